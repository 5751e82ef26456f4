export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
DT=tf32 T=64 timeout 120 python tools/layer_timing.py 1024 1024 1 64 2>&1 | head -3
timeout 900 python -m pytest tests/test_gpu.py -m gpu -x -q -k "small or c1 or parity" > gpurun_out/gputest43.txt 2>&1; tail -3 gpurun_out/gputest43.txt
