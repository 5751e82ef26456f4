export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
DT=tf32 T=64 timeout 120 python tools/layer_timing.py 1024 1024 1 64 2>&1 | head -3
T=64 timeout 120 python tools/layer_timing.py 1024 1024 1 64 2>&1 | head -3
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_shapes.py -m gpu -x -q -k "small or c1 or ragged or gradcheck or identity or (parity and (-64] or -50] or -77]))" > gpurun_out/gputest46.txt 2>&1; tail -3 gpurun_out/gputest46.txt
