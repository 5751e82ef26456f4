export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
DT=tf32 T=64 timeout 120 python tools/layer_timing.py 1024 1024 1 64 2>&1 | head -3
T=64 timeout 120 python tools/layer_timing.py 1024 1024 1 64 2>&1 | head -3
SKL_SMALL=0 DT=tf32 T=64 timeout 120 python tools/layer_timing.py 1024 1024 1 64 2>&1 | head -3
timeout 2000 python -m pytest tests -m gpu -x -q > gpurun_out/gputest44.txt 2>&1; tail -3 gpurun_out/gputest44.txt
