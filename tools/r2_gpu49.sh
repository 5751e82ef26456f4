export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 300 python tools/kernel_table.py c5,c2,c4 > gpurun_out/kt49.json 2>&1
timeout 900 python -m pytest tests/test_gpu.py -m gpu -x -q > gpurun_out/gputest49.txt 2>&1; tail -3 gpurun_out/gputest49.txt
