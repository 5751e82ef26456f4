export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest50.txt 2>&1; tail -3 gpurun_out/gputest50.txt
for i in 1 2; do timeout 300 python tools/kernel_table.py c2 2>&1 | grep c2; done
