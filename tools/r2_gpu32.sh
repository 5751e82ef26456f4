export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
SKL_LIB=scratch/libskl.so timeout 120 python tools/trace_b2b.py 768 768 1 128 32768 fwd > gpurun_out/trace32.txt 2>&1
grep -A3 "slot 0" gpurun_out/trace32.txt | grep "role [12]" | cut -c1-900
timeout 300 python tools/kernel_table.py c5,c2,c4 > gpurun_out/kt32.json 2>&1
timeout 900 python -m pytest tests/test_gpu.py -m gpu -x -q > gpurun_out/gputest32.txt 2>&1; tail -3 gpurun_out/gputest32.txt
