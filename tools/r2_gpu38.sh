export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
SKL_DUT=1 timeout 300 python tools/kernel_table.py c5,c4 > gpurun_out/kt38_dut.json 2>&1
SKL_DUT=1 timeout 900 python -m pytest tests/test_gpu.py -m gpu -x -q -k "backward or chain" > gpurun_out/gputest38.txt 2>&1; tail -3 gpurun_out/gputest38.txt
