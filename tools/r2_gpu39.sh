export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 300 python tools/kernel_table.py c5,c2,c4 > gpurun_out/kt39.json 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest39.txt 2>&1; tail -3 gpurun_out/gputest39.txt
timeout 900 python bench.py > gpurun_out/bench39.json 2> gpurun_out/bench39.err
tail -c 300 gpurun_out/bench39.json
