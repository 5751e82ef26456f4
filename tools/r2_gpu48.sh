export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:"out_gemm|reduce_rank|proj_part" --launch-skip 6 -c 3 -o gpurun_out/small2 -f python tools/one_step.py "c1 fp32" > gpurun_out/ncu48.log 2>&1
ncu -i gpurun_out/small2.ncu-rep --page details 2>&1 | grep -E "^  [a-z_ ]+.*\(|Duration|Elapsed Cycles|SM Frequency|L2 Hit|DRAM Throughput|One or More|No Eligible|Issue Slots" | head -40
