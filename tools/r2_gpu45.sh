export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
DT=tf32 ncu --set full --import-source on -k regex:"proj_part|reduce_rank|out_gemm|grads_small" -c 4 -o gpurun_out/small -f python tools/one_step.py "c1 fp32" > gpurun_out/ncu45.log 2>&1
ncu -i gpurun_out/small.ncu-rep --page details 2>&1 | grep -E "^  [a-z_]+.*\(|Duration|Elapsed Cycles|SM Frequency|Registers|Achieved Occupancy|Block Limit|Waves Per SM|Theoretical Occupancy" | head -60
