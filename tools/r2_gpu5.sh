export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
python tools/workload_ab.py c3 2>&1 | tail -1
SKL_B2B_RSPLIT=0 python tools/workload_ab.py c3 2>&1 | tail -1
python tools/workload_ab.py "c2 bf16" 2>&1 | tail -1
ncu --set full --clock-control none --import-source on -k regex:"b2b_kernel" -c 2 -o gpurun_out/r2_c3_rsplit python tools/one_step.py c3 > gpurun_out/ncu_c3.log 2>&1
tail -2 gpurun_out/ncu_c3.log
