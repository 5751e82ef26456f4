export PATH=/usr/local/cuda/bin:$PATH
SKL_CHAIN_L2_MB=64 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:gemm_kernel -c 40 python tools/one_step.py "c3 bf16" > gpurun_out/c3_chain_ncu.txt 2>&1
SKL_CHAIN_L2_MB=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:gemm_kernel -c 10 python tools/one_step.py "c3 bf16" > gpurun_out/c3_chain_ncu0.txt 2>&1
grep -c gemm_kernel gpurun_out/c3_chain_ncu.txt
