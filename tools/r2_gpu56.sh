export PATH=/usr/local/cuda/bin:$PATH
for mb in 0 48 32 64; do
  echo "== SKL_CHAIN_L2_MB=$mb"; SKL_CHAIN_L2_MB=$mb timeout 300 python tools/workload_ab.py c3 2>&1 | tail -1
done
SKL_CHAIN_L2_MB=48 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:gemm_kernel --launch-skip 40 -c 20 python tools/one_step.py "c3 bf16" 2>&1 | grep -E "gemm_kernel|dram__bytes|duration" | head -60 > gpurun_out/c3_chain_ncu.txt
SKL_CHAIN_L2_MB=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:gemm_kernel --launch-skip 8 -c 4 python tools/one_step.py "c3 bf16" 2>&1 | grep -E "gemm_kernel|dram__bytes|duration" | head -30 > gpurun_out/c3_chain_ncu0.txt
timeout 900 python -m pytest tests/test_gpu.py -m gpu -x -q -k "parity and (4096-4096-3-256 or 2048-1024-4-256 or 512-768-3 or 1024-1536)" 2>&1 | tail -2
