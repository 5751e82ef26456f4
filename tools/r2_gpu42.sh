# Round-2 evidence (part 2): --set full of the c3 step (unfused tcgen05 GEMM chain) and of the
# c4 L1 k16 step (packed-panel b2b + dut); c1 per-kernel timing.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel" -c 4 -o gpurun_out/r2_c3 -f python tools/one_step.py "c3 bf16" > gpurun_out/ncu42a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"b2b_kernel|dut" -c 4 -o gpurun_out/r2_c4k16 -f python tools/one_step.py "c4 bf16 4096 L1 k16" > gpurun_out/ncu42b.log 2>&1
DT=tf32 T=64 timeout 120 python tools/layer_timing.py 1024 1024 1 64 > gpurun_out/c1_timing.txt 2>&1
ls -la gpurun_out/*.ncu-rep; cat gpurun_out/c1_timing.txt
