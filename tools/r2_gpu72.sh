# --set full of the remaining c4 lines (bf16 L2 k32, L4 k64)
export PATH=/usr/local/cuda/bin:$PATH
ncu --set full --clock-control none -k regex:"b2b_kernel|dut|du_kernel" -c 4 -o gpurun_out/r2_c4k32 -f python tools/one_step.py "c4 bf16 4096 L2 k32" > gpurun_out/ncu72a.log 2>&1
ncu --set full --clock-control none -k regex:"b2b_kernel|dut|du_kernel" -c 3 -o gpurun_out/r2_c4k64 -f python tools/one_step.py "c4 bf16 4096 L4 k64" > gpurun_out/ncu72b.log 2>&1
ls -la gpurun_out/*.ncu-rep
