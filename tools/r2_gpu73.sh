# --set full of the c4 TF32 lines (L1 k16, L2 k64)
export PATH=/usr/local/cuda/bin:$PATH
ncu --set full --clock-control none -k regex:"b2b|dut|du_kernel|pack" -c 5 -o gpurun_out/r2_c4tf32k16 -f python tools/one_step.py "c4 TF32 4096 L1 k16" > gpurun_out/ncu73a.log 2>&1
ncu --set full --clock-control none -k regex:"b2b|dut|du_kernel|pack" -c 5 -o gpurun_out/r2_c4tf32k64 -f python tools/one_step.py "c4 TF32 4096 L2 k64" > gpurun_out/ncu73b.log 2>&1
ls -la gpurun_out/*.ncu-rep
