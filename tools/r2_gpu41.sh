# Round-2 evidence (part 1) after the TMA saves / per-warp stores / du tail changes: launch list of
# the bench command, --set full captures of the c2 step, the c2-TF32 step (b2b_tf32 wide kernel)
# and the 768x768 projection step.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sweep > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"b2b_kernel|du_kernel" -c 3 -o gpurun_out/r2_c2_full -f python tools/one_step.py "c2 bf16" > gpurun_out/ncu41a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"b2b|du_kernel|pack" -c 4 -o gpurun_out/r2_c2tf32 -f python tools/one_step.py "c2 TF32" > gpurun_out/ncu41b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"b2b_kernel|du_kernel" -c 3 -o gpurun_out/r2_proj -f python tools/one_step.py 768 768 1 128 > gpurun_out/ncu41c.log 2>&1
ls -la gpurun_out/*.ncu-rep
