export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err
T=131072 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"b2b_kernel|dut|du_kernel" --launch-skip 3 -c 4 -o gpurun_out/r2_c4k16_step python tools/layer_timing.py 4096 4096 1 16 > gpurun_out/ncu_c4step.log 2>&1
T=32768 SKL_DU_NOCOOP=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"b2b_kernel|du_kernel" --launch-skip 5 -c 3 -o gpurun_out/r2_proj_step python tools/layer_timing.py 768 768 1 128 > gpurun_out/ncu_projstep.log 2>&1
tail -2 gpurun_out/ncu_c4step.log gpurun_out/ncu_projstep.log
