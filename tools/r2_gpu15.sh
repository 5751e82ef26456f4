# Final round-2 evidence: launch list of the bench command, --set full of the c2 step and of the
# small-rank dut kernel, then the bench line (N=1, with CPU baseline) and the reference arm.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sweep > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"b2b_kernel|du_kernel" -c 3 -o gpurun_out/r2_c2_full python tools/one_step.py "c2 bf16" > gpurun_out/ncu_c2.log 2>&1
T=131072 ncu --set full --clock-control none --import-source on -k regex:"dut" -c 2 -o gpurun_out/r2_c4k16_dut python tools/layer_timing.py 4096 4096 1 16 > gpurun_out/ncu_dut.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r2_final.json 2> gpurun_out/bench_r2_final.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_r2_ref.json 2> gpurun_out/bench_r2_ref.err
tail -c 600 gpurun_out/bench_r2_final.json; tail -c 400 gpurun_out/bench_r2_ref.json
