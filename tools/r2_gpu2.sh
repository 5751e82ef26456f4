mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
T=32768 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"b2b|du_kernel" -c 3 -o gpurun_out/r2_proj python tools/layer_timing.py 768 768 1 128 > gpurun_out/ncu_proj.log 2>&1
T=131072 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"b2b|du_kernel" -c 3 -o gpurun_out/r2_c4k16 python tools/layer_timing.py 4096 4096 1 16 > gpurun_out/ncu_c4.log 2>&1
for tool in memcheck synccheck racecheck; do
  for c in 0 1 2 3 4 5; do
    timeout 400 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_case.py $c > gpurun_out/san_${tool}_$c.log 2>&1; echo "$tool case $c rc=$?" >> gpurun_out/san_summary.txt
  done
done
cat gpurun_out/san_summary.txt
tail -3 gpurun_out/ncu_proj.log gpurun_out/ncu_c4.log
