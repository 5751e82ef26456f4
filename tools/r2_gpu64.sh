# Round-2 closing evidence: GPU suite, compute-sanitizer on every kernel family (incl. the
# small-batch path), the bench launch list, the default bench line and the reference arm.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest64.txt 2>&1; tail -2 gpurun_out/gputest64.txt
rm -f gpurun_out/san_summary.txt gpurun_out/san_*.log
for tool in memcheck synccheck racecheck; do
  for c in 0 1 2 3 4 5 6 7; do
    timeout 400 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_case.py $c > gpurun_out/san_${tool}_$c.log 2>&1; echo "$tool case $c rc=$?" >> gpurun_out/san_summary.txt
  done
done
cat gpurun_out/san_summary.txt | tr '\n' ' '; echo
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sweep > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench64.json 2> gpurun_out/bench64.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench64_ref.json 2> gpurun_out/bench64_ref.err
tail -c 300 gpurun_out/bench64.json; tail -c 300 gpurun_out/bench64_ref.json
