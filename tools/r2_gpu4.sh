mkdir -p gpurun_out
SKL_PARITY_LOG=$PWD/gpurun_out/parity_errors.jsonl timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -25 > gpurun_out/gpu_all.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
cat gpurun_out/gpu_all.log; tail -c 3000 gpurun_out/bench_r2a.json
