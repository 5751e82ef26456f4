export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest67.txt 2>&1; tail -2 gpurun_out/gputest67.txt
timeout 300 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_case.py 0 > gpurun_out/san67_mem.log 2>&1; echo "memcheck c2 rc=$?"
timeout 300 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_case.py 0 > gpurun_out/san67_sync.log 2>&1; echo "synccheck c2 rc=$?"
for rep in 1 2; do for mc in 1 0; do echo "== MC=$mc"; SKL_B2B_MC=$mc timeout 300 python tools/kernel_table.py c2 2>&1 | grep "c2 bf16"; done; done
