# Round-2 re-entry: GPU parity suite + smoke, then the final evidence script.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?"
bash tools/r2_gpu15.sh
