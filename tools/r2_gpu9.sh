timeout 900 python -m pytest tests/test_gpu.py -x -q -m gpu -k "parity_bf16 or parity_tf32 or deterministic" 2>&1 | tail -3
for env in "" "SKL_DUT=1" "SKL_DUT=0"; do
  echo "== $env"; env $env T=32768 python tools/layer_timing.py 768 768 1 128 2>&1 | grep -E "^step"
  env $env T=131072 python tools/layer_timing.py 4096 4096 1 16 2>&1 | grep -E "^step"
  env $env T=131072 python tools/layer_timing.py 4096 4096 2 32 2>&1 | grep -E "^step"
  env $env T=131072 DT=tf32 python tools/layer_timing.py 4096 4096 2 64 2>&1 | grep -E "^step"
  env $env T=131072 DT=tf32 python tools/layer_timing.py 4096 4096 1 16 2>&1 | grep -E "^step"
done
