export PATH=/usr/local/cuda/bin:$PATH
SKL_B2B_MC=1 timeout 120 python tools/dbg_bwd.py 768 768 1 128 600 > /dev/null 2>&1; echo "smoke rc=$?"
SKL_B2B_MC=1 timeout 300 python -m pytest tests/test_gpu.py -m gpu -x -q -k "forward_parity_bf16" 2>&1 | tail -2
for rep in 1 2; do for mc in 1 0; do echo "== MC=$mc"; SKL_B2B_MC=$mc timeout 120 python tools/layer_timing.py 768 768 1 128 2>&1 | sed -n 1p; SKL_B2B_MC=$mc timeout 120 python tools/layer_timing.py 768 3072 2 128 2>&1 | sed -n 1p; done; done
