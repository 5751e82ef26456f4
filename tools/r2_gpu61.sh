export PATH=/usr/local/cuda/bin:$PATH
timeout 300 python -m pytest tests/test_gpu.py -m gpu -x -q -k "parity and 768-768-1-128" 2>&1 | tail -2
for rep in 1 2; do for il in 1 0; do echo "== IL=$il"; SKL_B2B_IL=$il timeout 120 python tools/layer_timing.py 768 768 1 128 2>&1 | sed -n 1,3p; done; done
