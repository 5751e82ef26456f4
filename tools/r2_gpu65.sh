export PATH=/usr/local/cuda/bin:$PATH
SKL_B2B_DT=2 timeout 300 python -m pytest tests/test_gpu.py tests/test_gpu_shapes.py -m gpu -x -q -k "(parity and (768-768-1-128 or 1023-1025)) or ragged_shapes" 2>&1 | tail -2
for rep in 1 2; do for dt in 2 1; do echo "== DT=$dt"; SKL_B2B_DT=$dt timeout 120 python tools/layer_timing.py 768 768 1 128 2>&1 | sed -n 1,3p; done; done
for rep in 1 2; do for dt in 2 1; do SKL_B2B_DT=$dt python tools/stack_ab.py 2>&1 | tail -1; done; done
