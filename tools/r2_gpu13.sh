timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_shapes.py -x -q -m gpu -k "chain or bert or graph or dp" 2>&1 | tail -2
python tools/stack_time.py | tail -1
SKL_PDL=0 python tools/stack_time.py | tail -1
