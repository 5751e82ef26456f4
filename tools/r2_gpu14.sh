timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_shapes.py -x -q -m gpu -k "parity or chain or bert or graph or deterministic or ragged" 2>&1 | tail -3
python tools/workload_ab.py "c2 bf16" | tail -1
python tools/stack_time.py | tail -1
T=32768 python tools/layer_timing.py 768 768 1 128 2>&1 | grep -E "^step"
