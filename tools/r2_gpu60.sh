export PATH=/usr/local/cuda/bin:$PATH
for rep in 1 2; do GRAPH=1 timeout 120 python tools/workload_ab.py c1 2>&1 | tail -1; SKL_PDL=0 GRAPH=1 timeout 120 python tools/workload_ab.py c1 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_shapes.py tests/test_model_io.py -m gpu -x -q -k "small or c1 or ragged or gradcheck or identity or model or (parity and (-64] or -50] or -77]))" 2>&1 | tail -2
