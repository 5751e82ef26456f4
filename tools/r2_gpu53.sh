export PATH=/usr/local/cuda/bin:$PATH
bash tools/ab_lib.sh scratch/ab/pkg/libskl.so paper_2601_15473_b200/libskl.so "python tools/kernel_table.py c4" 2
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_shapes.py -m gpu -x -q -k "parity or ragged or chain" 2>&1 | tail -2
