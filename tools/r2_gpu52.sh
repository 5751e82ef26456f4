export PATH=/usr/local/cuda/bin:$PATH
python tools/conv_timing.py; python tools/conv_timing.py 32 256 256 14 14 3 1 1 1 64; python tools/conv_timing.py 8 3 64 224 224 7 2 3 1 32
timeout 900 python -m pytest tests -m gpu -x -q -k "conv" 2>&1 | tail -3
