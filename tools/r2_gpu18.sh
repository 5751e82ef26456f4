export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 300 python tools/phased_ab.py 2>&1 | tee gpurun_out/phased_ab2.txt
python - <<'PY'
import sys; sys.path.insert(0, '.')
import torch, paper_2601_15473_b200 as skl
PY
