export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for sh in "768 3072 2 128 300" "768 768 1 128 600" "768 3072 2 128 32768"; do
SKL_B2B_WSTORE=1 python tools/dbg_bwd.py $sh; SKL_B2B_WSTORE=0 python tools/dbg_bwd.py $sh
python - <<'PY'
import torch
a=torch.load('/tmp/gx_1.pt').float(); b=torch.load('/tmp/gx_0.pt').float()
d=(a-b).abs()
print("max diff", d.max().item(), (d>0).sum().item())
PY
done
timeout 300 python tools/kernel_table.py c5,c2,c4 > gpurun_out/kt33.json 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest33.txt 2>&1; tail -3 gpurun_out/gputest33.txt
