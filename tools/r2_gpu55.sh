export PATH=/usr/local/cuda/bin:$PATH
for sp in "" 4 5 6 7 8; do
  echo "== SKL_DU_SPLITS=$sp"; SKL_DU_CR_MAX=8 SKL_DU_SPLITS=$sp T=32768 timeout 120 python tools/layer_timing.py 768 768 1 128 2>&1 | sed -n 2,3p
done
