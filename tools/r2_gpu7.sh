# du split A/B on the c5 projection layer (768x768, L1 k128, T=32768) and FFN shapes
for env in "" "SKL_DU_SPLITS=4" "SKL_DU_SPLITS=6" "SKL_DU_SPLITS=8 SKL_DU_CR_MAX=8" "SKL_DU_SPLITS=12 SKL_DU_CR_MAX=8" "SKL_DU_CR=0"; do
  echo "== $env"; env $env T=32768 python tools/layer_timing.py 768 768 1 128 2>&1 | grep -E "^bwd batch|^step"
done
for env in "" "SKL_DU_SPLITS=2" "SKL_DU_SPLITS=3"; do
  echo "== FFN1 $env"; env $env T=32768 python tools/layer_timing.py 768 3072 2 128 2>&1 | grep -E "^bwd batch|^step"
done
