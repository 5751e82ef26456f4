export PATH=/usr/local/cuda/bin:$PATH
(
for rep in 1 2; do
echo "== default"; SKL_PDL=0 timeout 300 python tools/phased_ab.py dxdu2:0 fused:0 phased:0
echo "== SPLITS=''"; SKL_DU_SPLITS= SKL_PDL=0 timeout 300 python tools/phased_ab.py dxdu2:0 fused:0 phased:0
echo "== DEEP_CR=0"; SKL_DU_DEEP_CR=0 SKL_PDL=0 timeout 300 python tools/phased_ab.py dxdu2:0 fused:0 phased:0
done
) 2>&1 | tee gpurun_out/phased_ab6.txt
