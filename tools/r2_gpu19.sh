export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
(
echo "== PDL off"; SKL_PDL=0 timeout 300 python tools/phased_ab.py fused:0 phased:0 phased:8 du1:0 dxdu2:0 du1:8 dxdu2:8
for sp in 2 3 4 6 8; do echo "== SKL_DU_SPLITS=$sp PDL off"; SKL_PDL=0 SKL_DU_SPLITS=$sp timeout 300 python tools/phased_ab.py du1:0 dxdu2:0; done
echo "== SKL_DU_CR=0 PDL off"; SKL_PDL=0 SKL_DU_CR=0 timeout 300 python tools/phased_ab.py du1:0 dxdu2:0
) 2>&1 | tee gpurun_out/phased_ab3.txt
