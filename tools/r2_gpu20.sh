export PATH=/usr/local/cuda/bin:$PATH
(
for sp in "" 1 2 3 4 5 6 7 8; do echo "== SKL_DU_SPLITS=$sp PDL off"; SKL_DU_VERBOSE=1 SKL_PDL=0 SKL_DU_SPLITS=$sp timeout 300 python tools/phased_ab.py du1:0 dxdu2:0 2>&1 | sort | uniq -c | sort -rn | head -6; done
for sp in "" 4 6 8 12 16 24; do echo "== CR=0 SKL_DU_SPLITS=$sp PDL off"; SKL_DU_CR=0 SKL_DU_VERBOSE=1 SKL_PDL=0 SKL_DU_SPLITS=$sp timeout 300 python tools/phased_ab.py du1:0 dxdu2:0 2>&1 | sort | uniq -c | sort -rn | head -6; done
) 2>&1 | tee gpurun_out/phased_ab4.txt
