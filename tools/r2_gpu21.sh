export PATH=/usr/local/cuda/bin:$PATH
(
echo "== default, PDL on"; SKL_DU_VERBOSE=1 timeout 300 python tools/phased_ab.py fused:0 phased:0 phased:8 du1:0 dxdu2:0 2>&1 | sort | uniq -c | sort -rn | head -12
echo "== default, PDL off"; SKL_PDL=0 timeout 300 python tools/phased_ab.py fused:0 phased:0 phased:8 du1:0 dxdu2:0 du1:8 dxdu2:8
echo "== c5 proj layer"; timeout 300 python tools/layer_timing.py 768 768 1 128
) 2>&1 | tee gpurun_out/phased_ab5.txt
