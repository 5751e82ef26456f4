export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for pf in 0 12 24; do
  echo "== PF $pf"; SKL_B2B_PF=$pf timeout 300 python tools/kernel_table.py c5,c2,c4 > gpurun_out/kt31_$pf.json 2>&1
done
SKL_LIB=scratch/libskl.so timeout 120 python tools/trace_b2b.py 768 768 1 128 32768 fwd > gpurun_out/trace31.txt 2>&1
grep -A3 "slot 0" gpurun_out/trace31.txt | grep "role 1" | cut -c1-700
