export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for a in "768 768 1 128 32768 bwd"; do
  echo "=== $a SKL_DUT=1"; SKL_DUT=1 SLOTS=0,2,4,6 SKL_LIB=scratch/libskl.so timeout 120 python tools/trace_b2b.py $a
done > gpurun_out/trace37.txt 2>&1
cut -c1-400 gpurun_out/trace37.txt
