export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for a in "768 768 1 128 32768 fwd"; do
  echo "=== $a"; SKL_LIB=scratch/libskl.so timeout 120 python tools/trace_b2b.py $a
done > gpurun_out/trace30.txt 2>&1
grep -A3 "slot 0" gpurun_out/trace30.txt | grep "role [23]" | cut -c1-1200
