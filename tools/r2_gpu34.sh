export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for a in "768 768 1 128 32768 bwd" "768 3072 2 128 32768 bwd"; do
  echo "=== $a"; SLOTS=4,6 SKL_LIB=scratch/libskl.so timeout 120 python tools/trace_b2b.py $a
done > gpurun_out/trace34.txt 2>&1
cut -c1-1500 gpurun_out/trace34.txt
