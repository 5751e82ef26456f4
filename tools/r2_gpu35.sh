export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for a in "768 768 1 128 32768 bwd"; do
  echo "=== $a SKL_DUT=1"; SKL_DUT=1 SLOTS=4,6 SKL_LIB=scratch/libskl.so timeout 120 python tools/trace_b2b.py $a
done > gpurun_out/trace35.txt 2>&1
for a in "4096 4096 1 16 131072 bwd"; do
  echo "=== $a"; SLOTS=4,6 SKL_LIB=scratch/libskl.so timeout 120 python tools/trace_b2b.py $a
done >> gpurun_out/trace35.txt 2>&1
SKL_DUT=1 T=32768 timeout 120 python tools/layer_timing.py 768 768 1 128 | head -3 >> gpurun_out/trace35.txt 2>&1
cut -c1-1200 gpurun_out/trace35.txt
