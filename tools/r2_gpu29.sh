export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for a in "768 768 1 128 32768 fwd" "768 3072 2 128 32768 bwd" "768 3072 2 128 32768 fwd"; do
  echo "=== $a"; SKL_LIB=scratch/libskl.so timeout 120 python tools/trace_b2b.py $a
done > gpurun_out/trace29.txt 2>&1
grep -A3 "slot 0" gpurun_out/trace29.txt | grep "role 2" | cut -c1-500
timeout 300 python tools/kernel_table.py c5,c2 > gpurun_out/kt29.json 2>&1
timeout 900 python -m pytest tests/test_gpu.py -m gpu -x -q > gpurun_out/gputest29.txt 2>&1; tail -3 gpurun_out/gputest29.txt
