# TMA-stored saved columns: timelines, kernel table, A/B against SKL_SAVE_TMA=0, GPU suite.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for a in "768 768 1 128 32768 fwd" "768 768 1 128 32768 bwd" "768 3072 2 128 32768 bwd"; do
  echo "=== $a"; SKL_LIB=scratch/libskl.so timeout 120 python tools/trace_b2b.py $a
done > gpurun_out/trace27.txt 2>&1
timeout 300 python tools/kernel_table.py c5,c2 > gpurun_out/kt27.json 2>&1
SKL_SAVE_TMA=0 timeout 300 python tools/kernel_table.py c5,c2 > gpurun_out/kt27_off.json 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest27.txt 2>&1; tail -3 gpurun_out/gputest27.txt
