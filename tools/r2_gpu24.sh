# c5 breakdown: per-shape kernel table and the stack's per-kernel totals.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 300 python tools/kernel_table.py c5,c2 > gpurun_out/kt24.json 2>&1
timeout 300 python tools/stack_profile.py > gpurun_out/stack24.txt 2>&1
cat gpurun_out/stack24.txt
