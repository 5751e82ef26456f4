# DP-phased backward breakdown (c2), c5 stack per-kernel totals, c5/c3 kernel tables.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 300 python tools/phased_ab.py > gpurun_out/phased_ab.txt 2>&1
timeout 300 python tools/stack_profile.py > gpurun_out/stack_profile.txt 2>&1
timeout 300 python tools/kernel_table.py c5 > gpurun_out/ktab_c5.json 2>&1
timeout 300 python tools/kernel_table.py c3 > gpurun_out/ktab_c3.json 2>&1
cat gpurun_out/phased_ab.txt gpurun_out/stack_profile.txt
