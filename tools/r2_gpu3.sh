mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
N=$(python tools/stack_ncu.py count | tail -1)
echo "launches per step: $N" > gpurun_out/stack_ncu.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"b2b_kernel|du_kernel|gemm_kernel|pack_tiles|repad|convert|transpose" --launch-skip $((2*N)) --launch-count $N --csv --log-file gpurun_out/stack_launches.csv python tools/stack_ncu.py 3 >> gpurun_out/stack_ncu.log 2>&1
python tools/layer_timing.py 768 768 1 128 > gpurun_out/proj_timing.log 2>&1
