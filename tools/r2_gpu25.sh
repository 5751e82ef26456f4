# ncu --set full with source of the c5 projection layer (fwd, bwd, du): where each warp role waits.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"b2b_kernel|du_kernel" --launch-skip 3 -c 3 -o gpurun_out/r2_proj_src python tools/one_step.py 768 768 1 128 > gpurun_out/ncu25.log 2>&1
tail -3 gpurun_out/ncu25.log
