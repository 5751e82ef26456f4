export PATH=/usr/local/cuda/bin:$PATH
for rep in 1 2 3; do for dt in 1 0; do echo "== DT=$dt"; SKL_B2B_DT=$dt timeout 120 python tools/layer_timing.py 768 768 1 128 2>&1 | sed -n 2,3p; done; done
for rep in 1 2; do for dt in 1 0; do SKL_B2B_DT=$dt python tools/stack_ab.py 2>&1 | tail -1; done; done
