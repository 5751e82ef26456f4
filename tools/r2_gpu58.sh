export PATH=/usr/local/cuda/bin:$PATH
for rep in 1 2; do
python tools/stack_ab.py 2>&1 | tail -1
SKL_B2B_L2HINT=0 python tools/stack_ab.py 2>&1 | tail -1
SKL_B2B_L2HINT=3 python tools/stack_ab.py 2>&1 | tail -1
SKL_DU_L2HINT=0 python tools/stack_ab.py 2>&1 | tail -1
SKL_DU_L2HINT=3 python tools/stack_ab.py 2>&1 | tail -1
done
