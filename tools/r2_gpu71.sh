export PATH=/usr/local/cuda/bin:$PATH
for rep in 1 2; do for h in -1 3; do echo "== L2HINT=$h"; SKL_B2B_L2HINT=$h timeout 300 python tools/kernel_table.py c2,c5,c4 2>&1 | grep -E "^\{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  ', d['shape'][:24], d['step_us'])"; done; done
