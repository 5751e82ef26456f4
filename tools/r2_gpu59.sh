export PATH=/usr/local/cuda/bin:$PATH
for rep in 1 2; do
for sp in -1 1; do echo "== SKL_FWD_SP=$sp"; SKL_FWD_SP=$sp timeout 300 python tools/kernel_table.py c2 2>&1 | grep "c2 bf16"; done
done
