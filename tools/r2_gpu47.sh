export PATH=/usr/local/cuda/bin:$PATH
for sm in 1 0; do
  SKL_SMALL=$sm GRAPH=1 timeout 120 python tools/workload_ab.py c1 2>&1 | tail -1
done
