# One fwd+bwd step of a bench.SWEEP workload (for ncu captures).
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_15473_b200 as skl
import bench
name = sys.argv[1]
cases = bench.SWEEP + [("c2 bf16", 768, 3072, 2, 128, 32768, "bf16")]
c = [c for c in cases if name in c[0]][0]
bench.measure_workload(skl, torch, torch.device("cuda", 0), *c, steps=1, warmup=1)
torch.cuda.synchronize()
print("done", c[0])
