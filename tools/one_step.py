# One fwd+bwd step of a bench.SWEEP workload, or of an explicit shape "d_in d_out L k [T]" (for ncu captures).
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_15473_b200 as skl
import bench
if len(sys.argv) >= 5:
    d_in, d_out, L, k = (int(v) for v in sys.argv[1:5])
    T = int(sys.argv[5]) if len(sys.argv) > 5 else 32768
    c = (f"{d_in}x{d_out} L{L} k{k} T{T}", d_in, d_out, L, k, T, os.environ.get("DT", "bf16"))
else:
    cases = bench.SWEEP + [("c2 bf16", 768, 3072, 2, 128, 32768, "bf16")]
    c = [c for c in cases if sys.argv[1] in c[0]][0]
bench.measure_workload(skl, torch, torch.device("cuda", 0), *c, steps=1, warmup=1)
torch.cuda.synchronize()
print("done", c[0])
