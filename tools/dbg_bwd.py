import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2601_15473_b200 as skl
d_in, d_out, L, k, T = [int(v) for v in sys.argv[1:6]]
lyr = skl.SkLinear(d_in, d_out, L, k, seed=3, dtype=skl.BF16)
torch.manual_seed(0)
X = torch.randn(T, d_in, device="cuda").bfloat16(); G = torch.randn(T, d_out, device="cuda").bfloat16()
sv = torch.empty(L * k, (T + 7) // 8 * 8, dtype=torch.bfloat16, device="cuda")
lyr.forward(X, saved=sv)
g = lyr.backward(X, G, saved=sv)
torch.cuda.synchronize()
torch.save(g.grad_x.cpu(), f"/tmp/gx_{os.environ.get('SKL_B2B_WSTORE','1')}.pt")
