import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_15473_b200 as skl
from paper_2601_15473_b200.model import bert_ffn_stack, wait_all
dev = torch.device("cuda", 0)
chain = bert_ffn_stack(num_layers=12, device=dev)
T = 32768
x = torch.randn(T, 768, device=dev).to(torch.bfloat16)
g = torch.randn(T, 768, device=dev).to(torch.bfloat16)
buckets = chain.allocate_grads(dev)
def step():
    chain.forward(x)
    chain.backward(g, buckets=buckets, need_grad_x=False, overlap=False)
for _ in range(2): step()
torch.cuda.synchronize()
t0 = time.perf_counter(); step(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print("host enqueue %.2f ms, total %.2f ms" % ((t1 - t0) * 1e3, (t2 - t0) * 1e3))
skl.profile_enable(True); skl.profile_collect()
step(); torch.cuda.synchronize()
prof = skl.profile_collect(); skl.profile_enable(False)
tot = sum(t for _, t in prof.values())
for k, (n, t) in prof.items(): print(f"{k:12s} x{n:4d} {t:8.3f} ms  {t/n*1e3:8.1f} us/launch  {t/tot*100:5.1f}%")
# per layer type breakdown
