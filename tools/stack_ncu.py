"""The c5 stack (bench.measure_stack's chain) for an ncu launch list: `count`
prints libskl launches per step; otherwise runs `steps` eager steps (the
caller skips the warm-up ones with ncu --launch-skip)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_15473_b200 as skl  # noqa: E402
from paper_2601_15473_b200.model import bert_ffn_stack  # noqa: E402

dev = torch.device("cuda", 0)
chain = bert_ffn_stack(num_layers=12, device=dev)
T = 32768
x = torch.randn(T, 768, device=dev).to(torch.bfloat16)
g = torch.randn(T, 768, device=dev).to(torch.bfloat16)
buckets = chain.allocate_grads(dev)


def step():
    chain.forward(x)
    chain.backward(g, buckets=buckets, need_grad_x=False, overlap=False)


if sys.argv[1] == "count":
    step()
    torch.cuda.synchronize()
    n0 = skl.launch_count()
    step()
    torch.cuda.synchronize()
    print(skl.launch_count() - n0)
else:
    for _ in range(int(sys.argv[1])):
        step()
    torch.cuda.synchronize()
