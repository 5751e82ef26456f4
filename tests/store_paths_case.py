"""Helper for test_gpu.py::test_store_and_tile_variants_are_bitwise_identical: one
forward + backward of a 768x768 L1 k128 layer (and a c2-shaped one) under the SKL_*
switches of the calling process, outputs written to the .pt file given."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_15473_b200 as skl  # noqa: E402

out = {}
for (d_in, d_out, L, k, T) in ((768, 768, 1, 128, 1300), (768, 3072, 2, 128, 700)):
    lyr = skl.SkLinear(d_in, d_out, L, k, seed=9, dtype=skl.BF16)
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    with torch.no_grad():
        lyr.bias.copy_((torch.randn(d_out, device="cuda", generator=g) * 0.1).to(torch.bfloat16))
    X = torch.randn(T, d_in, device="cuda", generator=g).to(torch.bfloat16)
    G = torch.randn(T, d_out, device="cuda", generator=g).to(torch.bfloat16)
    sv = torch.empty(L * k, (T + 7) // 8 * 8, dtype=torch.bfloat16, device="cuda")
    y = lyr.forward(X, saved=sv)
    gr = lyr.backward(X, G, saved=sv)
    torch.cuda.synchronize()
    key = f"{d_in}x{d_out}"
    out[key] = {"y": y.cpu(), "saved": sv[:, :T].cpu(), "gx": gr.grad_x.cpu(), "du1": gr.grad_u1.cpu(),
                "du2": gr.grad_u2.cpu(), "db": gr.grad_b.cpu()}
torch.save(out, sys.argv[1])
