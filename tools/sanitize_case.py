"""Small fwd+bwd launches of every fused kernel family for compute-sanitizer
(memcheck / synccheck / racecheck): bf16 c2-shaped (b2b fwd/bwd + du with the
cluster reduction), a ragged shape (padded dispatch), the TF32 wide-rank kernel
(R = 512), the unfused chain (R = 1536), the 768x768 projection (du deep-split
cluster reduction), the small-batch path (T <= 128) and a DenseLinear layer.  Exits non-zero on an error status."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_15473_b200 as skl  # noqa: E402

CASES = [(768, 3072, 2, 128, 600, skl.BF16), (6, 8, 2, 3, 300, skl.BF16), (768, 3072, 2, 128, 300, skl.F32_TF32),
         (512, 512, 3, 256, 300, skl.BF16), (768, 768, 1, 128, 2048, skl.BF16),
         # small-batch path (small.cu): the c1 shape in TF32, a ragged bf16 layer through the padded dispatch
         (1024, 1024, 1, 64, 64, skl.F32_TF32), (30, 70, 2, 12, 97, skl.BF16)]
which = sys.argv[1:] or [str(i) for i in range(len(CASES) + 1)]
for i, (d_in, d_out, L, k, T, dt) in enumerate(CASES):
    if str(i) not in which:
        continue
    td = skl.torch_dtype(dt)
    lyr = skl.SkLinear(d_in, d_out, L, k, seed=3, dtype=dt)
    X = torch.randn(T, d_in, device="cuda").to(td)
    G = torch.randn(T, d_out, device="cuda").to(td)
    sv = torch.empty(L * k, (T + 7) // 8 * 8, dtype=td, device="cuda")
    lyr.forward(X, saved=sv)
    lyr.backward(X, G, saved=sv)
    torch.cuda.synchronize()
    print("case", i, (d_in, d_out, L, k, T, "bf16" if dt == skl.BF16 else "tf32"), "ok", flush=True)
if str(len(CASES)) in which:
    dn = skl.DenseLinear(200, 136, seed=1)
    X = torch.randn(300, 200, device="cuda").to(torch.bfloat16)
    dn.backward(X, dn.forward(X))
    torch.cuda.synchronize()
    print("case dense ok", flush=True)
