"""FFN2-shaped backward (3072 -> 768, L2 k128, T = 32768) plain, with the fused x-mask
(SKL_FUSE_RELU_IN) and with the 1-bit mask: per-kernel device times (profile events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_15473_b200 as skl  # noqa: E402

d_in, d_out, L, k, T = 3072, 768, 2, 128, 32768
s = skl.shape(d_in, d_out, L, k, skl.BF16)
lyr = skl.SkLinear(d_in, d_out, L, k, seed=1, dtype=skl.BF16)
dev = torch.device("cuda", 0)
X = torch.randn(T, d_in, device=dev).bfloat16()
G = torch.randn(T, d_out, device=dev).bfloat16()
sv = torch.empty(L * k, T, dtype=torch.bfloat16, device=dev)
gx = torch.empty(T, d_in, dtype=torch.bfloat16, device=dev)
du1 = torch.empty(L, k, d_out, device=dev)
du2 = torch.empty(L, d_in, k, device=dev)
db = torch.empty(d_out, device=dev)
ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device=dev)
bits = torch.randint(-2**31, 2**31 - 1, (T, skl.relu_bits_row_words(d_in)), dtype=torch.int32, device=dev)
args = (s, G, X, sv, lyr.S1s, lyr.S2s, lyr.U1s, lyr.U2s, gx, du1, du2, db, ws)
skl.forward(s, X, lyr.S1s, lyr.S2s, lyr.U1s, lyr.U2s, lyr.bias, torch.empty(T, d_out, dtype=torch.bfloat16, device=dev), sv, ws)
variants = {
    "plain": lambda: skl.backward_phase(*args[:1], skl.BWD_ALL, *args[1:]),
    "xmask": lambda: skl.backward_phase(*args[:1], skl.BWD_ALL, *args[1:], fuse=skl.FUSE_RELU_IN),
    "bits": lambda: skl.backward_phase(*args[:1], skl.BWD_ALL, *args[1:], fuse=skl.FUSE_RELU_IN, relu_bits=bits),
}
for name, fn in variants.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    skl.profile_enable(True)
    skl.profile_collect()
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    prof = skl.profile_collect()
    skl.profile_enable(False)
    print(name, {kk: round(t / n * 1e3, 1) for kk, (n, t) in prof.items()})
