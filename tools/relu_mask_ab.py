# FFN2-shaped backward (3072 -> 768, L2 k128, T=32768): no mask vs x-mask vs 1-bit mask
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_15473_b200 as skl
dev = torch.device("cuda", 0)
d_in, d_out, l, k, T = 3072, 768, 2, 128, 32768
s = skl.shape(d_in, d_out, l, k, skl.BF16)
td = torch.bfloat16
S1s = torch.empty(l, d_in, k, dtype=td, device=dev); S2s = torch.empty(l, k, d_out, dtype=td, device=dev)
U1s = torch.empty(l, k, d_out, dtype=td, device=dev); U2s = torch.empty(l, d_in, k, dtype=td, device=dev)
skl.generate_sketches(s, 0, 1, S1s, S2s); skl.init_params(s, 1, U1s, U2s)
X = torch.relu(torch.randn(T, d_in, device=dev)).to(td); G = torch.randn(T, d_out, device=dev).to(td)
GX = torch.empty(T, d_in, dtype=td, device=dev)
sv = torch.empty(l * k, T, dtype=td, device=dev)
du1 = torch.empty(l * k * d_out, device=dev); du2 = torch.empty(l * k * d_in, device=dev); db = torch.empty(d_out, device=dev)
ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device=dev)
W = skl.relu_bits_row_words(d_in)
bits = torch.randint(0, 2**31 - 1, (T, W), dtype=torch.int32, device=dev)
skl.forward(s, X, S1s, S2s, U1s, U2s, None, torch.empty(T, d_out, dtype=td, device=dev), sv, ws)
cases = {"none": dict(fuse=0), "xmask": dict(fuse=skl.FUSE_RELU_IN), "bits": dict(fuse=skl.FUSE_RELU_IN, relu_bits=bits)}
for name, kw in cases.items():
    fn = lambda: skl.backward_phase(s, skl.BWD_DX_DU2, G, X, sv, S1s, S2s, U1s, U2s, GX, None, du2, None, ws, **kw)
    for _ in range(5): fn()
    torch.cuda.synchronize()
    skl.profile_enable(True); skl.profile_collect()
    for _ in range(20): fn()
    torch.cuda.synchronize()
    prof = skl.profile_collect(); skl.profile_enable(False)
    print(name, {kk: round(t / n * 1e3, 1) for kk, (n, t) in prof.items()})
