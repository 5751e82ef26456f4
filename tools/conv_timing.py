"""SkConv2d fwd+bwd on the device (explicit im2col lowering onto the SKLinear
path): per-kernel device times and the traffic the lowering adds.

    python tools/conv_timing.py [B C_in C_out H W k_h stride pad L k]   (default: a ResNet-50 3x3 stage-1 conv)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_15473_b200 as skl  # noqa: E402
from paper_2601_15473_b200.conv import ConvShape, SkConv2d  # noqa: E402

a = [int(v) for v in sys.argv[1:]] or [32, 64, 64, 56, 56, 3, 1, 1, 1, 64]
B, C, CO, H, W, KH, ST, PD, L, K = a
cs = ConvShape(C, CO, KH, KH, ST, PD)
conv = SkConv2d(cs, L, K, seed=1)
x = torch.randn(B, C, H, W, device="cuda").bfloat16()
oh, ow = cs.out_h(H), cs.out_w(W)
g = torch.randn(B, CO, oh, ow, device="cuda").bfloat16()


def step():
    keep = {}
    conv.forward(x, keep=keep)
    conv.backward(x, g, keep=keep)


for _ in range(3):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
skl.profile_enable(True)
skl.profile_collect()
for _ in range(5):
    step()
torch.cuda.synchronize()
prof = skl.profile_collect()
T, d_in = B * oh * ow, C * KH * KH
img = (B * C * H * W + B * CO * oh * ow) * 2          # NCHW input + output (or grad) per pass
patches = T * d_in * 2                                 # the lowered patch matrix
print(json.dumps({"conv": dict(B=B, c_in=C, c_out=CO, H=H, W=W, k=KH, stride=ST, pad=PD, L=L, rank=K),
                  "tokens": T, "lowered_d_in": d_in, "ms_per_step": round(ms, 4),
                  "image_MB_per_pass": round(img / 1e6, 1), "patch_matrix_MB": round(patches / 1e6, 1),
                  "kernels_us": {k: round(t / n * 1e3, 1) for k, (n, t) in prof.items()}}))
