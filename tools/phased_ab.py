# c2 backward schedules on one GPU: fused (one du launch) vs the DP-phased split
# (du(dU1|db), then b2b_bwd + du(dU2)), each with 0 and 8 reserved SMs.
# Prints batch-timed step time and per-kernel event times.
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_15473_b200 as skl
from paper_2601_15473_b200.dp import GradBucket
dev = torch.device("cuda", 0)
d_in, d_out, l, k = 768, 3072, 2, 128
T = int(os.environ.get("T", "32768"))
s = skl.shape(d_in, d_out, l, k, skl.BF16)
td = torch.bfloat16
S1s = torch.empty(l, d_in, k, dtype=td, device=dev); S2s = torch.empty(l, k, d_out, dtype=td, device=dev)
U1s = torch.empty(l, k, d_out, dtype=td, device=dev); U2s = torch.empty(l, d_in, k, dtype=td, device=dev)
skl.generate_sketches(s, 0, 1, S1s, S2s); skl.init_params(s, 1, U1s, U2s)
X = torch.randn(T, d_in, device=dev).to(td); Y = torch.empty(T, d_out, dtype=td, device=dev)
G = torch.randn(T, d_out, device=dev).to(td); GX = torch.empty(T, d_in, dtype=td, device=dev)
B = torch.zeros(d_out, dtype=td, device=dev)
sv = torch.empty(l * k, (T + 7) // 8 * 8, dtype=td, device=dev)
gb = GradBucket.allocate(d_in, d_out, l, k, device=dev)
ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device=dev)
fw = lambda: skl.forward(s, X, S1s, S2s, U1s, U2s, B, Y, sv, ws)


def fused():
    fw()
    skl.backward(s, G, X, sv, S1s, S2s, U1s, U2s, GX, gb.dU1s, gb.dU2s, gb.db, ws)


def phased():
    fw()
    skl.backward_phase(s, skl.BWD_DU1_DB, G, X, sv, S1s, S2s, U1s, U2s, None, gb.dU1s, None, gb.db, ws)
    skl.backward_phase(s, skl.BWD_DX_DU2, G, X, sv, S1s, S2s, U1s, U2s, GX, None, gb.dU2s, None, ws)


def du1():
    skl.backward_phase(s, skl.BWD_DU1_DB, G, X, sv, S1s, S2s, U1s, U2s, None, gb.dU1s, None, gb.db, ws)


def dxdu2():
    skl.backward_phase(s, skl.BWD_DX_DU2, G, X, sv, S1s, S2s, U1s, U2s, GX, None, gb.dU2s, None, ws)


variants = [a for a in sys.argv[1:]] or ["fused:0", "fused:8", "phased:0", "phased:8"]
for v in variants:
    name, res = v.split(":")
    fn = {"fused": fused, "phased": phased, "du1": du1, "dxdu2": dxdu2}[name]
    skl.set_reserved_sms(int(res))
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 40
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    batch = e0.elapsed_time(e1) / n * 1e3
    skl.profile_enable(True); skl.profile_collect()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    prof = skl.profile_collect(); skl.profile_enable(False)
    print("%-8s res=%s step %.1f us" % (name, res, batch),
          {kk: (cnt // n, round(t / n * 1e3, 1)) for kk, (cnt, t) in prof.items()}, flush=True)
skl.set_reserved_sms(0)
