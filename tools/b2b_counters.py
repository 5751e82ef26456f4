import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_15473_b200 as skl
dev = torch.device("cuda", 0)
d_in, d_out, l, k = [int(v) for v in sys.argv[1:5]]
which = sys.argv[5]
T = int(os.environ.get("T", "32768"))
s = skl.shape(d_in, d_out, l, k, skl.BF16)
td = torch.bfloat16
S1s = torch.empty(l, d_in, k, dtype=td, device=dev); S2s = torch.empty(l, k, d_out, dtype=td, device=dev)
U1s = torch.empty(l, k, d_out, dtype=td, device=dev); U2s = torch.empty(l, d_in, k, dtype=td, device=dev)
skl.generate_sketches(s, 0, 1, S1s, S2s); skl.init_params(s, 1, U1s, U2s)
X = torch.randn(T, d_in, device=dev).to(td); Y = torch.empty(T, d_out, dtype=td, device=dev)
G = torch.randn(T, d_out, device=dev).to(td); GX = torch.empty(T, d_in, dtype=td, device=dev)
B = torch.zeros(d_out, dtype=td, device=dev)
sv = torch.empty(l * k, T, dtype=td, device=dev)
du1 = torch.empty(l, k, d_out, device=dev); du2 = torch.empty(l, d_in, k, device=dev); db = torch.empty(d_out, device=dev)
ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device=dev)
def run():
    if which == "fwd": skl.forward(s, X, S1s, S2s, U1s, U2s, B, Y, sv, ws)
    else: skl.backward_phase(s, skl.BWD_DX_DU2, G, X, sv, S1s, S2s, U1s, U2s, GX, None, du2, None, ws)
for _ in range(3): run()
torch.cuda.synchronize(); run(); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (296 * 8))()
skl.lib().skl_debug_b2b_prof(buf, 296 * 8); p = np.array(buf, dtype=np.float64).reshape(296, 8)[:148] / 1965.0
skl.lib().skl_debug_b2b_eprof(buf, 296 * 8); e = np.array(buf, dtype=np.float64).reshape(296, 8)[:148] / 1965.0
names = ["mma wait G1 stage", "mma wait G2 stage", "mma wait tmem slot", "mma wait H ready", "mma total", "prod wait G1", "prod wait G2", "prod total"]
en = ["ep wait acc", "ep bulk reuse", "ep bar a", "ep bar b", "ep wait G1 chunk", "ep total", "ep convert", "ep tmem ld"]
lead = p[0::2]
print(which, (d_in, d_out, l, k))
print(" MMA:", {n: round(v, 2) for n, v in zip(names[:5], lead[:, :5].mean(0))})
print(" prod:", {n: round(v, 2) for n, v in zip(names[5:], p[:, 5:].mean(0))})
print(" epi:", {n: round(v, 2) for n, v in zip(en, e.mean(0))})
