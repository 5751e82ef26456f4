# Timeline of b2b_bwd CTAs (exit) vs du CTAs (entry/exit) in one c2 backward.
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_15473_b200 as skl
dev = torch.device("cuda", 0)
d_in, d_out, l, k, T = [int(v) for v in (sys.argv[1:6] if len(sys.argv) > 5 else (768, 3072, 2, 128, 32768))]
s = skl.shape(d_in, d_out, l, k, skl.BF16)
td = torch.bfloat16
S1s = torch.empty(l, d_in, k, dtype=td, device=dev); S2s = torch.empty(l, k, d_out, dtype=td, device=dev)
U1s = torch.empty(l, k, d_out, dtype=td, device=dev); U2s = torch.empty(l, d_in, k, dtype=td, device=dev)
skl.generate_sketches(s, 0, 1, S1s, S2s); skl.init_params(s, 1, U1s, U2s)
X = torch.randn(T, d_in, device=dev).to(td); Y = torch.empty(T, d_out, dtype=td, device=dev)
G = torch.randn(T, d_out, device=dev).to(td); GX = torch.empty(T, d_in, dtype=td, device=dev)
B = torch.zeros(d_out, dtype=td, device=dev)
sv = torch.empty(l * k, T, dtype=td, device=dev)
dU1 = torch.empty(l * k * d_out, device=dev); dU2 = torch.empty(l * k * d_in, device=dev); db = torch.empty(d_out, device=dev)
ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device=dev)
def step():
    skl.forward(s, X, S1s, S2s, U1s, U2s, B, Y, sv, ws)
    skl.backward(s, G, X, sv, S1s, S2s, U1s, U2s, GX, dU1, dU2, db, ws)
for _ in range(5): step()
torch.cuda.synchronize()
# the b2b trace holds the LAST b2b launch (bwd) since both write the same array
step(); torch.cuda.synchronize()
bb = (ctypes.c_ulonglong * (296 * 4))(); skl.lib().skl_debug_b2b_ts(bb, 296 * 4)
b = np.array(bb, dtype=np.float64).reshape(296, 4)[:148]
du = (ctypes.c_ulonglong * (296 * 12))(); skl.lib().skl_debug_du_ts(du, 296 * 12)
u = np.array(du, dtype=np.float64).reshape(296, 12)
x3 = u[:, 6:12].copy()
clk = u[:, 5] - u[:, 4]; gt = u[:, 3] - u[:, 2]
loopclk = u[:, 4].copy()
u = u[:, :4]
keep = u[:, 0] > 0
u = u[keep]; clk = clk[keep]; gt = gt[keep]; x3 = x3[keep]
print("effective SM MHz over main+drain: min %.0f med %.0f max %.0f" % ((clk/gt*1e3).min(), np.median(clk/gt*1e3), (clk/gt*1e3).max()))
t0 = b[:, 0].min()
wb = (ctypes.c_ulonglong * (296 * 16))(); skl.lib().skl_debug_du_wend(wb, 296 * 16)
w = (np.array(wb, dtype=np.float64).reshape(296, 16)[:len(keep)][keep] - t0) / 1e3
b = (b - t0) / 1e3; u = (u - t0) / 1e3
print("b2b_bwd entry %.1f..%.1f  exit: min %.1f  p25 %.1f  med %.1f  max %.1f" % (b[:,0].min(), b[:,0].max(), b[:,3].min(), np.percentile(b[:,3],25), np.median(b[:,3]), b[:,3].max()))
print("du CTAs", len(u))
print("du entry sorted (us):", np.round(np.sort(u[:, 0]), 1).tolist())
print("du exit  sorted (us):", np.round(np.sort(u[:, 1]), 1).tolist())
pb = (ctypes.c_ulonglong * (296 * 8))(); skl.lib().skl_debug_du_prof(pb, 296 * 8)
p = np.array(pb, dtype=np.float64).reshape(296, 8)[:len(u)] / 1965.0  # cycles -> us
names = ["prod_wait_empty", "prod_total", "mma_wait_full", "mma_total", "ep_colsum", "ep_wait_acc", "ep_part", "ep_red"]
for i, nm in enumerate(names):
    print("%-16s min %6.1f med %6.1f max %6.1f" % (nm, p[:, i].min(), np.median(p[:, i]), p[:, i].max()))
print("per-CTA rows (leader CTAs of first 4 clusters):")
for c in range(0, min(len(u), 32), 2): print(c, np.round(p[c], 1).tolist(), np.round(u[c], 1).tolist())

print("columns: entry, exit, prologue done, reduce start (us)")
for c in range(0, len(u), 8): print(c, np.round(u[c], 1).tolist(), "main+drain %.1f reduce %.1f" % (u[c,3]-u[c,2], u[c,1]-u[c,3]))

print("per-warp reduce-loop end / kernel end (us), CTA 0, 8, 96:")
for c in (0, 8, 96):
    if c < len(w): print(c, "reduce start %.1f" % u[c, 3], np.round(w[c, :8], 1).tolist(), np.round(w[c, 8:], 1).tolist(), "exit %.1f" % u[c, 1])

print("reduce-loop cycles (clock64) CTA 0, 8, 96:", [loopclk[c] for c in (0, 8, 96) if c < len(loopclk)])

x3 = (x3 - t0) / 1e3
print("issue-done / wait-done / tail-done (us) for CTA 0, 8, 96:")
for c in (0, 8, 96):
    if c < len(x3): print(c, "start %.1f" % u[c, 3], np.round(x3[c], 1).tolist(), "exit %.1f" % u[c, 1])
print("timeline per CTA (entry, prologue-done, reduce-start, exit):")
for c in (0, 8, 96):
    if c < len(u): print(c, np.round(u[c, [0, 2, 3, 1]], 1).tolist())

print("main-loop done (tfull) / partial stored (us):")
for c in (0, 8, 96):
    if c < len(u): print(c, "tfull %.1f" % x3[c, 3], "dumped %.1f" % x3[c, 4], "stored %.1f" % x3[c, 5], "reduce start %.1f" % u[c, 3], "sum done %.1f" % x3[c, 2], "exit %.1f" % u[c, 1])

