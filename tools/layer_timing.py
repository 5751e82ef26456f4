# Back-to-back launches of one layer's forward (and backward): batch-timed vs per-launch profiler.
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_15473_b200 as skl
dev = torch.device("cuda", 0)
d_in, d_out, l, k = [int(v) for v in sys.argv[1:5]]
T = int(os.environ.get("T", "32768"))
tf32 = os.environ.get('DT') == 'tf32'
s = skl.shape(d_in, d_out, l, k, skl.F32_TF32 if tf32 else skl.BF16)
td = torch.float32 if tf32 else torch.bfloat16
S1s = torch.empty(l, d_in, k, dtype=td, device=dev); S2s = torch.empty(l, k, d_out, dtype=td, device=dev)
U1s = torch.empty(l, k, d_out, dtype=td, device=dev); U2s = torch.empty(l, d_in, k, dtype=td, device=dev)
skl.generate_sketches(s, 0, 1, S1s, S2s); skl.init_params(s, 1, U1s, U2s)
X = torch.randn(T, d_in, device=dev).to(td); Y = torch.empty(T, d_out, dtype=td, device=dev)
G = torch.randn(T, d_out, device=dev).to(td); GX = torch.empty(T, d_in, dtype=td, device=dev)
B = torch.zeros(d_out, dtype=td, device=dev)
sv = torch.empty(l * k, T, dtype=td, device=dev)
du1 = torch.empty(l * k * d_out, device=dev); du2 = torch.empty(l * k * d_in, device=dev); db = torch.empty(d_out, device=dev)
ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device=dev)
fw = lambda: skl.forward(s, X, S1s, S2s, U1s, U2s, B, Y, sv, ws)
bw = lambda: skl.backward(s, G, X, sv, S1s, S2s, U1s, U2s, GX, du1, du2, db, ws)
for name, fn in (("fwd", fw), ("bwd", bw), ("step", lambda: (fw(), bw()))):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    batch = e0.elapsed_time(e1) / n * 1e3
    skl.profile_enable(True); skl.profile_collect()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    prof = skl.profile_collect(); skl.profile_enable(False)
    print(name, "batch-timed %.1f us/call" % batch, {kk: round(t / cnt * 1e3, 1) for kk, (cnt, t) in prof.items()})
import time
for name, fn in (("fwd", fw), ("bwd", bw)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(100): fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(name, "host enqueue %.1f us/call" % ((t1 - t0) / 100 * 1e6))
