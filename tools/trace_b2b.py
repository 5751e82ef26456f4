"""Per-role event timelines of one b2b / du launch (trace build, csrc/trace.cuh):

    make -C scratch/csrc_trace EXTRA=-DSKL_TRACE=1   (a copy of csrc -> scratch/libskl.so)
    SKL_LIB=scratch/libskl.so python tools/trace_b2b.py d_in d_out L k [T] [fwd|bwd]

Prints, for the traced CTAs, each role's events as code@kilocycles (from the
first event of the CTA).  Codes: producer 1 = G1 stage acquired, 2 = G2 stage;
MMA 10 = G2 slots acquired for chunk 1, 11 = G1 stage full, 12 = H ready,
13 = G2 slot free, 14 = G2 stage full; epilogue 21 = G1 chunk accumulated,
22 = chunk converted, 23 = saves done, 24 = G2 tile accumulated,
25 = staging buffer free, 26 = tile store issued.  Slots 4-7 (SLOTS=4,6) are
the du kernel: producer 1 = stage acquired; MMA 12 = unit start, 11 = stage
full; epilogue 21 = accumulator ready, 22 = dumped to smem; tail 23 = after
the cluster barrier, 24 = partial slices loaded, 25 = reduced and stored."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_15473_b200 as skl  # noqa: E402

d_in, d_out, L, k = (int(v) for v in sys.argv[1:5])
T = int(sys.argv[5]) if len(sys.argv) > 5 else 32768
which = sys.argv[6] if len(sys.argv) > 6 else "fwd"
lib = skl.lib()
lib.skl_trace_dump.argtypes = [ctypes.c_void_p, ctypes.c_int]
dev = torch.device("cuda", 0)
lyr = skl.SkLinear(d_in, d_out, L, k, seed=1, dtype=skl.BF16)
X = torch.randn(T, d_in, device=dev).to(torch.bfloat16)
G = torch.randn(T, d_out, device=dev).to(torch.bfloat16)
sv = torch.empty(L * k, (T + 7) // 8 * 8, dtype=torch.bfloat16, device=dev)
for _ in range(3):
    lyr.forward(X, saved=sv)
    lyr.backward(X, G, saved=sv)
torch.cuda.synchronize()
if which == "bwd":
    lyr.forward(X, saved=sv)
    torch.cuda.synchronize()
lib.skl_trace_reset()
if which == "fwd":
    lyr.forward(X, saved=sv)
else:
    lyr.backward(X, G, saved=sv)
torch.cuda.synchronize()
n = 8 * 4 * 2 * 1024
buf = (ctypes.c_uint64 * n)()
assert lib.skl_trace_dump(buf, n) == n, lib.skl_trace_dump(buf, n)
slots = os.environ.get("SLOTS", "0,2").split(",")
for s in (int(v) for v in slots):
    rows = []
    for r in range(4):
        base = (s * 4 + r) * 2048
        ev = [(buf[base + 2 * i], buf[base + 2 * i + 1]) for i in range(1024) if buf[base + 2 * i]]
        rows.append(ev)
    t0 = min((e[0][0] for e in rows if e), default=0)
    print(f"== slot {s}")
    for r, ev in enumerate(rows):
        print(f"  role {r} ({len(ev)} events):", " ".join(f"{c}@{(t - t0) / 1e3:.1f}" for t, c in ev))
