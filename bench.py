#!/usr/bin/env python3
"""bench.py -- SKLinear fwd+bwd tokens/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1, one rank per GPU)

A step is one SKLinear forward + backward (dX, dU1s, dU2s, db) over one batch
of synthetic tokens, through the C-ABI of libskl.so:
  workload c2 (BASELINE.json configs[1], the BERT-base FFN shape):
    d_in=768, d_out=3072, L=2, k=128, 32768 tokens per GPU, bf16.
Multi-GPU: token sharding (weak scaling, 32768 tokens per GPU); forward needs
no communication; the backward all-reduces the fp32 gradient bucket
(dU1s | db | dU2s) with NCCL, the dU1s | db part overlapped with the dX kernel.
Rank 0 prints one JSON line.  At N=1 the line also carries "workloads": the
other BASELINE.json configs (c1, c2-TF32, c3, c4 sweep) measured briefly, each
with its own binding-roofline fraction.

--impl reference times the reference's own CPU implementation
(oracle/_ref/librnla_ref.so: the unmodified reference sources, timed by the
reference's bench::time_op) on all host threads, on the same workload (c2 at
full T per step, OMP_PROC_BIND=close OMP_WAIT_POLICY=active; timed calls capped
at REF_BUDGET_S); rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SKLinear fwd+bwd tokens/s and % roofline at 1/2/4/8 B200 vs host-CPU reference"
D_IN, D_OUT, L, K_RANK, T_GPU = 768, 3072, 2, 128, 32768
SEED = 42
WORKLOAD = (f"c2: SKLinear fwd+bwd d_in={D_IN} d_out={D_OUT} L={L} k={K_RANK}, "
            f"{T_GPU} tokens per GPU (BERT-base FFN shape)")
# SMs libskl leaves free for NCCL when N > 1.  0: measured on one B200, 8
# reserved SMs cost the phased step 28 us (312 vs 284 us) while the persistent
# b2b_bwd kernel frees 40 SMs after its first wave anyway (128 tiles on 74
# pairs), under which the head all-reduce runs -- its NCCL stream is created
# high-priority so its CTAs take those SMs first.
RESERVED_SMS = 0
NCCL_CTAS = 8        # NCCL_MAX_CTAS for the ~3-4 MB gradient buckets


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["bf16_tflops"]), float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json, burst)"
    return 1590.0, 6650.0, "fallback (B200_PROFILING.md)"


def sustained_tflops(dtype):
    """The sustained (4 s back-to-back) dense peak for the long sweep workloads, reported
    next to the burst-based fraction: bf16 from MEASURED_PEAKS.json, TF32 from
    profiles/r2_tf32_peak.json."""
    if dtype == "bf16":
        p = os.path.join(ROOT, "MEASURED_PEAKS.json")
        if os.path.exists(p):
            with open(p) as f:
                d = json.load(f)
            if "bf16_tflops_sustained" in d:
                return float(d["bf16_tflops_sustained"])
        return None
    with open(os.path.join(ROOT, "profiles", "r2_tf32_peak.json")) as f:
        return float(json.load(f)["tf32_tflops_sustained"])


def tf32_peak():
    """Dense TF32 peak: MEASURED_PEAKS.json when the driver measured it, else the
    figure tools/measure_tf32_peak.py measured on a B200 (cuBLAS fp32 8192^3 with
    TF32, burst), committed as profiles/r2_tf32_peak.json."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        if "tf32_tflops" in d:
            return float(d["tf32_tflops"]), "measured (MEASURED_PEAKS.json, burst)"
    q = os.path.join(ROOT, "profiles", "r2_tf32_peak.json")
    with open(q) as f:
        d = json.load(f)
    return float(d["tf32_tflops"]), "measured (profiles/r2_tf32_peak.json: cuBLAS TF32 8192^3, burst)"


def flops_per_token(d_in=D_IN, d_out=D_OUT, l=L, k=K_RANK):
    R, D = 2 * l * k, d_in + d_out
    return {"fwd": 2 * R * D, "bwd": 3 * R * D, "b2b": 2 * R * D,
            "dU1": 2 * l * k * d_out, "dU2": 2 * l * k * d_in}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            with open(self.path) as f:
                for line in f:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        except Exception:
            pass
        finally:
            try:
                os.unlink(self.path)
            except Exception:
                pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        loaded = [s for s in sm if s > 0.5 * (max(sm) if sm else 1)] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


OMP_ENV = {"OMP_PROC_BIND": "close", "OMP_WAIT_POLICY": "active"}  # BASELINE.md §3 (set before libgomp loads)
CPU_SLICE_1T = 1024  # tokens of the single-thread sample (a full-T call takes ~2 min on one core)


def _cpu_ref_time(T, threads, trials, warmup):
    """Reference SkLinear fwd+bwd on the c2 layer (oracle/_ref: the unmodified
    reference sources, timed by its own bench::time_op) -> (mean ms, std ms)."""
    import oracle
    o = oracle.Oracle("reference")
    return o.time_fwd_bwd(D_IN, D_OUT, L, K_RANK, T, SEED, threads, trials, warmup)


def cpu_probe(args):
    """--impl cpu-probe: the N=1 line's cpu_baseline, in its own process so the
    OpenMP environment applies: c2 at full T on every host core,
    plus a single-thread sample.  Prints one JSON object."""
    import oracle
    threads = os.cpu_count() or 1
    if not oracle.available("reference"):  # scalar C restatement (oracle/skl_oracle.c), single thread
        o = oracle.Oracle("port")
        t = 256
        p = o.sk_linear_fresh(D_IN, D_OUT, L, K_RANK, SEED)
        x, g, b = oracle.inputs(D_IN, D_OUT, t, SEED, o)
        t0 = time.perf_counter()
        o.forward(p, b, x)
        o.backward(p, x, g)
        ms = (time.perf_counter() - t0) * 1e3
        print(json.dumps({"value": t / (ms / 1e3), "unit": "tokens/s", "cores": 1, "kind": "port",
                          "sample": f"c2 shape, {t}-token slice, scalar f64 port, 1 call ({ms:.0f} ms)"}))
        return
    full_ms, full_std = _cpu_ref_time(T_GPU, threads, 1, 1)
    one_ms, _ = _cpu_ref_time(CPU_SLICE_1T, 1, 1, 0)
    print(json.dumps({
        "value": T_GPU / (full_ms / 1e3), "unit": "tokens/s", "cores": threads, "kind": "reference",
        "sample": (f"c2 at full T={T_GPU} (same config as the GPU line), fwd+bwd f64 through the reference's "
                   f"bench::time_op: 1 warm-up + 1 timed call = {full_ms:.0f} ms on {threads} threads, "
                   f"OMP_PROC_BIND=close OMP_WAIT_POLICY=active"),
        "same_config": True,
        "single_thread": {"value": CPU_SLICE_1T / (one_ms / 1e3), "unit": "tokens/s", "cores": 1,
                          "sample": f"{CPU_SLICE_1T}-token slice of c2, 1 timed call = {one_ms:.0f} ms"}}))


def cpu_baseline_reference():
    """The N=1 line's cpu_baseline: cpu_probe in a subprocess (own OpenMP env)."""
    env = dict(os.environ, **OMP_ENV)
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--impl", "cpu-probe"], env=env,
                       capture_output=True, text=True, timeout=900)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    if r.returncode != 0 or not lines:
        raise RuntimeError((r.stderr or r.stdout)[-300:])
    return json.loads(lines[-1])


# Other BASELINE.json configs (parity-tested in tests/; reported, not the headline):
#   name, d_in, d_out, L, k, tokens, dtype
SWEEP = [
    ("c1 fp32/TF32 1024->1024 L1 k64 T64", 1024, 1024, 1, 64, 64, "tf32"),
    ("c2 TF32 768->3072 L2 k128 T32768", 768, 3072, 2, 128, 32768, "tf32"),
    ("c3 bf16 4096->4096 L3 k256 T65536", 4096, 4096, 3, 256, 65536, "bf16"),
    ("c4 bf16 4096 L1 k16 T131072", 4096, 4096, 1, 16, 131072, "bf16"),
    ("c4 bf16 4096 L2 k32 T131072", 4096, 4096, 2, 32, 131072, "bf16"),
    ("c4 bf16 4096 L4 k64 T131072", 4096, 4096, 4, 64, 131072, "bf16"),
    ("c4 TF32 4096 L1 k16 T131072", 4096, 4096, 1, 16, 131072, "tf32"),
    ("c4 TF32 4096 L2 k64 T131072", 4096, 4096, 2, 64, 131072, "tf32"),
]


def roofline_time(d_in, d_out, l, k, T, ebytes, peak_tf, peak_bw):
    """Binding roofline of one fwd+bwd step: FLOPs 5·R·D per token;
    algorithmic bytes (2D + d_in + 2Lk)·e per token (fwd: X, Y, saved; bwd: G,
    X, saved, dX) -- params/grads are per-call and negligible."""
    R, D = 2 * l * k, d_in + d_out
    flops = 5 * R * D * T
    bytes_ = (2 * D + d_in + 2 * l * k) * ebytes * T
    t_tensor, t_hbm = flops / (peak_tf * 1e12), bytes_ / (peak_bw * 1e9)
    return max(t_tensor, t_hbm), ("tensor" if t_tensor >= t_hbm else "hbm"), flops, bytes_


def _time_steps(torch, fn, steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.current_stream()
    e0.record(st)
    for _ in range(steps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def measure_workload(skl, torch, dev, name, d_in, d_out, l, k, T, dtype, steps=10, warmup=3, phased=False,
                     graph=False):
    kind = skl.BF16 if dtype == "bf16" else skl.F32_TF32
    td = torch.bfloat16 if dtype == "bf16" else torch.float32
    s = skl.shape(d_in, d_out, l, k, kind)
    S1s = torch.empty(l, d_in, k, dtype=td, device=dev)
    S2s = torch.empty(l, k, d_out, dtype=td, device=dev)
    U1s = torch.empty(l, k, d_out, dtype=td, device=dev)
    U2s = torch.empty(l, d_in, k, dtype=td, device=dev)
    skl.generate_sketches(s, skl.GAUSSIAN, SEED, S1s, S2s)
    skl.init_params(s, SEED, U1s, U2s)
    gen = torch.Generator(device=dev)
    gen.manual_seed(7)
    bias = torch.randn(d_out, device=dev, generator=gen).to(td)
    X = torch.randn(T, d_in, device=dev, generator=gen).to(td)
    G = torch.randn(T, d_out, device=dev, generator=gen).to(td)
    Y = torch.empty(T, d_out, dtype=td, device=dev)
    GX = torch.empty(T, d_in, dtype=td, device=dev)
    saved = torch.empty(l * k, (T + 7) // 8 * 8, dtype=td, device=dev)
    du1 = torch.empty(l, k, d_out, device=dev)
    du2 = torch.empty(l, d_in, k, device=dev)
    db = torch.empty(d_out, device=dev)
    ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device=dev)

    def step():
        skl.forward(s, X, S1s, S2s, U1s, U2s, bias, Y, saved, ws)
        if phased:
            skl.backward_phase(s, skl.BWD_DU1_DB, G, X, saved, S1s, S2s, U1s, U2s, None, du1, None, db, ws)
            skl.backward_phase(s, skl.BWD_DX_DU2, G, X, saved, S1s, S2s, U1s, U2s, GX, None, du2, None, ws)
        else:
            skl.backward(s, G, X, saved, S1s, S2s, U1s, U2s, GX, du1, du2, db, ws)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ms = ms_eager = _time_steps(torch, step, steps)
    if graph:  # launch-bound shapes: the same step replayed from a CUDA graph
        from paper_2601_15473_b200.graphs import capture
        g = capture(step)
        ms = _time_steps(torch, g.replay, steps)
    peak_bf16, peak_bw, _ = peaks()
    peak_tf, tf_src = (peak_bf16, "bf16 burst") if dtype == "bf16" else tf32_peak()
    t_roof, bound, flops, bytes_ = roofline_time(d_in, d_out, l, k, T, 2 if dtype == "bf16" else 4, peak_tf, peak_bw)
    r_pad = (2 * l * k + 63) // 64 * 64
    small = T <= 128 and 2.0 * 2 * l * k * (d_in + d_out) * T <= 0.5e9  # skl.cu use_small
    sus = sustained_tflops(dtype)
    t_roof_s = roofline_time(d_in, d_out, l, k, T, 2 if dtype == "bf16" else 4, sus, peak_bw)[0] if sus else None
    return {"workload": name, "dtype": dtype, "tokens": T, "ms_per_step": ms, "tokens_per_s": T / (ms / 1e3),
            "bound": bound, "roofline_ms": t_roof * 1e3, "roofline_frac": t_roof / (ms / 1e3),
            "roofline_frac_sustained_peak": (t_roof_s / (ms / 1e3)) if t_roof_s else None,
            "tflops": flops / (ms / 1e3) / 1e12, "hbm_gbs_alg": bytes_ / (ms / 1e3) / 1e9,
            # on-chip H: bf16 b2b kernel (R <= 512), TF32 b2b kernel (R <= 256) or wide-rank TF32 kernel (R <= 512);
            # T <= 128 takes the small-batch path (rank intermediate in a 32 KB fp32 buffer, L2-resident)
            "fused": bool(r_pad <= 512) and not small,
            "path": ("small-batch (small.cu: T <= 128, fp32 FMA over parameter slices)" if small
                     else "fused b2b (H on chip)" if r_pad <= 512 else "unfused tcgen05 GEMM chain (H through HBM)"),
            "peak_tflops_used": peak_tf, "peak_source": tf_src, "phased_backward": phased, "cuda_graph": graph,
            "ms_per_step_eager": ms_eager}


def measure_stack(skl, torch, dev, world, steps=5, warmup=2, T=T_GPU, num_layers=12):
    """BASELINE config 5: the 12-layer BERT-base stack of SKLinear FFN/proj
    layers (paper_2601_15473_b200.model.bert_ffn_stack: 72 SKLinear layers,
    ReLU fused), fwd + bwd of T tokens per GPU; at N > 1 every layer's dU
    bucket is all-reduced (NCCL) overlapped with the layers below it."""
    import torch.distributed as dist
    from paper_2601_15473_b200.model import bert_ffn_stack, wait_all
    chain = bert_ffn_stack(num_layers=num_layers, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(11)
    x = torch.randn(T, 768, device=dev, generator=gen).to(torch.bfloat16)
    g = torch.randn(T, 768, device=dev, generator=gen).to(torch.bfloat16)
    buckets = chain.allocate_grads(dev)

    def step():
        chain.forward(x)
        _, works = chain.backward(g, buckets=buckets, need_grad_x=False, overlap=world > 1)
        wait_all(works)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ms_eager = _time_steps(torch, step, steps)
    graph = world == 1  # one process: replay the 72-layer step from a CUDA graph (no per-call host work)
    if graph:
        from paper_2601_15473_b200.graphs import capture
        gr = capture(step)
        ms = _time_steps(torch, gr.replay, steps)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    peak_bf16, peak_bw, _ = peaks()
    sus = sustained_tflops("bf16")
    t_roof = t_roof_s = 0.0
    flops = 0
    for stp in chain.steps:
        L = stp.layer
        tr, _, f, _ = roofline_time(L.d_in, L.d_out, L.num_terms, L.low_rank, T, 2, peak_bf16, peak_bw)
        t_roof += tr
        if sus:
            t_roof_s += roofline_time(L.d_in, L.d_out, L.num_terms, L.low_rank, T, 2, sus, peak_bw)[0]
        flops += f
    del chain, buckets
    torch.cuda.empty_cache()
    return {"workload": f"c5 BERT-base {num_layers}-layer SKLinear FFN/proj stack ({6 * num_layers} SKLinear, "
                        f"fused ReLU), fwd+bwd, {T} tokens per GPU" + (f", dp{world} overlapped all-reduce"
                                                                        if world > 1 else ""),
            "dtype": "bf16", "tokens": T * world, "ms_per_step": ms, "tokens_per_s": world * T / (ms / 1e3),
            "bound": "tensor", "roofline_ms": t_roof * 1e3, "roofline_frac": t_roof / (ms / 1e3),
            "roofline_frac_sustained_peak": (t_roof_s / (ms / 1e3)) if sus else None,
            "tflops": flops / (ms / 1e3) / 1e12, "n_gpus": world, "cuda_graph": graph, "ms_per_step_eager": ms_eager}


REF_BUDGET_S = 150.0  # wall-clock cap of the reference arm's timed calls (full-T calls take seconds each)


def run_reference(args, rank):
    """--impl reference: the reference's CPU implementation (oracle/_ref, all host
    threads, OMP env of BASELINE.md §3) on THIS arm's workload, c2 at full
    T = 32768 per step.  Warm-up capped at 1 call and the timed calls at what
    fits REF_BUDGET_S (each call takes seconds); both counts are in the line."""
    if rank != 0:
        return
    import oracle
    threads = os.cpu_count() or 1
    if not oracle.available("reference"):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/librnla_ref.so not built"}))
        return
    warm = min(1, max(0, args.warmup))
    t0 = time.perf_counter()
    first_ms, _ = _cpu_ref_time(T_GPU, threads, 1, warm)
    per_call = (time.perf_counter() - t0) / (1 + warm)
    extra = max(0, min(args.steps - 1, int(REF_BUDGET_S / max(per_call, 1e-3)) - 1))
    ms = first_ms
    if extra > 0:
        m2, _ = _cpu_ref_time(T_GPU, threads, extra, 0)
        ms = (first_ms + extra * m2) / (1 + extra)
    timed = 1 + extra
    v = T_GPU / (ms / 1e3)
    cb = {"value": v, "unit": "tokens/s", "cores": threads, "kind": "reference", "same_config": True,
          "sample": (f"c2 at full T={T_GPU} per step (the GPU arm's workload), fwd+bwd f64 via the reference's "
                     f"bench::time_op, {timed} timed call(s) after {warm} warm-up (capped at {REF_BUDGET_S:.0f} s; "
                     f"--steps {args.steps}), OMP_PROC_BIND=close OMP_WAIT_POLICY=active")}
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": timed,
            "warmup": warm, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "d_in": D_IN, "d_out": D_OUT, "num_terms": L, "low_rank": K_RANK,
                       "tokens_per_step": T_GPU, "parallelism": f"host OpenMP, {threads} threads"},
            "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _relaunch_under_torchrun(n):
    """`python bench.py --gpus N` without a launcher: re-exec this command under
    torch.distributed.run with N ranks (one per GPU) on 127.0.0.1."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference", "cpu-probe"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the other-config workloads at N=1")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup) if args.impl == "ours" else args.warmup

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        _relaunch_under_torchrun(args.gpus)  # one process per GPU (does not return)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "ours" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    if args.impl == "cpu-probe":
        cpu_probe(args)
        return
    if args.impl == "reference":
        for k_, v_ in OMP_ENV.items():  # before the reference library (libgomp) loads
            os.environ.setdefault(k_, v_)
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_2601_15473_b200 as skl

    torch.cuda.set_device(local_rank)
    if world > 1:
        os.environ.setdefault("NCCL_MAX_CTAS", str(NCCL_CTAS))
        opts = dist.ProcessGroupNCCL.Options()
        opts.is_high_priority_stream = True
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank), pg_options=opts)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream()

    s = skl.shape(D_IN, D_OUT, L, K_RANK, skl.BF16)
    bf = torch.bfloat16
    # Replicated parameters: every rank regenerates the same sketches / U from the seed.
    S1s = torch.empty(L, D_IN, K_RANK, dtype=bf, device=dev)
    S2s = torch.empty(L, K_RANK, D_OUT, dtype=bf, device=dev)
    U1s = torch.empty(L, K_RANK, D_OUT, dtype=bf, device=dev)
    U2s = torch.empty(L, D_IN, K_RANK, dtype=bf, device=dev)
    skl.generate_sketches(s, skl.GAUSSIAN, SEED, S1s, S2s)
    skl.init_params(s, SEED, U1s, U2s)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)
    bias = (torch.randn(D_OUT, device=dev, generator=gen) * 0.1).to(bf)
    T = T_GPU
    X = torch.randn(T, D_IN, device=dev, generator=gen).to(bf)
    G = torch.randn(T, D_OUT, device=dev, generator=gen).to(bf)
    Y = torch.empty(T, D_OUT, dtype=bf, device=dev)
    saved = torch.empty(L * K_RANK, (T + 7) // 8 * 8, dtype=bf, device=dev)  # Savedᵀ [L*k][round8(T)]
    GX = torch.empty(T, D_IN, dtype=bf, device=dev)
    from paper_2601_15473_b200.dp import GradBucket, backward_overlapped
    gb = GradBucket.allocate(D_IN, D_OUT, L, K_RANK, device=dev)  # dU1s | db | dU2s (fp32)
    bucket = gb.flat
    ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device=dev)
    if world > 1:
        # leave SMs for the NCCL kernel that runs concurrently with the dX kernel
        skl.set_reserved_sms(RESERVED_SMS)

    def step(x=X, g=G):
        skl.forward(s, x, S1s, S2s, U1s, U2s, bias, Y, saved, ws)
        if world > 1:  # phased backward: all-reduce of dU1s|db overlaps the dX kernel
            for w in backward_overlapped(skl, s, g, x, saved, S1s, S2s, U1s, U2s, GX, gb, ws):
                w.wait()
        else:
            skl.backward(s, g, x, saved, S1s, S2s, U1s, U2s, GX, gb.dU1s, gb.dU2s, gb.db, ws)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    barrier()

    # ---------------- timed region: device-resident inputs (X, G > L2 each step)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = skl.launch_count()
    with ClockSampler(local_rank) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        barrier()
    launches = skl.launch_count() - launches0
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    clocks = clk.summary()
    value = world * T / (ms / 1e3)

    # ---------------- per-kernel device times (CUDA events on the launch stream)
    skl.profile_enable(True)
    skl.profile_collect()
    barrier()
    for _ in range(args.steps):
        step()
    barrier()
    prof = skl.profile_collect()
    skl.profile_enable(False)
    per_kernel = {k: {"launches": n, "avg_ms": t / n, "share": None} for k, (n, t) in prof.items()}
    tot = sum(t for (_, t) in prof.values()) or 1.0
    for k, (n, t) in prof.items():
        per_kernel[k]["share"] = t / tot
    dom = max(prof.items(), key=lambda kv: kv[1][1])[0] if prof else None
    fpt = flops_per_token()
    alg_flops = {"b2b_fwd": fpt["b2b"] * T, "b2b_bwd": fpt["b2b"] * T, "gemm_dU1": fpt["dU1"] * T,
                 "gemm_dU2": fpt["dU2"] * T}
    peak_tf, peak_bw, peak_src = peaks()
    roof = None
    if dom in alg_flops:
        avg_ms = per_kernel[dom]["avg_ms"]
        achieved = alg_flops[dom] / (avg_ms / 1e3) / 1e12
        # dram__bytes_read.sum + dram__bytes_write.sum of this kernel from one `ncu --set full`
        # capture (not measured in this run: ncu replays kernels); the capture is named in the line
        traffic, traffic_src = None, None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                tj = json.load(f)
            traffic, traffic_src = tj.get(dom), tj.get("_source", "profiles/traffic.json")
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": achieved / peak_tf, "traffic": traffic, "traffic_source": traffic_src, "kernel": dom,
                "kernel_ms": avg_ms, "peak_source": peak_src}
    step_flops = (fpt["fwd"] + fpt["bwd"]) * T
    step_roof = step_flops / (ms / 1e3) / 1e12

    # ---------------- end to end: host buffers through the public API
    # Every step copies its X, G from pinned host memory and reads the gradient
    # bucket back.  The copy of step i+1 runs on a copy stream while step i
    # computes (double-buffered device inputs, as a data loader would), so the
    # step is bound by the PCIe H2D of its 252 MB, not copy + compute.
    Xh = X.cpu().pin_memory()
    Gh = G.cpu().pin_memory()
    Xd = [torch.empty_like(X), torch.empty_like(X)]
    Gd = [torch.empty_like(G), torch.empty_like(G)]
    out_h = torch.empty(bucket.numel(), dtype=torch.float32).pin_memory()
    copy_stream = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]

    def e2e_run(n):
        with torch.cuda.stream(copy_stream):
            Xd[0].copy_(Xh, non_blocking=True)
            Gd[0].copy_(Gh, non_blocking=True)
            copied[0].record(copy_stream)
        for i in range(n):
            cur, nxt = i % 2, (i + 1) % 2
            if i + 1 < n:
                with torch.cuda.stream(copy_stream):
                    if i >= 1:
                        copy_stream.wait_event(consumed[nxt])  # step i-1 finished reading buffer nxt
                    Xd[nxt].copy_(Xh, non_blocking=True)
                    Gd[nxt].copy_(Gh, non_blocking=True)
                    copied[nxt].record(copy_stream)
            stream.wait_event(copied[cur])
            step(Xd[cur], Gd[cur])
            consumed[cur].record(stream)
            out_h.copy_(bucket, non_blocking=True)

    e2e_run(2)
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    copy_stream.wait_stream(stream)  # the first H2D starts inside the timed region
    e2e_run(args.steps)
    f1.record(stream)
    barrier()
    ms_e2e = max_over_ranks(f0.elapsed_time(f1) / args.steps)
    e2e = {"value": world * T / (ms_e2e / 1e3), "unit": "tokens/s",
           "h2d_bytes_per_step": Xh.numel() * 2 + Gh.numel() * 2, "d2h_bytes_per_step": out_h.numel() * 4,
           "ms_per_step": ms_e2e,
           # the binding resource end to end is the host link: achieved H2D rate over the step
           "h2d_gbs": (Xh.numel() * 2 + Gh.numel() * 2) / (ms_e2e / 1e3) / 1e9,
           "bound": "PCIe host->device copy of X and G (the device step is %.0f%% of it)" % (100 * ms / ms_e2e),
           "path": "pinned host X,G -(copy stream, double-buffered)-> sketched_linear_forward/backward -> "
                   "grad bucket to pinned host, every step"}

    workloads = None
    if world > 1 and not args.no_sweep:  # the stack exercises the per-layer overlapped all-reduce
        try:
            workloads = [measure_stack(skl, torch, dev, world)]
        except Exception as e:
            workloads = [{"workload": "c5 stack", "error": str(e)[:200]}]
    if world == 1 and not args.no_sweep:
        workloads = []
        for (name, di, do, l, k, tt, dt) in SWEEP:
            try:
                # launch-bound (T=64): replayed from a CUDA graph; ms_per_step_eager keeps the per-call figure
                workloads.append(measure_workload(skl, torch, dev, name, di, do, l, k, tt, dt, graph=tt < 4096))
            except Exception as e:  # report, never fake
                workloads.append({"workload": name, "error": str(e)[:200]})
            torch.cuda.empty_cache()
        try:
            workloads.append(measure_stack(skl, torch, dev, world))
        except Exception as e:
            workloads.append({"workload": "c5 stack", "error": str(e)[:200]})
        try:  # the DP schedule's phased backward (two dU launches, RESERVED_SMS left to NCCL), no collective
            skl.set_reserved_sms(RESERVED_SMS)
            workloads.append(measure_workload(skl, torch, dev,
                                              f"c2 bf16, DP-phased backward ({RESERVED_SMS} SMs reserved)",
                                              D_IN, D_OUT, L, K_RANK, T_GPU, "bf16", phased=True))
        finally:
            skl.set_reserved_sms(0)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_reference()
        except Exception as e:  # report, never fake
            cpu = {"value": None, "unit": "tokens/s", "cores": None, "kind": None, "sample": f"failed: {e}"}

    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded Gaussian activations; sketches/U from the reference seed chain)",
            "config": {"workload": WORKLOAD, "d_in": D_IN, "d_out": D_OUT, "num_terms": L, "low_rank": K_RANK,
                       "tokens_per_gpu": T, "global_tokens": world * T,
                       "parallelism": (f"dp{world} (token sharding; NCCL all-reduce of dU1s|db overlapped with "
                                       f"the dX kernel, then dU2s)") if world > 1
                                      else "dp1 (one GPU: fused backward, no collective)",
                       "l2": "inputs larger than L2 (X 50 MB + G 201 MB read, Y 201 MB written per step)"},
            "roofline": roof,
            "step_tflops": step_roof, "step_roofline_frac": step_roof / peak_tf,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
            "kernels": per_kernel,
            "workloads": workloads,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
