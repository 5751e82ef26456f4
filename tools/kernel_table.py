"""Per-kernel device times of one SKLinear fwd+bwd step for a list of shapes,
with each kernel's algorithmic bytes / FLOPs and the fraction of the measured
peaks (MEASURED_PEAKS.json).  Run on a B200:

    python tools/kernel_table.py [c4|c5|c2|all] > table.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_15473_b200 as skl  # noqa: E402

SHAPES = {
    "c2": [("c2 bf16", 768, 3072, 2, 128, 32768, "bf16"), ("c2 tf32", 768, 3072, 2, 128, 32768, "tf32")],
    "c4": [("c4 bf16 L1 k16", 4096, 4096, 1, 16, 131072, "bf16"), ("c4 bf16 L2 k32", 4096, 4096, 2, 32, 131072, "bf16"),
           ("c4 bf16 L4 k64", 4096, 4096, 4, 64, 131072, "bf16"), ("c4 tf32 L1 k16", 4096, 4096, 1, 16, 131072, "tf32"),
           ("c4 tf32 L2 k64", 4096, 4096, 2, 64, 131072, "tf32")],
    "c5": [("c5 proj 768x768 L1 k128", 768, 768, 1, 128, 32768, "bf16"),
           ("c5 FFN1 768->3072 L2 k128", 768, 3072, 2, 128, 32768, "bf16"),
           ("c5 FFN2 3072->768 L2 k128", 3072, 768, 2, 128, 32768, "bf16")],
    "c3": [("c3 bf16 4096 L3 k256", 4096, 4096, 3, 256, 65536, "bf16")],
}


def alg(name, d_in, d_out, Lk, T, e):
    R = 2 * Lk
    if name.startswith("b2b_fwd") or name == "gemm_H":
        return T * (d_in + d_out + Lk) * e, 2 * T * R * (d_in + d_out)
    if name.startswith("b2b_bwd"):
        return T * (d_out + d_in + Lk) * e, 2 * T * R * (d_in + d_out)
    if name.startswith("du"):
        return T * (d_out + d_in + 2 * Lk) * e, 2 * T * Lk * (d_in + d_out)
    return None, None


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    names = list(SHAPES) if which == "all" else which.split(",")
    pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
    bw, tf = pk["hbm_gbs"], pk["bf16_tflops"]
    dev = torch.device("cuda", 0)
    out = []
    for grp in names:
        for (label, d_in, d_out, L, k, T, dt) in SHAPES[grp]:
            kind = skl.BF16 if dt == "bf16" else skl.F32_TF32
            td = skl.torch_dtype(kind)
            e = 2 if dt == "bf16" else 4
            lyr = skl.SkLinear(d_in, d_out, L, k, seed=1, dtype=kind)
            X = torch.randn(T, d_in, device=dev).to(td)
            G = torch.randn(T, d_out, device=dev).to(td)
            sv = torch.empty(L * k, (T + 7) // 8 * 8, dtype=td, device=dev)

            def step():
                lyr.forward(X, saved=sv)
                lyr.backward(X, G, saved=sv)
            for _ in range(5):
                step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 20
            e0.record()
            for _ in range(n):
                step()
            e1.record()
            torch.cuda.synchronize()
            step_us = e0.elapsed_time(e1) / n * 1e3
            skl.profile_enable(True)
            skl.profile_collect()
            for _ in range(n):
                step()
            torch.cuda.synchronize()
            prof = skl.profile_collect()
            skl.profile_enable(False)
            row = {"shape": label, "step_us": round(step_us, 1), "kernels": {}}
            for kn, (cnt, ms) in prof.items():
                us = ms / cnt * 1e3
                b, f = alg(kn, d_in, d_out, L * k, T, e)
                ent = {"us": round(us, 1)}
                if b:
                    ent["alg_GBps"] = round(b / us / 1e3, 1)
                    ent["hbm_frac"] = round(b / us / 1e3 / bw, 3)
                    peak_tf = tf if dt == "bf16" else tf / 2
                    ent["tflops"] = round(f / us / 1e6, 1)
                    ent["tensor_frac"] = round(f / us / 1e6 / peak_tf, 3)
                row["kernels"][kn] = ent
            print(json.dumps(row), flush=True)
            out.append(row)
            del lyr, X, G, sv
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
