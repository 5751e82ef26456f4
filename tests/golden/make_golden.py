#!/usr/bin/env python3
"""Generate tests/golden/*.json from the REFERENCE implementation itself.

Runs the unmodified reference sources compiled by oracle/Makefile into
oracle/_ref/librnla_ref.so (never the C restatement), so the fixtures pin
the restatement and the device kernels to the reference's own outputs.
Values are stored as C99 hex floats (exact).  Regenerate with

    make -C oracle && python tests/golden/make_golden.py

Pinned reference behaviour:
  * Splitmix64 golden u64s            test_sketch.cpp:25-33
  * derive_seed / sketches / U init   rng.hpp:66-69, sketch.cpp:34-49, nn_layers.cpp:133-147
  * SkLinear forward / backward       nn_layers.cpp:61-101
  * SURVEY.md Appendix A known-answer values (c1 shape, seed 42)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402


def hx(a):
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel()]


def main():
    ref = oracle.Oracle("reference")
    out = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref/librnla_ref.so (reference sources)",
           "rng_algorithm": ref.lib.ref_rng_algorithm().decode()}
    out["splitmix64"] = {str(s): [f"{int(v):016x}" for v in ref.splitmix64_stream(s, 8)] for s in (0, 42, 2**64 - 1)}
    out["derive_seed"] = {f"{m},{i}": f"{ref.derive_seed(m, i):016x}"
                          for m in (0, 42, 12345) for i in (0, 1, 2, 3, 7, 9, 11, 1000, 1001)}
    out["gaussian_stream"] = {str(s): hx(ref.gaussian_stream(s, 9)) for s in (7, 42)}
    sk = []
    for dist, k, d, seed in [(0, 4, 10, 7), (0, 3, 7, 42), (1, 4, 10, 7), (1, 2, 3, 123), (0, 64, 1024, 42)]:
        m = ref.realize_sketch(dist, k, d, seed)
        sk.append({"dist": dist, "k": k, "d": d, "seed": seed, "head": hx(m.ravel()[:24]),
                   "tail": hx(m.ravel()[-8:]), "sum": float(m.sum()).hex()})
    out["sketches"] = sk
    # small full layer (SURVEY §0.3 algebra-check shape)
    d_in, d_out, L, k, T = 37, 53, 3, 5, 11
    p = ref.sk_linear_fresh(d_in, d_out, L, k, 42)
    x = ref.gaussian_matrix(d_in, T, ref.derive_seed(42, 7))
    g = ref.gaussian_matrix(d_out, T, ref.derive_seed(42, 9))
    b = ref.gaussian_matrix(1, d_out, ref.derive_seed(42, 11))[0]
    y = ref.forward(p, b, x)
    gx, gu1, gu2, gb = ref.backward(p, x, g)
    out["layer_small"] = {"d_in": d_in, "d_out": d_out, "L": L, "k": k, "T": T, "seed": 42,
                          "s1": hx(p.s1), "u1": hx(p.u1), "s2": hx(p.s2), "u2": hx(p.u2), "x": hx(x), "g": hx(g),
                          "b": hx(b), "y": hx(y), "grad_x": hx(gx), "grad_u1": hx(gu1), "grad_u2": hx(gu2),
                          "grad_b": hx(gb)}
    # c1 shape, seed 42, x = gaussian_matrix(1024,64,7), G = (..,9), zero bias
    p = ref.sk_linear_fresh(1024, 1024, 1, 64, 42)
    x = ref.gaussian_matrix(1024, 64, 7)
    g = ref.gaussian_matrix(1024, 64, 9)
    y = ref.forward(p, np.zeros(1024), x)
    gx, gu1, gu2, gb = ref.backward(p, x, g)
    out["kat_c1"] = {"s1_row0": hx(p.s1[0, 0, :4]), "s2_row0": hx(p.s2[0, 0, :4]), "u1_00_01": hx(p.u1[0, 0, :2]),
                     "u2_00_01": hx(p.u2[0, 0, :2]), "u2_last": float(p.u2[0, -1, -1]).hex(),
                     "y_0_0": float(y[0, 0]).hex(), "y_1023_63": float(y[1023, 63]).hex(),
                     "sum_y": float(np.sum(y)).hex(), "sum_abs_y": float(np.sum(np.abs(y))).hex(),
                     "grad_x_0_0": float(gx[0, 0]).hex(), "grad_u1_0_0_0": float(gu1[0, 0, 0]).hex(),
                     "grad_u2_0_0_0": float(gu2[0, 0, 0]).hex(), "grad_b_0": float(gb[0]).hex()}
    path = os.path.join(HERE, "reference_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
