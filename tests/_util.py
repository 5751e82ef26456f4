"""Shared helpers for the parity tests (numpy side of the checker)."""
from __future__ import annotations

import json
import os

import numpy as np


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round f64 values to the nearest bfloat16 (ties to even), returned as f64."""
    a = np.asarray(a, dtype=np.float64)
    m, e = np.frexp(a)                 # a = m * 2**e, 0.5 <= |m| < 1
    return np.ldexp(np.rint(m * 256.0) / 256.0, e)   # 8 significant bits


def f32_round(a: np.ndarray) -> np.ndarray:
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def tf32_round(a: np.ndarray) -> np.ndarray:
    """fp32 -> TF32 round-to-nearest (cvt.rna: ties away from zero)."""
    f = np.asarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    f = ((f + 0x1000) & 0xFFFFE000).astype(np.uint32)
    return f.view(np.float32).astype(np.float64)


def rel_fro(approx, exact) -> float:
    approx = np.asarray(approx, dtype=np.float64)
    exact = np.asarray(exact, dtype=np.float64)
    ref = np.linalg.norm(exact)
    return float(np.linalg.norm(approx - exact) / (ref if ref > 0 else 1.0))


def max_abs_rel(approx, exact) -> float:
    """max |approx - exact| / max |exact|."""
    approx = np.asarray(approx, dtype=np.float64)
    exact = np.asarray(exact, dtype=np.float64)
    den = np.max(np.abs(exact))
    return float(np.max(np.abs(approx - exact)) / (den if den > 0 else 1.0))


# Tolerance gates vs the f64 oracle on identical (already rounded) inputs,
# BASELINE.md §5 / SURVEY.md §8(c).
GATES = {
    "bf16": dict(rel_fro=1e-2, max_abs=2e-2),
    "tf32": dict(rel_fro=2e-3, max_abs=2e-3),
}


# Regression bounds: about 2x the rel_fro the kernels measure on the parity
# shapes (per output, from a GPU run with SKL_PARITY_LOG set:
# tests/golden/parity_errors_r2.json).  Far inside the gates above, so a
# numerics regression that stays within tolerance -- e.g. truncating H to bf16
# / TF32 instead of rounding to nearest -- still fails.  Applied with
# check_close(..., regress=True).
REGRESS = {
    "bf16": {"y": 4.1e-3, "saved": 3.4e-3, "grad_x": 4.8e-3, "dU": 3.5e-3, "db": 1e-6},
    "tf32": {"y": 8e-4, "saved": 8e-4, "grad_x": 1.2e-3, "dU": 1.7e-3, "db": 1e-6},
}


def _kind(name: str) -> str:
    n = name.lower()
    for key, kind in (("grad_x", "grad_x"), ("du1", "dU"), ("du2", "dU"), ("saved", "saved"), ("db", "db")):
        if key in n:
            return kind
    return "y"


def check_close(name, approx, exact, variant="bf16", regress=False):
    g = GATES[variant]
    rf, ma = rel_fro(approx, exact), max_abs_rel(approx, exact)
    log = os.environ.get("SKL_PARITY_LOG")
    if log:
        with open(log, "a") as f:
            f.write(json.dumps({"test": os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0], "name": name,
                                "variant": variant, "rel_fro": rf, "max_abs": ma}) + "\n")
    assert rf <= g["rel_fro"] and ma <= g["max_abs"], (
        f"{name}: rel_fro={rf:.3e} (gate {g['rel_fro']:.0e}), max_abs/max|ref|={ma:.3e} (gate {g['max_abs']:.0e})")
    if regress:
        bound = REGRESS[variant][_kind(name)]
        assert rf <= bound, f"{name}: rel_fro={rf:.3e} above the regression bound {bound:.1e}"
    return rf, ma
