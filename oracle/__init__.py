"""oracle -- CPU parity checker for the B200 SKLinear hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package, and only as the checker / the timed reference arm, never as the
thing measured or shipped.  The product (``paper_2601_15473_b200``) never
imports it and has no CPU fallback.

Two interchangeable back ends with the same numpy API:

* ``kind="port"``      -- ``liboracle.so``: ``skl_oracle.c``, a plain-C f64
  restatement of the reference algorithm (every function cites the reference
  file:line it follows);
* ``kind="reference"`` -- ``_ref/librnla_ref.so``: the unmodified reference
  sources (/root/reference/proj/src) compiled by ``oracle/Makefile`` plus the
  thin ``ref_shim.cpp`` adapter.

Pinning: tests/test_oracle.py checks the port bit-for-bit against the
reference library and both against the reference's golden u64s
(test_sketch.cpp:25-33) and the known-answer values in tests/golden/.

Layout helpers convert between the reference's column convention / per-term
matrices (layers.hpp:52-81) and the pawX row convention / ``[L, d, k]``
stacks exported at the C-ABI (include/skl.h):

    S1s[i] = s2_iᵀ  [d_in, k]      U2s[i] = u1_iᵀ  [d_in, k]
    U1s[i] = u2_iᵀ  [k, d_out]     S2s[i] = s1_i   [k, d_out]
    dU1s[i] = grad_u2_iᵀ           dU2s[i] = grad_u1_iᵀ
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_u64 = ctypes.c_uint64
_dp = ctypes.POINTER(ctypes.c_double)
_up = ctypes.POINTER(ctypes.c_uint64)

GAUSSIAN = 0
RADEMACHER = 1


class OracleError(RuntimeError):
    pass


class ShapeError(OracleError):
    """Mirror of rnla::shape_error (errors.hpp:10-13)."""


class ParameterError(OracleError):
    """Mirror of rnla::parameter_error (errors.hpp:16-19)."""


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _lib_path(kind: str) -> str:
    if kind == "port":
        return os.path.join(_HERE, "liboracle.so")
    if kind == "reference":
        return os.path.join(_HERE, "_ref", "librnla_ref.so")
    raise ValueError(kind)


def available(kind: str) -> bool:
    return os.path.exists(_lib_path(kind))


@dataclass
class Params:
    """Reference-layout SKLinear parameters (f64, column convention)."""

    d_in: int
    d_out: int
    l: int
    k: int
    s1: np.ndarray  # [l, k, d_out]
    u1: np.ndarray  # [l, k, d_in]
    s2: np.ndarray  # [l, k, d_in]
    u2: np.ndarray  # [l, d_out, k]


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = _lib_path(kind)
        if not os.path.exists(path):
            raise OracleError(f"oracle library {path} not built (run `make -C oracle`)")
        self.lib = lib = ctypes.CDLL(path)
        pre = "orc_" if kind == "port" else "ref_"
        self._pre = pre
        f = lambda n: getattr(lib, pre + n)
        f("derive_seed").restype = _u64
        f("derive_seed").argtypes = [_u64, _u64]
        f("splitmix64_stream").argtypes = [_u64, _u64, _up]
        f("gaussian_stream").argtypes = [_u64, _u64, _dp]
        f("realize_sketch").argtypes = [ctypes.c_int, _u64, _u64, _u64, _dp]
        f("sk_linear_fresh").argtypes = [_u64, _u64, _u64, _u64, _u64, ctypes.c_int, _dp, _dp, _dp, _dp]
        f("sk_forward").argtypes = [_u64] * 5 + [_dp] * 7
        f("sk_backward").argtypes = [_u64] * 5 + [_dp] * 10
        if kind == "reference":
            lib.ref_last_error.restype = ctypes.c_char_p
            lib.ref_rng_algorithm.restype = ctypes.c_char_p
            lib.ref_time_fwd_bwd.argtypes = [_u64] * 6 + [ctypes.c_int, _u64, _u64, _dp, _dp]
            lib.ref_sk_forward_checked.argtypes = [_u64] * 6
            lib.ref_gaussian_matrix.argtypes = [_u64, _u64, _u64, _dp]
        else:
            lib.orc_gaussian_matrix.argtypes = [_u64, _u64, _u64, _dp]
            lib.orc_exceeds_dense.argtypes = [_u64] * 4
            lib.orc_sk_stored_coeffs.argtypes = [_u64] * 4
            lib.orc_sk_stored_coeffs.restype = _u64

    # -- error mapping (errors.hpp) --------------------------------------
    def _check(self, rc: int, what: str):
        if rc == 0:
            return
        msg = what
        if self.kind == "reference":
            msg = f"{what}: {self.lib.ref_last_error().decode()}"
        if rc == 1:
            raise ShapeError(msg)
        if rc == 2:
            raise ParameterError(msg)
        raise OracleError(f"{msg} (rc={rc})")

    def _fn(self, name):
        return getattr(self.lib, self._pre + name)

    # -- rng.hpp ----------------------------------------------------------
    def derive_seed(self, master: int, index: int) -> int:
        return int(self._fn("derive_seed")(master, index))

    def splitmix64_stream(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        self._fn("splitmix64_stream")(seed, n, out.ctypes.data_as(_up))
        return out

    def gaussian_stream(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self._fn("gaussian_stream")(seed, n, _p(out))
        return out

    # -- sketch.cpp -------------------------------------------------------
    def realize_sketch(self, dist: int, k: int, d: int, seed: int) -> np.ndarray:
        out = np.empty((k, d), dtype=np.float64)
        self._check(self._fn("realize_sketch")(dist, k, d, seed, _p(out)), "realize_sketch")
        return out

    def gaussian_matrix(self, rows: int, cols: int, seed: int) -> np.ndarray:
        out = np.empty((rows, cols), dtype=np.float64)
        rc = self._fn("gaussian_matrix")(rows, cols, seed, _p(out))
        if self.kind == "reference":
            self._check(rc, "gaussian_matrix")
        return out

    # -- nn_layers.cpp ----------------------------------------------------
    def sk_linear_fresh(self, d_in, d_out, l, k, seed, dist=GAUSSIAN) -> Params:
        s1 = np.empty((max(l, 1), max(k, 1), d_out))
        u1 = np.empty((max(l, 1), max(k, 1), d_in))
        s2 = np.empty((max(l, 1), max(k, 1), d_in))
        u2 = np.empty((max(l, 1), d_out, max(k, 1)))
        rc = self._fn("sk_linear_fresh")(d_in, d_out, l, k, seed, dist, _p(s1), _p(u1), _p(s2), _p(u2))
        self._check(rc, "sk_linear_fresh")
        return Params(d_in, d_out, l, k, s1, u1, s2, u2)

    def forward(self, p: Params, bias: np.ndarray, x: np.ndarray) -> np.ndarray:
        """SkLinear::forward, column convention: x [d_in, T] -> y [d_out, T]."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape[0] != p.d_in:
            raise ShapeError("SkLinear::forward: input rows != d_in")
        T = x.shape[1]
        y = np.empty((p.d_out, T))
        b = np.ascontiguousarray(bias, dtype=np.float64)
        rc = self._fn("sk_forward")(p.d_in, p.d_out, p.l, p.k, T, _p(p.s1), _p(p.u1), _p(p.s2), _p(p.u2),
                                    _p(b), _p(x), _p(y))
        self._check(rc, "sk_forward")
        return y

    def backward(self, p: Params, x: np.ndarray, g: np.ndarray):
        """SkLinear::backward -> (grad_x [d_in,T], grad_u1 [l,k,d_in], grad_u2 [l,d_out,k], grad_b [d_out])."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        g = np.ascontiguousarray(g, dtype=np.float64)
        if x.shape[0] != p.d_in or g.shape[0] != p.d_out or x.shape[1] != g.shape[1]:
            raise ShapeError("SkLinear::backward: shape mismatch")
        T = x.shape[1]
        gx = np.empty((p.d_in, T))
        gu1 = np.empty_like(p.u1)
        gu2 = np.empty_like(p.u2)
        gb = np.empty(p.d_out)
        rc = self._fn("sk_backward")(p.d_in, p.d_out, p.l, p.k, T, _p(p.s1), _p(p.u1), _p(p.s2), _p(p.u2),
                                     _p(x), _p(g), _p(gx), _p(gu1), _p(gu2), _p(gb))
        self._check(rc, "sk_backward")
        return gx, gu1, gu2, gb

    # -- DenseLinear (nn_layers.cpp:32-59) ------------------------------------
    def _dense_fn(self, name, argtypes):
        f = self._fn(name)
        f.argtypes = argtypes
        return f

    def dense_init(self, d_in, d_out, seed):
        """dense_linear_init -> (w [d_out, d_in], b [d_out])."""
        w, b = np.empty((d_out, d_in)), np.empty(d_out)
        rc = self._dense_fn("dense_init", [_u64] * 3 + [_dp] * 2)(d_in, d_out, seed, _p(w), _p(b))
        if self.kind == "reference":
            self._check(rc, "dense_init")
        return w, b

    def dense_forward(self, w, b, x):
        """DenseLinear::forward, column convention: x [d_in, T] -> y [d_out, T]."""
        w = np.ascontiguousarray(w, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        d_out, d_in = w.shape
        if x.shape[0] != d_in:
            raise ShapeError("DenseLinear::forward: input rows != d_in")
        y = np.empty((d_out, x.shape[1]))
        rc = self._dense_fn("dense_forward", [_u64] * 3 + [_dp] * 4)(d_in, d_out, x.shape[1], _p(w), _p(b), _p(x),
                                                                      _p(y))
        self._check(rc, "dense_forward")
        return y

    def dense_backward(self, w, x, g):
        """DenseLinear::backward -> (grad_x [d_in, T], grad_w [d_out, d_in], grad_b [d_out])."""
        w = np.ascontiguousarray(w, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        g = np.ascontiguousarray(g, dtype=np.float64)
        d_out, d_in = w.shape
        if x.shape[0] != d_in or g.shape[0] != d_out or x.shape[1] != g.shape[1]:
            raise ShapeError("DenseLinear::backward: shape mismatch")
        T = x.shape[1]
        gx, gw, gb = np.empty((d_in, T)), np.empty((d_out, d_in)), np.empty(d_out)
        rc = self._dense_fn("dense_backward", [_u64] * 3 + [_dp] * 6)(d_in, d_out, T, _p(w), _p(x), _p(g), _p(gx),
                                                                       _p(gw), _p(gb))
        self._check(rc, "dense_backward")
        return gx, gw, gb

    # -- reference-only -----------------------------------------------------
    def time_fwd_bwd(self, d_in, d_out, l, k, T, seed=42, threads=1, trials=3, warmup=1):
        """Reference SkLinear fwd+bwd timed by bench::time_op (ms mean, ms std)."""
        if self.kind != "reference":
            raise OracleError("time_fwd_bwd needs the reference library")
        m = ctypes.c_double()
        s = ctypes.c_double()
        rc = self.lib.ref_time_fwd_bwd(d_in, d_out, l, k, T, seed, threads, trials, warmup,
                                       ctypes.byref(m), ctypes.byref(s))
        self._check(rc, "time_fwd_bwd")
        return m.value, s.value


# ---------------------------------------------------------------------------
# Layout helpers: reference (column convention, per-term) <-> ABI (row
# convention, pawX [L, d, k] stacks).  Pure data movement, exact.
# ---------------------------------------------------------------------------
def sk_linear_from_dense(o: "Oracle", W: np.ndarray, l: int, k: int, seed: int, dist: int = GAUSSIAN) -> Params:
    """sk_linear_from_dense (nn_layers.cpp:149-160): sketches seeded like
    sk_linear_shell (:124-127), u1_i = s1_i·W [k, d_in], u2_i = W·s2_iᵀ
    [d_out, k] (f64 matmul; the reference's gemm_rows order is irrelevant at f64
    against the bf16/TF32 gates)."""
    d_out, d_in = W.shape
    p = o.sk_linear_fresh(d_in, d_out, l, k, seed, dist)   # same sketches; U replaced below
    u1 = np.stack([p.s1[i] @ W for i in range(l)])
    u2 = np.stack([W @ p.s2[i].T for i in range(l)])
    return Params(d_in, d_out, l, k, p.s1, u1, p.s2, u2)


def skconv_forward(ref: "Oracle", geo, p: Params, bias, x):
    """The REFERENCE's SkConv2d::forward (nn_layers.cpp:226-244, via oracle/_ref)
    on explicit parameters.  geo = (c_in, c_out, kh, kw, stride, padding); x NCHW."""
    B, C, H, W = x.shape
    c_in, c_out, kh, kw, st, pad = geo
    oh, ow = (H + 2 * pad - kh) // st + 1, (W + 2 * pad - kw) // st + 1
    y = np.empty((B, c_out, oh, ow))
    g = np.array(geo, dtype=np.uint64)
    f = ref.lib.ref_skconv_forward
    f.argtypes = [_up, _u64, _u64] + [_dp] * 5 + [_u64] * 3 + [_dp, _dp]
    ref._check(f(g.ctypes.data_as(_up), p.l, p.k, _p(p.s1), _p(p.u1), _p(p.s2), _p(p.u2), _p(np.ascontiguousarray(bias)),
                 B, H, W, _p(np.ascontiguousarray(x)), _p(y)), "skconv_forward")
    return y


def skconv_backward(ref: "Oracle", geo, p: Params, x, g):
    """The REFERENCE's SkConv2d::backward (nn_layers.cpp:280-314) -> (grad_x, gu1, gu2, gb)."""
    B, C, H, W = x.shape
    gx = np.empty_like(x)
    gu1 = np.empty((p.l, p.k, p.d_in))
    gu2 = np.empty((p.l, p.d_out, p.k))
    gb = np.empty(p.d_out)
    geo_a = np.array(geo, dtype=np.uint64)
    f = ref.lib.ref_skconv_backward
    f.argtypes = [_up, _u64, _u64] + [_dp] * 4 + [_u64] * 3 + [_dp] * 6
    ref._check(f(geo_a.ctypes.data_as(_up), p.l, p.k, _p(p.s1), _p(p.u1), _p(p.s2), _p(p.u2), B, H, W,
                 _p(np.ascontiguousarray(x)), _p(np.ascontiguousarray(g)), _p(gx), _p(gu1), _p(gu2), _p(gb)),
               "skconv_backward")
    return gx, gu1, gu2, gb


def to_abi(p: Params):
    """-> dict(S1s [L,d_in,k], U1s [L,k,d_out], U2s [L,d_in,k], S2s [L,k,d_out])."""
    return dict(
        S1s=np.ascontiguousarray(p.s2.transpose(0, 2, 1)),
        U1s=np.ascontiguousarray(p.u2.transpose(0, 2, 1)),
        U2s=np.ascontiguousarray(p.u1.transpose(0, 2, 1)),
        S2s=np.ascontiguousarray(p.s1),
    )


def from_abi(d_in, d_out, S1s, U1s, U2s, S2s) -> Params:
    L, _, k = S1s.shape
    return Params(d_in, d_out, L, k,
                  s1=np.ascontiguousarray(S2s, dtype=np.float64),
                  u1=np.ascontiguousarray(U2s.transpose(0, 2, 1), dtype=np.float64),
                  s2=np.ascontiguousarray(S1s.transpose(0, 2, 1), dtype=np.float64),
                  u2=np.ascontiguousarray(U1s.transpose(0, 2, 1), dtype=np.float64))


def grads_to_abi(gx, gu1, gu2, gb):
    """Reference grads -> (dX [T,d_in], dU1s [L,k,d_out], dU2s [L,d_in,k], db [d_out])."""
    return (np.ascontiguousarray(gx.T), np.ascontiguousarray(gu2.transpose(0, 2, 1)),
            np.ascontiguousarray(gu1.transpose(0, 2, 1)), gb.copy())


def inputs(d_in, d_out, T, seed=42, oracle: Oracle | None = None):
    """BASELINE.md §3 inputs: x, G, bias from derive_seed(seed, 7/9/11) (column convention)."""
    o = oracle or Oracle("port")
    x = o.gaussian_matrix(d_in, T, o.derive_seed(seed, 7))
    g = o.gaussian_matrix(d_out, T, o.derive_seed(seed, 9))
    b = o.gaussian_matrix(1, d_out, o.derive_seed(seed, 11))[0]
    return x, g, b
