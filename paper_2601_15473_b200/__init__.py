"""paper_2601_15473_b200 -- B200-native SKLinear hot path (Panther / pawX).

Python host mirror of the reference's ``rnla::nn::SkLinear`` API
(/root/reference/proj/include/rnla/nn/layers.hpp:52-92) over the C-ABI of
``libskl.so`` (include/skl.h).  PyTorch is used only for device memory and
streams; all arithmetic runs in the sm_100a kernels of ``libskl.so``.  There
is no CPU fallback: importing works anywhere, but every compute call raises
when the library or an sm_100 GPU is missing.

    layer = SkLinear(d_in=768, d_out=3072, num_terms=2, low_rank=128, seed=42)
    y = layer.forward(x)                      # x [T, d_in]   (row convention)
    grads = layer.backward(x, g)              # Grads(grad_x, grad_u1, grad_u2, grad_b)

Naming follows pawX (row convention, [L, d, k] stacks; see include/skl.h for
the exact mapping onto the reference's per-term s1/u1/s2/u2).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

_HERE = os.path.dirname(os.path.abspath(__file__))
# SKL_LIB overrides the library path (A/B timing of two builds); default: in-tree build.
LIB_PATH = os.environ.get("SKL_LIB") or os.path.join(_HERE, "libskl.so")

SKL_OK = 0
STATUS = {0: "SKL_OK", 1: "SKL_ERR_SHAPE", 2: "SKL_ERR_PARAM", 3: "SKL_ERR_CUDA", 4: "SKL_ERR_NCCL",
          5: "SKL_ERR_UNSUPPORTED", 6: "SKL_ERR_WORKSPACE"}
GAUSSIAN, RADEMACHER = 0, 1
F32_TF32, BF16 = 0, 1
OUT_F64, OUT_F32, OUT_BF16 = 0, 1, 2

ABI_SYMBOLS = (
    "skl_version", "skl_last_error", "skl_rng_algorithm", "skl_derive_seed", "skl_params", "skl_exceeds_dense",
    "skl_generate_sketches", "skl_init_params", "skl_realize_sketch", "skl_workspace_size",
    "sketched_linear_forward", "sketched_linear_backward", "skl_allreduce_grads", "skl_launch_count",
    "skl_profile_enable", "skl_profile_collect", "sketched_linear_backward_phase", "skl_set_reserved_sms",
    "sketched_linear_forward_ex", "sketched_linear_backward_ex", "skl_from_dense", "skl_from_dense_workspace_size",
    "skl_conv_workspace_size", "sketched_conv2d_forward", "sketched_conv2d_backward",
    "sketched_linear_forward_bits", "sketched_linear_backward_bits", "skl_relu_bits_row_words",
    "skl_relu_bits_supported", "skl_dense_workspace_size", "skl_dense_init", "dense_linear_forward",
    "dense_linear_backward",
)
BWD_DU1_DB, BWD_DX_DU2, BWD_ALL = 1, 2, 3
FUSE_RELU_OUT, FUSE_RELU_IN, FUSE_RELU_BITS = 1, 2, 4


class SklError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class ShapeError(SklError, ValueError):
    """rnla::shape_error (errors.hpp:10-13)."""


class ParameterError(SklError, ValueError):
    """rnla::parameter_error (errors.hpp:16-19)."""


class LoadError(SklError):
    """rnla::nn::load_error (errors.hpp:40-45): malformed or incompatible model file."""


class _Shape(ctypes.Structure):
    _fields_ = [("d_in", ctypes.c_int64), ("d_out", ctypes.c_int64), ("num_terms", ctypes.c_int64),
                ("low_rank", ctypes.c_int64), ("dtype", ctypes.c_int)]


class _DenseShape(ctypes.Structure):
    _fields_ = [("d_in", ctypes.c_int64), ("d_out", ctypes.c_int64), ("dtype", ctypes.c_int)]


class _ParamCount(ctypes.Structure):
    _fields_ = [("learnable", ctypes.c_uint64), ("total_stored", ctypes.c_uint64),
                ("dense_equivalent", ctypes.c_uint64)]


class _ProfEntry(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 48), ("launches", ctypes.c_uint64), ("total_ms", ctypes.c_double)]


def launch_count() -> int:
    """Kernels launched by libskl in this process (native counter)."""
    return int(lib().skl_launch_count())


def profile_enable(on: bool = True):
    _check(lib().skl_profile_enable(int(on)))


def profile_collect(max_entries: int = 64):
    """-> {kernel name: (launches, total device ms)} since the last collect."""
    buf = (_ProfEntry * max_entries)()
    n = lib().skl_profile_collect(buf, max_entries)
    return {buf[i].name.decode(): (int(buf[i].launches), float(buf[i].total_ms)) for i in range(n)}


_lib = None


def lib() -> ctypes.CDLL:
    """Load libskl.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, u64, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t
    sp = ctypes.POINTER(_Shape)
    for name in ("skl_version", "skl_last_error", "skl_rng_algorithm"):
        getattr(L, name).restype = ctypes.c_char_p
    L.skl_derive_seed.restype = u64
    L.skl_derive_seed.argtypes = [u64, u64]
    L.skl_params.argtypes = [sp, ctypes.POINTER(_ParamCount)]
    L.skl_exceeds_dense.argtypes = [u64] * 4
    L.skl_generate_sketches.argtypes = [sp, ctypes.c_int, u64, vp, vp, vp]
    L.skl_init_params.argtypes = [sp, u64, vp, vp, vp]
    L.skl_realize_sketch.argtypes = [ctypes.c_int, i64, i64, u64, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp]
    L.skl_workspace_size.argtypes = [sp, i64, ctypes.POINTER(sz), ctypes.POINTER(sz)]
    L.sketched_linear_forward.argtypes = [sp, i64] + [vp] * 9 + [sz, vp]
    L.sketched_linear_backward.argtypes = [sp, i64] + [vp] * 12 + [sz, vp]
    L.sketched_linear_backward_phase.argtypes = [sp, i64, ctypes.c_uint] + [vp] * 12 + [sz, vp]
    L.skl_set_reserved_sms.argtypes = [ctypes.c_int]
    L.skl_from_dense_workspace_size.argtypes = [sp, ctypes.POINTER(sz)]
    L.skl_from_dense.argtypes = [sp, ctypes.c_int, u64] + [vp] * 8 + [sz, vp]
    L.sketched_linear_forward_ex.argtypes = [sp, i64, ctypes.c_uint] + [vp] * 9 + [sz, vp]
    L.sketched_linear_backward_ex.argtypes = [sp, i64, ctypes.c_uint, ctypes.c_uint] + [vp] * 12 + [sz, vp]
    L.sketched_linear_forward_bits.argtypes = [sp, i64, ctypes.c_uint] + [vp] * 10 + [sz, vp]
    L.sketched_linear_backward_bits.argtypes = [sp, i64, ctypes.c_uint, ctypes.c_uint] + [vp] * 13 + [sz, vp]
    L.skl_relu_bits_row_words.argtypes = [i64]
    L.skl_relu_bits_supported.argtypes = [sp]
    L.skl_allreduce_grads.argtypes = [vp, vp, sz, vp]
    dp = ctypes.POINTER(_DenseShape)
    L.skl_dense_workspace_size.argtypes = [dp, i64, ctypes.POINTER(sz), ctypes.POINTER(sz)]
    L.skl_dense_init.argtypes = [dp, u64, vp, vp, vp]
    L.dense_linear_forward.argtypes = [dp, i64, ctypes.c_uint] + [vp] * 4 + [vp, sz, vp]
    L.dense_linear_backward.argtypes = [dp, i64, ctypes.c_uint] + [vp] * 6 + [vp, sz, vp]
    L.skl_launch_count.restype = u64
    L.skl_profile_enable.argtypes = [ctypes.c_int]
    L.skl_profile_enable.restype = ctypes.c_int
    L.skl_profile_collect.argtypes = [ctypes.POINTER(_ProfEntry), ctypes.c_int]
    L.skl_profile_collect.restype = ctypes.c_int
    for name in ABI_SYMBOLS:
        if name not in ("skl_version", "skl_last_error", "skl_rng_algorithm", "skl_derive_seed",
                        "skl_exceeds_dense", "skl_launch_count", "skl_relu_bits_row_words"):
            getattr(L, name).restype = ctypes.c_int
    L.skl_relu_bits_row_words.restype = i64
    _lib = L
    return L


def _check(status: int):
    if status == SKL_OK:
        return
    msg = lib().skl_last_error().decode()
    if status == 1:
        raise ShapeError(status, msg)
    if status == 2:
        raise ParameterError(status, msg)
    raise SklError(status, msg)


def derive_seed(master: int, index: int) -> int:
    return int(lib().skl_derive_seed(master, index))


def exceeds_dense(l, k, d_in, d_out) -> bool:
    return bool(lib().skl_exceeds_dense(l, k, d_in, d_out))


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def shape(d_in, d_out, num_terms, low_rank, dtype=BF16) -> _Shape:
    return _Shape(d_in, d_out, num_terms, low_rank, dtype)


def torch_dtype(dtype: int):
    import torch
    return torch.bfloat16 if dtype == BF16 else torch.float32


def workspace_size(s: _Shape, T: int):
    f, b = ctypes.c_size_t(), ctypes.c_size_t()
    _check(lib().skl_workspace_size(ctypes.byref(s), T, ctypes.byref(f), ctypes.byref(b)))
    return f.value, b.value


def params(s: _Shape):
    pc = _ParamCount()
    _check(lib().skl_params(ctypes.byref(s), ctypes.byref(pc)))
    return pc.learnable, pc.total_stored, pc.dense_equivalent


def realize_sketch(dist, k, d, seed, out, unit_variance=False, transpose=False, stream=None):
    """realize_sketch / gaussian_matrix on device into `out` (f64/f32/bf16 tensor)."""
    import torch
    ot = {torch.float64: OUT_F64, torch.float32: OUT_F32, torch.bfloat16: OUT_BF16}[out.dtype]
    _check(lib().skl_realize_sketch(dist, k, d, seed, int(unit_variance), int(transpose), ot, _ptr(out),
                                    _stream(stream)))
    return out


def generate_sketches(s: _Shape, dist, seed, S1s, S2s, stream=None):
    _check(lib().skl_generate_sketches(ctypes.byref(s), dist, seed, _ptr(S1s), _ptr(S2s), _stream(stream)))


def init_params(s: _Shape, seed, U1s, U2s, stream=None):
    _check(lib().skl_init_params(ctypes.byref(s), seed, _ptr(U1s), _ptr(U2s), _stream(stream)))


def _validate(s: _Shape, elem=(), f32=(), device=None):
    """The C-ABI takes raw device pointers: reject what it would misread.  `elem`
    are (name, tensor) pairs in the layer's element type, `f32` fp32 gradients;
    None entries are skipped.  Every tensor must be a contiguous CUDA tensor on
    one device."""
    import torch
    want = torch_dtype(s.dtype)
    for group, dt in ((elem, want), (f32, torch.float32)):
        for name, t in group:
            if t is None:
                continue
            if not isinstance(t, torch.Tensor) or not t.is_cuda:
                raise ParameterError(2, f"{name}: expected a CUDA tensor")
            if t.dtype != dt:
                raise ParameterError(2, f"{name}: dtype {t.dtype}, expected {dt}")
            if not t.is_contiguous():
                raise ParameterError(2, f"{name}: tensor must be contiguous")
            if device is None:
                device = t.device
            elif t.device != device:
                raise ParameterError(2, f"{name}: on {t.device}, expected {device}")


def forward(s: _Shape, x, S1s, S2s, U1s, U2s, bias, y, saved, workspace, stream=None, fuse=0, relu_bits=None):
    """sketched_linear_forward(_ex/_bits): fuse = FUSE_RELU_OUT applies the following ReLU;
    with relu_bits (int32 [T, relu_bits_row_words(d_out)]) it also writes the 1-bit ReLU mask."""
    _validate(s, (("x", x), ("S1s", S1s), ("S2s", S2s), ("U1s", U1s), ("U2s", U2s), ("bias", bias), ("y", y),
                  ("saved", saved)))
    T = x.shape[0]
    if relu_bits is not None:
        _check(lib().sketched_linear_forward_bits(ctypes.byref(s), T, fuse | FUSE_RELU_BITS, _ptr(x), _ptr(S1s),
                                                  _ptr(S2s), _ptr(U1s), _ptr(U2s), _ptr(bias), _ptr(y), _ptr(saved),
                                                  _ptr(relu_bits), _ptr(workspace),
                                                  workspace.numel() if workspace is not None else 0, _stream(stream)))
        return
    _check(lib().sketched_linear_forward_ex(ctypes.byref(s), T, fuse, _ptr(x), _ptr(S1s), _ptr(S2s), _ptr(U1s),
                                            _ptr(U2s), _ptr(bias), _ptr(y), _ptr(saved), _ptr(workspace),
                                            workspace.numel() if workspace is not None else 0, _stream(stream)))


def relu_bits_row_words(width: int) -> int:
    """skl_relu_bits_row_words: int32 words per token of a 1-bit ReLU mask of `width` columns."""
    return int(lib().skl_relu_bits_row_words(int(width)))


def relu_bits_supported(s: _Shape) -> bool:
    """skl_relu_bits_supported: whether this shape's kernels take 1-bit ReLU masks."""
    return bool(lib().skl_relu_bits_supported(ctypes.byref(s)))


def backward(s: _Shape, g, x, saved, S1s, S2s, U1s, U2s, grad_x, dU1s, dU2s, db, workspace, stream=None):
    _validate(s, (("g", g), ("x", x), ("saved", saved), ("S1s", S1s), ("S2s", S2s), ("U1s", U1s), ("U2s", U2s),
                  ("grad_x", grad_x)), (("dU1s", dU1s), ("dU2s", dU2s), ("db", db)))
    T = x.shape[0]
    _check(lib().sketched_linear_backward(ctypes.byref(s), T, _ptr(g), _ptr(x), _ptr(saved), _ptr(S1s), _ptr(S2s),
                                          _ptr(U1s), _ptr(U2s), _ptr(grad_x), _ptr(dU1s), _ptr(dU2s), _ptr(db),
                                          _ptr(workspace), workspace.numel() if workspace is not None else 0,
                                          _stream(stream)))


def backward_phase(s: _Shape, phases, g, x, saved, S1s, S2s, U1s, U2s, grad_x, dU1s, dU2s, db, workspace,
                   stream=None, fuse=0, relu_bits=None):
    """sketched_linear_backward_ex/_bits: phases BWD_DU1_DB (dU1s, db) / BWD_DX_DU2 (grad_x, dU2s) / BWD_ALL;
    fuse = FUSE_RELU_IN masks grad_x by (x > 0) (the preceding ReLU's backward), read from
    relu_bits (the previous layer's 1-bit mask) when given."""
    _validate(s, (("g", g), ("x", x), ("saved", saved), ("S1s", S1s), ("S2s", S2s), ("U1s", U1s), ("U2s", U2s),
                  ("grad_x", grad_x)), (("dU1s", dU1s), ("dU2s", dU2s), ("db", db)))
    T = x.shape[0]
    if relu_bits is not None:
        _check(lib().sketched_linear_backward_bits(ctypes.byref(s), T, phases, fuse | FUSE_RELU_BITS, _ptr(g), _ptr(x),
                                                   _ptr(saved), _ptr(S1s), _ptr(S2s), _ptr(U1s), _ptr(U2s),
                                                   _ptr(grad_x), _ptr(dU1s), _ptr(dU2s), _ptr(db), _ptr(relu_bits),
                                                   _ptr(workspace), workspace.numel() if workspace is not None else 0,
                                                   _stream(stream)))
        return
    _check(lib().sketched_linear_backward_ex(ctypes.byref(s), T, phases, fuse, _ptr(g), _ptr(x), _ptr(saved),
                                             _ptr(S1s), _ptr(S2s), _ptr(U1s), _ptr(U2s), _ptr(grad_x),
                                             _ptr(dU1s), _ptr(dU2s), _ptr(db), _ptr(workspace),
                                             workspace.numel() if workspace is not None else 0,
                                             _stream(stream)))


def set_reserved_sms(n: int):
    """Leave n SMs free for a concurrent NCCL kernel (skl_set_reserved_sms)."""
    _check(lib().skl_set_reserved_sms(int(n)))


@dataclass
class Grads:
    """SkLinear::Grads (layers.hpp:72-78) in ABI layout."""

    grad_x: object   # [T, d_in]
    grad_u1: object  # dU1s [L, k, d_out] fp32
    grad_u2: object  # dU2s [L, d_in, k] fp32
    grad_b: object   # [d_out] fp32


class SkLinear:
    """Device-resident mirror of rnla::nn::SkLinear (layers.hpp:62-81).

    Construction follows sk_linear_fresh (nn_layers.cpp:133-147): sketches from
    derive_seed(seed, 2i / 2i+1), U ~ N(0, 2/(d_in+d_out)) from
    derive_seed(seed, 1000+i), zero bias -- all generated on the GPU.
    """

    def __init__(self, d_in, d_out, num_terms, low_rank, seed=0, dist=GAUSSIAN, dtype=BF16, device="cuda",
                 _fresh=True):
        import torch
        if num_terms < 1 or low_rank < 1:
            raise ParameterError(2, "SkLinear: num_terms and low_rank must be >= 1")
        self.d_in, self.d_out, self.num_terms, self.low_rank = d_in, d_out, num_terms, low_rank
        self.seed, self.dist, self.dtype = seed, dist, dtype
        self.shape = shape(d_in, d_out, num_terms, low_rank, dtype)
        td = torch_dtype(dtype)
        L, k = num_terms, low_rank
        self.S1s = torch.empty(L, d_in, k, dtype=td, device=device)
        self.S2s = torch.empty(L, k, d_out, dtype=td, device=device)
        self.U1s = torch.empty(L, k, d_out, dtype=td, device=device)
        self.U2s = torch.empty(L, d_in, k, dtype=td, device=device)
        self.bias = torch.zeros(d_out, dtype=td, device=device)
        # sketch descriptors in reference order [s1_0, s2_0, s1_1, ...] (dist, rows, cols, seed):
        # what model_save serialises instead of the values (nn_model.cpp:250-265)
        dname = "gaussian" if dist == GAUSSIAN else "rademacher"
        self.sketches = [d for i in range(L) for d in ((dname, k, d_out, derive_seed(seed, 2 * i)),
                                                         (dname, k, d_in, derive_seed(seed, 2 * i + 1)))]
        if _fresh:
            generate_sketches(self.shape, dist, seed, self.S1s, self.S2s)
            init_params(self.shape, seed, self.U1s, self.U2s)
        self._ws = None

    @classmethod
    def from_dense(cls, W, bias, num_terms, low_rank, seed=0, dist=GAUSSIAN, dtype=BF16):
        """sk_linear_from_dense (nn_layers.cpp:149-160), computed on the device:
        W [d_out, d_in] (the reference's DenseLinear::w), bias [d_out] or None."""
        import torch
        d_out, d_in = W.shape
        if bias is not None and bias.numel() != d_out:
            raise ShapeError(1, "sk_linear_from_dense: bias length != d_out")
        lyr = cls(d_in, d_out, num_terms, low_rank, seed=seed, dist=dist, dtype=dtype, device=W.device, _fresh=False)
        td = torch_dtype(dtype)
        Wd = W.to(td).contiguous()
        bd = bias.to(td).contiguous() if bias is not None else None
        n = ctypes.c_size_t()
        _check(lib().skl_from_dense_workspace_size(ctypes.byref(lyr.shape), ctypes.byref(n)))
        ws = torch.empty(n.value, dtype=torch.uint8, device=W.device)
        _check(lib().skl_from_dense(ctypes.byref(lyr.shape), dist, seed, _ptr(Wd), _ptr(bd), _ptr(lyr.S1s),
                                    _ptr(lyr.S2s), _ptr(lyr.U1s), _ptr(lyr.U2s), _ptr(lyr.bias), _ptr(ws), n.value,
                                    _stream(None)))
        return lyr

    @classmethod
    def from_parts(cls, d_in, d_out, num_terms, low_rank, sketches, u1, u2, bias, dtype=BF16, device="cuda"):
        """A layer from sketch DESCRIPTORS plus explicit U / bias in the reference's
        layout (sk_linear_from_json, nn_model.cpp:290-311): the sketches are
        re-realised on the device from (dist, rows, cols, seed) -- bit-identical to
        SketchOp::realized -- and u1 [L][k][d_in], u2 [L][d_out][k] are transposed
        into the U2s / U1s stacks."""
        import numpy as np
        import torch
        L, k = num_terms, low_rank
        if len(sketches) != 2 * L:
            raise ShapeError(1, "SKLinear: expected 2*num_terms sketches")
        lyr = cls(d_in, d_out, L, k, seed=0, dtype=dtype, device=device, _fresh=False)
        for i in range(L):
            for j, (dname, rows, cols, seed) in enumerate(sketches[2 * i: 2 * i + 2]):
                if dname not in ("gaussian", "rademacher"):
                    raise ParameterError(2, f"SKLinear: sketch distribution {dname!r} is not on this path")
                want = d_out if j == 0 else d_in
                if rows != k or cols != want:
                    raise ShapeError(1, f"SKLinear: sketch {2 * i + j} is {rows}x{cols}, expected {k}x{want}")
                dist = GAUSSIAN if dname == "gaussian" else RADEMACHER
                if j == 0:   # s1_i == S2s[i] [k, d_out]
                    realize_sketch(dist, k, d_out, seed, lyr.S2s[i])
                else:        # s2_i == S1s[i]ᵀ  [d_in, k]
                    realize_sketch(dist, k, d_in, seed, lyr.S1s[i], transpose=True)
        lyr.sketches = [tuple(s) for s in sketches]
        td = torch_dtype(dtype)
        u1 = np.asarray(u1, dtype=np.float64).reshape(L, k, d_in)
        u2 = np.asarray(u2, dtype=np.float64).reshape(L, d_out, k)
        lyr.U2s.copy_(torch.from_numpy(np.ascontiguousarray(u1.transpose(0, 2, 1))).to(device=device, dtype=td))
        lyr.U1s.copy_(torch.from_numpy(np.ascontiguousarray(u2.transpose(0, 2, 1))).to(device=device, dtype=td))
        lyr.bias.copy_(torch.from_numpy(np.asarray(bias, dtype=np.float64)).to(device=device, dtype=td))
        return lyr

    def params(self):
        """SkLinear::params -> (learnable, total_stored, dense_equivalent)."""
        return params(self.shape)

    def workspace(self, T):
        import torch
        need = max(workspace_size(self.shape, T))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.S1s.device)
        return self._ws

    def forward(self, x, saved=None):
        import torch
        if x.dim() != 2 or x.shape[1] != self.d_in:
            raise ShapeError(1, "SkLinear::forward: input columns != d_in")
        y = torch.empty(x.shape[0], self.d_out, dtype=x.dtype, device=x.device)
        forward(self.shape, x, self.S1s, self.S2s, self.U1s, self.U2s, self.bias, y, saved,
                self.workspace(x.shape[0]))
        return y

    def backward(self, x, g, saved=None) -> Grads:
        import torch
        if x.shape[1] != self.d_in or g.shape[1] != self.d_out or x.shape[0] != g.shape[0]:
            raise ShapeError(1, "SkLinear::backward: shape mismatch")
        T = x.shape[0]
        dev = x.device
        gx = torch.empty(T, self.d_in, dtype=x.dtype, device=dev)
        du1 = torch.empty(self.num_terms, self.low_rank, self.d_out, dtype=torch.float32, device=dev)
        du2 = torch.empty(self.num_terms, self.d_in, self.low_rank, dtype=torch.float32, device=dev)
        db = torch.empty(self.d_out, dtype=torch.float32, device=dev)
        backward(self.shape, g, x, saved, self.S1s, self.S2s, self.U1s, self.U2s, gx, du1, du2, db,
                 self.workspace(T))
        return Grads(gx, du1, du2, db)


# --------------------------------------------------------------------------- DenseLinear
def dense_shape(d_in, d_out, dtype=BF16) -> _DenseShape:
    return _DenseShape(d_in, d_out, dtype)


def dense_workspace_size(s: _DenseShape, T: int):
    f, b = ctypes.c_size_t(), ctypes.c_size_t()
    _check(lib().skl_dense_workspace_size(ctypes.byref(s), T, ctypes.byref(f), ctypes.byref(b)))
    return f.value, b.value


def dense_forward(s: _DenseShape, x, W, bias, y, workspace, stream=None, fuse=0):
    """dense_linear_forward: y = x·Wᵀ + b (fuse = FUSE_RELU_OUT applies a following ReLU)."""
    _validate(s, (("x", x), ("W", W), ("bias", bias), ("y", y)))
    _check(lib().dense_linear_forward(ctypes.byref(s), x.shape[0], fuse, _ptr(x), _ptr(W), _ptr(bias), _ptr(y),
                                      _ptr(workspace), workspace.numel() if workspace is not None else 0,
                                      _stream(stream)))


def dense_backward(s: _DenseShape, g, x, W, grad_x, dW, db, workspace, stream=None, fuse=0):
    """dense_linear_backward: grad_x = G·W (× (x > 0) with FUSE_RELU_IN), dW = Gᵀ·x, db = Σ_t G."""
    _validate(s, (("g", g), ("x", x), ("W", W), ("grad_x", grad_x)), (("dW", dW), ("db", db)))
    _check(lib().dense_linear_backward(ctypes.byref(s), x.shape[0], fuse, _ptr(g), _ptr(x), _ptr(W), _ptr(grad_x),
                                       _ptr(dW), _ptr(db), _ptr(workspace),
                                       workspace.numel() if workspace is not None else 0, _stream(stream)))


@dataclass
class DenseGrads:
    """DenseLinear::Grads (layers.hpp:42-46), row convention."""

    grad_x: object  # [T, d_in]
    grad_w: object  # [d_out, d_in] fp32
    grad_b: object  # [d_out] fp32


class DenseLinear:
    """Device-resident rnla::nn::DenseLinear (layers.hpp:33-48): W [d_out, d_in]
    (the reference's w), bias [d_out].  Construction follows dense_linear_init
    (nn_layers.cpp:51-59), generated on the GPU from `seed`."""

    def __init__(self, d_in, d_out, seed=0, dtype=BF16, device="cuda", _init=True):
        import torch
        if d_in < 1 or d_out < 1:
            raise ShapeError(1, "DenseLinear: d_in and d_out must be >= 1")
        self.d_in, self.d_out, self.dtype, self.seed = d_in, d_out, dtype, seed
        self.shape = dense_shape(d_in, d_out, dtype)
        td = torch_dtype(dtype)
        self.W = torch.empty(d_out, d_in, dtype=td, device=device)
        self.bias = torch.zeros(d_out, dtype=td, device=device)
        if _init:
            _check(lib().skl_dense_init(ctypes.byref(self.shape), seed, _ptr(self.W), _ptr(self.bias),
                                        _stream(None)))
        self._ws = None

    @classmethod
    def from_parts(cls, w, b, dtype=BF16, device="cuda"):
        """A layer from explicit w [d_out, d_in] and b [d_out] (numpy or torch)."""
        import numpy as np
        import torch
        w = np.asarray(w, dtype=np.float64)
        lyr = cls(w.shape[1], w.shape[0], dtype=dtype, device=device, _init=False)
        td = torch_dtype(dtype)
        lyr.W.copy_(torch.from_numpy(np.ascontiguousarray(w)).to(device=device, dtype=td))
        lyr.bias.copy_(torch.from_numpy(np.asarray(b, dtype=np.float64)).to(device=device, dtype=td))
        return lyr

    def params(self):
        """(learnable, total_stored, dense_equivalent) -- all d_in*d_out + d_out for a dense layer."""
        n = self.d_in * self.d_out + self.d_out
        return n, n, n

    def workspace(self, T):
        import torch
        need = max(dense_workspace_size(self.shape, T))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.W.device)
        return self._ws

    def forward(self, x):
        import torch
        if x.dim() != 2 or x.shape[1] != self.d_in:
            raise ShapeError(1, "DenseLinear::forward: input rows != d_in")
        y = torch.empty(x.shape[0], self.d_out, dtype=x.dtype, device=x.device)
        dense_forward(self.shape, x, self.W, self.bias, y, self.workspace(x.shape[0]))
        return y

    def backward(self, x, g) -> DenseGrads:
        import torch
        if x.shape[1] != self.d_in or g.shape[1] != self.d_out or x.shape[0] != g.shape[0]:
            raise ShapeError(1, "DenseLinear::backward: shape mismatch")
        T = x.shape[0]
        gx = torch.empty(T, self.d_in, dtype=x.dtype, device=x.device)
        dW = torch.empty(self.d_out, self.d_in, dtype=torch.float32, device=x.device)
        db = torch.empty(self.d_out, dtype=torch.float32, device=x.device)
        dense_backward(self.shape, g, x, self.W, gx, dW, db, self.workspace(T))
        return DenseGrads(gx, dW, db)
