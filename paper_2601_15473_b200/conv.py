"""SkConv2d on the device: im2col lowering onto the SKLinear path.

Mirror of rnla::nn::SkConv2d (layers.hpp:94-158, nn_layers.cpp:176-314) over
the C-ABI sketched_conv2d_forward / _backward: NCHW images, the inner
SKLinear has d_in = c_in*kh*kw and d_out = c_out, the B*oh*ow patches of a
batch are its tokens.  Construction follows sk_conv2d_fresh
(nn_layers.cpp:316-322): the inner layer is sk_linear_fresh(c_in*kh*kw,
c_out, l, k, seed).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import BF16, GAUSSIAN, Grads, ShapeError, SkLinear, _check, _ptr, _Shape, _stream, lib


class _ConvShape(ctypes.Structure):
    _fields_ = [("c_in", ctypes.c_int64), ("c_out", ctypes.c_int64), ("kernel_h", ctypes.c_int64),
                ("kernel_w", ctypes.c_int64), ("stride", ctypes.c_int64), ("padding", ctypes.c_int64)]


@dataclass(frozen=True)
class ConvShape:
    """rnla::nn::ConvShape (layers.hpp:96-107)."""

    c_in: int
    c_out: int
    kernel_h: int
    kernel_w: int
    stride: int = 1
    padding: int = 0

    def lowered_d_in(self):
        return self.c_in * self.kernel_h * self.kernel_w

    def out_h(self, h):
        if h + 2 * self.padding < self.kernel_h:
            raise ShapeError(1, "conv: kernel taller than padded image")
        return (h + 2 * self.padding - self.kernel_h) // self.stride + 1

    def out_w(self, w):
        if w + 2 * self.padding < self.kernel_w:
            raise ShapeError(1, "conv: kernel wider than padded image")
        return (w + 2 * self.padding - self.kernel_w) // self.stride + 1

    def _c(self):
        return _ConvShape(self.c_in, self.c_out, self.kernel_h, self.kernel_w, self.stride, self.padding)


def _bind():
    L = lib()
    if getattr(L, "_conv_bound", False):
        return L
    vp, i64, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t
    sp = ctypes.POINTER(_Shape)
    cp = ctypes.POINTER(_ConvShape)
    L.skl_conv_workspace_size.argtypes = [sp, cp, i64, i64, i64, ctypes.POINTER(sz), ctypes.POINTER(sz)]
    L.skl_conv_workspace_size.restype = ctypes.c_int
    L.sketched_conv2d_forward.argtypes = [sp, cp, i64, i64, i64, ctypes.c_uint] + [vp] * 10 + [sz, vp]
    L.sketched_conv2d_forward.restype = ctypes.c_int
    L.sketched_conv2d_backward.argtypes = [sp, cp, i64, i64, i64] + [vp] * 13 + [sz, vp]
    L.sketched_conv2d_backward.restype = ctypes.c_int
    L._conv_bound = True
    return L


class SkConv2d:
    """Device-resident rnla::nn::SkConv2d."""

    def __init__(self, shape: ConvShape, num_terms, low_rank, seed=0, dist=GAUSSIAN, dtype=BF16, device="cuda",
                 inner: SkLinear | None = None):
        self.shape = shape
        self.inner = inner or SkLinear(shape.lowered_d_in(), shape.c_out, num_terms, low_rank, seed=seed, dist=dist,
                                       dtype=dtype, device=device)
        if self.inner.d_in != shape.lowered_d_in() or self.inner.d_out != shape.c_out:
            raise ShapeError(1, "SKConv2d: inner dims disagree with conv shape")
        self._ws = None

    def _workspace(self, B, H, W):
        import torch
        L = _bind()
        f, b = ctypes.c_size_t(), ctypes.c_size_t()
        _check(L.skl_conv_workspace_size(ctypes.byref(self.inner.shape), ctypes.byref(self.shape._c()), B, H, W,
                                         ctypes.byref(f), ctypes.byref(b)))
        need = max(f.value, b.value)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.inner.S1s.device)
        return self._ws

    def forward(self, x, keep=None, fuse=0):
        """SkConv2d::forward: x [B, c_in, H, W] -> y [B, c_out, oh, ow].  keep: optional
        dict receiving the patch matrix and saved projection for backward()."""
        import torch
        B, C, H, W = x.shape
        if C != self.shape.c_in:
            raise ShapeError(1, "conv forward: channel count mismatch")
        oh, ow = self.shape.out_h(H), self.shape.out_w(W)
        y = torch.empty(B, self.shape.c_out, oh, ow, dtype=x.dtype, device=x.device)
        cols = saved = None
        if keep is not None:
            T = B * oh * ow
            cols = torch.empty(T, self.inner.d_in, dtype=x.dtype, device=x.device)
            saved = torch.empty(self.inner.num_terms * self.inner.low_rank, (T + 7) // 8 * 8, dtype=x.dtype,
                                device=x.device)
            keep.update(cols=cols, saved=saved)
        ws = self._workspace(B, H, W)
        L, s = _bind(), self.inner
        _check(L.sketched_conv2d_forward(ctypes.byref(s.shape), ctypes.byref(self.shape._c()), B, H, W, fuse, _ptr(x),
                                         _ptr(s.S1s), _ptr(s.S2s), _ptr(s.U1s), _ptr(s.U2s), _ptr(s.bias), _ptr(y),
                                         _ptr(cols), _ptr(saved), _ptr(ws), ws.numel(), _stream(None)))
        return y

    def backward(self, x, g, keep=None) -> Grads:
        """SkConv2d::backward -> Grads(grad_x [B,c_in,H,W], dU1s, dU2s, db)."""
        import torch
        B, C, H, W = x.shape
        s = self.inner
        gx = torch.empty_like(x)
        du1 = torch.empty(s.num_terms, s.low_rank, s.d_out, dtype=torch.float32, device=x.device)
        du2 = torch.empty(s.num_terms, s.d_in, s.low_rank, dtype=torch.float32, device=x.device)
        db = torch.empty(s.d_out, dtype=torch.float32, device=x.device)
        keep = keep or {}
        ws = self._workspace(B, H, W)
        _check(_bind().sketched_conv2d_backward(
            ctypes.byref(s.shape), ctypes.byref(self.shape._c()), B, H, W, _ptr(g), _ptr(x), _ptr(keep.get("cols")),
            _ptr(keep.get("saved")), _ptr(s.S1s), _ptr(s.S2s), _ptr(s.U1s), _ptr(s.U2s), _ptr(gx), _ptr(du1),
            _ptr(du2), _ptr(db), _ptr(ws), ws.numel(), _stream(None)))
        return Grads(gx, du1, du2, db)
