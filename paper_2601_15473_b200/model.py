"""Linear/ReLU chains of SKLinear layers on the device.

Mirror of the reference's model container for this path:
    model_forward(model, x): Linear/SKLinear/ReLU layers applied in order
                                               nn_model.cpp:111-122
    Relu::forward / Relu::backward           nn_layers.cpp:341-354

Every ReLU is fused into its neighbours instead of running as a kernel:
the forward applies it in the epilogue of the SKLinear it follows
(SKL_FUSE_RELU_OUT), and the backward applies its mask in the dX epilogue of
the SKLinear it feeds (SKL_FUSE_RELU_IN: grad *= (x > 0), x being that
layer's input = the ReLU's output, positive exactly where the ReLU's input
was).  A chain therefore launches only the SKLinear kernels.

Data-parallel training (token sharding): `backward(...,
buckets=...)` all-reduces each layer's dU1s | db bucket asynchronously as soon
as its phase-1 kernel has run and its dU2s after phase 2, so every
collective overlaps the backward of the layers below it; the caller waits on
the returned works (or `wait_all`) before the optimizer step.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import (BF16, BWD_ALL, BWD_DU1_DB, BWD_DX_DU2, FUSE_RELU_IN, FUSE_RELU_OUT, DenseLinear, ShapeError,
               SkLinear, SklError, backward_phase, dense_backward, dense_forward, dense_workspace_size, forward,
               relu_bits_row_words, relu_bits_supported, torch_dtype, workspace_size)


class Relu:
    """ReLU layer of a chain (Relu, layers.hpp; nn_layers.cpp:341-354) -- always fused."""

    def __repr__(self):
        return "Relu()"


@dataclass
class _Step:
    layer: object           # SkLinear or DenseLinear
    relu_out: bool          # a ReLU follows (fused into this layer's forward epilogue)
    relu_in: bool = False   # the input came out of a ReLU (its mask is fused into this layer's dX)
    x: object = None        # saved input (needed by the backward: dU2s, the ReLU mask)
    saved: object = None    # saved projection x·S1 [L*k][round8(T)]
    bits: object = None     # relu_in: the 1-bit ReLU mask of x written by the previous layer's forward


@dataclass
class ChainGrads:
    """Per-SKLinear-layer gradients (chain order) and the input gradient."""

    grad_x: object
    layers: list = field(default_factory=list)  # GradBucket per SKLinear layer


class SkChain:
    """model_forward over a list of SkLinear / DenseLinear / Relu layers, with a training backward."""

    def __init__(self, layers, relu_bits=True):
        """relu_bits: carry each fused ReLU's mask from the forward to the next
        layer's backward as 1 bit per element (skl.h SKL_FUSE_RELU_BITS) where both
        layers' kernels support it, instead of re-reading the ReLU output."""
        layers = list(layers)
        self._layers = layers
        self.relu_bits = relu_bits
        if not layers or not isinstance(layers[0], (SkLinear, DenseLinear)):
            raise ShapeError(1, "SkChain: a chain starts with a Linear / SKLinear layer (a leading ReLU has no "
                                "producing layer to fuse into)")
        self.steps: list[_Step] = []
        prev_relu = False
        for i, lyr in enumerate(layers):
            if isinstance(lyr, Relu):
                if prev_relu:
                    continue  # ReLU∘ReLU == ReLU
                self.steps[-1].relu_out = True
                prev_relu = True
                continue
            if not isinstance(lyr, (SkLinear, DenseLinear)):  # nn_model.cpp:117-119
                raise ShapeError(1, f"model_forward: layer {i} is not part of a Linear/ReLU chain")
            if self.steps and self.steps[-1].layer.d_out != lyr.d_in:
                raise ShapeError(1, f"SkChain: layer {i} d_in={lyr.d_in} != previous d_out="
                                    f"{self.steps[-1].layer.d_out}")
            if self.steps and self.steps[-1].layer.dtype != lyr.dtype:
                raise SklError(5, "SkChain: all layers must share one element type")
            self.steps.append(_Step(lyr, relu_out=False, relu_in=prev_relu))
            prev_relu = False
        self.dtype = self.steps[0].layer.dtype
        self._ws = None

    def layers(self):
        """The chain's layer list as given (SkLinear / DenseLinear / Relu, repeated
        ReLUs kept), e.g. for model_save with the names model_load returned."""
        return list(self._layers)

    @property
    def d_in(self):
        return self.steps[0].layer.d_in

    @property
    def d_out(self):
        return self.steps[-1].layer.d_out

    def _workspace(self, T, device):
        import torch
        need = max(max(dense_workspace_size(st.layer.shape, T) if isinstance(st.layer, DenseLinear)
                       else workspace_size(st.layer.shape, T)) for st in self.steps)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=device)
        return self._ws

    def forward(self, x, train=True):
        """model_forward (nn_model.cpp:111-122).  train=True keeps each layer's
        input and saved projection for backward()."""
        import torch
        T = x.shape[0]
        if x.dim() != 2 or x.shape[1] != self.d_in:
            raise ShapeError(1, "model_forward: input columns != d_in")
        ws = self._workspace(T, x.device)
        td = torch_dtype(self.dtype)
        cur = x
        for i, st in enumerate(self.steps):
            L = st.layer
            y = torch.empty(T, L.d_out, dtype=td, device=x.device)
            if isinstance(L, DenseLinear):
                dense_forward(L.shape, cur, L.W, L.bias, y, ws, fuse=FUSE_RELU_OUT if st.relu_out else 0)
                if train:
                    st.x = cur
                    if i + 1 < len(self.steps):
                        self.steps[i + 1].bits = None
                cur = y
                continue
            saved = torch.empty(L.num_terms * L.low_rank, (T + 7) // 8 * 8, dtype=td, device=x.device) \
                if train else None
            bits = None
            if train and st.relu_out and self.relu_bits and i + 1 < len(self.steps) and \
                    isinstance(self.steps[i + 1].layer, SkLinear) and \
                    relu_bits_supported(L.shape) and relu_bits_supported(self.steps[i + 1].layer.shape):
                bits = torch.empty(T, relu_bits_row_words(L.d_out), dtype=torch.int32, device=x.device)
            forward(L.shape, cur, L.S1s, L.S2s, L.U1s, L.U2s, L.bias, y, saved, ws,
                    fuse=FUSE_RELU_OUT if st.relu_out else 0, relu_bits=bits)
            if train:
                st.x, st.saved = cur, saved
                if i + 1 < len(self.steps):
                    self.steps[i + 1].bits = bits
            cur = y
        return cur

    def allocate_grads(self, device="cuda"):
        """Per-layer fp32 gradient buckets: GradBucket (dU1s | db | dU2s) for an
        SKLinear, DenseBucket (dW | db) for a Linear."""
        from .dp import DenseBucket, GradBucket
        return [DenseBucket.allocate(st.layer.d_in, st.layer.d_out, device=device)
                if isinstance(st.layer, DenseLinear) else
                GradBucket.allocate(st.layer.d_in, st.layer.d_out, st.layer.num_terms, st.layer.low_rank,
                                    device=device) for st in self.steps]

    def backward(self, g, buckets=None, group=None, need_grad_x=True, overlap=None, phased=False):
        """Backward of the whole chain from the output gradient g [T, d_out].

        buckets: per-layer GradBucket (dU1s | db | dU2s, fp32), allocated if None.
        overlap: all-reduce each bucket across `group` as soon as it is ready,
        overlapped with the backward of the layers below; defaults to True when
        torch.distributed is initialised.  phased: split each layer's backward
        (dU1s|db first, its all-reduce overlapping that layer's own dX kernel)
        -- the single-layer schedule; for a stack the per-layer fused backward
        is faster (c2 layer: one du launch instead of two, -22 us).
        Returns (ChainGrads, works) -- wait on `works` before reading the grads."""
        import torch
        import torch.distributed as dist
        if self.steps[-1].x is None:
            raise SklError(2, "SkChain.backward: run forward(train=True) first")
        T = g.shape[0]
        if overlap is None:
            overlap = dist.is_available() and dist.is_initialized()
        if buckets is None:
            buckets = self.allocate_grads(g.device)
        ws = self._workspace(T, g.device)
        td = torch_dtype(self.dtype)
        works = []
        cur = g
        for i in range(len(self.steps) - 1, -1, -1):
            st, b = self.steps[i], buckets[i]
            L = st.layer
            gx = torch.empty(T, L.d_in, dtype=td, device=g.device) if (i > 0 or need_grad_x) else None
            fuse = FUSE_RELU_IN if st.relu_in else 0
            if isinstance(L, DenseLinear):
                dense_backward(L.shape, cur, st.x, L.W, gx, b.dW, b.db, ws, fuse=fuse)
                if overlap:
                    w = b.allreduce_(group, async_op=True)
                    if w is not None:
                        works.append(w)
            elif overlap and phased:
                backward_phase(L.shape, BWD_DU1_DB, cur, st.x, st.saved, L.S1s, L.S2s, L.U1s, L.U2s, None,
                               b.dU1s, None, b.db, ws)
                w = b.allreduce_head(group, async_op=True)
                if w is not None:
                    works.append(w)
                backward_phase(L.shape, BWD_DX_DU2, cur, st.x, st.saved, L.S1s, L.S2s, L.U1s, L.U2s, gx,
                               None, b.dU2s, None, ws, fuse=fuse, relu_bits=st.bits if st.relu_in else None)
                w = b.allreduce_tail(group, async_op=True)
                if w is not None:
                    works.append(w)
            elif overlap:
                # one fused backward per layer, then its whole bucket all-reduced on
                # NCCL's stream while the layers below run theirs (SURVEY §8e "in the
                # stack"); the phased split would cost a second du launch per layer
                backward_phase(L.shape, BWD_ALL, cur, st.x, st.saved, L.S1s, L.S2s, L.U1s, L.U2s, gx,
                               b.dU1s, b.dU2s, b.db, ws, fuse=fuse, relu_bits=st.bits if st.relu_in else None)
                w = b.allreduce_(group, async_op=True)
                if w is not None:
                    works.append(w)
            else:
                backward_phase(L.shape, BWD_ALL, cur, st.x, st.saved, L.S1s, L.S2s, L.U1s, L.U2s, gx,
                               b.dU1s, b.dU2s, b.db, ws, fuse=fuse, relu_bits=st.bits if st.relu_in else None)
            cur = gx
        return ChainGrads(cur, buckets), works


def wait_all(works):
    for w in works:
        w.wait()


def bert_ffn_stack(num_layers=12, d_model=768, d_ff=3072, k=128, seed=42, dtype=BF16, device="cuda"):
    """BASELINE config 5: per encoder layer 4 x SKLinear(768,768,L=1,k=128) (the
    projections; attention itself is not on this path) then SKLinear(768,3072,
    L=2,k=128) + ReLU + SKLinear(3072,768,L=2,k=128).  L=1 for the 768x768
    projections: L=2,k=128 would store more than the dense layer
    (exceeds_dense, layers.hpp:28-31).  Layer j's seed is
    derive_seed(seed, j) (SPEC.md:414 convention)."""
    from . import derive_seed
    layers = []
    j = 0
    for _ in range(num_layers):
        for _p in range(4):
            layers.append(SkLinear(d_model, d_model, 1, k, seed=derive_seed(seed, j), dtype=dtype, device=device))
            j += 1
        layers.append(SkLinear(d_model, d_ff, 2, k, seed=derive_seed(seed, j), dtype=dtype, device=device))
        j += 1
        layers.append(Relu())
        layers.append(SkLinear(d_ff, d_model, 2, k, seed=derive_seed(seed, j), dtype=dtype, device=device))
        j += 1
    return SkChain(layers)
