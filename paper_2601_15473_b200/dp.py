"""Data-parallel (token-sharded) SKLinear: host-side plumbing.

The path shards along tokens only: every rank holds the full
replicated layer (sketches regenerated from the same seed -- bit-identical, no
broadcast), the forward needs no communication, and the backward's parameter
gradients dU1s / dU2s / db are sums over tokens, so they are all-reduced
(sum) across ranks.  dX stays local.

Overlap: the backward runs in two phases (skl.h sketched_linear_backward_phase):
phase DU1_DB produces dU1s and db -- 80 % of the bucket at c2 -- whose
all-reduce is issued asynchronously and runs on NCCL's stream while phase
DX_DU2 computes dX (the fused b2b kernel) and dU2s; the small dU2s all-reduce
follows.  The bucket is laid out dU1s | db | dU2s so each collective is one
contiguous slice (no packing copy).  libskl leaves `reserved_sms` SMs free so
the NCCL kernel is co-resident with the persistent compute kernels.

torch.distributed is the plumbing (NCCL on GPUs, gloo in the CPU tests); the
C-ABI also offers skl_allreduce_grads for C++ hosts holding an ncclComm_t.
"""
from __future__ import annotations

from dataclasses import dataclass


def shard_range(T: int, rank: int, world: int):
    """Contiguous token range [lo, hi) of `rank` (balanced, deterministic)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, rem = divmod(T, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


@dataclass
class GradBucket:
    """One flat fp32 buffer holding dU1s [L,k,d_out] | db [d_out] | dU2s [L,d_in,k].

    The backward writes straight into the views, so the all-reduces need no
    packing copy: `head` (dU1s | db) is reduced while dX is computed, `tail`
    (dU2s) after.
    """

    flat: object
    dU1s: object
    db: object
    dU2s: object
    head: object
    tail: object

    @staticmethod
    def numel(d_in, d_out, L, k):
        return L * k * d_out + d_out + L * d_in * k

    @classmethod
    def from_flat(cls, flat, d_in, d_out, L, k):
        n1, n2 = L * k * d_out, d_out
        return cls(flat, flat[:n1].view(L, k, d_out), flat[n1:n1 + n2], flat[n1 + n2:].view(L, d_in, k),
                   flat[:n1 + n2], flat[n1 + n2:])

    @classmethod
    def allocate(cls, d_in, d_out, L, k, device="cuda", dtype=None):
        import torch
        flat = torch.zeros(cls.numel(d_in, d_out, L, k), dtype=dtype or torch.float32, device=device)
        return cls.from_flat(flat, d_in, d_out, L, k)

    @staticmethod
    def _reduce(t, group, async_op):
        import torch.distributed as dist
        if not dist.is_initialized():
            return None
        return dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group, async_op=async_op)

    def allreduce_head(self, group=None, async_op=False):
        """Sum dU1s | db over the ranks of `group` (in place)."""
        return self._reduce(self.head, group, async_op)

    def allreduce_tail(self, group=None, async_op=False):
        """Sum dU2s over the ranks of `group` (in place)."""
        return self._reduce(self.tail, group, async_op)

    def allreduce_(self, group=None, async_op=False):
        """Sum the whole bucket (one collective, no overlap)."""
        return self._reduce(self.flat, group, async_op)


@dataclass
class DenseBucket:
    """One flat fp32 buffer holding a DenseLinear's dW [d_out, d_in] | db [d_out]
    (same all-reduce interface as GradBucket; the whole bucket is the head)."""

    flat: object
    dW: object
    db: object

    @staticmethod
    def numel(d_in, d_out):
        return d_out * d_in + d_out

    @classmethod
    def allocate(cls, d_in, d_out, device="cuda", dtype=None):
        import torch
        flat = torch.zeros(cls.numel(d_in, d_out), dtype=dtype or torch.float32, device=device)
        return cls(flat, flat[:d_out * d_in].view(d_out, d_in), flat[d_out * d_in:])

    def allreduce_(self, group=None, async_op=False):
        return GradBucket._reduce(self.flat, group, async_op)

    allreduce_head = allreduce_

    def allreduce_tail(self, group=None, async_op=False):
        return None


def backward_overlapped(skl, s, g, x, saved, S1s, S2s, U1s, U2s, grad_x, bucket: GradBucket, workspace,
                        group=None):
    """Token-sharded backward of one SKLinear layer with the gradient
    all-reduce overlapped with the dX kernel.  Returns the pending collective
    works; `w.wait()` makes the current stream wait for them (NCCL)."""
    works = []
    skl.backward_phase(s, skl.BWD_DU1_DB, g, x, saved, S1s, S2s, U1s, U2s, None, bucket.dU1s, None, bucket.db,
                       workspace)
    w = bucket.allreduce_head(group, async_op=True)
    if w is not None:
        works.append(w)
    skl.backward_phase(s, skl.BWD_DX_DU2, g, x, saved, S1s, S2s, U1s, U2s, grad_x, None, bucket.dU2s, None,
                       workspace)
    w = bucket.allreduce_tail(group, async_op=True)
    if w is not None:
        works.append(w)
    return works
