"""Data-parallel (token-sharded) SKLinear: host-side plumbing.

The path shards along tokens only: every rank holds the full
replicated layer (sketches regenerated from the same seed -- bit-identical, no
broadcast), the forward needs no communication, and the backward's parameter
gradients dU1s / dU2s / db are sums over tokens, so one all-reduce (sum) of a
single contiguous fp32 bucket per layer combines the shards.  dX stays local.

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
    """One flat fp32 buffer holding dU1s [L,k,d_out] | dU2s [L,d_in,k] | db [d_out].

    The backward writes straight into the views, so the all-reduce needs no
    packing copy.
    """

    flat: object
    dU1s: object
    dU2s: object
    db: object

    @staticmethod
    def numel(d_in, d_out, L, k):
        return L * k * d_out + L * d_in * k + d_out

    @classmethod
    def allocate(cls, d_in, d_out, L, k, device="cuda"):
        import torch
        flat = torch.zeros(cls.numel(d_in, d_out, L, k), dtype=torch.float32, device=device)
        n1, n2 = L * k * d_out, L * d_in * k
        return cls(flat, flat[:n1].view(L, k, d_out), flat[n1:n1 + n2].view(L, d_in, k), flat[n1 + n2:])

    def allreduce_(self, group=None, async_op=False):
        """Sum the bucket over the ranks of `group` (in place)."""
        import torch.distributed as dist
        if not dist.is_initialized() or dist.get_world_size(group) == 1:
            return None
        return dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
