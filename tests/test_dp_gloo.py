"""Multi-process (gloo, world_size 2) test of the token-sharded DP logic:
per-rank token shards -> local backward -> all-reduce of the flat gradient
bucket == full-batch gradients.  The per-shard compute is the oracle (CPU),
so this checks the host-side sharding / bucket / collective logic that
bench.py runs over NCCL on GPUs."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from paper_2601_15473_b200.dp import GradBucket, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d_in, d_out, L, k, T = 24, 40, 2, 4, 37
    o = oracle.Oracle("port")
    p = o.sk_linear_fresh(d_in, d_out, L, k, 42)  # replicated: same seed on every rank
    x, g, _ = oracle.inputs(d_in, d_out, T, 7, o)
    lo, hi = shard_range(T, rank, world)
    gx, gu1, gu2, gb = o.backward(p, x[:, lo:hi].copy(), g[:, lo:hi].copy())
    _, du1, du2, db = oracle.grads_to_abi(gx, gu1, gu2, gb)
    bucket = GradBucket.allocate(d_in, d_out, L, k, device="cpu", dtype=torch.float64)
    # phase DU1_DB writes dU1s | db, its all-reduce is issued async; phase
    # DX_DU2 writes dU2s, then the tail all-reduce (the overlapped DP schedule)
    bucket.dU1s.copy_(torch.from_numpy(du1))
    bucket.db.copy_(torch.from_numpy(db))
    w1 = bucket.allreduce_head(async_op=True)
    bucket.dU2s.copy_(torch.from_numpy(du2))
    w2 = bucket.allreduce_tail(async_op=True)
    w1.wait()
    w2.wait()
    if rank == 0:
        full = oracle.grads_to_abi(*o.backward(p, x, g))
        ref = np.concatenate([full[1].ravel(), full[3], full[2].ravel()])  # dU1s | db | dU2s
        q.put(float(np.max(np.abs(bucket.flat.numpy() - ref)) / np.max(np.abs(ref))))
    dist.destroy_process_group()


def test_shard_range_partitions_tokens():
    from paper_2601_15473_b200.dp import shard_range
    for T in (0, 1, 7, 32768, 32769):
        for world in (1, 2, 3, 8):
            spans = [shard_range(T, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == T
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_gloo_world2_allreduce_equals_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err < 1e-12
