"""Token-sharded data parallelism with the DEVICE kernels doing the compute:
two ranks (two processes sharing cuda:0; torch.distributed gloo, which
all-reduces CUDA tensors through the host -- NCCL refuses two ranks on one GPU)
run the overlapped schedules of dp.py / model.py on their token shards, and the
all-reduced gradients equal the single-process full-batch gradients.

The NCCL path itself is exercised by tests/cpp/test_chain_dp.cpp (C++ host,
world 1) and test_gpu.py::test_dp_overlapped_step_over_nccl.
"""
from __future__ import annotations

import os
import socket

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

D_IN, D_OUT, L, K, T = 768, 3072, 2, 128, 3000


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(torch, skl):
    gen = torch.Generator(device="cuda").manual_seed(5)
    X = torch.randn(T, D_IN, device="cuda", generator=gen).to(torch.bfloat16)
    G = torch.randn(T, D_OUT, device="cuda", generator=gen).to(torch.bfloat16)
    return X, G


def _worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2601_15473_b200 as skl
    from paper_2601_15473_b200.dp import GradBucket, backward_overlapped, shard_range
    from paper_2601_15473_b200.model import Relu, SkChain
    layer = skl.SkLinear(D_IN, D_OUT, L, K, seed=42)      # replicated: same seed on every rank
    X, G = _inputs(torch, skl)
    lo, hi = shard_range(T, rank, world)
    x, g = X[lo:hi].contiguous(), G[lo:hi].contiguous()
    saved = torch.empty(L * K, (hi - lo + 7) // 8 * 8, dtype=torch.bfloat16, device="cuda")
    layer.forward(x, saved=saved)
    gb = GradBucket.allocate(D_IN, D_OUT, L, K)
    gx = torch.empty(hi - lo, D_IN, dtype=torch.bfloat16, device="cuda")
    for w in backward_overlapped(skl, layer.shape, g, x, saved, layer.S1s, layer.S2s, layer.U1s, layer.U2s, gx, gb,
                                 layer.workspace(hi - lo)):
        w.wait()
    # a 2-layer chain with a fused ReLU, per-layer bucket all-reduce overlapping the layer below
    a = skl.SkLinear(D_IN, D_OUT, L, K, seed=7)
    b = skl.SkLinear(D_OUT, D_IN, L, K, seed=8)
    chain = SkChain([a, Relu(), b])
    chain.forward(x)
    cg, works = chain.backward(g[:, :D_IN].contiguous(), overlap=True)
    for w in works:
        w.wait()
    torch.cuda.synchronize()
    if rank == 0:
        torch.save({"layer": gb.flat.cpu(), "gx": gx.cpu(), "lo": lo, "hi": hi,
                    "chain": [bk.flat.cpu() for bk in cg.layers]}, out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_dp_with_device_kernels(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    import paper_2601_15473_b200 as skl
    from paper_2601_15473_b200.model import Relu, SkChain
    out = str(tmp_path / "dp.pt")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = torch.load(out)
    # single-process full batch
    layer = skl.SkLinear(D_IN, D_OUT, L, K, seed=42)
    X, G = _inputs(torch, skl)
    full = layer.backward(X, G)
    ref = torch.cat([full.grad_u1.flatten(), full.grad_b, full.grad_u2.flatten()]).cpu()
    rel = ((got["layer"] - ref).norm() / ref.norm()).item()
    assert rel < 1e-5, rel            # fp32 sums over the same tokens in another split order
    assert torch.equal(got["gx"], full.grad_x[got["lo"]:got["hi"]].cpu())   # dX is local: bitwise
    a = skl.SkLinear(D_IN, D_OUT, L, K, seed=7)
    b = skl.SkLinear(D_OUT, D_IN, L, K, seed=8)
    chain = SkChain([a, Relu(), b])
    chain.forward(X)
    cg, _ = chain.backward(G[:, :D_IN].contiguous(), overlap=False)
    torch.cuda.synchronize()
    for i, bk in enumerate(cg.layers):
        r = bk.flat.cpu()
        rel = ((got["chain"][i] - r).norm() / r.norm()).item()
        assert rel < 1e-5, (i, rel)
