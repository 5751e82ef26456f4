"""GPU parity tests: the sm_100a kernels (through the C-ABI of libskl.so)
against the oracle (oracle/, the reference algorithm in f64) on identical
seeded inputs.  Run on a B200:  python -m pytest tests -m gpu -x -q
"""
from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def skl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_15473_b200 as skl
    skl.lib()  # loud failure if libskl.so is missing
    return skl


def _np(t):
    return t.detach().double().cpu().numpy()


def _tdev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


# --------------------------------------------------------------------------- B1
@pytest.mark.parametrize("k,d,seed", [(64, 1024, 0xE816C0EF88EC839C), (3, 7, 42), (128, 3072, 12345)])
def test_gaussian_sketch_entries(skl, port, k, d, seed):
    """realize_sketch(Gaussian) on device: integer chain exact, values equal
    after rounding to f32/bf16 on every entry; f64 within 4 ulp."""
    ref = port.realize_sketch(0, k, d, seed)
    out64 = torch.empty(k, d, dtype=torch.float64, device="cuda")
    skl.realize_sketch(0, k, d, seed, out64)
    dev = _np(out64)
    ulp = np.abs(dev.view(np.int64) - ref.view(np.int64))
    assert ulp.max() <= 4, f"f64 ulp max {ulp.max()}"
    out32 = torch.empty(k, d, dtype=torch.float32, device="cuda")
    skl.realize_sketch(0, k, d, seed, out32)
    assert np.array_equal(_np(out32), ref.astype(np.float32).astype(np.float64))
    outb = torch.empty(k, d, dtype=torch.bfloat16, device="cuda")
    skl.realize_sketch(0, k, d, seed, outb)
    from tests._util import bf16_round
    assert np.array_equal(_np(outb), bf16_round(ref))


def test_rademacher_bit_exact(skl, port):
    ref = port.realize_sketch(1, 33, 517, 99)
    out = torch.empty(33, 517, dtype=torch.float64, device="cuda")
    skl.realize_sketch(1, 33, 517, 99, out)
    assert np.array_equal(_np(out), ref)


def test_gaussian_matrix_unit_variance(skl, port):
    ref = port.gaussian_matrix(37, 11, 7)
    out = torch.empty(37, 11, dtype=torch.float64, device="cuda")
    skl.realize_sketch(0, 37, 11, 7, out, unit_variance=True)
    assert np.abs(_np(out).view(np.int64) - ref.view(np.int64)).max() <= 4


@pytest.mark.parametrize("dist", [0, 1])
@pytest.mark.parametrize("d_in,d_out,L,k", [(1024, 1024, 1, 64), (768, 3072, 2, 128), (40, 24, 3, 8)])
def test_generate_layer_matches_sk_linear_fresh(skl, port, dist, d_in, d_out, L, k):
    """Device sketches + U init in the ABI stacks == sk_linear_fresh (f32 rounding)."""
    import oracle
    seed = 42
    p = port.sk_linear_fresh(d_in, d_out, L, k, seed, dist)
    abi = oracle.to_abi(p)
    s = skl.shape(d_in, d_out, L, k, skl.F32_TF32)
    S1s = torch.empty(L, d_in, k, device="cuda")
    S2s = torch.empty(L, k, d_out, device="cuda")
    U1s = torch.empty(L, k, d_out, device="cuda")
    U2s = torch.empty(L, d_in, k, device="cuda")
    skl.generate_sketches(s, dist, seed, S1s, S2s)
    skl.init_params(s, seed, U1s, U2s)
    for name, t in (("S1s", S1s), ("S2s", S2s), ("U1s", U1s), ("U2s", U2s)):
        assert np.array_equal(_np(t), abi[name].astype(np.float32).astype(np.float64)), name


# --------------------------------------------------------------------------- B2/B3
def _make_case(skl, port, d_in, d_out, L, k, T, dtype, seed=42, dist=0):
    """Device layer + inputs, and the same (rounded) values as f64 for the oracle."""
    import oracle
    td = skl.torch_dtype(dtype)
    s = skl.shape(d_in, d_out, L, k, dtype)
    S1s = torch.empty(L, d_in, k, dtype=td, device="cuda")
    S2s = torch.empty(L, k, d_out, dtype=td, device="cuda")
    U1s = torch.empty(L, k, d_out, dtype=td, device="cuda")
    U2s = torch.empty(L, d_in, k, dtype=td, device="cuda")
    skl.generate_sketches(s, dist, seed, S1s, S2s)
    skl.init_params(s, seed, U1s, U2s)
    x, g, b = oracle.inputs(d_in, d_out, T, seed, port)
    X = _tdev(x.T, td)
    G = _tdev(g.T, td)
    B = _tdev(b, td)
    P = oracle.from_abi(d_in, d_out, _np(S1s), _np(U1s), _np(U2s), _np(S2s))
    return s, (S1s, S2s, U1s, U2s), X, G, B, P, _np(X).T.copy(), _np(G).T.copy(), _np(B)


def _variant(dtype, skl):
    return "bf16" if dtype == skl.BF16 else "tf32"


CASES = [
    (1024, 1024, 1, 64, 64),       # c1 shape
    (768, 3072, 2, 128, 300),      # c2 shape, ragged token count
    (256, 512, 3, 32, 129),        # R = 192 (single GEMM1 chunk), ragged
    (512, 256, 4, 64, 200),        # R = 512, d_out < d_in
    (128, 64, 1, 16, 50),          # small rank R = 32 (padded to 64)
    (768, 768, 1, 128, 600),       # c5 projection: R = 256 (one chunk, saves deferred after hready), du M = 128
    (1024, 512, 1, 64, 20000),     # R = 128 ping-pong H: > 74 pair tiles, so CTAs alternate TMEM regions
    (4096, 4096, 1, 16, 300),      # c4 L1 k16 shape: R = 32 on d = 4096 (packed panels, 32 GEMM2 tiles)
    (4096, 4096, 4, 64, 257),      # c4 L4 k64 shape: R = 512, ragged T
    # R > 512: R-split clusters of CTA pairs, partial sums chained over DSMEM
    (512, 768, 3, 128, 1000),      # R = 768: 2 pairs x 384 (chunks 256 + 128), direct stacks
    (1024, 1536, 3, 100, 700),     # R = 600 -> 640: 2 pairs x 320, packed panels (k % 64 != 0)
    (2048, 1024, 4, 256, 2000),    # R = 2048: 4 pairs (cluster of 8 CTAs), several tiles per cluster
    (4096, 4096, 3, 256, 3000),    # c3 shape: R = 1536, 3 pairs x 512
]


@pytest.mark.parametrize("unfused", [False, True])
@pytest.mark.parametrize("d_in,d_out,L,k,T", CASES)
def test_forward_parity_bf16(skl, port, monkeypatch, unfused, d_in, d_out, L, k, T):
    if unfused and os.environ.get("SKL_FORCE_UNFUSED") is None:
        pytest.skip("unfused path is exercised in a separate process (SKL_FORCE_UNFUSED=1)")
    s, (S1s, S2s, U1s, U2s), X, G, B, P, x64, g64, b64 = _make_case(skl, port, d_in, d_out, L, k, T, skl.BF16)
    y = torch.empty(T, d_out, dtype=torch.bfloat16, device="cuda")
    saved = torch.empty(L * k, (T + 7) // 8 * 8, dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device="cuda")
    skl.forward(s, X, S1s, S2s, U1s, U2s, B, y, saved, ws)
    torch.cuda.synchronize()
    y_ref = port.forward(P, b64, x64).T
    from tests._util import check_close
    check_close("y", _np(y), y_ref, "bf16", regress=True)
    # saved projection (x·S1_i, term-major) is kept transposed: [L*k][round8(T)]
    sv_ref = np.concatenate([x64.T @ P.s2[i].T for i in range(L)], axis=1)
    check_close("saved", _np(saved)[:, :T].T, sv_ref, "bf16", regress=True)


@pytest.mark.parametrize("d_in,d_out,L,k,T", CASES)
def test_backward_parity_bf16(skl, port, d_in, d_out, L, k, T):
    import oracle
    s, (S1s, S2s, U1s, U2s), X, G, B, P, x64, g64, b64 = _make_case(skl, port, d_in, d_out, L, k, T, skl.BF16)
    y = torch.empty(T, d_out, dtype=torch.bfloat16, device="cuda")
    saved = torch.empty(L * k, (T + 7) // 8 * 8, dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device="cuda")
    skl.forward(s, X, S1s, S2s, U1s, U2s, B, y, saved, ws)
    gx = torch.empty(T, d_in, dtype=torch.bfloat16, device="cuda")
    du1 = torch.empty(L, k, d_out, device="cuda")
    du2 = torch.empty(L, d_in, k, device="cuda")
    db = torch.empty(d_out, device="cuda")
    skl.backward(s, G, X, saved, S1s, S2s, U1s, U2s, gx, du1, du2, db, ws)
    torch.cuda.synchronize()
    rgx, rgu1, rgu2, rgb = oracle.grads_to_abi(*port.backward(P, x64, g64))
    from tests._util import check_close
    check_close("grad_x", _np(gx), rgx, "bf16", regress=True)
    check_close("dU1s", _np(du1), rgu1, "bf16", regress=True)
    check_close("dU2s", _np(du2), rgu2, "bf16", regress=True)
    check_close("db", _np(db), rgb, "bf16", regress=True)
    # recompute path (no saved projection) gives the same gradients
    du1b = torch.empty_like(du1)
    du2b = torch.empty_like(du2)
    skl.backward(s, G, X, None, S1s, S2s, U1s, U2s, None, du1b, du2b, None, ws)
    torch.cuda.synchronize()
    check_close("dU1s(recompute)", _np(du1b), rgu1, "bf16", regress=True)
    check_close("dU2s(recompute)", _np(du2b), rgu2, "bf16", regress=True)


# --------------------------------------------------------------------------- TF32 (fp32 I/O)
TF32_CASES = [
    (1024, 1024, 1, 64, 64),       # c1 shape (fused, R = 128)
    (256, 512, 2, 64, 300),        # R = 256 (fused, widest on-chip TF32 H), ragged
    (768, 3072, 2, 128, 200),      # c2 shape, R = 512 (TF32 H through HBM)
    (128, 64, 1, 16, 50),          # small rank R = 32 (padded to 64)
    (96, 160, 3, 8, 77),           # k % 64 != 0, odd tokens
    (512, 512, 1, 64, 20000),      # R = 128 ping-pong H in TF32, several tiles per CTA
    (768, 768, 1, 128, 600),       # c5 projection shape in TF32 (R = 256, the widest TMEM-only TF32 H)
    (4096, 4096, 2, 64, 130),      # c4 TF32 L2 k64 shape (R = 256), ragged T
]


@pytest.mark.parametrize("d_in,d_out,L,k,T", TF32_CASES)
def test_forward_backward_parity_tf32(skl, port, d_in, d_out, L, k, T):
    """fp32-in/fp32-out TF32 variant vs the f64 oracle: rel_fro <= 2e-3 and
    max_abs <= 2e-3 * max|ref| on y, grad_x, dU1s, dU2s, db (tests/_util.py)."""
    import oracle
    from tests._util import check_close
    s, (S1s, S2s, U1s, U2s), X, G, B, P, x64, g64, b64 = _make_case(skl, port, d_in, d_out, L, k, T, skl.F32_TF32)
    y = torch.empty(T, d_out, device="cuda")
    saved = torch.empty(L * k, (T + 7) // 8 * 8, device="cuda")
    ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device="cuda")
    skl.forward(s, X, S1s, S2s, U1s, U2s, B, y, saved, ws)
    gx = torch.empty(T, d_in, device="cuda")
    du1 = torch.empty(L, k, d_out, device="cuda")
    du2 = torch.empty(L, d_in, k, device="cuda")
    db = torch.empty(d_out, device="cuda")
    skl.backward(s, G, X, saved, S1s, S2s, U1s, U2s, gx, du1, du2, db, ws)
    torch.cuda.synchronize()
    check_close("y(tf32)", _np(y), port.forward(P, b64, x64).T, "tf32", regress=True)
    rgx, rgu1, rgu2, rgb = oracle.grads_to_abi(*port.backward(P, x64, g64))
    check_close("grad_x(tf32)", _np(gx), rgx, "tf32", regress=True)
    check_close("dU1s(tf32)", _np(du1), rgu1, "tf32", regress=True)
    check_close("dU2s(tf32)", _np(du2), rgu2, "tf32", regress=True)
    check_close("db(tf32)", _np(db), rgb, "tf32", regress=True)
    # recompute path (no saved projection)
    du1b, du2b = torch.empty_like(du1), torch.empty_like(du2)
    skl.backward(s, G, X, None, S1s, S2s, U1s, U2s, None, du1b, du2b, None, ws)
    torch.cuda.synchronize()
    check_close("dU1s(tf32, recompute)", _np(du1b), rgu1, "tf32", regress=True)
    check_close("dU2s(tf32, recompute)", _np(du2b), rgu2, "tf32", regress=True)


def test_backward_is_deterministic(skl, port):
    """Split-T reduction order is fixed: two runs are bitwise identical."""
    s, (S1s, S2s, U1s, U2s), X, G, B, P, x64, g64, b64 = _make_case(skl, port, 768, 3072, 2, 128, 4096, skl.BF16)
    ws = torch.empty(max(skl.workspace_size(s, 4096)), dtype=torch.uint8, device="cuda")
    saved = torch.empty(256, 4096, dtype=torch.bfloat16, device="cuda")
    y = torch.empty(4096, 3072, dtype=torch.bfloat16, device="cuda")
    skl.forward(s, X, S1s, S2s, U1s, U2s, B, y, saved, ws)
    outs = []
    for _ in range(2):
        gx = torch.empty(4096, 768, dtype=torch.bfloat16, device="cuda")
        du1 = torch.empty(2, 128, 3072, device="cuda")
        du2 = torch.empty(2, 768, 128, device="cuda")
        db = torch.empty(3072, device="cuda")
        skl.backward(s, G, X, saved, S1s, S2s, U1s, U2s, gx, du1, du2, db, ws)
        outs.append((gx, du1, du2, db))
    torch.cuda.synchronize()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
def test_phased_backward_matches_oracle(skl, port, dtype_name):
    """sketched_linear_backward_phase(DU1_DB) then (DX_DU2), with SMs reserved
    for a concurrent collective, gives the same gradients (within the gates)."""
    import oracle
    from tests._util import check_close
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    d_in, d_out, L, k, T = 768, 3072, 2, 128, 1000
    s, (S1s, S2s, U1s, U2s), X, G, B, P, x64, g64, b64 = _make_case(skl, port, d_in, d_out, L, k, T, dtype)
    td = skl.torch_dtype(dtype)
    y = torch.empty(T, d_out, dtype=td, device="cuda")
    saved = torch.empty(L * k, (T + 7) // 8 * 8, dtype=td, device="cuda")
    ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device="cuda")
    skl.set_reserved_sms(8)
    try:
        skl.forward(s, X, S1s, S2s, U1s, U2s, B, y, saved, ws)
        gx = torch.empty(T, d_in, dtype=td, device="cuda")
        du1 = torch.empty(L, k, d_out, device="cuda")
        du2 = torch.empty(L, d_in, k, device="cuda")
        db = torch.empty(d_out, device="cuda")
        skl.backward_phase(s, skl.BWD_DU1_DB, G, X, saved, S1s, S2s, U1s, U2s, None, du1, None, db, ws)
        skl.backward_phase(s, skl.BWD_DX_DU2, G, X, saved, S1s, S2s, U1s, U2s, gx, None, du2, None, ws)
        torch.cuda.synchronize()
    finally:
        skl.set_reserved_sms(0)
    rgx, rgu1, rgu2, rgb = oracle.grads_to_abi(*port.backward(P, x64, g64))
    check_close("grad_x(phased)", _np(gx), rgx, dtype_name)
    check_close("dU1s(phased)", _np(du1), rgu1, dtype_name)
    check_close("dU2s(phased)", _np(du2), rgu2, dtype_name)
    check_close("db(phased)", _np(db), rgb, dtype_name)


@pytest.mark.parametrize("reserved", [0, 8])
def test_phased_backward_full_c2_matches_fused(skl, reserved):
    """At the bench's full c2 size (T = 32768) the phased launches take other
    dU tilings than the fused one (dU1-only: 12 tiles, cooperative reduction
    when clusters of 2S CTAs do not all fit; dU2-only: 3 tiles, S = 23-24):
    grad_x is the same kernel (bitwise), the fp32 gradients differ only by the
    order of the split partial sums."""
    d_in, d_out, L, k, T = 768, 3072, 2, 128, 32768
    s = skl.shape(d_in, d_out, L, k, skl.BF16)
    bf = torch.bfloat16
    S1s = torch.empty(L, d_in, k, dtype=bf, device="cuda")
    S2s = torch.empty(L, k, d_out, dtype=bf, device="cuda")
    U1s = torch.empty(L, k, d_out, dtype=bf, device="cuda")
    U2s = torch.empty(L, d_in, k, dtype=bf, device="cuda")
    skl.generate_sketches(s, skl.GAUSSIAN, 5, S1s, S2s)
    skl.init_params(s, 5, U1s, U2s)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)
    X = torch.randn(T, d_in, device="cuda", generator=gen).to(bf)
    G = torch.randn(T, d_out, device="cuda", generator=gen).to(bf)
    B = torch.zeros(d_out, dtype=bf, device="cuda")
    y = torch.empty(T, d_out, dtype=bf, device="cuda")
    saved = torch.empty(L * k, T, dtype=bf, device="cuda")
    ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device="cuda")
    skl.forward(s, X, S1s, S2s, U1s, U2s, B, y, saved, ws)
    outs = []
    for phased in (False, True):
        gx = torch.empty(T, d_in, dtype=bf, device="cuda")
        du1 = torch.empty(L, k, d_out, device="cuda")
        du2 = torch.empty(L, d_in, k, device="cuda")
        db = torch.empty(d_out, device="cuda")
        skl.set_reserved_sms(reserved if phased else 0)
        try:
            if phased:
                skl.backward_phase(s, skl.BWD_DU1_DB, G, X, saved, S1s, S2s, U1s, U2s, None, du1, None, db, ws)
                skl.backward_phase(s, skl.BWD_DX_DU2, G, X, saved, S1s, S2s, U1s, U2s, gx, None, du2, None, ws)
            else:
                skl.backward(s, G, X, saved, S1s, S2s, U1s, U2s, gx, du1, du2, db, ws)
            torch.cuda.synchronize()
        finally:
            skl.set_reserved_sms(0)
        outs.append((gx, du1, du2, db))
    (gx0, a0, b0, c0), (gx1, a1, b1, c1) = outs
    assert torch.equal(gx0, gx1)
    for name, u, v in (("dU1s", a0, a1), ("dU2s", b0, b1), ("db", c0, c1)):
        rel = float((u - v).norm() / v.norm())
        assert rel <= 1e-5, f"{name}: phased vs fused rel_fro {rel:.2e}"


def test_dp_overlapped_step_over_nccl(skl, port):
    """The DP schedule bench.py runs at N > 1 (dp.backward_overlapped: async
    NCCL all-reduce of dU1s|db issued before the dX kernel), on a world-1 NCCL
    group: the collectives run and the bucket equals the plain backward."""
    import socket
    import torch.distributed as dist
    from paper_2601_15473_b200.dp import GradBucket, backward_overlapped
    d_in, d_out, L, k, T = 768, 3072, 2, 128, 2048
    s, (S1s, S2s, U1s, U2s), X, G, B, P, x64, g64, b64 = _make_case(skl, port, d_in, d_out, L, k, T, skl.BF16)
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port_ = sock.getsockname()[1]
    sock.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port_}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        y = torch.empty(T, d_out, dtype=torch.bfloat16, device="cuda")
        saved = torch.empty(L * k, T, dtype=torch.bfloat16, device="cuda")
        ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device="cuda")
        skl.forward(s, X, S1s, S2s, U1s, U2s, B, y, saved, ws)
        gb = GradBucket.allocate(d_in, d_out, L, k)
        gx = torch.empty(T, d_in, dtype=torch.bfloat16, device="cuda")
        works = backward_overlapped(skl, s, G, X, saved, S1s, S2s, U1s, U2s, gx, gb, ws)
        assert len(works) == 2
        for w in works:
            w.wait()
        ref = GradBucket.allocate(d_in, d_out, L, k)
        gx2 = torch.empty_like(gx)
        skl.backward(s, G, X, saved, S1s, S2s, U1s, U2s, gx2, ref.dU1s, ref.dU2s, ref.db, ws)
        torch.cuda.synchronize()
        assert torch.equal(gx, gx2)
        rel = (gb.flat - ref.flat).norm() / ref.flat.norm()
        assert rel < 1e-5, rel
    finally:
        dist.destroy_process_group()


# --------------------------------------------------------------------------- Linear/ReLU chains
@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
def test_chain_with_fused_relu_matches_oracle(skl, port, dtype_name):
    """model_forward over SKLinear / ReLU layers (nn_model.cpp:111-122) with the
    ReLU fused into the neighbouring kernels, forward + training backward, vs
    the layer-by-layer f64 oracle composition (Relu::forward/backward,
    nn_layers.cpp:341-354) on the same rounded parameters and input."""
    import oracle
    from paper_2601_15473_b200.model import Relu, SkChain
    from tests._util import check_close
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    dims = [(96, 160, 2, 32), (160, 128, 1, 64), (128, 64, 3, 16)]
    T = 150
    layers = []
    gen = torch.Generator(device="cuda").manual_seed(5)
    for i, (di, do, L, k) in enumerate(dims):
        lyr = skl.SkLinear(di, do, L, k, seed=100 + i, dtype=dtype)
        lyr.bias.copy_((torch.randn(do, device="cuda", generator=gen) * 0.3).to(td))
        layers.append(lyr)
    chain = SkChain([layers[0], Relu(), layers[1], layers[2]])
    x = torch.randn(T, 96, device="cuda", generator=gen).to(td)
    g = torch.randn(T, 64, device="cuda", generator=gen).to(td)
    y = chain.forward(x)
    grads, works = chain.backward(g, overlap=False)
    torch.cuda.synchronize()
    # oracle, layer by layer on the device's own (rounded) layer inputs, so each
    # fused kernel is checked at its own tolerance (an all-f64 composition
    # would compound the rounding of the bf16 activations and flip ReLU masks
    # at pre-activations within one rounding step of zero)
    P = [oracle.from_abi(l.d_in, l.d_out, _np(l.S1s), _np(l.U1s), _np(l.U2s), _np(l.S2s)) for l in layers]
    B = [_np(l.bias) for l in layers]
    a0 = _np(x).T.copy()
    a1 = _np(chain.steps[1].x).T.copy()
    a2 = _np(chain.steps[2].x).T.copy()
    check_close("chain relu(layer0)", a1, np.maximum(port.forward(P[0], B[0], a0), 0.0), dtype_name)
    check_close("chain layer1", a2, port.forward(P[1], B[1], a1), dtype_name)
    check_close("chain y", _np(y), port.forward(P[2], B[2], a2).T, dtype_name)
    g3 = _np(g).T.copy()
    gx3, *r3 = port.backward(P[2], a2, g3)
    gx2, *r2 = port.backward(P[1], a1, gx3)
    g1 = np.where(a1 > 0, gx2, 0.0)                      # Relu::backward
    gx1, *r1 = port.backward(P[0], a0, g1)
    check_close("chain grad_x", _np(grads.grad_x), gx1.T, dtype_name)
    for i, r in enumerate((r1, r2, r3)):
        _, du1, du2, db = oracle.grads_to_abi(np.zeros((1, 1)), *r)
        b = grads.layers[i]
        check_close(f"chain dU1s[{i}]", _np(b.dU1s), du1, dtype_name)
        check_close(f"chain dU2s[{i}]", _np(b.dU2s), du2, dtype_name)
        check_close(f"chain db[{i}]", _np(b.db), db, dtype_name)


@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
@pytest.mark.parametrize("unfused", [False, True])
def test_fused_relu_mask_is_exact_at_scale(skl, dtype_name, unfused):
    """The backward's fused ReLU mask (FUSE_RELU_IN, Relu::backward nn_layers.cpp:347-354)
    equals the plain backward's grad_x times (x > 0), bitwise, at a size where
    every CTA runs several output tiles and more than one row tile (the mask
    tiles are prefetched one tile ahead), with ragged T and N2 % 128 != 0."""
    if unfused and os.environ.get("SKL_FORCE_UNFUSED") is None:
        pytest.skip("unfused path is exercised in a separate process (SKL_FORCE_UNFUSED=1)")
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    d_in, d_out, L, k, T = 1088, 512, 2, 64, 20003
    lyr = skl.SkLinear(d_in, d_out, L, k, seed=77, dtype=dtype)
    gen = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn(T, d_in, device="cuda", generator=gen).to(td)
    g = torch.randn(T, d_out, device="cuda", generator=gen).to(td)
    s = lyr.shape
    ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device="cuda")
    out = []
    for fuse in (0, skl.FUSE_RELU_IN):
        gx = torch.empty(T, d_in, dtype=td, device="cuda")
        du1 = torch.empty(L, k, d_out, device="cuda")
        du2 = torch.empty(L, d_in, k, device="cuda")
        db = torch.empty(d_out, device="cuda")
        skl.backward_phase(s, skl.BWD_ALL, g, x, None, lyr.S1s, lyr.S2s, lyr.U1s, lyr.U2s, gx, du1, du2, db, ws,
                           fuse=fuse)
        out.append((gx, du1, du2, db))
    torch.cuda.synchronize()
    plain, fused = out
    assert torch.equal(fused[0], plain[0] * (x > 0).to(td))
    for a, b in zip(fused[1:], plain[1:]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
def test_chain_relu_bits_match_x_mask_bitwise(skl, dtype_name):
    """The 1-bit ReLU mask carried from FFN1's forward to FFN2's backward
    (SKL_FUSE_RELU_BITS) gives bitwise the same activations and gradients as
    re-reading the ReLU output, at a c5 FFN shape with ragged T and several
    row tiles per CTA."""
    from paper_2601_15473_b200.model import Relu, SkChain
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    k = 128 if dtype_name == "bf16" else 64  # TF32: R = 256 stays on the CTA-pair kernel
    l1 = skl.SkLinear(768, 3072, 2, k, seed=11, dtype=dtype)
    l2 = skl.SkLinear(3072, 768, 2, k, seed=12, dtype=dtype)
    if not (skl.relu_bits_supported(l1.shape) and skl.relu_bits_supported(l2.shape)):
        assert os.environ.get("SKL_FORCE_UNFUSED") is not None  # only the unfused chain lacks them
        pytest.skip("1-bit masks are a fused-kernel feature")
    T = 20003  # > 74 pair tiles: the bits of the next row tile are prefetched across tiles
    gen = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(T, 768, device="cuda", generator=gen).to(td)
    g = torch.randn(T, 768, device="cuda", generator=gen).to(td)
    res = []
    for bits in (False, True):
        chain = SkChain([l1, Relu(), l2], relu_bits=bits)
        y = chain.forward(x)
        assert (chain.steps[1].bits is not None) == bits
        grads, _ = chain.backward(g, overlap=False)
        torch.cuda.synchronize()
        res.append((y.clone(), grads.grad_x.clone(), [(b.dU1s.clone(), b.dU2s.clone(), b.db.clone())
                                                       for b in grads.layers]))
    (y0, gx0, l0), (y1, gx1, lb) = res
    assert torch.equal(y0, y1) and torch.equal(gx0, gx1)
    for a, b in zip(l0, lb):
        for u, v in zip(a, b):
            assert torch.equal(u, v)
    # the bits are the ReLU output's sign, bit (c % 32) of word c / 32
    chain = SkChain([l1, Relu(), l2], relu_bits=True)
    h = chain.forward(x)
    bits = chain.steps[1].bits
    a1 = chain.steps[1].x
    w = skl.relu_bits_row_words(3072)
    assert bits.shape == (T, w)
    cols = torch.arange(3072, device="cuda")
    got = (bits[:, cols // 32] >> (cols % 32)) & 1
    assert torch.equal(got.bool(), a1 > 0)


def test_bert_stack_overlapped_dp_step_runs(skl):
    """Config 5 at reduced depth: the BERT FFN/proj stack with the per-layer
    all-reduce schedules (whole bucket after each layer's fused backward, or the
    phased split) on a world-1 NCCL group gives the same gradients as the plain
    backward."""
    import socket
    import torch.distributed as dist
    from paper_2601_15473_b200.model import bert_ffn_stack, wait_all
    chain = bert_ffn_stack(num_layers=2)
    T = 1024
    x = torch.randn(T, 768, device="cuda").to(torch.bfloat16)
    g = torch.randn(T, 768, device="cuda").to(torch.bfloat16)
    chain.forward(x)
    ref, _ = chain.backward(g, overlap=False)
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port_ = sock.getsockname()[1]
    sock.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port_}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        for phased in (False, True):  # per-layer fused backward + bucket all-reduce / phased split
            got, works = chain.backward(g, overlap=True, phased=phased)
            assert len(works) == (2 if phased else 1) * len(chain.steps)
            wait_all(works)
            torch.cuda.synchronize()
            assert torch.equal(got.grad_x, ref.grad_x)
            for a, b in zip(got.layers, ref.layers):
                rel = (a.flat - b.flat).norm() / b.flat.norm()
                assert rel < 1e-5, rel
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
@pytest.mark.parametrize("d_in,d_out,L,k", [(256, 384, 2, 64), (96, 160, 3, 16)])
def test_from_dense_matches_oracle(skl, port, dtype_name, d_in, d_out, L, k):
    """sk_linear_from_dense on device (tcgen05 GEMMs) == the reference algorithm
    (u1 = s1·W, u2 = W·s2ᵀ, nn_layers.cpp:149-160) on the same rounded W."""
    import oracle
    from tests._util import check_close
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    gen = torch.Generator(device="cuda").manual_seed(3)
    W = (torch.randn(d_out, d_in, device="cuda", generator=gen) * 0.05).to(td)
    b = torch.randn(d_out, device="cuda", generator=gen).to(td)
    lyr = skl.SkLinear.from_dense(W, b, L, k, seed=77, dtype=dtype)
    torch.cuda.synchronize()
    P = oracle.sk_linear_from_dense(port, _np(W), L, k, 77)
    abi = oracle.to_abi(P)
    from tests._util import bf16_round, f32_round
    rnd = bf16_round if dtype == skl.BF16 else f32_round   # direct f64 -> element rounding (no double rounding)
    assert np.array_equal(_np(lyr.S2s), rnd(abi["S2s"]))   # sketches bit-exact
    assert np.array_equal(_np(lyr.S1s), rnd(abi["S1s"]))
    check_close("from_dense U1s", _np(lyr.U1s), abi["U1s"], dtype_name)
    check_close("from_dense U2s", _np(lyr.U2s), abi["U2s"], dtype_name)
    assert torch.equal(lyr.bias, b)


# --------------------------------------------------------------------------- SkConv2d
@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
@pytest.mark.parametrize("stride,pad", [(1, 1), (2, 0)])
def test_skconv2d_matches_reference(skl, ref, dtype_name, stride, pad):
    """SkConv2d forward/backward on device (im2col -> SKLinear -> NCHW, col2im)
    vs the REFERENCE's own SkConv2d (oracle/_ref) on the same parameters."""
    import oracle
    from paper_2601_15473_b200.conv import ConvShape, SkConv2d
    from tests._util import check_close
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    cs = ConvShape(c_in=8, c_out=24, kernel_h=3, kernel_w=3, stride=stride, padding=pad)
    conv = SkConv2d(cs, 2, 16, seed=9, dtype=dtype)
    gen = torch.Generator(device="cuda").manual_seed(4)
    conv.inner.bias.copy_((torch.randn(24, device="cuda", generator=gen) * 0.2).to(td))
    B, H, W = 3, 10, 11
    x = torch.randn(B, 8, H, W, device="cuda", generator=gen).to(td)
    keep = {}
    y = conv.forward(x, keep=keep)
    g = torch.randn_like(y.float()).to(td)
    gr = conv.backward(x, g, keep=keep)
    gr2 = conv.backward(x, g)                       # recompute path (no kept patches)
    torch.cuda.synchronize()
    s = conv.inner
    P = oracle.from_abi(s.d_in, s.d_out, _np(s.S1s), _np(s.U1s), _np(s.U2s), _np(s.S2s))
    geo = (cs.c_in, cs.c_out, cs.kernel_h, cs.kernel_w, cs.stride, cs.padding)
    y_ref = oracle.skconv_forward(ref, geo, P, _np(s.bias), _np(x))
    check_close("conv y", _np(y), y_ref, dtype_name)
    gx, gu1, gu2, gb = oracle.skconv_backward(ref, geo, P, _np(x), _np(g))
    _, du1, du2, db = oracle.grads_to_abi(np.zeros((1, 1)), gu1, gu2, gb)
    for tag, G in (("kept", gr), ("recompute", gr2)):
        check_close(f"conv grad_x ({tag})", _np(G.grad_x), gx, dtype_name)
        check_close(f"conv dU1s ({tag})", _np(G.grad_u1), du1, dtype_name)
        check_close(f"conv dU2s ({tag})", _np(G.grad_u2), du2, dtype_name)
        check_close(f"conv db ({tag})", _np(G.grad_b), db, dtype_name)


# --------------------------------------------------------------------------- edge cases and full-size properties
@pytest.mark.parametrize("T", [0, 1, 7, 255, 257])
def test_edge_token_counts(skl, port, T):
    """Empty, single-token and ragged batches (the reference handles any T,
    nn_layers.cpp:61-101): T = 0 is a no-op forward and zero gradients."""
    import oracle
    from tests._util import check_close
    d_in, d_out, L, k = 256, 384, 2, 64
    s, (S1s, S2s, U1s, U2s), X, G, B, P, x64, g64, b64 = _make_case(skl, port, d_in, d_out, L, k, max(T, 1), skl.BF16)
    X, G = X[:T], G[:T]
    y = torch.full((T, d_out), 7.0, dtype=torch.bfloat16, device="cuda")
    saved = torch.empty(L * k, max(8, (T + 7) // 8 * 8), dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device="cuda")
    skl.forward(s, X, S1s, S2s, U1s, U2s, B, y, saved, ws)
    gx = torch.empty(T, d_in, dtype=torch.bfloat16, device="cuda")
    du1 = torch.full((L, k, d_out), 5.0, device="cuda")
    du2 = torch.full((L, d_in, k), 5.0, device="cuda")
    db = torch.full((d_out,), 5.0, device="cuda")
    skl.backward(s, G, X, saved, S1s, S2s, U1s, U2s, gx, du1, du2, db, ws)
    torch.cuda.synchronize()
    if T == 0:
        assert du1.abs().max().item() == 0 and du2.abs().max().item() == 0 and db.abs().max().item() == 0
        return
    x64, g64 = x64[:, :T].copy(), g64[:, :T].copy()
    check_close(f"y T={T}", _np(y), port.forward(P, b64, x64).T, "bf16")
    rgx, rgu1, rgu2, rgb = oracle.grads_to_abi(*port.backward(P, x64, g64))
    check_close(f"grad_x T={T}", _np(gx), rgx, "bf16")
    check_close(f"dU1s T={T}", _np(du1), rgu1, "bf16")
    check_close(f"dU2s T={T}", _np(du2), rgu2, "bf16")
    check_close(f"db T={T}", _np(db), rgb, "bf16")


def test_c3_shape_slice_matches_oracle(skl, port):
    """BASELINE config 3 shape (4096 -> 4096, L=3, k=256: R = 1536, the unfused
    chain) on a 512-token slice vs the f64 oracle (c3 parity on a
    token slice; the f64 reference is too slow at 64k tokens)."""
    import oracle
    from tests._util import check_close
    d_in, d_out, L, k, T = 4096, 4096, 3, 256, 512
    s, (S1s, S2s, U1s, U2s), X, G, B, P, x64, g64, b64 = _make_case(skl, port, d_in, d_out, L, k, T, skl.BF16)
    y = torch.empty(T, d_out, dtype=torch.bfloat16, device="cuda")
    saved = torch.empty(L * k, T, dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device="cuda")
    skl.forward(s, X, S1s, S2s, U1s, U2s, B, y, saved, ws)
    gx = torch.empty(T, d_in, dtype=torch.bfloat16, device="cuda")
    du1 = torch.empty(L, k, d_out, device="cuda")
    du2 = torch.empty(L, d_in, k, device="cuda")
    db = torch.empty(d_out, device="cuda")
    skl.backward(s, G, X, saved, S1s, S2s, U1s, U2s, gx, du1, du2, db, ws)
    torch.cuda.synchronize()
    check_close("c3 y", _np(y), port.forward(P, b64, x64).T, "bf16")
    rgx, rgu1, rgu2, rgb = oracle.grads_to_abi(*port.backward(P, x64, g64))
    check_close("c3 grad_x", _np(gx), rgx, "bf16")
    check_close("c3 dU1s", _np(du1), rgu1, "bf16")
    check_close("c3 dU2s", _np(du2), rgu2, "bf16")
    check_close("c3 db", _np(db), rgb, "bf16")


@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
def test_full_size_c2_properties(skl, dtype_name):
    """BASELINE config 2 at its full 32768 tokens, checked through
    size-independent properties (the f64 oracle would take minutes):
      * row independence: the forward of a token slice equals the same rows
        of the full forward, bitwise;
      * gradient additivity: dU1s/dU2s/db of the batch == the sums over two
        ragged halves (reduction over tokens, nn_layers.cpp:90-99);
      * determinism: a second backward is bitwise identical."""
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    d_in, d_out, L, k, T = 768, 3072, 2, 128, 32768
    lyr = skl.SkLinear(d_in, d_out, L, k, seed=42, dtype=dtype)
    gen = torch.Generator(device="cuda").manual_seed(1)
    lyr.bias.copy_(torch.randn(d_out, device="cuda", generator=gen).to(td))
    X = torch.randn(T, d_in, device="cuda", generator=gen).to(td)
    G = torch.randn(T, d_out, device="cuda", generator=gen).to(td)
    y = lyr.forward(X)
    y_part = lyr.forward(X[1000:3000].contiguous())
    torch.cuda.synchronize()
    assert torch.equal(y[1000:3000], y_part)
    h = 12345
    full = lyr.backward(X, G)
    a = lyr.backward(X[:h].contiguous(), G[:h].contiguous())
    b = lyr.backward(X[h:].contiguous(), G[h:].contiguous())
    again = lyr.backward(X, G)
    torch.cuda.synchronize()
    for name, f, p, q in (("dU1s", full.grad_u1, a.grad_u1, b.grad_u1), ("dU2s", full.grad_u2, a.grad_u2, b.grad_u2),
                          ("db", full.grad_b, a.grad_b, b.grad_b)):
        rel = ((f - (p + q)).norm() / f.norm()).item()
        assert rel < 1e-4, (name, rel)  # fp32 sums of 32768 tokens in a different split order
    assert torch.equal(full.grad_x[:h], a.grad_x) and torch.equal(full.grad_x[h:], b.grad_x)
    for u, v in zip((full.grad_x, full.grad_u1, full.grad_u2, full.grad_b),
                    (again.grad_x, again.grad_u1, again.grad_u2, again.grad_b)):
        assert torch.equal(u, v)


def test_unfused_path_parity_in_subprocess():
    """Every parity test above once more with SKL_FORCE_UNFUSED=1 (the env switch is
    read once per process): the unfused GEMM chain -- the path for R > 512 --
    against the same oracle gates."""
    import subprocess
    import sys
    if os.environ.get("SKL_FORCE_UNFUSED") is not None:
        pytest.skip("already the unfused process")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SKL_FORCE_UNFUSED="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_gpu.py", "-k",
                        "parity or mask_is_exact or chain or edge or deterministic"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]


def test_fused_path_small_batches_in_subprocess():
    """The parity tests once more with SKL_SMALL=0: batches of T <= 128 tokens (the
    c1 shape, T = 64; ragged 50 / 77) take the fused tcgen05 kernels instead of the
    small-batch path (small.cu), against the same oracle gates."""
    import subprocess
    import sys
    if os.environ.get("SKL_SMALL") is not None:
        pytest.skip("already the SKL_SMALL process")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SKL_SMALL="0")
    # the parametrised cases with T <= 128 (ids end in the token count) and the small-shape tests
    sel = ("(parity and (-64] or -50] or -77] or -20])) or c1 or gradcheck or identity or criterion or zero or "
           "ragged or deterministic_small")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_gpu.py", "tests/test_gpu_shapes.py",
                        "-k", sel],
                       env=env, cwd=root, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]


def test_small_batch_path_is_deterministic_and_matches_fused(skl, port):
    """T <= 128: the small-batch path (fp32 FMA over parameter slices) against the
    oracle at the c1 shape in both dtypes, bitwise reproducible, for every phase
    split and a fused ReLU / x-mask."""
    import oracle
    from tests._util import check_close
    for kind, name in ((skl.F32_TF32, "tf32"), (skl.BF16, "bf16")):
        d_in, d_out, L, k, T = 1024, 1024, 1, 64, 64
        s, (S1s, S2s, U1s, U2s), X, G, B, P, x64, g64, b64 = _make_case(skl, port, d_in, d_out, L, k, T, kind)
        td = skl.torch_dtype(kind)
        ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device="cuda")
        sv = torch.empty(L * k, (T + 7) // 8 * 8, dtype=td, device="cuda")
        runs = []
        for _ in range(2):
            y = torch.empty(T, d_out, dtype=td, device="cuda")
            skl.forward(s, X, S1s, S2s, U1s, U2s, B, y, sv, ws)
            gx = torch.empty(T, d_in, dtype=td, device="cuda")
            du1 = torch.empty(L, k, d_out, device="cuda")
            du2 = torch.empty(L, d_in, k, device="cuda")
            db = torch.empty(d_out, device="cuda")
            skl.backward(s, G, X, sv, S1s, S2s, U1s, U2s, gx, du1, du2, db, ws)
            runs.append((y, gx, du1, du2, db))
        torch.cuda.synchronize()
        for a, b in zip(*runs):
            assert torch.equal(a, b)
        y, gx, du1, du2, db = runs[0]
        check_close(f"small y {name}", _np(y), port.forward(P, b64, x64).T, name)
        rgx, rgu1, rgu2, rgb = oracle.grads_to_abi(*port.backward(P, x64, g64))
        check_close(f"small grad_x {name}", _np(gx), rgx, name)
        check_close(f"small dU1s {name}", _np(du1), rgu1, name)
        check_close(f"small dU2s {name}", _np(du2), rgu2, name)
        check_close(f"small db {name}", _np(db), rgb, name)
        # the DP phases give the same gradients bitwise
        du1p, du2p, dbp = torch.empty_like(du1), torch.empty_like(du2), torch.empty_like(db)
        gxp = torch.empty_like(gx)
        skl.backward_phase(s, skl.BWD_DU1_DB, G, X, sv, S1s, S2s, U1s, U2s, None, du1p, None, dbp, ws)
        skl.backward_phase(s, skl.BWD_DX_DU2, G, X, sv, S1s, S2s, U1s, U2s, gxp, None, du2p, None, ws)
        torch.cuda.synchronize()
        assert torch.equal(du1p, du1) and torch.equal(du2p, du2) and torch.equal(dbp, db) and torch.equal(gxp, gx)


def test_rsplit_path_parity_in_subprocess():
    """The parity tests once more with SKL_B2B_RSPLIT=1: shapes with R > 512 (the
    R = 768 / 640 / 2048 and c3 R = 1536 cases) run on the R-split clusters (H on
    chip, GEMM2 partials chained over DSMEM in fixed pair order) against the same
    oracle gates, and stay bitwise deterministic."""
    import subprocess
    import sys
    if os.environ.get("SKL_B2B_RSPLIT") is not None:
        pytest.skip("already the R-split process")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SKL_B2B_RSPLIT="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_gpu.py", "-k",
                        "parity_bf16 or c3_shape or rsplit_is_deterministic"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]


@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
@pytest.mark.parametrize("d_in,d_out,L,k,T", [
    (1024, 1024, 1, 64, 1),     # one token
    (512, 768, 3, 48, 128),     # the largest small batch, L = 3, k % 64 != 0
    (512, 768, 3, 48, 129),     # one past it: the fused kernels
    (64, 4096, 2, 32, 17),      # wide output, ragged T
])
def test_small_batch_edges_match_oracle(skl, port, dtype_name, d_in, d_out, L, k, T):
    """Edges of the small-batch path (T <= 128) and its hand-over to the fused
    kernels at T = 129: forward and every gradient against the f64 oracle."""
    import oracle
    from tests._util import check_close
    kind = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    s, (S1s, S2s, U1s, U2s), X, G, B, P, x64, g64, b64 = _make_case(skl, port, d_in, d_out, L, k, T, kind)
    td = skl.torch_dtype(kind)
    ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device="cuda")
    sv = torch.empty(L * k, (T + 7) // 8 * 8, dtype=td, device="cuda")
    y = torch.empty(T, d_out, dtype=td, device="cuda")
    skl.forward(s, X, S1s, S2s, U1s, U2s, B, y, sv, ws)
    gx = torch.empty(T, d_in, dtype=td, device="cuda")
    du1 = torch.empty(L, k, d_out, device="cuda")
    du2 = torch.empty(L, d_in, k, device="cuda")
    db = torch.empty(d_out, device="cuda")
    skl.backward(s, G, X, sv, S1s, S2s, U1s, U2s, gx, du1, du2, db, ws)
    torch.cuda.synchronize()
    check_close("y", _np(y), port.forward(P, b64, x64).T, dtype_name)
    rgx, rgu1, rgu2, rgb = oracle.grads_to_abi(*port.backward(P, x64, g64))
    check_close("grad_x", _np(gx), rgx, dtype_name)
    check_close("dU1s", _np(du1), rgu1, dtype_name)
    check_close("dU2s", _np(du2), rgu2, dtype_name)
    check_close("db", _np(db), rgb, dtype_name)


@pytest.mark.parametrize("T", [200, 256, 513, 4096 + 77])
def test_double_tile_backward_edges_match_oracle(skl, port, T):
    """The double-tile R = 256 backward at one (half-empty) double tile, exactly
    one, an odd tile count and a ragged multi-wave T; the DP phase split and the
    recompute path (no saved projection) give the same dX bitwise (same b2b
    kernel) and gradients within the gates (the phased du launches may split T
    differently, so their fp32 sums may round differently)."""
    import oracle
    from tests._util import check_close
    d_in, d_out, L, k = 768, 768, 1, 128
    s, (S1s, S2s, U1s, U2s), X, G, B, P, x64, g64, b64 = _make_case(skl, port, d_in, d_out, L, k, T, skl.BF16)
    ws = torch.empty(max(skl.workspace_size(s, T)), dtype=torch.uint8, device="cuda")
    sv = torch.empty(L * k, (T + 7) // 8 * 8, dtype=torch.bfloat16, device="cuda")
    skl.forward(s, X, S1s, S2s, U1s, U2s, B, torch.empty(T, d_out, dtype=torch.bfloat16, device="cuda"), sv, ws)
    gx = torch.empty(T, d_in, dtype=torch.bfloat16, device="cuda")
    du1, du2, db = torch.empty(L, k, d_out, device="cuda"), torch.empty(L, d_in, k, device="cuda"), torch.empty(d_out, device="cuda")
    skl.backward(s, G, X, sv, S1s, S2s, U1s, U2s, gx, du1, du2, db, ws)
    torch.cuda.synchronize()
    rgx, rgu1, rgu2, rgb = oracle.grads_to_abi(*port.backward(P, x64, g64))
    check_close("grad_x", _np(gx), rgx, "bf16")
    check_close("dU1s", _np(du1), rgu1, "bf16")
    check_close("dU2s", _np(du2), rgu2, "bf16")
    check_close("db", _np(db), rgb, "bf16")
    gxp, du2p = torch.empty_like(gx), torch.empty_like(du2)
    du1p, dbp = torch.empty_like(du1), torch.empty_like(db)
    skl.backward_phase(s, skl.BWD_DU1_DB, G, X, None, S1s, S2s, U1s, U2s, None, du1p, None, dbp, ws)
    skl.backward_phase(s, skl.BWD_DX_DU2, G, X, None, S1s, S2s, U1s, U2s, gxp, None, du2p, None, ws)
    torch.cuda.synchronize()
    assert torch.equal(gxp, gx)
    check_close("dU1s (phased, recomputed saved)", _np(du1p), rgu1, "bf16")
    check_close("dU2s (phased)", _np(du2p), rgu2, "bf16")
    check_close("db (phased)", _np(dbp), rgb, "bf16")


def test_store_and_tile_variants_are_bitwise_identical(tmp_path):
    """The round-2 store and tiling variants change where bytes go, not the
    arithmetic: the saved columns through per-warp TMA stores (SKL_SAVE_TMA) or
    per-thread stores, per-warp or group output stores (SKL_B2B_WSTORE), and the
    double-tile R = 256 backward (SKL_B2B_DT) or one tile per pair give bitwise
    the same y, saved projection, dX, dU1s, dU2s and db."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    runs = {"default": {}, "no_tma_saves": {"SKL_SAVE_TMA": "0"}, "group_stores": {"SKL_B2B_WSTORE": "0"},
            "single_tiles": {"SKL_B2B_DT": "0"}}
    outs = {}
    for name, extra in runs.items():
        f = str(tmp_path / f"{name}.pt")
        r = subprocess.run([sys.executable, "tests/store_paths_case.py", f], env=dict(os.environ, **extra), cwd=root,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        outs[name] = torch.load(f)
    for name in runs:
        for shape, tensors in outs["default"].items():
            for key, t in tensors.items():
                assert torch.equal(t, outs[name][shape][key]), f"{name}: {shape} {key} differs"


def test_rsplit_is_deterministic(skl):
    """R > 512 backward twice: bitwise identical (both the default chain and, in
    the SKL_B2B_RSPLIT=1 subprocess, the DSMEM partial chain)."""
    d_in, d_out, L, k, T = 2048, 1024, 4, 256, 1500
    lyr = skl.SkLinear(d_in, d_out, L, k, seed=5, dtype=skl.BF16)
    X = torch.randn(T, d_in, device="cuda").to(torch.bfloat16)
    G = torch.randn(T, d_out, device="cuda").to(torch.bfloat16)
    y1, y2 = lyr.forward(X), lyr.forward(X)
    a, b = lyr.backward(X, G), lyr.backward(X, G)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    for u, v in zip((a.grad_x, a.grad_u1, a.grad_u2, a.grad_b), (b.grad_x, b.grad_u1, b.grad_u2, b.grad_b)):
        assert torch.equal(u, v)


def test_graph_replay_is_bitwise_equal(skl):
    """A fixed-shape chain step (forward + backward through SkChain, 2 encoder
    layers of the c5 stack) recorded with graphs.capture replays to bitwise the
    eager results -- what bench.py relies on for the launch-bound lines."""
    from paper_2601_15473_b200.graphs import capture
    from paper_2601_15473_b200.model import bert_ffn_stack
    chain = bert_ffn_stack(num_layers=1)
    T = 1000
    gen = torch.Generator(device="cuda").manual_seed(21)
    x = torch.randn(T, 768, device="cuda", generator=gen).to(torch.bfloat16)
    g = torch.randn(T, 768, device="cuda", generator=gen).to(torch.bfloat16)
    buckets = chain.allocate_grads("cuda")

    def step():
        chain.forward(x)
        chain.backward(g, buckets=buckets, need_grad_x=False, overlap=False)

    step()
    torch.cuda.synchronize()
    ref = [b.flat.clone() for b in buckets]
    for b in buckets:
        b.flat.zero_()
    gr = capture(step)
    for b in buckets:
        b.flat.zero_()
    gr.replay()
    torch.cuda.synchronize()
    for a, b in zip(ref, buckets):
        assert torch.equal(a, b.flat)


def test_from_dense_is_unbiased_over_sketch_seeds(skl):
    """Acceptance criterion 2 (acceptance.cpp:113-156) on the device
    path: over 5000 sketch seeds, the seed-averaged output of sk_linear_from_dense(W)
    is within 3 standard errors of the dense layer for l = 1 and l = 4, and
    var(l = 4) / var(l = 1) lies in [0.2, 0.35].  Shapes are widened to the ABI's
    16-byte row alignment (d_in 6 -> 16, k 3 -> 4); TF32 I/O."""
    from paper_2601_15473_b200 import derive_seed
    dtype = skl.F32_TF32
    d_in, d_out, k, seeds = 16, 8, 4, 5000
    gen = torch.Generator(device="cuda").manual_seed(201)
    W = torch.randn(d_out, d_in, device="cuda", generator=gen)
    b = 0.05 * torch.arange(1, d_out + 1, device="cuda", dtype=torch.float32)
    x = torch.randn(2, d_in, device="cuda", generator=gen)
    expect = x.double() @ W.double().T + b.double()             # [2, d_out]
    slack = 2e-3 * expect.abs() + 1e-4                          # TF32 operand rounding, far below 3 SE

    def run(l, tag):
        ys = torch.stack([skl.SkLinear.from_dense(W, b, l, k, seed=derive_seed(tag, s), dtype=dtype).forward(x).double()
                          for s in range(seeds)])               # [seeds, 2, d_out]
        mean, var = ys.mean(0), ys.var(0, unbiased=True)
        z = ((mean - expect).abs() - slack).clamp(min=0) / (var / seeds).sqrt()
        return z.max().item(), var.mean().item()

    z1, v1 = run(1, 1000)
    z4, v4 = run(4, 2000)
    assert z1 <= 3.0 and z4 <= 3.0, (z1, z4)
    assert 0.2 <= v4 / v1 <= 0.35, v4 / v1


def test_sketched_conv_from_dense_is_unbiased(skl):
    """test_nn_montecarlo.cpp:80-114 on the device path: a SkConv2d whose inner
    SKLinear comes from sk_linear_from_dense of a dense conv's lowered weight
    (sk_conv2d_from_dense) averages, over 600 sketch seeds, to the dense conv within
    3 standard errors per output.  Channels widened 2 -> 4 for the ABI's 16-byte rows."""
    import torch.nn.functional as F
    from paper_2601_15473_b200 import derive_seed
    from paper_2601_15473_b200.conv import ConvShape, SkConv2d
    c_in, c_out, kh = 4, 4, 3
    shape = ConvShape(c_in, c_out, kh, kh, 1, 0)
    gen = torch.Generator(device="cuda").manual_seed(31)
    Wc = torch.randn(c_out, c_in, kh, kh, device="cuda", generator=gen)      # [c_out][c_in][kh][kw]
    b = torch.tensor([0.2, -0.1, 0.05, 0.0], device="cuda")
    x = torch.randn(1, c_in, 5, 5, device="cuda", generator=gen)
    expect = F.conv2d(x.double(), Wc.double(), b.double())                   # [1, c_out, 3, 3]
    W = Wc.reshape(c_out, c_in * kh * kh)   # lowered feature order (channel, kernel row, kernel col)
    ys = []
    for s in range(600):
        inner = skl.SkLinear.from_dense(W, b, 1, 4, seed=derive_seed(888, s), dtype=skl.F32_TF32)
        ys.append(SkConv2d(shape, 1, 4, dtype=skl.F32_TF32, inner=inner).forward(x).double())
    ys = torch.stack(ys)
    mean, se = ys.mean(0), ys.std(0, unbiased=True) / 600 ** 0.5
    slack = 2e-3 * expect.abs() + 1e-4  # TF32 operand rounding
    assert bool(((mean - expect).abs() <= 3 * se + slack).all()), ((mean - expect).abs() / se).max()


@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
def test_from_dense_zero_weights_leaves_bias(skl, dtype_name):
    """test_nn_layers.cpp:99-111: sk_linear_from_dense of a zero W has zero U1s / U2s
    and its forward is exactly the bias, on the device path."""
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    d_in, d_out = 16, 8
    b = torch.tensor([1.5, -2.0, 0.25, 3.0, -1.0, 0.5, 0.0, 2.0], device="cuda").to(td)
    lyr = skl.SkLinear.from_dense(torch.zeros(d_out, d_in, device="cuda", dtype=td), b, 2, 8, seed=17, dtype=dtype)
    assert not bool(lyr.U1s.any()) and not bool(lyr.U2s.any())
    x = torch.randn(40, d_in, device="cuda").to(td)
    y = lyr.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(y, b.expand(40, d_out))


@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
def test_conv_zero_input_gives_bias_colored_maps(skl, dtype_name):
    """test_nn_layers.cpp:263-281 on the device path (channels widened for the
    ABI's 16-byte rows): a zero image maps to each output channel's bias."""
    from paper_2601_15473_b200.conv import ConvShape, SkConv2d
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    conv = SkConv2d(ConvShape(8, 8, 3, 3, 1, 0), 1, 8, seed=59, dtype=dtype)
    bias = torch.linspace(-0.7, 0.7, 8, device="cuda").to(td)
    conv.inner.bias.copy_(bias)
    y = conv.forward(torch.zeros(2, 8, 5, 5, device="cuda", dtype=td))
    torch.cuda.synchronize()
    assert y.shape == (2, 8, 3, 3)
    assert torch.equal(y, bias.view(1, 8, 1, 1).expand(2, 8, 3, 3))
