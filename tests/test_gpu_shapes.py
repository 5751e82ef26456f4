"""GPU parity at the shapes the reference itself tests, UNMODIFIED: rows that
are not 16-byte multiples (d_in = 6, k = 3, 2 conv channels, ...) go through the
same kernels on zero-padded copies (skl.cu, padded dispatch) and must match the
oracle at the bf16 / TF32 gates.  Also the DenseLinear layer of a chain and the
c1 end-to-end tolerance against the reference's unrounded f64 output.

Run on a B200:  python -m pytest tests -m gpu -x -q
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def skl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_15473_b200 as skl
    skl.lib()
    return skl


def _np(t):
    return t.detach().double().cpu().numpy()


def _tdev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def _variant(skl, dtype):
    return "bf16" if dtype == skl.BF16 else "tf32"


def _layer_f64(skl, layer):
    import oracle
    return oracle.from_abi(layer.d_in, layer.d_out, _np(layer.S1s), _np(layer.U1s), _np(layer.U2s), _np(layer.S2s))


# --------------------------------------------------------------------------- ragged parity sweep
RAGGED = [
    (6, 8, 2, 3, 2),          # test_nn_layers.cpp:158 GradCheck / acceptance.cpp:113 shape
    (5, 3, 2, 2, 4),          # test_nn_layers.cpp:92 zero-input shape (sk_linear_fresh(5, 3, 2, 2, 11))
    (7, 13, 1, 5, 33),        # everything odd
    (100, 36, 2, 10, 257),    # d_out only 4-aligned (TF32 ok, bf16 padded)
    (770, 3070, 1, 37, 300),  # near-c2 widths, odd k
    (1023, 1025, 2, 64, 129), # k % 64 == 0 but ragged d (direct mode off: padded dims are direct-capable)
]


@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
@pytest.mark.parametrize("d_in,d_out,L,k,T", RAGGED)
def test_ragged_shapes_match_oracle(skl, port, dtype_name, d_in, d_out, L, k, T):
    """Forward, backward (fused and phased) and the saved-projection recompute
    at ragged shapes vs the f64 oracle on the same rounded values."""
    import oracle
    from tests._util import check_close
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    layer = skl.SkLinear(d_in, d_out, L, k, seed=42, dtype=dtype)
    x, g, b = oracle.inputs(d_in, d_out, T, 42, port)
    X, G = _tdev(x.T, td), _tdev(g.T, td)
    layer.bias.copy_(_tdev(b, td))
    P = _layer_f64(skl, layer)
    x64, g64, b64 = _np(X).T.copy(), _np(G).T.copy(), _np(layer.bias)
    saved = torch.empty(L * k, (T + 7) // 8 * 8, dtype=td, device="cuda")
    y = layer.forward(X, saved=saved)
    gr = layer.backward(X, G, saved=saved)
    torch.cuda.synchronize()
    v = dtype_name
    check_close("y", _np(y), port.forward(P, b64, x64).T, v)
    rgx, rgu1, rgu2, rgb = oracle.grads_to_abi(*port.backward(P, x64, g64))
    check_close("grad_x", _np(gr.grad_x), rgx, v)
    check_close("dU1s", _np(gr.grad_u1), rgu1, v)
    check_close("dU2s", _np(gr.grad_u2), rgu2, v)
    check_close("db", _np(gr.grad_b), rgb, v)
    # phased (DP) backward and the recompute path give the same gradients
    s = layer.shape
    ws = layer.workspace(T)
    du1, du2 = torch.empty_like(gr.grad_u1), torch.empty_like(gr.grad_u2)
    db, gx = torch.empty_like(gr.grad_b), torch.empty_like(gr.grad_x)
    skl.backward_phase(s, skl.BWD_DU1_DB, G, X, None, layer.S1s, layer.S2s, layer.U1s, layer.U2s, None, du1, None,
                       db, ws)
    skl.backward_phase(s, skl.BWD_DX_DU2, G, X, None, layer.S1s, layer.S2s, layer.U1s, layer.U2s, gx, None, du2,
                       None, ws)
    torch.cuda.synchronize()
    check_close("dU1s(phased)", _np(du1), rgu1, v)
    check_close("dU2s(phased)", _np(du2), rgu2, v)
    check_close("db(phased)", _np(db), rgb, v)
    check_close("grad_x(phased)", _np(gx), rgx, v)


@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
def test_ragged_chain_with_fused_relu_and_bits(skl, port, dtype_name):
    """A Linear/ReLU chain whose widths are ragged (1-bit ReLU masks keep their
    64-column-group layout under padding) equals the oracle chain."""
    import oracle
    from paper_2601_15473_b200.model import Relu, SkChain
    from tests._util import check_close
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    l1 = skl.SkLinear(30, 70, 2, 12, seed=5, dtype=dtype)
    l2 = skl.SkLinear(70, 21, 1, 9, seed=6, dtype=dtype)
    chain = SkChain([l1, Relu(), l2])
    T = 97
    x = port.gaussian_matrix(30, T, 3)
    g = port.gaussian_matrix(21, T, 4)
    X, G = _tdev(x.T, td), _tdev(g.T, td)
    y = chain.forward(X)
    cg, _ = chain.backward(G)
    torch.cuda.synchronize()
    P1, P2 = _layer_f64(skl, l1), _layer_f64(skl, l2)
    x64, g64 = _np(X).T.copy(), _np(G).T.copy()
    z1 = port.forward(P1, np.zeros(70), x64)
    a1 = _np(chain.steps[1].x).T.copy()              # the device's ReLU output (rounded), as the oracle input
    check_close("relu out", a1, np.maximum(z1, 0), dtype_name)
    check_close("y", _np(y), port.forward(P2, np.zeros(21), a1).T, dtype_name)
    gx2, gu1b, gu2b, gbb = port.backward(P2, a1, g64)
    r = oracle.grads_to_abi(gx2, gu1b, gu2b, gbb)
    check_close("layer2 dU1s", _np(cg.layers[1].dU1s), r[1], dtype_name)
    check_close("layer2 dU2s", _np(cg.layers[1].dU2s), r[2], dtype_name)
    gz = gx2 * (a1 > 0)
    rgx, rgu1, rgu2, rgb = oracle.grads_to_abi(*port.backward(P1, x64, gz))
    check_close("layer1 dU1s", _np(cg.layers[0].dU1s), rgu1, dtype_name)
    check_close("grad_x", _np(cg.grad_x), rgx, dtype_name)


# --------------------------------------------------------------------------- the reference's own cases
@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
def test_gradcheck_case_unmodified(skl, port, dtype_name):
    """test_nn_layers.cpp:158-176 at its own shape: sk_linear_fresh(6, 8, 2, 3,
    41), x = random_matrix(6, 2, 43), loss = 1/2 |forward(x)|^2, grads =
    backward(x, forward(x)).  The device backward equals the oracle's, and the
    oracle's gradients pass the reference's central-difference GradCheck
    (oracles.hpp:105-132: h = 1e-6, relative error <= 1e-4) on the same values."""
    import oracle
    from tests._util import check_close
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    layer = skl.SkLinear(6, 8, 2, 3, seed=41, dtype=dtype)
    x = port.gaussian_matrix(6, 2, 43)
    X = _tdev(x.T, td)
    y = layer.forward(X)
    gr = layer.backward(X, y)
    torch.cuda.synchronize()
    P = _layer_f64(skl, layer)
    x64, G64 = _np(X).T.copy(), _np(y).T.copy()
    b0 = np.zeros(8)
    check_close("y", _np(y), port.forward(P, b0, x64).T, dtype_name)
    og = port.backward(P, x64, G64)
    rgx, rgu1, rgu2, rgb = oracle.grads_to_abi(*og)
    check_close("grad_x", _np(gr.grad_x), rgx, dtype_name)
    check_close("dU1s", _np(gr.grad_u1), rgu1, dtype_name)
    check_close("dU2s", _np(gr.grad_u2), rgu2, dtype_name)
    check_close("db", _np(gr.grad_b), rgb, dtype_name)
    # GradCheck of the oracle on these exact values (loss gradient at y = forward(x))
    ga = port.backward(P, x64, port.forward(P, b0, x64))

    def loss():
        yy = port.forward(P, b0, x64)
        return 0.5 * float(np.sum(yy * yy))

    h = 1e-6
    for arr, grad in ((P.u1, ga[1]), (P.u2, ga[2]), (x64, ga[0])):
        flat, gflat = arr.reshape(-1), grad.reshape(-1)
        for i in range(0, flat.size, max(1, flat.size // 12)):
            v = flat[i]
            flat[i] = v + h
            lp = loss()
            flat[i] = v - h
            lm = loss()
            flat[i] = v
            num = (lp - lm) / (2 * h)
            assert abs(num - gflat[i]) <= 1e-4 * max(1.0, abs(num)), (i, num, gflat[i])


@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
def test_identity_sketches_collapse_to_average_dense(skl, port, dtype_name):
    """test_nn_layers.cpp:69-90 at its own shape (d = k = 4, one term, identity
    s1 / s2 injected like SketchOp::with_realized): y = 1/2 (u1 + u2) x + b."""
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    d = 4
    layer = skl.SkLinear(d, d, 1, d, dtype=dtype, _fresh=False)
    u1 = port.gaussian_matrix(d, d, 5)   # random_matrix(d, d, 5)
    u2 = port.gaussian_matrix(d, d, 6)
    eye = np.eye(d)
    layer.S1s[0].copy_(_tdev(eye, td))      # s2ᵀ
    layer.S2s[0].copy_(_tdev(eye, td))      # s1
    layer.U2s[0].copy_(_tdev(u1.T, td))     # u1ᵀ
    layer.U1s[0].copy_(_tdev(u2.T, td))     # u2ᵀ
    layer.bias.copy_(_tdev(np.array([0.1, 0.2, 0.3, 0.4]), td))
    x = port.gaussian_matrix(d, 3, 7)
    X = _tdev(x.T, td)
    y = layer.forward(X)
    torch.cuda.synchronize()
    U1, U2 = _np(layer.U2s[0]).T, _np(layer.U1s[0]).T   # the rounded u1, u2 the device used
    expect = 0.5 * (U1 + U2) @ _np(X).T + _np(layer.bias)[:, None]
    from tests._util import check_close
    check_close("identity-sketch y", _np(y), expect.T, dtype_name)


@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
def test_from_dense_zero_weights_unmodified(skl, dtype_name):
    """test_nn_layers.cpp:99-111 at its own shape: sk_linear_from_dense(Matrix(2, 6),
    {1.5, -2}, 2, 3, 17) has zero U and maps random_matrix(6, 2, 19) to the bias."""
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    b = torch.tensor([1.5, -2.0], device="cuda").to(td)
    lyr = skl.SkLinear.from_dense(torch.zeros(2, 6, device="cuda", dtype=td), b, 2, 3, seed=17, dtype=dtype)
    assert not bool(lyr.U1s.any()) and not bool(lyr.U2s.any())
    y = lyr.forward(torch.randn(2, 6, device="cuda").to(td))
    torch.cuda.synchronize()
    assert torch.equal(y, b.expand(2, 2))


@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
def test_from_dense_ragged_matches_oracle(skl, port, dtype_name):
    """sk_linear_from_dense at ragged d_in / d_out / k: U1s / U2s equal the
    oracle's s1·W / W·s2ᵀ on the same rounded sketches and W."""
    import oracle
    from tests._util import check_close
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    d_in, d_out, L, k = 6, 8, 4, 3
    W = _tdev(port.gaussian_matrix(d_out, d_in, 201), td)
    lyr = skl.SkLinear.from_dense(W, None, L, k, seed=99, dtype=dtype)
    torch.cuda.synchronize()
    P = oracle.sk_linear_from_dense(port, _np(W), L, k, 99)
    # the device sketches are the oracle's, rounded; U from the rounded values
    S1 = _np(lyr.S1s)
    S2 = _np(lyr.S2s)
    w64 = _np(W)
    u1_ref = np.stack([S2[i] @ w64 for i in range(L)])          # s1_i·W   [k, d_in]
    u2_ref = np.stack([w64 @ S1[i] for i in range(L)])          # W·s2_iᵀ  [d_out, k]
    check_close("U2s = u1ᵀ", _np(lyr.U2s), u1_ref.transpose(0, 2, 1), dtype_name)
    check_close("U1s = u2ᵀ", _np(lyr.U1s), u2_ref.transpose(0, 2, 1), dtype_name)
    assert np.allclose(S2, P.s1, rtol=1e-2 if dtype_name == "bf16" else 1e-6, atol=0)


def test_acceptance_criterion_2_unmodified(skl):
    """acceptance.cpp:113-156 at its own shapes (d_in = 6, d_out = 8, batch 2,
    k = 3, 5000 seeds) on the device path (TF32 I/O): the seed-averaged output of
    sk_linear_from_dense(W, b, l, 3, derive_seed(tag, s)) is within 3 standard
    errors of the dense layer for l = 1 and l = 4, and var(l=4)/var(l=1) lies in
    [0.2, 0.35].  W = gaussian_matrix(8, 6, 201), x = gaussian_matrix(6, 2, 202),
    b_i = 0.05 (i + 1), exactly as the reference."""
    import oracle
    from paper_2601_15473_b200 import derive_seed
    port = oracle.Oracle("port")
    dtype = skl.F32_TF32
    d_in, d_out, k, seeds = 6, 8, 3, 5000
    w64 = port.gaussian_matrix(d_out, d_in, 201)
    x64 = port.gaussian_matrix(d_in, 2, 202)
    b64 = 0.05 * np.arange(1, d_out + 1)
    W, b, x = _tdev(w64, torch.float32), _tdev(b64, torch.float32), _tdev(x64.T, torch.float32)
    expect = torch.from_numpy((w64 @ x64 + b64[:, None]).T).cuda()          # [2, d_out] f64
    slack = 2e-3 * expect.abs() + 1e-4                                       # TF32 operand rounding, << 3 SE

    def run(l, tag):
        ys = torch.stack([skl.SkLinear.from_dense(W, b, l, k, seed=derive_seed(tag, s), dtype=dtype).forward(x).double()
                          for s in range(seeds)])
        mean, var = ys.mean(0), ys.var(0, unbiased=True)
        z = ((mean - expect).abs() - slack).clamp(min=0) / (var / seeds).sqrt()
        return z.max().item(), var.mean().item()

    z1, v1 = run(1, 1000)
    z4, v4 = run(4, 2000)
    assert z1 <= 3.0 and z4 <= 3.0, (z1, z4)
    assert 0.2 <= v4 / v1 <= 0.35, v4 / v1


def test_sketched_conv_montecarlo_unmodified(skl):
    """test_nn_montecarlo.cpp:80-114 at its own shape (c_in = c_out = 2, 3x3,
    5x5 image, l = 1, k = 4, 600 seeds, derive_seed(888, s)): the seed-averaged
    sketched conv built from a dense conv is within 3 SE of the dense conv.  The
    dense conv is dense_conv2d_init(shape, 31) (= dense_linear_init of the
    lowered weight) with b = {0.2, -0.1}; x = gaussian_matrix(1, 50, 32)."""
    import oracle
    from paper_2601_15473_b200 import derive_seed
    from paper_2601_15473_b200.conv import ConvShape, SkConv2d
    port = oracle.Oracle("port")
    shape = ConvShape(2, 2, 3, 3, 1, 0)
    w64, _ = port.dense_init(18, 2, 31)                 # [c_out][c_in*kh*kw]
    b64 = np.array([0.2, -0.1])
    x64 = port.gaussian_matrix(1, 2 * 5 * 5, 32).reshape(1, 2, 5, 5)
    cols = np.stack([x64[0, :, i:i + 3, j:j + 3].reshape(-1) for i in range(3) for j in range(3)])  # [9][18]
    expect = (cols @ w64.T + b64).T.reshape(1, 2, 3, 3)
    W, b, x = _tdev(w64, torch.float32), _tdev(b64, torch.float32), _tdev(x64, torch.float32)
    ys = []
    for s in range(600):
        inner = skl.SkLinear.from_dense(W, b, 1, 4, seed=derive_seed(888, s), dtype=skl.F32_TF32)
        ys.append(SkConv2d(shape, 1, 4, dtype=skl.F32_TF32, inner=inner).forward(x).double())
    ys = torch.stack(ys)
    mean, se = ys.mean(0), ys.std(0, unbiased=True) / 600 ** 0.5
    e = torch.from_numpy(expect).cuda()
    slack = 2e-3 * e.abs() + 1e-4
    assert bool(((mean - e).abs() <= 3 * se + slack).all()), ((mean - e).abs() / se).max()


@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
def test_conv_zero_input_unmodified(skl, dtype_name):
    """test_nn_layers.cpp:263-281 at its own shape: c_in = 1, c_out = 2, 3x3
    kernel, sk_conv2d_fresh(shape, 1, 4, 59), bias {0.7, -0.3}: a zero 5x5 image
    gives 3x3 maps equal to each channel's bias."""
    from paper_2601_15473_b200.conv import ConvShape, SkConv2d
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    conv = SkConv2d(ConvShape(1, 2, 3, 3, 1, 0), 1, 4, seed=59, dtype=dtype)
    bias = torch.tensor([0.7, -0.3], device="cuda").to(td)
    conv.inner.bias.copy_(bias)
    y = conv.forward(torch.zeros(1, 1, 5, 5, device="cuda", dtype=td))
    torch.cuda.synchronize()
    assert y.shape == (1, 2, 3, 3)
    assert torch.equal(y, bias.view(1, 2, 1, 1).expand(1, 2, 3, 3))


def test_ragged_conv_matches_reference(skl, ref):
    """SkConv2d with 2 input channels (d_in = 18) and 3 output channels against
    the reference's own SkConv2d (oracle/_ref), forward and backward, TF32."""
    import oracle
    from paper_2601_15473_b200.conv import ConvShape, SkConv2d
    from tests._util import check_close
    geo = (2, 3, 3, 3, 1, 1)
    conv = SkConv2d(ConvShape(*geo), 2, 3, seed=77, dtype=skl.F32_TF32)
    conv.inner.bias.copy_(torch.tensor([0.3, -0.2, 0.1], device="cuda"))
    x64 = ref.gaussian_matrix(1, 2 * 2 * 6 * 6, 61).reshape(2, 2, 6, 6)
    X = _tdev(x64, torch.float32)
    keep = {}
    y = conv.forward(X, keep=keep)
    g64 = ref.gaussian_matrix(1, y.numel(), 62).reshape(tuple(y.shape))
    G = _tdev(g64, torch.float32)
    gr = conv.backward(X, G, keep=keep)
    torch.cuda.synchronize()
    P = _layer_f64(skl, conv.inner)
    xb = _np(X)
    check_close("conv y", _np(y), oracle.skconv_forward(ref, geo, P, _np(conv.inner.bias), xb), "tf32")
    gx, gu1, gu2, gb = oracle.skconv_backward(ref, geo, P, xb, _np(G))
    _, rgu1, rgu2, rgb = oracle.grads_to_abi(np.zeros((P.d_in, 1)), gu1, gu2, gb)
    check_close("conv grad_x", _np(gr.grad_x), gx, "tf32")
    check_close("conv dU1s", _np(gr.grad_u1), rgu1, "tf32")
    check_close("conv dU2s", _np(gr.grad_u2), rgu2, "tf32")
    check_close("conv db", _np(gr.grad_b), rgb, "tf32")


# --------------------------------------------------------------------------- c1 end to end
def test_c1_end_to_end_against_unrounded_reference(skl, port):
    """BASELINE config 1 (the reference CPU correctness case) end to end: device
    sk_linear_fresh(1024, 1024, 1, 64, 42) in TF32 on x = gaussian_matrix(1024,
    64, 7) against the reference's f64 output on the UNROUNDED seeded values
    (y(0,0) = -0x1.d635314abae0ep-1), gate rel_fro / max_abs 2e-3."""
    from tests._util import check_close
    P = port.sk_linear_fresh(1024, 1024, 1, 64, 42)
    x = port.gaussian_matrix(1024, 64, 7)
    y_ref = port.forward(P, np.zeros(1024), x)
    assert y_ref[0, 0] == float.fromhex("-0x1.d635314abae0ep-1")
    layer = skl.SkLinear(1024, 1024, 1, 64, seed=42, dtype=skl.F32_TF32)
    y = layer.forward(_tdev(x.T, torch.float32))
    torch.cuda.synchronize()
    rf, ma = check_close("c1 y (unrounded reference)", _np(y), y_ref.T, "tf32")
    assert rf <= 2e-3 and ma <= 2e-3


# --------------------------------------------------------------------------- DenseLinear
DENSE = [(768, 3072, 300), (256, 128, 1000), (6, 8, 2), (50, 37, 129)]


@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
@pytest.mark.parametrize("d_in,d_out,T", DENSE)
def test_dense_linear_matches_oracle(skl, port, dtype_name, d_in, d_out, T):
    """DenseLinear::forward / backward (nn_layers.cpp:32-49) on the device vs the
    oracle (bit-exact with the reference's DenseLinear, tests/test_oracle.py),
    including dense_linear_init from the seed."""
    from tests._util import check_close
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    lyr = skl.DenseLinear(d_in, d_out, seed=31, dtype=dtype)
    w_ref, _ = port.dense_init(d_in, d_out, 31)
    tol = 2 ** -8 if dtype_name == "bf16" else 2 ** -23
    assert np.allclose(_np(lyr.W), w_ref, rtol=tol, atol=0)
    b = port.gaussian_matrix(1, d_out, 9)[0]
    lyr.bias.copy_(_tdev(b, td))
    x = port.gaussian_matrix(d_in, T, 3)
    g = port.gaussian_matrix(d_out, T, 4)
    X, G = _tdev(x.T, td), _tdev(g.T, td)
    y = lyr.forward(X)
    gr = lyr.backward(X, G)
    torch.cuda.synchronize()
    w64, b64, x64, g64 = _np(lyr.W), _np(lyr.bias), _np(X).T.copy(), _np(G).T.copy()
    check_close("dense y", _np(y), port.dense_forward(w64, b64, x64).T, dtype_name)
    gx, gw, gb = port.dense_backward(w64, x64, g64)
    check_close("dense grad_x", _np(gr.grad_x), gx.T, dtype_name)
    check_close("dense grad_w", _np(gr.grad_w), gw, dtype_name)
    check_close("dense grad_b", _np(gr.grad_b), gb, dtype_name)


@pytest.mark.parametrize("dtype_name", ["bf16", "tf32"])
def test_mixed_chain_with_dense_layer(skl, port, dtype_name):
    """model_forward over SKLinear + ReLU + Linear + ReLU + SKLinear
    (nn_model.cpp:111-122) and its training backward vs the oracle layer by layer."""
    import oracle
    from paper_2601_15473_b200.model import Relu, SkChain
    from tests._util import check_close
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    td = skl.torch_dtype(dtype)
    a = skl.SkLinear(64, 96, 2, 16, seed=1, dtype=dtype)
    dn = skl.DenseLinear(96, 50, seed=2, dtype=dtype)
    dn.bias.copy_(_tdev(port.gaussian_matrix(1, 50, 8)[0], td))
    c = skl.SkLinear(50, 40, 1, 8, seed=3, dtype=dtype)
    chain = SkChain([a, Relu(), dn, Relu(), c])
    T = 77
    X = _tdev(port.gaussian_matrix(64, T, 5).T, td)
    G = _tdev(port.gaussian_matrix(40, T, 6).T, td)
    y = chain.forward(X)
    cg, _ = chain.backward(G)
    torch.cuda.synchronize()
    Pa, Pc = _layer_f64(skl, a), _layer_f64(skl, c)
    w64, b64 = _np(dn.W), _np(dn.bias)
    a1 = _np(chain.steps[1].x).T.copy()   # device ReLU outputs, as the oracle inputs
    a2 = _np(chain.steps[2].x).T.copy()
    check_close("relu1", a1, np.maximum(port.forward(Pa, np.zeros(96), _np(X).T.copy()), 0), dtype_name)
    check_close("relu2", a2, np.maximum(port.dense_forward(w64, b64, a1), 0), dtype_name)
    check_close("y", _np(y), port.forward(Pc, np.zeros(40), a2).T, dtype_name)
    g64 = _np(G).T.copy()
    gx3, gu1, gu2, gb = port.backward(Pc, a2, g64)
    gz2 = gx3 * (a2 > 0)
    gxd, gw, gbd = port.dense_backward(w64, a1, gz2)
    check_close("dense dW", _np(cg.layers[1].dW), gw, dtype_name)
    check_close("dense db", _np(cg.layers[1].db), gbd, dtype_name)
    gz1 = gxd * (a1 > 0)
    rgx, rgu1, rgu2, rgb = oracle.grads_to_abi(*port.backward(Pa, _np(X).T.copy(), gz1))
    check_close("layer0 dU1s", _np(cg.layers[0].dU1s), rgu1, dtype_name)
    check_close("layer0 dU2s", _np(cg.layers[0].dU2s), rgu2, dtype_name)
    check_close("grad_x", _np(cg.grad_x), rgx, dtype_name)


# --------------------------------------------------------------------------- seeded generation at scale
LAYER_SHAPES = [
    (4096, 4096, 3, 256),   # c3 (6.29 M sketch entries)
    (4096, 4096, 4, 64),    # c4 L4 k64
    (4096, 4096, 1, 16),    # c4 L1 k16
    (768, 768, 1, 128),     # c5 projection
    (768, 3072, 2, 128),    # c5 FFN1 / c2
    (3072, 768, 2, 128),    # c5 FFN2
]


@pytest.mark.parametrize("dtype_name", ["bf16", "f32"])
@pytest.mark.parametrize("d_in,d_out,L,k", LAYER_SHAPES)
def test_generated_layer_rounds_equal_at_config_shapes(skl, port, dtype_name, d_in, d_out, L, k):
    """sk_linear_fresh(seed 42) on the device -- Gaussian sketches and U, written
    into the ABI stacks -- equals the reference stream rounded to the element type
    on EVERY entry, at the c3 / c4 / c5 layer shapes (CUDA's f64
    log/sin/cos are within 4 ulp of glibc, so only the rounded values can be
    exact; this checks they are, everywhere)."""
    import oracle
    from tests._util import bf16_round
    dtype = skl.BF16 if dtype_name == "bf16" else skl.F32_TF32
    lyr = skl.SkLinear(d_in, d_out, L, k, seed=42, dtype=dtype)
    torch.cuda.synchronize()
    abi = oracle.to_abi(port.sk_linear_fresh(d_in, d_out, L, k, 42))
    rnd = bf16_round if dtype_name == "bf16" else (lambda a: a.astype(np.float32).astype(np.float64))
    for name in ("S1s", "S2s", "U1s", "U2s"):
        dev = _np(getattr(lyr, name))
        ref = rnd(abi[name])
        bad = int(np.count_nonzero(dev != ref))
        assert bad == 0, f"{name}: {bad} of {ref.size} entries differ after rounding"


def test_c2_full_size_against_reference(skl, ref):
    """BASELINE config 2 at its FULL 32768 tokens against the reference itself
    (oracle/_ref, multithreaded f64, ~10-30 s): forward and every gradient of the
    bf16 device path on the same rounded inputs, at the bf16 gates."""
    import oracle
    from tests._util import check_close
    d_in, d_out, L, k, T = 768, 3072, 2, 128, 32768
    td = torch.bfloat16
    layer = skl.SkLinear(d_in, d_out, L, k, seed=42, dtype=skl.BF16)
    x, g, b = oracle.inputs(d_in, d_out, T, 42, ref)
    X, G = _tdev(x.T, td), _tdev(g.T, td)
    layer.bias.copy_(_tdev(b, td))
    saved = torch.empty(L * k, T, dtype=td, device="cuda")
    y = layer.forward(X, saved=saved)
    gr = layer.backward(X, G, saved=saved)
    torch.cuda.synchronize()
    P = _layer_f64(skl, layer)
    x64, g64, b64 = _np(X).T.copy(), _np(G).T.copy(), _np(layer.bias)
    check_close("c2 full y", _np(y), ref.forward(P, b64, x64).T, "bf16", regress=True)
    rgx, rgu1, rgu2, rgb = oracle.grads_to_abi(*ref.backward(P, x64, g64))
    check_close("c2 full grad_x", _np(gr.grad_x), rgx, "bf16", regress=True)
    check_close("c2 full dU1s", _np(gr.grad_u1), rgu1, "bf16", regress=True)
    check_close("c2 full dU2s", _np(gr.grad_u2), rgu2, "bf16", regress=True)
    check_close("c2 full db", _np(gr.grad_b), rgb, "bf16", regress=True)
