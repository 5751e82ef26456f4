"""CPU tests of the oracle (the parity checker): the C restatement against the
reference library compiled from /root/reference sources, against the
reference's own golden vectors (test_sketch.cpp:25-33), the known-answer values
in tests/golden/ (generated from the reference itself), and ports of the
reference's SKLinear unit tests (test_nn_layers.cpp, oracles.hpp)."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import oracle
from tests._util import bf16_round, tf32_round

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def fx(h):
    return np.array([float.fromhex(v) for v in h])


# ---------------------------------------------------------------- golden vectors
@pytest.mark.parametrize("kind", ["port", "reference"])
def test_splitmix64_golden_u64(kind):
    if not oracle.available(kind):
        pytest.skip(kind)
    o = oracle.Oracle(kind)
    # test_sketch.cpp:25-33
    s0 = o.splitmix64_stream(0, 2)
    assert int(s0[0]) == 0xE220A8397B1DCDAF and int(s0[1]) == 0x6E789E6AA1B965F4
    assert int(o.splitmix64_stream(42, 1)[0]) == 0xBDD732262FEB6E95


def test_port_matches_golden_file(port, golden):
    for seed, vals in golden["splitmix64"].items():
        assert [f"{int(v):016x}" for v in port.splitmix64_stream(int(seed), 8)] == vals
    for key, val in golden["derive_seed"].items():
        m, i = (int(t) for t in key.split(","))
        assert f"{port.derive_seed(m, i):016x}" == val
    for seed, vals in golden["gaussian_stream"].items():
        assert np.array_equal(port.gaussian_stream(int(seed), 9), fx(vals))
    for sk in golden["sketches"]:
        m = port.realize_sketch(sk["dist"], sk["k"], sk["d"], sk["seed"]).ravel()
        assert np.array_equal(m[:24], fx(sk["head"])) and np.array_equal(m[-8:], fx(sk["tail"]))
        assert float(m.sum()).hex() == sk["sum"]


def test_port_layer_matches_golden(port, golden):
    g = golden["layer_small"]
    p = port.sk_linear_fresh(g["d_in"], g["d_out"], g["L"], g["k"], g["seed"])
    for name in ("s1", "u1", "s2", "u2"):
        assert np.array_equal(getattr(p, name).ravel(), fx(g[name])), name
    x = fx(g["x"]).reshape(g["d_in"], g["T"])
    gg = fx(g["g"]).reshape(g["d_out"], g["T"])
    b = fx(g["b"])
    assert np.array_equal(port.forward(p, b, x).ravel(), fx(g["y"]))
    gx, gu1, gu2, gb = port.backward(p, x, gg)
    for name, v in (("grad_x", gx), ("grad_u1", gu1), ("grad_u2", gu2), ("grad_b", gb)):
        assert np.array_equal(v.ravel(), fx(g[name])), name


def test_port_kat_c1(port, golden):
    """SURVEY.md Appendix A values (sk_linear_fresh(1024,1024,1,64,42))."""
    k = golden["kat_c1"]
    p = port.sk_linear_fresh(1024, 1024, 1, 64, 42)
    assert np.array_equal(p.s1[0, 0, :4], fx(k["s1_row0"]))
    assert np.array_equal(p.s2[0, 0, :4], fx(k["s2_row0"]))
    assert np.array_equal(p.u1[0, 0, :2], fx(k["u1_00_01"]))
    assert p.u2[0, -1, -1] == float.fromhex(k["u2_last"])
    x = port.gaussian_matrix(1024, 64, 7)
    g = port.gaussian_matrix(1024, 64, 9)
    y = port.forward(p, np.zeros(1024), x)
    assert y[0, 0] == float.fromhex(k["y_0_0"]) and y[1023, 63] == float.fromhex(k["y_1023_63"])
    gx, gu1, gu2, gb = port.backward(p, x, g)
    assert gx[0, 0] == float.fromhex(k["grad_x_0_0"])
    assert gu1[0, 0, 0] == float.fromhex(k["grad_u1_0_0_0"])
    assert gu2[0, 0, 0] == float.fromhex(k["grad_u2_0_0_0"])
    assert gb[0] == float.fromhex(k["grad_b_0"])


# ---------------------------------------------------------------- port == reference (bit-exact)
@pytest.mark.parametrize("d_in,d_out,L,k,T,dist", [(6, 8, 2, 3, 2, 0), (37, 53, 3, 5, 11, 1), (64, 48, 1, 16, 9, 0),
                                                   (5, 3, 2, 2, 4, 1)])
def test_port_bitexact_vs_reference(port, ref, d_in, d_out, L, k, T, dist):
    pp = port.sk_linear_fresh(d_in, d_out, L, k, 1234, dist)
    pr = ref.sk_linear_fresh(d_in, d_out, L, k, 1234, dist)
    for name in ("s1", "u1", "s2", "u2"):
        assert np.array_equal(getattr(pp, name), getattr(pr, name)), name
    x, g, b = oracle.inputs(d_in, d_out, T, 99, port)
    assert np.array_equal(port.forward(pp, b, x), ref.forward(pr, b, x))
    for a, c in zip(port.backward(pp, x, g), ref.backward(pr, x, g)):
        assert np.array_equal(a, c)


def test_zero_skip_and_sign_of_zero(port, ref):
    """gemm_rows skips zero A entries (linalg.cpp:24): the port must too."""
    p = port.sk_linear_fresh(4, 3, 1, 2, 5)
    x = np.zeros((4, 3))
    x[1, 2] = -0.0
    b = np.array([-0.0, 0.0, 1.5])
    assert np.array_equal(port.forward(p, b, x).view(np.int64), ref.forward(p, b, x).view(np.int64))


# ---------------------------------------------------------------- reference unit tests, ported
def test_identity_sketches_collapse_to_average_dense(port):
    """test_nn_layers.cpp:69-90: S1 = S2 = I, l=1, k=d -> y = ((U1+U2)/2) x + b."""
    d = 4
    u1 = port.gaussian_matrix(d, d, 5)
    u2 = port.gaussian_matrix(d, d, 6)
    p = oracle.Params(d, d, 1, d, np.eye(d)[None], u1[None], np.eye(d)[None], u2[None])
    x = port.gaussian_matrix(d, 3, 7)
    b = np.array([0.1, 0.2, 0.3, 0.4])
    y = port.forward(p, b, x)
    expect = 0.5 * (u1 + u2) @ x + b[:, None]
    assert np.max(np.abs(y - expect)) < 1e-14


def test_zero_input_gives_bias(port):
    """test_nn_layers.cpp:92-97."""
    p = port.sk_linear_fresh(5, 3, 2, 2, 11)
    b = np.array([0.5, -1.0, 2.0])
    assert np.allclose(port.forward(p, b, np.zeros((5, 4))), b[:, None])


def test_backward_zero_upstream_and_batch_additivity(port):
    """test_nn_layers.cpp:113-140."""
    p = port.sk_linear_fresh(6, 8, 2, 3, 23)
    x = port.gaussian_matrix(6, 2, 29)
    gx, gu1, gu2, gb = port.backward(p, x, np.zeros((8, 2)))
    assert not gx.any() and not gu1.any() and not gu2.any() and not gb.any()
    go = port.gaussian_matrix(8, 2, 31)
    both = port.backward(p, x, go)
    parts = [port.backward(p, x[:, j:j + 1].copy(), go[:, j:j + 1].copy()) for j in range(2)]
    for i in (1, 2):
        assert np.max(np.abs(both[i] - (parts[0][i] + parts[1][i]))) < 1e-12
    assert np.allclose(both[3], parts[0][3] + parts[1][3])


def test_gradcheck_central_differences(port):
    """oracles.hpp:105-132 GradCheck (h=1e-5, rel 1e-4) on the 8x6, l=2, k=3 case (test_nn_layers.cpp:158-176)."""
    p = port.sk_linear_fresh(6, 8, 2, 3, 41)
    x = port.gaussian_matrix(6, 2, 43)
    b = np.zeros(8)

    def loss():
        y = port.forward(p, b, x)
        return 0.5 * float(np.sum(y * y))

    gx, gu1, gu2, gb = port.backward(p, x, port.forward(p, b, x))
    h, worst, scale = 1e-5, 0.0, max(np.abs(gx).max(), np.abs(gu1).max(), np.abs(gu2).max(), np.abs(gb).max())
    for arr, grad in ((p.u1, gu1), (p.u2, gu2), (b, gb), (x, gx)):
        flat, gflat = arr.reshape(-1), grad.reshape(-1)
        for i in range(flat.size):
            s = flat[i]
            flat[i] = s + h
            up = loss()
            flat[i] = s - h
            dn = loss()
            flat[i] = s
            num = (up - dn) / (2 * h)
            err = abs(gflat[i] - num)
            rel = 0.0 if err <= 1e-8 * max(scale, 1.0) else err / max(abs(gflat[i]), abs(num), 1e-12)
            worst = max(worst, rel)
    assert worst <= 1e-4


def test_param_count_and_skip_rule(port):
    """test_nn_layers.cpp:178-192 closed forms."""
    assert port.lib.orc_sk_stored_coeffs(1, 16, 8192, 8192) == 524288
    assert port.lib.orc_sk_stored_coeffs(2, 64, 256, 256) == 131072
    assert port.lib.orc_exceeds_dense(2, 64, 256, 256) == 1
    assert port.lib.orc_exceeds_dense(1, 64, 256, 256) == 0  # equality admitted
    # BERT FFN config c2 is admissible; 768x768 with L=2,k=128 is not
    assert port.lib.orc_exceeds_dense(2, 128, 768, 3072) == 0
    assert port.lib.orc_exceeds_dense(2, 128, 768, 768) == 1


def test_error_contract(port, ref):
    """shape_error / parameter_error (errors.hpp:10-19, nn_layers.cpp:62,116)."""
    with pytest.raises(oracle.ParameterError):
        port.sk_linear_fresh(4, 4, 0, 2, 1)
    with pytest.raises(oracle.ParameterError):
        ref.sk_linear_fresh(4, 4, 1, 0, 1)
    assert ref.lib.ref_sk_forward_checked(4, 3, 1, 2, 5, 2) == 1  # shape_error
    assert ref.lib.ref_sk_forward_checked(4, 3, 1, 2, 4, 2) == 0
    with pytest.raises(oracle.ShapeError):
        port.realize_sketch(0, 0, 5, 1)


def test_rademacher_support(port):
    """test_sketch.cpp:35-42."""
    s = port.realize_sketch(1, 2, 3, 123)
    v = 1.0 / np.sqrt(2.0)
    assert set(np.unique(s)) <= {v, -v}


def test_gaussian_sketch_rounding_fragility(port):
    """H4: Gaussian entries are far from bf16/tf32 rounding ties, so a 1-2 ulp
    f64 perturbation (device libm vs glibc) cannot change the rounded value.
    Counted on the c2 sketches (L=2, k=128)."""
    p = port.sk_linear_fresh(768, 3072, 2, 128, 42)
    vals = np.concatenate([p.s1.ravel(), p.s2.ravel()])
    flips = 0
    for d in (-2, -1, 1, 2):
        pert = (vals.view(np.int64) + d).view(np.float64)
        flips += int(np.sum(bf16_round(pert) != bf16_round(vals)))
        flips += int(np.sum(tf32_round(pert) != tf32_round(vals)))
    assert flips == 0


def test_dense_port_is_bit_exact_with_reference():
    """DenseLinear init / forward / backward of the port (skl_oracle.c) equal the
    reference's own DenseLinear (nn_layers.cpp:32-59, oracle/_ref) bit for bit."""
    import oracle
    if not oracle.available("reference"):
        pytest.skip("oracle/_ref not built")
    po, ro = oracle.Oracle("port"), oracle.Oracle("reference")
    for d_in, d_out, T, seed in ((6, 8, 2, 31), (37, 13, 11, 5), (96, 50, 20, 202)):
        w, b = po.dense_init(d_in, d_out, seed)
        w2, b2 = ro.dense_init(d_in, d_out, seed)
        assert np.array_equal(w, w2) and np.array_equal(b, b2)
        b = ro.gaussian_matrix(1, d_out, 9)[0]
        x = ro.gaussian_matrix(d_in, T, 3)
        g = ro.gaussian_matrix(d_out, T, 4)
        assert np.array_equal(po.dense_forward(w, b, x), ro.dense_forward(w, b, x))
        for a, c in zip(po.dense_backward(w, x, g), ro.dense_backward(w, x, g)):
            assert np.array_equal(a, c)
