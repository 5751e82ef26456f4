// test_sklinear.cpp -- C++ host parity test of the B200 SKLinear path.
//
// Drives libskl.so through the C++ host mirror include/skl.hpp (no PyTorch)
// and checks it against the oracle (oracle/liboracle.so, the f64 C
// restatement of the reference; TEST INFRASTRUCTURE, linked only here).
// Structured like the reference's acceptance.cpp: one PASS/FAIL line per
// criterion, exit code = number of failures.  Needs an sm_100 GPU.
//
// Ported reference cases (/root/reference/proj/tests):
//   identity sketches, l=1, k=d -> y = ((U1+U2)/2) x + b   test_nn_layers.cpp:69-90
//   zero input -> bias                                       test_nn_layers.cpp:92-97
//   zero upstream -> zero gradients; batch additivity        test_nn_layers.cpp:113-140
//   parameter / shape errors                                 nn_layers.cpp:62,79-80,116
//   params closed forms                                      test_nn_layers.cpp:178-192
//   sketch entries == realize_sketch (seed chain bit-exact)  sketch.cpp:34-49, rng.hpp:13-69
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include <dlfcn.h>

#include "skl.hpp"

extern "C" {
uint64_t orc_derive_seed(uint64_t master, uint64_t index);
int orc_realize_sketch(int dist, uint64_t k, uint64_t d, uint64_t seed, double* out);
void orc_gaussian_matrix(uint64_t rows, uint64_t cols, uint64_t seed, double* out);
int orc_sk_forward(uint64_t d_in, uint64_t d_out, uint64_t l, uint64_t k, uint64_t T, const double* s1,
                   const double* u1, const double* s2, const double* u2, const double* bias, const double* x,
                   double* y);
int orc_sk_backward(uint64_t d_in, uint64_t d_out, uint64_t l, uint64_t k, uint64_t T, const double* s1,
                    const double* u1, const double* s2, const double* u2, const double* x, const double* g,
                    double* gx, double* gu1, double* gu2, double* gb);
}

namespace {

int g_fail = 0;
void report(const char* name, bool ok, const std::string& detail = "") {
    std::printf("%s %s%s%s\n", ok ? "PASS" : "FAIL", name, detail.empty() ? "" : "  ", detail.c_str());
    if (!ok) ++g_fail;
}

using vec = std::vector<double>;

// ---- element conversion (host) -------------------------------------------
uint16_t f2bf(float f) {  // round to nearest even
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
float bf2f(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
std::vector<uint8_t> to_dev(const vec& a, skl_dtype t) {
    std::vector<uint8_t> out(a.size() * skl::elem_bytes(t));
    for (size_t i = 0; i < a.size(); ++i) {
        if (t == SKL_BF16) {
            const uint16_t b = f2bf((float)a[i]);
            std::memcpy(out.data() + 2 * i, &b, 2);
        } else {
            const float f = (float)a[i];
            std::memcpy(out.data() + 4 * i, &f, 4);
        }
    }
    return out;
}
vec from_dev(const void* p, size_t n, skl_dtype t) {
    vec out(n);
    for (size_t i = 0; i < n; ++i) {
        if (t == SKL_BF16) {
            uint16_t b;
            std::memcpy(&b, (const uint8_t*)p + 2 * i, 2);
            out[i] = bf2f(b);
        } else {
            float f;
            std::memcpy(&f, (const uint8_t*)p + 4 * i, 4);
            out[i] = f;
        }
    }
    return out;
}
vec download(const void* dptr, size_t n, skl_dtype t) {
    std::vector<uint8_t> h(n * skl::elem_bytes(t));
    skl::check_cuda(cudaMemcpy(h.data(), dptr, h.size(), cudaMemcpyDeviceToHost), "download");
    return from_dev(h.data(), n, t);
}
vec download_f32(const void* dptr, size_t n) { return download(dptr, n, SKL_F32_TF32); }

double rel_fro(const vec& a, const vec& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        num += (a[i] - b[i]) * (a[i] - b[i]);
        den += b[i] * b[i];
    }
    return std::sqrt(num) / (den > 0 ? std::sqrt(den) : 1.0);
}
double max_abs_rel(const vec& a, const vec& b) {
    double m = 0, r = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        m = std::fmax(m, std::fabs(a[i] - b[i]));
        r = std::fmax(r, std::fabs(b[i]));
    }
    return m / (r > 0 ? r : 1.0);
}
// Gates vs the f64 oracle (tests/_util.py GATES).
bool gate(const vec& a, const vec& b, skl_dtype t, std::string& detail) {
    const double rf = rel_fro(a, b), ma = max_abs_rel(a, b);
    const double g_rf = t == SKL_BF16 ? 1e-2 : 2e-3, g_ma = t == SKL_BF16 ? 2e-2 : 2e-3;
    char buf[160];
    std::snprintf(buf, sizeof buf, "rel_fro=%.3e max_abs/max|ref|=%.3e", rf, ma);
    detail = buf;
    return rf <= g_rf && ma <= g_ma;
}

// ABI stacks (row convention) <-> reference per-term matrices (column convention).
struct RefParams {
    vec s1, u1, s2, u2;  // [l][k][d_out], [l][k][d_in], [l][k][d_in], [l][d_out][k]
};
RefParams ref_from_layer(const skl::SkLinear& L) {
    const int64_t di = L.d_in(), dn = L.d_out(), l = L.num_terms(), k = L.low_rank();
    const skl_dtype t = L.dtype();
    const vec S1 = download(L.S1s(), l * di * k, t), S2 = download(L.S2s(), l * k * dn, t);
    const vec U1 = download(L.U1s(), l * k * dn, t), U2 = download(L.U2s(), l * di * k, t);
    RefParams p{vec(l * k * dn), vec(l * k * di), vec(l * k * di), vec(l * dn * k)};
    for (int64_t i = 0; i < l; ++i)
        for (int64_t j = 0; j < k; ++j) {
            for (int64_t o = 0; o < dn; ++o) {
                p.s1[(i * k + j) * dn + o] = S2[(i * k + j) * dn + o];  // s1 = S2s
                p.u2[(i * dn + o) * k + j] = U1[(i * k + j) * dn + o];  // u2 = U1sᵀ
            }
            for (int64_t c = 0; c < di; ++c) {
                p.s2[(i * k + j) * di + c] = S1[(i * di + c) * k + j];  // s2 = S1sᵀ
                p.u1[(i * k + j) * di + c] = U2[(i * di + c) * k + j];  // u1 = U2sᵀ
            }
        }
    return p;
}

struct Case {
    int64_t d_in, d_out, l, k, T;
    skl_dtype dtype;
};

// Seeded inputs exactly as SURVEY §8d / oracle.inputs: x = gaussian_matrix(d_in, T,
// derive_seed(seed,7)) (column convention), g from derive_seed(seed,9), bias
// from derive_seed(seed,11); rounded to the variant's element type.
struct Inputs {
    vec x_ref, g_ref, b;                 // rounded, reference layout
    std::vector<uint8_t> x_abi, g_abi, b_abi;  // row convention, device element type
};
Inputs make_inputs(const Case& c, uint64_t seed) {
    Inputs in;
    vec x(c.d_in * c.T), g(c.d_out * c.T), b(c.d_out);
    orc_gaussian_matrix(c.d_in, c.T, orc_derive_seed(seed, 7), x.data());
    orc_gaussian_matrix(c.d_out, c.T, orc_derive_seed(seed, 9), g.data());
    orc_gaussian_matrix(1, c.d_out, orc_derive_seed(seed, 11), b.data());
    vec xa(c.T * c.d_in), ga(c.T * c.d_out);
    for (int64_t r = 0; r < c.d_in; ++r)
        for (int64_t t = 0; t < c.T; ++t) xa[t * c.d_in + r] = x[r * c.T + t];
    for (int64_t r = 0; r < c.d_out; ++r)
        for (int64_t t = 0; t < c.T; ++t) ga[t * c.d_out + r] = g[r * c.T + t];
    in.x_abi = to_dev(xa, c.dtype);
    in.g_abi = to_dev(ga, c.dtype);
    in.b_abi = to_dev(b, c.dtype);
    const vec xr = from_dev(in.x_abi.data(), xa.size(), c.dtype), gr = from_dev(in.g_abi.data(), ga.size(), c.dtype);
    in.x_ref.resize(x.size());
    in.g_ref.resize(g.size());
    for (int64_t r = 0; r < c.d_in; ++r)
        for (int64_t t = 0; t < c.T; ++t) in.x_ref[r * c.T + t] = xr[t * c.d_in + r];
    for (int64_t r = 0; r < c.d_out; ++r)
        for (int64_t t = 0; t < c.T; ++t) in.g_ref[r * c.T + t] = gr[t * c.d_out + r];
    in.b = from_dev(in.b_abi.data(), b.size(), c.dtype);
    return in;
}

// Parity of a fresh layer: forward (saving the projection) + backward vs the oracle.
void parity_case(const char* name, const Case& c, skl_dist dist = SKL_DIST_GAUSSIAN) {
    const uint64_t seed = 42;
    skl::SkLinear fresh = skl::SkLinear::fresh(c.d_in, c.d_out, c.l, c.k, seed, dist, c.dtype);
    const Inputs in = make_inputs(c, seed);
    std::vector<uint8_t> s1, s2, u1, u2;
    const size_t e = skl::elem_bytes(c.dtype);
    auto grab = [&](void* p, size_t n) {
        std::vector<uint8_t> h(n * e);
        skl::check_cuda(cudaMemcpy(h.data(), p, h.size(), cudaMemcpyDeviceToHost), "grab");
        return h;
    };
    s1 = grab(fresh.S1s(), c.l * c.d_in * c.k);
    s2 = grab(fresh.S2s(), c.l * c.k * c.d_out);
    u1 = grab(fresh.U1s(), c.l * c.k * c.d_out);
    u2 = grab(fresh.U2s(), c.l * c.d_in * c.k);
    // same parameters + a nonzero bias (a fresh bias is zero and would hide bias bugs)
    skl::SkLinear L = skl::SkLinear::with_params(c.d_in, c.d_out, c.l, c.k, c.dtype, s1.data(), s2.data(), u1.data(),
                                                 u2.data(), in.b_abi.data());
    const RefParams P = ref_from_layer(L);

    skl::DeviceBuffer X(in.x_abi.size()), G(in.g_abi.size()), Y(c.T * c.d_out * e), S(L.saved_bytes(c.T));
    X.upload(in.x_abi.data(), in.x_abi.size());
    G.upload(in.g_abi.data(), in.g_abi.size());
    L.forward(X.get(), c.T, Y.get(), S.get());
    skl::SkLinear::Grads gr = L.backward(X.get(), G.get(), c.T, S.get());
    skl::check_cuda(cudaDeviceSynchronize(), "sync");

    vec y_ref(c.d_out * c.T), gx(c.d_in * c.T), gu1(c.l * c.k * c.d_in), gu2(c.l * c.d_out * c.k), gb(c.d_out);
    orc_sk_forward(c.d_in, c.d_out, c.l, c.k, c.T, P.s1.data(), P.u1.data(), P.s2.data(), P.u2.data(), in.b.data(),
                   in.x_ref.data(), y_ref.data());
    orc_sk_backward(c.d_in, c.d_out, c.l, c.k, c.T, P.s1.data(), P.u1.data(), P.s2.data(), P.u2.data(),
                    in.x_ref.data(), in.g_ref.data(), gx.data(), gu1.data(), gu2.data(), gb.data());
    // device results -> reference layout
    const vec y = download(Y.get(), c.T * c.d_out, c.dtype), dx = download(gr.grad_x.get(), c.T * c.d_in, c.dtype);
    const vec du1 = download_f32(gr.grad_u1.get(), c.l * c.k * c.d_out);
    const vec du2 = download_f32(gr.grad_u2.get(), c.l * c.d_in * c.k);
    const vec db = download_f32(gr.grad_b.get(), c.d_out);
    vec yr(y.size()), dxr(dx.size()), gu1d(gu1.size()), gu2d(gu2.size());
    for (int64_t t = 0; t < c.T; ++t) {
        for (int64_t o = 0; o < c.d_out; ++o) yr[o * c.T + t] = y[t * c.d_out + o];
        for (int64_t r = 0; r < c.d_in; ++r) dxr[r * c.T + t] = dx[t * c.d_in + r];
    }
    for (int64_t i = 0; i < c.l; ++i)
        for (int64_t j = 0; j < c.k; ++j) {
            for (int64_t r = 0; r < c.d_in; ++r) gu1d[(i * c.k + j) * c.d_in + r] = du2[(i * c.d_in + r) * c.k + j];
            for (int64_t o = 0; o < c.d_out; ++o) gu2d[(i * c.d_out + o) * c.k + j] = du1[(i * c.k + j) * c.d_out + o];
        }
    std::string d;
    std::string n(name);
    report((n + " forward").c_str(), gate(yr, y_ref, c.dtype, d), d);
    report((n + " grad_x").c_str(), gate(dxr, gx, c.dtype, d), d);
    report((n + " grad_u1").c_str(), gate(gu1d, gu1, c.dtype, d), d);
    report((n + " grad_u2").c_str(), gate(gu2d, gu2, c.dtype, d), d);
    report((n + " grad_b").c_str(), gate(db, gb, c.dtype, d), d);
}

void test_sketch_bit_exact() {
    // S2s[i] == realize_sketch(dist, k, d_out, derive_seed(seed, 2i)) and
    // S1s[i] == realize_sketch(dist, k, d_in, derive_seed(seed, 2i+1))ᵀ, fp32-rounded.
    for (int dist = 0; dist < 2; ++dist) {
        const int64_t d_in = 96, d_out = 160, l = 2, k = 24;
        skl::SkLinear L = skl::SkLinear::fresh(d_in, d_out, l, k, 42, (skl_dist)dist, SKL_F32_TF32);
        const vec S1 = download_f32(L.S1s(), l * d_in * k), S2 = download_f32(L.S2s(), l * k * d_out);
        bool ok = true;
        for (int64_t i = 0; i < l && ok; ++i) {
            vec a(k * d_out), b(k * d_in);
            orc_realize_sketch(dist, k, d_out, orc_derive_seed(42, 2 * i), a.data());
            orc_realize_sketch(dist, k, d_in, orc_derive_seed(42, 2 * i + 1), b.data());
            for (int64_t j = 0; j < k; ++j) {
                for (int64_t o = 0; o < d_out; ++o) ok &= (float)a[j * d_out + o] == (float)S2[(i * k + j) * d_out + o];
                for (int64_t c = 0; c < d_in; ++c) ok &= (float)b[j * d_in + c] == (float)S1[(i * d_in + c) * k + j];
            }
        }
        report(dist == 0 ? "sketch entries bit-exact (Gaussian, f32)" : "sketch entries bit-exact (Rademacher)", ok);
    }
}

void test_identity_sketches() {
    // test_nn_layers.cpp:69-90: with_realized(I), l=1, k=d -> y = ((U1+U2)/2) x + b
    const int64_t d = 64, T = 40;
    const skl_dtype t = SKL_F32_TF32;
    vec I(d * d, 0.0), u1(d * d), u2(d * d), b(d), x(T * d);
    for (int64_t i = 0; i < d; ++i) I[i * d + i] = 1.0;
    orc_gaussian_matrix(d, d, 5, u1.data());
    orc_gaussian_matrix(d, d, 6, u2.data());
    orc_gaussian_matrix(1, d, 8, b.data());
    orc_gaussian_matrix(T, d, 9, x.data());
    const auto Ih = to_dev(I, t), U1h = to_dev(u1, t), U2h = to_dev(u2, t), bh = to_dev(b, t), xh = to_dev(x, t);
    skl::SkLinear L = skl::SkLinear::with_params(d, d, 1, d, t, Ih.data(), Ih.data(), U1h.data(), U2h.data(), bh.data());
    const std::vector<uint8_t> yh = L.forward_host(xh.data(), T);
    const vec y = from_dev(yh.data(), T * d, t), xr = from_dev(xh.data(), T * d, t);
    const vec u1r = from_dev(U1h.data(), d * d, t), u2r = from_dev(U2h.data(), d * d, t), br = from_dev(bh.data(), d, t);
    vec ref(T * d);
    for (int64_t s = 0; s < T; ++s)
        for (int64_t o = 0; o < d; ++o) {
            double acc = 0;
            for (int64_t c = 0; c < d; ++c) acc += xr[s * d + c] * 0.5 * (u1r[c * d + o] + u2r[c * d + o]);
            ref[s * d + o] = acc + br[o];
        }
    std::string det;
    report("identity sketches collapse to ((U1+U2)/2)x+b", gate(y, ref, t, det), det);
}

void test_zero_cases() {
    for (skl_dtype t : {SKL_F32_TF32, SKL_BF16}) {
        const int64_t d_in = 128, d_out = 192, l = 2, k = 64, T = 130;
        const size_t e = skl::elem_bytes(t);
        vec b(d_out);
        orc_gaussian_matrix(1, d_out, 3, b.data());
        const auto bh = to_dev(b, t);
        skl::SkLinear f = skl::SkLinear::fresh(d_in, d_out, l, k, 7, SKL_DIST_GAUSSIAN, t);
        // zero input -> y == bias exactly (test_nn_layers.cpp:92-97)
        skl::DeviceBuffer X(T * d_in * e), Y(T * d_out * e), G(T * d_out * e);
        X.zero();
        G.zero();
        skl::check_cuda(cudaMemcpy(f.bias(), bh.data(), bh.size(), cudaMemcpyHostToDevice), "bias");
        f.forward(X.get(), T, Y.get());
        skl::check_cuda(cudaDeviceSynchronize(), "sync");
        const vec y = download(Y.get(), T * d_out, t), br = from_dev(bh.data(), d_out, t);
        bool ok = true;
        for (int64_t s = 0; s < T; ++s)
            for (int64_t o = 0; o < d_out; ++o) ok &= y[s * d_out + o] == br[o];
        report(t == SKL_BF16 ? "zero input gives bias (bf16)" : "zero input gives bias (tf32)", ok);
        // zero upstream -> all gradients exactly zero (test_nn_layers.cpp:113-120)
        vec xv(T * d_in);
        orc_gaussian_matrix(T, d_in, 4, xv.data());
        const auto xh = to_dev(xv, t);
        X.upload(xh.data(), xh.size());
        skl::SkLinear::Grads g = f.backward(X.get(), G.get(), T);
        skl::check_cuda(cudaDeviceSynchronize(), "sync");
        ok = true;
        for (double v : download(g.grad_x.get(), T * d_in, t)) ok &= v == 0.0;
        for (double v : download_f32(g.grad_u1.get(), l * k * d_out)) ok &= v == 0.0;
        for (double v : download_f32(g.grad_u2.get(), l * d_in * k)) ok &= v == 0.0;
        for (double v : download_f32(g.grad_b.get(), d_out)) ok &= v == 0.0;
        report(t == SKL_BF16 ? "zero upstream gives zero grads (bf16)" : "zero upstream gives zero grads (tf32)", ok);
    }
}

void test_batch_additivity() {
    // test_nn_layers.cpp:122-140: grads over [x1;x2] == grads(x1) + grads(x2)
    const Case c{256, 384, 2, 64, 512, SKL_F32_TF32};
    skl::SkLinear L = skl::SkLinear::fresh(c.d_in, c.d_out, c.l, c.k, 11, SKL_DIST_GAUSSIAN, c.dtype);
    const Inputs in = make_inputs(c, 11);
    skl::DeviceBuffer X(in.x_abi.size()), G(in.g_abi.size());
    X.upload(in.x_abi.data(), in.x_abi.size());
    G.upload(in.g_abi.data(), in.g_abi.size());
    const int64_t h = 200;  // ragged split
    skl::SkLinear::Grads all = L.backward(X.get(), G.get(), c.T);
    skl::SkLinear::Grads a = L.backward(X.get(), G.get(), h);
    skl::SkLinear::Grads b = L.backward(X.as<float>() + h * c.d_in, G.as<float>() + h * c.d_out, c.T - h);
    skl::check_cuda(cudaDeviceSynchronize(), "sync");
    vec sum, ref;
    auto add = [&](const skl::DeviceBuffer& p, const skl::DeviceBuffer& q, const skl::DeviceBuffer& r, size_t n) {
        const vec x = download_f32(p.get(), n), y = download_f32(q.get(), n), z = download_f32(r.get(), n);
        for (size_t i = 0; i < n; ++i) {
            sum.push_back(y[i] + z[i]);
            ref.push_back(x[i]);
        }
    };
    add(all.grad_u1, a.grad_u1, b.grad_u1, c.l * c.k * c.d_out);
    add(all.grad_u2, a.grad_u2, b.grad_u2, c.l * c.d_in * c.k);
    add(all.grad_b, a.grad_b, b.grad_b, c.d_out);
    const double rf = rel_fro(sum, ref);
    char buf[64];
    std::snprintf(buf, sizeof buf, "rel_fro=%.3e", rf);
    report("backward batch additivity (split 200 + 312 tokens)", rf < 1e-5, buf);
}

void test_errors() {
    bool ok = false;
    try {
        skl::SkLinear::fresh(64, 64, 0, 8, 1);
    } catch (const skl::parameter_error&) {
        ok = true;
    }
    report("l < 1 throws parameter_error (nn_layers.cpp:116)", ok);
    ok = false;
    try {
        skl::SkLinear::fresh(64, 64, 1, 0, 1);
    } catch (const skl::parameter_error&) {
        ok = true;
    }
    report("k < 1 throws parameter_error", ok);
    ok = false;
    try {
        skl_shape s{0, 64, 1, 8, SKL_BF16};
        size_t f, b;
        skl::check(skl_workspace_size(&s, 16, &f, &b));
    } catch (const skl::shape_error&) {
        ok = true;
    }
    report("d_in < 1 throws shape_error", ok);
}

void test_params() {
    // test_nn_layers.cpp:178-192 closed forms
    skl_shape s{1024, 1024, 1, 64, SKL_BF16};
    skl_param_count pc;
    skl::check(skl_params(&s, &pc));
    bool ok = pc.learnable == 64ull * 2048 + 1024 && pc.total_stored == 2ull * 64 * 2048 + 1024 &&
              pc.dense_equivalent == 1024ull * 1024 + 1024;
    ok &= skl_exceeds_dense(1, 128, 4096, 4096) == 0 && skl_exceeds_dense(2, 1024, 4096, 4096) == 1;
    ok &= skl_exceeds_dense(2, 128, 768, 768) == 1 && skl_exceeds_dense(2, 128, 768, 3072) == 0;
    report("params / exceeds_dense closed forms", ok);
}

void test_from_dense() {
    // sk_linear_from_dense (nn_layers.cpp:149-160): u1_i = s1_i·W, u2_i = W·s2_iᵀ
    const int64_t d_in = 96, d_out = 160, l = 2, k = 16;
    const skl_dtype t = SKL_F32_TF32;
    vec W(d_out * d_in), b(d_out);
    orc_gaussian_matrix(d_out, d_in, 21, W.data());
    orc_gaussian_matrix(1, d_out, 22, b.data());
    for (double& v : W) v *= 0.05;
    const auto Wh = to_dev(W, t), bh = to_dev(b, t);
    skl::DeviceBuffer Wd(Wh.size()), bd(bh.size());
    Wd.upload(Wh.data(), Wh.size());
    bd.upload(bh.data(), bh.size());
    skl::SkLinear L = skl::SkLinear::from_dense(Wd.get(), bd.get(), d_in, d_out, l, k, 33, SKL_DIST_GAUSSIAN, t);
    const RefParams P = ref_from_layer(L);  // device sketches (bit-exact) and device U
    const vec Wr = from_dev(Wh.data(), W.size(), t);
    vec u1(l * k * d_in, 0.0), u2(l * d_out * k, 0.0), u1d, u2d;
    for (int64_t i = 0; i < l; ++i)
        for (int64_t j = 0; j < k; ++j) {
            for (int64_t c = 0; c < d_in; ++c) {
                double acc = 0;
                for (int64_t o = 0; o < d_out; ++o) acc += P.s1[(i * k + j) * d_out + o] * Wr[o * d_in + c];
                u1[(i * k + j) * d_in + c] = acc;
            }
            for (int64_t o = 0; o < d_out; ++o) {
                double acc = 0;
                for (int64_t c = 0; c < d_in; ++c) acc += Wr[o * d_in + c] * P.s2[(i * k + j) * d_in + c];
                u2[(i * d_out + o) * k + j] = acc;
            }
        }
    std::string d1, d2;
    const bool ok1 = gate(P.u1, u1, t, d1), ok2 = gate(P.u2, u2, t, d2);
    report("from_dense u1 = s1·W (tcgen05)", ok1, d1);
    report("from_dense u2 = W·s2ᵀ (tcgen05)", ok2, d2);
    const vec bias = download(L.bias(), d_out, t), br = from_dev(bh.data(), d_out, t);
    report("from_dense bias copied", bias == br);
}

void test_fused_relu_forward() {
    // SKL_FUSE_RELU_OUT == max(0, plain forward), bitwise
    const int64_t d_in = 128, d_out = 192, l = 2, k = 64, T = 200;
    skl::SkLinear L = skl::SkLinear::fresh(d_in, d_out, l, k, 5, SKL_DIST_GAUSSIAN, SKL_BF16);
    vec xv(T * d_in), bv(d_out);
    orc_gaussian_matrix(T, d_in, 6, xv.data());
    orc_gaussian_matrix(1, d_out, 7, bv.data());
    const auto xh = to_dev(xv, SKL_BF16), bh = to_dev(bv, SKL_BF16);
    skl::check_cuda(cudaMemcpy(L.bias(), bh.data(), bh.size(), cudaMemcpyHostToDevice), "bias");
    skl::DeviceBuffer X(xh.size()), Y(T * d_out * 2), R(T * d_out * 2);
    X.upload(xh.data(), xh.size());
    L.forward(X.get(), T, Y.get());
    L.forward(X.get(), T, R.get(), nullptr, nullptr, SKL_FUSE_RELU_OUT);
    skl::check_cuda(cudaDeviceSynchronize(), "sync");
    const vec y = download(Y.get(), T * d_out, SKL_BF16), r = download(R.get(), T * d_out, SKL_BF16);
    bool ok = true;
    for (size_t i = 0; i < y.size(); ++i) ok &= r[i] == (y[i] > 0 ? y[i] : 0.0);
    report("fused ReLU forward == max(0, forward) bitwise", ok);
    // 1-bit masks: bits == (relu(y) > 0), and the next layer's backward with the
    // bits equals its backward with the x-mask, bitwise (skl.h SKL_FUSE_RELU_BITS)
    if (!L.relu_bits_supported()) {
        std::printf("SKIP relu bits (shape not on the CTA-pair kernel)\n");
        return;
    }
    const int64_t W = skl_relu_bits_row_words(d_out);
    skl::DeviceBuffer Bits((size_t)(T * W) * 4), R2(T * d_out * 2);
    L.forward(X.get(), T, R2.get(), nullptr, nullptr, SKL_FUSE_RELU_OUT, Bits.as<uint32_t>());
    skl::check_cuda(cudaDeviceSynchronize(), "sync");
    std::vector<uint32_t> bits((size_t)(T * W));
    Bits.download(bits.data(), bits.size() * 4);
    const vec r2 = download(R2.get(), T * d_out, SKL_BF16);
    bool okb = r2 == r;
    for (int64_t t = 0; t < T; ++t)
        for (int64_t c = 0; c < d_out; ++c)
            okb &= (((bits[t * W + c / 32] >> (c % 32)) & 1u) != 0) == (r[t * d_out + c] > 0);
    report("relu bits from the forward == (relu(y) > 0)", okb);
    skl::SkLinear L2 = skl::SkLinear::fresh(d_out, 96, 1, 64, 8, SKL_DIST_GAUSSIAN, SKL_BF16);
    if (!L2.relu_bits_supported()) return;
    vec gv(T * 96);
    orc_gaussian_matrix(T, 96, 9, gv.data());
    const auto gh = to_dev(gv, SKL_BF16);
    skl::DeviceBuffer G(gh.size());
    G.upload(gh.data(), gh.size());
    std::vector<vec> out[2];
    for (int mode = 0; mode < 2; ++mode) {
        skl::DeviceBuffer GX(T * d_out * 2), D1(64 * 96 * 4), D2(d_out * 64 * 4), DB(96 * 4);
        L2.backward_into(R.get(), G.get(), T, nullptr, GX.get(), D1.as<float>(), D2.as<float>(), DB.as<float>(),
                         nullptr, SKL_BWD_ALL, SKL_FUSE_RELU_IN, mode ? Bits.as<uint32_t>() : nullptr);
        skl::check_cuda(cudaDeviceSynchronize(), "sync");
        out[mode] = {download(GX.get(), T * d_out, SKL_BF16), download_f32(D1.get(), 64 * 96),
                     download_f32(D2.get(), d_out * 64), download_f32(DB.get(), 96)};
    }
    report("next layer's backward: relu bits == x-mask, bitwise", out[0] == out[1]);
}

void test_nccl_allreduce_world1() {
    // skl_allreduce_grads over a real ncclComm_t (one rank): the C-ABI entry a
    // C++ data-parallel host calls on the gradient bucket.
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        std::printf("SKIP nccl (libnccl.so.2 not loadable)\n");
        return;
    }
    using init_all_fn = int (*)(void**, int, const int*);
    using destroy_fn = int (*)(void*);
    auto init_all = reinterpret_cast<init_all_fn>(dlsym(h, "ncclCommInitAll"));
    auto destroy = reinterpret_cast<destroy_fn>(dlsym(h, "ncclCommDestroy"));
    void* comm = nullptr;
    const int dev0 = 0;
    bool ok = init_all && destroy && init_all(&comm, 1, &dev0) == 0;
    const size_t n = 1000;
    std::vector<float> hv(n);
    for (size_t i = 0; i < n; ++i) hv[i] = 0.5f * (float)i - 7.f;
    skl::DeviceBuffer B(n * 4);
    B.upload(hv.data(), n * 4);
    if (ok) ok = skl_allreduce_grads(comm, B.as<float>(), n, nullptr) == SKL_OK;
    skl::check_cuda(cudaDeviceSynchronize(), "sync");
    std::vector<float> back(n);
    B.download(back.data(), n * 4);
    skl::check_cuda(cudaDeviceSynchronize(), "sync");
    ok = ok && back == hv;  // sum over one rank
    ok = ok && skl_allreduce_grads(nullptr, B.as<float>(), n, nullptr) == SKL_ERR_PARAM;
    if (comm) destroy(comm);
    report("skl_allreduce_grads over an NCCL communicator (world 1)", ok);
}

}  // namespace

int main() {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        std::printf("SKIP no CUDA device\n");
        return 77;
    }
    std::printf("libskl %s, rng %s\n", skl_version(), skl_rng_algorithm());
    try {
        test_sketch_bit_exact();
        parity_case("c1 tf32 1024->1024 l1 k64 T64", {1024, 1024, 1, 64, 64, SKL_F32_TF32});
        parity_case("c2 bf16 768->3072 l2 k128 T300", {768, 3072, 2, 128, 300, SKL_BF16});
        parity_case("tf32 768->3072 l2 k128 T130 (R=512, unfused)", {768, 3072, 2, 128, 130, SKL_F32_TF32});
        parity_case("rademacher bf16 256->512 l3 k32 T129", {256, 512, 3, 32, 129, SKL_BF16}, SKL_DIST_RADEMACHER);
        // shapes whose rows are not 16-byte multiples (any shape the reference accepts)
        parity_case("ragged bf16 7->64 l1 k8 T16", {7, 64, 1, 8, 16, SKL_BF16});
        parity_case("GradCheck shape tf32 6->8 l2 k3 T2 (test_nn_layers.cpp:158)", {6, 8, 2, 3, 2, SKL_F32_TF32});
        test_identity_sketches();
        test_zero_cases();
        test_batch_additivity();
        test_errors();
        test_params();
        test_from_dense();
        test_fused_relu_forward();
        test_nccl_allreduce_world1();
    } catch (const std::exception& e) {
        std::printf("FAIL uncaught exception: %s\n", e.what());
        ++g_fail;
    }
    std::printf("%d failure(s)\n", g_fail);
    return g_fail;
}
