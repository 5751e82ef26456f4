// ref_shim.cpp -- extern "C" adapter over the UNMODIFIED reference sources.
//
// TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline timer).  Built by
// oracle/Makefile together with /root/reference/proj/src/{linalg,sketch,
// nn_layers,bench,nn_attention,decomp}.cpp into oracle/_ref/librnla_ref.so,
// using the reference's own flags (-std=c++20 -O3 -DNDEBUG -fopenmp, no
// -march; proj/CMakeLists.txt:3-12).  Nothing here re-implements the
// algorithm: every entry point calls the reference's public C++ API
//   rnla::derive_seed / Splitmix64 / GaussianStream   rng.hpp:13-69
//   rnla::sketch::make_sketch / realized             sketch.cpp:72-108
//   rnla::nn::sk_linear_fresh                         nn_layers.cpp:133-147
//   rnla::nn::SkLinear::forward / backward            nn_layers.cpp:61-101
//   rnla::bench::time_op / set_timing_threads         bench.cpp:28-76
// Layouts are the reference's (column convention, row-major f64 stacks:
// s1[l][k][d_out], u1[l][k][d_in], s2[l][k][d_in], u2[l][d_out][k]).
// Exceptions never cross this boundary: shape_error -> 1, parameter_error
// -> 2, anything else -> 9, with the message kept for ref_last_error().
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "rnla/bench.hpp"
#include "rnla/errors.hpp"
#include "rnla/nn/layers.hpp"
#include "rnla/rng.hpp"
#include "rnla/sketch.hpp"

using rnla::Matrix;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const rnla::shape_error& e) {
        g_err = e.what();
        return 1;
    } catch (const rnla::parameter_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

Matrix from_ptr(std::size_t r, std::size_t c, const double* p) {
    return Matrix(r, c, std::vector<double>(p, p + r * c));
}

void to_ptr(const Matrix& m, double* p) { std::memcpy(p, m.data(), m.size() * sizeof(double)); }

rnla::sketch::SketchDist dist_of(int d) {
    if (d == 0) return rnla::sketch::SketchDist::Gaussian;
    if (d == 1) return rnla::sketch::SketchDist::Rademacher;
    throw rnla::parameter_error("ref_shim: dist must be 0 (gaussian) or 1 (rademacher)");
}

// A layer whose sketches are injected through the reference's test hook
// SketchOp::with_realized (sketch.hpp:36-38), so forward/backward run on
// exactly the matrices the caller provides.
rnla::nn::SkLinear make_layer(std::uint64_t d_in, std::uint64_t d_out, std::uint64_t l,
                              std::uint64_t k, const double* s1, const double* u1,
                              const double* s2, const double* u2, const double* bias) {
    rnla::nn::SkLinear layer;
    layer.d_in = d_in;
    layer.d_out = d_out;
    layer.num_terms = l;
    layer.low_rank = k;
    layer.bias.assign(bias ? bias : nullptr, bias ? bias + d_out : nullptr);
    if (!bias) layer.bias.assign(d_out, 0.0);
    layer.terms.resize(l);
    for (std::size_t i = 0; i < l; ++i) {
        layer.terms[i].s1 = rnla::sketch::SketchOp::with_realized(from_ptr(k, d_out, s1 + i * k * d_out));
        layer.terms[i].u1 = from_ptr(k, d_in, u1 + i * k * d_in);
        layer.terms[i].s2 = rnla::sketch::SketchOp::with_realized(from_ptr(k, d_in, s2 + i * k * d_in));
        layer.terms[i].u2 = from_ptr(d_out, k, u2 + i * d_out * k);
    }
    return layer;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

const char* ref_rng_algorithm(void) { return rnla::kRngAlgorithm; }

std::uint64_t ref_derive_seed(std::uint64_t master, std::uint64_t index) {
    return rnla::derive_seed(master, index);
}

void ref_splitmix64_stream(std::uint64_t seed, std::uint64_t n, std::uint64_t* out) {
    rnla::Splitmix64 s(seed);
    for (std::uint64_t i = 0; i < n; ++i) out[i] = s.next_u64();
}

void ref_gaussian_stream(std::uint64_t seed, std::uint64_t n, double* out) {
    rnla::GaussianStream g(seed);
    for (std::uint64_t i = 0; i < n; ++i) out[i] = g.next();
}

int ref_realize_sketch(int dist, std::uint64_t k, std::uint64_t d, std::uint64_t seed, double* out) {
    return guard([&] { to_ptr(rnla::sketch::make_sketch(dist_of(dist), k, d, seed).realized(), out); });
}

int ref_gaussian_matrix(std::uint64_t rows, std::uint64_t cols, std::uint64_t seed, double* out) {
    return guard([&] { to_ptr(rnla::sketch::gaussian_matrix(rows, cols, seed), out); });
}

int ref_sk_linear_fresh(std::uint64_t d_in, std::uint64_t d_out, std::uint64_t l, std::uint64_t k,
                        std::uint64_t seed, int dist, double* s1, double* u1, double* s2, double* u2) {
    return guard([&] {
        const auto layer = rnla::nn::sk_linear_fresh(d_in, d_out, l, k, seed, dist_of(dist));
        for (std::size_t i = 0; i < l; ++i) {
            to_ptr(layer.terms[i].s1.realized(), s1 + i * k * d_out);
            to_ptr(layer.terms[i].u1, u1 + i * k * d_in);
            to_ptr(layer.terms[i].s2.realized(), s2 + i * k * d_in);
            to_ptr(layer.terms[i].u2, u2 + i * d_out * k);
        }
    });
}

int ref_sk_forward(std::uint64_t d_in, std::uint64_t d_out, std::uint64_t l, std::uint64_t k,
                   std::uint64_t T, const double* s1, const double* u1, const double* s2,
                   const double* u2, const double* bias, const double* x, double* y) {
    return guard([&] {
        const auto layer = make_layer(d_in, d_out, l, k, s1, u1, s2, u2, bias);
        to_ptr(layer.forward(from_ptr(d_in, T, x)), y);
    });
}

// Shape-checked forward on an arbitrary x (x_rows may differ from d_in, to
// pin the reference's shape_error contract, nn_layers.cpp:62).
int ref_sk_forward_checked(std::uint64_t d_in, std::uint64_t d_out, std::uint64_t l,
                           std::uint64_t k, std::uint64_t x_rows, std::uint64_t T) {
    return guard([&] {
        const auto layer = rnla::nn::sk_linear_fresh(d_in, d_out, l, k, 1);
        (void)layer.forward(Matrix(x_rows, T));
    });
}

int ref_sk_backward(std::uint64_t d_in, std::uint64_t d_out, std::uint64_t l, std::uint64_t k,
                    std::uint64_t T, const double* s1, const double* u1, const double* s2,
                    const double* u2, const double* x, const double* g, double* gx, double* gu1,
                    double* gu2, double* gb) {
    return guard([&] {
        const auto layer = make_layer(d_in, d_out, l, k, s1, u1, s2, u2, nullptr);
        const auto grads = layer.backward(from_ptr(d_in, T, x), from_ptr(d_out, T, g));
        to_ptr(grads.grad_x, gx);
        for (std::size_t i = 0; i < l; ++i) {
            to_ptr(grads.grad_u1[i], gu1 + i * k * d_in);
            to_ptr(grads.grad_u2[i], gu2 + i * d_out * k);
        }
        std::memcpy(gb, grads.grad_b.data(), d_out * sizeof(double));
    });
}

// DenseLinear (nn_layers.cpp:32-59) through the reference's own API.
int ref_dense_init(std::uint64_t d_in, std::uint64_t d_out, std::uint64_t seed, double* w, double* b) {
    return guard([&] {
        const auto layer = rnla::nn::dense_linear_init(d_in, d_out, seed);
        to_ptr(layer.w, w);
        std::memcpy(b, layer.b.data(), d_out * sizeof(double));
    });
}

int ref_dense_forward(std::uint64_t d_in, std::uint64_t d_out, std::uint64_t T, const double* w, const double* b,
                      const double* x, double* y) {
    return guard([&] {
        rnla::nn::DenseLinear layer;
        layer.w = from_ptr(d_out, d_in, w);
        layer.b.assign(b, b + d_out);
        to_ptr(layer.forward(from_ptr(d_in, T, x)), y);
    });
}

int ref_dense_backward(std::uint64_t d_in, std::uint64_t d_out, std::uint64_t T, const double* w, const double* x,
                       const double* g, double* gx, double* gw, double* gb) {
    return guard([&] {
        rnla::nn::DenseLinear layer;
        layer.w = from_ptr(d_out, d_in, w);
        layer.b.assign(d_out, 0.0);
        const auto grads = layer.backward(from_ptr(d_in, T, x), from_ptr(d_out, T, g));
        to_ptr(grads.grad_x, gx);
        to_ptr(grads.grad_w, gw);
        std::memcpy(gb, grads.grad_b.data(), d_out * sizeof(double));
    });
}

// CPU baseline: the reference's own SkLinear forward+backward timed by the
// reference's own harness (bench::time_op, bench.cpp:28-76) on `threads`
// OpenMP workers.  Inputs follow BASELINE.md §3: layer sk_linear_fresh(seed),
// x = gaussian_matrix(d_in,T,derive_seed(seed,7)), G = gaussian_matrix(d_out,
// T,derive_seed(seed,9)), bias = gaussian_matrix(1,d_out,derive_seed(seed,11)).
int ref_time_fwd_bwd(std::uint64_t d_in, std::uint64_t d_out, std::uint64_t l, std::uint64_t k,
                     std::uint64_t T, std::uint64_t seed, int threads, std::uint64_t trials,
                     std::uint64_t warmup, double* mean_ms, double* std_ms) {
    return guard([&] {
        auto layer = rnla::nn::sk_linear_fresh(d_in, d_out, l, k, seed);
        const Matrix b = rnla::sketch::gaussian_matrix(1, d_out, rnla::derive_seed(seed, 11));
        layer.bias.assign(b.data(), b.data() + d_out);
        for (auto& t : layer.terms) {  // realize outside the timed region
            (void)t.s1.realized();
            (void)t.s2.realized();
        }
        const Matrix x = rnla::sketch::gaussian_matrix(d_in, T, rnla::derive_seed(seed, 7));
        const Matrix g = rnla::sketch::gaussian_matrix(d_out, T, rnla::derive_seed(seed, 9));
        rnla::bench::set_timing_threads(threads);
        double sink = 0.0;
        const auto st = rnla::bench::time_op(
            [&] {
                const Matrix y = layer.forward(x);
                const auto gr = layer.backward(x, g);
                sink += y.data()[0] + gr.grad_x.data()[0];
            },
            trials, warmup);
        *mean_ms = st.mean_ms;
        *std_ms = st.std_ms + 0.0 * sink;
    });
}

int ref_max_threads(void) {
#ifdef _OPENMP
    return omp_get_num_procs();
#else
    return 1;
#endif
}

}  // extern "C"

// ---- SkConv2d (nn_layers.cpp:226-314) on explicit parameters -------------------
namespace {
rnla::nn::SkConv2d make_conv(const std::uint64_t* geo, std::uint64_t l, std::uint64_t k, const double* s1,
                             const double* u1, const double* s2, const double* u2, const double* bias) {
    rnla::nn::SkConv2d c;
    c.shape.c_in = geo[0];
    c.shape.c_out = geo[1];
    c.shape.kernel_h = geo[2];
    c.shape.kernel_w = geo[3];
    c.shape.stride = geo[4];
    c.shape.padding = geo[5];
    c.inner = make_layer(c.shape.lowered_d_in(), c.shape.c_out, l, k, s1, u1, s2, u2, bias);
    return c;
}
rnla::nn::ImageBatch make_images(std::uint64_t B, std::uint64_t C, std::uint64_t H, std::uint64_t W, const double* p) {
    rnla::nn::ImageBatch x;
    x.batch = B;
    x.channels = C;
    x.height = H;
    x.width = W;
    x.data.assign(p, p + B * C * H * W);
    return x;
}
}  // namespace

extern "C" {
// geo = {c_in, c_out, kernel_h, kernel_w, stride, padding}; x NCHW [B, c_in, H, W]; y [B, c_out, oh, ow]
int ref_skconv_forward(const std::uint64_t* geo, std::uint64_t l, std::uint64_t k, const double* s1,
                       const double* u1, const double* s2, const double* u2, const double* bias, std::uint64_t B,
                       std::uint64_t H, std::uint64_t W, const double* x, double* y) {
    return guard([&] {
        const auto c = make_conv(geo, l, k, s1, u1, s2, u2, bias);
        const auto out = c.forward(make_images(B, geo[0], H, W, x));
        std::memcpy(y, out.data.data(), out.data.size() * sizeof(double));
    });
}

int ref_skconv_backward(const std::uint64_t* geo, std::uint64_t l, std::uint64_t k, const double* s1,
                        const double* u1, const double* s2, const double* u2, std::uint64_t B, std::uint64_t H,
                        std::uint64_t W, const double* x, const double* g, double* gx, double* gu1, double* gu2,
                        double* gb) {
    return guard([&] {
        const auto c = make_conv(geo, l, k, s1, u1, s2, u2, nullptr);
        const std::uint64_t oh = c.shape.out_h(H), ow = c.shape.out_w(W);
        const auto gr = c.backward(make_images(B, geo[0], H, W, x), make_images(B, geo[1], oh, ow, g));
        std::memcpy(gx, gr.grad_x.data.data(), gr.grad_x.data.size() * sizeof(double));
        const std::uint64_t d_in = c.shape.lowered_d_in(), d_out = c.shape.c_out;
        for (std::uint64_t i = 0; i < l; ++i) {
            std::memcpy(gu1 + i * k * d_in, gr.grad_u1[i].data(), k * d_in * sizeof(double));
            std::memcpy(gu2 + i * d_out * k, gr.grad_u2[i].data(), d_out * k * sizeof(double));
        }
        std::memcpy(gb, gr.grad_b.data(), d_out * sizeof(double));
    });
}
}  // extern "C"
