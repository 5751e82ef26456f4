// ref_model_shim.cpp -- extern "C" adapter over the UNMODIFIED reference model
// container (/root/reference/proj/src/nn_model.cpp): model_save / model_load /
// model_forward (nn_model.cpp:111-122, 396-531).
//
// TEST INFRASTRUCTURE ONLY.  Used to produce reference-written model files
// (tests/golden/make_golden_model.py) and to run the reference's own
// model_forward on a file this repo wrote (round-trip test).  Built into
// oracle/_ref/librnla_ref.so by oracle/Makefile when nlohmann/json.hpp is
// available (the reference's vendor/ tree is absent).
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "rnla/errors.hpp"
#include "rnla/nn/layers.hpp"
#include "rnla/nn/model.hpp"
#include "rnla/rng.hpp"
#include "rnla/sketch.hpp"

namespace {
thread_local std::string g_merr;

template <class F>
int mguard(F&& f) {
    try {
        f();
        return 0;
    } catch (const rnla::shape_error& e) {
        g_merr = e.what();
        return 1;
    } catch (const rnla::parameter_error& e) {
        g_merr = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_merr = e.what();
        return 9;
    }
}
}  // namespace

extern "C" {

const char* ref_model_last_error(void) { return g_merr.c_str(); }

// Build a Linear/ReLU chain with the reference's own constructors and save it.
// spec: n rows of {type (0 = SKLinear, 1 = ReLU, 2 = Linear), d_in, d_out, l, k, seed, dist}.
// SKLinear layers are sk_linear_fresh(d_in, d_out, l, k, seed, dist) with bias
// gaussian_matrix(1, d_out, derive_seed(seed, 11)) * 0.5 (a fresh bias is zero).
int ref_model_save_chain(const char* path, int f32, int n, const std::uint64_t* spec) {
    return mguard([&] {
        rnla::nn::Model m;
        m.dtype = f32 ? "f32" : "f64";
        for (int i = 0; i < n; ++i) {
            const std::uint64_t* s = spec + 7 * i;
            rnla::nn::NamedLayer nl;
            nl.name = "layer" + std::to_string(i);
            if (s[0] == 1) {
                nl.layer = rnla::nn::Relu{};
            } else if (s[0] == 2) {  // DenseLinear: dense_linear_init(d_in, d_out, seed), bias as below
                rnla::nn::DenseLinear d = rnla::nn::dense_linear_init(s[1], s[2], s[5]);
                const rnla::Matrix b = rnla::sketch::gaussian_matrix(1, s[2], rnla::derive_seed(s[5], 11));
                for (std::size_t j = 0; j < s[2]; ++j) d.b[j] = 0.5 * b.data()[j];
                nl.layer = std::move(d);
            } else {
                rnla::nn::SkLinear l = rnla::nn::sk_linear_fresh(
                    s[1], s[2], s[3], s[4], s[5], s[6] ? rnla::sketch::SketchDist::Rademacher
                                                       : rnla::sketch::SketchDist::Gaussian);
                const rnla::Matrix b = rnla::sketch::gaussian_matrix(1, s[2], rnla::derive_seed(s[5], 11));
                for (std::size_t j = 0; j < s[2]; ++j) l.bias[j] = 0.5 * b.data()[j];
                nl.layer = std::move(l);
            }
            m.layers.push_back(std::move(nl));
        }
        rnla::nn::model_save(m, path);
    });
}

// model_load(path) then model_forward(x): x is [d_in x T] (column convention).
int ref_model_forward_file(const char* path, std::uint64_t d_in, std::uint64_t T, const double* x,
                           std::uint64_t d_out, double* y) {
    return mguard([&] {
        const rnla::nn::Model m = rnla::nn::model_load(path);
        rnla::Matrix xm(d_in, T, std::vector<double>(x, x + d_in * T));
        const rnla::Matrix ym = rnla::nn::model_forward(m, xm);
        if (ym.rows() != d_out || ym.cols() != T) throw rnla::shape_error("ref_model_forward_file: output shape");
        std::memcpy(y, ym.data(), d_out * T * sizeof(double));
    });
}

}  // extern "C"
