/*
 * skl.hpp -- C++ host mirror of rnla::nn::SkLinear over the C-ABI (skl.h).
 *
 * Reference interface this mirrors (/root/reference/proj):
 *   class SkLinear { forward(x) -> Matrix; backward(x, grad_out) -> Grads; params(); }
 *                                                     include/rnla/nn/layers.hpp:52-81
 *   sk_linear_fresh(d_in, d_out, l, k, seed, dist)    layers.hpp:85-88, nn_layers.cpp:133-147
 *   SketchOp::with_realized (test hook: explicit sketches) sketch.hpp:36-38
 *   shape_error / parameter_error                     include/rnla/errors.hpp:10-19
 *
 * Same names, same argument meaning, same error behaviour (exceptions of the
 * same names), but DEVICE-resident and row convention (x [T, d_in]) with the
 * pawX [L, d, k] stacks of skl.h.  No PyTorch: memory is cudaMalloc'ed here,
 * all arithmetic runs in libskl.so's sm_100a kernels.  Header-only; link
 * with -lskl -lcudart.
 */
#ifndef SKL_HPP_
#define SKL_HPP_

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "skl.h"

namespace skl {

// ---------------------------------------------------------------- errors (errors.hpp:10-19)
struct shape_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct parameter_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(skl_status s) {
    if (s == SKL_OK) return;
    const std::string msg = skl_last_error();
    if (s == SKL_ERR_SHAPE) throw shape_error(msg);
    if (s == SKL_ERR_PARAM) throw parameter_error(msg);
    throw cuda_error(msg);
}
inline void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e));
}

inline size_t elem_bytes(skl_dtype t) { return t == SKL_BF16 ? 2 : 4; }

// Host value -> element i of an array of the variant's element type (fp32, or
// bf16 rounded to nearest even from the fp32 value).
inline void put_elem(uint8_t* dst, size_t i, double v, skl_dtype t) {
    float f = (float)v;
    if (t != SKL_BF16) {
        std::memcpy(dst + 4 * i, &f, 4);
        return;
    }
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    const uint16_t h = (uint16_t)(u >> 16);
    std::memcpy(dst + 2 * i, &h, 2);
}

// ---------------------------------------------------------------- device memory (RAII)
class DeviceBuffer {
  public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(size_t bytes) : bytes_(bytes) {
        if (bytes_) check_cuda(cudaMalloc(&ptr_, bytes_), "cudaMalloc");
    }
    ~DeviceBuffer() {
        if (ptr_) cudaFree(ptr_);
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : ptr_(std::exchange(o.ptr_, nullptr)), bytes_(std::exchange(o.bytes_, 0)) {}
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        if (this != &o) {
            if (ptr_) cudaFree(ptr_);
            ptr_ = std::exchange(o.ptr_, nullptr);
            bytes_ = std::exchange(o.bytes_, 0);
        }
        return *this;
    }
    void* get() const { return ptr_; }
    template <class T>
    T* as() const { return static_cast<T*>(ptr_); }
    size_t bytes() const { return bytes_; }
    void upload(const void* host, size_t n, cudaStream_t st = nullptr) {
        check_cuda(cudaMemcpyAsync(ptr_, host, n, cudaMemcpyHostToDevice, st), "upload");
    }
    void download(void* host, size_t n, cudaStream_t st = nullptr) const {
        check_cuda(cudaMemcpyAsync(host, ptr_, n, cudaMemcpyDeviceToHost, st), "download");
    }
    void zero(cudaStream_t st = nullptr) {
        if (bytes_) check_cuda(cudaMemsetAsync(ptr_, 0, bytes_, st), "memset");
    }

  private:
    void* ptr_ = nullptr;
    size_t bytes_ = 0;
};

// ---------------------------------------------------------------- SkLinear
class SkLinear {
  public:
    // SkLinear::Grads (layers.hpp:72-78) in ABI layout: grad_x [T, d_in]
    // (element type of the variant), grad_u1 = dU1s [L,k,d_out], grad_u2 =
    // dU2s [L,d_in,k], grad_b [d_out] (fp32).
    struct Grads {
        DeviceBuffer grad_x, grad_u1, grad_u2, grad_b;
    };

    // sk_linear_fresh (nn_layers.cpp:133-147): sketches from derive_seed(seed,
    // 2i / 2i+1), U ~ N(0, 2/(d_in+d_out)) from derive_seed(seed, 1000+i),
    // zero bias -- generated on the device, bit-matching the reference stream.
    static SkLinear fresh(int64_t d_in, int64_t d_out, int64_t l, int64_t k, uint64_t seed,
                          skl_dist dist = SKL_DIST_GAUSSIAN, skl_dtype dtype = SKL_BF16,
                          cudaStream_t st = nullptr) {
        SkLinear s(d_in, d_out, l, k, dtype);
        check(skl_generate_sketches(&s.shape_, dist, seed, s.S1s_.get(), s.S2s_.get(), st));
        check(skl_init_params(&s.shape_, seed, s.U1s_.get(), s.U2s_.get(), st));
        s.bias_.zero(st);
        return s;
    }

    // sk_linear_from_dense (nn_layers.cpp:149-160) on the device: W [d_out, d_in]
    // and bias [d_out] (nullable) are DEVICE arrays in the variant's element type.
    static SkLinear from_dense(const void* W, const void* bias, int64_t d_in, int64_t d_out, int64_t l, int64_t k,
                               uint64_t seed, skl_dist dist = SKL_DIST_GAUSSIAN, skl_dtype dtype = SKL_BF16,
                               cudaStream_t st = nullptr) {
        SkLinear s(d_in, d_out, l, k, dtype);
        size_t n = 0;
        check(skl_from_dense_workspace_size(&s.shape_, &n));
        DeviceBuffer ws(n);
        check(skl_from_dense(&s.shape_, dist, seed, W, bias, s.S1s_.get(), s.S2s_.get(), s.U1s_.get(),
                             s.U2s_.get(), s.bias_.get(), ws.get(), n, st));
        check_cuda(cudaStreamSynchronize(st), "sync");  // ws is released on return
        return s;
    }

    // Explicit parameters (host arrays in the variant's element type, ABI
    // layouts) -- the analogue of SketchOp::with_realized (sketch.hpp:36-38).
    static SkLinear with_params(int64_t d_in, int64_t d_out, int64_t l, int64_t k, skl_dtype dtype,
                                const void* S1s, const void* S2s, const void* U1s, const void* U2s,
                                const void* bias /*nullable*/, cudaStream_t st = nullptr) {
        SkLinear s(d_in, d_out, l, k, dtype);
        const size_t e = elem_bytes(dtype);
        s.S1s_.upload(S1s, (size_t)(l * d_in * k) * e, st);
        s.S2s_.upload(S2s, (size_t)(l * k * d_out) * e, st);
        s.U1s_.upload(U1s, (size_t)(l * k * d_out) * e, st);
        s.U2s_.upload(U2s, (size_t)(l * d_in * k) * e, st);
        if (bias) s.bias_.upload(bias, (size_t)d_out * e, st);
        else s.bias_.zero(st);
        return s;
    }

    // A layer from sketch DESCRIPTORS and explicit U / bias in the reference's
    // layout (sk_linear_from_json, nn_model.cpp:290-311): descs = [s1_0, s2_0,
    // s1_1, ...] (dist, seed) re-realised on the device -- bit-identical to
    // SketchOp::realized -- and host f64 u1 [L][k][d_in], u2 [L][d_out][k], bias
    // [d_out] rounded to the element type and transposed into U2s / U1s.
    struct SketchDesc {
        skl_dist dist;
        int64_t rows, cols;
        uint64_t seed;
    };
    static SkLinear from_parts(int64_t d_in, int64_t d_out, int64_t l, int64_t k, skl_dtype dtype,
                               const std::vector<SketchDesc>& descs, const double* u1, const double* u2,
                               const double* bias, cudaStream_t st = nullptr) {
        SkLinear s(d_in, d_out, l, k, dtype);
        if ((int64_t)descs.size() != 2 * l) throw shape_error("SKLinear: expected 2*num_terms sketches");
        const size_t e = elem_bytes(dtype);
        const skl_out_type ot = dtype == SKL_BF16 ? SKL_OUT_BF16 : SKL_OUT_F32;
        for (int64_t i = 0; i < l; ++i) {
            const SketchDesc& s1 = descs[2 * i];
            const SketchDesc& s2 = descs[2 * i + 1];
            if (s1.rows != k || s1.cols != d_out || s2.rows != k || s2.cols != d_in)
                throw shape_error("SKLinear: sketch shape disagrees with the layer");
            check(skl_realize_sketch(s1.dist, k, d_out, s1.seed, 0, 0, ot,
                                     static_cast<uint8_t*>(s.S2s_.get()) + (size_t)(i * k * d_out) * e, st));
            check(skl_realize_sketch(s2.dist, k, d_in, s2.seed, 0, 1, ot,
                                     static_cast<uint8_t*>(s.S1s_.get()) + (size_t)(i * d_in * k) * e, st));
        }
        std::vector<uint8_t> U1((size_t)(l * k * d_out) * e), U2((size_t)(l * d_in * k) * e), b((size_t)d_out * e);
        for (int64_t i = 0; i < l; ++i)
            for (int64_t j = 0; j < k; ++j) {
                for (int64_t c = 0; c < d_in; ++c)  // U2s[i][c][j] = u1[i][j][c]
                    put_elem(U2.data(), (size_t)((i * d_in + c) * k + j), u1[(i * k + j) * d_in + c], dtype);
                for (int64_t o = 0; o < d_out; ++o)  // U1s[i][j][o] = u2[i][o][j]
                    put_elem(U1.data(), (size_t)((i * k + j) * d_out + o), u2[(i * d_out + o) * k + j], dtype);
            }
        for (int64_t o = 0; o < d_out; ++o) put_elem(b.data(), (size_t)o, bias ? bias[o] : 0.0, dtype);
        s.U1s_.upload(U1.data(), U1.size(), st);
        s.U2s_.upload(U2.data(), U2.size(), st);
        s.bias_.upload(b.data(), b.size(), st);
        check_cuda(cudaStreamSynchronize(st), "sync");  // host staging is released on return
        return s;
    }

    int64_t d_in() const { return shape_.d_in; }
    int64_t d_out() const { return shape_.d_out; }
    int64_t num_terms() const { return shape_.num_terms; }
    int64_t low_rank() const { return shape_.low_rank; }
    skl_dtype dtype() const { return shape_.dtype; }
    const skl_shape& shape() const { return shape_; }

    void* S1s() const { return S1s_.get(); }
    void* S2s() const { return S2s_.get(); }
    void* U1s() const { return U1s_.get(); }
    void* U2s() const { return U2s_.get(); }
    void* bias() const { return bias_.get(); }

    // SkLinear::params (nn_layers.cpp:103-110)
    skl_param_count params() const {
        skl_param_count pc;
        check(skl_params(&shape_, &pc));
        return pc;
    }

    // Row stride (elements) of the saved projection [L*k][round8(T)].
    static int64_t saved_ld(int64_t T) { return (T + 7) / 8 * 8; }
    size_t saved_bytes(int64_t T) const {
        return (size_t)(shape_.num_terms * shape_.low_rank) * (size_t)saved_ld(T) * elem_bytes(shape_.dtype);
    }

    // SkLinear::forward (nn_layers.cpp:61-76), device pointers:
    // x [T, d_in] -> y [T, d_out]; saved (nullable) [L*k][round8(T)] keeps x·S1_i.
    // fuse = SKL_FUSE_RELU_OUT applies a following ReLU in the epilogue.
    // relu_bits (with SKL_FUSE_RELU_OUT): also write the 1-bit ReLU mask,
    // [T][skl_relu_bits_row_words(d_out)] uint32, for the next layer's backward.
    void forward(const void* x, int64_t T, void* y, void* saved = nullptr, cudaStream_t st = nullptr,
                 unsigned fuse = 0, uint32_t* relu_bits = nullptr) const {
        if (T < 0) throw shape_error("SkLinear::forward: negative token count");
        void* ws = workspace(T, st);
        if (relu_bits) {
            check(sketched_linear_forward_bits(&shape_, T, fuse | SKL_FUSE_RELU_BITS, x, S1s_.get(), S2s_.get(),
                                               U1s_.get(), U2s_.get(), bias_.get(), y, saved, relu_bits, ws,
                                               ws_.bytes(), st));
            return;
        }
        check(sketched_linear_forward_ex(&shape_, T, fuse, x, S1s_.get(), S2s_.get(), U1s_.get(), U2s_.get(),
                                         bias_.get(), y, saved, ws, ws_.bytes(), st));
    }
    // Whether this layer's kernels take 1-bit ReLU masks (skl_relu_bits_supported).
    bool relu_bits_supported() const { return skl_relu_bits_supported(&shape_) != 0; }

    // SkLinear::backward (nn_layers.cpp:78-101): gradients allocated here.
    Grads backward(const void* x, const void* grad_out, int64_t T, const void* saved = nullptr,
                   cudaStream_t st = nullptr) const {
        Grads g{DeviceBuffer((size_t)(T * shape_.d_in) * elem_bytes(shape_.dtype)),
                DeviceBuffer((size_t)(shape_.num_terms * shape_.low_rank * shape_.d_out) * 4),
                DeviceBuffer((size_t)(shape_.num_terms * shape_.low_rank * shape_.d_in) * 4),
                DeviceBuffer((size_t)shape_.d_out * 4)};
        backward_into(x, grad_out, T, saved, g.grad_x.get(), g.grad_u1.as<float>(), g.grad_u2.as<float>(),
                      g.grad_b.as<float>(), st);
        return g;
    }

    // Allocation-free backward into caller buffers (e.g. one contiguous
    // dU1s | dU2s | db bucket for the NCCL all-reduce).  grad_x / grad_b nullable.
    // phases: SKL_BWD_ALL, or SKL_BWD_DU1_DB then SKL_BWD_DX_DU2 (data-parallel overlap);
    // fuse = SKL_FUSE_RELU_IN masks grad_x by (x > 0) (the preceding ReLU's backward).
    // relu_bits (with SKL_FUSE_RELU_IN): the previous layer's 1-bit ReLU mask instead of x.
    void backward_into(const void* x, const void* grad_out, int64_t T, const void* saved, void* grad_x, float* dU1s,
                       float* dU2s, float* db, cudaStream_t st = nullptr, unsigned phases = SKL_BWD_ALL,
                       unsigned fuse = 0, const uint32_t* relu_bits = nullptr) const {
        if (T < 0) throw shape_error("SkLinear::backward: negative token count");
        void* ws = workspace(T, st);
        if (relu_bits) {
            check(sketched_linear_backward_bits(&shape_, T, phases, fuse | SKL_FUSE_RELU_BITS, grad_out, x, saved,
                                                S1s_.get(), S2s_.get(), U1s_.get(), U2s_.get(), grad_x, dU1s, dU2s,
                                                db, relu_bits, ws, ws_.bytes(), st));
            return;
        }
        check(sketched_linear_backward_ex(&shape_, T, phases, fuse, grad_out, x, saved, S1s_.get(), S2s_.get(),
                                          U1s_.get(), U2s_.get(), grad_x, dU1s, dU2s, db, ws, ws_.bytes(), st));
    }

    // Host-buffer convenience (the reference's value-semantics call):
    // x_host [T, d_in] in the variant's element type -> y_host [T, d_out].
    std::vector<uint8_t> forward_host(const void* x_host, int64_t T, cudaStream_t st = nullptr) const {
        const size_t e = elem_bytes(shape_.dtype);
        DeviceBuffer x((size_t)(T * shape_.d_in) * e), y((size_t)(T * shape_.d_out) * e);
        x.upload(x_host, x.bytes(), st);
        forward(x.get(), T, y.get(), nullptr, st);
        std::vector<uint8_t> out(y.bytes());
        y.download(out.data(), out.size(), st);
        check_cuda(cudaStreamSynchronize(st), "sync");
        return out;
    }

  private:
    SkLinear(int64_t d_in, int64_t d_out, int64_t l, int64_t k, skl_dtype dtype) {
        if (l < 1 || k < 1) throw parameter_error("SkLinear: l and k must be >= 1");  // nn_layers.cpp:116
        if (d_in < 1 || d_out < 1) throw shape_error("SkLinear: d_in and d_out must be >= 1");
        shape_ = skl_shape{d_in, d_out, l, k, dtype};
        const size_t e = elem_bytes(dtype);
        S1s_ = DeviceBuffer((size_t)(l * d_in * k) * e);
        U2s_ = DeviceBuffer((size_t)(l * d_in * k) * e);
        U1s_ = DeviceBuffer((size_t)(l * k * d_out) * e);
        S2s_ = DeviceBuffer((size_t)(l * k * d_out) * e);
        bias_ = DeviceBuffer((size_t)d_out * e);
    }

    void* workspace(int64_t T, cudaStream_t st) const {
        size_t f = 0, b = 0;
        check(skl_workspace_size(&shape_, T, &f, &b));
        const size_t need = f > b ? f : b;
        if (ws_.bytes() < need) {
            check_cuda(cudaStreamSynchronize(st), "sync");  // the old workspace may still be in use
            ws_ = DeviceBuffer(need);
        }
        return ws_.get();
    }

    skl_shape shape_{};
    DeviceBuffer S1s_, S2s_, U1s_, U2s_, bias_;
    mutable DeviceBuffer ws_;
};

// ---------------------------------------------------------------- DenseLinear
// rnla::nn::DenseLinear (layers.hpp:33-48; nn_layers.cpp:32-59), device-resident,
// row convention: y = x·Wᵀ + b with W [d_out, d_in] (the reference's w).
class DenseLinear {
  public:
    // dense_linear_init (nn_layers.cpp:51-59): W = gaussian_matrix(d_out, d_in,
    // seed) * sqrt(2/(d_in+d_out)) generated on the device; zero bias.
    static DenseLinear fresh(int64_t d_in, int64_t d_out, uint64_t seed, skl_dtype dtype = SKL_BF16,
                             cudaStream_t st = nullptr) {
        DenseLinear d(d_in, d_out, dtype);
        check(skl_dense_init(&d.shape_, seed, d.W_.get(), d.bias_.get(), st));
        return d;
    }
    // Explicit W [d_out, d_in] and bias [d_out] (host arrays, element type of the variant).
    static DenseLinear with_params(int64_t d_in, int64_t d_out, skl_dtype dtype, const void* W, const void* bias,
                                   cudaStream_t st = nullptr) {
        DenseLinear d(d_in, d_out, dtype);
        d.W_.upload(W, d.W_.bytes(), st);
        if (bias) d.bias_.upload(bias, d.bias_.bytes(), st);
        else d.bias_.zero(st);
        return d;
    }

    // From host f64 w [d_out][d_in] and b [d_out] (a model file's Linear record).
    static DenseLinear from_parts(int64_t d_in, int64_t d_out, skl_dtype dtype, const double* w, const double* b,
                                  cudaStream_t st = nullptr) {
        const size_t e = elem_bytes(dtype);
        std::vector<uint8_t> W((size_t)(d_out * d_in) * e), B((size_t)d_out * e);
        for (int64_t i = 0; i < d_out * d_in; ++i) put_elem(W.data(), (size_t)i, w[i], dtype);
        for (int64_t o = 0; o < d_out; ++o) put_elem(B.data(), (size_t)o, b ? b[o] : 0.0, dtype);
        DenseLinear d = with_params(d_in, d_out, dtype, W.data(), B.data(), st);
        check_cuda(cudaStreamSynchronize(st), "sync");
        return d;
    }

    int64_t d_in() const { return shape_.d_in; }
    int64_t d_out() const { return shape_.d_out; }
    skl_dtype dtype() const { return shape_.dtype; }
    const skl_dense_shape& shape() const { return shape_; }
    void* W() const { return W_.get(); }
    void* bias() const { return bias_.get(); }

    // DenseLinear::forward: x [T, d_in] -> y [T, d_out]; fuse = SKL_FUSE_RELU_OUT.
    void forward(const void* x, int64_t T, void* y, cudaStream_t st = nullptr, unsigned fuse = 0) const {
        if (T < 0) throw shape_error("DenseLinear::forward: negative token count");
        void* ws = workspace(T, st);
        check(dense_linear_forward(&shape_, T, fuse, x, W_.get(), bias_.get(), y, ws, ws_.bytes(), st));
    }
    // DenseLinear::backward into caller buffers: grad_x [T, d_in] (nullable),
    // dW [d_out, d_in] and db [d_out] fp32 (db nullable); fuse = SKL_FUSE_RELU_IN.
    void backward_into(const void* x, const void* grad_out, int64_t T, void* grad_x, float* dW, float* db,
                       cudaStream_t st = nullptr, unsigned fuse = 0) const {
        if (T < 0) throw shape_error("DenseLinear::backward: negative token count");
        void* ws = workspace(T, st);
        check(dense_linear_backward(&shape_, T, fuse, grad_out, x, W_.get(), grad_x, dW, db, ws, ws_.bytes(), st));
    }

  private:
    DenseLinear(int64_t d_in, int64_t d_out, skl_dtype dtype) {
        if (d_in < 1 || d_out < 1) throw shape_error("DenseLinear: d_in and d_out must be >= 1");
        shape_ = skl_dense_shape{d_in, d_out, dtype};
        W_ = DeviceBuffer((size_t)(d_out * d_in) * elem_bytes(dtype));
        bias_ = DeviceBuffer((size_t)d_out * elem_bytes(dtype));
    }
    void* workspace(int64_t T, cudaStream_t st) const {
        size_t f = 0, b = 0;
        check(skl_dense_workspace_size(&shape_, T, &f, &b));
        const size_t need = f > b ? f : b;
        if (ws_.bytes() < need) {
            check_cuda(cudaStreamSynchronize(st), "sync");
            ws_ = DeviceBuffer(need);
        }
        return ws_.get();
    }

    skl_dense_shape shape_{};
    DeviceBuffer W_, bias_;
    mutable DeviceBuffer ws_;
};

}  // namespace skl

#endif  // SKL_HPP_
