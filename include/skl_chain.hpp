/*
 * skl_chain.hpp -- model_forward over Linear / SKLinear / ReLU layers, with a
 * training backward, in C++ over the C-ABI (no PyTorch).
 *
 * Reference (/root/reference/proj):
 *   Matrix model_forward(const Model&, const Matrix& x)   nn_model.cpp:111-122
 *   Relu::forward / Relu::backward                         nn_layers.cpp:341-354
 *   DenseLinear / SkLinear forward + backward              nn_layers.cpp:32-101
 * Same layer order and the same shape_error for a layer that is not part of a
 * Linear/ReLU chain; device-resident, row convention (x [T, d_in]).
 *
 * Every ReLU is fused into its neighbours instead of running as a kernel: the
 * forward applies it in the epilogue of the layer it follows
 * (SKL_FUSE_RELU_OUT) and the backward applies its mask in the dX epilogue of
 * the layer it feeds (SKL_FUSE_RELU_IN, x > 0 with x that layer's input).
 * Between two SKLinear layers whose kernels support it the mask travels as
 * 1 bit per element (SKL_FUSE_RELU_BITS).  With a Dp (skl_dp.hpp) each layer's
 * fp32 gradient bucket is all-reduced as soon as its backward is done, the
 * collective overlapping the backward of the layers below.
 */
#ifndef SKL_CHAIN_HPP_
#define SKL_CHAIN_HPP_

#include <variant>

#include "skl.hpp"
#include "skl_dp.hpp"

namespace skl {

struct Relu {};  // rnla::nn::Relu (layers.hpp) -- always fused

class Chain {
  public:
    using Layer = std::variant<SkLinear, DenseLinear, Relu>;

    explicit Chain(std::vector<Layer> layers, bool relu_bits = true) : layers_(std::move(layers)) {
        bool prev_relu = false;
        for (size_t i = 0; i < layers_.size(); ++i) {
            if (std::holds_alternative<Relu>(layers_[i])) {
                if (steps_.empty())
                    throw shape_error("Chain: a leading ReLU has no producing layer to fuse into");
                steps_.back().relu_out = true;  // ReLU∘ReLU == ReLU
                prev_relu = true;
                continue;
            }
            Step s;
            s.idx = i;
            s.relu_in = prev_relu;
            if (!steps_.empty() && d_out_of(steps_.back()) != d_in_of(s))
                throw shape_error("model_forward: layer " + std::to_string(i) + " d_in != previous d_out");
            if (!steps_.empty() && dtype_of(steps_.back()) != dtype_of(s))
                throw parameter_error("Chain: all layers must share one element type");
            steps_.push_back(std::move(s));
            prev_relu = false;
        }
        if (steps_.empty()) throw shape_error("Chain: no Linear / SKLinear layer");
        for (size_t i = 0; i + 1 < steps_.size(); ++i) {  // 1-bit masks between two bit-capable SKLinear layers
            const SkLinear* a = std::get_if<SkLinear>(&layers_[steps_[i].idx]);
            const SkLinear* b = std::get_if<SkLinear>(&layers_[steps_[i + 1].idx]);
            steps_[i].bits_out = relu_bits && steps_[i].relu_out && a && b && a->relu_bits_supported() &&
                                 b->relu_bits_supported();
        }
        for (Step& s : steps_) {  // gradient bucket layouts
            if (const SkLinear* L = std::get_if<SkLinear>(&layers_[s.idx])) s.grad_count = SkBucket::of(*L).count();
            else {
                const DenseLinear& D = std::get<DenseLinear>(layers_[s.idx]);
                s.grad_count = (size_t)(D.d_out() * D.d_in() + D.d_out());
            }
            s.grads = DeviceBuffer(s.grad_count * 4);
        }
    }

    size_t num_layers() const { return layers_.size(); }
    const Layer& layer(size_t i) const { return layers_[i]; }
    int64_t d_in() const { return d_in_of(steps_.front()); }
    int64_t d_out() const { return d_out_of(steps_.back()); }
    skl_dtype dtype() const { return dtype_of(steps_.front()); }

    // model_forward: x [T, d_in] (device; kept by pointer for backward) ->
    // y [T, d_out] in an internal buffer valid until the next forward.
    const void* forward(const void* x, int64_t T, cudaStream_t st = nullptr, bool train = true) {
        if (T < 0) throw shape_error("model_forward: negative token count");
        reserve(T);
        const void* cur = x;
        for (size_t i = 0; i < steps_.size(); ++i) {
            Step& s = steps_[i];
            s.x = cur;
            const unsigned fuse = s.relu_out ? SKL_FUSE_RELU_OUT : 0;
            if (const SkLinear* L = std::get_if<SkLinear>(&layers_[s.idx])) {
                L->forward(cur, T, s.y.get(), train ? s.saved.get() : nullptr, st, fuse,
                           (train && s.bits_out) ? s.bits.as<uint32_t>() : nullptr);
            } else {
                std::get<DenseLinear>(layers_[s.idx]).forward(cur, T, s.y.get(), st, fuse);
            }
            cur = s.y.get();
        }
        T_ = T;
        return cur;
    }

    // Training backward from grad_out [T, d_out]: layer gradients into each
    // layer's fp32 bucket (grads(i)); grad_x [T, d_in] (nullable).  With dp,
    // each bucket's all-reduce is issued right after that layer's backward.
    void backward(const void* grad_out, int64_t T, cudaStream_t st = nullptr, void* grad_x = nullptr,
                  Dp* dp = nullptr) {
        if (T != T_) throw shape_error("Chain::backward: token count differs from the forward's");
        const void* g = grad_out;
        for (size_t i = steps_.size(); i-- > 0;) {
            Step& s = steps_[i];
            void* gx = i > 0 ? gbuf_[i & 1].get() : grad_x;
            const unsigned fuse = s.relu_in ? SKL_FUSE_RELU_IN : 0;
            float* b = s.grads.as<float>();
            if (const SkLinear* L = std::get_if<SkLinear>(&layers_[s.idx])) {
                const SkBucket k = SkBucket::of(*L);
                const uint32_t* bits = (s.relu_in && steps_[i - 1].bits_out) ? steps_[i - 1].bits.as<uint32_t>()
                                                                             : nullptr;
                L->backward_into(s.x, g, T, s.saved.get(), gx, k.dU1s(b), k.dU2s(b), k.db(b), st, SKL_BWD_ALL,
                                 fuse, bits);
            } else {
                const DenseLinear& D = std::get<DenseLinear>(layers_[s.idx]);
                D.backward_into(s.x, g, T, gx, b, b + D.d_out() * D.d_in(), st, fuse);
            }
            if (dp) dp->allreduce_async(b, s.grad_count, st);
            g = gx;
        }
    }

    // fp32 gradient bucket of chain step `j` (j-th Linear / SKLinear layer):
    // SKLinear dU1s | db | dU2s (SkBucket), Linear dW [d_out, d_in] | db.
    const DeviceBuffer& grads(size_t j) const { return steps_.at(j).grads; }
    size_t num_steps() const { return steps_.size(); }
    size_t layer_index(size_t j) const { return steps_.at(j).idx; }
    // The input the j-th Linear / SKLinear layer saw in the last forward (device).
    const void* step_input(size_t j) const { return steps_.at(j).x; }

  private:
    struct Step {
        size_t idx = 0;
        bool relu_in = false, relu_out = false, bits_out = false;
        const void* x = nullptr;
        DeviceBuffer y, saved, bits, grads;
        size_t grad_count = 0;
    };

    int64_t d_in_of(const Step& s) const {
        if (const SkLinear* L = std::get_if<SkLinear>(&layers_[s.idx])) return L->d_in();
        return std::get<DenseLinear>(layers_[s.idx]).d_in();
    }
    int64_t d_out_of(const Step& s) const {
        if (const SkLinear* L = std::get_if<SkLinear>(&layers_[s.idx])) return L->d_out();
        return std::get<DenseLinear>(layers_[s.idx]).d_out();
    }
    skl_dtype dtype_of(const Step& s) const {
        if (const SkLinear* L = std::get_if<SkLinear>(&layers_[s.idx])) return L->dtype();
        return std::get<DenseLinear>(layers_[s.idx]).dtype();
    }

    void reserve(int64_t T) {
        if (T <= cap_T_) return;
        check_cuda(cudaDeviceSynchronize(), "sync");  // buffers may still be in use
        const size_t e = elem_bytes(dtype());
        int64_t dmax = 1;
        for (Step& s : steps_) {
            s.y = DeviceBuffer((size_t)(T * d_out_of(s)) * e);
            dmax = std::max(dmax, std::max(d_in_of(s), d_out_of(s)));
            if (const SkLinear* L = std::get_if<SkLinear>(&layers_[s.idx])) {
                s.saved = DeviceBuffer(L->saved_bytes(T));
                if (s.bits_out) s.bits = DeviceBuffer((size_t)T * (size_t)skl_relu_bits_row_words(L->d_out()) * 4);
            }
        }
        gbuf_[0] = DeviceBuffer((size_t)(T * dmax) * e);
        gbuf_[1] = DeviceBuffer((size_t)(T * dmax) * e);
        cap_T_ = T;
    }

    std::vector<Layer> layers_;
    std::vector<Step> steps_;
    DeviceBuffer gbuf_[2];
    int64_t cap_T_ = 0, T_ = -1;
};

}  // namespace skl

#endif  // SKL_CHAIN_HPP_
