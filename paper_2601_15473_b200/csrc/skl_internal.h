// skl_internal.h -- shared declarations between the C-ABI dispatch (skl.cu)
// and the kernel translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace skl {

enum { ELEM_F64 = 0, ELEM_F32 = 1, ELEM_BF16 = 2 };

struct SklDims {
    int64_t d_in, d_out, L, k;
    int64_t Lk, R, R_pad;  // R = 2Lk, R_pad = R rounded up to 64
};

cudaError_t launch_gen_sketches(int dist, uint64_t seed, const SklDims& d, int elem, void* S1s, void* S2s,
                                cudaStream_t st);
cudaError_t launch_init_u(uint64_t seed, const SklDims& d, int elem, void* U1s, void* U2s, cudaStream_t st);
cudaError_t launch_realize(int dist, int64_t k, int64_t dd, uint64_t seed, int unit_var, int transpose, int elem,
                           void* out, cudaStream_t st);

cudaError_t launch_pack2(const SklDims& d, int elem, const void* S1s, const void* U2s, const void* U1s,
                         const void* S2s, void* Acat, void* Bcat, void* AcatT, void* BcatT, const void* bias,
                         float* bias32, cudaStream_t st);
// Convolution geometry of one SkConv2d call (ConvShape, layers.hpp:96-107).
struct ConvGeom {
    int B, c, h, w, kh, kw, stride, pad, oh, ow;
};
cudaError_t launch_im2col(const void* img, int elem, const ConvGeom& g, void* cols, cudaStream_t st);
cudaError_t launch_col2im(const void* cols, int elem, const ConvGeom& g, void* img, cudaStream_t st);
cudaError_t launch_tokens_planes(const void* in, int elem, int64_t B, int64_t P, int64_t C, void* out, int to_planes,
                                 cudaStream_t st);
// [B][R][C] -> [B][R2][C2], zero fill outside the source (pads or crops the inner dims).
cudaError_t launch_repad(const void* src, int elem_bytes, int64_t B, int64_t R, int64_t C, void* dst, int64_t R2,
                         int64_t C2, cudaStream_t st);
// out[c * ld_out + r] = in[r * cols + c]; ld_out <= 0 means rows.
cudaError_t launch_transpose(const void* in, int elem, int64_t rows, int64_t cols, void* out, cudaStream_t st,
                             int64_t ld_out = 0);
cudaError_t launch_gaussian_scaled(int64_t rows, int64_t cols, uint64_t seed, double scale, int elem, void* out,
                                   cudaStream_t st);
// fp32 copy of an element-type vector (NULL in -> zeros), optionally TF32-rounded (cvt.rna).
cudaError_t launch_to_f32(const void* in, int elem, int64_t n, float* out, int round_tf32, cudaStream_t st);
// Small-batch path (small.cu): T <= kSmallT tokens, fp32 FMA over parameter slices.
constexpr int kSmallT = 128;
struct SmallArgs {
    int elem, T, d_in, d_out, k, Lk, R;
    float alpha;
    const void *x, *grad_y, *S1s, *S2s, *U1s, *U2s, *bias, *mask;
    int relu;
    void *out, *grad_x;
    void* save;         // forward: saved projection (nullable); backward: recomputed Saved^T target
    const void* saved;  // backward: the caller's saved projection (when !need_saved)
    void* p2t;          // backward: P_S2^T [Lk][ld_save]
    long long ld_save;
    float *part, *H;    // workspace: [splits][T][R] partials, [T][R] rank intermediate
    int need_saved, data, u1;
    float *grad_U1s, *grad_U2s, *grad_bias;
};
cudaError_t launch_small_forward(const SmallArgs& a, cudaStream_t st);
cudaError_t launch_small_backward(const SmallArgs& a, cudaStream_t st);
}  // namespace skl
