// aux.cu -- the non-GEMM kernels of the SKLinear path (all HBM/latency-bound
// integer or byte work, written as plain coalesced CUDA):
//
//   * device sketch generator: counter-based SplitMix64 -> Box-Muller /
//     sign bit, bit-exact integer chain of the reference stream
//     (rng.hpp:13-69, sketch.cpp:34-49, nn_layers.cpp:124-145)
//   * parameter packing: pawX [L,d,k] stacks -> the K-major operand panels the
//     tcgen05 kernels stream when they cannot read the stacks in place
//     (Acat / Bcat and their transposes, one tiled launch), with TF32
//     round-to-nearest for the fp32 variant
// (db and the dU reductions are fused into the du kernel, du.cuh.)
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "skl_internal.h"
#include "prof.h"
#include "sm100.cuh"

namespace skl {
namespace {

// ---------------------------------------------------------------- RNG
// Draw j (0-based) of Splitmix64(seed): state after j+1 increments.
__device__ __forceinline__ uint64_t sm64_draw(uint64_t seed, uint64_t j) {
    uint64_t z = seed + (j + 1) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t derive_seed_dev(uint64_t master, uint64_t index) {
    return sm64_draw(master ^ (0x517cc1b727220a95ULL + index), 0);
}
// rng.hpp:25-27 next_open01, IEEE ops spelled out (no contraction).
__device__ __forceinline__ double open01(uint64_t x) {
    return __dmul_rn(__dadd_rn((double)(x >> 11), 0.5), 0x1.0p-53);
}
// Entry e of GaussianStream(seed) (rng.hpp:45-57): pair p = e/2 uses draws
// 2p and 2p+1; even e -> r cos(theta), odd e -> the cached r sin(theta).
__device__ __forceinline__ double gauss_at(uint64_t seed, uint64_t e) {
    const uint64_t p = e >> 1;
    const double u1 = open01(sm64_draw(seed, 2 * p));
    const double u2 = open01(sm64_draw(seed, 2 * p + 1));
    const double r = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
    const double theta = __dmul_rn(6.283185307179586, u2);  // 2.0 * 3.14159265358979323846
    double s, c;
    sincos(theta, &s, &c);
    return __dmul_rn(r, (e & 1) ? s : c);
}

template <typename T>
__device__ __forceinline__ void store_val(void* out, uint64_t idx, double v);
template <>
__device__ __forceinline__ void store_val<double>(void* out, uint64_t idx, double v) {
    reinterpret_cast<double*>(out)[idx] = v;
}
template <>
__device__ __forceinline__ void store_val<float>(void* out, uint64_t idx, double v) {
    reinterpret_cast<float*>(out)[idx] = __double2float_rn(v);
}
template <>
__device__ __forceinline__ void store_val<__nv_bfloat16>(void* out, uint64_t idx, double v) {
    reinterpret_cast<__nv_bfloat16*>(out)[idx] = __double2bfloat16(v);
}

// realize_sketch(dist, k, d, seed) entry (row, col) of the [k, d] matrix.
__device__ __forceinline__ double sketch_entry(int dist, uint64_t seed, uint64_t d, uint64_t row, uint64_t col,
                                               double scale) {
    const uint64_t e = row * d + col;
    if (dist == 1) return (sm64_draw(seed, e) >> 63) ? scale : -scale;  // rng.hpp:30, sketch.cpp:44-49
    return __dmul_rn(gauss_at(seed, e), scale);                          // sketch.cpp:38-43
}

// All sketches of a layer, directly in the ABI stacks:
//   S1s[i][c][j] = realize(dist,k,d_in, derive_seed(seed,2i+1))[j][c]
//   S2s[i][j][o] = realize(dist,k,d_out,derive_seed(seed,2i))[j][o]
template <typename T>
__global__ void gen_sketches_kernel(int dist, uint64_t layer_seed, int64_t L, int64_t k, int64_t d_in,
                                    int64_t d_out, double scale, void* S1s, void* S2s) {
    const uint64_t n1 = (uint64_t)L * d_in * k;
    const uint64_t n2 = (uint64_t)L * k * d_out;
    for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < n1 + n2;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        if (idx < n1) {
            const uint64_t i = idx / (d_in * k), rem = idx % (d_in * k);
            const uint64_t c = rem / k, j = rem % k;
            const uint64_t seed = derive_seed_dev(layer_seed, 2 * i + 1);
            store_val<T>(S1s, idx, sketch_entry(dist, seed, d_in, j, c, scale));
        } else {
            const uint64_t id2 = idx - n1;
            const uint64_t i = id2 / (k * d_out), rem = id2 % (k * d_out);
            const uint64_t j = rem / d_out, o = rem % d_out;
            const uint64_t seed = derive_seed_dev(layer_seed, 2 * i);
            store_val<T>(S2s, id2, sketch_entry(dist, seed, d_out, j, o, scale));
        }
    }
}

// sk_linear_fresh U (nn_layers.cpp:136-145): stream g_i = GaussianStream(
// derive_seed(seed,1000+i)); u1 [k][d_in] = g[0 .. k*d_in), u2 [d_out][k]
// = g[k*d_in ..).  U2s[i][c][j] = u1[j][c], U1s[i][j][o] = u2[o][j].
template <typename T>
__global__ void init_u_kernel(uint64_t layer_seed, int64_t L, int64_t k, int64_t d_in, int64_t d_out,
                              double std_dev, void* U1s, void* U2s) {
    const uint64_t n2 = (uint64_t)L * d_in * k;
    const uint64_t n1 = (uint64_t)L * k * d_out;
    for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < n1 + n2;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        if (idx < n2) {
            const uint64_t i = idx / (d_in * k), rem = idx % (d_in * k);
            const uint64_t c = rem / k, j = rem % k;
            const uint64_t seed = derive_seed_dev(layer_seed, 1000 + i);
            store_val<T>(U2s, idx, __dmul_rn(gauss_at(seed, j * d_in + c), std_dev));
        } else {
            const uint64_t id1 = idx - n2;
            const uint64_t i = id1 / (k * d_out), rem = id1 % (k * d_out);
            const uint64_t j = rem / d_out, o = rem % d_out;
            const uint64_t seed = derive_seed_dev(layer_seed, 1000 + i);
            store_val<T>(U1s, id1, __dmul_rn(gauss_at(seed, (uint64_t)k * d_in + o * k + j), std_dev));
        }
    }
}

template <typename T>
__global__ void realize_kernel(int dist, int64_t k, int64_t d, uint64_t seed, double scale, int unit_var,
                               int transpose, void* out) {
    const uint64_t n = (uint64_t)k * d;
    for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t row, col;
        if (transpose) { col = idx / k; row = idx % k; }
        else { row = idx / d; col = idx % d; }
        double v;
        if (unit_var) v = gauss_at(seed, row * d + col);  // gaussian_matrix, sketch.cpp:120-125
        else v = sketch_entry(dist, seed, d, row, col, scale);
        store_val<T>(out, idx, v);
    }
}

// ---------------------------------------------------------------- packing
template <typename T>
__device__ __forceinline__ float ld_f(const void* p, uint64_t i) {
    if constexpr (sizeof(T) == 2) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
    else return reinterpret_cast<const float*>(p)[i];
}

inline int grid_for(uint64_t n, int block = 256) {
    uint64_t g = (n + block - 1) / block;
    if (g > 148ull * 16) g = 148ull * 16;
    return (int)(g ? g : 1);
}

}  // namespace

// ---------------------------------------------------------------- launchers
cudaError_t launch_gen_sketches(int dist, uint64_t seed, const SklDims& d, int elem, void* S1s, void* S2s,
                                cudaStream_t st) {
    ProfScope ps_("gen_sketches", st);
    const double scale = 1.0 / sqrt((double)d.k);
    const uint64_t n = (uint64_t)d.L * d.k * (d.d_in + d.d_out);
    if (elem == ELEM_BF16)
        gen_sketches_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(dist, seed, d.L, d.k, d.d_in, d.d_out,
                                                                        scale, S1s, S2s);
    else if (elem == ELEM_F32)
        gen_sketches_kernel<float><<<grid_for(n), 256, 0, st>>>(dist, seed, d.L, d.k, d.d_in, d.d_out, scale, S1s,
                                                                S2s);
    else
        gen_sketches_kernel<double><<<grid_for(n), 256, 0, st>>>(dist, seed, d.L, d.k, d.d_in, d.d_out, scale,
                                                                 S1s, S2s);
    return cudaGetLastError();
}

cudaError_t launch_init_u(uint64_t seed, const SklDims& d, int elem, void* U1s, void* U2s, cudaStream_t st) {
    ProfScope ps_("init_u", st);
    const double std_dev = sqrt(2.0 / (double)(d.d_in + d.d_out));
    const uint64_t n = (uint64_t)d.L * d.k * (d.d_in + d.d_out);
    if (elem == ELEM_BF16)
        init_u_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(seed, d.L, d.k, d.d_in, d.d_out, std_dev, U1s,
                                                                  U2s);
    else if (elem == ELEM_F32)
        init_u_kernel<float><<<grid_for(n), 256, 0, st>>>(seed, d.L, d.k, d.d_in, d.d_out, std_dev, U1s, U2s);
    else
        init_u_kernel<double><<<grid_for(n), 256, 0, st>>>(seed, d.L, d.k, d.d_in, d.d_out, std_dev, U1s, U2s);
    return cudaGetLastError();
}

cudaError_t launch_realize(int dist, int64_t k, int64_t dd, uint64_t seed, int unit_var, int transpose, int elem,
                           void* out, cudaStream_t st) {
    ProfScope ps_("realize", st);
    const double scale = 1.0 / sqrt((double)k);
    const uint64_t n = (uint64_t)k * dd;
    if (elem == ELEM_BF16)
        realize_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(dist, k, dd, seed, scale, unit_var, transpose,
                                                                   out);
    else if (elem == ELEM_F32)
        realize_kernel<float><<<grid_for(n), 256, 0, st>>>(dist, k, dd, seed, scale, unit_var, transpose, out);
    else
        realize_kernel<double><<<grid_for(n), 256, 0, st>>>(dist, k, dd, seed, scale, unit_var, transpose, out);
    return cudaGetLastError();
}

// One launch packs both operand panels in every requested layout: each block
// moves a 32x32 tile (coalesced read of the contiguous stack dimension,
// coalesced write of the natural layout, smem transpose for the other), and
// block 0 also converts the bias to fp32.
template <typename T>
__global__ void __launch_bounds__(256) pack_tiles_kernel(const void* S1s, const void* U2s, const void* U1s,
                                                         const void* S2s, int64_t L, int64_t k64, int64_t d_in64,
                                                         int64_t d_out64, int64_t R_pad64, void* Acat, void* Bcat,
                                                         void* AcatT, void* BcatT, const void* bias, float* bias32) {
    // 32-bit index math: every panel here is far below 2^31 elements, and 64-bit
    // division / modulo (emulated, ~70 instructions each) made this kernel
    // instruction-bound (13 us for 8 MB at c2-TF32).  The per-thread column of
    // a tile is fixed across its 4 rows, so its term / rank split is hoisted.
    __shared__ float tile[32][33];
    const int k = (int)k64, d_in = (int)d_in64, d_out = (int)d_out64, R_pad = (int)R_pad64;
    const int Lk = (int)L * k;
    const int ta_r = R_pad / 32, ta_c = (d_in + 31) / 32;
    const int tb_c = (d_out + 31) / 32;
    const int nA = ta_r * ta_c, nB = ta_r * tb_c;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    // the bias -> fp32 copy is spread over the whole grid: block 0 looping over
    // it alone was the kernel's critical path (c2-TF32: 13.8 us with the SMs
    // active half of that; the loop's dependent load/store pairs serialise)
    if (bias32)
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d_out; i += gridDim.x * blockDim.x)
            bias32[i] = bias ? ld_f<T>(bias, i) : 0.f;
    for (int b = blockIdx.x; b < nA + nB; b += gridDim.x) {
        const bool isA = b < nA;
        int row0, col0, rows, cols;  // natural layout: A = [d_in][R_pad], B = [R_pad][d_out]
        if (isA) { row0 = (b / ta_r) * 32; col0 = (b % ta_r) * 32; rows = d_in; cols = R_pad; }
        else { const int bb = b - nA; row0 = (bb / tb_c) * 32; col0 = (bb % tb_c) * 32; rows = R_pad; cols = d_out; }
        // A: column c = rank index -> (source stack, term, rank-in-term), fixed for this thread
        const int c = col0 + tx;
        const void* asrc = nullptr;
        int64_t abase = 0;
        if (isA && c < 2 * Lk) {
            const int cc = c < Lk ? c : c - Lk;
            asrc = c < Lk ? S1s : U2s;
            abase = (int64_t)(cc / k) * d_in * k + cc % k;  // + r * k
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = row0 + ty + 8 * i;
            float v = 0.f;
            if (r < rows && c < cols) {
                if (isA) {  // (c_in = r, rank = c)
                    if (asrc) v = ld_f<T>(asrc, abase + (int64_t)r * k);
                } else {    // (rank = r, c_out = c)
                    if (r < Lk) v = ld_f<T>(U1s, (int64_t)r * d_out + c);
                    else if (r < 2 * Lk) v = ld_f<T>(S2s, (int64_t)(r - Lk) * d_out + c);
                }
            }
            if constexpr (sizeof(T) == 4) v = dev::tf32_rna(v);
            tile[ty + 8 * i][tx] = v;
            void* nat = isA ? Acat : Bcat;
            if (nat && r < rows && c < cols) {
                if constexpr (sizeof(T) == 2) reinterpret_cast<__nv_bfloat16*>(nat)[(int64_t)r * cols + c] = __float2bfloat16_rn(v);
                else reinterpret_cast<float*>(nat)[(int64_t)r * cols + c] = v;
            }
        }
        void* tr = isA ? AcatT : BcatT;
        if (!tr) continue;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int cT = col0 + ty + 8 * i, rT = row0 + tx;  // transposed: [cols][rows]
            if (rT < rows && cT < cols) {
                const float v = tile[tx][ty + 8 * i];
                if constexpr (sizeof(T) == 2) reinterpret_cast<__nv_bfloat16*>(tr)[(int64_t)cT * rows + rT] = __float2bfloat16_rn(v);
                else reinterpret_cast<float*>(tr)[(int64_t)cT * rows + rT] = v;
            }
        }
    }
}

cudaError_t launch_pack2(const SklDims& d, int elem, const void* S1s, const void* U2s, const void* U1s,
                         const void* S2s, void* Acat, void* Bcat, void* AcatT, void* BcatT, const void* bias,
                         float* bias32, cudaStream_t st) {
    ProfScope ps_("pack", st);
    const int64_t tiles = (d.R_pad / 32) * ((d.d_in + 31) / 32 + (d.d_out + 31) / 32);
    const int grid = (int)std::min<int64_t>(tiles, 148 * 8);
    if (elem == ELEM_BF16)
        pack_tiles_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(S1s, U2s, U1s, S2s, d.L, d.k, d.d_in, d.d_out, d.R_pad,
                                                               Acat, Bcat, AcatT, BcatT, bias, bias32);
    else
        pack_tiles_kernel<float><<<grid, 256, 0, st>>>(S1s, U2s, U1s, S2s, d.L, d.k, d.d_in, d.d_out, d.R_pad, Acat,
                                                       Bcat, AcatT, BcatT, bias, bias32);
    return cudaGetLastError();
}

// out[c][r] = in[r][c] for a [rows][cols] matrix; 32x32 smem tiles (coalesced
// both ways).  Used once per conversion by skl_from_dense (W -> Wᵀ).
template <typename T>
__global__ void __launch_bounds__(256) transpose_kernel(const T* __restrict__ in, T* __restrict__ out, int64_t rows,
                                                        int64_t cols, int64_t ld_out) {
    __shared__ T tile[32][33];
    const int64_t tr = (rows + 31) / 32, tc = (cols + 31) / 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int64_t b = blockIdx.x; b < tr * tc; b += gridDim.x) {
        const int64_t r0 = (b / tc) * 32, c0 = (b % tc) * 32;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t r = r0 + ty + 8 * i, c = c0 + tx;
            if (r < rows && c < cols) tile[ty + 8 * i][tx] = in[r * cols + c];
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t c = c0 + ty + 8 * i, r = r0 + tx;
            if (r < rows && c < cols) out[c * ld_out + r] = tile[tx][ty + 8 * i];
        }
    }
}

cudaError_t launch_transpose(const void* in, int elem, int64_t rows, int64_t cols, void* out, cudaStream_t st,
                             int64_t ld_out) {
    ProfScope ps_("transpose", st);
    const int64_t tiles = ((rows + 31) / 32) * ((cols + 31) / 32);
    const int grid = (int)std::min<int64_t>(tiles, 148 * 8);
    if (ld_out <= 0) ld_out = rows;
    if (elem == ELEM_BF16)
        transpose_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)in, (__nv_bfloat16*)out, rows, cols,
                                                              ld_out);
    else
        transpose_kernel<float><<<grid, 256, 0, st>>>((const float*)in, (float*)out, rows, cols, ld_out);
    return cudaGetLastError();
}

// DenseLinear init (dense_linear_init, nn_layers.cpp:51-59): w = the first
// rows*cols entries of GaussianStream(seed) (row-major) times `scale`.
cudaError_t launch_gaussian_scaled(int64_t rows, int64_t cols, uint64_t seed, double scale, int elem, void* out,
                                   cudaStream_t st) {
    ProfScope ps_("realize", st);
    const uint64_t n = (uint64_t)rows * cols;
    if (elem == ELEM_BF16)
        realize_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(0, rows, cols, seed, scale, 0, 0, out);
    else if (elem == ELEM_F32)
        realize_kernel<float><<<grid_for(n), 256, 0, st>>>(0, rows, cols, seed, scale, 0, 0, out);
    else
        realize_kernel<double><<<grid_for(n), 256, 0, st>>>(0, rows, cols, seed, scale, 0, 0, out);
    return cudaGetLastError();
}

// out[i] = tf32_rna(in[i]) (operands a TF32 GEMM reads; in place allowed), or,
// with to_f32 set, out[i] = float(in[i]) for an element-type vector (bias).
__global__ void __launch_bounds__(256) convert_kernel(const void* in, int in_bf16, float* out, int64_t n, int rna) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float v = in == nullptr ? 0.f
                  : in_bf16     ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(in)[i])
                                : reinterpret_cast<const float*>(in)[i];
        out[i] = rna ? dev::tf32_rna(v) : v;
    }
}

cudaError_t launch_to_f32(const void* in, int elem, int64_t n, float* out, int round_tf32, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    ProfScope ps_("convert", st);
    convert_kernel<<<grid_for((uint64_t)n), 256, 0, st>>>(in, elem == ELEM_BF16, out, n, round_tf32);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- convolution lowering
// SkConv2d (nn_layers.cpp:176-314) = im2col + SkLinear + reshape.  Token t =
// b*oh*ow + oy*ow + ox; lowered feature f = ch*kh*kw + kr*kw + kc (im2col's
// row order, nn_layers.cpp:176-200).  All kernels are gathers (each output
// element written once, fixed summation order): deterministic, no atomics.
template <typename T>
__global__ void __launch_bounds__(256) im2col_tokens_kernel(const T* __restrict__ img, T* __restrict__ cols,
                                                            ConvGeom g) {
    const int64_t d = (int64_t)g.c * g.kh * g.kw;
    const int64_t n = (int64_t)g.B * g.oh * g.ow * d;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i / d, f = i % d;
        const int64_t b = t / ((int64_t)g.oh * g.ow), p = t % ((int64_t)g.oh * g.ow);
        const int oy = (int)(p / g.ow), ox = (int)(p % g.ow);
        const int ch = (int)(f / (g.kh * g.kw)), kr = (int)((f / g.kw) % g.kh), kc = (int)(f % g.kw);
        const int iy = oy * g.stride + kr - g.pad, ix = ox * g.stride + kc - g.pad;
        cols[i] = (iy >= 0 && iy < g.h && ix >= 0 && ix < g.w)
                      ? img[(((int64_t)b * g.c + ch) * g.h + iy) * g.w + ix]
                      : T(0.f);
    }
}

// col2im (nn_layers.cpp:202-224) as a gather: input pixel (b, ch, iy, ix)
// sums the patch entries that read it, in (kr, kc) order.
template <typename T>
__global__ void __launch_bounds__(256) col2im_gather_kernel(const T* __restrict__ cols, T* __restrict__ img,
                                                            ConvGeom g) {
    const int64_t d = (int64_t)g.c * g.kh * g.kw;
    const int64_t n = (int64_t)g.B * g.c * g.h * g.w;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        // one 64-bit split into (image plane, pixel), then 32-bit arithmetic
        const int64_t plane = i / ((int64_t)g.w * g.h);
        const int pix = (int)(i - plane * g.w * g.h);
        const int iy = pix / g.w, ix = pix - iy * g.w;
        const int ch = (int)(plane % g.c);
        const int64_t b = plane / g.c;
        float acc = 0.f;
        for (int kr = 0; kr < g.kh; ++kr) {
            const int ty = iy + g.pad - kr;
            if (ty < 0 || ty % g.stride) continue;
            const int oy = ty / g.stride;
            if (oy >= g.oh) continue;
            for (int kc = 0; kc < g.kw; ++kc) {
                const int tx = ix + g.pad - kc;
                if (tx < 0 || tx % g.stride) continue;
                const int ox = tx / g.stride;
                if (ox >= g.ow) continue;
                const int64_t t = (b * g.oh + oy) * g.ow + ox;
                acc += (float)cols[t * d + ((int64_t)ch * g.kh + kr) * g.kw + kc];
            }
        }
        img[i] = T(acc);
    }
}

// Bandwidth-shaped im2col (round 2; the per-element kernel above spent 430 us
// at a 64-channel 56x56 3x3 layer, B = 32, on 64-bit index arithmetic and
// channel-strided reads; this one 80 us for the 116 MB patch matrix).  One warp per token, lanes along the lowered features (coalesced
// row writes); the (channel plane offset, kr, kc) of every feature comes from
// a shared-memory table built once per block, so the inner loop is a bounds
// test, one L2 load and one store.  Same values, same layout.
template <typename T>
__global__ void __launch_bounds__(256) im2col_warp_kernel(const T* __restrict__ img, T* __restrict__ cols,
                                                          ConvGeom g) {
    extern __shared__ int im_tab[];  // [d] channel plane offsets, then [d] (kr << 16 | kc)
    const int d = g.c * g.kh * g.kw, khw = g.kh * g.kw;
    int* ch_off = im_tab;
    int* rc = im_tab + d;
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
        const int ch = f / khw, r = f % khw;
        ch_off[f] = ch * g.h * g.w;
        rc[f] = ((r / g.kw) << 16) | (r % g.kw);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warps = blockDim.x >> 5;
    const long long tokens = (long long)g.B * g.oh * g.ow;
    for (long long t = (long long)blockIdx.x * warps + (threadIdx.x >> 5); t < tokens; t += (long long)gridDim.x * warps) {
        const int b = (int)(t / ((long long)g.oh * g.ow)), p = (int)(t % ((long long)g.oh * g.ow));
        const int y0 = (p / g.ow) * g.stride - g.pad, x0 = (p % g.ow) * g.stride - g.pad;
        const T* src = img + (long long)b * g.c * g.h * g.w;
        T* dst = cols + t * d;
        for (int f = lane; f < d; f += 32) {
            const int iy = y0 + (rc[f] >> 16), ix = x0 + (rc[f] & 0xFFFF);
            dst[f] = (iy >= 0 && iy < g.h && ix >= 0 && ix < g.w) ? src[ch_off[f] + iy * g.w + ix] : T(0.f);
        }
    }
}

// col2im, channel-parallel: a block owns 32 channels x 32 pixels of one image
// row.  Lanes run along the channels, so each patch-matrix load of a warp
// covers one token's 32 x (kh x kw) contiguous entries (the neighbours' (kr,
// kc) entries of the same sectors are read by the neighbouring pixels of the
// block, from L1); the sums (in (kr, kc) order, as the per-pixel gather above:
// bitwise the same) are transposed through shared memory so the image row is
// written 64 contiguous bytes per warp store.
template <typename T>
__global__ void __launch_bounds__(256) col2im_chan_kernel(const T* __restrict__ cols, T* __restrict__ img,
                                                          ConvGeom g) {
    __shared__ float tile[32][33];  // [channel][pixel]
    const int khw = g.kh * g.kw;
    const long long d = (long long)g.c * khw;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nxb = (g.w + 31) / 32, ncb = (g.c + 31) / 32;
    const long long nblk = (long long)g.B * g.h * nxb * ncb;
    for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const int cb = (int)(blk % ncb), xb = (int)((blk / ncb) % nxb);
        const int iy = (int)((blk / ((long long)ncb * nxb)) % g.h);
        const long long b = blk / ((long long)ncb * nxb * g.h);
        const int ch = cb * 32 + lane, x0 = xb * 32;
        __syncthreads();  // the previous tile's stores have read `tile`
#pragma unroll 1
        for (int j = 0; j < 4; ++j) {
            const int px = warp + 8 * j, ix = x0 + px;
            float acc = 0.f;
            if (ch < g.c && ix < g.w) {
                const T* base = cols + (long long)ch * khw;
                for (int kr = 0; kr < g.kh; ++kr) {
                    const int ty = iy + g.pad - kr;
                    if (ty < 0 || ty % g.stride) continue;
                    const int oy = ty / g.stride;
                    if (oy >= g.oh) continue;
                    for (int kc = 0; kc < g.kw; ++kc) {
                        const int tx = ix + g.pad - kc;
                        if (tx < 0 || tx % g.stride) continue;
                        const int ox = tx / g.stride;
                        if (ox >= g.ow) continue;
                        acc += (float)base[((b * g.oh + oy) * g.ow + ox) * d + kr * g.kw + kc];
                    }
                }
            }
            tile[lane][px] = acc;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // warp -> channel rows, lanes along the pixels
            const int cl = warp + 8 * j, c = cb * 32 + cl, ix = x0 + lane;
            if (c < g.c && ix < g.w) img[((b * g.c + c) * g.h + iy) * g.w + ix] = T(tile[cl][lane]);
        }
    }
}

// [B*P, C] token rows <-> [B, C, P] planes (P = oh*ow): 32x32 smem tiles per image.
template <typename T>
__global__ void __launch_bounds__(256) tokens_planes_kernel(const T* __restrict__ in, T* __restrict__ out, int64_t B,
                                                            int64_t P, int64_t C, int to_planes) {
    __shared__ float tile[32][33];
    const int64_t tp = (P + 31) / 32, tc = (C + 31) / 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int64_t blk = blockIdx.x; blk < B * tp * tc; blk += gridDim.x) {
        const int64_t b = blk / (tp * tc), r = blk % (tp * tc);
        const int64_t p0 = (r / tc) * 32, c0 = (r % tc) * 32;
        __syncthreads();
        if (to_planes) {  // in [b*P + p][c] -> out [b][c][p]
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int64_t p = p0 + ty + 8 * i, c = c0 + tx;
                if (p < P && c < C) tile[ty + 8 * i][tx] = (float)in[(b * P + p) * C + c];
            }
            __syncthreads();
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int64_t c = c0 + ty + 8 * i, p = p0 + tx;
                if (p < P && c < C) out[(b * C + c) * P + p] = T(tile[tx][ty + 8 * i]);
            }
        } else {          // in [b][c][p] -> out [b*P + p][c]
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int64_t c = c0 + ty + 8 * i, p = p0 + tx;
                if (p < P && c < C) tile[tx][ty + 8 * i] = (float)in[(b * C + c) * P + p];
            }
            __syncthreads();
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int64_t p = p0 + ty + 8 * i, c = c0 + tx;
                if (p < P && c < C) out[(b * P + p) * C + c] = T(tile[ty + 8 * i][tx]);
            }
        }
    }
}

cudaError_t launch_im2col(const void* img, int elem, const ConvGeom& g, void* cols, cudaStream_t st) {
    ProfScope ps_("im2col", st);
    const uint64_t n = (uint64_t)g.B * g.oh * g.ow * g.c * g.kh * g.kw;
    const int d = g.c * g.kh * g.kw;
    const size_t tab = (size_t)d * 8;
    if (tab <= 48 * 1024 && (uint64_t)g.c * g.h * g.w < (1ull << 31)) {  // table in static-limit smem, 32-bit offsets
        const uint64_t tokens = (uint64_t)g.B * g.oh * g.ow;
        const int grid = (int)std::min<uint64_t>((tokens + 7) / 8, 148 * 16);
        if (elem == ELEM_BF16)
            im2col_warp_kernel<__nv_bfloat16><<<grid, 256, tab, st>>>((const __nv_bfloat16*)img, (__nv_bfloat16*)cols, g);
        else
            im2col_warp_kernel<float><<<grid, 256, tab, st>>>((const float*)img, (float*)cols, g);
        return cudaGetLastError();
    }
    if (elem == ELEM_BF16)
        im2col_tokens_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>((const __nv_bfloat16*)img, (__nv_bfloat16*)cols, g);
    else
        im2col_tokens_kernel<float><<<grid_for(n), 256, 0, st>>>((const float*)img, (float*)cols, g);
    return cudaGetLastError();
}

cudaError_t launch_col2im(const void* cols, int elem, const ConvGeom& g, void* img, cudaStream_t st) {
    ProfScope ps_("col2im", st);
    const uint64_t n = (uint64_t)g.B * g.c * g.h * g.w;
    if (g.c >= 16) {  // channel-parallel tiles (fewer channels would leave most lanes idle)
        const uint64_t blocks = (uint64_t)g.B * g.h * ((g.w + 31) / 32) * ((g.c + 31) / 32);
        const int grid = (int)std::min<uint64_t>(blocks, 148 * 16);
        if (elem == ELEM_BF16)
            col2im_chan_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)cols, (__nv_bfloat16*)img, g);
        else
            col2im_chan_kernel<float><<<grid, 256, 0, st>>>((const float*)cols, (float*)img, g);
        return cudaGetLastError();
    }
    if (elem == ELEM_BF16)
        col2im_gather_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>((const __nv_bfloat16*)cols, (__nv_bfloat16*)img, g);
    else
        col2im_gather_kernel<float><<<grid_for(n), 256, 0, st>>>((const float*)cols, (float*)img, g);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- row padding
// dst[b][r][c] = (r < R && c < C) ? src[b][r][c] : 0 for a [B][R2][C2] dst:
// pads (R2 >= R, C2 >= C) or crops (R2 <= R, C2 <= C) the two inner dims of a
// row-major stack.  Shapes whose rows are not 16-byte multiples go through the
// TMA-fed kernels on zero-padded copies (skl.cu, padded dispatch); zero rank or
// feature columns contribute nothing to any product, so the cropped results
// equal the unpadded computation.  Elements move as raw bits (2 or 4 bytes).
template <typename T>
__global__ void __launch_bounds__(256) repad_kernel(const T* __restrict__ src, int64_t R, int64_t C,
                                                    T* __restrict__ dst, int64_t R2, int64_t C2, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i % C2, rest = i / C2;
        const int64_t r = rest % R2, b = rest / R2;
        dst[i] = (r < R && c < C) ? src[(b * R + r) * C + c] : T(0);
    }
}

cudaError_t launch_repad(const void* src, int elem_bytes, int64_t B, int64_t R, int64_t C, void* dst, int64_t R2,
                         int64_t C2, cudaStream_t st) {
    const uint64_t n = (uint64_t)B * R2 * C2;
    if (n == 0) return cudaSuccess;
    ProfScope ps_("repad", st);
    if (elem_bytes == 2)
        repad_kernel<uint16_t><<<grid_for(n), 256, 0, st>>>((const uint16_t*)src, R, C, (uint16_t*)dst, R2, C2, n);
    else
        repad_kernel<uint32_t><<<grid_for(n), 256, 0, st>>>((const uint32_t*)src, R, C, (uint32_t*)dst, R2, C2, n);
    return cudaGetLastError();
}

cudaError_t launch_tokens_planes(const void* in, int elem, int64_t B, int64_t P, int64_t C, void* out, int to_planes,
                                 cudaStream_t st) {
    ProfScope ps_(to_planes ? "to_planes" : "to_tokens", st);
    const int64_t blocks = B * ((P + 31) / 32) * ((C + 31) / 32);
    const int grid = (int)std::min<int64_t>(blocks, 148 * 8);
    if (elem == ELEM_BF16)
        tokens_planes_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)in, (__nv_bfloat16*)out, B, P, C,
                                                                  to_planes);
    else
        tokens_planes_kernel<float><<<grid, 256, 0, st>>>((const float*)in, (float*)out, B, P, C, to_planes);
    return cudaGetLastError();
}

}  // namespace skl
