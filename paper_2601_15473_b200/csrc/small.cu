// small.cu -- the small-batch SKLinear path (T <= kSmallT tokens, e.g. the
// reference's CPU correctness case c1: 1024 -> 1024, L = 1, k = 64, T = 64).
//
// At a few dozen tokens the fused tcgen05 kernels run ONE 256-token tile on
// one CTA pair, which must stream the whole parameter set through two SMs
// (1 MB at c1: ~26 us per kernel, traced).  Here the work is spread over the
// parameters instead: every CTA reads a 64 x 32 slice of one weight panel,
// the token dimension stays whole, and the rank-R intermediate is reduced in
// fixed split order (deterministic) in a 32 KB fp32 buffer.  The arithmetic
// is fp32 FMA on the CUDA cores (2 x 33 MFLOP at c1; the tensor cores would
// idle on tiles this small), so every variant -- bf16 and the fp32/TF32 one --
// is at least as accurate as the fused path.
//
//   forward  (nn_layers.cpp:61-76):  part[s] = X[:, Ks] . Acat[Ks, :]   (proj_part, K split 64)
//                                    H = sum_s part[s]; saved = (x.S1)^T   (reduce_rank)
//                                    y = inv . H . Bcat + b (ReLU)        (out_gemm)
//   backward (nn_layers.cpp:78-101): P = G . Bcat^T (proj_part + reduce_rank, P_S2^T saved)
//                                    dX = inv . P . Acat^T (x > 0 mask)    (out_gemm)
//                                    dU1 = inv . Saved^T . G, db = colsum G,
//                                    dU2^T = inv . P_S2^T . X             (grads_small)
//
// Acat / Bcat are never packed: their entries are read from the ABI stacks
// ([L, d, k] S1s / U2s, [L, k, d] U1s / S2s) by index (SURVEY §8b mapping).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "prof.h"
#include "skl_internal.h"

namespace skl {
namespace {

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename E>
__device__ __forceinline__ E from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

struct Stacks {
    const void *S1s, *S2s, *U1s, *U2s;
    int d_in, d_out, k, Lk, R;
};
// Acat(i, r): column r < Lk is S1s[r / k][i][r % k], else U2s[(r - Lk) / k][i][(r - Lk) % k]
template <typename E>
__device__ __forceinline__ float acat(const Stacks& p, int i, int r) {
    const bool s = r < p.Lk;
    const int rr = s ? r : r - p.Lk;
    const E* src = static_cast<const E*>(s ? p.S1s : p.U2s);
    return to_f(src[((long long)(rr / p.k) * p.d_in + i) * p.k + rr % p.k]);
}
// Bcat(r, o): row r < Lk is U1s[r / k][r % k][o], else S2s[(r - Lk) / k][(r - Lk) % k][o]
template <typename E>
__device__ __forceinline__ float bcat(const Stacks& p, int r, int o) {
    const bool u = r < p.Lk;
    const E* src = static_cast<const E*>(u ? p.U1s : p.S2s);
    return to_f(src[(long long)(u ? r : r - p.Lk) * p.d_out + o]);
}

// Programmatic dependent launch, as every other kernel of the library: the next
// kernel's launch and prologue overlap this one's tail; each kernel waits for
// its predecessor before touching data and only then lets its dependent start
// (seven dependent launches per c1 step, each a few microseconds of work).
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, cudaStream_t st, Args... args) {
    static const bool pdl = !(getenv("SKL_PDL") && atoi(getenv("SKL_PDL")) == 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

#define SMALL_LAUNCH(kern, grid, st, ...)                                \
    do {                                                                 \
        const cudaError_t e_ = launch_pdl(kern, grid, st, __VA_ARGS__); \
        if (e_ != cudaSuccess) return e_;                                \
    } while (0)

constexpr int kKS = 64;  // K slice per CTA (proj_part) / K chunk (out_gemm)
constexpr int kNC = 32;  // output columns per CTA

constexpr int kTP = kSmallT + 4, kWP = kNC + 4;  // padded rows: 16-B aligned, bank-spread
// acc[i][j] += sum_c A[c][t0 + i] . W[c][c0 + j]: thread -> 4 tokens x 4 columns
// (t0 = (tid / 8) * 4 covers 128 tokens, c0 = (tid % 8) * 4 covers 32 columns), two
// 16-B shared loads per 16 FMAs.
__device__ __forceinline__ void micro_tile(const float (*A)[kTP], const float (*W)[kWP], float (&acc)[4][4]) {
    const int tid = threadIdx.x, t0 = (tid / 8) * 4, c0 = (tid % 8) * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll 8
    for (int c = 0; c < kKS; ++c) {
        const float4 a = *reinterpret_cast<const float4*>(&A[c][t0]);
        const float4 w = *reinterpret_cast<const float4*>(&W[c][c0]);
        const float av[4] = {a.x, a.y, a.z, a.w}, wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], wv[j], acc[i][j]);
    }
}

// part[s][t][r] = sum_{c in slice s} In[t][c] . W(c, r), r in [r0, r0 + 32), for
// r < r_end.  mode 0: In = X [T][d_in], W = Acat; mode 1: In = G [T][d_out], W = Bcat^T.
template <typename E, int kMode>
__global__ void __launch_bounds__(256) proj_part_kernel(const E* __restrict__ in, Stacks p, int T, int r_end,
                                                        float* __restrict__ part) {
    pdl_enter();
    __shared__ __align__(16) float in_s[kKS][kTP];  // transposed: [k][token]
    __shared__ __align__(16) float w_s[kKS][kWP];
    const int K = kMode == 0 ? p.d_in : p.d_out;
    const int r0 = blockIdx.x * kNC, k0 = blockIdx.y * kKS;
    const int tid = threadIdx.x;
    // all of this thread's global loads are issued before any is stored (latency, not
    // bandwidth, bounds these few-KB tiles)
    float vi[kSmallT * kKS / 256], vw[kKS * kNC / 256];
#pragma unroll
    for (int q = 0; q < kSmallT * kKS / 256; ++q) {
        const int e = tid + 256 * q, t = e / kKS, c = e % kKS;
        vi[q] = (t < T && k0 + c < K) ? to_f(in[(long long)t * K + k0 + c]) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < kKS * kNC / 256; ++q) {
        // mode 0: lanes along r (a term's k columns are contiguous); mode 1: lanes along c (U1s / S2s rows)
        const int e = tid + 256 * q;
        const int c = kMode == 0 ? e / kNC : e % kKS, rl = kMode == 0 ? e % kNC : e / kKS;
        const int kc = k0 + c, r = r0 + rl;
        vw[q] = (kc < K && r < r_end) ? (kMode == 0 ? acat<E>(p, kc, r) : bcat<E>(p, r, kc)) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < kSmallT * kKS / 256; ++q) {
        const int e = tid + 256 * q;
        in_s[e % kKS][e / kKS] = vi[q];
    }
#pragma unroll
    for (int q = 0; q < kKS * kNC / 256; ++q) {
        const int e = tid + 256 * q;
        if (kMode == 0) w_s[e / kNC][e % kNC] = vw[q];
        else w_s[e % kKS][e / kKS] = vw[q];
    }
    __syncthreads();
    float acc[4][4];
    micro_tile(in_s, w_s, acc);
    const int t0 = (tid / 8) * 4, c0 = (tid % 8) * 4;
    float* dst = part + (long long)blockIdx.y * T * p.R;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int t = t0 + i, r = r0 + c0 + j;
            if (t < T && r < r_end) dst[(long long)t * p.R + r] = acc[i][j];
        }
}

// H[t][r] = sum_s part[s][t][r] (split order), r < r_end; columns [c0, c0 + Lk) also
// go to save[(r - c0) * ld_save + t] in the element type (the transposed layout of
// the fused path's saved projection / P_S2).
template <typename E>
__global__ void __launch_bounds__(256) reduce_rank_kernel(const float* __restrict__ part, int S, int T, int R,
                                                          int r_end, float* __restrict__ H, E* __restrict__ save,
                                                          int c0, int Lk, long long ld_save) {
    pdl_enter();
    const long long n = (long long)T * r_end;
    for (long long e = blockIdx.x * 256LL + threadIdx.x; e < n; e += (long long)gridDim.x * 256) {
        const int r = (int)(e % r_end), t = (int)(e / r_end);  // r fastest: coalesced partial loads
        float v = 0.f;
        for (int s0 = 0; s0 < S; s0 += 8) {  // 8 loads in flight, then the ordered adds
            float w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = s0 + i < S ? part[((long long)(s0 + i) * T + t) * R + r] : 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (s0 + i < S) v += w[i];
        }
        if (H) H[(long long)t * R + r] = v;
        if (save && r >= c0 && r < c0 + Lk) save[(long long)(r - c0) * ld_save + t] = from_f<E>(v);
    }
}

// out[t][n] = alpha . sum_r H[t][r] . W(r, n) (+ bias[n]) (ReLU / x-mask), n in [n0, n0 + 32).
// mode 0 (forward): W = Bcat, N = d_out; mode 1 (dX): W(r, i) = Acat(i, r), N = d_in.
template <typename E, int kMode>
__global__ void __launch_bounds__(256) out_gemm_kernel(const float* __restrict__ H, Stacks p, int T, float alpha,
                                                       const E* __restrict__ bias, int relu, const E* __restrict__ mask,
                                                       E* __restrict__ out) {
    pdl_enter();
    __shared__ __align__(16) float h_s[kKS][kTP];  // transposed: [rank][token]
    __shared__ __align__(16) float w_s[kKS][kWP];
    const int N = kMode == 0 ? p.d_out : p.d_in;
    const int n0 = blockIdx.x * kNC;
    const int tid = threadIdx.x;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    for (int r0 = 0; r0 < p.R; r0 += kKS) {
        float vh[kSmallT * kKS / 256], vw[kKS * kNC / 256];
#pragma unroll
        for (int q = 0; q < kSmallT * kKS / 256; ++q) {
            const int e = tid + 256 * q, t = e / kKS, c = e % kKS;
            vh[q] = (t < T && r0 + c < p.R) ? H[(long long)t * p.R + r0 + c] : 0.f;
        }
#pragma unroll
        for (int q = 0; q < kKS * kNC / 256; ++q) {
            // mode 0: lanes along n (Bcat rows); mode 1: lanes along the rank (Acat rows)
            const int e = tid + 256 * q;
            const int c = kMode == 0 ? e / kNC : e % kKS, nl = kMode == 0 ? e % kNC : e / kKS;
            const int r = r0 + c, nn = n0 + nl;
            vw[q] = (r < p.R && nn < N) ? (kMode == 0 ? bcat<E>(p, r, nn) : acat<E>(p, nn, r)) : 0.f;
        }
        __syncthreads();  // the previous chunk's FMAs are done with h_s / w_s
#pragma unroll
        for (int q = 0; q < kSmallT * kKS / 256; ++q) {
            const int e = tid + 256 * q;
            h_s[e % kKS][e / kKS] = vh[q];
        }
#pragma unroll
        for (int q = 0; q < kKS * kNC / 256; ++q) {
            const int e = tid + 256 * q;
            if (kMode == 0) w_s[e / kNC][e % kNC] = vw[q];
            else w_s[e % kKS][e / kKS] = vw[q];
        }
        __syncthreads();
        float part_acc[4][4];
        micro_tile(h_s, w_s, part_acc);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] += part_acc[i][j];
    }
    const int t0 = (tid / 8) * 4, c0 = (tid % 8) * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int n = n0 + c0 + j;
        if (n >= N) continue;
        const float b = bias ? to_f(bias[n]) : 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int t = t0 + i;
            if (t >= T) continue;
            float v = fmaf(acc[i][j], alpha, b);
            if (relu) v = fmaxf(v, 0.f);
            if (mask && !(to_f(mask[(long long)t * N + n]) > 0.f)) v = 0.f;
            out[(long long)t * N + n] = from_f<E>(v);
        }
    }
}

// Parameter gradients over the T tokens (K = T, no split).  blockIdx.x < g1: dU1 /
// db column group (32 d_out columns x 32 rank rows of blockIdx.y); otherwise dU2
// (32 d_in rows x 32 rank columns).  Saved / P_S2 are the transposed [Lk][ld] buffers.
template <typename E>
__global__ void __launch_bounds__(256) grads_small_kernel(const E* __restrict__ G, const E* __restrict__ X,
                                                          const E* __restrict__ saved, const E* __restrict__ p2t,
                                                          long long ld, Stacks p, int T, float alpha, int g1,
                                                          float* __restrict__ dU1, float* __restrict__ dU2,
                                                          float* __restrict__ db) {
    pdl_enter();
    __shared__ __align__(16) float a_s[kSmallT][kWP];  // activation columns: G (dU1) or X (dU2)
    __shared__ __align__(16) float r_s[kSmallT][kWP];  // rank columns: Saved (dU1) or P_S2 (dU2), token-major
    const bool u1 = (int)blockIdx.x < g1;
    const int c0 = (u1 ? blockIdx.x : blockIdx.x - g1) * kNC, j0 = blockIdx.y * kNC;
    const int N = u1 ? p.d_out : p.d_in;
    const E* act = u1 ? G : X;
    const E* rk = u1 ? saved : p2t;
    const int tid = threadIdx.x;
    float va[kSmallT * kNC / 256], vr[kSmallT * kNC / 256];
#pragma unroll
    for (int q = 0; q < kSmallT * kNC / 256; ++q) {
        const int e = tid + 256 * q, t = e / kNC, c = e % kNC;
        va[q] = (t < T && c0 + c < N) ? to_f(act[(long long)t * N + c0 + c]) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < kSmallT * kNC / 256; ++q) {
        const int e = tid + 256 * q, j = e / kSmallT, t = e % kSmallT;  // tokens contiguous in the transposed buffer
        vr[q] = (t < T && j0 + j < p.Lk) ? to_f(rk[(long long)(j0 + j) * ld + t]) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < kSmallT * kNC / 256; ++q) {
        const int e = tid + 256 * q;
        a_s[e / kNC][e % kNC] = va[q];
        r_s[e % kSmallT][e / kSmallT] = vr[q];
    }
    __syncthreads();
    // thread -> (rank row j, 4 activation columns), the activation index fastest
    const int cl = tid % 8 * 4, jl = tid / 8;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int t = 0; t < T; ++t) {
        const float rv = r_s[t][jl];
        const float4 a = *reinterpret_cast<const float4*>(&a_s[t][cl]);
        acc[0] = fmaf(rv, a.x, acc[0]);
        acc[1] = fmaf(rv, a.y, acc[1]);
        acc[2] = fmaf(rv, a.z, acc[2]);
        acc[3] = fmaf(rv, a.w, acc[3]);
    }
    const int j = j0 + jl;
    if (j < p.Lk) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c = c0 + cl + q;
            if (c >= N) continue;
            if (u1) dU1[(long long)j * p.d_out + c] = acc[q] * alpha;                              // [Lk][d_out]
            else dU2[((long long)(j / p.k) * p.d_in + c) * p.k + j % p.k] = acc[q] * alpha;        // [L][d_in][k]
        }
    }
    if (u1 && db && blockIdx.y == 0 && tid < kNC && c0 + tid < N) {  // db = sum_t G (unscaled)
        float s = 0.f;
        for (int t = 0; t < T; ++t) s += a_s[t][tid];
        db[c0 + tid] = s;
    }
}

template <typename E>
cudaError_t small_forward_t(const SmallArgs& a, cudaStream_t st) {
    const Stacks p{a.S1s, a.S2s, a.U1s, a.U2s, a.d_in, a.d_out, a.k, a.Lk, a.R};
    const int S = (a.d_in + kKS - 1) / kKS;
    {
        ProfScope ps_("small_proj", st);
        SMALL_LAUNCH((proj_part_kernel<E, 0>), dim3((a.R + kNC - 1) / kNC, S), st, static_cast<const E*>(a.x), p, a.T,
                                                                              a.R, a.part);
    }
    {
        ProfScope ps_("small_reduce", st);
        const long long n = (long long)a.T * a.R;
        SMALL_LAUNCH(reduce_rank_kernel<E>, dim3((unsigned)((n + 255) / 256)), st, a.part, S, a.T, a.R, a.R, a.H,
                                                                             static_cast<E*>(a.save), 0, a.Lk, a.ld_save);
    }
    ProfScope ps_("small_out", st);
    SMALL_LAUNCH((out_gemm_kernel<E, 0>), dim3((a.d_out + kNC - 1) / kNC), st, a.H, p, a.T, a.alpha, static_cast<const E*>(a.bias),
                                                                    a.relu, nullptr, static_cast<E*>(a.out));
    return cudaGetLastError();
}

template <typename E>
cudaError_t small_backward_t(const SmallArgs& a, cudaStream_t st) {
    const Stacks p{a.S1s, a.S2s, a.U1s, a.U2s, a.d_in, a.d_out, a.k, a.Lk, a.R};
    const E* saved = static_cast<const E*>(a.saved);
    if (a.need_saved) {  // Saved^T = (x . S1)^T: the first Lk rank columns only
        const int S = (a.d_in + kKS - 1) / kKS;
        {
            ProfScope ps_("small_proj", st);
            SMALL_LAUNCH((proj_part_kernel<E, 0>), dim3((a.Lk + kNC - 1) / kNC, S), st, static_cast<const E*>(a.x), p, a.T,
                                                                                   a.Lk, a.part);
        }
        ProfScope ps_("small_reduce", st);
        const long long n = (long long)a.T * a.Lk;
        SMALL_LAUNCH(reduce_rank_kernel<E>, dim3((unsigned)((n + 255) / 256)), st, 
            a.part, S, a.T, a.R, a.Lk, nullptr, static_cast<E*>(a.save), 0, a.Lk, a.ld_save);
        saved = static_cast<const E*>(a.save);
    }
    if (a.data) {  // P = G . Bcat^T (P_S2^T saved), dX = inv . P . Acat^T
        const int S = (a.d_out + kKS - 1) / kKS;
        {
            ProfScope ps_("small_proj", st);
            SMALL_LAUNCH((proj_part_kernel<E, 1>), dim3((a.R + kNC - 1) / kNC, S), st, static_cast<const E*>(a.grad_y), p,
                                                                                  a.T, a.R, a.part);
        }
        {
            ProfScope ps_("small_reduce", st);
            const long long n = (long long)a.T * a.R;
            SMALL_LAUNCH(reduce_rank_kernel<E>, dim3((unsigned)((n + 255) / 256)), st, 
                a.part, S, a.T, a.R, a.R, a.H, static_cast<E*>(a.p2t), a.Lk, a.Lk, a.ld_save);
        }
        if (a.grad_x) {
            ProfScope ps_("small_out", st);
            SMALL_LAUNCH((out_gemm_kernel<E, 1>), dim3((a.d_in + kNC - 1) / kNC), st, 
                a.H, p, a.T, a.alpha, nullptr, 0, static_cast<const E*>(a.mask), static_cast<E*>(a.grad_x));
        }
    }
    const int g1 = a.u1 ? (a.d_out + kNC - 1) / kNC : 0, g2 = a.data ? (a.d_in + kNC - 1) / kNC : 0;
    if (g1 + g2 == 0) return cudaGetLastError();
    ProfScope ps_("small_grads", st);
    SMALL_LAUNCH(grads_small_kernel<E>, dim3(g1 + g2, (a.Lk + kNC - 1) / kNC), st, 
        static_cast<const E*>(a.grad_y), static_cast<const E*>(a.x), saved, static_cast<const E*>(a.p2t), a.ld_save,
        p, a.T, a.alpha, g1, a.grad_U1s, a.grad_U2s, a.u1 ? a.grad_bias : nullptr);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_small_forward(const SmallArgs& a, cudaStream_t st) {
    return a.elem == ELEM_BF16 ? small_forward_t<__nv_bfloat16>(a, st) : small_forward_t<float>(a, st);
}
cudaError_t launch_small_backward(const SmallArgs& a, cudaStream_t st) {
    return a.elem == ELEM_BF16 ? small_backward_t<__nv_bfloat16>(a, st) : small_backward_t<float>(a, st);
}

}  // namespace skl
