// gemm.cuh -- persistent, warp-specialised tcgen05 GEMM for sm_100a.
//
//   D[m, n] = alpha * sum_k A(m, k) * B(n, k)   (+ bias[n])
//
// Used by the SKLinear path for the contractions that do not run inside the
// fused back-to-back kernel (b2b.cuh): the unfused H = x·Acat / y = H·Bcat
// (+b) / P = G·Bcatᵀ / dX = P·Acatᵀ chain when the rank R = 2Lk is too large
// for the on-chip intermediate (bf16 R > 512, TF32 R > 256), and the saved-
// projection recompute.  Both operands are K-major.
//
// Structure (one CTA pair per two SMs, cta_group::2):
//   warp 0      TMA producer   (one elected lane)  smem ring of kStages
//   warp 1      MMA issuer     (one elected lane, leader CTA only)
//   warp 2      TMEM allocator (512 columns = 2 accumulator stages)
//   warps 4..7  epilogue       TMEM -> registers -> alpha/bias -> swizzled
//                              smem -> TMA bulk store (coalesced, async)
// The pair runs M = 256 (each CTA keeps its 128 rows of A and half of the
// kBN rows of B), so per SM one 128x256x16 MMA reads 8 KB of smem per 64
// cycles -- exactly the 128 B/clk smem port -- where a single CTA would need
// 12 KB and be smem-bound at 2/3 of the tensor peak.  Accumulators are
// double-buffered in TMEM so the epilogue of tile i overlaps tile i+1.
#pragma once

#include "sm100.cuh"

namespace skl {

struct GemmArgs {
    int M, N, K;
    int l2hint;  // bit 1: B loads evict_last
    int num_m_tiles, num_n_tiles, k_blocks;
    float alpha;
    const float* bias;  // [N] fp32, nullable
    // all columns -> out through the tmOut tensor map (nullable); columns
    // [out2_c0, out2_c1) are additionally written transposed to out2
    // (out2[(n - out2_c0) * ldo2 + m]) -- the layout the dU kernel reads.
    void* out;
    long long ldo;
    void* out2;
    long long ldo2;
    int out2_c0, out2_c1;
    int out_f32;     // 1: fp32 output, 0: bf16 output
    int round_tf32;  // 1: round outputs to TF32 (cvt.rna) -- they feed a TF32 GEMM
    int relu;        // out = max(0, ·)            (fused Relu::forward)
    const void* mask;  // out *= (mask > 0), mask [M][ld_mask] in the output type (fused Relu::backward)
    long long ld_mask;
};

namespace dev {

template <int kKind>
struct KindTraits;
template <>
struct KindTraits<0> {  // bf16
    static constexpr int kElem = 2, kBK = 64, kUK = 16;
};
template <>
struct KindTraits<1> {  // tf32 (fp32 words)
    static constexpr int kElem = 4, kBK = 32, kUK = 8;
};

template <int kCG, int kKind, int kBN, int kStages>
struct GemmCfg {
    static constexpr int kBK = KindTraits<kKind>::kBK;
    static constexpr int kUK = KindTraits<kKind>::kUK;
    static constexpr int kElem = KindTraits<kKind>::kElem;
    static constexpr int kBM = 128;           // rows per CTA
    static constexpr int kNcta = kBN / kCG;   // B rows staged per CTA
    static constexpr int kABytes = kBM * 128; // one 128-B row (one k-block) per M row
    static constexpr int kBBytes = kNcta * 128;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kTmemCols = 512;
    static constexpr int kOutBytes = 16384;   // one [128 rows x 128 B] output box
    static constexpr int kSmem = kStages * kStageBytes + 2 * kOutBytes + 1024 /*align*/ + 256 /*barriers*/;
    static_assert(kBN % (16 * kCG) == 0 && kBN <= 256 && kBN >= 16 * kCG, "bad BLOCK_N");
    static_assert(kBN % 64 == 0, "epilogue stores 64-column (bf16) / 32-column (fp32) boxes");
    static_assert(2 * kBN <= kTmemCols, "two accumulator stages must fit TMEM");
    static_assert(kSmem <= 232448, "exceeds the 227 KB dynamic shared memory limit");
};

template <int kCG, int kKind, int kBN, int kStages>
__global__ void __launch_bounds__(256, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmOut, GemmArgs args) {
    using C = GemmCfg<kCG, kKind, kBN, kStages>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base_u32 - smem_u32(smem_raw));
    uint8_t* sA = smem;
    uint8_t* sB = smem + kStages * C::kABytes;
    uint8_t* sOut = smem + kStages * C::kStageBytes;  // 2 x 16 KB output staging
    uint64_t* bars = reinterpret_cast<uint64_t*>(sOut + 2 * C::kOutBytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages;
    uint64_t* tfull = bars + 2 * kStages;
    uint64_t* tempty = bars + 2 * kStages + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);

    const uint32_t warp = warp_id();
    const uint32_t rank = kCG == 2 ? cluster_ctarank() : 0;
    const bool leader = rank == 0;

    if (warp == 0 && elect_one()) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
        if (args.out) prefetch_tmap(&tmOut);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], kCG);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4 * kCG);
        }
        fence_barrier_init();
    }
    if (warp == 2) {
        tmem_alloc<kCG>(tmem_slot, C::kTmemCols);
        tmem_relinquish<kCG>();
    }
    tc_fence_before();
    if constexpr (kCG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();
    pdl_launch_dependents();  // after the wait: a dependent starts only once our predecessor completed

    const int num_tiles = args.num_m_tiles * args.num_n_tiles;
    const int cluster_id = blockIdx.x / kCG;
    const int num_clusters = gridDim.x / kCG;

    // n fastest: the clusters working at the same time share one A row panel
    // (activations, large -- read from HBM once) and sweep the B panel
    // (parameters, a few MB -- L2-resident).  m-fastest order re-read A once
    // per N tile (ncu: 542 MB read vs 73 MB algorithmic for the c2 TF32 y GEMM).
    auto decode = [&](int t, int& m0, int& n0) {
        m0 = (t / args.num_n_tiles) * (C::kBM * kCG);
        n0 = (t % args.num_n_tiles) * kBN;
    };

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            // B (the weight panel) is re-read by every m tile: evict_last.  A keeps the
            // default: n-fastest order re-reads each activation panel from L2.
            const uint64_t pol_a = l2_evict_normal();
            const uint64_t pol_b = (args.l2hint & 2) ? l2_evict_last() : pol_a;
            for (int t = cluster_id; t < num_tiles; t += num_clusters) {
                int m0, n0;
                decode(t, m0, n0);
                const int am = m0 + (int)rank * C::kBM;
                const int bn = n0 + (int)rank * C::kNcta;
                for (int kb = 0; kb < args.k_blocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    const int k0 = kb * C::kBK;
                    if (leader)
                        mbar_arrive_expect_tx(&full[stage], C::kStageBytes * kCG);
                    else
                        mbar_arrive_cluster(&full[stage], 0);
                    tma_load_2d_hint<kCG>(&tmA, &full[stage], sA + stage * C::kABytes, k0, am, pol_a);
                    tma_load_2d_hint<kCG>(&tmB, &full[stage], sB + stage * C::kBBytes, k0, bn, pol_b);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (leader && elect_one()) {
            constexpr uint32_t idesc = make_idesc(kKind, C::kBM * kCG, kBN, 0, 0);
            int stage = 0;
            uint32_t phase = 0;
            int iter = 0;
            for (int t = cluster_id; t < num_tiles; t += num_clusters, ++iter) {
                const int acc = iter & 1;
                mbar_wait(&tempty[acc], ((iter >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * kBN;
                for (int kb = 0; kb < args.k_blocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_addr = smem_u32(sA + stage * C::kABytes);
                    const uint32_t b_addr = smem_u32(sB + stage * C::kBBytes);
#pragma unroll
                    for (int k = 0; k < C::kBK / C::kUK; ++k)
                        mma_ss<kCG, kKind>(d_tmem, make_sdesc(a_addr + k * C::kUK * C::kElem, 0, 1024),
                                           make_sdesc(b_addr + k * C::kUK * C::kElem, 0, 1024), idesc,
                                           (kb > 0 || k > 0) ? 1u : 0u);
                    mma_commit<kCG>(&empty[stage]);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
                mma_commit<kCG>(&tfull[acc]);
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue
        // Thread = one accumulator row (TMEM lane).  Each 128-B column slice
        // (64 bf16 / 32 fp32 columns) goes TMEM -> registers -> alpha/bias
        // (/TF32 rounding) -> 128B-swizzled smem box -> one TMA bulk store
        // (two boxes in flight).
        const uint32_t q = warp & 3;  // TMEM lane quarter
        const uint32_t lane = lane_id();
        const uint32_t srow = q * 32 + lane;
        const bool issuer = (q == 0 && lane == 0);
        const int ecols = args.out_f32 ? 32 : 64;
        int iter = 0, nbox = 0;
        for (int t = cluster_id; t < num_tiles; t += num_clusters, ++iter) {
            int m0, n0;
            decode(t, m0, n0);
            const int acc = iter & 1;
            mbar_wait(&tfull[acc], (iter >> 1) & 1);
            tc_fence_after();
            const int row0 = m0 + (int)rank * C::kBM;
            const int row = row0 + (int)srow;
            const uint32_t t_row = tmem_base + ((q * 32u) << 16) + acc * kBN;
#pragma unroll 1
            for (int c = 0; c < kBN; c += ecols) {
                const int n = n0 + c;
                if (n >= args.N) break;  // uniform across the CTA
                uint32_t ra[32], rb[32];
                tmem_ld32(t_row + c, ra);
                if (!args.out_f32) tmem_ld32(t_row + c + 32, rb);
                tmem_ld_wait();
                float v[64];
#pragma unroll
                for (int j = 0; j < 64; ++j) {
                    if (j >= ecols) break;
                    const uint32_t bits = j < 32 ? ra[j] : rb[j - 32];
                    const float b = (args.bias != nullptr && n + j < args.N) ? __ldg(args.bias + n + j) : 0.f;
                    v[j] = fmaf(__uint_as_float(bits), args.alpha, b);
                    if (args.relu) v[j] = fmaxf(v[j], 0.f);
                    if (args.round_tf32) v[j] = tf32_rna(v[j]);
                }
                if (args.mask && row < args.M) {
                    // 128 B of the ReLU mask row (the layer input) covering these columns
                    const uint8_t* mrow = reinterpret_cast<const uint8_t*>(args.mask) +
                                          ((long long)row * args.ld_mask + n) * (args.out_f32 ? 4 : 2);
                    if (args.out_f32) {
#pragma unroll
                        for (int ch = 0; ch < 8; ++ch) {
                            if (n + 4 * ch >= args.N) break;
                            const uint4 mk = __ldg(reinterpret_cast<const uint4*>(mrow + ch * 16));
                            const uint32_t m[4] = {mk.x, mk.y, mk.z, mk.w};
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                if (__uint_as_float(m[i]) <= 0.f) v[4 * ch + i] = 0.f;
                        }
                    } else {
#pragma unroll
                        for (int ch = 0; ch < 8; ++ch) {
                            if (n + 8 * ch >= args.N) break;
                            const uint4 mk = __ldg(reinterpret_cast<const uint4*>(mrow + ch * 16));
                            const uint32_t m[4] = {mk.x, mk.y, mk.z, mk.w};
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&m[i]));
                                if (f.x <= 0.f) v[8 * ch + 2 * i] = 0.f;
                                if (f.y <= 0.f) v[8 * ch + 2 * i + 1] = 0.f;
                            }
                        }
                    }
                }
                // columns [out2_c0, out2_c1) also go out transposed: out2[(n - c0) * ldo2 + row]
                if (args.out2 && row < args.M && n + ecols > args.out2_c0 && n < args.out2_c1) {
#pragma unroll
                    for (int j = 0; j < 64; ++j) {
                        const int nn = n + j;
                        if (j >= ecols || nn < args.out2_c0 || nn >= args.out2_c1 || nn >= args.N) continue;
                        const long long o = (long long)(nn - args.out2_c0) * args.ldo2 + row;
                        if (args.out_f32) reinterpret_cast<float*>(args.out2)[o] = v[j];
                        else reinterpret_cast<__nv_bfloat16*>(args.out2)[o] = __float2bfloat16_rn(v[j]);
                    }
                }
                if (!args.out) continue;
                uint8_t* buf = sOut + (nbox & 1) * C::kOutBytes;
                if (issuer) bulk_wait_read<1>();  // the store that last used `buf` has read it
                named_bar_sync(1, 128);
                const uint32_t row_addr = smem_u32(buf) + srow * 128;
#pragma unroll
                for (int ch = 0; ch < 8; ++ch) {
                    uint32_t w[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        w[i] = args.out_f32 ? __float_as_uint(v[4 * ch + i])
                                            : pack_bf16x2(v[8 * ch + 2 * i], v[8 * ch + 2 * i + 1]);
                    st_shared_v4(row_addr + ((uint32_t)(ch ^ (srow & 7)) << 4), w[0], w[1], w[2], w[3]);
                }
                fence_proxy_async_smem();
                named_bar_sync(1, 128);
                if (issuer) {
                    tma_store_2d(&tmOut, buf, n, row0);  // rows >= M / cols >= N are clipped
                    bulk_commit();
                }
                ++nbox;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(&tempty[acc]);
                else mbar_arrive_cluster(&tempty[acc], 0);
            }
        }
        if (issuer) bulk_wait<0>();
    }

    tc_fence_before();
    if constexpr (kCG == 2) cluster_sync(); else __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<kCG>(tmem_base, C::kTmemCols);
    }
}

}  // namespace dev
}  // namespace skl
