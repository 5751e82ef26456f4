// gemm.cuh -- persistent, warp-specialised tcgen05 GEMM for sm_100a.
//
//   D[m, n] = alpha * sum_k A(m, k) * B(n, k)   (+ bias[n])
//
// Used by the SKLinear path for every contraction that does not run inside
// the fused back-to-back kernel (b2b.cuh):
//   * dU1s = inv * Savedᵀ·G     (split-K over tokens, A and B MN-major)
//   * dU2s = inv * Xᵀ·P_S2      (split-K over tokens, A and B MN-major)
//   * the unfused H = X·Acat / Y = H·Bcat (+b) / P / dX chain when the
//     rank R = 2Lk is too large for the on-chip intermediate (R > 512).
//
// Structure (one CTA per SM, or one CTA pair per TPC when kCG == 2):
//   warp 0      TMA producer   (one elected lane)  smem ring of kStages
//   warp 1      MMA issuer     (one elected lane, leader CTA only)
//   warp 2      TMEM allocator (512 columns = 2 accumulator stages)
//   warps 4..7  epilogue       TMEM -> registers -> alpha/bias -> global
// Operands are staged with 128B-swizzled TMA tiles; accumulators live in TMEM
// (double-buffered so the epilogue of tile i overlaps the MMAs of tile i+1).
// With kCG == 2 the pair runs cta_group::2 MMAs (M = 256, each CTA holds its
// 128 rows of A and half of the N rows of B), halving per-SM operand traffic.
//
// Split-K writes raw fp32 partials [split][M][N]; reduce_partials (aux.cu)
// sums them in a fixed order (deterministic) and applies alpha / layout.
#pragma once

#include "sm100.cuh"

namespace skl {

struct GemmArgs {
    int M, N, K;
    int num_m_tiles, num_n_tiles, splits, k_blocks;
    float alpha;
    const float* bias;  // [N] fp32, nullable (direct mode only)
    // direct mode (partial == nullptr): all columns -> out (nullable); columns
    // [out2_c0, out2_c1) are additionally written transposed to out2
    // (out2[(n - out2_c0) * ldo2 + m]) -- the layout the dU kernel reads.
    void* out;
    long long ldo;
    void* out2;
    long long ldo2;
    int out2_c0, out2_c1;
    int out_f32;  // 1: fp32 output, 0: bf16 output
    int round_tf32;  // 1: round direct-mode outputs to TF32 (cvt.rna) -- they feed a TF32 GEMM
    // split-K mode
    float* partial;  // [splits][M][N] fp32
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

template <int kCG, int kKind, bool kAMN, bool kBMN, int kBN, int kStages>
struct GemmCfg {
    static constexpr int kBK = KindTraits<kKind>::kBK;
    static constexpr int kUK = KindTraits<kKind>::kUK;
    static constexpr int kElem = KindTraits<kKind>::kElem;
    static constexpr int kBM = 128;           // rows per CTA
    static constexpr int kNcta = kBN / kCG;   // B rows staged per CTA
    static constexpr int kABytes = kBM * 128; // one 128-B row per M row (K-major) / BK rows x 128 B x 2 blocks
    static constexpr int kBBytes = kNcta * 128;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kTmemCols = 512;
    static constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
    static_assert(kBN % (16 * kCG) == 0 && kBN <= 256 && kBN >= 16 * kCG, "bad BLOCK_N");
    static_assert(!kBMN || kNcta % 64 == 0, "MN-major B needs 64-wide blocks");
    static_assert(!(kKind == 1 && (kAMN || kBMN)), "MN-major TF32 operands are not supported");
    static_assert(2 * kBN <= kTmemCols, "two accumulator stages must fit TMEM");
};

template <int kCG, int kKind, bool kAMN, bool kBMN, int kBN, int kStages>
__global__ void __launch_bounds__(256, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs args) {
    using C = GemmCfg<kCG, kKind, kAMN, kBMN, kBN, kStages>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base_u32 - smem_u32(smem_raw));
    uint8_t* sA = smem;
    uint8_t* sB = smem + kStages * C::kABytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * C::kStageBytes);
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

    const int num_tiles = args.num_m_tiles * args.num_n_tiles * args.splits;
    const int cluster_id = blockIdx.x / kCG;
    const int num_clusters = gridDim.x / kCG;

    auto decode = [&](int t, int& m0, int& n0, int& kb0, int& kb1, int& split) {
        const int mt = t % args.num_m_tiles;
        const int rest = t / args.num_m_tiles;
        const int nt = rest % args.num_n_tiles;
        split = rest / args.num_n_tiles;
        m0 = mt * (C::kBM * kCG);
        n0 = nt * kBN;
        kb0 = (int)(((long long)split * args.k_blocks) / args.splits);
        kb1 = (int)(((long long)(split + 1) * args.k_blocks) / args.splits);
    };

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cluster_id; t < num_tiles; t += num_clusters) {
                int m0, n0, kb0, kb1, split;
                decode(t, m0, n0, kb0, kb1, split);
                const int am = m0 + (int)rank * C::kBM;
                const int bn = n0 + (int)rank * C::kNcta;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* a_dst = sA + stage * C::kABytes;
                    uint8_t* b_dst = sB + stage * C::kBBytes;
                    const int k0 = kb * C::kBK;
                    if (leader)
                        mbar_arrive_expect_tx(&full[stage], C::kStageBytes * kCG);
                    else
                        mbar_arrive_cluster(&full[stage], 0);
                    if constexpr (!kAMN) {
                        tma_load_2d<kCG>(&tmA, &full[stage], a_dst, k0, am);
                    } else {
                        // two 64-wide M blocks, each [BK rows x 128 B]
                        tma_load_2d<kCG>(&tmA, &full[stage], a_dst, am, k0);
                        tma_load_2d<kCG>(&tmA, &full[stage], a_dst + C::kBK * 128, am + 64, k0);
                    }
                    if constexpr (!kBMN) {
                        tma_load_2d<kCG>(&tmB, &full[stage], b_dst, k0, bn);
                    } else {
#pragma unroll
                        for (int j = 0; j < C::kNcta / 64; ++j)
                            tma_load_2d<kCG>(&tmB, &full[stage], b_dst + j * C::kBK * 128, bn + 64 * j, k0);
                    }
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (leader && elect_one()) {
            constexpr uint32_t idesc = make_idesc(kKind, C::kBM * kCG, kBN, kAMN ? 1 : 0, kBMN ? 1 : 0);
            int stage = 0;
            uint32_t phase = 0;
            int iter = 0;
            for (int t = cluster_id; t < num_tiles; t += num_clusters, ++iter) {
                int m0, n0, kb0, kb1, split;
                decode(t, m0, n0, kb0, kb1, split);
                const int acc = iter & 1;
                mbar_wait(&tempty[acc], ((iter >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * kBN;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_addr = smem_u32(sA + stage * C::kABytes);
                    const uint32_t b_addr = smem_u32(sB + stage * C::kBBytes);
#pragma unroll
                    for (int k = 0; k < C::kBK / C::kUK; ++k) {
                        uint64_t ad, bd;
                        if constexpr (!kAMN)
                            ad = make_sdesc(a_addr + k * C::kUK * C::kElem, 0, 1024);
                        else
                            ad = make_sdesc(a_addr + k * C::kUK * 128, C::kBK * 128, 1024);
                        if constexpr (!kBMN)
                            bd = make_sdesc(b_addr + k * C::kUK * C::kElem, 0, 1024);
                        else
                            bd = make_sdesc(b_addr + k * C::kUK * 128, C::kBK * 128, 1024);
                        mma_ss<kCG, kKind>(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
                    }
                    mma_commit<kCG>(&empty[stage]);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
                mma_commit<kCG>(&tfull[acc]);
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue
        const uint32_t q = warp & 3;  // TMEM lane quarter
        const uint32_t lane = lane_id();
        int iter = 0;
        for (int t = cluster_id; t < num_tiles; t += num_clusters, ++iter) {
            int m0, n0, kb0, kb1, split;
            decode(t, m0, n0, kb0, kb1, split);
            const int acc = iter & 1;
            mbar_wait(&tfull[acc], (iter >> 1) & 1);
            tc_fence_after();
            const int row = m0 + (int)rank * C::kBM + (int)(q * 32 + lane);
            const uint32_t t_row = tmem_base + ((q * 32u) << 16) + acc * kBN;
#pragma unroll 1
            for (int c = 0; c < kBN; c += 16) {
                uint32_t r[16];
                tmem_ld16(t_row + c, r);
                tmem_ld_wait();
                const int n = n0 + c;
                if (row >= args.M || n >= args.N) continue;
                float v[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
                if (args.partial) {
                    float* dst = args.partial + ((long long)split * args.M + row) * args.N + n;
                    if (n + 16 <= args.N && (args.N & 3) == 0) {
#pragma unroll
                        for (int j = 0; j < 16; j += 4)
                            *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                    } else {
                        for (int j = 0; j < 16 && n + j < args.N; ++j) dst[j] = v[j];
                    }
                    continue;
                }
                float bv[16];
                load_bias16(args.bias, n, args.N, bv);
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] = fmaf(v[j], args.alpha, bv[j]);
                if (args.round_tf32) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[j] = tf32_rna(v[j]);
                }
                const int nvalid = min(16, args.N - n);
                // columns [out2_c0, out2_c1) also go out transposed: out2[(n - c0) * ldo2 + row]
                if (args.out2 && n + 16 > args.out2_c0 && n < args.out2_c1) {
                    for (int j = 0; j < 16; ++j) {
                        const int nn = n + j;
                        if (nn < args.out2_c0 || nn >= args.out2_c1 || nn >= args.N) continue;
                        const long long o = (long long)(nn - args.out2_c0) * args.ldo2 + row;
                        if (args.out_f32) reinterpret_cast<float*>(args.out2)[o] = v[j];
                        else reinterpret_cast<__nv_bfloat16*>(args.out2)[o] = __float2bfloat16_rn(v[j]);
                    }
                }
                if (args.out) {
                    void* obase = args.out;
                    const long long ld = args.ldo;
                    const int nv = nvalid;
                    if (args.out_f32) {
                        float* dst = reinterpret_cast<float*>(obase) + (long long)row * ld + n;
                        if (nv == 16 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
                            for (int j = 0; j < 16; j += 4)
                                *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                        } else {
                            for (int j = 0; j < nv; ++j) dst[j] = v[j];
                        }
                    } else {
                        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(obase) + (long long)row * ld + n;
                        if (nv == 16 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
                            uint4 w0 = make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                                                  pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
                            uint4 w1 = make_uint4(pack_bf16x2(v[8], v[9]), pack_bf16x2(v[10], v[11]),
                                                  pack_bf16x2(v[12], v[13]), pack_bf16x2(v[14], v[15]));
                            reinterpret_cast<uint4*>(dst)[0] = w0;
                            reinterpret_cast<uint4*>(dst)[1] = w1;
                        } else {
                            for (int j = 0; j < nv; ++j) dst[j] = __float2bfloat16_rn(v[j]);
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(&tempty[acc]);
                else mbar_arrive_cluster(&tempty[acc], 0);
            }
        }
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
