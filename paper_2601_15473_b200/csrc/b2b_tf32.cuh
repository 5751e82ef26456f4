// b2b_tf32.cuh -- fused back-to-back kernel for the TF32 variant with a wide
// rank, 256 < R_pad <= 512 (c2-TF32: R = 512).
//
// Same contraction as b2b.cuh (forward H = x·Acat, y = inv·H·Bcat + b;
// backward P = G·Bcatᵀ, dX = inv·P·Acatᵀ), but the fp32 (TF32) intermediate
// [256 tokens x R] of a CTA pair no longer fits TMEM next to the GEMM2
// accumulators (one fp32 word per column: R = 512 is all 512 columns).  So H
// is split across the two on-chip memories and still never touches HBM:
//
//   H columns [0, 256)      stay in TMEM (cvt.rna in place) -> GEMM2 "TS" MMAs
//   H columns [256, R_pad)  go to SMEM as K-major SW128 tiles -> GEMM2 "SS" MMAs
//
// both accumulating into the same TMEM slot.  The 128 KB SMEM home of the
// upper half doubles as the GEMM1 operand ring (ring A: 4 x 32 KB stages)
// while GEMM1 runs -- the upper half of the previous tile is dead by then --
// and GEMM2 streams its B2 tiles through a separate 2-stage ring (ring B)
// with its own producer warp.  Lifetimes:
//   GEMM1(t) chunk 0 -> TMEM [0,256), chunk 1 -> TMEM [256,512) (GEMM2 slots)
//   convert: chunk 0 in place; chunk 1 -> SMEM upper half, slots released
//   GEMM2(t): TS over [0,256) + SS over SMEM; last MMA commits hhi_free
//   producer A waits hhi_free before loading GEMM1(t+1) into that SMEM.
//
// Warp roles: 0 producer A (GEMM1), 1 MMA issuer, 2 TMEM allocator,
// 3 producer B (GEMM2), 4..11 two epilogue warpgroups.  CTA pairs
// (cta_group::2, M = 256 tokens); operands are the packed K-major panels.
#pragma once

#include "b2b.cuh"

namespace skl {
namespace dev {

// kSP (single pass): GEMM1 stages carry the A tile and BOTH B1 chunks, so A is
// read once -- the backward's A is G (fp32, K1 = d_out), where a second pass
// would stream it from HBM twice.  The forward (K1 = d_in) keeps two passes and
// deeper rings.
template <bool kSP>
struct B2BT32Cfg {
    static constexpr int kBK = 32;                      // fp32 per 128-B k-block
    static constexpr int kStageA = kSP ? 48 * 1024 : 32 * 1024;  // X/G k-block + B1 chunk(s)
    static constexpr int kRingA = kSP ? 3 : 4;
    static constexpr int kRingABytes = kRingA * kStageA;  // 144 / 128 KB
    static constexpr int kHhiBytes = 128 * 1024;          // up to 8 k-blocks of [128 x 32 fp32]
    static_assert(kHhiBytes <= kRingABytes, "the SMEM half of H lives inside ring A");
    static constexpr int kB2Rows = 64;                  // B2 rows per CTA per 128-wide N tile
    static constexpr int kB2KbBytes = kB2Rows * 128;    // 8 KB
    static constexpr int kKbPerStageB = kSP ? 2 : 4;
    static constexpr int kStageB = kKbPerStageB * kB2KbBytes;
    static constexpr int kRingB = 2;
    static constexpr int kOutBytes = 16384;             // one [128 x 32 fp32] output box per group
    static constexpr int kSmem = kRingABytes + kRingB * kStageB + 2 * kOutBytes + 1024 /*bias*/ + 1024 /*align*/ +
                                 256 /*barriers*/;
    static_assert(kSmem <= 232448, "exceeds the 227 KB dynamic shared memory limit");
};

template <bool kSP>
__global__ void __launch_bounds__(384, 1)
    b2b_tf32_kernel(const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
                    const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmY, B2BArgs args) {
    using C = B2BT32Cfg<kSP>;
    constexpr int kCG = 2;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base_u32 - smem_u32(smem_raw));
    uint8_t* hhi = smem;                                   // ring A while GEMM1 runs, H upper half after
    uint8_t* ringB = smem + C::kRingABytes;
    uint8_t* stage_out = ringB + C::kRingB * C::kStageB;  // 2 x 16 KB (one per epilogue group)
    float* bias_s = reinterpret_cast<float*>(stage_out + 2 * C::kOutBytes);  // [group][slot][64]
    uint64_t* bars = reinterpret_cast<uint64_t*>(stage_out + 2 * C::kOutBytes + 1024);
    uint64_t* fullA = bars;                      // [kRingA]
    uint64_t* emptyA = fullA + C::kRingA;        // [kRingA]
    uint64_t* fullB = emptyA + C::kRingA;        // [kRingB]
    uint64_t* emptyB = fullB + C::kRingB;        // [kRingB]
    uint64_t* tfull1 = emptyB + C::kRingB;       // [2] GEMM1 chunk accumulated
    uint64_t* hready = tfull1 + 2;               // [2] chunk converted (TMEM in place / SMEM)
    uint64_t* tfull2 = hready + 2;               // [2] GEMM2 slot accumulated
    uint64_t* tempty2 = tfull2 + 2;              // [2] GEMM2 slot drained
    uint64_t* hhi_free = tempty2 + 2;            // GEMM2 of the tile has finished reading SMEM H
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hhi_free + 1);

    const uint32_t warp = warp_id();
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;

    if (warp == 0 && elect_one()) {
        prefetch_tmap(&tmA1);
        prefetch_tmap(&tmB1);
        prefetch_tmap(&tmB2);
        prefetch_tmap(&tmY);
        for (int s = 0; s < C::kRingA; ++s) {
            mbar_init(&fullA[s], kCG);
            mbar_init(&emptyA[s], 1);
        }
        for (int s = 0; s < C::kRingB; ++s) {
            mbar_init(&fullB[s], kCG);
            mbar_init(&emptyB[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull1[i], 1);
            mbar_init(&hready[i], 8 * kCG);
            mbar_init(&tfull2[i], 1);
            mbar_init(&tempty2[i], 8 * kCG);
        }
        mbar_init(hhi_free, 1);
        fence_barrier_init();
    }
    if (warp == 2) {
        tmem_alloc<kCG>(tmem_slot, 512);
        tmem_relinquish<kCG>();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();
    pdl_launch_dependents();  // after the wait: a dependent starts only once our predecessor completed

    const int tile_rows = 256;
    const int num_tiles = (args.T + tile_rows - 1) / tile_rows;
    const int cluster_id = blockIdx.x / kCG;
    const int num_clusters = gridDim.x / kCG;
    const int nkb1 = (args.K1 + C::kBK - 1) / C::kBK;
    const int nkb2 = args.R_pad / C::kBK;                // 16 at R = 512: 8 from TMEM, rest from SMEM
    const int nkb_lo = 256 / C::kBK;                      // k-blocks held in TMEM
    const int w1 = args.R_pad - 256;                      // width of GEMM1 chunk 1 (upper half)
    const int nstB = (nkb2 + C::kKbPerStageB - 1) / C::kKbPerStageB;
    const int n2_tiles = (args.N2 + 127) / 128;

    if (warp == 0) {
        // ---------------------------------------------------------------- producer A (GEMM1)
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int t = cluster_id; t < num_tiles; t += num_clusters, ++it) {
                if (it > 0) mbar_wait(hhi_free, (it - 1) & 1);  // previous tile's SMEM H is dead
                const int am = t * tile_rows + (int)rank * 128;
                for (int pass = 0; pass < (kSP ? 1 : 2); ++pass) {
                    const int c_lo = kSP ? 0 : pass, c_hi = kSP ? 2 : pass + 1;
                    uint32_t bytes = 16384;
                    for (int c = c_lo; c < c_hi; ++c) bytes += (uint32_t)((c == 0 ? 256 : w1) / kCG) * 128;
                    for (int kb = 0; kb < nkb1; ++kb) {
                        mbar_wait(&emptyA[stage], phase ^ 1);
                        uint8_t* st = hhi + stage * C::kStageA;
                        if (leader) mbar_arrive_expect_tx(&fullA[stage], bytes * kCG);
                        else mbar_arrive_cluster(&fullA[stage], 0);
                        tma_load_2d<kCG>(&tmA1, &fullA[stage], st, kb * C::kBK, am);
                        for (int c = c_lo; c < c_hi; ++c) {
                            const int brows = (c == 0 ? 256 : w1) / kCG;
                            const int b0 = 256 * c + (int)rank * brows;
                            uint8_t* bst = st + 16384 + (c - c_lo) * 16384;
                            for (int r = 0; r < brows; r += args.b1rows)
                                tma_load_2d<kCG>(&tmB1, &fullA[stage], bst + r * 128, kb * C::kBK, b0 + r);
                        }
                        if (++stage == C::kRingA) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 3) {
        // ---------------------------------------------------------------- producer B (GEMM2 B2 tiles)
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cluster_id; t < num_tiles; t += num_clusters) {
                for (int j = 0; j < n2_tiles; ++j) {
                    const int brow = j * 128 + (int)rank * C::kB2Rows;
                    for (int s = 0; s < nstB; ++s) {
                        const int kb0 = s * C::kKbPerStageB;
                        const int nk = min(C::kKbPerStageB, nkb2 - kb0);
                        mbar_wait(&emptyB[stage], phase ^ 1);
                        uint8_t* st = ringB + stage * C::kStageB;
                        if (leader) mbar_arrive_expect_tx(&fullB[stage], (uint32_t)(nk * C::kB2KbBytes * kCG));
                        else mbar_arrive_cluster(&fullB[stage], 0);
                        for (int q = 0; q < nk; ++q)
                            tma_load_2d<kCG>(&tmB2, &fullB[stage], st + q * C::kB2KbBytes, (kb0 + q) * C::kBK, brow);
                        if (++stage == C::kRingB) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA issuer
        if (leader && elect_one()) {
            int sa = 0, sb = 0;
            uint32_t pa = 0, pb = 0;
            uint32_t slot_seq = 0;
            const uint32_t idesc2 = make_idesc(1, 256, 128, 0, 0);
            int it = 0;
            for (int t = cluster_id; t < num_tiles; t += num_clusters, ++it) {
                // ---- GEMM1: chunk 0 -> TMEM [0,256), chunk 1 -> [256, 256 + w1) (the GEMM2 slots)
                for (int pass = 0; pass < (kSP ? 1 : 2); ++pass) {
                    const int c_lo = kSP ? 0 : pass, c_hi = kSP ? 2 : pass + 1;
                    if (c_hi > 1) {  // chunk 1 overlays both GEMM2 slots
                        for (int u = 0; u < 2; ++u, ++slot_seq)
                            mbar_wait(&tempty2[slot_seq & 1], ((slot_seq >> 1) & 1) ^ 1);
                        tc_fence_after();
                    }
                    for (int kb = 0; kb < nkb1; ++kb) {
                        mbar_wait(&fullA[sa], pa);
                        tc_fence_after();
                        const uint32_t a_addr = smem_u32(hhi + sa * C::kStageA);
                        for (int c = c_lo; c < c_hi; ++c) {
                            const uint32_t idesc1 = make_idesc(1, 256, c == 0 ? 256 : w1, 0, 0);
                            const uint32_t d = tmem_base + 256 * c;
                            const uint32_t b_addr = a_addr + 16384 + (c - c_lo) * 16384;
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                mma_ss<kCG, 1>(d, make_sdesc(a_addr + k * 32, 0, 1024), make_sdesc(b_addr + k * 32, 0, 1024),
                                               idesc1, (kb > 0 || k > 0) ? 1u : 0u);
                        }
                        mma_commit<kCG>(&emptyA[sa]);
                        if (++sa == C::kRingA) { sa = 0; pa ^= 1; }
                    }
                    for (int c = c_lo; c < c_hi; ++c) mma_commit<kCG>(&tfull1[c]);
                }
                // ---- wait for the converted H (TMEM lower half, SMEM upper half) of both CTAs
                for (int c = 0; c < 2; ++c) mbar_wait(&hready[c], it & 1);
                tc_fence_after();
                // ---- GEMM2: 128-wide output tiles, K = R_pad (TS over TMEM, SS over SMEM)
                const uint32_t hhi_addr = smem_u32(hhi);
                for (int j = 0; j < n2_tiles; ++j, ++slot_seq) {
                    const uint32_t s = slot_seq & 1;
                    mbar_wait(&tempty2[s], ((slot_seq >> 1) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t d = tmem_base + 256 + 128 * s;
                    for (int st2 = 0; st2 < nstB; ++st2) {
                        const int kb0 = st2 * C::kKbPerStageB;
                        const int nk = min(C::kKbPerStageB, nkb2 - kb0);
                        mbar_wait(&fullB[sb], pb);
                        tc_fence_after();
                        const uint32_t b_addr = smem_u32(ringB + sb * C::kStageB);
                        for (int q = 0; q < nk; ++q) {
                            const int kb = kb0 + q;
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const uint64_t bdesc = make_sdesc(b_addr + q * C::kB2KbBytes + k * 32, 0, 1024);
                                const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
                                if (kb < nkb_lo)
                                    mma_ts<kCG, 1>(d, tmem_base + (uint32_t)(kb * 32 + k * 8), bdesc, idesc2, acc);
                                else
                                    mma_ss<kCG, 1>(d, make_sdesc(hhi_addr + (kb - nkb_lo) * 16384 + k * 32, 0, 1024),
                                                   bdesc, idesc2, acc);
                            }
                        }
                        mma_commit<kCG>(&emptyB[sb]);
                        if (++sb == C::kRingB) { sb = 0; pb ^= 1; }
                    }
                    mma_commit<kCG>(&tfull2[s]);
                }
                mma_commit<kCG>(hhi_free);  // every GEMM2 MMA of this tile (SMEM H readers) has completed
            }
        }
    } else if (warp >= 4) {
        // ---------------------------------------------------------------- epilogue
        const uint32_t q = warp & 3;
        const uint32_t wg = (warp - 4) >> 2;
        const uint32_t lane = lane_id();
        const uint32_t lane_base = (q * 32u) << 16;
        const uint32_t srow = q * 32 + lane;
        const bool issuer = (q == 0 && lane == 0);
        uint8_t* buf = stage_out + wg * C::kOutBytes;
        float* bias_g = bias_s + wg * 128;
        uint32_t slot_seq = 0;
        uint32_t tf_par0 = 0, tf_par1 = 0;
        auto load_bias_col = [&](int col) -> float {
            return (args.bias == nullptr || col >= args.N2) ? 0.f : __ldg(args.bias + col);
        };
        float bias_pref = load_bias_col((int)(wg * 64 + (srow & 63)));
        auto arrive_leader = [&](uint64_t* bar) {
            if (leader) mbar_arrive(bar);
            else mbar_arrive_cluster(bar, 0);
        };
        auto save_cols = [&](int row, bool row_ok, int col, const uint32_t (&r)[16]) {
            if (args.save && row_ok && col + 16 > args.save_col0 && col < args.save_col0 + args.save_cols) {
                float* dst = reinterpret_cast<float*>(args.save) + row;
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    if (col + i >= args.save_col0 && col + i < args.save_col0 + args.save_cols)
                        dst[(long long)(col + i - args.save_col0) * args.ld_save] = __uint_as_float(r[i]);
            }
        };
        int it = 0;
        for (int t = cluster_id; t < num_tiles; t += num_clusters, ++it) {
            const int row = t * tile_rows + (int)rank * 128 + (int)srow;
            const bool row_ok = row < args.T;
            // ---- chunk 0: TF32-round in place in TMEM (group wg: columns [128 wg, 128 wg + 128))
            mbar_wait(&tfull1[0], it & 1);
            tc_fence_after();
#pragma unroll 1
            for (int cl = (int)wg * 128; cl < ((int)wg + 1) * 128; cl += 16) {
                uint32_t r[16];
                tmem_ld16(tmem_base + lane_base + cl, r);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(tf32_rna(__uint_as_float(r[i])));
                uint32_t lo[8], hi[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) { lo[i] = r[i]; hi[i] = r[8 + i]; }
                tmem_st8(tmem_base + lane_base + cl, lo);
                tmem_st8(tmem_base + lane_base + cl + 8, hi);
                save_cols(row, row_ok, cl, r);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive_leader(&hready[0]);
            // ---- chunk 1: TMEM [256, 256 + w1) -> TF32 -> SMEM upper half (K-major SW128 tiles)
            mbar_wait(&tfull1[1], it & 1);   // also: every GEMM1 MMA (ring A reader) has completed
            tc_fence_after();
            const int half = w1 / 2;
#pragma unroll 1
            for (int cl = (int)wg * half; cl < ((int)wg + 1) * half; cl += 16) {
                uint32_t r[16];
                tmem_ld16(tmem_base + lane_base + 256 + cl, r);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(tf32_rna(__uint_as_float(r[i])));
                const int kb = cl / C::kBK, cc = cl % C::kBK;   // k-block, column inside it
                const uint32_t rowa = smem_u32(hhi) + kb * 16384 + srow * 128;
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const uint32_t ch = (uint32_t)(cc / 4 + g);
                    st_shared_v4(rowa + ((ch ^ (srow & 7)) << 4), r[4 * g], r[4 * g + 1], r[4 * g + 2], r[4 * g + 3]);
                }
                save_cols(row, row_ok, 256 + cl, r);
            }
            fence_proxy_async_smem();  // generic smem writes -> visible to the tensor core (async proxy)
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                arrive_leader(&hready[1]);
                arrive_leader(&tempty2[slot_seq & 1]);        // chunk 1 overlaid both GEMM2 slots
                arrive_leader(&tempty2[(slot_seq + 1) & 1]);
            }
            slot_seq += 2;
            // ---- GEMM2 output tiles: this group's 64 columns, as two [128 x 32 fp32] boxes
            for (int j = 0; j < n2_tiles; ++j, ++slot_seq) {
                const uint32_t s = slot_seq & 1;
                const float bval = bias_pref;
                bias_pref = load_bias_col((j + 1 == n2_tiles ? 0 : j + 1) * 128 + (int)(wg * 64 + (srow & 63)));
                mbar_wait(&tfull2[s], s ? tf_par1 : tf_par0);
                if (s) tf_par1 ^= 1u; else tf_par0 ^= 1u;
                tc_fence_after();
                if (srow < 64) bias_g[s * 64 + srow] = bval;
                uint32_t ra[32], rb[32];
                tmem_ld32(tmem_base + lane_base + 256 + 128 * s + 64 * wg, ra);
                tmem_ld32(tmem_base + lane_base + 256 + 128 * s + 64 * wg + 32, rb);
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive_leader(&tempty2[s]);
                const int n0 = j * 128 + 64 * (int)wg;
                const uint32_t row_addr = smem_u32(buf) + srow * 128;
#pragma unroll
                for (int box = 0; box < 2; ++box) {
                    if (issuer) bulk_wait_read<0>();  // the previous box has left `buf`
                    named_bar_sync(1 + wg, 128);
                    const uint32_t* src = box == 0 ? ra : rb;
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float4 b4 = reinterpret_cast<const float4*>(bias_g + s * 64)[box * 8 + c];
                        float v[4] = {fmaf(__uint_as_float(src[4 * c]), args.alpha, b4.x),
                                      fmaf(__uint_as_float(src[4 * c + 1]), args.alpha, b4.y),
                                      fmaf(__uint_as_float(src[4 * c + 2]), args.alpha, b4.z),
                                      fmaf(__uint_as_float(src[4 * c + 3]), args.alpha, b4.w)};
                        if (args.relu) {
#pragma unroll
                            for (int i = 0; i < 4; ++i) v[i] = fmaxf(v[i], 0.f);
                        }
                        if (args.mask && row_ok && n0 + 32 * box + 4 * c < args.N2) {
                            const uint4 mk = __ldg(reinterpret_cast<const uint4*>(
                                reinterpret_cast<const float*>(args.mask) + (long long)row * args.ld_mask + n0 +
                                32 * box + 4 * c));
                            const uint32_t m[4] = {mk.x, mk.y, mk.z, mk.w};
#pragma unroll
                            for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(m[i]) > 0.f ? v[i] : 0.f;
                        }
                        st_shared_v4(row_addr + ((uint32_t)(c ^ (srow & 7)) << 4), __float_as_uint(v[0]),
                                     __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3]));
                    }
                    fence_proxy_async_smem();
                    named_bar_sync(1 + wg, 128);
                    if (issuer) {
                        tma_store_2d(&tmY, buf, n0 + 32 * box, t * tile_rows + (int)rank * 128);
                        bulk_commit();
                    }
                }
            }
        }
        if (issuer) bulk_wait<0>();
    }

    tc_fence_before();
    cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<kCG>(tmem_base, 512);
    }
}

}  // namespace dev

// Host side: the wide-rank TF32 fused kernel covers 256 < R_pad <= 512.
inline bool b2b_tf32_wide_supported(long long R_pad) { return R_pad > 256 && R_pad <= 512; }

}  // namespace skl
