// b2b.cuh -- fused back-to-back tcgen05 kernel: the SKLinear hot op.
//
// Forward  (nn_layers.cpp:61-76, row convention):
//     H = X · Acat                  [tile, R]   (R = 2Lk: all L terms, both branches)
//     Y = inv · H · Bcat + b        [tile, d_out]
// Backward data path (nn_layers.cpp:78-101):
//     P  = G · Bcatᵀ                [tile, R]
//     dX = inv · P · Acatᵀ          [tile, d_in]
// Both are   OUT = alpha · (A1 · B1ᵀ) · B2ᵀ (+ bias),  so one kernel serves both.
//
// The rank-R intermediate never touches HBM: GEMM1 accumulates H in TMEM
// (fp32), the epilogue warps round it to bf16 and write it back into TMEM,
// and GEMM2 consumes it directly as the A operand (tcgen05.mma ... [a_tmem],
// the "TS" form).  The Σ over the L terms and the two branches is simply the
// K = R reduction of GEMM2, i.e. one TMEM accumulator per output tile; the
// 1/(2L) scale and the bias are fused into the GEMM2 epilogue.  Columns of H
// the backward needs (x·S1 in the forward, G·S2ᵀ in the backward) are
// streamed out by the conversion epilogue, from registers, at no extra read.
//
// TMEM map (512 columns, one CTA per SM):
//   GEMM1 chunk c (<= 256 wide) accumulates fp32 in [256c, 256c + W_c)
//   bf16 H (2 values / column)          lives in [0, R/2)   (in-place compaction)
//   GEMM2 double-buffered slots         [256, 384) and [384, 512)
// Chunk 1 and the GEMM2 slots share [256, 512); chunk 1 therefore acquires
// both slots from the slot ring and releases them once converted.
//
// Warp roles: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 4..7 epilogue.
// kCG == 2 runs cta_group::2 (M = 256 tokens per CTA pair, each CTA keeps
// its 128 rows of H in its own TMEM, B operands are split across the pair).
#pragma once

#include "sm100.cuh"

namespace skl {

struct B2BArgs {
    int T, K1, R, R_pad, N2;
    float alpha;
    const float* bias;  // [N2] fp32, nullable
    void* out;          // [T, N2] bf16, row stride ldo
    long long ldo;
    void* save;         // H columns [save_col0, save_col0 + save_cols) -> save[t][c - save_col0]
    int save_col0, save_cols;
    int Lk, k, dS;      // direct modes: L*k, k, and the term row stride of the [L*d][k] views
    int bias_bf16;      // bias pointer holds bf16 (direct modes skip the fp32 copy)
    int dbg;            // perf-bisection switches (SKL_B2B_DEBUG): 1 skip GEMM2 epilogue math/stores, 4 skip GEMM2 MMAs
    long long ld_save;
};

namespace dev {

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem]  (kind::f16, A K-major bf16 packed 2/column)
template <int kCG>
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
    if constexpr (kCG == 1)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
            "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
            "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

template <int kCG>
struct B2BCfg {
    static constexpr int kStageBytes = kCG == 1 ? 48 * 1024 : 32 * 1024;
    static constexpr int kStages = kCG == 1 ? 4 : 6;
    static constexpr int kB2Rows = 128 / kCG;               // B2 rows per CTA per 128-wide N tile
    static constexpr int kB2KbBytes = kB2Rows * 128;         // one 64-wide k-block of B2
    static constexpr int kKbPerStage2 = kStageBytes / kB2KbBytes;
    static constexpr int kB1BoxRows = 32;
    static constexpr int kSmem = kStages * kStageBytes + 2 * 16384 + 1024 /*bias*/ + 1024 /*align*/ + 256;
    static_assert(kSmem <= 232448, "exceeds the 227 KB dynamic shared memory limit");
};

// kMode 0: B1 / B2 are packed K-major panels (any k).
// kMode 1: forward straight from the ABI stacks (k % 64 == 0): B1 = S1s|U2s
//          viewed as [L*d_in][k] (MN-major tiles), B2 = U1s|S2s viewed as
//          [L*k][d_out] (MN-major tiles).  No packing pass.
// kMode 2: backward straight from the stacks: B1 = U1s|S2s [L*k][d_out]
//          (K-major), B2 = S1s|U2s [L*d_in][k] (K-major, per-term row offset).
template <int kCG, int kMode>
__global__ void __launch_bounds__(256, 1)
    b2b_kernel(const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
               const __grid_constant__ CUtensorMap tmB1b, const __grid_constant__ CUtensorMap tmB2,
               const __grid_constant__ CUtensorMap tmB2b, const __grid_constant__ CUtensorMap tmY, B2BArgs args) {
    using C = B2BCfg<kCG>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base_u32 - smem_u32(smem_raw));
    uint8_t* stage_out = smem + C::kStages * C::kStageBytes;  // 2 x 16 KB output staging
    float* bias_s = reinterpret_cast<float*>(stage_out + 2 * 16384);  // 2 slots x 128 bias values
    uint64_t* bars = reinterpret_cast<uint64_t*>(stage_out + 2 * 16384 + 1024);
    uint64_t* full = bars;                            // [kStages]
    uint64_t* empty = bars + C::kStages;              // [kStages]
    uint64_t* tfull1 = bars + 2 * C::kStages;         // [2] GEMM1 chunk accumulated
    uint64_t* hready = tfull1 + 2;                    // [2] chunk converted to bf16 H
    uint64_t* tfull2 = hready + 2;                    // [2] GEMM2 slot accumulated
    uint64_t* tempty2 = tfull2 + 2;                   // [2] GEMM2 slot drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty2 + 2);

    const uint32_t warp = warp_id();
    const uint32_t rank = kCG == 2 ? cluster_ctarank() : 0;
    const bool leader = rank == 0;

    if (warp == 0 && elect_one()) {
        prefetch_tmap(&tmA1);
        prefetch_tmap(&tmB1);
        prefetch_tmap(&tmB2);
        if constexpr (kMode != 0) {
            prefetch_tmap(&tmB1b);
            prefetch_tmap(&tmB2b);
        }
        prefetch_tmap(&tmY);
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], kCG);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull1[i], 1);
            mbar_init(&hready[i], 4 * kCG);
            mbar_init(&tfull2[i], 1);
            mbar_init(&tempty2[i], 4 * kCG);
        }
        fence_barrier_init();
    }
    if (warp == 2) {
        tmem_alloc<kCG>(tmem_slot, 512);
        tmem_relinquish<kCG>();
    }
    tc_fence_before();
    if constexpr (kCG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int tile_rows = 128 * kCG;
    const int num_tiles = (args.T + tile_rows - 1) / tile_rows;
    const int cluster_id = blockIdx.x / kCG;
    const int num_clusters = gridDim.x / kCG;
    const int nch = (args.R_pad + 255) / 256;
    const int nkb1 = (args.K1 + 63) / 64;
    const int nkb2 = args.R_pad / 64;
    const int nst2 = (nkb2 + C::kKbPerStage2 - 1) / C::kKbPerStage2;
    const int n2_tiles = (args.N2 + 127) / 128;

    if (warp == 0) {
        // ---------------------------------------------------------------- producer
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            auto next = [&]() { if (++stage == C::kStages) { stage = 0; phase ^= 1; } };
            for (int t = cluster_id; t < num_tiles; t += num_clusters) {
                const int am = t * tile_rows + (int)rank * 128;
                for (int c = 0; c < nch; ++c) {
                    const int wc = min(256, args.R_pad - 256 * c);
                    const int brows = wc / kCG;
                    const int b0 = 256 * c + (int)rank * brows;
                    const uint32_t bytes = 16384 + brows * 128;
                    for (int kb = 0; kb < nkb1; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* st = smem + stage * C::kStageBytes;
                        if (leader) mbar_arrive_expect_tx(&full[stage], bytes * kCG);
                        else mbar_arrive_cluster(&full[stage], 0);
                        tma_load_2d<kCG>(&tmA1, &full[stage], st, kb * 64, am);
                        if constexpr (kMode == 0) {
                            for (int r = 0; r < brows; r += C::kB1BoxRows)
                                tma_load_2d<kCG>(&tmB1, &full[stage], st + 16384 + r * 128, kb * 64, b0 + r);
                        } else if constexpr (kMode == 2) {  // rows of [U1s ; S2s]
                            for (int r = 0; r < brows; r += C::kB1BoxRows) {
                                const int rg = b0 + r;
                                tma_load_2d<kCG>(rg < args.Lk ? &tmB1 : &tmB1b, &full[stage], st + 16384 + r * 128, kb * 64,
                                                 rg < args.Lk ? rg : rg - args.Lk);
                            }
                        } else {  // MN-major [64 d_in rows x 64 rank cols] blocks of S1s | U2s
                            for (int jb = 0; jb < brows / 64; ++jb) {
                                const int rg = b0 + 64 * jb;
                                const int rr = rg < args.Lk ? rg : rg - args.Lk;
                                tma_load_2d<kCG>(rg < args.Lk ? &tmB1 : &tmB1b, &full[stage], st + 16384 + jb * 8192,
                                                 rr % args.k, (rr / args.k) * args.dS + kb * 64);
                            }
                        }
                        next();
                    }
                }
                for (int j = 0; j < n2_tiles; ++j) {
                    const int brow = j * 128 + (int)rank * C::kB2Rows;
                    for (int s = 0; s < nst2; ++s) {
                        const int kb0 = s * C::kKbPerStage2;
                        const int nk = min(C::kKbPerStage2, nkb2 - kb0);
                        mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* st = smem + stage * C::kStageBytes;
                        if (leader) mbar_arrive_expect_tx(&full[stage], (uint32_t)(nk * C::kB2KbBytes * kCG));
                        else mbar_arrive_cluster(&full[stage], 0);
                        for (int q = 0; q < nk; ++q) {
                            const int r0 = (kb0 + q) * 64;  // rank index of this k-block
                            if constexpr (kMode == 0) {
                                tma_load_2d<kCG>(&tmB2, &full[stage], st + q * C::kB2KbBytes, r0, brow);
                            } else if constexpr (kMode == 1) {  // MN-major rows of [U1s ; S2s]
                                const CUtensorMap* m = r0 < args.Lk ? &tmB2 : &tmB2b;
                                const int rr = r0 < args.Lk ? r0 : r0 - args.Lk;
                                for (int jb = 0; jb < C::kB2Rows / 64; ++jb)
                                    tma_load_2d<kCG>(m, &full[stage], st + q * C::kB2KbBytes + jb * 8192, brow + 64 * jb, rr);
                            } else {  // K-major [d_in rows x 64 rank cols] of S1s | U2s, term row offset
                                const int rr = r0 < args.Lk ? r0 : r0 - args.Lk;
                                tma_load_2d<kCG>(r0 < args.Lk ? &tmB2 : &tmB2b, &full[stage], st + q * C::kB2KbBytes,
                                                 rr % args.k, (rr / args.k) * args.dS + brow);
                            }
                        }
                        next();
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA issuer
        if (leader && elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            auto next = [&]() { if (++stage == C::kStages) { stage = 0; phase ^= 1; } };
            uint32_t slot_seq = 0;
            const uint32_t idesc2 = make_idesc(0, 128 * kCG, 128, 0, kMode == 1 ? 1 : 0);
            int it = 0;
            for (int t = cluster_id; t < num_tiles; t += num_clusters, ++it) {
                // ---- GEMM1: H chunks
                for (int c = 0; c < nch; ++c) {
                    const int wc = min(256, args.R_pad - 256 * c);
                    if (c == 1) {  // chunk 1 overlays both GEMM2 slots
                        for (int u = 0; u < 2; ++u, ++slot_seq)
                            mbar_wait(&tempty2[slot_seq & 1], ((slot_seq >> 1) & 1) ^ 1);
                        tc_fence_after();
                    }
                    const uint32_t idesc1 = make_idesc(0, 128 * kCG, wc, 0, kMode == 1 ? 1 : 0);
                    const uint32_t d = tmem_base + 256 * c;
                    for (int kb = 0; kb < nkb1; ++kb) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint32_t a_addr = smem_u32(smem + stage * C::kStageBytes);
                        const uint32_t b_addr = a_addr + 16384;
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            mma_ss<kCG, 0>(d, make_sdesc(a_addr + k * 32, 0, 1024),
                                           kMode == 1 ? make_sdesc(b_addr + k * 2048, 8192, 1024)
                                                      : make_sdesc(b_addr + k * 32, 0, 1024),
                                           idesc1, (kb > 0 || k > 0) ? 1u : 0u);
                        mma_commit<kCG>(&empty[stage]);
                        next();
                    }
                    mma_commit<kCG>(&tfull1[c]);
                }
                // ---- wait for the bf16 H of this tile (both CTAs)
                for (int c = 0; c < nch; ++c) mbar_wait(&hready[c], it & 1);
                tc_fence_after();
                // ---- GEMM2: 128-wide output tiles, A = H from TMEM
                for (int j = 0; j < n2_tiles; ++j, ++slot_seq) {
                    const uint32_t s = slot_seq & 1;
                    mbar_wait(&tempty2[s], ((slot_seq >> 1) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t d = tmem_base + 256 + 128 * s;
                    for (int st2 = 0; st2 < nst2; ++st2) {
                        const int kb0 = st2 * C::kKbPerStage2;
                        const int nk = min(C::kKbPerStage2, nkb2 - kb0);
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint32_t b_addr = smem_u32(smem + stage * C::kStageBytes);
                        for (int q = 0; q < nk; ++q) {
                            if (args.dbg & 4) break;  // perf bisection: skip GEMM2 MMAs
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const uint32_t a_t = tmem_base + (uint32_t)((kb0 + q) * 32 + k * 8);
                                const uint64_t bdesc = kMode == 1
                                    ? make_sdesc(b_addr + q * C::kB2KbBytes + k * 2048, 8192, 1024)
                                    : make_sdesc(b_addr + q * C::kB2KbBytes + k * 32, 0, 1024);
                                mma_ts<kCG>(d, a_t, bdesc, idesc2, (st2 > 0 || q > 0 || k > 0) ? 1u : 0u);
                            }
                        }
                        mma_commit<kCG>(&empty[stage]);
                        next();
                    }
                    mma_commit<kCG>(&tfull2[s]);
                }
            }
        }
    } else if (warp >= 4) {
        // ---------------------------------------------------------------- epilogue
        const uint32_t q = warp & 3;
        const uint32_t lane = lane_id();
        const uint32_t lane_base = (q * 32u) << 16;
        uint32_t slot_seq = 0;
        uint32_t tf_par0 = 0, tf_par1 = 0;
        uint32_t sbuf = 0;                       // output staging buffer toggle
        const bool issuer = (q == 0 && lane == 0);  // issues / waits the bulk stores
        int it = 0;
        for (int t = cluster_id; t < num_tiles; t += num_clusters, ++it) {
            const int row = t * tile_rows + (int)rank * 128 + (int)(q * 32 + lane);
            const bool row_ok = row < args.T;
            // ---- convert GEMM1 chunks: fp32 -> bf16 H in TMEM (+ saved columns)
            for (int c = 0; c < nch; ++c) {
                const int wc = min(256, args.R_pad - 256 * c);
                mbar_wait(&tfull1[c], it & 1);
                tc_fence_after();
#pragma unroll 1
                for (int g2 = 0; g2 < wc / 32; ++g2) {
                  uint32_t rr[2][16];
                  tmem_ld16(tmem_base + lane_base + 256 * c + 32 * g2, rr[0]);
                  tmem_ld16(tmem_base + lane_base + 256 * c + 32 * g2 + 16, rr[1]);
                  tmem_ld_wait();
#pragma unroll
                  for (int hh = 0; hh < 2; ++hh) {
                    const int g = 2 * g2 + hh;
                    const uint32_t (&r)[16] = rr[hh];
                    uint32_t p[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) p[i] = pack_bf16x2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
                    tmem_st8(tmem_base + lane_base + 128 * c + 8 * g, p);
                    const int col = 256 * c + 16 * g;  // H column (R order)
                    if (args.save && row_ok && col + 16 > args.save_col0 && col < args.save_col0 + args.save_cols) {
                        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(args.save) +
                                             (long long)row * args.ld_save + (col - args.save_col0);
                        if (col >= args.save_col0 && col + 16 <= args.save_col0 + args.save_cols &&
                            (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                            reinterpret_cast<uint4*>(dst)[0] = make_uint4(p[0], p[1], p[2], p[3]);
                            reinterpret_cast<uint4*>(dst)[1] = make_uint4(p[4], p[5], p[6], p[7]);
                        } else {
                            const __nv_bfloat16* pb = reinterpret_cast<const __nv_bfloat16*>(p);
                            for (int i = 0; i < 16; ++i)
                                if (col + i >= args.save_col0 && col + i < args.save_col0 + args.save_cols)
                                    dst[i] = pb[i];
                        }
                    }
                  }
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (leader) mbar_arrive(&hready[c]);
                    else mbar_arrive_cluster(&hready[c], 0);
                    if (c == 1) {  // release the two slots chunk 1 overlaid
                        for (int u = 0; u < 2; ++u) {
                            const uint32_t s = (slot_seq + u) & 1;
                            if (leader) mbar_arrive(&tempty2[s]);
                            else mbar_arrive_cluster(&tempty2[s], 0);
                        }
                    }
                }
                if (c == 1) slot_seq += 2;
            }
            // ---- GEMM2 output tiles
            for (int j = 0; j < n2_tiles; ++j, ++slot_seq) {
                const uint32_t s = slot_seq & 1;
                const uint32_t srow = q * 32 + lane;
                // The tile's 128 bias values go through shared memory: with
                // ~226 KB of smem in use L1 is tiny, so per-thread global bias
                // loads would each pay L2 latency inside the epilogue.
                const int bcol = j * 128 + (int)srow;
                float bval = 0.f;
                if (args.bias != nullptr && bcol < args.N2)
                    bval = args.bias_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(args.bias)[bcol])
                                          : __ldg(args.bias + bcol);
                // tfull2[s] completes once per GEMM2 job on slot s (chunk-1
                // acquisitions never commit it), so count its phases per slot.
                mbar_wait(&tfull2[s], s ? tf_par1 : tf_par0);
                if (s) tf_par1 ^= 1u; else tf_par0 ^= 1u;
                tc_fence_after();
                bias_s[s * 128 + srow] = bval;  // published by the named barrier below
                // Two 64-column halves per tile: TMEM -> alpha*acc + b -> bf16 ->
                // 128B-swizzled smem staging buffer -> one TMA bulk store each
                // (coalesced, clipped at T / N2 by the tensor map).
                if (args.dbg & 1) {  // perf bisection: release the slot without reading it
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if (leader) mbar_arrive(&tempty2[s]);
                        else mbar_arrive_cluster(&tempty2[s], 0);
                    }
                    continue;
                }
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {
                    uint32_t ra[32], rb[32];
                    tmem_ld32(tmem_base + lane_base + 256 + 128 * s + 64 * h, ra);
                    tmem_ld32(tmem_base + lane_base + 256 + 128 * s + 64 * h + 32, rb);
                    tmem_ld_wait();
                    if (h == 1) {  // every TMEM read of this slot has completed
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) {
                            if (leader) mbar_arrive(&tempty2[s]);
                            else mbar_arrive_cluster(&tempty2[s], 0);
                        }
                    }
                    const int n0 = j * 128 + 64 * h;
                    if (args.dbg & 16) continue;  // perf bisection: TMEM reads only
                    uint8_t* buf = stage_out + sbuf * 16384;
                    if (issuer) bulk_wait_read<1>();  // the store that used `buf` has read it
                    named_bar_sync(1, 128);
                    const uint32_t row_addr = smem_u32(buf) + srow * 128;
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float4* bp = reinterpret_cast<const float4*>(bias_s + s * 128 + 64 * h + 8 * c);
                        const float4 b0 = bp[0], b1 = bp[1];
                        const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                        const uint32_t* src = (c < 4) ? ra : rb;
                        const int o = (c & 3) * 8;
                        uint32_t w[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            w[i] = pack_bf16x2(fmaf(__uint_as_float(src[o + 2 * i]), args.alpha, bv[2 * i]),
                                               fmaf(__uint_as_float(src[o + 2 * i + 1]), args.alpha, bv[2 * i + 1]));
                        st_shared_v4(row_addr + ((uint32_t)(c ^ (srow & 7)) << 4), w[0], w[1], w[2], w[3]);
                    }
                    fence_proxy_async_smem();
                    named_bar_sync(1, 128);
                    if (issuer && !(args.dbg & 8)) {
                        tma_store_2d(&tmY, buf, n0, t * tile_rows + (int)rank * 128);
                        bulk_commit();
                    }
                    sbuf ^= 1;
                }
            }
        }
        if (issuer) bulk_wait<0>();
    }

    tc_fence_before();
    if constexpr (kCG == 2) cluster_sync(); else __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<kCG>(tmem_base, 512);
    }
}

}  // namespace dev

// Host side (skl.cu): whether the fused path handles this rank / dtype.
inline bool b2b_supported(long long R_pad, int kind) { return kind == 0 && R_pad <= 512; }

}  // namespace skl
