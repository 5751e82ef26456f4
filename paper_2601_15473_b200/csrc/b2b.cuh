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
// Warp roles: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 4..11 epilogue
// (two warpgroups splitting the columns of every tile).
// kCG == 2 runs cta_group::2 (M = 256 tokens per CTA pair, each CTA keeps
// its 128 rows of H in its own TMEM, B operands are split across the pair).
//
// R-split (kRS, R > 512, e.g. BASELINE c3: R = 1536).  A CTA pair holds at most
// R = 512 of bf16 H next to its GEMM2 accumulators, so a cluster of nsplit
// pairs (2 * nsplit CTAs) shares one 256-token tile: pair p computes the
// R-slice H_p = X · Acat[:, p*r_loc, +r_loc) (GEMM1, as above) and the partial
// D_p = H_p · Bcat[p*r_loc, +r_loc) of every output tile (GEMM2).  The partials
// are summed over DSMEM along the chain 0 -> 1 -> ... -> nsplit-1 (each pair
// adds the running sum it receives to its own accumulator and forwards it, in
// 32-column halves through one 16 KB slot per epilogue warpgroup), so the sum
// order is fixed (deterministic) and only the last pair applies alpha / bias
// and stores the tile.  H still never leaves the chip.
#pragma once

#include "sm100.cuh"
#include "trace.cuh"

#ifndef SKL_FWD_BIAS_TAB
#define SKL_FWD_BIAS_TAB 1  // 0 measured: 96 -> 106 us at c2 (per-tile bias loads cost more than the 6th stage)
#endif
namespace skl {

struct B2BArgs {
    int T, K1, R, R_pad, N2;
    float alpha;
    const float* bias;  // [N2] fp32, nullable
    void* out;          // [T, N2] bf16, row stride ldo
    long long ldo;
    void* save;         // H columns [save_col0, save_col0 + save_cols) -> save[c - save_col0][t] (transposed)
    int save_col0, save_cols;
    int Lk, k, dS;      // direct modes: L*k, k, and the term row stride of the [L*d][k] views
    int bias_bf16;      // bias pointer holds bf16 (direct modes skip the fp32 copy)
    int b1rows;         // rows per K-major B1 TMA box (largest that tiles every chunk; big boxes
                        // matter: per-SM TMA ingest grows ~2.5x from 4 KB to 16 KB boxes)
    int nsplit, r_loc;  // R-split (kRS): pairs per cluster and R columns per pair (else 1, R_pad)
    long long ld_save;
    // Fused neighbours of the layer in a Linear/ReLU chain (nn_model.cpp:111-122):
    int relu;           // forward: out = max(0, ·)  (Relu::forward, nn_layers.cpp:341-345)
    const void* mask;   // backward: out *= (mask > 0), mask = the layer input [T, N2] that a ReLU
                        // produced (Relu::backward, nn_layers.cpp:347-354); nullable
    long long ld_mask;
    // 1-bit ReLU masks (kPost == 2): bit (c % 32) of word [t * bits_ld + c / 32] is (out[t][c] > 0).
    uint32_t* relu_bits;         // forward with relu: written alongside out
    const uint32_t* mask_bits;   // backward: out *= bit, instead of reading `mask`
    long long bits_ld;           // words per row (even: 64-column groups are 8-B aligned)
    int l2hint;                  // L2 cache-hint policy bits for the producer's TMA loads
    int save_tma;                // saved columns leave through TMA stores (tmS) in 64-column boxes
    int wstore;                  // per-warp output stores allowed (tmYw)
};

namespace dev {

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem].  kKind 0: kind::f16, A = bf16 packed 2 per
// TMEM column; kKind 1: kind::tf32, A = one fp32 (TF32-rounded) per column.
template <int kCG, int kKind>
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
    if constexpr (kCG == 1 && kKind == 0)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
            "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
    else if constexpr (kCG == 2 && kKind == 0)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
            "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
    else if constexpr (kCG == 1)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
            "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
            "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

template <int kCG, int kMode, int kKind = 0, bool kMask = false, bool kRS = false, bool kSP = false>
struct B2BCfg {
    // kKind 1 (TF32, fp32 I/O): a k-block is 32 fp32 (still 128 B per row, so
    // every smem tile / descriptor has the bf16 byte geometry); the output
    // staging doubles (fp32 tiles) and costs one stage.
    static_assert(kKind == 0 || kMode == 0, "the TF32 fused kernel streams packed panels (kMode 0)");
    static_assert(!kRS || (kCG == 2 && kKind == 0 && !kMask), "the R-split runs bf16 CTA pairs, no fused mask");
    static constexpr int kElem = kKind == 0 ? 2 : 4;
    static constexpr int kBK = 128 / kElem;                  // elements per k-block
    static constexpr int kOutBytes = kKind == 0 ? 16384 : 32768;  // per epilogue group
    // The backward's GEMM1 (K = d_out, 80% of its MMAs) runs single-pass: one
    // A1 tile feeds both 256-wide chunks, so G is read once instead of twice;
    // its stages therefore hold A1 + B1 for all of R (48 KB).  kSP does the same
    // for a forward whose x is long (K1 = d_in >= 2048: the c5 FFN2 layer, c4),
    // where the second pass would re-read a 1.5-2 MB x tile per pair that no
    // longer fits L2 with every pair streaming.
    static constexpr bool kSinglePassG1 = (kMode == 2 || kSP) && kCG == 2;
    static constexpr int kStageBytes = (kCG == 1 || kSinglePassG1) ? 48 * 1024 : 32 * 1024;
    // The forward keeps the whole bias (fp32, N2 <= kMaxBiasTab) resident in
    // smem and gives up one stage for it; its GEMM2 stages are 4 k-blocks deep.
    static constexpr bool kBiasTab = kMode == 1 && !kRS;
    static constexpr int kBiasTabBytes = kBiasTab ? 32 * 1024 : 0;
    static constexpr int kMaxBiasTab = kBiasTabBytes / 4;
    // kMask (backward with a fused ReLU mask): the mask tile of the next output
    // tile is TMA-loaded into smem one tile ahead (one kOutBytes buffer per
    // epilogue group); the ring gives up the stages that space takes.
    static constexpr bool kMaskStage = kMask;
    static constexpr int kMaskBytes = kMask ? 2 * kOutBytes : 0;
    // kRS: one 16 KB receive slot per epilogue warpgroup ([128 rows][32 fp32],
    // chunk-swizzled) for the running GEMM2 partial of the previous pair.
    static constexpr int kRecvBytes = kRS ? 2 * 16384 : 0;
    static constexpr int kStages = (kSinglePassG1 ? (kBiasTab ? 3 : 4) : (kCG == 1 ? 4 : 6) - (kBiasTab ? 1 : 0) - kKind) -
                                   (kMaskBytes + kRecvBytes + kStageBytes - 1) / kStageBytes;
    static constexpr int kAOff = 16384;                      // B1 offset inside a GEMM1 stage
    static constexpr int kRingBytes = kStages * kStageBytes;
    static constexpr int kB2Rows = 128 / kCG;               // B2 rows per CTA per 128-wide N tile
    static constexpr int kB2KbBytes = kB2Rows * 128;         // one 64-wide k-block of B2
    static constexpr int kKbPerStage2 = kStageBytes / kB2KbBytes;
    static constexpr int kB1BoxRows = 32;
    static constexpr int kSmem = kRingBytes + 2 * kOutBytes + 1024 /*bias ring*/ + kBiasTabBytes + kMaskBytes +
                                 kRecvBytes + 1024 /*align*/ + 512;
    static_assert(kStages >= 3, "operand ring too shallow");
    static_assert(kSmem <= 232448, "exceeds the 227 KB dynamic shared memory limit");
};

// kMode 0: B1 / B2 are packed K-major panels (any k).
// kMode 1: forward straight from the ABI stacks (k % 64 == 0): B1 = S1s|U2s
//          viewed as [L*d_in][k] (MN-major tiles), B2 = U1s|S2s viewed as
//          [L*k][d_out] (MN-major tiles).  No packing pass.
// kMode 2: backward straight from the stacks: B1 = U1s|S2s [L*k][d_out]
//          (K-major), B2 = S1s|U2s [L*d_in][k] (K-major, per-term row offset).
// kPost: 1 = the epilogue also applies the fused ReLU / ReLU mask (B2BArgs::relu /
// mask), 2 = the same with 1-bit masks (relu_bits / mask_bits); separate
// instantiations so the plain layer keeps its register budget.
template <int kCG, int kMode, int kKind, int kPost, bool kRS = false, bool kSP = false, bool kDT = false>
__global__ void __launch_bounds__(384, 1)
    b2b_kernel(const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
               const __grid_constant__ CUtensorMap tmB1b, const __grid_constant__ CUtensorMap tmB2,
               const __grid_constant__ CUtensorMap tmB2b, const __grid_constant__ CUtensorMap tmY,
               const __grid_constant__ CUtensorMap tmM, const __grid_constant__ CUtensorMap tmS,
               const __grid_constant__ CUtensorMap tmYw, B2BArgs args) {
    using C = B2BCfg<kCG, kMode, kKind, kPost == 1 && kMode != 1, kRS, kSP || kDT>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base_u32 - smem_u32(smem_raw));
    uint8_t* stage_out = smem + C::kRingBytes;                  // 2 x kOutBytes output staging
    float* bias_s = reinterpret_cast<float*>(stage_out + 2 * C::kOutBytes);  // 2 slots x 128 bias values
    float* bias_tab = reinterpret_cast<float*>(stage_out + 2 * C::kOutBytes + 1024);  // kMode 1: bias[N2]
    uint8_t* mask_s = stage_out + 2 * C::kOutBytes + 1024 + C::kBiasTabBytes;  // kMask: [2 groups][kOutBytes]
    uint8_t* recv_s = mask_s + C::kMaskBytes;                   // kRS: [2 groups][128 rows][32 fp32]
    uint64_t* bars = reinterpret_cast<uint64_t*>(recv_s + C::kRecvBytes);
    uint64_t* full = bars;                            // [kStages]
    uint64_t* empty = bars + C::kStages;              // [kStages]
    uint64_t* tfull1 = bars + 2 * C::kStages;         // [2] GEMM1 chunk accumulated
    uint64_t* hready = tfull1 + 2;                    // [2] chunk converted to bf16 H
    uint64_t* tfull2 = hready + 2;                    // [2] GEMM2 slot accumulated
    uint64_t* tempty2 = tfull2 + 2;                   // [2] GEMM2 slot drained
    uint64_t* mfull = tempty2 + 2;                    // [2] kMask: this group's mask tile landed
    uint64_t* rfull = mfull + 2;                      // [2] kRS: this group's receive slot holds a partial
    uint64_t* sfree = rfull + 2;                      // [2] kRS: the next pair's receive slot is free
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sfree + 2);

    const uint32_t warp = warp_id();
    // Cluster layout: pairs are CTA ranks (2p, 2p+1); kRS clusters hold nsplit pairs.
    const uint32_t crank = kCG == 2 ? cluster_ctarank() : 0;
    const uint32_t rank = crank & 1u;                 // rank inside the MMA pair
    const uint32_t lead = crank & ~1u;                // cluster rank of the pair's leader
    const uint16_t pmask = (uint16_t)(3u << lead);
    const bool leader = rank == 0;
    const int nsplit = kRS ? args.nsplit : 1;
    const int sp = kRS ? (int)(crank >> 1) : 0;       // this pair's R-slice
    const int r_loc = kRS ? args.r_loc : args.R_pad;  // R columns of this pair
    const int r_off = sp * r_loc;                     // ... starting at this rank index
    auto commit = [&](uint64_t* bar) {  // MMA completion -> both CTAs of this pair
        if constexpr (kCG == 2) mma_commit_pair(bar, pmask);
        else mma_commit<1>(bar);
    };

    if (warp == 0 && elect_one()) {
        prefetch_tmap(&tmA1);
        prefetch_tmap(&tmB1);
        prefetch_tmap(&tmB2);
        if constexpr (kMode != 0) {
            prefetch_tmap(&tmB1b);
            prefetch_tmap(&tmB2b);
        }
        prefetch_tmap(&tmY);
        if constexpr (kKind == 0) prefetch_tmap(&tmYw);
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], kCG);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull1[i], 1);
            mbar_init(&hready[i], 8 * kCG);   // 8 epilogue warps per CTA
            mbar_init(&tfull2[i], 1);
            mbar_init(&tempty2[i], 8 * kCG);
            mbar_init(&mfull[i], 1);
            mbar_init(&rfull[i], 4);          // the 4 sender warps of the previous pair's group
            mbar_init(&sfree[i], 4);          // the 4 receiver warps of the next pair's group
        }
        if constexpr (C::kMaskStage) prefetch_tmap(&tmM);
        if (args.save_tma) prefetch_tmap(&tmS);
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
    pdl_wait();  // inputs of this launch may come from the previous kernel in the stream
    pdl_launch_dependents();  // after the wait: a dependent starts only once our predecessor completed

    const int tile_rows = 128 * kCG;
    const int num_tiles = (args.T + tile_rows - 1) / tile_rows;
    const int cluster_id = blockIdx.x / (kCG * nsplit);
    const int num_clusters = gridDim.x / (kCG * nsplit);
    const int nch = (r_loc + 255) / 256;
    const int nkb1 = (args.K1 + C::kBK - 1) / C::kBK;
    const int nkb2 = r_loc / C::kBK;
    const int nst2 = (nkb2 + C::kKbPerStage2 - 1) / C::kKbPerStage2;
    const int n2_tiles = (args.N2 + 127) / 128;
    // Ping-pong H (R_pad <= 128): tile t's H lives in TMEM region (t & 1) * 128, so
    // GEMM1 of the next tile is issued BEFORE GEMM2 of this one and its HBM reads
    // overlap this tile's output drain (the epilogue's stores) instead of
    // alternating with it.  Producer, MMA issuer and epilogue all follow this order.
    const bool pp = nch == 1 && r_loc <= 128;

    if (warp == 0) {
        // ---------------------------------------------------------------- producer
        if (elect_one()) {
            Tr tr(0);
            int stage = 0;
            uint32_t phase = 0;
            // activations (x / G) stream through L2 once; the weight panels are re-read by every tile
            // (l2hint bit 0: activations evict_first when GEMM1 reads them once, bit 1: weights
            // evict_last; a two-pass GEMM1 re-reads its activation tile from L2, so it keeps the default)
            const int hint = args.l2hint;
            const uint64_t pol_norm = l2_evict_normal();
            const uint64_t pol_act = ((hint & 1) && (C::kSinglePassG1 || nch == 1)) ? l2_evict_first() : pol_norm;
            const uint64_t pol_w = (hint & 2) ? l2_evict_last() : pol_norm;
            auto next = [&]() { if (++stage == C::kStages) { stage = 0; phase ^= 1; } };
            auto load_g1 = [&](int t) {
                const int am = t * tile_rows + (int)rank * 128;
                // GEMM1 passes: one per chunk, or (single-pass mode) one pass that
                // feeds every chunk from the same A1 stage -> A1 is read once.
                const int npass = C::kSinglePassG1 ? 1 : nch;
                for (int pass = 0; pass < npass; ++pass) {
                    const int c_lo = C::kSinglePassG1 ? 0 : pass, c_hi = C::kSinglePassG1 ? nch : pass + 1;
                    uint32_t bytes = 16384;
                    for (int c = c_lo; c < c_hi; ++c) bytes += (min(256, r_loc - 256 * c) / kCG) * 128;
                    for (int kb = 0; kb < nkb1; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        tr(1);
                        uint8_t* st = smem + stage * C::kStageBytes;
                        if (leader) mbar_arrive_expect_tx(&full[stage], bytes * kCG);
                        else mbar_arrive_cluster(&full[stage], lead);
                        tma_load_2d_hint<kCG>(&tmA1, &full[stage], st, kb * C::kBK, am, pol_act);
                        for (int c = c_lo; c < c_hi; ++c) {
                            const int wc = min(256, r_loc - 256 * c);
                            const int brows = wc / kCG;
                            const int b0 = r_off + 256 * c + (int)rank * brows;  // global rank index
                            uint8_t* bst = st + C::kAOff + (c - c_lo) * (256 / kCG) * 128;
                            if constexpr (kMode == 0) {
                                for (int r = 0; r < brows; r += args.b1rows)
                                    tma_load_2d_hint<kCG>(&tmB1, &full[stage], bst + r * 128, kb * C::kBK, b0 + r, pol_w);
                            } else if constexpr (kMode == 2) {  // rows of [U1s ; S2s]
                                for (int r = 0; r < brows; r += args.b1rows) {
                                    const int rg = b0 + r;
                                    tma_load_2d_hint<kCG>(rg < args.Lk ? &tmB1 : &tmB1b, &full[stage], bst + r * 128, kb * 64,
                                                     rg < args.Lk ? rg : rg - args.Lk, pol_w);
                                }
                            } else {  // MN-major [64 d_in rows x 64 rank cols] blocks of S1s | U2s
                                for (int jb = 0; jb < brows / 64; ++jb) {
                                    const int rg = b0 + 64 * jb;
                                    const int rr = rg < args.Lk ? rg : rg - args.Lk;
                                    tma_load_2d_hint<kCG>(rg < args.Lk ? &tmB1 : &tmB1b, &full[stage], bst + jb * 8192,
                                                     rr % args.k, (rr / args.k) * args.dS + kb * 64, pol_w);
                                }
                            }
                        }
                        next();
                    }
                }
            };
            auto load_g2 = [&]() {
                for (int j = 0; j < n2_tiles; ++j) {
                    const int brow = j * 128 + (int)rank * C::kB2Rows;
                    for (int s = 0; s < nst2; ++s) {
                        const int kb0 = s * C::kKbPerStage2;
                        const int nk = min(C::kKbPerStage2, nkb2 - kb0);
                        mbar_wait(&empty[stage], phase ^ 1);
                        tr(2);
                        uint8_t* st = smem + stage * C::kStageBytes;
                        if (leader) mbar_arrive_expect_tx(&full[stage], (uint32_t)(nk * C::kB2KbBytes * kCG));
                        else mbar_arrive_cluster(&full[stage], lead);
                        for (int q = 0; q < nk; ++q) {
                            const int r0 = r_off + (kb0 + q) * C::kBK;  // global rank index of this k-block
                            if constexpr (kMode == 0) {
                                tma_load_2d_hint<kCG>(&tmB2, &full[stage], st + q * C::kB2KbBytes, r0, brow, pol_w);
                            } else if constexpr (kMode == 1) {  // MN-major rows of [U1s ; S2s]
                                const CUtensorMap* m = r0 < args.Lk ? &tmB2 : &tmB2b;
                                const int rr = r0 < args.Lk ? r0 : r0 - args.Lk;
                                for (int jb = 0; jb < C::kB2Rows / 64; ++jb)
                                    tma_load_2d_hint<kCG>(m, &full[stage], st + q * C::kB2KbBytes + jb * 8192, brow + 64 * jb, rr, pol_w);
                            } else {  // K-major [d_in rows x 64 rank cols] of S1s | U2s, term row offset
                                const int rr = r0 < args.Lk ? r0 : r0 - args.Lk;
                                tma_load_2d_hint<kCG>(r0 < args.Lk ? &tmB2 : &tmB2b, &full[stage], st + q * C::kB2KbBytes,
                                                 rr % args.k, (rr / args.k) * args.dS + brow, pol_w);
                            }
                        }
                        next();
                    }
                }
            };
            if constexpr (kDT) {
                // Double tiles (R = 256): a GEMM1 stage holds the A tiles of two pair
                // tiles (2u, 2u + 1) around one B1 k-block, so every weight byte
                // brought in feeds twice the MMAs (the weight panels are two thirds of
                // a 768x768 projection tile's operand traffic).
                const int ndt = (num_tiles + 1) / 2;
                for (int u = cluster_id; u < ndt; u += num_clusters) {
                    for (int kb = 0; kb < nkb1; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        tr(1);
                        uint8_t* st = smem + stage * C::kStageBytes;
                        if (leader) mbar_arrive_expect_tx(&full[stage], 3u * 16384u * kCG);
                        else mbar_arrive_cluster(&full[stage], lead);
                        tma_load_2d_hint<kCG>(&tmA1, &full[stage], st, kb * C::kBK, 2 * u * tile_rows + (int)rank * 128,
                                              pol_act);
                        tma_load_2d_hint<kCG>(&tmA1, &full[stage], st + 32768, kb * C::kBK,
                                              (2 * u + 1) * tile_rows + (int)rank * 128, pol_act);
                        const int brows = 256 / kCG, b0 = (int)rank * brows;
                        uint8_t* bst = st + C::kAOff;
                        if constexpr (kMode == 2) {  // rows of [U1s ; S2s]
                            for (int r = 0; r < brows; r += args.b1rows) {
                                const int rg = b0 + r;
                                tma_load_2d_hint<kCG>(rg < args.Lk ? &tmB1 : &tmB1b, &full[stage], bst + r * 128, kb * 64,
                                                      rg < args.Lk ? rg : rg - args.Lk, pol_w);
                            }
                        } else {  // MN-major [64 d_in rows x 64 rank cols] blocks of S1s | U2s
                            for (int jb = 0; jb < brows / 64; ++jb) {
                                const int rg = b0 + 64 * jb;
                                const int rr = rg < args.Lk ? rg : rg - args.Lk;
                                tma_load_2d_hint<kCG>(rg < args.Lk ? &tmB1 : &tmB1b, &full[stage], bst + jb * 8192,
                                                      rr % args.k, (rr / args.k) * args.dS + kb * 64, pol_w);
                            }
                        }
                        next();
                    }
                    load_g2();
                }
            } else {
            if (pp && cluster_id < num_tiles) load_g1(cluster_id);
            for (int t = cluster_id; t < num_tiles; t += num_clusters) {
                if (!pp) load_g1(t);
                else if (t + num_clusters < num_tiles) load_g1(t + num_clusters);
                load_g2();
            }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA issuer
        if (leader && elect_one()) {
            Tr tr(1);
            int stage = 0;
            uint32_t phase = 0;
            auto next = [&]() { if (++stage == C::kStages) { stage = 0; phase ^= 1; } };
            uint32_t slot_seq = 0;
            const uint32_t idesc2 = make_idesc(kKind, 128 * kCG, 128, 0, kMode == 1 ? 1 : 0);
            int it = 0;
            auto issue_g1 = [&](uint32_t hoff, int r) {  // hoff: TMEM column of this tile's H (ping-pong)
                // ---- GEMM1: H chunks (one pass per chunk, or one pass for all)
                const int npass = C::kSinglePassG1 ? 1 : nch;
                for (int pass = 0; pass < npass; ++pass) {
                    const int c_lo = C::kSinglePassG1 ? 0 : pass, c_hi = C::kSinglePassG1 ? nch : pass + 1;
                    if (c_hi > 1 && c_lo <= 1) {  // chunk 1 overlays both GEMM2 slots
                        for (int u = 0; u < 2; ++u, ++slot_seq)
                            mbar_wait(&tempty2[slot_seq & 1], ((slot_seq >> 1) & 1) ^ 1);
                        tc_fence_after();
                        tr(10);
                    }
                    for (int kb = 0; kb < nkb1; ++kb) {
                        mbar_wait(&full[stage], phase);
                        tr(11);
                        tc_fence_after();
                        const uint32_t a_addr = smem_u32(smem + stage * C::kStageBytes);
                        for (int c = c_lo; c < c_hi; ++c) {
                            const int wc = min(256, r_loc - 256 * c);
                            const uint32_t idesc1 = make_idesc(kKind, 128 * kCG, wc, 0, kMode == 1 ? 1 : 0);
                            const uint32_t d = tmem_base + 256 * c + hoff;
                            const uint32_t b_addr = a_addr + C::kAOff + (c - c_lo) * (256 / kCG) * 128;
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                mma_ss<kCG, kKind>(d, make_sdesc(a_addr + k * 32, 0, 1024),
                                               kMode == 1 ? make_sdesc(b_addr + k * 2048, 8192, 1024)
                                                          : make_sdesc(b_addr + k * 32, 0, 1024),
                                               idesc1, (kb > 0 || k > 0) ? 1u : 0u);
                        }
                        commit(&empty[stage]);
                        next();
                    }
                    for (int c = c_lo; c < c_hi; ++c) commit(&tfull1[pp ? r : c]);
                }
            };
            auto issue_g2 = [&](uint32_t hoff) {
                // ---- GEMM2: 128-wide output tiles, A = H from TMEM
                for (int j = 0; j < n2_tiles; ++j, ++slot_seq) {
                    const uint32_t s = slot_seq & 1;
                    mbar_wait(&tempty2[s], ((slot_seq >> 1) & 1) ^ 1);
                    tr(13);
                    tc_fence_after();
                    const uint32_t d = tmem_base + 256 + 128 * s;
                    for (int st2 = 0; st2 < nst2; ++st2) {
                        const int kb0 = st2 * C::kKbPerStage2;
                        const int nk = min(C::kKbPerStage2, nkb2 - kb0);
                        mbar_wait(&full[stage], phase);
                        tr(14);
                        tc_fence_after();
                        const uint32_t b_addr = smem_u32(smem + stage * C::kStageBytes);
                        for (int q = 0; q < nk; ++q) {
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const uint32_t a_t = tmem_base + hoff + (uint32_t)((kb0 + q) * 32 + k * 8);
                                const uint64_t bdesc = kMode == 1
                                    ? make_sdesc(b_addr + q * C::kB2KbBytes + k * 2048, 8192, 1024)
                                    : make_sdesc(b_addr + q * C::kB2KbBytes + k * 32, 0, 1024);
                                mma_ts<kCG, kKind>(d, a_t, bdesc, idesc2, (st2 > 0 || q > 0 || k > 0) ? 1u : 0u);
                            }
                        }
                        commit(&empty[stage]);
                        next();
                    }
                    commit(&tfull2[s]);
                }
            };
            if constexpr (kDT) {
                // Double tiles: TMEM [0, 256) and [256, 512) take tile a's and tile b's
                // GEMM1 (fp32), compacted to H_a = [0, 128), H_b = [256, 384); GEMM2 of
                // each output column tile accumulates a in [128, 256) and b in [384, 512)
                // from the same B2 stage.  Each slot's drains are waited exactly once, in
                // order: by the next output tile, the last one by the next double tile's
                // GEMM1 (which overwrites the whole of TMEM).
                const uint32_t idesc1 = make_idesc(kKind, 128 * kCG, 256, 0, kMode == 1 ? 1 : 0);
                uint32_t dwait[2] = {0u, 0u};
                auto wait_drain = [&](int h) {
                    mbar_wait(&tempty2[h], dwait[h] & 1);
                    ++dwait[h];
                };
                const int ndt = (num_tiles + 1) / 2;
                for (int u = cluster_id; u < ndt; u += num_clusters, ++it) {
                    if (it > 0) {
                        wait_drain(0);
                        wait_drain(1);
                        tc_fence_after();
                    }
                    for (int kb = 0; kb < nkb1; ++kb) {
                        mbar_wait(&full[stage], phase);
                        tr(11);
                        tc_fence_after();
                        const uint32_t a_addr = smem_u32(smem + stage * C::kStageBytes);
                        const uint32_t b_addr = a_addr + C::kAOff;
#pragma unroll
                        for (int h = 0; h < 2; ++h)
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                mma_ss<kCG, kKind>(tmem_base + 256u * h, make_sdesc(a_addr + 32768u * h + k * 32, 0, 1024),
                                                   kMode == 1 ? make_sdesc(b_addr + k * 2048, 8192, 1024)
                                                              : make_sdesc(b_addr + k * 32, 0, 1024),
                                                   idesc1, (kb > 0 || k > 0) ? 1u : 0u);
                        commit(&empty[stage]);
                        next();
                    }
                    commit(&tfull1[0]);
                    commit(&tfull1[1]);
                    mbar_wait(&hready[0], it & 1);
                    mbar_wait(&hready[1], it & 1);
                    tr(12);
                    tc_fence_after();
                    for (int j = 0; j < n2_tiles; ++j) {
                        if (j > 0) {
                            wait_drain(0);
                            wait_drain(1);
                            tc_fence_after();
                        }
                        for (int st2 = 0; st2 < nst2; ++st2) {
                            const int kb0 = st2 * C::kKbPerStage2;
                            const int nk = min(C::kKbPerStage2, nkb2 - kb0);
                            mbar_wait(&full[stage], phase);
                            tr(14);
                            tc_fence_after();
                            const uint32_t b_addr = smem_u32(smem + stage * C::kStageBytes);
#pragma unroll
                            for (int h = 0; h < 2; ++h)
                                for (int q = 0; q < nk; ++q) {
#pragma unroll
                                    for (int k = 0; k < 4; ++k) {
                                        const uint32_t a_t = tmem_base + 256u * h + (uint32_t)((kb0 + q) * 32 + k * 8);
                                        const uint64_t bdesc = kMode == 1
                                            ? make_sdesc(b_addr + q * C::kB2KbBytes + k * 2048, 8192, 1024)
                                            : make_sdesc(b_addr + q * C::kB2KbBytes + k * 32, 0, 1024);
                                        mma_ts<kCG, kKind>(tmem_base + 256u * h + 128u, a_t, bdesc, idesc2,
                                                           (st2 > 0 || q > 0 || k > 0) ? 1u : 0u);
                                    }
                                }
                            commit(&empty[stage]);
                            next();
                        }
                        commit(&tfull2[0]);
                        commit(&tfull2[1]);
                    }
                }
            } else {
            if (pp && cluster_id < num_tiles) issue_g1(0, 0);
            for (int t = cluster_id; t < num_tiles; t += num_clusters, ++it) {
                if (!pp) issue_g1(0, 0);
                else if (t + num_clusters < num_tiles) issue_g1(128u * ((it + 1) & 1), (it + 1) & 1);
                // ---- wait for the bf16 H of this tile (both CTAs)
                if (pp) mbar_wait(&hready[it & 1], (it >> 1) & 1);
                else for (int c = 0; c < nch; ++c) mbar_wait(&hready[c], it & 1);
                tr(12);
                tc_fence_after();
                issue_g2(pp ? 128u * (it & 1) : 0u);
            }
            }
        }
    } else if (warp >= 4) {
        // ---------------------------------------------------------------- epilogue
        // Two warpgroups (warps 4-7, 8-11).  A warp may only touch its TMEM lane
        // quarter (warp % 4), so both groups cover all 128 rows and split the
        // columns: group wg converts / stores columns [wg*W/2, (wg+1)*W/2) of
        // every GEMM1 chunk and GEMM2 tile.
        const uint32_t q = warp & 3;
        const uint32_t wg = (warp - 4) >> 2;
        const uint32_t lane = lane_id();
        const uint32_t lane_base = (q * 32u) << 16;
        const uint32_t srow = q * 32 + lane;  // TMEM lane == tile row
        uint32_t slot_seq = 0;
        uint32_t tf_par0 = 0, tf_par1 = 0;
        uint32_t xch = 0;                     // kRS: partial hand-offs of this group so far
        Tr tr((lane == 0 && wg == 0 && (q == 0 || q == 3)) ? 2 + (q == 3 ? 1 : 0) : -1);
        const bool issuer = (q == 0 && lane == 0);  // per group: issues / waits its bulk stores
        // Per-warp output stores (bf16, no fused mask, bias resident or absent): each
        // warp writes its 32 rows of the output tile with its own TMA store and
        // waits only for its own previous store, so the two group barriers per
        // output tile go away (the 768x768 projection's GEMM2 is epilogue-bound).
        // Otherwise the group shares one store per tile (staged bias / mask tiles
        // are published by the group barrier).
        uint8_t* buf = stage_out + wg * C::kOutBytes;  // this group's output staging buffer
        uint8_t* mbuf = mask_s + wg * C::kOutBytes;    // kMask: this group's mask tile (same layout as buf)
        uint32_t mph = 0;
        const bool use_mask = C::kMaskStage && args.mask != nullptr;
        const bool use_bits_in = kPost == 2 && args.mask_bits != nullptr;
        const bool use_bits_out = kPost == 2 && args.relu_bits != nullptr;
        const bool wstore = kKind == 0 && args.wstore && !use_mask && (C::kBiasTab || args.bias == nullptr);
        const bool storer = wstore ? lane == 0 : issuer;  // threads that own bulk stores
        uint2 mbits = make_uint2(0u, 0u), mbits_next = make_uint2(0u, 0u);
        // mask tile of output tile (t, j) for this group's 64 columns -> mbuf (issuer only)
        auto issue_mask = [&](int t_, int j_) {
            const int mn0 = j_ * 128 + 64 * (int)wg, mr0 = t_ * tile_rows + (int)rank * 128;
            mbar_arrive_expect_tx(&mfull[wg], C::kOutBytes);
            tma_load_2d<1>(&tmM, &mfull[wg], mbuf, mn0, mr0);
            if constexpr (kKind == 1) tma_load_2d<1>(&tmM, &mfull[wg], mbuf + 16384, mn0 + 32, mr0);
        };
        float* bias_g = bias_s + wg * 128;            // [2 slots][64]
        auto load_bias_col = [&](int col) -> float {
            if (args.bias == nullptr || col >= args.N2) return 0.f;
            return args.bias_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(args.bias)[col])
                                  : __ldg(args.bias + col);
        };
        float bias_pref = 0.f;
        if constexpr (C::kBiasTab) {
            // whole bias resident in smem for the kernel's lifetime
            const int tid = (int)((warp - 4) * 32 + lane);
            for (int i = tid; i < args.N2; i += 256) bias_tab[i] = load_bias_col(i);
            named_bar_sync(3, 256);
        } else {
            bias_pref = load_bias_col((int)(wg * 64 + (srow & 63)));  // tile j = 0
        }
        const float alpha = args.alpha;
        auto arrive_leader = [&](uint64_t* bar) {
            if (leader) mbar_arrive(bar);
            else mbar_arrive_cluster(bar, lead);
        };
        // The backward's single-pass GEMM1 finishes both H chunks at once, so the
        // MMA idles while they convert: there the saved columns (P_S2) are written
        // AFTER hready, from the bf16 H in TMEM, under the first GEMM2 MMAs.  The
        // next tile's GEMM1 cannot overwrite H before that: its pass first waits
        // for both GEMM2 slots, which this group releases only after its drain.
        // Same for a single chunk (R <= 256): its conversion has no other chunk's
        // GEMM1 to hide under.  Needs >= 3 GEMM2 tiles, so that the MMA issuer
        // has waited on a slot this group released after its saves before it
        // issues the next tile's GEMM1 (which overwrites, or -- ping-pong -- is
        // followed by a GEMM1 that overwrites, this H).
        const bool defer_save = kKind == 0 && ((C::kSinglePassG1 && nch == 2) || (nch == 1 && n2_tiles >= 3));
        int cur_t = 0;
        // Saved columns go out TRANSPOSED, save[c - save_col0][t] (row stride
        // ld_save = round8(T)): the token-reduction GEMMs then read them K-major.
        // Each warp owns a 4 KB slice of the group's staging buffer (its 32
        // tokens).  `col` is the global rank index (r_off + the pair-local column).
        uint8_t* wbuf = buf + q * 4096;
        bool save_pend = false;  // this warp's TMA save store may still be reading wbuf
        auto reclaim_wbuf = [&]() {  // before wbuf is written again
            if (save_pend) {
                if (lane == 0) bulk_wait_read<0>();
                __syncwarp();
                save_pend = false;
            }
        };
        // Fallback (columns straddling the save window, TF32-free shapes whose
        // quarters are not 64 wide): the warp's [32 tokens x 16 cols] block is
        // transposed through wbuf so every lane writes two 16-B chunks (8 tokens
        // of one column) instead of 16 scattered 2-B stores.
        auto save_cols16 = [&](const uint32_t (&p)[8], int col) {
            reclaim_wbuf();
            const __nv_bfloat16* pb = reinterpret_cast<const __nv_bfloat16*>(p);
            __nv_bfloat16* scr = reinterpret_cast<__nv_bfloat16*>(wbuf);  // [16 cols][32 tokens]
#pragma unroll
            for (int i = 0; i < 16; ++i) scr[i * 32 + lane] = pb[i];
            __syncwarp();
            const long long tok0 = (long long)cur_t * tile_rows + (int)rank * 128 + q * 32;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int id = (int)lane * 2 + hh, i = id >> 2, j = id & 3;
                const long long tok = tok0 + 8 * j;
                if (col + i >= args.save_col0 && col + i < args.save_col0 + args.save_cols && tok < args.ld_save) {
                    const uint4 v = *reinterpret_cast<const uint4*>(scr + i * 32 + 8 * j);
                    *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(args.save) +
                                              (long long)(col + i - args.save_col0) * args.ld_save + tok) = v;
                }
            }
            __syncwarp();
        };
        // TMA route (bf16, 64-column quarters inside the save window): the warp
        // stages its [64 cols][32 tokens] block in wbuf (64-B rows; lane pairs
        // swap halves so each lane stores two tokens of one column, even lanes
        // filling one row and odd lanes the next: 128 B per store, no bank
        // conflict) and lane 0 issues one TMA store of it.  The async engine then
        // does the strided writes the threads did one 16-B chunk at a time
        // (3.8k cycles per tile of the 768x768 projection, 7k of the c2 backward).
        auto quarter_tma = [&](int col, int W) -> bool {
            return kKind == 0 && args.save_tma && W == 64 && col >= args.save_col0 &&
                   col + 64 <= args.save_col0 + args.save_cols;
        };
        auto stage16 = [&](const uint32_t (&p)[8], int j) {  // columns [16j, 16j + 16) of the quarter
            const bool odd = lane & 1u;
            const uint32_t a = smem_u32(wbuf) + (uint32_t)(16 * j + (odd ? 1 : 0)) * 64u + (lane & ~1u) * 2u;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t x = __shfl_xor_sync(0xffffffffu, p[i], 1);
                // even lane: column 2i of tokens (lane, lane+1); odd lane: column 2i+1 of (lane-1, lane)
                const uint32_t w = odd ? ((x >> 16) | (p[i] & 0xFFFF0000u)) : ((p[i] & 0xFFFFu) | (x << 16));
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(a + (uint32_t)(2 * i) * 64u), "r"(w));
            }
        };
        auto flush_quarter = [&](int col) {  // the warp staged its 32 rows of the quarter
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                tma_store_2d(&tmS, wbuf, cur_t * tile_rows + (int)rank * 128 + (int)q * 32, col - args.save_col0);
                bulk_commit();
            }
            save_pend = true;
        };
        // kRS: add the running partial of the previous pair (if any) to this
        // group's 32 accumulator columns `r`, then pass the sum to the next pair
        // (if any).  Partials move fp32 through one [128 rows][32] slot per
        // group, 16-B chunk j of row srow at j ^ (srow & 7): each thread reads
        // back exactly the row the same-index thread of the previous pair wrote.
        auto chain_reduce = [&](uint32_t (&r)[32]) {
            const uint32_t slot = smem_u32(recv_s) + wg * 16384 + srow * 128;
            if (sp > 0) {
                mbar_wait_cluster(&rfull[wg], xch & 1);
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    uint32_t v[4];
                    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                                 : "r"(slot + ((uint32_t)(jj ^ (srow & 7)) << 4)));
#pragma unroll
                    for (int i = 0; i < 4; ++i)  // (D_0 + ... + D_{sp-1}) + D_sp
                        r[4 * jj + i] = __float_as_uint(__uint_as_float(v[i]) + __uint_as_float(r[4 * jj + i]));
                }
                __syncwarp();
                if (lane == 0) mbar_arrive_remote_release(&sfree[wg], crank - 2);  // slot consumed
            }
            if (sp + 1 < nsplit) {
                mbar_wait_cluster(&sfree[wg], (xch & 1) ^ 1);  // the next pair's slot is free
#pragma unroll
                for (int jj = 0; jj < 8; ++jj)
                    st_dsmem_v4(slot + ((uint32_t)(jj ^ (srow & 7)) << 4), crank + 2, r[4 * jj], r[4 * jj + 1],
                                r[4 * jj + 2], r[4 * jj + 3]);
                __syncwarp();
                if (lane == 0) mbar_arrive_remote_release(&rfull[wg], crank + 2);
            }
            ++xch;
        };
        if constexpr (kDT) {
            // Double tiles (see the MMA issuer): convert both halves, save their
            // columns (from the bf16 H), then per output column tile drain slot a and
            // slot b.  Per-warp stores; the bias, when any, is the resident table.
            int it = 0;
            uint32_t tpar[2] = {0u, 0u};
            const int ndt = (num_tiles + 1) / 2;
            for (int u = cluster_id; u < ndt; u += num_clusters, ++it) {
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {
                    const uint32_t hoff = 256u * (uint32_t)h;
                    mbar_wait(&tfull1[h], it & 1);
                    tr(21);
                    tc_fence_after();
#pragma unroll 1
                    for (int rd = 0; rd < 2; ++rd) {  // in-place compaction as in the one-tile path (W = 64)
                        const int qi = 2 * rd + (int)wg;
                        uint32_t rr[4][16];
#pragma unroll
                        for (int g = 0; g < 4; ++g) tmem_ld16(tmem_base + lane_base + hoff + qi * 64 + 16 * g, rr[g]);
                        tmem_ld_wait();
                        if (rd == 0) {
                            tc_fence_before();
                            named_bar_sync(3, 256);
                            tc_fence_after();
                        }
#pragma unroll
                        for (int g = 0; g < 4; ++g) {
                            uint32_t pk[8];
#pragma unroll
                            for (int i = 0; i < 8; ++i)
                                pk[i] = pack_bf16x2(__uint_as_float(rr[g][2 * i]), __uint_as_float(rr[g][2 * i + 1]));
                            tmem_st8(tmem_base + lane_base + hoff + (qi * 64 + 16 * g) / 2, pk);
                        }
                    }
                    tmem_st_wait();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        tr(22);
                        arrive_leader(&hready[h]);
                    }
                }
                if (args.save) {  // saved columns of both halves, under the first GEMM2 MMAs
                    if (storer) bulk_wait_read<0>();
                    named_bar_sync(1 + wg, 128);
                    save_pend = false;
#pragma unroll 1
                    for (int h = 0; h < 2; ++h) {
                        cur_t = 2 * u + h;
#pragma unroll 1
                        for (int rd = 0; rd < 2; ++rd) {
                            const int qi = 2 * rd + (int)wg, qcol = qi * 64;
                            if (!(qcol + 64 > args.save_col0 && qcol < args.save_col0 + args.save_cols)) continue;
                            if (quarter_tma(qcol, 64)) {
                                reclaim_wbuf();
                                uint32_t pq[4][8];
#pragma unroll
                                for (int g = 0; g < 4; ++g)
                                    tmem_ld8(tmem_base + lane_base + 256u * h + (qcol + 16 * g) / 2, pq[g]);
                                tmem_ld_wait();
#pragma unroll
                                for (int g = 0; g < 4; ++g) stage16(pq[g], g);
                                flush_quarter(qcol);
                                continue;
                            }
#pragma unroll 1
                            for (int g = 0; g < 4; ++g) {
                                const int col = qcol + 16 * g;
                                if (!(col + 16 > args.save_col0 && col < args.save_col0 + args.save_cols)) continue;
                                uint32_t pk[8];
                                tmem_ld8(tmem_base + lane_base + 256u * h + col / 2, pk);
                                tmem_ld_wait();
                                save_cols16(pk, col);
                            }
                        }
                    }
                }
                tr(23);
#pragma unroll 1
                for (int j = 0; j < n2_tiles; ++j) {
                    const int n0 = j * 128 + 64 * (int)wg;
#pragma unroll 1
                    for (int h = 0; h < 2; ++h) {
                        mbar_wait(&tfull2[h], tpar[h]);
                        tpar[h] ^= 1u;
                        tr(24);
                        tc_fence_after();
                        uint32_t ra[32], rb[32];
                        const uint32_t scol = 256u * h + 128u + 64u * wg;
                        tmem_ld32(tmem_base + lane_base + scol, ra);
                        tmem_ld32(tmem_base + lane_base + scol + 32, rb);
                        tmem_ld_wait();
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) arrive_leader(&tempty2[h]);
                        if (lane == 0) bulk_wait_read<0>();  // this warp's previous stores have read `buf`
                        save_pend = false;
                        __syncwarp();
                        const uint32_t row_addr = smem_u32(buf) + srow * 128;
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            float4 b0 = make_float4(0.f, 0.f, 0.f, 0.f), b1 = b0;
                            if constexpr (C::kBiasTab) {
                                b0 = reinterpret_cast<const float4*>(bias_tab + n0 + 8 * c)[0];
                                b1 = reinterpret_cast<const float4*>(bias_tab + n0 + 8 * c)[1];
                            }
                            const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                            const uint32_t* src = (c < 4) ? ra : rb;
                            const int o = (c & 3) * 8;
                            uint32_t w[4];
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                w[i] = pack_bf16x2(fmaf(__uint_as_float(src[o + 2 * i]), alpha, bv[2 * i]),
                                                   fmaf(__uint_as_float(src[o + 2 * i + 1]), alpha, bv[2 * i + 1]));
                            st_shared_v4(row_addr + ((uint32_t)(c ^ (srow & 7)) << 4), w[0], w[1], w[2], w[3]);
                        }
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_2d(&tmYw, buf + q * 4096, n0, (2 * u + h) * tile_rows + (int)rank * 128 + (int)q * 32);
                            bulk_commit();
                        }
                        tr(26);
                    }
                }
            }
        } else {
        int it = 0;
        for (int t = cluster_id; t < num_tiles; t += num_clusters, ++it) {
            cur_t = t;
            const int row = t * tile_rows + (int)rank * 128 + (int)srow;
            const bool row_ok = row < args.T;
            if (use_mask && issuer) issue_mask(t, 0);  // lands during the GEMM1 conversion
            // this row's mask bits of output tile jj, this group's 64 columns (one 8-B load)
            auto load_bits = [&](int jj) -> uint2 {
                const int col = jj * 128 + 64 * (int)wg;
                if (!row_ok || col >= args.N2) return make_uint2(0u, 0u);
                return __ldg(reinterpret_cast<const uint2*>(args.mask_bits + (long long)row * args.bits_ld + col / 32));
            };
            if (use_bits_in) mbits_next = load_bits(0);
            // ---- convert GEMM1 chunks: fp32 -> bf16 H in TMEM (+ saved columns)
            for (int c = 0; c < nch; ++c) {
                const int wc = min(256, r_loc - 256 * c);
                // In-place fp32 -> bf16 compaction, split over both warpgroups in
                // two rounds of quarter-chunks (W = wc/4 columns each).  Quarter qi
                // lands in fp32 columns [qi*W/2, (qi+1)*W/2), i.e. inside quarters
                // 0/1, so round 0 reads Q0,Q1 before anyone writes (barrier), and
                // round 1's writes only hit Q1, which round 0 already consumed.
                const int W = wc / 4;
                const int hb = pp ? (int)(it & 1) : c;            // tfull1 / hready index
                const uint32_t hoff = pp ? 128u * (it & 1) : 0u;  // TMEM column of this tile's H
                mbar_wait(&tfull1[hb], pp ? ((it >> 1) & 1) : (it & 1));
                tr(21);
                tc_fence_after();
                if constexpr (kKind == 1) {
                    // TF32: H stays one fp32 word per column; round in place with
                    // cvt.rna, group wg owns columns [wg*wc/2, (wg+1)*wc/2).
#pragma unroll 1
                    for (int cl = (int)wg * (wc / 2); cl < ((int)wg + 1) * (wc / 2); cl += 16) {
                        uint32_t r[16];
                        tmem_ld16(tmem_base + lane_base + hoff + 256 * c + cl, r);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(tf32_rna(__uint_as_float(r[i])));
                        uint32_t lo[8], hi[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) { lo[i] = r[i]; hi[i] = r[8 + i]; }
                        tmem_st8(tmem_base + lane_base + hoff + 256 * c + cl, lo);
                        tmem_st8(tmem_base + lane_base + hoff + 256 * c + cl + 8, hi);
                        const int col = r_off + 256 * c + cl;
                        if (args.save && row_ok && col + 16 > args.save_col0 && col < args.save_col0 + args.save_cols) {
                            float* dst = reinterpret_cast<float*>(args.save) + row;
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (col + i >= args.save_col0 && col + i < args.save_col0 + args.save_cols)
                                    dst[(long long)(col + i - args.save_col0) * args.ld_save] = __uint_as_float(r[i]);
                        }
                    }
                } else {
                if (args.save && !defer_save) {  // buf doubles as the transpose scratch: the last store must have left it
                    if (storer) bulk_wait_read<0>();
                    named_bar_sync(1 + wg, 128);
                }
#pragma unroll 1
                for (int rd = 0; rd < 2; ++rd) {
                    const int qi = 2 * rd + (int)wg;
                    const bool qt = args.save && !defer_save && quarter_tma(r_off + 256 * c + qi * W, W);
                    if (qt) reclaim_wbuf();
                    uint32_t rr[4][16];
#pragma unroll
                    for (int g = 0; g < 4; ++g)
                        if (16 * g < W) tmem_ld16(tmem_base + lane_base + hoff + 256 * c + qi * W + 16 * g, rr[g]);
                    tmem_ld_wait();
                    if (rd == 0) {
                        tc_fence_before();
                        named_bar_sync(3, 256);  // both groups hold Q0/Q1 in registers
                        tc_fence_after();
                    }
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        if (16 * g >= W) break;
                        const uint32_t(&r)[16] = rr[g];
                        uint32_t p[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            p[i] = pack_bf16x2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
                        const int cl = qi * W + 16 * g;  // chunk-local fp32 column
                        tmem_st8(tmem_base + lane_base + hoff + 128 * c + cl / 2, p);
                        const int col = r_off + 256 * c + cl;  // H column (global R order)
                        if (qt)
                            stage16(p, g);
                        else if (args.save && !defer_save && col + 16 > args.save_col0 &&
                                 col < args.save_col0 + args.save_cols)
                            save_cols16(p, col);
                    }
                    if (qt) flush_quarter(r_off + 256 * c + qi * W);
                }
                }  // bf16 conversion
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    tr(22);
                    arrive_leader(&hready[hb]);
                    if (c == 1) {  // release the two slots chunk 1 overlaid
                        arrive_leader(&tempty2[slot_seq & 1]);
                        arrive_leader(&tempty2[(slot_seq + 1) & 1]);
                    }
                }
                if (c == 1) slot_seq += 2;
            }
            if (defer_save && args.save) {  // saved columns from the bf16 H, under the first GEMM2 MMAs
                if (storer) bulk_wait_read<0>();  // buf is the transpose scratch
                named_bar_sync(1 + wg, 128);
                for (int c = 0; c < nch; ++c) {
                    const int W = min(256, r_loc - 256 * c) / 4;
#pragma unroll 1
                    for (int rd = 0; rd < 2; ++rd) {
                        const int qi = 2 * rd + (int)wg;
                        const int qcol = r_off + 256 * c + qi * W;
                        if (!(qcol + W > args.save_col0 && qcol < args.save_col0 + args.save_cols)) continue;
                        tr(27);
                        if (quarter_tma(qcol, W)) {
                            reclaim_wbuf();
                            uint32_t pq[4][8];
#pragma unroll
                            for (int g = 0; g < 4; ++g)
                                tmem_ld8(tmem_base + lane_base + (pp ? 128u * (it & 1) : 0u) + 128 * c + (qi * W + 16 * g) / 2, pq[g]);
                            tmem_ld_wait();
                            tr(28);
#pragma unroll
                            for (int g = 0; g < 4; ++g) stage16(pq[g], g);
                            tr(29);
                            flush_quarter(qcol);
                            tr(30);
                            continue;
                        }
#pragma unroll 1
                        for (int g = 0; g < 4 && 16 * g < W; ++g) {
                            const int cl = qi * W + 16 * g, col = r_off + 256 * c + cl;
                            if (!(col + 16 > args.save_col0 && col < args.save_col0 + args.save_cols)) continue;
                            uint32_t p[8];
                            tmem_ld8(tmem_base + lane_base + (pp ? 128u * (it & 1) : 0u) + 128 * c + cl / 2, p);
                            tmem_ld_wait();
                            save_cols16(p, col);
                        }
                    }
                }
            }
            tr(23);
            // ---- GEMM2 output tiles: this group's 64 columns of every 128-wide tile
            for (int j = 0; j < n2_tiles; ++j, ++slot_seq) {
                const uint32_t s = slot_seq & 1;
                // Bias through smem (L1 is tiny with ~226 KB of smem in use);
                // software-pipelined: this tile's value was loaded one tile ago.
                float bval = 0.f;
                if constexpr (!C::kBiasTab) {
                    bval = bias_pref;
                    bias_pref = load_bias_col((j + 1 == n2_tiles ? 0 : j + 1) * 128 + (int)(wg * 64 + (srow & 63)));
                }
                // tfull2[s] completes once per GEMM2 job on slot s (chunk-1
                // acquisitions never commit it), so count its phases per slot.
                mbar_wait(&tfull2[s], s ? tf_par1 : tf_par0);
                if (s) tf_par1 ^= 1u; else tf_par0 ^= 1u;
                tr(24);
                tc_fence_after();
                if (!C::kBiasTab && srow < 64) bias_g[s * 64 + srow] = bval;  // published by the barrier below
                uint32_t ra[32], rb[32];
                tmem_ld32(tmem_base + lane_base + 256 + 128 * s + 64 * wg, ra);
                tmem_ld32(tmem_base + lane_base + 256 + 128 * s + 64 * wg + 32, rb);
                tmem_ld_wait();
                tr(31);
                // every TMEM read of this slot by this warp has completed
                tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive_leader(&tempty2[s]);
                if constexpr (kRS) {
                    if (nsplit > 1) {
                        chain_reduce(ra);
                        chain_reduce(rb);
                        if (sp + 1 < nsplit) continue;  // only the last pair of the chain writes the tile
                    }
                }
                const int n0 = j * 128 + 64 * (int)wg;
                if (use_bits_in) {  // this tile's bits were loaded one tile ago; fetch the next tile's
                    mbits = mbits_next;
                    if (j + 1 < n2_tiles) mbits_next = load_bits(j + 1);
                }
                uint32_t bo0 = 0u, bo1 = 0u;  // use_bits_out: this row's bits of the group's 64 columns
                if (storer || (save_pend && lane == 0)) bulk_wait_read<0>();  // our previous stores have read `buf`
                save_pend = false;
                tr(25);
                if (wstore) __syncwarp();
                else named_bar_sync(1 + wg, 128);
                tr(32);
                const uint32_t row_addr = smem_u32(buf) + srow * 128;
                const uint32_t mrow_addr = smem_u32(mbuf) + srow * 128;
                if (use_mask) {
                    mbar_wait(&mfull[wg], mph);
                    mph ^= 1u;
                }
                // 16-B chunk of the ReLU mask (the layer input) at staging offset `off`
                // (the TMA-loaded mask tile has the output tile's layout; OOB is zero)
                auto mask_chunk = [&](uint32_t off) -> uint4 {
                    uint4 v;
                    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                                 : "r"(mrow_addr + off));
                    return v;
                };
                if constexpr (kKind == 1) {
                    // fp32 output: the group's 64 columns are two [128 x 32] fp32 boxes
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const float4 b4 = reinterpret_cast<const float4*>(bias_g + s * 64)[c];
                        const uint32_t* src = (c < 8) ? ra : rb;
                        const int o = (c & 7) * 4;
                        float v[4] = {fmaf(__uint_as_float(src[o]), alpha, b4.x),
                                      fmaf(__uint_as_float(src[o + 1]), alpha, b4.y),
                                      fmaf(__uint_as_float(src[o + 2]), alpha, b4.z),
                                      fmaf(__uint_as_float(src[o + 3]), alpha, b4.w)};
                        if (kPost && args.relu) {
#pragma unroll
                            for (int i = 0; i < 4; ++i) v[i] = fmaxf(v[i], 0.f);
                        }
                        if (kPost == 2) {
                            const int sh = 4 * (c & 7);
                            if (use_bits_in) {
                                const uint32_t b4 = ((c < 8 ? mbits.x : mbits.y) >> sh) & 0xFu;
#pragma unroll
                                for (int i = 0; i < 4; ++i) v[i] = ((b4 >> i) & 1u) ? v[i] : 0.f;
                            }
                            if (use_bits_out) {
                                uint32_t b4 = 0u;
#pragma unroll
                                for (int i = 0; i < 4; ++i) b4 |= (v[i] > 0.f ? 1u : 0u) << i;
                                if (c < 8) bo0 |= b4 << sh; else bo1 |= b4 << sh;
                            }
                        }
                        if (use_mask) {
                            const uint4 mk = mask_chunk((c >> 3) * 16384 + ((uint32_t)((c & 7) ^ (srow & 7)) << 4));
                            const uint32_t m[4] = {mk.x, mk.y, mk.z, mk.w};
#pragma unroll
                            for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(m[i]) > 0.f ? v[i] : 0.f;
                        }
                        st_shared_v4(row_addr + (c >> 3) * 16384 + ((uint32_t)((c & 7) ^ (srow & 7)) << 4),
                                     __float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]),
                                     __float_as_uint(v[3]));
                    }
                    if (use_bits_out && row_ok && n0 < args.N2)
                        *reinterpret_cast<uint2*>(args.relu_bits + (long long)row * args.bits_ld + n0 / 32) =
                            make_uint2(bo0, bo1);
                    fence_proxy_async_smem();
                    named_bar_sync(1 + wg, 128);
                    if (issuer) {
                        tma_store_2d(&tmY, buf, n0, t * tile_rows + (int)rank * 128);
                        tma_store_2d(&tmY, buf + 16384, n0 + 32, t * tile_rows + (int)rank * 128);
                        bulk_commit();
                        if (use_mask && j + 1 < n2_tiles) issue_mask(t, j + 1);  // mbuf was read by all
                    }
                    continue;
                }
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    // (per-warp stores without the bias table means no bias: the group
                    // barrier that publishes bias_g is gone, so it is not read)
                    const float4* bp = C::kBiasTab ? reinterpret_cast<const float4*>(bias_tab + n0 + 8 * c)
                                                  : reinterpret_cast<const float4*>(bias_g + s * 64 + 8 * c);
                    const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
                    const float4 b0 = (!C::kBiasTab && wstore) ? zero4 : bp[0];
                    const float4 b1 = (!C::kBiasTab && wstore) ? zero4 : bp[1];
                    const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                    const uint32_t* src = (c < 4) ? ra : rb;
                    const int o = (c & 3) * 8;
                    float v[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] = fmaf(__uint_as_float(src[o + i]), alpha, bv[i]);
                    if (kPost && args.relu) {
#pragma unroll
                        for (int i = 0; i < 8; ++i) v[i] = fmaxf(v[i], 0.f);
                    }
                    if (kPost == 2) {
                        const int sh = 8 * (c & 3);
                        if (use_bits_in) {
                            const uint32_t b8 = ((c < 4 ? mbits.x : mbits.y) >> sh) & 0xFFu;
#pragma unroll
                            for (int i = 0; i < 8; ++i) v[i] = ((b8 >> i) & 1u) ? v[i] : 0.f;
                        }
                        if (use_bits_out) {
                            uint32_t b8 = 0u;
#pragma unroll
                            for (int i = 0; i < 8; ++i) b8 |= (v[i] > 0.f ? 1u : 0u) << i;
                            if (c < 4) bo0 |= b8 << sh; else bo1 |= b8 << sh;
                        }
                    }
                    if (use_mask) {
                        const uint4 mk = mask_chunk((uint32_t)(c ^ (srow & 7)) << 4);
                        const uint32_t m[4] = {mk.x, mk.y, mk.z, mk.w};
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&m[i]));
                            v[2 * i] = f.x > 0.f ? v[2 * i] : 0.f;
                            v[2 * i + 1] = f.y > 0.f ? v[2 * i + 1] : 0.f;
                        }
                    }
                    uint32_t w[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) w[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
                    st_shared_v4(row_addr + ((uint32_t)(c ^ (srow & 7)) << 4), w[0], w[1], w[2], w[3]);
                }
                if (use_bits_out && row_ok && n0 < args.N2)
                    *reinterpret_cast<uint2*>(args.relu_bits + (long long)row * args.bits_ld + n0 / 32) =
                        make_uint2(bo0, bo1);
                tr(33);
                fence_proxy_async_smem();
                if (wstore) {
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_2d(&tmYw, buf + q * 4096, n0, t * tile_rows + (int)rank * 128 + (int)q * 32);
                        bulk_commit();
                    }
                    tr(26);
                    continue;
                }
                named_bar_sync(1 + wg, 128);
                tr(34);
                if (issuer) {
                    tma_store_2d(&tmY, buf, n0, t * tile_rows + (int)rank * 128);
                    bulk_commit();
                    tr(26);
                }
                if (use_mask && issuer && j + 1 < n2_tiles) issue_mask(t, j + 1);  // mbuf was read by all
            }
        }
        }  // kDT
        if (storer) bulk_wait<0>();
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
// bf16: H compacts to R/2 TMEM columns, R <= 512 per CTA pair, and the R-split
// cluster (kRS) of up to 4 pairs takes R <= 2048.  TF32: H keeps one column per
// rank index next to the two 128-column GEMM2 slots, R <= 256.
constexpr int kMaxSplit = 4;
inline int b2b_split(long long R_pad) { return (int)((R_pad + 511) / 512); }  // pairs per cluster
inline bool b2b_supported(long long R_pad, int kind) {
    return kind == 0 ? b2b_split(R_pad) <= kMaxSplit : R_pad <= 256;
}

}  // namespace skl
