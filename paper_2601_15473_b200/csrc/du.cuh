// du.cuh -- the fused parameter-gradient kernel of the SKLinear backward.
//
//   dU1s  = inv · Savedᵀ · G      [L·k, d_out]                Saved = x·S1 (forward)
//   dU2sᵀ = inv · P_S2ᵀ · X       [L·k, d_in] -> [L][d_in][k] P_S2  = G·S2ᵀ (b2b_bwd)
//   db    = Σ_t G[t, :]                                        (nn_layers.cpp:99, unscaled)
//
// Reference: SkLinear::backward grad_u1 / grad_u2 / grad_b (nn_layers.cpp:88-99).
// All three reduce over the T tokens.  One persistent launch covers both GEMMs
// as a grouped problem list (both have M = L·k), split along T so every CTA
// pair has a unit.  The fused kernels wrote Saved and P_S2 TRANSPOSED
// ([L·k][T]), so A is a K-major operand (one 16 KB TMA box per stage); G and
// X are token-major, i.e. MN-major B tiles.  MMAs are cta_group::2 (M = 256:
// each CTA keeps 128 rows of A and half of the 256 B columns), which halves
// per-SM operand ingest versus one CTA per tile.
//
// db rides along: the column sums of G are taken by the epilogue warps from
// the G tiles already staged in shared memory for dU1.  Because cta_group::2
// TMA completion only reaches the leader's barrier, each CTA here loads its
// own half with plain TMA onto its OWN full barrier, and a relay thread on
// the peer CTA forwards completion to the leader (so both CTAs can observe
// their own stages).
//
// Reduction is deterministic and in-kernel: every (tile, split, rank) writes
// its fp32 partial and the 2·S CTAs of a tile each reduce a 1/(2S) slice in
// split order 0..S-1.  Default (DuArgs::cr): the S split pairs of a tile are
// one thread-block cluster; partials move with single bulk copies (smem ->
// global -> the reducing CTA's smem) around one cluster barrier.  Fallbacks
// (S > 4): a cooperative launch with a grid-wide ticket barrier, or the last
// CTA of a tile reducing it alone (SKL_DU_NOCOOP).
#pragma once

#include "sm100.cuh"
#include "trace.cuh"

namespace skl {

struct DuProblem {
    int M, N;             // output is M x N
    int m_tiles, n_tiles;  // 256 x 256 pair tiles
    int tile0;            // first global tile index of this problem
    int splits;           // T split of this problem's tiles (per-problem: balances colsum vs plain tiles)
    int unit0, slot0;     // first work unit / first partial slot of this problem
    int colsum;           // 1: also sum the B operand over K (db)
    float alpha;
    float* out;           // out[(m / mb) * mbs + (m % mb) * ms + n * ns]
    long long mb, mbs, ms, ns;
    float* db;            // [N] when colsum
};

struct DuArgs {
    int k_blocks, num_units, num_tiles;
    DuProblem p[2];
    float* part;     // [slot0 + tile * splits + split][256][256] per problem
    float* cpart;    // [p0.n_tiles][p0.splits][256]
    int* tickets;    // [num_tiles], zero on entry, left zero on exit
    int coop;        // 1: cooperative launch (all units co-resident) -> slice-parallel reduction
    int relay;       // 1: per-CTA TMA barriers + peer relay (needed when colsum reads both halves)
    int l2hint;      // L2 cache-hint policy bits for the operand loads (see the producer)
    int cr;          // cluster reduction: one cluster of 2S CTAs per tile (S splits = S pairs); each CTA
                     // bulk-stores its partial, the cluster barrier publishes it, each CTA bulk-loads its slice
};

namespace dev {

// A k-block is 128 bytes of tokens: 64 bf16 (kKind 0) or 32 fp32 words (kKind 1,
// TF32).  Every tile therefore has the same byte geometry in both variants;
// only the MN-major B blocks narrow from 64 to 32 columns.
constexpr int kDuBM = 128, kDuBN = 256, kDuStages = 6;
constexpr int kDuABytes = kDuBM * 128;        // K-major [128 rows x 128 B of tokens]
constexpr int kDuBBytes = (kDuBN / 2) * 128;  // MN-major blocks [tokens x 128 B of columns]
constexpr int kDuStageBytes = kDuABytes + kDuBBytes;
constexpr int kDuSmem = kDuStages * kDuStageBytes + 1024 + 256 + 8 * 128 * 4 + 128 * 4;
template <int kKind>
struct DuKind {
    static constexpr int kElem = kKind == 0 ? 2 : 4;
    static constexpr int kBK = 128 / kElem;   // tokens per k-block
    static constexpr int kW = 128 / kElem;    // columns per MN-major block
    static constexpr int kUK = kKind == 0 ? 16 : 8;  // K per MMA instruction
};

// Cluster-reduce tail parameters, precomputed at kernel start into shared memory:
// the tail runs once per CTA with a cold instruction cache (ncu: stall_no_inst),
// so it is kept short and free of the unit decode.
struct DuTail {
    float* out;        // P.out
    float* db;         // P.db (colsum units)
    const float* g0;   // split-0 partial of this pair rank: [128][256]; splits 2*128*256 apart
    const float* c0;   // split-0 column sums of this rank; splits 256 apart
    long long mbs, ms, ns;
    int mb, M, N, m0, n0, r0, rows, S, colsum, vec;
    int valid;         // rows of this CTA's 128-row half inside M (only those move)
    float alpha;
};
static_assert(136 * kDuBN * 4 + 8 * 512 <= kDuStages * kDuStageBytes, "cluster-reduce staging exceeds the ring");

template <int kKind>
__global__ void __launch_bounds__(256, 1)
    du_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
              const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1, DuArgs args) {
    using KT = DuKind<kKind>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base_u32 - smem_u32(smem_raw));
    uint8_t* sA = smem;
    uint8_t* sB = smem + kDuStages * kDuABytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kDuStages * kDuStageBytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + kDuStages;
    uint64_t* tfull = bars + 2 * kDuStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int* ticket_s = reinterpret_cast<int*>(tmem_slot + 1);
    uint64_t* rbar = tempty + 3;  // (8-B slot after tmem_slot/ticket_s) reduction bulk-load barrier
    float* csum_s = reinterpret_cast<float*>(smem + kDuStages * kDuStageBytes + 256);  // [8][128]
    float* cr_part = reinterpret_cast<float*>(smem);        // [128][256] chunk-swizzled accumulator (cluster reduce)

    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    const uint32_t crank = cluster_ctarank();
    const uint32_t rank = crank & 1u;           // rank inside the MMA pair
    const uint32_t lead_cta = crank & ~1u;      // cluster rank of the pair's leader
    const uint16_t pair_mask = (uint16_t)(3u << lead_cta);
    const bool leader = rank == 0;

    if (warp == 0 && elect_one()) {
        prefetch_tmap(&tmA0);
        prefetch_tmap(&tmB0);
        prefetch_tmap(&tmA1);
        prefetch_tmap(&tmB1);
        for (int s = 0; s < kDuStages; ++s) {
            mbar_init(&full[s], leader ? 2 : 1);  // leader: own tx + peer relay
            mbar_init(&empty[s], 5);              // MMA commit + 4 colsum warps (or 4 extra commits)
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 8);
        }
        mbar_init(rbar, 1);
        fence_barrier_init();
    }
    if (warp == 2) {
        tmem_alloc<2>(tmem_slot, 512);
        tmem_relinquish<2>();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();
    pdl_launch_dependents();

    const int units = args.num_units;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    struct Unit {
        int p, mt, nt, tile, split, kb0, kb1, slot, nsplit;
        bool colsum;
    };
    auto decode = [&](int u) {
        Unit x;
        x.p = u >= args.p[1].unit0 && args.p[1].m_tiles > 0 ? 1 : 0;
        const DuProblem& P = args.p[x.p];
        const int ptiles = P.m_tiles * P.n_tiles;
        const int lu = u - P.unit0;
        // split-major within the problem (concurrent units share a token window);
        // cluster-reduce mode: tile-major, the S splits of a tile are one cluster
        x.split = args.cr ? lu % P.splits : lu / ptiles;
        const int lt = args.cr ? lu / P.splits : lu % ptiles;
        x.tile = P.tile0 + lt;
        x.slot = P.slot0 + lt * P.splits;
        x.nsplit = P.splits;
        x.mt = lt % P.m_tiles;
        x.nt = lt / P.m_tiles;
        x.kb0 = (int)(((long long)x.split * args.k_blocks) / P.splits);
        x.kb1 = (int)(((long long)(x.split + 1) * args.k_blocks) / P.splits);
        x.colsum = args.p[x.p].colsum && x.mt == 0;
        return x;
    };

    DuTail* tail = reinterpret_cast<DuTail*>(csum_s + 8 * 128);  // 512 B slot after the colsum scratch
    if (args.cr && threadIdx.x == 0 && pair < units) {
        const Unit x = decode(pair);
        const DuProblem& P = args.p[x.p];
        DuTail d;
        d.out = P.out;
        d.db = P.db;
        d.g0 = args.part + ((long long)(pair - x.split) * 2 + rank) * 128 * kDuBN;
        d.c0 = args.cpart + (long long)x.nt * x.nsplit * kDuBN + rank * 128;
        d.mbs = P.mbs;
        d.ms = P.ms;
        d.ns = P.ns;
        d.mb = P.mb >= P.M ? P.M : (int)P.mb;
        d.M = P.M;
        d.N = P.N;
        d.r0 = x.split * 128 / x.nsplit;
        d.rows = (x.split + 1) * 128 / x.nsplit - d.r0;
        d.valid = min(128, max(0, P.M - (x.mt * 256 + (int)rank * 128)));
        d.m0 = x.mt * 256 + (int)rank * 128 + d.r0;
        d.n0 = x.nt * 256;
        d.S = x.nsplit;
        d.colsum = x.colsum ? 1 : 0;
        d.vec = P.ns == 1 && ((P.ms | P.mbs) & 3) == 0 && (reinterpret_cast<uintptr_t>(P.out) & 15) == 0;
        d.alpha = P.alpha;
        *tail = d;
    }

    if (warp == 0) {
        // ------------------------------------------------------------ producer (both CTAs, own half)
        if (elect_one()) {
            Tr tr(0, 4);
            int stage = 0;
            uint32_t phase = 0;
            // A (Savedᵀ / P_S2ᵀ) is re-read by every N tile of the same split; B (G / X) once
            // (DuArgs::l2hint bit 0: A evict_last, bit 1: B evict_first; 0 = the default policy)
            const uint64_t pol_norm = l2_evict_normal();
            const uint64_t pol_a = (args.l2hint & 1) ? l2_evict_last() : pol_norm;
            const uint64_t pol_b = (args.l2hint & 2) ? l2_evict_first() : pol_norm;
            for (int u = pair; u < units; u += npairs) {
                const Unit x = decode(u);
                const CUtensorMap* ma = x.p ? &tmA1 : &tmA0;
                const CUtensorMap* mb = x.p ? &tmB1 : &tmB0;
                const int m0 = x.mt * 256 + (int)rank * 128, n0 = x.nt * 256 + (int)rank * 128;
                for (int kb = x.kb0; kb < x.kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    tr(1);
                    uint8_t* a_dst = sA + stage * kDuABytes;
                    uint8_t* b_dst = sB + stage * kDuBBytes;
                    const int k0 = kb * KT::kBK;
                    if (!args.relay) {
                        // no colsum anywhere: pair-signalled TMA straight onto the leader's barrier
                        if (leader) mbar_arrive_expect_tx(&full[stage], 2 * kDuStageBytes);
                        else mbar_arrive_cluster(&full[stage], lead_cta);
                        tma_load_2d_hint<2>(ma, &full[stage], a_dst, k0, m0, pol_a);
#pragma unroll
                        for (int j = 0; j < 128 / KT::kW; ++j)
                            tma_load_2d_hint<2>(mb, &full[stage], b_dst + j * KT::kBK * 128, n0 + j * KT::kW, k0, pol_b);
                        if (++stage == kDuStages) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    mbar_arrive_expect_tx(&full[stage], kDuStageBytes);
                    tma_load_2d_hint<1>(ma, &full[stage], a_dst, k0, m0, pol_a);
#pragma unroll
                    for (int j = 0; j < 128 / KT::kW; ++j)
                        tma_load_2d_hint<1>(mb, &full[stage], b_dst + j * KT::kBK * 128, n0 + j * KT::kW, k0, pol_b);
                    if (++stage == kDuStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer (leader)
        if (leader && elect_one()) {
            Tr tr(1, 4);
            constexpr uint32_t idesc = make_idesc(kKind, 256, kDuBN, 0, 1);
            int stage = 0;
            uint32_t phase = 0;
            int iter = 0;
            for (int u = pair; u < units; u += npairs, ++iter) {
                const Unit x = decode(u);
                const int acc = iter & 1;
                mbar_wait(&tempty[acc], ((iter >> 1) & 1) ^ 1);
                tr(12);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * kDuBN;
                for (int kb = x.kb0; kb < x.kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tr(11);
                    tc_fence_after();
                    const uint32_t a_addr = smem_u32(sA + stage * kDuABytes);
                    const uint32_t b_addr = smem_u32(sB + stage * kDuBBytes);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        mma_ss<2, kKind>(d_tmem, make_sdesc(a_addr + k * 32, 0, 1024),
                                         kKind == 0 ? make_sdesc(b_addr + k * KT::kUK * 128, KT::kBK * 128, 1024)
                                                    : make_sdesc(b_addr + k * KT::kUK * 128, KT::kBK * 128, 512, 1),
                                         idesc, (kb > x.kb0 || k > 0) ? 1u : 0u);
                    mma_commit_pair(&empty[stage], pair_mask);
                    if (!x.colsum)  // stand in for the 4 colsum warps (multicast to both CTAs)
                        for (int i = 0; i < 4; ++i) mma_commit_pair(&empty[stage], pair_mask);
                    if (++stage == kDuStages) { stage = 0; phase ^= 1; }
                }
                mma_commit_pair(&tfull[acc], pair_mask);
            }
        }
    } else if (warp == 3) {
        // ------------------------------------------------------------ relay (peer CTA)
        if (!leader && args.relay && elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int u = pair; u < units; u += npairs) {
                const Unit x = decode(u);
                for (int kb = x.kb0; kb < x.kb1; ++kb) {
                    mbar_wait(&full[stage], phase);        // our half has landed
                    mbar_arrive_cluster(&full[stage], lead_cta);  // tell the leader's MMA issuer
                    if (++stage == kDuStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue warps (colsum + partials + reduce)
        const uint32_t q = warp & 3;
        const int t = (int)(q * 32 + lane);  // 0..127
        Tr tr((lane == 0 && warp == 4) ? 2 : -1, 4);
        int stage = 0;
        uint32_t phase = 0;
        uint32_t red_phase = 0;
        int iter = 0;
        for (int u = pair; u < units; u += npairs, ++iter) {
            const Unit x = decode(u);
            const DuProblem& P = args.p[x.p];
            const int m0 = x.mt * 256, n0 = x.nt * 256;
            if (x.colsum) {
                // ---- column sums of this CTA's 128 staged G columns: thread ->
                // one 16-B chunk (kCPC columns) of one kW-column block, 8 token rows.
                constexpr int kCPC = 16 / KT::kElem;          // columns per 16-B chunk
                constexpr int kChunks = 128 / kCPC;           // chunks across 128 columns
                constexpr int kGroups = 128 / kChunks;        // row groups of 8 tokens (= kBK / 8)
                const int chunk = t % kChunks, blk = chunk >> 3, ch = chunk & 7, r0 = (t / kChunks) * 8;
                float cs[kCPC];
#pragma unroll
                for (int i = 0; i < kCPC; ++i) cs[i] = 0.f;
                for (int kb = x.kb0; kb < x.kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    const uint32_t b_addr = smem_u32(sB + stage * kDuBBytes) + blk * KT::kBK * 128;
#pragma unroll
                    for (int r = r0; r < r0 + 8; ++r) {
                        uint32_t w[4];
                        // physical 16-B chunk: 128B swizzle (bf16) / 128B-atom-32B swizzle (tf32)
                        const uint32_t pch = kKind == 0 ? (uint32_t)(ch ^ (r & 7))
                                                        : (uint32_t)((((ch >> 1) ^ (r & 3)) << 1) | (ch & 1));
                        asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                                     : "r"(b_addr + r * 128 + (pch << 4)));
                        if constexpr (kKind == 0) {
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
                                cs[2 * i] += f.x;
                                cs[2 * i + 1] += f.y;
                            }
                        } else {
#pragma unroll
                            for (int i = 0; i < 4; ++i) cs[i] += __uint_as_float(w[i]);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[stage]);
                    if (++stage == kDuStages) { stage = 0; phase ^= 1; }
                }
                // combine the row groups in order -> cpart[nt][split][rank*128 + col]
#pragma unroll
                for (int i = 0; i < kCPC; ++i) csum_s[(t / kChunks) * 128 + chunk * kCPC + i] = cs[i];
                named_bar_sync(2, 128);
                {
                    float s = 0.f;
#pragma unroll
                    for (int g = 0; g < kGroups; ++g) s += csum_s[g * 128 + t];
                    __stcg(args.cpart + ((long long)x.nt * x.nsplit + x.split) * kDuBN + rank * 128 + t, s);
                }
                named_bar_sync(2, 128);
            } else {
                // the MMA issuer arrives for us on non-colsum units; keep the ring position
                for (int kb = x.kb0; kb < x.kb1; ++kb)
                    if (++stage == kDuStages) { stage = 0; phase ^= 1; }
            }
            // ---- accumulator -> fp32 partial [tile][split][256][256], our 128 rows
            const int acc = iter & 1;
            mbar_wait(&tfull[acc], (iter >> 1) & 1);
            tr(21);
            tc_fence_after();
            if (args.cr) {
                // accumulator -> this CTA's smem (the operand ring is idle now); the
                // cluster sums it with its peers' after the kernel-wide cluster barrier
                const uint32_t t_row = tmem_base + ((q * 32u) << 16) + acc * kDuBN;
                // row t, 16-B chunk j at chunk (j ^ (t & 7)): conflict-free, and rows stay
                // contiguous so the partial moves with one bulk copy
                float* srow = cr_part + t * kDuBN;
#pragma unroll 1
                for (int c = 0; c < kDuBN; c += 32) {
                    uint32_t v[32];
                    tmem_ld32(t_row + c, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; i += 4)
                        *reinterpret_cast<float4*>(srow + ((((c + i) >> 2) ^ (t & 7)) << 2)) =
                            make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                                        __uint_as_float(v[i + 3]));
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (leader) mbar_arrive(&tempty[acc]);
                    else mbar_arrive_cluster(&tempty[acc], lead_cta);
                }
                tr(22);
                continue;
            }
            {
                float* prow = args.part + (((long long)x.slot + x.split) * 256 + rank * 128 + t) * kDuBN;
                const uint32_t t_row = tmem_base + ((q * 32u) << 16) + acc * kDuBN;
#pragma unroll 1
                for (int c = 0; c < kDuBN; c += 32) {
                    uint32_t v[32];
                    tmem_ld32(t_row + c, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; i += 4)
                        __stcg(reinterpret_cast<float4*>(prow + c + i),
                               make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                                           __uint_as_float(v[i + 3])));
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(&tempty[acc]);
                else mbar_arrive_cluster(&tempty[acc], lead_cta);
            }

            // ---- deterministic split reduction (sum in split order 0..S-1)
            __threadfence();
            named_bar_sync(2, 128);
            int* tk = args.tickets + x.tile;
            const int parts = 2 * x.nsplit;  // CTAs contributing to this tile
            int row_lo, row_hi, col_lo, col_hi;
            if (args.coop) {
                if (t == 0) {
                    atomicAdd(tk, 1);
                    uint64_t t0, t1;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
                    while (ld_acquire_gpu(tk) < parts) {  // bounded: a scheduling bug traps, never hangs
                        __nanosleep(64);
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
                        if (t1 - t0 > 10000000000ull) __trap();
                    }
                }
                named_bar_sync(2, 128);
                const int z = 2 * x.split + (int)rank;
                row_lo = z * 256 / parts;
                row_hi = (z + 1) * 256 / parts;
                col_lo = z * kDuBN / parts;
                col_hi = (z + 1) * kDuBN / parts;
            } else {
                if (t == 0) *ticket_s = atomicAdd(tk, 1);
                named_bar_sync(2, 128);
                const bool last = *ticket_s == parts - 1;
                named_bar_sync(2, 128);
                row_lo = 0; row_hi = last ? 256 : 0;
                col_lo = 0; col_hi = last ? kDuBN : 0;
            }
            __threadfence();
            const float* pbase = args.part + (long long)x.slot * 256 * kDuBN;
            const bool vec = P.ns == 1 && (P.ms & 3) == 0 && (P.mbs & 3) == 0 &&
                             (reinterpret_cast<uintptr_t>(P.out) & 15) == 0;
            if (args.coop) {
                // Cooperative (one unit per pair): the operand ring is idle now, so the
                // S partial slices of this CTA's rows (S x rows x 1 KB = 128 KB, since
                // rows = 256 / 2S) are pulled into smem with bulk copies -- all in flight
                // at once -- and summed from smem.  (Register loads from far L2 were
                // latency-bound: ~10 us for 128 KB.)
                const int rows = row_hi - row_lo;
                const uint32_t slice = (uint32_t)rows * kDuBN * 4;
                if (t == 0 && rows > 0) {
                    fence_proxy_async_global();  // partials were written by other CTAs' generic stores
                    mbar_arrive_expect_tx(rbar, slice * (uint32_t)x.nsplit);
                    for (int sp = 0; sp < x.nsplit; ++sp)
                        bulk_load_1d(smem + (size_t)sp * slice, pbase + ((long long)sp * 256 + row_lo) * kDuBN, slice,
                                     rbar);
                }
                if (rows > 0) mbar_wait(rbar, red_phase);
                red_phase ^= 1u;
                const float4* s4 = reinterpret_cast<const float4*>(smem);
                for (int f = t; f < rows * (kDuBN / 4); f += 128) {
                    const int r = row_lo + f / (kDuBN / 4), c = (f % (kDuBN / 4)) * 4;
                    const int m = m0 + r, n = n0 + c;
                    float4 sum = s4[f];
                    for (int sp = 1; sp < x.nsplit; ++sp) {
                        const float4 v = s4[(size_t)sp * (slice / 16) + f];
                        sum.x += v.x; sum.y += v.y; sum.z += v.z; sum.w += v.w;
                    }
                    if (m >= P.M || n >= P.N) continue;
                    const float o[4] = {sum.x * P.alpha, sum.y * P.alpha, sum.z * P.alpha, sum.w * P.alpha};
                    const long long mo = P.mb >= P.M ? (long long)m * P.ms : (m / P.mb) * P.mbs + (m % P.mb) * P.ms;
                    if (vec && n + 4 <= P.N) {
                        *reinterpret_cast<float4*>(P.out + mo + n) = make_float4(o[0], o[1], o[2], o[3]);
                    } else {
                        for (int i = 0; i < 4 && n + i < P.N; ++i) P.out[mo + (long long)(n + i) * P.ns] = o[i];
                    }
                }
            } else {
            // Last-CTA reduction (non-cooperative): each thread gathers kU float4 outputs at once
            // (kU x splits independent L2 loads in flight) before any store.
            constexpr int kU = 8;
            const int nf = (row_hi - row_lo) * (kDuBN / 4);
            for (int f0 = t; f0 < nf; f0 += 128 * kU) {
                float4 sum[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u) sum[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int sp = 0; sp < x.nsplit; ++sp) {
                    float4 v[kU];
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const int f = f0 + 128 * u;
                        const int r = row_lo + f / (kDuBN / 4), c = (f % (kDuBN / 4)) * 4;
                        v[u] = f < nf ? __ldcg(reinterpret_cast<const float4*>(pbase + ((long long)sp * 256 + r) * kDuBN + c))
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        sum[u].x += v[u].x; sum[u].y += v[u].y; sum[u].z += v[u].z; sum[u].w += v[u].w;
                    }
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const int f = f0 + 128 * u;
                    if (f >= nf) break;
                    const int r = row_lo + f / (kDuBN / 4), c = (f % (kDuBN / 4)) * 4;
                    const int m = m0 + r, n = n0 + c;
                    if (m >= P.M || n >= P.N) continue;
                    const float o[4] = {sum[u].x * P.alpha, sum[u].y * P.alpha, sum[u].z * P.alpha, sum[u].w * P.alpha};
                    const long long mo = (m / P.mb) * P.mbs + (m % P.mb) * P.ms;
                    if (vec && n + 4 <= P.N) {
                        *reinterpret_cast<float4*>(P.out + mo + n) = make_float4(o[0], o[1], o[2], o[3]);
                    } else {
                        for (int i = 0; i < 4 && n + i < P.N; ++i) P.out[mo + (long long)(n + i) * P.ns] = o[i];
                    }
                }
            }
            }
            if (x.colsum) {
                for (int c = col_lo + t; c < col_hi; c += 128) {
                    const int n = n0 + c;
                    if (n >= P.N) continue;
                    float sum = 0.f;
                    for (int sp = 0; sp < x.nsplit; ++sp)
                        sum += __ldcg(args.cpart + ((long long)x.nt * x.nsplit + sp) * kDuBN + c);
                    P.db[n] = sum;
                }
            }
            // ---- ticket release: the last CTA of the tile to get here resets it
            named_bar_sync(2, 128);
            if (t == 0) {
                if (args.coop) {
                    if (atomicAdd(tk, 1) == 2 * parts - 1) atomicExch(tk, 0);
                } else if (*ticket_s == parts - 1) {
                    atomicExch(tk, 0);
                }
            }
        }
    }
    if (args.cr && pair < units) {
        // ---- cluster reduction.  Every CTA bulk-stores its (chunk-swizzled) smem
        // partial to its global slot [unit][rank][128][256]; the cluster barrier
        // publishes them; this CTA (split sp, pair rank r) then bulk-loads rows
        // [sp*128/S, (sp+1)*128/S) of its rank's 128 rows from every split (one
        // copy per split) plus the splits' column sums, and sums in split order
        // 0..S-1.  Few, large copies: per-copy TMA overhead and the cold tail code
        // (ncu: stall_no_inst) are what this phase costs.
        __syncthreads();
        if (threadIdx.x == 0) {
            fence_proxy_async_smem();  // the dump was written by generic stores
            if (tail->valid > 0)
                bulk_store_1d(args.part + ((long long)pair * 2 + rank) * 128 * kDuBN, cr_part,
                              (uint32_t)tail->valid * kDuBN * 4);
            bulk_commit();
            bulk_wait<0>();
            __threadfence();
        }
        tc_fence_before();
        cluster_sync();
        Tr trr((threadIdx.x == 128) ? 3 : -1, 4);
        trr(23);
        const DuTail d = *tail;  // registers: the output stores must not force reloads
        const int S = d.S, rows = max(0, min(d.rows, d.valid - d.r0));  // slice rows inside M
        float* cs = cr_part + 136 * kDuBN;  // past S * ceil(128 / S) <= 135 slice rows (S <= 8)
        if (threadIdx.x == 0) {
            fence_proxy_async_global();  // order the acquired view before the bulk reads
            mbar_arrive_expect_tx(rbar, (uint32_t)(S * rows * kDuBN * 4 + (d.colsum ? S * 512 : 0)));
            for (int q2 = 0; q2 < S; ++q2) {
                if (rows > 0)
                    bulk_load_1d(cr_part + q2 * rows * kDuBN, d.g0 + ((long long)q2 * 256 + d.r0) * kDuBN,
                                 (uint32_t)rows * kDuBN * 4, rbar);
                if (d.colsum) bulk_load_1d(cs + q2 * 128, d.c0 + q2 * kDuBN, 512, rbar);
            }
        }
        mbar_wait(rbar, 0);
        trr(24);
        // element (slice row r, column c) of split q2: row q2 * rows + r, chunk (c/4) ^ ((r0 + r) & 7)
        if (d.ns == 1) {
            // row-contiguous output (dU1): lanes over 4-column chunks, float4 stores
#pragma unroll 1
            for (int f = (int)threadIdx.x; f < rows * (kDuBN / 4); f += 256) {
                const int r = f >> 6, j = f & 63;
                const int m = d.m0 + r, n = d.n0 + j * 4;
                if (m >= d.M || n >= d.N) continue;
                const float* src = cr_part + r * kDuBN + ((j ^ ((d.r0 + r) & 7)) << 2);
                float4 v[8];  // up to 8 partial loads in flight, then the ordered sum (split 0, 1, ...)
#pragma unroll
                for (int q2 = 0; q2 < 8; ++q2)
                    if (q2 < S) v[q2] = *reinterpret_cast<const float4*>(src + q2 * rows * kDuBN);
                float4 a = v[0];
#pragma unroll
                for (int q2 = 1; q2 < 8; ++q2)
                    if (q2 < S) { a.x += v[q2].x; a.y += v[q2].y; a.z += v[q2].z; a.w += v[q2].w; }
                const long long mo = d.mb >= d.M ? (long long)m * d.ms
                                                 : (long long)(m / d.mb) * d.mbs + (long long)(m % d.mb) * d.ms;
                float* o = d.out + mo + n;
                if (d.vec && n + 4 <= d.N) {
                    *reinterpret_cast<float4*>(o) = make_float4(a.x * d.alpha, a.y * d.alpha, a.z * d.alpha, a.w * d.alpha);
                } else {
                    const float av[4] = {a.x, a.y, a.z, a.w};
                    for (int i = 0; i < 4 && n + i < d.N; ++i) o[i] = av[i] * d.alpha;
                }
            }
        } else {
            // strided columns (dU2ᵀ: consecutive rows contiguous): lanes over rows,
            // one 4-column chunk per step, so each scalar store covers 32 rows
#pragma unroll 1
            for (int j = (int)warp; j < kDuBN / 4; j += 8) {
                const int n = d.n0 + j * 4;
                if (n >= d.N) break;
#pragma unroll 1
                for (int r = (int)lane; r < rows; r += 32) {
                    const int m = d.m0 + r;
                    if (m >= d.M) break;
                    const float* src = cr_part + r * kDuBN + ((j ^ ((d.r0 + r) & 7)) << 2);
                    float4 v[8];  // all partial loads in flight, then the ordered sum
#pragma unroll
                    for (int q2 = 0; q2 < 8; ++q2)
                        if (q2 < S) v[q2] = *reinterpret_cast<const float4*>(src + q2 * rows * kDuBN);
                    float4 a = v[0];
#pragma unroll
                    for (int q2 = 1; q2 < 8; ++q2)
                        if (q2 < S) { a.x += v[q2].x; a.y += v[q2].y; a.z += v[q2].z; a.w += v[q2].w; }
                    float* o = d.out + (long long)(m / d.mb) * d.mbs + (long long)(m % d.mb) * d.ms + n * d.ns;
                    const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (n + i < d.N) o[i * d.ns] = av[i] * d.alpha;
                }
            }
        }
        trr(25);
        if (d.colsum) {
            for (int c = d.r0 + (int)threadIdx.x; c < d.r0 + d.rows; c += 256) {  // columns: not clamped by M
                const int n = d.n0 + (int)rank * 128 + c;
                if (n >= d.N) continue;
                float sum = cs[c];
                for (int q2 = 1; q2 < S; ++q2) sum += cs[q2 * 128 + c];
                d.db[n] = sum;
            }
        }
    } else {
        tc_fence_before();
        cluster_sync();  // the pair's MMAs into this CTA's TMEM are done before it is freed
    }
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<2>(tmem_base, 512);
    }
}

}  // namespace dev
}  // namespace skl
