// dut.cuh -- the parameter gradients of the SKLinear backward for SMALL rank
// L·k <= 128, as the transposed problem (no padded MMA rows).
//
//   dU1sᵀ = inv · Gᵀ · Saved     [d_out, L·k]     Saved = x·S1 (forward)
//   dU2s  = inv · Xᵀ · P_S2      [d_in,  L·k]     P_S2  = G·S2ᵀ (b2b_bwd)
//   db    = Σ_t G[t, :]                           (nn_layers.cpp:99, unscaled)
//
// Reference: SkLinear::backward grad_u1 / grad_u2 / grad_b (nn_layers.cpp:88-99).
// du.cuh computes dU1s = inv·Savedᵀ·G with M = L·k on a 256-row CTA-pair tile:
// at L·k = 16 (c4 L1 k16) 15/16 of its MMA rows are padding, enough to make that
// HBM-bound kernel tensor-bound too, and at L·k = 128 (the c5 768x768
// projections) half.  Here M is the feature dimension d (256-row pair chunks,
// A = G / X token-major, i.e. MN-major operand tiles) and N = L·k padded to 16
// (B = Savedᵀ / P_S2ᵀ, [L·k][T8], K-major).  A unit is (problem, group of up to
// kDutGroup M-chunks, token split): all its chunks accumulate in TMEM at once
// (chunks x N_pad <= 512 columns), so the activation G / X is read exactly once
// and the small rank operand once per group.  Units write fp32 partials; a
// second launch (dut_reduce_kernel) sums them in split order (deterministic),
// applies inv and scatters into the ABI layouts, and sums the db partials.
#pragma once

#include "sm100.cuh"
#include "trace.cuh"

namespace skl {

constexpr int kDutGroup = 4;  // M-chunks (256 rows each) per unit

struct DutProblem {
    int M;              // output rows (d_out for dU1ᵀ, d_in for dU2)
    int groups;         // ceil(M / (256 * kDutGroup))
    int unit0;          // first unit of this problem
    int colsum;         // 1: also column sums of A (db)
    float* out;         // element (m, n) at (n / nb) * nbs + (n % nb) * ns + m * ms
    long long nb, nbs, ns, ms;
    float* db;          // [M] when colsum
};

struct DutArgs {
    int N, N_pad;       // L·k and its 16-padded MMA width
    int k_blocks;       // token k-blocks (64 bf16 / 32 fp32 tokens each)
    int splits;         // token splits per (problem, group)
    int num_units, stages, stage_bytes, b_bytes;  // stage = B tile (b_bytes, 1 KB aligned) + A chunks
    float alpha;
    DutProblem p[2];
    float* part;        // [unit][2 ranks][kDutGroup][128][N_pad]
    float* cpart;       // [unit][2 ranks][kDutGroup][128]  (colsum units)
};

namespace dev {

template <int kKind>
__global__ void __launch_bounds__(256, 1)
    dut_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
               const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1, DutArgs args) {
    constexpr int kElem = kKind == 0 ? 2 : 4;
    constexpr int kBK = 128 / kElem;   // tokens per k-block
    constexpr int kW = 128 / kElem;    // MN-major block width (columns of A per 128-B row)
    constexpr int kUK = kKind == 0 ? 16 : 8;
    constexpr int kChunkBytes = 128 * 128;  // one 128-row A chunk per CTA per k-block (16 KB)
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base_u32 - smem_u32(smem_raw));
    const int S = args.stages, SB = args.stage_bytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * SB);
    uint64_t* full = bars;                // [S] this CTA's stage landed (leader: + peer relay)
    uint64_t* empty = bars + S;           // [S] MMA commit + the 4 colsum warps
    uint64_t* tfull = bars + 2 * S;       // accumulators complete
    uint64_t* tempty = tfull + 1;         // accumulators drained (8 arrivals: 4 warps x 2 CTAs)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
    float* csum_s = reinterpret_cast<float*>(smem + S * SB + 256);  // [kDutGroup][8][128] colsum scratch

    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    const uint32_t rank = cluster_ctarank() & 1u;  // rank inside the MMA pair (clusters of 2)
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

    if (warp == 0 && elect_one()) {
        prefetch_tmap(&tmA0);
        prefetch_tmap(&tmB0);
        prefetch_tmap(&tmA1);
        prefetch_tmap(&tmB1);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], leader ? 2 : 1);  // leader: own tx + the peer's relay
            mbar_init(&empty[s], 5);              // MMA commit + 4 colsum warps (or 4 extra commits)
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, 8);
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

    struct Unit {
        int p, g, s, kb0, kb1, chunks, m0;
        bool colsum;
    };
    auto decode = [&](int u) {
        Unit x;
        x.p = (args.p[1].groups > 0 && u >= args.p[1].unit0) ? 1 : 0;
        const DutProblem& P = args.p[x.p];
        const int lu = u - P.unit0;
        x.g = lu / args.splits;
        x.s = lu % args.splits;
        x.kb0 = (int)(((long long)x.s * args.k_blocks) / args.splits);
        x.kb1 = (int)(((long long)(x.s + 1) * args.k_blocks) / args.splits);
        x.m0 = x.g * 256 * kDutGroup;
        x.chunks = min(kDutGroup, (P.M - x.m0 + 255) / 256);
        x.colsum = P.colsum != 0;
        return x;
    };
    const int units = args.num_units;

    if (warp == 0) {
        // ---------------------------------------------------------------- producer (own half, own barrier)
        if (elect_one()) {
            Tr tr(0, 4);
            int stage = 0;
            uint32_t phase = 0;
            const uint64_t pol_a = l2_evict_first();   // G / X: read once
            const uint64_t pol_b = l2_evict_normal();  // Savedᵀ / P_S2ᵀ: re-read by every group
            for (int u = pair; u < units; u += npairs) {
                const Unit x = decode(u);
                const CUtensorMap* ma = x.p ? &tmA1 : &tmA0;
                const CUtensorMap* mb = x.p ? &tmB1 : &tmB0;
                const uint32_t bytes = (uint32_t)(x.chunks * kChunkBytes + (args.N_pad / 2) * 128);
                for (int kb = x.kb0; kb < x.kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    tr(1);
                    uint8_t* st = smem + stage * SB;
                    const int k0 = kb * kBK;
                    mbar_arrive_expect_tx(&full[stage], bytes);
                    for (int c = 0; c < x.chunks; ++c) {
                        const int mc = x.m0 + c * 256 + (int)rank * 128;  // this CTA's 128 rows of chunk c
#pragma unroll
                        for (int j = 0; j < 128 / kW; ++j)
                            tma_load_2d_hint<1>(ma, &full[stage], st + args.b_bytes + c * kChunkBytes + j * kBK * 128, mc + j * kW,
                                                k0, pol_a);
                    }
                    tma_load_2d_hint<1>(mb, &full[stage], st, k0, (int)rank * (args.N_pad / 2), pol_b);
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 3) {
        // ---------------------------------------------------------------- relay (peer CTA)
        if (!leader && elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int u = pair; u < units; u += npairs) {
                const Unit x = decode(u);
                for (int kb = x.kb0; kb < x.kb1; ++kb) {
                    mbar_wait(&full[stage], phase);      // our half has landed
                    mbar_arrive_cluster(&full[stage], 0);  // tell the leader's MMA issuer
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA issuer (leader)
        if (leader && elect_one()) {
            Tr tr(1, 4);
            const uint32_t idesc = make_idesc(kKind, 256, args.N_pad, 1, 0);
            int stage = 0;
            uint32_t phase = 0;
            int iter = 0;
            for (int u = pair; u < units; u += npairs, ++iter) {
                const Unit x = decode(u);
                mbar_wait(tempty, (iter & 1) ^ 1);
                tr(12);
                tc_fence_after();
                for (int kb = x.kb0; kb < x.kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tr(11);
                    tc_fence_after();
                    const uint32_t st = smem_u32(smem + stage * SB);
                    const uint32_t b_addr = st;
                    for (int c = 0; c < x.chunks; ++c) {
                        const uint32_t a_addr = st + args.b_bytes + c * kChunkBytes;
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            mma_ss<2, kKind>(tmem_base + c * args.N_pad,
                                             kKind == 0 ? make_sdesc(a_addr + k * kUK * 128, kBK * 128, 1024)
                                                        : make_sdesc(a_addr + k * kUK * 128, kBK * 128, 512, 1),
                                             make_sdesc(b_addr + k * 32, 0, 1024), idesc,
                                             (kb > x.kb0 || k > 0) ? 1u : 0u);
                    }
                    mma_commit_pair(&empty[stage], 3);
                    if (!x.colsum)  // stand in for the 4 colsum warps (multicast to both CTAs)
                        for (int i = 0; i < 4; ++i) mma_commit_pair(&empty[stage], 3);
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
                mma_commit_pair(tfull, 3);
            }
        }
    } else if (warp >= 4) {
        // ---------------------------------------------------------------- epilogue (colsum, partials)
        const uint32_t q = warp & 3;
        const int t = (int)(q * 32 + lane);  // 0..127: TMEM lane == A row of this CTA's chunk
        Tr tr((lane == 0 && warp == 4) ? 2 : -1, 4);
        int stage = 0;
        uint32_t phase = 0;
        int iter = 0;
        for (int u = pair; u < units; u += npairs, ++iter) {
            const Unit x = decode(u);
            if (x.colsum) {
                // column sums of this CTA's staged A rows (= G columns) over the unit's tokens:
                // thread -> one 16-B chunk (kCPC columns) of one kW-wide block, 8 token rows.
                constexpr int kCPC = 16 / kElem;   // columns per 16-B chunk
                constexpr int kChunks = 128 / kCPC;  // 16-B chunks across 128 columns
                constexpr int kGroups = 128 / kChunks;  // row groups of 8 tokens
                const int chunk = t % kChunks, blk = chunk >> 3, ch = chunk & 7, r0 = (t / kChunks) * 8;
                float cs[kDutGroup][kCPC];
#pragma unroll
                for (int c = 0; c < kDutGroup; ++c)
#pragma unroll
                    for (int i = 0; i < kCPC; ++i) cs[c][i] = 0.f;
                for (int kb = x.kb0; kb < x.kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
#pragma unroll
                    for (int c = 0; c < kDutGroup; ++c) {
                        if (c >= x.chunks) break;
                        const uint32_t a = smem_u32(smem + stage * SB + args.b_bytes + c * kChunkBytes) + blk * kBK * 128;
#pragma unroll
                        for (int r = r0; r < r0 + 8; ++r) {
                            uint32_t w[4];
                            const uint32_t pch = kKind == 0 ? (uint32_t)(ch ^ (r & 7))
                                                            : (uint32_t)((((ch >> 1) ^ (r & 3)) << 1) | (ch & 1));
                            asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                                         : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                                         : "r"(a + r * 128 + (pch << 4)));
                            if constexpr (kKind == 0) {
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
                                    cs[c][2 * i] += f.x;
                                    cs[c][2 * i + 1] += f.y;
                                }
                            } else {
#pragma unroll
                                for (int i = 0; i < 4; ++i) cs[c][i] += __uint_as_float(w[i]);
                            }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[stage]);
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
                // combine the row groups in order -> cpart[u][rank][c][row]
                for (int c = 0; c < x.chunks; ++c) {
#pragma unroll
                    for (int i = 0; i < kCPC; ++i) csum_s[(c * 8 + t / kChunks) * 128 + chunk * kCPC + i] = cs[c][i];
                }
                named_bar_sync(2, 128);
                for (int c = 0; c < x.chunks; ++c) {
                    float s = 0.f;
#pragma unroll
                    for (int gq = 0; gq < kGroups; ++gq) s += csum_s[(c * 8 + gq) * 128 + t];
                    __stcg(args.cpart + (((long long)u * 2 + rank) * kDutGroup + c) * 128 + t, s);
                }
                named_bar_sync(2, 128);
            } else {
                for (int kb = x.kb0; kb < x.kb1; ++kb)  // keep the ring position; the MMA issuer arrives for us
                    if (++stage == S) { stage = 0; phase ^= 1; }
            }
            // ---- accumulators -> fp32 partials [u][rank][c][row t][N_pad]
            mbar_wait(tfull, iter & 1);
            tr(21);
            tc_fence_after();
            const int cbytes = 128 * args.N_pad * 4;  // one chunk's partial: 128 contiguous rows
            if (u + npairs >= units && 2 * cbytes <= S * SB) {
                // Last unit of this pair: the operand ring is idle, so each chunk is
                // staged in smem (row t at t * N_pad, the row's 16-B chunks written
                // in a lane-rotated order to spread banks) and leaves with ONE bulk
                // store, double-buffered.  Per-thread 16-B global stores along
                // 512-B rows ran at ~15 B/cycle (13k cycles for the 768x768
                // projection's 3 chunks).
                for (int c = 0; c < x.chunks; ++c) {
                    uint8_t* buf = smem + (c & 1) * cbytes;
                    if (c >= 2) {  // the store issued from this buffer two chunks ago has read it
                        if (t == 0) bulk_wait_read<1>();
                        named_bar_sync(2, 128);
                    }
                    const uint32_t row_s = smem_u32(buf) + (uint32_t)t * args.N_pad * 4;
                    const uint32_t t_row = tmem_base + ((q * 32u) << 16) + c * args.N_pad;
                    for (int n = 0; n < args.N_pad; n += 16) {
                        uint32_t v[16];
                        tmem_ld16(t_row + n, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int j = (i + t) & 3;
                            st_shared_v4(row_s + (uint32_t)(n + 4 * j) * 4, v[4 * j], v[4 * j + 1], v[4 * j + 2],
                                         v[4 * j + 3]);
                        }
                    }
                    fence_proxy_async_smem();
                    named_bar_sync(2, 128);
                    if (t == 0) {
                        bulk_store_1d(args.part + (((long long)u * 2 + rank) * kDutGroup + c) * 128 * args.N_pad, buf,
                                      (uint32_t)cbytes);
                        bulk_commit();
                    }
                }
                if (t == 0) bulk_wait<0>();
            } else
            for (int c = 0; c < x.chunks; ++c) {
                float* prow = args.part + ((((long long)u * 2 + rank) * kDutGroup + c) * 128 + t) * args.N_pad;
                const uint32_t t_row = tmem_base + ((q * 32u) << 16) + c * args.N_pad;
                for (int n = 0; n < args.N_pad; n += 16) {
                    uint32_t v[16];
                    tmem_ld16(t_row + n, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 16; i += 4)
                        __stcg(reinterpret_cast<float4*>(prow + n + i),
                               make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                                           __uint_as_float(v[i + 3])));
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(tempty);
                else mbar_arrive_cluster(tempty, 0);
            }
            tr(22);
        }
    }
    tc_fence_before();
    cluster_sync();  // the pair's MMAs into this CTA's TMEM are done before it is freed
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<2>(tmem_base, 512);
    }
}

// Split reduction of the dut partials: output (problem p, row m, rank column n)
// = alpha * sum over splits s = 0..S-1 of part[unit(p, g, s)][...] -- in split
// order, so bitwise reproducible -- scattered into the ABI layout; db likewise
// from the column-sum partials (unscaled).  A block reduces a tile of kRedRows
// consecutive partial rows: threads read float4s along the rows (coalesced,
// 8 splits x kRedV float4s in flight), park the sums in smem, then write the
// output with lanes along whichever index is contiguous in the ABI layout --
// m for dU1s (out[n][m]), n for dU2s -- so every warp store is one segment.
constexpr int kRedRows = 16, kRedCols = 32;  // block tile: 16 partial rows x 32 rank columns
__global__ void __launch_bounds__(128) dut_reduce_kernel(DutArgs args) {
    pdl_wait();
    pdl_launch_dependents();
    __shared__ float tile_s[kRedRows * (kRedCols + 1)];
    constexpr int ld = kRedCols + 1;
    const int S = args.splits, Np = args.N_pad;
    const long long ustride = 2LL * kDutGroup * 128 * Np;
    const int n0 = (int)blockIdx.y * kRedCols;                 // this block's rank columns
    const int ncols = min(kRedCols, args.N - n0);
    const int rr_t = (int)threadIdx.x / (kRedCols / 4), c4 = ((int)threadIdx.x % (kRedCols / 4)) * 4;
    for (int p = 0; p < 2; ++p) {
        const DutProblem& P = args.p[p];
        if (P.groups == 0 || ncols <= 0) continue;
        const int tiles = (P.M + kRedRows - 1) / kRedRows;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            const int m0 = tile * kRedRows;  // kRedRows divides 128: inside one partial half-chunk
            const int g = m0 / (256 * kDutGroup), mr = m0 % (256 * kDutGroup);
            const int c = mr / 256, r = (mr % 256) / 128, row0 = mr % 128;
            // thread: partial row row0 + rr_t, columns n0 + c4 .. + 3 (one float4 per split)
            if (n0 + c4 < Np) {
                const float* src = args.part + (long long)(P.unit0 + g * S) * ustride +
                                   (((long long)r * kDutGroup + c) * 128 + row0 + rr_t) * Np + n0 + c4;
                float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int s0 = 0; s0 < S; s0 += 16) {
                    float4 v[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (s0 + i < S) v[i] = __ldcg(reinterpret_cast<const float4*>(src + (long long)(s0 + i) * ustride));
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (s0 + i < S) { acc.x += v[i].x; acc.y += v[i].y; acc.z += v[i].z; acc.w += v[i].w; }
                }
                float* d = tile_s + rr_t * ld + c4;
                d[0] = acc.x * args.alpha; d[1] = acc.y * args.alpha;
                d[2] = acc.z * args.alpha; d[3] = acc.w * args.alpha;
            }
            __syncthreads();
            const int rows = min(kRedRows, P.M - m0);
            if (P.ms == 1) {  // out[n][m]: lanes along m, kRedRows consecutive floats per column
                for (int i = (int)threadIdx.x; i < rows * ncols; i += 128) {
                    const int nl = i / rows, rr = i % rows, n = n0 + nl;
                    P.out[(n / P.nb) * P.nbs + (n % P.nb) * P.ns + (long long)(m0 + rr)] = tile_s[rr * ld + nl];
                }
            } else {          // lanes along n
                for (int i = (int)threadIdx.x; i < rows * ncols; i += 128) {
                    const int rr = i / ncols, nl = i % ncols, n = n0 + nl;
                    P.out[(n / P.nb) * P.nbs + (n % P.nb) * P.ns + (long long)(m0 + rr) * P.ms] = tile_s[rr * ld + nl];
                }
            }
            __syncthreads();
        }
        if (P.colsum && P.db && blockIdx.y == 0) {
            for (long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x; m < P.M;
                 m += (long long)gridDim.x * blockDim.x) {
                const int g = (int)(m / (256 * kDutGroup)), mr = (int)(m % (256 * kDutGroup));
                const int c = mr / 256, r = (mr % 256) / 128, row = mr % 128;
                float acc = 0.f;
                for (int s = 0; s < S; ++s) {
                    const long long u = P.unit0 + (long long)g * S + s;
                    acc += __ldcg(args.cpart + ((u * 2 + r) * kDutGroup + c) * 128 + row);
                }
                P.db[m] = acc;
            }
        }
    }
}

}  // namespace dev
}  // namespace skl
