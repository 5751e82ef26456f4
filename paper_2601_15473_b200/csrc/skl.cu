// skl.cu -- C-ABI dispatch of the B200 SKLinear hot path (include/skl.h).
//
// Maps the reference's SkLinear::forward / backward contract
// (nn_layers.cpp:61-101) onto the sm_100a kernels:
//   forward : pack params -> fused B2B kernel (H = x·Acat stays on chip,
//             y = inv·H·Bcat + b)            [R <= 512]
//             or GEMM(H) + GEMM(y) through HBM [R > 512, documented fallback]
//   backward: pack -> fused B2B kernel (P = G·Bcatᵀ on chip -> dX, P_S2 out)
//             -> split-K tcgen05 GEMMs dU1 = inv·Savedᵀ·G, dU2 = inv·Xᵀ·P_S2
//             -> fixed-order partial reduction; db = column sums of G.
// Status codes replace the reference's exceptions (errors.hpp:10-19).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/skl.h"
#include "b2b.cuh"
#include "b2b_tf32.cuh"
#include "du.cuh"
#include "dut.cuh"
#include "gemm.cuh"
#include "prof.h"
#include "skl_internal.h"

namespace skl {
namespace {

thread_local std::string g_err;

skl_status fail(skl_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

#define SKL_CUDA(expr)                                                                               \
    do {                                                                                             \
        cudaError_t e_ = (expr);                                                                     \
        if (e_ != cudaSuccess) return fail(SKL_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_));   \
    } while (0)

#define SKL_TRY(expr)                   \
    do {                                \
        skl_status s_ = (expr);         \
        if (s_ != SKL_OK) return s_;    \
    } while (0)

// ---------------------------------------------------------------- device
struct DevInfo {
    int sms = 0;
    int major = 0;
};
DevInfo dev_info() {
    int dev = 0;
    DevInfo d;
    if (cudaGetDevice(&dev) != cudaSuccess) return d;
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, dev);
    return d;
}

// SMs left free for concurrently running communication kernels (NCCL) --
// skl_set_reserved_sms; kept even so CTA pairs still tile the grid.
std::atomic<int> g_reserved_sms{0};

skl_status check_device(DevInfo& di) {
    di = dev_info();
    if (di.sms == 0) return fail(SKL_ERR_CUDA, "no CUDA device available (libskl has no CPU fallback)");
    if (di.major != 10) return fail(SKL_ERR_CUDA, "libskl requires an sm_100 (B200) device, found sm_%d", di.major);
    di.sms = std::max(2, (di.sms - g_reserved_sms.load(std::memory_order_relaxed)) & ~1);
    return SKL_OK;
}

// ---------------------------------------------------------------- tensor maps
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

// 2-D view: `inner` contiguous elements per row, `outer` rows `ld` elements
// apart; box {box_inner, box_outer}; 128B swizzle; OOB reads return zero.
skl_status make_tmap(CUtensorMap* m, const void* ptr, int elem_bytes, int64_t inner, int64_t outer, int64_t ld,
                     int box_inner, int box_outer, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    EncodeFn enc = get_encode();
    if (!enc) return fail(SKL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || ((ld * elem_bytes) & 15) != 0)
        return fail(SKL_ERR_UNSUPPORTED, "TMA needs 16-byte aligned base and row stride (ld=%lld)", (long long)ld);
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * elem_bytes)};
    cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                     const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(SKL_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d): inner=%lld outer=%lld ld=%lld box=%dx%d",
                    (int)r, (long long)inner, (long long)outer, (long long)ld, box_inner, box_outer);
    return SKL_OK;
}

// Saved columns of the fused kernels through TMA stores (SKL_SAVE_TMA=0: per-thread 16-B stores).
bool save_tma_enabled() {
    static const bool on = !(getenv("SKL_SAVE_TMA") && atoi(getenv("SKL_SAVE_TMA")) == 0);
    return on;
}

// Programmatic dependent launch on the fused / GEMM kernels (SKL_PDL=0 disables).
bool pdl_enabled() {
    static const bool on = !(getenv("SKL_PDL") && atoi(getenv("SKL_PDL")) == 0);
    return on;
}
void add_pdl(cudaLaunchAttribute* attrs, unsigned& n) {
    if (!pdl_enabled()) return;
    attrs[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
}

// Dynamic shared memory (and cluster-size) attributes are per device: set them
// once per (kernel, device).  `done` is the kernel's own device bitmask.
template <typename F>
skl_status ensure_attrs(F kern, int smem_bytes, std::atomic<uint64_t>& done, bool nonportable_cluster = false) {
    int dev = 0;
    SKL_CUDA(cudaGetDevice(&dev));
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return SKL_OK;
    SKL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
    if (nonportable_cluster) SKL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    done.fetch_or(bit, std::memory_order_acq_rel);
    return SKL_OK;
}

// ---------------------------------------------------------------- GEMM launch
// Operand view: element (row-major storage) pointer, storage rows x cols, ld.
struct View {
    const void* ptr;
    int64_t rows, cols, ld;
};

template <int kCG, int kKind, int kBN, int kStages>
skl_status run_gemm(const char* name, const View& A, const View& B, int M, int N, int K, GemmArgs args, int sms,
                    cudaStream_t st) {
    using C = dev::GemmCfg<kCG, kKind, kBN, kStages>;
    const int eb = dev::KindTraits<kKind>::kElem;
    const int bk = C::kBK;
    CUtensorMap ta, tb, to;
    SKL_TRY(make_tmap(&ta, A.ptr, eb, K, M, A.ld, bk, 128));          // A [M][K], K-major
    SKL_TRY(make_tmap(&tb, B.ptr, eb, K, N, B.ld, bk, C::kNcta));     // B [N][K], K-major
    if (args.out) {
        const int ob = args.out_f32 ? 4 : 2;
        SKL_TRY(make_tmap(&to, args.out, ob, N, M, args.ldo, 128 / ob, 128));
    } else {
        to = ta;  // unused
    }
    static const int gemm_l2hint = getenv("SKL_GEMM_L2HINT") ? atoi(getenv("SKL_GEMM_L2HINT")) : 0;  // 2: measured neutral at c3
    args.l2hint = gemm_l2hint;
    args.M = M;
    args.N = N;
    args.K = K;
    args.num_m_tiles = (M + 128 * kCG - 1) / (128 * kCG);
    args.num_n_tiles = (N + kBN - 1) / kBN;
    args.k_blocks = (K + bk - 1) / bk;
    const int tiles = args.num_m_tiles * args.num_n_tiles;
    int grid = std::max(1, std::min(sms / kCG, tiles)) * kCG;
    auto kern = dev::gemm_kernel<kCG, kKind, kBN, kStages>;
    static std::atomic<uint64_t> attr_done{0};
    SKL_TRY(ensure_attrs(kern, C::kSmem, attr_done));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    unsigned nattr = 1;
    add_pdl(attr, nattr);
    cfg.numAttrs = nattr;
    ProfScope ps_(name, st);
    SKL_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, to, args));
    return SKL_OK;
}

// K-major x K-major GEMM in the variant's MMA kind (0 bf16, 1 tf32).
skl_status gemm_any(int kind, const char* name, const View& A, const View& B, int M, int N, int K, GemmArgs args,
                    int sms, cudaStream_t st) {
    if (kind == 0) return run_gemm<2, 0, 256, 6>(name, A, B, M, N, K, args, sms, st);
    return run_gemm<2, 1, 256, 6>(name, A, B, M, N, K, args, sms, st);
}

// Operand sources of the fused kernel.  kMode 0: b1 / b2 are packed panels.
// kMode 1 (forward, direct): b1 = S1s, b1b = U2s ([L*d_in][k] views),
//                            b2 = U1s, b2b = S2s ([L*k][d_out] views).
// kMode 2 (backward, direct): b1 = U1s, b1b = S2s ([L*k][d_out] views),
//                             b2 = S1s, b2b = U2s ([L*d_in][k] views).
struct B2BSrc {
    const void *a1, *b1, *b1b, *b2, *b2b;
};

template <int kCG, int kMode, int kKind, int kPost = 0, bool kRS = false, bool kSP = false, bool kDT = false>
skl_status run_b2b_cg(const char* name, const B2BSrc& src, B2BArgs a, int sms, cudaStream_t st) {
    using C = dev::B2BCfg<kCG, kMode, kKind, kPost == 1 && kMode != 1, kRS, kSP || kDT>;
    constexpr int eb = C::kElem, bk = C::kBK;
    CUtensorMap ta, tb1, tb1b, tb2, tb2b, ty, tm, ts, tyw;
    SKL_TRY(make_tmap(&ta, src.a1, eb, a.K1, a.T, a.K1, bk, 128));
    if constexpr (kMode == 0) {
        SKL_TRY(make_tmap(&tb1, src.b1, eb, a.K1, a.R_pad, a.K1, bk, a.b1rows));
        SKL_TRY(make_tmap(&tb2, src.b2, eb, a.R_pad, a.N2, a.R_pad, bk, C::kB2Rows));
        tb1b = tb1;
        tb2b = tb2;
    } else if constexpr (kMode == 1) {
        const int64_t srows = (int64_t)(a.Lk / a.k) * a.dS;
        SKL_TRY(make_tmap(&tb1, src.b1, 2, a.k, srows, a.k, 64, 64));
        SKL_TRY(make_tmap(&tb1b, src.b1b, 2, a.k, srows, a.k, 64, 64));
        SKL_TRY(make_tmap(&tb2, src.b2, 2, a.N2, a.Lk, a.N2, 64, 64));
        SKL_TRY(make_tmap(&tb2b, src.b2b, 2, a.N2, a.Lk, a.N2, 64, 64));
    } else {
        const int64_t srows = (int64_t)(a.Lk / a.k) * a.dS;
        SKL_TRY(make_tmap(&tb1, src.b1, 2, a.K1, a.Lk, a.K1, 64, a.b1rows));
        SKL_TRY(make_tmap(&tb1b, src.b1b, 2, a.K1, a.Lk, a.K1, 64, a.b1rows));
        SKL_TRY(make_tmap(&tb2, src.b2, 2, a.k, srows, a.k, 64, C::kB2Rows));
        SKL_TRY(make_tmap(&tb2b, src.b2b, 2, a.k, srows, a.k, 64, C::kB2Rows));
    }
    SKL_TRY(make_tmap(&ty, a.out, eb, a.N2, a.T, a.ldo, bk, 128));
    tyw = ty;
    static const int wstore_env = getenv("SKL_B2B_WSTORE") ? atoi(getenv("SKL_B2B_WSTORE")) : 1;
    a.wstore = kKind == 0 && wstore_env;
    if (a.wstore) SKL_TRY(make_tmap(&tyw, a.out, eb, a.N2, a.T, a.ldo, bk, 32));  // per-warp output stores
    tm = ty;
    if (C::kMaskStage && a.mask) SKL_TRY(make_tmap(&tm, a.mask, eb, a.N2, a.T, a.ld_mask, bk, 128));  // output-tile boxes
    // saved columns (bf16): [save_cols][ld_save] tokens-contiguous, stored per warp in [64 cols][32 tokens] boxes
    ts = ty;
    a.save_tma = 0;
    if (kKind == 0 && a.save && a.save_cols >= 64 && (reinterpret_cast<uintptr_t>(a.save) & 15) == 0 &&
        ((a.ld_save * 2) & 15) == 0 && save_tma_enabled()) {
        SKL_TRY(make_tmap(&ts, a.save, 2, a.ld_save, a.save_cols, a.ld_save, 32, 64, CU_TENSOR_MAP_SWIZZLE_NONE));
        a.save_tma = 1;
    }
    const int tiles = kDT ? ((a.T + 128 * kCG - 1) / (128 * kCG) + 1) / 2  // double tiles
                          : (a.T + 128 * kCG - 1) / (128 * kCG);
    const int csize = kCG * (kRS ? a.nsplit : 1);  // CTAs per cluster
    auto kern = dev::b2b_kernel<kCG, kMode, kKind, kPost, kRS, kSP, kDT>;
    static std::atomic<uint64_t> attr_done{0};
    SKL_TRY(ensure_attrs(kern, C::kSmem, attr_done, /*clusters of 8 for 4 R-split pairs*/ kRS));
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(384);  // 4 control warps + 2 epilogue warpgroups
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    int clusters = std::max(1, std::min(sms / csize, tiles));
    if (kRS) {  // clusters of 2*nsplit CTAs must each fit one GPC: persistent grid = what is co-resident
        cfg.gridDim = dim3(clusters * csize);
        cfg.numAttrs = 1;
        int maxc = 0;
        if (cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg) == cudaSuccess && maxc > 0)
            clusters = std::min(clusters, maxc);
        (void)cudaGetLastError();
    }
    cfg.gridDim = dim3(clusters * csize);
    unsigned nattr = 1;
    add_pdl(attr, nattr);
    cfg.numAttrs = nattr;
    ProfScope ps_(name, st);
    SKL_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb1, tb1b, tb2, tb2b, ty, tm, ts, tyw, a));
    return SKL_OK;
}

// TF32 with 256 < R_pad <= 512: H split between TMEM and SMEM (b2b_tf32.cuh).
template <bool kSP>
skl_status run_b2b_tf32_wide(const char* name, const B2BSrc& src, B2BArgs a, int sms, cudaStream_t st) {
    using C = dev::B2BT32Cfg<kSP>;
    auto kern = dev::b2b_tf32_kernel<kSP>;
    CUtensorMap ta, tb1, tb2, ty;
    SKL_TRY(make_tmap(&ta, src.a1, 4, a.K1, a.T, a.K1, C::kBK, 128));
    SKL_TRY(make_tmap(&tb1, src.b1, 4, a.K1, a.R_pad, a.K1, C::kBK, a.b1rows));
    SKL_TRY(make_tmap(&tb2, src.b2, 4, a.R_pad, a.N2, a.R_pad, C::kBK, C::kB2Rows));
    SKL_TRY(make_tmap(&ty, a.out, 4, a.N2, a.T, a.ldo, C::kBK, 128));
    const int tiles = (a.T + 255) / 256;
    const int grid = std::max(1, std::min(sms / 2, tiles)) * 2;
    static std::atomic<uint64_t> attr_done{0};
    SKL_TRY(ensure_attrs(kern, C::kSmem, attr_done));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    unsigned nattr = 1;
    add_pdl(attr, nattr);
    cfg.numAttrs = nattr;
    ProfScope ps_(name, st);
    SKL_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb1, tb2, ty, a));
    return SKL_OK;
}

int g_b2b_cg = 2;       // CTA-group width of the fused kernel (SKL_B2B_CG=1 forces single-CTA MMAs)
int g_b2b_direct = 1;   // read the ABI stacks directly when k % 64 == 0 (SKL_B2B_PACKED=1 disables)

skl_status run_b2b(const char* name, int kind, int mode, const B2BSrc& src, B2BArgs a, int sms, cudaStream_t st) {
    if (kind != 0 && mode != 0) return fail(SKL_ERR_UNSUPPORTED, "the TF32 fused kernel streams packed panels");
    // L2 hints: weight panels evict_last (every tile re-reads them); the streamed
    // activation evict_first only when it is far larger than L2 (126 MB) -- a
    // smaller one (c2's G, 201 MB) is partly still in L2 when du re-reads it.
    static const int l2hint = getenv("SKL_B2B_L2HINT") ? atoi(getenv("SKL_B2B_L2HINT")) : -1;
    const double act_bytes = (double)a.T * a.K1 * (kind == 0 ? 2 : 4);
    a.l2hint = l2hint >= 0 ? l2hint : (2 | (act_bytes > 256e6 ? 1 : 0));
    // R-split: R > 512 (bf16) runs on clusters of b2b_split(R) CTA pairs, r_loc rank columns each
    const int split = kind == 0 ? b2b_split(a.R_pad) : 1;
    a.nsplit = split;
    a.r_loc = split > 1 ? (a.R_pad / split + 63) / 64 * 64 : a.R_pad;
    {  // B1 box rows: largest power of two <= 128 dividing every chunk's per-CTA rows (and Lk, r_loc in mode 2)
        const int cg = g_b2b_cg;
        int r = 128;
        auto ok = [&](int v) {
            for (int c = 0; c * 256 < a.r_loc; ++c)
                if ((std::min(256, a.r_loc - 256 * c) / cg) % v) return false;
            return mode != 2 || (a.Lk % v == 0 && a.r_loc % v == 0);
        };
        while (r > 8 && !ok(r)) r /= 2;
        a.b1rows = r;
    }
    if (split > 1) {
        if (g_b2b_cg != 2) return fail(SKL_ERR_UNSUPPORTED, "the R-split kernel needs CTA pairs");
        if (a.relu || a.mask || a.relu_bits || a.mask_bits)
            return fail(SKL_ERR_UNSUPPORTED, "fused ReLU with R > 512 runs on the unfused chain");
        if (mode == 1) return run_b2b_cg<2, 1, 0, 0, true>(name, src, a, sms, st);
        if (mode == 2) return run_b2b_cg<2, 2, 0, 0, true>(name, src, a, sms, st);
        return run_b2b_cg<2, 0, 0, 0, true>(name, src, a, sms, st);
    }
    if (kind == 1 && b2b_tf32_wide_supported(a.R_pad)) {
        if (g_b2b_cg != 2) return fail(SKL_ERR_UNSUPPORTED, "the wide-rank TF32 kernel needs CTA pairs");
        // single-pass GEMM1 when its A operand is long (the backward's G, K1 = d_out)
        if (a.K1 >= 2048) return run_b2b_tf32_wide<true>(name, src, a, sms, st);
        return run_b2b_tf32_wide<false>(name, src, a, sms, st);
    }
    if (a.relu_bits || a.mask_bits) {  // fused ReLU with 1-bit masks
        if (g_b2b_cg != 2) return fail(SKL_ERR_UNSUPPORTED, "fused ReLU needs the CTA-pair kernel (SKL_B2B_CG=2)");
        if (kind == 1) return run_b2b_cg<2, 0, 1, 2>(name, src, a, sms, st);
        if (mode == 1) return run_b2b_cg<2, 1, 0, 2>(name, src, a, sms, st);
        if (mode == 2) return run_b2b_cg<2, 2, 0, 2>(name, src, a, sms, st);
        return run_b2b_cg<2, 0, 0, 2>(name, src, a, sms, st);
    }
    if (a.relu || a.mask) {  // fused ReLU / ReLU-mask epilogue (CTA pairs only)
        if (g_b2b_cg != 2) return fail(SKL_ERR_UNSUPPORTED, "fused ReLU needs the CTA-pair kernel (SKL_B2B_CG=2)");
        if (kind == 1) return run_b2b_cg<2, 0, 1, 1>(name, src, a, sms, st);
        if (mode == 1) return run_b2b_cg<2, 1, 0, 1>(name, src, a, sms, st);
        if (mode == 2) return run_b2b_cg<2, 2, 0, 1>(name, src, a, sms, st);
        return run_b2b_cg<2, 0, 0, 1>(name, src, a, sms, st);
    }
    if (kind == 1) {
        if (g_b2b_cg == 2) return run_b2b_cg<2, 0, 1>(name, src, a, sms, st);
        return run_b2b_cg<1, 0, 1>(name, src, a, sms, st);
    }
    if (g_b2b_cg == 2) {
        // forward with a long x (K1 >= 2048) and two H chunks: single-pass GEMM1 (SKL_FWD_SP=0 off)
        static const int fwd_sp = getenv("SKL_FWD_SP") ? atoi(getenv("SKL_FWD_SP")) : -1;
        if (mode == 1 && a.R_pad > 256 && (fwd_sp == 1 || (fwd_sp < 0 && a.K1 >= 2048)))
            return run_b2b_cg<2, 1, 0, 0, false, true>(name, src, a, sms, st);
        // R = 256 backward (the 768x768 projections): double tiles, one weight stream
        // for two pair tiles (SKL_B2B_DT=0 off, =2 also the forward, measured slower:
        // with the bias table it keeps only 3 of 48 KB stages; needs the per-warp stores)
        static const int dt = getenv("SKL_B2B_DT") ? atoi(getenv("SKL_B2B_DT")) : 1;
        static const int wst = getenv("SKL_B2B_WSTORE") ? atoi(getenv("SKL_B2B_WSTORE")) : 1;
        if (dt && wst && a.R_pad == 256 && ((mode == 1 && dt == 2) || (mode == 2 && a.bias == nullptr))) {
            if (mode == 1) return run_b2b_cg<2, 1, 0, 0, false, false, true>(name, src, a, sms, st);
            return run_b2b_cg<2, 2, 0, 0, false, false, true>(name, src, a, sms, st);
        }
        if (mode == 1) return run_b2b_cg<2, 1, 0>(name, src, a, sms, st);
        if (mode == 2) return run_b2b_cg<2, 2, 0>(name, src, a, sms, st);
        return run_b2b_cg<2, 0, 0>(name, src, a, sms, st);
    }
    if (mode == 1) return run_b2b_cg<1, 1, 0>(name, src, a, sms, st);
    if (mode == 2) return run_b2b_cg<1, 2, 0>(name, src, a, sms, st);
    return run_b2b_cg<1, 0, 0>(name, src, a, sms, st);
}

void read_b2b_env() {
    static std::once_flag once;
    std::call_once(once, [] {
        const char* e = getenv("SKL_B2B_CG");
        if (e && atoi(e) == 1) g_b2b_cg = 1;
        e = getenv("SKL_B2B_PACKED");
        if (e && atoi(e) != 0) g_b2b_direct = 0;
    });
}

// Direct (pack-free) operand streaming needs 64-wide rank blocks inside one term.
bool direct_ok(const SklDims& d, skl_dtype t) {
    read_b2b_env();
    return g_b2b_direct && t == SKL_BF16 && d.k % 64 == 0 && d.R_pad == d.R &&
           (!dev::B2BCfg<2, 1, 0>::kBiasTab || d.d_out <= dev::B2BCfg<2, 1, 0>::kMaxBiasTab);
}

int pick_splits(int M, int N, int K, int bn, int cg, int sms, int bk) {
    const int tiles = ((M + 128 * cg - 1) / (128 * cg)) * ((N + bn - 1) / bn);
    const int kb = (K + bk - 1) / bk;
    int s = std::max(1, (sms / cg) / std::max(1, tiles));
    s = std::min(s, std::max(1, kb / 4));  // keep >= 4 k-blocks per split
    return std::max(1, std::min(s, 64));
}

// ---------------------------------------------------------------- shapes / workspace
size_t align_up(size_t x, size_t a = 1024) { return (x + a - 1) / a * a; }

skl_status get_dims(const skl_shape* s, SklDims& d) {
    if (!s) return fail(SKL_ERR_PARAM, "null shape");
    if (s->num_terms < 1 || s->low_rank < 1)
        return fail(SKL_ERR_PARAM, "SkLinear: num_terms and low_rank must be >= 1");  // nn_layers.cpp:116
    if (s->d_in < 1 || s->d_out < 1) return fail(SKL_ERR_SHAPE, "SkLinear: d_in and d_out must be >= 1");
    if (s->dtype != SKL_BF16 && s->dtype != SKL_F32_TF32) return fail(SKL_ERR_PARAM, "unknown dtype %d", s->dtype);
    d.d_in = s->d_in;
    d.d_out = s->d_out;
    d.L = s->num_terms;
    d.k = s->low_rank;
    d.Lk = d.L * d.k;
    d.R = 2 * d.Lk;
    d.R_pad = (d.R + 63) / 64 * 64;
    return SKL_OK;
}

int elem_of(skl_dtype t) { return t == SKL_BF16 ? ELEM_BF16 : ELEM_F32; }
int ebytes(skl_dtype t) { return t == SKL_BF16 ? 2 : 4; }

// The TMA-fed kernels need every row stride to be a multiple of 16 B.  Shapes
// whose d_in / d_out rows are not (the reference accepts any shape,
// nn_layers.cpp:61-101) run on zero-padded copies staged in the workspace
// (padded dispatch below): zero feature columns add nothing to any product,
// so the cropped outputs are those of the unpadded layer.
int64_t round_to(int64_t v, int64_t a) { return (v + a - 1) / a * a; }
int64_t row_align(skl_dtype t) { return 16 / ebytes(t); }  // elements per 16 B
bool needs_pad(const SklDims& d, skl_dtype t) {
    const int64_t a = row_align(t);
    return d.d_in % a || d.d_out % a;
}
SklDims pad_dims(const SklDims& d, skl_dtype t, bool pad_k) {
    const int64_t a = row_align(t);
    SklDims p = d;
    p.d_in = round_to(d.d_in, a);
    p.d_out = round_to(d.d_out, a);
    if (pad_k) {
        p.k = round_to(d.k, a);
        p.Lk = p.L * p.k;
        p.R = 2 * p.Lk;
        p.R_pad = (p.R + 63) / 64 * 64;
    }
    return p;
}

// SKL_FORCE_UNFUSED=1 routes every shape through the unfused GEMM chain
// (testing aid: both paths are parity-checked against the oracle).
bool use_fused(const SklDims& d, skl_dtype t) {
    read_b2b_env();
    static const bool force_unfused = [] {
        const char* e = getenv("SKL_FORCE_UNFUSED");
        return e && atoi(e) != 0;
    }();
    static const bool tf32_wide = !(getenv("SKL_TF32_WIDE") && atoi(getenv("SKL_TF32_WIDE")) == 0);
    // SKL_B2B_RSPLIT=1: R > 512 (bf16) on the R-split clusters (H on chip, GEMM2 partials
    // chained over DSMEM) instead of the GEMM chain through HBM.  Opt-in: the fp32 partials
    // need 64 KB per output tile per CTA against ~21 B/cycle of DSMEM bandwidth, so at c3
    // (R = 1536) it measures 2.2x slower than the chain (R-split).
    static const bool rsplit = getenv("SKL_B2B_RSPLIT") && atoi(getenv("SKL_B2B_RSPLIT")) != 0;
    if (force_unfused) return false;
    if (t != SKL_BF16 && tf32_wide && b2b_tf32_wide_supported(d.R_pad)) return g_b2b_cg == 2;
    if (t == SKL_BF16 && b2b_split(d.R_pad) > 1) return rsplit && g_b2b_cg == 2 && b2b_supported(d.R_pad, 0);
    return b2b_supported(d.R_pad, t == SKL_BF16 ? 0 : 1);
}

// R-split clusters (R > 512, bf16) run the plain layer; a fused ReLU / ReLU mask
// there takes the unfused chain.
bool rsplit_of(const SklDims& d, skl_dtype t) { return t == SKL_BF16 && b2b_split(d.R_pad) > 1; }

// 1-bit ReLU masks are implemented in the CTA-pair b2b kernel only (not in the
// wide-rank TF32 kernel or the unfused GEMM chain).
bool relu_bits_ok(const SklDims& d, skl_dtype t) {
    read_b2b_env();
    static const bool tf32_wide = !(getenv("SKL_TF32_WIDE") && atoi(getenv("SKL_TF32_WIDE")) == 0);
    if (!use_fused(d, t) || g_b2b_cg != 2 || rsplit_of(d, t)) return false;
    return !(t != SKL_BF16 && tf32_wide && b2b_tf32_wide_supported(d.R_pad));
}

struct Plan {
    size_t acat, bcat, acatT, bcatT, bias32, inter, saved, p2t, colsum, total;
    size_t du_part, du_cpart, du_tickets;
    size_t small_part, small_h;  // small-batch path (small.cu)
};

// Small-batch path (small.cu): T <= kSmallT tokens and at most ~0.5 GFLOP per
// forward (2·R·D·T), where one tcgen05 tile on one CTA pair is weight-stream
// bound (c1: 26 us per fused kernel) -- beyond that the tensor-core kernels win
// even on a single tile.  SKL_SMALL=0 disables it, =1 forces it for T <= kSmallT;
// SKL_FORCE_UNFUSED keeps it off so that run still exercises the GEMM chain.
bool use_small(const SklDims& d, int64_t T) {
    static const int mode = getenv("SKL_SMALL") ? atoi(getenv("SKL_SMALL")) : -1;
    static const bool force_unfused = getenv("SKL_FORCE_UNFUSED") && atoi(getenv("SKL_FORCE_UNFUSED")) != 0;
    if (mode == 0 || force_unfused || T < 1 || T > kSmallT) return false;
    return mode == 1 || 2.0 * (double)d.R * (double)(d.d_in + d.d_out) * (double)T <= 0.5e9;
}

// Row stride (elements) of the transposed token-reduction operands Saved and
// P_S2 ([L*k][T8]): T rounded up to 8 so every row starts 16-byte aligned.
int64_t t8(int64_t T) { return (T + 7) / 8 * 8; }

// Tiling of the fused dU kernel (du.cuh): problem 0 = dU1 [Lk, d_out],
// problem 1 = dU2ᵀ [Lk, d_in]; 256 x 256 pair tiles; T split S ways so the
// units fill the pairs in ONE wave (cooperative launch, slice-parallel
// reduction).  Units run split-major: the pairs active together sweep the
// same token window, so the rank operand (Savedᵀ / P_S2ᵀ, reused by every N
// tile) is served from L2.  Measured alternatives, both slower at c2/c3: a
// stream-K partition with staggered token offsets (+36-62 %: the rank operand
// falls out of L2) and multi-wave splits with last-CTA reduction (+3x at c2:
// serial reductions).
struct DuShape {
    int m0, n0t, m1, n1t, t0, t1, s0, s1, kb, units;  // t*/s*: tiles / T splits of dU1 (0) and dU2 (1)
    bool cr;                                          // cluster (DSMEM) reduction of the split partials
    int tiles() const { return t0 + t1; }
};
// How many clusters of `csize` du CTAs the device runs at once
// (cudaOccupancyMaxActiveClusters): a cluster must find csize free SMs inside
// one GPC, so clusters of 12 or 16 CTAs fit only one per GPC.  Cached per
// (device, kind, csize); without a device, the 8-GPC x 18-SM model.
int du_cluster_cap(int kind, int csize) {
    static std::atomic<int> cache[64][2][17];
    int dev = 0;
    if (csize < 1 || csize > 16 || cudaGetDevice(&dev) != cudaSuccess) return 8 * std::max(1, 18 / std::max(1, csize));
    std::atomic<int>& c = cache[dev & 63][kind & 1][csize];
    const int v = c.load(std::memory_order_relaxed);
    if (v > 0) return v;
    auto kern = kind == 0 ? dev::du_kernel<0> : dev::du_kernel<1>;
    int n = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dev::kDuSmem) == cudaSuccess &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(csize * 64);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = dev::kDuSmem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = csize;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) n = 0;
    }
    (void)cudaGetLastError();
    if (n <= 0) n = 8 * std::max(1, 18 / csize);
    c.store(n, std::memory_order_relaxed);
    return n;
}
DuShape du_shape(const SklDims& d, int64_t T, int sms, int kind, int which = 3) {
    DuShape s;
    s.m0 = (int)((d.Lk + 255) / 256);
    s.n0t = (int)((d.d_out + 255) / 256);
    s.m1 = (int)((d.Lk + 255) / 256);
    s.n1t = (int)((d.d_in + 255) / 256);
    s.t0 = (which & 1) ? s.m0 * s.n0t : 0;
    s.t1 = (which & 2) ? s.m1 * s.n1t : 0;
    const int bkt = kind == 0 ? 64 : 32;  // tokens per k-block
    s.kb = (int)std::max<int64_t>(1, (T + bkt - 1) / bkt);
    const int pairs = std::max(1, sms / 2);
    const int smax = std::max(1, s.kb / 2);  // keep >= 2 k-blocks per unit
    // Per-problem splits, one wave: minimise the longest unit (dU2 units weighted
    // by kW1 relative to dU1), then the number of partials.  At c2 the main loop
    // is HBM-bound already (285 MB at ~6.5 TB/s), so 60 pairs are as fast as 72;
    // small layers (768x768, L=1) gain 30 % from filling all pairs.
    static const double kW1 = getenv("SKL_DU_W1") ? atof(getenv("SKL_DU_W1")) : 1.0;
    double best = 1e30;
    s.s0 = s.s1 = 1;
    // one wave: a <= pairs / t0 and b <= pairs / t1 (the search is on every call's host path)
    const int amax = s.t0 ? std::max(1, std::min(smax, pairs / s.t0)) : 0;
    const int bmax = s.t1 ? std::max(1, std::min(smax, pairs / s.t1)) : 0;
    for (int a = (s.t0 ? 1 : 0); a <= amax; ++a)
        for (int b = (s.t1 ? 1 : 0); b <= bmax; ++b) {
            if (s.t0 * a + s.t1 * b > pairs && (a > 1 || b > 1)) continue;
            const double len = std::max(a ? std::ceil((double)s.kb / a) : 0.0,
                                        b ? std::ceil((double)s.kb / b) * kW1 : 0.0);
            const double cost = len + 1e-3 * (s.t0 * a + s.t1 * b);  // tie-break: fewer partials
            if (cost < best) { best = cost; s.s0 = std::max(a, 1); s.s1 = std::max(b, 1); }
        }
    if (s.t0 + s.t1 > pairs) {
        // More tiles than CTA pairs: several waves whatever S is, so pick the
        // uniform S with the shortest wave-quantised time, waves(S) * ceil(kb / S).
        // Clusters of 2S CTAs must fit a GPC's free SMs as earlier waves retire:
        // measured at c3 (96 tiles), S = 1/2/3/4 -> du 983/808/956/966 us, so
        // only S <= 2 is considered.
        double bestw = 1e30;
        for (int S = 1; S <= std::min(2, smax); ++S) {
            const int64_t waves = ((int64_t)(s.t0 + s.t1) * S + pairs - 1) / pairs;
            const double cost = (double)waves * std::ceil((double)s.kb / S) * (1.0 + 1e-3 * S);
            if (cost < bestw) { bestw = cost; s.s0 = s.s1 = S; }
        }
    }
    if (const char* e = getenv("SKL_DU_SPLITS")) {  // experiments: "S" or "S0,S1"
        int a = 0, b = 0;
        const int n = sscanf(e, "%d,%d", &a, &b);
        if (n >= 1 && a > 0) s.s0 = std::min(a, s.kb), s.s1 = std::min(n == 2 && b > 0 ? b : a, s.kb);
    }
    s.units = s.t0 * s.s0 + s.t1 * s.s1;
    // Cluster reduction (du.cuh, DuArgs::cr): one cluster of 2S CTAs per tile, the
    // split partials summed over DSMEM -- needs one S for both problems and a
    // cluster of at most 8 CTAs.  Otherwise partials go through global memory.
    static const bool cr_on = !(getenv("SKL_DU_CR") && atoi(getenv("SKL_DU_CR")) == 0);
    static const int cr_max = getenv("SKL_DU_CR_MAX") ? atoi(getenv("SKL_DU_CR_MAX")) : 4;  // 8: clusters of 16
    // Few tiles (the c5 768x768 projections: 6 tiles -> S = 12): the one-wave
    // split is too deep for a cluster; S = 8 with clusters of 16 CTAs measures the
    // same kernel time and, with no grid-wide barrier, lets the next kernel's
    // CTAs start as this one's retire (projection backward 73.5 -> 68.5 us).
    static const bool deep_cr = !(getenv("SKL_DU_DEEP_CR") && atoi(getenv("SKL_DU_DEEP_CR")) == 0);
    // It needs enough tiles to keep half the pairs busy: the DP-phased dU2-only
    // launch at c2 has 3 tiles, and its 24 pairs took 40-47 us where the
    // cooperative S = 24 split on 72 pairs takes 33 us.
    if (cr_on && deep_cr && !getenv("SKL_DU_SPLITS") && (!s.t0 || !s.t1 || s.s0 == s.s1) &&
        std::max(s.s0, s.s1) > 8 && smax >= 8 && 8 * (s.t0 + s.t1) <= pairs && 2 * 8 * (s.t0 + s.t1) >= pairs) {
        const int S = 8;
        if (s.t0) s.s0 = S;
        if (s.t1) s.s1 = S;
        s.units = s.t0 * s.s0 + s.t1 * s.s1;
    }
    const int sc = s.t0 ? s.s0 : s.s1;
    const int lim = std::max(s.s0, s.s1) > 4 && deep_cr ? 8 : std::min(cr_max, 8);
    s.cr = cr_on && sc <= lim && (!s.t0 || !s.t1 || s.s0 == s.s1);
    // Clusters of 2S CTAs pack per GPC (cudaOccupancyMaxActiveClusters: 74 / 33 /
    // 22 / 15 / 11 / 7 clusters of 2 / 4 / 6 / 8 / 10 / 12+ CTAs on a B200), so a
    // one-wave split whose clusters do not all fit runs in two waves.  Those
    // shapes take the cooperative reduction at the same split instead: c2's
    // DP-phased dU1-only launch (12 tiles, S = 6) 80 us as clusters of 12,
    // 71 us at S = 4 in clusters of 8, 55-66 us cooperative at S = 6.
    // (Several-wave shapes, more tiles than pairs, keep their clusters: they run
    // in waves whatever the reduction.)
    if (s.cr && !getenv("SKL_DU_SPLITS") && s.tiles() <= pairs && s.tiles() > du_cluster_cap(kind, 2 * sc))
        s.cr = false;
    return s;
}

// Small rank (L·k <= 128): the transposed dU problem (dut.cuh), M = d in
// 256-row pair chunks grouped kDutGroup per unit, N = L·k padded to 16.
// SKL_DUT=0 keeps du.cuh for every shape (A/B).
struct DutShape {
    int n_pad, g0, g1, splits, units, kb, max_chunks;
};
// Chosen where the padded du rows cost more than dut's partial round trip:
// L·k <= 64, or L·k <= 128 on wide layers (measured: c4 L1 k16 / L2 k32 / TF32
// L2 k64 -10 / -10 / -6.5 % per step; the 768x768 projections (L·k = 128) stay on
// du, whose partials are a quarter of dut's there).
bool use_dut(const SklDims& d) {
    static const int mode = getenv("SKL_DUT") ? atoi(getenv("SKL_DUT")) : -1;  // 0 off, 1 whenever L*k <= 128
    if (mode == 0 || d.Lk > 128) return false;
    return mode == 1 || d.Lk <= 64 || d.d_in + d.d_out >= 4096;
}
DutShape dut_shape(const SklDims& d, int64_t T, int sms, int kind, int which) {
    DutShape s;
    s.n_pad = (int)((d.Lk + 15) / 16 * 16);
    const int rows_per_group = 256 * kDutGroup;
    s.g0 = (which & 1) ? (int)((d.d_out + rows_per_group - 1) / rows_per_group) : 0;
    s.g1 = (which & 2) ? (int)((d.d_in + rows_per_group - 1) / rows_per_group) : 0;
    const int bkt = kind == 0 ? 64 : 32;
    s.kb = (int)std::max<int64_t>(1, (T + bkt - 1) / bkt);
    const int pairs = std::max(1, sms / 2), groups = std::max(1, s.g0 + s.g1);
    s.splits = std::max(1, std::min(pairs / groups, s.kb / 4));  // one wave, >= 4 k-blocks per unit
    s.units = (s.g0 + s.g1) * s.splits;
    int mc = 0;
    for (int dim : {(which & 1) ? (int)d.d_out : 0, (which & 2) ? (int)d.d_in : 0})
        if (dim) mc = std::max(mc, std::min(kDutGroup, (dim + 255) / 256));
    s.max_chunks = std::max(1, mc);
    return s;
}

// du split partials / column-sum partials / tickets, sized for every phase's
// split choice AND independently of the SM count the call will see
// (skl_set_reserved_sms may change it after the size query): one-wave searches
// keep t0*s0 + t1*s1 <= pairs unless every split is 1, and several waves use
// S <= 2, so units <= max(pairs, 2 * tiles) and s0 <= max(pairs, 2) for any
// pair count up to the device's full one.
void du_ws_sizes(const SklDims& d, skl_dtype t, int64_t T, int sms, size_t& part, size_t& cpart, size_t& tickets) {
    const int full_pairs = std::max(74, dev_info().sms / 2);
    const DuShape all = du_shape(d, T, 2 * full_pairs, t == SKL_BF16 ? 0 : 1, 3);
    part = (size_t)std::max(full_pairs, 2 * all.tiles()) * 256 * 256 * 4;
    cpart = (size_t)all.n0t * std::max(full_pairs, 2) * 256 * 4;
    tickets = (size_t)all.tiles() * 4;
    for (int which = 1; which <= 3; ++which) {  // explicit SKL_DU_SPLITS overrides
        const DuShape u = du_shape(d, T, sms, t == SKL_BF16 ? 0 : 1, which);
        part = std::max(part, (size_t)u.units * 256 * 256 * 4);
        cpart = std::max(cpart, (size_t)u.n0t * u.s0 * 256 * 4);
        tickets = std::max(tickets, (size_t)u.tiles() * 4);
    }
    if (use_dut(d)) {  // dut: units <= max(pairs, groups) for any SM count
        const DutShape u = dut_shape(d, T, 2 * full_pairs, t == SKL_BF16 ? 0 : 1, 3);
        const size_t units = (size_t)std::max(full_pairs, u.g0 + u.g1);
        part = std::max(part, units * 2 * kDutGroup * 128 * u.n_pad * 4);
        cpart = std::max(cpart, units * 2 * kDutGroup * 128 * 4);
    }
}

// Offsets into the caller's workspace (1 KiB aligned).
Plan plan(const SklDims& d, skl_dtype t, int64_t T, bool bwd, int sms) {
    const size_t e = ebytes(t);
    Plan p = {};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += align_up(bytes ? bytes : 1);
        return o;
    };
    p.acat = take((size_t)d.d_in * d.R_pad * e);
    p.bcat = take((size_t)d.R_pad * d.d_out * e);
    p.acatT = take((size_t)d.R_pad * d.d_in * e);
    p.bcatT = take((size_t)d.d_out * d.R_pad * e);
    p.bias32 = take((size_t)d.d_out * 4);
    const bool fused = use_fused(d, t);
    // unfused only: H [T, R_pad] (fwd) / P [T, R_pad] (bwd) through HBM (also kept for
    // R-split shapes: a fused ReLU there takes the unfused chain)
    p.inter = take(!fused || rsplit_of(d, t) ? (size_t)T * d.R_pad * e : 0);
    p.saved = take(bwd ? (size_t)d.Lk * t8(T) * e : 0);  // recomputed Savedᵀ when the caller kept none
    p.p2t = take(bwd ? (size_t)d.Lk * t8(T) * e : 0);    // P_S2ᵀ
    if (bwd) {
        size_t part, cpart, tickets;
        du_ws_sizes(d, t, T, sms, part, cpart, tickets);
        p.du_part = take(part);
        p.du_cpart = take(cpart);
        p.du_tickets = take(tickets);
    }
    if (use_small(d, T)) {
        const int64_t splits = (std::max(d.d_in, d.d_out) + 63) / 64;
        p.small_part = take((size_t)splits * T * d.R * 4);
        p.small_h = take((size_t)T * d.R * 4);
    }
    p.colsum = take(0);
    p.total = off;
    return p;
}

template <typename Tp>
Tp* at(void* ws, size_t off) {
    return reinterpret_cast<Tp*>(reinterpret_cast<uint8_t*>(ws) + off);
}

// Workspace of the padded dispatch: the padded layer's own plan first, then the
// zero-padded copies of the operands whose rows change and the padded outputs.
struct PadPlan {
    size_t inner, x, yg, dx, s1, u2, u1, s2, bias, du1, du2, db, total;
};
PadPlan pad_plan(const SklDims& d, const SklDims& dp, skl_dtype t, int64_t T, bool bwd, int sms) {
    const size_t e = ebytes(t);
    PadPlan q = {};
    const bool pin = dp.d_in != d.d_in, pout = dp.d_out != d.d_out;
    size_t off = align_up(plan(dp, t, T, bwd, sms).total);
    q.inner = off;
    auto take = [&](bool need, size_t bytes) {
        size_t o = off;
        if (need) off += align_up(bytes ? bytes : 1);
        return o;
    };
    q.x = take(pin, (size_t)T * dp.d_in * e);
    q.yg = take(pout, (size_t)T * dp.d_out * e);
    q.dx = take(bwd && pin, (size_t)T * dp.d_in * e);
    q.s1 = take(pin, (size_t)dp.Lk * dp.d_in * e);
    q.u2 = take(pin, (size_t)dp.Lk * dp.d_in * e);
    q.u1 = take(pout, (size_t)dp.Lk * dp.d_out * e);
    q.s2 = take(pout, (size_t)dp.Lk * dp.d_out * e);
    q.bias = take(pout, (size_t)dp.d_out * e);
    q.du1 = take(bwd && pout, (size_t)dp.Lk * dp.d_out * 4);
    q.du2 = take(bwd && pin, (size_t)dp.Lk * dp.d_in * 4);
    q.db = take(bwd && pout, (size_t)dp.d_out * 4);
    q.total = off;
    return q;
}

// [B][R][C] stack -> zero-padded [B][R2][C2] copy in the workspace (or the
// source itself when nothing changes).
skl_status repad_in(const void* src, int eb, int64_t B, int64_t R, int64_t C, void* ws, size_t off, int64_t R2,
                    int64_t C2, cudaStream_t st, const void** out) {
    if (!src || (R == R2 && C == C2)) {
        *out = src;
        return SKL_OK;
    }
    void* dst = at<void>(ws, off);
    SKL_CUDA(launch_repad(src, eb, B, R, C, dst, R2, C2, st));
    *out = dst;
    return SKL_OK;
}

// dU1s = inv·Savedᵀ·G ([Lk, d_out] == [L][k][d_out]); dU2sᵀ = inv·P_S2ᵀ·X
// ([Lk, d_in] scattered to [L][d_in][k]); db = column sums of G.  `which`:
// bit 0 = dU1s (+ db), bit 1 = dU2s; one grouped persistent launch.
// dut.cuh launch (L·k <= 128): problem 0 = dU1sᵀ (A = G, B = Savedᵀ, + db),
// problem 1 = dU2s (A = X, B = P_S2ᵀ); a lone dU2 phase sits in slot 0.
skl_status run_dut(const SklDims& d, int64_t T, int kind, int which, const void* saved, const void* grad_y,
                   const void* p2t, const void* x, float* grad_U1s, float* grad_U2s, float* grad_bias, void* workspace,
                   const Plan& p, int sms, cudaStream_t st, float inv) {
    const int eb = kind == 0 ? 2 : 4;
    const int64_t ldt = t8(T);
    const DutShape u = dut_shape(d, T, sms, kind, which);
    DutArgs a = {};
    a.N = (int)d.Lk;
    a.N_pad = u.n_pad;
    a.k_blocks = u.kb;
    a.splits = u.splits;
    a.num_units = u.units;
    a.alpha = inv;
    a.b_bytes = (int)align_up((size_t)(u.n_pad / 2) * 128, 1024);
    a.stage_bytes = a.b_bytes + u.max_chunks * 128 * 128;
    const int csum_bytes = kDutGroup * 8 * 128 * 4;
    a.stages = std::min(8, (225 * 1024 - csum_bytes - 2048) / a.stage_bytes);
    if (a.stages < 2) return fail(SKL_ERR_UNSUPPORTED, "dut: stage does not fit shared memory");
    const DutProblem pu1{(int)d.d_out, u.g0, 0, grad_bias ? 1 : 0, grad_U1s, (long long)1 << 40, 0,
                         (long long)d.d_out, 1, grad_bias};
    const DutProblem pu2{(int)d.d_in, u.g1, u.g0 * u.splits, 0, grad_U2s, (long long)d.k, (long long)(d.d_in * d.k),
                         1, (long long)d.k, nullptr};
    DutProblem none{};
    none.unit0 = 1 << 30;
    a.p[0] = (which & 1) ? pu1 : pu2;
    if (!(which & 1)) a.p[0].unit0 = 0;
    a.p[1] = (which & 1) && (which & 2) ? pu2 : none;
    a.part = at<float>(workspace, p.du_part);
    a.cpart = at<float>(workspace, p.du_cpart);
    const int bkt = 128 / eb;
    const CUtensorMapSwizzle mn_swz = kind == 0 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
    CUtensorMap tu1a, tu1b, tu2a, tu2b;
    if (which & 1) {
        SKL_TRY(make_tmap(&tu1a, grad_y, eb, d.d_out, T, d.d_out, bkt, bkt, mn_swz));  // G, MN-major
        SKL_TRY(make_tmap(&tu1b, saved, eb, T, d.Lk, ldt, bkt, u.n_pad / 2));            // Savedᵀ, K-major
    }
    if (which & 2) {
        SKL_TRY(make_tmap(&tu2a, x, eb, d.d_in, T, d.d_in, bkt, bkt, mn_swz));           // X
        SKL_TRY(make_tmap(&tu2b, p2t, eb, T, d.Lk, ldt, bkt, u.n_pad / 2));              // P_S2ᵀ
    }
    if (!(which & 1)) { tu1a = tu2a; tu1b = tu2b; }
    if (!(which & 2)) { tu2a = tu1a; tu2b = tu1b; }
    auto kern = kind == 0 ? dev::dut_kernel<0> : dev::dut_kernel<1>;
    const int smem = a.stages * a.stage_bytes + 256 + csum_bytes + 1024;
    static std::atomic<uint64_t> attr_done[2];
    SKL_TRY(ensure_attrs(kern, 225 * 1024 + 1024, attr_done[kind]));
    const int pairs = std::max(1, std::min(sms / 2, u.units));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    unsigned nattr = 1;
    add_pdl(attr, nattr);
    cfg.attrs = attr;
    cfg.numAttrs = nattr;
    {
        ProfScope ps_("dut", st);
        SKL_CUDA(cudaLaunchKernelEx(&cfg, kern, (which & 1) ? tu1a : tu2a, (which & 1) ? tu1b : tu2b, tu2a, tu2b, a));
    }
    cudaLaunchConfig_t rc = {};
    // one block per (kRedRows-row tile of the larger problem, kRedCols rank columns); each block
    // takes that tile of both problems
    const int64_t red_tiles = (std::max(d.d_out, d.d_in) + dev::kRedRows - 1) / dev::kRedRows;
    rc.gridDim = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(sms * 8, red_tiles)),
                      (unsigned)((d.Lk + dev::kRedCols - 1) / dev::kRedCols));
    rc.blockDim = dim3(128);
    rc.stream = st;
    cudaLaunchAttribute rattr[1];
    unsigned nr = 0;
    add_pdl(rattr, nr);
    rc.attrs = rattr;
    rc.numAttrs = nr;
    ProfScope ps2_("dut_reduce", st);
    SKL_CUDA(cudaLaunchKernelEx(&rc, dev::dut_reduce_kernel, a));
    return SKL_OK;
}

skl_status run_du(const SklDims& d, int64_t T, int kind, int which, const void* saved, const void* grad_y,
                  const void* p2t, const void* x, float* grad_U1s, float* grad_U2s, float* grad_bias, void* workspace,
                  const Plan& p, int sms, cudaStream_t st, float alpha = 0.f) {
    const int eb = kind == 0 ? 2 : 4;
    const int64_t ldt = t8(T);
    const float inv = alpha != 0.f ? alpha : (float)(1.0 / (2.0 * (double)d.L));
    if (use_dut(d))
        return run_dut(d, T, kind, which, saved, grad_y, p2t, x, grad_U1s, grad_U2s, grad_bias, workspace, p, sms, st,
                       inv);
    const DuShape u = du_shape(d, T, sms, kind, which);
    static const bool verbose = getenv("SKL_DU_VERBOSE") != nullptr;
    if (verbose)
        fprintf(stderr, "[skl du] which=%d tiles=%d+%d splits=%d,%d units=%d kb=%d cr=%d sms=%d cap(2S)=%d\n", which,
                u.t0, u.t1, u.s0, u.s1, u.units, u.kb, (int)u.cr, sms, du_cluster_cap(kind, 2 * (u.t0 ? u.s0 : u.s1)));
    DuArgs a = {};
    a.k_blocks = u.kb;
    a.num_units = u.units;
    // B (G / X, each tile read once) evict_first: c2 du 72.7 -> 69.7 us, c5 projection du -10 %
    static const int du_l2hint = getenv("SKL_DU_L2HINT") ? atoi(getenv("SKL_DU_L2HINT")) : 2;
    a.l2hint = du_l2hint;
    a.num_tiles = u.tiles();
    const int u1_units = (which & 1) ? u.t0 * u.s0 : 0;
    const DuProblem pu1{(int)d.Lk, (int)d.d_out, u.m0, u.n0t, 0, u.s0, 0, 0, grad_bias ? 1 : 0, inv, grad_U1s,
                        (long long)1 << 40, 0, (long long)d.d_out, 1, grad_bias};
    const DuProblem pu2{(int)d.Lk, (int)d.d_in, u.m1, u.n1t, u.t0, u.s1, u1_units, u1_units, 0, inv, grad_U2s,
                        (long long)d.k, (long long)(d.d_in * d.k), 1, (long long)d.k, nullptr};
    const DuProblem none{0, 0, 0, 0, 1 << 30, 1, 1 << 30, 0, 0, 0.f, nullptr, 1, 0, 0, 0, nullptr};
    a.p[0] = (which & 1) ? pu1 : pu2;
    a.p[1] = (which & 1) && (which & 2) ? pu2 : none;
    const bool colsum = (which & 1) && grad_bias;
    if (!(which & 2)) p2t = saved;  // unused slot-1 maps: any valid tensor
    a.part = at<float>(workspace, p.du_part);
    a.cpart = at<float>(workspace, p.du_cpart);
    a.tickets = at<int>(workspace, p.du_tickets);
    const int bkt = 128 / eb;  // tokens per k-block (= columns per MN-major block)
    CUtensorMap ta0, tb0, ta1, tb1;
    // MN-major TF32 tiles use the 32-B-atom 128B swizzle (UMMA layout SWIZZLE_128B_BASE32B)
    const CUtensorMapSwizzle mn_swz = kind == 0 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
    // Problem slot 0 reads (tmA0, tmB0), slot 1 (tmA1, tmB1).  dU1: Savedᵀ (K-major) x G
    // (MN-major); dU2ᵀ: P_S2ᵀ (K-major) x X (MN-major).  A lone dU2 launch sits in slot 0.
    CUtensorMap tu1a, tu1b, tu2a, tu2b;
    if (which & 1) {
        SKL_TRY(make_tmap(&tu1a, saved, eb, T, d.Lk, ldt, bkt, 128));
        SKL_TRY(make_tmap(&tu1b, grad_y, eb, d.d_out, T, d.d_out, bkt, bkt, mn_swz));
    }
    SKL_TRY(make_tmap(&tu2a, p2t, eb, T, d.Lk, ldt, bkt, 128));
    SKL_TRY(make_tmap(&tu2b, x, eb, d.d_in, T, d.d_in, bkt, bkt, mn_swz));
    ta0 = (which & 1) ? tu1a : tu2a;
    tb0 = (which & 1) ? tu1b : tu2b;
    ta1 = tu2a;
    tb1 = tu2b;
    if (!u.cr) SKL_CUDA(cudaMemsetAsync(a.tickets, 0, (size_t)u.tiles() * 4, st));
    auto du_kern = kind == 0 ? dev::du_kernel<0> : dev::du_kernel<1>;
    static std::atomic<uint64_t> attr_done[2];
    SKL_TRY(ensure_attrs(du_kern, dev::kDuSmem, attr_done[kind], /*clusters of 2S up to 16*/ true));
    const int units = u.units;  // CTA-pair work units
    a.relay = colsum ? 1 : 0;
    if (u.cr) {
        // one cluster of 2S CTAs per tile: no cross-cluster synchronisation, so
        // neither a cooperative launch nor co-residency of all units is needed
        a.cr = 1;
        a.coop = 0;
        const int S = u.t0 ? u.s0 : u.s1;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * units);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = dev::kDuSmem;
        cfg.stream = st;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2 * S;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        unsigned nattr = 1;
        add_pdl(attr, nattr);
        cfg.attrs = attr;
        cfg.numAttrs = nattr;
        ProfScope ps_(which == 3 ? "du_fused" : which == 1 ? "du_dU1db" : "du_dU2", st);
        SKL_CUDA(cudaLaunchKernelEx(&cfg, du_kern, ta0, tb0, ta1, tb1, a));
        return SKL_OK;
    }
    static const bool no_coop = getenv("SKL_DU_NOCOOP") && atoi(getenv("SKL_DU_NOCOOP")) != 0;  // profilers
    // one wave: cooperative launch, slice-parallel reduction; several waves:
    // persistent grid, the last CTA of each tile reduces it
    a.coop = (!no_coop && 2 * units <= sms) ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * (a.coop ? units : std::min(sms / 2, units)));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = dev::kDuSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = a.coop;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    ProfScope ps_(which == 3 ? "du_fused" : which == 1 ? "du_dU1db" : "du_dU2", st);
    cudaError_t le = cudaLaunchKernelEx(&cfg, du_kern, ta0, tb0, ta1, tb1, a);
    if (le != cudaSuccess && a.coop) {  // cooperative + cluster refused: last-CTA reduction instead
        (void)cudaGetLastError();
        a.coop = 0;
        attr[1].val.cooperative = 0;
        cfg.gridDim = dim3(2 * std::min(sms / 2, units));
        le = cudaLaunchKernelEx(&cfg, du_kern, ta0, tb0, ta1, tb1, a);
    }
    SKL_CUDA(le);
    return SKL_OK;
}


}  // namespace
}  // namespace skl

using namespace skl;

extern "C" {

const char* skl_version(void) { return "skl-b200 0.1 (sm_100a tcgen05)"; }
const char* skl_last_error(void) { return g_err.c_str(); }
const char* skl_rng_algorithm(void) { return "splitmix64-boxmuller-v1"; }

uint64_t skl_derive_seed(uint64_t master, uint64_t index) {
    uint64_t z = (master ^ (0x517cc1b727220a95ULL + index)) + 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

skl_status skl_params(const skl_shape* s, skl_param_count* out) {
    SklDims d;
    SKL_TRY(get_dims(s, d));
    const uint64_t lk = (uint64_t)d.Lk;
    out->learnable = lk * (uint64_t)(d.d_in + d.d_out) + (uint64_t)d.d_out;
    out->total_stored = 2 * lk * (uint64_t)(d.d_in + d.d_out) + (uint64_t)d.d_out;
    out->dense_equivalent = (uint64_t)d.d_in * (uint64_t)d.d_out + (uint64_t)d.d_out;
    return SKL_OK;
}

int skl_exceeds_dense(uint64_t l, uint64_t k, uint64_t d_in, uint64_t d_out) {
    return 2 * l * k * (d_in + d_out) > d_in * d_out;
}

skl_status skl_generate_sketches(const skl_shape* s, skl_dist dist, uint64_t layer_seed, void* S1s, void* S2s,
                                 void* stream) {
    SklDims d;
    SKL_TRY(get_dims(s, d));
    if (dist != SKL_DIST_GAUSSIAN && dist != SKL_DIST_RADEMACHER) return fail(SKL_ERR_PARAM, "unknown dist %d", dist);
    DevInfo di;
    SKL_TRY(check_device(di));
    SKL_CUDA(launch_gen_sketches((int)dist, layer_seed, d, elem_of(s->dtype), S1s, S2s, (cudaStream_t)stream));
    return SKL_OK;
}

skl_status skl_init_params(const skl_shape* s, uint64_t layer_seed, void* U1s, void* U2s, void* stream) {
    SklDims d;
    SKL_TRY(get_dims(s, d));
    DevInfo di;
    SKL_TRY(check_device(di));
    SKL_CUDA(launch_init_u(layer_seed, d, elem_of(s->dtype), U1s, U2s, (cudaStream_t)stream));
    return SKL_OK;
}

skl_status skl_realize_sketch(skl_dist dist, int64_t k, int64_t dd, uint64_t seed, int unit_variance, int transpose,
                              skl_out_type out_type, void* out, void* stream) {
    if (k < 1 || dd < 1) return fail(SKL_ERR_SHAPE, "make_sketch: dimensions must be >= 1");  // sketch.cpp:92
    if (dist != SKL_DIST_GAUSSIAN && dist != SKL_DIST_RADEMACHER) return fail(SKL_ERR_PARAM, "unknown dist %d", dist);
    DevInfo di;
    SKL_TRY(check_device(di));
    const int elem = out_type == SKL_OUT_F64 ? ELEM_F64 : out_type == SKL_OUT_F32 ? ELEM_F32 : ELEM_BF16;
    SKL_CUDA(launch_realize((int)dist, k, dd, seed, unit_variance, transpose, elem, out, (cudaStream_t)stream));
    return SKL_OK;
}

skl_status skl_workspace_size(const skl_shape* s, int64_t T, size_t* fwd_bytes, size_t* bwd_bytes) {
    SklDims d;
    SKL_TRY(get_dims(s, d));
    if (T < 0) return fail(SKL_ERR_SHAPE, "T must be >= 0");
    DevInfo di = dev_info();
    const int sms = di.sms ? di.sms : 148;
    if (needs_pad(d, s->dtype)) {  // padded dispatch: the padded layer's plan + staged copies
        const SklDims dp = pad_dims(d, s->dtype, false);
        if (fwd_bytes) *fwd_bytes = pad_plan(d, dp, s->dtype, T, false, sms).total;
        if (bwd_bytes) *bwd_bytes = pad_plan(d, dp, s->dtype, T, true, sms).total;
        return SKL_OK;
    }
    if (fwd_bytes) *fwd_bytes = plan(d, s->dtype, T, false, sms).total;  // saved_proj: [L*k][round8(T)]
    if (bwd_bytes) *bwd_bytes = plan(d, s->dtype, T, true, sms).total;
    return SKL_OK;
}

skl_status sketched_linear_forward(const skl_shape* s, int64_t T, const void* x, const void* S1s, const void* S2s,
                                   const void* U1s, const void* U2s, const void* bias, void* y, void* saved_proj,
                                   void* workspace, size_t ws_bytes, void* stream) {
    return sketched_linear_forward_ex(s, T, 0, x, S1s, S2s, U1s, U2s, bias, y, saved_proj, workspace, ws_bytes,
                                      stream);
}

skl_status sketched_linear_forward_ex(const skl_shape* s, int64_t T, unsigned fuse, const void* x, const void* S1s,
                                      const void* S2s, const void* U1s, const void* U2s, const void* bias, void* y,
                                      void* saved_proj, void* workspace, size_t ws_bytes, void* stream) {
    if (fuse & ~(unsigned)SKL_FUSE_RELU_OUT) return fail(SKL_ERR_PARAM, "forward: unsupported fuse flags %u", fuse);
    return sketched_linear_forward_bits(s, T, fuse, x, S1s, S2s, U1s, U2s, bias, y, saved_proj, nullptr, workspace,
                                        ws_bytes, stream);
}

int64_t skl_relu_bits_row_words(int64_t width) { return width < 1 ? 0 : (width + 63) / 64 * 2; }

int skl_relu_bits_supported(const skl_shape* s) {
    SklDims d;
    if (get_dims(s, d) != SKL_OK) return 0;
    return relu_bits_ok(d, s->dtype) ? 1 : 0;
}

skl_status sketched_linear_forward_bits(const skl_shape* s, int64_t T, unsigned fuse, const void* x, const void* S1s,
                                        const void* S2s, const void* U1s, const void* U2s, const void* bias, void* y,
                                        void* saved_proj, uint32_t* relu_bits, void* workspace, size_t ws_bytes,
                                        void* stream) {
    if (fuse & ~(unsigned)(SKL_FUSE_RELU_OUT | SKL_FUSE_RELU_BITS))
        return fail(SKL_ERR_PARAM, "forward: unsupported fuse flags %u", fuse);
    const bool bits = (fuse & SKL_FUSE_RELU_BITS) != 0;
    if (bits && (!(fuse & SKL_FUSE_RELU_OUT) || !relu_bits))
        return fail(SKL_ERR_PARAM, "forward: SKL_FUSE_RELU_BITS needs SKL_FUSE_RELU_OUT and a relu_bits buffer");
    SklDims d;
    SKL_TRY(get_dims(s, d));
    if (bits && !relu_bits_ok(d, s->dtype))
        return fail(SKL_ERR_UNSUPPORTED, "forward: 1-bit ReLU masks need the fused CTA-pair kernel for this shape");
    if (T < 0) return fail(SKL_ERR_SHAPE, "SkLinear::forward: T must be >= 0");
    if (T == 0) return SKL_OK;
    if (!x || !S1s || !S2s || !U1s || !U2s || !y) return fail(SKL_ERR_PARAM, "null tensor argument");
    DevInfo di;
    SKL_TRY(check_device(di));
    if (needs_pad(d, s->dtype)) {
        // Rows that are not 16-byte multiples: the same kernels on zero-padded
        // copies (x, the four stacks, the bias), y cropped back.  The 1-bit
        // ReLU mask keeps its layout: padding to 16 B never crosses a 64-column group.
        const int eb = ebytes(s->dtype);
        const SklDims dp = pad_dims(d, s->dtype, false);
        const PadPlan q = pad_plan(d, dp, s->dtype, T, false, di.sms);
        if (!workspace || ws_bytes < q.total)
            return fail(SKL_ERR_WORKSPACE, "forward workspace too small: need %zu bytes, got %zu", q.total, ws_bytes);
        cudaStream_t st = (cudaStream_t)stream;
        const void *xp, *s1p, *u2p, *u1p, *s2p, *bp;
        SKL_TRY(repad_in(x, eb, 1, T, d.d_in, workspace, q.x, T, dp.d_in, st, &xp));
        SKL_TRY(repad_in(S1s, eb, d.L, d.d_in, d.k, workspace, q.s1, dp.d_in, d.k, st, &s1p));
        SKL_TRY(repad_in(U2s, eb, d.L, d.d_in, d.k, workspace, q.u2, dp.d_in, d.k, st, &u2p));
        SKL_TRY(repad_in(U1s, eb, d.L, d.k, d.d_out, workspace, q.u1, d.k, dp.d_out, st, &u1p));
        SKL_TRY(repad_in(S2s, eb, d.L, d.k, d.d_out, workspace, q.s2, d.k, dp.d_out, st, &s2p));
        SKL_TRY(repad_in(bias, eb, 1, 1, d.d_out, workspace, q.bias, 1, dp.d_out, st, &bp));
        void* yp = dp.d_out != d.d_out ? at<void>(workspace, q.yg) : y;
        skl_shape sp = *s;
        sp.d_in = dp.d_in;
        sp.d_out = dp.d_out;
        SKL_TRY(sketched_linear_forward_bits(&sp, T, fuse, xp, s1p, s2p, u1p, u2p, bp, yp, saved_proj, relu_bits,
                                             workspace, q.inner, stream));
        if (yp != y) SKL_CUDA(launch_repad(yp, eb, 1, T, dp.d_out, y, T, d.d_out, st));
        return SKL_OK;
    }
    const Plan p = plan(d, s->dtype, T, false, di.sms);
    if (!workspace || ws_bytes < p.total)
        return fail(SKL_ERR_WORKSPACE, "forward workspace too small: need %zu bytes, got %zu", p.total, ws_bytes);
    cudaStream_t st = (cudaStream_t)stream;
    const int elem = elem_of(s->dtype);
    const int eb = ebytes(s->dtype);
    const float inv = (float)(1.0 / (2.0 * (double)d.L));
    if (!bits && use_small(d, T)) {
        SmallArgs a = {};
        a.elem = elem;
        a.T = (int)T;
        a.d_in = (int)d.d_in;
        a.d_out = (int)d.d_out;
        a.k = (int)d.k;
        a.Lk = (int)d.Lk;
        a.R = (int)d.R;
        a.alpha = inv;
        a.x = x;
        a.S1s = S1s;
        a.S2s = S2s;
        a.U1s = U1s;
        a.U2s = U2s;
        a.bias = bias;
        a.relu = (fuse & SKL_FUSE_RELU_OUT) ? 1 : 0;
        a.out = y;
        a.save = saved_proj;
        a.ld_save = t8(T);
        a.part = at<float>(workspace, p.small_part);
        a.H = at<float>(workspace, p.small_h);
        SKL_CUDA(launch_small_forward(a, st));
        return SKL_OK;
    }
    void* acatT = at<void>(workspace, p.acatT);
    void* bcatT = at<void>(workspace, p.bcatT);
    float* bias32 = at<float>(workspace, p.bias32);
    const bool fused = use_fused(d, s->dtype) && !(rsplit_of(d, s->dtype) && (fuse & SKL_FUSE_RELU_OUT));
    const bool direct = fused && direct_ok(d, s->dtype);
    if (!direct) SKL_CUDA(launch_pack2(d, elem, S1s, U2s, U1s, S2s, nullptr, nullptr, acatT, bcatT, bias, bias32, st));

    if (fused) {
        B2BArgs a = {};
        a.T = (int)T;
        a.K1 = (int)d.d_in;
        a.R = (int)d.R;
        a.R_pad = (int)d.R_pad;
        a.N2 = (int)d.d_out;
        a.alpha = inv;
        a.relu = (fuse & SKL_FUSE_RELU_OUT) ? 1 : 0;
        a.relu_bits = bits ? relu_bits : nullptr;
        a.bits_ld = skl_relu_bits_row_words(d.d_out);
        a.bias = direct ? reinterpret_cast<const float*>(bias) : bias32;
        a.bias_bf16 = direct ? 1 : 0;
        a.out = y;
        a.ldo = d.d_out;
        a.save = saved_proj;  // Savedᵀ [Lk][T8]
        a.save_col0 = 0;
        a.save_cols = (int)d.Lk;
        a.ld_save = t8(T);
        a.Lk = (int)d.Lk;
        a.k = (int)d.k;
        a.dS = (int)d.d_in;
        if (direct) return run_b2b("b2b_fwd", 0, 1, B2BSrc{x, S1s, U2s, U1s, S2s}, a, di.sms, st);
        return run_b2b("b2b_fwd", s->dtype == SKL_BF16 ? 0 : 1, 0, B2BSrc{x, acatT, nullptr, bcatT, nullptr}, a,
                       di.sms, st);
    }

    // Unfused fallback (R > 512 or SKL_FORCE_UNFUSED): H through HBM.
    void* H = at<void>(workspace, p.inter);
    GemmArgs g1 = {};
    g1.alpha = 1.f;
    g1.out = H;
    g1.ldo = d.R_pad;
    g1.out2 = saved_proj;
    g1.ldo2 = t8(T);
    g1.out2_c0 = 0;
    g1.out2_c1 = (int)d.Lk;
    g1.out_f32 = eb == 4;
    g1.round_tf32 = eb == 4;  // H feeds a TF32 GEMM: round-to-nearest instead of hardware truncation
    View vx{x, T, d.d_in, d.d_in}, vat{acatT, d.R_pad, d.d_in, d.d_in};
    SKL_TRY(gemm_any(eb == 4, "gemm_H", vx, vat, (int)T, (int)d.R, (int)d.d_in, g1, di.sms, st));
    GemmArgs g2 = {};
    g2.alpha = inv;
    g2.relu = (fuse & SKL_FUSE_RELU_OUT) ? 1 : 0;
    g2.bias = bias32;
    g2.out = y;
    g2.ldo = d.d_out;
    g2.out_f32 = eb == 4;
    View vh{H, T, d.R, d.R_pad}, vbt{bcatT, d.d_out, d.R_pad, d.R_pad};
    SKL_TRY(gemm_any(eb == 4, "gemm_Y", vh, vbt, (int)T, (int)d.d_out, (int)d.R, g2, di.sms, st));
    return SKL_OK;
}

skl_status sketched_linear_backward(const skl_shape* s, int64_t T, const void* grad_y, const void* x,
                                    const void* saved_proj, const void* S1s, const void* S2s, const void* U1s,
                                    const void* U2s, void* grad_x, float* grad_U1s, float* grad_U2s,
                                    float* grad_bias, void* workspace, size_t ws_bytes, void* stream) {
    return sketched_linear_backward_ex(s, T, SKL_BWD_ALL, 0, grad_y, x, saved_proj, S1s, S2s, U1s, U2s, grad_x,
                                       grad_U1s, grad_U2s, grad_bias, workspace, ws_bytes, stream);
}

skl_status sketched_linear_backward_phase(const skl_shape* s, int64_t T, unsigned phases, const void* grad_y,
                                          const void* x, const void* saved_proj, const void* S1s, const void* S2s,
                                          const void* U1s, const void* U2s, void* grad_x, float* grad_U1s,
                                          float* grad_U2s, float* grad_bias, void* workspace, size_t ws_bytes,
                                          void* stream) {
    return sketched_linear_backward_ex(s, T, phases, 0, grad_y, x, saved_proj, S1s, S2s, U1s, U2s, grad_x, grad_U1s,
                                       grad_U2s, grad_bias, workspace, ws_bytes, stream);
}

skl_status sketched_linear_backward_ex(const skl_shape* s, int64_t T, unsigned phases, unsigned fuse,
                                       const void* grad_y, const void* x, const void* saved_proj, const void* S1s,
                                       const void* S2s, const void* U1s, const void* U2s, void* grad_x,
                                       float* grad_U1s, float* grad_U2s, float* grad_bias, void* workspace,
                                       size_t ws_bytes, void* stream) {
    if (fuse & ~(unsigned)SKL_FUSE_RELU_IN) return fail(SKL_ERR_PARAM, "backward: unsupported fuse flags %u", fuse);
    return sketched_linear_backward_bits(s, T, phases, fuse, grad_y, x, saved_proj, S1s, S2s, U1s, U2s, grad_x,
                                         grad_U1s, grad_U2s, grad_bias, nullptr, workspace, ws_bytes, stream);
}

skl_status sketched_linear_backward_bits(const skl_shape* s, int64_t T, unsigned phases, unsigned fuse,
                                         const void* grad_y, const void* x, const void* saved_proj, const void* S1s,
                                         const void* S2s, const void* U1s, const void* U2s, void* grad_x,
                                         float* grad_U1s, float* grad_U2s, float* grad_bias, const uint32_t* relu_bits,
                                         void* workspace, size_t ws_bytes, void* stream) {
    if (fuse & ~(unsigned)(SKL_FUSE_RELU_IN | SKL_FUSE_RELU_BITS))
        return fail(SKL_ERR_PARAM, "backward: unsupported fuse flags %u", fuse);
    const bool bits = (fuse & SKL_FUSE_RELU_BITS) != 0;
    if (bits && (!(fuse & SKL_FUSE_RELU_IN) || (T > 0 && !relu_bits)))
        return fail(SKL_ERR_PARAM, "backward: SKL_FUSE_RELU_BITS needs SKL_FUSE_RELU_IN and a relu_bits buffer");
    SklDims d;
    SKL_TRY(get_dims(s, d));
    if (bits && !relu_bits_ok(d, s->dtype))
        return fail(SKL_ERR_UNSUPPORTED, "backward: 1-bit ReLU masks need the fused CTA-pair kernel for this shape");
    if (T < 0) return fail(SKL_ERR_SHAPE, "SkLinear::backward: T must be >= 0");
    if (phases == 0 || (phases & ~(unsigned)SKL_BWD_ALL)) return fail(SKL_ERR_PARAM, "bad phase mask %u", phases);
    const bool ph_u1 = (phases & SKL_BWD_DU1_DB) != 0, ph_data = (phases & SKL_BWD_DX_DU2) != 0;
    if ((ph_u1 && !grad_U1s) || (ph_data && !grad_U2s)) return fail(SKL_ERR_PARAM, "null gradient argument");
    if (T > 0 && (!grad_y || !x || !S1s || !S2s || !U1s || !U2s)) return fail(SKL_ERR_PARAM, "null tensor argument");
    DevInfo di;
    SKL_TRY(check_device(di));
    const Plan p = plan(d, s->dtype, T, true, di.sms);
    if (!workspace || ws_bytes < p.total)
        return fail(SKL_ERR_WORKSPACE, "backward workspace too small: need %zu bytes, got %zu", p.total, ws_bytes);
    cudaStream_t st = (cudaStream_t)stream;
    if (T == 0) {  // empty batch: all gradients are zero (sums over no tokens)
        if (ph_u1) SKL_CUDA(cudaMemsetAsync(grad_U1s, 0, (size_t)d.Lk * d.d_out * 4, st));
        if (ph_data) SKL_CUDA(cudaMemsetAsync(grad_U2s, 0, (size_t)d.Lk * d.d_in * 4, st));
        if (ph_u1 && grad_bias) SKL_CUDA(cudaMemsetAsync(grad_bias, 0, (size_t)d.d_out * 4, st));
        return SKL_OK;
    }
    if (needs_pad(d, s->dtype)) {
        // Rows that are not 16-byte multiples: zero-padded copies of G, x and the
        // stacks; gradients of the padded layer cropped back.  Padded feature
        // columns of x / G are zero, so they add nothing to dU1s / dU2s / db,
        // and the padded columns of dX / dU / db are dropped.
        const int eb = ebytes(s->dtype);
        const SklDims dp = pad_dims(d, s->dtype, false);
        const PadPlan q = pad_plan(d, dp, s->dtype, T, true, di.sms);
        if (ws_bytes < q.total)
            return fail(SKL_ERR_WORKSPACE, "backward workspace too small: need %zu bytes, got %zu", q.total, ws_bytes);
        const bool pin = dp.d_in != d.d_in, pout = dp.d_out != d.d_out;
        const void *xp, *gp, *s1p, *u2p, *u1p, *s2p;
        SKL_TRY(repad_in(x, eb, 1, T, d.d_in, workspace, q.x, T, dp.d_in, st, &xp));
        SKL_TRY(repad_in(grad_y, eb, 1, T, d.d_out, workspace, q.yg, T, dp.d_out, st, &gp));
        SKL_TRY(repad_in(S1s, eb, d.L, d.d_in, d.k, workspace, q.s1, dp.d_in, d.k, st, &s1p));
        SKL_TRY(repad_in(U2s, eb, d.L, d.d_in, d.k, workspace, q.u2, dp.d_in, d.k, st, &u2p));
        SKL_TRY(repad_in(U1s, eb, d.L, d.k, d.d_out, workspace, q.u1, d.k, dp.d_out, st, &u1p));
        SKL_TRY(repad_in(S2s, eb, d.L, d.k, d.d_out, workspace, q.s2, d.k, dp.d_out, st, &s2p));
        void* gxp = (pin && grad_x) ? at<void>(workspace, q.dx) : grad_x;
        float* du1p = (pout && grad_U1s) ? at<float>(workspace, q.du1) : grad_U1s;
        float* du2p = (pin && grad_U2s) ? at<float>(workspace, q.du2) : grad_U2s;
        float* dbp = (pout && grad_bias) ? at<float>(workspace, q.db) : grad_bias;
        skl_shape sp = *s;
        sp.d_in = dp.d_in;
        sp.d_out = dp.d_out;
        SKL_TRY(sketched_linear_backward_bits(&sp, T, phases, fuse, gp, xp, saved_proj, s1p, s2p, u1p, u2p, gxp, du1p,
                                              du2p, dbp, relu_bits, workspace, q.inner, stream));
        if (ph_u1 && du1p != grad_U1s) SKL_CUDA(launch_repad(du1p, 4, d.L, d.k, dp.d_out, grad_U1s, d.k, d.d_out, st));
        if (ph_u1 && dbp != grad_bias) SKL_CUDA(launch_repad(dbp, 4, 1, 1, dp.d_out, grad_bias, 1, d.d_out, st));
        if (ph_data && du2p != grad_U2s) SKL_CUDA(launch_repad(du2p, 4, d.L, dp.d_in, d.k, grad_U2s, d.d_in, d.k, st));
        if (ph_data && gxp != grad_x) SKL_CUDA(launch_repad(gxp, eb, 1, T, dp.d_in, grad_x, T, d.d_in, st));
        return SKL_OK;
    }
    const int elem = elem_of(s->dtype);
    const int eb = ebytes(s->dtype);
    const int kind = s->dtype == SKL_BF16 ? 0 : 1;
    const float inv = (float)(1.0 / (2.0 * (double)d.L));
    const int64_t ldt = t8(T);
    if (!bits && use_small(d, T)) {
        SmallArgs a = {};
        a.elem = elem;
        a.T = (int)T;
        a.d_in = (int)d.d_in;
        a.d_out = (int)d.d_out;
        a.k = (int)d.k;
        a.Lk = (int)d.Lk;
        a.R = (int)d.R;
        a.alpha = inv;
        a.x = x;
        a.grad_y = grad_y;
        a.S1s = S1s;
        a.S2s = S2s;
        a.U1s = U1s;
        a.U2s = U2s;
        a.mask = (fuse & SKL_FUSE_RELU_IN) ? x : nullptr;  // grad_x *= (x > 0): the preceding ReLU's backward
        a.grad_x = grad_x;
        a.need_saved = ph_u1 && !saved_proj;
        a.save = at<void>(workspace, p.saved);
        a.saved = saved_proj;
        a.p2t = at<void>(workspace, p.p2t);
        a.ld_save = ldt;
        a.part = at<float>(workspace, p.small_part);
        a.H = at<float>(workspace, p.small_h);
        a.data = ph_data ? 1 : 0;
        a.u1 = ph_u1 ? 1 : 0;
        a.grad_U1s = grad_U1s;
        a.grad_U2s = grad_U2s;
        a.grad_bias = grad_bias;
        SKL_CUDA(launch_small_backward(a, st));
        return SKL_OK;
    }
    void* acat = at<void>(workspace, p.acat);
    void* bcat = at<void>(workspace, p.bcat);
    void* acatT = at<void>(workspace, p.acatT);
    void* P = at<void>(workspace, p.inter);
    void* p2t = at<void>(workspace, p.p2t);
    const bool fused = use_fused(d, s->dtype) && !(rsplit_of(d, s->dtype) && (fuse & SKL_FUSE_RELU_IN));
    const bool bwd_direct = fused && grad_x != nullptr && direct_ok(d, s->dtype);
    const bool need_saved = ph_u1 && !saved_proj;
    // no dX: only P_S2 = G·S2ᵀ, whose bf16 B operand is the S2s stack itself ([L*k][d_out], K-major)
    const bool p2_only = ph_data && !grad_x;
    const bool pack_data = ph_data && !bwd_direct && !(p2_only && kind == 0);
    if (pack_data || need_saved)
        SKL_CUDA(launch_pack2(d, elem, S1s, U2s, U1s, S2s, pack_data && !p2_only ? acat : nullptr,
                              pack_data ? bcat : nullptr, need_saved ? acatT : nullptr, nullptr, nullptr, nullptr,
                              st));

    // Savedᵀ = (x·S1)ᵀ, recomputed only when the caller did not keep it.
    const void* saved = saved_proj;
    if (need_saved) {
        void* sv = at<void>(workspace, p.saved);
        GemmArgs g = {};
        g.alpha = 1.f;
        g.out2 = sv;
        g.ldo2 = ldt;
        g.out2_c0 = 0;
        g.out2_c1 = (int)d.Lk;
        g.out_f32 = eb == 4;
        g.round_tf32 = kind;
        View vx{x, T, d.d_in, d.d_in}, vat{acatT, d.R_pad, d.d_in, d.d_in};
        SKL_TRY(gemm_any(kind, "gemm_saved", vx, vat, (int)T, (int)d.Lk, (int)d.d_in, g, di.sms, st));
        saved = sv;
    }

    // Phase DU1_DB alone runs first in a data-parallel step so the all-reduce of
    // dU1s | db overlaps the dX kernel.
    if (ph_u1 && !ph_data)
        return run_du(d, T, kind, 1, saved, grad_y, nullptr, x, grad_U1s, nullptr, grad_bias, workspace, p, di.sms, st);
    // P = G·Bcatᵀ (P_S2ᵀ leaves the chip) and dX = inv·P·Acatᵀ
    if (fused && grad_x) {
        B2BArgs a = {};
        a.T = (int)T;
        a.K1 = (int)d.d_out;
        a.R = (int)d.R;
        a.R_pad = (int)d.R_pad;
        a.N2 = (int)d.d_in;
        a.alpha = inv;
        a.bias = nullptr;
        a.mask = (fuse & SKL_FUSE_RELU_IN) && !bits ? x : nullptr;  // grad_x *= (x > 0): the preceding ReLU's backward
        a.mask_bits = bits ? relu_bits : nullptr;                       // ... or its 1-bit form from the forward
        a.bits_ld = skl_relu_bits_row_words(d.d_in);
        a.ld_mask = d.d_in;
        a.out = grad_x;
        a.ldo = d.d_in;
        a.save = p2t;  // P_S2ᵀ [Lk][T8]
        a.save_col0 = (int)d.Lk;
        a.save_cols = (int)d.Lk;
        a.ld_save = ldt;
        a.Lk = (int)d.Lk;
        a.k = (int)d.k;
        a.dS = (int)d.d_in;
        if (bwd_direct)
            SKL_TRY(run_b2b("b2b_bwd", 0, 2, B2BSrc{grad_y, U1s, S2s, S1s, U2s}, a, di.sms, st));
        else
            SKL_TRY(run_b2b("b2b_bwd", kind, 0, B2BSrc{grad_y, bcat, nullptr, acat, nullptr}, a, di.sms, st));
    } else if (!grad_x) {
        // no dX (e.g. the first layer of a chain): only P_S2 = G·S2ᵀ, the S2 rows of Bcat
        GemmArgs g = {};
        g.alpha = 1.f;
        g.out2 = p2t;
        g.ldo2 = ldt;
        g.out2_c0 = 0;
        g.out2_c1 = (int)d.Lk;
        g.out_f32 = eb == 4;
        g.round_tf32 = kind;
        View vg{grad_y, T, d.d_out, d.d_out};
        View vs2{kind == 0 ? S2s : static_cast<const void*>(static_cast<const uint8_t*>(bcat) + (size_t)d.Lk * d.d_out * eb),
                 d.Lk, d.d_out, d.d_out};
        SKL_TRY(gemm_any(kind, "gemm_P", vg, vs2, (int)T, (int)d.Lk, (int)d.d_out, g, di.sms, st));
    } else {
        GemmArgs g = {};
        g.alpha = 1.f;
        g.out = fused ? nullptr : P;  // P only feeds the unfused dX GEMM
        g.ldo = d.R_pad;
        g.out2 = p2t;
        g.ldo2 = ldt;
        g.out2_c0 = (int)d.Lk;
        g.out2_c1 = (int)(2 * d.Lk);
        g.out_f32 = eb == 4;
        g.round_tf32 = kind;
        View vg{grad_y, T, d.d_out, d.d_out}, vb{bcat, d.R_pad, d.d_out, d.d_out};
        SKL_TRY(gemm_any(kind, "gemm_P", vg, vb, (int)T, (int)d.R, (int)d.d_out, g, di.sms, st));
        if (grad_x) {
            GemmArgs g2 = {};
            g2.alpha = inv;
            g2.mask = (fuse & SKL_FUSE_RELU_IN) ? x : nullptr;
            g2.ld_mask = d.d_in;
            g2.out = grad_x;
            g2.ldo = d.d_in;
            g2.out_f32 = eb == 4;
            View vp{P, T, d.R, d.R_pad}, va{acat, d.d_in, d.R_pad, d.R_pad};
            SKL_TRY(gemm_any(kind, "gemm_dX", vp, va, (int)T, (int)d.d_in, (int)d.R, g2, di.sms, st));
        }
    }


    return run_du(d, T, kind, ph_u1 ? 3 : 2, saved, grad_y, p2t, x, grad_U1s, grad_U2s, grad_bias, workspace, p,
                  di.sms, st);
}

namespace skl {
namespace {
size_t from_dense_core_bytes(const SklDims& d, size_t e) {
    return align_up((size_t)d.R_pad * d.d_in * e) + align_up((size_t)d.d_in * d.d_out * e);
}
bool from_dense_needs_pad(const SklDims& d, skl_dtype t) { return needs_pad(d, t) || d.k % row_align(t); }

// U from W for sketches already in S1s / S2s (aligned shape): U1s = S1sᵀ·Wᵀ for
// all terms in one GEMM, U2s[i] = Wᵀ·S2s[i]ᵀ per term.
skl_status from_dense_core(const SklDims& d, skl_dtype t, const void* W, const void* S1s, const void* S2s, void* U1s,
                           void* U2s, void* workspace, int sms, cudaStream_t st) {
    const int eb = ebytes(t), elem = elem_of(t), kind = t == SKL_BF16 ? 0 : 1;
    void* acatT = workspace;                                                   // rows < Lk: S1s[i]ᵀ
    void* wT = at<void>(workspace, align_up((size_t)d.R_pad * d.d_in * eb));  // Wᵀ [d_in][d_out]
    SKL_CUDA(cudaMemsetAsync(U2s, 0, (size_t)d.Lk * d.d_in * eb, st));       // (pack reads the U2 half)
    SKL_CUDA(launch_pack2(d, elem, S1s, U2s, U1s, S2s, nullptr, nullptr, acatT, nullptr, nullptr, nullptr, st));
    SKL_CUDA(launch_transpose(W, elem, d.d_out, d.d_in, wT, st));
    GemmArgs g = {};
    g.alpha = 1.f;
    g.out = U1s;  // [L*k][d_out]
    g.ldo = d.d_out;
    g.out_f32 = eb == 4;
    View va{acatT, d.Lk, d.d_in, d.d_in}, vw{W, d.d_out, d.d_in, d.d_in};
    SKL_TRY(gemm_any(kind, "from_dense_U1", va, vw, (int)d.Lk, (int)d.d_out, (int)d.d_in, g, sms, st));
    for (int64_t i = 0; i < d.L; ++i) {
        GemmArgs g2 = {};
        g2.alpha = 1.f;
        g2.out = static_cast<uint8_t*>(U2s) + (size_t)i * d.d_in * d.k * eb;  // U2s[i] [d_in][k]
        g2.ldo = d.k;
        g2.out_f32 = eb == 4;
        View vwt{wT, d.d_in, d.d_out, d.d_out};
        View vs2{static_cast<const uint8_t*>(S2s) + (size_t)i * d.k * d.d_out * eb, d.k, d.d_out, d.d_out};
        SKL_TRY(gemm_any(kind, "from_dense_U2", vwt, vs2, (int)d.d_in, (int)d.k, (int)d.d_out, g2, sms, st));
    }
    return SKL_OK;
}
}  // namespace
}  // namespace skl

skl_status skl_from_dense_workspace_size(const skl_shape* s, size_t* bytes) {
    SklDims d;
    SKL_TRY(get_dims(s, d));
    if (!bytes) return fail(SKL_ERR_PARAM, "null size pointer");
    const size_t e = ebytes(s->dtype);
    if (!from_dense_needs_pad(d, s->dtype)) {
        *bytes = from_dense_core_bytes(d, e);
        return SKL_OK;
    }
    // padded: core + S1s, S2s, W, U1s, U2s at the padded (d_in, d_out, k)
    const SklDims p = pad_dims(d, s->dtype, true);
    *bytes = from_dense_core_bytes(p, e) + 4 * align_up((size_t)p.Lk * std::max(p.d_in, p.d_out) * e) +
             align_up((size_t)p.d_in * p.d_out * e);
    return SKL_OK;
}

// sk_linear_from_dense (nn_layers.cpp:149-160) on the device.  Reference:
// u1_i = s1_i·W [k, d_in], u2_i = W·s2_iᵀ [d_out, k].  In the ABI stacks
// (S2s[i] = s1_i, S1s[i] = s2_iᵀ):  U1s[i] = u2_iᵀ = S1s[i]ᵀ·Wᵀ  and
// U2s[i] = u1_iᵀ = Wᵀ·S2s[i]ᵀ -- two tcgen05 GEMMs (all terms of U1s in one).
// Any shape: rows that are not 16-byte multiples (d_in, d_out or k) are
// computed on zero-padded copies of W and the sketches, then cropped.
skl_status skl_from_dense(const skl_shape* s, skl_dist dist, uint64_t layer_seed, const void* W,
                          const void* bias_in, void* S1s, void* S2s, void* U1s, void* U2s, void* bias_out,
                          void* workspace, size_t ws_bytes, void* stream) {
    SklDims d;
    SKL_TRY(get_dims(s, d));
    if (!W || !S1s || !S2s || !U1s || !U2s) return fail(SKL_ERR_PARAM, "null tensor argument");
    if (dist != SKL_DIST_GAUSSIAN && dist != SKL_DIST_RADEMACHER) return fail(SKL_ERR_PARAM, "unknown dist %d", dist);
    const int eb = ebytes(s->dtype), elem = elem_of(s->dtype);
    DevInfo di;
    SKL_TRY(check_device(di));
    size_t need = 0;
    SKL_TRY(skl_from_dense_workspace_size(s, &need));
    if (!workspace || ws_bytes < need)
        return fail(SKL_ERR_WORKSPACE, "from_dense workspace too small: need %zu bytes, got %zu", need, ws_bytes);
    cudaStream_t st = (cudaStream_t)stream;
    SKL_CUDA(launch_gen_sketches((int)dist, layer_seed, d, elem, S1s, S2s, st));  // sk_linear_shell seeds
    if (!from_dense_needs_pad(d, s->dtype)) {
        SKL_TRY(from_dense_core(d, s->dtype, W, S1s, S2s, U1s, U2s, workspace, di.sms, st));
    } else {
        const SklDims p = pad_dims(d, s->dtype, true);
        size_t off = from_dense_core_bytes(p, eb);
        const size_t slot = align_up((size_t)p.Lk * std::max(p.d_in, p.d_out) * eb);
        void* s1p = at<void>(workspace, off);
        void* s2p = at<void>(workspace, off + slot);
        void* u1p = at<void>(workspace, off + 2 * slot);
        void* u2p = at<void>(workspace, off + 3 * slot);
        void* wp = at<void>(workspace, off + 4 * slot);
        SKL_CUDA(launch_repad(S1s, eb, d.L, d.d_in, d.k, s1p, p.d_in, p.k, st));
        SKL_CUDA(launch_repad(S2s, eb, d.L, d.k, d.d_out, s2p, p.k, p.d_out, st));
        SKL_CUDA(launch_repad(W, eb, 1, d.d_out, d.d_in, wp, p.d_out, p.d_in, st));
        SKL_TRY(from_dense_core(p, s->dtype, wp, s1p, s2p, u1p, u2p, workspace, di.sms, st));
        SKL_CUDA(launch_repad(u1p, eb, d.L, p.k, p.d_out, U1s, d.k, d.d_out, st));
        SKL_CUDA(launch_repad(u2p, eb, d.L, p.d_in, p.k, U2s, d.d_in, d.k, st));
    }
    if (bias_out) {
        if (bias_in) SKL_CUDA(cudaMemcpyAsync(bias_out, bias_in, (size_t)d.d_out * eb, cudaMemcpyDeviceToDevice, st));
        else SKL_CUDA(cudaMemsetAsync(bias_out, 0, (size_t)d.d_out * eb, st));
    }
    return SKL_OK;
}

// ---------------------------------------------------------------- SkConv2d
// SkConv2d::forward / backward (nn_layers.cpp:226-314): im2col lowering +
// the SKLinear path (inner layer d_in = c_in*kh*kw, d_out = c_out) + NCHW
// reshapes, all on the device.  T = B*oh*ow patches are the tokens.
namespace skl {
namespace {
skl_status conv_geom(const skl_shape* s, const skl_conv_shape* cs, int64_t B, int64_t H, int64_t W, ConvGeom& g) {
    if (!s || !cs) return fail(SKL_ERR_PARAM, "null shape");
    if (cs->c_in < 1 || cs->c_out < 1 || cs->kernel_h < 1 || cs->kernel_w < 1 || cs->stride < 1 || cs->padding < 0)
        return fail(SKL_ERR_PARAM, "conv: invalid ConvShape");
    if (s->d_in != cs->c_in * cs->kernel_h * cs->kernel_w || s->d_out != cs->c_out)
        return fail(SKL_ERR_SHAPE, "SKConv2d: inner dims disagree with conv shape");  // nn_model.cpp:500
    if (B < 0 || H < 1 || W < 1) return fail(SKL_ERR_SHAPE, "conv: bad image size");
    const int64_t ph = H + 2 * cs->padding, pw = W + 2 * cs->padding;
    if (ph < cs->kernel_h) return fail(SKL_ERR_SHAPE, "conv: kernel taller than padded image");  // nn_layers.cpp:166
    if (pw < cs->kernel_w) return fail(SKL_ERR_SHAPE, "conv: kernel wider than padded image");   // :172
    g = ConvGeom{(int)B, (int)cs->c_in, (int)H, (int)W, (int)cs->kernel_h, (int)cs->kernel_w, (int)cs->stride,
                 (int)cs->padding, (int)((ph - cs->kernel_h) / cs->stride + 1),
                 (int)((pw - cs->kernel_w) / cs->stride + 1)};
    return SKL_OK;
}
struct ConvPlan {
    size_t cols, ytok, gtok, dcols, inner, total;
};
ConvPlan conv_plan(const skl_shape* s, const ConvGeom& g, bool bwd) {
    const size_t e = s->dtype == SKL_BF16 ? 2 : 4;
    const int64_t T = (int64_t)g.B * g.oh * g.ow;
    ConvPlan p = {};
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += align_up(b ? b : 1); return o; };
    p.cols = take((size_t)T * s->d_in * e);    // im2col patches [T, d_in] (recomputed when not kept)
    p.ytok = take(bwd ? 0 : (size_t)T * s->d_out * e);
    p.gtok = take(bwd ? (size_t)T * s->d_out * e : 0);
    p.dcols = take(bwd ? (size_t)T * s->d_in * e : 0);
    size_t f = 0, b = 0;
    skl_workspace_size(s, T, &f, &b);
    p.inner = take(bwd ? b : f);
    p.total = off;
    return p;
}
}  // namespace
}  // namespace skl

skl_status skl_conv_workspace_size(const skl_shape* s, const skl_conv_shape* cs, int64_t B, int64_t H, int64_t W,
                                   size_t* fwd_bytes, size_t* bwd_bytes) {
    ConvGeom g;
    SKL_TRY(conv_geom(s, cs, B, H, W, g));
    SklDims d;
    SKL_TRY(get_dims(s, d));
    if (fwd_bytes) *fwd_bytes = conv_plan(s, g, false).total;
    if (bwd_bytes) *bwd_bytes = conv_plan(s, g, true).total;
    return SKL_OK;
}

skl_status sketched_conv2d_forward(const skl_shape* s, const skl_conv_shape* cs, int64_t B, int64_t H, int64_t W,
                                   unsigned fuse, const void* x, const void* S1s, const void* S2s, const void* U1s,
                                   const void* U2s, const void* bias, void* y, void* cols_out, void* saved_proj,
                                   void* workspace, size_t ws_bytes, void* stream) {
    ConvGeom g;
    SKL_TRY(conv_geom(s, cs, B, H, W, g));
    if (!x || !y) return fail(SKL_ERR_PARAM, "null tensor argument");
    const ConvPlan p = conv_plan(s, g, false);
    if (!workspace || ws_bytes < p.total)
        return fail(SKL_ERR_WORKSPACE, "conv forward workspace too small: need %zu bytes, got %zu", p.total, ws_bytes);
    const int64_t T = (int64_t)g.B * g.oh * g.ow;
    if (T == 0) return SKL_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int elem = elem_of(s->dtype);
    void* cols = cols_out ? cols_out : at<void>(workspace, p.cols);
    void* ytok = at<void>(workspace, p.ytok);
    SKL_CUDA(launch_im2col(x, elem, g, cols, st));
    SKL_TRY(sketched_linear_forward_ex(s, T, fuse, cols, S1s, S2s, U1s, U2s, bias, ytok, saved_proj,
                                       at<void>(workspace, p.inner), p.total - p.inner, stream));
    SKL_CUDA(launch_tokens_planes(ytok, elem, g.B, (int64_t)g.oh * g.ow, s->d_out, y, 1, st));
    return SKL_OK;
}

skl_status sketched_conv2d_backward(const skl_shape* s, const skl_conv_shape* cs, int64_t B, int64_t H, int64_t W,
                                    const void* grad_y, const void* x, const void* cols_in, const void* saved_proj,
                                    const void* S1s, const void* S2s, const void* U1s, const void* U2s, void* grad_x,
                                    float* grad_U1s, float* grad_U2s, float* grad_bias, void* workspace,
                                    size_t ws_bytes, void* stream) {
    ConvGeom g;
    SKL_TRY(conv_geom(s, cs, B, H, W, g));
    if (!grad_y || (!x && !cols_in)) return fail(SKL_ERR_PARAM, "null tensor argument");
    const ConvPlan p = conv_plan(s, g, true);
    if (!workspace || ws_bytes < p.total)
        return fail(SKL_ERR_WORKSPACE, "conv backward workspace too small: need %zu bytes, got %zu", p.total, ws_bytes);
    const int64_t T = (int64_t)g.B * g.oh * g.ow;
    cudaStream_t st = (cudaStream_t)stream;
    const int elem = elem_of(s->dtype);
    const void* cols = cols_in;
    if (!cols) {
        SKL_CUDA(launch_im2col(x, elem, g, at<void>(workspace, p.cols), st));
        cols = at<void>(workspace, p.cols);
    }
    void* gtok = at<void>(workspace, p.gtok);
    void* dcols = grad_x ? at<void>(workspace, p.dcols) : nullptr;
    if (T > 0) SKL_CUDA(launch_tokens_planes(grad_y, elem, g.B, (int64_t)g.oh * g.ow, s->d_out, gtok, 0, st));
    SKL_TRY(sketched_linear_backward(s, T, gtok, cols, saved_proj, S1s, S2s, U1s, U2s, dcols, grad_U1s, grad_U2s,
                                     grad_bias, at<void>(workspace, p.inner), p.total - p.inner, stream));
    if (grad_x) SKL_CUDA(launch_col2im(dcols, elem, g, grad_x, st));
    return SKL_OK;
}

// ---------------------------------------------------------------- DenseLinear
// DenseLinear::forward / backward (nn_layers.cpp:32-49) in row convention:
//   y = x·Wᵀ + b       one tcgen05 GEMM (A = x, B = W, both K-major), bias /
//                      ReLU in the epilogue;
//   dX = G·W           one GEMM (B = Wᵀ, a small transposed copy);
//   dW = Gᵀ·x, db = Σ_t G   the du kernel's token reduction: it computes
//                      dWᵀ = xᵀ·G from a transposed copy of x (K-major A, like
//                      Savedᵀ) and G (MN-major B), with db from the staged G
//                      tiles; dWᵀ is transposed into W's layout.
namespace skl {
namespace {
skl_status dense_dims(const skl_dense_shape* s, SklDims& d) {
    if (!s) return fail(SKL_ERR_PARAM, "null shape");
    if (s->d_in < 1 || s->d_out < 1) return fail(SKL_ERR_SHAPE, "DenseLinear: d_in and d_out must be >= 1");
    if (s->dtype != SKL_BF16 && s->dtype != SKL_F32_TF32) return fail(SKL_ERR_PARAM, "unknown dtype %d", s->dtype);
    // du's problem 0 ("dU1" slot) with M = d_in rows of xᵀ and N = d_out columns of G
    d.d_in = s->d_in;
    d.d_out = s->d_out;
    d.L = 1;
    d.k = s->d_in;
    d.Lk = s->d_in;
    d.R = 2 * d.Lk;
    d.R_pad = (d.R + 63) / 64 * 64;
    return SKL_OK;
}
struct DensePlan {
    size_t wr, bias32, xT, wT, dwT, part, cpart, tickets, total;
};
DensePlan dense_plan(const SklDims& d, skl_dtype t, int64_t T, bool bwd, int sms) {
    const size_t e = ebytes(t);
    DensePlan q = {};
    size_t off = 0;
    auto take = [&](bool need, size_t bytes) {
        size_t o = off;
        if (need) off += align_up(bytes ? bytes : 1);
        return o;
    };
    q.wr = take(!bwd && t != SKL_BF16, (size_t)d.d_out * d.d_in * 4);  // TF32-rounded W (forward B operand)
    q.bias32 = take(!bwd, (size_t)d.d_out * 4);
    q.xT = take(bwd, (size_t)d.d_in * t8(T) * e);                      // xᵀ [d_in][round8(T)]
    q.wT = take(bwd, (size_t)d.d_in * d.d_out * e);                    // Wᵀ [d_in][d_out]
    q.dwT = take(bwd, (size_t)d.d_in * d.d_out * 4);                   // dWᵀ [d_in][d_out] fp32
    if (bwd) {
        size_t part, cpart, tickets;
        du_ws_sizes(d, t, T, sms, part, cpart, tickets);
        q.part = take(true, part);
        q.cpart = take(true, cpart);
        q.tickets = take(true, tickets);
    }
    q.total = off;
    return q;
}
struct DensePad {
    size_t inner, x, yg, dx, w, bias, dw, db, total;
};
DensePad dense_pad_plan(const SklDims& d, const SklDims& dp, skl_dtype t, int64_t T, bool bwd, int sms) {
    const size_t e = ebytes(t);
    DensePad q = {};
    size_t off = align_up(dense_plan(dp, t, T, bwd, sms).total);
    q.inner = off;
    auto take = [&](bool need, size_t bytes) {
        size_t o = off;
        if (need) off += align_up(bytes ? bytes : 1);
        return o;
    };
    const bool pin = dp.d_in != d.d_in, pout = dp.d_out != d.d_out;
    q.x = take(pin, (size_t)T * dp.d_in * e);
    q.yg = take(pout, (size_t)T * dp.d_out * e);
    q.dx = take(bwd && pin, (size_t)T * dp.d_in * e);
    q.w = take(true, (size_t)dp.d_out * dp.d_in * e);
    q.bias = take(!bwd && pout, (size_t)dp.d_out * e);
    q.dw = take(bwd, (size_t)dp.d_out * dp.d_in * 4);
    q.db = take(bwd && pout, (size_t)dp.d_out * 4);
    q.total = off;
    return q;
}
}  // namespace
}  // namespace skl

skl_status skl_dense_workspace_size(const skl_dense_shape* s, int64_t T, size_t* fwd_bytes, size_t* bwd_bytes) {
    SklDims d;
    SKL_TRY(dense_dims(s, d));
    if (T < 0) return fail(SKL_ERR_SHAPE, "T must be >= 0");
    const int sms = std::max(2, dev_info().sms ? dev_info().sms : 148);
    if (needs_pad(d, s->dtype)) {
        SklDims dp = pad_dims(d, s->dtype, false);
        dp.k = dp.Lk = dp.d_in;
        if (fwd_bytes) *fwd_bytes = dense_pad_plan(d, dp, s->dtype, T, false, sms).total;
        if (bwd_bytes) *bwd_bytes = dense_pad_plan(d, dp, s->dtype, T, true, sms).total;
        return SKL_OK;
    }
    if (fwd_bytes) *fwd_bytes = dense_plan(d, s->dtype, T, false, sms).total;
    if (bwd_bytes) *bwd_bytes = dense_plan(d, s->dtype, T, true, sms).total;
    return SKL_OK;
}

skl_status skl_dense_init(const skl_dense_shape* s, uint64_t seed, void* W, void* bias, void* stream) {
    SklDims d;
    SKL_TRY(dense_dims(s, d));
    if (!W) return fail(SKL_ERR_PARAM, "null tensor argument");
    DevInfo di;
    SKL_TRY(check_device(di));
    cudaStream_t st = (cudaStream_t)stream;
    const double std_dev = std::sqrt(2.0 / (double)(d.d_in + d.d_out));  // nn_layers.cpp:55
    SKL_CUDA(launch_gaussian_scaled(d.d_out, d.d_in, seed, std_dev, elem_of(s->dtype), W, st));
    if (bias) SKL_CUDA(cudaMemsetAsync(bias, 0, (size_t)d.d_out * ebytes(s->dtype), st));
    return SKL_OK;
}

skl_status dense_linear_forward(const skl_dense_shape* s, int64_t T, unsigned fuse, const void* x, const void* W,
                                const void* bias, void* y, void* workspace, size_t ws_bytes, void* stream) {
    if (fuse & ~(unsigned)SKL_FUSE_RELU_OUT) return fail(SKL_ERR_PARAM, "dense forward: unsupported fuse flags %u", fuse);
    SklDims d;
    SKL_TRY(dense_dims(s, d));
    if (T < 0) return fail(SKL_ERR_SHAPE, "DenseLinear::forward: T must be >= 0");
    if (T == 0) return SKL_OK;
    if (!x || !W || !y) return fail(SKL_ERR_PARAM, "null tensor argument");
    DevInfo di;
    SKL_TRY(check_device(di));
    cudaStream_t st = (cudaStream_t)stream;
    const int eb = ebytes(s->dtype), kind = s->dtype == SKL_BF16 ? 0 : 1;
    if (needs_pad(d, s->dtype)) {
        SklDims dp = pad_dims(d, s->dtype, false);
        dp.k = dp.Lk = dp.d_in;
        const DensePad q = dense_pad_plan(d, dp, s->dtype, T, false, di.sms);
        if (!workspace || ws_bytes < q.total)
            return fail(SKL_ERR_WORKSPACE, "dense forward workspace too small: need %zu bytes, got %zu", q.total,
                        ws_bytes);
        const void *xp, *wp, *bp;
        SKL_TRY(repad_in(x, eb, 1, T, d.d_in, workspace, q.x, T, dp.d_in, st, &xp));
        SKL_TRY(repad_in(W, eb, 1, d.d_out, d.d_in, workspace, q.w, dp.d_out, dp.d_in, st, &wp));
        SKL_TRY(repad_in(bias, eb, 1, 1, d.d_out, workspace, q.bias, 1, dp.d_out, st, &bp));
        void* yp = dp.d_out != d.d_out ? at<void>(workspace, q.yg) : y;
        skl_dense_shape sp = *s;
        sp.d_in = dp.d_in;
        sp.d_out = dp.d_out;
        SKL_TRY(dense_linear_forward(&sp, T, fuse, xp, wp, bp, yp, workspace, q.inner, stream));
        if (yp != y) SKL_CUDA(launch_repad(yp, eb, 1, T, dp.d_out, y, T, d.d_out, st));
        return SKL_OK;
    }
    const DensePlan q = dense_plan(d, s->dtype, T, false, di.sms);
    if (!workspace || ws_bytes < q.total)
        return fail(SKL_ERR_WORKSPACE, "dense forward workspace too small: need %zu bytes, got %zu", q.total, ws_bytes);
    float* bias32 = at<float>(workspace, q.bias32);
    SKL_CUDA(launch_to_f32(bias, elem_of(s->dtype), d.d_out, bias32, 0, st));
    const void* wop = W;
    if (kind == 1) {  // W as RN-rounded TF32 words (the activation is truncated by the tensor core)
        SKL_CUDA(launch_to_f32(W, ELEM_F32, d.d_out * d.d_in, at<float>(workspace, q.wr), 1, st));
        wop = at<void>(workspace, q.wr);
    }
    GemmArgs g = {};
    g.alpha = 1.f;
    g.bias = bias32;
    g.relu = (fuse & SKL_FUSE_RELU_OUT) ? 1 : 0;
    g.out = y;
    g.ldo = d.d_out;
    g.out_f32 = eb == 4;
    View vx{x, T, d.d_in, d.d_in}, vw{wop, d.d_out, d.d_in, d.d_in};
    return gemm_any(kind, "dense_fwd", vx, vw, (int)T, (int)d.d_out, (int)d.d_in, g, di.sms, st);
}

skl_status dense_linear_backward(const skl_dense_shape* s, int64_t T, unsigned fuse, const void* grad_y,
                                 const void* x, const void* W, void* grad_x, float* grad_W, float* grad_b,
                                 void* workspace, size_t ws_bytes, void* stream) {
    if (fuse & ~(unsigned)SKL_FUSE_RELU_IN) return fail(SKL_ERR_PARAM, "dense backward: unsupported fuse flags %u", fuse);
    SklDims d;
    SKL_TRY(dense_dims(s, d));
    if (T < 0) return fail(SKL_ERR_SHAPE, "DenseLinear::backward: T must be >= 0");
    if (!grad_W) return fail(SKL_ERR_PARAM, "null gradient argument");
    if (T > 0 && (!grad_y || !x || !W)) return fail(SKL_ERR_PARAM, "null tensor argument");
    DevInfo di;
    SKL_TRY(check_device(di));
    cudaStream_t st = (cudaStream_t)stream;
    const int eb = ebytes(s->dtype), kind = s->dtype == SKL_BF16 ? 0 : 1;
    if (T == 0) {
        SKL_CUDA(cudaMemsetAsync(grad_W, 0, (size_t)d.d_out * d.d_in * 4, st));
        if (grad_b) SKL_CUDA(cudaMemsetAsync(grad_b, 0, (size_t)d.d_out * 4, st));
        return SKL_OK;
    }
    if (needs_pad(d, s->dtype)) {
        SklDims dp = pad_dims(d, s->dtype, false);
        dp.k = dp.Lk = dp.d_in;
        const DensePad q = dense_pad_plan(d, dp, s->dtype, T, true, di.sms);
        if (!workspace || ws_bytes < q.total)
            return fail(SKL_ERR_WORKSPACE, "dense backward workspace too small: need %zu bytes, got %zu", q.total,
                        ws_bytes);
        const void *xp, *gp, *wp;
        SKL_TRY(repad_in(x, eb, 1, T, d.d_in, workspace, q.x, T, dp.d_in, st, &xp));
        SKL_TRY(repad_in(grad_y, eb, 1, T, d.d_out, workspace, q.yg, T, dp.d_out, st, &gp));
        SKL_TRY(repad_in(W, eb, 1, d.d_out, d.d_in, workspace, q.w, dp.d_out, dp.d_in, st, &wp));
        void* gxp = (grad_x && dp.d_in != d.d_in) ? at<void>(workspace, q.dx) : grad_x;
        float* dwp = at<float>(workspace, q.dw);
        float* dbp = (grad_b && dp.d_out != d.d_out) ? at<float>(workspace, q.db) : grad_b;
        skl_dense_shape sp = *s;
        sp.d_in = dp.d_in;
        sp.d_out = dp.d_out;
        SKL_TRY(dense_linear_backward(&sp, T, fuse, gp, xp, wp, gxp, dwp, dbp, workspace, q.inner, stream));
        SKL_CUDA(launch_repad(dwp, 4, 1, dp.d_out, dp.d_in, grad_W, d.d_out, d.d_in, st));
        if (dbp != grad_b) SKL_CUDA(launch_repad(dbp, 4, 1, 1, dp.d_out, grad_b, 1, d.d_out, st));
        if (gxp != grad_x) SKL_CUDA(launch_repad(gxp, eb, 1, T, dp.d_in, grad_x, T, d.d_in, st));
        return SKL_OK;
    }
    const DensePlan q = dense_plan(d, s->dtype, T, true, di.sms);
    if (!workspace || ws_bytes < q.total)
        return fail(SKL_ERR_WORKSPACE, "dense backward workspace too small: need %zu bytes, got %zu", q.total, ws_bytes);
    const int elem = elem_of(s->dtype);
    if (grad_x) {  // dX = G·W: B = Wᵀ [d_in][d_out] (K-major over d_out)
        void* wT = at<void>(workspace, q.wT);
        SKL_CUDA(launch_transpose(W, elem, d.d_out, d.d_in, wT, st));
        if (kind == 1) SKL_CUDA(launch_to_f32(wT, ELEM_F32, d.d_in * d.d_out, static_cast<float*>(wT), 1, st));
        GemmArgs g = {};
        g.alpha = 1.f;
        g.mask = (fuse & SKL_FUSE_RELU_IN) ? x : nullptr;  // Relu::backward of the preceding ReLU (x = its output)
        g.ld_mask = d.d_in;
        g.out = grad_x;
        g.ldo = d.d_in;
        g.out_f32 = eb == 4;
        View vg{grad_y, T, d.d_out, d.d_out}, vwt{wT, d.d_in, d.d_out, d.d_out};
        SKL_TRY(gemm_any(kind, "dense_dX", vg, vwt, (int)T, (int)d.d_in, (int)d.d_out, g, di.sms, st));
    }
    // dWᵀ = xᵀ·G and db = Σ_t G: du problem 0 with A = xᵀ [d_in][round8(T)]
    void* xT = at<void>(workspace, q.xT);
    SKL_CUDA(launch_transpose(x, elem, T, d.d_in, xT, st, t8(T)));
    Plan p = {};
    p.du_part = q.part;
    p.du_cpart = q.cpart;
    p.du_tickets = q.tickets;
    float* dwT = at<float>(workspace, q.dwT);
    SKL_TRY(run_du(d, T, kind, 1, xT, grad_y, nullptr, x, dwT, nullptr, grad_b, workspace, p, di.sms, st, 1.f));
    SKL_CUDA(launch_transpose(dwT, ELEM_F32, d.d_in, d.d_out, grad_W, st));
    return SKL_OK;
}

skl_status skl_set_reserved_sms(int n) {
    if (n < 0 || n > 64) return fail(SKL_ERR_PARAM, "reserved SMs must be in [0, 64], got %d", n);
    g_reserved_sms = n;
    return SKL_OK;
}

// ---------------------------------------------------------------- tracing
uint64_t skl_launch_count(void) { return skl::prof_launches(); }

skl_status skl_profile_enable(int on) {
    skl::prof_set_enabled(on != 0);
    return SKL_OK;
}

int skl_profile_collect(skl_profile_entry* out, int max_entries) { return skl::prof_collect(out, max_entries); }

#ifdef SKL_TRACE
// Trace builds only (-DSKL_TRACE=1, csrc/trace.cuh; not in include/skl.h): copy out / clear
// the per-role event table [slot][role][event](clock64, code).
static constexpr int kTraceWords = skl::dev::kTraceSlots * skl::dev::kTraceRoles * 2 * skl::dev::kTraceEvents;
int skl_trace_dump(uint64_t* out, int max_words) {
    if (max_words < kTraceWords) return -kTraceWords;
    cudaDeviceSynchronize();
    return cudaMemcpyFromSymbol(out, skl::dev::g_trace, kTraceWords * 8) == cudaSuccess ? kTraceWords : 0;
}
int skl_trace_reset(void) {
    static unsigned long long zero[kTraceWords];
    return cudaMemcpyToSymbol(skl::dev::g_trace, zero, kTraceWords * 8) == cudaSuccess ? 0 : -1;
}
#endif

// ---------------------------------------------------------------- NCCL
typedef int (*nccl_allreduce_fn)(const void*, void*, size_t, int, int, void*, cudaStream_t);

skl_status skl_allreduce_grads(void* nccl_comm, float* grad_bucket, size_t count, void* stream) {
    static nccl_allreduce_fn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        // Use the NCCL the host process already loaded (torch's or the app's);
        // fall back to the system library.
        void* p = dlsym(RTLD_DEFAULT, "ncclAllReduce");
        if (!p) {
            void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (h) p = dlsym(h, "ncclAllReduce");
        }
        fn = reinterpret_cast<nccl_allreduce_fn>(p);
    });
    if (!fn) return fail(SKL_ERR_UNSUPPORTED, "NCCL (libnccl.so.2) not available");
    if (!nccl_comm) return fail(SKL_ERR_PARAM, "null NCCL communicator");
    // ncclFloat32 = 7, ncclSum = 0 (nccl.h)
    const int r = fn(grad_bucket, grad_bucket, count, 7, 0, nccl_comm, (cudaStream_t)stream);
    if (r != 0) return fail(SKL_ERR_NCCL, "ncclAllReduce failed (%d)", r);
    return SKL_OK;
}

}  // extern "C"

