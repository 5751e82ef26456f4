// trace.cuh -- per-role event timelines of the persistent kernels (build with
// -DSKL_TRACE=1; otherwise every call compiles to nothing).
//
// Four CTAs per kernel are traced: the first CTA pair and the last one of the grid
// (slots 0-3: b2b, 4-7: du).  Each
// traced thread (producer, MMA issuer, one lane per epilogue warpgroup) owns a
// role row of g_trace and appends (clock64, code) pairs; skl_trace_dump copies
// the table out.  Used to find where a kernel's roles wait.
#pragma once

#include <cstdint>

namespace skl {
namespace dev {

constexpr int kTraceSlots = 8, kTraceRoles = 4, kTraceEvents = 1024;
#ifdef SKL_TRACE
__device__ unsigned long long g_trace[kTraceSlots][kTraceRoles][2 * kTraceEvents];
__device__ __forceinline__ int trace_slot() {
    const int b = (int)blockIdx.x, g = (int)gridDim.x;
    return b < 2 ? b : (b >= g - 2 ? 2 + (b - (g - 2)) : -1);
}
#endif

struct Tr {
#ifdef SKL_TRACE
    unsigned long long* row;
    int n;
    __device__ explicit Tr(int role, int base = 0) : row(nullptr), n(0) {  // base: 0 b2b, 4 du
        const int s = trace_slot() < 0 ? -1 : base + trace_slot();
        if (s >= 0 && role >= 0) row = g_trace[s][role];
    }
    __device__ __forceinline__ void operator()(int code) {
        if (row != nullptr && n < kTraceEvents) {
            row[2 * n] = clock64();
            row[2 * n + 1] = (unsigned long long)code;
            ++n;
        }
    }
#else
    __device__ explicit Tr(int, int = 0) {}
    __device__ __forceinline__ void operator()(int) {}
#endif
};

}  // namespace dev
}  // namespace skl
