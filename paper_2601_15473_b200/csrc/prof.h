// prof.h -- native launch tracing for libskl (the SURVEY §5 tracing hook).
//
// Every kernel launch in the library is wrapped in a ProfScope.  It always
// bumps a process-wide launch counter (skl_launch_count); when tracing is on
// (skl_profile_enable / SKL_PROFILE=1) it also brackets the launch with CUDA
// events recorded on the launching stream, so skl_profile_collect can report
// per-kernel device time without a profiler attached.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/skl.h"

namespace skl {

bool prof_enabled();
void prof_set_enabled(bool on);
uint64_t prof_launches();
int prof_collect(skl_profile_entry* out, int max_entries);
void prof_count();
void prof_record(const char* name, cudaEvent_t begin, cudaEvent_t end);
cudaEvent_t prof_event();

class ProfScope {
public:
    ProfScope(const char* name, cudaStream_t st) : name_(name), st_(st) {
        prof_count();
        if (prof_enabled()) {
            b_ = prof_event();
            e_ = prof_event();
            if (b_ && e_) cudaEventRecord(b_, st_);
        }
    }
    ~ProfScope() {
        if (b_ && e_) {
            cudaEventRecord(e_, st_);
            prof_record(name_, b_, e_);
        }
    }
    ProfScope(const ProfScope&) = delete;
    ProfScope& operator=(const ProfScope&) = delete;

private:
    const char* name_;
    cudaStream_t st_;
    cudaEvent_t b_ = nullptr, e_ = nullptr;
};

}  // namespace skl
