// prof.cpp -- launch counter and CUDA-event tracing registry (see prof.h).
#include "prof.h"

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/skl.h"

namespace skl {
namespace {

std::atomic<uint64_t> g_launches{0};
std::atomic<int> g_enabled{-1};  // -1: read SKL_PROFILE on first use

struct Rec {
    const char* name;
    cudaEvent_t b, e;
};

std::mutex g_mu;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

}  // namespace

uint64_t prof_launches() { return g_launches.load(std::memory_order_relaxed); }

void prof_set_enabled(bool on) { g_enabled.store(on ? 1 : 0); }

bool prof_enabled() {
    int v = g_enabled.load(std::memory_order_relaxed);
    if (v < 0) {
        const char* e = std::getenv("SKL_PROFILE");
        v = (e && std::atoi(e) != 0) ? 1 : 0;
        g_enabled.store(v);
    }
    return v == 1;
}

void prof_count() { g_launches.fetch_add(1, std::memory_order_relaxed); }

cudaEvent_t prof_event() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_pool.empty()) {
        cudaEvent_t ev = g_pool.back();
        g_pool.pop_back();
        return ev;
    }
    cudaEvent_t ev = nullptr;
    if (cudaEventCreate(&ev) != cudaSuccess) return nullptr;
    return ev;
}

void prof_record(const char* name, cudaEvent_t b, cudaEvent_t e) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_recs.push_back({name, b, e});
}

int prof_collect(skl_profile_entry* out, int max_entries) {
    std::vector<Rec> recs;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        recs.swap(g_recs);
    }
    std::map<std::string, std::pair<uint64_t, double>> agg;
    std::vector<std::string> order;
    for (const Rec& r : recs) {
        float ms = 0.f;
        cudaEventSynchronize(r.e);
        cudaEventElapsedTime(&ms, r.b, r.e);
        auto it = agg.find(r.name);
        if (it == agg.end()) {
            order.push_back(r.name);
            agg[r.name] = {1, (double)ms};
        } else {
            it->second.first += 1;
            it->second.second += ms;
        }
    }
    {
        std::lock_guard<std::mutex> lk(g_mu);
        for (const Rec& r : recs) {
            g_pool.push_back(r.b);
            g_pool.push_back(r.e);
        }
    }
    int n = 0;
    for (const std::string& name : order) {
        if (n >= max_entries) break;
        std::memset(&out[n], 0, sizeof(out[n]));
        std::strncpy(out[n].name, name.c_str(), sizeof(out[n].name) - 1);
        out[n].launches = agg[name].first;
        out[n].total_ms = agg[name].second;
        ++n;
    }
    return n;
}

}  // namespace skl
