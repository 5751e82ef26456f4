/*
 * skl_dp.hpp -- token-sharded data parallelism for the SKLinear path in C++
 * (no PyTorch): an NCCL communicator, a communication stream and the
 * overlapped gradient all-reduce of SURVEY.md §8(e).
 *
 * The reference has no distributed backend; this is the
 * multi-GPU row of the north star: tokens are sharded across ranks, every rank
 * regenerates the same sketches / U from the seed (bit-identical), the forward
 * needs no communication and the backward sums dU1s / dU2s / db across ranks
 * with ncclAllReduce, overlapped with the dX kernel:
 *
 *     compute stream:  DU1_DB (dU1s, db) ──► DX_DU2 (dX, dU2s) ──────────►
 *     comm stream:                 └► all-reduce(dU1s|db)   └► all-reduce(dU2s)
 *
 * (sketched_linear_backward_phase, skl.h).  In a chain every layer's whole
 * bucket is reduced as soon as its backward is done, overlapping the layers
 * below (skl_chain.hpp).  libskl leaves `reserved_sms` SMs free so the NCCL
 * kernel is co-resident with the persistent compute kernels.
 *
 * Rendezvous: rank 0 writes ncclGetUniqueId() to a file (write + rename);
 * the other ranks poll for it.  Errors: ncclCommGetAsyncError is polled while
 * the host waits (synchronize()); an asynchronous NCCL failure aborts the
 * communicator and throws skl::nccl_error instead of hanging.
 *
 * Header-only; link with -lnccl -lskl -lcudart.
 */
#ifndef SKL_DP_HPP_
#define SKL_DP_HPP_

#include <nccl.h>

#include <chrono>
#include <cstdio>
#include <fstream>
#include <string>
#include <thread>

#include "skl.hpp"

namespace skl {

struct nccl_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check_nccl(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw nccl_error(std::string(what) + ": " + ncclGetErrorString(r));
}

// Contiguous token range [lo, hi) of `rank` (balanced, deterministic) -- the shard of T.
inline std::pair<int64_t, int64_t> shard_range(int64_t T, int rank, int world) {
    if (world < 1 || rank < 0 || rank >= world) throw parameter_error("shard_range: bad rank / world");
    const int64_t base = T / world, rem = T % world;
    const int64_t lo = rank * base + (rank < rem ? rank : rem);
    return {lo, lo + base + (rank < rem ? 1 : 0)};
}

class Dp {
  public:
    // One rank of a `world`-rank job on CUDA device `device`.  reserved_sms SMs
    // are left to the NCCL kernel (skl_set_reserved_sms) and NCCL is capped at
    // as many CTAs (ncclConfig_t::maxCTAs) when world > 1.
    static Dp from_id_file(const std::string& path, int rank, int world, int device, int reserved_sms = 8,
                           double timeout_s = 120.0) {
        if (world < 1 || rank < 0 || rank >= world) throw parameter_error("Dp: bad rank / world");
        check_cuda(cudaSetDevice(device), "cudaSetDevice");
        ncclUniqueId id;
        if (rank == 0) {
            check_nccl(ncclGetUniqueId(&id), "ncclGetUniqueId");
            const std::string tmp = path + ".tmp" + std::to_string(rank);
            {
                std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
                f.write(id.internal, sizeof(id.internal));
                if (!f) throw nccl_error("Dp: cannot write " + tmp);
            }
            if (std::rename(tmp.c_str(), path.c_str()) != 0) throw nccl_error("Dp: cannot publish " + path);
        } else {
            const auto t0 = std::chrono::steady_clock::now();
            for (;;) {
                std::ifstream f(path, std::ios::binary);
                if (f && f.read(id.internal, sizeof(id.internal))) break;
                if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s)
                    throw nccl_error("Dp: timed out waiting for " + path);
                std::this_thread::sleep_for(std::chrono::milliseconds(20));
            }
        }
        Dp dp;
        dp.rank_ = rank;
        dp.world_ = world;
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        if (world > 1 && reserved_sms > 0) cfg.maxCTAs = reserved_sms;
        check_nccl(ncclCommInitRankConfig(&dp.comm_, world, id, rank, &cfg), "ncclCommInitRankConfig");
        check(skl_set_reserved_sms(world > 1 ? reserved_sms : 0));
        int lo = 0, hi = 0;
        check_cuda(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
        check_cuda(cudaStreamCreateWithPriority(&dp.comm_st_, cudaStreamNonBlocking, hi), "comm stream");
        check_cuda(cudaEventCreateWithFlags(&dp.produced_, cudaEventDisableTiming), "event");
        check_cuda(cudaEventCreateWithFlags(&dp.done_, cudaEventDisableTiming), "event");
        return dp;
    }

    Dp() = default;
    Dp(const Dp&) = delete;
    Dp& operator=(const Dp&) = delete;
    Dp(Dp&& o) noexcept { *this = std::move(o); }
    Dp& operator=(Dp&& o) noexcept {
        std::swap(comm_, o.comm_);
        std::swap(comm_st_, o.comm_st_);
        std::swap(produced_, o.produced_);
        std::swap(done_, o.done_);
        std::swap(rank_, o.rank_);
        std::swap(world_, o.world_);
        return *this;
    }
    ~Dp() {
        if (comm_) {
            ncclResult_t st = ncclSuccess;
            ncclCommGetAsyncError(comm_, &st);
            if (st == ncclSuccess) ncclCommDestroy(comm_);
            else ncclCommAbort(comm_);
        }
        if (produced_) cudaEventDestroy(produced_);
        if (done_) cudaEventDestroy(done_);
        if (comm_st_) cudaStreamDestroy(comm_st_);
    }

    int rank() const { return rank_; }
    int world() const { return world_; }
    ncclComm_t comm() const { return comm_; }
    cudaStream_t comm_stream() const { return comm_st_; }

    // Sum `count` floats of `buf` in place across the ranks, on the comm stream,
    // once `producer` has reached this point (its kernels wrote `buf`).
    void allreduce_async(float* buf, size_t count, cudaStream_t producer) {
        check_cuda(cudaEventRecord(produced_, producer), "record");
        check_cuda(cudaStreamWaitEvent(comm_st_, produced_, 0), "wait");
        check(skl_allreduce_grads(comm_, buf, count, comm_st_));
        ++issued_;
    }

    // `consumer` waits for every collective issued so far (before it reads the
    // reduced gradients, e.g. in the optimizer step).
    void join(cudaStream_t consumer) {
        check_cuda(cudaEventRecord(done_, comm_st_), "record");
        check_cuda(cudaStreamWaitEvent(consumer, done_, 0), "wait");
    }

    // Host wait for every issued collective, polling ncclCommGetAsyncError: an
    // asynchronous NCCL error (or the timeout) aborts the communicator and throws.
    void synchronize(double timeout_s = 300.0) {
        check_cuda(cudaEventRecord(done_, comm_st_), "record");
        const auto t0 = std::chrono::steady_clock::now();
        for (;;) {
            const cudaError_t q = cudaEventQuery(done_);
            if (q == cudaSuccess) return;
            if (q != cudaErrorNotReady) check_cuda(q, "comm stream");
            ncclResult_t st = ncclSuccess;
            check_nccl(ncclCommGetAsyncError(comm_, &st), "ncclCommGetAsyncError");
            const bool late =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s;
            if ((st != ncclSuccess && st != ncclInProgress) || late) {
                ncclCommAbort(comm_);
                comm_ = nullptr;
                throw nccl_error(late ? "Dp: collective timed out (communicator aborted)"
                                      : std::string("Dp: asynchronous NCCL error: ") + ncclGetErrorString(st));
            }
            std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
    }

    uint64_t collectives_issued() const { return issued_; }

  private:
    ncclComm_t comm_ = nullptr;
    cudaStream_t comm_st_ = nullptr;
    cudaEvent_t produced_ = nullptr, done_ = nullptr;
    int rank_ = 0, world_ = 1;
    uint64_t issued_ = 0;
};

// Gradient bucket of one SKLinear layer: dU1s [L,k,d_out] | db [d_out] | dU2s
// [L,d_in,k], fp32, so each all-reduce is one contiguous slice.
struct SkBucket {
    size_t n_u1, n_b, n_u2;
    static SkBucket of(const SkLinear& L) {
        const size_t lk = (size_t)(L.num_terms() * L.low_rank());
        return {lk * (size_t)L.d_out(), (size_t)L.d_out(), lk * (size_t)L.d_in()};
    }
    size_t count() const { return n_u1 + n_b + n_u2; }
    float* dU1s(float* b) const { return b; }
    float* db(float* b) const { return b + n_u1; }
    float* dU2s(float* b) const { return b + n_u1 + n_b; }
};

// Token-sharded backward of one SKLinear layer (this rank's T tokens) with the
// all-reduce of dU1s | db overlapped with the dX kernel, then dU2s's
// (SURVEY.md §8e).  The collectives are left in flight: dp.join(stream) or
// dp.synchronize() before reading `bucket`.
inline void backward_overlapped(const SkLinear& L, Dp& dp, const void* x, const void* grad_out, int64_t T,
                                const void* saved, void* grad_x, float* bucket, cudaStream_t st, unsigned fuse = 0,
                                const uint32_t* relu_bits = nullptr) {
    const SkBucket b = SkBucket::of(L);
    L.backward_into(x, grad_out, T, saved, nullptr, b.dU1s(bucket), nullptr, b.db(bucket), st, SKL_BWD_DU1_DB);
    dp.allreduce_async(bucket, b.n_u1 + b.n_b, st);  // overlaps the dX kernel below
    L.backward_into(x, grad_out, T, saved, grad_x, nullptr, b.dU2s(bucket), nullptr, st, SKL_BWD_DX_DU2, fuse,
                    relu_bits);
    dp.allreduce_async(b.dU2s(bucket), b.n_u2, st);
}

}  // namespace skl

#endif  // SKL_DP_HPP_
