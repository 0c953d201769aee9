// Host-side plumbing shared by the C ABI translation units (dg_capi.cpp,
// dg_io.cpp): error codes -> thread-local message, stream-ordered device
// memory, the engine and lattice handles. Internal; not installed.
#pragma once

#include <cuda_runtime.h>

#include <exception>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "b200geo.h"

namespace dg {

std::string& last_error();  // thread-local (dg_capi.cpp)

struct DgError {
    int code;
    std::string msg;
};

[[noreturn]] inline void raise(int code, const std::string& msg) { throw DgError{code, msg}; }

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess)                                                             \
            ::dg::raise(e_ == cudaErrorMemoryAllocation ? DG_ENOMEM : DG_ERUNTIME,         \
                        std::string(#x) + ": " + cudaGetErrorString(e_));                  \
    } while (0)

template <class F>
int guard(F&& f) {
    try {
        f();
        return DG_OK;
    } catch (const DgError& e) {
        last_error() = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        last_error() = "host out of memory";
        return DG_ENOMEM;
    } catch (const std::exception& e) {
        last_error() = e.what();
        return DG_ERUNTIME;
    }
}

// owning device allocation for objects that outlive a call (staged captures,
// lattices): taken from the device's stream-ordered pool, which keeps freed
// memory mapped (release threshold set at engine creation), so re-staging a
// run every call costs no cudaMalloc/cudaFree device synchronisation.
struct DevMem {
    void* p = nullptr;
    size_t bytes = 0;
    explicit DevMem(size_t n) : bytes(n) {
        if (n) {
            CK(cudaMallocAsync(&p, n, cudaStreamPerThread));
            CK(cudaStreamSynchronize(cudaStreamPerThread));
        }
    }
    ~DevMem() {
        if (p) cudaFreeAsync(p, cudaStreamPerThread);
    }
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
};

// Engine-owned device workspace of the run drivers: one allocation reused by
// every call, grown to the previous calls' high-water mark, so a solve never
// waits in the host for the stream-ordered pool to grow by gigabytes
// (intermittent 3-600 ms stalls at C5 in r01). One call at a time uses it
// (try_lock); a concurrent call on the same engine takes pool memory instead.
struct Arena {
    std::mutex mu;
    char* base = nullptr;
    size_t cap = 0, want = 0;
    ~Arena() {
        if (base) cudaFree(base);
    }
};

// scratch for one call: bump allocation in the engine's arena when it holds
// it, else stream-ordered pool memory
struct Scratch {
    cudaStream_t st;
    std::vector<void*> ptrs;
    Arena* arena = nullptr;
    size_t used = 0, total = 0;
    explicit Scratch(cudaStream_t s, Arena* a = nullptr) : st(s) {
        if (a && a->mu.try_lock()) {
            arena = a;
            if (a->want > a->cap) {  // grow to the last call's need (calls are synchronous)
                if (a->base) CK(cudaFree(a->base));
                a->base = nullptr;
                a->cap = 0;
                // the pool memory those calls took goes back to the driver first
                int dev = 0;
                cudaMemPool_t pool;
                CK(cudaGetDevice(&dev));
                CK(cudaDeviceGetDefaultMemPool(&pool, dev));
                CK(cudaDeviceSynchronize());
                CK(cudaMemPoolTrimTo(pool, 0));
                void* p = nullptr;
                CK(cudaMalloc(&p, a->want));
                a->base = static_cast<char*>(p);
                a->cap = a->want;
            }
        }
    }
    template <class T>
    T* alloc(size_t n) {
        if (n == 0) n = 1;
        const size_t bytes = (n * sizeof(T) + 255) & ~size_t(255);
        total += bytes;
        if (arena && used + bytes <= arena->cap) {
            void* p = arena->base + used;
            used += bytes;
            return static_cast<T*>(p);
        }
        void* p = nullptr;
        CK(cudaMallocAsync(&p, n * sizeof(T), st));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    ~Scratch() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
        if (arena) {
            // an error may leave work queued on the arena: finish it first
            if (std::uncaught_exceptions() > 0) cudaDeviceSynchronize();
            if (total > arena->want) arena->want = total;
            arena->mu.unlock();
        }
    }
};

// the caller's stream, else the engine's persistent stream (a fresh stream per
// call would defeat the stream-ordered memory pool's reuse), else a private one
struct StreamGuard {
    cudaStream_t st = nullptr;
    bool own = false;
    explicit StreamGuard(void* user, cudaStream_t fallback = nullptr) {
        if (user) {
            st = static_cast<cudaStream_t>(user);
        } else if (fallback) {
            st = fallback;
        } else {
            CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            own = true;
        }
    }
    ~StreamGuard() {
        if (own) cudaStreamDestroy(st);
    }
};

}  // namespace dg

struct dg_engine {
    int device = 0;
    int sm_count = 148;
    dg_tuning tuning{};  // validated by dg_engine_set_tuning; read once per call
    // multi-GPU engine (dg_engine_create_multi): this engine drives devices[0],
    // `peers` the others; whole-run calls shard the run across all of them
    std::vector<dg_engine*> peers;
    int n_devices() const { return 1 + (int)peers.size(); }
    dg_engine* dev(int k) { return k == 0 ? this : peers[k - 1]; }
    cudaStream_t stream = nullptr;  // default stream of calls that pass none
    cudaStream_t upload = nullptr;  // capture uploads overlapped with the geometry phase
    // the second correlation lane and the side refinement of a run, created once
    // (stream creation costs ~0.1-0.3 ms of host time per call)
    cudaStream_t lane = nullptr, refine = nullptr;
    // the correlator's Chebyshev tables, uploaded once (a per-call upload over
    // 64 KB queued behind capture uploads on the copy engine)
    std::mutex tables_mu;
    std::unique_ptr<dg::DevMem> tables;
    dg::Arena arena;  // workspace of the whole-run drivers
    // pinned double buffer of the file writers (dg_io.cpp), kept across calls
    std::mutex stage_mu;
    void* stage_host[2] = {nullptr, nullptr};
    size_t stage_bytes = 0;
    ~dg_engine() {
        for (dg_engine* e : peers) delete e;
        for (void* p : stage_host)
            if (p) cudaFreeHost(p);
        if (stream) cudaStreamDestroy(stream);
        if (upload) cudaStreamDestroy(upload);
        if (lane) cudaStreamDestroy(lane);
        if (refine) cudaStreamDestroy(refine);
    }
};

struct dg_grid;
struct dg_staged;
namespace dg {
// copies of a grid / staged run on the other devices of a multi-GPU engine,
// made by peer copies on first use and kept with the object
template <class T>
struct Replicas {
    std::mutex mu;
    std::vector<std::pair<const dg_engine*, std::unique_ptr<T>>> v;
};
}  // namespace dg

struct dg_grid {
    dg_engine* eng = nullptr;
    std::shared_ptr<dg::Replicas<dg_grid>> replicas = std::make_shared<dg::Replicas<dg_grid>>();
    double lat_start = 0, lat_step = 0, lon_start = 0, lon_step = 0, alt = 0;
    int64_t n_lat = 0, n_lon = 0, row_offset = 0;
    std::shared_ptr<dg::DevMem> mem;  // x | y | z of the full lattice
    const double *x = nullptr, *y = nullptr, *z = nullptr;
    // the FULL lattice (shared by every slab): FP32 positions relative to its
    // centre, for partition-independent correlator planning
    std::shared_ptr<dg::DevMem> rel;
    int64_t full_size = 0;
    double cx = 0, cy = 0, cz = 0;
    int64_t size() const { return n_lat * n_lon; }
    const float4* rel32() const { return static_cast<const float4*>(rel->p); }
};

// captures of a run resident in HBM: [S][R] rows of `stride` elements, data
// kCapturePad elements in (dg_internal.cuh), FP32 for the correlator, FP64 for
// centring / refinement
struct dg_staged {
    dg_engine* eng = nullptr;
    std::shared_ptr<dg::Replicas<dg_staged>> replicas = std::make_shared<dg::Replicas<dg_staged>>();
    int64_t S = 0, R = 0, N = 0, stride = 0;
    double fs = 0, fc = 0;
    std::unique_ptr<dg::DevMem> y32, y64;
    std::vector<dg_state> states;
    cudaEvent_t ready = nullptr;  // async staging: the upload's completion
    // per capture [S*R][N+1] exclusive prefix sums of |y|^2 (FP64), made on first
    // use (the moment path's refinement floor, launch_energy_prefix)
    mutable std::mutex e_mu;
    mutable std::unique_ptr<dg::DevMem> e64;
    mutable cudaEvent_t e_ready = nullptr;
    ~dg_staged() {
        if (ready) cudaEventDestroy(ready);
        if (e_ready) cudaEventDestroy(e_ready);
    }
};

namespace dg {
inline void set_device(const dg_engine* e) { CK(cudaSetDevice(e->device)); }
}  // namespace dg
