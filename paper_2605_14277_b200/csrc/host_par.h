// Host-side parallel loops and a pinned staging arena for scfr_create.
//
// Creating a Goofspiel-5 handle walks ~5 M decision points and sequences per
// player (validation, level statistics, affine shape detection) and converts
// two 2.7 M-row CSR matrices to int32.  Done serially that is ~65 ms, 5x the
// cost of 50 iterations.  The loops below split the work over the host cores.
// The copies go through a pinned arena that is reused across handles, like
// the device memory pool.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <vector>

namespace scfr {

inline int host_threads() {
    static const int n = [] {
        // three quarters of the cores: a worker descheduled behind another
        // busy thread stalls the whole split.  Goofspiel-5 create on a
        // 16-vCPU B200 host: 16 threads 22-43 ms, 12 threads 20-28 ms,
        // 8 threads 24-71 ms, 4 threads 27 ms.
        int v = (int)std::thread::hardware_concurrency() * 3 / 4;
        // one process per GPU (torchrun): share the host among the local ranks
        if (const char* lw = std::getenv("LOCAL_WORLD_SIZE")) v /= std::max(1, std::atoi(lw));
        if (const char* e = std::getenv("SCFR_HOST_THREADS")) v = std::atoi(e);
        return std::max(1, std::min(v, 32));
    }();
    return n;
}

// f(chunk, lo, hi) over [0, n) in contiguous chunks (at most host_threads(),
// each >= grain).  f must not throw: workers report errors through their
// own state, checked by the caller after the join.
template <class F>
int parallel_chunks(int64_t n, int64_t grain, F&& f) {
    const int64_t want = std::max<int64_t>(1, (n + grain - 1) / std::max<int64_t>(grain, 1));
    const int chunks = (int)std::min<int64_t>(host_threads(), want);
    if (chunks <= 1) {
        f(0, (int64_t)0, n);
        return 1;
    }
    std::vector<std::thread> th;
    th.reserve(chunks - 1);
    for (int c = 1; c < chunks; ++c) th.emplace_back([&f, c, n, chunks] { f(c, n * c / chunks, n * (c + 1) / chunks); });
    f(0, (int64_t)0, n / chunks);
    for (auto& t : th) t.join();
    return chunks;
}

// Pinned host staging, grow-only, shared by every handle of the process
// (hold `lock` while a create uses it).
struct PinnedArena {
    std::mutex lock;
    char* base = nullptr;
    size_t cap = 0, used = 0;
    void reset() { used = 0; }
    // Buffers stay valid until the next reset(); returns nullptr if pinning fails.
    void* take(size_t n) {
        n = (n + 255) & ~size_t(255);
        if (used + n > cap) return nullptr;
        void* p = base + used;
        used += n;
        return p;
    }
    bool reserve(size_t n) {
        static const bool off = [] {
            const char* e = std::getenv("SCFR_NO_PINNED");
            return e && e[0] == '1';
        }();
        if (off) return false;
        if (n <= cap) return true;
        if (base) cudaFreeHost(base);
        base = nullptr;
        cap = used = 0;
        if (cudaHostAlloc(reinterpret_cast<void**>(&base), n, cudaHostAllocDefault) != cudaSuccess) {
            base = nullptr;
            return false;
        }
        cap = n;
        return true;
    }
};
// Host scratch of scfr_create, grow-only and reused (fresh multi-MB vectors
// cost more in first-touch page faults than the loops that fill them).
// Guarded by the pinned arena's lock.
struct HostScratch {
    std::vector<int> sp[2], par[2];  // per player: int32 seq_ptr / dp_parent
    std::vector<int> ccnt, cfirst;   // per sequence: child-DP group
    std::vector<int64_t> dpd;        // per DP: depth
};
inline HostScratch& host_scratch() {
    static HostScratch* s = new HostScratch();
    return *s;
}

inline PinnedArena& pinned_arena() {
    static PinnedArena* a = new PinnedArena();  // never destroyed: process lifetime
    return *a;
}

}  // namespace scfr
