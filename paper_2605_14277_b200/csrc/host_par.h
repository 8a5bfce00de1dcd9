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
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace scfr {

// Per-thread override of the worker count: scfr_create runs its two upload
// pipelines (player 1 + U, player 2 + Uᵀ) side by side, each on half.
inline thread_local int tl_host_threads = 0;

inline int host_threads() {
    if (tl_host_threads > 0) return tl_host_threads;
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

// Process-wide worker pool for parallel_chunks: threads are started once and
// reused (spawning ~80 threads per scfr_create cost milliseconds and, with
// two upload pipelines, stalled page faults behind the stack mmaps).
class HostPool {
  public:
    static HostPool& get() {
        static HostPool* p = new HostPool();  // never destroyed: workers park at exit
        return *p;
    }
    void submit(std::function<void()> f) {
        {
            std::lock_guard<std::mutex> g(m_);
            q_.push_back(std::move(f));
            // one worker per queued task: never leave a task waiting behind
            // another caller's chunks (idle_ counts workers not yet woken)
            if ((int)q_.size() > idle_ && (int)workers_.size() < kMax) workers_.emplace_back([this] { loop(); });
        }
        cv_.notify_one();
    }

  private:
    static constexpr int kMax = 64;
    void loop() {
        std::unique_lock<std::mutex> lk(m_);
        for (;;) {
            ++idle_;
            cv_.wait(lk, [this] { return !q_.empty(); });
            --idle_;
            std::function<void()> f = std::move(q_.front());
            q_.pop_front();
            lk.unlock();
            f();
            lk.lock();
        }
    }
    std::mutex m_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
    std::vector<std::thread> workers_;
    int idle_ = 0;
};

// f(chunk, lo, hi) over [0, n) in contiguous chunks (at most host_threads(),
// each >= grain); chunk 0 runs on the caller, the rest on the pool.  f must
// not throw: workers report errors through their own state, checked by the
// caller after the join.
template <class F>
int parallel_chunks(int64_t n, int64_t grain, F&& f) {
    const int64_t want = std::max<int64_t>(1, (n + grain - 1) / std::max<int64_t>(grain, 1));
    const int chunks = (int)std::min<int64_t>(host_threads(), want);
    if (chunks <= 1) {
        f(0, (int64_t)0, n);
        return 1;
    }
    // the count is only touched under dm, so the caller cannot return (and
    // destroy dm / dcv) while a worker still holds them
    int left = chunks - 1;
    std::mutex dm;
    std::condition_variable dcv;
    HostPool& pool = HostPool::get();
    for (int c = 1; c < chunks; ++c)
        pool.submit([&f, &left, &dm, &dcv, c, n, chunks] {
            f(c, n * c / chunks, n * (c + 1) / chunks);
            std::lock_guard<std::mutex> g(dm);
            if (--left == 0) dcv.notify_all();
        });
    f(0, (int64_t)0, n / chunks);
    std::unique_lock<std::mutex> lk(dm);
    dcv.wait(lk, [&] { return left == 0; });
    return chunks;
}

// Pinned host staging, grow-only, shared by every handle of the process
// (hold `lock` while a create uses it).
struct PinnedArena {
    std::mutex lock;
    char* base = nullptr;
    size_t cap = 0;
    std::atomic<size_t> used{0};  // take() may run on both upload pipelines
    void reset() { used = 0; }
    // Buffers stay valid until the next reset(); returns nullptr if pinning fails.
    void* take(size_t n) {
        n = (n + 255) & ~size_t(255);
        const size_t at = used.fetch_add(n);
        if (at + n > cap) return nullptr;
        return base + at;
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
        cap = 0;
        used = 0;
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
// Grow-only host vector whose buffer stays page-locked (cudaHostRegister), so
// the structure uploads DMA straight from it; plain pageable memory if
// registration fails or SCFR_NO_PINNED=1.
inline void resize_pinned(std::vector<int>& v, size_t n) {
    static const bool off = [] {
        const char* e = std::getenv("SCFR_NO_PINNED");
        return e && e[0] == '1';
    }();
    if (!off && v.capacity() < n) {
        if (v.data() && v.capacity()) cudaHostUnregister(v.data());
        std::vector<int>().swap(v);
        v.reserve(n + n / 8);
        if (cudaHostRegister(v.data(), v.capacity() * sizeof(int), cudaHostRegisterDefault) != cudaSuccess)
            cudaGetLastError();  // stays pageable
    }
    v.resize(n);
}

struct HostScratch {  // per player (the two upload pipelines run concurrently)
    std::vector<int> sp[2], par[2];  // int32 seq_ptr / dp_parent
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
