// hoststage.h -- host side of pmsz_run_correction_host for PAGEABLE caller
// buffers (numpy arrays behind the reference's ScalarField, grid.py:35-82).
//
// The driver copies pageable memory at ~11 GB/s (1 GiB H2D: 95 ms) and
// cudaHostRegister costs ~50 ms per GiB (register + unregister), against
// 19 ms for a pinned copy.  So the input slabs are staged through a small
// pinned ring by a pool of host threads (pageable -> pinned memcpy at
// ~75 GB/s with 8+ threads) while the DMA of the previous chunk is on the
// link, and a pageable corrected field is filled on the host from fhat in the
// same pass (one load, two streaming stores) and patched with the edit record
// at the end -- no device-to-host copy of the field at all.
//
// Host-only C++ (no device code); included by pmsz.cu.
#pragma once
#include <cuda_runtime.h>
#if defined(__x86_64__) || defined(_M_X64)
#include <emmintrin.h>
#define PMSZ_HOST_SSE2 1
#else
#define PMSZ_HOST_SSE2 0
#endif
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace pmsz {

// True when ptr is page-locked host memory (cudaMallocHost / cudaHostRegister /
// a pinned torch tensor): the DMA engines read it directly.
inline bool host_pinned(const void* ptr) {
    if (!ptr) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Streaming (non-temporal) stores for the staging copies: the pinned slot
// and the corrected-field fill are written once and read by the DMA engine /
// the caller much later, so a regular store's read-for-ownership of every
// destination line (~2.7 GB of extra DRAM reads at 512^3) is pure waste.
// SSE2 only (the x86-64 baseline); the caller fences (_mm_sfence) before the
// DMA is issued.  Unaligned destinations fall back to memcpy.
// store fence after streaming stores / spin-wait hint (no-ops off x86-64)
inline void host_sfence() {
#if PMSZ_HOST_SSE2
    _mm_sfence();
#endif
}
inline void host_pause() {
#if PMSZ_HOST_SSE2
    _mm_pause();
#endif
}

inline void nt_copy(char* d1, char* d2, const char* src, size_t bytes) {
#if !PMSZ_HOST_SSE2
    memcpy(d1, src, bytes);
    if (d2) memcpy(d2, src, bytes);
    return;
#else
    if ((((uintptr_t)d1 | (uintptr_t)(d2 ? d2 : d1)) & 15) != 0) {
        memcpy(d1, src, bytes);
        if (d2) memcpy(d2, src, bytes);
        return;
    }
    size_t i = 0;
    if (d2) {
        for (; i + 64 <= bytes; i += 64) {
            const __m128i a = _mm_loadu_si128((const __m128i*)(src + i));
            const __m128i b = _mm_loadu_si128((const __m128i*)(src + i + 16));
            const __m128i c = _mm_loadu_si128((const __m128i*)(src + i + 32));
            const __m128i e = _mm_loadu_si128((const __m128i*)(src + i + 48));
            _mm_stream_si128((__m128i*)(d1 + i), a);
            _mm_stream_si128((__m128i*)(d1 + i + 16), b);
            _mm_stream_si128((__m128i*)(d1 + i + 32), c);
            _mm_stream_si128((__m128i*)(d1 + i + 48), e);
            _mm_stream_si128((__m128i*)(d2 + i), a);
            _mm_stream_si128((__m128i*)(d2 + i + 16), b);
            _mm_stream_si128((__m128i*)(d2 + i + 32), c);
            _mm_stream_si128((__m128i*)(d2 + i + 48), e);
        }
    } else {
        for (; i + 64 <= bytes; i += 64) {
            const __m128i a = _mm_loadu_si128((const __m128i*)(src + i));
            const __m128i b = _mm_loadu_si128((const __m128i*)(src + i + 16));
            const __m128i c = _mm_loadu_si128((const __m128i*)(src + i + 32));
            const __m128i e = _mm_loadu_si128((const __m128i*)(src + i + 48));
            _mm_stream_si128((__m128i*)(d1 + i), a);
            _mm_stream_si128((__m128i*)(d1 + i + 16), b);
            _mm_stream_si128((__m128i*)(d1 + i + 32), c);
            _mm_stream_si128((__m128i*)(d1 + i + 48), e);
        }
    }
    if (i < bytes) {
        memcpy(d1 + i, src + i, bytes - i);
        if (d2) memcpy(d2 + i, src + i, bytes - i);
    }
#endif
}

// f64 -> f32 with streaming stores; true when some value does not survive the
// round trip (NaN compares unequal, an overflow becomes inf != v).
inline bool nt_narrow(float* dst, const double* src, size_t n) {
    size_t i = 0;
    bool nb = false;
#if PMSZ_HOST_SSE2
    __m128d bad = _mm_setzero_pd();
    if (((uintptr_t)dst & 15) == 0) {
        for (; i + 4 <= n; i += 4) {
            const __m128d a = _mm_loadu_pd(src + i), b = _mm_loadu_pd(src + i + 2);
            const __m128 fa = _mm_cvtpd_ps(a), fb = _mm_cvtpd_ps(b);
            _mm_stream_ps(dst + i, _mm_movelh_ps(fa, fb));
            bad = _mm_or_pd(bad, _mm_cmpneq_pd(_mm_cvtps_pd(fa), a));
            bad = _mm_or_pd(bad, _mm_cmpneq_pd(_mm_cvtps_pd(fb), b));
        }
    }
    nb = _mm_movemask_pd(bad) != 0;
#endif
    for (; i < n; ++i) {
        const float v = (float)src[i];
        dst[i] = v;
        nb |= (double)v != src[i];
    }
    return nb;
}

// Persistent fork-join pool: run(fn) calls fn(t, nt) on nt threads (t = 0 on
// the caller) and returns when all are done.  One job at a time.
class HostPool {
   public:
    static HostPool& get() {
        // never destroyed (idle workers at exit); a forked child, which has no
        // copies of the workers, builds its own
        static std::atomic<HostPool*> pool{nullptr};
        static std::mutex m;
        HostPool* p = pool.load();
        if (p && p->pid_ == getpid()) return *p;
        std::lock_guard<std::mutex> lk(m);
        p = pool.load();
        if (!p || p->pid_ != getpid()) {
            p = new HostPool();
            pool.store(p);
        }
        return *p;
    }
    int threads() const { return nt_; }
    void run(const std::function<void(int, int)>& fn, int want = 0) {
        std::lock_guard<std::mutex> one(run_m_);
        const int jn = want > 0 ? std::min(want, nt_) : nt_;
        if (jn <= 1 || nt_ == 1) {
            fn(0, 1);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(m_);
            job_ = &fn;
            job_nt_ = jn;
            pending_ = nt_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        fn(0, jn);
        std::unique_lock<std::mutex> lk(m_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
    }

   private:
    HostPool() : pid_(getpid()) {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const int want = (int)std::min(16u, hw);
        nt_ = 1;
        for (int t = 1; t < want; ++t) {   // (a thread that cannot start just shrinks the pool)
            try {
                std::thread([this, t] { loop(t); }).detach();
            } catch (...) {
                break;
            }
            nt_ = t + 1;
        }
    }
    void loop(int t) {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(m_);
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
            const std::function<void(int, int)>* job = job_;
            const int jn = job_nt_;
            lk.unlock();
            if (t < jn) (*job)(t, jn);
            lk.lock();
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    pid_t pid_;
    int nt_ = 1;
    std::mutex run_m_, m_;
    std::condition_variable cv_, done_cv_;
    uint64_t gen_ = 0;
    int pending_ = 0;
    const std::function<void(int, int)>* job_ = nullptr;
    int job_nt_ = 1;
};

// [a, b) share of thread t of nt over `bytes`, cut on 64-byte lines.
inline void share(size_t bytes, int t, int nt, size_t* a, size_t* b) {
    *a = (bytes * t / nt) & ~(size_t)63;
    *b = t + 1 == nt ? bytes : (bytes * (t + 1) / nt) & ~(size_t)63;
}

// The same share with its cut points on `align`-byte boundaries of the
// destination address dst (transparent huge pages: two threads first-touching
// one 2 MiB page serialise on its zeroing).  Falls back to share() when the
// shares would be smaller than `align`.
inline void share_at(uintptr_t dst, size_t bytes, int t, int nt, size_t align, size_t* a, size_t* b) {
    if (bytes / nt < align) {
        share(bytes, t, nt, a, b);
        return;
    }
    auto cut = [&](int k) -> size_t {
        if (k <= 0) return 0;
        if (k >= nt) return bytes;
        const uintptr_t p = (dst + bytes * k / nt + align - 1) & ~(uintptr_t)(align - 1);
        return std::min<size_t>(bytes, p - dst);
    };
    *a = cut(t);
    *b = cut(t + 1);
}

// Parallel memcpy on the pool (the record copy-out, a fill without staging).
inline void pool_memcpy(void* dst, const void* src, size_t bytes) {
    if (bytes < ((size_t)1 << 20)) {
        memcpy(dst, src, bytes);
        return;
    }
    HostPool::get().run([&](int t, int nt) {
        size_t a, b;
        share_at((uintptr_t)dst, bytes, t, nt, (size_t)2 << 20, &a, &b);
        nt_copy((char*)dst + a, nullptr, (const char*)src + a, b - a);
        host_sfence();
    });
}

// Progress of the staging thread, read by K0's slab launches (prep()).
struct StageFeed {
    std::mutex m;
    std::condition_variable cv;
    int slabs = 0;            // slabs whose copies are enqueued (stage_ev[1 + c] recorded)
    bool done = false;        // the feeder has finished (or stopped)
    bool inexact = false;     // a narrowed f64 original value did not survive the round trip
    cudaError_t err = cudaSuccess;
    std::atomic<bool> stop{false};   // set by the consumer: stop staging
    void publish(int c) {
        {
            std::lock_guard<std::mutex> lk(m);
            slabs = c;
        }
        cv.notify_all();
    }
    void finish(cudaError_t e, bool bad) {
        {
            std::lock_guard<std::mutex> lk(m);
            done = true;
            if (e != cudaSuccess && err == cudaSuccess) err = e;
            inexact = inexact || bad;
        }
        cv.notify_all();
    }
    void mark_inexact() {
        {
            std::lock_guard<std::mutex> lk(m);
            inexact = true;
        }
        cv.notify_all();
    }
    // Block until slab count c is enqueued (or the feeder stopped); false when
    // the staged data cannot be used (inexact narrowing or a CUDA error).
    bool wait(int c) {
        std::unique_lock<std::mutex> lk(m);
        cv.wait(lk, [&] { return slabs >= c || done || inexact; });
        return !inexact && err == cudaSuccess;
    }
};

}  // namespace pmsz
