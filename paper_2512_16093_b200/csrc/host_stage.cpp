// host_stage.cpp -- host-side staging for the drop-in's numpy in / numpy out
// path (attention.sla_attention on host arrays at scale, ops.sla_attention_host).
//
// The reference API hands the attention pageable numpy f32 arrays.  DMA from
// pageable memory runs at ~12 GB/s, so every head chunk is first copied into
// page-locked staging buffers and uploaded from there at PCIe rate.  That copy
// (and, for V, the f32 -> bf16 rounding the kernels consume) is host-memory
// bound: a persistent pool of worker threads splits it into
// spans (64 Ki elements each) and writes the staging buffer with non-temporal stores (no
// read-for-ownership of the destination lines, which would otherwise add a
// third of the traffic and contend with the DMA engine reading the previous
// chunk out of the same memory).
//
// bf16-valued f32 arrays (low 16 bits zero -- a bf16 model's activations handed
// over as f32) can be staged as their bf16 bit patterns instead
// (tb_host_stage_bf16_exact): lossless, half the PCIe bytes; the check rides
// along with the copy and gives up at the first inexact value.
//
// Not a compute path: the values are moved (or rounded to bf16 exactly like
// __float2bfloat16_rn / torch's cast), never computed on.
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <unistd.h>

#include "../../include/tb_capi.h"

namespace {

// -------------------------------------------------------------- thread pool
class Pool {
  public:
    explicit Pool(int n) : n_(n) {
        for (int i = 1; i < n_; i++) workers_.emplace_back([this, i] { loop(i); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
            gen_++;
        }
        cv_.notify_all();
        for (auto &t : workers_) t.join();
    }
    int size() const { return n_; }
    // runs fn(i) for i in [0, parts) over the pool; the caller takes part of the work
    void run(int parts, const std::function<void(int)> &fn) {
        std::unique_lock<std::mutex> g(run_m_);          // one job at a time
        {
            std::lock_guard<std::mutex> l(m_);
            fn_ = &fn;
            parts_ = parts;
            next_.store(0);
            done_.store(0);
            gen_++;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> l(m_);
        done_cv_.wait(l, [&] { return done_.load() == parts_; });
        fn_ = nullptr;
    }

  private:
    void work() {
        for (;;) {
            const int i = next_.fetch_add(1);
            if (i >= parts_) return;
            (*fn_)(i);
            if (done_.fetch_add(1) + 1 == parts_) {
                std::lock_guard<std::mutex> l(m_);
                done_cv_.notify_all();
            }
        }
    }
    void loop(int) {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> l(m_);
                cv_.wait(l, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                if (fn_ == nullptr) continue;
            }
            work();
        }
    }
    int n_;
    std::vector<std::thread> workers_;
    std::mutex m_, run_m_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)> *fn_ = nullptr;
    int parts_ = 0;
    std::atomic<int> next_{0}, done_{0};
    uint64_t gen_ = 0;
    bool stop_ = false;
};

Pool &pool(int want) {
    static Pool *p = nullptr;
    static pid_t owner = 0;
    static std::mutex m;
    std::lock_guard<std::mutex> g(m);
    // a forked child inherits the pointer but not the worker threads: start a
    // fresh pool there (the parent's object is left alone)
    if (p != nullptr && owner != getpid()) p = nullptr;
    if (p == nullptr) {
        owner = getpid();
        int n = want;
        if (n <= 0) {
            const char *e = getenv("TB_HOST_THREADS");
            n = e ? atoi(e) : (int)std::thread::hardware_concurrency();
        }
        p = new Pool(std::max(1, std::min(n, 64)));      // process lifetime (never joined at exit)
    }
    return *p;
}

// ------------------------------------------------------------ span kernels
inline uint16_t bf16_rn(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7FFFFFFFu) > 0x7F800000u) return (uint16_t)((u >> 16) | 0x40);   // quiet NaN
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

__attribute__((target("avx2"))) void copy_avx2(uint8_t *dst, const uint8_t *src, int64_t bytes) {
    int64_t i = 0;
    // align the destination to 32 B for the streaming stores
    while (i < bytes && ((uintptr_t)(dst + i) & 31)) { dst[i] = src[i]; i++; }
    for (; i + 128 <= bytes; i += 128) {
        const __m256i a = _mm256_loadu_si256((const __m256i *)(src + i));
        const __m256i b = _mm256_loadu_si256((const __m256i *)(src + i + 32));
        const __m256i c = _mm256_loadu_si256((const __m256i *)(src + i + 64));
        const __m256i d = _mm256_loadu_si256((const __m256i *)(src + i + 96));
        _mm256_stream_si256((__m256i *)(dst + i), a);
        _mm256_stream_si256((__m256i *)(dst + i + 32), b);
        _mm256_stream_si256((__m256i *)(dst + i + 64), c);
        _mm256_stream_si256((__m256i *)(dst + i + 96), d);
    }
    for (; i < bytes; i++) dst[i] = src[i];
    _mm_sfence();                                         // this thread's streaming stores drained
}

// 8 x f32 -> bf16 round-to-nearest-even (NaN stays NaN), in the low half of each lane
__attribute__((target("avx2"))) inline __m256i cvt8_bf16(const float *p) {
    const __m256i bias = _mm256_set1_epi32(0x7FFF), one = _mm256_set1_epi32(1);
    const __m256i absm = _mm256_set1_epi32(0x7FFFFFFF), inf = _mm256_set1_epi32(0x7F800000);
    const __m256i qnan = _mm256_set1_epi32(0x00400000);
    __m256i u = _mm256_castps_si256(_mm256_loadu_ps(p));
    const __m256i nan = _mm256_cmpgt_epi32(_mm256_and_si256(u, absm), inf);
    const __m256i r = _mm256_add_epi32(u, _mm256_add_epi32(bias, _mm256_and_si256(_mm256_srli_epi32(u, 16), one)));
    u = _mm256_blendv_epi8(r, _mm256_or_si256(u, qnan), nan);
    return _mm256_srli_epi32(u, 16);
}

__attribute__((target("avx2"))) void to_bf16_avx2(uint16_t *dst, const float *src, int64_t n) {
    int64_t i = 0;
    while (i < n && ((uintptr_t)(dst + i) & 31)) { dst[i] = bf16_rn(src[i]); i++; }
    for (; i + 16 <= n; i += 16) {
        const __m256i lo = cvt8_bf16(src + i), hi = cvt8_bf16(src + i + 8);
        // packus works per 128-bit lane: [lo0 hi0 lo1 hi1] -> reorder the 64-bit quarters
        const __m256i pk = _mm256_permute4x64_epi64(_mm256_packus_epi32(lo, hi), 0xD8);
        _mm256_stream_si256((__m256i *)(dst + i), pk);
    }
    for (; i < n; i++) dst[i] = bf16_rn(src[i]);
    _mm_sfence();
}

// f32 -> bf16 when every value is exactly representable (low 16 bits zero):
// the upper halves, streamed; false as soon as a 1 K-element run holds a value
// that is not (the destination is then unspecified)
__attribute__((target("avx2"))) bool to_bf16_exact_avx2(uint16_t *dst, const float *src, int64_t n) {
    const uint32_t *u = reinterpret_cast<const uint32_t *>(src);
    int64_t i = 0;
    for (; i < n && ((uintptr_t)(dst + i) & 31); i++) {
        if (u[i] & 0xFFFFu) return false;
        dst[i] = (uint16_t)(u[i] >> 16);
    }
    const __m256i low = _mm256_set1_epi32(0xFFFF);
    while (i + 16 <= n) {
        const int64_t run = std::min<int64_t>(n - (n - i) % 16, i + 1024);
        __m256i seen = _mm256_setzero_si256();
        for (; i < run; i += 16) {
            const __m256i a = _mm256_loadu_si256((const __m256i *)(u + i));
            const __m256i b = _mm256_loadu_si256((const __m256i *)(u + i + 8));
            seen = _mm256_or_si256(seen, _mm256_or_si256(a, b));
            const __m256i pk = _mm256_permute4x64_epi64(
                _mm256_packus_epi32(_mm256_srli_epi32(a, 16), _mm256_srli_epi32(b, 16)), 0xD8);
            _mm256_stream_si256((__m256i *)(dst + i), pk);
        }
        if (!_mm256_testz_si256(seen, low)) { _mm_sfence(); return false; }
    }
    for (; i < n; i++) {
        if (u[i] & 0xFFFFu) { _mm_sfence(); return false; }
        dst[i] = (uint16_t)(u[i] >> 16);
    }
    _mm_sfence();
    return true;
}

bool to_bf16_exact_scalar(uint16_t *dst, const float *src, int64_t n) {
    const uint32_t *u = reinterpret_cast<const uint32_t *>(src);
    for (int64_t i = 0; i < n; i++) {
        if (u[i] & 0xFFFFu) return false;
        dst[i] = (uint16_t)(u[i] >> 16);
    }
    return true;
}

void copy_scalar(uint8_t *dst, const uint8_t *src, int64_t bytes) { std::memcpy(dst, src, (size_t)bytes); }
void to_bf16_scalar(uint16_t *dst, const float *src, int64_t n) {
    for (int64_t i = 0; i < n; i++) dst[i] = bf16_rn(src[i]);
}

bool have_avx2() {
    static const bool ok = __builtin_cpu_supports("avx2");
    return ok;
}

// elements per work item (256 KB of f32): ~18 spans per thread for a 2-head
// cfg4 chunk keeps the 16 threads evenly loaded (2^18: 74 spans, 5 rounds with
// the last one 10/16 full -- 73 vs 75 ms drop-in e2e; 2^20: 86 ms)
constexpr int64_t SPAN = 1 << 16;

}  // namespace

extern "C" int tb_host_stage(void *dst, const void *src, int64_t n, int src_dtype, int dst_dtype,
                             int64_t nthreads) {
    if (n < 0 || (n > 0 && (dst == nullptr || src == nullptr))) return TB_EINVAL;
    const bool copy = src_dtype == dst_dtype && (src_dtype == TB_F32 || src_dtype == TB_BF16 || src_dtype == TB_I8);
    const bool cvt = src_dtype == TB_F32 && dst_dtype == TB_BF16;
    if (!copy && !cvt) return TB_EINVAL;
    if (n == 0) return TB_OK;
    const int64_t es = src_dtype == TB_F32 ? 4 : src_dtype == TB_BF16 ? 2 : 1;
    const int64_t parts = (n + SPAN - 1) / SPAN;
    Pool &p = pool((int)nthreads);
    const bool v = have_avx2();
    auto body = [&](int i) {
        const int64_t a = (int64_t)i * SPAN, z = std::min(n, a + SPAN);
        if (copy) {
            uint8_t *d = (uint8_t *)dst + a * es;
            const uint8_t *s = (const uint8_t *)src + a * es;
            v ? copy_avx2(d, s, (z - a) * es) : copy_scalar(d, s, (z - a) * es);
        } else {
            uint16_t *d = (uint16_t *)dst + a;
            const float *s = (const float *)src + a;
            v ? to_bf16_avx2(d, s, z - a) : to_bf16_scalar(d, s, z - a);
        }
    };
    if (parts == 1 || p.size() == 1) {
        for (int i = 0; i < (int)parts; i++) body(i);
    } else {
        p.run((int)parts, body);
    }
    return TB_OK;                                         // every span ended with its sfence
}

extern "C" int64_t tb_host_threads(void) { return pool(0).size(); }

extern "C" int tb_host_stage_bf16_exact(void *dst, const float *src, int64_t n, int64_t nthreads) {
    if (n < 0 || (n > 0 && (dst == nullptr || src == nullptr))) return TB_EINVAL;
    if (n == 0) return 1;
    const int64_t parts = (n + SPAN - 1) / SPAN;
    Pool &p = pool((int)nthreads);
    const bool v = have_avx2();
    std::atomic<bool> inexact{false};
    auto body = [&](int i) {
        if (inexact.load(std::memory_order_relaxed)) return;     // another span already failed
        const int64_t a = (int64_t)i * SPAN, z = std::min(n, a + SPAN);
        uint16_t *d = (uint16_t *)dst + a;
        const bool ok = v ? to_bf16_exact_avx2(d, src + a, z - a) : to_bf16_exact_scalar(d, src + a, z - a);
        if (!ok) inexact.store(true, std::memory_order_relaxed);
    };
    if (parts == 1 || p.size() == 1) {
        for (int i = 0; i < (int)parts && !inexact.load(); i++) body(i);
    } else {
        p.run((int)parts, body);
    }
    return inexact.load() ? 0 : 1;
}
