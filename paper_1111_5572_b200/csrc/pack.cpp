// pack.cpp -- host-side read packing for the batch path.
//
// The batch call takes reads as ASCII (one byte per base, REF
// include/seedaln/genome.hpp Read::bases).  Shipping those bytes over PCIe is
// the e2e bound at C1 (108 MB per 1 M reads at ~54 GB/s = 2.0 ms, the same as
// the kernels), so the seeded pipeline packs each chunk on the host into three
// bit planes before the copy:
//
//   plane 0 (lo): bit i = base i is C or T      (2-bit code bit 0, A=0 C=1 G=2 T=3)
//   plane 1 (hi): bit i = base i is G or T      (code bit 1)
//   plane 2 (n) : bit i = base i is N
//
// 3 bits per base, 0.375 B instead of 1 B.  A byte outside {A,C,G,T,N} is
// marked lo = n = 1 (a combination no base has), so the seed kernel still sees
// the bad character and fails the batch exactly as it does on ASCII input
// (REF src/genome.cpp:182-200 reverse_complement throws for the read).
//
// Packing runs on a small persistent thread pool (AVX-512BW, AVX2 or scalar,
// chosen at run time), one slice of whole 64-base groups per task.
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "host_common.h"

namespace sab {
namespace {

// byte -> {lo, hi, n} bits (bit 0, 1, 2)
struct CodeLut {
    uint8_t v[256];
    CodeLut() {
        for (int c = 0; c < 256; ++c) v[c] = 5;  // invalid: lo = n = 1
        v['A'] = 0;
        v['C'] = 1;
        v['G'] = 2;
        v['T'] = 3;
        v['N'] = 4;
    }
};
const CodeLut kLut;

// scalar reference: one 32-base word
inline void pack_word_scalar(const char* s, int n, uint32_t& lo, uint32_t& hi, uint32_t& nn) {
    lo = hi = nn = 0;
    for (int i = 0; i < n; ++i) {
        const uint32_t c = kLut.v[static_cast<uint8_t>(s[i])];
        lo |= (c & 1u) << i;
        hi |= ((c >> 1) & 1u) << i;
        nn |= ((c >> 2) & 1u) << i;
    }
}

// words [w0, w1) of the planes from src[0, n)
void pack_scalar(const char* src, uint64_t n, uint64_t w0, uint64_t w1, uint32_t* lo, uint32_t* hi,
                 uint32_t* nn) {
    for (uint64_t w = w0; w < w1; ++w) {
        const uint64_t b = 32 * w;
        const int k = b >= n ? 0 : static_cast<int>(std::min<uint64_t>(32, n - b));
        pack_word_scalar(src + b, k, lo[w], hi[w], nn[w]);
    }
}

__attribute__((target("avx2"))) void pack_avx2(const char* src, uint64_t n, uint64_t w0, uint64_t w1,
                                                uint32_t* lo, uint32_t* hi, uint32_t* nn) {
    const __m256i A = _mm256_set1_epi8('A'), C = _mm256_set1_epi8('C'), G = _mm256_set1_epi8('G');
    const __m256i T = _mm256_set1_epi8('T'), N = _mm256_set1_epi8('N');
    uint64_t w = w0;
    for (; w < w1 && 32 * w + 32 <= n; ++w) {
        const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + 32 * w));
        const uint32_t a = static_cast<uint32_t>(_mm256_movemask_epi8(_mm256_cmpeq_epi8(v, A)));
        const uint32_t c = static_cast<uint32_t>(_mm256_movemask_epi8(_mm256_cmpeq_epi8(v, C)));
        const uint32_t g = static_cast<uint32_t>(_mm256_movemask_epi8(_mm256_cmpeq_epi8(v, G)));
        const uint32_t t = static_cast<uint32_t>(_mm256_movemask_epi8(_mm256_cmpeq_epi8(v, T)));
        const uint32_t x = static_cast<uint32_t>(_mm256_movemask_epi8(_mm256_cmpeq_epi8(v, N)));
        const uint32_t bad = ~(a | c | g | t | x);
        lo[w] = c | t | bad;
        hi[w] = g | t;
        nn[w] = x | bad;
    }
    pack_scalar(src, n, w, w1, lo, hi, nn);
}

__attribute__((target("avx512f,avx512bw"))) void pack_avx512(const char* src, uint64_t n, uint64_t w0,
                                                              uint64_t w1, uint32_t* lo, uint32_t* hi,
                                                              uint32_t* nn) {
    const __m512i A = _mm512_set1_epi8('A'), C = _mm512_set1_epi8('C'), G = _mm512_set1_epi8('G');
    const __m512i T = _mm512_set1_epi8('T'), N = _mm512_set1_epi8('N');
    uint64_t w = w0;
    for (; w + 1 < w1 && 32 * w + 64 <= n; w += 2) {
        const __m512i v = _mm512_loadu_si512(src + 32 * w);
        const uint64_t a = _mm512_cmpeq_epi8_mask(v, A), c = _mm512_cmpeq_epi8_mask(v, C);
        const uint64_t g = _mm512_cmpeq_epi8_mask(v, G), t = _mm512_cmpeq_epi8_mask(v, T);
        const uint64_t x = _mm512_cmpeq_epi8_mask(v, N);
        const uint64_t bad = ~(a | c | g | t | x);
        const uint64_t l = c | t | bad, h = g | t, m = x | bad;
        std::memcpy(lo + w, &l, 8);
        std::memcpy(hi + w, &h, 8);
        std::memcpy(nn + w, &m, 8);
    }
    pack_avx2(src, n, w, w1, lo, hi, nn);
}

using PackFn = void (*)(const char*, uint64_t, uint64_t, uint64_t, uint32_t*, uint32_t*, uint32_t*);

PackFn pick(int isa) {  // isa: 0 auto, 1 scalar, 2 avx2, 3 avx512
    if (isa == 0) {
        __builtin_cpu_init();
        if (__builtin_cpu_supports("avx512bw")) return pack_avx512;
        if (__builtin_cpu_supports("avx2")) return pack_avx2;
        return pack_scalar;
    }
    return isa == 3 ? pack_avx512 : isa == 2 ? pack_avx2 : pack_scalar;
}

// Persistent workers; the caller takes tasks too.  One job at a time.  The
// task cursor carries the job generation in its high half, so a worker that
// wakes late for an old job can neither run nor steal a task of the next one.
class PackPool {
  public:
    explicit PackPool(int n_threads) {
        for (int i = 0; i < n_threads; ++i) th_.emplace_back([this] { loop(); });
    }
    ~PackPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void run(PackFn fn, const char* src, uint64_t n, uint32_t* planes, uint64_t wpp) {
        std::lock_guard<std::mutex> one(job_mu_);
        Job j;
        j.fn = fn;
        j.src = src;
        j.n = n;
        j.lo = planes;
        j.hi = planes + wpp;
        j.nn = planes + 2 * wpp;
        j.words = (n + 31) / 32;
        j.n_tasks = (j.words + kTaskWords - 1) / kTaskWords;
        {
            std::lock_guard<std::mutex> g(mu_);
            j.gen = ++gen_;
            job_ = j;
            done_.store(0);
            cursor_.store(j.gen << 32);
        }
        if (j.n_tasks > 1 && !th_.empty()) cv_.notify_all();
        work(j);
        while (done_.load(std::memory_order_acquire) < j.n_tasks) std::this_thread::yield();
    }

  private:
    static constexpr uint64_t kTaskWords = 8192;  // 256 k bases per task; no word is shared
    struct Job {
        PackFn fn = nullptr;
        const char* src = nullptr;
        uint64_t n = 0, words = 0, n_tasks = 0, gen = 0;
        uint32_t *lo = nullptr, *hi = nullptr, *nn = nullptr;
    };
    void work(const Job& j) {
        uint64_t c = cursor_.load();
        for (;;) {
            if ((c >> 32) != j.gen || (c & 0xffffffffu) >= j.n_tasks) return;
            if (!cursor_.compare_exchange_weak(c, c + 1)) continue;
            const uint64_t w0 = (c & 0xffffffffu) * kTaskWords, w1 = std::min(j.words, w0 + kTaskWords);
            j.fn(j.src, j.n, w0, w1, j.lo, j.hi, j.nn);
            done_.fetch_add(1, std::memory_order_release);
            c = cursor_.load();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            Job j;
            {
                std::unique_lock<std::mutex> g(mu_);
                cv_.wait(g, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                j = job_;
            }
            work(j);
        }
    }
    std::vector<std::thread> th_;
    std::mutex mu_, job_mu_;
    std::condition_variable cv_;
    bool stop_ = false;
    uint64_t gen_ = 0;
    Job job_;
    std::atomic<uint64_t> cursor_{0}, done_{0};
};

// SA_PACK_THREADS=n (n > 0) turns packing on with n threads (0: never).
// Unset: pinned callers send ASCII (8 threads pack ~22 GB/s, host memory
// bound, slower than the 54 GB/s copy engine moves it unpacked), pageable
// callers are packed by every host thread -- their bytes must cross host
// memory once anyway, and packing writes 3/8 of what a staging copy writes
// (C2 pageable e2e 52.4 -> 43.4 ms).
int pack_threads_for(bool pageable) {
    const char* e = getenv("SA_PACK_THREADS");
    if (e) return std::max(0, std::min(64, atoi(e)));
    if (!pageable) return 0;
    return std::max(4, std::min(64, static_cast<int>(std::thread::hardware_concurrency())));
}

// Generic persistent worker pool for host copies into pinned staging
// buffers (the batcher's pageable-input path): tasks of one job are claimed
// from a generation-tagged cursor exactly like PackPool's.
class CopyPool {
  public:
    explicit CopyPool(int n_threads) {
        for (int i = 0; i < n_threads; ++i) th_.emplace_back([this] { loop(); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void run(char* dst, const char* src, uint64_t n) {
        std::lock_guard<std::mutex> one(job_mu_);
        Job j;
        j.dst = dst;
        j.src = src;
        j.n = n;
        j.n_tasks = (n + kTaskBytes - 1) / kTaskBytes;
        {
            std::lock_guard<std::mutex> g(mu_);
            j.gen = ++gen_;
            job_ = j;
            done_.store(0);
            cursor_.store(j.gen << 32);
        }
        if (j.n_tasks > 1 && !th_.empty()) cv_.notify_all();
        work(j);
        while (done_.load(std::memory_order_acquire) < j.n_tasks) std::this_thread::yield();
    }

  private:
    static constexpr uint64_t kTaskBytes = 1ull << 20;
    struct Job {
        char* dst = nullptr;
        const char* src = nullptr;
        uint64_t n = 0, n_tasks = 0, gen = 0;
    };
    void work(const Job& j) {
        uint64_t c = cursor_.load();
        for (;;) {
            if ((c >> 32) != j.gen || (c & 0xffffffffu) >= j.n_tasks) return;
            if (!cursor_.compare_exchange_weak(c, c + 1)) continue;
            const uint64_t b0 = (c & 0xffffffffu) * kTaskBytes, b1 = std::min(j.n, b0 + kTaskBytes);
            std::memcpy(j.dst + b0, j.src + b0, b1 - b0);
            done_.fetch_add(1, std::memory_order_release);
            c = cursor_.load();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            Job j;
            {
                std::unique_lock<std::mutex> g(mu_);
                cv_.wait(g, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                j = job_;
            }
            work(j);
        }
    }
    std::vector<std::thread> th_;
    std::mutex mu_, job_mu_;
    std::condition_variable cv_;
    bool stop_ = false;
    uint64_t gen_ = 0;
    Job job_;
    std::atomic<uint64_t> cursor_{0}, done_{0};
};

// SA_STAGE_THREADS=n: host threads copying pageable input into the pinned
// staging buffers (default: half the host's threads, 4..16).
int stage_threads_setting() {
    const char* e = getenv("SA_STAGE_THREADS");
    if (e) return std::max(1, std::min(64, atoi(e)));
    const int hw = static_cast<int>(std::thread::hardware_concurrency());
    return std::max(4, std::min(16, hw / 2));
}

}  // namespace

void parallel_copy(void* dst, const void* src, uint64_t n) {
    if (n < (4ull << 20)) {
        std::memcpy(dst, src, n);
        return;
    }
    static CopyPool pool(stage_threads_setting() - 1);  // the caller is one of the copiers
    pool.run(static_cast<char*>(dst), static_cast<const char*>(src), n);
}

bool pack_enabled(bool pageable) { return pack_threads_for(pageable) > 0; }

uint64_t pack_words_per_plane(uint64_t n_bases) { return (n_bases + 31) / 32 + 2; }

// Planes of src[0, n) into planes[3 * wpp] (wpp >= pack_words_per_plane(n));
// the two pad words of each plane are zeroed (the kernel's funnel shift reads
// one word past a read's last block).
void pack_planar(const char* src, uint64_t n, uint32_t* planes, uint64_t wpp) {
    static PackPool pool(std::max(1, pack_threads_for(true)) - 1);  // sized at first use
    static const PackFn fn = pick(0);
    const uint64_t words = (n + 31) / 32;
    for (int p = 0; p < 3; ++p)
        for (uint64_t w = words; w < wpp && w < words + 2; ++w) planes[p * wpp + w] = 0;
    pool.run(fn, src, n, planes, wpp);
}

}  // namespace sab

// test hook (not in include/): pack with a given ISA, single-threaded
extern "C" int sab_debug_pack(const char* src, uint64_t n, uint32_t* planes, uint64_t wpp, int isa) {
    if (wpp < sab::pack_words_per_plane(n) || isa < 0 || isa > 3) return SA_EINVAL;
    if (isa == 3 && !__builtin_cpu_supports("avx512bw")) return SA_ERUNTIME;
    if (isa == 2 && !__builtin_cpu_supports("avx2")) return SA_ERUNTIME;
    const uint64_t words = (n + 31) / 32;
    for (int p = 0; p < 3; ++p)
        for (uint64_t w = words; w < words + 2; ++w) planes[p * wpp + w] = 0;
    sab::pick(isa)(src, n, 0, words, planes, planes + wpp, planes + 2 * wpp);
    return SA_OK;
}
