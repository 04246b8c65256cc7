// Host-side packing for hs_eval_host: uint8 genomes in the reference's
// layout (one byte per gene) are packed to 2 bits per gene by a pool of
// host threads into pinned staging buffers while the GPU evaluates the
// previous chunk, so the PCIe link carries ceil(V/4) bytes per candidate
// instead of V (the host path is PCIe-bound). Genes >= K are detected on
// the way (the caller then sends that chunk unpacked, where the kernel
// flags them exactly as before).
#include <cuda_runtime.h>

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

#include <immintrin.h>

#include "host_pack.hpp"

namespace hs {
namespace {

// A fixed pool of worker threads running the parts of one job at a time.
// Parts are claimed from one 64-bit word holding the job number, the job's
// part count and the claim counter, so a worker that wakes late for a
// finished job can never run a part of the next one (the count is read
// from the same word it claims with, never from a separately published
// field the next job may already have overwritten);
// workers spin ~100 us on the job number before sleeping (the host-packing
// pipeline issues its chunks back to back, and a condition-variable wake-up
// of 15 threads per chunk cost ~0.25 ms, r3y), and the caller spins on the
// pending count.
class Pool {
  public:
    explicit Pool(int n) {
        for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_.store(true);
        }
        cv_.notify_all();
        for (auto &t : workers_) t.join();
    }
    int size() const { return int(workers_.size()) + 1; }
    // fn(part) for part in [0, parts), the caller thread taking part too
    void run(int parts, const std::function<void(int)> &fn) {
        std::lock_guard<std::mutex> lk(job_m_);  // one job at a time
        const uint64_t j = job_.load(std::memory_order_relaxed) + 1;
        fn_.store(&fn, std::memory_order_relaxed);
        pending_.store(parts, std::memory_order_relaxed);
        next_.store((j << 32) | (uint64_t(parts) << 16), std::memory_order_release);
        {
            std::lock_guard<std::mutex> g(m_);
            job_.store(j, std::memory_order_release);
        }
        cv_.notify_all();
        work(j);
        while (pending_.load(std::memory_order_acquire) > 0) _mm_pause();
    }

  private:
    static constexpr int kSpin = 2000;
    void work(uint64_t j) {
        for (;;) {
            // next_ = job << 32 | parts << 16 | claimed
            uint64_t v = next_.load(std::memory_order_acquire);
            for (;;) {
                if ((v >> 32) != j || (v & 0xFFFFu) >= ((v >> 16) & 0xFFFFu)) return;
                if (next_.compare_exchange_weak(v, v + 1, std::memory_order_acq_rel)) break;
            }
            // a claimed part keeps job j unfinished, so fn_ is still job j's
            (*fn_.load(std::memory_order_relaxed))(int(v & 0xFFFFu));
            pending_.fetch_sub(1, std::memory_order_release);
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            uint64_t j = job_.load(std::memory_order_acquire);
            for (int i = 0; j == seen && i < kSpin && !stop_.load(); ++i) {
                _mm_pause();
                j = job_.load(std::memory_order_acquire);
            }
            if (j == seen) {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return stop_.load() || job_.load() != seen; });
                if (stop_.load()) return;
                j = job_.load(std::memory_order_acquire);
            }
            if (stop_.load()) return;
            seen = j;
            work(j);
        }
    }
    std::vector<std::thread> workers_;
    std::mutex m_, job_m_;
    std::condition_variable cv_;
    std::atomic<const std::function<void(int)> *> fn_{nullptr};
    std::atomic<uint64_t> next_{0}, job_{0};
    std::atomic<int> pending_{0};
    std::atomic<bool> stop_{false};
};

Pool &pool() {
    static Pool p([] {
        int n = int(std::thread::hardware_concurrency());
        if (const char *v = getenv("HS_HOST_THREADS")) n = std::atoi(v);
        return std::max(0, std::min(n, 64) - 1);
    }());
    return p;
}

constexpr uint64_t kLow7 = 0x7F7F7F7F7F7F7F7Full, kHigh = 0x8080808080808080ull;

// 2-bit packing of one row: genes 4j..4j+3 -> byte j (gene 4j+q in bits
// 2q); returns nonzero when a gene is >= K
inline uint64_t pack_row(const uint8_t *src, int V, uint8_t *dst, int pld, uint64_t kadd) {
    uint64_t bad = 0;
    int i = 0, o = 0;
    for (; i + 8 <= V; i += 8, o += 2) {
        uint64_t x;
        std::memcpy(&x, src + i, 8);
        bad |= (x & kHigh) | (((x & kLow7) + kadd) & kHigh);
        // bytes b0..b7 (each < 4): y byte k = b_k | b_{k+1} << 2, then
        // z byte 0 = b0 | b1 << 2 | b2 << 4 | b3 << 6 (byte 4 likewise)
        const uint64_t y = x | (x >> 6);
        const uint64_t z = y | (y >> 12);
        dst[o] = uint8_t(z);
        dst[o + 1] = uint8_t(z >> 32);
    }
    uint32_t acc = 0;
    int sh = 0;
    for (; i < V; ++i) {
        const uint8_t b = src[i];
        bad |= (uint64_t(b) & 0x80) | ((uint64_t(b & 0x7F) + (kadd & 0xFF)) & 0x80);
        acc |= uint32_t(b & 3) << sh;
        sh += 2;
        if (sh == 8) {
            dst[o++] = uint8_t(acc);
            acc = 0;
            sh = 0;
        }
    }
    if (sh) dst[o++] = uint8_t(acc);
    for (; o < pld; ++o) dst[o] = 0;
    return bad;
}

// AVX2: 32 genes -> 8 bytes per step (maddubs pairs b0 + 4 b1, madd quads
// (b0 + 4 b1) + 16 (b2 + 4 b3), then 32 -> 16 -> 8-bit packs). The row's
// last < 32 genes come from one 32-byte load masked to the row (the bytes
// past it belong to the next row, so only the very last row of the buffer
// takes the scalar tail: any row whose 32-byte tail load would run past
// `end`, the readable bytes of the buffer); genes >= K are found by one
// unsigned max kept across all rows of the range.
__attribute__((target("avx2"))) inline __m256i pack32_avx2(__m256i x) {
    const __m256i m14 = _mm256_set1_epi16(0x0401);       // bytes (1, 4)
    const __m256i m116 = _mm256_set1_epi32(0x00100001);  // words (1, 16)
    const __m256i p = _mm256_maddubs_epi16(x, m14);      // 16 x (b0 + 4 b1)
    const __m256i q = _mm256_madd_epi16(p, m116);        // 8 x packed byte in int32
    const __m256i w = _mm256_packus_epi32(q, q);         // per 128-bit half
    const __m256i b = _mm256_packus_epi16(w, w);         // bytes 0..3 and 16..19
    // both halves' 4 bytes into the low 8 bytes
    return _mm256_permutevar8x32_epi32(b, _mm256_setr_epi32(0, 4, 0, 0, 0, 0, 0, 0));
}

__attribute__((target("avx2"))) uint64_t pack_rows_avx2(const uint8_t *src, int64_t ld,
                                                         int V, int K, int64_t r0, int64_t r1,
                                                         int64_t end, uint8_t *dst,
                                                         int64_t pld, uint64_t kadd) {
    alignas(32) static const uint8_t ones[64] = {
        0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF,
        0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF,
        0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF};  // then 32 zeros
    const int full = V / 32 * 32, t = V - full, o_t = full / 4;
    const int tail_bytes = int(pld) - o_t;  // packed tail + zero padding
    const __m256i tmask =
        _mm256_loadu_si256(reinterpret_cast<const __m256i *>(ones + 32 - t));
    static const int64_t pf_bytes = getenv("HS_PACK_PF") ? atoll(getenv("HS_PACK_PF")) : 4096;
    const int64_t pf_dist = std::max<int64_t>(2, pf_bytes / ld) * ld;
    __m256i mx = _mm256_setzero_si256();
    uint64_t bad = 0;
    for (int64_t r = r0; r < r1; ++r) {
        const uint8_t *s = src + r * ld;
        uint8_t *d = dst + r * pld;
        // ~4 KB ahead: more lines in flight per core than the hardware
        // prefetcher keeps (+15-30 % read rate; prefetches never fault)
        for (int64_t q = 0; q < ld; q += 64)
            _mm_prefetch(reinterpret_cast<const char *>(s + pf_dist + q), _MM_HINT_T0);
        int i = 0, o = 0;
        for (; i < full; i += 32, o += 8) {
            const __m256i x = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(s + i));
            mx = _mm256_max_epu8(mx, x);
            _mm_storel_epi64(reinterpret_cast<__m128i *>(d + o),
                             _mm256_castsi256_si128(pack32_avx2(x)));
        }
        if (t == 0) {
            for (; o < pld; ++o) d[o] = 0;
        } else if (r * ld + i + 32 <= end) {
            const __m256i x = _mm256_and_si256(
                _mm256_loadu_si256(reinterpret_cast<const __m256i *>(s + i)), tmask);
            mx = _mm256_max_epu8(mx, x);
            alignas(16) uint8_t tb[16];
            _mm_store_si128(reinterpret_cast<__m128i *>(tb),
                            _mm256_castsi256_si128(pack32_avx2(x)));
            for (int k = 0; k < tail_bytes; ++k) d[o_t + k] = k < 8 ? tb[k] : 0;
        } else {
            bad |= pack_row(s + i, t, d + o, int(pld) - o, kadd);
        }
    }
    alignas(32) uint8_t m[32];
    _mm256_store_si256(reinterpret_cast<__m256i *>(m), mx);
    for (int k = 0; k < 32; ++k) bad |= m[k] >= K;
    return bad;
}

}  // namespace

int host_pack_threads() { return pool().size(); }

bool pack2_rows(const uint8_t *src, int64_t ld, int V, int K, int64_t rows, uint8_t *dst,
                int64_t pld) {
    const uint64_t kadd = uint64_t(0x80 - K) * 0x0101010101010101ull;
    static const bool avx2 = __builtin_cpu_supports("avx2");
    Pool &pl = pool();
    // (at most 65535 parts: the claim word's 16-bit fields)
    const int parts = int(std::min<int64_t>({rows, int64_t(pl.size()) * 4, 65535}));
    if (parts <= 0) return true;
    std::atomic<uint64_t> bad{0};
    pl.run(parts, [&](int k) {
        const int64_t a = rows * k / parts, b = rows * (k + 1) / parts;
        uint64_t bd = 0;
        if (avx2)
            bd = pack_rows_avx2(src, ld, V, K, a, b, (rows - 1) * ld + V, dst, pld, kadd);
        else
            for (int64_t r = a; r < b; ++r)
                bd |= pack_row(src + r * ld, V, dst + r * pld, int(pld), kadd);
        if (bd) bad.fetch_or(1);
    });
    return bad.load() == 0;
}

// pinned staging buffers, per calling thread (the C ABI is thread-safe)
namespace {
struct Staging {
    void *p[2] = {nullptr, nullptr};
    size_t bytes = 0;
    ~Staging() {
        for (void *q : p)
            if (q) cudaFreeHost(q);
    }
};
thread_local Staging t_stage;
}  // namespace

uint8_t *pinned_staging(int which, size_t bytes) {
    if (bytes > t_stage.bytes) {
        for (void *&q : t_stage.p) {
            if (q) cudaFreeHost(q);
            q = nullptr;
        }
        t_stage.bytes = 0;
        for (void *&q : t_stage.p)
            if (cudaHostAlloc(&q, bytes, cudaHostAllocDefault) != cudaSuccess) {
                q = nullptr;
                return nullptr;
            }
        t_stage.bytes = bytes;
    }
    return static_cast<uint8_t *>(t_stage.p[which & 1]);
}

}  // namespace hs
