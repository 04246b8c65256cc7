// Host memory read ceiling vs the hs_eval_host packer on the same rows:
// T threads stream-read (AVX2 loads, OR-reduce) a 1.7 GB buffer -- the
// uint8 rows of one 8.4 M-candidate WS200 call -- and the packer
// (csrc/host_pack.cpp) packs the same buffer in 512 K-row chunks.
//   g++ -O3 -mavx2 -std=c++17 -I paper_2308_00127_b200/csrc tools/native/host_read_bw.cpp \
//       paper_2308_00127_b200/csrc/host_pack.cpp -lcudart -lpthread
#include <immintrin.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "host_pack.hpp"

int main(int argc, char **argv) {
    const int V = 202;
    const int64_t rows = int64_t(1) << 23, chunk = int64_t(1) << 19;
    const int64_t pld = ((V + 3) / 4 + 3) / 4 * 4;
    const size_t bytes = size_t(rows) * V;
    uint8_t *src = nullptr;
    const bool pinned = argc > 1 && atoi(argv[1]);  // cudaHostAlloc, as torch pin_memory
    if (pinned) {
        if (cudaHostAlloc(reinterpret_cast<void **>(&src), bytes, cudaHostAllocDefault) != cudaSuccess)
            return 1;
    } else {
        src = static_cast<uint8_t *>(aligned_alloc(64, (bytes + 63) / 64 * 64));
    }
    for (size_t i = 0; i < bytes; ++i) src[i] = uint8_t(i % 3);
    std::vector<uint8_t> dst(size_t(chunk) * pld);
    for (int T : {16}) {
        if (T > int(std::thread::hardware_concurrency())) break;
        std::vector<uint64_t> out(T);
        double best = 1e30;
        for (int rep = 0; rep < 3; ++rep) {
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t)
                th.emplace_back([&, t] {
                    const size_t a = bytes / 32 * t / T * 32, b = bytes / 32 * (t + 1) / T * 32;
                    __m256i acc = _mm256_setzero_si256();
                    for (size_t i = a; i < b; i += 32)
                        acc = _mm256_or_si256(
                            acc, _mm256_load_si256(reinterpret_cast<const __m256i *>(src + i)));
                    alignas(32) uint64_t m[4];
                    _mm256_store_si256(reinterpret_cast<__m256i *>(m), acc);
                    out[t] = m[0] | m[1] | m[2] | m[3];
                });
            for (auto &x : th) x.join();
            best = std::min(best, std::chrono::duration<double>(
                                      std::chrono::steady_clock::now() - t0).count());
        }
        printf("read  T=%2d: %6.1f GB/s\n", T, bytes / best / 1e9);
    }
    double best = 1e30;
    for (int rep = 0; rep < 3; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        for (int64_t r = 0; r < rows; r += chunk)
            hs::pack2_rows(src + r * V, V, V, 3, chunk, dst.data(), pld);
        best = std::min(best, std::chrono::duration<double>(
                                  std::chrono::steady_clock::now() - t0).count());
    }
    printf("pack  T=%2d: %6.1f GB/s (%.3g rows/s)\n", hs::host_pack_threads(), bytes / best / 1e9,
           rows / best);
    return 0;
}
