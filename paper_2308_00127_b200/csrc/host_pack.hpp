// Host-side 2-bit packing of uint8 genomes for the host-buffer path
// (host_pack.cpp).
#pragma once

#include <cstddef>
#include <cstdint>

namespace hs {

// rows x V genes (row stride ld) -> rows x pld bytes of 2-bit genes
// (hs_eval_packed's layout), on the host thread pool; false when some gene
// is >= K (K <= 4).
bool pack2_rows(const uint8_t *src, int64_t ld, int V, int K, int64_t rows, uint8_t *dst,
                int64_t pld);
// pinned staging buffer `which` (0 / 1) of at least `bytes`, per calling
// thread (reused across calls); nullptr if pinning fails
uint8_t *pinned_staging(int which, size_t bytes);
int host_pack_threads();

}  // namespace hs
