// Stream-ordered scratch for the C ABI's per-call buffers (speculation
// scratch, host-pipeline chunk buffers, reductions, validator tables).
// Allocations come from a library-owned memory pool per device whose
// release threshold is unlimited: freed blocks stay mapped for the next
// call instead of being returned to the driver at every synchronisation (the
// default pool's threshold is 0, and re-mapping cost 5–40 ms per call on the
// host, measured r3s). The pool keeps its high-water mark until
// hs_scratch_trim() or process exit.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace hs {
cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t s);
int scratch_trim();  // hs_scratch_trim
}
