// Kernel parameter blocks and launchers (kernels.cu), used by capi.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "plan.hpp"

namespace hs {

// runtime-uniform feature flags of the evaluator
enum : uint32_t {
    F_MEM = 1u,   // capacity can bind (heuristics.py:98-100)
    F_OKL = 2u,   // some device lacks batch size L (heuristics.py:96)
    F_MISS = 4u,  // some (task, dev, L) latency entry is missing
    F_NAN = 8u,   // a NaN can reach a time: keep the running makespan max
};

struct EvalParams {
    const uint8_t *blob;  // device plan blob (slots pre-scaled by lanes)
    DevLayout lay;
    int64_t eval_bytes;
    int V, K;
    uint32_t flags;
    int plan_smem;
    int lanes, ld_s, slots;
    int bulk;             // genome tiles may use cp.async.bulk
    // candidates
    const uint8_t *genes;
    int64_t n, ld;
    int gen;              // 1: hash-random, 2: enumerate (K6); 0: staged genes
    uint64_t seed;
    int64_t first;
    const uint8_t *tmpl;  // [V] fixed genes where group < 0
    const int16_t *group; // [V] group per position (null: identity)
    int n_groups;
    // outputs (each may be null)
    double *makespan;
    uint8_t *status;
    double *starts;       // trace: [n][V]
    uint8_t *genes_out;   // gen: [n][V]
    hs_best *best;
    hs_best *partial;     // [grid]
    unsigned int *ticket;
    int64_t index_base;
};

int eval_occupancy(int kt, bool cls, int T, size_t smem, int *blocks);
int launch_eval(const DevState &ds, bool cls, const EvalParams &p, int grid,
                cudaStream_t stream, std::string *err);
int launch_cp(const uint8_t *blob, const DevLayout &lay, int V, int words,
              const uint64_t *masks, int64_t nsub, double *out, uint8_t *status,
              double *scratch, cudaStream_t stream, std::string *err);
int launch_reach(const uint8_t *blob, const DevLayout &lay, int NT, int words,
                 uint64_t *desc, uint64_t *anc, cudaStream_t stream,
                 std::string *err);

}  // namespace hs
