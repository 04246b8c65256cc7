// Per-graph specialised evaluator (jit.cpp).
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "eval_common.cuh"
#include "plan.hpp"

namespace hs {

// Code-generation choices (HS_JIT_OPTS="regs=20,win=48,avail=reg,dur=sel")
struct JitOpts {
    // defaults from the B200 A/B sweep (profiles/README.md, r1c)
    int reg_budget = 64;   // end times kept in registers at once
    int reg_window = 400;  // ... when consumed within this many positions
    bool avail_smem = true;   // per-device available times in shared memory
    bool dur_smem = true;     // latency table in shared memory (else selects)
    bool int_max = false;     // max via int64 compare of bit patterns
    int lanes = 256;          // threads (= candidates) per CTA, at most
    bool dbuf = true;         // (set by jit_build) double-buffered genome tile
    static JitOpts from_env();
};

struct JitModule {
    int device = -1;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kern = nullptr, kern_trace = nullptr;
    int T = 0, lanes = 0, slots = 0, ld_cap = 0, blocks_per_sm = 1, sms = 0;
    size_t smem = 0;
    int64_t smem_tile = 0, smem_tile2 = 0, smem_ends = 0, smem_kstate = 0;
    JitOpts opts;
    size_t src_bytes = 0;
    double compile_ms = 0.0;
};

bool jit_eligible(const Plan &p);
// Emits the kernel for T lanes; returns the number of shared-memory slots.
int jit_emit(const Plan &p, int T, const JitOpts &o, std::string *src);
int jit_build(const Plan &p, int device, JitModule **out, std::string *err);
void jit_free(JitModule *m);
int jit_launch(const JitModule &m, const hsk::EvalParams &a, int grid,
               cudaStream_t stream, std::string *err);

}  // namespace hs
