// Per-graph specialised evaluator (jit.cpp).
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "eval_common.cuh"
#include "plan.hpp"

namespace hs {

// Code-generation choices (HS_JIT_OPTS="regs=20,win=48,avail=reg,dur=sel")
struct JitOpts {
    // defaults from the B200 A/B sweeps (profiles/README.md, r1c and r1g)
    int reg_budget = 64;   // end times kept in registers at once
    int reg_window = 400;  // ... when consumed within this many positions
    bool avail_smem = true;   // per-device available times in shared memory
    bool dur_smem = true;     // latency table in shared memory (else selects)
    int dur_smem_max = 1 << 30;  // ... up to this many bytes, else read through L1
                              // (measured slower on tf96: 8.3e8 vs 1.16e9)
    bool int_max = false;     // max via int64 compare of bit patterns
    bool genes_reg = false;   // genes 2 bits each in registers (K <= 4)
    int near = 8;             // > 0: split residency (registers for consumers
                              // within `near` positions, long storage beyond)
    int lanes = 256;          // threads (= candidates) per CTA, at most
    bool lanes_set = false;   // `lanes` given explicitly (HS_JIT_OPTS)
    int ahead = 2;            // software pipelining distance (tasks)
    bool dom = true;          // drop same-device predecessor terms (dominated)
    bool gword = false;       // genes read four per 32-bit shared-memory load
    bool fma = false;         // communication term as one fma (exact)
    int ctas = 1;             // CTAs per SM the direct-load kernel is built for
    bool dbuf = true;         // (set by jit_build) double-buffered genome tile
    bool gslots = false;      // (set by jit_build) end-time slots in global memory
    int sync = 0;             // CTA barrier every `sync` tasks (0: none)
    bool tmem = true;         // end-time slots in tensor memory (TMEM) when they fit
    int tm_lanes = 384;       // lanes per CTA with TMEM slots (12 warps)
    int tm_regs = 40;         // long-lived end times in registers with TMEM slots
    int tm_cols = 0;          // (set by jit_build) TMEM columns per warp group
    int tm_ctas = 1;          // CTAs per SM on the TMEM tier (each allocates
                              // 512 / tm_ctas columns, lanes / tm_ctas lanes)
    bool tm_dev = false;      // TMEM slots also hold the producer's device
                              // (4 columns per slot: the consumer's device
                              // compare needs no shared-memory gene load);
                              // measured neutral on WS200, -3 % on the WS
                              // 10x20 stack (profiles r2e), so off
    int gslot_lanes = 192;    // lanes per CTA with global-memory slots (sweep r1h)
    bool blk = true;          // node-block link classes computed, not looked up
                              // (full mesh; same device / same node / other)
    static JitOpts from_env();
};

struct JitModule {
    int device = -1;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kern = nullptr, kern_trace = nullptr;
    cudaKernel_t kern_direct = nullptr;  // genes from global into registers
    cudaKernel_t kern_sa = nullptr, kern_ea = nullptr;  // single-CTA search
    size_t smem_direct = 0;
    bool ends_global = false;  // end-time slots in global memory
    bool tmem = false;         // end-time slots in tensor memory
    int blocks_per_sm_direct = 0;
    int T = 0, lanes = 0, slots = 0, ld_cap = 0, blocks_per_sm = 1, sms = 0;
    size_t smem = 0;
    int64_t smem_tile = 0, smem_tile2 = 0, smem_ends = 0, smem_kstate = 0;
    JitOpts opts;
    size_t src_bytes = 0;
    double compile_ms = 0.0;
};

bool jit_eligible(const Plan &p);
bool jit_search_ok(const Plan &p);
// Emits the kernel for T lanes; returns the number of shared-memory slots.
int jit_emit(const Plan &p, int T, const JitOpts &o, std::string *src);
// batched-variant plans (extended genomes): the K8 semantics as straight-line code
int jit_emit_batched(const Plan &p, int T, const JitOpts &o, std::string *src, bool dbuf);
int jit_build(const Plan &p, int device, JitModule **out, std::string *err);
void jit_free(JitModule *m);
// the launch may use the direct-load kernel (explicit u8 genes, 4-aligned)
bool jit_direct_ok(const JitModule &m, const hsk::EvalParams &a);
int jit_launch(const JitModule &m, const hsk::EvalParams &a, int grid,
               cudaStream_t stream, std::string *err);
// one CTA of the SA (mode 1) or EA (mode 2) search kernel; `ps` -> params
int jit_launch_search(const JitModule &m, int mode, const hsk::EvalParams &a,
                      const void *ps, cudaStream_t stream, std::string *err, int grid = 1);

}  // namespace hs
