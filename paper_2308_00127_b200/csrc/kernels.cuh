// Launchers of the ahead-of-time kernels (kernels.cu), used by capi.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "eval_common.cuh"
#include "plan.hpp"

namespace hs {

using hsk::EvalParams;
using hsk::F_MEM;
using hsk::F_MISS;
using hsk::F_NAN;
using hsk::F_OKL;

int eval_occupancy(int kt, bool cls, int T, size_t smem, int *blocks);
int beval_occupancy(int T, size_t smem, int *blocks);
int launch_beval(const DevState &ds, const EvalParams &p, int grid,
                 cudaStream_t stream, std::string *err);
int launch_eval(const DevState &ds, bool cls, const EvalParams &p, int grid,
                cudaStream_t stream, std::string *err);
// (1+1) EA accept chain (K9): every child's mutations, drawn on the host
struct EaParams {
    uint8_t *parent;      // [V] in: start genome, out: final genome
    double cur_fit;       // fitness of the start genome
    const int32_t *moff;  // [budget + 1] CSR offsets into mpos / mval
    const int32_t *mpos;  // mutated genome positions
    const uint8_t *mval;  // new genes
    int budget;
    double *out_fit;      // [1] final fitness
    int32_t *info;        // [4] accepted, rounds, raising child (-1), status
};

// simulated annealing (K10); all state in/out so a run can resume
struct SaParams {
    uint8_t *genes;    // [V] current genome (in/out)
    uint8_t *best;     // [V] best-ever genome (in/out)
    uint64_t *rng;     // [4] PCG64 state lo, hi, increment lo, hi (in/out)
    uint32_t *buf;     // [2] has_uint32, cached upper half (in/out)
    double *f;         // [5] cur, best, temp (in/out); stop 3: cand, u
    int32_t *istate;   // [6] step, k (in/out); stop (0 done, 2 raised, 3
                       // host decides), raised status, stop 3: pos, new
    int32_t *spos;     // [window] speculative moves
    uint8_t *snew;
    double *sfit;      // [window] speculative fitness, status
    uint8_t *sst;
    double alpha;
    int n_dev, budget, window;
    int host_exp;      // test hook: hand every Metropolis test to the host
};

int launch_sa(const DevState &ds, bool cls, const EvalParams &p, const SaParams &sa,
              cudaStream_t stream, std::string *err);
int launch_ea(const DevState &ds, bool cls, const EvalParams &p, const EaParams &ea,
              cudaStream_t stream, std::string *err);
int launch_cp(const uint8_t *blob, const DevLayout &lay, int V, int words,
              const uint64_t *masks, int64_t nsub, double *out, uint8_t *status,
              double *scratch, cudaStream_t stream, std::string *err);
int launch_modularity(const uint8_t *blob, const DevLayout &lay, int NT,
                      const int32_t *labels, int64_t P, int ncomm, double res,
                      double m, double norm, double *out, uint8_t *status,
                      cudaStream_t stream, std::string *err);
int launch_reach(const uint8_t *blob, const DevLayout &lay, int NT, int words,
                 uint64_t *desc, uint64_t *anc, cudaStream_t stream,
                 std::string *err);

}  // namespace hs
