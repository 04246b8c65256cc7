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
using hsk::EaParams;
using hsk::SaParams;

int eval_occupancy(int kt, bool cls, int T, size_t smem, int *blocks);
int beval_occupancy(int T, size_t smem, int *blocks);
int launch_beval(const DevState &ds, const EvalParams &p, int grid,
                 cudaStream_t stream, std::string *err);
int launch_eval(const DevState &ds, bool cls, const EvalParams &p, int grid,
                cudaStream_t stream, std::string *err);
// grid = number of independent chains (one CTA each)
int launch_sa(const DevState &ds, bool cls, const EvalParams &p, const SaParams &sa,
              cudaStream_t stream, std::string *err, int grid = 1);
int launch_ea(const DevState &ds, bool cls, const EvalParams &p, const EaParams &ea,
              cudaStream_t stream, std::string *err, int grid = 1);
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
