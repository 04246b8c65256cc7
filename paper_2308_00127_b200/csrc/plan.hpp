// Plan: the immutable, flattened form of (graph, hardware, latency, L) that
// the evaluator kernels walk. Built once on the host (plan.cpp) and uploaded
// lazily, once per device, as one contiguous blob (DevPlan offsets).
#pragma once

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hetsched_b200.h"
#include "eval_common.cuh"

namespace hs {

constexpr uint8_t kNoLink = 255;   // comm class of a missing link
constexpr int kMaxRegK = 4;        // K <= 4: per-device state in registers

using hsk::DevLayout;
using hsk::EdgeRec;
using hsk::NodeRec;
static_assert(sizeof(EdgeRec) == 16, "EdgeRec layout");
static_assert(sizeof(NodeRec) == 16, "NodeRec layout");

struct DevState;
struct JitModule;

struct Plan {
    // ---- description
    int V = 0, E = 0, K = 0, L = 0, NT = 0;  // NT = n_tasks (== V)
    int n_classes = 0;                        // distinct bandwidths
    int live_slots = 0;
    bool uniform_comm = false, full_mesh = false, mem_check = true;
    bool all_batch_ok = true, latency_complete = true, nan_possible = false;
    int words = 0;

    std::vector<int32_t> order;       // position -> task index
    std::vector<int32_t> bfs;         // bfs_topological_order (task idx)
    std::vector<int32_t> dev_order;   // gene k -> device insertion index
    std::vector<std::string> task_ids;

    // ---- evaluator tables (genome order)
    std::vector<NodeRec> nodes;
    std::vector<EdgeRec> edges;
    std::vector<double> dur;          // [V*K]
    std::vector<uint8_t> dur_ok;      // [V*K]
    std::vector<double> extra;        // [V]
    std::vector<double> ctab;         // [V*n_cls] (CLASS mode), class 0 = 0.0
    std::vector<uint8_t> bclass;      // [K*K] class of (u,v); 0 same device
    std::vector<double> cap;          // [K]
    std::vector<uint8_t> okL;         // [K]
    int n_cls = 1;                    // classes incl. class 0

    // ---- critical path (bounds.py:57-72), BFS order
    std::vector<double> cp_fast;      // [V] fastest over all (dev, batch)
    std::vector<uint8_t> cp_fast_ok;  // [V]
    std::vector<int32_t> cp_pred_off; // [V+1]
    std::vector<int32_t> cp_pred_pos; // [E] pred BFS positions

    // ---- reachability (task insertion index)
    std::vector<int32_t> rc_succ_off, rc_succ, rc_pred_off, rc_pred;

    // ---- batched variants (heuristics.py:337-433): extended genomes, one
    // option (decomposition of L x distinct devices) per genome position
    bool batched = false;
    int n_opt = 0, P = 1;
    std::vector<int32_t> opt_np;    // [n_opt]
    std::vector<int32_t> opt_tab;   // [n_opt][P][4] = dev, lo, hi, size
    std::vector<double> bdur;       // [V][n_opt][P]
    std::vector<uint8_t> bdur_ok;   // [V][n_opt][P]

    DevLayout lay{};
    std::vector<uint8_t> blob;        // host image of the device blob

    // ---- lazily uploaded per-device state
    mutable std::mutex mu;
    mutable std::vector<DevState *> devs;  // index = device ordinal
    mutable std::vector<JitModule *> jits;  // index = device ordinal

    int pref_ld() const {
        // genome row stride with an odd number of 32-bit words: lane-strided
        // byte reads of the staged genomes are then bank-conflict free
        int w = (V + 3) / 4;
        if ((w & 1) == 0) ++w;
        return 4 * w;
    }
    ~Plan();
};

// Launch configuration and device copy of the blob, per (plan, device).
struct DevState {
    int device = -1;
    uint8_t *blob = nullptr;  // slot offsets pre-scaled by `lanes`
    int T = 0;                // threads per CTA == candidates per CTA tile
    int lanes = 0;
    int ld_cap = 0;           // largest genome row stride staged as-is
    int blocks_per_sm = 0, sms = 0;
    bool plan_smem = false;
    size_t smem = 0;          // dynamic shared memory per CTA
    int64_t smem_tile = 0, smem_ends = 0, smem_kstate = 0;
    int kt = 0;               // K template (2,3,4) or 0 = generic K
    bool ends_global = false; // end-time slots in global memory (L2 tier)
};

// Batched-variant options: allowed sub-batch sizes (null = L/4, L/2, 3L/4,
// L where integral, heuristics.py:337-342).
struct BatchedSpec {
    const int32_t *splits = nullptr;
    int n_splits = 0;
};

// Builds the plan; on failure returns an HS_E* code and sets *err.
int build_plan(const hs_instance_desc &d, Plan &p, std::string *err,
               const BatchedSpec *batched = nullptr);

// Device state for the current device (configures + uploads on first use).
int get_dev_state(const Plan &p, const DevState **out, std::string *err);

// Specialised module of the plan for `dev`, or null (HS_JIT=0 disables).
const JitModule *find_jit(const Plan &p, int dev);

}  // namespace hs
