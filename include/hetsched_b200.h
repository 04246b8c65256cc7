/*
 * hetsched_b200.h -- C ABI of the B200-native candidate-mapping evaluator.
 *
 * Drop-in boundary for the data-parallel hot path of the DiviML reference
 * (`hetsched`, /root/reference/pkg/src/hetsched). Every entry point takes
 * plain pointers and sizes (no torch or Python types), is thread-safe (the
 * reference's ModuleSolver may be called from a thread pool,
 * splitting.py:342-344), and runs its device work on the caller's stream.
 * Device pointers are marked d_, host pointers h_.
 *
 * Reference interface each entry point replaces:
 *   hs_plan_create  -- per-call setup inside decode(): sorted(hw.devices)
 *                      heuristics.py:132, _ListScheduler heuristics.py:46-58,
 *                      bfs_topological_order core.py:82-101, comm_time
 *                      core.py:148-155, LatencyTable.get core.py:166-170,
 *                      _mem_extra heuristics.py:60-65.
 *   hs_eval         -- fitness(genome, g, hw, table, L) heuristics.py:146-148
 *                      (decode heuristics.py:127-143) over a batch.
 *   hs_eval_host    -- same, host buffers in/out (the e2e call a binding
 *                      makes; H2D / D2H inside).
 *   hs_eval_gen     -- the candidate draws of the search loops
 *                      (heuristics.py:276-283, 322-325) fused with fitness.
 *   hs_trace        -- decode() heuristics.py:127-143 returning the per-task
 *                      start times that rebuild the Schedule.
 *   hs_cp_bound     -- critical_path_bound bounds.py:57-72, batched masks.
 *   hs_reach        -- dep_subgraph / pre_subgraph bounds.py:29-54 and
 *                      transitive_closure core.py:104-111 as bitsets.
 *   hs_best_merge   -- (no reference counterpart) lexicographic
 *                      (cost, index) merge of per-rank bests.
 *   hs_best_allreduce -- the same merge across GPUs over NCCL.
 *   hs_bridges_articulation / hs_k_edge_components -- module detection,
 *                      splitting.py:36-81, 178-219.
 *   hs_validate_schedules -- validate_schedule core.py:206-291, batched.
 */
#ifndef HETSCHED_B200_H
#define HETSCHED_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HS_ABI_VERSION 1

/* return codes */
#define HS_OK 0
#define HS_EINVAL 1   /* -> hetsched GraphError (bad description, bad gene) */
#define HS_ECYCLE 2   /* -> GraphError("cycle detected"), core.py:94-95   */
#define HS_ECUDA 3    /* -> RuntimeError                                   */
#define HS_ENOMEM 4   /* -> MemoryError                                    */
#define HS_EHOST 5    /* case left to the host restatement, which raises the
                         reference's exception (hs_plan_greedy)            */

/* per-candidate status (hs_eval*, hs_trace) */
#define HS_ST_OK 0        /* feasible: makespan finite or +inf by latency */
#define HS_ST_BATCH 1     /* unsupported full-batch size heuristics.py:96 */
#define HS_ST_MEMORY 2    /* capacity exceeded heuristics.py:98-100       */
#define HS_ST_LINK 3      /* missing link core.py:153-154                 */
#define HS_ST_MISSING 4   /* missing latency entry: GraphError core.py:169 */
#define HS_ST_GENE 5      /* gene out of range: GraphError heuristics.py:133 */

typedef struct hs_plan hs_plan; /* opaque, immutable after creation */

/* Instance description, reference wire model (core.py:25-179). Strings are
 * UTF-8 bytes concatenated with [n+1] offsets; indices refer to insertion
 * order (tasks dict order, edges list order, devices dict order). */
typedef struct hs_instance_desc {
    int32_t n_tasks;
    const char *task_ids;
    const int64_t *task_id_off;   /* [n_tasks+1] */
    const double *wm, *im, *om;   /* [n_tasks] bytes */
    int32_t n_edges;
    const int32_t *edge_src;      /* [n_edges] task index */
    const int32_t *edge_dst;      /* [n_edges] task index */
    int32_t n_devices;
    const char *dev_ids;
    const int64_t *dev_id_off;    /* [n_devices+1] */
    const double *memory;         /* [n_devices] bytes */
    const int32_t *batch_off;     /* [n_devices+1] into batch_sizes */
    const int32_t *batch_sizes;   /* ascending per device */
    const double *bandwidth;      /* [n_devices^2] beta(a->b) bytes/ms; <=0 = no link */
    int32_t L;                    /* inputs per task batch (decode's L) */
    const double *latency;        /* [n_tasks x n_cols], col j = (device, batch) pairs
                                     enumerated device-major in insertion order,
                                     batch sizes ascending: table.get(task, dev, b) */
    const uint8_t *latency_ok;    /* [n_tasks x n_cols] 1 = entry present */
    const int32_t *order;         /* optional [n_tasks] genome order (task index per
                                     position); NULL = bfs_topological_order */
} hs_instance_desc;

typedef struct hs_plan_info {
    int32_t V, E, K, L;
    int32_t live_slots;           /* max live end-times per candidate */
    int32_t n_classes;            /* distinct link bandwidths (comm classes) */
    int32_t uniform_comm;         /* full mesh, one bandwidth */
    int32_t full_mesh;
    int32_t mem_check;            /* 0 = capacity provably never binds */
    int32_t all_batch_ok;         /* every device supports L */
    int32_t latency_complete;     /* every needed (task, dev, L) present */
    int32_t words;                /* ceil(n_tasks/64) for masks / bitsets */
    int32_t pref_ld;              /* genome row stride that makes the staged
                                     tile bank-conflict free (>= V) */
    int32_t specializable;        /* hs_plan_specialize can serve this plan */
    int32_t batched_options;      /* batched-variant plans: options (genes) */
    int32_t max_parts;            /* batched-variant plans: parts per task */
} hs_plan_info;

typedef struct hs_best {
    double cost;                  /* makespan (ms); +inf if none feasible */
    int64_t index;                /* global candidate index, first minimum */
} hs_best;

/* thread-local message of the last failure in this thread */
const char *hs_last_error(void);
int hs_abi_version(void);
/* Per-call scratch (speculation buffers, host-pipeline chunks, reductions)
 * comes from a library-owned stream-ordered pool per device that keeps its
 * high-water mark between calls; this returns that memory to the driver
 * (all devices). Call with no library work in flight. */
int hs_scratch_trim(void);

int hs_plan_create(const hs_instance_desc *desc, hs_plan **out);
void hs_plan_destroy(hs_plan *plan);
/* Batched-variant plan (heuristics.py:337-433, bMET / bGreedy placement):
 * the genome holds one OPTION index per position, an option being a
 * decomposition of the L inputs into allowed sub-batch sizes (`splits`, or
 * L/4, L/2, 3L/4, L where integral) on distinct devices, enumerated in
 * batched_variant's order. hs_eval* / hs_trace then evaluate extended
 * genomes (hs_trace writes starts [n x V x max_parts]). */
int hs_plan_create_batched(const hs_instance_desc *desc, const int32_t *splits,
                           int32_t n_splits, hs_plan **out);
/* Option table: [n_opt][max_parts][4] = sorted-device index, first input,
 * last input (1-based), size; unused parts are -1. */
int hs_plan_batched_options(const hs_plan *plan, int32_t *n_opt,
                            int32_t *max_parts, int32_t *table);
int hs_plan_get_info(const hs_plan *plan, hs_plan_info *info);

/* greedy (heuristics.py:192-210, replaces _ListScheduler-driven greedy for
 * SA's start): BFS order, each task on the sorted-order device whose
 * placement grows the partial makespan least (by more than 1e-12), with
 * try_place's checks (heuristics.py:86-124). Host only, no CUDA. genes[V]
 * = sorted-device index per BFS position, starts[V] (may be NULL),
 * *makespan. HS_EHOST when the cost model can produce NaN, a reached
 * latency entry is missing or a task has no feasible device: the caller's
 * host scheduler then raises the reference's exception. */
int hs_plan_greedy(const hs_plan *plan, uint8_t *genes, double *starts,
                   double *makespan);
/* Specialise the evaluator to this plan on the current device: the plan is
 * emitted as straight-line CUDA (predecessor slots, communication and
 * latency constants baked in) and compiled by NVRTC for sm_100a (one-time
 * cost, reported in *compile_ms); later hs_eval* calls on this device use
 * it. HS_EINVAL when the plan is outside the specialised scope (batched
 * plans, K > 64, V > 1100, E > 2600, or a NaN in the cost model); the
 * ahead-of-time kernel then keeps serving the plan. */
int hs_plan_specialize(const hs_plan *plan, double *compile_ms);
/* The CUDA source the specialiser would compile for `lanes` lanes. */
int hs_plan_emit_specialized(const hs_plan *plan, int32_t lanes, char *buf,
                             int64_t cap, int64_t *len);
/* genome order (task index per position) and sorted device order */
int hs_plan_order(const hs_plan *plan, int32_t *order, int32_t *dev_order);

/* Batch fitness. d_genes: uint8 [n x ld] row-major, gene = sorted-device
 * index per genome position. Outputs (each may be NULL): d_makespan f64[n]
 * (+inf when infeasible, NaN on status >= 4), d_status u8[n], d_best =
 * first-index argmin with indices offset by index_base. */
int hs_eval(const hs_plan *plan, const uint8_t *d_genes, int64_t n, int64_t ld,
            double *d_makespan, uint8_t *d_status, hs_best *d_best,
            int64_t index_base, void *stream);

/* Same with host buffers; h_genes should be pinned for full PCIe rate.
 * Copies are chunked and overlapped with the kernels on `stream`; returns
 * after the results are in host memory. When K <= 4 and the host has >= 8
 * hardware threads (HS_HOST_PACK=0 / 1 overrides), a pool of host threads
 * packs the rows to 2 bits per gene into pinned staging while the GPU works
 * on the previous chunk, so PCIe carries a quarter of the bytes; a chunk
 * holding a gene >= K is sent unpacked (same statuses as hs_eval). */
int hs_eval_host(const hs_plan *plan, const uint8_t *h_genes, int64_t n,
                 int64_t ld, double *h_makespan, uint8_t *h_status,
                 hs_best *h_best, int64_t index_base, void *stream);
/* 1 when hs_eval_host packs n rows on the host (the rule above), else 0;
 * negative HS_E* on a bad plan. */
int hs_eval_host_packs(const hs_plan *plan, int64_t n);

/* Host-only: the packer hs_eval_host runs on its thread pool, for callers
 * that keep genomes packed (hs_eval_packed / hs_eval_host_packed input).
 * n rows of V uint8 genes (row stride ld) -> n rows of pld bytes, gene i in
 * bits 2*(i%4) of byte i/4, bytes past ceil(V/4) zero. *all_ok = 0 when
 * some gene is >= K (those bytes are then unspecified). No CUDA calls.
 * Replaces nothing in the reference (its genomes are Python lists,
 * heuristics.py:24-40); see heuristics.pack_genes. */
int hs_pack_genes2(const uint8_t *h_genes, int64_t n, int64_t ld, int32_t V,
                   int32_t K, uint8_t *h_packed, int64_t pld, int32_t *all_ok);

/* 2-bit packed genomes (K <= 4, or <= 4 batched options): gene i of a row
 * is bits 2*(i%4)..2*(i%4)+1 of byte i/4; rows of `ld` bytes with ld % 4
 * == 0 and ceil(V/4) <= ld <= pref_ld. A quarter of the bytes of hs_eval's
 * input (the host path is PCIe-bound); expanded in shared memory. */
int hs_eval_packed(const hs_plan *plan, const uint8_t *d_packed, int64_t n,
                   int64_t ld, double *d_makespan, uint8_t *d_status,
                   hs_best *d_best, int64_t index_base, void *stream);
int hs_eval_host_packed(const hs_plan *plan, const uint8_t *h_packed, int64_t n,
                        int64_t ld, double *h_makespan, uint8_t *h_status,
                        hs_best *h_best, int64_t index_base, void *stream);

/* Base-3 packed genomes (K <= 3, or <= 3 batched options): gene i of a row
 * is base-3 digit i%5 (least significant first) of byte i/5, i.e. byte j =
 * sum_d gene[5j+d] * 3^d; rows of `ld` bytes with ceil(V/5) <= ld <=
 * pref_ld. 1.6 bits per gene (WS200: 41 B per candidate instead of 52 B
 * 2-bit or 204 B u8) for the PCIe-bound host path; expanded in shared
 * memory. A byte >= 243 decodes to an out-of-range gene (status 4). */
int hs_eval_packed3(const hs_plan *plan, const uint8_t *d_packed, int64_t n,
                    int64_t ld, double *d_makespan, uint8_t *d_status,
                    hs_best *d_best, int64_t index_base, void *stream);
int hs_eval_host_packed3(const hs_plan *plan, const uint8_t *h_packed, int64_t n,
                         int64_t ld, double *h_makespan, uint8_t *h_status,
                         hs_best *h_best, int64_t index_base, void *stream);

/* The whole (1+1) EA accept chain in one launch (replaces the loop of
 * heuristics.py:302-334 around fitness). Child c (0 <= c < budget) is the
 * current parent with genes d_mpos[q] := d_mval[q] for q in
 * [d_moff[c], d_moff[c+1]) -- the mutation stream does not depend on
 * fitness, so the caller draws it up front; a child is accepted when its
 * fitness <= the current one (:328). d_parent [V] holds the start genome
 * (fitness cur_fit) and receives the final one; d_fit[0] = final fitness;
 * d_info = {accepted, rounds, first child whose evaluation raised (-1 if
 * none; the chain stops there as the reference's does), its status}. */
int hs_ea_run(const hs_plan *plan, uint8_t *d_parent, double cur_fit,
              const int32_t *d_moff, const int32_t *d_mpos, const uint8_t *d_mval,
              int32_t budget, double *d_fit, int32_t *d_info, void *stream);

/* The same accept chain in chained chunks, so the caller can draw the next
 * chunk's mutations while this one runs: children first_child ..
 * first_child + n_children - 1 with CSR lists relative to the chunk; the
 * current fitness is read from and written back to d_fit[0]; d_info
 * accumulates (the caller sets it to {0, 0, -1, 0} once) and a chunk does
 * nothing when an earlier one raised (d_info[2] >= 0, absolute child). */
int hs_ea_run_chunk(const hs_plan *plan, uint8_t *d_parent, double *d_fit,
                    const int32_t *d_moff, const int32_t *d_mpos, const uint8_t *d_mval,
                    int32_t n_children, int32_t first_child, int32_t *d_info,
                    void *stream);

/* The EA's mutation stream on the device (K12), for `chains` independent
 * numpy PCG64 generators: chain c starts at d_rng + 4c = {state lo, state
 * hi, inc lo, inc hi} with d_buf + 2c = {has_uint32, uinteger} and draws,
 * for each of `budget` children and each of n_tasks positions, random() <
 * p and on a hit integers(n_dev) (heuristics.py:318-325). Output as CSR
 * for hs_ea_run_multi: d_moff + c * (budget + 1) (absolute offsets), the
 * mutated positions / values at d_mpos / d_mval + c * cap_per_chain.
 * d_status[c] = 0 ok, 1 more than cap_per_chain mutations, 2 Lemire's
 * rejection branch was reached (probability < n_dev / 2^32): the caller
 * redraws such a chain on the host. The generators are not advanced. */
int hs_ea_draw(int32_t chains, const uint64_t *d_rng, const uint32_t *d_buf,
               int32_t n_tasks, int32_t n_dev, double p, int32_t budget,
               int32_t *d_moff, int32_t *d_mpos, uint8_t *d_mval,
               int64_t cap_per_chain, int32_t *d_status, void *stream);

/* Simulated annealing (heuristics.py:259-299) in one launch, resumable.
 * All state lives in device buffers (in/out): d_genes [V] current genome,
 * d_best [V] best-ever genome, d_rng = numpy PCG64 {state lo, state hi,
 * inc lo, inc hi}, d_buf = {has_uint32, uinteger}, d_f = {cur_fit,
 * best_fit, temp, -, -}, d_istate = {step, k (speculation window, start
 * 8), stop, status, pos, new, rounds (accumulated)}. Runs steps until `budget`; stop = 0 done,
 * 2 a fitness evaluation raised (status = its code; GraphError), 3 the
 * Metropolis test at this step is within a few ulp of the device exp():
 * the caller decides it with the host exp (u = d_f[4], candidate fitness
 * d_f[3], move pos/new), applies it and calls again. */
int hs_sa_run(const hs_plan *plan, uint8_t *d_genes, uint8_t *d_best, uint64_t *d_rng,
              uint32_t *d_buf, double *d_f, int32_t *d_istate, double alpha,
              int32_t n_dev, int32_t budget, int32_t window, void *stream);

/* Independent annealing chains in one launch, one CTA (one SM) each -- e.g.
 * the reference's simulated_annealing at `chains` seeds at once. Chain c's
 * state sits at d_genes / d_best + c * chain_stride (chain_stride >= V),
 * d_rng + 4c, d_buf + 2c, d_f + 8c, d_istate + 8c, each laid out as in
 * hs_sa_run; every chain follows its own seed's reference trajectory. */
int hs_sa_run_multi(const hs_plan *plan, int32_t chains, int64_t chain_stride,
                    uint8_t *d_genes, uint8_t *d_best, uint64_t *d_rng, uint32_t *d_buf,
                    double *d_f, int32_t *d_istate, double alpha, int32_t n_dev,
                    int32_t budget, int32_t window, void *stream);

/* Independent (1+1) EA accept chains in one launch, one CTA each: chain c's
 * parent at d_parent + c * chain_stride with fitness d_cur_fit[c], its
 * mutation lists as CSR with offsets d_moff + c * (budget + 1) (absolute
 * indices into d_mpos / d_mval), result d_fit[c] and d_info + 4c as in
 * hs_ea_run. */
int hs_ea_run_multi(const hs_plan *plan, int32_t chains, int64_t chain_stride,
                    uint8_t *d_parent, const double *d_cur_fit, const int32_t *d_moff,
                    const int32_t *d_mpos, const uint8_t *d_mval, int32_t budget,
                    double *d_fit, int32_t *d_info, void *stream);

/* On-device candidates: candidate c in [first, first+n) has genes
 * oracle/hs_oracle.py::gen_genes(seed, c). Optional d_genes_out [n x V]. */
int hs_eval_gen(const hs_plan *plan, uint64_t seed, int64_t first, int64_t n,
                double *d_makespan, uint8_t *d_status, uint8_t *d_genes_out,
                hs_best *d_best, void *stream);

/* Generated candidates over genome groups. Position i takes the fixed gene
 * d_template[i] when d_group[i] < 0, else the value of group d_group[i]
 * (groups numbered by first position, so d_group[i] <= i); NULL template and
 * group map = one group per position. HS_GEN_RANDOM: group values of
 * candidate c are gen_genes(seed, c) over n_groups; HS_GEN_ENUM: group j is
 * digit j of c in base K (requires first + n <= K^n_groups). Used for the
 * pinned / co-located module sweeps of the split heuristic's ModuleSolver
 * (splitting.py:225-245, pins and same_device of milp.py:277-291). */
#define HS_GEN_RANDOM 1
#define HS_GEN_ENUM 2
/* HS_GEN_NEIGHBOR: the one- and two-group moves of the incumbent genome
 * d_template (every position's gene): index c < n_groups*K sets group c/K
 * to c%K; index n_groups*K + ((j*n_groups + l)*K + a)*K + b sets group j
 * to a and, when l > j, group l to b (the module solver's local search). */
#define HS_GEN_NEIGHBOR 3
int hs_eval_gen_ex(const hs_plan *plan, int mode, uint64_t seed, int64_t first,
                   int64_t n, const uint8_t *d_template, const int16_t *d_group,
                   int32_t n_groups, double *d_makespan, uint8_t *d_status,
                   uint8_t *d_genes_out, hs_best *d_best, void *stream);

/* decode(): per-position start times d_start f64[n x V] (row per genome). */
int hs_trace(const hs_plan *plan, const uint8_t *d_genes, int64_t n, int64_t ld,
             double *d_start, double *d_makespan, uint8_t *d_status,
             void *stream);

/* critical_path_bound over nsub task masks (bit t = task insertion index t,
 * words = ceil(n_tasks/64) per mask). d_status[k] = 1 when a task of the
 * mask lacks a latency entry (GraphError). */
int hs_cp_bound(const hs_plan *plan, const uint64_t *d_masks, int64_t nsub,
                double *d_out, uint8_t *d_status, void *stream);

/* Descendant / ancestor bitsets [n_tasks x words] (task insertion index). */
int hs_reach(const hs_plan *plan, uint64_t *d_desc, uint64_t *d_anc,
             void *stream);

/* Newman modularity (resolution gamma) of P partitions of the graph's
 * undirected shadow: d_labels int32 [P x n_tasks] community index per task
 * (insertion order), communities 0..n_comm-1 summed in index order, same
 * binary64 sequence as networkx.community.modularity. The split
 * heuristic's module partition (splitting.py:178-219) is one such
 * partition; the reference itself computes no score.
 * d_status[k] = 1 when a label is out of range. */
int hs_modularity(const hs_plan *plan, const int32_t *d_labels, int64_t P,
                  int32_t n_comm, double resolution, double *d_out,
                  uint8_t *d_status, void *stream);

/* host: lexicographic (cost, index) minimum of n bests */
int hs_best_merge(const hs_best *bests, int64_t n, hs_best *out);

/* Module detection of the split heuristic (host, one-time per graph; no
 * device work). Graph = n_tasks tasks (insertion order) and n_edges directed
 * edges; both work on the undirected shadow (splitting.py:28-33).
 *
 * hs_bridges_articulation -- find_bridges_and_articulation_points
 *   (splitting.py:36-81): is_bridge[e] = 1 when edge e (either orientation)
 *   is a bridge, is_articulation[v] = 1 for cut vertices, *connected = 1
 *   when the shadow is connected. Any output may be NULL.
 * hs_k_edge_components -- k_edge_components(g, c) (splitting.py:178-219)
 *   with k = c + 1: module_of[v] = the module index of task v, modules being
 *   the k-edge-connected components of the shadow (networkx semantics:
 *   maximal sets with pairwise edge connectivity >= k), cycles of the module
 *   digraph merged, numbered by the lexicographic topological order keyed
 *   by each module's smallest task id (UTF-8 bytes, = Python str order). */
int hs_bridges_articulation(int32_t n_tasks, int32_t n_edges, const int32_t *edge_src,
                            const int32_t *edge_dst, uint8_t *is_bridge,
                            uint8_t *is_articulation, int32_t *connected);
int hs_k_edge_components(int32_t n_tasks, const char *task_ids,
                         const int64_t *task_id_off, int32_t n_edges,
                         const int32_t *edge_src, const int32_t *edge_dst, int32_t k,
                         int32_t *module_of, int32_t *n_modules);

/* Schedule validation on the GPU (K11): validate_schedule core.py:206-291
 * for n_sched schedules in one call (one CTA each). The instance is a
 * description as for hs_plan_create (L and order are ignored; latency holds
 * every (device, batch size) column). Schedule q owns batches
 * [h_batch_off[q], h_batch_off[q+1]) in its own order, input values
 * h_inputs[in_off .. in_off + n_inputs), input_count h_input_count[q] and
 * stated objective h_objective[q]. h_out[q] receives the FIRST violation in
 * the reference's check order (code 0 = valid, v0 = makespan), with the
 * indices / values its message needs; all buffers are host memory. */
typedef struct hs_sched_batch {
    int32_t task;       /* task insertion index, -1 = not in the graph    */
    int32_t device;     /* device insertion index, -1 = unknown device    */
    int32_t size;       /* b.size (-1 if outside int32)                   */
    int32_t n_inputs;   /* len(b.inputs)                                  */
    int64_t in_off;     /* first input value in h_inputs                  */
    double start;       /* b.start                                        */
    int32_t flags;      /* bit 0: b.inputs repeats a value                */
    int32_t pad;
} hs_sched_batch;

typedef struct hs_violation {
    int32_t code;       /* HS_V_*                                          */
    int32_t a, b, c;    /* batch / task / edge / device indices, see codes */
    double v0, v1, v2;  /* values of the message (v0 = makespan if valid)  */
} hs_violation;

#define HS_V_OK 0
#define HS_V_UNKNOWN_TASK 1    /* a = batch                                 */
#define HS_V_UNKNOWN_DEVICE 2  /* a = batch                                 */
#define HS_V_SIZE 3            /* a = batch: size vs inputs                 */
#define HS_V_BATCH_SIZE 4      /* a = batch: size not supported by device   */
#define HS_V_NEGATIVE_START 5  /* a = batch                                 */
#define HS_V_INPUT_RANGE 6     /* a = batch, c = position in its inputs     */
#define HS_V_DOUBLE 7          /* a = batch, c = position: assigned twice   */
#define HS_V_LATENCY 8         /* a = batch: missing entry (GraphError)     */
#define HS_V_UNASSIGNED 9      /* a = task, c = input (1-based)             */
#define HS_V_NO_LINK 10        /* a = edge, b = producer batch, c = input   */
#define HS_V_PRECEDENCE 11     /* a = edge, b = producer batch, c = input;
                                  v0 = consumer start, v1 = producer end,
                                  v2 = comm                                 */
#define HS_V_OVERLAP 12        /* a, b = batches (sorted order), c = device;
                                  v0, v1 = their ends                       */
#define HS_V_MEMORY 13         /* a = device, v0 = used, v1 = memory        */
#define HS_V_OBJECTIVE 14      /* v0 = makespan, v1 = stated objective      */

int hs_validate_schedules(const hs_instance_desc *desc, int64_t n_sched,
                          const int64_t *h_batch_off, const hs_sched_batch *h_batches,
                          const int64_t *h_inputs, const int32_t *h_input_count,
                          const double *h_objective, double tol, hs_violation *h_out,
                          void *stream);

/* Multi-GPU: the global best over every rank of an NCCL communicator. Each
 * rank passes its device-resident local best (hs_eval's d_best, indices
 * already global through index_base); d_out (device) receives the
 * lexicographic (cost, index) minimum on every rank. One ncclAllGather of
 * 16 B per rank on `stream` plus a one-thread merge kernel (NCCL has no
 * argmin operator). NCCL is bound at run time
 * (dlopen("libnccl.so.2")), so `comm` must come from the NCCL already loaded
 * in the process (e.g. torch's ProcessGroupNCCL._comm_ptr()). No reference
 * counterpart: the reference runs on one host and never reduces. */
struct ncclComm;
int hs_best_allreduce(const hs_best *d_in, hs_best *d_out, struct ncclComm *comm,
                      void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HETSCHED_B200_H */
