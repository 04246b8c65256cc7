// Ahead-of-time sm_100a kernels of the candidate-mapping evaluator.
//
//  K1 eval_kernel   batched list-scheduling makespan, one lane per candidate
//                   (decode/fitness, heuristics.py:43-148), walking the plan's
//                   node/edge records; genomes staged HBM -> shared memory by
//                   a TMA bulk copy per CTA tile; fused first-index argmin
//                   (K2), on-device candidate generation (K6) and start-time
//                   trace (K3) come from the shared tile driver
//                   (eval_common.cuh). jit.cpp emits the same computation as
//                   straight-line code specialised to one graph.
//  K4 cp_kernel     critical_path_bound over task masks (bounds.py:57-72).
//  K5 reach_kernel  descendant / ancestor bitsets (bounds.py:29-54,
//                   core.py:104-111).
//
// Exactness: every floating-point operation is the reference's binary64
// operation in the reference's order -- additions `end + comm`, `start +
// dur`, `mem + extra`, and Python's max(a, b) written as `b > a ? b : a`
// (DSETP + SEL, which also reproduces Python's NaN behaviour). There are no
// multiplications on the path, and the file is compiled with --fmad=false.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "kernels.cuh"

namespace hs {

using namespace hsk;

namespace {

// ---- per-device state of one candidate: registers for K <= 4
template <int KT>
struct DevRegs {
    double v[KT];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int k = 0; k < KT; ++k) v[k] = 0.0;
    }
    __device__ __forceinline__ double get(int d) const {
        double x = v[0];
#pragma unroll
        for (int k = 1; k < KT; ++k) x = (d == k) ? v[k] : x;
        return x;
    }
    __device__ __forceinline__ void set(int d, double x) {
#pragma unroll
        for (int k = 0; k < KT; ++k) v[k] = (d == k) ? x : v[k];
    }
};

// generic K: [K][lanes] column in shared memory
struct DevSmem {
    double *col;  // &base[lane]
    int stride;   // lanes
    int K;
    __device__ __forceinline__ void zero() {
        for (int k = 0; k < K; ++k) col[k * stride] = 0.0;
    }
    __device__ __forceinline__ double get(int d) const { return col[d * stride]; }
    __device__ __forceinline__ void set(int d, double x) { col[d * stride] = x; }
};

template <int KT>
struct DevStateSel {
    using type = DevRegs<KT>;
};
template <>
struct DevStateSel<0> {
    using type = DevSmem;
};

// The data-driven list scheduler of one candidate (heuristics.py:127-143).
// FAST: no capacity / batch-size / missing-entry checks and no NaN can
// occur (plan flags all clear), so those branches are compiled out.
template <int KT, bool CLASS, bool FAST>
struct PlanBody {
    const NodeRec *nodes;
    const EdgeRec *edges;
    const double *dur;
    const hs_u8 *dur_ok;
    const double *extra;
    const double *ctab;
    const hs_u16 *bclass;
    const double *cap;
    const hs_u8 *okL;
    double *ends;
    double *kstate;
    double *starts;
    int lanes, V, K;
    hs_u32 flags;

    __device__ __forceinline__ void run(const hs_u8 *grow, int li, hs_i64 cand,
                                        bool valid, int, double &ms_out, int &st_out) {
        double *ecol = ends + li;
        typename DevStateSel<KT>::type avail, mem;
        if constexpr (KT == 0) {
            avail.col = kstate + li;
            avail.stride = lanes;
            avail.K = K;
            mem.col = kstate + (hs_i64)K * lanes + li;
            mem.stride = lanes;
            mem.K = K;
        }
        const hs_u32 fl = FAST ? 0u : flags;
        avail.zero();
        if (fl & F_MEM) mem.zero();
        double ms = 0.0;
        int st = 0, bad = 0;
        for (int i = 0; i < V; ++i) {
            const NodeRec nr = nodes[i];
            int d = grow[i];
            bad |= d >= K;
            d = d < K ? d : 0;
            if (fl & F_OKL) {  // try_place batch-size check, :96
                if (!okL[d] && !st) st = ST_BATCH;
            }
            double mcur = 0.0;
            if (fl & F_MEM) {  // memory check, :98-100
                mcur = mem.get(d);
                if (mcur + extra[i] > cap[d] && !st) st = ST_MEMORY;
            }
            // ready_time, :67-78 (the L inputs repeat the same value)
            double r = 0.0;
            int nolink = 0;
#pragma unroll 2
            for (int e = nr.e_begin; e < nr.e_end; ++e) {
                const EdgeRec er = edges[e];
                const int gp = grow[er.gpos];
                const double ep = ecol[er.slot];
                double x;
                if constexpr (!CLASS) {
                    x = ep + (gp == d ? 0.0 : er.c);
                } else {
                    const int g2 = gp < K ? gp : 0;
                    int cls = bclass[g2 * K + d];
                    if (cls == 0xFFFF) {
                        nolink = 1;
                        cls = 0;
                    }
                    x = ep + ctab[er.crow + cls];
                }
                r = pymax(r, x);
            }
            if (CLASS && nolink && !st) st = ST_LINK;
            const double du = dur[i * K + d];
            if (fl & F_MISS) {  // LatencyTable.get raises, core.py:169
                if (!dur_ok[i * K + d] && !st) st = ST_MISSING;
            }
            const double s = pymax(r, avail.get(d));  // _slot, :80-84
            const double e = s + du;
            if (starts && valid) starts[cand * V + i] = s;
            if (nr.out_slot >= 0) ecol[nr.out_slot] = e;
            avail.set(d, e);
            if (fl & F_MEM) mem.set(d, mcur + extra[i]);
            if (fl & F_NAN) ms = pymax(ms, e);
        }
        if (!(fl & F_NAN)) {
            // ends per device never decrease without NaN: the makespan is
            // the largest device-available time
            for (int k = 0; k < K; ++k) ms = pymax(ms, avail.get(k));
        }
        if (bad) st = ST_GENE;
        if (st) ms = st >= ST_MISSING ? knan() : kinf();
        ms_out = ms;
        st_out = st;
    }
};

// Batched-variant extended genome (heuristics.py:363-433, non-insertion):
// gene = option (decomposition of L x distinct devices); per part, ready
// time over the predecessors' parts holding the part's inputs, start at
// max(ready, last end on the device). Like batched_variant, no memory or
// batch-size check (options are pre-filtered to supported sizes).
struct BatchedBody {
    const NodeRec *nodes;
    const EdgeRec *edges;
    const int *bopt;     // [n_opt][P][4] = dev, lo, hi, size
    const int *bnp;      // [n_opt]
    const double *bdur;  // [V][n_opt][P]
    const hs_u8 *bdur_ok;
    const double *ctab;
    const hs_u16 *bclass;
    double *ends;        // [slot * P + part][lanes]
    double *kstate;      // [K][lanes] device-available times
    double *starts;      // [n][V][P]
    int lanes, V, K, n_opt, P, ncls;
    bool nan;

    // P <= PM parts per option (PM = 2 or 4; every L <= 8 with the default
    // sub-batch sizes): each predecessor's option and parts are loaded once per edge
    // and every own part is relaxed from them (per-part maxima in
    // registers, the same order of max operations per part as below)
    template <int PM>
    __device__ __forceinline__ void runp(const hs_u8 *grow, int li, hs_i64 cand,
                                         bool valid, double &ms_out, int &st_out) {
        double *ecol = ends + li;
        double *av = kstate + li;
        for (int k = 0; k < K; ++k) av[k * lanes] = 0.0;
        double ms = 0.0;
        int st = 0, bad = 0;
        for (int i = 0; i < V; ++i) {
            const NodeRec nr = nodes[i];
            int o = grow[i];
            bad |= o >= n_opt;
            o = o < n_opt ? o : 0;
            const int np = bnp[o];
            int dk[PM], lok[PM], hik[PM], nl[PM];
            double r[PM];
#pragma unroll
            for (int k = 0; k < PM; ++k) {
                const int *q = bopt + (o * P + (k < np ? k : 0)) * 4;
                dk[k] = q[0];
                lok[k] = q[1];
                hik[k] = q[2];
                r[k] = 0.0;
                nl[k] = 0;
            }
            for (int e = nr.e_begin; e < nr.e_end; ++e) {
                const EdgeRec er = edges[e];
                int op = grow[er.gpos];
                op = op < n_opt ? op : 0;
                const int npp = bnp[op];
                for (int m = 0; m < npp; ++m) {
                    const int *qq = bopt + (op * P + m) * 4;
                    const int dm = qq[0], lom = qq[1], him = qq[2];
                    const double em = ecol[(er.slot * P + m) * lanes];
#pragma unroll
                    for (int k = 0; k < PM; ++k) {
                        if (k >= np || him < lok[k] || lom > hik[k]) continue;
                        int cls = bclass[dm * K + dk[k]];
                        if (cls == 0xFFFF) {
                            nl[k] = 1;
                            cls = 0;
                        }
                        r[k] = pymax(r[k], em + ctab[er.crow + cls]);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < PM; ++k) {
                if (k >= np) continue;
                const int d = dk[k];
                if (nl[k] && !st) st = ST_LINK;
                const hs_i64 at = ((hs_i64)i * n_opt + o) * P + k;
                if (!bdur_ok[at] && !st) st = ST_MISSING;
                const double s = pymax(r[k], av[d * lanes]);
                const double e = s + bdur[at];
                if (starts && valid) starts[(cand * V + i) * P + k] = s;
                if (nr.out_slot >= 0) ecol[(nr.out_slot * P + k) * lanes] = e;
                av[d * lanes] = e;
                ms = pymax(ms, e);
            }
        }
        if (bad) st = ST_GENE;
        if (st) ms = st >= ST_MISSING ? knan() : kinf();
        ms_out = ms;
        st_out = st;
    }

    __device__ __forceinline__ void run(const hs_u8 *grow, int li, hs_i64 cand,
                                        bool valid, int, double &ms_out, int &st_out) {
        if (P <= 2) {
            runp<2>(grow, li, cand, valid, ms_out, st_out);
            return;
        }
        if (P <= 4) {
            runp<4>(grow, li, cand, valid, ms_out, st_out);
            return;
        }
        double *ecol = ends + li;
        double *av = kstate + li;
        for (int k = 0; k < K; ++k) av[k * lanes] = 0.0;
        double ms = 0.0;
        int st = 0, bad = 0;
        for (int i = 0; i < V; ++i) {
            const NodeRec nr = nodes[i];
            int o = grow[i];
            bad |= o >= n_opt;
            o = o < n_opt ? o : 0;
            const int np = bnp[o];
            for (int k = 0; k < np; ++k) {
                const int *q = bopt + (o * P + k) * 4;
                const int d = q[0], lo = q[1], hi = q[2];
                double r = 0.0;
                int nolink = 0;
                for (int e = nr.e_begin; e < nr.e_end; ++e) {
                    const EdgeRec er = edges[e];
                    int op = grow[er.gpos];
                    op = op < n_opt ? op : 0;
                    const int npp = bnp[op];
                    // the predecessor's parts holding inputs lo..hi, in
                    // input order (Python iterates l = lo..hi)
                    for (int m = 0; m < npp; ++m) {
                        const int *qq = bopt + (op * P + m) * 4;
                        if (qq[2] < lo || qq[1] > hi) continue;
                        int cls = bclass[qq[0] * K + d];
                        if (cls == 0xFFFF) {
                            nolink = 1;
                            cls = 0;
                        }
                        const double x = ecol[(er.slot * P + m) * lanes] + ctab[er.crow + cls];
                        r = pymax(r, x);
                    }
                }
                if (nolink && !st) st = ST_LINK;
                const hs_i64 at = ((hs_i64)i * n_opt + o) * P + k;
                if (!bdur_ok[at] && !st) st = ST_MISSING;
                const double s = pymax(r, av[d * lanes]);
                const double e = s + bdur[at];
                if (starts && valid) starts[(cand * V + i) * P + k] = s;
                if (nr.out_slot >= 0) ecol[(nr.out_slot * P + k) * lanes] = e;
                av[d * lanes] = e;
                ms = pymax(ms, e);
            }
        }
        if (bad) st = ST_GENE;
        if (st) ms = st >= ST_MISSING ? knan() : kinf();
        ms_out = ms;
        st_out = st;
    }
};

}  // namespace

// Batched-variant evaluator (one lane per extended genome).
__global__ void __launch_bounds__(512) beval_kernel(const EvalParams a) {
    extern __shared__ __align__(16) hs_u8 smem[];
    const hs_u8 *plan = a.blob;
    if (a.plan_smem) {
        hs_u8 *sp = smem + 16;
        const uint4 *src = reinterpret_cast<const uint4 *>(a.blob);
        uint4 *dst = reinterpret_cast<uint4 *>(sp);
        for (hs_i64 q = threadIdx.x; q < a.eval_bytes / 16; q += blockDim.x)
            dst[q] = src[q];
        plan = sp;
    }
    BatchedBody body;
    body.nodes = reinterpret_cast<const NodeRec *>(plan + a.lay.node);
    body.edges = reinterpret_cast<const EdgeRec *>(plan + a.lay.edge);
    body.bopt = reinterpret_cast<const int *>(plan + a.lay.bopt);
    body.bnp = reinterpret_cast<const int *>(plan + a.lay.bnp);
    body.bdur = reinterpret_cast<const double *>(plan + a.lay.bdur);
    body.bdur_ok = plan + a.lay.bdur_ok;
    body.ctab = reinterpret_cast<const double *>(plan + a.lay.ctab);
    body.bclass = reinterpret_cast<const hs_u16 *>(plan + a.lay.bclass);
    body.ends = a.ends_g ? a.ends_g + blockIdx.x * a.ends_g_cta
                         : reinterpret_cast<double *>(smem + a.smem_ends);
    body.kstate = reinterpret_cast<double *>(smem + a.smem_kstate);
    body.starts = a.starts;
    body.lanes = a.lanes;
    body.V = a.V;
    body.K = a.K;
    body.n_opt = a.n_opt;
    body.P = a.P;
    body.ncls = a.n_cls;
    body.nan = (a.flags & F_NAN) != 0;
    eval_tiles(a, smem, body);
}

// K1: one lane per candidate; every lane walks the same record sequence
// (broadcast reads), only gene-indexed lookups diverge.
template <int KT, bool CLASS, bool FAST>
__global__ void __launch_bounds__(512) eval_kernel(const EvalParams a) {
    extern __shared__ __align__(16) hs_u8 smem[];
    const hs_u8 *plan = a.blob;
    if (a.plan_smem) {
        hs_u8 *sp = smem + 16;
        const uint4 *src = reinterpret_cast<const uint4 *>(a.blob);
        uint4 *dst = reinterpret_cast<uint4 *>(sp);
        for (hs_i64 q = threadIdx.x; q < a.eval_bytes / 16; q += blockDim.x)
            dst[q] = src[q];
        plan = sp;
    }
    PlanBody<KT, CLASS, FAST> body;
    body.nodes = reinterpret_cast<const NodeRec *>(plan + a.lay.node);
    body.edges = reinterpret_cast<const EdgeRec *>(plan + a.lay.edge);
    body.dur = reinterpret_cast<const double *>(plan + a.lay.dur);
    body.dur_ok = plan + a.lay.dur_ok;
    body.extra = reinterpret_cast<const double *>(plan + a.lay.extra);
    body.ctab = reinterpret_cast<const double *>(plan + a.lay.ctab);
    body.bclass = reinterpret_cast<const hs_u16 *>(plan + a.lay.bclass);
    body.cap = reinterpret_cast<const double *>(plan + a.lay.cap);
    body.okL = plan + a.lay.okL;
    body.ends = a.ends_g ? a.ends_g + blockIdx.x * a.ends_g_cta
                         : reinterpret_cast<double *>(smem + a.smem_ends);
    body.kstate = reinterpret_cast<double *>(smem + a.smem_kstate);
    body.starts = a.starts;
    body.lanes = a.lanes;
    body.V = a.V;
    body.K = a.K;
    body.flags = a.flags;
    eval_tiles(a, smem, body);  // __syncthreads() before first use of plan
}

// Plan tables (staged into shared memory when the layout says so) and the
// evaluator body of a single-CTA search kernel (K9 / K10).
template <class Body>
__device__ __forceinline__ void single_cta_body(const EvalParams &a, hs_u8 *smem, Body &body) {
    const hs_u8 *plan = a.blob;
    if (a.plan_smem) {
        hs_u8 *sp = smem + 16;
        const uint4 *src = reinterpret_cast<const uint4 *>(a.blob);
        uint4 *dst = reinterpret_cast<uint4 *>(sp);
        for (hs_i64 q = threadIdx.x; q < a.eval_bytes / 16; q += blockDim.x)
            dst[q] = src[q];
        plan = sp;
    }
    body.nodes = reinterpret_cast<const NodeRec *>(plan + a.lay.node);
    body.edges = reinterpret_cast<const EdgeRec *>(plan + a.lay.edge);
    body.dur = reinterpret_cast<const double *>(plan + a.lay.dur);
    body.dur_ok = plan + a.lay.dur_ok;
    body.extra = reinterpret_cast<const double *>(plan + a.lay.extra);
    body.ctab = reinterpret_cast<const double *>(plan + a.lay.ctab);
    body.bclass = reinterpret_cast<const hs_u16 *>(plan + a.lay.bclass);
    body.cap = reinterpret_cast<const double *>(plan + a.lay.cap);
    body.okL = plan + a.lay.okL;
    // one CTA per chain (hs_sa_run_multi / hs_ea_run_multi): each its own
    // region of the global slot tier
    body.ends = a.ends_g ? a.ends_g + blockIdx.x * a.ends_g_cta
                         : reinterpret_cast<double *>(smem + a.smem_ends);
    body.kstate = reinterpret_cast<double *>(smem + a.smem_kstate);
    body.starts = nullptr;
    body.lanes = a.lanes;
    body.V = a.V;
    body.K = a.K;
    body.flags = a.flags;
    __syncthreads();
}

// ---------------------------------------------------------------------------
// K10: simulated annealing (heuristics.py:259-299) in one launch. Rounds of
// speculation: thread 0 draws the next k steps' moves assuming each is
// rejected after a random() draw (a finite, worse candidate -- the only way
// a step continues a round); the lanes evaluate those k candidates against
// the current genome; thread 0 then replays the steps with the real
// generator and ends the round at the first acceptance or infinite
// candidate (where the speculated draws diverge). Metropolis needs exp():
// when u lies within a few ulp of the device exp the step is handed back to
// the host (CPython's math.exp decides; never observed in practice), so
// the trajectory is the reference's exactly.
template <int KT, bool CLASS, bool FAST>
__global__ void __launch_bounds__(512) sa_kernel(const EvalParams a, const SaParams e) {
    extern __shared__ __align__(16) hs_u8 smem[];
    PlanBody<KT, CLASS, FAST> body;
    single_cta_body(a, smem, body);
    sa_chain(a, e, smem, body);
}

// ---------------------------------------------------------------------------
// K9: the whole (1+1) EA accept chain in one launch (heuristics.py:302-334).
// The EA's mutation stream does not depend on fitness, so the host draws
// every child's mutation list up front (CSR: moff/mpos/mval). One CTA runs
// rounds: lane l evaluates child j+l = (current parent + its mutations);
// the first lane whose child is not worse (`fit <= cur`, the reference's
// acceptance, :328) -- or whose evaluation raised (status >= 4, GraphError
// in the reference) -- decides the round: its child becomes the parent and
// j moves past it; with no such lane j advances by a full round. Children
// after an acceptance are re-evaluated against the new parent in the next
// round, so the trajectory is the reference's exactly.
template <int KT, bool CLASS, bool FAST>
__global__ void __launch_bounds__(512) ea_kernel(const EvalParams a, const EaParams e) {
    extern __shared__ __align__(16) hs_u8 smem[];
    PlanBody<KT, CLASS, FAST> body;
    single_cta_body(a, smem, body);
    ea_chain(a, e, smem, body);
}

// ---------------------------------------------------------------------------
// K4: one thread per task mask; best[] scratch is [V][nsub] (coalesced).
__global__ void cp_kernel(const uint8_t *blob, DevLayout lay, int V, int words,
                          const uint64_t *masks, int64_t nsub, double *out,
                          uint8_t *status, double *scratch) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nsub) return;
    const double *fast = reinterpret_cast<const double *>(blob + lay.cp_fast);
    const uint8_t *fast_ok = blob + lay.cp_fast_ok;
    const int32_t *task = reinterpret_cast<const int32_t *>(blob + lay.cp_task);
    const int32_t *poff = reinterpret_cast<const int32_t *>(blob + lay.cp_pred_off);
    const int32_t *ppos = reinterpret_cast<const int32_t *>(blob + lay.cp_pred_pos);
    const uint64_t *m = masks + k * words;
    double res = 0.0;
    bool have = false;
    int err = 0;
    for (int i = 0; i < V; ++i) {
        const int t = task[i];
        if (!((m[t >> 6] >> (t & 63)) & 1ull)) continue;
        if (!fast_ok[i]) err = 1;
        double inc = 0.0;
        bool hi = false;
        for (int e = poff[i]; e < poff[i + 1]; ++e) {
            const int p = ppos[e];
            const int tp = task[p];
            if (!((m[tp >> 6] >> (tp & 63)) & 1ull)) continue;
            const double v = scratch[(int64_t)p * nsub + k];
            inc = hi ? pymax(inc, v) : v;
            hi = true;
        }
        const double b = fast[i] + (hi ? inc : 0.0);
        scratch[(int64_t)i * nsub + k] = b;
        res = have ? pymax(res, b) : b;
        have = true;
    }
    out[k] = have ? res : 0.0;
    if (status) status[k] = (uint8_t)err;
}

// K5: thread w owns bit-word w of every row; rows are finished in reverse
// (descendants) / forward (ancestors) topological order by the same thread,
// so no synchronisation is needed.
__global__ void reach_kernel(const uint8_t *blob, DevLayout lay, int NT, int words,
                             uint64_t *desc, uint64_t *anc) {
    const int32_t *order = reinterpret_cast<const int32_t *>(blob + lay.rc_order);
    const int32_t *so = reinterpret_cast<const int32_t *>(blob + lay.rc_succ_off);
    const int32_t *sv = reinterpret_cast<const int32_t *>(blob + lay.rc_succ);
    const int32_t *po = reinterpret_cast<const int32_t *>(blob + lay.rc_pred_off);
    const int32_t *pv = reinterpret_cast<const int32_t *>(blob + lay.rc_pred);
    for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < words;
         w += gridDim.x * blockDim.x) {
        if (desc) {
            for (int q = NT - 1; q >= 0; --q) {
                const int t = order[q];
                uint64_t acc = 0;
                for (int e = so[t]; e < so[t + 1]; ++e) {
                    const int s = sv[e];
                    if ((s >> 6) == w) acc |= 1ull << (s & 63);
                    acc |= desc[(int64_t)s * words + w];
                }
                desc[(int64_t)t * words + w] = acc;
            }
        }
        if (anc) {
            for (int q = 0; q < NT; ++q) {
                const int t = order[q];
                uint64_t acc = 0;
                for (int e = po[t]; e < po[t + 1]; ++e) {
                    const int s = pv[e];
                    if ((s >> 6) == w) acc |= 1ull << (s & 63);
                    acc |= anc[(int64_t)s * words + w];
                }
                anc[(int64_t)t * words + w] = acc;
            }
        }
    }
}

// K7: Newman modularity of many partitions of the undirected shadow, one
// CTA per partition: integer intra-edge counts and degree sums per
// community by shared-memory atomics (exact), then the same binary64
// sequence as networkx.community.modularity: per community
// L_c / m - ((res * d_c) * d_c) * norm, summed in community order by
// CPython's compensated float sum().
__global__ void modularity_kernel(const uint8_t *blob, DevLayout lay, int NT,
                                  const int32_t *labels, int ncomm, double res,
                                  double m, double norm, double *out,
                                  uint8_t *status) {
    extern __shared__ __align__(16) uint8_t sm[];
    unsigned long long *Lc = reinterpret_cast<unsigned long long *>(sm);
    unsigned long long *Dc = Lc + ncomm;
    __shared__ int bad;
    const int32_t *so = reinterpret_cast<const int32_t *>(blob + lay.rc_succ_off);
    const int32_t *sv = reinterpret_cast<const int32_t *>(blob + lay.rc_succ);
    const int32_t *lab = labels + (int64_t)blockIdx.x * NT;
    for (int c = threadIdx.x; c < ncomm; c += blockDim.x) Lc[c] = Dc[c] = 0ull;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < NT; t += blockDim.x) {
        const int a = lab[t];
        if (a < 0 || a >= ncomm) {
            bad = 1;
            continue;
        }
        const unsigned long long deg =
            (unsigned long long)(so[t + 1] - so[t]);  // out-degree
        atomicAdd(&Dc[a], deg);
        for (int e = so[t]; e < so[t + 1]; ++e) {
            const int b = lab[sv[e]];
            if (b >= 0 && b < ncomm) {
                atomicAdd(&Dc[b], 1ull);  // in-degree of the successor
                if (b == a) atomicAdd(&Lc[a], 1ull);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // Python >= 3.12 sum() over floats: Neumaier-compensated, with the
        // compensation added once at the end when finite and nonzero
        double f = 0.0, comp = 0.0;
        for (int c = 0; c < ncomm; ++c) {
            const double x = __ddiv_rn((double)Lc[c], m) -
                             __dmul_rn(__dmul_rn(__dmul_rn(res, (double)Dc[c]),
                                                 (double)Dc[c]), norm);
            const double t = f + x;
            if (fabs(f) >= fabs(x))
                comp += (f - t) + x;
            else
                comp += (x - t) + f;
            f = t;
        }
        if (comp != 0.0 && isfinite(comp)) f += comp;
        out[blockIdx.x] = f;
        if (status) status[blockIdx.x] = (uint8_t)bad;
    }
}

// ---------------------------------------------------------------------------
// launchers

static int cuda_fail(cudaError_t e, std::string *err, const char *what) {
    if (err) *err = std::string(what) + ": " + cudaGetErrorString(e);
    return HS_ECUDA;
}

template <int KT, bool CLASS>
static void *eval_fn(bool fast) {
    return fast ? (void *)eval_kernel<KT, CLASS, true>
                : (void *)eval_kernel<KT, CLASS, false>;
}

static void *pick_eval(int kt, bool cls, bool fast) {
    switch (kt) {
        case 2: return cls ? eval_fn<2, true>(fast) : eval_fn<2, false>(fast);
        case 3: return cls ? eval_fn<3, true>(fast) : eval_fn<3, false>(fast);
        case 4: return cls ? eval_fn<4, true>(fast) : eval_fn<4, false>(fast);
        default: return cls ? eval_fn<0, true>(fast) : eval_fn<0, false>(fast);
    }
}

int beval_occupancy(int T, size_t smem, int *blocks) {
    if (cudaFuncSetAttribute(beval_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return HS_ECUDA;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, beval_kernel, T, smem) !=
        cudaSuccess)
        return HS_ECUDA;
    return HS_OK;
}

int launch_beval(const DevState &ds, const EvalParams &p, int grid,
                 cudaStream_t stream, std::string *err) {
    cudaError_t e = cudaFuncSetAttribute(
        beval_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ds.smem);
    if (e != cudaSuccess) return cuda_fail(e, err, "cudaFuncSetAttribute");
    void *args[] = {(void *)&p};
    e = cudaLaunchKernel((const void *)beval_kernel, dim3(grid), dim3(ds.T), args,
                         ds.smem, stream);
    if (e != cudaSuccess) return cuda_fail(e, err, "batched eval launch");
    return HS_OK;
}

int eval_occupancy(int kt, bool cls, int T, size_t smem, int *blocks) {
    int worst = 1 << 30;
    for (int f = 0; f < 2; ++f) {
        void *fn = pick_eval(kt, cls, f == 1);
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess)
            return HS_ECUDA;
        int b = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, T, smem) !=
            cudaSuccess)
            return HS_ECUDA;
        worst = b < worst ? b : worst;
    }
    *blocks = worst;
    return HS_OK;
}

int launch_eval(const DevState &ds, bool cls, const EvalParams &p, int grid,
                cudaStream_t stream, std::string *err) {
    void *fn = pick_eval(ds.kt, cls, p.flags == 0);
    cudaError_t e = cudaFuncSetAttribute(
        fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ds.smem);
    if (e != cudaSuccess) return cuda_fail(e, err, "cudaFuncSetAttribute");
    void *args[] = {(void *)&p};
    e = cudaLaunchKernel(fn, dim3(grid), dim3(ds.T), args, ds.smem, stream);
    if (e != cudaSuccess) return cuda_fail(e, err, "eval launch");
    return HS_OK;
}

template <int KT, bool CLASS>
static void *ea_fn(bool fast) {
    return fast ? (void *)ea_kernel<KT, CLASS, true> : (void *)ea_kernel<KT, CLASS, false>;
}

static void *pick_ea(int kt, bool cls, bool fast) {
    switch (kt) {
        case 2: return cls ? ea_fn<2, true>(fast) : ea_fn<2, false>(fast);
        case 3: return cls ? ea_fn<3, true>(fast) : ea_fn<3, false>(fast);
        case 4: return cls ? ea_fn<4, true>(fast) : ea_fn<4, false>(fast);
        default: return cls ? ea_fn<0, true>(fast) : ea_fn<0, false>(fast);
    }
}

int launch_ea(const DevState &ds, bool cls, const EvalParams &p, const EaParams &ea,
              cudaStream_t stream, std::string *err, int grid) {
    void *fn = pick_ea(ds.kt, cls, p.flags == 0);
    cudaError_t e = cudaFuncSetAttribute(
        fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ds.smem);
    if (e != cudaSuccess) return cuda_fail(e, err, "cudaFuncSetAttribute");
    void *args[] = {(void *)&p, (void *)&ea};
    e = cudaLaunchKernel(fn, dim3(grid), dim3(ds.T), args, ds.smem, stream);
    if (e != cudaSuccess) return cuda_fail(e, err, "ea launch");
    return HS_OK;
}

template <int KT, bool CLASS>
static void *sa_fn(bool fast) {
    return fast ? (void *)sa_kernel<KT, CLASS, true> : (void *)sa_kernel<KT, CLASS, false>;
}

static void *pick_sa(int kt, bool cls, bool fast) {
    switch (kt) {
        case 2: return cls ? sa_fn<2, true>(fast) : sa_fn<2, false>(fast);
        case 3: return cls ? sa_fn<3, true>(fast) : sa_fn<3, false>(fast);
        case 4: return cls ? sa_fn<4, true>(fast) : sa_fn<4, false>(fast);
        default: return cls ? sa_fn<0, true>(fast) : sa_fn<0, false>(fast);
    }
}

int launch_sa(const DevState &ds, bool cls, const EvalParams &p, const SaParams &sa,
              cudaStream_t stream, std::string *err, int grid) {
    void *fn = pick_sa(ds.kt, cls, p.flags == 0);
    cudaError_t e = cudaFuncSetAttribute(
        fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ds.smem);
    if (e != cudaSuccess) return cuda_fail(e, err, "cudaFuncSetAttribute");
    void *args[] = {(void *)&p, (void *)&sa};
    e = cudaLaunchKernel(fn, dim3(grid), dim3(ds.T), args, ds.smem, stream);
    if (e != cudaSuccess) return cuda_fail(e, err, "sa launch");
    return HS_OK;
}

int launch_cp(const uint8_t *blob, const DevLayout &lay, int V, int words,
              const uint64_t *masks, int64_t nsub, double *out, uint8_t *status,
              double *scratch, cudaStream_t stream, std::string *err) {
    const int T = 128;
    const int64_t grid = (nsub + T - 1) / T;
    cp_kernel<<<(unsigned)grid, T, 0, stream>>>(blob, lay, V, words, masks, nsub,
                                                out, status, scratch);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HS_OK : cuda_fail(e, err, "cp launch");
}

int launch_modularity(const uint8_t *blob, const DevLayout &lay, int NT,
                      const int32_t *labels, int64_t P, int ncomm, double res,
                      double m, double norm, double *out, uint8_t *status,
                      cudaStream_t stream, std::string *err) {
    const size_t smem = size_t(ncomm) * 16;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(
            modularity_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return cuda_fail(e, err, "modularity smem");
    }
    for (int64_t lo = 0; lo < P; lo += 65535) {
        const int64_t nb = P - lo < 65535 ? P - lo : 65535;
        modularity_kernel<<<(unsigned)nb, 256, smem, stream>>>(
            blob, lay, NT, labels + lo * NT, ncomm, res, m, norm, out + lo,
            status ? status + lo : nullptr);
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HS_OK : cuda_fail(e, err, "modularity launch");
}

int launch_reach(const uint8_t *blob, const DevLayout &lay, int NT, int words,
                 uint64_t *desc, uint64_t *anc, cudaStream_t stream,
                 std::string *err) {
    const int T = 64;
    const int grid = (words + T - 1) / T;
    reach_kernel<<<grid > 0 ? grid : 1, T, 0, stream>>>(blob, lay, NT, words, desc,
                                                       anc);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HS_OK : cuda_fail(e, err, "reach launch");
}

}  // namespace hs
