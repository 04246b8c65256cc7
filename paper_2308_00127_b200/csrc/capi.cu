// extern "C" boundary (include/hetsched_b200.h): argument checking, device
// state (launch configuration + plan upload per device), scratch, and the
// host-buffer pipeline. All device work is issued on the caller's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "host_pack.hpp"
#include "jit.hpp"
#include "kernels.cuh"
#include "plan.hpp"
#include "scratch.hpp"

struct hs_plan {
    hs::Plan p;
};

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

int cuda_err(cudaError_t e, const char *what) {
    return set_err(HS_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                          \
    do {                                                  \
        cudaError_t e_ = (call);                          \
        if (e_ != cudaSuccess) return cuda_err(e_, #call); \
    } while (0)

int kt_of(int K) { return K <= 2 ? 2 : (K <= 4 ? K : 0); }

uint32_t flags_of(const hs::Plan &p) {
    uint32_t f = 0;
    if (p.mem_check) f |= hs::F_MEM;
    if (!p.all_batch_ok) f |= hs::F_OKL;
    if (!p.latency_complete) f |= hs::F_MISS;
    if (p.nan_possible) f |= hs::F_NAN;
    return f;
}

}  // namespace

namespace hs {

namespace {
constexpr int kMaxDevices = 64;
std::mutex g_pool_m;
cudaMemPool_t g_pools[kMaxDevices] = {};
}  // namespace

cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaMallocAsync(p, bytes, s);
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> g(g_pool_m);
        if (!g_pools[dev]) {
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            e = cudaMemPoolCreate(&g_pools[dev], &props);
            if (e != cudaSuccess) {
                g_pools[dev] = nullptr;
                return e;
            }
            uint64_t keep = ~uint64_t(0);
            cudaMemPoolSetAttribute(g_pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
        }
        pool = g_pools[dev];
    }
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

int scratch_trim() {
    std::lock_guard<std::mutex> g(g_pool_m);
    for (cudaMemPool_t pool : g_pools)
        if (pool) {
            const cudaError_t e = cudaMemPoolTrimTo(pool, 0);
            if (e != cudaSuccess) return cuda_err(e, "hs_scratch_trim");
        }
    return HS_OK;
}

// the thread-local error message of hs_last_error(), for the other
// translation units of the library (decomp.cpp, validate.cu)
int set_error(int code, const std::string &msg) { return set_err(code, msg); }

Plan::~Plan() {
    int cur = -1;
    cudaGetDevice(&cur);
    for (DevState *d : devs) {
        if (!d) continue;
        if (d->blob) {
            cudaSetDevice(d->device);
            cudaFree(d->blob);
        }
        delete d;
    }
    for (JitModule *m : jits) {
        if (!m) continue;
        cudaSetDevice(m->device);
        jit_free(m);
    }
    if (cur >= 0) cudaSetDevice(cur);
}

static bool jit_enabled() {
    const char *v = getenv("HS_JIT");
    return !(v && v[0] == '0');
}

// specialised module for the current device, or null
const JitModule *find_jit(const Plan &p, int dev) {
    if (!jit_enabled()) return nullptr;
    std::lock_guard<std::mutex> lk(p.mu);
    return (int)p.jits.size() > dev ? p.jits[dev] : nullptr;
}

int get_dev_state(const Plan &p, const DevState **out, std::string *err) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        if (err) *err = std::string("cudaGetDevice: ") + cudaGetErrorString(e);
        return HS_ECUDA;
    }
    std::lock_guard<std::mutex> lk(p.mu);
    if ((int)p.devs.size() > dev && p.devs[dev]) {
        *out = p.devs[dev];
        return HS_OK;
    }
    int optin = 0, sms = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    DevState *ds = new DevState();
    ds->device = dev;
    ds->sms = sms;
    ds->kt = kt_of(p.K);
    ds->ld_cap = p.pref_ld() + 16;
    const bool cls = !p.uniform_comm;
    if (p.batched) ds->kt = 0;  // device state in shared memory
    const int64_t slot_bytes = int64_t(p.live_slots) * 8 * (p.batched ? p.P : 1);
    const int64_t per_lane = ds->ld_cap + slot_bytes +
                             (ds->kt == 0 ? int64_t(16) * p.K : 0);
    const int64_t budget = int64_t(optin) - 16 - 1024;
    auto lanes_for = [&](int64_t plan_bytes) {
        int64_t l = (budget - plan_bytes) / per_lane;
        l = std::min<int64_t>(l, 256);
        return int(l / 32 * 32);
    };
    int la = lanes_for(p.lay.eval_bytes), lb = lanes_for(0);
    // Graphs whose live end times leave fewer than kMinLanes lanes per SM
    // (WS1000: 478 slots = 3.8 KB per candidate, one warp) keep the slots in
    // global memory instead -- an L2-resident [slot][lane] array per CTA,
    // coalesced like the shared-memory one -- so several warps share an SM
    // and hide its latency; shared memory then holds tiles and tables.
    constexpr int kMinLanes = 128;
    if (std::max(la, lb) < kMinLanes && slot_bytes > 0) {
        const int64_t pl = ds->ld_cap + (ds->kt == 0 ? int64_t(16) * p.K : 0);
        // lanes per CTA bound the scratch footprint (SMs x lanes x slots x
        // 8 B) that has to stay L2-resident
        int64_t cap_l = 256;
        if (const char *v = getenv("HS_GSLOT_LANES")) cap_l = std::max(32, atoi(v));
        auto lanes_g = [&](int64_t plan_bytes) {
            int64_t l = (budget - plan_bytes) / pl;
            l = std::min<int64_t>(l, cap_l);
            return int(l / 32 * 32);
        };
        const int ga = lanes_g(p.lay.eval_bytes), gb = lanes_g(0);
        if (std::max(ga, gb) > std::max(la, lb)) {
            ds->ends_global = true;
            la = ga;
            lb = gb;
        }
    }
    // plan tables in shared memory unless that costs more than one warp
    ds->plan_smem = la >= 32 && la >= lb - 32;
    auto configure = [&](bool psm) {
        ds->plan_smem = psm;
        ds->T = psm ? la : lb;
        ds->blocks_per_sm = 0;
        if (ds->T < 32) return;
        ds->lanes = ds->T;
        ds->smem_tile = 16 + (ds->plan_smem ? p.lay.eval_bytes : 0);
        ds->smem_ends = ds->smem_tile +
                        ((int64_t(ds->T) * ds->ld_cap + 15) & ~int64_t(15));
        ds->smem_kstate = ds->smem_ends + (ds->ends_global ? 0 : slot_bytes * ds->T);
        ds->smem = ds->smem_kstate +
                   (ds->kt == 0 ? int64_t(2) * p.K * ds->T * 8 : 0);
        int blocks = 0;
        const int orc = p.batched ? beval_occupancy(ds->T, ds->smem, &blocks)
                                  : eval_occupancy(ds->kt, cls, ds->T, ds->smem, &blocks);
        if (orc != HS_OK) blocks = 0;
        ds->blocks_per_sm = blocks;
    };
    configure(ds->plan_smem);
    // the batched-variant kernel is latency-bound at one CTA per SM (ncu
    // r2w: 12.5 % occupancy, 7 cycles per issue): when its tables read
    // through L1 leave room for more resident lanes (several CTAs per SM),
    // take that configuration
    if (p.batched && ds->plan_smem) {
        const int64_t with = int64_t(ds->T) * ds->blocks_per_sm;
        configure(false);
        if (int64_t(ds->T) * ds->blocks_per_sm <= with) configure(true);
    }
    if (ds->blocks_per_sm < 1) {  // eval unusable; bounds kernels still run
        ds->T = ds->lanes = 0;
        ds->smem = 0;
    }
    // device blob with slot indices scaled to element offsets in [slot][lane]
    std::vector<uint8_t> img = p.blob;
    NodeRec *nodes = reinterpret_cast<NodeRec *>(img.data() + p.lay.node);
    EdgeRec *edges = reinterpret_cast<EdgeRec *>(img.data() + p.lay.edge);
    if (!p.batched) {  // batched: the kernel scales (slot * P + part) itself
        for (int i = 0; i < p.V; ++i)
            if (nodes[i].out_slot >= 0) nodes[i].out_slot *= ds->lanes;
        for (size_t q = 0; q < p.edges.size(); ++q) edges[q].slot *= ds->lanes;
    }
    cudaGetLastError();  // clear a sticky-free error from the occupancy probe
    e = cudaMalloc(&ds->blob, img.size());
    if (e == cudaSuccess)
        e = cudaMemcpy(ds->blob, img.data(), img.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        if (ds->blob) cudaFree(ds->blob);
        delete ds;
        if (err) *err = std::string("plan upload: ") + cudaGetErrorString(e);
        return HS_ECUDA;
    }
    if (ds->ends_global) {
        // the per-launch slot scratch (tens of MB) comes from the device's
        // default stream-ordered pool: keep freed blocks in the pool instead
        // of unmapping them at every synchronisation
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
    }
    if ((int)p.devs.size() <= dev) p.devs.resize(dev + 1, nullptr);
    p.devs[dev] = ds;
    *out = ds;
    return HS_OK;
}

}  // namespace hs

namespace {

struct Scratch {
    void *ptr = nullptr;
    cudaStream_t s = nullptr;
    ~Scratch() {
        if (ptr) cudaFreeAsync(ptr, s);
    }
};

// Common body of hs_eval / hs_eval_gen / hs_trace.
int run_eval(const hs_plan *plan, const uint8_t *genes, int64_t n, int64_t ld,
             int gen, uint64_t seed, int64_t first, const uint8_t *tmpl,
             const int16_t *group, int n_groups, double *makespan,
             uint8_t *status, double *starts, uint8_t *genes_out, hs_best *best,
             int64_t index_base, cudaStream_t stream, int packed = 0) {
    if (!plan) return set_err(HS_EINVAL, "null plan");
    const hs::Plan &p = plan->p;
    if (n < 0) return set_err(HS_EINVAL, "n < 0");
    if (packed == 2) {
        // base-3 genes, 5 per byte: rows of ld bytes, 5*ld >= V, at most
        // the staged tile row (expanded in place)
        if (p.batched ? p.n_opt > 3 : p.K > 3)
            return set_err(HS_EINVAL, "base-3 packed genomes need at most 3 gene values");
        if (n > 0 && p.V > 0 &&
            (!genes || ld * 5 < p.V || ld > p.pref_ld() || ld > 256))
            return set_err(HS_EINVAL, "base-3 packed genes must be [n x ld], "
                                      "5*ld >= V, ld <= preferred stride");
    } else if (packed) {
        // 2-bit genes: rows of ld bytes, ld a multiple of 4, >= ceil(V/4),
        // at most the staged tile row (expanded in place)
        if (p.batched ? p.n_opt > 4 : p.K > 4)
            return set_err(HS_EINVAL, "2-bit packed genomes need at most 4 gene values");
        if (n > 0 && p.V > 0 &&
            (!genes || ld % 4 || ld * 4 < p.V || ld > p.pref_ld() || ld > 256))
            return set_err(HS_EINVAL, "packed genes must be [n x ld], ld % 4 == 0, "
                                      "4*ld >= V, ld <= preferred stride");
    } else if (!gen && n > 0 && p.V > 0 && (!genes || ld < p.V)) {
        return set_err(HS_EINVAL, "genes must be [n x ld] with ld >= V");
    }
    const hs::DevState *ds = nullptr;
    std::string err;
    int rc = hs::get_dev_state(p, &ds, &err);
    if (rc) return set_err(rc, err);
    if (ds->lanes == 0)
        return set_err(HS_EINVAL, "graph too large for the shared-memory "
                                  "evaluator (live end-time slots of one warp "
                                  "exceed the per-CTA shared memory)");

    const hs::JitModule *jm = hs::find_jit(p, ds->device);
    Scratch repack;
    repack.s = stream;
    // the specialised kernel reads its staged rows as 32-bit words
    if (!gen && !packed && n > 0 && (ld > ds->ld_cap || (jm && ld % 4))) {
        // exotic row stride: compact to the preferred stride first
        const int64_t pl = p.pref_ld();
        CK(hs::scratch_alloc(&repack.ptr, size_t(n * pl), stream));
        CK(cudaMemcpy2DAsync(repack.ptr, size_t(pl), genes, size_t(ld),
                             size_t(p.V), size_t(n), cudaMemcpyDeviceToDevice,
                             stream));
        genes = static_cast<const uint8_t *>(repack.ptr);
        ld = pl;
    }
    const int lanes = jm ? jm->lanes : ds->lanes;
    const int64_t ntiles = (n + lanes - 1) / lanes;
    // the direct-load kernel (jit_direct_ok) packs several CTAs per SM
    const bool direct = jm && jm->kern_direct && !starts && !gen && !packed && ld % 4 == 0 &&
                        (reinterpret_cast<uintptr_t>(genes) & 3) == 0;
    const int64_t cap = jm ? int64_t(jm->sms) *
                                 (direct ? jm->blocks_per_sm_direct : jm->blocks_per_sm)
                           : int64_t(ds->sms) * ds->blocks_per_sm;
    const int grid = int(std::max<int64_t>(1, std::min(ntiles, cap)));

    Scratch red;
    red.s = stream;
    hs::EvalParams a{};
    if (best) {
        CK(hs::scratch_alloc(&red.ptr, size_t(grid) * sizeof(hs_best) + 16, stream));
        a.partial = static_cast<hsk::Best *>(red.ptr);
        a.ticket = reinterpret_cast<unsigned int *>(
            static_cast<uint8_t *>(red.ptr) + size_t(grid) * sizeof(hs_best));
        CK(cudaMemsetAsync(a.ticket, 0, 16, stream));
    }
    a.blob = ds->blob;
    a.lay = p.lay;
    a.eval_bytes = p.lay.eval_bytes;
    a.V = p.V;
    a.K = p.K;
    a.gene_range = p.batched ? p.n_opt : p.K;
    a.n_opt = p.n_opt;
    a.P = p.P;
    a.n_cls = p.n_cls;
    a.flags = flags_of(p);
    a.plan_smem = ds->plan_smem ? 1 : 0;
    a.lanes = lanes;
    a.ld_s = (gen || packed) ? p.pref_ld() : int(ld);
    a.packed = packed;
    a.slots = p.live_slots;
    a.bulk = (!gen && (reinterpret_cast<uintptr_t>(genes) & 15) == 0) ? 1 : 0;
    a.genes = genes;
    a.n = n;
    a.ld = ld;
    a.gen = gen;
    a.seed = seed;
    a.first = first;
    a.tmpl = tmpl;
    a.group = group;
    a.n_groups = group ? n_groups : p.V;
    a.makespan = makespan;
    a.status = status;
    a.starts = starts;
    a.genes_out = genes_out;
    a.best = reinterpret_cast<hsk::Best *>(best);
    a.index_base = index_base;
    a.smem_tile = jm ? jm->smem_tile : ds->smem_tile;
    if (jm) {
        // hash-random rows without a template or group map are in range by
        // construction and fill whole 4-gene words (gen_row): no check pass
        a.sanitize = (gen == 1 && !tmpl && !group) ? 0 : 1;
        // double-buffered TMA staging when every tile is one bulk copy
        const int64_t tail = n % lanes;
        if (!gen && !packed && a.bulk && (tail * ld) % 16 == 0 && n > 0)
            a.smem_tile2 = jm->smem_tile2;
    }
    a.smem_ends = jm ? jm->smem_ends : ds->smem_ends;
    a.smem_kstate = jm ? jm->smem_kstate : ds->smem_kstate;
    Scratch ends_g;
    ends_g.s = stream;
    if ((jm ? jm->ends_global : ds->ends_global) && n > 0) {
        a.ends_g_cta = int64_t(jm ? jm->slots : p.live_slots) * (p.batched ? p.P : 1) * lanes;
        CK(hs::scratch_alloc(&ends_g.ptr, size_t(grid) * size_t(a.ends_g_cta) * 8, stream));
        a.ends_g = static_cast<double *>(ends_g.ptr);
    }
    if (jm) {
        a.slots = jm->slots;
        rc = hs::jit_launch(*jm, a, grid, stream, &err);
    } else if (p.batched) {
        rc = hs::launch_beval(*ds, a, grid, stream, &err);
    } else {
        rc = hs::launch_eval(*ds, !p.uniform_comm, a, grid, stream, &err);
    }
    if (rc) return set_err(rc, err);
    return HS_OK;
}

// K9 / K10 setup: the evaluator parameters of one CTA of ds->T lanes (AOT
// body); `ends_g` receives the global slot tier's scratch when needed.
int single_cta_params(const hs_plan *plan, const hs::DevState **dsp, hs::EvalParams &a,
                      Scratch &ends_g, cudaStream_t stream, const hs::JitModule **jmp,
                      int chains = 1) {
    if (!plan) return set_err(HS_EINVAL, "null plan");
    const hs::Plan &p = plan->p;
    if (p.batched) return set_err(HS_EINVAL, "the search kernels run on non-batched plans");
    const hs::DevState *ds = nullptr;
    std::string err;
    int rc = hs::get_dev_state(p, &ds, &err);
    if (rc) return set_err(rc, err);
    if (ds->lanes == 0)
        return set_err(HS_EINVAL, "graph too large for the shared-memory evaluator");
    *dsp = ds;
    a.blob = ds->blob;
    a.lay = p.lay;
    a.eval_bytes = p.lay.eval_bytes;
    a.V = p.V;
    a.K = p.K;
    a.gene_range = p.K;
    a.n_opt = p.n_opt;
    a.P = p.P;
    a.n_cls = p.n_cls;
    a.flags = flags_of(p);
    a.plan_smem = ds->plan_smem ? 1 : 0;
    a.lanes = ds->lanes;
    a.ld_s = p.pref_ld();
    a.slots = p.live_slots;
    a.smem_tile = ds->smem_tile;
    a.smem_ends = ds->smem_ends;
    a.smem_kstate = ds->smem_kstate;
    // the graph-specialised module's search kernels when it has them
    const hs::JitModule *jm = hs::find_jit(p, ds->device);
    if (jm && (!jm->kern_sa || !jm->kern_ea)) jm = nullptr;
    if (const char *v = getenv("HS_SEARCH_AOT"))
        if (atoi(v)) jm = nullptr;
    *jmp = jm;
    if (jm) {
        a.sanitize = 1;
        a.lanes = jm->lanes;
        a.slots = jm->slots;
        a.smem_tile = jm->smem_tile;
        a.smem_ends = jm->smem_ends;
        a.smem_kstate = jm->smem_kstate;
    }
    ends_g.s = stream;
    if (jm ? jm->ends_global : ds->ends_global) {
        a.ends_g_cta = int64_t(a.slots) * a.lanes;
        CK(hs::scratch_alloc(&ends_g.ptr, size_t(a.ends_g_cta) * 8 * size_t(chains), stream));
        a.ends_g = static_cast<double *>(ends_g.ptr);
    }
    return HS_OK;
}

int run_ea(const hs_plan *plan, uint8_t *parent, double cur_fit, const int32_t *moff,
           const int32_t *mpos, const uint8_t *mval, int32_t budget, double *out_fit,
           int32_t *info, cudaStream_t stream, const double *cur_in = nullptr,
           int32_t first_child = -1, int32_t chains = 1, int64_t chain_stride = 0) {
    if (budget < 0 || !parent || !out_fit || !info || (budget > 0 && !moff))
        return set_err(HS_EINVAL, "bad EA arguments");
    const hs::DevState *ds = nullptr;
    const hs::JitModule *jm = nullptr;
    hs::EvalParams a{};
    Scratch ends_g;
    if (chains < 1 || (chains > 1 && chain_stride < plan->p.V))
        return set_err(HS_EINVAL, "bad EA chain count / stride");
    int rc = single_cta_params(plan, &ds, a, ends_g, stream, &jm, chains);
    if (rc) return rc;
    std::string err;
    hs::EaParams e{};
    e.chain_stride = chains > 1 ? chain_stride : 0;
    e.parent = parent;
    e.cur_fit = cur_fit;
    e.moff = moff;
    e.mpos = mpos;
    e.mval = mval;
    e.budget = budget;
    const char *lv = getenv("HS_EA_LEVELS");
    e.two_level = lv ? atoi(lv) >= 2 : 1;
    e.out_fit = out_fit;
    e.info = info;
    e.cur_in = cur_in;
    e.first_child = first_child;
    e.accumulate = first_child >= 0;
    if (!e.accumulate) CK(cudaMemsetAsync(info, 0, 4 * sizeof(int32_t) * size_t(chains), stream));
    rc = jm ? hs::jit_launch_search(*jm, 2, a, &e, stream, &err, chains)
            : hs::launch_ea(*ds, !plan->p.uniform_comm, a, e, stream, &err, chains);
    if (rc) return set_err(rc, err);
    return HS_OK;
}

int run_sa(const hs_plan *plan, uint8_t *genes, uint8_t *best, uint64_t *rng,
           uint32_t *buf, double *f, int32_t *istate, double alpha, int32_t n_dev,
           int32_t budget, int32_t window, cudaStream_t stream, int32_t chains = 1,
           int64_t chain_stride = 0) {
    if (!genes || !best || !rng || !buf || !f || !istate || n_dev < 1 || n_dev > 256 ||
        budget < 0 || window < 1)
        return set_err(HS_EINVAL, "bad SA arguments");
    const hs::DevState *ds = nullptr;
    const hs::JitModule *jm = nullptr;
    hs::EvalParams a{};
    Scratch ends_g;
    if (chains < 1 || (chains > 1 && chain_stride < plan->p.V))
        return set_err(HS_EINVAL, "bad SA chain count / stride");
    int rc = single_cta_params(plan, &ds, a, ends_g, stream, &jm, chains);
    if (rc) return rc;
    if (n_dev != plan->p.K) return set_err(HS_EINVAL, "n_dev != number of devices");
    std::string err;
    hs::SaParams e{};
    e.window = std::min(window, a.lanes);
    Scratch spec;
    spec.s = stream;
    // speculation scratch per chain: window base steps + 32 continuation
    // steps (two-level): [fit f64 | pos i32 | new u8 | status u8]
    e.spec_stride = int64_t(e.window) + 32;
    const size_t nw = size_t(e.spec_stride) * size_t(chains);
    CK(hs::scratch_alloc(&spec.ptr, nw * 16 + 64, stream));
    uint8_t *sp = static_cast<uint8_t *>(spec.ptr);
    e.sfit = reinterpret_cast<double *>(sp);
    e.spos = reinterpret_cast<int32_t *>(sp + nw * 8);
    e.snew = sp + nw * 12;
    e.sst = sp + nw * 13;
    e.chain_stride = chains > 1 ? chain_stride : 0;
    e.genes = genes;
    e.best = best;
    e.rng = reinterpret_cast<hs_u64 *>(rng);
    e.buf = buf;
    e.f = f;
    e.istate = istate;
    e.alpha = alpha;
    e.n_dev = n_dev;
    e.budget = budget;
    const char *hx = getenv("HS_SA_HOST_EXP");
    e.host_exp = hx && atoi(hx) ? 1 : 0;
    // second level: continuation steps per branch (0 = off; HS_SA_LEVEL2)
    const char *lv = getenv("HS_SA_LEVEL2");
    e.two_level = lv ? std::max(0, std::min(16, atoi(lv))) : 8;
    rc = jm ? hs::jit_launch_search(*jm, 1, a, &e, stream, &err, chains)
            : hs::launch_sa(*ds, !plan->p.uniform_comm, a, e, stream, &err, chains);
    if (rc) return set_err(rc, err);
    return HS_OK;
}

}  // namespace

extern "C" {

const char *hs_last_error(void) { return g_err.c_str(); }

int hs_abi_version(void) { return HS_ABI_VERSION; }

int hs_scratch_trim(void) { return hs::scratch_trim(); }

int hs_plan_create(const hs_instance_desc *desc, hs_plan **out) {
    if (!desc || !out) return set_err(HS_EINVAL, "null argument");
    hs_plan *pl = new (std::nothrow) hs_plan();
    if (!pl) return set_err(HS_ENOMEM, "out of host memory");
    std::string err;
    int rc = hs::build_plan(*desc, pl->p, &err);
    if (rc) {
        delete pl;
        return set_err(rc, err);
    }
    *out = pl;
    return HS_OK;
}

void hs_plan_destroy(hs_plan *plan) { delete plan; }

int hs_plan_create_batched(const hs_instance_desc *desc, const int32_t *splits,
                           int32_t n_splits, hs_plan **out) {
    if (!desc || !out) return set_err(HS_EINVAL, "null argument");
    hs_plan *pl = new (std::nothrow) hs_plan();
    if (!pl) return set_err(HS_ENOMEM, "out of host memory");
    std::string err;
    hs::BatchedSpec bs;
    bs.splits = splits;
    bs.n_splits = n_splits;
    int rc = hs::build_plan(*desc, pl->p, &err, &bs);
    if (rc) {
        delete pl;
        return set_err(rc, err);
    }
    *out = pl;
    return HS_OK;
}

int hs_plan_batched_options(const hs_plan *plan, int32_t *n_opt, int32_t *max_parts,
                            int32_t *table) {
    if (!plan) return set_err(HS_EINVAL, "null plan");
    const hs::Plan &p = plan->p;
    if (!p.batched) return set_err(HS_EINVAL, "not a batched-variant plan");
    if (n_opt) *n_opt = p.n_opt;
    if (max_parts) *max_parts = p.P;
    if (table) std::copy(p.opt_tab.begin(), p.opt_tab.end(), table);
    return HS_OK;
}

int hs_plan_specialize(const hs_plan *plan, double *compile_ms) {
    if (!plan) return set_err(HS_EINVAL, "null plan");
    const hs::Plan &p = plan->p;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaFree(nullptr));  // make sure the primary context exists
    {
        std::lock_guard<std::mutex> lk(p.mu);
        if ((int)p.jits.size() > dev && p.jits[dev]) {
            if (compile_ms) *compile_ms = p.jits[dev]->compile_ms;
            return HS_OK;
        }
    }
    if (!hs::jit_eligible(p))
        return set_err(HS_EINVAL, "plan not eligible for the specialised "
                                  "evaluator (needs a non-batched plan with "
                                  "K <= 64, V <= 1100, E <= 2600 and no NaN "
                                  "in the cost model)");
    hs::JitModule *m = nullptr;
    std::string err;
    int rc = hs::jit_build(p, dev, &m, &err);
    if (rc) return set_err(rc, err);
    std::lock_guard<std::mutex> lk(p.mu);
    if ((int)p.jits.size() <= dev) p.jits.resize(dev + 1, nullptr);
    if (p.jits[dev]) {
        hs::jit_free(m);
    } else {
        p.jits[dev] = m;
    }
    if (compile_ms) *compile_ms = p.jits[dev]->compile_ms;
    return HS_OK;
}

int hs_plan_emit_specialized(const hs_plan *plan, int32_t lanes, char *buf,
                             int64_t cap, int64_t *len) {
    if (!plan || lanes < 1) return set_err(HS_EINVAL, "bad argument");
    if (!hs::jit_eligible(plan->p))
        return set_err(HS_EINVAL, "plan not eligible for the specialised evaluator");
    std::string src;
    if (plan->p.batched)
        hs::jit_emit_batched(plan->p, lanes, hs::JitOpts::from_env(), &src, true);
    else
        hs::jit_emit(plan->p, lanes, hs::JitOpts::from_env(), &src);
    if (len) *len = int64_t(src.size());
    if (buf && cap > 0) {
        const size_t m = std::min<size_t>(src.size(), size_t(cap - 1));
        std::memcpy(buf, src.data(), m);
        buf[m] = 0;
    }
    return HS_OK;
}

int hs_plan_greedy(const hs_plan *plan, uint8_t *genes, double *starts, double *makespan) {
    // greedy (heuristics.py:192-210) over the plan's tables: BFS order, each
    // task on the device (sorted order) whose placement grows the partial
    // makespan least by more than 1e-12; try_place's checks in its order
    // (batch size, memory, links, then the latency entry)
    if (!plan || !genes) return set_err(HS_EINVAL, "null argument");
    const hs::Plan &p = plan->p;
    if (p.batched) return set_err(HS_EINVAL, "greedy needs a non-batched plan");
    // NaN comparisons, missing latency entries and infeasible tasks are left
    // to the Python scheduler, which raises the reference's exceptions
    if (p.nan_possible) return set_err(HS_EHOST, "greedy: NaN in the cost model");
    const int V = p.V, K = p.K;
    std::vector<double> avail(size_t(K), 0.0), mem(size_t(K), 0.0), endt(size_t(V), 0.0);
    double ms = 0.0;
    auto cls_of = [&](int u, int v) {
        const size_t at = 2 * (size_t(u) * K + v);
        return int(p.bclass[at]) | (int(p.bclass[at + 1]) << 8);
    };
    for (int i = 0; i < V; ++i) {
        const hs::NodeRec &nr = p.nodes[i];
        const double ex = p.extra[i];
        int bk = -1;
        double bc = 0.0, bs = 0.0, be = 0.0;
        for (int k = 0; k < K; ++k) {
            if (!p.okL[k]) continue;
            if (mem[k] + ex > p.cap[k]) continue;
            double ready = 0.0;
            bool nolink = false;
            for (int e = nr.e_begin; e < nr.e_end; ++e) {
                const hs::EdgeRec &er = p.edges[e];
                const int src = genes[er.gpos];
                double c;
                if (p.uniform_comm) {
                    c = src == k ? 0.0 : er.c;
                } else {
                    const int cl = cls_of(src, k);
                    if (cl == 0xFFFF) {
                        nolink = true;
                        break;
                    }
                    c = p.ctab[size_t(er.crow) + cl];
                }
                const double x = endt[er.gpos] + c;
                if (x > ready) ready = x;
            }
            if (nolink) continue;
            if (!p.dur_ok[size_t(i) * K + k])
                return set_err(HS_EHOST, "greedy: missing latency entry");
            const double a = avail[k];
            const double st = a > ready ? a : ready;
            const double en = st + p.dur[size_t(i) * K + k];
            const double cand = en > ms ? en : ms;
            if (bk < 0 || cand < bc - 1e-12) {
                bk = k;
                bc = cand;
                bs = st;
                be = en;
            }
        }
        if (bk < 0) return set_err(HS_EHOST, "greedy: no feasible placement");
        avail[bk] = be;
        mem[bk] += ex;
        endt[i] = be;
        genes[i] = uint8_t(bk);
        if (starts) starts[i] = bs;
        if (be > ms) ms = be;
    }
    if (makespan) *makespan = ms;
    return HS_OK;
}

int hs_plan_get_info(const hs_plan *plan, hs_plan_info *info) {
    if (!plan || !info) return set_err(HS_EINVAL, "null argument");
    const hs::Plan &p = plan->p;
    info->V = p.V;
    info->E = p.E;
    info->K = p.K;
    info->L = p.L;
    info->live_slots = p.live_slots;
    info->n_classes = p.n_classes;
    info->uniform_comm = p.uniform_comm;
    info->full_mesh = p.full_mesh;
    info->mem_check = p.mem_check;
    info->all_batch_ok = p.all_batch_ok;
    info->latency_complete = p.latency_complete;
    info->words = p.words;
    info->pref_ld = p.pref_ld();
    info->specializable = hs::jit_eligible(p) ? 1 : 0;
    info->batched_options = p.batched ? p.n_opt : 0;
    info->max_parts = p.batched ? p.P : 1;
    return HS_OK;
}

int hs_plan_order(const hs_plan *plan, int32_t *order, int32_t *dev_order) {
    if (!plan) return set_err(HS_EINVAL, "null plan");
    if (order) std::copy(plan->p.order.begin(), plan->p.order.end(), order);
    if (dev_order)
        std::copy(plan->p.dev_order.begin(), plan->p.dev_order.end(), dev_order);
    return HS_OK;
}

int hs_eval(const hs_plan *plan, const uint8_t *d_genes, int64_t n, int64_t ld,
            double *d_makespan, uint8_t *d_status, hs_best *d_best,
            int64_t index_base, void *stream) {
    return run_eval(plan, d_genes, n, ld, 0, 0, 0, nullptr, nullptr, 0,
                    d_makespan, d_status, nullptr, nullptr, d_best, index_base,
                    static_cast<cudaStream_t>(stream));
}

int hs_eval_packed(const hs_plan *plan, const uint8_t *d_packed, int64_t n,
                   int64_t ld, double *d_makespan, uint8_t *d_status,
                   hs_best *d_best, int64_t index_base, void *stream) {
    return run_eval(plan, d_packed, n, ld, 0, 0, 0, nullptr, nullptr, 0, d_makespan,
                    d_status, nullptr, nullptr, d_best, index_base,
                    static_cast<cudaStream_t>(stream), 1);
}

int hs_eval_gen_ex(const hs_plan *plan, int mode, uint64_t seed, int64_t first,
                   int64_t n, const uint8_t *d_template, const int16_t *d_group,
                   int32_t n_groups, double *d_makespan, uint8_t *d_status,
                   uint8_t *d_genes_out, hs_best *d_best, void *stream) {
    if (!plan) return set_err(HS_EINVAL, "null plan");
    if (first < 0) return set_err(HS_EINVAL, "first < 0");
    if (mode != HS_GEN_RANDOM && mode != HS_GEN_ENUM && mode != HS_GEN_NEIGHBOR)
        return set_err(HS_EINVAL, "unknown generation mode");
    if (mode == HS_GEN_NEIGHBOR) {
        if (!d_group || !d_template || n_groups < 1)
            return set_err(HS_EINVAL, "neighbour moves need a template and groups");
        const long double k = plan->p.K, ng = n_groups;
        if ((long double)first + (long double)n > ng * k + ng * ng * k * k)
            return set_err(HS_EINVAL, "neighbour index out of range");
    }
    if (d_group && (n_groups < 0 || n_groups > plan->p.V || !d_template))
        return set_err(HS_EINVAL, "group map needs a template and "
                                  "0 <= n_groups <= V");
    if (mode == HS_GEN_ENUM) {
        // every enumerated index must be < K^n_groups
        const int ng = d_group ? n_groups : plan->p.V;
        long double space = 1.0L;
        for (int j = 0; j < ng && space < 1e19L; ++j) space *= plan->p.K;
        if ((long double)first + (long double)n > space)
            return set_err(HS_EINVAL, "enumeration range exceeds K^groups");
    }
    return run_eval(plan, nullptr, n, 0, mode, seed, first, d_template, d_group,
                    n_groups, d_makespan, d_status, nullptr, d_genes_out, d_best,
                    first, static_cast<cudaStream_t>(stream));
}

int hs_eval_gen(const hs_plan *plan, uint64_t seed, int64_t first, int64_t n,
                double *d_makespan, uint8_t *d_status, uint8_t *d_genes_out,
                hs_best *d_best, void *stream) {
    return hs_eval_gen_ex(plan, HS_GEN_RANDOM, seed, first, n, nullptr, nullptr,
                          0, d_makespan, d_status, d_genes_out, d_best, stream);
}

int hs_trace(const hs_plan *plan, const uint8_t *d_genes, int64_t n, int64_t ld,
             double *d_start, double *d_makespan, uint8_t *d_status,
             void *stream) {
    return run_eval(plan, d_genes, n, ld, 0, 0, 0, nullptr, nullptr, 0,
                    d_makespan, d_status, d_start, nullptr, nullptr, 0,
                    static_cast<cudaStream_t>(stream));
}

namespace {

// Per-thread staging for small host batches (search-loop windows): one
// pinned host buffer and one device buffer reused across calls, so a call
// is one H2D, one launch, one D2H and one stream sync.
struct SmallWs {
    int dev = -1;
    uint8_t *d = nullptr, *h = nullptr;
    size_t cap = 0;
    ~SmallWs() {
        if (d) cudaFree(d);
        if (h) cudaFreeHost(h);
    }
};
thread_local SmallWs g_small;
constexpr int64_t kSmallN = 1 << 16;

int eval_host_small(const hs_plan *plan, const uint8_t *h_genes, int64_t n,
                    int64_t ld, double *h_makespan, uint8_t *h_status,
                    hs_best *h_best, int64_t index_base, cudaStream_t s,
                    int packed) {
    const int64_t V = packed ? ld : plan->p.V;  // bytes of a row
    const int64_t lds = packed ? ld : plan->p.pref_ld();  // TMA-friendly stride
    const size_t gb = (size_t(n * lds) + 255) & ~size_t(255);
    const size_t need = gb + size_t(n) * 9 + 64;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    SmallWs &w = g_small;
    if (w.dev != dev || w.cap < need) {
        if (w.d) cudaFree(w.d);
        if (w.h) cudaFreeHost(w.h);
        w.d = w.h = nullptr;
        const size_t cap = std::max(need, size_t(1) << 20);
        CK(cudaMalloc(&w.d, cap));
        CK(cudaMallocHost(&w.h, cap));
        w.cap = cap;
        w.dev = dev;
    }
    for (int64_t r = 0; r < n; ++r)
        std::memcpy(w.h + r * lds, h_genes + r * ld, size_t(V));
    double *dm = reinterpret_cast<double *>(w.d + gb);
    uint8_t *dst = w.d + gb + size_t(n) * 8;
    hs_best *db = reinterpret_cast<hs_best *>(w.d + ((gb + size_t(n) * 9 + 15) & ~size_t(15)));
    CK(cudaMemcpyAsync(w.d, w.h, size_t(n * lds), cudaMemcpyHostToDevice, s));
    int rc = run_eval(plan, w.d, n, lds, 0, 0, 0, nullptr, nullptr, 0, dm, dst,
                      nullptr, nullptr, h_best ? db : nullptr, index_base, s, packed);
    if (rc) return rc;
    // results come back contiguously: makespans, statuses, best
    const size_t back = (reinterpret_cast<uint8_t *>(db) - reinterpret_cast<uint8_t *>(dm)) +
                        (h_best ? sizeof(hs_best) : 0);
    CK(cudaMemcpyAsync(w.h, dm, back, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (h_makespan) std::memcpy(h_makespan, w.h, size_t(n) * 8);
    if (h_status) std::memcpy(h_status, w.h + size_t(n) * 8, size_t(n));
    if (h_best)
        std::memcpy(h_best, w.h + (reinterpret_cast<uint8_t *>(db) -
                                   reinterpret_cast<uint8_t *>(dm)),
                    sizeof(hs_best));
    return HS_OK;
}

// uint8 host genomes (the reference's layout), K <= 4 (host_pack_enabled):
// the host thread pool packs each chunk to 2 bits per gene into a pinned
// staging buffer while the GPU copies and evaluates the previous one
// (double-buffered), so the PCIe link carries ceil(V/4) instead of V bytes
// per candidate. The call is then bound by the host threads' read rate of
// the uint8 rows (r3u: 3.0-3.2e8 candidates/s on 16 vCPUs against 2.67e8
// for the DMA of the bytes). A chunk holding a gene >= K goes over
// unpacked, so the kernel flags it (status 5) exactly as on the unpacked
// path.
int eval_host_u8_packed(const hs_plan *plan, const uint8_t *h_genes, int64_t n, int64_t ld,
                        double *h_makespan, uint8_t *h_status, hs_best *h_best,
                        int64_t index_base, cudaStream_t s0) {
    const hs::Plan &p = plan->p;
    const int V = p.V;
    const int64_t pld = ((V + 3) / 4 + 3) / 4 * 4;
    const int64_t chunk = std::min<int64_t>(n, 1 << 19);
    const int64_t nchunks = (n + chunk - 1) / chunk;
    const size_t gbytes = size_t(chunk) * size_t(std::max<int64_t>(ld, pld));
    const size_t per = ((gbytes + 255) & ~size_t(255)) + size_t(chunk) * 8 +
                       ((size_t(chunk) + 255) & ~size_t(255));
    uint8_t *stage[2] = {hs::pinned_staging(0, size_t(chunk * pld)),
                         hs::pinned_staging(1, size_t(chunk * pld))};
    if (!stage[0] || !stage[1]) return set_err(HS_ENOMEM, "pinned staging buffers");
    cudaStream_t ss[2] = {s0, nullptr};
    CK(cudaStreamCreateWithFlags(&ss[1], cudaStreamNonBlocking));
    cudaEvent_t ev0 = nullptr, copied[2] = {nullptr, nullptr};
    uint8_t *buf = nullptr;
    hs_best *bests = nullptr;
    int rc = HS_OK;
    do {
        cudaError_t e = cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming);
        for (auto &c : copied)
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c, cudaEventDisableTiming);
        if (e == cudaSuccess) e = hs::scratch_alloc((void **)&buf, 2 * per, s0);
        if (e == cudaSuccess)
            e = hs::scratch_alloc((void **)&bests, size_t(nchunks) * sizeof(hs_best), s0);
        if (e == cudaSuccess) e = cudaEventRecord(ev0, s0);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(ss[1], ev0, 0);
        if (e != cudaSuccess) {
            rc = cuda_err(e, "hs_eval_host (packing) setup");
            break;
        }
        double t_wait = 0, t_pack = 0, t_enq = 0;
        auto now = [] { return std::chrono::steady_clock::now(); };
        auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
        for (int64_t c = 0; c < nchunks && rc == HS_OK; ++c) {
            auto q0 = now();
            const int k = int(c & 1);
            cudaStream_t s = ss[k];
            uint8_t *b = buf + k * per;
            double *dm = reinterpret_cast<double *>(b + ((gbytes + 255) & ~size_t(255)));
            uint8_t *dsx = reinterpret_cast<uint8_t *>(dm + chunk);
            const int64_t lo = c * chunk, rows = std::min(chunk, n - lo);
            // the staging buffer's previous copy (chunk c-2) has left it
            if (c >= 2) {
                e = cudaEventSynchronize(copied[k]);
                if (e != cudaSuccess) {
                    rc = cuda_err(e, "staging reuse");
                    break;
                }
            }
            auto q1 = now();
            const bool ok = hs::pack2_rows(h_genes + lo * ld, ld, V, p.K, rows, stage[k], pld);
            auto q2 = now();
            t_wait += sec(q0, q1); t_pack += sec(q1, q2);
            if (ok)
                e = cudaMemcpyAsync(b, stage[k], size_t(rows * pld), cudaMemcpyHostToDevice, s);
            else
                e = cudaMemcpyAsync(b, h_genes + lo * ld, size_t((rows - 1) * ld + V),
                                    cudaMemcpyHostToDevice, s);
            if (e == cudaSuccess) e = cudaEventRecord(copied[k], s);
            if (e != cudaSuccess) {
                rc = cuda_err(e, "H2D genes");
                break;
            }
            rc = run_eval(plan, b, rows, ok ? pld : ld, 0, 0, 0, nullptr, nullptr, 0,
                          h_makespan ? dm : nullptr, h_status ? dsx : nullptr, nullptr,
                          nullptr, h_best ? bests + c : nullptr, index_base + lo, s,
                          ok ? 1 : 0);
            if (rc) break;
            if (h_makespan)
                e = cudaMemcpyAsync(h_makespan + lo, dm, size_t(rows) * 8,
                                    cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess && h_status)
                e = cudaMemcpyAsync(h_status + lo, dsx, size_t(rows), cudaMemcpyDeviceToHost,
                                    s);
            if (e != cudaSuccess) rc = cuda_err(e, "D2H results");
            t_enq += sec(q2, now());
        }
        auto q3 = now();
        if (rc) break;
        e = cudaEventRecord(ev0, ss[1]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s0, ev0, 0);
        std::vector<hs_best> hb(static_cast<size_t>(nchunks));
        if (e == cudaSuccess && h_best)
            e = cudaMemcpyAsync(hb.data(), bests, size_t(nchunks) * sizeof(hs_best),
                                cudaMemcpyDeviceToHost, s0);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s0);
        if (e != cudaSuccess) {
            rc = cuda_err(e, "hs_eval_host sync");
            break;
        }
        if (h_best) hs_best_merge(hb.data(), nchunks, h_best);
        if (getenv("HS_PACK_TRACE"))
            fprintf(stderr, "pack trace: wait %.2f pack %.2f enqueue %.2f drain %.2f ms\n",
                    t_wait * 1e3, t_pack * 1e3, t_enq * 1e3, sec(q3, now()) * 1e3);
    } while (0);
    // the second stream may still read `buf` when the loop broke early: it
    // drains before the stream-ordered frees on s0
    cudaStreamSynchronize(ss[1]);
    if (buf) cudaFreeAsync(buf, s0);
    if (bests) cudaFreeAsync(bests, s0);
    cudaStreamSynchronize(s0);  // staging buffers are reused by the next call
    cudaStreamDestroy(ss[1]);
    if (ev0) cudaEventDestroy(ev0);
    for (auto c : copied)
        if (c) cudaEventDestroy(c);
    return rc;
}

bool host_pack_enabled(const hs::Plan &p, int64_t n, int packed) {
    if (packed || p.batched || p.K > 4 || p.V < 16 || n <= kSmallN) return false;
    const int64_t pld = ((p.V + 3) / 4 + 3) / 4 * 4;
    if (pld > p.pref_ld() || pld > 256) return false;
    // on by default with >= 8 host threads: r3t measured 3.35e8 cand/s
    // packed on 16 threads against 2.67e8 for the uint8 DMA (WS200, 8.4 M
    // rows per call), once the device scratch stays mapped between calls
    const char *v = getenv("HS_HOST_PACK");
    if (v && *v) return std::atoi(v) != 0;
    return hs::host_pack_threads() >= 8;
}

}  // namespace

static int eval_host_impl(const hs_plan *plan, const uint8_t *h_genes, int64_t n,
                          int64_t ld, double *h_makespan, uint8_t *h_status,
                          hs_best *h_best, int64_t index_base, void *stream,
                          int packed) {
    if (!plan) return set_err(HS_EINVAL, "null plan");
    if (n < 0 || (n > 0 && (!h_genes || (!packed && ld < plan->p.V))))
        return set_err(HS_EINVAL, "genes must be [n x ld] with ld >= V");
    cudaStream_t s0 = static_cast<cudaStream_t>(stream);
    if (n > 0 && n <= kSmallN && plan->p.V > 0)
        return eval_host_small(plan, h_genes, n, ld, h_makespan, h_status, h_best,
                               index_base, s0, packed);
    if (host_pack_enabled(plan->p, n, packed))
        return eval_host_u8_packed(plan, h_genes, n, ld, h_makespan, h_status, h_best,
                                   index_base, s0);
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n, 1 << 19));
    const int64_t nchunks = n > 0 ? (n + chunk - 1) / chunk : 1;
    const size_t gbytes = size_t(chunk * ld);
    const size_t per = ((gbytes + 255) & ~size_t(255)) + size_t(chunk) * 8 +
                       ((size_t(chunk) + 255) & ~size_t(255));
    cudaStream_t s1 = nullptr;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    uint8_t *buf = nullptr;
    hs_best *bests = nullptr;
    int rc = HS_OK;
    do {
        cudaError_t e = cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev1, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventRecord(ev0, s0);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s1, ev0, 0);
        if (e == cudaSuccess) e = hs::scratch_alloc((void **)&buf, 2 * per, s0);
        if (e == cudaSuccess)
            e = hs::scratch_alloc((void **)&bests, size_t(nchunks) * sizeof(hs_best), s0);
        if (e == cudaSuccess) e = cudaEventRecord(ev0, s0);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s1, ev0, 0);
        if (e != cudaSuccess) {
            rc = cuda_err(e, "hs_eval_host setup");
            break;
        }
        for (int64_t c = 0; c < nchunks && rc == HS_OK; ++c) {
            cudaStream_t s = (c & 1) ? s1 : s0;
            uint8_t *b = buf + (c & 1) * per;
            uint8_t *dg = b;
            double *dm = reinterpret_cast<double *>(b + ((gbytes + 255) & ~size_t(255)));
            uint8_t *dsx = reinterpret_cast<uint8_t *>(dm + chunk);
            const int64_t lo = c * chunk, rows = std::min(chunk, n - lo);
            if (rows > 0) {
                // the last row ends at its last gene byte: a row-strided view
                // owns nothing past it
                const int64_t row_bytes = packed ? ld : plan->p.V;
                e = cudaMemcpyAsync(dg, h_genes + lo * ld,
                                    size_t((rows - 1) * ld + row_bytes),
                                    cudaMemcpyHostToDevice, s);
                if (e != cudaSuccess) {
                    rc = cuda_err(e, "H2D genes");
                    break;
                }
            }
            rc = run_eval(plan, dg, std::max<int64_t>(rows, 0), ld, 0, 0, 0,
                          nullptr, nullptr, 0, h_makespan ? dm : nullptr, h_status ? dsx : nullptr,
                          nullptr, nullptr, h_best ? bests + c : nullptr,
                          index_base + lo, s, packed);
            if (rc) break;
            if (h_makespan && rows > 0)
                e = cudaMemcpyAsync(h_makespan + lo, dm, size_t(rows) * 8,
                                    cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess && h_status && rows > 0)
                e = cudaMemcpyAsync(h_status + lo, dsx, size_t(rows),
                                    cudaMemcpyDeviceToHost, s);
            if (e != cudaSuccess) rc = cuda_err(e, "D2H results");
        }
        if (rc) break;
        e = cudaEventRecord(ev1, s1);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s0, ev1, 0);
        std::vector<hs_best> hb(static_cast<size_t>(nchunks));
        if (e == cudaSuccess && h_best)
            e = cudaMemcpyAsync(hb.data(), bests, size_t(nchunks) * sizeof(hs_best),
                                cudaMemcpyDeviceToHost, s0);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s0);
        if (e != cudaSuccess) {
            rc = cuda_err(e, "hs_eval_host sync");
            break;
        }
        if (h_best) hs_best_merge(hb.data(), nchunks, h_best);
    } while (0);
    cudaStreamSynchronize(s1);  // s1 may still read `buf` after an early break
    if (buf) cudaFreeAsync(buf, s0);
    if (bests) cudaFreeAsync(bests, s0);
    cudaStreamDestroy(s1);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    return rc;
}

int hs_eval_host(const hs_plan *plan, const uint8_t *h_genes, int64_t n,
                 int64_t ld, double *h_makespan, uint8_t *h_status,
                 hs_best *h_best, int64_t index_base, void *stream) {
    return eval_host_impl(plan, h_genes, n, ld, h_makespan, h_status, h_best,
                          index_base, stream, 0);
}

int hs_eval_host_packs(const hs_plan *plan, int64_t n) {
    if (!plan) return set_err(HS_EINVAL, "null plan");
    if (n <= kSmallN || plan->p.V <= 0) return 0;
    return host_pack_enabled(plan->p, n, 0) ? 1 : 0;
}

int hs_pack_genes2(const uint8_t *h_genes, int64_t n, int64_t ld, int32_t V, int32_t K,
                   uint8_t *h_packed, int64_t pld, int32_t *all_ok) {
    if (n < 0 || V <= 0 || K < 1 || K > 4 || ld < V || pld < (V + 3) / 4)
        return set_err(HS_EINVAL, "hs_pack_genes2: need n >= 0, V > 0, 1 <= K <= 4, "
                                  "ld >= V, pld >= ceil(V/4)");
    if (n > 0 && (!h_genes || !h_packed)) return set_err(HS_EINVAL, "hs_pack_genes2: null buffer");
    const bool ok = n == 0 || hs::pack2_rows(h_genes, ld, V, K, n, h_packed, pld);
    if (all_ok) *all_ok = ok ? 1 : 0;
    return HS_OK;
}

int hs_eval_host_packed(const hs_plan *plan, const uint8_t *h_packed, int64_t n,
                        int64_t ld, double *h_makespan, uint8_t *h_status,
                        hs_best *h_best, int64_t index_base, void *stream) {
    return eval_host_impl(plan, h_packed, n, ld, h_makespan, h_status, h_best,
                          index_base, stream, 1);
}

int hs_eval_packed3(const hs_plan *plan, const uint8_t *d_packed, int64_t n,
                    int64_t ld, double *d_makespan, uint8_t *d_status,
                    hs_best *d_best, int64_t index_base, void *stream) {
    return run_eval(plan, d_packed, n, ld, 0, 0, 0, nullptr, nullptr, 0, d_makespan,
                    d_status, nullptr, nullptr, d_best, index_base,
                    static_cast<cudaStream_t>(stream), 2);
}

int hs_eval_host_packed3(const hs_plan *plan, const uint8_t *h_packed, int64_t n,
                         int64_t ld, double *h_makespan, uint8_t *h_status,
                         hs_best *h_best, int64_t index_base, void *stream) {
    return eval_host_impl(plan, h_packed, n, ld, h_makespan, h_status, h_best,
                          index_base, stream, 2);
}

int hs_ea_run(const hs_plan *plan, uint8_t *d_parent, double cur_fit,
              const int32_t *d_moff, const int32_t *d_mpos, const uint8_t *d_mval,
              int32_t budget, double *d_fit, int32_t *d_info, void *stream) {
    return run_ea(plan, d_parent, cur_fit, d_moff, d_mpos, d_mval, budget, d_fit, d_info,
                  static_cast<cudaStream_t>(stream));
}

int hs_ea_run_chunk(const hs_plan *plan, uint8_t *d_parent, double *d_fit,
                    const int32_t *d_moff, const int32_t *d_mpos, const uint8_t *d_mval,
                    int32_t n_children, int32_t first_child, int32_t *d_info,
                    void *stream) {
    if (first_child < 0 || !d_fit) return set_err(HS_EINVAL, "bad EA chunk arguments");
    return run_ea(plan, d_parent, 0.0, d_moff, d_mpos, d_mval, n_children, d_fit, d_info,
                  static_cast<cudaStream_t>(stream), d_fit, first_child);
}

int hs_sa_run(const hs_plan *plan, uint8_t *d_genes, uint8_t *d_best, uint64_t *d_rng,
              uint32_t *d_buf, double *d_f, int32_t *d_istate, double alpha,
              int32_t n_dev, int32_t budget, int32_t window, void *stream) {
    return run_sa(plan, d_genes, d_best, d_rng, d_buf, d_f, d_istate, alpha, n_dev, budget,
                  window, static_cast<cudaStream_t>(stream));
}

int hs_sa_run_multi(const hs_plan *plan, int32_t chains, int64_t chain_stride,
                    uint8_t *d_genes, uint8_t *d_best, uint64_t *d_rng, uint32_t *d_buf,
                    double *d_f, int32_t *d_istate, double alpha, int32_t n_dev,
                    int32_t budget, int32_t window, void *stream) {
    return run_sa(plan, d_genes, d_best, d_rng, d_buf, d_f, d_istate, alpha, n_dev, budget,
                  window, static_cast<cudaStream_t>(stream), chains, chain_stride);
}

int hs_ea_run_multi(const hs_plan *plan, int32_t chains, int64_t chain_stride,
                    uint8_t *d_parent, const double *d_cur_fit, const int32_t *d_moff,
                    const int32_t *d_mpos, const uint8_t *d_mval, int32_t budget,
                    double *d_fit, int32_t *d_info, void *stream) {
    if (!d_cur_fit) return set_err(HS_EINVAL, "null start fitness");
    return run_ea(plan, d_parent, 0.0, d_moff, d_mpos, d_mval, budget, d_fit, d_info,
                  static_cast<cudaStream_t>(stream), d_cur_fit, -1, chains, chain_stride);
}

int hs_cp_bound(const hs_plan *plan, const uint64_t *d_masks, int64_t nsub,
                double *d_out, uint8_t *d_status, void *stream) {
    if (!plan) return set_err(HS_EINVAL, "null plan");
    if (nsub < 0 || (nsub > 0 && (!d_masks || !d_out)))
        return set_err(HS_EINVAL, "bad mask arguments");
    if (nsub == 0) return HS_OK;
    const hs::Plan &p = plan->p;
    const hs::DevState *ds = nullptr;
    std::string err;
    int rc = hs::get_dev_state(p, &ds, &err);
    if (rc) return set_err(rc, err);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t step = std::max<int64_t>(
        1, std::min<int64_t>(nsub, (int64_t(1) << 25) / std::max(p.V, 1)));
    Scratch sc;
    sc.s = s;
    CK(hs::scratch_alloc(&sc.ptr, size_t(std::max(p.V, 1)) * size_t(step) * 8, s));
    for (int64_t lo = 0; lo < nsub; lo += step) {
        const int64_t m = std::min(step, nsub - lo);
        rc = hs::launch_cp(ds->blob, p.lay, p.V, std::max(p.words, 1),
                           d_masks + lo * std::max(p.words, 1), m, d_out + lo,
                           d_status ? d_status + lo : nullptr,
                           static_cast<double *>(sc.ptr), s, &err);
        if (rc) return set_err(rc, err);
    }
    return HS_OK;
}

int hs_reach(const hs_plan *plan, uint64_t *d_desc, uint64_t *d_anc,
             void *stream) {
    if (!plan) return set_err(HS_EINVAL, "null plan");
    const hs::Plan &p = plan->p;
    if (p.NT == 0) return HS_OK;
    const hs::DevState *ds = nullptr;
    std::string err;
    int rc = hs::get_dev_state(p, &ds, &err);
    if (rc) return set_err(rc, err);
    rc = hs::launch_reach(ds->blob, p.lay, p.NT, p.words, d_desc, d_anc,
                          static_cast<cudaStream_t>(stream), &err);
    return rc ? set_err(rc, err) : HS_OK;
}

int hs_modularity(const hs_plan *plan, const int32_t *d_labels, int64_t P,
                  int32_t n_comm, double resolution, double *d_out,
                  uint8_t *d_status, void *stream) {
    if (!plan) return set_err(HS_EINVAL, "null plan");
    if (P < 0 || n_comm < 1 || (P > 0 && (!d_labels || !d_out)))
        return set_err(HS_EINVAL, "bad partition arguments");
    const hs::Plan &p = plan->p;
    if (P == 0) return HS_OK;
    if (p.E == 0)
        return set_err(HS_EINVAL, "modularity is undefined without edges");
    if (int64_t(n_comm) * 16 > 200 * 1024)
        return set_err(HS_EINVAL, "too many communities");
    const hs::DevState *ds = nullptr;
    std::string err;
    int rc = hs::get_dev_state(p, &ds, &err);
    if (rc) return set_err(rc, err);
    // undirected shadow of a DAG without duplicate edges: deg_sum = 2E
    const double deg_sum = 2.0 * double(p.E);
    const double m = deg_sum / 2.0;
    const double norm = 1.0 / (deg_sum * deg_sum);
    rc = hs::launch_modularity(ds->blob, p.lay, p.NT, d_labels, P, n_comm,
                               resolution, m, norm, d_out, d_status,
                               static_cast<cudaStream_t>(stream), &err);
    return rc ? set_err(rc, err) : HS_OK;
}

int hs_best_merge(const hs_best *bests, int64_t n, hs_best *out) {
    if (!out || (n > 0 && !bests)) return set_err(HS_EINVAL, "null argument");
    hs_best b{__builtin_huge_val(), -1};
    for (int64_t k = 0; k < n; ++k) {
        if (bests[k].index < 0) continue;
        const double c = bests[k].cost;
        if (b.index < 0 || c < b.cost || (c == b.cost && bests[k].index < b.index))
            b = bests[k];
    }
    *out = b;
    return HS_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Multi-GPU best: one NCCL all-gather of 16 B per rank + an on-device
// lexicographic merge (NCCL has no argmin operator). NCCL is
// resolved at run time with dlopen("libnccl.so.2"): when the caller's NCCL is
// already in the process (torch's, or the application's) the loader returns
// that very library, so the communicator handed in is always used with the
// NCCL that created it, and the library carries no link-time NCCL dependency.
#include <dlfcn.h>

#include <mutex>

namespace {

typedef int (*nccl_allgather_fn)(const void *, void *, size_t, int, ncclComm *,
                                 cudaStream_t);
typedef int (*nccl_count_fn)(const ncclComm *, int *);
typedef const char *(*nccl_errstr_fn)(int);
constexpr int kNcclInt64 = 4;  // ncclInt64 in nccl.h's ncclDataType_t

struct NcclApi {
    nccl_allgather_fn allgather = nullptr;
    nccl_count_fn count = nullptr;
    nccl_errstr_fn errstr = nullptr;
    bool ok = false;
    std::string why;
};

const NcclApi &nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("dlopen libnccl.so.2: ") + dlerror();
            return;
        }
        api.allgather = reinterpret_cast<nccl_allgather_fn>(dlsym(h, "ncclAllGather"));
        api.count = reinterpret_cast<nccl_count_fn>(dlsym(h, "ncclCommCount"));
        api.errstr = reinterpret_cast<nccl_errstr_fn>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.allgather && api.count;
        if (!api.ok) api.why = "libnccl.so.2 lacks ncclAllGather / ncclCommCount";
    });
    return api;
}

// the same rule as hs_best_merge, on the device, over the gathered ranks
__global__ void best_merge_kernel(const hs_best *in, int n, hs_best *out) {
    if (threadIdx.x != 0) return;
    hs_best b{__longlong_as_double(0x7FF0000000000000LL), -1};
    for (int k = 0; k < n; ++k) {
        const hs_best c = in[k];
        if (c.index < 0) continue;
        if (b.index < 0 || c.cost < b.cost || (c.cost == b.cost && c.index < b.index))
            b = c;
    }
    *out = b;
}

}  // namespace

extern "C" int hs_best_allreduce(const hs_best *d_in, hs_best *d_out, ncclComm *comm,
                                 void *stream) {
    if (!d_in || !d_out || !comm) return set_err(HS_EINVAL, "null argument");
    const NcclApi &api = nccl_api();
    if (!api.ok) return set_err(HS_ECUDA, api.why);
    int nranks = 0;
    int nr = api.count(comm, &nranks);
    if (nr != 0 || nranks < 1)
        return set_err(HS_ECUDA, std::string("ncclCommCount: ") +
                                     (api.errstr ? api.errstr(nr) : "failed"));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    hs_best *all = nullptr;
    CK(hs::scratch_alloc(reinterpret_cast<void **>(&all), sizeof(hs_best) * size_t(nranks), s));
    nr = api.allgather(d_in, all, 2, kNcclInt64, comm, s);
    if (nr != 0) {
        cudaFreeAsync(all, s);
        return set_err(HS_ECUDA, std::string("ncclAllGather: ") +
                                     (api.errstr ? api.errstr(nr) : "failed"));
    }
    best_merge_kernel<<<1, 32, 0, s>>>(all, nranks, d_out);
    cudaError_t e = cudaGetLastError();
    cudaFreeAsync(all, s);
    if (e != cudaSuccess) return cuda_err(e, "best_merge_kernel");
    return HS_OK;
}
