// sm_100a kernels of the candidate-mapping evaluator.
//
//  K1 eval_kernel   batched list-scheduling makespan, one lane per candidate
//                   (decode/fitness, heuristics.py:43-148), genomes staged
//                   HBM -> shared memory by a TMA bulk copy per CTA tile,
//                   fused first-index argmin epilogue (K2) and optional
//                   on-device candidate generation (K6) and start-time trace
//                   (K3).
//  K4 cp_kernel     critical_path_bound over task masks (bounds.py:57-72).
//  K5 reach_kernel  descendant / ancestor bitsets (bounds.py:29-54,
//                   core.py:104-111).
//
// Exactness: every floating-point operation is the reference's own binary64
// operation in the reference's order -- additions `end + comm`, `start +
// dur`, `mem + extra`, and Python's max(a, b) written as `b > a ? b : a`
// (DSETP + SEL, which also reproduces Python's NaN behaviour). There are no
// multiplications on the path, and the file is compiled with --fmad=false.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

#include "kernels.cuh"

namespace hs {

namespace {

constexpr double kInf = __builtin_huge_val();

__device__ __forceinline__ double pymax(double a, double b) {
    return b > a ? b : a;  // Python max(a, b): a unless b > a
}

__device__ __forceinline__ bool best_less(double c1, int64_t i1, double c2,
                                          int64_t i2) {
    return c1 < c2 || (c1 == c2 && i1 < i2);
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

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

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src,
                                         uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
            smem_addr(bar)),
        "r"(bytes)
        : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}

// lexicographic (cost, index) min across the CTA, then across CTAs through
// `partial` + a ticket: the last CTA to finish writes *best.
__device__ void reduce_best(double bc, int64_t bi, hs_best *partial,
                            unsigned int *ticket, hs_best *best) {
    __shared__ double s_c[32];
    __shared__ int64_t s_i[32];
    __shared__ bool s_last;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double oc = __shfl_down_sync(0xffffffffu, bc, o);
        const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
        if (best_less(oc, oi, bc, bi)) {
            bc = oc;
            bi = oi;
        }
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        s_c[warp] = bc;
        s_i[warp] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (best_less(s_c[w], s_i[w], bc, bi)) {
                bc = s_c[w];
                bi = s_i[w];
            }
        partial[blockIdx.x].cost = bc;
        partial[blockIdx.x].index = bi;
        __threadfence();
        const unsigned t = atomicAdd(ticket, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    bc = kInf;
    bi = INT64_MAX;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
        const double c = ((volatile double *)&partial[b].cost)[0];
        const int64_t i = ((volatile int64_t *)&partial[b].index)[0];
        if (best_less(c, i, bc, bi)) {
            bc = c;
            bi = i;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double oc = __shfl_down_sync(0xffffffffu, bc, o);
        const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
        if (best_less(oc, oi, bc, bi)) {
            bc = oc;
            bi = oi;
        }
    }
    __syncthreads();
    if (lane == 0) {
        s_c[warp] = bc;
        s_i[warp] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (best_less(s_c[w], s_i[w], bc, bi)) {
                bc = s_c[w];
                bi = s_i[w];
            }
        best->cost = bc;
        best->index = bi == INT64_MAX ? -1 : bi;
        *ticket = 0;  // reusable by the next launch on this stream
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// K1: one lane per candidate. Every lane walks the same node / edge record
// sequence (broadcast reads); only gene-indexed lookups diverge.
template <int KT, bool CLASS>
__global__ void __launch_bounds__(512)
eval_kernel(const EvalParams a) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    const int T = blockDim.x, tid = threadIdx.x;
    const int lanes = a.lanes;  // == T
    const int V = a.V, K = a.K;

    // ---- plan tables: staged once per CTA or read through L1
    const uint8_t *plan = a.blob;
    int64_t off = 16;
    if (a.plan_smem) {
        uint8_t *sp = smem + off;
        const uint4 *src = reinterpret_cast<const uint4 *>(a.blob);
        uint4 *dst = reinterpret_cast<uint4 *>(sp);
        for (int64_t q = tid; q < a.eval_bytes / 16; q += T) dst[q] = src[q];
        plan = sp;
        off += a.eval_bytes;
    }
    const NodeRec *nodes = reinterpret_cast<const NodeRec *>(plan + a.lay.node);
    const EdgeRec *edges = reinterpret_cast<const EdgeRec *>(plan + a.lay.edge);
    const double *dur = reinterpret_cast<const double *>(plan + a.lay.dur);
    const uint8_t *dur_ok = plan + a.lay.dur_ok;
    const double *extra = reinterpret_cast<const double *>(plan + a.lay.extra);
    const double *ctab = reinterpret_cast<const double *>(plan + a.lay.ctab);
    const uint16_t *bclass = reinterpret_cast<const uint16_t *>(plan + a.lay.bclass);
    const double *cap = reinterpret_cast<const double *>(plan + a.lay.cap);
    const uint8_t *okL = plan + a.lay.okL;

    uint8_t *gtile = smem + off;  // [lanes][ld_s] genomes of this tile
    off += ((int64_t)lanes * a.ld_s + 15) & ~int64_t(15);
    double *ends = reinterpret_cast<double *>(smem + off);  // [slots][lanes]
    off += (int64_t)a.slots * lanes * 8;
    double *kstate = reinterpret_cast<double *>(smem + off);  // [2K][lanes]

    if (tid == 0) mbar_init(bar);
    __syncthreads();

    const uint32_t flags = a.flags;
    double bc = kInf;
    int64_t bi = INT64_MAX;
    uint32_t phase = 0;
    const int64_t ntiles = (a.n + lanes - 1) / lanes;
    const bool bulk = a.bulk;

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t c0 = tile * lanes;
        const int64_t left = a.n - c0;
        const int rows = left < lanes ? (int)left : lanes;
        __syncthreads();  // the previous tile's genomes are no longer read
        if (a.gen) {
            // K6: on-device candidates (oracle gen_genes / enumeration)
            if (tid < rows) {
                const int NG = a.n_groups;
                const uint64_t c = (uint64_t)(a.first + c0 + tid);
                uint8_t *r8 = gtile + (int64_t)tid * a.ld_s;
                if (a.gen == 1) {
                    const int W4 = (NG + 3) >> 2;
                    uint32_t *row = reinterpret_cast<uint32_t *>(r8);
                    for (int w = 0; w < W4; ++w) {
                        const uint64_t ctr = c * (uint64_t)W4 + (uint64_t)w + 1ull;
                        const uint64_t h =
                            splitmix64(a.seed + ctr * 0x9E3779B97F4A7C15ull);
                        uint32_t pk = 0;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t v16 = (uint32_t)((h >> (16 * q)) & 0xFFFFull);
                            pk |= ((v16 * (uint32_t)K) >> 16) << (8 * q);
                        }
                        row[w] = pk;
                    }
                } else if (c < (1ull << 32)) {  // mixed-radix digits of c
                    uint32_t x = (uint32_t)c;
                    for (int j = 0; j < NG; ++j) {
                        r8[j] = (uint8_t)(x % (uint32_t)K);
                        x /= (uint32_t)K;
                    }
                } else {
                    uint64_t x = c;
                    for (int j = 0; j < NG; ++j) {
                        r8[j] = (uint8_t)(x % (uint64_t)K);
                        x /= (uint64_t)K;
                    }
                }
                if (a.group) {
                    // group ids are numbered by first position (group[p] <= p),
                    // so a backward sweep expands the compact values in place
                    for (int q = V - 1; q >= 0; --q) {
                        const int gq = a.group[q];
                        r8[q] = gq < 0 ? a.tmpl[q] : r8[gq];
                    }
                }
                if (a.genes_out) {
                    uint8_t *o = a.genes_out + (c0 + tid) * (int64_t)V;
                    for (int i = 0; i < V; ++i) o[i] = r8[i];
                }
            }
        } else {
            const int64_t bytes = (int64_t)rows * a.ld;
            const uint8_t *src = a.genes + c0 * a.ld;
            if (bulk && bytes > 0 && (bytes & 15) == 0) {
                if (tid == 0) bulk_g2s(gtile, src, (uint32_t)bytes, bar);
                mbar_wait(bar, phase);
                phase ^= 1u;
            } else {
                for (int64_t b = tid; b < bytes; b += T) gtile[b] = src[b];
            }
        }
        __syncthreads();

        // ---- the list scheduler of one candidate (heuristics.py:127-143)
        const int li = tid;
        const uint8_t *grow = gtile + (int64_t)li * a.ld_s;
        double *ecol = ends + li;
        typename DevStateSel<KT>::type avail, mem;
        if constexpr (KT == 0) {
            avail.col = kstate + li;
            avail.stride = lanes;
            avail.K = K;
            mem.col = kstate + (int64_t)K * lanes + li;
            mem.stride = lanes;
            mem.K = K;
        }
        avail.zero();
        if (flags & F_MEM) mem.zero();
        double ms = 0.0;
        int st = 0, bad = 0;
        const int64_t cand = c0 + li;
        for (int i = 0; i < V; ++i) {
            const NodeRec nr = nodes[i];
            int d = grow[i];
            bad |= d >= K;
            d = d < K ? d : 0;
            if (flags & F_OKL) {  // try_place batch-size check, :96
                if (!okL[d] && !st) st = HS_ST_BATCH;
            }
            double mcur = 0.0;
            if (flags & F_MEM) {  // memory check, :98-100
                mcur = mem.get(d);
                if (mcur + extra[i] > cap[d] && !st) st = HS_ST_MEMORY;
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
            if (CLASS && nolink && !st) st = HS_ST_LINK;
            const double du = dur[i * K + d];
            if (flags & F_MISS) {  // LatencyTable.get raises, core.py:169
                if (!dur_ok[i * K + d] && !st) st = HS_ST_MISSING;
            }
            const double s = pymax(r, avail.get(d));  // _slot, :80-84
            const double e = s + du;
            if (a.starts && li < rows) a.starts[cand * V + i] = s;
            if (nr.out_slot >= 0) ecol[nr.out_slot] = e;
            avail.set(d, e);
            if (flags & F_MEM) mem.set(d, mcur + extra[i]);
            if (flags & F_NAN) ms = pymax(ms, e);
        }
        if (!(flags & F_NAN)) {
            // ends per device are non-decreasing without NaN: the makespan
            // is the largest device-available time
            for (int k = 0; k < K; ++k) ms = pymax(ms, avail.get(k));
        }
        if (bad) st = HS_ST_GENE;
        if (st) ms = st >= HS_ST_MISSING ? __longlong_as_double(0x7ff8000000000000ll) : kInf;
        if (li < rows) {
            if (a.makespan) a.makespan[cand] = ms;
            if (a.status) a.status[cand] = (uint8_t)st;
            const double key = (ms != ms) ? kInf : ms;
            const int64_t gidx = a.index_base + cand;
            if (best_less(key, gidx, bc, bi)) {
                bc = key;
                bi = gidx;
            }
        }
    }
    if (a.best) reduce_best(bc, bi, a.partial, a.ticket, a.best);
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

// ---------------------------------------------------------------------------
// launchers

static int cuda_fail(cudaError_t e, std::string *err, const char *what) {
    if (err) *err = std::string(what) + ": " + cudaGetErrorString(e);
    return HS_ECUDA;
}

template <int KT, bool CLASS>
static void *eval_fn() {
    return (void *)eval_kernel<KT, CLASS>;
}

static void *pick_eval(int kt, bool cls) {
    switch (kt) {
        case 2: return cls ? eval_fn<2, true>() : eval_fn<2, false>();
        case 3: return cls ? eval_fn<3, true>() : eval_fn<3, false>();
        case 4: return cls ? eval_fn<4, true>() : eval_fn<4, false>();
        default: return cls ? eval_fn<0, true>() : eval_fn<0, false>();
    }
}

int eval_occupancy(int kt, bool cls, int T, size_t smem, int *blocks) {
    void *fn = pick_eval(kt, cls);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return HS_ECUDA;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, fn, T, smem) !=
        cudaSuccess)
        return HS_ECUDA;
    return HS_OK;
}

int launch_eval(const DevState &ds, bool cls, const EvalParams &p, int grid,
                cudaStream_t stream, std::string *err) {
    void *fn = pick_eval(ds.kt, cls);
    cudaError_t e = cudaFuncSetAttribute(
        fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ds.smem);
    if (e != cudaSuccess) return cuda_fail(e, err, "cudaFuncSetAttribute");
    void *args[] = {(void *)&p};
    e = cudaLaunchKernel(fn, dim3(grid), dim3(ds.T), args, ds.smem, stream);
    if (e != cudaSuccess) return cuda_fail(e, err, "eval launch");
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
