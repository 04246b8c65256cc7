// Shared between the ahead-of-time evaluator (kernels.cu, nvcc) and the
// per-graph specialised evaluator (jit.cpp, NVRTC): plain-old-data layouts
// and the CTA tile driver -- genome staging (TMA bulk copy or on-device
// generation), per-lane evaluation via a Body, outputs, and the fused
// first-index argmin. Self-contained: no standard headers under NVRTC.
#pragma once

typedef long long hs_i64;
typedef unsigned long long hs_u64;
typedef unsigned int hs_u32;
typedef unsigned short hs_u16;
typedef unsigned char hs_u8;

namespace hsk {

// Byte offsets of the sections of the device plan blob.
struct DevLayout {
    hs_i64 node, edge, dur, dur_ok, extra, ctab, bclass, cap, okL;
    hs_i64 cp_fast, cp_fast_ok, cp_task, cp_pred_off, cp_pred_pos;
    hs_i64 rc_succ_off, rc_succ, rc_pred_off, rc_pred, rc_order;
    hs_i64 total;
    hs_i64 eval_bytes;  // [0, eval_bytes) = evaluator tables, 16-aligned
    // batched-variant plans: option table [n_opt][P] of {dev, lo, hi, size}
    // (int32 x4), parts per option [n_opt], durations [V][n_opt][P] + flags
    hs_i64 bopt, bnp, bdur, bdur_ok;
};

// One predecessor relaxation: `slot` = the predecessor's end-time slot
// (element offset in the [slot][lane] array after per-device scaling),
// `gpos` = its genome position. UNIFORM comm: `c` = om_p / beta; CLASS
// comm: `crow` = p * n_classes row into ctab.
struct alignas(16) EdgeRec {
    int slot;
    int gpos;
    union {
        double c;
        hs_i64 crow;
    };
};

// One placement, in genome order.
struct alignas(16) NodeRec {
    int e_begin, e_end;
    int out_slot;  // -1: nothing reads this end time
    int pad;
};

struct Best {
    double cost;
    hs_i64 index;
};

// runtime-uniform feature flags of the evaluator
enum : hs_u32 {
    F_MEM = 1u,   // capacity can bind (heuristics.py:98-100)
    F_OKL = 2u,   // some device lacks batch size L (heuristics.py:96)
    F_MISS = 4u,  // some (task, dev, L) latency entry is missing
    F_NAN = 8u,   // a NaN can reach a time: keep the running makespan max
};

// status codes (include/hetsched_b200.h)
enum { ST_OK = 0, ST_BATCH = 1, ST_MEMORY = 2, ST_LINK = 3, ST_MISSING = 4,
       ST_GENE = 5 };

struct EvalParams {
    const hs_u8 *blob;  // device plan blob
    DevLayout lay;
    hs_i64 eval_bytes;
    int V, K;
    int gene_range;     // genes are in [0, gene_range): K, or n_opt (batched)
    int n_opt, P;       // batched-variant plans
    int n_cls;
    hs_u32 flags;
    int plan_smem;
    int lanes, ld_s, slots;
    int bulk;           // genome tiles may use cp.async.bulk
    int packed;         // 1: genes arrive 2 bits each (K <= 4); 2: base-3,
                        // 5 per byte (K <= 3); `ld` bytes/row
    const hs_u8 *genes;
    hs_i64 n, ld;
    int gen;            // 1 hash-random, 2 enumerate (K6); 0 staged genes
    hs_u64 seed;
    hs_i64 first;
    const hs_u8 *tmpl;  // [V] fixed genes where group < 0
    const short *group; // [V] group per position (null: identity)
    int n_groups;
    double *makespan;
    hs_u8 *status;
    double *starts;     // trace [n][V]
    hs_u8 *genes_out;   // [n][V]
    Best *best;
    Best *partial;      // [grid]
    hs_u32 *ticket;
    hs_i64 index_base;
    hs_i64 smem_tile2;  // second genome tile (double buffering), 0 = none
    int sanitize;       // clamp staged genes to < gene_range, flag overflows
    hs_i64 smem_tile;   // byte offsets in shared memory: genome tile,
    hs_i64 smem_ends;   // [slot][lane] end times,
    hs_i64 smem_kstate; // [2K][lane] device state (generic K)
    // global-memory tier of the end-time slots (graphs whose live end times
    // do not fit shared memory): CTA b owns ends_g[b * ends_g_cta ...],
    // laid out [slot][lane] like the shared-memory slots (coalesced)
    double *ends_g;
    hs_i64 ends_g_cta;
};

// (1+1) EA accept chain (K9): every child's mutations, drawn on the host
struct EaParams {
    hs_u8 *parent;        // [V] in: start genome, out: final genome
    double cur_fit;       // fitness of the start genome
    const int *moff;      // [budget + 1] CSR offsets into mpos / mval
    const int *mpos;      // mutated genome positions
    const hs_u8 *mval;    // new genes
    int budget;
    int two_level;        // evaluate children of child j speculatively
    // chained chunks (hs_ea_run_chunk): fitness read from cur_in, counters
    // accumulated into info, nothing done when an earlier chunk raised
    const double *cur_in;
    int first_child, accumulate;
    double *out_fit;      // [1] final fitness
    int *info;            // [4] accepted, rounds, raising child (-1), status
    // independent chains (hs_ea_run_multi): CTA c runs chain c with its
    // parent at parent + c * chain_stride, its CSR offsets at moff + c *
    // (budget + 1) (absolute indices into mpos / mval), out_fit + c and
    // info + 4 c; 0 = one chain
    hs_i64 chain_stride;
};

// simulated annealing (K10); all state in/out so a run can resume
struct SaParams {
    hs_u8 *genes;      // [V] current genome (in/out)
    hs_u8 *best;       // [V] best-ever genome (in/out)
    hs_u64 *rng;       // [4] PCG64 state lo, hi, increment lo, hi (in/out)
    hs_u32 *buf;       // [2] has_uint32, cached upper half (in/out)
    double *f;         // [5] cur, best, temp (in/out); stop 3: cand, u
    int *istate;       // [7] step, k (in/out); stop (0 done, 2 raised, 3
                       // host decides), raised status, stop 3: pos, new;
                       // rounds (accumulated)
    int *spos;         // [window] speculative moves
    hs_u8 *snew;
    double *sfit;      // [window] speculative fitness, status
    hs_u8 *sst;
    double alpha;
    int n_dev, budget, window;
    int host_exp;      // test hook: hand every Metropolis test to the host
    // independent chains (hs_sa_run_multi): CTA c runs chain c with genes /
    // best at + c * chain_stride, rng + 4c, buf + 2c, f + 8c, istate + 8c and
    // its own speculation scratch (+ c * spec_stride); 0 = one chain
    hs_i64 chain_stride;
    // speculation scratch entries per chain: window (base steps) + 32 (the
    // second level's continuation warp: two branches of 16)
    hs_i64 spec_stride;
    int two_level;     // second level: continuation steps per branch (0: off)
};

#if defined(__CUDACC__) || defined(__CUDACC_RTC__)

__device__ __forceinline__ double kinf() { return __longlong_as_double(0x7ff0000000000000ll); }
__device__ __forceinline__ double knan() { return __longlong_as_double(0x7ff8000000000000ll); }

__device__ __forceinline__ double pymax(double a, double b) {
    // Python max(a, b): a unless b > a (NaN compares false: a)
    double r;
    asm("{\n .reg .pred p;\n setp.gt.f64 p, %2, %1;\n selp.f64 %0, %2, %1, p;\n}"
        : "=d"(r) : "d"(a), "d"(b));
    return r;
}

// Tensor-memory tier of the specialised kernel's end-time slots: each
// thread owns one TMEM lane (its warp's lane quadrant) and a band of
// columns; a double is two 32-bit columns. tcgen05.ld/st are asynchronous:
// loads are waited before use (tm_wait_ld, registers tied to the wait),
// stores are waited before any later load of the same columns (tm_wait_st).
__device__ __forceinline__ void tm_st2(hs_u32 addr, double v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};"
                 ::"r"(addr), "r"(__double2loint(v)), "r"(__double2hiint(v)) : "memory");
}
// end time + producer device (4 columns: lo, hi, device, unused)
__device__ __forceinline__ void tm_st4(hs_u32 addr, double v, int dev) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %3};"
                 ::"r"(addr), "r"(__double2loint(v)), "r"(__double2hiint(v)), "r"(dev)
                 : "memory");
}
__device__ __forceinline__ void tm_ld2(hs_u32 addr, hs_u32 &lo, hs_u32 &hi) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                 : "=r"(lo), "=r"(hi) : "r"(addr) : "memory");
}
__device__ __forceinline__ void tm_wait_st() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ double tm_val(hs_u32 lo, hs_u32 hi) {
    return __hiloint2double((int)hi, (int)lo);
}

// (p && v > r) ? v : r -- one compare with a predicate input and a 64-bit
// select (the specialised kernel's dominance-pruned relaxation term)
__device__ __forceinline__ double maxsel(double r, bool p, double v) {
    // one compare with the predicate folded in (setp.gt.and) + one select
    double out;
    asm("{\n .reg .pred q, s;\n setp.ne.b32 q, %3, 0;\n"
        " setp.gt.and.f64 s, %2, %1, q;\n selp.f64 %0, %2, %1, s;\n}"
        : "=d"(out) : "d"(r), "d"(v), "r"((int)p));
    return out;
}

// Python max(a, b) for a, b >= +0.0 and not NaN: the binary64 bit patterns
// of non-negative doubles order like the values (ALU compare, not FP64)
__device__ __forceinline__ double pymax_nn(double a, double b) {
    return __double_as_longlong(b) > __double_as_longlong(a) ? b : a;
}

// four genes (bytes <= 3) -> 8 bits, byte b at bits 2b..2b+1
__device__ __forceinline__ hs_u32 pack4(hs_u32 w) {
    const hs_u32 x = w | (w >> 6);
    return (x | (x >> 12)) & 0xFFu;
}
__device__ __forceinline__ hs_u32 pack16(hs_u32 a, hs_u32 b, hs_u32 c, hs_u32 d) {
    return pack4(a) | (pack4(b) << 8) | (pack4(c) << 16) | (pack4(d) << 24);
}

// branch-free select (kept as FSEL pairs: the specialised code relies on it
// to stay divergence free when lanes map tasks to different devices)
__device__ __forceinline__ double dsel(bool p, double a, double b) {
    double r;
    asm("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n selp.f64 %0, %1, %2, q;\n}"
        : "=d"(r) : "d"(a), "d"(b), "r"((int)p));
    return r;
}

// Shared-memory accesses the optimiser cannot see through. The specialised
// kernels keep per-device state at A + d * T (d = the lane's gene): if the
// front end could relate those addresses it would rewrite the array into
// K-way select chains per task -- super-linear compile time for K ~ 30.
// No memory clobber: the regions accessed this way are accessed only this
// way, so ordinary loads and stores may still be scheduled around them.
__device__ __forceinline__ double ld_shared_f64(hs_u32 a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void st_shared_f64(hs_u32 a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v));
}

// branch-free status update: keep the first failing check's code (the
// optimiser must not turn hundreds of these into nested branches)
__device__ __forceinline__ int first_status(int st, bool fail, int code) {
    int r;
    asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n selp.b32 %0, %1, %3, q;\n}"
        : "=r"(r) : "r"(code), "r"((int)(fail && st == 0)), "r"(st));
    return r;
}

__device__ __forceinline__ bool best_less(double c1, hs_i64 i1, double c2, hs_i64 i2) {
    return c1 < c2 || (c1 == c2 && i1 < i2);
}

__device__ __forceinline__ hs_u64 splitmix64(hs_u64 z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ hs_u32 smem_addr(const void *p) {
    return (hs_u32)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_inval(hs_u64 *bar) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init(hs_u64 *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// TMA 1-D bulk copy global -> shared, completion on the mbarrier
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, hs_u32 bytes,
                                         hs_u64 *bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
                 "[%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(hs_u64 *bar, hs_u32 phase) {
    asm volatile("{\n"
                 ".reg .pred p;\n"
                 "WAIT_%=:\n"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                 "@!p bra WAIT_%=;\n"
                 "}\n" ::"r"(smem_addr(bar)), "r"(phase) : "memory");
}

// lexicographic (cost, index) min across the CTA, then across CTAs through
// `partial` + a ticket: the last CTA to finish writes *best.
__device__ __forceinline__ void warp_best(double &bc, hs_i64 &bi) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double oc = __shfl_down_sync(0xffffffffu, bc, o);
        const hs_i64 oi = __shfl_down_sync(0xffffffffu, bi, o);
        if (best_less(oc, oi, bc, bi)) {
            bc = oc;
            bi = oi;
        }
    }
}

static __device__ __noinline__ void reduce_best(double bc, hs_i64 bi, Best *partial,
                                         hs_u32 *ticket, Best *best) {
    __shared__ double s_c[32];
    __shared__ hs_i64 s_i[32];
    __shared__ int s_last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = (blockDim.x + 31) >> 5;
    warp_best(bc, bi);
    if (lane == 0) {
        s_c[warp] = bc;
        s_i[warp] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < nw; ++w)
            if (best_less(s_c[w], s_i[w], bc, bi)) {
                bc = s_c[w];
                bi = s_i[w];
            }
        partial[blockIdx.x].cost = bc;
        partial[blockIdx.x].index = bi;
        __threadfence();
        const hs_u32 t = atomicAdd(ticket, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    bc = kinf();
    bi = 0x7fffffffffffffffll;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
        const double c = ((volatile double *)&partial[b].cost)[0];
        const hs_i64 i = ((volatile hs_i64 *)&partial[b].index)[0];
        if (best_less(c, i, bc, bi)) {
            bc = c;
            bi = i;
        }
    }
    warp_best(bc, bi);
    __syncthreads();
    if (lane == 0) {
        s_c[warp] = bc;
        s_i[warp] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < nw; ++w)
            if (best_less(s_c[w], s_i[w], bc, bi)) {
                bc = s_c[w];
                bi = s_i[w];
            }
        best->cost = bc;
        best->index = bi == 0x7fffffffffffffffll ? -1 : bi;
        *ticket = 0;  // reusable by the next launch on this stream
    }
}

// four bytes b -> four genes (b * K) >> 8 (K <= 256): even and odd bytes
// multiplied in 16-bit lanes, the high byte of each lane kept
__device__ __forceinline__ hs_u32 gen_bytes_to_genes(hs_u32 x, hs_u32 K) {
    const hs_u32 e = x & 0x00FF00FFu, o = (x >> 8) & 0x00FF00FFu;
    return (((e * K) >> 8) & 0x00FF00FFu) | ((o * K) & 0xFF00FF00u);
}

// K6: on-device candidate rows (oracle/hs_oracle.py::gen_genes, or
// mixed-radix enumeration), expanded over the group map.
__device__ __forceinline__ void gen_row(const EvalParams &a, hs_u8 *r8, hs_i64 cidx) {
    const int NG = a.n_groups, K = a.gene_range, V = a.V;
    const hs_u64 c = (hs_u64)cidx;
    if (a.gen == 3) {
        // neighbours of the incumbent a.tmpl: index < NG*K moves one group
        // (j -> va), the rest two groups ((j*NG + l)*K + va)*K + vb (j >= l
        // leaves l alone); positions outside every group (group -1) keep
        // the template, so "no second group" is -2
        int j, l = -2, va, vb = 0;
        const hs_u64 singles = (hs_u64)NG * (hs_u64)K;
        if (c < singles) {
            j = (int)(c / (hs_u64)K);
            va = (int)(c % (hs_u64)K);
        } else {
            hs_u64 p = c - singles;
            vb = (int)(p % (hs_u64)K);
            p /= (hs_u64)K;
            va = (int)(p % (hs_u64)K);
            p /= (hs_u64)K;
            l = (int)(p % (hs_u64)NG);
            j = (int)(p / (hs_u64)NG);
            if (l <= j) l = -2;
        }
        for (int q = 0; q < V; ++q) {
            const int gq = a.group[q];
            r8[q] = gq == j ? (hs_u8)va : (gq == l ? (hs_u8)vb : a.tmpl[q]);
        }
        for (int q = V; q < ((V + 3) & ~3); ++q) r8[q] = 0;
        return;
    }
    if (a.gen == 1) {
        // one splitmix64 per candidate, then per 8 genes one 64-bit
        // multiply-xorshift of h + (w+1) * C; each byte b of it gives the
        // gene (b * K) >> 8, four at a time in two 16-bit-lane products
        // (b * K < 2^16 for K <= 256): ~4 instructions per gene where a
        // splitmix64 per 4 genes cost ~8 (the generator was a quarter of the
        // generated-candidate evaluation's issue slots)
        const int W4 = (NG + 3) >> 2, W8 = (W4 + 1) >> 1;
        hs_u32 *row = reinterpret_cast<hs_u32 *>(r8);
        const hs_u64 h = splitmix64(a.seed + (c + 1ull) * 0x9E3779B97F4A7C15ull);
        const hs_u32 Ku = (hs_u32)K;
        hs_u64 zc = h;
        for (int w = 0; w < W8; ++w) {
            zc += 0xD1B54A32D192ED03ull;
            hs_u64 z = zc ^ (zc >> 32);
            z *= 0xD6E8FEB86659FD93ull;
            z ^= z >> 32;
            const hs_u32 lo = (hs_u32)z, hi = (hs_u32)(z >> 32);
            row[2 * w] = gen_bytes_to_genes(lo, Ku);
            if (2 * w + 1 < W4) row[2 * w + 1] = gen_bytes_to_genes(hi, Ku);
        }
    } else if (c < (1ull << 32)) {
        hs_u32 x = (hs_u32)c;
        for (int j = 0; j < NG; ++j) {
            r8[j] = (hs_u8)(x % (hs_u32)K);
            x /= (hs_u32)K;
        }
    } else {
        hs_u64 x = c;
        for (int j = 0; j < NG; ++j) {
            r8[j] = (hs_u8)(x % (hs_u64)K);
            x /= (hs_u64)K;
        }
    }
    if (a.group) {
        // group ids are numbered by first position (group[p] <= p), so a
        // backward sweep expands the compact values in place
        for (int q = V - 1; q >= 0; --q) {
            const int gq = a.group[q];
            r8[q] = gq < 0 ? a.tmpl[q] : r8[gq];
        }
    }
}

// Issue the TMA bulk copy of a tile's genome rows (one elected thread).
__device__ __forceinline__ void issue_tile(const EvalParams &a, hs_i64 tile, hs_u8 *dst,
                                           hs_u64 *bar) {
    const hs_i64 c0 = tile * a.lanes;
    const hs_i64 left = a.n - c0;
    const hs_i64 rows = left < a.lanes ? left : a.lanes;
    bulk_g2s(dst, a.genes + c0 * a.ld, (hs_u32)(rows * a.ld), bar);
}

// The CTA tile loop. `body.run(row, lane, cand, valid, gene_bad, ms, st)`
// evaluates the lane's candidate from its staged genome row; `gene_bad` is
// set when the row was sanitised (a.sanitize) and held a gene >= K.
template <class Body>
__device__ __forceinline__ void eval_tiles(const EvalParams &a, hs_u8 *smem, Body &body) {
    hs_u64 *bar = reinterpret_cast<hs_u64 *>(smem);  // two mbarriers
    hs_u8 *gtile = smem + a.smem_tile;
    // double-buffered TMA staging: tile t+grid streams in while t computes
    const bool dbuf = a.smem_tile2 != 0;
    const int T = blockDim.x, tid = threadIdx.x;
    const int lanes = a.lanes;
    if (tid == 0) {
        mbar_init(bar);
        mbar_init(bar + 1);
    }
    __syncthreads();
    double bc = kinf();
    hs_i64 bi = 0x7fffffffffffffffll;
    hs_u32 phase0 = 0, phase1 = 0;
    const hs_i64 ntiles = (a.n + lanes - 1) / lanes;
    if (dbuf && tid == 0 && (hs_i64)blockIdx.x < ntiles)
        issue_tile(a, blockIdx.x, gtile, bar);
    int it = 0;
    for (hs_i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const hs_i64 c0 = tile * lanes;
        const hs_i64 left = a.n - c0;
        const int rows = left < lanes ? (int)left : lanes;
        hs_u8 *cur = gtile;
        if (dbuf) {
            const int b = it & 1;
            cur = b ? smem + a.smem_tile2 : gtile;
            if (b) {
                mbar_wait(bar + 1, phase1);
                phase1 ^= 1u;
            } else {
                mbar_wait(bar, phase0);
                phase0 ^= 1u;
            }
            __syncthreads();  // every lane is done with the other buffer
            if (tid == 0 && tile + gridDim.x < ntiles)
                issue_tile(a, tile + gridDim.x, b ? gtile : smem + a.smem_tile2,
                           b ? bar : bar + 1);
        } else {
            // generated rows are written and read by their own lane only:
            // no CTA barrier, so generation (IMAD pipe) of one warp overlaps
            // the evaluation (ALU / FP64 / LSU) of the others
            if (!a.gen) __syncthreads();  // the previous tile is no longer read
            if (a.gen) {
                if (tid < rows) {
                    hs_u8 *r8 = gtile + (hs_i64)tid * a.ld_s;
                    gen_row(a, r8, a.first + c0 + tid);
                    if (a.genes_out) {
                        hs_u8 *o = a.genes_out + (c0 + tid) * (hs_i64)a.V;
                        for (int i = 0; i < a.V; ++i) o[i] = r8[i];
                    }
                }
            } else {
                const hs_i64 bytes = (hs_i64)rows * a.ld;
                const hs_u8 *src = a.genes + c0 * a.ld;
                // packed rows land in the last bytes of the tile and are
                // expanded in place (all rows read before any row is written)
                hs_u8 *dst = a.packed ? gtile + (hs_i64)lanes * a.ld_s - (hs_i64)lanes * a.ld
                                      : gtile;
                if (a.bulk && bytes > 0 && (bytes & 15) == 0) {
                    if (tid == 0) bulk_g2s(dst, src, (hs_u32)bytes, bar);
                    mbar_wait(bar, phase0);
                    phase0 ^= 1u;
                } else {
                    for (hs_i64 b = tid; b < bytes; b += T) dst[b] = src[b];
                }
                if (a.packed == 2) {
                    __syncthreads();
                    // base-3 genes, 5 per byte (least significant digit
                    // first): 4 row bytes -> 20 genes -> five 4-gene words
                    hs_u32 pk[64];
                    const int nb = (int)a.ld;
                    const int nw = (nb + 3) >> 2;
                    const hs_u8 *prow = dst + (hs_i64)tid * a.ld;
#pragma unroll 4
                    for (int w = 0; w < nw && w < 64; ++w) {
                        hs_u32 x = 0u;
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (tid < rows && 4 * w + j < nb)
                                x |= (hs_u32)prow[4 * w + j] << (8 * j);
                        pk[w] = x;
                    }
                    __syncthreads();
                    hs_u32 *orow = reinterpret_cast<hs_u32 *>(gtile + (hs_i64)tid * a.ld_s);
                    const int nout = a.ld_s >> 2;
#pragma unroll 2
                    for (int w = 0; w < nw && w < 64; ++w) {
                        const hs_u32 x = pk[w];
                        hs_u32 o[5] = {0u, 0u, 0u, 0u, 0u};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            hs_u32 b = (x >> (8 * j)) & 0xFFu;
#pragma unroll
                            for (int d = 0; d < 5; ++d) {
                                // b / 3 for b < 256; the last digit keeps the
                                // quotient whole, so a byte >= 243 yields a
                                // gene >= 3 (flagged out of range)
                                const hs_u32 q = (b * 171u) >> 9;
                                const int gi = 5 * j + d;
                                o[gi >> 2] |= (d < 4 ? b - 3u * q : b) << (8 * (gi & 3));
                                b = q;
                            }
                        }
#pragma unroll
                        for (int k = 0; k < 5; ++k)
                            if (5 * w + k < nout) orow[5 * w + k] = o[k];
                    }
                } else if (a.packed) {
                    __syncthreads();
                    // 2-bit genes, 16 per word: word w -> four 4-gene words
                    hs_u32 pk[64];
                    const int nw = (int)(a.ld >> 2);
                    const hs_u32 *prow =
                        reinterpret_cast<const hs_u32 *>(dst + (hs_i64)tid * a.ld);
#pragma unroll 4
                    for (int w = 0; w < nw && w < 64; ++w) pk[w] = tid < rows ? prow[w] : 0u;
                    __syncthreads();
                    hs_u32 *orow = reinterpret_cast<hs_u32 *>(gtile + (hs_i64)tid * a.ld_s);
                    const int nout = a.ld_s >> 2;
#pragma unroll 4
                    for (int w = 0; w < nw && w < 64; ++w) {
                        const hs_u32 x = pk[w];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int o = 4 * w + j;
                            if (o < nout) {
                                const hs_u32 b = (x >> (8 * j)) & 0xFFu;
                                orow[o] = (b & 3u) | ((b & 0xCu) << 6) | ((b & 0x30u) << 12) |
                                          ((b & 0xC0u) << 18);
                            }
                        }
                    }
                }
            }
            if (!a.gen) __syncthreads();
        }
        const int li = tid;
        const hs_i64 cand = c0 + li;
        const bool valid = li < rows;
        hs_u8 *row = cur + (hs_i64)li * a.ld_s;
        int gene_bad = 0;
        if (a.sanitize) {
            // one pass over the lane's own row: flag genes >= K, clamp every
            // byte to K-1 so the specialised code can index by gene freely
            // (rows past the last candidate hold stale bytes)
            // read-only check; the clamping rewrite only for a row that
            // holds a gene >= K (the rare error path: status 5)
            hs_u32 *w = reinterpret_cast<hs_u32 *>(row);
            const int nw = (a.V + 3) >> 2;
            const hs_u32 kmax = (hs_u32)(a.gene_range - 1) * 0x01010101u;
            const int tail = a.V & 3;
            hs_u32 any = 0u, over_tail = 0u;
            for (int j = 0; j + 1 < nw; ++j) any |= __vcmpgtu4(w[j], kmax);
            if (nw > 0) {
                over_tail = __vcmpgtu4(w[nw - 1], kmax);
                if (tail) over_tail &= (1u << (8 * tail)) - 1u;
            }
            gene_bad = (any | over_tail) != 0u;
            // bytes past V in the last word are clamped too (the body may
            // read whole words)
            if (gene_bad || __vcmpgtu4(nw > 0 ? w[nw - 1] : 0u, kmax))
                for (int j = 0; j < nw; ++j) w[j] = __vminu4(w[j], kmax);
        }
        double ms;
        int st;
        body.run(row, li, cand, valid, gene_bad, ms, st);
        if (valid) {
            if (a.makespan) a.makespan[cand] = ms;
            if (a.status) a.status[cand] = (hs_u8)st;
            const double key = (ms != ms) ? kinf() : ms;
            const hs_i64 gidx = a.index_base + cand;
            if (best_less(key, gidx, bc, bi)) {
                bc = key;
                bi = gidx;
            }
        }
    }
    // the mbarriers' lifetime ends with the tile loop (no copy in flight):
    // invalidate them before the shared memory is reused
    __syncthreads();
    if (tid == 0) {
        mbar_inval(bar);
        mbar_inval(bar + 1);
    }
    if (a.best) reduce_best(bc, bi, a.partial, a.ticket, a.best);
}

// numpy Generator(PCG64) on the device (oracle restatement: rng.py): the
// 128-bit LCG step then the XSL-RR output; 32-bit draws take the buffered
// upper half of the previous word; integers(high) is Lemire's method on
// 32-bit draws; random() = (word >> 11) * 2^-53.
struct Pcg64 {
    hs_u64 slo, shi, ilo, ihi;
    hs_u32 has, cached;
    __device__ __forceinline__ hs_u64 next64() {
        const hs_u64 ml = 4865540595714422341ull, mh = 2549297995355413924ull;
        const hs_u64 lo = slo * ml;
        hs_u64 hi = __umul64hi(slo, ml) + slo * mh + shi * ml;
        const hs_u64 lo2 = lo + ilo;
        hi += ihi + (lo2 < lo ? 1ull : 0ull);
        slo = lo2;
        shi = hi;
        const hs_u64 x = hi ^ lo2;
        const unsigned rot = (unsigned)(hi >> 58);
        return (x >> rot) | (x << ((64u - rot) & 63u));
    }
    __device__ __forceinline__ hs_u32 next32() {
        if (has) {
            has = 0;
            return cached;
        }
        const hs_u64 x = next64();
        has = 1;
        cached = (hs_u32)(x >> 32);
        return (hs_u32)x;
    }
    __device__ __forceinline__ int integers(hs_u32 high) {
        if (high <= 1) return 0;
        hs_u64 m = (hs_u64)next32() * high;
        hs_u32 left = (hs_u32)m;
        if (left < high) {
            const hs_u32 thr = (0xFFFFFFFFu - (high - 1)) % high;
            while (left < thr) {
                m = (hs_u64)next32() * high;
                left = (hs_u32)m;
            }
        }
        return (int)(m >> 32);
    }
    __device__ __forceinline__ double random() {
        return (double)(next64() >> 11) * (1.0 / 9007199254740992.0);
    }
};

// K10 driver: simulated annealing (heuristics.py:259-299) in one launch of
// a single CTA per chain. Rounds of speculation: thread 0 draws the next k
// steps' moves assuming each is rejected after a random() draw (a finite,
// worse candidate -- the only way a step continues a round); the lanes
// evaluate those k candidates against the current genome; thread 0 then
// replays the steps with the real generator and ends the round at the first
// acceptance or infinite candidate (where the speculated draws diverge).
// Second level (e.two_level steps, when one more warp fits): the commonest
// round ends with step 0 accepted, so one extra warp evaluates further
// steps on top of step 0's move for each way step 0 can be accepted
// (delta <= 0: no random() drawn; delta > 0 and the Metropolis test passed:
// random() drawn) -- lanes 0-15 and 16-31 --, their moves drawn by threads
// 32 and 64 from the two generator states while thread 0 draws the base
// steps; such a round goes on into the matching branch and can make two
// acceptances. Metropolis needs exp():
// when u lies within a few ulp of the device exp the step is handed back to
// the host (CPython's math.exp decides; never observed in practice), so the
// trajectory is the reference's exactly. Shared by the AOT kernel
// (kernels.cu) and the specialised module (jit.cpp).
template <class Body>
__device__ __forceinline__ void sa_chain(const EvalParams &a, const SaParams &e0, hs_u8 *smem,
                                         Body &body) {
    __shared__ int s_k, s_step, s_go, s_apos, s_apos2, s_pos0, s_new0;
    __shared__ hs_u64 s_q[2][4];  // branch starts: after step 0's draws (A), + random() (B)
    __shared__ hs_u32 s_qb[2][2];
    SaParams e = e0;  // this CTA's chain
    const hs_i64 sp = e0.spec_stride;
    if (e0.chain_stride) {
        const hs_i64 c = blockIdx.x;
        e.genes += c * e0.chain_stride;
        e.best += c * e0.chain_stride;
        e.rng += 4 * c;
        e.buf += 2 * c;
        e.f += 8 * c;
        e.istate += 8 * c;
        e.spos += c * sp;
        e.snew += c * sp;
        e.sfit += c * sp;
        e.sst += c * sp;
    }
    const int l = threadIdx.x;
    hs_u8 *row = smem + a.smem_tile + (hs_i64)l * a.ld_s;
    hs_u8 *genes = e.genes;
    // a lane's row stays the current genome between rounds: it undoes its
    // own move(s) and takes the round's accepted moves (s_apos, s_apos2)
    // instead of re-copying V bytes; a lane that sat a round out copies in
    // full
    int prev = -1, prev0 = -1;
    bool synced = false;
    // the row's bytes past V stay 0 (the specialised body may read whole
    // words of the row and rely on every byte being a valid gene)
    for (int i = a.V; i < a.ld_s; ++i) row[i] = 0;
    const int V = a.V, budget = e.budget, W = e.window;
    const hs_u32 nd1 = (hs_u32)(e.n_dev - 1);
    Pcg64 r;
    double cur = 0.0, bestf = 0.0, temp = 0.0;
    int step = 0, stop = 0, rounds = 0;
    if (e.istate[2] != 0) return;  // a chained earlier launch stopped
    if (l == 0) {
        r.slo = e.rng[0];
        r.shi = e.rng[1];
        r.ilo = e.rng[2];
        r.ihi = e.rng[3];
        r.has = e.buf[0];
        r.cached = e.buf[1];
        cur = e.f[0];
        bestf = e.f[1];
        temp = e.f[2];
        step = e.istate[0];
        // the first round's window comes from the caller: at most the
        // scratch arrays' length (e.window <= lanes)
        s_k = e.istate[1] < 1 ? 1 : (e.istate[1] < W ? e.istate[1] : W);
        s_step = step;
        s_go = 1;
        s_apos = s_apos2 = -1;
    }
    __syncthreads();
    auto draw_move = [&](Pcg64 &q, int &pos, int &nw, int pos0, int new0) {
        pos = q.integers((hs_u32)V);
        const int old = pos == pos0 ? new0 : genes[pos];
        nw = old;
        if (e.n_dev > 1) {
            nw = q.integers(nd1);
            if (nw >= old) ++nw;
        }
    };
    for (;;) {
        const int kk = s_k, stp = s_step;
        if (!s_go || stp >= budget) break;
        const int n = kk < budget - stp ? kk : budget - stp;
        const int wb = (n + 31) & ~31;  // first lane after the base warps
        // one more warp: branch A in its lanes 0..15, branch B in 16..31,
        // e.two_level continuation steps each (at most 16)
        const bool lvl2 = e.two_level > 0 && e.n_dev > 1 && wb + 32 <= a.lanes &&
                          budget - stp > 1;
        const int m2 = e.two_level < 16 ? e.two_level : 16;
        const int m = lvl2 ? (m2 < budget - stp - 1 ? m2 : budget - stp - 1) : 0;
        Pcg64 q;
        if (l == 0) {  // speculative moves of the next n steps: step 0 first
            q = r;
            int pos, nw;
            draw_move(q, pos, nw, -1, 0);
            e.spos[0] = pos;
            e.snew[0] = (hs_u8)nw;
            if (lvl2) {
                s_pos0 = pos;
                s_new0 = nw;
                s_q[0][0] = q.slo, s_q[0][1] = q.shi, s_qb[0][0] = q.has, s_qb[0][1] = q.cached;
            }
            (void)q.random();
            if (lvl2) s_q[1][0] = q.slo, s_q[1][1] = q.shi, s_qb[1][0] = q.has, s_qb[1][1] = q.cached;
        }
        if (lvl2) __syncthreads();  // the branch starts are published
        if (l == 0) {  // the remaining base steps
            int pos, nw;
            for (int i = 1; i < n; ++i) {
                draw_move(q, pos, nw, -1, 0);
                e.spos[i] = pos;
                e.snew[i] = (hs_u8)nw;
                (void)q.random();
            }
        } else if (lvl2 && (l == 32 || l == 64)) {
            // the two continuation streams, drawn by warps 1 and 2 while
            // thread 0 draws the base steps
            const int b = l == 32 ? 0 : 1;
            q.slo = s_q[b][0];
            q.shi = s_q[b][1];
            q.ilo = e.rng[2];
            q.ihi = e.rng[3];
            q.has = s_qb[b][0];
            q.cached = s_qb[b][1];
            const int p0 = s_pos0, n0 = s_new0;
            for (int j = 0; j < m; ++j) {
                int pos, nw;
                draw_move(q, pos, nw, p0, n0);
                e.spos[W + 16 * b + j] = pos;
                e.snew[W + 16 * b + j] = (hs_u8)nw;
                (void)q.random();
            }
        }
        __syncthreads();
        const int w0 = l & ~31;
        const bool active = w0 < wb || (lvl2 && w0 == wb);
        if (active) {  // warp-uniform: warps past the window sit out
            if (synced) {
                if (prev0 >= 0) row[prev0] = genes[prev0];
                if (prev >= 0) row[prev] = genes[prev];
                const int ap = s_apos, ap2 = s_apos2;
                if (ap >= 0) row[ap] = genes[ap];
                if (ap2 >= 0) row[ap2] = genes[ap2];
            } else {
                for (int i = 0; i < V; ++i) row[i] = genes[i];
                synced = true;
            }
            prev = prev0 = -1;
            int slot;
            bool valid;
            if (w0 < wb) {
                slot = l;
                valid = l < n;
            } else {
                const int b = (l - wb) >> 4, j = (l - wb) & 15;
                slot = W + 16 * b + j;
                valid = j < m;
                prev0 = e.spos[0];
                row[prev0] = e.snew[0];  // on top of step 0's move
            }
            if (valid) {
                prev = e.spos[slot];
                row[prev] = e.snew[slot];
            }
            double ms = 0.0;
            int st = 0;
            body.run(row, l, stp + slot, valid, 0, ms, st);
            if (valid) {
                e.sfit[slot] = ms;
                e.sst[slot] = (hs_u8)st;
            }
        } else {
            synced = false;
        }
        __syncthreads();
        if (l == 0) {  // replay with the real generator
            bool acc = false, acc0 = false, mh0 = false;
            int i = 0;
            ++rounds;
            s_apos = s_apos2 = -1;
            // one step at scratch slot `slot` (kind: 0 base, 1 continuation);
            // returns true when the round ends here
            auto replay = [&](int slot, int kind) -> bool {
                int pos, nw;
                draw_move(r, pos, nw, -1, 0);
                const double cand = e.sfit[slot];
                if (e.sst[slot] >= ST_MISSING) {  // fitness raised
                    stop = 2;
                    e.istate[3] = e.sst[slot];
                    return true;
                }
                const double delta = cand - cur;
                acc = delta <= 0.0;
                const bool fin = isfinite(cand);
                bool drew = false;
                if (!acc && fin) {
                    const double u = r.random();
                    drew = true;
                    const double ex = exp(-delta / temp);
                    // temp == 0 (cooled to underflow): the reference's
                    // -delta / temp raises ZeroDivisionError -- the host's
                    // Python division decides, as it does for a close call
                    if (e.host_exp || temp == 0.0 || u == 0.0 ||
                        fabs(u - ex) <= ex * 0x1p-48) {
                        stop = 3;  // too close to call against CPython's exp
                        e.istate[4] = pos;
                        e.istate[5] = nw;
                        e.f[3] = cand;
                        e.f[4] = u;
                        return true;
                    }
                    acc = u < ex;
                }
                ++step;
                if (acc) {
                    genes[pos] = (hs_u8)nw;
                    if (kind == 0) s_apos = pos; else s_apos2 = pos;
                    cur = cand;
                    if (cand < bestf) {
                        bestf = cand;
                        for (int j = 0; j < V; ++j) e.best[j] = genes[j];
                    }
                }
                temp *= e.alpha;
                if (kind == 0 && slot == 0) {
                    acc0 = acc;
                    mh0 = drew;
                }
                return acc || !fin;
            };
            for (i = 0; i < n; ++i)
                if (replay(i, 0)) break;
            // step 0 accepted: the round goes on into the matching branch
            if (lvl2 && !stop && acc0 && i == 0) {
                acc = false;
                const int base = W + (mh0 ? 16 : 0);
                for (int j = 0; j < m && step < budget; ++j)
                    if (replay(base + j, 1)) break;
            }
            s_k = acc ? 8 : (2 * kk < W ? 2 * kk : W);
            s_step = step;
            if (stop) s_go = 0;
        }
        __syncthreads();
    }
    if (l == 0) {
        e.rng[0] = r.slo;
        e.rng[1] = r.shi;
        e.buf[0] = r.has;
        e.buf[1] = r.cached;
        e.f[0] = cur;
        e.f[1] = bestf;
        e.f[2] = temp;
        e.istate[0] = step;
        e.istate[1] = s_k;
        e.istate[2] = stop;
        e.istate[6] += rounds;
    }
}

// K9 driver: the whole (1+1) EA accept chain (heuristics.py:302-334) in
// one launch of a single CTA. The EA's mutation stream does not depend on
// fitness, so the host draws every child's mutation list up front (CSR:
// moff/mpos/mval). Rounds: lane l evaluates child j+l = (current parent +
// its mutations); the first lane whose child is not worse (`fit <= cur`,
// the reference's acceptance, :328) -- or whose evaluation raised (status
// >= 4, GraphError in the reference) -- decides the round: its child
// becomes the parent and j moves past it; with no such lane j advances by
// a full round. Children after an acceptance are re-evaluated against the
// new parent in the next round, so the trajectory is the reference's.
template <class Body>
__device__ __forceinline__ void ea_chain(const EvalParams &a, const EaParams &e0, hs_u8 *smem,
                                         Body &body) {
    __shared__ int s_first, s_first2;
    EaParams e = e0;  // this CTA's chain
    if (e0.chain_stride) {
        const hs_i64 c = blockIdx.x;
        e.parent += c * e0.chain_stride;
        e.moff += c * (hs_i64)(e0.budget + 1);
        e.out_fit += c;
        e.info += 4 * c;
        if (e.cur_in) e.cur_in += c;
    }
    __shared__ double s_fit, s_fit2;
    const int l = threadIdx.x;
    hs_u8 *row = smem + a.smem_tile + (hs_i64)l * a.ld_s;
    hs_u8 *parent = e.parent;  // [V], global; written by one lane per acceptance
    if (e.accumulate && e.info[2] >= 0) return;  // an earlier chunk raised
    double cur = e.cur_in ? *e.cur_in : e.cur_fit;
    int acc = 0, rounds = 0, err_child = -1, err_st = 0;
    // children per round: one warp after an acceptance, doubling while
    // rounds reject (whole warps sit a round out: a lone warp's evaluation
    // is the round's latency, and it is shortest without co-issuing warps)
    int k = 32 < a.lanes ? 32 : a.lanes;
    double ms = 0.0;
    int st = 0;
    // a lane's row stays the parent between rounds: it undoes the
    // mutations it applied (its child's, and child j's on the second level)
    // and takes the accepted children's (cacc, cacc2) instead of re-copying
    // V bytes; a lane that sat a round out copies in full
    int bprev = -1, cprev = -1, cacc = -1, cacc2 = -1;
    bool synced = false;
    // the row's bytes past V stay 0 (the specialised body may read whole
    // words of the row and rely on every byte being a valid gene)
    for (int i = a.V; i < a.ld_s; ++i) row[i] = 0;
    for (int j = 0; j < e.budget;) {
        if (l == 0) {
            s_first = a.lanes;
            s_first2 = 32;
        }
        __syncthreads();  // parent / s_first of the previous round settled
        // second level: one more warp evaluates children j+1.. on top of
        // child j, for the case that child j is accepted (the commonest
        // first acceptance) -- then one round makes two acceptances
        const bool lvl2 = e.two_level && k + 32 <= a.lanes;
        const int w0 = l & ~31;
        const int c = w0 < k ? j + l : j + 1 + (l - k);
        const bool valid = c < e.budget && (w0 < k ? l < k : lvl2 && w0 == k);
        if (w0 < k || (lvl2 && w0 == k)) {  // warp-uniform (warp-collective body ops)
            const bool is2 = w0 >= k;
            if (synced) {
                const int undo[4] = {bprev, cprev, cacc, cacc2};
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (undo[u] >= 0)
                        for (int q = e.moff[undo[u]]; q < e.moff[undo[u] + 1]; ++q)
                            row[e.mpos[q]] = parent[e.mpos[q]];
            } else {
                for (int i = 0; i < a.V; ++i) row[i] = parent[i];
                synced = true;
            }
            bprev = cprev = -1;
            if (is2) {  // second level: on top of child j
                bprev = j;
                for (int q = e.moff[j]; q < e.moff[j + 1]; ++q) row[e.mpos[q]] = e.mval[q];
            }
            if (valid) {
                cprev = c;
                for (int q = e.moff[c]; q < e.moff[c + 1]; ++q) row[e.mpos[q]] = e.mval[q];
            }
            body.run(row, l, c, valid, 0, ms, st);
            if (!is2 && valid && (st >= ST_MISSING || ms <= cur)) atomicMin(&s_first, l);
        } else {
            synced = false;
        }
        __syncthreads();
        const int r = s_first;
        ++rounds;
        cacc = cacc2 = -1;
        if (r == a.lanes) {
            j += k;
            k = 2 * k < a.lanes ? 2 * k : a.lanes;
            continue;
        }
        cacc = j + r;
        if (l == r) {
            if (st >= ST_MISSING) {
                s_fit = -1.0;
            } else {
                for (int q = e.moff[c]; q < e.moff[c + 1]; ++q) parent[e.mpos[q]] = e.mval[q];
                s_fit = ms;
            }
        }
        __syncthreads();
        if (s_fit < 0.0) {  // fitness raised: the reference stops here
            err_child = j + r;
            if (l == r) err_st = st;
            break;
        }
        cur = s_fit;
        ++acc;
        const int k1 = k;
        k = 32 < a.lanes ? 32 : a.lanes;
        if (r != 0 || !lvl2) {
            j += r + 1;
            continue;
        }
        // child j was accepted: the second level's children are children
        // j+1.. of the new parent
        if (valid && w0 == k1 && (st >= ST_MISSING || ms <= cur)) atomicMin(&s_first2, l - k1);
        __syncthreads();
        const int r2 = s_first2;
        if (r2 == 32) {
            j += 1 + 32;
            continue;
        }
        if (w0 == k1 && l - k1 == r2) {
            if (st >= ST_MISSING) {
                s_fit2 = -1.0;
            } else {
                for (int q = e.moff[c]; q < e.moff[c + 1]; ++q) parent[e.mpos[q]] = e.mval[q];
                s_fit2 = ms;
            }
        }
        __syncthreads();
        if (s_fit2 < 0.0) {
            err_child = j + 1 + r2;
            if (w0 == k1 && l - k1 == r2) err_st = st;
            break;
        }
        cur = s_fit2;
        ++acc;
        cacc2 = j + 1 + r2;
        j += r2 + 2;
    }
    if (err_st) e.info[3] = err_st;  // the raising lane only
    if (l == 0) {
        e.out_fit[0] = cur;
        if (e.accumulate) {
            e.info[0] += acc;
            e.info[1] += rounds;
            if (err_child >= 0) e.info[2] = e.first_child + err_child;
        } else {
            e.info[0] = acc;
            e.info[1] = rounds;
            e.info[2] = err_child;
        }
    }
}

#endif  // device code

}  // namespace hsk
