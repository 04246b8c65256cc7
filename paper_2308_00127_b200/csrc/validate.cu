// K11: schedule validation on the GPU -- the counterpart of the reference's
// validate_schedule (core.py:206-291), for many schedules per launch (one
// CTA per schedule). Every check is the reference's, in the reference's
// order, and the FIRST violation in that order is reported, so the caller
// can raise the same ScheduleError (GraphError for a missing latency
// entry) with the same message:
//
//   per batch, in batch order (core.py:217-240), thread 0: unknown task /
//   device, size vs inputs, unsupported batch size, negative start, input
//   index range and double assignment (input by input), end = start +
//   latency (a missing entry raises GraphError);
//   then in parallel, each reduced to its first violation by an atomicMin
//   over the reference's iteration order:
//   every (task, input) assigned (tasks x inputs, :242-245),
//   precedence with communication per edge and input (:247-259),
//   pairwise overlap per device, devices in first-appearance order, batches
//   sorted stably by (start, end) (:261-271),
//   preemptive-residency memory per device in hardware order (:273-286,
//   one thread per device: the sum is sequential in batch order),
//   makespan = max end vs the stated objective (:288-291).
//
// All float arithmetic is the reference's binary64 operations (no FMA:
// built with --fmad=false).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hetsched_b200.h"
#include "scratch.hpp"

namespace hs {
int set_error(int code, const std::string &msg);
}

namespace {

struct VTables {
    int V, E, K, n_cols;
    const double *wm, *im, *om;     // [V]
    const int32_t *esrc, *edst;     // [E]
    const double *bw;               // [K*K], <= 0 = no link
    const double *memory;           // [K]
    const int32_t *boff, *bsz;      // device batch sizes
    const double *lat;              // [V x n_cols]
    const uint8_t *lat_ok;          // [V x n_cols]
};

struct VJob {
    int64_t n_sched;
    const int64_t *sb;              // [n+1] batch offsets
    const hs_sched_batch *b;        // batches
    const int64_t *inputs;          // input values
    const int32_t *L;               // [n] input_count
    const double *obj;              // [n] stated objective
    double tol;
    const int64_t *by_off;          // [n] offset into by_input (V * L_s each)
    int32_t *by_input;              // (task, input) -> batch
    const int64_t *seen_off;        // [n] offset into seen (K * words each)
    uint32_t *seen;                 // per device: task seen bitset
    double *ends;                   // [batches]
    int32_t *dlist;                 // [batches] batches grouped by device
    int32_t *rank;                  // [batches] stable (start, end) rank
    int32_t *dinfo;                 // [n x 3K]: list start, count, first-seen order
    hs_violation *out;
};

constexpr int kThreads = 256;

__device__ __forceinline__ bool key_less(double s1, double e1, double s2, double e2) {
    return s1 < s2 || (s1 == s2 && e1 < e2);  // Python tuple (start, end) order
}

__global__ void validate_kernel(VTables t, VJob j) {
    __shared__ int s_code;
    __shared__ unsigned long long s_key;
    __shared__ double s_red[kThreads];
    __shared__ hs_violation s_out;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int64_t q = blockIdx.x; q < j.n_sched; q += gridDim.x) {
        const int64_t b0 = j.sb[q], b1 = j.sb[q + 1];
        const int nb = int(b1 - b0);
        const int L = j.L[q];
        const double tol = j.tol;
        int32_t *byi = j.by_input + j.by_off[q];
        uint32_t *seen = j.seen + j.seen_off[q];
        int32_t *dinfo = j.dinfo + q * 3 * t.K;  // start | count | order
        const int words = (t.V + 31) / 32;
        for (int64_t k = tid; k < int64_t(t.V) * L; k += nt) byi[k] = -1;
        for (int k = tid; k < t.K * words; k += nt) seen[k] = 0;
        for (int k = tid; k < 3 * t.K; k += nt) dinfo[k] = k < 2 * t.K ? 0 : -1;
        if (tid == 0) {
            s_code = 0;
            memset(&s_out, 0, sizeof(s_out));
        }
        __syncthreads();
        // ---- per-batch checks, in batch order (thread 0)
        if (tid == 0) {
            int code = 0, a = 0, c = 0, nd = 0;
            for (int jj = 0; jj < nb && !code; ++jj) {
                const hs_sched_batch B = j.b[b0 + jj];
                a = jj;
                if (B.task < 0) { code = HS_V_UNKNOWN_TASK; break; }
                if (B.device < 0) { code = HS_V_UNKNOWN_DEVICE; break; }
                if (B.size != B.n_inputs || (B.flags & 1)) { code = HS_V_SIZE; break; }
                int col = -1;
                for (int x = t.boff[B.device]; x < t.boff[B.device + 1]; ++x)
                    if (t.bsz[x] == B.size) col = x;
                if (col < 0) { code = HS_V_BATCH_SIZE; break; }
                if (B.start < -tol) { code = HS_V_NEGATIVE_START; break; }
                for (int x = 0; x < B.n_inputs; ++x) {
                    const int64_t l = j.inputs[B.in_off + x];
                    c = x;
                    if (l < 1 || l > L) { code = HS_V_INPUT_RANGE; break; }
                    int32_t &slot = byi[int64_t(B.task) * L + (l - 1)];
                    if (slot >= 0) { code = HS_V_DOUBLE; break; }
                    slot = jj;
                }
                if (code) break;
                const int64_t li = int64_t(B.task) * t.n_cols + col;
                if (!t.lat_ok[li]) { code = HS_V_LATENCY; break; }
                j.ends[b0 + jj] = B.start + t.lat[li];
                dinfo[t.K + B.device] += 1;
                if (dinfo[2 * t.K + B.device] < 0) dinfo[2 * t.K + B.device] = nd++;
            }
            if (code) {
                s_code = code;
                s_out.code = code;
                s_out.a = a;
                s_out.c = c;
            } else {  // group batch indices by device (batch order kept)
                int acc = 0;
                for (int d = 0; d < t.K; ++d) {
                    dinfo[d] = acc;
                    acc += dinfo[t.K + d];
                    dinfo[t.K + d] = 0;
                }
                for (int jj = 0; jj < nb; ++jj) {
                    const int d = j.b[b0 + jj].device;
                    j.dlist[b0 + dinfo[d] + dinfo[t.K + d]++] = jj;
                }
            }
        }
        __syncthreads();
        // ---- every (task, input) assigned, tasks x inputs order
        if (!s_code) {
            if (tid == 0) s_key = ~0ull;
            __syncthreads();
            for (int64_t k = tid; k < int64_t(t.V) * L; k += nt)
                if (byi[k] < 0) atomicMin(&s_key, (unsigned long long)k);
            __syncthreads();
            if (tid == 0 && s_key != ~0ull) {
                s_code = s_out.code = HS_V_UNASSIGNED;
                s_out.a = int(s_key / L);
                s_out.c = int(s_key % L) + 1;
            }
            __syncthreads();
        }
        // ---- precedence with communication, edges x inputs order
        if (!s_code) {
            if (tid == 0) s_key = ~0ull;
            __syncthreads();
            for (int64_t k = tid; k < int64_t(t.E) * L; k += nt) {
                const int e = int(k / L), l = int(k % L);
                const int src = t.esrc[e], dst = t.edst[e];
                const int bi = byi[int64_t(src) * L + l], bj = byi[int64_t(dst) * L + l];
                const int du = j.b[b0 + bi].device, dv = j.b[b0 + bj].device;
                bool bad;
                if (du == dv) {
                    bad = j.b[b0 + bj].start + tol < j.ends[b0 + bi] + 0.0;
                } else {
                    const double beta = t.bw[du * t.K + dv];
                    bad = !(beta > 0.0) ||
                          j.b[b0 + bj].start + tol < j.ends[b0 + bi] + t.om[src] / beta;
                }
                if (bad) atomicMin(&s_key, (unsigned long long)k);
            }
            __syncthreads();
            if (tid == 0 && s_key != ~0ull) {
                const int e = int(s_key / L), l = int(s_key % L);
                const int src = t.esrc[e], dst = t.edst[e];
                const int bi = byi[int64_t(src) * L + l], bj = byi[int64_t(dst) * L + l];
                const int du = j.b[b0 + bi].device, dv = j.b[b0 + bj].device;
                const double beta = du == dv ? 1.0 : t.bw[du * t.K + dv];
                s_out.a = e;
                s_out.b = bi;
                s_out.c = l + 1;
                if (du != dv && !(beta > 0.0)) {
                    s_out.code = HS_V_NO_LINK;
                } else {
                    s_out.code = HS_V_PRECEDENCE;
                    s_out.v0 = j.b[b0 + bj].start;
                    s_out.v1 = j.ends[b0 + bi];
                    s_out.v2 = du == dv ? 0.0 : t.om[src] / beta;
                }
                s_code = s_out.code;
            }
            __syncthreads();
        }
        // ---- overlap per device: stable (start, end) ranks, then the first
        // overlapping pair in (device first-seen order, rank, rank) order
        if (!s_code) {
            for (int x = tid; x < nb; x += nt) {
                const hs_sched_batch B = j.b[b0 + x];
                const int d = B.device, lo = dinfo[d], cnt = dinfo[t.K + d];
                const double sx = B.start, ex = j.ends[b0 + x];
                int r = 0;
                for (int y = 0; y < cnt; ++y) {
                    const int yy = j.dlist[b0 + lo + y];
                    const double sy = j.b[b0 + yy].start, ey = j.ends[b0 + yy];
                    if (key_less(sy, ey, sx, ex) || (!key_less(sx, ex, sy, ey) && yy < x)) ++r;
                }
                j.rank[b0 + x] = r;
            }
            if (tid == 0) s_key = ~0ull;
            __syncthreads();
            for (int d = 0; d < t.K; ++d) {
                const int lo = dinfo[d], cnt = dinfo[t.K + d], ord = dinfo[2 * t.K + d];
                const int64_t pairs = int64_t(cnt) * cnt;
                for (int64_t k = tid; k < pairs; k += nt) {
                    const int x = j.dlist[b0 + lo + int(k / cnt)];
                    const int y = j.dlist[b0 + lo + int(k % cnt)];
                    const int rx = j.rank[b0 + x], ry = j.rank[b0 + y];
                    if (rx >= ry) continue;
                    const double sx = j.b[b0 + x].start, sy = j.b[b0 + y].start;
                    const double ex = j.ends[b0 + x], ey = j.ends[b0 + y];
                    const double hi = sx > sy ? sx : sy;  // max(b1.start, b2.start)
                    const double lo2 = ex < ey ? ex : ey;
                    if (hi < lo2 - tol)
                        atomicMin(&s_key, ((unsigned long long)ord << 42) |
                                              ((unsigned long long)rx << 21) |
                                              (unsigned long long)ry);
                }
            }
            __syncthreads();
            if (tid == 0 && s_key != ~0ull) {
                const int ord = int(s_key >> 42), rx = int((s_key >> 21) & 0x1FFFFF),
                          ry = int(s_key & 0x1FFFFF);
                int d = 0;
                for (int x = 0; x < t.K; ++x)
                    if (dinfo[2 * t.K + x] == ord) d = x;
                const int lo = dinfo[d], cnt = dinfo[t.K + d];
                int bx = -1, by = -1;
                for (int y = 0; y < cnt; ++y) {
                    const int yy = j.dlist[b0 + lo + y];
                    if (j.rank[b0 + yy] == rx) bx = yy;
                    if (j.rank[b0 + yy] == ry) by = yy;
                }
                s_out.code = HS_V_OVERLAP;
                s_out.a = bx;
                s_out.b = by;
                s_out.c = d;
                s_out.v0 = j.ends[b0 + bx];
                s_out.v1 = j.ends[b0 + by];
                s_code = s_out.code;
            }
            __syncthreads();
        }
        // ---- memory per device (hardware order), sequential sums
        if (!s_code) {
            if (tid == 0) s_key = ~0ull;
            __syncthreads();
            if (tid < t.K) {
                const int d = tid, lo = dinfo[d], cnt = dinfo[t.K + d];
                double used = 0.0;
                uint32_t *sd = seen + d * words;
                for (int y = 0; y < cnt; ++y) {
                    const hs_sched_batch B = j.b[b0 + j.dlist[b0 + lo + y]];
                    const double per = t.im[B.task] + t.om[B.task];
                    used += per * double(B.size);
                    const uint32_t bit = 1u << (B.task & 31);
                    if (!(sd[B.task >> 5] & bit)) {
                        sd[B.task >> 5] |= bit;
                        used += t.wm[B.task];
                    }
                }
                if (used > t.memory[d] + tol) atomicMin(&s_key, (unsigned long long)d);
            }
            __syncthreads();
            if (tid == 0 && s_key != ~0ull) {
                const int d = int(s_key), lo = dinfo[d], cnt = dinfo[t.K + d];
                double used = 0.0;
                for (int w = 0; w < words; ++w) seen[d * words + w] = 0;
                uint32_t *sd = seen + d * words;
                for (int y = 0; y < cnt; ++y) {
                    const hs_sched_batch B = j.b[b0 + j.dlist[b0 + lo + y]];
                    const double per = t.im[B.task] + t.om[B.task];
                    used += per * double(B.size);
                    const uint32_t bit = 1u << (B.task & 31);
                    if (!(sd[B.task >> 5] & bit)) {
                        sd[B.task >> 5] |= bit;
                        used += t.wm[B.task];
                    }
                }
                s_out.code = HS_V_MEMORY;
                s_out.a = d;
                s_out.v0 = used;
                s_out.v1 = t.memory[d];
                s_code = s_out.code;
            }
            __syncthreads();
        }
        // ---- makespan vs the stated objective
        if (!s_code) {
            double m = -__longlong_as_double(0x7FF0000000000000LL);
            for (int x = tid; x < nb; x += nt) {
                const double e = j.ends[b0 + x];
                m = e > m ? e : m;
            }
            s_red[tid] = m;
            __syncthreads();
            for (int w = nt / 2; w > 0; w >>= 1) {
                if (tid < w) s_red[tid] = s_red[tid + w] > s_red[tid] ? s_red[tid + w] : s_red[tid];
                __syncthreads();
            }
            if (tid == 0) {
                const double mk = nb > 0 ? s_red[0] : 0.0;  // max(ends) or 0.0
                s_out.v0 = mk;
                if (fabs(mk - j.obj[q]) > tol) {
                    s_out.code = HS_V_OBJECTIVE;
                    s_out.v1 = j.obj[q];
                }
            }
            __syncthreads();
        }
        if (tid == 0) j.out[q] = s_out;
        __syncthreads();
    }
}

}  // namespace

namespace {

struct DevBuf {
    void *p = nullptr;
    cudaStream_t s = nullptr;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
};

}  // namespace

extern "C" int hs_validate_schedules(const hs_instance_desc *d, int64_t n_sched,
                                     const int64_t *h_batch_off,
                                     const hs_sched_batch *h_batches,
                                     const int64_t *h_inputs,
                                     const int32_t *h_input_count,
                                     const double *h_objective, double tol,
                                     hs_violation *h_out, void *stream) {
    if (!d || n_sched < 0 || (n_sched > 0 && (!h_batch_off || !h_input_count ||
                                               !h_objective || !h_out)))
        return hs::set_error(HS_EINVAL, "hs_validate_schedules: null argument");
    if (n_sched == 0) return HS_OK;
    const int V = d->n_tasks, E = d->n_edges, K = d->n_devices;
    if (V < 0 || E < 0 || K < 1 || (E > 0 && (!d->edge_src || !d->edge_dst)))
        return hs::set_error(HS_EINVAL, "hs_validate_schedules: bad instance");
    const int n_cols = d->batch_off[K];
    const int64_t nbt = h_batch_off[n_sched];
    if (nbt < 0 || (nbt > 0 && !h_batches))
        return hs::set_error(HS_EINVAL, "hs_validate_schedules: bad batch offsets");
    int64_t n_in = 0;
    for (int64_t x = 0; x < nbt; ++x) {
        const hs_sched_batch &B = h_batches[x];
        if (B.task >= V || B.device >= K || B.n_inputs < 0 || B.in_off < 0)
            return hs::set_error(HS_EINVAL, "hs_validate_schedules: bad batch record");
        n_in = std::max<int64_t>(n_in, B.in_off + B.n_inputs);
    }
    if (n_in > 0 && !h_inputs)
        return hs::set_error(HS_EINVAL, "hs_validate_schedules: null inputs");
    for (int64_t q = 0; q < n_sched; ++q)
        if (h_batch_off[q + 1] < h_batch_off[q] || h_batch_off[q + 1] - h_batch_off[q] > (1 << 20) ||
            h_input_count[q] < 0)
            return hs::set_error(HS_EINVAL, "hs_validate_schedules: bad schedule");
    for (int x = 0; x < E; ++x)
        if (d->edge_src[x] < 0 || d->edge_src[x] >= V || d->edge_dst[x] < 0 ||
            d->edge_dst[x] >= V)
            return hs::set_error(HS_EINVAL, "hs_validate_schedules: bad edge");
    const int words = (V + 31) / 32;
    std::vector<int64_t> by_off(size_t(n_sched) + 1, 0), seen_off(size_t(n_sched) + 1, 0);
    for (int64_t q = 0; q < n_sched; ++q) {
        by_off[q + 1] = by_off[q] + int64_t(V) * h_input_count[q];
        seen_off[q + 1] = seen_off[q] + int64_t(K) * words;
    }
    // one device arena: tables | job arrays | scratch
    std::vector<std::pair<const void *, size_t>> up;
    size_t total = 0;
    auto place = [&](size_t bytes) {
        const size_t at = total;
        total += (bytes + 255) & ~size_t(255);
        return at;
    };
    const size_t o_wm = place(8 * size_t(V)), o_im = place(8 * size_t(V)),
                 o_om = place(8 * size_t(V)), o_es = place(4 * size_t(E)),
                 o_ed = place(4 * size_t(E)), o_bw = place(8 * size_t(K) * K),
                 o_mem = place(8 * size_t(K)), o_bo = place(4 * size_t(K + 1)),
                 o_bs = place(4 * size_t(n_cols)),
                 o_lat = place(8 * size_t(V) * n_cols), o_ok = place(size_t(V) * n_cols),
                 o_sb = place(8 * size_t(n_sched + 1)),
                 o_b = place(sizeof(hs_sched_batch) * size_t(nbt)),
                 o_in = place(8 * size_t(n_in)), o_L = place(4 * size_t(n_sched)),
                 o_obj = place(8 * size_t(n_sched)), o_byo = place(8 * size_t(n_sched)),
                 o_so = place(8 * size_t(n_sched)), o_out = place(sizeof(hs_violation) * size_t(n_sched)),
                 o_by = place(4 * size_t(by_off[n_sched])),
                 o_seen = place(4 * size_t(seen_off[n_sched])),
                 o_ends = place(8 * size_t(nbt)), o_dl = place(4 * size_t(nbt)),
                 o_rk = place(4 * size_t(nbt)), o_di = place(4 * size_t(n_sched) * 3 * K);
    const size_t upload_end = o_out;
    std::vector<uint8_t> host(upload_end, 0);
    auto put = [&](size_t at, const void *src, size_t bytes) {
        if (bytes) std::memcpy(host.data() + at, src, bytes);
    };
    put(o_wm, d->wm, 8 * size_t(V));
    put(o_im, d->im, 8 * size_t(V));
    put(o_om, d->om, 8 * size_t(V));
    put(o_es, d->edge_src, 4 * size_t(E));
    put(o_ed, d->edge_dst, 4 * size_t(E));
    put(o_bw, d->bandwidth, 8 * size_t(K) * K);
    put(o_mem, d->memory, 8 * size_t(K));
    put(o_bo, d->batch_off, 4 * size_t(K + 1));
    put(o_bs, d->batch_sizes, 4 * size_t(n_cols));
    put(o_lat, d->latency, 8 * size_t(V) * n_cols);
    put(o_ok, d->latency_ok, size_t(V) * n_cols);
    put(o_sb, h_batch_off, 8 * size_t(n_sched + 1));
    put(o_b, h_batches, sizeof(hs_sched_batch) * size_t(nbt));
    put(o_in, h_inputs, 8 * size_t(n_in));
    put(o_L, h_input_count, 4 * size_t(n_sched));
    put(o_obj, h_objective, 8 * size_t(n_sched));
    put(o_byo, by_off.data(), 8 * size_t(n_sched));
    put(o_so, seen_off.data(), 8 * size_t(n_sched));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DevBuf buf;
    buf.s = s;
    cudaError_t e = hs::scratch_alloc(&buf.p, total, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(buf.p, host.data(), upload_end, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess)
        return hs::set_error(HS_ECUDA, std::string("hs_validate_schedules: ") +
                                           cudaGetErrorString(e));
    uint8_t *base = static_cast<uint8_t *>(buf.p);
    VTables t{V, E, K, n_cols,
              reinterpret_cast<const double *>(base + o_wm),
              reinterpret_cast<const double *>(base + o_im),
              reinterpret_cast<const double *>(base + o_om),
              reinterpret_cast<const int32_t *>(base + o_es),
              reinterpret_cast<const int32_t *>(base + o_ed),
              reinterpret_cast<const double *>(base + o_bw),
              reinterpret_cast<const double *>(base + o_mem),
              reinterpret_cast<const int32_t *>(base + o_bo),
              reinterpret_cast<const int32_t *>(base + o_bs),
              reinterpret_cast<const double *>(base + o_lat),
              reinterpret_cast<const uint8_t *>(base + o_ok)};
    VJob j{n_sched,
           reinterpret_cast<const int64_t *>(base + o_sb),
           reinterpret_cast<const hs_sched_batch *>(base + o_b),
           reinterpret_cast<const int64_t *>(base + o_in),
           reinterpret_cast<const int32_t *>(base + o_L),
           reinterpret_cast<const double *>(base + o_obj),
           tol,
           reinterpret_cast<const int64_t *>(base + o_byo),
           reinterpret_cast<int32_t *>(base + o_by),
           reinterpret_cast<const int64_t *>(base + o_so),
           reinterpret_cast<uint32_t *>(base + o_seen),
           reinterpret_cast<double *>(base + o_ends),
           reinterpret_cast<int32_t *>(base + o_dl),
           reinterpret_cast<int32_t *>(base + o_rk),
           reinterpret_cast<int32_t *>(base + o_di),
           reinterpret_cast<hs_violation *>(base + o_out)};
    const int grid = int(std::min<int64_t>(n_sched, 148 * 8));
    validate_kernel<<<grid, kThreads, 0, s>>>(t, j);
    e = cudaGetLastError();
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(h_out, base + o_out, sizeof(hs_violation) * size_t(n_sched),
                            cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess)
        return hs::set_error(HS_ECUDA, std::string("validate_kernel: ") + cudaGetErrorString(e));
    return HS_OK;
}
