// Per-graph specialised evaluator: the plan is emitted as straight-line
// CUDA (one block of code per task placement, the graph's predecessor
// positions, end-time slots, communication and latency constants baked in
// as immediates), compiled by NVRTC for sm_100a at plan time and driven by
// the same tile loop as the ahead-of-time kernel (eval_common.cuh).
//
// Compared with walking node/edge records, this removes every plan load and
// address computation from the inner loop. On top of that (defaults from
// the B200 sweeps in profiles/README.md):
//  * software pipelining: relaxation terms of task t are emitted beside the
//    dependent per-device chain of task t - ahead;
//  * split residency: every end time is a register value for consumers
//    within `near` positions; values read farther away get long storage --
//    registers (greedy interval selection), then end-time slots in tensor
//    memory (tcgen05.ld/st, 12 warps/SM), shared memory, or a global-memory
//    tier for graphs whose live end times exceed the SM;
//  * dominance pruning: same-device predecessor terms never exceed the
//    device's available time and are dropped.
// The arithmetic is the reference decoder's binary64 sequence
// (heuristics.py:43-148) up to reorderings that are exact without NaN
// (max is associative); results are checked bit-for-bit against the golden
// fixtures by the same GPU tests as the AOT kernel.
//
// Scope (everything else uses the AOT kernel): non-batched plans with
// K <= 64 devices, V <= 1100 tasks, E <= 2600 edges and no NaN anywhere in
// the cost model (max is then associative, so predecessor maxima may be
// reordered). Capacity, batch-size, missing-entry and missing-link checks
// are emitted only when the plan needs them.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <queue>
#include <string>
#include <vector>

#include "jit.hpp"

namespace hs {
namespace {

#include "eval_common_src.inc"  // kEvalCommonSrc: text of eval_common.cuh

// ---- NVRTC through dlopen: the library loads on hosts without CUDA
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram *nvrtcProgram_t;
struct Nvrtc {
    void *h = nullptr;
    nvrtcResult_t (*create)(nvrtcProgram_t *, const char *, const char *, int,
                            const char *const *, const char *const *) = nullptr;
    nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char *const *) = nullptr;
    nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t *) = nullptr;
    nvrtcResult_t (*log)(nvrtcProgram_t, char *) = nullptr;
    nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t *) = nullptr;
    nvrtcResult_t (*cubin)(nvrtcProgram_t, char *) = nullptr;
    nvrtcResult_t (*destroy)(nvrtcProgram_t *) = nullptr;
    bool ok = false;
};

Nvrtc &nvrtc() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *names[] = {"/usr/local/cuda/lib64/libnvrtc.so.12",
                               "libnvrtc.so.12", "libnvrtc.so"};
        for (const char *nm : names) {
            n.h = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
            if (n.h) break;
        }
        if (!n.h) return;
        n.create = (decltype(n.create))dlsym(n.h, "nvrtcCreateProgram");
        n.compile = (decltype(n.compile))dlsym(n.h, "nvrtcCompileProgram");
        n.log_size = (decltype(n.log_size))dlsym(n.h, "nvrtcGetProgramLogSize");
        n.log = (decltype(n.log))dlsym(n.h, "nvrtcGetProgramLog");
        n.cubin_size = (decltype(n.cubin_size))dlsym(n.h, "nvrtcGetCUBINSize");
        n.cubin = (decltype(n.cubin))dlsym(n.h, "nvrtcGetCUBIN");
        n.destroy = (decltype(n.destroy))dlsym(n.h, "nvrtcDestroyProgram");
        n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size &&
               n.cubin && n.destroy;
    });
    return n;
}

std::string lit(double v) {
    if (std::isinf(v)) return v > 0 ? "kinf()" : "(-kinf())";
    if (std::isnan(v)) return "knan()";
    char buf[64];
    std::snprintf(buf, sizeof buf, "%a", v);
    return std::string("(") + buf + ")";
}

std::string sel(const std::string &d, const std::vector<std::string> &vals) {
    // vals[k] for gene d, as a select chain (K <= 4)
    bool same = true;
    for (auto &v : vals) same = same && v == vals[0];
    if (same) return vals[0];
    std::string out = vals[0];
    for (size_t k = 1; k < vals.size(); ++k)
        out = "dsel(" + d + " == " + std::to_string(k) + ", " + vals[k] + ", " + out + ")";
    return out;
}

}  // namespace

JitOpts JitOpts::from_env() {
    JitOpts o;
    const char *env = getenv("HS_JIT_OPTS");
    if (!env) return o;
    std::string s(env);
    size_t at = 0;
    while (at < s.size()) {
        size_t end = s.find(',', at);
        if (end == std::string::npos) end = s.size();
        const std::string kv = s.substr(at, end - at);
        const size_t eq = kv.find('=');
        if (eq != std::string::npos) {
            const std::string k = kv.substr(0, eq), v = kv.substr(eq + 1);
            if (k == "regs") o.reg_budget = std::atoi(v.c_str());
            if (k == "win") o.reg_window = std::atoi(v.c_str());
            if (k == "avail") o.avail_smem = v == "smem";
            if (k == "dur") o.dur_smem = v == "smem";
            if (k == "max") o.int_max = v == "int";
            if (k == "genes") o.genes_reg = v == "reg";
            if (k == "near") o.near = std::atoi(v.c_str());
            if (k == "ctas") o.ctas = std::max(1, std::atoi(v.c_str()));
            if (k == "ahead") o.ahead = std::atoi(v.c_str());
            if (k == "fma") o.fma = std::atoi(v.c_str()) != 0;
            if (k == "glanes") o.gslot_lanes = std::max(32, std::atoi(v.c_str()));
            // end-time slots in the global-memory tier regardless of fit
            // (normally chosen by jit_build; also for hs_plan_emit_specialized)
            if (k == "gslots") o.gslots = std::atoi(v.c_str()) != 0;
            if (k == "sync") o.sync = std::atoi(v.c_str());
            if (k == "gword") o.gword = std::atoi(v.c_str()) != 0;
            if (k == "dom") o.dom = std::atoi(v.c_str()) != 0;
            if (k == "tmem") o.tmem = std::atoi(v.c_str()) != 0;
            if (k == "tlanes") o.tm_lanes = std::max(32, std::atoi(v.c_str()));
            if (k == "tregs") o.tm_regs = std::max(0, std::atoi(v.c_str()));
            if (k == "tdev") o.tm_dev = std::atoi(v.c_str()) != 0;
            if (k == "tctas") o.tm_ctas = std::atoi(v.c_str()) >= 2 ? 2 : 1;
            if (k == "blk") o.blk = std::atoi(v.c_str()) != 0;
            // emission-only (hs_plan_emit_specialized): TMEM columns per warp
            // group, normally chosen by jit_build
            if (k == "tcols") o.tm_cols = std::max(0, std::atoi(v.c_str()));
            if (k == "dsmem") o.dur_smem_max = std::atoi(v.c_str());
            if (k == "lanes") {
                o.lanes = std::max(32, std::min(1024, std::atoi(v.c_str())));
                o.lanes_set = true;
            }
        }
        at = end + 1;
    }
    return o;
}

static int64_t a16(int64_t x) { return (x + 15) & ~int64_t(15); }

// Straight-line code grows with V + E and NVRTC time super-linearly (about
// 20 s at V ~ 1000 on the GPU box's host), so larger graphs stay on the AOT
// kernel.
constexpr int kJitMaxV = 1100, kJitMaxE = 2600, kJitMaxK = 64;

bool jit_batched_ok(const Plan &p);

bool jit_eligible(const Plan &p) {
    if (p.batched) return jit_batched_ok(p);
    return p.K <= kJitMaxK && !p.nan_possible && p.V > 0 && p.V <= kJitMaxV &&
           p.E <= kJitMaxE;
}

namespace {

// Link classes of a multi-server platform (the paper's case study,
// benchgen.gen_transformer_stack): a full mesh whose class of (u, v) is 0
// on the same device, `ci` between devices of the same node and `co`
// across nodes, nodes being blocks of B consecutive sorted devices. The
// class is then (u == v, u / B == v / B) -- a multiply-shift and two
// compares instead of two table loads per edge. (M, S): d / B == (d * M)
// >> S for every d < K.
struct BlockClasses {
    bool ok = false;
    int B = 0, ci = 0, co = 0, M = 0, S = 0;
};

BlockClasses block_classes(const Plan &p) {
    BlockClasses b;
    if (p.uniform_comm || !p.full_mesh || p.n_cls != 3 || p.K < 3) return b;
    const int K = p.K;
    for (int B = 2; B < K && !b.ok; ++B) {
        if (K % B) continue;
        int ci = -1, co = -1;
        bool ok = true;
        for (int u = 0; u < K && ok; ++u)
            for (int v = 0; v < K && ok; ++v) {
                const size_t at = 2 * (size_t(u) * K + v);  // uint16 little-endian
                const int c = p.bclass[at] | (p.bclass[at + 1] << 8);
                if (u == v) {
                    ok = c == 0;
                    continue;
                }
                int &want = (u / B == v / B) ? ci : co;
                if (want < 0) want = c;
                ok = c == want && c != 0 && c != 0xFFFF;
            }
        if (ok && ci > 0 && co > 0 && ci != co) {
            b.B = B;
            b.ci = ci;
            b.co = co;
            for (int S = 6; S < 24 && !b.ok; ++S) {
                const int M = ((1 << S) + B - 1) / B;
                bool good = true;
                for (int d = 0; d < K && good; ++d) good = (d * M) >> S == d / B;
                if (good) {
                    b.M = M;
                    b.S = S;
                    b.ok = true;
                }
            }
        }
    }
    return b;
}

// Shared-memory layout of the specialised kernel (byte offsets); every
// table is staged from the plan blob once per CTA.
struct JitLayout {
    bool dur = false, durg = false, cls = false, mem = false, avail = false, dbuf = true;
    int64_t dur_off = 0, ctab_off = 0, bcl_off = 0, cap_off = 0, head = 16;
    int64_t tile = 0, tile2 = 0, ends = 0, avail_off = 0, mem_off = 0, total = 0;
};

JitLayout jit_layout(const Plan &p, const JitOpts &o, int T, int slots, int ld_cap,
                     bool dbuf = true) {
    JitLayout l;
    if (o.gslots || o.tmem) slots = 0;  // end-time slots in global / tensor memory
    l.dbuf = dbuf;
    l.dur = o.dur_smem || p.K > 4;
    // a large latency table (many devices: the transformer case study has
    // 288 x 30 entries = 69 KB) is read through L1 from the plan blob
    // instead of occupying shared memory that would otherwise hold lanes
    if (l.dur && int64_t(p.V) * p.K * 8 > o.dur_smem_max) {
        l.dur = false;
        l.durg = true;
    }
    l.avail = o.avail_smem || p.K > 4;
    // node-block classes need no class tables (computed from the genes)
    l.cls = !p.uniform_comm && !(o.blk && block_classes(p).ok);
    l.mem = p.mem_check;
    int64_t at = 16;
    if (l.dur) { l.dur_off = at; at += a16(int64_t(p.V) * p.K * 8); }
    if (l.cls) {
        l.ctab_off = at; at += a16(int64_t(p.V) * p.n_cls * 8);
        l.bcl_off = at; at += a16(int64_t(p.K) * p.K * 2);
    }
    if (l.mem) { l.cap_off = at; at += a16(int64_t(p.K) * 8); }
    l.head = at;
    // per-lane state first, genome tiles last: the direct-load kernel
    // (genes read from global memory into registers) needs only [0, tile)
    l.ends = at;
    at = l.ends + int64_t(slots) * T * 8;
    if (l.avail) { l.avail_off = at; at += int64_t(p.K) * T * 8; }
    if (l.mem) { l.mem_off = at; at += int64_t(p.K) * T * 8; }
    at = a16(at);
    l.tile = at;
    l.tile2 = dbuf ? l.tile + a16(int64_t(T) * ld_cap) : 0;
    at = l.tile + a16(int64_t(T) * ld_cap) * (dbuf ? 2 : 1);
    l.total = at;
    return l;
}

int64_t per_lane_bytes(const Plan &p, const JitOpts &o, int slots, int ld_cap,
                       bool dbuf) {
    if (p.batched)  // tiles, [slot][part] end times, device-available times
        return (dbuf ? 2 : 1) * ld_cap + int64_t(o.gslots ? 0 : slots) * 8 * p.P + 8 * p.K;
    const bool avail = o.avail_smem || p.K > 4;
    if (o.gslots || o.tmem) slots = 0;
    return (dbuf ? 2 : 1) * ld_cap + int64_t(slots) * 8 + (avail ? 8 * p.K : 0) + (p.mem_check ? 8 * p.K : 0);
}

int64_t head_bytes(const Plan &p, const JitOpts &o) {
    if (p.batched) {  // bat_layout's tables
        const int64_t NO = p.n_opt, VNP = int64_t(p.V) * p.n_opt * p.P;
        return 16 + a16(NO * NO * 2) + a16(NO * 8) + a16(VNP * 8) +
               (p.latency_complete ? 0 : a16(VNP));
    }
    return jit_layout(p, o, 32, 0, 0).head;
}

std::string stage(int64_t dst, const char *section, int64_t bytes) {
    char buf[512];
    std::snprintf(buf, sizeof buf,
                  "  { const uint4 *src = reinterpret_cast<const uint4 *>(a.blob + a.lay.%s);\n"
                  "    uint4 *dst = reinterpret_cast<uint4 *>(smem + %lld);\n"
                  "    for (int q = threadIdx.x; q < %lld; q += blockDim.x) dst[q] = src[q]; }\n",
                  section, (long long)dst, (long long)(a16(bytes) / 16));
    return buf;
}

}  // namespace

// ---------------------------------------------------------------------------
// Batched-variant plans (K8's semantics, heuristics.py:363-433): the gene is
// an option (a decomposition of L over distinct devices) and each task has
// up to P parts. Straight-line code per task like K1', with the option
// structure folded into two small shared-memory tables built here:
//   OPT[o]      part k of option o: device in bits 16k..16k+7, "part
//               exists" in bit 16k+8;
//   OVD[oq][oi] bit 4m+k set when part m of the producer's option oq and
//               part k of the consumer's option oi both exist, hold a common
//               input (the reference's per-input ready time) and sit on
//               different devices -- a same-device term is dominated by
//               the device's available time (no NaN), as in K1'.
// Each term is then one bit test folded into the predicated max. Uniform
// full-mesh bandwidth only (one om/beta per producer); the parts' end times
// live in registers for consumers within `near` positions, else in
// shared-memory slots [slot][part][lane] -- or, when those leave fewer than
// 96 lanes per CTA (WS200 at L = 4: ~100 far-read producers x 3 parts -> 64
// lanes), in the global-memory tier ([slot][part][lane] per CTA, L2-resident,
// like K1''s).
bool jit_batched_ok(const Plan &p) {
    if (!(p.batched && p.P <= 4 && p.n_opt <= 255 && p.full_mesh && p.n_classes <= 1 &&
          p.K <= kJitMaxK && !p.nan_possible && p.V > 0 && p.V <= kJitMaxV &&
          p.E <= kJitMaxE))
        return false;
    JitOpts o = JitOpts::from_env();
    const int slots = jit_emit_batched(p, 32, o, nullptr, true);
    const int64_t head = head_bytes(p, o);
    auto lanes = [&](const JitOpts &oo) {
        return (227 * 1024 - 2048 - head) /
               std::max<int64_t>(1, per_lane_bytes(p, oo, slots, p.pref_ld() + 16, false));
    };
    if (lanes(o) >= 96) return true;
    o.gslots = true;
    return lanes(o) >= 96;
}

namespace {

struct BatLayout {
    int64_t ovd = 16, opt = 0, bd = 0, bok = 0, head = 0, ends = 0, avail = 0, tile = 0,
            tile2 = 0, total = 0;
    bool bok_on = false;
};

BatLayout bat_layout(const Plan &p, int T, int slots, int ld_cap, bool dbuf) {
    BatLayout l;
    const int NO = p.n_opt, P = p.P;
    int64_t at = 16;
    l.ovd = at;
    at += a16(int64_t(NO) * NO * 2);
    l.opt = at;
    at += a16(int64_t(NO) * 8);
    l.bd = at;
    at += a16(int64_t(p.V) * NO * P * 8);
    l.bok_on = !p.latency_complete;
    if (l.bok_on) {
        l.bok = at;
        at += a16(int64_t(p.V) * NO * P);
    }
    l.head = at;
    l.ends = at;
    at += int64_t(slots) * P * T * 8;
    l.avail = at;
    at += int64_t(p.K) * T * 8;
    at = a16(at);
    l.tile = at;
    l.tile2 = dbuf ? at + a16(int64_t(T) * ld_cap) : 0;
    at += a16(int64_t(T) * ld_cap) * (dbuf ? 2 : 1);
    l.total = at;
    return l;
}

}  // namespace

// Emits the batched kernel for T lanes; returns the number of slots.
int jit_emit_batched(const Plan &p, int T, const JitOpts &o, std::string *src, bool dbuf) {
    const int V = p.V, K = p.K, P = p.P, NO = p.n_opt;
    std::vector<int> last(V, -1), far_last(V, -1);
    std::vector<std::vector<int>> preds(V);
    for (int i = 0; i < V; ++i)
        for (int e = p.nodes[i].e_begin; e < p.nodes[i].e_end; ++e) {
            const int q = p.edges[e].gpos;
            preds[i].push_back(q);
            last[q] = std::max(last[q], i);
        }
    const int near = std::max(1, o.near);
    for (int i = 0; i < V; ++i)
        for (int q : preds[i])
            if (i - q > near) far_last[q] = std::max(far_last[q], i);
    // interval colouring of the far-read producers' slots
    std::vector<int> where(V, -1);
    std::vector<std::vector<int>> dies(V);
    for (int q = 0; q < V; ++q)
        if (far_last[q] >= 0) dies[far_last[q]].push_back(q);
    std::priority_queue<int, std::vector<int>, std::greater<int>> freel;
    int next = 0;
    for (int i = 0; i < V; ++i) {
        for (int q : dies[i]) freel.push(where[q]);
        if (far_last[i] < 0) continue;
        if (!freel.empty()) {
            where[i] = freel.top();
            freel.pop();
        } else {
            where[i] = next++;
        }
    }
    if (src == nullptr) return next;
    const int ld_cap = p.pref_ld() + 16;
    const BatLayout l = bat_layout(p, T, o.gslots ? 0 : next, ld_cap, dbuf);
    // the option tables
    std::vector<uint64_t> opt(NO, 0);
    for (int oo = 0; oo < NO; ++oo)
        for (int k = 0; k < p.opt_np[oo]; ++k)
            opt[oo] |= (uint64_t(uint32_t(p.opt_tab[(size_t(oo) * P + k) * 4]) & 0xFFu) |
                        0x100ull) << (16 * k);
    std::vector<uint16_t> ovd(size_t(NO) * NO, 0);
    for (int a = 0; a < NO; ++a)
        for (int b = 0; b < NO; ++b)
            for (int m = 0; m < p.opt_np[a]; ++m)
                for (int k = 0; k < p.opt_np[b]; ++k) {
                    const int32_t *qa = &p.opt_tab[(size_t(a) * P + m) * 4];
                    const int32_t *qb = &p.opt_tab[(size_t(b) * P + k) * 4];
                    const bool overlap = !(qa[2] < qb[1] || qa[1] > qb[2]);
                    if (overlap && qa[0] != qb[0]) ovd[size_t(a) * NO + b] |= uint16_t(1u << (4 * m + k));
                }
    // per-producer om / beta (class 1 of the single bandwidth; 0 when the
    // mesh has no second device)
    std::vector<double> cq(V, 0.0);
    if (p.n_cls > 1)
        for (int q = 0; q < V; ++q) cq[q] = p.ctab[size_t(q) * p.n_cls + 1];
    std::string &s = *src;
    s.clear();
    char buf[512];
    s += "#include \"eval_common.cuh\"\nusing namespace hsk;\n";
    s += "__constant__ unsigned long long HOPT[" + std::to_string(NO) + "] = {";
    for (int oo = 0; oo < NO; ++oo) s += (oo ? ", " : "") + std::to_string(opt[oo]) + "ull";
    s += "};\n__constant__ unsigned short HOVD[" + std::to_string(size_t(NO) * NO) + "] = {";
    for (size_t q = 0; q < ovd.size(); ++q) s += (q ? ", " : "") + std::to_string(ovd[q]);
    s += "};\n";
    std::vector<double> cconst;
    auto cst = [&](double v) {
        if (!std::isfinite(v)) return lit(v);
        cconst.push_back(v);
        return "HSC[" + std::to_string(cconst.size() - 1) + "]";
    };
    s += "template <bool TRACE, bool SYNC>\n__device__ __forceinline__ void jit_body(hs_u8 *smem, "
         "const hs_u8 *g, int li, hs_i64 cand, bool valid, int gene_bad, double *starts, "
         "double &ms_out, int &st_out, double *EG, hs_u32 TB, const double *DG) {\n";
    // parts' end-time slots [slot][part][lane]: shared memory, or this
    // CTA's region of the global-memory tier
    if (o.gslots)
        s += "    double *E = EG + li;\n    (void)E; (void)TB; (void)DG;\n";
    else
        s += "    double *E = reinterpret_cast<double *>(smem + " + std::to_string(l.ends) +
             ") + li;\n    (void)E; (void)EG; (void)TB; (void)DG;\n";
    s += "    const hs_u16 *OVD = reinterpret_cast<const hs_u16 *>(smem + " +
         std::to_string(l.ovd) + ");\n";
    s += "    const unsigned long long *OPT = reinterpret_cast<const unsigned long long *>(smem + " +
         std::to_string(l.opt) + ");\n";
    s += "    const double *BD = reinterpret_cast<const double *>(smem + " + std::to_string(l.bd) +
         ");\n";
    if (l.bok_on)
        s += "    const hs_u8 *BOK = smem + " + std::to_string(l.bok) + ";\n";
    s += "    const hs_u32 A = smem_addr(smem + " + std::to_string(l.avail) + ") + li * 8;\n";
    for (int k = 0; k < K; ++k)
        s += "    st_shared_f64(A + " + std::to_string(k * T * 8) + ", 0.0);\n";
    s += "    int st = 0;\n";
    const std::string PS = std::to_string(P), NOS = std::to_string(NO);
    for (int i = 0; i < V; ++i) {
        const std::string is = std::to_string(i);
        s += "    // " + p.task_ids[p.order[i]] + "\n";
        s += "    const int o" + is + " = g[" + is + "];\n";
        s += "    const unsigned long long W" + is + " = OPT[o" + is + "];\n";
        for (int k = 0; k < P; ++k)
            s += "    double r" + is + "_" + std::to_string(k) + " = 0.0;\n";
        for (size_t e = 0; e < preds[i].size(); ++e) {
            const int q = preds[i][e];
            const std::string qs = std::to_string(q);
            const bool in_reg = i - q <= near;
            const std::string oq = in_reg ? "o" + qs : "(int)g[" + qs + "]";
            const std::string mk = "M" + is + "_" + std::to_string(e);
            s += "    const hs_u32 " + mk + " = OVD[" + oq + " * " + NOS + " + o" + is + "];\n";
            for (int m = 0; m < P; ++m) {
                const std::string fv = in_reg
                    ? "f" + qs + "_" + std::to_string(m)
                    : "E[" + std::to_string((int64_t(where[q]) * P + m) * T) + "]";
                for (int k = 0; k < P; ++k) {
                    std::snprintf(buf, sizeof buf, "(%s & 0x%xu) != 0u", mk.c_str(),
                                  1u << (4 * m + k));
                    const std::string r = "r" + is + "_" + std::to_string(k);
                    s += "    " + r + " = maxsel(" + r + ", " + buf + ", " + fv + ");\n";
                }
            }
        }
        for (int k = 0; k < P; ++k) {
            const std::string ks = std::to_string(k), ik = is + "_" + ks;
            s += "    const int d" + ik + " = (int)((W" + is + " >> " + std::to_string(16 * k) +
                 ") & 0xFFull);\n";
            s += "    const bool v" + ik + " = ((W" + is + " >> " + std::to_string(16 * k + 8) +
                 ") & 1ull) != 0ull;\n";
            s += "    const hs_u32 A" + ik + " = A + d" + ik + " * " + std::to_string(T * 8) + ";\n";
            s += "    const double s" + ik + " = pymax(r" + ik + ", ld_shared_f64(A" + ik + "));\n";
            const std::string bi = "(" + std::to_string(size_t(i) * NO * P + k) + " + o" + is +
                                   " * " + PS + ")";
            if (l.bok_on)
                s += "    st = first_status(st, v" + ik + " && !BOK[" + bi + "], ST_MISSING);\n";
            s += "    const double e" + ik + " = s" + ik + " + BD[" + bi + "];\n";
            std::snprintf(buf, sizeof buf,
                          "    if (TRACE && valid && v%s) starts[(cand * %d + %d) * %d + %d] = s%s;\n",
                          ik.c_str(), V, i, P, k, ik.c_str());
            s += buf;
            s += "    if (v" + ik + ") st_shared_f64(A" + ik + ", e" + ik + ");\n";
            if (last[i] >= 0) {
                const bool zero = cq[i] == 0.0 && !std::signbit(cq[i]);
                s += "    const double f" + ik + " = " +
                     (zero ? "e" + ik : "e" + ik + " + " + cst(cq[i])) + ";\n";
                if (where[i] >= 0)
                    s += "    E[" + std::to_string((int64_t(where[i]) * P + k) * T) + "] = f" + ik +
                         ";\n";
            }
        }
    }
    s += "    double ms = 0.0;\n";
    for (int k = 0; k < K; ++k)
        s += "    ms = pymax(ms, ld_shared_f64(A + " + std::to_string(k * T * 8) + "));\n";
    s += "    if (gene_bad) st = ST_GENE;\n"
         "    ms_out = st ? (st >= ST_MISSING ? knan() : kinf()) : ms;\n"
         "    st_out = st;\n}\n";
    if (!cconst.empty()) {
        std::string decl = "__constant__ double HSC[" + std::to_string(cconst.size()) + "] = {";
        for (size_t k = 0; k < cconst.size(); ++k) decl += (k ? ", " : "") + lit(cconst[k]);
        decl += "};\n";
        const size_t at = s.find("template <bool TRACE");
        s.insert(at, decl);
    }
    s += "template <bool TRACE>\nstruct JitBody {\n  hs_u8 *smem; double *starts; double *eg; "
         "hs_u32 tb;\n  const double *dg;\n"
         "  __device__ __forceinline__ void run(const hs_u8 *g, int li, hs_i64 cand, "
         "bool valid, int gene_bad, double &ms, int &st) {\n"
         "    jit_body<TRACE, true>(smem, g, li, cand, valid, gene_bad, starts, ms, st, eg, tb, dg);\n"
         "  }\n};\n";
    s += "template <bool TRACE>\n__device__ __forceinline__ void jit_main(const EvalParams &a) {\n"
         "  extern __shared__ __align__(16) hs_u8 smem[];\n";
    s += "  for (int q = threadIdx.x; q < " + std::to_string(size_t(NO) * NO) +
         "; q += blockDim.x) reinterpret_cast<hs_u16 *>(smem + " + std::to_string(l.ovd) +
         ")[q] = HOVD[q];\n";
    s += "  for (int q = threadIdx.x; q < " + NOS + "; q += blockDim.x) "
         "reinterpret_cast<unsigned long long *>(smem + " + std::to_string(l.opt) + ")[q] = HOPT[q];\n";
    s += stage(l.bd, "bdur", int64_t(V) * NO * P * 8);
    if (l.bok_on) s += stage(l.bok, "bdur_ok", int64_t(V) * NO * P);
    s += "  JitBody<TRACE> body;\n  body.smem = smem;\n  body.starts = a.starts;\n"
         "  body.eg = a.ends_g ? a.ends_g + blockIdx.x * a.ends_g_cta : nullptr;\n"
         "  body.tb = 0u;\n  body.dg = nullptr;\n"
         "  eval_tiles(a, smem, body);\n}\n";
    // o.ctas: the CTAs per SM jit_build sized the shared memory for
    std::snprintf(buf, sizeof buf,
                  "extern \"C\" __global__ void __launch_bounds__(%d, %d) "
                  "hs_jit_eval(const EvalParams a) { jit_main<false>(a); }\n"
                  "extern \"C\" __global__ void __launch_bounds__(%d, 1) "
                  "hs_jit_trace(const EvalParams a) { jit_main<true>(a); }\n",
                  T, std::max(1, o.ctas), T);
    s += buf;
    return next;
}

// Emits the kernel for T lanes; returns the number of shared-memory slots.
int jit_emit(const Plan &p, int T, const JitOpts &o_in, std::string *src) {
    JitOpts o = o_in;
    if (o.tm_cols <= 0) o.tmem = false;  // TMEM columns are chosen by jit_build
    const int V = p.V, K = p.K;
    const int reg_budget = o.reg_budget, reg_window = o.reg_window;
    std::vector<int> last(V, -1);
    std::vector<std::vector<int>> preds(V);  // positions
    for (int i = 0; i < V; ++i)
        for (int e = p.nodes[i].e_begin; e < p.nodes[i].e_end; ++e) {
            const int q = p.edges[e].gpos;
            preds[i].push_back(q);
            last[q] = std::max(last[q], i);
        }
    // register residency for short-lived end times, slots for the rest
    std::vector<int> where(V, -2);  // -2 none, -1 register, >=0 slot
    int next = 0;
    const int near = o.near;
    if (near > 0) {
        // split residency: every end time is a register value for the
        // consumers within `near` positions; a value with farther consumers
        // also gets long storage, a register when at most `reg_budget` such
        // values overlap (greedy by end point = the maximum number of
        // intervals), else a shared-memory slot (interval colouring)
        std::vector<int> far_last(V, -1);
        for (int i = 0; i < V; ++i)
            for (int q : preds[i])
                if (i - q > near) far_last[q] = std::max(far_last[q], i);
        std::vector<int> byend;
        for (int q = 0; q < V; ++q) {
            if (last[q] < 0) continue;
            if (far_last[q] < 0) where[q] = -1;
            else byend.push_back(q);
        }
        std::sort(byend.begin(), byend.end(), [&](int a, int b) {
            return far_last[a] != far_last[b] ? far_last[a] < far_last[b] : a < b;
        });
        std::vector<int> load(V + 1, 0);
        std::vector<char> to_slot(V, 0);
        for (int q : byend) {
            int mx = 0;
            for (int t = q; t < far_last[q]; ++t) mx = std::max(mx, load[t]);
            if (mx < reg_budget) {
                where[q] = -1;
                for (int t = q; t < far_last[q]; ++t) ++load[t];
            } else {
                to_slot[q] = 1;
            }
        }
        std::vector<std::vector<int>> dies(V);
        for (int q = 0; q < V; ++q)
            if (to_slot[q]) dies[far_last[q]].push_back(q);
        std::priority_queue<int, std::vector<int>, std::greater<int>> freel;
        for (int i = 0; i < V; ++i) {
            for (int q : dies[i]) freel.push(where[q]);
            if (!to_slot[i]) continue;
            if (!freel.empty()) {
                where[i] = freel.top();
                freel.pop();
            } else {
                where[i] = next++;
            }
        }
    } else {
        std::vector<std::vector<int>> dies(V);
        for (int i = 0; i < V; ++i)
            if (last[i] >= 0) dies[last[i]].push_back(i);
        std::priority_queue<int, std::vector<int>, std::greater<int>> freel;
        int live_regs = 0;
        for (int i = 0; i < V; ++i) {
            for (int q : dies[i]) {
                if (where[q] >= 0) freel.push(where[q]);
                else if (where[q] == -1) --live_regs;
            }
            if (last[i] < 0) continue;
            if (last[i] - i <= reg_window && live_regs < reg_budget) {
                where[i] = -1;
                ++live_regs;
            } else if (!freel.empty()) {
                where[i] = freel.top();
                freel.pop();
            } else {
                where[i] = next++;
            }
        }
    }
    if (src == nullptr) return next;
    const int ld_cap = p.pref_ld() + 16;
    const JitLayout l = jit_layout(p, o, T, next, ld_cap, o.dbuf);
    const bool checks = p.mem_check || !p.all_batch_ok || !p.latency_complete || l.cls;
    const std::string mx = o.int_max ? "pymax_nn" : "pymax";
    std::string &s = *src;
    s.clear();
    char buf[1024];
    s += "#include \"eval_common.cuh\"\nusing namespace hsk;\n";
    const bool greg = o.genes_reg && K <= 4;
    const int NP = (V + 15) / 16, NW = (V + 3) / 4;
    s += "template <bool TRACE, bool SYNC>\n__device__ __forceinline__ void jit_body(hs_u8 *smem, " +
         std::string(greg ? "const hs_u32 *GPA" : "const hs_u8 *g") +
         ", int li, hs_i64 cand, bool valid, int gene_bad, double *starts, "
         "double &ms_out, int &st_out, double *EG, hs_u32 TB, const double *DG) {\n";
    // end-time slots [slot][lane]: shared memory, or this CTA's region of
    // the global-memory tier (graphs whose live end times exceed it)
    if (o.gslots)
        s += "    double *E = EG + li;\n    (void)E;\n";
    else
        s += "    double *E = reinterpret_cast<double *>(smem + " + std::to_string(l.ends) +
             ") + li;\n    (void)E;\n";
    if (l.dur)
        s += "    const double *DUR = reinterpret_cast<const double *>(smem + " +
             std::to_string(l.dur_off) + ");\n";
    if (l.cls) {
        s += "    const double *CT = reinterpret_cast<const double *>(smem + " +
             std::to_string(l.ctab_off) + ");\n";
        s += "    const hs_u16 *BCL = reinterpret_cast<const hs_u16 *>(smem + " +
             std::to_string(l.bcl_off) + ");\n";
    }
    if (l.avail) {
        s += "    const hs_u32 A = smem_addr(smem + " + std::to_string(l.avail_off) +
             ") + li * 8;\n";
        for (int k = 0; k < K; ++k)
            s += "    st_shared_f64(A + " + std::to_string(k * T * 8) + ", 0.0);\n";
    } else {
        for (int k = 0; k < K; ++k) s += "    double a" + std::to_string(k) + " = 0.0;\n";
    }
    if (l.mem) {
        s += "    const double *CAP = reinterpret_cast<const double *>(smem + " +
             std::to_string(l.cap_off) + ");\n";
        s += "    const hs_u32 M = smem_addr(smem + " + std::to_string(l.mem_off) +
             ") + li * 8;\n";
        for (int k = 0; k < K; ++k)
            s += "    st_shared_f64(M + " + std::to_string(k * T * 8) + ", 0.0);\n";
    }
    // genes 2 bits each in registers: no shared-memory gene loads on the
    // per-task chain, and no aliasing between gene reads and slot stores
    auto gexpr = [&](int q) {
        const int j = q >> 4, sh = 2 * (q & 15);
        std::string w = "GP" + std::to_string(j);
        if (sh) w = "(" + w + " >> " + std::to_string(sh) + ")";
        return sh == 30 ? "(int)" + w : "(int)(" + w + " & 3u)";
    };
    if (greg)
        for (int j = 0; j < NP; ++j)
            s += "    const hs_u32 GP" + std::to_string(j) + " = GPA[" + std::to_string(j) +
                 "];\n";
    s += "    int st = 0;\n";
    uint64_t okmask = 0;
    for (int k = 0; k < K; ++k)
        if (p.okL[k]) okmask |= 1ull << k;
    // max over a list of terms: a balanced tree (no NaN can occur, so max
    // is associative and the result equals the reference's fold)
    auto max_tree = [&](std::vector<std::string> xs, const std::string &tag) {
        int lvl = 0;
        while (xs.size() > 1) {
            std::vector<std::string> nx;
            for (size_t k = 0; k + 1 < xs.size(); k += 2) {
                const std::string m = "m" + tag + "_" + std::to_string(lvl) + "_" +
                                      std::to_string(k);
                s += "    const double " + m + " = " + mx + "(" + xs[k] + ", " + xs[k + 1] +
                     ");\n";
                nx.push_back(m);
            }
            if (xs.size() & 1) nx.push_back(xs.back());
            xs.swap(nx);
            ++lvl;
        }
        return xs[0];
    };
    std::vector<double> cconst;  // fma communication constants (HSC[])
    // Dominance pruning (uniform bandwidth, o.dom): a predecessor on the
    // consumer's device contributes end + 0.0, which never exceeds the
    // device's available time (per-device ends never decrease without NaN,
    // and every time is >= +0.0), so max(ready, avail) is unchanged when it
    // is dropped. Each producer then carries one value f = end + om/beta
    // (one add per producer instead of per edge) and each edge is one
    // predicated compare-and-select: acc = (d_q != d_i && f > acc) ? f : acc.
    const BlockClasses bk = o.blk && !greg ? block_classes(p) : BlockClasses{};
    const bool blk = bk.ok && !l.cls;
    const bool dom = o.dom && !l.cls && !greg && !blk;
    // both fold "cond|value" terms with the same-device terms dropped
    const bool domlike = dom || blk;
    auto node_of = [&](const std::string &d) {
        return "((" + d + " * " + std::to_string(bk.M) + ") >> " + std::to_string(bk.S) + ")";
    };
    std::vector<double> prod_c(V, 0.0);
    for (int i = 0; i < V; ++i)
        for (int e = p.nodes[i].e_begin; e < p.nodes[i].e_end; ++e)
            prod_c[p.edges[e].gpos] = p.edges[e].c;
    auto zero_c = [&](int q) { return prod_c[q] == 0.0 && !std::signbit(prod_c[q]); };
    // one relaxation term end(q) + comm(q -> i) per predecessor
    auto edge_terms = [&](int i, int k0, int k1) {
        const std::string is = std::to_string(i), di = "d" + is;
        std::vector<std::string> xs;
        for (int k = k0; k < k1; ++k) {
            const int q = preds[i][k];
            const EdgeRec &er = p.edges[p.nodes[i].e_begin + k];
            const bool in_reg = where[q] == -1 || (near > 0 && i - q <= near);
            const std::string endq = in_reg
                ? "e" + std::to_string(q)
                : o.tmem ? "TV" + is + "_" + std::to_string(q)  // loaded by tm_loads()
                : "E[" + std::to_string((long long)where[q] * T) + "]";
            const bool tdev = o.tmem && o.tm_dev && !in_reg && !greg;
            const std::string gq = greg ? gexpr(q)
                : in_reg ? "d" + std::to_string(q)
                : tdev ? "TD" + is + "_" + std::to_string(q)  // device from TMEM
                : "(int)g[" + std::to_string(q) + "]";
            const std::string x = "x" + is + "_" + std::to_string(k);
            if (dom) {
                // the producer's f (register name f<q>, or its slot)
                const std::string fq = in_reg ? "f" + std::to_string(q) : endq;
                xs.push_back((zero_c(q) ? std::string() : gq + " != " + di) + "|" + fq);
                continue;
            }
            if (blk) {
                // same device: dominated (dropped); same node: class ci;
                // other node: class co (om / beta of either, constant memory)
                const std::string nq = (near > 0 && i - q <= near)
                                           ? "n" + std::to_string(q) : node_of(gq);
                const double cin = p.ctab[size_t(q) * p.n_cls + bk.ci];
                const double cout = p.ctab[size_t(q) * p.n_cls + bk.co];
                std::string ci_s = lit(cin), co_s = lit(cout);
                if (std::isfinite(cin) && std::isfinite(cout)) {
                    ci_s = "HSC[" + std::to_string(cconst.size()) + "]";
                    cconst.push_back(cin);
                    co_s = "HSC[" + std::to_string(cconst.size()) + "]";
                    cconst.push_back(cout);
                }
                s += "    const double " + x + " = " + endq + " + dsel(" + nq + " == n" + is +
                     ", " + ci_s + ", " + co_s + ");\n";
                xs.push_back(gq + " != " + di + "|" + x);
                continue;
            }
            if (l.cls) {
                // comm class of (producer device, consumer device); 0xFFFF =
                // missing link (core.py:153-154), class 0 = same device
                const std::string c = "c" + is + "_" + std::to_string(k);
                s += "    const int " + c + "r = BCL[" + gq + " * " + std::to_string(K) + " + " +
                     di + "];\n";
                s += "    nl" + is + " |= " + c + "r == 0xFFFF;\n";
                s += "    const int " + c + " = min(" + c + "r, " + std::to_string(p.n_cls - 1) +
                     ");\n";
                s += "    const double " + x + " = " + endq + " + CT[" +
                     std::to_string((long long)q * p.n_cls) + " + " + c + "];\n";
            } else if (er.c == 0.0 && !std::signbit(er.c)) {
                // zero-byte output: end + 0.0 == end for end >= +0
                s += "    const double " + x + " = " + endq + ";\n";
            } else if (o.fma && std::isfinite(er.c) && !greg) {
                // end + (same ? 0 : c) as fma(c, 0.0 or 1.0, end): one FP64
                // op and one 32-bit select instead of an add and a 64-bit
                // select; exact: c*1 + end rounds once like end + c, and
                // c*0 + end == end for finite c and end >= +0
                // the constant comes from constant memory (an operand of
                // DFMA, no register moves)
                s += "    const double " + x + " = __fma_rn(HSC[" +
                     std::to_string(cconst.size()) + "], dsel(" + gq + " == " + di +
                     ", 0.0, 1.0), " + endq + ");\n";
                cconst.push_back(er.c);
            } else if (greg) {
                // same device <=> the 2-bit fields agree: one LOP3 per edge
                const int j = q >> 4, sh = 2 * (q & 15);
                char mk[32];
                std::snprintf(mk, sizeof mk, "0x%xu", 3u << sh);
                s += "    const double " + x + " = " + endq + " + dsel(((GP" +
                     std::to_string(j) + " ^ DP" + is + ") & " + mk + ") == 0u, 0.0, " +
                     lit(er.c) + ");\n";
            } else {
                s += "    const double " + x + " = " + endq + " + dsel(" + gq + " == " + di +
                     ", 0.0, " + lit(er.c) + ");\n";
            }
            xs.push_back(x);
        }
        return xs;
    };
    // dom: fold "cond|value" terms into a running maximum named `acc`
    auto fold = [&](const std::vector<std::string> &terms, const std::string &acc,
                    const std::string &init) {
        size_t k0 = 0;
        if (init == "0.0" && !terms.empty()) {
            // first term against the 0.0 start: a plain select (v >= +0.0)
            const size_t bar = terms[0].find('|');
            const std::string cond = terms[0].substr(0, bar), v = terms[0].substr(bar + 1);
            s += "    double " + acc + " = " +
                 (cond.empty() ? v : "dsel(" + cond + ", " + v + ", 0.0)") + ";\n";
            k0 = 1;
        } else {
            s += "    double " + acc + " = " + init + ";\n";
        }
        for (size_t k = k0; k < terms.size(); ++k) {
            const std::string &t = terms[k];
            const size_t bar = t.find('|');
            const std::string cond = t.substr(0, bar), v = t.substr(bar + 1);
            if (cond.empty())
                s += "    " + acc + " = " + mx + "(" + acc + ", " + v + ");\n";
            else
                s += "    " + acc + " = maxsel(" + acc + ", " + cond + ", " + v + ");\n";
        }
        return acc;
    };
    // Software pipelining (o.ahead = D): the relaxation terms of task t over
    // predecessors placed at least D positions earlier are emitted next to
    // the dependent per-device chain of task t - D, so the two interleave.
    // Status codes are still applied in try_place order inside the tail.
    const int D = std::max(0, o.ahead);
    std::vector<std::string> early(V);
    // TMEM tier: load every slot-resident predecessor value of task i that
    // is read by the early terms, then one wait with the registers tied to it
    auto tm_loads = [&](int i) {
        std::vector<int> qs;
        for (size_t k = 0; k < preds[i].size(); ++k) {
            const int q = preds[i][k];
            if (q > i - D - 1) continue;  // late term: a register value
            const bool in_reg = where[q] == -1 || (near > 0 && i - q <= near);
            if (!in_reg) qs.push_back(q);
        }
        const std::string is = std::to_string(i);
        // one asm block per group of <= 8: the loads into 32-bit temporaries,
        // one wait, then each pair moved into a true 64-bit output (a double
        // assembled from two separately-tied registers costs ptxas a
        // register-pair copy before every 64-bit use)
        // TMEM slot layout: {end lo, end hi} (2 columns per slot) or, with
        // tm_dev, {end lo, end hi, device, -} (4 columns; one .x4 load)
        const int cps = o.tm_dev ? 4 : 2;
        for (size_t c = 0; c < qs.size(); c += 8) {
            const size_t m = std::min(qs.size(), c + 8) - c;
            std::string body = "{\\n .reg .b32 ";
            for (size_t k = 0; k < m; ++k)
                body += (k ? ", " : "") + std::string("l") + std::to_string(k) + ", h" +
                        std::to_string(k) + (o.tm_dev ? ", x" + std::to_string(k) +
                                                         ", y" + std::to_string(k) : "");
            body += ";\\n";
            const size_t no = o.tm_dev ? 2 * m : m;  // outputs: value (+ device) each
            for (size_t k = 0; k < m; ++k) {
                const std::string ks = std::to_string(k);
                body += o.tm_dev
                    ? " tcgen05.ld.sync.aligned.32x32b.x4.b32 {l" + ks + ", h" + ks + ", x" + ks +
                          ", y" + ks + "}, [%" + std::to_string(no + k) + "];\\n"
                    : " tcgen05.ld.sync.aligned.32x32b.x2.b32 {l" + ks + ", h" + ks + "}, [%" +
                          std::to_string(no + k) + "];\\n";
            }
            body += " tcgen05.wait::ld.sync.aligned;\\n";
            for (size_t k = 0; k < m; ++k) {
                const std::string ks = std::to_string(k);
                body += " mov.b64 %" + ks + ", {l" + ks + ", h" + ks + "};\\n";
                if (o.tm_dev) body += " mov.b32 %" + std::to_string(m + k) + ", x" + ks + ";\\n";
            }
            body += "}";
            std::string outs, outs_d, ins;
            for (size_t k = 0; k < m; ++k) {
                const std::string v = "TV" + is + "_" + std::to_string(qs[c + k]);
                s += "    double " + v + ";\n";
                outs += std::string(k ? ", " : "") + "\"=d\"(" + v + ")";
                if (o.tm_dev) {
                    const std::string dv = "TD" + is + "_" + std::to_string(qs[c + k]);
                    s += "    int " + dv + ";\n";
                    outs_d += ", \"=r\"(" + dv + ")";
                }
                ins += std::string(k ? ", " : "") + "\"r\"(TB + " +
                       std::to_string(cps * where[qs[c + k]]) + "u)";
            }
            s += "    asm volatile(\"" + body + "\" : " + outs + outs_d + " : " + ins +
                 " : \"memory\");\n";
        }
    };
    auto head = [&](int i) {
        const std::string is = std::to_string(i), di = "d" + is;
        s += "    // " + p.task_ids[p.order[i]] + "\n";
        // genes were range-checked and clamped when the row was staged
        if (!greg && o.gword) {
            // one 32-bit shared-memory load per four genes (1 wavefront
            // instead of 4), bytes extracted in registers
            if ((i & 3) == 0)
                s += "    const hs_u32 GWD" + std::to_string(i >> 2) +
                     " = reinterpret_cast<const hs_u32 *>(g)[" + std::to_string(i >> 2) + "];\n";
            s += "    const int " + di + " = (int)((GWD" + std::to_string(i >> 2) + " >> " +
                 std::to_string(8 * (i & 3)) + ") & 0xFFu);\n";
        } else {
            s += "    const int " + di + " = " + (greg ? gexpr(i) : "g[" + is + "]") + ";\n";
        }
        if (greg && !preds[i].empty())
            s += "    const hs_u32 DP" + is + " = (hs_u32)" + di + " * 0x55555555u;\n";
        if (blk) s += "    const int n" + is + " = " + node_of(di) + ";\n";
        if (l.cls) s += "    int nl" + is + " = 0;\n";
        if (o.tmem) tm_loads(i);
        // early terms: predecessors placed at or before i - D - 1 (in edge
        // order; the max over them is exact in any order)
        std::vector<std::string> xs;
        for (size_t k = 0; k < preds[i].size(); ++k)
            if (preds[i][k] <= i - D - 1) {
                auto t = edge_terms(i, int(k), int(k) + 1);
                xs.push_back(t[0]);
            }
        if (!xs.empty())
            early[i] = domlike ? fold(xs, "re" + is, "0.0") : max_tree(xs, is + "e");
    };
    auto tail = [&](int i) {
        const std::string is = std::to_string(i), di = "d" + is;
        // try_place order (heuristics.py:92-106): batch size, memory, links,
        // latency entry; the first failing check decides the status
        if (!p.all_batch_ok) {
            std::snprintf(buf, sizeof buf,
                          "    st = first_status(st, !((0x%llxull >> %s) & 1ull), ST_BATCH);\n",
                          (unsigned long long)okmask, di.c_str());
            s += buf;
        }
        if (l.mem) {
            s += "    const hs_u32 M" + is + " = M + " + di + " * " + std::to_string(T * 8) +
                 ";\n";
            s += "    const double m" + is + " = ld_shared_f64(M" + is + ");\n";
            s += "    st = first_status(st, m" + is + " + " + lit(p.extra[i]) + " > CAP[" +
                 di + "], ST_MEMORY);\n";
        }
        std::vector<std::string> xs;
        for (size_t k = 0; k < preds[i].size(); ++k)
            if (preds[i][k] > i - D - 1) {
                auto t = edge_terms(i, int(k), int(k) + 1);
                xs.push_back(t[0]);
            }
        if (!early[i].empty() && !domlike) xs.push_back(early[i]);
        if (l.cls) s += "    st = first_status(st, nl" + is + ", ST_LINK);\n";
        if (!p.latency_complete) {
            uint64_t miss = 0;
            for (int k = 0; k < K; ++k)
                if (p.okL[k] && !p.dur_ok[size_t(i) * K + k]) miss |= 1ull << k;
            if (miss) {
                std::snprintf(buf, sizeof buf,
                              "    st = first_status(st, (0x%llxull >> %s) & 1ull, ST_MISSING);\n",
                              (unsigned long long)miss, di.c_str());
                s += buf;
            }
        }
        const std::string r = "r" + is;
        if (domlike)
            fold(xs, r, early[i].empty() ? "0.0" : early[i]);
        else if (xs.empty())
            s += "    const double " + r + " = 0.0;\n";
        else
            s += "    const double " + r + " = " + max_tree(xs, is) + ";\n";  // max(0.0, x) == x
        std::vector<std::string> av, du;
        for (int k = 0; k < K; ++k) {
            av.push_back("a" + std::to_string(k));
            du.push_back(lit(p.dur[size_t(i) * K + k]));
        }
        const std::string si = "s" + is, ei = "e" + is, Ai = "A" + is;
        if (l.avail) {
            s += "    const hs_u32 " + Ai + " = A + " + di + " * " + std::to_string(T * 8) +
                 ";\n";
            s += "    const double " + si + " = " + mx + "(" + r + ", ld_shared_f64(" + Ai +
                 "));\n";
        } else {
            s += "    const double " + si + " = " + mx + "(" + r + ", " + sel(di, av) + ");\n";
        }
        std::string dsrc = l.dur    ? "DUR[" + std::to_string(i * K) + " + " + di + "]"
                           : l.durg ? "__ldg(DG + " + std::to_string(i * K) + " + " + di + ")"
                                    : sel(di, du);
        if (l.dur || l.durg) {
            bool same = true;
            for (auto &v : du) same = same && v == du[0];
            if (same) dsrc = du[0];
        }
        s += "    const double " + ei + " = " + si + " + " + dsrc + ";\n";
        std::snprintf(buf, sizeof buf,
                      "    if (TRACE && valid) starts[cand * %d + %d] = %s;\n", V, i, si.c_str());
        s += buf;
        std::string stored = ei;
        if (dom && last[i] >= 0) {
            stored = "f" + is;
            // the constant from constant memory: a DADD operand (c[3][..]),
            // where an immediate double costs two UMOVs per task
            std::string cv = lit(prod_c[i]);
            if (!zero_c(i) && std::isfinite(prod_c[i])) {
                cv = "HSC[" + std::to_string(cconst.size()) + "]";
                cconst.push_back(prod_c[i]);
            }
            s += "    const double " + stored + " = " + (zero_c(i) ? ei : ei + " + " + cv) +
                 ";\n";
        }
        if (where[i] >= 0) {
            if (o.tmem && o.tm_dev)
                s += "    tm_st4(TB + " + std::to_string(4 * where[i]) + ", " + stored + ", " + di +
                     ");\n";
            else if (o.tmem)
                s += "    tm_st2(TB + " + std::to_string(2 * where[i]) + ", " + stored + ");\n";
            else
                s += "    E[" + std::to_string((long long)where[i] * T) + "] = " + stored + ";\n";
        }
        if (l.avail) {
            s += "    st_shared_f64(" + Ai + ", " + ei + ");\n";
        } else {
            for (int k = 0; k < K; ++k) {
                const std::string a = "a" + std::to_string(k);
                s += "    " + a + " = dsel(" + di + " == " + std::to_string(k) + ", " + ei +
                     ", " + a + ");\n";
            }
        }
        if (l.mem)
            s += "    st_shared_f64(M" + is + ", m" + is + " + " + lit(p.extra[i]) + ");\n";
    };
    // Optional CTA barrier every `sync` tasks (tile driver only, where every
    // thread of the CTA runs the body) to keep the warps of a CTA within one
    // window of the straight-line code. Measured (profiles r1h): no gain on
    // WS1000, whose fetch stalls come from the code streaming through the
    // instruction caches once per tile, and a loss on WS200 -- off by default.
    const int sync_every = std::max(0, o.sync);
    // a slot written at step q + D is read at step >= q + near + 1: waiting
    // for the stores every W <= near + 1 - D steps orders every store
    // before its first load
    const int wst = std::max(1, std::min(16, near + 1 - D));
    for (int t = 0; t < V + D; ++t) {
        if (o.tmem && t % wst == 0 && t > 0) s += "    tm_wait_st();\n";
        if (t < V) head(t);
        if (t - D >= 0) tail(t - D);
        if (sync_every && t % sync_every == sync_every - 1 && t + 1 < V + D)
            s += "    if (SYNC) __syncthreads();\n";
    }
    s += "    double ms = 0.0;\n";
    for (int k = 0; k < K; ++k)
        s += l.avail ? "    ms = pymax(ms, ld_shared_f64(A + " + std::to_string(k * T * 8) +
                           "));\n"
                     : "    ms = pymax(ms, a" + std::to_string(k) + ");\n";
    std::snprintf(buf, sizeof buf,
                  "    if (gene_bad) st = ST_GENE;\n"
                  "    ms_out = st ? (st >= ST_MISSING ? knan() : kinf()) : ms;\n"
                  "    st_out = st;\n}\n");
    s += buf;
    (void)checks;
    // pack16 over the row's 32-bit words (4 genes each) -> GPA[NP]
    auto pack_words = [&](const std::string &w) {
        std::string out = "    hs_u32 GPA[" + std::to_string(NP) + "];\n";
        for (int j = 0; j < NP; ++j) {
            std::string args;
            for (int q = 0; q < 4; ++q) {
                const int k = 4 * j + q;
                args += (q ? ", " : "") + (k < NW ? w + std::to_string(k) : std::string("0u"));
            }
            out += "    GPA[" + std::to_string(j) + "] = pack16(" + args + ");\n";
        }
        return out;
    };
    if (!cconst.empty()) {
        std::string decl = "__constant__ double HSC[" + std::to_string(cconst.size()) + "] = {";
        for (size_t k = 0; k < cconst.size(); ++k)
            decl += (k ? ", " : "") + lit(cconst[k]);
        decl += "};\n";
        const size_t at = s.find("template <bool TRACE");
        s.insert(at, decl);
    }
    s += "template <bool TRACE>\nstruct JitBody {\n  hs_u8 *smem; double *starts; double *eg; hs_u32 tb;\n  const double *dg;\n"
         "  __device__ __forceinline__ void run(const hs_u8 *g, int li, hs_i64 cand, "
         "bool valid, int gene_bad, double &ms, int &st) {\n";
    if (greg) {
        // the staged row was sanitised by eval_tiles: every byte <= K-1
        s += "    const hs_u32 *GW = reinterpret_cast<const hs_u32 *>(g);\n";
        for (int k = 0; k < NW; ++k)
            s += "    const hs_u32 w" + std::to_string(k) + " = GW[" + std::to_string(k) + "];\n";
        s += pack_words("w");
        s += "    jit_body<TRACE, true>(smem, GPA, li, cand, valid, gene_bad, starts, ms, st, eg, tb, dg);\n";
    } else {
        s += "    jit_body<TRACE, true>(smem, g, li, cand, valid, gene_bad, starts, ms, st, eg, tb, dg);\n";
    }
    s += "  }\n};\n";
    s += "template <bool TRACE, int MODE>\n__device__ __forceinline__ void jit_main("
         "const EvalParams &a, const SaParams *sa, const EaParams *ea) {\n"
         "  extern __shared__ __align__(16) hs_u8 smem[];\n";
    if (l.dur) s += stage(l.dur_off, "dur", int64_t(V) * K * 8);
    if (l.cls) {
        s += stage(l.ctab_off, "ctab", int64_t(V) * p.n_cls * 8);
        s += stage(l.bcl_off, "bclass", int64_t(K) * K * 2);
    }
    if (l.mem) s += stage(l.cap_off, "cap", int64_t(K) * 8);
    s += "  JitBody<TRACE> body;\n  body.smem = smem;\n  body.starts = a.starts;\n"
         "  body.eg = a.ends_g ? a.ends_g + blockIdx.x * a.ends_g_cta : nullptr;\n"
         "  body.tb = 0u;\n"
         "  body.dg = reinterpret_cast<const double *>(a.blob + a.lay.dur);\n";
    if (o.tmem) {
        // the TMEM of the SM (512 columns, or its share with tm_ctas CTAs
        // per SM): warp 0 allocates; each warp uses its lane quadrant and a
        // column band
        const std::string ncols = std::to_string(512 / std::max(1, o.tm_ctas));
        s += "  __shared__ hs_u32 tm_base_s;\n"
             "  if (threadIdx.x < 32) {\n"
             "    asm volatile(\"tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], " + ncols + ";\" "
             ":: \"r\"(smem_addr(&tm_base_s)) : \"memory\");\n"
             "    asm volatile(\"tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\" ::: \"memory\");\n"
             "  }\n"
             "  asm volatile(\"tcgen05.fence::before_thread_sync;\" ::: \"memory\");\n"
             "  __syncthreads();\n"
             "  asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n";
        s += "  body.tb = tm_base_s + ((((threadIdx.x >> 5) & 3u) * 32u) << 16) + (threadIdx.x >> 7) * " +
             std::to_string(o.tm_cols) + "u;\n";
    }
    s += "  if constexpr (MODE == 0) eval_tiles(a, smem, body);\n"
         "  else if constexpr (MODE == 1) sa_chain(a, *sa, smem, body);\n"
         "  else ea_chain(a, *ea, smem, body);\n";
    if (o.tmem)
        s += "  asm volatile(\"tcgen05.fence::before_thread_sync;\" ::: \"memory\");\n"
             "  __syncthreads();\n"
             "  if (threadIdx.x < 32) {\n"
             "    asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n"
             "    asm volatile(\"tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, " +
             std::to_string(512 / std::max(1, o.tm_ctas)) + ";\" "
             ":: \"r\"(tm_base_s) : \"memory\");\n"
             "  }\n";
    s += "}\n";
    const int min_blocks = o.tmem ? std::max(1, o.tm_ctas) : 1;
    std::snprintf(buf, sizeof buf,
                  "extern \"C\" __global__ void __launch_bounds__(%d, %d) "
                  "hs_jit_eval(const EvalParams a) { jit_main<false, 0>(a, nullptr, nullptr); }\n"
                  "extern \"C\" __global__ void __launch_bounds__(%d, %d) "
                  "hs_jit_trace(const EvalParams a) { jit_main<true, 0>(a, nullptr, nullptr); }\n",
                  T, min_blocks, T, min_blocks);
    s += buf;
    if (jit_search_ok(p) && o.sync == 0) {
        // single-CTA search drivers (SA K10, EA K9) over the specialised body
        // (they leave idle warps out of a round: no CTA barriers in the body)
        std::snprintf(buf, sizeof buf,
                      "extern \"C\" __global__ void __launch_bounds__(%d, 1) "
                      "hs_jit_sa(const EvalParams a, const SaParams e) "
                      "{ jit_main<false, 1>(a, &e, nullptr); }\n"
                      "extern \"C\" __global__ void __launch_bounds__(%d, 1) "
                      "hs_jit_ea(const EvalParams a, const EaParams e) "
                      "{ jit_main<false, 2>(a, nullptr, &e); }\n",
                      T, T);
        s += buf;
    }
    if (greg) {
        // Direct-load kernel: no genome tile and no CTA barrier per tile.
        // Each thread reads its own row from global memory (L1-cached
        // 32-bit loads: a warp's 32 rows are one contiguous span), clamps
        // and flags genes >= K, packs them into registers and evaluates;
        // shared memory holds only the tables and the per-lane state, so
        // several CTAs share an SM.
        std::snprintf(buf, sizeof buf,
                      "extern \"C\" __global__ void __launch_bounds__(%d, %d) "
                      "hs_jit_direct(const EvalParams a) {\n"
                      "  extern __shared__ __align__(16) hs_u8 smem[];\n", T, std::max(1, o.ctas));
        s += buf;
        if (l.dur) s += stage(l.dur_off, "dur", int64_t(V) * K * 8);
        if (l.cls) {
            s += stage(l.ctab_off, "ctab", int64_t(V) * p.n_cls * 8);
            s += stage(l.bcl_off, "bclass", int64_t(K) * K * 2);
        }
        if (l.mem) s += stage(l.cap_off, "cap", int64_t(K) * 8);
        s += "  __syncthreads();\n"
             "  double *EGC = a.ends_g ? a.ends_g + blockIdx.x * a.ends_g_cta : nullptr;\n"
             "  const int li = threadIdx.x;\n"
             "  double bc = kinf();\n  hs_i64 bi = 0x7fffffffffffffffll;\n"
             "  const hs_i64 stride = (hs_i64)gridDim.x * blockDim.x;\n";
        std::snprintf(buf, sizeof buf, "  const hs_u32 kmax = 0x%08xu;\n",
                      unsigned(K - 1) * 0x01010101u);
        s += buf;
        s += "  for (hs_i64 cand = (hs_i64)blockIdx.x * blockDim.x + li; cand < a.n; "
             "cand += stride) {\n"
             "    const hs_u32 *rw = reinterpret_cast<const hs_u32 *>(a.genes + cand * a.ld);\n";
        for (int k = 0; k < NW; ++k)
            s += "    hs_u32 w" + std::to_string(k) + " = __ldg(rw + " + std::to_string(k) +
                 ");\n";
        // the next row of this thread into L2 while this one computes
        s += "    if (cand + stride < a.n) {\n"
             "      const hs_u8 *nx = a.genes + (cand + stride) * a.ld;\n";
        for (int off = 0; off < 4 * NW; off += 128)
            s += "      asm volatile(\"prefetch.global.L2 [%0];\" :: \"l\"(nx + " +
                 std::to_string(off) + "));\n";
        s += "      asm volatile(\"prefetch.global.L2 [%0];\" :: \"l\"(nx + " +
             std::to_string(4 * NW - 1) + "));\n    }\n";
        s += "    hs_u32 over = 0u;\n";
        for (int k = 0; k < NW; ++k) {
            const std::string w = "w" + std::to_string(k);
            std::string ov = "__vcmpgtu4(" + w + ", kmax)";
            if (k == NW - 1 && (V & 3)) {
                char mk[32];
                std::snprintf(mk, sizeof mk, "0x%xu", (1u << (8 * (V & 3))) - 1u);
                ov = "(" + ov + " & " + mk + ")";
            }
            s += "    over |= " + ov + ";\n    " + w + " = __vminu4(" + w + ", kmax);\n";
        }
        s += pack_words("w");
        s += "    double ms;\n    int st;\n"
             "    jit_body<false, false>(smem, GPA, li, cand, true, over != 0u, nullptr, ms, st, EGC, 0u, "
             "reinterpret_cast<const double *>(a.blob + a.lay.dur));\n"
             "    if (a.makespan) a.makespan[cand] = ms;\n"
             "    if (a.status) a.status[cand] = (hs_u8)st;\n"
             "    const double key = (ms != ms) ? kinf() : ms;\n"
             "    const hs_i64 gidx = a.index_base + cand;\n"
             "    if (best_less(key, gidx, bc, bi)) {\n      bc = key;\n      bi = gidx;\n    }\n"
             "  }\n"
             "  if (a.best) reduce_best(bc, bi, a.partial, a.ticket, a.best);\n}\n";
    }
    return next;
}

bool jit_search_ok(const Plan &p) {
    // the search kernels double the inlined straight-line code: only where
    // NVRTC stays fast
    if (const char *v = getenv("HS_JIT_SEARCH"))
        if (!atoi(v)) return false;
    return p.V <= 512 && !p.batched;
}

int jit_build(const Plan &p, int device, JitModule **out, std::string *err) {
    if (!jit_eligible(p)) {
        if (err) *err = "plan not eligible for the specialised evaluator";
        return HS_EINVAL;
    }
    Nvrtc &nv = nvrtc();
    if (!nv.ok) {
        if (err) *err = "libnvrtc.so.12 not found";
        return HS_ECUDA;
    }
    auto t0 = std::chrono::steady_clock::now();
    int optin = 0, sms = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const JitOpts o = JitOpts::from_env();
    const int slots = p.batched ? jit_emit_batched(p, 32, o, nullptr, true)
                                : jit_emit(p, 32, o, nullptr);
    const int ld_cap = p.pref_ld() + 16;
    const int64_t head = head_bytes(p, o);
    const int64_t budget = int64_t(optin) - head - 1024;
    JitOpts ob = o;  // slots in shared memory
    ob.tmem = false;
    // no end-time slots and the device state in shared memory (K > 4, the
    // multi-server platforms): 12 warps like the TMEM tier (tf96 +11 %,
    // profiles r2o); otherwise `lanes`
    const int cap_lanes = slots == 0 && p.K > kMaxRegK && !o.lanes_set
                              ? std::max(o.lanes, o.tm_lanes) : o.lanes;
    auto lanes_for = [&](bool db) {
        return int(std::min<int64_t>(budget / per_lane_bytes(p, ob, slots, ld_cap, db),
                                     cap_lanes) / 32 * 32);
    };
    // double-buffer the genome tile only when it costs no lanes
    bool dbuf = lanes_for(true) >= lanes_for(false);
    int T = lanes_for(dbuf);
    JitOpts oe = ob;
    // too few lanes with the end times in shared memory: move them to the
    // global-memory tier ([slot][lane] per CTA, L2-resident; `gslot_lanes`
    // bounds the footprint SMs x lanes x slots x 8 B)
    int smem_sm_all = 0;
    cudaDeviceGetAttribute(&smem_sm_all, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
    const int64_t smem_lanes_sm =
        p.batched && slots > 0
            ? int64_t(T) * std::max<int64_t>(1, smem_sm_all /
                                                   (bat_layout(p, std::max(T, 32), slots, ld_cap,
                                                               dbuf).total + 1024))
            : 0;
    if (p.batched && slots > 0 && smem_lanes_sm < o.gslot_lanes) {
        // K8': the parts' slots to the global-memory tier when shared
        // memory holds fewer lanes per SM than that tier runs (r4e, WS200:
        // L = 2 109 lanes in shared memory 2.5e8 -> 192 lanes 5.9e8 cand/s;
        // jit_batched_ok)
        JitOpts og = ob;
        og.gslots = true;
        auto lanes_g = [&](bool db) {
            return int(std::min<int64_t>(budget / per_lane_bytes(p, og, slots, ld_cap, db),
                                         std::min(o.lanes, o.gslot_lanes)) / 32 * 32);
        };
        const bool dg = lanes_g(true) >= lanes_g(false);
        if (lanes_g(dg) > T) {
            oe.gslots = true;
            dbuf = dg;
            T = lanes_g(dg);
        }
    }
    if (T < 128 && slots > 0 && !p.batched) {
        JitOpts og = ob;
        og.gslots = true;
        auto lanes_g = [&](bool db) {
            return int(std::min<int64_t>(budget / per_lane_bytes(p, og, slots, ld_cap, db),
                                         std::min(o.lanes, o.gslot_lanes)) / 32 * 32);
        };
        const bool dg = lanes_g(true) >= lanes_g(false);
        if (lanes_g(dg) > T) {
            oe.gslots = true;
            dbuf = dg;
            T = lanes_g(dg);
        }
    }
    // tensor-memory tier (o.tmem): the end-time slots move to TMEM (512
    // columns x 128 lanes per SM), shared memory keeps tiles and tables
    // with its own lane count and long-lived register budget (more warps,
    // fewer registers each); otherwise the shared-memory sizing above stands
    int n_slots = slots;
    if (o.tmem && !oe.gslots && slots > 0 && !p.batched) {
        JitOpts ot = o;
        ot.lanes = o.tm_lanes / o.tm_ctas;
        ot.reg_budget = o.tm_regs;
        const int slots_t = jit_emit(p, 32, ot, nullptr);
        // several CTAs per SM share its shared memory and its 512 columns
        int smem_sm = 0;
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
        const int64_t budget_t = o.tm_ctas > 1
            ? std::min<int64_t>(budget, int64_t(smem_sm) / o.tm_ctas - 1024 - head - 1024)
            : budget;
        auto lanes_t = [&](bool db) {
            return int(std::min<int64_t>(budget_t / per_lane_bytes(p, ot, slots_t, ld_cap, db),
                                         ot.lanes) / 32 * 32);
        };
        const bool dt = lanes_t(true) >= lanes_t(false);
        const int Tt = std::min(lanes_t(dt), 512);
        const int groups = (Tt / 32 + 3) / 4;
        // column bands 4-aligned (the .x4 slot accesses start on them)
        const int cols = groups > 0 ? (512 / o.tm_ctas / groups) & ~3 : 0;
        if (Tt >= 32 && slots_t > 0 && (ot.tm_dev ? 4 : 2) * slots_t > cols)
            ot.tm_dev = false;  // the device column does not fit: end times only
        if (Tt >= 32 && slots_t > 0 && 2 * slots_t <= cols) {
            oe = ot;
            oe.tm_cols = cols;
            dbuf = dt;
            T = Tt;
            n_slots = slots_t;
        } else if (Tt >= 32 && slots_t == 0) {
            // every end time fits the smaller register budget: the same
            // 12-warp configuration without any slot tier
            oe = ot;
            oe.tmem = false;
            dbuf = dt;
            T = Tt;
            n_slots = 0;
        }
    }
    oe.tmem = oe.tmem && oe.tm_cols > 0;
    if (T < 32) {
        if (err) *err = "graph too large for the specialised evaluator";
        return HS_EINVAL;
    }
    if (p.batched) {
        // K8': lanes per SM, not per CTA, is what hides latency. A CTA
        // whose tables + tiles take more than half of the SM's shared memory
        // leaves it at one CTA (Inception-v3 at L = 4: 140 KB -> 256 lanes
        // per SM where ResNet-50's 114 KB CTAs run two): search the lane
        // count and tile double-buffering for the most resident lanes per SM
        // (ties: the larger CTA, then double-buffered)
        int smem_sm = 0;
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
        const int ns = oe.gslots ? 0 : slots;
        // at most two CTAs per SM: three single-buffered 224-lane CTAs
        // (672 lanes, 97 registers) ran ResNet-50 at L = 4 at 1.5e9 where
        // two double-buffered 256-lane CTAs run 2.2e9 (r4g vs r4c)
        auto per_sm = [&](int t, bool db, int *ctas) {
            const int64_t sm = bat_layout(p, t, ns, ld_cap, db).total;
            if (sm > optin - 1024) return 0;
            *ctas = int(std::min<int64_t>({int64_t(2048 / t), int64_t(smem_sm) / (sm + 1024), 2}));
            // the global slot tier's L2 footprint grows with the lanes per SM
            if (oe.gslots) *ctas = std::min(*ctas, std::max(1, o.gslot_lanes / t));
            return t * *ctas;
        };
        int c0 = 1;
        int best = per_sm(T, dbuf, &c0), bctas = 0;
        // only where the default configuration leaves one CTA per SM (and
        // not under HS_JIT_OPTS=lanes=N): elsewhere it stays as shared
        // memory allows (ResNet-50 at L = 2: three 256-lane CTAs)
        for (int db = 1; db >= 0 && c0 < 2 && !o.lanes_set; --db)
            for (int t = std::min(o.lanes, 512) / 32 * 32; t >= 64; t -= 32) {
                int c = 1;
                const int l = per_sm(t, db != 0, &c);
                if (l > best) {
                    best = l;
                    T = t;
                    dbuf = db != 0;
                    bctas = c;
                }
            }
        if (bctas > 0) oe.ctas = bctas;  // the searched configuration
    }
    std::string src;
    oe.dbuf = dbuf;
    if (p.batched)
        jit_emit_batched(p, T, oe, &src, dbuf);
    else
        jit_emit(p, T, oe, &src);
    const char *hdr_src[] = {kEvalCommonSrc};
    const char *hdr_name[] = {"eval_common.cuh"};
    nvrtcProgram_t prog = nullptr;
    if (nv.create(&prog, src.c_str(), "hs_jit.cu", 1, hdr_src, hdr_name) != 0) {
        if (err) *err = "nvrtcCreateProgram failed";
        return HS_ECUDA;
    }
    const char *opts[] = {"--gpu-architecture=sm_100a", "--std=c++17",
                          "--fmad=false", "-lineinfo", "--restrict"};
    const int rc = nv.compile(prog, 5, opts);
    size_t lsz = 0;
    nv.log_size(prog, &lsz);
    std::string log(lsz, '\0');
    if (lsz) nv.log(prog, &log[0]);
    if (rc != 0) {
        nv.destroy(&prog);
        if (err) *err = "NVRTC compile failed: " + log.substr(0, 2000);
        return HS_ECUDA;
    }
    size_t csz = 0;
    nv.cubin_size(prog, &csz);
    std::vector<char> cubin(csz);
    nv.cubin(prog, cubin.data());
    nv.destroy(&prog);
    // HS_JIT_DUMP=<dir>: keep the emitted source and cubin (cuobjdump -sass
    // for the SASS listings under profiles/)
    if (const char *dir = getenv("HS_JIT_DUMP")) {
        char stem[512];
        std::snprintf(stem, sizeof stem, "%s/hs_jit_V%d_E%d_K%d_L%d_T%d", dir, p.V, p.E,
                      p.K, p.L, T);
        if (FILE *f = std::fopen((std::string(stem) + ".cu").c_str(), "wb")) {
            std::fwrite(src.data(), 1, src.size(), f);
            std::fclose(f);
        }
        if (FILE *f = std::fopen((std::string(stem) + ".cubin").c_str(), "wb")) {
            std::fwrite(cubin.data(), 1, cubin.size(), f);
            std::fclose(f);
        }
    }

    JitModule *m = new JitModule();
    m->device = device;
    m->T = m->lanes = T;
    m->slots = n_slots;
    m->ld_cap = ld_cap;
    m->opts = oe;
    m->ends_global = oe.gslots;
    m->tmem = oe.tmem;
    if (p.batched) {
        const BatLayout l = bat_layout(p, T, oe.gslots ? 0 : n_slots, ld_cap, dbuf);
        m->smem_tile = l.tile;
        m->smem_tile2 = l.tile2;
        m->smem_ends = l.ends;
        m->smem_kstate = l.avail;
        m->smem = size_t(l.total);
    } else {
        const JitLayout l = jit_layout(p, oe, T, n_slots, ld_cap, dbuf);
        m->smem_tile = l.tile;
        m->smem_tile2 = l.tile2;
        m->smem_ends = l.ends;
        m->smem_kstate = l.avail_off;
        m->smem = size_t(l.total);
    }
    cudaError_t e = cudaLibraryLoadData(&m->lib, cubin.data(), nullptr, nullptr, 0,
                                        nullptr, nullptr, 0);
    if (e == cudaSuccess) e = cudaLibraryGetKernel(&m->kern, m->lib, "hs_jit_eval");
    if (e == cudaSuccess) e = cudaLibraryGetKernel(&m->kern_trace, m->lib, "hs_jit_trace");
    if (e == cudaSuccess)
        e = cudaKernelSetAttributeForDevice(
            m->kern_trace, cudaFuncAttributeMaxDynamicSharedMemorySize, int(m->smem), device);
    if (e == cudaSuccess)
        e = cudaKernelSetAttributeForDevice(
            m->kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(m->smem), device);
    if (e == cudaSuccess && jit_search_ok(p) &&
        cudaLibraryGetKernel(&m->kern_sa, m->lib, "hs_jit_sa") == cudaSuccess) {
        e = cudaLibraryGetKernel(&m->kern_ea, m->lib, "hs_jit_ea");
        if (e == cudaSuccess)
            e = cudaKernelSetAttributeForDevice(
                m->kern_sa, cudaFuncAttributeMaxDynamicSharedMemorySize, int(m->smem), device);
        if (e == cudaSuccess)
            e = cudaKernelSetAttributeForDevice(
                m->kern_ea, cudaFuncAttributeMaxDynamicSharedMemorySize, int(m->smem), device);
    }
    if (e == cudaSuccess && o.genes_reg && p.K <= 4) {
        m->smem_direct = size_t(m->smem_tile);
        e = cudaLibraryGetKernel(&m->kern_direct, m->lib, "hs_jit_direct");
        if (e == cudaSuccess)
            e = cudaKernelSetAttributeForDevice(m->kern_direct,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                int(m->smem_direct), device);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &m->blocks_per_sm_direct, (const void *)m->kern_direct, T, m->smem_direct);
        if (e == cudaSuccess && m->blocks_per_sm_direct < 1)
            e = cudaErrorInvalidConfiguration;
    }
    if (e != cudaSuccess) {
        if (m->lib) cudaLibraryUnload(m->lib);
        delete m;
        if (err) *err = std::string("loading the specialised kernel: ") +
                        cudaGetErrorString(e);
        return HS_ECUDA;
    }
    int smem_sm = 0;
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
    m->blocks_per_sm = std::max(1, std::min(2048 / T, int(smem_sm / (m->smem + 1024))));
    // each CTA allocates 512 / tm_ctas TMEM columns
    if (m->tmem) m->blocks_per_sm = std::min(m->blocks_per_sm, oe.tm_ctas);
    // K8': the CTAs per SM the lane search sized it for (launch bounds, L2)
    if (p.batched && oe.ctas > 1) m->blocks_per_sm = std::min(m->blocks_per_sm, oe.ctas);
    m->sms = sms;
    m->src_bytes = src.size();
    m->compile_ms = std::chrono::duration<double, std::milli>(
                        std::chrono::steady_clock::now() - t0).count();
    *out = m;
    return HS_OK;
}

void jit_free(JitModule *m) {
    if (!m) return;
    if (m->lib) cudaLibraryUnload(m->lib);
    delete m;
}

bool jit_direct_ok(const JitModule &m, const hsk::EvalParams &a) {
    return m.kern_direct && !a.starts && !a.gen && !a.packed && a.ld % 4 == 0 &&
           (reinterpret_cast<uintptr_t>(a.genes) & 3) == 0;
}

int jit_launch_search(const JitModule &m, int mode, const hsk::EvalParams &a,
                      const void *ps, cudaStream_t stream, std::string *err, int grid) {
    const cudaKernel_t k = mode == 1 ? m.kern_sa : m.kern_ea;
    if (!k) {
        if (err) *err = "specialised module has no search kernels";
        return HS_EINVAL;
    }
    void *args[] = {(void *)&a, const_cast<void *>(ps)};
    cudaError_t e = cudaLaunchKernel((const void *)k, dim3(grid), dim3(m.T), args, m.smem, stream);
    if (e != cudaSuccess) {
        if (err) *err = std::string("specialised search launch: ") + cudaGetErrorString(e);
        return HS_ECUDA;
    }
    return HS_OK;
}

int jit_launch(const JitModule &m, const hsk::EvalParams &a, int grid, cudaStream_t stream,
               std::string *err) {
    void *args[] = {(void *)&a};
    const bool direct = jit_direct_ok(m, a);
    const cudaKernel_t k = a.starts ? m.kern_trace : direct ? m.kern_direct : m.kern;
    cudaError_t e = cudaLaunchKernel((const void *)k, dim3(grid), dim3(m.T), args,
                                     direct ? m.smem_direct : m.smem, stream);
    if (e != cudaSuccess) {
        if (err) *err = std::string("specialised eval launch: ") + cudaGetErrorString(e);
        return HS_ECUDA;
    }
    return HS_OK;
}

}  // namespace hs
