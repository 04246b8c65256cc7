// Per-graph specialised evaluator: the plan is emitted as straight-line
// CUDA (one block of code per task placement, the graph's predecessor
// positions, end-time slots, communication and latency constants baked in
// as immediates), compiled by NVRTC for sm_100a at plan time and driven by
// the same tile loop as the ahead-of-time kernel (eval_common.cuh).
//
// Compared with walking node/edge records, this removes every plan load and
// address computation from the inner loop, keeps short-lived end times in
// registers, and lets ptxas schedule the loads of later placements early.
// The arithmetic is the same binary64 sequence as the reference decoder
// (heuristics.py:43-148); results are checked bit-for-bit against the
// golden fixtures by the same GPU tests as the AOT kernel.
//
// Scope (everything else uses the AOT kernel): K <= 4 devices, one
// bandwidth over a full mesh, and no capacity / batch-size / missing-entry /
// NaN cases (plan flags clear) -- the benchmark graphs of the paper.
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
            if (k == "lanes") o.lanes = std::max(32, std::min(1024, std::atoi(v.c_str())));
        }
        at = end + 1;
    }
    return o;
}

static int64_t a16(int64_t x) { return (x + 15) & ~int64_t(15); }

// Straight-line code grows with V + E and ptxas time super-linearly
// (minutes at V ~ 1000), so very large graphs stay on the AOT kernel.
constexpr int kJitMaxV = 512, kJitMaxE = 2048, kJitMaxK = 64;

bool jit_eligible(const Plan &p) {
    return !p.batched && p.K <= kJitMaxK && !p.nan_possible && p.V > 0 &&
           p.V <= kJitMaxV && p.E <= kJitMaxE;
}

namespace {

// Shared-memory layout of the specialised kernel (byte offsets); every
// table is staged from the plan blob once per CTA.
struct JitLayout {
    bool dur = false, cls = false, mem = false, avail = false, dbuf = true;
    int64_t dur_off = 0, ctab_off = 0, bcl_off = 0, cap_off = 0, head = 16;
    int64_t tile = 0, tile2 = 0, ends = 0, avail_off = 0, mem_off = 0, total = 0;
};

JitLayout jit_layout(const Plan &p, const JitOpts &o, int T, int slots, int ld_cap,
                     bool dbuf = true) {
    JitLayout l;
    l.dbuf = dbuf;
    l.dur = o.dur_smem || p.K > 4;
    l.avail = o.avail_smem || p.K > 4;
    l.cls = !p.uniform_comm;
    l.mem = p.mem_check;
    int64_t at = 16;
    if (l.dur) { l.dur_off = at; at += a16(int64_t(p.V) * p.K * 8); }
    if (l.cls) {
        l.ctab_off = at; at += a16(int64_t(p.V) * p.n_cls * 8);
        l.bcl_off = at; at += a16(int64_t(p.K) * p.K * 2);
    }
    if (l.mem) { l.cap_off = at; at += a16(int64_t(p.K) * 8); }
    l.head = at;
    l.tile = at;
    l.tile2 = dbuf ? l.tile + a16(int64_t(T) * ld_cap) : 0;
    l.ends = l.tile + a16(int64_t(T) * ld_cap) * (dbuf ? 2 : 1);
    at = l.ends + int64_t(slots) * T * 8;
    if (l.avail) { l.avail_off = at; at += int64_t(p.K) * T * 8; }
    if (l.mem) { l.mem_off = at; at += int64_t(p.K) * T * 8; }
    l.total = at;
    return l;
}

int64_t per_lane_bytes(const Plan &p, const JitOpts &o, int slots, int ld_cap,
                       bool dbuf) {
    const bool avail = o.avail_smem || p.K > 4;
    return (dbuf ? 2 : 1) * ld_cap + int64_t(slots) * 8 + (avail ? 8 * p.K : 0) + (p.mem_check ? 8 * p.K : 0);
}

int64_t head_bytes(const Plan &p, const JitOpts &o) {
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

// Emits the kernel for T lanes; returns the number of shared-memory slots.
int jit_emit(const Plan &p, int T, const JitOpts &o, std::string *src) {
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
    {
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
    s += "template <bool TRACE>\n__device__ __forceinline__ void jit_body(hs_u8 *smem, "
         "const hs_u8 *g, int li, hs_i64 cand, bool valid, int gene_bad, double *starts, "
         "double &ms_out, int &st_out) {\n";
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
    s += "    int st = 0;\n";
    uint64_t okmask = 0;
    for (int k = 0; k < K; ++k)
        if (p.okL[k]) okmask |= 1ull << k;
    for (int i = 0; i < V; ++i) {
        const std::string is = std::to_string(i);
        const std::string di = "d" + is;
        s += "    // " + p.task_ids[p.order[i]] + "\n";
        // raw gene for the range check; clamped for table / state indexing
        // (lanes past the last row read stale tile bytes)
        // genes were range-checked and clamped when the row was staged
        s += "    const int " + di + " = g[" + is + "];\n";
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
        if (l.cls) s += "    int nl" + is + " = 0;\n";
        for (size_t k = 0; k < preds[i].size(); ++k) {
            const int q = preds[i][k];
            const EdgeRec &er = p.edges[p.nodes[i].e_begin + k];
            const std::string endq = where[q] == -1
                ? "e" + std::to_string(q)
                : "E[" + std::to_string((long long)where[q] * T) + "]";
            const std::string gq = where[q] == -1
                ? "d" + std::to_string(q)
                : "(int)g[" + std::to_string(q) + "]";
            const std::string x = "x" + is + "_" + std::to_string(k);
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
            } else {
                s += "    const double " + x + " = " + endq + " + dsel(" + gq + " == " + di +
                     ", 0.0, " + lit(er.c) + ");\n";
            }
            xs.push_back(x);
        }
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
        // max over predecessors: a balanced tree (no NaN can occur, so max
        // is associative and the result equals the reference's fold)
        const std::string r = "r" + is;
        if (xs.empty()) {
            s += "    const double " + r + " = 0.0;\n";
        } else {
            int lvl = 0;
            while (xs.size() > 1) {
                std::vector<std::string> nx;
                for (size_t k = 0; k + 1 < xs.size(); k += 2) {
                    const std::string m = "m" + is + "_" + std::to_string(lvl) + "_" +
                                          std::to_string(k);
                    s += "    const double " + m + " = " + mx + "(" + xs[k] + ", " +
                         xs[k + 1] + ");\n";
                    nx.push_back(m);
                }
                if (xs.size() & 1) nx.push_back(xs.back());
                xs.swap(nx);
                ++lvl;
            }
            s += "    const double " + r + " = " + xs[0] + ";\n";  // max(0.0, x) == x
        }
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
        std::string dsrc = l.dur ? "DUR[" + std::to_string(i * K) + " + " + di + "]" : sel(di, du);
        if (l.dur) {
            bool same = true;
            for (auto &v : du) same = same && v == du[0];
            if (same) dsrc = du[0];
        }
        s += "    const double " + ei + " = " + si + " + " + dsrc + ";\n";
        std::snprintf(buf, sizeof buf,
                      "    if (TRACE && valid) starts[cand * %d + %d] = %s;\n", V, i, si.c_str());
        s += buf;
        if (where[i] >= 0)
            s += "    E[" + std::to_string((long long)where[i] * T) + "] = " + ei + ";\n";
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
    s += "template <bool TRACE>\nstruct JitBody {\n  hs_u8 *smem; double *starts;\n"
         "  __device__ __forceinline__ void run(const hs_u8 *g, int li, hs_i64 cand, "
         "bool valid, int gene_bad, double &ms, int &st) {\n"
         "    jit_body<TRACE>(smem, g, li, cand, valid, gene_bad, starts, ms, st);\n  }\n};\n";
    s += "template <bool TRACE>\n__device__ __forceinline__ void jit_main(const EvalParams &a) {\n"
         "  extern __shared__ __align__(16) hs_u8 smem[];\n";
    if (l.dur) s += stage(l.dur_off, "dur", int64_t(V) * K * 8);
    if (l.cls) {
        s += stage(l.ctab_off, "ctab", int64_t(V) * p.n_cls * 8);
        s += stage(l.bcl_off, "bclass", int64_t(K) * K * 2);
    }
    if (l.mem) s += stage(l.cap_off, "cap", int64_t(K) * 8);
    s += "  JitBody<TRACE> body;\n  body.smem = smem;\n  body.starts = a.starts;\n"
         "  eval_tiles(a, smem, body);\n}\n";
    std::snprintf(buf, sizeof buf,
                  "extern \"C\" __global__ void __launch_bounds__(%d, 1) "
                  "hs_jit_eval(const EvalParams a) { jit_main<false>(a); }\n"
                  "extern \"C\" __global__ void __launch_bounds__(%d, 1) "
                  "hs_jit_trace(const EvalParams a) { jit_main<true>(a); }\n", T, T);
    s += buf;
    return next;
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
    const int slots = jit_emit(p, 32, o, nullptr);
    const int ld_cap = p.pref_ld() + 16;
    const int64_t head = head_bytes(p, o);
    const int64_t budget = int64_t(optin) - head - 1024;
    auto lanes_for = [&](bool db) {
        return int(std::min<int64_t>(budget / per_lane_bytes(p, o, slots, ld_cap, db),
                                     o.lanes) / 32 * 32);
    };
    // double-buffer the genome tile only when it costs no lanes
    const bool dbuf = lanes_for(true) >= lanes_for(false);
    int T = lanes_for(dbuf);
    if (T < 32) {
        if (err) *err = "graph too large for the specialised evaluator";
        return HS_EINVAL;
    }
    std::string src;
    JitOpts oe = o;
    oe.dbuf = dbuf;
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

    JitModule *m = new JitModule();
    m->device = device;
    m->T = m->lanes = T;
    m->slots = slots;
    m->ld_cap = ld_cap;
    m->opts = o;
    {
        const JitLayout l = jit_layout(p, o, T, slots, ld_cap, dbuf);
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

int jit_launch(const JitModule &m, const hsk::EvalParams &a, int grid, cudaStream_t stream,
               std::string *err) {
    void *args[] = {(void *)&a};
    const cudaKernel_t k = a.starts ? m.kern_trace : m.kern;
    cudaError_t e = cudaLaunchKernel((const void *)k, dim3(grid), dim3(m.T), args,
                                     m.smem, stream);
    if (e != cudaSuccess) {
        if (err) *err = std::string("specialised eval launch: ") + cudaGetErrorString(e);
        return HS_ECUDA;
    }
    return HS_OK;
}

}  // namespace hs
