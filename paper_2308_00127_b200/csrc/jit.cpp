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
        }
        at = end + 1;
    }
    return o;
}

static int64_t dur_bytes(const Plan &p) {
    return (int64_t(p.V) * p.K * 8 + 15) & ~int64_t(15);
}

// Straight-line code grows with V + E and ptxas time super-linearly
// (minutes at V ~ 1000), so very large graphs stay on the AOT kernel.
constexpr int kJitMaxV = 512, kJitMaxE = 2048;

bool jit_eligible(const Plan &p) {
    return !p.batched && p.K <= 4 && p.uniform_comm && !p.mem_check && p.all_batch_ok &&
           p.latency_complete && !p.nan_possible && p.V > 0 &&
           p.V <= kJitMaxV && p.E <= kJitMaxE;
}

// Emits the body for T lanes. Returns the number of shared-memory slots.
int jit_emit(const Plan &p, int T, const JitOpts &o, std::string *src) {
    const int V = p.V, K = p.K;
    const int reg_budget = o.reg_budget, reg_window = o.reg_window;
    // lifetimes in genome order
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
    {
        std::vector<std::vector<int>> dies(V);
        for (int i = 0; i < V; ++i)
            if (last[i] >= 0) dies[last[i]].push_back(i);
        std::priority_queue<int, std::vector<int>, std::greater<int>> freel;
        int next = 0, live_regs = 0;
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
        if (src == nullptr) return next;
        (void)0;
        std::string &s = *src;
        s.clear();
        s += "#include \"eval_common.cuh\"\nusing namespace hsk;\n";
        s += "template <bool TRACE>\nstruct JitBody {\n  double *ends; double *avail; "
             "const double *dur; double *starts;\n";
        s += "  __device__ __forceinline__ void run(const hs_u8 *g, int li, "
             "hs_i64 cand, bool valid, double &ms_out, int &st_out) {\n";
        s += "    double *E = ends + li;\n";
        if (o.avail_smem) {
            s += "    double *A = avail + li;\n";
            for (int k = 0; k < K; ++k)
                s += "    A[" + std::to_string(k * T) + "] = 0.0;\n";
        } else {
            for (int k = 0; k < K; ++k)
                s += "    double a" + std::to_string(k) + " = 0.0;\n";
        }
        s += "    int gmax = 0;\n";
        // no NaN and no negative times inside the specialised scope: max on
        // the binary64 bit patterns equals Python's max (ALU, not FP64)
        const std::string mx = o.int_max ? "pymax_nn" : "pymax";
        char buf[1024];
        for (int i = 0; i < V; ++i) {
            const std::string di = "d" + std::to_string(i);
            s += "    // " + p.task_ids[p.order[i]] + "\n";
            // raw gene for the range check; clamped for table / state
            // indexing (lanes past the last row read stale tile bytes)
            std::snprintf(buf, sizeof buf,
                          "    const int g%d = g[%d]; gmax = max(gmax, g%d);\n"
                          "    const int %s = min(g%d, %d);\n",
                          i, i, i, di.c_str(), i, K - 1);
            s += buf;
            // arrivals of the predecessors (ready_time, :67-78)
            std::vector<std::string> xs;
            for (size_t k = 0; k < preds[i].size(); ++k) {
                const int q = preds[i][k];
                const EdgeRec &er = p.edges[p.nodes[i].e_begin + k];
                const std::string endq = where[q] == -1
                    ? "e" + std::to_string(q)
                    : "E[" + std::to_string((long long)where[q] * T) + "]";
                const std::string gq = where[q] == -1
                    ? "d" + std::to_string(q) : "(int)g[" + std::to_string(q) + "]";
                const std::string x = "x" + std::to_string(i) + "_" + std::to_string(k);
                if (er.c == 0.0 && !std::signbit(er.c)) {
                    // zero-byte output: end + 0.0 == end for end >= +0
                    s += "    const double " + x + " = " + endq + ";\n";
                } else {
                    s += "    const double " + x + " = " + endq + " + dsel(" + gq + " == " +
                         di + ", 0.0, " + lit(er.c) + ");\n";
                }
                xs.push_back(x);
            }
            // max over predecessors: a balanced tree (no NaN can occur, so
            // max is associative and the result equals the reference's fold)
            std::string r = "r" + std::to_string(i);
            if (xs.empty()) {
                s += "    const double " + r + " = 0.0;\n";
            } else {
                int lvl = 0;
                while (xs.size() > 1) {
                    std::vector<std::string> nx;
                    for (size_t k = 0; k + 1 < xs.size(); k += 2) {
                        const std::string m = "m" + std::to_string(i) + "_" +
                                              std::to_string(lvl) + "_" + std::to_string(k);
                        s += "    const double " + m + " = " + mx + "(" + xs[k] + ", " +
                             xs[k + 1] + ");\n";
                        nx.push_back(m);
                    }
                    if (xs.size() & 1) nx.push_back(xs.back());
                    xs.swap(nx);
                    ++lvl;
                }
                // pymax(0.0, x) == x for x >= +0
                s += "    const double " + r + " = " + xs[0] + ";\n";
            }
            std::vector<std::string> av, du;
            for (int k = 0; k < K; ++k) {
                av.push_back("a" + std::to_string(k));
                du.push_back(lit(p.dur[size_t(i) * K + k]));
            }
            const std::string si = "s" + std::to_string(i);
            const std::string Ai = "A" + std::to_string(i);
            if (o.avail_smem) {
                s += "    double *" + Ai + " = A + " + di + " * " + std::to_string(T) + ";\n";
                s += "    const double " + si + " = " + mx + "(" + r + ", *" + Ai + ");\n";
            } else {
                s += "    const double " + si + " = " + mx + "(" + r + ", " + sel(di, av) + ");\n";
            }
            std::string dsrc = sel(di, du);
            if (o.dur_smem && dsrc != du[0])
                dsrc = "dur[" + std::to_string(i * K) + " + " + di + "]";
            const std::string ei = "e" + std::to_string(i);
            s += "    const double " + ei + " = " + si + " + " + dsrc + ";\n";
            std::snprintf(buf, sizeof buf,
                          "    if (TRACE && valid) starts[cand * %d + %d] = %s;\n", V, i,
                          si.c_str());
            s += buf;
            if (where[i] >= 0)
                s += "    E[" + std::to_string((long long)where[i] * T) + "] = " + ei + ";\n";
            if (o.avail_smem) {
                s += "    *" + Ai + " = " + ei + ";\n";
            } else {
                for (int k = 0; k < K; ++k) {
                    const std::string a = "a" + std::to_string(k);
                    s += "    " + a + " = dsel(" + di + " == " + std::to_string(k) + ", " +
                         ei + ", " + a + ");\n";
                }
            }
        }
        s += "    double ms = 0.0;\n";
        for (int k = 0; k < K; ++k)
            s += o.avail_smem ? "    ms = pymax(ms, A[" + std::to_string(k * T) + "]);\n"
                              : "    ms = pymax(ms, a" + std::to_string(k) + ");\n";
        std::snprintf(buf, sizeof buf,
                      "    const int st = gmax >= %d ? ST_GENE : ST_OK;\n"
                      "    ms_out = st ? knan() : ms;\n    st_out = st;\n  }\n};\n", K);
        s += buf;
        s += "template <bool TRACE>\n__device__ __forceinline__ void jit_main(const EvalParams &a) {\n"
             "  extern __shared__ __align__(16) hs_u8 smem[];\n"
             "  JitBody<TRACE> body;\n"
             "  body.ends = reinterpret_cast<double *>(smem + a.smem_ends);\n"
             "  body.avail = reinterpret_cast<double *>(smem + a.smem_kstate);\n"
             "  body.dur = reinterpret_cast<const double *>(smem + 16);\n"
             "  body.starts = a.starts;\n";
        if (o.dur_smem) {
            std::snprintf(buf, sizeof buf,
                          "  { const uint4 *src = reinterpret_cast<const uint4 *>(a.blob + "
                          "a.lay.dur);\n    uint4 *dst = reinterpret_cast<uint4 *>(smem + 16);\n"
                          "    for (int q = threadIdx.x; q < %lld; q += blockDim.x) dst[q] = "
                          "src[q]; }\n", (long long)(dur_bytes(p) / 16));
            s += buf;
        }
        s += "  eval_tiles(a, smem, body);\n}\n";
        std::snprintf(buf, sizeof buf,
                      "extern \"C\" __global__ void __launch_bounds__(%d, 1) "
                      "hs_jit_eval(const EvalParams a) { jit_main<false>(a); }\n"
                      "extern \"C\" __global__ void __launch_bounds__(%d, 1) "
                      "hs_jit_trace(const EvalParams a) { jit_main<true>(a); }\n", T, T);
        s += buf;
        return next;
    }
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
    const int64_t per_lane = ld_cap + int64_t(slots) * 8 + (o.avail_smem ? 8 * p.K : 0);
    const int64_t head = 16 + (o.dur_smem ? dur_bytes(p) : 0);
    const int64_t budget = int64_t(optin) - head - 1024;
    int T = int(std::min<int64_t>(budget / per_lane, 256) / 32 * 32);
    if (T < 32) {
        if (err) *err = "graph too large for the specialised evaluator";
        return HS_EINVAL;
    }
    std::string src;
    jit_emit(p, T, o, &src);
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
    m->smem_tile = head;
    m->smem_ends = head + ((int64_t(T) * ld_cap + 15) & ~int64_t(15));
    m->smem_kstate = m->smem_ends + int64_t(slots) * T * 8;
    m->smem = size_t(m->smem_kstate + (o.avail_smem ? int64_t(8) * p.K * T : 0));
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
