// Plan compiler: (graph, hardware, latency table, L) -> flat tables.
//
// Restates, once per instance, everything the reference recomputes inside
// every decode() call (heuristics.py:127-143): the genome order
// (bfs_topological_order = heap-Kahn on string ids, core.py:82-101), the
// device numbering sorted(hw.devices) (heuristics.py:132), comm_time
// (core.py:148-155: 0 on the same device, missing link, om / beta as an IEEE
// division), LatencyTable.get at batch L (core.py:166-170), _mem_extra
// ((im + om) * L then + wm, heuristics.py:60-65) and the capacity test
// memory + 1e-9 (heuristics.py:99). Compiled with -ffp-contract=off: no
// multiply-add may be fused, every value is the reference's binary64.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <queue>
#include <set>
#include <unordered_set>

#include "plan.hpp"

namespace hs {
namespace {

bool bytes_less(const std::string &a, const std::string &b) {
    // std::string::compare is an unsigned bytewise compare: UTF-8 byte
    // order equals Python's code-point order of the decoded strings.
    return a.compare(b) < 0;
}

int fail(std::string *err, int code, const std::string &msg) {
    if (err) *err = msg;
    return code;
}

int64_t align16(int64_t x) { return (x + 15) & ~int64_t(15); }

}  // namespace

int build_plan(const hs_instance_desc &d, Plan &p, std::string *err,
               const BatchedSpec *bspec) {
    if (d.n_tasks < 0 || d.n_edges < 0 || d.n_devices < 1)
        return fail(err, HS_EINVAL, "need n_tasks >= 0, n_edges >= 0, "
                                    "n_devices >= 1");
    if (d.n_devices > 255)
        return fail(err, HS_EINVAL, "at most 255 devices (uint8 genes)");
    const int NT = d.n_tasks, K = d.n_devices, E = d.n_edges;
    p.NT = p.V = NT;
    p.K = K;
    p.E = E;
    p.L = d.L;
    p.words = (NT + 63) / 64;

    // ---- ids
    p.task_ids.resize(NT);
    for (int t = 0; t < NT; ++t)
        p.task_ids[t].assign(d.task_ids + d.task_id_off[t],
                             size_t(d.task_id_off[t + 1] - d.task_id_off[t]));
    std::vector<std::string> dev_ids(K);
    for (int k = 0; k < K; ++k)
        dev_ids[k].assign(d.dev_ids + d.dev_id_off[k],
                          size_t(d.dev_id_off[k + 1] - d.dev_id_off[k]));
    {
        std::set<std::string> seen(p.task_ids.begin(), p.task_ids.end());
        if ((int)seen.size() != NT)
            return fail(err, HS_EINVAL, "duplicate task id");
        std::set<std::string> sd(dev_ids.begin(), dev_ids.end());
        if ((int)sd.size() != K)
            return fail(err, HS_EINVAL, "duplicate device id");
    }
    for (int t = 0; t < NT; ++t)
        if (d.wm[t] < 0 || d.im[t] < 0 || d.om[t] < 0)  // core.py:33
            return fail(err, HS_EINVAL, "task " + p.task_ids[t] +
                                            ": wm/im/om must be >= 0");

    // ---- edges: succ / pred in insertion order (core.py:47-59)
    std::vector<std::vector<int>> succ(NT), pred(NT);
    {
        std::unordered_set<int64_t> seen;
        for (int e = 0; e < E; ++e) {
            const int a = d.edge_src[e], b = d.edge_dst[e];
            if (a < 0 || a >= NT || b < 0 || b >= NT)
                return fail(err, HS_EINVAL, "dangling edge endpoint");
            if (!seen.insert(int64_t(a) * NT + b).second)
                return fail(err, HS_EINVAL, "duplicate edge");
            succ[a].push_back(b);
            pred[b].push_back(a);
        }
    }

    // ---- bfs_topological_order: Kahn, smallest id first (core.py:82-96)
    {
        std::vector<int> indeg(NT);
        for (int t = 0; t < NT; ++t) indeg[t] = (int)pred[t].size();
        auto gt = [&](int a, int b) {
            return bytes_less(p.task_ids[b], p.task_ids[a]);
        };
        std::priority_queue<int, std::vector<int>, decltype(gt)> heap(gt);
        for (int t = 0; t < NT; ++t)
            if (indeg[t] == 0) heap.push(t);
        p.bfs.clear();
        while (!heap.empty()) {
            const int t = heap.top();
            heap.pop();
            p.bfs.push_back(t);
            for (int s : succ[t])
                if (--indeg[s] == 0) heap.push(s);
        }
        if ((int)p.bfs.size() != NT)
            return fail(err, HS_ECYCLE, "cycle detected");
    }
    if (d.order) {
        p.order.assign(d.order, d.order + NT);
        std::vector<int> seen(NT, 0);
        for (int t : p.order) {
            if (t < 0 || t >= NT || seen[t]++)
                return fail(err, HS_EINVAL, "genome order is not a "
                                            "permutation of the tasks");
        }
    } else {
        p.order = p.bfs;
    }
    std::vector<int> pos(NT);
    for (int i = 0; i < NT; ++i) pos[p.order[i]] = i;
    for (int i = 0; i < NT; ++i)
        for (int q : pred[p.order[i]])
            if (pos[q] >= i)
                return fail(err, HS_EINVAL, "genome order is not a "
                                            "topological order");

    // ---- devices: gene k -> k-th smallest id (heuristics.py:132)
    p.dev_order.resize(K);
    for (int k = 0; k < K; ++k) p.dev_order[k] = k;
    std::sort(p.dev_order.begin(), p.dev_order.end(), [&](int a, int b) {
        return bytes_less(dev_ids[a], dev_ids[b]);
    });

    // ---- latency at batch L, capacity, batch support
    const int ncols = d.batch_off[K];
    auto lat = [&](int t, int col) { return d.latency[int64_t(t) * ncols + col]; };
    auto lat_ok = [&](int t, int col) {
        return d.latency_ok[int64_t(t) * ncols + col] != 0;
    };
    p.okL.assign(K, 0);
    p.cap.assign(K, 0.0);
    std::vector<int> colL(K, -1);
    for (int k = 0; k < K; ++k) {
        const int dv = p.dev_order[k];
        for (int c = d.batch_off[dv]; c < d.batch_off[dv + 1]; ++c)
            if (d.batch_sizes[c] == d.L) colL[k] = c;
        p.okL[k] = colL[k] >= 0;
        p.cap[k] = d.memory[dv] + 1e-9;
        if (!p.okL[k]) p.all_batch_ok = false;
    }
    const int V = NT;
    p.dur.assign(size_t(V) * K, 0.0);
    p.dur_ok.assign(size_t(V) * K, 0);
    for (int i = 0; i < V; ++i) {
        const int t = p.order[i];
        for (int k = 0; k < K; ++k) {
            if (colL[k] < 0) continue;
            if (lat_ok(t, colL[k])) {
                const double v = lat(t, colL[k]);
                if (v < 0)
                    return fail(err, HS_EINVAL, "negative latency");
                p.dur[size_t(i) * K + k] = v;
                p.dur_ok[size_t(i) * K + k] = 1;
                if (std::isnan(v)) p.nan_possible = true;
            } else {
                p.latency_complete = false;
            }
        }
    }
    p.extra.resize(V);
    for (int i = 0; i < V; ++i) {
        const int t = p.order[i];
        double x = (d.im[t] + d.om[t]) * double(d.L);
        x += d.wm[t];
        p.extra[i] = x;
    }
    // capacity can never bind if the whole graph fits on every device: the
    // rounded running sum is monotone over non-negative terms
    {
        double total = 0.0;
        for (int i = 0; i < V; ++i) total += p.extra[i];
        bool fits = true;
        for (int k = 0; k < K; ++k)
            if (!(total <= p.cap[k])) fits = false;
        p.mem_check = !fits;
    }

    // ---- comm classes (core.py:148-155)
    std::vector<uint64_t> betas;  // distinct bit patterns, first-seen order
    p.full_mesh = true;
    std::vector<int> bcls(size_t(K) * K, 0);
    for (int u = 0; u < K; ++u)
        for (int v = 0; v < K; ++v) {
            if (u == v) continue;
            const double b = d.bandwidth[size_t(p.dev_order[u]) * K + p.dev_order[v]];
            if (b <= 0) {
                bcls[size_t(u) * K + v] = -1;
                p.full_mesh = false;
                continue;
            }
            uint64_t bits;
            std::memcpy(&bits, &b, 8);
            auto it = std::find(betas.begin(), betas.end(), bits);
            if (it == betas.end()) {
                betas.push_back(bits);
                it = betas.end() - 1;
            }
            bcls[size_t(u) * K + v] = 1 + int(it - betas.begin());
        }
    p.n_classes = (int)betas.size();
    // batched plans always carry the class tables (the batched evaluator
    // looks communication up by (source device, destination device))
    p.uniform_comm = p.full_mesh && betas.size() <= 1 && !bspec;
    p.n_cls = 1 + (int)betas.size();
    if (!p.uniform_comm && p.n_cls > 65535)
        return fail(err, HS_EINVAL, "too many distinct bandwidths");
    p.bclass.assign(size_t(K) * K * 2, 0);  // uint16 little-endian
    for (size_t q = 0; q < bcls.size(); ++q) {
        const int c = bcls[q] < 0 ? 0xFFFF : bcls[q];
        p.bclass[2 * q] = uint8_t(c & 0xFF);
        p.bclass[2 * q + 1] = uint8_t(c >> 8);
    }
    std::vector<double> beta_val(betas.size());
    for (size_t c = 0; c < betas.size(); ++c) std::memcpy(&beta_val[c], &betas[c], 8);
    if (!p.uniform_comm) {
        p.ctab.assign(size_t(V) * p.n_cls, 0.0);
        for (int i = 0; i < V; ++i)
            for (int c = 1; c < p.n_cls; ++c) {
                const double x = d.om[p.order[i]] / beta_val[c - 1];
                p.ctab[size_t(i) * p.n_cls + c] = x;
                if (std::isnan(x)) p.nan_possible = true;
            }
    }
    for (int i = 0; i < V; ++i)
        if (std::isnan(p.extra[i])) p.nan_possible = true;

    // ---- live end-time slots (interval colouring in genome order)
    std::vector<int> last_use(V, -1), slot(V, -1);
    for (int i = 0; i < V; ++i)
        for (int s : succ[p.order[i]]) last_use[i] = std::max(last_use[i], pos[s]);
    {
        std::priority_queue<int, std::vector<int>, std::greater<int>> freel;
        int next = 0;
        std::vector<std::vector<int>> dies(V);
        for (int i = 0; i < V; ++i)
            if (last_use[i] >= 0) dies[last_use[i]].push_back(i);
        for (int i = 0; i < V; ++i) {
            // predecessors whose last reader is i are read before i's end
            // is written, so their slots can be recycled for i -- except
            // in batched plans, where part k's end is written before part
            // k+1 reads the predecessors
            if (!bspec)
                for (int q : dies[i]) freel.push(slot[q]);
            if (last_use[i] >= 0) {
                if (!freel.empty()) {
                    slot[i] = freel.top();
                    freel.pop();
                } else {
                    slot[i] = next++;
                }
            }
            if (bspec)
                for (int q : dies[i]) freel.push(slot[q]);
        }
        p.live_slots = next;
    }

    // ---- node / edge records
    p.nodes.resize(V);
    p.edges.clear();
    p.edges.reserve(E);
    for (int i = 0; i < V; ++i) {
        NodeRec nr{};
        nr.e_begin = (int)p.edges.size();
        for (int q : pred[p.order[i]]) {
            EdgeRec er{};
            er.slot = slot[pos[q]];
            er.gpos = pos[q];
            if (p.uniform_comm) {
                er.c = betas.empty() ? 0.0 : d.om[q] / beta_val[0];
                if (std::isnan(er.c)) p.nan_possible = true;
            } else {
                er.crow = int64_t(pos[q]) * p.n_cls;
            }
            p.edges.push_back(er);
        }
        nr.e_end = (int)p.edges.size();
        nr.out_slot = slot[i];
        p.nodes[i] = nr;
    }

    // ---- critical path tables (bounds.py:57-72) over g._topo
    p.cp_fast.assign(V, 0.0);
    p.cp_fast_ok.assign(V, 1);
    p.cp_pred_off.assign(V + 1, 0);
    p.cp_pred_pos.clear();
    std::vector<int> bpos(NT);
    for (int i = 0; i < NT; ++i) bpos[p.bfs[i]] = i;
    for (int i = 0; i < V; ++i) {
        const int t = p.bfs[i];
        bool have = false;
        double best = 0.0;
        // min over hw.devices.values() (insertion order) x batch_sizes
        for (int dv = 0; dv < K && p.cp_fast_ok[i]; ++dv)
            for (int c = d.batch_off[dv]; c < d.batch_off[dv + 1]; ++c) {
                if (!lat_ok(t, c)) {
                    p.cp_fast_ok[i] = 0;
                    break;
                }
                const double v = lat(t, c);
                if (!have || v < best) {
                    best = v;
                    have = true;
                }
            }
        p.cp_fast[i] = best;
        for (int q : pred[t]) p.cp_pred_pos.push_back(bpos[q]);
        p.cp_pred_off[i + 1] = (int)p.cp_pred_pos.size();
    }

    // ---- reachability CSR (task insertion index)
    p.rc_succ_off.assign(NT + 1, 0);
    p.rc_pred_off.assign(NT + 1, 0);
    p.rc_succ.clear();
    p.rc_pred.clear();
    for (int t = 0; t < NT; ++t) {
        for (int s : succ[t]) p.rc_succ.push_back(s);
        for (int q : pred[t]) p.rc_pred.push_back(q);
        p.rc_succ_off[t + 1] = (int)p.rc_succ.size();
        p.rc_pred_off[t + 1] = (int)p.rc_pred.size();
    }

    // ---- batched-variant options (heuristics.py:337-392)
    if (bspec) {
        p.batched = true;
        std::vector<int> sizes;
        if (bspec->splits && bspec->n_splits > 0) {
            sizes.assign(bspec->splits, bspec->splits + bspec->n_splits);
        } else {
            for (int k = 1; k <= 4; ++k)
                if ((d.L * k) % 4 == 0 && d.L * k / 4 >= 1) sizes.push_back(d.L * k / 4);
        }
        std::sort(sizes.begin(), sizes.end());
        sizes.erase(std::unique(sizes.begin(), sizes.end()), sizes.end());
        std::vector<std::vector<int>> decomps;
        std::vector<int> acc;
        std::function<void(int, int)> rec = [&](int remaining, int start) {
            if (remaining == 0) {
                decomps.push_back(acc);
                return;
            }
            if ((int)acc.size() >= K) return;
            for (int k = start; k < (int)sizes.size(); ++k)
                if (sizes[k] <= remaining) {
                    acc.push_back(sizes[k]);
                    rec(remaining - sizes[k], k);
                    acc.pop_back();
                }
        };
        if (d.L >= 1) rec(d.L, 0);
        bool hasL = false, Lallowed = false;
        for (auto &dc : decomps) hasL |= dc.size() == 1 && dc[0] == d.L;
        for (int s2 : sizes) Lallowed |= s2 == d.L;
        if (!hasL && Lallowed) decomps.push_back({d.L});
        // device support of a size, by sorted device index
        auto supports = [&](int k, int size) {
            const int dv = p.dev_order[k];
            for (int c = d.batch_off[dv]; c < d.batch_off[dv + 1]; ++c)
                if (d.batch_sizes[c] == size) return true;
            return false;
        };
        std::vector<std::vector<int>> opt_sizes, opt_devs;
        for (auto &dc : decomps) {
            const int r = (int)dc.size();
            std::vector<int> perm;
            std::vector<char> used(K, 0);
            std::function<void()> gen = [&]() {  // itertools.permutations order
                if ((int)perm.size() == r) {
                    for (int k = 0; k < r; ++k)
                        if (!supports(perm[k], dc[k])) return;
                    opt_sizes.push_back(dc);
                    opt_devs.push_back(perm);
                    return;
                }
                for (int k = 0; k < K; ++k) {
                    if (used[k]) continue;
                    used[k] = 1;
                    perm.push_back(k);
                    gen();
                    perm.pop_back();
                    used[k] = 0;
                    if (opt_sizes.size() > 255) return;
                }
            };
            gen();
            if (opt_sizes.size() > 255)
                return fail(err, HS_EINVAL, "more than 255 batched options "
                                            "(uint8 extended genes)");
        }
        p.n_opt = (int)opt_sizes.size();
        p.P = 1;
        for (auto &o : opt_sizes) p.P = std::max(p.P, (int)o.size());
        if (p.P > 8) return fail(err, HS_EINVAL, "more than 8 sub-batches per task");
        const int P = p.P, NO = p.n_opt;
        p.opt_np.assign(NO, 0);
        p.opt_tab.assign(size_t(NO) * P * 4, -1);
        for (int o = 0; o < NO; ++o) {
            p.opt_np[o] = (int)opt_sizes[o].size();
            int lo = 1;
            for (int k = 0; k < p.opt_np[o]; ++k) {
                int32_t *q = &p.opt_tab[(size_t(o) * P + k) * 4];
                q[0] = opt_devs[o][k];
                q[1] = lo;
                q[2] = lo + opt_sizes[o][k] - 1;
                q[3] = opt_sizes[o][k];
                lo += opt_sizes[o][k];
            }
        }
        p.bdur.assign(size_t(V) * NO * P, 0.0);
        p.bdur_ok.assign(size_t(V) * NO * P, 0);
        for (int i = 0; i < V; ++i) {
            const int t = p.order[i];
            for (int o = 0; o < NO; ++o)
                for (int k = 0; k < p.opt_np[o]; ++k) {
                    const int32_t *q = &p.opt_tab[(size_t(o) * P + k) * 4];
                    const int dv = p.dev_order[q[0]];
                    for (int c = d.batch_off[dv]; c < d.batch_off[dv + 1]; ++c)
                        if (d.batch_sizes[c] == q[3] && lat_ok(t, c)) {
                            const size_t at = (size_t(i) * NO + o) * P + k;
                            p.bdur[at] = lat(t, c);
                            p.bdur_ok[at] = 1;
                            if (std::isnan(p.bdur[at])) p.nan_possible = true;
                        }
                }
        }
        // class tables are needed even for one bandwidth
        if (p.ctab.empty()) {
            p.ctab.assign(size_t(V) * p.n_cls, 0.0);
            for (int i = 0; i < V; ++i)
                for (int c = 1; c < p.n_cls; ++c)
                    p.ctab[size_t(i) * p.n_cls + c] = d.om[p.order[i]] / beta_val[c - 1];
        }
        for (double x : p.ctab)
            if (std::isnan(x)) p.nan_possible = true;
    }

    // ---- blob layout (host image; slots are re-scaled per device config)
    DevLayout &L = p.lay;
    int64_t off = 0;
    auto put = [&](int64_t bytes) {
        const int64_t o = off;
        off = align16(off + bytes);
        return o;
    };
    L.node = put(int64_t(V) * sizeof(NodeRec));
    L.edge = put(int64_t(p.edges.size()) * sizeof(EdgeRec));
    L.dur = put(int64_t(V) * K * 8);
    L.dur_ok = put(int64_t(V) * K);
    L.extra = put(int64_t(V) * 8);
    L.ctab = put(int64_t(p.ctab.size()) * 8);
    L.bclass = put(int64_t(p.bclass.size()));
    L.cap = put(int64_t(K) * 8);
    L.okL = put(int64_t(K));
    L.bopt = put(int64_t(p.opt_tab.size()) * 4);
    L.bnp = put(int64_t(p.opt_np.size()) * 4);
    L.bdur = put(int64_t(p.bdur.size()) * 8);
    L.bdur_ok = put(int64_t(p.bdur_ok.size()));
    L.eval_bytes = off;
    L.cp_fast = put(int64_t(V) * 8);
    L.cp_fast_ok = put(int64_t(V));
    L.cp_task = put(int64_t(V) * 4);
    L.cp_pred_off = put(int64_t(V + 1) * 4);
    L.cp_pred_pos = put(int64_t(p.cp_pred_pos.size()) * 4);
    L.rc_succ_off = put(int64_t(NT + 1) * 4);
    L.rc_succ = put(int64_t(p.rc_succ.size()) * 4);
    L.rc_pred_off = put(int64_t(NT + 1) * 4);
    L.rc_pred = put(int64_t(p.rc_pred.size()) * 4);
    L.rc_order = put(int64_t(NT) * 4);
    L.total = off;
    p.blob.assign(size_t(std::max<int64_t>(off, 16)), 0);
    auto cpy = [&](int64_t o, const void *src, size_t bytes) {
        if (bytes) std::memcpy(p.blob.data() + o, src, bytes);
    };
    cpy(L.node, p.nodes.data(), p.nodes.size() * sizeof(NodeRec));
    cpy(L.edge, p.edges.data(), p.edges.size() * sizeof(EdgeRec));
    cpy(L.dur, p.dur.data(), p.dur.size() * 8);
    cpy(L.dur_ok, p.dur_ok.data(), p.dur_ok.size());
    cpy(L.extra, p.extra.data(), p.extra.size() * 8);
    cpy(L.ctab, p.ctab.data(), p.ctab.size() * 8);
    cpy(L.bclass, p.bclass.data(), p.bclass.size());
    cpy(L.cap, p.cap.data(), p.cap.size() * 8);
    cpy(L.okL, p.okL.data(), p.okL.size());
    cpy(L.bopt, p.opt_tab.data(), p.opt_tab.size() * 4);
    cpy(L.bnp, p.opt_np.data(), p.opt_np.size() * 4);
    cpy(L.bdur, p.bdur.data(), p.bdur.size() * 8);
    cpy(L.bdur_ok, p.bdur_ok.data(), p.bdur_ok.size());
    cpy(L.cp_fast, p.cp_fast.data(), p.cp_fast.size() * 8);
    cpy(L.cp_fast_ok, p.cp_fast_ok.data(), p.cp_fast_ok.size());
    cpy(L.cp_task, p.bfs.data(), p.bfs.size() * 4);
    cpy(L.cp_pred_off, p.cp_pred_off.data(), p.cp_pred_off.size() * 4);
    cpy(L.cp_pred_pos, p.cp_pred_pos.data(), p.cp_pred_pos.size() * 4);
    cpy(L.rc_succ_off, p.rc_succ_off.data(), p.rc_succ_off.size() * 4);
    cpy(L.rc_succ, p.rc_succ.data(), p.rc_succ.size() * 4);
    cpy(L.rc_pred_off, p.rc_pred_off.data(), p.rc_pred_off.size() * 4);
    cpy(L.rc_pred, p.rc_pred.data(), p.rc_pred.size() * 4);
    cpy(L.rc_order, p.bfs.data(), p.bfs.size() * 4);
    return HS_OK;
}

}  // namespace hs
