// Module decomposition of a task graph for the split heuristic -- the native
// counterpart of the reference's module detection (splitting.py:28-219):
//
//  * bridges and articulation points of the undirected shadow
//    (find_bridges_and_articulation_points, splitting.py:36-81). Both sets
//    are properties of the graph, independent of DFS order; an iterative
//    low-link DFS finds them.
//  * the (c+1)-edge-connected components of the shadow
//    (networkx.k_edge_components as called at splitting.py:184): maximal
//    node sets whose every pair has local edge connectivity >= k in the
//    whole graph. Pairwise connectivities come from Gusfield's equivalent
//    flow tree (n-1 unit-capacity max flows, each an exact min cut); two
//    tasks share a component iff every tree edge on their path carries
//    >= k, so the components are the connected pieces of the tree after
//    dropping the lighter edges. For k = 2 the components are those of the
//    shadow without its bridges (the partition networkx uses for k = 2).
//  * the reference's post-processing (splitting.py:186-208): cycles of the
//    component digraph merged (strongly connected components), then the
//    modules ordered by Kahn's algorithm with the smallest "min task id"
//    first (networkx.lexicographical_topological_sort keyed by
//    min(comps[k]); ids compare bytewise = Python code-point order).
//
// Everything here is a one-time O(n * k * E) host computation per graph.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <functional>
#include <queue>
#include <string>
#include <vector>

#include "../../include/hetsched_b200.h"

namespace {

struct Shadow {
    int n = 0;
    std::vector<int> off, adj;  // CSR of the simple undirected shadow
};

Shadow make_shadow(int n, int m, const int32_t *src, const int32_t *dst) {
    std::vector<std::pair<int, int>> e;
    e.reserve(size_t(m) * 2);
    for (int i = 0; i < m; ++i) {
        const int a = src[i], b = dst[i];
        if (a == b) continue;
        e.emplace_back(a, b);
        e.emplace_back(b, a);
    }
    std::sort(e.begin(), e.end());
    e.erase(std::unique(e.begin(), e.end()), e.end());
    Shadow s;
    s.n = n;
    s.off.assign(size_t(n) + 1, 0);
    for (auto &p : e) s.off[p.first + 1]++;
    for (int i = 0; i < n; ++i) s.off[i + 1] += s.off[i];
    s.adj.resize(e.size());
    std::vector<int> fill(s.off.begin(), s.off.end() - 1);
    for (auto &p : e) s.adj[fill[p.first]++] = p.second;
    return s;
}

// unit-capacity max flow s -> t on the shadow (each undirected edge is a
// pair of opposite arcs of capacity 1); returns the flow value and marks
// the source side of a minimum cut in `side`.
struct MaxFlow {
    const Shadow &g;
    std::vector<int> rev;   // index of the opposite arc
    std::vector<int> flow;  // flow on arc (-1, 0, 1)
    std::vector<int> prev_arc, seen;
    int stamp = 0;
    explicit MaxFlow(const Shadow &sh) : g(sh) {
        rev.resize(g.adj.size());
        for (int u = 0; u < g.n; ++u)
            for (int a = g.off[u]; a < g.off[u + 1]; ++a) {
                const int v = g.adj[a];
                const int *lo = g.adj.data() + g.off[v], *hi = g.adj.data() + g.off[v + 1];
                rev[a] = int(std::lower_bound(lo, hi, u) - g.adj.data());
            }
        flow.assign(g.adj.size(), 0);
        prev_arc.assign(size_t(g.n), -1);
        seen.assign(size_t(g.n), 0);
    }
    // BFS in the residual graph from s; true if t was reached
    bool bfs(int s, int t) {
        ++stamp;
        std::queue<int> q;
        q.push(s);
        seen[s] = stamp;
        while (!q.empty()) {
            const int u = q.front();
            q.pop();
            for (int a = g.off[u]; a < g.off[u + 1]; ++a) {
                const int v = g.adj[a];
                if (seen[v] == stamp || flow[a] >= 1) continue;
                seen[v] = stamp;
                prev_arc[v] = a;
                if (v == t) return true;
                q.push(v);
            }
        }
        return false;
    }
    int run(int s, int t, std::vector<char> &side) {
        std::fill(flow.begin(), flow.end(), 0);
        int f = 0;
        while (bfs(s, t)) {
            for (int v = t; v != s;) {
                const int a = prev_arc[v];
                flow[a] += 1;
                flow[rev[a]] -= 1;
                v = g.adj[rev[a]];
            }
            ++f;
        }
        // the last (failed) BFS marked the residual-reachable set
        side.assign(size_t(g.n), 0);
        for (int v = 0; v < g.n; ++v) side[v] = seen[v] == stamp;
        return f;
    }
};

struct Ids {
    const char *bytes;
    const int64_t *off;
    bool less(int a, int b) const {
        const int64_t la = off[a + 1] - off[a], lb = off[b + 1] - off[b];
        const int c = std::memcmp(bytes + off[a], bytes + off[b], size_t(std::min(la, lb)));
        return c < 0 || (c == 0 && la < lb);
    }
};

// low-link DFS (iterative): bridge flag per shadow arc (both directions of
// a bridge edge get it) and articulation flag per vertex; returns the
// number of DFS roots (connected components)
int bridge_dfs(const Shadow &g, std::vector<char> &bridge_arc, std::vector<char> &art) {
    const int n = g.n;
    std::vector<int> disc(size_t(n), -1), low(size_t(n), 0), parent(size_t(n), -1);
    art.assign(size_t(n), 0);
    bridge_arc.assign(g.adj.size(), 0);
    auto arc = [&](int a, int b) {
        const int *lo = g.adj.data() + g.off[a], *hi = g.adj.data() + g.off[a + 1];
        return size_t(std::lower_bound(lo, hi, b) - g.adj.data());
    };
    int counter = 0, roots = 0;
    std::vector<std::pair<int, int>> stack;  // (vertex, next arc)
    for (int root = 0; root < n; ++root) {
        if (disc[root] >= 0) continue;
        ++roots;
        disc[root] = low[root] = counter++;
        int root_children = 0;
        stack.assign(1, {root, g.off[root]});
        while (!stack.empty()) {
            const int v = stack.back().first;
            if (stack.back().second < g.off[v + 1]) {
                const int w = g.adj[stack.back().second++];
                if (disc[w] < 0) {
                    parent[w] = v;
                    disc[w] = low[w] = counter++;
                    if (v == root) ++root_children;
                    stack.push_back({w, g.off[w]});
                } else if (w != parent[v]) {
                    low[v] = std::min(low[v], disc[w]);
                }
                continue;
            }
            stack.pop_back();
            if (stack.empty()) break;
            const int p = stack.back().first;
            low[p] = std::min(low[p], low[v]);
            if (low[v] > disc[p]) bridge_arc[arc(p, v)] = bridge_arc[arc(v, p)] = 1;
            if (p != root && low[v] >= disc[p]) art[p] = 1;
        }
        if (root_children > 1) art[root] = 1;
    }
    return roots;
}

}  // namespace

extern "C" int hs_bridges_articulation(int32_t n_tasks, int32_t n_edges,
                                       const int32_t *edge_src, const int32_t *edge_dst,
                                       uint8_t *is_bridge, uint8_t *is_articulation,
                                       int32_t *connected) {
    if (n_tasks < 0 || n_edges < 0 || (n_edges > 0 && (!edge_src || !edge_dst)))
        return HS_EINVAL;
    for (int i = 0; i < n_edges; ++i)
        if (edge_src[i] < 0 || edge_src[i] >= n_tasks || edge_dst[i] < 0 ||
            edge_dst[i] >= n_tasks)
            return HS_EINVAL;
    const Shadow g = make_shadow(n_tasks, n_edges, edge_src, edge_dst);
    std::vector<char> bridge_arc, art;
    const int roots = bridge_dfs(g, bridge_arc, art);
    if (is_bridge)
        for (int i = 0; i < n_edges; ++i) {
            const int a = edge_src[i], b = edge_dst[i];
            bool br = false;
            if (a != b) {
                const int *lo = g.adj.data() + g.off[a], *hi = g.adj.data() + g.off[a + 1];
                br = bridge_arc[size_t(std::lower_bound(lo, hi, b) - g.adj.data())];
            }
            is_bridge[i] = br;
        }
    if (is_articulation)
        for (int v = 0; v < g.n; ++v) is_articulation[v] = uint8_t(art[v]);
    if (connected) *connected = roots <= 1;
    return HS_OK;
}

extern "C" int hs_k_edge_components(int32_t n_tasks, const char *task_ids,
                                    const int64_t *task_id_off, int32_t n_edges,
                                    const int32_t *edge_src, const int32_t *edge_dst,
                                    int32_t k, int32_t *module_of, int32_t *n_modules) {
    if (n_tasks < 0 || n_edges < 0 || k < 1 || !module_of || !n_modules ||
        (n_tasks > 0 && (!task_ids || !task_id_off)) ||
        (n_edges > 0 && (!edge_src || !edge_dst)))
        return HS_EINVAL;
    for (int i = 0; i < n_edges; ++i)
        if (edge_src[i] < 0 || edge_src[i] >= n_tasks || edge_dst[i] < 0 ||
            edge_dst[i] >= n_tasks)
            return HS_EINVAL;
    const int n = n_tasks;
    *n_modules = 0;
    if (n == 0) return HS_OK;
    const Shadow g = make_shadow(n, n_edges, edge_src, edge_dst);
    // Gusfield: equivalent flow tree (p[s], fl[s]) for s = 1..n-1
    std::vector<int> p(size_t(n), 0), fl(size_t(n), 0);
    std::vector<char> bridge_arc;
    if (k == 2) {  // 2-edge-connected = connected without the bridges
        std::vector<char> art;
        bridge_dfs(g, bridge_arc, art);
    } else if (k > 2) {
        MaxFlow mf(g);
        std::vector<char> side;
        for (int s = 1; s < n; ++s) {
            const int t = p[s];
            fl[s] = mf.run(s, t, side);
            for (int i = s + 1; i < n; ++i)
                if (side[i] && p[i] == t) p[i] = s;
        }
    }
    // components: union over tree edges with connectivity >= k (k == 1:
    // plain connected components, every pair with a path)
    std::vector<int> uf(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) uf[i] = i;
    std::function<int(int)> find = [&](int x) {
        while (uf[x] != x) x = uf[x] = uf[uf[x]];
        return x;
    };
    auto unite = [&](int a, int b) {
        a = find(a);
        b = find(b);
        if (a != b) uf[std::max(a, b)] = std::min(a, b);
    };
    if (k == 2) {
        for (int u = 0; u < n; ++u)
            for (int a = g.off[u]; a < g.off[u + 1]; ++a)
                if (!bridge_arc[size_t(a)]) unite(u, g.adj[a]);
    } else if (k > 2) {
        for (int s = 1; s < n; ++s)
            if (fl[s] >= k) unite(s, p[s]);
    } else {
        for (int u = 0; u < n; ++u)
            for (int a = g.off[u]; a < g.off[u + 1]; ++a) unite(u, g.adj[a]);
    }
    std::vector<int> comp(size_t(n), -1), rep_of;
    for (int i = 0; i < n; ++i) {
        const int r = find(i);
        if (comp[r] < 0) {
            comp[r] = int(rep_of.size());
            rep_of.push_back(r);
        }
        comp[i] = comp[r];
    }
    int C = int(rep_of.size());
    // merge cycles of the component digraph (Tarjan SCC, iterative)
    auto build_red = [&](std::vector<std::vector<int>> &out) {
        out.assign(size_t(C), {});
        for (int i = 0; i < n_edges; ++i) {
            const int a = comp[edge_src[i]], b = comp[edge_dst[i]];
            if (a != b) out[a].push_back(b);
        }
        for (auto &v : out) {
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end()), v.end());
        }
    };
    std::vector<std::vector<int>> red;
    build_red(red);
    {
        std::vector<int> idx(size_t(C), -1), lowl(size_t(C), 0), scc(size_t(C), -1);
        std::vector<char> on(size_t(C), 0);
        std::vector<int> st;
        int counter = 0, nscc = 0;
        std::vector<std::pair<int, size_t>> cs;
        for (int r = 0; r < C; ++r) {
            if (idx[r] >= 0) continue;
            cs.assign(1, {r, 0});
            idx[r] = lowl[r] = counter++;
            st.push_back(r);
            on[r] = 1;
            while (!cs.empty()) {
                const int v = cs.back().first;
                size_t &it = cs.back().second;
                if (it < red[v].size()) {
                    const int w = red[v][it++];
                    if (idx[w] < 0) {
                        idx[w] = lowl[w] = counter++;
                        st.push_back(w);
                        on[w] = 1;
                        cs.push_back({w, 0});
                    } else if (on[w]) {
                        lowl[v] = std::min(lowl[v], idx[w]);
                    }
                    continue;
                }
                if (lowl[v] == idx[v]) {
                    for (;;) {
                        const int w = st.back();
                        st.pop_back();
                        on[w] = 0;
                        scc[w] = nscc;
                        if (w == v) break;
                    }
                    ++nscc;
                }
                cs.pop_back();
                if (!cs.empty()) {
                    const int u = cs.back().first;
                    lowl[u] = std::min(lowl[u], lowl[v]);
                }
            }
        }
        if (nscc < C) {
            for (int i = 0; i < n; ++i) comp[i] = scc[comp[i]];
            C = nscc;
            build_red(red);
        }
    }
    // smallest task id per component, then lexicographic Kahn
    const Ids ids{task_ids, task_id_off};
    std::vector<int> key(size_t(C), -1);
    for (int i = 0; i < n; ++i) {
        int &kk = key[comp[i]];
        if (kk < 0 || ids.less(i, kk)) kk = i;
    }
    std::vector<int> indeg(size_t(C), 0);
    for (int c = 0; c < C; ++c)
        for (int d : red[c]) indeg[d]++;
    auto cmp = [&](int a, int b) { return ids.less(key[b], key[a]); };  // min-heap
    std::priority_queue<int, std::vector<int>, decltype(cmp)> heap(cmp);
    for (int c = 0; c < C; ++c)
        if (!indeg[c]) heap.push(c);
    std::vector<int> rank(size_t(C), -1);
    int r = 0;
    while (!heap.empty()) {
        const int c = heap.top();
        heap.pop();
        rank[c] = r++;
        for (int d : red[c])
            if (--indeg[d] == 0) heap.push(d);
    }
    if (r != C) return HS_ECYCLE;  // cannot happen after the SCC merge
    for (int i = 0; i < n; ++i) module_of[i] = rank[comp[i]];
    *n_modules = C;
    return HS_OK;
}
