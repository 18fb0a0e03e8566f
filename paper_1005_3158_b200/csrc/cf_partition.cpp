// cf_partition.cpp — graph partitioning for genuinely unstructured multi-GPU meshes (SURVEY §8(f)
// rank 4): the reference's decoupled-mesh partitioner and its quality metrics, on the host (a
// setup step, off the per-step path; the default decomposition is RCB, cf_mesh.cpp).
//
//   dual graph          build_dual_graph mesh.hpp:119-126 (tets sharing a face; a face shared by
//                       more tets links consecutive holders only, as the reference's sorted scan)
//   virtual elements    augment_virtual_elements partition.hpp:43-91: one zero-weight vertex per
//                       interface pair (cast side only), linked to the facet owner and the sister,
//                       so decoupled regions are partitioned together (paper 4.1.1)
//   greedy growing      partition_graph partition.hpp:134-232: parts grown by BFS to a weight
//                       quota from the farthest unassigned vertex, zero-weight leftovers follow
//                       their lowest-id assigned neighbour, then 8 boundary-refinement passes
//   quality             partition_metrics :250-272, count_split_interface_pairs :276-283
// The partitions are the reference's vertex for vertex (tests/test_host.py); every choice that
// decides ties (BFS queue order over ascending neighbour lists, lowest index among equally far
// vertices, first part among equally adjacent ones) is the reference's.
#include <algorithm>
#include <cstring>
#include <deque>
#include <limits>
#include <numeric>
#include <string>
#include <utility>
#include <vector>

#include "cf_internal.hpp"

namespace cfb {
namespace {

// sorted, deduplicated CSR from an undirected edge list (AdjacencyGraph::from_edge_list graph.hpp:36-55)
Graph csr_from_edges(int32_t n, std::vector<std::pair<int32_t, int32_t>>& und) {
    std::vector<std::pair<int32_t, int32_t>> dir;
    dir.reserve(2 * und.size());
    for (const auto& [a, b] : und)
        if (a != b) {
            dir.emplace_back(a, b);
            dir.emplace_back(b, a);
        }
    std::vector<std::pair<int32_t, int32_t>>().swap(und);
    std::sort(dir.begin(), dir.end());
    dir.erase(std::unique(dir.begin(), dir.end()), dir.end());
    Graph g;
    g.n = n;
    g.off.assign((size_t)n + 1, 0);
    for (const auto& e : dir) ++g.off[e.first + 1];
    for (int32_t v = 0; v < n; ++v) g.off[v + 1] += g.off[v];
    g.adj.resize(dir.size());
    for (size_t i = 0; i < dir.size(); ++i) g.adj[i] = dir[i].second;
    return g;
}

// the element-adjacency edges (face neighbours), u < v not required
std::vector<std::pair<int32_t, int32_t>> dual_edges(const MeshData& m) {
    struct Face {
        int32_t k[3];
        int32_t e;
    };
    static constexpr int kFaces[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
    std::vector<Face> faces((size_t)4 * m.E);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m.E; ++e)
        for (int f = 0; f < 4; ++f) {
            int32_t k[3] = {m.tets[4 * e + kFaces[f][0]], m.tets[4 * e + kFaces[f][1]], m.tets[4 * e + kFaces[f][2]]};
            std::sort(k, k + 3);
            faces[4 * e + f] = {{k[0], k[1], k[2]}, (int32_t)e};
        }
    auto key_less = [](const Face& a, const Face& b) {
        if (a.k[0] != b.k[0]) return a.k[0] < b.k[0];
        if (a.k[1] != b.k[1]) return a.k[1] < b.k[1];
        if (a.k[2] != b.k[2]) return a.k[2] < b.k[2];
        return a.e < b.e;
    };
    std::sort(faces.begin(), faces.end(), key_less);
    std::vector<std::pair<int32_t, int32_t>> edges;
    for (size_t i = 0; i + 1 < faces.size(); ++i)
        if (faces[i].k[0] == faces[i + 1].k[0] && faces[i].k[1] == faces[i + 1].k[1] &&
            faces[i].k[2] == faces[i + 1].k[2])
            edges.emplace_back(faces[i].e, faces[i + 1].e);
    return edges;
}

// the unassigned vertex farthest (BFS hops) from the assigned set; unreachable vertices are
// farthest; the lowest index wins ties (farthest_unassigned partition.hpp:97-126)
int32_t farthest_unassigned(const Graph& g, const std::vector<int32_t>& assign, std::vector<int32_t>& dist,
                            std::vector<int32_t>& queue) {
    constexpr int32_t kUnreached = std::numeric_limits<int32_t>::max();
    dist.assign(g.n, kUnreached);
    queue.clear();
    for (int32_t v = 0; v < g.n; ++v)
        if (assign[v] >= 0) {
            dist[v] = 0;
            queue.push_back(v);
        }
    for (size_t h = 0; h < queue.size(); ++h) {
        const int32_t v = queue[h];
        for (int64_t j = g.off[v]; j < g.off[v + 1]; ++j) {
            const int32_t u = g.adj[j];
            if (assign[u] < 0 && dist[u] == kUnreached) {
                dist[u] = dist[v] + 1;
                queue.push_back(u);
            }
        }
    }
    int32_t best = -1, best_d = -1;
    for (int32_t v = 0; v < g.n; ++v)
        if (assign[v] < 0 && dist[v] > best_d) {
            best_d = dist[v];
            best = v;
        }
    return best;
}

}  // namespace

std::vector<int32_t> partition_graph(const Graph& g, const std::vector<int32_t>& w, int32_t k, double tol) {
    const int32_t n = g.n;
    if (k < 1) raise(CF_VALIDATION, "part count must be >= 1");
    if ((int64_t)w.size() != n) raise(CF_VALIDATION, "weight array size mismatch");
    int64_t total = 0;
    for (int32_t x : w) total += x;
    if (k > total)
        raise(CF_VALIDATION, "requested " + std::to_string(k) + " parts for " + std::to_string(total) +
                                 " weighted elements");
    std::vector<int32_t> assign(n, -1);
    if (k == 1) {
        std::fill(assign.begin(), assign.end(), 0);
        return assign;
    }
    std::vector<int64_t> pw(k, 0);
    std::vector<int32_t> stamp(n, -1), dist, scratch;
    int64_t done = 0;
    std::deque<int32_t> q;
    for (int32_t p = 0; p < k; ++p) {
        const int64_t target = (total - done + (k - p) - 1) / (k - p);  // ceil of the remaining share
        int32_t seed = p == 0 ? 0 : farthest_unassigned(g, assign, dist, scratch);
        while (pw[p] < target && seed >= 0) {
            q.assign(1, seed);
            stamp[seed] = p;
            while (!q.empty() && pw[p] < target) {
                const int32_t v = q.front();
                q.pop_front();
                if (assign[v] >= 0) continue;
                assign[v] = p;
                pw[p] += w[v];
                done += w[v];
                for (int64_t j = g.off[v]; j < g.off[v + 1]; ++j) {
                    const int32_t u = g.adj[j];
                    if (assign[u] < 0 && stamp[u] != p) {
                        stamp[u] = p;
                        q.push_back(u);
                    }
                }
            }
            if (pw[p] < target) seed = farthest_unassigned(g, assign, dist, scratch);
        }
    }
    for (int32_t v = 0; v < n; ++v) {  // zero-weight leftovers join their lowest-id assigned neighbour
        if (assign[v] >= 0) continue;
        int32_t p = k - 1;
        for (int64_t j = g.off[v]; j < g.off[v + 1]; ++j)
            if (assign[g.adj[j]] >= 0) {
                p = assign[g.adj[j]];
                break;
            }
        assign[v] = p;
        pw[p] += w[v];
    }
    // boundary refinement: a boundary vertex moves to its most adjacent other part when that
    // strictly cuts fewer edges and keeps the part weights within the cap
    const double mean = (double)total / k;
    const int64_t cap = std::max<int64_t>((total + k - 1) / k, (int64_t)(mean * (1.0 + tol)));
    std::vector<int32_t> adjc(k, 0);
    for (int pass = 0; pass < 8; ++pass) {
        bool moved = false;
        for (int32_t v = 0; v < n; ++v) {
            const int32_t p = assign[v];
            bool boundary = false;
            for (int64_t j = g.off[v]; j < g.off[v + 1]; ++j) boundary = boundary || assign[g.adj[j]] != p;
            if (!boundary) continue;
            for (int64_t j = g.off[v]; j < g.off[v + 1]; ++j) ++adjc[assign[g.adj[j]]];
            int32_t best = -1;
            for (int32_t c = 0; c < k; ++c)
                if (c != p && adjc[c] > 0 && (best < 0 || adjc[c] > adjc[best])) best = c;
            const int32_t gain = best >= 0 ? adjc[best] - adjc[p] : 0;
            for (int64_t j = g.off[v]; j < g.off[v + 1]; ++j) adjc[assign[g.adj[j]]] = 0;
            if (best < 0 || gain <= 0) continue;
            if (pw[p] - w[v] < 1 || pw[best] + w[v] > cap) continue;
            assign[v] = best;
            pw[p] -= w[v];
            pw[best] += w[v];
            moved = true;
        }
        if (!moved) break;
    }
    return assign;
}

Graph dual_graph(const MeshData& m) {
    auto e = dual_edges(m);
    return csr_from_edges(m.E, e);
}

std::vector<int32_t> partition_elements(const MeshData& m, int32_t k, double tol, bool augment) {
    auto edges = dual_edges(m);
    int32_t nv = m.E;
    if (augment) {
        // augment_virtual_elements (one side): vertex E + i for the i-th cast-side interface pair
        const std::vector<Pair> pairs = pair_sister_facets(m);
        for (const Pair& pr : pairs) {
            if (pr.contact < 0 || 2 * pr.contact + 1 >= (int32_t)m.contacts.size())
                raise(CF_VALIDATION, "interface pair references unknown contact");
            if (m.facet_tag[pr.facet] != m.contacts[2 * pr.contact]) continue;
            edges.emplace_back(nv, m.owner[pr.facet]);
            edges.emplace_back(nv, pr.sister);
            ++nv;
        }
    }
    const Graph g = csr_from_edges(nv, edges);
    std::vector<int32_t> w(nv, 0);
    std::fill(w.begin(), w.begin() + m.E, 1);
    std::vector<int32_t> part = partition_graph(g, w, k, tol);
    part.resize(m.E);  // the virtual tail is dropped (partition_elements partition.hpp:236-241)
    return part;
}

PartitionQuality partition_metrics(const MeshData& m, const int32_t* part, int32_t k) {
    PartitionQuality q;
    const Graph g = dual_graph(m);
    std::vector<char> adj((size_t)k * k, 0);
    for (int32_t u = 0; u < g.n; ++u)
        for (int64_t j = g.off[u]; j < g.off[u + 1]; ++j) {
            const int32_t v = g.adj[j];
            if (u >= v) continue;
            const int32_t pu = part[u], pv = part[v];
            if (pu != pv) {
                ++q.edge_cut;
                adj[(size_t)pu * k + pv] = adj[(size_t)pv * k + pu] = 1;
            }
        }
    q.neighbor_counts.assign(k, 0);
    for (int32_t p = 0; p < k; ++p)
        for (int32_t c = 0; c < k; ++c) q.neighbor_counts[p] += adj[(size_t)p * k + c];
    std::vector<int64_t> count(k, 0);
    for (int32_t e = 0; e < m.E; ++e) ++count[part[e]];
    const int64_t mx = m.E ? *std::max_element(count.begin(), count.end()) : 0;
    q.imbalance = m.E ? (double)mx * k / m.E : 1.0;
    return q;
}

int64_t count_split_interface_pairs(const MeshData& m, const int32_t* part) {
    int64_t split = 0;
    for (const Pair& pr : pair_sister_facets(m)) split += part[m.owner[pr.facet]] != part[pr.sister];
    return split;
}

}  // namespace cfb
