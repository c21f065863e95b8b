// partition.cu -- host side of the multi-GPU path: the bus-graph
// cut and the rank-local problem with its halo.
//
// Ownership: bus i -> part[i]; generator g -> part[gen_bus[g]]; branch l = (i -> j) ->
// part[i].  Every period of a component stays on its rank, so the DP, the ramp rows and the RC
// rows are local.  The only cross-rank coupling is the bus update (7d) of a cut branch's
// to-bus j: the branch owner sends the four bus-side targets (tauhat of FP_ji, FQ_ji, W_j, A_j)
// and receives bus j's (muP, muQ, dwbar, dthbar, wbar, thbar) back.
//
// Rank-local numbering (all lists sorted by global id, so the bus sums run in the single-GPU
// canonical (l, side) order and the partitioned iteration is bitwise the single-GPU one):
//   buses    : owned [0, Bo) then ghosts [Bo, Bo + Bg) (remote to-buses of local branches)
//   branches : local [0, Lo) then phantoms [Lo, Lo + Lp) (remote branches whose to-bus is owned)
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

#include "ucac.h"
#include "ucac_part.h"

namespace ucac {

// weighted recursive coordinate bisection (coordinates given) or weighted BFS-order split
static void rcb(std::vector<int> &idx, const double *xy, const std::vector<double> &w, int p0, int np,
                int32_t *part) {
    if (np == 1) {
        for (int i : idx) part[i] = p0;
        return;
    }
    double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
    for (int i : idx) {
        xmin = std::min(xmin, xy[2 * i]);
        xmax = std::max(xmax, xy[2 * i]);
        ymin = std::min(ymin, xy[2 * i + 1]);
        ymax = std::max(ymax, xy[2 * i + 1]);
    }
    const int ax = (xmax - xmin) >= (ymax - ymin) ? 0 : 1;
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
        if (xy[2 * a + ax] != xy[2 * b + ax]) return xy[2 * a + ax] < xy[2 * b + ax];
        return a < b;
    });
    const int n1 = np / 2;
    double wt = 0.0;
    for (int i : idx) wt += w[i];
    const double target = wt * (double)n1 / (double)np;
    double acc = 0.0;
    size_t cut = 0;
    while (cut < idx.size() && acc + w[idx[cut]] * 0.5 <= target) acc += w[idx[cut++]];
    cut = std::max<size_t>(1, std::min(cut, idx.size() - 1));
    std::vector<int> a(idx.begin(), idx.begin() + cut), b(idx.begin() + cut, idx.end());
    rcb(a, xy, w, p0, n1, part);
    rcb(b, xy, w, p0 + n1, np - n1, part);
}

// Greedy boundary refinement with Fiduccia-Mattheyses gains: a bus moves to the neighbouring part
// that cuts the most incident branches less (gain = branches to that part - branches to its own),
// if the gain is positive and both parts stay within +-tol of the mean weight.  Buses in index
// order, passes until no move (at most 20): deterministic, and the cut only shrinks.
static void fm_refine(int nbus, int nbranch, const int32_t *from, const int32_t *to, const std::vector<double> &w,
                      int nparts, int32_t *part, double tol) {
    std::vector<std::vector<int>> adj(nbus);
    for (int l = 0; l < nbranch; l++) {
        adj[from[l]].push_back(to[l]);
        adj[to[l]].push_back(from[l]);
    }
    std::vector<double> load(nparts, 0.0);
    double tot = 0.0;
    for (int i = 0; i < nbus; i++) {
        load[part[i]] += w[i];
        tot += w[i];
    }
    const double hi = (1.0 + tol) * tot / nparts, lo = (1.0 - tol) * tot / nparts;
    std::vector<int> cnt(nparts, 0);
    for (int pass = 0; pass < 20; pass++) {
        int moved = 0;
        for (int i = 0; i < nbus; i++) {
            const int a = part[i];
            for (int v : adj[i]) cnt[part[v]]++;
            int best = a, bg = 0;
            for (int v : adj[i]) {
                const int b = part[v];
                const int g = cnt[b] - cnt[a];
                if (b != a && (g > bg || (g == bg && best != a && b < best)) && load[b] + w[i] <= hi && load[a] - w[i] >= lo) {
                    best = b;
                    bg = g;
                }
            }
            for (int v : adj[i]) cnt[part[v]] = 0;
            if (best != a && bg > 0) {
                part[i] = best;
                load[a] -= w[i];
                load[best] += w[i];
                moved++;
            }
        }
        if (!moved) break;
    }
}

int partition_buses(int nbus, int nbranch, const int32_t *from, const int32_t *to, const double *xy, int nparts,
                    int32_t *part, const double *branch_w) {
    if (nbus <= 0 || nparts <= 0 || nparts > nbus) return 1;
    // weight: one unit per bus plus, per owned branch, its expected solve work (1 when not given; a
    // caller can pass e.g. 1 + the branch's thermal-AL Newton share)
    std::vector<double> w(nbus, 1.0);
    for (int l = 0; l < nbranch; l++) w[from[l]] += branch_w ? branch_w[l] : 1.0;
    if (xy) {
        std::vector<int> idx(nbus);
        std::iota(idx.begin(), idx.end(), 0);
        rcb(idx, xy, w, 0, nparts, part);
        fm_refine(nbus, nbranch, from, to, w, nparts, part, 0.05);
        return 0;
    }
    // no coordinates: BFS order from bus 0 (neighbours in id order), contiguous weighted chunks
    std::vector<std::vector<int>> adj(nbus);
    for (int l = 0; l < nbranch; l++) {
        adj[from[l]].push_back(to[l]);
        adj[to[l]].push_back(from[l]);
    }
    for (auto &a : adj) std::sort(a.begin(), a.end());
    std::vector<int> order;
    std::vector<char> seen(nbus, 0);
    for (int s = 0; s < nbus; s++) {
        if (seen[s]) continue;
        seen[s] = 1;
        size_t h = order.size();
        order.push_back(s);
        while (h < order.size()) {
            int u = order[h++];
            for (int v : adj[u])
                if (!seen[v]) {
                    seen[v] = 1;
                    order.push_back(v);
                }
        }
    }
    double wt = 0.0;
    for (double x : w) wt += x;
    double acc = 0.0;
    for (int i : order) {
        int p = (int)std::min<double>(nparts - 1, (acc + 0.5 * w[i]) * nparts / wt);
        part[i] = p;
        acc += w[i];
    }
    fm_refine(nbus, nbranch, from, to, w, nparts, part, 0.05);
    return 0;
}

Halo build_halo(int nbus, int nbranch, const int32_t *from, const int32_t *to, const int32_t *part, int nparts,
                int rank) {
    Halo h;
    h.nparts = nparts;
    h.rank = rank;
    h.bus_local.assign(nbus, -1);
    for (int i = 0; i < nbus; i++)
        if (part[i] == rank) h.own_bus.push_back(i);
    for (int l = 0; l < nbranch; l++) {
        if (part[from[l]] == rank) {
            h.local_branch.push_back(l);
            if (part[to[l]] != rank) h.ghost_bus.push_back(to[l]);
        } else if (part[to[l]] == rank) {
            h.phantom.push_back(l);
        }
    }
    std::sort(h.ghost_bus.begin(), h.ghost_bus.end());
    h.ghost_bus.erase(std::unique(h.ghost_bus.begin(), h.ghost_bus.end()), h.ghost_bus.end());
    for (size_t a = 0; a < h.own_bus.size(); a++) h.bus_local[h.own_bus[a]] = (int)a;
    for (size_t a = 0; a < h.ghost_bus.size(); a++) h.bus_local[h.ghost_bus[a]] = (int)(h.own_bus.size() + a);
    // every rank's cut-branch list (local branches with a remote to-bus) and export-bus list
    // (owned buses that are the to-bus of a remote branch), in global id order
    std::vector<std::vector<int>> cut(nparts), exp(nparts);
    for (int l = 0; l < nbranch; l++)
        if (part[from[l]] != part[to[l]]) {
            cut[part[from[l]]].push_back(l);
            exp[part[to[l]]].push_back(to[l]);
        }
    for (auto &e : exp) {
        std::sort(e.begin(), e.end());
        e.erase(std::unique(e.begin(), e.end()), e.end());
    }
    size_t maxc = 0, maxe = 0;
    for (int q = 0; q < nparts; q++) {
        maxc = std::max(maxc, cut[q].size());
        maxe = std::max(maxe, exp[q].size());
    }
    h.max_cut = (int)maxc;
    h.max_export = (int)maxe;
    // local ids of my cut branches, my export buses
    std::vector<int> br_local(nbranch, -1);
    for (size_t a = 0; a < h.local_branch.size(); a++) br_local[h.local_branch[a]] = (int)a;
    for (size_t a = 0; a < h.phantom.size(); a++) br_local[h.phantom[a]] = (int)(h.local_branch.size() + a);
    for (int l : cut[rank]) h.cut_local.push_back(br_local[l]);
    for (int i : exp[rank]) h.export_local.push_back(h.bus_local[i]);
    // where each phantom / ghost comes from in the gathered buffers: (owner rank, position)
    for (int l : h.phantom) {
        int q = part[from[l]];
        int pos = (int)(std::lower_bound(cut[q].begin(), cut[q].end(), l) - cut[q].begin());
        h.phantom_src.push_back(q * (int)maxc + pos);
    }
    for (int i : h.ghost_bus) {
        int q = part[i];
        int pos = (int)(std::lower_bound(exp[q].begin(), exp[q].end(), i) - exp[q].begin());
        h.ghost_src.push_back(q * (int)maxe + pos);
    }
    h.br_local = br_local;
    return h;
}

}  // namespace ucac

extern "C" ucac_status ucac_partition(int32_t nbus, int32_t nbranch, const int32_t *br_from, const int32_t *br_to,
                                      const double *bus_xy, int32_t nparts, int32_t *part, const double *branch_w) {
    if (!br_from || !br_to || !part || nbus <= 0 || nbranch < 0 || nparts < 1 || nparts > nbus) return UCAC_EINVAL;
    for (int l = 0; l < nbranch; l++)
        if (br_from[l] < 0 || br_from[l] >= nbus || br_to[l] < 0 || br_to[l] >= nbus) return UCAC_EINVAL;
    return ucac::partition_buses(nbus, nbranch, br_from, br_to, bus_xy, nparts, part, branch_w) ? UCAC_EINVAL : UCAC_OK;
}

extern "C" ucac_status ucac_halo_lists(int32_t nbus, int32_t nbranch, const int32_t *br_from, const int32_t *br_to,
                                       const int32_t *part, int32_t nparts, int32_t rank, int32_t *sizes,
                                       int32_t *own_bus, int32_t *ghost_bus, int32_t *local_branch,
                                       int32_t *phantom, int32_t *cut_branch, int32_t *export_bus) {
    if (!br_from || !br_to || !part || !sizes || nparts < 1 || rank < 0 || rank >= nparts) return UCAC_EINVAL;
    for (int i = 0; i < nbus; i++)
        if (part[i] < 0 || part[i] >= nparts) return UCAC_EINVAL;
    ucac::Halo h = ucac::build_halo(nbus, nbranch, br_from, br_to, part, nparts, rank);
    sizes[0] = (int32_t)h.own_bus.size();
    sizes[1] = (int32_t)h.ghost_bus.size();
    sizes[2] = (int32_t)h.local_branch.size();
    sizes[3] = (int32_t)h.phantom.size();
    sizes[4] = (int32_t)h.cut_local.size();
    sizes[5] = (int32_t)h.export_local.size();
    auto cp = [](int32_t *dst, const std::vector<int> &v) {
        if (dst) std::copy(v.begin(), v.end(), dst);
    };
    cp(own_bus, h.own_bus);
    cp(ghost_bus, h.ghost_bus);
    cp(local_branch, h.local_branch);
    cp(phantom, h.phantom);
    if (cut_branch)
        for (size_t a = 0; a < h.cut_local.size(); a++) cut_branch[a] = h.local_branch[h.cut_local[a]];
    if (export_bus)
        for (size_t a = 0; a < h.export_local.size(); a++) export_bus[a] = h.own_bus[h.export_local[a]];
    return UCAC_OK;
}
