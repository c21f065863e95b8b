// ucac.cu -- host runtime of libucac.so: the C ABI of include/ucac.h.
//
// create: validate -> build the rank-local problem (the whole problem on one GPU; the bus-graph
// cut with its halo on several) -> device layout (SoA, CSR incidence in canonical
// order) -> cold start kernel -> CUDA graphs of 1 and 16 inner iterations.  iterate: graph
// launches back to back; the device status word carries the inner test, the outer (lambda,
// beta) decision and the stop-on-primal flag, so the host never looks at the iterate.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <limits>
#include <vector>

#include "ucac.h"

// NVTX ranges (tracing): one per public call, one per ucac_create phase and one per eager
// kernel of ucac_iterate_timed, named as the call / phase / kernel.  Header-only NVTX v3: without a
// profiler attached each push/pop is a test of a null callback.
#include <nvtx3/nvToolsExt.h>
namespace {
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};
}  // namespace
#define UCAC_NVTX(name) NvtxRange nvtx_range_(name)

// graph shape: the generator chain forks at the start of the iteration, on a
// higher-priority stream
#ifndef UCAC_EARLY_FORK
#define UCAC_EARLY_FORK 1
#endif
#ifndef UCAC_UNROLL_MAX_LT
#define UCAC_UNROLL_MAX_LT 50000   // L*T above which no 16-iteration graph is built
#endif
#ifndef UCAC_NODE_PRIO
#define UCAC_NODE_PRIO 0   // honouring node priorities measured neutral (0.1700-0.1712 ms)
#endif
#ifndef UCAC_UBAR_AFTER_BUS
#define UCAC_UBAR_AFTER_BUS 0   // 1 measured slower (0.186 vs 0.181 ms): k_ubar then delays the early fold
#endif
#ifndef UCAC_EXEC_POOL
#define UCAC_EXEC_POOL 1   // recycle instantiated graphs across contexts (cudaGraphExecUpdate)
#endif
#ifndef UCAC_FUSE_ROWS
#define UCAC_FUSE_ROWS 0   // measured slower: 0.203 vs 0.182 ms (per-thread end loops lengthen the late chains)
#endif
#ifndef UCAC_PIPE_DP
#define UCAC_PIPE_DP 1
#endif
#ifndef UCAC_S2_PRIO
#define UCAC_S2_PRIO 1
#endif
#include "ucac_dev.cuh"
static_assert(UCAC_HIST_CAP == ucac::HIST_CAP && UCAC_HIST_FIELDS == ucac::HIST_FIELDS, "ucac_history layout");
#include "ucac_part.h"

namespace ucac {
void launch_apply_outer(const Dev &d, cudaStream_t s);
cudaError_t gen_set_smem_attr(int T);
size_t gen_smem_bytes(int T);
}  // namespace ucac

using namespace ucac;

static thread_local std::string g_create_err;

// ------------------------------------------------------------------------------------------
// the rank-local problem (host vectors) -- identity for a single GPU
// ------------------------------------------------------------------------------------------
struct Local {
    int B = 0, Bo = 0, G = 0, L = 0, Lp = 0, T = 0, ref = -1;
    double S = 100.0;
    std::vector<double> gs, bs, vmin, vmax;                      // buses (own + ghost)
    std::vector<int> from, to;                                    // local branches (local bus ids)
    std::vector<double> ysoa, rate;
    std::vector<int> gbus, tu, td, u0, hold;                      // local generators
    std::vector<double> pmin, pmax, qmin, qmax, c2, c1, c0, csu, csd, rup, rdn, sup, sdn, p0;
    std::vector<int8_t> uinit;                                    // [G*T] or empty
    std::vector<int> bgp, bgi, bep, bei;                          // CSR for owned buses
    std::vector<int> gen_global, branch_global, bus_global;      // local -> global (owned buses)
    // halo
    std::vector<int> cut_local, export_local, phantom_src, ghost_src;
    int max_cut = 0, max_export = 0;
    std::vector<int> phantom_bus;                                 // [Lp] owned local bus of each phantom
    std::vector<int> gep, gei;                                    // CSR ghost bus -> local end codes
    // periods: local period t = global t + t_off of Tg, owned [own0, own1) (time cut, NEXT-4(c))
    int t_off = 0, Tg = 0, own0 = 0, own1 = 0, Tmax = 0;
    std::vector<int> tstart;                                       // [nranks + 1] owned global ranges
};

// NEXT-4(c) time cut: rank r owns the global periods [r Tg / n, (r + 1) Tg / n) of every
// component, plus one halo period on each side that is not the horizon's end.
static void time_split(int Tg, int nranks, std::vector<int> &t0) {
    t0.assign(nranks + 1, 0);
    for (int r = 0; r <= nranks; r++) t0[r] = (int)(((long long)r * Tg) / nranks);
}
static Local localize_periods(Local P, const ucac_horizon *hz, const ucac_uc *uc, int nranks, int rank) {
    const int Tg = P.T;
    time_split(Tg, nranks, P.tstart);
    const int g0 = P.tstart[rank], g1 = P.tstart[rank + 1];
    const int hl = g0 > 0, hh = g1 < Tg;
    const int Tl = (g1 - g0) + hl + hh;
    P.Tg = Tg;
    P.t_off = g0 - hl;
    P.own0 = hl;
    P.own1 = hl + (g1 - g0);
    P.Tmax = 0;
    for (int r = 0; r < nranks; r++) P.Tmax = std::max(P.Tmax, P.tstart[r + 1] - P.tstart[r]);
    if (!P.uinit.empty()) {
        std::vector<int8_t> u((size_t)P.G * Tl);
        for (int g = 0; g < P.G; g++)
            for (int t = 0; t < Tl; t++) u[(size_t)g * Tl + t] = P.uinit[(size_t)g * Tg + P.t_off + t];
        P.uinit.swap(u);
    }
    (void)hz;
    (void)uc;
    P.T = Tl;
    return P;
}

static Local build_local(const ucac_network *net, const ucac_horizon *hz, const ucac_costs *co, const ucac_uc *uc,
                         const int32_t *part, int nranks, int rank) {
    Local P;
    const int B = net->nbus, G = net->ngen, L = net->nbranch, T = hz->T;
    P.T = T;
    P.S = net->base_mva;
    Halo h;
    if (nranks > 1) {
        h = build_halo(B, L, net->br_from, net->br_to, part, nranks, rank);
    } else {
        h.own_bus.resize(B);
        for (int i = 0; i < B; i++) h.own_bus[i] = i;
        h.local_branch.resize(L);
        for (int l = 0; l < L; l++) h.local_branch[l] = l;
        h.bus_local.resize(B);
        for (int i = 0; i < B; i++) h.bus_local[i] = i;
        h.br_local.resize(L);
        for (int l = 0; l < L; l++) h.br_local[l] = l;
    }
    P.Bo = (int)h.own_bus.size();
    P.B = P.Bo + (int)h.ghost_bus.size();
    P.L = (int)h.local_branch.size();
    P.Lp = (int)h.phantom.size();
    std::vector<int> bus_glob(h.own_bus);
    bus_glob.insert(bus_glob.end(), h.ghost_bus.begin(), h.ghost_bus.end());
    P.bus_global = h.own_bus;
    for (int a = 0; a < P.B; a++) {
        int i = bus_glob[a];
        P.gs.push_back(net->bus_gs[i]);
        P.bs.push_back(net->bus_bs[i]);
        P.vmin.push_back(net->bus_vmin[i]);
        P.vmax.push_back(net->bus_vmax[i]);
    }
    P.ref = h.bus_local[net->ref_bus] >= 0 && h.bus_local[net->ref_bus] < P.Bo ? h.bus_local[net->ref_bus] : -1;
    P.ysoa.assign((size_t)8 * P.L, 0.0);
    P.from.reserve(P.L);
    P.to.reserve(P.L);
    P.rate.reserve(P.L);
    for (int a = 0; a < P.L; a++) {
        int l = h.local_branch[a];
        P.from.push_back(h.bus_local[net->br_from[l]]);
        P.to.push_back(h.bus_local[net->br_to[l]]);
        P.rate.push_back(net->br_rate[l]);
        for (int k = 0; k < 8; k++) P.ysoa[(size_t)k * P.L + a] = net->br_y[(size_t)l * 8 + k];
    }
    P.branch_global = h.local_branch;
    for (int g = 0; g < G; g++) {
        int lb = h.bus_local[net->gen_bus[g]];
        if (lb < 0 || lb >= P.Bo) continue;
        P.gen_global.push_back(g);
        P.gbus.push_back(lb);
        P.tu.push_back(uc->min_up[g]);
        P.td.push_back(uc->min_dn[g]);
        P.u0.push_back(uc->u0[g]);
        P.hold.push_back(uc->hold[g]);
        P.pmin.push_back(net->gen_pmin[g]);
        P.pmax.push_back(net->gen_pmax[g]);
        P.qmin.push_back(net->gen_qmin[g]);
        P.qmax.push_back(net->gen_qmax[g]);
        P.c2.push_back(co->c2[g]);
        P.c1.push_back(co->c1[g]);
        P.c0.push_back(co->c0[g]);
        P.csu.push_back(co->startup[g]);
        P.csd.push_back(co->shutdown[g]);
        P.rup.push_back(uc->ramp_up[g]);
        P.rdn.push_back(uc->ramp_dn[g]);
        P.sup.push_back(uc->su_ramp[g]);
        P.sdn.push_back(uc->sd_ramp[g]);
        P.p0.push_back(uc->p0[g]);
        if (uc->u_init)
            for (int t = 0; t < T; t++) P.uinit.push_back(uc->u_init[(size_t)g * T + t]);
    }
    P.G = (int)P.gen_global.size();
    // CSR of the owned buses in canonical order: generators by global index, then branch ends by
    // global (l, side) -- local and phantom branches interleaved exactly as on one GPU
    P.bgp.assign(P.Bo + 1, 0);
    P.bep.assign(P.Bo + 1, 0);
    for (int a = 0; a < P.G; a++) P.bgp[P.gbus[a] + 1]++;
    struct End { int gl, side, bus, code; };
    std::vector<End> ends;
    ends.reserve((size_t)2 * L);
    for (int l = 0; l < L; l++) {
        int lf = h.bus_local[net->br_from[l]], lt = h.bus_local[net->br_to[l]];
        int ll = h.br_local[l];
        if (ll < 0) continue;
        if (lf >= 0 && lf < P.Bo && ll < P.L) ends.push_back({l, 0, lf, 2 * ll});
        if (lt >= 0 && lt < P.Bo) ends.push_back({l, 1, lt, 2 * ll + 1});
    }
    for (auto &e : ends) P.bep[e.bus + 1]++;
    for (int i = 0; i < P.Bo; i++) {
        P.bgp[i + 1] += P.bgp[i];
        P.bep[i + 1] += P.bep[i];
    }
    P.bgi.assign(P.G, 0);
    P.bei.assign(ends.size(), 0);
    {
        std::vector<int> fg(P.Bo, 0), fe(P.Bo, 0);
        for (int a = 0; a < P.G; a++) P.bgi[P.bgp[P.gbus[a]] + fg[P.gbus[a]]++] = a;
        for (auto &e : ends) P.bei[P.bep[e.bus] + fe[e.bus]++] = e.code;   // ends already in (l, side) order
    }
    P.cut_local = h.cut_local;
    P.export_local = h.export_local;
    P.phantom_src = h.phantom_src;
    P.ghost_src = h.ghost_src;
    P.max_cut = h.max_cut;
    P.max_export = h.max_export;
    // early/late split across ranks: the owned to-bus of every phantom, and per ghost
    // bus the local branch ends at it (end codes 2 l + 1, l ascending)
    for (int p = 0; p < P.Lp; p++) P.phantom_bus.push_back(h.bus_local[net->br_to[h.phantom[p]]]);
    const int Bg = P.B - P.Bo;
    P.gep.assign(Bg + 1, 0);
    for (int a = 0; a < P.L; a++)
        if (P.to[a] >= P.Bo) P.gep[P.to[a] - P.Bo + 1]++;
    for (int g = 0; g < Bg; g++) P.gep[g + 1] += P.gep[g];
    P.gei.assign(P.gep[Bg], 0);
    {
        std::vector<int> fill(Bg, 0);
        for (int a = 0; a < P.L; a++)
            if (P.to[a] >= P.Bo) {
                const int g = P.to[a] - P.Bo;
                P.gei[P.gep[g] + fill[g]++] = 2 * a + 1;
            }
    }
    return P;
}

struct ucac_ctx {
    Dev d{};
    Local P;
    int G = 0, L = 0, B = 0, T = 0;      // local counts (B = owned buses)
    int nranks = 1, rank = 0, comm_mode = 0;
    bool multi = false;                  // the multi-rank iteration graph (nranks > 1, or UCAC_NCCL_ONE_RANK)
    ncclComm_t comm = nullptr;
    ncclComm_t comm2 = nullptr;          // bus cut: the early exchanges' communicator (stream s3)
    cudaStream_t s = nullptr, s2 = nullptr, s3 = nullptr;
    bool own_stream = false;
    long long hist_base = 0;             // inner_total when the record history was last emptied
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_genx = nullptr, ev_early = nullptr, ev_branch = nullptr,
                ev_tail = nullptr, ev_bus = nullptr;
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    int gunroll[2] = {1, 16};
    std::vector<void *> dalloc;
    DevStatus *st_host = nullptr;        // pinned mirror
    double *xpose = nullptr;             // [4 LT] scratch for SoA -> AoS read-back
    std::string err;
    std::vector<cudaEvent_t> tev;        // timed-iteration event pool
    ucac_params prm{};
    bool ctl_dirty = true;               // device control fields may hold a stop/done state
    void *xbuf = nullptr;                // time cut: receive buffers + flags (cudaMalloc, IPC-mappable)
    size_t xoff[4] = {0, 0, 0, 0}, xbytes = 0;
    std::vector<void *> peer_maps;       // CUDA IPC mappings of the peers' xbuf
    Dev *xdevs = nullptr;                // loopback group: device copy of the group's Dev records
    ncclResult_t nccl_err = ncclSuccess; // first failed collective of a graph capture
};

#define CK(call)                                                                           \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) {                                                           \
            ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);                \
            return UCAC_ECUDA;                                                             \
        }                                                                                  \
    } while (0)
#define NK(call)                                                                           \
    do {                                                                                   \
        ncclResult_t r_ = (call);                                                          \
        if (r_ != ncclSuccess) {                                                           \
            ctx->err = std::string(#call) + ": " + ncclGetErrorString(r_);                \
            return UCAC_ENCCL;                                                             \
        }                                                                                  \
    } while (0)

static ucac_status fail(ucac_ctx *ctx, ucac_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (ctx) ctx->err = buf;
    else g_create_err = buf;
    return s;
}

template <class Tp>
static cudaError_t up(ucac_ctx *ctx, Tp *dst, const Tp *src, size_t n) {
    if (n == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, n * sizeof(Tp), cudaMemcpyHostToDevice, ctx->s);
}

// Pinned DevStatus buffers are recycled across contexts: a page-locked allocation costs
// milliseconds, a context needs one small buffer.
static std::mutex g_pinned_mu;
static std::vector<DevStatus *> g_pinned_free;
static DevStatus *pinned_status_get() {
    {
        std::lock_guard<std::mutex> lk(g_pinned_mu);
        if (!g_pinned_free.empty()) {
            DevStatus *p = g_pinned_free.back();
            g_pinned_free.pop_back();
            return p;
        }
    }
    void *p = nullptr;
    return cudaMallocHost(&p, sizeof(DevStatus)) == cudaSuccess ? (DevStatus *)p : nullptr;
}
static void pinned_status_put(DevStatus *p) {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    g_pinned_free.push_back(p);
}

// Page-locked staging image for ucac_create's upload, kept across contexts and grown on demand
// (the upload is one DMA from it instead of the driver's pageable double copy); held under its
// mutex from the host-side layout to the end of the upload.  It lives for the process (as the
// pinned status records do): its size is the largest problem's input image (2.8 MB for pegase
// T = 48), and freeing it at the last context would make the next ucac_create pay the pinning.
// The upload out of it is asynchronous: g_stage_ev, recorded after the copy, is waited for before
// the image is written or freed again.
static std::mutex g_stage_mu;
static char *g_stage = nullptr;
static size_t g_stage_cap = 0;
static cudaEvent_t g_stage_ev = nullptr;
static bool g_stage_ev_pending = false;
static char *stage_get(size_t n) {   // caller holds g_stage_mu
    if (g_stage_ev_pending) {
        if (cudaEventSynchronize(g_stage_ev) != cudaSuccess) return nullptr;
        g_stage_ev_pending = false;
    }
    if (n <= g_stage_cap) return g_stage;
    if (g_stage) cudaFreeHost(g_stage);
    g_stage = nullptr;
    g_stage_cap = 0;
    const size_t cap = std::max<size_t>(n + n / 4, 1 << 20);
    void *p = nullptr;
    if (cudaMallocHost(&p, cap) != cudaSuccess) return nullptr;
    g_stage = (char *)p;
    g_stage_cap = cap;
    return g_stage;
}

// Bump allocator over one device allocation: 256-byte aligned slices.  With base == 0 it only
// measures (the sizing pass); with `stage` set, put() also copies the host vector into the
// staging image at the slice's offset.
struct Arena {
    uintptr_t base = 0;
    size_t off = 0, up_end = 0;
    char *stage = nullptr;
    template <class Tp> Tp *take(size_t n) {
        const size_t o = (off + 255) & ~(size_t)255;
        off = o + std::max<size_t>(n, 1) * sizeof(Tp);
        return base ? (Tp *)(base + o) : nullptr;
    }
    // a slice of n elements written by fill(dst) straight into the staging image
    template <class Tp, class F> Tp *put_fill(size_t n, F fill) {
        const size_t o = (off + 255) & ~(size_t)255;
        Tp *p = take<Tp>(n);
        if (stage) fill((Tp *)(stage + o));
        return p;
    }
    template <class Tp> Tp *put(const std::vector<Tp> &v) {
        const size_t o = (off + 255) & ~(size_t)255;
        Tp *p = take<Tp>(v.size());
        if (stage && !v.empty()) memcpy(stage + o, v.data(), v.size() * sizeof(Tp));
        if (stage && v.empty()) memset(stage + o, 0, sizeof(Tp));   // (the staging image is reused)
        return p;
    }
};

static bool finite_all(const double *a, size_t n) {
    // exponent all ones <=> inf or NaN; a branch-free OR over the bits (vectorises)
    const uint64_t E = 0x7ff0000000000000ull;
    uint64_t bad = 0;
    for (size_t i = 0; i < n; i++) {
        uint64_t b;
        memcpy(&b, a + i, sizeof b);
        bad |= (uint64_t)((b & E) == E);
    }
    return bad == 0;
}

// scan_demand = false: the demand's finiteness is checked while ucac_create transposes it into the
// staging image (one pass over the caller's arrays instead of two; single rank only)
static ucac_status validate(const ucac_network *net, const ucac_horizon *hz, const ucac_costs *co,
                            const ucac_uc *uc, const ucac_params *p, bool scan_demand) {
#define BAD(...) return fail(nullptr, UCAC_EINVAL, __VA_ARGS__)
    if (!net || !hz || !co || !uc || !p) BAD("null argument");
    const int B = net->nbus, G = net->ngen, L = net->nbranch, T = hz->T;
    if (B <= 0 || G <= 0 || L <= 0 || T <= 0) BAD("empty problem: nbus=%d ngen=%d nbranch=%d T=%d", B, G, L, T);
    if (net->ref_bus < 0 || net->ref_bus >= B) BAD("ref_bus %d out of range", net->ref_bus);
    if (!(net->base_mva > 0)) BAD("base_mva must be > 0");
    if (!(p->rho_pq > 0) || !(p->rho_va > 0) || !(p->rho_uc > 0)) BAD("rho must be > 0");
    if (!(p->beta0 > 0) || !(p->tau > 1) || !(p->theta > 0 && p->theta < 1)) BAD("bad beta0/tau/theta");
    const double *dd[] = {net->bus_gs, net->bus_bs, net->bus_vmin, net->bus_vmax};
    for (auto a : dd)
        if (!a || !finite_all(a, B)) BAD("bus arrays must be finite");
    for (int i = 0; i < B; i++)
        if (!(net->bus_vmin[i] > 0) || net->bus_vmin[i] > net->bus_vmax[i]) BAD("bus %d: need 0 < vmin <= vmax", i);
    if (!hz->pd || !hz->qd) BAD("demand arrays missing");
    if (scan_demand && (!finite_all(hz->pd, (size_t)T * B) || !finite_all(hz->qd, (size_t)T * B)))
        BAD("demand must be finite");
    if (!net->br_from || !net->br_to || !net->br_y || !net->br_rate) BAD("branch arrays missing");
    if (!finite_all(net->br_y, (size_t)L * 8) || !finite_all(net->br_rate, L)) BAD("branch data must be finite");
    std::vector<int> deg(B, 0);
    for (int l = 0; l < L; l++) {
        int i = net->br_from[l], j = net->br_to[l];
        if (i < 0 || i >= B || j < 0 || j >= B) BAD("branch %d: bus index out of range", l);
        if (i == j) BAD("branch %d: from == to", l);
        if (net->br_rate[l] < 0) BAD("branch %d: negative rate", l);
        deg[i]++;
        deg[j]++;
    }
    for (int i = 0; i < B; i++)
        if (deg[i] == 0) BAD("bus %d has no branch (bus 2x2 system singular)", i);
    const double *gd[] = {net->gen_pmin, net->gen_pmax, net->gen_qmin, net->gen_qmax, co->c2, co->c1, co->c0,
                          co->startup, co->shutdown, uc->ramp_up, uc->ramp_dn, uc->su_ramp, uc->sd_ramp, uc->p0};
    for (auto a : gd)
        if (!a || !finite_all(a, G)) BAD("generator arrays must be finite");
    if (!net->gen_bus || !uc->min_up || !uc->min_dn || !uc->u0 || !uc->hold) BAD("generator index arrays missing");
    for (int g = 0; g < G; g++) {
        if (net->gen_bus[g] < 0 || net->gen_bus[g] >= B) BAD("gen %d: bus out of range", g);
        if (net->gen_pmin[g] > net->gen_pmax[g]) BAD("gen %d: pmin > pmax", g);
        if (net->gen_qmin[g] > net->gen_qmax[g]) BAD("gen %d: qmin > qmax", g);
        if (co->c2[g] < 0) BAD("gen %d: c2 < 0", g);
        if (uc->min_up[g] < 1 || uc->min_up[g] > T || uc->min_dn[g] < 1 || uc->min_dn[g] > T)
            BAD("gen %d: min up/down must be in [1, T] (R15)", g);
        if (uc->u0[g] != 0 && uc->u0[g] != 1) BAD("gen %d: u0 must be 0/1", g);
        if (uc->hold[g] < 0 || uc->hold[g] > T) BAD("gen %d: hold must be in [0, T]", g);
    }
    if (uc->u_init)
        for (size_t k = 0; k < (size_t)G * T; k++)
            if (uc->u_init[k] != 0 && uc->u_init[k] != 1) BAD("u_init must be 0/1");
    if (p->tron_maxit < 1 || p->al_maxit < 1 || p->inner_min < 0 || p->inner_cap < 1) BAD("bad iteration caps");
    if (p->diverge_window < 0 || p->diverge_window >= HIST_CAP || (p->diverge_window > 0 && !std::isfinite(p->diverge_factor)))
        BAD("diverge_window must be in [0, %d) with a finite diverge_factor", HIST_CAP);
    return UCAC_OK;
#undef BAD
}

static ucac_status build_graphs(ucac_ctx *ctx);

// The side streams and fork/join events of destroyed contexts, kept for the next ucac_create on
// the same device (creating them took ~0.17 ms of every create; the e2e path creates per call).
struct StreamSet {
    int dev;
    cudaStream_t s2, s3;
    cudaEvent_t ev[7];
};
static std::mutex g_ss_mu;
static std::vector<StreamSet> g_ss_free;
static bool stream_set_get(ucac_ctx *ctx) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    std::lock_guard<std::mutex> lk(g_ss_mu);
    for (size_t i = 0; i < g_ss_free.size(); i++) {
        if (g_ss_free[i].dev != dev) continue;
        const StreamSet q = g_ss_free[i];
        g_ss_free.erase(g_ss_free.begin() + i);
        ctx->s2 = q.s2; ctx->s3 = q.s3;
        ctx->ev_fork = q.ev[0]; ctx->ev_join = q.ev[1]; ctx->ev_genx = q.ev[2]; ctx->ev_early = q.ev[3];
        ctx->ev_branch = q.ev[4]; ctx->ev_tail = q.ev[5]; ctx->ev_bus = q.ev[6];
        return true;
    }
    return false;
}
static void stream_set_put(ucac_ctx *ctx) {
    const cudaEvent_t ev[7] = {ctx->ev_fork, ctx->ev_join, ctx->ev_genx, ctx->ev_early, ctx->ev_branch, ctx->ev_tail, ctx->ev_bus};
    if (!ctx->s2 || !ctx->s3) return;
    for (auto e : ev)
        if (!e) return;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaStreamSynchronize(ctx->s2) != cudaSuccess ||
        cudaStreamSynchronize(ctx->s3) != cudaSuccess)
        return;
    StreamSet q{dev, ctx->s2, ctx->s3, {}};
    for (int i = 0; i < 7; i++) q.ev[i] = ev[i];
    {
        std::lock_guard<std::mutex> lk(g_ss_mu);
        if (g_ss_free.size() >= 16) return;   // (then ucac_destroy destroys them)
        g_ss_free.push_back(q);
    }
    ctx->s2 = ctx->s3 = nullptr;
    ctx->ev_fork = ctx->ev_join = ctx->ev_genx = ctx->ev_early = ctx->ev_branch = ctx->ev_tail = ctx->ev_bus = nullptr;
}

extern "C" ucac_status ucac_nccl_unique_id(unsigned char *id) {
    if (!id) return UCAC_EINVAL;
    ncclUniqueId u;
    ncclResult_t r = ncclGetUniqueId(&u);
    if (r != ncclSuccess) {
        g_create_err = ncclGetErrorString(r);
        return UCAC_ENCCL;
    }
    static_assert(sizeof(ncclUniqueId) <= 128, "ncclUniqueId size");
    memcpy(id, &u, sizeof(u));
    return UCAC_OK;
}

extern "C" ucac_status ucac_create(const ucac_network *net, const ucac_horizon *hz, const ucac_costs *co,
                                   const ucac_uc *uc, const ucac_params *prm, const ucac_dist *dist,
                                   void *cuda_stream, ucac_ctx **out) {
    UCAC_NVTX("ucac_create");
    if (!out) return fail(nullptr, UCAC_EINVAL, "out is NULL");
    *out = nullptr;
    // UCAC_CREATE_TRACE=1: phase times of ucac_create on stderr (diagnostics)
    static const bool trace = getenv("UCAC_CREATE_TRACE") != nullptr;
    auto tp0 = std::chrono::steady_clock::now(), tpl = tp0;
    auto mark = [&](const char *what) {
        nvtxMarkA(what);   // (phase boundaries on the NVTX timeline)
        if (!trace) return;
        auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "ucac_create %-12s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - tpl).count());
        tpl = now;
    };
    const bool stage_scan = !dist || dist->nranks == 1;   // demand finiteness checked while staging it
    ucac_status vs = validate(net, hz, co, uc, prm, !stage_scan);
    mark("validate");
    if (vs != UCAC_OK) return vs;
    const int nranks = dist ? dist->nranks : 1;
    const int rank = dist ? dist->rank : 0;
    if (nranks < 1 || rank < 0 || rank >= nranks || nranks > net->nbus)
        return fail(nullptr, UCAC_EINVAL, "bad rank %d / nranks %d", rank, nranks);
    if (dist && nranks > 1 && dist->comm_mode != 0 && dist->comm_mode != 1)
        return fail(nullptr, UCAC_EINVAL, "comm_mode must be 0 (NCCL) or 1 (loopback group)");
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(nullptr, UCAC_ECUDA, "no CUDA device: %s", cudaGetErrorString(e));
    int cc_major = 0, cc_minor = 0;
    e = cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (e != cudaSuccess) return fail(nullptr, UCAC_ECUDA, "%s", cudaGetErrorString(e));
    if (cc_major != 10) return fail(nullptr, UCAC_ECUDA, "libucac is built for sm_100a; device is sm_%d%d", cc_major, cc_minor);

    // (a one-rank time cut is allowed: it runs the time-cut graph with local exchanges, for tests)
    const int tcut = dist ? (dist->cut != 0) : 0;
    // UCAC_NCCL_ONE_RANK=1 (tests): a one-rank bus-cut dist with comm_mode 0 still builds an NCCL
    // communicator (of one rank) and runs the multi-rank iteration graph with its captured
    // collectives, so that the NCCL path executes on a one-GPU box
    const char *one_env = getenv("UCAC_NCCL_ONE_RANK");
    const bool nccl1 = dist && nranks == 1 && dist->comm_mode == 0 && one_env && atoi(one_env) == 1;
    if (dist && dist->cut != 0 && dist->cut != 1) return fail(nullptr, UCAC_EINVAL, "cut must be 0 or 1");
    if (tcut && nranks > hz->T) return fail(nullptr, UCAC_EINVAL, "time cut: T=%d < nranks=%d", hz->T, nranks);
    if (tcut && (prm->variant & (4 | 16)))
        return fail(nullptr, UCAC_EUNSUPPORTED, "time cut: variant bits 4 (ramp-aware DP) and 16 (literal Eq. 5f) are not supported");
    std::vector<int32_t> part;
    if (nranks > 1 && !tcut) {
        part.assign(net->nbus, 0);
        if (dist->bus_part) {
            for (int i = 0; i < net->nbus; i++) {
                if (dist->bus_part[i] < 0 || dist->bus_part[i] >= nranks) return fail(nullptr, UCAC_EINVAL, "bus_part out of range");
                part[i] = dist->bus_part[i];
            }
        } else if (partition_buses(net->nbus, net->nbranch, net->br_from, net->br_to, dist->bus_xy, nranks, part.data(),
                                   dist->branch_w)) {
            return fail(nullptr, UCAC_EINVAL, "partitioner failed");
        }
        // every rank checks every part (the partition is global and deterministic), so a part
        // without generators or branches fails on all ranks together, before any of them enters
        // ncclCommInitRank and waits there for the others
        std::vector<int> ng(nranks, 0), nl(nranks, 0);
        for (int g = 0; g < net->ngen; g++) ng[part[net->gen_bus[g]]]++;
        for (int l = 0; l < net->nbranch; l++) nl[part[net->br_from[l]]]++;
        for (int r = 0; r < nranks; r++)
            if (ng[r] == 0 || nl[r] == 0)
                return fail(nullptr, UCAC_EUNSUPPORTED, "part %d owns no generator or no branch; use fewer ranks", r);
    }
    ucac_ctx *ctx = new ucac_ctx();
    ctx->prm = *prm;
    ctx->nranks = nranks;
    ctx->rank = rank;
    ctx->comm_mode = dist && nranks > 1 ? dist->comm_mode : 0;
    ctx->multi = nranks > 1 || nccl1;
    mark("device/part");
    if (tcut) {
        std::vector<int32_t> one(net->nbus, 0);
        ctx->P = localize_periods(build_local(net, hz, co, uc, one.data(), 1, 0), hz, uc, nranks, rank);
    } else {
        ctx->P = build_local(net, hz, co, uc, part.data(), nranks, rank);
        ctx->P.Tg = ctx->P.T;
        ctx->P.own1 = ctx->P.T;
        ctx->P.Tmax = ctx->P.T;
        ctx->P.tstart = {0, ctx->P.T};
    }
    mark("build_local");
    Local &P = ctx->P;
    const int B = P.B, G = P.G, L = P.L, T = P.T;
    ctx->B = P.Bo;
    ctx->G = G;
    ctx->L = L;
    ctx->T = T;
    // the 16-iteration graph amortises launch latency where an iteration is short; a large case
    // (an iteration of ~0.1 ms) runs single-iteration graphs back to back and skips capturing and
    // instantiating the long one in ucac_create
    if ((long long)L * T > UCAC_UNROLL_MAX_LT) ctx->gunroll[1] = 1;
    auto bail = [&](ucac_status s) {
        g_create_err = ctx->err;
        ucac_destroy(ctx);
        return s;
    };
    if (G == 0 || L == 0) return bail(fail(ctx, UCAC_EUNSUPPORTED, "rank %d owns no generator or no branch; use fewer ranks", rank));
    if (cuda_stream) {
        ctx->s = (cudaStream_t)cuda_stream;
    } else {
        if (cudaStreamCreateWithFlags(&ctx->s, cudaStreamNonBlocking) != cudaSuccess) return bail(fail(ctx, UCAC_ECUDA, "stream"));
        ctx->own_stream = true;
    }
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if (stream_set_get(ctx)) {
        // recycled from a destroyed context (stream_set_put)
    } else if (cudaStreamCreateWithPriority(&ctx->s2, cudaStreamNonBlocking, UCAC_S2_PRIO ? prio_hi : prio_lo) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->s3, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_genx, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_early, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_branch, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_tail, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_bus, cudaEventDisableTiming) != cudaSuccess)
        return bail(fail(ctx, UCAC_ECUDA, "stream/event creation failed"));
    mark("streams");
    if ((ctx->st_host = pinned_status_get()) == nullptr) return bail(fail(ctx, UCAC_ENOMEM, "pinned status"));
    mark("pinned");
    memset(ctx->st_host, 0, sizeof(DevStatus));
    if ((nranks > 1 && ctx->comm_mode == 0) || nccl1) {
        ncclUniqueId id;
        memcpy(&id, dist->nccl_id, sizeof(id));
        ncclResult_t r = ncclCommInitRank(&ctx->comm, nranks, id, rank);
        if (r != ncclSuccess) return bail(fail(ctx, UCAC_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r)));
        if (!tcut) {   // the early exchanges run on their own stream, so on their own communicator
            r = ncclCommSplit(ctx->comm, 0, rank, &ctx->comm2, nullptr);
            if (r != ncclSuccess) return bail(fail(ctx, UCAC_ENCCL, "ncclCommSplit: %s", ncclGetErrorString(r)));
        }
    }

    Dev &d = ctx->d;
    d.G = G; d.L = L; d.B = B; d.T = T;
    d.B_own = P.Bo;
    d.Lph = P.Lp;
    d.nranks = nranks;
    d.xrank_rec = (nranks > 1 || ctx->multi) ? 1 : 0;
    d.ncut = (int)P.cut_local.size();
    d.nexport = (int)P.export_local.size();
    d.nphantom_src = (int)P.phantom_src.size();
    d.nghost = B - P.Bo;
    d.max_cut = P.max_cut;
    d.max_export = P.max_export;
    d.ref_bus = P.ref;
    d.S = P.S;
    d.t_off = P.t_off;
    d.Tg = P.Tg;
    d.own0 = P.own0;
    d.own1 = P.own1;
    d.tcut = tcut;
    d.Tmax = P.Tmax;
    d.rank = rank;
    d.rpq = prm->rho_pq; d.rva = prm->rho_va; d.ruc = prm->rho_uc;
    d.irpq = 1.0 / prm->rho_pq; d.irva = 1.0 / prm->rho_va; d.iruc = 1.0 / prm->rho_uc;
    d.tau = prm->tau; d.theta = prm->theta; d.lambda_max = prm->lambda_max; d.beta_max = prm->beta_max;
    d.eps_inner_abs = prm->eps_inner_abs;
    d.inner_min = prm->inner_min; d.inner_cap = prm->inner_cap; d.outer_enabled = prm->outer_enabled;
    d.tron_gtol = prm->tron_gtol_rel * std::max(prm->rho_pq, prm->rho_va);
    d.tron_maxit = prm->tron_maxit; d.al_maxit = prm->al_maxit;
    d.al_eta_star = prm->al_eta_star; d.al_sigma0_rel = prm->al_sigma0_rel;
    d.al_sigma_max_rel = prm->al_sigma_max_rel; d.al_sigma_decay = prm->al_sigma_decay;
    d.uc_fixed = prm->uc_fixed;
    d.div_window = prm->diverge_window;
    d.div_factor = prm->diverge_factor;
    d.fuse_rows = (nranks == 1 && !nccl1 && UCAC_FUSE_ROWS) ? 1 : 0;
    d.variant = prm->variant;
    d.strict = prm->strict_fp != 0;
    d.nblk_bus = nblk_bus(P.Bo, T);
    d.nblk_ubar = nblk_ubar(G, T);
    d.nblk_rows = nblk_rows(L, T);

    const size_t GT = (size_t)G * T, LT = (size_t)L * T, BT = (size_t)B * T;
    // One device arena for every array of the context: the uploaded inputs form
    // its prefix, staged contiguously on the host and sent with one copy; the rest is zeroed with
    // one memset.  A first pass over the same layout sizes it.
    int8_t *uinit = nullptr;
    uint64_t demand_bad = 0;   // inf/NaN met while staging the demand (single rank)
    auto layout = [&](Arena &A) {
        d.gbus = A.put(P.gbus);
        d.tu = A.put(P.tu);
        d.td = A.put(P.td);
        d.u0 = A.put(P.u0);
        d.hold = A.put(P.hold);
        d.pmin = A.put(P.pmin);
        d.pmax = A.put(P.pmax);
        d.qmin = A.put(P.qmin);
        d.qmax = A.put(P.qmax);
        d.c2 = A.put(P.c2);
        d.c1 = A.put(P.c1);
        d.c0 = A.put(P.c0);
        d.csu = A.put(P.csu);
        d.csd = A.put(P.csd);
        d.rup = A.put(P.rup);
        d.rdn = A.put(P.rdn);
        d.sup = A.put(P.sup);
        d.sdn = A.put(P.sdn);
        d.p0 = A.put(P.p0);
        d.y = A.put(P.ysoa);
        d.rate = A.put(P.rate);
        d.bfrom = A.put(P.from);
        d.bto = A.put(P.to);
        d.gs = A.put(P.gs);
        d.bs = A.put(P.bs);
        d.vmin = A.put(P.vmin);
        d.vmax = A.put(P.vmax);
        // demand [bus][local period], owned buses (ghost rows 0), transposed from the caller's
        // [period][bus] arrays straight into the staging image (reads in input order)
        // (single rank: every value passes here, and an exponent of all ones flags inf/NaN, the
        // finiteness check validate() leaves to this pass)
        auto demand = [&](const double *src) {
            return [&, src](double *dst) {
                const uint64_t E = 0x7ff0000000000000ull;
                uint64_t bad = 0;
                for (int a = P.Bo; a < P.B; a++)
                    for (int t = 0; t < T; t++) dst[(size_t)a * T + t] = 0.0;
                // blocks of 64 buses: the transposed writes of a block stay in a few KB of cache
                for (int a0 = 0; a0 < P.Bo; a0 += 64) {
                    const int a1 = std::min(P.Bo, a0 + 64);
                    for (int t = 0; t < T; t++)
                        for (int a = a0; a < a1; a++) {
                            const double v = src[(size_t)(P.t_off + t) * net->nbus + P.bus_global[a]];
                            uint64_t b;
                            memcpy(&b, &v, sizeof b);
                            bad |= (uint64_t)((b & E) == E);
                            dst[(size_t)a * T + t] = v;
                        }
                }
                demand_bad |= bad;
            };
        };
        d.pd = A.put_fill<double>((size_t)B * T, demand(hz->pd));
        d.qd = A.put_fill<double>((size_t)B * T, demand(hz->qd));
        d.bg_ptr = A.put(P.bgp);
        d.bg_idx = A.put(P.bgi);
        d.be_ptr = A.put(P.bep);
        d.be_idx = A.put(P.bei);
        d.cut_local = A.put(P.cut_local);
        d.export_local = A.put(P.export_local);
        d.phantom_src = A.put(P.phantom_src);
        d.ghost_src = A.put(P.ghost_src);
        d.tc_t0 = A.put(P.tstart);
        d.phantom_bus = A.put(P.phantom_bus);
        d.ghost_eptr = A.put(P.gep);
        d.ghost_eidx = A.put(P.gei);
        uinit = P.uinit.empty() ? nullptr : A.put(P.uinit);
        A.up_end = A.off;
        // iterate (zeroed, then set by launch_init)
        d.u = A.take<int8_t>(GT);
        d.p = A.take<double>(GT);
        d.q = A.take<double>(GT);
        d.ph = A.take<double>(GT);
        d.ub_on = A.take<double>(GT);
        d.ub_su = A.take<double>(GT);
        d.ub_sd = A.take<double>(GT);
        d.pbar = A.take<double>(GT);
        d.qbar = A.take<double>(GT);
        d.zg = A.take<double>(NGROW * GT);
        d.yg = A.take<double>(NGROW * GT);
        d.lg = A.take<double>(NGROW * GT);
        d.x = A.take<double>(4 * LT);
        d.f = A.take<double>(4 * LT);
        d.fbar = A.take<double>(4 * LT);
        d.al = A.take<double>(3 * LT);
        d.zb = A.take<double>(NBROW * LT);
        d.yb = A.take<double>(NBROW * LT);
        d.lb = A.take<double>(NBROW * LT);
        d.wbar = A.take<double>(BT);
        d.thbar = A.take<double>(BT);
        d.part_bus = A.take<double>((size_t)d.nblk_bus * NPART);
        d.part_ubar = A.take<double>((size_t)d.nblk_ubar * NPART);
        d.part_rows = A.take<double>((size_t)d.nblk_rows * NPART);
        d.nblk_lbus = nblk_lbus(P.Bo * T);
        d.nblk_lrows = nblk_lrows(L * T);
        d.part_lbus = A.take<double>((size_t)d.nblk_lbus * NPART);
        d.part_lrows = A.take<double>((size_t)d.nblk_lrows * NPART);
        d.lbus = A.take<int>((size_t)d.nblk_bus * 128);          // BUS_THREADS items per k_bus block
        d.lbus_cnt = A.take<unsigned>((size_t)d.nblk_bus);
        d.lrow = A.take<int>((size_t)d.nblk_rows * 2 * 128);     // 2 ROWS_THREADS items per k_rows block
        d.lrow_cnt = A.take<unsigned>((size_t)d.nblk_rows);
        d.part_efold = A.take<double>((size_t)fold_blocks() * NPART);
        d.rec_part = A.take<double>(3 * NPART);
        d.kdone = A.take<unsigned>(3);
        d.bmark = A.take<unsigned>(BT);
        d.tauh = A.take<double>((size_t)NBROW * (L + P.Lp) * T);
        d.bmu = A.take<double>(4 * BT);
        d.cnt = A.take<unsigned long long>(NCNT);
        d.alq = A.take<int>((size_t)UCAC_AL_BUCKETS * LT);
        d.alq_cnt = A.take<unsigned>(UCAC_AL_BUCKETS + 1);
        d.alq_x = A.take<double>(4 * LT);
        d.alits = A.take<uint8_t>(LT);
        d.u_next = A.take<int8_t>(GT);
        d.unext_ok = A.take<unsigned>(1);
        d.rec = A.take<double>(NREC);
        d.hist = A.take<double>((size_t)HIST_CAP * HIST_FIELDS);
        d.tl = A.take<unsigned long long>(2 * NKERN);
        // bus cut: early exchanges carry a late flag (5 and 7 values), late ones the plain values (4, 6)
        d.xsend1 = A.take<double>((size_t)P.max_cut * 5 * T);
        d.xrecv1 = A.take<double>((size_t)nranks * P.max_cut * 5 * T);
        d.xsend2 = A.take<double>((size_t)P.max_export * 7 * T);
        d.xrecv2 = A.take<double>((size_t)nranks * P.max_export * 7 * T);
        d.xsend3 = A.take<double>((size_t)P.max_cut * 4 * T);
        d.xrecv3 = A.take<double>((size_t)nranks * P.max_cut * 4 * T);
        d.xsend4 = A.take<double>((size_t)P.max_export * 6 * T);
        d.xrecv4 = A.take<double>((size_t)nranks * P.max_export * 6 * T);
        d.qmark = A.take<unsigned>((size_t)(L + P.Lp) * T);
        d.st = A.take<DevStatus>(1);
        if (tcut) {   // (the receive buffers live in ctx->xbuf, a plain cudaMalloc block peers can map)
            d.tc_stage_send = A.take<double>((size_t)G * P.Tmax * 4);
            d.tc2_send = A.take<double>((size_t)G * 2);
            d.tc3_send = A.take<double>((size_t)G * 12);
            d.xarrive = A.take<unsigned>(3);
        }
        d.rmark[0] = A.take<unsigned>((size_t)(L + P.Lp) * T);
        d.rmark[1] = A.take<unsigned>((size_t)(L + P.Lp) * T);
        ctx->xpose = A.take<double>(4 * LT);
    };
    {
        mark("setup");
        Arena sizing;
        layout(sizing);
        void *base = nullptr;
        // stream-ordered from the device's default pool, whose release threshold is raised once:
        // a context created after another was destroyed reuses its pages instead of mapping new
        // ones (create/destroy cycles of the public API, the e2e path)
        static const bool pool_ready = [] {
            int dv = 0;
            cudaMemPool_t pool;
            if (cudaGetDevice(&dv) != cudaSuccess || cudaDeviceGetDefaultMemPool(&pool, dv) != cudaSuccess) return false;
            unsigned long long keep = ~0ull;
            return cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep) == cudaSuccess;
        }();
        (void)pool_ready;
        e = cudaMallocAsync(&base, sizing.off, ctx->s);
        if (e != cudaSuccess) return bail(fail(ctx, UCAC_ENOMEM, "cudaMalloc arena of %zu B", sizing.off));
        ctx->dalloc.push_back(base);
        std::lock_guard<std::mutex> lk(g_stage_mu);
        std::vector<char> pageable;   // if no page-locked memory can be had
        char *stage = stage_get(sizing.up_end);
        if (!stage) {
            pageable.assign(sizing.up_end, 0);
            stage = pageable.data();
        }
        Arena A;
        A.base = (uintptr_t)base;
        A.stage = stage;
        layout(A);
        if (stage_scan && demand_bad) return bail(fail(ctx, UCAC_EINVAL, "demand must be finite"));
        if (cudaMemcpyAsync(base, stage, A.up_end, cudaMemcpyHostToDevice, ctx->s) != cudaSuccess ||
            cudaMemsetAsync((char *)base + A.up_end, 0, A.off - A.up_end, ctx->s) != cudaSuccess)
            return bail(fail(ctx, UCAC_ECUDA, "arena upload"));
        // the staging image is reused by the next create: it waits for this event (stage_get);
        // without the event (or with a page-able image), the copy is waited for here
        if (!g_stage_ev && cudaEventCreateWithFlags(&g_stage_ev, cudaEventDisableTiming) != cudaSuccess) g_stage_ev = nullptr;
        if (stage == g_stage && g_stage_ev && cudaEventRecord(g_stage_ev, ctx->s) == cudaSuccess) {
            g_stage_ev_pending = true;
        } else if (cudaStreamSynchronize(ctx->s) != cudaSuccess) {
            return bail(fail(ctx, UCAC_ECUDA, "arena upload"));
        }
    }
    if (tcut) {
        // receive buffers and arrival flags of the time cut's exchanges, one cudaMalloc block (not
        // the pool arena) so a device-initiated exchange can map it from other processes (CUDA IPC)
        const size_t a0 = 0, a1 = a0 + (size_t)nranks * G * P.Tmax * 4 * 8, a2 = a1 + (size_t)nranks * G * 2 * 8,
                     a3 = a2 + (size_t)nranks * G * 12 * 8, a4 = a3 + 3 * UCAC_MAX_P2P * 8;
        if (cudaMalloc(&ctx->xbuf, a4) != cudaSuccess) return bail(fail(ctx, UCAC_ENOMEM, "exchange buffers"));
        if (cudaMemset(ctx->xbuf, 0, a4) != cudaSuccess) return bail(fail(ctx, UCAC_ECUDA, "exchange buffers"));
        char *xb = (char *)ctx->xbuf;
        d.tc_stage_recv = (double *)(xb + a0);
        d.tc2_recv = (double *)(xb + a1);
        d.tc3_recv = (double *)(xb + a2);
        d.xflags = (unsigned long long *)(xb + a3);
        ctx->xoff[0] = a0; ctx->xoff[1] = a1; ctx->xoff[2] = a2; ctx->xoff[3] = a3;
        ctx->xbytes = a4;
    }
    // status: beta = beta0, k = 1 (R21)
    DevStatus st0{};
    st0.beta = prm->beta0;
    st0.outer_k = 1;
    *ctx->st_host = st0;
    if (cudaMemcpyAsync(d.st, ctx->st_host, sizeof(DevStatus), cudaMemcpyHostToDevice, ctx->s) != cudaSuccess)
        return bail(fail(ctx, UCAC_ECUDA, "status upload"));
    if (gen_set_smem_attr(P.Tg) != cudaSuccess) return bail(fail(ctx, UCAC_ECUDA, "T=%d needs %zu B of shared memory", P.Tg, gen_smem_bytes(P.Tg)));
    mark("arena");
    // an empty record history: all-ones bytes are NaN doubles, which the detector's test rejects
    if (cudaMemsetAsync(d.hist, 0xFF, (size_t)HIST_CAP * HIST_FIELDS * sizeof(double), ctx->s) != cudaSuccess)
        return bail(fail(ctx, UCAC_ECUDA, "history"));
    launch_init(d, uinit, ctx->s);
    e = cudaGetLastError();
    if (e != cudaSuccess) return bail(fail(ctx, UCAC_ECUDA, "init kernel: %s", cudaGetErrorString(e)));
    mark("init");
    // the graphs are captured while the upload, the memset and the init kernel run (capture
    // records only the work enqueued after it begins), then the stream is waited for once
    if (!(nranks > 1 && ctx->comm_mode == 1)) {
        ucac_status gs = build_graphs(ctx);
        if (gs != UCAC_OK) {
            cudaStreamSynchronize(ctx->s);
            return bail(gs);
        }
    }
    mark("graphs");
    e = cudaStreamSynchronize(ctx->s);
    if (e != cudaSuccess) return bail(fail(ctx, UCAC_ECUDA, "init: %s", cudaGetErrorString(e)));
    mark("sync");
    *out = ctx;
    return UCAC_OK;
#undef ALLOC
#undef UPLOAD
}

// ------------------------------------------------------------------------------------------
// one inner iteration.  Dependency order (also the order of the eager, timed path):
//   (7a) k_gen -> (7b) k_genx, k_branch -> (7d) k_bus, k_rows [early] -> (7b) k_branch_al
//   -> (7c) k_ubar -> k_late [(7d) late bus + rows, S8/S9].
// The fast-path branch kernel marks the bus-periods touched by a thermal-AL solve; the bus
// solve and row update of everything else only need the fast path and the generator x-update
// (early phase), the marked ones wait for the AL tail (late phase).  In the single-GPU graph:
//   s : k_branch ---------------------------> k_branch_al --------> [join] k_late
//   s2:           k_gen -> k_genx -> k_ubar ---------------------------^
//   s3:                      `-> k_bus/k_rows early -------------------^
// i.e. the early sweep (~90 % of the bus/row work) and the generator chain (which never reads a
// branch result) run in the shadow of the latency-bound AL tail.  The generator chain forks AFTER
// the register-bound fast path (sharing the SMs with it halves its occupancy).  Several ranks
// add the halo exchange: the cut ends' tauhat before the bus solve, the bus results
// before the row update, the reduction record before the inner/outer decision; there both bus
// phases run after the tauhat exchange and both row phases after the bus exchange.
// ------------------------------------------------------------------------------------------
static const int kOrder[NKERN] = {K_GEN, K_GENX, K_BRANCH, K_BUS, K_ROWS, K_BRANCH_AL, K_UBAR, K_FOLD,
                                  K_BUS_LATE, K_ROWS_LATE};

static void launch_kernel(ucac_ctx *ctx, int k, cudaStream_t s) {
    switch (k) {
        case K_BRANCH: if (ctx->d.strict) launch_branch_strict(ctx->d, s); else launch_branch(ctx->d, s); break;
        case K_BRANCH_AL: launch_branch_al(ctx->d, s); break;
        case K_GEN: launch_gen(ctx->d, s); break;
        case K_GENX: launch_genx(ctx->d, s); break;
        case K_BUS: launch_bus(ctx->d, s); break;
        case K_ROWS: if (!ctx->d.fuse_rows) launch_rows(ctx->d, s); break;   // fused: inside k_bus
        case K_BUS_LATE: launch_bus_late(ctx->d, s); break;
        case K_ROWS_LATE: if (!ctx->d.fuse_rows) launch_rows_late(ctx->d, s, 1); break;
        case K_FOLD: launch_fold_early(ctx->d, s); break;
        case K_UBAR: launch_ubar(ctx->d, s); break;
        default: break;
    }
}

// NCCL return codes of the captured collectives: the first failure is kept and reported by build_graphs
#define NC(call)                                                              \
    do {                                                                      \
        ncclResult_t r_ = (call);                                             \
        if (r_ != ncclSuccess && ctx->nccl_err == ncclSuccess) ctx->nccl_err = r_; \
    } while (0)

// NEXT-4(c) time cut, one rank per GPU.  The single-GPU graph's three streams with
// the exchanges inserted where their data are final:
//   s : k_branch ------------------------> k_branch_al -> [bus list] k_bus_late -> [fold] k_rows_late
//         -> pack 3 -> exchange 3 -> unpack 3 -> S8 all-reduce -> finalize
//   s2:   stage costs -> exchange 1 -> DP -> k_genx -> pack 2 -> exchange 2 -> unpack 2 -> k_ubar
//   s3:   [k_branch, unpack 2] k_bus -> k_rows -> [k_ubar] k_fold_early
// so the early bus/row sweep and the generator chain run in the shadow of the AL tail, as on one GPU.
// The collectives are totally ordered by the graph's dependencies (1 and 2 on s2 after the iteration
// fork, 3 and the all-reduce on s after the early fold), so one communicator serves them all.
// d.p2p: the three exchanges are device-initiated stores into the peers' buffers (k_xchg.cu).
// One rank (tests): the stage costs are copied locally and the neighbour exchanges vanish.
static void enqueue_iteration_tc(ucac_ctx *ctx) {
    const Dev &d = ctx->d;
    const bool multi = ctx->multi;
    cudaStream_t s = ctx->s, s2 = ctx->s2, s3 = ctx->s3;
    cudaEventRecord(ctx->ev_fork, s);
    cudaStreamWaitEvent(s2, ctx->ev_fork, 0);
    launch_kernel(ctx, K_BRANCH, s);
    cudaEventRecord(ctx->ev_branch, s);
    // generator chain with exchanges 1 and 2
    launch_stage_tc(d, s2);
    const size_t n1 = (size_t)d.G * d.Tmax * 4;
    if (!multi) cudaMemcpyAsync(d.tc_stage_recv, d.tc_stage_send, n1 * sizeof(double), cudaMemcpyDeviceToDevice, s2);
    else if (d.p2p) launch_xchg(d, 1, s2);
    else NC(ncclAllGather(d.tc_stage_send, d.tc_stage_recv, n1, ncclDouble, ctx->comm, s2));
    launch_dp_tc(d, s2);
    launch_kernel(ctx, K_GENX, s2);
    if (multi) {
        launch_pack_tc2(d, s2);
        if (d.p2p) launch_xchg(d, 2, s2);
        else NC(ncclAllGather(d.tc2_send, d.tc2_recv, (size_t)d.G * 2, ncclDouble, ctx->comm, s2));
        launch_unpack_tc2(d, s2);
    }
    cudaEventRecord(ctx->ev_genx, s2);
    // early sweep
    cudaStreamWaitEvent(s3, ctx->ev_genx, 0);
    cudaStreamWaitEvent(s3, ctx->ev_branch, 0);
    launch_kernel(ctx, K_BUS, s3);
    cudaEventRecord(ctx->ev_bus, s3);
    launch_kernel(ctx, K_ROWS, s3);
    launch_kernel(ctx, K_UBAR, s2);
    cudaEventRecord(ctx->ev_join, s2);
    cudaStreamWaitEvent(s3, ctx->ev_join, 0);
    launch_kernel(ctx, K_FOLD, s3);
    cudaEventRecord(ctx->ev_early, s3);
    // AL tail, late sweep
    launch_kernel(ctx, K_BRANCH_AL, s);
    cudaStreamWaitEvent(s, ctx->ev_genx, 0);
    cudaStreamWaitEvent(s, ctx->ev_bus, 0);
    launch_kernel(ctx, K_BUS_LATE, s);
    cudaStreamWaitEvent(s, ctx->ev_early, 0);
    launch_kernel(ctx, K_ROWS_LATE, s);
    if (!multi) return;   // one rank: k_rows_late's final fold applied S8/S9 itself
    launch_pack_tc3(d, s);
    if (d.p2p) launch_xchg(d, 3, s);
    else NC(ncclAllGather(d.tc3_send, d.tc3_recv, (size_t)d.G * 12, ncclDouble, ctx->comm, s));
    launch_unpack_tc3(d, s);
    NC(ncclGroupStart());
    NC(ncclAllReduce(d.rec, d.rec, NREC_SUM, ncclDouble, ncclSum, ctx->comm, s));
    NC(ncclAllReduce(d.rec + NREC_SUM, d.rec + NREC_SUM, NREC - NREC_SUM, ncclDouble, ncclMax, ctx->comm, s));
    NC(ncclGroupEnd());
    launch_finalize(d, s);
}

// Bus cut over NCCL ranks: the single-GPU overlap kept across ranks.  The early
// exchanges (cut ends' tauhat with a "queued" flag, then early bus results with a "late" flag) run
// on s3 on their own communicator, so the interior buses and rows proceed during the AL tail; the
// late ones (final tauhat of the queued cut ends, late bus results) and the S8 all-reduce on s.
//   s : k_branch ----------------> k_branch_al -> tau late -> [bus list] k_bus_late -> bus late
//         -> [early fold] k_rows_late -> all-reduce -> finalize
//   s2:   k_gen -> k_genx -> k_ubar
//   s3:   [k_branch, k_genx] tau early -> k_bus -> bus early -> k_rows -> [k_ubar] k_fold_early
static void enqueue_iteration_bus_multi(ucac_ctx *ctx) {
    const Dev &d = ctx->d;
    cudaStream_t s = ctx->s, s2 = ctx->s2, s3 = ctx->s3;
    const size_t T = d.T;
    cudaEventRecord(ctx->ev_fork, s);
    cudaStreamWaitEvent(s2, ctx->ev_fork, 0);
    launch_kernel(ctx, K_BRANCH, s);
    cudaEventRecord(ctx->ev_branch, s);
    launch_kernel(ctx, K_GEN, s2);
    launch_kernel(ctx, K_GENX, s2);
    cudaEventRecord(ctx->ev_genx, s2);
    launch_kernel(ctx, K_UBAR, s2);
    cudaEventRecord(ctx->ev_join, s2);
    // early sweep with the early exchanges
    cudaStreamWaitEvent(s3, ctx->ev_branch, 0);
    cudaStreamWaitEvent(s3, ctx->ev_genx, 0);
    if (d.max_cut > 0) {
        launch_pack_tau_early(d, s3);
        NC(ncclAllGather(d.xsend1, d.xrecv1, (size_t)d.max_cut * 5 * T, ncclDouble, ctx->comm2, s3));
        launch_unpack_tau_early(d, s3);
    }
    launch_kernel(ctx, K_BUS, s3);
    cudaEventRecord(ctx->ev_bus, s3);
    if (d.max_export > 0) {
        launch_pack_bus_early(d, s3);
        NC(ncclAllGather(d.xsend2, d.xrecv2, (size_t)d.max_export * 7 * T, ncclDouble, ctx->comm2, s3));
        launch_unpack_bus_early(d, s3);
    }
    launch_kernel(ctx, K_ROWS, s3);
    cudaStreamWaitEvent(s3, ctx->ev_join, 0);
    launch_kernel(ctx, K_FOLD, s3);
    cudaEventRecord(ctx->ev_early, s3);
    // AL tail, late exchanges, late sweep
    launch_kernel(ctx, K_BRANCH_AL, s);
    if (d.max_cut > 0) launch_pack_tau(d, s);
    cudaStreamWaitEvent(s, ctx->ev_bus, 0);   // the early unpack's queued flags, the bus lists
    if (d.max_cut > 0) {
        NC(ncclAllGather(d.xsend3, d.xrecv3, (size_t)d.max_cut * 4 * T, ncclDouble, ctx->comm, s));
        launch_unpack_tau(d, s);
    }
    launch_kernel(ctx, K_BUS_LATE, s);
    if (d.max_export > 0) launch_pack_bus(d, s);
    cudaStreamWaitEvent(s, ctx->ev_early, 0);   // the early ghost flags, the early rows and fold
    if (d.max_export > 0) {
        NC(ncclAllGather(d.xsend4, d.xrecv4, (size_t)d.max_export * 6 * T, ncclDouble, ctx->comm, s));
        launch_unpack_bus(d, s);
    }
    launch_kernel(ctx, K_ROWS_LATE, s);
    NC(ncclGroupStart());
    NC(ncclAllReduce(d.rec, d.rec, NREC_SUM, ncclDouble, ncclSum, ctx->comm, s));
    NC(ncclAllReduce(d.rec + NREC_SUM, d.rec + NREC_SUM, NREC - NREC_SUM, ncclDouble, ncclMax, ctx->comm, s));
    NC(ncclGroupEnd());
    launch_finalize(d, s);
}

static void enqueue_iteration(ucac_ctx *ctx) {
    if (ctx->d.tcut) {
        enqueue_iteration_tc(ctx);
        return;
    }
    if (ctx->multi) {
        enqueue_iteration_bus_multi(ctx);
        return;
    }
    const Dev &d = ctx->d;
    const bool multi = ctx->nranks > 1;
    const bool early_fork = !multi && UCAC_EARLY_FORK;
    if (early_fork) {
        // the generator chain (7a, 7b gens, 7c) reads only the previous iterate: it runs beside the
        // branch fast path at high launch priority, in the SM slots k_branch's grid leaves free
        //
        // (enqueuing the chain before k_branch, or a larger shared-memory carveout for k_branch
        // so k_gen co-resides from the start, measured slower: k_branch is throughput-bound)
        cudaEventRecord(ctx->ev_fork, ctx->s);
        cudaStreamWaitEvent(ctx->s2, ctx->ev_fork, 0);
        launch_kernel(ctx, K_BRANCH, ctx->s);
        cudaEventRecord(ctx->ev_branch, ctx->s);
        launch_kernel(ctx, K_GEN, ctx->s2);
        launch_kernel(ctx, K_GENX, ctx->s2);
    } else {
        launch_kernel(ctx, K_BRANCH, ctx->s);
        cudaEventRecord(ctx->ev_fork, ctx->s);
        cudaStreamWaitEvent(ctx->s2, ctx->ev_fork, 0);
        launch_kernel(ctx, K_GEN, ctx->s2);
        launch_kernel(ctx, K_GENX, ctx->s2);
    }
    if (!multi) {
        cudaEventRecord(ctx->ev_genx, ctx->s2);
        cudaStreamWaitEvent(ctx->s3, ctx->ev_genx, 0);
        if (early_fork) cudaStreamWaitEvent(ctx->s3, ctx->ev_branch, 0);
        launch_kernel(ctx, K_BUS, ctx->s3);
        cudaEventRecord(ctx->ev_bus, ctx->s3);   // k_bus_late reads the bus lists k_bus compacts
        launch_kernel(ctx, K_ROWS, ctx->s3);
    }
    // k_ubar is off the critical path (it only has to finish before the early fold): after
    // k_bus it no longer competes with it for SMs (UCAC_UBAR_AFTER_BUS)
    if (!multi && UCAC_UBAR_AFTER_BUS) cudaStreamWaitEvent(ctx->s2, ctx->ev_bus, 0);
    launch_kernel(ctx, K_UBAR, ctx->s2);
    cudaEventRecord(ctx->ev_join, ctx->s2);
    if (early_fork && UCAC_PIPE_DP) {
        // the next iteration's (7a) DP, overlapping the rest of this one (k_gen tail launch)
        launch_gen(d, ctx->s2, 1);
        cudaEventRecord(ctx->ev_tail, ctx->s2);
    }
    if (!multi) {   // fold the early partials in the shadow of the AL tail
        cudaStreamWaitEvent(ctx->s3, ctx->ev_join, 0);
        launch_kernel(ctx, K_FOLD, ctx->s3);
        cudaEventRecord(ctx->ev_early, ctx->s3);
    }
    launch_kernel(ctx, K_BRANCH_AL, ctx->s);
    if (multi && d.max_cut > 0) {
        launch_pack_tau(d, ctx->s);
        NC(ncclAllGather(d.xsend1, d.xrecv1, (size_t)d.max_cut * 4 * d.T, ncclDouble, ctx->comm, ctx->s));
        launch_unpack_tau(d, ctx->s);
    }
    if (!multi) {
        // the late bus solve needs the AL results and the generator x-update only (not k_ubar);
        // the late rows' final fold needs every early partial (k_fold_early, after k_ubar)
        cudaStreamWaitEvent(ctx->s, ctx->ev_genx, 0);
        // fused rows: k_bus_late does the final fold, so it needs the folded early partials
        if (d.fuse_rows) cudaStreamWaitEvent(ctx->s, ctx->ev_early, 0);
        cudaStreamWaitEvent(ctx->s, ctx->ev_bus, 0);
        launch_kernel(ctx, K_BUS_LATE, ctx->s);
        cudaStreamWaitEvent(ctx->s, ctx->ev_early, 0);
        launch_kernel(ctx, K_ROWS_LATE, ctx->s);
        if (early_fork && UCAC_PIPE_DP) cudaStreamWaitEvent(ctx->s, ctx->ev_tail, 0);
        return;
    }
    cudaStreamWaitEvent(ctx->s, ctx->ev_join, 0);
    launch_kernel(ctx, K_BUS, ctx->s);
    launch_kernel(ctx, K_BUS_LATE, ctx->s);
    if (d.max_export > 0) {
        launch_pack_bus(d, ctx->s);
        NC(ncclAllGather(d.xsend2, d.xrecv2, (size_t)d.max_export * 6 * d.T, ncclDouble, ctx->comm, ctx->s));
        launch_unpack_bus(d, ctx->s);
    }
    launch_kernel(ctx, K_ROWS, ctx->s);
    launch_kernel(ctx, K_FOLD, ctx->s);
    launch_kernel(ctx, K_ROWS_LATE, ctx->s);
    NC(ncclGroupStart());
    NC(ncclAllReduce(d.rec, d.rec, NREC_SUM, ncclDouble, ncclSum, ctx->comm, ctx->s));
    NC(ncclAllReduce(d.rec + NREC_SUM, d.rec + NREC_SUM, NREC - NREC_SUM, ncclDouble, ncclMax, ctx->comm, ctx->s));
    NC(ncclGroupEnd());
    launch_finalize(d, ctx->s);
}

// Instantiated single-iteration graphs of destroyed single-rank contexts: the next ucac_create
// captures its own graph and, where the topology is the same (same kernels, same edges), loads it
// into one of these with cudaGraphExecUpdate (new kernel parameters and grids) instead of
// instantiating anew.  A pooled graph is never launched before that update.
static std::mutex g_exec_mu;
static std::vector<std::pair<int, cudaGraphExec_t>> g_exec_free;   // (device, graph)
static cudaGraphExec_t exec_pool_get() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lk(g_exec_mu);
    for (size_t i = 0; i < g_exec_free.size(); i++)
        if (g_exec_free[i].first == dev) {
            cudaGraphExec_t x = g_exec_free[i].second;
            g_exec_free.erase(g_exec_free.begin() + i);
            return x;
        }
    return nullptr;
}
static bool exec_pool_put(cudaGraphExec_t x) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    std::lock_guard<std::mutex> lk(g_exec_mu);
    if (g_exec_free.size() >= 4) return false;
    g_exec_free.emplace_back(dev, x);
    return true;
}

static ucac_status build_graphs(ucac_ctx *ctx) {
    for (int gi = 0; gi < 2; gi++) {
        if (gi == 1 && ctx->gunroll[1] == 1) break;   // single-iteration graphs only
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(ctx->s, cudaStreamCaptureModeThreadLocal));
        ctx->nccl_err = ncclSuccess;
        for (int k = 0; k < ctx->gunroll[gi]; k++) enqueue_iteration(ctx);
        CK(cudaStreamEndCapture(ctx->s, &g));
        if (ctx->nccl_err != ncclSuccess) {
            cudaGraphDestroy(g);
            return fail(ctx, UCAC_ENCCL, "NCCL collective in the iteration graph: %s", ncclGetErrorString(ctx->nccl_err));
        }
        // single rank: load the new graph into this context's previous one (ucac_set_rho) or a
        // pooled one; multi-rank graphs are instantiated anew
        cudaGraphExec_t x = ctx->gexec[gi];
        ctx->gexec[gi] = nullptr;
        if (!x && gi == 0 && !ctx->multi && UCAC_EXEC_POOL) x = exec_pool_get();
        if (x && !ctx->multi) {
            cudaGraphExecUpdateResultInfo info;
            if (cudaGraphExecUpdate(x, g, &info) == cudaSuccess) {
                ctx->gexec[gi] = x;
                cudaGraphDestroy(g);
                continue;
            }
            cudaGetLastError();   // (a different topology: instantiate instead)
        }
        if (x) cudaGraphExecDestroy(x);
        // per-node launch priorities (launch_hi_prio) are honoured only with this flag
        cudaError_t e = cudaGraphInstantiate(&ctx->gexec[gi], g, UCAC_NODE_PRIO ? cudaGraphInstantiateFlagUseNodePriority : 0);
        cudaGraphDestroy(g);
        CK(e);
    }
    return UCAC_OK;
}

static ucac_status set_control(ucac_ctx *ctx, int stop, double target) {
    // write stop_on_primal, primal_target and clear done (three fields of the device status);
    // nothing to do when the last call ran without stop_on_primal and this one does too
    // (with the divergence detector on, every call starts with done cleared: a call it ended is over)
    if (!stop && !ctx->ctl_dirty && ctx->prm.diverge_window == 0) return UCAC_OK;
    ctx->ctl_dirty = stop != 0;
    DevStatus *h = ctx->st_host;
    h->stop_on_primal = stop;
    h->primal_target = target;
    h->done = 0;
    DevStatus *dd = ctx->d.st;
    CK(cudaMemcpyAsync(&dd->done, &h->done, sizeof(int), cudaMemcpyHostToDevice, ctx->s));
    CK(cudaMemcpyAsync(&dd->stop_on_primal, &h->stop_on_primal, sizeof(int), cudaMemcpyHostToDevice, ctx->s));
    CK(cudaMemcpyAsync(&dd->primal_target, &h->primal_target, sizeof(double), cudaMemcpyHostToDevice, ctx->s));
    return UCAC_OK;
}

static ucac_status pull_status(ucac_ctx *ctx) {
    CK(cudaMemcpyAsync(ctx->st_host, ctx->d.st, sizeof(DevStatus), cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    return UCAC_OK;
}

extern "C" ucac_status ucac_iterate(ucac_ctx *ctx, int32_t n, int32_t stop_on_primal, double primal_target,
                                    int32_t *n_done) {
    UCAC_NVTX("ucac_iterate");
    if (!ctx) return UCAC_EINVAL;
    if (n < 0) return fail(ctx, UCAC_EINVAL, "n < 0");
    if (ctx->nranks > 1 && ctx->comm_mode == 1)
        return fail(ctx, UCAC_ESTATE, "loopback-group contexts iterate through ucac_iterate_group");
    long long before = 0;
    if (n_done) {
        ucac_status s = pull_status(ctx);
        if (s != UCAC_OK) return s;
        before = ctx->st_host->inner_total;
    }
    ucac_status s = set_control(ctx, stop_on_primal > 0, primal_target);
    if (s != UCAC_OK) return s;
    const int big = ctx->gexec[1] ? ctx->gunroll[1] : n + 1;
    const int nb = n / big, nr = n % big;
    for (int k = 0; k < nb; k++) CK(cudaGraphLaunch(ctx->gexec[1], ctx->s));
    for (int k = 0; k < nr; k++) CK(cudaGraphLaunch(ctx->gexec[0], ctx->s));
    CK(cudaGetLastError());
    if (n_done) {
        s = pull_status(ctx);
        if (s != UCAC_OK) return s;
        *n_done = (int32_t)(ctx->st_host->inner_total - before);
        if (ctx->st_host->err_kernel) return fail(ctx, UCAC_ENUMERIC, "non-finite iterate at iteration %d", ctx->st_host->err_iter);
    }
    return UCAC_OK;
}

extern "C" ucac_status ucac_set_rho(ucac_ctx *ctx, double rho_pq, double rho_va, double rho_uc) {
    UCAC_NVTX("ucac_set_rho");
    if (!ctx) return UCAC_EINVAL;
    if (!(rho_pq > 0.0 && rho_va > 0.0 && rho_uc > 0.0) || !std::isfinite(rho_pq) || !std::isfinite(rho_va) ||
        !std::isfinite(rho_uc))
        return fail(ctx, UCAC_EINVAL, "rho must be positive and finite");
    CK(cudaStreamSynchronize(ctx->s));
    ucac_params &prm = ctx->prm;
    prm.rho_pq = rho_pq;
    prm.rho_va = rho_va;
    prm.rho_uc = rho_uc;
    Dev &d = ctx->d;
    d.rpq = rho_pq; d.rva = rho_va; d.ruc = rho_uc;
    d.irpq = 1.0 / rho_pq; d.irva = 1.0 / rho_va; d.iruc = 1.0 / rho_uc;
    d.tron_gtol = prm.tron_gtol_rel * std::max(rho_pq, rho_va);
    // the pipelined tail DP (k_gen tail) already ran the next (7a) with the old rho_uc: drop it
    CK(cudaMemsetAsync(d.unext_ok, 0, sizeof(unsigned), ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    // the graphs captured the old Dev by value: capture them again (build_graphs updates the
    // instantiated ones in place where it can)
    if (!(ctx->nranks > 1 && ctx->comm_mode == 1)) return build_graphs(ctx);
    return UCAC_OK;
}

// In-process loopback group: the partition contexts of one problem (comm_mode 1, same device)
// step through the same phases as the NCCL graph; the exchanges are device-to-device copies
// driven from the host between phases (no kernel ever waits on another context).
extern "C" ucac_status ucac_iterate_group(ucac_ctx **ctxs, int32_t n, int32_t iters) {
    UCAC_NVTX("ucac_iterate_group");
    if (!ctxs || n < 1 || iters < 0) return UCAC_EINVAL;
    for (int r = 0; r < n; r++)
        if (!ctxs[r] || ctxs[r]->nranks != n || ctxs[r]->rank != r || (n > 1 && ctxs[r]->comm_mode != 1))
            return fail(ctxs[r], UCAC_EINVAL, "group: context %d is not rank %d of a %d-rank loopback group", r, r, n);
    ucac_ctx *ctx = ctxs[0];
    auto sync_all = [&]() -> cudaError_t {
        for (int r = 0; r < n; r++) {
            cudaError_t e = cudaStreamSynchronize(ctxs[r]->s);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    };
    for (int r = 0; r < n; r++) {
        ucac_status s = set_control(ctxs[r], 0, 0.0);
        if (s != UCAC_OK) return s;
    }
    // all-gather of `count` doubles from every rank's send buffer into every rank's receive buffer
    auto allgather = [&](double *Dev::*snd, double *Dev::*rcv, size_t count) -> cudaError_t {
        for (int r = 0; r < n; r++)
            for (int q = 0; q < n; q++) {
                cudaError_t e = cudaMemcpyAsync(ctxs[r]->d.*rcv + (size_t)q * count, ctxs[q]->d.*snd, count * sizeof(double),
                                                cudaMemcpyDeviceToDevice, ctxs[r]->s);
                if (e != cudaSuccess) return e;
            }
        return cudaSuccess;
    };
    for (int it = 0; it < iters; it++) {
        if (ctx->d.tcut) {   // NEXT-4(c) time cut: the phases of enqueue_iteration_tc
            // d.p2p: each exchange is ONE cooperative launch emulating every rank's device-initiated
            // sends and waits (k_xchg.cu); else host-driven device-to-device copies
            std::vector<Dev> devs;
            for (int r = 0; r < n; r++) devs.push_back(ctxs[r]->d);
            auto exchange = [&](int phase, double *Dev::*snd, double *Dev::*rcv, size_t count) -> cudaError_t {
                if (ctx->d.p2p) return launch_xchg_group(devs.data(), n, phase, ctx->s, ctx->xdevs);
                return allgather(snd, rcv, count);
            };
            for (int r = 0; r < n; r++) launch_stage_tc(ctxs[r]->d, ctxs[r]->s);
            CK(sync_all());
            CK(exchange(1, &Dev::tc_stage_send, &Dev::tc_stage_recv, (size_t)ctx->d.G * ctx->d.Tmax * 4));
            CK(sync_all());
            for (int r = 0; r < n; r++) {
                ucac_ctx *c = ctxs[r];
                launch_dp_tc(c->d, c->s);
                launch_kernel(c, K_GENX, c->s);
                launch_pack_tc2(c->d, c->s);
            }
            CK(sync_all());
            CK(exchange(2, &Dev::tc2_send, &Dev::tc2_recv, (size_t)ctx->d.G * 2));
            CK(sync_all());
            for (int r = 0; r < n; r++) {
                ucac_ctx *c = ctxs[r];
                launch_unpack_tc2(c->d, c->s);
                const int seq[] = {K_BRANCH, K_UBAR, K_BUS, K_BRANCH_AL, K_BUS_LATE, K_ROWS, K_FOLD, K_ROWS_LATE};
                for (int k : seq) launch_kernel(c, k, c->s);
                launch_pack_tc3(c->d, c->s);
            }
            CK(sync_all());
            CK(exchange(3, &Dev::tc3_send, &Dev::tc3_recv, (size_t)ctx->d.G * 12));
            CK(sync_all());
            for (int r = 0; r < n; r++) launch_unpack_tc3(ctxs[r]->d, ctxs[r]->s);
            CK(sync_all());
        } else {
        // bus cut: the phases of enqueue_iteration_bus_multi (early exchanges before the AL tail's
        // results are used, late ones after), each exchange a copy of every rank's send buffer
        auto gather = [&](double *Dev::*snd, double *Dev::*rcv, int per, int Dev::*cnt, int Dev::*mx) -> cudaError_t {
            for (int r = 0; r < n; r++)
                for (int q = 0; q < n; q++) {
                    const Dev &dr = ctxs[r]->d, &dq = ctxs[q]->d;
                    const size_t blk = (size_t)(dr.*mx) * per * dr.T;
                    if (dq.*cnt > 0) {
                        cudaError_t e = cudaMemcpyAsync(dr.*rcv + q * blk, dq.*snd, (size_t)(dq.*cnt) * per * dq.T * sizeof(double),
                                                        cudaMemcpyDeviceToDevice, ctxs[r]->s);
                        if (e != cudaSuccess) return e;
                    }
                }
            return cudaSuccess;
        };
        for (int r = 0; r < n; r++) {
            ucac_ctx *c = ctxs[r];
            const int ph1[] = {K_BRANCH, K_GEN, K_GENX, K_UBAR};
            for (int k : ph1) launch_kernel(c, k, c->s);
            if (c->d.max_cut > 0) launch_pack_tau_early(c->d, c->s);
        }
        CK(sync_all());
        CK(gather(&Dev::xsend1, &Dev::xrecv1, 5, &Dev::ncut, &Dev::max_cut));
        CK(sync_all());
        for (int r = 0; r < n; r++) {
            ucac_ctx *c = ctxs[r];
            if (c->d.max_cut > 0) launch_unpack_tau_early(c->d, c->s);
            launch_kernel(c, K_BUS, c->s);
            if (c->d.max_export > 0) launch_pack_bus_early(c->d, c->s);
        }
        CK(sync_all());
        CK(gather(&Dev::xsend2, &Dev::xrecv2, 7, &Dev::nexport, &Dev::max_export));
        CK(sync_all());
        for (int r = 0; r < n; r++) {
            ucac_ctx *c = ctxs[r];
            if (c->d.max_export > 0) launch_unpack_bus_early(c->d, c->s);
            launch_kernel(c, K_ROWS, c->s);
            launch_kernel(c, K_FOLD, c->s);
            launch_kernel(c, K_BRANCH_AL, c->s);
            if (c->d.max_cut > 0) launch_pack_tau(c->d, c->s);
        }
        CK(sync_all());
        CK(gather(&Dev::xsend3, &Dev::xrecv3, 4, &Dev::ncut, &Dev::max_cut));
        CK(sync_all());
        for (int r = 0; r < n; r++) {
            ucac_ctx *c = ctxs[r];
            if (c->d.max_cut > 0) launch_unpack_tau(c->d, c->s);
            launch_kernel(c, K_BUS_LATE, c->s);
            if (c->d.max_export > 0) launch_pack_bus(c->d, c->s);
        }
        CK(sync_all());
        CK(gather(&Dev::xsend4, &Dev::xrecv4, 6, &Dev::nexport, &Dev::max_export));
        CK(sync_all());
        for (int r = 0; r < n; r++) {
            ucac_ctx *c = ctxs[r];
            if (c->d.max_export > 0) launch_unpack_bus(c->d, c->s);
            launch_kernel(c, K_ROWS_LATE, c->s);
        }
        CK(sync_all());
        }
        if (n > 1) {
            std::vector<double> all((size_t)n * NREC), red(NREC, 0.0);
            for (int r = 0; r < n; r++)
                CK(cudaMemcpy(all.data() + (size_t)r * NREC, ctxs[r]->d.rec, NREC * sizeof(double), cudaMemcpyDeviceToHost));
            for (int c = 0; c < NREC; c++) {
                double v = all[c];
                for (int r = 1; r < n; r++) v = c < NREC_SUM ? v + all[(size_t)r * NREC + c] : std::max(v, all[(size_t)r * NREC + c]);
                red[c] = v;
            }
            for (int r = 0; r < n; r++) {
                CK(cudaMemcpy(ctxs[r]->d.rec, red.data(), NREC * sizeof(double), cudaMemcpyHostToDevice));
                launch_finalize(ctxs[r]->d, ctxs[r]->s);
            }
            CK(sync_all());
        }
    }
    CK(cudaGetLastError());
    return UCAC_OK;
}

static const char *kNames[NKERN] = {"k_branch", "k_gen", "k_bus", "k_ubar", "k_bus_late", "k_branch_al", "k_rows",
                                    "k_genx", "k_rows_late", "k_fold_early"};
extern "C" const char *ucac_kernel_name(int32_t k) { return (k >= 0 && k < NKERN) ? kNames[k] : "?"; }

extern "C" ucac_status ucac_iterate_timed(ucac_ctx *ctx, int32_t n, double *kernel_ms, int64_t *launches) {
    UCAC_NVTX("ucac_iterate_timed");
    if (!ctx || n < 0) return UCAC_EINVAL;
    if (ctx->multi) return fail(ctx, UCAC_EUNSUPPORTED, "timed iterations are single-GPU");
    ucac_status s = set_control(ctx, 0, 0.0);
    if (s != UCAC_OK) return s;
    // eager iterations have no tail DP launch: every k_gen computes its own (7a)
    CK(cudaMemsetAsync(ctx->d.unext_ok, 0, sizeof(unsigned), ctx->s));
    const size_t need = (size_t)n * NKERN * 2;
    while (ctx->tev.size() < need) {
        cudaEvent_t ev;
        CK(cudaEventCreate(&ev));
        ctx->tev.push_back(ev);
    }
    for (int it = 0; it < n; it++) {
        for (int j = 0; j < NKERN; j++) {
            const int k = kOrder[j];   // the graph's dependency order; events indexed by kernel id
            cudaEvent_t a = ctx->tev[((size_t)it * NKERN + k) * 2], b = ctx->tev[((size_t)it * NKERN + k) * 2 + 1];
            CK(cudaEventRecord(a, ctx->s));
            {
                UCAC_NVTX(kNames[k]);
                launch_kernel(ctx, k, ctx->s);
            }
            CK(cudaEventRecord(b, ctx->s));
        }
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->s));
    for (int k = 0; k < NKERN; k++) {
        double tot = 0.0;
        for (int it = 0; it < n; it++) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ctx->tev[((size_t)it * NKERN + k) * 2], ctx->tev[((size_t)it * NKERN + k) * 2 + 1]));
            tot += ms;
        }
        if (kernel_ms) kernel_ms[k] = tot;
        if (launches) launches[k] = n;
    }
    return UCAC_OK;
}

// the component of a non-finite report as a global index of the kernel's component kind
static int32_t err_global_comp(const ucac_ctx *ctx, int err_kernel, int comp) {
    if (!err_kernel || comp < 0) return -1;
    const int k = err_kernel - 1;
    const std::vector<int> &v = (k == K_BRANCH || k == K_BRANCH_AL || k == K_ROWS || k == K_ROWS_LATE)
                                    ? ctx->P.branch_global
                                    : (k == K_BUS || k == K_BUS_LATE) ? ctx->P.bus_global : ctx->P.gen_global;
    return comp < (int)v.size() ? v[comp] : comp;
}

extern "C" ucac_status ucac_residuals(ucac_ctx *ctx, ucac_report *r) {
    UCAC_NVTX("ucac_residuals");
    if (!ctx || !r) return UCAC_EINVAL;
    ucac_status s = pull_status(ctx);
    if (s != UCAC_OK) return s;
    const DevStatus *h = ctx->st_host;
    r->primal_inf = h->primal_inf;
    r->rz_inf = h->rz_inf;
    r->rz_2 = h->rz_2;
    r->z_inf = h->z_inf;
    r->z_2 = h->z_2;
    r->dual_inf = h->dual_inf;
    r->objective = h->objective;
    r->beta = h->beta;
    r->inner_total = h->inner_total;
    r->outer_total = h->outer_k - 1;
    r->tron_iters = (int64_t)h->tron_iters;
    r->tron_capped = (int64_t)h->tron_capped;
    r->al_active = (int64_t)h->al_active;
    r->al_capped = (int64_t)h->al_capped;
    r->al_tron_iters = (int64_t)h->al_tron_iters;
    r->inner_since_outer = (int32_t)h->inner_since;
    r->outer_k = (int32_t)h->outer_k;
    r->err_kernel = h->err_kernel;
    r->err_iter = h->err_iter;
    r->err_comp = err_global_comp(ctx, h->err_kernel, h->err_comp);
    r->err_period = h->err_kernel ? h->err_period : -1;
    r->diverged_iter = h->diverged_iter;
    r->hist_len = (int32_t)std::max(0LL, std::min<long long>(h->inner_total - ctx->hist_base, HIST_CAP));
    if (h->err_kernel) return fail(ctx, UCAC_ENUMERIC, "non-finite iterate at iteration %d", h->err_iter);
    return UCAC_OK;
}

extern "C" ucac_status ucac_history(ucac_ctx *ctx, double *out, int32_t n, int32_t *got) {
    UCAC_NVTX("ucac_history");
    if (!ctx || n < 0 || (n > 0 && !out)) return UCAC_EINVAL;
    ucac_status s = pull_status(ctx);
    if (s != UCAC_OK) return s;
    const long long it = ctx->st_host->inner_total;
    const int have = (int)std::max(0LL, std::min<long long>(it - ctx->hist_base, HIST_CAP));
    const int m = std::min<int>(n, have);
    std::vector<double> all((size_t)HIST_CAP * HIST_FIELDS);
    CK(cudaMemcpyAsync(all.data(), ctx->d.hist, all.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    for (int j = 0; j < m; j++) {   // iterations it - m + 1 ... it, oldest first
        const long long iter = it - m + 1 + j;
        memcpy(out + (size_t)j * HIST_FIELDS, all.data() + (size_t)((iter - 1) % HIST_CAP) * HIST_FIELDS,
               HIST_FIELDS * sizeof(double));
    }
    if (got) *got = m;
    return UCAC_OK;
}

template <class Tp>
static cudaError_t down(ucac_ctx *ctx, Tp *dst, const Tp *src, size_t n) {
    if (n == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, n * sizeof(Tp), cudaMemcpyDeviceToHost, ctx->s);
}

// [K][n] device SoA <-> [n][K] canonical host
// out[j] = in[(j % K) * n + j / K]: one coalesced write per output element
__global__ void k_soa_to_aos(const double *__restrict__ in, double *__restrict__ out, size_t n, int K) {
    const size_t N = n * (size_t)K;
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < N; j += (size_t)gridDim.x * blockDim.x)
        out[j] = in[(j % K) * n + j / K];
}
static ucac_status soa_to_aos(ucac_ctx *ctx, double *host, const double *dev, size_t n, int K) {
    if (n == 0) return UCAC_OK;
    // transposed on the device into the context's scratch, then one copy
    k_soa_to_aos<<<148 * 8, 256, 0, ctx->s>>>(dev, ctx->xpose, n, K);
    CK(cudaGetLastError());
    CK(down(ctx, host, (const double *)ctx->xpose, n * K));
    CK(cudaStreamSynchronize(ctx->s));
    return UCAC_OK;
}
static ucac_status aos_to_soa(ucac_ctx *ctx, double *dev, const double *host, size_t n, int K) {
    std::vector<double> tmp(n * K);
    for (size_t i = 0; i < n; i++)
        for (int k = 0; k < K; k++) tmp[(size_t)k * n + i] = host[i * K + k];
    CK(up(ctx, dev, tmp.data(), n * K));
    CK(cudaStreamSynchronize(ctx->s));
    return UCAC_OK;
}

// State of the (rank-local) problem: generators, local branches and OWNED buses.
extern "C" ucac_status ucac_get_state(ucac_ctx *ctx, ucac_state *st) {
    UCAC_NVTX("ucac_get_state");
    if (!ctx || !st) return UCAC_EINVAL;
    launch_apply_outer(ctx->d, ctx->s);
    CK(cudaGetLastError());
    const Dev &d = ctx->d;
    const size_t GT = (size_t)ctx->G * ctx->T, LT = (size_t)ctx->L * ctx->T, BT = (size_t)ctx->B * ctx->T;
    CK(down(ctx, st->u, d.u, GT));
    CK(down(ctx, st->p, d.p, GT));
    CK(down(ctx, st->q, d.q, GT));
    CK(down(ctx, st->ph, d.ph, GT));
    CK(down(ctx, st->ub_on, d.ub_on, GT));
    CK(down(ctx, st->ub_su, d.ub_su, GT));
    CK(down(ctx, st->ub_sd, d.ub_sd, GT));
    CK(down(ctx, st->pbar, d.pbar, GT));
    CK(down(ctx, st->qbar, d.qbar, GT));
    CK(down(ctx, st->zg, d.zg, NGROW * GT));
    CK(down(ctx, st->yg, d.yg, NGROW * GT));
    CK(down(ctx, st->lg, d.lg, NGROW * GT));
    CK(down(ctx, st->zb, d.zb, NBROW * LT));
    CK(down(ctx, st->yb, d.yb, NBROW * LT));
    CK(down(ctx, st->lb, d.lb, NBROW * LT));
    CK(down(ctx, st->wbar, d.wbar, BT));
    CK(down(ctx, st->thbar, d.thbar, BT));
    ucac_status s;
    if ((s = soa_to_aos(ctx, st->x, d.x, LT, 4)) != UCAC_OK) return s;
    if ((s = soa_to_aos(ctx, st->f, d.f, LT, 4)) != UCAC_OK) return s;
    if ((s = soa_to_aos(ctx, st->fbar, d.fbar, LT, 4)) != UCAC_OK) return s;
    if ((s = soa_to_aos(ctx, st->al, d.al, LT, 3)) != UCAC_OK) return s;
    if ((s = pull_status(ctx)) != UCAC_OK) return s;
    const DevStatus *h = ctx->st_host;
    st->scal[0] = h->beta;
    st->scal[1] = h->znorm_prev;
    st->scal[2] = (double)h->outer_k;
    st->scal[3] = (double)h->inner_total;
    st->scal[4] = (double)h->inner_since;
    st->scal[5] = st->scal[6] = st->scal[7] = 0.0;
    return UCAC_OK;
}

extern "C" ucac_status ucac_set_state(ucac_ctx *ctx, const ucac_state *st) {
    UCAC_NVTX("ucac_set_state");
    if (!ctx || !st) return UCAC_EINVAL;
    if (ctx->nranks > 1) return fail(ctx, UCAC_EUNSUPPORTED, "set_state is single-GPU (ghost buses would be stale)");
    const Dev &d = ctx->d;
    const size_t GT = (size_t)ctx->G * ctx->T, LT = (size_t)ctx->L * ctx->T, BT = (size_t)ctx->B * ctx->T;
    CK(cudaStreamSynchronize(ctx->s));
    CK(up(ctx, d.u, (const int8_t *)st->u, GT));
    CK(up(ctx, d.p, (const double *)st->p, GT));
    CK(up(ctx, d.q, (const double *)st->q, GT));
    CK(up(ctx, d.ph, (const double *)st->ph, GT));
    CK(up(ctx, d.ub_on, (const double *)st->ub_on, GT));
    CK(up(ctx, d.ub_su, (const double *)st->ub_su, GT));
    CK(up(ctx, d.ub_sd, (const double *)st->ub_sd, GT));
    CK(up(ctx, d.pbar, (const double *)st->pbar, GT));
    CK(up(ctx, d.qbar, (const double *)st->qbar, GT));
    CK(up(ctx, d.zg, (const double *)st->zg, NGROW * GT));
    CK(up(ctx, d.yg, (const double *)st->yg, NGROW * GT));
    CK(up(ctx, d.lg, (const double *)st->lg, NGROW * GT));
    CK(up(ctx, d.zb, (const double *)st->zb, NBROW * LT));
    CK(up(ctx, d.yb, (const double *)st->yb, NBROW * LT));
    CK(up(ctx, d.lb, (const double *)st->lb, NBROW * LT));
    CK(up(ctx, d.wbar, (const double *)st->wbar, BT));
    CK(up(ctx, d.thbar, (const double *)st->thbar, BT));
    ucac_status s;
    if ((s = aos_to_soa(ctx, d.x, st->x, LT, 4)) != UCAC_OK) return s;
    if ((s = aos_to_soa(ctx, d.f, st->f, LT, 4)) != UCAC_OK) return s;
    if ((s = aos_to_soa(ctx, d.fbar, st->fbar, LT, 4)) != UCAC_OK) return s;
    if ((s = aos_to_soa(ctx, d.al, st->al, LT, 3)) != UCAC_OK) return s;
    if ((s = pull_status(ctx)) != UCAC_OK) return s;
    DevStatus *h = ctx->st_host;
    h->beta = st->scal[0];
    h->beta_lam = 0.0;
    h->znorm_prev = st->scal[1];
    h->outer_k = (long long)st->scal[2];
    h->inner_total = (long long)st->scal[3];
    h->inner_since = (long long)st->scal[4];
    h->pending_outer = 0;
    h->done = 0;
    h->err_kernel = 0;
    h->err_iter = 0;
    h->err_comp = -1;
    h->err_period = -1;
    h->diverged_iter = 0;
    CK(cudaMemcpyAsync(d.st, h, sizeof(DevStatus), cudaMemcpyHostToDevice, ctx->s));
    // the record history belongs to the replaced trajectory
    CK(cudaMemsetAsync(d.hist, 0xFF, (size_t)HIST_CAP * HIST_FIELDS * sizeof(double), ctx->s));
    ctx->hist_base = h->inner_total;
    CK(cudaMemsetAsync(d.cnt, 0, NCNT * sizeof(unsigned long long), ctx->s));
    CK(cudaMemsetAsync(d.unext_ok, 0, sizeof(unsigned), ctx->s));   // the pipelined DP result is stale
    CK(cudaMemsetAsync(d.alq_cnt, 0, (UCAC_AL_BUCKETS + 1) * sizeof(unsigned), ctx->s));
    CK(cudaMemsetAsync(d.alits, 0, (size_t)ctx->L * ctx->T, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    return UCAC_OK;
}

extern "C" ucac_status ucac_get_solution(ucac_ctx *ctx, ucac_solution *sol) {
    UCAC_NVTX("ucac_get_solution");
    if (!ctx || !sol) return UCAC_EINVAL;
    const Dev &d = ctx->d;
    const size_t GT = (size_t)ctx->G * ctx->T, LT = (size_t)ctx->L * ctx->T, BT = (size_t)ctx->B * ctx->T;
    if (sol->u_on) CK(down(ctx, sol->u_on, d.u, GT));
    if (sol->p) CK(down(ctx, sol->p, d.p, GT));
    if (sol->q) CK(down(ctx, sol->q, d.q, GT));
    if (sol->wbar) CK(down(ctx, sol->wbar, d.wbar, BT));
    if (sol->thetabar) CK(down(ctx, sol->thetabar, d.thbar, BT));
    if (sol->flows) {
        ucac_status s = soa_to_aos(ctx, sol->flows, d.f, LT, 4);
        if (s != UCAC_OK) return s;
    }
    CK(cudaStreamSynchronize(ctx->s));
    return UCAC_OK;
}

// NEXT-2: the UC warm start.  The multiperiod ACOPF with every unit on
// after its held prefix and the schedule held (uc_fixed), `iters` inner iterations; then on the
// device the Hamming stage costs to [p > threshold] and one batched DP pass (Algorithm 2) give the
// nearest schedule satisfying Eq. 3.  Single GPU.
extern "C" ucac_status ucac_uc_warm_start(const ucac_network *net, const ucac_horizon *hz, const ucac_costs *cost,
                                          const ucac_uc *uc, const ucac_params *prm, int32_t iters,
                                          double threshold, int8_t *u_out) {
    UCAC_NVTX("ucac_uc_warm_start");
    if (!net || !hz || !cost || !uc || !prm || !u_out || iters < 0) {
        g_create_err = "ucac_uc_warm_start: bad arguments";
        return UCAC_EINVAL;
    }
    const int G = net->ngen, T = hz->T;
    std::vector<int8_t> uinit((size_t)G * T);
    for (int g = 0; g < G; g++)
        for (int t = 0; t < T; t++) uinit[(size_t)g * T + t] = t < uc->hold[g] ? (int8_t)uc->u0[g] : (int8_t)1;
    ucac_uc uc2 = *uc;
    uc2.u_init = uinit.data();
    ucac_params p2 = *prm;
    p2.uc_fixed = 1;
    ucac_ctx *ctx = nullptr;
    ucac_status s = ucac_create(net, hz, cost, &uc2, &p2, nullptr, nullptr, &ctx);
    if (s != UCAC_OK) return s;
    s = ucac_iterate(ctx, iters, 0, 0.0, nullptr);
    double *L = nullptr, *c = nullptr;
    int8_t *sched = nullptr;
    cudaError_t e = cudaSuccess;
    if (s == UCAC_OK) {
        const Dev &d = ctx->d;
        const size_t GT = (size_t)G * T;
        if ((e = cudaMallocAsync((void **)&L, GT * 4 * sizeof(double), ctx->s)) == cudaSuccess &&
            (e = cudaMallocAsync((void **)&c, G * sizeof(double), ctx->s)) == cudaSuccess &&
            (e = cudaMallocAsync((void **)&sched, GT, ctx->s)) == cudaSuccess) {
            launch_hamming_costs((int)GT, d.p, threshold, L, ctx->s);
            e = launch_dp_batch(G, T, L, d.tu, d.td, d.u0, d.hold, sched, c, ctx->s);
            if (e == cudaSuccess) e = cudaMemcpyAsync(u_out, sched, GT, cudaMemcpyDeviceToHost, ctx->s);
            cudaFreeAsync(L, ctx->s);
            cudaFreeAsync(c, ctx->s);
            cudaFreeAsync(sched, ctx->s);
            cudaError_t e2 = cudaStreamSynchronize(ctx->s);
            if (e == cudaSuccess) e = e2;
        }
        if (e != cudaSuccess) {
            g_create_err = cudaGetErrorString(e);
            s = UCAC_ECUDA;
        }
    }
    ucac_destroy(ctx);
    return s;
}

extern "C" ucac_status ucac_local_map(ucac_ctx *ctx, int32_t which, int32_t *ids, int32_t *count) {
    if (!ctx || !count || which < 0 || which > 3) return UCAC_EINVAL;
    if (which == 3) {
        *count = 4;
        if (ids) {
            ids[0] = ctx->P.t_off;
            ids[1] = ctx->P.own0;
            ids[2] = ctx->P.own1;
            ids[3] = ctx->P.T;
        }
        return UCAC_OK;
    }
    const std::vector<int> &v = which == 0 ? ctx->P.gen_global : (which == 1 ? ctx->P.branch_global : ctx->P.bus_global);
    *count = (int32_t)v.size();
    if (ids) std::copy(v.begin(), v.end(), ids);
    return UCAC_OK;
}

extern "C" ucac_status ucac_dp_batch(int32_t ngen, int32_t T, const double *L, const int32_t *min_up,
                                     const int32_t *min_dn, const int32_t *u0, const int32_t *hold, int8_t *sched,
                                     double *cost, int32_t on_device, void *cuda_stream) {
    UCAC_NVTX("ucac_dp_batch");
    if (ngen <= 0 || T <= 0 || !L || !min_up || !min_dn || !u0 || !hold || !sched || !cost) {
        g_create_err = "ucac_dp_batch: bad arguments";
        return UCAC_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)cuda_stream;
    if (gen_set_smem_attr(T) != cudaSuccess) {
        g_create_err = "ucac_dp_batch: shared memory";
        return UCAC_ECUDA;
    }
    if (on_device) {
        cudaError_t e = launch_dp_batch(ngen, T, L, min_up, min_dn, u0, hold, sched, cost, s);
        if (e != cudaSuccess) {
            g_create_err = cudaGetErrorString(e);
            return UCAC_ECUDA;
        }
        return UCAC_OK;
    }
    for (int g = 0; g < ngen; g++)
        if (min_up[g] < 1 || min_up[g] > T || min_dn[g] < 1 || min_dn[g] > T || hold[g] < 0 || hold[g] > T ||
            (u0[g] != 0 && u0[g] != 1)) {
            g_create_err = "ucac_dp_batch: min_up/min_dn in [1,T], hold in [0,T], u0 in {0,1}";
            return UCAC_EINVAL;
        }
    double *dL = nullptr, *dc = nullptr;
    int *dtu = nullptr, *dtd = nullptr, *du0 = nullptr, *dh = nullptr;
    int8_t *ds = nullptr;
    const size_t GT = (size_t)ngen * T;
    cudaError_t e = cudaSuccess;
    if ((e = cudaMalloc(&dL, GT * 4 * 8)) != cudaSuccess || (e = cudaMalloc(&dc, ngen * 8)) != cudaSuccess ||
        (e = cudaMalloc(&dtu, ngen * 4)) != cudaSuccess || (e = cudaMalloc(&dtd, ngen * 4)) != cudaSuccess ||
        (e = cudaMalloc(&du0, ngen * 4)) != cudaSuccess || (e = cudaMalloc(&dh, ngen * 4)) != cudaSuccess ||
        (e = cudaMalloc(&ds, GT)) != cudaSuccess) {
    } else {
        cudaMemcpyAsync(dL, L, GT * 4 * 8, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(dtu, min_up, ngen * 4, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(dtd, min_dn, ngen * 4, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(du0, u0, ngen * 4, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(dh, hold, ngen * 4, cudaMemcpyHostToDevice, s);
        e = launch_dp_batch(ngen, T, dL, dtu, dtd, du0, dh, ds, dc, s);
        cudaMemcpyAsync(sched, ds, GT, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(cost, dc, ngen * 8, cudaMemcpyDeviceToHost, s);
        cudaError_t e2 = cudaStreamSynchronize(s);
        if (e == cudaSuccess) e = e2;
    }
    cudaFree(dL); cudaFree(dc); cudaFree(dtu); cudaFree(dtd); cudaFree(du0); cudaFree(dh); cudaFree(ds);
    if (e != cudaSuccess) {
        g_create_err = cudaGetErrorString(e);
        return UCAC_ECUDA;
    }
    return UCAC_OK;
}

extern "C" ucac_status ucac_get_sizes(ucac_ctx *ctx, ucac_sizes *sz) {
    if (!ctx || !sz) return UCAC_EINVAL;
    const int64_t G = ctx->G, L = ctx->L, B = ctx->B, T = ctx->T;
    const int64_t GT = G * T, LT = L * T, BT = B * T;
    sz->nrows = G * (12 * T - 1) + 8 * LT;
    sz->gen_periods = GT;
    sz->branch_periods = LT;
    sz->bus_periods = BT;
    // Algorithmic bytes: every array element a kernel must read or write once.
    // k_branch: read fbar(4) z(8) y(8) x(4) al(3) + wbar/thbar of both ends (4); write x(4) f(4) al(3) tauhat(8)
    sz->alg_bytes[K_BRANCH] = LT * 46 * 8 + L * (9 * 8 + 2 * 4);
    // k_gen (DP): read ubar, z, y of the 3 duplicate rows (9); write u (1 B)
    sz->alg_bytes[K_GEN] = GT * (9 * 8 + 1);
    // k_genx: read ubar(3) pbar qbar (2) z,y of 9 rows (18); write p q ph (3)
    sz->alg_bytes[K_GENX] = GT * 26 * 8 + G * 24 * 8;
    // k_bus: per gen-period read p q ph z,y,lambda of GP GQ RC (9) pbar qbar (2), write pbar qbar z y (8);
    //        per end-period read tauhat (4); per bus-period read pd qd wbar thbar, write wbar thbar + 4 bmu
    sz->alg_bytes[K_BUS] = GT * 19 * 8 + 2 * LT * 4 * 8 + BT * 10 * 8;
    // k_rows: per (l,t) read tauhat p,q (4) f (4) x (4) z,y,lambda (24) fbar (4) + bmu/wbar/thbar of 2 buses (12);
    //         write fbar (4) z y (16)
    sz->alg_bytes[K_ROWS] = LT * 72 * 8;
    // k_ubar: per gen-period: read u p q ph ubar(3) z,y,lambda of 9 rows (27); write ubar(3) z,y (18)
    sz->alg_bytes[K_UBAR] = GT * (51 * 8 + 1);
    // the early/late split of the bus solve and row update is data-dependent: the k_bus and k_rows
    // figures above cover all bus- and branch-periods (plus the marks they read); the late
    // kernels are charged only their own scan of the marks
    sz->alg_bytes[K_BUS] += BT * 4;
    sz->alg_bytes[K_ROWS] += 2 * LT * 4;
    sz->alg_bytes[K_BUS_LATE] = BT * 4;
    sz->alg_bytes[K_ROWS_LATE] = 2 * LT * 4;
    sz->alg_bytes[K_FOLD] = (int64_t)(ctx->d.nblk_bus + ctx->d.nblk_ubar + ctx->d.nblk_rows) * NPART * 8;
    sz->alg_bytes[K_BRANCH_AL] = 0;  // data-dependent: 49 doubles per queued (l,t)
    int64_t tot = 0;
    for (int k = 0; k < NKERN; k++) tot += sz->alg_bytes[k];
    sz->alg_bytes_per_iter = tot;
    return UCAC_OK;
}

extern "C" void *ucac_stream(ucac_ctx *ctx) { return ctx ? (void *)ctx->s : nullptr; }

extern "C" const char *ucac_last_error(const ucac_ctx *ctx) {
    if (!ctx) return g_create_err.c_str();
    return ctx->err.c_str();
}

extern "C" void ucac_destroy(ucac_ctx *ctx) {
    if (!ctx) return;
    stream_set_put(ctx);   // (its streams are idle once s is: every fork in the graphs joins s)
    if (ctx->s) cudaStreamSynchronize(ctx->s);
    if (ctx->gexec[0] && !ctx->multi && UCAC_EXEC_POOL && exec_pool_put(ctx->gexec[0])) ctx->gexec[0] = nullptr;
    for (auto &g : ctx->gexec)
        if (g) cudaGraphExecDestroy(g);
    for (auto ev : ctx->tev) cudaEventDestroy(ev);
    for (void *p : ctx->dalloc) cudaFreeAsync(p, ctx->s);
    if (ctx->s && !ctx->dalloc.empty()) cudaStreamSynchronize(ctx->s);
    for (void *p : ctx->peer_maps) cudaIpcCloseMemHandle(p);
    if (ctx->xbuf) cudaFree(ctx->xbuf);
    if (ctx->xdevs) cudaFree(ctx->xdevs);
    if (ctx->comm2) ncclCommDestroy(ctx->comm2);
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    if (ctx->st_host) pinned_status_put(ctx->st_host);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->ev_genx) cudaEventDestroy(ctx->ev_genx);
    if (ctx->ev_early) cudaEventDestroy(ctx->ev_early);
    if (ctx->ev_branch) cudaEventDestroy(ctx->ev_branch);
    if (ctx->ev_tail) cudaEventDestroy(ctx->ev_tail);
    if (ctx->ev_bus) cudaEventDestroy(ctx->ev_bus);
    if (ctx->s2) cudaStreamDestroy(ctx->s2);
    if (ctx->s3) cudaStreamDestroy(ctx->s3);
    if (ctx->own_stream && ctx->s) cudaStreamDestroy(ctx->s);
    delete ctx;
}

#ifdef UCAC_PROF
// diagnostic builds only: reset / read the kernel timeline (2*NKERN u64: first start, last exit)
extern "C" int ucac_debug_timeline(ucac_ctx *ctx, unsigned long long *host, int reset) {
    if (reset) {
        std::vector<unsigned long long> v(2 * NKERN);
        for (int k = 0; k < NKERN; k++) {
            v[2 * k] = ~0ull;
            v[2 * k + 1] = 0ull;
        }
        return (int)cudaMemcpy(ctx->d.tl, v.data(), v.size() * 8, cudaMemcpyHostToDevice);
    }
    return (int)cudaMemcpy(host, ctx->d.tl, 2 * NKERN * 8, cudaMemcpyDeviceToHost);
}
// diagnostic builds only: a one-thread kernel on the context's stream stores the global timer in
// slot (0..7) when the stream reaches it (graph start / end latencies, tools/timeline.py); slot < 0
// copies the 8 slots to host
__device__ unsigned long long g_stamp[8];
__global__ void k_stamp(int slot) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_stamp[slot] = t;
}
extern "C" int ucac_debug_stamp(ucac_ctx *ctx, unsigned long long *host, int slot) {
    if (slot >= 0 && slot < 8) {
        k_stamp<<<1, 1, 0, ctx->s>>>(slot);
        return (int)cudaGetLastError();
    }
    return (int)cudaMemcpyFromSymbol(host, g_stamp, sizeof(g_stamp));
}
#endif

extern "C" ucac_status ucac_debug_poison(ucac_ctx *ctx, int32_t field, int64_t index) {
    if (!ctx) return UCAC_EINVAL;
    const Dev &d = ctx->d;
    const int64_t GT = (int64_t)ctx->G * ctx->T, LT = (int64_t)ctx->L * ctx->T;
    double *base = field == 0 ? d.zb : field == 1 ? d.yb : field == 2 ? d.zg : field == 3 ? d.yg : nullptr;
    const int64_t n = field < 2 ? NBROW * LT : NGROW * GT;
    if (!base || index < 0 || index >= n) return fail(ctx, UCAC_EINVAL, "poison: field %d index %lld", field, (long long)index);
    const double nan = std::numeric_limits<double>::quiet_NaN();
    CK(cudaStreamSynchronize(ctx->s));
    CK(cudaMemcpyAsync(base + index, &nan, sizeof(double), cudaMemcpyHostToDevice, ctx->s));
    CK(cudaMemsetAsync(d.unext_ok, 0, sizeof(unsigned), ctx->s));   // the pipelined DP read the old value
    CK(cudaStreamSynchronize(ctx->s));
    return UCAC_OK;
}

extern "C" ucac_status ucac_time_split(int32_t T, int32_t nranks, int32_t rank, int32_t *out) {
    if (T < 1 || nranks < 1 || nranks > T || rank < 0 || rank >= nranks || !out) return UCAC_EINVAL;
    std::vector<int> t0;
    time_split(T, nranks, t0);
    const int g0 = t0[rank], g1 = t0[rank + 1];
    const int hl = g0 > 0, hh = g1 < T;
    out[0] = g0 - hl;                 // global period of local period 0
    out[1] = hl;                      // first owned local period
    out[2] = hl + (g1 - g0);          // end of the owned local periods
    out[3] = (g1 - g0) + hl + hh;     // local periods (halos included)
    return UCAC_OK;
}

extern "C" int32_t ucac_comm_nccl(const ucac_ctx *ctx) { return ctx ? (ctx->comm != nullptr ? 1 : 0) : -1; }

extern "C" ucac_status ucac_comm_info(ucac_ctx *ctx, int32_t *nranks, int32_t *rank) {
    if (!ctx || !nranks || !rank) return UCAC_EINVAL;
    if (ctx->comm) {   // what the NCCL communicator itself reports
        int n = 0, r = 0;
        NK(ncclCommCount(ctx->comm, &n));
        NK(ncclCommUserRank(ctx->comm, &r));
        *nranks = n;
        *rank = r;
    } else {
        *nranks = ctx->nranks;
        *rank = ctx->rank;
    }
    return UCAC_OK;
}

// ---- device-initiated exchange of the time cut (NEXT-4(c), k_xchg.cu)
static void set_peer(Dev &d, int q, char *xb, const size_t *off) {
    d.peer_stage_recv[q] = (double *)(xb + off[0]);
    d.peer_tc2_recv[q] = (double *)(xb + off[1]);
    d.peer_tc3_recv[q] = (double *)(xb + off[2]);
    d.peer_flags[q] = (unsigned long long *)(xb + off[3]);
}

extern "C" ucac_status ucac_p2p_group(ucac_ctx **ctxs, int32_t n) {
    UCAC_NVTX("ucac_p2p_group");
    if (!ctxs || n < 2 || n > UCAC_MAX_P2P) return UCAC_EINVAL;
    for (int r = 0; r < n; r++)
        if (!ctxs[r] || !ctxs[r]->d.tcut || ctxs[r]->comm_mode != 1 || ctxs[r]->rank != r || ctxs[r]->nranks != n)
            return fail(ctxs[r], UCAC_EINVAL, "p2p group: context %d is not rank %d of a time-cut loopback group", r, r);
    for (int r = 0; r < n; r++) {
        Dev &d = ctxs[r]->d;
        for (int q = 0; q < n; q++) set_peer(d, q, (char *)ctxs[q]->xbuf, ctxs[q]->xoff);
        d.p2p = 1;
    }
    ucac_ctx *ctx = ctxs[0];
    if (!ctx->xdevs) CK(cudaMalloc(&ctx->xdevs, sizeof(Dev) * UCAC_MAX_P2P));
    return UCAC_OK;
}

// blob = cudaIpcMemHandle_t of the exchange block, then its 4 offsets (uint64)
extern "C" ucac_status ucac_p2p_export(ucac_ctx *ctx, unsigned char *blob) {
    if (!ctx || !blob) return UCAC_EINVAL;
    if (!ctx->d.tcut || !ctx->xbuf) return fail(ctx, UCAC_EUNSUPPORTED, "p2p: not a time-cut context");
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, ctx->xbuf));
    memcpy(blob, &h, sizeof(h));
    uint64_t off[4] = {ctx->xoff[0], ctx->xoff[1], ctx->xoff[2], ctx->xoff[3]};
    memcpy(blob + sizeof(h), off, sizeof(off));
    return UCAC_OK;
}

extern "C" ucac_status ucac_p2p_import(ucac_ctx *ctx, const unsigned char *blobs) {
    UCAC_NVTX("ucac_p2p_import");
    if (!ctx || !blobs) return UCAC_EINVAL;
    if (!ctx->d.tcut || ctx->comm_mode != 0 || ctx->nranks > UCAC_MAX_P2P)
        return fail(ctx, UCAC_EUNSUPPORTED, "p2p: an NCCL time-cut context of at most %d ranks", UCAC_MAX_P2P);
    Dev &d = ctx->d;
    for (int q = 0; q < ctx->nranks; q++) {
        const unsigned char *b = blobs + (size_t)q * UCAC_P2P_BLOB;
        uint64_t off64[4];
        memcpy(off64, b + sizeof(cudaIpcMemHandle_t), sizeof(off64));
        const size_t off[4] = {(size_t)off64[0], (size_t)off64[1], (size_t)off64[2], (size_t)off64[3]};
        if (q == ctx->rank) {
            set_peer(d, q, (char *)ctx->xbuf, off);
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, b, sizeof(h));
        void *p = nullptr;
        CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        ctx->peer_maps.push_back(p);
        set_peer(d, q, (char *)p, off);
    }
    d.p2p = 1;
    for (auto &g : ctx->gexec)
        if (g) {
            cudaGraphExecDestroy(g);
            g = nullptr;
        }
    return build_graphs(ctx);
}
