// k_sweep.cu -- steps (7c) ubar, (7d) bus, (7e) z, (7f) y for every coupling row, the
// residual/objective partial reductions (S8), the final reduction with the inner test and
// the outer (lambda, beta) decision (S9).  Compiled with -fmad=false (operation
// order as written, matching the oracle's definitions).
//
// Ownership (no write conflicts, no atomics): every coupling row's xbar side, z and y are
// written by exactly one thread:
//   k_bus   thread (i,t): the generator copies pbar_g,t, qbar_g,t of g at i (rows GP_t, GQ_t and
//           RC_{t+1}), the flow copies of every branch end at i (FP, FQ) and wbar_i,t, thbar_i,t
//           (rows W, A of every end at i);
//   k_ubar  thread (g,t): the group (ubar^on_t, ubar^sd_t, ubar^su_{t+1}) and its rows D_ON_t,
//           D_SD_t, PL_t..RD_t, D_SU_{t+1}, RU_{t+1}; thread (g,0) also group 0 (ubar^su_1).
// The outer update lambda <- clip(lambda + beta z) decided at the end of iteration l is
// applied lazily by the owning thread at the start of its row update in iteration l+1 (the
// x-steps never read lambda), which saves a full pass over all rows.
#include <algorithm>
#include <cstdlib>

#include "ucac_dev.cuh"

namespace ucac {
namespace {

struct Acc {
    double v[NPART];
    __device__ Acc() {
#pragma unroll
        for (int k = 0; k < NPART; k++) v[k] = 0.0;
    }
};

// (7e) z = -(lambda + y + rho r)/(beta + rho), (7f) y += rho (r + z); S8 terms.
// ib = 1/(beta + rho), formed once per thread: the quotient becomes a product (within one ulp of
// the oracle's), with no division slow path to spill around.
__device__ __forceinline__ void zy_row(double r, double rho, double ib, double *zp, double *yp, double *lp,
                                       int pending, double beta_lam, double lmax, double dxb, Acc &a,
                                       double bpr = 0.0) {
    double lam = *lp;
    double zo = *zp;
    if (pending) {
        double v = lam + beta_lam * zo;
        lam = v < -lmax ? -lmax : (v > lmax ? lmax : v);
        *lp = lam;
    }
    double y = *yp;
    double zz = (bpr > 0.0 ? -((lam + y) + rho * r) / bpr : -((lam + y) + rho * r) * ib);
    *zp = zz;
    *yp = y + rho * (r + zz);
    double rz = r + zz;
    a.v[P_PINF] = fmax(a.v[P_PINF], fabs(r));
    a.v[P_RZINF] = fmax(a.v[P_RZINF], fabs(rz));
    a.v[P_RZ2] = a.v[P_RZ2] + rz * rz;
    a.v[P_ZINF] = fmax(a.v[P_ZINF], fabs(zz));
    a.v[P_Z2] = a.v[P_Z2] + zz * zz;
    a.v[P_DINF] = fmax(a.v[P_DINF], rho * fabs(dxb));
    if (!isfinite(r) || !isfinite(zz)) a.v[P_BAD] = 1.0;
}

// the same update on values (loads hoisted by the caller): returns z, y and lambda in place
__device__ __forceinline__ void zy_vals(double r, double rho, double ib, double &z, double &y, double &lam,
                                        int pending, double beta_lam, double lmax, double dxb, Acc &a,
                                        double bpr = 0.0) {
    if (pending) {
        const double v = lam + beta_lam * z;
        lam = v < -lmax ? -lmax : (v > lmax ? lmax : v);
    }
    const double zz = (bpr > 0.0 ? -((lam + y) + rho * r) / bpr : -((lam + y) + rho * r) * ib);
    y = y + rho * (r + zz);
    z = zz;
    const double rz = r + zz;
    a.v[P_PINF] = fmax(a.v[P_PINF], fabs(r));
    a.v[P_RZINF] = fmax(a.v[P_RZINF], fabs(rz));
    a.v[P_RZ2] = a.v[P_RZ2] + rz * rz;
    a.v[P_ZINF] = fmax(a.v[P_ZINF], fabs(zz));
    a.v[P_Z2] = a.v[P_Z2] + zz * zz;
    a.v[P_DINF] = fmax(a.v[P_DINF], rho * fabs(dxb));
    if (!isfinite(r) || !isfinite(zz)) a.v[P_BAD] = 1.0;
}

// k_ubar's twins of zy_row / zy_vals with the oracle's exact quotient (bpr = beta + rho): the
// (7c) box-QP can be ill-conditioned, and k_ubar/k_genx keep the oracle's bits
__device__ __forceinline__ void zy_row_div(double r, double rho, double bpr, double *zp, double *yp, double *lp,
                                           int pending, double beta_lam, double lmax, double dxb, Acc &a) {
    zy_row(r, rho, 0.0, zp, yp, lp, pending, beta_lam, lmax, dxb, a, bpr);
}
__device__ __forceinline__ void zy_vals_div(double r, double rho, double bpr, double &z, double &y, double &lam,
                                            int pending, double beta_lam, double lmax, double dxb, Acc &a) {
    zy_vals(r, rho, 0.0, z, y, lam, pending, beta_lam, lmax, dxb, a, bpr);
}

#ifndef UCAC_RED_SKIP
#define UCAC_RED_SKIP 1   // idle warps skip the block reduction's shuffle tree (bitwise neutral)
#endif
// deterministic block reduction -> part[blockIdx.x][NPART]
__device__ void block_reduce_store(Acc &a, double *part, int vb = -1) {
    if (vb < 0) vb = blockIdx.x;
    __shared__ double sh[32][NPART];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // A warp none of whose lanes touched its accumulator (every slot still +0.0, compared
    // bitwise) folds to +0.0 in every slot (0 + 0 and fmax(0, 0)), so it skips the shuffle tree
    // and stores that directly: the same bits.  Most warps of the late kernels are such warps.
    bool touched = !UCAC_RED_SKIP;
#pragma unroll
    for (int k = 0; k < NPART; k++) touched |= __double_as_longlong(a.v[k]) != 0;
    if (!__any_sync(0xffffffffu, touched)) {
        if (lane < NPART) sh[warp][lane] = 0.0;
    } else {
#pragma unroll
        for (int k = 0; k < NPART; k++) {
            double v = a.v[k];
            const bool isum = (k == P_RZ2 || k == P_Z2 || k == P_OBJ);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                double w = __shfl_down_sync(0xffffffffu, v, o);
                v = isum ? v + w : fmax(v, w);
            }
            if (lane == 0) sh[warp][k] = v;
        }
    }
    __syncthreads();
    if (threadIdx.x < NPART) {
        const int k = threadIdx.x;
        const bool isum = (k == P_RZ2 || k == P_Z2 || k == P_OBJ);
        double v = sh[0][k];
        for (int w = 1; w < nw; w++) v = isum ? v + sh[w][k] : fmax(v, sh[w][k]);
        part[(size_t)vb * NPART + k] = v;
    }
}

#define ZG(k, i) d.zg[(size_t)(k) * GT + (i)]
#define YG(k, i) d.yg[(size_t)(k) * GT + (i)]
#define LG(k, i) d.lg[(size_t)(k) * GT + (i)]
#define ZB(k, i) d.zb[(size_t)(k) * LT + (i)]
#define YB(k, i) d.yb[(size_t)(k) * LT + (i)]
#define LB(k, i) d.lb[(size_t)(k) * LT + (i)]
#define FX(k, i) d.f[(size_t)(k) * LT + (i)]
#define FB(k, i) d.fbar[(size_t)(k) * LT + (i)]
#define XX(k, i) d.x[(size_t)(k) * LT + (i)]
#define TH(k, i) d.tauh[(size_t)(k) * LTH + (i)]

constexpr int BUS_THREADS = 128;
// __launch_bounds__ minimum resident blocks per SM (register caps), unset = none: an explicit 1
// is not the same as none (ptxas gave k_bus 148 instead of 128 registers, +3 us); measured
// DESIGN.md 7
#ifdef UCAC_BUS_MINB
#define BUS_BOUNDS __launch_bounds__(BUS_THREADS, UCAC_BUS_MINB)
#else
#define BUS_BOUNDS __launch_bounds__(BUS_THREADS)
#endif
#ifdef UCAC_ROWS_MINB
#define ROWS_BOUNDS __launch_bounds__(ROWS_THREADS, UCAC_ROWS_MINB)
#else
#define ROWS_BOUNDS __launch_bounds__(ROWS_THREADS)
#endif
#ifdef UCAC_UBAR_MINB
#define UBAR_BOUNDS __launch_bounds__(UBAR_THREADS, UCAC_UBAR_MINB)
#else
#define UBAR_BOUNDS __launch_bounds__(UBAR_THREADS)
#endif
constexpr int UBAR_THREADS = 64;
constexpr int ROWS_THREADS = 128;
// late kernels: most threads skip (unmarked rows), so the block waits on its slowest chain.
// The bus kernel keeps 1024-thread blocks; the rows kernel, whose row updates need more than the
// 64 registers of a 1024-thread block, runs 256-thread blocks (measured)
#ifndef UCAC_LBUS_THREADS
#define UCAC_LBUS_THREADS 128
#endif
#ifndef UCAC_LROWS_THREADS
#define UCAC_LROWS_THREADS 256
#endif
constexpr int LBUS_THREADS = UCAC_LBUS_THREADS, LROWS_THREADS = UCAC_LROWS_THREADS;

// ------------------------------------------------------------------------- S8 partials
// Every kernel that updates rows leaves one partial per block.  The early ones (k_bus, k_ubar,
// k_rows) are folded by k_fold_early off the critical path (in the shadow of the AL tail); the
// LAST block of k_rows_late (threadfence + counter) folds the late kernels' partials (k_bus_late's,
// then its own; k_bus_late itself when the rows are fused into it), and the last block of the
// iteration's last kernel folds the three records.  Fixed slots, fixed order: deterministic.
enum RecKind { RK_EARLY = 0, RK_BUS_LATE, RK_ROWS_LATE, NRK };

// fold slots [0, n) of part into out[NPART]: 32 groups of NPART threads take every 32nd slot
// (independent loads in flight), then the groups are folded in order
__device__ __forceinline__ double fold(int k, double a, double b) {
    return (k == P_RZ2 || k == P_Z2 || k == P_OBJ) ? a + b : fmax(a, b);
}
#ifndef UCAC_FOLD_BATCH
#define UCAC_FOLD_BATCH 16
#endif
constexpr int FOLD_BATCH = UCAC_FOLD_BATCH;
__device__ void fold_slots(const double *part, int n, double *out) {
    __shared__ double grp[32][NPART];
    const int ng = min(32, (int)blockDim.x / NPART);   // groups (blockDim is a multiple of NPART)
    const int k = threadIdx.x % NPART, g = threadIdx.x / NPART;
    if (g < ng) {
        double v = 0.0;
        // FOLD_BATCH independent loads in flight per round trip, folded in slot order (g, g+ng, ...):
        // the last block's fold is on the iteration's critical path, and with 4 in flight the
        // ~860 partials of k_rows_late took 7 dependent L2 round trips
        for (int j = g; j < n; j += FOLD_BATCH * ng) {
            double a[FOLD_BATCH];
#pragma unroll
            for (int u = 0; u < FOLD_BATCH; u++) {
                const int jj = j + u * ng;
                a[u] = jj < n ? __ldcg(part + (size_t)jj * NPART + k) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < FOLD_BATCH; u++)
                if (j + u * ng < n) v = fold(k, v, a[u]);
        }
        grp[g][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < NPART) {
        double v = grp[0][threadIdx.x];
        for (int q = 1; q < ng; q++) v = fold(threadIdx.x, v, grp[q][threadIdx.x]);
        out[threadIdx.x] = v;
    }
    __syncthreads();
}

// store this block's partial; true in the last block of the launch (which then folds)
__device__ bool store_partial_last(Acc &acc, double *part, unsigned *counter) {
    block_reduce_store(acc, part);
    __shared__ bool last;
    if (threadIdx.x < NPART) __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last) {
        __threadfence();
        if (threadIdx.x == 0) *counter = 0;   // ready for the next launch
    }
    return last;
}

__device__ void finalize_status(const Dev &d, const double *rec);

// last block of the iteration: fold the three records (fixed order) -> S8 record -> S9
__device__ void final_fold(const Dev &d) {
    __shared__ double fin[NPART];
    if (threadIdx.x < NPART) {
        const int k = threadIdx.x;
        double v = __ldcg(d.rec_part + k);
        for (int r = 1; r < NRK; r++) v = fold(k, v, __ldcg(d.rec_part + r * NPART + k));
        fin[k] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double rec[NREC];
        rec[R_RZ2] = fin[P_RZ2];
        rec[R_Z2] = fin[P_Z2];
        rec[R_OBJ] = fin[P_OBJ];
        for (int q = 0; q < NCNT; q++) rec[R_C0 + q] = (double)__ldcg(d.cnt + q);
        rec[R_PINF] = fin[P_PINF];
        rec[R_RZINF] = fin[P_RZINF];
        rec[R_ZINF] = fin[P_ZINF];
        rec[R_DINF] = fin[P_DINF];
        rec[R_BAD] = fin[P_BAD];
        for (int q = 0; q < NCNT; q++) d.cnt[q] = 0;
        for (int q = 0; q <= UCAC_AL_BUCKETS; q++) d.alq_cnt[q] = 0;
        if (d.xrank_rec) {
            for (int q = 0; q < NREC; q++) d.rec[q] = rec[q];   // cross-rank all-reduce, then k_finalize
        } else {
            finalize_status(d, rec);
        }
    }
}

__device__ __forceinline__ void kernel_tail(const Dev &d, Acc &acc, double *part, int kind, bool final) {
    if (store_partial_last(acc, part, d.kdone + kind)) {
        fold_slots(part, gridDim.x, d.rec_part + kind * NPART);
        if (final) {
            __threadfence();
            final_fold(d);
        }
    }
}


// ------------------------------------------------------------------------- (7d) bus
// k_bus: one thread per (i,t) solves the bus 2x2 KKT system from the bus-side targets of its
// generators' rows (read here) and of its incident branch ends (tauhat, written by k_branch),
// in canonical CSR order; writes the generator copies (and their rows GP, GQ, RC_{t+1}),
// wbar, thbar and (muP, muQ, dwbar, dthbar) for k_rows.
//
// Split: k_bus (early) takes the bus-periods with no thermal-AL solve at an
// incident branch end -- their inputs are final after the fast path, so in the single-GPU graph
// it runs in the shadow of k_branch_al -- and k_late the marked ones after the AL tail.
// STRICT (strict_fp parity mode): the oracle's quotients y/rho, mu/rho and /(beta + rho)
// instead of products with reciprocals, so the bus and row updates are the oracle's bits
struct Ctl {
    double rpq, rva, irpq, beta, beta_lam, lmax, ibpq, ibva, bpq, bva;
    int pending;
    unsigned stamp;
    __device__ explicit Ctl(const Dev &d)
        : rpq(d.rpq), rva(d.rva), irpq(d.irpq), beta(d.st->beta), beta_lam(d.st->beta_lam), lmax(d.lambda_max),
          ibpq(1.0 / (beta + d.rpq)), ibva(1.0 / (beta + d.rva)), bpq(beta + d.rpq), bva(beta + d.rva),
          pending(d.st->pending_outer), stamp(mark_stamp(d)) {}
};
template <bool STRICT>
__device__ __forceinline__ double over_rho(double v, double rho, double irho) { return STRICT ? v / rho : v * irho; }
// (7e)/(7f) of one row with the reciprocal (default) or the oracle's quotient (STRICT)
template <bool STRICT>
__device__ __forceinline__ void zy_s(double r, double rho, double ib, double bpr, double &z, double &y, double &lam,
                                     int pending, double beta_lam, double lmax, double dxb, Acc &a) {
    if (STRICT) zy_vals(r, rho, 0.0, z, y, lam, pending, beta_lam, lmax, dxb, a, bpr);
    else zy_vals(r, rho, ib, z, y, lam, pending, beta_lam, lmax, dxb, a);
}

// ---- compacted late lists.  The early kernels see every mark: each block writes its
// marked items, in thread order, to its own fixed slot range list[blockIdx.x * cap ...] and the
// count to cnt[blockIdx.x].  A late block turns the counts into exclusive offsets (shared memory)
// and takes items j = its thread id + k * grid stride of the concatenation -- a deterministic
// list in index order, so the late kernels need a grid sized to the marked work only, and
// their fold order is fixed.
__device__ __forceinline__ void block_compact(int nitems, const int *items, int *list, unsigned *cnt, int cap, int vb = -1) {
    if (vb < 0) vb = blockIdx.x;
    __shared__ int wsum[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int incl = nitems;   // inclusive warp scan of the per-thread counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < nw; w++) {
        if (w < warp) off += wsum[w];
        tot += wsum[w];
    }
    off += incl - nitems;
    for (int q = 0; q < nitems; q++) list[(size_t)vb * cap + off + q] = items[q];
    if (threadIdx.x == 0) cnt[vb] = (unsigned)tot;
    __syncthreads();
}
// exclusive offsets pre[0..n] of cnt[0..n) in shared memory (block-wide); returns the total
__device__ __forceinline__ int block_offsets(const unsigned *cnt, int n, int *pre) {
    __shared__ int wsum[32];
    const int nt = blockDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = nt >> 5;
    // one coalesced pass of independent loads into shared memory, then the scan from there
    // (unrolled so all of a thread's loads are in flight together: one L2 round trip, not n / nt)
    {
        constexpr int U = 16;
        for (int i0 = threadIdx.x; i0 < n; i0 += U * nt) {
            int v[U];
#pragma unroll
            for (int u = 0; u < U; u++) v[u] = i0 + u * nt < n ? (int)__ldcg(cnt + i0 + u * nt) : 0;
#pragma unroll
            for (int u = 0; u < U; u++)
                if (i0 + u * nt < n) pre[i0 + u * nt] = v[u];
        }
    }
    __syncthreads();
    const int per = (n + nt - 1) / nt;
    const int beg = min(n, (int)threadIdx.x * per), end = min(n, beg + per);
    int sum = 0;
    for (int i = beg; i < end; i++) sum += pre[i];
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int off = 0;
    for (int w = 0; w < warp; w++) off += wsum[w];
    off += incl - sum;
    for (int i = beg; i < end; i++) {
        const int c = pre[i];
        pre[i] = off;
        off += c;
    }
    if (threadIdx.x == nt - 1) pre[n] = off;
    __syncthreads();
    return pre[n];
}
// item j of the concatenated lists: source block by binary search over the offsets
__device__ __forceinline__ int list_item(const int *pre, int n, const int *list, int cap, int j) {
    int lo = 0, hi = n;   // largest src with pre[src] <= j (pre[n] > j)
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (pre[mid] <= j) lo = mid;
        else hi = mid;
    }
    return __ldcg(list + (size_t)lo * cap + (j - pre[lo]));
}

// bus-period k = i*T + t of an owned bus (ghost buses are solved by their owner)
template <bool STRICT>
__device__ __forceinline__ void bus_solve(const Dev &d, const Ctl &c, int k, Acc &acc) {
    const int T = d.T;
    const size_t GT = (size_t)d.G * T, BT = (size_t)d.B * T;
    const size_t LTH = (size_t)(d.L + d.Lph) * T;
    const double rpq = c.rpq, rva = c.rva;
    const double irpq = c.irpq, ibpq = c.ibpq, beta_lam = c.beta_lam, lmax = c.lmax;
    const int pending = c.pending;
    {
        const int i = k / T, t = k - i * T;
        const int g0 = d.bg_ptr[i], g1 = d.bg_ptr[i + 1];
        const int e0 = d.be_ptr[i], e1 = d.be_ptr[i + 1];
        const int ne = e1 - e0;
        // ---- sums of the 2x2 KKT system, canonical order (gens, ends, wbar)
        const bool has_next = tglob(d, t) < d.Tg - 1;   // a ramp-copy row RC_{t+1} exists
        double AP = 0.0, AQ = 0.0, C = 0.0, rP = d.pd[k], rQ = d.qd[k];
        const double wbo = d.wbar[k], tbo = d.thbar[k];
        // (loops unrolled so the loads of several gens / ends are in flight together)
#pragma unroll 2
        for (int a = g0; a < g1; a++) {
            const size_t gi = (size_t)d.bg_idx[a] * T + t;
            const double tgp = d.p[gi] + ZG(G_GP, gi) + over_rho<STRICT>(YG(G_GP, gi), rpq, irpq);
            double th, aa;
            if (has_next) {
                const double trc = d.ph[gi + 1] + ZG(G_RC, gi + 1) + over_rho<STRICT>(YG(G_RC, gi + 1), rpq, irpq);
                th = (tgp + trc) * 0.5;
                aa = 2.0 * rpq;
            } else {
                th = tgp;
                aa = rpq;
            }
            AP = AP + 1.0 / aa;
            rP = rP - th;
            const double thq = d.q[gi] + ZG(G_GQ, gi) + over_rho<STRICT>(YG(G_GQ, gi), rpq, irpq);
            AQ = AQ + irpq;
            rQ = rQ - thq;
        }
        double wsum = 0.0, tsum = 0.0;
#pragma unroll 4
        for (int a = e0; a < e1; a++) {
            const int code = d.be_idx[a];
            const int l = code >> 1, side = code & 1;
            const size_t li = (size_t)l * T + t;
            const int kp = side ? B_FPJI : B_FPIJ, kq = side ? B_FQJI : B_FQIJ;
            const int kw = side ? B_WJ : B_WI, ka = side ? B_AJ : B_AI;
            const double thp = TH(kp, li), thq = TH(kq, li), thw = TH(kw, li), tha = TH(ka, li);
            AP = AP + irpq;
            rP = rP + thp;
            AQ = AQ + irpq;
            rQ = rQ + thq;
            wsum = wsum + thw;
            tsum = tsum + tha;
        }
        const double thw = wsum / (double)ne;
        const double aw = (double)ne * rva;
        const double alw = -d.gs[i], bew = d.bs[i];
        AP = AP + alw * alw / aw;
        AQ = AQ + bew * bew / aw;
        C = C + alw * bew / aw;
        rP = rP - alw * thw;
        rQ = rQ - bew * thw;
        const double det = AP * AQ - C * C;
        const double muP = (rP * AQ - C * rQ) / det;
        const double muQ = (AP * rQ - C * rP) / det;
        if (!isfinite(muP + muQ)) report_nonfinite(d, K_BUS, i, t);
        // ---- generator copies and their rows (each gen: all loads, then the updates, then the stores)
        for (int a = g0; a < g1; a++) {
            const size_t gi = (size_t)d.bg_idx[a] * T + t;
            const bool rc = has_next;
            const double pg = d.p[gi], qg = d.q[gi], pbo = d.pbar[gi], qbo = d.qbar[gi];
            double zp = ZG(G_GP, gi), yp = YG(G_GP, gi), lp = LG(G_GP, gi);
            double zq = ZG(G_GQ, gi), yq = YG(G_GQ, gi), lq = LG(G_GQ, gi);
            double phn = 0.0, zr = 0.0, yr = 0.0, lr = 0.0;
            if (rc) {
                phn = d.ph[gi + 1];
                zr = ZG(G_RC, gi + 1);
                yr = YG(G_RC, gi + 1);
                lr = LG(G_RC, gi + 1);
            }
            const double tgp = pg + zp + over_rho<STRICT>(yp, rpq, irpq);
            double th, aa;
            if (rc) {
                const double trc = phn + zr + over_rho<STRICT>(yr, rpq, irpq);
                th = (tgp + trc) * 0.5;
                aa = 2.0 * rpq;
            } else {
                th = tgp;
                aa = rpq;
            }
            const double pb = th + muP / aa;
            const double thq = qg + zq + over_rho<STRICT>(yq, rpq, irpq);
            const double qb = thq + over_rho<STRICT>(muQ, rpq, irpq);
            zy_s<STRICT>(pg - pb, rpq, ibpq, c.bpq, zp, yp, lp, pending, beta_lam, lmax, pb - pbo, acc);
            zy_s<STRICT>(qg - qb, rpq, ibpq, c.bpq, zq, yq, lq, pending, beta_lam, lmax, qb - qbo, acc);
            if (rc) zy_s<STRICT>(phn - pb, rpq, ibpq, c.bpq, zr, yr, lr, pending, beta_lam, lmax, pb - pbo, acc);
            d.pbar[gi] = pb;
            d.qbar[gi] = qb;
            ZG(G_GP, gi) = zp;
            YG(G_GP, gi) = yp;
            ZG(G_GQ, gi) = zq;
            YG(G_GQ, gi) = yq;
            if (pending) {
                LG(G_GP, gi) = lp;
                LG(G_GQ, gi) = lq;
            }
            if (rc) {
                ZG(G_RC, gi + 1) = zr;
                YG(G_RC, gi + 1) = yr;
                if (pending) LG(G_RC, gi + 1) = lr;
            }
        }
        double wb = thw + (alw * muP + bew * muQ) / aw;
        if (d.variant & 2) {   // NEXT-3 variant 2 (R47): SPEC's clip of wbar to the voltage box
            const double vl = d.vmin[i] * d.vmin[i], vh = d.vmax[i] * d.vmax[i];
            wb = wb < vl ? vl : (wb > vh ? vh : wb);
        }
        // NEXT-3 variant 8 (R51): no angle rows, thetabar is not a variable (kept at its start value)
        const double tb = (d.variant & 8) ? tbo : ((i == d.ref_bus) ? 0.0 : tsum / (double)ne);
        d.wbar[k] = wb;
        d.thbar[k] = tb;
        d.bmu[0 * BT + k] = muP;
        d.bmu[1 * BT + k] = muQ;
        d.bmu[2 * BT + k] = wb - wbo;
        d.bmu[3 * BT + k] = tb - tbo;
    }
}

// Single GPU (d.fuse_rows): after its bus solve, the (i,t) thread also updates the rows of every
// branch end at bus i (they need only this bus's result; a bus is marked iff all its ends are),
// so the end rows need no kernel of their own.  Consecutive threads are consecutive t of one bus,
// so each end's row accesses stay coalesced.
template <bool STRICT>
__device__ __forceinline__ void end_rows(const Dev &d, const Ctl &c, int l, int t, int side, Acc &acc);
template <bool STRICT>
__device__ __forceinline__ void bus_end_rows(const Dev &d, const Ctl &c, int k, Acc &acc) {
    const int i = k / d.T, t = k - i * d.T;
    for (int a = d.be_ptr[i]; a < d.be_ptr[i + 1]; a++) {
        const int code = d.be_idx[a];
        end_rows<STRICT>(d, c, code >> 1, t, code & 1, acc);
    }
}

template <bool STRICT>
__global__ void BUS_BOUNDS k_bus(Dev d) {
    TL_KERNEL(K_BUS);
    if (d.st->done) return;
    const Ctl c(d);
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    Acc acc;
    const bool own = k < d.B_own * d.T && own_t(d, k % d.T);   // (time cut: owned periods only)
    const bool marked = own && d.bmark[k] == c.stamp;
    if (own && !marked) {
        bus_solve<STRICT>(d, c, k, acc);
        if (d.fuse_rows) bus_end_rows<STRICT>(d, c, k, acc);
    }
    block_compact(marked ? 1 : 0, &k, d.lbus, d.lbus_cnt, BUS_THREADS);   // the late bus list
    block_reduce_store(acc, d.part_bus);
}

// The four rows of branch end (l, side) at period t -- flow copies fbar = tauhat - mu/rho_pq,
// then (7e)/(7f) for FP, FQ, W, A of that end -- need only that end's bus result.
template <bool STRICT>
__device__ __forceinline__ void end_rows(const Dev &d, const Ctl &c, int l, int t, int side, Acc &acc) {
    const int T = d.T;
    const size_t LT = (size_t)d.L * T, BT = (size_t)d.B * T;
    const size_t LTH = (size_t)(d.L + d.Lph) * T;
    const size_t k = (size_t)l * T + t;
    const int bus = side ? d.bto[l] : d.bfrom[l];
    const size_t bk = (size_t)bus * T + t;
    const int kp = side ? B_FPJI : B_FPIJ, kq = side ? B_FQJI : B_FQIJ;
    const int kw = side ? B_WJ : B_WI, ka = side ? B_AJ : B_AI;
    const int rows[4] = {kp, kq, kw, ka};
    // every load first (no store in between: one round of memory latency, not four)
    const double muP = d.bmu[0 * BT + bk], muQ = d.bmu[1 * BT + bk];
    const double dwb = d.bmu[2 * BT + bk], dtb = d.bmu[3 * BT + bk];
    const double wb = d.wbar[bk], tb = d.thbar[bk];
    const double thp = TH(kp, k), thq = TH(kq, k), pbo = FB(kp, k), qbo = FB(kq, k);
    const double fp = FX(kp, k), fq = FX(kq, k), xw = XX(side ? 1 : 0, k), xa = XX(side ? 3 : 2, k);
    double z[4], y[4], lam[4];
#pragma unroll
    for (int r = 0; r < 4; r++) {
        z[r] = ZB(rows[r], k);
        y[r] = YB(rows[r], k);
        lam[r] = LB(rows[r], k);
    }
    const double pb = thp + over_rho<STRICT>(-muP, c.rpq, c.irpq);
    const double qb = thq + over_rho<STRICT>(-muQ, c.rpq, c.irpq);
    zy_s<STRICT>(fp - pb, c.rpq, c.ibpq, c.bpq, z[0], y[0], lam[0], c.pending, c.beta_lam, c.lmax, pb - pbo, acc);
    zy_s<STRICT>(fq - qb, c.rpq, c.ibpq, c.bpq, z[1], y[1], lam[1], c.pending, c.beta_lam, c.lmax, qb - qbo, acc);
    zy_s<STRICT>(xw - wb, c.rva, c.ibva, c.bva, z[2], y[2], lam[2], c.pending, c.beta_lam, c.lmax, dwb, acc);
    if (!(d.variant & 8))   // R51: without angle rows their z, y, lambda stay 0
        zy_s<STRICT>(xa - tb, c.rva, c.ibva, c.bva, z[3], y[3], lam[3], c.pending, c.beta_lam, c.lmax, dtb, acc);
    if (!isfinite(nf0(z[0]) + nf0(z[1]) + nf0(z[2]) + nf0(z[3]) + nf0(y[0]) + nf0(y[1]) + nf0(y[2]) + nf0(y[3])))
        report_nonfinite(d, K_ROWS, l, t);
    FB(kp, k) = pb;
    FB(kq, k) = qb;
#pragma unroll
    for (int r = 0; r < 4; r++) {
        ZB(rows[r], k) = z[r];
        YB(rows[r], k) = y[r];
        if (c.pending) LB(rows[r], k) = lam[r];
    }
    (void)LTH;
    (void)LT;
}

// k_rows (early): one thread per (l,t), the ends whose bus is not marked (coalesced row
// arrays, as k_branch); the marked ends are done by k_rows_late.
template <bool STRICT>
__global__ void ROWS_BOUNDS k_rows(Dev d) {
    TL_KERNEL(K_ROWS);
    if (d.st->done) return;
    const Ctl c(d);
    // virtual blocks: with a capped grid (UCAC_ROWS_BPSM) each block takes blocks vb, vb + grid, ...
    // of the full launch, each with its own list slot range and partial slot -- the same lists and
    // partials, so the same bits, in fewer SM slots (room for k_bus_late when the AL tail ends)
    for (int vb = blockIdx.x; vb < d.nblk_rows; vb += gridDim.x) {
        if (vb != (int)blockIdx.x) __syncthreads();   // shared scratch of the previous pass
        const int k = vb * blockDim.x + threadIdx.x;
        Acc acc;
        int items[2], ni = 0;
        if (k < d.L * d.T && own_t(d, k % d.T)) {
            const int l = k / d.T, t = k - l * d.T;
            if (d.rmark[0][k] != c.stamp) end_rows<STRICT>(d, c, l, t, 0, acc);
            else items[ni++] = k << 1;
            if (d.rmark[1][k] != c.stamp) end_rows<STRICT>(d, c, l, t, 1, acc);
            else items[ni++] = (k << 1) | 1;
        }
        block_compact(ni, items, d.lrow, d.lrow_cnt, 2 * ROWS_THREADS, vb);   // the late end list
        block_reduce_store(acc, d.part_rows, vb);
    }
}

// Late phase (after the AL tail): k_bus_late solves the marked bus-periods, k_rows_late updates
// the marked ends (k_bus_late: 1024-thread blocks, few partial slots, so the final fold is short;
// k_rows_late: 256-thread blocks, one wave grid-striding over (l,t)).
// Single GPU: k_rows_late is the last kernel of the iteration (final = 1).
template <bool STRICT>
__global__ void __launch_bounds__(LBUS_THREADS) k_bus_late(Dev d) {
    pdl_wait();
    TL_KERNEL(K_BUS_LATE);
    if (d.st->done) return;
    extern __shared__ int pre[];   // [nblk_bus + 1] offsets of the compacted bus lists
    Acc acc;
    const int n = block_offsets(d.lbus_cnt, d.nblk_bus, pre);
    if ((int)(blockIdx.x * blockDim.x) < n) {   // the control values (two divisions) only with work
        const Ctl c(d);
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
            const int k = list_item(pre, d.nblk_bus, d.lbus, BUS_THREADS, j);
            bus_solve<STRICT>(d, c, k, acc);
            if (d.fuse_rows) bus_end_rows<STRICT>(d, c, k, acc);
        }
    }
    // fused rows: this is the iteration's last kernel and does the final fold; otherwise its
    // partials are folded by k_rows_late's last block, after its own (no last-block fold here, on
    // the critical path between the AL tail and the late rows)
    if (d.fuse_rows) kernel_tail(d, acc, d.part_lbus, RK_BUS_LATE, true);
    else block_reduce_store(acc, d.part_lbus);
}

// k_fold_early: the block partials of k_bus, k_ubar and k_rows (in that order) -> rec_part[RK_EARLY]
#ifndef UCAC_FOLD_BLOCKS
#define UCAC_FOLD_BLOCKS 64
#endif
constexpr int FOLD_BLOCKS = UCAC_FOLD_BLOCKS, FOLD_THREADS = 256;
__global__ void __launch_bounds__(FOLD_THREADS) k_fold_early(Dev d) {
    TL_KERNEL(K_FOLD);
    if (d.st->done) return;
    const int nb = d.nblk_bus, nu = d.nblk_ubar, nr = d.nblk_rows, n = nb + nu + nr;
    const int chunk = (n + FOLD_BLOCKS - 1) / FOLD_BLOCKS;
    const int j0 = min(n, (int)blockIdx.x * chunk), j1 = min(n, j0 + chunk);
    __shared__ double grp[FOLD_THREADS / NPART][NPART];
    const int k = threadIdx.x % NPART, g = threadIdx.x / NPART, ng = FOLD_THREADS / NPART;
    double v = 0.0;
    // FOLD_BATCH loads in flight, folded in slot order (as fold_slots)
    for (int j = j0 + g; j < j1; j += FOLD_BATCH * ng) {
        double a[FOLD_BATCH];
#pragma unroll
        for (int u = 0; u < FOLD_BATCH; u++) {
            const int jj = j + u * ng;
            const double *p = jj < nb ? d.part_bus + (size_t)jj * NPART
                            : jj < nb + nu ? d.part_ubar + (size_t)(jj - nb) * NPART
                                           : d.part_rows + (size_t)(jj - nb - nu) * NPART;
            a[u] = jj < j1 ? __ldcg(p + k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < FOLD_BATCH; u++)
            if (j + u * ng < j1) v = fold(k, v, a[u]);
    }
    grp[g][k] = v;
    __syncthreads();
    if (threadIdx.x < NPART) {
        double w = grp[0][threadIdx.x];
        for (int q = 1; q < ng; q++) w = fold(threadIdx.x, w, grp[q][threadIdx.x]);
        d.part_efold[(size_t)blockIdx.x * NPART + threadIdx.x] = w;
        __threadfence();
    }
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(d.kdone + RK_EARLY, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (threadIdx.x == 0) d.kdone[RK_EARLY] = 0;
    fold_slots(d.part_efold, gridDim.x, d.rec_part + RK_EARLY * NPART);
}

template <bool STRICT>
__global__ void __launch_bounds__(LROWS_THREADS) k_rows_late(Dev d, int final) {
    pdl_wait();
    TL_KERNEL(K_ROWS_LATE);
    if (d.st->done) return;
    extern __shared__ int pre[];   // [nblk_rows + 1] offsets of the compacted end lists
    Acc acc;
    const int n = block_offsets(d.lrow_cnt, d.nblk_rows, pre);
    if ((int)(blockIdx.x * blockDim.x) < n) {
        const Ctl c(d);
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
            const int code = list_item(pre, d.nblk_rows, d.lrow, 2 * ROWS_THREADS, j);
            const int k = code >> 1, l = k / d.T, t = k - l * d.T;
            end_rows<STRICT>(d, c, l, t, code & 1, acc);
        }
    }
    if (store_partial_last(acc, d.part_lrows, d.kdone + RK_ROWS_LATE)) {
        fold_slots(d.part_lbus, d.nblk_lbus, d.rec_part + RK_BUS_LATE * NPART);   // k_bus_late's partials
        fold_slots(d.part_lrows, gridDim.x, d.rec_part + RK_ROWS_LATE * NPART);
        if (final) {
            __threadfence();
            final_fold(d);
        }
    }
}

// ------------------------------------------------------------------------- (7c) ubar
__device__ __forceinline__ double clamp01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

__device__ __forceinline__ void solve_small(int nf, double A[3][3], const double *b, double *x) {
    if (nf == 1) {
        x[0] = b[0] / A[0][0];
        return;
    }
    if (nf == 2) {
        double det = A[0][0] * A[1][1] - A[0][1] * A[1][0];
        x[0] = (b[0] * A[1][1] - A[0][1] * b[1]) / det;
        x[1] = (A[0][0] * b[1] - b[0] * A[1][0]) / det;
        return;
    }
    double det = A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1]) - A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0]) +
                 A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
    for (int k = 0; k < 3; k++) {
        double M[3][3];
        for (int i = 0; i < 3; i++)
            for (int j = 0; j < 3; j++) M[i][j] = (j == k) ? b[i] : A[i][j];
        double dk = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) - M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                    M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
        x[k] = dk / det;
    }
}

// exact box-QP over [0,1]^n, n <= 3, by the 3^n activity states: candidates
// [c0, c1) of the enumeration, first minimum kept (best, bidx); boxqp3 runs all of them
__device__ __forceinline__ int boxqp3_ncand(int n) { return n == 3 ? 27 : (n == 2 ? 9 : 3); }
__device__ void boxqp3_range(int n, int m, const double (*c)[3], const double *e, int c0, int c1, double *v,
                             double &best, int &bidx) {
    double H[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, bb[3] = {0, 0, 0};
    for (int i = 0; i < n; i++) {
        for (int j = 0; j < n; j++) {
            double s = 0.0;
            for (int k = 0; k < m; k++) s = s + c[k][i] * c[k][j];
            H[i][j] = s;
        }
        double s = 0.0;
        for (int k = 0; k < m; k++) s = s + c[k][i] * e[k];
        bb[i] = s;
    }
    best = INFINITY;
    bidx = 0x7fffffff;
    for (int i = 0; i < n; i++) v[i] = 0.0;
    for (int idx = c0; idx < c1; idx++) {
        int st[3], r = idx;
        for (int i = 0; i < n; i++) {
            st[i] = r % 3;
            r /= 3;
        }
        double vv[3] = {0, 0, 0};
        int fi[3], nf = 0;
        for (int i = 0; i < n; i++) {
            if (st[i] == 0) fi[nf++] = i;
            else vv[i] = (st[i] == 1) ? 0.0 : 1.0;
        }
        if (nf > 0) {
            double A[3][3], rhs[3], sol[3];
            for (int a = 0; a < nf; a++) {
                double s = bb[fi[a]];
                for (int j = 0; j < n; j++)
                    if (st[j] != 0) s = s - H[fi[a]][j] * vv[j];
                rhs[a] = s;
                for (int b2 = 0; b2 < nf; b2++) A[a][b2] = H[fi[a]][fi[b2]];
            }
            solve_small(nf, A, rhs, sol);
            for (int a = 0; a < nf; a++) vv[fi[a]] = sol[a];
        }
        for (int i = 0; i < n; i++) vv[i] = clamp01(vv[i]);
        double obj = 0.0;
        for (int k = 0; k < m; k++) {
            double rr = e[k];
            for (int i = 0; i < n; i++) rr = rr - c[k][i] * vv[i];
            obj = obj + 0.5 * rr * rr;
        }
        if (obj < best) {
            best = obj;
            bidx = idx;
            for (int i = 0; i < n; i++) v[i] = vv[i];
        }
    }
}
// The same enumeration with the problem size fixed at compile time: every loop unrolls, the
// activity states, the free index lists and the reduced systems become constants and registers
// (boxqp3_range's runtime n, m keep them in local memory, a ~30-cycle dependent access each), and
// the 3^N independent candidates interleave.  Identical operations in identical order (this unit
// builds with -fmad=false and IEEE division), so the pick and its bits are boxqp3_range's.
template <int N, int M>
__device__ __forceinline__ void boxqp3_fixed(const double (*c)[3], const double *e, double *v) {
    double H[3][3], bb[3];
#pragma unroll
    for (int i = 0; i < N; i++) {
#pragma unroll
        for (int j = 0; j < N; j++) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < M; k++) s = s + c[k][i] * c[k][j];
            H[i][j] = s;
        }
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < M; k++) s = s + c[k][i] * e[k];
        bb[i] = s;
    }
    double best = INFINITY;
#pragma unroll
    for (int i = 0; i < 3; i++) v[i] = 0.0;
    constexpr int NC = N == 3 ? 27 : (N == 2 ? 9 : 3);
#pragma unroll
    for (int idx = 0; idx < NC; idx++) {
        int st[3] = {0, 0, 0}, r = idx;
#pragma unroll
        for (int i = 0; i < N; i++) {
            st[i] = r % 3;
            r /= 3;
        }
        double vv[3] = {0, 0, 0};
        int fi[3] = {0, 0, 0}, nf = 0;
#pragma unroll
        for (int i = 0; i < N; i++) {
            if (st[i] == 0) fi[nf++] = i;
            else vv[i] = (st[i] == 1) ? 0.0 : 1.0;
        }
        if (nf > 0) {
            double A[3][3], rhs[3], sol[3];
#pragma unroll
            for (int a = 0; a < 3; a++) {
                if (a >= nf) break;
                double s = bb[fi[a]];
#pragma unroll
                for (int j = 0; j < N; j++)
                    if (st[j] != 0) s = s - H[fi[a]][j] * vv[j];
                rhs[a] = s;
#pragma unroll
                for (int b2 = 0; b2 < 3; b2++)
                    if (b2 < nf) A[a][b2] = H[fi[a]][fi[b2]];
            }
            solve_small(nf, A, rhs, sol);
#pragma unroll
            for (int a = 0; a < 3; a++)
                if (a < nf) vv[fi[a]] = sol[a];
        }
#pragma unroll
        for (int i = 0; i < N; i++) vv[i] = clamp01(vv[i]);
        double obj = 0.0;
#pragma unroll
        for (int k = 0; k < M; k++) {
            double rr = e[k];
#pragma unroll
            for (int i = 0; i < N; i++) rr = rr - c[k][i] * vv[i];
            obj = obj + 0.5 * rr * rr;
        }
        if (obj < best) {
            best = obj;
#pragma unroll
            for (int i = 0; i < N; i++) v[i] = vv[i];
        }
    }
}
#ifndef UCAC_UBAR_FIXED
#define UCAC_UBAR_FIXED 1
#endif
__device__ void boxqp3(int n, int m, const double (*c)[3], const double *e, double *v) {
    double best;
    int bidx;
    boxqp3_range(n, m, c, e, 0, boxqp3_ncand(n), v, best, bidx);
}
// UBAR_LANES consecutive lanes per (g, group) split the enumeration into contiguous candidate
// ranges; each keeps its first minimum, and the (objective, index) combine -- smaller objective,
// then smaller index -- returns the sequential enumeration's pick bit for bit (as k_genx does)
#ifndef UCAC_UBAR_LANES
#define UCAC_UBAR_LANES 1   // measured (eager, pegase T=48): 1 lane 38.6 us, 2 lanes 54.6, 4 lanes 66.4 -- the
                            // per-thread chain shrinks but 2-4x the threads (and their loads) run in 2-4 waves
#endif
constexpr int UBAR_LANES = UCAC_UBAR_LANES;
__device__ void boxqp3_lanes(int n, int m, const double (*c)[3], const double *e, double *v, int sub,
                             unsigned mask) {
    const int nc = boxqp3_ncand(n);
    v[0] = v[1] = v[2] = 0.0;
    const int c0 = (nc * sub + UBAR_LANES - 1) / UBAR_LANES, c1 = (nc * (sub + 1) + UBAR_LANES - 1) / UBAR_LANES;
    double best;
    int bidx;
    boxqp3_range(n, m, c, e, c0, c1, v, best, bidx);
#pragma unroll
    for (int o = 1; o < UBAR_LANES; o <<= 1) {
        const double ob = __shfl_xor_sync(mask, best, o);
        const int oi = __shfl_xor_sync(mask, bidx, o);
        const double o0 = __shfl_xor_sync(mask, v[0], o), o1 = __shfl_xor_sync(mask, v[1], o),
                     o2 = __shfl_xor_sync(mask, v[2], o);
        if (ob < best || (ob == best && oi < bidx)) {
            best = ob;
            bidx = oi;
            v[0] = o0;
            v[1] = o1;
            v[2] = o2;
        }
    }
}

// LIT: the literal Eq. 5f ramp-down row (variant bit 16, R52), a separate instantiation so the
// default kernel carries none of its code
template <bool LIT>
__global__ void UBAR_BOUNDS k_ubar(Dev d) {
    TL_KERNEL(K_UBAR);
    if (d.st->done) return;
    const int T = d.T;
    const size_t GT = (size_t)d.G * T;
    // UBAR_LANES consecutive lanes per (g, group); the group's lanes are all in or all out of range
    const int k4 = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = k4 / UBAR_LANES, sub = k4 % UBAR_LANES;
    const unsigned mask = __ballot_sync(0xffffffffu, k < d.G * T && own_t(d, k % T));
    const double ruc = d.ruc;
    const double beta_lam = d.st->beta_lam, lmax = d.lambda_max, bpr = d.st->beta + ruc;
    const int pending = d.st->pending_outer;
    Acc acc;
    if (k < d.G * T && own_t(d, k % T)) {   // whole lane groups in or out (the shuffle mask above)
        const int g = k / T, t = k - g * T;
        const int tg = tglob(d, t);
        const size_t i = (size_t)k;
        const double Pm = d.pmin[g], PM = d.pmax[g], Qm = d.qmin[g], QM = d.qmax[g];
        const double RDn = d.rdn[g], SDn = d.sdn[g], RUp = d.rup[g], SUp = d.sup[g];
        const int u0 = d.u0[g];
        // old group values (iterate l) -- the x-step's shifted bounds use them (R19)
        const double on_o = d.ub_on[i], sd_o = d.ub_sd[i], su_o = d.ub_su[i];
        const double onp_o = tg == 0 ? (double)u0 : d.ub_on[i - 1];
        const int ut = d.u[i], up = tg == 0 ? u0 : d.u[i - 1];
        const int sdt = up > ut, sut = ut > up;
        const double p = d.p[i], q = d.q[i], ph = d.ph[i];
        // slacks (x-variables of 7b) recomputed exactly as the x-step defines them
        const double bpl = Pm * on_o - ZG(G_PL, i) - YG(G_PL, i) / ruc;
        const double bpu = PM * on_o - ZG(G_PU, i) - YG(G_PU, i) / ruc;
        const double bql = Qm * on_o - ZG(G_QL, i) - YG(G_QL, i) / ruc;
        const double bqu = QM * on_o - ZG(G_QU, i) - YG(G_QU, i) / ruc;
        // NEXT-3 variant 16 (R52): the literal Eq. 5f ramp-down row R_D ubar^on_{t-1} + S_D ubar^su_t
        constexpr bool lit = LIT;
        const double brl = lit ? -RDn * onp_o - SDn * su_o - ZG(G_RD, i) - YG(G_RD, i) / ruc
                               : -RDn * on_o - SDn * sd_o - ZG(G_RD, i) - YG(G_RD, i) / ruc;
        const double dd = p - ph;
        const double spl = fmax(0.0, p - bpl), spu = fmax(0.0, bpu - p);
        const double sql = fmax(0.0, q - bql), squ = fmax(0.0, bqu - q);
        const double srd = fmax(0.0, dd - brl);
        double cm[9][3], e[9];
        int m = 0;
#define ROW(a0, a1, a2, ev)   \
    do {                      \
        cm[m][0] = (a0);      \
        cm[m][1] = (a1);      \
        cm[m][2] = (a2);      \
        e[m++] = (ev);        \
    } while (0)
        ROW(1.0, 0.0, 0.0, (double)ut + ZG(G_DON, i) + YG(G_DON, i) / ruc);
        ROW(0.0, 1.0, 0.0, (double)sdt + ZG(G_DSD, i) + YG(G_DSD, i) / ruc);
        ROW(Pm, 0.0, 0.0, (p - spl) + ZG(G_PL, i) + YG(G_PL, i) / ruc);
        ROW(PM, 0.0, 0.0, (p + spu) + ZG(G_PU, i) + YG(G_PU, i) / ruc);
        ROW(Qm, 0.0, 0.0, (q - sql) + ZG(G_QL, i) + YG(G_QL, i) / ruc);
        ROW(QM, 0.0, 0.0, (q + squ) + ZG(G_QU, i) + YG(G_QU, i) / ruc);
        if (!lit) ROW(-RDn, -SDn, 0.0, (dd - srd) + ZG(G_RD, i) + YG(G_RD, i) / ruc);
        int n = 2;
        int sun = 0;
        double pn = 0.0, phn = 0.0, sru_n = 0.0, su_on = 0.0, srd_n = 0.0;
        const bool nxt = tg < d.Tg - 1;
        if (nxt) {
            const size_t j = i + 1;
            const int un = d.u[j];
            sun = un > ut;
            pn = d.p[j];
            phn = d.ph[j];
            su_on = d.ub_su[j];
            const double bru_n = RUp * on_o + SUp * su_on - ZG(G_RU, j) - YG(G_RU, j) / ruc;
            sru_n = fmax(0.0, bru_n - (pn - phn));
            ROW(0.0, 0.0, 1.0, (double)sun + ZG(G_DSU, j) + YG(G_DSU, j) / ruc);
            ROW(RUp, 0.0, SUp, ((pn - phn) + sru_n) + ZG(G_RU, j) + YG(G_RU, j) / ruc);
            if (lit) {   // RD_{t+1} = (d - s) + R_D ubar^on_t + S_D ubar^su_{t+1}: this group's row
                const double brl_n = -RDn * on_o - SDn * su_on - ZG(G_RD, j) - YG(G_RD, j) / ruc;
                srd_n = fmax(0.0, (pn - phn) - brl_n);
                ROW(-RDn, 0.0, -SDn, ((pn - phn) - srd_n) + ZG(G_RD, j) + YG(G_RD, j) / ruc);
            }
            n = 3;
        }
#undef ROW
        // z, y, lambda of the group's rows, all loaded before any store (a store to one row array
        // would otherwise order every later row's loads behind it)
        const int rk[7] = {G_DON, G_DSD, G_PL, G_PU, G_QL, G_QU, G_RD};
        double zr[10], yr[10], lr[10];
#pragma unroll
        for (int q2 = 0; q2 < 7; q2++) {
            zr[q2] = ZG(rk[q2], i);
            yr[q2] = YG(rk[q2], i);
            lr[q2] = LG(rk[q2], i);
        }
        if (nxt) {
            zr[7] = ZG(G_DSU, i + 1); yr[7] = YG(G_DSU, i + 1); lr[7] = LG(G_DSU, i + 1);
            zr[8] = ZG(G_RU, i + 1);  yr[8] = YG(G_RU, i + 1);  lr[8] = LG(G_RU, i + 1);
            if (lit) { zr[9] = ZG(G_RD, i + 1); yr[9] = YG(G_RD, i + 1); lr[9] = LG(G_RD, i + 1); }
        }
        double v[3];
        if (UBAR_LANES == 1 && UCAC_UBAR_FIXED) {   // (the row arrays stay in registers)
            if (nxt) boxqp3_fixed<3, 9>(cm, e, v);
            else boxqp3_fixed<2, lit ? 6 : 7>(cm, e, v);
        } else {
            boxqp3_lanes(n, m, cm, e, v, sub, mask);
        }
        if (sub == 0) {
        {
            double chk = nf0(v[0]) + nf0(v[1]) + nf0(v[2]);
#pragma unroll
            for (int q2 = 0; q2 < 9; q2++)
                if (q2 < m) chk = chk + nf0(e[q2]);
            if (!isfinite(chk)) report_nonfinite(d, K_UBAR, g, t);
        }
        const double on_n = v[0], sd_n = v[1];
        // rows of the group with the new ubar (r = x-part - c'ubar)
        const double don = on_n - on_o, dsd = sd_n - sd_o;
        zy_vals_div((double)ut - on_n, ruc, bpr, zr[0], yr[0], lr[0], pending, beta_lam, lmax, don, acc);
        zy_vals_div((double)sdt - sd_n, ruc, bpr, zr[1], yr[1], lr[1], pending, beta_lam, lmax, dsd, acc);
        zy_vals_div((p - spl) - Pm * on_n, ruc, bpr, zr[2], yr[2], lr[2], pending, beta_lam, lmax, Pm * don, acc);
        zy_vals_div((p + spu) - PM * on_n, ruc, bpr, zr[3], yr[3], lr[3], pending, beta_lam, lmax, PM * don, acc);
        zy_vals_div((q - sql) - Qm * on_n, ruc, bpr, zr[4], yr[4], lr[4], pending, beta_lam, lmax, Qm * don, acc);
        zy_vals_div((q + squ) - QM * on_n, ruc, bpr, zr[5], yr[5], lr[5], pending, beta_lam, lmax, QM * don, acc);
        if (!lit)
            zy_vals_div((dd - srd) + RDn * on_n + SDn * sd_n, ruc, bpr, zr[6], yr[6], lr[6], pending, beta_lam, lmax,
                    RDn * don + SDn * dsd, acc);
        double su_n = 0.0;
        if (nxt) {
            su_n = v[2];
            const double dsu = su_n - su_on;
            zy_vals_div((double)sun - su_n, ruc, bpr, zr[7], yr[7], lr[7], pending, beta_lam, lmax, dsu, acc);
            zy_vals_div(((pn - phn) + sru_n) - RUp * on_n - SUp * su_n, ruc, bpr, zr[8], yr[8], lr[8], pending, beta_lam,
                    lmax, RUp * don + SUp * dsu, acc);
            if (lit)
                zy_vals_div(((pn - phn) - srd_n) + RDn * on_n + SDn * su_n, ruc, bpr, zr[9], yr[9], lr[9], pending,
                        beta_lam, lmax, RDn * don + SDn * dsu, acc);
        }
        d.ub_on[i] = on_n;
        d.ub_sd[i] = sd_n;
        // (literal Eq. 5f: RD_t belongs to group t-1, whose thread stores it; not stored here)
#pragma unroll
        for (int q2 = 0; q2 < 7; q2++) {
            if (lit && q2 == 6) continue;
            ZG(rk[q2], i) = zr[q2];
            YG(rk[q2], i) = yr[q2];
            if (pending) LG(rk[q2], i) = lr[q2];
        }
        if (nxt) {
            d.ub_su[i + 1] = su_n;
            ZG(G_DSU, i + 1) = zr[7]; YG(G_DSU, i + 1) = yr[7];
            ZG(G_RU, i + 1) = zr[8];  YG(G_RU, i + 1) = yr[8];
            if (pending) {
                LG(G_DSU, i + 1) = lr[7];
                LG(G_RU, i + 1) = lr[8];
            }
            if (lit) {
                ZG(G_RD, i + 1) = zr[9]; YG(G_RD, i + 1) = yr[9];
                if (pending) LG(G_RD, i + 1) = lr[9];
            }
        }
        if (tg == 0) {
            // group 0 = (ubar^su_1): rows D_SU_1, RU_1 (ubar^on_0 := u0, R4)
            const double bru = RUp * onp_o + SUp * su_o - ZG(G_RU, i) - YG(G_RU, i) / ruc;
            const double sru = fmax(0.0, bru - dd);
            double c1[3][3] = {{1.0, 0.0, 0.0}, {SUp, 0.0, 0.0}, {-SDn, 0.0, 0.0}};
            double e1[3];
            e1[0] = (double)sut + ZG(G_DSU, i) + YG(G_DSU, i) / ruc;
            e1[1] = (dd + sru) - RUp * (double)u0 + ZG(G_RU, i) + YG(G_RU, i) / ruc;
            // literal Eq. 5f (R52): RD_1 = (d - s) + R_D u0 + S_D ubar^su_1 joins this group
            e1[2] = ((dd - srd) + RDn * (double)u0) + ZG(G_RD, i) + YG(G_RD, i) / ruc;
            double v1[3];
            if (UCAC_UBAR_FIXED) boxqp3_fixed<1, lit ? 3 : 2>(c1, e1, v1);
            else boxqp3(1, lit ? 3 : 2, c1, e1, v1);
            d.ub_su[i] = v1[0];
            const double dsu = v1[0] - su_o;
            zy_row_div((double)sut - v1[0], ruc, bpr, &ZG(G_DSU, i), &YG(G_DSU, i), &LG(G_DSU, i), pending, beta_lam, lmax, dsu,
                   acc);
            zy_row_div((dd + sru) - RUp * (double)u0 - SUp * v1[0], ruc, bpr, &ZG(G_RU, i), &YG(G_RU, i), &LG(G_RU, i),
                   pending, beta_lam, lmax, SUp * dsu, acc);
            if (lit)
                zy_row_div((dd - srd) + RDn * (double)u0 + SDn * v1[0], ruc, bpr, &ZG(G_RD, i), &YG(G_RD, i), &LG(G_RD, i),
                       pending, beta_lam, lmax, SDn * dsu, acc);
        }
        // objective, Eq. 1a with f^OPF = c2 (S p)^2 + c1 S p and f^UC (R13)
        const double Sp = d.S * p;
        acc.v[P_OBJ] = d.c2[g] * Sp * Sp + d.c1[g] * Sp + d.c0[g] * (double)ut + d.csu[g] * (double)sut +
                       d.csd[g] * (double)sdt;
        }   // sub == 0
    }
    block_reduce_store(acc, d.part_ubar);
}

// ------------------------------------------------------------------------- S8 / S9
// S8 norms, inner test and the outer (lambda, beta) decision from a reduction record (R20-R22)
__device__ void finalize_status(const Dev &d, const double *rec) {
    DevStatus *st = d.st;
    st->primal_inf = rec[R_PINF];
    st->rz_inf = rec[R_RZINF];
    st->rz_2 = sqrt(rec[R_RZ2]);
    st->z_inf = rec[R_ZINF];
    st->z_2 = sqrt(rec[R_Z2]);
    st->dual_inf = rec[R_DINF];
    st->objective = rec[R_OBJ];
    st->tron_iters += (unsigned long long)rec[R_C0];
    st->tron_capped += (unsigned long long)rec[R_C1];
    st->al_active += (unsigned long long)rec[R_C2];
    st->al_capped += (unsigned long long)rec[R_C3];
    st->al_tron_iters += (unsigned long long)rec[R_C4];
    st->inner_total += 1;
    st->inner_since += 1;
    if ((rec[R_BAD] != 0.0 || !isfinite(rec[R_RZ2]) || !isfinite(rec[R_OBJ])) && st->err_kernel == 0) {
        st->err_kernel = 1 + K_ROWS_LATE;
        st->err_iter = (int)st->inner_total;
    }
    st->pending_outer = 0;
    if (d.outer_enabled && st->inner_since >= d.inner_min) {
        const double thr = fmax(d.eps_inner_abs, 1e-2 / (double)st->outer_k);
        if (st->rz_inf <= thr || st->inner_since >= d.inner_cap) {
            const double zn = st->z_2;
            st->pending_outer = 1;
            st->beta_lam = st->beta;
            if (st->outer_k > 1 && zn > d.theta * st->znorm_prev) st->beta = fmin(d.tau * st->beta, d.beta_max);
            st->znorm_prev = zn;
            st->outer_k += 1;
            st->inner_since = 0;
        }
    }
    // the iteration's record (ucac_history) and the divergence detector: primal_inf >
    // factor x its value div_window iterations earlier ends the call (done), once per run
    {
        const long long it = st->inner_total;
        double *hr = d.hist + (size_t)((it - 1) % HIST_CAP) * HIST_FIELDS;
        hr[0] = st->primal_inf;
        hr[1] = st->dual_inf;
        hr[2] = st->z_inf;
        hr[3] = st->z_2;
        hr[4] = st->objective;
        hr[5] = st->beta;
        if (d.div_window > 0 && it > d.div_window && st->diverged_iter == 0) {
            const double old = d.hist[(size_t)((it - 1 - d.div_window) % HIST_CAP) * HIST_FIELDS];
            if (st->primal_inf > d.div_factor * old) {   // (false against a NaN: an emptied history)
                st->diverged_iter = (int)it;
                st->done = 1;
            }
        }
    }
    if (st->stop_on_primal && st->primal_inf <= st->primal_target) st->done = 1;
}

// S8/S9 on the (all-rank) reduction record
__global__ void k_finalize(Dev d) {
    if (d.st->done) return;
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double rec[NREC];
        for (int c = 0; c < NREC; c++) rec[c] = d.rec[c];
        finalize_status(d, rec);
    }
}

// ---- halo exchange: pack/unpack of the cut ends' tauhat and of bus results
__device__ __forceinline__ int to_kind(int kk) { return kk == 0 ? B_FPJI : (kk == 1 ? B_FQJI : (kk == 2 ? B_WJ : B_AJ)); }
// Early exchanges (before the AL tail ends): every cut branch-period's to-end tauhat with a flag
// that the (l,t) went to the AL queue (its tauhat is then not final: the to-bus and its ends go late
// on the owner), and every export bus-period's results with a flag that it is late (its ghost copies
// and the local ends at them go late).  Late exchanges carry the final values of the flagged ones.
__global__ void k_pack_tau_early(Dev d) {
    if (d.st->done) return;
    const int T = d.T;
    const size_t LTH = (size_t)(d.L + d.Lph) * T;
    const unsigned stamp = mark_stamp(d);
    const int n = d.ncut * T;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int t = k % T, c = k / T;
        const size_t lk = (size_t)d.cut_local[c] * T + t;
        const bool q = d.qmark[lk] == stamp;
        double *o = d.xsend1 + (size_t)c * 5 * T;
        for (int kk = 0; kk < 4; kk++) o[kk * T + t] = q ? 0.0 : TH(to_kind(kk), lk);
        o[4 * T + t] = q ? 1.0 : 0.0;
    }
}
__global__ void k_unpack_tau_early(Dev d) {
    if (d.st->done) return;
    const int T = d.T;
    const size_t LTH = (size_t)(d.L + d.Lph) * T;
    const unsigned stamp = mark_stamp(d);
    const int n = d.Lph * T;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int t = k % T, p = k / T;
        const double *src = d.xrecv1 + (size_t)d.phantom_src[p] * 5 * T;
        const size_t pk = (size_t)(d.L + p) * T + t;
        if (src[4 * T + t] != 0.0) {
            // a remote AL solve at this owned bus: the bus and every end at it go late (as k_branch marks)
            d.qmark[pk] = stamp;
            const int bus = d.phantom_bus[p];
            d.bmark[(size_t)bus * T + t] = stamp;
            for (int a = d.be_ptr[bus]; a < d.be_ptr[bus + 1]; a++) {
                const int code = d.be_idx[a];
                d.rmark[code & 1][(size_t)(code >> 1) * T + t] = stamp;
            }
        } else {
            for (int kk = 0; kk < 4; kk++) TH(to_kind(kk), pk) = src[kk * T + t];
        }
    }
}
__global__ void k_pack_bus_early(Dev d) {
    if (d.st->done) return;
    const int T = d.T;
    const size_t BT = (size_t)d.B * T;
    const unsigned stamp = mark_stamp(d);
    const int n = d.nexport * T;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int t = k % T, e = k / T;
        const size_t bk = (size_t)d.export_local[e] * T + t;
        const bool late = d.bmark[bk] == stamp;
        double *o = d.xsend2 + (size_t)e * 7 * T;
        for (int f = 0; f < 6; f++) o[f * T + t] = late ? 0.0 : (f < 4 ? d.bmu[f * BT + bk] : (f == 4 ? d.wbar[bk] : d.thbar[bk]));
        o[6 * T + t] = late ? 1.0 : 0.0;
    }
}
__global__ void k_unpack_bus_early(Dev d) {
    if (d.st->done) return;
    const int T = d.T;
    const size_t BT = (size_t)d.B * T;
    const unsigned stamp = mark_stamp(d);
    const int n = d.nghost * T;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int t = k % T, gb = k / T;
        const double *src = d.xrecv2 + (size_t)d.ghost_src[gb] * 7 * T;
        const size_t bk = (size_t)(d.B_own + gb) * T + t;
        if (src[6 * T + t] != 0.0) {
            // late on its owner: the local ends at this ghost bus wait for the late exchange
            d.bmark[bk] = stamp;
            for (int a = d.ghost_eptr[gb]; a < d.ghost_eptr[gb + 1]; a++) {
                const int code = d.ghost_eidx[a];
                d.rmark[code & 1][(size_t)(code >> 1) * T + t] = stamp;
            }
        } else {
            for (int f = 0; f < 4; f++) d.bmu[f * BT + bk] = src[f * T + t];
            d.wbar[bk] = src[4 * T + t];
            d.thbar[bk] = src[5 * T + t];
        }
    }
}
// late: the final tauhat of the queued cut ends / the results of the late export buses
__global__ void k_pack_tau(Dev d) {
    if (d.st->done) return;
    const int T = d.T;
    const size_t LTH = (size_t)(d.L + d.Lph) * T;
    const int n = d.ncut * 4 * T;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int t = k % T, kk = (k / T) % 4, c = k / (4 * T);
        d.xsend3[k] = TH(to_kind(kk), (size_t)d.cut_local[c] * T + t);
    }
}
__global__ void k_unpack_tau(Dev d) {
    if (d.st->done) return;
    const int T = d.T;
    const size_t LTH = (size_t)(d.L + d.Lph) * T;
    const unsigned stamp = mark_stamp(d);
    const int n = d.Lph * 4 * T;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int t = k % T, kk = (k / T) % 4, p = k / (4 * T);
        const size_t pk = (size_t)(d.L + p) * T + t;
        if (d.qmark[pk] == stamp) TH(to_kind(kk), pk) = d.xrecv3[((size_t)d.phantom_src[p] * 4 + kk) * T + t];
    }
}
__global__ void k_pack_bus(Dev d) {
    if (d.st->done) return;
    const int T = d.T;
    const size_t BT = (size_t)d.B * T;
    const int n = d.nexport * 6 * T;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int t = k % T, f = (k / T) % 6, e = k / (6 * T);
        const size_t bk = (size_t)d.export_local[e] * T + t;
        d.xsend4[k] = f < 4 ? d.bmu[f * BT + bk] : (f == 4 ? d.wbar[bk] : d.thbar[bk]);
    }
}
__global__ void k_unpack_bus(Dev d) {
    if (d.st->done) return;
    const int T = d.T;
    const size_t BT = (size_t)d.B * T;
    const unsigned stamp = mark_stamp(d);
    const int n = d.nghost * 6 * T;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int t = k % T, f = (k / T) % 6, gb = k / (6 * T);
        const size_t bk = (size_t)(d.B_own + gb) * T + t;
        if (d.bmark[bk] != stamp) continue;   // early ghost: already delivered by the early exchange
        const double v = d.xrecv4[((size_t)d.ghost_src[gb] * 6 + f) * T + t];
        if (f < 4) d.bmu[f * BT + bk] = v;
        else if (f == 4) d.wbar[bk] = v;
        else d.thbar[bk] = v;
    }
}

// materialise a pending lambda update (before a state dump)
__global__ void k_apply_outer(Dev d) {
    if (!d.st->pending_outer) return;
    const double bl = d.st->beta_lam, lmax = d.lambda_max;
    const size_t ng = (size_t)NGROW * d.G * d.T, nbr = (size_t)NBROW * d.L * d.T;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < ng + nbr; k += (size_t)gridDim.x * blockDim.x) {
        double *lp = k < ng ? d.lg + k : d.lb + (k - ng);
        const double z = k < ng ? d.zg[k] : d.zb[k - ng];
        const double v = *lp + bl * z;
        *lp = v < -lmax ? -lmax : (v > lmax ? lmax : v);
    }
}
__global__ void k_clear_pending(Dev d) { d.st->pending_outer = 0; }

}  // namespace

int nblk_bus(int B, int T) { return (B * T + BUS_THREADS - 1) / BUS_THREADS; }
int nblk_ubar(int G, int T) { return (G * T * UBAR_LANES + UBAR_THREADS - 1) / UBAR_THREADS; }
int nblk_rows(int L, int T) { return (L * T + ROWS_THREADS - 1) / ROWS_THREADS; }

// launch priority of the sweep chain k_bus -> k_rows -> (fold) -> k_rows_late, the critical path
// once the AL tail ends first; k_ubar, off that path, keeps normal priority
#ifndef UCAC_SWEEP_PRIO
#define UCAC_SWEEP_PRIO 0   // 1 measured equal (0.1879 vs 0.1877 ms)
#endif
#ifndef UCAC_UBAR_PRIO
#define UCAC_UBAR_PRIO 1
#endif
static int sm_count();
template <typename... KArgs>
static void launch_sweep(bool hi, void (*k)(KArgs...), dim3 g, dim3 b, cudaStream_t s, KArgs... args) {
    if (hi) launch_hi_prio(k, g, b, 0, s, args...);
    else k<<<g, b, 0, s>>>(args...);
}
void launch_bus(const Dev &d, cudaStream_t s) {
    launch_sweep(UCAC_SWEEP_PRIO, d.strict ? k_bus<true> : k_bus<false>, dim3(d.nblk_bus), dim3(BUS_THREADS), s, d);
}
// k_rows grid: UCAC_ROWS_BPSM blocks per SM (virtual blocks; 0 = one block per 128 (l,t)).  At 112
// registers 4 blocks fit an SM; 3 leave one block's registers free, so k_bus_late starts as soon as
// the AL tail ends instead of after k_rows' last blocks (timeline: 131 -> 124 us; step 0.1676 ->
// 0.1656 ms, iterate bitwise unchanged; 2: 0.1699, 4: 0.1670)
// Only where the row sweep is short next to the AL tail: at T = 168 (L*T = 770 k) the sweep is
// HBM-bound and the full grid is faster (k_rows 85.0 -> 72.3 us, step 0.4023/0.4040 -> 0.3988/0.4002
// ms), so the cap applies up to L*T = UCAC_ROWS_BPSM_MAX_LT (pegase T = 48: 220 k).
#ifndef UCAC_ROWS_BPSM
#define UCAC_ROWS_BPSM 3
#endif
#ifndef UCAC_ROWS_BPSM_MAX_LT
#define UCAC_ROWS_BPSM_MAX_LT 400000
#endif
void launch_rows(const Dev &d, cudaStream_t s) {
    const bool cap = UCAC_ROWS_BPSM > 0 && (long long)d.L * d.T <= UCAC_ROWS_BPSM_MAX_LT;
    const int grid = cap ? std::min(d.nblk_rows, UCAC_ROWS_BPSM * sm_count()) : d.nblk_rows;
    launch_sweep(UCAC_SWEEP_PRIO, d.strict ? k_rows<true> : k_rows<false>, dim3(grid), dim3(ROWS_THREADS), s, d);
}
#ifndef UCAC_LATE_PRIO
#define UCAC_LATE_PRIO 1
#endif
// The late kernels: one wave, grid-striding over the compacted lists (their items are ~10 % of the
// bus-periods / ends); at high launch priority, so they take SM slots ahead of pending early
// blocks when the AL tail ends.  Dynamic shared memory: the offsets of the early blocks' lists.
static int sm_count() {
    static const int n = [] {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        return std::max(1, sms);
    }();
    return n;
}
template <typename K>
static size_t late_smem(K k, int nsrc) {
    const size_t b = (size_t)(nsrc + 1) * sizeof(int);
    if (b > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b);
    return b;
}
void launch_bus_late(const Dev &d, cudaStream_t s) {
    auto k = d.strict ? k_bus_late<true> : k_bus_late<false>;
    launch_ex(k, dim3(d.nblk_lbus), dim3(LBUS_THREADS), late_smem(k, d.nblk_bus), s,
              UCAC_SWEEP_PRIO || UCAC_LATE_PRIO, (pdl_mask() & 2) != 0, d);
}
void launch_rows_late(const Dev &d, cudaStream_t s, int final) {
    auto k = d.strict ? k_rows_late<true> : k_rows_late<false>;
    launch_ex(k, dim3(d.nblk_lrows), dim3(LROWS_THREADS), late_smem(k, d.nblk_rows), s,
              UCAC_SWEEP_PRIO || UCAC_LATE_PRIO, (pdl_mask() & 4) != 0, d, final);
}
#ifndef UCAC_LATE_WAVES
#define UCAC_LATE_WAVES 1
#endif
// late grids: enough threads for every marked item of a wave-sized grid (at most one per SM x
// UCAC_LATE_WAVES), never more blocks than the full range would need
int nblk_lbus(int n) { return std::max(1, std::min((n + LBUS_THREADS - 1) / LBUS_THREADS, sm_count() * UCAC_LATE_WAVES)); }
int nblk_lrows(int n) { return std::max(1, std::min((n + LROWS_THREADS - 1) / LROWS_THREADS, 2 * sm_count() * UCAC_LATE_WAVES)); }
int fold_blocks() { return FOLD_BLOCKS; }
void launch_fold_early(const Dev &d, cudaStream_t s) { k_fold_early<<<FOLD_BLOCKS, FOLD_THREADS, 0, s>>>(d); }
void launch_ubar(const Dev &d, cudaStream_t s) {
    if (d.variant & 16) launch_sweep(UCAC_UBAR_PRIO, k_ubar<true>, dim3(d.nblk_ubar), dim3(UBAR_THREADS), s, d);
    else launch_sweep(UCAC_UBAR_PRIO, k_ubar<false>, dim3(d.nblk_ubar), dim3(UBAR_THREADS), s, d);
}
void launch_finalize(const Dev &d, cudaStream_t s) { k_finalize<<<1, 32, 0, s>>>(d); }
static int xgrid(int n) { return std::max(1, std::min(296, (n + 255) / 256)); }
void launch_pack_tau(const Dev &d, cudaStream_t s) { k_pack_tau<<<xgrid(d.ncut * 4 * d.T), 256, 0, s>>>(d); }
void launch_pack_tau_early(const Dev &d, cudaStream_t s) { k_pack_tau_early<<<xgrid(d.ncut * d.T), 256, 0, s>>>(d); }
void launch_unpack_tau_early(const Dev &d, cudaStream_t s) { k_unpack_tau_early<<<xgrid(d.Lph * d.T), 256, 0, s>>>(d); }
void launch_pack_bus_early(const Dev &d, cudaStream_t s) { k_pack_bus_early<<<xgrid(d.nexport * d.T), 256, 0, s>>>(d); }
void launch_unpack_bus_early(const Dev &d, cudaStream_t s) { k_unpack_bus_early<<<xgrid(d.nghost * d.T), 256, 0, s>>>(d); }
void launch_unpack_tau(const Dev &d, cudaStream_t s) { k_unpack_tau<<<xgrid(d.Lph * 4 * d.T), 256, 0, s>>>(d); }
void launch_pack_bus(const Dev &d, cudaStream_t s) { k_pack_bus<<<xgrid(d.nexport * 6 * d.T), 256, 0, s>>>(d); }
void launch_unpack_bus(const Dev &d, cudaStream_t s) { k_unpack_bus<<<xgrid(d.nghost * 6 * d.T), 256, 0, s>>>(d); }
void launch_apply_outer(const Dev &d, cudaStream_t s) {
    k_apply_outer<<<296, 256, 0, s>>>(d);
    k_clear_pending<<<1, 1, 0, s>>>(d);
}

}  // namespace ucac
