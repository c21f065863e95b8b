// k_gen.cu -- steps (7a) (k_gen: UC DP, warp per generator) and (7b, generator part; k_genx:
// thread per (g,t)), plus the cold-start kernel (S0) and the
// standalone batched DP.  Compiled with -fmad=false: every expression here is evaluated
// in the operation order written (the same order the oracle's definition uses), so that the
// integer DP decisions ("stay" when c_stay <= c_switch) are taken on the same fp64
// values and commitment schedules match the oracle bit for bit.
//
// Mapping: one WARP per generator.  Lanes = periods for the stage costs L_t(a,b), the
// switch-window sums and the per-(g,t) generator x-update (t = lane, lane+32, ...); the
// backward recursion of Algorithm 2 is inherently sequential in t and runs on
// lane 0 over a shared-memory table (O(T) with 2 states).
#include <mutex>
#include <algorithm>

#include "ucac_dev.cuh"

namespace ucac {
namespace {

// phi_v(b) = y (b - ubar + z) + rho/2 (b - ubar + z)^2 (duplicate rows; R18)
__device__ __forceinline__ double phi(double b, double ub, double y, double z, double rho) {
    double e = (b - ub) + z;
    return y * e + 0.5 * rho * e * e;
}

// stage cost L^UC_{g,t}(a,b) with su, sd inferred, f^UC (R13)
__device__ __forceinline__ double stage_cost(int a, int b, double c0, double csu, double csd, double rho,
                                             const double *ub, const double *y, const double *z) {
    int su = b > a, sd = a > b;
    double v = c0 * (double)b;
    v = v + csu * (double)su;
    v = v + csd * (double)sd;
    v = v + phi((double)b, ub[0], y[0], z[0], rho);
    v = v + phi((double)su, ub[1], y[1], z[1], rho);
    v = v + phi((double)sd, ub[2], y[2], z[2], rho);
    return v;
}

#ifndef UCAC_DP_PAIR
#define UCAC_DP_PAIR 1   // the batch kernel (NEXT-1): two instances per warp
#endif
struct DpSmem {
    double *L;     // [T*4 + 4] L_t(a, b) at t*4 + 2a + b; once the switch costs are formed, the
                   // continuation costs c_t(s) (Eq. 10-11) reuse the dead off-diagonal slots,
                   // c_t(s) at t*4 + 1 + s (t = 0..T): per instance ~8.3 KB at T = 168, not 13.7
    double *acc;   // [T*2] switch cost before continuation: L_t(s,n) + sum_{t'} L_{t'}(n,n)
    unsigned *sw;  // [2][W], W = ceil(T/32): decision "switch" of state s at t, bit t%32 of word t/32
    int8_t *u;     // [T]
};
#define DP_C(t, st) s.L[(t) * 4 + 1 + (st)]

__host__ __device__ inline size_t dp_smem_bytes(int T) {
    const size_t W = (size_t)(T + 31) / 32;
    const size_t b = (size_t)(T * 4 + 4 + T * 2) * 8 + 2 * W * 4 + (size_t)T;
    return (b + 15) & ~(size_t)15;   // every warp's slice 16-byte aligned (the paired loads below)
}

__device__ __forceinline__ DpSmem dp_carve(char *base, int T) {
    DpSmem s;
    s.L = (double *)base;
    s.acc = s.L + T * 4 + 4;
    s.sw = (unsigned *)(s.acc + T * 2);
    s.u = (int8_t *)(s.sw + 2 * ((T + 31) / 32));
    return s;
}

// Algorithm 2 on a warp; s.L must be filled.  Returns the optimal cost on lane 0.
// Lanes: the switch costs of every (t, state) (Eq. 11's window sums).  Lane 0: the backward
// recursion (Eq. 10-11, P:380's tie rule) and the traceback.  The recursion's short
// dependency c_{t+1} is carried in registers, the window ends are computed, the switch costs of a
// period come in one 16-byte shared load, the decisions are kept as bits and the
// traceback jumps to the next switch bit instead of stepping through every period -- the same
// additions and comparisons in the same order, so the same costs and decisions bit for bit.
// GL: lanes per instance (32: a warp; 16: two instances per warp, each half running its own serial
// part on its lane 0 -- the batch kernel, whose single active lane left the issue slots idle);
// act = false: this group has no instance but still meets the warp's __syncwarp.
template <int GL = 32>
__device__ double dp_warp(const DpSmem &s, int T, int TU, int TD, int u0, int hold, bool act = true) {
    const int lane = threadIdx.x & (GL - 1);
    for (int t = lane; t < T && act; t += GL) {
#pragma unroll
        for (int st = 0; st < 2; st++) {
            int n = 1 - st;
            int m = n ? TU : TD;
            int e = t + m - 1;
            if (e > T - 1) e = T - 1;
            double acc = s.L[t * 4 + st * 2 + n];
            for (int tt = t + 1; tt <= e; tt++) acc = acc + s.L[tt * 4 + n * 2 + n];   // R17
            s.acc[t * 2 + st] = acc;
        }
    }
    __syncwarp();
    double cost = 0.0;
    if (lane == 0 && act) {
        DP_C(T, 0) = 0.0;   // (L's off-diagonal slots are dead from here on)
        DP_C(T, 1) = 0.0;
        const int W = (T + 31) / 32;
        double cn0 = 0.0, cn1 = 0.0;   // c_{t+1}(off), c_{t+1}(on)
        unsigned b0 = 0u, b1 = 0u;
        for (int t = T - 1; t >= 0; t--) {
            const int e0 = min(t + TU - 1, T - 1), e1 = min(t + TD - 1, T - 1);   // R15 clip
            const double2 a2 = *reinterpret_cast<const double2 *>(s.acc + t * 2);
            const double sw0 = a2.x + DP_C(e0 + 1, 1);                                    // Eq. 11
            const double sw1 = a2.y + DP_C(e1 + 1, 0);
            const double stay0 = s.L[t * 4 + 0] + cn0, stay1 = s.L[t * 4 + 3] + cn1;      // Eq. 10
            const bool k0 = stay0 <= sw0, k1 = stay1 <= sw1;
            cn0 = k0 ? stay0 : sw0;
            cn1 = k1 ? stay1 : sw1;
            DP_C(t, 0) = cn0;
            DP_C(t, 1) = cn1;
            b0 |= (k0 ? 0u : 1u) << (t & 31);
            b1 |= (k1 ? 0u : 1u) << (t & 31);
            if ((t & 31) == 0) {
                s.sw[t >> 5] = b0;
                s.sw[W + (t >> 5)] = b1;
                b0 = b1 = 0u;
            }
        }
        for (int t = 0; t < hold; t++) {                                                  // R14
            s.u[t] = (int8_t)u0;
            cost = cost + s.L[t * 4 + u0 * 3];
        }
        cost = cost + DP_C(hold, u0);
        int t = hold, st = u0;
        while (t < T) {
            // the next period from t on where state st switches (the stay run before it keeps st)
            const unsigned *bits = s.sw + st * W;
            int tp = T;
            for (int w = t >> 5; w < W; w++) {
                unsigned word = bits[w];
                if (w == (t >> 5)) word &= ~0u << (t & 31);
                if (word) {
                    tp = (w << 5) + __ffs(word) - 1;
                    break;
                }
            }
            for (int tt = t; tt < tp; tt++) s.u[tt] = (int8_t)st;
            if (tp >= T) break;
            const int e = min(tp + (st == 0 ? TU : TD) - 1, T - 1);   // the forced window of 1 - st
            for (int tt = tp; tt <= e; tt++) s.u[tt] = (int8_t)(1 - st);
            st = 1 - st;
            t = e + 1;
        }
    }
    __syncwarp();
    return cost;
}

// ---------------------------------------------------------------- generator x-update (S2)
struct GenIn {
    int first;
    double c2S2, c1S, rpq, ruc, tp, tq, tph, p0, bpl, bpu, bql, bqu, brl, bru, pL, pU, qL, qU;
};

__device__ __forceinline__ double gen_obj_p(const GenIn &g, double p, double ph) {
    double v = g.c2S2 * p * p + g.c1S * p;
    double e = p - g.tp;
    v = v + 0.5 * g.rpq * e * e;
    if (!g.first) {
        e = ph - g.tph;
        v = v + 0.5 * g.rpq * e * e;
    }
    e = p - g.bpl;
    if (e < 0.0) v = v + 0.5 * g.ruc * e * e;
    e = p - g.bpu;
    if (e > 0.0) v = v + 0.5 * g.ruc * e * e;
    double dd = p - ph;
    e = dd - g.brl;
    if (e < 0.0) v = v + 0.5 * g.ruc * e * e;
    e = dd - g.bru;
    if (e > 0.0) v = v + 0.5 * g.ruc * e * e;
    return v;
}
__device__ __forceinline__ double gen_obj_q(const GenIn &g, double q) {
    double e = q - g.tq;
    double v = 0.5 * g.rpq * e * e;
    e = q - g.bql;
    if (e < 0.0) v = v + 0.5 * g.ruc * e * e;
    e = q - g.bqu;
    if (e > 0.0) v = v + 0.5 * g.ruc * e * e;
    return v;
}

// exact minimiser of the generator subproblem by activity-pattern enumeration
// (DESIGN.md 5.2): 16 patterns x {p free} + 4 ramp patterns x {p = pL, p = pU}.
__device__ void gen_solve(const GenIn &g, double &po, double &qo, double &pho) {
    double best = INFINITY, bp = g.pL, bph = g.first ? g.p0 : g.tph;
    if (g.first) {
        for (int pat = 0; pat < 16; pat++) {
            int alo = pat & 1, ahi = (pat >> 1) & 1, rlo = (pat >> 2) & 1, rhi = (pat >> 3) & 1;
            double den = 2.0 * g.c2S2 + g.rpq;
            double num = -g.c1S + g.rpq * g.tp;
            if (alo) { den = den + g.ruc; num = num + g.ruc * g.bpl; }
            if (ahi) { den = den + g.ruc; num = num + g.ruc * g.bpu; }
            if (rlo) { den = den + g.ruc; num = num + g.ruc * (g.brl + g.p0); }
            if (rhi) { den = den + g.ruc; num = num + g.ruc * (g.bru + g.p0); }
            double p = num / den;
            if (p >= g.pL && p <= g.pU) {
                double v = gen_obj_p(g, p, g.p0);
                if (v < best) { best = v; bp = p; }
            }
        }
        double v = gen_obj_p(g, g.pL, g.p0);
        if (v < best) { best = v; bp = g.pL; }
        v = gen_obj_p(g, g.pU, g.p0);
        if (v < best) { best = v; bp = g.pU; }
        bph = g.p0;
    } else {
        for (int pat = 0; pat < 16; pat++) {
            int alo = pat & 1, ahi = (pat >> 1) & 1, rlo = (pat >> 2) & 1, rhi = (pat >> 3) & 1;
            double A = 2.0 * g.c2S2 + g.rpq;
            double b1 = -g.c1S + g.rpq * g.tp;
            if (alo) { A = A + g.ruc; b1 = b1 + g.ruc * g.bpl; }
            if (ahi) { A = A + g.ruc; b1 = b1 + g.ruc * g.bpu; }
            double R = 0.0, rb = 0.0;
            if (rlo) { R = R + g.ruc; rb = rb + g.ruc * g.brl; }
            if (rhi) { R = R + g.ruc; rb = rb + g.ruc * g.bru; }
            b1 = b1 + rb;
            double b2 = g.rpq * g.tph - rb;
            double det = (A + R) * (g.rpq + R) - R * R;
            double p = (b1 * (g.rpq + R) + R * b2) / det;
            double ph = ((A + R) * b2 + R * b1) / det;
            if (p >= g.pL && p <= g.pU) {
                double v = gen_obj_p(g, p, ph);
                if (v < best) { best = v; bp = p; bph = ph; }
            }
        }
        for (int kb = 0; kb < 2; kb++) {
            double pb = kb ? g.pU : g.pL;
            for (int pat = 0; pat < 4; pat++) {
                int rlo = pat & 1, rhi = (pat >> 1) & 1;
                double R = 0.0, rb = 0.0;
                if (rlo) { R = R + g.ruc; rb = rb + g.ruc * g.brl; }
                if (rhi) { R = R + g.ruc; rb = rb + g.ruc * g.bru; }
                double ph = (g.rpq * g.tph - rb + R * pb) / (g.rpq + R);
                double v = gen_obj_p(g, pb, ph);
                if (v < best) { best = v; bp = pb; bph = ph; }
            }
        }
    }
    double bestq = INFINITY, bq = g.qL;
    for (int pat = 0; pat < 4; pat++) {
        int lo = pat & 1, hi = (pat >> 1) & 1;
        double den = g.rpq, num = g.rpq * g.tq;
        if (lo) { den = den + g.ruc; num = num + g.ruc * g.bql; }
        if (hi) { den = den + g.ruc; num = num + g.ruc * g.bqu; }
        double qq = num / den;
        if (qq >= g.qL && qq <= g.qU) {
            double v = gen_obj_q(g, qq);
            if (v < bestq) { bestq = v; bq = qq; }
        }
    }
    double v = gen_obj_q(g, g.qL);
    if (v < bestq) { bestq = v; bq = g.qL; }
    v = gen_obj_q(g, g.qU);
    if (v < bestq) { bestq = v; bq = g.qU; }
    po = bp;
    qo = bq;
    pho = bph;
}

// The same enumeration split over GENX_LANES consecutive lanes: lane `sub` evaluates the
// candidates with index = sub (mod GENX_LANES), each exactly as gen_solve does, and the lanes
// combine (value, index) keeping the smallest value and, on ties, the smallest index -- which is
// the candidate gen_solve's sequential "if (v < best)" keeps.  Bitwise the same result with
// GENX_LANES x the threads per (g,t).
#ifndef UCAC_GENX_LANES
#define UCAC_GENX_LANES 2   // measured: 1 lane 20.8 us, 2 lanes 16.8, 4 lanes 20.9, 8 lanes 25.1 (eager)
#endif
constexpr int GENX_LANES = UCAC_GENX_LANES;
__device__ __forceinline__ void lane_min(double &v, int &idx, double &a, double &b) {
    const unsigned m = __activemask();   // whole lane groups: past the end of the grid they left together
#pragma unroll
    for (int o = 1; o < GENX_LANES; o <<= 1) {
        const double v2 = __shfl_xor_sync(m, v, o, GENX_LANES);
        const int i2 = __shfl_xor_sync(m, idx, o, GENX_LANES);
        const double a2 = __shfl_xor_sync(m, a, o, GENX_LANES);
        const double b2 = __shfl_xor_sync(m, b, o, GENX_LANES);
        if (v2 < v || (v2 == v && i2 < idx)) { v = v2; idx = i2; a = a2; b = b2; }
    }
}
__device__ void gen_solve_lanes(const GenIn &g, int sub, double &po, double &qo, double &pho) {
    // candidate index: 0..15 the interior patterns, then the bound candidates in gen_solve's order
    double best = INFINITY, bp = g.pL, bph = g.first ? g.p0 : g.tph;
    int bidx = 1 << 30;
    const int ncand = g.first ? 18 : 24;
    for (int c = sub; c < ncand; c += GENX_LANES) {
        double v = NAN, p = 0.0, ph = 0.0;
        bool ok = false;
        if (c < 16) {
            const int pat = c;
            const int alo = pat & 1, ahi = (pat >> 1) & 1, rlo = (pat >> 2) & 1, rhi = (pat >> 3) & 1;
            if (g.first) {
                double den = 2.0 * g.c2S2 + g.rpq;
                double num = -g.c1S + g.rpq * g.tp;
                if (alo) { den = den + g.ruc; num = num + g.ruc * g.bpl; }
                if (ahi) { den = den + g.ruc; num = num + g.ruc * g.bpu; }
                if (rlo) { den = den + g.ruc; num = num + g.ruc * (g.brl + g.p0); }
                if (rhi) { den = den + g.ruc; num = num + g.ruc * (g.bru + g.p0); }
                p = num / den;
                ph = g.p0;
            } else {
                double A = 2.0 * g.c2S2 + g.rpq;
                double b1 = -g.c1S + g.rpq * g.tp;
                if (alo) { A = A + g.ruc; b1 = b1 + g.ruc * g.bpl; }
                if (ahi) { A = A + g.ruc; b1 = b1 + g.ruc * g.bpu; }
                double R = 0.0, rb = 0.0;
                if (rlo) { R = R + g.ruc; rb = rb + g.ruc * g.brl; }
                if (rhi) { R = R + g.ruc; rb = rb + g.ruc * g.bru; }
                b1 = b1 + rb;
                double b2 = g.rpq * g.tph - rb;
                double det = (A + R) * (g.rpq + R) - R * R;
                p = (b1 * (g.rpq + R) + R * b2) / det;
                ph = ((A + R) * b2 + R * b1) / det;
            }
            ok = p >= g.pL && p <= g.pU;
        } else if (g.first) {
            p = c == 16 ? g.pL : g.pU;
            ph = g.p0;
            ok = true;
        } else {
            const int kb = (c - 16) >> 2, pat = (c - 16) & 3;
            p = kb ? g.pU : g.pL;
            const int rlo = pat & 1, rhi = (pat >> 1) & 1;
            double R = 0.0, rb = 0.0;
            if (rlo) { R = R + g.ruc; rb = rb + g.ruc * g.brl; }
            if (rhi) { R = R + g.ruc; rb = rb + g.ruc * g.bru; }
            ph = (g.rpq * g.tph - rb + R * p) / (g.rpq + R);
            ok = true;
        }
        if (ok) v = gen_obj_p(g, p, ph);
        if (v < best) { best = v; bidx = c; bp = p; bph = ph; }
    }
    lane_min(best, bidx, bp, bph);
    if (g.first) bph = g.p0;
    double bestq = INFINITY, bq = g.qL;
    int qidx = 1 << 30;
    for (int c = sub; c < 6; c += GENX_LANES) {
        double qq, v = NAN;
        if (c < 4) {
            const int lo = c & 1, hi = (c >> 1) & 1;
            double den = g.rpq, num = g.rpq * g.tq;
            if (lo) { den = den + g.ruc; num = num + g.ruc * g.bql; }
            if (hi) { den = den + g.ruc; num = num + g.ruc * g.bqu; }
            qq = num / den;
            if (qq >= g.qL && qq <= g.qU) v = gen_obj_q(g, qq);
        } else {
            qq = c == 4 ? g.qL : g.qU;
            v = gen_obj_q(g, qq);
        }
        if (v < bestq) { bestq = v; qidx = c; bq = qq; }
    }
    double dummy = 0.0;
    lane_min(bestq, qidx, bq, dummy);
    po = bp;
    qo = bq;
    pho = bph;
}

#define ZG(k, i) d.zg[(size_t)(k) * GT + (i)]
#define YG(k, i) d.yg[(size_t)(k) * GT + (i)]

// tail = 0: the iteration's own (7a), skipped when the previous iteration's tail launch already
// computed it (u_next valid).  tail = 1: launched right after k_ubar, it computes the NEXT
// iteration's (7a) -- its inputs (ubar, y, z of the duplicate rows, p) are final once k_ubar has
// run -- so the DP overlaps the rest of this iteration.  The schedule becomes state
// only when k_genx adopts u_next, after the done check, so a stopped run is unchanged.
__global__ void __launch_bounds__(128) k_gen(Dev d, int tail) {
    TL_KERNEL(K_GEN);
    if (d.st->done || d.uc_fixed) return;   // uc_fixed: the schedule is held (NEXT-2)
    if (!tail && *((volatile unsigned *)d.unext_ok)) return;
    extern __shared__ __align__(16) char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x * (blockDim.x >> 5) + warp;
    if (g >= d.G) return;
    const int T = d.T;
    const size_t GT = (size_t)d.G * T;
    DpSmem s = dp_carve(smem + (size_t)warp * dp_smem_bytes(T), T);
    const double ruc = d.ruc;
    // ---- (7a): stage costs on iterate l (ubar^l, y^l, z^l of the duplicate rows)
    const double c0 = d.c0[g], csu = d.csu[g], csd = d.csd[g];
    for (int t = lane; t < T; t += 32) {
        const size_t i = (size_t)g * T + t;
        double ub[3] = {d.ub_on[i], d.ub_su[i], d.ub_sd[i]};
        double yy[3] = {YG(G_DON, i), YG(G_DSU, i), YG(G_DSD, i)};
        double zz[3] = {ZG(G_DON, i), ZG(G_DSU, i), ZG(G_DSD, i)};
        if (!isfinite(nf0(ub[0]) + nf0(ub[1]) + nf0(ub[2]) + nf0(yy[0]) + nf0(yy[1]) + nf0(yy[2]) + nf0(zz[0]) +
                      nf0(zz[1]) + nf0(zz[2])))
            report_nonfinite(d, K_GEN, g, t);
#pragma unroll
        for (int a = 0; a < 2; a++)
#pragma unroll
            for (int b = 0; b < 2; b++) s.L[t * 4 + a * 2 + b] = stage_cost(a, b, c0, csu, csd, ruc, ub, yy, zz);
        // NEXT-4(a) ramp-aware DP (variant bit 4, R50): no shutdown at t while the current dispatch
        // p_{t-1} exceeds the shutdown ramp S^D (Eq. 4d would be infeasible)
        if (d.variant & 4) {
            const double pprev = t == 0 ? d.p0[g] : d.p[i - 1];
            if (pprev > d.sdn[g]) s.L[t * 4 + 1 * 2 + 0] = INFINITY;
        }
    }
    __syncwarp();
    dp_warp(s, T, d.tu[g], d.td[g], d.u0[g], d.hold[g]);
    for (int t = lane; t < T; t += 32) d.u_next[(size_t)g * T + t] = s.u[t];
    if (tail && g == 0 && lane == 0) *d.unext_ok = 1u;   // read only by later launches (stream order)
}

// (7b) generator part on iterate l: one thread per (g,t) (S2)
__global__ void __launch_bounds__(128) k_genx(Dev d) {
    TL_KERNEL(K_GENX);
    if (d.st->done) return;
    const int T = d.T;
    const size_t GT = (size_t)d.G * T;
    // GENX_LANES consecutive lanes per (g,t): a group never straddles the end of the range, so
    // whole groups past it leave together and the shuffles stay within the active groups
    const int k4 = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = k4 / GENX_LANES, sub = k4 % GENX_LANES;
    if (k >= d.G * T) return;
    if (sub == 0) {
        if (!d.uc_fixed) d.u[k] = d.u_next[k];   // adopt this iteration's (7a) schedule
        if (k == 0) *d.unext_ok = 0u;              // u_next is consumed: stale for the next state
    }
    const int g = k / T, t = k - g * T;
    if (!own_t(d, t)) return;   // time cut: halo periods belong to the neighbour (the lane group leaves together)
    const int tg = tglob(d, t);
    const double ruc = d.ruc, rpq = d.rpq;
    const double S = d.S;
    GenIn in;
    in.c2S2 = d.c2[g] * S * S;
    in.c1S = d.c1[g] * S;
    in.rpq = rpq;
    in.ruc = ruc;
    in.p0 = d.p0[g];
    in.pL = fmin(0.0, d.pmin[g]);
    in.pU = d.pmax[g];
    in.qL = fmin(0.0, d.qmin[g]);
    in.qU = fmax(0.0, d.qmax[g]);
    const double pmin = d.pmin[g], pmax = d.pmax[g], qmin = d.qmin[g], qmax = d.qmax[g];
    const double rdn = d.rdn[g], sdn = d.sdn[g], rup = d.rup[g], sup = d.sup[g];
    const double u0 = (double)d.u0[g];
    const size_t i = (size_t)k;
    const double on = d.ub_on[i], su = d.ub_su[i], sd = d.ub_sd[i];
    const double onp = tg == 0 ? u0 : d.ub_on[i - 1];
    in.first = tg == 0;
    in.tp = d.pbar[i] - ZG(G_GP, i) - YG(G_GP, i) / d.rpq;
    in.tq = d.qbar[i] - ZG(G_GQ, i) - YG(G_GQ, i) / d.rpq;
    in.tph = tg == 0 ? 0.0 : d.pbar[i - 1] - ZG(G_RC, i) - YG(G_RC, i) / d.rpq;
    in.bpl = pmin * on - ZG(G_PL, i) - YG(G_PL, i) / d.ruc;
    in.bpu = pmax * on - ZG(G_PU, i) - YG(G_PU, i) / d.ruc;
    in.bql = qmin * on - ZG(G_QL, i) - YG(G_QL, i) / d.ruc;
    in.bqu = qmax * on - ZG(G_QU, i) - YG(G_QU, i) / d.ruc;
    // RD row: Eq. 4d, or the literal Eq. 5f with variant bit 16 (R52)
    in.brl = (d.variant & 16) ? -rdn * onp - sdn * su - ZG(G_RD, i) - YG(G_RD, i) / d.ruc
                              : -rdn * on - sdn * sd - ZG(G_RD, i) - YG(G_RD, i) / d.ruc;
    in.bru = rup * onp + sup * su - ZG(G_RU, i) - YG(G_RU, i) / d.ruc;
    double po, qo, pho;
    gen_solve_lanes(in, sub, po, qo, pho);
    if (sub == 0) {
        d.p[i] = po;
        d.q[i] = qo;
        d.ph[i] = pho;
        if (!isfinite(nf0(in.tp) + nf0(in.tq) + nf0(in.tph) + nf0(in.bpl) + nf0(in.bpu) + nf0(in.bql) + nf0(in.bqu) +
                      nf0(in.brl) + nf0(in.bru) + nf0(po) + nf0(qo) + nf0(pho)))
            report_nonfinite(d, K_GENX, g, t);
    }
}

// ---------------------------------------------------------------- NEXT-4(c) time cut
// (P:166-167).  Stage costs of the owned periods (the same stage_cost as k_gen), laid out
// [g][Tmax][4] for the all-gather.
__global__ void k_stage_tc(Dev d) {
    if (d.st->done || d.uc_fixed) return;
    const int T = d.T, n = d.own1 - d.own0;
    const size_t GT = (size_t)d.G * T;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < d.G * n; k += gridDim.x * blockDim.x) {
        const int g = k / n, t = d.own0 + (k - g * n);
        const size_t i = (size_t)g * T + t;
        double ub[3] = {d.ub_on[i], d.ub_su[i], d.ub_sd[i]};
        double yy[3] = {YG(G_DON, i), YG(G_DSU, i), YG(G_DSD, i)};
        double zz[3] = {ZG(G_DON, i), ZG(G_DSU, i), ZG(G_DSD, i)};
        if (!isfinite(nf0(ub[0]) + nf0(ub[1]) + nf0(ub[2]) + nf0(yy[0]) + nf0(yy[1]) + nf0(yy[2]) + nf0(zz[0]) +
                      nf0(zz[1]) + nf0(zz[2])))
            report_nonfinite(d, K_GEN, g, t);
        double *o = d.tc_stage_send + ((size_t)g * d.Tmax + (t - d.own0)) * 4;
#pragma unroll
        for (int a = 0; a < 2; a++)
#pragma unroll
            for (int b = 0; b < 2; b++) o[a * 2 + b] = stage_cost(a, b, d.c0[g], d.csu[g], d.csd[g], d.ruc, ub, yy, zz);
    }
}

// the full-horizon DP (Alg. 2) on every rank from the gathered stage costs; the schedule of the
// local periods (halos included) goes to u and u_next (k_genx's adoption is then a copy)
__global__ void __launch_bounds__(128) k_dp_tc(Dev d) {
    if (d.st->done || d.uc_fixed) return;
    extern __shared__ __align__(16) char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x * (blockDim.x >> 5) + warp;
    if (g >= d.G) return;
    const int Tg = d.Tg;
    DpSmem s = dp_carve(smem + (size_t)warp * dp_smem_bytes(Tg), Tg);
    for (int k = lane; k < Tg * 4; k += 32) {
        const int tg = k >> 2;
        int r = 0;
        while (d.tc_t0[r + 1] <= tg) r++;
        s.L[k] = __ldcg(d.tc_stage_recv + (((size_t)r * d.G + g) * d.Tmax + (tg - d.tc_t0[r])) * 4 + (k & 3));
    }
    __syncwarp();
    dp_warp(s, Tg, d.tu[g], d.td[g], d.u0[g], d.hold[g]);
    for (int t = lane; t < d.T; t += 32) {
        const int8_t v = s.u[tglob(d, t)];
        d.u[(size_t)g * d.T + t] = v;
        d.u_next[(size_t)g * d.T + t] = v;
    }
}

// p and phat of the first owned period, for the previous rank's last-period ramp rows
__global__ void k_pack_tc2(Dev d) {
    if (d.st->done) return;
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < d.G; g += gridDim.x * blockDim.x) {
        const size_t i = (size_t)g * d.T + d.own0;
        d.tc2_send[(size_t)g * 2 + 0] = d.p[i];
        d.tc2_send[(size_t)g * 2 + 1] = d.ph[i];
    }
}
__global__ void k_unpack_tc2(Dev d) {
    if (d.st->done || d.own1 >= d.T) return;   // no next rank
    const double *src = d.tc2_recv + (size_t)(d.rank + 1) * d.G * 2;
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < d.G; g += gridDim.x * blockDim.x) {
        const size_t i = (size_t)g * d.T + d.own1;
        d.p[i] = src[(size_t)g * 2 + 0];
        d.ph[i] = src[(size_t)g * 2 + 1];
    }
}
// the values this rank computed that the next rank owns or reads next iteration: ubar^on and pbar
// of the last owned period, ubar^su and the D_SU / RU / RC rows (z, y, lambda) of the next period
__global__ void k_pack_tc3(Dev d) {
    if (d.st->done || d.own1 >= d.T) return;
    const size_t GT = (size_t)d.G * d.T;
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < d.G; g += gridDim.x * blockDim.x) {
        const size_t i = (size_t)g * d.T + d.own1 - 1, j = i + 1;
        double *o = d.tc3_send + (size_t)g * 12;
        o[0] = d.ub_on[i];
        o[1] = d.pbar[i];
        o[2] = d.ub_su[j];
        const int rows[3] = {G_DSU, G_RU, G_RC};
        for (int q = 0; q < 3; q++) {
            o[3 + 3 * q] = d.zg[(size_t)rows[q] * GT + j];
            o[4 + 3 * q] = d.yg[(size_t)rows[q] * GT + j];
            o[5 + 3 * q] = d.lg[(size_t)rows[q] * GT + j];
        }
    }
}
__global__ void k_unpack_tc3(Dev d) {
    if (d.st->done || d.own0 == 0) return;   // no previous rank
    const size_t GT = (size_t)d.G * d.T;
    const double *src = d.tc3_recv + (size_t)(d.rank - 1) * d.G * 12;
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < d.G; g += gridDim.x * blockDim.x) {
        const size_t i = (size_t)g * d.T + d.own0 - 1, j = i + 1;
        const double *o = src + (size_t)g * 12;
        d.ub_on[i] = o[0];
        d.pbar[i] = o[1];
        d.ub_su[j] = o[2];
        const int rows[3] = {G_DSU, G_RU, G_RC};
        for (int q = 0; q < 3; q++) {
            d.zg[(size_t)rows[q] * GT + j] = o[3 + 3 * q];
            d.yg[(size_t)rows[q] * GT + j] = o[4 + 3 * q];
            d.lg[(size_t)rows[q] * GT + j] = o[5 + 3 * q];
        }
    }
}

__global__ void k_dp_batch(int G, int T, const double *L, const int *tu, const int *td, const int *u0,
                           const int *hold, int8_t *sched, double *cost) {
    extern __shared__ __align__(16) char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x * (blockDim.x >> 5) + warp;
    if (g >= G) return;
    // on-device inputs are not validated by the host: an out-of-range instance gets a NaN cost and
    // an all-zero schedule instead of indexing past its shared-memory slice (ucac.h ucac_dp_batch)
    if (tu[g] < 1 || tu[g] > T || td[g] < 1 || td[g] > T || hold[g] < 0 || hold[g] > T || (u0[g] != 0 && u0[g] != 1)) {
        for (int t = lane; t < T; t += 32) sched[(size_t)g * T + t] = 0;
        if (lane == 0) cost[g] = __longlong_as_double(0x7ff8000000000000ll);
        return;
    }
    DpSmem s = dp_carve(smem + (size_t)warp * dp_smem_bytes(T), T);
    for (int k = lane; k < T * 4; k += 32) s.L[k] = L[(size_t)g * T * 4 + k];
    __syncwarp();
    double c = dp_warp(s, T, tu[g], td[g], u0[g], hold[g]);
    for (int t = lane; t < T; t += 32) sched[(size_t)g * T + t] = s.u[t];
    if (lane == 0) cost[g] = c;
}
// several instances per warp (GL lanes each, UCAC_DP_PAIR): the same per-instance code and
// arithmetic.  Worth it while the block (WARPS x 32/GL instances) stays small enough for three or
// more blocks per SM; measured (G = 10^4; ms at T = 24/48/96/168): one instance per warp (4 warps)
// 0.029/0.047/0.079/0.142; 16 lanes x 4 warps 0.023/0.038/0.064/0.132; 16 x 3 0.023/0.039/0.063/
// 0.128; 16 x 2 0.024/0.037/0.063/0.129; 8 x 2 0.021/0.032/0.063/0.149; 8 x 1 0.020/0.031/0.062/
// 0.145 -- so 8 lanes x 2 warps up to T = 48 and 16 x 3 above
inline int dp_group_per(int T) { return T <= 48 ? 8 : 6; }
inline bool dp_pair_fits(int T) { return dp_smem_bytes(T) * dp_group_per(T) <= 76 * 1024; }
template <int GL, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_dp_batch_group(int G, int T, const double *L, const int *tu,
                                                              const int *td, const int *u0, const int *hold,
                                                              int8_t *sched, double *cost) {
    extern __shared__ __align__(16) char smem[];
    constexpr int PER = WARPS * (32 / GL);
    const int half = threadIdx.x / GL, lane = threadIdx.x & (GL - 1);
    const int g = blockIdx.x * PER + half;
    const bool in = g < G;
    const bool ok = in && !(tu[g] < 1 || tu[g] > T || td[g] < 1 || td[g] > T || hold[g] < 0 || hold[g] > T ||
                            (u0[g] != 0 && u0[g] != 1));
    if (in && !ok) {   // as k_dp_batch: an out-of-range instance gets a NaN cost and a zero schedule
        for (int t = lane; t < T; t += GL) sched[(size_t)g * T + t] = 0;
        if (lane == 0) cost[g] = __longlong_as_double(0x7ff8000000000000ll);
    }
    DpSmem s = dp_carve(smem + (size_t)half * dp_smem_bytes(T), T);
    if (ok)
        for (int k = lane; k < T * 4; k += GL) s.L[k] = L[(size_t)g * T * 4 + k];
    __syncwarp();
    const double c = dp_warp<GL>(s, T, ok ? tu[g] : 1, ok ? td[g] : 1, ok ? u0[g] : 0, ok ? hold[g] : 0, ok);
    if (ok) {
        for (int t = lane; t < T; t += GL) sched[(size_t)g * T + t] = s.u[t];
        if (lane == 0) cost[g] = c;
    }
}

// NEXT-2: stage costs of the repair DP, L_t(a, b) = [b != (p_t > threshold)] -- the
// Hamming distance to the thresholded multiperiod-ACOPF dispatch (SPEC warm_start_uc)
__global__ void k_hamming_costs(int n, const double *p, double threshold, double *L) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int ut = p[k] > threshold;
#pragma unroll
        for (int a = 0; a < 2; a++)
#pragma unroll
            for (int b = 0; b < 2; b++) L[(size_t)k * 4 + a * 2 + b] = (b != ut) ? 1.0 : 0.0;
    }
}

// ---------------------------------------------------------------- cold start (S0)
__global__ void k_init(Dev d, const int8_t *u_init) {
    const int T = d.T;
    const long long GT = (long long)d.G * T, LT = (long long)d.L * T, BT = (long long)d.B * T;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < GT + LT + BT;
         k += (long long)gridDim.x * blockDim.x) {
        if (k < GT) {
            const int g = (int)(k / T), t = (int)(k - (long long)g * T);
            const int tg = tglob(d, t);   // global period (time cut: local period 0 may be a halo)
            const int ut = u_init ? u_init[k] : d.u0[g];
            // (a halo period's predecessor is not local: its ubar^su/sd are never read here)
            const int up = tg == 0 ? d.u0[g] : (t == 0 ? ut : (u_init ? u_init[k - 1] : d.u0[g]));
            const double pm = 0.5 * (d.pmin[g] + d.pmax[g]);
            d.u[k] = (int8_t)ut;
            d.p[k] = pm;
            d.q[k] = 0.5 * (d.qmin[g] + d.qmax[g]);
            d.ph[k] = tg == 0 ? d.p0[g] : pm;
            d.ub_on[k] = (double)ut;
            d.ub_su[k] = ut > up ? 1.0 : 0.0;
            d.ub_sd[k] = up > ut ? 1.0 : 0.0;
            d.pbar[k] = pm;
            d.qbar[k] = d.q[k];
        } else if (k < GT + LT) {
            const long long kk = k - GT;
            const int l = (int)(kk / T);
            const int i = d.bfrom[l], j = d.bto[l];
            const double vi = 0.5 * (d.vmin[i] + d.vmax[i]), vj = 0.5 * (d.vmin[j] + d.vmax[j]);
            const double wi = vi * vi, wj = vj * vj;
            const double R = sqrt(wi * wj);
            const double C = R * cos(0.0), S = R * sin(0.0);
            const double Gii = d.y[0 * d.L + l], Gij = d.y[1 * d.L + l], Gji = d.y[2 * d.L + l], Gjj = d.y[3 * d.L + l];
            const double Bii = d.y[4 * d.L + l], Bij = d.y[5 * d.L + l], Bji = d.y[6 * d.L + l], Bjj = d.y[7 * d.L + l];
            // Eq. 2e-2h, evaluated in the oracle's order (a w_i + b w_j) + c C + d S
            const double f0 = Gii * wi + 0.0 * wj + Gij * C + Bij * S;
            const double f1 = -Bii * wi + 0.0 * wj + -Bij * C + Gij * S;
            const double f2 = 0.0 * wi + Gjj * wj + Gji * C + -Bji * S;
            const double f3 = 0.0 * wi + -Bjj * wj + -Bji * C + -Gji * S;
            const double r = d.rate[l];
            d.x[0 * LT + kk] = wi;
            d.x[1 * LT + kk] = wj;
            d.x[2 * LT + kk] = 0.0;
            d.x[3 * LT + kk] = 0.0;
            d.f[0 * LT + kk] = f0; d.f[1 * LT + kk] = f1; d.f[2 * LT + kk] = f2; d.f[3 * LT + kk] = f3;
            d.fbar[0 * LT + kk] = f0; d.fbar[1 * LT + kk] = f1; d.fbar[2 * LT + kk] = f2; d.fbar[3 * LT + kk] = f3;
            d.al[0 * LT + kk] = 0.0;
            d.al[1 * LT + kk] = 0.0;
            d.al[2 * LT + kk] = d.al_sigma0_rel * d.rpq * (r * r);
        } else {
            const long long kk = k - GT - LT;
            const int i = (int)(kk / T);
            const double v = 0.5 * (d.vmin[i] + d.vmax[i]);
            d.wbar[kk] = v * v;
            d.thbar[kk] = 0.0;
        }
    }
}

}  // namespace

static size_t gen_smem(int T, int warps) { return dp_smem_bytes(T) * warps; }

void launch_gen(const Dev &d, cudaStream_t s, int tail) {
    const int warps = 4;
    launch_hi_prio(k_gen, dim3((d.G + warps - 1) / warps), dim3(warps * 32), gen_smem(d.T, warps), s, d, tail);
}
void launch_genx(const Dev &d, cudaStream_t s) {
    launch_hi_prio(k_genx, dim3((GENX_LANES * d.G * d.T + 127) / 128), dim3(128), 0, s, d);
}

cudaError_t launch_dp_batch(int G, int T, const double *L, const int *tu, const int *td, const int *u0,
                            const int *hold, int8_t *sched, double *cost, cudaStream_t s) {
    const int warps = 4;
    if (UCAC_DP_PAIR && dp_pair_fits(T)) {
        const int per = dp_group_per(T);
        const size_t sm = dp_smem_bytes(T) * per;
        if (T <= 48)
            k_dp_batch_group<8, 2><<<(G + per - 1) / per, 64, sm, s>>>(G, T, L, tu, td, u0, hold, sched, cost);
        else
            k_dp_batch_group<16, 3><<<(G + per - 1) / per, 96, sm, s>>>(G, T, L, tu, td, u0, hold, sched, cost);
        return cudaGetLastError();
    }
    k_dp_batch<<<(G + warps - 1) / warps, warps * 32, gen_smem(T, warps), s>>>(G, T, L, tu, td, u0, hold,
                                                                                sched, cost);
    return cudaGetLastError();
}

void launch_hamming_costs(int n, const double *p, double threshold, double *L, cudaStream_t s) {
    k_hamming_costs<<<std::max(1, std::min(592, (n + 255) / 256)), 256, 0, s>>>(n, p, threshold, L);
}

void launch_init(const Dev &d, const int8_t *u_init_dev, cudaStream_t s) {
    k_init<<<296, 256, 0, s>>>(d, u_init_dev);
}

size_t gen_smem_bytes(int T) { return gen_smem(T, 4); }
void launch_stage_tc(const Dev &d, cudaStream_t s) {
    const int n = d.G * (d.own1 - d.own0);
    k_stage_tc<<<std::max(1, std::min(592, (n + 127) / 128)), 128, 0, s>>>(d);
}
void launch_dp_tc(const Dev &d, cudaStream_t s) {
    const int warps = 4;
    k_dp_tc<<<(d.G + warps - 1) / warps, warps * 32, gen_smem(d.Tg, warps), s>>>(d);
}
static int tcgrid(int n) { return std::max(1, std::min(148, (n + 127) / 128)); }
void launch_pack_tc2(const Dev &d, cudaStream_t s) { k_pack_tc2<<<tcgrid(d.G), 128, 0, s>>>(d); }
void launch_unpack_tc2(const Dev &d, cudaStream_t s) { k_unpack_tc2<<<tcgrid(d.G), 128, 0, s>>>(d); }
void launch_pack_tc3(const Dev &d, cudaStream_t s) { k_pack_tc3<<<tcgrid(d.G), 128, 0, s>>>(d); }
void launch_unpack_tc3(const Dev &d, cudaStream_t s) { k_unpack_tc3<<<tcgrid(d.G), 128, 0, s>>>(d); }
// The attribute is process-wide per kernel: only ever raise it, so a later context or dp_batch
// with a smaller T never lowers the limit under a live larger-T context.
cudaError_t gen_set_smem_attr(int T) {
    static std::mutex mu;
    static size_t cur = 0;
    std::lock_guard<std::mutex> lk(mu);
    // the grouped batch kernels run only while their block needs <= 76 KB (dp_pair_fits): that
    // limit, once, whatever T comes first
    static bool group_set = false;
    if (!group_set) {
        cudaError_t eg = cudaFuncSetAttribute(k_dp_batch_group<16, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 76 * 1024);
        if (eg == cudaSuccess)
            eg = cudaFuncSetAttribute(k_dp_batch_group<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 76 * 1024);
        if (eg != cudaSuccess) return eg;
        group_set = true;
    }
    const size_t b = gen_smem(T, 4);
    if (b <= cur) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k_gen, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_dp_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b);

    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_dp_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b);
    if (e == cudaSuccess) cur = b;
    return e;
}

}  // namespace ucac
