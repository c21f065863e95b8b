/*
 * oracle.c -- PLAIN CPU ORACLE for the UC-ACOPF two-level ADMM of arXiv 2310.13145
 * ("On Solving Unit Commitment with AC Optimal Power Flow on GPU").
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Single threaded, fp64, plain loops in the
 * paper's order; compiled with -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 * It shares no code with the CUDA path.  Where the paper is silent the reading taken is
 * the one registered in DESIGN.md section 3 ("R1".."R42", mirroring SURVEY.md c.4).
 *
 * Parity pins (tests/test_oracle_*.py) check every function here against something
 * other than itself: brute force over Eq. (3) schedules, exact active-set enumeration
 * of the generator / ubar QPs, dense KKT solves of the bus QP, KKT + finite differences
 * + grid search for the branch problem, closed forms and the MATPOWER case9 optimum.
 */
#include "oracle.h"
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdlib.h>
#include <string.h>

/* Row kinds of the coupling constraints, Eq. (5)-(6) as read in DESIGN.md 3.
 * gen rows per (g,t) */
enum { D_ON, D_SU, D_SD, PL, PU, QL, QU, RD, RU, GP, GQ, RC, NGR };
/* branch rows per (l,t) */
enum { FP_IJ, FQ_IJ, FP_JI, FQ_JI, W_I, W_J, A_I, A_J, NBR };

#define MAXN 8

struct orc_ctx {
    orc_problem pb;      /* pointers below own deep copies */
    orc_params pr;
    void *blk[40]; int nblk;
    /* x side */
    int8_t *u;                      /* [G*T] u_on */
    double *p, *q, *ph;             /* [G*T] */
    double *sl;                     /* [6*G*T] slacks pl pu ql qu rd ru (x-variables) */
    double *x, *f, *al;             /* branch x [L*T*4], flows [L*T*4], AL [L*T*3] */
    /* xbar side */
    double *ub[3];                  /* ubar on, su, sd [G*T] */
    double *pbar, *qbar;            /* [G*T] */
    double *fbar;                   /* [L*T*4] */
    double *wbar, *thbar;           /* [B*T] */
    /* multipliers */
    double *zg, *yg, *lg;           /* [12*G*T] */
    double *zb, *yb, *lb;           /* [8*L*T] */
    double beta, znorm_prev;
    int64_t outer_k, inner_total, inner_since;
    /* divergence detector: primal residual of the last 256 iterations (NaN = none) */
    double phist[256];
    int done;
    /* CSR incidence, canonical order (gens by index, then ends by (l, side)) */
    int32_t *bg_ptr, *bg_idx, *be_ptr, *be_idx;
    orc_report rep;
};

static void *cpy(orc_ctx *c, const void *src, size_t bytes) {
    void *d = malloc(bytes ? bytes : 1);
    if (src && bytes) memcpy(d, src, bytes);
    else memset(d, 0, bytes ? bytes : 1);
    c->blk[c->nblk++] = d;
    return d;
}
static double *dz(size_t n) { return (double *)calloc(n ? n : 1, sizeof(double)); }

static double dmax(double a, double b) { return a > b ? a : b; }
static double dmin(double a, double b) { return a < b ? a : b; }
static double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* Algorithmic flop counter of the branch solves (R55): each +, -, *, /, sqrt is one
 * flop, counted per operation as the plain algorithm states it (comparisons, clamps, copies and
 * sign flips are not flops).  Per thread, so the OpenMP build counts per solve. */
static __thread double g_fl;
#define FL(n) (g_fl += (double)(n))

/* sin and cos of one argument (R54).  An explicit polynomial instead of libm, so the
 * strict_fp GPU build can run the identical operation sequence and the two codes agree bit for
 * bit.  Cody-Waite reduction a = k pi/2 + r with k = floor(a 2/pi + 1/2) and fdlibm's split of
 * pi/2 (33 leading bits + tail), then the Taylor series of sin to r^17 and of cos to r^18 on
 * |r| <= pi/4 (truncation < 1e-19); quadrant by k mod 4.  Pinned against libm in
 * tests/test_oracle_branch.py (<= 2 ulp on [-4 pi, 4 pi], the range of theta_i - theta_j).
 * 43 flops. */
void orc_sincos(double a, double *s, double *c) {
    const double k = floor(a * 0x1.45f306dc9c883p-1 + 0.5);
    const double r = (a - k * 0x1.921fb544p+0) - k * 0x1.0b4611a626331p-34;
    const double z = r * r;
    double ps = 0x1.952c77030ad4ap-49;
    ps = ps * z + -0x1.ae7f3e733b81fp-41;
    ps = ps * z + 0x1.6124613a86d09p-33;
    ps = ps * z + -0x1.ae64567f544e4p-26;
    ps = ps * z + 0x1.71de3a556c734p-19;
    ps = ps * z + -0x1.a01a01a01a01ap-13;
    ps = ps * z + 0x1.1111111111111p-7;
    ps = ps * z + -0x1.5555555555555p-3;
    const double sr = r + (r * z) * ps;
    double pc = -0x1.6827863b97d97p-53;
    pc = pc * z + 0x1.ae7f3e733b81fp-45;
    pc = pc * z + -0x1.93974a8c07c9dp-37;
    pc = pc * z + 0x1.1eed8eff8d898p-29;
    pc = pc * z + -0x1.27e4fb7789f5cp-22;
    pc = pc * z + 0x1.a01a01a01a01ap-16;
    pc = pc * z + -0x1.6c16c16c16c17p-10;
    pc = pc * z + 0x1.5555555555555p-5;
    const double cr = (1.0 - 0.5 * z) + (z * z) * pc;
    FL(43);
    switch (((long long)k) & 3) {
        case 0: *s = sr; *c = cr; break;
        case 1: *s = cr; *c = -sr; break;
        case 2: *s = -sr; *c = -cr; break;
        default: *s = -cr; *c = sr; break;
    }
}

/* ========================================================================== */
/* S1: UC subproblem by dynamic programming (Section III-B, Algorithm 2).      */
/* ========================================================================== */

/* phi_v(b) = y_v (b - ubar_v + z_v) + rho/2 (b - ubar_v + z_v)^2: the augmented
 * Lagrangian terms of the duplicate rows x^UC - xbar^UC -- the only rows
 * containing x^UC (R18). */
static double phi(double b, double ub, double y, double z, double rho) {
    double e = (b - ub) + z;
    return y * e + 0.5 * rho * e * e;
}

/* Stage cost L^UC_{g,t}(a, b) with u^su, u^sd inferred from u^on:
 * f^UC_{t,g} = c0 u^on + C^SU u^su + C^SD u^sd (R13) plus the three phi terms,
 * summed left to right. */
void orc_stage_costs(int32_t T, double c0, double csu, double csd, double rho_uc,
                     const double *ub, const double *y, const double *z, double *L) {
    for (int t = 0; t < T; t++) {
        for (int a = 0; a < 2; a++) {
            for (int b = 0; b < 2; b++) {
                int su = b > a, sd = a > b;
                double v = c0 * (double)b;
                v = v + csu * (double)su;
                v = v + csd * (double)sd;
                v = v + phi((double)b, ub[0 * T + t], y[0 * T + t], z[0 * T + t], rho_uc);
                v = v + phi((double)su, ub[1 * T + t], y[1 * T + t], z[1 * T + t], rho_uc);
                v = v + phi((double)sd, ub[2 * T + t], y[2 * T + t], z[2 * T + t], rho_uc);
                L[t * 4 + a * 2 + b] = v;
            }
        }
    }
}

/* Algorithm 2 with Eq. (10) stay and Eq. (11) switch
 * (P:331-350).  c[t][s] is the optimal cost of periods t..T given the state s before t
 * (P:309).  Readings: window clipped at T with c_{T+1} = 0 (R15); direct left-to-right
 * window sum (R17); tie -> stay (R16); initial obligation = forced prefix of
 * `hold` periods at u0 (R14, Eq. 3a-3b).  Returns the optimal cost. */
double orc_dp(int32_t T, const double *L, int32_t TU, int32_t TD, int32_t u0,
              int32_t hold, int8_t *sched) {
    double *c = dz((size_t)(T + 1) * 2);
    int32_t *d = (int32_t *)calloc((size_t)(T + 1) * 2, sizeof(int32_t));
    c[T * 2 + 0] = 0.0;
    c[T * 2 + 1] = 0.0;
    for (int t = T - 1; t >= 0; t--) {
        for (int s = 0; s < 2; s++) {
            double stay = L[t * 4 + s * 2 + s] + c[(t + 1) * 2 + s];
            int n = 1 - s;
            int m = n ? TU : TD;
            int e = t + m - 1;
            if (e > T - 1) e = T - 1;
            double acc = L[t * 4 + s * 2 + n];
            for (int tt = t + 1; tt <= e; tt++) acc = acc + L[tt * 4 + n * 2 + n];
            double sw = acc + c[(e + 1) * 2 + n];
            if (stay <= sw) {
                c[t * 2 + s] = stay;
                d[t * 2 + s] = -1;
            } else {
                c[t * 2 + s] = sw;
                d[t * 2 + s] = e;
            }
        }
    }
    double cost = 0.0;
    int P = hold;
    for (int t = 0; t < P; t++) {
        sched[t] = (int8_t)u0;
        cost = cost + L[t * 4 + u0 * 2 + u0];
    }
    cost = cost + c[P * 2 + u0];
    int t = P, s = u0;
    while (t < T) {
        if (d[t * 2 + s] < 0) {
            sched[t] = (int8_t)s;
            t++;
        } else {
            int e = d[t * 2 + s];
            for (int tt = t; tt <= e; tt++) sched[tt] = (int8_t)(1 - s);
            s = 1 - s;
            t = e + 1;
        }
    }
    free(c);
    free(d);
    return cost;
}

/* NEXT-2: threshold the multiperiod-ACOPF dispatch, then one DP pass (Algorithm 2) whose
 * stage cost is the Hamming distance to the thresholded schedule: the nearest schedule that
 * satisfies Eq. 3 (SPEC warm_start_uc). */
void orc_uc_repair(int32_t T, const double *p, double threshold, int32_t TU, int32_t TD, int32_t u0,
                   int32_t hold, int8_t *u_out) {
    double *L = (double *)calloc((size_t)T * 4, sizeof(double));
    for (int t = 0; t < T; t++) {
        int ut = p[t] > threshold;
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 2; b++) L[t * 4 + a * 2 + b] = (b != ut) ? 1.0 : 0.0;
    }
    orc_dp(T, L, TU, TD, u0, hold, u_out);
    free(L);
}

/* ========================================================================== */
/* S2: generator x-update (7b restricted to p, q, phat, slacks).               */
/* ========================================================================== */
/* in[] layout: 0 first(0/1), 1 c2S2, 2 c1S, 3 rho_pq, 4 rho_uc, 5 tau_p, 6 tau_q,
 * 7 tau_ph, 8 p0, 9 b_pl, 10 b_pu, 11 b_ql, 12 b_qu, 13 b_rl, 14 b_ru,
 * 15 pL, 16 pU, 17 qL, 18 qU.
 * The subproblem (rows P:186-191 with Eq. 4d for ramp-down (R3) and the
 * ramp copy phat (R6)): minimise c2(Sp)^2 + c1 Sp + rho_pq/2[(p-tau_p)^2 + (q-tau_q)^2
 * + (phat-tau_ph)^2] + rho_uc/2 sum_rows (row - b)^2 over slacks >= 0 and the box.
 * Each slack minimises out exactly to a one-sided square; the remaining
 * convex piecewise quadratic is solved by enumerating activity patterns x {p free,
 * p = pL, p = pU} and keeping the smallest true objective (ties -> first). */
static double gen_obj_p(const double *in, double p, double ph) {
    double v = in[1] * p * p + in[2] * p;
    double e = p - in[5];
    v = v + 0.5 * in[3] * e * e;
    if (!(in[0] != 0.0)) {
        e = ph - in[7];
        v = v + 0.5 * in[3] * e * e;
    }
    e = p - in[9];
    if (e < 0.0) v = v + 0.5 * in[4] * e * e;
    e = p - in[10];
    if (e > 0.0) v = v + 0.5 * in[4] * e * e;
    double d = p - ph;
    e = d - in[13];
    if (e < 0.0) v = v + 0.5 * in[4] * e * e;
    e = d - in[14];
    if (e > 0.0) v = v + 0.5 * in[4] * e * e;
    return v;
}
static double gen_obj_q(const double *in, double q) {
    double e = q - in[6];
    double v = 0.5 * in[3] * e * e;
    e = q - in[11];
    if (e < 0.0) v = v + 0.5 * in[4] * e * e;
    e = q - in[12];
    if (e > 0.0) v = v + 0.5 * in[4] * e * e;
    return v;
}

void orc_gen_x(const double *in, double *out) {
    int first = in[0] != 0.0;
    double c2S2 = in[1], c1S = in[2], rpq = in[3], ruc = in[4];
    double tp = in[5], tq = in[6], tph = in[7], p0 = in[8];
    double bpl = in[9], bpu = in[10], bql = in[11], bqu = in[12], brl = in[13], bru = in[14];
    double pL = in[15], pU = in[16], qL = in[17], qU = in[18];
    double best = INFINITY, bp = pL, bph = first ? p0 : tph;
    if (first) {
        /* t = 1: phat = p_{0,g} is data (R5); 1-D convex. */
        for (int pat = 0; pat < 16; pat++) {
            int alo = pat & 1, ahi = (pat >> 1) & 1, rlo = (pat >> 2) & 1, rhi = (pat >> 3) & 1;
            double den = 2.0 * c2S2 + rpq;
            double num = -c1S + rpq * tp;
            if (alo) { den = den + ruc; num = num + ruc * bpl; }
            if (ahi) { den = den + ruc; num = num + ruc * bpu; }
            if (rlo) { den = den + ruc; num = num + ruc * (brl + p0); }
            if (rhi) { den = den + ruc; num = num + ruc * (bru + p0); }
            double p = num / den;
            if (p >= pL && p <= pU) {
                double v = gen_obj_p(in, p, p0);
                if (v < best) { best = v; bp = p; }
            }
        }
        double pb[2] = {pL, pU};
        for (int k = 0; k < 2; k++) {
            double v = gen_obj_p(in, pb[k], p0);
            if (v < best) { best = v; bp = pb[k]; }
        }
        bph = p0;
    } else {
        for (int pat = 0; pat < 16; pat++) {
            int alo = pat & 1, ahi = (pat >> 1) & 1, rlo = (pat >> 2) & 1, rhi = (pat >> 3) & 1;
            double A = 2.0 * c2S2 + rpq;
            double b1 = -c1S + rpq * tp;
            if (alo) { A = A + ruc; b1 = b1 + ruc * bpl; }
            if (ahi) { A = A + ruc; b1 = b1 + ruc * bpu; }
            double R = 0.0, rb = 0.0;
            if (rlo) { R = R + ruc; rb = rb + ruc * brl; }
            if (rhi) { R = R + ruc; rb = rb + ruc * bru; }
            b1 = b1 + rb;
            double b2 = rpq * tph - rb;
            /* [[A+R, -R], [-R, rpq+R]] (p, phat) = (b1, b2) */
            double det = (A + R) * (rpq + R) - R * R;
            double p = (b1 * (rpq + R) + R * b2) / det;
            double ph = ((A + R) * b2 + R * b1) / det;
            if (p >= pL && p <= pU) {
                double v = gen_obj_p(in, p, ph);
                if (v < best) { best = v; bp = p; bph = ph; }
            }
        }
        double pbs[2] = {pL, pU};
        for (int k = 0; k < 2; k++) {
            for (int pat = 0; pat < 4; pat++) {
                int rlo = pat & 1, rhi = (pat >> 1) & 1;
                double R = 0.0, rb = 0.0;
                if (rlo) { R = R + ruc; rb = rb + ruc * brl; }
                if (rhi) { R = R + ruc; rb = rb + ruc * bru; }
                double ph = (rpq * tph - rb + R * pbs[k]) / (rpq + R);
                double v = gen_obj_p(in, pbs[k], ph);
                if (v < best) { best = v; bp = pbs[k]; bph = ph; }
            }
        }
    }
    /* q: 1-D convex piecewise quadratic, patterns + bounds. */
    double bestq = INFINITY, bq = qL;
    for (int pat = 0; pat < 4; pat++) {
        int lo = pat & 1, hi = (pat >> 1) & 1;
        double den = rpq, num = rpq * tq;
        if (lo) { den = den + ruc; num = num + ruc * bql; }
        if (hi) { den = den + ruc; num = num + ruc * bqu; }
        double qq = num / den;
        if (qq >= qL && qq <= qU) {
            double v = gen_obj_q(in, qq);
            if (v < bestq) { bestq = v; bq = qq; }
        }
    }
    {
        double qb[2] = {qL, qU};
        for (int k = 0; k < 2; k++) {
            double v = gen_obj_q(in, qb[k]);
            if (v < bestq) { bestq = v; bq = qb[k]; }
        }
    }
    out[0] = bp;
    out[1] = bq;
    out[2] = bph;
}

/* ========================================================================== */
/* S4: ubar update (7c), exact box-QP over one group of <= 3 variables.        */
/* ========================================================================== */
/* minimise 0.5 sum_k (e_k - c_k' v)^2 over [0,1]^n (argmin over [0,1]).
 * Enumerate 3^n activity states (free / at 0 / at 1), solve the reduced SPD system
 * (H >= I because every variable has its duplicate row), clamp, keep the smallest true
 * objective (ties -> lowest state index). */
static int solve_small(int nf, double A[3][3], double *b, double *x) {
    if (nf == 1) { x[0] = b[0] / A[0][0]; return 0; }
    if (nf == 2) {
        double det = A[0][0] * A[1][1] - A[0][1] * A[1][0];
        x[0] = (b[0] * A[1][1] - A[0][1] * b[1]) / det;
        x[1] = (A[0][0] * b[1] - b[0] * A[1][0]) / det;
        return 0;
    }
    double det = A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1])
               - A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0])
               + A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
    for (int k = 0; k < 3; k++) {
        double M[3][3];
        for (int i = 0; i < 3; i++)
            for (int j = 0; j < 3; j++) M[i][j] = (j == k) ? b[i] : A[i][j];
        double dk = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1])
                  - M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0])
                  + M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
        x[k] = dk / det;
    }
    return 0;
}

void orc_boxqp3(int32_t n, int32_t m, const double *c, const double *e, double *v) {
    double H[3][3] = {{0}}, bb[3] = {0};
    for (int i = 0; i < n; i++) {
        for (int j = 0; j < n; j++) {
            double s = 0.0;
            for (int k = 0; k < m; k++) s = s + c[k * 3 + i] * c[k * 3 + j];
            H[i][j] = s;
        }
        double s = 0.0;
        for (int k = 0; k < m; k++) s = s + c[k * 3 + i] * e[k];
        bb[i] = s;
    }
    int ncand = 1;
    for (int i = 0; i < n; i++) ncand *= 3;
    double best = INFINITY;
    for (int i = 0; i < n; i++) v[i] = 0.0;
    for (int idx = 0; idx < ncand; idx++) {
        int st[3], r = idx;
        for (int i = 0; i < n; i++) { st[i] = r % 3; r /= 3; }
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
        for (int i = 0; i < n; i++) vv[i] = clampd(vv[i], 0.0, 1.0);
        double obj = 0.0;
        for (int k = 0; k < m; k++) {
            double rr = e[k];
            for (int i = 0; i < n; i++) rr = rr - c[k * 3 + i] * vv[i];
            obj = obj + 0.5 * rr * rr;
        }
        if (obj < best) {
            best = obj;
            for (int i = 0; i < n; i++) v[i] = vv[i];
        }
    }
}

/* ========================================================================== */
/* S5: bus update (7d), equality-constrained QP with the two balance rows.    */
/* ========================================================================== */
/* minimise sum_k a_k/2 (v_k - tauhat_k)^2 s.t. sum alpha_k v_k = P, sum beta_k v_k = Q
 * (Eq. 2a-2b; bus subproblem P:411/418).  Lagrange: v_k = tauhat_k +
 * (alpha_k muP + beta_k muQ)/a_k, with the 2x2 system solved by Cramer's rule. */
void orc_bus_kkt(int32_t k, const double *alpha, const double *beta, const double *a,
                 const double *tauhat, double P, double Q, double *v, double *mu) {
    double AP = 0, AQ = 0, C = 0, rP = P, rQ = Q;
    for (int i = 0; i < k; i++) {
        AP = AP + alpha[i] * alpha[i] / a[i];
        AQ = AQ + beta[i] * beta[i] / a[i];
        C = C + alpha[i] * beta[i] / a[i];
        rP = rP - alpha[i] * tauhat[i];
        rQ = rQ - beta[i] * tauhat[i];
    }
    double det = AP * AQ - C * C;
    double muP = (rP * AQ - C * rQ) / det;
    double muQ = (AP * rQ - C * rP) / det;
    for (int i = 0; i < k; i++) v[i] = tauhat[i] + (alpha[i] * muP + beta[i] * muQ) / a[i];
    mu[0] = muP;
    mu[1] = muQ;
}

/* ========================================================================== */
/* S3: branch x-update (7b line part): flows, TRON, augmented Lagrangian.      */
/* ========================================================================== */

/* Flows of branch (i->j) as functions of x = (w_i, w_j, theta_i, theta_j) through
 * C = sqrt(w_i w_j) cos(theta_i - theta_j), S = sqrt(w_i w_j) sin(...), i.e. the
 * rectangular products w^R_ij, w^I_ij of P:106-113 (Eq. 2i-2j hold identically).
 * Eq. 2e-2h (with the to-side labels read as ji, R1):
 *   p_ij =  Gii w_i + Gij C + Bij S      q_ij = -Bii w_i - Bij C + Gij S
 *   p_ji =  Gjj w_j + Gji C - Bji S      q_ji = -Bjj w_j - Bji C - Gji S
 * J[k*4+m] = d f_k / d x_m; H[k*16+m*4+n] = d^2 f_k / d x_m d x_n. */
void orc_branch_flows(const double *y, const double *x, double *f, double *J, double *H) {
    double Gii = y[0], Gij = y[1], Gji = y[2], Gjj = y[3];
    double Bii = y[4], Bij = y[5], Bji = y[6], Bjj = y[7];
    double wi = x[0], wj = x[1], d = x[2] - x[3];
    double R = sqrt(wi * wj);
    double sn, cs;
    orc_sincos(d, &sn, &cs);
    double C = R * cs, S = R * sn;
    /* flops: R, d, C, S 5 (+ 43 sincos); f 28; with J, H the textbook tables: dC, dS 8, HC/HS 34,
     * J 56, H 192 (R55) */
    FL(5 + 28);
    if (J || H) FL(8 + 34 + (J ? 56 : 0) + (H ? 192 : 0));
    double dC[4] = {C / (2.0 * wi), C / (2.0 * wj), -S, S};
    double dS[4] = {S / (2.0 * wi), S / (2.0 * wj), C, -C};
    double HC[4][4], HS[4][4];
    HC[0][0] = -C / (4.0 * wi * wi);  HS[0][0] = -S / (4.0 * wi * wi);
    HC[1][1] = -C / (4.0 * wj * wj);  HS[1][1] = -S / (4.0 * wj * wj);
    HC[0][1] = C / (4.0 * wi * wj);   HS[0][1] = S / (4.0 * wi * wj);
    HC[0][2] = -S / (2.0 * wi);       HS[0][2] = C / (2.0 * wi);
    HC[0][3] = S / (2.0 * wi);        HS[0][3] = -C / (2.0 * wi);
    HC[1][2] = -S / (2.0 * wj);       HS[1][2] = C / (2.0 * wj);
    HC[1][3] = S / (2.0 * wj);        HS[1][3] = -C / (2.0 * wj);
    HC[2][2] = -C;                    HS[2][2] = -S;
    HC[3][3] = -C;                    HS[3][3] = -S;
    HC[2][3] = C;                     HS[2][3] = S;
    for (int m = 0; m < 4; m++)
        for (int n = 0; n < m; n++) { HC[m][n] = HC[n][m]; HS[m][n] = HS[n][m]; }
    /* f_k = a_k w_i + b_k w_j + c_k C + d_k S */
    double ca[4] = {Gii, -Bii, 0.0, 0.0};
    double cb[4] = {0.0, 0.0, Gjj, -Bjj};
    double cc[4] = {Gij, -Bij, Gji, -Bji};
    double cd[4] = {Bij, Gij, -Bji, -Gji};
    for (int k = 0; k < 4; k++) {
        f[k] = ca[k] * wi + cb[k] * wj + cc[k] * C + cd[k] * S;
        if (J) {
            for (int m = 0; m < 4; m++) {
                double v = cc[k] * dC[m] + cd[k] * dS[m];
                if (m == 0) v = v + ca[k];
                if (m == 1) v = v + cb[k];
                J[k * 4 + m] = v;
            }
        }
        if (H) {
            for (int m = 0; m < 4; m++)
                for (int n = 0; n < 4; n++)
                    H[k * 16 + m * 4 + n] = cc[k] * HC[m][n] + cd[k] * HS[m][n];
        }
    }
}

typedef void (*eval_fn)(void *ctx, const double *x, double *f, double *g, double *H);

static double dot(int n, const double *a, const double *b) {
    FL(2 * n);
    double s = 0.0;
    for (int i = 0; i < n; i++) s = s + a[i] * b[i];
    return s;
}
static double nrm2(int n, const double *a) { FL(1); return sqrt(dot(n, a, a)); }
static void matvec(int n, const double *H, const double *v, double *o) {
    FL(2 * n * n);
    for (int i = 0; i < n; i++) {
        double s = 0.0;
        for (int j = 0; j < n; j++) s = s + H[i * n + j] * v[j];
        o[i] = s;
    }
}
/* quadratic model q(s) = g's + 1/2 s'Hs */
static double qmodel(int n, const double *g, const double *H, const double *s) {
    double Hs[MAXN];
    matvec(n, H, s, Hs);
    FL(2);
    return dot(n, g, s) + 0.5 * dot(n, s, Hs);
}

/* TRON-style projected trust-region Newton (Lin & More 1999; "ExaTron"), as
 * specified in DESIGN.md 5.3 (constants R10).  Returns 1 if ||P(x-g)-x||_inf <= gtol. */
static const double TR_MU0 = 0.01, TR_ETA0 = 1e-4, TR_ETA1 = 0.25, TR_ETA2 = 0.75;
static const double TR_SIG1 = 0.25, TR_SIG3 = 4.0, TR_DELTA0 = 1.0, TR_CGTOL = 1e-12;
static const double TR_EPSF = 1e-10, TR_STALL = 1e-13;   /* R48 */
static const double TR_STALL_R34 = 1e-14;                  /* R34, the plain mode */

static void pstep(int n, const double *x, const double *lo, const double *hi,
                  const double *d, double a, double *s) {
    FL(3 * n);
    for (int i = 0; i < n; i++) s[i] = clampd(x[i] + a * d[i], lo[i], hi[i]) - x[i];
}
static int cauchy_ok(int n, const double *g, const double *H, const double *s, double delta) {
    FL(1);
    return nrm2(n, s) <= delta && qmodel(n, g, H, s) <= TR_MU0 * dot(n, g, s);
}
static void cauchy(int n, const double *x, const double *lo, const double *hi,
                   const double *g, const double *H, double delta, double *alpha, double *s) {
    double mg[MAXN], sp[MAXN];
    for (int i = 0; i < n; i++) mg[i] = -g[i];
    double a = *alpha;
    pstep(n, x, lo, hi, mg, a, s);
    if (!cauchy_ok(n, g, H, s, delta)) {
        for (int k = 0; k < 60; k++) {
            a = a * 0.1;
            FL(1);
            pstep(n, x, lo, hi, mg, a, s);
            if (cauchy_ok(n, g, H, s, delta)) break;
        }
    } else {
        for (int k = 0; k < 20; k++) {
            double ap = a;
            for (int i = 0; i < n; i++) sp[i] = s[i];
            a = a * 10.0;
            FL(1);
            pstep(n, x, lo, hi, mg, a, s);
            int same = 1;
            for (int i = 0; i < n; i++) if (s[i] != sp[i]) same = 0;
            if (!cauchy_ok(n, g, H, s, delta) || same) {
                a = ap;
                for (int i = 0; i < n; i++) s[i] = sp[i];
                break;
            }
        }
    }
    *alpha = a;
}
/* tau >= 0 with ||a + tau p||_2 = delta */
static double bnd_tau(int n, const double *a, const double *p, double delta) {
    double aa = dot(n, a, a), ap = dot(n, a, p), pp = dot(n, p, p);
    if (pp <= 0.0) return 0.0;
    FL(8);
    double gap = delta * delta - aa;
    if (gap < 0.0) gap = 0.0;
    double rad = sqrt(ap * ap + pp * gap);
    if (ap > 0.0) return gap / (ap + rad);
    return (rad - ap) / pp;
}
/* Steihaug-Toint CG on the free variables for the model at s_c, trust region on the
 * total step s_c + w. */
static void steihaug(int n, const double *H, const double *gq, const int *fr,
                     const double *sc, double delta, double *w) {
    double r[MAXN], p[MAXN], Hp[MAXN], t[MAXN];
    for (int i = 0; i < n; i++) {
        w[i] = 0.0;
        r[i] = fr[i] ? -gq[i] : 0.0;
        p[i] = r[i];
    }
    double rr = dot(n, r, r);
    if (rr == 0.0) return;
    double tol2 = TR_CGTOL * TR_CGTOL * rr;
    FL(2);
    for (int k = 0; k < n; k++) {
        matvec(n, H, p, Hp);
        for (int i = 0; i < n; i++) if (!fr[i]) Hp[i] = 0.0;
        double kap = dot(n, p, Hp);
        for (int i = 0; i < n; i++) t[i] = sc[i] + w[i];
        FL(n);
        if (kap <= 0.0) {
            double tau = bnd_tau(n, t, p, delta);
            for (int i = 0; i < n; i++) w[i] = w[i] + tau * p[i];
            FL(2 * n);
            return;
        }
        double a = rr / kap;
        for (int i = 0; i < n; i++) t[i] = sc[i] + w[i] + a * p[i];
        FL(1 + 3 * n);
        if (nrm2(n, t) >= delta) {
            for (int i = 0; i < n; i++) t[i] = sc[i] + w[i];
            double tau = bnd_tau(n, t, p, delta);
            for (int i = 0; i < n; i++) w[i] = w[i] + tau * p[i];
            FL(3 * n);
            return;
        }
        for (int i = 0; i < n; i++) { w[i] = w[i] + a * p[i]; r[i] = r[i] - a * Hp[i]; }
        FL(4 * n);
        double rn = dot(n, r, r);
        if (rn <= tol2) return;
        double b = rn / rr;
        for (int i = 0; i < n; i++) p[i] = r[i] + b * p[i];
        FL(1 + 2 * n);
        rr = rn;
    }
}
/* projected search along w from the Cauchy point */
static void prsrch(int n, const double *x, const double *lo, const double *hi,
                   const double *g, const double *H, const double *sc, const double *w,
                   double *s) {
    double gq[MAXN], Hs[MAXN], ds[MAXN];
    matvec(n, H, sc, Hs);
    for (int i = 0; i < n; i++) gq[i] = g[i] + Hs[i];
    FL(n);
    double qc = qmodel(n, g, H, sc);
    double b = 1.0;
    for (int k = 0; k < 20; k++) {
        for (int i = 0; i < n; i++) {
            s[i] = clampd(x[i] + sc[i] + b * w[i], lo[i], hi[i]) - x[i];
            ds[i] = s[i] - sc[i];
        }
        FL(5 * n + 2);
        if (qmodel(n, g, H, s) <= qc + TR_MU0 * dot(n, gq, ds)) return;
        b = b * 0.5;
        FL(1);
    }
    for (int i = 0; i < n; i++) s[i] = sc[i];
}
static double pgnorm(int n, const double *x, const double *g, const double *lo,
                     const double *hi) {
    FL(2 * n);
    double m = 0.0;
    for (int i = 0; i < n; i++) {
        double v = fabs(clampd(x[i] - g[i], lo[i], hi[i]) - x[i]);
        if (v > m) m = v;
    }
    return m;
}
/* plain = 1: the first-order reading of SURVEY 8(c) S3 with none of the solver accelerations
 * R41 (first Cauchy trial = model minimiser) or R48 (stall step 1e-13; plain keeps R34's 1e-14) */
static int tron_r(int n, double *x, const double *lo, const double *hi, eval_fn ev, void *ctx,
                  double gtol, int maxit, int *iters, double delta0, int plain);
static int tron(int n, double *x, const double *lo, const double *hi, eval_fn ev, void *ctx,
                double gtol, int maxit, int *iters) {
    return tron_r(n, x, lo, hi, ev, ctx, gtol, maxit, iters, TR_DELTA0, 0);
}
static int tron_r(int n, double *x, const double *lo, const double *hi, eval_fn ev, void *ctx,
                  double gtol, int maxit, int *iters, double delta0, int plain) {
    double f, g[MAXN], H[MAXN * MAXN], fn, gn[MAXN], Hn[MAXN * MAXN];
    double sc[MAXN], w[MAXN], s[MAXN], xn[MAXN], gq[MAXN], Hs[MAXN];
    int fr[MAXN];
    const double stall = plain ? TR_STALL_R34 : TR_STALL;
    for (int i = 0; i < n; i++) x[i] = clampd(x[i], lo[i], hi[i]);
    ev(ctx, x, &f, g, H);
    double delta = delta0, alpha = 1.0;
    if (!plain) {
        /* first Cauchy trial length: the model minimiser along -g (R41) */
        double Hg[MAXN];
        matvec(n, H, g, Hg);
        double gHg = dot(n, g, Hg), gg = dot(n, g, g);
        if (gHg > 0.0 && gg > 0.0) { alpha = gg / gHg; FL(1); }
    }
    int it;
    for (it = 0; it < maxit; it++) {
        if (pgnorm(n, x, g, lo, hi) <= gtol) { *iters = it; return 1; }
        cauchy(n, x, lo, hi, g, H, delta, &alpha, sc);
        for (int i = 0; i < n; i++) {
            double xc = x[i] + sc[i];
            fr[i] = (xc > lo[i] && xc < hi[i]);
        }
        matvec(n, H, sc, Hs);
        for (int i = 0; i < n; i++) gq[i] = g[i] + Hs[i];
        FL(2 * n);
        steihaug(n, H, gq, fr, sc, delta, w);
        prsrch(n, x, lo, hi, g, H, sc, w, s);
        /* stall: a step below 1e-13 (1 + |x|) means the rounding floor of the gradient is reached;
         * for the AL's sigma J'J curvature that floor lies above gtol (R48) */
        {
            double xm = 0.0;
            for (int i = 0; i < n; i++) xm = dmax(xm, fabs(x[i]));
            FL(2);
            if (nrm2(n, s) <= stall * (1.0 + xm)) { *iters = it; return 1; }
        }
        double pred = -qmodel(n, g, H, s);
        for (int i = 0; i < n; i++) xn[i] = clampd(x[i] + s[i], lo[i], hi[i]);
        ev(ctx, xn, &fn, gn, Hn);
        double ared = f - fn;
        FL(n + 1);
        /* when the predicted reduction is below the rounding level of f, f - fn is noise:
         * use the trapezoidal estimate -(g + gn)'s / 2 instead. */
        if (fabs(pred) <= TR_EPSF * fabs(f)) { ared = -0.5 * (dot(n, g, s) + dot(n, gn, s)); FL(2); }
        FL(1);
        double ratio = (pred > 0.0) ? ared / pred : -1.0;
        FL(pred > 0.0);
        double snorm = nrm2(n, s);
        if (ratio > TR_ETA0) {
            for (int i = 0; i < n; i++) x[i] = xn[i];
            f = fn;
            memcpy(g, gn, sizeof(double) * n);
            memcpy(H, Hn, sizeof(double) * n * n);
        }
        if (ratio < TR_ETA1) { delta = TR_SIG1 * dmin(snorm, delta); FL(1); }
        else if (ratio > TR_ETA2) { delta = dmax(delta, TR_SIG3 * snorm); FL(1); }
    }
    *iters = it;
    return pgnorm(n, x, g, lo, hi) <= gtol;
}

typedef struct { const double *A, *b; int n; } qctx;
static void q_eval(void *vc, const double *x, double *f, double *g, double *H) {
    qctx *c = (qctx *)vc;
    int n = c->n;
    matvec(n, c->A, x, g);
    *f = 0.5 * dot(n, x, g) + dot(n, c->b, x);
    for (int i = 0; i < n; i++) g[i] = g[i] + c->b[i];
    for (int i = 0; i < n * n; i++) H[i] = c->A[i];
}
int orc_tron_quadratic(int32_t n, const double *A, const double *b, const double *lo,
                       const double *hi, double gtol, int32_t maxit, double *x) {
    qctx c = {A, b, n};
    int it;
    return tron(n, x, lo, hi, q_eval, &c, gtol, maxit, &it) ? it : -1;
}

/* Branch objective: F = sum_k rho_pq/2 (f_k - tau_k)^2 + sum_m rho_va/2 (x_m - tau_{4+m})^2
 * (the x-step minimises sum_rows rho/2 (row - tau)^2).  With al != 0 the
 * variables are (x, s_ij, s_ji) and Phi = F + sum_m mu_m h_m + sigma/2 h_m^2 with
 * h_m = (p_m^2 + q_m^2)/rbar^2 - 1 + s_m, s_m in [0,1] (Eq. 2c-2d, R9). */
typedef struct {
    const double *y, *tau;
    double rpq, rva, r2, mu[2], sig;
    int al;
    int nva;   /* 4 (w and theta rows) or 2 (no angle rows, R51) */
} bctx;
static void br_eval(void *vc, const double *X, double *fo, double *g, double *H) {
    bctx *c = (bctx *)vc;
    int n = c->al ? 6 : 4;
    double f[4], J[16], Hf[64];
    orc_branch_flows(c->y, X, f, J, Hf);
    /* flops (R55): flow rows 4 x 97, va rows 8 each, AL 2 x 334 (dense 6x6 Hessian terms) */
    FL(4 * 97 + 8 * c->nva + (c->al ? 2 * 334 : 0));
    double F = 0.0;
    for (int i = 0; i < n; i++) g[i] = 0.0;
    for (int i = 0; i < n * n; i++) H[i] = 0.0;
    for (int k = 0; k < 4; k++) {
        double e = f[k] - c->tau[k];
        F = F + 0.5 * c->rpq * e * e;
        for (int a = 0; a < 4; a++) {
            g[a] = g[a] + c->rpq * e * J[k * 4 + a];
            for (int b = 0; b < 4; b++)
                H[a * n + b] = H[a * n + b] + c->rpq * (J[k * 4 + a] * J[k * 4 + b] + e * Hf[k * 16 + a * 4 + b]);
        }
    }
    for (int m = 0; m < c->nva; m++) {   /* nva = 2 without the angle rows (R51) */
        double e = X[m] - c->tau[4 + m];
        F = F + 0.5 * c->rva * e * e;
        g[m] = g[m] + c->rva * e;
        H[m * n + m] = H[m * n + m] + c->rva;
    }
    if (c->al) {
        for (int m = 0; m < 2; m++) {
            int kp = 2 * m, kq = 2 * m + 1;
            double P = f[kp], Q = f[kq];
            double h = (P * P + Q * Q) / c->r2 - 1.0 + X[4 + m];
            double gh[6] = {0, 0, 0, 0, 0, 0};
            for (int a = 0; a < 4; a++) gh[a] = 2.0 * (P * J[kp * 4 + a] + Q * J[kq * 4 + a]) / c->r2;
            gh[4 + m] = 1.0;
            double lam = c->mu[m] + c->sig * h;
            F = F + c->mu[m] * h + 0.5 * c->sig * h * h;
            for (int a = 0; a < 6; a++) g[a] = g[a] + lam * gh[a];
            for (int a = 0; a < 6; a++) {
                for (int b = 0; b < 6; b++) {
                    double hh = 0.0;
                    if (a < 4 && b < 4)
                        hh = 2.0 * (J[kp * 4 + a] * J[kp * 4 + b] + P * Hf[kp * 16 + a * 4 + b]
                                    + J[kq * 4 + a] * J[kq * 4 + b] + Q * Hf[kq * 16 + a * 4 + b]) / c->r2;
                    H[a * 6 + b] = H[a * 6 + b] + lam * hh + c->sig * gh[a] * gh[b];
                }
            }
        }
    }
    *fo = F;
}

/* Second-order multiplier update of the method of multipliers (R42).  Near the round's
 * minimiser X(mu) of the AL Phi on the box, with the active bounds fixed, the constraint values
 * move as dh/dmu = -M, M = J_F H_FF^{-1} J_F' (J = dh/dX, H = Hessian of Phi, F = the
 * variables strictly inside their bounds), so the Newton step on h(mu) = 0 is dmu = M^{-1} h.
 * For sigma -> inf, M -> I/sigma and this is the first-order update dmu = sigma h.
 * Returns 0 (caller keeps the first-order update) if H_FF or M is not positive definite. */
#define AL_NEWTON_C 10.0
#define AL_R1_DELTA0 0.03
static int al_newton_dmu(bctx *c, const double *X, const double *lo, const double *hi,
                         const double *h, double *dmu, double *dx) {
    double F, g[6], H[36], f[4], Jf[16];
    br_eval(c, X, &F, g, H);
    orc_branch_flows(c->y, X, f, Jf, NULL);
    /* J rows: dh_m/dX = 2 (P_m dP_m/dx + Q_m dQ_m/dx) / rbar^2, and 1 for the slack s_m */
    double J[2][6];
    for (int m = 0; m < 2; m++) {
        int kp = 2 * m, kq = 2 * m + 1;
        for (int a = 0; a < 4; a++) J[m][a] = 2.0 * (f[kp] * Jf[kp * 4 + a] + f[kq] * Jf[kq * 4 + a]) / c->r2;
        FL(4 * 5);
        J[m][4] = m == 0 ? 1.0 : 0.0;
        J[m][5] = m == 1 ? 1.0 : 0.0;
    }
    int idx[6], nf = 0;
    for (int i = 0; i < 6; i++)
        if (X[i] > lo[i] && X[i] < hi[i]) idx[nf++] = i;
    /* Cholesky H_FF = L L' (textbook, column by column) */
    double L[36];
    for (int j = 0; j < nf; j++) {
        double d = H[idx[j] * 6 + idx[j]];
        for (int k = 0; k < j; k++) d = d - L[j * 6 + k] * L[j * 6 + k];
        FL(2 * j + 1);
        if (!(d > 0.0)) return 0;
        L[j * 6 + j] = sqrt(d);
        for (int i = j + 1; i < nf; i++) {
            double v = H[idx[i] * 6 + idx[j]];
            for (int k = 0; k < j; k++) v = v - L[i * 6 + k] * L[j * 6 + k];
            L[i * 6 + j] = v / L[j * 6 + j];
            FL(2 * j + 1);
        }
    }
    /* V_m = H_FF^{-1} J_m,F by forward and back substitution; M_mn = J_m,F . V_n */
    double V[2][6];
    for (int m = 0; m < 2; m++) {
        double z[6];
        for (int i = 0; i < nf; i++) {
            double v = J[m][idx[i]];
            for (int k = 0; k < i; k++) v = v - L[i * 6 + k] * z[k];
            z[i] = v / L[i * 6 + i];
        }
        for (int i = nf - 1; i >= 0; i--) {
            double v = z[i];
            for (int k = i + 1; k < nf; k++) v = v - L[k * 6 + i] * V[m][k];
            V[m][i] = v / L[i * 6 + i];
        }
        FL(2 * nf * nf);
    }
    double M[2][2];
    for (int m = 0; m < 2; m++)
        for (int n = 0; n < 2; n++) {
            double v = 0.0;
            for (int i = 0; i < nf; i++) v = v + J[m][idx[i]] * V[n][i];
            M[m][n] = v;
            FL(2 * nf);
        }
    /* Spectral safeguard: in each eigen-direction v of M (eigenvalue lam in (0, 1/sigma]) take
     * the Newton factor 1/lam where lam >= 1/(C sigma), and the first-order factor sigma where M
     * is nearly singular (both ends of a near-lossless line binding: their multipliers are not
     * separately determined, and 1/lam would amplify rounding along that direction). */
    double a = M[0][0], b = 0.5 * (M[0][1] + M[1][0]), d = M[1][1];
    double mean = 0.5 * (a + d), half = 0.5 * (a - d);
    double r = sqrt(half * half + b * b);
    double lam[2] = {mean + r, mean - r};
    FL(13);
    double v[2][2];
    if (r == 0.0) {
        v[0][0] = 1.0; v[0][1] = 0.0;
    } else if (a >= d) {
        double n = sqrt((lam[0] - d) * (lam[0] - d) + b * b);
        v[0][0] = (lam[0] - d) / n; v[0][1] = b / n;
        FL(9);
    } else {
        double n = sqrt(b * b + (lam[0] - a) * (lam[0] - a));
        v[0][0] = b / n; v[0][1] = (lam[0] - a) / n;
        FL(9);
    }
    v[1][0] = -v[0][1]; v[1][1] = v[0][0];
    dmu[0] = 0.0;
    dmu[1] = 0.0;
    for (int e = 0; e < 2; e++) {
        double fac = lam[e] >= 1.0 / (AL_NEWTON_C * c->sig) ? 1.0 / lam[e] : c->sig;
        double ph = v[e][0] * h[0] + v[e][1] * h[1];
        dmu[0] = dmu[0] + fac * ph * v[e][0];
        dmu[1] = dmu[1] + fac * ph * v[e][1];
        FL(3 + 3 + 4);
    }
    /* first-order move of the round's minimiser with mu (R43): dX_F = -H_FF^{-1} J_F' dmu */
    for (int i = 0; i < 6; i++) dx[i] = 0.0;
    for (int i = 0; i < nf; i++) dx[idx[i]] = -(V[0][i] * dmu[0] + V[1][i] * dmu[1]);
    FL(3 * nf);
    return 1;
}

/* One branch solve (R9/R10/R12): TRON on the 4-variable box; if the rate is
 * 0 (unlimited) or both ends satisfy Eq. 2c-2d, done (thermal multipliers 0).  Otherwise
 * method of multipliers on the 6-variable slack form, warm-starting (mu, sigma).
 * pr->plain = 1 switches off every solver acceleration (R41-R44, R48, R49): the first-order
 * AL of SURVEY 8(c) S3 with R36's sigma rule -- the plain twin that pins the accelerated path
 * (tests/test_oracle_branch.py::test_plain_and_accelerated_al_same_kkt_point).
 * stats: 0 TRON iterations, 1 TRON capped, 2 AL active, 3 AL rounds, 4 AL capped,
 *        5 flops of the fast path, 6 flops of the AL, 7 fast-path Newton its, 8 AL Newton its (R55). */
void orc_branch_solve(const double *y, const double *wlo, const double *whi, double rate,
                      const double *tau, double rpq, double rva, const orc_params *pr,
                      double *x, double *al, double *f, int64_t *stats) {
    const double TWO_PI = 6.283185307179586;
    const int plain = pr->plain != 0;
    double lo[6] = {wlo[0], wlo[1], -TWO_PI, -TWO_PI, 0.0, 0.0};
    double hi[6] = {whi[0], whi[1], TWO_PI, TWO_PI, 1.0, 1.0};
    /* NEXT-3 variant 8 (R51): no angle consensus rows; the line's angles are local,
     * with its own reference theta_i = 0 (only theta_i - theta_j enters the flows) */
    if (pr->variant & 8) lo[2] = hi[2] = 0.0;
    double gtol = pr->tron_gtol_rel * dmax(rpq, rva);
    bctx c;
    c.y = y; c.tau = tau; c.rpq = rpq; c.rva = rva; c.al = 0;
    c.nva = (pr->variant & 8) ? 2 : 4;
    c.r2 = rate * rate; c.mu[0] = c.mu[1] = 0.0; c.sig = 0.0;
    int it = 0;
    const double fl0 = g_fl;
    /* NEXT-3 variant 1 (R47): every rated branch goes straight to the six-variable AL from the
     * warm start (clipped to the box), as ExaTron solves it; else the 4-variable fast path first */
    const int al_always = (pr->variant & 1) && rate > 0.0;
    int ok = 1;
    /* the previous iterate, clipped to the box: the second candidate start of the AL (R49) */
    double xprev[4];
    for (int i = 0; i < 4; i++) xprev[i] = clampd(x[i], lo[i], hi[i]);
    if (al_always)
        for (int i = 0; i < 4; i++) x[i] = clampd(x[i], lo[i], hi[i]);
    else
        ok = tron_r(4, x, lo, hi, br_eval, &c, gtol, pr->tron_maxit, &it, TR_DELTA0, plain);
    stats[0] = it; stats[1] = !ok; stats[2] = 0; stats[3] = 0; stats[4] = 0;
    stats[7] = it; stats[8] = 0;
    double sig0 = pr->al_sigma0_rel * rpq * c.r2;
    orc_branch_flows(y, x, f, NULL, NULL);
    const double fl1 = g_fl;
    stats[5] = (int64_t)(fl1 - fl0); stats[6] = 0;
    if (rate > 0.0) {
        double s1 = f[0] * f[0] + f[1] * f[1], s2 = f[2] * f[2] + f[3] * f[3];
        if (al_always || s1 > c.r2 || s2 > c.r2) {
            double X[6] = {x[0], x[1], x[2], x[3],
                           clampd(1.0 - s1 / c.r2, 0.0, 1.0), clampd(1.0 - s2 / c.r2, 0.0, 1.0)};
            FL(6 + 4);
            c.al = 1;
            c.mu[0] = al[0]; c.mu[1] = al[1];
            c.sig = dmax(sig0, al[2] * pr->al_sigma_decay);
            double smax = pr->al_sigma_max_rel * sig0;
            double hprev = INFINITY;
            int k;
            stats[2] = 1;
            if (!plain) {
                /* R49: round 1 starts from whichever of the fast-path point and the previous
                 * iterate (each with its slacks from its flows) has the lower AL value */
                double fp[4], Xp[6], Fa, Fb, gs[6], Hs[36];
                orc_branch_flows(y, xprev, fp, NULL, NULL);
                for (int i = 0; i < 4; i++) Xp[i] = xprev[i];
                Xp[4] = clampd(1.0 - (fp[0] * fp[0] + fp[1] * fp[1]) / c.r2, 0.0, 1.0);
                Xp[5] = clampd(1.0 - (fp[2] * fp[2] + fp[3] * fp[3]) / c.r2, 0.0, 1.0);
                FL(10);
                br_eval(&c, X, &Fa, gs, Hs);
                br_eval(&c, Xp, &Fb, gs, Hs);
                if (Fb < Fa)
                    for (int i = 0; i < 6; i++) X[i] = Xp[i];
            }
            for (k = 0; k < pr->al_maxit; k++) {
                /* round 1 starts at the fast-path point, which violates Eq. 2c-2d: a small first
                 * trust region (R44) keeps the first model step where sigma h^2 is modelled well */
                const double d0 = (k == 0 && !plain) ? AL_R1_DELTA0 : TR_DELTA0;
                ok = tron_r(6, X, lo, hi, br_eval, &c, gtol, pr->tron_maxit, &it, d0, plain);
                stats[0] += it;
                stats[8] += it;
                stats[1] += !ok;
                orc_branch_flows(y, X, f, NULL, NULL);
                double h1 = (f[0] * f[0] + f[1] * f[1]) / c.r2 - 1.0 + X[4];
                double h2 = (f[2] * f[2] + f[3] * f[3]) / c.r2 - 1.0 + X[5];
                FL(12);
                double hm = dmax(fabs(h1), fabs(h2));
                if (hm <= pr->al_eta_star) break;
                double hv[2] = {h1, h2}, dmu[2], dx[6];
                if (!plain && al_newton_dmu(&c, X, lo, hi, hv, dmu, dx)) {
#ifndef ORC_NO_PREDICTOR
                    for (int i = 0; i < 6; i++) X[i] = clampd(X[i] + dx[i], lo[i], hi[i]);
                    FL(6);
#endif
                } else {
                    /* first-order method of multipliers (Nocedal-Wright 17.4), R36 */
                    dmu[0] = c.sig * h1;
                    dmu[1] = c.sig * h2;
                    FL(2);
                }
                c.mu[0] = c.mu[0] + dmu[0];
                c.mu[1] = c.mu[1] + dmu[1];
                FL(3);
                if (hm > 0.25 * hprev) { c.sig = dmin(10.0 * c.sig, smax); FL(1); }
                hprev = hm;
            }
            stats[3] = k < pr->al_maxit ? k + 1 : k;
            stats[4] = k >= pr->al_maxit;
            for (int i = 0; i < 4; i++) x[i] = X[i];
            al[0] = c.mu[0]; al[1] = c.mu[1]; al[2] = c.sig;
            stats[6] = (int64_t)(g_fl - fl1);
            return;
        }
    }
    al[0] = 0.0; al[1] = 0.0; al[2] = sig0;
}

/* ========================================================================== */
/* Context, initialisation (S0), the inner iteration (Alg. 1 lines 4-9).       */
/* ========================================================================== */

static int bad(double v) { return !(v == v) || v == INFINITY || v == -INFINITY; }

int orc_create(const orc_problem *pb, const orc_params *pr, orc_ctx **out) {
    *out = NULL;
    if (pr->diverge_window < 0 || pr->diverge_window >= 256) return 1;
    int B = pb->nbus, G = pb->ngen, L = pb->nbranch, T = pb->T;
    if (B <= 0 || G <= 0 || L <= 0 || T <= 0 || pb->ref_bus < 0 || pb->ref_bus >= B) return 1;
    if (!(pr->rho_pq > 0) || !(pr->rho_va > 0) || !(pr->rho_uc > 0)) return 1;
    for (int i = 0; i < B; i++)
        if (!(pb->bus_vmin[i] > 0) || pb->bus_vmin[i] > pb->bus_vmax[i]) return 1;
    for (int g = 0; g < G; g++) {
        if (pb->gen_bus[g] < 0 || pb->gen_bus[g] >= B) return 1;
        if (pb->pmin[g] > pb->pmax[g] || pb->qmin[g] > pb->qmax[g] || pb->c2[g] < 0) return 1;
        if (pb->min_up[g] < 1 || pb->min_up[g] > T || pb->min_dn[g] < 1 || pb->min_dn[g] > T) return 1;
        if (pb->hold[g] < 0 || pb->hold[g] > T || (pb->u0[g] != 0 && pb->u0[g] != 1)) return 1;
    }
    for (int l = 0; l < L; l++) {
        if (pb->br_from[l] == pb->br_to[l]) return 1;
        if (pb->br_from[l] < 0 || pb->br_from[l] >= B || pb->br_to[l] < 0 || pb->br_to[l] >= B) return 1;
        for (int k = 0; k < 8; k++) if (bad(pb->br_y[l * 8 + k])) return 1;
    }
    orc_ctx *c = (orc_ctx *)calloc(1, sizeof(orc_ctx));
    c->pr = *pr;
    orc_problem *q = &c->pb;
    *q = *pb;
    size_t sB = sizeof(double) * B, sG = sizeof(double) * G, sL = sizeof(double) * L;
    q->bus_gs = cpy(c, pb->bus_gs, sB); q->bus_bs = cpy(c, pb->bus_bs, sB);
    q->bus_vmin = cpy(c, pb->bus_vmin, sB); q->bus_vmax = cpy(c, pb->bus_vmax, sB);
    q->pd = cpy(c, pb->pd, sB * T); q->qd = cpy(c, pb->qd, sB * T);
    q->br_from = cpy(c, pb->br_from, 4 * L); q->br_to = cpy(c, pb->br_to, 4 * L);
    q->br_y = cpy(c, pb->br_y, sL * 8); q->br_rate = cpy(c, pb->br_rate, sL);
    q->gen_bus = cpy(c, pb->gen_bus, 4 * G);
    q->pmin = cpy(c, pb->pmin, sG); q->pmax = cpy(c, pb->pmax, sG);
    q->qmin = cpy(c, pb->qmin, sG); q->qmax = cpy(c, pb->qmax, sG);
    q->c2 = cpy(c, pb->c2, sG); q->c1 = cpy(c, pb->c1, sG); q->c0 = cpy(c, pb->c0, sG);
    q->csu = cpy(c, pb->csu, sG); q->csd = cpy(c, pb->csd, sG);
    q->ramp_up = cpy(c, pb->ramp_up, sG); q->ramp_dn = cpy(c, pb->ramp_dn, sG);
    q->su_ramp = cpy(c, pb->su_ramp, sG); q->sd_ramp = cpy(c, pb->sd_ramp, sG);
    q->min_up = cpy(c, pb->min_up, 4 * G); q->min_dn = cpy(c, pb->min_dn, 4 * G);
    q->u0 = cpy(c, pb->u0, 4 * G); q->hold = cpy(c, pb->hold, 4 * G);
    q->p0 = cpy(c, pb->p0, sG);
    q->u_init = NULL;

    size_t GT = (size_t)G * T, LT = (size_t)L * T, BT = (size_t)B * T;
    c->u = (int8_t *)calloc(GT, 1);
    c->p = dz(GT); c->q = dz(GT); c->ph = dz(GT); c->sl = dz(6 * GT);
    c->x = dz(LT * 4); c->f = dz(LT * 4); c->al = dz(LT * 3);
    for (int k = 0; k < 3; k++) c->ub[k] = dz(GT);
    c->pbar = dz(GT); c->qbar = dz(GT); c->fbar = dz(LT * 4);
    c->wbar = dz(BT); c->thbar = dz(BT);
    c->zg = dz(NGR * GT); c->yg = dz(NGR * GT); c->lg = dz(NGR * GT);
    c->zb = dz(NBR * LT); c->yb = dz(NBR * LT); c->lb = dz(NBR * LT);

    /* CSR incidence in canonical order */
    c->bg_ptr = (int32_t *)calloc(B + 1, 4); c->be_ptr = (int32_t *)calloc(B + 1, 4);
    c->bg_idx = (int32_t *)calloc(G ? G : 1, 4); c->be_idx = (int32_t *)calloc(2 * L, 4);
    for (int g = 0; g < G; g++) c->bg_ptr[q->gen_bus[g] + 1]++;
    for (int l = 0; l < L; l++) { c->be_ptr[q->br_from[l] + 1]++; c->be_ptr[q->br_to[l] + 1]++; }
    for (int i = 0; i < B; i++) { c->bg_ptr[i + 1] += c->bg_ptr[i]; c->be_ptr[i + 1] += c->be_ptr[i]; }
    {
        int32_t *fg = (int32_t *)calloc(B, 4), *fe = (int32_t *)calloc(B, 4);
        for (int g = 0; g < G; g++) { int i = q->gen_bus[g]; c->bg_idx[c->bg_ptr[i] + fg[i]++] = g; }
        for (int l = 0; l < L; l++) {
            int i = q->br_from[l], j = q->br_to[l];
            c->be_idx[c->be_ptr[i] + fe[i]++] = 2 * l + 0;
            c->be_idx[c->be_ptr[j] + fe[j]++] = 2 * l + 1;
        }
        free(fg); free(fe);
    }
    for (int i = 0; i < B; i++) if (c->be_ptr[i + 1] == c->be_ptr[i]) { orc_destroy(c); return 1; }

    /* S0, cold start: p, q, |V| at bound midpoints, angles 0, flows from the
     * initial voltages; xbar = x so every consensus row starts at 0; schedule u_init or
     * "continue u0" (R23); y = z = lambda = 0; beta = beta0 (R21). */
    for (int g = 0; g < G; g++) {
        for (int t = 0; t < T; t++) {
            size_t k = (size_t)g * T + t;
            c->u[k] = pb->u_init ? pb->u_init[k] : (int8_t)q->u0[g];
            c->p[k] = 0.5 * (q->pmin[g] + q->pmax[g]);
            c->q[k] = 0.5 * (q->qmin[g] + q->qmax[g]);
        }
        for (int t = 0; t < T; t++) {
            size_t k = (size_t)g * T + t;
            c->ph[k] = t == 0 ? q->p0[g] : c->p[k - 1];
            int up = t == 0 ? q->u0[g] : c->u[k - 1];
            c->ub[0][k] = c->u[k];
            c->ub[1][k] = c->u[k] > up ? 1.0 : 0.0;
            c->ub[2][k] = up > c->u[k] ? 1.0 : 0.0;
            c->pbar[k] = c->p[k];
            c->qbar[k] = c->q[k];
        }
    }
    for (int i = 0; i < B; i++) {
        double v = 0.5 * (q->bus_vmin[i] + q->bus_vmax[i]);
        for (int t = 0; t < T; t++) { c->wbar[(size_t)i * T + t] = v * v; c->thbar[(size_t)i * T + t] = 0.0; }
    }
    for (int l = 0; l < L; l++) {
        int i = q->br_from[l], j = q->br_to[l];
        double vi = 0.5 * (q->bus_vmin[i] + q->bus_vmax[i]);
        double vj = 0.5 * (q->bus_vmin[j] + q->bus_vmax[j]);
        double r2 = q->br_rate[l] * q->br_rate[l];
        for (int t = 0; t < T; t++) {
            size_t k = (size_t)l * T + t;
            double *x = c->x + 4 * k;
            x[0] = vi * vi; x[1] = vj * vj; x[2] = 0.0; x[3] = 0.0;
            orc_branch_flows(q->br_y + 8 * l, x, c->f + 4 * k, NULL, NULL);
            for (int m = 0; m < 4; m++) c->fbar[4 * k + m] = c->f[4 * k + m];
            c->al[3 * k + 0] = 0.0; c->al[3 * k + 1] = 0.0;
            c->al[3 * k + 2] = pr->al_sigma0_rel * pr->rho_pq * r2;
        }
    }
    c->beta = pr->beta0;
    c->znorm_prev = 0.0;
    c->outer_k = 1;
    c->inner_total = 0;
    c->inner_since = 0;
    memset(&c->rep, 0, sizeof(c->rep));
    c->rep.beta = c->beta;
    for (int k = 0; k < 256; k++) c->phist[k] = NAN;
    c->done = 0;
    *out = c;
    return 0;
}

void orc_destroy(orc_ctx *c) {
    if (!c) return;
    for (int i = 0; i < c->nblk; i++) free(c->blk[i]);
    free(c->u); free(c->p); free(c->q); free(c->ph); free(c->sl);
    free(c->x); free(c->f); free(c->al);
    for (int k = 0; k < 3; k++) free(c->ub[k]);
    free(c->pbar); free(c->qbar); free(c->fbar); free(c->wbar); free(c->thbar);
    free(c->zg); free(c->yg); free(c->lg); free(c->zb); free(c->yb); free(c->lb);
    free(c->bg_ptr); free(c->bg_idx); free(c->be_ptr); free(c->be_idx);
    free(c);
}

#define ZG(k, i) c->zg[(size_t)(k) * GT + (i)]
#define YG(k, i) c->yg[(size_t)(k) * GT + (i)]
#define LG(k, i) c->lg[(size_t)(k) * GT + (i)]
#define ZB(k, i) c->zb[(size_t)(k) * LT + (i)]
#define YB(k, i) c->yb[(size_t)(k) * LT + (i)]
#define LB(k, i) c->lb[(size_t)(k) * LT + (i)]

typedef struct { double pinf, rzinf, rz2, zinf, z2, dinf; } norms;
/* (7e) z = argmin_z L = -(lambda + y + rho r)/(beta + rho), (7f) y += rho(r+z)
 * (P:238); norms for S8. */
/* the row's S8 terms are returned in rec[4] = (r, r + z, z, rho |dxbar|) and folded into the norms
 * afterwards in the canonical row order (so the OpenMP build sums in the same order) */
static void zy_row(double r, double rho, double beta, double *z, double *y, const double *lam,
                   double dxb, double *rec) {
    double zz = -((*lam + *y) + rho * r) / (beta + rho);
    *z = zz;
    *y = *y + rho * (r + zz);
    rec[0] = r;
    rec[1] = r + zz;
    rec[2] = zz;
    rec[3] = rho * fabs(dxb);
}
static void fold_row(const double *rec, norms *n) {
    n->pinf = dmax(n->pinf, fabs(rec[0]));
    n->rzinf = dmax(n->rzinf, fabs(rec[1]));
    n->rz2 = n->rz2 + rec[1] * rec[1];
    n->zinf = dmax(n->zinf, fabs(rec[2]));
    n->z2 = n->z2 + rec[2] * rec[2];
    n->dinf = dmax(n->dinf, rec[3]);
}

static void one_iteration(orc_ctx *c) {
    const orc_problem *q = &c->pb;
    const orc_params *pr = &c->pr;
    int B = q->nbus, G = q->ngen, L = q->nbranch, T = q->T;
    size_t GT = (size_t)G * T, LT = (size_t)L * T;
    double S = q->base_mva, rpq = pr->rho_pq, rva = pr->rho_va, ruc = pr->rho_uc;
    double beta = c->beta;

    /* keep x-bar^l for the dual residual */
    double *ubo[3], *pbo = dz(GT), *qbo = dz(GT), *fbo = dz(LT * 4);
    double *wbo = dz((size_t)B * T), *tbo = dz((size_t)B * T);
    for (int k = 0; k < 3; k++) { ubo[k] = dz(GT); memcpy(ubo[k], c->ub[k], sizeof(double) * GT); }
    memcpy(pbo, c->pbar, sizeof(double) * GT); memcpy(qbo, c->qbar, sizeof(double) * GT);
    memcpy(fbo, c->fbar, sizeof(double) * LT * 4);
    memcpy(wbo, c->wbar, sizeof(double) * B * T); memcpy(tbo, c->thbar, sizeof(double) * B * T);

    /* ---- (7a) x^UC by DP per generator (Alg. 2), on iterate l ---- */
    int8_t *unew = (int8_t *)calloc(GT, 1);
    if (pr->uc_fixed) {
        memcpy(unew, c->u, GT);   /* NEXT-2: the multiperiod ACOPF with the schedule held */
    } else {
#pragma omp parallel
        {
        double *Lt = dz((size_t)T * 4), *ub3 = dz((size_t)3 * T), *y3 = dz((size_t)3 * T), *z3 = dz((size_t)3 * T);
#pragma omp for schedule(static)
        for (int g = 0; g < G; g++) {
            for (int v = 0; v < 3; v++)
                for (int t = 0; t < T; t++) {
                    size_t i = (size_t)g * T + t;
                    ub3[v * T + t] = c->ub[v][i];
                    y3[v * T + t] = YG(D_ON + v, i);
                    z3[v * T + t] = ZG(D_ON + v, i);
                }
            orc_stage_costs(T, q->c0[g], q->csu[g], q->csd[g], ruc, ub3, y3, z3, Lt);
            if (pr->variant & 4) {
                /* NEXT-4(a), R50: a shutdown at t (u_{t-1} = 1, u_t = 0) needs p_{t-1} <= S^D by
                 * Eq. 4d; with the current dispatch above S^D that transition is excluded */
                for (int t = 0; t < T; t++) {
                    double pprev = t == 0 ? q->p0[g] : c->p[(size_t)g * T + t - 1];
                    if (pprev > q->sd_ramp[g]) Lt[t * 4 + 1 * 2 + 0] = INFINITY;
                }
            }
            orc_dp(T, Lt, q->min_up[g], q->min_dn[g], q->u0[g], q->hold[g], unew + (size_t)g * T);
        }
        free(Lt); free(ub3); free(y3); free(z3);
        }
    }

    /* ---- (7b) x^OPF: generators on iterate l ---- */
#pragma omp parallel for schedule(static)
    for (int g = 0; g < G; g++) {
        double pL = dmin(0.0, q->pmin[g]), pU = q->pmax[g];
        double qL = dmin(0.0, q->qmin[g]), qU = dmax(0.0, q->qmax[g]);
        for (int t = 0; t < T; t++) {
            size_t i = (size_t)g * T + t;
            double on = c->ub[0][i], su = c->ub[1][i], sd = c->ub[2][i];
            double onp = t == 0 ? (double)q->u0[g] : c->ub[0][i - 1];
            double in[19];
            in[0] = t == 0 ? 1.0 : 0.0;
            in[1] = q->c2[g] * S * S;
            in[2] = q->c1[g] * S;
            in[3] = rpq; in[4] = ruc;
            in[5] = c->pbar[i] - ZG(GP, i) - YG(GP, i) / rpq;
            in[6] = c->qbar[i] - ZG(GQ, i) - YG(GQ, i) / rpq;
            in[7] = t == 0 ? 0.0 : c->pbar[i - 1] - ZG(RC, i) - YG(RC, i) / rpq;
            in[8] = q->p0[g];
            in[9] = q->pmin[g] * on - ZG(PL, i) - YG(PL, i) / ruc;
            in[10] = q->pmax[g] * on - ZG(PU, i) - YG(PU, i) / ruc;
            in[11] = q->qmin[g] * on - ZG(QL, i) - YG(QL, i) / ruc;
            in[12] = q->qmax[g] * on - ZG(QU, i) - YG(QU, i) / ruc;
            /* RD row: Eq. 4d (R_D ubar^on_t + S_D ubar^sd_t), or the literal Eq. 5f
             * (R_D ubar^on_{t-1} + S_D ubar^su_t) with variant bit 16 (R52) */
            in[13] = (pr->variant & 16)
                ? -q->ramp_dn[g] * onp - q->sd_ramp[g] * su - ZG(RD, i) - YG(RD, i) / ruc
                : -q->ramp_dn[g] * on - q->sd_ramp[g] * sd - ZG(RD, i) - YG(RD, i) / ruc;
            in[14] = q->ramp_up[g] * onp + q->su_ramp[g] * su - ZG(RU, i) - YG(RU, i) / ruc;
            in[15] = pL; in[16] = pU; in[17] = qL; in[18] = qU;
            double o[3];
            orc_gen_x(in, o);
            c->p[i] = o[0]; c->q[i] = o[1]; c->ph[i] = o[2];
            double d = o[0] - o[2];
            double *s = c->sl + 6 * i;
            s[0] = dmax(0.0, o[0] - in[9]);
            s[1] = dmax(0.0, in[10] - o[0]);
            s[2] = dmax(0.0, o[1] - in[11]);
            s[3] = dmax(0.0, in[12] - o[1]);
            s[4] = dmax(0.0, d - in[13]);
            s[5] = dmax(0.0, in[14] - d);
        }
    }
    /* ---- (7b) x^OPF: branches ("six variables", P:456 ExaTron) ---- */
    int64_t tit = 0, tcap = 0, alact = 0, alcap = 0, nfast = 0, nal = 0;
    double ffast = 0.0, fal = 0.0;
    /* integer-valued sums: exact in any order */
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : tit, tcap, alact, alcap, nfast, nal, ffast, fal)
    for (int l = 0; l < L; l++) {
        int bi = q->br_from[l], bj = q->br_to[l];
        double wlo[2] = {q->bus_vmin[bi] * q->bus_vmin[bi], q->bus_vmin[bj] * q->bus_vmin[bj]};
        double whi[2] = {q->bus_vmax[bi] * q->bus_vmax[bi], q->bus_vmax[bj] * q->bus_vmax[bj]};
        for (int t = 0; t < T; t++) {
            size_t i = (size_t)l * T + t;
            double tau[8];
            for (int k = 0; k < 4; k++) tau[k] = c->fbar[4 * i + k] - ZB(k, i) - YB(k, i) / rpq;
            tau[4] = c->wbar[(size_t)bi * T + t] - ZB(W_I, i) - YB(W_I, i) / rva;
            tau[5] = c->wbar[(size_t)bj * T + t] - ZB(W_J, i) - YB(W_J, i) / rva;
            tau[6] = c->thbar[(size_t)bi * T + t] - ZB(A_I, i) - YB(A_I, i) / rva;
            tau[7] = c->thbar[(size_t)bj * T + t] - ZB(A_J, i) - YB(A_J, i) / rva;
            int64_t st[9];
            orc_branch_solve(q->br_y + 8 * l, wlo, whi, q->br_rate[l], tau, rpq, rva, pr,
                             c->x + 4 * i, c->al + 3 * i, c->f + 4 * i, st);
            tit += st[0];
            tcap += st[1];
            alact += st[2];
            alcap += st[4];
            ffast += (double)st[5];
            fal += (double)st[6];
            nfast += st[7];
            nal += st[8];
        }
    }
    memcpy(c->u, unew, GT);
    free(unew);

    /* ---- (7c) xbar^UC: ubar per (g, group) on x^{l+1}, u^{l+1} (R19) ---- */
    const int lit5f = (pr->variant & 16) != 0;
#pragma omp parallel for schedule(static)
    for (int g = 0; g < G; g++) {
        double Pm = q->pmin[g], PM = q->pmax[g], Qm = q->qmin[g], QM = q->qmax[g];
        double RDn = q->ramp_dn[g], SDn = q->sd_ramp[g], RUp = q->ramp_up[g], SUp = q->su_ramp[g];
        for (int t = -1; t < T; t++) {
            double cm[9 * 3], e[9];
            int m = 0, n;
            if (t < 0) {
                /* group 0 = (ubar^su_1): rows D_SU_1 and RU_1 (ubar^on_0 := u0, R4) */
                size_t i = (size_t)g * T;
                int u1 = c->u[i], su1 = u1 > q->u0[g];
                n = 1;
                cm[m * 3 + 0] = 1.0; cm[m * 3 + 1] = 0; cm[m * 3 + 2] = 0;
                e[m++] = (double)su1 + ZG(D_SU, i) + YG(D_SU, i) / ruc;
                cm[m * 3 + 0] = SUp; cm[m * 3 + 1] = 0; cm[m * 3 + 2] = 0;
                e[m++] = (c->p[i] - c->ph[i]) + c->sl[6 * i + 5] - RUp * (double)q->u0[g] + ZG(RU, i) + YG(RU, i) / ruc;
                if (lit5f) {   /* R52: RD_1 = (d - s) + R_D u0 + S_D ubar^su_1 */
                    cm[m * 3 + 0] = -SDn; cm[m * 3 + 1] = 0; cm[m * 3 + 2] = 0;
                    e[m++] = ((c->p[i] - c->ph[i]) - c->sl[6 * i + 4]) + RDn * (double)q->u0[g] + ZG(RD, i) + YG(RD, i) / ruc;
                }
                double v[3];
                orc_boxqp3(n, m, cm, e, v);
                c->ub[1][i] = v[0];
                continue;
            }
            size_t i = (size_t)g * T + t;
            int ut = c->u[i], uprev = t == 0 ? q->u0[g] : c->u[i - 1];
            int sdt = uprev > ut;
            n = (t < T - 1) ? 3 : 2;
            /* columns: (ubar^on_t, ubar^sd_t, ubar^su_{t+1}) */
#define ROW(c0_, c1_, c2_, ev) do { cm[m*3+0]=(c0_); cm[m*3+1]=(c1_); cm[m*3+2]=(c2_); e[m++]=(ev); } while (0)
            ROW(1.0, 0.0, 0.0, (double)ut + ZG(D_ON, i) + YG(D_ON, i) / ruc);
            ROW(0.0, 1.0, 0.0, (double)sdt + ZG(D_SD, i) + YG(D_SD, i) / ruc);
            ROW(Pm, 0.0, 0.0, (c->p[i] - c->sl[6 * i + 0]) + ZG(PL, i) + YG(PL, i) / ruc);
            ROW(PM, 0.0, 0.0, (c->p[i] + c->sl[6 * i + 1]) + ZG(PU, i) + YG(PU, i) / ruc);
            ROW(Qm, 0.0, 0.0, (c->q[i] - c->sl[6 * i + 2]) + ZG(QL, i) + YG(QL, i) / ruc);
            ROW(QM, 0.0, 0.0, (c->q[i] + c->sl[6 * i + 3]) + ZG(QU, i) + YG(QU, i) / ruc);
            if (!lit5f)
                ROW(-RDn, -SDn, 0.0, ((c->p[i] - c->ph[i]) - c->sl[6 * i + 4]) + ZG(RD, i) + YG(RD, i) / ruc);
            if (t < T - 1) {
                size_t j = i + 1;
                int sun = c->u[j] > ut;
                ROW(0.0, 0.0, 1.0, (double)sun + ZG(D_SU, j) + YG(D_SU, j) / ruc);
                ROW(RUp, 0.0, SUp, ((c->p[j] - c->ph[j]) + c->sl[6 * j + 5]) + ZG(RU, j) + YG(RU, j) / ruc);
                if (lit5f)   /* R52: RD_{t+1} = (d - s) + R_D ubar^on_t + S_D ubar^su_{t+1} */
                    ROW(-RDn, 0.0, -SDn, ((c->p[j] - c->ph[j]) - c->sl[6 * j + 4]) + ZG(RD, j) + YG(RD, j) / ruc);
            }
#undef ROW
            double v[3];
            orc_boxqp3(n, m, cm, e, v);
            c->ub[0][i] = v[0];
            c->ub[2][i] = v[1];
            if (t < T - 1) c->ub[1][i + 1] = v[2];
        }
    }

    /* ---- (7d) xbar^OPF: bus per (i,t) on x^{l+1} (R8) ---- */
    {
        int maxk = 0;
        for (int i = 0; i < B; i++) {
            int k = 2 * (c->bg_ptr[i + 1] - c->bg_ptr[i]) + 2 * (c->be_ptr[i + 1] - c->be_ptr[i]) + 1;
            if (k > maxk) maxk = k;
        }
#pragma omp parallel
        {
        double *al_ = dz(maxk), *be_ = dz(maxk), *aa = dz(maxk), *th = dz(maxk), *vv = dz(maxk);
#pragma omp for schedule(static)
        for (int i = 0; i < B; i++) {
            int ne = c->be_ptr[i + 1] - c->be_ptr[i];
            for (int t = 0; t < T; t++) {
                int k = 0;
                for (int a = c->bg_ptr[i]; a < c->bg_ptr[i + 1]; a++) {
                    int g = c->bg_idx[a];
                    size_t gi = (size_t)g * T + t;
                    double tgp = c->p[gi] + ZG(GP, gi) + YG(GP, gi) / rpq;
                    if (t < T - 1) {
                        double trc = c->ph[gi + 1] + ZG(RC, gi + 1) + YG(RC, gi + 1) / rpq;
                        th[k] = (tgp + trc) * 0.5;
                        aa[k] = 2.0 * rpq;
                    } else {
                        th[k] = tgp;
                        aa[k] = rpq;
                    }
                    al_[k] = 1.0; be_[k] = 0.0; k++;
                    th[k] = c->q[gi] + ZG(GQ, gi) + YG(GQ, gi) / rpq;
                    aa[k] = rpq; al_[k] = 0.0; be_[k] = 1.0; k++;
                }
                double wsum = 0.0, tsum = 0.0;
                for (int a = c->be_ptr[i]; a < c->be_ptr[i + 1]; a++) {
                    int l = c->be_idx[a] >> 1, side = c->be_idx[a] & 1;
                    size_t li = (size_t)l * T + t;
                    int kp = side ? FP_JI : FP_IJ, kq = side ? FQ_JI : FQ_IJ;
                    int kw = side ? W_J : W_I, ka = side ? A_J : A_I;
                    th[k] = c->f[4 * li + kp] + ZB(kp, li) + YB(kp, li) / rpq;
                    aa[k] = rpq; al_[k] = -1.0; be_[k] = 0.0; k++;
                    th[k] = c->f[4 * li + kq] + ZB(kq, li) + YB(kq, li) / rpq;
                    aa[k] = rpq; al_[k] = 0.0; be_[k] = -1.0; k++;
                    wsum = wsum + (c->x[4 * li + (side ? 1 : 0)] + ZB(kw, li) + YB(kw, li) / rva);
                    tsum = tsum + (c->x[4 * li + (side ? 3 : 2)] + ZB(ka, li) + YB(ka, li) / rva);
                }
                th[k] = wsum / (double)ne;
                aa[k] = (double)ne * rva;
                al_[k] = -q->bus_gs[i];
                be_[k] = q->bus_bs[i];
                k++;
                double mu[2];
                orc_bus_kkt(k, al_, be_, aa, th, q->pd[(size_t)t * B + i], q->qd[(size_t)t * B + i], vv, mu);
                /* scatter */
                k = 0;
                for (int a = c->bg_ptr[i]; a < c->bg_ptr[i + 1]; a++) {
                    int g = c->bg_idx[a];
                    size_t gi = (size_t)g * T + t;
                    c->pbar[gi] = vv[k++];
                    c->qbar[gi] = vv[k++];
                }
                for (int a = c->be_ptr[i]; a < c->be_ptr[i + 1]; a++) {
                    int l = c->be_idx[a] >> 1, side = c->be_idx[a] & 1;
                    size_t li = (size_t)l * T + t;
                    c->fbar[4 * li + (side ? FP_JI : FP_IJ)] = vv[k++];
                    c->fbar[4 * li + (side ? FQ_JI : FQ_IJ)] = vv[k++];
                }
                /* NEXT-3 variant 2 (R47): SPEC's clip of wbar to the voltage box */
                c->wbar[(size_t)i * T + t] = (pr->variant & 2)
                    ? clampd(vv[k], q->bus_vmin[i] * q->bus_vmin[i], q->bus_vmax[i] * q->bus_vmax[i]) : vv[k];
                /* R51: without angle rows thetabar is not a variable (kept at its start value) */
                if (!(pr->variant & 8))
                    c->thbar[(size_t)i * T + t] = (i == q->ref_bus) ? 0.0 : tsum / (double)ne;
            }
        }
        free(al_); free(be_); free(aa); free(th); free(vv);
        }
    }

    /* ---- (7e) z and (7f) y for every row; S8 norms ---- */
    norms nm = {0, 0, 0, 0, 0, 0};
    double obj = 0.0;
    /* per-row S8 terms (4 each) and per-(g,t) costs, folded below in the canonical row order */
    double *grec = dz((size_t)GT * NGR * 4), *brec = dz((size_t)LT * NBR * 4), *gcost = dz(GT);
#pragma omp parallel for schedule(static)
    for (int g = 0; g < G; g++) {
        double Pm = q->pmin[g], PM = q->pmax[g], Qm = q->qmin[g], QM = q->qmax[g];
        for (int t = 0; t < T; t++) {
            size_t i = (size_t)g * T + t;
            int ut = c->u[i], up = t == 0 ? q->u0[g] : c->u[i - 1];
            int su = ut > up, sd = up > ut;
            double on = c->ub[0][i], ubsu = c->ub[1][i], ubsd = c->ub[2][i];
            double onp = t == 0 ? (double)q->u0[g] : c->ub[0][i - 1];
            double don = on - ubo[0][i], dsu = ubsu - ubo[1][i], dsd = ubsd - ubo[2][i];
            double donp = t == 0 ? 0.0 : c->ub[0][i - 1] - ubo[0][i - 1];
            const double *s = c->sl + 6 * i;
            double p = c->p[i], qq = c->q[i], d = p - c->ph[i];
            double r[NGR], dx[NGR];
            r[D_ON] = (double)ut - on;            dx[D_ON] = don;
            r[D_SU] = (double)su - ubsu;          dx[D_SU] = dsu;
            r[D_SD] = (double)sd - ubsd;          dx[D_SD] = dsd;
            r[PL] = (p - s[0]) - Pm * on;         dx[PL] = Pm * don;
            r[PU] = (p + s[1]) - PM * on;         dx[PU] = PM * don;
            r[QL] = (qq - s[2]) - Qm * on;        dx[QL] = Qm * don;
            r[QU] = (qq + s[3]) - QM * on;        dx[QU] = QM * don;
            if (pr->variant & 16) {   /* literal Eq. 5f (R52) */
                r[RD] = (d - s[4]) + q->ramp_dn[g] * onp + q->sd_ramp[g] * ubsu;
                dx[RD] = q->ramp_dn[g] * donp + q->sd_ramp[g] * dsu;
            } else {
                r[RD] = (d - s[4]) + q->ramp_dn[g] * on + q->sd_ramp[g] * ubsd;
                dx[RD] = q->ramp_dn[g] * don + q->sd_ramp[g] * dsd;
            }
            r[RU] = (d + s[5]) - q->ramp_up[g] * onp - q->su_ramp[g] * ubsu;
            dx[RU] = q->ramp_up[g] * donp + q->su_ramp[g] * dsu;
            r[GP] = p - c->pbar[i];               dx[GP] = c->pbar[i] - pbo[i];
            r[GQ] = qq - c->qbar[i];              dx[GQ] = c->qbar[i] - qbo[i];
            r[RC] = t == 0 ? 0.0 : c->ph[i] - c->pbar[i - 1];
            dx[RC] = t == 0 ? 0.0 : c->pbar[i - 1] - pbo[i - 1];
            for (int k = 0; k < NGR; k++) {
                if (k == RC && t == 0) continue;
                double rho = (k >= GP) ? rpq : ruc;
                zy_row(r[k], rho, beta, &ZG(k, i), &YG(k, i), &LG(k, i), dx[k], grec + (i * NGR + k) * 4);
            }
            double Sp = S * p;
            gcost[i] = q->c2[g] * Sp * Sp + q->c1[g] * Sp + q->c0[g] * (double)ut
                     + q->csu[g] * (double)su + q->csd[g] * (double)sd;
        }
    }
#pragma omp parallel for schedule(static)
    for (int l = 0; l < L; l++) {
        int bi = q->br_from[l], bj = q->br_to[l];
        for (int t = 0; t < T; t++) {
            size_t i = (size_t)l * T + t;
            size_t wi = (size_t)bi * T + t, wj = (size_t)bj * T + t;
            double r[NBR], dx[NBR];
            for (int k = 0; k < 4; k++) {
                r[k] = c->f[4 * i + k] - c->fbar[4 * i + k];
                dx[k] = c->fbar[4 * i + k] - fbo[4 * i + k];
            }
            r[W_I] = c->x[4 * i + 0] - c->wbar[wi];   dx[W_I] = c->wbar[wi] - wbo[wi];
            r[W_J] = c->x[4 * i + 1] - c->wbar[wj];   dx[W_J] = c->wbar[wj] - wbo[wj];
            r[A_I] = c->x[4 * i + 2] - c->thbar[wi];  dx[A_I] = c->thbar[wi] - tbo[wi];
            r[A_J] = c->x[4 * i + 3] - c->thbar[wj];  dx[A_J] = c->thbar[wj] - tbo[wj];
            for (int k = 0; k < NBR; k++) {
                if ((pr->variant & 8) && (k == A_I || k == A_J)) continue;   /* R51 */
                double rho = (k < W_I) ? rpq : rva;
                zy_row(r[k], rho, beta, &ZB(k, i), &YB(k, i), &LB(k, i), dx[k], brec + (i * NBR + k) * 4);
            }
        }
    }
    /* S8 norms and the objective (Eq. 1a), sequential in the canonical order: gens (g, t, row
     * kind), then branches (l, t, row kind) */
    for (size_t i = 0; i < GT; i++) {
        int t = (int)(i % (size_t)T);
        for (int k = 0; k < NGR; k++) {
            if (k == RC && t == 0) continue;
            fold_row(grec + (i * NGR + k) * 4, &nm);
        }
        obj = obj + gcost[i];
    }
    for (size_t i = 0; i < LT; i++)
        for (int k = 0; k < NBR; k++) {
            if ((pr->variant & 8) && (k == A_I || k == A_J)) continue;
            fold_row(brec + (i * NBR + k) * 4, &nm);
        }
    free(grec); free(brec); free(gcost);
    for (int k = 0; k < 3; k++) free(ubo[k]);
    free(pbo); free(qbo); free(fbo); free(wbo); free(tbo);

    c->inner_total++;
    c->inner_since++;
    orc_report *rp = &c->rep;
    rp->primal_inf = nm.pinf; rp->rz_inf = nm.rzinf; rp->rz_2 = sqrt(nm.rz2);
    rp->z_inf = nm.zinf; rp->z_2 = sqrt(nm.z2); rp->dual_inf = nm.dinf; rp->objective = obj;
    rp->tron_iters += tit; rp->tron_capped += tcap; rp->al_active += alact; rp->al_capped += alcap;
    rp->flops_fast = ffast; rp->flops_al = fal; rp->newton_fast = nfast; rp->newton_al = nal;

    /* ---- S8 inner test, S9 outer update (Alg. 1 line 10; R20-R22) ---- */
    if (pr->outer_enabled && c->inner_since >= pr->inner_min) {
        double thr = dmax(pr->eps_inner_abs, 1e-2 / (double)c->outer_k);
        if (nm.rzinf <= thr || c->inner_since >= pr->inner_cap) {
            double zn = sqrt(nm.z2);
            for (size_t a = 0; a < NGR * GT; a++)
                c->lg[a] = clampd(c->lg[a] + beta * c->zg[a], -pr->lambda_max, pr->lambda_max);
            for (size_t a = 0; a < NBR * LT; a++)
                c->lb[a] = clampd(c->lb[a] + beta * c->zb[a], -pr->lambda_max, pr->lambda_max);
            if (c->outer_k > 1 && zn > pr->theta * c->znorm_prev)
                c->beta = dmin(pr->tau * c->beta, pr->beta_max);
            c->znorm_prev = zn;
            c->outer_k++;
            c->inner_since = 0;
        }
    }
    rp->beta = c->beta;
    rp->inner_total = c->inner_total;
    rp->outer_total = c->outer_k - 1;
    rp->inner_since_outer = (int32_t)c->inner_since;
    rp->outer_k = (int32_t)c->outer_k;

    /* ---- divergence detector ("primal residual grows 10x over 200 inner iterations
     * -> abort with diagnostics"): primal_i > factor * primal_{i - window} ends the call ---- */
    {
        const int64_t it = c->inner_total;
        c->phist[(it - 1) % 256] = nm.pinf;
        const int w = pr->diverge_window;
        if (w > 0 && it > w && rp->diverged_iter == 0) {
            const double old = c->phist[(it - 1 - w) % 256];
            if (nm.pinf > pr->diverge_factor * old) {
                rp->diverged_iter = (int32_t)it;
                c->done = 1;
            }
        }
    }
}

int orc_iterate(orc_ctx *c, int32_t n) {
    c->done = 0;   /* (a call that the detector ended: the next call continues) */
    for (int k = 0; k < n && !c->done; k++) one_iteration(c);
    return 0;
}

void orc_report_get(const orc_ctx *c, orc_report *r) { *r = c->rep; }

/* NEXT-4(b), R53: new penalty classes between iterations; every rho-derived quantity of the
 * steps is formed from c->pr at its use, and the iterate is kept. */
void orc_set_rho(orc_ctx *c, double rho_pq, double rho_va, double rho_uc) {
    c->pr.rho_pq = rho_pq;
    c->pr.rho_va = rho_va;
    c->pr.rho_uc = rho_uc;
}

void orc_get_state(const orc_ctx *c, orc_state *s) {
    size_t GT = (size_t)c->pb.ngen * c->pb.T, LT = (size_t)c->pb.nbranch * c->pb.T;
    size_t BT = (size_t)c->pb.nbus * c->pb.T, D = sizeof(double);
    memcpy(s->u, c->u, GT);
    memcpy(s->p, c->p, D * GT); memcpy(s->q, c->q, D * GT); memcpy(s->ph, c->ph, D * GT);
    memcpy(s->ub_on, c->ub[0], D * GT); memcpy(s->ub_su, c->ub[1], D * GT); memcpy(s->ub_sd, c->ub[2], D * GT);
    memcpy(s->pbar, c->pbar, D * GT); memcpy(s->qbar, c->qbar, D * GT);
    memcpy(s->zg, c->zg, D * GT * NGR); memcpy(s->yg, c->yg, D * GT * NGR); memcpy(s->lg, c->lg, D * GT * NGR);
    memcpy(s->x, c->x, D * LT * 4); memcpy(s->f, c->f, D * LT * 4); memcpy(s->fbar, c->fbar, D * LT * 4);
    memcpy(s->al, c->al, D * LT * 3);
    memcpy(s->zb, c->zb, D * LT * NBR); memcpy(s->yb, c->yb, D * LT * NBR); memcpy(s->lb, c->lb, D * LT * NBR);
    memcpy(s->wbar, c->wbar, D * BT); memcpy(s->thbar, c->thbar, D * BT);
    s->scal[0] = c->beta; s->scal[1] = c->znorm_prev; s->scal[2] = (double)c->outer_k;
    s->scal[3] = (double)c->inner_total; s->scal[4] = (double)c->inner_since;
    s->scal[5] = s->scal[6] = s->scal[7] = 0.0;
}

void orc_set_state(orc_ctx *c, const orc_state *s) {
    size_t GT = (size_t)c->pb.ngen * c->pb.T, LT = (size_t)c->pb.nbranch * c->pb.T;
    size_t BT = (size_t)c->pb.nbus * c->pb.T, D = sizeof(double);
    memcpy(c->u, s->u, GT);
    memcpy(c->p, s->p, D * GT); memcpy(c->q, s->q, D * GT); memcpy(c->ph, s->ph, D * GT);
    memcpy(c->ub[0], s->ub_on, D * GT); memcpy(c->ub[1], s->ub_su, D * GT); memcpy(c->ub[2], s->ub_sd, D * GT);
    memcpy(c->pbar, s->pbar, D * GT); memcpy(c->qbar, s->qbar, D * GT);
    memcpy(c->zg, s->zg, D * GT * NGR); memcpy(c->yg, s->yg, D * GT * NGR); memcpy(c->lg, s->lg, D * GT * NGR);
    memcpy(c->x, s->x, D * LT * 4); memcpy(c->f, s->f, D * LT * 4); memcpy(c->fbar, s->fbar, D * LT * 4);
    memcpy(c->al, s->al, D * LT * 3);
    memcpy(c->zb, s->zb, D * LT * NBR); memcpy(c->yb, s->yb, D * LT * NBR); memcpy(c->lb, s->lb, D * LT * NBR);
    memcpy(c->wbar, s->wbar, D * BT); memcpy(c->thbar, s->thbar, D * BT);
    c->beta = s->scal[0]; c->znorm_prev = s->scal[1]; c->outer_k = (int64_t)s->scal[2];
    c->inner_total = (int64_t)s->scal[3]; c->inner_since = (int64_t)s->scal[4];
    /* the residual history belongs to the replaced trajectory */
    for (int k = 0; k < 256; k++) c->phist[k] = NAN;
    c->rep.diverged_iter = 0;
}

void orc_get_slacks(const orc_ctx *c, double *sl) {
    memcpy(sl, c->sl, sizeof(double) * 6 * (size_t)c->pb.ngen * c->pb.T);
}

/* The all-core build (liboracle_omp.so, -fopenmp): the per-component loops of
 * each step run in parallel, every reduction (S8 norms, objective) stays sequential in the
 * canonical order, so its iterates are bitwise those of the single-thread build
 * (tests/test_oracle_admm.py::test_openmp_build_is_bitwise_the_serial_oracle). */
int orc_threads(int32_t n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}
