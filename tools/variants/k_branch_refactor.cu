// k_branch.cu -- step (7b) line part: one bound-constrained trust-region Newton solve per
// (branch, period) ("tiny nonlinear optimization problem with six variables",
// P:456 ExaTron), batched over all L*T pairs, fp64 on sm_100a.
//
// Mapping: one THREAD per (l,t) solve -- the 4- (or 6-) variable Newton
// system, its gradient and Hessian live in registers; there is no cross-lane work at all,
// so all 32 lanes do useful FP64 math (a warp-per-solve mapping would leave >= 28 lanes
// idle for n <= 6).  Consecutive threads are consecutive (l,t) pairs, so every row array
// load/store of the warp is one coalesced 256-B segment.
//
// Flows are linear in phi = (w_i, w_j, C, S) with C = sqrt(w_i w_j) cos(th_i - th_j),
// S = sqrt(w_i w_j) sin(...) (Eq. 2e-2j): f = M phi.  Hence
//   grad_x F = J^T G_phi + rho_va (x - tau_x),
//   Hess_x F = J^T K_phi J + G_C d2C + G_S d2S + rho_va I,  K_phi = rho_pq M^T M (+ AL terms)
// with J = d phi / d x.  K_phi has 7 distinct entries for the plain problem.
//
// The TRON variant (Cauchy search, Steihaug-Toint CG on the free variables, projected
// search, ratio test) is the one specified in DESIGN.md 5.3; the oracle implements the same
// algorithm independently (oracle/oracle.c) with a straightforward evaluation.
#include "ucac_dev.cuh"
#ifdef UCAC_PROF
#include <cstdio>
#endif

#ifndef UCAC_TRON_DIRECT
#define UCAC_TRON_DIRECT 0   // 1: Newton step by LDL^T when it is interior (tried)
#endif

namespace ucac {
namespace {

constexpr double TR_MU0 = 0.01, TR_ETA0 = 1e-4, TR_ETA1 = 0.25, TR_ETA2 = 0.75;
constexpr double TR_SIG1 = 0.25, TR_SIG3 = 4.0, TR_DELTA0 = 1.0, TR_CGTOL = 1e-12;
constexpr double TR_EPSF = 1e-10, TR_STALL = 1e-14;
constexpr double TWO_PI = 6.283185307179586;

template <bool AL>
struct BrFun {
    double Gii, Gij, Gji, Gjj, Bii, Bij, Bji, Bjj;
    double tau[8];
    double rpq, rva;
    double K00, K02, K03, K11, K12, K13, K22;   // rho_pq M^T M (K01 = K23 = 0, K33 = K22)
    double mu0, mu1, sig, r2inv;                // AL only

    __device__ __forceinline__ void setup() {
        K00 = rpq * (Gii * Gii + Bii * Bii);
        K02 = rpq * (Gii * Gij + Bii * Bij);
        K03 = rpq * (Gii * Bij - Bii * Gij);
        K11 = rpq * (Gjj * Gjj + Bjj * Bjj);
        K12 = rpq * (Gjj * Gji + Bjj * Bji);
        K13 = rpq * (Bjj * Gji - Gjj * Bji);
        K22 = rpq * (Gij * Gij + Bij * Bij + Gji * Gji + Bji * Bji);
    }

    __device__ __forceinline__ void flows(const double *x, double &C, double &S, double &f0,
                                          double &f1, double &f2, double &f3) const {
        double R = sqrt(x[0] * x[1]);
        double sn, cs;
        sincos(x[2] - x[3], &sn, &cs);
        C = R * cs;
        S = R * sn;
        f0 = Gii * x[0] + Gij * C + Bij * S;
        f1 = -Bii * x[0] - Bij * C + Gij * S;
        f2 = Gjj * x[1] + Gji * C - Bji * S;
        f3 = -Bjj * x[1] - Bji * C - Gji * S;
    }

    // objective only
    __device__ __forceinline__ double value(const double *x) const {
        double C, S, f0, f1, f2, f3;
        flows(x, C, S, f0, f1, f2, f3);
        double e0 = f0 - tau[0], e1 = f1 - tau[1], e2 = f2 - tau[2], e3 = f3 - tau[3];
        double F = 0.5 * rpq * (e0 * e0 + e1 * e1 + e2 * e2 + e3 * e3);
        double v = 0.0;
#pragma unroll
        for (int m = 0; m < 4; m++) {
            double d = x[m] - tau[4 + m];
            v += d * d;
        }
        F += 0.5 * rva * v;
        if (AL) {
            double h0 = (f0 * f0 + f1 * f1) * r2inv - 1.0 + x[4];
            double h1 = (f2 * f2 + f3 * f3) * r2inv - 1.0 + x[5];
            F += mu0 * h0 + 0.5 * sig * h0 * h0 + mu1 * h1 + 0.5 * sig * h1 * h1;
        }
        return F;
    }

    // objective, gradient and (optionally) Hessian
    template <int N, bool HESS>
    __device__ __forceinline__ void eval(const double *x, double &F, double *g, double (*H)[N]) const {
        double C, S, f0, f1, f2, f3;
        flows(x, C, S, f0, f1, f2, f3);
        double e0 = f0 - tau[0], e1 = f1 - tau[1], e2 = f2 - tau[2], e3 = f3 - tau[3];
        F = 0.5 * rpq * (e0 * e0 + e1 * e1 + e2 * e2 + e3 * e3);
        double v = 0.0;
#pragma unroll
        for (int m = 0; m < 4; m++) {
            double d = x[m] - tau[4 + m];
            v += d * d;
        }
        F += 0.5 * rva * v;
        // phi-space gradient rho_pq M^T e
        double Gw0 = rpq * (e0 * Gii - e1 * Bii);
        double Gw1 = rpq * (e2 * Gjj - e3 * Bjj);
        double GC = rpq * (e0 * Gij - e1 * Bij + e2 * Gji - e3 * Bji);
        double GS = rpq * (e0 * Bij + e1 * Gij - e2 * Bji - e3 * Gji);
        double k00 = K00, k01 = 0.0, k02 = K02, k03 = K03, k11 = K11, k12 = K12, k13 = K13;
        double k22 = K22, k23 = 0.0, k33 = K22;
        double dh0[4], dh1[4], lam0 = 0.0, lam1 = 0.0;
        if (AL) {
            double h0 = (f0 * f0 + f1 * f1) * r2inv - 1.0 + x[4];
            double h1 = (f2 * f2 + f3 * f3) * r2inv - 1.0 + x[5];
            F += mu0 * h0 + 0.5 * sig * h0 * h0 + mu1 * h1 + 0.5 * sig * h1 * h1;
            double tw = 2.0 * r2inv;
            dh0[0] = tw * (f0 * Gii - f1 * Bii);
            dh0[1] = 0.0;
            dh0[2] = tw * (f0 * Gij - f1 * Bij);
            dh0[3] = tw * (f0 * Bij + f1 * Gij);
            dh1[0] = 0.0;
            dh1[1] = tw * (f2 * Gjj - f3 * Bjj);
            dh1[2] = tw * (f2 * Gji - f3 * Bji);
            dh1[3] = tw * (-f2 * Bji - f3 * Gji);
            lam0 = mu0 + sig * h0;
            lam1 = mu1 + sig * h1;
            Gw0 += lam0 * dh0[0];
            Gw1 += lam1 * dh1[1];
            GC += lam0 * dh0[2] + lam1 * dh1[2];
            GS += lam0 * dh0[3] + lam1 * dh1[3];
            if (HESS) {
                double a0 = lam0 * tw, a1 = lam1 * tw;
                k00 += a0 * (Gii * Gii + Bii * Bii) + sig * dh0[0] * dh0[0];
                k02 += a0 * (Gii * Gij + Bii * Bij) + sig * dh0[0] * dh0[2];
                k03 += a0 * (Gii * Bij - Bii * Gij) + sig * dh0[0] * dh0[3];
                k11 += a1 * (Gjj * Gjj + Bjj * Bjj) + sig * dh1[1] * dh1[1];
                k12 += a1 * (Gjj * Gji + Bjj * Bji) + sig * dh1[1] * dh1[2];
                k13 += a1 * (Bjj * Gji - Gjj * Bji) + sig * dh1[1] * dh1[3];
                double m0 = a0 * (Gij * Gij + Bij * Bij), m1 = a1 * (Gji * Gji + Bji * Bji);
                k22 += m0 + m1 + sig * (dh0[2] * dh0[2] + dh1[2] * dh1[2]);
                k33 += m0 + m1 + sig * (dh0[3] * dh0[3] + dh1[3] * dh1[3]);
                k23 += sig * (dh0[2] * dh0[3] + dh1[2] * dh1[3]);
                k01 += sig * (dh0[0] * dh0[1] + dh1[0] * dh1[1]);
            }
        }
        double i2wi = 0.5 / x[0], i2wj = 0.5 / x[1];
        double dC[4] = {C * i2wi, C * i2wj, -S, S};
        double dS[4] = {S * i2wi, S * i2wj, C, -C};
#pragma unroll
        for (int m = 0; m < 4; m++) g[m] = GC * dC[m] + GS * dS[m] + rva * (x[m] - tau[4 + m]);
        g[0] += Gw0;
        g[1] += Gw1;
        if (AL) {
            g[4] = lam0;
            g[5] = lam1;
        }
        if (!HESS) return;
        // P = K_phi J  (rows a = phi index, cols m = x index)
        double P[4][4];
        const double Kr[4][4] = {{k00, k01, k02, k03}, {k01, k11, k12, k13}, {k02, k12, k22, k23},
                                 {k03, k13, k23, k33}};
#pragma unroll
        for (int a = 0; a < 4; a++) {
#pragma unroll
            for (int m = 0; m < 4; m++) P[a][m] = Kr[a][2] * dC[m] + Kr[a][3] * dS[m];
            P[a][0] += Kr[a][0];
            P[a][1] += Kr[a][1];
        }
#pragma unroll
        for (int m = 0; m < 4; m++) {
#pragma unroll
            for (int n = m; n < 4; n++) {
                double h = dC[m] * P[2][n] + dS[m] * P[3][n];
                if (m == 0) h += P[0][n];
                if (m == 1) h += P[1][n];
                H[m][n] = h;
            }
        }
        // curvature of C, S
        double A = GC * C + GS * S, Bq = GS * C - GC * S;
        H[0][0] += -A * i2wi * i2wi;
        H[1][1] += -A * i2wj * i2wj;
        H[0][1] += A * i2wi * i2wj;
        H[0][2] += Bq * i2wi;
        H[0][3] += -Bq * i2wi;
        H[1][2] += Bq * i2wj;
        H[1][3] += -Bq * i2wj;
        H[2][2] += -A;
        H[3][3] += -A;
        H[2][3] += A;
#pragma unroll
        for (int m = 0; m < 4; m++) H[m][m] += rva;
        if (AL) {
#pragma unroll
            for (int m = 0; m < 4; m++) {
                double j0 = dh0[2] * dC[m] + dh0[3] * dS[m];
                double j1 = dh1[2] * dC[m] + dh1[3] * dS[m];
                if (m == 0) { j0 += dh0[0]; j1 += dh1[0]; }
                if (m == 1) { j0 += dh0[1]; j1 += dh1[1]; }
                H[m][4] = sig * j0;
                H[m][5] = sig * j1;
            }
            H[4][4] = sig;
            H[5][5] = sig;
            H[4][5] = 0.0;
        }
#pragma unroll
        for (int m = 0; m < N; m++)
#pragma unroll
            for (int n = 0; n < m; n++) H[m][n] = H[n][m];
    }
};

// pairwise partial sums: half the dependent-FMA chain of a running sum
template <int N>
__device__ __forceinline__ double dotn(const double *a, const double *b) {
    double s = a[0] * b[0] + a[1] * b[1];
#pragma unroll
    for (int i = 2; i + 1 < N; i += 2) s += a[i] * b[i] + a[i + 1] * b[i + 1];
    if (N & 1) s += a[N - 1] * b[N - 1];
    return s;
}
template <int N>
__device__ __forceinline__ void matvec(const double (*H)[N], const double *v, double *o) {
#pragma unroll
    for (int i = 0; i < N; i++) o[i] = dotn<N>(H[i], v);
}
// compare/select clamp (the oracle's form; cheaper than fmin/fmax with their NaN handling)
__device__ __forceinline__ double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

template <int N>
__device__ __forceinline__ void pstep(const double *x, const double *lo, const double *hi,
                                      const double *g, double a, double *s) {
#pragma unroll
    for (int i = 0; i < N; i++) s[i] = clampd(x[i] - a * g[i], lo[i], hi[i]) - x[i];
}
template <int N>
__device__ __forceinline__ double bnd_tau(const double *a, const double *p, double delta) {
    double aa = dotn<N>(a, a), ap = dotn<N>(a, p), pp = dotn<N>(p, p);
    if (pp <= 0.0) return 0.0;
    double gap = fmax(delta * delta - aa, 0.0);
    double rad = sqrt(ap * ap + pp * gap);
    return ap > 0.0 ? gap / (ap + rad) : (rad - ap) / pp;
}

// Projected trust-region Newton, split into begin / converged / iterate so a
// caller can interleave iterations of different solves (the flattened AL loop of k_branch_al).
template <int N>
struct Tron {
    double f, g[N], H[N][N], delta, alpha;
    int it;

    template <class Fun>
    __device__ __forceinline__ void begin(const Fun &fn, double *x, const double *lo, const double *hi) {
#pragma unroll
        for (int i = 0; i < N; i++) x[i] = clampd(x[i], lo[i], hi[i]);
        fn.template eval<N, true>(x, f, g, H);
        delta = TR_DELTA0;
        alpha = 1.0;
        it = 0;
        // first Cauchy trial length: the model minimiser along -g (R41)
        double Hg[N];
        matvec<N>(H, g, Hg);
        const double gHg = dotn<N>(g, Hg), gg = dotn<N>(g, g);
        if (gHg > 0.0 && gg > 0.0) alpha = gg / gHg;
    }
    // ||P(x - g) - x||_inf <= gtol
    __device__ __forceinline__ bool converged(const double *x, const double *lo, const double *hi,
                                              double gtol) const {
        double pgn = 0.0;
#pragma unroll
        for (int i = 0; i < N; i++) pgn = fmax(pgn, fabs(clampd(x[i] - g[i], lo[i], hi[i]) - x[i]));
        return pgn <= gtol;
    }
    // one iteration (Cauchy point, CG, projected search, ratio test); true = stall stop
    template <class Fun>
    __device__ __forceinline__ bool iterate(const Fun &fn, double *x, const double *lo, const double *hi);
};

// One Cauchy trial s = P(x - a g) - x: returns whether the sufficient-decrease and trust-region
// tests hold, and the model value q(s).  While only the coordinates pinned at a bound (gm = 0)
// are clamped, s = -a gm and q(s) = -a gm.gm + a^2/2 gm'H gm, O(N) instead of a mat-vec.
template <int N>
__device__ __forceinline__ bool cauchy_trial(const double *x, const double *lo, const double *hi, const double *g,
                                             const double *gm, const double (*H)[N], double gg, double gHg,
                                             double a, double d2, double *s, double &q, bool &simple) {
    simple = true;
#pragma unroll
    for (int i = 0; i < N; i++) {
        const double v = x[i] - a * g[i];
        s[i] = clampd(v, lo[i], hi[i]) - x[i];
        simple = simple && (gm[i] == 0.0 || (v >= lo[i] && v <= hi[i]));
    }
    double ss, gs;
    if (simple) {
        ss = a * a * gg;
        gs = -a * gg;
        q = gs + 0.5 * a * a * gHg;
    } else {
        double Hs[N];
        matvec<N>(H, s, Hs);
        ss = dotn<N>(s, s);
        gs = dotn<N>(g, s);
        q = gs + 0.5 * dotn<N>(s, Hs);
    }
    return ss <= d2 && q <= TR_MU0 * gs;
}

// Newton step on the free set F by an LDL^T factorisation of H_FF (fixed rows/columns
// replaced by the identity).  Returns false if H_FF is not positive definite.
template <int N>
__device__ __forceinline__ bool newton_free(const double (*H)[N], const bool *fr, const double *r, double *w) {
    double Lm[N][N], D[N];
    bool pd = true;
#pragma unroll
    for (int j = 0; j < N; j++) {
        double dj = fr[j] ? H[j][j] : 1.0;
#pragma unroll
        for (int k = 0; k < j; k++) dj -= Lm[j][k] * Lm[j][k] * D[k];
        pd = pd && dj > 0.0;
        D[j] = dj;
        const double inv = 1.0 / dj;
#pragma unroll
        for (int i = j + 1; i < N; i++) {
            double v = (fr[i] && fr[j]) ? H[i][j] : 0.0;
#pragma unroll
            for (int k = 0; k < j; k++) v -= Lm[i][k] * Lm[j][k] * D[k];
            Lm[i][j] = v * inv;
        }
    }
    if (!pd) return false;
    double z[N];
#pragma unroll
    for (int i = 0; i < N; i++) {
        double v = r[i];
#pragma unroll
        for (int k = 0; k < i; k++) v -= Lm[i][k] * z[k];
        z[i] = v;
    }
#pragma unroll
    for (int i = N - 1; i >= 0; i--) {
        double v = z[i] / D[i];
#pragma unroll
        for (int k = i + 1; k < N; k++) v -= Lm[k][i] * w[k];
        w[i] = fr[i] ? v : 0.0;
    }
    return true;
}

template <int N>
template <class Fun>
__device__ __forceinline__ bool Tron<N>::iterate(const Fun &fn, double *x, const double *lo, const double *hi) {
    const double d2 = delta * delta;
    // --- Cauchy point: backtrack (x0.1) or extrapolate (x10) along P(x - a g)
    double sc[N], qc, gq[N];   // Cauchy step, its model value, model gradient g + H sc
    bool csimple;
    {
        double gm[N], Hgm[N];
#pragma unroll
        for (int i = 0; i < N; i++) {
            const bool pinned = (x[i] <= lo[i] && g[i] > 0.0) || (x[i] >= hi[i] && g[i] < 0.0);
            gm[i] = pinned ? 0.0 : g[i];
        }
        matvec<N>(H, gm, Hgm);
        const double gg = dotn<N>(gm, gm), gHg = dotn<N>(gm, Hgm);
        double a = alpha;
        if (!cauchy_trial<N>(x, lo, hi, g, gm, H, gg, gHg, a, d2, sc, qc, csimple)) {
            for (int k = 0; k < 60; k++) {
                a *= 0.1;
                if (cauchy_trial<N>(x, lo, hi, g, gm, H, gg, gHg, a, d2, sc, qc, csimple)) break;
            }
        } else {
            for (int k = 0; k < 20; k++) {
                double sn[N], qn;
                bool sim;
                const bool ok = cauchy_trial<N>(x, lo, hi, g, gm, H, gg, gHg, 10.0 * a, d2, sn, qn, sim);
                bool same = true;
#pragma unroll
                for (int i = 0; i < N; i++) same = same && (sn[i] == sc[i]);
                if (!ok || same) break;
                a *= 10.0;
#pragma unroll
                for (int i = 0; i < N; i++) sc[i] = sn[i];
                qc = qn;
                csimple = sim;
            }
        }
        alpha = a;
        // gradient of the model at the Cauchy point, gq = g + H sc
        if (csimple) {
#pragma unroll
            for (int i = 0; i < N; i++) gq[i] = g[i] - a * Hgm[i];
        } else {
            double Hs[N];
            matvec<N>(H, sc, Hs);
#pragma unroll
            for (int i = 0; i < N; i++) gq[i] = g[i] + Hs[i];
        }
    }
    // --- subspace step on the free variables at x + sc, region ||sc + w|| <= delta:
    // the Newton step when H_FF is positive definite and it lies inside the region (the point
    // Steihaug-Toint CG converges to), otherwise Steihaug-Toint CG itself
    bool fr[N];
    double w[N];
    {
        double r[N];
#pragma unroll
        for (int i = 0; i < N; i++) {
            const double xc = x[i] + sc[i];
            fr[i] = (xc > lo[i]) && (xc < hi[i]);
            r[i] = fr[i] ? -gq[i] : 0.0;
            w[i] = 0.0;
        }
        double rr = dotn<N>(r, r);
        if (rr != 0.0) {
            bool done = false;
            if (UCAC_TRON_DIRECT && newton_free<N>(H, fr, r, w)) {
                double t[N];
#pragma unroll
                for (int i = 0; i < N; i++) t[i] = sc[i] + w[i];
                done = dotn<N>(t, t) < d2;
            }
            if (!done) {
                double p[N];
#pragma unroll
                for (int i = 0; i < N; i++) {
                    w[i] = 0.0;
                    p[i] = r[i];
                }
                const double tol2 = TR_CGTOL * TR_CGTOL * rr;
                for (int k = 0; k < N; k++) {
                    double Hp[N], t[N];
                    matvec<N>(H, p, Hp);
#pragma unroll
                    for (int i = 0; i < N; i++) if (!fr[i]) Hp[i] = 0.0;
                    double kap = dotn<N>(p, Hp);
#pragma unroll
                    for (int i = 0; i < N; i++) t[i] = sc[i] + w[i];
                    if (kap <= 0.0) {
                        double tau = bnd_tau<N>(t, p, delta);
#pragma unroll
                        for (int i = 0; i < N; i++) w[i] += tau * p[i];
                        break;
                    }
                    double a = rr / kap;
                    double tt[N];
#pragma unroll
                    for (int i = 0; i < N; i++) tt[i] = t[i] + a * p[i];
                    if (dotn<N>(tt, tt) >= d2) {
                        double tau = bnd_tau<N>(t, p, delta);
#pragma unroll
                        for (int i = 0; i < N; i++) w[i] += tau * p[i];
                        break;
                    }
#pragma unroll
                    for (int i = 0; i < N; i++) {
                        w[i] += a * p[i];
                        r[i] -= a * Hp[i];
                    }
                    double rn = dotn<N>(r, r);
                    if (rn <= tol2) break;
                    double b = rn / rr;
#pragma unroll
                    for (int i = 0; i < N; i++) p[i] = r[i] + b * p[i];
                    rr = rn;
                }
            }
        }
    }
    // --- projected search along w from the Cauchy point; q(sc + d) = qc + gq.d + d'Hd/2
    double s[N], qs = qc;
    {
        double b = 1.0;
        bool found = false;
        for (int k = 0; k < 20; k++) {
            double ds[N], Hd[N];
#pragma unroll
            for (int i = 0; i < N; i++) {
                s[i] = clampd(x[i] + sc[i] + b * w[i], lo[i], hi[i]) - x[i];
                ds[i] = s[i] - sc[i];
            }
            matvec<N>(H, ds, Hd);
            const double gd = dotn<N>(gq, ds);
            const double q = qc + gd + 0.5 * dotn<N>(ds, Hd);
            if (q <= qc + TR_MU0 * gd) {
                found = true;
                qs = q;
                break;
            }
            b *= 0.5;
        }
        if (!found) {
#pragma unroll
            for (int i = 0; i < N; i++) s[i] = sc[i];
        }
    }
    const double ss = dotn<N>(s, s);
    // --- stall: a step at the rounding level of x means the gradient floor is reached
    {
        double xm = 0.0;
#pragma unroll
        for (int i = 0; i < N; i++) xm = fmax(xm, fabs(x[i]));
        const double tol = TR_STALL * (1.0 + xm);
        if (ss <= tol * tol) return true;
    }
    // --- ratio test
    const double pred = -qs;
    double xn[N], gn[N], fnew;
#pragma unroll
    for (int i = 0; i < N; i++) xn[i] = clampd(x[i] + s[i], lo[i], hi[i]);
    fn.template eval<N, false>(xn, fnew, gn, nullptr);
    double ared = f - fnew;
    if (fabs(pred) <= TR_EPSF * fabs(f)) ared = -0.5 * (dotn<N>(g, s) + dotn<N>(gn, s));
    const double ratio = pred > 0.0 ? ared / pred : -1.0;
    const double snorm = sqrt(ss);
    if (ratio > TR_ETA0) {
#pragma unroll
        for (int i = 0; i < N; i++) x[i] = xn[i];
        fn.template eval<N, true>(x, f, g, H);
    }
    if (ratio < TR_ETA1) delta = TR_SIG1 * fmin(snorm, delta);
    else if (ratio > TR_ETA2) delta = fmax(delta, TR_SIG3 * snorm);
    it++;
    return false;
}

// Whole solve.  Returns true when ||P(x-g)-x||_inf <= gtol (or the step stalled at rounding).
template <int N, class Fun>
__device__ __forceinline__ bool tron(const Fun &fn, double *x, const double *lo, const double *hi, double gtol,
                                     int maxit, int &iters) {
    Tron<N> S;
    S.begin(fn, x, lo, hi);
    for (;;) {
        if (S.converged(x, lo, hi, gtol)) break;
        if (S.it >= maxit) {
            iters = S.it;
            return false;
        }
        if (S.iterate(fn, x, lo, hi)) break;
    }
    iters = S.it;
    return true;
}

__device__ __forceinline__ void warp_add_u64(unsigned long long *dst, unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// load the data of solve k = l*T + t: admittances, targets tau = xbar - z - y/rho (5.1), w bounds
__device__ __forceinline__ void load_solve(const Dev &d, int k, BrFun<false> &F, double *wlo, double *whi) {
    const size_t LTs = (size_t)d.L * d.T;
    const int l = k / d.T, t = k - l * d.T;
    const int bi = d.bfrom[l], bj = d.bto[l];
    F.Gii = d.y[0 * d.L + l]; F.Gij = d.y[1 * d.L + l]; F.Gji = d.y[2 * d.L + l]; F.Gjj = d.y[3 * d.L + l];
    F.Bii = d.y[4 * d.L + l]; F.Bij = d.y[5 * d.L + l]; F.Bji = d.y[6 * d.L + l]; F.Bjj = d.y[7 * d.L + l];
    F.rpq = d.rpq;
    F.rva = d.rva;
#pragma unroll
    for (int r = 0; r < 4; r++) F.tau[r] = d.fbar[r * LTs + k] - d.zb[r * LTs + k] - d.yb[r * LTs + k] / d.rpq;
    const size_t wi = (size_t)bi * d.T + t, wj = (size_t)bj * d.T + t;
    F.tau[4] = d.wbar[wi] - d.zb[B_WI * LTs + k] - d.yb[B_WI * LTs + k] / d.rva;
    F.tau[5] = d.wbar[wj] - d.zb[B_WJ * LTs + k] - d.yb[B_WJ * LTs + k] / d.rva;
    F.tau[6] = d.thbar[wi] - d.zb[B_AI * LTs + k] - d.yb[B_AI * LTs + k] / d.rva;
    F.tau[7] = d.thbar[wj] - d.zb[B_AJ * LTs + k] - d.yb[B_AJ * LTs + k] / d.rva;
    F.setup();
    wlo[0] = d.vmin[bi] * d.vmin[bi];
    whi[0] = d.vmax[bi] * d.vmax[bi];
    wlo[1] = d.vmin[bj] * d.vmin[bj];
    whi[1] = d.vmax[bj] * d.vmax[bj];
}

// Phase 1: 4-variable fast path for every (l,t).  Solves whose result violates Eq. 2c-2d are
// appended to the AL queue and finished by k_branch_al (R9); the rest are final here.
// Bus-side targets of the 8 rows of solve k for step (7d): tauhat = x-part + z + y/rho
// (DESIGN.md 5.5), written right after the solve so the bus kernel reads 4 values per incident
// end instead of the row state.  (x + z) + y/rho has no multiply-add to contract, so this is
// the same value the oracle forms.
__device__ __forceinline__ void emit_tauhat(const Dev &d, int k, const double *x, double f0, double f1,
                                            double f2, double f3) {
    const size_t LTs = (size_t)d.L * d.T;                // row-state kind stride
    const size_t LTH = (size_t)(d.L + d.Lph) * d.T;      // tauhat kind stride includes phantom branches
    const double xs[8] = {f0, f1, f2, f3, x[0], x[1], x[2], x[3]};
#pragma unroll
    for (int r = 0; r < 8; r++) {
        const double rho = r < 4 ? d.rpq : d.rva;
        d.tauh[r * LTH + k] = xs[r] + d.zb[r * LTs + k] + d.yb[r * LTs + k] / rho;
    }
}

#ifndef UCAC_BRANCH_TPB
#define UCAC_BRANCH_TPB 128
#endif
#ifndef UCAC_BRANCH_MINB
#define UCAC_BRANCH_MINB 3
#endif
#ifndef UCAC_AL_DEAL
#define UCAC_AL_DEAL 0
#endif
#ifndef UCAC_AL_FLAT
#define UCAC_AL_FLAT 0
#endif
#ifndef UCAC_AL_BLOCKS_PER_SM
#define UCAC_AL_BLOCKS_PER_SM 4
#endif
__global__ void __launch_bounds__(UCAC_BRANCH_TPB, UCAC_BRANCH_MINB) k_branch(Dev d) {
    if (d.st->done) return;
    const int LT = d.L * d.T;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long c_it = 0, c_cap = 0;
    if (k < LT) {
        const size_t LTs = (size_t)LT;
        BrFun<false> F4;
        double lo[4], hi[4];
        load_solve(d, k, F4, lo, hi);
        lo[2] = -TWO_PI; hi[2] = TWO_PI; lo[3] = -TWO_PI; hi[3] = TWO_PI;
        double x[4];
#pragma unroll
        for (int m = 0; m < 4; m++) x[m] = d.x[m * LTs + k];
        int it = 0;
        bool ok = tron<4>(F4, x, lo, hi, d.tron_gtol, d.tron_maxit, it);
        c_it = it;
        c_cap = !ok;
        double C, S, f0, f1, f2, f3;
        F4.flows(x, C, S, f0, f1, f2, f3);
        const double rate = d.rate[k / d.T];
        const double r2 = rate * rate;
#pragma unroll
        for (int m = 0; m < 4; m++) d.x[m * LTs + k] = x[m];
        d.f[0 * LTs + k] = f0;
        d.f[1 * LTs + k] = f1;
        d.f[2 * LTs + k] = f2;
        d.f[3 * LTs + k] = f3;
        if (rate > 0.0 && (f0 * f0 + f1 * f1 > r2 || f2 * f2 + f3 * f3 > r2)) {
            const unsigned pos = atomicAdd(d.alq_cnt, 1u);
            d.alq[pos] = k;
        } else {
            d.al[0 * LTs + k] = 0.0;
            d.al[1 * LTs + k] = 0.0;
            d.al[2 * LTs + k] = d.al_sigma0_rel * d.rpq * r2;
            emit_tauhat(d, k, x, f0, f1, f2, f3);
        }
    }
    warp_add_u64(d.cnt + 0, c_it);
    warp_add_u64(d.cnt + 1, c_cap);
}

// Phase 2: the queued thermal-active solves (6-variable slack AL, R36).
//
// The warp executes the union of its lanes' control flow, so a nested "AL round { TRON }" loop
// costs sum over rounds of the max over lanes.  The loop is therefore FLATTENED: every pass does
// one TRON iteration of whatever round each lane is in, and a lane whose round ends updates
// (mu, sigma) -- or finishes its solve and takes the next queued item -- in the same pass.  The
// per-solve arithmetic is exactly the nested algorithm's (oracle orc_branch_solve).
//
// Items are dealt lane-major over all warps of the grid (item = lane * nwarps + warp, then
// strided by 32 * nwarps), so with a short queue each warp carries only a few solves and the
// max over its lanes stays close to the single longest solve.
struct AlItem {
    BrFun<true> F;
    double lo[6], hi[6], x[6];
    double r2, sig0, smax, hprev;
    int k, kk;
};

__device__ __forceinline__ void al_begin(const Dev &d, int k, AlItem &A) {
    const size_t LTs = (size_t)d.L * d.T;
    {
        BrFun<false> F4;
        load_solve(d, k, F4, A.lo, A.hi);
        A.F.Gii = F4.Gii; A.F.Gij = F4.Gij; A.F.Gji = F4.Gji; A.F.Gjj = F4.Gjj;
        A.F.Bii = F4.Bii; A.F.Bij = F4.Bij; A.F.Bji = F4.Bji; A.F.Bjj = F4.Bjj;
#pragma unroll
        for (int r = 0; r < 8; r++) A.F.tau[r] = F4.tau[r];
        A.F.rpq = F4.rpq; A.F.rva = F4.rva;
        A.F.K00 = F4.K00; A.F.K02 = F4.K02; A.F.K03 = F4.K03; A.F.K11 = F4.K11;
        A.F.K12 = F4.K12; A.F.K13 = F4.K13; A.F.K22 = F4.K22;
    }
    A.lo[2] = -TWO_PI; A.hi[2] = TWO_PI; A.lo[3] = -TWO_PI; A.hi[3] = TWO_PI;
    A.lo[4] = 0.0; A.hi[4] = 1.0; A.lo[5] = 0.0; A.hi[5] = 1.0;
    const double rate = d.rate[k / d.T];
    A.r2 = rate * rate;
    A.sig0 = d.al_sigma0_rel * d.rpq * A.r2;
    A.F.r2inv = 1.0 / A.r2;
#pragma unroll
    for (int m = 0; m < 4; m++) A.x[m] = d.x[m * LTs + k];
    {
        const double f0 = d.f[0 * LTs + k], f1 = d.f[1 * LTs + k], f2 = d.f[2 * LTs + k], f3 = d.f[3 * LTs + k];
        A.x[4] = clampd(1.0 - (f0 * f0 + f1 * f1) / A.r2, 0.0, 1.0);
        A.x[5] = clampd(1.0 - (f2 * f2 + f3 * f3) / A.r2, 0.0, 1.0);
    }
    A.F.mu0 = d.al[0 * LTs + k];
    A.F.mu1 = d.al[1 * LTs + k];
    A.F.sig = fmax(A.sig0, d.al[2 * LTs + k] * d.al_sigma_decay);
    A.smax = d.al_sigma_max_rel * A.sig0;
    A.hprev = INFINITY;
    A.k = k;
    A.kk = 0;
}

__device__ __forceinline__ void al_finish(const Dev &d, const AlItem &A) {
    const size_t LTs = (size_t)d.L * d.T;
    const int k = A.k;
    double C, S, f0, f1, f2, f3;
    A.F.flows(A.x, C, S, f0, f1, f2, f3);
#pragma unroll
    for (int m = 0; m < 4; m++) d.x[m * LTs + k] = A.x[m];
    d.f[0 * LTs + k] = f0;
    d.f[1 * LTs + k] = f1;
    d.f[2 * LTs + k] = f2;
    d.f[3 * LTs + k] = f3;
    d.al[0 * LTs + k] = A.F.mu0;
    d.al[1 * LTs + k] = A.F.mu1;
    d.al[2 * LTs + k] = A.F.sig;
    emit_tauhat(d, k, A.x, f0, f1, f2, f3);
}

__global__ void __launch_bounds__(64) k_branch_al(Dev d) {
    if (d.st->done) return;
    const unsigned n = *((volatile unsigned *)d.alq_cnt);
    const unsigned nwarps = (gridDim.x * blockDim.x) >> 5;
    const unsigned lane = threadIdx.x & 31, gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
#if UCAC_AL_DEAL
    unsigned next = lane * nwarps + gwarp;   // lane-major: few solves per warp
#else
    unsigned next = gwarp * 32 + lane;       // dense: full warps
#endif
    unsigned long long c_it = 0, c_cap = 0, c_al = 0, c_alcap = 0;
    AlItem A;
#if !UCAC_AL_FLAT
    // nested form: AL rounds around whole TRON solves
    for (; next < n; next += 32 * nwarps) {
#ifdef UCAC_PROF
        const long long t0 = clock64();
        unsigned long long it0 = c_it, cap0 = c_cap;
#endif
        al_begin(d, d.alq[next], A);
        c_al += 1;
        for (;;) {
            int it = 0;
            const bool ok = tron<6>(A.F, A.x, A.lo, A.hi, d.tron_gtol, d.tron_maxit, it);
            c_it += it;
            c_cap += !ok;
            double C, Sn, f0, f1, f2, f3;
            A.F.flows(A.x, C, Sn, f0, f1, f2, f3);
            const double h1 = (f0 * f0 + f1 * f1) / A.r2 - 1.0 + A.x[4];
            const double h2 = (f2 * f2 + f3 * f3) / A.r2 - 1.0 + A.x[5];
            const double hm = fmax(fabs(h1), fabs(h2));
            if (hm <= d.al_eta_star) break;
            A.F.mu0 += A.F.sig * h1;
            A.F.mu1 += A.F.sig * h2;
            if (hm > 0.25 * A.hprev) A.F.sig = fmin(10.0 * A.F.sig, A.smax);
            A.hprev = hm;
            if (++A.kk >= d.al_maxit) {
                c_alcap += 1;
                break;
            }
        }
        al_finish(d, A);
#ifdef UCAC_PROF
        // diagnostic build only: report solves slower than UCAC_PROF cycles
        const long long dt = clock64() - t0;
        if (dt > UCAC_PROF)
            printf("ALPROF k %d l %d t %d cycles %lld tron_iters %llu rounds %d tron_caps %llu warp %u lane %u\n",
                   A.k, A.k / d.T, A.k % d.T, dt, c_it - it0, A.kk + 1, c_cap - cap0, gwarp, lane);
#endif
    }
#else
    Tron<6> S;
    bool busy = false;
    for (;;) {
        if (!busy) {
            if (next >= n) break;
            al_begin(d, d.alq[next], A);
            next += 32 * nwarps;
            c_al += 1;
            S.begin(A.F, A.x, A.lo, A.hi);
            busy = true;
        }
        // one TRON pass of the current round
        bool round_done = false, ok = true;
        if (S.converged(A.x, A.lo, A.hi, d.tron_gtol)) {
            round_done = true;
        } else if (S.it >= d.tron_maxit) {
            round_done = true;
            ok = false;
        } else {
            round_done = S.iterate(A.F, A.x, A.lo, A.hi);
        }
        if (!round_done) continue;
        // round end: the method-of-multipliers update (R9)
        c_it += S.it;
        c_cap += !ok;
        double C, Sn, f0, f1, f2, f3;
        A.F.flows(A.x, C, Sn, f0, f1, f2, f3);
        const double h1 = (f0 * f0 + f1 * f1) / A.r2 - 1.0 + A.x[4];
        const double h2 = (f2 * f2 + f3 * f3) / A.r2 - 1.0 + A.x[5];
        const double hm = fmax(fabs(h1), fabs(h2));
        bool fin = hm <= d.al_eta_star;
        if (!fin) {
            A.F.mu0 += A.F.sig * h1;
            A.F.mu1 += A.F.sig * h2;
            if (hm > 0.25 * A.hprev) A.F.sig = fmin(10.0 * A.F.sig, A.smax);
            A.hprev = hm;
            if (++A.kk >= d.al_maxit) {
                fin = true;
                c_alcap += 1;
            }
        }
        if (fin) {
            al_finish(d, A);
            busy = false;
        } else {
            S.begin(A.F, A.x, A.lo, A.hi);
        }
    }
#endif
    if (c_it) atomicAdd(d.cnt + 0, c_it);
    if (c_cap) atomicAdd(d.cnt + 1, c_cap);
    if (c_al) atomicAdd(d.cnt + 2, c_al);
    if (c_alcap) atomicAdd(d.cnt + 3, c_alcap);
}

}  // namespace

void launch_branch(const Dev &d, cudaStream_t s) {
    const int n = d.L * d.T;
    k_branch<<<(n + UCAC_BRANCH_TPB - 1) / UCAC_BRANCH_TPB, UCAC_BRANCH_TPB, 0, s>>>(d);
}
void launch_branch_al(const Dev &d, cudaStream_t s) { k_branch_al<<<148 * UCAC_AL_BLOCKS_PER_SM, 64, 0, s>>>(d); }

}  // namespace ucac
