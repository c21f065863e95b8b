// k_strict.cu -- step (7b) line part in the strict_fp parity mode (ucac_params.strict_fp = 1,
// SURVEY.md 8(b), 8(c).4 A31).  Compiled with -fmad=false.
//
// One thread per (branch, period) runs the branch solve of DESIGN.md 5.3 exactly as the plain
// CPU oracle states it -- the same algorithm, the same operation order, IEEE divisions and
// square roots, no FMA contraction and the explicit sin/cos polynomial of R54 -- so that with
// the oracle's arithmetic and this kernel's in agreement the whole iterate is reproduced bit
// for bit (the generator, ubar and DP kernels already are; the bus and row kernels have strict
// instantiations with the oracle's quotients, k_sweep.cu).  It is the same method as k_branch
// + k_branch_al (fast path, then the six-variable slack AL with the second-order multiplier
// step, the predictor, the two-point start and the small first radius, R41-R49), written a
// second time: the code is not shared with oracle/ (the oracle is test infrastructure), it
// restates the same definitions, as k_gen.cu does for the DP (category (b)).
//
// This mode exists for parity (the north star's 1e-9 per-iteration contract over 50 free-running
// iterations); it is not the throughput path: it keeps the oracle's dense 4x4x4 flow-Hessian
// tables and Steihaug CG in local memory.  The default path is k_branch.cu.
#include <algorithm>

#include "ucac_dev.cuh"

namespace ucac {
namespace {

constexpr double S_MU0 = 0.01, S_ETA0 = 1e-4, S_ETA1 = 0.25, S_ETA2 = 0.75;
constexpr double S_SIG1 = 0.25, S_SIG3 = 4.0, S_DELTA0 = 1.0, S_CGTOL = 1e-12;
constexpr double S_EPSF = 1e-10, S_STALL = 1e-13;   // R48
constexpr double S_AL_NEWTON_C = 10.0, S_AL_R1_DELTA0 = 0.03;
constexpr double S_TWO_PI = 6.283185307179586;
constexpr int SN = 6;   // the largest subproblem (six-variable AL)

__device__ __forceinline__ double smax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double smin(double a, double b) { return a < b ? a : b; }
__device__ __forceinline__ double sclamp(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

// sin, cos by R54's polynomial: Cody-Waite reduction by pi/2 (33-bit head + tail) and the
// Taylor series of sin to r^17, of cos to r^18 on |r| <= pi/4
__device__ void s_sincos(double a, double *s, double *c) {
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
    switch (((long long)k) & 3) {
        case 0: *s = sr; *c = cr; break;
        case 1: *s = cr; *c = -sr; break;
        case 2: *s = -sr; *c = -cr; break;
        default: *s = -cr; *c = sr; break;
    }
}

// flows of branch (i->j), Eq. 2e-2h with R1's to-side labels, through C = sqrt(w_i w_j)
// cos(th_i - th_j), S = ... sin(...); J[k*4+m] = df_k/dx_m, H[k*16+m*4+n] = d2f_k/dx_m dx_n
__device__ void s_flows(const double *y, const double *x, double *f, double *J, double *H) {
    const double Gii = y[0], Gij = y[1], Gji = y[2], Gjj = y[3];
    const double Bii = y[4], Bij = y[5], Bji = y[6], Bjj = y[7];
    const double wi = x[0], wj = x[1], d = x[2] - x[3];
    const double R = sqrt(wi * wj);
    double sn, cs;
    s_sincos(d, &sn, &cs);
    const double C = R * cs, S = R * sn;
    const double dC[4] = {C / (2.0 * wi), C / (2.0 * wj), -S, S};
    const double dS[4] = {S / (2.0 * wi), S / (2.0 * wj), C, -C};
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
    const double ca[4] = {Gii, -Bii, 0.0, 0.0};
    const double cb[4] = {0.0, 0.0, Gjj, -Bjj};
    const double cc[4] = {Gij, -Bij, Gji, -Bji};
    const double cd[4] = {Bij, Gij, -Bji, -Gji};
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
                for (int n = 0; n < 4; n++) H[k * 16 + m * 4 + n] = cc[k] * HC[m][n] + cd[k] * HS[m][n];
        }
    }
}

__device__ __forceinline__ double s_dot(int n, const double *a, const double *b) {
    double s = 0.0;
    for (int i = 0; i < n; i++) s = s + a[i] * b[i];
    return s;
}
__device__ __forceinline__ double s_nrm2(int n, const double *a) { return sqrt(s_dot(n, a, a)); }
__device__ __forceinline__ void s_matvec(int n, const double *H, const double *v, double *o) {
    for (int i = 0; i < n; i++) {
        double s = 0.0;
        for (int j = 0; j < n; j++) s = s + H[i * n + j] * v[j];
        o[i] = s;
    }
}
__device__ __forceinline__ double s_qmodel(int n, const double *g, const double *H, const double *s) {
    double Hs[SN];
    s_matvec(n, H, s, Hs);
    return s_dot(n, g, s) + 0.5 * s_dot(n, s, Hs);
}

// the branch objective F (+ the thermal AL terms when al != 0) with its gradient and Hessian
struct SCtx {
    const double *y, *tau;
    double rpq, rva, r2, mu[2], sig;
    int al, nva;
};
__device__ void s_eval(const SCtx *c, const double *X, double *fo, double *g, double *H) {
    const int n = c->al ? 6 : 4;
    double f[4], J[16], Hf[64];
    s_flows(c->y, X, f, J, Hf);
    double F = 0.0;
    for (int i = 0; i < n; i++) g[i] = 0.0;
    for (int i = 0; i < n * n; i++) H[i] = 0.0;
    for (int k = 0; k < 4; k++) {
        const double e = f[k] - c->tau[k];
        F = F + 0.5 * c->rpq * e * e;
        for (int a = 0; a < 4; a++) {
            g[a] = g[a] + c->rpq * e * J[k * 4 + a];
            for (int b = 0; b < 4; b++)
                H[a * n + b] = H[a * n + b] + c->rpq * (J[k * 4 + a] * J[k * 4 + b] + e * Hf[k * 16 + a * 4 + b]);
        }
    }
    for (int m = 0; m < c->nva; m++) {
        const double e = X[m] - c->tau[4 + m];
        F = F + 0.5 * c->rva * e * e;
        g[m] = g[m] + c->rva * e;
        H[m * n + m] = H[m * n + m] + c->rva;
    }
    if (c->al) {
        for (int m = 0; m < 2; m++) {
            const int kp = 2 * m, kq = 2 * m + 1;
            const double P = f[kp], Q = f[kq];
            const double h = (P * P + Q * Q) / c->r2 - 1.0 + X[4 + m];
            double gh[6] = {0, 0, 0, 0, 0, 0};
            for (int a = 0; a < 4; a++) gh[a] = 2.0 * (P * J[kp * 4 + a] + Q * J[kq * 4 + a]) / c->r2;
            gh[4 + m] = 1.0;
            const double lam = c->mu[m] + c->sig * h;
            F = F + c->mu[m] * h + 0.5 * c->sig * h * h;
            for (int a = 0; a < 6; a++) g[a] = g[a] + lam * gh[a];
            for (int a = 0; a < 6; a++) {
                for (int b = 0; b < 6; b++) {
                    double hh = 0.0;
                    if (a < 4 && b < 4)
                        hh = 2.0 * (J[kp * 4 + a] * J[kp * 4 + b] + P * Hf[kp * 16 + a * 4 + b] + J[kq * 4 + a] * J[kq * 4 + b] +
                                    Q * Hf[kq * 16 + a * 4 + b]) / c->r2;
                    H[a * 6 + b] = H[a * 6 + b] + lam * hh + c->sig * gh[a] * gh[b];
                }
            }
        }
    }
    *fo = F;
}

__device__ void s_pstep(int n, const double *x, const double *lo, const double *hi, const double *d, double a, double *s) {
    for (int i = 0; i < n; i++) s[i] = sclamp(x[i] + a * d[i], lo[i], hi[i]) - x[i];
}
__device__ bool s_cauchy_ok(int n, const double *g, const double *H, const double *s, double delta) {
    return s_nrm2(n, s) <= delta && s_qmodel(n, g, H, s) <= S_MU0 * s_dot(n, g, s);
}
__device__ void s_cauchy(int n, const double *x, const double *lo, const double *hi, const double *g, const double *H,
                         double delta, double *alpha, double *s) {
    double mg[SN], sp[SN];
    for (int i = 0; i < n; i++) mg[i] = -g[i];
    double a = *alpha;
    s_pstep(n, x, lo, hi, mg, a, s);
    if (!s_cauchy_ok(n, g, H, s, delta)) {
        for (int k = 0; k < 60; k++) {
            a = a * 0.1;
            s_pstep(n, x, lo, hi, mg, a, s);
            if (s_cauchy_ok(n, g, H, s, delta)) break;
        }
    } else {
        for (int k = 0; k < 20; k++) {
            const double ap = a;
            for (int i = 0; i < n; i++) sp[i] = s[i];
            a = a * 10.0;
            s_pstep(n, x, lo, hi, mg, a, s);
            bool same = true;
            for (int i = 0; i < n; i++)
                if (s[i] != sp[i]) same = false;
            if (!s_cauchy_ok(n, g, H, s, delta) || same) {
                a = ap;
                for (int i = 0; i < n; i++) s[i] = sp[i];
                break;
            }
        }
    }
    *alpha = a;
}
__device__ double s_bnd_tau(int n, const double *a, const double *p, double delta) {
    const double aa = s_dot(n, a, a), ap = s_dot(n, a, p), pp = s_dot(n, p, p);
    if (pp <= 0.0) return 0.0;
    double gap = delta * delta - aa;
    if (gap < 0.0) gap = 0.0;
    const double rad = sqrt(ap * ap + pp * gap);
    if (ap > 0.0) return gap / (ap + rad);
    return (rad - ap) / pp;
}
__device__ void s_steihaug(int n, const double *H, const double *gq, const int *fr, const double *sc, double delta,
                           double *w) {
    double r[SN], p[SN], Hp[SN], t[SN];
    for (int i = 0; i < n; i++) {
        w[i] = 0.0;
        r[i] = fr[i] ? -gq[i] : 0.0;
        p[i] = r[i];
    }
    double rr = s_dot(n, r, r);
    if (rr == 0.0) return;
    const double tol2 = S_CGTOL * S_CGTOL * rr;
    for (int k = 0; k < n; k++) {
        s_matvec(n, H, p, Hp);
        for (int i = 0; i < n; i++)
            if (!fr[i]) Hp[i] = 0.0;
        const double kap = s_dot(n, p, Hp);
        for (int i = 0; i < n; i++) t[i] = sc[i] + w[i];
        if (kap <= 0.0) {
            const double tau = s_bnd_tau(n, t, p, delta);
            for (int i = 0; i < n; i++) w[i] = w[i] + tau * p[i];
            return;
        }
        const double a = rr / kap;
        for (int i = 0; i < n; i++) t[i] = sc[i] + w[i] + a * p[i];
        if (s_nrm2(n, t) >= delta) {
            for (int i = 0; i < n; i++) t[i] = sc[i] + w[i];
            const double tau = s_bnd_tau(n, t, p, delta);
            for (int i = 0; i < n; i++) w[i] = w[i] + tau * p[i];
            return;
        }
        for (int i = 0; i < n; i++) {
            w[i] = w[i] + a * p[i];
            r[i] = r[i] - a * Hp[i];
        }
        const double rn = s_dot(n, r, r);
        if (rn <= tol2) return;
        const double b = rn / rr;
        for (int i = 0; i < n; i++) p[i] = r[i] + b * p[i];
        rr = rn;
    }
}
__device__ void s_prsrch(int n, const double *x, const double *lo, const double *hi, const double *g, const double *H,
                         const double *sc, const double *w, double *s) {
    double gq[SN], Hs[SN], ds[SN];
    s_matvec(n, H, sc, Hs);
    for (int i = 0; i < n; i++) gq[i] = g[i] + Hs[i];
    const double qc = s_qmodel(n, g, H, sc);
    double b = 1.0;
    for (int k = 0; k < 20; k++) {
        for (int i = 0; i < n; i++) {
            s[i] = sclamp(x[i] + sc[i] + b * w[i], lo[i], hi[i]) - x[i];
            ds[i] = s[i] - sc[i];
        }
        if (s_qmodel(n, g, H, s) <= qc + S_MU0 * s_dot(n, gq, ds)) return;
        b = b * 0.5;
    }
    for (int i = 0; i < n; i++) s[i] = sc[i];
}
__device__ double s_pgnorm(int n, const double *x, const double *g, const double *lo, const double *hi) {
    double m = 0.0;
    for (int i = 0; i < n; i++) {
        const double v = fabs(sclamp(x[i] - g[i], lo[i], hi[i]) - x[i]);
        if (v > m) m = v;
    }
    return m;
}

// projected trust-region Newton with the R41 first Cauchy length and the R48 stall
__device__ bool s_tron(int n, double *x, const double *lo, const double *hi, const SCtx *ctx, double gtol, int maxit,
                       int *iters, double delta0) {
    double f, g[SN], H[SN * SN], fn, gn[SN], Hn[SN * SN];
    double sc[SN], w[SN], s[SN], xn[SN], gq[SN], Hs[SN];
    int fr[SN];
    for (int i = 0; i < n; i++) x[i] = sclamp(x[i], lo[i], hi[i]);
    s_eval(ctx, x, &f, g, H);
    double delta = delta0, alpha = 1.0;
    {
        double Hg[SN];
        s_matvec(n, H, g, Hg);
        const double gHg = s_dot(n, g, Hg), gg = s_dot(n, g, g);
        if (gHg > 0.0 && gg > 0.0) alpha = gg / gHg;
    }
    int it;
    for (it = 0; it < maxit; it++) {
        if (s_pgnorm(n, x, g, lo, hi) <= gtol) {
            *iters = it;
            return true;
        }
        s_cauchy(n, x, lo, hi, g, H, delta, &alpha, sc);
        for (int i = 0; i < n; i++) {
            const double xc = x[i] + sc[i];
            fr[i] = (xc > lo[i] && xc < hi[i]);
        }
        s_matvec(n, H, sc, Hs);
        for (int i = 0; i < n; i++) gq[i] = g[i] + Hs[i];
        s_steihaug(n, H, gq, fr, sc, delta, w);
        s_prsrch(n, x, lo, hi, g, H, sc, w, s);
        {
            double xm = 0.0;
            for (int i = 0; i < n; i++) xm = smax(xm, fabs(x[i]));
            if (s_nrm2(n, s) <= S_STALL * (1.0 + xm)) {
                *iters = it;
                return true;
            }
        }
        const double pred = -s_qmodel(n, g, H, s);
        for (int i = 0; i < n; i++) xn[i] = sclamp(x[i] + s[i], lo[i], hi[i]);
        s_eval(ctx, xn, &fn, gn, Hn);
        double ared = f - fn;
        if (fabs(pred) <= S_EPSF * fabs(f)) ared = -0.5 * (s_dot(n, g, s) + s_dot(n, gn, s));
        const double ratio = (pred > 0.0) ? ared / pred : -1.0;
        const double snorm = s_nrm2(n, s);
        if (ratio > S_ETA0) {
            for (int i = 0; i < n; i++) x[i] = xn[i];
            f = fn;
            for (int i = 0; i < n; i++) g[i] = gn[i];
            for (int i = 0; i < n * n; i++) H[i] = Hn[i];
        }
        if (ratio < S_ETA1) delta = S_SIG1 * smin(snorm, delta);
        else if (ratio > S_ETA2) delta = smax(delta, S_SIG3 * snorm);
    }
    *iters = it;
    return s_pgnorm(n, x, g, lo, hi) <= gtol;
}

// second-order multiplier step with the spectral safeguard and the primal predictor (R42, R43)
__device__ bool s_al_newton_dmu(const SCtx *c, const double *X, const double *lo, const double *hi, const double *h,
                                double *dmu, double *dx) {
    double F, g[6], H[36], f[4], Jf[16];
    s_eval(c, X, &F, g, H);
    s_flows(c->y, X, f, Jf, nullptr);
    double J[2][6];
    for (int m = 0; m < 2; m++) {
        const int kp = 2 * m, kq = 2 * m + 1;
        for (int a = 0; a < 4; a++) J[m][a] = 2.0 * (f[kp] * Jf[kp * 4 + a] + f[kq] * Jf[kq * 4 + a]) / c->r2;
        J[m][4] = m == 0 ? 1.0 : 0.0;
        J[m][5] = m == 1 ? 1.0 : 0.0;
    }
    int idx[6], nf = 0;
    for (int i = 0; i < 6; i++)
        if (X[i] > lo[i] && X[i] < hi[i]) idx[nf++] = i;
    double L[36];
    for (int j = 0; j < nf; j++) {
        double d = H[idx[j] * 6 + idx[j]];
        for (int k = 0; k < j; k++) d = d - L[j * 6 + k] * L[j * 6 + k];
        if (!(d > 0.0)) return false;
        L[j * 6 + j] = sqrt(d);
        for (int i = j + 1; i < nf; i++) {
            double v = H[idx[i] * 6 + idx[j]];
            for (int k = 0; k < j; k++) v = v - L[i * 6 + k] * L[j * 6 + k];
            L[i * 6 + j] = v / L[j * 6 + j];
        }
    }
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
    }
    double M[2][2];
    for (int m = 0; m < 2; m++)
        for (int n = 0; n < 2; n++) {
            double v = 0.0;
            for (int i = 0; i < nf; i++) v = v + J[m][idx[i]] * V[n][i];
            M[m][n] = v;
        }
    const double a = M[0][0], b = 0.5 * (M[0][1] + M[1][0]), d = M[1][1];
    const double mean = 0.5 * (a + d), half = 0.5 * (a - d);
    const double r = sqrt(half * half + b * b);
    const double lam[2] = {mean + r, mean - r};
    double v[2][2];
    if (r == 0.0) {
        v[0][0] = 1.0; v[0][1] = 0.0;
    } else if (a >= d) {
        const double nn = sqrt((lam[0] - d) * (lam[0] - d) + b * b);
        v[0][0] = (lam[0] - d) / nn; v[0][1] = b / nn;
    } else {
        const double nn = sqrt(b * b + (lam[0] - a) * (lam[0] - a));
        v[0][0] = b / nn; v[0][1] = (lam[0] - a) / nn;
    }
    v[1][0] = -v[0][1]; v[1][1] = v[0][0];
    dmu[0] = 0.0;
    dmu[1] = 0.0;
    for (int e = 0; e < 2; e++) {
        const double fac = lam[e] >= 1.0 / (S_AL_NEWTON_C * c->sig) ? 1.0 / lam[e] : c->sig;
        const double ph = v[e][0] * h[0] + v[e][1] * h[1];
        dmu[0] = dmu[0] + fac * ph * v[e][0];
        dmu[1] = dmu[1] + fac * ph * v[e][1];
    }
    for (int i = 0; i < 6; i++) dx[i] = 0.0;
    for (int i = 0; i < nf; i++) dx[idx[i]] = -(V[0][i] * dmu[0] + V[1][i] * dmu[1]);
    return true;
}

// counters: 0 TRON iterations, 1 capped, 2 AL active, 3 AL capped, 4 TRON iterations in the AL
__device__ void s_branch_solve(const double *y, const double *wlo, const double *whi, double rate, const double *tau,
                               const Dev &d, double *x, double *al, double *f, unsigned long long *cnt) {
    double lo[6] = {wlo[0], wlo[1], -S_TWO_PI, -S_TWO_PI, 0.0, 0.0};
    double hi[6] = {whi[0], whi[1], S_TWO_PI, S_TWO_PI, 1.0, 1.0};
    if (d.variant & 8) lo[2] = hi[2] = 0.0;   // R51
    const double gtol = d.tron_gtol;           // tron_gtol_rel * max(rho_pq, rho_va), formed once on the host
    SCtx c;
    c.y = y; c.tau = tau; c.rpq = d.rpq; c.rva = d.rva; c.al = 0;
    c.nva = (d.variant & 8) ? 2 : 4;
    c.r2 = rate * rate; c.mu[0] = c.mu[1] = 0.0; c.sig = 0.0;
    int it = 0;
    const bool al_always = (d.variant & 1) && rate > 0.0;   // R47
    bool ok = true;
    double xprev[4];
    for (int i = 0; i < 4; i++) xprev[i] = sclamp(x[i], lo[i], hi[i]);
    if (al_always)
        for (int i = 0; i < 4; i++) x[i] = sclamp(x[i], lo[i], hi[i]);
    else
        ok = s_tron(4, x, lo, hi, &c, gtol, d.tron_maxit, &it, S_DELTA0);
    cnt[0] += it;
    cnt[1] += !ok;
    const double sig0 = d.al_sigma0_rel * d.rpq * c.r2;
    s_flows(y, x, f, nullptr, nullptr);
    if (rate > 0.0) {
        const double s1 = f[0] * f[0] + f[1] * f[1], s2 = f[2] * f[2] + f[3] * f[3];
        if (al_always || s1 > c.r2 || s2 > c.r2) {
            double X[6] = {x[0], x[1], x[2], x[3], sclamp(1.0 - s1 / c.r2, 0.0, 1.0), sclamp(1.0 - s2 / c.r2, 0.0, 1.0)};
            c.al = 1;
            c.mu[0] = al[0]; c.mu[1] = al[1];
            c.sig = smax(sig0, al[2] * d.al_sigma_decay);
            const double sgmax = d.al_sigma_max_rel * sig0;
            double hprev = INFINITY;
            int k;
            cnt[2] += 1;
            {
                // R49: the lower-AL start of the fast-path point and the previous iterate
                double fp[4], Xp[6], Fa, Fb, gs[6], Hs[36];
                s_flows(y, xprev, fp, nullptr, nullptr);
                for (int i = 0; i < 4; i++) Xp[i] = xprev[i];
                Xp[4] = sclamp(1.0 - (fp[0] * fp[0] + fp[1] * fp[1]) / c.r2, 0.0, 1.0);
                Xp[5] = sclamp(1.0 - (fp[2] * fp[2] + fp[3] * fp[3]) / c.r2, 0.0, 1.0);
                s_eval(&c, X, &Fa, gs, Hs);
                s_eval(&c, Xp, &Fb, gs, Hs);
                if (Fb < Fa)
                    for (int i = 0; i < 6; i++) X[i] = Xp[i];
            }
            for (k = 0; k < d.al_maxit; k++) {
                ok = s_tron(6, X, lo, hi, &c, gtol, d.tron_maxit, &it, k == 0 ? S_AL_R1_DELTA0 : S_DELTA0);   // R44
                cnt[0] += it;
                cnt[4] += it;
                cnt[1] += !ok;
                s_flows(y, X, f, nullptr, nullptr);
                const double h1 = (f[0] * f[0] + f[1] * f[1]) / c.r2 - 1.0 + X[4];
                const double h2 = (f[2] * f[2] + f[3] * f[3]) / c.r2 - 1.0 + X[5];
                const double hm = smax(fabs(h1), fabs(h2));
                if (hm <= d.al_eta_star) break;
                const double hv[2] = {h1, h2};
                double dmu[2], dx[6];
                if (s_al_newton_dmu(&c, X, lo, hi, hv, dmu, dx)) {
                    for (int i = 0; i < 6; i++) X[i] = sclamp(X[i] + dx[i], lo[i], hi[i]);
                } else {
                    dmu[0] = c.sig * h1;
                    dmu[1] = c.sig * h2;
                }
                c.mu[0] = c.mu[0] + dmu[0];
                c.mu[1] = c.mu[1] + dmu[1];
                if (hm > 0.25 * hprev) c.sig = smin(10.0 * c.sig, sgmax);
                hprev = hm;
            }
            cnt[3] += k >= d.al_maxit;
            for (int i = 0; i < 4; i++) x[i] = X[i];
            al[0] = c.mu[0]; al[1] = c.mu[1]; al[2] = c.sig;
            return;
        }
    }
    al[0] = 0.0; al[1] = 0.0; al[2] = sig0;
}

__device__ __forceinline__ void s_warp_add(unsigned long long *dst, unsigned long long v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

constexpr int STRICT_TPB = 128;
__global__ void __launch_bounds__(STRICT_TPB) k_branch_strict(Dev d) {
    pdl_wait();
    TL_KERNEL(K_BRANCH);
    if (d.st->done) return;
    const int LT = d.L * d.T;
    const size_t LTs = (size_t)LT, LTH = (size_t)(d.L + d.Lph) * d.T;
    unsigned long long cnt[NCNT] = {0, 0, 0, 0, 0};
    for (int base = blockIdx.x * blockDim.x; base < LT; base += gridDim.x * blockDim.x) {
        const int k = base + threadIdx.x;
        if (k < LT && own_t(d, k % d.T)) {   // (time cut: owned periods only)
            const int l = k / d.T, t = k - l * d.T;
            const int bi = d.bfrom[l], bj = d.bto[l];
            double y[8];
            for (int r = 0; r < 8; r++) y[r] = d.y[r * d.L + l];
            const size_t wi = (size_t)bi * d.T + t, wj = (size_t)bj * d.T + t;
            // targets tau = xbar - z - y/rho, the oracle's quotient
            const double xb[8] = {d.fbar[0 * LTs + k], d.fbar[1 * LTs + k], d.fbar[2 * LTs + k], d.fbar[3 * LTs + k],
                                  d.wbar[wi], d.wbar[wj], d.thbar[wi], d.thbar[wj]};
            double tau[8], zz[8], yy[8];
            for (int r = 0; r < 8; r++) {
                zz[r] = d.zb[r * LTs + k];
                yy[r] = d.yb[r * LTs + k];
                tau[r] = xb[r] - zz[r] - yy[r] / (r < 4 ? d.rpq : d.rva);
            }
            const double wlo[2] = {d.vmin[bi] * d.vmin[bi], d.vmin[bj] * d.vmin[bj]};
            const double whi[2] = {d.vmax[bi] * d.vmax[bi], d.vmax[bj] * d.vmax[bj]};
            double x[4], al[3], f[4];
            for (int m = 0; m < 4; m++) x[m] = d.x[m * LTs + k];
            for (int m = 0; m < 3; m++) al[m] = d.al[m * LTs + k];
            s_branch_solve(y, wlo, whi, d.rate[l], tau, d, x, al, f, cnt);
            for (int m = 0; m < 4; m++) d.x[m * LTs + k] = x[m];
            for (int m = 0; m < 4; m++) d.f[m * LTs + k] = f[m];
            for (int m = 0; m < 3; m++) d.al[m * LTs + k] = al[m];
            // bus-side targets tauhat = x-part + z + y/rho of the 8 rows, for (7d)
            const double xs[8] = {f[0], f[1], f[2], f[3], x[0], x[1], x[2], x[3]};
            double chk = 0.0;
            for (int r = 0; r < 8; r++) {
                const double th = xs[r] + zz[r] + yy[r] / (r < 4 ? d.rpq : d.rva);
                d.tauh[r * LTH + k] = th;
                chk = chk + nf0(tau[r]) + nf0(th);
            }
            if (chk != 0.0) report_nonfinite(d, K_BRANCH, l, t);   // NaN/inf anywhere in tau or tauhat
        }
    }
    s_warp_add(d.cnt + 0, cnt[0]);
    s_warp_add(d.cnt + 1, cnt[1]);
    s_warp_add(d.cnt + 2, cnt[2]);
    s_warp_add(d.cnt + 3, cnt[3]);
    s_warp_add(d.cnt + 4, cnt[4]);
}

}  // namespace

void launch_branch_strict(const Dev &d, cudaStream_t s) {
    const int n = d.L * d.T;
    const int grid = std::max(1, std::min((n + STRICT_TPB - 1) / STRICT_TPB, 148 * 4));
    k_branch_strict<<<grid, STRICT_TPB, 0, s>>>(d);
}

}  // namespace ucac
