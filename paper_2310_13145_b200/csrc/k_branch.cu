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

// Subspace step of TRON for N <= UCAC_TRON_DIRECT_MAXN variables: LDL^T Newton step when H_FF is
// positive definite and the step is interior, else Steihaug-Toint CG.
#ifndef UCAC_TRON_DIRECT_MAXN
#define UCAC_TRON_DIRECT_MAXN 6
#endif

namespace ucac {
#ifdef UCAC_PROF
// diagnostic builds only: per queued AL solve (k, start ns, end ns, Newton its, rounds, warp<<8|lane)
__device__ unsigned long long g_prof[6 << 16];
#endif
namespace {

constexpr double TR_MU0 = 0.01, TR_ETA0 = 1e-4, TR_ETA1 = 0.25, TR_ETA2 = 0.75;
constexpr double TR_SIG1 = 0.25, TR_SIG3 = 4.0, TR_DELTA0 = 1.0, TR_CGTOL = 1e-12;
constexpr double TR_EPSF = 1e-10, TR_STALL = 1e-13;   // R48
constexpr double TWO_PI = 6.283185307179586;

// 1/x for normal x: the MUFU reciprocal approximation refined by two Newton steps (relative error
// 2^-22 -> 2^-44 -> rounding), i.e. within an ulp of the IEEE quotient the oracle forms, without
// the division's slow-path call (and the register spills around it).  Callers guarantee a normal
// x; a subnormal x flushes to zero (result inf), where the quotient would be large but finite.
__device__ __forceinline__ double rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

// sin and cos of the angle difference: CUDA's sincos, or (UCAC_POLY_SINCOS) R54's Cody-Waite +
// Taylor polynomial (the oracle's operation sequence, here with FMA contraction: within 2 ulp, no
// slow-path range reduction -- the angle differences stay in [-4 pi, 4 pi])
#ifndef UCAC_POLY_SINCOS
#define UCAC_POLY_SINCOS 0
#endif
__device__ __forceinline__ void br_sincos(double a, double *s, double *c) {
    if (!UCAC_POLY_SINCOS) {
        sincos(a, s, c);
        return;
    }
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
    const int q = ((int)(long long)k) & 3;
    const double sa = (q & 1) ? cr : sr, ca = (q & 1) ? sr : cr;
    *s = (q & 2) ? -sa : sa;
    *c = ((q + 1) & 2) ? -ca : ca;
}

// NOANG: no angle consensus rows (variant bit 8, R51) -- a separate instantiation, so the default
// kernels carry none of its code
template <bool AL, bool NOANG = false>
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
        br_sincos(x[2] - x[3], &sn, &cs);
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
        for (int m = 0; m < (NOANG ? 2 : 4); m++) {
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
        for (int m = 0; m < (NOANG ? 2 : 4); m++) {
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
        const double ixx = 0.5 * rcp(x[0] * x[1]);   // one reciprocal for both 1/(2 w)
        double i2wi = x[1] * ixx, i2wj = x[0] * ixx;
        double dC[4] = {C * i2wi, C * i2wj, -S, S};
        double dS[4] = {S * i2wi, S * i2wj, C, -C};
#pragma unroll
        for (int m = 0; m < 4; m++) g[m] = GC * dC[m] + GS * dS[m] + ((NOANG && m >= 2) ? 0.0 : rva * (x[m] - tau[4 + m]));
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
        for (int m = 0; m < (NOANG ? 2 : 4); m++) H[m][m] += rva;
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

template <int N>
__device__ __forceinline__ double dotn(const double *a, const double *b) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N; i++) s += a[i] * b[i];
    return s;
}
template <int N>
__device__ __forceinline__ void matvec(const double (*H)[N], const double *v, double *o) {
#pragma unroll
    for (int i = 0; i < N; i++) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < N; j++) s += H[i][j] * v[j];
        o[i] = s;
    }
}
template <int N>
__device__ __forceinline__ double qmodel(const double *g, const double (*H)[N], const double *s) {
    double Hs[N];
    matvec<N>(H, s, Hs);
    return dotn<N>(g, s) + 0.5 * dotn<N>(s, Hs);
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
__device__ __forceinline__ bool cauchy_ok(const double *g, const double (*H)[N], const double *s, double delta) {
    return dotn<N>(s, s) <= delta * delta && qmodel<N>(g, H, s) <= TR_MU0 * dotn<N>(g, s);
}
template <int N>
__device__ __forceinline__ double bnd_tau(const double *a, const double *p, double delta) {
    double aa = dotn<N>(a, a), ap = dotn<N>(a, p), pp = dotn<N>(p, p);
    if (pp <= 0.0) return 0.0;
    double gap = fmax(delta * delta - aa, 0.0);
    double rad = sqrt(ap * ap + pp * gap);
    return ap > 0.0 ? gap * rcp(ap + rad) : (rad - ap) * rcp(pp);
}

template <int N>
__device__ __forceinline__ void copy_h(const double (*H)[N], double (*o)[N]) {
#pragma unroll
    for (int i = 0; i < N; i++)
#pragma unroll
        for (int j = 0; j < N; j++) o[i][j] = H[i][j];
}

// Second-order multiplier update of the thermal AL (R42) with the primal predictor (R43):
// dmu = M^{-1} h in the well-conditioned
// eigen-directions of M = J_F H_FF^{-1} J_F' and sigma h in the others.  H is the AL Hessian at
// the round's end point x (6 variables); its slack columns are sigma * dh/dx, so
// J_m = (H[0..3][4+m] / sigma, e_{4+m}).  F = variables strictly inside their bounds; H_FF is
// factored as L D L' with the fixed rows and columns replaced by the identity.  Returns false
// (keep the first-order step) if H_FF is not positive definite.
constexpr double AL_NEWTON_C = 10.0;
constexpr double AL_R1_DELTA0 = 0.03;
__device__ __forceinline__ bool al_newton_dmu(const double (*H)[6], const double *x, const double *lo,
                                              const double *hi, double sig, const double *h, double *dmu,
                                              double *dx) {
    bool fr[6];
#pragma unroll
    for (int i = 0; i < 6; i++) fr[i] = x[i] > lo[i] && x[i] < hi[i];
    double J[2][6];
    const double isig = rcp(sig);
#pragma unroll
    for (int m = 0; m < 2; m++) {
#pragma unroll
        for (int a = 0; a < 4; a++) J[m][a] = fr[a] ? H[a][4 + m] * isig : 0.0;
        J[m][4] = (m == 0 && fr[4]) ? 1.0 : 0.0;
        J[m][5] = (m == 1 && fr[5]) ? 1.0 : 0.0;
    }
    double Lm[6][6], D[6];
    bool pd = true;
#pragma unroll
    for (int j = 0; j < 6; j++) {
        double dj = fr[j] ? H[j][j] : 1.0;
#pragma unroll
        for (int k = 0; k < j; k++) dj -= Lm[j][k] * Lm[j][k] * D[k];
        pd = pd && dj > 1e-300;
        D[j] = dj;
        const double inv = rcp(dj);
#pragma unroll
        for (int i = j + 1; i < 6; i++) {
            double v = (fr[i] && fr[j]) ? H[i][j] : 0.0;
#pragma unroll
            for (int k = 0; k < j; k++) v -= Lm[i][k] * Lm[j][k] * D[k];
            Lm[i][j] = v * inv;
        }
    }
    if (!pd) return false;
    // V_n = H_FF^{-1} J_n (zero on fixed coordinates), M_mn = J_m . V_n
    double V[2][6];
#pragma unroll
    for (int n = 0; n < 2; n++) {
        double z[6];
#pragma unroll
        for (int i = 0; i < 6; i++) {
            double v = J[n][i];
#pragma unroll
            for (int k = 0; k < i; k++) v -= Lm[i][k] * z[k];
            z[i] = v;
        }
#pragma unroll
        for (int i = 5; i >= 0; i--) {
            double v = z[i] * rcp(D[i]);
#pragma unroll
            for (int k = i + 1; k < 6; k++) v -= Lm[k][i] * V[n][k];
            V[n][i] = v;
        }
    }
    const double a = dotn<6>(J[0], V[0]), d = dotn<6>(J[1], V[1]);
    const double b = 0.5 * (dotn<6>(J[0], V[1]) + dotn<6>(J[1], V[0]));
    const double mean = 0.5 * (a + d), half = 0.5 * (a - d);
    const double r = sqrt(half * half + b * b);
    const double lam0 = mean + r, lam1 = mean - r;
    double v0, v1;
    if (r == 0.0) {
        v0 = 1.0;
        v1 = 0.0;
    } else if (a >= d) {
        const double in = rcp(sqrt((lam0 - d) * (lam0 - d) + b * b));
        v0 = (lam0 - d) * in;
        v1 = b * in;
    } else {
        const double in = rcp(sqrt(b * b + (lam0 - a) * (lam0 - a)));
        v0 = b * in;
        v1 = (lam0 - a) * in;
    }
    const double thr = rcp(AL_NEWTON_C * sig);
    const double f0 = lam0 >= thr ? rcp(lam0) : sig, f1 = lam1 >= thr ? rcp(lam1) : sig;
    const double p0 = v0 * h[0] + v1 * h[1], p1 = -v1 * h[0] + v0 * h[1];
    dmu[0] = f0 * p0 * v0 - f1 * p1 * v1;
    dmu[1] = f0 * p0 * v1 + f1 * p1 * v0;
    // first-order move of the round's minimiser with mu (R43): dx_F = -H_FF^{-1} J_F' dmu
#pragma unroll
    for (int i = 0; i < 6; i++) dx[i] = -(V[0][i] * dmu[0] + V[1][i] * dmu[1]);
    return true;
}

// Newton step on the free set F by an LDL^T factorisation of H_FF (fixed rows/columns
// replaced by the identity).  Returns false if H_FF is not positive definite.
template <int N>
__device__ __forceinline__ bool newton_free(const double (*H)[N], const bool *fr, const double *r, double *w) {
    // L D L' with LD[i][j] = L[i][j] D[j] kept (no triple products) and the pivots inverted once
    double Lm[N][N], LD[N][N], iD[N];
    bool pd = true;
#pragma unroll
    for (int j = 0; j < N; j++) {
        double dj = fr[j] ? H[j][j] : 1.0;
#pragma unroll
        for (int k = 0; k < j; k++) dj -= Lm[j][k] * LD[j][k];
        pd = pd && dj > 1e-300;
        const double inv = rcp(dj);
        iD[j] = inv;
#pragma unroll
        for (int i = j + 1; i < N; i++) {
            double v = (fr[i] && fr[j]) ? H[i][j] : 0.0;
#pragma unroll
            for (int k = 0; k < j; k++) v -= Lm[i][k] * LD[j][k];
            LD[i][j] = v;
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
        double v = z[i] * iD[i];
#pragma unroll
        for (int k = i + 1; k < N; k++) v -= Lm[k][i] * w[k];
        w[i] = fr[i] ? v : 0.0;
    }
    return true;
}

#ifndef UCAC_NEWTON_FIRST
#define UCAC_NEWTON_FIRST 1
#endif
// Projected trust-region Newton.  Returns true when ||P(x-g)-x||_inf <= gtol.
template <int N, class Fun>
__device__ bool tron(const Fun &fn, double *x, const double *lo, const double *hi, double gtol,
                     int maxit, int &iters, double (*Hout)[N] = nullptr, double delta0 = TR_DELTA0) {
    double f, g[N], H[N][N];
#pragma unroll
    for (int i = 0; i < N; i++) x[i] = clampd(x[i], lo[i], hi[i]);
    fn.template eval<N, true>(x, f, g, H);
    double delta = delta0, alpha = 1.0;
    {
        // first Cauchy trial length: the model minimiser along -g (R41)
        double Hg[N];
        matvec<N>(H, g, Hg);
        const double gHg = dotn<N>(g, Hg), gg = dotn<N>(g, g);
        if (gHg > 0.0 && gg > 0.0) alpha = gg * rcp(gHg);
    }
    int it = 0;
    for (; it < maxit; it++) {
        double pgn = 0.0;
#pragma unroll
        for (int i = 0; i < N; i++) pgn = fmax(pgn, fabs(clampd(x[i] - g[i], lo[i], hi[i]) - x[i]));
        if (pgn <= gtol) {
            iters = it;
            if (Hout) copy_h<N>(H, Hout);
            return true;
        }
        double s[N], qs;   // step and its model value (reused by the ratio test)
        bool have_step = false;
        if (UCAC_NEWTON_FIRST && N == 4) {   // fast path only: in the 6-variable AL it cost spills
            // Newton first: with x strictly inside the box and H positive definite, TRON's step
            // from the Cauchy point sc is sc + w = -H^{-1} g whenever every coordinate stays free
            // (w solves H w = -(g + H sc)).  So when -H^{-1} g is interior and inside the trust
            // region it is taken directly, without computing sc; else the full step.
            bool inside = true;
#pragma unroll
            for (int i = 0; i < N; i++) inside = inside && x[i] > lo[i] && x[i] < hi[i];
            if (inside) {
                bool fr[N];
                double r[N], w[N];
#pragma unroll
                for (int i = 0; i < N; i++) {
                    fr[i] = true;
                    r[i] = -g[i];
                }
                if (newton_free<N>(H, fr, r, w) && dotn<N>(w, w) < delta * delta) {
                    bool in2 = true;
#pragma unroll
                    for (int i = 0; i < N; i++) in2 = in2 && x[i] + w[i] > lo[i] && x[i] + w[i] < hi[i];
                    if (in2) {
#pragma unroll
                        for (int i = 0; i < N; i++) s[i] = w[i];
                        qs = qmodel<N>(g, H, s);
                        have_step = qs < 0.0;
                    }
                }
            }
        }
        if (!have_step) {
            // --- Cauchy point: backtrack (x0.1) or extrapolate (x10) along P(x - a g)
            double sc[N];
            {
                double a = alpha;
                pstep<N>(x, lo, hi, g, a, sc);
                if (!cauchy_ok<N>(g, H, sc, delta)) {
                    for (int k = 0; k < 60; k++) {
                        a *= 0.1;
                        pstep<N>(x, lo, hi, g, a, sc);
                        if (cauchy_ok<N>(g, H, sc, delta)) break;
                    }
                } else {
                    for (int k = 0; k < 20; k++) {
                        double sp[N];
    #pragma unroll
                        for (int i = 0; i < N; i++) sp[i] = sc[i];
                        double ap = a;
                        a *= 10.0;
                        pstep<N>(x, lo, hi, g, a, sc);
                        bool same = true;
    #pragma unroll
                        for (int i = 0; i < N; i++) same = same && (sc[i] == sp[i]);
                        if (!cauchy_ok<N>(g, H, sc, delta) || same) {
                            a = ap;
    #pragma unroll
                            for (int i = 0; i < N; i++) sc[i] = sp[i];
                            break;
                        }
                    }
                }
                alpha = a;
            }
            // --- Steihaug-Toint CG on the free variables at x + sc, region ||sc + w|| <= delta
            bool fr[N];
            double gq[N], w[N];
            {
                double Hs[N];
                matvec<N>(H, sc, Hs);
    #pragma unroll
                for (int i = 0; i < N; i++) {
                    double xc = x[i] + sc[i];
                    fr[i] = (xc > lo[i]) && (xc < hi[i]);
                    gq[i] = g[i] + Hs[i];
                    w[i] = 0.0;
                }
                double r[N], p[N];
    #pragma unroll
                for (int i = 0; i < N; i++) {
                    r[i] = fr[i] ? -gq[i] : 0.0;
                    p[i] = r[i];
                }
                double rr = dotn<N>(r, r);
                bool direct = false;
                if (rr != 0.0 && N <= UCAC_TRON_DIRECT_MAXN) {
                    // the point CG converges to, when it is interior: the Newton step on the free set
                    if (newton_free<N>(H, fr, r, w)) {
                        double t[N];
    #pragma unroll
                        for (int i = 0; i < N; i++) t[i] = sc[i] + w[i];
                        direct = dotn<N>(t, t) < delta * delta;
                    }
                    if (!direct) {
    #pragma unroll
                        for (int i = 0; i < N; i++) w[i] = 0.0;
                    }
                }
                if (rr != 0.0 && !direct) {
                    double tol2 = TR_CGTOL * TR_CGTOL * rr;
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
                        double a = rr * rcp(kap);
                        double tt[N];
    #pragma unroll
                        for (int i = 0; i < N; i++) tt[i] = t[i] + a * p[i];
                        if (dotn<N>(tt, tt) >= delta * delta) {
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
                        double b = rn * rcp(rr);
    #pragma unroll
                        for (int i = 0; i < N; i++) p[i] = r[i] + b * p[i];
                        rr = rn;
                    }
                }
            }
            // --- projected search along w from the Cauchy point
            {
                const double qc = qmodel<N>(g, H, sc);
                double b = 1.0;
                bool found = false;
                for (int k = 0; k < 20; k++) {
                    double ds[N];
    #pragma unroll
                    for (int i = 0; i < N; i++) {
                        s[i] = clampd(x[i] + sc[i] + b * w[i], lo[i], hi[i]) - x[i];
                        ds[i] = s[i] - sc[i];
                    }
                    qs = qmodel<N>(g, H, s);
                    if (qs <= qc + TR_MU0 * dotn<N>(gq, ds)) {
                        found = true;
                        break;
                    }
                    b *= 0.5;
                }
                if (!found) {
    #pragma unroll
                    for (int i = 0; i < N; i++) s[i] = sc[i];
                    qs = qc;
                }
            }
        }
        const double ss = dotn<N>(s, s);
        // --- stall: a step at the rounding level of x means the gradient floor is reached
        {
            double xm = 0.0;
#pragma unroll
            for (int i = 0; i < N; i++) xm = fmax(xm, fabs(x[i]));
            const double tol = TR_STALL * (1.0 + xm);
            if (ss <= tol * tol) {
                iters = it;
                if (Hout) copy_h<N>(H, Hout);
                return true;
            }
        }
        // --- ratio test
        double pred = -qs;
        double xn[N], gn[N], fnew;
#pragma unroll
        for (int i = 0; i < N; i++) xn[i] = clampd(x[i] + s[i], lo[i], hi[i]);
        // one evaluation with the Hessian at the trial point, adopted if the step is accepted
        // (accepted steps are the common case: this saves the second flow evaluation)
        double Hn[N][N];
        fn.template eval<N, true>(xn, fnew, gn, Hn);
        double ared = f - fnew;
        if (fabs(pred) <= TR_EPSF * fabs(f)) ared = -0.5 * (dotn<N>(g, s) + dotn<N>(gn, s));
        double ratio = pred > 0.0 ? ared * rcp(pred) : -1.0;
        double snorm = sqrt(ss);
        if (ratio > TR_ETA0) {
#pragma unroll
            for (int i = 0; i < N; i++) x[i] = xn[i];
            f = fnew;
#pragma unroll
            for (int i = 0; i < N; i++) {
                g[i] = gn[i];
#pragma unroll
                for (int j = 0; j < N; j++) H[i][j] = Hn[i][j];
            }
        }
        if (ratio < TR_ETA1) delta = TR_SIG1 * fmin(snorm, delta);
        else if (ratio > TR_ETA2) delta = fmax(delta, TR_SIG3 * snorm);
    }
    iters = it;
    if (Hout) copy_h<N>(H, Hout);
    double pgn = 0.0;
#pragma unroll
    for (int i = 0; i < N; i++) pgn = fmax(pgn, fabs(clampd(x[i] - g[i], lo[i], hi[i]) - x[i]));
    return pgn <= gtol;
}

__device__ __forceinline__ void warp_add_u64(unsigned long long *dst, unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// load the data of solve k = l*T + t: admittances, targets tau = xbar - z - y/rho (5.1), w bounds
// zs/ys (optional, stride `ss`): keep z and y/rho of the 8 rows for the tauhat emission
template <bool NOANG>
__device__ __forceinline__ void load_solve(const Dev &d, int k, BrFun<false, NOANG> &F, double *wlo, double *whi,
                                           double *zs = nullptr, double *ys = nullptr, int ss = 0) {
    const size_t LTs = (size_t)d.L * d.T;
    const int l = k / d.T, t = k - l * d.T;
    const int bi = d.bfrom[l], bj = d.bto[l];
    F.Gii = d.y[0 * d.L + l]; F.Gij = d.y[1 * d.L + l]; F.Gji = d.y[2 * d.L + l]; F.Gjj = d.y[3 * d.L + l];
    F.Bii = d.y[4 * d.L + l]; F.Bij = d.y[5 * d.L + l]; F.Bji = d.y[6 * d.L + l]; F.Bjj = d.y[7 * d.L + l];
    F.rpq = d.rpq;
    F.rva = d.rva;
    const size_t wi = (size_t)bi * d.T + t, wj = (size_t)bj * d.T + t;
    const double xb[8] = {d.fbar[0 * LTs + k], d.fbar[1 * LTs + k], d.fbar[2 * LTs + k], d.fbar[3 * LTs + k],
                          d.wbar[wi], d.wbar[wj], d.thbar[wi], d.thbar[wj]};
#pragma unroll
    for (int r = 0; r < 8; r++) {
        // y * (1/rho) instead of y / rho: within one ulp of the oracle's quotient, and no division
        // (whose slow-path call made the compiler spill around each of the eight loads)
        const double z = d.zb[r * LTs + k], yr = d.yb[r * LTs + k] * (r < 4 ? d.irpq : d.irva);
        F.tau[r] = xb[r] - z - yr;
        if (zs) {
            zs[r * ss] = z;
            ys[r * ss] = yr;
        }
    }
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
// end instead of the row state.  y/rho is formed as y * (1/rho) (within one ulp of the
// oracle's quotient).
__device__ __forceinline__ void emit_tauhat_zy(const Dev &d, int k, const double *x, double f0, double f1,
                                               double f2, double f3, const double *zs, const double *ys, int ss) {
    const size_t LTH = (size_t)(d.L + d.Lph) * d.T;      // tauhat kind stride includes phantom branches
    const double xs[8] = {f0, f1, f2, f3, x[0], x[1], x[2], x[3]};
#pragma unroll
    for (int r = 0; r < 8; r++) d.tauh[r * LTH + k] = xs[r] + zs[r * ss] + ys[r * ss];
}
__device__ __forceinline__ void emit_tauhat(const Dev &d, int k, const double *x, double f0, double f1,
                                            double f2, double f3) {
    const size_t LTs = (size_t)d.L * d.T;                // row-state kind stride
    const size_t LTH = (size_t)(d.L + d.Lph) * d.T;      // tauhat kind stride includes phantom branches
    const double xs[8] = {f0, f1, f2, f3, x[0], x[1], x[2], x[3]};
#pragma unroll
    for (int r = 0; r < 8; r++) {
        d.tauh[r * LTH + k] = xs[r] + d.zb[r * LTs + k] + d.yb[r * LTs + k] * (r < 4 ? d.irpq : d.irva);
    }
}

#ifndef UCAC_BRANCH_TPB
#define UCAC_BRANCH_TPB 128
#endif
#ifndef UCAC_BRANCH_MINB
#define UCAC_BRANCH_MINB 3
#endif
#ifndef UCAC_AL_TPB
#define UCAC_AL_TPB 256
#endif
#ifndef UCAC_AL_DEAL
#define UCAC_AL_DEAL 2
#endif
#ifndef UCAC_AL_BLOCKS_PER_SM
#define UCAC_AL_BLOCKS_PER_SM 1
#endif
template <bool NOANG>
__global__ void __launch_bounds__(UCAC_BRANCH_TPB, UCAC_BRANCH_MINB) k_branch(Dev d) {
    pdl_wait();
    TL_KERNEL(K_BRANCH);
    if (d.st->done) return;
    const int LT = d.L * d.T;
    unsigned long long c_it = 0, c_cap = 0;
    // grid-stride over 128-solve chunks: the grid is sized to leave SM slots free for the
    // generator chain that runs beside this kernel (launch_branch)
    for (int base = blockIdx.x * blockDim.x; base < LT; base += gridDim.x * blockDim.x) {
    const int k = base + threadIdx.x;
    if (k < LT && own_t(d, k % d.T)) {   // (time cut: owned periods only)
        const size_t LTs = (size_t)LT;
        BrFun<false, NOANG> F4;
        double lo[4], hi[4];
        // z and y/rho of the 8 rows, kept in shared memory for the tauhat emission
        __shared__ double s_z[8][UCAC_BRANCH_TPB], s_y[8][UCAC_BRANCH_TPB];
        load_solve(d, k, F4, lo, hi, &s_z[0][threadIdx.x], &s_y[0][threadIdx.x], UCAC_BRANCH_TPB);
        lo[2] = -TWO_PI; hi[2] = TWO_PI; lo[3] = -TWO_PI; hi[3] = TWO_PI;
        if (NOANG) lo[2] = hi[2] = 0.0;   // R51: the line's own angle reference
        double x[4];
#pragma unroll
        for (int m = 0; m < 4; m++) x[m] = d.x[m * LTs + k];
        const double rate = d.rate[k / d.T];
        const double r2 = rate * rate;
        // NEXT-3 variant 1 (R47): every rated branch goes straight to the AL from the clipped warm start
        const bool al_always = (d.variant & 1) && rate > 0.0;
        if (al_always) {
#pragma unroll
            for (int m = 0; m < 4; m++) x[m] = clampd(x[m], lo[m], hi[m]);
        } else {
            int it = 0;
            const bool ok = tron<4>(F4, x, lo, hi, d.tron_gtol, d.tron_maxit, it);
            c_it += it;
            c_cap += !ok;
        }
        double C, S, f0, f1, f2, f3;
        F4.flows(x, C, S, f0, f1, f2, f3);
        {
            double chk = nf0(f0) + nf0(f1) + nf0(f2) + nf0(f3);
#pragma unroll
            for (int r = 0; r < 8; r++) chk += nf0(F4.tau[r]);
            if (!isfinite(chk)) report_nonfinite(d, K_BRANCH, k / d.T, k - (k / d.T) * d.T);
        }
        const bool queue = rate > 0.0 && (al_always || f0 * f0 + f1 * f1 > r2 || f2 * f2 + f3 * f3 > r2);
        if (queue) {
            // AL queue buckets by the solve's previous AL Newton count: heavy and newly
            // active solves first, so the block-major dealing groups similar chains per warp and the
            // blocks holding light solves release their SMs early
            const int pit = UCAC_AL_BUCKETS > 1 ? d.alits[k] : 0;
            const int b = UCAC_AL_BUCKETS == 1 ? 0 : (pit == 0 || pit >= 9 ? 0 : (pit >= 6 || UCAC_AL_BUCKETS == 2 ? 1 : 2));
            const unsigned pos = atomicAdd(d.alq_cnt + b, 1u);
            d.alq[(size_t)b * LTs + pos] = k;
            d.qmark[k] = mark_stamp(d);   // (multi-rank: flags a cut end's tauhat as not final)
            // the previous iterate (still in d.x): the AL's second candidate start (R49)
#pragma unroll
            for (int m = 0; m < 4; m++) d.alq_x[m * LTs + k] = d.x[m * LTs + k];
        } else if (UCAC_AL_BUCKETS > 1 && d.alits[k]) {
            d.alits[k] = 0;
        }
#pragma unroll
        for (int m = 0; m < 4; m++) d.x[m * LTs + k] = x[m];
        d.f[0 * LTs + k] = f0;
        d.f[1 * LTs + k] = f1;
        d.f[2 * LTs + k] = f2;
        d.f[3 * LTs + k] = f3;
        if (queue) {
            // mark both end buses and every branch end at them: their bus solve and end rows move
            // to the late phase, after the AL tail
            const int l = k / d.T, t = k - l * d.T;
            const unsigned stamp = mark_stamp(d);
#pragma unroll
            for (int side = 0; side < 2; side++) {
                const int bus = side ? d.bto[l] : d.bfrom[l];
                d.bmark[(size_t)bus * d.T + t] = stamp;
                if (bus < d.B_own)
                    for (int a = d.be_ptr[bus]; a < d.be_ptr[bus + 1]; a++) {
                        const int code = d.be_idx[a];
                        d.rmark[code & 1][(size_t)(code >> 1) * d.T + t] = stamp;
                    }
            }
        } else {
            d.al[0 * LTs + k] = 0.0;
            d.al[1 * LTs + k] = 0.0;
            d.al[2 * LTs + k] = d.al_sigma0_rel * d.rpq * r2;
            emit_tauhat_zy(d, k, x, f0, f1, f2, f3, &s_z[0][threadIdx.x], &s_y[0][threadIdx.x], UCAC_BRANCH_TPB);
        }
    }
    }
    warp_add_u64(d.cnt + 0, c_it);
    warp_add_u64(d.cnt + 1, c_cap);
}

// Phase 2: the queued thermal-active solves (6-variable slack AL, R36), pulled one at a time
// by every thread of a persistent grid, so the heavy tail is spread over all SMs.
template <bool NOANG>
__global__ void __launch_bounds__(UCAC_AL_TPB) k_branch_al(Dev d) {
    pdl_wait();
    TL_KERNEL(K_BRANCH_AL);
    if (d.st->done) return;
    const size_t LTs = (size_t)d.L * d.T;
    unsigned nb[UCAC_AL_BUCKETS], n = 0;
#pragma unroll
    for (int b = 0; b < UCAC_AL_BUCKETS; b++) {
        nb[b] = *((volatile unsigned *)d.alq_cnt + b);
        n += nb[b];
    }
    unsigned long long c_it = 0, c_cap = 0, c_al = 0, c_alcap = 0, c_alit = 0;
#if UCAC_AL_DEAL == 2
    // block-major static dealing: the queue fills the first blocks, so the AL work sits on few SMs
    // (with full-register-file blocks, exclusively) and the other SMs run the concurrent sweeps
    for (unsigned idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += gridDim.x * blockDim.x) {
#elif UCAC_AL_DEAL == 1
    // lane-major static dealing: item lane * nwarps + warp, so each warp carries few solves
    const unsigned nwarps = (gridDim.x * blockDim.x) >> 5;
    const unsigned gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    for (unsigned idx = lane * nwarps + gwarp; idx < n; idx += 32 * nwarps) {
#else
    for (;;) {
        const unsigned idx = atomicAdd(d.alq_cnt + UCAC_AL_BUCKETS, 1u);
        if (idx >= n) break;
#endif
        int k;
        {
            unsigned b = 0, p = idx;
            while (b + 1 < UCAC_AL_BUCKETS && p >= nb[b]) p -= nb[b++];
            k = d.alq[(size_t)b * LTs + p];
        }
        const unsigned long long alit0 = c_alit;
#ifdef UCAC_PROF
        unsigned long long t_start;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
        const unsigned long long it0 = c_it;
#endif
        BrFun<true, NOANG> F6;
        double lo[6], hi[6];
        {
            BrFun<false, NOANG> F4;
            load_solve(d, k, F4, lo, hi);
            F6.Gii = F4.Gii; F6.Gij = F4.Gij; F6.Gji = F4.Gji; F6.Gjj = F4.Gjj;
            F6.Bii = F4.Bii; F6.Bij = F4.Bij; F6.Bji = F4.Bji; F6.Bjj = F4.Bjj;
#pragma unroll
            for (int r = 0; r < 8; r++) F6.tau[r] = F4.tau[r];
            F6.rpq = F4.rpq; F6.rva = F4.rva;
            F6.K00 = F4.K00; F6.K02 = F4.K02; F6.K03 = F4.K03; F6.K11 = F4.K11;
            F6.K12 = F4.K12; F6.K13 = F4.K13; F6.K22 = F4.K22;
        }
        lo[2] = -TWO_PI; hi[2] = TWO_PI; lo[3] = -TWO_PI; hi[3] = TWO_PI;
        if (NOANG) lo[2] = hi[2] = 0.0;   // R51
        lo[4] = 0.0; hi[4] = 1.0; lo[5] = 0.0; hi[5] = 1.0;
        const double rate = d.rate[k / d.T];
        const double r2 = rate * rate;
        const double sig0 = d.al_sigma0_rel * d.rpq * r2;
        F6.r2inv = rcp(r2);
        double x[6];
#pragma unroll
        for (int m = 0; m < 4; m++) x[m] = d.x[m * LTs + k];
        {
            const double f0 = d.f[0 * LTs + k], f1 = d.f[1 * LTs + k], f2 = d.f[2 * LTs + k], f3 = d.f[3 * LTs + k];
            x[4] = clampd(1.0 - (f0 * f0 + f1 * f1) * F6.r2inv, 0.0, 1.0);
            x[5] = clampd(1.0 - (f2 * f2 + f3 * f3) * F6.r2inv, 0.0, 1.0);
        }
        double mu0 = d.al[0 * LTs + k], mu1 = d.al[1 * LTs + k];
        double sig = fmax(sig0, d.al[2 * LTs + k] * d.al_sigma_decay);
        {
            // R49: round 1 starts from whichever of the fast-path point and the previous iterate
            // (each with its slacks from its flows) has the lower AL value
            double xp[6], C0, S0, p0, p1, p2, p3;
#pragma unroll
            for (int m = 0; m < 4; m++) xp[m] = clampd(d.alq_x[m * LTs + k], lo[m], hi[m]);
            F6.flows(xp, C0, S0, p0, p1, p2, p3);
            xp[4] = clampd(1.0 - (p0 * p0 + p1 * p1) * F6.r2inv, 0.0, 1.0);
            xp[5] = clampd(1.0 - (p2 * p2 + p3 * p3) * F6.r2inv, 0.0, 1.0);
            F6.mu0 = mu0; F6.mu1 = mu1; F6.sig = sig;
            if (F6.value(xp) < F6.value(x)) {
#pragma unroll
                for (int m = 0; m < 6; m++) x[m] = xp[m];
            }
        }
        const double smax = d.al_sigma_max_rel * sig0;
        double hprev = INFINITY;
        double C, S, f0, f1, f2, f3;
        int kk = 0;
        c_al += 1;
        for (; kk < d.al_maxit; kk++) {
            F6.mu0 = mu0; F6.mu1 = mu1; F6.sig = sig;
            int it = 0;
            double Hx[6][6];
            // round 1 starts at the fast-path point, which violates Eq. 2c-2d: small first radius (R44)
            bool ok = tron<6>(F6, x, lo, hi, d.tron_gtol, d.tron_maxit, it, Hx, kk == 0 ? AL_R1_DELTA0 : TR_DELTA0);
            c_it += it;
            c_alit += it;
            c_cap += !ok;
            F6.flows(x, C, S, f0, f1, f2, f3);
            double h1 = (f0 * f0 + f1 * f1) * F6.r2inv - 1.0 + x[4];
            double h2 = (f2 * f2 + f3 * f3) * F6.r2inv - 1.0 + x[5];
            double hm = fmax(fabs(h1), fabs(h2));
            if (hm <= d.al_eta_star) break;
            const double hv[2] = {h1, h2};
            double dmu[2], dx[6];
            if (al_newton_dmu(Hx, x, lo, hi, sig, hv, dmu, dx)) {
#pragma unroll
                for (int i = 0; i < 6; i++) x[i] = clampd(x[i] + dx[i], lo[i], hi[i]);
            } else {
                dmu[0] = sig * h1;
                dmu[1] = sig * h2;
            }
            mu0 += dmu[0];
            mu1 += dmu[1];
            if (hm > 0.25 * hprev) sig = fmin(10.0 * sig, smax);
            hprev = hm;
        }
        c_alcap += kk >= d.al_maxit;
        F6.flows(x, C, S, f0, f1, f2, f3);
        if (!isfinite(nf0(f0) + nf0(f1) + nf0(f2) + nf0(f3) + nf0(mu0) + nf0(mu1)))
            report_nonfinite(d, K_BRANCH_AL, k / d.T, k - (k / d.T) * d.T);
#pragma unroll
        for (int m = 0; m < 4; m++) d.x[m * LTs + k] = x[m];
        d.f[0 * LTs + k] = f0;
        d.f[1 * LTs + k] = f1;
        d.f[2 * LTs + k] = f2;
        d.f[3 * LTs + k] = f3;
        d.al[0 * LTs + k] = mu0;
        d.al[1 * LTs + k] = mu1;
        d.al[2 * LTs + k] = sig;
        if (UCAC_AL_BUCKETS > 1) d.alits[k] = (uint8_t)min(255ull, max(1ull, c_alit - alit0));
        emit_tauhat(d, k, x, f0, f1, f2, f3);
#ifdef UCAC_PROF
        {
            unsigned long long t_end;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
            if (idx < (1u << 16)) {
                unsigned long long *r = g_prof + 6ull * idx;
                r[0] = k; r[1] = t_start; r[2] = t_end; r[3] = c_it - it0; r[4] = kk + 1;
                r[5] = ((unsigned long long)(blockIdx.x * blockDim.x + threadIdx.x) >> 5) << 8 | (threadIdx.x & 31);
            }
        }
#endif
    }
    if (c_it) atomicAdd(d.cnt + 0, c_it);
    if (c_cap) atomicAdd(d.cnt + 1, c_cap);
    if (c_al) atomicAdd(d.cnt + 2, c_al);
    if (c_alcap) atomicAdd(d.cnt + 3, c_alcap);
    if (c_alit) atomicAdd(d.cnt + 4, c_alit);
}

}  // namespace

#ifndef UCAC_BRANCH_FREE_SLOTS
#define UCAC_BRANCH_FREE_SLOTS 24
#endif
#ifndef UCAC_BRANCH_CARVEOUT
#define UCAC_BRANCH_CARVEOUT -1   // driver default; 50 and 100 measured slower
#endif
void launch_branch(const Dev &d, cudaStream_t s) {
    // shared-memory carveout: 3 k_branch blocks need 52 KB; a larger carveout lets the generator
    // chain's blocks (k_gen: 4 x dp_smem_bytes(T), ~10 KB at T = 48) co-reside in the free slots instead of waiting for the
    // SM to drain
    static const bool carve = [] {
        return UCAC_BRANCH_CARVEOUT < 0 ||
               cudaFuncSetAttribute(k_branch<false>, cudaFuncAttributePreferredSharedMemoryCarveout, UCAC_BRANCH_CARVEOUT) == cudaSuccess;
    }();
    (void)carve;
    const int n = d.L * d.T, chunks = (n + UCAC_BRANCH_TPB - 1) / UCAC_BRANCH_TPB;
    // 148 SMs x UCAC_BRANCH_MINB resident blocks, minus the slots left to the generator chain
    const int grid = std::max(1, std::min(chunks, 148 * UCAC_BRANCH_MINB - UCAC_BRANCH_FREE_SLOTS));
    if (pdl_mask() & 8) {   // after the previous iteration's last kernel (experiments)
        if (d.variant & 8) launch_ex(k_branch<true>, dim3(grid), dim3(UCAC_BRANCH_TPB), 0, s, false, true, d);
        else launch_ex(k_branch<false>, dim3(grid), dim3(UCAC_BRANCH_TPB), 0, s, false, true, d);
        return;
    }
    if (d.variant & 8) k_branch<true><<<grid, UCAC_BRANCH_TPB, 0, s>>>(d);
    else k_branch<false><<<grid, UCAC_BRANCH_TPB, 0, s>>>(d);
}
#ifndef UCAC_AL_PRIO
#define UCAC_AL_PRIO 0
#endif
#ifndef UCAC_AL_SMEM
#define UCAC_AL_SMEM 0   // dynamic shared memory per AL block (bytes): > 0 reserves SMs for the AL work
#endif
void launch_branch_al(const Dev &d, cudaStream_t s) {
    if (UCAC_AL_SMEM > 48 * 1024) {
        cudaFuncSetAttribute(k_branch_al<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, UCAC_AL_SMEM);
        cudaFuncSetAttribute(k_branch_al<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, UCAC_AL_SMEM);
    }
    const dim3 grid(148 * UCAC_AL_BLOCKS_PER_SM), block(UCAC_AL_TPB);
    const bool pdl = (pdl_mask() & 1) != 0;
    if (UCAC_AL_PRIO || pdl) {   // high launch priority: its full-SM blocks take SMs as k_branch drains
        if (d.variant & 8) launch_ex(k_branch_al<true>, grid, block, (size_t)UCAC_AL_SMEM, s, UCAC_AL_PRIO != 0, pdl, d);
        else launch_ex(k_branch_al<false>, grid, block, (size_t)UCAC_AL_SMEM, s, UCAC_AL_PRIO != 0, pdl, d);
    } else {
        if (d.variant & 8) k_branch_al<true><<<grid, block, UCAC_AL_SMEM, s>>>(d);
        else k_branch_al<false><<<grid, block, UCAC_AL_SMEM, s>>>(d);
    }
}

}  // namespace ucac

#ifdef UCAC_PROF
extern "C" int ucac_debug_prof(void *host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, ucac::g_prof, bytes < sizeof(ucac::g_prof) ? bytes : sizeof(ucac::g_prof));
}
#endif
