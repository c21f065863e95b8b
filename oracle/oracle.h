/*
 * oracle.h -- PLAIN CPU ORACLE for the UC-ACOPF two-level ADMM (arXiv 2310.13145).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load liboracle.so.  The product path
 * (paper_2310_13145_b200/, libucac.so) never includes, links or calls anything here,
 * and this file shares no code, header, table or constant with it.
 *
 * Citations "P:n" are lines of /root/reference/PAPER.md (the paper's LaTeX source);
 * "Rk" are the readings registered in DESIGN.md section 3.
 *
 * Everything is fp64, single threaded, canonical order: component index, then period.
 * Arrays indexed [c*T + t] (t = 0..T-1 stands for the paper's period t+1).
 */
#ifndef UCAC_ORACLE_H
#define UCAC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Problem data, per unit on base_mva.  Same semantics as the product ABI but an
 * independent declaration (the two codes share no header). */
typedef struct {
    int32_t nbus, ngen, nbranch, T, ref_bus;
    double base_mva;
    const double *bus_gs, *bus_bs, *bus_vmin, *bus_vmax;      /* [nbus]            */
    const double *pd, *qd;                                    /* [T*nbus] t-major  */
    const int32_t *br_from, *br_to;                           /* [nbranch]         */
    const double *br_y;        /* [nbranch*8] Gii,Gij,Gji,Gjj,Bii,Bij,Bji,Bjj       */
    const double *br_rate;     /* [nbranch] r-bar pu, 0 = unlimited                 */
    const int32_t *gen_bus;                                   /* [ngen]            */
    const double *pmin, *pmax, *qmin, *qmax;                  /* [ngen] pu         */
    const double *c2, *c1, *c0, *csu, *csd;                   /* $/MW^2h, $/MWh, $/h */
    const double *ramp_up, *ramp_dn, *su_ramp, *sd_ramp;      /* pu / period       */
    const int32_t *min_up, *min_dn, *u0, *hold;               /* [ngen]            */
    const double *p0;                                         /* [ngen] pu         */
    const int8_t *u_init;      /* [ngen*T] (g-major) or NULL                        */
} orc_problem;

typedef struct {
    double rho_pq, rho_va, rho_uc;
    double beta0, tau, theta, lambda_max, beta_max;
    double eps_inner_abs;
    int32_t inner_min, inner_cap, outer_enabled;
    double tron_gtol_rel;
    int32_t tron_maxit, al_maxit;
    double al_eta_star, al_sigma0_rel, al_sigma_max_rel, al_sigma_decay;
    int32_t uc_fixed;   /* 1: step (7a) keeps u (the NEXT-2 warm start's multiperiod ACOPF) */
    int32_t variant;    /* NEXT-3 formulation variants (bitmask, R47): 1 = every rated branch solves the
                           six-variable AL (no fast path), 2 = wbar clipped to [Vmin^2, Vmax^2] */
    int32_t plain;      /* 1: the branch solver without the accelerations R41-R44, R48, R49 (the plain
                           first-order AL that pins the accelerated one; oracle only) */
    int32_t diverge_window;   /* SPEC S:431 divergence detector: > 0 = an iterate call stops when the
                                 primal residual exceeds diverge_factor x its value diverge_window
                                 iterations earlier (first time only); 0 = off */
    double diverge_factor;
} orc_params;

typedef struct {
    double primal_inf, rz_inf, rz_2, z_inf, z_2, dual_inf, objective, beta;
    int64_t inner_total, outer_total, tron_iters, tron_capped, al_active, al_capped;
    int32_t inner_since_outer, outer_k;
    /* the last iteration's branch solves (R55): algorithmic flops and Newton iterations of the
     * 4-variable fast path and of the 6-variable AL */
    double flops_fast, flops_al;
    int64_t newton_fast, newton_al;
    int32_t diverged_iter, pad_;   /* first iteration the divergence detector fired (0 = never) */
} orc_report;

/* Canonical state (section 4 of DESIGN.md).  Row kinds:
 * gen rows   (12 per (g,t)): D_ON D_SU D_SD PL PU QL QU RD RU GP GQ RC
 * branch rows (8 per (l,t)): FP_IJ FQ_IJ FP_JI FQ_JI W_I W_J A_I A_J
 * row arrays are [kind][comp*T + t]. */
typedef struct {
    int8_t *u;                               /* [ngen*T] */
    double *p, *q, *ph, *ub_on, *ub_su, *ub_sd, *pbar, *qbar;           /* [ngen*T] */
    double *zg, *yg, *lg;                    /* [12*ngen*T] */
    double *x;                               /* [nbranch*T*4] w_i w_j th_i th_j */
    double *f;                               /* [nbranch*T*4] p_ij q_ij p_ji q_ji */
    double *fbar;                            /* [nbranch*T*4] bus-side flow copies */
    double *al;                              /* [nbranch*T*3] mu_ij mu_ji sigma */
    double *zb, *yb, *lb;                    /* [8*nbranch*T] */
    double *wbar, *thbar;                    /* [nbus*T] */
    double *scal;  /* [8]: beta, znorm_prev, outer_k, inner_total, inner_since, 0,0,0 */
} orc_state;

typedef struct orc_ctx orc_ctx;

int  orc_create(const orc_problem *pb, const orc_params *pr, orc_ctx **out);
void orc_destroy(orc_ctx *c);
int  orc_iterate(orc_ctx *c, int32_t n);                 /* n inner iterations */
void orc_set_rho(orc_ctx *c, double rho_pq, double rho_va, double rho_uc);   /* NEXT-4(b), R53 */
void orc_report_get(const orc_ctx *c, orc_report *r);
void orc_get_state(const orc_ctx *c, orc_state *s);
void orc_set_state(orc_ctx *c, const orc_state *s);

/* ---- single-step entry points used by the pin tests ---- */
/* S1 stage cost table L[t][a][b] for one generator (Section III-B). */
void orc_stage_costs(int32_t T, double c0, double csu, double csd, double rho_uc,
                     const double *ub /*[3*T]: on,su,sd t-minor blocks*/,
                     const double *y /*[3*T]*/, const double *z /*[3*T]*/, double *L /*[T*4]*/);
/* S1 DP, Algorithm 2.  Returns the optimal cost; sched[T]. */
/* NEXT-2 warm start (SPEC warm_start_uc): u = [p > threshold] repaired to the nearest
 * schedule satisfying Eq. 3 (min-up/down, held prefix) by one DP pass with stage costs
 * L_t(a, b) = [b != u_t] (Hamming distance; ties as the DP: stay). */
void orc_uc_repair(int32_t T, const double *p, double threshold, int32_t TU, int32_t TD, int32_t u0,
                   int32_t hold, int8_t *u_out);
double orc_dp(int32_t T, const double *L /*[T*4] L[t*4+a*2+b]*/, int32_t TU, int32_t TD,
              int32_t u0, int32_t hold, int8_t *sched);
/* S2 generator x-update for one (g,t). in[]: see oracle.c gen_x_update. out: p,q,ph. */
void orc_gen_x(const double *in, double *out);
/* S4 ubar group box-QP: n vars, m rows, c[m*3] (row-major, 3 cols), e[m] -> v[n]. */
void orc_boxqp3(int32_t n, int32_t m, const double *c, const double *e, double *v);
/* S5 bus closed form: k copies with (alpha,beta,a,tauhat) -> v; returns muP,muQ. */
void orc_bus_kkt(int32_t k, const double *alpha, const double *beta, const double *a,
                 const double *tauhat, double P, double Q, double *v, double *mu);
/* S3 branch solve.  y[8] admittance, lo/hi[2] w bounds (i,j), rate (0=unlimited),
 * tau[8] row targets, x[4] in/out, al[3] in/out, f[4] out, stats[9] out
 * (tron iterations, tron capped, al active, al iterations, al capped, flops fast path,
 * flops AL, Newton its fast path, Newton its AL). */
void orc_branch_solve(const double *y, const double *wlo, const double *whi, double rate,
                      const double *tau, double rho_pq, double rho_va, const orc_params *pr,
                      double *x, double *al, double *f, int64_t *stats);
/* Generic TRON on a dense quadratic 0.5 x'Ax + b'x over a box (pin: active-set enum). */
int orc_tron_quadratic(int32_t n, const double *A, const double *b, const double *lo,
                       const double *hi, double gtol, int32_t maxit, double *x);
/* Flows of one branch (Eq. 2e-2h) and derivative tables, for finite-difference pins. */
void orc_branch_flows(const double *y, const double *x, double *f, double *J /*[16]*/,
                      double *H /*[64]*/);
/* sin and cos by the explicit polynomial of R54 (the flows' only transcendental). */
void orc_sincos(double a, double *s, double *c);
/* the generator slacks of the current x (s^pl s^pu s^ql s^qu s^rd s^ru per (g,t), [6*ngen*T]) */
void orc_get_slacks(const orc_ctx *c, double *sl);
/* threads of the all-core build (n > 0 sets them); 1 for the single-thread build */
int orc_threads(int32_t n);

#ifdef __cplusplus
}
#endif
#endif
