/*
 * ucac.h -- C ABI of the B200-native hot path of the component-decomposed two-level ADMM
 * for unit commitment with AC optimal power flow (Zhang, Kim & Kim, arXiv 2310.13145,
 * "On Solving Unit Commitment with Alternating Current Optimal Power Flow on GPU").
 *
 * Citations "P:n" are lines of the paper's LaTeX source; "Rk" are the readings
 * registered in DESIGN.md section 3 where the paper is silent or garbled.
 *
 * One inner ADMM iteration (Alg. 1 lines 4-9; steps (7a)-(7f)) runs
 * entirely on the device as hand-written fp64 sm_100a kernels:
 *   (7a) UC dynamic program per generator            (Alg. 2)
 *   (7b) generator closed form per (g,t) + branch trust-region Newton per (l,t)
 *   (7c) ubar box-QP per (g, period group)
 *   (7d) bus closed form per (i,t)
 *   (7e) z, (7f) y per coupling row
 *   residual reduction, inner test and outer (lambda, beta) update.
 *
 * Conventions (all entry points):
 *  - Units: per unit on base_mva (p, q, flows in pu; w = |V|^2 in pu^2; angles in rad);
 *    costs in $ per 1-h period with p in MW inside the cost (c2 (S p)^2 + c1 S p).
 *  - Arrays: plain HOST pointers unless a name says "_dev".  Component-major, period-minor:
 *    element (c, t) of a [C*T] array is at c*T + t (t = 0 is the paper's period 1), except
 *    the demand arrays pd/qd which are period-major [T*nbus] (P_{t,i} at t*nbus + i).
 *  - Ownership: ucac_create deep-copies every input; the caller may free them on return.
 *    The context owns all device memory.  Output buffers are caller-allocated with the sizes
 *    stated per call.
 *  - Errors: every call returns ucac_status; nothing throws or aborts across the ABI.
 *    ucac_last_error(ctx) (or ucac_last_error(NULL) after a failed create) gives a message.
 *  - Threading: one context per host thread; no global mutable state.
 *  - The library requires a CUDA device of compute capability 10.0 (B200, sm_100a).  It never
 *    falls back to the CPU: without a device every call returns UCAC_ECUDA.
 */
#ifndef UCAC_H
#define UCAC_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ucac_ctx ucac_ctx;

typedef enum {
    UCAC_OK = 0,
    UCAC_EINVAL = 1,       /* invalid argument or problem data (message says which)        */
    UCAC_ENOMEM = 2,       /* device or host allocation failed                               */
    UCAC_ECUDA = 3,        /* CUDA runtime error or no sm_100 device                         */
    UCAC_ENCCL = 4,        /* NCCL error (multi-GPU contexts)                                */
    UCAC_ENUMERIC = 5,     /* a non-finite iterate was produced (report.err_* say where)     */
    UCAC_ESTATE = 6,       /* call not valid in the current state                            */
    UCAC_EUNSUPPORTED = 7
} ucac_status;

/* Network, Eq. (2).  Branch l = (i -> j) carries the MATPOWER two-port
 * admittance entries of Eq. 2e-2h: br_y[8*l + k], k = Gii,Gij,Gji,Gjj,Bii,Bij,Bji,Bjj (R1:
 * the to-side equations 2g-2h are read with ji labels).  br_rate = rbar_ij of Eq. 2c-2d,
 * 0 = unlimited (R12).  Bus voltage bounds enter as w in [vmin^2, vmax^2] (Eq. 2k). */
typedef struct {
    int32_t nbus, ngen, nbranch, ref_bus;
    double base_mva;
    const double *bus_gs, *bus_bs, *bus_vmin, *bus_vmax;   /* [nbus]                     */
    const int32_t *br_from, *br_to;                         /* [nbranch], 0-based         */
    const double *br_y;                                     /* [nbranch*8]                */
    const double *br_rate;                                  /* [nbranch] pu               */
    const int32_t *gen_bus;                                 /* [ngen]                     */
    const double *gen_pmin, *gen_pmax, *gen_qmin, *gen_qmax; /* [ngen] pu, Eq. 4a-4b      */
} ucac_network;

/* Horizon and demand P_{t,i}, Q_{t,i}. */
typedef struct {
    int32_t T;
    const double *pd, *qd;                                  /* [T*nbus] period-major      */
} ucac_horizon;

/* f^OPF = c2 (S p)^2 + c1 S p; f^UC = c0 u^on + C^SU u^su + C^SD u^sd (R13). */
typedef struct {
    const double *c2, *c1, *c0, *startup, *shutdown;        /* [ngen]                     */
} ucac_costs;

/* UC data: ramps (Eq. 4c-4d), min up/down (Eq. 3d-3e) and the
 * initial state x_0: u0, hold = L_g if u0 = 1 else F_g (Eq. 3a-3b), p0 = p_{0,g}. */
typedef struct {
    const double *ramp_up, *ramp_dn, *su_ramp, *sd_ramp;    /* [ngen] pu / period         */
    const int32_t *min_up, *min_dn;                         /* [ngen] in [1, T] (R15)     */
    const int32_t *u0, *hold;                               /* [ngen]                     */
    const double *p0;                                       /* [ngen] pu                  */
    const int8_t *u_init;   /* [ngen*T] initial schedule or NULL = continue u0 (R23)       */
} ucac_uc;

/* ADMM parameters: rho per class; tau, theta; beta0, bounds and the inner
 * test (R20-R22); branch solver constants (R9, R10). */
typedef struct {
    double rho_pq, rho_va, rho_uc;
    double beta0, tau, theta, lambda_max, beta_max;
    double eps_inner_abs;
    int32_t inner_min, inner_cap, outer_enabled;
    double tron_gtol_rel;
    int32_t tron_maxit, al_maxit;
    double al_eta_star, al_sigma0_rel, al_sigma_max_rel, al_sigma_decay;
    int32_t uc_fixed;   /* 1: step (7a) keeps the schedule (NEXT-2 warm start, ucac_uc_warm_start) */
    int32_t variant;    /* NEXT-3 formulation variants (bitmask, R47): 1 = every rated branch
                           solves the six-variable thermal AL (no 4-variable fast path, as ExaTron),
                           2 = wbar clipped to [Vmin^2, Vmax^2] after the bus solve (SPEC),
                           4 = ramp-aware DP (NEXT-4(a), R50): no shutdown at t while the current
                           dispatch p_{t-1} (p0 at t = 1) exceeds the shutdown ramp S^D,
                           8 = no angle consensus rows (SPEC, R51): each line keeps theta_i = 0 and
                           its own angle difference; thetabar is not updated,
                           16 = the literal Eq. 5f ramp-down row R_D ubar^on_{t-1} + S_D ubar^su_t
                           (R52) instead of Eq. 4d's R_D ubar^on_t + S_D ubar^sd_t */
    int32_t strict_fp;  /* 1 = strict parity mode: the branch solves run the plain
                           oracle algorithm (k_strict.cu) and every quotient is the IEEE quotient, no
                           FMA contraction, sin/cos by the explicit polynomial of R54 -- the iterate
                           then equals the CPU oracle's bit for bit (up to the order of the S8 sums,
                           which feed only the inner/outer decisions).  Slower; for parity runs. */
    int32_t diverge_window;  /* divergence detector ("primal residual grows 10x over 200
                                inner iterations -> abort with diagnostics"): 0 = off; in [1, 255] an
                                ucac_iterate call stops (as at stop_on_primal) at the first iteration i
                                with primal_inf_i > diverge_factor * primal_inf_{i - diverge_window},
                                once per run; ucac_report.diverged_iter names it.  The next call
                                continues.  EINVAL outside [0, 255]. */
    double diverge_factor;   /* (SPEC: window 200, factor 10) */
} ucac_params;

/* Multi-GPU (bus-graph cut).  NULL = single GPU.
 * Bus i belongs to rank bus_part[i]; generators follow their bus, branch (i -> j) follows bus
 * i.  Every rank passes the SAME global problem and builds its local part with a halo: each
 * inner iteration exchanges the cut ends' bus targets (4 doubles per cut branch-period) and
 * the to-bus results back (6 per export bus-period), plus a 12-double reduction record
 * (all-gather / all-reduce, NCCL over NVLink, captured in the iteration graph).
 * comm_mode 0: one process per GPU, NCCL communicator from nccl_id (ucac_nccl_unique_id on rank
 * 0, broadcast by the caller); the caller selects the device before create.
 * comm_mode 1: in-process loopback group of nranks contexts on one device, iterated together
 * with ucac_iterate_group (bitwise the single-GPU iteration; for tests and one-GPU runs). */
typedef struct {
    int32_t rank, nranks, comm_mode;
    unsigned char nccl_id[128];     /* ncclUniqueId (comm_mode 0)                          */
    const int32_t *bus_part;        /* [nbus] owner rank, or NULL = ucac_partition(bus_xy)  */
    const double *bus_xy;           /* [nbus*2] bus coordinates for the partitioner, or NULL */
    const double *branch_w;         /* [nbranch] partition weights (ucac_partition), or NULL = 1  */
    int32_t cut;                    /* 0 = bus-graph cut (above); 1 = time cut (NEXT-4(c), SURVEY
                                       8(f) row 4; P:166-167 temporal decomposition): rank r owns the
                                       periods [r T / n, (r+1) T / n) of every component, keeps one
                                       halo period on each side, all-gathers the DP stage costs
                                       (4 doubles per (g,t)) for a full-horizon DP on every rank, and
                                       exchanges with its neighbours the ramp rows' period-boundary
                                       values (2 doubles per generator forward after (7b), 12 back
                                       after (7c)/(7d)); bus_part / bus_xy are ignored.  Requires
                                       T >= nranks; variant bits 4 and 16 are EUNSUPPORTED. */
} ucac_dist;

/* Deterministic bus-graph cut: weighted recursive coordinate bisection on bus_xy, or weighted
 * BFS-order chunks when bus_xy is NULL, then a greedy boundary refinement with Fiduccia-Mattheyses
 * gains (a bus moves to a neighbouring part when that cuts fewer branches and both parts stay
 * within 5 % of the mean weight; index order, deterministic).  Bus weight = 1 + the weights of its
 * owned branches (branch_w[nbranch], NULL = 1 each: the branch solves dominate; pass the expected
 * per-branch solve work, e.g. 1 + its thermal-AL share, to balance the AL tail).  part[nbus]
 * receives ranks in [0, nparts).  Host only (no device needed). */
ucac_status ucac_partition(int32_t nbus, int32_t nbranch, const int32_t *br_from, const int32_t *br_to,
                           const double *bus_xy, int32_t nparts, int32_t *part, const double *branch_w);
/* Halo of rank `rank` under `part` (host only): sizes[6] = owned buses, ghost buses, local
 * branches, phantom branches (remote branches whose to-bus is owned), cut branches (local
 * branches with a remote to-bus), export buses (owned to-buses of phantoms); the lists (global
 * ids, ascending; any may be NULL) are caller-allocated with those sizes. */
ucac_status ucac_halo_lists(int32_t nbus, int32_t nbranch, const int32_t *br_from, const int32_t *br_to,
                            const int32_t *part, int32_t nparts, int32_t rank, int32_t *sizes,
                            int32_t *own_bus, int32_t *ghost_bus, int32_t *local_branch, int32_t *phantom,
                            int32_t *cut_branch, int32_t *export_bus);
ucac_status ucac_nccl_unique_id(unsigned char *id /* [128] */);
/* Period split of the time cut (ucac_dist.cut = 1, NEXT-4(c)), host only: rank owns the global
 * periods [rank T / n, (rank + 1) T / n); out[4] = (global period of local period 0, first owned
 * local period, end of the owned local periods, local periods incl. one halo period on each side
 * that is not the horizon's end).  EINVAL unless 1 <= nranks <= T and 0 <= rank < nranks. */
ucac_status ucac_time_split(int32_t T, int32_t nranks, int32_t rank, int32_t *out);
/* The context's communicator: ncclCommCount / ncclCommUserRank for an NCCL context (comm_mode 0),
 * else the ucac_dist ranks (1 / 0 for a single-GPU context). */
ucac_status ucac_comm_info(ucac_ctx *ctx, int32_t *nranks, int32_t *rank);
/* 1 if the context iterates through an NCCL communicator (comm_mode 0 with several ranks, or one
 * rank under UCAC_NCCL_ONE_RANK=1 -- the multi-rank graph and its captured collectives on a one-GPU
 * box, for tests), else 0; -1 for a NULL context. */
int32_t ucac_comm_nccl(const ucac_ctx *ctx);

/* Device-initiated exchange of the time cut (NEXT-4(c)): the three exchanges of
 * each iteration (stage costs to every rank, the boundary values to the neighbours) become stores
 * by the sender's blocks into the receivers' buffers in peer memory, published by a system-scope
 * release of the iteration's epoch in the receivers' flags; the receivers spin on acquire loads.
 * Only the S8 all-reduce stays on NCCL.  Ranks of at most 8 (one NVSwitch node).
 * ucac_p2p_export: this context's blob (UCAC_P2P_BLOB bytes: a CUDA IPC handle of its receive
 * buffers + offsets); the caller all-gathers the blobs of the ranks (rank order) and passes them to
 * ucac_p2p_import on every rank, which maps the peers (cudaIpcOpenMemHandle) and re-captures the
 * iteration graph.  ucac_p2p_group: the same for a comm_mode-1 loopback group on one device, where
 * every exchange is one cooperative launch over all ranks' blocks (co-resident, so their waits
 * cannot deadlock).  EUNSUPPORTED unless time cut. */
#define UCAC_P2P_BLOB 96
ucac_status ucac_p2p_export(ucac_ctx *ctx, unsigned char *blob);
ucac_status ucac_p2p_import(ucac_ctx *ctx, const unsigned char *blobs /* [nranks * UCAC_P2P_BLOB] */);
ucac_status ucac_p2p_group(ucac_ctx **ctxs, int32_t n);

/* Create a context: validate (EINVAL with a message: non-finite data, vmin <= 0 or
 * vmin > vmax, pmin > pmax, qmin > qmax, c2 < 0, min_up/min_dn outside [1,T], hold outside
 * [0,T], from == to, bus without branch, bad indices, rho <= 0), lay the data out on the
 * device, and run the cold start of P:459 (R23).  cuda_stream: a cudaStream_t to run on,
 * or NULL for a context-owned stream.  On failure *out = NULL. */
ucac_status ucac_create(const ucac_network *net, const ucac_horizon *hz, const ucac_costs *cost,
                        const ucac_uc *uc, const ucac_params *prm, const ucac_dist *dist,
                        void *cuda_stream, ucac_ctx **out);

/* Run n inner iterations (each = steps 7a-7f + residuals + the outer update when the inner
 * test fires), asynchronously on the context stream.  If stop_on_primal > 0 the loop stops on
 * the device after the first iteration whose primal infeasibility ||Ax+Bxbar||_inf
 * is <= primal_target; *n_done (if not NULL) then receives the number run (synchronises).
 * Hitting n is not an error.  ENUMERIC when an iterate became non-finite. */
ucac_status ucac_iterate(ucac_ctx *ctx, int32_t n, int32_t stop_on_primal, double primal_target,
                         int32_t *n_done);

/* NEXT-4(b) adaptive rho ("future work", R53): replace the three penalty classes
 * rho_pq, rho_va, rho_uc between iterations.  Synchronises the context stream, updates
 * every rho-derived constant (1/rho, the TRON tolerance gtol_rel * max(rho_pq, rho_va), the AL's
 * sigma_0) and re-instantiates the iteration graphs (~2 ms).  The iterate (x, xbar, z, y,
 * lambda, beta) is kept as is.  EINVAL for a non-positive or non-finite rho. */
ucac_status ucac_set_rho(ucac_ctx *ctx, double rho_pq, double rho_va, double rho_uc);

/* n inner iterations of a comm_mode-1 loopback group: ctxs[r] is rank r of nranks = n contexts
 * of one problem on the current device.  Synchronous. */
ucac_status ucac_iterate_group(ucac_ctx **ctxs, int32_t n, int32_t iters);

/* Global ids of the context's local components (which: 0 generators, 1 branches, 2 owned
 * buses), ascending; ids may be NULL to query *count.  The state/solution arrays of a
 * multi-rank context are laid out over exactly these components.  which = 3: the local periods,
 * ids[4] = (global index of local period 0, first owned local period, end of the owned local
 * periods, local periods); the state/solution arrays hold every local period (a time-cut rank's
 * halo periods included), a rank's own values are those of its owned periods. */
ucac_status ucac_local_map(ucac_ctx *ctx, int32_t which, int32_t *ids, int32_t *count);

/* Same iterations launched kernel by kernel with a CUDA event pair around every launch;
 * kernel_ms[k] receives the summed device time of kernel k (order: ucac_kernel_name(k)),
 * launches[k] the number of launches.  Used by the benchmark for per-kernel rooflines. */
#define UCAC_NKERNELS 10
ucac_status ucac_iterate_timed(ucac_ctx *ctx, int32_t n, double *kernel_ms, int64_t *launches);
const char *ucac_kernel_name(int32_t k);

/* Status after the last iteration (synchronises the stream). */
typedef struct {
    double primal_inf, rz_inf, rz_2, z_inf, z_2, dual_inf, objective, beta;
    int64_t inner_total, outer_total, tron_iters, tron_capped, al_active, al_capped;
    int64_t al_tron_iters;            /* TRON iterations inside thermal-AL solves (part of tron_iters) */
    int32_t inner_since_outer, outer_k;
    int32_t err_kernel, err_iter;     /* first non-finite: kernel id + 1 (0 = none), iteration */
    int32_t err_comp, err_period;     /* ... and where: the component (global generator, branch or
                                         bus index, by the kernel's kind) and the period (0-based) */
    int32_t diverged_iter;            /* first iteration the divergence detector fired (0 = never) */
    int32_t hist_len;                 /* records in ucac_history (min(inner_total, UCAC_HIST_CAP)) */
} ucac_report;
ucac_status ucac_residuals(ucac_ctx *ctx, ucac_report *rep);

/* Per-iteration record history ("||z|| history"): the device keeps the last
 * UCAC_HIST_CAP inner iterations' (primal_inf, dual_inf, z_inf, z_2, objective, beta), written by
 * the iteration's final fold.  out (host) receives the last min(n, hist_len) records, oldest first,
 * UCAC_HIST_FIELDS doubles each; *got their number.  ucac_set_state empties it. */
#define UCAC_HIST_CAP 256
#define UCAC_HIST_FIELDS 6
ucac_status ucac_history(ucac_ctx *ctx, double *out, int32_t n, int32_t *got);

/* Solution (host buffers): u_on [ngen*T]; p, q [ngen*T]; wbar, thetabar [nbus*T];
 * flows [nbranch*T*4] = (p_ij, q_ij, p_ji, q_ji) of the branch x-side. */
typedef struct {
    int8_t *u_on;
    double *p, *q, *wbar, *thetabar, *flows;
} ucac_solution;
ucac_status ucac_get_solution(ucac_ctx *ctx, ucac_solution *sol);

/* Full iterate in the canonical layout of DESIGN.md 4 (host buffers, sizes in brackets;
 * GT = ngen*T, LT = nbranch*T, BT = nbus*T).  Row kinds per (g,t): D_ON D_SU D_SD PL PU QL
 * QU RD RU GP GQ RC; per (l,t): FP_IJ FQ_IJ FP_JI FQ_JI W_I W_J A_I A_J; row arrays are
 * [kind][comp*T + t].  x and f are [LT][4] (w_i w_j th_i th_j / p_ij q_ij p_ji q_ji),
 * fbar [LT][4], al [LT][3] = (mu_ij, mu_ji, sigma) of the thermal AL.
 * scal[8] = beta, ||z||_prev, outer k, inner total, inner since outer, 0, 0, 0.
 * Used for checkpoint/resume and for iteration-by-iteration parity with the oracle. */
typedef struct {
    int8_t *u;                                               /* [GT]        */
    double *p, *q, *ph, *ub_on, *ub_su, *ub_sd, *pbar, *qbar; /* [GT]        */
    double *zg, *yg, *lg;                                    /* [12*GT]     */
    double *x, *f, *fbar;                                    /* [4*LT]      */
    double *al;                                              /* [3*LT]      */
    double *zb, *yb, *lb;                                    /* [8*LT]      */
    double *wbar, *thbar;                                    /* [BT]        */
    double *scal;                                            /* [8]         */
} ucac_state;
ucac_status ucac_get_state(ucac_ctx *ctx, ucac_state *st);
ucac_status ucac_set_state(ucac_ctx *ctx, const ucac_state *st);

/* NEXT-2 UC warm start (R46): solve the multiperiod
 * ACOPF with every unit on after its held prefix and the schedule held (uc_fixed = 1) for
 * `iters` inner iterations, then u_out[g*T+t] = the nearest schedule satisfying Eq. 3 (one DP
 * pass, stage cost = Hamming distance to [p > threshold], threshold in pu, e.g. 1e-3).  Pass
 * u_out as ucac_uc.u_init of the UC-ACOPF context.  Single GPU; host buffers; synchronous. */
ucac_status ucac_uc_warm_start(const ucac_network *net, const ucac_horizon *hz, const ucac_costs *cost,
                               const ucac_uc *uc, const ucac_params *prm, int32_t iters, double threshold,
                               int8_t *u_out);

/* Batched UC DP (Alg. 2) on caller stage costs: L [ngen*T*4] with L[(g*T+t)*4 + a*2 + b] =
 * L^UC_{g,t}(a, b).  Outputs sched [ngen*T] (int8) and cost [ngen].  Tie -> stay
 * (P:380), windows clipped at T (R15), forced prefix of hold periods (R14).  When on_device
 * != 0 all five array arguments are device pointers and the call runs asynchronously on
 * cuda_stream (NULL = legacy default stream); otherwise they are host pointers.  Host inputs are
 * validated (min_up, min_dn in [1, T], hold in [0, T], u0 in {0, 1}; else UCAC_EINVAL); device
 * inputs cannot be checked without a sync, so an out-of-range instance gets cost NaN and an
 * all-zero schedule from the kernel (no out-of-range access). */
ucac_status ucac_dp_batch(int32_t ngen, int32_t T, const double *L, const int32_t *min_up,
                          const int32_t *min_dn, const int32_t *u0, const int32_t *hold,
                          int8_t *sched, double *cost, int32_t on_device, void *cuda_stream);

/* Bytes moved and sizes, for the benchmark's roofline arithmetic. */
typedef struct {
    int64_t nrows, gen_periods, branch_periods, bus_periods;
    int64_t alg_bytes_per_iter;         /* algorithmic HBM bytes of one inner iteration   */
    int64_t alg_bytes[UCAC_NKERNELS];   /* per kernel                                     */
} ucac_sizes;
ucac_status ucac_get_sizes(ucac_ctx *ctx, ucac_sizes *sz);

/* Fault injection for the non-finite path: overwrite one element of a row-state
 * array with NaN, between iterations.  field: 0 = branch-row z, 1 = branch-row y, 2 = generator-row
 * z, 3 = generator-row y; index in the canonical [kind][comp*T + t] layout of ucac_state (local
 * components on a multi-rank context).  The next ucac_iterate then returns UCAC_ENUMERIC and
 * ucac_residuals names the first kernel that met the value (err_kernel, err_comp, err_period,
 * err_iter).  EINVAL for a bad field or index.  Synchronous.  Test use only. */
ucac_status ucac_debug_poison(ucac_ctx *ctx, int32_t field, int64_t index);

/* Measured FP64 (non-tensor) pipe peak of the current device, the denominator of the branch
 * kernels' roofline: a DFMA-chain microbenchmark (8 independent fma chains per
 * thread, 8 x 256-thread blocks per SM, best of 5 timed launches of 64 x iters DFMA per thread).
 * *tflops = 2 flop x DFMA count / time; *ms (may be NULL) the best launch time. */
ucac_status ucac_measure_fp64_peak(int32_t iters, double *tflops, double *ms);
/* Dependent-chain latencies of the current device in SM cycles per link, one warp, clock64:
 * cycles[0] DFMA, [1] DADD, [2] a double __shfl_xor_sync + add (one warp-reduction step), [3] the
 * branch kernels' reciprocal (rcp.approx.f64 + two Newton steps), [4] IEEE sqrt.  Diagnostics
 * (why one lane per small solve). */
ucac_status ucac_measure_latencies(double *cycles);

void *ucac_stream(ucac_ctx *ctx);                 /* the cudaStream_t the context runs on */
const char *ucac_last_error(const ucac_ctx *ctx); /* NULL ctx: last create failure (thread-local) */
/* Waits for the context's stream, frees its device memory and destroys it.  Its side streams,
 * fork/join events and instantiated single-iteration graph are kept (process lifetime, per device)
 * for the next ucac_create, which loads its own graph into the kept one (cudaGraphExecUpdate) --
 * so no cudaDeviceReset between contexts.  NULL: no-op. */
void ucac_destroy(ucac_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif
