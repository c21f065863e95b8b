// ucac_dev.cuh -- device-side layout of the UC-ACOPF ADMM hot path (B200, sm_100a, fp64).
//
// Everything the kernels touch lives in one POD `Dev` passed by value to every kernel.
// Layout: component-major, period-minor SoA; row state is [kind][comp*T + t]
// so that a warp whose lanes are consecutive periods of one component (or consecutive
// (component, period) pairs) reads each row kind as one coalesced 256-B segment.
#pragma once
#ifndef UCAC_PDL_DEFAULT
#define UCAC_PDL_DEFAULT 1   // k_branch_al after k_branch (measured)
#endif
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef UCAC_AL_BUCKETS
#define UCAC_AL_BUCKETS 1   // AL queue buckets by the previous AL Newton count (heavy / new first); 2 and
                            // 3 measured neutral (0.1664-0.1672 ms vs 0.1666-0.1669), DESIGN.md 7
#endif
#ifndef UCAC_MAX_P2P
#define UCAC_MAX_P2P 8   // ranks of a device-initiated exchange group (one node: 8 GPUs on NVSwitch)
#endif

namespace ucac {

// coupling-row kinds (Eq. 5; R3 ramp-down in the Eq. 4d form, R6 ramp copy,
// R7 angle consensus)
enum GenRow { G_DON = 0, G_DSU, G_DSD, G_PL, G_PU, G_QL, G_QU, G_RD, G_RU, G_GP, G_GQ, G_RC, NGROW };
enum BrRow { B_FPIJ = 0, B_FQIJ, B_FPJI, B_FQJI, B_WI, B_WJ, B_AI, B_AJ, NBROW };

// kernel ids (ucac_kernel_name)
enum KernelId { K_BRANCH = 0, K_GEN = 1, K_BUS = 2, K_UBAR = 3, K_BUS_LATE = 4, K_BRANCH_AL = 5, K_ROWS = 6,
                K_GENX = 7, K_ROWS_LATE = 8, K_FOLD = 9, NKERN = 10 };

// per-block reduction record (S8): max |r|, max |r+z|, sum (r+z)^2, max |z|, sum z^2,
// max rho |dxbar|, objective, non-finite flag
enum Part { P_PINF = 0, P_RZINF, P_RZ2, P_ZINF, P_Z2, P_DINF, P_OBJ, P_BAD, NPART };
// cross-rank reduction record: 7 sums (RZ2, Z2, OBJ, 4 TRON counters) then 5 maxes
enum Rec { R_RZ2 = 0, R_Z2, R_OBJ, R_C0, R_C1, R_C2, R_C3, R_C4, NREC_SUM, R_PINF = NREC_SUM, R_RZINF, R_ZINF, R_DINF, R_BAD,
           NREC };
constexpr int NCNT = 5;   // TRON iterations, TRON caps, AL solves, AL caps, TRON iterations inside the AL

struct DevStatus {
    double beta;          // current beta^k
    double beta_lam;      // beta used by the pending lambda update
    double znorm_prev;    // ||z||_2 at the previous outer update
    long long outer_k;    // k (starts at 1)
    long long inner_total;
    long long inner_since;
    int pending_outer;    // lambda <- clip(lambda + beta_lam z) to apply at the next sweep
    int done;             // stop_on_primal reached: kernels return immediately
    int stop_on_primal;
    int err_kernel, err_iter;         // first non-finite value: kernel id + 1, iteration (1-based)
    int err_comp, err_period;         // ... its component (rank-local index) and period
    int diverged_iter;                // divergence detector: first iteration it fired
    double primal_target;
    double primal_inf, rz_inf, rz_2, z_inf, z_2, dual_inf, objective;
    unsigned long long tron_iters, tron_capped, al_active, al_capped, al_tron_iters;
};

// per-iteration records (ucac_history): primal_inf, dual_inf, z_inf, z_2, objective, beta
constexpr int HIST_CAP = 256, HIST_FIELDS = 6;

struct Dev {
    int G, L, B, T;
    int ref_bus;
    int nblk_bus, nblk_ubar, nblk_rows;
    double S;                         // base MVA
    double rpq, rva, ruc;             // rho classes
    double irpq, irva, iruc;          // 1/rho: every kernel forms y/rho as y * (1/rho)
    double tau, theta, lambda_max, beta_max, eps_inner_abs;
    int inner_min, inner_cap, outer_enabled;
    double tron_gtol;                 // absolute: tron_gtol_rel * max(rho_pq, rho_va)
    int tron_maxit, al_maxit;
    double al_eta_star, al_sigma0_rel, al_sigma_max_rel, al_sigma_decay;
    int uc_fixed;                     // 1: k_gen keeps u (NEXT-2)
    int div_window;                   // divergence detector (0 = off)
    double div_factor;
    double *hist;                     // [HIST_CAP][HIST_FIELDS], slot (iteration - 1) % HIST_CAP
    int variant;                      // NEXT-3 bitmask: 1 = AL for every rated branch, 2 = wbar clip
    int strict;                       // strict_fp parity mode: oracle quotients / operation order (k_strict.cu)
    // ---- periods (NEXT-4(c) time cut): local period t is global period t + t_off of Tg; the kernels
    // update the owned periods [own0, own1) only (single GPU / bus cut: 0, T, T, 0)
    int t_off, Tg, own0, own1;
    int tcut, Tmax, rank;                   // time cut on; longest owned range of any rank
    const int *tc_t0;                 // [nranks + 1] owned global period ranges of the ranks
    double *tc_stage_send, *tc_stage_recv;   // [G][Tmax][4], [nranks][G][Tmax][4]: DP stage costs
    double *tc2_send, *tc2_recv;             // [G][2], [nranks][G][2]: p, phat of the first owned period
    double *tc3_send, *tc3_recv;             // [G][12], [nranks][G][12]: the boundary values sent forward
    // device-initiated exchange of the time cut (NEXT-4(c), k_xchg.cu): the other ranks' receive
    // buffers and arrival flags (peer memory: CUDA IPC across GPUs, plain pointers in a loopback group)
    int p2p;                                  // 1: the three exchanges by k_xchg instead of NCCL
    double *peer_stage_recv[UCAC_MAX_P2P], *peer_tc2_recv[UCAC_MAX_P2P], *peer_tc3_recv[UCAC_MAX_P2P];
    unsigned long long *peer_flags[UCAC_MAX_P2P];   // rank q's flags [3 phases][UCAC_MAX_P2P sources]
    unsigned long long *xflags;               // mine, written by the senders
    unsigned *xarrive;                        // [3] blocks of this rank done sending (last one signals)

    // ---- static generator data [G]
    const int *gbus, *tu, *td, *u0, *hold;
    const double *pmin, *pmax, *qmin, *qmax, *c2, *c1, *c0, *csu, *csd;
    const double *rup, *rdn, *sup, *sdn, *p0;
    // ---- static branch data
    const double *y;                  // [8][L] SoA: Gii Gij Gji Gjj Bii Bij Bji Bjj
    const double *rate;               // [L]
    const int *bfrom, *bto;           // [L]
    // ---- static bus data
    const double *gs, *bs, *vmin, *vmax;  // [B]
    const double *pd, *qd;            // [B][T]
    const int *bg_ptr, *bg_idx;       // CSR bus -> generators (index order)
    const int *be_ptr, *be_idx;       // CSR bus -> branch ends (2*l + side), (l, side) order

    // ---- iterate
    int8_t *u;                        // [G*T]
    double *p, *q, *ph;               // [G*T]
    double *ub_on, *ub_su, *ub_sd;    // [G*T]
    double *pbar, *qbar;              // [G*T]
    double *zg, *yg, *lg;             // [12][G*T]
    double *x;                        // [4][L*T]  w_i w_j th_i th_j
    double *f;                        // [4][L*T]  p_ij q_ij p_ji q_ji
    double *fbar;                     // [4][L*T]
    double *al;                       // [3][L*T]  mu_ij mu_ji sigma
    double *zb, *yb, *lb;             // [8][L*T]
    double *wbar, *thbar;             // [B*T]

    // ---- reduction scratch
    double *part_bus;                 // [nblk_bus][NPART]
    double *part_ubar;                // [nblk_ubar][NPART]
    unsigned long long *cnt;          // [NCNT] per-iteration solver counters (zeroed by the final fold)
    // ---- multi-rank; single GPU: B_own = B, Lph = 0, nothing to exchange
    int B_own;                        // owned buses [0, B_own); ghosts [B_own, B)
    int Lph;                          // phantom branches [L, L + Lph) (tauhat only)
    int ncut, nexport, nphantom_src, nghost, max_cut, max_export, nranks;
    int xrank_rec;                    // 1: the final fold leaves the S8 record to a cross-rank all-reduce
    const int *cut_local, *export_local, *phantom_src, *ghost_src;
    double *xsend1, *xrecv1, *xsend2, *xrecv2;   // halo exchange buffers: early tauhat + late flag (5 per
                                                 // cut branch-period), early bus results + late flag (7)
    double *xsend3, *xrecv3, *xsend4, *xrecv4;   // late tauhat (4), late bus results (6)
    const int *phantom_bus;           // [Lp] owned local bus of each phantom branch's to-end
    const int *ghost_eptr, *ghost_eidx;   // CSR ghost bus -> local branch end codes at it
    unsigned *qmark;                  // [(L + Lp) T] = stamp: the (l,t) went to the AL queue (local, or remote for a phantom)
    double *rec;                      // [NREC] local reduction record (sums then maxes)
    double *tauh;                     // [8][(L+Lph)*T] bus-side targets x + z + y/rho of the branch rows
    double *bmu;                      // [4][B*T] muP, muQ, wbar - wbar_old, thbar - thbar_old
    double *part_rows;                // [nblk_rows][NPART]
    int *alq;                         // [L*T] queue of thermal-active solves (phase 2)
    unsigned *bmark;                  // [B*T] = stamp(iteration) if an incident (l,t) is queued:
                                      // its bus solve waits for the AL tail (k_bus_late)
    unsigned *rmark[2];               // [(L+Lph)*T] per side: = stamp if that end's bus is marked
    int nblk_lbus, nblk_lrows;        // late-phase grids (one wave over the compacted lists)
    int *lbus;                        // [nblk_bus][BUS_THREADS]: marked bus-periods, per k_bus block
    unsigned *lbus_cnt;               // [nblk_bus] their counts
    int *lrow;                        // [nblk_rows][2 ROWS_THREADS]: marked ends (k << 1 | side), per k_rows block
    unsigned *lrow_cnt;               // [nblk_rows]
    double *part_lbus, *part_lrows;   // their block partials
    double *part_efold;               // [fold_blocks()][NPART] first-level fold of the early partials
    double *rec_part;                 // [3][NPART] folded records: early, bus late, rows late
    unsigned *kdone;                  // [3] last-block counters of the kernels producing them
    unsigned *alq_cnt;                // [UCAC_AL_BUCKETS + 1] bucket lengths, next item (zeroed by the final fold)
    double *alq_x;                    // [4][L*T] by (l,t): the previous x of a queued solve (R49)
    uint8_t *alits;                   // [L*T] TRON iterations of the (l,t)'s last AL solve (0: none last iteration)
    int fuse_rows;                    // 1 GPU: the end rows of a bus are updated by its bus thread (no k_rows)
    int8_t *u_next;                   // [G*T] the DP's schedule for the next (7b): written by k_gen, adopted by k_genx
    unsigned *unext_ok;               // 1: u_next holds the DP of the current state (set by the tail k_gen)
    DevStatus *st;
    unsigned long long *tl;           // [2*NKERN] diagnostic timeline (UCAC_PROF builds only)
};

// UCAC_PROF builds: per kernel, the earliest block start and the latest warp exit (lane 0 of every
// warp: a block's warps can outlive its thread 0, as the AL solves do) on the global timer (ns),
// for graph timelines (tools/timeline.py).  Empty otherwise.
#ifdef UCAC_PROF
struct TlGuard {
    unsigned long long *p;
    __device__ TlGuard(unsigned long long *tl, int kid) : p(tl + 2 * kid) {
        if (threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            atomicMin(p, t);
        }
    }
    __device__ ~TlGuard() {
        if ((threadIdx.x & 31) == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            atomicMax(p + 1, t);
        }
    }
};
#define TL_KERNEL(kid) TlGuard tl_guard_(d.tl, (kid))
#else
#define TL_KERNEL(kid) \
    do {               \
    } while (0)
#endif

__host__ __device__ inline size_t gi(const Dev &d, int g, int t) { return (size_t)g * d.T + t; }
// owned local period / its global index (time cut, NEXT-4(c)); trivially true / t otherwise
__device__ __forceinline__ bool own_t(const Dev &d, int t) { return t >= d.own0 && t < d.own1; }
__device__ __forceinline__ int tglob(const Dev &d, int t) { return t + d.t_off; }

// SPEC S:322 non-finite handling: the first kernel that meets a NaN/inf records (kernel,
// component, period, iteration); ucac_iterate / ucac_residuals then return UCAC_ENUMERIC
__device__ __forceinline__ void report_nonfinite(const Dev &d, int kid, int comp, int t) {
    if (atomicCAS(&d.st->err_kernel, 0, kid + 1) == 0) {
        d.st->err_comp = comp;
        d.st->err_period = t;
        d.st->err_iter = (int)d.st->inner_total + 1;
    }
}
// 0 for finite v, NaN otherwise: sums of these flag a non-finite operand
__device__ __forceinline__ double nf0(double v) { return v * 0.0; }
// per-iteration stamp of bmark (read before k_reduce advances inner_total; never 0)
__device__ __forceinline__ unsigned mark_stamp(const Dev &d) { return (unsigned)(d.st->inner_total + 1); }

}  // namespace ucac

// launch wrappers (one per translation unit)
namespace ucac {
void launch_branch(const Dev &d, cudaStream_t s);
void launch_branch_al(const Dev &d, cudaStream_t s);
void launch_branch_strict(const Dev &d, cudaStream_t s);
// time cut (NEXT-4(c)): DP stage costs of the owned periods, the full-horizon DP, boundary exchange
void launch_stage_tc(const Dev &d, cudaStream_t s);
void launch_dp_tc(const Dev &d, cudaStream_t s);
void launch_pack_tc2(const Dev &d, cudaStream_t s);
void launch_unpack_tc2(const Dev &d, cudaStream_t s);
void launch_pack_tc3(const Dev &d, cudaStream_t s);
void launch_unpack_tc3(const Dev &d, cudaStream_t s);
// device-initiated exchange (k_xchg.cu): phase 1 stage costs to every rank, 2 p/phat to the
// previous rank, 3 the boundary values to the next rank; each sends, signals, then waits for its sources
void launch_xchg(const Dev &d, int phase, cudaStream_t s);
cudaError_t launch_xchg_group(const Dev *devs_host, int n, int phase, cudaStream_t s, Dev *scratch);
// Launch with the device's highest execution priority (a launch attribute, kept by graph capture):
// the generator chain (k_gen, k_genx, k_ubar) forks at the start of the iteration and should take
// SM slots as k_branch blocks retire rather than queue behind them.
// Programmatic dependent launch (PDL) of the critical chain's kernels, bit mask from UCAC_PDL
// (1 = k_branch_al after k_branch, 2 = k_bus_late after k_branch_al, 4 = k_rows_late after
// k_bus_late, 8 = k_branch after the previous iteration's last kernel): the dependent grid is scheduled as the primary's blocks exit and waits in
// griddepcontrol.wait (pdl_wait, first statement of those kernels; a no-op without the attribute)
// until the primary grid has completed and its memory is visible.  Experiments.
inline int pdl_mask() {
    static const int m = [] { const char *e = getenv("UCAC_PDL"); return e ? atoi(e) : UCAC_PDL_DEFAULT; }();
    return m;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
template <typename... KArgs>
inline cudaError_t launch_ex(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool hi,
                             bool pdl, KArgs... args) {
    static int prio = [] { int lo = 0, hi_ = 0; cudaDeviceGetStreamPriorityRange(&lo, &hi_); return hi_; }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int n = 0;
    if (hi) {
        at[n].id = cudaLaunchAttributePriority;
        at[n++].val.priority = prio;
    }
    if (pdl) {
        at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[n++].val.programmaticStreamSerializationAllowed = 1;
    }
    cfg.attrs = at;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, k, args...);
}
template <typename... KArgs>
inline cudaError_t launch_hi_prio(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, KArgs... args) {
    static int prio = [] { int lo = 0, hi = 0; cudaDeviceGetStreamPriorityRange(&lo, &hi); return hi; }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributePriority;
    at[0].val.priority = prio;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, args...);
}
void launch_gen(const Dev &d, cudaStream_t s, int tail = 0);
void launch_genx(const Dev &d, cudaStream_t s);
void launch_bus(const Dev &d, cudaStream_t s);
void launch_rows(const Dev &d, cudaStream_t s);
void launch_bus_late(const Dev &d, cudaStream_t s);
void launch_rows_late(const Dev &d, cudaStream_t s, int final);
int nblk_lbus(int n);
int nblk_lrows(int n);
int fold_blocks();
void launch_fold_early(const Dev &d, cudaStream_t s);
int nblk_rows(int L, int T);
// multi-rank
void launch_finalize(const Dev &d, cudaStream_t s);
void launch_pack_tau(const Dev &d, cudaStream_t s);
void launch_pack_tau_early(const Dev &d, cudaStream_t s);
void launch_unpack_tau_early(const Dev &d, cudaStream_t s);
void launch_pack_bus_early(const Dev &d, cudaStream_t s);
void launch_unpack_bus_early(const Dev &d, cudaStream_t s);
void launch_unpack_tau(const Dev &d, cudaStream_t s);
void launch_pack_bus(const Dev &d, cudaStream_t s);
void launch_unpack_bus(const Dev &d, cudaStream_t s);
void launch_ubar(const Dev &d, cudaStream_t s);
void launch_init(const Dev &d, const int8_t *u_init_dev, cudaStream_t s);
void launch_hamming_costs(int n, const double *p, double threshold, double *L, cudaStream_t s);
cudaError_t launch_dp_batch(int G, int T, const double *L, const int *tu, const int *td, const int *u0,
                            const int *hold, int8_t *sched, double *cost, cudaStream_t s);
int nblk_bus(int B, int T);
int nblk_ubar(int G, int T);
}  // namespace ucac
