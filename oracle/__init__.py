"""ctypes wrapper of the plain CPU oracle (oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product path
(paper_2310_13145_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_HDR = os.path.join(_HERE, "oracle.h")
_LIB = os.path.join(_HERE, "_build", "liboracle.so")
_LIB_OMP = os.path.join(_HERE, "_build", "liboracle_omp.so")
_lock = threading.Lock()
_lib = None
_lib_omp = None

CFLAGS = ["-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall",
          "-Wno-unknown-pragmas"]


def build(force: bool = False) -> str:
    """compile liboracle.so with gcc (-O2 -ffp-contract=off, no fast-math, single thread) and the
    all-core twin liboracle_omp.so (the same source with -fopenmp)."""
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    for out, extra in ((_LIB, []), (_LIB_OMP, ["-fopenmp"])):
        stale = force or not os.path.exists(out) or any(
            os.path.getmtime(p) > os.path.getmtime(out) for p in (_SRC, _HDR))
        if stale:
            tmp = out + f".{os.getpid()}.tmp"
            subprocess.check_call(["gcc", *CFLAGS, *extra, "-o", tmp, _SRC, "-lm"])
            os.replace(tmp, out)
    return _LIB


def lib(omp: bool = False):
    """the single-thread oracle, or (omp=True) its all-core OpenMP build"""
    global _lib, _lib_omp
    with _lock:
        if omp:
            if _lib_omp is None:
                build()
                _lib_omp = C.CDLL(_LIB_OMP)
                _declare(_lib_omp)
            return _lib_omp
        if _lib is None:
            _lib = C.CDLL(build())
            _declare(_lib)
    return _lib


def threads(n: int = 0) -> int:
    """threads of the all-core build (n > 0 sets them)"""
    return lib(omp=True).orc_threads(int(n))


dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int32)
i8p = C.POINTER(C.c_int8)
i64p = C.POINTER(C.c_int64)


class Problem_c(C.Structure):
    _fields_ = [("nbus", C.c_int32), ("ngen", C.c_int32), ("nbranch", C.c_int32), ("T", C.c_int32),
                ("ref_bus", C.c_int32), ("base_mva", C.c_double),
                ("bus_gs", dp), ("bus_bs", dp), ("bus_vmin", dp), ("bus_vmax", dp),
                ("pd", dp), ("qd", dp), ("br_from", ip), ("br_to", ip), ("br_y", dp), ("br_rate", dp),
                ("gen_bus", ip), ("pmin", dp), ("pmax", dp), ("qmin", dp), ("qmax", dp),
                ("c2", dp), ("c1", dp), ("c0", dp), ("csu", dp), ("csd", dp),
                ("ramp_up", dp), ("ramp_dn", dp), ("su_ramp", dp), ("sd_ramp", dp),
                ("min_up", ip), ("min_dn", ip), ("u0", ip), ("hold", ip), ("p0", dp), ("u_init", i8p)]


class Params_c(C.Structure):
    _fields_ = [("rho_pq", C.c_double), ("rho_va", C.c_double), ("rho_uc", C.c_double),
                ("beta0", C.c_double), ("tau", C.c_double), ("theta", C.c_double),
                ("lambda_max", C.c_double), ("beta_max", C.c_double), ("eps_inner_abs", C.c_double),
                ("inner_min", C.c_int32), ("inner_cap", C.c_int32), ("outer_enabled", C.c_int32),
                ("tron_gtol_rel", C.c_double), ("tron_maxit", C.c_int32), ("al_maxit", C.c_int32),
                ("al_eta_star", C.c_double), ("al_sigma0_rel", C.c_double), ("al_sigma_max_rel", C.c_double),
                ("al_sigma_decay", C.c_double), ("uc_fixed", C.c_int32), ("variant", C.c_int32),
                ("plain", C.c_int32), ("diverge_window", C.c_int32), ("diverge_factor", C.c_double)]


class Report_c(C.Structure):
    _fields_ = [("primal_inf", C.c_double), ("rz_inf", C.c_double), ("rz_2", C.c_double),
                ("z_inf", C.c_double), ("z_2", C.c_double), ("dual_inf", C.c_double),
                ("objective", C.c_double), ("beta", C.c_double),
                ("inner_total", C.c_int64), ("outer_total", C.c_int64), ("tron_iters", C.c_int64),
                ("tron_capped", C.c_int64), ("al_active", C.c_int64), ("al_capped", C.c_int64),
                ("inner_since_outer", C.c_int32), ("outer_k", C.c_int32),
                ("flops_fast", C.c_double), ("flops_al", C.c_double),
                ("newton_fast", C.c_int64), ("newton_al", C.c_int64),
                ("diverged_iter", C.c_int32), ("pad_", C.c_int32)]


STATE_FIELDS = [("u", np.int8, "GT"), ("p", np.float64, "GT"), ("q", np.float64, "GT"),
                ("ph", np.float64, "GT"), ("ub_on", np.float64, "GT"), ("ub_su", np.float64, "GT"),
                ("ub_sd", np.float64, "GT"), ("pbar", np.float64, "GT"), ("qbar", np.float64, "GT"),
                ("zg", np.float64, "12GT"), ("yg", np.float64, "12GT"), ("lg", np.float64, "12GT"),
                ("x", np.float64, "4LT"), ("f", np.float64, "4LT"), ("fbar", np.float64, "4LT"),
                ("al", np.float64, "3LT"), ("zb", np.float64, "8LT"), ("yb", np.float64, "8LT"),
                ("lb", np.float64, "8LT"), ("wbar", np.float64, "BT"), ("thbar", np.float64, "BT"),
                ("scal", np.float64, "8")]


class State_c(C.Structure):
    _fields_ = [(n, i8p if t == np.int8 else dp) for n, t, _ in STATE_FIELDS]


def _declare(L):
    L.orc_create.argtypes = [C.POINTER(Problem_c), C.POINTER(Params_c), C.POINTER(C.c_void_p)]
    L.orc_create.restype = C.c_int
    L.orc_destroy.argtypes = [C.c_void_p]
    L.orc_iterate.argtypes = [C.c_void_p, C.c_int32]
    L.orc_set_rho.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double]
    L.orc_set_rho.restype = None
    L.orc_report_get.argtypes = [C.c_void_p, C.POINTER(Report_c)]
    L.orc_get_state.argtypes = [C.c_void_p, C.POINTER(State_c)]
    L.orc_set_state.argtypes = [C.c_void_p, C.POINTER(State_c)]
    L.orc_stage_costs.argtypes = [C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double, dp, dp, dp, dp]
    L.orc_dp.argtypes = [C.c_int32, dp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, i8p]
    L.orc_dp.restype = C.c_double
    L.orc_uc_repair.argtypes = [C.c_int32, dp, C.c_double, C.c_int32, C.c_int32, C.c_int32, C.c_int32, i8p]
    L.orc_uc_repair.restype = None
    L.orc_gen_x.argtypes = [dp, dp]
    L.orc_boxqp3.argtypes = [C.c_int32, C.c_int32, dp, dp, dp]
    L.orc_bus_kkt.argtypes = [C.c_int32, dp, dp, dp, dp, C.c_double, C.c_double, dp, dp]
    L.orc_branch_solve.argtypes = [dp, dp, dp, C.c_double, dp, C.c_double, C.c_double,
                                   C.POINTER(Params_c), dp, dp, dp, i64p]
    L.orc_tron_quadratic.argtypes = [C.c_int32, dp, dp, dp, dp, C.c_double, C.c_int32, dp]
    L.orc_tron_quadratic.restype = C.c_int
    L.orc_branch_flows.argtypes = [dp, dp, dp, dp, dp]
    L.orc_sincos.argtypes = [C.c_double, dp, dp]
    L.orc_sincos.restype = None
    L.orc_get_slacks.argtypes = [C.c_void_p, dp]
    L.orc_get_slacks.restype = None
    L.orc_threads.argtypes = [C.c_int32]
    L.orc_threads.restype = C.c_int


def _p(a, t=dp):
    return a.ctypes.data_as(t) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def params_c(pr, plain: bool = False) -> Params_c:
    """plain: the branch solver without the accelerations R41-R44/R48/R49 (oracle-only twin)"""
    return Params_c(pr.rho_pq, pr.rho_va, pr.rho_uc, pr.beta0, pr.tau, pr.theta, pr.lambda_max,
                    pr.beta_max, pr.eps_inner_abs, pr.inner_min, pr.inner_cap, pr.outer_enabled,
                    pr.tron_gtol_rel, pr.tron_maxit, pr.al_maxit, pr.al_eta_star, pr.al_sigma0_rel,
                    pr.al_sigma_max_rel, pr.al_sigma_decay, pr.uc_fixed, pr.variant, int(plain),
                    pr.diverge_window, pr.diverge_factor)


class Oracle:
    """One oracle context (Algorithm 1 run on the CPU)."""

    def __init__(self, pb, pr, plain: bool = False, omp: bool = False):
        """omp: the all-core build (bitwise the same iterates)"""
        self.L = lib(omp)
        pb = pb.normalized()
        self.pb = pb
        self.pr = pr
        self._keep = []

        def k(a, t=dp):
            a = np.ascontiguousarray(a)
            self._keep.append(a)
            return a.ctypes.data_as(t)
        ui = None
        if pb.u_init is not None:
            ui = k(np.ascontiguousarray(pb.u_init, dtype=np.int8).reshape(-1), i8p)
        self._pbc = Problem_c(pb.nbus, pb.ngen, pb.nbranch, pb.T, pb.ref_bus, pb.base_mva,
                              k(pb.bus_gs), k(pb.bus_bs), k(pb.bus_vmin), k(pb.bus_vmax),
                              k(pb.pd.reshape(-1)), k(pb.qd.reshape(-1)), k(pb.br_from, ip), k(pb.br_to, ip),
                              k(pb.br_y.reshape(-1)), k(pb.br_rate), k(pb.gen_bus, ip),
                              k(pb.pmin), k(pb.pmax), k(pb.qmin), k(pb.qmax),
                              k(pb.c2), k(pb.c1), k(pb.c0), k(pb.csu), k(pb.csd),
                              k(pb.ramp_up), k(pb.ramp_dn), k(pb.su_ramp), k(pb.sd_ramp),
                              k(pb.min_up, ip), k(pb.min_dn, ip), k(pb.u0, ip), k(pb.hold, ip), k(pb.p0), ui)
        self._prc = params_c(pr, plain)
        h = C.c_void_p()
        rc = self.L.orc_create(C.byref(self._pbc), C.byref(self._prc), C.byref(h))
        if rc != 0:
            raise ValueError("orc_create rejected the problem")
        self.h = h

    def close(self):
        if self.h:
            self.L.orc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def iterate(self, n: int = 1):
        self.L.orc_iterate(self.h, n)

    def set_rho(self, rho_pq: float, rho_va: float, rho_uc: float):
        """NEXT-4(b), R53: new penalty classes between iterations (the iterate is kept)."""
        self.L.orc_set_rho(self.h, rho_pq, rho_va, rho_uc)

    def report(self) -> dict:
        r = Report_c()
        self.L.orc_report_get(self.h, C.byref(r))
        return {n: getattr(r, n) for n, _ in Report_c._fields_}

    def _sizes(self):
        pb = self.pb
        GT, LT, BT = pb.ngen * pb.T, pb.nbranch * pb.T, pb.nbus * pb.T
        return {"GT": GT, "12GT": 12 * GT, "4LT": 4 * LT, "3LT": 3 * LT, "8LT": 8 * LT, "BT": BT, "8": 8}

    def get_state(self) -> dict:
        sz = self._sizes()
        st = {n: np.zeros(sz[s], dtype=t) for n, t, s in STATE_FIELDS}
        sc = State_c(*[_p(st[n], i8p if t == np.int8 else dp) for n, t, _ in STATE_FIELDS])
        self.L.orc_get_state(self.h, C.byref(sc))
        return st

    def slacks(self) -> np.ndarray:
        """generator slacks of the current x, [ngen*T, 6] (pl, pu, ql, qu, rd, ru)"""
        out = np.zeros(6 * self.pb.ngen * self.pb.T)
        self.L.orc_get_slacks(self.h, _p(out))
        return out.reshape(-1, 6)

    def set_state(self, st: dict):
        sz = self._sizes()
        arrs = {n: np.ascontiguousarray(st[n], dtype=t).reshape(-1) for n, t, _ in STATE_FIELDS}
        for n, t, s in STATE_FIELDS:
            assert arrs[n].size == sz[s], n
        sc = State_c(*[_p(arrs[n], i8p if t == np.int8 else dp) for n, t, _ in STATE_FIELDS])
        self.L.orc_set_state(self.h, C.byref(sc))


# ---- single-step wrappers ----
def stage_costs(T, c0, csu, csd, rho, ub, y, z):
    L = np.zeros(T * 4)
    lib().orc_stage_costs(T, c0, csu, csd, rho, _p(_f64(ub)), _p(_f64(y)), _p(_f64(z)), _p(L))
    return L.reshape(T, 2, 2)


def uc_repair(p, threshold, TU, TD, u0, hold):
    """NEXT-2: [p > threshold] repaired to the nearest Eq. 3 schedule (one DP pass)."""
    p = _f64(p).reshape(-1)
    u = np.zeros(p.size, dtype=np.int8)
    lib().orc_uc_repair(p.size, _p(p), float(threshold), int(TU), int(TD), int(u0), int(hold), _p(u, i8p))
    return u


def uc_warm_start(pb, pr, iters: int, threshold: float = 1e-3):
    """NEXT-2 (SPEC warm_start_uc): the multiperiod ACOPF with every unit on (after its held
    prefix) and the schedule held, `iters` inner iterations, then threshold + repair per generator."""
    import dataclasses
    G, T = pb.ngen, pb.T
    uinit = np.ones((G, T), dtype=np.int8)
    for g in range(G):
        uinit[g, :int(pb.hold[g])] = int(pb.u0[g])
    o = Oracle(dataclasses.replace(pb, u_init=uinit), dataclasses.replace(pr, uc_fixed=1))
    o.iterate(iters)
    p = o.get_state()["p"].reshape(G, T)
    o.close()
    u = np.stack([uc_repair(p[g], threshold, pb.min_up[g], pb.min_dn[g], pb.u0[g], pb.hold[g]) for g in range(G)])
    return u, p


def dp_solve(L, TU, TD, u0, hold):
    L = _f64(L).reshape(-1)
    T = L.size // 4
    s = np.zeros(T, dtype=np.int8)
    cost = lib().orc_dp(T, _p(L), TU, TD, u0, hold, _p(s, i8p))
    return s, cost


def gen_x(vec):
    vec = _f64(vec)
    out = np.zeros(3)
    lib().orc_gen_x(_p(vec), _p(out))
    return out


def boxqp3(c, e):
    c = _f64(c)
    e = _f64(e)
    m, n = c.shape
    cc = np.zeros((m, 3))
    cc[:, :n] = c
    v = np.zeros(3)
    lib().orc_boxqp3(n, m, _p(cc), _p(e), _p(v))
    return v[:n]


def bus_kkt(alpha, beta, a, tauhat, P, Q):
    alpha, beta, a, tauhat = map(_f64, (alpha, beta, a, tauhat))
    v = np.zeros(alpha.size)
    mu = np.zeros(2)
    lib().orc_bus_kkt(alpha.size, _p(alpha), _p(beta), _p(a), _p(tauhat), P, Q, _p(v), _p(mu))
    return v, mu


def branch_solve(y, wlo, whi, rate, tau, rho_pq, rho_va, pr, x, al, plain=False):
    """stats: tron its, capped, al active, al rounds, al capped, flops fast, flops al,
    Newton its fast, Newton its al"""
    x = _f64(x).copy()
    al = _f64(al).copy()
    f = np.zeros(4)
    st = np.zeros(9, dtype=np.int64)
    prc = params_c(pr, plain)
    lib().orc_branch_solve(_p(_f64(y)), _p(_f64(wlo)), _p(_f64(whi)), rate, _p(_f64(tau)),
                           rho_pq, rho_va, C.byref(prc), _p(x), _p(al), _p(f), _p(st, i64p))
    return x, al, f, st


def tron_quadratic(A, b, lo, hi, x0, gtol=1e-10, maxit=200):
    A = _f64(A)
    n = b.size
    x = _f64(x0).copy()
    it = lib().orc_tron_quadratic(n, _p(A.reshape(-1)), _p(_f64(b)), _p(_f64(lo)), _p(_f64(hi)),
                                  gtol, maxit, _p(x))
    return x, it


def sincos(a):
    """(sin a, cos a) by the oracle's explicit polynomial (R54)"""
    s, c = C.c_double(), C.c_double()
    lib().orc_sincos(float(a), C.byref(s), C.byref(c))
    return s.value, c.value


def branch_flows(y, x):
    f = np.zeros(4)
    J = np.zeros(16)
    H = np.zeros(64)
    lib().orc_branch_flows(_p(_f64(y)), _p(_f64(x)), _p(f), _p(J), _p(H))
    return f, J.reshape(4, 4), H.reshape(4, 4, 4)
