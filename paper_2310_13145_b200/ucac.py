"""Thin ctypes binding of libucac.so (include/ucac.h).  Argument marshalling only: every
step of the ADMM hot path runs in the CUDA kernels behind the C ABI.  There is no CPU
fallback: if the library or a B200 is missing, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import build as _build

_lock = threading.Lock()
_lib = None

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int32)
i8p = C.POINTER(C.c_int8)
i64p = C.POINTER(C.c_int64)

NKERNELS = 10
KERNELS = ["k_branch", "k_gen", "k_bus", "k_ubar", "k_bus_late", "k_branch_al", "k_rows", "k_genx", "k_rows_late",
           "k_fold_early"]
STATUS = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "ECUDA", 4: "ENCCL", 5: "ENUMERIC", 6: "ESTATE", 7: "EUNSUPPORTED"}


class UcacError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"ucac {STATUS.get(code, code)}: {msg}")
        self.code = code


class Network(C.Structure):
    _fields_ = [("nbus", C.c_int32), ("ngen", C.c_int32), ("nbranch", C.c_int32), ("ref_bus", C.c_int32),
                ("base_mva", C.c_double), ("bus_gs", dp), ("bus_bs", dp), ("bus_vmin", dp), ("bus_vmax", dp),
                ("br_from", ip), ("br_to", ip), ("br_y", dp), ("br_rate", dp), ("gen_bus", ip),
                ("gen_pmin", dp), ("gen_pmax", dp), ("gen_qmin", dp), ("gen_qmax", dp)]


class Horizon(C.Structure):
    _fields_ = [("T", C.c_int32), ("pd", dp), ("qd", dp)]


class Costs(C.Structure):
    _fields_ = [("c2", dp), ("c1", dp), ("c0", dp), ("startup", dp), ("shutdown", dp)]


class Uc(C.Structure):
    _fields_ = [("ramp_up", dp), ("ramp_dn", dp), ("su_ramp", dp), ("sd_ramp", dp), ("min_up", ip),
                ("min_dn", ip), ("u0", ip), ("hold", ip), ("p0", dp), ("u_init", i8p)]


class Params(C.Structure):
    _fields_ = [("rho_pq", C.c_double), ("rho_va", C.c_double), ("rho_uc", C.c_double),
                ("beta0", C.c_double), ("tau", C.c_double), ("theta", C.c_double),
                ("lambda_max", C.c_double), ("beta_max", C.c_double), ("eps_inner_abs", C.c_double),
                ("inner_min", C.c_int32), ("inner_cap", C.c_int32), ("outer_enabled", C.c_int32),
                ("tron_gtol_rel", C.c_double), ("tron_maxit", C.c_int32), ("al_maxit", C.c_int32),
                ("al_eta_star", C.c_double), ("al_sigma0_rel", C.c_double), ("al_sigma_max_rel", C.c_double),
                ("al_sigma_decay", C.c_double), ("uc_fixed", C.c_int32), ("variant", C.c_int32),
                ("strict_fp", C.c_int32), ("diverge_window", C.c_int32), ("diverge_factor", C.c_double)]


class Dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("comm_mode", C.c_int32),
                ("nccl_id", C.c_ubyte * 128), ("bus_part", ip), ("bus_xy", dp), ("branch_w", dp),
                ("cut", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("primal_inf", C.c_double), ("rz_inf", C.c_double), ("rz_2", C.c_double),
                ("z_inf", C.c_double), ("z_2", C.c_double), ("dual_inf", C.c_double),
                ("objective", C.c_double), ("beta", C.c_double),
                ("inner_total", C.c_int64), ("outer_total", C.c_int64), ("tron_iters", C.c_int64),
                ("tron_capped", C.c_int64), ("al_active", C.c_int64), ("al_capped", C.c_int64),
                ("al_tron_iters", C.c_int64),
                ("inner_since_outer", C.c_int32), ("outer_k", C.c_int32),
                ("err_kernel", C.c_int32), ("err_iter", C.c_int32),
                ("err_comp", C.c_int32), ("err_period", C.c_int32),
                ("diverged_iter", C.c_int32), ("hist_len", C.c_int32)]


class Solution(C.Structure):
    _fields_ = [("u_on", i8p), ("p", dp), ("q", dp), ("wbar", dp), ("thetabar", dp), ("flows", dp)]


STATE_FIELDS = [("u", np.int8, "GT"), ("p", np.float64, "GT"), ("q", np.float64, "GT"),
                ("ph", np.float64, "GT"), ("ub_on", np.float64, "GT"), ("ub_su", np.float64, "GT"),
                ("ub_sd", np.float64, "GT"), ("pbar", np.float64, "GT"), ("qbar", np.float64, "GT"),
                ("zg", np.float64, "12GT"), ("yg", np.float64, "12GT"), ("lg", np.float64, "12GT"),
                ("x", np.float64, "4LT"), ("f", np.float64, "4LT"), ("fbar", np.float64, "4LT"),
                ("al", np.float64, "3LT"), ("zb", np.float64, "8LT"), ("yb", np.float64, "8LT"),
                ("lb", np.float64, "8LT"), ("wbar", np.float64, "BT"), ("thbar", np.float64, "BT"),
                ("scal", np.float64, "8")]


class State(C.Structure):
    _fields_ = [(n, i8p if t == np.int8 else dp) for n, t, _ in STATE_FIELDS]


class Sizes(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("gen_periods", C.c_int64), ("branch_periods", C.c_int64),
                ("bus_periods", C.c_int64), ("alg_bytes_per_iter", C.c_int64),
                ("alg_bytes", C.c_int64 * NKERNELS)]


def library_path() -> str:
    return _build.LIB


def lib(build_if_missing: bool = True):
    """Load libucac.so (building it in-tree with nvcc if missing)."""
    global _lib
    with _lock:
        if _lib is None:
            path = _build.LIB
            if not os.path.exists(path):
                if not build_if_missing:
                    raise UcacError(3, f"{path} missing; run __graft_entry__.build()")
                _build.build()
            L = C.CDLL(path)
            _declare(L)
            _lib = L
    return _lib


def _declare(L):
    L.ucac_create.argtypes = [C.POINTER(Network), C.POINTER(Horizon), C.POINTER(Costs), C.POINTER(Uc),
                              C.POINTER(Params), C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
    L.ucac_create.restype = C.c_int
    L.ucac_uc_warm_start.argtypes = [C.POINTER(Network), C.POINTER(Horizon), C.POINTER(Costs), C.POINTER(Uc),
                                     C.POINTER(Params), C.c_int32, C.c_double, i8p]
    L.ucac_uc_warm_start.restype = C.c_int
    L.ucac_iterate.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_double, C.POINTER(C.c_int32)]
    L.ucac_set_rho.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double]
    L.ucac_iterate.restype = C.c_int
    L.ucac_iterate_timed.argtypes = [C.c_void_p, C.c_int32, dp, i64p]
    L.ucac_iterate_timed.restype = C.c_int
    L.ucac_kernel_name.argtypes = [C.c_int32]
    L.ucac_kernel_name.restype = C.c_char_p
    L.ucac_residuals.argtypes = [C.c_void_p, C.POINTER(Report)]
    L.ucac_residuals.restype = C.c_int
    L.ucac_history.argtypes = [C.c_void_p, dp, C.c_int32, C.POINTER(C.c_int32)]
    L.ucac_history.restype = C.c_int
    L.ucac_get_solution.argtypes = [C.c_void_p, C.POINTER(Solution)]
    L.ucac_get_solution.restype = C.c_int
    L.ucac_get_state.argtypes = [C.c_void_p, C.POINTER(State)]
    L.ucac_get_state.restype = C.c_int
    L.ucac_set_state.argtypes = [C.c_void_p, C.POINTER(State)]
    L.ucac_set_state.restype = C.c_int
    L.ucac_dp_batch.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
    L.ucac_dp_batch.restype = C.c_int
    L.ucac_get_sizes.argtypes = [C.c_void_p, C.POINTER(Sizes)]
    L.ucac_get_sizes.restype = C.c_int
    L.ucac_stream.argtypes = [C.c_void_p]
    L.ucac_stream.restype = C.c_void_p
    L.ucac_last_error.argtypes = [C.c_void_p]
    L.ucac_last_error.restype = C.c_char_p
    L.ucac_destroy.argtypes = [C.c_void_p]
    L.ucac_destroy.restype = None
    L.ucac_partition.argtypes = [C.c_int32, C.c_int32, ip, ip, dp, C.c_int32, ip, dp]
    L.ucac_partition.restype = C.c_int
    L.ucac_halo_lists.argtypes = [C.c_int32, C.c_int32, ip, ip, ip, C.c_int32, C.c_int32, ip, ip, ip, ip, ip, ip, ip]
    L.ucac_halo_lists.restype = C.c_int
    L.ucac_nccl_unique_id.argtypes = [C.POINTER(C.c_ubyte)]
    L.ucac_nccl_unique_id.restype = C.c_int
    L.ucac_iterate_group.argtypes = [C.POINTER(C.c_void_p), C.c_int32, C.c_int32]
    L.ucac_iterate_group.restype = C.c_int
    L.ucac_local_map.argtypes = [C.c_void_p, C.c_int32, ip, ip]
    L.ucac_local_map.restype = C.c_int
    L.ucac_debug_poison.argtypes = [C.c_void_p, C.c_int32, C.c_int64]
    L.ucac_debug_poison.restype = C.c_int
    L.ucac_p2p_group.argtypes = [C.POINTER(C.c_void_p), C.c_int32]
    L.ucac_p2p_group.restype = C.c_int
    L.ucac_p2p_export.argtypes = [C.c_void_p, C.c_void_p]
    L.ucac_p2p_export.restype = C.c_int
    L.ucac_p2p_import.argtypes = [C.c_void_p, C.c_void_p]
    L.ucac_p2p_import.restype = C.c_int
    L.ucac_comm_info.argtypes = [C.c_void_p, ip, ip]
    L.ucac_comm_info.restype = C.c_int
    L.ucac_comm_nccl.argtypes = [C.c_void_p]
    L.ucac_comm_nccl.restype = C.c_int32
    L.ucac_measure_latencies.argtypes = [dp]
    L.ucac_measure_latencies.restype = C.c_int
    L.ucac_time_split.argtypes = [C.c_int32, C.c_int32, C.c_int32, ip]
    L.ucac_time_split.restype = C.c_int
    L.ucac_measure_fp64_peak.argtypes = [C.c_int32, dp, dp]
    L.ucac_measure_fp64_peak.restype = C.c_int


EXPORTED = ["ucac_create", "ucac_iterate", "ucac_set_rho", "ucac_iterate_timed", "ucac_kernel_name", "ucac_residuals",
            "ucac_get_solution", "ucac_get_state", "ucac_set_state", "ucac_dp_batch", "ucac_get_sizes",
            "ucac_stream", "ucac_last_error", "ucac_destroy", "ucac_partition", "ucac_halo_lists",
            "ucac_nccl_unique_id", "ucac_iterate_group", "ucac_local_map", "ucac_uc_warm_start",
            "ucac_debug_poison", "ucac_measure_fp64_peak", "ucac_time_split", "ucac_comm_info",
            "ucac_p2p_group", "ucac_p2p_export", "ucac_p2p_import", "ucac_history", "ucac_comm_nccl",
            "ucac_measure_latencies"]


def _check(rc, h=None):
    if rc != 0:
        msg = lib().ucac_last_error(h)
        raise UcacError(rc, msg.decode() if msg else "")


def params_struct(pr) -> Params:
    return Params(pr.rho_pq, pr.rho_va, pr.rho_uc, pr.beta0, pr.tau, pr.theta, pr.lambda_max, pr.beta_max,
                  pr.eps_inner_abs, pr.inner_min, pr.inner_cap, pr.outer_enabled, pr.tron_gtol_rel,
                  pr.tron_maxit, pr.al_maxit, pr.al_eta_star, pr.al_sigma0_rel, pr.al_sigma_max_rel,
                  pr.al_sigma_decay, pr.uc_fixed, pr.variant, pr.strict_fp, pr.diverge_window, pr.diverge_factor)


def problem_structs(pb, keep: list):
    """ucac_network / horizon / costs / uc of a normalized Problem (arrays kept alive in `keep`)."""
    def a(x, t=dp):
        x = np.ascontiguousarray(x)
        keep.append(x)
        return x.ctypes.data_as(t)
    net = Network(pb.nbus, pb.ngen, pb.nbranch, pb.ref_bus, pb.base_mva, a(pb.bus_gs), a(pb.bus_bs),
                  a(pb.bus_vmin), a(pb.bus_vmax), a(pb.br_from, ip), a(pb.br_to, ip), a(pb.br_y.reshape(-1)),
                  a(pb.br_rate), a(pb.gen_bus, ip), a(pb.pmin), a(pb.pmax), a(pb.qmin), a(pb.qmax))
    hz = Horizon(pb.T, a(pb.pd.reshape(-1)), a(pb.qd.reshape(-1)))
    co = Costs(a(pb.c2), a(pb.c1), a(pb.c0), a(pb.csu), a(pb.csd))
    ui = a(np.ascontiguousarray(pb.u_init, dtype=np.int8).reshape(-1), i8p) if pb.u_init is not None else None
    uc = Uc(a(pb.ramp_up), a(pb.ramp_dn), a(pb.su_ramp), a(pb.sd_ramp), a(pb.min_up, ip), a(pb.min_dn, ip),
            a(pb.u0, ip), a(pb.hold, ip), a(pb.p0), ui)
    return net, hz, co, uc


def uc_warm_start(pb, pr, iters: int, threshold: float = 1e-3) -> np.ndarray:
    """NEXT-2 UC warm start (ucac_uc_warm_start): the schedule [ngen, T] to pass as u_init."""
    pb = pb.normalized()
    keep = []
    net, hz, co, uc = problem_structs(pb, keep)
    prm = params_struct(pr)
    u = np.zeros(pb.ngen * pb.T, dtype=np.int8)
    _check(lib().ucac_uc_warm_start(C.byref(net), C.byref(hz), C.byref(co), C.byref(uc), C.byref(prm), int(iters),
                                    float(threshold), u.ctypes.data_as(i8p)), None)
    return u.reshape(pb.ngen, pb.T)


class Context:
    """One ADMM context on the current CUDA device (ucac_create .. ucac_destroy)."""

    def __init__(self, pb, pr, stream: int = 0, dist: dict | None = None):
        """dist: None (one GPU) or {"rank", "nranks", "comm_mode" (0 NCCL / 1 loopback group),
        "nccl_id" (bytes, mode 0), "bus_part" (optional), "bus_xy" (optional),
        "cut" (0 bus-graph cut, 1 time cut NEXT-4(c))}"""
        self.L = lib()
        pb = pb.normalized()
        self.pb, self.pr = pb, pr
        keep = []

        def a(x, t=dp):
            x = np.ascontiguousarray(x)
            keep.append(x)
            return x.ctypes.data_as(t)
        net, hz, co, uc = problem_structs(pb, keep)
        prm = params_struct(pr)
        dist_c = None
        if dist is not None:
            dist_c = Dist()
            dist_c.rank, dist_c.nranks, dist_c.comm_mode = dist["rank"], dist["nranks"], dist.get("comm_mode", 0)
            if dist.get("nccl_id") is not None:
                dist_c.nccl_id[:] = list(bytes(dist["nccl_id"]))
            dist_c.bus_part = a(np.asarray(dist["bus_part"], dtype=np.int32), ip) if dist.get("bus_part") is not None else None
            xy = dist.get("bus_xy", pb.bus_xy)
            dist_c.bus_xy = a(np.asarray(xy, dtype=np.float64).reshape(-1)) if xy is not None else None
            dist_c.cut = int(dist.get("cut", 0))
            if dist.get("branch_w") is not None:
                dist_c.branch_w = a(np.asarray(dist["branch_w"], dtype=np.float64))
        h = C.c_void_p()
        rc = self.L.ucac_create(C.byref(net), C.byref(hz), C.byref(co), C.byref(uc), C.byref(prm),
                                C.byref(dist_c) if dist_c is not None else None,
                                C.c_void_p(stream) if stream else None, C.byref(h))
        _check(rc, None)
        self.h = h
        self.dist = dist
        self._local = {}
        for which, name in ((0, "gen"), (1, "branch"), (2, "bus")):
            cnt = C.c_int32(0)
            _check(self.L.ucac_local_map(self.h, which, None, C.byref(cnt)), self.h)
            ids = np.zeros(cnt.value, dtype=np.int32)
            _check(self.L.ucac_local_map(self.h, which, ids.ctypes.data_as(ip), C.byref(cnt)), self.h)
            self._local[name] = ids
        per = np.zeros(4, dtype=np.int32)
        cnt = C.c_int32(0)
        _check(self.L.ucac_local_map(self.h, 3, per.ctypes.data_as(ip), C.byref(cnt)), self.h)
        # local periods: global index of local period 0, owned [own0, own1), local count
        self.t_off, self.own0, self.own1, self.Tl = (int(v) for v in per)

    def local_ids(self, which: str) -> np.ndarray:
        """global ids of the local generators / branches / owned buses (state layout order)"""
        return self._local[which]

    def close(self):
        if getattr(self, "h", None):
            self.L.ucac_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(self.L.ucac_stream(self.h) or 0)

    def iterate(self, n: int = 1, stop_on_primal: float | None = None) -> int | None:
        done = C.c_int32(0)
        if stop_on_primal is None:
            _check(self.L.ucac_iterate(self.h, n, 0, 0.0, None), self.h)
            return None
        _check(self.L.ucac_iterate(self.h, n, 1, float(stop_on_primal), C.byref(done)), self.h)
        return done.value

    def set_rho(self, rho_pq: float, rho_va: float, rho_uc: float):
        """NEXT-4(b), R53: new penalty classes between iterations (ucac_set_rho)."""
        _check(self.L.ucac_set_rho(self.h, float(rho_pq), float(rho_va), float(rho_uc)), self.h)

    def p2p_export(self) -> bytes:
        """ucac_p2p_export: this rank's IPC blob for the device-initiated exchange (time cut)"""
        buf = (C.c_ubyte * P2P_BLOB)()
        _check(self.L.ucac_p2p_export(self.h, buf), self.h)
        return bytes(buf)

    def p2p_import(self, blobs):
        """ucac_p2p_import: map every rank's exchange buffers (blobs in rank order)"""
        raw = b"".join(blobs)
        buf = (C.c_ubyte * len(raw)).from_buffer_copy(raw)
        _check(self.L.ucac_p2p_import(self.h, buf), self.h)

    def comm_info(self) -> dict:
        """ucac_comm_info: the communicator's own rank count and rank (NCCL contexts)"""
        n, r = C.c_int32(), C.c_int32()
        _check(self.L.ucac_comm_info(self.h, C.byref(n), C.byref(r)), self.h)
        return {"nranks": n.value, "rank": r.value, "nccl": self.L.ucac_comm_nccl(self.h) == 1}

    def poison(self, field: str, index: int):
        """fault injection (ucac_debug_poison): NaN into one element of zb / yb / zg / yg"""
        _check(self.L.ucac_debug_poison(self.h, {"zb": 0, "yb": 1, "zg": 2, "yg": 3}[field], int(index)), self.h)

    def report_raw(self) -> dict:
        """ucac_residuals without raising on UCAC_ENUMERIC (the err_* fields say where)"""
        r = Report()
        rc = self.L.ucac_residuals(self.h, C.byref(r))
        d = {n: getattr(r, n) for n, _ in Report._fields_}
        d["status"] = STATUS.get(rc, rc)
        return d

    def iterate_timed(self, n: int):
        ms = np.zeros(NKERNELS)
        cnt = np.zeros(NKERNELS, dtype=np.int64)
        _check(self.L.ucac_iterate_timed(self.h, n, ms.ctypes.data_as(dp), cnt.ctypes.data_as(i64p)), self.h)
        return dict(zip(KERNELS, ms)), dict(zip(KERNELS, cnt))

    HIST_FIELDS = ("primal_inf", "dual_inf", "z_inf", "z_2", "objective", "beta")

    def history(self, n: int = 256) -> np.ndarray:
        """the last min(n, 256) iterations' records (ucac_history), oldest first: a structured
        array with the fields HIST_FIELDS"""
        buf = np.zeros((max(0, int(n)), len(self.HIST_FIELDS)))
        got = C.c_int32(0)
        _check(self.L.ucac_history(self.h, buf.ctypes.data_as(dp), int(n), C.byref(got)), self.h)
        return np.rec.fromarrays(buf[:got.value].T.copy(), names=list(self.HIST_FIELDS))

    def report(self) -> dict:
        r = Report()
        _check(self.L.ucac_residuals(self.h, C.byref(r)), self.h)
        return {n: getattr(r, n) for n, _ in Report._fields_}

    def solution_shapes(self) -> dict:
        """{field: (size, dtype)} of solution()'s arrays (for caller-owned, e.g. pinned, buffers)"""
        GT, LT, BT = (len(self._local["gen"]) * self.Tl, len(self._local["branch"]) * self.Tl,
                      len(self._local["bus"]) * self.Tl)
        return {"u_on": (GT, np.int8), "p": (GT, np.float64), "q": (GT, np.float64), "wbar": (BT, np.float64),
                "thetabar": (BT, np.float64), "flows": (4 * LT, np.float64)}

    def solution(self, out: dict | None = None) -> dict:
        """ucac_get_solution into fresh arrays, or into `out` (caller-owned contiguous arrays of
        solution_shapes(), e.g. page-locked buffers reused across calls)"""
        shapes = self.solution_shapes()
        if out is None:
            out = {k: np.zeros(n, t) for k, (n, t) in shapes.items()}
        else:
            for k, (n, t) in shapes.items():
                a = out[k]
                if a.dtype != t or a.size != n or not a.flags["C_CONTIGUOUS"]:
                    raise ValueError(f"solution buffer {k}: need {n} contiguous {np.dtype(t)}")
        s = Solution(out["u_on"].ctypes.data_as(i8p), *[out[k].ctypes.data_as(dp) for k in
                                                         ("p", "q", "wbar", "thetabar", "flows")])
        _check(self.L.ucac_get_solution(self.h, C.byref(s)), self.h)
        return out

    def _sizes(self):
        GT, LT, BT = (len(self._local["gen"]) * self.Tl, len(self._local["branch"]) * self.Tl,
                      len(self._local["bus"]) * self.Tl)
        return {"GT": GT, "12GT": 12 * GT, "4LT": 4 * LT, "3LT": 3 * LT, "8LT": 8 * LT, "BT": BT, "8": 8}

    def get_state(self) -> dict:
        sz = self._sizes()
        st = {n: np.zeros(sz[s], dtype=t) for n, t, s in STATE_FIELDS}
        sc = State(*[st[n].ctypes.data_as(i8p if t == np.int8 else dp) for n, t, _ in STATE_FIELDS])
        _check(self.L.ucac_get_state(self.h, C.byref(sc)), self.h)
        return st

    def set_state(self, st: dict):
        sz = self._sizes()
        arr = {n: np.ascontiguousarray(st[n], dtype=t).reshape(-1) for n, t, _ in STATE_FIELDS}
        for n, t, s in STATE_FIELDS:
            if arr[n].size != sz[s]:
                raise ValueError(f"state field {n}: {arr[n].size} != {sz[s]}")
        sc = State(*[arr[n].ctypes.data_as(i8p if t == np.int8 else dp) for n, t, _ in STATE_FIELDS])
        _check(self.L.ucac_set_state(self.h, C.byref(sc)), self.h)

    def sizes(self) -> dict:
        s = Sizes()
        _check(self.L.ucac_get_sizes(self.h, C.byref(s)), self.h)
        d = {n: getattr(s, n) for n, _ in Sizes._fields_ if n != "alg_bytes"}
        d["alg_bytes"] = dict(zip(KERNELS, list(s.alg_bytes)))
        return d


def measure_fp64_peak(iters: int = 4096) -> dict:
    """ucac_measure_fp64_peak: the DFMA-chain FP64 peak of the current device"""
    tf, ms = C.c_double(), C.c_double()
    _check(lib().ucac_measure_fp64_peak(int(iters), C.byref(tf), C.byref(ms)), None)
    return {"tflops": tf.value, "ms": ms.value, "iters": int(iters)}


def measure_latencies() -> dict:
    """ucac_measure_latencies: dependent-chain latencies (SM cycles per link) of the current device"""
    out = np.zeros(5)
    _check(lib().ucac_measure_latencies(out.ctypes.data_as(dp)), None)
    return dict(zip(("dfma", "dadd", "shfl_add", "rcp", "sqrt"), (float(v) for v in out)))


def dp_batch(L, min_up, min_dn, u0, hold):
    """Batched DP (Alg. 2) on host arrays; L [ngen, T, 2, 2]."""
    Lh = np.ascontiguousarray(L, dtype=np.float64)
    G, T = Lh.shape[0], Lh.shape[1]
    sched = np.zeros((G, T), dtype=np.int8)
    cost = np.zeros(G)
    arrs = [np.ascontiguousarray(v, dtype=np.int32) for v in (min_up, min_dn, u0, hold)]
    rc = lib().ucac_dp_batch(G, T, Lh.ctypes.data, *[x.ctypes.data for x in arrs], sched.ctypes.data,
                             cost.ctypes.data, 0, None)
    _check(rc, None)
    return sched, cost


def dp_batch_device(G, T, L_ptr, tu_ptr, td_ptr, u0_ptr, hold_ptr, sched_ptr, cost_ptr, stream=0):
    """Batched DP on device pointers (asynchronous on `stream`)."""
    rc = lib().ucac_dp_batch(G, T, L_ptr, tu_ptr, td_ptr, u0_ptr, hold_ptr, sched_ptr, cost_ptr, 1,
                             C.c_void_p(stream) if stream else None)
    _check(rc, None)


def partition(pb, nparts: int, use_xy: bool = True, branch_w=None) -> np.ndarray:
    """bus -> rank (ucac_partition: weighted RCB on the bus coordinates, or BFS chunks, then FM-gain
    boundary refinement; branch_w = per-branch solve weights or None)"""
    pb = pb.normalized()
    part = np.zeros(pb.nbus, dtype=np.int32)
    xy = np.ascontiguousarray(pb.bus_xy, dtype=np.float64).reshape(-1) if (use_xy and pb.bus_xy is not None) else None
    bw = np.ascontiguousarray(branch_w, dtype=np.float64) if branch_w is not None else None
    rc = lib().ucac_partition(pb.nbus, pb.nbranch, pb.br_from.ctypes.data_as(ip), pb.br_to.ctypes.data_as(ip),
                              xy.ctypes.data_as(dp) if xy is not None else None, nparts, part.ctypes.data_as(ip),
                              bw.ctypes.data_as(dp) if bw is not None else None)
    _check(rc, None)
    return part


def halo_lists(pb, part, rank: int) -> dict:
    """ucac_halo_lists: the rank-local components and halo (global ids)"""
    pb = pb.normalized()
    part = np.ascontiguousarray(part, dtype=np.int32)
    nparts = int(part.max()) + 1
    sizes = np.zeros(6, dtype=np.int32)
    args = [pb.nbus, pb.nbranch, pb.br_from.ctypes.data_as(ip), pb.br_to.ctypes.data_as(ip), part.ctypes.data_as(ip),
            nparts, rank, sizes.ctypes.data_as(ip)]
    _check(lib().ucac_halo_lists(*args, None, None, None, None, None, None), None)
    names = ["own_bus", "ghost_bus", "local_branch", "phantom", "cut_branch", "export_bus"]
    out = {n: np.zeros(int(s), dtype=np.int32) for n, s in zip(names, sizes)}
    _check(lib().ucac_halo_lists(*args, *[out[n].ctypes.data_as(ip) for n in names]), None)
    return out


def time_split(T: int, nranks: int, rank: int) -> dict:
    """ucac_time_split: the periods of `rank` under the time cut (host only)"""
    out = np.zeros(4, dtype=np.int32)
    _check(lib().ucac_time_split(int(T), int(nranks), int(rank), out.ctypes.data_as(ip)), None)
    return {"t_off": int(out[0]), "own0": int(out[1]), "own1": int(out[2]), "Tl": int(out[3])}


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(lib().ucac_nccl_unique_id(buf), None)
    return bytes(buf)


P2P_BLOB = 96


def p2p_group(ctxs):
    """ucac_p2p_group: device-initiated exchanges for a time-cut loopback group (one device)"""
    arr = (C.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])
    _check(lib().ucac_p2p_group(arr, len(ctxs)), ctxs[0].h)


def iterate_group(ctxs, iters: int):
    """ucac_iterate_group over comm_mode-1 contexts (rank order)"""
    arr = (C.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])
    _check(lib().ucac_iterate_group(arr, len(ctxs), iters), ctxs[0].h)


def local_part(ctx) -> dict:
    """what a rank contributes to the global state: its local component ids, periods and state"""
    return {"gen": ctx.local_ids("gen"), "branch": ctx.local_ids("branch"), "bus": ctx.local_ids("bus"),
            "t_off": ctx.t_off, "own0": ctx.own0, "own1": ctx.own1, "Tl": ctx.Tl, "state": ctx.get_state()}


def assemble_state(pb, ctxs) -> dict:
    """global canonical state from the local states of a partition group (contexts, or the
    local_part() dicts of the ranks)"""
    return assemble_parts(pb, [c if isinstance(c, dict) else local_part(c) for c in ctxs])


def assemble_parts(pb, parts) -> dict:
    pb = pb.normalized()
    T, G, L, B = pb.T, pb.ngen, pb.nbranch, pb.nbus
    out = {n: np.zeros({"GT": G * T, "12GT": 12 * G * T, "4LT": 4 * L * T, "3LT": 3 * L * T, "8LT": 8 * L * T,
                        "BT": B * T, "8": 8}[s], dtype=t) for n, t, s in STATE_FIELDS}
    for c in parts:
        st = c["state"]
        g, l, b = (np.asarray(c[k]) for k in ("gen", "branch", "bus"))
        # the owned periods of this part (all of them unless time cut): local -> global index
        tl = np.arange(c["own0"], c["own1"])
        tg = tl + c["t_off"]
        Tl = c["Tl"]
        gl = (np.arange(len(g))[:, None] * Tl + tl).reshape(-1)
        ll = (np.arange(len(l))[:, None] * Tl + tl).reshape(-1)
        bl = (np.arange(len(b))[:, None] * Tl + tl).reshape(-1)
        gi = (g[:, None] * T + tg).reshape(-1)
        li = (l[:, None] * T + tg).reshape(-1)
        bi = (b[:, None] * T + tg).reshape(-1)
        for n, t, s in STATE_FIELDS:
            v = st[n]
            if s == "GT":
                out[n][gi] = v[gl]
            elif s == "12GT":
                out[n].reshape(12, -1)[:, gi] = v.reshape(12, -1)[:, gl]
            elif s == "8LT":
                out[n].reshape(8, -1)[:, li] = v.reshape(8, -1)[:, ll]
            elif s in ("4LT", "3LT"):
                k = 4 if s == "4LT" else 3
                out[n].reshape(-1, k)[li] = v.reshape(-1, k)[ll]
            elif s == "BT":
                out[n][bi] = v[bl]
            else:
                out[n] = v
    return out
