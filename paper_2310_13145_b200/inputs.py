"""Seeded synthetic inputs for the UC-ACOPF ADMM hot path (arXiv 2310.13145).

This module holds NO arithmetic of the method (no ADMM step, no subproblem solve).  It
only builds problem data, and both sides (the CPU oracle under ``oracle/`` and the CUDA
path behind ``include/ucac.h``) consume its output:

* ``case9()`` -- MATPOWER case9 (public data) turned into the paper's
  UC-ACOPF instance shape (0.7 demand discount, ramps 10 % of P-max).
* ``synthetic_case(...)`` -- deterministic IEEE-shaped grids (case30/118/300-shaped and a
  2869-bus pegase-shaped grid) built from a splitmix64 stream (never NumPy's
  distribution streams, which are not version stable), with a planted AC power flow at
  peak load as a feasibility certificate (DESIGN.md section 6 gives the recipe).
* ``Problem`` / ``Params`` containers and the ``CONFIGS`` registry of BASELINE.json.

The Newton-Raphson power flow below is input generation (it certifies that a synthetic
grid is AC-feasible); it is not part of the paper's method.
"""
from __future__ import annotations

import dataclasses
import functools
import hashlib
import math
from typing import Optional

import numpy as np

MASK64 = (1 << 64) - 1


class SplitMix64:
    """splitmix64 (Steele, Lea & Flood 2014); doubles as (x >> 11) * 2^-53."""

    def __init__(self, seed: int):
        self.s = seed & MASK64

    def next(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & MASK64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self, a: float = 0.0, b: float = 1.0) -> float:
        return a + (b - a) * ((self.next() >> 11) * (2.0 ** -53))

    def normal(self) -> float:
        u1 = max(self.uniform(), 1e-300)
        u2 = self.uniform()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)

    def randint(self, lo: int, hi: int) -> int:
        """uniform integer in [lo, hi]"""
        return lo + int(self.uniform() * (hi - lo + 1)) % (hi - lo + 1)

    def permutation(self, n: int) -> list:
        a = list(range(n))
        for i in range(n - 1, 0, -1):
            j = self.randint(0, i)
            a[i], a[j] = a[j], a[i]
        return a


# --------------------------------------------------------------------------------------
# containers
# --------------------------------------------------------------------------------------
@dataclasses.dataclass
class Problem:
    """UC-ACOPF instance, per unit on ``base_mva`` (SURVEY.md 8(b) ucac_network etc.)."""

    name: str
    base_mva: float
    ref_bus: int
    bus_gs: np.ndarray
    bus_bs: np.ndarray
    bus_vmin: np.ndarray
    bus_vmax: np.ndarray
    pd: np.ndarray  # [T, nbus]
    qd: np.ndarray  # [T, nbus]
    br_from: np.ndarray
    br_to: np.ndarray
    br_y: np.ndarray  # [nbranch, 8] Gii Gij Gji Gjj Bii Bij Bji Bjj
    br_rate: np.ndarray  # [nbranch] pu, 0 = unlimited
    gen_bus: np.ndarray
    pmin: np.ndarray
    pmax: np.ndarray
    qmin: np.ndarray
    qmax: np.ndarray
    c2: np.ndarray  # $/MW^2 h
    c1: np.ndarray  # $/MW h
    c0: np.ndarray  # $/h when on
    csu: np.ndarray
    csd: np.ndarray
    ramp_up: np.ndarray
    ramp_dn: np.ndarray
    su_ramp: np.ndarray
    sd_ramp: np.ndarray
    min_up: np.ndarray
    min_dn: np.ndarray
    u0: np.ndarray
    hold: np.ndarray
    p0: np.ndarray
    u_init: Optional[np.ndarray] = None  # [ngen, T] int8
    bus_xy: Optional[np.ndarray] = None  # coordinates (partitioner)

    @property
    def nbus(self) -> int:
        return int(self.bus_gs.shape[0])

    @property
    def ngen(self) -> int:
        return int(self.gen_bus.shape[0])

    @property
    def nbranch(self) -> int:
        return int(self.br_from.shape[0])

    @property
    def T(self) -> int:
        return int(self.pd.shape[0])

    def nrows(self) -> int:
        """number of coupling rows: 12 per (g,t) minus the t=1 RC row,
        8 per (l,t)."""
        return self.ngen * (12 * self.T - 1) + 8 * self.nbranch * self.T

    def normalized(self) -> "Problem":
        """contiguous arrays with the ABI dtypes"""
        d = {}
        for f in dataclasses.fields(self):
            v = getattr(self, f.name)
            if isinstance(v, np.ndarray):
                if f.name in ("br_from", "br_to", "gen_bus", "min_up", "min_dn", "u0", "hold"):
                    v = np.ascontiguousarray(v, dtype=np.int32)
                elif f.name == "u_init":
                    v = np.ascontiguousarray(v, dtype=np.int8)
                else:
                    v = np.ascontiguousarray(v, dtype=np.float64)
            d[f.name] = v
        return Problem(**d)

    def digest(self) -> str:
        h = hashlib.sha256()
        for f in dataclasses.fields(self):
            v = getattr(self, f.name)
            if isinstance(v, np.ndarray):
                h.update(f.name.encode())
                h.update(np.ascontiguousarray(v).tobytes())
        return h.hexdigest()

    def restricted(self, T: int) -> "Problem":
        d = dataclasses.asdict(self)
        d = {k: getattr(self, k) for k in d}
        d["pd"] = self.pd[:T].copy()
        d["qd"] = self.qd[:T].copy()
        if self.u_init is not None:
            d["u_init"] = self.u_init[:, :T].copy()
        d["min_up"] = np.minimum(self.min_up, T)
        d["min_dn"] = np.minimum(self.min_dn, T)
        d["hold"] = np.minimum(self.hold, T)
        return Problem(**d)


@dataclasses.dataclass
class Params:
    """ADMM parameters.  rho per class; tau, theta; the rest are the
    readings of DESIGN.md 3 (R10, R20, R21)."""

    rho_pq: float
    rho_va: float
    rho_uc: float
    beta0: float = 1e3
    tau: float = 6.0
    theta: float = 0.8
    lambda_max: float = 1e12
    beta_max: float = 1e12
    eps_inner_abs: float = 1e-6
    inner_min: int = 5
    inner_cap: int = 1000
    outer_enabled: int = 1
    tron_gtol_rel: float = 1e-11
    tron_maxit: int = 100
    al_maxit: int = 50
    al_eta_star: float = 1e-10
    al_sigma0_rel: float = 10.0
    al_sigma_max_rel: float = 1e3
    al_sigma_decay: float = 0.1
    uc_fixed: int = 0          # 1: step (7a) keeps u (NEXT-2 warm start's multiperiod ACOPF)
    variant: int = 0           # NEXT-3 bitmask: 1 = AL for every rated branch (no fast path), 2 = wbar clip
    strict_fp: int = 0         # 1: strict parity mode (oracle operation order / quotients, R54 sin/cos)
    diverge_window: int = 0    # SPEC S:431 divergence detector (0 = off, < 256): an iterate call stops when
    diverge_factor: float = 10.0   # primal > factor x its value `window` iterations earlier (SPEC: 200, 10)


# --------------------------------------------------------------------------------------
# network primitives (input preparation)
# --------------------------------------------------------------------------------------
def branch_admittance(r, x, b, tap=1.0, shift_deg=0.0):
    """MATPOWER pi-model two-port (Y_ff, Y_ft, Y_tf, Y_tt) as the 8 real entries
    (Gii, Gij, Gji, Gjj, Bii, Bij, Bji, Bjj) of Eq. 2e-2h."""
    ys = 1.0 / complex(r, x)
    tap = tap if tap else 1.0
    a = tap * complex(math.cos(math.radians(shift_deg)), math.sin(math.radians(shift_deg)))
    ytt = ys + 1j * b / 2.0
    yff = ytt / (a * a.conjugate())
    yft = -ys / a.conjugate()
    ytf = -ys / a
    return np.array([yff.real, yft.real, ytf.real, ytt.real, yff.imag, yft.imag, ytf.imag, ytt.imag])


def _ybus(nb, fr, to, y8, gs, bs):
    import scipy.sparse as sp

    yff = y8[:, 0] + 1j * y8[:, 4]
    yft = y8[:, 1] + 1j * y8[:, 5]
    ytf = y8[:, 2] + 1j * y8[:, 6]
    ytt = y8[:, 3] + 1j * y8[:, 7]
    rows = np.concatenate([fr, fr, to, to, np.arange(nb)])
    cols = np.concatenate([fr, to, fr, to, np.arange(nb)])
    vals = np.concatenate([yff, yft, ytf, ytt, gs + 1j * bs])
    return sp.csr_matrix((vals, (rows, cols)), shape=(nb, nb))


def power_flow(Y, sbus, v0, ref, pv, pq, tol=1e-10, maxit=40):
    """Polar Newton-Raphson power flow (input certification only)."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl

    V = v0.astype(complex).copy()
    Vm = np.abs(V)
    Va = np.angle(V)
    pvpq = np.concatenate([pv, pq]).astype(int)
    pq = np.asarray(pq, dtype=int)
    for _ in range(maxit):
        Ibus = Y @ V
        mis = V * np.conj(Ibus) - sbus
        F = np.concatenate([mis[pvpq].real, mis[pq].imag])
        if np.max(np.abs(F)) < tol:
            return V, True
        dV = sp.diags(V)
        dI = sp.diags(Ibus)
        Vn = sp.diags(V / np.abs(V))
        dS_dVa = 1j * dV @ np.conj(dI - Y @ dV)
        dS_dVm = dV @ np.conj(Y @ Vn) + np.conj(dI) @ Vn
        J11 = dS_dVa[pvpq][:, pvpq].real
        J12 = dS_dVm[pvpq][:, pq].real
        J21 = dS_dVa[pq][:, pvpq].imag
        J22 = dS_dVm[pq][:, pq].imag
        J = sp.bmat([[J11, J12], [J21, J22]], format="csc")
        dx = spl.spsolve(J, -F)
        if not np.all(np.isfinite(dx)):
            return V, False
        Va[pvpq] += dx[: len(pvpq)]
        Vm[pq] += dx[len(pvpq):]
        V = Vm * np.exp(1j * Va)
        if np.max(Vm) > 3 or np.min(Vm) < 0.3:
            return V, False
    return V, False


# --------------------------------------------------------------------------------------
# demand profile (the ISO-NE factors of P:465 are unpublished, R24)
# --------------------------------------------------------------------------------------
def diurnal_profile(T: int) -> np.ndarray:
    """smooth double-peaked diurnal curve in [0.6, 1.0], period 24, deterministic."""
    h = np.arange(24, dtype=np.float64)
    g = 0.85 * np.exp(-((h - 9.0) / 3.0) ** 2) + 1.0 * np.exp(-((h - 19.0) / 2.5) ** 2) \
        + 0.15 * np.sin(2 * np.pi * h / 24.0)
    g = (g - g.min()) / (g.max() - g.min())
    f = 0.6 + 0.4 * g
    return np.array([f[t % 24] for t in range(T)], dtype=np.float64)


# --------------------------------------------------------------------------------------
# case9 (MATPOWER, public data)
# --------------------------------------------------------------------------------------
CASE9_BRANCH = [  # from to r x b rateA
    (1, 4, 0.0, 0.0576, 0.0, 250), (4, 5, 0.017, 0.092, 0.158, 250), (5, 6, 0.039, 0.17, 0.358, 150),
    (3, 6, 0.0, 0.0586, 0.0, 300), (6, 7, 0.0119, 0.1008, 0.209, 150), (7, 8, 0.0085, 0.072, 0.149, 250),
    (8, 2, 0.0, 0.0625, 0.0, 250), (8, 9, 0.032, 0.161, 0.306, 250), (9, 4, 0.01, 0.085, 0.176, 250),
]
CASE9_GEN = [  # bus Pmin Pmax Qmin Qmax startup shutdown c2 c1 c0
    (1, 10, 250, -300, 300, 1500, 0, 0.11, 5.0, 150),
    (2, 10, 300, -300, 300, 2000, 0, 0.085, 1.2, 600),
    (3, 10, 270, -300, 300, 3000, 0, 0.1225, 1.0, 335),
]
CASE9_LOAD = {5: (90.0, 30.0), 7: (100.0, 35.0), 9: (125.0, 50.0)}


def case9(T: int = 4, factors=None, discount: float = 0.7, rates: bool = True,
          min_up: int = 2, min_dn: int = 2, ramps: bool = True) -> Problem:
    """MATPOWER case9 as a UC-ACOPF instance (BASELINE.json configs[0]).

    factors default (0.75, 0.90, 1.00, 0.80) for T=4, else the diurnal profile;
    demand = discount * factor_t * base load; R = 0.1 Pmax;
    S^U = S^D = max(Pmin, R, p0) (S:138 + R5); p0 = proportional dispatch of 1.02x the
    t=1 load; u0 = 1, L_g = 0 (R25)."""
    base = 100.0
    nb = 9
    if factors is None:
        factors = [0.75, 0.90, 1.00, 0.80] if T == 4 else list(diurnal_profile(T))
    factors = np.asarray(factors, dtype=np.float64)[:T]
    pd0 = np.zeros(nb)
    qd0 = np.zeros(nb)
    for b, (p, q) in CASE9_LOAD.items():
        pd0[b - 1] = p / base
        qd0[b - 1] = q / base
    pd = np.array([discount * factors[t] * pd0 for t in range(T)])
    qd = np.array([discount * factors[t] * qd0 for t in range(T)])
    fr = np.array([b[0] - 1 for b in CASE9_BRANCH])
    to = np.array([b[1] - 1 for b in CASE9_BRANCH])
    y = np.array([branch_admittance(b[2], b[3], b[4]) for b in CASE9_BRANCH])
    rate = np.array([b[5] / base if rates else 0.0 for b in CASE9_BRANCH])
    g = np.array(CASE9_GEN, dtype=np.float64)
    ng = g.shape[0]
    pmin, pmax = g[:, 1] / base, g[:, 2] / base
    load1 = 1.02 * pd[0].sum()
    p0 = np.clip(load1 * pmax / pmax.sum(), pmin, pmax)
    R = 0.1 * pmax if ramps else 10.0 * pmax
    sur = np.maximum(np.maximum(pmin, R), p0) if ramps else 10.0 * pmax
    return Problem(
        name=f"case9_T{T}", base_mva=base, ref_bus=0,
        bus_gs=np.zeros(nb), bus_bs=np.zeros(nb), bus_vmin=np.full(nb, 0.9), bus_vmax=np.full(nb, 1.1),
        pd=pd, qd=qd, br_from=fr, br_to=to, br_y=y, br_rate=rate,
        gen_bus=(g[:, 0] - 1).astype(np.int32), pmin=pmin, pmax=pmax, qmin=g[:, 3] / base, qmax=g[:, 4] / base,
        c2=g[:, 7], c1=g[:, 8], c0=g[:, 9], csu=g[:, 5], csd=g[:, 6],
        ramp_up=R.copy(), ramp_dn=R.copy(), su_ramp=sur.copy(), sd_ramp=sur.copy(),
        min_up=np.full(ng, min(min_up, T)), min_dn=np.full(ng, min(min_dn, T)),
        u0=np.ones(ng, dtype=np.int32), hold=np.zeros(ng, dtype=np.int32), p0=p0,
    ).normalized()


# --------------------------------------------------------------------------------------
# synthetic IEEE-shaped grids (SURVEY.md 8(d) recipe)
# --------------------------------------------------------------------------------------
def _topology(rng: SplitMix64, nb: int, nl: int, clusters: int):
    if clusters <= 1:
        xy = np.array([[rng.uniform(), rng.uniform()] for _ in range(nb)])
    else:
        cent = np.array([[rng.uniform(0.15, 0.85), rng.uniform(0.15, 0.85)] for _ in range(clusters)])
        xy = np.array([cent[i % clusters] + 0.1 * np.array([rng.normal(), rng.normal()]) for i in range(nb)])
    order = rng.permutation(nb)
    conn = np.zeros(nb, dtype=bool)
    conn[order[0]] = True
    conn_list = [order[0]]
    edges = []
    for b in order[1:]:
        cl = np.array(conn_list)
        d = np.hypot(xy[cl, 0] - xy[b, 0], xy[cl, 1] - xy[b, 1])
        k = int(np.argmin(d))
        edges.append((min(b, cl[k]), max(b, cl[k])))
        conn[b] = True
        conn_list.append(b)
    have = set(edges)
    need = nl - (nb - 1)
    kn = 6
    while need > 0:
        cand = {}
        for b in range(nb):
            d = np.hypot(xy[:, 0] - xy[b, 0], xy[:, 1] - xy[b, 1])
            d[b] = np.inf
            for o in np.argsort(d, kind="stable")[:kn]:
                e = (min(b, int(o)), max(b, int(o)))
                if e not in have:
                    cand[e] = float(d[o])
        if len(cand) >= need or kn > 30:
            break
        kn += 4
    extra = sorted(cand.items(), key=lambda kv: (kv[1], kv[0]))[:need]
    edges += [e for e, _ in extra]
    return xy, edges


def synthetic_case(nbus: int, ngen: int, nbranch: int, seed: int, T: int = 24,
                   clusters: int = 1, binding_frac: float = 0.1, discount: float = 0.7,
                   vhi_thresh: float = 1.05, name: Optional[str] = None) -> Problem:
    """Deterministic IEEE-shaped UC-ACOPF instance with a planted peak AC power flow.

    Recipe: geometric spanning tree + shortest k-NN meshing; lines
    x = 0.01 + 0.25*len*U(.6,1.4), r = x*U(.05,.35), b = x*U(0,3); 15 % transformers;
    generators on high-degree buses, Pmax lognormal(200 MW, 0.8) clipped to [20,1000];
    loads local to generation (0.45 of total capacity); shunts at high-Q buses; a
    Newton-Raphson power flow at peak with a reinforcement loop; rates from the planted
    flows (binding_frac of them tight).  UC data per S:137-138 and P:465."""
    rng = SplitMix64(seed)
    base = 100.0
    nb, ng, nl = nbus, ngen, nbranch
    xy, edges = _topology(rng, nb, nl, clusters)
    nl = len(edges)
    fr = np.array([e[0] for e in edges])
    to = np.array([e[1] for e in edges])
    length = np.hypot(xy[fr, 0] - xy[to, 0], xy[fr, 1] - xy[to, 1])
    is_tr = np.array([rng.uniform() < 0.15 for _ in range(nl)])
    xs = np.zeros(nl)
    rs = np.zeros(nl)
    bs_ch = np.zeros(nl)
    tap = np.ones(nl)
    for k in range(nl):
        if is_tr[k]:
            xs[k] = rng.uniform(0.02, 0.2)
            tap[k] = rng.uniform(0.95, 1.05)
        else:
            xs[k] = 0.01 + 0.25 * length[k] * rng.uniform(0.6, 1.4)
            rs[k] = xs[k] * rng.uniform(0.05, 0.35)
            bs_ch[k] = xs[k] * rng.uniform(0.0, 3.0)
    deg = np.bincount(np.concatenate([fr, to]), minlength=nb)
    # generators on distinct buses, weighted by degree
    w = (deg + 1.0).astype(float)
    gb = []
    avail = np.ones(nb, dtype=bool)
    for _ in range(ng):
        ww = np.where(avail, w, 0.0)
        c = np.cumsum(ww)
        r = rng.uniform() * c[-1]
        b = int(np.searchsorted(c, r, side="right"))
        b = min(b, nb - 1)
        while not avail[b]:
            b = (b + 1) % nb
        gb.append(b)
        avail[b] = False
    gb = np.array(gb)
    pmax = np.array([min(max(200.0 * math.exp(0.8 * rng.normal()), 20.0), 1000.0) for _ in range(ng)]) / base
    pmin = pmax * np.array([rng.uniform(0.1, 0.4) for _ in range(ng)])
    qmax = 0.6 * pmax
    qmin = -0.4 * pmax
    lam = float(np.median(length[~is_tr])) if np.any(~is_tr) else 0.05
    # loads local to generation
    dist_bg = np.hypot(xy[:, None, 0] - xy[None, gb, 0], xy[:, None, 1] - xy[None, gb, 1])
    dens = (pmax[None, :] * np.exp(-dist_bg / lam)).sum(axis=1)
    has_load = np.array([rng.uniform() < 0.65 for _ in range(nb)])
    ln = np.array([math.exp(0.8 * rng.normal()) for _ in range(nb)])
    pd0 = np.where(has_load, ln * dens, 0.0)
    pd0 *= 0.45 * pmax.sum() / pd0.sum()
    qd0 = pd0 * np.array([rng.uniform(0.1, 0.35) for _ in range(nb)])
    gs = np.zeros(nb)
    bsh = np.zeros(nb)
    medq = np.median(qd0[has_load]) if np.any(has_load) else 0.0
    for i in range(nb):
        u = rng.uniform(0.3, 0.8)
        if has_load[i] and qd0[i] > medq:
            bsh[i] = qd0[i] * u
    ref = int(gb[int(np.argmax(pmax))])

    # local-balancing dispatch serving 1.03 x load
    wgt = pmax[None, :] * np.exp(-dist_bg / lam)
    share = (pd0[:, None] * wgt / wgt.sum(axis=1, keepdims=True)).sum(axis=0) * 1.03
    pg = np.clip(share, pmin, pmax)
    for _ in range(20):
        rem = 1.03 * pd0.sum() - pg.sum()
        if abs(rem) < 1e-9:
            break
        head = (pmax - pg) if rem > 0 else (pg - pmin)
        if head.sum() <= 0:
            break
        pg = np.clip(pg + rem * head / head.sum(), pmin, pmax)

    pv = np.array(sorted(set(gb.tolist()) - {ref}), dtype=int)
    pq = np.array(sorted(set(range(nb)) - set(gb.tolist())), dtype=int)
    scale = 1.0
    Vsol = None
    for _pass in range(25):
        y8 = np.array([branch_admittance(rs[k], xs[k], bs_ch[k], tap[k]) for k in range(nl)])
        Y = _ybus(nb, fr, to, y8, gs, bsh)
        sg = np.zeros(nb, dtype=complex)
        np.add.at(sg, gb, pg * scale)
        sbus = sg - scale * (pd0 + 1j * qd0)
        v0 = np.ones(nb, dtype=complex) * 1.0
        v0[gb] = 1.03
        V, ok = power_flow(Y, sbus, v0, ref, pv, pq)
        if not ok:
            scale *= 0.9
            continue
        Vm = np.abs(V)
        Va = np.angle(V)
        changed = False
        for i in pq:
            if Vm[i] < 0.96:
                bsh[i] += 0.5 * (0.99 - Vm[i]) * (1 + 4 * qd0[i] * scale)
                changed = True
            elif Vm[i] > vhi_thresh:
                bsh[i] -= 0.5 * (Vm[i] - 1.02) * (1 + 4 * qd0[i] * scale)
                changed = True
        dth = np.abs(Va[fr] - Va[to])
        for k in np.nonzero(dth > math.radians(25.0))[0]:
            xs[k] *= 0.7
            rs[k] *= 0.7
            changed = True
        Ibus = Y @ V
        sinj = V * np.conj(Ibus) + scale * (pd0 + 1j * qd0)
        for gi, b in enumerate(gb):
            qg = sinj[b].imag  # one generator per bus
            if qg > qmax[gi]:
                qmax[gi] = 1.2 * qg
                changed = True
            if qg < qmin[gi]:
                qmin[gi] = 1.2 * qg
                changed = True
        gref = int(np.nonzero(gb == ref)[0][0])
        pref = sinj[ref].real
        if pref > pmax[gref]:
            pmax[gref] = 1.1 * pref
            changed = True
        if pref < pmin[gref]:
            pmin[gref] = max(0.0, 0.9 * pref)
            changed = True
        Vsol = V
        if not changed:
            break
    if Vsol is None:
        raise RuntimeError("synthetic grid: power flow never converged")
    pd0 *= scale
    qd0 *= scale
    y8 = np.array([branch_admittance(rs[k], xs[k], bs_ch[k], tap[k]) for k in range(nl)])
    V = Vsol
    sf = V[fr] * np.conj(y8[:, 0] * V[fr] + 1j * y8[:, 4] * V[fr] + (y8[:, 1] + 1j * y8[:, 5]) * V[to])
    st = V[to] * np.conj((y8[:, 2] + 1j * y8[:, 6]) * V[fr] + (y8[:, 3] + 1j * y8[:, 7]) * V[to])
    smax = np.maximum(np.abs(sf), np.abs(st))
    rate = np.zeros(nl)
    for k in range(nl):
        if rng.uniform() < binding_frac:
            rate[k] = max(smax[k] * rng.uniform(1.05, 1.2), 0.05)
        else:
            rate[k] = max(smax[k] * rng.uniform(1.3, 2.5), 0.1)
    # costs and UC data
    c2 = np.array([rng.uniform(0.002, 0.05) for _ in range(ng)])
    c1 = np.array([rng.uniform(10.0, 40.0) for _ in range(ng)])
    c0 = np.array([rng.uniform(50.0, 600.0) for _ in range(ng)])
    csu = np.array([rng.uniform(100.0, 3000.0) for _ in range(ng)])
    csd = np.zeros(ng)
    min_up = np.array([rng.randint(1, 4) for _ in range(ng)])
    min_dn = np.array([rng.randint(1, 4) for _ in range(ng)])
    u0 = np.array([1 if rng.uniform() < 0.8 else 0 for _ in range(ng)])
    hold = np.array([rng.randint(0, 2) if (u0[g] == 1 and rng.uniform() < 0.3) else 0 for g in range(ng)])
    fac = diurnal_profile(T)
    pd = np.array([discount * fac[t] * pd0 for t in range(T)])
    qd = np.array([discount * fac[t] * qd0 for t in range(T)])
    sinj = V * np.conj(_ybus(nb, fr, to, y8, gs, bsh) @ V) + (pd0 + 1j * qd0)
    pplant = np.array([sinj[b].real for b in gb])
    p0 = np.where(u0 == 1, np.clip(pplant * discount * fac[0], pmin, pmax), 0.0)
    R = 0.1 * pmax
    sur = np.maximum(np.maximum(pmin, R), p0)
    return Problem(
        name=name or f"synth{nb}_T{T}_s{seed}", base_mva=base, ref_bus=ref,
        bus_gs=gs, bus_bs=bsh, bus_vmin=np.full(nb, 0.94), bus_vmax=np.full(nb, 1.06),
        pd=pd, qd=qd, br_from=fr, br_to=to, br_y=y8, br_rate=rate,
        gen_bus=gb, pmin=pmin, pmax=pmax, qmin=qmin, qmax=qmax,
        c2=c2, c1=c1, c0=c0, csu=csu, csd=csd,
        ramp_up=R.copy(), ramp_dn=R.copy(), su_ramp=sur.copy(), sd_ramp=sur.copy(),
        min_up=min_up, min_dn=min_dn, u0=u0, hold=hold, p0=p0, bus_xy=xy,
    ).normalized()


def random_problem(seed: int, nbus: int = 6, ngen: int = 3, nbranch: int = 8, T: int = 5) -> Problem:
    """small synthetic instance for parity tests (several tiles + ragged tails)."""
    return synthetic_case(nbus, ngen, nbranch, seed, T=T, name=f"rand{nbus}_T{T}_s{seed}")


# --------------------------------------------------------------------------------------
# BASELINE.json configs as concrete inputs
# --------------------------------------------------------------------------------------
CONFIGS = {
    # name: (builder kwargs, params, iterations)
    "case9": dict(kind="case9", T=4, rho=(5e3, 1e4, 1e4), iters=200),
    "case30": dict(kind="synth", nbus=30, ngen=6, nbranch=41, seed=30, T=24, rho=(5e3, 1e4, 1e4),
                   iters=20000, vhi=1.058),
    "case118": dict(kind="synth", nbus=118, ngen=54, nbranch=186, seed=118, T=24, rho=(5e3, 1e4, 1e4),
                    iters=1000),
    "case300": dict(kind="synth", nbus=300, ngen=69, nbranch=411, seed=300, T=24, rho=(5e3, 1e4, 1e4),
                    iters=1000),
    "pegase2869": dict(kind="synth", nbus=2869, ngen=510, nbranch=4582, seed=2869, T=48,
                       rho=(5e3, 1e4, 1e4), iters=200, clusters=6),
}


@functools.lru_cache(maxsize=8)
def build_config(name: str, T: Optional[int] = None):
    """(Problem, Params) for a BASELINE.json config."""
    c = CONFIGS[name]
    TT = T or c["T"]
    if c["kind"] == "case9":
        pb = case9(T=TT)
    else:
        pb = synthetic_case(c["nbus"], c["ngen"], c["nbranch"], c["seed"], T=TT,
                            clusters=c.get("clusters", 1), vhi_thresh=c.get("vhi", 1.05), name=name)
    rp, rv, ru = c["rho"]
    return pb, Params(rho_pq=rp, rho_va=rv, rho_uc=ru)


# ---------------------------------------------------------------------------------------------
# NEXT-1 workload (Fig. 1 shape): batches of independent UC DP instances with random
# stage costs.  Per generator and period, L(a, b) is the cost of being in state b at t after
# state a at t-1: L(0,0) = 0, L(1,1) = on-cost, L(0,1) = on-cost + start-up cost,
# L(1,0) = shut-down cost; min up/down times in [1, 8], initial state, held prefix in [0, 3].
# Plain data generation: no DP arithmetic here.
def dp_workload(G: int, T: int, seed: int = 1):
    rng = np.random.default_rng(seed)
    on = rng.uniform(-1.0, 1.0, (G, T)) + 0.3 * np.sin(np.linspace(0, 4 * np.pi, T))[None, :]
    csu = rng.uniform(0.0, 2.0, (G, 1))
    csd = rng.uniform(0.0, 0.5, (G, 1))
    L = np.zeros((G, T, 2, 2))
    L[:, :, 1, 1] = on
    L[:, :, 0, 1] = on + csu
    L[:, :, 1, 0] = csd
    tu = rng.integers(1, 9, G).astype(np.int32)
    td = rng.integers(1, 9, G).astype(np.int32)
    u0 = rng.integers(0, 2, G).astype(np.int32)
    hold = rng.integers(0, 4, G).astype(np.int32)
    hold = np.minimum(hold, T).astype(np.int32)
    return L, tu, td, u0, hold
