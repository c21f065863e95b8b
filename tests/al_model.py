"""The augmented Lagrangian of the two-level ADMM written out from the paper, row by row.

An independent model for the `-m "not gpu"` pins of the oracle's steps (7a), (7c) and (7d): it is
written from the paper's definitions, not from oracle.c, and shares nothing with it but the
state layout.

  L_{beta,rho}(x, xbar, z, y, lambda)
    = sum_t f^OPF_t + f^UC + lambda'z + beta/2 |z|^2 + sum_rows [ y (r + z) + rho/2 (r + z)^2 ],
  r = A x + B xbar, one entry per coupling row:
    x^UC - xbar^UC                          (Eq. 5a)            rho_uc   D_ON, D_SU, D_SD
    p -/+ s - Pmin/Pmax ubar^on                rho_uc   PL, PU
    q -/+ s - Qmin/Qmax ubar^on                rho_uc   QL, QU
    p_t - p_{t-1} - s + R^D ubar^on_t + S^D ubar^sd_t   (Eq. 4d form, R3)  rho_uc   RD
    p_t - p_{t-1} + s - R^U ubar^on_{t-1} - S^U ubar^su_t     rho_uc   RU
    component consensus (A_3 x + B_3 xbar, R7): p - pbar, q - qbar,
      phat_t - pbar_{t-1} (the ramp copy, R6), flows - fbar, w - wbar, theta - thetabar
                                            rho_pq (p, q, flows) / rho_va (w, theta)   (R32)
  f^OPF = c2 (S p)^2 + c1 S p, f^UC = c0 u^on + C^SU u^su + C^SD u^sd (R13),
  u^su_t = max(0, u_t - u_{t-1}), u^sd_t = max(0, u_{t-1} - u_t) with u_0 = u0 (R4).

`terms(...)` returns every row's contribution separately, so a pin can difference two states
row by row without the cancellation error of two large sums.
"""
from __future__ import annotations

import numpy as np

GEN_KINDS = ["D_ON", "D_SU", "D_SD", "PL", "PU", "QL", "QU", "RD", "RU", "GP", "GQ", "RC"]
BR_KINDS = ["FP_IJ", "FQ_IJ", "FP_JI", "FQ_JI", "W_I", "W_J", "A_I", "A_J"]


def switching(u, u0):
    """(su, sd) [G, T] inferred from u^on [G, T] and the initial state."""
    prev = np.concatenate([np.asarray(u0, float)[:, None], u[:, :-1]], axis=1)
    return np.maximum(0.0, u - prev), np.maximum(0.0, prev - u)


def gen_rows(pb, st, sl):
    """r for the 12 generator row kinds, [12, G, T] (RC at t = 1 does not exist: 0 there)."""
    G, T = pb.ngen, pb.T
    sh = lambda k: np.asarray(st[k], float).reshape(G, T)
    u = np.asarray(st["u"], float).reshape(G, T)
    su, sd = switching(u, pb.u0)
    on, usu, usd = sh("ub_on"), sh("ub_su"), sh("ub_sd")
    p, q, ph, pbar, qbar = sh("p"), sh("q"), sh("ph"), sh("pbar"), sh("qbar")
    s = np.asarray(sl, float).reshape(G, T, 6)
    on_prev = np.concatenate([np.asarray(pb.u0, float)[:, None], on[:, :-1]], axis=1)
    col = lambda a: np.asarray(a, float)[:, None]
    d = p - ph
    r = np.zeros((12, G, T))
    r[0] = u - on
    r[1] = su - usu
    r[2] = sd - usd
    r[3] = p - s[..., 0] - col(pb.pmin) * on
    r[4] = p + s[..., 1] - col(pb.pmax) * on
    r[5] = q - s[..., 2] - col(pb.qmin) * on
    r[6] = q + s[..., 3] - col(pb.qmax) * on
    r[7] = d - s[..., 4] + col(pb.ramp_dn) * on + col(pb.sd_ramp) * usd
    r[8] = d + s[..., 5] - col(pb.ramp_up) * on_prev - col(pb.su_ramp) * usu
    r[9] = p - pbar
    r[10] = q - qbar
    r[11, :, 1:] = ph[:, 1:] - pbar[:, :-1]
    return r


def branch_rows(pb, st):
    """r for the 8 branch row kinds, [8, L, T]."""
    L, T = pb.nbranch, pb.T
    x = np.asarray(st["x"], float).reshape(L, T, 4)
    f = np.asarray(st["f"], float).reshape(L, T, 4)
    fb = np.asarray(st["fbar"], float).reshape(L, T, 4)
    wb = np.asarray(st["wbar"], float).reshape(pb.nbus, T)
    tb = np.asarray(st["thbar"], float).reshape(pb.nbus, T)
    i, j = np.asarray(pb.br_from), np.asarray(pb.br_to)
    r = np.zeros((8, L, T))
    for k in range(4):
        r[k] = f[..., k] - fb[..., k]
    r[4] = x[..., 0] - wb[i]
    r[5] = x[..., 1] - wb[j]
    r[6] = x[..., 2] - tb[i]
    r[7] = x[..., 3] - tb[j]
    return r


def terms(pb, pr, st, sl, z=None, y=None, lam=None, beta=None):
    """Per-row and per-(g,t) cost contributions of L_{beta,rho}.

    z, y, lambda default to the state's own; pass the iterate-l values to evaluate a step of
    iteration l (the x-bar steps use z^l, y^l).  Returns (gen [12,G,T], branch [8,L,T],
    cost [G,T]); the AL is the sum of all three."""
    G, T, L = pb.ngen, pb.T, pb.nbranch
    z = st if z is None else z
    y = st if y is None else y
    lam = st if lam is None else lam
    beta = float(st["scal"][0]) if beta is None else beta
    rg, rb = gen_rows(pb, st, sl), branch_rows(pb, st)
    rho_g = np.array([pr.rho_uc] * 9 + [pr.rho_pq] * 3)[:, None, None]
    rho_b = np.array([pr.rho_pq] * 4 + [pr.rho_va] * 4)[:, None, None]

    def rowterm(r, zz, yy, ll, rho):
        v = r + zz
        return ll * zz + 0.5 * beta * zz * zz + yy * v + 0.5 * rho * v * v

    zg =np.asarray(z["zg"], float).reshape(12, G, T)
    yg = np.asarray(y["yg"], float).reshape(12, G, T)
    lg = np.asarray(lam["lg"], float).reshape(12, G, T)
    zb = np.asarray(z["zb"], float).reshape(8, L, T)
    yb = np.asarray(y["yb"], float).reshape(8, L, T)
    lb = np.asarray(lam["lb"], float).reshape(8, L, T)
    tg = rowterm(rg, zg, yg, lg, rho_g)
    tg[11, :, 0] = 0.0                         # no RC row at the first period
    tb = rowterm(rb, zb, yb, lb, rho_b)
    u = np.asarray(st["u"], float).reshape(G, T)
    su, sd = switching(u, pb.u0)
    Sp = pb.base_mva * np.asarray(st["p"], float).reshape(G, T)
    col = lambda a: np.asarray(a, float)[:, None]
    cost = col(pb.c2) * Sp * Sp + col(pb.c1) * Sp + col(pb.c0) * u + col(pb.csu) * su + col(pb.csd) * sd
    return tg, tb, cost


def total(pb, pr, st, sl, **kw):
    tg, tb, c = terms(pb, pr, st, sl, **kw)
    return float(np.sum(tg) + np.sum(tb) + np.sum(c))


def delta(pb, pr, st_a, st_b, sl, **kw):
    """L(st_b) - L(st_a), differenced row by row (no cancellation of the unchanged rows)."""
    a, b = terms(pb, pr, st_a, sl, **kw), terms(pb, pr, st_b, sl, **kw)
    return float(sum(np.sum(y - x) for x, y in zip(a, b)))
