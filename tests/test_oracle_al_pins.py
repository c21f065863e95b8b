"""Pins of the oracle's (7a) stage cost and its (7c)/(7d) assembly against the augmented
Lagrangian written out from the paper (tests/al_model.py), at states with nonzero
y and z.

* (7a): the DP's stage costs L^UC_{g,t}(a, b) must reproduce, summed over a schedule, the
  change of the full L_{beta,rho} when only x^UC moves -- for random schedules, including every
  sign of the y (r + z) term.
* (7c), and (7d): after one oracle iteration, no feasible move of a ubar group
  inside [0,1]^3, and no move of a bus's copies along the null space of its two balance rows
  (Eq. 2a-2b), may lower L(x^{l+1}, xbar, z^l, y^l) -- block descent.  That pins
  which rows each group and bus assembles, their coefficients, the 2 rho_pq weight of a
  generator copy with a ramp-copy row and the n_i rho_va weight of wbar, and the targets.
"""
import dataclasses

import numpy as np
import pytest

import oracle
from paper_2310_13145_b200 import inputs

import al_model


def _run(name, iters, T=None):
    pb, pr = inputs.build_config(name)
    if T is not None:
        pb = pb.restricted(T)
    pb = pb.normalized()
    o = oracle.Oracle(pb, pr)
    o.iterate(iters)
    return pb, pr, o


def _states(name, iters, T=None):
    """(pb, pr, state at iterate l, state at l+1, slacks of x^{l+1})"""
    pb, pr, o = _run(name, iters, T)
    st0 = o.get_state()
    o.iterate(1)
    st1 = o.get_state()
    sl = o.slacks()
    o.close()
    return pb, pr, st0, st1, sl


# ------------------------------------------------------------------------------------ (7a)
@pytest.mark.parametrize("name,iters", [("case9", 30), ("case30", 12)])
def test_stage_cost_equals_full_al_difference(name, iters):
    """Sum_t L_t(u_{t-1}, u_t) over a schedule differs from the full AL at that schedule by a
    constant (the UC subproblem's objective is L restricted to x^UC).  Checked on the
    differences between random schedules, at a state with nonzero y and z."""
    pb, pr, o = _run(name, iters)
    st, sl = o.get_state(), o.slacks()
    o.close()
    G, T = pb.ngen, pb.T
    zg, yg = st["zg"].reshape(12, G, T), st["yg"].reshape(12, G, T)
    assert np.abs(yg[:3]).max() > 0 and np.abs(zg[:3]).max() > 0
    ub = np.stack([st["ub_on"], st["ub_su"], st["ub_sd"]]).reshape(3, G, T)
    rng = np.random.default_rng(7)
    checked = 0
    for g in range(G):
        L = oracle.stage_costs(T, pb.c0[g], pb.csu[g], pb.csd[g], pr.rho_uc, ub[:, g], yg[:3, g], zg[:3, g])
        scheds = [rng.integers(0, 2, T) for _ in range(6)] + [np.zeros(T, int), np.ones(T, int)]
        base = st["u"].reshape(G, T).copy()
        def dp_cost(u):
            prev, c = int(pb.u0[g]), 0.0
            for t in range(T):
                c += L[t, prev, int(u[t])]
                prev = int(u[t])
            return c
        ref_u = scheds[0]
        sa = dict(st)
        ua = base.copy()
        ua[g] = ref_u
        sa["u"] = ua.reshape(-1).astype(np.int8)
        for u in scheds[1:]:
            sb = dict(st)
            ub_ = base.copy()
            ub_[g] = u
            sb["u"] = ub_.reshape(-1).astype(np.int8)
            d_al = al_model.delta(pb, pr, sa, sb, sl)
            d_dp = dp_cost(u) - dp_cost(ref_u)
            scale = np.abs(L).max() * T
            assert abs(d_al - d_dp) <= 1e-11 * scale, (g, u, d_al, d_dp)
            checked += 1
    assert checked >= 7 * G


def test_stage_cost_pin_detects_sign_error():
    """Power of the pin above: a stage cost with the y (r + z) sign flipped, or without z in the
    penalty, disagrees with the AL difference (so the pin can see such a mistake)."""
    pb, pr, o = _run("case9", 30)
    st, sl = o.get_state(), o.slacks()
    o.close()
    G, T = pb.ngen, pb.T
    zg, yg = st["zg"].reshape(12, G, T), st["yg"].reshape(12, G, T)
    ub = np.stack([st["ub_on"], st["ub_su"], st["ub_sd"]]).reshape(3, G, T)
    g = int(np.argmax(np.abs(yg[0]).sum(axis=1)))
    base = st["u"].reshape(G, T).copy()
    u1, u2 = np.ones(T, int), np.zeros(T, int)

    def d_al():
        sa, sb = dict(st), dict(st)
        a, b = base.copy(), base.copy()
        a[g], b[g] = u1, u2
        sa["u"], sb["u"] = a.reshape(-1).astype(np.int8), b.reshape(-1).astype(np.int8)
        return al_model.delta(pb, pr, sa, sb, sl)

    def cost(L, u):
        prev, c = int(pb.u0[g]), 0.0
        for t in range(T):
            c += L[t, prev, int(u[t])]
            prev = int(u[t])
        return c
    good = oracle.stage_costs(T, pb.c0[g], pb.csu[g], pb.csd[g], pr.rho_uc, ub[:, g], yg[:3, g], zg[:3, g])
    flipped = oracle.stage_costs(T, pb.c0[g], pb.csu[g], pb.csd[g], pr.rho_uc, ub[:, g], -yg[:3, g], zg[:3, g])
    noz = oracle.stage_costs(T, pb.c0[g], pb.csu[g], pb.csd[g], pr.rho_uc, ub[:, g], yg[:3, g], 0 * zg[:3, g])
    ref = d_al()
    scale = 1e-11 * np.abs(good).max() * T
    assert abs(cost(good, u2) - cost(good, u1) - ref) <= scale
    assert abs(cost(flipped, u2) - cost(flipped, u1) - ref) > 1e3 * scale
    assert abs(cost(noz, u2) - cost(noz, u1) - ref) > 1e3 * scale


# ------------------------------------------------------------------------------------ (7c)
def _ubar_groups(G, T):
    """the (7c) groups as lists of (field, g, t): (ubar^on_t, ubar^sd_t, ubar^su_{t+1}) and
    group 0 = (ubar^su_1)"""
    out = []
    for g in range(G):
        out.append([("ub_su", g, 0)])
        for t in range(T):
            grp = [("ub_on", g, t), ("ub_sd", g, t)]
            if t < T - 1:
                grp.append(("ub_su", g, t + 1))
            out.append(grp)
    return out


def _descent_ubar(pb, pr, st0, st1, sl, eps_list=(1e-7, 1e-4, 1e-2), nrand=3, seed=0):
    """smallest AL change over feasible group moves, relative to the move's curvature scale"""
    G, T = pb.ngen, pb.T
    rng = np.random.default_rng(seed)
    kw = dict(z=st0, y=st0, lam=st0, beta=float(st0["scal"][0]))
    worst = np.inf
    for grp in _ubar_groups(G, T):
        n = len(grp)
        v0 = np.array([st1[f][g * T + t] for f, g, t in grp])
        dirs = [np.eye(n)[i] * s for i in range(n) for s in (1.0, -1.0)]
        dirs += [d / np.linalg.norm(d) for d in rng.normal(size=(nrand, n))]
        for d in dirs:
            for eps in eps_list:
                v = np.clip(v0 + eps * d, 0.0, 1.0)
                if np.array_equal(v, v0):
                    continue
                s2 = {k: (a.copy() if k in ("ub_on", "ub_su", "ub_sd") else a) for k, a in st1.items()}
                for (f, g, t), val in zip(grp, v):
                    s2[f][g * T + t] = val
                dl = al_model.delta(pb, pr, st1, s2, sl, **kw)
                # the group's Hessian is >= rho_uc I (its duplicate rows): a minimiser gains at
                # least rho_uc/2 |move|^2 -- allow a quarter of it to rounding
                gain = 0.25 * 0.5 * pr.rho_uc * float(np.sum((v - v0) ** 2))
                worst = min(worst, dl / gain)
    return worst


@pytest.mark.parametrize("name,iters,T", [("case9", 25, None), ("case30", 8, 12)])
def test_ubar_step_is_block_minimiser(name, iters, T):
    """(7c): ubar^{l+1} minimises L(x^{l+1}, ubar, z^l, y^l) over [0,1]: every feasible
    move of a group raises L by at least a quarter of the duplicate rows' curvature."""
    pb, pr, st0, st1, sl = _states(name, iters, T)
    assert _descent_ubar(pb, pr, st0, st1, sl) >= 1.0


def test_ubar_pin_detects_displacement():
    """Power of the pin: the oracle's ubar displaced by 1e-5 in one group fails it."""
    pb, pr, st0, st1, sl = _states("case9", 25)
    G, T = pb.ngen, pb.T
    bad = {k: a.copy() for k, a in st1.items()}
    k = 1 * T + 2
    bad["ub_on"][k] = np.clip(bad["ub_on"][k] + (1e-5 if bad["ub_on"][k] < 0.5 else -1e-5), 0, 1)
    assert _descent_ubar(pb, pr, st0, bad, sl, eps_list=(1e-7,), nrand=0) < 1.0


# ------------------------------------------------------------------------------------ (7d)
def _bus_vars(pb, i):
    """the bus-side copies of bus i: (field, index-in-field-array at t=0 minus t, alpha, beta);
    Eq. 2a: sum_g pbar_g - sum_ends pbar_end - G^s wbar = P_d, Eq. 2b: sum_g qbar_g -
    sum_ends qbar_end + B^s wbar = Q_d"""
    T = pb.T
    out = []
    for g in np.nonzero(pb.gen_bus == i)[0]:
        out.append(("pbar", lambda t, g=g: g * T + t, 1.0, 0.0))
        out.append(("qbar", lambda t, g=g: g * T + t, 0.0, 1.0))
    for l in range(pb.nbranch):
        for side, bus in ((0, pb.br_from[l]), (1, pb.br_to[l])):
            if bus == i:
                out.append(("fbar", lambda t, l=l, s=side: (l * T + t) * 4 + 2 * s, -1.0, 0.0))
                out.append(("fbar", lambda t, l=l, s=side: (l * T + t) * 4 + 2 * s + 1, 0.0, -1.0))
    out.append(("wbar", lambda t: i * T + t, -pb.bus_gs[i], pb.bus_bs[i]))
    return out


def _descent_bus(pb, pr, st0, st1, sl, buses, eps_list=(1e-7, 1e-4), seed=0):
    T = pb.T
    kw = dict(z=st0, y=st0, lam=st0, beta=float(st0["scal"][0]))
    worst, bal = np.inf, 0.0
    rho_min = min(pr.rho_pq, pr.rho_va)
    for i in buses:
        vs = _bus_vars(pb, i)
        N = np.array([[a for _, _, a, _ in vs], [b for _, _, _, b in vs]])
        _, sv, Vt = np.linalg.svd(N)
        basis = Vt[int(np.sum(sv > 1e-12 * sv.max())):]
        for t in range(T):
            v0 = np.array([st1[f][ix(t)] for f, ix, _, _ in vs])
            bal = max(bal, abs(N[0] @ v0 - pb.pd[t, i]), abs(N[1] @ v0 - pb.qd[t, i]))
            dirs = [s * b for b in basis for s in (1.0, -1.0)]
            for d in dirs:
                for eps in eps_list:
                    s2 = {k: (a.copy() if k in ("pbar", "qbar", "fbar", "wbar") else a) for k, a in st1.items()}
                    for (f, ix, _, _), dv in zip(vs, eps * d):
                        s2[f][ix(t)] += dv
                    dl = al_model.delta(pb, pr, st1, s2, sl, **kw)
                    gain = 0.25 * 0.5 * rho_min * eps * eps
                    worst = min(worst, dl / gain)
            if i != pb.ref_bus:   # thetabar is free except at the reference bus
                for s in (1.0, -1.0):
                    s2 = {k: (a.copy() if k == "thbar" else a) for k, a in st1.items()}
                    s2["thbar"][i * T + t] += s * 1e-6
                    dl = al_model.delta(pb, pr, st1, s2, sl, **kw)
                    worst = min(worst, dl / (0.25 * 0.5 * pr.rho_va * 1e-12))
    return worst, bal


@pytest.mark.parametrize("name,iters,T,nb", [("case9", 25, None, 9), ("case30", 8, 12, 30)])
def test_bus_step_is_block_minimiser(name, iters, T, nb):
    """(7d): the bus copies minimise L(x^{l+1}, xbar^OPF, z^l, y^l) subject to Eq. 2a-2b:
    no move along the null space of the balance rows lowers L, thetabar is stationary, and the
    balance rows hold."""
    pb, pr, st0, st1, sl = _states(name, iters, T)
    worst, bal = _descent_bus(pb, pr, st0, st1, sl, range(nb))
    assert worst >= 1.0, worst
    assert bal <= 1e-10, bal


def test_bus_pin_detects_displacement():
    """Power of the pin: the oracle's bus copies displaced by 1e-4 along a feasible direction
    (a generator copy and an incident end copy, the P balance kept) fail it."""
    pb, pr, st0, st1, sl = _states("case9", 25)
    T = pb.T
    bad = {k: a.copy() for k, a in st1.items()}
    # shift pbar of generator 0 at t=1 by 1e-4 and the same on an incident end's copy, which
    # keeps Eq. 2a: a feasible point that is not the minimiser
    g, t = 0, 1
    i = int(pb.gen_bus[g])
    l = int(np.nonzero((pb.br_from == i) | (pb.br_to == i))[0][0])
    side = 0 if pb.br_from[l] == i else 1
    bad["pbar"][g * T + t] += 1e-4
    bad["fbar"][(l * T + t) * 4 + 2 * side] += 1e-4
    worst, _ = _descent_bus(pb, pr, st0, bad, sl, [i], eps_list=(1e-7,))
    assert worst < 1.0
