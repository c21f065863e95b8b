"""Whole-iteration pins for the oracle's two-level ADMM (Alg. 1).

* (7e)/(7f) exactness: z^{l+1}, y^{l+1} of every row recomputed here from the rows of
  Eq. (5) (R3/R6/R7) evaluated on the state the oracle returned, and the z
  closed form checked against 1-D numerical minimisation of the row's L terms;
* the outer update: lambda <- clip(lambda + beta z), beta x tau iff
  ||z|| > theta ||z||_prev, tau = 6, theta = 0.8;
* MATPOWER case9 single-period ACOPF optimum (golden, 5296.69 $/h) and AC feasibility of
  the converged consensus point;
* Eq. 3 feasibility of every schedule, determinism."""
import dataclasses
import json
import os

import numpy as np
import pytest
from scipy.optimize import minimize_scalar

import oracle
from paper_2310_13145_b200 import inputs

from test_oracle_dp import feasible

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "case9_acopf.json")))
SPEC = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def rows_residual(pb, pr, s0, s1):
    """r = A x^{l+1} + B xbar^{l+1} per row (Eq. 5) from two consecutive states; slacks are
    the exact minimisers given the x-step's shifted bounds (built from s0)."""
    T, G, L = pb.T, pb.ngen, pb.nbranch
    rpq, rva, ruc = pr.rho_pq, pr.rho_va, pr.rho_uc
    zg0, yg0 = s0["zg"].reshape(12, G, T), s0["yg"].reshape(12, G, T)
    u = s1["u"].reshape(G, T).astype(float)
    p, q, ph = (s1[k].reshape(G, T) for k in ("p", "q", "ph"))
    on0, su0, sd0 = (s0[k].reshape(G, T) for k in ("ub_on", "ub_su", "ub_sd"))
    on1, su1, sd1 = (s1[k].reshape(G, T) for k in ("ub_on", "ub_su", "ub_sd"))
    pbar, qbar = s1["pbar"].reshape(G, T), s1["qbar"].reshape(G, T)
    rg = np.zeros((12, G, T))
    for g in range(G):
        for t in range(T):
            up = pb.u0[g] if t == 0 else u[g, t - 1]
            su, sd = max(0.0, u[g, t] - up), max(0.0, up - u[g, t])
            onp0 = pb.u0[g] if t == 0 else on0[g, t - 1]
            onp1 = pb.u0[g] if t == 0 else on1[g, t - 1]

            def b(k, v):
                return v - zg0[k, g, t] - yg0[k, g, t] / ruc
            bpl, bpu = b(3, pb.pmin[g] * on0[g, t]), b(4, pb.pmax[g] * on0[g, t])
            bql, bqu = b(5, pb.qmin[g] * on0[g, t]), b(6, pb.qmax[g] * on0[g, t])
            brl = b(7, -pb.ramp_dn[g] * on0[g, t] - pb.sd_ramp[g] * sd0[g, t])
            bru = b(8, pb.ramp_up[g] * onp0 + pb.su_ramp[g] * su0[g, t])
            d = p[g, t] - ph[g, t]
            spl, spu = max(0, p[g, t] - bpl), max(0, bpu - p[g, t])
            sql, squ = max(0, q[g, t] - bql), max(0, bqu - q[g, t])
            srd, sru = max(0, d - brl), max(0, bru - d)
            rg[0, g, t] = u[g, t] - on1[g, t]
            rg[1, g, t] = su - su1[g, t]
            rg[2, g, t] = sd - sd1[g, t]
            rg[3, g, t] = p[g, t] - spl - pb.pmin[g] * on1[g, t]
            rg[4, g, t] = p[g, t] + spu - pb.pmax[g] * on1[g, t]
            rg[5, g, t] = q[g, t] - sql - pb.qmin[g] * on1[g, t]
            rg[6, g, t] = q[g, t] + squ - pb.qmax[g] * on1[g, t]
            rg[7, g, t] = d - srd + pb.ramp_dn[g] * on1[g, t] + pb.sd_ramp[g] * sd1[g, t]  # Eq. 4d
            rg[8, g, t] = d + sru - pb.ramp_up[g] * onp1 - pb.su_ramp[g] * su1[g, t]
            rg[9, g, t] = p[g, t] - pbar[g, t]
            rg[10, g, t] = q[g, t] - qbar[g, t]
            rg[11, g, t] = 0.0 if t == 0 else ph[g, t] - pbar[g, t - 1]
    x, f, fb = s1["x"].reshape(L, T, 4), s1["f"].reshape(L, T, 4), s1["fbar"].reshape(L, T, 4)
    wb, tb = s1["wbar"].reshape(-1, T), s1["thbar"].reshape(-1, T)
    rb = np.zeros((8, L, T))
    for k in range(4):
        rb[k] = f[:, :, k] - fb[:, :, k]
    rb[4] = x[:, :, 0] - wb[pb.br_from]
    rb[5] = x[:, :, 1] - wb[pb.br_to]
    rb[6] = x[:, :, 2] - tb[pb.br_from]
    rb[7] = x[:, :, 3] - tb[pb.br_to]
    rhog = np.array([ruc] * 9 + [rpq] * 3)[:, None, None] * np.ones((12, G, T))
    rhob = np.array([rpq] * 4 + [rva] * 4)[:, None, None] * np.ones((8, L, T))
    return rg, rb, rhog, rhob


def test_z_y_updates_exact():
    pb = inputs.case9(T=4)
    pr = inputs.Params(rho_pq=5e3, rho_va=1e4, rho_uc=1e4, outer_enabled=0)
    o = oracle.Oracle(pb, pr)
    o.iterate(3)
    s0 = o.get_state()
    o.iterate(1)
    s1 = o.get_state()
    rg, rb, rhog, rhob = rows_residual(pb, pr, s0, s1)
    beta = s0["scal"][0]
    for r, rho, z0k, y0k, l0k, z1k, y1k, n in ((rg, rhog, "zg", "yg", "lg", "zg", "yg", 12),
                                               (rb, rhob, "zb", "yb", "lb", "zb", "yb", 8)):
        lam = s0[l0k].reshape(n, -1)
        y0 = s0[y0k].reshape(n, -1)
        z1 = s1[z1k].reshape(n, -1)
        y1 = s1[y1k].reshape(n, -1)
        r = r.reshape(n, -1)
        rho = rho.reshape(n, -1)
        zref = -(lam + y0 + rho * r) / (beta + rho)
        if n == 12:
            zref[11].reshape(pb.ngen, pb.T)[:, 0] = 0.0     # no RC row at t = 1
        assert np.allclose(z1, zref, rtol=1e-9, atol=1e-11)
        yref = y0 + rho * (r + z1)
        if n == 12:
            yref[11].reshape(pb.ngen, pb.T)[:, 0] = y0[11].reshape(pb.ngen, pb.T)[:, 0]
        assert np.allclose(y1, yref, rtol=1e-9, atol=1e-9)
    # the closed form is the argmin of lambda z + beta/2 z^2 + y(r+z) + rho/2 (r+z)^2 (7e)
    for k in range(5):
        lam, y, rho, r = 0.3 * k, 1.0 - k, 1e4, 1e-3 * (k - 2)
        z = -(lam + y + rho * r) / (beta + rho)
        res = minimize_scalar(lambda v: lam * v + beta / 2 * v * v + y * (r + v) + rho / 2 * (r + v) ** 2,
                              bracket=(-1, 1), tol=1e-14)
        assert z == pytest.approx(res.x, abs=1e-9)
    g = SPEC["z_update"]
    assert -(g["lambda"] + g["y"] + g["rho"] * g["r"]) / (g["beta"] + g["rho"]) == pytest.approx(g["z"], rel=1e-15)


def test_outer_update_rule():
    pb = inputs.case9(T=4)
    pr = inputs.Params(rho_pq=5e3, rho_va=1e4, rho_uc=1e4)
    o = oracle.Oracle(pb, pr)
    seen = 0
    prev = o.get_state()
    for _ in range(200):
        o.iterate(1)
        cur = o.get_state()
        b0, b1 = prev["scal"][0], cur["scal"][0]
        k0, k1 = prev["scal"][2], cur["scal"][2]
        if k1 != k0:
            seen += 1
            assert k1 == k0 + 1
            for zk, lk in (("zg", "lg"), ("zb", "lb")):
                ref = np.clip(prev[lk] + b0 * cur[zk], -pr.lambda_max, pr.lambda_max)
                assert np.allclose(cur[lk], ref, rtol=1e-15, atol=0)
            zn = np.sqrt(np.sum(cur["zg"] ** 2) + np.sum(cur["zb"] ** 2))
            if k0 > 1 and zn > pr.theta * prev["scal"][1] * (1 + 1e-12):
                assert b1 == min(pr.tau * b0, pr.beta_max)
            elif k0 == 1 or zn < pr.theta * prev["scal"][1] * (1 - 1e-12):
                assert b1 == b0
            assert cur["scal"][1] == pytest.approx(zn, rel=1e-12)
        else:
            assert b1 == b0 and np.array_equal(cur["lg"], prev["lg"])
        prev = cur
    assert seen >= 3


def test_case9_acopf_optimum():
    """T=1, all units forced on (hold = 1), discount 1, no ramps -> MATPOWER optimum."""
    pb = inputs.case9(T=1, factors=[1.0], discount=1.0, ramps=False)
    pb.hold[:] = 1
    assert pb.pd.sum() * pb.base_mva == pytest.approx(GOLD["total_load_mw"])
    assert pb.qd.sum() * pb.base_mva == pytest.approx(GOLD["total_load_mvar"])
    pr = inputs.Params(rho_pq=5e3, rho_va=1e4, rho_uc=1e4)
    o = oracle.Oracle(pb, pr)
    o.iterate(1000)
    rep = o.report()
    assert rep["primal_inf"] < 1e-5
    assert rep["objective"] == pytest.approx(GOLD["objective"], abs=0.01)
    st = o.get_state()
    assert np.allclose(st["p"] * pb.base_mva, GOLD["pg_mw"], atol=0.02)
    # AC feasibility of the consensus point: V = sqrt(wbar) e^{j thbar}, S = V conj(Ybus V)
    V = np.sqrt(st["wbar"]) * np.exp(1j * st["thbar"])
    S = np.zeros(pb.nbus, dtype=complex)
    for l in range(pb.nbranch):
        y = pb.br_y[l]
        i, j = pb.br_from[l], pb.br_to[l]
        S[i] += V[i] * np.conj((y[0] + 1j * y[4]) * V[i] + (y[1] + 1j * y[5]) * V[j])
        S[j] += V[j] * np.conj((y[2] + 1j * y[6]) * V[i] + (y[3] + 1j * y[7]) * V[j])
    inj = np.zeros(pb.nbus, dtype=complex)
    np.add.at(inj, pb.gen_bus, st["pbar"] + 1j * st["qbar"])
    inj -= pb.pd[0] + 1j * pb.qd[0]
    assert np.max(np.abs(S - inj)) < 100 * rep["primal_inf"] + 1e-9
    assert np.all(st["wbar"] >= pb.bus_vmin ** 2 - 1e-4) and np.all(st["wbar"] <= pb.bus_vmax ** 2 + 1e-4)


def test_case9_uc_schedules_and_determinism():
    pb, pr = inputs.build_config("case9")
    a = oracle.Oracle(pb, pr)
    b = oracle.Oracle(pb, pr)
    for _ in range(20):
        a.iterate(10)
        b.iterate(10)
        sa, sb = a.get_state(), b.get_state()
        for k in sa:
            assert np.array_equal(sa[k], sb[k]), k
        u = sa["u"].reshape(pb.ngen, pb.T)
        for g in range(pb.ngen):
            assert feasible(list(u[g]), int(pb.u0[g]), int(pb.min_up[g]), int(pb.min_dn[g]), int(pb.hold[g]))
    rep = a.report()
    assert rep["inner_total"] == 200
    assert rep["primal_inf"] < 5e-2


def test_dp_switching_instance():
    """SURVEY 8(d) #1b: an expensive unit whose commitment the DP switches off."""
    pb = inputs.case9(T=6, factors=[0.6, 0.7, 1, 1, 0.7, 0.6], discount=0.5)
    pb.c0[2] = 5000.0
    pb.sd_ramp[:] = pb.pmax
    pr = inputs.Params(rho_pq=5e3, rho_va=1e4, rho_uc=3e3)
    o = oracle.Oracle(pb, pr)
    o.iterate(400)
    st = o.get_state()
    u = st["u"].reshape(pb.ngen, pb.T)
    assert u[2].sum() == 0 and u[0].sum() == pb.T
    assert o.report()["primal_inf"] < 1e-3


def test_consensus_fixed_point():
    """A converged point is (numerically) a fixed point of one more sweep."""
    pb = inputs.case9(T=1, factors=[1.0], discount=1.0, ramps=False)
    pb.hold[:] = 1
    pr = inputs.Params(rho_pq=5e3, rho_va=1e4, rho_uc=1e4)
    o = oracle.Oracle(pb, pr)
    o.iterate(1500)
    s0 = o.get_state()
    o.iterate(1)
    s1 = o.get_state()
    res = o.report()["primal_inf"]
    assert res < 1e-5
    for k in ("p", "q", "pbar", "qbar", "wbar", "x", "f"):
        assert np.allclose(s0[k], s1[k], atol=100 * res), k


def test_variant_wbar_clip_keeps_voltage_box():
    """NEXT-3 variant 2 (R47): with SPEC's clip every bus copy w-bar lies in [Vmin^2, Vmax^2];
    without it the exact bus QP may leave the box (A8)."""
    import dataclasses
    pb, pr = inputs.build_config("case30")
    o = oracle.Oracle(pb, dataclasses.replace(pr, variant=2))
    o.iterate(15)
    w = o.get_state()["wbar"].reshape(pb.nbus, pb.T)
    lo, hi = (pb.bus_vmin ** 2)[:, None], (pb.bus_vmax ** 2)[:, None]
    assert np.all(w >= lo) and np.all(w <= hi)


def test_variant_al_always_every_rated_branch_takes_the_al():
    """NEXT-3 variant 1 (R47): every rated (l,t) solves the AL each iteration."""
    import dataclasses
    pb, pr = inputs.build_config("case30")
    o = oracle.Oracle(pb, dataclasses.replace(pr, variant=1))
    o.iterate(2)
    rated = int(np.sum(pb.br_rate > 0)) * pb.T
    assert o.report()["al_active"] == 2 * rated


def _ulp_response(pr, iters=2, seed=0):
    pb = inputs.build_config("case30")[0]
    o = oracle.Oracle(pb, pr)
    o.iterate(iters)
    st = o.get_state()
    o.close()
    rng = np.random.default_rng(seed)
    pert = {k: (v * (1 + rng.choice([-1.0, 1.0], v.shape) * 2.0 ** -52) if v.dtype == np.float64 and k != "scal" else v)
            for k, v in st.items()}
    xs = []
    for s in (st, pert):
        a = oracle.Oracle(pb, pr)
        a.set_state(s)
        a.iterate(1)
        xs.append(a.get_state()["x"].reshape(-1, 4))
        a.close()
    scale = np.maximum(np.abs(xs[0]), np.sqrt(np.mean(xs[0] ** 2, axis=0)))
    return float(np.max(np.abs(xs[1] - xs[0]) / scale))


def test_variant1_conditioning():
    """DESIGN.md 10 / R47: the oracle's own response to a one-ulp perturbation of its input state
    is at rounding level for the default formulation and bounded (<= 1e-8) for variant 1, whose
    slack-form AL of inactive lines is ill-conditioned.  The GPU parity tolerance for variant 1 is
    10x this measured response, so this pins that it cannot hide a default-path error."""
    import dataclasses
    pr = inputs.build_config("case30")[1]
    r0 = _ulp_response(pr)
    r1 = _ulp_response(dataclasses.replace(pr, variant=1))
    assert r0 < 1e-13, r0
    assert 1e-13 < r1 < 1e-8, r1


def _shutdowns_above_sd(pb, pr, iters):
    """(violations, shutdowns): shutdowns at t whose previous-iterate dispatch p_{t-1} exceeds S^D."""
    import dataclasses  # noqa: F401
    q = pb.normalized()
    G, T = q.ngen, q.T
    o = oracle.Oracle(pb, pr)
    viol = shut = 0
    for _ in range(iters):
        p = o.get_state()["p"].reshape(G, T).copy()
        o.iterate(1)
        u = o.get_state()["u"].reshape(G, T)
        for g in range(G):
            for t in range(T):
                prev_on = q.u0[g] if t == 0 else u[g, t - 1]
                if prev_on == 1 and u[g, t] == 0:
                    shut += 1
                    pprev = q.p0[g] if t == 0 else p[g, t - 1]
                    viol += pprev > q.sd_ramp[g]
    o.close()
    return viol, shut


def test_ramp_aware_dp_next4():
    """NEXT-4(a), R50 (variant bit 4): no DP schedule shuts a unit down at t while its current
    dispatch p_{t-1} (or p_0) exceeds the shutdown ramp S^D -- the Eq. 4d-infeasible transition
    of SURVEY A5.  Scenario: case30 with S^D = Pmin/2, where the default formulation takes such
    transitions (71 in 300 iterations) and the ramp-aware DP takes none but still shuts units down."""
    import dataclasses
    pb, pr = inputs.build_config("case30")
    pb = dataclasses.replace(pb, sd_ramp=pb.pmin * 0.5)
    v4, s4 = _shutdowns_above_sd(pb, dataclasses.replace(pr, variant=4), 300)
    v0, s0 = _shutdowns_above_sd(pb, pr, 300)
    assert v4 == 0 and s4 > 0, (v4, s4)
    assert v0 > 0, (v0, s0)


def test_no_angle_consensus_variant_next3():
    """NEXT-3 variant 8 (R51): without angle consensus rows the A_I/A_J rows keep
    z = y = lambda = 0, thetabar stays at its start value, every line keeps its own reference
    theta_i = 0, and a line's solution does not depend on the angle targets tau_6, tau_7."""
    import dataclasses
    pb, pr = inputs.build_config("case30")
    pr8 = dataclasses.replace(pr, variant=8)
    o = oracle.Oracle(pb, pr8)
    o.iterate(60)
    st = o.get_state()
    LT = pb.nbranch * pb.T
    zb, yb, lb = (st[k].reshape(8, LT) for k in ("zb", "yb", "lb"))
    assert np.all(zb[6:] == 0) and np.all(yb[6:] == 0) and np.all(lb[6:] == 0)
    assert np.all(st["thbar"] == 0)
    x = st["x"].reshape(LT, 4)
    assert np.all(x[:, 2] == 0) and np.any(x[:, 3] != 0)
    assert o.report()["outer_total"] >= 1
    o.close()
    # angle targets do not enter the line problem
    rng = np.random.default_rng(5)
    y = pb.br_y[0]
    xs = np.array([1.0, 0.98, 0.0, -0.05])
    tau = np.concatenate([oracle.branch_flows(y, xs)[0] * 1.1, xs])
    tau2 = tau.copy()
    tau2[6:] += rng.normal(size=2)
    a = oracle.branch_solve(y, [0.81, 0.81], [1.21, 1.21], 0.0, tau, pr.rho_pq, pr.rho_va, pr8, xs.copy(), np.zeros(3))
    b = oracle.branch_solve(y, [0.81, 0.81], [1.21, 1.21], 0.0, tau2, pr.rho_pq, pr.rho_va, pr8, xs.copy(), np.zeros(3))
    assert np.array_equal(a[0], b[0]) and a[0][2] == 0.0
    c = oracle.branch_solve(y, [0.81, 0.81], [1.21, 1.21], 0.0, tau2, pr.rho_pq, pr.rho_va, pr, xs.copy(), np.zeros(3))
    assert not np.array_equal(a[0], c[0])



def test_literal_eq5f_ramp_down_next3():
    """NEXT-3 variant 16 (R52): the ramp-down row is the literal Eq. 5f,
    (p_t - p^_t) - s + R_D ubar^on_{t-1} + S_D ubar^su_t, instead of Eq. 4d.
    Pins, one iteration from a mid-run state:
    * the RD row residual recovered from the y update, r = (y+ - y)/rho - z+, equals the
      literal row evaluated on the new iterate (slack from the x-step's bound on the old ubar);
    * ubar^sd is in no physical row any more, so (7c) gives it the projection of its duplicate
      row's target: clip(u^sd + z + y/rho, 0, 1)."""
    import dataclasses
    pb, pr = inputs.build_config("case30")
    pr16 = dataclasses.replace(pr, variant=16, outer_enabled=0)
    q = pb.normalized()
    G, T = q.ngen, q.T
    o = oracle.Oracle(pb, pr16)
    o.iterate(25)
    s0 = o.get_state()
    o.iterate(1)
    s1 = o.get_state()
    o.close()
    ruc = pr.rho_uc
    RD, DSD = 7, 2
    z0, y0 = s0["zg"].reshape(12, G, T), s0["yg"].reshape(12, G, T)
    z1, y1 = s1["zg"].reshape(12, G, T), s1["yg"].reshape(12, G, T)
    on0, su0 = s0["ub_on"].reshape(G, T), s0["ub_su"].reshape(G, T)
    on1, su1, sd1 = (s1[k].reshape(G, T) for k in ("ub_on", "ub_su", "ub_sd"))
    u1 = s1["u"].reshape(G, T)
    dd = (s1["p"] - s1["ph"]).reshape(G, T)
    worst = 0.0
    for g in range(G):
        for t in range(T):
            onp0 = q.u0[g] if t == 0 else on0[g, t - 1]
            onp1 = q.u0[g] if t == 0 else on1[g, t - 1]
            brl = -q.ramp_dn[g] * onp0 - q.sd_ramp[g] * su0[g, t] - z0[RD, g, t] - y0[RD, g, t] / ruc
            s4 = max(0.0, dd[g, t] - brl)
            r_lit = (dd[g, t] - s4) + q.ramp_dn[g] * onp1 + q.sd_ramp[g] * su1[g, t]
            r_y = (y1[RD, g, t] - y0[RD, g, t]) / ruc - z1[RD, g, t]
            worst = max(worst, abs(r_lit - r_y))
            up = q.u0[g] if t == 0 else u1[g, t - 1]
            sd = float(up > u1[g, t])
            assert abs(sd1[g, t] - np.clip(sd + z0[DSD, g, t] + y0[DSD, g, t] / ruc, 0.0, 1.0)) <= 1e-12
    assert worst <= 1e-9, worst


def test_set_rho_equals_fresh_context_next4():
    """NEXT-4(b), R53: orc_set_rho between iterations is the same as a context created with the
    new rho and handed the current state (every rho-derived quantity is formed at its use)."""
    import dataclasses
    pb, pr = inputs.build_config("case30")
    a = oracle.Oracle(pb, pr)
    a.iterate(7)
    st = a.get_state()
    a.set_rho(2 * pr.rho_pq, 0.5 * pr.rho_va, 3 * pr.rho_uc)
    a.iterate(3)
    b = oracle.Oracle(pb, dataclasses.replace(pr, rho_pq=2 * pr.rho_pq, rho_va=0.5 * pr.rho_va, rho_uc=3 * pr.rho_uc))
    b.set_state(st)
    b.iterate(3)
    sa, sb = a.get_state(), b.get_state()
    for k in sa:
        assert np.array_equal(sa[k], sb[k]), k
    a.close()
    b.close()


def test_openmp_build_is_bitwise_the_serial_oracle():
    """the all-core oracle (liboracle_omp.so, the same source with -fopenmp,
    per-component loops in parallel, reductions sequential in the canonical order) produces the
    single-thread oracle's iterates bit for bit."""
    import oracle
    from paper_2310_13145_b200 import inputs
    pb, pr = inputs.build_config("case30")
    a, b = oracle.Oracle(pb, pr), oracle.Oracle(pb, pr, omp=True)
    oracle.threads(4)
    a.iterate(25)
    b.iterate(25)
    sa, sb = a.get_state(), b.get_state()
    assert all(sa[k].tobytes() == sb[k].tobytes() for k in sa)
    assert a.report() == b.report()
