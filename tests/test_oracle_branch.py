"""Pins for oracle S3: branch flows (Eq. 2e-2j), the TRON solver and the branch solve
(7b line part, "six variables", P:456 ExaTron).

Independent references: complex power S = V conj(Y V) of the MATPOWER pi-model, torch
autograd (fp64) for first and second derivatives, SciPy BVLS for box QPs, a planted exact
power-flow point, and a dense grid search for a binding thermal limit (Eq. 2c-2d)."""
import dataclasses

import numpy as np
import pytest
import torch
from scipy.optimize import lsq_linear

import oracle
from paper_2310_13145_b200 import inputs

TWO_PI = 2 * np.pi


def flows_complex(y, x):
    wi, wj, ti, tj = x
    Vi = np.sqrt(wi) * np.exp(1j * ti)
    Vj = np.sqrt(wj) * np.exp(1j * tj)
    yff, yft = y[0] + 1j * y[4], y[1] + 1j * y[5]
    ytf, ytt = y[2] + 1j * y[6], y[3] + 1j * y[7]
    sij = Vi * np.conj(yff * Vi + yft * Vj)
    sji = Vj * np.conj(ytf * Vi + ytt * Vj)
    return np.array([sij.real, sij.imag, sji.real, sji.imag])


def flows_torch(y, x):
    wi, wj, ti, tj = x[0], x[1], x[2], x[3]
    vi, vj = torch.sqrt(wi), torch.sqrt(wj)
    # V_i = vi e^{j ti}; write complex products out in real arithmetic
    yffr, yftr, ytfr, yttr, yffi, yfti, ytfi, ytti = [float(v) for v in y]
    Vir, Vii = vi * torch.cos(ti), vi * torch.sin(ti)
    Vjr, Vji = vj * torch.cos(tj), vj * torch.sin(tj)

    def cm(ar, ai, br, bi):
        return ar * br - ai * bi, ar * bi + ai * br
    Iir = cm(yffr, yffi, Vir, Vii)[0] + cm(yftr, yfti, Vjr, Vji)[0]
    Iii = cm(yffr, yffi, Vir, Vii)[1] + cm(yftr, yfti, Vjr, Vji)[1]
    Ijr = cm(ytfr, ytfi, Vir, Vii)[0] + cm(yttr, ytti, Vjr, Vji)[0]
    Iji = cm(ytfr, ytfi, Vir, Vii)[1] + cm(yttr, ytti, Vjr, Vji)[1]
    sij = cm(Vir, Vii, Iir, -Iii)
    sji = cm(Vjr, Vji, Ijr, -Iji)
    return torch.stack([sij[0], sij[1], sji[0], sji[1]])


def test_admittance_symmetric_and_ybus():
    """tap = 1, shift = 0 -> symmetric two-port; tap/shift vs a dense Y-bus."""
    y = inputs.branch_admittance(0.01, 0.1, 0.02)
    assert y[1] == y[2] and y[5] == y[6]
    r, x, b, tap, sh = 0.02, 0.08, 0.03, 1.04, 5.0
    y = inputs.branch_admittance(r, x, b, tap, sh)
    ys = 1 / complex(r, x)
    a = tap * np.exp(1j * np.radians(sh))
    # textbook: I_f = (ys + jb/2)/|a|^2 V_f - ys/conj(a) V_t ; I_t = -ys/a V_f + (ys + jb/2) V_t
    Vf, Vt = 1.02 * np.exp(0.1j), 0.97 * np.exp(-0.05j)
    If = (ys + 1j * b / 2) / abs(a) ** 2 * Vf - ys / np.conj(a) * Vt
    It = -ys / a * Vf + (ys + 1j * b / 2) * Vt
    f = flows_complex(y, [abs(Vf) ** 2, abs(Vt) ** 2, np.angle(Vf), np.angle(Vt)])
    assert np.allclose(f, [(Vf * np.conj(If)).real, (Vf * np.conj(If)).imag,
                           (Vt * np.conj(It)).real, (Vt * np.conj(It)).imag], atol=1e-12)


def test_flows_and_derivatives():
    rng = np.random.default_rng(1)
    for _ in range(50):
        y = inputs.branch_admittance(rng.uniform(0, 0.05), rng.uniform(0.02, 0.3), rng.uniform(0, 0.3),
                                     rng.uniform(0.95, 1.05), rng.uniform(-5, 5))
        x = np.array([rng.uniform(0.8, 1.2), rng.uniform(0.8, 1.2), rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5)])
        f, J, H = oracle.branch_flows(y, x)
        assert np.allclose(f, flows_complex(y, x), atol=1e-12)
        xt = torch.tensor(x, dtype=torch.float64, requires_grad=True)
        Jt = torch.autograd.functional.jacobian(lambda v: flows_torch(y, v), xt).numpy()
        assert np.allclose(J, Jt, atol=1e-10)
        for k in range(4):
            Hk = torch.autograd.functional.hessian(lambda v: flows_torch(y, v)[k], xt).numpy()
            assert np.allclose(H[k], Hk, atol=1e-10)
    # flat start identities: w_i = w_j = 1, theta_i = theta_j -> C = 1, S = 0
    y = inputs.branch_admittance(0.0, 0.1, 0.0)
    f, _, _ = oracle.branch_flows(y, np.array([1.0, 1.0, 0.2, 0.2]))
    assert np.allclose(f, 0.0, atol=1e-12)


def test_tron_on_box_qps():
    """TRON on random convex box QPs (n <= 8) matches BVLS."""
    rng = np.random.default_rng(9)
    for _ in range(200):
        n = int(rng.integers(1, 9))
        M = rng.normal(size=(n + 2, n))
        A = M.T @ M + 0.1 * np.eye(n)
        b = rng.normal(size=n) * 3
        lo = -rng.uniform(0, 1, n)
        hi = rng.uniform(0, 1, n)
        x, it = oracle.tron_quadratic(A, b, lo, hi, np.zeros(n), gtol=1e-11, maxit=300)
        assert it >= 0
        Lc = np.linalg.cholesky(A)
        ref = lsq_linear(Lc.T, -np.linalg.solve(Lc, b), bounds=(lo, hi), method="bvls", tol=1e-15).x
        fo = 0.5 * x @ A @ x + b @ x
        fr = 0.5 * ref @ A @ ref + b @ ref
        assert fo <= fr + 1e-9 * (1 + abs(fr))
        assert np.allclose(x, ref, atol=1e-7)


def test_tron_scalar_examples():
    """(x-0.3)^2 -> 0.3 and (x+1)^2 -> 0 on [0,1]."""
    x, _ = oracle.tron_quadratic(np.array([[2.0]]), np.array([-0.6]), np.array([0.0]), np.array([1.0]), np.array([0.9]))
    assert x[0] == pytest.approx(0.3, abs=1e-12)
    x, _ = oracle.tron_quadratic(np.array([[2.0]]), np.array([2.0]), np.array([0.0]), np.array([1.0]), np.array([0.9]))
    assert x[0] == 0.0


def F_branch(y, x, tau, rpq, rva):
    f = flows_complex(y, x)
    return 0.5 * rpq * np.sum((f - tau[:4]) ** 2) + 0.5 * rva * np.sum((np.asarray(x) - tau[4:]) ** 2)


def grad_torch(y, x, tau, rpq, rva):
    xt = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    f = flows_torch(y, xt)
    t = torch.tensor(tau, dtype=torch.float64)
    F = 0.5 * rpq * torch.sum((f - t[:4]) ** 2) + 0.5 * rva * torch.sum((xt - t[4:]) ** 2)
    F.backward()
    return xt.grad.numpy()


PR = inputs.Params(rho_pq=5e3, rho_va=1e4, rho_uc=1e4)


def test_branch_planted_point():
    """targets = an exact power-flow point -> the solver returns it."""
    rng = np.random.default_rng(2)
    for _ in range(40):
        y = inputs.branch_admittance(rng.uniform(0, 0.04), rng.uniform(0.03, 0.2), rng.uniform(0, 0.2))
        xs = np.array([rng.uniform(0.85, 1.15), rng.uniform(0.85, 1.15), rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3)])
        tau = np.concatenate([flows_complex(y, xs), xs])
        x0 = xs + rng.normal(size=4) * 0.02
        x, al, f, st = oracle.branch_solve(y, [0.81, 0.81], [1.21, 1.21], 0.0, tau, 5e3, 1e4, PR, x0, np.zeros(3))
        assert np.allclose(x, xs, atol=1e-8)
        assert np.allclose(f, flows_complex(y, x), atol=1e-12)   # Eq. 2i-2j by construction
        assert st[1] == 0


def test_branch_kkt_random():
    """Projected gradient (torch autograd) at the returned point <= TRON tolerance."""
    rng = np.random.default_rng(3)
    lo = np.array([0.81, 0.81, -TWO_PI, -TWO_PI])
    hi = np.array([1.21, 1.21, TWO_PI, TWO_PI])
    for _ in range(60):
        y = inputs.branch_admittance(rng.uniform(0, 0.04), rng.uniform(0.03, 0.2), rng.uniform(0, 0.2))
        tau = np.concatenate([rng.normal(size=4) * 0.5, [rng.uniform(0.7, 1.3), rng.uniform(0.7, 1.3)],
                              rng.normal(size=2) * 0.1])
        x0 = np.array([1.0, 1.0, 0.0, 0.0])
        x, al, f, st = oracle.branch_solve(y, lo[:2], hi[:2], 0.0, tau, 5e3, 1e4, PR, x0, np.zeros(3))
        g = grad_torch(y, x, tau, 5e3, 1e4)
        pg = np.clip(x - g, lo, hi) - x
        assert np.max(np.abs(pg)) <= 2e-9 * 1e4
        assert st[1] == 0
        # a local minimum: no better point nearby within the box
        F0 = F_branch(y, x, tau, 5e3, 1e4)
        for _k in range(20):
            xp = np.clip(x + rng.normal(size=4) * 1e-4, lo, hi)
            assert F_branch(y, xp, tau, 5e3, 1e4) >= F0 - 1e-9


def test_branch_huge_rate_inactive():
    """rate huge -> thermal multipliers stay 0 and the result equals the unlimited one."""
    rng = np.random.default_rng(4)
    y = inputs.branch_admittance(0.01, 0.08, 0.1)
    tau = np.concatenate([rng.normal(size=4) * 0.5, [1.0, 1.0, 0.05, -0.05]])
    x0 = np.array([1.0, 1.0, 0.0, 0.0])
    a = oracle.branch_solve(y, [0.81, 0.81], [1.21, 1.21], 0.0, tau, 5e3, 1e4, PR, x0, np.zeros(3))
    b = oracle.branch_solve(y, [0.81, 0.81], [1.21, 1.21], 1e6, tau, 5e3, 1e4, PR, x0, np.zeros(3))
    assert np.array_equal(a[0], b[0]) and b[1][0] == 0 and b[1][1] == 0 and b[3][2] == 0


def test_branch_binding_limit_grid_search():
    """Binding Eq. 2c-2d: the AL result is feasible and at least as good as the best point
    of a dense feasible grid over (w_i, w_j, delta) with the optimal angle mean."""
    y = inputs.branch_admittance(0.01, 0.1, 0.05)
    rpq, rva = 5e3, 1e4
    rate = 0.6
    for seed in range(4):
        rng = np.random.default_rng(100 + seed)
        xs = np.array([1.0, 0.98, 0.12, 0.0]) + rng.normal(size=4) * 0.01
        fs = flows_complex(y, xs)
        tau = np.concatenate([fs * 1.15, xs])         # targets push the flow above the rate
        x, al, f, st = oracle.branch_solve(y, [0.81, 0.81], [1.21, 1.21], rate, tau, rpq, rva, PR,
                                           xs.copy(), np.zeros(3))
        assert st[2] == 1                              # AL path taken
        assert f[0] ** 2 + f[1] ** 2 <= rate ** 2 * (1 + 1e-8)
        assert f[2] ** 2 + f[3] ** 2 <= rate ** 2 * (1 + 1e-8)
        Fx = F_branch(y, x, tau, rpq, rva)
        # grid: w_i, w_j, delta; theta mean chosen optimally for the va terms
        wi = np.linspace(x[0] - 0.02, x[0] + 0.02, 41)
        wj = np.linspace(x[1] - 0.02, x[1] + 0.02, 41)
        dl = np.linspace((x[2] - x[3]) - 0.02, (x[2] - x[3]) + 0.02, 41)
        Wi, Wj, D = np.meshgrid(wi, wj, dl, indexing="ij")
        m = 0.5 * (tau[6] + tau[7] - D)            # theta_j minimising the va terms given delta
        Ti, Tj = m + D, m
        Vi = np.sqrt(Wi) * np.exp(1j * Ti)
        Vj = np.sqrt(Wj) * np.exp(1j * Tj)
        yff, yft, ytf, ytt = y[0] + 1j * y[4], y[1] + 1j * y[5], y[2] + 1j * y[6], y[3] + 1j * y[7]
        sij = Vi * np.conj(yff * Vi + yft * Vj)
        sji = Vj * np.conj(ytf * Vi + ytt * Vj)
        F = 0.5 * rpq * ((sij.real - tau[0]) ** 2 + (sij.imag - tau[1]) ** 2 + (sji.real - tau[2]) ** 2
                         + (sji.imag - tau[3]) ** 2) \
            + 0.5 * rva * ((Wi - tau[4]) ** 2 + (Wj - tau[5]) ** 2 + (Ti - tau[6]) ** 2 + (Tj - tau[7]) ** 2)
        feas = (np.abs(sij) <= rate) & (np.abs(sji) <= rate)
        assert feas.any()
        Fg = F[feas].min()
        assert Fx <= Fg + 1e-6 * abs(Fg)


def _lagrangian_grad(y, x, s, mu, tau, rpq, rva, r2):
    """Gradient of F + sum_m mu_m h_m over (x, s) by torch autograd (fp64), h_m the normalised
    Eq. 2c-2d constraint in slack form (R36)."""
    xt = torch.tensor(np.concatenate([x, s]), dtype=torch.float64, requires_grad=True)
    f = flows_torch(y, xt[:4])
    tt = torch.tensor(tau, dtype=torch.float64)
    F = 0.5 * rpq * torch.sum((f - tt[:4]) ** 2) + 0.5 * rva * torch.sum((xt[:4] - tt[4:]) ** 2)
    h0 = (f[0] ** 2 + f[1] ** 2) / r2 - 1.0 + xt[4]
    h1 = (f[2] ** 2 + f[3] ** 2) / r2 - 1.0 + xt[5]
    Lg = F + float(mu[0]) * h0 + float(mu[1]) * h1
    (g,) = torch.autograd.grad(Lg, xt)
    return g.numpy(), np.array([h0.item(), h1.item()])


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("seed", range(6))
def test_branch_al_kkt_multipliers(seed, variant):
    """The returned (x, mu) is a KKT point of the thermally constrained branch problem
    (Eq. 2c-2d): h ~ 0, mu >= 0 on a binding end, mu ~ 0 where the slack is interior, and the
    Lagrangian gradient vanishes on the free variables (autograd, independent of the oracle's
    derivative code and of its multiplier update rule).  Second-order multiplier steps (R42)
    reach it in a few rounds (a first-order update needs about twice as many)."""
    rng = np.random.default_rng(300 + seed)
    y = inputs.branch_admittance(rng.uniform(0.005, 0.03), rng.uniform(0.05, 0.2), rng.uniform(0.0, 0.1))
    rpq, rva = 5e3, 1e4
    rate = 0.5 + 0.2 * rng.uniform()
    xs = np.array([1.0, 0.98, 0.12, 0.0]) + rng.normal(size=4) * 0.01
    tau = np.concatenate([flows_complex(y, xs) * (1.2 + 0.2 * rng.uniform()), xs])
    lo, hi = np.array([0.81, 0.81]), np.array([1.21, 1.21])
    pr = dataclasses.replace(PR, variant=variant)   # variant 1 (R47): no fast path, the AL from the warm start
    x, al, f, st = oracle.branch_solve(y, lo, hi, rate, tau, rpq, rva, pr, xs.copy(), np.zeros(3))
    assert st[2] == 1 and st[4] == 0
    r2 = rate ** 2
    s = np.clip(1.0 - np.array([f[0] ** 2 + f[1] ** 2, f[2] ** 2 + f[3] ** 2]) / r2, 0.0, 1.0)
    g, h = _lagrangian_grad(y, x, s, al[:2], tau, rpq, rva, r2)
    assert np.max(np.abs(h)) <= 1e-8
    scale = rpq * np.max(np.abs(flows_complex(y, x))) ** 2
    for i in range(4):
        if lo[min(i, 1)] < x[i] < hi[min(i, 1)] or i >= 2:
            assert abs(g[i]) <= 1e-6 * scale, (i, g)
    for m in range(2):
        if s[m] > 1e-6:
            assert abs(al[m]) <= 1e-6 * scale
        else:
            assert al[m] >= -1e-6 * scale
    assert st[3] <= 6 and st[0] <= 40 + 20 * variant, st


def test_sincos_polynomial_against_libm():
    """R54: the oracle's explicit sin/cos polynomial (shared operation sequence with the strict_fp
    GPU build) is within 2 ulp of libm on [-4 pi, 4 pi] (the range of theta_i - theta_j over the
    box [-2 pi, 2 pi]^2), exact at 0, and odd/even."""
    rng = np.random.default_rng(54)
    a = np.concatenate([rng.uniform(-4 * np.pi, 4 * np.pi, 20000), rng.normal(0, 0.3, 20000),
                        np.arange(-8, 9) * np.pi / 2 + rng.normal(0, 1e-3, 17), [0.0, 1e-300, -1e-8, 0.7853981633974483]])
    worst = 0.0
    for v in a:
        s, c = oracle.sincos(v)
        rs, rc = np.sin(v), np.cos(v)
        # error in ulps of the larger of the value and 1e-16 (|sin| near k pi is limited by the
        # absolute accuracy of the argument reduction, ~1e-26)
        es = abs(s - rs) / np.spacing(max(abs(rs), 1e-16))
        ec = abs(c - rc) / np.spacing(max(abs(rc), 1e-16))
        worst = max(worst, es, ec)
        s2, c2 = oracle.sincos(-v)
        assert s2 == -s and c2 == c
    assert worst <= 2.0, worst
    assert oracle.sincos(0.0) == (0.0, 1.0)


def _harvest(name, iters):
    """every (l,t) branch-solve input of the oracle's next iteration at its state after `iters`
    iterations (targets tau = xbar - z - y/rho, warm x, AL state)"""
    pb, pr = inputs.build_config(name)
    pb = pb.normalized()
    o = oracle.Oracle(pb, pr)
    o.iterate(iters)
    st = o.get_state()
    o.close()
    L, T = pb.nbranch, pb.T
    LT = L * T
    zb, yb = st["zb"].reshape(8, LT), st["yb"].reshape(8, LT)
    fb, x, al = st["fbar"].reshape(LT, 4), st["x"].reshape(LT, 4), st["al"].reshape(LT, 3)
    wb, tb = st["wbar"].reshape(pb.nbus, T), st["thbar"].reshape(pb.nbus, T)
    rho = np.array([pr.rho_pq] * 4 + [pr.rho_va] * 4)
    for l in range(L):
        i, j = pb.br_from[l], pb.br_to[l]
        for t in range(T):
            k = l * T + t
            xb = np.array([fb[k, 0], fb[k, 1], fb[k, 2], fb[k, 3], wb[i, t], wb[j, t], tb[i, t], tb[j, t]])
            tau = xb - zb[:, k] - yb[:, k] / rho
            yield pr, (pb.br_y[l], [pb.bus_vmin[i] ** 2, pb.bus_vmin[j] ** 2],
                       [pb.bus_vmax[i] ** 2, pb.bus_vmax[j] ** 2], pb.br_rate[l], tau, x[k].copy(), al[k].copy())


def test_plain_and_accelerated_al_same_kkt_point():
    """The accelerated branch solver (R41-R44, R48, R49: solver engineering, not readings of the
    paper) and the plain first-order AL of SURVEY 8(c) S3 (oracle plain mode) reach the same KKT
    point on every solve of the case300 and pegase-shaped configs' states: x within 1e-11, the
    flows within 1e-9 relative, the thermal multipliers within 10 sigma eta* (the AL stops at
    |h| <= eta*, so mu is only defined to sigma eta*).  All thermally active solves
    are compared, plus every 20th inactive one."""
    n_al = n_fast = 0
    its = np.zeros(2)
    for name, iters in (("case300", 20), ("pegase2869", 3)):
        for k, (pr, (y, lo, hi, rate, tau, x0, al0)) in enumerate(_harvest(name, iters)):
            xa, ala, fa, sa = oracle.branch_solve(y, lo, hi, rate, tau, pr.rho_pq, pr.rho_va, pr, x0, al0)
            if sa[2] == 0 and k % 20:
                continue
            xp, alp, fp, sp = oracle.branch_solve(y, lo, hi, rate, tau, pr.rho_pq, pr.rho_va, pr, x0, al0, plain=True)
            assert sa[1] == 0 and sp[1] == 0 and sp[2] == sa[2] and sp[4] == 0
            assert np.max(np.abs(xa - xp)) <= 1e-11, (name, k, xa, xp)
            assert np.max(np.abs(fa - fp)) <= 1e-9 * max(1.0, np.max(np.abs(fa))), (name, k)
            if sa[2]:
                sig = max(ala[2], alp[2])
                assert np.max(np.abs(ala[:2] - alp[:2])) <= 10 * sig * pr.al_eta_star + 1e-9 * np.max(np.abs(ala[:2])), (name, k, ala, alp)
                n_al += 1
                its += (sa[8], sp[8])
            else:
                n_fast += 1
    print(f"plain vs accelerated: {n_al} AL solves, {n_fast} fast-path solves, Newton its {its}")
    assert n_al + n_fast >= 1000 and n_al >= 250, (n_al, n_fast)
    assert its[0] < its[1]   # the accelerations cut the AL's Newton iterations
