"""Pins for the oracle's closed-form steps: S2 generator (7b), S4 ubar (7c), S5 bus (7d).

Each is compared with an independent solver of the SAME optimization problem written out
from the paper's rows (P:186-191 with Eq. 4d, R3; generator consensus and ramp copy, R6;
Eq. 2a-2b for the bus), not with a retyped formula:
* generator / ubar: the bound-constrained least-squares problem solved by SciPy's BVLS
  (an exact active-set method) on the full variable set including all six slacks;
* bus: the dense KKT system of the equality-constrained QP solved with numpy.linalg.
"""
import numpy as np
import pytest
from scipy.optimize import lsq_linear

import oracle


def gen_reference(vec):
    """Exact minimiser of the 9-variable generator QP (p, q, phat, 6 slacks)."""
    first = vec[0] != 0
    c2S2, c1S, rpq, ruc, tp, tq, tph, p0 = vec[1:9]
    bpl, bpu, bql, bqu, brl, bru, pL, pU, qL, qU = vec[9:19]
    # variables: p q ph spl spu sql squ srd sru  (ph dropped when first)
    names = ["p", "q", "ph", "spl", "spu", "sql", "squ", "srd", "sru"]
    if first:
        names.remove("ph")
    ix = {n: i for i, n in enumerate(names)}
    rows, rhs = [], []

    def term(w, coef, b):
        a = np.zeros(len(names))
        for n, v in coef.items():
            a[ix[n]] += v
        rows.append(np.sqrt(w) * a)
        rhs.append(np.sqrt(w) * b)
    # c2S2 p^2 + c1S p = c2S2 (p + c1S/(2 c2S2))^2 + const  (requires c2 > 0)
    term(2 * c2S2, {"p": 1.0}, -c1S / (2 * c2S2))
    term(rpq, {"p": 1.0}, tp)                                   # GP row
    term(rpq, {"q": 1.0}, tq)                                   # GQ row
    term(ruc, {"p": 1.0, "spl": -1.0}, bpl)                     # PL
    term(ruc, {"p": 1.0, "spu": 1.0}, bpu)                      # PU
    term(ruc, {"q": 1.0, "sql": -1.0}, bql)                     # QL
    term(ruc, {"q": 1.0, "squ": 1.0}, bqu)                      # QU
    if first:
        term(ruc, {"p": 1.0, "srd": -1.0}, brl + p0)            # RD (Eq. 4d), phat_1 = p0
        term(ruc, {"p": 1.0, "sru": 1.0}, bru + p0)             # RU
    else:
        term(rpq, {"ph": 1.0}, tph)                             # RC row
        term(ruc, {"p": 1.0, "ph": -1.0, "srd": -1.0}, brl)
        term(ruc, {"p": 1.0, "ph": -1.0, "sru": 1.0}, bru)
    lo = np.zeros(len(names))
    hi = np.full(len(names), np.inf)
    lo[ix["p"]], hi[ix["p"]] = pL, pU
    lo[ix["q"]], hi[ix["q"]] = qL, qU
    if not first:
        lo[ix["ph"]], hi[ix["ph"]] = -np.inf, np.inf
    res = lsq_linear(np.array(rows), np.array(rhs), bounds=(lo, hi), method="bvls", tol=1e-15,
                     lsq_solver="exact")
    v = res.x
    return np.array([v[ix["p"]], v[ix["q"]], p0 if first else v[ix["ph"]]])


def random_gen_vec(rng, first):
    S = 100.0
    pmin, pmax = rng.uniform(0.1, 0.5), rng.uniform(0.8, 3.0)
    qmin, qmax = -rng.uniform(0.1, 1.0), rng.uniform(0.1, 1.0)
    on, su, sd, onp = rng.uniform(0, 1, 4)
    rd = ru = 0.1 * pmax
    s = max(pmin, rd)
    rpq = 10 ** rng.uniform(2.5, 4.5)
    ruc = 10 ** rng.uniform(2.5, 4.5)
    z = rng.normal(size=9) * 0.05
    vec = np.zeros(19)
    vec[0] = 1.0 if first else 0.0
    vec[1] = rng.uniform(0.002, 0.12) * S * S
    vec[2] = rng.uniform(1, 40) * S
    vec[3], vec[4] = rpq, ruc
    vec[5] = rng.uniform(0, pmax) + z[0]
    vec[6] = rng.uniform(qmin, qmax) + z[1]
    vec[7] = rng.uniform(0, pmax) + z[2]
    vec[8] = rng.uniform(pmin, pmax)
    vec[9] = pmin * on + z[3]
    vec[10] = pmax * on + z[4]
    vec[11] = qmin * on + z[5]
    vec[12] = qmax * on + z[6]
    vec[13] = -rd * on - s * sd + z[7]
    vec[14] = ru * onp + s * su + z[8]
    vec[15], vec[16] = min(0.0, pmin), pmax
    vec[17], vec[18] = min(0.0, qmin), max(0.0, qmax)
    return vec


@pytest.mark.parametrize("first", [False, True])
def test_gen_vs_exact_qp(first):
    rng = np.random.default_rng(7 + first)
    worst = 0.0
    for _ in range(300):
        vec = random_gen_vec(rng, first)
        got = oracle.gen_x(vec)
        ref = gen_reference(vec)
        worst = max(worst, np.max(np.abs(got - ref)))
        assert np.allclose(got, ref, rtol=1e-9, atol=1e-9), (vec, got, ref)
    assert worst < 1e-9


def test_gen_pure_projection():
    """c2 = c1 = 0, only the consensus row: p = clip(tau_p)."""
    vec = np.zeros(19)
    vec[3], vec[4] = 1e4, 1e-12
    vec[5], vec[6] = 2.5, -0.7
    vec[9], vec[10], vec[11], vec[12] = -1e9, 1e9, -1e9, 1e9
    vec[13], vec[14] = -1e9, 1e9
    vec[7] = 0.3
    vec[15], vec[16], vec[17], vec[18] = 0.0, 2.0, -0.5, 0.5
    out = oracle.gen_x(vec)
    assert out[0] == pytest.approx(2.0, abs=1e-12)
    assert out[1] == pytest.approx(-0.5, abs=1e-12)
    assert out[2] == pytest.approx(0.3, abs=1e-9)


def ubar_reference(c, e):
    res = lsq_linear(c, e, bounds=(0.0, 1.0), method="bvls", tol=1e-15, lsq_solver="exact")
    return res.x


def test_ubar_vs_bvls():
    rng = np.random.default_rng(21)
    for _ in range(400):
        n = int(rng.integers(1, 4))
        # duplicate rows (identity) + bound/ramp rows with the paper's coefficient shapes
        rows = [np.eye(3)[i][:n] for i in range(n)]
        pm, PM, qm, QM = rng.uniform(0.1, 0.5), rng.uniform(1, 3), -rng.uniform(0.1, 1), rng.uniform(0.1, 1)
        RD, SD, RU, SU = 0.2, 0.5, 0.2, 0.5
        cand = [[pm, 0, 0], [PM, 0, 0], [qm, 0, 0], [QM, 0, 0], [-RD, -SD, 0], [RU, 0, SU]]
        for cc in cand[: int(rng.integers(0, 7))]:
            rows.append(np.array(cc[:n], dtype=float))
        C = np.array(rows)
        e = rng.normal(size=C.shape[0]) * 1.5 + 0.5
        got = oracle.boxqp3(C, e)
        ref = ubar_reference(C, e)
        fg = 0.5 * np.sum((e - C @ got) ** 2)
        fr = 0.5 * np.sum((e - C @ ref) ** 2)
        assert fg <= fr + 1e-12 * (1 + abs(fr))
        assert np.allclose(got, ref, atol=1e-8)
        assert np.all(got >= 0) and np.all(got <= 1)


def test_ubar_dup_only_is_clip():
    """Only duplicate rows: ubar = clip(e)."""
    e = np.array([1.7, -0.3, 0.4])
    assert np.array_equal(oracle.boxqp3(np.eye(3), e), np.array([1.0, 0.0, 0.4]))


def test_ubar_scale_invariance():
    """rho scaling leaves the argmin unchanged."""
    rng = np.random.default_rng(2)
    C = np.vstack([np.eye(3), rng.normal(size=(4, 3))])
    e = rng.normal(size=7)
    a = oracle.boxqp3(C, e)
    b = oracle.boxqp3(3.0 * C, 3.0 * e)
    assert np.allclose(a, b, atol=1e-12)


def bus_dense(alpha, beta, a, th, P, Q):
    k = len(a)
    K = np.zeros((k + 2, k + 2))
    K[:k, :k] = np.diag(a)
    K[:k, k] = -alpha
    K[:k, k + 1] = -beta
    K[k, :k] = alpha
    K[k + 1, :k] = beta
    rhs = np.concatenate([a * th, [P, Q]])
    sol = np.linalg.solve(K, rhs)
    return sol[:k], sol[k:]


def test_bus_vs_dense_kkt():
    rng = np.random.default_rng(4)
    for _ in range(300):
        ng, ne = int(rng.integers(0, 3)), int(rng.integers(1, 6))
        alpha, beta, a, th = [], [], [], []
        for _g in range(ng):
            alpha += [1.0, 0.0]
            beta += [0.0, 1.0]
            a += [rng.choice([1e4, 2e4]), 1e4]
            th += list(rng.normal(size=2))
        for _e in range(ne):
            alpha += [-1.0, 0.0]
            beta += [0.0, -1.0]
            a += [1e4, 1e4]
            th += list(rng.normal(size=2))
        gs, bs = rng.normal() * 0.05, rng.normal() * 0.2
        alpha.append(-gs)
        beta.append(bs)
        a.append(ne * 2e4)
        th.append(1.0 + 0.05 * rng.normal())
        alpha, beta, a, th = map(np.array, (alpha, beta, a, th))
        P, Q = rng.normal(), rng.normal()
        v, mu = oracle.bus_kkt(alpha, beta, a, th, P, Q)
        vr, mur = bus_dense(alpha, beta, a, th, P, Q)
        assert np.allclose(v, vr, rtol=1e-11, atol=1e-12)
        assert abs(alpha @ v - P) < 1e-10 and abs(beta @ v - Q) < 1e-10   # Eq. 2a-2b


def test_bus_balanced_targets_fixed_point():
    """targets already satisfying Eq. 2a-2b are returned unchanged."""
    alpha = np.array([1.0, 0.0, -1.0, 0.0, -0.0])
    beta = np.array([0.0, 1.0, 0.0, -1.0, 0.0])
    th = np.array([0.8, 0.3, 0.5, 0.1, 1.0])
    a = np.array([1e4, 1e4, 1e4, 1e4, 2e4])
    v, mu = oracle.bus_kkt(alpha, beta, a, th, alpha @ th, beta @ th)
    assert np.allclose(v, th, atol=1e-15) and np.allclose(mu, 0.0, atol=1e-9)
