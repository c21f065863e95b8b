"""Pins for oracle S1 (UC dynamic program, Section III-B, Alg. 2).

The DP is checked against brute force over every schedule satisfying Eq. (3a)-(3f)
 written out here independently, the SPEC worked examples, and the shift
invariance of Section III-B's recursion."""
import itertools
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def feasible(u, u0, TU, TD, hold):
    """Eq. 3 with su/sd inferred from u (t=1 uses u0, R4)."""
    T = len(u)
    if u0 == 1 and any(u[t] != 1 for t in range(hold)):      # Eq. 3a, L_g = hold
        return False
    if u0 == 0 and any(u[t] != 0 for t in range(hold)):      # Eq. 3b, F_g = hold
        return False
    prev = [u0] + list(u[:-1])
    su = [max(0, u[t] - prev[t]) for t in range(T)]
    sd = [max(0, prev[t] - u[t]) for t in range(T)]
    for t in range(TU - 1, T):                               # Eq. 3d, t in {T^U..T}
        if sum(su[t - TU + 1:t + 1]) > u[t]:
            return False
    for t in range(TD - 1, T):                               # Eq. 3e
        if sum(sd[t - TD + 1:t + 1]) > 1 - u[t]:
            return False
    return True


def sched_cost(L, u, u0):
    c = 0.0
    prev = u0
    for t, b in enumerate(u):
        c += L[t, prev, b]
        prev = b
    return c


def brute(L, u0, TU, TD, hold):
    T = L.shape[0]
    best, arg, costs = np.inf, None, []
    for u in itertools.product([0, 1], repeat=T):
        if feasible(u, u0, TU, TD, hold):
            c = sched_cost(L, u, u0)
            costs.append(c)
            if c < best:
                best, arg = c, u
    return best, arg, sorted(costs)


def test_spec_T1():
    g = GOLD["dp_T1"]
    L = np.zeros((1, 2, 2))
    L[0, 1, 1] = g["L11"]
    L[0, 1, 0] = g["L10"]
    L[0, 0, 0] = 100.0
    L[0, 0, 1] = 100.0
    s, c = oracle.dp_solve(L, g["TU"], g["TD"], g["u0"], g["hold"])
    assert list(s) == g["schedule"] and c == g["cost"]


def test_spec_T3_minup():
    g = GOLD["dp_T3_minup"]
    L = np.zeros((3, 2, 2))
    L[:, :, 1] = g["L_on"]
    L[:, :, 0] = g["L_off"]
    s, c = oracle.dp_solve(L, g["TU"], g["TD"], g["u0"], g["hold"])
    assert list(s) == g["schedule"] and c == g["cost"]


def test_stage_cost_spec():
    g = GOLD["stage_cost_su"]
    ub = np.array(g["ubar"])[:, None]
    L = oracle.stage_costs(1, 0.0, 0.0, 0.0, g["rho"], ub, np.zeros((3, 1)), np.zeros((3, 1)))
    a, b = g["transition"]
    assert L[0, a, b] == g["L"]
    assert L[0, 1, 1] == 0.0


# The stage cost's definition is pinned against the full augmented Lagrangian in
# tests/test_oracle_al_pins.py::test_stage_cost_equals_full_al_difference.


@pytest.mark.parametrize("seed", range(6))
def test_dp_vs_bruteforce(seed):
    """S:517 acceptance 1: exact optimum over Eq. 3; schedule feasible; argmin when unique."""
    rng = np.random.default_rng(seed)
    for _ in range(60):
        T = int(rng.integers(1, 10))
        TU, TD = int(rng.integers(1, min(4, T) + 1)), int(rng.integers(1, min(4, T) + 1))
        u0 = int(rng.integers(0, 2))
        hold = int(rng.integers(0, min(2, T) + 1)) if rng.uniform() < 0.4 else 0
        L = rng.uniform(-1, 1, (T, 2, 2))
        s, c = oracle.dp_solve(L, TU, TD, u0, hold)
        best, arg, costs = brute(L, u0, TU, TD, hold)
        assert feasible(list(s), u0, TU, TD, hold)
        assert c == pytest.approx(best, rel=1e-12, abs=1e-12)
        assert sched_cost(L, list(s), u0) == pytest.approx(best, rel=1e-12, abs=1e-12)
        if len(costs) > 1 and costs[1] - costs[0] > 1e-9:
            assert tuple(s) == arg


def test_dp_shift_invariance():
    """Adding kappa to every table entry adds kappa*T and keeps the schedule."""
    rng = np.random.default_rng(11)
    for _ in range(50):
        T = int(rng.integers(2, 12))
        L = rng.uniform(-1, 1, (T, 2, 2))
        s1, c1 = oracle.dp_solve(L, 2, 3, 1, 0)
        s2, c2 = oracle.dp_solve(L + 0.5, 2, 3, 1, 0)
        assert list(s1) == list(s2)
        assert c2 == pytest.approx(c1 + 0.5 * T, rel=1e-12, abs=1e-12)


def test_dp_tie_rule_stay():
    """c_stay <= c_switch -> stay.  All-zero costs: the unit stays at u0."""
    for u0 in (0, 1):
        s, c = oracle.dp_solve(np.zeros((6, 2, 2)), 2, 2, u0, 0)
        assert list(s) == [u0] * 6 and c == 0.0


def test_dp_linear_time():
    """O(T): 168 periods on a window of 4 is cheap; brute force is impossible."""
    rng = np.random.default_rng(5)
    L = rng.uniform(-1, 1, (168, 2, 2))
    s, c = oracle.dp_solve(L, 4, 4, 1, 2)
    assert feasible(list(s), 1, 4, 4, 2)
    assert sched_cost(L, list(s), 1) == pytest.approx(c, rel=1e-12)
