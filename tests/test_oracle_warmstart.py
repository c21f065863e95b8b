"""Pins for the NEXT-2 UC warm start (SPEC warm_start_uc): the threshold + one-DP-pass
repair is checked against brute force over every schedule (small T): the repaired schedule
satisfies Eq. 3 (min-up/down, held prefix) and has the minimal Hamming distance to the
thresholded dispatch; plus SPEC's worked examples and the held-schedule ACOPF run."""
import dataclasses
import itertools

import numpy as np
import pytest

import oracle
from paper_2310_13145_b200 import inputs


def feasible(u, TU, TD, u0, hold):
    """Eq. 3 on a schedule, with the initial state u0 held for `hold` periods (R14): every run
    that starts inside the horizon lasts min-up (on) / min-down (off) periods or reaches T."""
    T = len(u)
    if any(u[t] != u0 for t in range(min(hold, T))):
        return False
    prev, start = u0, None
    for t in range(T):
        if u[t] != prev:
            start = t
            prev = u[t]
            m = TU if u[t] == 1 else TD
            end = min(T, t + m)
            if any(u[k] != u[t] for k in range(t, end)):
                return False
    return True


def test_spec_examples():
    assert list(oracle.uc_repair([0.5, 0.6, 0.7], 1e-3, 1, 1, 1, 0)) == [1, 1, 1]
    assert list(oracle.uc_repair([0.0, 0.0, 0.0], 1e-3, 2, 2, 0, 0)) == [0, 0, 0]
    u = oracle.uc_repair([0.0, 0.6, 0.0], 1e-3, 2, 1, 0, 0)
    assert feasible(list(u), 2, 1, 0, 0) and sum(a != b for a, b in zip(u, [0, 1, 0])) == 1


@pytest.mark.parametrize("seed", range(40))
def test_repair_is_nearest_feasible_schedule(seed):
    rng = np.random.default_rng(seed)
    T = int(rng.integers(1, 9))
    TU, TD = int(rng.integers(1, T + 1)), int(rng.integers(1, T + 1))
    u0 = int(rng.integers(0, 2))
    hold = int(rng.integers(0, min(3, T) + 1))
    p = rng.uniform(-0.5, 1.0, T) * (rng.uniform(size=T) < 0.6)
    thr = 1e-3
    target = (p > thr).astype(int)
    u = [int(v) for v in oracle.uc_repair(p, thr, TU, TD, u0, hold)]
    assert feasible(u, TU, TD, u0, hold)
    best = min(sum(a != b for a, b in zip(s, target))
               for s in itertools.product((0, 1), repeat=T) if feasible(list(s), TU, TD, u0, hold))
    assert sum(a != b for a, b in zip(u, target)) == best


def test_held_schedule_acopf_keeps_u():
    """uc_fixed: step (7a) is skipped, the all-on (after the held prefix) schedule stays."""
    pb, pr = inputs.build_config("case9")
    u, p = oracle.uc_warm_start(pb, pr, iters=30)
    assert u.shape == (pb.ngen, pb.T)
    G, T = pb.ngen, pb.T
    uinit = np.ones((G, T), dtype=np.int8)
    for g in range(G):
        uinit[g, :int(pb.hold[g])] = int(pb.u0[g])
    o = oracle.Oracle(dataclasses.replace(pb, u_init=uinit), dataclasses.replace(pr, uc_fixed=1))
    o.iterate(30)
    assert np.array_equal(o.get_state()["u"].reshape(G, T), uinit)
    for g in range(G):
        assert feasible(list(u[g]), int(pb.min_up[g]), int(pb.min_dn[g]), int(pb.u0[g]), int(pb.hold[g]))
