"""The oracle's divergence detector ("non-decreasing divergence detector (primal residual
grows 10x over 200 inner iterations) -> abort with diagnostics"), pinned against the rule
evaluated by brute force on the per-iteration primal residuals of a detector-off run."""
import dataclasses

import pytest

import oracle
from paper_2310_13145_b200 import inputs


def _primal_sequence(pb, pr, n):
    o = oracle.Oracle(pb, pr)
    seq = []
    for _ in range(n):
        o.iterate(1)
        seq.append(o.report()["primal_inf"])
    o.close()
    return seq


def test_detector_off_by_default_and_factor_extremes():
    pb, pr = inputs.build_config("case9")
    assert pr.diverge_window == 0
    # factor 0: primal_i > 0 * primal_{i-w} from the first iteration that has a predecessor w back
    w = 5
    o = oracle.Oracle(pb, dataclasses.replace(pr, diverge_window=w, diverge_factor=0.0))
    o.iterate(50)
    r = o.report()
    assert r["diverged_iter"] == w + 1 and r["inner_total"] == w + 1
    o.iterate(3)   # the call the detector ended is over: the next one continues, the flag stays
    r = o.report()
    assert r["inner_total"] == w + 4 and r["diverged_iter"] == w + 1
    # an unreachable factor never fires
    o = oracle.Oracle(pb, dataclasses.replace(pr, diverge_window=w, diverge_factor=1e300))
    o.iterate(40)
    assert o.report()["diverged_iter"] == 0 and o.report()["inner_total"] == 40


@pytest.mark.parametrize("w,factor", [(3, 1.0), (7, 0.9), (20, 0.5)])
def test_detector_stops_where_the_rule_first_holds(w, factor):
    """The stop iteration is the first i > w with p_i > factor * p_{i-w} (1-based), computed from
    a detector-off run's per-iteration reports; the iterate up to there is unchanged."""
    pb, pr = inputs.build_config("case9")
    n = 120
    p = _primal_sequence(pb, pr, n)
    first = next((i for i in range(w + 1, n + 1) if p[i - 1] > factor * p[i - 1 - w]), 0)
    assert first, "the rule never holds on this run: choose another (w, factor)"
    o = oracle.Oracle(pb, dataclasses.replace(pr, diverge_window=w, diverge_factor=factor))
    o.iterate(n)
    r = o.report()
    assert r["diverged_iter"] == first and r["inner_total"] == first
    assert r["primal_inf"] == p[first - 1]


def test_window_range_and_state_reset():
    pb, pr = inputs.build_config("case9")
    with pytest.raises(ValueError):
        oracle.Oracle(pb, dataclasses.replace(pr, diverge_window=256))
    # set_state replaces the trajectory: the history restarts (no detection until w iterations)
    w = 4
    o = oracle.Oracle(pb, dataclasses.replace(pr, diverge_window=w, diverge_factor=0.0))
    o.iterate(10)
    assert o.report()["diverged_iter"] == w + 1
    o.set_state(o.get_state())
    assert o.report()["diverged_iter"] == 0
    o.iterate(20)
    assert o.report()["diverged_iter"] == (w + 1) + (w + 1)
