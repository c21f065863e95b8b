"""The scheduling knobs of the iteration graph change WHEN work runs, never what it computes.

DESIGN.md 7 claims that the one-wave `k_rows_late` grid (UCAC_LROWS_GRID), the programmatic
dependent launches of the critical chain (UCAC_PDL) and the batched last-block folds leave the
iterate bitwise unchanged.  Each knob is read once per process, so every setting runs in its own
subprocess (tools/ab_state.py) and the full iterates are compared byte for byte.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _state(tmp_path, tag, env_over, case="case118", iters=40):
    out = str(tmp_path / f"{tag}.npz")
    env = dict(os.environ)
    for k, v in env_over.items():
        if v is None:
            env.pop(k, None)
        else:
            env[k] = v
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ab_state.py"), out, case, str(iters)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    return np.load(out)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["case118", "case300"])
def test_schedule_knobs_bitwise(tmp_path, case):
    base = _state(tmp_path, "default", {"UCAC_LROWS_GRID": None, "UCAC_PDL": None}, case)
    variants = {
        "rows_one_thread_per_lt": {"UCAC_LROWS_GRID": "-1", "UCAC_PDL": None},
        "rows_grid_37": {"UCAC_LROWS_GRID": "37", "UCAC_PDL": None},   # several grid-stride passes
        "no_pdl": {"UCAC_LROWS_GRID": None, "UCAC_PDL": "0"},
        "pdl_all": {"UCAC_LROWS_GRID": None, "UCAC_PDL": "7"},
    }
    for tag, env in variants.items():
        st = _state(tmp_path, tag, env, case)
        bad = [k for k in base.files if k != "scal" and base[k].tobytes() != st[k].tobytes()]
        assert not bad, f"{case} {tag}: iterate differs from the default schedule in {bad}"
        # scal[1] = ||z|| at the last outer update: a sum whose block grouping follows the grid,
        # so only the rounding of the fold may move (relative n * eps); the rest is exact
        a, b = base["scal"], st["scal"]
        assert np.array_equal(np.delete(a, 1), np.delete(b, 1)), f"{case} {tag}: scal {a} vs {b}"
        assert abs(a[1] - b[1]) <= 1e-12 * abs(a[1]), f"{case} {tag}: ||z|| {a[1]!r} vs {b[1]!r}"
