"""Per-field GPU-vs-oracle difference report (diagnostic; not a test).

For each config: run the GPU k iterations, hand its state to the oracle, run one more
iteration on both, print max |diff| and max |diff|/|oracle| per state field.
usage: python tools/parity_report.py [config ...]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2310_13145_b200 import inputs, ucac  # noqa: E402


def report(name, k=5):
    pb, pr = inputs.build_config(name)
    g = ucac.Context(pb, pr)
    g.iterate(k)
    st = g.get_state()
    o = oracle.Oracle(pb, pr)
    o.set_state(st)
    g.iterate(1)
    o.iterate(1)
    a, b = g.get_state(), o.get_state()
    print(f"== {name}: {pb.nbus} buses, {pb.nbranch} branches, T={pb.T}; after iteration {k + 1}")
    print(f"   schedule equal: {np.array_equal(a['u'], b['u'])}")
    for f in a:
        if f in ("u", "scal"):
            continue
        d = np.abs(a[f] - b[f])
        rel = d / np.maximum(np.abs(b[f]), 1e-300)
        i = int(np.argmax(d))
        over = np.mean(d > 1e-12 + 1e-9 * np.abs(b[f]))
        print(f"   {f:6s} max|d| {d.max():.3e} (oracle {b[f][i]: .6e})  max rel {np.max(np.where(np.abs(b[f]) > 1e-6, rel, 0)):.3e}"
              f"  frac>tol {over:.2e}")


if __name__ == "__main__":
    for n in sys.argv[1:] or ["case30", "case118", "pegase2869"]:
        report(n)
