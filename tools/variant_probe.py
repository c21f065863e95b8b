"""One-step GPU vs oracle error distribution of the branch outputs (x, al) per iteration, for a
formulation variant (diagnostic; prints per-iteration quantiles and the worst branches)."""
import dataclasses
import sys

import numpy as np

import oracle
from paper_2310_13145_b200 import inputs, ucac

variant = int(sys.argv[1]) if len(sys.argv) > 1 else 1
case = sys.argv[2] if len(sys.argv) > 2 else "case30"
pb, pr = inputs.build_config(case)
pr = dataclasses.replace(pr, variant=variant)
gpu = ucac.Context(pb, pr)
for it in range(8):
    one = oracle.Oracle(pb, pr)
    st0 = gpu.get_state()
    one.set_state(st0)
    gpu.iterate(1)
    one.iterate(1)
    gs, os_ = gpu.get_state(), one.get_state()
    x, xo = gs["x"].reshape(-1, 4), os_["x"].reshape(-1, 4)
    al, alo = gs["al"].reshape(-1, 3), os_["al"].reshape(-1, 3)
    scale = np.maximum(np.abs(xo), np.sqrt(np.mean(xo * xo, axis=0)))
    rel = np.max(np.abs(x - xo) / scale, axis=1)
    dmu = np.max(np.abs(al[:, :2] - alo[:, :2]), axis=1) / np.maximum(alo[:, 2], 1e-300)
    order = np.argsort(-rel)[:5]
    print(f"it {it+1}: x rel q50 {np.median(rel):.2e} q99 {np.quantile(rel, .99):.2e} max {rel.max():.2e}; "
          f"n>1e-12 {(rel > 1e-12).sum()} / {len(rel)}; sig mismatch {(al[:, 2] != alo[:, 2]).sum()}")
    for r in order:
        print(f"   lt {r}: rel {rel[r]:.2e} x {x[r]} xo {xo[r]} mu {al[r]} muo {alo[r]} dmu/sig {dmu[r]:.2e}"
              f" prev mu {st0['al'].reshape(-1, 3)[r]}")
    one.close()
