"""Dump the GPU iterate after N graph iterations of a config to an .npz (A/B bitwise checks of
scheduling-only kernel changes).  usage: python tools/ab_state.py OUT.npz [config] [iters]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_13145_b200 import inputs, ucac  # noqa: E402

out = sys.argv[1]
case = sys.argv[2] if len(sys.argv) > 2 else "pegase2869"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 100
pb, pr = inputs.build_config(case)
ctx = ucac.Context(pb, pr)
ctx.iterate(n)
np.savez(out, **ctx.get_state())
print(out, case, n, ctx.report())
