"""Where does GPU/oracle drift start?  Runs both on a test case iteration by iteration and,
at every iteration, restarts a fresh oracle from the GPU state to separate one-iteration
differences from accumulated ones; prints the worst branch solves (diagnostic).
usage: python tools/drift_probe.py ragged SEED ITERS | config NAME ITERS"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from paper_2310_13145_b200 import inputs, ucac  # noqa: E402
from test_gpu_parity import ATOL, RTOL, kind_scale, FLOAT_FIELDS  # noqa: E402


def case(kind, arg):
    if kind == "ragged":
        seed = int(arg)
        rng = np.random.default_rng(seed)
        nb = int(rng.integers(30, 60))
        ng = int(rng.integers(5, 12))
        pb = inputs.synthetic_case(nb, ng, nb + int(rng.integers(5, 20)), seed=1000 + seed, T=int(rng.integers(5, 9)))
        return pb, inputs.Params(rho_pq=5e3, rho_va=1e4, rho_uc=1e4)
    return inputs.build_config(arg)


def rel(a, b, k):
    return np.abs(a - b) / (1e-300 + kind_scale(k, b))


def main(kind, arg, iters):
    pb, pr = case(kind, arg)
    g = ucac.Context(pb, pr)
    o = oracle.Oracle(pb, pr)
    T = pb.T
    for it in range(int(iters)):
        s0 = g.get_state()
        o1 = oracle.Oracle(pb, pr)
        o1.set_state(s0)
        g.iterate(1)
        o.iterate(1)
        o1.iterate(1)
        a, b, c = g.get_state(), o.get_state(), o1.get_state()
        acc = {k: float(np.max(rel(a[k], b[k], k))) if a[k].size else 0.0 for k in FLOAT_FIELDS}
        one = {k: float(np.max(rel(a[k], c[k], k))) if a[k].size else 0.0 for k in FLOAT_FIELDS}
        wa, wo = max(acc, key=acc.get), max(one, key=one.get)
        sa, sb = a['al'].reshape(-1, 3)[:, 2], b['al'].reshape(-1, 3)[:, 2]
        print(f"it {it + 1:3d} accumulated worst {wa} {acc[wa]:.2e} | one-step worst {wo} {one[wo]:.2e} "
              f"| al sigma equal: one-step {np.array_equal(sa, c['al'].reshape(-1, 3)[:, 2])} "
              f"accumulated {np.array_equal(sa, sb)} (n diff {int(np.sum(sa != sb))})")
        top = sorted(((v, k) for k, v in acc.items() if k != "al"), reverse=True)[:4]
        print("     accumulated top:", ", ".join(f"{k} {v:.1e}" for v, k in top))
        if acc.get("zg", 0) > 1e-9:
            r = rel(a["zg"], b["zg"], "zg").reshape(12, pb.ngen, T)
            for j in np.argsort(-r.ravel())[:4]:
                kk, gg, tt = np.unravel_index(j, r.shape)
                print(f"     zg kind {kk} g {gg} t {tt}: gpu {a['zg'].reshape(12, pb.ngen, T)[kk, gg, tt]!r} "
                      f"oracle {b['zg'].reshape(12, pb.ngen, T)[kk, gg, tt]!r}")
            ds = np.nonzero(sa != sb)[0]
            for i in ds[:6]:
                print(f"     sigma differs at (l,t)=({i // T},{i % T}): gpu {a['al'].reshape(-1, 3)[i]} "
                      f"oracle {b['al'].reshape(-1, 3)[i]}")
        if one[wo] > 1e-10:
            xa, xc = a["x"].reshape(-1, 4), c["x"].reshape(-1, 4)
            la, lc = a["al"].reshape(-1, 3), c["al"].reshape(-1, 3)
            d = np.max(np.abs(xa - xc), axis=1)
            for i in np.argsort(-d)[:5]:
                print(f"    (l,t)=({i // T},{i % T}) |dx| {d[i]:.2e} al gpu {la[i]} oracle {lc[i]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
