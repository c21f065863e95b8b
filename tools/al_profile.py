"""Distribution of the per-solve work of the branch step (7b) at a given inner iteration,
computed with the oracle on CPU (diagnostic; tools/ only).  Reports how many (l,t) solves
enter the thermal AL, and the TRON-iteration / AL-round histograms, i.e. the length of the
longest single-thread chain that bounds k_branch_al.
usage: python tools/al_profile.py [config] [iterations]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2310_13145_b200 import inputs  # noqa: E402


def profile(name="pegase2869", iters=10):
    pb, pr = inputs.build_config(name)
    o = oracle.Oracle(pb, pr, omp=True)
    o.iterate(int(iters))
    s = o.get_state()
    L, T = pb.nbranch, pb.T
    LT = L * T
    rpq, rva = pr.rho_pq, pr.rho_va
    zb, yb = s["zb"].reshape(8, LT), s["yb"].reshape(8, LT)
    fbar, x, al = s["fbar"].reshape(LT, 4), s["x"].reshape(LT, 4), s["al"].reshape(LT, 3)
    wbar, thbar = s["wbar"], s["thbar"]
    rows = []
    for l in range(L):
        bi, bj = pb.br_from[l], pb.br_to[l]
        wlo = [pb.bus_vmin[bi] ** 2, pb.bus_vmin[bj] ** 2]
        whi = [pb.bus_vmax[bi] ** 2, pb.bus_vmax[bj] ** 2]
        for t in range(T):
            i = l * T + t
            tau = np.empty(8)
            tau[:4] = fbar[i] - zb[:4, i] - yb[:4, i] / rpq
            tau[4] = wbar[bi * T + t] - zb[4, i] - yb[4, i] / rva
            tau[5] = wbar[bj * T + t] - zb[5, i] - yb[5, i] / rva
            tau[6] = thbar[bi * T + t] - zb[6, i] - yb[6, i] / rva
            tau[7] = thbar[bj * T + t] - zb[7, i] - yb[7, i] / rva
            _, _, _, st = oracle.branch_solve(pb.br_y[l], wlo, whi, pb.br_rate[l], tau, rpq, rva, pr,
                                              x[i], al[i])
            rows.append((l, t, *st))
    a = np.array(rows)
    it, al_on, al_rounds = a[:, 2], a[:, 4] == 1, a[:, 5]
    print(f"{name} after {iters} iterations: {LT} solves, {al_on.sum()} thermal-AL")
    print("TRON iterations, fast path: mean %.2f max %d" % (it[~al_on].mean(), it[~al_on].max()))
    if al_on.any():
        ia = it[al_on]
        print("TRON iterations, AL solves: mean %.1f  p50 %d p90 %d p99 %d max %d" % (
            ia.mean(), *np.percentile(ia, [50, 90, 99]).astype(int), ia.max()))
        print("AL rounds: mean %.2f max %d; histogram %s" % (al_rounds[al_on].mean(), al_rounds[al_on].max(),
                                                               np.bincount(al_rounds[al_on].astype(int)).tolist()))
        top = np.argsort(-ia)[:8]
        idx = np.nonzero(al_on)[0][top]
        for j in idx:
            print("  l %d t %d iters %d rounds %d" % (a[j, 0], a[j, 1], a[j, 2], a[j, 5]))
    return a


if __name__ == "__main__":
    profile(*sys.argv[1:])
