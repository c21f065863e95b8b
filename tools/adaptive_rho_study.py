"""NEXT-4(b) adaptive rho (R53): residual balancing on the GPU through
ucac_set_rho.  Every K inner iterations the primal infeasibility r (max |Ax + Bxbar|) and the
dual residual s (max rho |dxbar|) are compared; r > mu s scales all three penalty classes by
tau, s > mu r by 1/tau, within [lo, hi] x the initial values (Boyd et al. 2011, 3.4.1).  Reports
the best primal reached and the time to 1e-2 / 1e-3 / 1e-4 against the fixed-rho run.
usage: python tools/adaptive_rho_study.py [out.json] [max_iters]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_13145_b200 import inputs, ucac  # noqa: E402

THRESHOLDS = (1e-2, 1e-3, 1e-4)


def run(pb, pr, max_iters, adaptive, K=50, mu=10.0, tau=2.0, lo=1e-2, hi=1e2):
    import torch
    c = ucac.Context(pb, pr)
    rho0 = (pr.rho_pq, pr.rho_va, pr.rho_uc)
    scale, changes = 1.0, 0
    out = {"to": {}, "best_primal": float("inf")}
    done, secs, nxt = 0, 0.0, 0
    while done < max_iters:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        c.iterate(K)
        r = c.report()
        if adaptive:
            new = scale
            if r["primal_inf"] > mu * r["dual_inf"]:
                new = min(scale * tau, hi)
            elif r["dual_inf"] > mu * r["primal_inf"]:
                new = max(scale / tau, lo)
            if new != scale:
                scale = new
                changes += 1
                c.set_rho(*(v * scale for v in rho0))
        torch.cuda.synchronize()
        secs += time.perf_counter() - t0
        done += K
        out["best_primal"] = min(out["best_primal"], r["primal_inf"])
        while nxt < len(THRESHOLDS) and r["primal_inf"] <= THRESHOLDS[nxt]:
            out["to"][f"{THRESHOLDS[nxt]:g}"] = {"iterations": done, "seconds": secs}
            nxt += 1
    r = c.report()
    out.update(iterations=done, seconds=secs, final_primal=r["primal_inf"], objective=r["objective"],
               outer=r["outer_total"], rho_scale=scale, rho_changes=changes)
    c.close()
    return out


def main(out=None, max_iters="20000"):
    rows = []
    for name in ("case9", "case30", "case118", "case300"):
        pb, pr = inputs.build_config(name)
        for adaptive in (False, True):
            row = {"config": name, "adaptive_rho": adaptive}
            row.update(run(pb, pr, int(max_iters), adaptive))
            rows.append(row)
            print(json.dumps(row), flush=True)
    if out:
        json.dump(rows, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
