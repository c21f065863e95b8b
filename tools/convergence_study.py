"""Time to primal infeasibility (the "time-to-residual" part of BASELINE.json's metric) on one
B200: for each config, rho setting (the bench's (5e3, 1e4, 1e4) and Table I's per-case values,
P:440) and initial schedule (cold: u0 held through the horizon; warm: NEXT-2 ucac_uc_warm_start),
the GPU iterations and device seconds to primal <= 1e-2, 1e-3, 1e-4, and the best primal seen.
usage: python tools/convergence_study.py [out.json] [max_iters]"""
import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_13145_b200 import inputs, ucac  # noqa: E402

TABLE1_RHO = {"case9": (5e3, 1e4, 1e4), "case30": (5e5, 1e6, 1e6), "case118": (5e4, 1e5, 1e5),
              "case300": (5e3, 1e4, 1e4)}
THRESHOLDS = (1e-2, 1e-3, 1e-4)


def run(pb, pr, max_iters, chunk=500):
    import torch
    c = ucac.Context(pb, pr)
    out = {"to": {}, "best_primal": float("inf")}
    done, secs = 0, 0.0
    for thr in THRESHOLDS:
        reached = False
        while done < max_iters:
            n = min(chunk, max_iters - done)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            k = c.iterate(n, stop_on_primal=thr)
            torch.cuda.synchronize()
            secs += time.perf_counter() - t0
            done += k
            r = c.report()
            out["best_primal"] = min(out["best_primal"], r["primal_inf"])
            if r["primal_inf"] <= thr:
                out["to"][f"{thr:g}"] = {"iterations": done, "seconds": secs, "outer": r["outer_total"],
                                         "objective": r["objective"]}
                reached = True
                break
        if not reached:
            break
    r = c.report()
    out.update(iterations=done, seconds=secs, final_primal=r["primal_inf"], objective=r["objective"],
               outer=r["outer_total"], beta=r["beta"])
    c.close()
    return out


def main(out=None, max_iters="20000"):
    max_iters = int(max_iters)
    rows = []
    for name in ("case9", "case30", "case118", "case300"):
        pb0, pr0 = inputs.build_config(name)
        for rho_name, rho in (("bench", (pr0.rho_pq, pr0.rho_va, pr0.rho_uc)), ("table1", TABLE1_RHO[name])):
            if rho_name == "table1" and rho == (pr0.rho_pq, pr0.rho_va, pr0.rho_uc):
                continue
            pr = dataclasses.replace(pr0, rho_pq=rho[0], rho_va=rho[1], rho_uc=rho[2])
            for start in ("cold", "warm"):
                pb = pb0
                if start == "warm":
                    pb = dataclasses.replace(pb0, u_init=ucac.uc_warm_start(pb0, pr, 200))
                row = {"config": name, "rho": rho_name, "rho_values": rho, "start": start}
                row.update(run(pb, pr, max_iters))
                rows.append(row)
                print(json.dumps(row), flush=True)
    if out:
        json.dump(rows, open(out, "w"), indent=1)


def sweep(out=None, max_iters="20000", key="beta_max", values="2.5e3,5e3,1e4,2e4,5e4,1e12",
          cases="case30,case118,case300"):
    """one parameter of the outer loop swept on the bench rho, cold start."""
    rows = []
    for name in cases.split(","):
        pb, pr0 = inputs.build_config(name)
        for v in values.split(","):
            pr = dataclasses.replace(pr0, **{key: type(getattr(pr0, key))(float(v))})
            row = {"config": name, key: float(v)}
            row.update(run(pb, pr, int(max_iters)))
            rows.append(row)
            print(json.dumps(row), flush=True)
    if out:
        json.dump(rows, open(out, "w"), indent=1)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "sweep":
        sweep(*sys.argv[2:])
    else:
        main(*sys.argv[1:])
