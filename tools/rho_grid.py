"""SURVEY.md 8(d) rho grid for the time-to-residual configs (BASELINE configs[1]-[3]).

For each of case30/118/300 and every (rho_pq, rho_va, rho_uc) = Table I x 10^(k_pq, k_va, k_uc),
k in {-2, -1, 0, 1} per class, run the GPU ADMM from the cold start until primal infeasibility
 <= 1e-4 or `max_iters`, and record the iterations to 1e-2 / 1e-3 / 1e-4 and the best primal.
The GPU iterate equals the oracle's within the parity tolerance (tests/test_gpu_parity.py), so the
grid is searched here and the chosen rho is then confirmed on the oracle (tests/test_oracle_admm.py).

usage: python tools/rho_grid.py OUT.jsonl [max_iters] [cases] [extra k=v params ...]
"""
import dataclasses
import itertools
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_13145_b200 import inputs, ucac  # noqa: E402

TABLE1_RHO = {"case30": (5e5, 1e6, 1e6), "case118": (5e4, 1e5, 1e5), "case300": (5e3, 1e4, 1e4)}
THRESHOLDS = (1e-2, 1e-3, 1e-4)


def run(pb, pr, max_iters, chunk=1000):
    import torch
    c = ucac.Context(pb, pr)
    out = {"to": {}, "best_primal": float("inf")}
    done, secs, ti = 0, 0.0, 0
    while done < max_iters and ti < len(THRESHOLDS):
        thr = THRESHOLDS[ti]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        k = c.iterate(min(chunk, max_iters - done), stop_on_primal=thr)
        torch.cuda.synchronize()
        secs += time.perf_counter() - t0
        done += k
        r = c.report()
        out["best_primal"] = min(out["best_primal"], r["primal_inf"])
        while ti < len(THRESHOLDS) and r["primal_inf"] <= THRESHOLDS[ti]:
            out["to"][f"{THRESHOLDS[ti]:g}"] = {"iterations": done, "seconds": round(secs, 4),
                                                "outer": r["outer_total"], "objective": r["objective"]}
            ti += 1
    r = c.report()
    out.update(iterations=done, seconds=round(secs, 4), final_primal=r["primal_inf"], objective=r["objective"],
               outer=r["outer_total"], beta=r["beta"], z_inf=r["z_inf"], rz_inf=r["rz_inf"])
    c.close()
    return out


def main(out, max_iters="20000", cases="case30,case118,case300", *extra):
    kw = {}
    for e in extra:
        k, v = e.split("=")
        kw[k] = v
    max_iters = int(max_iters)
    f = open(out, "a")
    for name in cases.split(","):
        pb, pr0 = inputs.build_config(name)
        base = TABLE1_RHO[name]
        pr1 = dataclasses.replace(pr0, **{k: type(getattr(pr0, k))(float(v)) for k, v in kw.items()})
        for kp, kv, ku in itertools.product((-2, -1, 0, 1), repeat=3):
            rho = (base[0] * 10.0 ** kp, base[1] * 10.0 ** kv, base[2] * 10.0 ** ku)
            pr = dataclasses.replace(pr1, rho_pq=rho[0], rho_va=rho[1], rho_uc=rho[2])
            row = {"config": name, "k": [kp, kv, ku], "rho": rho, **kw}
            try:
                row.update(run(pb, pr, max_iters))
            except Exception as e:  # a diverging rho is a result, not a crash
                row["error"] = str(e)
            f.write(json.dumps(row) + "\n")
            f.flush()
            print(json.dumps({k: row.get(k) for k in ("config", "k", "best_primal", "final_primal", "to")}),
                  flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
