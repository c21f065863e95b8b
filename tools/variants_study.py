"""NEXT-3 ablation (R47): for each formulation variant, the GPU
iterations to primal infeasibility <= 1e-4, the objective and the device time (one B200).
usage: python tools/variants_study.py [out.json]"""
import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_13145_b200 import inputs, ucac  # noqa: E402

NAMES = {0: "paper reading (fast path + AL when violated)", 1: "AL for every rated branch (ExaTron-faithful)",
         2: "w-bar clipped to the voltage box (SPEC)", 3: "1 + 2", 4: "ramp-aware DP (NEXT-4a)",
         8: "no angle consensus rows (SPEC)", 16: "literal Eq. 5f ramp-down (A3)"}


def main(out=None):
    import torch
    rows = []
    for name in ("case30", "case118", "case300"):
        pb, pr = inputs.build_config(name)
        for v in (0, 1, 2, 3, 4, 8, 16):
            c = ucac.Context(pb, dataclasses.replace(pr, variant=v))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            n = c.iterate(20000, stop_on_primal=1e-4)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            r = c.report()
            rows.append({"config": name, "variant": v, "what": NAMES[v], "iterations": n,
                         "primal_inf": r["primal_inf"], "objective": r["objective"], "seconds": dt,
                         "al_solves": r["al_active"], "newton_iters": r["tron_iters"]})
            print(json.dumps(rows[-1]), flush=True)
            c.close()
    if out:
        json.dump(rows, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
