"""FP64 flops per TRON Newton iteration of the two branch kernels, for bench.py's roofline.

Run under ncu (one GPU), e.g.
  ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,\
smsp__sass_thread_inst_executed_op_dmul_pred_on.sum -k regex:k_branch --csv --log-file gpurun_out/flops.csv \
      python tools/calibrate_flops.py gpurun_out/flops_counts.json
This script runs WARM eager iterations, then CAL iterations and records, per iteration, the Newton
iterations the solver counted (fast path = all - inside the AL, AL); the ncu log holds the lane
FP64 instruction counts of the same launches.  `python tools/calibrate_flops.py --reduce csv json`
divides them (flops = 2 DFMA + DADD + DMUL).
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

WARM, CAL = 8, 4


def run(out):
    from paper_2310_13145_b200 import inputs, ucac
    pb, pr = inputs.build_config("pegase2869")
    c = ucac.Context(pb, pr)
    c.iterate_timed(WARM)
    rows = []
    for _ in range(CAL):
        r0 = c.report()
        c.iterate_timed(1)
        r1 = c.report()
        al = r1["al_tron_iters"] - r0["al_tron_iters"]
        rows.append({"fast": r1["tron_iters"] - r0["tron_iters"] - al, "al": al})
    json.dump({"warm": WARM, "cal": rows}, open(out, "w"))


def reduce(csv_path, json_path):
    cnt = json.load(open(json_path))
    rows = list(csv.reader(open(csv_path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    per = {}
    for r in rows[i + 1:]:
        d = dict(zip(h, r))
        # "void (anonymous namespace)::k_branch<0>(Dev)" -> "k_branch" (template instantiations)
        key = (int(d["ID"]), d["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0])
        per.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    launches = {"k_branch": [], "k_branch_al": []}
    for (lid, name), m in sorted(per.items()):
        f = 2 * m["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"] + \
            m["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"] + m["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]
        if name in launches:
            launches[name].append(f)
    w = cnt["warm"]
    fast = sum(launches["k_branch"][w:w + len(cnt["cal"])])
    al = sum(launches["k_branch_al"][w:w + len(cnt["cal"])])
    nf = sum(r["fast"] for r in cnt["cal"])
    na = sum(r["al"] for r in cnt["cal"])
    print(json.dumps({"flops_per_newton_fast": fast / nf, "flops_per_newton_al": al / na,
                      "newton_fast": nf, "newton_al": na, "iterations": len(cnt["cal"])}))


if __name__ == "__main__":
    if sys.argv[1] == "--reduce":
        reduce(sys.argv[2], sys.argv[3])
    else:
        run(sys.argv[1])
