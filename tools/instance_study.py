"""Why do the synthetic case30/118/300-shaped configs not reach primal 1e-4?

Runs the GPU ADMM (parity-equal to the oracle) on instance variants of the synthetic generator --
generator minimum output (the synthetic recipe draws Pmin = Pmax U(0.1, 0.4); the MATPOWER
case30/118 files have Pmin = 0), no-load cost c0 against rho_uc, initially-off units, the
outer-loop beta cap -- and records primal infeasibility reached, the schedule's
movement over the last iterations, and the beta it ended at.

usage: python tools/instance_study.py OUT.jsonl [max_iters] [cases]
"""
import dataclasses
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_13145_b200 import inputs, ucac  # noqa: E402

TABLE1_RHO = {"case30": (5e5, 1e6, 1e6), "case118": (5e4, 1e5, 1e5), "case300": (5e3, 1e4, 1e4)}


def variants(pb):
    G = pb.ngen
    lowmin = pb.pmin * 0.25
    yield "base", pb, {}
    yield "pmin/4", dataclasses.replace(pb, pmin=lowmin, su_ramp=np.maximum(np.maximum(lowmin, pb.ramp_up), pb.p0),
                                        sd_ramp=np.maximum(np.maximum(lowmin, pb.ramp_up), pb.p0)), {}
    z = np.zeros(G)
    yield "pmin0", dataclasses.replace(pb, pmin=z, su_ramp=np.maximum(pb.ramp_up, pb.p0),
                                       sd_ramp=np.maximum(pb.ramp_up, pb.p0)), {}
    yield "c0/10", dataclasses.replace(pb, c0=pb.c0 * 0.1), {}
    yield "pmin/4,c0/10", dataclasses.replace(pb, pmin=lowmin, c0=pb.c0 * 0.1,
                                              su_ramp=np.maximum(np.maximum(lowmin, pb.ramp_up), pb.p0),
                                              sd_ramp=np.maximum(np.maximum(lowmin, pb.ramp_up), pb.p0)), {}
    p0on = np.clip(np.where(pb.u0 == 1, pb.p0, pb.pmin), pb.pmin, pb.pmax)
    yield "all-on-u0", dataclasses.replace(pb, u0=np.ones(G, np.int32), hold=np.zeros(G, np.int32), p0=p0on,
                                           su_ramp=np.maximum(pb.su_ramp, p0on), sd_ramp=np.maximum(pb.sd_ramp, p0on)), {}
    yield "uc_fixed(all on)", dataclasses.replace(pb, pmin=z, u_init=np.ones((G, pb.T), np.int8),
                                                  su_ramp=np.maximum(pb.ramp_up, pb.p0),
                                                  sd_ramp=np.maximum(pb.ramp_up, pb.p0)), {"uc_fixed": 1}
    yield "base,beta_max=1e5", pb, {"beta_max": 1e5}
    yield "pmin/4,beta_max=1e5", dataclasses.replace(
        pb, pmin=lowmin, su_ramp=np.maximum(np.maximum(lowmin, pb.ramp_up), pb.p0),
        sd_ramp=np.maximum(np.maximum(lowmin, pb.ramp_up), pb.p0)), {"beta_max": 1e5}


def run(pb, pr, max_iters):
    import torch
    c = ucac.Context(pb, pr)
    best, done, t0 = np.inf, 0, time.perf_counter()
    hit = {}
    trace = []
    u_prev = None
    flips = 0
    while done < max_iters:
        n = c.iterate(min(500, max_iters - done), stop_on_primal=1e-4)
        done += n
        r = c.report()
        best = min(best, r["primal_inf"])
        trace.append(round(r["primal_inf"], 6))
        for thr in (1e-2, 1e-3, 1e-4):
            if r["primal_inf"] <= thr and f"{thr:g}" not in hit:
                hit[f"{thr:g}"] = done
        if done >= max_iters - 1000:
            u = c.get_state()["u"]
            if u_prev is not None:
                flips += int(np.sum(u != u_prev))
            u_prev = u
        if r["primal_inf"] <= 1e-4:
            break
    torch.cuda.synchronize()
    r = c.report()
    st = c.get_state()
    out = dict(iterations=done, seconds=round(time.perf_counter() - t0, 3), best_primal=best,
               final_primal=r["primal_inf"], z_inf=r["z_inf"], rz_inf=r["rz_inf"], beta=r["beta"],
               outer=r["outer_total"], objective=r["objective"], to=hit, on_frac=float(np.mean(st["u"])),
               u_flips_last=flips, trace=trace[::max(1, len(trace) // 20)])
    c.close()
    return out


def main(out, max_iters="20000", cases="case30,case118,case300"):
    f = open(out, "a")
    for name in cases.split(","):
        pb0, pr0 = inputs.build_config(name)
        for rho_name, rho in (("bench", (pr0.rho_pq, pr0.rho_va, pr0.rho_uc)), ("table1", TABLE1_RHO[name])):
            if rho_name == "table1" and tuple(rho) == (pr0.rho_pq, pr0.rho_va, pr0.rho_uc):
                continue
            for vname, pb, kw in variants(pb0):
                pr = dataclasses.replace(pr0, rho_pq=rho[0], rho_va=rho[1], rho_uc=rho[2], **kw)
                row = {"config": name, "rho": rho_name, "variant": vname}
                try:
                    row.update(run(pb.normalized(), pr, int(max_iters)))
                except Exception as e:
                    row["error"] = str(e)
                f.write(json.dumps(row) + "\n")
                f.flush()
                print(json.dumps({k: row.get(k) for k in ("config", "rho", "variant", "best_primal", "final_primal",
                                                           "to", "beta", "u_flips_last", "on_frac")}), flush=True)




def grid2(out, max_iters="20000", cases="case30,case118,case300"):
    """second pass: minimum output scaled x {1, 1/4, 0}, beta capped at rho_min x {0.05, 0.5, 5, inf}
    (Sun & Sun's two-level ADMM needs rho >= 2 beta for the inner loop), Table I and bench rho"""
    f = open(out, "a")
    for name in cases.split(","):
        pb0, pr0 = inputs.build_config(name)
        for rho_name, rho in (("bench", (pr0.rho_pq, pr0.rho_va, pr0.rho_uc)), ("table1", TABLE1_RHO[name])):
            if rho_name == "table1" and tuple(rho) == (pr0.rho_pq, pr0.rho_va, pr0.rho_uc):
                continue
            for pscale in (1.0, 0.25, 0.0):
                lowmin = pb0.pmin * pscale
                pb = dataclasses.replace(pb0, pmin=lowmin, su_ramp=np.maximum(np.maximum(lowmin, pb0.ramp_up), pb0.p0),
                                         sd_ramp=np.maximum(np.maximum(lowmin, pb0.ramp_up), pb0.p0))
                for bfac in (0.05, 0.5, 5.0, None):
                    bmax = 1e12 if bfac is None else bfac * min(rho)
                    pr = dataclasses.replace(pr0, rho_pq=rho[0], rho_va=rho[1], rho_uc=rho[2], beta_max=bmax,
                                             beta0=min(pr0.beta0, bmax))
                    row = {"config": name, "rho": rho_name, "pmin_scale": pscale, "beta_max": bmax}
                    try:
                        row.update(run(pb.normalized(), pr, int(max_iters)))
                    except Exception as e:
                        row["error"] = str(e)
                    f.write(json.dumps(row) + "\n")
                    f.flush()
                    print(json.dumps({k: row.get(k) for k in ("config", "rho", "pmin_scale", "beta_max", "best_primal",
                                                               "final_primal", "to", "u_flips_last")}), flush=True)


def grid3(out, max_iters="20000", cases="case30,case118,case300"):
    """third pass: the schedule held at all-on (uc_fixed: the continuous multiperiod ACOPF of the
    NEXT-2 warm start), minimum output x {1, 0}, beta capped at rho_min x {0.05, 0.5, inf}"""
    f = open(out, "a")
    for name in cases.split(","):
        pb0, pr0 = inputs.build_config(name)
        G = pb0.ngen
        for rho_name, rho in (("bench", (pr0.rho_pq, pr0.rho_va, pr0.rho_uc)), ("table1", TABLE1_RHO[name])):
            if rho_name == "table1" and tuple(rho) == (pr0.rho_pq, pr0.rho_va, pr0.rho_uc):
                continue
            for pscale in (1.0, 0.0):
                lowmin = pb0.pmin * pscale
                pb = dataclasses.replace(pb0, pmin=lowmin, u_init=np.ones((G, pb0.T), np.int8),
                                         su_ramp=np.maximum(np.maximum(lowmin, pb0.ramp_up), pb0.p0),
                                         sd_ramp=np.maximum(np.maximum(lowmin, pb0.ramp_up), pb0.p0))
                for bfac in (0.05, 0.5, None):
                    bmax = 1e12 if bfac is None else bfac * min(rho)
                    pr = dataclasses.replace(pr0, rho_pq=rho[0], rho_va=rho[1], rho_uc=rho[2], beta_max=bmax,
                                             beta0=min(pr0.beta0, bmax), uc_fixed=1)
                    row = {"config": name, "rho": rho_name, "variant": "uc_fixed(all on)", "pmin_scale": pscale,
                           "beta_max": bmax}
                    try:
                        row.update(run(pb.normalized(), pr, int(max_iters)))
                    except Exception as e:
                        row["error"] = str(e)
                    f.write(json.dumps(row) + "\n")
                    f.flush()
                    print(json.dumps({k: row.get(k) for k in ("config", "rho", "pmin_scale", "beta_max", "best_primal",
                                                               "final_primal", "to", "iterations")}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "grid2":
        grid2(*sys.argv[2:])
    elif len(sys.argv) > 1 and sys.argv[1] == "grid3":
        grid3(*sys.argv[2:])
    else:
        main(*sys.argv[1:])
