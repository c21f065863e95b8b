#!/usr/bin/env python
"""Benchmark of the UC-ACOPF two-level ADMM hot path (arXiv 2310.13145) on B200.

A "step" is one inner ADMM iteration = all hot-path rows of SURVEY.md 8(a): UC DP (7a),
generator closed form + batched branch TRON solves (7b), ubar box-QPs (7c), bus closed form
(7d), z/y for every coupling row (7e-7f), residual reduction, inner test and outer
(lambda, beta) update.  Workload at N=1: BASELINE.json configs[4], the 2869-bus
pegase-shaped synthetic grid with T=48 (the largest single-GPU configuration; the north
star's "largest case").  Inputs are seeded synthetic data (paper_2310_13145_b200.inputs).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ucac|reference] [--config NAME]

Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle (oracle/) on the
host cores on a bounded sample of the same workload (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ADMM iters/sec & branch-subproblem solves/sec; time-to-residual 1e-4, 1/2/4/8 B200"
UNIT = "ADMM inner iterations/s"
# SASS-executed FP64 flops per TRON Newton iteration of the two branch kernels: lane-level SASS
# counts of the same launches (2 DFMA + DADD + DMUL) / the Newton iterations the solver counted in
# them (tools/calibrate_flops.py; profiles/r01/flops_calibration.json) -- reported beside the
# algorithmic figure (the oracle's counted flops of the same solves, R55), which sets roofline.frac.
FLOPS_PER_NEWTON_FAST = 717.0
FLOPS_PER_NEWTON_AL = 2147.0


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except Exception:
        return {}


def fp64_peak_tflops(sm_mhz: float) -> float:
    """B200 FP64 (non-tensor) peak: 148 SMs x 64 FP64 FMA lanes/clk x 2 flop."""
    return 148 * 64 * 2 * sm_mhz * 1e6 / 1e12


class ClockSampler:
    """SM clock and clock-event reasons sampled DURING the timed region: NVML polled every
    millisecond from a thread (the timed region lasts tens of ms, shorter than nvidia-smi's own
    start-up), nvidia-smi -lms 100 if NVML is unavailable."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.rows = []          # (sm_mhz, max_mhz, reason mask)
        self.stop = threading.Event()
        self.t = None
        self.src = "none"

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def loop():
                while not self.stop.is_set():
                    try:
                        self.rows.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), mx, get_reasons(h)))
                    except Exception:
                        pass
                    time.sleep(0.001)
            self.src = "nvml"
            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
            time.sleep(0.005)
        except Exception:
            self._smi()
        return self

    def _smi(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_power_cap,"
                  "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")
        try:
            proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={fields}",
                                     "--format=csv,noheader,nounits", "-lms", "100"],
                                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            return
        self.src = "nvidia-smi"
        bits = [0x8, 0x4, 0x40, 0x20]

        def read():
            for line in proc.stdout:
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 6 and p[0].replace(".", "").isdigit():
                    mask = sum(b for b, v in zip(bits, p[2:6]) if v.lower() == "active")
                    self.rows.append((float(p[0]), float(p[1]), mask))
                if self.stop.is_set():
                    break
            proc.terminate()
        self.t = threading.Thread(target=read, daemon=True)
        self.t.start()
        time.sleep(1.0)   # nvidia-smi start-up

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"], "samples": 0,
                    "source": self.src}
        reasons = sorted({n for _, _, m in self.rows for b, n in self.REASONS.items() if m & b})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows), "source": self.src}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample(pb, pr, steps: int, budget_s: float, omp: bool = False):
    """time the oracle (as it stands; single thread, or its all-core OpenMP build) on a bounded
    number of iterations."""
    import oracle
    o = oracle.Oracle(pb, pr, omp=omp)
    t0 = time.perf_counter()
    n = 0
    while n < steps:
        o.iterate(1)
        n += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return n, dt, o.report()


REF_BUDGET_S = 150.0


def run_reference(args, pb, pr, rank, world):
    if rank != 0:
        return
    import numpy as np  # noqa: F401
    import oracle
    # the all-core build of the oracle (same source with OpenMP over the components of each step,
    # reductions in canonical order: bitwise the single-thread iterates) on every host core
    ncores = oracle.threads(os.cpu_count() or 1)
    o = oracle.Oracle(pb, pr, omp=True)
    for _ in range(args.warmup):
        o.iterate(1)
    # a bounded sample: at most REF_BUDGET_S seconds of timed oracle iterations (the oracle runs
    # ~3 it/s on the pegase config), so a large --steps still ends within a few minutes
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        o.iterate(1)
        times.append(time.perf_counter() - t0)
        if sum(times) > REF_BUDGET_S:
            break
    tot = sum(times)
    v = len(times) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(times), "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, paper_2310_13145_b200.inputs)",
        "config": {"workload": f"{args.config} (B={pb.nbus}, G={pb.ngen}, L={pb.nbranch}, T={pb.T})",
                   "rows": pb.nrows(), "branch_solves_per_step": pb.nbranch * pb.T, "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": ncores, "kind": "oracle", "cpu_model": cpu_model(),
                         "sample": f"{len(times)} timed inner iterations (of {args.steps} requested, {REF_BUDGET_S:.0f} s cap) after {args.warmup} warm-up, "
                                   f"C oracle, all-core OpenMP build (-O2 -ffp-contract=off -fopenmp, {ncores} threads)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "branch_solves_per_s": v * pb.nbranch * pb.T,
    }
    print(json.dumps(line), flush=True)


DP_METRIC = "UC DP instances/s (batched Alg. 2, Fig. 1 shape)"
DP_SIZES = [(1000, 24), (1000, 48), (1000, 96), (1000, 168), (10000, 24), (10000, 48), (10000, 96), (10000, 168)]


def run_dp(args, rank, world):
    """NEXT-1: batched UC DP on random stage costs, G in {1e3, 1e4}, T = 24..168.
    Device-timed ucac_dp_batch calls (inputs resident, L2 flushed between calls); the CPU
    baseline is the oracle's DP (one core) on the same instances; outputs checked bitwise
    against it on a sample.  Value = instances/s at the largest size."""
    if rank != 0:
        return
    import numpy as np
    import torch

    import oracle
    from paper_2310_13145_b200 import inputs, ucac
    torch.cuda.set_device(0)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    peaks = measured_peaks()
    rows = []
    with ClockSampler(0) as clk:
        for G, T in DP_SIZES:
            L, tu, td, u0, hold = inputs.dp_workload(G, T, seed=G + T)
            dL = torch.from_numpy(L.reshape(-1)).cuda()
            dint = [torch.from_numpy(a).cuda() for a in (tu, td, u0, hold)]
            sched = torch.zeros(G * T, dtype=torch.int8, device="cuda")
            cost = torch.zeros(G, dtype=torch.float64, device="cuda")
            st = torch.cuda.current_stream()

            def call():
                ucac.dp_batch_device(G, T, dL.data_ptr(), *[a.data_ptr() for a in dint], sched.data_ptr(),
                                     cost.data_ptr(), st.cuda_stream)
            for _ in range(max(args.warmup, 3)):
                call()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
            for a, b in ev:
                flush.zero_()
                a.record(st)
                call()
                b.record(st)
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
            # oracle on a bounded sample (<= 2 s per size), bitwise check on it
            s_h, c_h = sched.cpu().numpy().reshape(G, T), cost.cpu().numpy()
            t0, n = time.perf_counter(), 0
            ok = True
            while n < G and time.perf_counter() - t0 < 2.0:
                so, co = oracle.dp_solve(L[n], int(tu[n]), int(td[n]), int(u0[n]), int(hold[n]))
                ok = ok and bool(np.array_equal(so, s_h[n])) and bool(co == c_h[n])
                n += 1
            cpu_s = (time.perf_counter() - t0) / n
            byts = G * T * (4 * 8 + 1) + G * (4 * 4 + 8)
            rows.append({"G": G, "T": T, "ms": ms, "instances_per_s": G / (ms * 1e-3),
                         "alg_GBps": byts / (ms * 1e-3) / 1e9, "us_per_period": ms * 1e3 / T,
                         "cpu_instances_per_s": 1.0 / cpu_s, "cpu_sample": n, "bitwise_equal_on_sample": ok})
    big = rows[-1]
    hbm = peaks.get("hbm_gbs", 6650.0)
    t10k = [r for r in rows if r["G"] == 10000]
    line = {
        "metric": DP_METRIC, "value": big["instances_per_s"], "unit": "DP instances/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": big["ms"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (inputs.dp_workload, seeded)",
        "config": {"workload": f"UC DP batch G={big['G']} T={big['T']} (NEXT-1, Fig. 1 shape)",
                   "l2": "flushed (256 MiB memset) before every timed call"},
        "roofline": {"bound": "hbm", "kernel": "k_dp_batch", "achieved": big["alg_GBps"], "peak": hbm,
                     "unit": "GB/s", "frac": big["alg_GBps"] / hbm, "traffic": None,
                     "note": "the O(T) backward recursion of each instance is sequential (one lane); "
                             "bytes = stage costs 32 B + schedule 1 B per (g,t)"},
        "linear_in_T": {"us_per_period_G10000": {r["T"]: r["us_per_period"] for r in t10k}},
        "table": rows,
        "cpu_baseline": {"value": big["cpu_instances_per_s"], "unit": "DP instances/s", "cores": 1, "kind": "oracle",
                         "sample": f"{big['cpu_sample']} instances of G={big['G']} T={big['T']}, C oracle orc_dp"},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def run_warmstart(args, pb, pr, rank):
    """NEXT-2: the UC warm start through ucac_uc_warm_start (context creation,
    held-schedule ACOPF iterations, device Hamming costs + batched DP repair), wall clock, against
    the oracle's warm start on the same workload and iteration count (one core)."""
    if rank != 0:
        return
    import numpy as np

    import oracle
    from paper_2310_13145_b200 import ucac
    iters = args.steps
    ucac.uc_warm_start(pb, pr, 1)                     # warm-up (library load, first context)
    t0 = time.perf_counter()
    u = ucac.uc_warm_start(pb, pr, iters)
    gpu_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    uo, _ = oracle.uc_warm_start(pb, pr, iters)
    cpu_s = time.perf_counter() - t0
    line = {
        "metric": "UC warm starts/s (NEXT-2: held-schedule ACOPF + DP repair)", "value": 1.0 / gpu_s,
        "unit": "warm starts/s", "n_gpus": 1, "steps": iters, "warmup": 1, "ms_per_step": 1e3 * gpu_s / iters,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, paper_2310_13145_b200.inputs)",
        "config": {"workload": f"{args.config} warm start, {iters} held-schedule iterations, threshold 1e-3 pu"},
        "units_on": int(u.sum()), "units_on_of": int(u.size), "schedule_equal_to_oracle": bool(np.array_equal(u, uo)),
        "cpu_baseline": {"value": 1.0 / cpu_s, "unit": "warm starts/s", "cores": 1, "kind": "oracle",
                         "sample": f"the same warm start ({iters} iterations) by the C oracle"},
        "note": "wall clock including context creation (H2D of the problem) and the D2H of the schedule",
    }
    print(json.dumps(line), flush=True)


def ncu_traffic() -> dict:
    """DRAM bytes per launch (read + write) of the dominant kernels from the committed ncu
    --set full capture (profiles/r02/ncu_traffic.json, tools/ncu_traffic.py; cold-cache, one launch each)."""
    try:
        path = os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json")
        if not os.path.exists(path):
            path = os.path.join(ROOT, "profiles", "r01", "ncu_traffic.json")
        d = json.load(open(path))
        out = {k: v["traffic"] for k, v in d["kernels"].items()}
        out["_note"] = "dram bytes per launch, " + d["source"]
        return out
    except (OSError, ValueError, KeyError):
        return {}


def time_to_residual(name: str = "case9", targets=(1e-2, 1e-3, 1e-4), cap: int = 5000, chunk: int = 25):
    """The "time-to-residual 1e-4" part of the metric: from the cold start, the GPU iterates in
    chunks with the on-device primal stop (P:486 primal infeasibility) until the next target is
    met; wall time around each chunk with a device synchronize on both sides (ucac_create not
    included).  Every target is reported as reached (iterations, seconds) or not within `cap`
    iterations, with the best primal seen (the synthetic case30/118/300-shaped
    configs stall at 1e-2..1e-1, as the paper's own UC runs end at 1.8e-3..1.2e-2)."""
    import torch
    from paper_2310_13145_b200 import inputs, ucac
    pb, pr = inputs.build_config(name)
    c = ucac.Context(pb, pr)
    done, secs, r, best = 0, 0.0, None, float("inf")
    reached = {}
    ti = 0
    while done < cap and ti < len(targets):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        k = c.iterate(min(chunk, cap - done), stop_on_primal=targets[ti])
        torch.cuda.synchronize()
        secs += time.perf_counter() - t0
        done += k
        r = c.report()
        best = min(best, r["primal_inf"])
        while ti < len(targets) and r["primal_inf"] <= targets[ti]:
            reached[f"{targets[ti]:g}"] = {"iterations": done, "seconds": round(secs, 5), "outer": r["outer_total"],
                                          "objective": r["objective"]}
            ti += 1
    c.close()
    return {"config": f"{name} T={pb.T}, cold start, rho {(pr.rho_pq, pr.rho_va, pr.rho_uc)}",
            "target_primal": targets[-1], "reached": reached, "all_reached": len(reached) == len(targets),
            "iterations_run": done, "seconds": round(secs, 5), "best_primal": best,
            "final_primal": r["primal_inf"] if r else None}


def problem_bytes(pb) -> int:
    import numpy as np
    tot = 0
    for v in vars(pb).values():
        if isinstance(v, np.ndarray):
            tot += v.nbytes
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ucac", choices=["ucac", "reference"])
    ap.add_argument("--config", default="pegase2869")
    ap.add_argument("--T", type=int, default=None, help="override the config's horizon (SURVEY 8(a) stress: pegase T=168)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cut", default="bus", choices=["bus", "time"],
                    help="N > 1: bus-graph cut (DESIGN.md 9, default) or time cut (NEXT-4(c))")
    ap.add_argument("--ttr-cap", type=int, default=20000,
                    help="iteration cap of the time-to-residual runs on configs[1]-[3]")
    ap.add_argument("--no-ttr-all", action="store_true", help="time-to-residual on configs[0] only")
    ap.add_argument("--kernel-window", type=int, default=100,
                    help="eager iterations (at least --steps) for the per-kernel figures and the roofline")
    ap.add_argument("--kernel-window-start", type=int, default=106,
                    help="first iteration of that window (the default 100-step run's: warm-up 5 + 100 timed + 1)")
    ap.add_argument("--p2p", action="store_true",
                    help="N > 1 with --cut time: device-initiated NVLink exchanges (CUDA IPC peer stores) instead of NCCL")
    ap.add_argument("--selfcheck-iters", type=int, default=10,
                    help="N > 1: iterations of the rank-assembled vs 1-GPU bitwise self-check (0 = off)")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--workload", default="admm", choices=["admm", "dp", "warmstart"],
                    help="admm: the inner-iteration hot path (default); dp: NEXT-1 batched UC DP; "
                         "warmstart: NEXT-2 UC warm start")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    from paper_2310_13145_b200 import inputs
    pb, pr = inputs.build_config(args.config, args.T)

    if args.impl == "reference":
        run_reference(args, pb, pr, rank, world)
        return
    if args.workload == "dp":
        run_dp(args, rank, world)
        return
    if args.workload == "warmstart":
        run_warmstart(args, pb, pr, rank)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2310_13145_b200 import ucac

    branch_w = None
    if world > 1 and args.cut == "bus":
        # partition weights from the expected branch-solve work: a short 1-GPU run
        # (deterministic, so every rank computes the same weights) marks the (l,t) whose thermal AL
        # has been active (mu != 0); weight = 1 + 8 x the branch's active share (an AL solve costs
        # ~8 fast-path solves, R55)
        wc = ucac.Context(pb, pr)
        wc.iterate(20)
        al = wc.get_state()["al"].reshape(pb.nbranch, pb.T, 3)
        wc.close()
        branch_w = 1.0 + 8.0 * np.mean((al[:, :, 0] != 0) | (al[:, :, 1] != 0), axis=1)

    def make_dist():
        """N > 1: the bus-graph cut or the time cut (9.1) of the same problem"""
        if world == 1:
            return None
        obj = [ucac.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return {"rank": rank, "nranks": world, "comm_mode": 0, "nccl_id": obj[0], "cut": int(args.cut == "time"),
                "branch_w": branch_w}

    def make_ctx():
        c = ucac.Context(pb, pr, dist=make_dist())
        if world > 1 and args.p2p:
            blobs = [None] * world
            dist.all_gather_object(blobs, c.p2p_export())
            c.p2p_import(blobs)
        return c

    ctx = make_ctx()
    stream = torch.cuda.ExternalStream(ctx.stream)
    sizes = ctx.sizes()
    l2_flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    # warm-up
    ctx.iterate(args.warmup)
    torch.cuda.synchronize()
    rep0 = ctx.report()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(v):
        if world == 1:
            return v
        t = torch.tensor([float(v)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(v):
        if world == 1:
            return v
        t = torch.tensor([float(v)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # ---- timed region: one graph-launched step per event pair, L2 flushed between steps
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            for k in range(args.steps):
                l2_flush.zero_()
                starts[k].record(stream)
                ctx.iterate(1)
                ends[k].record(stream)
        barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    tot_ms = allmax(sum(step_ms))
    rep1 = ctx.report()
    newton = allsum(rep1["tron_iters"] - rep0["tron_iters"])
    peaks = measured_peaks()
    clocks = clk.summary()

    # ---- per-kernel device times (same kernels launched eagerly with an event pair each), 1 GPU
    roofline, kernels, kms = None, None, None
    kw = args.steps
    fused = False
    fp64_meas = None
    if world == 1:
        # a fixed window of >= 100 eager iterations right after the timed region, so that the
        # per-kernel figures do not depend on --steps (the AL tail's length is set by its longest
        # solve, its flops by the number of thermal-active lines, which grows over the first ~50)
        kw = max(args.steps, args.kernel_window)
        # ... starting at a fixed iteration (untimed graph iterations up to it when --steps is small),
        # so that runs with different --steps report the same window
        k0 = args.warmup + args.steps + 1
        if k0 < args.kernel_window_start:
            ctx.iterate(args.kernel_window_start - k0)
            k0 = args.kernel_window_start
        repk = ctx.report()
        kms, klaunch = ctx.iterate_timed(kw)
        rep2 = ctx.report()
        n_al = rep2["al_tron_iters"] - repk["al_tron_iters"]
        n_fast = rep2["tron_iters"] - repk["tron_iters"] - n_al
        al_solves = (rep2["al_active"] - repk["al_active"]) / kw
        ksum = sum(kms.values())
        # the FP64 (non-tensor) peak measured in this process: DFMA chains, ucac_measure_fp64_peak
        with ClockSampler(local) as clk64:
            fp64_meas = ucac.measure_fp64_peak()
        fp64_meas["clocks"] = clk64.summary()
        fp64 = fp64_meas["tflops"]
        hbm = peaks.get("hbm_gbs", 6650.0)
        fp64_note = ("FP64 non-tensor peak measured in this run (DFMA-chain microbenchmark, "
                     "ucac_measure_fp64_peak; see fp64_peak)")
        # algorithmic flops (R55): the oracle replays one iteration from the GPU's state and counts the
        # flops of its branch solves (per-operation counts of the plain algorithm); per fast-path solve
        # and per AL solve, times the GPU's live solve counts
        alg = None
        if rank == 0:
            import oracle
            oracle.threads(os.cpu_count() or 1)
            o = oracle.Oracle(pb, pr, omp=True)
            o.set_state(ctx.get_state())
            o.iterate(1)
            ro = o.report()
            o.close()
            LT = pb.nbranch * pb.T
            alg = {"flops_per_fast_solve": ro["flops_fast"] / LT,
                   "flops_per_al_solve": ro["flops_al"] / max(1, ro["al_active"]),
                   "oracle_newton_per_fast_solve": ro["newton_fast"] / LT,
                   "oracle_newton_per_al_solve": ro["newton_al"] / max(1, ro["al_active"]),
                   "oracle_al_solves": ro["al_active"],
                   "source": "oracle one-step replay from the GPU state after the per-kernel window (R55)"}
        kernels = {}
        for k, n, fpn, alg_flops in (
                ("k_branch", n_fast, FLOPS_PER_NEWTON_FAST,
                 alg["flops_per_fast_solve"] * pb.nbranch * pb.T if alg else None),
                ("k_branch_al", n_al, FLOPS_PER_NEWTON_AL,
                 alg["flops_per_al_solve"] * al_solves if alg else None)):
            sass = n * fpn / (kms[k] * 1e-3) / 1e12
            a_ = alg_flops / (kms[k] / kw * 1e-3) / 1e12 if alg_flops is not None else sass
            kernels[k] = {"bound": "alu", "achieved": a_, "peak": fp64, "unit": "TFLOP/s", "frac": a_ / fp64,
                          "flops_per_step_algorithmic": alg_flops,
                          "sass_achieved": sass, "sass_frac": sass / fp64,
                          "newton_iters_per_step": n / kw, "sass_flops_per_newton": fpn,
                          "ms_per_step": kms[k] / kw, "share_of_step": kms[k] / ksum}
        kernels["k_branch_al"]["al_solves_per_step"] = al_solves
        fused = kms.get("k_rows", 0.0) + kms.get("k_rows_late", 0.0) < 1e-3 * kms["k_bus"]
        for k in (("k_bus",) if fused else ("k_rows", "k_bus")) + ("k_ubar", "k_genx", "k_gen"):
            t = kms[k] + kms.get(k + "_late", 0.0)       # early + late launches
            nbytes = sizes["alg_bytes"][k] + (sizes["alg_bytes"]["k_rows"] if fused and k == "k_bus" else 0)
            gbs = nbytes * kw / (t * 1e-3) / 1e9
            name = "k_bus+rows(+late)" if fused and k == "k_bus" else k + ("+late" if k + "_late" in kms else "")
            kernels[name] = {
                "bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                "ms_per_step": t / kw, "share_of_step": t / ksum}
        dom = max(("k_branch", "k_branch_al"), key=lambda k: kms[k])
        traffic = ncu_traffic()
        if max(kms, key=kms.get) == dom:
            roofline = dict(kernels[dom], kernel=dom, traffic=traffic.get(dom),
                            traffic_note=traffic.get("_note"),
                            peak_note=fp64_note + "; achieved = algorithmic flops per step (the oracle's counted "
                                      "flops per solve x the GPU's live solve counts, R55) / the kernel's "
                                      "event-timed ms per step; sass_* = Newton iterations x ncu SASS flops")
        else:
            dom = max(kms, key=kms.get)
            roofline = {"bound": "hbm", "kernel": dom, "achieved": sizes["alg_bytes"][dom] * kw /
                        (kms[dom] * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s", "traffic": traffic.get(dom),
                        "ms_per_step": kms[dom] / kw, "share_of_step": kms[dom] / ksum}
            roofline["frac"] = roofline["achieved"] / hbm

    # ---- e2e: the public API from host buffers (create = H2D of the problem, iterate,
    #      residuals + solution = D2H), per step = one inner iteration, max over ranks
    # the result is read into page-locked host buffers the caller owns and reuses (allocated once,
    # outside the timed region, as the inputs' pinned copies would be)
    sol_buf = {k: torch.empty(n, dtype=torch.int8 if t == np.int8 else torch.float64, pin_memory=True).numpy()
               for k, (n, t) in ctx.solution_shapes().items()}

    def e2e_run():
        barrier()
        t0 = time.perf_counter()
        c2 = make_ctx()
        ta = time.perf_counter()
        c2.iterate(args.steps)
        _ = c2.report()
        tb = time.perf_counter()
        sol_ = c2.solution(out=sol_buf)
        t1 = time.perf_counter()
        c2.close()
        return t1 - t0, sol_, {"create_ms": 1e3 * (ta - t0), "iterate_report_ms": 1e3 * (tb - ta),
                               "solution_ms": 1e3 * (t1 - tb)}

    e2e_run()   # untimed warm-up of the public-API path (first-call driver work)
    dt, sol, parts = e2e_run()
    e2e_s = allmax(dt)
    h2d = problem_bytes(pb.normalized()) * world
    d2h = allsum(sum(v.nbytes for v in sol.values()) + 200)
    e2e = {"value": args.steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d / args.steps),
           "d2h_bytes_per_step": int(d2h / args.steps),
           "note": "ucac_create(host arrays) + ucac_iterate(K) + ucac_residuals + ucac_get_solution (into "
                   "caller-owned page-locked buffers allocated once), wall clock, after one untimed warm-up "
                   "run of the same calls", "parts_rank0": parts}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        n, dt, _ = oracle_sample(pb, pr, 10 ** 6, args.cpu_budget)
        ncores = oracle.threads(os.cpu_count() or 1)
        n2, dt2, _ = oracle_sample(pb, pr, 10 ** 6, args.cpu_budget, omp=True)
        cpu = {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{n} inner iterations of the same workload from the cold start, "
                         f"single-threaded C oracle ({dt:.1f} s budget {args.cpu_budget:.0f} s)",
               "all_cores": {"value": n2 / dt2, "unit": UNIT, "cores": ncores, "nproc": os.cpu_count(),
                             "cpu_model": cpu_model(), "kind": "oracle (all-core OpenMP build, bitwise the same iterates)",
                             "sample": f"{n2} inner iterations from the cold start ({dt2:.1f} s, budget {args.cpu_budget:.0f} s)"}}

    ttr = None
    if rank == 0 and world == 1:
        ttr = {"case9": time_to_residual("case9", targets=(1e-4,))}
        if not args.no_ttr_all:
            for nm in ("case30", "case118", "case300"):
                ttr[nm] = time_to_residual(nm, cap=args.ttr_cap, chunk=250)

    # N > 1: on-box self-check -- a fresh partitioned run of K iterations, the local states gathered
    # and assembled on rank 0, compared bitwise with a 1-GPU run of the same K iterations
    selfcheck = None
    if world > 1 and args.selfcheck_iters > 0:
        kc = args.selfcheck_iters
        cchk = make_ctx()
        info = cchk.comm_info()
        cchk.iterate(kc)
        torch.cuda.synchronize()
        parts = [None] * world
        dist.all_gather_object(parts, ucac.local_part(cchk))
        cchk.close()
        if rank == 0:
            one = ucac.Context(pb, pr)
            one.iterate(kc)
            ref = one.get_state()
            one.close()
            got = ucac.assemble_parts(pb, parts)
            bad = [k for k in ref if k != "scal" and not np.array_equal(got[k], ref[k])]
            if not np.array_equal(got["scal"][[0, 2, 3, 4]], ref["scal"][[0, 2, 3, 4]]):
                bad.append("scal")
            selfcheck = {"iterations": kc, "bitwise_equal_to_1gpu": not bad, "differ": bad,
                         "nccl_nranks": info["nranks"], "cut": args.cut, "p2p": bool(args.p2p)}

    if rank == 0:
        v = args.steps / (tot_ms * 1e-3)
        line = {
            "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, paper_2310_13145_b200.inputs)",
            "config": {"workload": f"{args.config} (B={pb.nbus}, G={pb.ngen}, L={pb.nbranch}, T={pb.T})",
                       "rows": pb.nrows(), "branch_solves_per_step": pb.nbranch * pb.T,
                       "l2": "flushed (256 MiB memset) before every timed step",
                       "parallelism": (f"{args.cut} cut over {world} GPUs, NCCL exchange" if world > 1
                                       else "single GPU")},
            "branch_solves_per_s": v * pb.nbranch * pb.T,
            "newton_iters_per_s": newton / (tot_ms * 1e-3),
            "newton_per_solve": newton / max(1, args.steps * pb.nbranch * pb.T),
            "branch_stats_per_step": {k: (rep1[k] - rep0[k]) / args.steps
                                      for k in ("tron_capped", "al_active", "al_capped")},
            "primal_inf": rep1["primal_inf"],
            "roofline": roofline,
            "fp64_peak": fp64_meas,
            "algorithmic_flops": alg if world == 1 else None,
            "kernels": kernels,
            "kernel_ms_per_step": {k: v_ / kw for k, v_ in kms.items()} if kms else None,
            "kernel_window": ({"iterations": kw, "first": k0,
                               "note": "per-kernel figures (kernels, roofline, kernel_ms_per_step): the same kernels "
                                       "launched eagerly with an event pair each over this window of iterations, "
                                       "after the timed region"} if kms else None),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "time_to_residual": ttr,
            "multi_gpu_selfcheck": selfcheck,
            # 1 GPU: branch, gen (head), genx, bus, rows, ubar, fold, branch_al, bus_late, rows_late and
            # the tail gen (9 with the rows fused into the bus kernels, UCAC_FUSE_ROWS)
            "gpu_launches": ((9 if fused else 11) if world == 1 else (15 if args.cut == "bus" else 16)) * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
