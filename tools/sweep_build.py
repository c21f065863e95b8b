"""Rebuild libucac.so with each set of extra nvcc flags and run a short bench for each
(tuning sweeps on the GPU box; restores the default build at the end).
usage: python tools/sweep_build.py "-DFOO=1" "-DBAR=2 -DBAZ=3" ...
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(flags, steps=20):
    # a variant is "nvcc flags" or "src:k_branch.cu=path [nvcc flags]" (compile another file for a unit)
    src = ""
    if flags.startswith("src:"):
        src, _, flags = flags[4:].partition(" ")
    env = dict(os.environ, UCAC_EXTRA_NVCC=flags, UCAC_SRC_OVERRIDE=src)
    subprocess.run([sys.executable, os.path.join(ROOT, "paper_2310_13145_b200", "build.py"), "--force"], env=env,
                   check=True, capture_output=True)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", str(steps), "--warmup", "5",
                          "--no-cpu-baseline"], capture_output=True, text=True, env=env)
    line = [x for x in out.stdout.splitlines() if x.startswith("{")]
    if not line:
        return {"flags": flags, "error": out.stderr[-500:]}
    d = json.loads(line[-1])
    return {"flags": (src + " " + flags).strip(), "value": round(d["value"], 1), "ms_step": round(d["ms_per_step"], 4),
            "kernels_ms": {k: round(v, 4) for k, v in d["kernel_ms_per_step"].items()},
            "newton_per_solve": round(d["newton_per_solve"], 3)}


if __name__ == "__main__":
    variants = sys.argv[1:] or [""]
    for v in variants:
        print(json.dumps(run(v)), flush=True)
    subprocess.run([sys.executable, os.path.join(ROOT, "paper_2310_13145_b200", "build.py"), "--force"], check=True,
                   capture_output=True)
