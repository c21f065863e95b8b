"""Build libucac.so (the CUDA hot path behind include/ucac.h) in-tree with nvcc for sm_100a.

Translation units and their arithmetic contract:
  k_branch.cu  batched TRON branch solves          -fmad=true  (FP64-pipe bound; FMA)
  k_gen.cu     UC DP + generator x-update + S0      -fmad=false (bit-exact DP decisions)
  k_sweep.cu   bus / ubar / z / y / reductions      -fmad=false (oracle operation order)
  ucac.cu      host runtime (C ABI)
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_build")
LIB = os.path.join(OUT, "libucac.so")
INCLUDE = os.path.join(ROOT, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC,
          "--expt-relaxed-constexpr"]
UNITS = {
    "k_branch.cu": ["-fmad=true"],
    "k_gen.cu": ["-fmad=false"],
    "k_sweep.cu": ["-fmad=false"],
    "k_strict.cu": ["-fmad=false"],
    "k_measure.cu": [],
    "k_xchg.cu": [],
    "ucac.cu": [],
    "partition.cu": [],
}


def _nccl_dirs():
    """The NCCL that PyTorch loads (the venv's nvidia-nccl wheel): libucac is compiled against its
    header and linked to its libnccl.so.2 with an rpath, so that both libraries resolve to the same
    NCCL whichever is imported first (linked to the system libnccl.so.2 instead, loading libucac
    before torch made torch's own NCCL symbols unresolvable).  (None, None) if absent."""
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        for base in (list(spec.submodule_search_locations) if spec and spec.submodule_search_locations else []):
            inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
            if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
                return inc, lib
    except Exception:
        pass
    return None, None


NCCL_INC, NCCL_LIB = _nccl_dirs()
if NCCL_LIB:
    COMMON = COMMON + ["-I", NCCL_INC]
    LIBS = ["-L", NCCL_LIB, "-Xlinker", "-l:libnccl.so.2", "-Xlinker", "-rpath", "-Xlinker", NCCL_LIB]
else:
    LIBS = ["-lnccl"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OUT, exist_ok=True)
    headers = [os.path.join(CSRC, "ucac_dev.cuh"), os.path.join(CSRC, "ucac_part.h"), os.path.join(INCLUDE, "ucac.h")]
    objs = []
    jobs = []
    # tuning A/B only: UCAC_SRC_OVERRIDE="k_branch.cu=/path/variant.cu" compiles another file for a unit
    override = dict(kv.split("=", 1) for kv in os.environ.get("UCAC_SRC_OVERRIDE", "").split(",") if "=" in kv)
    for src, flags in UNITS.items():
        s = override.get(src, os.path.join(CSRC, src))
        o = os.path.join(OUT, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers + [os.path.abspath(__file__)]):
            extra = os.environ.get("UCAC_EXTRA_NVCC", "").split()   # tuning sweeps only
            cmd = [nvcc(), *ARCH, *COMMON, *flags, *extra, "-Xptxas", "-v", "-c", s, "-o", o]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        return r.stderr

    with ThreadPoolExecutor(max_workers=len(UNITS)) as ex:
        logs = list(ex.map(run, jobs))
    if verbose:
        for lg in logs:
            sys.stderr.write(lg)
    if force or jobs or _stale(LIB, objs):
        tmp = LIB + f".{os.getpid()}.tmp"
        r = subprocess.run([nvcc(), *ARCH, "-shared", "-o", tmp, *objs, *LIBS], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
