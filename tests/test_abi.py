"""Host-side checks of the C ABI (no GPU): libucac.so builds for sm_100a, loads, and exports
every function include/ucac.h declares; the ctypes structs of the binding have exactly the
sizes and field offsets gcc computes from the header; the SASS contains only sm_100a code;
and without a device every entry point fails loudly (no CPU fallback)."""
import os
import re
import subprocess

import pytest

from paper_2310_13145_b200 import build as B
from paper_2310_13145_b200 import ucac

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "ucac.h")


def declared_functions():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ucac_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    path = B.build()
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (ucac_\w+)", out))
    decl = declared_functions()
    assert decl, "no declarations parsed"
    missing = [f for f in decl if f not in exported]
    assert not missing, missing
    assert set(decl) == set(ucac.EXPORTED)
    L = ucac.lib()
    for f in decl:
        getattr(L, f)


def test_struct_layouts_match_header(tmp_path):
    import ctypes as C
    structs = {"ucac_network": ucac.Network, "ucac_horizon": ucac.Horizon, "ucac_costs": ucac.Costs,
               "ucac_uc": ucac.Uc, "ucac_params": ucac.Params, "ucac_report": ucac.Report,
               "ucac_solution": ucac.Solution, "ucac_state": ucac.State, "ucac_sizes": ucac.Sizes,
               "ucac_dist": ucac.Dist}
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "ucac.h"', "int main(void){"]
    for cname, py in structs.items():
        src.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            src.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    src.append("return 0;}")
    c = tmp_path / "lay.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "lay"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n") if line)
    for cname, py in structs.items():
        assert int(got[cname]) == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)


def test_sass_is_sm100a_and_fp64():
    path = B.build()
    out = subprocess.run(["cuobjdump", "-lelf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "DFMA" in sass and "DADD" in sass          # fp64 pipe
    assert "HMMA" not in sass                         # no legacy tensor path


def test_no_cpu_fallback_without_device():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("device present")
    except Exception:
        pass
    from paper_2310_13145_b200 import inputs
    pb, pr = inputs.build_config("case9")
    with pytest.raises(ucac.UcacError) as e:
        ucac.Context(pb, pr)
    assert e.value.code == 3


def test_library_then_torch_import_order():
    """libucac.so links the NCCL that PyTorch loads (the venv's nvidia-nccl wheel, by rpath): loading
    the library before torch must not leave torch's NCCL symbols unresolved (linked to the system
    libnccl.so.2, `import torch` after `ucac.lib()` failed with an undefined ncclDevCommCreate)."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r); from paper_2310_13145_b200 import ucac; ucac.lib(); "
            "import torch; print('ok', torch.__version__)") % ROOT
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
