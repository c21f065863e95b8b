"""Phase times of the public-API path on pegase T=48 (create / iterate 100 / report / solution /
close), three times; with UCAC_CREATE_TRACE=1 also ucac_create's phases (diagnostic).
usage: UCAC_CREATE_TRACE=1 python tools/e2e_probe.py"""
import time, torch, sys
sys.path.insert(0, ".")
from paper_2310_13145_b200 import inputs, ucac
pb, pr = inputs.build_config("pegase2869")
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    c = ucac.Context(pb, pr); torch.cuda.synchronize(); t1 = time.perf_counter()
    c.iterate(100); torch.cuda.synchronize(); t2 = time.perf_counter()
    r = c.report(); t3 = time.perf_counter()
    s = c.solution(); t4 = time.perf_counter()
    c.close(); t5 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms iterate {1e3*(t2-t1):.1f} report {1e3*(t3-t2):.1f} solution {1e3*(t4-t3):.1f} close {1e3*(t5-t4):.1f}")
