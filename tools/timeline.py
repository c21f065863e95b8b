"""Graph timeline of one inner iteration (diagnostic; needs a -DUCAC_PROF build): per kernel the
first block start and the last block exit relative to the iteration start (global timer).
usage: python tools/timeline.py [config] [warm iterations]"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_13145_b200 import inputs, ucac  # noqa: E402


def main(name="pegase2869", warm=10):
    import torch
    pb, pr = inputs.build_config(name)
    c = ucac.Context(pb, pr)
    c.iterate(int(warm))
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    L = ucac.lib()
    buf = np.zeros(2 * ucac.NKERNELS, dtype=np.uint64)
    rows, ev_ms = [], []
    st = torch.cuda.ExternalStream(c.stream)
    for rep in range(5):
        flush.zero_()
        torch.cuda.synchronize()
        L.ucac_debug_timeline(c.h, None, 1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        c.iterate(1)
        b.record(st)
        c.report()
        ev_ms.append(a.elapsed_time(b))
        L.ucac_debug_timeline(c.h, buf.ctypes.data_as(C.c_void_p), 0)
        rows.append(buf.astype(np.int64).reshape(-1, 2).copy())
    r = np.median(np.stack(rows), axis=0)
    t0 = r[:, 0].min()
    order = np.argsort(r[:, 0])
    print(f"event-timed step {np.median(ev_ms) * 1e3:.1f} us; kernels span {(r[:, 1].max() - t0) / 1e3:.1f} us")
    for k in order:
        print(f"{ucac.KERNELS[k]:14s} start {(r[k, 0] - t0) / 1e3:8.1f} us  end {(r[k, 1] - t0) / 1e3:8.1f} us  "
              f"span {(r[k, 1] - r[k, 0]) / 1e3:7.1f} us")


if __name__ == "__main__":
    main(*sys.argv[1:])
