"""Graph timeline of one inner iteration (diagnostic; needs a -DUCAC_PROF build): per kernel the
first block start and the last block exit relative to the iteration start (global timer).
usage: python tools/timeline.py [config] [warm iterations] [T]"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_13145_b200 import inputs, ucac  # noqa: E402


def main(name="pegase2869", warm=10, T=None):
    import torch
    pb, pr = inputs.build_config(name, int(T)) if T else inputs.build_config(name)
    c = ucac.Context(pb, pr)
    c.iterate(int(warm))
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    L = ucac.lib()
    buf = np.zeros(2 * ucac.NKERNELS, dtype=np.uint64)
    rows, ev_ms, stamps = [], [], []
    st = torch.cuda.ExternalStream(c.stream)
    stamp = getattr(L, "ucac_debug_stamp", None)
    sbuf = np.zeros(8, dtype=np.uint64)
    for rep in range(5):
        flush.zero_()
        torch.cuda.synchronize()
        L.ucac_debug_timeline(c.h, None, 1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            if stamp:
                stamp(c.h, None, 0)
            c.iterate(1)
            if stamp:
                stamp(c.h, None, 1)
            b.record(st)
        c.report()
        ev_ms.append(a.elapsed_time(b))
        L.ucac_debug_timeline(c.h, buf.ctypes.data_as(C.c_void_p), 0)
        rows.append(buf.astype(np.int64).reshape(-1, 2).copy())
        if stamp:
            stamp(c.h, sbuf.ctypes.data_as(C.c_void_p), -1)
            stamps.append(sbuf[:2].astype(np.int64).copy())
    r = np.median(np.stack(rows), axis=0)
    t0 = r[:, 0].min()
    order = np.argsort(r[:, 0])
    print(f"event-timed step {np.median(ev_ms) * 1e3:.1f} us; kernels span {(r[:, 1].max() - t0) / 1e3:.1f} us")
    if stamps:
        # stamp kernels just before and after the graph launch on the same stream
        lead = np.median([rr[:, 0].min() - s[0] for rr, s in zip(rows, stamps)]) / 1e3
        tail = np.median([s[1] - rr[:, 1].max() for rr, s in zip(rows, stamps)]) / 1e3
        print(f"stamp before graph -> first kernel start {lead:.1f} us; last kernel exit -> stamp after {tail:.1f} us")
    if stamp and os.environ.get("TIMELINE_B2B"):
        # back to back: stamp, n single-iteration graphs, stamp
        for n in (1, 2, 8):
            vals = []
            for rep in range(3):
                torch.cuda.synchronize()
                stamp(c.h, None, 2)
                c.iterate(n)
                stamp(c.h, None, 3)
                c.report()
                stamp(c.h, sbuf.ctypes.data_as(C.c_void_p), -1)
                vals.append((int(sbuf[3]) - int(sbuf[2])) / 1e3)
            print(f"back to back: {n} iterations stamp to stamp {np.median(vals):.1f} us = {np.median(vals) / n:.1f} us each")
    for k in order:
        print(f"{ucac.KERNELS[k]:14s} start {(r[k, 0] - t0) / 1e3:8.1f} us  end {(r[k, 1] - t0) / 1e3:8.1f} us  "
              f"span {(r[k, 1] - r[k, 0]) / 1e3:7.1f} us")


if __name__ == "__main__":
    main(*sys.argv[1:])
