"""Where does a step's time go?  graph vs eager, with and without an L2 flush (diagnostic).
usage: python tools/step_breakdown.py [config]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2310_13145_b200 import inputs, ucac  # noqa: E402


def main(name="pegase2869", steps=20):
    pb, pr = inputs.build_config(name)
    ctx = ucac.Context(pb, pr)
    st = torch.cuda.ExternalStream(ctx.stream)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    ctx.iterate(5)
    torch.cuda.synchronize()
    out = {}
    with torch.cuda.stream(st):
        for mode in ("graph_flush", "graph_noflush", "graph_batched"):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            if mode == "graph_batched":
                a, b = ev[0]
                a.record(st)
                ctx.iterate(steps)
                b.record(st)
                torch.cuda.synchronize()
                out[mode] = a.elapsed_time(b) / steps
                continue
            for a, b in ev:
                if mode == "graph_flush":
                    flush.zero_()
                a.record(st)
                ctx.iterate(1)
                b.record(st)
            torch.cuda.synchronize()
            out[mode] = sum(a.elapsed_time(b) for a, b in ev) / steps
        for mode in ("eager_flush", "eager_noflush"):
            tot = {}
            for _ in range(steps):
                if mode == "eager_flush":
                    flush.zero_()
                ms, _ = ctx.iterate_timed(1)
                for k, v in ms.items():
                    tot[k] = tot.get(k, 0.0) + v / steps
            out[mode] = {k: round(v, 4) for k, v in tot.items()}
            out[mode]["sum"] = round(sum(tot.values()), 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main(*sys.argv[1:])
