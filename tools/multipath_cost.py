"""Step time of the multi-rank iteration graphs on one GPU (diagnostic): a one-rank NCCL context
(UCAC_NCCL_ONE_RANK=1, the bus cut's and the time cut's graphs with their captured collectives)
against the single-GPU graph, pegase T=48, 100 iterations each, CUDA events on the library stream.
usage: UCAC_NCCL_ONE_RANK=1 python tools/multipath_cost.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2310_13145_b200 import inputs, ucac  # noqa: E402


def timed(ctx, n=100):
    s = torch.cuda.ExternalStream(ctx.stream)
    ctx.iterate(10)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(n):
        ctx.iterate(1)
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def main():
    assert os.environ.get("UCAC_NCCL_ONE_RANK") == "1"
    pb, pr = inputs.build_config("pegase2869")
    out = {"single_gpu_graph_ms": timed(ucac.Context(pb, pr))}
    for cut in (0, 1):
        c = ucac.Context(pb, pr, dist={"rank": 0, "nranks": 1, "comm_mode": 0, "nccl_id": ucac.nccl_unique_id(), "cut": cut})
        assert c.comm_info()["nccl"]
        out[("bus" if cut == 0 else "time") + "_cut_graph_one_rank_nccl_ms"] = timed(c)
    print(out)


if __name__ == "__main__":
    main()
