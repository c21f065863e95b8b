"""Compare a loopback partition group with the single-GPU context field by field (diagnostic)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_13145_b200 import inputs, ucac  # noqa: E402


def main(name="case30", P=2, iters=1):
    pb, pr = inputs.build_config(name)
    P, iters = int(P), int(iters)
    one = ucac.Context(pb, pr)
    part = ucac.partition(pb, P)
    ctxs = [ucac.Context(pb, pr, dist={"rank": r, "nranks": P, "comm_mode": 1, "bus_part": part}) for r in range(P)]
    s0 = one.get_state()
    g0 = ucac.assemble_state(pb, ctxs)
    print("init equal:", {k: bool(np.array_equal(s0[k], g0[k])) for k in s0})
    for it in range(iters):
        one.iterate(1)
        ucac.iterate_group(ctxs, 1)
        ref, got = one.get_state(), ucac.assemble_state(pb, ctxs)
        bad = [k for k in ref if k != "scal" and not np.array_equal(ref[k], got[k])]
        print("iteration", it + 1, "mismatching fields:", bad)
        for k in bad[:4]:
            d = np.nonzero(ref[k] != got[k])[0]
            print("  ", k, "n", d.size, "first idx", d[:10], "ref", ref[k][d[:4]], "got", got[k][d[:4]])
    T = pb.T
    halos = [ucac.halo_lists(pb, part, r) for r in range(P)]
    cut = set(np.concatenate([h["cut_branch"] for h in halos]).tolist())
    exports = set(np.concatenate([h["export_bus"] for h in halos]).tolist())
    ref, got = one.get_state(), ucac.assemble_state(pb, ctxs)
    bw = np.nonzero(ref["wbar"] != got["wbar"])[0] // T
    print("mismatching wbar buses", sorted(set(bw.tolist())), "export buses", sorted(exports))
    bf = np.nonzero(ref["fbar"] != got["fbar"])[0]
    br = sorted(set((bf // 4 // T).tolist()))
    print("mismatching fbar branches", br[:20], "cut branches", sorted(cut)[:20])
    for l in br[:6]:
        print("  branch", l, "from", pb.br_from[l], "to", pb.br_to[l], "part", part[pb.br_from[l]], part[pb.br_to[l]],
              "rate", pb.br_rate[l])
    al_ref = ref["al"].reshape(-1, 3)
    act = np.nonzero(np.abs(al_ref[:, 0]) + np.abs(al_ref[:, 1]) > 0)[0] // T
    print("AL-active branches", sorted(set(act.tolist()))[:20])
    for r, c in enumerate(ctxs):
        print("rank", r, "gens", c.local_ids("gen")[:10], "buses", len(c.local_ids("bus")), "branches",
              len(c.local_ids("branch")))
    print("gen buses", pb.gen_bus, "part of gen buses", part[pb.gen_bus])


if __name__ == "__main__":
    main(*sys.argv[1:])
