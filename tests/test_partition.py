"""Host-side logic of the multi-GPU path, no GPU needed:
the bus-graph cut (ucac_partition) and the rank-local halo (ucac_halo_lists), checked for
global consistency across ranks with torch.distributed over gloo, world_size 2 (and 3)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_13145_b200 import inputs, ucac


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partition_deterministic_and_balanced():
    for name in ("case30", "case118", "case300"):
        pb, _ = inputs.build_config(name)
        for P in (2, 3, 4, 8):
            a = ucac.partition(pb, P)
            b = ucac.partition(pb, P)
            assert np.array_equal(a, b)
            assert a.min() == 0 and a.max() == P - 1
            # weight = 1 + owned branches, balanced within a factor 2 of the mean
            w = np.ones(pb.nbus)
            np.add.at(w, pb.br_from, 1.0)
            load = np.bincount(a, weights=w, minlength=P)
            assert load.max() <= 2.0 * load.mean()
            # no coordinates: BFS chunks
            c = ucac.partition(pb, P, use_xy=False)
            assert np.array_equal(c, ucac.partition(pb, P, use_xy=False)) and c.max() == P - 1


def test_partition_rejects_bad_input():
    pb, _ = inputs.build_config("case9")
    with pytest.raises(ucac.UcacError):
        ucac.partition(pb, pb.nbus + 1)


def _halo_worker(rank, world, port, name, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pb, _ = inputs.build_config(name)
    part = ucac.partition(pb, world)
    mine = ucac.halo_lists(pb, part, rank)
    gathered = [None] * world
    dist.all_gather_object(gathered, {k: v.tolist() for k, v in mine.items()})
    ok = True
    msg = []
    try:
        own = np.concatenate([np.array(g["own_bus"], dtype=int) for g in gathered])
        assert np.array_equal(np.sort(own), np.arange(pb.nbus)), "owned buses are not a partition"
        lb = np.concatenate([np.array(g["local_branch"], dtype=int) for g in gathered])
        assert np.array_equal(np.sort(lb), np.arange(pb.nbranch)), "local branches are not a partition"
        for r, g in enumerate(gathered):
            assert all(part[pb.br_from[l]] == r for l in g["local_branch"])
            assert set(g["phantom"]) == {l for l in range(pb.nbranch)
                                         if part[pb.br_to[l]] == r and part[pb.br_from[l]] != r}
            assert set(g["ghost_bus"]) == {int(pb.br_to[l]) for l in g["local_branch"] if part[pb.br_to[l]] != r}
            assert set(g["cut_branch"]) == {l for l in g["local_branch"] if part[pb.br_to[l]] != r}
            assert set(g["export_bus"]) == {int(pb.br_to[l]) for l in g["phantom"]}
        # every cut branch is exactly one phantom at its to-bus owner, every ghost an export
        cuts = sorted(l for g in gathered for l in g["cut_branch"])
        ph = sorted(l for g in gathered for l in g["phantom"])
        assert cuts == ph
        ghosts = sorted(b for g in gathered for b in g["ghost_bus"])
        exports = {b for g in gathered for b in g["export_bus"]}
        assert set(ghosts) <= exports
    except AssertionError as e:
        ok = False
        msg.append(str(e))
    flags = [None] * world
    dist.all_gather_object(flags, ok)
    if rank == 0:
        out.put((all(flags), msg))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,name", [(2, "case118"), (3, "case300")])
def test_halo_consistent_across_gloo_ranks(world, name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert res[0], res[1]
    assert all(p.exitcode == 0 for p in procs)


def _time_split_worker(rank, world, port, T, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = ucac.time_split(T, world, rank)
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    ok, msg = True, []
    try:
        # owned global ranges tile [0, T) in rank order
        owned = [(g["t_off"] + g["own0"], g["t_off"] + g["own1"]) for g in gathered]
        assert owned[0][0] == 0 and owned[-1][1] == T
        assert all(a[1] == b[0] and a[0] < a[1] for a, b in zip(owned, owned[1:]))
        for r, g in enumerate(gathered):
            lo, hi = g["t_off"], g["t_off"] + g["Tl"]   # local periods, halos included
            # a halo below iff not the horizon's start: the previous rank's last owned period
            assert (g["own0"] == 1) == (r > 0) and (r == 0 or lo == owned[r - 1][1] - 1)
            # a halo above iff not the horizon's end: the next rank's first owned period
            assert (hi > owned[r][1]) == (r < world - 1) and (r == world - 1 or hi - 1 == owned[r + 1][0])
    except AssertionError as e:
        ok = False
        msg.append(str(e))
    flags = [None] * world
    dist.all_gather_object(flags, ok)
    if rank == 0:
        out.put((all(flags), msg))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,T", [(2, 24), (3, 48), (2, 3)])
def test_time_split_consistent_across_gloo_ranks(world, T):
    """NEXT-4(c) host logic: every rank's period split (ucac_time_split) agrees with its
    neighbours' -- the owned ranges tile the horizon and each halo period is the neighbour's
    boundary period (the values exchanged there)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_time_split_worker, args=(r, world, port, T, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert res[0], res[1]
    assert all(p.exitcode == 0 for p in procs)
    with pytest.raises(ucac.UcacError):
        ucac.time_split(3, 4, 0)


def test_fm_refinement_cut_and_weighted_balance():
    """The FM-gain boundary refinement after RCB: case300 over 8 parts cuts 37 of
    411 branches (RCB alone: 69), every part within 10 % of the mean weight; with per-branch weights
    (every 10th branch 10x, standing in for thermal-AL lines) the weighted loads balance too."""
    pb, _ = inputs.build_config("case300")
    part = ucac.partition(pb, 8)
    assert int(np.sum(part[pb.br_from] != part[pb.br_to])) <= 40
    w = np.ones(pb.nbus)
    np.add.at(w, pb.br_from, 1.0)
    load = np.bincount(part, weights=w, minlength=8)
    assert load.max() <= 1.1 * load.mean()
    bw = np.ones(pb.nbranch)
    bw[::10] = 10.0
    p2 = ucac.partition(pb, 8, branch_w=bw)
    w2 = np.ones(pb.nbus)
    np.add.at(w2, pb.br_from, bw)
    l2 = np.bincount(p2, weights=w2, minlength=8)
    assert l2.max() <= 1.1 * l2.mean()
    assert not np.array_equal(part, p2)
