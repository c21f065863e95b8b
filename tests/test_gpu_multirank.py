"""Multi-rank path on one GPU: a comm_mode-1 loopback group of P partition contexts runs the
same phases and halo exchanges as the NCCL graph.  Every component is computed
by exactly the kernel that computes it on one GPU, and the bus sums run in the same canonical
order, so the assembled iterate must equal the single-GPU iterate BIT FOR BIT (only the
global 2-norm sums differ in summation order; they feed the outer-update test, which flips
only at exact ties)."""
import numpy as np
import pytest

from paper_2310_13145_b200 import inputs, ucac

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,P,iters", [("case30", 2, 30), ("case118", 3, 25), ("case300", 4, 20),
                                          ("pegase2869", 8, 6)])
def test_loopback_group_bitwise_equals_single_gpu(name, P, iters):
    pb, pr = inputs.build_config(name)
    one = ucac.Context(pb, pr)
    one.iterate(iters)
    ref = one.get_state()
    part = ucac.partition(pb, P)
    ctxs = [ucac.Context(pb, pr, dist={"rank": r, "nranks": P, "comm_mode": 1, "bus_part": part}) for r in range(P)]
    ucac.iterate_group(ctxs, iters)
    got = ucac.assemble_state(pb, ctxs)
    for k in ref:
        if k == "scal":
            assert np.array_equal(got[k][[0, 2, 3, 4]], ref[k][[0, 2, 3, 4]]), (k, got[k], ref[k])
            continue
        assert np.array_equal(got[k], ref[k]), (name, P, k, np.max(np.abs(got[k].astype(float) - ref[k])))
    r1 = one.report()
    for c in ctxs:
        rp = c.report()
        assert rp["primal_inf"] == r1["primal_inf"] and rp["inner_total"] == iters
        assert rp["objective"] == pytest.approx(r1["objective"], rel=1e-12)
    # each rank holds only its part
    assert sum(len(c.local_ids("bus")) for c in ctxs) == pb.nbus
    assert sum(len(c.local_ids("branch")) for c in ctxs) == pb.nbranch


def test_group_rejects_mismatched_contexts():
    pb, pr = inputs.build_config("case30")
    part = ucac.partition(pb, 2)
    a = ucac.Context(pb, pr, dist={"rank": 0, "nranks": 2, "comm_mode": 1, "bus_part": part})
    b = ucac.Context(pb, pr, dist={"rank": 1, "nranks": 2, "comm_mode": 1, "bus_part": part})
    with pytest.raises(ucac.UcacError):
        ucac.iterate_group([b, a], 1)
    with pytest.raises(ucac.UcacError):
        a.iterate(1)   # loopback contexts iterate as a group


@pytest.mark.parametrize("name,P,iters,p2p", [("case30", 2, 30, False), ("case30", 5, 25, False),
                                              ("case118", 3, 20, False), ("case300", 4, 15, False),
                                              ("pegase2869", 8, 5, False), ("case30", 5, 25, True),
                                              ("case118", 3, 20, True), ("pegase2869", 8, 5, True)])
def test_time_cut_group_bitwise_equals_single_gpu(name, P, iters, p2p):
    """NEXT-4(c) (P:166-167 temporal decomposition): the periods split over P
    ranks (T=24 over 5 ranks is ragged), every component on every rank, the DP stage costs
    all-gathered, the ramp rows' boundary values exchanged with the neighbours.  Each (component,
    period) is computed by the same kernel code as on one GPU, so the assembled iterate equals the
    single-GPU iterate bit for bit.  p2p: the exchanges are the device-initiated ones (k_xchg.cu:
    sender stores into the receivers' buffers, epoch flags with release/acquire), the group's ranks
    emulated by one cooperative launch per exchange."""
    pb, pr = inputs.build_config(name)
    one = ucac.Context(pb, pr)
    one.iterate(iters)
    ref = one.get_state()
    ctxs = [ucac.Context(pb, pr, dist={"rank": r, "nranks": P, "comm_mode": 1, "cut": 1}) for r in range(P)]
    if p2p:
        ucac.p2p_group(ctxs)
    # each rank owns a contiguous period range; together they cover the horizon once
    owned = sorted((c.t_off + c.own0, c.t_off + c.own1) for c in ctxs)
    assert owned[0][0] == 0 and owned[-1][1] == pb.T and all(a[1] == b[0] for a, b in zip(owned, owned[1:]))
    ucac.iterate_group(ctxs, iters)
    got = ucac.assemble_state(pb, ctxs)
    for k in ref:
        if k == "scal":
            assert np.array_equal(got[k][[0, 2, 3, 4]], ref[k][[0, 2, 3, 4]]), (k, got[k], ref[k])
            continue
        assert np.array_equal(got[k], ref[k]), (name, P, k, np.max(np.abs(got[k].astype(float) - ref[k])))
    r1 = one.report()
    for c in ctxs:
        rp = c.report()
        assert rp["primal_inf"] == r1["primal_inf"] and rp["inner_total"] == iters
        assert rp["objective"] == pytest.approx(r1["objective"], rel=1e-12)
        assert len(c.local_ids("gen")) == pb.ngen and len(c.local_ids("branch")) == pb.nbranch


def test_time_cut_rejects_unsupported():
    pb, pr = inputs.build_config("case9")
    with pytest.raises(ucac.UcacError):   # T = 4 < 5 ranks
        ucac.Context(pb, pr, dist={"rank": 0, "nranks": 5, "comm_mode": 1, "cut": 1})
    import dataclasses
    with pytest.raises(ucac.UcacError):   # the ramp-aware DP needs p_{t-1} across the cut
        ucac.Context(pb, dataclasses.replace(pr, variant=4), dist={"rank": 0, "nranks": 2, "comm_mode": 1, "cut": 1})


@pytest.mark.parametrize("name,iters", [("case30", 40), ("case300", 20), ("pegase2869", 6)])
def test_time_cut_graph_one_rank_bitwise_equals_single_gpu(name, iters):
    """The time cut's iteration GRAPH (three streams, the exchanges placed where their data are
    final) run with one rank -- local exchanges, no NCCL -- gives the single-GPU
    iterate bit for bit: its stream and event dependencies order every read after its write (the
    loopback tests above check the exchanges themselves, phase by phase)."""
    pb, pr = inputs.build_config(name)
    one = ucac.Context(pb, pr)
    one.iterate(iters)
    ref = one.get_state()
    tc = ucac.Context(pb, pr, dist={"rank": 0, "nranks": 1, "comm_mode": 0, "cut": 1})
    tc.iterate(iters)
    got = tc.get_state()
    for k in ref:
        assert np.array_equal(got[k], ref[k]), (name, k)
    assert tc.report()["objective"] == one.report()["objective"]


def test_nccl_one_rank_multirank_graph_bitwise_equals_single_gpu(monkeypatch):
    """The NCCL transport on a one-GPU box ("the NCCL path has never executed"): under
    UCAC_NCCL_ONE_RANK=1 a one-rank comm_mode-0 context builds a real NCCL communicator (and the
    early exchanges' split one) and iterates through the multi-rank graph -- the S8 record leaves
    the final fold for a captured ncclAllReduce and k_finalize applies S8/S9; with the time cut,
    the captured all-gathers of the DP stage costs and the neighbour values run too.  Its iterate
    and report equal the single-GPU graph's bit for bit."""
    monkeypatch.setenv("UCAC_NCCL_ONE_RANK", "1")
    for name, cut in (("case30", 0), ("pegase2869", 0), ("case118", 1)):
        pb, pr = inputs.build_config(name)
        ref = ucac.Context(pb, pr)
        one = ucac.Context(pb, pr, dist={"rank": 0, "nranks": 1, "comm_mode": 0, "nccl_id": ucac.nccl_unique_id(),
                                         "cut": cut})
        info = one.comm_info()
        assert info == {"nranks": 1, "rank": 0, "nccl": True} and not ref.comm_info()["nccl"]
        for _ in range(3):
            ref.iterate(7)
            one.iterate(7)
        a, b = ref.get_state(), one.get_state()
        assert all(a[k].tobytes() == b[k].tobytes() for k in a), name
        ra, rb = ref.report(), one.report()
        for k in ("primal_inf", "objective", "inner_total", "outer_total", "tron_iters", "al_active"):
            assert ra[k] == rb[k], (name, k)


@pytest.mark.parametrize("cut,P", [(0, 3), (1, 4)])
def test_strict_multirank_groups_bitwise_equal_the_oracle(cut, P):
    """The multi-rank paths in strict mode against the CPU oracle itself (not only against one
    GPU): the bus cut (halo exchanges, early/late flags) and the time cut (stage-cost all-gather,
    neighbour ramp values) on the case118-shaped config, 25 free-running iterations, the assembled
    iterate bitwise equal to the oracle's."""
    import dataclasses
    import oracle
    pb, pr = inputs.build_config("case118")
    pr = dataclasses.replace(pr, strict_fp=1)
    if cut == 0:
        part = ucac.partition(pb, P)
        ctxs = [ucac.Context(pb, pr, dist={"rank": r, "nranks": P, "comm_mode": 1, "bus_part": part}) for r in range(P)]
    else:
        ctxs = [ucac.Context(pb, pr, dist={"rank": r, "nranks": P, "comm_mode": 1, "cut": 1}) for r in range(P)]
    orc = oracle.Oracle(pb, pr)
    for it in range(25):
        ucac.iterate_group(ctxs, 1)
        orc.iterate(1)
        got, ref = ucac.assemble_state(pb, ctxs), orc.get_state()
        for k in ref:
            if k == "scal":
                assert np.array_equal(got[k][[0, 2, 3, 4]], ref[k][[0, 2, 3, 4]]), (it, k)
                continue
            assert got[k].tobytes() == ref[k].tobytes(), (cut, P, it + 1, k)
