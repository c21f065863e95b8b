"""The north star's parity contract taken literally (BASELINE.json; PAPER.md:231-238 for the
iterates): per-iteration fp64 primal and dual variables within 1e-9 relative / 1e-12 absolute,
element by element, for the first 50 FREE-RUNNING iterations -- no per-kind RMS scale, no
rho-scaled floor -- in the strict_fp mode (ucac_params.strict_fp), where the
GPU runs the oracle's arithmetic (k_strict.cu, the strict sweep instantiations).  In that mode the
iterates are expected to agree bit for bit; the test reports how many fields do.

Also: the default (FMA) mode's free-running drift quantified against the oracle's own response
to rounding-level noise; the non-finite fault path (err_kernel / err_comp / err_period /
err_iter); the ADVICE r01 regressions (set_rho and the pipelined DP, the k_gen shared-memory
attribute across contexts)."""
import dataclasses
import os

import numpy as np
import pytest

import oracle
from paper_2310_13145_b200 import inputs, ucac

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-9, 1e-12
FLOAT_FIELDS = ["p", "q", "ph", "ub_on", "ub_su", "ub_sd", "pbar", "qbar", "zg", "yg", "lg", "x", "f", "fbar",
                "al", "zb", "yb", "lb", "wbar", "thbar"]


def elementwise(gs, os_, where):
    """|gpu - oracle| <= 1e-12 + 1e-9 |oracle| for every element of every field; returns the
    number of fields that are bitwise equal"""
    assert np.array_equal(gs["u"], os_["u"]), f"schedule {where}"
    same = 0
    for k in FLOAT_FIELDS:
        a, b = gs[k], os_[k]
        err = np.abs(a - b) - (ATOL + RTOL * np.abs(b))
        if err.size and np.max(err) > 0:
            i = int(np.argmax(err))
            raise AssertionError(f"{where} {k}[{i}]: gpu {a[i]!r} oracle {b[i]!r}")
        same += int(a.tobytes() == b.tobytes())
    # beta, outer k, inner total, inner since: exact; ||z||_prev is a sum (tree vs sequential order)
    assert np.array_equal(gs["scal"][[0, 2, 3, 4]], os_["scal"][[0, 2, 3, 4]]), f"scalars {where}"
    assert gs["scal"][1] == pytest.approx(os_["scal"][1], rel=1e-12, abs=1e-300)
    return same


@pytest.mark.parametrize("name", ["case9", "case30", "case118", "case300"])
def test_strict_free_run_50_iterations_elementwise(name):
    """configs[0] and the case30/118/300-shaped configs, strict mode, 50 free-running
    iterations, every iteration compared element by element at 1e-9 rel / 1e-12 abs."""
    pb, pr = inputs.build_config(name)
    pr = dataclasses.replace(pr, strict_fp=1)
    gpu = ucac.Context(pb, pr)
    orc = oracle.Oracle(pb, pr)
    bitwise = []
    bitwise.append(elementwise(gpu.get_state(), orc.get_state(), "init"))
    for it in range(50):
        gpu.iterate(1)
        orc.iterate(1)
        bitwise.append(elementwise(gpu.get_state(), orc.get_state(), f"strict iteration {it + 1}"))
    rg, ro = gpu.report(), orc.report()
    assert rg["objective"] == pytest.approx(ro["objective"], rel=1e-12)
    assert rg["inner_total"] == ro["inner_total"] == 50 and rg["outer_total"] == ro["outer_total"]
    assert rg["tron_iters"] == ro["tron_iters"] and rg["al_active"] == ro["al_active"]
    # the strict mode reproduces the oracle's arithmetic: every field bitwise, every iteration
    assert min(bitwise) == len(FLOAT_FIELDS), bitwise


def test_strict_pegase_one_iteration_bitwise():
    """the strict kernels at full size (pegase-shaped, T=48): one iteration from a GPU state,
    every field within the contract (and bitwise, as above)."""
    pb, pr = inputs.build_config("pegase2869")
    pr = dataclasses.replace(pr, strict_fp=1)
    gpu = ucac.Context(pb, pr)
    gpu.iterate(3)
    orc = oracle.Oracle(pb, pr)
    orc.set_state(gpu.get_state())
    gpu.iterate(1)
    orc.iterate(1)
    assert elementwise(gpu.get_state(), orc.get_state(), "pegase strict") == len(FLOAT_FIELDS)


def test_strict_pegase_free_run_50_iterations_bitwise():
    """The full-size case (pegase-shaped, T = 48, 220 k branch solves per iteration) free-running
    from the cold start for 50 iterations in strict mode against the all-core oracle build (bitwise
    the serial oracle's iterates, test_openmp_build_is_bitwise_the_serial_oracle): every field of
    every iteration bitwise."""
    pb, pr = inputs.build_config("pegase2869")
    pr = dataclasses.replace(pr, strict_fp=1)
    oracle.threads(os.cpu_count() or 1)
    gpu = ucac.Context(pb, pr)
    orc = oracle.Oracle(pb, pr, omp=True)
    for it in range(50):
        gpu.iterate(1)
        orc.iterate(1)
        assert elementwise(gpu.get_state(), orc.get_state(), f"pegase strict iteration {it + 1}") == len(FLOAT_FIELDS)
    assert gpu.report()["tron_iters"] == orc.report()["tron_iters"]


def test_strict_t168_free_run_bitwise():
    """The horizon of P:478's longest runs (pegase-shaped, T = 168), strict mode, 10 free-running
    iterations from the cold start: every field bitwise."""
    pb, pr = inputs.build_config("pegase2869", 168)
    pr = dataclasses.replace(pr, strict_fp=1)
    oracle.threads(os.cpu_count() or 1)
    gpu = ucac.Context(pb, pr)
    orc = oracle.Oracle(pb, pr, omp=True)
    for it in range(10):
        gpu.iterate(1)
        orc.iterate(1)
        assert elementwise(gpu.get_state(), orc.get_state(), f"T=168 strict iteration {it + 1}") == len(FLOAT_FIELDS)


@pytest.mark.parametrize("variant", [1, 2, 4, 8, 16])
def test_strict_variants_free_run_bitwise(variant):
    """Each NEXT-3/NEXT-4(a) formulation variant (R47, R50-R52) in strict mode: 30 free-running
    iterations of the case30-shaped config bitwise equal to the oracle's same variant."""
    pb, pr = inputs.build_config("case30")
    pr = dataclasses.replace(pr, strict_fp=1, variant=variant)
    gpu = ucac.Context(pb, pr)
    orc = oracle.Oracle(pb, pr)
    for it in range(30):
        gpu.iterate(1)
        orc.iterate(1)
        assert elementwise(gpu.get_state(), orc.get_state(), f"variant {variant} iteration {it + 1}") == len(FLOAT_FIELDS)


@pytest.mark.parametrize("name,iters", [("case30", 60), ("case118", 40)])
def test_strict_uc_warm_start_bitwise(name, iters):
    """NEXT-2 in strict mode: the held-schedule multiperiod ACOPF, the device Hamming costs and
    the repair DP reproduce the oracle's repaired schedule exactly -- no rounding-ambiguous
    thresholds to excuse, since the dispatch p the threshold reads is the oracle's bit for bit."""
    pb, pr = inputs.build_config(name)
    pr = dataclasses.replace(pr, strict_fp=1)
    ug = ucac.uc_warm_start(pb, pr, iters)
    uo, _ = oracle.uc_warm_start(pb, pr, iters)
    assert np.array_equal(ug, uo)


def _perturbed(st, rel, rng):
    return {k: (v * (1.0 + rel * rng.uniform(-1.0, 1.0, v.shape)) if v.dtype == np.float64 and k != "scal" else v)
            for k, v in st.items()}


def _normdiff(a, b):
    """per field max |a - b| / max(1, max |b|) over the float fields"""
    return {k: float(np.max(np.abs(a[k] - b[k])) / max(1.0, float(np.max(np.abs(b[k]))))) if b[k].size else 0.0
            for k in FLOAT_FIELDS}


@pytest.mark.parametrize("name", ["case9", "case30"])
def test_default_mode_free_run_drift_within_oracle_noise_envelope(name):
    """Default (FMA) mode, 50 free-running iterations.  The GPU's iteration map differs from the
    oracle's by delta per step (FMA, CUDA sin/cos, the LDL^T Newton steps stopping at the same
    tolerance); delta is measured one-step on this run.  The oracle is run a second time with a
    random relative perturbation of size delta injected into its state after every iteration:
    its distance from the clean oracle run is the envelope any fp64 implementation with that
    per-step rounding would show.  The GPU's distance from the clean oracle must stay within 10x
    that envelope (floor 1e-12) on every field at every iteration, and the schedule must match."""
    pb, pr = inputs.build_config(name)
    gpu = ucac.Context(pb, pr)
    ref = oracle.Oracle(pb, pr)
    noisy = oracle.Oracle(pb, pr)
    rng = np.random.default_rng(11)
    # delta: the largest one-step relative difference over the first iterations
    delta = 1e-15
    for it in range(5):
        st = gpu.get_state()
        one = oracle.Oracle(pb, pr)
        one.set_state(st)
        one.iterate(1)
        gpu.iterate(1)
        d = _normdiff(gpu.get_state(), one.get_state())
        delta = max(delta, max(d.values()))
        one.close()
    gpu.close()
    gpu = ucac.Context(pb, pr)
    worst = 0.0
    for it in range(50):
        gpu.iterate(1)
        ref.iterate(1)
        noisy.iterate(1)
        noisy.set_state(_perturbed(noisy.get_state(), delta, rng))
        gs, rs, ns = gpu.get_state(), ref.get_state(), noisy.get_state()
        assert np.array_equal(gs["u"], rs["u"]), f"schedule, iteration {it + 1}"
        dg, dn = _normdiff(gs, rs), _normdiff(ns, rs)
        for k in FLOAT_FIELDS:
            assert dg[k] <= max(10.0 * dn[k], 1e-12), (it + 1, k, dg[k], dn[k], delta)
            worst = max(worst, dg[k] / max(dn[k], 1e-300))
    print(f"{name}: delta {delta:.2e}, worst GPU/envelope ratio {worst:.3f}")


def test_nonfinite_fault_injection_reports_kernel_component_iteration():
    """a NaN planted in one branch row's z (l = 5, t = 7, row FP_IJ) is met first by
    the branch kernel at the next iteration; a NaN in one generator's D_ON z (g = 2, t = 3) by
    the DP kernel.  ucac_iterate returns UCAC_ENUMERIC and the report names kernel, component,
    period and iteration."""
    pb, pr = inputs.build_config("case30")
    T, L = pb.T, pb.nbranch
    c = ucac.Context(pb, pr)
    c.iterate(3)
    c.report()
    c.poison("zb", 0 * L * T + 5 * T + 7)
    with pytest.raises(ucac.UcacError) as e:
        c.iterate(1, stop_on_primal=0.0)
    assert e.value.code == 5
    r = c.report_raw()
    assert r["status"] == "ENUMERIC"
    assert ucac.KERNELS[r["err_kernel"] - 1] == "k_branch"
    assert (r["err_comp"], r["err_period"], r["err_iter"]) == (5, 7, 4), r
    c2 = ucac.Context(pb, pr)
    c2.iterate(2)
    c2.poison("zg", 0 * pb.ngen * T + 2 * T + 3)
    with pytest.raises(ucac.UcacError):
        c2.iterate(1, stop_on_primal=0.0)
    r = c2.report_raw()
    assert ucac.KERNELS[r["err_kernel"] - 1] == "k_gen"
    assert (r["err_comp"], r["err_period"], r["err_iter"]) == (2, 3, 3), r
    # a clean state resets the report
    c2.set_state(ucac.Context(pb, pr).get_state())
    c2.iterate(1)
    assert c2.report()["err_kernel"] == 0
    with pytest.raises(ucac.UcacError):
        c2.poison("zb", 10 ** 12)


def test_set_rho_flips_dp_decision_first_iteration():
    """after ucac_set_rho the next iteration's DP (7a) must use the new rho_uc (the
    pipelined tail DP computed with the old one is dropped).  rho_uc is changed enough to flip a
    commitment decision; u after the first iteration equals the oracle's."""
    pb, pr = inputs.build_config("case30")
    for factor in (1e-2, 1e-3, 1e2):
        gpu = ucac.Context(pb, pr)
        orc = oracle.Oracle(pb, pr)
        keep = oracle.Oracle(pb, pr)
        for o in (gpu, orc, keep):
            o.iterate(12)
        gpu.set_rho(pr.rho_pq, pr.rho_va, factor * pr.rho_uc)
        orc.set_rho(pr.rho_pq, pr.rho_va, factor * pr.rho_uc)
        for o in (gpu, orc, keep):
            o.iterate(1)
        gu, ou, ku = gpu.get_state()["u"], orc.get_state()["u"], keep.get_state()["u"]
        assert np.array_equal(gu, ou), factor
        if not np.array_equal(ou, ku):
            return   # the change flipped a decision and the GPU followed it
    pytest.fail("no rho_uc change flipped a DP decision")


def test_gen_smem_attribute_survives_smaller_T():
    """the k_gen / k_dp_batch dynamic shared-memory limit only grows, so a T=168
    context still launches (eagerly and through a re-captured graph) after a T=4 dp_batch."""
    pb, pr = inputs.build_config("case30", 168)
    c = ucac.Context(pb, pr)
    L, tu, td, u0, hold = inputs.dp_workload(8, 8, seed=1)   # T=8 < 168: a smaller smem need
    ucac.dp_batch(L, tu, td, u0, hold)
    c.iterate_timed(2)
    c.set_rho(pr.rho_pq, pr.rho_va, pr.rho_uc)
    c.iterate(2)
    assert c.report()["inner_total"] == 4


def test_measure_latencies_sane():
    """ucac_measure_latencies (DESIGN.md 11's lane-split argument): positive cycle counts, a DFMA
    link no shorter than the pipe's issue interval, a shuffle-and-add step longer than an add"""
    lat = ucac.measure_latencies()
    assert all(v > 0 for v in lat.values()), lat
    assert lat["dfma"] >= 2 and lat["shfl_add"] > lat["dadd"], lat
