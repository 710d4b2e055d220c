"""CUDA-graph replay of the asynchronous step (timestepping.StepGraph, the
small-grid latency path): the same kernels with the same arguments in the
same order as the uncaptured steps, so the runs must agree bit for bit, with
identical iteration lists (timestepping.py:475-515)."""

import numpy as np
import pytest

import paper_2404_14864_b200 as k
from conftest import BOX, PI_BOX

pytestmark = pytest.mark.gpu


def _spec(eq, tau, t_final):
    heat, wave, schr = k.HeatPlaneDecay(), k.WaveStanding(), k.SchrodingerPhaseRotation()
    if eq == "heat":
        return BOX, k.StarCurve(1.0, c=0.2, lobes=8), dict(
            equation="heat", bc_kind="dirichlet", g=heat.dirichlet, u0=heat.u0,
            lap_u0=heat.lap_u0, tau=tau, t_final=t_final)
    if eq == "wave":
        return BOX, k.EllipseCurve(1.2, 0.8), dict(
            equation="wave", bc_kind="dirichlet", g=wave.dirichlet, u0=wave.u0,
            lap_u0=wave.lap_u0, v0=wave.v0, lap_v0=wave.lap_v0, tau=tau, t_final=t_final)
    return PI_BOX, k.StarCurve(1.5, c=0.2, lobes=3), dict(
        equation="schrodinger", bc_kind="dirichlet", g=schr.dirichlet, u0=schr.u0,
        lap_u0=schr.lap_u0, potential=schr.potential, tau=tau, t_final=t_final)


@pytest.mark.parametrize("fresh", [False, True], ids=["shared-context", "fresh-contexts"])
@pytest.mark.parametrize("eq", ["heat", "wave", "schrodinger"])
def test_graph_replay_bit_identical(eq, fresh):
    box, curve, kw = _spec(eq, 1 / 64, 12 / 64)
    geo = k.build_grid(box, 128, curve)
    spec = k.ProblemSpec(**kw)
    be = k.CudaBackend(0, timing=False)
    ctx = k.StepContext(geo, operator=True, backend=be)
    # fresh: the captured run goes first, on its own context
    ctx2 = k.StepContext(geo, operator=True, backend=be) if fresh else ctx
    b = k.run(spec, geo, context=ctx2, operator=True, graph=True, snapshot_times=(6 / 64,))
    a = k.run(spec, geo, context=ctx, operator=True, graph=False, snapshot_times=(6 / 64,))
    assert getattr(ctx2, "_step_graph", None) is not None
    assert a.iterations == b.iterations
    assert np.array_equal(a.state.u, b.state.u)
    assert np.array_equal(a.snapshots[0][1], b.snapshots[0][1])
    dens_a, dens_b = np.asarray(a.state.density), np.asarray(b.state.density)
    assert np.array_equal(dens_a, dens_b)


def test_graph_replay_reports_instability():
    heat = k.HeatPlaneDecay()
    geo = k.build_grid(BOX, 64, k.StarCurve(1.0, c=0.2, lobes=5))
    spec = k.ProblemSpec(equation="heat", bc_kind="dirichlet", g=heat.dirichlet, u0=heat.u0,
                         lap_u0=heat.lap_u0, tau=0.05, t_final=1.0, blowup_threshold=0.5)
    with pytest.raises(k.InstabilityError):
        k.run(spec, geo, operator=True, graph=True)


def test_graph_c1_config_matches_golden_iterations():
    # BASELINE configs[0] (C1, heat flower8 128^2, tau = 0.01, 100 steps):
    # the captured run reproduces the reference's iteration list
    from conftest import golden, rel_linf, run_cases

    box, m, curve, kw = run_cases()["c1_heat_flower128"]
    geo = k.build_grid(box, m, curve)
    ctx = k.StepContext(geo, backend=k.CudaBackend(0, timing=False))
    res = k.run(k.ProblemSpec(**kw), geo, context=ctx, operator=True, graph=True)
    g = golden("runs")
    assert ctx._step_graph is not None
    assert res.iterations == list(g["c1_heat_flower128__iterations"])
    assert rel_linf(res.state.u, g["c1_heat_flower128__u"]) < 1e-10


def test_graph_reuse_and_log_ring_wrap(monkeypatch):
    # a context keeps its captured step across runs; the step log is a fixed
    # ring (captured steps write to it by address): a 64-entry ring wraps
    # several times in two 100-step runs and every iteration list still
    # matches the reference's
    from conftest import golden, run_cases
    from paper_2404_14864_b200 import timestepping as ts

    monkeypatch.setattr(ts, "LOG_RING", 64)
    box, m, curve, kw = run_cases()["c1_heat_flower128"]
    geo = k.build_grid(box, m, curve)
    ctx = k.StepContext(geo, backend=k.CudaBackend(0, timing=False))
    g = list(golden("runs")["c1_heat_flower128__iterations"])
    first = k.run(k.ProblemSpec(**kw), geo, context=ctx, operator=True, graph=True)
    sg = ctx._step_graph
    second = k.run(k.ProblemSpec(**kw), geo, context=ctx, operator=True, graph=True)
    assert ctx._step_graph is sg                     # reused, not recaptured
    assert first.iterations == g and second.iterations == g
    assert np.array_equal(first.state.u, second.state.u)


@pytest.mark.parametrize("cplx", [False, True], ids=["f64", "c128"])
def test_one_cta_operator_sweeps_match_grid_kernels(monkeypatch, cplx):
    # op_solve_cta_kernel (n_ctl <= 160, no grid barrier) against the
    # cooperative grid kernels (KFBI_OP_CTA=0): same sweeps, same field to
    # rounding (the row sums are ordered differently)
    from paper_2404_14864_b200 import boxsolve

    res = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("KFBI_OP_CTA", flag)
        boxsolve._GRID_PLANS.clear()
        box, curve, kw = _spec("schrodinger" if cplx else "heat", 1 / 64, 8 / 64)
        geo = k.build_grid(box, 128, curve)
        ctx = k.StepContext(geo, backend=k.CudaBackend(0, timing=False))
        assert ctx.n_ctl <= 160
        res[flag] = k.run(k.ProblemSpec(**kw), geo, context=ctx, operator=True, graph=False)
    boxsolve._GRID_PLANS.clear()
    assert res["1"].iterations == res["0"].iterations
    a, b = np.asarray(res["1"].state.u), np.asarray(res["0"].state.u)
    assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))


def test_staged_edge_values_bit_identical(monkeypatch):
    # corr_edges_smem_kernel (JM staged per CTA) against the per-warp W-row
    # kernel: the same per-lane summation order, so the same bits
    import torch

    from paper_2404_14864_b200 import boxsolve

    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("KFBI_EDGES_SMEM", flag)
        boxsolve._GRID_PLANS.clear()
        ws = k.InterfaceWorkspace(k.build_grid(PI_BOX, 512, k.StarCurve(1.5, c=0.2, lobes=3)))
        ws.plan.set_interp("w")
        g = torch.Generator(device="cuda").manual_seed(3)
        jm = torch.randn((6, ws.cps.m), generator=g, device="cuda", dtype=torch.complex128)
        jv = torch.zeros(3 * ws.plan.n_edges, device="cuda", dtype=torch.complex128)
        ws.plan.edge_values(jm, jv)
        out[flag] = jv.cpu()
    boxsolve._GRID_PLANS.clear()
    assert torch.equal(out["1"], out["0"])


@pytest.mark.parametrize("eq", ["heat", "wave"])
def test_graph_replay_neumann(eq):
    # Neumann runs close the recurrences with the extracted trace (the step's
    # output, not host data): the captured step carries it through its state
    heat, wave = k.HeatPlaneDecay(c=1.0), k.WaveStanding(phase=0.0)
    if eq == "heat":
        box, curve, kw = BOX, k.StarCurve(1.0, c=0.2, lobes=5), dict(
            equation="heat", bc_kind="neumann", g=heat.neumann, u0=heat.u0,
            lap_u0=heat.lap_u0, tau=1 / 32, t_final=10 / 32, c=1.0)
    else:
        box, curve, kw = BOX, k.EllipseCurve(1.2, 0.8), dict(
            equation="wave", bc_kind="neumann", g=wave.neumann, u0=wave.u0,
            lap_u0=wave.lap_u0, v0=wave.v0, lap_v0=wave.lap_v0, tau=0.25, t_final=2.5)
        # (tau 1/32 does not converge within max_iter for Neumann wave on 64^2
        # in the reference's Richardson either)
    geo = k.build_grid(box, 64, curve)
    spec = k.ProblemSpec(**kw)
    be = k.CudaBackend(0, timing=False)
    ctx = k.StepContext(geo, operator=True, backend=be)
    b = k.run(spec, geo, context=ctx, operator=True, graph=True)
    assert ctx._step_graph is not None
    a = k.run(spec, geo, context=k.StepContext(geo, operator=True, backend=be), operator=True,
              graph=False)
    assert a.iterations == b.iterations
    assert np.array_equal(a.state.u, b.state.u)
