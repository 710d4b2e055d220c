"""Benchmark: KFBI time steps/s at 4096² for heat, wave and Schrödinger.

One bench step = one time step of EACH of the three equations (BASELINE.json
metric: "KFBI time steps/sec at 4096² (heat/wave/Schrödinger)"):

  heat         Crank-Nicolson, flower star(1, 0.2, k=8) on [-1.5,1.5]²
  wave         implicit θ = 1/4, ellipse (1.2, 0.8) on [-1.5,1.5]²
  schrodinger  Strang splitting (complex128), star(1.5, 0.2, 3) on [-π,π]²

all Dirichlet, M = 4096, τ = 0.25·64/M (the convergence-sweep rule of
SURVEY §6.3 / BASELINE §2), closed-form manufactured solutions (synthetic
data, no RNG).  Setup, startup and the cold first steps (warm-up) are
untimed; K bench steps are timed with CUDA events, bracketed by a barrier +
synchronize, max over ranks.  Per-equation working sets (W rows, panels,
fields) exceed the 126 MB L2, so no flush is needed between steps.

  value  time steps/s, device-resident (the public per-step API, boundary
         data evaluated and uploaded by it every step); the three equations
         are independent problems, each stepped on its own CUDA stream
         (`sequential` in the line: the same steps on one stream)
  e2e    same loop plus a device->host copy of every step's solution field
         into pinned memory (what a user saving each step pays): its interior
         values (the masked exterior is zero by construction), packed by a
         device gather and copied on a side stream (StepContext.field_to_host)
         so the copy engine overlaps the following steps; the timed region
         ends when every copy is done

Also in the ours-line: `pipeline` (the same K steps with every Richardson
sweep through the full pipeline, no trace operator), `operator_build_s`,
`t1_time_to_solution_s` (a T = 1 run per equation, operator form incl. its
build vs pipeline form), `repeats` (value = median of 5 timed regions of K
steps each), the `roofline` of the dominant box-solve pass, and `slab_c5`
(BASELINE configs[4]: one 16384² solve, star3 on [-π,π]², slab-decomposed
over the N ranks, NCCL all-to-all and fused peer-store transposes).

`--impl reference` times the CPU reference path (the oracle port of the
reference package, numpy/scipy with all host threads) on the same workload
with real, untruncated time steps (one cold warm-up step per equation, then
whole bench steps until --steps or --ref-budget-s); rank 0 only.

Launch: python bench.py [--gpus N --steps K --warmup W]; for N > 1 under
torchrun every rank runs an independent replica of the 4096² workload (weak
scaling) and all ranks share the C5 slab solve (strong scaling).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

M_DEFAULT = 4096
EQUATIONS = ("heat", "wave", "schrodinger")
METRIC = "KFBI time steps/sec at 4096² (heat/wave/Schrödinger); speedup vs host CPU"


def workload(m):
    import paper_2404_14864_b200 as k

    box = (-1.5, 1.5, -1.5, 1.5)
    pibox = (-np.pi, np.pi, -np.pi, np.pi)
    tau = 0.25 * 64 / m
    heat, wave, schr = k.HeatPlaneDecay(1.0), k.WaveStanding(0.0), k.SchrodingerPhaseRotation()
    horizon = 10_000 * tau
    return {
        "heat": (box, k.StarCurve(1.0, c=0.2, lobes=8), dict(
            equation="heat", bc_kind="dirichlet", g=heat.dirichlet, u0=heat.u0,
            lap_u0=heat.lap_u0, tau=tau, t_final=horizon, c=1.0)),
        "wave": (box, k.EllipseCurve(1.2, 0.8), dict(
            equation="wave", bc_kind="dirichlet", g=wave.dirichlet, u0=wave.u0,
            lap_u0=wave.lap_u0, v0=wave.v0, lap_v0=wave.lap_v0, tau=tau, t_final=horizon,
            theta=0.25)),
        "schrodinger": (pibox, k.StarCurve(1.5, c=0.2, lobes=3), dict(
            equation="schrodinger", bc_kind="dirichlet", g=schr.dirichlet, u0=schr.u0,
            lap_u0=schr.lap_u0, potential=schr.potential, w=1.0, tau=tau, t_final=horizon)),
    }


def config_obj(m, eqs, n, mode=None):
    return {
        "workload": f"KFBI per-step solve, {m}x{m} grid, one time step each of "
                    + "/".join(eqs) + " (heat flower8, wave ellipse, Schrodinger star3)",
        "grid": m, "tau": 0.25 * 64 / m, "equations": list(eqs),
        "boundary": "dirichlet", "l2": "per-equation working set > 126 MB L2 (no flush)",
        "parallelism": f"replicas{n}",
    }


# ---------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md)."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        # the timed region starts only once the sampler is producing samples
        t0 = time.time()
        while self.proc is not None and time.time() - t0 < 5.0:
            try:
                if os.path.getsize(self.path) > 0:
                    break
            except OSError:
                pass
            time.sleep(0.01)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm.append(float(f[1]))
                    mx = float(f[2])
                except ValueError:
                    continue
                for nm, v in zip(names, f[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        except OSError:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
def _dist():
    import torch.distributed as dist

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1 and not dist.is_initialized():
        import torch

        from datetime import timedelta

        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        # a stuck collective fails the run after 5 minutes instead of hanging it
        dist.init_process_group(backend=backend, timeout=timedelta(seconds=300))
    return ws, rank, local


def _max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def _bytes_cols(m, cplx):
    # algorithmic bytes of one fused column pass: read + write the interior spectrum
    return 2 * (m - 1) ** 2 * (16 if cplx else 8)


def run_ours(args):
    import torch

    import paper_2404_14864_b200 as k
    from paper_2404_14864_b200.timestepping import _stepper_for

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    m = args.m
    eqs = args.equations
    wl = workload(m)
    backend = k.CudaBackend(local, timing=False)
    ctxs, specs, states, steppers = {}, {}, {}, {}
    kappas, op_build_s, startups = {}, {}, {}
    setup_parts = {}
    t_setup = time.time()

    # the trace operators of the three independent problems are built
    # concurrently (one host thread and one CUDA stream each; the build of a
    # column is a chain of short kernels, so three chains overlap), each
    # started as soon as its context exists so that the host-side startups
    # (initial fields evaluated with numpy, uploaded) overlap the device
    # builds; one at a time after the startups with --sequential
    def build(eq):
        s_b = torch.cuda.Stream() if not args.sequential else torch.cuda.current_stream()
        with torch.cuda.stream(s_b):
            t_op = time.perf_counter()
            ctxs[eq].workspace.ensure_operator(kappas[eq], eq == "schrodinger")
            s_b.synchronize()
            op_build_s[eq] = time.perf_counter() - t_op

    import threading
    ths = []
    concurrent = not args.pipeline and not args.sequential
    t_all = time.perf_counter()
    for eq in eqs:
        box, curve, kw = wl[eq]
        part = {}
        t_p = time.perf_counter()
        geo = k.build_grid(box, m, curve)
        part["build_grid"] = time.perf_counter() - t_p
        t_p = time.perf_counter()
        ctxs[eq] = k.StepContext(geo, backend=backend, operator=not args.pipeline)
        specs[eq] = k.ProblemSpec(**kw)
        startup, step = _stepper_for(specs[eq])
        steppers[eq] = step
        startups[eq] = startup
        part["context"] = time.perf_counter() - t_p
        kap = {"heat": 2.0 * specs[eq].c / specs[eq].tau,
               "wave": 1.0 / (specs[eq].theta * specs[eq].tau ** 2),
               "schrodinger": 2j / specs[eq].tau}[eq]
        kappas[eq] = kap
        if concurrent:
            torch.cuda.current_stream().synchronize()    # the context's uploads
            if not ths:
                t_all = time.perf_counter()              # first build starts
            ths.append(threading.Thread(target=build, args=(eq,)))
            ths[-1].start()
        t_p = time.perf_counter()
        states[eq] = startup(specs[eq], ctxs[eq])
        torch.cuda.current_stream().synchronize()
        part["startup"] = time.perf_counter() - t_p
        setup_parts[eq] = part
    if not args.pipeline:
        torch.cuda.synchronize()
        if args.sequential:
            for eq in eqs:
                build(eq)
        else:
            for th in ths:
                th.join()
            op_build_s["all_concurrent"] = time.perf_counter() - t_all
    torch.cuda.synchronize()
    t_setup = time.time() - t_setup

    # the three equations are independent problems: each steps on its own
    # CUDA stream (their latency-bound phases overlap the others' kernels);
    # --sequential puts them on one stream
    main_stream = torch.cuda.current_stream()
    eq_stream = {eq: (main_stream if args.sequential else torch.cuda.Stream()) for eq in eqs}

    def advance(eq):
        with torch.cuda.stream(eq_stream[eq]):
            st = steppers[eq](states[eq], specs[eq], ctxs[eq])
            ctxs[eq].check_stable(st, specs[eq])
        states[eq] = st
        return st

    def fork():
        for eq in eqs:
            eq_stream[eq].wait_stream(main_stream)

    def join():
        for eq in eqs:
            main_stream.wait_stream(eq_stream[eq])

    def fresh():
        # every timed region starts from t = 0: startup + W untimed warm-up
        # steps (the cold first step included), so the timed window is
        # steps W+1..W+K of each equation, the same early regime the
        # reference arm times (the wave iteration counts grow later in the
        # run)
        torch.cuda.synchronize()
        for c in ctxs.values():
            c.flush()
        for eq in eqs:
            with torch.cuda.stream(eq_stream[eq]):
                states[eq] = startups[eq](specs[eq], ctxs[eq])
        for _ in range(args.warmup):
            for eq in eqs:
                advance(eq)
        torch.cuda.synchronize()
        for c in ctxs.values():
            c.flush()

    def seq_advance(eq):
        st = steppers[eq](states[eq], specs[eq], ctxs[eq])
        ctxs[eq].check_stable(st, specs[eq])
        states[eq] = st
        return st

    def fresh_seq():
        # as fresh(), everything on the launching stream
        torch.cuda.synchronize()
        for c in ctxs.values():
            c.flush()
        for eq in eqs:
            states[eq] = startups[eq](specs[eq], ctxs[eq])
        for _ in range(args.warmup):
            for eq in eqs:
                seq_advance(eq)
        torch.cuda.synchronize()
        for c in ctxs.values():
            c.flush()

    fresh()

    plans = [c.plan for c in ctxs.values()]
    for p in plans:
        p.set_timing(False)
    launches0 = sum(p.launch_count() for p in plans)
    stream = torch.cuda.current_stream()
    ev = {eq: [] for eq in eqs}
    iters = {eq: [] for eq in eqs}
    reps_ms = []
    with Clocks(local) as clk:
        for rep in range(args.repeats):
            if rep:
                fresh()
            _barrier(ws)
            torch.cuda.synchronize()
            start = torch.cuda.Event(enable_timing=True)
            end = torch.cuda.Event(enable_timing=True)
            if args.profile and rep == 0:
                torch.cuda.profiler.start()
            start.record(stream)
            fork()
            for _ in range(args.steps):
                for eq in eqs:
                    st = advance(eq)
                    if st.log_slot is None:
                        iters[eq].append(st.last_iterations)
            join()
            end.record(stream)
            torch.cuda.synchronize()
            if args.profile and rep == 0:
                torch.cuda.profiler.stop()
            _barrier(ws)
            reps_ms.append(_max_over_ranks(start.elapsed_time(end), ws))
            for eq in eqs:             # asynchronous stepping: per-step log (+ error checks)
                if ctxs[eq].asynchronous:
                    iters[eq].extend(ctxs[eq].flush())
    elapsed_ms = float(np.median(reps_ms))
    launches = (sum(p.launch_count() for p in plans) - launches0) // args.repeats

    # per-equation rates and the one-stream rate: the same K steps with the
    # equations one after another on one stream, each bracketed by events
    fresh_seq()
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(args.steps):
        for eq in eqs:
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            seq_advance(eq)
            b.record(stream)
            ev[eq].append((a, b))
    s1.record(stream)
    torch.cuda.synchronize()
    seq_iters = {eq: ctxs[eq].flush() for eq in eqs}
    seq_ms = _max_over_ranks(s0.elapsed_time(s1), ws)
    per_eq_ms = {eq: sum(a.elapsed_time(b) for a, b in ev[eq]) / args.steps for eq in eqs}

    # kernel-duration pass: the same K steps again, one stream, with every
    # launch of our kernels bracketed by CUDA events on the launching stream
    # (kept out of the headline pass, whose host side it would slow down)
    fresh_seq()
    for p in plans:
        p.reset_kernel_times()
        p.set_timing(True)
    for _ in range(args.steps):
        for eq in eqs:
            seq_advance(eq)
    torch.cuda.synchronize()
    for c in ctxs.values():
        c.flush()
    # per-kernel device times over the timed region
    kt_ms, kt_calls = {}, {}
    # box-solve passes, algorithmic bytes per launch in units of (M-1)^2 s
    # (SURVEY §8(d)): three-pass solve 2 per row pass and 2 for the column
    # stage; FACR(1) rows_fwd 1.5 / rows_inv 1 (average 1.25 over
    # the alternating launches), column stage 1 (M/2 rows), odd rows 1.5
    pas = {n: {"bytes": 0.0, "ms": 0.0, "calls": 0}
           for n in ("transform-rows", "transform-cols", "diagonal-scale")}
    work_fr = {}
    for eq, c in ctxs.items():
        ms, calls = c.plan.kernel_times()
        cplx = eq == "schrodinger"
        unit = _bytes_cols(m, cplx) / 2.0
        facr = c.plan.facr_for(kappas[eq])
        # FACR per step: the trace-only first sweep (inverse of the even rows
        # its stencils read, odd-row chunks of the stencils) and the masked
        # final sweep (even rows of the domain's band, odd-row chunk ranges of
        # the interior): the plan's work fractions scale those launches' bytes
        fr = c.plan.work_fractions() if facr else (1.0, 1.0, 1.0, 1.0)
        per = ({"transform-rows": (1.5 + fr[0] + 1.5 + fr[1]) / 4.0, "transform-cols": 1.0,
                "diagonal-scale": 1.5 * (fr[2] + fr[3]) / 2.0} if facr
               else {"transform-rows": 2.0, "transform-cols": 2.0, "diagonal-scale": 0.0})
        work_fr[eq] = fr
        for n in pas:
            pas[n]["bytes"] += calls[n] * per[n] * unit
            pas[n]["ms"] += ms[n]
            pas[n]["calls"] += calls[n]
        for name in ms:
            kt_ms[name] = kt_ms.get(name, 0.0) + ms[name]
            kt_calls[name] = kt_calls.get(name, 0) + calls[name]
    for p in plans:
        p.set_timing(False)
    clocks = clk.summary()

    # matrix-free edge values (fp64-bound): spec_block (DFT of
    # the five used jump columns) + edges_spectral_res (one frequency sum per
    # crossing) on the heat geometry, event-timed; flops counted per (control,
    # frequency) and per (crossing, frequency)
    mf = None
    hp = ctxs.get("heat")
    if hp is not None and hp.plan.spectral_edges:
        n = hp.plan.n_ctl
        jm = torch.randn((6, n), dtype=torch.float64, device=f"cuda:{local}")
        jv = torch.empty(3 * hp.plan.n_edges, dtype=torch.float64, device=f"cuda:{local}")
        hp.plan.edge_values(jm, jv)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(20):
            hp.plan.edge_values(jm, jv)
        e1.record(stream)
        torch.cuda.synchronize()
        t_ms = e0.elapsed_time(e1) / 20
        K = n // 2 + 1
        flops = 26.0 * n * K + 18.0 * hp.plan.n_edges * (n // 2 - 1)
        mf = {"kernels": "spec_block_kernel + edges_spectral_res_kernel (heat, flower8)",
              "n_ctl": n, "n_edges": hp.plan.n_edges, "flops_per_call": flops, "ms_per_call": t_ms,
              "achieved_tflops": flops / (t_ms / 1e3) / 1e12, "peak_tflops": FP64_PEAK_TFLOPS,
              "peak_source": "measured fp64 FMA peak (tools/mb/dfma.cu, DESIGN.md §4)",
              "frac": flops / (t_ms / 1e3) / 1e12 / FP64_PEAK_TFLOPS, "bound": "fp64"}

    elapsed_max = elapsed_ms
    n_time_steps = args.steps * len(eqs)
    value = n_time_steps * ws / (elapsed_max / 1e3)

    # ---- e2e: same loop + D2H of each step's solution field (pinned) ----
    # the step's result = the solution field, copied as its interior values
    # (the exterior is zero by construction; StepContext.unpack_interior
    # restores the full array on the host)
    pinned = {eq: torch.empty(ctxs[eq].interior_index.numel(),
                              dtype=torch.complex128 if eq == "schrodinger" else torch.float64,
                              pin_memory=True) for eq in eqs}
    h2d = sum(ctxs[eq].n_ctl * (16 if eq == "schrodinger" else 8) for eq in eqs)
    d2h = sum(pinned[eq].numel() * pinned[eq].element_size() for eq in eqs)
    # link probe (untimed): device -> pinned host bandwidth of this box
    probe = torch.empty(max(p.numel() for p in pinned.values()) * 2 // 2, dtype=torch.float64,
                        device=f"cuda:{local}")
    host = torch.empty(probe.numel(), dtype=torch.float64, pin_memory=True)
    host.copy_(probe)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        host.copy_(probe)
    torch.cuda.synchronize()
    d2h_gbps = 3 * probe.numel() * 8 / (time.perf_counter() - t0) / 1e9
    del probe, host
    # warm-up of the e2e path (untimed): first DMA into fresh pinned pages and
    # the staging buffers' first use cost ~2x a steady step
    fresh()
    for _ in range(args.warmup):
        for eq in eqs:
            st = advance(eq)
            ctxs[eq].field_to_host(st.u, pinned[eq], packed=True)
    for c in ctxs.values():
        c.host_sync()
    torch.cuda.synchronize()
    # three timed regions (each from t = 0, exactly K steps); e2e = the median
    e2e_runs = []
    for _ in range(3):
        fresh()
        _barrier(ws)
        torch.cuda.synchronize()
        s2 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        s2.record(stream)
        fork()
        for _ in range(args.steps):
            for eq in eqs:
                st = advance(eq)
                # D2H on the context's copy stream, overlapping the next steps
                with torch.cuda.stream(eq_stream[eq]):
                    ctxs[eq].field_to_host(st.u, pinned[eq], packed=True)
        for eq, c in ctxs.items():
            with torch.cuda.stream(eq_stream[eq]):
                c.host_sync()
        join()
        e2.record(stream)
        torch.cuda.synchronize()
        for c in ctxs.values():
            c.flush()
        _barrier(ws)
        e2e_runs.append(_max_over_ranks(s2.elapsed_time(e2), ws))
    e2e_ms = statistics.median(e2e_runs)
    e2e_value = n_time_steps * ws / (e2e_ms / 1e3)

    # ---- pipeline form: every Richardson sweep through the full pipeline ----
    # (jumps -> edge values -> box solve -> extraction; the algorithm of
    # bvp.py:312-351 without the trace operator), same K steps
    pipe = None
    if not args.pipeline and not args.no_pipeline_pass:
        for c in ctxs.values():
            c.flush()
            c.operator = False
        fresh_seq()
        torch.cuda.synchronize()
        pipe_it = {eq: [] for eq in eqs}
        pev = {eq: [] for eq in eqs}
        _barrier(ws)
        torch.cuda.synchronize()
        s3 = torch.cuda.Event(enable_timing=True)
        e3 = torch.cuda.Event(enable_timing=True)
        s3.record(stream)
        for _ in range(args.steps):
            for eq in eqs:
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                st = seq_advance(eq)
                b.record(stream)
                pev[eq].append((a, b))
                pipe_it[eq].append(st.last_iterations)
        e3.record(stream)
        torch.cuda.synchronize()
        _barrier(ws)
        pipe_ms = _max_over_ranks(s3.elapsed_time(e3), ws)
        pipe_eq_ms = {eq: sum(a.elapsed_time(b) for a, b in pev[eq]) / args.steps for eq in eqs}
        sweeps = sum(sum(v) for v in pipe_it.values())
        pipe = {"value": n_time_steps * ws / (pipe_ms / 1e3), "unit": "time steps/s",
                "ms_per_step": pipe_ms / args.steps,
                "sweeps_per_s": sweeps * ws / (pipe_ms / 1e3),
                "per_equation": {eq: {"steps_per_s": 1e3 / pipe_eq_ms[eq],
                                      "ms_per_step": pipe_eq_ms[eq],
                                      "ms_per_sweep": pipe_eq_ms[eq] / max(np.mean(pipe_it[eq]), 1),
                                      "iterations": pipe_it[eq]} for eq in eqs}}
        for c in ctxs.values():
            c.operator = True

    # ---- BASELINE configs[0..2] (C1-C3) through run(), rank-local
    configs = None
    if not args.no_configs:
        configs = run_configs(args, local, with_cpu=(rank == 0 and ws == 1 and not args.no_cpu_baseline))

    # ---- C5 (BASELINE configs[4]): one 16384^2 solve, slab-decomposed over the N ranks
    slab = None
    if not args.no_slab:
        slab = {}
        for mode in ("carry", "a2a", "p2p"):
            name = {"a2a": "nccl", "p2p": "p2p", "carry": "carry"}[mode]
            try:
                slab[name] = slab_c5(args, ws, rank, local, mode)
            except Exception as e:          # reported, never fatal for the headline
                slab[name] = {"error": f"{type(e).__name__}: {e}"}
            torch.cuda.empty_cache()
        if ws == 1:
            try:
                slab["one_gpu"] = c5_one_gpu(args, local)
            except Exception as e:
                slab["one_gpu"] = {"error": f"{type(e).__name__}: {e}"}
            torch.cuda.empty_cache()

    if rank != 0:
        return None
    peaks = _peaks()
    traffic = _ncu_traffic() or {}
    roof = {}
    pas = {n: v for n, v in pas.items() if v["calls"]}
    for n, v in pas.items():
        avg = v["ms"] / max(v["calls"], 1)
        ach = (v["bytes"] / max(v["calls"], 1)) / (avg / 1e3) / 1e9 if v["calls"] else 0.0
        roof[n] = {"achieved": ach, "frac": ach / peaks["hbm_gbs"], "avg_launch_ms": avg,
                   "launches": v["calls"], "ms_per_bench_step": v["ms"] / args.steps}
    dom = max(pas, key=lambda n: pas[n]["ms"])     # the dominant kernel of the step
    kernel_name = {"transform-rows": "rows_fwd_facr / rows_inv_reg (DST-I along x of the even rows, "
                                     "transform-rows)",
                   "transform-cols": "cols_tri (tridiagonal column solves, transform-cols)",
                   "diagonal-scale": "rows_odd_facr (odd rows by x recurrences)"}
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "time steps/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": elapsed_max / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64 (heat, wave) / c128 (schrodinger)",
        "data": "synthetic: closed-form manufactured solutions (no RNG), random-free geometry",
        "config": config_obj(m, eqs, ws),
        "schedule": ("one CUDA stream per equation (the three problems are independent; "
                     "their latency-bound phases overlap)" if not args.sequential else
                     "one stream (equations one after another)"),
        "sequential": {"value": n_time_steps * ws / (seq_ms / 1e3), "ms_per_step": seq_ms / args.steps,
                       "note": "the same K steps on one stream, equations one after another"},
        "per_equation": {eq: {"steps_per_s": 1e3 / per_eq_ms[eq], "ms_per_step": per_eq_ms[eq],
                              "iterations": iters[eq],
                              "iterations_one_stream_equal": seq_iters[eq] == iters[eq][:len(seq_iters[eq])]}
                         for eq in eqs},
        "kernel_ms_per_bench_step": {kname: v / args.steps for kname, v in kt_ms.items() if v},
        "kernel_calls": {kname: v for kname, v in kt_calls.items() if v},
        "roofline": {
            "matrix_free_edges": mf,
            "kernel": kernel_name[dom],
            "bound": "hbm", "achieved": roof[dom]["achieved"], "peak": peaks["hbm_gbs"],
            "unit": "GB/s", "frac": roof[dom]["frac"],
            "traffic": traffic.get(dom),
            "peak_source": peaks["source"],
            "algorithmic_bytes_per_launch": "transform-rows under FACR(1): 1.5 (forward) / 1.0 x f "
                                            "(inverse, f = the fraction of even rows the trace-only "
                                            "first sweep / the masked final sweep transform) x "
                                            "(M-1)^2 s, averaged over the alternating launches; "
                                            "three-pass: 2 (M-1)^2 s",
            "work_fractions": work_fr,
            "avg_launch_ms": roof[dom]["avg_launch_ms"],
            "per_pass": roof,
        },
        "e2e": {"value": e2e_value, "unit": "time steps/s", "d2h_link_GBps": d2h_gbps,
                "ms_per_step_runs": e2e_runs and [r / args.steps for r in e2e_runs],
                "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "setup_s": t_setup,
        "setup_parts_s": setup_parts,
        "sweep_mode": "pipeline" if args.pipeline else
        "operator (sweep 1 + returned field by the full pipeline, sweeps >= 2 via the trace operator)",
        "repeats": {"n": args.repeats, "ms_per_step": [r / args.steps for r in reps_ms],
                    "value_is": "median of the repeats (each exactly K steps)"},
    }
    if op_build_s:
        line["operator_build_s"] = op_build_s
    if pipe is not None:
        line["pipeline"] = pipe
        # time to solution of a T = 1 run (1/tau steps, the C4 rule) per equation:
        # operator form incl. its one-off build vs. the pipeline form
        n_t1 = int(round(1.0 / specs[eqs[0]].tau))
        line["t1_time_to_solution_s"] = {
            eq: {"steps": n_t1,
                 "operator_incl_build": op_build_s.get(eq, 0.0) + n_t1 * per_eq_ms[eq] / 1e3,
                 "pipeline": n_t1 * pipe["per_equation"][eq]["ms_per_step"] / 1e3}
            for eq in eqs}
    if configs is not None:
        line["configs"] = configs
    if slab is not None:
        line["slab_c5"] = slab
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(ctxs, specs, iters, args)
    return line


def config_cases():
    """BASELINE.json configs[0..2] as run() specs."""
    import paper_2404_14864_b200 as k

    box = (-1.5, 1.5, -1.5, 1.5)
    pibox = (-np.pi, np.pi, -np.pi, np.pi)
    heat, wave, schr = k.HeatPlaneDecay(1.0), k.WaveStanding(0.0), k.SchrodingerPhaseRotation()
    return {
        "C1": ("heat CN, flower star(1, 0.2, 8), 128^2, tau 0.01, T 1 (100 steps)",
               box, 128, k.StarCurve(1.0, c=0.2, lobes=8),
               dict(equation="heat", bc_kind="dirichlet", g=heat.dirichlet, u0=heat.u0,
                    lap_u0=heat.lap_u0, tau=0.01, t_final=1.0, c=1.0)),
        "C2": ("wave theta 1/4, ellipse (1.2, 0.8), 1024^2, tau 1/64, T 1 (64 steps)",
               box, 1024, k.EllipseCurve(1.2, 0.8),
               dict(equation="wave", bc_kind="dirichlet", g=wave.dirichlet, u0=wave.u0,
                    lap_u0=wave.lap_u0, v0=wave.v0, lap_v0=wave.lap_v0, tau=1 / 64, t_final=1.0,
                    theta=0.25)),
        "C3": ("Schrodinger Strang (c128), star(1.5, 0.2, 3) on [-pi, pi]^2, 2048^2, tau 1/128, "
               "T 1 (128 steps)", pibox, 2048, k.StarCurve(1.5, c=0.2, lobes=3),
               dict(equation="schrodinger", bc_kind="dirichlet", g=schr.dirichlet, u0=schr.u0,
                    lap_u0=schr.lap_u0, potential=schr.potential, w=1.0, tau=1 / 128, t_final=1.0)),
    }


def run_configs(args, local, with_cpu):
    """Each config end to end through the public run() API (numpy in, numpy
    out: setup, operator build when run(operator="auto") picks it, every
    step, the final field copied to the host), wall-clocked after a warm-up
    run; C1 also on the host CPU with the oracle port (the reference's own
    size)."""
    import torch

    import paper_2404_14864_b200 as k

    out = {}
    backend = k.CudaBackend(local, timing=False)
    for name, (desc, box, m, curve, kw) in config_cases().items():
        geo = k.build_grid(box, m, curve)
        spec = k.ProblemSpec(**kw)
        k.run(spec, geo, backend=backend)              # warm-up (first-use allocations)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = k.run(spec, geo, backend=backend)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ctx = k.StepContext(geo, backend=backend)
        n = spec.n_steps()
        from paper_2404_14864_b200.timestepping import operator_pays
        row = {"workload": desc, "steps": n, "run_wall_s": wall, "steps_per_s_run": n / wall,
               "iterations_total": int(sum(res.iterations)),
               "operator_form": bool(operator_pays(ctx, n)), "n_ctl": int(ctx.n_ctl)}
        # steady stepping rate: the same run() with the context (setup) reused
        k.run(spec, geo, context=ctx)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res2 = k.run(spec, geo, context=ctx)
        torch.cuda.synchronize()
        row["steps_per_s_steady"] = n / (time.perf_counter() - t0)
        row["iterations_match"] = res2.iterations == res.iterations
        if with_cpu and name == "C1":
            from oracle import kfbi_oracle as O
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            from conftest import oracle_spec

            O.WORKERS = _cpu_threads()
            tabs = O.tables_from_workspace(ctx.workspace)
            t0 = time.perf_counter()
            st = O.run(tabs, oracle_spec(kw))
            cpu = time.perf_counter() - t0
            row["cpu_oracle"] = {"wall_s": cpu, "steps_per_s": n / cpu, "cores": _cpu_threads(),
                                 "iterations_match": list(st.iterations) == list(res.iterations),
                                 "max_rel_diff": float(np.max(np.abs(res.state.u - st.u))
                                                       / np.max(np.abs(st.u)))}
        out[name] = row
        del ctx
        torch.cuda.empty_cache()
    return out


def c5_problem(m, rank, ws, local, mode, torch):
    """StaticPlaneWave on star(1.5, 0.2, 3) over [-pi, pi]^2,
    kappa = 2 / tau with tau = 0.25 * 64 / m (kappa = 2048 at m = 16384)."""
    import paper_2404_14864_b200 as k
    from paper_2404_14864_b200 import dist as D

    tau = 0.25 * 64 / m
    kappa = 2.0 / tau
    geo = k.build_grid((-np.pi, np.pi, -np.pi, np.pi), m, k.StarCurve(1.5, c=0.2, lobes=3))
    wsp = k.InterfaceWorkspace(geo, backend=k.CudaBackend(local, timing=False))
    sol = k.StaticPlaneWave(kappa=kappa)
    cps = wsp.cps
    solver = D.SlabRichardson(wsp, nranks=ws, rank=rank, mode=mode)
    r0, r1 = solver.rows
    X, Y = geo.grid.X[r0:r1], geo.grid.Y[r0:r1]
    F = torch.from_numpy(np.where(geo.classification.interior[r0:r1], sol.f(X, Y), 0.0)).cuda()
    fg = torch.from_numpy(np.asarray(sol.f(cps.x, cps.y))).cuda()
    g = torch.from_numpy(np.asarray(sol.dirichlet(cps.x, cps.y))).cuda()
    wsp.plan                                   # geometry upload
    return geo, wsp, sol, solver, F, fg, g, kappa


def c5_one_gpu(args, local):
    """C5 on one GPU through the plan's own device Richardson solve
    (bvp.solve_device: FACR(1) box solve, no slab layout)."""
    import torch

    import paper_2404_14864_b200 as k
    from paper_2404_14864_b200.bvp import solve_device

    m = args.slab_m
    t0 = time.time()
    tau = 0.25 * 64 / m
    kappa = 2.0 / tau
    geo = k.build_grid((-np.pi, np.pi, -np.pi, np.pi), m, k.StarCurve(1.5, c=0.2, lobes=3))
    wsp = k.InterfaceWorkspace(geo, backend=k.CudaBackend(local, timing=False))
    sol = k.StaticPlaneWave(kappa=kappa)
    cps = wsp.cps
    X, Y = geo.grid.X, geo.grid.Y
    interior = geo.classification.interior
    F = torch.from_numpy(np.where(interior, sol.f(X, Y), 0.0).reshape(-1)).cuda()
    fg = torch.from_numpy(np.asarray(sol.f(cps.x, cps.y))).cuda()
    g = torch.from_numpy(np.asarray(sol.dirichlet(cps.x, cps.y))).cuda()
    wsp.plan
    torch.cuda.synchronize()
    setup_s = time.time() - t0

    def solve():
        dens = torch.zeros(cps.m, dtype=torch.float64, device="cuda")
        return solve_device(wsp, kappa=kappa, F=F, f_gamma=fg, g=g, density=dens)

    solve()
    reps = max(1, args.slab_steps)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = solve()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    u = out.u.reshape(m + 1, m + 1).cpu().numpy()
    err = float(np.max(np.abs(u[interior] - sol.u(X, Y)[interior])))
    return {"metric": f"KFBI solves/s at {m}^2 (C5, one GPU, plan box solve)",
            "value": 1e3 / ms, "unit": "solves/s", "ms_per_solve": ms, "solves": reps,
            "n_ranks": 1, "iterations": out.iterations, "max_err_interior": err,
            "setup_s": setup_s, "n_ctl": int(cps.m), "kappa": kappa,
            "facr": bool(wsp.plan.facr_for(kappa)),
            "geometry": "star(1.5, 0.2, 3) on [-pi, pi]^2 (SURVEY §8(d) C5)", "mode": "plan"}


def slab_c5(args, ws, rank, local, mode):
    """C5 solves/s over the N ranks (strong scaling) inside the headline run."""
    import torch

    m = args.slab_m
    t0 = time.time()
    geo, wsp, sol, solver, F, fg, g, kappa = c5_problem(m, rank, ws, local, mode, torch)
    torch.cuda.synchronize()
    setup_s = time.time() - t0

    def solve():
        dens = torch.zeros(wsp.cps.m, dtype=torch.float64, device="cuda")
        return solver.solve(kappa=kappa, F=F, f_gamma=fg, g=g, density=dens)

    solve()
    reps = max(1, args.slab_steps)
    _barrier(ws)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = solve()
    b.record()
    torch.cuda.synchronize()
    _barrier(ws)
    ms = _max_over_ranks(a.elapsed_time(b), ws) / reps
    u, tu, tn, it, res, hist = out
    r0, r1 = solver.rows
    interior = geo.classification.interior[r0:r1]
    X, Y = geo.grid.X[r0:r1], geo.grid.Y[r0:r1]
    err = float(np.max(np.abs(u.cpu().numpy()[interior] - sol.u(X, Y)[interior]))) if interior.any() else 0.0
    err = _max_over_ranks(err, ws)
    return {"metric": f"KFBI solves/s at {m}^2 (C5, slab-decomposed over the ranks)",
            "value": 1e3 / ms, "unit": "solves/s", "ms_per_solve": ms, "solves": reps,
            "scaling": "strong", "n_ranks": ws, "iterations": it, "max_err_interior": err,
            "setup_s": setup_s, "n_ctl": int(wsp.cps.m), "kappa": kappa,
            "geometry": "star(1.5, 0.2, 3) on [-pi, pi]^2 (SURVEY §8(d) C5)",
            "mode": mode,
            "transport": {"a2a": "NCCL all_to_all_single x2 + all_reduce per sweep",
                          "p2p": "transposes fused into the passes (CUDA IPC peer stores + "
                                 "peer-flag barrier) + NCCL all_reduce",
                          "carry": "no transposes: tridiagonal column stage pushes 3 values per "
                                   "column to every rank over CUDA IPC peer memory inside the "
                                   "kernel + NCCL all_reduce"}[mode]
                         + (" (1 rank: no traffic)" if ws == 1 else "")}


def c4_cases():
    """SURVEY §6.3 / BASELINE configs[3]: the reference CLI's convergence
    geometries (heat star k=5, wave ellipse, Schrodinger star3 on [-pi, pi]^2)."""
    import paper_2404_14864_b200 as k

    box = (-1.5, 1.5, -1.5, 1.5)
    pibox = (-np.pi, np.pi, -np.pi, np.pi)
    heat, wave, schr = k.HeatPlaneDecay(1.0), k.WaveStanding(0.0), k.SchrodingerPhaseRotation()
    return {
        "heat": (box, k.StarCurve(1.0, c=0.2, lobes=5), heat, dict(
            equation="heat", bc_kind="dirichlet", g=heat.dirichlet, u0=heat.u0,
            lap_u0=heat.lap_u0, c=1.0)),
        "wave": (box, k.EllipseCurve(1.2, 0.8), wave, dict(
            equation="wave", bc_kind="dirichlet", g=wave.dirichlet, u0=wave.u0,
            lap_u0=wave.lap_u0, v0=wave.v0, lap_v0=wave.lap_v0, theta=0.25)),
        "schrodinger": (pibox, k.StarCurve(1.5, c=0.2, lobes=3), schr, dict(
            equation="schrodinger", bc_kind="dirichlet", g=schr.dirichlet, u0=schr.u0,
            lap_u0=schr.lap_u0, potential=schr.potential, w=1.0)),
    }


def run_c4(args):
    """--workload c4 (BASELINE configs[3], report.py:183-225 convergence_study):
    every equation at M = 256..4096, tau = 0.25 * 64 / M, T = 1, errors
    against the exact solution over the interior nodes, orders log2(e_M /
    e_2M), and the steady steps/s of each size (run() with the context
    reused, after one untimed run)."""
    import torch

    import paper_2404_14864_b200 as k

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    sizes = [int(x) for x in args.c4_sizes.split(",")]
    backend = k.CudaBackend(local, timing=False)
    table = {}
    t_all = time.time()
    for eq, (box, curve, sol, kw) in c4_cases().items():
        rows = []
        for m in sizes:
            t0 = time.time()
            geo = k.build_grid(box, m, curve)
            spec = k.ProblemSpec(tau=0.25 * 64 / m, t_final=1.0, **kw)
            ctx = k.StepContext(geo, backend=backend)
            setup = time.time() - t0
            t0 = time.perf_counter()
            res = k.run(spec, geo, context=ctx)        # incl. the operator build
            torch.cuda.synchronize()
            first = time.perf_counter() - t0
            t0 = time.perf_counter()
            res = k.run(spec, geo, context=ctx)
            torch.cuda.synchronize()
            steady = time.perf_counter() - t0
            e_inf, e_2 = k.compute_errors(res.state.u, lambda x, y: sol.u(x, y, 1.0), geo.grid,
                                          geo.classification)
            n = spec.n_steps()
            rows.append({"m": m, "steps": n, "e_inf": float(e_inf), "e_2": float(e_2),
                         "mean_iterations": float(np.mean(res.iterations)),
                         "steps_per_s": n / steady, "first_run_s": first, "setup_s": setup,
                         "operator_form": bool(ctx.operator)})
            del ctx
            torch.cuda.empty_cache()
        for a, b in zip(rows[:-1], rows[1:]):
            b["order_inf"] = float(np.log2(a["e_inf"] / b["e_inf"]))
            b["order_2"] = float(np.log2(a["e_2"] / b["e_2"]))
        table[eq] = rows
    if rank != 0:
        return None
    return {"metric": "KFBI convergence sweep (C4): errors, orders and steps/s per size",
            "value": min(r["steps_per_s"] for rows in table.values() for r in rows if r["m"] == sizes[-1]),
            "unit": f"time steps/s at {sizes[-1]}^2 (slowest equation)", "n_gpus": ws,
            "higher_is_better": True, "dtype": "f64 (heat, wave) / c128 (schrodinger)",
            "data": "synthetic: closed-form manufactured solutions",
            "config": {"workload": "C4: heat star5, wave ellipse, Schrodinger star3; tau = 16/M, T = 1",
                       "sizes": sizes}, "table": table, "wall_s": time.time() - t_all}


def run_c5(args):
    """--workload c5 (BASELINE.json configs[4]): one modified-Helmholtz KFBI
    solve per step at M = 16384 (flower star, StaticPlaneWave, kappa = 2/tau
    with tau = 1/1024), the box solve slab-decomposed over the N ranks
    (dist.SlabRichardson: NCCL all-to-all transposes + one stencil-value
    all-reduce per sweep).  Strong scaling: the N ranks share one problem."""
    import torch

    import paper_2404_14864_b200 as k
    from paper_2404_14864_b200 import dist as D

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    m = args.m if args.m != M_DEFAULT else 16384
    t0 = time.time()
    geo, wsp, sol, solver, F, fg, g, kappa = c5_problem(m, rank, ws, local, args.slab_mode or ("p2p" if args.p2p else "a2a"), torch)
    cps = wsp.cps
    r0, r1 = solver.rows
    X, Y = geo.grid.X[r0:r1], geo.grid.Y[r0:r1]
    torch.cuda.synchronize()
    setup_s = time.time() - t0

    def step():
        dens = torch.zeros(cps.m, dtype=torch.float64, device="cuda")
        return solver.solve(kappa=kappa, F=F, f_gamma=fg, g=g, density=dens)

    for _ in range(args.warmup):
        out = step()
    _barrier(ws)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        out = step()
    b.record()
    torch.cuda.synchronize()
    _barrier(ws)
    ms = _max_over_ranks(a.elapsed_time(b), ws) / args.steps
    u, tu, tn, it, res, hist = out
    interior = geo.classification.interior[r0:r1]
    err = float(np.max(np.abs(u.cpu().numpy()[interior] - sol.u(X, Y)[interior]))) if interior.any() else 0.0
    err = _max_over_ranks(err, ws)
    if rank != 0:
        return None
    return {
        "metric": "KFBI modified-Helmholtz solves/s at 16384^2 (C5, slab-decomposed box solve)",
        "value": 1e3 / ms, "unit": "solves/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: StaticPlaneWave manufactured solution (no RNG)",
        "config": {"workload": f"C5: one KFBI solve per step, {m}x{m}, star(1.5, 0.2, 3) on [-pi, pi]^2, kappa={kappa}",
                   "grid": m, "parallelism": f"slab{ws}",
                   "transport": ("none (1 rank)" if ws == 1 else
                                 "transposes fused into the passes (CUDA IPC peer stores + "
                                 "peer-flag barrier) + NCCL all_reduce" if args.p2p else
                                 "NCCL all_to_all_single + all_reduce"),
                   "p2p": bool(args.p2p)},
        "iterations": it, "residual": res, "max_err_interior": err, "setup_s": setup_s,
        "n_ctl": int(cps.m),
    }


FP64_PEAK_TFLOPS = 33.7     # measured DFMA throughput, tools/mb/dfma.cu


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def _ncu_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(path))
    except Exception:
        return None


# ---------------------------------------------------------------------------
def _oracle_sample(tables, spec_kw, sweeps):
    """Wall time of one oracle time step truncated after `sweeps` sweeps
    (after a warm-up step so the density is warm)."""
    from oracle import kfbi_oracle as O

    keys = ("equation", "g", "u0", "lap_u0", "tau", "t_final", "c", "theta", "w", "potential",
            "splitting", "v0", "lap_v0")
    spec = O.Spec(**{k: spec_kw[k] for k in keys if k in spec_kw})
    st = O.Stepper(tables, spec, max_sweeps=1)
    st.step()                      # untimed: leaves the cold first-step path
    st.max_sweeps = sweeps
    t0 = time.perf_counter()
    st.step()
    return time.perf_counter() - t0


def _cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model(tables_by_eq, spec_kw_by_eq, iters_by_eq, samples=1):
    """Per-step CPU time model: t(step) = t_glue + iters * t_sweep, with t_sweep
    and t_glue from truncated oracle steps of 1 and 2 sweeps."""
    from oracle import kfbi_oracle as O

    O.WORKERS = _cpu_threads()
    out = {}
    for eq, t in tables_by_eq.items():
        t1 = min(_oracle_sample(t, spec_kw_by_eq[eq], 1) for _ in range(samples))
        t2 = min(_oracle_sample(t, spec_kw_by_eq[eq], 2) for _ in range(samples))
        sweep = max(t2 - t1, 1e-9)
        glue = max(t1 - sweep, 0.0)
        it = iters_by_eq[eq]
        out[eq] = {"sweep_s": sweep, "glue_s": glue, "iterations": it,
                   "step_s": glue + it * sweep}
    return out


def cpu_baseline(ctxs, specs, iters, args):
    from oracle import kfbi_oracle as O

    wl = workload(args.m)
    tables = {eq: O.tables_from_workspace(c.workspace) for eq, c in ctxs.items()}
    its = {eq: int(round(float(np.median(iters[eq])))) for eq in ctxs}
    t0 = time.time()
    model = cpu_model(tables, {eq: wl[eq][2] for eq in ctxs}, its)
    total = sum(v["step_s"] for v in model.values())
    return {
        "value": len(ctxs) / total, "unit": "time steps/s", "cores": _cpu_threads(),
        "kind": "port",
        "sample": ("oracle port of the reference (numpy/scipy, scipy.fft workers = all host "
                   "threads, OpenBLAS threads) on the same 4096^2 workload: per equation one "
                   "time step truncated after 1 and after 2 Richardson sweeps gives t_sweep and "
                   "t_glue; step time = t_glue + t_sweep * (iterations per step measured on the "
                   "GPU in this run, identical to the reference's by parity)"),
        "per_equation": model, "sample_wall_s": time.time() - t0,
    }


def run_reference(args):
    """--impl reference: the CPU reference path on the host cores, rank 0 only.

    The oracle port of the reference (oracle/kfbi_oracle.py: numpy/scipy, the
    reference's algorithm line by line, pinned bit for bit to the unmodified
    reference by tests/test_oracle.py) advances each equation of the same
    4096^2 workload with REAL, untruncated Richardson solves: one warm-up step
    (the cold first step), then whole bench steps (one step of every
    equation) until --steps or the time budget is reached; the line reports
    the number of bench steps actually timed and the per-step iterations."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import paper_2404_14864_b200 as k
    from oracle import kfbi_oracle as O

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from conftest import oracle_spec

    O.WORKERS = _cpu_threads()
    m = args.m
    eqs = args.equations
    wl = workload(m)
    t_setup = time.time()
    steppers = {}
    for eq in eqs:
        box, curve, kw = wl[eq]
        # host setup shared with the product (identical to the reference's, tests/test_setup.py)
        tables = O.tables_from_workspace(k.InterfaceWorkspace(k.build_grid(box, m, curve)))
        steppers[eq] = O.Stepper(tables, oracle_spec(kw))
    t_setup = time.time() - t_setup
    t_warm = time.time()
    for eq in eqs:                       # warm-up: the cold first step of every equation
        steppers[eq].step()
    t_warm = time.time() - t_warm
    budget = time.time() + args.ref_budget_s
    step_s, iters = [], {eq: [] for eq in eqs}
    per_eq = {eq: [] for eq in eqs}
    while len(step_s) < max(args.steps, 1):
        tot = 0.0
        for eq in eqs:
            t0 = time.perf_counter()
            steppers[eq].step()
            dt = time.perf_counter() - t0
            per_eq[eq].append(dt)
            iters[eq].append(steppers[eq].iterations[-1])
            tot += dt
        step_s.append(tot)
        if time.time() > budget:
            break
    n = len(step_s)
    per_step = float(np.mean(step_s))
    value = len(eqs) / per_step
    sample = (f"{n} untruncated bench step(s) (one time step of each of {', '.join(eqs)} at "
              f"{m}^2, full Richardson solves to tol 1e-8) after one untimed cold step per "
              f"equation; oracle port of the reference, scipy.fft workers and OpenBLAS on "
              f"{_cpu_threads()} host threads")
    return {
        "metric": METRIC, "value": value, "unit": "time steps/s", "n_gpus": ws,
        "steps": n, "steps_requested": args.steps, "warmup": 1, "ms_per_step": per_step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 (heat, wave) / c128 (schrodinger)",
        "data": "synthetic: closed-form manufactured solutions", "config": config_obj(m, eqs, ws),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "time steps/s", "cores": _cpu_threads(),
                         "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "time steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "per_equation": {eq: {"s_per_step": float(np.mean(per_eq[eq])), "iterations": iters[eq],
                              "warmup_iterations": steppers[eq].iterations[:1]} for eq in eqs},
        "setup_s": t_setup, "warmup_s": t_warm,
    }


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--m", "--grid", dest="m", type=int, default=M_DEFAULT)
    ap.add_argument("--equations", default=",".join(EQUATIONS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", choices=["steps", "c4", "c5"], default="steps",
                    help="steps: the 4096^2 time-step metric (default); c5: one 16384^2 "
                         "KFBI solve per step, slab-decomposed over the ranks")
    ap.add_argument("--profile", action="store_true",
                    help="bracket the headline loop with cudaProfilerStart/Stop (for ncu "
                         "--profile-from-start off launch lists of the timed region only)")
    ap.add_argument("--p2p", action="store_true",
                    help="c5: fuse the slab transposes into the passes (peer-memory stores)")
    ap.add_argument("--ref-budget-s", type=float, default=90.0,
                    help="reference arm: stop after the bench step that crosses this budget")
    ap.add_argument("--repeats", type=int, default=5,
                    help="timed regions of K steps each; value = their median")
    ap.add_argument("--no-pipeline-pass", action="store_true",
                    help="skip the pipeline-form measurement")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the C1-C3 run() measurements")
    ap.add_argument("--no-slab", action="store_true",
                    help="skip the C5 slab-decomposed solve measurement")
    ap.add_argument("--slab-m", type=int, default=16384)
    ap.add_argument("--c4-sizes", default="256,512,1024,2048,4096")
    ap.add_argument("--slab-steps", type=int, default=3)
    ap.add_argument("--slab-mode", choices=["a2a", "p2p", "carry"], default=None,
                    help="c5: slab exchange (default a2a, or p2p with --p2p)")
    ap.add_argument("--sequential", action="store_true",
                    help="step the three equations on one stream (default: one stream each)")
    ap.add_argument("--pipeline", action="store_true",
                    help="run every Richardson sweep through the full pipeline (no trace operator)")
    args = ap.parse_args(argv)
    args.equations = tuple(e for e in args.equations.split(",") if e)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        line = run_reference(args)
    elif args.workload == "c5":
        line = run_c5(args)
    elif args.workload == "c4":
        line = run_c4(args)
    else:
        line = run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
