"""Multi-process host logic of bench.py on CPU (gloo, world_size 2): ranks
agree on the max-over-ranks time, the barrier completes, and the reference
arm runs on rank 0 only.  The KFBI time loop itself is sequential, so
`bench.py --gpus N` runs N independent replicas."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist

    import bench

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        v = bench._max_over_ranks(1.5 + rank, world)
        bench._barrier(world)

        class A:
            steps, warmup, m, equations = 1, 3, 64, ("heat",)

        ref = bench.run_reference(A()) if rank != 0 else "rank0-skipped"
        out[rank] = (v, ref)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_reduction_and_rank0_only_reference():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert out[0][0] == pytest.approx(2.5) and out[1][0] == pytest.approx(2.5)
    assert out[1][1] is None          # non-zero ranks do no reference work


def test_torchrun_two_ranks_reference_arm_contract():
    # the driver's exact launch (torch.distributed.run, 127.0.0.1) of the
    # reference arm on CPU: rank 0 prints ONE JSON line, rank 1 exits 0 silently
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3", "--grid", "64",
           "--equations", "heat", "--ref-budget-s", "20"]
    env = dict(os.environ, OMP_NUM_THREADS="1", CUDA_VISIBLE_DEVICES="")
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["n_gpus"] == 2
    assert d["e2e"]["h2d_bytes_per_step"] == 0
