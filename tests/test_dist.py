"""N>1 path on CPU (gloo, world_size 2): the bench's timing reduction (max
over ranks), the whole-job weak-scaling rate, per-rank independent objects,
and that only rank 0 prints a JSON line (the reference arm's other ranks do
no work)."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        sys.path.insert(0, str(ROOT))
        import bench

        ms = [3.5, 7.25][rank]
        got = bench.max_over_ranks(ms, ws, device="cpu")
        from paper_2203_12339_b200.config import C1
        from paper_2203_12339_b200.geometry import make_geometry_image

        g = make_geometry_image(C1.side, C1.radius, C1.bump_amp, C1.bump_terms, C1.seed + rank)
        digest = float(np.asarray(g.positions, np.float64).sum())
        dist.barrier()
        q.put((rank, got, digest))
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_and_independent_objects_gloo():
    ws, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [7.25, 7.25]  # every rank sees the slowest time
    assert res[0][2] != res[1][2]  # rank-seeded, independent objects


def test_whole_job_rate_weak_scaling():
    sys.path.insert(0, str(ROOT))
    import bench

    one = bench.whole_job_rate(65536, 1, 100, 50.0)
    two = bench.whole_job_rate(65536, 2, 100, 50.0)
    assert two == pytest.approx(2 * one)
    assert one == pytest.approx(65536 * 100 / 0.05)


def test_reference_arm_other_ranks_exit_quietly():
    """`bench.py --impl reference` under torchrun: rank != 0 returns without
    work or output (only rank 0 prints the JSON line)."""
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0"], env=env, capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0
    assert r.stdout.strip() == ""
