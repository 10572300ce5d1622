"""Multi-process host logic on CPU (gloo, world_size 2): the replica bench's
max-over-ranks aggregation, and the reference arm's CLI contract."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    sys.path.insert(0, str(ROOT))
    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank r "took" 10*(r+1) ms for 5 steps of a 1000-edge replica
    value, tmax = bench.replica_value(10.0 * (rank + 1), world, 1000, 5, dist, "cpu")
    q.put((rank, value, tmax))
    dist.barrier()
    dist.destroy_process_group()


def test_replica_max_over_ranks_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = sorted(q.get(timeout=10) for _ in range(2))
    for rank, value, tmax in got:
        assert tmax == 20.0  # the slowest rank defines the job time
        assert value == pytest.approx(2 * 1000 * 5 / 0.020)


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=300,
                         cwd=str(ROOT))
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    assert line["value"] > 0


def test_bench_spawns_n_ranks():
    """``bench.py --gpus 2`` outside torchrun re-launches itself as 2 ranks
    (gloo here, NCCL on a GPU box) -- the replica bench's process plumbing."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--check-ranks"],
                         capture_output=True, text=True, timeout=300, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["ranks"] == 2 and line["allreduce_sum"] == 2.0
