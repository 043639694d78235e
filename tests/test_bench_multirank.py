"""The N>1 plumbing of bench.py on CPU (gloo, world size 2): single-token
decode does not shard ("replicas only"), so the only
cross-rank steps are the barrier and the max-over-ranks timing; the reference
arm runs on rank 0 alone and the other ranks exit without work."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, local = bench.dist_env()
        assert (r, w, local) == (rank, world, rank)
        bench.barrier(world)
        got = bench.max_over_ranks(10.0 + 5.0 * rank, world, device="cpu")
        q.put((rank, got))
        bench.barrier(world)
    finally:
        dist.destroy_process_group()


def test_barrier_and_max_over_ranks_gloo():
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
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: 15.0, 1: 15.0}


def test_reference_arm_nonzero_rank_exits_without_work():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "1"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip() == ""


def test_replica_value_is_whole_job_throughput():
    """value = N * steps / max-over-ranks time: the units all ranks processed."""
    sys.path.insert(0, str(ROOT))
    import bench
    assert bench.whole_job_value(1, 20, 1000.0) == 20.0
    assert bench.whole_job_value(4, 20, 2000.0) == 40.0  # 4 ranks x 20 tokens in 2 s
    assert bench.max_over_ranks(3.5, 1) == 3.5


def test_ep_mode_under_torchrun_gloo():
    """bench.py --ep (config 5) under torchrun at world size 2: experts sharded,
    all-to-all dispatch/combine, max-over-ranks timing; gloo + a toy shape on
    CPU (--ep-cpu), the same plumbing NCCL runs on GPUs."""
    import json
    port = _free_port()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", str(port), str(ROOT / "bench.py"), "--gpus", "2",
                        "--ep-cpu", "--steps", "2", "--warmup", "1"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["experts_per_rank"] == 4 and d["value"] > 0
    assert d["scaling"] == "strong"
