"""CPU coverage of bench.py's N > 1 path (replicas only) with world_size-2 gloo process groups:
max-over-ranks timing, whole-job throughput, and the reference arm exiting 0 on ranks != 0."""
import os
import socket
import subprocess
import sys

import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    t = [3.0, 5.0][rank]                           # per-rank device time of the timed region
    tmax = bench.max_over_ranks(t)
    v = bench.replica_throughput(world, 1.0e9, tmax)
    out[rank] = (tmax, v)
    dist.destroy_process_group()


def test_max_over_ranks_and_replica_throughput_gloo():
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        tmax, v = out[r]
        assert tmax == 5.0                          # every rank sees the slowest rank's time
        assert abs(v - 2 * 1.0e9 / 5.0) < 1e-6      # whole-job value: both replicas' work / slowest time


def test_single_process_identity():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.max_over_ranks(2.5) == 2.5
    assert bench.replica_throughput(1, 10.0, 2.0) == 5.0


def test_reference_arm_nonzero_rank_exits_quietly():
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == ""
