"""Host-side logic of bench.py's N>1 path (replicas only), on CPU with gloo, world size 2.

The B200 path does not shard: --gpus N runs N independent
replicas, and the only cross-rank steps are a barrier and the max of the
device-timed step time.  These tests run that plumbing in two processes."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


WORKER = r"""
import json, os, sys
sys.path.insert(0, sys.argv[1])
import bench
rank, ws = bench.dist_setup()
bench.barrier(ws)
# each rank pretends its replica took (rank + 1) * 10 ms for 1e9 edges
t = bench.reduce_max((rank + 1) * 10.0, ws)
v = bench.aggregate_value(1e9, t * 1e-3, ws)
# the reference arm prints on rank 0 only
print(json.dumps({"rank": rank, "ws": ws, "max_ms": t, "value": v}), flush=True)
import torch.distributed as dist
dist.destroy_process_group()
"""


def test_two_rank_max_and_aggregate(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    port = _free_port()
    procs = []
    for rank in range(2):
        env = dict(os.environ, RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, str(script), ROOT], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = []
    for p in procs:
        out, err = p.communicate(timeout=180)
        assert p.returncode == 0, err
        outs.append(json.loads(out.strip().splitlines()[-1]))
    for o in outs:
        assert o["ws"] == 2
        assert o["max_ms"] == pytest.approx(20.0)          # max over ranks, not the local time
        assert o["value"] == pytest.approx(2 * 1e9 / 0.020)  # all ranks' units / slowest rank's time


def test_reference_arm_other_ranks_silent(tmp_path):
    """--impl reference under torchrun: rank 0 alone runs and prints; others exit 0 without work."""
    port = _free_port()
    env = dict(os.environ, RANK="1", LOCAL_RANK="1", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
               MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""
