"""The N > 1 bench plumbing (replicas only) on CPU: two gloo ranks launched the way the driver
launches bench.py (torch.distributed.run, 127.0.0.1); barrier, max-over-ranks timing and the whole-job value."""
import os
import socket
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

WORKER = r"""
import json, os, sys
sys.path.insert(0, os.environ["KSB_ROOT"])
import bench
world, rank, local = bench.dist_init("gloo")
bench.barrier(world)
ms_local = 10.0 * (rank + 1)                 # rank 1 is the slow one
value, ms = bench.replica_value(1000.0, ms_local, world)
with open(os.path.join(os.environ["KSB_OUT"], f"rank{rank}.json"), "w") as f:
    json.dump({"rank": rank, "world": world, "ms": ms, "value": value}, f)
import torch.distributed as dist
dist.destroy_process_group()
"""


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_gloo_replicas(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, KSB_ROOT=str(ROOT), KSB_OUT=str(tmp_path), CUDA_VISIBLE_DEVICES="")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(free_port()), str(script)]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    import json
    lines = [json.loads((tmp_path / f"rank{r}.json").read_text()) for r in range(2)]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    for d in lines:
        assert d["world"] == 2
        assert d["ms"] == 20.0                         # max over ranks, every rank sees it
        assert abs(d["value"] - 2 * 1000.0 / 0.020) < 1e-6  # all ranks' units over the slowest time
