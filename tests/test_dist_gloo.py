"""Multi-process (one process per rank) host path on CPU: torchrun + gloo,
world sizes 2 and 3 (tree + broadcast for non-power-of-two P)."""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3, 4])
def test_dist_host_path(world):
    env = dict(os.environ)
    env.pop("CUDA_VISIBLE_DEVICES", None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "tests", "dist_worker.py")]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=240, env=env, cwd=ROOT)
    assert proc.returncode == 0, proc.stderr[-3000:]
    dec = json.JSONDecoder()  # ranks share stdout: split on the marker, not on lines
    results = [dec.raw_decode(chunk.strip())[0] for chunk in proc.stdout.split("RESULT ")[1:]]
    assert len(results) == world
    for res in results:
        r = res["rank"]
        assert res["ring"] == f"hi{(r - 1) % world}"
        assert res["allgather"] == [f"from-{q}" for q in range(world)]
        assert res["bcast"] == "root"
        assert res["tree_ok"], res
        assert res["butterfly_ok"], res
