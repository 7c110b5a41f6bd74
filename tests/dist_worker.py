"""Worker for tests/test_dist_gloo.py, launched with torch.distributed.run on CPU
(gloo).  Exercises the one-process-per-rank host plumbing of dist.py: byte
send/recv, barrier, allgather / binomial broadcast, and the per-rank exchange
SCHEDULES the NVLink kernel executes (butterfly / tree + broadcast) -- here
run step by step with encode_sparse messages over gloo and the CPU oracle's ⊤
as the merge (the oracle is the checker; the GPU kernel is tested on GPUs).
Prints one JSON line per rank."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import gtopk_oracle as orc  # noqa: E402
from paper_1901_04359_b200 import collectives as coll  # noqa: E402
from paper_1901_04359_b200.dist import init_dist_cluster  # noqa: E402
from paper_1901_04359_b200.sparse import SparseVector  # noqa: E402
from paper_1901_04359_b200.transport import decode_sparse, encode_sparse  # noqa: E402


def run_schedule(ep, steps, local: SparseVector, k: int) -> SparseVector:
    acc = local
    for j, (send_to, recv_from, merge) in enumerate(steps):
        if send_to >= 0:
            ep.send(send_to, 0x4000 + j, encode_sparse(acc))
        if recv_from >= 0:
            got = decode_sparse(ep.recv(recv_from, 0x4000 + j), local.dim)
            if merge:
                i, v = orc.top_op(got.indices, got.values, acc.indices, acc.values, k)
                acc = SparseVector(local.dim, i, v)
            else:
                acc = got
    return acc


def main():
    ep = init_dist_cluster(device_collectives=False, timeout=30)
    r, P = ep.rank, ep.world_size
    out = {"rank": r, "world": P}
    # byte transport + barrier
    ep.barrier()
    ep.send((r + 1) % P, 7, f"hi{r}".encode())
    out["ring"] = ep.recv((r - 1) % P, 7).decode()
    out["allgather"] = [b.decode() for b in coll.allgather(ep, f"from-{r}".encode())]
    out["bcast"] = coll.binomial_bcast(ep, 0, b"root" if r == 0 else None).decode()
    ep.barrier()
    # exchange schedules vs the reference tree fold
    rng = np.random.default_rng(4242)
    ok_tree, ok_fly, trials = True, True, 25
    for _ in range(trials):
        m = int(rng.integers(12, 200))
        k = int(rng.integers(1, 12))
        lists = [orc.top_k_select(rng.integers(-3, 4, m).astype(np.float32), k)[:2] for _ in range(P)]
        wi, wv = orc.tree_fold(lists, k)
        mine = SparseVector(m, *lists[r])
        before = ep.stats.snapshot()
        got = run_schedule(ep, coll.tree_schedule(r, P), mine, k)
        d = ep.stats.snapshot().delta(before)
        ok_tree &= np.array_equal(got.indices, wi) and np.array_equal(got.values.view(np.uint32),
                                                                     np.asarray(wv, np.float32).view(np.uint32))
        counts = orc.gtopk_message_counts(P)[r]
        ok_tree &= d.msgs_sent == counts["msgs_sent"] and d.msgs_recv == counts["msgs_recv"]
        if P & (P - 1) == 0:
            got = run_schedule(ep, coll.butterfly_schedule(r, P), mine, k)
            ok_fly &= np.array_equal(got.indices, wi) and np.array_equal(got.values, wv)
    out["tree_ok"] = bool(ok_tree)
    out["butterfly_ok"] = bool(ok_fly)
    ep.barrier()
    print("RESULT " + json.dumps(out), flush=True)
    ep.close()  # wait for this rank's in-flight sends before tearing gloo down
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
