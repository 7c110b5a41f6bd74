"""Latency of the TCP backend's host-staged gTopKAllReduce (tcp.py): P ranks
as threads of one process on cuda:0 over a 127.0.0.1 mesh, device lists of
k entries (the headline k = 25,600 by default); median wall time per call
over 30 calls after 5 warm-up calls, max over ranks.  One JSON line per P."""
import json
import os
import socket
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1901_04359_b200 as gk  # noqa: E402
from paper_1901_04359_b200 import collectives as coll  # noqa: E402
from paper_1901_04359_b200 import tcp  # noqa: E402
from paper_1901_04359_b200.device import DeviceList  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 25_600
dev = torch.device("cuda", 0)


def mesh(P):
    socks = [socket.socket() for _ in range(P)]
    for s in socks:
        s.bind(("127.0.0.1", 0))
    cfg = tcp.ClusterConfig(P, "tcp", [("127.0.0.1", s.getsockname()[1]) for s in socks], 60.0)
    for s in socks:
        s.close()
    eps = [None] * P
    ts = [threading.Thread(target=lambda r=r: eps.__setitem__(r, tcp.connect_tcp_cluster(cfg, r, dev)))
          for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return eps


for P in (2, 4, 8):
    rng = np.random.default_rng(P)
    lists = []
    for _ in range(P):
        idx = np.sort(rng.choice(m, k, replace=False))
        lists.append(gk.DeviceSparseVector(DeviceList.from_host(m, idx, rng.standard_normal(k).astype(np.float32), dev)))
    eps = mesh(P)

    def worker(ep):
        times = []
        for it in range(35):
            ep.barrier()
            t0 = time.perf_counter()
            coll.gtopk_allreduce(ep, lists[ep.rank], k)
            torch.cuda.synchronize(dev)
            if it >= 5:
                times.append(time.perf_counter() - t0)
        return float(np.median(times))

    try:
        med = gk.run_workers(eps, worker)
    finally:
        for ep in eps:
            ep.close()
    print(json.dumps({"backend": "tcp (127.0.0.1, ranks as threads on one GPU)", "P": P, "m": m, "k": k,
                      "gtopk_allreduce_ms_median_max_over_ranks": round(max(med) * 1e3, 3),
                      "wire_bytes_per_message": 12 + 12 * k}), flush=True)
