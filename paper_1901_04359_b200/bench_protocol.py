"""The reference's collective benchmark protocol on the device collectives.

Mirrors reference `cli.py:246-294` (`run_bench`): for each collective
("dense", "topk", "gtopk") a fresh cluster of P ranks, every rank's input drawn
exactly as the reference draws it (`np.random.default_rng(seed)`, one
N(0,1) vector of m float32 per rank, its exact top-k as the sparse input),
`warmup_reps` untimed calls, `repeats` timed calls, and one CSV row per rank:
`CollectiveStats` (bytes / messages per call from the endpoint's stats,
`comm_rounds`, mean wall ms) plus the wall-time standard deviation --
`BENCH_HEADER` is the reference's header.

Differences, by design: the inputs are resident in HBM (DeviceSparseVector /
CUDA tensors, the device API of `collectives.py`), every call is followed by
a device synchronisation so the wall time covers the kernels, and the
cluster is `create_local_cluster(P)` on one GPU (in-process ranks, like the
reference's threads) or -- `endpoint` given -- this torchrun rank's endpoint
of a one-process-per-GPU job (init_dist_cluster).  `device_ms` adds the
CUDA-event time of the same calls.
"""

from __future__ import annotations

import time

import numpy as np
import torch

from . import collectives
from .collectives import CollectiveStats
from .device import DeviceList
from .sparse import DeviceSparseVector, k_from_density, top_k_select
from .transport import create_local_cluster, run_workers

BENCH_HEADER = CollectiveStats.CSV_HEADER + ",wall_ms_std"
ALGOS = ("dense", "topk", "gtopk")


def bench_inputs(P: int, m: int, k: int, seed: int = 0):
    """The reference's inputs (cli.py:249-252): per rank a dense N(0,1) float32
    vector and its exact top-k (host SparseVector)."""
    rng = np.random.default_rng(seed)
    dense_in = [rng.standard_normal(m).astype(np.float32) for _ in range(P)]
    sparse_in = [top_k_select(v, k)[0] for v in dense_in]
    return dense_in, sparse_in


def _rank_bench(ep, algo, g_dev, s_dev, k, P, m, warmup_reps, repeats):
    dev = g_dev.device

    def once():
        if algo == "dense":
            collectives.dense_ring_allreduce(ep, g_dev)
        elif algo == "topk":
            collectives.topk_allreduce(ep, s_dev, P)
        else:
            collectives.gtopk_allreduce(ep, s_dev, k, P)
        torch.cuda.synchronize(dev)

    for _ in range(warmup_reps):
        once()
    walls, devs = [], []
    before = ep.stats.snapshot()
    for _ in range(repeats):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        once()
        e1.record()
        walls.append((time.perf_counter() - t0) * 1e3)
        e1.synchronize()
        devs.append(e0.elapsed_time(e1))
    delta = ep.stats.snapshot().delta(before)
    stats = CollectiveStats(collective=algo, P=P, m=m, k=k, rank=ep.rank,
                            bytes_sent=delta.bytes_sent // repeats, bytes_recv=delta.bytes_recv // repeats,
                            msgs=delta.msgs_sent // repeats, rounds=collectives.comm_rounds(algo, P),
                            wall_ms=float(np.mean(walls)))
    return stats, float(np.std(walls)), float(np.mean(devs))


def run_bench(P: int, m: int = 10000, k: int | None = None, rho: float = 0.001, seed: int = 0,
              warmup_reps: int = 3, repeats: int = 10, device=None, endpoint=None,
              with_device_ms: bool = False) -> list[str]:
    """CSV rows (no header) of the reference's bench for P ranks; with
    `endpoint` (a torchrun rank) only that rank's rows."""
    k = k if k is not None else k_from_density(rho, m)
    dense_in, sparse_in = bench_inputs(P, m, k, seed)
    rows = []
    for algo in ALGOS:
        if endpoint is not None:
            eps = None
            dev = endpoint.group.device
        else:
            dev = torch.device("cuda", 0) if device is None else torch.device(device)
            eps = create_local_cluster(P, device=dev)

        def worker(ep, algo=algo, dev=dev):
            g_dev = torch.from_numpy(dense_in[ep.rank]).to(dev)
            s = sparse_in[ep.rank]
            s_dev = DeviceSparseVector(DeviceList.from_host(m, s.indices, s.values, dev, k))
            return _rank_bench(ep, algo, g_dev, s_dev, k, P, m, warmup_reps, repeats)

        results = [worker(endpoint)] if eps is None else run_workers(eps, worker)
        for stats, std, dms in results:
            row = f"{stats.csv_row()},{std:.6f}"
            if with_device_ms:
                row += f",{dms:.6f}"
            rows.append(row)
        if eps is not None:
            for ep in eps:
                ep.close()
    return rows
