"""BASELINE.json configs 1-5 on the GPU (development/evidence tool, not the bench).

    python tools/sweep.py [--configs 1,2,3,4,5] [--steps 50] [--out f.jsonl]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tools/sweep.py ...

Per config and P (= the torchrun world size, one rank per GPU):
  pipeline_ms : gtopk S-SGD step (K1 -> fused NVLink exchange -> K3) replayed
                from CUDA graphs, gradients resident in HBM, steady-state
                residual (precondition ~2/rho untimed steps), CUDA events,
                max over ranks -- bench.py's `value` at this (m, rho, P).
  api_ms      : the public optimizer step (gtopk_step / topk_step / dense_step)
                with device-resident gradients, one status read per step
                (host syncs included), max over ranks.
  cpu_ref     : the reference's CPU path at the same (m, rho, P) -- the oracle
                port (numpy, one host thread per rank like run_workers), full
                size, mean over `--cpu-steps` timed steps -- with the host's
                core count and CPU model (rank 0 only; `--no-cpu` skips it).
  protocol    : `--protocol`: the reference's collective benchmark
                (cli.py:246-294: warmup 3, repeats 10, per-rank rows of bytes
                / messages / rounds / mean wall ms / std) for configs 1 and 3
                through bench_protocol.run_bench, CSV with the reference's header.
Config 1 (m=1M, P=4 simulated workers) runs in-process on one GPU: 4 logical
ranks (create_local_cluster + run_workers), the reference's own harness.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def k_from_density(rho, m):
    return max(1, min(m, round(rho * m)))


CONFIGS = {
    2: [("resnet20", 270_000, 0.001)],
    3: [("vgg16", 14_700_000, 0.001)],
    4: [("resnet50", 25_600_000, 0.001)],
    5: [(name, m, rho) for name, m in (("alexnet", 61_000_000), ("lstm-ptb", 66_000_000))
        for rho in (0.0005, 0.001, 0.002, 0.005, 0.01)],
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=1)
    ap.add_argument("--protocol", action="store_true")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_1901_04359_b200 as gk
    from paper_1901_04359_b200 import optimizer as opt
    from paper_1901_04359_b200.pipeline import GTopKPipeline

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        from paper_1901_04359_b200.dist import init_dist_cluster

        ep = init_dist_cluster(timeout=60.0)
    else:
        torch.cuda.set_device(0)
        ep = gk.create_local_cluster(1)[0]
        dist = None
    dev = ep.group.device
    P = world
    rows = []

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, steps):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        e1.synchronize()
        return max_over_ranks(e0.elapsed_time(e1) / steps)

    from bench import cpu_model, host_cores, oracle_steps

    def cpu_ref(m, rho, Pc):
        if rank != 0 or args.no_cpu:
            return None
        ms, desc = oracle_steps(m, rho, Pc, args.cpu_steps, 0)
        return {"ms": round(ms, 1), "kind": "port", "cores": min(Pc, host_cores()),
                "host_cores": host_cores(), "cpu": cpu_model(), "sample": desc}

    def emit(row):
        row.update(P=P, n_gpus=world)
        rows.append(row)
        if rank == 0:
            print(json.dumps(row), flush=True)

    wanted = [int(c) for c in args.configs.split(",") if c]

    if 1 in wanted and world == 1:
        # config 1: P=4 simulated workers on one GPU through the reference harness
        m, rho, Pl = 1_000_000, 0.001, 4
        k = k_from_density(rho, m)
        rng = np.random.default_rng(0)
        grads = [torch.from_numpy(rng.standard_normal(m).astype(np.float32)).to(dev) for _ in range(Pl)]
        eps = gk.create_local_cluster(Pl)
        states = [opt.make_state(torch.zeros(m, device=dev), lr=0.01) for _ in range(Pl)]

        def worker(e):
            for _ in range(3):
                opt.gtopk_step(states[e.rank], e, grads[e.rank], k, Pl)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            for _ in range(args.steps):
                opt.gtopk_step(states[e.rank], e, grads[e.rank], k, Pl)
            torch.cuda.synchronize(dev)
            return (time.perf_counter() - t0) * 1e3 / args.steps

        ts = gk.run_workers(eps, worker)
        row = {"config": 1, "model": "synthetic-1M", "m": m, "rho": rho, "k": k,
               "note": "P=4 logical ranks on one GPU (create_local_cluster + run_workers), host wall clock",
               "api_ms": {"gtopk_step": round(max(ts), 4)}, "cpu_ref": cpu_ref(m, rho, Pl)}
        rows.append(row)
        print(json.dumps(row), flush=True)

    for c in wanted:
        for name, m, rho in CONFIGS.get(c, []):
            k = k_from_density(rho, m)
            rng = np.random.default_rng(0)
            host = []
            for j in range(P + rank + 1):
                x = rng.standard_normal(m).astype(np.float32)
                if j in (rank, P + rank):
                    host.append(x)
            grads = [torch.from_numpy(x).to(dev) for x in host]
            del host
            state = opt.make_state(torch.zeros(m, device=dev), lr=0.01)
            pipe = GTopKPipeline(ep, state, k, grads)
            pipe.capture()
            pipe.run(min(3000, int(2 / rho)))
            pipe.status.zero_()
            pipe.run(10)
            pipe_ms = timed(lambda: pipe.run(args.steps), 1) / args.steps  # block-graph replays
            fb = bool(int(pipe.status.item()) & 0x2)
            pipe.check()
            pipe.sync_state()
            row = {"config": c, "model": name, "m": m, "rho": rho, "k": k,
                   "pipeline_ms": round(pipe_ms, 4), "dense_fallback_in_timed_steps": fb,
                   "select_gbs_12m": round(12 * m / (pipe_ms * 1e-3) / 1e9, 1) if P == 1 else None}
            api = {}
            n_api = max(5, args.steps // 5)
            it = [0]

            def g_step():
                opt.gtopk_step(state, ep, grads[it[0] % 2], k, P)
                it[0] += 1

            g_step()
            api["gtopk_step"] = round(timed(g_step, n_api), 4)
            if c == 3:
                st_t = opt.make_state(torch.zeros(m, device=dev), lr=0.01)
                st_d = opt.make_state(torch.zeros(m, device=dev), lr=0.01)
                opt.topk_step(st_t, ep, grads[0], k, P)
                opt.dense_step(st_d, ep, grads[0], P)
                api["topk_step"] = round(timed(lambda: opt.topk_step(st_t, ep, grads[0], k, P), n_api), 4)
                api["dense_step"] = round(timed(lambda: opt.dense_step(st_d, ep, grads[0], P), n_api), 4)
                del st_t, st_d
            row["api_ms"] = api
            row["cpu_ref"] = cpu_ref(m, rho, P)
            emit(row)
            del pipe, state, grads
            torch.cuda.empty_cache()

    if args.protocol:
        from paper_1901_04359_b200 import bench_protocol

        cases = []
        if world == 1:
            cases.append((4, 1_000_000, 0.001, None))  # config 1: P=4 in-process ranks on one GPU
        cases.append((P, 14_700_000, 0.001, ep if world > 1 else None))  # config 3 at this job's P
        for Pc, m, rho, e in cases:
            rws = bench_protocol.run_bench(Pc, m=m, rho=rho, endpoint=e, with_device_ms=True)
            if world > 1:
                allr = [None] * world
                dist.all_gather_object(allr, rws)
                rws = [r for part in allr for r in part]
            if rank == 0:
                print(bench_protocol.BENCH_HEADER + ",device_ms", flush=True)
                for r in rws:
                    print(r, flush=True)
                rows.append({"protocol": {"P": Pc, "m": m, "rho": rho, "rows": rws}})

    if rank == 0 and args.out:
        with open(args.out, "w") as fh:
            for r in rows:
                fh.write(json.dumps(r) + "\n")
    if dist is not None:
        dist.barrier()
        ep.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
