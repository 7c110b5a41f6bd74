"""Benchmark: gTopKAllReduce+select ms/iter at m=25.6M, rho=0.001 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    # N>1: python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
    #      --master-port P bench.py --gpus N ...

A "step" is one iteration of the gTop-k S-SGD communication hot path on every
rank (reference optimizer.py:199-252): K1 residual-add + exact top-k select
over the rank's m-length gradient, gTopKAllReduce over the P = N ranks (the
fused NVLink exchange kernel; absent at N = 1), K3 sparse update + extra
residual.  Weak scaling: every rank owns a full m = 25.6M gradient (ResNet-50
size, BASELINE configs[3]).

value : ms/iter of the device-resident pipeline (gradients already in HBM,
        steps replayed from CUDA graphs), CUDA events on the launching
        stream, max over ranks.  Each step streams 307 MB through K1 -- far
        above the 126 MB L2 -- so no explicit L2 flush is needed.
e2e   : the same metric through the public API `optimizer.gtopk_step` with
        the gradient in pinned HOST memory: H2D of 4m bytes and a D2H of the
        8-byte (status, global nnz) word inside every timed step.
roofline : K1's main HBM pass, 12m algorithmic bytes / its CUDA-event
        duration (measured live on its stream: back-to-back launches of the
        pass alone on the steady-state residual and window) vs the measured
        HBM peak.
cpu_baseline : the numpy oracle port of the reference (oracle/) on host cores.
--impl reference : the reference arm -- the oracle port of the reference's CPU
        path (the reference is pure Python/numpy; it cannot run on the GPU).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "gTopKAllReduce+select ms/iter at m=25.6M ρ=0.001 @1/2/4/8 B200; select HBM GB/s"
DATA = "synthetic: cli.run_bench draws (seed 0, rank r = draw r; next batch = draw P + r)"
M_DEFAULT = 25_600_000
RHO_DEFAULT = 0.001


def k_from_density(rho, m):
    return max(1, min(m, round(rho * m)))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic():
    """dram bytes per launch of K1's main pass from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "select_main_ncu.json")) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the GPU is busy."""

    QUERY = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def mark(self):
        return time.monotonic()

    def stop(self, t0, t1):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        for t, line in self.lines:
            if not (t0 <= t <= t1):
                continue
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for name, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle port of the reference's CPU path
# ---------------------------------------------------------------------------


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def workload_config(m, rho, P):
    """The `config` both arms report, key for key (the driver compares them)."""
    k = k_from_density(rho, m)
    return {"workload": f"resnet50-size gradient m={m} rho={rho} (k={k}), P={P} ranks, one per GPU",
            "m": m, "k": k, "rho": rho, "P": P}


def oracle_steps(m, rho, P, steps, warmup):
    """The reference's CPU path (the oracle port: numpy, one host thread per
    rank like run_workers) on the FULL workload: `warmup` untimed and `steps`
    timed gtopk steps (residual-add + select + tree fold + update) on the same
    gradients as the GPU arm (cli.run_bench draws: seed 0, rank r = draw r;
    next batch = draw P + r).  Returns (ms per step, description)."""
    from oracle import gtopk_oracle as orc

    k = k_from_density(rho, m)
    rng = np.random.default_rng(0)
    draws = [rng.standard_normal(m).astype(np.float32) for _ in range(2 * P)]
    batches = [draws[:P], draws[P:]]
    states = [orc.State(np.zeros(m, np.float32), 0.01) for _ in range(P)]
    for i in range(warmup):
        orc.threaded_gtopk_step(states, batches[i % 2], k)
    times = []
    for i in range(steps):
        t0 = time.perf_counter()
        orc.threaded_gtopk_step(states, batches[(warmup + i) % 2], k)
        times.append(time.perf_counter() - t0)
    ms = statistics.mean(times) * 1e3
    sd = statistics.pstdev(times) * 1e3 if len(times) > 1 else 0.0
    desc = (f"{steps} timed (+{warmup} untimed) full-size oracle gtopk steps (m={m}, k={k}) on {P} host "
            f"thread(s), one per rank; mean {ms:.1f} ms, std {sd:.1f} ms; {host_cores()} cores available "
            f"({cpu_model()})")
    return ms, desc


# ---------------------------------------------------------------------------
# reference arm: the reference's CPU path (oracle port) on the host cores
# ---------------------------------------------------------------------------


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    P = max(1, world)
    m, rho = args.m, args.rho
    # full size, no extrapolation: ~3.6 s per step at the headline, so the
    # driver's --steps 20 --warmup 5 run takes ~1.5 min; the warm-up is capped
    # at 3 steps (the CPU path has no caches to warm beyond the first call)
    ms, sample = oracle_steps(m, rho, P, args.steps, min(args.warmup, 3))
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(ms, 3),
        "unit": "ms",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 3),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": DATA,
        "config": workload_config(m, rho, P),
        "cpu_baseline": {"value": round(ms, 3), "unit": "ms", "cores": min(P, host_cores()), "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(ms, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# the B200 arm
# ---------------------------------------------------------------------------


def run_b200(args, rank, world):
    import torch

    import paper_1901_04359_b200 as gk
    from paper_1901_04359_b200 import _lib
    from paper_1901_04359_b200 import optimizer as opt
    from paper_1901_04359_b200.pipeline import GTopKPipeline

    lib = _lib.load()
    if world > 1:
        from paper_1901_04359_b200.dist import init_dist_cluster
        import torch.distributed as dist

        ep = init_dist_cluster(timeout=60.0, mode=args.mode)
    else:
        torch.cuda.set_device(0)
        ep = gk.create_local_cluster(1)[0]
        dist = None
    dev = ep.group.device
    P = world
    m, rho = args.m, args.rho
    k = k_from_density(rho, m)

    # synthetic gradients, cli.run_bench's stream (cli.py:249-250): seed 0,
    # rank r's gradient is the r-th sequential draw; the pipeline alternates it
    # with the (P + r)-th draw as the next batch's gradient
    rng = np.random.default_rng(0)
    host_grads = []
    for j in range(P + rank + 1):
        x = rng.standard_normal(m).astype(np.float32)
        if j == rank or j == P + rank:
            host_grads.append(x)
    dgrads = [torch.from_numpy(g).to(dev) for g in host_grads]

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

    # ---- device-resident pipeline, CUDA graphs ------------------------------
    trace = None
    if os.environ.get("GTK_TRACE") and world > 1:
        trace = torch.zeros(128, dtype=torch.int64, device=dev)
        lib.gtk_exchange_set_trace(ctypes.c_void_p(trace.data_ptr()))
    state = opt.make_state(torch.zeros(m, device=dev), lr=0.01)
    pipe = GTopKPipeline(ep, state, k, dgrads)
    pipe.capture()
    # mid-training residual: gTop-k's residual builds up over ~1/rho steps
    # before its magnitudes settle; precondition it (untimed) so the timed
    # steps see the steady state a long training run spends its time in
    pipe.run(args.precondition)
    torch.cuda.synchronize(dev)
    pipe.status.zero_()  # (misses while the residual built up are informational)
    sampler = ClockSampler(dev.index) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    pipe.run(args.warmup)
    barrier()
    t_clk0 = time.monotonic()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lib.gtk_launch_count()
    ev0.record()
    pipe.run(args.steps)
    ev1.record()
    ev1.synchronize()
    elapsed = ev0.elapsed_time(ev1)
    timed_fallback = bool(int(pipe.status.item()) & 0x2)  # any dense-fallback select in the timed steps
    dbg = bool(os.environ.get("GTK_PROF_DEBUG"))
    if dbg:
        print(f"[rank {rank}] after timed loop: status=0x{int(pipe.status.item()):x}", flush=True)
    # keep the GPU busy until the clock sampler has seen it under load: ~0.5 s
    # of pipeline steps -- the SAME number on every rank (each step is a
    # collective; a wall-clock loop let ranks run different counts, and the
    # extra steps' exchanges then waited out their peers' timeouts)
    n_soak = max(1, int(math.ceil(500.0 / max(elapsed / args.steps * 20, 1e-3))))
    n_soak = int(max_over_ranks(n_soak))
    for _ in range(n_soak):
        pipe.run(20)
        torch.cuda.synchronize(dev)
    t_clk1 = time.monotonic()
    barrier()
    pipe.check()
    pipe.sync_state()
    if trace is not None:
        t = trace.cpu().numpy().astype(np.int64)
        ns = pipe.plan.nsteps
        stamps = [("start", t[0])] + [(f"s{j}.{w}", t[2 + 4 * j + i]) for j in range(ns)
                                      for i, w in enumerate(("push", "flag", "merge", "bar"))] + [("end", t[1])]
        stamps += [(f"s{j}.copied", t[96 + j]) for j in range(min(ns, 4))]
        stamps += [(f"s{j}.released", t[100 + j]) for j in range(min(ns, 4))]
        mnames = ["path", "slots", "hist_bar", "engine_end", "bin", "gather_bar", "ranked", "written"]
        for j in range(min(ns, 2)):
            mt = t[32 + 16 * j:32 + 16 * j + 9]
            if mt[0]:
                stamps += [(f"s{j}.m.{n}", v) for n, v in zip(mnames, mt[1:]) if v]
                b = 32 + 16 * j
                print(f"[rank {rank}] merge step {j} window lo={t[b + 14]} shift={t[b + 15]} rec0={t[b + 10]} "
                      f"tau={t[b + 11]} tau2={t[b + 12]} -> next lo={t[b + 13]}; round-0 in_bin={t[b + 9]}",
                      flush=True)
        base = t[0]
        print(f"[rank {rank}] exchange trace (us from start): " +
              " ".join(f"{n}={(v - base) / 1e3:.1f}" for n, v in stamps if v), flush=True)
        lib.gtk_exchange_set_trace(None)
    ms_step = max_over_ranks(elapsed / args.steps)
    gpu_launches = pipe.kernels_per_step * args.steps

    # ---- stage breakdown + roofline: CUDA event nodes inside a step graph ----
    if dbg:
        print(f"[rank {rank}] after soak ({pipe.t} steps): status=0x{int(pipe.status.item()):x}", flush=True)
    stage = pipe.profile(steps=max(10, min(args.steps, 30)))
    pipe.sync_state()
    if dbg:
        print(f"[rank {rank}] after profile: status=0x{int(pipe.status.item()):x}", flush=True)
    pipe.check()
    # the roofline kernel alone: back-to-back launches of K1's HBM pass on the
    # steady-state residual and window, CUDA events on its stream
    main_ms = max_over_ranks(pipe.time_main_pass(reps=20))
    hbm_peak, peak_kind = peaks()
    algo_bytes = 12 * m
    achieved = algo_bytes / (main_ms * 1e-3) / 1e9
    traffic = ncu_traffic()

    # ---- e2e: public API with pinned host gradients --------------------------
    pinned = [torch.from_numpy(g).pin_memory() for g in host_grads]
    st2 = state  # the same (steady-state) training state, continued through the public API
    for i in range(max(2, args.warmup)):
        opt.gtopk_step(st2, ep, pinned[i % 2], k, P)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_fallbacks = 0
    e0.record()
    for i in range(args.steps):
        rep = opt.gtopk_step(st2, ep, pinned[i % 2], k, P)
        e2e_fallbacks += bool(st2._bufs.get("last_status", 0) & 0x2)  # (host int: no device work)
        if os.environ.get("GTK_E2E_DEBUG") and i < 8:
            print(f"e2e step {i}: status 0x{st2._bufs.get('last_status', 0):x} "
                  f"window {st2._window.cpu().numpy().tolist()}", file=sys.stderr, flush=True)
    e1.record()
    e1.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    assert rep.selected_k == k

    clocks = sampler.stop(t_clk0, t_clk1) if sampler else None

    # ---- CPU baseline (rank 0, N = 1 only) -----------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cms, sample = oracle_steps(m, rho, 1, 3, 0)  # ~11 s of CPU work
        cpu = {"value": round(cms, 3), "unit": "ms", "cores": 1, "kind": "port", "sample": sample}

    if rank == 0:
        exch = "none (P=1)" if P == 1 else pipe.plan.mode
        line = {
            "metric": METRIC,
            "value": round(ms_step, 4),
            "unit": "ms",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4),
            "higher_is_better": False,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": DATA,
            "config": workload_config(m, rho, P),
            "run": {
                "exchange": exch,
                "step": "K1 select + gTopKAllReduce + K3 update, CUDA-graph replay",
                "select_mode": pipe.mode + (" (the next step's HBM pass overlaps this step's finish"
                                            + (" and exchange" if P > 1 else "") + ")"
                                            if pipe.mode == "defer" else ""),
                "l2": "inputs larger than L2: 307 MB streamed by K1 per step vs 126 MB L2",
                "residual": f"steady state: {args.precondition} untimed preconditioning steps before warmup",
                "dense_fallback_in_timed_steps": timed_fallback,
            },
            "roofline": {"bound": "hbm", "kernel": "select_main_kernel (K1 HBM pass)",
                         "achieved": round(achieved, 1), "peak": hbm_peak, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                         "algorithmic_bytes_per_launch": algo_bytes, "launch_ms": round(main_ms, 5),
                         "timing": "CUDA events around 20 back-to-back launches of the main pass "
                                   "(steady-state residual and window), max over ranks"},
            "stages_ms": {k_: (round(v, 5) if v is not None else None) for k_, v in stage.items()},
            "exchange_rounds": None if P == 1 else {
                "rounds": pipe.plan.nsteps,
                "us_per_round": (round(stage["exchange"] * 1e3 / pipe.plan.nsteps, 2)
                                 if stage.get("exchange") else None),
                # k LL records of 16 B (idx|tag, value|tag) per round over 900 GB/s NVLink 5
                "nvlink_floor_us_per_round": round(16 * k / 900e3, 3),
                "note": "per round: LL records pushed by the partner + merge (+ K3 after the last round); latency-bound"},
            "e2e": {"value": round(e2e_ms, 4), "unit": "ms", "h2d_bytes_per_step": 4 * m,
                    "d2h_bytes_per_step": 8, "dense_fallback_steps": e2e_fallbacks},
            "gpu_launches": gpu_launches,
            "kernels_per_step": pipe.kernels_per_step,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        ep.close()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--m", "--numel", dest="m", type=int, default=M_DEFAULT,
                    help="gradient length (use --numel under torchrun: --m is ambiguous there)")
    ap.add_argument("--rho", type=float, default=RHO_DEFAULT)
    ap.add_argument("--mode", choices=["auto", "butterfly", "tree"], default="auto")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline")
    ap.add_argument("--precondition", type=int, default=1500,
                    help="untimed steps that build the residual up to its steady state")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if os.environ.get("GTK_HANG_DUMP"):  # diagnostics: every thread's Python stack after N s, to stderr
        import faulthandler

        faulthandler.dump_traceback_later(float(os.environ["GTK_HANG_DUMP"]), exit=False)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_b200(args, rank, world)


if __name__ == "__main__":
    sys.exit(main())
