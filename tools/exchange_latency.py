"""Latency of one rank's fused exchange kernel (gtk_gtopk_exchange_update)
on ONE GPU, partners emulated by a pre-filled inbox (the loopback harness of
tests/test_gpu_exchange_loopback.py): the merge rounds + fused K3 without the
partner's skew.  Prints one JSON line per (P, mode, k) with the CUDA-event
median per call and the %globaltimer phase stamps of block 0.

    python tools/exchange_latency.py [--k 270 25600] [--P 2 4 8] [--calls 30]

GTK_MERGE_GRID / GTK_MERGE_CLUSTER select the merge grid (csrc/gtk_merge.cu).
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import test_gpu_exchange_loopback as lbt  # noqa: E402


def run(P, mode, k, calls, rank=0, deferred=False, thrash_mb=0):
    rng = np.random.default_rng(11 + k)
    m = max(1_000_000, 20 * k)
    lists = lbt._lists(rng, P, m, k, "normal")
    scheds = lbt.schedules_for(P, mode)
    lb = lbt.Loopback(rank, P, scheds[rank], k, m)
    _sent, recv, _final = lbt.simulate(lists, k, scheds)
    d = lb.d
    w = torch.randn(m, device=d)
    res = torch.zeros(m, device=d)
    local = lb.dv.DeviceList.from_host(m, lists[rank][0], lists[rank][1], d, k)
    local.count[1] = lbt.hint_of(lists[rank][0], lists[rank][1], k)
    # every call's inbox words, built once (tag = call number)
    words = {}
    tr = torch.zeros(256, dtype=torch.int64, device=d)
    thrash = torch.zeros(thrash_mb * 262144, device=d) if thrash_mb else None
    times = []
    trace = None
    for call in range(calls):
        tag = call + 1
        for s, got in enumerate(recv[rank]):
            if got is not None:
                key = (s, tag & 1)
                if key not in words:
                    words[key] = lbt.encode_slot(k, 0, *got)
                wv = (words[key] & np.uint64(0xFFFFFFFF)) | (np.uint64(tag) << np.uint64(32))
                lb.prefill(s, tag, wv)
        lb.status.zero_()
        last = call == calls - 1
        if last:
            tr.zero_()
            lb.lib.gtk_exchange_set_trace(ctypes.c_void_p(tr.data_ptr()))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        P_ = lb.dv.P
        args = [lb.rank, lb.P, lb.sched, lb.nsteps, lb.peer, P_(lb.epoch), P_(lb.acc.idx), P_(lb.acc.val),
                P_(lb.acc.count), k, P_(lb.status), None, ctypes.c_int64(int(5e9)), P_(lb.counts),
                P_(local.idx), P_(local.val), P_(local.count), P_(lb.ws), ctypes.c_size_t(lb.ws.numel())]
        st = lb.dv.stream_of(d)  # torch's current stream: the events below see the kernel
        # the GPU is kept busy (SM clocks up) and the start event lands after the
        # spin, with the exchange launch already queued behind it
        if thrash is not None:
            thrash.add_(1.0)  # stream a buffer larger than L2 through it (evicts the kernel's code lines)
        torch.cuda._sleep(400_000)
        e0.record()
        rc = lb.lib.gtk_gtopk_exchange_update(*args, P_(w), P_(None if deferred else res), ctypes.c_float(0.01), 0,
                                              P_(lb.tags), st)
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0, rc
        assert int(lb.status.item()) == 0, hex(int(lb.status.item()))
        if call >= 3:
            times.append(e0.elapsed_time(e1) * 1e3)
        if last:
            lb.lib.gtk_exchange_set_trace(None)
            trace = tr.cpu().tolist()
    # the final global list matches the oracle's fold
    from oracle import gtopk_oracle as orc
    want_i, _ = orc.tree_fold(lists, k)
    ai, _ = lb.acc.to_host()
    assert np.array_equal(ai, want_i)
    t0 = trace[0]
    us = lambda v: round((v - t0) / 1e3, 2) if v else None  # noqa: E731
    phases = {"end": us(trace[1])}
    if trace[121] and trace[1] > t0:  # SM clock of block 0's SM over the call
        phases["sm_mhz"] = round((trace[121] - trace[120]) / ((trace[1] - t0) / 1e3), 1)
    for s in range(lb.nsteps):
        phases[f"s{s}"] = {"hdr": us(trace[3 + 4 * s]), "merge": us(trace[4 + 4 * s]), "bar": us(trace[5 + 4 * s])}
        mb = 32 + 16 * s
        names = ["m.start", "m.path", "m.slots", "m.hist_bar", "m.engine_end", "bin", "gather_bar", "ranked",
                 "written"]
        if os.environ.get("GTK_MERGE_SOLO", "1") != "0" and k <= 2048 and os.environ.get("GTK_MERGE_GRID", "1") == "1":
            # one-CTA merge_solo stamps: start, loaded, union, selected, written,
            # bin found, gathered, ranked; diagnostics [10..12] = bin, in_bin, above
            names = ["m.start", "m.loaded", "m.union", "m.selected", "m.written", "s.bin", "s.gathered", "s.ranked"]
            phases[f"s{s}"]["diag"] = trace[mb + 10:mb + 13]
        phases[f"s{s}"].update({n: us(trace[mb + i]) for i, n in enumerate(names) if trace[mb + i]})
        if os.environ.get("GTK_TRACE_FINE"):  # a GTK_MERGE_TRACE_FINE build: staged / union 0 / union last
            phases[f"s{s}"].update({n: us(trace[mb + 10 + i]) for i, n in enumerate(["f.staged0", "f.union0",
                                                                                      "f.union_last"])})
        if s < 4 and trace[104 + 2 * s]:  # histogram-barrier arrivals: the latest block, block 0
            phases[f"s{s}"]["arr.last"] = us(trace[104 + 2 * s])
            phases[f"s{s}"]["arr.blk0"] = us(trace[105 + 2 * s])
    return {"P": P, "mode": mode, "k": k, "us_median": round(statistics.median(times), 2),
            "us_min": round(min(times), 2), "grid": os.environ.get("GTK_MERGE_GRID", "auto"),
            "cluster": os.environ.get("GTK_MERGE_CLUSTER", "auto"), "phases": phases}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, nargs="+", default=[270, 25600])
    ap.add_argument("--P", type=int, nargs="+", default=[2, 4])
    ap.add_argument("--calls", type=int, default=30)
    ap.add_argument("--thrash-mb", type=int, default=0, help="stream this many MB through L2 before each call")
    ap.add_argument("--deferred", action="store_true", help="res = NULL: the deferred step's exchange (compact grid)")
    a = ap.parse_args()
    for P in a.P:
        for k in a.k:
            r = run(P, "butterfly", k, a.calls, deferred=a.deferred, thrash_mb=a.thrash_mb)
            r["deferred"] = a.deferred
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
