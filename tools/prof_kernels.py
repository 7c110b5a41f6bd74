"""Per-kernel timing aid: back-to-back submission (host gaps hidden) and CUDA
graph replay.  Usage: python tools/prof_kernels.py [m] [k] [iters]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1901_04359_b200.device as dev

m = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 25_600
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
d = torch.device("cuda", 0)
g = torch.randn(m, device=d); r = 0.1 * torch.randn(m, device=d); out = torch.empty_like(g)
lst = dev.DeviceList(m, k, d); st = torch.zeros(1, dtype=torch.int32, device=d)
a = dev.DeviceList(m, k, d); b = dev.DeviceList(m, k, d); o = dev.DeviceList(m, k, d)
dev.select(None, g, out, k, a, st); dev.select(None, r, out, k, b, st)

def batch(fn, n):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / n * 1e3

sel_us = batch(lambda: dev.select(r, g, out, k, lst, st), iters)
print(f"select m={m} k={k}: {sel_us:.1f} us/call back-to-back -> {12*m/sel_us/1e3:.0f} GB/s", flush=True)
mrg_us = batch(lambda: dev.top_op(a, b, k, o), iters)
print(f"merge k={k}: {mrg_us:.1f} us/call back-to-back", flush=True)
try:
    gr = torch.cuda.CUDAGraph()
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        dev.select(r, g, out, k, lst, st)
        dev.top_op(a, b, k, o)
    torch.cuda.synchronize()
    with torch.cuda.graph(gr, stream=s2):
        dev.select(r, g, out, k, lst, st)
        dev.top_op(a, b, k, o)
    gr.replay(); torch.cuda.synchronize()
    us = batch(gr.replay, iters)
    print(f"graph(select+merge): {us:.1f} us/replay", flush=True)
except Exception as exc:
    print("graph capture failed:", repr(exc), flush=True)
print("status", int(st.item()), "nnz", lst.nnz(), o.nnz())
