"""Ad-hoc CUDA-event timing of the kernels (development aid, not the bench)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1901_04359_b200.device as dev

d = torch.device("cuda", 0)
def timeit(fn, n=20, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(n):
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    return float(np.median(ts)), float(np.min(ts))

for m, k in ((270_000, 270), (1_000_000, 1000), (14_700_000, 14700), (25_600_000, 25600), (66_000_000, 66000), (66_000_000, 660000)):
    g = torch.randn(m, device=d); r = 0.1 * torch.randn(m, device=d); out = torch.empty_like(g)
    lst = dev.DeviceList(m, k, d); st = torch.zeros(1, dtype=torch.int32, device=d)
    flush = torch.empty(256 * 1024 * 1024 // 4, device=d)
    def f():
        dev.select(r, g, out, k, lst, st)
    med, mn = timeit(f)
    gbs = 12 * m / (med * 1e-3) / 1e9
    print(f"select m={m} k={k}: median {med*1e3:.1f} us min {mn*1e3:.1f} us  -> {gbs:.0f} GB/s (12m bytes) status={int(st.item())}", flush=True)
    # merge of two k-lists
    a = dev.DeviceList(m, k, d); b = dev.DeviceList(m, k, d); o = dev.DeviceList(m, k, d)
    dev.select(None, g, out, k, a, st); dev.select(None, r, out, k, b, st)
    med, mn = timeit(lambda: dev.top_op(a, b, k, o))
    print(f"  merge k={k}: median {med*1e3:.1f} us min {mn*1e3:.1f} us nnz={o.nnz()}", flush=True)
    del g, r, out, flush
    torch.cuda.empty_cache()
