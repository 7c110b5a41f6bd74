"""Merge-kernel timing/profiling aid at several k."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_04359_b200.device as dev
d = torch.device("cuda", 0)
ks = [int(x) for x in sys.argv[1:]] or [270, 1000, 14700, 25600, 66000, 660000]
st = torch.zeros(1, dtype=torch.int32, device=d)
for k in ks:
    m = max(1000 * k, 4 * k)
    m = min(m, 66_000_000)
    g = torch.randn(m, device=d); r = torch.randn(m, device=d); out = torch.empty_like(g)
    a = dev.DeviceList(m, k, d); b = dev.DeviceList(m, k, d); o = dev.DeviceList(m, k, d)
    dev.select(None, g, out, k, a, st); dev.select(None, r, out, k, b, st)
    for _ in range(3): dev.top_op(a, b, k, o)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): dev.top_op(a, b, k, o)
    e.record(); e.synchronize()
    print(f"merge k={k}: {s.elapsed_time(e)/20*1e3:.1f} us", flush=True)
    del g, r, out
