"""Chunked public step: where the time goes (copy events vs compute events)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1901_04359_b200 as gk  # noqa: E402
from paper_1901_04359_b200 import optimizer as opt  # noqa: E402

m, k = 25_600_000, 25_600
d = torch.device("cuda", 0)
rng = np.random.default_rng(0)
host = [torch.from_numpy(rng.standard_normal(m).astype(np.float32)).pin_memory() for _ in range(2)]
print("pinned:", host[0].is_pinned(), host[0][5:100].is_pinned())
dev_g = [h.to(d) for h in host]
ep = gk.create_local_cluster(1)[0]
st = opt.make_state(torch.zeros(m, device=d), lr=0.01)
for i in range(100):
    opt.gtopk_step(st, ep, dev_g[i % 2], k, 1)
for i in range(5):
    opt.gtopk_step(st, ep, host[i % 2], k, 1)
torch.cuda.synchronize()
print("chunked path used:", "gbuf" in st._bufs, "window cold:", st._bufs.get("window_cold"))
cur = torch.cuda.current_stream()
for trial in range(3):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    t0 = time.perf_counter()
    opt.gtopk_step(st, ep, host[trial % 2], k, 1)
    t1 = time.perf_counter()
    e1.record(cur)
    e1.synchronize()
    print(f"step: events {e0.elapsed_time(e1):.3f} ms, host {1e3 * (t1 - t0):.3f} ms")
# copy stream timing: chunk events are not timing events; time the copies alone
cs = st._bufs["copy_stream"]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
ev[0].record(cs)
with torch.cuda.stream(cs):
    per = 6_400_000
    for c in range(4):
        st._bufs["gbuf"][c * per:(c + 1) * per].copy_(host[0][c * per:(c + 1) * per], non_blocking=True)
        ev[c + 1].record(cs)
t0 = time.perf_counter()
ev[4].synchronize()
print("host returned after enqueue in %.3f ms" % ((time.perf_counter() - t0) * 1e3))
print("chunk arrivals (ms):", [round(ev[0].elapsed_time(e), 3) for e in ev[1:]])
