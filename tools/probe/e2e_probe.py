"""Where the public-API e2e step (pinned host gradient) spends its time."""
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
host = [rng.standard_normal(m).astype(np.float32) for _ in range(2)]
pinned = [torch.from_numpy(g).pin_memory() for g in host]
dev_g = [p.to(d) for p in pinned]
ep = gk.create_local_cluster(1)[0]
st = opt.make_state(torch.zeros(m, device=d), lr=0.01)
for i in range(200):
    opt.gtopk_step(st, ep, dev_g[i % 2], k, 1)
torch.cuda.synchronize()


def ev_time(fn, n=30):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for i in range(n):
        fn(i)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / n, (time.perf_counter() - t0) / n * 1e3


buf = torch.empty(m, device=d)
print("h2d copy_ into a fixed buffer: %.3f ms (wall %.3f)" % ev_time(lambda i: buf.copy_(pinned[i % 2], non_blocking=True)))
print("h2d .to(device): %.3f ms (wall %.3f)" % ev_time(lambda i: pinned[i % 2].to(d, non_blocking=True)))
print("gtopk_step device grads: %.3f ms (wall %.3f)" % ev_time(lambda i: opt.gtopk_step(st, ep, dev_g[i % 2], k, 1)))
print("gtopk_step pinned grads: %.3f ms (wall %.3f)" % ev_time(lambda i: opt.gtopk_step(st, ep, pinned[i % 2], k, 1)))
t0 = time.perf_counter()
for i in range(30):
    pinned[i % 2].is_pinned()
print("is_pinned: %.1f us" % ((time.perf_counter() - t0) / 30 * 1e6))

# the same with bench.py's nvidia-smi clock sampler running beside it
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402

smp = bench.ClockSampler(0)
smp.start()
time.sleep(0.5)
print("gtopk_step pinned grads, sampler on: %.3f ms (wall %.3f)" % ev_time(lambda i: opt.gtopk_step(st, ep, pinned[i % 2], k, 1)))
print("h2d copy_, sampler on: %.3f ms (wall %.3f)" % ev_time(lambda i: buf.copy_(pinned[i % 2], non_blocking=True)))
print("gtopk_step device grads, sampler on: %.3f ms (wall %.3f)" % ev_time(lambda i: opt.gtopk_step(st, ep, dev_g[i % 2], k, 1)))
smp.stop(0, 1e18)
