"""Public-API step cost at P = 1 (optimizer.gtopk_step, device gradients):
per-call time and how many calls took the exact dense fallback."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1901_04359_b200 as gk  # noqa: E402
from paper_1901_04359_b200 import optimizer as opt  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 25_600
d = torch.device("cuda", 0)
gen = torch.Generator(device=d).manual_seed(5)
grads = [torch.randn(m, device=d, generator=gen) for _ in range(2)]
ep = gk.create_local_cluster(1)[0]
st = opt.make_state(torch.zeros(m, device=d), lr=0.01)
for i in range(300):
    opt.gtopk_step(st, ep, grads[i % 2], k, 1)
torch.cuda.synchronize()
fb = 0
t0 = time.perf_counter()
n = 100
for i in range(n):
    opt.gtopk_step(st, ep, grads[i % 2], k, 1)
    fb += bool(st._bufs.get("last_status", 0) & 0x2)
torch.cuda.synchronize()
print(f"gtopk_step m={m} k={k}: {(time.perf_counter() - t0) / n * 1e3:.3f} ms per call, dense fallbacks {fb}/{n}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(n):
    opt.gtopk_step(st, ep, grads[i % 2], k, 1)
e1.record()
e1.synchronize()
print(f"  device-event span per call: {e0.elapsed_time(e1) / n:.3f} ms")

if os.environ.get("API_PROFILE"):
    import cProfile
    import pstats

    pr = cProfile.Profile()
    pr.enable()
    for i in range(200):
        opt.gtopk_step(st, ep, grads[i % 2], k, 1)
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
