"""Baseline steps at P = 1 (topk_step / dense_step / gtopk_step, device
gradients, VGG-16 size by default): per-call time and the per-kernel device
time of one call (torch.profiler), to see where a baseline step goes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1901_04359_b200 as gk  # noqa: E402
from paper_1901_04359_b200 import optimizer as opt  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 14_700_000
k = gk.k_from_density(0.001, m)
d = torch.device("cuda", 0)
gen = torch.Generator(device=d).manual_seed(5)
grads = [torch.randn(m, device=d, generator=gen) for _ in range(2)]
ep = gk.create_local_cluster(1)[0]

for name in ("gtopk_step", "topk_step", "dense_step"):
    st = opt.make_state(torch.zeros(m, device=d), lr=0.01)
    fn = getattr(opt, name)

    def call(i):
        if name == "dense_step":
            fn(st, ep, grads[i % 2], 1)
        else:
            fn(st, ep, grads[i % 2], k, 1)

    for i in range(50):
        call(i)
    torch.cuda.synchronize()
    n = 100
    t0 = time.perf_counter()
    for i in range(n):
        call(i)
    torch.cuda.synchronize()
    print(f"{name} m={m} k={k}: {(time.perf_counter() - t0) / n * 1e3:.3f} ms per call")
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for i in range(5):
            call(i)
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
