"""H2D bandwidth of a 102.4 MB pinned gradient: one copy vs chunks on several streams."""
import time

import torch

n = 25_600_000
h = torch.empty(n, dtype=torch.float32).pin_memory()
h.normal_()
d = torch.empty(n, device="cuda")
main = torch.cuda.current_stream()


def one():
    d.copy_(h, non_blocking=True)


streams = [torch.cuda.Stream() for _ in range(8)]


def multi(ns, chunks):
    ev0 = torch.cuda.Event()
    ev0.record(main)
    per = (n + chunks - 1) // chunks
    evs = []
    for c in range(chunks):
        s = streams[c % ns]
        s.wait_event(ev0)
        with torch.cuda.stream(s):
            d[c * per:(c + 1) * per].copy_(h[c * per:(c + 1) * per], non_blocking=True)
            e = torch.cuda.Event()
            e.record(s)
            evs.append(e)
    for e in evs:
        main.wait_event(e)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


ms = timeit(one)
print(f"single copy: {ms:.3f} ms  {n * 4 / ms / 1e6:.1f} GB/s")
for ns, ch in ((1, 4), (2, 2), (2, 4), (2, 8), (4, 4), (4, 8), (8, 8), (8, 16)):
    ms = timeit(lambda: multi(ns, ch))
    print(f"{ns} streams x {ch} chunks: {ms:.3f} ms  {n * 4 / ms / 1e6:.1f} GB/s")
