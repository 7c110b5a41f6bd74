"""Timeline (%globaltimer, block 0 / last block) of consecutive pipeline
steps enqueued back to back -- each step's kernels stamp into their own trace
buffer -- to see how the next step's main pass overlaps this step's finish
(GTK_PIPE_MODE=defer) or follows it (chain / plain)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1901_04359_b200 as gk  # noqa: E402
from paper_1901_04359_b200 import _lib  # noqa: E402
from paper_1901_04359_b200 import optimizer as opt  # noqa: E402
from paper_1901_04359_b200.pipeline import GTopKPipeline  # noqa: E402

lib = _lib.load()
if int(os.environ.get("WORLD_SIZE", "1")) > 1:  # torchrun: one process per GPU, the real exchange
    from paper_1901_04359_b200.dist import init_dist_cluster

    ep = init_dist_cluster(timeout=60.0)
    d = ep.group.device
else:
    ep = gk.create_local_cluster(1)[0]
    d = torch.device("cuda", 0)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 25_600
npre = int(sys.argv[3]) if len(sys.argv) > 3 else 400
nst = 4
gen = torch.Generator(device=d).manual_seed(5)
grads = [torch.randn(m, device=d, generator=gen) for _ in range(2)]
st = opt.make_state(torch.zeros(m, device=d), lr=0.01)
pipe = GTopKPipeline(ep, st, k, grads)
pipe.capture()
pipe.run(npre)
torch.cuda.synchronize()
trs = [torch.zeros(256, dtype=torch.int64, device=d) for _ in range(nst)]
torch.cuda._sleep(int(2e7))  # the steps below queue behind a spin: no host gaps
for i in range(nst):
    lib.gtk_exchange_set_trace(ctypes.c_void_p(trs[i].data_ptr()))
    pipe.step_eager()
lib.gtk_exchange_set_trace(None)
torch.cuda.synchronize()
T = [t.cpu().tolist() for t in trs]
base = T[0][112]
us = lambda v: round((v - base) / 1e3, 1) if v else None  # noqa: E731
lines = [f"[rank {ep.rank}] mode={pipe.mode} m={m} k={k} P={ep.world_size}"]
for i, t in enumerate(T):
    ex = f" | exchange {us(t[0])} .. {us(t[1])}" if ep.world_size > 1 else ""
    lines.append(f"[rank {ep.rank}] step {i}: main {us(t[112])} .. {us(t[113])} | finish {us(t[48])} "
                 f"fixup_done {us(t[68])} scanned {us(t[49])} copied {us(t[50])} bin {us(t[51])} "
                 f"gather_bar {us(t[52])} ranked {us(t[53])} written {us(t[54])} last_end {us(t[114])}{ex} "
                 f"| n_fix={t[62]} n_ins={t[63]}")
print("\n".join(lines), flush=True)
