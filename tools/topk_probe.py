"""TopK-AllReduce baseline cost breakdown under torchrun (device lists):
    python -m torch.distributed.run --nproc-per-node 2 ... tools/topk_probe.py [m] [k]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1901_04359_b200 import collectives as coll  # noqa: E402
from paper_1901_04359_b200 import device as dv  # noqa: E402
from paper_1901_04359_b200 import optimizer as opt  # noqa: E402
from paper_1901_04359_b200.dist import init_dist_cluster  # noqa: E402
from paper_1901_04359_b200.sparse import DeviceSparseVector  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 14_700_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 14_700
ep = init_dist_cluster(timeout=60.0)
d = ep.group.device
g = torch.randn(m, device=d)
lst = dv.DeviceList(m, k, d)
st = torch.zeros(1, dtype=torch.int32, device=d)
out = torch.empty(m, device=d)
dv.select(None, g, out, k, lst, st)
sv = DeviceSparseVector(lst)


def timed(fn, n=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


res = {}
res["topk_allreduce"] = timed(lambda: coll.topk_allreduce(ep, sv, ep.world_size))
cnts = torch.empty(ep.world_size, dtype=torch.int32, device=d)
res["count_allgather+item"] = timed(lambda: (dist.all_gather_into_tensor(cnts, lst.n), int(cnts.max().item())))
buf = torch.zeros(ep.world_size * k, dtype=torch.int32, device=d)
res["allgather_k_int32"] = timed(lambda: dist.all_gather_into_tensor(buf, lst.idx[:k]))
res["accumulate"] = timed(lambda: dv.topk_accumulate(buf, buf.view(torch.float32), cnts, ep.world_size, k, m, out))
state = opt.make_state(torch.zeros(m, device=d), lr=0.01)
res["topk_step"] = timed(lambda: opt.topk_step(state, ep, g, k, ep.world_size), 20)
res["gtopk_step"] = timed(lambda: opt.gtopk_step(state, ep, g, k, ep.world_size), 20)
if ep.rank == 0:
    print({a: round(b, 4) for a, b in res.items()}, flush=True)
if os.environ.get("TOPK_PROFILE"):
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            opt.topk_step(state, ep, g, k, ep.world_size)
        torch.cuda.synchronize()
    if ep.rank == 0:
        print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=25), flush=True)
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12), flush=True)
ep.close()
dist.destroy_process_group()
