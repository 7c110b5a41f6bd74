"""One rank of a 2-process gTopKAllReduce loop (k = 25.6K lists of a 25.6M
gradient), for an ncu capture of the exchange kernel's NVLink bytes on rank 0
(tools/gpu/nvl_ncu.sh launches the two ranks by hand, rank 0 under ncu with a
single-pass metric set).  Env: RANK, WORLD_SIZE, LOCAL_RANK, MASTER_ADDR/PORT."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1901_04359_b200 import collectives as coll  # noqa: E402
from paper_1901_04359_b200 import device as dv  # noqa: E402
from paper_1901_04359_b200.dist import init_dist_cluster  # noqa: E402
from paper_1901_04359_b200.sparse import DeviceSparseVector  # noqa: E402

m, k = 25_600_000, 25_600
ep = init_dist_cluster(timeout=20.0)
d = ep.group.device
gen = torch.Generator(device=d).manual_seed(3 + ep.rank)
g = torch.randn(m, device=d, generator=gen)
lst = dv.DeviceList(m, k, d)
st = torch.zeros(1, dtype=torch.int32, device=d)
out = torch.empty(m, device=d)
dv.select(None, g, out, k, lst, st)
sv = DeviceSparseVector(lst)
for i in range(6):
    res = coll.gtopk_allreduce(ep, sv, k, ep.world_size)
    torch.cuda.synchronize()
    dist.barrier()
print(f"rank {ep.rank}: {res.global_topk.nnz} entries", flush=True)
ep.close()
dist.destroy_process_group()
