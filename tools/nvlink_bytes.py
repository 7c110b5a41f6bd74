"""NVLink bytes per pipeline step, from the driver's own counters (NVML
field values NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX, KiB, summed over
the links) read around `steps` graph-replayed steps on every rank -- the
exchange's wire bytes against the LL-record floor 16 B x (k + 1) per round.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29600 tools/nvlink_bytes.py [m] [k] [steps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1901_04359_b200 import optimizer as opt  # noqa: E402
from paper_1901_04359_b200.dist import init_dist_cluster  # noqa: E402
from paper_1901_04359_b200.pipeline import GTopKPipeline  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 25_600
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
ep = init_dist_cluster(timeout=60.0)
dev = ep.group.device
rank, P = ep.rank, ep.world_size
gen = torch.Generator(device=dev).manual_seed(11 + rank)
grads = [torch.randn(m, device=dev, generator=gen) for _ in range(2)]
st = opt.make_state(torch.zeros(m, device=dev), lr=0.01)
pipe = GTopKPipeline(ep, st, k, grads)
pipe.capture()
pipe.run(400)
torch.cuda.synchronize(dev)
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
nlinks = 18


def counters():
    ids = [(pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, l) for l in range(nlinks)]
    ids += [(pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, l) for l in range(nlinks)]
    vals = pynvml.nvmlDeviceGetFieldValues(h, ids)
    tx = rx = 0
    for i, v in enumerate(vals):
        if v.nvmlReturn != 0:
            continue
        x = v.value.ullVal
        if i < nlinks:
            tx += x
        else:
            rx += x
    return tx, rx


dist.barrier()
tx0, rx0 = counters()
pipe.run(steps)
torch.cuda.synchronize(dev)
tx1, rx1 = counters()
dist.barrier()
pipe.check()
rounds = pipe.plan.nsteps
rec = {"rank": rank, "P": P, "m": m, "k": k, "steps": steps, "rounds": rounds,
       "tx_bytes_per_step": round((tx1 - tx0) * 1024 / steps), "rx_bytes_per_step": round((rx1 - rx0) * 1024 / steps),
       "ll_floor_bytes_per_step": 16 * (k + 1) * rounds,
       "note": "NVML NVLINK_THROUGHPUT_DATA counters (KiB) summed over links; LL records: 16 B per entry + header"}
allr = [None] * P
dist.all_gather_object(allr, rec)
if rank == 0:
    for r in allr:
        print(json.dumps(r), flush=True)
ep.close()
dist.destroy_process_group()
