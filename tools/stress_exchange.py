"""Long-run consistency check of the fused exchange (LL records, fused pushes):
python -m torch.distributed.run --nproc-per-node N tools/stress_exchange.py [steps] [mode]
Runs the CUDA-graph pipeline for `steps` steps; every rank applies the same
global update, so the weights must stay bit-identical across ranks, and the
sticky status must stay clean (no timeout, no peer failure)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
from paper_1901_04359_b200 import optimizer as opt
from paper_1901_04359_b200.dist import init_dist_cluster
from paper_1901_04359_b200.pipeline import GTopKPipeline

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
mode = sys.argv[2] if len(sys.argv) > 2 else "auto"
ep = init_dist_cluster(timeout=30.0, mode=mode)
r, P = ep.rank, ep.world_size
dev = ep.group.device
m, k = 2_560_000, 2560
rng = np.random.default_rng(1000 + r)
grads = [torch.from_numpy(rng.standard_normal(m).astype(np.float32)).to(dev) for _ in range(2)]
st = opt.make_state(torch.zeros(m, device=dev), lr=0.01)
pipe = GTopKPipeline(ep, st, k, grads)
pipe.capture()
done = 0
while done < steps:
    n = min(2000, steps - done)
    pipe.run(n)
    done += n
torch.cuda.synchronize(dev)
word = int(pipe.status.item())
pipe.sync_state()
h = hashlib.sha256(st.weights.cpu().numpy().tobytes()).hexdigest()[:16]
hs = [None] * P
dist.all_gather_object(hs, (h, word))
if r == 0:
    same = len({x[0] for x in hs}) == 1
    clean = all((w & 0x1D) == 0 for _, w in hs)
    print(f"STRESS mode={mode} P={P} steps={steps} weights identical across ranks: {same}; "
          f"status clean: {clean}; {hs}", flush=True)
dist.barrier()
ep.close()
dist.destroy_process_group()
