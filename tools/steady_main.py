"""Steady-state pipeline then a few eager steps: the ncu target for profiling
the main pass in its real L2 state (ncu -k regex:select_main -s <n> -c 1)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_04359_b200 as gk
from paper_1901_04359_b200 import optimizer as opt
from paper_1901_04359_b200.pipeline import GTopKPipeline
d = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
m = int(sys.argv[2]) if len(sys.argv) > 2 else 25_600_000
k = int(sys.argv[3]) if len(sys.argv) > 3 else 25_600
gen = torch.Generator(device=d).manual_seed(5)
grads = [torch.randn(m, device=d, generator=gen) for _ in range(2)]
ep = gk.create_local_cluster(1)[0]
st = opt.make_state(torch.zeros(m, device=d), lr=0.01)
pipe = GTopKPipeline(ep, st, k, grads, use_graph=False)
for _ in range(n):
    pipe.step_eager()
torch.cuda.synchronize()
for _ in range(4):
    pipe.step_eager()
torch.cuda.synchronize()
print("status", int(pipe.status.item()))
