"""Stage times of the steady-state pipeline by both profilers (eager events vs
graph event nodes) -- which one measures the main pass as ncu does?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_04359_b200 as gk
from paper_1901_04359_b200 import optimizer as opt
from paper_1901_04359_b200.pipeline import GTopKPipeline
d = torch.device("cuda", 0)
m, k = 25_600_000, 25_600
gen = torch.Generator(device=d).manual_seed(5)
grads = [torch.randn(m, device=d, generator=gen) for _ in range(2)]
ep = gk.create_local_cluster(1)[0]
st = opt.make_state(torch.zeros(m, device=d), lr=0.01)
pipe = GTopKPipeline(ep, st, k, grads)
pipe.capture()
pipe.run(1500)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); pipe.run(200); e.record(); e.synchronize()
print("graph step:", s.elapsed_time(e) / 200 * 1e3, "us")
print("eager profile:", {k_: (round(v * 1e3, 2) if v else None) for k_, v in pipe.profile(30).items()})
print("graph profile:", {k_: (round(v * 1e3, 2) if v else None) for k_, v in pipe.profile_graph(30).items()})
print("eager profile:", {k_: (round(v * 1e3, 2) if v else None) for k_, v in pipe.profile(30).items()})
