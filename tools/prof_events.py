"""Check CUDA-event stage timing (eager hooks and graph event nodes) against
whole-step timing, to validate bench.py's roofline measurement."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_04359_b200 as gk
import paper_1901_04359_b200.device as dev
from paper_1901_04359_b200 import _lib, optimizer as opt
from paper_1901_04359_b200.pipeline import GTopKPipeline
lib = _lib.load()
d = torch.device("cuda", 0)
m, k = 25_600_000, 25_600
g = torch.randn(m, device=d); r = 0.1 * torch.randn(m, device=d); out = torch.empty_like(g)
lst = dev.DeviceList(m, k, d); st = torch.zeros(1, dtype=torch.int32, device=d)
for _ in range(3): dev.select(r, g, out, k, lst, st)
torch.cuda.synchronize()
# eager, back-to-back selects with hooks
lib.gtk_prof_reset(); lib.gtk_prof_enable(1)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): dev.select(r, g, out, k, lst, st)
e.record(); e.synchronize(); lib.gtk_prof_enable(0)
print("eager select loop total/call us", s.elapsed_time(e) / 20 * 1e3)
for pid, name in ((0, "main"), (1, "select")):
    ms, n = _lib.prof_read(pid); print(f"  eager {name}: {ms / max(n,1) * 1e3:.1f} us over {n}")
lib.gtk_prof_reset()
# graph with event nodes
ep = gk.create_local_cluster(1)[0]
state = opt.make_state(torch.zeros(m, device=d), lr=0.01)
pipe = GTopKPipeline(ep, state, k, [g, r])
pipe.capture()
s.record(); pipe.run(20); e.record(); e.synchronize()
print("graph step us", s.elapsed_time(e) / 20 * 1e3)
lib.gtk_prof_enable(1)
stream = torch.cuda.Stream(d)
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=stream):
    pipe._enqueue(0)
lib.gtk_prof_enable(0)
for i in range(6):
    s.record(stream); gr.replay(); e.record(stream); torch.cuda.synchronize()
    vals = {name: _lib.prof_graph_read(pid) for pid, name in ((0, "main"), (1, "select"), (4, "update"))}
    print(f"replay {i}: total {s.elapsed_time(e)*1e3:.1f} us  " + "  ".join(f"{n}={ms*1e3:.1f}us/{c}" for n, (ms, c) in vals.items()))
