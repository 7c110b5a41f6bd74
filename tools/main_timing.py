"""Steady-state K1 main-pass timing (gtk_select_main_pass), development aid:
python tools/main_timing.py [m] [k] [precondition]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_04359_b200 as gk
from paper_1901_04359_b200 import optimizer as opt
from paper_1901_04359_b200.pipeline import GTopKPipeline
d = torch.device("cuda", 0)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 25_600
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1500
gen = torch.Generator(device=d).manual_seed(5)
grads = [torch.randn(m, device=d, generator=gen) for _ in range(2)]
ep = gk.create_local_cluster(1)[0]
st = opt.make_state(torch.zeros(m, device=d), lr=0.01)
pipe = GTopKPipeline(ep, st, k, grads)
pipe.capture()
pipe.run(n)
ts = [pipe.time_main_pass(20) for _ in range(5)]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
pipe.run(10); e0.record(); pipe.run(100); e1.record(); e1.synchronize()
print(f"m={m} k={k}: main pass {min(ts)*1e3:.2f} us (min of 5) {sorted(ts)[2]*1e3:.2f} (median) -> "
      f"{12*m/min(ts)/1e6:.0f} GB/s; step {e0.elapsed_time(e1)*10:.2f} us", flush=True)
