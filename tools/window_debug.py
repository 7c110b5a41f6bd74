"""Step-by-step eager pipeline: report which steps hit the dense fallback and
the carried key window (lo, shift) around them."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_04359_b200 as gk
from paper_1901_04359_b200 import optimizer as opt
from paper_1901_04359_b200.pipeline import GTopKPipeline

d = torch.device("cuda", 0)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
n = int(sys.argv[3]) if len(sys.argv) > 3 else 400
gen = torch.Generator(device=d).manual_seed(5)
grads = [torch.randn(m, device=d, generator=gen) for _ in range(2)]
ep = gk.create_local_cluster(1)[0]
st = opt.make_state(torch.zeros(m, device=d), lr=0.01)
pipe = GTopKPipeline(ep, st, k, grads, use_graph=False)
bad = 0
for t in range(n):
    w0 = pipe.window.cpu().tolist()
    pipe.status.zero_()
    pipe.step_eager()
    s = int(pipe.status.item())
    w1 = pipe.window.cpu().tolist()
    if s & 2 or t < 4 or t % 500 == 0:
        res_out = pipe.res[pipe.t % 2]
        lo = w0[1] if w0[0] & 1 else 0
        kr = res_out.view(torch.int32) & 0x7FFFFFFF
        ks = pipe.sel.val[:k].view(torch.int32) & 0x7FFFFFFF
        C = int((kr >= lo).sum()) + int((ks >= lo).sum())
        tau = int(ks.min())
        print(f"step {t}: status={s} window_in={w0} window_out={w1} C={C} tau={tau} tau-lo={tau - lo}", flush=True)
        bad += bool(s & 2)
        if bad > 10:
            break
print("fallback steps:", bad)
