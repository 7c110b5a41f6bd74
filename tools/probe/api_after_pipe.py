"""Public gtopk_step after the pipeline (bench.py's e2e order): per-call status and window record."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1901_04359_b200 as gk  # noqa: E402
from paper_1901_04359_b200 import optimizer as opt  # noqa: E402
from paper_1901_04359_b200.pipeline import GTopKPipeline  # noqa: E402

m, k = 25_600_000, 25_600
pre = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
torch.cuda.set_device(0)
d = torch.device("cuda", 0)
rng = np.random.default_rng(0)
host = [rng.standard_normal(m).astype(np.float32) for _ in range(2)]
dg = [torch.from_numpy(g).to(d) for g in host]
ep = gk.create_local_cluster(1)[0]
st = opt.make_state(torch.zeros(m, device=d), lr=0.01)
pipe = GTopKPipeline(ep, st, k, dg)
pipe.capture()
pipe.run(pre)
torch.cuda.synchronize()
pipe.check()
pipe.sync_state()
print("pipeline dwin records:", [w.cpu().numpy().tolist() for w in pipe.dwin])
pinned = [torch.from_numpy(g).pin_memory() for g in host]
src = pinned if os.environ.get("PINNED") else dg
for i in range(30):
    opt.gtopk_step(st, ep, src[i % 2], k, 1)
    win = st._window.cpu().numpy()
    print(i, hex(st._bufs.get("last_status", 0)), "rec", win.tolist())
