"""Step-by-step eager deferred pipeline (P = 1): which steps take the dense
fallback, the two parity records, and the candidate count the main pass saw."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GTK_PIPE_MODE", "defer")
import torch  # noqa: E402

import paper_1901_04359_b200 as gk  # noqa: E402
from paper_1901_04359_b200 import optimizer as opt  # noqa: E402
from paper_1901_04359_b200.pipeline import GTopKPipeline  # noqa: E402

d = torch.device("cuda", 0)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
n = int(sys.argv[3]) if len(sys.argv) > 3 else 60
gen = torch.Generator(device=d).manual_seed(5)
grads = [torch.randn(m, device=d, generator=gen) for _ in range(2)]
ep = gk.create_local_cluster(1)[0]
st = opt.make_state(torch.zeros(m, device=d), lr=0.01)
pipe = GTopKPipeline(ep, st, k, grads, use_graph=False)
import ctypes  # noqa: E402

from paper_1901_04359_b200 import _lib  # noqa: E402

tr = torch.zeros(256, dtype=torch.int64, device=d)
_lib.load().gtk_exchange_set_trace(ctypes.c_void_p(tr.data_ptr()))
bad = 0
for t in range(n):
    tr.zero_()
    p = t % 2
    w0 = pipe.dwin[p].cpu().tolist()
    pipe.status.zero_()
    pipe.step_eager()
    s = int(pipe.status.item())
    w1 = pipe.dwin[p].cpu().tolist()
    ws = pipe.dws[p]
    ctl = ws[:64].view(torch.int32).cpu().tolist()  # SelectCtl: lo, shift, ovf_cursor, overflow, nonfinite
    f = tr[48:68].cpu().tolist()
    print(f"step {t}: status={s:#x} rec_in={w0[:6]} rec_out={w1[:6]} lo,shift={ctl[:2]} "
          f"own={f[10]} cap={f[11]} C={f[12]} G={f[13]} n_fix={f[14]} n_ins={f[15]} ovf={f[16]} C2={f[17]} "
          f"ord_cap={f[18]} fell={f[19]}", flush=True)
    bad += bool(s & 2)
print("fallback steps:", bad)
