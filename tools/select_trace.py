"""Phase timestamps (block 0, %globaltimer) of the select finish kernel."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_04359_b200.device as dev
from paper_1901_04359_b200 import _lib
lib = _lib.load()
d = torch.device("cuda", 0)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 25_600
g = torch.randn(m, device=d); r = 0.1 * torch.randn(m, device=d); out = torch.empty_like(g)
lst = dev.DeviceList(m, k, d); st = torch.zeros(1, dtype=torch.int32, device=d)
for _ in range(3): dev.select(r, g, out, k, lst, st)
tr = torch.zeros(128, dtype=torch.int64, device=d)
lib.gtk_exchange_set_trace(ctypes.c_void_p(tr.data_ptr()))
names = ["start", "scanned", "copied", "bin", "gather_bar", "ranked", "written"]
for rep in range(3):
    tr.zero_(); torch.cuda.synchronize()
    dev.select(r, g, out, k, lst, st); torch.cuda.synchronize()
    t = tr.cpu().tolist()[48:55]
    print(f"finish rep{rep}: " + " ".join(f"{n}={(v - t[0]) / 1e3:.1f}" for n, v in zip(names, t) if v), flush=True)
    u = tr.cpu().tolist()[64:71]
    sn = ["start", "loaded", "radix", "emitted", "last_start", "last_loaded", "last_radix"]
    print(f"sample rep{rep}: " + " ".join(f"{n}={(v - u[0]) / 1e3:.1f}" for n, v in zip(sn, u) if v)
          + f" | finish_start={(t[0] - u[0]) / 1e3:.1f}", flush=True)
    w = tr.cpu().tolist()[72:78]
    x = tr.cpu().tolist()[80:86]
    print("  phaseA levels: " + " ".join(f"{(v - u[0]) / 1e3:.2f}" for v in w if v)
          + " | last levels: " + " ".join(f"{(v - u[0]) / 1e3:.2f}" for v in x if v), flush=True)
lib.gtk_exchange_set_trace(None)
