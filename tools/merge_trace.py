"""Phase timestamps (block 0, %globaltimer) of one standalone merge."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_04359_b200.device as dev
from paper_1901_04359_b200 import _lib
lib = _lib.load()
d = torch.device("cuda", 0)
st = torch.zeros(1, dtype=torch.int32, device=d)
for k in [int(x) for x in sys.argv[1:]] or [270, 25600, 66000]:
    m = min(max(1000 * k, 4 * k), 66_000_000)
    g = torch.randn(m, device=d); r = torch.randn(m, device=d); out = torch.empty_like(g)
    a = dev.DeviceList(m, k, d); b = dev.DeviceList(m, k, d); o = dev.DeviceList(m, k, d)
    dev.select(None, g, out, k, a, st); dev.select(None, r, out, k, b, st)
    for _ in range(3): dev.top_op(a, b, k, o)
    tr = torch.zeros(64, dtype=torch.int64, device=d)
    lib.gtk_exchange_set_trace(ctypes.c_void_p(tr.data_ptr()))
    for rep in range(3):
        tr.zero_(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); dev.top_op(a, b, k, o); e.record(); e.synchronize()
        t = tr.cpu().tolist()[32:41]
        names = ["path", "slots", "hist_bar", "engine_end", "bin", "gather_bar", "ranked", "written"]
        base = t[0]
        print(f"k={k} rep{rep}: event {s.elapsed_time(e)*1e3:.1f}us | " +
              " ".join(f"{n}={(v-base)/1e3:.1f}" for n, v in zip(["start"] + names, t) if v), flush=True)
    lib.gtk_exchange_set_trace(None)
