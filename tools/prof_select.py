"""Back-to-back select timing + launch list helper (ncu wrapper target)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_04359_b200.device as dev
m = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 25_600
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
d = torch.device("cuda", 0)
g = torch.randn(m, device=d); r = 0.1 * torch.randn(m, device=d); out = torch.empty_like(g)
lst = dev.DeviceList(m, k, d); st = torch.zeros(1, dtype=torch.int32, device=d)
for _ in range(3): dev.select(r, g, out, k, lst, st)
torch.cuda.synchronize()
torch.cuda._sleep(int(4e7))
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(n): dev.select(r, g, out, k, lst, st)
e.record(); e.synchronize()
print(f"select m={m} k={k}: {s.elapsed_time(e)/n*1e3:.1f} us/call (GPU-saturated) status={int(st.item())}")
