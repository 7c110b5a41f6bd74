"""Phase stamps (block 0, %globaltimer) of the finish kernel in the steady
state (carried window), plus the sample kernel's publish."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_04359_b200 as gk
from paper_1901_04359_b200 import optimizer as opt, _lib
from paper_1901_04359_b200.pipeline import GTopKPipeline
lib = _lib.load()
d = torch.device("cuda", 0)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 25_600
npre = int(sys.argv[3]) if len(sys.argv) > 3 else 1500
gen = torch.Generator(device=d).manual_seed(5)
grads = [torch.randn(m, device=d, generator=gen) for _ in range(2)]
ep = gk.create_local_cluster(1)[0]
st = opt.make_state(torch.zeros(m, device=d), lr=0.01)
pipe = GTopKPipeline(ep, st, k, grads)
pipe.capture()
pipe.run(npre)
torch.cuda.synchronize()
tr = torch.zeros(128, dtype=torch.int64, device=d)
lib.gtk_exchange_set_trace(ctypes.c_void_p(tr.data_ptr()))
names = ["start", "scanned", "copied", "bin", "gather_bar", "ranked", "written"]
for rep in range(4):
    tr.zero_(); torch.cuda.synchronize()
    pipe.step_eager(); torch.cuda.synchronize()
    t = tr.cpu().tolist()
    s0 = t[64]  # sample kernel, block 0 after its pdl_wait
    print(f"timeline rep{rep} (us from sample start): main start={(t[112]-s0)/1e3:.1f} main end={(t[113]-s0)/1e3:.1f} "
          f"finish start={(t[48]-s0)/1e3:.1f} finish end={(t[114]-s0)/1e3:.1f}", flush=True)
    f = t[48:55]
    print(f"finish rep{rep}: " + " ".join(f"{n}={(v - f[0]) / 1e3:.1f}" for n, v in zip(names, f) if v)
          + f" | round-0 in_bin={t[55]} w_scanned={(t[56]-f[0])/1e3:.1f} w_put={(t[57]-f[0])/1e3:.1f} own={t[58]} cap={t[59]} C={t[60]} G={t[61]}", flush=True)
lib.gtk_exchange_set_trace(None)
