"""Small invocations of every device path for compute-sanitizer
(racecheck / synccheck / memcheck): K1 plain / windowed / chained / deferred,
K2 top_op (grid and cluster merges), the fused exchange (+K3) on a loopback
inbox, and the sparse update.  Exits non-zero if any result differs from the
oracle.  Usage: compute-sanitizer --tool racecheck python tools/sanitize_paths.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1901_04359_b200.device as dev  # noqa: E402
from oracle import gtopk_oracle as orc  # noqa: E402

F32 = np.float32
d = torch.device("cuda", 0)
rng = np.random.default_rng(3)
m, k = 300_000, 300
ok = True


def same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint32) if np.asarray(a).dtype == F32 else a,
                          np.asarray(b).view(np.uint32) if np.asarray(b).dtype == F32 else b)


# K1: plain, windowed (two calls), forced exact
st = torch.zeros(1, dtype=torch.int32, device=d)
g = rng.standard_normal(m).astype(F32)
r = (0.3 * rng.standard_normal(m)).astype(F32)
out = torch.empty(m, device=d)
lst = dev.DeviceList(m, k, d)
win = dev.new_window(d)
for flags in ("plain", "win", "win", "exact"):
    dev.select(torch.from_numpy(r).to(d), torch.from_numpy(g).to(d), out, k, lst, st,
               force_exact=flags == "exact", window=win if flags == "win" else None)
    i, v = lst.to_host()
    wi, wv, wr = orc.top_k_select(r + g, k)
    ok &= same(i, wi) and same(v, wv) and same(out.cpu().numpy(), wr)
print("K1 select:", ok, flush=True)

# K1 + K3 deferred, 4 steps
R = [torch.zeros(m, device=d), torch.empty(m, device=d)]
w = torch.zeros(m, device=d)
wins = [dev.new_window(d) for _ in range(2)]
wss = [dev.select_workspace(m, k, d, slot=21 + i) for i in range(2)]
sels = [dev.DeviceList(m, k, d) for _ in range(2)]
ref = orc.State(np.zeros(m, F32), 0.05)
for t in range(4):
    g = rng.standard_normal(m).astype(F32)
    p = t % 2
    dev.select_update_deferred(R[p], torch.from_numpy(g).to(d), R[1 - p], k, sels[p], st, wins[p], wss[p],
                               sels[1 - p] if t else None, w, float(F32(0.05)), 1, 0, prev_ws=wss[1 - p])
    (gi, gv), _ = orc.gtopk_step_all([ref], [g], k)
    i, v = sels[p].to_host()
    ok &= same(i, gi) and same(v, gv) and same(w.cpu().numpy(), ref.weights)
print("K1 deferred:", ok, flush=True)

# K2 top_op: cluster (small k) and cooperative grid
for kk, env in ((1500, "1"), (1500, "0"), (20_000, None)):
    if env is None:
        os.environ.pop("GTK_MERGE_CLUSTER", None)
    else:
        os.environ["GTK_MERGE_CLUSTER"] = env
    a = orc.top_k_select(rng.standard_normal(m).astype(F32), kk)[:2]
    b = orc.top_k_select(rng.standard_normal(m).astype(F32), kk)[:2]
    A = dev.DeviceList.from_host(m, *a, d, kk)
    B = dev.DeviceList.from_host(m, *b, d, kk)
    o = dev.DeviceList(m, kk, d)
    dev.top_op(A, B, kk, o)
    oi, ov = o.to_host()
    wi, wv = orc.top_op(*a, *b, kk)
    ok &= same(oi, wi) and same(ov, wv)
os.environ.pop("GTK_MERGE_CLUSTER", None)
print("K2 top_op:", ok, flush=True)

# the fused exchange + K3 on a loopback inbox (rank 1 of P = 2 and rank 3 of P = 4)
import test_gpu_exchange_loopback as lbt  # noqa: E402

for P in (2, 4):
    lists = lbt._lists(rng, P, m, k, "normal")
    lbt.check_rank(P - 1, P, "butterfly", lists, k, m, rng, calls=2)
print("exchange loopback:", ok, flush=True)
sys.exit(0 if ok else 1)
