"""Worker for tests/test_gpu_dist.py: one process per GPU (torchrun, NCCL +
IPC).  Checks the fused NVLink exchange kernel and the full gtopk_step
against the CPU oracle (the checker), bit-exactly, for the butterfly and the
tree + broadcast schedules, the poison path and the CUDA-graph pipeline.
Prints one JSON line per rank."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import gtopk_oracle as orc  # noqa: E402
from paper_1901_04359_b200 import collectives as coll  # noqa: E402
from paper_1901_04359_b200 import optimizer as opt  # noqa: E402
from paper_1901_04359_b200.dist import init_dist_cluster  # noqa: E402
from paper_1901_04359_b200.pipeline import GTopKPipeline  # noqa: E402
from paper_1901_04359_b200.device import DeviceList  # noqa: E402
from paper_1901_04359_b200.sparse import DeviceSparseVector, SparseVector  # noqa: E402
from paper_1901_04359_b200.transport import TransportError  # noqa: E402

F32 = np.float32


def bits(a):
    return np.asarray(a, F32).view(np.uint32)


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "auto"
    ep = init_dist_cluster(timeout=30.0, mode=mode)
    r, P = ep.rank, ep.world_size
    out = {"rank": r, "P": P, "mode": mode, "fails": []}

    def check(cond, what):
        if not cond:
            out["fails"].append(what)

    # 1. gtopk_allreduce on random / tied / cancelling inputs vs the tree fold
    rng = np.random.default_rng(77)
    for trial in range(12):
        m = int(rng.integers(50, 300_000))
        k = int(rng.integers(1, min(3000, m // 4) + 2))
        kind = trial % 3
        base = rng.standard_normal(m).astype(F32)
        lists = []
        for q in range(P):
            if kind == 0:
                g = rng.standard_normal(m).astype(F32)
            elif kind == 1:
                g = rng.integers(-3, 4, m).astype(F32)
            else:  # odd ranks cancel even ranks exactly on shared indices
                g = base if q % 2 == 0 else -base
            lists.append(orc.top_k_select(g, k)[:2])
        want_i, want_v = orc.tree_fold(lists, k)
        before = ep.stats.snapshot()
        res = coll.gtopk_allreduce(ep, SparseVector(m, *lists[r]), k, P)
        d = ep.stats.snapshot().delta(before)
        check(np.array_equal(res.global_topk.indices, want_i), f"idx trial {trial}")
        check(np.array_equal(bits(res.global_topk.values), bits(want_v)), f"val trial {trial}")
        check(d.msgs_sent >= 1, f"stats trial {trial}")

    # 1b. large k (the density sweep's regime): union slices of the exchange
    #     kernel's merges beyond the minimum shared-memory capacity, LL
    #     records of 400K entries per step
    m, k = 4_000_000, 400_000
    lr_rng = np.random.default_rng(9)
    lists = [orc.top_k_select(lr_rng.standard_normal(m).astype(F32), k)[:2] for _ in range(P)]
    want_i, want_v = orc.tree_fold(lists, k)
    res = coll.gtopk_allreduce(ep, SparseVector(m, *lists[r]), k, P)
    check(np.array_equal(res.global_topk.indices, want_i), "large-k idx")
    check(np.array_equal(bits(res.global_topk.values), bits(want_v)), "large-k val")

    # 1b. the TopK-AllReduce baseline (NCCL count + packed all-gather, rank-order
    #     accumulation, division at the touched entries) bitwise vs the
    #     reference's dense accumulation (collectives.py:148-165), device lists
    for trial in range(4):
        m = int(rng.integers(1000, 200_000))
        k = int(rng.integers(1, min(2000, m // 4) + 2))
        lists = [orc.top_k_select((rng.integers(-3, 4, m) if trial % 2 else rng.standard_normal(m)).astype(F32),
                                  k)[:2] for _ in range(P)]
        want = orc.topk_allreduce(lists, m, P)
        dl = DeviceList.from_host(m, *lists[r], ep.group.device, k)
        got = coll.topk_allreduce(ep, DeviceSparseVector(dl), P).cpu().numpy()
        check(np.array_equal(bits(got), bits(want)), f"topk_allreduce trial {trial}")

    # 2. full gtopk_step trajectories vs the oracle (m=270K ResNet-20 size)
    m, k, steps = 270_000, 270, 4
    g_rng = np.random.default_rng(5)
    grads = [[g_rng.standard_normal(m).astype(F32) for _ in range(P)] for _ in range(steps)]
    st = opt.make_state(np.zeros(m, F32), lr=0.1)
    for it in range(steps):
        rep = opt.gtopk_step(st, ep, grads[it][r], k, P)
    ref = [orc.State(np.zeros(m, F32), 0.1) for _ in range(P)]
    for it in range(steps):
        orc.gtopk_step_all(ref, grads[it], k)
    check(np.array_equal(bits(st.weights), bits(ref[r].weights)), "step weights")
    check(np.array_equal(bits(st.residual), bits(ref[r].residual)), "step residual")
    check(rep.selected_k == k, "selected_k")

    # 2b. topk_step trajectories (momentum 0: the touched-entry update,
    # gtk_topk_apply; momentum 0.9: the dense update) vs the oracle
    for mom in (0.0, 0.9):
        stt = opt.make_state(np.zeros(m, F32), lr=0.1, momentum=mom)
        for it in range(steps):
            opt.topk_step(stt, ep, grads[it][r], k, P)
        reft = [orc.State(np.zeros(m, F32), 0.1, mom) for _ in range(P)]
        for it in range(steps):
            orc.topk_step_all(reft, grads[it], k)
        check(np.array_equal(bits(stt.weights), bits(reft[r].weights)), f"topk_step weights mom={mom}")
        check(np.array_equal(bits(stt.residual), bits(reft[r].residual)), f"topk_step residual mom={mom}")

    # 2b'. a non-finite gradient on rank 0 in topk_step (status carried in
    # the all-gather): rank 0 raises FloatingPointError, the others
    # TransportError, nobody's state moves, and the next step is exact
    from paper_1901_04359_b200.transport import TransportError as _TE

    stp = opt.make_state(np.zeros(m, F32), lr=0.1)
    opt.topk_step(stp, ep, grads[0][r], k, P)
    w_before, res_before = stp.weights.copy(), stp.residual.copy()
    badg = grads[1][r].copy()
    if r == 0:
        badg[17] = np.nan
    try:
        opt.topk_step(stp, ep, badg, k, P)
        check(False, "poisoned topk_step did not raise")
    except FloatingPointError:
        check(r == 0, "FloatingPointError on a healthy rank")
    except _TE:
        check(r != 0, "TransportError on the failing rank")
    check(np.array_equal(bits(stp.weights), bits(w_before)), "poisoned topk_step moved the weights")
    check(np.array_equal(bits(stp.residual), bits(res_before)), "poisoned topk_step moved the residual")
    opt.topk_step(stp, ep, grads[2][r], k, P)
    refp = [orc.State(np.zeros(m, F32), 0.1) for _ in range(P)]
    orc.topk_step_all(refp, [grads[0][q] for q in range(P)], k)
    orc.topk_step_all(refp, [grads[2][q] for q in range(P)], k)
    check(np.array_equal(bits(stp.weights), bits(refp[r].weights)), "topk_step after a poisoned step")
    check(np.array_equal(bits(stp.residual), bits(refp[r].residual)), "topk_step residual after a poisoned step")

    # 2c. mismatched dense lengths raise ProtocolError on every rank
    # (collectives.py:113-117), and the group stays usable
    from paper_1901_04359_b200.transport import ProtocolError

    try:
        coll.dense_ring_allreduce(ep, np.ones(8 + r, F32))
        check(False, "dense length mismatch: no ProtocolError")
    except ProtocolError:
        pass
    ok = coll.dense_ring_allreduce(ep, np.full(9, r + 1.0, F32))
    check(np.array_equal(ok, np.full(9, P * (P + 1) / 2, F32)), "dense allreduce after a mismatch")

    # 3. the CUDA-graph pipeline gives the same trajectory
    dev = ep.group.device
    dg = [torch.from_numpy(grads[0][r]).to(dev), torch.from_numpy(grads[1][r]).to(dev)]
    st2 = opt.make_state(torch.zeros(m, device=dev), lr=0.1)
    pipe = GTopKPipeline(ep, st2, k, dg)
    pipe.capture()  # two eager steps
    pipe.run(30)  # graph replays: the carried select/merge key windows get used and adapt
    pipe.check()
    pipe.sync_state()
    ref2 = [orc.State(np.zeros(m, F32), 0.1) for _ in range(P)]
    for it in range(32):
        orc.gtopk_step_all(ref2, grads[it % 2], k)
    check(np.array_equal(bits(st2.weights.cpu().numpy()), bits(ref2[r].weights)), "pipeline weights")
    check(np.array_equal(bits(st2.residual.cpu().numpy()), bits(ref2[r].residual)), "pipeline residual")
    check(pipe.deferred, "pipeline: deferred steps (the default mode)")
    # 3b. the non-deferred step (select_push + exchange with the residual restore)
    os.environ["GTK_PIPE_MODE"] = "plain"
    try:
        st2b = opt.make_state(torch.zeros(m, device=dev), lr=0.1)
        pipeb = GTopKPipeline(ep, st2b, k, dg)
        pipeb.capture()
        pipeb.run(30)
        pipeb.check()
        pipeb.sync_state()
        check(not pipeb.deferred, "plain pipeline mode")
        check(np.array_equal(bits(st2b.weights.cpu().numpy()), bits(ref2[r].weights)), "plain pipeline weights")
        check(np.array_equal(bits(st2b.residual.cpu().numpy()), bits(ref2[r].residual)), "plain pipeline residual")
    finally:
        del os.environ["GTK_PIPE_MODE"]

    # 4. poison: a non-finite gradient on rank P-1 fails the step everywhere,
    #    state untouched
    st3 = opt.make_state(np.zeros(1000, F32), lr=0.1)
    g = np.ones(1000, F32)
    if r == P - 1:
        g[17] = np.inf
    w_before = st3.weights.copy()
    try:
        opt.gtopk_step(st3, ep, g, 10, P)
        check(False, "poison: no exception")
    except FloatingPointError:
        check(r == P - 1, "poison: FloatingPointError on a healthy rank")
    except TransportError:
        check(r != P - 1, "poison: TransportError on the failing rank")
    check(np.array_equal(st3.weights, w_before) and st3.iteration == 0, "poison: state changed")
    # 5. poison through the graph pipeline (the selection goes to the first
    #    partner straight from K1's finish: a non-finite input sends count -1
    #    from there): every rank's sticky status fails, K3 never ran after it
    m5, k5 = 50_000, 50
    gp = [np.random.default_rng(100 + r).standard_normal(m5).astype(F32) for _ in range(2)]
    if r == P - 1:
        gp[1][77] = np.inf
    st5 = opt.make_state(torch.zeros(m5, device=dev), lr=0.1)
    pipe5 = GTopKPipeline(ep, st5, k5, [torch.from_numpy(x).to(dev) for x in gp])
    try:
        pipe5.capture()  # step 1 (the second gradient) is poisoned
        pipe5.run(3)
        pipe5.check()
        check(False, "pipeline poison: no exception")
    except FloatingPointError:
        check(r == P - 1, "pipeline poison: FloatingPointError on a healthy rank")
    except TransportError:
        check(r != P - 1, "pipeline poison: TransportError on the failing rank")
    # the cluster is still usable afterwards
    res = coll.gtopk_allreduce(ep, SparseVector(100, [r], [1.0 + r]), 1, P)
    check(res.global_topk.indices.tolist() == [P - 1], "after poison")

    print("RESULT " + json.dumps(out), flush=True)
    dist.barrier()
    ep.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
