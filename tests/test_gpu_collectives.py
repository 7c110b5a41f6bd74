"""GPU parity of the collectives and optimizer steps (in-process cluster on
cuda:0, one host thread per rank), against golden vectors from the reference,
the reference's own test expectations (pkg/tests/test_collectives.py,
test_optimizer.py) and the CPU oracle at BASELINE config 1/2 sizes."""

import numpy as np
import pytest

from conftest import cuda_ok, load_golden

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA GPU")]

F32 = np.float32


def bits(a):
    return np.asarray(a, F32).view(np.uint32)


@pytest.fixture(scope="module")
def gk():
    import paper_1901_04359_b200 as gk

    return gk


@pytest.fixture(scope="module")
def opt():
    from paper_1901_04359_b200 import optimizer as opt

    return opt


@pytest.fixture(scope="module")
def coll():
    from paper_1901_04359_b200 import collectives as coll

    return coll


def sv(gk, dim, pairs):
    return gk.SparseVector.from_pairs(dim, pairs)


def zeros(m):
    return np.zeros(m, dtype=F32)


def random_sparse(gk, rng, m, k):
    from oracle import gtopk_oracle as orc

    i, v, _ = orc.top_k_select(rng.standard_normal(m).astype(F32), k)
    return gk.SparseVector(m, i, v)


# ---- golden: the reference's own cluster outputs and accounting -------------


def test_allreduce_golden(gk, coll):
    z = load_golden("allreduce.npz")
    for c in range(int(z["n"])):
        P, m, k = int(z[f"c{c}_P"]), int(z[f"c{c}_m"]), int(z[f"c{c}_k"])
        ins = [gk.SparseVector(m, z[f"c{c}_in{r}_idx"], z[f"c{c}_in{r}_val"]) for r in range(P)]
        dense = [z[f"c{c}_dense{r}"] for r in range(P)]

        def worker(ep):
            before = ep.stats.snapshot()
            g = coll.gtopk_allreduce(ep, ins[ep.rank], k, P)
            d = ep.stats.snapshot().delta(before)
            t = coll.topk_allreduce(ep, ins[ep.rank], P)
            r = coll.dense_ring_allreduce(ep, dense[ep.rank])
            return g, d, t, r

        outs = gk.run_workers(gk.create_local_cluster(P), worker)
        for r in range(P):
            g, d, t, ring = outs[r]
            assert np.array_equal(g.global_topk.indices, z[f"c{c}_g_idx"]), (c, r)
            assert np.array_equal(bits(g.global_topk.values), bits(z[f"c{c}_g_val"])), (c, r)
            assert g.global_mask.indices.tolist() == z[f"c{c}_g_idx"].tolist()
            st = z[f"c{c}_stats{r}"]
            assert [d.bytes_sent, d.bytes_recv, d.msgs_sent, d.msgs_recv] == st.tolist(), (c, r)
            assert np.array_equal(bits(t), bits(z[f"c{c}_topk"])), (c, r)
            np.testing.assert_allclose(ring, z[f"c{c}_ring"], rtol=1e-4, atol=1e-5)
            assert np.array_equal(bits(ring), bits(outs[0][3]))


def test_steps_golden(gk, opt):
    z = load_golden("steps.npz")
    for c in range(int(z["n"])):
        algo = str(z[f"c{c}_algo"])
        P, m, k = int(z[f"c{c}_P"]), int(z[f"c{c}_m"]), int(z[f"c{c}_k"])
        lr, mom, scaling = float(z[f"c{c}_lr"]), float(z[f"c{c}_mom"]), str(z[f"c{c}_scaling"])
        grads = z[f"c{c}_grads"]
        winit = z[f"c{c}_winit"]  # NpzFile reads are not thread-safe: load before the workers
        fn = opt.STEP_FNS[algo]

        def worker(ep):
            st = opt.make_state(winit, lr=lr, momentum=mom, update_scaling=scaling)
            ks = []
            for it in range(grads.shape[0]):
                if algo == "dense":
                    rep = fn(st, ep, grads[it][ep.rank], P, rank_order_sum=True)
                else:
                    rep = fn(st, ep, grads[it][ep.rank], k, P)
                ks.append(rep.selected_k)
            return st.weights.copy(), st.residual.copy(), ks

        outs = gk.run_workers(gk.create_local_cluster(P), worker)
        for r in range(P):
            if algo == "dense":  # ring order in the reference vs rank order here
                np.testing.assert_allclose(outs[r][0], z[f"c{c}_w{r}"], rtol=1e-5, atol=1e-6)
                continue
            assert np.array_equal(bits(outs[r][0]), bits(z[f"c{c}_w{r}"])), (c, algo, r)
            assert np.array_equal(bits(outs[r][1]), bits(z[f"c{c}_res{r}"])), (c, algo, r)
            assert outs[r][2] == z[f"c{c}_selk{r}"].tolist(), (c, algo, r)


# ---- reference test_collectives.py expectations --------------------------------


def test_gtopk_known_answers(gk, coll):
    (ep,) = gk.create_local_cluster(1)
    local = sv(gk, 8, [(2, 1.0), (5, -4.0)])
    res = coll.gtopk_allreduce(ep, local, 2, 1)
    assert res.global_topk == local and res.global_mask.indices.tolist() == [2, 5]
    with pytest.raises(ValueError):
        coll.gtopk_allreduce(ep, sv(gk, 8, [(0, 1.0), (1, 1.0), (2, 1.0)]), 2, 1)
    eps = gk.create_local_cluster(2)
    ins = [sv(gk, 6, [(1, 0.5), (3, -2.0)]), sv(gk, 6, [(1, 0.6), (4, 1.0)])]
    outs = gk.run_workers(eps, lambda ep: coll.gtopk_allreduce(ep, ins[ep.rank], 2, 2))
    want = sv(gk, 6, [(1, np.float32(0.5) + np.float32(0.6)), (3, -2.0)])
    assert all(r.global_topk == want for r in outs)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8, 16])
def test_gtopk_matches_tree_fold(gk, coll, P):
    from oracle import gtopk_oracle as orc

    rng = np.random.default_rng(100 + P)
    eps = gk.create_local_cluster(P)
    for _ in range(12):
        m = int(rng.integers(4, 65))
        k = int(rng.integers(1, min(8, m) + 1))
        ins = [random_sparse(gk, rng, m, k) for _ in range(P)]
        wi, wv = orc.tree_fold([(s.indices, s.values) for s in ins], k)
        outs = gk.run_workers(eps, lambda ep: coll.gtopk_allreduce(ep, ins[ep.rank], k, P))
        for res in outs:
            assert res.global_topk.indices.tolist() == wi.tolist()
            assert np.array_equal(bits(res.global_topk.values), bits(wv))


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_rank0_message_accounting(gk, coll, n):
    P, k, m = 2 ** n, 4, 128
    rng = np.random.default_rng(200 + n)
    ins = [random_sparse(gk, rng, m, k) for _ in range(P)]

    def worker(ep):
        before = ep.stats.snapshot()
        coll.gtopk_allreduce(ep, ins[ep.rank], k, P)
        return ep.stats.snapshot().delta(before)

    d = gk.run_workers(gk.create_local_cluster(P), worker)
    msg = 12 + 12 * k
    assert (d[0].msgs_recv, d[0].msgs_sent, d[0].bytes_recv, d[0].bytes_sent) == (n, n, n * msg, n * msg)


def test_gtopk_cardinality_and_containment(gk, coll):
    rng = np.random.default_rng(56)
    P, m, k = 4, 64, 6
    ins = [random_sparse(gk, rng, m, k) for _ in range(P)]
    outs = gk.run_workers(gk.create_local_cluster(P), lambda ep: coll.gtopk_allreduce(ep, ins[ep.rank], k, P))
    assert all(res.global_topk.nnz == k for res in outs)
    union = set().union(*[set(s.indices.tolist()) for s in ins])
    assert all(set(r.global_topk.indices.tolist()) <= union for r in outs)


def test_topk_allreduce(gk, coll):
    (ep,) = gk.create_local_cluster(1)
    local = sv(gk, 4, [(1, 3.0)])
    assert np.array_equal(coll.topk_allreduce(ep, local, 1), gk.densify(local))
    ins = [sv(gk, 4, [(0, 1.0)]), sv(gk, 4, [(0, 3.0)])]
    outs = gk.run_workers(gk.create_local_cluster(2), lambda ep: coll.topk_allreduce(ep, ins[ep.rank], 2))
    assert all(np.array_equal(o, np.array([2, 0, 0, 0], F32)) for o in outs)
    rng = np.random.default_rng(10)
    P, m, k = 4, 32, 4
    for _ in range(10):
        ins = [random_sparse(gk, rng, m, k) for _ in range(P)]
        want = np.zeros(m, F32)
        for s in ins:
            want[s.indices] += s.values
        want /= F32(P)
        outs = gk.run_workers(gk.create_local_cluster(P), lambda ep: coll.topk_allreduce(ep, ins[ep.rank], P))
        assert all(np.array_equal(o, want) for o in outs)

    def worker(ep):
        before = ep.stats.snapshot()
        coll.topk_allreduce(ep, ins[ep.rank], P)
        return ep.stats.snapshot().delta(before)

    for d in gk.run_workers(gk.create_local_cluster(P), worker):
        assert d.bytes_sent == coll.predicted_bytes("topk", P, m, k)


def test_dense_allreduce(gk, coll):
    from paper_1901_04359_b200.transport import ProtocolError

    (ep,) = gk.create_local_cluster(1)
    g = np.array([1.0, -2.0], F32)
    assert np.array_equal(coll.dense_ring_allreduce(ep, g), g)
    outs = gk.run_workers(gk.create_local_cluster(3),
                          lambda ep: coll.dense_ring_allreduce(ep, np.full(6, ep.rank + 1.0, F32)))
    assert all(np.array_equal(o, np.full(6, 6.0, F32)) for o in outs)
    rng = np.random.default_rng(7)
    for m in (5, 16, 64, 257):
        ins = [rng.standard_normal(m).astype(F32) for _ in range(4)]
        want = np.sum(np.stack(ins), axis=0, dtype=np.float64)
        outs = gk.run_workers(gk.create_local_cluster(4), lambda ep: coll.dense_ring_allreduce(ep, ins[ep.rank]))
        from oracle import gtopk_oracle as orc

        ring = orc.dense_ring_allreduce(ins)  # the reference's ring order, simulated
        for r, o in enumerate(outs):
            np.testing.assert_allclose(o, want, rtol=1e-4, atol=1e-5)
            assert np.array_equal(bits(o), bits(ring[r]))  # bitwise the ring's sum
    with pytest.raises(ProtocolError):
        gk.run_workers(gk.create_local_cluster(2, timeout=5),
                       lambda ep: coll.dense_ring_allreduce(ep, np.ones([8, 12][ep.rank], F32)))

    def worker(ep):
        before = ep.stats.snapshot()
        coll.dense_ring_allreduce(ep, ins[ep.rank][:33] if ep.rank < 4 else None)
        return ep.stats.snapshot().delta(before)

    for d in gk.run_workers(gk.create_local_cluster(4), worker):
        assert d.bytes_sent == coll.predicted_bytes("dense", 4, 33, 0) and d.msgs_sent == 6


# ---- reference test_optimizer.py expectations ----------------------------------


def test_dense_step_known_answers(gk, opt):
    (ep,) = gk.create_local_cluster(1)
    st = opt.make_state(zeros(1), lr=0.1)
    opt.dense_step(st, ep, np.array([1.0], F32), 1)
    assert np.array_equal(st.weights, np.array([-0.1], F32)) and st.iteration == 1
    grads = [np.array([1.0], F32), np.array([3.0], F32)]

    def worker(ep):
        s = opt.make_state(zeros(1), lr=0.1)
        opt.dense_step(s, ep, grads[ep.rank], 2)
        return s.weights

    assert all(np.array_equal(w, np.array([-0.2], F32)) for w in gk.run_workers(gk.create_local_cluster(2), worker))
    (ep,) = gk.create_local_cluster(1)
    st = opt.make_state(zeros(2), lr=1.0, momentum=0.5)
    g = np.array([1.0, 0.0], F32)
    opt.dense_step(st, ep, g, 1)
    opt.dense_step(st, ep, g, 1)
    assert np.array_equal(st.weights, np.array([-2.5, 0.0], F32))


def test_topk_step_known_answers(gk, opt):
    grads = [np.array([1.0, 0.0, 0.0, 0.1], F32), np.array([0.0, 2.0, 0.0, 0.1], F32)]

    def worker(ep):
        st = opt.make_state(zeros(4), lr=1.0)
        opt.topk_step(st, ep, grads[ep.rank], 1, 2)
        return st

    states = gk.run_workers(gk.create_local_cluster(2), worker)
    for st in states:
        assert np.array_equal(st.weights, -np.array([0.5, 1.0, 0.0, 0.0], F32))
        assert np.array_equal(st.residual, np.array([0, 0, 0, 0.1], F32))
    (ep,) = gk.create_local_cluster(1)
    st = opt.make_state(zeros(2), lr=1.0)
    g = np.array([0.3, 0.5], F32)
    opt.topk_step(st, ep, g, 1, 1)
    assert np.array_equal(st.weights, np.array([0.0, -0.5], F32))
    assert np.array_equal(st.residual, np.array([0.3, 0.0], F32))
    opt.topk_step(st, ep, g, 1, 1)
    assert np.array_equal(st.weights, np.array([-0.6, -0.5], F32))
    assert np.array_equal(st.residual, np.array([0.0, 0.5], F32))


def test_gtopk_step_known_answers(gk, opt):
    grads = [np.array([1.0, 0, 0, 0], F32), np.array([0, 2.0, 0, 0], F32)]

    def worker(ep):
        st = opt.make_state(zeros(4), lr=1.0)
        rep = opt.gtopk_step(st, ep, grads[ep.rank], 1, 2)
        return st, rep

    outs = gk.run_workers(gk.create_local_cluster(2), worker)
    for st, rep in outs:
        assert np.array_equal(st.weights, np.array([0, -1.0, 0, 0], F32)) and rep.selected_k == 1
        assert rep.t_compress_ms >= 0.0 and rep.t_communicate_ms >= 0.0
    assert np.array_equal(outs[0][0].residual, np.array([1, 0, 0, 0], F32))
    assert not outs[1][0].residual.any()
    # sum scaling
    grads = [np.array([1.0, 0.0], F32), np.array([3.0, 0.0], F32)]

    def w2(ep):
        st = opt.make_state(zeros(2), lr=1.0, update_scaling="sum")
        opt.gtopk_step(st, ep, grads[ep.rank], 1, 2)
        return st.weights

    assert all(np.array_equal(w, np.array([-4.0, 0.0], F32)) for w in gk.run_workers(gk.create_local_cluster(2), w2))


def test_single_worker_gtopk_equals_topk_and_naive(gk, opt):
    m, k, steps = 16, 3, 20
    rng = np.random.default_rng(5)
    grads = [rng.standard_normal(m).astype(F32) for _ in range(steps)]

    def run(fn):
        (ep,) = gk.create_local_cluster(1)
        st = opt.make_state(zeros(m), lr=0.3)
        for g in grads:
            fn(st, ep, g, k, 1)
        return st

    a, b, c = run(opt.topk_step), run(opt.gtopk_step), run(opt.gtopk_naive_step)
    for s in (b, c):
        assert np.array_equal(a.weights, s.weights) and np.array_equal(a.residual, s.residual)


def test_divergence_and_lost_mass(gk, opt):
    P, m, k = 4, 8, 2
    grads = [zeros(m) for _ in range(P)]
    for r, v in enumerate([0.9, 0.8, 0.7, 0.6]):
        grads[r][r] = v
        grads[r][4] = 0.25

    def tree(ep):
        st = opt.make_state(zeros(m), lr=1.0)
        rep = opt.gtopk_step(st, ep, grads[ep.rank], k, P, measure_divergence=True)
        return st.weights, rep

    def naive(ep):
        st = opt.make_state(zeros(m), lr=1.0)
        rep = opt.gtopk_naive_step(st, ep, grads[ep.rank], k, P, measure_divergence=True)
        return st.weights, rep

    tw, trep = gk.run_workers(gk.create_local_cluster(P), tree)[0]
    nw, nrep = gk.run_workers(gk.create_local_cluster(P), naive)[0]
    assert tw.nonzero()[0].tolist() == [0, 1] and nw.nonzero()[0].tolist() == [0, 4]
    assert trep.divergence == nrep.divergence == 0.5
    assert trep.lost_mass == 0.0 and nrep.lost_mass == 0.0

    P, m, k = 4, 10, 3
    grads = [zeros(m) for _ in range(P)]
    grads[0][[0, 5, 6]] = [0.9, 0.3, 0.25]
    grads[1][[1, 5, 6]] = [0.8, 0.3, 0.25]
    grads[2][[2, 6, 7]] = [0.7, 2.0, 0.1]
    grads[3][[3, 5, 7]] = [0.6, 0.3, 0.1]

    def w(ep):
        st = opt.make_state(zeros(m), lr=1.0)
        return opt.gtopk_step(st, ep, grads[ep.rank], k, P, measure_divergence=True), st

    outs = gk.run_workers(gk.create_local_cluster(P), w)
    rep0, st0 = outs[0]
    assert st0.weights.nonzero()[0].tolist() == [0, 1, 6]
    assert rep0.lost_mass == pytest.approx(0.5, abs=1e-6)
    assert rep0.divergence == pytest.approx(1 / 3)
    assert outs[0][1].residual[6] == 0.0 and outs[1][1].residual[6] == 0.0


def test_divergence_lost_mass_bitwise(gk, opt):
    """measure_divergence at a real size, bitwise against the reference's own
    formulas (optimizer.py:232-241) on the oracle's selections: the mass is
    numpy's sum over all m slots (zeros included), the divergence the set
    arithmetic of _mask_divergence."""
    from oracle import gtopk_oracle as orc

    P, m, k = 4, 200_003, 1500
    rng = np.random.default_rng(23)
    grads = [rng.standard_normal(m).astype(np.float32) for _ in range(P)]
    # correlated coordinates, so the tree prunes mass that lands in the mask
    hot = rng.choice(m, 400, replace=False)
    for g in grads:
        g[hot] += np.float32(2.5)
    sels = [orc.top_k_select(g, k)[:2] for g in grads]
    total = np.zeros(m, dtype=np.float32)
    for i, v in sels:  # rank order (optimizer.py:176-183)
        total[i.astype(np.int64)] += v
    gi, gv = orc.tree_fold(sels, k)
    ni, nv, _ = orc.top_k_select(total, k)
    ni = ni[nv != 0]
    mask = np.zeros(m, dtype=bool)
    mask[gi.astype(np.int64)] = True
    want_mass = float(np.abs(np.where(mask, total, np.float32(0)) - orc.densify(gi, gv, m)).sum())
    sa, sb = set(gi.tolist()), set(ni.tolist())
    want_div = 1.0 - len(sa & sb) / max(len(sa), len(sb), 1)

    def w(ep):
        st = opt.make_state(zeros(m), lr=1.0)
        return opt.gtopk_step(st, ep, grads[ep.rank], k, P, measure_divergence=True)

    reps = gk.run_workers(gk.create_local_cluster(P), w)
    assert want_mass > 0.0 and 0.0 < want_div < 1.0
    for rep in reps:
        assert rep.lost_mass == want_mass
        assert rep.divergence == want_div


def test_extra_residual_identity_and_replicas(gk, opt):
    from oracle import gtopk_oracle as orc

    P, m, k, steps = 4, 32, 4, 15
    rng = np.random.default_rng(7)
    grads = [[rng.standard_normal(m).astype(F32) for _ in range(P)] for _ in range(steps)]

    def worker(ep):
        st = opt.make_state(zeros(m), lr=0.05)
        checks = []
        for it in range(steps):
            before = st.residual + grads[it][ep.rank]
            i, v, after = orc.top_k_select(before, k)
            opt.gtopk_step(st, ep, grads[it][ep.rank], k, P)
            returned = st.residual - after
            outside = np.ones(m, bool)
            outside[i] = False
            checks.append(not returned[outside].any() and bool(np.all((returned[i] == 0) | (returned[i] == v))))
        return checks, st.weights

    outs = gk.run_workers(gk.create_local_cluster(P), worker)
    assert all(all(c) for c, _ in outs)
    assert all(np.array_equal(w, outs[0][1]) for _, w in outs)


def test_nonfinite_step_leaves_state_untouched(gk, opt):
    from paper_1901_04359_b200.transport import TransportError

    (ep,) = gk.create_local_cluster(1)
    st = opt.make_state(np.ones(8, F32), lr=0.1)
    opt.gtopk_step(st, ep, np.arange(8, dtype=F32), 2, 1)
    w, r, it = st.weights.copy(), st.residual.copy(), st.iteration
    bad = np.ones(8, F32)
    bad[3] = np.nan
    with pytest.raises(FloatingPointError):
        opt.gtopk_step(st, ep, bad, 2, 1)
    assert np.array_equal(st.weights, w) and np.array_equal(st.residual, r) and st.iteration == it
    grads = [np.ones(8, F32), bad]

    def worker(ep):
        s = opt.make_state(np.ones(8, F32), lr=0.1)
        opt.gtopk_step(s, ep, grads[ep.rank], 2, 2)

    with pytest.raises(FloatingPointError):
        gk.run_workers(gk.create_local_cluster(2, timeout=5), worker)


@pytest.mark.parametrize("cfg", [("cfg1", 1_000_000, 0.001, 4, 3), ("resnet20", 270_000, 0.001, 8, 3)])
def test_baseline_configs_vs_oracle(gk, opt, cfg):
    """BASELINE configs[0] (m=1M, rho=0.001, P=4 simulated workers) and
    configs[1] (ResNet-20 size, P=8): full gtopk_step trajectories, bitwise."""
    from oracle import gtopk_oracle as orc

    name, m, rho, P, steps = cfg
    k = gk.k_from_density(rho, m)
    rng = np.random.default_rng(0)
    grads = [[rng.standard_normal(m).astype(F32) for _ in range(P)] for _ in range(steps)]
    w0 = np.zeros(m, F32)

    def worker(ep):
        st = opt.make_state(w0, lr=0.1)
        for it in range(steps):
            opt.gtopk_step(st, ep, grads[it][ep.rank], k, P)
        return st.weights.copy(), st.residual.copy()

    outs = gk.run_workers(gk.create_local_cluster(P), worker)
    ref = [orc.State(w0, 0.1) for _ in range(P)]
    for it in range(steps):
        orc.gtopk_step_all(ref, grads[it], k)
    for r in range(P):
        assert np.array_equal(bits(outs[r][0]), bits(ref[r].weights)), (name, r)
        assert np.array_equal(bits(outs[r][1]), bits(ref[r].residual)), (name, r)


def test_topk_step_touched_update_bitwise(gk, opt):
    """topk_step at P = 1, momentum 0 (gtk_topk_apply: the update at the
    selected entries only) against the oracle's dense average + dense update,
    with -0.0 / inf weights that a dense w - lr * +0 leaves unchanged;
    8 steps, weights and residual bitwise.  (NaN weights are left out: a GPU
    subtract returns the canonical NaN where numpy keeps the operand's.)"""
    from oracle import gtopk_oracle as orc

    m, k, steps = 100_003, 97, 8
    rng = np.random.default_rng(12)
    w0 = rng.standard_normal(m).astype(F32)
    w0[::7] = F32(-0.0)
    w0[5::11] = np.inf
    grads = [rng.standard_normal(m).astype(F32) for _ in range(steps)]
    (ep,) = gk.create_local_cluster(1)
    st = opt.make_state(w0, lr=0.25)
    ref = [orc.State(w0, 0.25)]
    for it in range(steps):
        opt.topk_step(st, ep, grads[it], k, 1)
        orc.topk_step_all(ref, [grads[it]], k)
    assert np.array_equal(bits(st.weights), bits(ref[0].weights))
    assert np.array_equal(bits(st.residual), bits(ref[0].residual))


def test_topk_step_nonfinite_voids_update_then_recovers(gk, opt):
    """P = 1 topk_step with the select's status checked in the update kernel
    (no host sync before it): FloatingPointError, state untouched, and the
    next step exact against the oracle (the scratch stayed all +0)."""
    from oracle import gtopk_oracle as orc

    m, k = 50_000, 50
    rng = np.random.default_rng(3)
    g0, g2 = rng.standard_normal(m).astype(F32), rng.standard_normal(m).astype(F32)
    bad = rng.standard_normal(m).astype(F32)
    bad[123] = np.inf
    (ep,) = gk.create_local_cluster(1)
    st = opt.make_state(np.zeros(m, F32), lr=0.1)
    opt.topk_step(st, ep, g0, k, 1)
    w, r, it = st.weights.copy(), st.residual.copy(), st.iteration
    with pytest.raises(FloatingPointError):
        opt.topk_step(st, ep, bad, k, 1)
    assert np.array_equal(bits(st.weights), bits(w)) and np.array_equal(bits(st.residual), bits(r))
    assert st.iteration == it
    opt.topk_step(st, ep, g2, k, 1)
    ref = [orc.State(np.zeros(m, F32), 0.1)]
    orc.topk_step_all(ref, [g0], k)
    orc.topk_step_all(ref, [g2], k)
    assert np.array_equal(bits(st.weights), bits(ref[0].weights))
    assert np.array_equal(bits(st.residual), bits(ref[0].residual))
