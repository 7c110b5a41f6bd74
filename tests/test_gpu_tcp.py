"""GPU parity of the TCP backend's host-staged collectives (tcp.py): P ranks
as threads of one process on cuda:0, linked by a real 127.0.0.1 TCP mesh in
the reference's wire format, each rank's merges / accumulations on the GPU.
Compared bitwise with the oracle (collectives.py:88-219, optimizer.py:199-252)."""

import threading

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA GPU")]

F32 = np.float32


def bits(a):
    return np.asarray(a, F32).view(np.uint32)


def tcp_mesh(P, timeout=60.0):
    import socket

    from paper_1901_04359_b200 import tcp

    socks = [socket.socket() for _ in range(P)]
    for s in socks:
        s.bind(("127.0.0.1", 0))
    addrs = [("127.0.0.1", s.getsockname()[1]) for s in socks]
    for s in socks:
        s.close()
    cfg = tcp.ClusterConfig(P, "tcp", addrs, timeout)
    eps = [None] * P
    ts = [threading.Thread(target=lambda r=r: eps.__setitem__(r, tcp.connect_tcp_cluster(cfg, r, "cuda:0")))
          for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert all(e is not None for e in eps)
    return eps


def run(eps, fn):
    import paper_1901_04359_b200 as gk

    try:
        return gk.run_workers(eps, fn)
    finally:
        for ep in eps:
            ep.close()


def sparse_lists(rng, P, m, k):
    import paper_1901_04359_b200 as gk

    out = []
    for _ in range(P):
        n = int(rng.integers(0, k + 1))
        idx = np.sort(rng.choice(m, n, replace=False)).astype(np.uint64)
        val = rng.standard_normal(n).astype(F32)
        val[rng.random(n) < 0.1] = F32(0.5)  # ties across ranks
        out.append(gk.SparseVector(m, idx, val))
    return out


@pytest.mark.parametrize("P", [2, 3, 4, 5])
def test_tcp_gtopk_allreduce_vs_oracle(P):
    from oracle import gtopk_oracle as orc

    rng = np.random.default_rng(P)
    m, k = 50_000, 300
    lists = sparse_lists(rng, P, m, k)
    ref_i, ref_v = orc.gtopk_allreduce([(s.indices, s.values) for s in lists], k)

    from paper_1901_04359_b200 import collectives as coll

    outs = run(tcp_mesh(P), lambda ep: coll.gtopk_allreduce(ep, lists[ep.rank], k))
    for r, res in enumerate(outs):
        g = res.global_topk
        assert np.array_equal(np.asarray(g.indices, np.uint64), ref_i), r
        assert np.array_equal(bits(g.values), bits(ref_v)), r


@pytest.mark.parametrize("P", [2, 3, 4])
def test_tcp_topk_and_dense_allreduce_vs_oracle(P):
    from oracle import gtopk_oracle as orc
    from paper_1901_04359_b200 import collectives as coll

    rng = np.random.default_rng(10 + P)
    m, k = 20_001, 200
    lists = sparse_lists(rng, P, m, k)
    dense = [rng.standard_normal(m).astype(F32) for _ in range(P)]
    ref_t = orc.topk_allreduce([(s.indices, s.values) for s in lists], m, P)
    ref_d = orc.dense_ring_allreduce(dense)

    outs = run(tcp_mesh(P), lambda ep: (coll.topk_allreduce(ep, lists[ep.rank]),
                                        coll.dense_ring_allreduce(ep, dense[ep.rank])))
    for r, (t, d) in enumerate(outs):
        assert np.array_equal(bits(t), bits(ref_t)), r
        assert np.array_equal(bits(d), bits(ref_d[r])), r


@pytest.mark.parametrize("P,momentum", [(4, 0.0), (3, 0.0), (2, 0.9)])
def test_tcp_gtopk_step_trajectory_vs_oracle(P, momentum):
    """gtopk_step over the TCP mesh (select on the GPU, host-staged tree +
    broadcast, K3 on the GPU), 4 steps, weights and residual bitwise."""
    from oracle import gtopk_oracle as orc
    from paper_1901_04359_b200 import optimizer as opt

    m, k, steps = 30_000, 60, 4
    rng = np.random.default_rng(7)
    grads = [[rng.standard_normal(m).astype(F32) for _ in range(P)] for _ in range(steps)]
    w0 = rng.standard_normal(m).astype(F32)

    def worker(ep):
        st = opt.make_state(w0, lr=0.05, momentum=momentum)
        for it in range(steps):
            opt.gtopk_step(st, ep, grads[it][ep.rank], k, P)
        return st.weights.copy(), st.residual.copy()

    outs = run(tcp_mesh(P), worker)
    ref = [orc.State(w0, 0.05, momentum) for _ in range(P)]
    for it in range(steps):
        orc.gtopk_step_all(ref, grads[it], k)
    for r in range(P):
        assert np.array_equal(bits(outs[r][0]), bits(ref[r].weights)), r
        assert np.array_equal(bits(outs[r][1]), bits(ref[r].residual)), r


def test_tcp_local_backend_equivalence_bitwise():
    """reference pkg/tests/test_transport.py:255-298: identical inputs through
    the in-process and the TCP backends give identical results for every
    collective -- and identical byte / message accounting."""
    import paper_1901_04359_b200 as gk
    from paper_1901_04359_b200 import collectives as coll

    rng = np.random.default_rng(21)
    P, m, k = 3, 24, 3
    sparse_in = sparse_lists(rng, P, m, k)
    dense_in = [rng.standard_normal(m).astype(F32) for _ in range(P)]

    def all_collectives(ep):
        r = ep.rank
        out = (coll.gtopk_allreduce(ep, sparse_in[r], k, P), coll.topk_allreduce(ep, sparse_in[r], P),
               coll.dense_ring_allreduce(ep, dense_in[r]))
        st = ep.stats
        return out, (st.bytes_sent, st.bytes_recv, st.msgs_sent, st.msgs_recv)

    local = gk.run_workers(gk.create_local_cluster(P), all_collectives)
    over_tcp = run(tcp_mesh(P), all_collectives)
    for r in range(P):
        (g_t, t_t, d_t), s_t = over_tcp[r]
        (g_l, t_l, d_l), s_l = local[r]
        assert g_t.global_topk == g_l.global_topk
        assert np.array_equal(bits(t_t), bits(t_l))
        assert np.array_equal(bits(d_t), bits(d_l))
        assert s_t == s_l, (r, s_t, s_l)


@pytest.mark.parametrize("P,momentum", [(3, 0.0), (2, 0.9)])
def test_tcp_topk_step_trajectory_vs_oracle(P, momentum):
    """topk_step over the TCP mesh: momentum 0 takes the touched-entry update
    (gtk_topk_apply), momentum 0.9 the dense one; 4 steps bitwise."""
    from oracle import gtopk_oracle as orc
    from paper_1901_04359_b200 import optimizer as opt

    m, k, steps = 30_000, 60, 4
    rng = np.random.default_rng(8)
    grads = [[rng.standard_normal(m).astype(F32) for _ in range(P)] for _ in range(steps)]
    w0 = rng.standard_normal(m).astype(F32)

    def worker(ep):
        st = opt.make_state(w0, lr=0.05, momentum=momentum)
        for it in range(steps):
            opt.topk_step(st, ep, grads[it][ep.rank], k, P)
        return st.weights.copy(), st.residual.copy()

    outs = run(tcp_mesh(P), worker)
    ref = [orc.State(w0, 0.05, momentum) for _ in range(P)]
    for it in range(steps):
        orc.topk_step_all(ref, grads[it], k)
    for r in range(P):
        assert np.array_equal(bits(outs[r][0]), bits(ref[r].weights)), r
        assert np.array_equal(bits(outs[r][1]), bits(ref[r].residual)), r
