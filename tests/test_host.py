"""Host-side logic on CPU: data types, wire codec, schedules, accounting,
the in-process cluster's byte transport and error propagation.  Mirrors the
reference's test_sparse.py / test_transport.py / test_collectives.py host
checks; no kernel launches."""

import threading

import numpy as np
import pytest

import paper_1901_04359_b200 as gk
from paper_1901_04359_b200 import collectives as coll
from paper_1901_04359_b200 import optimizer as opt
from paper_1901_04359_b200.transport import ProtocolError, TransportError
from conftest import load_golden
from oracle import gtopk_oracle as orc

F32 = np.float32


def sv(dim, pairs):
    return gk.SparseVector.from_pairs(dim, pairs)


# ---- types ------------------------------------------------------------------


def test_sparse_vector_semantics():
    s = sv(6, [(3, -2.0), (1, 0.5)])
    assert s.indices.dtype == np.uint64 and s.values.dtype == np.float32
    assert s.indices.tolist() == [1, 3] and s.nnz == 2
    assert s == sv(6, [(1, 0.5), (3, -2.0)])
    assert s != sv(7, [(1, 0.5), (3, -2.0)])
    s.validate()
    with pytest.raises(ValueError):
        gk.SparseVector(4, [2, 1], [1.0, 1.0]).validate()
    with pytest.raises(ValueError):
        gk.SparseVector(2, [0, 5], [1.0, 1.0]).validate()
    assert gk.SparseVector.empty(3).nnz == 0


def test_index_mask():
    a = gk.IndexMask.from_indices(5, [0, 2, 4])
    b = gk.IndexMask.from_indices(5, [2, 3, 4])
    assert (~a).indices.tolist() == [1, 3]
    assert (a & b).indices.tolist() == [2, 4]
    assert a.count == 3 and a.flags.tolist() == [True, False, True, False, True]
    with pytest.raises(ValueError):
        gk.IndexMask.from_indices(2, [2])
    with pytest.raises(ValueError):
        gk.IndexMask.from_indices(2, [0]) & gk.IndexMask.from_indices(3, [0])
    g = [1.0, 2.0, 3.0]
    assert np.array_equal(gk.masked_extract(g, gk.IndexMask.from_indices(3, [1])), np.array([0, 2, 0], F32))
    with pytest.raises(ValueError):
        gk.masked_extract([1.0, 2.0], gk.IndexMask.from_indices(3, [0]))


def test_densify_host_and_density():
    assert np.array_equal(gk.densify(sv(3, [(1, 2.0)])), np.array([0, 2, 0], F32))
    assert gk.k_from_density(0.001, 100) == 1
    assert gk.k_from_density(0.01, 256) == 3
    assert gk.k_from_density(0.001, 25_600_000) == 25_600
    with pytest.raises(ValueError):
        gk.k_from_density(0.0, 10)
    with pytest.raises(ValueError):
        gk.as_dense(np.zeros((2, 2)))


# ---- codec ------------------------------------------------------------------


def test_codec_golden_bytes():
    z = load_golden("codec.npz")
    for c in range(int(z["n"])):
        s = gk.SparseVector(int(z[f"c{c}_m"]), z[f"c{c}_idx"], z[f"c{c}_val"])
        buf = gk.encode_sparse(s)
        assert buf == z[f"c{c}_bytes"].tobytes()
        assert gk.decode_sparse(buf, s.dim) == s


def test_codec_errors():
    buf = gk.encode_sparse(sv(10, [(1, 1.0), (4, 2.0)]))
    with pytest.raises(ProtocolError):
        gk.decode_sparse(buf[:5], 10)
    with pytest.raises(ProtocolError):
        gk.decode_sparse(b"\x00" * 12, 10)
    with pytest.raises(ProtocolError):
        gk.decode_sparse(buf + b"\x00", 10)
    with pytest.raises(ProtocolError):
        gk.decode_sparse(buf, 3)  # index out of range
    bad = gk.encode_sparse(gk.SparseVector(10, [4, 1], [1.0, 2.0]))
    with pytest.raises(ProtocolError):
        gk.decode_sparse(bad, 10)


# ---- schedules / accounting -------------------------------------------------


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8, 16])
def test_tree_schedule_matches_reference_message_counts(P):
    want = orc.gtopk_message_counts(P)
    for r in range(P):
        steps = coll.tree_schedule(r, P)
        assert len(steps) == 2 * coll.ceil_log2(P)
        assert sum(s >= 0 for s, _, _ in steps) == want[r]["msgs_sent"]
        assert sum(v >= 0 for _, v, _ in steps) == want[r]["msgs_recv"]


@pytest.mark.parametrize("P", [1, 2, 3, 5, 8, 16])
def test_tree_schedule_executes_to_tree_fold(P):
    """Run every rank's steps in lock-step with the oracle's ⊤: all ranks end
    with the reference tree fold."""
    rng = np.random.default_rng(P)
    for _ in range(20):
        m = int(rng.integers(8, 100))
        k = int(rng.integers(1, 9))
        lists = [orc.top_k_select(rng.standard_normal(m).astype(F32), k)[:2] for _ in range(P)]
        want = orc.tree_fold(lists, k)
        acc = [tuple(x) for x in lists]
        scheds = [coll.tree_schedule(r, P) for r in range(P)]
        for j in range(len(scheds[0]) if P > 1 else 0):
            inbox = {}
            for r in range(P):
                s, _, _ = scheds[r][j]
                if s >= 0:
                    inbox[s] = acc[r]
            new = list(acc)
            for r in range(P):
                _, src, merge = scheds[r][j]
                if src >= 0:
                    assert src in [q for q in range(P) if scheds[q][j][0] == r]
                    new[r] = orc.top_op(*inbox[r], *acc[r], k) if merge else inbox[r]
            acc = new
        for r in range(P):
            assert np.array_equal(acc[r][0], want[0]) and np.array_equal(acc[r][1], want[1])


def test_butterfly_schedule():
    assert coll.butterfly_schedule(5, 8) == [(4, 4, 1), (7, 7, 1), (1, 1, 1)]
    with pytest.raises(ValueError):
        coll.butterfly_schedule(0, 6)


def test_comm_rounds_and_predicted_bytes():
    assert coll.comm_rounds("gtopk", 8) == 6
    assert coll.comm_rounds("dense", 4) == 6
    assert coll.comm_rounds("topk", 4) == 3
    assert coll.comm_rounds("bcast", 5) == 3
    assert coll.comm_rounds("gtopk", 1) == 0
    assert coll.ceil_log2(8) == 3 and coll.ceil_log2(5) == 3 and coll.ceil_log2(1) == 0
    assert coll.predicted_bytes("dense", 4, 64, 0) == 2 * 3 * 16 * 4
    assert coll.predicted_bytes("topk", 4, 64, 5) == 3 * (12 + 12 * 5)
    with pytest.raises(ValueError):
        coll.predicted_bytes("gtopk", 4, 64, 5)
    row = coll.CollectiveStats("gtopk", 4, 64, 5, 0, 10, 20, 2, 4, 1.5).csv_row()
    assert row == "gtopk,4,64,5,0,10,20,2,4,1.500000"


def test_transport_stats_lazy_counts():
    st = gk.TransportStats()
    st.add_sparse(5, sent=True)
    st.add_sparse(0, sent=False)
    assert st.msgs_sent == 1 and st.msgs_recv == 1
    assert st.bytes_sent == 72 and st.bytes_recv == 12
    d = st.snapshot().delta(gk.TransportStats())
    assert d.bytes_sent == 72


# ---- in-process byte transport (transport.py semantics) ----------------------


def test_local_cluster_send_recv_barrier():
    eps = gk.create_local_cluster(4, timeout=5)

    def worker(ep):
        ep.barrier()
        right, left = (ep.rank + 1) % 4, (ep.rank - 1) % 4
        ep.send(right, 7, f"hi{ep.rank}".encode())
        got = ep.recv(left, 7)
        ep.barrier()
        return got

    assert gk.run_workers(eps, worker) == [b"hi3", b"hi0", b"hi1", b"hi2"]


def test_local_cluster_errors():
    (ep,) = gk.create_local_cluster(1)
    with pytest.raises(ValueError):
        ep.send(0, 1, b"x")  # self
    eps = gk.create_local_cluster(2, timeout=0.3)
    with pytest.raises(ValueError):
        eps[0].send(5, 1, b"x")
    with pytest.raises(ValueError):
        eps[0].send(1, -1, b"x")
    with pytest.raises(TransportError):
        eps[0].recv(1, 3)  # timeout
    with pytest.raises(ValueError):
        gk.create_local_cluster(0)


def test_run_workers_prefers_root_cause():
    eps = gk.create_local_cluster(3, timeout=5)

    def worker(ep):
        if ep.rank == 2:
            raise KeyError("boom")
        ep.recv((ep.rank + 1) % 3, 1)  # blocks until the abort

    with pytest.raises(KeyError):
        gk.run_workers(eps, worker)


def test_byte_allgather_and_bcast():
    eps = gk.create_local_cluster(4)
    outs = gk.run_workers(eps, lambda ep: coll.allgather(ep, f"from-{ep.rank}".encode()))
    assert all(o == [f"from-{r}".encode() for r in range(4)] for o in outs)
    eps = gk.create_local_cluster(3)
    outs = gk.run_workers(eps, lambda ep: coll.allgather(ep, b"x" * (ep.rank * 10)))
    assert all(o == [b"", b"x" * 10, b"x" * 20] for o in outs)
    eps = gk.create_local_cluster(8)

    def bc(ep):
        before = ep.stats.snapshot()
        out = coll.binomial_bcast(ep, 0, b"data" if ep.rank == 0 else None)
        return out, ep.stats.snapshot().delta(before)

    outs = gk.run_workers(eps, bc)
    assert all(o == b"data" for o, _ in outs)
    assert outs[0][1].msgs_sent == 3 and sum(d.msgs_sent for _, d in outs) == 7
    eps = gk.create_local_cluster(6)
    outs = gk.run_workers(eps, lambda ep: coll.binomial_bcast(ep, 2, b"rooted" if ep.rank == 2 else None))
    assert all(o == b"rooted" for o in outs)
    (ep,) = gk.create_local_cluster(1)
    assert coll.allgather(ep, b"solo") == [b"solo"]
    assert coll.binomial_bcast(ep, 0, b"p") == b"p"


def test_group_rendezvous_abort():
    """A failing rank aborts the device-group rendezvous of the others."""
    g = gk.transport.LocalDeviceGroup(2, device="cpu", timeout=5)
    errs = []

    def waiter():
        try:
            g.run(1, None, lambda ops: None)
        except TransportError as exc:
            errs.append(exc)

    t = threading.Thread(target=waiter)
    t.start()
    g.abort()
    t.join(5)
    assert errs and "aborted" in str(errs[0])


# ---- optimizer host-side pieces ------------------------------------------------


def test_density_schedule():
    sched = opt.DensitySchedule()
    assert [opt.density_at(sched, e) for e in range(6)] == [0.25, 0.0725, 0.015, 0.004, 0.001, 0.001]
    assert opt.density_at(opt.DensitySchedule(warmup=(), terminal=0.05), 100) == 0.05
    with pytest.raises(ValueError):
        opt.density_at(sched, -1)
    assert opt.DEFAULT_WARMUP == (0.25, 0.0725, 0.015, 0.004)


def test_make_state_validation():
    st = opt.make_state(np.ones(4, F32), lr=0.1)
    assert st.weights.tolist() == [1, 1, 1, 1] and not st.residual.any() and st.iteration == 0
    with pytest.raises(ValueError):
        opt.make_state(np.ones(4, F32), lr=0.1, momentum=1.0)
    with pytest.raises(ValueError):
        opt.make_state(np.ones(4, F32), lr=0.1, update_scaling="mean")
    with pytest.raises(ValueError):
        opt.OptimizerState(np.ones(4, F32), np.zeros(3, F32), 0.1)
    assert set(opt.STEP_FNS) == {"dense", "topk", "gtopk", "gtopk-naive"}


# ---- drop-in surface ----------------------------------------------------------

# reference pkg/src/gtopk/__init__.py:3-44, minus the out-of-scope modules
# (cost_model, models: SURVEY.md §2) and the TCP mesh (ClusterConfig,
# connect_tcp_cluster: SURVEY.md §8(f) row 4)
REFERENCE_HOT_PATH_EXPORTS = [
    "CollectiveStats", "GTopKResult", "allgather", "binomial_bcast", "dense_ring_allreduce", "gtopk_allreduce",
    "topk_allreduce", "DensitySchedule", "OptimizerState", "StepReport", "dense_step", "density_at",
    "gtopk_naive_step", "gtopk_step", "make_state", "topk_step", "IndexMask", "SparseVector", "densify",
    "k_from_density", "masked_extract", "top_k_select", "top_op", "Endpoint", "ProtocolError", "TransportError",
    "create_local_cluster", "decode_sparse", "encode_sparse", "run_workers",
]
OUT_OF_SCOPE = {"CostParams", "FitResult", "fit_alpha_beta", "scaling_efficiency", "t_dense", "t_gtopk", "t_topk",
                "SyntheticDataset", "ToyModel", "gen_dataset", "grad", "shard_batches", "ClusterConfig",
                "connect_tcp_cluster"}


def test_top_level_exports_every_reference_hot_path_name():
    import paper_1901_04359_b200 as gtopk

    for name in REFERENCE_HOT_PATH_EXPORTS:
        assert hasattr(gtopk, name), name
        assert name in dir(gtopk) and name in gtopk.__all__, name
    # the lazily resolved names are the submodules' own objects
    assert gtopk.gtopk_step is opt.gtopk_step and gtopk.gtopk_allreduce is coll.gtopk_allreduce
    assert gtopk.STEP_FNS["gtopk"] is opt.gtopk_step
    with pytest.raises(AttributeError):
        gtopk.no_such_name  # noqa: B018


def test_export_list_matches_reference_init():
    """The list above is the reference's own __init__ (checked where the
    reference checkout exists, i.e. in the build container)."""
    import ast
    import os

    path = "/root/reference/pkg/src/gtopk/__init__.py"
    if not os.path.exists(path):
        pytest.skip("reference checkout not present")
    names = set()
    for node in ast.parse(open(path).read()).body:
        if isinstance(node, ast.ImportFrom):
            names |= {a.name for a in node.names}
    assert names == set(REFERENCE_HOT_PATH_EXPORTS) | OUT_OF_SCOPE
