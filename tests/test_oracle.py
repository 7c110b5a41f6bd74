"""Pin the CPU oracle (oracle/gtopk_oracle.py) to the reference: golden vectors
produced by running the reference itself (tests/golden/make_golden.py) and the
reference's own known-answer tests (pkg/tests/test_sparse.py,
test_collectives.py, test_optimizer.py), restated.  CPU only."""

import hashlib

import numpy as np
import pytest

from conftest import load_golden
from oracle import gtopk_oracle as orc

F32 = np.float32


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits(a):
    return np.asarray(a, F32).view(np.uint32)


# ---- golden vectors --------------------------------------------------------


def test_select_golden_small():
    z = load_golden("select_small.npz")
    for c in range(int(z["n"])):
        i, v, r = orc.top_k_select(z[f"c{c}_g"], int(z[f"c{c}_k"]))
        assert np.array_equal(i, z[f"c{c}_idx"]), c
        assert np.array_equal(bits(v), bits(z[f"c{c}_val"])), c
        if f"c{c}_res" in z:
            assert np.array_equal(bits(r), bits(z[f"c{c}_res"])), c
        else:
            assert sha(r) == str(z[f"c{c}_res_sha"]), c


def test_select_golden_large_recipe():
    z = load_golden("select_large.npz")
    for name in ("cfg1", "resnet20"):
        m, k, P = int(z[f"{name}_m"]), int(z[f"{name}_k"]), int(z[f"{name}_P"])
        rng = np.random.default_rng(0)
        for r in range(P):
            g = rng.standard_normal(m).astype(F32)
            i, v, res = orc.top_k_select(g, k)
            assert np.array_equal(i, z[f"{name}_r{r}_idx"])
            assert np.array_equal(v, z[f"{name}_r{r}_val"])
            assert sha(res) == str(z[f"{name}_r{r}_res_sha"])


def test_top_op_golden():
    z = load_golden("top_op.npz")
    for c in range(int(z["n"])):
        k = int(z[f"c{c}_k"])
        oi, ov = orc.top_op(z[f"c{c}_a_idx"], z[f"c{c}_a_val"], z[f"c{c}_b_idx"], z[f"c{c}_b_val"], k)
        assert np.array_equal(oi, z[f"c{c}_o_idx"]), c
        assert np.array_equal(bits(ov), bits(z[f"c{c}_o_val"])), c


def test_allreduce_golden():
    z = load_golden("allreduce.npz")
    for c in range(int(z["n"])):
        P, m, k = int(z[f"c{c}_P"]), int(z[f"c{c}_m"]), int(z[f"c{c}_k"])
        lists = [(z[f"c{c}_in{r}_idx"], z[f"c{c}_in{r}_val"]) for r in range(P)]
        gi, gv = orc.gtopk_allreduce(lists, k)
        assert np.array_equal(gi, z[f"c{c}_g_idx"]), c
        assert np.array_equal(bits(gv), bits(z[f"c{c}_g_val"])), c
        assert np.array_equal(bits(orc.topk_allreduce(lists, m, P)), bits(z[f"c{c}_topk"])), c
        ring = orc.dense_ring_allreduce([z[f"c{c}_dense{r}"] for r in range(P)])
        assert np.array_equal(bits(ring[0]), bits(z[f"c{c}_ring"])), c
        # message counts of the tree + broadcast
        counts = orc.gtopk_message_counts(P)
        for r in range(P):
            st = z[f"c{c}_stats{r}"]
            assert counts[r]["msgs_sent"] == st[2] and counts[r]["msgs_recv"] == st[3], (c, r)


def test_steps_golden():
    z = load_golden("steps.npz")
    for c in range(int(z["n"])):
        algo = str(z[f"c{c}_algo"])
        if algo == "gtopk-naive":
            continue  # the oracle restates the tree path; naive is covered on the GPU side
        P, m, k = int(z[f"c{c}_P"]), int(z[f"c{c}_m"]), int(z[f"c{c}_k"])
        lr, mom, scaling = float(z[f"c{c}_lr"]), float(z[f"c{c}_mom"]), str(z[f"c{c}_scaling"])
        grads = z[f"c{c}_grads"]
        states = [orc.State(z[f"c{c}_winit"], lr, mom, scaling) for _ in range(P)]
        for it in range(grads.shape[0]):
            if algo == "gtopk":
                orc.gtopk_step_all(states, list(grads[it]), k)
            elif algo == "topk":
                orc.topk_step_all(states, list(grads[it]), k)
            else:
                orc.dense_step_all(states, list(grads[it]))
        for r in range(P):
            assert np.array_equal(bits(states[r].weights), bits(z[f"c{c}_w{r}"])), (c, algo, r)
            assert np.array_equal(bits(states[r].residual), bits(z[f"c{c}_res{r}"])), (c, algo, r)


def test_codec_golden():
    z = load_golden("codec.npz")
    for c in range(int(z["n"])):
        buf = orc.encode_sparse(z[f"c{c}_idx"], z[f"c{c}_val"])
        assert buf == z[f"c{c}_bytes"].tobytes()
        i, v = orc.decode_sparse(buf, int(z[f"c{c}_m"]))
        assert np.array_equal(i, z[f"c{c}_idx"]) and np.array_equal(bits(v), bits(z[f"c{c}_val"]))


# ---- the reference's known-answer tests, restated -----------------------------


def test_known_answers_select():
    i, v, r = orc.top_k_select([0.1, -0.5, 0.3, 0.05], 2)  # test_sparse.py:23-27
    assert i.tolist() == [1, 2] and v.tolist() == [F32(-0.5), F32(0.3)]
    assert np.array_equal(r, np.array([0.1, 0, 0, 0.05], F32))
    assert orc.top_k_select([2.0, -2.0, 1.0], 2)[0].tolist() == [0, 1]  # :36-38
    i, _, r = orc.top_k_select([1.0, -1.0, 1.0], 2)  # :40-44
    assert i.tolist() == [0, 1] and r[2] == F32(1.0)
    with pytest.raises(ValueError):
        orc.top_k_select([1.0, 2.0], 0)
    with pytest.raises(FloatingPointError):
        orc.top_k_select([1.0, np.nan], 1)


def test_known_answers_top_op():
    oi, ov = orc.top_op([1, 3], [0.5, -2.0], [1, 4], [0.6, 1.0], 2)  # test_sparse.py:87-91
    assert oi.tolist() == [1, 3] and ov.tolist() == [F32(0.5) + F32(0.6), F32(-2.0)]
    oi, ov = orc.top_op([0], [1.0], [0], [-1.0], 1)  # cancellation -> empty
    assert oi.size == 0
    oi, ov = orc.top_op([0, 5], [1.0, -3.0], [], [], 2)
    assert oi.tolist() == [0, 5]


def test_known_answers_density():
    assert orc.k_from_density(0.001, 100) == 1
    assert orc.k_from_density(0.01, 256) == 3
    assert orc.k_from_density(0.001, 25_000_000) == 25_000
    assert orc.k_from_density(1.0, 7) == 7
    assert orc.k_from_density(0.001, 25_600_000) == 25_600


def test_tree_fold_p2_exchange():
    # test_collectives.py:204-210
    gi, gv = orc.gtopk_allreduce([([1, 3], [0.5, -2.0]), ([1, 4], [0.6, 1.0])], 2)
    assert gi.tolist() == [1, 3] and gv.tolist() == [F32(0.5) + F32(0.6), F32(-2.0)]


def test_gtopk_step_hand_trace():
    # test_optimizer.py:167-186
    states = [orc.State(np.zeros(4, F32), 1.0) for _ in range(2)]
    orc.gtopk_step_all(states, [np.array([1.0, 0, 0, 0], F32), np.array([0, 2.0, 0, 0], F32)], 1)
    for st in states:
        assert np.array_equal(st.weights, np.array([0, -1.0, 0, 0], F32))
    assert np.array_equal(states[0].residual, np.array([1, 0, 0, 0], F32))
    assert not states[1].residual.any()


def test_butterfly_equals_tree_fold():
    """The recursive-doubling butterfly used by the NVLink kernel for P = 2^n
    gives every rank the tree fold bitwise (⊤ is commutative)."""
    rng = np.random.default_rng(99)
    for P in (2, 4, 8, 16):
        for _ in range(40):
            m = int(rng.integers(8, 200))
            k = int(rng.integers(1, min(12, m) + 1))
            lists = [orc.top_k_select(rng.integers(-3, 4, m).astype(F32) if rng.random() < 0.5
                                      else rng.standard_normal(m).astype(F32), k)[:2] for _ in range(P)]
            want = orc.tree_fold(lists, k)
            acc = [(np.asarray(i), np.asarray(v)) for i, v in lists]
            for j in range(orc.ceil_log2(P)):
                acc = [orc.top_op(*acc[r ^ (1 << j)], *acc[r], k) for r in range(P)]
            for r in range(P):
                assert np.array_equal(acc[r][0], want[0])
                assert np.array_equal(bits(acc[r][1]), bits(want[1]))
