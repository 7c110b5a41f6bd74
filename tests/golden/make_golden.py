"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the reference package `gtopk` (pure Python + numpy) and records
inputs/outputs of the hot-path functions into `tests/golden/*.npz`.  The
fixtures are committed; nothing at test/bench time reads /root/reference.

Inputs are either stored verbatim (small cases) or as a numpy
`default_rng(seed)` recipe (large cases; PCG64 + standard_normal streams are
stable across numpy >= 1.17), with the expected outputs stored verbatim.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from gtopk import collectives, optimizer, sparse, transport  # noqa: E402  (the reference)

F32 = np.float32


def adversarial(kind: str, rng, m: int) -> np.ndarray:
    """Input families from SURVEY.md §8(d): ties, ±const, subnormals, signed zeros."""
    if kind == "normal":
        return rng.standard_normal(m).astype(F32)
    if kind == "int":
        return rng.integers(-3, 4, m).astype(F32)
    if kind == "pmconst":
        return (np.where(rng.random(m) < 0.5, -1.0, 1.0) * 0.75).astype(F32)
    if kind == "subnormal":
        return (rng.standard_normal(m) * 1e-40).astype(F32)
    if kind == "zeros":
        z = np.zeros(m, F32)
        z[rng.random(m) < 0.5] = -0.0
        return z
    if kind == "mixed":
        g = rng.standard_normal(m).astype(F32)
        g[rng.random(m) < 0.3] = 0.0
        g[rng.random(m) < 0.1] = -0.0
        g[rng.random(m) < 0.2] = 2.0
        g[rng.random(m) < 0.05] = -2.0
        return g
    if kind == "layered":  # structured magnitudes, like per-layer gradient scales
        g = rng.standard_normal(m).astype(F32)
        cut = np.linspace(0, m, 6).astype(int)
        for j in range(5):
            g[cut[j]:cut[j + 1]] *= F32(10.0 ** (j - 2))
        return g
    raise ValueError(kind)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_select():
    rng = np.random.default_rng(2024)
    cases = {}
    n = 0
    for kind in ("normal", "int", "pmconst", "subnormal", "zeros", "mixed", "layered"):
        for m in (1, 2, 7, 64, 1000, 4099, 20000):
            for kfrac in (0.0, 0.01, 0.3, 1.0):
                k = max(1, min(m, int(round(kfrac * m)) or 1))
                g = adversarial(kind, rng, m)
                sel, res = sparse.top_k_select(g, k)
                cases[f"c{n}_g"] = g
                cases[f"c{n}_k"] = np.array(k)
                cases[f"c{n}_idx"] = sel.indices
                cases[f"c{n}_val"] = sel.values
                if m <= 1000:
                    cases[f"c{n}_res"] = res
                else:
                    cases[f"c{n}_res_sha"] = np.array(sha(res))
                n += 1
    cases["n"] = np.array(n)
    np.savez_compressed(os.path.join(HERE, "select_small.npz"), **cases)


def gen_select_large():
    """BASELINE configs' selection, inputs by recipe (cli.py:250-251 draw order)."""
    out = {}
    for name, m, rho, P in (("cfg1", 1_000_000, 0.001, 4), ("resnet20", 270_000, 0.001, 2)):
        rng = np.random.default_rng(0)
        k = sparse.k_from_density(rho, m)
        for r in range(P):
            g = rng.standard_normal(m).astype(F32)
            sel, res = sparse.top_k_select(g, k)
            out[f"{name}_r{r}_idx"] = sel.indices
            out[f"{name}_r{r}_val"] = sel.values
            out[f"{name}_r{r}_res_sha"] = np.array(sha(res))
        out[f"{name}_m"] = np.array(m)
        out[f"{name}_k"] = np.array(k)
        out[f"{name}_P"] = np.array(P)
    np.savez_compressed(os.path.join(HERE, "select_large.npz"), **out)


def gen_top_op():
    rng = np.random.default_rng(77)
    cases = {}
    n = 0
    for trial in range(400):
        m = int(rng.integers(1, 200))
        k = int(rng.integers(1, m + 1))
        ka = int(rng.integers(0, k + 1))
        kb = int(rng.integers(0, k + 1))
        kind = ["normal", "int", "pmconst", "mixed"][trial % 4]
        ga = adversarial(kind, rng, m)
        gb = adversarial(kind, rng, m)
        if trial % 7 == 0:  # force cancellation on shared indices
            gb = -ga.copy()
        a = sparse.top_k_select(ga, ka)[0] if ka else sparse.SparseVector.empty(m)
        b = sparse.top_k_select(gb, kb)[0] if kb else sparse.SparseVector.empty(m)
        o = sparse.top_op(a, b, k)
        for nm, s in (("a", a), ("b", b), ("o", o)):
            cases[f"c{n}_{nm}_idx"] = s.indices
            cases[f"c{n}_{nm}_val"] = s.values
        cases[f"c{n}_m"] = np.array(m)
        cases[f"c{n}_k"] = np.array(k)
        n += 1
    # pathological: overflow to inf, then inf + -inf = NaN (top_op has no finiteness check)
    big = F32(3e38)
    a = sparse.SparseVector(8, [1, 2, 3, 5], [big, -big, 1.0, np.inf])
    b = sparse.SparseVector(8, [1, 2, 4, 5], [big, -big, -2.0, -np.inf])
    for k in (1, 2, 3, 4, 5):
        o = sparse.top_op(a, b, k)
        for nm, s in (("a", a), ("b", b), ("o", o)):
            cases[f"c{n}_{nm}_idx"] = s.indices
            cases[f"c{n}_{nm}_val"] = s.values
        cases[f"c{n}_m"] = np.array(8)
        cases[f"c{n}_k"] = np.array(k)
        n += 1
    cases["n"] = np.array(n)
    np.savez_compressed(os.path.join(HERE, "top_op.npz"), **cases)


def gen_allreduce():
    """gtopk_allreduce / topk_allreduce / dense ring run through the reference's
    own in-process cluster (create_local_cluster + run_workers)."""
    cases = {}
    n = 0
    for P in (1, 2, 3, 4, 5, 8, 16):
        rng = np.random.default_rng(500 + P)
        for trial in range(6):
            m = int(rng.integers(4, 300))
            k = int(rng.integers(1, min(40, m) + 1))
            kind = ["normal", "int", "mixed"][trial % 3]
            dense_in = [adversarial(kind, rng, m) for _ in range(P)]
            sparse_in = [sparse.top_k_select(adversarial(kind, rng, m), k)[0] for _ in range(P)]

            def worker(ep):
                before = ep.stats.snapshot()
                g = collectives.gtopk_allreduce(ep, sparse_in[ep.rank], k, P)
                d = ep.stats.snapshot().delta(before)
                t = collectives.topk_allreduce(ep, sparse_in[ep.rank], P)
                r = collectives.dense_ring_allreduce(ep, dense_in[ep.rank])
                return g, d, t, r

            outs = transport.run_workers(transport.create_local_cluster(P), worker)
            g0 = outs[0][0].global_topk
            for r in range(P):
                assert outs[r][0].global_topk == g0
                cases[f"c{n}_in{r}_idx"] = sparse_in[r].indices
                cases[f"c{n}_in{r}_val"] = sparse_in[r].values
                cases[f"c{n}_dense{r}"] = dense_in[r]
                d = outs[r][1]
                cases[f"c{n}_stats{r}"] = np.array(
                    [d.bytes_sent, d.bytes_recv, d.msgs_sent, d.msgs_recv], dtype=np.int64
                )
            cases[f"c{n}_g_idx"] = g0.indices
            cases[f"c{n}_g_val"] = g0.values
            cases[f"c{n}_topk"] = outs[0][2]
            cases[f"c{n}_ring"] = outs[0][3]
            cases[f"c{n}_P"] = np.array(P)
            cases[f"c{n}_m"] = np.array(m)
            cases[f"c{n}_k"] = np.array(k)
            n += 1
    cases["n"] = np.array(n)
    np.savez_compressed(os.path.join(HERE, "allreduce.npz"), **cases)


def gen_steps():
    """Multi-step optimizer trajectories through the reference's STEP_FNS."""
    cases = {}
    n = 0
    configs = [
        ("gtopk", 1, 16, 3, 0.3, 0.0, "average"),
        ("gtopk", 2, 40, 4, 0.1, 0.0, "average"),
        ("gtopk", 4, 64, 5, 0.05, 0.0, "average"),
        ("gtopk", 4, 64, 5, 0.05, 0.0, "sum"),
        ("gtopk", 2, 33, 3, 0.1, 0.9, "average"),
        ("gtopk", 3, 50, 4, 0.2, 0.0, "average"),
        ("gtopk", 8, 128, 6, 0.01, 0.0, "average"),
        ("topk", 4, 48, 5, 0.1, 0.0, "average"),
        ("topk", 2, 20, 20, 0.1, 0.5, "average"),
        ("dense", 4, 30, 0, 0.1, 0.0, "average"),
        ("gtopk-naive", 4, 40, 4, 0.1, 0.0, "average"),
    ]
    for algo, P, m, k, lr, mom, scaling in configs:
        rng = np.random.default_rng(900 + n)
        steps = 8
        grads = [[rng.standard_normal(m).astype(F32) for _ in range(P)] for _ in range(steps)]
        w0 = rng.standard_normal(m).astype(F32)
        fn = optimizer.STEP_FNS[algo]

        def worker(ep):
            st = optimizer.make_state(w0, lr=lr, momentum=mom, update_scaling=scaling)
            sel_k = []
            for it in range(steps):
                if algo == "dense":
                    rep = fn(st, ep, grads[it][ep.rank], P)
                else:
                    rep = fn(st, ep, grads[it][ep.rank], k, P)
                sel_k.append(rep.selected_k)
            return st.weights.copy(), st.residual.copy(), sel_k

        outs = transport.run_workers(transport.create_local_cluster(P), worker)
        cases[f"c{n}_algo"] = np.array(algo)
        cases[f"c{n}_P"] = np.array(P)
        cases[f"c{n}_m"] = np.array(m)
        cases[f"c{n}_k"] = np.array(k)
        cases[f"c{n}_lr"] = np.array(lr)
        cases[f"c{n}_mom"] = np.array(mom)
        cases[f"c{n}_scaling"] = np.array(scaling)
        cases[f"c{n}_winit"] = w0
        cases[f"c{n}_grads"] = np.array(grads)
        for r in range(P):
            cases[f"c{n}_w{r}"] = outs[r][0]
            cases[f"c{n}_res{r}"] = outs[r][1]
            cases[f"c{n}_selk{r}"] = np.array(outs[r][2])
        n += 1
    cases["n"] = np.array(n)
    np.savez_compressed(os.path.join(HERE, "steps.npz"), **cases)


def gen_codec():
    rng = np.random.default_rng(31)
    cases = {}
    for n, m in enumerate((1, 5, 100)):
        s = sparse.top_k_select(rng.standard_normal(m).astype(F32), max(1, m // 3))[0]
        cases[f"c{n}_idx"] = s.indices
        cases[f"c{n}_val"] = s.values
        cases[f"c{n}_m"] = np.array(m)
        cases[f"c{n}_bytes"] = np.frombuffer(transport.encode_sparse(s), dtype=np.uint8)
    cases["n"] = np.array(3)
    np.savez_compressed(os.path.join(HERE, "codec.npz"), **cases)


if __name__ == "__main__":
    gen_select()
    gen_select_large()
    gen_top_op()
    gen_allreduce()
    gen_steps()
    gen_codec()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
