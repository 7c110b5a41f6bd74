"""CPU oracle for the gTop-k hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain numpy restatement of the reference algorithm
(`/root/reference/pkg/src/gtopk`, arXiv 1901.04359 desk reproduction).  It is
the *checker*: only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` leg may import it.  The product package
(`paper_1901_04359_b200`) never imports or calls anything in here; its CUDA
path fails loudly when the native library is missing.

Parity pinning: every function below is checked against golden vectors that
were produced by importing the reference itself (`tests/golden/make_golden.py`
writes `tests/golden/*.npz`; `tests/test_oracle.py` replays them), plus the
reference's own known-answer tests (test_sparse.py / test_collectives.py /
test_optimizer.py hand traces), restated in `tests/test_oracle.py`.

All arithmetic is IEEE-754 fp32 single-op rounding (numpy ufuncs), exactly as
the reference does it; the functions mirror the reference's structure so that
timing the oracle is a fair stand-in for timing the reference (kind "port").
"""

from __future__ import annotations

import struct
import threading

import numpy as np

F32 = np.float32
U64 = np.uint64

SPARSE_MAGIC = 0x67544B31  # transport.py:31
_SPARSE_HEADER = struct.Struct("<IQ")  # transport.py:34


# ---------------------------------------------------------------------------
# sparse.py restatement
# ---------------------------------------------------------------------------


def as_dense(values) -> np.ndarray:
    """sparse.py:19-24 -- coerce to 1-D float32."""
    arr = np.asarray(values, dtype=F32)
    if arr.ndim != 1:
        raise ValueError(f"dense vector must be 1-D, got shape {arr.shape}")
    return arr


def k_from_density(rho: float, m: int) -> int:
    """sparse.py:27-31 -- Python (banker's) round, clamp to [1, m]."""
    if not 0.0 < rho <= 1.0:
        raise ValueError(f"density must be in (0, 1], got {rho}")
    return max(1, min(m, round(rho * m)))


def top_k_select(g, k: int):
    """sparse.py:135-154 -- exact top-k by |g|, lower index wins ties.

    Returns (indices u64 ascending, values f32, residual f32[m]).
    The stable argsort on -|g| is the reference's own ordering rule
    (sparse.py:149); kept entries are copied bitwise and zeroed (+0.0) in the
    residual (sparse.py:151-153).
    """
    g = as_dense(g)
    m = g.size
    if not 1 <= k <= m:
        raise ValueError(f"k must be in [1, {m}], got {k}")
    if not np.isfinite(g).all():
        raise FloatingPointError("non-finite values in dense input")
    order = np.argsort(-np.abs(g), kind="stable")
    keep = np.sort(order[:k]).astype(U64)
    vals = g[keep].copy()
    residual = g.copy()
    residual[keep] = F32(0)
    return keep, vals, residual


def top_op(a_idx, a_val, b_idx, b_val, k: int):
    """sparse.py:157-195 -- the ⊤ merge.

    Union by index, a+b on shared indices (fp32), drop exact zeros, keep the
    k largest |v| (ties -> lower index; NaN magnitudes rank last, as numpy's
    lexsort puts NaN last), return index-ascending.
    """
    if k < 1:
        raise ValueError(f"k must be positive, got {k}")
    a_idx = np.asarray(a_idx, dtype=U64)
    b_idx = np.asarray(b_idx, dtype=U64)
    a_val = np.asarray(a_val, dtype=F32)
    b_val = np.asarray(b_val, dtype=F32)
    if a_idx.size == 0 and b_idx.size == 0:
        return np.empty(0, U64), np.empty(0, F32)
    common, ia, ib = np.intersect1d(a_idx, b_idx, assume_unique=True, return_indices=True)
    a_only = np.ones(a_idx.size, bool)
    a_only[ia] = False
    b_only = np.ones(b_idx.size, bool)
    b_only[ib] = False
    idx = np.concatenate([common, a_idx[a_only], b_idx[b_only]])
    val = np.concatenate([a_val[ia] + b_val[ib], a_val[a_only], b_val[b_only]]).astype(F32)
    nz = val != 0
    idx, val = idx[nz], val[nz]
    if idx.size > k:
        pick = np.lexsort((idx, -np.abs(val)))[:k]
        idx, val = idx[pick], val[pick]
    order = np.argsort(idx)
    return idx[order], val[order]


def densify(idx, val, m: int) -> np.ndarray:
    """sparse.py:198-202."""
    out = np.zeros(m, dtype=F32)
    out[np.asarray(idx, dtype=U64)] = np.asarray(val, dtype=F32)
    return out


# ---------------------------------------------------------------------------
# transport.py codec restatement
# ---------------------------------------------------------------------------


def encode_sparse(idx, val) -> bytes:
    """transport.py:56-61 -- magic u32 | n u64 | idx u64[n] | val f32[n]."""
    idx = np.ascontiguousarray(idx, dtype="<u8")
    val = np.ascontiguousarray(val, dtype="<f4")
    return _SPARSE_HEADER.pack(SPARSE_MAGIC, idx.size) + idx.tobytes() + val.tobytes()


def decode_sparse(buf: bytes, dim: int):
    """transport.py:64-82 (validation errors raised as ValueError here)."""
    magic, n = _SPARSE_HEADER.unpack_from(buf, 0)
    if magic != SPARSE_MAGIC or len(buf) != _SPARSE_HEADER.size + 12 * n:
        raise ValueError("bad sparse buffer")
    off = _SPARSE_HEADER.size
    idx = np.frombuffer(buf, dtype="<u8", count=n, offset=off).astype(U64)
    val = np.frombuffer(buf, dtype="<f4", count=n, offset=off + 8 * n).astype(F32)
    if n and (not np.all(idx[:-1] < idx[1:]) or int(idx[-1]) >= dim):
        raise ValueError("bad sparse indices")
    return idx, val


# ---------------------------------------------------------------------------
# collectives.py restatement (single-threaded simulation of all P ranks)
# ---------------------------------------------------------------------------


def ceil_log2(P: int) -> int:
    """collectives.py:36-37."""
    return (P - 1).bit_length() if P > 1 else 0


def tree_fold(lists, k: int):
    """collectives.py:206-214 / tests/conftest.py:17-28 -- the recursive-halving
    reduce tree; round j: rank r (r % 2^j == 0) folds top_op(acc[r+half], acc[r])."""
    P = len(lists)
    acc = {r: (np.asarray(i, U64), np.asarray(v, F32)) for r, (i, v) in enumerate(lists)}
    for j in range(1, ceil_log2(P) + 1):
        half, span = 1 << (j - 1), 1 << j
        for r in range(0, P, span):
            if r + half < P:
                ri, rv = acc[r + half]
                oi, ov = acc[r]
                acc[r] = top_op(ri, rv, oi, ov, k)
    return acc[0]


def gtopk_allreduce(lists, k: int):
    """collectives.py:188-219 -- every rank ends with the rank-0 fold (binomial
    bcast of the encoded bytes is value-preserving).  Returns (idx, val)."""
    for i, _ in lists:
        if len(i) > k:
            raise ValueError("local sparse vector has more than k entries")
    return tree_fold(lists, k)


def gtopk_message_counts(P: int, nnz_per_rank_round=None):
    """Message accounting of collectives.py:206-217 + 168-185 for each rank:
    list of dicts {msgs_sent, msgs_recv}.  (Bytes depend on nnz and are
    12 + 12*nnz per message, collectives.py:210-211.)"""
    out = [dict(msgs_sent=0, msgs_recv=0) for _ in range(P)]
    for j in range(1, ceil_log2(P) + 1):
        half, span = 1 << (j - 1), 1 << j
        for r in range(P):
            if r % span == half:
                out[r]["msgs_sent"] += 1
            elif r % span == 0 and r + half < P:
                out[r]["msgs_recv"] += 1
    for j in range(1, ceil_log2(P) + 1):
        half = 1 << (j - 1)
        for rel in range(P):
            if rel < half and rel + half < P:
                out[rel]["msgs_sent"] += 1
            elif half <= rel < 2 * half:
                out[rel]["msgs_recv"] += 1
    return out


def topk_allreduce(lists, m: int, P: int) -> np.ndarray:
    """collectives.py:148-165 -- rank-order dense accumulation then / FLOAT(P)."""
    acc = np.zeros(m, dtype=F32)
    for idx, val in lists:
        acc[np.asarray(idx, U64)] += np.asarray(val, F32)
    acc /= F32(P)
    return acc


def dense_ring_allreduce(vectors) -> list[np.ndarray]:
    """collectives.py:88-128 -- reduce-scatter + allgather rings, simulated for
    all ranks with the exact chunk/step order of the reference.  Returns the
    per-rank outputs (identical by construction)."""
    P = len(vectors)
    g = [as_dense(v) for v in vectors]
    if P == 1:
        return [g[0].copy()]
    m = g[0].size
    chunk = -(-m // P)
    bufs = []
    for v in g:
        b = np.zeros(chunk * P, dtype=F32)
        b[:m] = v
        bufs.append(b)

    def piece(r, c):
        return bufs[r][c * chunk:(c + 1) * chunk]

    for step in range(P - 1):
        sends = [piece(r, (r - step) % P).copy() for r in range(P)]
        for r in range(P):
            left = (r - 1) % P
            c = (r - step - 1) % P
            piece(r, c)[:] = piece(r, c) + sends[left]
    for step in range(P - 1):
        sends = [piece(r, (r - step + 1) % P).copy() for r in range(P)]
        for r in range(P):
            left = (r - 1) % P
            c = (r - step) % P
            piece(r, c)[:] = sends[left]
    return [b[:m].copy() for b in bufs]


# ---------------------------------------------------------------------------
# optimizer.py restatement
# ---------------------------------------------------------------------------


class State:
    """optimizer.py:54-78 (OptimizerState / make_state)."""

    def __init__(self, weights, lr, momentum=0.0, update_scaling="average"):
        self.weights = as_dense(weights).copy()
        self.residual = np.zeros_like(self.weights)
        self.lr = lr
        self.momentum = momentum
        self.update_scaling = update_scaling
        self.velocity = None
        self.iteration = 0


def apply_update(state: State, update: np.ndarray) -> None:
    """optimizer.py:92-99."""
    if state.momentum > 0.0:
        if state.velocity is None:
            state.velocity = np.zeros_like(state.weights)
        state.velocity = F32(state.momentum) * state.velocity + update
        update = state.velocity
    state.weights -= F32(state.lr) * update
    state.iteration += 1


def scaled(state: State, merged: np.ndarray, P: int) -> np.ndarray:
    """optimizer.py:102-105."""
    return merged / F32(P) if state.update_scaling == "average" else merged


def gtopk_step_all(states, grads, k: int):
    """optimizer.py:199-252 for all P ranks at once (measure_divergence off).

    Returns the global (idx, val) and the per-rank local selections."""
    P = len(states)
    sels = []
    resid_after = []
    for st, g in zip(states, grads):
        acc = st.residual + as_dense(g)
        i, v, r = top_k_select(acc, k)
        sels.append((i, v))
        resid_after.append(r)
    gi, gv = gtopk_allreduce(sels, k)
    gmask = np.zeros(states[0].weights.size, bool)
    gmask[gi] = True
    for st, (i, v), r in zip(states, sels, resid_after):
        outside = ~gmask[i]
        r[i[outside]] += v[outside]
        st.residual = r
    m = states[0].weights.size
    for st in states:
        apply_update(st, scaled(st, densify(gi, gv, m), P))
    return (gi, gv), sels


def topk_step_all(states, grads, k: int):
    """optimizer.py:145-173 for all ranks."""
    P = len(states)
    sels = []
    for st, g in zip(states, grads):
        i, v, r = top_k_select(st.residual + as_dense(g), k)
        sels.append((i, v))
        st.residual = r
    avg = topk_allreduce(sels, states[0].weights.size, P)
    for st in states:
        apply_update(st, avg)
    return sels


def dense_step_all(states, grads, rank_order_sum=False):
    """optimizer.py:118-142 for all ranks."""
    P = len(states)
    if rank_order_sum:
        acc = np.zeros_like(as_dense(grads[0]))
        for g in grads:
            acc = acc + as_dense(g)
        totals = [acc] * P
    else:
        totals = dense_ring_allreduce(grads)
    for st, t in zip(states, totals):
        apply_update(st, t / F32(P))


# ---------------------------------------------------------------------------
# CPU baseline harness: thread-per-rank, like transport.run_workers
# (transport.py:507-539); numpy's argsort releases the GIL.
# ---------------------------------------------------------------------------


def threaded_gtopk_step(states, grads, k: int):
    """One gtopk step for all ranks with one host thread per rank doing its
    own residual-add + select (the reference's per-rank compress phase), then
    the tree fold + update.  Used only as the timed CPU baseline."""
    P = len(states)
    sels = [None] * P
    resid = [None] * P

    def work(r):
        i, v, res = top_k_select(states[r].residual + grads[r], k)
        sels[r] = (i, v)
        resid[r] = res

    threads = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    gi, gv = gtopk_allreduce(sels, k)
    m = states[0].weights.size
    gmask = np.zeros(m, bool)
    gmask[gi] = True
    dense = densify(gi, gv, m)
    for r, st in enumerate(states):
        i, v = sels[r]
        outside = ~gmask[i]
        resid[r][i[outside]] += v[outside]
        st.residual = resid[r]
        apply_update(st, scaled(st, dense, P))
    return gi, gv
