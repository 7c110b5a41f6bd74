"""Gradient aggregation collectives -- drop-in for the reference's
`gtopk.collectives` (pkg/src/gtopk/collectives.py).

The three aggregation paths keep their reference semantics and accounting:

* gtopk_allreduce   -- ⌈log2 P⌉-round ⊤ merge tree + broadcast (:188-219);
                       every rank returns the identical global top-k, NOT
                       divided by P.  On the GPU: in-process clusters run the
                       exact reduce-tree as a chain of K2 merge kernels; one
                       process per GPU runs the fused NVLink exchange kernel
                       (butterfly for P = 2^n -- bitwise equal to tree+bcast
                       because ⊤ is commutative -- tree+bcast otherwise).
* topk_allreduce    -- allgather + rank-order dense accumulation / P (:148-165).
* dense_ring_allreduce -- elementwise sum (:88-128); within rtol 1e-4 of the
                       sequential sum, bitwise identical on all ranks.

Byte-level helpers (allgather, binomial_bcast) run the reference's ring and
binomial message patterns over Endpoint.send/recv (the accounting depends on
them).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device as _dev
from .device import DeviceList
from .sparse import FLOAT, DeviceSparseVector, IndexMask, SparseVector, as_dense
from .transport import Endpoint, ProtocolError, sparse_msg_bytes

_TAG_GATHER = 0x3000
_TAG_BCAST = 0x5000


def ceil_log2(P: int) -> int:
    """collectives.py:36-37."""
    return (P - 1).bit_length() if P > 1 else 0


@dataclass
class CollectiveStats:
    """Per-rank accounting for one collective invocation (collectives.py:40-62)."""

    collective: str
    P: int
    m: int
    k: int
    rank: int
    bytes_sent: int
    bytes_recv: int
    msgs: int
    rounds: int
    wall_ms: float

    CSV_HEADER = "collective,P,m,k,rank,bytes_sent,bytes_recv,msgs,rounds,wall_ms"

    def csv_row(self) -> str:
        return (
            f"{self.collective},{self.P},{self.m},{self.k},{self.rank},"
            f"{self.bytes_sent},{self.bytes_recv},{self.msgs},{self.rounds},"
            f"{self.wall_ms:.6f}"
        )


@dataclass
class GTopKResult:
    """Global top-k (identical on all ranks) and its index mask."""

    global_topk: object  # SparseVector (host inputs) or DeviceSparseVector
    global_mask: IndexMask


def comm_rounds(collective: str, P: int) -> int:
    """collectives.py:73-85."""
    if P == 1:
        return 0
    if collective == "dense":
        return 2 * (P - 1)
    if collective in ("topk", "allgather"):
        return P - 1
    if collective == "gtopk":
        return 2 * ceil_log2(P)
    if collective == "bcast":
        return ceil_log2(P)
    raise ValueError(f"unknown collective {collective!r}")


def predicted_bytes(collective: str, P: int, m: int, k: int) -> int:
    """collectives.py:222-234."""
    if P == 1:
        return 0
    if collective == "dense":
        return 2 * (P - 1) * (-(-m // P)) * 4
    if collective == "topk":
        return (P - 1) * sparse_msg_bytes(k)
    if collective == "gtopk":
        raise ValueError("gtopk send volume is rank dependent; use endpoint stats")
    raise ValueError(f"unknown collective {collective!r}")


# ---------------------------------------------------------------------------
# schedules (host logic; shared by the local and the NVLink backends)
# ---------------------------------------------------------------------------


def tree_schedule(rank: int, P: int):
    """Per-rank steps of the reference structure: reduce tree (:206-214) then
    binomial broadcast from rank 0 (:168-185).  Each step is
    (send_to, recv_from, merge) with -1 for none."""
    steps = []
    n = ceil_log2(P)
    for j in range(1, n + 1):
        half, span = 1 << (j - 1), 1 << j
        if rank % span == half:
            steps.append((rank - half, -1, 0))
        elif rank % span == 0 and rank + half < P:
            steps.append((-1, rank + half, 1))
        else:
            steps.append((-1, -1, 0))
    for j in range(1, n + 1):
        half = 1 << (j - 1)
        if rank < half:
            steps.append((rank + half if rank + half < P else -1, -1, 0))
        elif rank < 2 * half:
            steps.append((-1, rank - half, 0))
        else:
            steps.append((-1, -1, 0))
    return steps


def butterfly_schedule(rank: int, P: int):
    """Recursive doubling for P = 2^n: round j exchanges with rank ^ 2^j and
    both sides merge -- no broadcast rounds.  Bitwise equal to the tree +
    broadcast because ⊤ is commutative and the butterfly's pairings are the
    tree's pairings."""
    if P & (P - 1):
        raise ValueError("butterfly needs a power-of-two P")
    return [(rank ^ (1 << j), rank ^ (1 << j), 1) for j in range(ceil_log2(P))]


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


def _group_device(ep: Endpoint):
    g = getattr(ep, "group", None)
    if g is None:
        raise TypeError("endpoint has no device group (use create_local_cluster or init_dist_cluster)")
    return g.device


def _to_device_list(local, device, cap) -> tuple[DeviceList, bool]:
    """(device list with capacity >= cap, input_was_host)"""
    if isinstance(local, DeviceSparseVector):
        lst = local.list
        if lst.device != device or lst.cap < cap:
            lst = lst.clone(cap=max(cap, lst.cap))
            if lst.device != device:
                lst = DeviceList.from_host(local.dim, *local.list.to_host(), device, cap)
        return lst, False
    return DeviceList.from_host(local.dim, local.indices, local.values, device, cap), True


# ---------------------------------------------------------------------------
# gTopKAllReduce
# ---------------------------------------------------------------------------


def _local_gtopk_leader(ops):
    """Run the reduce tree over all ranks' lists on the leader's stream.
    ops[r] = (ep, DeviceList acc (private copy), k)."""
    P = len(ops)
    k = ops[0][2]
    acc = [o[1] for o in ops]
    dev = acc[0].device
    nmsg = 0
    log = torch.zeros(max(2 * P, 1), dtype=torch.int32, device=dev)  # sent counts per message
    sends = []  # (sender rank, receiver rank, log slot)
    for j in range(1, ceil_log2(P) + 1):
        half, span = 1 << (j - 1), 1 << j
        for r in range(0, P, span):
            if r + half < P:
                log[nmsg:nmsg + 1].copy_(acc[r + half].n)
                sends.append((r + half, r, nmsg))
                nmsg += 1
                _dev.top_op(acc[r + half], acc[r], k, acc[r])
    final = acc[0]
    # accounting: tree messages carry the sender's accumulator; the binomial
    # broadcast carries the final list (collectives.py:216-217)
    for s, r, slot in sends:
        cnt = log[slot:slot + 1]
        ops[s][0].stats.add_sparse(cnt, sent=True)
        ops[r][0].stats.add_sparse(cnt, sent=False)
    n = ceil_log2(P)
    for j in range(1, n + 1):
        half = 1 << (j - 1)
        for rel in range(P):
            if rel < half and rel + half < P:
                ops[rel][0].stats.add_sparse(final.n, sent=True)
                ops[rel + half][0].stats.add_sparse(final.n, sent=False)
    return final


def gtopk_allreduce(ep: Endpoint, local, k: int, P: int | None = None) -> GTopKResult:
    """collectives.py:188-219 -- global top-k of the P local top-k vectors via
    the ⊤ merge tree; identical result on every rank; values NOT divided by P."""
    P = ep.world_size if P is None else P
    if P != ep.world_size:
        raise ValueError("P must match the cluster size")
    if local.nnz > k:
        raise ValueError(f"local sparse vector has {local.nnz} entries, k={k}")
    group = ep.group
    if hasattr(group, "gtopk"):  # one process per GPU: fused NVLink exchange
        dev = group.device
        lst, was_host = _to_device_list(local, dev, k)
        out = group.gtopk(ep, lst, k)
    else:
        dev = _group_device(ep)
        lst, was_host = _to_device_list(local, dev, k)
        # private accumulator (the merges update it in place)
        mine = lst if was_host else lst.clone(cap=max(k, lst.cap))
        out = mine if P == 1 else group.run(ep.rank, (ep, mine, k), _local_gtopk_leader)
    if was_host:
        i, v = out.to_host()
        g = SparseVector(local.dim, i, v)
        return GTopKResult(g, IndexMask.from_indices(local.dim, g.indices))
    # a fresh list per rank and call, like the reference's decode
    # (collectives.py:216-219): the exchange plan's accumulator (and the
    # in-process leader's list, shared by every rank) is reused by later calls
    dsv = DeviceSparseVector(out.clone(cap=k))
    return GTopKResult(dsv, _LazyDeviceMask(dsv))


class _LazyDeviceMask(IndexMask):
    """Global mask of a device-resident result: indices fetched on demand."""

    def __init__(self, dsv: DeviceSparseVector):
        self.dim = dsv.dim
        self._dsv = dsv
        self._flags = None
        self._indices = None

    def _load(self):
        if self._indices is None and self._flags is None:
            self._indices = self._dsv.to_host().indices

    @property
    def flags(self):
        self._load()
        return IndexMask.flags.fget(self)

    @property
    def indices(self):
        self._load()
        return IndexMask.indices.fget(self)

    @property
    def count(self):
        self._load()
        return IndexMask.count.fget(self)


# ---------------------------------------------------------------------------
# TopKAllReduce (allgather baseline)
# ---------------------------------------------------------------------------


def _allgather_stats(ops, counts_dev):
    """Ring allgather accounting (collectives.py:140-144): at step s rank r
    forwards block (r - s) % P to the right and receives (r - s - 1) % P."""
    P = len(ops)
    for s in range(P - 1):
        for r in range(P):
            ops[r][0].stats.add_sparse(counts_dev[(r - s) % P:(r - s) % P + 1], sent=True)
            ops[r][0].stats.add_sparse(counts_dev[(r - s - 1) % P:(r - s - 1) % P + 1], sent=False)


def _local_topk_leader(ops, divide=True):
    P = len(ops)
    dev = ops[0][1].device
    m = ops[0][1].dim
    cap = max(o[1].cap for o in ops)
    idx = torch.empty((P, cap), dtype=torch.int32, device=dev)
    val = torch.empty((P, cap), dtype=torch.float32, device=dev)
    cnt = torch.empty(P, dtype=torch.int32, device=dev)
    for r, (_ep, lst) in enumerate(ops):
        if lst.dim != m:
            raise ProtocolError("sparse dim mismatch in topk_allreduce")
        idx[r, : lst.cap].copy_(lst.idx)
        val[r, : lst.cap].copy_(lst.val)
        cnt[r:r + 1].copy_(lst.n)
    out = torch.empty(m, dtype=torch.float32, device=dev)
    _dev.topk_accumulate(idx, val, cnt, P, cap, m, out, divide=divide)
    _allgather_stats(ops, cnt)
    return out


def topk_allreduce(ep: Endpoint, local, P: int | None = None):
    """collectives.py:148-165 -- dense average of all ranks' sparse vectors,
    accumulated in rank order 0..P-1 then divided by FLOAT(P) (bitwise equal
    to the reference).  Host input -> numpy; device input -> CUDA tensor."""
    P = ep.world_size if P is None else P
    if P != ep.world_size:
        raise ValueError("P must match the cluster size")
    group = ep.group
    if hasattr(group, "topk"):
        dev = group.device
        lst, was_host = _to_device_list(local, dev, max(local.nnz, 1))
        out = group.topk(ep, lst, divide=True)
    else:
        dev = _group_device(ep)
        lst, was_host = _to_device_list(local, dev, max(local.nnz, 1))
        out = group.run(ep.rank, (ep, lst), _local_topk_leader)
    return out.cpu().numpy() if was_host else out


def rank_order_sparse_sum(ep: Endpoint, local):
    """Unscaled rank-order sum of everyone's selection (optimizer.py:176-183)."""
    group = ep.group
    if hasattr(group, "topk"):
        lst, _ = _to_device_list(local, group.device, max(local.nnz, 1))
        return group.topk(ep, lst, divide=False)
    lst, _ = _to_device_list(local, _group_device(ep), max(local.nnz, 1))
    return group.run(ep.rank, (ep, lst), lambda ops: _local_topk_leader(ops, divide=False))


# ---------------------------------------------------------------------------
# dense allreduce baseline
# ---------------------------------------------------------------------------


def _local_dense_leader(ops, ring_stats=True):
    """Sum of every rank's dense vector in one kernel: in the ring's order
    (bitwise the reference's dense_ring_allreduce) or, with ring_stats=False,
    in rank order from +0 (the rank-order sum).  Accounting:
    the ring allreduce's 2(P-1) chunk messages (collectives.py:101-126), or
    with ring_stats=False the allgather of whole vectors (optimizer.py:108-115)."""
    P = len(ops)
    m = ops[0][1].numel()
    for _ep, g in ops:
        if g.numel() != m:
            raise ProtocolError(
                f"ring chunk size mismatch: got {4 * (-(-g.numel() // P))} bytes, expected {4 * (-(-m // P))}"
            )
    out = torch.empty(m, dtype=torch.float32, device=ops[0][1].device)
    _dev.dense_sum([g for _ep, g in ops], m, out, ring=ring_stats)
    msgs, nbytes = (2 * (P - 1), 4 * -(-m // P)) if ring_stats else (P - 1, 4 * m)
    for ep_r, _g in ops:
        ep_r.stats.msgs_sent += msgs
        ep_r.stats.msgs_recv += msgs
        ep_r.stats.bytes_sent += msgs * nbytes
        ep_r.stats.bytes_recv += msgs * nbytes
    return out


def dense_ring_allreduce(ep: Endpoint, g):
    """collectives.py:88-128 -- elementwise SUM over ranks (not the average).
    Host input -> numpy; device input -> CUDA tensor.  Mismatched dims raise
    ProtocolError on every rank."""
    on_device = isinstance(g, torch.Tensor) and g.is_cuda
    P = ep.world_size
    group = ep.group
    if on_device:
        gd = g.contiguous().to(torch.float32)
    else:
        gh = as_dense(g)
        if P == 1:
            return gh.copy()
    if hasattr(group, "dense"):
        dev = group.device
        if not on_device:
            gd = torch.from_numpy(np.ascontiguousarray(gh)).to(dev)
        out = group.dense(ep, gd)
    else:
        dev = _group_device(ep)
        if not on_device:
            gd = torch.from_numpy(np.ascontiguousarray(gh)).to(dev)
        if P == 1:
            return gd.clone()
        out = group.run(ep.rank, (ep, gd), _local_dense_leader)
    return out if on_device else out.cpu().numpy()


def rank_order_dense_sum(ep: Endpoint, g):
    """optimizer.py:105-115 (_rank_order_dense_sum): every rank's dense vector
    gathered and accumulated from +0 in rank order 0..P-1 -- the summation
    order of topk_allreduce, so k = m trajectories compare bitwise.  Host
    input -> numpy; device input -> CUDA tensor (identical on every rank)."""
    on_device = isinstance(g, torch.Tensor) and g.is_cuda
    group = ep.group
    gh = None if on_device else as_dense(g)
    if hasattr(group, "dense_rank_order"):
        dev = group.device
        gd = g.contiguous().to(torch.float32) if on_device else torch.from_numpy(np.ascontiguousarray(gh)).to(dev)
        out = group.dense_rank_order(ep, gd)
    else:
        dev = _group_device(ep)
        gd = g.contiguous().to(torch.float32) if on_device else torch.from_numpy(np.ascontiguousarray(gh)).to(dev)
        out = group.run(ep.rank, (ep, gd), lambda ops: _local_dense_leader(ops, ring_stats=False))
    return out if on_device else out.cpu().numpy()


# ---------------------------------------------------------------------------
# byte-level helpers (host; the reference's message patterns)
# ---------------------------------------------------------------------------


def _ring_allgather_plan(rank: int, P: int):
    """Step s of the ring: forward block (rank - s) to the right neighbour,
    receive block (rank - s - 1) from the left one (collectives.py:138-144)."""
    return [(s, (rank - s) % P, (rank - s - 1) % P) for s in range(P - 1)]


def allgather(ep: Endpoint, payload: bytes) -> list[bytes]:
    """collectives.py:131-145 -- every rank's payload, indexed by source rank,
    in P - 1 ring steps (P - 1 messages sent and received per rank)."""
    P, me = ep.world_size, ep.rank
    right, left = (me + 1) % P, (me - 1) % P
    have = {me: bytes(payload)}
    for step, fwd, want in _ring_allgather_plan(me, P):
        ep.send(right, _TAG_GATHER + step, have[fwd])
        have[want] = ep.recv(left, _TAG_GATHER + step)
    return [have[r] for r in range(P)]


def _binomial_plan(rel: int, P: int):
    """(round j, peer offset, sends?) of a binomial broadcast for the rank at
    distance `rel` from the root: in round j the ranks that already hold the
    payload (rel < 2^(j-1)) forward it 2^(j-1) further (collectives.py:176-184)."""
    plan = []
    for j in range(1, ceil_log2(P) + 1):
        half = 1 << (j - 1)
        if rel < half and rel + half < P:
            plan.append((j, half, True))
        elif half <= rel < 2 * half:
            plan.append((j, -half, False))
    return plan


def binomial_bcast(ep: Endpoint, root: int, payload: bytes | None) -> bytes:
    """collectives.py:168-185 -- the root's payload on every rank after
    ceil(log2 P) rounds."""
    P = ep.world_size
    rel = (ep.rank - root) % P
    if rel == 0 and payload is None:
        raise ValueError("root must supply the payload")
    data = bytes(payload) if rel == 0 else b""
    for j, off, sends in _binomial_plan(rel, P):
        peer = (root + rel + off) % P
        if sends:
            ep.send(peer, _TAG_BCAST + j, data)
        else:
            data = ep.recv(peer, _TAG_BCAST + j)
    return data
