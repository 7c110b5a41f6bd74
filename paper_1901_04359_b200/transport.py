"""Rank-addressed endpoints -- drop-in for the reference's `gtopk.transport`
(pkg/src/gtopk/transport.py), re-designed for GPUs.

* The Endpoint contract is kept: rank, world_size, timeout, stats, blocking
  byte-level send/recv matched on (source, tag) with FIFO channels, a
  dissemination barrier, abort/close (transport.py:156-220), and the sparse
  wire codec encode_sparse/decode_sparse (transport.py:56-82).
* The collectives of the hot path do NOT move bytes through this host API:
  each endpoint carries a *device group* through which gTopKAllReduce /
  TopKAllReduce / dense allreduce run as kernels on the GPU
  (collectives.py).  Two backends:
    - `create_local_cluster(P)`: P ranks in one process (one host thread
      each, `run_workers`), all on one GPU -- the reference's in-process
      cluster (transport.py:279-284), used for parity tests and the
      single-GPU benchmark with simulated workers.
    - `init_dist_cluster()`: one process per GPU under torchrun
      (torch.distributed over NCCL for plumbing), with the fused NVLink
      peer-memory exchange kernel for gTopKAllReduce (`dist.py`).
* `stats` keeps the reference's accounting (bytes = 12 + 12*nnz per sparse
  message, collectives.py:210-211); device-resident counts are resolved
  lazily so a step never synchronises just to count bytes.
"""

from __future__ import annotations

import collections
import logging
import struct
import threading

import numpy as np

from .sparse import FLOAT, INDEX, SparseVector

log = logging.getLogger("gtopk_b200.transport")

FRAME_MAGIC = 0x6754524E
SPARSE_MAGIC = 0x67544B31
_SPARSE_HEADER = struct.Struct("<IQ")
_MAX_PAYLOAD = 2**32 - 1
BARRIER_TAG = 0x7FFF0000
DEFAULT_TIMEOUT = 30.0


class TransportError(Exception):
    """Connection failure, timeout, or aborted cluster (transport.py:43-44)."""


class ProtocolError(Exception):
    """Malformed frame, bad magic, or size mismatch (transport.py:47-48)."""


# ---------------------------------------------------------------------------
# sparse wire codec (transport.py:56-82) -- bit-exact wire format
# ---------------------------------------------------------------------------


def encode_sparse(s) -> bytes:
    """magic u32 | count u64 | indices u64[] | values f32[], little-endian."""
    if hasattr(s, "to_host") and not isinstance(s, SparseVector):
        s = s.to_host()
    header = _SPARSE_HEADER.pack(SPARSE_MAGIC, s.nnz)
    idx = np.ascontiguousarray(s.indices, dtype="<u8").tobytes()
    val = np.ascontiguousarray(s.values, dtype="<f4").tobytes()
    return header + idx + val


def decode_sparse(buf: bytes, dim: int) -> SparseVector:
    """Inverse of encode_sparse; validates magic, length, order and range."""
    if len(buf) < _SPARSE_HEADER.size:
        raise ProtocolError(f"sparse buffer truncated: {len(buf)} bytes")
    magic, n = _SPARSE_HEADER.unpack_from(buf, 0)
    if magic != SPARSE_MAGIC:
        raise ProtocolError(f"bad sparse magic 0x{magic:08X}")
    expect = _SPARSE_HEADER.size + 12 * n
    if len(buf) != expect:
        raise ProtocolError(f"sparse buffer length {len(buf)}, expected {expect}")
    off = _SPARSE_HEADER.size
    indices = np.frombuffer(buf, dtype="<u8", count=n, offset=off).astype(INDEX)
    values = np.frombuffer(buf, dtype="<f4", count=n, offset=off + 8 * n).astype(FLOAT)
    if n > 0:
        if not np.all(indices[:-1] < indices[1:]):
            raise ProtocolError("sparse indices not strictly ascending")
        if int(indices[-1]) >= dim:
            raise ProtocolError(f"sparse index {int(indices[-1])} >= dim {dim}")
    return SparseVector(dim, indices, values)


def sparse_msg_bytes(nnz: int) -> int:
    """Wire size of one encoded sparse message (transport.py:56-61)."""
    return 12 + 12 * int(nnz)


# ---------------------------------------------------------------------------
# stats with lazily resolved device counts
# ---------------------------------------------------------------------------


class TransportStats:
    """Byte/message counters (transport.py:135-153).  `add_sparse_*` accepts
    a device count tensor; it is resolved (one small D2H) only when read."""

    def __init__(self, bytes_sent=0, bytes_recv=0, msgs_sent=0, msgs_recv=0):
        self._bs = int(bytes_sent)
        self._br = int(bytes_recv)
        self.msgs_sent = int(msgs_sent)
        self.msgs_recv = int(msgs_recv)
        self._pending: list = []  # (count_tensor_or_int, sent: bool)

    def _resolve(self) -> None:
        if not self._pending:
            return
        pend, self._pending = self._pending, []
        for cnt, sent in pend:
            n = int(cnt.item()) if hasattr(cnt, "item") else int(cnt)
            if sent:
                self._bs += sparse_msg_bytes(n)
            else:
                self._br += sparse_msg_bytes(n)

    def add_sparse(self, count, sent: bool) -> None:
        if sent:
            self.msgs_sent += 1
        else:
            self.msgs_recv += 1
        self._pending.append((count, sent))

    @property
    def bytes_sent(self) -> int:
        self._resolve()
        return self._bs

    @bytes_sent.setter
    def bytes_sent(self, v) -> None:
        self._resolve()
        self._bs = int(v)

    @property
    def bytes_recv(self) -> int:
        self._resolve()
        return self._br

    @bytes_recv.setter
    def bytes_recv(self, v) -> None:
        self._resolve()
        self._br = int(v)

    def snapshot(self) -> "TransportStats":
        return TransportStats(self.bytes_sent, self.bytes_recv, self.msgs_sent, self.msgs_recv)

    def delta(self, earlier: "TransportStats") -> "TransportStats":
        return TransportStats(
            self.bytes_sent - earlier.bytes_sent,
            self.bytes_recv - earlier.bytes_recv,
            self.msgs_sent - earlier.msgs_sent,
            self.msgs_recv - earlier.msgs_recv,
        )

    def __repr__(self) -> str:
        return (
            f"TransportStats(bytes_sent={self.bytes_sent}, bytes_recv={self.bytes_recv}, "
            f"msgs_sent={self.msgs_sent}, msgs_recv={self.msgs_recv})"
        )


# ---------------------------------------------------------------------------
# endpoints
# ---------------------------------------------------------------------------


def _dissemination_rounds(rank: int, P: int):
    """(send_to, recv_from) of each round of a dissemination barrier: round r
    pairs rank with rank +- 2^r (mod P), ceil(log2 P) rounds (transport.py:197-206)."""
    return [((rank + (1 << r)) % P, (rank - (1 << r)) % P) for r in range((P - 1).bit_length())]


class Endpoint:
    """One rank's handle (transport.py:156-220): blocking byte messages to and
    from the other ranks, matched on (peer, tag) in FIFO order, plus the
    device group the GPU collectives run on.  Backends implement the
    reference's plug points `_send_impl` / `_recv_impl`."""

    def __init__(self, rank: int, world_size: int, timeout: float = DEFAULT_TIMEOUT):
        self.rank = rank
        self.world_size = world_size
        self.timeout = timeout
        self.stats = TransportStats()
        self.group = None  # device group used by the GPU collectives

    def _validate(self, peer: int, tag: int) -> None:
        # argument errors are ValueError, raised before any transfer
        if peer == self.rank:
            raise ValueError("send/recv to self is not allowed")
        if peer < 0 or peer >= self.world_size:
            raise ValueError(f"rank {peer} out of range [0, {self.world_size})")
        if tag < 0 or tag >= 1 << 32:
            raise ValueError(f"tag must fit in 32 bits, got {tag}")

    def send(self, dest: int, tag: int, payload: bytes) -> None:
        self._validate(dest, tag)
        data = bytes(payload)
        if len(data) > _MAX_PAYLOAD:
            raise ValueError("payload too large")
        self._send_impl(dest, tag, data)
        self.stats.msgs_sent += 1
        self.stats.bytes_sent += len(data)

    def recv(self, source: int, tag: int) -> bytes:
        self._validate(source, tag)
        data = self._recv_impl(source, tag)
        self.stats.msgs_recv += 1
        self.stats.bytes_recv += len(data)
        return data

    def barrier(self) -> None:
        """Dissemination barrier: ceil(log2 P) rounds of empty messages."""
        for r, (to, frm) in enumerate(_dissemination_rounds(self.rank, self.world_size)):
            self.send(to, BARRIER_TAG + r, b"")
            self.recv(frm, BARRIER_TAG + r)

    def abort(self) -> None:
        """Wake blocked peers with TransportError."""

    def close(self) -> None:
        pass

    def _send_impl(self, dest: int, tag: int, payload: bytes) -> None:
        raise NotImplementedError

    def _recv_impl(self, source: int, tag: int) -> bytes:
        raise NotImplementedError


class _Mailboxes:
    """Byte channels of one in-process cluster: one mailbox per destination
    rank, each a condition variable over per-(source, tag) FIFOs, so a receiver
    sleeps until its own mailbox changes (no polling) and an abort wakes every
    receiver at once."""

    def __init__(self, P: int):
        self._cond = [threading.Condition() for _ in range(P)]
        self._fifo: list[dict] = [collections.defaultdict(collections.deque) for _ in range(P)]
        self.aborted = False

    def post(self, src: int, dst: int, tag: int, payload: bytes) -> None:
        if self.aborted:
            raise TransportError("cluster aborted")
        with self._cond[dst]:
            self._fifo[dst][(src, tag)].append(payload)
            self._cond[dst].notify_all()

    def take(self, src: int, dst: int, tag: int, timeout: float) -> bytes:
        key = (src, tag)
        cond, fifo = self._cond[dst], self._fifo[dst]
        with cond:
            ready = cond.wait_for(lambda: self.aborted or bool(fifo.get(key)), timeout)
            if fifo.get(key):  # delivered messages are still handed out after an abort
                return fifo[key].popleft()
            if self.aborted:
                raise TransportError("cluster aborted")
            assert not ready
            raise TransportError(f"rank {dst}: recv from {src} tag {tag} timed out")

    def abort(self) -> None:
        self.aborted = True
        for cond in self._cond:
            with cond:
                cond.notify_all()


class LocalEndpoint(Endpoint):
    """Endpoint of an in-process cluster (transport.py:250-276)."""

    def __init__(self, rank, world_size, boxes: _Mailboxes, group, timeout):
        super().__init__(rank, world_size, timeout)
        self._boxes = boxes
        self.group = group

    def _send_impl(self, dest, tag, payload):
        self._boxes.post(self.rank, dest, tag, payload)

    def _recv_impl(self, source, tag):
        return self._boxes.take(source, self.rank, tag, self.timeout)

    def abort(self):
        self._boxes.abort()
        if self.group is not None:
            self.group.abort()


class LocalDeviceGroup:
    """Rendezvous for the in-process GPU collectives.

    Every rank thread deposits its operand; the LAST rank to arrive runs the
    whole collective as a chain of kernels on its stream (kernels that waited
    on each other would not be guaranteed to be co-scheduled on one GPU) and
    publishes the result; every rank returns it.  One condition-variable
    rendezvous per collective: a rank can only enter the next collective after
    it has read this one's result, and the next result is only written once
    every rank has entered, so results alternate between two slots.
    """

    def __init__(self, P: int, device=None, timeout: float = DEFAULT_TIMEOUT):
        self.P = P
        self._device = device
        self.timeout = timeout
        self._cond = threading.Condition()
        self._operands = [None] * P
        self._arrived = 0
        self._generation = 0
        self._outcome = [None, None]  # (result, error) per generation parity
        self.aborted = False

    @property
    def device(self):
        if self._device is None:
            from . import device as _dev

            self._device = _dev.default_device()
        return self._device

    def abort(self) -> None:
        with self._cond:
            self.aborted = True
            self._cond.notify_all()

    def run(self, rank: int, operand, leader_fn):
        """Collective call: returns leader_fn(all operands, rank order) to every rank."""
        with self._cond:
            if self.aborted:
                raise TransportError("cluster aborted")
            gen = self._generation
            self._operands[rank] = operand
            self._arrived += 1
            if self._arrived == self.P:
                ops, self._operands = self._operands, [None] * self.P
                self._arrived = 0
                try:
                    self._outcome[gen & 1] = (leader_fn(ops), None)
                except BaseException as exc:  # noqa: BLE001 - re-raised on every rank
                    self._outcome[gen & 1] = (None, exc)
                self._generation += 1
                self._cond.notify_all()
            elif not self._cond.wait_for(lambda: self._generation != gen or self.aborted, self.timeout):
                raise TransportError("collective rendezvous timed out")
            if self._generation == gen:  # woken by an abort before completion
                raise TransportError("cluster aborted")
            result, err = self._outcome[gen & 1]
        if err is not None:
            raise err
        return result


def create_local_cluster(P: int, timeout: float = DEFAULT_TIMEOUT, device=None) -> list[Endpoint]:
    """P mutually connected in-process endpoints (transport.py:279-284) that
    share one GPU device group."""
    if P < 1:
        raise ValueError(f"P must be >= 1, got {P}")
    boxes = _Mailboxes(P)
    group = LocalDeviceGroup(P, device, timeout)
    return [LocalEndpoint(r, P, boxes, group, timeout) for r in range(P)]


def _root_cause(failures: dict) -> BaseException:
    """The failure to report: a rank's own error before the TransportErrors
    the abort induced in the others, lowest rank first (transport.py:535-538)."""
    own = sorted(r for r, e in failures.items() if not isinstance(e, TransportError))
    return failures[own[0] if own else min(failures)]


def run_workers(endpoints: list[Endpoint], fn) -> list:
    """fn(ep) for every endpoint concurrently, one host thread per rank
    (transport.py:507-539); results in rank order.  The first failure aborts
    every endpoint (waking blocked receives and rendezvous) and the root
    cause is re-raised.  Worker threads run on the caller's CUDA device."""
    from concurrent.futures import ThreadPoolExecutor

    n = len(endpoints)
    results: list = [None] * n
    failures: dict[int, BaseException] = {}
    device = None
    try:
        import torch

        if torch.cuda.is_available():
            device = torch.cuda.current_device()
    except Exception:  # pragma: no cover - torch absent
        device = None

    def body(i: int) -> None:
        try:
            if device is not None:
                import torch

                torch.cuda.set_device(device)
            results[i] = fn(endpoints[i])
        except BaseException as exc:  # noqa: BLE001 - reported to the caller
            failures[i] = exc
            for ep in endpoints:
                ep.abort()

    if n:
        with ThreadPoolExecutor(max_workers=n, thread_name_prefix="gtopk-b200-rank") as pool:
            for fut in [pool.submit(body, i) for i in range(n)]:
                fut.result()
    if failures:
        raise _root_cause(failures)
    return results
