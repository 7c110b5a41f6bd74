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

import logging
import queue
import struct
import threading
import time

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


class Endpoint:
    """One rank's handle (transport.py:156-220) plus its device group."""

    def __init__(self, rank: int, world_size: int, timeout: float = DEFAULT_TIMEOUT):
        self.rank = rank
        self.world_size = world_size
        self.timeout = timeout
        self.stats = TransportStats()
        self.group = None  # device group used by the GPU collectives

    def send(self, dest: int, tag: int, payload: bytes) -> None:
        self._check_peer(dest)
        self._check_tag(tag)
        if len(payload) > _MAX_PAYLOAD:
            raise ValueError("payload too large")
        self._send_impl(dest, tag, bytes(payload))
        self.stats.msgs_sent += 1
        self.stats.bytes_sent += len(payload)

    def recv(self, source: int, tag: int) -> bytes:
        self._check_peer(source)
        self._check_tag(tag)
        payload = self._recv_impl(source, tag)
        self.stats.msgs_recv += 1
        self.stats.bytes_recv += len(payload)
        return payload

    def _check_peer(self, other: int) -> None:
        if other == self.rank:
            raise ValueError("send/recv to self is not allowed")
        if not 0 <= other < self.world_size:
            raise ValueError(f"rank {other} out of range [0, {self.world_size})")

    @staticmethod
    def _check_tag(tag: int) -> None:
        if not 0 <= tag < 2**32:
            raise ValueError(f"tag must fit in 32 bits, got {tag}")

    def barrier(self) -> None:
        """Dissemination barrier, ceil(log2 P) rounds (transport.py:197-206)."""
        P = self.world_size
        if P == 1:
            return
        for r in range((P - 1).bit_length()):
            step = 1 << r
            self.send((self.rank + step) % P, BARRIER_TAG + r, b"")
            self.recv((self.rank - step) % P, BARRIER_TAG + r)

    def abort(self) -> None:
        """Wake blocked peers with TransportError."""

    def close(self) -> None:
        pass

    def _send_impl(self, dest: int, tag: int, payload: bytes) -> None:
        raise NotImplementedError

    def _recv_impl(self, source: int, tag: int) -> bytes:
        raise NotImplementedError


class _LocalRouter:
    """FIFO byte channels of one in-process cluster (transport.py:228-248)."""

    def __init__(self, P: int):
        self.P = P
        self._queues: dict = {}
        self._lock = threading.Lock()
        self.aborted = False

    def channel(self, src: int, dst: int, tag: int) -> queue.SimpleQueue:
        key = (src, dst, tag)
        with self._lock:
            q = self._queues.get(key)
            if q is None:
                q = self._queues[key] = queue.SimpleQueue()
            return q

    def abort(self) -> None:
        self.aborted = True


class LocalEndpoint(Endpoint):
    def __init__(self, rank, world_size, router: _LocalRouter, group, timeout):
        super().__init__(rank, world_size, timeout)
        self._router = router
        self.group = group

    def _send_impl(self, dest, tag, payload):
        if self._router.aborted:
            raise TransportError("cluster aborted")
        self._router.channel(self.rank, dest, tag).put(payload)

    def _recv_impl(self, source, tag):
        q = self._router.channel(source, self.rank, tag)
        deadline = time.monotonic() + self.timeout
        while True:
            remaining = deadline - time.monotonic()
            if remaining <= 0:
                raise TransportError(f"rank {self.rank}: recv from {source} tag {tag} timed out")
            try:
                return q.get(timeout=min(0.1, remaining))
            except queue.Empty:
                if self._router.aborted:
                    raise TransportError("cluster aborted") from None

    def abort(self):
        self._router.abort()
        if self.group is not None:
            self.group.abort()


class LocalDeviceGroup:
    """Rendezvous for the in-process GPU collectives.

    Every rank thread deposits its operand, one leader thread runs the whole
    collective as a chain of kernels on one stream (no device-side waits
    between separately launched kernels -- they would not be guaranteed to
    be co-scheduled on one GPU), then every rank picks up its result.
    """

    def __init__(self, P: int, device=None, timeout: float = DEFAULT_TIMEOUT):
        self.P = P
        self._device = device
        self.timeout = timeout
        self._slots = [None] * P
        self._result = None
        self._error = None
        self._barrier = threading.Barrier(P)
        self.aborted = False

    @property
    def device(self):
        if self._device is None:
            from . import device as _dev

            self._device = _dev.default_device()
        return self._device

    def abort(self) -> None:
        self.aborted = True
        self._barrier.abort()

    def _wait(self) -> None:
        if self.aborted:
            raise TransportError("cluster aborted")
        try:
            self._barrier.wait(timeout=self.timeout)
        except threading.BrokenBarrierError:
            if self.aborted:
                raise TransportError("cluster aborted") from None
            raise TransportError("collective rendezvous timed out") from None

    def run(self, rank: int, operand, leader_fn):
        """Collective call: returns leader_fn(all operands) to every rank."""
        self._slots[rank] = operand
        self._wait()
        if rank == 0:
            try:
                self._result = leader_fn(list(self._slots))
                self._error = None
            except BaseException as exc:  # noqa: BLE001 - re-raised on every rank
                self._result = None
                self._error = exc
        self._wait()
        res, err = self._result, self._error
        self._slots[rank] = None
        self._wait()
        if err is not None:
            raise err
        return res


def create_local_cluster(P: int, timeout: float = DEFAULT_TIMEOUT, device=None) -> list[Endpoint]:
    """P mutually connected in-process endpoints (transport.py:279-284) that
    share one GPU device group."""
    if P < 1:
        raise ValueError(f"P must be >= 1, got {P}")
    router = _LocalRouter(P)
    group = LocalDeviceGroup(P, device, timeout)
    return [LocalEndpoint(r, P, router, group, timeout) for r in range(P)]


def run_workers(endpoints: list[Endpoint], fn) -> list:
    """Run fn(ep) on one thread per endpoint (transport.py:507-539); on any
    failure abort the cluster and re-raise the root cause (non-TransportError
    preferred, lowest rank first).  Worker threads inherit the caller's CUDA
    device."""
    results = [None] * len(endpoints)
    failures: dict[int, BaseException] = {}
    lock = threading.Lock()
    dev_idx = None
    try:
        import torch

        if torch.cuda.is_available():
            dev_idx = torch.cuda.current_device()
    except Exception:  # pragma: no cover
        dev_idx = None

    def runner(i: int, ep: Endpoint):
        try:
            if dev_idx is not None:
                import torch

                torch.cuda.set_device(dev_idx)
            results[i] = fn(ep)
        except BaseException as exc:  # noqa: BLE001
            with lock:
                failures[i] = exc
            for other in endpoints:
                other.abort()

    threads = [
        threading.Thread(target=runner, args=(i, ep), name=f"gtopk-b200-worker-{i}")
        for i, ep in enumerate(endpoints)
    ]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if failures:
        primary = [r for r, e in failures.items() if not isinstance(e, TransportError)]
        rank = min(primary) if primary else min(failures)
        raise failures[rank]
    return results
