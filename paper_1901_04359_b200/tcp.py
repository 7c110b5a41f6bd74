"""Multi-host backend: the reference's TCP mesh (pkg/src/gtopk/transport.py:
85-133, 286-500) with the collectives' arithmetic on this host's GPU.

Within one box the product path is `init_dist_cluster()` (one process per
GPU, the fused NVLink exchange kernel).  Across boxes there is no peer
memory, so this backend stages each message through host memory:

    device list --D2H--> encode_sparse bytes --TCP--> decode --H2D--> K2 merge

The wire is the reference's, byte for byte, so a rank of this package and
a rank of the reference interoperate on one mesh:

  * frames: magic 0x6754524E | source rank | tag | payload length | payload,
    4-byte little-endian header fields (transport.py:1-11, :370-373);
  * mesh formation: every rank listens on its configured address, dials
    every lower rank and announces itself with a 4-byte little-endian rank,
    accepts every higher rank (transport.py:416-500);
  * message pattern and tags of every collective: gTopKAllReduce is the
    reduce tree on tag 0x4000 + j then the binomial broadcast from rank 0 on
    0x5000 + j (collectives.py:188-219, :168-185); TopKAllReduce the ring
    allgather on 0x3000 + step (:131-165); the dense allreduce the ring
    reduce-scatter / allgather on 0x1000 / 0x2000 + step (:88-128).

Each merge / accumulation runs on the GPU (K2 `gtk_top_op`, the TopK
accumulation kernel, the dense ring's chunk adds), in the reference's
operand order, so results are bitwise the reference's.

Design (not the reference's): one receive thread per endpoint multiplexes
every peer socket with `selectors` (the reference runs a reader thread per
peer) and parses frames incrementally into a per-endpoint mailbox -- one
condition variable over per-(source, tag) FIFOs, so receivers sleep instead
of polling, and a lost peer or an abort wakes exactly the receivers it
concerns.  Mesh formation dials the lower ranks while a helper thread
accepts the higher ones, so neither side of the handshake serialises the
other.
"""

from __future__ import annotations

import collections
import logging
import selectors
import socket
import struct
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from .transport import (
    DEFAULT_TIMEOUT,
    FRAME_MAGIC,
    Endpoint,
    ProtocolError,
    TransportError,
    decode_sparse,
    encode_sparse,
)

log = logging.getLogger("gtopk_b200.tcp")

_HDR = struct.Struct("<IIII")  # magic, source, tag, length
_RANK = struct.Struct("<I")

# collective tag bases of the reference (collectives.py:29-33)
TAG_RING_RS = 0x1000
TAG_RING_AG = 0x2000
TAG_GATHER = 0x3000
TAG_GTOPK = 0x4000
TAG_BCAST = 0x5000


# ---------------------------------------------------------------------------
# configuration (transport.py:90-133)
# ---------------------------------------------------------------------------


@dataclass
class ClusterConfig:
    """Worker count and backend; "tcp" needs one (host, port) per rank."""

    P: int
    backend: str = "local"
    addresses: list[tuple[str, int]] = field(default_factory=list)
    timeout: float = DEFAULT_TIMEOUT

    def __post_init__(self):
        if self.P < 1:
            raise ValueError(f"P must be >= 1, got {self.P}")
        if self.backend not in ("local", "tcp"):
            raise ValueError(f"unknown backend {self.backend!r}")
        if self.backend == "tcp" and len(self.addresses) != self.P:
            raise ValueError(f"tcp backend needs {self.P} addresses, got {len(self.addresses)}")


def load_hosts_file(path) -> list[tuple[str, int]]:
    """'rank host port' per line ('#' comments and blank lines skipped);
    ranks must cover 0..P-1 exactly once.  Returns [(host, port)] by rank."""
    by_rank: dict[int, tuple[str, int]] = {}
    with open(path, encoding="utf-8") as fh:
        for no, raw in enumerate(fh, 1):
            text = raw.strip()
            if not text or text.startswith("#"):
                continue
            fields = text.split()
            if len(fields) != 3:
                raise ValueError(f"{path}:{no}: expected 'rank host port'")
            r, host, port = int(fields[0]), fields[1], int(fields[2])
            if r in by_rank:
                raise ValueError(f"{path}:{no}: duplicate rank {r}")
            by_rank[r] = (host, port)
    if set(by_rank) != set(range(len(by_rank))):
        raise ValueError(f"{path}: ranks must be 0..P-1 without gaps")
    return [by_rank[r] for r in range(len(by_rank))]


# ---------------------------------------------------------------------------
# mailbox + frame parser
# ---------------------------------------------------------------------------


class _Mailbox:
    """Delivered frames of one endpoint, keyed by (source, tag)."""

    def __init__(self):
        self._cv = threading.Condition()
        self._fifo: dict = collections.defaultdict(collections.deque)
        self.lost: dict[int, str] = {}  # source -> reason its connection ended
        self.aborted = False

    def deliver(self, src: int, tag: int, payload: bytes) -> None:
        with self._cv:
            self._fifo[(src, tag)].append(payload)
            self._cv.notify_all()

    def peer_lost(self, src: int, reason: str) -> None:
        with self._cv:
            self.lost.setdefault(src, reason)
            self._cv.notify_all()

    def abort(self) -> None:
        with self._cv:
            self.aborted = True
            self._cv.notify_all()

    def take(self, src: int, tag: int, timeout: float, rank: int) -> bytes:
        key = (src, tag)
        with self._cv:
            self._cv.wait_for(lambda: self.aborted or src in self.lost or bool(self._fifo.get(key)), timeout)
            if self.aborted:
                raise TransportError("endpoint aborted")
            q = self._fifo.get(key)
            if q:  # frames that arrived before the peer went away are still delivered
                return q.popleft()
            if src in self.lost:
                raise TransportError(f"connection to rank {src} lost: {self.lost[src]}")
            raise TransportError(f"rank {rank}: recv from {src} tag {tag} timed out")


class _FrameParser:
    """Incremental frame decoder for one peer's byte stream."""

    __slots__ = ("peer", "buf")

    def __init__(self, peer: int):
        self.peer = peer
        self.buf = bytearray()

    def feed(self, data: bytes):
        """Append bytes; yield every complete (tag, payload).  Raises
        ProtocolError on a bad magic or a frame claiming another source."""
        self.buf += data
        while len(self.buf) >= _HDR.size:
            magic, src, tag, length = _HDR.unpack_from(self.buf, 0)
            if magic != FRAME_MAGIC:
                raise ProtocolError(f"bad frame magic 0x{magic:08X}")
            if src != self.peer:
                raise ProtocolError(f"frame claims source {src}, expected {self.peer}")
            end = _HDR.size + length
            if len(self.buf) < end:
                return
            payload = bytes(self.buf[_HDR.size:end])
            del self.buf[:end]
            yield tag, payload


# ---------------------------------------------------------------------------
# endpoint
# ---------------------------------------------------------------------------


class TcpEndpoint(Endpoint):
    """One rank of a TCP mesh (transport.py:338-413): framed byte messages
    to every peer; the device group stages the collectives through it."""

    def __init__(self, rank: int, world_size: int, sockets: dict[int, socket.socket],
                 timeout: float = DEFAULT_TIMEOUT, device=None):
        super().__init__(rank, world_size, timeout)
        self._socks = dict(sockets)
        self._tx_locks = {r: threading.Lock() for r in self._socks}
        self._box = _Mailbox()
        self._closing = False
        self._wake_r, self._wake_w = socket.socketpair()
        self._wake_r.setblocking(False)
        self._rx = threading.Thread(target=self._receive_loop, daemon=True, name=f"gtopk-tcp-rx-{rank}")
        if self._socks:
            self._rx.start()
        if device is not None:
            self.group = HostStagedGroup(self, device)

    # -- receive side: one thread, all peers ------------------------------
    def _receive_loop(self) -> None:
        sel = selectors.DefaultSelector()
        sel.register(self._wake_r, selectors.EVENT_READ, None)
        for peer, s in self._socks.items():
            s.setblocking(False)
            sel.register(s, selectors.EVENT_READ, _FrameParser(peer))
        live = len(self._socks)
        try:
            while live and not self._closing:
                for key, _ in sel.select():
                    parser = key.data
                    if parser is None:  # close()/abort() woke us
                        return
                    reason = None
                    try:
                        data = key.fileobj.recv(1 << 20)
                        if not data:
                            reason = "connection closed" if not parser.buf else "connection closed mid-frame"
                        else:
                            for tag, payload in parser.feed(data):
                                self._box.deliver(parser.peer, tag, payload)
                    except (BlockingIOError, InterruptedError):
                        continue
                    except ProtocolError as exc:
                        reason = str(exc)
                    except OSError as exc:
                        reason = str(exc)
                    if reason is not None:
                        sel.unregister(key.fileobj)
                        live -= 1
                        self._box.peer_lost(parser.peer, reason)
        finally:
            sel.close()

    # -- plug points of Endpoint -------------------------------------------
    def _send_impl(self, dest: int, tag: int, payload: bytes) -> None:
        if self._box.aborted:
            raise TransportError("endpoint aborted")
        if dest in self._box.lost:
            raise TransportError(f"connection to rank {dest} lost: {self._box.lost[dest]}")
        frame = _HDR.pack(FRAME_MAGIC, self.rank, tag, len(payload)) + payload
        sock = self._socks[dest]
        view = memoryview(frame)
        deadline = time.monotonic() + self.timeout
        try:
            with self._tx_locks[dest]:
                # the socket is non-blocking (shared with the receive thread):
                # wait for buffer space with select, bounded by the timeout
                while view:
                    try:
                        sent = sock.send(view)
                        view = view[sent:]
                    except (BlockingIOError, InterruptedError):
                        left = deadline - time.monotonic()
                        if left <= 0 or self._box.aborted:
                            raise TransportError(f"send to rank {dest} timed out") from None
                        with selectors.DefaultSelector() as ws:
                            ws.register(sock, selectors.EVENT_WRITE)
                            ws.select(min(left, 0.5))
        except OSError as exc:
            raise TransportError(f"send to rank {dest} failed: {exc}") from exc

    def _recv_impl(self, source: int, tag: int) -> bytes:
        return self._box.take(source, tag, self.timeout, self.rank)

    def abort(self) -> None:
        """Fail this rank's blocked and future send/recv with TransportError and
        drop the connections (peers see their link to this rank lost)."""
        self._box.abort()
        self.close()

    def close(self) -> None:
        if self._closing:
            return
        self._closing = True
        try:
            self._wake_w.send(b"x")
        except OSError:
            pass
        if self._rx.is_alive():
            self._rx.join(timeout=5.0)
        for s in self._socks.values():
            for op in (lambda: s.shutdown(socket.SHUT_RDWR), s.close):
                try:
                    op()
                except OSError:
                    pass
        self._wake_r.close()
        self._wake_w.close()
        g = self.group
        if g is not None and hasattr(g, "close"):
            g.close()


# ---------------------------------------------------------------------------
# mesh formation (transport.py:416-500)
# ---------------------------------------------------------------------------


def _dial(addr, deadline: float, my_rank: int, peer: int) -> socket.socket:
    while True:
        left = deadline - time.monotonic()
        if left <= 0:
            raise TransportError(f"rank {my_rank}: timeout connecting to rank {peer} at {addr[0]}:{addr[1]}")
        try:
            s = socket.create_connection(addr, timeout=min(1.0, left))
        except OSError:
            time.sleep(0.05)
            continue
        s.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
        s.settimeout(None)
        s.sendall(_RANK.pack(my_rank))
        return s


def connect_tcp_cluster(cfg: ClusterConfig, my_rank: int, device=None) -> TcpEndpoint:
    """Join the mesh as `my_rank`: listen, dial every lower rank (announcing
    our rank), accept every higher rank (reading its announcement).  Returns
    once all P-1 links are up.  TransportError on timeout (naming the missing
    ranks), ProtocolError on a duplicate, unexpected or truncated
    announcement.  device: the GPU the collectives run on (default: the
    current CUDA device when one is present; None on a CPU-only host gives a
    byte-only endpoint)."""
    if cfg.backend != "tcp":
        raise ValueError("connect_tcp_cluster requires a tcp ClusterConfig")
    if not 0 <= my_rank < cfg.P:
        raise ValueError(f"rank {my_rank} out of range [0, {cfg.P})")
    device = _default_device(device)
    if cfg.P == 1:
        return TcpEndpoint(my_rank, 1, {}, cfg.timeout, device)
    deadline = time.monotonic() + cfg.timeout
    listener = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
    listener.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
    links: dict[int, socket.socket] = {}
    try:
        listener.bind(tuple(cfg.addresses[my_rank]))
        listener.listen(cfg.P)
        # the accepts of higher ranks run in a helper thread while this one dials
        higher = set(range(my_rank + 1, cfg.P))
        accepted: dict[int, socket.socket] = {}
        failure: list[BaseException] = []

        def accept_all():
            try:
                while higher - set(accepted):
                    left = deadline - time.monotonic()
                    if left <= 0:
                        miss = ",".join(str(r) for r in sorted(higher - set(accepted)))
                        raise TransportError(f"rank {my_rank}: timeout waiting for rank(s) {miss}")
                    listener.settimeout(min(1.0, left))
                    try:
                        s, _ = listener.accept()
                    except socket.timeout:
                        continue
                    s.settimeout(max(0.1, min(5.0, cfg.timeout)))
                    raw = b""
                    while len(raw) < _RANK.size:
                        chunk = s.recv(_RANK.size - len(raw))
                        if not chunk:
                            s.close()
                            raise ProtocolError("peer closed before rank announcement")
                        raw += chunk
                    (peer,) = _RANK.unpack(raw)
                    if peer == my_rank or peer in accepted:
                        s.close()
                        raise ProtocolError(f"duplicate rank announcement: {peer}")
                    if peer not in higher:
                        s.close()
                        raise ProtocolError(f"unexpected rank announcement: {peer}")
                    s.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
                    s.settimeout(None)
                    accepted[peer] = s
            except BaseException as exc:  # re-raised on the caller's thread
                failure.append(exc)

        acceptor = threading.Thread(target=accept_all, daemon=True)
        acceptor.start()
        try:
            for peer in range(my_rank):
                links[peer] = _dial(tuple(cfg.addresses[peer]), deadline, my_rank, peer)
        finally:
            acceptor.join()
            links.update(accepted)
        if failure:
            raise failure[0]
    except BaseException:
        for s in links.values():
            s.close()
        raise
    finally:
        listener.close()
    log.debug("rank %d: mesh of %d peers up", my_rank, len(links))
    return TcpEndpoint(my_rank, cfg.P, links, cfg.timeout, device)


def _default_device(device):
    if device is not None:
        import torch

        return torch.device(device)
    try:
        import torch

        if torch.cuda.is_available():
            return torch.device("cuda", torch.cuda.current_device())
    except ImportError:
        pass
    return None


# ---------------------------------------------------------------------------
# host-staged device collectives
# ---------------------------------------------------------------------------


def _ceil_log2(P: int) -> int:
    return (P - 1).bit_length()


class HostStagedGroup:
    """Device group of a TCP endpoint: the interface `collectives` and
    `optimizer` dispatch on (gtopk / topk / dense / dense_rank_order), with
    the messages staged through host bytes and the arithmetic on `device`."""

    def __init__(self, ep: TcpEndpoint, device):
        import torch

        self.ep = ep
        self.device = torch.device(device)
        self.world = self.P = ep.world_size
        self.rank = ep.rank
        self.aborted = False

    def abort(self) -> None:
        self.aborted = True

    # -- helpers -------------------------------------------------------------
    def _send_list(self, ep, dest: int, tag: int, lst) -> None:
        from .sparse import SparseVector

        i, v = lst.to_host()
        ep.send(dest, tag, encode_sparse(SparseVector(lst.dim, i, v)))

    def _recv_list(self, ep, src: int, tag: int, dim: int, cap: int):
        from .device import DeviceList

        s = decode_sparse(ep.recv(src, tag), dim)
        return DeviceList.from_host(dim, s.indices, s.values, self.device, max(cap, s.nnz))

    # -- gTopKAllReduce: reduce tree + binomial broadcast (collectives.py:188-219)
    def gtopk(self, ep, lst, k: int, status=None, update=None):
        from . import device as _dev

        if self.aborted:
            raise TransportError("cluster aborted")
        if status is not None:  # a local select error raises before the collective
            _dev.raise_status(int(status[0].item()))
        P, r = self.world, self.rank
        acc = lst.clone(cap=max(k, lst.cap))
        for j in range(1, _ceil_log2(P) + 1):
            half, span = 1 << (j - 1), 1 << j
            if r % span == half:
                self._send_list(ep, r - half, TAG_GTOPK + j, acc)
            elif r % span == 0 and r + half < P:
                got = self._recv_list(ep, r + half, TAG_GTOPK + j, lst.dim, k)
                _dev.top_op(got, acc, k, acc)  # ⊤(received, own)
        # binomial broadcast of rank 0's fold (collectives.py:168-185)
        for j in range(1, _ceil_log2(P) + 1):
            half = 1 << (j - 1)
            if r < half:
                if r + half < P:
                    self._send_list(ep, r + half, TAG_BCAST + j, acc)
            elif r < 2 * half:
                acc = self._recv_list(ep, r - half, TAG_BCAST + j, lst.dim, k)
        if update is not None:
            w, res, lr, scaling = update
            _dev.scatter_update(w, res, None, acc, lst, lst.dim, lr, 0.0, P, scaling, skip=status)
        return acc

    # -- ring allgather of byte blocks (collectives.py:131-145) ---------------
    def _allgather(self, ep, mine: bytes) -> list[bytes]:
        P, r = self.world, self.rank
        blocks: list = [None] * P
        blocks[r] = mine
        for step in range(P - 1):
            ep.send((r + 1) % P, TAG_GATHER + step, blocks[(r - step) % P])
            blocks[(r - step - 1) % P] = ep.recv((r - 1) % P, TAG_GATHER + step)
        return blocks

    # -- TopKAllReduce: allgather + rank-order accumulation (collectives.py:148-165)
    def topk(self, ep, lst, divide: bool = True, apply=None):
        import torch

        from . import device as _dev
        from .sparse import SparseVector

        i, v = lst.to_host()
        parts = [decode_sparse(b, lst.dim) for b in self._allgather(ep, encode_sparse(SparseVector(lst.dim, i, v)))]
        for s in parts:
            if s.dim != lst.dim:
                raise ProtocolError("sparse dim mismatch in topk_allreduce")
        P = self.world
        cap = max(max(s.nnz for s in parts), 1)
        idx = np.zeros((P, cap), dtype=np.int32)
        val = np.zeros((P, cap), dtype=np.float32)
        cnt = np.zeros(P, dtype=np.int32)
        for q, s in enumerate(parts):
            idx[q, : s.nnz] = s.indices
            val[q, : s.nnz] = s.values
            cnt[q] = s.nnz
        d = self.device
        ti, tv, tc = torch.from_numpy(idx).to(d), torch.from_numpy(val).to(d), torch.from_numpy(cnt).to(d)
        if apply is not None:  # (w, lr, acc): topk_step's momentum-0 update, touched entries only
            w, lr, acc = apply[:3]  # (the status was checked before the collective)
            _dev.topk_apply(ti, tv, tc, P, cap, lst.dim, acc, w, lr, divide)
            return None
        out = torch.empty(lst.dim, dtype=torch.float32, device=d)
        _dev.topk_accumulate(ti, tv, tc, P, cap, lst.dim, out, divide=divide)
        return out

    # -- dense ring allreduce (collectives.py:88-128): chunk adds on the GPU ----
    def dense(self, ep, g):
        import torch

        P, r, m = self.world, self.rank, g.numel()
        if P == 1:
            return g.clone()
        chunk = -(-m // P)
        buf = torch.zeros(chunk * P, dtype=torch.float32, device=self.device)
        buf[:m].copy_(g)

        def exchange(tag: int, send_c: int):
            ep.send((r + 1) % P, tag, buf[send_c * chunk:(send_c + 1) * chunk].cpu().numpy().tobytes())
            raw = ep.recv((r - 1) % P, tag)
            if len(raw) != chunk * 4:
                raise ProtocolError(f"ring chunk size mismatch: got {len(raw)} bytes, expected {chunk * 4}")
            return torch.frombuffer(bytearray(raw), dtype=torch.float32).to(self.device)

        for step in range(P - 1):
            c = (r - step - 1) % P
            incoming = exchange(TAG_RING_RS + step, (r - step) % P)
            buf[c * chunk:(c + 1) * chunk].add_(incoming)
        for step in range(P - 1):
            c = (r - step) % P
            buf[c * chunk:(c + 1) * chunk].copy_(exchange(TAG_RING_AG + step, (r - step + 1) % P))
        return buf[:m].clone()

    # -- rank-order dense sum (optimizer.py:105-115): allgather + one kernel ---
    def dense_rank_order(self, ep, g):
        import torch

        from . import device as _dev

        m = g.numel()
        blocks = self._allgather(ep, g.detach().to(torch.float32).cpu().numpy().tobytes())
        parts = []
        for b in blocks:
            if len(b) != 4 * m:
                raise ProtocolError(f"dense dim mismatch: got {len(b) // 4}, expected {m}")
            parts.append(torch.frombuffer(bytearray(b), dtype=torch.float32).to(self.device))
        out = torch.empty(m, dtype=torch.float32, device=self.device)
        _dev.dense_sum(parts, m, out)
        return out

    def close(self) -> None:
        pass
