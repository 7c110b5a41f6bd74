"""TCP mesh backend (paper_1901_04359_b200/tcp.py) on CPU: configuration,
mesh formation, the reference's frame format byte for byte, FIFO matching,
barrier, peer loss, abort, and -- in this container, where the reference is
importable -- a mixed mesh of this package's ranks and the reference's own
TcpEndpoint ranks (pkg/src/gtopk/transport.py:286-500)."""

import os
import socket
import struct
import sys
import threading
import time

import pytest

from paper_1901_04359_b200 import tcp
from paper_1901_04359_b200.transport import TransportError

REF_SRC = "/root/reference/pkg/src"


def free_ports(n):
    socks, ports = [], []
    for _ in range(n):
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        socks.append(s)
        ports.append(s.getsockname()[1])
    for s in socks:
        s.close()
    return ports


def mesh(P, timeout=10.0, connect=None):
    """P endpoints on 127.0.0.1, formed concurrently (one thread per rank)."""
    addrs = [("127.0.0.1", p) for p in free_ports(P)]
    cfg = tcp.ClusterConfig(P, "tcp", addrs, timeout)
    eps, errs = [None] * P, []

    def join(r):
        try:
            eps[r] = (connect[r] if connect else tcp.connect_tcp_cluster)(cfg, r)
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)

    ts = [threading.Thread(target=join, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return eps


def run_all(eps, fn):
    out, errs = [None] * len(eps), []

    def body(i):
        try:
            out[i] = fn(eps[i])
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)

    ts = [threading.Thread(target=body, args=(i,)) for i in range(len(eps))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(30)
    if errs:
        raise errs[0]
    return out


def test_cluster_config_validation():
    assert tcp.ClusterConfig(2).backend == "local"
    with pytest.raises(ValueError):
        tcp.ClusterConfig(0)
    with pytest.raises(ValueError):
        tcp.ClusterConfig(2, "udp")
    with pytest.raises(ValueError):
        tcp.ClusterConfig(2, "tcp", [("h", 1)])
    with pytest.raises(ValueError):
        tcp.connect_tcp_cluster(tcp.ClusterConfig(2), 0)
    with pytest.raises(ValueError):
        tcp.connect_tcp_cluster(tcp.ClusterConfig(1, "tcp", [("127.0.0.1", 1)]), 1)


def test_load_hosts_file(tmp_path):
    p = tmp_path / "hosts"
    p.write_text("# ranks\n1 b 5001\n\n0 a 5000\n")
    assert tcp.load_hosts_file(p) == [("a", 5000), ("b", 5001)]
    for bad in ("0 a\n", "0 a 1\n0 b 2\n", "0 a 1\n2 b 2\n"):
        p.write_text(bad)
        with pytest.raises(ValueError):
            tcp.load_hosts_file(p)


@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_mesh_send_recv_fifo_barrier(P):
    eps = mesh(P)
    try:
        def body(ep):
            for d in range(P):
                if d != ep.rank:
                    for i in range(3):  # FIFO per (source, tag), tags independent
                        ep.send(d, 7, bytes([ep.rank, d, i]))
                    ep.send(d, 9, b"")
            got = {}
            for s in range(P):
                if s != ep.rank:
                    assert ep.recv(s, 9) == b""
                    got[s] = [ep.recv(s, 7) for _ in range(3)]
            ep.barrier()
            return got

        res = run_all(eps, body)
        for r in range(P):
            for s, msgs in res[r].items():
                assert msgs == [bytes([s, r, i]) for i in range(3)]
        ep0 = eps[0]
        assert ep0.stats.msgs_sent >= 4 * (P - 1)
        assert ep0.stats.bytes_sent >= 9 * (P - 1)
    finally:
        for ep in eps:
            ep.close()


def test_byte_collectives_over_tcp():
    from paper_1901_04359_b200 import collectives as coll

    P = 4
    eps = mesh(P)
    try:
        gathered = run_all(eps, lambda ep: coll.allgather(ep, bytes([ep.rank]) * (ep.rank + 1)))
        for g in gathered:
            assert g == [bytes([r]) * (r + 1) for r in range(P)]
        got = run_all(eps, lambda ep: coll.binomial_bcast(ep, 2, b"root" if ep.rank == 2 else None))
        assert got == [b"root"] * P
    finally:
        for ep in eps:
            ep.close()


class FakePeer:
    """Rank 0 of a P = 2 mesh spoken by hand, to pin the wire bytes."""

    def __init__(self):
        self.port0, self.port1 = free_ports(2)
        self.lst = socket.socket()
        self.lst.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
        self.lst.bind(("127.0.0.1", self.port0))
        self.lst.listen(1)
        cfg = tcp.ClusterConfig(2, "tcp", [("127.0.0.1", self.port0), ("127.0.0.1", self.port1)], 5.0)
        box = {}
        t = threading.Thread(target=lambda: box.setdefault("ep", tcp.connect_tcp_cluster(cfg, 1)))
        t.start()
        self.conn, _ = self.lst.accept()
        self.announce = self._read(4)
        t.join()
        self.ep = box["ep"]

    def _read(self, n):
        buf = b""
        while len(buf) < n:
            c = self.conn.recv(n - len(buf))
            assert c
            buf += c
        return buf

    def close(self):
        self.ep.close()
        self.conn.close()
        self.lst.close()


def test_wire_bytes_match_reference_format():
    f = FakePeer()
    try:
        assert f.announce == struct.pack("<I", 1)  # transport.py:468
        f.ep.send(0, 0x4001, b"\x01\x02\x03")
        assert f._read(19) == struct.pack("<IIII", 0x6754524E, 1, 0x4001, 3) + b"\x01\x02\x03"
        # frames split at arbitrary byte boundaries reassemble
        frame = struct.pack("<IIII", 0x6754524E, 0, 5, 4) + b"wxyz"
        for i in range(len(frame)):
            f.conn.sendall(frame[i:i + 1])
            time.sleep(0.001)
        f.conn.sendall(struct.pack("<IIII", 0x6754524E, 0, 6, 0))
        assert f.ep.recv(0, 5) == b"wxyz"
        assert f.ep.recv(0, 6) == b""
    finally:
        f.close()


def test_bad_magic_and_wrong_source_fail_the_link():
    for hdr in (struct.pack("<IIII", 0xDEADBEEF, 0, 1, 0), struct.pack("<IIII", 0x6754524E, 3, 1, 0)):
        f = FakePeer()
        try:
            f.conn.sendall(hdr)
            with pytest.raises(TransportError, match="lost"):
                f.ep.recv(0, 1)
        finally:
            f.close()


def test_peer_loss_wakes_receiver_promptly():
    f = FakePeer()
    try:
        f.conn.sendall(struct.pack("<IIII", 0x6754524E, 0, 2, 1) + b"z")
        f.conn.close()
        t0 = time.monotonic()
        assert f.ep.recv(0, 2) == b"z"  # delivered before the loss
        with pytest.raises(TransportError, match="lost"):
            f.ep.recv(0, 2)
        assert time.monotonic() - t0 < 2.0  # not the 5 s timeout
        with pytest.raises(TransportError):
            f.ep.send(0, 2, b"x")
    finally:
        f.close()


def test_abort_wakes_blocked_recv():
    eps = mesh(2, timeout=20.0)
    try:
        err = []

        def waiter():
            try:
                eps[1].recv(0, 3)
            except TransportError as exc:
                err.append(exc)

        t = threading.Thread(target=waiter)
        t0 = time.monotonic()
        t.start()
        time.sleep(0.2)
        eps[1].abort()
        t.join(5)
        assert err and "aborted" in str(err[0])
        assert time.monotonic() - t0 < 5.0
        # the surviving rank sees its link to the aborted rank lost
        with pytest.raises(TransportError, match="lost"):
            eps[0].recv(1, 3)
    finally:
        for ep in eps:
            ep.close()


def test_recv_timeout_and_missing_rank():
    eps = mesh(2, timeout=0.3)
    try:
        with pytest.raises(TransportError, match="timed out"):
            eps[0].recv(1, 1)
    finally:
        for ep in eps:
            ep.close()
    port = free_ports(2)
    cfg = tcp.ClusterConfig(2, "tcp", [("127.0.0.1", port[0]), ("127.0.0.1", port[1])], 0.5)
    with pytest.raises(TransportError, match="rank\\(s\\) 1"):
        tcp.connect_tcp_cluster(cfg, 0)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference sources not present")
def test_mixed_mesh_with_reference_ranks():
    """Ranks 0 and 2 run the reference's TcpEndpoint, ranks 1 and 3 this
    package's: one mesh, byte messages, barrier, allgather and broadcast of
    both implementations interleaved."""
    sys.path.insert(0, REF_SRC)
    try:
        from gtopk import collectives as ref_coll
        from gtopk import transport as ref_tp
    finally:
        sys.path.remove(REF_SRC)
    from paper_1901_04359_b200 import collectives as coll

    def ref_connect(cfg, r):
        return ref_tp.connect_tcp_cluster(ref_tp.ClusterConfig(cfg.P, "tcp", cfg.addresses, cfg.timeout), r)

    P = 4
    eps = mesh(P, connect=[ref_connect, tcp.connect_tcp_cluster, ref_connect, tcp.connect_tcp_cluster])
    try:
        def body(ep):
            c = ref_coll if ep.rank % 2 == 0 else coll
            ep.barrier()
            g = c.allgather(ep, b"r%d" % ep.rank)
            b = c.binomial_bcast(ep, 1, b"from-1" if ep.rank == 1 else None)
            ep.barrier()
            return g, b

        for g, b in run_all(eps, body):
            assert g == [b"r%d" % r for r in range(P)]
            assert b == b"from-1"
    finally:
        for ep in eps:
            ep.close()


def test_duplicate_announcement_is_protocol_error():
    """reference pkg/tests/test_transport.py:232-253."""
    from paper_1901_04359_b200.transport import ProtocolError

    ports = free_ports(3)
    cfg = tcp.ClusterConfig(3, "tcp", [("127.0.0.1", p) for p in ports], 5.0)
    err = {}

    def node0():
        try:
            tcp.connect_tcp_cluster(cfg, 0)
        except Exception as exc:  # noqa: BLE001
            err["exc"] = exc

    t = threading.Thread(target=node0)
    t.start()
    time.sleep(0.2)
    socks = []
    for _ in range(2):  # two sockets both claim rank 1
        s = socket.create_connection(("127.0.0.1", ports[0]), timeout=5)
        s.sendall(struct.pack("<I", 1))
        socks.append(s)
    t.join(10)
    for s in socks:
        s.close()
    assert isinstance(err.get("exc"), ProtocolError)
