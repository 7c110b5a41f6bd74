"""One-GPU loopback parity of the multi-GPU gTopKAllReduce device path.

The fused NVLink exchange kernel (`gtk_gtopk_exchange[_update]`,
csrc/gtk_comm.cu) of rank r only ever READS its own inbox and WRITES its
partners' inboxes.  So one GPU can run any rank of any P exactly as it runs in
a torchrun job: the test allocates rank r's inbox and pre-fills, for every
step of r's schedule, the low-latency (LL) records the oracle says r's partner
sends at that step; the partners' inboxes are local scratch buffers, decoded
afterwards.  Checked bitwise against the oracle (reference collectives.py:
188-219 reduce tree + :168-185 binomial broadcast, sparse.py:157-195 top_op,
optimizer.py:227-230/243 extra residual + update):

  * the global top-k every rank ends with (acc idx / val / count),
  * every list rank r pushes, step by step -- including the merge output the
    kernel pushes to the NEXT partner as it writes it (fused send), and the
    broadcast forwarding of the tree schedule,
  * the fused K3: w at the global entries, residual at the local entries that
    missed the global set, the membership tags, and the message counts,
  * poison (a partner sends count -1): PEER_FAILED, poison forwarded, K3
    skipped; self-poison; the host abort word and the %globaltimer timeout,
  * gtk_select_push: K1's finish writes the selection as step-0 LL records,
    and the exchange then runs with GTK_STEP_PREPUSHED.

LL record layout (include/gtopk_b200.h, gtk_gtopk_exchange): slot (step s,
call parity p) of an inbox starts at (2 s + p) * slot_bytes(k), slot_bytes(k)
= round_up(16 + 16 k, 256); a 16-byte header {count | tag << 32, k-th-key hint
| tag << 32}, then per entry {idx | tag << 32, value bits | tag << 32}; tag =
the call's epoch (= device epoch counter + 1).
"""

import ctypes
import time

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA GPU")]

F32 = np.float32
U64 = np.uint64
DEV_NONFINITE, DEV_TIMEOUT, DEV_ABORTED, DEV_PEER_FAILED = 0x1, 0x4, 0x8, 0x10
POISON = 0xFFFFFFFF


def slot_bytes(k):
    return (16 + 16 * k + 255) & ~255


def key_of(v):
    return np.asarray(v, F32).view(np.uint32) & 0x7FFFFFFF


def hint_of(idx, val, k):
    """the k-th-key hint a full list carries (0 = none)"""
    return int(key_of(val).min()) if len(idx) == k else 0


def encode_slot(k, tag, idx, val, count=None, hint=None):
    """LL words (uint64) of one inbox slot."""
    n = len(idx)
    w = np.zeros(slot_bytes(k) // 8, dtype=U64)
    t = U64(tag) << U64(32)
    c = n if count is None else count
    w[0] = U64(c) | t
    w[1] = U64(hint_of(idx, val, k) if hint is None else hint) | t
    if n:
        w[2:2 + 2 * n:2] = np.asarray(idx, U64) | t
        w[3:3 + 2 * n:2] = np.asarray(val, F32).view(np.uint32).astype(U64) | t
    return w


def decode_slot(words, k, tag):
    """(count, hint, idx, val) of a slot; asserts every word carries `tag`."""
    words = np.asarray(words, U64)
    assert int(words[0]) >> 32 == tag and int(words[1]) >> 32 == tag, "header not written for this call"
    n = int(words[0]) & 0xFFFFFFFF
    hint = int(words[1]) & 0xFFFFFFFF
    if n == POISON:
        return n, hint, None, None
    body = words[2:2 + 2 * n]
    assert np.all((body >> U64(32)) == U64(tag)), "stale entry record"
    idx = (body[0::2] & U64(0xFFFFFFFF)).astype(U64)
    val = (body[1::2] & U64(0xFFFFFFFF)).astype(np.uint32).view(F32)
    return n, hint, idx, val


# ---------------------------------------------------------------------------
# expected per-step traffic: every rank of the schedule simulated with the oracle


def simulate(lists, k, schedules):
    """schedules[q] = rank q's steps (send_to, recv_from, merge).  Returns
    (sent[q][s], received[q][s], final[q]) with lists as (idx u64, val f32)."""
    from oracle import gtopk_oracle as orc

    P = len(lists)
    cur = [(np.asarray(i, U64), np.asarray(v, F32)) for i, v in lists]
    nsteps = len(schedules[0])
    sent = [[None] * nsteps for _ in range(P)]
    recv = [[None] * nsteps for _ in range(P)]
    for s in range(nsteps):
        msgs = {}
        for q in range(P):
            to, _frm, _mg = schedules[q][s]
            if to >= 0:
                msgs[(q, to)] = cur[q]
                sent[q][s] = cur[q]
        nxt = list(cur)
        for q in range(P):
            _to, frm, mg = schedules[q][s]
            if frm >= 0:
                got = msgs[(frm, q)]
                recv[q][s] = got
                nxt[q] = orc.top_op(got[0], got[1], cur[q][0], cur[q][1], k) if mg else got
        cur = nxt
    return sent, recv, cur


def schedules_for(P, mode):
    from paper_1901_04359_b200 import collectives as coll

    if mode == "butterfly":
        return [coll.butterfly_schedule(q, P) for q in range(P)]
    return [coll.tree_schedule(q, P) for q in range(P)]


# ---------------------------------------------------------------------------
# one rank's exchange call on this GPU


class Loopback:
    """Rank `rank` of a P-rank schedule with its inbox and the partners'
    (scratch) inboxes in local device memory."""

    def __init__(self, rank, P, steps, k, m, prepushed=False):
        import torch

        from paper_1901_04359_b200 import _lib
        from paper_1901_04359_b200 import device as dv

        self.torch, self.lib, self.dv = torch, _lib.load(), dv
        self.d = torch.device("cuda", 0)
        self.rank, self.P, self.steps, self.k, self.m = rank, P, steps, k, m
        self.nsteps = len(steps)
        nb = ctypes.c_size_t()
        assert self.lib.gtk_exchange_inbox_bytes(k, self.nsteps, ctypes.byref(nb)) == 0
        self.words = nb.value // 8
        assert nb.value == 2 * self.nsteps * slot_bytes(k)
        # inbox[q] for every rank: own inbox at [rank], scratch for the others
        self.inbox = [torch.zeros(self.words, dtype=torch.int64, device=self.d) for _ in range(P)]
        self.peer = (ctypes.c_void_p * P)(*[t.data_ptr() for t in self.inbox])
        sched = []
        for j, (to, frm, mg) in enumerate(steps):
            sched += [to, frm, mg, j | (0x10000 if (prepushed and j == 0) else 0)]
        self.sched = (ctypes.c_int32 * max(len(sched), 1))(*sched)
        self.epoch = torch.zeros(1, dtype=torch.int64, device=self.d)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.d)
        self.counts = torch.zeros(2 * max(self.nsteps, 1), dtype=torch.int32, device=self.d)
        self.acc = dv.DeviceList(m, k, self.d)
        self.ws = dv.merge_workspace(k, k, self.d)
        self.tags = torch.zeros(m, dtype=torch.int32, device=self.d)

    def slot_range(self, s, par):
        w = slot_bytes(self.k) // 8
        o = (2 * s + par) * w
        return o, o + w

    def prefill(self, s, tag, words):
        o0, o1 = self.slot_range(s, tag & 1)
        self.inbox[self.rank][o0:o1].copy_(self.torch.from_numpy(words.view(np.int64)).to(self.d))

    def sent_slot(self, s, tag):
        to = self.steps[s][0]
        o0, o1 = self.slot_range(s, tag & 1)
        return self.inbox[to][o0:o1].cpu().numpy().view(U64)

    def call(self, local, w=None, res=None, lr=0.0, scaling=0, timeout_s=20.0, abort_dev=None, local_on_dev=None):
        """The exchange (+ fused K3 when w is given) on `local`, like one
        DistDeviceGroup.enqueue_exchange call."""
        dv, P_ = self.dv, self.dv.P
        if local_on_dev is None:
            local_on_dev = dv.DeviceList.from_host(self.m, local[0], local[1], self.d, self.k)
            local_on_dev.count[1] = hint_of(local[0], local[1], self.k)
        self.lst = local_on_dev
        args = [self.rank, self.P, self.sched, self.nsteps, self.peer, P_(self.epoch), P_(self.acc.idx),
                P_(self.acc.val), P_(self.acc.count), self.k, P_(self.status),
                ctypes.c_void_p(abort_dev) if abort_dev else None, ctypes.c_int64(int(timeout_s * 1e9)),
                P_(self.counts), P_(local_on_dev.idx), P_(local_on_dev.val), P_(local_on_dev.count), P_(self.ws),
                ctypes.c_size_t(self.ws.numel())]
        st = dv.stream_of(self.d)
        if w is None:
            rc = self.lib.gtk_gtopk_exchange(*args, st)
        else:
            rc = self.lib.gtk_gtopk_exchange_update(*args, P_(w), P_(res), ctypes.c_float(lr), scaling,
                                                    P_(self.tags), st)
        assert rc == 0, rc
        self.torch.cuda.synchronize()
        return int(self.status.item())


def _lists(rng, P, m, k, kind):
    from oracle import gtopk_oracle as orc

    base = rng.standard_normal(m).astype(F32)
    out = []
    for q in range(P):
        if kind == "normal":
            g = rng.standard_normal(m).astype(F32)
        elif kind == "ties":
            g = rng.integers(-3, 4, m).astype(F32)
        else:  # odd ranks cancel even ranks exactly on shared indices
            g = base if q % 2 == 0 else -base
        out.append(orc.top_k_select(g, k)[:2])
    return out


def bits(a):
    return np.asarray(a, F32).view(np.uint32)


def check_rank(rank, P, mode, lists, k, m, rng, calls=2):
    """Run rank `rank` for `calls` consecutive exchange calls (both inbox
    parities); each call's traffic and result are checked."""
    from oracle import gtopk_oracle as orc

    scheds = schedules_for(P, mode)
    steps = scheds[rank]
    lb = Loopback(rank, P, steps, k, m)
    want_i, want_v = orc.tree_fold(lists, k)
    for call in range(calls):
        tag = call + 1
        sent, recv, final = simulate(lists, k, scheds)
        for s, got in enumerate(recv[rank]):
            if got is not None:
                lb.prefill(s, tag, encode_slot(k, tag, *got))
        lb.status.zero_()
        word = lb.call(lists[rank])
        assert word == 0, hex(word)
        ai, av = lb.acc.to_host()
        # every rank ends with the reference's rank-0 fold, bitwise
        assert np.array_equal(ai, want_i), (rank, P, mode, call)
        assert np.array_equal(bits(av), bits(want_v)), (rank, P, mode, call)
        assert np.array_equal(ai, final[rank][0]) and np.array_equal(bits(av), bits(final[rank][1]))
        # every push of this rank, step by step (fused next-step sends included)
        counts = lb.counts.cpu().numpy()
        for s, msg in enumerate(sent[rank]):
            if msg is None:
                continue
            n, hint, si, sv_ = decode_slot(lb.sent_slot(s, tag), k, tag)
            assert n == len(msg[0]) and counts[2 * s] == n, (rank, s)
            assert np.array_equal(si, msg[0]) and np.array_equal(bits(sv_), bits(msg[1])), (rank, P, mode, s)
            assert hint in (0, hint_of(msg[0], msg[1], k))
        for s, got in enumerate(recv[rank]):
            if got is not None:
                assert counts[2 * s + 1] == len(got[0])
        assert int(lb.epoch.item()) == tag
        # the next call's lists (the other inbox parity)
        lists = _lists(rng, P, m, k, "normal")
        want_i, want_v = orc.tree_fold(lists, k)


@pytest.mark.parametrize("P,mode", [(2, "butterfly"), (4, "butterfly"), (8, "butterfly"), (2, "tree"),
                                    (3, "tree"), (4, "tree"), (5, "tree"), (8, "tree")])
def test_exchange_loopback_every_rank(P, mode):
    rng = np.random.default_rng(1000 + P)
    m, k = 200_003, 1500
    for rank in range(P):
        for kind in ("normal", "ties", "cancel"):
            lists = _lists(rng, P, m, k, kind)
            check_rank(rank, P, mode, lists, k, m, rng, calls=2 if kind == "normal" else 1)


@pytest.mark.parametrize("P,mode,k", [(4, "butterfly", 25_600), (3, "tree", 25_600), (2, "butterfly", 270),
                                      (8, "butterfly", 270), (2, "butterfly", 200_000)])
def test_exchange_loopback_sizes(P, mode, k):
    """The headline k (25.6K), ResNet-20's k = 270 and a large-k list whose
    union slices exceed the minimum shared-memory capacity."""
    rng = np.random.default_rng(7 + k)
    m = max(270_000, 10 * k)
    lists = _lists(rng, P, m, k, "normal")
    for rank in sorted({0, P // 2, P - 1}):
        check_rank(rank, P, mode, lists, k, m, rng, calls=1)


def _k3_expect(w0, res0, local, glob, lr, P, scaling):
    w = w0.copy()
    res = res0.copy()
    gi = np.asarray(glob[0], np.int64)
    u = glob[1] / F32(P) if scaling == 0 else glob[1]
    w[gi] = w[gi] - F32(lr) * u.astype(F32)
    li = np.asarray(local[0], np.int64)
    miss = ~np.isin(li, gi)
    res[li[miss]] = res[li[miss]] + local[1][miss]
    return w, res


@pytest.mark.parametrize("P,mode", [(2, "butterfly"), (4, "butterfly"), (3, "tree"), (8, "tree")])
def test_exchange_update_fused_k3(P, mode):
    """gtk_gtopk_exchange_update: optimizer.py:227-230 (extra residual) and
    :243 (w -= lr * global / P) inside the exchange kernel, bitwise."""
    import torch

    from oracle import gtopk_oracle as orc

    rng = np.random.default_rng(31 + P)
    m, k, lr = 150_000, 900, 0.05
    scheds = schedules_for(P, mode)
    for rank in range(P):
        grads = [rng.standard_normal(m).astype(F32) for _ in range(P)]
        sels = [orc.top_k_select(g, k) for g in grads]
        lists = [(s[0], s[1]) for s in sels]
        lb = Loopback(rank, P, scheds[rank], k, m)
        tag = 1
        _sent, recv, final = simulate(lists, k, scheds)
        for s, got in enumerate(recv[rank]):
            if got is not None:
                lb.prefill(s, tag, encode_slot(k, tag, *got))
        w0 = rng.standard_normal(m).astype(F32)
        res0 = sels[rank][2]  # the select's residual: zeros at the local winners
        w = torch.from_numpy(w0.copy()).cuda()
        res = torch.from_numpy(res0.copy()).cuda()
        for scaling in (0,):
            word = lb.call(lists[rank], w=w, res=res, lr=float(F32(lr)), scaling=scaling)
            assert word == 0
            ew, er = _k3_expect(w0, res0, lists[rank], final[rank], lr, P, scaling)
            assert np.array_equal(bits(w.cpu().numpy()), bits(ew)), (P, mode, rank)
            assert np.array_equal(bits(er), bits(res.cpu().numpy())), (P, mode, rank)
            tags = lb.tags.cpu().numpy().astype(np.uint32)
            member = np.zeros(m, bool)
            member[np.asarray(final[rank][0], np.int64)] = True
            assert np.all(tags[member] == tag) and not np.any(tags[~member] == tag)


@pytest.mark.parametrize("deferred", [False, True])
def test_exchange_poison_received_forwarded_and_k3_skipped(deferred):
    """A partner's count -1 (its K1 saw NaN/Inf): PEER_FAILED, every later
    send of this rank carries count -1, w and the residual stay untouched --
    also for the deferred step (res = NULL), whose final merge applies the w
    update itself."""
    import torch

    from oracle import gtopk_oracle as orc

    P, m, k = 4, 80_000, 300
    rng = np.random.default_rng(5)
    lists = _lists(rng, P, m, k, "normal")
    scheds = schedules_for(P, "butterfly")
    for rank in (0, 3):
        lb = Loopback(rank, P, scheds[rank], k, m)
        tag = 1
        _sent, recv, _final = simulate(lists, k, scheds)
        lb.prefill(0, tag, encode_slot(k, tag, [], [], count=POISON, hint=0))  # step 0: poisoned partner
        for s in range(1, lb.nsteps):
            lb.prefill(s, tag, encode_slot(k, tag, *recv[rank][s]))
        w0 = np.ones(m, F32)
        res0 = rng.standard_normal(m).astype(F32)
        w = torch.from_numpy(w0.copy()).cuda()
        res = torch.from_numpy(res0.copy()).cuda()
        word = lb.call(lists[rank], w=w, res=None if deferred else res, lr=0.1)
        assert word & DEV_PEER_FAILED and not word & (DEV_TIMEOUT | DEV_ABORTED)
        assert np.array_equal(w.cpu().numpy(), w0) and np.array_equal(res.cpu().numpy(), res0)
        n, _h, _i, _v = decode_slot(lb.sent_slot(1, tag), k, tag)  # the poison is forwarded
        assert n == POISON
    # self-poison: this rank's select flagged NONFINITE -> it sends count -1
    # itself (the status word is not cleared: the kernel reads it at entry)
    import ctypes as ct

    lb = Loopback(1, 2, schedules_for(2, "butterfly")[1], k, m)
    lb.prefill(0, 1, encode_slot(k, 1, *lists[0]))
    lb.status.fill_(DEV_NONFINITE)
    lst = lb.dv.DeviceList.from_host(m, lists[1][0], lists[1][1], lb.d, k)
    P_ = lb.dv.P
    rc = lb.lib.gtk_gtopk_exchange(1, 2, lb.sched, lb.nsteps, lb.peer, P_(lb.epoch), P_(lb.acc.idx),
                                   P_(lb.acc.val), P_(lb.acc.count), k, P_(lb.status), None,
                                   ct.c_int64(int(5e9)), P_(lb.counts), P_(lst.idx), P_(lst.val), P_(lst.count),
                                   P_(lb.ws), ct.c_size_t(lb.ws.numel()), lb.dv.stream_of(lb.d))
    assert rc == 0
    torch.cuda.synchronize()
    n, _h, _i, _v = decode_slot(lb.sent_slot(0, 1), k, 1)
    assert n == POISON


def test_exchange_timeout_and_host_abort():
    """Nothing ever arrives: the %globaltimer deadline raises TIMEOUT; with a
    long deadline the host abort word stops the wait within a fraction of a
    second (reference transport.py:210-214: abort wakes blocked peers)."""
    import threading

    from paper_1901_04359_b200 import _lib

    P, m, k = 2, 10_000, 50
    rng = np.random.default_rng(9)
    lists = _lists(rng, P, m, k, "normal")
    steps = schedules_for(P, "butterfly")[0]
    lb = Loopback(0, P, steps, k, m)
    t0 = time.monotonic()
    word = lb.call(lists[0], timeout_s=0.05)
    assert word & DEV_TIMEOUT and time.monotonic() - t0 < 5.0
    lib = _lib.load()
    host = ctypes.POINTER(ctypes.c_uint32)()
    devp = ctypes.POINTER(ctypes.c_uint32)()
    assert lib.gtk_abort_word_create(ctypes.byref(host), ctypes.byref(devp)) == 0
    try:
        lb2 = Loopback(0, P, steps, k, m)
        timer = threading.Timer(0.3, lambda: lib.gtk_abort_word_set(host, 1))
        timer.start()
        t0 = time.monotonic()
        word = lb2.call(lists[0], timeout_s=60.0, abort_dev=ctypes.cast(devp, ctypes.c_void_p).value)
        took = time.monotonic() - t0
        timer.join()
        assert word & DEV_ABORTED and not word & DEV_TIMEOUT
        assert took < 10.0, took  # far below the 60 s deadline
        with pytest.raises(Exception):
            from paper_1901_04359_b200 import device as dv

            dv.raise_status(word)
    finally:
        lib.gtk_abort_word_destroy(host)


@pytest.mark.parametrize("P", [2, 4])
def test_select_push_then_prepushed_exchange(P):
    """The pipeline's N > 1 step on rank r: gtk_select_push (K1 whose finish
    writes the selection as step-0 LL records into the first partner's inbox)
    then gtk_gtopk_exchange_update with GTK_STEP_PREPUSHED; checked against
    the oracle: the pushed records, the global list, w and the residual."""
    import torch

    from oracle import gtopk_oracle as orc

    m, k, lr = 300_000, 300, 0.1
    rng = np.random.default_rng(77 + P)
    scheds = schedules_for(P, "butterfly")
    for rank in range(P):
        res_prev = (rng.standard_normal(m) * 0.5).astype(F32)
        grads = [rng.standard_normal(m).astype(F32) for _ in range(P)]
        accs = [(res_prev + g).astype(F32) if q == rank else g for q, g in enumerate(grads)]
        sels = [orc.top_k_select(a, k) for a in accs]
        lists = [(s[0], s[1]) for s in sels]
        lb = Loopback(rank, P, scheds[rank], k, m, prepushed=True)
        tag = 1
        _sent, recv, final = simulate(lists, k, scheds)
        for s, got in enumerate(recv[rank]):
            if got is not None:
                lb.prefill(s, tag, encode_slot(k, tag, *got))
        d = lb.d
        rin = torch.from_numpy(res_prev).to(d)
        gd = torch.from_numpy(grads[rank]).to(d)
        rout = torch.empty_like(gd)
        sel = lb.dv.DeviceList(m, k, d)
        win = lb.dv.new_window(d)
        part = scheds[rank][0][0]
        lb.dv.select_push(rin, gd, rout, k, sel, lb.status, win, lb.inbox[part].data_ptr(), lb.epoch)
        torch.cuda.synchronize()
        assert int(lb.status.item()) == 0
        # step 0's records, written by K1's finish
        n, hint, si, sv_ = decode_slot(lb.sent_slot(0, tag), k, tag)
        assert n == k and np.array_equal(si, lists[rank][0]) and np.array_equal(bits(sv_), bits(lists[rank][1]))
        assert hint == hint_of(*lists[rank], k)
        assert np.array_equal(bits(rout.cpu().numpy()), bits(sels[rank][2]))
        w0 = rng.standard_normal(m).astype(F32)
        w = torch.from_numpy(w0.copy()).to(d)
        word = lb.call(None, w=w, res=rout, lr=float(F32(lr)), local_on_dev=sel)
        assert word == 0
        ai, av = lb.acc.to_host()
        assert np.array_equal(ai, final[rank][0]) and np.array_equal(bits(av), bits(final[rank][1]))
        ew, er = _k3_expect(w0, sels[rank][2], lists[rank], final[rank], lr, P, 0)
        assert np.array_equal(bits(w.cpu().numpy()), bits(ew))
        assert np.array_equal(bits(rout.cpu().numpy()), bits(er))
        # a non-finite gradient: the finish sends count -1 to the first partner
        gbad = grads[rank].copy()
        gbad[123] = np.nan
        lb.status.zero_()
        lb.dv.select_push(rin, torch.from_numpy(gbad).to(d), rout, k, sel, lb.status, win,
                          lb.inbox[part].data_ptr(), lb.epoch)
        torch.cuda.synchronize()
        assert int(lb.status.item()) & DEV_NONFINITE
        n, _h, _i, _v = decode_slot(lb.sent_slot(0, tag + 1), k, tag + 1)
        assert n == POISON


@pytest.mark.parametrize("P,k,grid", [(2, 1500, "auto"), (4, 1500, "auto"), (4, 25_600, "auto"),
                                      (2, 270, "auto"), (4, 3000, "grid")])
def test_exchange_successive_calls_carried_windows(P, k, grid, monkeypatch):
    """Successive calls of one exchange plan: every merge step carries its
    key window from the previous call (csrc/gtk_merge.cuh, MergeWindowRec).
    The call sequence drives steady windows (same distribution), misses
    (every value scaled x8: the k-th key jumps out of the window), massive
    ties (integer gradients: thousands of keys equal to the k-th) and
    cancellations (fewer than k union entries); every call's global list is
    checked bitwise against the oracle's tree fold, with the fused K3."""
    import torch

    from oracle import gtopk_oracle as orc

    if grid == "grid":  # the cooperative grid path (cluster merges are the default at this k)
        monkeypatch.setenv("GTK_MERGE_CLUSTER", "0")
    rng = np.random.default_rng(4242 + P + k)
    m = max(200_000, 12 * k)
    scheds = schedules_for(P, "butterfly")
    rank = P - 1
    lb = Loopback(rank, P, scheds[rank], k, m)
    w = torch.zeros(m, device=lb.d)
    res = torch.zeros(m, device=lb.d)
    seq = ["normal", "normal", "normal", "scaled", "scaled", "normal", "ties", "normal", "cancel", "normal",
           "normal"]
    for call, kind in enumerate(seq):
        tag = call + 1
        if kind == "scaled":
            lists = [(i, (v * F32(8.0 ** (call - 2))).astype(F32)) for i, v in _lists(rng, P, m, k, "normal")]
        else:
            lists = _lists(rng, P, m, k, kind)
        _sent, recv, final = simulate(lists, k, scheds)
        for s, got in enumerate(recv[rank]):
            if got is not None:
                lb.prefill(s, tag, encode_slot(k, tag, *got))
        lb.status.zero_()
        w0 = w.cpu().numpy()
        res0 = res.cpu().numpy()
        word = lb.call(lists[rank], w=w, res=res, lr=0.01)
        assert word == 0, (call, kind, hex(word))
        want_i, want_v = orc.tree_fold(lists, k)
        ai, av = lb.acc.to_host()
        assert np.array_equal(ai, want_i), (P, k, call, kind)
        assert np.array_equal(bits(av), bits(want_v)), (P, k, call, kind)
        ew, er = _k3_expect(w0, res0, lists[rank], final[rank], 0.01, P, 0)
        assert np.array_equal(bits(w.cpu().numpy()), bits(ew)), (P, k, call, kind)
        assert np.array_equal(bits(res.cpu().numpy()), bits(er)), (P, k, call, kind)


@pytest.mark.parametrize("P,kind", [(2, "normal"), (4, "normal"), (2, "ties")])
def test_deferred_p_gt_1_step_chain(P, kind):
    """The deferred P > 1 step on rank P - 1, partners emulated by the loopback
    inbox: gtk_select_push_deferred (winners pending, selection pushed, the
    previous step's winners settled by membership of the previous global
    list) then gtk_gtopk_exchange_update with res = NULL (w only).  Step by
    step against the oracle's P-rank trajectory (optimizer.py:199-252): the
    pushed selection, the global list, w, and the settled residual."""
    import torch

    from oracle import gtopk_oracle as orc

    m, k, lr = 200_003, 400, 0.05
    rng = np.random.default_rng(900 + P + (kind == "ties"))
    rank = P - 1
    scheds = schedules_for(P, "butterfly")
    lb = Loopback(rank, P, scheds[rank], k, m, prepushed=True)
    d = lb.d
    dv = lb.dv
    states = [orc.State(np.zeros(m, F32), lr) for _ in range(P)]
    R = [torch.zeros(m, device=d), torch.empty(m, device=d)]
    w = torch.zeros(m, device=d)
    wins = [dv.new_window(d) for _ in range(2)]
    wss = [dv.select_workspace(m, k, d, slot=31 + i) for i in range(2)]
    sels = [dv.DeviceList(m, k, d) for _ in range(2)]
    part = scheds[rank][0][0]
    cur = 0
    for t in range(8):
        tag = t + 1
        if kind == "ties":
            grads = [rng.integers(-3, 4, m).astype(F32) for _ in range(P)]
        else:
            grads = [rng.standard_normal(m).astype(F32) for _ in range(P)]
        # the oracle's step for every rank; what each rank sends at each step
        before = [(s.weights.copy(), s.residual.copy()) for s in states]
        (gi, gv), local = orc.gtopk_step_all(states, grads, k)
        _sent, recv, final = simulate([(i, v) for i, v in local], k, scheds)
        for s, got in enumerate(recv[rank]):
            if got is not None:
                lb.prefill(s, tag, encode_slot(k, tag, *got))
        par = t % 2
        lb.status.zero_()
        dv.select_push_deferred(R[cur], torch.from_numpy(grads[rank]).to(d), R[1 - cur], k, sels[par], lb.status,
                                wins[par], wss[par], sels[1 - par] if t else None, wss[1 - par], lb.tags,
                                lb.inbox[part].data_ptr(), lb.epoch)
        word = lb.call(None, w=w, res=None, lr=float(F32(lr)), local_on_dev=sels[par])
        assert word & 0x3D == 0, (t, hex(word))
        # the pushed selection (step 0 records written by K1's finish)
        n, _h, si, sv_ = decode_slot(lb.sent_slot(0, tag), k, tag)
        assert n == len(local[rank][0]) and np.array_equal(si, local[rank][0]), (P, kind, t)
        assert np.array_equal(bits(sv_), bits(local[rank][1])), (P, kind, t)
        ai, av = lb.acc.to_host()
        assert np.array_equal(ai, gi) and np.array_equal(bits(av), bits(gv)), (P, kind, t)
        assert np.array_equal(bits(w.cpu().numpy()), bits(states[rank].weights)), (P, kind, t)
        cur = 1 - cur
        settled = R[cur].clone()
        dv.settle_global(settled, sels[par], lb.tags, lb.epoch)
        assert np.array_equal(bits(settled.cpu().numpy()), bits(states[rank].residual)), (P, kind, t)
        del before
