"""One process per GPU (torchrun): the NVLink backend of the collectives.

`init_dist_cluster()` returns this rank's `DistEndpoint`.  torch.distributed
is the plumbing only:
  * NCCL carries the baselines (TopKAllReduce's allgather, the dense
    allreduce -- collectives.py:88-165),
  * a gloo group carries host bytes (Endpoint.send/recv, the CUDA IPC handle
    exchange, barriers).
gTopKAllReduce itself is ONE kernel per rank (`gtk_gtopk_exchange`): it
stores its accumulator into the partner's IPC-mapped inbox over NVLink as
self-validating low-latency records, polls its own inbox for the partner's
and merges (⊤), for every round of the schedule -- recursive-doubling butterfly for P = 2^n
(bitwise equal to the reference's tree + broadcast), the reference's exact
tree + binomial broadcast otherwise (collectives.py:206-217).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from . import collectives as _coll
from . import device as _dev
from .device import DeviceList, P
from .transport import DEFAULT_TIMEOUT, Endpoint, TransportError, TransportStats, sparse_msg_bytes


def _schedule(rank: int, world: int, mode: str):
    if mode == "auto":
        mode = "butterfly" if world & (world - 1) == 0 else "tree"
    if mode == "butterfly":
        return _coll.butterfly_schedule(rank, world), mode
    return _coll.tree_schedule(rank, world), mode


class _ExchangePlan:
    """Per-k resources of the fused exchange: own inbox (cudaMalloc,
    IPC-exported), the peers' mapped inboxes, accumulator and workspace."""

    def __init__(self, group: "DistDeviceGroup", k: int):
        lib = _lib.load()
        self.k = k
        steps, self.mode = _schedule(group.rank, group.world, group.mode)
        self.nsteps = len(steps)
        self.steps = steps
        sched = np.array([[s, r, mg, j] for j, (s, r, mg) in enumerate(steps)], dtype=np.int32).reshape(-1)
        self.schedule = (ctypes.c_int32 * max(len(sched), 1))(*sched.tolist())
        n_in = ctypes.c_size_t()
        _lib.check(lib.gtk_exchange_inbox_bytes(k, self.nsteps, ctypes.byref(n_in)))
        self.inbox = ctypes.c_void_p()
        _lib.check(lib.gtk_dev_alloc(n_in.value, ctypes.byref(self.inbox)))
        handle = np.zeros(64, dtype=np.uint8)
        _lib.check(lib.gtk_ipc_get_handle(self.inbox, handle.ctypes.data_as(ctypes.c_void_p)))
        allh = [torch.zeros(64, dtype=torch.uint8) for _ in range(group.world)]
        dist.all_gather(allh, torch.from_numpy(handle), group=group.gloo)
        W = group.world
        self.peer_inbox = (ctypes.c_void_p * W)()
        self._opened = []
        for r in range(W):
            if r == group.rank:
                self.peer_inbox[r] = self.inbox.value
                continue
            h = allh[r].numpy()
            pi = ctypes.c_void_p()
            _lib.check(lib.gtk_ipc_open_handle(h.ctypes.data_as(ctypes.c_void_p), ctypes.byref(pi)))
            self.peer_inbox[r] = pi.value
            self._opened.append(pi)
        dev = group.device
        self.acc = DeviceList(group.dim_hint, k, dev)
        self.ws = _dev.merge_workspace(k, k, dev)
        self.step_counts = torch.zeros(max(2 * self.nsteps, 2), dtype=torch.int32, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.epoch = torch.zeros(1, dtype=torch.int64, device=dev)  # advanced by the kernel
        self.tags = None  # u32[m] K3 membership tags (gtk_gtopk_exchange_update), allocated on first use
        # gtk_select_push: the first step's partner inbox (its step-0 slots),
        # and the schedule variant whose step 0 is marked as already pushed
        s0 = steps[0][0] if steps else -1
        self.push_slot0 = self.peer_inbox[s0] if s0 >= 0 else None
        if s0 >= 0:
            pre = sched.copy()
            pre[3] |= _lib.STEP_PREPUSHED
            self.schedule_prepushed = (ctypes.c_int32 * len(pre))(*pre.tolist())
        else:
            self.schedule_prepushed = None
        dist.barrier(group=group.gloo)  # every rank mapped every peer before first use
        self._gloo = group.gloo

    def close(self):
        """Unmap the peers' inboxes and free our own -- only once every rank's
        kernels are done with them: drain this device, then a host barrier
        (a peer may still be writing into our inbox until it has finished)."""
        lib = _lib.load()
        torch.cuda.synchronize(self.acc.device)
        try:
            dist.barrier(group=self._gloo)
        except Exception:  # noqa: BLE001 - a dead peer: nothing left to wait for
            pass
        for p in self._opened:
            lib.gtk_ipc_close_handle(p)
        self._opened = []
        if self.inbox:
            lib.gtk_dev_free(self.inbox)
            self.inbox = ctypes.c_void_p()


class DistDeviceGroup:
    """Device collectives for one rank of a torchrun job."""

    def __init__(self, rank: int, world: int, device: torch.device, gloo, timeout: float,
                 mode: str = "auto"):
        self.rank = rank
        self.world = world
        self.P = world
        self.device = device
        self.gloo = gloo
        self.timeout = timeout
        self.mode = mode
        self.dim_hint = 0
        self._plans: dict[int, _ExchangePlan] = {}
        self.aborted = False
        self.topk_status_in_band = True  # topk(apply=...) carries the select's status (optimizer.topk_step)
        # abort word: pinned host memory mapped into the device; the exchange
        # kernel polls it while it waits for a partner (transport.py:210-214)
        lib = _lib.load()
        self._abort_host = ctypes.POINTER(ctypes.c_uint32)()
        self._abort_dev = ctypes.POINTER(ctypes.c_uint32)()
        with torch.cuda.device(device):
            _lib.check(lib.gtk_abort_word_create(ctypes.byref(self._abort_host), ctypes.byref(self._abort_dev)),
                       "gtk_abort_word_create")

    def abort(self) -> None:
        """Wake this rank's waiting exchange kernel: it stops polling, the step
        raises TransportError("cluster aborted"); later calls raise at once."""
        self.aborted = True
        if self._abort_host:
            _lib.load().gtk_abort_word_set(self._abort_host, 1)

    def plan(self, k: int, dim: int) -> _ExchangePlan:
        p = self._plans.get(k)
        if p is None:
            self.dim_hint = dim
            p = self._plans[k] = _ExchangePlan(self, k)
        p.acc.dim = dim
        return p

    # -- gTopKAllReduce ----------------------------------------------------
    def gtopk(self, ep: Endpoint, lst: DeviceList, k: int, status: torch.Tensor | None = None,
              update=None) -> DeviceList:
        """Fused NVLink exchange; returns the plan's accumulator (valid until
        the next gtopk call with the same k).  update: see enqueue_exchange."""
        if self.aborted:
            raise TransportError("cluster aborted")
        plan = self.plan(k, lst.dim)
        if self.world == 1:
            if lst is not plan.acc:
                plan.acc.copy_from(lst)
            if update is not None:
                w, res, lr, scaling = update
                _dev.scatter_update(w, res, None, plan.acc, lst, lst.dim, lr, 0.0, 1, scaling, skip=status)
            return plan.acc
        st = status if status is not None else plan.status
        if status is None:
            st.zero_()
        self.enqueue_exchange(plan, lst, st, update=update)
        counts = plan.step_counts.clone()  # snapshot for lazy byte accounting
        for j, (s, r, _mg) in enumerate(plan.steps):
            if s >= 0:
                ep.stats.add_sparse(counts[2 * j:2 * j + 1], sent=True)
            if r >= 0:
                ep.stats.add_sparse(counts[2 * j + 1:2 * j + 2], sent=False)
        if status is None:
            word = int(st.item())
            _dev.raise_status(word)
        return plan.acc

    def enqueue_exchange(self, plan: _ExchangePlan, lst: DeviceList, status: torch.Tensor,
                         update=None, prepushed: bool = False) -> None:
        """Launch the fused exchange kernel on the current stream: plan.acc
        becomes the global top-k of every rank's `lst`.  No host sync; the
        launch is CUDA-graph capturable (device-side epoch).  update = (w,
        res, lr, scaling): K3's sparse form runs in the same kernel
        (gtk_gtopk_exchange_update; `lst` must not be plan.acc)."""
        src = None if lst is plan.acc else lst
        if prepushed and plan.schedule_prepushed is None:
            raise ValueError("no first-step partner to have pushed to")
        sched = plan.schedule_prepushed if prepushed else plan.schedule
        args = [self.rank, self.world, sched, plan.nsteps, plan.peer_inbox,
                P(plan.epoch), P(plan.acc.idx), P(plan.acc.val), P(plan.acc.count),
                plan.k, P(status), ctypes.cast(self._abort_dev, ctypes.c_void_p),
                ctypes.c_int64(int(self.timeout * 1e9)), P(plan.step_counts),
                P(src.idx if src else None), P(src.val if src else None), P(src.count if src else None),
                P(plan.ws), ctypes.c_size_t(plan.ws.numel())]
        if update is not None and src is not None and plan.nsteps > 0:
            w, res, lr, scaling = update
            if plan.tags is None or plan.tags.numel() < lst.dim:
                plan.tags = torch.zeros(lst.dim, dtype=torch.int32, device=self.device)  # membership tags
            _lib.call("gtk_gtopk_exchange_update", *args, P(w), P(res), ctypes.c_float(lr), scaling, P(plan.tags),
                      _dev.stream_of(self.device))
            return
        _lib.call("gtk_gtopk_exchange", *args, _dev.stream_of(self.device))
        if update is not None:  # (no exchange steps or in-place list: separate K3)
            w, res, lr, scaling = update
            _dev.scatter_update(w, res, None, plan.acc, lst, lst.dim, lr, 0.0, self.world, scaling, skip=status)

    # -- TopKAllReduce baseline: NCCL allgather + rank-order accumulation -----
    def topk(self, ep: Endpoint, lst: DeviceList, divide: bool = True, apply=None):
        """collectives.py:148-165: every rank's list (counts, then one packed
        all-gather of [idx | value bits] per rank), accumulated in rank order
        by gtk_topk_accumulate (scatter per rank, division at the touched
        entries only)."""
        W = self.world
        if apply is not None:
            # topk_step (w, lr, acc, status): every rank's list has the same capacity
            # (k), so one all-gather of [count | idx | value bits] per rank
            # carries the counts too -- no host read of the sizes -- and the
            # momentum-0 update runs at the touched entries only.  (Callers
            # pass the same k on every rank, like every step of the job.)
            # The select's status word travels in the same gather: any
            # rank's error voids the update everywhere (PEER_FAILED on the
            # healthy ranks) -- no host sync before the collective.
            w, lr, acc, status = apply
            cap = lst.cap
            stride = 2 * cap + 2
            mine = torch.empty(stride, dtype=torch.int32, device=self.device)
            mine[0:1].copy_(lst.n)
            mine[1:2].copy_(status[0:1])
            mine[2:2 + cap].copy_(lst.idx)
            mine[2 + cap:].copy_(lst.val.view(torch.int32))
            allv = torch.empty(W * stride, dtype=torch.int32, device=self.device)
            dist.all_gather_into_tensor(allv, mine)
            cnts = allv.view(W, stride)[:, 0].contiguous()
            _dev.topk_apply(allv[2:], allv[2 + cap:].view(torch.float32), cnts, W, stride, lst.dim, acc, w, lr,
                            divide, statuses=allv[1:], status_stride=stride, local_status=status[0:1])
            self._topk_stats(ep, cnts)
            return None
        cnts = torch.empty(W, dtype=torch.int32, device=self.device)
        dist.all_gather_into_tensor(cnts, lst.n)
        cap = max(int(cnts.max().item()), 1)  # (the gather's size: one host read)
        n = min(cap, lst.cap)
        mine = torch.empty(2 * cap, dtype=torch.int32, device=self.device)
        mine[:n].copy_(lst.idx[:n])
        mine[cap:cap + n].copy_(lst.val[:n].view(torch.int32))
        allv = torch.empty(W * 2 * cap, dtype=torch.int32, device=self.device)
        dist.all_gather_into_tensor(allv, mine)
        out = torch.empty(lst.dim, dtype=torch.float32, device=self.device)
        _dev.topk_accumulate(allv, allv[cap:].view(torch.float32), cnts, W, 2 * cap, lst.dim, out, divide=divide)
        self._topk_stats(ep, cnts)
        return out

    def _topk_stats(self, ep: Endpoint, cnts: torch.Tensor) -> None:
        """Ring-allgather accounting of the reference (collectives.py:140-144)."""
        W = self.world
        for s in range(W - 1):
            ep.stats.add_sparse(cnts[(self.rank - s) % W:(self.rank - s) % W + 1], sent=True)
            ep.stats.add_sparse(cnts[(self.rank - s - 1) % W:(self.rank - s - 1) % W + 1], sent=False)

    # -- dense baseline: NCCL allreduce (sum) -----------------------------------
    def dense(self, ep: Endpoint, g: torch.Tensor) -> torch.Tensor:
        W = self.world
        self._check_dims(g.numel())
        out = g.clone()
        if W > 1:
            dist.all_reduce(out, op=dist.ReduceOp.SUM)
        chunk = -(-g.numel() // W)
        ep.stats.msgs_sent += 2 * (W - 1)
        ep.stats.msgs_recv += 2 * (W - 1)
        ep.stats.bytes_sent += 2 * (W - 1) * chunk * 4
        ep.stats.bytes_recv += 2 * (W - 1) * chunk * 4
        return out

    # -- rank-order dense sum: NCCL allgather + one rank-ordered sum kernel ------
    def dense_rank_order(self, ep: Endpoint, g: torch.Tensor) -> torch.Tensor:
        """optimizer.py:105-115: the reference's allgather of whole vectors and
        +0-seeded accumulation in rank order (bitwise, unlike NCCL's sum)."""
        W, m = self.world, g.numel()
        self._check_dims(m)
        parts = torch.empty(W * m, dtype=torch.float32, device=self.device)
        if W > 1:
            dist.all_gather_into_tensor(parts, g)
        else:
            parts.copy_(g)
        out = torch.empty(m, dtype=torch.float32, device=self.device)
        _dev.dense_sum([parts[r * m:(r + 1) * m] for r in range(W)], m, out)
        ep.stats.msgs_sent += W - 1
        ep.stats.msgs_recv += W - 1
        ep.stats.bytes_sent += (W - 1) * 4 * m
        ep.stats.bytes_recv += (W - 1) * 4 * m
        return out

    def _check_dims(self, m: int) -> None:
        """ProtocolError on every rank when the ranks' vector lengths differ
        (collectives.py:113-117) -- checked before the size-dependent
        collective by one 2-element NCCL max-reduction of (m, -m), the same
        size on every rank (in place of a gloo all-gather of m)."""
        t = torch.tensor([m, -m], dtype=torch.int64).to(self.device, non_blocking=True)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        hi, neg_lo = t.tolist()
        if hi != m or -neg_lo != m:
            from .transport import ProtocolError

            raise ProtocolError("ring chunk size mismatch across ranks")

    def close(self) -> None:
        for p in self._plans.values():
            p.close()
        self._plans.clear()
        if self._abort_host:
            torch.cuda.synchronize(self.device)
            _lib.load().gtk_abort_word_destroy(self._abort_host)
            self._abort_host = ctypes.POINTER(ctypes.c_uint32)()


class DistEndpoint(Endpoint):
    """Endpoint of one torchrun rank; byte messages travel over gloo."""

    def __init__(self, rank: int, world_size: int, group, gloo, timeout: float = DEFAULT_TIMEOUT):
        super().__init__(rank, world_size, timeout)
        self.group = group
        self._gloo = gloo

    def _send_impl(self, dest, tag, payload):
        # non-blocking like the reference's queue put (transport.py:255-258):
        # gloo's blocking send would deadlock the dissemination barrier
        if self.group is not None and self.group.aborted:
            raise TransportError("endpoint aborted")
        self._pending = [(w, keep) for w, keep in getattr(self, "_pending", []) if not w.is_completed()]
        n = torch.tensor([len(payload)], dtype=torch.int64)
        self._pending.append((dist.isend(n, dest, group=self._gloo, tag=tag), n))
        if len(payload):
            buf = torch.frombuffer(bytearray(payload), dtype=torch.uint8)
            self._pending.append((dist.isend(buf, dest, group=self._gloo, tag=tag), buf))

    def _recv_impl(self, source, tag):
        n = torch.zeros(1, dtype=torch.int64)
        dist.recv(n, source, group=self._gloo, tag=tag)
        if int(n) == 0:
            return b""
        buf = torch.empty(int(n), dtype=torch.uint8)
        dist.recv(buf, source, group=self._gloo, tag=tag)
        return bytes(buf.numpy().tobytes())

    def abort(self):
        if self.group is not None:
            self.group.abort()

    def close(self):
        for w, _keep in getattr(self, "_pending", []):
            w.wait()
        self._pending = []
        if self.group is not None and hasattr(self.group, "close"):
            self.group.close()


def init_dist_cluster(timeout: float = DEFAULT_TIMEOUT, mode: str = "auto", device_collectives: bool = True):
    """Join the torchrun job (RANK/WORLD_SIZE/LOCAL_RANK/MASTER_* env) and
    return this rank's endpoint.  mode: "auto" | "butterfly" | "tree"."""
    backend = "nccl" if (device_collectives and torch.cuda.is_available()) else "gloo"
    if not dist.is_initialized():
        if backend == "nccl":
            local = int(os.environ.get("LOCAL_RANK", "0"))
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    gloo = dist.new_group(backend="gloo") if backend == "nccl" else dist.group.WORLD
    group = None
    if device_collectives:
        if not torch.cuda.is_available():
            raise _lib.NativeLibraryError("device collectives need a CUDA device")
        local = int(os.environ.get("LOCAL_RANK", str(rank % torch.cuda.device_count())))
        group = DistDeviceGroup(rank, world, torch.device("cuda", local), gloo, timeout, mode)
    return DistEndpoint(rank, world, group, gloo, timeout)
