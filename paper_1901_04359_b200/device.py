"""Device-side plumbing: sparse lists in HBM, workspaces, and thin wrappers
over the C-ABI kernels (`_lib`).  PyTorch is used only for device memory and
streams; every computation is a kernel of `libgtopk_b200.so`.

Device sparse list layout (one per rank per buffer): int32 idx[cap],
float32 val[cap], int32 count[1] -- index-ascending, count on the device so a
chain select -> merge rounds -> update never synchronises with the host.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

from . import _lib

U64 = np.uint64
F32 = np.float32


def require_cuda() -> None:
    _lib.load()
    if not torch.cuda.is_available():
        raise _lib.NativeLibraryError(
            "no CUDA device visible: the gTop-k hot path runs only on the GPU (no CPU fallback)"
        )


def default_device() -> torch.device:
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def P(t) -> ctypes.c_void_p:
    """Raw device pointer of a tensor (or NULL)."""
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


def stream_of(device: torch.device) -> ctypes.c_void_p:
    """torch's current stream on `device` as a raw cudaStream_t (the direct
    binding: torch.cuda.current_stream() costs ~10 us of Python per call)."""
    idx = device.index if device.index is not None else torch.cuda.current_device()
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(idx))


class DeviceList:
    """Index-sorted sparse list resident on one GPU."""

    __slots__ = ("dim", "cap", "idx", "val", "count", "device")

    def __init__(self, dim: int, cap: int, device: torch.device):
        self.dim = int(dim)
        self.cap = int(max(cap, 1))
        self.device = device
        self.idx = torch.empty(self.cap, dtype=torch.int32, device=device)
        self.val = torch.empty(self.cap, dtype=torch.float32, device=device)
        # {count, k-th key hint (0 = unknown)}: the hint lets a later merge
        # histogram a narrow key window in a single round
        self.count = torch.zeros(2, dtype=torch.int32, device=device)

    @classmethod
    def from_host(cls, dim, indices, values, device, cap=None) -> "DeviceList":
        indices = np.asarray(indices)
        n = int(indices.size)
        lst = cls(dim, max(n, cap or 0, 1), device)
        if n:
            lst.idx[:n].copy_(torch.from_numpy(indices.astype(np.int32)), non_blocking=False)
            lst.val[:n].copy_(torch.from_numpy(np.asarray(values, dtype=F32)), non_blocking=False)
        lst.count[0] = n
        lst.count[1] = 0
        return lst

    @property
    def n(self) -> torch.Tensor:
        """The 1-element device count (view)."""
        return self.count[0:1]

    def nnz(self) -> int:
        return int(self.count[0].item())

    def to_host(self):
        n = self.nnz()
        idx = self.idx[:n].cpu().numpy().astype(U64)
        val = self.val[:n].cpu().numpy().astype(F32)
        return idx, val

    def copy_from(self, other: "DeviceList") -> None:
        n = min(self.cap, other.cap)
        self.idx[:n].copy_(other.idx[:n], non_blocking=True)
        self.val[:n].copy_(other.val[:n], non_blocking=True)
        self.count.copy_(other.count, non_blocking=True)

    def clone(self, cap=None) -> "DeviceList":
        out = DeviceList(self.dim, cap or self.cap, self.device)
        out.copy_from(self)
        return out


# ---------------------------------------------------------------------------
# workspaces: one cache per host thread (one stream per worker thread), so
# concurrent ranks in one process never share a workspace.
# ---------------------------------------------------------------------------

_tls = threading.local()


def _cache() -> dict:
    c = getattr(_tls, "ws", None)
    if c is None:
        c = _tls.ws = {}
    return c


def _new_ws(nbytes: int, device) -> torch.Tensor:
    buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
    _lib.call("gtk_workspace_init", P(buf), ctypes.c_size_t(buf.numel()), stream_of(device))
    return buf


def select_workspace(m: int, k: int, device, slot: int = 0) -> torch.Tensor:
    """Select workspace for (m, k) on `device`; `slot` > 0 gives separate ones
    (deferred selects alternate two: gtk_select_update_deferred)."""
    key = ("select", device.index, m, k, slot)
    c = _cache()
    ws = c.get(key)
    if ws is None:
        n = ctypes.c_size_t()
        _lib.call("gtk_select_workspace_bytes", m, k, ctypes.byref(n))
        ws = c[key] = _new_ws(n.value, device)
    return ws


def merge_workspace(cap: int, k: int, device) -> torch.Tensor:
    key = ("merge", device.index, cap)
    c = _cache()
    ws = c.get(key)
    if ws is None:
        n = ctypes.c_size_t()
        _lib.call("gtk_merge_workspace_bytes", cap, k, ctypes.byref(n))
        ws = c[key] = _new_ws(n.value, device)
    return ws


# ---------------------------------------------------------------------------
# kernel wrappers
# ---------------------------------------------------------------------------


def new_window(device) -> torch.Tensor:
    """Per-parameter key-window record for select(window=...): uint32[8], zero
    = none yet (gtk_select_windowed)."""
    return torch.zeros(8, dtype=torch.int32, device=device)


def select(res_in, grad: torch.Tensor, res_out: torch.Tensor, k: int, out: DeviceList,
           status: torch.Tensor, force_exact: bool = False, window: torch.Tensor | None = None) -> None:
    """K1: res_out = res_in + grad (or grad), out = exact top-k of it, res_out
    zeroed at the winners.  Stream-ordered, no host sync.  `window` (from
    new_window, one per parameter) carries the key window between the
    successive selections of one residual; results are identical either way."""
    m = grad.numel()
    dev = grad.device
    ws = select_workspace(m, k, dev)
    _lib.call(
        "gtk_select_windowed", P(res_in), P(grad), P(res_out), m, k, P(out.idx), P(out.val), P(out.count),
        P(status), P(ws), ctypes.c_size_t(ws.numel()),
        _lib.SELECT_FORCE_EXACT if force_exact else 0, P(window), stream_of(dev),
    )


def select_push(res_in, grad: torch.Tensor, res_out: torch.Tensor, k: int, out: DeviceList,
                status: torch.Tensor, window: torch.Tensor | None, peer_slot0: int, epoch: torch.Tensor) -> None:
    """K1 whose selection also goes straight to the exchange's first partner
    (gtk_select_push): peer_slot0 = that partner's mapped inbox, epoch = the
    exchange plan's device epoch.  The next exchange runs prepushed."""
    m = grad.numel()
    dev = grad.device
    ws = select_workspace(m, k, dev)
    _lib.call(
        "gtk_select_push", P(res_in), P(grad), P(res_out), m, k, P(out.idx), P(out.val), P(out.count),
        P(status), P(ws), ctypes.c_size_t(ws.numel()), 0, P(window), ctypes.c_void_p(peer_slot0), P(epoch),
        stream_of(dev),
    )


def time_main_pass(res_in, grad: torch.Tensor, res_out: torch.Tensor, k: int, reps: int,
                   ws: torch.Tensor | None = None) -> float:
    """Measurement only: ms per launch of K1's HBM pass against the window the
    last select of this (m, k) published (gtk_select_main_pass): CUDA events
    on the library's stream around `reps` and `2 reps` back-to-back launches;
    the difference is exactly `reps` launches (the call's trailing workspace
    clear cancels).  res_out is overwritten with res_in + grad."""
    m = grad.numel()
    dev = grad.device
    if ws is None:
        ws = select_workspace(m, k, dev)
    st = torch.cuda.current_stream(dev)

    def timed(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        _lib.call("gtk_select_main_pass", P(res_in), P(grad), P(res_out), m, k, P(ws),
                  ctypes.c_size_t(ws.numel()), n, stream_of(dev))
        e1.record(st)
        e1.synchronize()
        return e0.elapsed_time(e1)

    timed(2)  # warm
    return (timed(2 * reps) - timed(reps)) / reps


def sparse_update_fusable(lr: float, momentum: float) -> bool:
    """K3's sparse-exact form applies (finite lr with the sign bit clear, no
    momentum): the update can ride on the select at P = 1."""
    lr32 = np.float32(lr)
    return momentum == 0.0 and bool(np.isfinite(lr32)) and not bool(np.signbit(lr32))


def select_update(res_in, grad: torch.Tensor, res_out: torch.Tensor, k: int, out: DeviceList,
                  status: torch.Tensor, window: torch.Tensor | None, w: torch.Tensor, lr: float, P_: int,
                  scaling: int, chain: bool = False) -> None:
    """K1 + K3 for P = 1 (gtk_select_update): the selection is the global
    top-k, and every selected entry also updates w exactly like
    scatter_update's sparse form.  chain=True (GTK_SELECT_CHAIN): no sampling
    kernel, res_in's pending winners (the previous chained call's) are zeroed
    on the fly and this call's stay pending in res_out until `settle`."""
    m = grad.numel()
    dev = grad.device
    ws = select_workspace(m, k, dev)
    _lib.call(
        "gtk_select_update", P(res_in), P(grad), P(res_out), m, k, P(out.idx), P(out.val), P(out.count),
        P(status), P(ws), ctypes.c_size_t(ws.numel()), _lib.SELECT_CHAIN if chain else 0, P(window), P(w),
        ctypes.c_float(lr), P_, scaling, stream_of(dev),
    )


def select_update_deferred(res_in, grad: torch.Tensor, res_out: torch.Tensor, k: int, out: DeviceList,
                           status: torch.Tensor, window: torch.Tensor, ws: torch.Tensor, prev: DeviceList | None,
                           w: torch.Tensor, lr: float, P_: int, scaling: int,
                           prev_ws: torch.Tensor | None = None) -> None:
    """K1 + K3 for P = 1 with the settle deferred (gtk_select_update_deferred):
    this call's winners stay pending in res_out, `prev` (the previous call's
    selection, pending in res_in) is corrected by this call's finish, which
    then releases the next call's HBM pass; the caller alternates two
    (window record, ws, out) sets (prev_ws = the previous call's ws).
    Bitwise the selection and update of select_update; `settle` after the
    last call."""
    m = grad.numel()
    _lib.call(
        "gtk_select_update_deferred", P(res_in), P(grad), P(res_out), m, k, P(out.idx), P(out.val),
        P(out.count), P(status), P(ws), ctypes.c_size_t(ws.numel()), P(window),
        P(prev.idx) if prev is not None else None, P(prev.count) if prev is not None else None,
        P(prev_ws) if prev is not None else None, P(w),
        ctypes.c_float(lr), P_, scaling, stream_of(grad.device),
    )


def select_push_deferred(res_in, grad: torch.Tensor, res_out: torch.Tensor, k: int, out: DeviceList,
                         status: torch.Tensor, window: torch.Tensor, ws: torch.Tensor, prev: DeviceList | None,
                         prev_ws: torch.Tensor | None, tags: torch.Tensor, peer_slot0: int | None,
                         epoch: torch.Tensor) -> None:
    """K1 for the deferred P > 1 step (gtk_select_push_deferred): winners stay
    pending in res_out, the selection goes to the exchange's first partner,
    `prev` is settled by membership of the previous global list (`tags` /
    `epoch`: the exchange plan's); the exchange then runs with res = None."""
    m = grad.numel()
    _lib.call(
        "gtk_select_push_deferred", P(res_in), P(grad), P(res_out), m, k, P(out.idx), P(out.val), P(out.count),
        P(status), P(ws), ctypes.c_size_t(ws.numel()), P(window),
        P(prev.idx) if prev is not None else None, P(prev.count) if prev is not None else None,
        P(prev_ws) if prev is not None else None, P(tags), ctypes.c_void_p(peer_slot0 or 0), P(epoch),
        stream_of(grad.device),
    )


def settle_global(res: torch.Tensor, sel: DeviceList, tags: torch.Tensor, epoch: torch.Tensor) -> None:
    """gtk_select_settle_global: the residual after the last deferred P > 1
    step (+0.0 at the local winners in the last global list)."""
    _lib.call("gtk_select_settle_global", P(res), P(sel.idx), P(sel.count), P(tags), P(epoch),
              stream_of(res.device))


def settle(res: torch.Tensor, sel: DeviceList, window: torch.Tensor) -> None:
    """gtk_select_settle: +0.0 at the last chained select's winners (the
    residual the reference keeps), and the record's pending flag cleared."""
    _lib.call("gtk_select_settle", P(res), P(sel.idx), P(sel.count), P(window), stream_of(res.device))


def top_op(a: DeviceList, b: DeviceList, k: int, out: DeviceList) -> None:
    """K2: out = ⊤(a, b, k) (a = received, b = own).  out may be b."""
    dev = b.device
    cap = max(a.cap, b.cap)
    ws = merge_workspace(cap, k, dev)
    _lib.call(
        "gtk_top_op", P(a.idx), P(a.val), P(a.count), P(b.idx), P(b.val), P(b.count), cap, k,
        P(out.idx), P(out.val), P(out.count), P(ws), ctypes.c_size_t(ws.numel()), stream_of(dev),
    )


def scatter_update(w, res, vel, glist: DeviceList, llist, m, lr, momentum, P_, scaling, skip=None) -> None:
    """K3: weights update from the global list + extra residual from the local
    list; a no-op on device if the status word `skip` carries an error bit."""
    dev = w.device
    _lib.call(
        "gtk_scatter_update", P(w), P(res), P(vel), P(glist.idx), P(glist.val), P(glist.count),
        P(llist.idx if llist is not None else None), P(llist.val if llist is not None else None),
        P(llist.count if llist is not None else None), m, ctypes.c_float(lr),
        ctypes.c_float(momentum), P_, scaling, P(skip), stream_of(dev),
    )


def dense_apply(w, vel, upd, lr, momentum, divide_by: int = 0) -> None:
    """optimizer.py:92-99 with a dense update vector (baselines)."""
    _lib.call("gtk_dense_apply", P(w), P(vel if momentum > 0 else None), P(upd), w.numel(),
              ctypes.c_float(lr), ctypes.c_float(momentum), int(divide_by), stream_of(w.device))


def densify(lst: DeviceList, m: int, out: torch.Tensor) -> None:
    _lib.call("gtk_densify", P(lst.idx), P(lst.val), P(lst.count), m, P(out), stream_of(out.device))


def topk_accumulate(idx: torch.Tensor, val: torch.Tensor, counts: torch.Tensor, P_: int,
                    stride: int, m: int, out: torch.Tensor, divide: bool = True) -> None:
    _lib.call(
        "gtk_topk_accumulate", P(idx), P(val), P(counts), P_, stride, m, P(out), 1 if divide else 0,
        stream_of(out.device),
    )


def topk_apply(idx: torch.Tensor, val: torch.Tensor, counts: torch.Tensor, P_: int, stride: int, m: int,
               acc: torch.Tensor, w: torch.Tensor, lr: float, divide: bool = True, statuses=None,
               status_stride: int = 1, local_status=None) -> None:
    """gtk_topk_apply: the topk baseline's momentum-0 update from the P
    gathered lists, at the touched entries only (acc: all-+0 f32[m] scratch,
    left all +0).  statuses: the P ranks' status words (status_stride apart);
    any error bit voids the update and flags local_status PEER_FAILED."""
    _lib.call("gtk_topk_apply", P(idx), P(val), P(counts), P_, stride, m, P(acc), P(w), ctypes.c_float(lr),
              1 if divide else 0, P(statuses), ctypes.c_int64(status_stride), P(local_status), stream_of(w.device))


def dense_sum(srcs, m: int, out: torch.Tensor, ring: bool = False) -> None:
    """Sum of the P vectors: in rank order from +0 (ring=False,
    optimizer.py:108-115) or in the ring allreduce's order (ring=True,
    collectives.py:119-122)."""
    ptrs = torch.tensor([t.data_ptr() for t in srcs], dtype=torch.int64, device=out.device)
    _lib.call("gtk_dense_ring_sum" if ring else "gtk_dense_sum", P(ptrs), len(srcs), m, P(out), stream_of(out.device))
    # keep the pointer table alive until the kernel has consumed it
    torch.cuda.current_stream(out.device).synchronize()


def divergence_terms(glist: DeviceList, naive: DeviceList, total: torch.Tensor):
    """gtk_divergence_terms: (pruned mass per global entry [device f32, gn],
    |shared indices| [device u32 as int32]) of optimizer.py:232-241."""
    dev = total.device
    pruned = torch.empty(glist.cap, dtype=torch.float32, device=dev)
    shared = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("gtk_divergence_terms", P(glist.idx), P(glist.val), P(glist.count), P(naive.idx), P(naive.count),
              P(total), total.numel(), P(pruned), P(shared), stream_of(dev))
    return pruned, shared


def read_status(status: torch.Tensor, count: torch.Tensor, host: torch.Tensor, reset: bool) -> tuple[int, int]:
    """gtk_status_read: (status word, count) in one D2H round trip into the
    pinned `host` pair, the status word zeroed behind it when `reset`."""
    _lib.call("gtk_status_read", P(status), P(count), ctypes.c_void_p(host.data_ptr()), int(reset),
              stream_of(status.device))
    h = host.numpy()
    return int(h[0]), int(h[1])


def raise_status(word: int) -> None:
    """Raise the reference exception for a device status word."""
    from .transport import TransportError

    if word & _lib.DEV_NONFINITE:
        raise FloatingPointError("non-finite values in dense input")
    if word & _lib.DEV_PENDING:
        raise RuntimeError("residual holds a chained select's pending winners: gtk_select_settle it first")
    if word & _lib.DEV_ABORTED:
        raise TransportError("cluster aborted")
    if word & _lib.DEV_TIMEOUT:
        raise TransportError("peer exchange timed out")
    if word & _lib.DEV_PEER_FAILED:
        raise TransportError("a peer rank failed during the exchange")
