"""Synchronous SGD step variants -- drop-in for the reference's
`gtopk.optimizer` (pkg/src/gtopk/optimizer.py).

The state lives in HBM: weights, a double-buffered residual (so a failed
step leaves the state untouched, optimizer.py:219-230) and the velocity.
States built from numpy arrays expose numpy arrays (copied back lazily);
states built from CUDA tensors expose the live tensors.

One gtopk_step is the hot path of this package:

    K1  select      residual + g -> exact local top-k, residual' (one HBM pass)
    ⊤   collective  gTopKAllReduce over the ranks (merge kernels / NVLink)
    K3  update      w -= lr * u at the k global entries; local entries that
                    missed the global set go back to residual'
    one 8-byte D2H  (status word, global nnz) -> exceptions + StepReport
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from . import collectives as _coll
from . import device as _dev
from .device import DeviceList
from .sparse import FLOAT, DeviceSparseVector, SparseVector, as_dense

DEFAULT_WARMUP = (0.25, 0.0725, 0.015, 0.004)
DEFAULT_TERMINAL_DENSITY = 0.001


@dataclass(frozen=True)
class DensitySchedule:
    """Warmup densities for the first epochs, then a constant terminal density
    (optimizer.py:38-43)."""

    warmup: tuple = DEFAULT_WARMUP
    terminal: float = DEFAULT_TERMINAL_DENSITY


def density_at(schedule: DensitySchedule, epoch: int) -> float:
    """optimizer.py:46-51."""
    if epoch < 0:
        raise ValueError("epoch must be >= 0")
    if epoch < len(schedule.warmup):
        return schedule.warmup[epoch]
    return schedule.terminal


def _is_cuda(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


class OptimizerState:
    """optimizer.py:54-73 with device-resident buffers."""

    def __init__(self, weights, residual, lr: float, iteration: int = 0, momentum: float = 0.0,
                 update_scaling: str = "average", schedule: DensitySchedule | None = None,
                 velocity=None):
        self._device_mode = _is_cuda(weights)
        self._dev = None
        self._w = self._res = self._res2 = self._vel = None
        self._w_np = self._res_np = self._vel_np = None
        self._host_cache = {}
        if self._device_mode:
            self._dev = weights.device
            self._w = weights.contiguous().to(torch.float32)
            self._res = residual.contiguous().to(torch.float32) if _is_cuda(residual) else \
                torch.from_numpy(as_dense(residual).copy()).to(self._dev)
            if self._res.numel() != self._w.numel():
                raise ValueError("residual dim must match weights dim")
            self._res2 = torch.empty_like(self._res)
            if velocity is not None:
                self._vel = velocity if _is_cuda(velocity) else torch.from_numpy(as_dense(velocity).copy()).to(self._dev)
        else:
            self._w_np = as_dense(weights)
            self._res_np = as_dense(residual)
            if self._res_np.size != self._w_np.size:
                raise ValueError("residual dim must match weights dim")
            self._vel_np = None if velocity is None else as_dense(velocity)
        self.lr = lr
        self.iteration = iteration
        self.momentum = momentum
        self.update_scaling = update_scaling
        self.schedule = schedule if schedule is not None else DensitySchedule()
        # a chained P = 1 select (gtk_select_update + GTK_SELECT_CHAIN) leaves its
        # winners pending in the live residual: (selection, key-window record)
        # until `_settle` zeroes them (lazily: the next chained step does it on
        # the fly, anything else that reads the residual settles first)
        self._pending = None
        if not 0.0 <= self.momentum < 1.0:
            raise ValueError("momentum must be in [0, 1)")
        if self.update_scaling not in ("average", "sum"):
            raise ValueError(f"unknown update scaling {self.update_scaling!r}")
        self._bufs = {}

    # ---- placement ---------------------------------------------------------
    @property
    def m(self) -> int:
        return self._w.numel() if self._w is not None else self._w_np.size

    def _settle(self) -> None:
        """Materialise the residual the reference keeps (+0.0 at the last
        chained step's winners, optimizer.py:230)."""
        if self._pending is not None:
            sel, win = self._pending
            self._pending = None
            _dev.settle(self._res, sel, win)
            self._host_cache.pop("r", None)

    def to_device(self, device) -> None:
        """Move the state into HBM on `device` (no-op if already there)."""
        if self._w is not None and self._w.device == device:
            return
        self._settle()
        if self._w is not None:  # move between devices
            self._w, self._res = self._w.to(device), self._res.to(device)
            self._vel = None if self._vel is None else self._vel.to(device)
        else:
            self._w = torch.from_numpy(np.array(self._w_np, dtype=FLOAT)).to(device)
            self._res = torch.from_numpy(np.array(self._res_np, dtype=FLOAT)).to(device)
            if self._vel_np is not None:
                self._vel = torch.from_numpy(np.array(self._vel_np, dtype=FLOAT)).to(device)
            self._w_np = self._res_np = self._vel_np = None
        self._res2 = torch.empty_like(self._res)
        self._dev = device
        self._host_cache.clear()

    def _host(self, name, t):
        if t is None:
            return None
        c = self._host_cache.get(name)
        if c is None:
            c = self._host_cache[name] = t.cpu().numpy()
        return c

    # ---- reference-visible fields -----------------------------------------
    @property
    def weights(self):
        if self._w is None:
            return self._w_np
        return self._w if self._device_mode else self._host("w", self._w)

    @weights.setter
    def weights(self, value) -> None:
        if self._w is not None:
            v = value if _is_cuda(value) else torch.from_numpy(as_dense(value).copy())
            self._w.copy_(v.reshape(-1))
            self._host_cache.pop("w", None)
        else:
            self._w_np = as_dense(value)

    @property
    def residual(self):
        if self._res is None:
            return self._res_np
        self._settle()
        return self._res if self._device_mode else self._host("r", self._res)

    @residual.setter
    def residual(self, value) -> None:
        self._settle()
        if self._res is not None:
            v = value if _is_cuda(value) else torch.from_numpy(as_dense(value).copy())
            self._res.copy_(v.reshape(-1))
            self._host_cache.pop("r", None)
        else:
            self._res_np = as_dense(value)

    @property
    def velocity(self):
        if self._vel is None:
            return self._vel_np
        return self._vel if self._device_mode else self._host("v", self._vel)

    @velocity.setter
    def velocity(self, value) -> None:
        if value is None:
            self._vel = self._vel_np = None
        elif self._w is not None:
            v = value if _is_cuda(value) else torch.from_numpy(as_dense(value).copy()).to(self._dev)
            self._vel = v.reshape(-1).to(torch.float32).clone()
        else:
            self._vel_np = as_dense(value)
        self._host_cache.pop("v", None)

    # ---- step plumbing -------------------------------------------------------
    def _list(self, name: str, k: int) -> DeviceList:
        key = (name, k)
        lst = self._bufs.get(key)
        if lst is None:
            lst = self._bufs[key] = DeviceList(self.m, k, self._dev)
        return lst

    def _status(self) -> torch.Tensor:
        st = self._bufs.get("status")
        if st is None:
            st = self._bufs["status"] = torch.zeros(2, dtype=torch.int32, device=self._dev)
        return st

    def _ensure_velocity(self) -> None:
        if self.momentum > 0.0 and self._vel is None:
            self._vel = torch.zeros_like(self._w)

    def _commit(self, swap_residual: bool) -> None:
        if swap_residual:
            self._res, self._res2 = self._res2, self._res
        self.iteration += 1
        self._host_cache.clear()

    def __repr__(self) -> str:
        return (f"OptimizerState(m={self.m}, lr={self.lr}, iteration={self.iteration}, "
                f"momentum={self.momentum}, update_scaling={self.update_scaling!r})")


def make_state(weights, lr: float, **kwargs) -> OptimizerState:
    """optimizer.py:76-78 -- residual starts at zeros."""
    if _is_cuda(weights):
        w = weights.detach().reshape(-1).to(torch.float32).clone()
        return OptimizerState(w, torch.zeros_like(w), lr, **kwargs)
    w = as_dense(weights).copy()
    return OptimizerState(w, np.zeros_like(w), lr, **kwargs)


@dataclass
class StepReport:
    """optimizer.py:81-89; phase times from CUDA events."""

    loss: float = 0.0
    t_compute_ms: float = 0.0
    t_compress_ms: float = 0.0
    t_communicate_ms: float = 0.0
    selected_k: int = 0
    lost_mass: float = 0.0
    divergence: float | None = None


# ---------------------------------------------------------------------------


def _grad_to_device(grad, device) -> torch.Tensor:
    if isinstance(grad, torch.Tensor):
        if grad.dim() != 1:
            raise ValueError(f"dense vector must be 1-D, got shape {tuple(grad.shape)}")
        g = grad.to(torch.float32)
        if g.device == device:
            return g
        # host tensor: async H2D when pinned (stream-ordered before K1)
        return g.to(device, non_blocking=g.is_pinned())
    g = as_dense(grad)
    return torch.from_numpy(np.ascontiguousarray(g)).to(device, non_blocking=False)


def _setup(state: OptimizerState, ep, grad):
    dev = ep.group.device
    state.to_device(dev)
    g = _grad_to_device(grad, dev)
    if g.numel() != state.m:
        raise ValueError(f"gradient dim {g.numel()} != state dim {state.m}")
    return dev, g


def _scaling_code(state: OptimizerState) -> int:
    return 0 if state.update_scaling == "average" else 1


class _Timer:
    """Phase events of a step (StepReport's t_compress / t_communicate),
    created once per state and recorded on the stream looked up once."""

    def __init__(self):
        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        self.stream = None

    def start(self, dev):
        self.stream = torch.cuda.current_stream(dev)
        return self

    def mark(self, i):
        self.ev[i].record(self.stream)

    def ms(self, i, j):
        return self.ev[i].elapsed_time(self.ev[j])


def _timer(state) -> _Timer:
    tm = state._bufs.get("timer")
    if tm is None:
        tm = state._bufs["timer"] = _Timer()
    return tm.start(state._dev)


def _select_checked(state, g, k, sel: DeviceList, status, fused_update: bool = False) -> None:
    """K1 into the spare residual; raises FloatingPointError with the state
    untouched (the live residual is never written; with fused_update the
    weights are only written when the input is finite).  fused_update (P = 1)
    runs chained: res_in's pending winners are zeroed on the fly and this
    step's stay pending (state._pending) until the residual is read."""
    m = state.m
    if not 1 <= k <= m:
        raise ValueError(f"k must be in [1, {m}], got {k}")
    win = getattr(state, "_window", None)
    if win is None or win.device != g.device:
        state._settle()
        win = state._window = _dev.new_window(g.device)  # this residual's key window (K1 hint)
    if fused_update:
        # chained (no sampling kernel, the window carried in `win`) once a
        # window is established; the first step and every step after an exact
        # dense fallback run the sampled form instead -- a window recorded by
        # the dense pass (2^20-key bins) can admit millions of keys of a
        # flat-topped residual, overflow again and never recover
        chain = not state._bufs.get("window_cold", True)
        if not chain:
            state._settle()
        _dev.select_update(state._res, g, state._res2, k, sel, status[0:1], win, state._w,
                           float(np.float32(state.lr)), 1, _scaling_code(state), chain=chain)
        state._bufs["chained"] = chain
    else:
        state._settle()
        _dev.select(state._res, g, state._res2, k, sel, status[0:1], window=win)


def _begin(state) -> torch.Tensor:
    """The step's device status word, zero (it is left zeroed by the previous
    step's _finish; anything else re-zeroes it)."""
    status = state._status()
    if not state._bufs.get("status_clean", False):
        status.zero_()
    state._bufs["status_clean"] = False
    return status


def _finish(state, count_src) -> tuple[int, int]:
    """The step's one host round trip (gtk_status_read): (status word, count),
    the status word re-zeroed for the next step."""
    host = state._bufs.get("status_host")
    if host is None:
        host = state._bufs["status_host"] = torch.zeros(2, dtype=torch.int32, pin_memory=True)
    word, cnt = _dev.read_status(state._status(), count_src, host, reset=True)
    state._bufs["status_clean"] = True
    state._bufs["last_status"] = word  # (diagnostics: e.g. the dense-fallback bit)
    return word, cnt


def gtopk_step(state: OptimizerState, ep, grad, k: int, P: int, *, loss: float = 0.0,
               t_compute_ms: float = 0.0, measure_divergence: bool = False) -> StepReport:
    """optimizer.py:199-252 on the GPU: K1 select -> gTopKAllReduce -> K3."""
    if P != ep.world_size:
        raise ValueError("P must match the cluster size")
    dev, g = _setup(state, ep, grad)
    state._ensure_velocity()
    status = _begin(state)
    sel = state._list("sel", k)
    tm = _timer(state)
    tm.mark(0)
    if P == 1 and not measure_divergence and _dev.sparse_update_fusable(state.lr, state.momentum):
        # one rank: gtopk_allreduce is the identity (collectives.py:188-219), no
        # extra residual can arise and K3 rides on K1's finish (gtk_select_update)
        _select_checked(state, g, k, sel, status, fused_update=True)
        tm.mark(1)
        tm.mark(2)
        word, gnnz = _finish(state, sel.n)
        state._bufs["window_cold"] = bool(word & (_lib.DEV_FALLBACK | _lib.DEV_ERROR_MASK))
        _dev.raise_status(word)
        state._commit(swap_residual=True)
        # a chained step's winners stay pending in the new residual (settled on
        # the fly by the next chained step); the sampled form zeroed them
        state._pending = (sel, state._window) if state._bufs["chained"] else None
        return StepReport(loss=loss, t_compute_ms=t_compute_ms, t_compress_ms=tm.ms(0, 1),
                          t_communicate_ms=tm.ms(1, 2), selected_k=gnnz)
    _select_checked(state, g, k, sel, status)
    tm.mark(1)
    fused_k3 = False
    if hasattr(ep.group, "gtopk"):
        # one process per GPU: the fused exchange kernel carries the select's
        # status (poison) to every rank, K3 skips on any error bit, and the
        # single status read below raises -- no mid-step host sync; with the
        # sparse-exact update K3 runs inside the same kernel
        fused_k3 = _dev.sparse_update_fusable(state.lr, state.momentum)
        upd = ((state._w, state._res2, float(np.float32(state.lr)), _scaling_code(state)) if fused_k3 else None)
        glist = ep.group.gtopk(ep, sel, k, status=status[0:1], update=upd)
    else:
        # in-process cluster: surface a local FloatingPointError before the
        # collective, exactly like the reference (other ranks then see the
        # cluster abort as TransportError)
        word = int(status[0].item())
        _dev.raise_status(word)
        result = _coll.gtopk_allreduce(ep, DeviceSparseVector(sel), k, P)
        glist = result.global_topk.list
    tm.mark(2)
    lost_mass, divergence = 0.0, None
    if measure_divergence:
        lost_mass, divergence = _divergence(ep, sel, glist, k, state.m)
    if not fused_k3:
        _dev.scatter_update(state._w, state._res2, state._vel, glist, sel, state.m, float(np.float32(state.lr)),
                            float(np.float32(state.momentum)), P, _scaling_code(state), skip=status[0:1])
    word, gnnz = _finish(state, glist.n)
    _dev.raise_status(word)
    state._commit(swap_residual=True)
    return StepReport(loss=loss, t_compute_ms=t_compute_ms, t_compress_ms=tm.ms(0, 1),
                      t_communicate_ms=tm.ms(1, 2), selected_k=gnnz, lost_mass=lost_mass,
                      divergence=divergence)


def topk_step(state: OptimizerState, ep, grad, k: int, P: int, *, loss: float = 0.0,
              t_compute_ms: float = 0.0) -> StepReport:
    """optimizer.py:145-173: K1 select -> TopKAllReduce (dense average) -> update."""
    if P != ep.world_size:
        raise ValueError("P must match the cluster size")
    dev, g = _setup(state, ep, grad)
    state._ensure_velocity()
    status = _begin(state)
    sel = state._list("sel", k)
    tm = _timer(state)
    tm.mark(0)
    _select_checked(state, g, k, sel, status)
    tm.mark(1)
    sparse = _dev.sparse_update_fusable(state.lr, state.momentum) and (P == 1 or hasattr(ep.group, "topk"))
    if not (sparse and (P == 1 or getattr(ep.group, "topk_status_in_band", False))):
        # surface a local FloatingPointError before the collective (the
        # in-band forms carry the status through it instead: a failed select
        # voids the update on every rank and raises at the status read below)
        word = int(status[0].item())
        _dev.raise_status(word)
    if sparse:
        # momentum 0, finite lr >= +0: the update touches only the gathered
        # lists' indices (w - lr * +0 leaves every other weight bitwise unchanged), so the
        # rank-ordered sums go to a persistent all-+0 scratch and the update
        # runs at those entries (gtk_topk_apply) -- no m-wide memset / apply
        acc = state._bufs.pop("topk_acc", None)
        if acc is None or acc.numel() != state.m or acc.device != dev:
            acc = torch.zeros(state.m, dtype=torch.float32, device=dev)
        lr = float(np.float32(state.lr))
        if P == 1:
            _dev.topk_apply(sel.idx, sel.val, sel.n, 1, sel.cap, state.m, acc, state._w, lr, divide=True,
                            statuses=status[0:1])
        else:
            ep.group.topk(ep, sel, divide=True, apply=(state._w, lr, acc, status[0:1]))
        state._bufs["topk_acc"] = acc  # (dropped above if the collective raised)
        tm.mark(2)
    else:
        averaged = _coll.topk_allreduce(ep, DeviceSparseVector(sel), P)
        tm.mark(2)
        _dense_update(state, averaged)
    word, nnz = _finish(state, sel.n)
    _dev.raise_status(word)
    state._commit(swap_residual=True)
    return StepReport(loss=loss, t_compute_ms=t_compute_ms, t_compress_ms=tm.ms(0, 1),
                      t_communicate_ms=tm.ms(1, 2), selected_k=nnz)


def _dense_update(state: OptimizerState, update: torch.Tensor, divide_by: int = 0) -> None:
    """optimizer.py:92-99 for a dense update vector (the baselines' path)."""
    _dev.dense_apply(state._w, state._vel, update, float(np.float32(state.lr)),
                     float(np.float32(state.momentum)), divide_by)


def dense_step(state: OptimizerState, ep, grad, P: int, *, loss: float = 0.0,
               t_compute_ms: float = 0.0, rank_order_sum: bool = False) -> StepReport:
    """optimizer.py:118-142: dense allreduce (sum) / P, then the update."""
    dev, g = _setup(state, ep, grad)
    state._ensure_velocity()
    t0 = time.perf_counter()
    if rank_order_sum:
        # allgather + rank-order accumulation (optimizer.py:108-115)
        total = _coll.rank_order_dense_sum(ep, g)
    elif ep.world_size == 1:
        # one rank: the ring allreduce is the identity (collectives.py:97-98
        # returns a copy); the update only reads it, so no copy is made
        total = g
    else:
        total = _coll.dense_ring_allreduce(ep, g)
    t_comm = (time.perf_counter() - t0) * 1e3
    _dense_update(state, total, divide_by=P)
    torch.cuda.current_stream(dev).synchronize()
    state._commit(swap_residual=False)
    return StepReport(loss=loss, t_compute_ms=t_compute_ms, t_communicate_ms=t_comm, selected_k=g.numel())


def _naive_global_select(total: torch.Tensor, k: int, dev) -> DeviceList:
    """optimizer.py:186-189: exact top-k of the dense sum, zeros dropped
    (K1 with no residual, then the merge kernel against an empty list, which
    drops exact zeros and keeps index order)."""
    m = total.numel()
    picked = DeviceList(m, k, dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    scratch = torch.empty_like(total)
    _dev.select(None, total, scratch, k, picked, st)
    empty = DeviceList(m, 1, dev)
    empty.count.zero_()
    out = DeviceList(m, k, dev)
    _dev.top_op(empty, picked, k, out)
    return out


def _divergence(ep, sel: DeviceList, glist: DeviceList, k: int, m: int):
    """optimizer.py:232-241: reference (allgather) selection vs tree result:
    mask divergence and the |mass| pruned mid-tree at indices that still
    landed in the global mask.  The intersection and the pruned terms come
    from one kernel (gtk_divergence_terms); the lost mass is then summed over
    the dense m-vector exactly as the reference does (np.abs(pruned).sum():
    numpy's pairwise order over all m slots, zeros included), so it matches
    bitwise -- a diagnostics-only host reduction of k D2H'd values."""
    dev = sel.device
    total = _coll.rank_order_sparse_sum(ep, DeviceSparseVector(sel))
    naive = _naive_global_select(total, k, dev)
    pruned, shared = _dev.divergence_terms(glist, naive, total)
    gn, nn, n_shared = (int(x) for x in torch.cat([glist.count[:1], naive.count[:1], shared]).cpu().tolist())
    divergence = 1.0 - n_shared / max(gn, nn, 1)
    dense = np.zeros(m, dtype=FLOAT)
    dense[glist.idx[:gn].cpu().numpy().astype(np.int64)] = pruned[:gn].cpu().numpy()
    lost_mass = float(np.abs(dense).sum())
    return lost_mass, divergence


def gtopk_naive_step(state: OptimizerState, ep, grad, k: int, P: int, *, loss: float = 0.0,
                     t_compute_ms: float = 0.0, measure_divergence: bool = False) -> StepReport:
    """optimizer.py:255-306: the reference global top-k of the true averaged
    sum (TopKAllReduce + a second exact select), used as the tree's oracle."""
    if P != ep.world_size:
        raise ValueError("P must match the cluster size")
    dev, g = _setup(state, ep, grad)
    state._ensure_velocity()
    status = _begin(state)
    sel = state._list("sel", k)
    tm = _timer(state)
    tm.mark(0)
    _select_checked(state, g, k, sel, status)
    tm.mark(1)
    word = int(status[0].item())
    _dev.raise_status(word)
    averaged = _coll.topk_allreduce(ep, DeviceSparseVector(sel), P)
    tm.mark(2)
    gsel = _naive_global_select(averaged, k, dev)
    divergence = None
    if measure_divergence:
        tree = _coll.gtopk_allreduce(ep, DeviceSparseVector(sel), k, P)
        ti, _ = tree.global_topk.list.to_host()
        ni, _ = gsel.to_host()
        sa, sb = set(ti.tolist()), set(ni.tolist())
        divergence = 1.0 - len(sa & sb) / max(len(sa), len(sb), 1)
    # averaged already carries 1/P; "sum" scaling multiplies it back (:293-296)
    scaling = 1 if state.update_scaling == "average" else 2
    _dev.scatter_update(state._w, state._res2, state._vel, gsel, sel, state.m, float(np.float32(state.lr)),
                        float(np.float32(state.momentum)), P, scaling, skip=status[0:1])
    word, nnz = _finish(state, gsel.n)
    _dev.raise_status(word)
    state._commit(swap_residual=True)
    return StepReport(loss=loss, t_compute_ms=t_compute_ms, t_compress_ms=tm.ms(0, 1),
                      t_communicate_ms=tm.ms(1, 2), selected_k=nnz, lost_mass=0.0, divergence=divergence)


STEP_FNS = {
    "dense": dense_step,
    "topk": topk_step,
    "gtopk": gtopk_step,
    "gtopk-naive": gtopk_naive_step,
}
