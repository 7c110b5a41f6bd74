"""Device-resident gTop-k S-SGD step for one rank, replayed from CUDA graphs.

`gtopk_step` (optimizer.py) is the reference-compatible API: one call per
step, one 8-byte status/count read per step.  `GTopKPipeline` is the same
hot path -- K1 select -> gTopKAllReduce -> K3 update, the identical kernels --
for a training loop that keeps gradients in HBM: the step is captured once
per residual parity into a CUDA graph and replayed with no host work; the
device status word is sticky (an error in any step makes every later K3 a
no-op) and is raised by `check()`.

The graph-capturability comes from the kernels keeping all per-call state on
the device (select workspace counters, the exchange's epoch counter).
"""

from __future__ import annotations

import os
import statistics

import numpy as np
import torch

from . import _lib
from . import device as _dev
from .device import DeviceList


class GTopKPipeline:
    kBlockSteps = 20  # steps per block graph (even: the residual parity returns)

    """gtopk_step for fixed (state, k, P, gradient buffers), graph-replayed.

    grads: list of device gradient tensors; step t reads grads[t % len(grads)].
    The residual alternates between the state's two buffers (parity t % 2),
    so len(grads) must be 1 or 2 for a graph per parity."""

    def __init__(self, ep, state, k: int, grads, use_graph: bool = True):
        from .optimizer import _scaling_code

        self.ep = ep
        self.group = ep.group
        self.P = ep.world_size
        self.dev = self.group.device
        state.to_device(self.dev)
        state._settle()  # the pipeline's own key-window record starts with nothing pending
        state._ensure_velocity()
        self.state = state
        self.m = state.m
        self.k = int(k)
        if not 1 <= self.k <= self.m:
            raise ValueError(f"k must be in [1, {self.m}], got {k}")
        if len(grads) not in (1, 2):
            raise ValueError("one or two gradient buffers")
        for g in grads:
            if not (g.is_cuda and g.device == self.dev and g.numel() == self.m and g.dtype == torch.float32):
                raise ValueError("gradients must be float32 tensors of the state's size on its device")
        self.grads = [g.contiguous() for g in grads]
        self.res = [state._res, state._res2]
        self.sel = DeviceList(self.m, self.k, self.dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.window = _dev.new_window(self.dev)  # K1 key window carried between steps
        self.lr = float(np.float32(state.lr))
        self.mom = float(np.float32(state.momentum))
        self.scaling = _scaling_code(state)
        self.plan = None
        if self.P > 1:
            if not hasattr(self.group, "enqueue_exchange"):
                raise TypeError("GTopKPipeline with P > 1 needs one process per GPU (init_dist_cluster)")
            self.plan = self.group.plan(self.k, self.m)
        self.t = 0
        self.graphs = None
        self.block_graph = None
        self.kernels_per_step = None
        self.use_graph = use_graph
        # P = 1 select mode (GTK_PIPE_MODE, A/B measurements):
        #  defer (default): gtk_select_update_deferred -- the next step's HBM
        #    pass streams while this step's finish ranks; two alternating
        #    (window record, workspace, selection) sets;
        #  chain: GTK_SELECT_CHAIN (no sampling kernel, winners zeroed on the fly);
        #  plain: gtk_select_update with the sampling kernel.
        self.mode = os.environ.get("GTK_PIPE_MODE", "defer")
        if self.mode not in ("defer", "chain", "plain"):
            raise ValueError(f"GTK_PIPE_MODE={self.mode!r}")
        self.chained = False  # steps leave their winners pending (settled by sync_state)
        self.deferred = False
        self._dsteps = 0  # deferred steps enqueued (the first has no previous selection)
        if self.mode == "defer":
            self.dsel = [DeviceList(self.m, self.k, self.dev) for _ in range(2)]
            self.dws = [_dev.select_workspace(self.m, self.k, self.dev, slot=1 + i) for i in range(2)]
            # the next main pass starts before this finish has written the next
            # window: it reads the record of the step before (one per parity)
            self.dwin = [_dev.new_window(self.dev) for _ in range(2)]

    # -- one step's launches (current stream) --------------------------------
    def _enqueue(self, parity: int) -> None:
        grad = self.grads[parity % len(self.grads)]
        res_in, res_out = self.res[parity], self.res[1 - parity]
        if self.P == 1 and _dev.sparse_update_fusable(self.lr, self.mom):
            # one rank: the global top-k is the selection; K3 rides on K1's finish
            if self.mode == "defer":
                prev = self.dsel[1 - parity] if self._dsteps > 0 else None
                try:
                    _dev.select_update_deferred(res_in, grad, res_out, self.k, self.dsel[parity], self.status,
                                                self.dwin[parity], self.dws[parity], prev, self.state._w, self.lr,
                                                1, self.scaling, prev_ws=self.dws[1 - parity])
                except ValueError:
                    if self._dsteps:
                        raise
                    # (very large k: the finish's fix list does not fit next to
                    # its slice in shared memory) -- chained selects instead
                    self.mode = "chain"
                    del self.dsel, self.dws, self.dwin
                    return self._enqueue(parity)
                self._dsteps += 1
                self.deferred = True
                return
            chain = self.mode == "chain"
            _dev.select_update(res_in, grad, res_out, self.k, self.sel, self.status, self.window,
                               self.state._w, self.lr, 1, self.scaling, chain=chain)
            self.chained = chain
            return
        if self.P > 1 and self.mode == "defer" and _dev.sparse_update_fusable(self.lr, self.mom):
            # deferred P > 1 step: the selection goes to the first partner as
            # it is written (unless this rank receives first), the exchange
            # updates w only (res = None) and lets the next step's HBM pass
            # run beside it; the next finish settles this step's winners by
            # membership of the global list
            plan = self.plan
            if plan.tags is None or plan.tags.numel() < self.m:
                plan.tags = torch.zeros(self.m, dtype=torch.int32, device=self.dev)
            prev = self.dsel[1 - parity] if self._dsteps > 0 else None
            try:
                _dev.select_push_deferred(res_in, grad, res_out, self.k, self.dsel[parity], self.status,
                                          self.dwin[parity], self.dws[parity], prev, self.dws[1 - parity],
                                          plan.tags, plan.push_slot0, plan.epoch)
            except ValueError:
                if self._dsteps:
                    raise
                self.mode = "plain"  # (very large k: see the P = 1 branch)
                del self.dsel, self.dws, self.dwin
                return self._enqueue(parity)
            self.group.enqueue_exchange(plan, self.dsel[parity], self.status,
                                        update=(self.state._w, None, self.lr, self.scaling),
                                        prepushed=plan.push_slot0 is not None)
            self._dsteps += 1
            self.deferred = True
            return
        if self.P > 1 and _dev.sparse_update_fusable(self.lr, self.mom) and self.plan.push_slot0 is not None:
            # the selection goes to the first partner as it is written
            # (gtk_select_push), K3 rides on the exchange kernel
            _dev.select_push(res_in, grad, res_out, self.k, self.sel, self.status, self.window,
                             self.plan.push_slot0, self.plan.epoch)
            self.group.enqueue_exchange(self.plan, self.sel, self.status,
                                        update=(self.state._w, res_out, self.lr, self.scaling), prepushed=True)
            return
        _dev.select(res_in, grad, res_out, self.k, self.sel, self.status, window=self.window)
        if self.P > 1 and _dev.sparse_update_fusable(self.lr, self.mom):
            # K3 rides on the exchange kernel (one launch fewer, no membership pass)
            self.group.enqueue_exchange(self.plan, self.sel, self.status,
                                        update=(self.state._w, res_out, self.lr, self.scaling))
            return
        if self.P > 1:
            self.group.enqueue_exchange(self.plan, self.sel, self.status)
            glist = self.plan.acc
        else:
            glist = self.sel
        _dev.scatter_update(self.state._w, res_out, self.state._vel, glist, self.sel, self.m, self.lr, self.mom,
                            self.P, self.scaling, skip=self.status)

    def capture(self) -> None:
        """Warm the workspaces with two eager steps, then capture one graph per
        residual parity."""
        for _ in range(2):
            self.step_eager()
        torch.cuda.synchronize(self.dev)
        stream = torch.cuda.Stream(self.dev)
        graphs = []
        n0 = _lib.load().gtk_launch_count()
        for parity in (0, 1):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                self._enqueue(parity)
            graphs.append(g)
        self.kernels_per_step = (_lib.load().gtk_launch_count() - n0) // 2
        # kBlockSteps steps (both parities, in order) in one graph: one graph
        # launch per block of steps instead of per step
        blk = torch.cuda.CUDAGraph()
        with torch.cuda.graph(blk, stream=stream):
            for j in range(self.kBlockSteps):
                self._enqueue(j % 2)
        self.graphs = graphs
        self.block_graph = blk
        torch.cuda.synchronize(self.dev)

    def profile(self, steps: int = 20) -> dict:
        """Per-stage device time (ms) of a step: CUDA events recorded by the
        library around each launch on its stream, for `steps` eager steps
        queued behind a long spin kernel -- so they execute back-to-back with
        no host gaps, exactly like graph replays."""
        lib = _lib.load()
        torch.cuda.synchronize(self.dev)
        lib.gtk_prof_reset()
        lib.gtk_prof_enable(1)
        try:
            torch.cuda._sleep(int(4e7))  # ~20 ms: covers the host enqueue of every step
            for _ in range(steps):
                self.step_eager()
        finally:
            lib.gtk_prof_enable(0)
        torch.cuda.synchronize(self.dev)
        ids = {"select_main": _lib.PROF_SELECT_MAIN, "select": _lib.PROF_SELECT,
               "exchange": _lib.PROF_EXCHANGE, "update": _lib.PROF_UPDATE}
        out = {}
        for name, pid in ids.items():
            ms, n = _lib.prof_read(pid)
            out[name] = ms / n if n else None
        lib.gtk_prof_reset()
        if os.environ.get("GTK_PROF_DEBUG"):
            print("profile (ms per launch):", out, flush=True)
        return out

    def time_main_pass(self, reps: int = 20) -> float:
        """ms per launch of K1's HBM pass on this pipeline's current residual
        and gradient, steady-state window (device.time_main_pass); the scratch
        residual buffer (the next step's output) is overwritten."""
        torch.cuda.synchronize(self.dev)
        p = self.t % 2
        # deferred steps keep their windows in their own two workspaces: the
        # one of this parity holds the window its last main pass used
        ws = self.dws[p] if self.deferred else None
        return _dev.time_main_pass(self.res[p], self.grads[p % len(self.grads)], self.res[1 - p], self.k, reps,
                                   ws=ws)

    def profile_graph(self, steps: int = 20) -> dict:
        """Per-stage device time (ms) from CUDA event nodes captured around
        each launch inside a step graph, replayed `steps` times and read back
        after each replay.  Event nodes serialise the launches they bracket,
        so each stage is timed alone (no overlap with its neighbours).  Every
        replay repeats the same step from the same residual (res[p] ->
        res[1-p]); the weights take `steps` updates (a measurement tool)."""
        lib = _lib.load()
        torch.cuda.synchronize(self.dev)
        lib.gtk_prof_reset()
        lib.gtk_prof_enable(1)
        stream = torch.cuda.Stream(self.dev)
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                self._enqueue(self.t % 2)
        finally:
            lib.gtk_prof_enable(0)
        ids = {"select_main": _lib.PROF_SELECT_MAIN, "select": _lib.PROF_SELECT,
               "exchange": _lib.PROF_EXCHANGE, "update": _lib.PROF_UPDATE}
        acc = {k_: [] for k_ in ids}
        for _ in range(steps):
            g.replay()
            torch.cuda.synchronize(self.dev)
            for name, pid in ids.items():
                ms, n = _lib.prof_graph_read(pid)
                if n:
                    acc[name].append(ms / n)
        self.t += 1  # the replays took this parity's step (res[p] -> res[1-p])
        lib.gtk_prof_reset()
        return {k_: (sum(v) / len(v) if v else None) for k_, v in acc.items()}

    def step_eager(self) -> None:
        self._enqueue(self.t % 2)
        self.t += 1

    def run(self, n: int) -> None:
        """Enqueue n steps (graph replays when captured)."""
        if self.graphs is not None:
            while n >= self.kBlockSteps and self.t % 2 == 0:
                self.block_graph.replay()
                self.t += self.kBlockSteps
                n -= self.kBlockSteps
        for _ in range(n):
            if self.graphs is not None:
                self.graphs[self.t % 2].replay()
                self.t += 1
            else:
                self.step_eager()

    def check(self) -> None:
        """Synchronise, raise the first error of any step, and hand the
        state's buffers back in their current roles."""
        word = int(self.status.item())
        _dev.raise_status(word)

    def sync_state(self) -> None:
        """Reflect the steps run so far in the OptimizerState (residual role
        and iteration count)."""
        st = self.state
        p = self.t % 2
        if self.chained and self.t > 0:
            # materialise the residual of the last step (+0.0 at its winners);
            # the next chained step would have zeroed them on the fly
            _dev.settle(self.res[p], self.sel, self.window)
        if self.deferred and self.t > 0:
            # the same for a deferred step (the next step's finish would have
            # corrected its own view of them); idempotent if the pipeline goes
            # on -- it owns the state's buffers until then
            self._settle_into(self.res[p], p)
        st._res, st._res2 = self.res[p], self.res[1 - p]
        st.iteration += self.t - getattr(self, "_synced_t", 0)
        self._synced_t = self.t
        st._host_cache.clear()

    def settled_residual(self) -> torch.Tensor:
        """A copy of the live residual with the last step's pending winners
        settled (+0.0), i.e. the reference's residual after self.t steps; the
        pipeline's own buffers are left as they are (tests)."""
        p = self.t % 2
        res = self.res[p].clone()
        if self.chained and self.t > 0:
            _dev.settle(res, self.sel, self.window.clone())
        if self.deferred and self.t > 0:
            self._settle_into(res, p)
        return res

    def _settle_into(self, res: torch.Tensor, p: int) -> None:
        """+0.0 at the last deferred step's winners (P > 1: those in its global list)."""
        if self.P == 1:
            _dev.settle(res, self.dsel[1 - p], self.dwin[1 - p].clone())
        else:
            _dev.settle_global(res, self.dsel[1 - p], self.plan.tags, self.plan.epoch)

    def global_list(self) -> DeviceList:
        if self.plan is not None:
            return self.plan.acc
        return self.dsel[(self.t - 1) % 2] if self.deferred else self.sel
