/*
 * gtopk_b200.h -- C ABI of the B200-native gTop-k hot path (arXiv 1901.04359).
 *
 * The reference (pure Python + numpy, /root/reference/pkg/src/gtopk) has no
 * FFI: its plug points are the Python functions re-exported by
 * gtopk/__init__.py:3-44.  Each entry point below states the reference
 * function it replaces (file:line); INTEGRATION.md shows the ctypes binding a
 * maintainer adds on the reference side.
 *
 * Conventions
 *  - Every pointer argument named d_* or documented "device" is a device
 *    pointer on the current CUDA device; `stream` is a cudaStream_t (void* so
 *    the header does not need cuda_runtime.h; NULL = legacy default stream).
 *  - Sparse lists on the device are (int32 idx[cap], float val[cap],
 *    int32 count[2]) with strictly increasing indices.  count[0] is the
 *    entry count; count[1] is a k-th-key hint written by select/merge (the
 *    key = bits & 0x7FFFFFFF of the list's k-th largest |value|, 0 = none)
 *    that lets a later merge histogram a narrow window in one round -- it
 *    never changes results.  Counts live in device memory so chains of
 *    kernels never synchronise with the host.
 *  - Every call returns a host status code (GTK_OK or GTK_E*).  Data-dependent
 *    errors (non-finite input, exchange timeout) are reported through a device
 *    status word (uint32, GTK_DEV_* bits) that the host reads once at the
 *    Python boundary and raises as the reference's exception type.
 *  - m < 2^31 (device indices are int32; all BASELINE configs satisfy this).
 */
#ifndef GTOPK_B200_H_
#define GTOPK_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* host status codes */
#define GTK_OK 0
#define GTK_EINVAL 1      /* -> ValueError        (sparse.py:144-145, collectives.py:199-203) */
#define GTK_ENONFINITE 2  /* -> FloatingPointError (sparse.py:146-147) */
#define GTK_EPROTO 3      /* -> ProtocolError     (transport.py:47-48) */
#define GTK_ETIMEOUT 4    /* -> TransportError    (transport.py:262-268) */
#define GTK_ECUDA 5       /* CUDA runtime failure */
#define GTK_ENOMEM 6      /* workspace too small */
#define GTK_EABORTED 7    /* -> TransportError("cluster aborted") (transport.py:256-257) */

/* device status word bits */
#define GTK_DEV_NONFINITE 0x1u  /* select input held NaN/Inf */
#define GTK_DEV_FALLBACK 0x2u   /* select used the exact dense fallback (informational) */
#define GTK_DEV_TIMEOUT 0x4u    /* peer flag wait timed out */
#define GTK_DEV_ABORTED 0x8u    /* abort flag observed */
#define GTK_DEV_PEER_FAILED 0x10u /* a peer's step failed (poisoned message received) */
#define GTK_DEV_PENDING 0x20u   /* plain select of a residual with unsettled chained winners (gtk_select_settle) */
#define GTK_DEV_ERROR_MASK 0x3Du  /* every bit except the informational FALLBACK */

/* gtk_select flags */
#define GTK_SELECT_FORCE_EXACT 0x1 /* skip the sampled-threshold fast path (testing) */
#define GTK_SELECT_CHAIN 0x2       /* chained windowed select, see gtk_select_settle */
#define GTK_STEP_PREPUSHED 0x10000  /* exchange schedule flag, see gtk_gtopk_exchange */

int gtk_version(void);
const char* gtk_strerror(int code);
/* last CUDA error string seen by the library on this thread ("" if none) */
const char* gtk_last_cuda_error(void);

/* ------------------------------------------------------------------------
 * K1: fused residual-add + exact top-k select.
 * Replaces optimizer.py:219-220 (`accumulated = residual + g;
 * top_k_select(accumulated, k)`) and sparse.py:135-154 (top_k_select).
 *   res_in  : device f32[m] residual, or NULL (then acc = grad: plain top_k_select)
 *   grad    : device f32[m]
 *   res_out : device f32[m]; receives acc with +0.0 at the k selected slots
 *             (may alias res_in or grad)
 *   sel_idx/sel_val : device int32[k] / f32[k], index-ascending, values bitwise acc
 *   d_count : device int32, set to k
 *   d_status: device uint32, OR-ed with GTK_DEV_* bits (caller zeroes it)
 *   ws      : device workspace of gtk_select_workspace_bytes(m,k) bytes,
 *             zeroed once with gtk_workspace_init before first use; one
 *             workspace per stream (calls on one workspace must be ordered).
 * ------------------------------------------------------------------------ */
int gtk_select_workspace_bytes(int64_t m, int32_t k, size_t* bytes);
int gtk_workspace_init(void* ws, size_t bytes, void* stream);
int gtk_select(const float* res_in, const float* grad, float* res_out, int64_t m, int32_t k,
               int32_t* sel_idx, float* sel_val, int32_t* d_count, uint32_t* d_status, void* ws,
               size_t ws_bytes, int32_t flags, void* stream);

/* gtk_select with a per-parameter key window carried from call to call.
 *   d_window : device uint32[8] owned by the caller, one per parameter (the
 *              residual whose selections follow each other), zeroed once.
 *              Each call leaves {valid | margin level << 8, lo, shift, k,
 *              approx. k-th key, previous one, 0, 0} measured from its own candidate
 *              histogram; the next call with the same k skips the sampling
 *              pass and streams against that window (shifted by the last
 *              growth of the k-th key).  A stale window can only cost the
 *              exact dense fallback (GTK_DEV_FALLBACK), after which the window
 *              is invalid (the next call samples again) and, if it admitted
 *              too few keys, its margin level rises.
 *              Results are bit-identical to gtk_select in every case. */
int gtk_select_windowed(const float* res_in, const float* grad, float* res_out, int64_t m, int32_t k,
                        int32_t* sel_idx, float* sel_val, int32_t* d_count, uint32_t* d_status, void* ws,
                        size_t ws_bytes, int32_t flags, uint32_t* d_window, void* stream);

/* gtk_select_windowed whose selection also goes out, as it is written, to
 * the gTopKAllReduce exchange's first partner: LL records (see
 * gtk_gtopk_exchange) into that partner's inbox step-0 slot of the upcoming
 * exchange call (tag = *d_epoch + 1, slot parity = tag & 1); a non-finite
 * input sends count -1.  The following exchange call must carry
 * GTK_STEP_PREPUSHED on step 0 of its schedule.
 *   peer_slot0: the partner's IPC-mapped inbox base (its step-0 slots);
 *   d_epoch: the exchange plan's device epoch counter. */
int gtk_select_push(const float* res_in, const float* grad, float* res_out, int64_t m, int32_t k,
                    int32_t* sel_idx, float* sel_val, int32_t* d_count, uint32_t* d_status, void* ws,
                    size_t ws_bytes, int32_t flags, uint32_t* d_window, void* peer_slot0,
                    const uint64_t* d_epoch, void* stream);

/* gtk_select_windowed + K3 in the same launches, for P = 1 where the global
 * top-k IS the local selection (gtopk_allreduce over one rank is the
 * identity, collectives.py:188-219): every selected entry also applies
 * w[idx] -= FLOAT(lr) * u(val) with u as in gtk_scatter_update (scaling 0:
 * val / FLOAT(P), 1: val, 2: val * FLOAT(P)).  Sparse-exact form only: lr
 * finite with the sign bit clear (else GTK_EINVAL: run gtk_scatter_update's
 * dense kernel instead), no momentum.  On a non-finite input w is untouched. */
int gtk_select_update(const float* res_in, const float* grad, float* res_out, int64_t m, int32_t k,
                      int32_t* sel_idx, float* sel_val, int32_t* d_count, uint32_t* d_status, void* ws,
                      size_t ws_bytes, int32_t flags, uint32_t* d_window, float* w, float lr, int32_t P,
                      int32_t scaling, void* stream);

/* Chained selects (flags |= GTK_SELECT_CHAIN on gtk_select_windowed /
 * gtk_select_update; d_window required): a training loop's successive
 * selections of one residual, two launches per call instead of three.
 *  - no sampling kernel: the window comes from the record (a record that
 *    holds none -- the first call, or after a miss -- costs one exact dense
 *    pass, which records a window for the next call);
 *  - the k winners' residual slots are left PENDING in res_out (holding acc)
 *    and the exact winner predicate goes to the record {tau = the k-th key,
 *    cut = the largest kept index with key == tau}: the next chained call
 *    zeroes them on the fly while it streams res_in = this call's res_out, so
 *    its loads never wait for this call's finish;
 *  - gtk_select_settle(res_out, sel_idx, d_count, d_window) materialises the
 *    residual the reference keeps (optimizer.py:230: +0.0 at the winners) --
 *    call it before the residual is read by anything but the next chained
 *    select.  Selections, values and the settled residual are bitwise those
 *    of gtk_select_windowed.  res_out must not alias res_in or grad. */
int gtk_select_settle(float* res, const int32_t* sel_idx, const int32_t* d_count, uint32_t* d_window,
                      void* stream);

/* Deferred-settle select + fused update (P = 1 training loop, the
 * pipeline's steady state; reference optimizer.py:219-230 + :243 per step):
 * the next step's HBM pass runs while this step's finish is still ranking.
 *  - the winners' residual slots are left PENDING in res_out (holding acc);
 *    the next call passes this call's selection as (prev_sel_idx, prev_count)
 *    and res_in = this call's res_out.  Its finish first corrects the
 *    previous winners' slots (res_out[i] = +0 + grad[i], histogram and
 *    candidates to match), then releases the call after it (programmatic
 *    dependent launch), whose main pass streams while this finish ranks and
 *    writes -- selections, values, w and the settled residual are bitwise
 *    those of gtk_select_update;
 *  - no sampling kernel: the window comes from d_window, and since the next
 *    call starts before this call has measured its window, the caller
 *    alternates TWO records (call t uses record t % 2: written two calls
 *    earlier), TWO workspaces `ws` and two selection buffers;
 *  - prev_ws: the previous call's workspace (its finish left each block's
 *    output range there, so the correction needs no search), may be NULL;
 *  - prev_sel_idx = NULL: res_in holds no pending winners (first call);
 *  - gtk_select_settle(last res_out, last sel_idx, last d_count, its record)
 *    materialises the residual after the last call.
 * w / lr / P / scaling as gtk_select_update. */
int gtk_select_update_deferred(const float* res_in, const float* grad, float* res_out, int64_t m, int32_t k,
                               int32_t* sel_idx, float* sel_val, int32_t* d_count, uint32_t* d_status, void* ws,
                               size_t ws_bytes, uint32_t* d_window, const int32_t* prev_sel_idx,
                               const int32_t* prev_count, const void* prev_ws, float* w, float lr, int32_t P,
                               int32_t scaling, void* stream);

/* Deferred-settle select for the P > 1 step (the pipeline's steady state;
 * reference optimizer.py:219-230): gtk_select_update_deferred's scheme
 * without the fused update, with gtk_select_push's send of the selection to
 * the exchange's first partner -- followed by gtk_gtopk_exchange_update with
 * res = NULL (w updated, the residual untouched).  The previous winners are
 * corrected by membership of the previous global list: prev_tags = the
 * exchange plan's uint32[m] tags, d_epoch = its epoch counter (the previous
 * exchange's epoch when this call's finish runs).  peer_slot0 = NULL: no
 * push (a rank whose schedule receives first).  Settle the last step with
 * gtk_select_settle_global. */
int gtk_select_push_deferred(const float* res_in, const float* grad, float* res_out, int64_t m, int32_t k,
                             int32_t* sel_idx, float* sel_val, int32_t* d_count, uint32_t* d_status, void* ws,
                             size_t ws_bytes, uint32_t* d_window, const int32_t* prev_sel_idx,
                             const int32_t* prev_count, const void* prev_ws, const uint32_t* prev_tags,
                             void* peer_slot0, const uint64_t* d_epoch, void* stream);

/* The residual after the last deferred P > 1 step: +0.0 at the local winners
 * in the global list (tags[i] == low word of *d_epoch), +0 + acc elsewhere
 * (optimizer.py:227-230). */
int gtk_select_settle_global(float* res, const int32_t* sel_idx, const int32_t* d_count, const uint32_t* tags,
                             const uint64_t* d_epoch, void* stream);

/* Measurement only (bench.py's roofline): `reps` back-to-back launches of
 * K1's HBM pass alone (res_out = res_in + grad, candidate compaction and the
 * window histogram) against the key window the last select on this
 * workspace published, then the workspace's histogram and counters are
 * cleared (cudaMemsetAsync), so the next select starts clean.  Must follow a
 * completed select of the same (m, k) on `ws`; sel lists are not written. */
int gtk_select_main_pass(const float* res_in, const float* grad, float* res_out, int64_t m, int32_t k,
                         void* ws, size_t ws_bytes, int32_t reps, void* stream);

/* ------------------------------------------------------------------------
 * K2: the sparse top-k merge operator ⊤.
 * Replaces sparse.py:157-195 (top_op(a, b, k)); a = received, b = own
 * (collectives.py:214).  Output may alias b (in-place accumulator update).
 *   a_idx/a_val/d_na, b_idx/b_val/d_nb : device lists (counts on device)
 *   cap = max entries either input may hold (<= k in gTopKAllReduce)
 * ------------------------------------------------------------------------ */
int gtk_merge_workspace_bytes(int32_t cap, int32_t k, size_t* bytes);
int gtk_top_op(const int32_t* a_idx, const float* a_val, const int32_t* d_na, const int32_t* b_idx,
               const float* b_val, const int32_t* d_nb, int32_t cap, int32_t k, int32_t* o_idx,
               float* o_val, int32_t* d_no, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------
 * K3: scatter the global top-k into the model update and return the
 * extra residuals.  Replaces optimizer.py:227-230 (extra residual) and
 * optimizer.py:243 + :92-105 (densify, /P, momentum, w -= lr*u).
 *   scaling: 0 = "average" (v / FLOAT(P)), 1 = "sum" (v), 2 = v * FLOAT(P)
 *            (2 is gtopk_naive_step's "sum" on pre-averaged values, optimizer.py:293-296)
 *   vel may be NULL when momentum == 0.  l_idx may be NULL (no extra residual).
 *   Bitwise identical to the reference's dense update.
 * ------------------------------------------------------------------------ */
/*   d_skip: optional device status word; if any GTK_DEV_* error bit is set
 *           the kernels leave w/res/vel untouched (a failed step must not
 *           change the state, optimizer.py:219-230). */
int gtk_scatter_update(float* w, float* res, float* vel, const int32_t* g_idx, const float* g_val,
                       const int32_t* d_gn, const int32_t* l_idx, const float* l_val,
                       const int32_t* d_ln, int64_t m, float lr, float momentum, int32_t P,
                       int32_t scaling, const uint32_t* d_skip, void* stream);

/* optimizer.py:92-99 with a dense update: u = divide_by > 0 ? upd / FLOAT(divide_by) : upd;
 * if vel: vel = FLOAT(mom)*vel + u, u = vel;  w -= FLOAT(lr) * u.  (dense/topk baselines) */
int gtk_dense_apply(float* w, float* vel, const float* upd, int64_t m, float lr, float momentum,
                    int32_t divide_by, void* stream);

/* sparse.py:198-202 densify: out = zeros(m); out[idx] = val */
int gtk_densify(const int32_t* idx, const float* val, const int32_t* d_n, int64_t m, float* out,
                void* stream);

/* collectives.py:158-164 (TopKAllReduce accumulate): out = zeros(m);
 * for r in 0..P-1: out[idx_r] += val_r;  if divide: out /= FLOAT(P).
 * (divide = 0 is the unscaled rank-order sum of optimizer.py:176-183.)
 * lists are packed [P][stride] with counts d_n[P]. */
int gtk_topk_accumulate(const int32_t* idx, const float* val, const int32_t* d_n, int32_t P,
                        int64_t stride, int64_t m, float* out, int32_t divide, void* stream);

/* the topk baseline's sparse update at momentum 0 (optimizer.py:145-173 with
 * _apply_update :92-99): the P lists (same layout as gtk_topk_accumulate)
 * summed in rank order into `acc` (f32[m], all +0 on entry, all +0 again on
 * return), then w[i] -= lr * (acc[i] / P if divide else acc[i]) at each
 * touched index once -- bitwise the dense average + dense update, at P x k
 * instead of m elements.  d_status (NULL = none): the P ranks' status words,
 * status_stride int32 apart; if any carries an error bit nothing is added or
 * applied and d_local_status (this rank's word, may be NULL) gets
 * GTK_DEV_PEER_FAILED unless it already holds an error. */
int gtk_topk_apply(const int32_t* idx, const float* val, const int32_t* d_n, int32_t P, int64_t stride, int64_t m,
                   float* acc, float* w, float lr, int32_t divide, const int32_t* d_status, int64_t status_stride,
                   int32_t* d_local_status, void* stream);

/* optimizer.py:232-241 (measure_divergence) terms: pruned[i] = total[g_idx[i]] -
 * g_val[i] for the global list's entries (the reference's masked sum minus
 * densify(global) at the mask), and *d_shared = |{global indices} ∩ {naive
 * indices}| (_mask_divergence, optimizer.py:192-196).  Both lists index-sorted. */
int gtk_divergence_terms(const int32_t* g_idx, const float* g_val, const int32_t* d_gn, const int32_t* n_idx,
                         const int32_t* d_nn, const float* total, int64_t m, float* pruned, uint32_t* d_shared,
                         void* stream);

/* The step's single host round trip (optimizer.py:246-252 builds the
 * StepReport and raises from it): h_out[0] = *d_status, h_out[1] = *d_count
 * (h_out: pinned host memory), then *d_status = 0 when reset; synchronises
 * the stream. */
int gtk_status_read(const int32_t* d_status, const int32_t* d_count, int32_t* h_out, int32_t reset, void* stream);

/* rank-ordered dense sum of P device vectors (in-process dense baseline;
 * optimizer.py:108-115 summation order). srcs: device array of P pointers. */
int gtk_dense_sum(const float* const* srcs, int32_t P, int64_t m, float* out, void* stream);

/* dense sum of P device vectors in the reference's ring reduce-scatter order
 * (collectives.py:88-128: chunk c = e / ceil(m/P) summed from rank c on),
 * bitwise the ring allreduce's result (in-process dense baseline). */
int gtk_dense_ring_sum(const float* const* srcs, int32_t P, int64_t m, float* out, void* stream);

/* ------------------------------------------------------------------------
 * gTopKAllReduce exchange (collectives.py:188-219) over NVLink peer memory.
 * One persistent cooperative kernel per rank runs every round of the
 * schedule: push the current list into the partner's inbox (self-validating
 * LL records, below), poll its own inbox for the partner's list, merge (⊤).
 *
 *  schedule (host array, nsteps entries of 4 int32: {send_to, recv_from,
 *  merge, flags}); send_to/recv_from = -1 for none; merge=1 -> acc = ⊤(recv, acc),
 *  merge=0 -> acc = recv (broadcast); flags: low 16 bits informational (the
 *  step index), GTK_STEP_PREPUSHED on step 0 = its send was done by
 *  gtk_select_push.
 *  peer_inbox: host array of P device pointers (IPC-mapped) to each rank's
 *  inbox region of gtk_exchange_inbox_bytes(k, nsteps) bytes (zeroed once).
 *  Lists travel as low-latency records: per entry one 16-byte store of two
 *  64-bit words {idx | tag << 32, val bits | tag << 32}, the slot header
 *  {count | tag, hint | tag}, tag = the call's epoch; the receiver polls the
 *  words until they carry its tag (no separate flag or fence).
 * ------------------------------------------------------------------------ */
int gtk_exchange_inbox_bytes(int32_t k, int32_t nsteps, size_t* bytes);
/* cudaMalloc'd + zeroed region (IPC handles need whole allocations) */
int gtk_dev_alloc(size_t bytes, void** dptr);
int gtk_dev_free(void* dptr);
int gtk_ipc_get_handle(void* dptr, void* handle_out /* 64 bytes */);
int gtk_ipc_open_handle(const void* handle /* 64 bytes */, void** dptr_out);
int gtk_ipc_close_handle(void* dptr);
/* Abort word of a device group (replaces the reference's cluster abort,
 * transport.py:210-214, :246-248): pinned host memory mapped into the device
 * address space.  gtk_abort_word_set(host, 1) while an exchange kernel waits
 * makes it stop polling within microseconds, OR GTK_DEV_ABORTED into its
 * status word and skip K3 -- the step then raises TransportError("cluster
 * aborted") instead of waiting out its timeout.  dev_ptr is the d_abort
 * argument of the exchange calls. */
int gtk_abort_word_create(uint32_t** host_ptr, uint32_t** dev_ptr);
int gtk_abort_word_set(uint32_t* host_ptr, uint32_t value);
int gtk_abort_word_destroy(uint32_t* host_ptr);
/*  d_epoch: device uint64 call counter, zero-initialised, advanced by the
 *         kernel itself (so the launch can be captured in a CUDA graph and
 *         replayed); it stays identical on every rank.
 *  acc_*: in = this rank's local selection (<= k entries), out = the global
 *         top-k, identical on all ranks.
 *  step_counts: optional device int32[nsteps][2] receiving the entry counts
 *         sent/received per step (message accounting, 12 + 12*n bytes each).
 *  in_*: optional input list; when given the kernel first copies it into acc
 *         (so the caller's local selection stays intact for K3).
 *  ws: a merge workspace of gtk_merge_workspace_bytes(k, k) bytes.
 *  d_abort: optional abort word (gtk_abort_word_create's dev_ptr) polled while waiting. */
int gtk_gtopk_exchange(int32_t rank, int32_t P, const int32_t* schedule, int32_t nsteps,
                       void* const* peer_inbox, uint64_t* d_epoch,
                       int32_t* acc_idx, float* acc_val, int32_t* d_acc_n, int32_t k,
                       uint32_t* d_status, const uint32_t* d_abort, int64_t timeout_ns,
                       int32_t* step_counts, const int32_t* in_idx, const float* in_val,
                       const int32_t* d_in_n, void* ws, size_t ws_bytes, void* stream);

/* gtk_gtopk_exchange + K3 in the same kernel (P > 1): the writer of the final
 * global list also updates w (w[i] -= FLOAT(lr) * u(v), u as in
 * gtk_scatter_update) and tags its members (d_tags[i] = low 32 bits of the
 * device epoch); after one grid barrier every entry of the local selection
 * in_* whose tag is stale returns to res (res[i] += v) -- optimizer.py:227-230,
 * :243.  Skipped on any GTK_DEV_* error bit, like gtk_scatter_update's d_skip.
 * Sparse-exact form only (finite lr, sign bit clear; no momentum); in_* is
 * required; nsteps > 0 (one rank: gtk_select_update).
 *   d_tags: device uint32[m], zeroed once, owned per exchange plan.
 *   res = NULL: the deferred step (gtk_select_push_deferred) -- no residual
 *   restore (the local winners stay pending for the next select's settle),
 *   the next kernel in the stream may launch at once (it is the next step's
 *   HBM pass), and the merges run on 32 blocks (+24 per further merge round) when the
 *   union fits their shared memory, leaving the rest of the GPU to that pass. */
int gtk_gtopk_exchange_update(int32_t rank, int32_t P, const int32_t* schedule, int32_t nsteps,
                              void* const* peer_inbox, uint64_t* d_epoch,
                              int32_t* acc_idx, float* acc_val, int32_t* d_acc_n, int32_t k,
                              uint32_t* d_status, const uint32_t* d_abort, int64_t timeout_ns,
                              int32_t* step_counts, const int32_t* in_idx, const float* in_val,
                              const int32_t* d_in_n, void* ws, size_t ws_bytes, float* w, float* res,
                              float lr, int32_t scaling, uint32_t* d_tags, void* stream);

/* ------------------------------------------------------------------------
 * Profiling hooks (bench.py; not part of the reference interface).
 * When enabled, CUDA events are recorded on the launching stream around:
 * id 0 = K1 main HBM pass, 1 = whole select, 2 = exchange kernel,
 * 3 = standalone merge, 4 = K3 update.  Skipped while a stream is captured.
 * ------------------------------------------------------------------------ */
int gtk_prof_enable(int on);
int gtk_prof_read(int id, double* total_ms, int64_t* count); /* synchronises pending events */
int gtk_prof_reset(void);
/* pairs recorded during stream capture are event-record graph nodes; after a
 * synchronised replay this returns the sum of their current durations */
int gtk_prof_graph_read(int id, double* ms, int64_t* count);
int64_t gtk_launch_count(void); /* kernels launched by this library so far */
/* subsequent gtk_gtopk_exchange launches stamp %globaltimer into d_trace[0..]:
 * [0] start, [1] end, [2+4s+{0,1,2,3}] step s: pushed, flag seen, merged, barrier
 * (NULL disables) */
int gtk_exchange_set_trace(int64_t* d_trace);

#ifdef __cplusplus
}
#endif
#endif /* GTOPK_B200_H_ */
