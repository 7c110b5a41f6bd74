// gTopKAllReduce over NVLink 5 / NVSwitch peer memory (reference
// collectives.py:188-219 + binomial_bcast :168-185), fused with the ⊤ merge.
//
// One persistent cooperative kernel per rank executes the rank's whole
// schedule (butterfly for P = 2^n, reduce-tree + binomial broadcast otherwise).
// Lists travel as low-latency (LL) records: every entry is one 16-byte store
// of two self-validating 64-bit words {idx | tag, val bits | tag} into the
// partner's IPC-mapped inbox slot (s, epoch & 1), the slot header likewise
// {count | tag, hint | tag}; tag = the call's epoch.  The receiver polls the
// words it reads (header, then the entries as the merge reads them) until
// they carry the call's tag -- no flag, no fence, no release round trip.
//
//   step s:  [send]  the list to send was pushed by the previous step's merge
//                    as it wrote it (fused: the merge's output goes to acc and
//                    to the next partner at once); otherwise (first step,
//                    poisoned, broadcast forwarding after a copy) every block
//                    pushes its share of the current list;
//            [recv]  every block polls the header (count, k-th key hint;
//                    count = -1: the sender is poisoned) with a %globaltimer
//                    timeout, then
//            [merge] acc = ⊤(inbox, acc) with the same device merge as K2
//                    (received-then-own, collectives.py:214), reading the
//                    inbox records as they arrive, or acc = inbox for a
//                    broadcast step.
//
// Inbox slots are double-buffered by call parity; a rank can only overwrite a
// slot of its partner after that partner finished the previous call that used
// it (every call exchanges in both directions), so records are never
// overwritten while read, and a stale record carries another call's tag.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include <cstring>

#include "gtk_internal.h"
#include "gtk_merge.cuh"

namespace gtk {

constexpr int kMaxSteps = 64;
constexpr int kMaxRanks = 64;

struct Step {
  int32_t send_to, recv_from, merge, tag;
};

struct ExchangeArgs {
  int32_t rank, P, nsteps, k;
  uint64_t* d_epoch;  // device call counter (identical on every rank): graph-replay safe
  Step steps[kMaxSteps];
  char* inbox[kMaxRanks];     // peer-mapped inbox bases (index = rank)
  int32_t* acc_idx;
  float* acc_val;
  int32_t* d_acc_n;
  uint32_t* d_status;
  const uint32_t* d_abort;  // host-mapped abort word (nullable)
  int64_t timeout_ns;
  int32_t* step_counts;  // [nsteps][2] (sent, received) entry counts, for stats
  int64_t* trace;        // optional %globaltimer phase stamps (block 0), see gtk_exchange_set_trace
  const int32_t* in_idx; // optional input list copied into acc first (keeps the
  const float* in_val;   // caller's local selection intact for K3)
  const int32_t* d_in_n;
  uint32_t* windows;     // [kMergeWindowSlots][8] carried merge key windows, one per step
  // fused K3 (gtk_gtopk_exchange_update; upd_w null = exchange only): the
  // global list updates w, local (in_*) entries missing from it return to res
  float* upd_w;
  float* upd_res;
  float upd_lr;
  int upd_scaling;
  uint32_t* upd_tags;    // u32[m]: tags[i] = low 32 bits of the epoch when i is in this call's global list
  MergeArgs merge;       // workspace pointers; list pointers filled per step
};


__host__ __device__ inline size_t slot_bytes(int32_t k) { return ll_slot_bytes(k); }
__device__ __forceinline__ uint64_t* slot_of(char* inbox, int s, uint32_t par, int32_t k) {
  GTK_DCHECK(s >= 0 && s < kMaxSteps && par < 2u);
  return reinterpret_cast<uint64_t*>(inbox + ((size_t)s * 2 + par) * slot_bytes(k));
}

// push entries [e0, e1) of (idx, val) as LL records to body (peer memory)
__device__ __forceinline__ void push_ll(uint64_t* body, const int32_t* idx, const float* val, uint32_t e0,
                                        uint32_t e1, uint32_t tag) {
  for (uint32_t e = e0 + threadIdx.x; e < e1; e += blockDim.x)
    st_ll_pair(body + 2 * (size_t)e, (uint32_t)__ldcg(idx + e), __float_as_uint(__ldcg(val + e)), tag);
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <bool kSolo>
__global__ void __launch_bounds__(kMergeThreads) exchange_kernel(ExchangeArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  MergeSmem& S = *reinterpret_cast<MergeSmem*>(dsm);
  __shared__ uint32_t s_n, s_hint;
  __shared__ bool s_poison;
  const unsigned G = gridDim.x, blk = blockIdx.x;
  // a deferred step (no residual to restore: the select left its winners
  // pending, the next select's finish settles them) lets the next step's HBM
  // pass launch at once -- it touches neither w nor anything we read or write
  const bool deferred = a.upd_w && !a.upd_res;
  if (deferred) pdl_launch_dependents();
  pdl_wait();  // launched programmatically behind the select
  if (!deferred) pdl_launch_dependents();
  grid_sync_begin(&a.merge.ews->bar);
  // every block reads the counter before anyone advances it (block 0 does so
  // after the final grid barrier)
  const uint64_t epoch = __ldcg((const unsigned long long*)a.d_epoch) + 1;
  const uint32_t par = (uint32_t)(epoch & 1u);
  // poison: a rank whose select failed (non-finite input) still runs every
  // step so no peer hangs, but sends count = -1; receivers flag PEER_FAILED
  // and forward the poison, so every rank fails the step and K3 is skipped.
  const bool self_poison = (__ldcg(a.d_status) & GTK_DEV_NONFINITE) != 0;
  const bool tr = a.trace && blk == 0 && threadIdx.x == 0;
  if (tr) {
    a.trace[0] = (int64_t)globaltimer();
    a.trace[120] = (int64_t)clock64();  // (with [121]: the SM clock over the call)
  }

  bool k3_fused = false;  // the final merge applied the w update (deferred steps)
  // the step whose receive writes the final global list into acc (K3's tags)
  int last_recv = -1;
  for (int s = 0; s < a.nsteps; ++s)
    if (a.steps[s].recv_from >= 0) last_recv = s;

  // the current list: the caller's input until the first merge/copy writes acc
  const int32_t* cur_idx = a.in_idx ? a.in_idx : a.acc_idx;
  const float* cur_val = a.in_idx ? a.in_val : a.acc_val;
  const int32_t* cur_n = a.in_idx ? a.d_in_n : a.d_acc_n;

  const uint32_t tag = (uint32_t)epoch;
  const LLPoll poll{a.timeout_ns > 0 ? globaltimer() + (uint64_t)a.timeout_ns : 0ull, a.d_status, a.d_abort};
  bool poisoned = self_poison;  // per block, but every block decides it from the same words
  // this step's send already went out: with the previous step's output, or
  // (step 0) with the select's output (gtk_select_push)
  bool pushed = (a.steps[0].tag & kStepPrepushed) != 0;
  for (int s = 0; s < a.nsteps; ++s) {
    const Step st = a.steps[s];
    // the next step sends the list this step's merge / copy produces: fuse
    const bool fuse_next = s + 1 < a.nsteps && a.steps[s + 1].send_to >= 0;
    if (st.send_to >= 0 && !pushed) {
      uint64_t* slot = slot_of(a.inbox[st.send_to], s, par, a.k);
      uint32_t n = poisoned ? 0u : (uint32_t)__ldcg(cur_n);
      if (n > (uint32_t)a.k) n = a.k;
      const uint32_t per = (n + G - 1) / G;
      const uint32_t e0 = min(n, blk * per), e1 = min(n, e0 + per);
      push_ll(slot + 2, cur_idx, cur_val, e0, e1, tag);
      if (blk == 0 && threadIdx.x == 0) {
        // the k-th key hint travels with the list; count -1 = poisoned
        st_ll_pair(slot, poisoned ? 0xFFFFFFFFu : n, poisoned ? 0u : (uint32_t)__ldcg(cur_n + 1), tag);
        if (a.step_counts) a.step_counts[2 * s] = (int32_t)n;
      }
      if (tr) a.trace[100 + s] = (int64_t)globaltimer();
    }
    if (st.send_to >= 0 && pushed && blk == 0 && threadIdx.x == 32 && a.step_counts)  // (not the polling thread)
      a.step_counts[2 * s] = min(__ldcg(cur_n), a.k);  // the previous merge's output (final after the barrier)
    pushed = false;
    if (tr) a.trace[2 + 4 * s] = (int64_t)globaltimer();
    if (st.recv_from >= 0) {
      // everything local the merge needs is loaded before the wait
      uint32_t* wrec = (st.merge && s < kMergeWindowSlots) ? a.windows + 8 * s : nullptr;
      const MergeWindowRec wv = load_window_rec(wrec);
      uint32_t n_own = 0, hint_own = 0;
      if (st.merge) {
        // every block reads the own count before the merge's first barrier;
        // the merge writes acc (and its count) only after that barrier
        n_own = self_poison ? 0u : (uint32_t)__ldcg(cur_n);
        if (n_own > (uint32_t)a.k) n_own = a.k;
        hint_own = self_poison ? 0u : (uint32_t)__ldcg(cur_n + 1);
      }
      const uint64_t* slot = slot_of(a.inbox[a.rank], s, par, a.k);
      auto merge_args = [&]() {
        MergeArgs m = a.merge;
        m.a_ll = slot + 2;
        m.a_tag = tag;
        m.poll = poll;
        m.b_idx = cur_idx;
        m.b_val = cur_val;
        m.o_idx = a.acc_idx;
        m.o_val = a.acc_val;
        m.d_no = a.d_acc_n;
        m.trace = a.trace ? a.trace + 32 + 16 * s : nullptr;
        m.trace_arrive = a.trace ? a.trace + 104 + 2 * s : nullptr;
        return m;
      };
      // one-CTA merge: every record this thread may read (k at most) and its
      // own entries are loaded before the header is polled -- records already
      // there cost no round trip of their own
      SoloIn pre;
      if constexpr (kSolo)
        if (st.merge) solo_preload(merge_args(), (uint32_t)a.k, n_own, pre);
      if (threadIdx.x == 0) {
        uint32_t n, hint;
        const bool ok = ld_ll_pair(slot, tag, poll, n, hint);
        const bool peer_poison = ok && n == 0xFFFFFFFFu;
        if (peer_poison && blk == 0) atomicOr(a.d_status, GTK_DEV_PEER_FAILED);
        s_n = (!ok || peer_poison) ? 0u : (n > (uint32_t)a.k ? (uint32_t)a.k : n);
        s_hint = hint;
        s_poison = !ok || peer_poison;
      }
      __syncthreads();
      const uint32_t n_in = s_n, hint_in = s_hint;
      poisoned = poisoned || s_poison;
      if (tr) a.trace[3 + 4 * s] = (int64_t)globaltimer();
      if (blk == 0 && threadIdx.x == 0 && a.step_counts) a.step_counts[2 * s + 1] = (int32_t)n_in;
      // fused send of this step's output (never for a poisoned rank: the next
      // push must carry count -1)
      uint64_t* out_slot = nullptr;
      if (fuse_next && !poisoned) {
        out_slot = slot_of(a.inbox[a.steps[s + 1].send_to], s + 1, par, a.k);
        pushed = true;
      }
      if (st.merge) {
        MergeArgs m = merge_args();
        if (a.upd_w && s == last_recv) {  // the final global list: K3's membership tags
          m.tag = a.upd_tags;
          m.tag_val = tag;
          if (!a.upd_res) {
            // deferred step (no residual restore): the final merge's writer
            // also updates w -- every LL record was read before the merge's
            // first barrier, so the status word it checks is final
            m.upd_w = a.upd_w;
            m.upd_lr = a.upd_lr;
            m.upd_Pf = (float)a.P;
            m.upd_scaling = a.upd_scaling;
            m.upd_skip = a.d_status;
            k3_fused = true;
          }
        }
        if (out_slot) {
          m.ll_body = out_slot + 2;
          m.ll_head = out_slot;
          m.ll_tag = tag;
        }
        if constexpr (kSolo)
          merge_solo(m, min(n_in, (uint32_t)kMergeSub), min(n_own, (uint32_t)kMergeSub), hint_in, hint_own, S, pre);
        else
          merge_device<false>(m, n_in, n_own, hint_in, hint_own, G, S, wrec, wv);
      } else {
        const uint32_t per = (n_in + G - 1) / G;
        const uint32_t e0 = min(n_in, blk * per), e1 = min(n_in, e0 + per);
        const bool k3 = a.upd_w && s == last_recv;  // the broadcast's copy is the final global list
        for (uint32_t e = e0 + threadIdx.x; e < e1; e += kMergeThreads) {
          uint32_t i, vb;
          ld_ll_pair(slot + 2 + 2 * (size_t)e, tag, poll, i, vb);
          a.acc_idx[e] = (int32_t)i;
          a.acc_val[e] = __uint_as_float(vb);
          if (k3) a.upd_tags[i] = tag;
          if (out_slot) st_ll_pair(out_slot + 2 + 2 * (size_t)e, i, vb, tag);
        }
        if (blk == 0 && threadIdx.x == 0) {
          a.d_acc_n[0] = (int32_t)n_in;
          a.d_acc_n[1] = (int32_t)hint_in;
          if (out_slot) st_ll_pair(out_slot, n_in, hint_in, tag);
        }
      }
      cur_idx = a.acc_idx;
      cur_val = a.acc_val;
      cur_n = a.d_acc_n;
      if (tr) a.trace[4 + 4 * s] = (int64_t)globaltimer();
    }
    // the next step's merge reads acc written by every block; no barrier after
    // the last step (the next call starts on a kernel boundary)
    if (s + 1 < a.nsteps) grid_sync(&a.merge.ews->bar, G);
    if (tr) a.trace[5 + 4 * s] = (int64_t)globaltimer();
  }
  if (a.in_idx && cur_idx != a.acc_idx) {  // no step wrote acc: it is the input
    uint32_t n = (uint32_t)__ldcg(a.d_in_n);
    if (n > (uint32_t)a.k) n = a.k;
    const uint32_t per = (n + G - 1) / G;
    const uint32_t e0 = min(n, blk * per), e1 = min(n, e0 + per);
    for (uint32_t e = e0 + threadIdx.x; e < e1; e += kMergeThreads) {
      const int32_t i = __ldcg(a.in_idx + e);
      a.acc_idx[e] = i;
      a.acc_val[e] = __ldcg(a.in_val + e);
      if (a.upd_w) a.upd_tags[i] = (uint32_t)epoch;
    }
    if (blk == 0 && threadIdx.x == 0) {
      a.d_acc_n[0] = (int32_t)n;
      a.d_acc_n[1] = __ldcg(a.d_in_n + 1);
    }
  }
  if (a.upd_w && !k3_fused) {
    // K3 once the status is final (a failed step must leave the state
    // untouched on every rank): the global list updates w; local entries
    // whose membership tag (set by the final list's writer) is not this
    // call's epoch missed the global list and return to the residual
    grid_sync(&a.merge.ews->bar, G);  // every tag and the status word final
    if (!(__ldcg(a.d_status) & GTK_DEV_ERROR_MASK)) {
      const uint32_t gn = min((uint32_t)__ldcg(a.d_acc_n), (uint32_t)a.k);
      // (no residual: a deferred select keeps the local winners pending)
      const uint32_t ln = a.upd_res ? min((uint32_t)__ldcg(a.d_in_n), (uint32_t)a.k) : 0u;
      const uint32_t ep32 = (uint32_t)epoch;
      const float Pf = (float)a.P;
      // kK3Batch entries per thread per round: every list load, then every
      // dependent w / tag / residual load, then the stores -- one memory round
      // trip per phase instead of three per entry (large k)
      constexpr int kK3Batch = 4;
      const uint32_t stride = G * kMergeThreads;
      const uint32_t nmax = max(gn, ln);
      for (uint32_t base = blk * kMergeThreads + threadIdx.x; base < nmax; base += kK3Batch * stride) {
        int32_t gi[kK3Batch], li[kK3Batch];
        float gv[kK3Batch], lv[kK3Batch], wv[kK3Batch], rv[kK3Batch];
        uint32_t tg[kK3Batch];
#pragma unroll
        for (int u = 0; u < kK3Batch; ++u) {
          const uint32_t e = base + u * stride;
          if (e < gn) {
            gi[u] = __ldcg(a.acc_idx + e);
            gv[u] = __ldcg(a.acc_val + e);
          }
          if (e < ln) {
            li[u] = __ldcg(a.in_idx + e);
            lv[u] = __ldcg(a.in_val + e);
          }
        }
#pragma unroll
        for (int u = 0; u < kK3Batch; ++u) {
          const uint32_t e = base + u * stride;
          GTK_DCHECK(e >= gn || gi[u] >= 0);
          if (e < gn) wv[u] = a.upd_w[gi[u]];
          if (e < ln) {
            tg[u] = __ldcg(a.upd_tags + li[u]);
            rv[u] = a.upd_res[li[u]];
          }
        }
#pragma unroll
        for (int u = 0; u < kK3Batch; ++u) {
          const uint32_t e = base + u * stride;
          if (e < gn) a.upd_w[gi[u]] = __fsub_rn(wv[u], __fmul_rn(a.upd_lr, scale_u(gv[u], Pf, a.upd_scaling)));
          if (e < ln && tg[u] != ep32) a.upd_res[li[u]] = __fadd_rn(rv[u], lv[u]);
        }
      }
    }
  }
  if (blk == 0 && threadIdx.x == 0) {
    *a.d_epoch = epoch;
    if (tr) {
      a.trace[1] = (int64_t)globaltimer();
      a.trace[121] = (int64_t)clock64();
    }
  }
}

}  // namespace gtk

using namespace gtk;

extern "C" int gtk_exchange_set_trace(int64_t* d_trace) {
  set_trace_buffer(d_trace);
  return GTK_OK;
}

extern "C" int gtk_exchange_inbox_bytes(int32_t k, int32_t nsteps, size_t* bytes) {
  if (!bytes || k < 1 || nsteps < 0 || nsteps > kMaxSteps) return GTK_EINVAL;
  *bytes = slot_bytes(k) * 2 * (size_t)(nsteps > 0 ? nsteps : 1);
  return GTK_OK;
}

// abort word of a device group: pinned host memory mapped into the device's
// address space, so the host sets it while an exchange kernel polls it
extern "C" int gtk_abort_word_create(uint32_t** host_ptr, uint32_t** dev_ptr) {
  if (!host_ptr || !dev_ptr) return GTK_EINVAL;
  void* h = nullptr;
  GTK_CUDA(cudaHostAlloc(&h, sizeof(uint32_t), cudaHostAllocMapped | cudaHostAllocPortable));
  *(volatile uint32_t*)h = 0u;
  void* d = nullptr;
  const cudaError_t e = cudaHostGetDevicePointer(&d, h, 0);
  if (e != cudaSuccess) {
    cudaFreeHost(h);
    set_last_cuda_error(e);
    return GTK_ECUDA;
  }
  *host_ptr = (uint32_t*)h;
  *dev_ptr = (uint32_t*)d;
  return GTK_OK;
}

extern "C" int gtk_abort_word_set(uint32_t* host_ptr, uint32_t value) {
  if (!host_ptr) return GTK_EINVAL;
  __atomic_store_n(host_ptr, value, __ATOMIC_SEQ_CST);
  return GTK_OK;
}

extern "C" int gtk_abort_word_destroy(uint32_t* host_ptr) {
  if (host_ptr) GTK_CUDA(cudaFreeHost(host_ptr));
  return GTK_OK;
}

extern "C" int gtk_dev_alloc(size_t bytes, void** dptr) {
  if (!dptr || bytes == 0) return GTK_EINVAL;
  GTK_CUDA(cudaMalloc(dptr, bytes));
  GTK_CUDA(cudaMemset(*dptr, 0, bytes));
  return GTK_OK;
}

extern "C" int gtk_dev_free(void* dptr) {
  if (dptr) GTK_CUDA(cudaFree(dptr));
  return GTK_OK;
}

extern "C" int gtk_ipc_get_handle(void* dptr, void* handle_out) {
  if (!dptr || !handle_out) return GTK_EINVAL;
  cudaIpcMemHandle_t h;
  GTK_CUDA(cudaIpcGetMemHandle(&h, dptr));
  static_assert(sizeof(h) == 64, "ipc handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  return GTK_OK;
}

extern "C" int gtk_ipc_open_handle(const void* handle, void** dptr_out) {
  if (!handle || !dptr_out) return GTK_EINVAL;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  GTK_CUDA(cudaIpcOpenMemHandle(dptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return GTK_OK;
}

extern "C" int gtk_ipc_close_handle(void* dptr) {
  if (!dptr) return GTK_EINVAL;
  GTK_CUDA(cudaIpcCloseMemHandle(dptr));
  return GTK_OK;
}

static int exchange_impl(int32_t rank, int32_t P, const int32_t* schedule, int32_t nsteps, void* const* peer_inbox,
                         uint64_t* d_epoch, int32_t* acc_idx, float* acc_val,
                         int32_t* d_acc_n, int32_t k, uint32_t* d_status, const uint32_t* d_abort,
                         int64_t timeout_ns, int32_t* step_counts, const int32_t* in_idx, const float* in_val,
                         const int32_t* d_in_n, void* ws, size_t ws_bytes, float* upd_w, float* upd_res,
                         float upd_lr, int32_t upd_scaling, uint32_t* upd_tags, void* stream);

extern "C" int gtk_gtopk_exchange(int32_t rank, int32_t P, const int32_t* schedule, int32_t nsteps,
                                  void* const* peer_inbox, uint64_t* d_epoch,
                                  int32_t* acc_idx, float* acc_val, int32_t* d_acc_n, int32_t k,
                                  uint32_t* d_status, const uint32_t* d_abort, int64_t timeout_ns,
                                  int32_t* step_counts, const int32_t* in_idx, const float* in_val,
                                  const int32_t* d_in_n, void* ws, size_t ws_bytes, void* stream) {
  return exchange_impl(rank, P, schedule, nsteps, peer_inbox, d_epoch, acc_idx, acc_val, d_acc_n, k,
                       d_status, d_abort, timeout_ns, step_counts, in_idx, in_val, d_in_n, ws, ws_bytes, nullptr,
                       nullptr, 0.0f, 0, nullptr, stream);
}

extern "C" int gtk_gtopk_exchange_update(int32_t rank, int32_t P, const int32_t* schedule, int32_t nsteps,
                                         void* const* peer_inbox, uint64_t* d_epoch,
                                         int32_t* acc_idx, float* acc_val, int32_t* d_acc_n, int32_t k,
                                         uint32_t* d_status, const uint32_t* d_abort, int64_t timeout_ns,
                                         int32_t* step_counts, const int32_t* in_idx, const float* in_val,
                                         const int32_t* d_in_n, void* ws, size_t ws_bytes, float* w, float* res,
                                         float lr, int32_t scaling, uint32_t* d_tags, void* stream) {
  // res = NULL: the deferred form -- the residual keeps every local winner
  // pending (gtk_select_push_deferred), only w is updated and the membership
  // tags written for the next select's settle
  if (!w || !in_idx || !d_tags || scaling < 0 || scaling > 2 || !std::isfinite(lr) || std::signbit(lr))
    return GTK_EINVAL;
  if (nsteps == 0) return GTK_EINVAL;  // one rank: gtk_select_update
  return exchange_impl(rank, P, schedule, nsteps, peer_inbox, d_epoch, acc_idx, acc_val, d_acc_n, k,
                       d_status, d_abort, timeout_ns, step_counts, in_idx, in_val, d_in_n, ws, ws_bytes, w, res, lr,
                       scaling, d_tags, stream);
}

static int exchange_impl(int32_t rank, int32_t P, const int32_t* schedule, int32_t nsteps, void* const* peer_inbox,
                         uint64_t* d_epoch, int32_t* acc_idx, float* acc_val,
                         int32_t* d_acc_n, int32_t k, uint32_t* d_status, const uint32_t* d_abort,
                         int64_t timeout_ns, int32_t* step_counts, const int32_t* in_idx, const float* in_val,
                         const int32_t* d_in_n, void* ws, size_t ws_bytes, float* upd_w, float* upd_res,
                         float upd_lr, int32_t upd_scaling, uint32_t* upd_tags, void* stream) {
  if (P < 1 || P > kMaxRanks || rank < 0 || rank >= P || nsteps < 0 || nsteps > kMaxSteps || k < 1)
    return GTK_EINVAL;
  if (!acc_idx || !acc_val || !d_acc_n || !d_status || !ws || !d_epoch) return GTK_EINVAL;
  if (nsteps > 0 && (!schedule || !peer_inbox)) return GTK_EINVAL;
  const MergeLayout L = merge_layout(k);
  if (ws_bytes < L.total) return GTK_ENOMEM;
  if (nsteps == 0) return GTK_OK;
  ExchangeArgs a;
  std::memset(&a, 0, sizeof(a));
  a.rank = rank;
  a.P = P;
  a.nsteps = nsteps;
  a.k = k;
  a.d_epoch = d_epoch;
  for (int s = 0; s < nsteps; ++s) {
    a.steps[s] = Step{schedule[4 * s], schedule[4 * s + 1], schedule[4 * s + 2], schedule[4 * s + 3]};
    if ((a.steps[s].tag & kStepPrepushed) && (s != 0 || a.steps[s].send_to < 0)) return GTK_EINVAL;
    if (a.steps[s].send_to >= P || a.steps[s].recv_from >= P) return GTK_EINVAL;
  }
  for (int r = 0; r < P; ++r) a.inbox[r] = (char*)peer_inbox[r];
  a.acc_idx = acc_idx;
  a.acc_val = acc_val;
  a.d_acc_n = d_acc_n;
  a.d_status = d_status;
  a.d_abort = d_abort;
  a.timeout_ns = timeout_ns;
  a.step_counts = step_counts;
  a.trace = trace_buffer();
  if (in_idx && (!in_val || !d_in_n)) return GTK_EINVAL;
  a.in_idx = in_idx;
  a.in_val = in_val;
  a.d_in_n = d_in_n;
  a.windows = (uint32_t*)((char*)ws + L.windows);
  a.upd_w = upd_w;
  a.upd_res = upd_res;
  a.upd_lr = upd_lr;
  a.upd_scaling = upd_scaling;
  a.upd_tags = upd_tags;
  char* base = (char*)ws;
  a.merge = MergeArgs{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, (uint32_t)k, nullptr, nullptr,
                      nullptr, (MergeCtl*)(base + L.ctl), (EngineWS*)(base + L.engine),
                      (int32_t*)(base + L.u_idx), (float*)(base + L.u_val)};
  MergeGrid g;
  // deferred (no residual): the exchange runs beside the next step's HBM pass
  // on 32 blocks for one merge round and 24 more per further round (measured
  // with the rotating-counter grid barrier, profiles/r2_compact_grid_sweep.txt:
  // N = 2 32 blocks 75.3 us/step, 24: 77.9, 40: 76.5, 16: 83.5; N = 4 56 blocks
  // 87.7, 48: 89.3, 64: 90.6, 40: 92.6, 32: 98.7, 80: 97.9 -- the earlier
  // {count, generation} barrier's slower rounds wanted 64 at N = 4)
  int merges = 0;
  for (int s = 0; s < nsteps; ++s) merges += schedule[4 * s + 2] ? 1 : 0;
  const int compact_g = (upd_w && !upd_res) ? 32 + 24 * (std::max(1, merges) - 1) : 0;
  if (!merge_grid_for((const void*)exchange_kernel<false>, k, &g, compact_g)) return GTK_ECUDA;
  const void* fn = merge_use_solo(g, k) ? (const void*)exchange_kernel<true> : (const void*)exchange_kernel<false>;
  if (!ensure_dyn_smem(fn, merge_smem_bytes(kMergeSliceCapMax))) return GTK_ECUDA;
  a.merge.slice_cap = g.slice_cap;
  void* args[] = {&a};
  ProfScope prof(kProfExchange, (cudaStream_t)stream);
  return merge_launch(fn, g, args, merge_smem_bytes(g.slice_cap), (cudaStream_t)stream, true);
}
