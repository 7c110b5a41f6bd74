// Common device helpers for the gTop-k B200 library (sm_100a).
//
// Key convention (SURVEY.md §8a "key equivalence"): the selection key of an
// fp32 value is its bit pattern with the sign cleared, key = bits & 0x7FFFFFFF.
// For finite inputs this is monotone in |x|, so "k largest |g|, lower index
// wins ties" (reference sparse.py:148-150) == "k largest key, lower index wins".
// Non-finite values have key >= 0x7F800000.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/gtopk_b200.h"

// GTK_CHECKED builds (tools/checked_build.sh): every shared / global index
// the kernels compute is asserted in range -- the bounds checks this GPU pool
// offers in place of compute-sanitizer (a failed check prints and traps)
#ifdef GTK_CHECKED
#include <cstdio>
#define GTK_DCHECK(cond)                                                                              \
  do {                                                                                                \
    if (!(cond)) {                                                                                    \
      printf("GTK_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__,     \
             (int)blockIdx.x, (int)threadIdx.x);                                                     \
      __trap();                                                                                       \
    }                                                                                                 \
  } while (0)
#else
#define GTK_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

namespace gtk {

constexpr uint32_t kKeyMask = 0x7FFFFFFFu;
constexpr uint32_t kInfKey = 0x7F800000u;
constexpr unsigned kFull = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t key_of(float x) { return __float_as_uint(x) & kKeyMask; }

// Merge-side key (reference sparse.py:190 lexsort on -|v|): NaN magnitudes sort
// LAST in numpy, below every nonzero finite or infinite value -> key 0.
__device__ __forceinline__ uint32_t merge_key_of(float x) {
  uint32_t k = __float_as_uint(x) & kKeyMask;
  return k > kInfKey ? 0u : k;
}

// fp32 add with x86 SSE NaN semantics (the reference runs numpy on x86): the
// result of a NaN-producing add of non-NaN operands is the "real indefinite"
// 0xFFC00000; a NaN operand propagates quieted (first operand wins).
__device__ __forceinline__ float add_x86(float a, float b) {
  const float r = __fadd_rn(a, b);
  if (r == r) return r;
  const uint32_t ua = __float_as_uint(a), ub = __float_as_uint(b);
  if ((ua & kKeyMask) > kInfKey) return __uint_as_float(ua | 0x00400000u);
  if ((ub & kKeyMask) > kInfKey) return __uint_as_float(ub | 0x00400000u);
  return __uint_as_float(0xFFC00000u);
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned warp_id() { return threadIdx.x >> 5; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t v) { return __reduce_add_sync(kFull, v); }

// ---- memory-order primitives (PTX ISA memory consistency model) ----------
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_gpu_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys_add_u64(uint64_t* p, uint64_t v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// streaming (evict-first) 128-bit global accesses for the single-use m-length
// arrays of the select pass.
__device__ __forceinline__ float4 ld_stream4(const float* p) {
  return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ void st_stream4(float* p, float4 v) {
  __stcs(reinterpret_cast<float4*>(p), v);
}

// ---- async global -> shared copies (cp.async, L1-bypassing for 16 B) -------
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// wait until at most N of this thread's committed groups are still pending
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---- bulk (TMA) global -> shared copies completing on an mbarrier ---------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");  // visible to the async (bulk-copy) proxy
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(mbar)),
      "r"(parity)
      : "memory");
}
// bytes (multiple of 16, 16-byte aligned both sides) of global memory to
// shared memory by the bulk-copy engine, evict-first in L2 (streamed once)
__device__ __forceinline__ void bulk_g2s_stream(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* mbar) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(mbar)), "l"(pol)
      : "memory");
}

// ---- programmatic dependent launch (sm_90+) ---------------------------------
// launch_dependents: let the next kernel in the stream (launched with the
// programmatic-serialization attribute) start now; wait: block until the
// previous kernel has completed and its memory is visible.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---- grid-wide barrier for cooperative launches ---------------------------
// Generation barrier; count returns to 0 after every use so the workspace
// needs a single zero-initialisation.
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// ---- low-latency (LL) peer records ------------------------------------------
// A 64-bit word {payload (low 32), tag (high 32)}, stored and loaded with
// single-copy-atomic 64-bit accesses at system scope: a receiver polls the
// word itself until the tag is the call's, so no separate flag, fence or
// release round trip is needed (NCCL's LL idea).  Pairs go out as one
// 16-byte store; each 8-byte half validates itself.
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void st_ll_pair(uint64_t* p, uint32_t a, uint32_t b, uint32_t tag) {
  const uint64_t x = ((uint64_t)tag << 32) | a, y = ((uint64_t)tag << 32) | b;
  asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(x), "l"(y) : "memory");
}
__device__ __forceinline__ void ld_ll_pair_raw(const uint64_t* p, uint64_t& x, uint64_t& y) {
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(p) : "memory");
}
// inbox slot of the exchange (one per step and call parity): 16 B LL header
// {count | tag, hint | tag} | k LL entries of 16 B {idx | tag, val bits | tag}
__host__ __device__ inline size_t ll_slot_bytes(int32_t k) { return (16 + (size_t)k * 16 + 255) & ~size_t(255); }
constexpr int32_t kStepPrepushed = 0x10000;  // schedule flag: step 0's send was done by gtk_select_push

// Polling context: give up (status |= TIMEOUT / ABORTED, payload 0) once the
// deadline passes or the host raises the abort flag.
struct LLPoll {
  uint64_t deadline;  // %globaltimer ns; 0 = none
  uint32_t* status;
  const uint32_t* abort;  // host-mapped abort word (gtk_abort_word_create), nullable
};
__device__ __forceinline__ uint32_t ld_relaxed_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
static __device__ __noinline__ bool ll_wait_failed(const LLPoll c) {
  if (c.abort && ld_relaxed_sys_u32(c.abort)) {
    atomicOr(c.status, 0x8u);  // GTK_DEV_ABORTED
    return true;
  }
  if (c.deadline && globaltimer_ns() > c.deadline) {
    atomicOr(c.status, 0x4u);  // GTK_DEV_TIMEOUT
    return true;
  }
  return false;
}
// the pair at p once both halves carry `tag`
__device__ __forceinline__ bool ld_ll_pair(const uint64_t* p, uint32_t tag, const LLPoll& c, uint32_t& a,
                                           uint32_t& b) {
  uint64_t x, y;
  ld_ll_pair_raw(p, x, y);
  uint32_t spins = 0;
  while ((uint32_t)(x >> 32) != tag || (uint32_t)(y >> 32) != tag) {
    if ((++spins & 255u) == 0 && ll_wait_failed(c)) {
      a = b = 0;
      return false;
    }
    ld_ll_pair_raw(p, x, y);
  }
  a = (uint32_t)x;
  b = (uint32_t)y;
  return true;
}

// Grid barrier over three rotating arrival counters: barrier instance i of a
// launch sends its arrivals (red.release, no return trip) to ctr[i % 3] and
// polls it (ld.acquire) until all G blocks are in; block 0, once past
// instance i, clears ctr[(i + 2) % 3] -- the counter of instance i - 1, which
// every block has stopped polling, and of instance i + 2, which nobody can
// reach before block 0's next (release) arrival -- and records i + 1 in
// `next`, where the next launch on this barrier starts (read by every block
// at its start, grid_sync_begin; block 0 writes it only after every block has
// arrived, i.e. started).  Invariant between launches: ctr[next] =
// ctr[next + 1] = 0.  Measured (tools/probe/lat_probe.cu, 100 blocks): 2.3K
// cycles per barrier vs 3.4K for a {count, generation} word whose last
// arriver bumps the generation behind its returning acq_rel arrival.
// (GTK_GRID_BAR_GEN=1 builds that protocol instead, for A/B.)
struct __align__(16) GridBarrier {
  uint32_t ctr[3];
  uint32_t next;
};

__device__ __forceinline__ uint32_t atom_add_acq_rel_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// wrapping ticket: old value; the counter returns to 0 after lim
__device__ __forceinline__ uint32_t atom_inc_acq_rel_gpu(uint32_t* p, uint32_t lim) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.inc.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(lim) : "memory");
  return old;
}

__device__ __forceinline__ uint64_t atom_add_acq_rel_gpu_u64(uint64_t* p, uint64_t v) {
  uint64_t old;
  asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release_gpu_u64(uint64_t* p, uint64_t v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_gpu_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_add_release_gpu_u32(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// A grid that is one thread-block cluster (cluster-mode merges) synchronises
// with barrier.cluster instead: release/acquire at cluster scope orders the
// blocks' global-memory writes too, and no global word is touched.
__device__ __forceinline__ uint32_t cluster_ncta() {
  uint32_t n;
  asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
  return n;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// a grid barrier that has not completed after kGridSyncTrapNs (a peer block
// that can never arrive) traps: the launch fails with an error instead of
// spinning forever
constexpr uint64_t kGridSyncTrapNs = 20ull * 1000 * 1000 * 1000;
__device__ __forceinline__ uint64_t grid_sync_now() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void grid_sync_check_stall(uint64_t& t0) {
  const uint64_t now = grid_sync_now();
  if (t0 == 0) t0 = now;
  else if (now - t0 > kGridSyncTrapNs) __trap();
}

// this block's next barrier instance (mod 3), thread 0 only
__device__ __forceinline__ uint32_t& grid_sync_inst() {
  __shared__ uint32_t s_inst;
  return s_inst;
}
// every kernel that may call grid_sync with G > 1 calls this first (after its
// griddepcontrol.wait: the previous launch on the barrier must be complete)
__device__ __forceinline__ void grid_sync_begin(const GridBarrier* b) {
  if (threadIdx.x == 0) grid_sync_inst() = __ldcg(&b->next) % 3u;
}

__device__ __forceinline__ void grid_sync(GridBarrier* b, unsigned nblocks) {
  if (nblocks == 1) {
    __syncthreads();
    return;
  }
  if (cluster_ncta() == nblocks) {
    cluster_sync_all();
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#if defined(GTK_GRID_BAR_GEN) && GTK_GRID_BAR_GEN
    // {count, generation} in ctr[0..1]: the last arriver (known from its
    // returning acq_rel arrival) resets the count and advances the generation
    uint64_t* word = reinterpret_cast<uint64_t*>(b->ctr);
    const uint64_t old = atom_add_acq_rel_gpu_u64(word, 1ull);
    const uint32_t g = (uint32_t)(old >> 32);
    if ((uint32_t)old == nblocks - 1) {
      red_add_release_gpu_u64(word, (1ull << 32) - nblocks);
    } else {
      uint64_t t0 = 0;
      for (uint32_t spins = 1; (uint32_t)(ld_acquire_gpu_u64(word) >> 32) == g; ++spins)
        if ((spins & 1023u) == 0) grid_sync_check_stall(t0);
    }
#else
    uint32_t& inst = grid_sync_inst();
    const uint32_t i = inst;
    GTK_DCHECK(i < 3u);
    uint32_t* c = &b->ctr[i];
    red_add_release_gpu_u32(c, 1u);
    uint64_t t0 = 0;
    for (uint32_t spins = 1; ld_acquire_gpu_u32(c) < nblocks; ++spins)
      if ((spins & 1023u) == 0) grid_sync_check_stall(t0);
    const uint32_t nx = i == 2u ? 0u : i + 1u;
    inst = nx;
    if (blockIdx.x == 0) {
      b->ctr[nx == 2u ? 0u : nx + 1u] = 0u;  // ctr[(i + 2) % 3]
      b->next = nx;
    }
#endif
  }
  __syncthreads();
}

// Block-wide exclusive scan of one uint32 per thread (NT threads, NT % 32 == 0).
// `scratch` needs NT/32 + 1 words. Returns the exclusive prefix; *total gets the sum.
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* scratch, uint32_t* total) {
  constexpr int NW = NT / 32;
  const unsigned lane = lane_id(), w = warp_id();
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= (unsigned)o) x += y;
  }
  if (lane == 31) scratch[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t s = lane < (unsigned)NW ? scratch[lane] : 0u;
    uint32_t t = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(kFull, t, o);
      if (lane >= (unsigned)o) t += y;
    }
    if (lane < (unsigned)NW) scratch[lane] = t - s;
    if (lane == 31) scratch[NW] = t;
  }
  __syncthreads();
  const uint32_t res = scratch[w] + x - v;
  *total = scratch[NW];
  __syncthreads();
  return res;
}

// K3's per-entry update factor u(v) (optimizer.py:243, _scaled): scaling 0 =
// "average" v / FLOAT(P), 1 = "sum" v, 2 = v * FLOAT(P) (naive gTop-k "sum")
__device__ __forceinline__ float scale_u(float v, float Pf, int scaling) {
  return scaling == 0 ? __fdiv_rn(v, Pf) : (scaling == 2 ? __fmul_rn(v, Pf) : v);
}

__host__ __device__ __forceinline__ uint32_t ceil_log2_u64(uint64_t x) {
  uint32_t s = 0;
  while ((1ull << s) < x) ++s;
  return s;
}

}  // namespace gtk
