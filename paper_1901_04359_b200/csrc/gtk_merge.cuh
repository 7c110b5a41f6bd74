// Device-side ⊤ merge (K2, reference sparse.py:157-195) shared by the
// standalone merge launch (gtk_merge.cu) and the fused NVLink exchange kernel
// (gtk_comm.cu).  Must run inside a cooperative launch of G blocks x
// kMergeThreads with sizeof(MergeSmem) bytes of dynamic shared memory.
//
// phase 0: the merged sequence of A (received) and B (own) -- A first on equal
//          indices -- is cut into G contiguous diagonal slices (merge path).
//          Every block finds the A/B split of each of its 2048-slot
//          sub-chunk boundaries in parallel (one warp per boundary, 33-ary
//          search), stages the inputs in shared memory and builds its slice of
//          union slots directly in shared memory: a shared index is summed once
//          (a + b with x86 NaN semantics -- fp32 add is commutative, so the
//          reference's received-then-own order, collectives.py:214, is met),
//          exact zeros (+0/-0) become empty slots (sparse.py:184-186), and a
//          2048-bin histogram of the top key bits is accumulated.
// phase 1: the exact engine keeps the k largest by (|v| desc, idx asc), NaN
//          magnitudes last (numpy lexsort, sparse.py:190), and compacts them in
//          index order -- already index-sorted (sparse.py:194), no sort.
// The output may alias B (in-place accumulator): every input read happens
// before the first grid barrier.  All list loads are ld.global.cg, so lists
// written by a peer GPU earlier in the same kernel are read correctly.
#pragma once

#include "gtk_engine.cuh"

namespace gtk {

constexpr int kMergeThreads = 512;
constexpr int kMergeSub = 2048;        // merged slots staged per sub-chunk
constexpr int kMergeSlotsPerBlock = 512;  // grid sizing target
constexpr int kMergeSliceCap = 4096;   // slice slots kept in shared memory (minimum)
constexpr int kMergeSliceCapMax = 20480;  // ... up to 160 KB of dynamic smem at large k
constexpr int kMergeMaxSplits = 65;
constexpr int kMergeMaxCluster = 16;   // CTAs of a cluster-mode merge (non-portable size above 8)
// cluster-mode sizing (measured, loopback exchange at P = 2: a CTA with more
// than ~640 union slots makes its phases longer than the cluster barriers
// save); up to 4K slots the one-CTA merge_solo beats any split (k = 1024:
// 6.9 us vs a 4-CTA cluster's 12.7; k = 2048: 11.7 vs 12.5)
constexpr int kMergeClusterSlots = 512;  // union slots per CTA in cluster mode
constexpr int kMergeSoloSlots = 4096;    // unions up to this many slots: one CTA (merge_solo), no grid barriers

struct MergeCtl {
  uint32_t n_valid;
  uint32_t pad[63];
};

struct MergeLayout {
  size_t ctl, engine, u_idx, u_val, windows, total;
};
constexpr int kMergeWindowSlots = 64;  // carried key windows (exchange steps), 8 words each

static inline MergeLayout merge_layout(int32_t cap) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  MergeLayout L{};
  size_t off = 0;
  L.ctl = off;
  off = al(off + sizeof(MergeCtl));
  L.engine = off;
  off = al(off + sizeof(EngineWS));
  L.u_idx = off;
  off = al(off + sizeof(int32_t) * 2 * (size_t)cap);
  L.u_val = off;
  off = al(off + sizeof(float) * 2 * (size_t)cap);
  L.windows = off;
  off = al(off + sizeof(uint32_t) * 8 * kMergeWindowSlots);
  L.total = off;
  return L;
}

struct MergeArgs {
  const int32_t* a_idx;
  const float* a_val;
  const int32_t* d_na;
  const int32_t* b_idx;
  const float* b_val;
  const int32_t* d_nb;
  uint32_t k;
  int32_t* o_idx;
  float* o_val;
  int32_t* d_no;
  MergeCtl* ctl;
  EngineWS* ews;
  int32_t* u_idx;  // global slot scratch for slices larger than kMergeSliceCap
  float* u_val;
  int64_t* trace;  // optional %globaltimer stamps of block 0 (phase boundaries)
  // fused K3 on the output (the exchange's last step): w update + membership tags
  float* upd_w;
  float upd_lr;
  float upd_Pf;
  int upd_scaling;
  uint32_t* tag;
  uint32_t tag_val;
  uint32_t slice_cap;  // slice slots staged in shared memory (behind MergeSmem)
  const uint32_t* upd_skip = nullptr;  // the fused update skips on an error bit here (Sink::upd_skip)
  // exchange: A arrives as LL records in the inbox (a_ll[2i] = {idx, val bits}
  // tagged a_tag; a_idx / a_val unused), polled as they are read
  const uint64_t* a_ll = nullptr;
  uint32_t a_tag = 0;
  LLPoll poll = {};
  // exchange: the output also goes to the next step's partner (see Sink)
  uint64_t* ll_body = nullptr;
  uint64_t* ll_head = nullptr;
  uint32_t ll_tag = 0;
  // diagnostics (nullable): [0] latest block arrival at the histogram
  // barrier (atomicMax of %globaltimer), [1] block 0's arrival
  int64_t* trace_arrive = nullptr;
};

// entry i of A (plain list or polled LL records)
__device__ __forceinline__ void a_entry(const MergeArgs& a, uint32_t i, int32_t& idx, float& val) {
  if (a.a_ll) {
    uint32_t x, y;
    ld_ll_pair(a.a_ll + 2 * (size_t)i, a.a_tag, a.poll, x, y);
    idx = (int32_t)x;
    val = __uint_as_float(y);
  } else {
    idx = __ldcg(a.a_idx + i);
    val = __ldcg(a.a_val + i);
  }
}
__device__ __forceinline__ int32_t a_index(const MergeArgs& a, uint32_t i) {
  if (a.a_ll) {
    int32_t idx;
    float v;
    a_entry(a, i, idx, v);
    return idx;
  }
  return __ldcg(a.a_idx + i);
}

__device__ __forceinline__ void merge_stamp(const MergeArgs& a, int i) {
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[i] = (int64_t)t;
  }
}

// dynamic shared memory: MergeSmem, then the slice (slice_cap idx, slice_cap val)
struct MergeSmem {
  EngineSmem<kMergeThreads> esm;
  int32_t sAi[kMergeSub], sBi[kMergeSub];
  float sAv[kMergeSub], sBv[kMergeSub];
  uint32_t split[kMergeMaxSplits];
  uint32_t s_valid;
};
constexpr size_t kMergeSmemFixed = (sizeof(MergeSmem) + 15) & ~size_t(15);
static inline size_t merge_smem_bytes(uint32_t slice_cap) {
  return kMergeSmemFixed + (size_t)slice_cap * (sizeof(int32_t) + sizeof(float));
}

// number of A elements among the first d merged elements (A before B on ties);
// executed by one full warp, result returned to every lane.
static __device__ __forceinline__ uint32_t merge_path_warp(const MergeArgs& a, uint32_t na, const int32_t* B,
                                                           uint32_t nb, uint32_t d) {
  uint32_t L = d > nb ? d - nb : 0u;
  uint32_t H = d < na ? d : na;
  const unsigned lane = lane_id();
  while (L < H) {
    const uint32_t n = H - L;
    if (n <= 32) {
      bool q = false;
      if (lane < n) {
        const uint32_t i = L + lane;
        q = a_index(a, i) <= __ldcg(B + (d - 1 - i));
      }
      L += __popc(__ballot_sync(kFull, q));
      break;
    }
    const uint32_t p = L + (uint32_t)(((uint64_t)n * (lane + 1)) / 33);
    const bool q = a_index(a, p) <= __ldcg(B + (d - 1 - p));
    const unsigned bal = __ballot_sync(kFull, q);
    const int t = __popc(bal);
    const uint32_t p_prev = __shfl_sync(kFull, p, t > 0 ? t - 1 : 0);
    const uint32_t p_t = __shfl_sync(kFull, p, t < 32 ? t : 31);
    if (t == 0) {
      H = p_t;
    } else {
      L = p_prev + 1;
      if (t < 32) H = p_t;
    }
  }
  return L;
}

// Window of the round-0 histogram from the inputs' k-th-key hints: a list with
// k entries has all of them >= its hint, so (cancellations aside) the union
// has >= k entries >= max(hint); 2048 linear bins over the 2 octaves above it
// (sums of correlated ranks' entries can double a value: +1 octave) isolate
// the k-th key in one round.  A miss (cancellation on shared indices) falls
// back to the full key range.
constexpr uint32_t kMergeWinShift = 13;  // 2048 << 13 = 2^24 keys = 2 octaves

// na/nb and the hints are passed by value: the caller read them before any
// output write.  rec (nullable): a key window carried from this merge's
// previous call (the same exchange step of the same parameter, same record
// format as gtk_select_windowed); used when valid, rewritten by block 0
// after the histogram barrier (every block has read it by then).
struct MergeWindowRec {  // a carried window record, loaded ahead of the merge
  uint32_t w0, lo, shift, k, tau, tau2;
};
__device__ __forceinline__ MergeWindowRec load_window_rec(const uint32_t* rec) {
  MergeWindowRec r{0u, 0u, 0u, 0u, 0u, 0u};
  if (rec) {
    r.w0 = __ldcg(rec);
    r.lo = __ldcg(rec + 1);
    r.shift = __ldcg(rec + 2);
    r.k = __ldcg(rec + 3);
    r.tau = __ldcg(rec + 4);
    r.tau2 = __ldcg(rec + 5);
  }
  return r;
}

// Union slots [s_lo, s_hi) of the merged sequence of the staged sA[0, la) and
// sB[0, lb) (index-sorted; A first on equal indices) for one thread: one
// merge-path search for the thread's first slot, then a sequential merge --
// ~log2(la + lb) + (s_hi - s_lo) dependent shared loads instead of one binary
// search per entry.  A shared index is summed once (received-then-own,
// collectives.py:214) in A's slot; B's copy leaves an empty slot.  prevA /
// (nextB, nextBv): the A entry before sA[0] and the B entry after sB[lb - 1]
// (-1: none).  emit(slot, idx, val, valid).
template <class Emit>
static __device__ __forceinline__ void union_by_path(const int32_t* sAi, const float* sAv, uint32_t la,
                                                     const int32_t* sBi, const float* sBv, uint32_t lb,
                                                     uint32_t s_lo, uint32_t s_hi, int32_t prevA, int32_t nextB,
                                                     float nextBv, Emit&& emit) {
  uint32_t lo = s_lo > lb ? s_lo - lb : 0u, hi = min(s_lo, la);
  while (lo < hi) {  // # A entries among the first s_lo merged ones
    const uint32_t mid = (lo + hi) >> 1;
    if (sAi[mid] <= sBi[s_lo - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  uint32_t i = lo, j = s_lo - lo;
  for (uint32_t sl = s_lo; sl < s_hi; ++sl) {
    if (i < la && (j >= lb || sAi[i] <= sBi[j])) {
      const int32_t x = sAi[i];
      float v = sAv[i];
      if (j < lb) {
        if (sBi[j] == x) v = add_x86(v, sBv[j]);
      } else if (nextB == x) {
        v = add_x86(v, nextBv);
      }
      emit(sl, x, v, v != 0.0f);
      ++i;
    } else {
      const int32_t x = sBi[j];
      const float v = sBv[j];
      const bool dup = i > 0 ? (sAi[i - 1] == x) : (prevA == x);
      emit(sl, x, v, !dup && v != 0.0f);
      ++j;
    }
  }
}

// ---- one-CTA merge of a small union (k <= 2K) -------------------------------
// The whole ⊤ in one block's shared memory with a dedicated pipeline -- no
// global workspace, no window record, ~10 block barriers in all:
//   load   every A record (LL words, polled only if not there yet) and B entry
//          of this thread in flight at once -- in the exchange issued before
//          the slot header is even polled (solo_preload);
//   union  each entry finds its union slot by one binary search in the other
//          list (slot = own position + rank in the other list, A first on
//          equal indices), a shared index summed once (received-then-own,
//          collectives.py:214), exact zeros dropped (sparse.py:184-186); a
//          2048-bin histogram of key bits 30..20 is built on the way;
//   select the bin holding rank k; its entries (a few dozen) are gathered and
//          ranked directly by (key desc, index asc) -- the reference's order,
//          sparse.py:188-192; a bin with more than kSoloGather entries is
//          refined by radix passes over key bits 19..9 and 8..0 instead (ties
//          on the exact k-th key: lowest index first -- the union slots ARE
//          index order, so the tie rank is a prefix count);
//   write  kept slots compacted in slot order (already index-sorted,
//          sparse.py:194): per-(row, warp) ballots, one 128-entry warp scan.
// Slots are laid out in rows of kMergeThreads (slot = row * NT + thread):
// conflict-free shared reads and coalesced output stores.
constexpr int kSoloRows = 8;
constexpr uint32_t kSoloMaxSlots = (uint32_t)kSoloRows * kMergeThreads;  // 4096
constexpr int kSoloPer = kMergeSub / kMergeThreads;                     // list entries per thread (4)
constexpr uint32_t kSoloGather = 128;  // in-bin entries ranked directly (else refined)
static_assert(kSoloMaxSlots <= (uint32_t)kMergeSliceCap, "solo union lives in the minimum slice area");
static_assert(kSoloRows * (kMergeThreads / 32) <= kMergeThreads, "solo row counts fit the engine's wcnt");
static_assert(kSoloMaxSlots <= kKeptBits && kSoloGather <= (uint32_t)kGatherCap, "solo bitmap / gather");

// this thread's share of both input lists, loads issued ahead of their use
struct SoloIn {
  uint64_t ax[kSoloPer], ay[kSoloPer];  // A: raw LL words (a_ll) or {idx, val bits}
  int32_t bi[kSoloPer];
  float bv[kSoloPer];
};
// A entries [0, na_max) (na_max >= the count still to be learnt: LL records
// past it are loaded and ignored) and B entries [0, nb)
static __device__ __forceinline__ void solo_preload(const MergeArgs& a, uint32_t na_max, uint32_t nb, SoloIn& in) {
  constexpr int NT = kMergeThreads;
  const uint32_t tid = threadIdx.x;
#pragma unroll
  for (int u = 0; u < kSoloPer; ++u) {
    const uint32_t e = u * NT + tid;
    if (e < na_max) {
      if (a.a_ll) {
        ld_ll_pair_raw(a.a_ll + 2 * (size_t)e, in.ax[u], in.ay[u]);
      } else {
        in.ax[u] = (uint32_t)__ldcg(a.a_idx + e);
        in.ay[u] = __float_as_uint(__ldcg(a.a_val + e));
      }
    }
    if (e < nb) {
      in.bi[u] = __ldcg(a.b_idx + e);
      in.bv[u] = __ldcg(a.b_val + e);
    }
  }
}

// exclusive slot-order ranks of per-row flags (bit r of `bits` = row r of this
// thread's slots); returns the total, positions through pos(r)
struct SoloRanks {
  uint32_t* cnt;  // [kSoloRows * NW] exclusive bases
  uint32_t* bal;  // [kSoloRows * NW] ballots
  __device__ __forceinline__ uint32_t pos(uint32_t r) const {
    const uint32_t i = r * (kMergeThreads / 32) + warp_id();
    return cnt[i] + __popc(bal[i] & lanemask_lt());
  }
};
static __device__ __forceinline__ uint32_t solo_rank(uint32_t bits, EngineSmem<kMergeThreads>& esm,
                                                     SoloRanks& R) {
  constexpr int NW = kMergeThreads / 32;
  uint32_t* cnt = esm.wcnt;
  uint32_t* bal = esm.wbal;
#pragma unroll
  for (int r = 0; r < kSoloRows; ++r) {
    const unsigned b = __ballot_sync(kFull, (bits >> r) & 1u);
    if (lane_id() == 0) {
      cnt[r * NW + warp_id()] = __popc(b);
      bal[r * NW + warp_id()] = b;
    }
  }
  __syncthreads();
  if (warp_id() == 0) {  // 128 counts, 4 per lane, in (row, warp) = slot order
    constexpr int PER = kSoloRows * NW / 32;
    uint32_t c[PER], s = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      c[j] = cnt[lane_id() * PER + j];
      s += c[j];
    }
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane_id() >= (unsigned)o) x += y;
    }
    uint32_t e = x - s;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      cnt[lane_id() * PER + j] = e;
      e += c[j];
    }
    if (lane_id() == 31) esm.bcast[7] = x;
  }
  __syncthreads();
  R.cnt = cnt;
  R.bal = bal;
  return esm.bcast[7];
}

// bin holding rank t (1-based from the top) of esm.hist[0, nbins), nbins <=
// 5 * NT; every thread gets (bin, count above it, count in it) and returns the
// histogram's total (< t: no such bin).  Two block barriers: each warp scans
// its 5 * 32 reversed bins, the warp totals are combined by every warp from
// shared memory.
static __device__ __forceinline__ uint32_t solo_find(uint32_t nbins, uint32_t t, EngineSmem<kMergeThreads>& esm,
                                                     uint32_t& bin, uint32_t& above, uint32_t& in_bin) {
  constexpr int PER = 5, NW = kMergeThreads / 32;
  uint32_t c[PER], sum = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {  // thread t owns reversed bins [5t, 5t + 5)
    const uint32_t rb = threadIdx.x * PER + j;
    c[j] = rb < nbins ? esm.hist[nbins - 1 - rb] : 0u;
    sum += c[j];
  }
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane_id() >= (unsigned)o) x += y;
  }
  if (lane_id() == 31) esm.scan[warp_id()] = x;
  __syncthreads();
  const uint32_t wt = lane_id() < (unsigned)NW ? esm.scan[lane_id()] : 0u;
  const uint32_t wpre = __reduce_add_sync(kFull, lane_id() < warp_id() ? wt : 0u);
  const uint32_t tot = __reduce_add_sync(kFull, wt);
  const uint32_t pre = wpre + x - sum;
  if (pre < t && pre + sum >= t) {
    uint32_t acc = pre;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      if (acc < t && acc + c[j] >= t) {
        esm.bcast[0] = nbins - 1 - (threadIdx.x * PER + j);
        esm.bcast[1] = acc;
        esm.bcast[2] = c[j];
      }
      acc += c[j];
    }
  }
  __syncthreads();
  bin = esm.bcast[0];
  above = esm.bcast[1];
  in_bin = esm.bcast[2];
  return tot;
}

// a = received (plain list or LL records), b = own; na, nb <= kMergeSub,
// na + nb <= kSoloMaxSlots <= slice_cap; `in` holds the preloaded entries;
// hint_a / hint_b: the lists' k-th keys (the first histogram's window)
static __device__ __forceinline__ void merge_solo(const MergeArgs& a, uint32_t na, uint32_t nb, uint32_t hint_a,
                                                  uint32_t hint_b, MergeSmem& S, const SoloIn& in) {
  constexpr int NT = kMergeThreads;
  EngineSmem<NT>& esm = S.esm;
  const uint32_t N = na + nb, tid = threadIdx.x;
  if (N == 0) {
    if (tid == 0) {
      a.d_no[0] = 0;
      a.d_no[1] = 0;
      if (a.ll_head) st_ll_pair(a.ll_head, 0u, 0u, a.ll_tag);
    }
    __syncthreads();
    return;
  }
  int32_t* const uI = reinterpret_cast<int32_t*>(reinterpret_cast<unsigned char*>(&S) + kMergeSmemFixed);
  float* const uV = reinterpret_cast<float*>(uI + a.slice_cap);
  // the first histogram's window: a full list has all k entries >= its hint,
  // so (cancellations aside) the union's k-th key is >= max(hint); 2048 bins
  // over the 2 octaves above it (+ OVER) leave ~1 entry per bin -- no
  // contended shared atomics, a tiny bin to rank
  uint32_t lo = 0;
  if (na >= a.k && hint_a < kInfKey) lo = max(lo, hint_a);
  if (nb >= a.k && hint_b < kInfKey) lo = max(lo, hint_b);
  uint32_t sh = lo ? kMergeWinShift : 20u;
  merge_stamp(a, 0);
  // ---- load: A records that were not there at preload time are polled now
  int32_t ai[kSoloPer];
  float av[kSoloPer];
#pragma unroll
  for (int u = 0; u < kSoloPer; ++u) {
    if (u * NT >= max(na, nb)) break;  // (block-uniform)
    const uint32_t e = u * NT + tid;
    if (e < na) {
      if (!a.a_ll || ((uint32_t)(in.ax[u] >> 32) == a.a_tag && (uint32_t)(in.ay[u] >> 32) == a.a_tag)) {
        ai[u] = (int32_t)(uint32_t)in.ax[u];
        av[u] = __uint_as_float((uint32_t)in.ay[u]);
      } else {
        a_entry(a, e, ai[u], av[u]);
      }
      S.sAi[e] = ai[u];
      S.sAv[e] = av[u];
    }
    if (e < nb) {
      S.sBi[e] = in.bi[u];
      S.sBv[e] = in.bv[u];
    }
  }
  for (uint32_t b = tid; b < (uint32_t)kHistLen; b += NT) esm.hist[b] = 0;
  for (uint32_t w = tid; w < kSoloMaxSlots / 32; w += NT) esm.kept_bits[w] = 0;
  if (tid == 0) {
    S.s_valid = 0;
    esm.ng = 0;
    esm.bcast[6] = 0xFFFFFFFFu;
  }
  __syncthreads();
  merge_stamp(a, 1);
  // ---- union slots + the window histogram
  uint32_t my_valid = 0;
  auto count = [&](int32_t i, float v) {
    ++my_valid;
    const uint32_t key = merge_key_of(v);
    if (key >= lo) {
      atomicAdd(&esm.hist[min((uint32_t)kBins, (key - lo) >> sh)], 1u);
      // a likely winner: its w line (the fused update) heads for L2 now
      if (a.upd_w) prefetch_l2(a.upd_w + i);
    }
  };
  {
    const uint32_t per = (N + NT - 1) / NT, s_lo = min(N, tid * per), s_hi = min(N, s_lo + per);
    union_by_path(S.sAi, S.sAv, na, S.sBi, S.sBv, nb, s_lo, s_hi, -1, -1, 0.0f,
                  [&](uint32_t sl, int32_t x, float v, bool valid) {
                    GTK_DCHECK(sl < N);
                    uI[sl] = valid ? x : -1;
                    uV[sl] = v;
                    if (valid) count(x, v);
                  });
  }
  my_valid = warp_sum(my_valid);
  if (lane_id() == 0 && my_valid) atomicAdd(&S.s_valid, my_valid);
  __syncthreads();
  merge_stamp(a, 2);
  const uint32_t n_valid = S.s_valid;
  const bool keep_all = n_valid <= a.k;
  // ---- the k-th key's bin [blo, bhi): kept(key) = key >= bhi, or key in the
  // bin and (mode) the whole bin / its gathered rank / its index-order tie
  // rank says so.  A bin too crowded to rank is refined 2^11-fold.
  enum { kWhole, kBitmap, kTies };
  int mode = kWhole;
  uint64_t blo = 0, bhi = 0;
  uint32_t t = a.k;
  if (!keep_all) {
    uint64_t hi = 0x80000000ull;
#pragma unroll 1
    for (int r = 0; r < 5; ++r) {
      if (r > 0) {  // rebuild over [lo, hi) (a refinement or the full range)
        for (uint32_t b = tid; b < (uint32_t)kHistLen; b += NT) esm.hist[b] = 0;
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kSoloRows; ++q) {
    if (q * NT >= N) break;  // (block-uniform: rows past the union)
          const uint32_t s = q * NT + tid;
          if (s < N && uI[s] >= 0) {
            const uint32_t key = merge_key_of(uV[s]);
            if (key >= lo && (uint64_t)key < hi) atomicAdd(&esm.hist[min((uint32_t)kBins, (key - lo) >> sh)], 1u);
          }
        }
        __syncthreads();
      }
      uint32_t bin, above, in_bin;
      if (solo_find(kHistLen, t, esm, bin, above, in_bin) < t) {
        // the window missed (cancellation on shared indices): the full range
        GTK_DCHECK(lo != 0);
        lo = 0;
        sh = 20;
        continue;
      }
      if (r == 0) merge_stamp(a, 5);
      if (a.trace && tid == 0 && r == 0) {  // diagnostics: the k-th key's bin
        a.trace[10] = bin;
        a.trace[11] = in_bin;
        a.trace[12] = lo;
      }
      blo = (uint64_t)lo + ((uint64_t)bin << sh);
      bhi = bin < (uint32_t)kBins ? min((uint64_t)(blo + (1ull << sh)), hi) : hi;
      t -= above;
      if (in_bin == t) break;  // every entry of the bin is kept
      if (in_bin <= kSoloGather) {
        // gather the bin and rank it directly: (key desc, index asc)
        mode = kBitmap;
#pragma unroll
        for (int q = 0; q < kSoloRows; ++q) {
    if (q * NT >= N) break;  // (block-uniform: rows past the union)
          const uint32_t s = q * NT + tid;
          if (s < N && uI[s] >= 0) {
            const uint32_t key = merge_key_of(uV[s]);
            if (key >= blo && key < bhi) {
              const uint32_t p = atomicAdd(&esm.ng, 1u);
              esm.keys[p] = key;
              esm.gidx[p] = uI[s];
              esm.gblk[p] = s;
            }
          }
        }
        __syncthreads();
        merge_stamp(a, 6);
        const uint32_t ng = esm.ng;
        for (uint32_t j = tid; j < ng; j += NT) {
          const uint32_t kj = esm.keys[j];
          const int32_t ij = esm.gidx[j];
          uint32_t rank = 0;
          for (uint32_t q0 = 0; q0 < ng; q0 += 8) {  // 8 independent loads in flight
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const uint32_t q = q0 + u;
              if (q < ng) {
                const uint32_t kq = esm.keys[q];
                const int32_t iq = esm.gidx[q];
                rank += (kq > kj) | ((kq == kj) & (iq < ij));
              }
            }
          }
          if (rank < t) atomicOr(&esm.kept_bits[esm.gblk[j] >> 5], 1u << (esm.gblk[j] & 31));
        }
        __syncthreads();
        merge_stamp(a, 7);
        break;
      }
      if (bhi - blo == 1) {  // one exact key: t of its in_bin entries, lowest index first
        mode = kTies;
        break;
      }
      lo = (uint32_t)blo;
      hi = bhi;
      sh = ceil_log2_u64((bhi - blo + kBins - 1) / kBins);
    }
  }
  merge_stamp(a, 3);
  // ---- kept flags in slot order
  uint32_t eq_bits = 0, kbits = 0;
#pragma unroll
  for (int q = 0; q < kSoloRows; ++q) {
    if (q * NT >= N) break;  // (block-uniform: rows past the union)
    const uint32_t s = q * NT + tid;
    if (s < N && uI[s] >= 0) {
      const uint32_t key = merge_key_of(uV[s]);
      bool kept = keep_all || key >= bhi;
      if (!kept && key >= blo) {
        if (mode == kWhole) kept = true;
        else if (mode == kBitmap) kept = (esm.kept_bits[s >> 5] >> (s & 31)) & 1u;
        else eq_bits |= 1u << q;
      }
      if (kept) kbits |= 1u << q;
    }
  }
  if (mode == kTies) {  // t entries of key == blo, lowest slots first
    SoloRanks E;
    solo_rank(eq_bits, esm, E);
#pragma unroll
    for (int q = 0; q < kSoloRows; ++q)
      if (((eq_bits >> q) & 1u) && E.pos(q) < t) kbits |= 1u << q;
    __syncthreads();  // esm.wcnt / wbal reused below
  }
  // the fused update's w loads go out before the compaction's barriers
  Sink out{a.o_idx, a.o_val, a.d_no, nullptr, true, nullptr, nullptr, 2u, 0u, 0u, 3u,
           a.upd_w, a.upd_lr, a.upd_Pf, a.upd_scaling, a.tag, a.tag_val, a.ll_body, a.ll_head, a.ll_tag};
  out.upd_skip = a.upd_skip;
  const Sink wout = sink_for_write(out);
  float wv[kSoloRows];
  if (wout.upd_w) {
#pragma unroll
    for (int q = 0; q < kSoloRows; ++q)
      if (q * NT < N && ((kbits >> q) & 1u)) wv[q] = wout.upd_w[uI[q * NT + tid]];
  }
  // the hint: the k-th key = the smallest kept key
  uint32_t kmin = 0xFFFFFFFFu;
#pragma unroll
  for (int q = 0; q < kSoloRows; ++q)
    if (q * NT < N && ((kbits >> q) & 1u)) kmin = min(kmin, merge_key_of(uV[q * NT + tid]));
  kmin = __reduce_min_sync(kFull, kmin);
  if (lane_id() == 0 && kmin != 0xFFFFFFFFu) atomicMin(&esm.bcast[6], kmin);
  SoloRanks R;
  const uint32_t n_out = solo_rank(kbits, esm, R);  // (its barriers publish bcast[6])
  GTK_DCHECK(n_out == (keep_all ? n_valid : a.k));
  // ---- write (+ the fused side effects of the exchange's final merge)
#pragma unroll
  for (int q = 0; q < kSoloRows; ++q) {
    if (q * NT >= N) break;  // (block-uniform: rows past the union)
    if ((kbits >> q) & 1u) {
      const uint32_t p = R.pos(q);
      const int32_t i = uI[q * NT + tid];
      const float v = uV[q * NT + tid];
      wout.o_idx[p] = i;
      wout.o_val[p] = v;
      if (wout.upd_w)
        wout.upd_w[i] = __fsub_rn(wv[q], __fmul_rn(wout.upd_lr, scale_u(v, wout.upd_Pf, wout.upd_scaling)));
      if (wout.tag) wout.tag[i] = wout.tag_val;
      if (wout.ll_body) st_ll_pair(wout.ll_body + 2 * (size_t)p, (uint32_t)i, __float_as_uint(v), wout.ll_tag);
    }
  }
  if (tid == 0) sink_count(out, n_out, keep_all ? 0u : esm.bcast[6]);
  merge_stamp(a, 4);
  __syncthreads();  // callers may reuse the inputs / shared memory right after
}

// kSolo: the instance for one-CTA grids of lists up to kSoloMaxSlots / 2
// entries (merge_solo only -- its own register allocation); the host picks it
// with merge_use_solo
template <bool kSolo = false>
static __device__ __forceinline__ void merge_device(const MergeArgs& a, uint32_t na, uint32_t nb, uint32_t hint_a,
                                                    uint32_t hint_b, unsigned G, MergeSmem& S,
                                                    uint32_t* rec = nullptr, MergeWindowRec rv = {}) {
  EngineSmem<kMergeThreads>& esm = S.esm;
  const unsigned blk = blockIdx.x;
  const uint32_t N = na + nb;
  if (N == 0) {
    if (blk == 0 && threadIdx.x == 0) {
      a.d_no[0] = 0;
      a.d_no[1] = 0;
      if (a.ll_head) st_ll_pair(a.ll_head, 0u, 0u, a.ll_tag);
    }
    grid_sync(&a.ews->bar, G);  // callers may reuse the inputs right after
    return;
  }
  if constexpr (kSolo) {
    // (the host guarantees na, nb <= kMergeSub: lists of <= cap <= kSoloMaxSlots / 2)
    GTK_DCHECK(G == 1 && na <= (uint32_t)kMergeSub && nb <= (uint32_t)kMergeSub && N <= a.slice_cap);
    na = min(na, (uint32_t)kMergeSub);
    nb = min(nb, (uint32_t)kMergeSub);
    SoloIn in;
    solo_preload(a, na, nb, in);
    merge_solo(a, na, nb, hint_a, hint_b, S, in);
    return;
  }
  uint32_t win_lo = 0;
  if (na >= a.k && hint_a < kInfKey) win_lo = max(win_lo, hint_a);
  if (nb >= a.k && hint_b < kInfKey) win_lo = max(win_lo, hint_b);
  uint32_t win_shift = win_lo ? kMergeWinShift : 20u;
  uint32_t rec_level = 2u, rec_tau = 0u, rec_tau2 = 0u;
  if (rec) {
    rec_level = min(4u, max(2u, rv.w0 >> 8));
    if (rv.k == a.k) {
      rec_tau = rv.tau;
      rec_tau2 = rv.tau2;
      if (rv.w0 & 1u) {  // the previous call measured the window of this step
        win_lo = rv.lo;
        win_shift = rv.shift;
      }
    }
  }
#ifndef GTK_MERGE_TRACE_FINE
  if (a.trace && blk == 0 && threadIdx.x == 0) {  // window used (diagnostics)
    a.trace[14] = win_lo;
    a.trace[15] = win_shift;
    a.trace[10] = rec ? (int64_t)rv.w0 : -1;
    a.trace[11] = rec_tau;
    a.trace[12] = rec_tau2;
  }
#endif
  for (int b = threadIdx.x; b < kHistLen; b += kMergeThreads) esm.hist[b] = 0;
  if (threadIdx.x == 0) S.s_valid = 0;
  if (blk == 0 && threadIdx.x < kRounds) a.ews->gather_n[threadIdx.x] = 0;  // read only after a barrier

  uint32_t d0, d1;
  slice_of(N, G, blk, d0, d1);
  const uint32_t L = d1 - d0;
  const bool in_smem = L <= a.slice_cap;
  int32_t* const slice_idx = reinterpret_cast<int32_t*>(reinterpret_cast<unsigned char*>(&S) + kMergeSmemFixed);
  float* const slice_val = reinterpret_cast<float*>(slice_idx + a.slice_cap);
  const uint32_t nsub = (L + kMergeSub - 1) / kMergeSub;
  merge_stamp(a, 0);
  uint32_t my_valid = 0;
  // sub-chunks in groups of kMergeMaxSplits - 1: all boundaries of a group,
  // one warp each, in parallel, then the group's union slots (any slice size)
  for (uint32_t j0 = 0; j0 < nsub; j0 += kMergeMaxSplits - 1) {
    const uint32_t jn = min(nsub - j0, (uint32_t)kMergeMaxSplits - 1);
    for (uint32_t j = warp_id(); j <= jn; j += kMergeThreads / 32) {
      const uint32_t d = min(d1, d0 + (j0 + j) * kMergeSub);
      const uint32_t i = merge_path_warp(a, na, a.b_idx, nb, d);
      GTK_DCHECK(j < (uint32_t)kMergeMaxSplits);
      if (lane_id() == 0) S.split[j] = i;
    }
    __syncthreads();
    if (j0 == 0) merge_stamp(a, 1);  // merge-path splits known
    for (uint32_t jj = 0; jj < jn; ++jj) {
      const uint32_t j = j0 + jj;
      const uint32_t sub = d0 + j * kMergeSub, sub_end = min(d1, sub + kMergeSub);
      const uint32_t ia = S.split[jj], ib = S.split[jj + 1];
      const uint32_t ja = sub - ia, jb = sub_end - ib;
      const uint32_t la = ib - ia, lb = jb - ja;
      // the neighbours across the sub-chunk edges go out first (an LL record of
      // A is only checked after the staging loads: no extra round trip)
      uint64_t pax = 0, pay = 0;
      int32_t prevA = -1;
      if (ia > 0) {
        if (a.a_ll) ld_ll_pair_raw(a.a_ll + 2 * (size_t)(ia - 1), pax, pay);
        else prevA = __ldcg(a.a_idx + ia - 1);
      }
      const int32_t nextB = jb < nb ? __ldcg(a.b_idx + jb) : -1;
      const float nextBv = jb < nb ? __ldcg(a.b_val + jb) : 0.0f;
      // stage A[ia, ib) and B[ja, jb): every load of the sub-chunk in flight at once
      GTK_DCHECK(la <= (uint32_t)kMergeSub && lb <= (uint32_t)kMergeSub);
      for (uint32_t base = 0; base < la + lb; base += 4 * kMergeThreads) {
        int32_t ri[4];
        float rv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t t = base + u * kMergeThreads + threadIdx.x;
          if (t < la) {
            a_entry(a, ia + t, ri[u], rv[u]);
          } else if (t < la + lb) {
            ri[u] = __ldcg(a.b_idx + ja + (t - la));
            rv[u] = __ldcg(a.b_val + ja + (t - la));
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t t = base + u * kMergeThreads + threadIdx.x;
          if (t < la) {
            S.sAi[t] = ri[u];
            S.sAv[t] = rv[u];
          } else if (t < la + lb) {
            S.sBi[t - la] = ri[u];
            S.sBv[t - la] = rv[u];
          }
        }
      }
      if (ia > 0 && a.a_ll)
        prevA = ((uint32_t)(pax >> 32) == a.a_tag && (uint32_t)(pay >> 32) == a.a_tag) ? (int32_t)(uint32_t)pax
                                                                                        : a_index(a, ia - 1);
      __syncthreads();
#ifdef GTK_MERGE_TRACE_FINE
      if (j == 0) merge_stamp(a, 10);  // (diagnostic build: first sub-chunk staged)
#endif
      {
        const uint32_t L = la + lb, per = (L + kMergeThreads - 1) / kMergeThreads;
        const uint32_t s_lo = min(L, threadIdx.x * per), s_hi = min(L, s_lo + per);
        union_by_path(S.sAi, S.sAv, la, S.sBi, S.sBv, lb, s_lo, s_hi, prevA, nextB, nextBv,
                      [&](uint32_t sl, int32_t x, float v, bool valid) {
                        const uint32_t slot = sub + sl;
                        GTK_DCHECK(slot >= d0 && slot < d1 && (!in_smem || slot - d0 < a.slice_cap));
                        if (in_smem) {
                          slice_idx[slot - d0] = valid ? x : -1;
                          slice_val[slot - d0] = v;
                        } else {
                          a.u_idx[slot] = valid ? x : -1;
                          a.u_val[slot] = v;
                        }
                        if (valid) {
                          ++my_valid;
                          const uint32_t key = merge_key_of(v);
                          if (key >= win_lo)
                            atomicAdd(&esm.hist[min((uint32_t)kBins, (key - win_lo) >> win_shift)], 1u);
                        }
                      });
      }
      __syncthreads();
#ifdef GTK_MERGE_TRACE_FINE
      if (j == 0) merge_stamp(a, 11);  // (first sub-chunk's union done)
      if (j + 1 == nsub) merge_stamp(a, 12);
#endif
    }
  }
  my_valid = warp_sum(my_valid);
  if (lane_id() == 0 && my_valid) atomicAdd(&S.s_valid, my_valid);
  __syncthreads();
  merge_stamp(a, 2);  // union slots + histogram built
  const bool solo = G == 1;
  const SliceSrc src{slice_idx, slice_val, a.u_idx, a.u_val, d0, in_smem, true};
  uint32_t n_valid;
  if (solo) {
    n_valid = S.s_valid;  // the histogram stays in shared memory
  } else {
    for (int b = threadIdx.x; b < kHistLen; b += kMergeThreads) {
      const uint32_t c = esm.hist[b];
      if (c) atomicAdd(&a.ews->hist[0][b], c);
    }
    if (threadIdx.x == 0 && S.s_valid) atomicAdd(&a.ctl->n_valid, S.s_valid);
    if (a.trace_arrive && threadIdx.x == 0) {
      const uint64_t tnow = globaltimer_ns();
      atomicMax((unsigned long long*)a.trace_arrive, (unsigned long long)tnow);
      if (blk == 0) a.trace_arrive[1] = (int64_t)tnow;
    }
    grid_sync(&a.ews->bar, G);
    // the global histogram -> shared memory by async copies, landing while
    // the valid count is read: the engine's bin search then needs no second
    // L2 round trip
    for (int b = threadIdx.x; b < kHistLen; b += kMergeThreads) cp_async4(&esm.hist[b], a.ews->hist[0] + b);
    cp_async_commit();
    n_valid = __ldcg(&a.ctl->n_valid);
    cp_async_wait_all();
    __syncthreads();
  }
  merge_stamp(a, 3);  // after the histogram barrier
  const bool keep_all = n_valid <= a.k;
  Sink out{a.o_idx, a.o_val, a.d_no, nullptr, true, a.trace ? a.trace + 5 : nullptr,
           keep_all ? nullptr : rec, rec_level, rec_tau, rec_tau2, 3u,
           a.upd_w, a.upd_lr, a.upd_Pf, a.upd_scaling, a.tag, a.tag_val,
           a.ll_body, a.ll_head, a.ll_tag};
  out.upd_skip = a.upd_skip;
  // one engine call site for both attempts (the window, then -- if it missed
  // through cancellation or a shifted carried window -- the full key range):
  // a single inlined copy of the engine keeps the kernel's code compact (its
  // phases run once per call; instruction fetch is a large share of its stalls)
  bool ok = false;
#pragma unroll 1
  for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
    const bool first = attempt == 0;
    if (!first) {
      if (rec && blk == 0 && threadIdx.x == 0) {
        rec[0] = min(4u, rec_level + 1) << 8;  // invalid, wider margin next time
        rec[4] = rec[5] = 0u;
      }
      if (!solo) {
        grid_sync(&a.ews->bar, G);
        if (blk == 0) {
          for (int r = 0; r < kRounds; ++r)
            for (int b = threadIdx.x; b < kHistLen; b += kMergeThreads) a.ews->hist[r][b] = 0;
          if (threadIdx.x < kRounds) a.ews->gather_n[threadIdx.x] = 0;
        }
        grid_sync(&a.ews->bar, G);
      }
    }
    const bool ka = first && keep_all;
    ok = engine_run<kMergeThreads>(src, d0, d1, ka ? n_valid : a.k, ka, first ? win_lo : 0u, first ? win_shift : 20u,
                                   first ? esm.hist : nullptr, first, a.ews, esm, out, G);
    if (first) {
      merge_stamp(a, 4);  // engine done
      if (a.trace && rec && blk == 0 && threadIdx.x == 0) a.trace[13] = __ldcg(rec + 1);
    }
  }
  // every block read n_valid before the engine's first barrier
  if (!solo && blk == 0 && threadIdx.x == 0) a.ctl->n_valid = 0;
}

}  // namespace gtk
