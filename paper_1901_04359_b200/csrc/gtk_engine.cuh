// Exact top-k "engine": given an index-ordered list of slots (each slot either
// empty or an (idx, val) entry with a 31-bit magnitude key), keep exactly the
// kt entries that are largest by (key desc, idx asc) -- the reference's rule
// (sparse.py:148-150 for select, sparse.py:188-192 for top_op) -- and write them
// out in index order (the input order IS the index order and the compaction is
// stable, so no sort is ever needed).
//
// Runs inside a cooperative kernel: G blocks, block b owning the contiguous
// slot range [s0, s1) (ranges ascending with b), normally staged in shared
// memory.  The k-th key tau is located with 2049-bin histograms (2048 window
// bins + OVER): find the bin b holding rank kt; if b is narrow enough
// (<= kGatherCap entries, or a single key) finish with ONE grid barrier:
//     every block counts its entries above b and gathers its entries inside b
//     as (key, idx, block); after the barrier every block derives tau, the
//     index-order tie ranks and its own output offset from the gathered set
//     and the per-block counts, and writes its winners;
// otherwise refine the window inside b (2^11-fold per round).
// With G == 1 histograms and the gather stay in shared memory (no barriers).
#pragma once

#include "gtk_common.cuh"

namespace gtk {

constexpr int kBins = 2048;                 // window bins
constexpr int kHistLen = kBins + 1;         // + OVER
constexpr int kHistStride = 2056;           // padded
constexpr int kRounds = 4;
constexpr int kGatherCap = 1024;  // gather buffer size
constexpr int kGatherMax = 384;   // gathered entries loaded speculatively with the count after the barrier
constexpr int kRankDirect = 96;   // gathers up to this size are ranked O(n^2) directly; larger via a sub-histogram
constexpr int kMaxBlocks = 1024;
#ifndef GTK_MERGE_BIN_TARGET
#define GTK_MERGE_BIN_TARGET 64
#endif
constexpr uint32_t kMergeBinTarget = GTK_MERGE_BIN_TARGET;  // merge windows: entries in the k-th key's bin

struct EngineWS {
  GridBarrier bar;
  uint32_t gather_n[kRounds];  // zeroed by the producer of the run's first histogram
  uint32_t pad0[10];
  uint32_t hist[kRounds][kHistStride];
  uint32_t gather_key[kGatherCap];
  int32_t gather_idx[kGatherCap];
  uint32_t gather_blk[kGatherCap];
  uint32_t cta_a[kMaxBlocks];
  uint32_t cta_b[kMaxBlocks];
};

constexpr uint32_t kKeptBits = 32768;  // slice slots covered by the kept bitmap (a finish slice is <= 20480)
constexpr uint32_t kSlotBits = 22;    // gather record: (block << 22) | slot within the block's slice
// slots past kSlotMax (a dense-fallback slice of m > ~600M elements) are
// recorded as kSlotMax: any slot >= kKeptBits is resolved by index (keep_fn's
// scan), so only the block field must stay exact; kSlotMax < 2^22 - 1 keeps
// the record of block 1023 distinct from the "not kept" mark 0xFFFFFFFF
constexpr uint32_t kSlotMax = (1u << kSlotBits) - 2;
static_assert(kKeptBits <= kSlotMax, "kept bitmap beyond the slot field");

template <int NT>
struct EngineSmem {
  uint32_t hist[kHistStride];
  uint32_t keys[kGatherCap];
  int32_t gidx[kGatherCap];
  uint32_t gblk[kGatherCap];
  uint32_t kept_bits[kKeptBits / 32];  // my slice's in-bin winners
  uint32_t wcnt[NT];                    // engine_write: kept per (row, warp), then their exclusive scan
  uint32_t wbal[NT];                    // engine_write: kept ballot per (row, warp)
  uint32_t scan[NT / 32 + 2];
  uint32_t bcast[8];
  uint32_t ng;
};

// binary searches over an ascending index list in shared memory
static __device__ __forceinline__ uint32_t lower_bound_s(const int32_t* s, uint32_t n, int32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (s[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
static __device__ __forceinline__ uint32_t upper_bound_s(const int32_t* s, uint32_t n, int32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (s[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// ---- slot sources -------------------------------------------------------------
// get(s, key, idx, val) -> slot s holds an entry?  Only s in the block's own
// [s0, s1) is ever requested.
// A block's slice, staged either in shared memory (the normal case: indexed
// s - s0) or -- when it does not fit -- in a global scratch list indexed by s
// (written by this same block earlier in the kernel).  idx < 0 = empty slot.
struct SliceSrc {
  const int32_t* sidx;  // shared
  const float* sval;
  const int32_t* gidx;  // global
  const float* gval;
  uint32_t s0;
  bool in_smem;
  bool merge_keys;  // ⊤ ordering: NaN magnitudes rank last (numpy lexsort)
  __device__ __forceinline__ bool get(uint32_t s, uint32_t& key, int32_t& i, float& v) const {
    if (in_smem) {
      i = sidx[s - s0];
      v = sval[s - s0];
    } else {
      i = __ldcg(gidx + s);
      v = __ldcg(gval + s);
    }
    key = merge_keys ? merge_key_of(v) : key_of(v);
    return i >= 0;
  }
};
struct DenseSrc {  // dense fallback: slot s is element s
  const float* val;
  __device__ __forceinline__ bool get(uint32_t s, uint32_t& key, int32_t& i, float& v) const {
    i = (int32_t)s;
    v = __ldcg(val + s);
    key = key_of(v);
    return true;
  }
};

struct Sink {
  int32_t* o_idx;
  float* o_val;
  int32_t* d_count;  // d_count[0] = kept entries; d_count[1] = kt-th key hint (0 = none)
  float* zero_at;    // select: res_out[idx] = +0.0 for kept entries (nullable)
  bool write_hint;
  int64_t* trace;    // optional %globaltimer stamps of block 0: [0] bin found, [1] after gather barrier, [2] ranked, [3] written
  uint32_t* next_window;  // select only (nullable): the next call's key window, see engine_run
  uint32_t window_level;  // margin level L >= 1: the next window admits ~k (1 + 2^L / 2) keys
  uint32_t prev_tau;      // the previous call's approximate k-th key (0: none)
  uint32_t prev_tau2;     // ... and the one before
  uint32_t window_rank_shift;  // lo' sits at rank kt (1 + 2^L >> shift): select 1, merge 3 (a union holds <= 2 kt)
  // select + K3 at P = 1 (gtk_select_update): w[idx] -= FLOAT(lr) * u(val) for
  // every kept entry, the sparse update of gtk_scatter_update (nullable)
  float* upd_w;
  float upd_lr;
  float upd_Pf;
  int upd_scaling;
  uint32_t* tag;      // exchange + K3: tag[idx] = tag_val marks membership of the final global list (nullable)
  uint32_t tag_val;
  // exchange: the output also goes straight to the next step's partner as LL
  // records (body[2p] = {idx, val bits}, head = {count, hint}), nullable
  uint64_t* ll_body = nullptr;
  uint64_t* ll_head = nullptr;
  uint32_t ll_tag = 0;
  // chained select (GTK_SELECT_CHAIN): the winners' residual slots are left
  // pending instead of zeroed; the exact winner predicate goes to the key
  // window record: rec[6] = tau (the k-th key), rec[7] = cut (the largest
  // index among the kept entries with key == tau), rec[0] |= kRecPending --
  // i is a winner iff key > tau || (key == tau && i <= cut) (nullable)
  uint32_t* pend_rec = nullptr;
  // deferred select: every block's first output position ([1 + blk]; [0] = G)
  uint32_t* blk_ofs = nullptr;
  // the fused w update is skipped when this status word holds an error bit,
  // read once per block after the engine's last barrier (nullable: always)
  const uint32_t* upd_skip = nullptr;
};

// the sink a block writes with: upd_w dropped when the status word (final
// behind the engine's last barrier) holds an error bit
__device__ __forceinline__ Sink sink_for_write(const Sink& out) {
  Sink o = out;
  if (o.upd_w && o.upd_skip && (__ldcg(o.upd_skip) & GTK_DEV_ERROR_MASK)) o.upd_w = nullptr;
  return o;
}

constexpr uint32_t kRecValid = 0x1u;    // window record word 0: lo/shift/k describe the next call's window
constexpr uint32_t kRecPending = 0x2u;  // ... the residual still holds the last chained call's winners

// block 0, thread 0, after the write: the pending-winner predicate (chained select)
__device__ __forceinline__ void sink_pending(const Sink& out, uint32_t tau) {
  if (out.pend_rec) {
    out.pend_rec[6] = tau;
    out.pend_rec[0] = out.pend_rec[0] | kRecPending;
  }
}

// block 0 publishes the output count (and the k-th-key hint)
__device__ __forceinline__ void sink_count(const Sink& out, uint32_t n, uint32_t hint) {
  out.d_count[0] = (int32_t)n;
  if (out.write_hint) out.d_count[1] = (int32_t)hint;
  if (out.ll_head) st_ll_pair(out.ll_head, n, out.write_hint ? hint : 0u, out.ll_tag);
}

// one kept entry to the output list (+ the select's side effects)
__device__ __forceinline__ void sink_put(const Sink& out, uint32_t p, int32_t i, float v) {
  GTK_DCHECK(i >= 0);
  out.o_idx[p] = i;
  out.o_val[p] = v;
  if (out.zero_at) out.zero_at[i] = 0.0f;
  if (out.upd_w) out.upd_w[i] = __fsub_rn(out.upd_w[i], __fmul_rn(out.upd_lr, scale_u(v, out.upd_Pf, out.upd_scaling)));
  if (out.tag) out.tag[i] = out.tag_val;
  if (out.ll_body) st_ll_pair(out.ll_body + 2 * (size_t)p, (uint32_t)i, __float_as_uint(v), out.ll_tag);
}

__device__ __forceinline__ void sink_stamp(const Sink& out, int i) {
  if (out.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    out.trace[i] = (int64_t)t;
  }
}

__device__ __forceinline__ void slice_of(uint32_t N, unsigned G, unsigned b, uint32_t& s0, uint32_t& s1) {
  const uint32_t S = (N + G - 1) / G;
  s0 = min((uint64_t)N, (uint64_t)b * S);
  s1 = min((uint64_t)N, (uint64_t)s0 + S);
}

// block-wide sum of one value per thread (all threads get the result)
template <int NT>
__device__ __forceinline__ uint32_t block_sum(uint32_t v, uint32_t* red) {
  v = warp_sum(v);
  __syncthreads();
  if (lane_id() == 0) red[warp_id()] = v;
  __syncthreads();
  const uint32_t t = warp_sum(lane_id() < (unsigned)(NT / 32) ? red[lane_id()] : 0u);
  __syncthreads();
  return t;
}

// Histogram my slice's keys in [lo, hi) into sm.hist; flush to ghist if given.
template <int NT, class Src>
__device__ void engine_hist(const Src& src, uint32_t s0, uint32_t s1, uint32_t lo, uint64_t hi,
                            uint32_t shift, uint32_t* ghist, EngineSmem<NT>& sm) {
  for (int b = threadIdx.x; b < kHistLen; b += NT) sm.hist[b] = 0;
  __syncthreads();
  for (uint32_t s = s0 + threadIdx.x; s < s1; s += NT) {
    uint32_t key;
    int32_t i;
    float v;
    if (src.get(s, key, i, v) && key >= lo && (uint64_t)key < hi) {
      const uint32_t bin = min((uint32_t)kBins, (key - lo) >> shift);
      GTK_DCHECK(bin < (uint32_t)kHistLen);
      atomicAdd(&sm.hist[bin], 1u);
    }
  }
  __syncthreads();
  if (ghist) {
    for (int b = threadIdx.x; b < kHistLen; b += NT) {
      const uint32_t c = sm.hist[b];
      if (c) atomicAdd(ghist + b, c);
    }
  }
}

// Find the bin holding rank t (1-based, from the top, OVER first) of a
// histogram in global (ldcg) or shared memory.  All blocks compute the same
// answer.  Returns false if the histogram holds < t entries.
template <int NT>
__device__ bool engine_find_bin(const uint32_t* hist, bool in_smem, uint32_t t, EngineSmem<NT>& sm,
                                uint32_t& bin, uint32_t& above, uint32_t& in_bin, uint32_t t2 = 0,
                                uint32_t t3 = 0, uint32_t* bin2 = nullptr, uint32_t* bin3 = nullptr,
                                uint32_t* above2 = nullptr) {
  constexpr int PER = (kHistLen + NT - 1) / NT;
  // thread t owns reversed positions [t*PER, t*PER+PER): rb = 0 is OVER (bin 2048)
  uint32_t c[PER];
  uint32_t sum = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int rb = threadIdx.x * PER + j;
    c[j] = rb < kHistLen ? (in_smem ? hist[kBins - rb] : __ldcg(hist + (kBins - rb))) : 0u;
    sum += c[j];
  }
  uint32_t tot;
  uint32_t pre = block_excl_scan<NT>(sum, sm.scan, &tot);
  if (threadIdx.x == 0) sm.bcast[0] = sm.bcast[5] = sm.bcast[6] = 0xFFFFFFFFu;
  __syncthreads();
  if (pre < t && pre + sum >= t) {
    uint32_t acc = pre;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      if (acc < t && acc + c[j] >= t) {
        sm.bcast[0] = kBins - (threadIdx.x * PER + j);
        sm.bcast[1] = acc;
        sm.bcast[2] = c[j];
      }
      acc += c[j];
    }
  }
  if (t2 != 0) {  // extra ranks (bins only), same scan
    uint32_t acc = pre;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      if (acc < t2 && acc + c[j] >= t2) {
        sm.bcast[5] = kBins - (threadIdx.x * PER + j);
        sm.bcast[3] = acc;  // (entries above rank t2's bin)
      }
      if (acc < t3 && acc + c[j] >= t3) sm.bcast[6] = kBins - (threadIdx.x * PER + j);
      acc += c[j];
    }
  }
  __syncthreads();
  bin = sm.bcast[0];
  above = sm.bcast[1];
  in_bin = sm.bcast[2];
  if (bin2) *bin2 = sm.bcast[5];
  if (bin3) *bin3 = sm.bcast[6];
  if (above2) *above2 = sm.bcast[3];
  __syncthreads();
  return tot >= t && bin != 0xFFFFFFFFu;
}

// Up to kSinkBatch kept entries (bi, bv) to output positions bp: every
// dependent load (w[idx] of the fused update) is issued before the first
// store, so a thread with many winners pays one memory round trip per batch,
// not one per entry (the stores could alias the next entry's load as far as
// the compiler knows, so a plain loop of sink_put serialises them).
constexpr int kSinkBatch = 4;
__device__ __forceinline__ void sink_put_batch(const Sink& out, const uint32_t (&bp)[kSinkBatch],
                                               const int32_t (&bi)[kSinkBatch], const float (&bv)[kSinkBatch],
                                               int n) {
  float wv[kSinkBatch];
  if (out.upd_w) {
#pragma unroll
    for (int j = 0; j < kSinkBatch; ++j)
      if (j < n) wv[j] = out.upd_w[bi[j]];
  }
#pragma unroll
  for (int j = 0; j < kSinkBatch; ++j) {
    if (j >= n) break;
    const int32_t i = bi[j];
    const float v = bv[j];
    GTK_DCHECK(i >= 0);
    out.o_idx[bp[j]] = i;
    out.o_val[bp[j]] = v;
    if (out.zero_at) out.zero_at[i] = 0.0f;
    if (out.upd_w) out.upd_w[i] = __fsub_rn(wv[j], __fmul_rn(out.upd_lr, scale_u(v, out.upd_Pf, out.upd_scaling)));
    if (out.tag) out.tag[i] = out.tag_val;
    if (out.ll_body) st_ll_pair(out.ll_body + 2 * (size_t)bp[j], (uint32_t)i, __float_as_uint(v), out.ll_tag);
  }
}

// Stable index-order write of my slice's kept entries at out_pos.. .
// keep(key, idx, slot) decides; positions via one block scan per chunk.
// A chunk is 32 rows of NT slots, thread t reading slot row * NT + t of
// each row (conflict-free shared-memory reads, consecutive lanes writing
// consecutive output positions); the per-(row, warp) kept counts -- 32 x
// NT/32 = NT of them -- are scanned in one block scan.
template <int NT, class Src, class Keep>
__device__ void engine_write(const Src& src, uint32_t s0, uint32_t s1, uint32_t out_pos, const Keep& keep_fn,
                             EngineSmem<NT>& sm, const Sink& out) {
  constexpr int NW = NT / 32;
  const unsigned lane = lane_id(), w = warp_id();
  for (uint32_t c0 = s0; c0 < s1; c0 += 32u * NT) {
    const uint32_t nrows = min(32u, (s1 - c0 + NT - 1) / NT);
    uint32_t kbits = 0;
    for (uint32_t r = 0; r < nrows; ++r) {
      const uint32_t s = c0 + r * NT + threadIdx.x;
      uint32_t key;
      int32_t i;
      float v;
      const bool kept = s < s1 && src.get(s, key, i, v) && keep_fn(key, i, s - s0);
      const unsigned bal = __ballot_sync(kFull, kept);
      GTK_DCHECK(r * NW + w < (uint32_t)NT);
      if (lane == 0) {
        sm.wcnt[r * NW + w] = __popc(bal);
        sm.wbal[r * NW + w] = bal;
      }
      kbits |= (uint32_t)kept << r;
    }
    __syncthreads();
    uint32_t k_tot;
    const uint32_t cnt = threadIdx.x < nrows * NW ? sm.wcnt[threadIdx.x] : 0u;
    const uint32_t ex = block_excl_scan<NT>(cnt, sm.scan, &k_tot);
    sm.wcnt[threadIdx.x] = ex;
    __syncthreads();
    if (c0 == s0 && out.zero_at) sink_stamp(out, 5);  // (select only: a merge keeps diagnostics there)
    const unsigned lt = lanemask_lt();
    while (kbits) {
      uint32_t bp[kSinkBatch];
      int32_t bi[kSinkBatch];
      float bv[kSinkBatch];
      int n = 0;
#pragma unroll
      for (int j = 0; j < kSinkBatch; ++j) {
        if (kbits) {
          const uint32_t r = __ffs(kbits) - 1;
          kbits &= kbits - 1;
          uint32_t key;
          src.get(c0 + r * NT + threadIdx.x, key, bi[j], bv[j]);
          bp[j] = out_pos + sm.wcnt[r * NW + w] + __popc(sm.wbal[r * NW + w] & lt);
          n = j + 1;
        }
      }
      sink_put_batch(out, bp, bi, bv, n);
    }
    out_pos += k_tot;
    __syncthreads();  // sm.wcnt is reused by the next chunk
    if (c0 == s0 && out.zero_at) sink_stamp(out, 6);
  }
}

// ---- finish from the bin [blo, bhi) of keys that holds the rank-kt key ----
// Every block gathers its in-bin entries (key, idx, block | slot) into the
// shared gather buffer (gcount: its global counter; nullptr = G == 1, all in
// shared memory) and counts its entries above the bin; after ONE grid
// barrier every block ranks the gathered keys (tau = the t_in-th largest of
// them, t_in = rank of the target inside the bin, ties at tau by index),
// derives its output offset and writes its winners.
template <int NT, class Src>
__device__ void engine_gather_finish(const Src& src, uint32_t s0, uint32_t s1, uint32_t kt, uint32_t t_in,
                                     uint64_t blo, uint64_t bhi, uint32_t* gcount, EngineWS* ws,
                                     EngineSmem<NT>& sm, const Sink& out, unsigned G) {
  const unsigned blk = blockIdx.x;
  const bool solo = gcount == nullptr;
  uint32_t n_above = 0;
  if (solo && threadIdx.x == 0) sm.ng = 0;
  if (solo) __syncthreads();
  // (block-uniform trip count: the in-bin slots are reserved with one
  // atomic per warp)
  for (uint32_t sb0 = s0; sb0 < s1; sb0 += NT) {
    const uint32_t s = sb0 + threadIdx.x;
    uint32_t key = 0;
    int32_t i = 0;
    float v;
    const bool valid = s < s1 && src.get(s, key, i, v);
    n_above += valid && (uint64_t)key >= bhi;
    const bool inb = valid && (uint64_t)key < bhi && key >= blo;
    // a potential winner: its w line (fused update) heads for L2 now, so
    // the write phase's read-modify-write after the barrier hits there
    if (out.upd_w && valid && key >= blo) prefetch_l2(out.upd_w + i);
    const unsigned bal = __ballot_sync(kFull, inb);
    if (bal == 0u) continue;
    uint32_t p0 = 0;
    if (lane_id() == (unsigned)(__ffs(bal) - 1))
      p0 = atomicAdd(solo ? &sm.ng : gcount, (uint32_t)__popc(bal));
    p0 = __shfl_sync(kFull, p0, __ffs(bal) - 1);
    if (inb) {
      const uint32_t p = p0 + __popc(bal & lanemask_lt());
      GTK_DCHECK(p < (uint32_t)kGatherCap);
      if (p >= (uint32_t)kGatherCap) continue;  // (cannot happen: in_bin <= kGatherCap)
      if (solo) {
        sm.keys[p] = key;
        sm.gidx[p] = i;
        sm.gblk[p] = (blk << kSlotBits) | min(s - s0, kSlotMax);
      } else {
        ws->gather_key[p] = key;
        ws->gather_idx[p] = i;
        ws->gather_blk[p] = (blk << kSlotBits) | min(s - s0, kSlotMax);
      }
    }
  }
  n_above = block_sum<NT>(n_above, sm.scan);
  uint32_t above_before = 0;
  if (!solo) {
    GTK_DCHECK(blk < (unsigned)kMaxBlocks);
    if (threadIdx.x == 0) ws->cta_a[blk] = n_above;
    grid_sync(&ws->bar, G);
    // one round trip: the count, the (at most kGatherMax) gathered entries
    // and the per-block counts are independent loads
    const uint32_t ng = min(__ldcg(gcount), (uint32_t)kGatherCap + 1u);
    for (uint32_t j = threadIdx.x; j < (uint32_t)kGatherMax; j += NT) {
      sm.keys[j] = __ldcg(&ws->gather_key[j]);
      sm.gidx[j] = __ldcg(&ws->gather_idx[j]);
      sm.gblk[j] = __ldcg(&ws->gather_blk[j]);
    }
    for (uint32_t j = kGatherMax + threadIdx.x; j < min(ng, (uint32_t)kGatherCap); j += NT) {  // up to kGatherCap
      sm.keys[j] = __ldcg(&ws->gather_key[j]);
      sm.gidx[j] = __ldcg(&ws->gather_idx[j]);
      sm.gblk[j] = __ldcg(&ws->gather_blk[j]);
    }
    for (unsigned j = threadIdx.x; j < blk; j += NT) above_before += __ldcg(&ws->cta_a[j]);
    if (threadIdx.x == 0) sm.ng = ng;
  }
  above_before = block_sum<NT>(above_before, sm.scan);  // also publishes sm.keys / sm.ng
  sink_stamp(out, 1);
  const uint32_t ng = sm.ng;
  // tau = t_in-th largest gathered key; gt = # gathered keys > tau.  A
  // large gather is first narrowed in shared memory: a 2048-way histogram
  // of the bin [blo, bhi) over the gathered keys (every block holds the
  // same gathered set, so no barrier), then the O(n^2) rank runs only over
  // the sub-bin holding t_in.
  const uint32_t* rk = sm.keys;  // the keys ranked below
  uint32_t nr = ng, r_t = t_in, r_above = 0;
  if (ng > (uint32_t)kRankDirect) {
    const uint64_t width = bhi - blo;
    const uint32_t ss = width <= (uint64_t)kBins ? 0u : ceil_log2_u64((width + kBins - 1) / kBins);
    for (int b = threadIdx.x; b < kHistLen; b += NT) sm.hist[b] = 0;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < ng; j += NT) atomicAdd(&sm.hist[(sm.keys[j] - (uint32_t)blo) >> ss], 1u);
    __syncthreads();
    uint32_t sb, sab, sin;
    engine_find_bin<NT>(sm.hist, true, t_in, sm, sb, sab, sin);
    const uint32_t r_lo = (uint32_t)blo + (sb << ss), r_hi = r_lo + ((1u << ss) - 1u);  // inclusive
    if (threadIdx.x == 0) sm.bcast[7] = 0;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < ng; j += NT) {  // the sub-bin's keys -> sm.hist[0, sin)
      const uint32_t x = sm.keys[j];
      if (x >= r_lo && x <= r_hi) sm.hist[atomicAdd(&sm.bcast[7], 1u)] = x;
    }
    rk = sm.hist;
    nr = sin;
    r_t = t_in - sab;
    r_above = sab;
  }
  if (threadIdx.x == 0) sm.bcast[3] = sm.bcast[4] = 0;
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < nr; j += NT) {
    const uint32_t x = rk[j];
    uint32_t gt = 0, ge = 0;
    for (uint32_t q = 0; q < nr; ++q) {
      const uint32_t y = rk[q];
      gt += (y > x);
      ge += (y >= x);
    }
    if (gt < r_t && ge >= r_t) {
      sm.bcast[3] = x;
      sm.bcast[4] = r_above + gt;
    }
  }
  __syncthreads();
  const uint32_t tau = sm.bcast[3];
  const uint32_t need = t_in - sm.bcast[4];  // entries with key == tau to keep, lowest idx first
  sink_stamp(out, 2);
  // kept flags of the gathered entries: winners of my slice go to a
  // bitmap indexed by slot (O(1) lookup in the write), the ones of
  // earlier blocks shift my output offset
  // the gathered entries equal to tau (their indices) -> sm.hist[0, n_eq):
  // the index-order tie ranks run over that short list only
  for (uint32_t w = threadIdx.x; w < kKeptBits / 32; w += NT) sm.kept_bits[w] = 0;
  if (threadIdx.x == 0) sm.bcast[7] = 0;
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < ng; j += NT)
    if (sm.keys[j] == tau) sm.hist[atomicAdd(&sm.bcast[7], 1u)] = (uint32_t)sm.gidx[j];
  __syncthreads();
  const uint32_t n_eq = sm.bcast[7];
  uint32_t extra = 0;
  for (uint32_t j = threadIdx.x; j < ng; j += NT) {
    const uint32_t x = sm.keys[j];
    bool kept = x > tau;
    if (x == tau) {
      uint32_t rank = 0;
      const int32_t ij = sm.gidx[j];
      for (uint32_t q = 0; q < n_eq; ++q) rank += (int32_t)sm.hist[q] < ij;
      kept = rank < need;
      if (out.pend_rec && blk == 0 && rank + 1 == need) out.pend_rec[7] = (uint32_t)ij;  // the last kept tie
    }
    const uint32_t gb = sm.gblk[j] >> kSlotBits, slot = sm.gblk[j] & ((1u << kSlotBits) - 1);
    if (kept) {
      if (gb < blk) ++extra;
      // (a slot beyond the bitmap -- large global-mode slice -- is found
      // by the scan in keep_fn instead)
      if (gb == blk && slot < kKeptBits) atomicOr(&sm.kept_bits[slot >> 5], 1u << (slot & 31));
    } else {
      sm.gblk[j] = 0xFFFFFFFFu;  // mark "not kept" for the large-slice scan
    }
  }
  extra = block_sum<NT>(extra, sm.scan);
  const uint32_t bl = (uint32_t)blo, bh32 = (uint32_t)min(bhi, (uint64_t)0xFFFFFFFFu);
  const bool bh_max = bhi > 0xFFFFFFFFull;
  auto keep_fn = [&](uint32_t key, int32_t i, uint32_t slot) -> bool {
    if (!bh_max && key >= bh32) return true;
    if (key < bl) return false;
    if (slot < kKeptBits) return (sm.kept_bits[slot >> 5] >> (slot & 31)) & 1u;
    for (uint32_t q = 0; q < ng; ++q)
      if (sm.gidx[q] == i) return sm.gblk[q] != 0xFFFFFFFFu;
    return false;
  };
  if (out.blk_ofs && threadIdx.x == 0) {
    out.blk_ofs[1 + blk] = above_before + extra;
    if (blk == 0) out.blk_ofs[0] = G;
  }
  engine_write<NT>(src, s0, s1, above_before + extra, keep_fn, sm, sink_for_write(out));
  sink_stamp(out, 3);
  if (blk == 0) {  // every block is past its last histogram read
    for (int rr = 0; rr < kRounds; ++rr)
      for (int b = threadIdx.x; b < kHistLen; b += NT) ws->hist[rr][b] = 0;
    if (threadIdx.x == 0) {
      sink_count(out, kt, tau);
      sink_pending(out, tau);
    }
  }
}

// The engine proper.  Every block calls it with its own slice [s0, s1).
// hist0: the round-0 histogram over [lo0, 2^31) with bin width 2^shift0,
//        already complete (global: built before a grid barrier / by an earlier
//        kernel; with G == 1 it may live in sm.hist: hist0_smem), or nullptr to
//        build it here.
// Returns false (consistently in all blocks) if round 0 holds fewer than kt
// entries (select: fallback needed; merge: widen the window).
// keep_all keeps every valid slot (kt = number of valid slots).
// slice_async: the slice is still landing by cp.async (the caller committed
// it as the last group); it is awaited after the round-0 bin is found.
template <int NT, class Src>
__device__ bool engine_run(const Src& src, uint32_t s0, uint32_t s1, uint32_t kt, bool keep_all, uint32_t lo0,
                           uint32_t shift0, const uint32_t* hist0, bool hist0_smem, EngineWS* ws,
                           EngineSmem<NT>& sm, const Sink& out, unsigned G, bool slice_async = false) {
  const unsigned blk = blockIdx.x;
  const bool solo = G == 1;

  if (slice_async && (keep_all || hist0 == nullptr)) {
    cp_async_wait_all();
    __syncthreads();
    slice_async = false;
  }
  if (keep_all) {
    uint32_t c = 0;
    for (uint32_t s = s0 + threadIdx.x; s < s1; s += NT) {
      uint32_t key;
      int32_t i;
      float v;
      c += src.get(s, key, i, v) ? 1u : 0u;
    }
    c = block_sum<NT>(c, sm.scan);
    uint32_t before = 0;
    if (!solo) {
      if (threadIdx.x == 0) ws->cta_a[blk] = c;
      grid_sync(&ws->bar, G);
      for (unsigned j = threadIdx.x; j < blk; j += NT) before += __ldcg(&ws->cta_a[j]);
      before = block_sum<NT>(before, sm.scan);
    }
    engine_write<NT>(src, s0, s1, before, [](uint32_t, int32_t, uint32_t) { return true; }, sm,
                     sink_for_write(out));
    if (blk == 0) {
      for (int r = 0; r < kRounds; ++r)
        for (int b = threadIdx.x; b < kHistLen; b += NT) ws->hist[r][b] = 0;
      if (threadIdx.x == 0) sink_count(out, kt, 0u);
    }
    return true;
  }

  uint32_t lo = lo0, shift = shift0;
  uint64_t hi = 0x80000000ull;
  uint32_t t = kt;
  const uint32_t* hist = hist0;
  bool hsm = hist0_smem;
  // a select's window recorded with no k-th-key history (the exact dense
  // pass): when the next window's lower rank t2 lies in the k-th key's bin,
  // its edge is refined with every refinement round (t2r = its rank inside
  // the current range; 0 = not tracked) -- one 2^20-key bin of a flat-topped
  // residual can hold millions of keys, and a window opening at its edge
  // overflows on every later call
  uint32_t t2r = 0;
  for (int r = 0; r < kRounds; ++r) {
    if (hist == nullptr) {
      engine_hist<NT>(src, s0, s1, lo, hi, shift, solo ? nullptr : ws->hist[r], sm);
      if (!solo) grid_sync(&ws->bar, G);
      hist = solo ? sm.hist : ws->hist[r];
      hsm = solo;
    }
    uint32_t bin, above, in_bin;
    if (r == 0 && out.next_window) {
      // select: besides rank kt, the ranks kt (1 + 2^L / 2) and kt/2 of this
      // window give the next call's window [lo', hi') -- the same parameter's
      // accumulated residual moves slowly from step to step, so next time
      // about that many candidates pass lo' (a miss costs one exact dense
      // fallback and raises L)
      uint32_t b2, b3, a2 = 0;
      const uint64_t t2w = (uint64_t)kt + (((uint64_t)kt << out.window_level) >> out.window_rank_shift);
      const uint32_t t2 = (uint32_t)min(t2w, (uint64_t)0xFFFFFFFFu), t3 = max(1u, kt / 2);
      if (!engine_find_bin<NT>(hist, hsm, t, sm, bin, above, in_bin, t2, t3, &b2, &b3, &a2)) return false;
      if (out.window_rank_shift == 1 && out.prev_tau == 0u && out.prev_tau2 == 0u && b2 == bin && t2 > a2)
        t2r = t2 - a2;
      if (blk == 0 && threadIdx.x == 0) {
        uint64_t lo_n = lo, hi_n = hi;
        if (b2 != 0xFFFFFFFFu) lo_n = (uint64_t)lo + ((uint64_t)b2 << shift);
        if (b3 != 0xFFFFFFFFu && b3 < (uint32_t)kBins) hi_n = (uint64_t)lo + ((uint64_t)(b3 + 1) << shift);
        if (hi_n > hi) hi_n = hi;
        // the k-th key's recent path (keys are log-scaled: a common relative
        // growth of the magnitudes is a common key offset):
        //  - jitter J = |second difference|: keep lo' at least 2^(L-1) J below
        //    the k-th key (flat-topped residuals pack many k below tau);
        //  - steady growth (the residual building up): shift by half the
        //    smaller of the last two increments.
        const uint32_t tau_n = (uint32_t)min((uint64_t)lo + ((uint64_t)bin << shift), (uint64_t)0x7FFFFFFFu);
        const uint32_t p1 = out.prev_tau, p2 = out.prev_tau2;
        if (p1 != 0 && p2 != 0) {
          const int64_t i1 = (int64_t)tau_n - (int64_t)p1, i2 = (int64_t)p1 - (int64_t)p2;
          const uint64_t jit = (uint64_t)(i1 > i2 ? i1 - i2 : i2 - i1);
          const uint64_t back = jit << (out.window_level - 1);
          const uint64_t lo_j = tau_n > back ? tau_n - back : 0u;
          if (lo_j < lo_n) lo_n = lo_j;
          if (i1 > 0 && i2 > 0) {
            const uint64_t d = (uint64_t)min(i1, i2) / 2;
            lo_n = min(lo_n + d, (uint64_t)0x7FFFFFFFu);
            hi_n = min(hi_n + d, (uint64_t)0x80000000u);
          }
        }
        if (hi_n <= lo_n) hi_n = lo_n + 1;
        const uint64_t width = hi_n - lo_n;
        uint32_t shift_n = width <= (uint64_t)kBins ? 0u : ceil_log2_u64((width + kBins - 1) / kBins);
        if (out.window_rank_shift >= 3 && bin < (uint32_t)kBins && in_bin > 0) {
          // merge: every union entry is processed whatever the window, so aim
          // for resolution instead -- bins narrow enough that the k-th key's
          // bin holds ~64 entries at the measured density, the k-th key in
          // the middle of the 2048 bins (>= 1024 bins of room to move down)
          const uint64_t dens_w = ((uint64_t)kMergeBinTarget << shift) / in_bin;  // key units per ~target entries
          uint32_t sd = 0;
          while (sd < 31 && (2ull << sd) <= dens_w) ++sd;
          sd += out.window_level - 2;  // a miss widens
          if (sd < shift_n) {
            shift_n = sd;
            const uint64_t half = (uint64_t)(kBins / 2) << shift_n;
            lo_n = tau_n > half ? tau_n - half : 0u;
          }
        }
        out.next_window[1] = (uint32_t)lo_n;
        out.next_window[2] = shift_n;
        out.next_window[3] = kt;
        out.next_window[4] = tau_n;
        out.next_window[5] = p1;
        out.next_window[0] = kRecValid | (out.window_level << 8);
      }
    } else if (t2r != 0) {
      uint32_t b2, a2 = 0;
      if (!engine_find_bin<NT>(hist, hsm, t, sm, bin, above, in_bin, t2r, 0u, &b2, nullptr, &a2)) return false;
      if (b2 != 0xFFFFFFFFu && b2 < (uint32_t)kBins && blk == 0 && threadIdx.x == 0) {
        // raise the recorded lower edge to rank t2's (finer) bin, same upper end
        const uint64_t lo_r = (uint64_t)lo + ((uint64_t)b2 << shift);
        const uint64_t lo_w = out.next_window[1], hi_w = lo_w + ((uint64_t)kBins << out.next_window[2]);
        if (lo_r > lo_w && lo_r < hi_w) {
          out.next_window[1] = (uint32_t)lo_r;
          const uint64_t width = hi_w - lo_r;
          out.next_window[2] = width <= (uint64_t)kBins ? 0u : ceil_log2_u64((width + kBins - 1) / kBins);
        }
      }
      t2r = (b2 == bin && t2r > a2) ? t2r - a2 : 0u;
    } else if (!engine_find_bin<NT>(hist, hsm, t, sm, bin, above, in_bin)) {
      return false;
    }
    sink_stamp(out, 0);
    if (out.trace && r == 0 && blk == 0 && threadIdx.x == 0) out.trace[4] = in_bin;  // diagnostics
    if (r == 0 && slice_async) {
      cp_async_wait_all();
      __syncthreads();
    }
    uint64_t blo, bhi;
    if (bin < (uint32_t)kBins) {
      blo = (uint64_t)lo + ((uint64_t)bin << shift);
      bhi = blo + (1ull << shift);
      if (bhi > hi) bhi = hi;
    } else {
      blo = (uint64_t)lo + ((uint64_t)kBins << shift);
      bhi = hi;
    }
    const uint32_t t_in = t - above;  // rank of the target inside the bin
    const bool single_key = (bhi - blo == 1);
    // the last round always gathers if it can (a bin is then at most 8 keys wide)
    if (in_bin <= (uint32_t)kGatherCap) {
      engine_gather_finish<NT>(src, s0, s1, kt, t_in, blo, bhi, solo ? nullptr : &ws->gather_n[r], ws, sm, out, G);
      return true;
    }
    if (single_key) {
      // ---- massive tie on one key: per-block gt/eq counts, one barrier -------
      const uint32_t tau = (uint32_t)blo;
      const uint32_t need = t_in;
      uint32_t c_gt = 0, c_eq = 0;
      for (uint32_t s = s0 + threadIdx.x; s < s1; s += NT) {
        uint32_t key;
        int32_t i;
        float v;
        if (src.get(s, key, i, v)) {
          c_gt += key > tau;
          c_eq += key == tau;
        }
      }
      c_gt = block_sum<NT>(c_gt, sm.scan);
      c_eq = block_sum<NT>(c_eq, sm.scan);
      uint32_t gt_before = 0, eq_before = 0;
      if (!solo) {
        if (threadIdx.x == 0) {
          ws->cta_a[blk] = c_gt;
          ws->cta_b[blk] = c_eq;
        }
        grid_sync(&ws->bar, G);
        for (unsigned j = threadIdx.x; j < blk; j += NT) {
          gt_before += __ldcg(&ws->cta_a[j]);
          eq_before += __ldcg(&ws->cta_b[j]);
        }
        gt_before = block_sum<NT>(gt_before, sm.scan);
        eq_before = block_sum<NT>(eq_before, sm.scan);
      }
      uint32_t out_pos = gt_before + min(eq_before, need);
      uint32_t eq_seen = eq_before;
      const Sink wout = sink_for_write(out);
      for (uint32_t base = s0; base < s1; base += NT) {
        const uint32_t s = base + threadIdx.x;
        uint32_t key = 0;
        int32_t i = 0;
        float v = 0.f;
        const bool valid = s < s1 && src.get(s, key, i, v);
        const uint32_t is_eq = valid && key == tau;
        bool keep = valid && key > tau;
        uint32_t eq_tot;
        const uint32_t eq_rank = block_excl_scan<NT>(is_eq, sm.scan, &eq_tot);
        if (is_eq && eq_seen + eq_rank < need) keep = true;
        if (is_eq && eq_seen + eq_rank + 1 == need && out.pend_rec) out.pend_rec[7] = (uint32_t)i;  // the last kept tie
        uint32_t k_tot;
        const uint32_t k_rank = block_excl_scan<NT>(keep ? 1u : 0u, sm.scan, &k_tot);
        if (keep) sink_put(wout, out_pos + k_rank, i, v);
        out_pos += k_tot;
        eq_seen += eq_tot;
      }
      if (blk == 0) {
        for (int rr = 0; rr < kRounds; ++rr)
          for (int b = threadIdx.x; b < kHistLen; b += NT) ws->hist[rr][b] = 0;
        if (threadIdx.x == 0) {
          sink_count(out, kt, tau);
          sink_pending(out, tau);
        }
      }
      return true;
    }
    // ---- refine inside the target bin ------------------------------------------
    t = t_in;
    lo = (uint32_t)blo;
    hi = bhi;
    const uint64_t width = bhi - blo;
    shift = width <= (uint64_t)kBins ? 0u : ceil_log2_u64((width + kBins - 1) / kBins);
    hist = nullptr;
  }
  return false;  // unreachable: a bin is one key wide after kRounds
}

}  // namespace gtk
