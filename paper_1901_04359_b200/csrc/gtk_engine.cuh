// Exact top-k "engine": given an index-ordered list of slots (each slot either
// empty or an (idx, val) entry with a 31-bit magnitude key), keep exactly the
// kt entries that are largest by (key desc, idx asc) -- the reference's rule
// (sparse.py:148-150 for select, sparse.py:188-192 for top_op) -- and write them
// out in index order (the input order IS the index order and the compaction is
// stable, so no sort is ever needed).
//
// Runs inside a cooperative kernel: G blocks, block b owning the contiguous
// slot range [s0, s1) (ranges ascending with b).  The slice normally lives in
// shared memory (SmemSrc), so every pass below is LDS-speed; the dense exact
// fallback streams its slice from global memory (DenseSrc).  The k-th key tau
// is found by radix refinement over 2049-bin histograms (2048 window bins +
// OVER), rounds shrinking the window 2^11-fold, finishing either when a bin is
// one key wide or when the target bin holds <= kGatherCap entries (gathered
// and ranked by brute force).  Ties at tau are resolved in index order with a
// grid-wide prefix of per-block equal-key counts.
#pragma once

#include "gtk_common.cuh"

namespace gtk {

constexpr int kBins = 2048;                 // window bins
constexpr int kHistLen = kBins + 1;         // + OVER
constexpr int kHistStride = 2056;           // padded
constexpr int kRounds = 4;
constexpr int kGatherCap = 1024;
constexpr int kMaxBlocks = 1024;

struct EngineWS {
  GridBarrier bar;
  uint32_t gather_n[kRounds];
  uint32_t pad0[10];
  uint32_t hist[kRounds][kHistStride];
  uint32_t gather_key[kGatherCap];
  uint32_t cta_a[kMaxBlocks];
  uint32_t cta_b[kMaxBlocks];
};

template <int NT>
struct EngineSmem {
  uint32_t hist[kHistStride];
  uint32_t keys[kGatherCap];
  uint32_t scan[NT / 32 + 2];
  uint32_t bcast[8];
};

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
  int32_t* d_count;
  float* zero_at;  // select: res_out[idx] = +0.0 for kept entries (nullable)
};

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
  uint32_t t = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) t += red[w];
  __syncthreads();
  return t;
}

// Histogram my slice's keys in [lo, hi) into a round's global histogram.
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
      atomicAdd(&sm.hist[bin], 1u);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kHistLen; b += NT) {
    const uint32_t c = sm.hist[b];
    if (c) atomicAdd(ghist + b, c);
  }
}

// Find the bin holding rank t (1-based, from the top, OVER first).  All blocks
// compute the same answer.  Returns false if the histogram holds < t entries.
template <int NT>
__device__ bool engine_find_bin(const uint32_t* ghist, uint32_t t, EngineSmem<NT>& sm, uint32_t& bin,
                                uint32_t& above, uint32_t& in_bin, uint32_t& total) {
  constexpr int PER = (kHistLen + NT - 1) / NT;
  // thread t owns reversed positions [t*PER, t*PER+PER): rb = 0 is OVER (bin 2048)
  uint32_t c[PER];
  uint32_t sum = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int rb = threadIdx.x * PER + j;
    c[j] = rb < kHistLen ? __ldcg(ghist + (kBins - rb)) : 0u;
    sum += c[j];
  }
  uint32_t tot;
  uint32_t pre = block_excl_scan<NT>(sum, sm.scan, &tot);
  if (threadIdx.x == 0) sm.bcast[0] = 0xFFFFFFFFu;
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
  __syncthreads();
  total = tot;
  bin = sm.bcast[0];
  above = sm.bcast[1];
  in_bin = sm.bcast[2];
  __syncthreads();
  return tot >= t && bin != 0xFFFFFFFFu;
}

// The engine proper.  Every block calls it with its own slice [s0, s1).
// Returns false (consistently in all blocks) if the round-0 histogram holds
// fewer than kt entries (select: fallback needed).
//   round0_ready: ws->hist[0] already holds the slots' histogram over
//                 [lo0, 2^31) with bin width 2^shift0 (built by the producer
//                 and made visible by a grid barrier or kernel boundary)
//   kt / keep_all: keep_all keeps every valid slot (kt is then ignored and the
//                 output count is the number of valid slots).
template <int NT, class Src>
__device__ bool engine_run(const Src& src, uint32_t s0, uint32_t s1, uint32_t kt, bool keep_all, uint32_t lo0,
                           uint32_t shift0, bool round0_ready, EngineWS* ws, EngineSmem<NT>& sm,
                           const Sink& out, unsigned G) {
  const unsigned blk = blockIdx.x;
  uint32_t tau = 0, n_gt = 0, need = 0;
  if (!keep_all) {
    uint32_t lo = lo0, shift = shift0;
    uint64_t hi = 0x80000000ull;
    uint32_t t = kt, acc_above = 0;
    bool done = false;
    for (int r = 0; r < kRounds && !done; ++r) {
      if (r > 0 || !round0_ready) {
        engine_hist<NT>(src, s0, s1, lo, hi, shift, ws->hist[r], sm);
        grid_sync(&ws->bar, G);
      }
      uint32_t bin, above, in_bin, total;
      if (!engine_find_bin<NT>(ws->hist[r], t, sm, bin, above, in_bin, total)) return false;
      uint64_t blo, bhi;
      if (bin < (uint32_t)kBins) {
        blo = (uint64_t)lo + ((uint64_t)bin << shift);
        bhi = blo + (1ull << shift);
        if (bhi > hi) bhi = hi;
      } else {
        blo = (uint64_t)lo + ((uint64_t)kBins << shift);
        bhi = hi;
      }
      const uint32_t t_in = t - above;
      if (bhi - blo == 1) {
        tau = (uint32_t)blo;
        n_gt = acc_above + above;
        done = true;
        break;
      }
      if (in_bin <= (uint32_t)kGatherCap) {
        // gather the keys of the target bin, rank them by brute force
        for (uint32_t s = s0 + threadIdx.x; s < s1; s += NT) {
          uint32_t key;
          int32_t i;
          float v;
          if (src.get(s, key, i, v) && key >= blo && key < bhi) {
            const uint32_t p = atomicAdd(&ws->gather_n[r], 1u);
            ws->gather_key[p] = key;
          }
        }
        grid_sync(&ws->bar, G);
        const uint32_t ng = __ldcg(&ws->gather_n[r]);
        for (uint32_t j = threadIdx.x; j < ng; j += NT) sm.keys[j] = __ldcg(&ws->gather_key[j]);
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < ng; j += NT) {
          const uint32_t x = sm.keys[j];
          uint32_t gt = 0, ge = 0;
          for (uint32_t q = 0; q < ng; ++q) {
            const uint32_t y = sm.keys[q];
            gt += (y > x);
            ge += (y >= x);
          }
          if (gt < t_in && ge >= t_in) {
            sm.bcast[3] = x;
            sm.bcast[4] = gt;
          }
        }
        __syncthreads();
        tau = sm.bcast[3];
        n_gt = acc_above + above + sm.bcast[4];
        __syncthreads();
        done = true;
        break;
      }
      // refine inside the target bin
      acc_above += above;
      t = t_in;
      lo = (uint32_t)blo;
      hi = bhi;
      const uint64_t width = bhi - blo;
      shift = width <= (uint64_t)kBins ? 0u : ceil_log2_u64((width + kBins - 1) / kBins);
    }
    if (!done) return false;  // unreachable: shift reaches 0 within kRounds
    need = kt - n_gt;
  }

  // ---- compaction: per-block counts, grid prefix, stable write -------------
  uint32_t c_a = 0, c_b = 0;  // keep_all: (valid, -)  else (gt, eq)
  for (uint32_t s = s0 + threadIdx.x; s < s1; s += NT) {
    uint32_t key;
    int32_t i;
    float v;
    if (src.get(s, key, i, v)) {
      if (keep_all) {
        c_a++;
      } else {
        c_a += key > tau;
        c_b += key == tau;
      }
    }
  }
  c_a = block_sum<NT>(c_a, sm.scan);
  c_b = block_sum<NT>(c_b, sm.scan);
  if (threadIdx.x == 0) {
    ws->cta_a[blk] = c_a;
    ws->cta_b[blk] = c_b;
  }
  grid_sync(&ws->bar, G);

  // self-clean the histogram/gather state for the next engine use (every block
  // is past its last histogram read)
  if (blk == 0) {
    for (int r = 0; r < kRounds; ++r)
      for (int b = threadIdx.x; b < kHistLen; b += NT) ws->hist[r][b] = 0;
    if (threadIdx.x < kRounds) ws->gather_n[threadIdx.x] = 0;
  }

  uint32_t a_before = 0, b_before = 0, a_all = 0;
  for (unsigned j = threadIdx.x; j < G; j += NT) {
    const uint32_t a = __ldcg(&ws->cta_a[j]);
    const uint32_t b = __ldcg(&ws->cta_b[j]);
    if (j < blk) {
      a_before += a;
      b_before += b;
    }
    a_all += a;
  }
  a_before = block_sum<NT>(a_before, sm.scan);
  b_before = block_sum<NT>(b_before, sm.scan);
  a_all = block_sum<NT>(a_all, sm.scan);

  uint32_t out_pos = keep_all ? a_before : a_before + min(b_before, need);
  uint32_t eq_seen = b_before;
  for (uint32_t base = s0; base < s1; base += NT) {
    const uint32_t s = base + threadIdx.x;
    uint32_t key = 0;
    int32_t i = 0;
    float v = 0.f;
    bool valid = false;
    if (s < s1) valid = src.get(s, key, i, v);
    bool keep;
    uint32_t is_eq = 0;
    if (keep_all) {
      keep = valid;
    } else {
      is_eq = valid && key == tau;
      keep = valid && key > tau;
    }
    uint32_t eq_tot = 0;
    uint32_t eq_rank = 0;
    if (!keep_all) eq_rank = block_excl_scan<NT>(is_eq, sm.scan, &eq_tot);
    if (is_eq && eq_seen + eq_rank < need) keep = true;
    uint32_t k_tot;
    const uint32_t k_rank = block_excl_scan<NT>(keep ? 1u : 0u, sm.scan, &k_tot);
    if (keep) {
      const uint32_t p = out_pos + k_rank;
      out.o_idx[p] = i;
      out.o_val[p] = v;
      if (out.zero_at) out.zero_at[i] = 0.0f;
    }
    out_pos += k_tot;
    eq_seen += eq_tot;
  }
  if (blk == 0 && threadIdx.x == 0) *out.d_count = (int32_t)(keep_all ? a_all : kt);
  return true;
}

}  // namespace gtk
