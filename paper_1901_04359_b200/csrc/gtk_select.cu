// K1: fused residual-add + exact top-k select (reference optimizer.py:219-220,
// sparse.py:135-154).
//
// Four launches per call, no host synchronisation:
//   1. select_sample  : ~128/rho sampled elements of acc = res + g (evenly
//                       strided 4 KB chunks, one per block); each block keeps
//                       its exact top-32 keys (bitwise binary search on counts).
//   2. select_window  : one block finds the exact sample order statistics
//                       around rank k*s/m (+-4 sigma) -> key window [lo, hi).
//   3. select_main    : THE HBM pass.  One 4096-element tile per block, no
//                       inter-block dependency: 128-bit streaming loads of res
//                       and g, acc = __fadd_rn(res, g) streamed to res_out, key
//                       test against lo, warp-ballot compaction of the tile's
//                       candidates (index order inside the tile) into the
//                       tile's own slot row -- or, for a dense tile, into an
//                       atomically reserved overflow region -- and a 2049-bin
//                       histogram of candidate keys over the window.
//   4. select_finish  : cooperative.  Block b owns a contiguous range of tiles;
//                       it copies their candidates (already index-ordered) into
//                       shared memory -- its slice of the global candidate
//                       list -- and the exact engine (gtk_engine.cuh) keeps the
//                       k winners, writes them in index order and zeroes their
//                       residual slots.  If the window missed (fewer than k
//                       candidates, or too many) the engine runs over the dense
//                       acc instead: the exact fallback.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "gtk_engine.cuh"
#include "gtk_internal.h"

namespace gtk {

constexpr int kMainThreads = 256;
constexpr int kMainVec = 4;                                  // float4 per thread per array
constexpr int kTile = kMainThreads * kMainVec * 4;          // 4096 elements
constexpr int kSampleThreads = 256;
constexpr int kSampleChunk = kSampleThreads * 4;            // 1024 elements per chunk
constexpr int kSampleTop = 32;                               // top keys kept per sample block
constexpr int kSampleMaxChunks = 1024;                       // sample blocks (window holds 32K keys)
constexpr int kFinishThreads = 512;
constexpr int kSliceCap = 3072;                              // candidates staged per finish block
constexpr uint32_t kOvfBit = 0x80000000u;

struct SelectCtl {
  uint32_t lo;
  uint32_t shift;
  uint32_t ovf_cursor;
  uint32_t overflow;
  uint32_t nonfinite;
  uint32_t pad[11];
};

struct SelectLayout {
  size_t ctl, sample_top, engine, tile_info, tile_ovf, slot_idx, slot_val, ovf_idx, ovf_val, ord_idx, ord_val,
      total;
  uint32_t ntiles, slots, ovf_cap, ord_cap;
};

static SelectLayout select_layout(int64_t m, int32_t k) {
  SelectLayout L{};
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  L.ntiles = (uint32_t)((m + kTile - 1) / kTile);
  // expected candidates per tile with the sample's oversampling (~1.6x, 2.5x budget)
  const double lam = (double)kTile * (double)k / (double)m * 2.5;
  const double want = lam + 6.0 * std::sqrt(lam) + 8.0;
  uint32_t s = 16;
  while (s < want && s < 1024) s <<= 1;
  L.slots = s;
  uint64_t ovf = (uint64_t)k * 4 + 65536;
  uint64_t ord = (uint64_t)k * 8 + 131072;
  if (ord > (uint64_t)m) ord = (uint64_t)m;
  if (ovf > (uint64_t)m) ovf = (uint64_t)m;
  L.ovf_cap = (uint32_t)ovf;
  L.ord_cap = (uint32_t)ord;
  size_t off = 0;
  L.ctl = off;
  off = al(off + sizeof(SelectCtl));
  L.sample_top = off;
  off = al(off + sizeof(uint32_t) * kSampleMaxChunks * kSampleTop);
  L.engine = off;
  off = al(off + sizeof(EngineWS));
  L.tile_info = off;
  off = al(off + sizeof(uint32_t) * L.ntiles);
  L.tile_ovf = off;
  off = al(off + sizeof(uint32_t) * L.ntiles);
  L.slot_idx = off;
  off = al(off + sizeof(int32_t) * (size_t)L.ntiles * L.slots);
  L.slot_val = off;
  off = al(off + sizeof(float) * (size_t)L.ntiles * L.slots);
  L.ovf_idx = off;
  off = al(off + sizeof(int32_t) * L.ovf_cap);
  L.ovf_val = off;
  off = al(off + sizeof(float) * L.ovf_cap);
  L.ord_idx = off;
  off = al(off + sizeof(int32_t) * L.ord_cap);
  L.ord_val = off;
  off = al(off + sizeof(float) * L.ord_cap);
  L.total = off;
  return L;
}

// ---------------------------------------------------------------------------
// 1. sampling pass: per-block top-kSampleTop keys (exact, no atomics)
// ---------------------------------------------------------------------------
// The threshold window must come from exact sample ORDER STATISTICS, not from
// histogram bin edges: an accumulated residual develops a flat-topped
// magnitude distribution (every entry grows until it is selected), where the
// top k all lie within ~0.1% of tau -- a bin edge would admit a large fraction
// of m as candidates.
struct SampleArgs {
  const float* res;
  const float* grad;
  uint32_t m;
  uint32_t stride;  // elements between chunk starts
  uint32_t* top;    // [nchunks][kSampleTop] block-local top keys (0-padded)
};

// The r1-th and r2-th largest of the keys held by the block (NT threads x PER
// keys each) in one bitwise binary search on counts (both counts packed in
// one word: fewer than 2^16 keys); r >= 1.  A rank beyond the number of
// nonzero keys yields 0.
template <int NT, int PER>
__device__ __forceinline__ uint2 block_rank_keys(const uint32_t (&keys)[PER], uint32_t r1, uint32_t r2,
                                                 uint32_t (&red)[2][NT / 32]) {
  static_assert(NT * PER < 65536, "packed 16-bit counts");
  uint32_t p1 = 0, p2 = 0;
#pragma unroll 1
  for (int bit = 30; bit >= 0; --bit) {
    const uint32_t c1 = p1 | (1u << bit), c2 = p2 | (1u << bit);
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) c += (keys[j] >= c1 ? 1u : 0u) + (keys[j] >= c2 ? 0x10000u : 0u);
    c = warp_sum(c);
    uint32_t* rb = red[bit & 1];  // double-buffered: one barrier per iteration
    if (lane_id() == 0) rb[warp_id()] = c;
    __syncthreads();
    uint32_t tot = lane_id() < (unsigned)(NT / 32) ? rb[lane_id()] : 0u;
    tot = warp_sum(tot);
    if ((tot & 0xFFFFu) >= r1) p1 = c1;
    if ((tot >> 16) >= r2) p2 = c2;
  }
  return make_uint2(p1, p2);
}

// r-th largest of the keys held by one warp (32 lanes x PER keys), bitwise
// binary search on warp-reduced counts; 0 if fewer than r nonzero keys.
template <int PER>
__device__ __forceinline__ uint32_t warp_rank_key(const uint32_t (&keys)[PER], uint32_t r) {
  uint32_t p = 0;
#pragma unroll 1
  for (int bit = 30; bit >= 0; --bit) {
    const uint32_t cand = p | (1u << bit);
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) c += keys[j] >= cand;
    if (warp_sum(c) >= r) p = cand;
  }
  return p;
}

// Write the warp's kSampleTop largest keys (all keys > th, then keys == th,
// order irrelevant, zero-padded) to out[0..kSampleTop).
template <int PER>
__device__ __forceinline__ void warp_emit_top(const uint32_t (&keys)[PER], uint32_t th, uint32_t* out) {
  const unsigned lane = lane_id();
  uint32_t n = 0;
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const bool f = pass == 0 ? keys[j] > th : (keys[j] == th && th > 0);
      const unsigned bal = __ballot_sync(kFull, f);
      const uint32_t pos = n + __popc(bal & lanemask_lt());
      if (f && pos < (uint32_t)kSampleTop) out[pos] = keys[j];
      n += __popc(bal);
    }
  }
  for (uint32_t p = n + lane; p < (uint32_t)kSampleTop; p += 32) out[p] = 0;
}

__global__ void __launch_bounds__(kSampleThreads) select_sample_kernel(SampleArgs a) {
  __shared__ uint32_t s_wtop[kSampleThreads / 32][kSampleTop];
  pdl_launch_dependents();  // the window kernel may launch (it waits for us)
  const uint64_t e0 = (uint64_t)blockIdx.x * a.stride + threadIdx.x * 4;
  float x[4];
  if (e0 + 4 <= a.m) {
    float4 g4 = ld_stream4(a.grad + e0);
    if (a.res) {
      const float4 r4 = ld_stream4(a.res + e0);
      g4.x = __fadd_rn(r4.x, g4.x);
      g4.y = __fadd_rn(r4.y, g4.y);
      g4.z = __fadd_rn(r4.z, g4.z);
      g4.w = __fadd_rn(r4.w, g4.w);
    }
    x[0] = g4.x;
    x[1] = g4.y;
    x[2] = g4.z;
    x[3] = g4.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t e = e0 + j;
      float v = 0.0f;
      if (e < a.m) {
        v = a.grad[e];
        if (a.res) v = __fadd_rn(a.res[e], v);
      }
      x[j] = v;
    }
  }
  uint32_t key[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t kk = key_of(x[j]);
    key[j] = kk < kInfKey ? kk : 0u;  // non-finite: ignored (K1 reports it)
  }
  // level 1: each warp's top-32 of its 128 keys (warp-only search, no barrier)
  const uint32_t wth = warp_rank_key<4>(key, kSampleTop);
  uint32_t* wtop = s_wtop[warp_id()];
  warp_emit_top<4>(key, wth, wtop);
  __syncthreads();
  // level 2: warp 0 takes the block's top-32 of the 8 x 32 warp winners
  if (warp_id() == 0) {
    uint32_t k2[kSampleThreads / 32];
#pragma unroll
    for (int w = 0; w < kSampleThreads / 32; ++w) k2[w] = s_wtop[w][lane_id()];
    const uint32_t bth = warp_rank_key<kSampleThreads / 32>(k2, kSampleTop);
    warp_emit_top<kSampleThreads / 32>(k2, bth, a.top + (size_t)blockIdx.x * kSampleTop);
  }
}

// ---------------------------------------------------------------------------
// 2. threshold window (one block): exact sample ranks r_lo / r_hi
// ---------------------------------------------------------------------------
constexpr int kWindowThreads = 512;  // x PER keys each, PER in {8, 16, 32, 64} by sample size

struct WindowArgs {
  uint32_t r_lo;         // sample rank (from top) whose key becomes lo
  uint32_t r_hi;         // sample rank whose key (+1) becomes hi
  uint32_t nkeys;        // nchunks * kSampleTop
  uint32_t force_exact;  // 1 -> lo = 0x7FFFFFFF (forces the dense fallback)
  SelectCtl* ctl;
  const uint32_t* top;
  EngineWS* ews;
};

template <int PER>
__global__ void __launch_bounds__(kWindowThreads) select_window_kernel(WindowArgs a) {
  __shared__ uint32_t red[2][kWindowThreads / 32];
  pdl_launch_dependents();  // the main pass may launch and start streaming its tiles
  pdl_wait();               // the sample tops are complete
  uint32_t key[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const uint32_t i = j * kWindowThreads + threadIdx.x;
    key[j] = i < a.nkeys ? __ldcg(a.top + i) : 0u;
  }
  const uint2 kk = block_rank_keys<kWindowThreads, PER>(key, a.r_lo, a.r_hi, red);
  const uint32_t klo = kk.x, khi = kk.y;
  if (threadIdx.x < kRounds) a.ews->gather_n[threadIdx.x] = 0;  // the finish engine's counters
  if (threadIdx.x == 0) {
    uint32_t lo = klo;  // 0 when the sample holds fewer than r_lo nonzero keys: take all
    uint32_t hi = khi >= lo ? khi + 1 : lo + 1;
    if (a.force_exact) {
      lo = 0x7FFFFFFFu;
      hi = 0x80000000u;
    }
    const uint64_t width = (uint64_t)hi - lo;
    const uint32_t shift = width <= (uint64_t)kBins ? 0u : ceil_log2_u64((width + kBins - 1) / kBins);
    SelectCtl* ctl = a.ctl;
    ctl->lo = lo;
    ctl->shift = shift;
    ctl->ovf_cursor = 0;
    ctl->overflow = 0;
    ctl->nonfinite = 0;
  }
}

// ---------------------------------------------------------------------------
// 3. main HBM pass
// ---------------------------------------------------------------------------
struct MainArgs {
  const float* res;  // nullable
  const float* grad;
  float* res_out;
  uint32_t m;
  uint32_t slots;
  uint32_t ovf_cap;
  SelectCtl* ctl;
  uint32_t* tile_info;
  uint32_t* tile_ovf;
  int32_t* slot_idx;
  float* slot_val;
  int32_t* ovf_idx;
  float* ovf_val;
  uint32_t* whist;  // engine round-0 histogram [kHistLen]
};

__global__ void __launch_bounds__(kMainThreads) select_main_kernel(MainArgs a) {
  __shared__ uint32_t s_wt[kMainVec * 8];  // per (vec, warp) candidate totals -> offsets
  __shared__ uint32_t s_total;
  __shared__ int32_t* s_didx;
  __shared__ float* s_dval;
  __shared__ uint32_t s_nonfinite;

  const uint32_t tile = blockIdx.x;
  const uint64_t tbase = (uint64_t)tile * kTile;
  const unsigned lane = lane_id(), w = warp_id();
  if (threadIdx.x == 0) s_nonfinite = 0;

  float v[kMainVec][4];
  const bool full = tbase + kTile <= a.m;
  if (full) {
    float4 gv[kMainVec], rv[kMainVec];
#pragma unroll
    for (int q = 0; q < kMainVec; ++q) {
      const uint64_t e = tbase + ((uint64_t)q * kMainThreads + threadIdx.x) * 4;
      gv[q] = ld_stream4(a.grad + e);
      if (a.res) rv[q] = ld_stream4(a.res + e);
    }
    // everything below consumes the window kernel's results (and may write
    // res_out = res in place, which the sample kernel reads): wait for it --
    // the loads above are already in flight (programmatic dependent launch)
    pdl_wait();
#pragma unroll
    for (int q = 0; q < kMainVec; ++q) {
      float4 x = gv[q];
      if (a.res) {
        x.x = __fadd_rn(rv[q].x, x.x);
        x.y = __fadd_rn(rv[q].y, x.y);
        x.z = __fadd_rn(rv[q].z, x.z);
        x.w = __fadd_rn(rv[q].w, x.w);
      }
      const uint64_t e = tbase + ((uint64_t)q * kMainThreads + threadIdx.x) * 4;
      st_stream4(a.res_out + e, x);
      v[q][0] = x.x;
      v[q][1] = x.y;
      v[q][2] = x.z;
      v[q][3] = x.w;
    }
  } else {
    pdl_wait();
#pragma unroll
    for (int q = 0; q < kMainVec; ++q)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t e = tbase + ((uint64_t)q * kMainThreads + threadIdx.x) * 4 + j;
        float x = 0.0f;
        if (e < a.m) {
          x = a.grad[e];
          if (a.res) x = __fadd_rn(a.res[e], x);
          a.res_out[e] = x;
        }
        v[q][j] = x;
      }
  }
  const uint32_t lo = __ldcg(&a.ctl->lo);  // issued after the tile loads: off the critical path
  const uint32_t shift = __ldcg(&a.ctl->shift);
  __syncthreads();  // s_nonfinite init visible

  // candidate flags, non-finite check, window histogram
  uint32_t flags = 0;  // bit q*4+j
  bool nonfinite = false;
#pragma unroll
  for (int q = 0; q < kMainVec; ++q)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t e = tbase + ((uint64_t)q * kMainThreads + threadIdx.x) * 4 + j;
      const uint32_t key = key_of(v[q][j]);
      const bool in = full || e < a.m;
      nonfinite |= in && key >= kInfKey;
      if (in && key >= lo) {
        flags |= 1u << (q * 4 + j);
        atomicAdd(a.whist + min((uint32_t)kBins, (key - lo) >> shift), 1u);
      }
    }
  if (__any_sync(kFull, nonfinite) && lane == 0) s_nonfinite = 1;

  // in-tile, index-ordered offsets: order is (q, warp, lane, j)
  uint32_t lane_pre[kMainVec];
#pragma unroll
  for (int q = 0; q < kMainVec; ++q) {
    uint32_t pre = 0, tot = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const unsigned bal = __ballot_sync(kFull, (flags >> (q * 4 + j)) & 1u);
      pre += __popc(bal & lanemask_lt());
      tot += __popc(bal);
    }
    lane_pre[q] = pre;
    if (lane == 0) s_wt[q * 8 + w] = tot;
  }
  __syncthreads();
  if (w == 0) {
    const uint32_t x = s_wt[lane];
    uint32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= (unsigned)o) incl += y;
    }
    s_wt[lane] = incl - x;
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    if (lane == 0) {
      s_total = total;
      uint32_t info = total;
      int32_t* didx = a.slot_idx + (size_t)tile * a.slots;
      float* dval = a.slot_val + (size_t)tile * a.slots;
      if (total > a.slots) {  // dense tile: reserve overflow space
        const uint32_t base = atomicAdd(&a.ctl->ovf_cursor, total);
        if (base + total > a.ovf_cap) {
          a.ctl->overflow = 1;
          didx = nullptr;
        } else {
          didx = a.ovf_idx + base;
          dval = a.ovf_val + base;
        }
        a.tile_ovf[tile] = base;
        info |= kOvfBit;
      }
      a.tile_info[tile] = info;
      s_didx = didx;
      s_dval = dval;
      if (s_nonfinite) a.ctl->nonfinite = 1;
    }
  }
  __syncthreads();
  int32_t* didx = s_didx;
  float* dval = s_dval;
  if (s_total == 0 || didx == nullptr) return;
#pragma unroll
  for (int q = 0; q < kMainVec; ++q) {
    uint32_t pos = s_wt[q * 8 + w] + lane_pre[q];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if ((flags >> (q * 4 + j)) & 1u) {
        didx[pos] = (int32_t)(tbase + ((uint64_t)q * kMainThreads + threadIdx.x) * 4 + j);
        dval[pos] = v[q][j];
        ++pos;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// 4. finish: per-block candidate slices in smem, exact engine / dense fallback
// ---------------------------------------------------------------------------
struct FinishArgs {
  float* res_out;
  uint32_t m;
  uint32_t k;
  uint32_t ntiles;
  uint32_t slots;
  uint32_t ord_cap;
  SelectCtl* ctl;
  EngineWS* ews;
  const uint32_t* tile_info;
  const uint32_t* tile_ovf;
  const int32_t* slot_idx;
  const float* slot_val;
  const int32_t* ovf_idx;
  const float* ovf_val;
  int32_t* ord_idx;  // global staging for a block whose slice exceeds kSliceCap
  float* ord_val;
  int32_t* sel_idx;
  float* sel_val;
  int32_t* d_count;
  uint32_t* d_status;
  int64_t* trace;  // optional phase stamps (block 0): [0] start [1] scanned [2] copied [3..6] engine
};

__device__ __forceinline__ void finish_stamp(const FinishArgs& a, int i) {
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[i] = (int64_t)t;
  }
}

__global__ void __launch_bounds__(kFinishThreads) select_finish_kernel(FinishArgs a) {
  __shared__ EngineSmem<kFinishThreads> sm;
  __shared__ int32_t s_idx[kSliceCap];
  __shared__ float s_val[kSliceCap];
  const unsigned G = gridDim.x, blk = blockIdx.x;
  if (__ldcg(&a.ctl->nonfinite)) {
    if (blk == 0) {
      for (int b = threadIdx.x; b < kHistLen; b += kFinishThreads) a.ews->hist[0][b] = 0;
      if (threadIdx.x == 0) atomicOr(a.d_status, GTK_DEV_NONFINITE);
    }
    return;
  }
  const Sink out{a.sel_idx, a.sel_val, a.d_count, a.res_out, true, a.trace ? a.trace + 3 : nullptr};
  finish_stamp(a, 0);

  // my tile range and its place in the global (index-ordered) candidate list
  const uint32_t per = (a.ntiles + G - 1) / G;
  const uint32_t t0 = min(a.ntiles, blk * per), t1 = min(a.ntiles, t0 + per);
  uint32_t before = 0, all = 0, own = 0;
  // tile_info is padded to a multiple of 4 with zeros: 128-bit loads
  const uint32_t n4 = (a.ntiles + 3) / 4;
#pragma unroll 4
  for (uint32_t t4 = threadIdx.x; t4 < n4; t4 += kFinishThreads) {
    const uint4 q = __ldcg(reinterpret_cast<const uint4*>(a.tile_info) + t4);
    const uint32_t c[4] = {q.x & ~kOvfBit, q.y & ~kOvfBit, q.z & ~kOvfBit, q.w & ~kOvfBit};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t t = 4 * t4 + j;
      all += c[j];
      before += t < t0 ? c[j] : 0u;
      own += (t >= t0 && t < t1) ? c[j] : 0u;
    }
  }
  before = block_sum<kFinishThreads>(before, sm.scan);
  own = block_sum<kFinishThreads>(own, sm.scan);
  const uint32_t C = block_sum<kFinishThreads>(all, sm.scan);
  const bool overflow = __ldcg(&a.ctl->overflow) != 0;
  finish_stamp(a, 1);
  if (!overflow && C >= a.k && C <= a.ord_cap) {
    // copy my tiles' candidates into my slice (smem if it fits)
    const bool in_smem = own <= (uint32_t)kSliceCap;
    int32_t* di = in_smem ? s_idx : a.ord_idx + before;
    float* dv = in_smem ? s_val : a.ord_val + before;
    uint32_t* s_dst = sm.keys;                   // per-tile destination (local)
    uint32_t* s_cnt = sm.hist;                   // per-tile info
    uint32_t* s_ovf = sm.hist + kFinishThreads;  // per-tile overflow base
    uint32_t run = 0;
    for (uint32_t tb = t0; tb < t1; tb += kFinishThreads) {
      const uint32_t t = tb + threadIdx.x;
      const uint32_t info = t < t1 ? __ldcg(a.tile_info + t) : 0u;
      uint32_t tot;
      const uint32_t pre = block_excl_scan<kFinishThreads>(info & ~kOvfBit, sm.scan, &tot);
      s_dst[threadIdx.x] = run + pre;
      s_cnt[threadIdx.x] = info;
      s_ovf[threadIdx.x] = (info & kOvfBit) ? __ldcg(a.tile_ovf + t) : 0u;
      __syncthreads();
      const uint32_t nt = min((uint32_t)kFinishThreads, t1 - tb);
      // entry-indexed gather: entry j of this chunk lives in tile q with
      // s_dst[q] - run <= j < s_dst[q+1] - run (binary search in smem)
#pragma unroll 4
      for (uint32_t j = threadIdx.x; j < tot; j += kFinishThreads) {
        const uint32_t jj = run + j;
        uint32_t lo = 0, hi = nt;  // last q with s_dst[q] <= jj
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (s_dst[mid] <= jj) lo = mid;
          else hi = mid;
        }
        const uint32_t inf = s_cnt[lo];
        if (inf & kOvfBit) continue;  // dense tiles are copied below
        const size_t src = (size_t)(tb + lo) * a.slots + (jj - s_dst[lo]);
        di[jj] = __ldcg(a.slot_idx + src);
        dv[jj] = __ldcg(a.slot_val + src);
      }
      for (uint32_t q = warp_id(); q < nt; q += kFinishThreads / 32) {  // dense tiles
        const uint32_t inf = s_cnt[q];
        if (!(inf & kOvfBit)) continue;
        const uint32_t cnt = inf & ~kOvfBit, ob = s_ovf[q], dst = s_dst[q];
        for (uint32_t e = lane_id(); e < cnt; e += 32) {
          di[dst + e] = __ldcg(a.ovf_idx + ob + e);
          dv[dst + e] = __ldcg(a.ovf_val + ob + e);
        }
      }
      run += tot;
      __syncthreads();
    }
    finish_stamp(a, 2);
    SliceSrc src{s_idx, s_val, a.ord_idx, a.ord_val, before, in_smem, false};
    if (engine_run<kFinishThreads>(src, before, before + own, a.k, false, __ldcg(&a.ctl->lo),
                                   __ldcg(&a.ctl->shift), a.ews->hist[0], false, a.ews, sm, out, G))
      return;
  }
  // exact dense fallback over acc (= res_out, untouched so far)
  grid_sync(&a.ews->bar, G);
  if (blk == 0) {
    for (int r = 0; r < kRounds; ++r)
      for (int b = threadIdx.x; b < kHistLen; b += kFinishThreads) a.ews->hist[r][b] = 0;
    if (threadIdx.x < kRounds) a.ews->gather_n[threadIdx.x] = 0;
    if (threadIdx.x == 0) atomicOr(a.d_status, GTK_DEV_FALLBACK);
  }
  grid_sync(&a.ews->bar, G);
  DenseSrc dsrc{a.res_out};
  uint32_t s0, s1;
  slice_of(a.m, G, blk, s0, s1);
  engine_run<kFinishThreads>(dsrc, s0, s1, a.k, false, 0u, 20u, nullptr, false, a.ews, sm, out, G);
}

}  // namespace gtk

using namespace gtk;

extern "C" int gtk_select_workspace_bytes(int64_t m, int32_t k, size_t* bytes) {
  if (!bytes || m < 1 || m >= (int64_t(1) << 31) || k < 1 || k > m) return GTK_EINVAL;
  *bytes = select_layout(m, k).total;
  return GTK_OK;
}

extern "C" int gtk_select(const float* res_in, const float* grad, float* res_out, int64_t m, int32_t k,
                          int32_t* sel_idx, float* sel_val, int32_t* d_count, uint32_t* d_status, void* ws,
                          size_t ws_bytes, int32_t flags, void* stream) {
  if (!grad || !res_out || !sel_idx || !sel_val || !d_count || !d_status || !ws) return GTK_EINVAL;
  if (m < 1 || m >= (int64_t(1) << 31) || k < 1 || k > m) return GTK_EINVAL;
  const SelectLayout L = select_layout(m, k);
  if (ws_bytes < L.total) return GTK_ENOMEM;
  const bool aligned = ((uintptr_t)grad % 16 == 0) && ((uintptr_t)res_out % 16 == 0) &&
                       (!res_in || (uintptr_t)res_in % 16 == 0);
  if (!aligned) return GTK_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  char* base = (char*)ws;
  SelectCtl* ctl = (SelectCtl*)(base + L.ctl);
  EngineWS* ews = (EngineWS*)(base + L.engine);
  uint32_t* stop = (uint32_t*)(base + L.sample_top);

  // sample plan: ~128 sampled elements expected above the k-th key, at most
  // kSampleMaxChunks chunks of 1024 (each keeps its top kSampleTop keys)
  const double mu_full = 128.0;
  const uint64_t chunks_all = (uint64_t)((m + kSampleChunk - 1) / kSampleChunk);
  uint64_t swant = (uint64_t)std::ceil(mu_full * (double)m / (double)k / kSampleChunk);
  if (swant < 1) swant = 1;
  uint32_t nchunks, stride, r_lo, r_hi;
  if (swant * 2 >= chunks_all && chunks_all <= (uint64_t)kSampleMaxChunks) {
    nchunks = (uint32_t)chunks_all;  // small problem: every element, exact rank k
    stride = kSampleChunk;
    r_lo = r_hi = (uint32_t)k;
  } else {
    nchunks = (uint32_t)(swant < (uint64_t)kSampleMaxChunks ? swant : (uint64_t)kSampleMaxChunks);
    stride = (uint32_t)((uint64_t)m / nchunks) & ~3u;
    if (stride < (uint32_t)kSampleChunk) stride = kSampleChunk;
    const double s = (double)nchunks * kSampleChunk;
    const double mu = (double)k * s / (double)m;
    const double sd = std::sqrt(mu);
    r_lo = (uint32_t)std::ceil(mu + 4.0 * sd + 4.0);
    const double rh = mu - 4.0 * sd - 4.0;
    r_hi = rh < 1.0 ? 1u : (uint32_t)rh;
  }
  ProfScope prof_all(kProfSelect, st);
  SampleArgs sa{res_in, grad, (uint32_t)m, stride, stop};
  select_sample_kernel<<<nchunks, kSampleThreads, 0, st>>>(sa);
  GTK_CHECK_LAUNCH();
  WindowArgs wa{r_lo, r_hi, nchunks * (uint32_t)kSampleTop, (uint32_t)((flags & GTK_SELECT_FORCE_EXACT) ? 1 : 0),
                ctl, stop, ews};
  {
    const uint32_t nk = wa.nkeys;
    auto* wk = nk <= 8 * kWindowThreads    ? select_window_kernel<8>
               : nk <= 16 * kWindowThreads ? select_window_kernel<16>
               : nk <= 32 * kWindowThreads ? select_window_kernel<32>
                                           : select_window_kernel<64>;
    GTK_CUDA(launch_pdl(wk, dim3(1), dim3(kWindowThreads), 0, st, wa));
  }
  GTK_CHECK_LAUNCH();

  MainArgs ma{res_in,
              grad,
              res_out,
              (uint32_t)m,
              L.slots,
              L.ovf_cap,
              ctl,
              (uint32_t*)(base + L.tile_info),
              (uint32_t*)(base + L.tile_ovf),
              (int32_t*)(base + L.slot_idx),
              (float*)(base + L.slot_val),
              (int32_t*)(base + L.ovf_idx),
              (float*)(base + L.ovf_val),
              ews->hist[0]};
  {
    ProfScope prof_main(kProfSelectMain, st);
    GTK_CUDA(launch_pdl(select_main_kernel, dim3(L.ntiles), dim3(kMainThreads), 0, st, ma));
    GTK_CHECK_LAUNCH();
  }

  FinishArgs fa{res_out,
                (uint32_t)m,
                (uint32_t)k,
                L.ntiles,
                L.slots,
                L.ord_cap,
                ctl,
                ews,
                (const uint32_t*)(base + L.tile_info),
                (const uint32_t*)(base + L.tile_ovf),
                (const int32_t*)(base + L.slot_idx),
                (const float*)(base + L.slot_val),
                (const int32_t*)(base + L.ovf_idx),
                (const float*)(base + L.ovf_val),
                (int32_t*)(base + L.ord_idx),
                (float*)(base + L.ord_val),
                sel_idx,
                sel_val,
                d_count,
                d_status,
                trace_buffer() ? trace_buffer() + 48 : nullptr};


  int G = coop_grid((const void*)select_finish_kernel, kFinishThreads, 0);
  if (G <= 0) return GTK_ECUDA;
  int want = (int)((L.ntiles + 39) / 40);  // ~40 tiles (~350 candidates) per block
  if ((int64_t)want * kSliceCap < (int64_t)k * 2) want = (int)(((int64_t)k * 2 + kSliceCap - 1) / kSliceCap);
  if (want < 8) want = 8;
  if ((uint32_t)want > L.ntiles) want = (int)L.ntiles;
  if (G > want) G = want;
  if (G > num_sms()) G = num_sms();
  if (G > kMaxBlocks) G = kMaxBlocks;
  void* args[] = {&fa};
  return coop_launch((const void*)select_finish_kernel, G, kFinishThreads, args, 0, st);
}
