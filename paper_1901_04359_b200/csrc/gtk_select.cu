// K1: fused residual-add + exact top-k select (reference optimizer.py:219-220,
// sparse.py:135-154).
//
// Four launches per call, no host synchronisation:
//   1. select_sample  : ~128/rho sampled elements of acc = res + g (evenly
//                       strided 4 KB chunks, one per block) into an 8192-bin
//                       histogram of the top key bits + a 256-bin exponent
//                       histogram.
//   2. select_window  : one block turns the sample histograms into a
//                       conservative key window [lo, hi) around the k-th key.
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
constexpr int kSampleBins = 8192;                            // key >> 18
constexpr int kSampleShift = 18;
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
  size_t ctl, sample_hist, engine, tile_info, tile_ovf, slot_idx, slot_val, ovf_idx, ovf_val, ord_idx, ord_val,
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
  L.sample_hist = off;
  off = al(off + sizeof(uint32_t) * (kSampleBins + 256));
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
// 1. sampling pass
// ---------------------------------------------------------------------------
struct SampleArgs {
  const float* res;
  const float* grad;
  uint32_t m;
  uint32_t stride;   // elements between chunk starts
  uint32_t* hist;    // [kSampleBins] fine, zero on entry (re-zeroed by the window kernel)
  uint32_t* coarse;  // [256] per-exponent sums, same protocol
};

__global__ void __launch_bounds__(kSampleThreads) select_sample_kernel(SampleArgs a) {
  // one 1024-element chunk per block: the per-element shared-memory atomics
  // (the cost of this kernel) are spread over ~1 block per SM
  __shared__ uint32_t sh[kSampleBins];
  static_assert(kSampleBins == 32 * kSampleThreads, "thread t owns exponent t's 32 fine bins");
  pdl_launch_dependents();  // the window kernel may launch (it waits for us)
  for (int b = threadIdx.x; b < kSampleBins; b += kSampleThreads) sh[b] = 0;
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
      float v = __int_as_float(0x7F800000);  // +inf: ignored below
      if (e < a.m) {
        v = a.grad[e];
        if (a.res) v = __fadd_rn(a.res[e], v);
      }
      x[j] = v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t key = key_of(x[j]);
    if (key < kInfKey) atomicAdd(&sh[key >> kSampleShift], 1u);
  }
  __syncthreads();
  // flush (fire-and-forget reductions): thread t owns exponent t's 32 fine bins
  uint32_t csum = 0;
#pragma unroll 8
  for (int j = 0; j < 32; ++j) {
    const int b = threadIdx.x * 32 + ((j + threadIdx.x) & 31);  // rotated: no bank conflicts
    const uint32_t v = sh[b];
    if (v) {
      atomicAdd(a.hist + b, v);
      csum += v;
    }
  }
  if (csum) atomicAdd(a.coarse + threadIdx.x, csum);
}

// ---------------------------------------------------------------------------
// 2. threshold window (one block)
// ---------------------------------------------------------------------------
struct WindowArgs {
  uint32_t r_lo;         // rank (from top) whose bin's LOWER edge becomes lo
  uint32_t r_hi;         // rank whose bin's UPPER edge bounds the window
  uint32_t force_exact;  // 1 -> lo = 0x7FFFFFFF (forces the dense fallback)
  SelectCtl* ctl;
  uint32_t* hist;
  uint32_t* coarse;
  EngineWS* ews;
};

__global__ void __launch_bounds__(kSampleThreads) select_window_kernel(WindowArgs a) {
  __shared__ uint32_t scan[kSampleThreads / 32 + 2];
  __shared__ uint32_t s_exp[2], s_above[2], s_bin[2];
  pdl_launch_dependents();  // the main pass may launch and start streaming its tiles
  pdl_wait();               // the sample histograms are complete
  const uint32_t ce = __ldcg(a.coarse + (kSampleThreads - 1 - threadIdx.x));  // descending exponent
  uint32_t tot;
  const uint32_t pre = block_excl_scan<kSampleThreads>(ce, scan, &tot);
  if (threadIdx.x == 0) {
    s_exp[0] = s_exp[1] = 0xFFFFFFFFu;
    s_bin[0] = s_bin[1] = 0xFFFFFFFFu;
  }
  __syncthreads();
  const uint32_t rk[2] = {a.r_lo, a.r_hi};
#pragma unroll
  for (int i = 0; i < 2; ++i)
    if (ce && pre < rk[i] && pre + ce >= rk[i]) {
      s_exp[i] = kSampleThreads - 1 - threadIdx.x;
      s_above[i] = pre;
    }
  __syncthreads();
  if (warp_id() < 2) {
    const int i = warp_id();
    const unsigned lane = lane_id();
    if (s_exp[i] != 0xFFFFFFFFu) {
      const uint32_t bin = s_exp[i] * 32 + 31 - lane;  // descending inside the exponent
      const uint32_t v = __ldcg(a.hist + bin);
      uint32_t incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= (unsigned)o) incl += y;
      }
      const uint32_t ex = s_above[i] + incl - v;
      if (v && ex < rk[i] && ex + v >= rk[i]) s_bin[i] = bin;
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kSampleBins; b += kSampleThreads) a.hist[b] = 0;
  a.coarse[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    uint32_t lo = s_bin[0] == 0xFFFFFFFFu ? 0u : (s_bin[0] << kSampleShift);  // too few samples: all
    uint32_t hi;
    if (s_bin[1] == 0xFFFFFFFFu) {
      hi = 0x80000000u;
    } else {
      hi = (s_bin[1] + 1) << kSampleShift;
      if (hi <= lo) hi = lo + (1u << kSampleShift);
    }
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
  if (threadIdx.x < kRounds) {  // the finish engine's gather counters (read only after its barrier)
    EngineWS* ews = a.ews;
    ews->gather_n[threadIdx.x] = 0;
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
};

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
  const Sink out{a.sel_idx, a.sel_val, a.d_count, a.res_out, true};

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
  uint32_t* shist = (uint32_t*)(base + L.sample_hist);

  // sample plan: expect ~128 sampled elements above the k-th key
  const double mu_full = 128.0;
  const uint64_t s_target = (uint64_t)std::ceil(mu_full * (double)m / (double)k);
  uint32_t nchunks, stride, r_lo, r_hi;
  if (s_target * 2 >= (uint64_t)m) {  // small problem: scan everything, exact window
    nchunks = (uint32_t)((m + kSampleChunk - 1) / kSampleChunk);
    stride = kSampleChunk;
    r_lo = (uint32_t)k;
    r_hi = (uint32_t)k;
  } else {
    nchunks = (uint32_t)((s_target + kSampleChunk - 1) / kSampleChunk);
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
  SampleArgs sa{res_in, grad, (uint32_t)m, stride, shist, shist + kSampleBins};
  select_sample_kernel<<<nchunks, kSampleThreads, 0, st>>>(sa);
  GTK_CHECK_LAUNCH();
  WindowArgs wa{r_lo, r_hi, (uint32_t)((flags & GTK_SELECT_FORCE_EXACT) ? 1 : 0), ctl, shist,
                shist + kSampleBins, ews};
  GTK_CUDA(launch_pdl(select_window_kernel, dim3(1), dim3(kSampleThreads), 0, st, wa));
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
                d_status};


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
