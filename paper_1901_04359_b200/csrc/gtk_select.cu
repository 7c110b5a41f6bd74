// K1: fused residual-add + exact top-k select (reference optimizer.py:219-220,
// sparse.py:135-154).
//
// Three launches per call (PDL-chained), no host synchronisation:
//   1. select_sample  : ~128/rho sampled elements of acc = res + g (evenly
//                       strided 4 KB chunks, one per block); each block keeps
//                       its exact top-32 keys (histogram levels in shared
//                       memory); the last block to finish finds the exact
//                       sample order statistics around rank k*s/m (+-4 sigma)
//                       -> key window [lo, hi).
//   2. select_main    : THE HBM pass.  One 4096-element tile per block, no
//                       inter-block dependency: 128-bit streaming loads of res
//                       and g, acc = __fadd_rn(res, g) streamed to res_out, key
//                       test against lo, warp-ballot compaction of the tile's
//                       candidates (index order inside the tile) into the
//                       tile's own slot row -- or, for a dense tile, into an
//                       atomically reserved overflow region -- and a 2049-bin
//                       histogram of candidate keys over the window.
//   3. select_finish  : cooperative.  Block b owns a contiguous range of tiles;
//                       it copies their candidates (already index-ordered) into
//                       shared memory -- its slice of the global candidate
//                       list -- and the exact engine (gtk_engine.cuh) keeps the
//                       k winners, writes them in index order and zeroes their
//                       residual slots.  If the window missed (fewer than k
//                       candidates, or too many) the engine runs over the dense
//                       acc instead: the exact fallback.
#include <cuda_runtime.h>

#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "gtk_engine.cuh"
#include "gtk_internal.h"

namespace gtk {

constexpr int kMainThreads = 256;
constexpr int kMainVec = 4;                                  // float4 per thread per array
constexpr int kTile = kMainThreads * kMainVec * 4;          // 4096 elements
constexpr int kMainTilesPerBlock = 2;                      // tiles loaded up front by one main-pass block
// main pass loads: 0 = float4 register loads (default), 1 = bulk copies (TMA)
// of the block's tiles into 64 KB of shared memory on one mbarrier.  The bulk
// form frees ~24 registers per thread but measured slower on the same box
// (profiles/r2_main_tma_ab.txt: main pass alone 53.0 -> 54.2 us, N = 1 step
// 61.9 -> 65.1 us, N = 2 75.1 -> 79.4): kept as an A/B switch
#ifndef GTK_MAIN_TMA
#define GTK_MAIN_TMA 0
#endif
constexpr size_t kMainStageBytes = GTK_MAIN_TMA ? (size_t)kMainTilesPerBlock * 2 * kTile * sizeof(float) : 0;
constexpr int kMainDenseHist = 48;                          // candidates per tile above which the histogram goes via smem
constexpr int kSampleThreads = 1024;
constexpr int kSampleChunk = kSampleThreads;                // 1024 elements per chunk (one per thread)
constexpr int kSampleTop = 32;                               // top keys kept per sample block
constexpr int kSampleMaxChunks = 1024;                       // sample blocks (window holds 32K keys)
#ifndef GTK_FINISH_THREADS
#define GTK_FINISH_THREADS 512
#endif
constexpr int kFinishThreads = GTK_FINISH_THREADS;
constexpr int kSliceCap = 3072;                              // candidates staged per finish block (minimum)
constexpr int kSliceCapMax = 20480;                          // ... up to 160 KB of dynamic smem at large k
constexpr size_t kFinishDynSmemMax = 192 * 1024;             // slice + (deferred) fix list
constexpr uint32_t kOvfBit = 0x80000000u;
constexpr uint32_t kMinWindowLevel = 2;  // carried-window margin: from k (1 + 2^2 / 2) = 3k candidates
constexpr uint32_t kMaxWindowLevel = 4;  // ... up to k (1 + 2^4 / 2) = 9k

constexpr uint32_t kCtlPendingViolation = 2u;
struct SelectCtl {
  uint32_t lo;
  uint32_t shift;
  uint32_t ovf_cursor;
  uint32_t overflow;
  uint32_t nonfinite;  // 1: non-finite input (main pass); kCtlPendingViolation (sample kernel)
  uint32_t sample_done;  // sample-block ticket (atomicInc, wraps to 0 per launch)
  uint32_t pad[10];
};

struct SelectLayout {
  size_t ctl, sample_top, group_cnt, blk_ofs, engine, tile_info, tile_ovf, slot_idx, slot_val, ovf_idx, ovf_val,
      ord_idx, ord_val, total;
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
  // generous: a carried window (gtk_select_windowed) admits ~3k-9k keys, tens
  // of k while a residual builds up; memory is cheap next to a dense fallback
  uint64_t ovf = (uint64_t)k * 64 + 262144;
  uint64_t ord = (uint64_t)k * 64 + 262144;
  if (ord > (uint64_t)m) ord = (uint64_t)m;
  if (ovf > (uint64_t)m) ovf = (uint64_t)m;
  L.ovf_cap = (uint32_t)ovf;
  L.ord_cap = (uint32_t)ord;
  size_t off = 0;
  L.ctl = off;
  off = al(off + sizeof(SelectCtl));
  L.sample_top = off;
  off = al(off + sizeof(uint32_t) * kSampleMaxChunks * kSampleTop);
  L.group_cnt = off;
  off = al(off + sizeof(uint32_t) * kMaxBlocks);
  L.blk_ofs = off;  // [0] = G of the finish that wrote [1 + b] = block b's first output position (0: none)
  off = al(off + sizeof(uint32_t) * (kMaxBlocks + 1));
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
// 1. sampling pass + threshold window (one launch)
// ---------------------------------------------------------------------------
// The threshold window must come from exact sample ORDER STATISTICS, not from
// histogram bin edges: an accumulated residual develops a flat-topped
// magnitude distribution (every entry grows until it is selected), where the
// top k all lie within ~0.1% of tau -- a bin edge would admit a large fraction
// of m as candidates.
//
// Each block keeps the exact top-kSampleTop keys of its 1024-element chunk;
// the last block to finish (ticket counter) takes the exact order statistics
// r_lo / r_hi of the union and publishes the window [lo, hi).

// ---- exact order statistics by histogram levels ---------------------------
// Three levels over the 31-bit key: bits 30..19 (4096 bins), 18..7 (4096
// bins), 6..0 (128 bins).  Each level histograms the keys that share the
// prefix resolved so far (plain shared atomics: a 12-bit digit spreads the
// keys), one block scan over the bins (both statistics' counts packed in one
// word) picks the digit.  Key 0 is "absent" (padding, zeros).
constexpr int kLvlBins = 4096;
struct LevelSmem {
  uint32_t hist[2][kLvlBins];  // per statistic; [0] alone while the prefixes agree
  uint32_t scan[kSampleThreads / 32 + 1];
  uint32_t pre[2];  // resolved key prefix per statistic
  uint32_t rem[2];  // rank still to find inside the prefix (0: fewer keys than the rank)
};

__device__ __forceinline__ void level_geom(int lvl, int& shift, uint32_t& mask, int& pshift) {
  shift = lvl == 0 ? 19 : (lvl == 1 ? 7 : 0);
  mask = lvl == 2 ? 0x7Fu : 0xFFFu;
  pshift = lvl == 0 ? 31 : (lvl == 1 ? 19 : 7);
}

// out[s] = rank[s]-th largest nonzero key (rank >= 1) of the multiset the
// block holds, 0 if there are fewer; for_each(f) calls f(key) for every key
// of this thread.  ghist0 (nullable): level 0 already histogrammed in global
// memory (read and re-zeroed here).  Precondition: sm.hist zero; kept zero.
template <int NS, class ForEach>
__device__ __forceinline__ void block_hist_select(const ForEach& for_each, const uint32_t (&rank)[NS],
                                                  uint32_t (&out)[NS], LevelSmem& sm, uint32_t* ghist0,
                                                  int64_t* tr = nullptr) {
  auto stamp = [&](int i) {
    if (tr && threadIdx.x == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      tr[i] = (int64_t)t;
    }
  };
  static_assert(NS == 1 || NS == 2, "one or two statistics");
  constexpr int NT = kSampleThreads;
  constexpr int PER = kLvlBins / NT;  // bins per thread in the scan
  static_assert(PER == 4, "scan layout");
  if (threadIdx.x < NS) {
    sm.pre[threadIdx.x] = 0;
    sm.rem[threadIdx.x] = rank[threadIdx.x];
  }
  __syncthreads();
#pragma unroll 1
  for (int lvl = 0; lvl < 3; ++lvl) {
    int shift, pshift;
    uint32_t mask;
    level_geom(lvl, shift, mask, pshift);
    uint32_t pre[NS], rem[NS];
    bool live[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      pre[s] = sm.pre[s];
      rem[s] = sm.rem[s];
      live[s] = rem[s] != 0;
    }
    const bool shared = NS == 1 || (live[0] && live[NS - 1] && pre[0] == pre[NS - 1]) || !live[NS - 1];
    const bool from_global = lvl == 0 && ghist0 != nullptr;
    if (!from_global) {
      for_each([&](uint32_t key) {
        if (key == 0) return;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          if (s > 0 && shared) break;
          const int ss = shared ? 0 : s;
          const bool lv = shared ? live[0] || live[NS - 1] : live[s];
          const uint32_t p = shared ? (live[0] ? pre[0] : pre[NS - 1]) : pre[s];
          if (lv && (lvl == 0 || (key >> pshift) == (p >> pshift))) atomicAdd(&sm.hist[ss][(key >> shift) & mask], 1u);
        }
      });
      __syncthreads();
    }
    stamp(2 * lvl);
    // thread t owns bins nb-4(t+1) .. nb-4t-1, read top-down
    const int nb = (int)mask + 1;
    const int b0 = nb - PER * ((int)threadIdx.x + 1);
    uint32_t c[PER];  // packed: low 16 bits hist[0], high 16 bits hist[1]
    uint32_t sum = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int b = b0 + (PER - 1 - j);
      uint32_t v = 0;
      if (b >= 0) {
        if (from_global) {
          v = __ldcg(ghist0 + b);
          ghist0[b] = 0u;
        } else {
          v = sm.hist[0][b];
          sm.hist[0][b] = 0u;
          if (!shared) {
            v |= sm.hist[NS - 1][b] << 16;
            sm.hist[NS - 1][b] = 0u;
          }
        }
      }
      c[j] = v;
      sum += v;
    }
    uint32_t tot;
    const uint32_t above = block_excl_scan<NT>(sum, sm.scan, &tot);
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (!live[s]) continue;
      const int sh = (shared || s == 0) ? 0 : 16;
      const uint32_t m16 = shared ? 0xFFFFFFFFu : 0xFFFFu;
      const uint32_t r = rem[s];
      const uint32_t my_above = (above >> sh) & m16, my_sum = (sum >> sh) & m16, total = (tot >> sh) & m16;
      if (total < r) {
        if (threadIdx.x == 0) sm.rem[s] = 0;
      } else if (my_above < r && my_above + my_sum >= r) {
        uint32_t acc = my_above;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const uint32_t cj = (c[j] >> sh) & m16;
          if (acc + cj >= r) {
            const uint32_t digit = (uint32_t)(b0 + (PER - 1 - j));
            sm.pre[s] = pre[s] | (digit << shift);
            sm.rem[s] = r - acc;
            break;
          }
          acc += cj;
        }
      }
    }
    __syncthreads();
    stamp(2 * lvl + 1);
  }
#pragma unroll
  for (int s = 0; s < NS; ++s) out[s] = sm.rem[s] ? sm.pre[s] : 0u;
}

struct SampleArgs {
  const float* res;
  const float* grad;
  uint32_t m;
  uint32_t stride;       // elements between chunk starts
  uint32_t nchunks;      // blocks
  uint32_t r_lo;         // sample rank (from top) whose key becomes lo
  uint32_t r_hi;         // sample rank whose key (+1) becomes hi
  uint32_t force_exact;  // 1 -> lo = 0x7FFFFFFF (forces the dense fallback)
  uint32_t* top;         // [nchunks][kSampleTop] block-local top keys (0-padded)
  const uint32_t* window; // nullable: {valid | level << 8, lo, shift, k, tau} left by the previous call
  uint32_t k;
  SelectCtl* ctl;
  EngineWS* ews;
  uint32_t* group_cnt;  // [kMaxBlocks] per-finish-block candidate counts, zeroed here
  int64_t* trace;       // optional stamps: [0..3] block 0 phases, [4..6] last block phases
};

__device__ __forceinline__ void sample_stamp(const SampleArgs& a, int i, bool who) {
  if (a.trace && who && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[i] = (int64_t)t;
  }
}

// a plain (unchained) select of a residual whose winners a chained call left
// pending (include/gtopk_b200.h: settle first): the finish fails the call with
// GTK_DEV_PENDING (the main pass never reads the record: any dependent load
// there measured +9 us per pass)
__device__ __forceinline__ uint32_t pending_violation(const SampleArgs& a) {
  return (a.window && a.res && (__ldcg(a.window) & kRecPending)) ? kCtlPendingViolation : 0u;
}

__global__ void __launch_bounds__(kSampleThreads) select_sample_kernel(SampleArgs a) {
  __shared__ LevelSmem sm;
  __shared__ uint32_t s_n, s_last;
  // the previous kernel (K3 of the last step) writes res: wait for it before
  // reading, and only then let the main pass launch (its early loads read res)
  pdl_wait();
  pdl_launch_dependents();
  sample_stamp(a, 0, blockIdx.x == 0);
  if (a.window && !a.force_exact && (__ldcg(a.window) & 1u) && __ldcg(a.window + 3) == a.k) {
    // the previous call of this parameter measured the window: no sampling
    if (blockIdx.x == 0) {
      for (int i = threadIdx.x; i < kMaxBlocks; i += kSampleThreads) a.group_cnt[i] = 0u;
      if (threadIdx.x < kRounds) a.ews->gather_n[threadIdx.x] = 0;
      if (threadIdx.x == 0) {
        SelectCtl* ctl = a.ctl;
        ctl->lo = __ldcg(a.window + 1);
        ctl->shift = __ldcg(a.window + 2);
        ctl->ovf_cursor = 0;
        ctl->overflow = 0;
        ctl->nonfinite = pending_violation(a);
      }
    }
    return;
  }
  sample_stamp(a, 0, blockIdx.x == 0);
  {
    uint4* h = reinterpret_cast<uint4*>(&sm.hist[0][0]);
    for (int i = threadIdx.x; i < 2 * kLvlBins / 4; i += kSampleThreads) h[i] = make_uint4(0, 0, 0, 0);
  }
  if (threadIdx.x == 0) s_n = 0;
  const uint64_t e = (uint64_t)blockIdx.x * a.stride + threadIdx.x;
  uint32_t key = 0;
  if (e < a.m) {
    float x = __ldcs(a.grad + e);
    if (a.res) x = __fadd_rn(__ldcs(a.res + e), x);
    const uint32_t kk = key_of(x);
    key = kk < kInfKey ? kk : 0u;  // non-finite: ignored (K1 reports it)
  }
  sample_stamp(a, 1, blockIdx.x == 0);
  // the chunk's kSampleTop-th key, then its top keys: > th first, == th to the cap
  const uint32_t rk[1] = {(uint32_t)kSampleTop};
  uint32_t th[1];
  block_hist_select<1>([&](auto&& f) { f(key); }, rk, th, sm, nullptr,
                       (a.trace && blockIdx.x == 0) ? a.trace + 8 : nullptr);
  sample_stamp(a, 2, blockIdx.x == 0);
  uint32_t* out = a.top + (size_t)blockIdx.x * kSampleTop;
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
    const bool f = key != 0 && (pass == 0 ? key > th[0] : key == th[0]);
    const unsigned bal = __ballot_sync(kFull, f);
    uint32_t base = 0;
    if (lane_id() == 0 && bal) base = atomicAdd(&s_n, (uint32_t)__popc(bal));
    base = __shfl_sync(kFull, base, 0);
    const uint32_t pos = base + __popc(bal & lanemask_lt());
    if (f && pos < (uint32_t)kSampleTop) out[pos] = key;
    __syncthreads();
  }
  if (threadIdx.x < (unsigned)kSampleTop && threadIdx.x >= s_n) out[threadIdx.x] = 0u;

  // ticket: the last block to arrive computes the window (the barrier orders
  // the block's writes before thread 0's acq_rel ticket; atom.inc wraps the
  // counter back to 0, so every complete launch leaves it clean)
  __syncthreads();
  if (threadIdx.x == 0) s_last = atom_inc_acq_rel_gpu(&a.ctl->sample_done, a.nchunks - 1) == a.nchunks - 1;
  __syncthreads();
  sample_stamp(a, 3, blockIdx.x == 0);
  if (!s_last) return;
  sample_stamp(a, 4, true);
  const uint32_t nkeys = a.nchunks * kSampleTop;
  const uint32_t rk2[2] = {a.r_lo, a.r_hi};
  uint32_t kk[2];
  constexpr int kRegKeys = 4;
  if (nkeys <= (uint32_t)(kSampleThreads * kRegKeys)) {
    uint32_t k2[kRegKeys];
#pragma unroll
    for (int j = 0; j < kRegKeys; ++j) {
      const uint32_t i = j * kSampleThreads + threadIdx.x;
      k2[j] = i < nkeys ? __ldcg(a.top + i) : 0u;
    }
    sample_stamp(a, 5, true);
    block_hist_select<2>(
        [&](auto&& f) {
#pragma unroll
          for (int j = 0; j < kRegKeys; ++j) f(k2[j]);
        },
        rk2, kk, sm, nullptr, a.trace ? a.trace + 16 : nullptr);
  } else {  // large samples: re-read the keys from L2 per level
    block_hist_select<2>(
        [&](auto&& f) {
#pragma unroll 4
          for (uint32_t i = threadIdx.x; i < nkeys; i += kSampleThreads) f(__ldcg(a.top + i));
        },
        rk2, kk, sm, nullptr);
  }
  sample_stamp(a, 6, true);
  if (threadIdx.x < kRounds) a.ews->gather_n[threadIdx.x] = 0;  // the finish engine's counters
  for (int i = threadIdx.x; i < kMaxBlocks; i += kSampleThreads) a.group_cnt[i] = 0u;
  if (threadIdx.x == 0) {
    uint32_t lo = kk[0];  // 0 when the sample holds fewer than r_lo nonzero keys: take all
    uint32_t hi = kk[1] >= lo ? kk[1] + 1 : lo + 1;
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
    ctl->nonfinite = pending_violation(a);
  }
}

// ---------------------------------------------------------------------------
// 2. main HBM pass
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
  uint32_t* whist;      // engine round-0 histogram [kHistLen]
  uint32_t* group_cnt;  // candidates per finish block (tiles_per_group tiles each)
  uint32_t tiles_per_group;
  uint32_t n2;  // blocks [0, n2) take two tiles, the rest one (the last wave is short)
  int64_t* trace = nullptr;  // optional timeline stamps: [0] block 0 start, [1] last block end (max)
  // key-window record (nullable): its pending-winner predicate (a chained
  // select left the winners of res in place) is applied to res on the fly;
  // chained calls (chain = 1) also take the window from it -- there is no
  // sampling kernel -- and reset the engine's gather counters
  const uint32_t* window = nullptr;
  uint32_t k = 0;
  uint32_t chain = 0;
  uint32_t force_exact = 0;
  uint32_t* gather_n = nullptr;
};

// res with a chained select's pending winners zeroed: the winner predicate of
// the previous call's exact top-k (gtk_engine.cuh, Sink::pend_rec)
__device__ __forceinline__ float settle_res(float r, uint64_t i, uint32_t ptau, uint32_t pcut) {
  const uint32_t kr = key_of(r);
  return (kr > ptau || (kr == ptau && i <= (uint64_t)pcut)) ? 0.0f : r;
}

// v[b >> 2][b & 3] without a dynamically indexed (local-memory) array
__device__ __forceinline__ float pick(const float (&v)[kMainVec][4], int b) {
  float x = v[0][0];
#pragma unroll
  for (int i = 1; i < kMainVec * 4; ++i) x = b == i ? v[i >> 2][i & 3] : x;
  return x;
}

// Everything after the loads for one tile whose acc values this thread holds
// (v[q][j] is element (q * 256 + tid) * 4 + j): candidate flags, index-ordered
// compaction into the tile's slot row (or the overflow region for a dense
// tile) and the window histogram.  One block barrier (three for a dense tile);
// the shared scratch alternates with `par` between a block's tiles.
__device__ __forceinline__ bool main_tile(const MainArgs& a, uint32_t tile, const float (&v)[kMainVec][4], bool full,
                                          uint32_t lo, uint32_t shift, int par, uint32_t (&s_wt)[2][16],
                                          int32_t* (&s_didx)[2], float* (&s_dval)[2], uint32_t* s_hist) {
  const uint64_t tbase = (uint64_t)tile * kTile;
  const unsigned lane = lane_id(), w = warp_id();
  // candidate flags (bit q*4+j) and the non-finite check
  uint32_t flags = 0;
  bool nonfinite = false;
#pragma unroll
  for (int q = 0; q < kMainVec; ++q)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t e = tbase + ((uint64_t)q * kMainThreads + threadIdx.x) * 4 + j;
      const uint32_t key = key_of(v[q][j]);
      const bool in = full || e < a.m;
      nonfinite |= in && key >= kInfKey;
      if (in && key >= lo) flags |= 1u << (q * 4 + j);
    }
  if (__any_sync(kFull, nonfinite) && lane == 0) atomicOr(&a.ctl->nonfinite, 1u);

  // index-ordered in-tile offsets, order (q, warp, lane, j): per-lane counts of
  // the four q segments packed two per word (16-bit fields: a warp's segment
  // holds <= 128, a tile's <= 1024), one warp scan per word
  const uint32_t c01 = __popc(flags & 0xFu) | (__popc(flags & 0xF0u) << 16);
  const uint32_t c23 = __popc(flags & 0xF00u) | (__popc(flags & 0xF000u) << 16);
  uint32_t i01 = c01, i23 = c23;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y01 = __shfl_up_sync(kFull, i01, o), y23 = __shfl_up_sync(kFull, i23, o);
    if (lane >= (unsigned)o) {
      i01 += y01;
      i23 += y23;
    }
  }
  if (lane == 31) {
    s_wt[par][2 * w] = i01;  // warp totals per q
    s_wt[par][2 * w + 1] = i23;
  }
  __syncthreads();
  // every warp derives its segment bases from the 8 warps' totals: no second barrier
  uint32_t before01 = 0, before23 = 0, all01 = 0, all23 = 0;
#pragma unroll
  for (int ww = 0; ww < 8; ++ww) {
    const uint32_t t01 = s_wt[par][2 * ww], t23 = s_wt[par][2 * ww + 1];
    if (ww < (int)w) {
      before01 += t01;
      before23 += t23;
    }
    all01 += t01;
    all23 += t23;
  }
  const uint32_t T0 = all01 & 0xFFFFu, T1 = all01 >> 16, T2 = all23 & 0xFFFFu, T3 = all23 >> 16;
  const uint32_t total = T0 + T1 + T2 + T3;
  // base of (q, this lane): segment start + earlier warps + earlier lanes
  const uint32_t e01 = i01 - c01, e23 = i23 - c23;
  const uint32_t base[kMainVec] = {(before01 & 0xFFFFu) + (e01 & 0xFFFFu),
                                   T0 + (before01 >> 16) + (e01 >> 16),
                                   T0 + T1 + (before23 & 0xFFFFu) + (e23 & 0xFFFFu),
                                   T0 + T1 + T2 + (before23 >> 16) + (e23 >> 16)};
  if (total == 0) {
    if (threadIdx.x == 0) a.tile_info[tile] = 0u;
    return false;
  }
  if (threadIdx.x == 0) atomicAdd(a.group_cnt + tile / a.tiles_per_group, total);
  int32_t* didx = a.slot_idx + (size_t)tile * a.slots;
  float* dval = a.slot_val + (size_t)tile * a.slots;
  const bool dense = total > a.slots;
  if (dense) {  // reserve overflow space (uniform branch)
    if (threadIdx.x == 0) {
      const uint32_t b = atomicAdd(&a.ctl->ovf_cursor, total);
      if (b + total > a.ovf_cap) {
        a.ctl->overflow = 1u;
        s_didx[par] = nullptr;
      } else {
        s_didx[par] = a.ovf_idx + b;
        s_dval[par] = a.ovf_val + b;
      }
      a.tile_ovf[tile] = b;
    }
    __syncthreads();
    didx = s_didx[par];
    dval = s_dval[par];
  }
  if (threadIdx.x == 0) a.tile_info[tile] = total | (dense ? kOvfBit : 0u);
  // my candidates (set bits only), and -- for a sparse tile -- their histogram
  // bins straight to the global window histogram
  const bool hist_direct = total <= (uint32_t)kMainDenseHist;
  for (uint32_t f = flags; f; f &= f - 1) {
    const int b = __ffs(f) - 1;
    const int q = b >> 2, j = b & 3;
    const float x = pick(v, b);
    if (didx) {
      const uint32_t bq = q == 0 ? base[0] : q == 1 ? base[1] : q == 2 ? base[2] : base[3];
      const uint32_t pos = bq + __popc(flags & ((1u << b) - 1u) & (0xFu << (4 * q)));
      GTK_DCHECK(pos < total && (dense || pos < a.slots));
      didx[pos] = (int32_t)(tbase + ((uint64_t)q * kMainThreads + threadIdx.x) * 4 + j);
      dval[pos] = x;
    }
    if (hist_direct) atomicAdd(a.whist + min((uint32_t)kBins, (key_of(x) - lo) >> shift), 1u);
  }
  if (!hist_direct) {
    // dense tile (large k, or a wide window while a residual builds up): the
    // block's shared histogram (cleared at block start, flushed once at block
    // end), so a hot bin costs one global atomic per block
    for (uint32_t f = flags; f; f &= f - 1) {
      const int b = __ffs(f) - 1;
      atomicAdd(&s_hist[min((uint32_t)kBins, (key_of(pick(v, b)) - lo) >> shift)], 1u);
    }
    return true;
  }
  return false;
}


// kMode: kMainPlain reads nothing but the sample kernel's window words after
// griddepcontrol.wait (every dependent load there delays the whole pass: up
// to +9 us measured); kMainChain (GTK_SELECT_CHAIN) takes the window from the
// record and zeroes the previous call's pending winners on the fly;
// kMainDefer (gtk_select_update_deferred) is released by the previous call's
// finish as soon as that finish has corrected the winners before it, and
// never waits for the rest of it (the finish after this pass corrects this
// pass's view of the previous winners; the window comes from the record of
// the call before the previous one) -- only the last block waits for the
// previous finish before exiting, so the grid's completion still orders
// everything after it behind that finish.
constexpr int kMainPlain = 0, kMainChain = 1, kMainDefer = 2;
template <int kMode>
__global__ void __launch_bounds__(kMainThreads, 3) select_main_kernel(MainArgs a) {
  __shared__ uint32_t s_wt[2][16];  // per warp: packed candidate totals of the q segments
  __shared__ int32_t* s_didx[2];
  __shared__ float* s_dval[2];
  __shared__ uint32_t s_hist[kHistLen];  // dense tiles only
  pdl_launch_dependents();  // the finish grid may become resident as our last wave drains

  // all of this block's tiles are loaded before any is processed: more bytes
  // in flight per resident block
  // blocks [0, n2) take two tiles; the last ~one wave of blocks takes one
  // tile each, so the grid's drain (blocks running alone on a few SMs) is short
  static_assert(kMainTilesPerBlock == 2, "two-tile / one-tile schedule");
  const uint32_t blk = blockIdx.x;
  constexpr bool kChain = kMode == kMainChain;
  constexpr bool kRecord = kMode != kMainPlain;
  if (a.trace && blk == 0 && threadIdx.x == 0) a.trace[0] = (int64_t)globaltimer_ns();
  const uint32_t t0 = blk < a.n2 ? 2 * blk : a.n2 + blk;
  const uint32_t ntile = blk < a.n2 ? 2u : 1u;
#if GTK_MAIN_TMA
  // the full tiles' gradient and residual by the bulk-copy engine into shared
  // memory (64 KB per block in flight without a register each: a block that
  // shares its SM with a finish or exchange block still streams at depth),
  // one mbarrier for all of them
  extern __shared__ __align__(128) float4 s_stage[];  // [tile][grad | res][kTile / 4]
  __shared__ __align__(8) uint64_t s_mbar;
  if (threadIdx.x == 0) {
    mbar_init(&s_mbar, 1);
    uint32_t bytes = 0;
    for (uint32_t u = 0; u < ntile; ++u)
      if ((uint64_t)(t0 + u + 1) * kTile <= a.m) bytes += (a.res ? 2u : 1u) * kTile * 4u;
    mbar_arrive_expect_tx(&s_mbar, bytes);
    for (uint32_t u = 0; u < ntile; ++u) {
      const uint64_t tbase = (uint64_t)(t0 + u) * kTile;
      if (tbase + kTile > a.m) break;
      bulk_g2s_stream(s_stage + (2 * u) * (kTile / 4), a.grad + tbase, kTile * 4u, &s_mbar);
      if (a.res) bulk_g2s_stream(s_stage + (2 * u + 1) * (kTile / 4), a.res + tbase, kTile * 4u, &s_mbar);
    }
  }
#else
  float4 gv[kMainTilesPerBlock][kMainVec], rv[kMainTilesPerBlock][kMainVec];
#pragma unroll
  for (int u = 0; u < kMainTilesPerBlock; ++u) {
    const uint64_t tbase = (uint64_t)(t0 + u) * kTile;
    if ((uint32_t)u < ntile && tbase + kTile <= a.m) {
#pragma unroll
      for (int q = 0; q < kMainVec; ++q) {
        const uint64_t e = tbase + ((uint64_t)q * kMainThreads + threadIdx.x) * 4;
        gv[u][q] = ld_stream4(a.grad + e);
        if (a.res) rv[u][q] = ld_stream4(a.res + e);
      }
    }
  }
#endif
  // the dense-tile histogram, cleared while the loads are in flight (the
  // first tile's barrier orders it before any use)
  for (int b = threadIdx.x; b < kHistLen; b += kMainThreads) s_hist[b] = 0u;
  // everything below consumes the sample kernel's window (and may write
  // res_out = res in place, which the sample kernel reads): wait for it --
  // the loads above are already in flight (programmatic dependent launch;
  // griddepcontrol.wait itself costs ~1 us per block, hidden behind them:
  // a variant without the sample kernel that had to wait before loading res
  // measured 6 us slower per step)
  if (kMode != kMainDefer) pdl_wait();
  uint32_t lo, shift;
  bool pend = false;
  uint32_t ptau = 0, pcut = 0;
  if (kRecord) {
    // the whole key-window record in one round trip (two independent 16-byte
    // loads, 32-byte aligned: gtk_select_windowed checks): the window of this
    // call and the pending-winner predicate of res_in
    const uint4 r0 = __ldcg(reinterpret_cast<const uint4*>(a.window));
    const uint4 r1 = __ldcg(reinterpret_cast<const uint4*>(a.window) + 1);
    const bool valid = !a.force_exact && (r0.x & kRecValid) && r0.w == a.k;
    lo = valid ? r0.y : 0x7FFFFFFFu;  // no window: nothing passes, the finish runs exact
    shift = valid ? r0.z : 0u;
    pend = kChain && a.res != nullptr && (r0.x & kRecPending) != 0;
    ptau = r1.z;
    pcut = r1.w;
    if (blk == 0) {  // the finish's engine counters and window (read only after this kernel)
      if (threadIdx.x < (unsigned)kRounds) a.gather_n[threadIdx.x] = 0u;
      if (threadIdx.x == 0) {
        a.ctl->lo = lo;
        a.ctl->shift = shift;
      }
    }
  } else {
    lo = __ldcg(&a.ctl->lo);
    shift = __ldcg(&a.ctl->shift);
  }
  bool any_dense = false;
#if GTK_MAIN_TMA
  __syncthreads();  // (the mbarrier's initialisation before anyone waits on it)
  mbar_wait_parity(&s_mbar, 0);
#endif
#pragma unroll
  for (int u = 0; u < kMainTilesPerBlock; ++u) {
    const uint32_t tile = t0 + u;
    const uint64_t tbase = (uint64_t)tile * kTile;
    if ((uint32_t)u >= ntile || tbase >= a.m) break;
    float v[kMainVec][4];
    const bool full = tbase + kTile <= a.m;
    if (full) {
#pragma unroll
      for (int q = 0; q < kMainVec; ++q) {
#if GTK_MAIN_TMA
        float4 x = s_stage[(2 * u) * (kTile / 4) + q * kMainThreads + threadIdx.x];
#else
        float4 x = gv[u][q];
#endif
        if (a.res) {
#if GTK_MAIN_TMA
          float4 r = s_stage[(2 * u + 1) * (kTile / 4) + q * kMainThreads + threadIdx.x];
#else
          float4 r = rv[u][q];
#endif
          // (chained: one max-key test per 4 elements; a pending winner is in
          // ~k/m of them)
          if (kChain && pend &&
              max(max(key_of(r.x), key_of(r.y)), max(key_of(r.z), key_of(r.w))) >= ptau) {
            const uint64_t e = tbase + ((uint64_t)q * kMainThreads + threadIdx.x) * 4;
            r.x = settle_res(r.x, e, ptau, pcut);
            r.y = settle_res(r.y, e + 1, ptau, pcut);
            r.z = settle_res(r.z, e + 2, ptau, pcut);
            r.w = settle_res(r.w, e + 3, ptau, pcut);
          }
          x.x = __fadd_rn(r.x, x.x);
          x.y = __fadd_rn(r.y, x.y);
          x.z = __fadd_rn(r.z, x.z);
          x.w = __fadd_rn(r.w, x.w);
        }
        st_stream4(a.res_out + tbase + ((uint64_t)q * kMainThreads + threadIdx.x) * 4, x);
        v[q][0] = x.x;
        v[q][1] = x.y;
        v[q][2] = x.z;
        v[q][3] = x.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < kMainVec; ++q)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t e = tbase + ((uint64_t)q * kMainThreads + threadIdx.x) * 4 + j;
          float x = 0.0f;
          if (e < a.m) {
            x = a.grad[e];
            if (a.res) x = __fadd_rn((kChain && pend) ? settle_res(a.res[e], e, ptau, pcut) : a.res[e], x);
            a.res_out[e] = x;
          }
          v[q][j] = x;
        }
    }
    any_dense |= main_tile(a, tile, v, full, lo, shift, u & 1, s_wt, s_didx, s_dval, s_hist);
  }
  if (any_dense) {  // block-uniform
    __syncthreads();
    for (int b = threadIdx.x; b < kHistLen; b += kMainThreads) {
      const uint32_t c = s_hist[b];
      if (c) atomicAdd(a.whist + b, c);
    }
  }
  if (a.trace) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax((unsigned long long*)a.trace + 1, (unsigned long long)globaltimer_ns());
  }
  if (kMode == kMainDefer && blk == gridDim.x - 1) pdl_wait();  // complete only after the previous finish
}

// ---------------------------------------------------------------------------
// 3. finish: per-block candidate slices in smem, exact engine / dense fallback
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
  int32_t* ord_idx;  // global staging for a block whose slice exceeds slice_cap
  float* ord_val;
  int32_t* sel_idx;
  float* sel_val;
  int32_t* d_count;
  uint32_t* d_status;
  int64_t* trace;  // optional phase stamps (block 0): [0] start [1] scanned [2] copied [3..6] engine
  uint32_t* window;  // nullable: {valid | level << 8, lo, shift, k, tau} for the next call (written here)
  uint32_t* group_cnt;  // candidates per block, counted by the main pass (reset here for the next call)
  uint32_t tiles_per_group;
  float* upd_w;      // nullable: fused K3 at P = 1 (gtk_select_update)
  float upd_lr;
  float upd_Pf;
  int upd_scaling;
  uint32_t slice_cap;  // candidates per block staged in (dynamic) shared memory
  // gtk_select_push: the selection also goes out as LL records to the
  // exchange's first partner (inbox step-0 slots at ll_base, slot parity and
  // tag from the upcoming exchange call's epoch = *ll_epoch + 1), nullable
  uint64_t* ll_base = nullptr;
  const uint64_t* ll_epoch = nullptr;
  uint32_t ll_slot_words = 0;
  uint32_t chain = 0;  // GTK_SELECT_CHAIN: winners stay pending in res_out (Sink::pend_rec)
  // gtk_select_update_deferred: winners stay pending; the previous call's
  // selection (prev_idx / prev_count, nullable) is corrected first (see
  // deferred_fixup); the dependent launch is released after that correction
  uint32_t defer = 0;
  const int32_t* prev_idx = nullptr;
  const int32_t* prev_count = nullptr;
  const float* grad = nullptr;
  uint32_t fix_cap = 0;  // fix-list entries staged in shared memory behind the slice
  // P > 1 (gtk_select_push_deferred): only previous winners that made the
  // previous global list were zeroed by the reference (optimizer.py:227-230
  // returns the others to the residual): membership = prev_tags[i] == the
  // low word of *prev_epoch (the exchange plan's tags / epoch); nullable (P = 1)
  const uint32_t* prev_tags = nullptr;
  const uint64_t* prev_epoch = nullptr;
  const float* res_in = nullptr;
  uint32_t* ofs_out = nullptr;       // this call's per-block output positions (deferred: the next call's j0 / j1)
  const uint32_t* prev_ofs = nullptr;  // the previous call's (in its workspace), nullable
};

// first index i of the ascending list a[0, n) with a[i] >= x; one full warp,
// 33-ary (a few dependent L2 round trips), result in every lane
__device__ __forceinline__ uint32_t lower_bound_warp(const int32_t* a, uint32_t n, int32_t x) {
  uint32_t L = 0, H = n;
  const unsigned lane = lane_id();
  while (L < H) {
    const uint32_t len = H - L;
    if (len <= 32) {
      const bool q = lane < len && __ldcg(a + L + lane) < x;
      L += __popc(__ballot_sync(kFull, q));
      break;
    }
    const uint32_t p = L + (uint32_t)(((uint64_t)len * (lane + 1)) / 33);
    const bool q = __ldcg(a + p) < x;
    const int t = __popc(__ballot_sync(kFull, q));
    const uint32_t p_prev = __shfl_sync(kFull, p, t > 0 ? t - 1 : 0);
    const uint32_t p_t = __shfl_sync(kFull, p, t < 32 ? t : 31);
    if (t > 0) L = p_prev + 1;
    if (t < 32) H = p_t;
  }
  return L;
}

constexpr uint32_t kFixWas = 1u, kFixNow = 2u;  // fix-list flags: a candidate before / after the correction

// Deferred settle, before the finish ranks anything: the previous call's
// winners in this block's tile range were pending in res_in, so this call's
// main pass streamed acc' = acc_prev + g there instead of +0 + g (reference
// optimizer.py:230 zeroes them first).  Each one gets res_out[i] = +0 + g[i];
// the window histogram moves it between bins / in or out of the window, and
// the candidate changes go to a fix list (index order) applied to the slice
// after the copy.  Returns the fix-list length (*n_ins: new candidates);
// raises the overflow flag (exact dense fallback over the corrected res_out)
// if the lists do not fit.
// The words the correction starts from, loaded right after griddepcontrol.wait
// in one round trip together with the non-finite check (they are independent:
// loading them inside deferred_fixup put two more dependent round trips ahead
// of the next pass's release)
struct FixupPre {
  uint32_t lo, shift, n_prev, ep32, ofs0, ofs_b;
};
__device__ __forceinline__ FixupPre fixup_preload(const FinishArgs& a) {
  FixupPre p;
  p.lo = __ldcg(&a.ctl->lo);
  p.shift = __ldcg(&a.ctl->shift);
  p.n_prev = (uint32_t)max(__ldcg(a.prev_count), 0);
  p.ep32 = a.prev_epoch ? (uint32_t)__ldcg((const unsigned long long*)a.prev_epoch) : 0u;
  p.ofs0 = a.prev_ofs ? __ldcg(a.prev_ofs) : 0u;
  const uint32_t b = blockIdx.x + threadIdx.x;  // (threads 0 / 1: my range's ends)
  p.ofs_b = (a.prev_ofs && threadIdx.x < 2 && b < gridDim.x) ? __ldcg(a.prev_ofs + 1 + b) : 0xFFFFFFFFu;
  return p;
}

__device__ uint32_t deferred_fixup(const FinishArgs& a, EngineSmem<kFinishThreads>& sm, int32_t* f_idx, float* f_val,
                                   uint32_t* f_flag, uint32_t t0, uint32_t t1, uint32_t* n_ins_out,
                                   const FixupPre& pre) {
  const uint32_t lo = pre.lo, shift = pre.shift;
  const uint32_t n_prev = min(pre.n_prev, a.m);
  const uint32_t ep32 = pre.ep32;
  const int32_t E0 = (int32_t)min((uint64_t)t0 * kTile, (uint64_t)a.m);
  const int32_t E1 = (int32_t)min((uint64_t)t1 * kTile, (uint64_t)a.m);
  // my range of the previous selection: its finish recorded every block's
  // first output position (same tile partition), else two warp searches
  const bool have_ofs = a.prev_ofs && pre.ofs0 == gridDim.x;
  if (have_ofs) {
    if (threadIdx.x < 2) sm.bcast[threadIdx.x] = min(pre.ofs_b, n_prev);  // (past the last block: n_prev)
  } else if (warp_id() < 2) {
    const uint32_t j = lower_bound_warp(a.prev_idx, n_prev, warp_id() == 0 ? E0 : E1);
    if (lane_id() == 0) sm.bcast[warp_id()] = j;
  }
  __syncthreads();
  const uint32_t j0 = sm.bcast[0], j1 = sm.bcast[1];
  // histogram moves of this block, aggregated in shared memory first (the
  // previous winners mostly sit in the same top bins: one global atomic per
  // bin and block instead of one per winner)
  for (int b = threadIdx.x; b < kHistLen; b += kFinishThreads) sm.hist[b] = 0u;
  __syncthreads();
  uint32_t n_fix = 0, n_ins = 0;
  for (uint32_t base = j0; base < j1; base += kFinishThreads) {  // block-uniform trip count
    const uint32_t j = base + threadIdx.x;
    const bool has = j < j1;
    int32_t e = 0;
    float ap = 0.0f, gv = 0.0f, rp = 0.0f;
    uint32_t tg = ep32;
    if (has) e = __ldcg(a.prev_idx + j);
    if (has) {
      ap = __ldcg(a.res_out + e);
      gv = __ldcg(a.grad + e);
      if (a.prev_tags) {
        tg = __ldcg(a.prev_tags + e);
        rp = __ldcg(a.res_in + e);
      }
    }
    // a member of the previous global list: res = +0 there; otherwise the
    // reference returned the value: res = +0 + acc (acc itself unless -0)
    const float A = (tg == ep32) ? __fadd_rn(0.0f, gv) : __fadd_rn(__fadd_rn(0.0f, rp), gv);
    bool was = false, now = false;
    if (has) {
      if (__float_as_uint(A) != __float_as_uint(ap)) a.res_out[e] = A;
      const uint32_t kw = key_of(ap), kn = key_of(A);
      was = kw >= lo;
      now = kn >= lo;
      const uint32_t bw = was ? min((uint32_t)kBins, (kw - lo) >> shift) : 0u;
      const uint32_t bn = now ? min((uint32_t)kBins, (kn - lo) >> shift) : 0u;
      if (was && !(now && bw == bn)) atomicSub(&sm.hist[bw], 1u);
      if (now && !(was && bw == bn)) atomicAdd(&sm.hist[bn], 1u);
    }
    const bool keep = was || now;
    uint32_t tot;
    const uint32_t pos = n_fix + block_excl_scan<kFinishThreads>(keep ? 1u : 0u, sm.scan, &tot);
    GTK_DCHECK(!has || (e >= 0 && (uint32_t)e < a.m));
    if (keep && pos < a.fix_cap) {
      f_idx[pos] = e;
      f_val[pos] = A;
      f_flag[pos] = (was ? kFixWas : 0u) | (now ? kFixNow : 0u);
    }
    n_fix += tot;
    n_ins += block_sum<kFinishThreads>((now && !was) ? 1u : 0u, sm.scan);
  }
  *n_ins_out = n_ins;
  return n_fix;  // (the histogram moves stay in sm.hist for deferred_fixup_publish)
}

// The fixup's effects on this finish's own bookkeeping -- the histogram moves
// (sm.hist), the new candidates of my tile range, the overflow flag -- after
// the next pass has been released: it reads none of them (it works in the
// other select workspace), and the grid barrier that follows orders them
// before this finish reads them.
__device__ void deferred_fixup_publish(const FinishArgs& a, EngineSmem<kFinishThreads>& sm, uint32_t n_fix,
                                       uint32_t n_ins) {
  for (int b = threadIdx.x; b < kHistLen; b += kFinishThreads) {  // (block_sum in the fixup synced sm.hist)
    const uint32_t dlt = sm.hist[b];
    if (dlt) atomicAdd(a.ews->hist[0] + b, dlt);  // (mod 2^32: negative moves wrap)
  }
  if (threadIdx.x == 0) {
    if (n_ins) atomicAdd(a.group_cnt + blockIdx.x, n_ins);
    if (n_fix > a.fix_cap || n_ins > (uint32_t)kGatherCap)
      atomicOr(&a.ctl->overflow, 1u);  // lists too long: exact dense fallback (res_out is corrected)
  }
}

// The fix list applied to the staged slice (index order, own_raw entries):
// a previous winner that was a candidate gets its corrected value or leaves
// (empty slot); one that became a candidate is inserted in index order.
// (s_idx / s_val: the slice in shared memory or in the global staging list)
__device__ void apply_fixes(int32_t* s_idx, float* s_val, uint32_t own_raw, const int32_t* f_idx, const float* f_val,
                            uint32_t* f_flag, uint32_t n_fix, uint32_t n_ins, EngineSmem<kFinishThreads>& sm) {
  // positions first (the slice is still sorted): a was-candidate's slot, an
  // insertion's rank r = # slice entries below it
  uint32_t* ins = sm.keys;  // compacted insertions: fix-list positions
  uint32_t n_seen = 0;
  for (uint32_t base = 0; base < n_fix; base += kFinishThreads) {
    const uint32_t f = base + threadIdx.x;
    const bool has = f < n_fix;
    const uint32_t fl = has ? f_flag[f] : 0u;
    const bool insert = has && (fl & kFixNow) && !(fl & kFixWas);
    if (has) f_flag[f] = (fl & 3u) | (lower_bound_s(s_idx, own_raw, f_idx[f]) << 2);
    uint32_t tot;
    const uint32_t p = n_seen + block_excl_scan<kFinishThreads>(insert ? 1u : 0u, sm.scan, &tot);
    if (insert) ins[p] = f;
    n_seen += tot;
  }
  __syncthreads();
  for (uint32_t f = threadIdx.x; f < n_fix; f += kFinishThreads) {
    const uint32_t fl = f_flag[f];
    if (fl & kFixWas) {
      const uint32_t pos = fl >> 2;
      if (fl & kFixNow) s_val[pos] = f_val[f];
      else s_idx[pos] = -1;  // empty slot (SliceSrc::get)
    }
  }
  __syncthreads();
  if (n_ins == 0) return;
  // slice entry p moves up by the insertions with r <= p: descending chunks,
  // all of a chunk read before any of it is written (targets lie at or above
  // the chunk, n_ins < one chunk)
  for (int c = (int)((own_raw + kFinishThreads - 1) / kFinishThreads) - 1; c >= 0; --c) {
    const uint32_t p = (uint32_t)c * kFinishThreads + threadIdx.x;
    int32_t xi = 0;
    float xv = 0.0f;
    uint32_t np = 0;
    if (p < own_raw) {
      xi = s_idx[p];
      xv = s_val[p];
      uint32_t lo_ = 0, hi_ = n_ins;  // # insertions with r <= p
      while (lo_ < hi_) {
        const uint32_t mid = (lo_ + hi_) >> 1;
        if ((f_flag[ins[mid]] >> 2) <= p) lo_ = mid + 1;
        else hi_ = mid;
      }
      np = p + lo_;
    }
    __syncthreads();
    GTK_DCHECK(p >= own_raw || np < own_raw + n_ins);
    if (p < own_raw) {
      s_idx[np] = xi;
      s_val[np] = xv;
    }
    __syncthreads();
  }
  for (uint32_t q = threadIdx.x; q < n_ins; q += kFinishThreads) {
    const uint32_t f = ins[q];
    const uint32_t np = (f_flag[f] >> 2) + q;
    GTK_DCHECK(np < own_raw + n_ins);
    s_idx[np] = f_idx[f];
    s_val[np] = f_val[f];
  }
  __syncthreads();
}

// block 0 of the finish, once every block has read them: the main pass's
// counters start the next call at zero (a chained call has no sampling kernel
// to reset them)
__device__ __forceinline__ void reset_select_counters(const FinishArgs& a, unsigned G) {
  for (unsigned i = threadIdx.x; i < G; i += blockDim.x) a.group_cnt[i] = 0u;
  if (threadIdx.x == 0) {
    a.ctl->ovf_cursor = 0u;
    a.ctl->overflow = 0u;
    a.ctl->nonfinite = 0u;
  }
}

__device__ __forceinline__ void finish_stamp(const FinishArgs& a, int i) {
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[i] = (int64_t)t;
  }
}

#ifndef GTK_FINISH_MIN_BLOCKS
#define GTK_FINISH_MIN_BLOCKS 2
#endif
__global__ void __launch_bounds__(kFinishThreads, GTK_FINISH_MIN_BLOCKS) select_finish_kernel(FinishArgs a) {
  __shared__ EngineSmem<kFinishThreads> sm;
  extern __shared__ __align__(16) unsigned char s_dyn[];  // the candidate slice: slice_cap (idx, val)
  int32_t* s_idx = reinterpret_cast<int32_t*>(s_dyn);
  float* s_val = reinterpret_cast<float*>(s_dyn + sizeof(int32_t) * a.slice_cap);
  const unsigned G = gridDim.x, blk = blockIdx.x;
  pdl_wait();  // launched programmatically behind the main pass
  grid_sync_begin(&a.ews->bar);
  // (a deferred call with a previous selection releases the next call's main
  // pass once that selection is corrected in res_out, below)
  const bool fixing = a.defer && a.prev_idx != nullptr;
  if (!fixing) pdl_launch_dependents();
  // margin level of the carried window (only block 0 writes the record)
  const uint32_t wlevel = (a.window && blk == 0) ? min(kMaxWindowLevel, max(kMinWindowLevel, __ldcg(a.window) >> 8)) : kMinWindowLevel;
  const bool wsame = a.window && blk == 0 && __ldcg(a.window + 3) == a.k;
  const uint32_t wtau = wsame ? __ldcg(a.window + 4) : 0u, wtau2 = wsame ? __ldcg(a.window + 5) : 0u;
  FixupPre fpre{};
  if (fixing) fpre = fixup_preload(a);
  if (const uint32_t bad = __ldcg(&a.ctl->nonfinite)) {
    grid_sync(&a.ews->bar, G);  // every block has read the counters
    if (blk == 0) {
      for (int b = threadIdx.x; b < kHistLen; b += kFinishThreads) a.ews->hist[0][b] = 0;
      reset_select_counters(a, G);
      if (threadIdx.x == 0) {
        atomicOr(a.d_status, ((bad & 1u) ? GTK_DEV_NONFINITE : 0u) |
                                 ((bad & kCtlPendingViolation) ? GTK_DEV_PENDING : 0u));
        if (a.ll_base) {  // the exchange's first partner learns it at once: count -1 (poisoned)
          const uint32_t tag = (uint32_t)(__ldcg((const unsigned long long*)a.ll_epoch) + 1ull);
          st_ll_pair(a.ll_base + (size_t)(tag & 1u) * a.ll_slot_words, 0xFFFFFFFFu, 0u, tag);
        }
        if (a.window) {
          // the step fails and the state keeps res_in: its pending winners
          // (a chained predecessor's) stay recorded
          a.window[0] = (wlevel << 8) | (__ldcg(a.window) & kRecPending);
          a.window[4] = a.window[5] = 0u;
        }
      }
    }
    return;
  }
  // the fused update skips on an error an EARLIER step left in the (sticky)
  // status word of a pipeline, like the exchange's K3: the weights keep the
  // last good step
  float* const upd_w = (a.upd_w && !(__ldcg(a.d_status) & GTK_DEV_ERROR_MASK)) ? a.upd_w : nullptr;
  Sink out{a.sel_idx, a.sel_val, a.d_count, (a.chain || a.defer) ? nullptr : a.res_out, true,
           a.trace ? a.trace + 3 : nullptr,
           a.window, wlevel, wtau, wtau2, 1u, upd_w, a.upd_lr, a.upd_Pf, a.upd_scaling};
  if (a.chain) out.pend_rec = a.window;
  if (a.ofs_out) {  // written by the candidate path's gather finish only (same tile partition next call)
    if (blk == 0 && threadIdx.x == 0) a.ofs_out[0] = 0u;
    out.blk_ofs = a.ofs_out;
  }
  if (a.ll_base) {  // the exchange's step 0 send, straight from the write phase
    const uint32_t tag = (uint32_t)(__ldcg((const unsigned long long*)a.ll_epoch) + 1ull);
    uint64_t* slot = a.ll_base + (size_t)(tag & 1u) * a.ll_slot_words;
    out.ll_body = slot + 2;
    out.ll_head = slot;
    out.ll_tag = tag;
  }
  finish_stamp(a, 0);
  const uint32_t per = a.tiles_per_group;
  const uint32_t t0 = min(a.ntiles, blk * per), t1 = min(a.ntiles, t0 + per);

  // deferred settle of the previous call's winners (histogram corrections
  // complete behind the grid barrier before anyone reads the histogram)
  int32_t* f_idx = reinterpret_cast<int32_t*>(s_dyn + (sizeof(int32_t) + sizeof(float)) * a.slice_cap);
  float* f_val = reinterpret_cast<float*>(f_idx + a.fix_cap);
  uint32_t* f_flag = reinterpret_cast<uint32_t*>(f_val + a.fix_cap);
  uint32_t n_fix = 0, n_ins = 0;
  if (fixing) {
    n_fix = deferred_fixup(a, sm, f_idx, f_val, f_flag, t0, t1, &n_ins, fpre);
    if (a.trace && blk == 0 && threadIdx.x == 0) {  // diagnostics (block 0's fix list)
      a.trace[14] = n_fix;
      a.trace[15] = n_ins;
    }
#ifdef GTK_FIXUP_PUBLISH_EARLY  // (A/B: the round-2 order, bookkeeping ahead of the release)
    deferred_fixup_publish(a, sm, n_fix, n_ins);
#endif
    __threadfence();  // res_out corrections visible before the next main pass is released
    __syncthreads();
    pdl_launch_dependents();
#ifndef GTK_FIXUP_PUBLISH_EARLY
    deferred_fixup_publish(a, sm, n_fix, n_ins);
#endif
    n_fix = min(n_fix, a.fix_cap);
    grid_sync(&a.ews->bar, G);
    finish_stamp(a, 20);  // (diagnostics: fixup + barrier done)
  }

  // the round-0 window histogram (main pass) -> sm.hist by async copies
  // issued now and awaited after the candidate copy: their L2 latency hides
  // behind it (the copy's scratch lives in the gather arrays instead)
  for (int b = threadIdx.x; b < kHistLen; b += kFinishThreads) cp_async4(&sm.hist[b], a.ews->hist[0] + b);
  cp_async_commit();  // group: histogram
  // my tile range and its place in the global (index-ordered) candidate list:
  // the main pass counted the candidates of every block's tile range
  uint32_t C;
  {
    const uint32_t c = threadIdx.x < G ? __ldcg(a.group_cnt + threadIdx.x) : 0u;
    const uint32_t ex = block_excl_scan<kFinishThreads>(c, sm.scan, &C);
    if (threadIdx.x == blk) {
      sm.bcast[0] = ex;
      sm.bcast[1] = c;
    }
    __syncthreads();
  }
  const uint32_t before = sm.bcast[0], own = sm.bcast[1];
  const bool overflow = __ldcg(&a.ctl->overflow) != 0;
  finish_stamp(a, 1);
  if (a.defer && a.trace && blk == 0 && threadIdx.x == 0) {  // diagnostics: the candidate-path decision
    a.trace[16] = overflow;
    a.trace[17] = C;
    a.trace[18] = a.ord_cap;
    a.trace[19] = 0;
  }
  if (!overflow && C >= a.k && C <= a.ord_cap) {
    // copy my tiles' candidates into my slice (smem if it fits)
    const bool in_smem = own <= a.slice_cap;
    int32_t* di = in_smem ? s_idx : a.ord_idx + before;
    float* dv = in_smem ? s_val : a.ord_val + before;
    static_assert(kGatherCap >= kFinishThreads, "copy scratch");
    uint32_t* s_dst = sm.keys;                               // per-tile destination (local)
    uint32_t* s_cnt = reinterpret_cast<uint32_t*>(sm.gidx);  // per-tile info
    uint32_t* s_ovf = sm.gblk;                               // per-tile overflow base
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
      // many candidates per tile (large k): one warp per tile, lanes over its
      // contiguous slot row (coalesced, no search); otherwise entry-indexed:
      // entry j of this chunk lives in tile q with s_dst[q] - run <= j <
      // s_dst[q+1] - run (binary search in smem)
      const bool per_tile = tot >= 8u * nt;
      if (per_tile) {
        for (uint32_t q = warp_id(); q < nt; q += kFinishThreads / 32) {
          const uint32_t inf = s_cnt[q];
          if (inf & kOvfBit) continue;  // dense tiles are copied below
          const uint32_t cnt = inf, dst = s_dst[q];
          const size_t sb = (size_t)(tb + q) * a.slots;
          for (uint32_t e = lane_id(); e < cnt; e += 32) {
            if (in_smem) {
              cp_async4(di + dst + e, a.slot_idx + sb + e);
              cp_async4(dv + dst + e, a.slot_val + sb + e);
            } else {
              di[dst + e] = __ldcg(a.slot_idx + sb + e);
              dv[dst + e] = __ldcg(a.slot_val + sb + e);
            }
          }
        }
      }
#pragma unroll 4
      for (uint32_t j = per_tile ? tot : threadIdx.x; j < tot; j += kFinishThreads) {
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
        GTK_DCHECK(jj - s_dst[lo] < a.slots && (!in_smem || jj < a.slice_cap));
        if (in_smem) {  // async: lands while the k-th key's bin is found
          cp_async4(di + jj, a.slot_idx + src);
          cp_async4(dv + jj, a.slot_val + src);
        } else {
          di[jj] = __ldcg(a.slot_idx + src);
          dv[jj] = __ldcg(a.slot_val + src);
        }
      }
      for (uint32_t q = warp_id(); q < nt; q += kFinishThreads / 32) {  // dense tiles
        const uint32_t inf = s_cnt[q];
        if (!(inf & kOvfBit)) continue;
        const uint32_t cnt = inf & ~kOvfBit, ob = s_ovf[q], dst = s_dst[q];
        for (uint32_t e = lane_id(); e < cnt; e += 32) {
          if (in_smem) {
            cp_async4(di + dst + e, a.ovf_idx + ob + e);
            cp_async4(dv + dst + e, a.ovf_val + ob + e);
          } else {
            di[dst + e] = __ldcg(a.ovf_idx + ob + e);
            dv[dst + e] = __ldcg(a.ovf_val + ob + e);
          }
        }
      }
      run += tot;
      __syncthreads();
    }
    finish_stamp(a, 2);
    if (a.trace && blk == 0 && threadIdx.x == 0) {  // diagnostics: slice sizes
      a.trace[10] = own;
      a.trace[11] = a.slice_cap;
      a.trace[12] = C;
      a.trace[13] = G;
    }
    cp_async_commit();    // group: the slice
    const bool fixes = n_fix > 0;  // (block-local)
    if (fixes) {  // the slice must have landed
      cp_async_wait_all();
      __syncthreads();
      apply_fixes(di, dv, own - n_ins, f_idx, f_val, f_flag, n_fix, n_ins, sm);
    } else {
      cp_async_wait<1>();   // the histogram has landed; the slice may still be in flight
      __syncthreads();
    }
    SliceSrc src{s_idx, s_val, a.ord_idx, a.ord_val, before, in_smem, false};
    if (engine_run<kFinishThreads>(src, before, before + own, a.k, false, __ldcg(&a.ctl->lo),
                                   __ldcg(&a.ctl->shift), sm.hist, true, a.ews, sm, out, G,
                                   /*slice_async=*/!fixes)) {
      if (a.trace && threadIdx.x == 0)  // timeline: last block end (trace_buffer()[114])
        atomicMax((unsigned long long*)a.trace + 66, (unsigned long long)globaltimer_ns());
      if (blk == 0) reset_select_counters(a, G);  // (the engine's grid barrier is behind every read)
      return;
    }
  }
  // exact dense fallback over acc (= res_out, untouched so far)
  if (a.defer && a.trace && blk == 0 && threadIdx.x == 0) a.trace[19] = 1;
  cp_async_wait_all();  // the histogram prefetch must land before sm.hist is reused
  grid_sync(&a.ews->bar, G);
  if (blk == 0) {
    for (int r = 0; r < kRounds; ++r)
      for (int b = threadIdx.x; b < kHistLen; b += kFinishThreads) a.ews->hist[r][b] = 0;
    if (threadIdx.x < kRounds) a.ews->gather_n[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
      atomicOr(a.d_status, GTK_DEV_FALLBACK);
      // the record is invalid until the exact pass below rewrites it; a
      // window that admitted too few keys widens its margin from then on
      const bool low_miss = !overflow && C < a.k;
      if (a.window) {
        a.window[0] = (low_miss ? min(kMaxWindowLevel, wlevel + 1) : wlevel) << 8;
        a.window[4] = a.window[5] = 0u;  // no growth estimate across a gap
      }
    }
  }
  grid_sync(&a.ews->bar, G);
  DenseSrc dsrc{a.res_out};
  uint32_t s0, s1;
  slice_of(a.m, G, blk, s0, s1);
  // the exact pass's own round-0 histogram (full key range, 2^20-key bins)
  // records a fresh window for the next call (block 0), at the raised margin
  // after a low miss and with no growth estimate across the gap
  Sink dout = out;
  dout.blk_ofs = nullptr;  // (the dense partition is not the tile partition)
  dout.window_level = (!overflow && C < a.k) ? min(kMaxWindowLevel, wlevel + 1) : wlevel;
  dout.prev_tau = dout.prev_tau2 = 0u;
  engine_run<kFinishThreads>(dsrc, s0, s1, a.k, false, 0u, 20u, nullptr, false, a.ews, sm, dout, G);
  if (blk == 0) reset_select_counters(a, G);
  // the record's k-th-key estimate: the exact k-th key (this thread wrote it
  // as the count's hint) instead of the edge of its 2^20-key bin -- a coarse
  // estimate would read as a jump of the k-th key two calls later and push
  // that window's lower edge far down (overflow, another fallback, ...)
  if (a.window && blk == 0 && threadIdx.x == 0) a.window[4] = (uint32_t)a.d_count[1];
}

}  // namespace gtk

using namespace gtk;

// main-pass grid: two tiles per block, except that about one wave of resident
// blocks at the end of the grid takes one tile each (a shorter drain)
static bool main_smem_ready() {
  if (kMainStageBytes == 0) return true;
  return ensure_dyn_smem((const void*)select_main_kernel<kMainPlain>, kMainStageBytes) &&
         ensure_dyn_smem((const void*)select_main_kernel<kMainChain>, kMainStageBytes) &&
         ensure_dyn_smem((const void*)select_main_kernel<kMainDefer>, kMainStageBytes);
}

static uint32_t main_grid(uint32_t ntiles, uint32_t* n2) {
  if (!main_smem_ready()) return 0;
  const int slots = coop_grid((const void*)select_main_kernel<kMainPlain>, kMainThreads, kMainStageBytes);  // resident blocks, all SMs
  if (slots <= 0) return 0;
  uint32_t n1 = std::min<uint32_t>(ntiles, (uint32_t)slots);
  uint32_t two = (ntiles - n1) / 2;
  n1 = ntiles - 2 * two;
  *n2 = two;
  return two + n1;
}

extern "C" int gtk_select_workspace_bytes(int64_t m, int32_t k, size_t* bytes) {
  if (!bytes || m < 1 || m >= (int64_t(1) << 31) || k < 1 || k > m) return GTK_EINVAL;
  *bytes = select_layout(m, k).total;
  return GTK_OK;
}

extern "C" int gtk_select(const float* res_in, const float* grad, float* res_out, int64_t m, int32_t k,
                          int32_t* sel_idx, float* sel_val, int32_t* d_count, uint32_t* d_status, void* ws,
                          size_t ws_bytes, int32_t flags, void* stream) {
  return gtk_select_windowed(res_in, grad, res_out, m, k, sel_idx, sel_val, d_count, d_status, ws, ws_bytes, flags,
                             nullptr, stream);
}

namespace {
struct FusedUpdate {
  float* w;
  float lr;
  float Pf;
  int scaling;
};
}  // namespace

struct PeerPush {
  uint64_t* slot0;
  const uint64_t* epoch;
};
struct Deferred {  // gtk_select_update_deferred / gtk_select_push_deferred
  bool on;
  const int32_t* prev_idx;
  const int32_t* prev_count;
  const void* prev_ws;
  const uint32_t* prev_tags = nullptr;
  const uint64_t* prev_epoch = nullptr;
};
static int select_impl(const float* res_in, const float* grad, float* res_out, int64_t m, int32_t k,
                       int32_t* sel_idx, float* sel_val, int32_t* d_count, uint32_t* d_status, void* ws,
                       size_t ws_bytes, int32_t flags, uint32_t* d_window, FusedUpdate upd, void* stream,
                       PeerPush push = {nullptr, nullptr}, Deferred dfr = {false, nullptr, nullptr, nullptr, nullptr, nullptr});

extern "C" int gtk_select_windowed(const float* res_in, const float* grad, float* res_out, int64_t m, int32_t k,
                                   int32_t* sel_idx, float* sel_val, int32_t* d_count, uint32_t* d_status,
                                   void* ws, size_t ws_bytes, int32_t flags, uint32_t* d_window, void* stream) {
  return select_impl(res_in, grad, res_out, m, k, sel_idx, sel_val, d_count, d_status, ws, ws_bytes, flags,
                     d_window, FusedUpdate{nullptr, 0.0f, 1.0f, 0}, stream);
}

extern "C" int gtk_select_push(const float* res_in, const float* grad, float* res_out, int64_t m, int32_t k,
                               int32_t* sel_idx, float* sel_val, int32_t* d_count, uint32_t* d_status, void* ws,
                               size_t ws_bytes, int32_t flags, uint32_t* d_window, void* peer_slot0,
                               const uint64_t* d_epoch, void* stream) {
  if (!peer_slot0 || !d_epoch) return GTK_EINVAL;
  return select_impl(res_in, grad, res_out, m, k, sel_idx, sel_val, d_count, d_status, ws, ws_bytes, flags,
                     d_window, FusedUpdate{nullptr, 0.0f, 1.0f, 0}, stream,
                     PeerPush{(uint64_t*)peer_slot0, d_epoch});
}

extern "C" int gtk_select_update(const float* res_in, const float* grad, float* res_out, int64_t m, int32_t k,
                                 int32_t* sel_idx, float* sel_val, int32_t* d_count, uint32_t* d_status, void* ws,
                                 size_t ws_bytes, int32_t flags, uint32_t* d_window, float* w, float lr, int32_t P,
                                 int32_t scaling, void* stream) {
  // only the sparse-exact form (see gtk_update.cu) fuses; the caller runs the
  // dense K3 for any other lr
  if (!w || P < 1 || scaling < 0 || scaling > 2 || !std::isfinite(lr) || std::signbit(lr)) return GTK_EINVAL;
  return select_impl(res_in, grad, res_out, m, k, sel_idx, sel_val, d_count, d_status, ws, ws_bytes, flags,
                     d_window, FusedUpdate{w, lr, (float)P, scaling}, stream);
}

extern "C" int gtk_select_update_deferred(const float* res_in, const float* grad, float* res_out, int64_t m,
                                          int32_t k, int32_t* sel_idx, float* sel_val, int32_t* d_count,
                                          uint32_t* d_status, void* ws, size_t ws_bytes, uint32_t* d_window,
                                          const int32_t* prev_sel_idx, const int32_t* prev_count,
                                          const void* prev_ws, float* w, float lr, int32_t P, int32_t scaling,
                                          void* stream) {
  if (!w || !res_in || P < 1 || scaling < 0 || scaling > 2 || !std::isfinite(lr) || std::signbit(lr))
    return GTK_EINVAL;
  return select_impl(res_in, grad, res_out, m, k, sel_idx, sel_val, d_count, d_status, ws, ws_bytes, 0, d_window,
                     FusedUpdate{w, lr, (float)P, scaling}, stream, PeerPush{nullptr, nullptr},
                     Deferred{true, prev_sel_idx, prev_count, prev_sel_idx ? prev_ws : nullptr});
}

extern "C" int gtk_select_push_deferred(const float* res_in, const float* grad, float* res_out, int64_t m, int32_t k,
                                        int32_t* sel_idx, float* sel_val, int32_t* d_count, uint32_t* d_status,
                                        void* ws, size_t ws_bytes, uint32_t* d_window, const int32_t* prev_sel_idx,
                                        const int32_t* prev_count, const void* prev_ws, const uint32_t* prev_tags,
                                        void* peer_slot0, const uint64_t* d_epoch, void* stream) {
  // peer_slot0 = NULL: this rank receives first (tree schedule root): no push
  if (!res_in || !d_epoch || (prev_sel_idx && !prev_tags)) return GTK_EINVAL;
  return select_impl(res_in, grad, res_out, m, k, sel_idx, sel_val, d_count, d_status, ws, ws_bytes, 0, d_window,
                     FusedUpdate{nullptr, 0.0f, 1.0f, 0}, stream, PeerPush{(uint64_t*)peer_slot0, d_epoch},
                     Deferred{true, prev_sel_idx, prev_count, prev_sel_idx ? prev_ws : nullptr, prev_tags, d_epoch});
}

static int select_impl(const float* res_in, const float* grad, float* res_out, int64_t m, int32_t k,
                       int32_t* sel_idx, float* sel_val, int32_t* d_count, uint32_t* d_status, void* ws,
                       size_t ws_bytes, int32_t flags, uint32_t* d_window, FusedUpdate upd, void* stream,
                       PeerPush push, Deferred dfr) {
  if (!grad || !res_out || !sel_idx || !sel_val || !d_count || !d_status || !ws) return GTK_EINVAL;
  if (dfr.on && (!d_window || (uintptr_t)d_window % 32 != 0 || res_out == res_in || res_out == grad ||
                 (dfr.prev_idx && (!dfr.prev_count || dfr.prev_idx == sel_idx || dfr.prev_ws == ws))))
    return GTK_EINVAL;
  if (m < 1 || m >= (int64_t(1) << 31) || k < 1 || k > m) return GTK_EINVAL;
  // a chained call needs the record that carries its window and the pending
  // winners, and its own output buffer (res_in is read early, before the
  // previous call's kernels have finished)
  if ((flags & GTK_SELECT_CHAIN) &&
      (!d_window || (uintptr_t)d_window % 32 != 0 || res_out == res_in || res_out == grad))
    return GTK_EINVAL;
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
  // the finish grid (cooperative): fixed before the main pass, which counts
  // the candidates of each finish block's tile range
  // slice capacity: a carried window admits ~3k candidates (9k at the widest
  // margin); stage ~4k / G per block in shared memory, at least kSliceCap
  const int nsm = num_sms();
  if (nsm <= 0) return GTK_ECUDA;
  uint32_t slice_cap = kSliceCap;
  {
    const uint64_t per = ((uint64_t)k * 4 + nsm - 1) / nsm;
    if (per > slice_cap) slice_cap = (uint32_t)std::min<uint64_t>((per + 1023) & ~1023ull, kSliceCapMax);
  }
  // deferred calls stage the previous winners of a block's tile range (~k/G,
  // room for 2x) behind the slice: the fix list
  uint32_t fix_cap = dfr.on ? (uint32_t)std::max<uint64_t>(512, ((2ull * k + nsm - 1) / nsm + 255) & ~255ull) : 0u;
  size_t fin_smem = (size_t)slice_cap * (sizeof(int32_t) + sizeof(float)) + (size_t)fix_cap * 12;
  if (fin_smem > kFinishDynSmemMax) return GTK_EINVAL;  // (deferred at very large k: use gtk_select_update)
  if (!ensure_dyn_smem((const void*)select_finish_kernel, kFinishDynSmemMax)) return GTK_ECUDA;
  int G = coop_grid((const void*)select_finish_kernel, kFinishThreads, fin_smem);
  if (G <= 0) return GTK_ECUDA;
  {
    int want = (int)((L.ntiles + 39) / 40);  // ~40 tiles per block (measured best of 22..150)
    if ((int64_t)want * slice_cap < (int64_t)k * 2) want = (int)(((int64_t)k * 2 + slice_cap - 1) / slice_cap);
    if (want < 8) want = 8;
    if ((uint32_t)want > L.ntiles) want = (int)L.ntiles;
    if (G > want) G = want;
    if (G > nsm) G = nsm;
    // deferred: the finish runs beside the next call's HBM pass; on ~2/5 of
    // the SMs it leaves the rest to that pass at full occupancy (measured at
    // the headline: 148 blocks 66.7 us/step, 100 64.0, 74 63.3, 60 62.9)
    if (dfr.on) {
      const int gd = std::max(8, (nsm * 2 + 4) / 5);
      const int gk = (int)(((int64_t)k * 2 + slice_cap - 1) / slice_cap);
      G = std::min(G, std::max(gd, gk));
    }
    const char* fg = getenv("GTK_FINISH_G");  // (measurement switch)
    if (fg && atoi(fg) > 0 && atoi(fg) < G && (int64_t)atoi(fg) * slice_cap >= (int64_t)k * 2) G = atoi(fg);
    if (dfr.on) {  // the fix list holds ~k / G previous winners per block: room for 2x
      fix_cap = (uint32_t)std::max<uint64_t>(512, ((2ull * k + G - 1) / G + 255) & ~255ull);
      fin_smem = (size_t)slice_cap * (sizeof(int32_t) + sizeof(float)) + (size_t)fix_cap * 12;
      if (fin_smem > kFinishDynSmemMax) return GTK_EINVAL;
    }
    if (G > kMaxBlocks) G = kMaxBlocks;
  }
  const uint32_t tiles_per_group = (L.ntiles + G - 1) / G;
  uint32_t* group_cnt = (uint32_t*)(base + L.group_cnt);

  const bool chain = (flags & GTK_SELECT_CHAIN) != 0;
  const bool defer = dfr.on;
  const bool force_exact = (flags & GTK_SELECT_FORCE_EXACT) != 0;
  ProfScope prof_all(kProfSelect, st);
  if (!chain && !defer) {  // a chained call takes its window from the record: no sampling pass
    SampleArgs sa{res_in, grad, (uint32_t)m, stride, nchunks, r_lo, r_hi, (uint32_t)(force_exact ? 1 : 0), stop,
                  d_window, (uint32_t)k, ctl, ews, group_cnt, trace_buffer() ? trace_buffer() + 64 : nullptr};
    GTK_CUDA(launch_pdl(select_sample_kernel, dim3(nchunks), dim3(kSampleThreads), 0, st, sa));
    GTK_CHECK_LAUNCH();
  }

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
              ews->hist[0],
              group_cnt,
              tiles_per_group};
  ma.window = d_window;
  ma.k = (uint32_t)k;
  ma.chain = (chain || defer) ? 1u : 0u;
  ma.force_exact = force_exact ? 1u : 0u;
  ma.gather_n = ews->gather_n;
  {
    ProfScope prof_main(kProfSelectMain, st);
    const uint32_t gmain = main_grid(L.ntiles, &ma.n2);
    if (gmain == 0) return GTK_ECUDA;
    ma.trace = trace_buffer() ? trace_buffer() + 112 : nullptr;
    auto* mk = defer ? select_main_kernel<kMainDefer>
                     : (chain ? select_main_kernel<kMainChain> : select_main_kernel<kMainPlain>);
    GTK_CUDA(launch_pdl(mk, dim3(gmain), dim3(kMainThreads), kMainStageBytes, st, ma));
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
                trace_buffer() ? trace_buffer() + 48 : nullptr,
                d_window,
                group_cnt,
                tiles_per_group,
                upd.w,
                upd.lr,
                upd.Pf,
                upd.scaling,
                slice_cap};
  fa.chain = chain ? 1u : 0u;
  if (defer) {
    fa.defer = 1u;
    fa.prev_idx = dfr.prev_idx;
    fa.prev_count = dfr.prev_count;
    fa.grad = grad;
    fa.fix_cap = fix_cap;
    fa.prev_tags = dfr.prev_tags;
    fa.prev_epoch = dfr.prev_epoch;
    fa.res_in = res_in;
    fa.ofs_out = (uint32_t*)(base + L.blk_ofs);
    fa.prev_ofs = dfr.prev_ws ? (const uint32_t*)((const char*)dfr.prev_ws + L.blk_ofs) : nullptr;
  }
  if (push.slot0) {
    fa.ll_base = push.slot0;
    fa.ll_epoch = push.epoch;
    fa.ll_slot_words = (uint32_t)(ll_slot_bytes(k) / sizeof(uint64_t));
  }


  void* args[] = {&fa};
  // GTK_FINISH_COOP=0: a plain (PDL) launch -- the finish's G <= #SMs blocks
  // are all resident once the main pass ahead of it has drained (A/B)
  const char* fc = getenv("GTK_FINISH_COOP");
  const bool coop = !(fc && *fc == '0');
  return coop_launch((const void*)select_finish_kernel, G, kFinishThreads, args, fin_smem, st, true, coop);
}

extern "C" int gtk_select_main_pass(const float* res_in, const float* grad, float* res_out, int64_t m, int32_t k,
                                    void* ws, size_t ws_bytes, int32_t reps, void* stream) {
  if (!grad || !res_out || !ws || reps < 1) return GTK_EINVAL;
  if (m < 1 || m >= (int64_t(1) << 31) || k < 1 || k > m) return GTK_EINVAL;
  const SelectLayout L = select_layout(m, k);
  if (ws_bytes < L.total) return GTK_ENOMEM;
  cudaStream_t st = (cudaStream_t)stream;
  char* base = (char*)ws;
  SelectCtl* ctl = (SelectCtl*)(base + L.ctl);
  EngineWS* ews = (EngineWS*)(base + L.engine);
  uint32_t* group_cnt = (uint32_t*)(base + L.group_cnt);
  const int nsm = num_sms();
  if (nsm <= 0) return GTK_ECUDA;
  // the finish grouping of select_impl (only the per-group counts depend on it)
  const uint32_t tiles_per_group = (L.ntiles + nsm - 1) / nsm;
  MainArgs ma{res_in, grad, res_out, (uint32_t)m, L.slots, L.ovf_cap, ctl,
              (uint32_t*)(base + L.tile_info), (uint32_t*)(base + L.tile_ovf), (int32_t*)(base + L.slot_idx),
              (float*)(base + L.slot_val), (int32_t*)(base + L.ovf_idx), (float*)(base + L.ovf_val),
              ews->hist[0], group_cnt, tiles_per_group};
  const uint32_t gmain = main_grid(L.ntiles, &ma.n2);
  if (gmain == 0) return GTK_ECUDA;
  for (int r = 0; r < reps; ++r) {
    select_main_kernel<kMainPlain><<<gmain, kMainThreads, kMainStageBytes, st>>>(ma);
    GTK_CHECK_LAUNCH();
  }
  // the repeated passes accumulated histogram / counter state: clear it
  GTK_CUDA(cudaMemsetAsync(ews->hist[0], 0, sizeof(uint32_t) * kHistStride, st));
  GTK_CUDA(cudaMemsetAsync(group_cnt, 0, sizeof(uint32_t) * kMaxBlocks, st));
  GTK_CUDA(cudaMemsetAsync(&ctl->ovf_cursor, 0, sizeof(ctl->ovf_cursor), st));
  GTK_CUDA(cudaMemsetAsync(&ctl->overflow, 0, sizeof(ctl->overflow), st));
  return GTK_OK;
}

__global__ void settle_kernel(float* res, const int32_t* sel_idx, const int32_t* d_count, uint32_t* window) {
  const uint32_t n = (uint32_t)__ldg(d_count);
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
    res[__ldg(sel_idx + e)] = 0.0f;
  if (blockIdx.x == 0 && threadIdx.x == 0) window[0] &= ~kRecPending;
}

// the residual after a deferred P > 1 step: +0.0 at the local winners that
// made the global list (tags == low word of *d_epoch), +0 + acc at the others
__global__ void settle_global_kernel(float* res, const int32_t* sel_idx, const int32_t* d_count, const uint32_t* tags,
                                     const uint64_t* d_epoch) {
  const uint32_t n = (uint32_t)__ldg(d_count);
  const uint32_t ep32 = (uint32_t)__ldcg((const unsigned long long*)d_epoch);
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int32_t i = __ldg(sel_idx + e);
    res[i] = __ldcg(tags + i) == ep32 ? 0.0f : __fadd_rn(0.0f, res[i]);
  }
}

extern "C" int gtk_select_settle_global(float* res, const int32_t* sel_idx, const int32_t* d_count,
                                        const uint32_t* tags, const uint64_t* d_epoch, void* stream) {
  if (!res || !sel_idx || !d_count || !tags || !d_epoch) return GTK_EINVAL;
  settle_global_kernel<<<num_sms(), 256, 0, (cudaStream_t)stream>>>(res, sel_idx, d_count, tags, d_epoch);
  GTK_CHECK_LAUNCH();
  return GTK_OK;
}

extern "C" int gtk_select_settle(float* res, const int32_t* sel_idx, const int32_t* d_count, uint32_t* d_window,
                                 void* stream) {
  if (!res || !sel_idx || !d_count || !d_window) return GTK_EINVAL;
  settle_kernel<<<num_sms(), 256, 0, (cudaStream_t)stream>>>(res, sel_idx, d_count, d_window);
  GTK_CHECK_LAUNCH();
  return GTK_OK;
}
