// K2: the sparse top-k merge operator ⊤ (reference sparse.py:157-195) as one
// cooperative launch; the algorithm lives in gtk_merge.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "gtk_internal.h"
#include "gtk_merge.cuh"

namespace gtk {

template <bool kSolo>
__global__ void __launch_bounds__(kMergeThreads, 1) merge_kernel(MergeArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  MergeSmem& S = *reinterpret_cast<MergeSmem*>(dsm);
  grid_sync_begin(&a.ews->bar);
  const uint32_t na = (uint32_t)__ldcg(a.d_na), nb = (uint32_t)__ldcg(a.d_nb);
  const uint32_t ha = (uint32_t)__ldcg(a.d_na + 1), hb = (uint32_t)__ldcg(a.d_nb + 1);
  merge_device<kSolo>(a, na, nb, ha, hb, gridDim.x, S);
}

// Grid of a merge over two lists of <= cap entries.
//  * cluster (default while the union fits the shared memory of <= 16 CTAs):
//    one thread-block cluster of G CTAs, ~kMergeClusterSlots union slots each;
//    the engine's barriers are barrier.cluster (~0.2 us) instead of the
//    global-atomic grid barrier (~2-5 us with block skew).
//  * cooperative grid: ~512 merged slots per block (the engine's phases are
//    latency-bound, more blocks shorten each: measured 2048 -> 512 takes
//    k = 25.6K from 21 to 16.5 us), at most one block per SM.
// Either way the slice capacity covers the expected slice up to
// kMergeSliceCapMax.  GTK_MERGE_GRID=n / GTK_MERGE_CLUSTER=0|1 override the
// choice (measurements).
static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

static bool cluster_fits(const void* func, int cs, size_t smem) {
  static std::mutex mu;
  static std::unordered_map<unsigned long long, bool> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  const unsigned long long key = ((unsigned long long)(uintptr_t)func) ^ ((unsigned long long)dev << 56) ^
                                 ((unsigned long long)cs << 40) ^ (unsigned long long)smem;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  bool ok = true;
  if (cs > 8 && cudaFuncSetAttribute(func, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) ok = false;
  if (ok) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kMergeThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cs;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    ok = cudaOccupancyMaxActiveClusters(&n, func, &cfg) == cudaSuccess && n >= 1;
  }
  cudaGetLastError();  // a refused size is an answer, not an error
  cache[key] = ok;
  return ok;
}

bool merge_grid_for(const void* func, int32_t cap, MergeGrid* out, int compact_g) {
  if (!ensure_dyn_smem(func, merge_smem_bytes(kMergeSliceCapMax))) return false;
  const int lim = num_sms();
  if (lim <= 0) return false;
  const uint64_t slots = 2ull * (uint64_t)(cap < 1 ? 1 : cap);
  const int force_g = env_int("GTK_MERGE_GRID", 0), force_c = env_int("GTK_MERGE_CLUSTER", -1);
  if (env_int("GTK_MERGE_COMPACT", 1) == 0) compact_g = 0;
  auto cap_for = [&](int g) {
    const uint64_t per = (slots + g - 1) / g;
    uint32_t sc = kMergeSliceCap;
    if (per > sc) sc = (uint32_t)std::min<uint64_t>((per + 255) & ~255ull, kMergeSliceCapMax);
    return sc;
  };
  if (compact_g > 0) {
    // a merge sharing the GPU with an HBM pass: at most compact_g blocks of a
    // cooperative grid (schedulable on whichever SMs are free -- a cluster
    // needs a whole GPC free, which the running finish blocks deny: measured
    // N = 2 16-CTA cluster 86.4 us/step vs 32-block grid 78.1).
    // GTK_MERGE_COMPACT_G / GTK_MERGE_COMPACT_CLUSTER override (A/B)
    const int cg = std::max(1, std::min(env_int("GTK_MERGE_COMPACT_G", compact_g), lim));
    const bool as_cluster = env_int("GTK_MERGE_COMPACT_CLUSTER", 0) != 0 && cg <= kMergeMaxCluster;
    const uint64_t want_c0 = slots <= (uint64_t)kMergeSoloSlots ? 1 : (slots + kMergeClusterSlots - 1) / kMergeClusterSlots;
    const int g = (int)std::min<uint64_t>(want_c0, (uint64_t)cg);
    if ((slots + g - 1) / g <= (uint64_t)kMergeSliceCapMax) {
      const uint32_t sc = cap_for(g);
      if (g == 1) {
        *out = MergeGrid{1, sc, false};
        return true;
      }
      if (as_cluster && cluster_fits(func, g, merge_smem_bytes(sc))) {
        *out = MergeGrid{g, sc, true};
        return true;
      }
      if (!as_cluster && coop_grid(func, kMergeThreads, merge_smem_bytes(sc)) >= g) {
        *out = MergeGrid{g, sc, false, env_int("GTK_MERGE_COMPACT_COOP", 1) != 0};
        return true;
      }
    }
  }
  // cluster candidate
  const uint64_t want_c = slots <= (uint64_t)kMergeSoloSlots ? 1 : (slots + kMergeClusterSlots - 1) / kMergeClusterSlots;
  int gc = (int)std::min<uint64_t>(want_c, kMergeMaxCluster);
  if (force_g > 0) gc = std::min(force_g, kMergeMaxCluster);
  if (gc < 1) gc = 1;
  const bool c_smem = (slots + gc - 1) / gc <= (uint64_t)kMergeSliceCapMax;
  // cluster mode only where the union spreads over <= 16 CTAs at the target density
  bool use_cluster = force_c != 0 && c_smem && (force_g > 0 ? force_g <= kMergeMaxCluster
                                                             : (force_c == 1 || want_c <= (uint64_t)kMergeMaxCluster));
  if (force_c == 1 && !c_smem) return false;
  if (use_cluster) {
    const uint32_t sc = cap_for(gc);
    if (gc == 1 || cluster_fits(func, gc, merge_smem_bytes(sc))) {
      *out = MergeGrid{gc, sc, gc > 1};
      return true;
    }
    if (force_c == 1) return false;
  }
  const int want = (int)((slots + kMergeSlotsPerBlock - 1) / kMergeSlotsPerBlock);
  int g = force_g > 0 ? force_g : (want < lim ? (want < 1 ? 1 : want) : lim);
  if (g > kMaxBlocks) g = kMaxBlocks;
  const uint32_t sc = cap_for(g);
  const int co = coop_grid(func, kMergeThreads, merge_smem_bytes(sc));
  if (co <= 0) return false;
  if (g > co) g = co;
  *out = MergeGrid{g, sc, false};
  return true;
}

bool merge_use_solo(const MergeGrid& g, int32_t cap) {
  // GTK_MERGE_SOLO=0: the generic engine on one CTA too (A/B)
  static const bool on = env_int("GTK_MERGE_SOLO", 1) != 0;
  return on && g.G == 1 && !g.cluster && 2ull * (uint64_t)(cap < 1 ? 1 : cap) <= kSoloMaxSlots;
}

int merge_launch(const void* func, const MergeGrid& g, void** args, size_t smem, cudaStream_t st, bool pdl) {
  if (!g.cluster) return coop_launch(func, g.G, kMergeThreads, args, smem, st, pdl, g.coop);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g.G);
  cfg.blockDim = dim3(kMergeThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = g.G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 2 : 1;
  const cudaError_t e = cudaLaunchKernelExC(&cfg, func, args);
  if (e != cudaSuccess) {
    set_last_cuda_error(e);
    return GTK_ECUDA;
  }
  count_launch();
  return GTK_OK;
}

int launch_merge(const MergeArgs& args, int32_t cap, cudaStream_t st) {
  MergeGrid g;
  if (!merge_grid_for((const void*)merge_kernel<false>, cap, &g)) return GTK_ECUDA;
  const void* fn = merge_use_solo(g, cap) ? (const void*)merge_kernel<true> : (const void*)merge_kernel<false>;
  if (!ensure_dyn_smem(fn, merge_smem_bytes(kMergeSliceCapMax))) return GTK_ECUDA;
  MergeArgs a = args;
  a.slice_cap = g.slice_cap;
  void* p[] = {&a};
  ProfScope prof(kProfMerge, st);
  return merge_launch(fn, g, p, merge_smem_bytes(g.slice_cap), st, false);
}

}  // namespace gtk

using namespace gtk;

extern "C" int gtk_merge_workspace_bytes(int32_t cap, int32_t k, size_t* bytes) {
  if (!bytes || cap < 0 || k < 1) return GTK_EINVAL;
  *bytes = merge_layout(cap < 1 ? 1 : cap).total;
  return GTK_OK;
}

extern "C" int gtk_top_op(const int32_t* a_idx, const float* a_val, const int32_t* d_na, const int32_t* b_idx,
                          const float* b_val, const int32_t* d_nb, int32_t cap, int32_t k, int32_t* o_idx,
                          float* o_val, int32_t* d_no, void* ws, size_t ws_bytes, void* stream) {
  if (!d_na || !d_nb || !o_idx || !o_val || !d_no || !ws || cap < 0 || k < 1) return GTK_EINVAL;
  const MergeLayout L = merge_layout(cap < 1 ? 1 : cap);
  if (ws_bytes < L.total) return GTK_ENOMEM;
  char* base = (char*)ws;
  MergeArgs args{a_idx, a_val, d_na, b_idx, b_val, d_nb, (uint32_t)k, o_idx, o_val, d_no,
                 (MergeCtl*)(base + L.ctl), (EngineWS*)(base + L.engine), (int32_t*)(base + L.u_idx),
                 (float*)(base + L.u_val), trace_buffer() ? trace_buffer() + 32 : nullptr};
  return launch_merge(args, cap < 1 ? 1 : cap, (cudaStream_t)stream);
}
