// K2: the sparse top-k merge operator ⊤ (reference sparse.py:157-195) as one
// cooperative launch; the algorithm lives in gtk_merge.cuh.
#include <cuda_runtime.h>

#include <algorithm>

#include "gtk_internal.h"
#include "gtk_merge.cuh"

namespace gtk {

__global__ void __launch_bounds__(kMergeThreads, 1) merge_kernel(MergeArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  MergeSmem& S = *reinterpret_cast<MergeSmem*>(dsm);
  const uint32_t na = (uint32_t)__ldcg(a.d_na), nb = (uint32_t)__ldcg(a.d_nb);
  const uint32_t ha = (uint32_t)__ldcg(a.d_na + 1), hb = (uint32_t)__ldcg(a.d_nb + 1);
  merge_device(a, na, nb, ha, hb, gridDim.x, S);
}

// blocks and shared-memory slice capacity for a merge of two lists of <= cap
// entries: ~512 merged slots per block (the engine's phases are latency-bound,
// more blocks shorten each: measured 2048 -> 512 takes k = 25.6K from 21 to
// 16.5 us), at most one block per SM; the slice capacity covers the expected
// slice (large k) up to kMergeSliceCapMax
int merge_grid_for(const void* func, int32_t cap, uint32_t* slice_cap) {
  if (!ensure_dyn_smem(func, merge_smem_bytes(kMergeSliceCapMax))) return 0;
  const int lim = num_sms();
  if (lim <= 0) return 0;
  const int want = (int)((2LL * cap + kMergeSlotsPerBlock - 1) / kMergeSlotsPerBlock);
  int g = want < lim ? (want < 1 ? 1 : want) : lim;
  if (g > kMaxBlocks) g = kMaxBlocks;
  const uint64_t per = (2ull * (uint64_t)cap + g - 1) / g;
  uint32_t sc = kMergeSliceCap;
  if (per > sc) sc = (uint32_t)std::min<uint64_t>((per + 255) & ~255ull, kMergeSliceCapMax);
  const int co = coop_grid(func, kMergeThreads, merge_smem_bytes(sc));
  if (co <= 0) return 0;
  if (g > co) g = co;
  *slice_cap = sc;
  return g;
}

int launch_merge(const MergeArgs& args, int32_t cap, cudaStream_t st) {
  uint32_t sc = 0;
  const int G = merge_grid_for((const void*)merge_kernel, cap, &sc);
  if (G <= 0) return GTK_ECUDA;
  MergeArgs a = args;
  a.slice_cap = sc;
  void* p[] = {&a};
  ProfScope prof(kProfMerge, st);
  return coop_launch((const void*)merge_kernel, G, kMergeThreads, p, merge_smem_bytes(sc), st);
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
