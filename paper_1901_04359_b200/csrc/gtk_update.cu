// K3: global top-k -> model update + extra residuals (reference
// optimizer.py:227-230, :243, :92-105), plus the densify / TopKAllReduce /
// dense-sum helpers of the baselines (sparse.py:198-202, collectives.py:158-164,
// optimizer.py:108-115).
//
// Bit-exactness of the sparse update: the reference computes
// u = densify(g)/FLOAT(P) densely and w -= FLOAT(lr)*u.  At untouched slots
// u = +0, FLOAT(lr)*(+0) = +0 for finite lr with the sign bit clear, and
// w - (+0) == w bitwise (including w = -0), so only the k touched slots change.
// For any other lr (negative, -0, inf, nan) or momentum > 0 the dense kernel
// runs instead.  All arithmetic uses explicit _rn intrinsics (no FMA
// contraction), matching numpy's single-op fp32 rounding.
#include <cuda_runtime.h>

#include <cmath>

#include "gtk_common.cuh"
#include "gtk_internal.h"

namespace gtk {

constexpr int kUpdThreads = 256;
constexpr int kDenseTile = 4096;  // elements per block in the dense update

__device__ __forceinline__ bool sorted_contains(const int32_t* a, uint32_t n, int32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const int32_t y = __ldg(a + mid);
    if (y < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < n && __ldg(a + lo) == x;
}

// sparse path: global entries update w; local entries outside the global set
// return to the residual.
__device__ __forceinline__ bool skipped(const uint32_t* d_skip) {
  return d_skip && (__ldcg(d_skip) & GTK_DEV_ERROR_MASK);
}

__global__ void __launch_bounds__(kUpdThreads)
    scatter_update_kernel(float* w, float* res, const int32_t* g_idx, const float* g_val, const int32_t* d_gn,
                          const int32_t* l_idx, const float* l_val, const int32_t* d_ln, float lr, float Pf,
                          int scaling, int do_weights, const uint32_t* d_skip) {
  pdl_wait();  // launched programmatically behind the exchange / select
  pdl_launch_dependents();
  if (skipped(d_skip)) return;
  const uint32_t gn = (uint32_t)__ldg(d_gn);
  const uint32_t ln = l_idx ? (uint32_t)__ldg(d_ln) : 0u;
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (do_weights) {
    for (uint32_t e = tid; e < gn; e += stride) {
      const int32_t i = __ldg(g_idx + e);
      const float u = scale_u(__ldg(g_val + e), Pf, scaling);
      w[i] = __fsub_rn(w[i], __fmul_rn(lr, u));
    }
  }
  for (uint32_t e = tid; e < ln; e += stride) {
    const int32_t i = __ldg(l_idx + e);
    if (!sorted_contains(g_idx, gn, i)) res[i] = __fadd_rn(res[i], __ldg(l_val + e));
  }
}

// dense path (momentum > 0 or an lr for which the sparse form is not exact):
// each block stages the global entries of its tile into shared memory.
__global__ void __launch_bounds__(kUpdThreads)
    dense_update_kernel(float* w, float* vel, const int32_t* g_idx, const float* g_val, const int32_t* d_gn,
                        uint32_t m, float lr, float mom, float Pf, int scaling, const uint32_t* d_skip) {
  __shared__ float su[kDenseTile];
  __shared__ uint32_t s_rng[2];
  pdl_wait();
  pdl_launch_dependents();
  if (skipped(d_skip)) return;
  const uint32_t gn = (uint32_t)__ldg(d_gn);
  const uint32_t t0 = blockIdx.x * kDenseTile;
  const uint32_t t1 = min(m, t0 + kDenseTile);
  for (int j = threadIdx.x; j < kDenseTile; j += kUpdThreads) su[j] = 0.0f;
  if (threadIdx.x < 2) {
    const int32_t x = (int32_t)(threadIdx.x == 0 ? t0 : t1);
    uint32_t lo = 0, hi = gn;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(g_idx + mid) < x) lo = mid + 1;
      else hi = mid;
    }
    s_rng[threadIdx.x] = lo;
  }
  __syncthreads();
  for (uint32_t e = s_rng[0] + threadIdx.x; e < s_rng[1]; e += kUpdThreads)
    su[__ldg(g_idx + e) - t0] = scale_u(__ldg(g_val + e), Pf, scaling);
  __syncthreads();
  for (uint32_t e = t0 + threadIdx.x; e < t1; e += kUpdThreads) {
    float u = su[e - t0];
    if (vel) {
      const float v2 = __fadd_rn(__fmul_rn(mom, vel[e]), u);
      vel[e] = v2;
      u = v2;
    }
    w[e] = __fsub_rn(w[e], __fmul_rn(lr, u));
  }
}

__device__ __forceinline__ float dense_apply_one(float w, float* vel_e, float u, float lr, float mom, float Pf,
                                                 bool divide) {
  if (divide) u = __fdiv_rn(u, Pf);
  if (vel_e) {
    u = __fadd_rn(__fmul_rn(mom, *vel_e), u);
    *vel_e = u;
  }
  return __fsub_rn(w, __fmul_rn(lr, u));
}

// elements [0, m4*4) as float4 (the host checks 16-byte alignment of all
// three arrays), [m4*4, m) scalar: 12 B/element (20 with momentum), one pass
__global__ void dense_apply_kernel(float* w, float* vel, const float* upd, uint32_t m, uint32_t m4, float lr,
                                   float mom, float Pf, int divide) {
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t t0 = blockIdx.x * blockDim.x + threadIdx.x;
  float4* w4 = reinterpret_cast<float4*>(w);
  float4* v4 = reinterpret_cast<float4*>(vel);
  const float4* u4 = reinterpret_cast<const float4*>(upd);
  for (uint32_t q = t0; q < m4; q += stride) {
    const float4 u = __ldcs(u4 + q);
    float4 x = w4[q];
    if (vel) {
      float4 v = v4[q];
      x.x = dense_apply_one(x.x, &v.x, u.x, lr, mom, Pf, divide);
      x.y = dense_apply_one(x.y, &v.y, u.y, lr, mom, Pf, divide);
      x.z = dense_apply_one(x.z, &v.z, u.z, lr, mom, Pf, divide);
      x.w = dense_apply_one(x.w, &v.w, u.w, lr, mom, Pf, divide);
      v4[q] = v;
    } else {
      x.x = dense_apply_one(x.x, nullptr, u.x, lr, mom, Pf, divide);
      x.y = dense_apply_one(x.y, nullptr, u.y, lr, mom, Pf, divide);
      x.z = dense_apply_one(x.z, nullptr, u.z, lr, mom, Pf, divide);
      x.w = dense_apply_one(x.w, nullptr, u.w, lr, mom, Pf, divide);
    }
    w4[q] = x;
  }
  for (uint32_t e = m4 * 4 + t0; e < m; e += stride)
    w[e] = dense_apply_one(w[e], vel ? vel + e : nullptr, upd[e], lr, mom, Pf, divide);
}

__global__ void scatter_kernel(const int32_t* idx, const float* val, const int32_t* d_n, float* out) {
  const uint32_t n = (uint32_t)__ldg(d_n);
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
    out[__ldg(idx + e)] = __ldg(val + e);
}

__global__ void scatter_add_kernel(const int32_t* idx, const float* val, const int32_t* d_n, float* out) {
  const uint32_t n = (uint32_t)__ldg(d_n);
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int32_t i = __ldg(idx + e);
    out[i] = __fadd_rn(out[i], __ldg(val + e));
  }
}

// entry e of rank r is an index's first occurrence unless an earlier rank's
// (ascending) list holds the same index: each touched index is handled by
// exactly one thread
__device__ __forceinline__ bool first_occurrence(const int32_t* idx, const int32_t* d_n, int32_t r, int64_t stride,
                                                 int32_t i) {
  for (int32_t s = 0; s < r; ++s) {
    const int32_t* a = idx + (uint64_t)s * stride;
    const uint32_t n = (uint32_t)__ldg(d_n + s);
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(a + mid) < i) lo = mid + 1;
      else hi = mid;
    }
    if (lo < n && __ldg(a + lo) == i) return false;
  }
  return true;
}

// out /= P at the touched entries only (untouched ones are +0 and +0 / P is
// +0): each index exactly once, like the reference's dense division
// (collectives.py:164), at P x k instead of m elements
__global__ void divide_touched_kernel(const int32_t* idx, const int32_t* d_n, int32_t P, int64_t stride, float* out,
                                      float Pf) {
  const uint64_t tot = (uint64_t)P * (uint64_t)stride;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < tot; q += (uint64_t)gridDim.x * blockDim.x) {
    const int32_t r = (int32_t)(q / (uint64_t)stride);
    const uint32_t e = (uint32_t)(q % (uint64_t)stride);
    if (e >= (uint32_t)__ldg(d_n + r)) continue;
    const int32_t i = __ldg(idx + (uint64_t)r * stride + e);
    if (first_occurrence(idx, d_n, r, stride, i)) out[i] = __fdiv_rn(out[i], Pf);
  }
}

// the topk baseline's update at momentum 0 (optimizer.py:92-99 with the
// averaged vector of collectives.py:158-165): w -= lr * (sum / P) at the
// touched entries only -- untouched entries would subtract lr * +0, which
// leaves every w bitwise unchanged -- and the rank-ordered sums in `acc` are
// reset to +0 for the next call
// any of the P status words (stride `sstride`) carries an error bit: the
// step is void on every rank (nothing is added or applied)
__device__ __forceinline__ bool any_rank_failed(const int32_t* d_st, int32_t P, int64_t sstride) {
  if (!d_st) return false;
  for (int32_t r = 0; r < P; ++r)
    if (__ldcg(d_st + (uint64_t)r * sstride) & GTK_DEV_ERROR_MASK) return true;
  return false;
}

__global__ void scatter_add_guarded_kernel(const int32_t* idx, const float* val, const int32_t* d_n, float* out,
                                           const int32_t* d_st, int32_t P, int64_t sstride) {
  if (any_rank_failed(d_st, P, sstride)) return;
  const uint32_t n = (uint32_t)__ldg(d_n);
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int32_t i = __ldg(idx + e);
    out[i] = __fadd_rn(out[i], __ldg(val + e));
  }
}

__global__ void apply_touched_kernel(const int32_t* idx, const int32_t* d_n, int32_t P, int64_t stride, float* acc,
                                     float* w, float lr, float Pf, int divide, const int32_t* d_st, int64_t sstride,
                                     int32_t* d_local) {
  if (any_rank_failed(d_st, P, sstride)) {
    // a healthy rank learns that a peer's selection failed (the failing
    // rank's own word already carries its error)
    if (blockIdx.x == 0 && threadIdx.x == 0 && d_local && !(*d_local & GTK_DEV_ERROR_MASK))
      atomicOr(d_local, GTK_DEV_PEER_FAILED);
    return;
  }
  const uint64_t tot = (uint64_t)P * (uint64_t)stride;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < tot; q += (uint64_t)gridDim.x * blockDim.x) {
    const int32_t r = (int32_t)(q / (uint64_t)stride);
    const uint32_t e = (uint32_t)(q % (uint64_t)stride);
    if (e >= (uint32_t)__ldg(d_n + r)) continue;
    const int32_t i = __ldg(idx + (uint64_t)r * stride + e);
    if (!first_occurrence(idx, d_n, r, stride, i)) continue;
    float u = acc[i];
    if (divide) u = __fdiv_rn(u, Pf);
    w[i] = __fsub_rn(w[i], __fmul_rn(lr, u));
    acc[i] = 0.0f;
  }
}

__global__ void dense_sum_kernel(const float* const* srcs, int P, uint32_t m, float* out) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    float acc = 0.0f;
    for (int r = 0; r < P; ++r) acc = __fadd_rn(acc, srcs[r][e]);
    out[e] = acc;
  }
}

// the reference's ring reduce-scatter order (collectives.py:119-122): element
// e lies in chunk c = e / chunk, whose sum starts at rank c's value and takes
// ranks c+1, c+2, ... (mod P) in turn -- bitwise the ring's result
__global__ void dense_ring_sum_kernel(const float* const* srcs, int P, uint32_t m, uint32_t chunk, float* out) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const int c = (int)(e / chunk);
    float acc = srcs[c][e];
    for (int j = 1; j < P; ++j) {
      const int r = c + j < P ? c + j : c + j - P;
      acc = __fadd_rn(acc, srcs[r][e]);
    }
    out[e] = acc;
  }
}

static int grid_for(uint64_t n, int threads) {
  uint64_t g = (n + threads - 1) / threads;
  const uint64_t cap = (uint64_t)num_sms() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace gtk

using namespace gtk;

extern "C" int gtk_scatter_update(float* w, float* res, float* vel, const int32_t* g_idx, const float* g_val,
                                  const int32_t* d_gn, const int32_t* l_idx, const float* l_val,
                                  const int32_t* d_ln, int64_t m, float lr, float momentum, int32_t P,
                                  int32_t scaling, const uint32_t* d_skip, void* stream) {
  if (!w || !g_idx || !g_val || !d_gn || m < 1 || m >= (int64_t(1) << 31) || P < 1) return GTK_EINVAL;
  if (scaling < 0 || scaling > 2) return GTK_EINVAL;
  if (l_idx && (!l_val || !d_ln || !res)) return GTK_EINVAL;
  if (momentum > 0.0f && !vel) return GTK_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const float Pf = (float)P;
  // the local list IS the global list (P = 1): no entry can miss the global set
  if (l_idx == g_idx && l_val == g_val && d_ln == d_gn) l_idx = nullptr;
  const bool sparse_exact = momentum == 0.0f && std::isfinite(lr) && !std::signbit(lr);
  ProfScope prof(kProfUpdate, st);
  if (!sparse_exact) {
    const int tiles = (int)((m + kDenseTile - 1) / kDenseTile);
    GTK_CUDA(launch_pdl(dense_update_kernel, dim3(tiles), dim3(kUpdThreads), 0, st, w,
                        momentum > 0.0f ? vel : nullptr, g_idx, g_val, d_gn, (uint32_t)m, lr, momentum, Pf, scaling,
                        d_skip));
    GTK_CHECK_LAUNCH();
    if (l_idx) {
      scatter_update_kernel<<<num_sms() * 2, kUpdThreads, 0, st>>>(w, res, g_idx, g_val, d_gn, l_idx, l_val, d_ln,
                                                                    lr, Pf, scaling, 0, d_skip);
      GTK_CHECK_LAUNCH();
    }
    return GTK_OK;
  }
  // k-length work: one launch updates w at the global entries and returns the
  // local entries that missed the global set to the residual
  GTK_CUDA(launch_pdl(scatter_update_kernel, dim3(num_sms() * 2), dim3(kUpdThreads), 0, st, w, res, g_idx, g_val,
                      d_gn, l_idx, l_val, d_ln, lr, Pf, scaling, 1, d_skip));
  GTK_CHECK_LAUNCH();
  return GTK_OK;
}

extern "C" int gtk_dense_apply(float* w, float* vel, const float* upd, int64_t m, float lr, float momentum,
                               int32_t divide_by, void* stream) {
  if (!w || !upd || m < 1 || m >= (int64_t(1) << 31) || divide_by < 0) return GTK_EINVAL;
  if (momentum > 0.0f && !vel) return GTK_EINVAL;
  float* v = momentum > 0.0f ? vel : nullptr;
  const bool aligned = ((uintptr_t)w | (uintptr_t)upd | (uintptr_t)v) % 16 == 0;
  const uint32_t m4 = aligned ? (uint32_t)(m / 4) : 0;
  dense_apply_kernel<<<grid_for(aligned ? (uint64_t)m4 : (uint64_t)m, 256), 256, 0, (cudaStream_t)stream>>>(
      w, v, upd, (uint32_t)m, m4, lr, momentum, (float)divide_by, divide_by > 0);
  GTK_CHECK_LAUNCH();
  return GTK_OK;
}

extern "C" int gtk_densify(const int32_t* idx, const float* val, const int32_t* d_n, int64_t m, float* out,
                           void* stream) {
  if (!idx || !val || !d_n || !out || m < 1 || m >= (int64_t(1) << 31)) return GTK_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  GTK_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * (size_t)m, st));
  scatter_kernel<<<num_sms() * 2, 256, 0, st>>>(idx, val, d_n, out);
  GTK_CHECK_LAUNCH();
  return GTK_OK;
}

extern "C" int gtk_topk_accumulate(const int32_t* idx, const float* val, const int32_t* d_n, int32_t P,
                                   int64_t stride, int64_t m, float* out, int32_t divide, void* stream) {
  if (!idx || !val || !d_n || !out || P < 1 || m < 1 || m >= (int64_t(1) << 31) || stride < 0)
    return GTK_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  GTK_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * (size_t)m, st));
  for (int r = 0; r < P; ++r) {  // rank order 0..P-1 (collectives.py:162-163)
    scatter_add_kernel<<<num_sms() * 2, 256, 0, st>>>(idx + r * stride, val + r * stride, d_n + r, out);
    GTK_CHECK_LAUNCH();
  }
  if (divide) {
    divide_touched_kernel<<<num_sms() * 2, 256, 0, st>>>(idx, d_n, P, stride, out, (float)P);
    GTK_CHECK_LAUNCH();
  }
  return GTK_OK;
}

extern "C" int gtk_topk_apply(const int32_t* idx, const float* val, const int32_t* d_n, int32_t P, int64_t stride,
                              int64_t m, float* acc, float* w, float lr, int32_t divide, const int32_t* d_status,
                              int64_t status_stride, int32_t* d_local_status, void* stream) {
  if (!idx || !val || !d_n || !acc || !w || P < 1 || m < 1 || m >= (int64_t(1) << 31) || stride < 0 ||
      status_stride < 0)
    return GTK_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  for (int r = 0; r < P; ++r) {  // rank order 0..P-1 (collectives.py:162-163), into the all-+0 acc
    scatter_add_guarded_kernel<<<num_sms() * 2, 256, 0, st>>>(idx + r * stride, val + r * stride, d_n + r, acc,
                                                             d_status, P, status_stride);
    GTK_CHECK_LAUNCH();
  }
  apply_touched_kernel<<<num_sms() * 2, 256, 0, st>>>(idx, d_n, P, stride, acc, w, lr, (float)P, divide, d_status,
                                                      status_stride, d_local_status);
  GTK_CHECK_LAUNCH();
  return GTK_OK;
}

// measure_divergence (optimizer.py:232-241): for every global entry i the
// pruned mass total[g_idx[i]] - g_val[i] (the reference's masked sum minus
// densify(global) at the mask, optimizer.py:238-240), and the number of global
// indices also in the naive list (|shared| of _mask_divergence, :192-196):
// one binary search per entry in the index-sorted naive list, warp-aggregated
__global__ void divergence_kernel(const int32_t* g_idx, const float* g_val, const int32_t* d_gn,
                                  const int32_t* n_idx, const int32_t* d_nn, const float* total, float* pruned,
                                  uint32_t* d_shared) {
  const uint32_t gn = (uint32_t)__ldg(d_gn), nn = (uint32_t)__ldg(d_nn);
  for (uint32_t base = blockIdx.x * blockDim.x; base < gn; base += gridDim.x * blockDim.x) {
    const uint32_t e = base + threadIdx.x;
    bool hit = false;
    if (e < gn) {
      const int32_t i = g_idx[e];
      pruned[e] = __fsub_rn(total[i], g_val[e]);
      uint32_t lo = 0, hi = nn;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (n_idx[mid] < i) lo = mid + 1;
        else hi = mid;
      }
      hit = lo < nn && n_idx[lo] == i;
    }
    const unsigned bal = __ballot_sync(0xFFFFFFFFu, hit);
    if ((threadIdx.x & 31) == 0 && bal) atomicAdd(d_shared, (uint32_t)__popc(bal));
  }
}

extern "C" int gtk_divergence_terms(const int32_t* g_idx, const float* g_val, const int32_t* d_gn,
                                    const int32_t* n_idx, const int32_t* d_nn, const float* total, int64_t m,
                                    float* pruned, uint32_t* d_shared, void* stream) {
  if (!g_idx || !g_val || !d_gn || !n_idx || !d_nn || !total || !pruned || !d_shared || m < 1 ||
      m >= (int64_t(1) << 31))
    return GTK_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  GTK_CUDA(cudaMemsetAsync(d_shared, 0, sizeof(uint32_t), st));
  divergence_kernel<<<num_sms() * 2, 256, 0, st>>>(g_idx, g_val, d_gn, n_idx, d_nn, total, pruned, d_shared);
  GTK_CHECK_LAUNCH();
  return GTK_OK;
}

// the step's one host round trip: status word and count -> pinned host pair
// (then, with reset, the status word back to 0 for the next step), synchronised
extern "C" int gtk_status_read(const int32_t* d_status, const int32_t* d_count, int32_t* h_out, int32_t reset,
                               void* stream) {
  if (!d_status || !d_count || !h_out) return GTK_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  GTK_CUDA(cudaMemcpyAsync(h_out, d_status, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GTK_CUDA(cudaMemcpyAsync(h_out + 1, d_count, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  if (reset) GTK_CUDA(cudaMemsetAsync(const_cast<int32_t*>(d_status), 0, sizeof(int32_t), st));
  GTK_CUDA(cudaStreamSynchronize(st));
  return GTK_OK;
}

extern "C" int gtk_dense_ring_sum(const float* const* srcs, int32_t P, int64_t m, float* out, void* stream) {
  if (!srcs || !out || P < 1 || m < 1 || m >= (int64_t(1) << 31)) return GTK_EINVAL;
  const int64_t chunk = (m + P - 1) / P;
  dense_ring_sum_kernel<<<grid_for(m, 256), 256, 0, (cudaStream_t)stream>>>(srcs, P, (uint32_t)m, (uint32_t)chunk,
                                                                             out);
  GTK_CHECK_LAUNCH();
  return GTK_OK;
}

extern "C" int gtk_dense_sum(const float* const* srcs, int32_t P, int64_t m, float* out, void* stream) {
  if (!srcs || !out || P < 1 || m < 1 || m >= (int64_t(1) << 31)) return GTK_EINVAL;
  dense_sum_kernel<<<grid_for(m, 256), 256, 0, (cudaStream_t)stream>>>(srcs, P, (uint32_t)m, out);
  GTK_CHECK_LAUNCH();
  return GTK_OK;
}
