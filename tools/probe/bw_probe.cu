// HBM probe: what does the 2-read/1-write streaming pattern of K1's main pass
// reach on this GPU, by launch shape?  (nvcc -O3 -arch=sm_100a bw_probe.cu)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float4 ldcs(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void stcs(float* p, float4 v) { __stcs(reinterpret_cast<float4*>(p), v); }

__global__ void copy_k(const float* a, float* o, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    stcs(o + 4 * i, ldcs(a + 4 * i));
}
// one 4096-element tile per block, 4 float4 per array per thread (K1 main's shape)
__global__ void __launch_bounds__(256) add_tile(const float* a, const float* b, float* o) {
  const size_t base = (size_t)blockIdx.x * 4096;
  float4 x[4], y[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    x[q] = ldcs(a + base + (q * 256 + threadIdx.x) * 4);
    y[q] = ldcs(b + base + (q * 256 + threadIdx.x) * 4);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float4 r = make_float4(x[q].x + y[q].x, x[q].y + y[q].y, x[q].z + y[q].z, x[q].w + y[q].w);
    stcs(o + base + (q * 256 + threadIdx.x) * 4, r);
  }
}
// persistent: grid-stride over tiles, next tile's loads issued before this tile's stores
__global__ void __launch_bounds__(256) add_persist(const float* a, const float* b, float* o, int ntiles) {
  int t = blockIdx.x;
  if (t >= ntiles) return;
  float4 x[4], y[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    x[q] = ldcs(a + (size_t)t * 4096 + (q * 256 + threadIdx.x) * 4);
    y[q] = ldcs(b + (size_t)t * 4096 + (q * 256 + threadIdx.x) * 4);
  }
  for (; t < ntiles; t += gridDim.x) {
    const int tn = t + gridDim.x;
    float4 xn[4], yn[4];
    if (tn < ntiles) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        xn[q] = ldcs(a + (size_t)tn * 4096 + (q * 256 + threadIdx.x) * 4);
        yn[q] = ldcs(b + (size_t)tn * 4096 + (q * 256 + threadIdx.x) * 4);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float4 r = make_float4(x[q].x + y[q].x, x[q].y + y[q].y, x[q].z + y[q].z, x[q].w + y[q].w);
      stcs(o + (size_t)t * 4096 + (q * 256 + threadIdx.x) * 4, r);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      x[q] = xn[q];
      y[q] = yn[q];
    }
  }
}
// 8 float4 per array per thread (8192-element tiles)
__global__ void __launch_bounds__(256) add_tile8(const float* a, const float* b, float* o) {
  const size_t base = (size_t)blockIdx.x * 8192;
  float4 x[8], y[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    x[q] = ldcs(a + base + (q * 256 + threadIdx.x) * 4);
    y[q] = ldcs(b + base + (q * 256 + threadIdx.x) * 4);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float4 r = make_float4(x[q].x + y[q].x, x[q].y + y[q].y, x[q].z + y[q].z, x[q].w + y[q].w);
    stcs(o + base + (q * 256 + threadIdx.x) * 4, r);
  }
}


__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
template <int S>
__global__ void __launch_bounds__(256) add_tma(const float* a, const float* b, float* o, int ntiles) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* sa = reinterpret_cast<float*>(smem);
  float* sb = sa + S * 4096;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + S * 4096);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(full + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int G = gridDim.x;
  if (threadIdx.x == 0)
    for (int s = 0; s < S; ++s) {
      const int t = blockIdx.x + s * G;
      if (t < ntiles) {
        mbar_expect(full + s, 32768);
        bulk_g2s(sa + s * 4096, a + (size_t)t * 4096, 16384, full + s);
        bulk_g2s(sb + s * 4096, b + (size_t)t * 4096, 16384, full + s);
      }
    }
  for (int i = 0;; ++i) {
    const int t = blockIdx.x + i * G;
    if (t >= ntiles) break;
    const int s = i % S;
    mbar_wait(full + s, (uint32_t)((i / S) & 1));
    float4 x[4], y[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      x[q] = reinterpret_cast<const float4*>(sa + s * 4096)[q * 256 + threadIdx.x];
      y[q] = reinterpret_cast<const float4*>(sb + s * 4096)[q * 256 + threadIdx.x];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int tn = t + S * G;
      if (tn < ntiles) {
        mbar_expect(full + s, 32768);
        bulk_g2s(sa + s * 4096, a + (size_t)tn * 4096, 16384, full + s);
        bulk_g2s(sb + s * 4096, b + (size_t)tn * 4096, 16384, full + s);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float4 r = make_float4(x[q].x + y[q].x, x[q].y + y[q].y, x[q].z + y[q].z, x[q].w + y[q].w);
      stcs(o + (size_t)t * 4096 + (q * 256 + threadIdx.x) * 4, r);
    }
  }
}

int main() {
  const size_t m = 25600000;
  float *a, *b, *o, *big;
  cudaMalloc(&a, m * 4);
  cudaMalloc(&b, m * 4);
  cudaMalloc(&o, m * 4);
  const size_t nbig = 1ull << 29;  // 1 Gi floats... use 512 Mi floats = 2 GiB for the copy reference
  cudaMalloc(&big, nbig * 4 * 2);
  cudaMemset(a, 0, m * 4);
  cudaMemset(b, 0, m * 4);
  cudaMemset(big, 0, nbig * 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, double bytes, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    const int it = 20;
    for (int i = 0; i < it; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-34s %8.2f us  %7.1f GB/s\n", name, ms / it * 1e3, bytes / (ms / it * 1e-3) / 1e9);
  };
  run("copy 4 GiB (1R1W), grid 16x", 2.0 * nbig * 4, [&] { copy_k<<<sms * 16, 256>>>(big, big + nbig, nbig / 4); });
  run("copy 102 MB (1R1W), grid 16x", 2.0 * m * 4, [&] { copy_k<<<sms * 16, 256>>>(a, o, m / 4); });
  run("add 2R1W tile/block 4096", 3.0 * m * 4, [&] { add_tile<<<m / 4096, 256>>>(a, b, o); });
  run("add 2R1W tile/block 8192", 3.0 * m * 4, [&] { add_tile8<<<m / 8192, 256>>>(a, b, o); });
  for (int per : {2, 3, 4, 6, 8})
    run(per == 2 ? "add 2R1W persistent 2/SM" : per == 3 ? "add 2R1W persistent 3/SM" : per == 4 ? "add 2R1W persistent 4/SM" : per == 6 ? "add 2R1W persistent 6/SM" : "add 2R1W persistent 8/SM",
        3.0 * m * 4, [&] { add_persist<<<sms * per, 256>>>(a, b, o, (int)(m / 4096)); });
  {
    auto go = [&](auto kern, int S, int per) {
      const size_t sm = (size_t)S * 32768 + 64;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      char name[64];
      snprintf(name, sizeof name, "add 2R1W TMA S=%d %d/SM", S, per);
      run(name, 3.0 * m * 4, [&] { kern<<<sms * per, 256, sm>>>(a, b, o, (int)(m / 4096)); });
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) printf("  %s\n", cudaGetErrorString(e));
    };
    go(add_tma<2>, 2, 3);
    go(add_tma<3>, 3, 2);
    go(add_tma<4>, 4, 1);
    go(add_tma<6>, 6, 1);
    go(add_tma<2>, 2, 2);
    go(add_tma<3>, 3, 1);
  }
  return 0;
}
