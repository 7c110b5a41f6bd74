// Primitive latencies on one B200 (clock64 cycles, block 0 thread 0):
//   load   one load per thread (512 threads) of an L2-resident buffer, then
//          __syncthreads: ld.global.cg u32, ld.relaxed.gpu v2.u64,
//          ld.relaxed.sys v2.u64, 4 independent ld.relaxed.sys v2.u64
//   gridbar  the repo's grid barrier (acq_rel arrival, release add, acquire poll)
//            over G blocks, per barrier
//   clusterbar barrier.cluster over a 16-CTA cluster, per barrier
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_probe tools/probe/lat_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld_sys(const uint64_t* p, uint64_t& x, uint64_t& y) {
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(p) : "memory");
}
__device__ __forceinline__ void ld_gpu(const uint64_t* p, uint64_t& x, uint64_t& y) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(p) : "memory");
}

__global__ void load_kernel(const uint64_t* buf, long long* out, int reps) {
  __shared__ uint64_t sink[512];
  const uint64_t* b = buf + 2 * (size_t)blockIdx.x * 4 * 512;
  long long t[6];
  uint64_t acc = 0;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    t[0] = clock64();
    acc += __ldcg((const unsigned*)b + threadIdx.x);
    __syncthreads();
    sink[threadIdx.x] = acc;
    __syncthreads();
    t[1] = clock64();
    uint64_t x, y;
    ld_gpu(b + 2 * threadIdx.x, x, y);
    acc += x ^ y;
    sink[threadIdx.x] = acc;
    __syncthreads();
    t[2] = clock64();
    ld_sys(b + 2 * threadIdx.x, x, y);
    acc += x ^ y;
    sink[threadIdx.x] = acc;
    __syncthreads();
    t[3] = clock64();
    uint64_t x1, y1, x2, y2, x3, y3;
    ld_sys(b + 2 * threadIdx.x, x, y);
    ld_sys(b + 2 * (threadIdx.x + 512), x1, y1);
    ld_sys(b + 2 * (threadIdx.x + 1024), x2, y2);
    ld_sys(b + 2 * (threadIdx.x + 1536), x3, y3);
    acc += x ^ y ^ x1 ^ y1 ^ x2 ^ y2 ^ x3 ^ y3;
    sink[threadIdx.x] = acc;
    __syncthreads();
    t[4] = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0 && r == reps - 1)
      for (int i = 0; i < 4; ++i) out[i] = t[i + 1] - t[i];
  }
  if (acc == 42) out[10] = sink[threadIdx.x];
}

struct Bar {
  unsigned count, gen;
};
__global__ void gridbar_kernel(Bar* bar, long long* out, int reps) {
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t* word = reinterpret_cast<uint64_t*>(bar);
      uint64_t old;
      asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(word), "l"(1ull) : "memory");
      const unsigned g = (unsigned)(old >> 32);
      if ((unsigned)old == gridDim.x - 1) {
        asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(word), "l"((1ull << 32) - gridDim.x) : "memory");
      } else {
        uint64_t v;
        do {
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(word) : "memory");
        } while ((unsigned)(v >> 32) == g);
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (clock64() - t0) / reps;
}

// {count, gen} barrier variants (the repo's protocol = mode 0):
//   0: atom.add.acq_rel arrival; last: red.release gen bump; others: ld.acquire poll (+ nanosleep after 64 spins)
//   1: as 0 without the nanosleep
//   2: as 1, the last arriver bumps gen with red.relaxed (its acq_rel arrival already ordered everything)
//   3: atom.add.release arrival; last: fence.acquire + red.relaxed bump; others: ld.acquire poll
template <int kMode>
__global__ void genbar_kernel(Bar* bar, long long* out, int reps) {
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t* word = reinterpret_cast<uint64_t*>(bar);
      uint64_t old;
      if (kMode == 3)
        asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(word), "l"(1ull) : "memory");
      else
        asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(word), "l"(1ull) : "memory");
      const unsigned g = (unsigned)(old >> 32);
      if ((unsigned)old == gridDim.x - 1) {
        if (kMode <= 1) {
          asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(word), "l"((1ull << 32) - gridDim.x) : "memory");
        } else {
          if (kMode == 3) asm volatile("fence.acq_rel.gpu;" ::: "memory");
          asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(word), "l"((1ull << 32) - gridDim.x) : "memory");
        }
      } else {
        uint64_t v;
        unsigned spins = 0;
        do {
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(word) : "memory");
          if (kMode == 0 && ++spins > 64) __nanosleep(20);
        } while ((unsigned)(v >> 32) == g);
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (clock64() - t0) / reps;
}

// barrier variants over a monotonic arrival counter (zeroed before the launch):
// barrier r completes when the counter reaches G * (r + 1)
//   mode 1: red.release arrival, ld.acquire poll
//   mode 2: fence.acq_rel.gpu; red.relaxed; ld.relaxed poll; fence.acq_rel.gpu
//   mode 3: red.relaxed arrival, ld.relaxed poll, no fence (lower bound, not a barrier for data)
//   mode 4: __threadfence(); atomicAdd; volatile poll; __threadfence()
//   mode 5: fence.sc.gpu only on arrival; ld.acquire poll
template <int kMode>
__global__ void ctrbar_kernel(unsigned* ctr, long long* out, int reps) {
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned target = gridDim.x * (unsigned)(r + 1);
      unsigned v;
      if (kMode == 1) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        do asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        while ((int)(v - target) < 0);
      } else if (kMode == 2) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        do asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        while ((int)(v - target) < 0);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else if (kMode == 3) {
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        do asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        while ((int)(v - target) < 0);
      } else if (kMode == 4) {
        __threadfence();
        atomicAdd(ctr, 1u);
        do v = *(volatile unsigned*)ctr;
        while ((int)(v - target) < 0);
        __threadfence();
      } else {
        asm volatile("fence.sc.gpu;" ::: "memory");
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        do asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        while ((int)(v - target) < 0);
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (clock64() - t0) / reps;
}

// cost of one fence / store pattern in a single thread
__global__ void fence_kernel(unsigned* buf, long long* out) {
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  for (int i = 0; i < 100; ++i) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  long long t1 = clock64();
  for (int i = 0; i < 100; ++i) {
    buf[i * 64] = i;
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  long long t2 = clock64();
  for (int i = 0; i < 100; ++i) asm volatile("fence.acq_rel.cluster;" ::: "memory");
  long long t3 = clock64();
  out[0] = (t1 - t0) / 100;
  out[1] = (t2 - t1) / 100;
  out[2] = (t3 - t2) / 100;
}

__global__ void __cluster_dims__(16, 1, 1) clusterbar_kernel(long long* out, int reps) {
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (clock64() - t0) / reps;
}

int main() {
  uint64_t* buf;
  long long* out;
  Bar* bar;
  const size_t words = 2 * 148 * 4 * 512;
  cudaMalloc(&buf, words * 8);
  cudaMemset(buf, 1, words * 8);
  cudaMalloc(&out, 64 * 8);
  cudaMalloc(&bar, sizeof(Bar));
  cudaMemset(bar, 0, sizeof(Bar));
  cudaFuncSetAttribute(clusterbar_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  long long h[16];
  for (int G : {1, 32, 100, 148}) {
    load_kernel<<<G, 512>>>(buf, out, 20);
    cudaMemcpy(h, out, 4 * 8, cudaMemcpyDeviceToHost);
    printf("load G=%3d  cycles: ldcg u32 %lld | relaxed.gpu v2 %lld | relaxed.sys v2 %lld | 4x relaxed.sys v2 %lld\n", G,
           h[0], h[1], h[2], h[3]);
  }
  for (int G : {2, 16, 32, 100, 148}) {
    gridbar_kernel<<<G, 512>>>(bar, out, 200);
    cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
    printf("gridbar G=%3d  cycles per barrier %lld\n", G, h[0]);
  }
  auto gen_run = [&](auto kern, int mode) {
    for (int G : {2, 32, 100}) {
      cudaMemset(bar, 0, sizeof(Bar));
      kern<<<G, 512>>>(bar, out, 200);
      cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
      printf("genbar mode %d G=%3d  cycles per barrier %lld\n", mode, G, h[0]);
    }
  };
  gen_run(genbar_kernel<0>, 0);
  gen_run(genbar_kernel<1>, 1);
  gen_run(genbar_kernel<2>, 2);
  gen_run(genbar_kernel<3>, 3);
  unsigned* ctr;
  cudaMalloc(&ctr, 4096);
  auto ctr_run = [&](auto kern, int mode) {
    for (int G : {2, 100, 148}) {
      cudaMemset(ctr, 0, 4);
      kern<<<G, 512>>>(ctr, out, 200);
      cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
      printf("ctrbar mode %d G=%3d  cycles per barrier %lld\n", mode, G, h[0]);
    }
  };
  ctr_run(ctrbar_kernel<1>, 1);
  ctr_run(ctrbar_kernel<2>, 2);
  ctr_run(ctrbar_kernel<3>, 3);
  ctr_run(ctrbar_kernel<4>, 4);
  ctr_run(ctrbar_kernel<5>, 5);
  fence_kernel<<<1, 32>>>(ctr, out);
  cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost);
  printf("fence.acq_rel.gpu alone %lld | after a store %lld | fence.acq_rel.cluster %lld cycles\n", h[0], h[1], h[2]);
  clusterbar_kernel<<<16, 512>>>(out, 200);
  cudaError_t e = cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
  printf("clusterbar 16 CTAs  cycles per barrier %lld (%s)\n", h[0], cudaGetErrorString(e));
  return 0;
}
