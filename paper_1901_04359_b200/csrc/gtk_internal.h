// Host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <utility>

#include "../../include/gtopk_b200.h"

namespace gtk {

void set_last_cuda_error(cudaError_t e);
int num_sms();
// max co-resident blocks of `func` (cooperative launch limit) on the current device
int coop_grid(const void* func, int threads, size_t smem);
// pdl: programmatic dependent launch on the previous kernel of the stream
// (the kernel must griddepcontrol.wait before consuming its outputs)
int coop_launch(const void* func, int grid, int threads, void** args, size_t smem, cudaStream_t st,
                bool pdl = false, bool cooperative = true);
// opt a kernel into > 48 KB of dynamic shared memory (once per device); false on error
bool ensure_dyn_smem(const void* func, size_t bytes);
// grid of a ⊤-merge kernel (merge_kernel / exchange_kernel) over lists of
// <= cap entries: G blocks of kMergeThreads, slice_cap union slots staged in
// shared memory per block, and either one thread-block cluster of G CTAs
// (cluster = true: the engine's grid barriers become barrier.cluster) or a
// cooperative grid
struct MergeGrid {
  int G;
  uint32_t slice_cap;
  bool cluster;
  // false: a plain launch (with PDL) instead of a cooperative one (the
  // deferred exchange, GTK_MERGE_COMPACT_COOP=0: its few blocks are all
  // resident before the next kernel can start, which launches only once every
  // block has released it).  Measured equal: the next HBM pass then starts
  // before the finish ends but loses the time to the SMs it shares
  bool coop = true;
};
// compact_g > 0: at most compact_g blocks whenever the union fits their
// shared memory (a merge that shares the GPU with an HBM pass)
bool merge_grid_for(const void* func, int32_t cap, MergeGrid* out, int compact_g = 0);
// a one-CTA merge of lists up to cap entries takes the merge_solo instance
bool merge_use_solo(const MergeGrid& g, int32_t cap);
// launch a merge-type kernel on its MergeGrid (cluster or cooperative)
int merge_launch(const void* func, const MergeGrid& g, void** args, size_t smem, cudaStream_t st, bool pdl);

// Launch with the programmatic-stream-serialization attribute: the kernel may
// start as soon as the previous kernel in the stream executes
// griddepcontrol.launch_dependents; it must griddepcontrol.wait before
// consuming that kernel's results.  Graph-capturable.
bool pdl_enabled();  // GTK_NO_PDL=1 disables (A/B measurements)
// debug trace buffer (gtk_exchange_set_trace): exchange stamps at [0..31],
// merge phase stamps at [32 + 16*step ..] (standalone merges use [32..])
int64_t* trace_buffer();
void set_trace_buffer(int64_t* p);

template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  if (!pdl_enabled()) {
    kernel<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---- profiling hooks (bench.py): CUDA events around a launch, recorded on the
// launching stream, only when enabled and the stream is not being captured ----
enum ProfId { kProfSelectMain = 0, kProfSelect = 1, kProfExchange = 2, kProfMerge = 3, kProfUpdate = 4, kProfN = 8 };
void prof_record(int id, cudaStream_t st, bool begin);
void count_launch(int n = 1);

struct ProfScope {
  int id;
  cudaStream_t st;
  ProfScope(int i, cudaStream_t s) : id(i), st(s) { prof_record(id, st, true); }
  ~ProfScope() { prof_record(id, st, false); }
};

}  // namespace gtk

#define GTK_CHECK_LAUNCH()                        \
  do {                                            \
    cudaError_t _e = cudaGetLastError();          \
    if (_e != cudaSuccess) {                      \
      gtk::set_last_cuda_error(_e);               \
      return GTK_ECUDA;                           \
    }                                             \
    gtk::count_launch();                          \
  } while (0)

#define GTK_CUDA(call)                            \
  do {                                            \
    cudaError_t _e = (call);                      \
    if (_e != cudaSuccess) {                      \
      gtk::set_last_cuda_error(_e);               \
      return GTK_ECUDA;                           \
    }                                             \
  } while (0)
