// Library-level C-ABI entry points: version, error strings, workspace init and
// the cooperative-launch helpers.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <vector>
#include <unordered_map>

#include "gtk_internal.h"

namespace gtk {

static thread_local char g_last_err[256] = "";

void set_last_cuda_error(cudaError_t e) {
  std::snprintf(g_last_err, sizeof(g_last_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
}

int num_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

int coop_grid(const void* func, int threads, size_t smem) {
  static std::mutex mu;
  static std::unordered_map<unsigned long long, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  const unsigned long long key = ((unsigned long long)(uintptr_t)func) ^ ((unsigned long long)dev << 56) ^
                                 ((unsigned long long)threads << 40) ^ (unsigned long long)smem;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, func, threads, smem);
  if (e != cudaSuccess) {
    set_last_cuda_error(e);
    return 0;
  }
  const int g = per_sm * num_sms();
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = g;
  return g;
}

bool ensure_dyn_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<unsigned long long, bool> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  const unsigned long long key = ((unsigned long long)(uintptr_t)func) ^ ((unsigned long long)dev << 56);
  std::lock_guard<std::mutex> g(mu);
  if (done.count(key)) return true;
  cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) {
    set_last_cuda_error(e);
    return false;
  }
  done[key] = true;
  return true;
}

int coop_launch(const void* func, int grid, int threads, void** args, size_t smem, cudaStream_t st, bool pdl,
                bool cooperative) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (cooperative) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na++].val.cooperative = 1;
  }
  if (pdl && pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelExC(&cfg, func, args);
  if (e != cudaSuccess) {
    set_last_cuda_error(e);
    return GTK_ECUDA;
  }
  count_launch();
  return GTK_OK;
}

// ---- profiling hooks -----------------------------------------------------------
static std::atomic<long long> g_launches{0};
static std::atomic<bool> g_prof_on{false};
static std::mutex g_prof_mu;
struct PendingPair {
  int id;
  cudaEvent_t a, b;
};
static std::vector<PendingPair> g_pending;
static std::vector<cudaEvent_t> g_open[kProfN];  // begin events awaiting their end, per id
static std::vector<cudaEvent_t> g_pool;
static double g_sum_ms[kProfN];
static long long g_cnt[kProfN];

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static int64_t* g_trace = nullptr;
int64_t* trace_buffer() { return g_trace; }
void set_trace_buffer(int64_t* p) { g_trace = p; }

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("GTK_NO_PDL");
    return !(v && v[0] && v[0] != '0');
  }();
  return on;
}

static cudaEvent_t pool_get() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// pairs recorded while a stream was being captured become event-record nodes
// of the graph: they are re-recorded on every replay and read in place
static std::vector<PendingPair> g_graph_pairs;
static std::vector<cudaEvent_t> g_graph_open[kProfN];

void prof_record(int id, cudaStream_t st, bool begin) {
  if (!g_prof_on.load(std::memory_order_relaxed) || id < 0 || id >= kProfN) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) return;
  const bool capturing = cs != cudaStreamCaptureStatusNone;
  std::lock_guard<std::mutex> g(g_prof_mu);
  cudaEvent_t e = pool_get();
  if (!e) return;
  if (capturing) {
    if (cudaEventRecordWithFlags(e, st, cudaEventRecordExternal) != cudaSuccess) return;
  } else if (cudaEventRecord(e, st) != cudaSuccess) {
    return;
  }
  auto& open = capturing ? g_graph_open[id] : g_open[id];
  if (begin) {
    open.push_back(e);
  } else if (!open.empty()) {
    cudaEvent_t a = open.back();
    open.pop_back();
    (capturing ? g_graph_pairs : g_pending).push_back(PendingPair{id, a, e});
  }
}

}  // namespace gtk

extern "C" int gtk_prof_enable(int on) {
  gtk::g_prof_on.store(on != 0);
  return GTK_OK;
}

extern "C" int gtk_prof_read(int id, double* total_ms, int64_t* count) {
  using namespace gtk;
  if (id < 0 || id >= kProfN || !total_ms || !count) return GTK_EINVAL;
  std::lock_guard<std::mutex> g(g_prof_mu);
  for (auto& p : g_pending) {
    float ms = 0.f;
    if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      g_sum_ms[p.id] += ms;
      g_cnt[p.id] += 1;
    }
    g_pool.push_back(p.a);
    g_pool.push_back(p.b);
  }
  g_pending.clear();
  *total_ms = g_sum_ms[id];
  *count = g_cnt[id];
  return GTK_OK;
}

extern "C" int gtk_prof_reset(void) {
  using namespace gtk;
  std::lock_guard<std::mutex> g(g_prof_mu);
  for (auto& p : g_pending) {
    cudaEventSynchronize(p.b);
    g_pool.push_back(p.a);
    g_pool.push_back(p.b);
  }
  g_pending.clear();
  for (auto& p : g_graph_pairs) {
    g_pool.push_back(p.a);
    g_pool.push_back(p.b);
  }
  g_graph_pairs.clear();
  for (int i = 0; i < kProfN; ++i) {
    g_sum_ms[i] = 0;
    g_cnt[i] = 0;
    g_open[i].clear();
    g_graph_open[i].clear();
  }
  return GTK_OK;
}

extern "C" int gtk_prof_graph_read(int id, double* ms, int64_t* count) {
  using namespace gtk;
  if (id < 0 || id >= kProfN || !ms || !count) return GTK_EINVAL;
  std::lock_guard<std::mutex> g(g_prof_mu);
  double s = 0;
  int64_t n = 0;
  for (auto& p : g_graph_pairs) {
    if (p.id != id) continue;
    float t = 0.f;
    if (cudaEventElapsedTime(&t, p.a, p.b) == cudaSuccess) {
      s += t;
      ++n;
    }
  }
  *ms = s;
  *count = n;
  return GTK_OK;
}

extern "C" int64_t gtk_launch_count(void) { return (int64_t)gtk::g_launches.load(); }

namespace gtk {

}  // namespace gtk

extern "C" int gtk_version(void) { return 10000; /* 1.0.0 */ }

extern "C" const char* gtk_strerror(int code) {
  switch (code) {
    case GTK_OK: return "ok";
    case GTK_EINVAL: return "invalid argument";
    case GTK_ENONFINITE: return "non-finite values in dense input";
    case GTK_EPROTO: return "protocol error";
    case GTK_ETIMEOUT: return "timed out";
    case GTK_ECUDA: return "CUDA error";
    case GTK_ENOMEM: return "workspace too small";
    case GTK_EABORTED: return "cluster aborted";
    default: return "unknown error";
  }
}

extern "C" const char* gtk_last_cuda_error(void) { return gtk::g_last_err; }

extern "C" int gtk_workspace_init(void* ws, size_t bytes, void* stream) {
  if (!ws) return GTK_EINVAL;
  GTK_CUDA(cudaMemsetAsync(ws, 0, bytes, (cudaStream_t)stream));
  return GTK_OK;
}
