// Library-wide entry points: version, last error, launch checking.
#include "hgb200.h"
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <map>
#include <set>
#include <tuple>
#include <string>

#include "hg_common.cuh"

namespace hg {

static thread_local std::string g_last_error;

void set_error(const char* where, const std::string& msg) { g_last_error = std::string(where) + ": " + msg; }

int fail(const char* where, int code, const std::string& msg) {
  set_error(where, msg);
  return code;
}

static std::atomic<long long> g_launches{0};

__global__ void k_mark_time(unsigned long long* slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *slot = t;
}

// one step's IterMetrics source row (trainer.py:86-104,407-421) written by
// the device at the end of the step: [loss, counter deltas since the previous
// row (prev updated in place), per-layer valid entries, n_src of block 0,
// the prune counts]; the host reads it with one async copy
__global__ void k_metrics_row(const long long* const* __restrict__ vecs, const int* __restrict__ lens, int nvec,
                              long long* __restrict__ prev, const double* loss, const int32_t* n_src0,
                              const int32_t* __restrict__ counts, int ncounts, int valid_idx, double* __restrict__ out) {
  int nv = 0;
  for (int v = 0; v < nvec; ++v) nv += lens[v];
  if (threadIdx.x == 0) out[0] = *loss;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    int v = 0, o = i;
    while (o >= lens[v]) o -= lens[v++];
    const long long cur = vecs[v][o];
    out[1 + i] = (double)(cur - prev[i]);
    prev[i] = cur;
  }
  const int nl = nvec - 1;   // every vector but the last (global) is a layer
  for (int l = threadIdx.x; l < nl; l += blockDim.x) out[1 + nv + l] = (double)vecs[l][valid_idx];
  if (threadIdx.x == 0) out[1 + nv + nl] = (double)*n_src0;
  for (int c = threadIdx.x; c < ncounts; c += blockDim.x) out[2 + nv + nl + c] = (double)counts[c];
}

bool pdl_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("HG_PDL");
    return !(e && e[0] == '0');
  }();
  return v;
}

bool node_prio_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("HG_NODE_PRIO");
    return e && e[0] == '1';
  }();
  return v;
}

const char* env_knob(const char* name) { return std::getenv(name); }

// raise (never lower) a kernel's dynamic shared-memory limit to >= bytes;
// launches below the 48 KB default need nothing
int ensure_smem_attr(const void* kernel, int bytes, const char* where) {
  if (bytes <= 48 * 1024) return kOk;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> set_to;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(where, kCuda, cudaGetErrorString(e));
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_pair(kernel, dev);
  const auto it = set_to.find(key);
  if (it != set_to.end() && it->second >= bytes) return kOk;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return fail(where, kCuda, cudaGetErrorString(e));
  set_to[key] = bytes;
  return kOk;
}

int check_launch(const char* where) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(where, kCuda, cudaGetErrorString(e));
  return kOk;
}

}  // namespace hg

extern "C" {

int hg_version(void) { return 10000; }  // 1.0.0

// device-side kernel timers (hg::KTimer[kNumTimers]; start fields = ~0), or NULL to disable
int hg_set_kernel_timers(void* buf) {
  int st = hg::set_timers_gather(buf);
  if (!st) st = hg::set_timers_layer(buf);
  if (!st) st = hg::set_timers_sampler(buf);
  if (!st) st = hg::set_timers_gemm(buf);
  return st;
}

// number of hand-written hg kernels launched by this process so far
long long hg_kernel_launches(void) { return hg::g_launches.load(std::memory_order_relaxed); }

// step timeline probe: *slot = %globaltimer when the stream reaches this point
int hg_mark_time(unsigned long long* slot, cudaStream_t stream) {
  hg::k_mark_time<<<1, 1, 0, stream>>>(slot);
  return hg::check_launch("hg_mark_time");
}

int hg_metrics_row(const long long* const* vecs, const int* lens, int nvec, long long* prev, const double* loss,
                   const int32_t* n_src0, const int32_t* counts, int ncounts, int valid_idx, double* out,
                   cudaStream_t stream) {
  if (nvec < 1) return hg::fail("hg_metrics_row", hg::kBadArg, "no counter vectors");
  hg::k_metrics_row<<<1, 64, 0, stream>>>(vecs, lens, nvec, prev, loss, n_src0, counts, ncounts, valid_idx, out);
  return hg::check_launch("hg_metrics_row");
}

// a CUDA graph replay re-executes the n hg kernels recorded at its capture
void hg_count_graph_replay(long long n) { hg::g_launches.fetch_add(n, std::memory_order_relaxed); }

// executable graph honouring per-node priorities (HG_NODE_PRIO=1 path of
// engine.StepEngine: the cache-update and training streams outrank the
// lookahead sampler inside one replay)
int hg_graph_instantiate(void* graph, void** exec_out) {
  if (!graph || !exec_out) return hg::fail("hg_graph_instantiate", hg::kBadArg, "null graph");
  cudaGraphExec_t ex = nullptr;
  cudaError_t e = cudaGraphInstantiateWithFlags(&ex, static_cast<cudaGraph_t>(graph),
                                                cudaGraphInstantiateFlagUseNodePriority);
  if (e != cudaSuccess) return hg::fail("hg_graph_instantiate", hg::kCuda, cudaGetErrorString(e));
  *exec_out = ex;
  return hg::kOk;
}

int hg_graph_launch(void* exec, cudaStream_t stream) {
  cudaError_t e = cudaGraphLaunch(static_cast<cudaGraphExec_t>(exec), stream);
  return e == cudaSuccess ? hg::kOk : hg::fail("hg_graph_launch", hg::kCuda, cudaGetErrorString(e));
}

int hg_graph_exec_destroy(void* exec) {
  cudaError_t e = cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(exec));
  return e == cudaSuccess ? hg::kOk : hg::fail("hg_graph_exec_destroy", hg::kCuda, cudaGetErrorString(e));
}

const char* hg_last_error(void) { return hg::g_last_error.c_str(); }

int hg_device_sync(void) {
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return hg::fail("hg_device_sync", hg::kCuda, cudaGetErrorString(e));
  return 0;
}

}  // extern "C"
