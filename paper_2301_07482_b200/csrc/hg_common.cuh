// Shared helpers for the hgb200 sm_100a kernels: status codes, launch checks,
// device-count-aware grid sizing and warp utilities.
//
// Conventions of every hg_* entry point (see include/hgb200.h):
//   * all memory is owned by the caller (PyTorch); pointers are device pointers
//     unless named *_host; nothing is allocated here except cuBLAS handles;
//   * every launch is asynchronous on the caller's stream;
//   * element counts that are produced on the device are passed as device
//     pointers (`const int32_t* n_dev`) together with a host upper bound
//     (`n_max`) that sizes the grid, so a whole iteration can run without a
//     host round trip;
//   * functions return 0 on success and a negative status otherwise; the
//     message is kept per thread and read with hg_last_error().
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

namespace hg {

enum Status : int {
  kOk = 0,
  kBadArg = -1,
  kCuda = -2,
  kCublas = -3,
  kUnsupported = -4,
};

void set_error(const char* where, const std::string& msg);
int fail(const char* where, int code, const std::string& msg);
int check_launch(const char* where);

constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs

inline unsigned grid_for(long long n, int per_block, unsigned cap = 148u * 64u) {
  long long g = (n + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > (long long)cap) g = cap;
  return (unsigned)g;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// fixed-order tree reduction (identical result on every run)
__device__ __forceinline__ double warp_sum_fixed(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return __shfl_sync(0xffffffffu, v, 0);
}

// warp-aggregated integer counter bump: one atomic per warp
__device__ __forceinline__ void warp_count_add(unsigned long long* ctr, bool pred) {
  unsigned m = __ballot_sync(__activemask(), pred);
  if (m && (lane_id() == (__ffs(__activemask()) - 1)))
    atomicAdd(ctr, (unsigned long long)__popc(m));
}

// 128-bit vector load that bypasses L1 allocation (streaming gathers)
__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint4 ldg_stream_u4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ---- device-side kernel timers (work inside CUDA graphs, where events can't
// bracket a single node): span from the first CTA start to the last CTA end
// (%globaltimer, ns), accumulated per launch by the last CTA to finish.
struct KTimer {
  unsigned long long start, end, total_ns, launches, done, pad[3];
};
enum TimerId : int { kTLoadRows = 0, kTAggregate = 1, kTTransposeAgg = 2, kTSelect = 3, kTGemmFwd = 4, kTGemmBwd = 5, kTGemmWgrad = 6,
                     kTAggregateFeat = 7, kNumTimers = 8 };

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void kt_begin(KTimer* kt) {
  if (kt && threadIdx.x == 0) atomicMin(&kt->start, gtimer());
}
// every thread of the CTA must reach this
__device__ __forceinline__ void kt_end(KTimer* kt) {
  if (!kt) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMax(&kt->end, gtimer());
    __threadfence();
    const unsigned long long n = (unsigned long long)gridDim.x * gridDim.y * gridDim.z;
    if (atomicAdd(&kt->done, 1ull) == n - 1) {
      __threadfence();
      const unsigned long long s = atomicAdd(&kt->start, 0ull), e = atomicAdd(&kt->end, 0ull);
      kt->total_ns += e - s;
      kt->launches += 1;
      kt->start = ~0ull;
      kt->end = 0;
      kt->done = 0;
      __threadfence();
    }
  }
}

// Programmatic dependent launch (PDL): kernels launched with launch_pdl may
// be scheduled while their predecessor in the stream is still finishing (its
// launch latency overlaps the predecessor's tail); they call pdl_wait() first,
// which blocks until the predecessor grid has completed and its writes are
// visible, so stream semantics are unchanged. A no-op for normal launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pdl_enabled();   // HG_PDL=0 disables (A/B)
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device);
// thread-safe (a mutex-guarded set), no process-global "done" flag
int ensure_smem_attr(const void* kernel, int bytes, const char* where);
// read an environment knob once (thread-safe static initialisation)
const char* env_knob(const char* name);
bool node_prio_enabled();   // HG_NODE_PRIO=1: kernel nodes carry their stream's priority

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args... args) {
  if (!pdl_enabled()) {
    kernel<<<grid, block, smem, stream>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (node_prio_enabled()) {
    // recorded on the kernel node at capture; honoured by graphs instantiated
    // with cudaGraphInstantiateFlagUseNodePriority (hg_graph_instantiate)
    int prio = 0;
    if (cudaStreamGetPriority(stream, &prio) == cudaSuccess) {
      attr[1].id = cudaLaunchAttributePriority;
      attr[1].val.priority = prio;
      cfg.numAttrs = 2;
    }
  }
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

int set_timers_gather(void* p);
int set_timers_layer(void* p);
int set_timers_sampler(void* p);
int set_timers_gemm(void* p);

}  // namespace hg

#define HG_CHECK_CUDA(where, expr)                                       \
  do {                                                                     \
    cudaError_t _e = (expr);                                               \
    if (_e != cudaSuccess)                                                 \
      return hg::fail(where, hg::kCuda, cudaGetErrorString(_e));           \
  } while (0)

#define HG_LAUNCHED(where)                        \
  do {                                            \
    int _s = hg::check_launch(where);             \
    if (_s) return _s;                            \
  } while (0)
