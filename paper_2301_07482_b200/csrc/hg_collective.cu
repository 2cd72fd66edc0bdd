// Gradient all-reduce fused with the SGD step over NVLink peer memory (the
// data-parallel exchange of SURVEY §8(e): trainer.py:423-433 + nn.py:355-360
// with the gradients averaged over P ranks). An alternative to the NCCL hook:
//   k_p2p_stage      copy this rank's flat gradient bucket into its exchange
//                    slot (double-buffered by step parity), fence at system
//                    scope, then the last CTA publishes flag = epoch
//   k_p2p_reduce_sgd every CTA waits until all P flags reach the epoch, sums
//                    the P slots in rank order 0..P-1 (identical bits on every
//                    rank), divides by P and applies p -= eta * g
// Slots and flags live in CUDA-IPC allocations mapped into every rank
// (distributed.P2PAllReduce). The epoch is a per-rank device counter that the
// last CTA of k_p2p_reduce_sgd advances, so it counts exchange steps and is
// the same on every rank at a step. Slot (epoch & 1) is rewritten at epoch + 2
// only after every rank passed the epoch + 1 barrier, i.e. finished reading it.
// The wait times out instead of hanging if a peer never arrives: the kernel
// records the timeout in the state word, skips the update and exits (the
// context stays usable); the host reads the word and raises.
#include "hgb200.h"

#include "hg_common.cuh"

namespace hg {
namespace {

constexpr unsigned long long kP2PTimeoutNs = 120ull * 1000000000ull;   // default when state[4] == 0

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// st: [0] stage arrivals, [1] reduce arrivals, [2] completed exchanges,
//     [3] timeout flag (sticky), [4] timeout in ns (0 = kP2PTimeoutNs)
__global__ void k_p2p_stage(const float* __restrict__ grads, long long n, float* __restrict__ my_slots,
                            unsigned long long* my_flag, unsigned long long* st) {
  pdl_wait();
  const unsigned long long epoch = st[2] + 1ull;
  float* slot = my_slots + (long long)(epoch & 1ull) * n;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) slot[i] = grads[i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(st, 1ull) == gridDim.x - 1) {
      st[0] = 0;
      __threadfence_system();
      st_release_sys(my_flag, epoch);
    }
  }
}

__global__ void k_p2p_reduce_sgd(float* __restrict__ params, long long n, const float* const* __restrict__ slots,
                                 unsigned long long* const* __restrict__ flags, int P, float eta,
                                 unsigned long long* st) {
  pdl_wait();
  __shared__ int s_abort;
  const unsigned long long epoch = st[2] + 1ull;
  if (threadIdx.x == 0) {
    const unsigned long long limit = st[4] ? st[4] : kP2PTimeoutNs;
    const unsigned long long t0 = globaltimer_ns();
    int abort = ld_acquire_sys(st + 3) != 0ull;   // an earlier exchange already failed
    for (int r = 0; r < P && !abort; ++r) {
      while (ld_acquire_sys(flags[r]) < epoch) {
        if (globaltimer_ns() - t0 > limit) {   // a peer never arrived: record it, never hang the GPU
          atomicExch(st + 3, 1ull);
          abort = 1;
          break;
        }
        __nanosleep(128);
      }
    }
    s_abort = abort;
  }
  __syncthreads();
  if (s_abort) return;   // parameters untouched; the host sees state[3] and raises
  const long long off = (long long)(epoch & 1ull) * n;
  const float inv = 1.0f / (float)P;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float s = __ldcg(slots[0] + off + i);       // L2 / NVLink, never a stale L1 line
    for (int r = 1; r < P; ++r) s = __fadd_rn(s, __ldcg(slots[r] + off + i));
    const float g = (P & (P - 1)) == 0 ? __fmul_rn(s, inv) : __fdiv_rn(s, (float)P);
    params[i] = __fsub_rn(params[i], __fmul_rn(eta, g));
  }
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(st + 1, 1ull) == gridDim.x - 1) {
    st[1] = 0;
    st[2] = epoch;
  }
}

}  // namespace
}  // namespace hg

using namespace hg;

extern "C" {

// one data-parallel step: average this rank's grads with the P-1 peers' over
// the IPC-mapped slots and apply SGD; slots[r] = rank r's 2 x n float slot
// area, flags[r] = rank r's flag word (device arrays of P pointers);
// state = 8 u64 words owned by this rank, zero-initialised except [4] (the
// peer-wait timeout in ns, 0 = 120 s); state[3] != 0 after a timed-out wait
int hg_p2p_allreduce_sgd(float* params, const float* grads, long long n, float* my_slots,
                         unsigned long long* my_flag, const float* const* slots, unsigned long long* const* flags,
                         int P, unsigned long long* state, float eta, cudaStream_t stream) {
  const char* W = "hg_p2p_allreduce_sgd";
  if (P < 1 || P > 64 || n < 1) return fail(W, kBadArg, "bad world size / bucket size");
  const unsigned grid = grid_for(n, 256, 148 * 2);
  { const cudaError_t pe = hg::launch_pdl(k_p2p_stage, dim3(grid), dim3(256), 0, stream, grads, n, my_slots,
                                          my_flag, state);
    if (pe != cudaSuccess) return fail(W, kCuda, cudaGetErrorString(pe)); }
  HG_LAUNCHED(W);
  { const cudaError_t pe = hg::launch_pdl(k_p2p_reduce_sgd, dim3(grid), dim3(256), 0, stream, params, n, slots, flags,
                                          P, eta, state);
    if (pe != cudaSuccess) return fail(W, kCuda, cudaGetErrorString(pe)); }
  HG_LAUNCHED(W);
  return kOk;
}

}  // extern "C"
