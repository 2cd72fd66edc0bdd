// Full-graph in-neighbour CSR2 on the device (histgnn/graphs.py:161-172,
// build_csr2): edges grouped by destination, the input edge order kept inside
// every row (the reference's stable argsort). No library sort:
//   k_csr_count   per-destination counts (atomics)
//   scan          start[v] = exclusive prefix, end[v] = start[v] + count
//   k_csr_place   each edge's index at an atomic cursor of its destination row
//   segsort       every row's edge indices ascending (= input order)
//   k_csr_gather  col[p] = src[index[p]]
// Startup only (the graph is built once); ids and edge indices are 32-bit
// (N < 2^31, E < 2^32), offsets 64-bit.
#include "hgb200.h"

#include "hg_common.cuh"
#include "hg_scan.cuh"
#include "hg_segsort.cuh"

namespace hg {
namespace {

__global__ void k_csr_count(const int32_t* __restrict__ dst, long long E, int32_t* __restrict__ cnt) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (long long)gridDim.x * blockDim.x)
    atomicAdd(&cnt[dst[e]], 1);
}

struct CsrCount {
  const int32_t* cnt;
  __device__ long long operator()(long long i) const { return cnt[i]; }
};
struct EmitCsr {
  int64_t* start;
  int64_t* end;
  unsigned long long* cursor;
  __device__ void operator()(long long i, long long excl, long long v) const {
    start[i] = excl;
    end[i] = excl + v;
    cursor[i] = (unsigned long long)excl;
  }
};
struct NoTotalL {
  __device__ void operator()(long long) const {}
};

__global__ void k_csr_place(const int32_t* __restrict__ dst, long long E, unsigned long long* __restrict__ cursor,
                            unsigned* __restrict__ idx) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (long long)gridDim.x * blockDim.x)
    idx[atomicAdd(&cursor[dst[e]], 1ull)] = (unsigned)e;
}

__global__ void k_csr_gather(const int32_t* __restrict__ src, const unsigned* __restrict__ idx, long long E,
                             int32_t* __restrict__ col) {
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < E; p += (long long)gridDim.x * blockDim.x)
    col[p] = src[idx[p]];
}

}  // namespace
}  // namespace hg

using namespace hg;

extern "C" {

long long hg_build_csr2_scratch_bytes(long long E, long long N) {
  // counts, cursors, long-segment list + count, scan partials, index + merge buffers
  return (N + 16) * (4 + 8 + 4) + 64 + (scan_tiles(N) + 1) * 8 + (E + 16) * 4 * 2 + 1024;
}

int hg_build_csr2(const int32_t* src, const int32_t* dst, long long E, long long N, int64_t* start, int64_t* end,
                  int32_t* col, void* scratch, long long scratch_bytes, cudaStream_t stream) {
  const char* W = "hg_build_csr2";
  if (N < 1 || N >= (1ll << 31) || E < 0 || E >= (1ll << 32)) return fail(W, kBadArg, "N < 2^31 and E < 2^32");
  if (scratch_bytes < hg_build_csr2_scratch_bytes(E, N)) return fail(W, kBadArg, "scratch too small");
  char* p = reinterpret_cast<char*>(scratch);
  int32_t* cnt = reinterpret_cast<int32_t*>(p);
  unsigned long long* cursor = reinterpret_cast<unsigned long long*>((reinterpret_cast<uintptr_t>(cnt + N + 16) + 15) &
                                                                     ~uintptr_t(15));
  int32_t* big = reinterpret_cast<int32_t*>(cursor + N + 16);
  int32_t* n_big = big + N + 16;
  long long* part = reinterpret_cast<long long*>((reinterpret_cast<uintptr_t>(n_big + 16) + 15) & ~uintptr_t(15));
  unsigned* idx = reinterpret_cast<unsigned*>(part + scan_tiles(N) + 1);
  unsigned* tmp = idx + E + 16;
  HG_CHECK_CUDA(W, cudaMemsetAsync(cnt, 0, (size_t)N * 4, stream));
  HG_CHECK_CUDA(W, cudaMemsetAsync(n_big, 0, 4, stream));
  const unsigned ge = grid_for(E, 256, 148 * 32);
  if (E > 0) {
    k_csr_count<<<ge, 256, 0, stream>>>(dst, E, cnt);
    HG_LAUNCHED(W);
  }
  const int s = scan_launch<long long>(W, CsrCount{cnt}, ConstCount{N}, N, part, EmitCsr{start, end, cursor},
                                       NoTotalL{}, stream);
  if (s) return s;
  if (E == 0) return kOk;
  k_csr_place<<<ge, 256, 0, stream>>>(dst, E, cursor, idx);
  HG_LAUNCHED(W);
  const int ss = segsort_launch<int64_t>(W, N, start, end, idx, tmp, big, n_big, stream);
  if (ss) return ss;
  k_csr_gather<<<ge, 256, 0, stream>>>(src, idx, E, col);
  HG_LAUNCHED(W);
  return kOk;
}

}  // extern "C"
