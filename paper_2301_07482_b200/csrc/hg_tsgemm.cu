// K7 product path: the dense per-layer transform on tcgen05 over TS operands.
//
// Operands are produced directly in the TS layout (hg_ts.cuh: bf16 hi/lo
// planes of 8x8 core matrices in row-group strips) by the aggregation, the dz
// gather and the per-step weight split, so the GEMM never stages operands
// through registers: a producer thread streams every K-chunk stage with ONE
// 4-D TMA box per operand (cp.async.bulk.tensor.4d, completion counted on an
// mbarrier) into a kStages-deep shared-memory ring; a single thread issues
// tcgen05.mma kind::f16 (bf16 x bf16 -> fp32 in TMEM) for the 3-term split
//   a.b ~= hi(a).hi(b) + hi(a).lo(b) + lo(a).hi(b)   (relative error ~1e-5)
// and releases each stage with tcgen05.commit; 4 x kEpiHalves warps drain TMEM
// through shared memory in the epilogue (coalesced row stores).
//   kMN = false: D = A . B^T, both operands K-major      (forward, data grad)
//   kMN = true : D = A^T . B over the stored rows, both read as MN-major
//                operands from the very same stored cores (weight grad,
//                split-K over rows + fixed-order reduction: deterministic).
#include "hgb200.h"
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "hg_common.cuh"
#include "hg_ts.cuh"

namespace hg {
namespace {

__device__ KTimer* g_kt = nullptr;
}  // namespace
int set_timers_gemm(void* p) {
  cudaError_t e = cudaMemcpyToSymbol(g_kt, &p, sizeof(p));
  return e == cudaSuccess ? kOk : fail("set_timers_gemm", kCuda, cudaGetErrorString(e));
}
namespace {

constexpr int kTM = 128;       // tile rows (MMA M)
constexpr int kBK = 32;        // K elements per stage
// Epilogue warps split a tile's columns in kEpiHalves parts per TMEM lane
// quadrant (4 * kEpiHalves epilogue warps): the drain is issue-latency bound
// (ncu: ~8 cycles per issued instruction, one epilogue warp per scheduler).
#ifndef HG_EPI_HALVES
#define HG_EPI_HALVES 2
#endif
constexpr int kEpiHalves = HG_EPI_HALVES;
constexpr int kEpiWarps = 4 * kEpiHalves;
constexpr int kThreads = 32 * kEpiWarps;   // one-tile kernel: every warp drains
constexpr int kStages = 4;

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(32);
  }
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// 32 consecutive accumulator columns of this thread's TMEM lane, one wait
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// no-swizzle UMMA shared-memory descriptor, Blackwell version bit
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// kind::f16 instruction descriptor: bf16 x bf16 -> f32, K- or MN-major operands
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void tma_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                       uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- epilogues
// Epilogues store acc at expand(key(i)) + n. The key is computed once per
// tile row by the lane that owns the row and shuffled to the storing lanes,
// so the store loop carries no index loads. Key widths are what measured
// best (C2/C5, kernel timers): the forward scatter shuffles the 32-bit
// rows[i] (forward GEMMs 0.51 -> 0.45 ms/step at C5), dgrad / wgrad shuffle
// the 64-bit row offset (-25 % / -13 % vs per-store arithmetic; a 32-bit
// key there was slower than either).
struct EpiScatterRelu {  // h_out[rows[i]][n] = act(acc)
  static constexpr bool kFwd = true;
  using Key = int;
  const int32_t* rows;
  float* out;
  int ldo;
  int relu;
  bool vec;   // 16-byte row segments possible (ldo % 4 == 0, aligned base)
  __device__ __forceinline__ Key key(int i) const { return rows[i]; }
  __device__ __forceinline__ long long expand(Key k) const { return (long long)k * ldo; }
  __device__ __forceinline__ void store(long long k, int n, float x) const {
    if (relu) x = x > 0.f ? x : 0.f;
    out[k + n] = x;
  }
  __device__ __forceinline__ void store4(long long k, int n, float4 x) const {
    if (relu) x = make_float4(fmaxf(x.x, 0.f), fmaxf(x.y, 0.f), fmaxf(x.z, 0.f), fmaxf(x.w, 0.f));
    *reinterpret_cast<float4*>(out + k + n) = x;
  }
};
struct EpiStore {
  static constexpr bool kFwd = false;
  using Key = long long;
  float* out;
  long long ldo;
  bool vec;
  __device__ __forceinline__ Key key(int i) const { return (long long)i * ldo; }
  __device__ __forceinline__ long long expand(Key k) const { return k; }
  __device__ __forceinline__ void store(long long k, int n, float x) const { out[k + n] = x; }
  __device__ __forceinline__ void store4(long long k, int n, float4 x) const {
    *reinterpret_cast<float4*>(out + k + n) = x;
  }
};
struct EpiPartial {      // part[z][i][n] = acc
  static constexpr bool kFwd = false;
  using Key = long long;
  float* part;
  long long ldo;
  long long stride;
  bool vec;
  __device__ __forceinline__ Key key(int i) const { return (long long)blockIdx.z * stride + (long long)i * ldo; }
  __device__ __forceinline__ long long expand(Key k) const { return k; }
  __device__ __forceinline__ void store(long long k, int n, float x) const { part[k + n] = x; }
  __device__ __forceinline__ void store4(long long k, int n, float4 x) const {
    *reinterpret_cast<float4*>(part + k + n) = x;
  }
};

// Epilogue staging: a warp moves its 32 tile rows x 32 columns through a
// 4 KB shared-memory chunk, float4 j of row r at slot j ^ (r & 7) (XOR
// swizzle, no padding): the row-per-lane STS.128 writes and the
// 4-rows-per-instruction LDS.128 reads are both bank-conflict free.
__device__ __forceinline__ int stage_at(int r, int c) { return r * 32 + ((((c >> 2) ^ r) & 7) << 2) + (c & 3); }

// Store one staged 32 x 32 chunk. Vector path: a warp instruction writes
// 4 rows x 128 B (8 lanes x 16 B per row), 8 instructions per chunk; columns
// past n_valid fall back to scalar stores.
template <typename Epi>
__device__ __forceinline__ void store_chunk(const Epi& epi, const float* stage_f, typename Epi::Key my_key,
                                            int row0, int M, int c0, int n0, int n_valid, int lane) {
  if (epi.vec) {
    const int rsub = lane >> 3, c4 = (lane & 7) * 4;
    const int col = c0 + c4;
#pragma unroll 4
    for (int rr = 0; rr < 32; rr += 4) {
      const int r = rr + rsub;
      const long long k = epi.expand(__shfl_sync(0xffffffffu, my_key, r));
      if (row0 + r < M) {
        const float4 v = *reinterpret_cast<const float4*>(stage_f + stage_at(r, c4));
        if (col + 3 < n_valid) {
          epi.store4(k, n0 + col, v);
        } else {
          const float e4[4] = {v.x, v.y, v.z, v.w};
          for (int e = 0; e < 4; ++e)
            if (col + e < n_valid) epi.store(k, n0 + col + e, e4[e]);
        }
      }
    }
  } else {
    const int col = c0 + lane;
    for (int r = 0; r < 32; ++r) {
      const long long k = epi.expand(__shfl_sync(0xffffffffu, my_key, r));
      if (row0 + r < M && col < n_valid) epi.store(k, n0 + col, stage_f[stage_at(r, lane)]);
    }
  }
}

// Drain accumulator columns [cb, ce) (multiples of 32 from cb) of the
// warp's TMEM lane quadrant: tmem_row = TMEM address of (quadrant lane 0,
// column 0 of the accumulator); zero = no K chunk was accumulated.
template <typename Epi>
__device__ __forceinline__ void drain_cols(const Epi& epi, uint32_t tmem_row, float* stage_f,
                                           typename Epi::Key my_key, int row0, int M, int cb, int ce, int n0,
                                           int n_valid, int lane, bool zero) {
  for (int c0 = cb; c0 < ce; c0 += 32) {
    uint32_t acc[32];
    if (!zero) {
      tmem_ld32(tmem_row + (uint32_t)c0, acc);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0u;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<float4*>(stage_f + stage_at(lane, 4 * j)) =
          make_float4(__uint_as_float(acc[4 * j]), __uint_as_float(acc[4 * j + 1]), __uint_as_float(acc[4 * j + 2]),
                      __uint_as_float(acc[4 * j + 3]));
    __syncwarp();
    store_chunk(epi, stage_f, my_key, row0, M, c0, n0, n_valid, lane);
    __syncwarp();
  }
}

__device__ __forceinline__ void epi_cols(int h, int n_valid, int& cb, int& ce) {
  const int per = ((n_valid + 32 * kEpiHalves - 1) / (32 * kEpiHalves)) * 32;
  cb = h * per;
  ce = min(n_valid, cb + per);
}

struct Shape {
  int M, N, K;              // M, K may be replaced by device counts
  const int32_t* M_dev;
  const int32_t* K_dev;
  int chunks_per_split;
};

template <bool kMN, typename Epi>
__global__ void __launch_bounds__(kThreads, 1) k_tsgemm(const __grid_constant__ CUtensorMap tmA,
                                                        const __grid_constant__ CUtensorMap tmB, Shape sh, Epi epi,
                                                        int N_pad, uint32_t tmem_cols) {
  pdl_wait();
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages], done_bar;
  __shared__ uint32_t tmem_slot;
  const int M = sh.M_dev ? *sh.M_dev : sh.M;
  const int K = sh.K_dev ? *sh.K_dev : sh.K;
  const int m0 = blockIdx.x * kTM;
  KTimer* kt = g_kt ? g_kt + (kMN ? kTGemmWgrad : (Epi::kFwd ? kTGemmFwd : kTGemmBwd)) : nullptr;
  kt_begin(kt);
  if (m0 >= M) {
    kt_end(kt);
    return;
  }
  const int n0 = blockIdx.y * N_pad;
  const int n_valid = min(N_pad, sh.N - n0);
  const int chunks = (K + kBK - 1) / kBK;
  // split-K (weight gradient): the device count of reduction rows is shared
  // evenly by the splits (the host's upper bound would leave the trailing
  // splits idle and the others each a bound-sized share)
  const int per = kMN && sh.K_dev ? (chunks + (int)gridDim.z - 1) / (int)gridDim.z : sh.chunks_per_split;
  const int c_begin = blockIdx.z * per;
  const int c_end = min(chunks, c_begin + per);
  const int nc = c_end > c_begin ? c_end - c_begin : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t a_half = 8192;                     // 128 x 32 bf16
  const uint32_t b_half = (uint32_t)N_pad * 64;     // N_pad x 32 bf16
  const uint32_t stage_bytes = 2 * a_half + 2 * b_half;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0 && lane == 0) {
    // producer: one TMA box per operand per stage (hi and lo planes together)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int i = 0; i < nc; ++i) {
      const int st = i % kStages;
      if (i >= kStages) mbar_wait(&empty_bar[st], ((i / kStages) - 1) & 1);
      uint8_t* base = smem + st * stage_bytes;
      const int c = c_begin + i;
      mbar_expect_tx(&full_bar[st], stage_bytes);
      if (!kMN) {
        tma_4d(base, &tmA, 0, 4 * c, m0 / 8, 0, &full_bar[st]);               // 128 rows x 32 k
        tma_4d(base + 2 * a_half, &tmB, 0, 4 * c, n0 / 8, 0, &full_bar[st]);  // N_pad rows x 32 k
      } else {
        tma_4d(base, &tmA, 0, m0 / 8, 4 * c, 0, &full_bar[st]);               // 32 rows x 128 cols
        tma_4d(base + 2 * a_half, &tmB, 0, n0 / 8, 4 * c, 0, &full_bar[st]);  // 32 rows x N_pad cols
      }
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer
    const uint32_t idesc = make_idesc(kTM, N_pad, kMN ? 1 : 0, kMN ? 1 : 0);
    for (int i = 0; i < nc; ++i) {
      const int st = i % kStages;
      mbar_wait(&full_bar[st], (i / kStages) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + st * stage_bytes);
      const uint32_t sb = sa + 2 * a_half;
#pragma unroll
      for (int ks = 0; ks < kBK / 16; ++ks) {
        uint64_t ah, al, bh, bl;
        if (!kMN) {  // K-major: SBO 512 B (row groups), LBO 128 B (k-cores); 16 k = 2 cores
          ah = make_desc(sa + ks * 256, 128, 512);
          al = make_desc(sa + a_half + ks * 256, 128, 512);
          bh = make_desc(sb + ks * 256, 128, 512);
          bl = make_desc(sb + b_half + ks * 256, 128, 512);
        } else {     // MN-major: SBO 128 B (MN groups), LBO = MN width * 16 B (k groups)
          ah = make_desc(sa + ks * 4096, 2048, 128);
          al = make_desc(sa + a_half + ks * 4096, 2048, 128);
          const uint32_t kg = (uint32_t)N_pad * 16;
          bh = make_desc(sb + ks * 2 * kg, kg, 128);
          bl = make_desc(sb + b_half + ks * 2 * kg, kg, 128);
        }
        const uint32_t acc0 = (i > 0 || ks > 0) ? 1u : 0u;
        mma_bf16(tmem, ah, bh, idesc, acc0);
        mma_bf16(tmem, ah, bl, idesc, 1u);
        mma_bf16(tmem, al, bh, idesc, 1u);
      }
      mma_commit(&empty_bar[st]);
    }
    mma_commit(&done_bar);
  }
  __syncwarp();
  // epilogue (every warp): TMEM lane = tile row, warp w drains lane quadrant
  // w % 4, column part w / 4; 32 x 32 sub-tiles staged through smem so every
  // global store instruction writes contiguous 128 B row segments
  if (nc > 0) mbar_wait(&done_bar, 0);
  tc_fence_after();
  __syncthreads();
  {
    const int q = warp & 3;
    int cb, ce;
    epi_cols(warp >> 2, n_valid, cb, ce);
    float* stage_f = reinterpret_cast<float*>(smem) + warp * 32 * 32;
    const typename Epi::Key my_key = (m0 + q * 32 + lane < M) ? epi.key(m0 + q * 32 + lane) : 0;
    drain_cols(epi, tmem + ((uint32_t)(q * 32) << 16), stage_f, my_key, m0 + q * 32, M, cb, ce, n0, n_valid, lane,
               nc == 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, tmem_cols);
  kt_end(kt);
}

// ---------------------------------------------------------------------------
// Persistent, warp-specialised variant for the K-major GEMMs (forward and
// data gradient): one CTA per SM loops over 128 x N_pad output tiles
// (tile t = blockIdx.x + k * gridDim.x, the row count read from the device).
//   warp 0 lane 0 : TMA producer, runs ahead through the stage ring across
//                   tile boundaries
//   warp 1 lane 0 : tcgen05.mma issuer into one of TWO TMEM accumulators
//                   (2 x N_pad columns), tcgen05.commit -> acc_full[buf]
//   warps 2..     : epilogue (TMEM lane quadrant = warp % 4, column part
//                   (warp - 2) / 4), drain tile i
//                   while the MMAs of tile i+1 run; arrive acc_empty[buf]
// The grid is sized to the SMs, so a row bound far above the actual count
// costs no empty waves of 200 KB CTAs.
constexpr int kPThreads = 64 + 32 * kEpiWarps;

template <typename Epi>
__global__ void __launch_bounds__(kPThreads, 1) k_tsgemm_p(const __grid_constant__ CUtensorMap tmA,
                                                           const __grid_constant__ CUtensorMap tmB, Shape sh, Epi epi,
                                                           int N_pad, int n_tiles, uint32_t tmem_cols) {
  pdl_wait();
  KTimer* kt = g_kt ? g_kt + (Epi::kFwd ? kTGemmFwd : kTGemmBwd) : nullptr;
  kt_begin(kt);
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_slot;
  const int M = sh.M_dev ? *sh.M_dev : sh.M;
  const int K = sh.K;
  const int chunks = (K + kBK - 1) / kBK;
  const int m_tiles = (M + kTM - 1) / kTM;
  const int total = m_tiles * n_tiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t a_half = 8192;
  const uint32_t b_half = (uint32_t)N_pad * 64;
  const uint32_t stage_bytes = 2 * a_half + 2 * b_half;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      int i = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int m0 = (t / n_tiles) * kTM, n0 = (t % n_tiles) * N_pad;
        for (int c = 0; c < chunks; ++c, ++i) {
          const int st = i % kStages;
          if (i >= kStages) mbar_wait(&empty_bar[st], ((i / kStages) - 1) & 1);
          uint8_t* base = smem + st * stage_bytes;
          mbar_expect_tx(&full_bar[st], stage_bytes);
          tma_4d(base, &tmA, 0, 4 * c, m0 / 8, 0, &full_bar[st]);
          tma_4d(base + 2 * a_half, &tmB, 0, 4 * c, n0 / 8, 0, &full_bar[st]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc(kTM, N_pad, 0, 0);
      int i = 0, lt = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++lt) {
        const int buf = lt & 1;
        if (lt >= 2) mbar_wait(&acc_empty[buf], ((lt >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(buf * N_pad);
        for (int c = 0; c < chunks; ++c, ++i) {
          const int st = i % kStages;
          mbar_wait(&full_bar[st], (i / kStages) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + st * stage_bytes);
          const uint32_t sb = sa + 2 * a_half;
#pragma unroll
          for (int ks = 0; ks < kBK / 16; ++ks) {
            const uint64_t ah = make_desc(sa + ks * 256, 128, 512);
            const uint64_t al = make_desc(sa + a_half + ks * 256, 128, 512);
            const uint64_t bh = make_desc(sb + ks * 256, 128, 512);
            const uint64_t bl = make_desc(sb + b_half + ks * 256, 128, 512);
            const uint32_t acc0 = (c > 0 || ks > 0) ? 1u : 0u;
            mma_bf16(d, ah, bh, idesc, acc0);
            mma_bf16(d, ah, bl, idesc, 1u);
            mma_bf16(d, al, bh, idesc, 1u);
          }
          mma_commit(&empty_bar[st]);
        }
        mma_commit(&acc_full[buf]);
      }
    }
  } else {
    // epilogue warps 2 .. 2 + kEpiWarps: TMEM lanes [32 q, 32 q + 32),
    // q = warp % 4, column part (warp - 2) / 4
    const int q = warp & 3;
    float* stage_f = reinterpret_cast<float*>(smem + (size_t)kStages * stage_bytes) + (warp - 2) * 32 * 32;
    int lt = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++lt) {
      const int buf = lt & 1;
      const int m0 = (t / n_tiles) * kTM, n0 = (t % n_tiles) * N_pad;
      const int n_valid = min(N_pad, sh.N - n0);
      int cb, ce;
      epi_cols((warp - 2) >> 2, n_valid, cb, ce);
      const typename Epi::Key my_key = (m0 + q * 32 + lane < M) ? epi.key(m0 + q * 32 + lane) : 0;
      mbar_wait(&acc_full[buf], (lt >> 1) & 1);
      tc_fence_after();
      drain_cols(epi, tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * N_pad), stage_f, my_key, m0 + q * 32, M,
                 cb, ce, n0, n_valid, lane, false);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, tmem_cols);
  kt_end(kt);
}

__global__ void k_splitk_sum(const float* __restrict__ part, int splits, long long n, long long stride,
                             float* __restrict__ out) {
  pdl_wait();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float s = part[i];
    for (int z = 1; z < splits; ++z) s = __fadd_rn(s, part[z * stride + i]);
    out[i] = s;
  }
}

// pack X[rows x cols] (element (r, c) = transposed ? src[c*ld + r] : src[r*ld + c]) into a TS buffer
// sized for rows_alloc rows; zero padding up to the 128-row / 32-column boundaries
__global__ void k_ts_pack(const float* __restrict__ src, long long ld, int transposed, int rows, int cols,
                          int rows_pad, int nCG, long long plane, uint8_t* __restrict__ dst) {
  pdl_wait();
  const long long groups = (long long)rows_pad * nCG;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < groups;
       t += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(t / nCG);
    const int g = (int)(t - (long long)r * nCG);
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = g * 8 + e;
      v[e] = (r < rows && c < cols) ? (transposed ? src[(long long)c * ld + r] : src[(long long)r * ld + c]) : 0.f;
    }
    ts_store8(dst, nCG, plane, r, g, v);
  }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::mutex g_encode_mu;

int get_encode(const char* W) {
  std::lock_guard<std::mutex> lk(g_encode_mu);
  if (g_encode) return kOk;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
    return fail(W, kCuda, "cuTensorMapEncodeTiled unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return kOk;
}

// 4-D view (core 128 B, column group, row group, plane) of a TS buffer
int make_map(const char* W, CUtensorMap* map, const void* base, long long rows_alloc, int cols, int box_cg,
             int box_g) {
  int st = get_encode(W);
  if (st) return st;
  const long long rows_pad = ts_rows_pad(rows_alloc);
  const int nCG = ts_ncg(cols);
  cuuint64_t dims[4] = {64, (cuuint64_t)nCG, (cuuint64_t)(rows_pad / 8), 2};
  cuuint64_t strides[3] = {128, (cuuint64_t)nCG * 128, (cuuint64_t)ts_plane_bytes(rows_alloc, cols)};
  cuuint32_t box[4] = {64, (cuuint32_t)box_cg, (cuuint32_t)box_g, 2};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(W, kCuda, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return kOk;
}

inline int pad_n(int n) {
  int p = (n + 15) / 16 * 16;
  return p < 16 ? 16 : p;
}
inline uint32_t tmem_cols_for(int n) {
  uint32_t c = 32;
  while ((int)c < n) c <<= 1;
  return c;
}

// fwd / dgrad use the persistent warp-specialised kernel (epilogue of tile i
// overlapping the MMAs of tile i+1). Before the epilogue rework the one-tile
// kernel was faster below ~256K rows (C3 forward 0.152 vs 0.178 ms/step);
// with the vector epilogue the persistent kernel wins at every measured
// shape: C2 1.080 -> 1.105e6, C3 0.99 -> 1.02e6 seeds/s, C5 layer 0
// 0.63 -> 0.30 ms/step of forward GEMMs. The one-tile kernel k_tsgemm serves
// the split-K weight gradients only.

template <typename Epi>
int launch_persistent(const char* W, const CUtensorMap& a, const CUtensorMap& b, Shape sh, Epi e, int n_tile,
                      cudaStream_t stream) {
  const int n_tiles = (sh.N + n_tile - 1) / n_tile;
  const size_t smem = (size_t)kStages * (2 * 8192 + 2 * (size_t)n_tile * 64) + kEpiWarps * 32 * 32 * 4;
  {
    const int max_smem = kStages * (2 * 8192 + 2 * 256 * 64) + kEpiWarps * 32 * 32 * 4;
    const int sa = ensure_smem_attr((const void*)k_tsgemm_p<Epi>, max_smem, W);
    if (sa) return sa;
  }
  const long long tiles = ((sh.M + kTM - 1) / kTM) * (long long)n_tiles;
  const unsigned grid = (unsigned)(tiles < 1 ? 1 : (tiles < 148 ? tiles : 148));
  uint32_t cols = tmem_cols_for(2 * n_tile);
  if (cols > 512) cols = 512;
  { const cudaError_t _pe = hg::launch_pdl(k_tsgemm_p<Epi>, dim3(grid), dim3(kPThreads), smem, stream, a, b, sh, e,
                                           n_tile, n_tiles, cols);
    if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  return kOk;
}

template <bool kMN, typename Epi>
int launch(const char* W, const CUtensorMap& a, const CUtensorMap& b, Shape sh, Epi e, int n_tile, int splits,
           cudaStream_t stream) {
  if constexpr (!kMN) {
    // row-major products (forward / dgrad): persistent kernel, one K pass
    if (splits != 1) return fail(W, kBadArg, "split-K is for the weight gradient only");
    return launch_persistent(W, a, b, sh, e, n_tile, stream);
  }
  const int n_tiles = (sh.N + n_tile - 1) / n_tile;
  const size_t smem = (size_t)kStages * (2 * 8192 + 2 * (size_t)n_tile * 64);
  {
    const int max_smem = kStages * (2 * 8192 + 2 * 256 * 64);
    const int sa = ensure_smem_attr((const void*)k_tsgemm<kMN, Epi>, max_smem, W);
    if (sa) return sa;
  }
  // an empty row range (R_max == 0: everything pruned or injected) still
  // launches one CTA, which exits at once (m0 >= M)
  const long long mt = (sh.M + kTM - 1) / kTM;
  dim3 grid((unsigned)(mt > 0 ? mt : 1), (unsigned)(n_tiles > 0 ? n_tiles : 1), (unsigned)splits);
  { const cudaError_t _pe = hg::launch_pdl(k_tsgemm<kMN, Epi>, dim3(grid), dim3(kThreads), smem, stream, a, b, sh, e, n_tile, tmem_cols_for(n_tile)); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  return kOk;
}

inline bool vec_ok(const float* p, long long ld) {
  return ld % 4 == 0 && (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}
inline int n_tile_for(int N) { return N > 256 ? 256 : pad_n(N); }

}  // namespace
}  // namespace hg

using namespace hg;

extern "C" {

long long hg_ts_bytes(long long rows, int cols) { return ts_bytes(rows, cols); }

int hg_ts_pack(const float* src, long long ld, int transposed, int rows, int cols, long long rows_alloc, void* dst,
               cudaStream_t stream) {
  const long long rows_pad = ts_rows_pad(rows_alloc);
  const int nCG = ts_ncg(cols);
  { const cudaError_t _pe = hg::launch_pdl(k_ts_pack, dim3(grid_for(rows_pad * nCG, 256)), dim3(256), 0, stream, src, ld, transposed, rows, cols, (int)rows_pad, nCG,
                                                               ts_plane_bytes(rows_alloc, cols),
                                                               static_cast<uint8_t*>(dst)); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED("hg_ts_pack");
  return kOk;
}

// h_out[rows[i]] = relu?( A[i, :K1] . PT[:, :K1]^T ); A: TS [R_max x K1], PT: TS of P^T [N x K1]
int hg_ts_linear_fwd(const int32_t* R_dev, long long R_max, const void* A_ts, int K1, const void* PT_ts, int N,
                     const int32_t* rows, int relu, float* h_out, cudaStream_t stream) {
  const char* W = "hg_ts_linear_fwd";
  const int nt = n_tile_for(N);
  CUtensorMap a, b;
  int st = make_map(W, &a, A_ts, R_max, K1, 4, 16);
  if (!st) st = make_map(W, &b, PT_ts, N, K1, 4, nt / 8);
  if (st) return st;
  Shape sh{(int)R_max, N, K1, R_dev, nullptr, (K1 + kBK - 1) / kBK};
  return launch<false>(W, a, b, sh, EpiScatterRelu{rows, h_out, N, relu, vec_ok(h_out, N)}, nt, 1, stream);
}

// SG[R x K] = dz[R x N] . W[K x N]^T; dz: TS [R_max x N], W: TS [K x N]
int hg_ts_linear_dgrad(const int32_t* R_dev, long long R_max, const void* dz_ts, int N, const void* W_ts, int K,
                       float* SG, cudaStream_t stream) {
  const char* W = "hg_ts_linear_dgrad";
  const int nt = n_tile_for(K);
  CUtensorMap a, b;
  int st = make_map(W, &a, dz_ts, R_max, N, 4, 16);
  if (!st) st = make_map(W, &b, W_ts, K, N, 4, nt / 8);
  if (st) return st;
  Shape sh{(int)R_max, K, N, R_dev, nullptr, (N + kBK - 1) / kBK};
  // dgrad row stores: with the 8-warp swizzled-stage epilogue the 16-byte
  // vector stores win (C2 dgrad 0.040 -> 0.025 ms/step, step 0.663 -> 0.655
  // ms); with the old 4-warp padded stage, scalar stores had measured better
#ifndef HG_DGRAD_VEC
#define HG_DGRAD_VEC 1
#endif
  return launch<false>(W, a, b, sh, EpiStore{SG, K, HG_DGRAD_VEC ? vec_ok(SG, K) : false}, nt, 1, stream);
}

// dP[K1 x N] = A[:R, :K1]^T . dz[:R, :N]  (split-K over the rows, fixed-order sum)
int hg_ts_linear_wgrad(const int32_t* R_dev, long long R_max, const void* A_ts, int K1, const void* dz_ts, int N,
                       float* dP, float* partial, int splits, cudaStream_t stream) {
  const char* W = "hg_ts_linear_wgrad";
  if (splits < 1) splits = 1;
  const int chunks = (int)((R_max + kBK - 1) / kBK);
  int per = (chunks + splits - 1) / splits;
  if (per < 1) per = 1;
  splits = (chunks + per - 1) / per;
  if (splits < 1) splits = 1;
  const int nt = n_tile_for(N);
  CUtensorMap a, b;
  int st = make_map(W, &a, A_ts, R_max, K1, 16, 4);
  if (!st) st = make_map(W, &b, dz_ts, R_max, N, nt / 8, 4);
  if (st) return st;
  const long long stride = (long long)K1 * N;
  Shape sh{K1, N, (int)R_max, nullptr, R_dev, per};
  st = launch<true>(W, a, b, sh, EpiPartial{partial, N, stride, vec_ok(partial, N) && stride % 4 == 0}, nt, splits, stream);
  if (st) return st;
  { const cudaError_t _pe = hg::launch_pdl(k_splitk_sum, dim3(grid_for(stride, 256)), dim3(256), 0, stream, partial, splits, stride, stride, dP); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  return kOk;
}

}  // extern "C"
