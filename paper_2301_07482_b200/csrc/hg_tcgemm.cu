// K7: the dense per-layer transform on the 5th-generation tensor cores.
//
// C[M x N] (+)= A[M x K] . B[K x N] in fp32 storage, computed with tcgen05.mma
// kind::f16 (bf16 inputs, fp32 accumulators in TMEM) using the 3-term split
//   x = hi(x) + lo(x),  hi = bf16(x), lo = bf16(x - hi)
//   a.b ~= hi(a).hi(b) + hi(a).lo(b) + lo(a).hi(b)
// which keeps ~16 mantissa bits per product (relative error ~1e-5), well
// inside the 1e-3 fp32 tolerance of the north star, at bf16 tensor-core rate.
//
// One CTA = 4 warps owns a 128 x N tile (N <= 256, one TMEM accumulator of
// N fp32 columns). Per K-chunk of 32, all threads load fp32 operands from
// global memory (any of the layouts the GNN layer needs: row-major,
// transposed, bias-augmented), split them to bf16 hi/lo and store them in the
// canonical K-major no-swizzle core-matrix layout (8 rows x 16 B); one elected
// thread issues 6 MMAs (2 k-steps x 3 terms) and commits them to an mbarrier
// that releases the smem stage (2-stage ring). The epilogue drains TMEM with
// tcgen05.ld (warp w owns lanes 32w..32w+31 = tile rows) and applies the
// layer-specific epilogue (ReLU + scatter to the block output rows, plain
// store, or a split-K partial). Deterministic: fixed reduction order.
#include "hgb200.h"
#include <cuda_bf16.h>

#include "hg_common.cuh"

namespace hg {
namespace {

constexpr int kTM = 128;   // tile rows (MMA M)
constexpr int kBK = 32;    // K elements per chunk
constexpr int kThreads = 128;

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "HG_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra HG_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
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

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// K-major, no swizzle: core matrix = 8 rows x 16 B contiguous; LBO = distance
// between the two 8-element K halves of one MMA (k-cores), SBO = distance
// between 8-row groups. Version 1 = Blackwell descriptor format.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, both K-major
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// smem byte offset of element (row, k) in a [rows x kBK] bf16 K-major tile
__device__ __forceinline__ uint32_t tile_off(int row, int kcore) {
  return (uint32_t)((row >> 3) * (kBK / 8) * 128 + kcore * 128 + (row & 7) * 16);
}

__device__ __forceinline__ void split_store(uint8_t* hi_tile, uint8_t* lo_tile, int row, const float (&v)[kBK]) {
#pragma unroll
  for (int kc = 0; kc < kBK / 8; ++kc) {
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float a = v[kc * 8 + 2 * q], b = v[kc * 8 + 2 * q + 1];
      const __nv_bfloat16 ah = __float2bfloat16_rn(a), bh = __float2bfloat16_rn(b);
      const __nv_bfloat16 al = __float2bfloat16_rn(a - __bfloat162float(ah));
      const __nv_bfloat16 bl = __float2bfloat16_rn(b - __bfloat162float(bh));
      hw[q] = (uint32_t)__bfloat16_as_ushort(ah) | ((uint32_t)__bfloat16_as_ushort(bh) << 16);
      lw[q] = (uint32_t)__bfloat16_as_ushort(al) | ((uint32_t)__bfloat16_as_ushort(bl) << 16);
    }
    const uint32_t off = tile_off(row, kc);
    *reinterpret_cast<uint4*>(hi_tile + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(lo_tile + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  }
}

// ------------------------------------------------------------ operand views
// operand(r, k) for r < rows, k < cols (zero outside)
struct OpRowMajor {      // element = p[r * ld + k]   (K contiguous)
  const float* p;
  long long ld;
  __device__ __forceinline__ void load(int r, int rows, int k0, int cols, float (&v)[kBK]) const {
    if (r >= rows) {
#pragma unroll
      for (int k = 0; k < kBK; ++k) v[k] = 0.f;
      return;
    }
    const float* src = p + (long long)r * ld + k0;
    const bool vec_ok = (k0 + kBK <= cols) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
    if (vec_ok) {
#pragma unroll
      for (int k = 0; k < kBK; k += 4) {
        const float4 x = *reinterpret_cast<const float4*>(src + k);
        v[k] = x.x; v[k + 1] = x.y; v[k + 2] = x.z; v[k + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kBK; ++k) v[k] = (k0 + k < cols) ? src[k] : 0.f;
    }
  }
};

struct OpTransposed {    // element = p[k * ld + r]   (r contiguous)
  const float* p;
  long long ld;
  __device__ __forceinline__ void load(int r, int rows, int k0, int cols, float (&v)[kBK]) const {
#pragma unroll
    for (int k = 0; k < kBK; ++k) v[k] = (r < rows && k0 + k < cols) ? p[(long long)(k0 + k) * ld + r] : 0.f;
  }
};

// ---------------------------------------------------------------- epilogues
struct EpiScatterRelu {  // h_out[rows[i]][n] = act(acc)
  const int32_t* rows;
  float* out;
  int ldo;
  int relu;
  __device__ __forceinline__ void store(int i, int n, float x) const {
    if (relu) x = x > 0.f ? x : 0.f;
    out[(long long)rows[i] * ldo + n] = x;
  }
};
struct EpiStore {        // out[i][n] = acc
  float* out;
  long long ldo;
  __device__ __forceinline__ void store(int i, int n, float x) const { out[(long long)i * ldo + n] = x; }
};

struct GemmShape {
  int M, N, K;              // host upper bounds / exact values
  const int32_t* M_dev;     // optional device count replacing M
  const int32_t* K_dev;     // optional device count replacing K
  int k_chunks_per_split;   // split-K: chunks per blockIdx.z
  long long partial_stride; // split-K: elements between split partial outputs
};

template <typename OpA, typename OpB, typename Epi>
__global__ void __launch_bounds__(kThreads, 1) k_tcgemm(GemmShape sh, OpA opA, OpB opB, Epi epi, int N_pad,
                                                        uint32_t tmem_cols) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // per stage: A hi, A lo (128 x 32 bf16 = 8 KB each), B hi, B lo (N_pad x 32 bf16 each)
  const uint32_t a_bytes = kTM * kBK * 2;
  const uint32_t b_bytes = (uint32_t)N_pad * kBK * 2;
  const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tmem_slot;

  const int M = sh.M_dev ? *sh.M_dev : sh.M;
  const int K = sh.K_dev ? *sh.K_dev : sh.K;
  const int m0 = blockIdx.x * kTM;
  if (m0 >= M) return;
  const int n0 = blockIdx.y * N_pad;
  const int n_valid = min(N_pad, sh.N - n0);
  const int chunks_total = (K + kBK - 1) / kBK;
  const int c_begin = blockIdx.z * sh.k_chunks_per_split;
  const int c_end = min(chunks_total, c_begin + sh.k_chunks_per_split);
  const int warp = threadIdx.x >> 5;
  const int tid = threadIdx.x;

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t idesc = make_idesc(kTM, N_pad);

  int uses[2] = {0, 0};
  for (int c = c_begin; c < c_end; ++c) {
    const int st = (c - c_begin) & 1;
    uint8_t* base = smem + st * stage_bytes;
    uint8_t* a_hi = base;
    uint8_t* a_lo = base + a_bytes;
    uint8_t* b_hi = base + 2 * a_bytes;
    uint8_t* b_lo = b_hi + b_bytes;
    const int k0 = c * kBK;
    // global loads of the A row first (in flight while we wait for the stage)
    float v[kBK];
    opA.load(m0 + tid, M, k0, K, v);
    // the stage must be free: the MMAs issued two chunks ago have completed
    // (while this CTA loaded chunk c-1 the tensor cores worked on chunk c-2)
    if (uses[st] > 0) mbar_wait(&mbar[st], (uses[st] - 1) & 1);
    split_store(a_hi, a_lo, tid, v);
    for (int r = tid; r < N_pad; r += kThreads) {
      opB.load(n0 + r, n0 + n_valid, k0, K, v);
      split_store(b_hi, b_lo, r, v);
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t sa_hi = smem_u32(a_hi), sa_lo = smem_u32(a_lo);
      const uint32_t sb_hi = smem_u32(b_hi), sb_lo = smem_u32(b_lo);
      const uint32_t lbo = 128, sbo = (kBK / 8) * 128;
#pragma unroll
      for (int ks = 0; ks < kBK / 16; ++ks) {
        const uint32_t koff = ks * 256;  // 16 bf16 = 2 k-cores
        const uint32_t acc0 = (c > c_begin || ks > 0) ? 1u : 0u;
        mma_bf16(tmem, make_desc(sa_hi + koff, lbo, sbo), make_desc(sb_hi + koff, lbo, sbo), idesc, acc0);
        mma_bf16(tmem, make_desc(sa_hi + koff, lbo, sbo), make_desc(sb_lo + koff, lbo, sbo), idesc, 1u);
        mma_bf16(tmem, make_desc(sa_lo + koff, lbo, sbo), make_desc(sb_hi + koff, lbo, sbo), idesc, 1u);
      }
      mma_commit(&mbar[st]);
    }
    uses[st]++;
  }
  // drain: wait for the last commit on each used stage
  for (int st = 0; st < 2; ++st)
    if (uses[st] > 0) mbar_wait(&mbar[st], (uses[st] - 1) & 1);
  tc_fence_after();

  // Epilogue: TMEM lane = tile row, so each thread holds one row; stage 32x32
  // sub-tiles through shared memory (the operand stages are free now) so the
  // global stores are row-contiguous (one 128 B segment per row per warp op).
  const int lane = tid & 31;
  const bool have = c_end > c_begin;
  float* stage_f = reinterpret_cast<float*>(smem) + warp * 32 * 33;
  for (int c0 = 0; c0 < n_valid; c0 += 32) {
    float acc[32];
    if (have) {
      float* a0 = acc;
      tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, *reinterpret_cast<float(*)[16]>(a0));
      tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(c0 + 16), *reinterpret_cast<float(*)[16]>(a0 + 16));
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) stage_f[lane * 33 + j] = acc[j];
    __syncwarp();
    const int col = c0 + lane;
    for (int r = 0; r < 32; ++r) {
      const int row = m0 + warp * 32 + r;
      if (row < M && col < n_valid) epi.store(row, n0 + col, stage_f[r * 33 + lane]);
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, tmem_cols);
}

// deterministic split-K reduction: out[i] = sum_z part[z][i] (fixed order)
__global__ void k_splitk_sum(const float* __restrict__ part, int splits, long long n, long long stride,
                             float* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float s = part[i];
    for (int z = 1; z < splits; ++z) s = __fadd_rn(s, part[z * stride + i]);
    out[i] = s;
  }
}

struct EpiPartial {      // part[z][i][n] = acc
  float* part;
  long long ldo;
  long long stride;
  __device__ __forceinline__ void store(int i, int n, float x) const {
    part[(long long)blockIdx.z * stride + (long long)i * ldo + n] = x;
  }
};

inline int pad_n(int n) {
  int p = (n + 15) / 16 * 16;
  return p < 16 ? 16 : p;
}
inline uint32_t tmem_cols_for(int n) {
  uint32_t c = 32;
  while ((int)c < n) c <<= 1;
  return c;
}

template <typename OpA, typename OpB, typename Epi>
int launch(const char* W, GemmShape sh, OpA a, OpB b, Epi e, int splits, cudaStream_t stream) {
  const int n_tile = sh.N > 256 ? 256 : pad_n(sh.N);
  const int n_tiles = (sh.N + n_tile - 1) / n_tile;
  const size_t smem = 2 * (2 * kTM * kBK * 2 + 2 * (size_t)n_tile * kBK * 2);
  static int attr_dev = -1;  // one opt-in per instantiation (per process, device 0..)
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    const int max_smem = 2 * (2 * kTM * kBK * 2 + 2 * 256 * kBK * 2);
    cudaError_t err = cudaFuncSetAttribute(k_tcgemm<OpA, OpB, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           max_smem);
    if (err != cudaSuccess) return fail(W, kCuda, cudaGetErrorString(err));
    attr_dev = dev;
  }
  const long long mt = (sh.M + kTM - 1) / kTM;   // R_max == 0 still launches one (exiting) CTA
  dim3 grid((unsigned)(mt > 0 ? mt : 1), (unsigned)(n_tiles > 0 ? n_tiles : 1), (unsigned)splits);
  if (grid.x == 0) return kOk;
  k_tcgemm<OpA, OpB, Epi><<<grid, kThreads, smem, stream>>>(sh, a, b, e, n_tile, tmem_cols_for(n_tile));
  HG_LAUNCHED(W);
  return kOk;
}


}  // namespace
}  // namespace hg

using namespace hg;

extern "C" {

// z = A[:, :K1] . P  -> h_out[rows[i]] = relu?(z[i])   (nn.py:150,156 + 161-162 + 289)
// A: [R x ldA] row-major (R on device via R_dev), P: [K1 x N] row-major.
int hg_tc_linear_fwd(const int32_t* R_dev, long long R_max, const float* A, long long ldA, int K1, const float* P,
                     int N, const int32_t* rows, int relu, float* h_out, cudaStream_t stream) {
  GemmShape sh{(int)R_max, N, K1, R_dev, nullptr, (K1 + kBK - 1) / kBK, 0};
  return launch("hg_tc_linear_fwd", sh, OpRowMajor{A, ldA}, OpTransposed{P, N}, EpiScatterRelu{rows, h_out, N, relu},
                1, stream);
}

// SG[R x K] = dz[R x N] . W^T, W = P[:K] ([K x N] row-major)      (nn.py:171,175-176)
int hg_tc_linear_dgrad(const int32_t* R_dev, long long R_max, const float* dz, int N, const float* P, int K,
                       float* SG, cudaStream_t stream) {
  GemmShape sh{(int)R_max, K, N, R_dev, nullptr, (N + kBK - 1) / kBK, 0};
  return launch("hg_tc_linear_dgrad", sh, OpRowMajor{dz, N}, OpRowMajor{P, N}, EpiStore{SG, K}, 1, stream);
}

// dP[K1 x N] = A[:, :K1]^T . dz  (reduction over the R rows, split-K, fixed order)
// partial: caller scratch of splits * K1 * N floats.                (nn.py:170,173-174)
int hg_tc_linear_wgrad(const int32_t* R_dev, long long R_max, const float* A, long long ldA, int K1, const float* dz,
                       int N, float* dP, float* partial, int splits, cudaStream_t stream) {
  if (splits < 1) splits = 1;
  const int chunks = (int)((R_max + kBK - 1) / kBK);
  const int per = (chunks + splits - 1) / splits > 0 ? (chunks + splits - 1) / splits : 1;
  splits = (chunks + per - 1) / per > 0 ? (chunks + per - 1) / per : 1;
  const long long stride = (long long)K1 * N;
  GemmShape sh{K1, N, (int)R_max, nullptr, R_dev, per, stride};
  int st = launch("hg_tc_linear_wgrad", sh, OpTransposed{A, ldA}, OpTransposed{dz, N}, EpiPartial{partial, N, stride},
                  splits, stream);
  if (st) return st;
  k_splitk_sum<<<grid_for(stride, 256), 256, 0, stream>>>(partial, splits, stride, stride, dP);
  HG_LAUNCHED("hg_tc_linear_wgrad");
  return kOk;
}


}  // extern "C"
