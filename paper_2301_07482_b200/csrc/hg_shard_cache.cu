// Owner-sharded historical cache (semantics: oracle/shardcache.py).
//
// P ranks, rank r trains batch P*s + r at step s; node v belongs to owner o
// with bounds[o] <= v < bounds[o+1] (comms.py:329-337). Owner o keeps, per
// cache layer, the reference's ring state for its ids only, indexed locally
// (row_of[v - lo], admit_iter[v - lo]; row_owner holds global ids), in
// CUDA-IPC memory that every peer maps. One step:
//   lookups   k_shard_lookup: pure reads of the owners' state after the
//             previous step (cache.py:103-129 judged at the rank's own
//             iteration); hits are recorded as (owner, row) and injected by
//             k_inject_sharded straight from the owner's ring (NVLink on a
//             multi-GPU box); expired entries are only reported (exp list)
//   request   hg_cache_request (hg_cache.cu): the batch-wide admission rank
//             (cache.py:188-191) as per-position actions, in this rank's memory
//   barrier A every rank's lookups and request done (hg_peer_barrier)
//   commit    per owner: every rank's expiries (k_sc_invalidate, one count per
//             entry still held), then for r = 0..P-1 rank r's request
//             restricted to owned ids: gradient evictions, the ring write in
//             admit-rank order with the overwrite accounting, retained
//             refreshes (cache.py:131-204), and end_iteration(it_r)'s sweep
//             (cache.py:206-211,330-334)
//   barrier B signalled after the commit, awaited before the next lookups
// With P = 1 this is the single-GPU cache bit for bit (lookups precede the
// update inside an iteration, so deferring expiries changes nothing).
#include "hgb200.h"

#include <cmath>

#include "hg_common.cuh"
#include "hg_scan.cuh"
#include "hg_state.h"

namespace hg {
namespace {

constexpr unsigned long long kBarrierTimeoutNs = 120ull * 1000000000ull;

__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_acq_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ int owner_of(const long long* __restrict__ bounds, int P, long long v) {
  int o = 0;
  while (o + 1 < P && v >= bounds[o + 1]) ++o;
  return o;
}

// ---------------------------------------------------------------- lookups
// one thread per live position: owner, row and freshness of its id; a hit
// is recorded as hit_row[loc] = owner << kOwnerShift | row and its row is
// injected straight from the owner's ring (k_inject_sharded, one-sided NVLink
// reads on a multi-GPU box); expired entries are only reported
constexpr int kOwnerShift = 26;   // rows < 2^26 per owner ring, owners < 32
__global__ void __launch_bounds__(256) k_shard_lookup(const int32_t* n_live_dev, const int32_t* __restrict__ live,
                                                      const int32_t* __restrict__ src_nodes, int P,
                                                      const long long* __restrict__ bounds,
                                                      const int32_t* const* __restrict__ row_of,
                                                      const int32_t* const* __restrict__ admit_iter,
                                                      const int32_t* it_dev, double t_stale, int t_inf,
                                                      uint8_t* __restrict__ hit_flag, int32_t* __restrict__ hit_row,
                                                      int32_t* __restrict__ exp_ids, long long* req_hdr, long long* ctr) {
  pdl_wait();
  const int n = *n_live_dev;
  const int it = *it_dev;
  unsigned long long* c = reinterpret_cast<unsigned long long*>(ctr);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j - (threadIdx.x & 31) < n; j += gridDim.x * blockDim.x) {
    bool fresh = false, expired = false;
    if (j < n) {
      const int loc = live[j];
      const int v = src_nodes[loc];
      const int o = owner_of(bounds, P, v);
      const long long li = (long long)v - bounds[o];
      const int row = __ldcg(row_of[o] + li);
      if (row >= 0) {
        fresh = true;
        if (!t_inf) {
          const double age = (double)(it - __ldcg(admit_iter[o] + li));
          if (!(age <= t_stale)) {
            fresh = false;
            expired = true;
          }
        }
      }
      hit_flag[loc] = fresh;
      hit_row[loc] = fresh ? (int32_t)(((unsigned)o << kOwnerShift) | (unsigned)row) : -1;
      if (expired) {
        const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(req_hdr) + 3, 1ull);
        exp_ids[slot] = v;
      }
    }
    warp_count_add(c + kCtrHits, j < n && fresh);
    warp_count_add(c + kCtrMisses, j < n && !fresh);
  }
}

// h_out[r] = owner ring row of hit r (rows decoded from hit_row), a warp per
// 32 output rows, 16-byte pieces
__global__ void k_inject_sharded(const int32_t* n_dev, const uint8_t* __restrict__ flag,
                                 const int32_t* __restrict__ hit_row, const float* const* __restrict__ tables, int dim,
                                 float* __restrict__ h_out) {
  pdl_wait();
  const int n = *n_dev;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int nv = dim >> 2;
  for (int r0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; r0 < n; r0 += warps * 32) {
    const int r = r0 + lane;
    const bool f = r < n && flag[r];
    const int hr = f ? hit_row[r] : 0;
    unsigned m = __ballot_sync(0xffffffffu, f);
    while (m) {
      const int q = __ffs(m) - 1;
      m &= m - 1;
      const unsigned code = (unsigned)__shfl_sync(0xffffffffu, hr, q);
      const float* src = tables[code >> kOwnerShift] + (long long)(code & ((1u << kOwnerShift) - 1)) * dim;
      const uint4* s4 = reinterpret_cast<const uint4*>(src);
      uint4* d4 = reinterpret_cast<uint4*>(h_out + (long long)(r0 + q) * dim);
      for (int x = lane; x < nv; x += 32) d4[x] = __ldcg(s4 + x);
    }
  }
}

// request header: [0] n, [1] k, [2] it, [3] n_expired
__global__ void k_req_reset(long long* hdr, const int32_t* it_dev) {
  pdl_wait();
  hdr[0] = 0;
  hdr[1] = 0;
  hdr[2] = *it_dev;
  hdr[3] = 0;
  hdr[4] = 0;
}

// ---------------------------------------------------------------- commit
__global__ void k_sc_invalidate(int P, const int32_t* const* __restrict__ exps, const long long* const* __restrict__ hdrs,
                                long long lo, long long hi, int32_t* __restrict__ row_of,
                                int32_t* __restrict__ row_owner, long long* ctr) {
  pdl_wait();
  unsigned long long* c = reinterpret_cast<unsigned long long*>(ctr);
  for (int r = 0; r < P; ++r) {
    const long long n = __ldcg(hdrs[r] + 3);
    for (long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x; m < n; m += (long long)gridDim.x * blockDim.x) {
      const long long v = __ldcg(exps[r] + m);
      bool hit = false;
      if (v >= lo && v < hi) {
        const int old = atomicExch(row_of + (v - lo), -1);
        if (old >= 0) {
          row_owner[old] = -1;
          hit = true;
        }
      }
      warp_count_add(c + kCtrStalenessEvictions, hit);
      if (hit) atomicAdd(c + kCtrValid, (unsigned long long)-1ll);
    }
  }
}

// not admitted & held -> gradient eviction; admitted & computed & owned -> write flag
__global__ void k_sc_evict(const long long* __restrict__ hdr, const int32_t* __restrict__ req_id,
                           const uint8_t* __restrict__ req_act, long long lo, long long hi,
                           int32_t* __restrict__ row_of, int32_t* __restrict__ row_owner, uint8_t* __restrict__ wflag,
                           long long* ctr) {
  pdl_wait();
  const long long n = __ldcg(hdr);
  unsigned long long* c = reinterpret_cast<unsigned long long*>(ctr);
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    const long long v = __ldcg(req_id + j);
    const int act = __ldcg(req_act + j);
    const bool owned = v >= lo && v < hi;
    bool evicted = false;
    if (owned && act == 0) {
      const int r = row_of[v - lo];
      if (r >= 0) {
        row_owner[r] = -1;
        row_of[v - lo] = -1;
        evicted = true;
      }
    }
    wflag[j] = owned && act == 1;
    warp_count_add(c + kCtrGradientEvictions, evicted);
    if (evicted) atomicAdd(c + kCtrValid, (unsigned long long)-1ll);
  }
}

struct HdrCount {
  const long long* p;
  __device__ long long get() const { return __ldcg(p); }
};
struct StoreNW {
  long long* ctr;
  __device__ void operator()(int t) const { ctr[kCtrNWrite] = t; }
};

// first use of the owner's ring (cache.py:79-91 on the owner's node count):
// every thread derives the same capacity; one writes it
__device__ __forceinline__ long long sc_capacity(long long* ctr, long long nw, long long cap_fixed, long long window,
                                                 long long n_owned, long long limit, long long min_cap) {
  long long cap = ctr[kCtrCapacity];
  if (cap != 0 || nw == 0) return cap;
  if (cap_fixed > 0) {
    cap = cap_fixed;
  } else if (window == 0) {   // t_stale = inf
    cap = n_owned;
  } else {
    cap = 2 * (nw > 1 ? nw : 1) * window;
    const long long top = n_owned > 1 ? n_owned : 1;
    cap = cap < min_cap ? min_cap : cap;
    cap = cap > top ? top : cap;
  }
  if (cap > limit) cap = limit;
  return cap > 1 ? cap : 1;
}

__global__ void k_sc_release_writes(const int32_t* __restrict__ wlist, const int32_t* __restrict__ req_id,
                                    long long lo, int32_t* __restrict__ row_of, int32_t* __restrict__ row_owner,
                                    long long* ctr, long long cap_fixed, long long window, long long n_owned,
                                    long long limit) {
  pdl_wait();
  const long long nw = ctr[kCtrNWrite];
  if (nw == 0) return;
  const long long cap = sc_capacity(ctr, nw, cap_fixed, window, n_owned, limit, 64);
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr[kCtrCapacity] = cap;
  const long long w0 = nw >= cap ? nw - cap : 0;
  for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < nw - w0;
       w += (long long)gridDim.x * blockDim.x) {
    const long long v = __ldcg(req_id + wlist[w0 + w]);
    const int r = row_of[v - lo];
    if (r >= 0) {
      row_owner[r] = -1;
      row_of[v - lo] = -1;
      atomicAdd(reinterpret_cast<unsigned long long*>(ctr) + kCtrValid, (unsigned long long)-1ll);
    }
  }
}

__global__ void k_sc_ring_scan(const long long* __restrict__ hdr, double t_stale, int t_inf, long long lo,
                               int32_t* __restrict__ row_of, int32_t* __restrict__ row_owner,
                               const int32_t* __restrict__ admit_iter, long long* ctr) {
  pdl_wait();
  const long long nw = ctr[kCtrNWrite];
  if (nw == 0) return;
  const long long cap = ctr[kCtrCapacity];
  const int it = (int)__ldcg(hdr + 2);
  const long long header = ctr[kCtrHeader];
  const bool wrap_all = nw >= cap;
  const long long n = wrap_all ? cap : nw;
  unsigned long long* c = reinterpret_cast<unsigned long long*>(ctr);
  for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < n; w += (long long)gridDim.x * blockDim.x) {
    const long long row = wrap_all ? w : (header + w) % cap;
    const int old = row_owner[row];
    bool forced = false, late = false;
    if (old >= 0) {
      const int age = it - admit_iter[old - lo];
      forced = t_inf || (double)age < t_stale;
      late = !forced;
      row_of[old - lo] = -1;
      if (wrap_all) row_owner[row] = -1;
    }
    warp_count_add(c + kCtrForcedEvictions, forced);
    warp_count_add(c + kCtrWindowForced, forced);
    warp_count_add(c + kCtrStalenessEvictions, late);
    if (forced || late) atomicAdd(c + kCtrValid, (unsigned long long)-1ll);
  }
}

// one warp per written row; the embedding row is read from the requesting
// rank's request area (req_emb[j], peer memory over CUDA IPC)
__global__ void k_sc_write_rows(const int32_t* __restrict__ wlist, const int32_t* __restrict__ req_id,
                                const float* __restrict__ req_emb, const long long* __restrict__ hdr, int row_words,
                                long long lo, float* __restrict__ table, int32_t* __restrict__ row_of,
                                int32_t* __restrict__ row_owner, int32_t* __restrict__ admit_iter, long long* ctr) {
  pdl_wait();
  const long long nw = ctr[kCtrNWrite];
  if (nw == 0) return;
  const long long cap = ctr[kCtrCapacity];
  const long long header = ctr[kCtrHeader];
  const bool wrap_all = nw >= cap;
  const long long w0 = wrap_all ? nw - cap : 0;
  const int it = (int)__ldcg(hdr + 2);
  const int lane = threadIdx.x & 31;
  const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int nv = row_words >> 2;
  for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nw - w0; w += warps) {
    const int j = wlist[w0 + w];
    const long long v = __ldcg(req_id + j);
    const long long row = wrap_all ? w : (header + w) % cap;
    const uint4* s = reinterpret_cast<const uint4*>(req_emb + (long long)j * row_words);
    uint4* d = reinterpret_cast<uint4*>(table + row * row_words);
    for (int x = lane; x < nv; x += 32) d[x] = __ldcg(s + x);
    if (lane == 0) {
      row_owner[row] = (int32_t)v;
      row_of[v - lo] = (int32_t)row;
      admit_iter[v - lo] = it;
    }
  }
}

// commit (header, admissions, window, valid), retained refreshes and that
// batch's end_iteration sweep (cache.py:206-211,330-334: t_int = 0 never)
__global__ void k_sc_finish(const long long* __restrict__ hdr, const int32_t* __restrict__ req_id,
                            const uint8_t* __restrict__ req_act, long long lo, long long hi,
                            const int32_t* __restrict__ row_of, int32_t* __restrict__ admit_iter, int refresh,
                            long long t_int, long long* ctr, long long limit) {
  pdl_wait();
  if (refresh) {
    const long long k = __ldcg(hdr + 1);
    const int it = (int)__ldcg(hdr + 2);
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (long long)gridDim.x * blockDim.x) {
      if (__ldcg(req_act + j) != 2) continue;
      const long long v = __ldcg(req_id + j);
      if (v >= lo && v < hi && row_of[v - lo] >= 0) admit_iter[v - lo] = it;
    }
  }
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const long long nw = ctr[kCtrNWrite];
  if (nw != 0) {
    const long long cap = ctr[kCtrCapacity];
    const bool wrap_all = nw >= cap;
    const long long neff = wrap_all ? cap : nw;
    ctr[kCtrHeader] = wrap_all ? neff % cap : (ctr[kCtrHeader] + nw) % cap;
    ctr[kCtrAdmissions] += neff;
    ctr[kCtrWindowAdmissions] += neff;
    ctr[kCtrValid] += neff;
  }
  if (t_int < 1) return;
  const long long it = __ldcg(hdr + 2);
  if ((it + 1) % t_int != 0) return;
  const long long wa = ctr[kCtrWindowAdmissions], wf = ctr[kCtrWindowForced];
  long long cap = ctr[kCtrCapacity];
  if (cap > 0 && wa != 0 && (double)wf > 0.01 * (double)wa && cap < limit) cap = cap * 2 < limit ? cap * 2 : limit;
  ctr[kCtrCapacity] = cap;
  ctr[kCtrWindowAdmissions] = 0;
  ctr[kCtrWindowForced] = 0;
  ctr[kCtrHeader] = 0;
}

// ---------------------------------------------------------------- barrier
// st: [0] epoch (signals so far), [1] timeout flag (sticky), [2] timeout ns
__global__ void k_peer_signal(unsigned long long* my_flag, unsigned long long* st) {
  pdl_wait();
  const unsigned long long e = st[0] + 1ull;
  st[0] = e;
  __threadfence_system();
  st_rel_sys(my_flag, e);
}

__global__ void k_peer_wait(unsigned long long* const* flags, int P, unsigned long long* st) {
  pdl_wait();
  const unsigned long long e = st[0];
  const unsigned long long limit = st[2] ? st[2] : kBarrierTimeoutNs;
  if (st[1]) return;
  const unsigned long long t0 = gtimer_ns();
  for (int r = 0; r < P; ++r) {
    while (ld_acq_sys(flags[r]) < e) {
      if (gtimer_ns() - t0 > limit) {
        st[1] = 1ull;
        return;
      }
      __nanosleep(256);
    }
  }
  __threadfence_system();
}

#define HG_SC_LAUNCH(W, K, G, B, ...)                                                         \
  do {                                                                                      \
    const cudaError_t _pe = hg::launch_pdl(K, dim3(G), dim3(B), 0, stream, __VA_ARGS__);    \
    if (_pe != cudaSuccess) return hg::fail(W, hg::kCuda, cudaGetErrorString(_pe));         \
    HG_LAUNCHED(W);                                                                         \
  } while (0)

}  // namespace
}  // namespace hg

using namespace hg;

extern "C" {

int hg_cache_request_reset(long long* req_hdr, const int32_t* it_dev, cudaStream_t stream) {
  HG_SC_LAUNCH("hg_cache_request_reset", k_req_reset, 1, 1, req_hdr, it_dev);
  return kOk;
}

int hg_cache_lookup_sharded(const int32_t* n_live_dev, long long n_live_max, const int32_t* live,
                            const int32_t* src_nodes, long long n_src_max, int P, const long long* bounds,
                            const int32_t* const* row_of, const int32_t* const* admit_iter, const int32_t* it_dev,
                            double t_stale, uint8_t* hit_flag, int32_t* hit_row, int32_t* exp_ids, long long* req_hdr,
                            long long* layer_ctr, cudaStream_t stream) {
  const char* W = "hg_cache_lookup_sharded";
  if (P < 1 || P > 32) return fail(W, kBadArg, "bad world size (1..32)");
  HG_CHECK_CUDA(W, cudaMemsetAsync(hit_flag, 0, (size_t)(n_src_max > 0 ? n_src_max : 1), stream));
  if (n_live_max <= 0) return kOk;
  HG_SC_LAUNCH(W, k_shard_lookup, grid_for(n_live_max, 256), 256, n_live_dev, live, src_nodes, P, bounds, row_of,
               admit_iter, it_dev, t_stale, std::isinf(t_stale) ? 1 : 0, hit_flag, hit_row, exp_ids, req_hdr,
               layer_ctr);
  return kOk;
}

int hg_inject_rows_sharded(const int32_t* n_dev, long long n_max, const uint8_t* flag, const int32_t* hit_row,
                           const float* const* tables, int dim, float* h_out, cudaStream_t stream) {
  if (dim < 4 || (dim & 3)) return fail("hg_inject_rows_sharded", kBadArg, "rows must be a multiple of 4 floats");
  HG_SC_LAUNCH("hg_inject_rows_sharded", k_inject_sharded, grid_for(n_max * 32, 256, 148 * 16), 256, n_dev, flag,
               hit_row, tables, dim, h_out);
  return kOk;
}

long long hg_cache_apply_scratch_bytes(long long n_max) {
  const long long n = n_max + 16;
  return n * 4 + n + (scan_tiles(n_max) + 1) * 4 + 256;
}

int hg_cache_invalidate(int P, const int32_t* const* exp_ids, const long long* const* req_hdrs, long long n_max,
                        long long lo, long long hi, int32_t* row_of, int32_t* row_owner, long long* layer_ctr,
                        cudaStream_t stream) {
  const char* W = "hg_cache_invalidate";
  if (P < 1 || P > 64) return fail(W, kBadArg, "bad world size");
  HG_SC_LAUNCH(W, k_sc_invalidate, grid_for(n_max, 256, 148 * 4), 256, P, exp_ids, req_hdrs, lo, hi, row_of,
               row_owner, layer_ctr);
  return kOk;
}

int hg_cache_apply(const long long* req_hdr, const int32_t* req_id, const uint8_t* req_act, const float* req_emb,
                   long long n_max, int row_words, long long lo, long long hi, double t_stale, int refresh_retained,
                   long long cap_fixed, long long n_owned, long long limit, float* table, int32_t* row_of,
                   int32_t* row_owner, int32_t* admit_iter, long long* layer_ctr, void* scratch,
                   long long scratch_bytes, cudaStream_t stream) {
  const char* W = "hg_cache_apply";
  if (scratch_bytes < hg_cache_apply_scratch_bytes(n_max)) return fail(W, kBadArg, "scratch too small");
  if (row_words < 4 || (row_words & 3) || limit < 1) return fail(W, kBadArg, "bad row width / limit");
  if (n_max <= 0) return kOk;
  const long long nn = n_max + 16;
  int32_t* wlist = reinterpret_cast<int32_t*>(scratch);
  uint8_t* wflag = reinterpret_cast<uint8_t*>(wlist + nn);
  int* part = reinterpret_cast<int*>((reinterpret_cast<uintptr_t>(wflag + nn) + 15) & ~uintptr_t(15));
  const int t_inf = std::isinf(t_stale) ? 1 : 0;
  const long long window = t_inf ? 0 : (long long)(t_stale >= 1.0 ? std::floor(t_stale) : 1.0);
  const long long t_int = t_inf ? 0 : (long long)std::floor(t_stale);
  HG_SC_LAUNCH(W, k_sc_evict, grid_for(n_max, 256), 256, req_hdr, req_id, req_act, lo, hi, row_of, row_owner, wflag,
               layer_ctr);
  const int s = scan_launch<int>(W, FlagU8{wflag}, HdrCount{req_hdr}, n_max, part, EmitCompact{wlist},
                                 StoreNW{layer_ctr}, stream);
  if (s) return s;
  HG_SC_LAUNCH(W, k_sc_release_writes, grid_for(n_max, 256), 256, (const int32_t*)wlist, req_id, lo, row_of,
               row_owner, layer_ctr, cap_fixed, window, n_owned, limit);
  HG_SC_LAUNCH(W, k_sc_ring_scan, grid_for(n_max, 256), 256, req_hdr, t_stale, t_inf, lo, row_of, row_owner,
               (const int32_t*)admit_iter, layer_ctr);
  HG_SC_LAUNCH(W, k_sc_write_rows, grid_for(n_max * 32, 256, 148 * 16), 256, (const int32_t*)wlist, req_id, req_emb,
               req_hdr, row_words, lo, table, row_of, row_owner, admit_iter, layer_ctr);
  HG_SC_LAUNCH(W, k_sc_finish, refresh_retained ? grid_for(n_max, 256) : 1u, refresh_retained ? 256 : 32, req_hdr,
               req_id, req_act, lo, hi, (const int32_t*)row_of, admit_iter, refresh_retained, t_int, layer_ctr, limit);
  return kOk;
}

int hg_peer_signal(unsigned long long* my_flag, unsigned long long* state, cudaStream_t stream) {
  HG_SC_LAUNCH("hg_peer_signal", k_peer_signal, 1, 1, my_flag, state);
  return kOk;
}

int hg_peer_wait(unsigned long long* const* flags, int P, unsigned long long* state, cudaStream_t stream) {
  if (P < 1 || P > 64) return fail("hg_peer_wait", kBadArg, "bad world size");
  HG_SC_LAUNCH("hg_peer_wait", k_peer_wait, 1, 1, flags, P, state);
  return kOk;
}

}  // extern "C"
