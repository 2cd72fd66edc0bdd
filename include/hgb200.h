/*
 * hgb200.h — C-ABI of the B200-native ReFresh per-iteration data path.
 *
 * The reference (`histgnn`, /root/reference/pkg/src/histgnn) is a pure-Python
 * package: its "plugin boundary" is its Python module API, and there is no FFI.
 * Each entry point below replaces the compute inside one reference function;
 * the Python package `paper_2301_07482_b200` keeps the reference signatures and
 * binds these symbols with ctypes.
 *
 * Conventions (all functions):
 *   - plain pointers + sizes, no torch types; every pointer is device memory
 *     (or UVA-mapped host memory where stated) owned by the caller;
 *   - asynchronous on the given stream; no host synchronisation inside;
 *   - counts produced on the device are passed as `const int32_t* *_dev`
 *     together with a host upper bound `*_max` that sizes the launch grid;
 *   - return 0 on success, < 0 on error; hg_last_error() describes it;
 *   - node ids and local ids are int32 (N < 2^31); full-graph CSR2 offsets int64;
 *   - scratch memory is caller supplied; *_scratch_bytes() give the sizes.
 * Compiled for sm_100a only.
 */
#ifndef HGB200_H_
#define HGB200_H_

#include <cuda_runtime.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int hg_version(void);
const char* hg_last_error(void);
int hg_device_sync(void);
/* number of hand-written hg kernels launched by this process (library GEMMs excluded) */
long long hg_kernel_launches(void);
/* step timeline probe: one-thread kernel writing %globaltimer (ns) to *slot */
int hg_mark_time(unsigned long long* slot, cudaStream_t stream);
/* add the n hg kernels of a replayed CUDA graph (counted at its capture) */
void hg_count_graph_replay(long long n);
/* instantiate a captured cudaGraph_t with per-node priorities
 * (cudaGraphInstantiateFlagUseNodePriority), launch it, destroy it */
int hg_graph_instantiate(void* graph, void** exec_out);
int hg_graph_launch(void* exec, cudaStream_t stream);
int hg_graph_exec_destroy(void* exec);
/* device-side kernel timers for kernels replayed inside CUDA graphs: buf is
 * u64[8 * 8] (per timer: start=~0, end, total_ns, launches, ...), NULL = off.
 * Timer 0 = k_load_rows, 1 = k_aggregate, 2 = k_transpose_agg, 3 = k_select. */
int hg_set_kernel_timers(void* buf);
/* IterMetrics row of one step (trainer.py:86-104,407-421), written on the
 * device at the end of the step: out = [*loss, vecs[...] - prev (prev := now),
 * vecs[l][valid_idx] for the nvec-1 layer vectors, *n_src0, counts[0..n)];
 * vecs / lens: device arrays of the counter vectors (layers, then global). */
int hg_metrics_row(const long long* const* vecs, const int* lens, int nvec, long long* prev, const double* loss,
                   const int32_t* n_src0, const int32_t* counts, int ncounts, int valid_idx, double* out,
                   cudaStream_t stream);

/* ---- K1+K2 sampler: histgnn/sampler.py:118-163 (_sample_in_neighbors,
 * _build_block), called per layer by sampler.py:166-190 (sample_layered).
 * state_dev (u64[6], device): [0..3] = PCG64 state hi/lo, inc hi/lo of
 * default_rng(SeedSequence((seed, batch))) (sampler.py:104-106); [4] = draws
 * consumed before this layer (advanced by sum(deg)); [5] = g2l stamp epoch
 * (start at 1, advanced per layer). Device-resident so a captured CUDA graph
 * replays with new batches.
 * Outputs: block CSR offsets blk_off[F+1] (start = blk_off[i], end = blk_end[i]),
 * dst_deg[F], col_local[E], src_out = frontier ++ sorted new nodes,
 * counts_dev[0] = E, counts_dev[1] = n_src. g2l (int64[N]) must start as -1;
 * bitmap (uint32[ceil(N/32)]) must start zero and is left zero. */
long long hg_sample_layer_scratch_bytes(long long F_max, long long num_nodes);
int hg_sample_layer(const int64_t* g_start, const int64_t* g_end, const int32_t* g_col, long long num_nodes,
                    const int32_t* frontier, const int32_t* F_dev, long long F_max, int fanout,
                    unsigned long long* state_dev, int64_t* g2l,
                    uint32_t* bitmap, int64_t* cand_off, int32_t* blk_off, int32_t* blk_end, int32_t* dst_deg,
                    int32_t* src_flat, int32_t* col_local, int32_t* src_out, int32_t* counts_dev, void* scratch,
                    long long scratch_bytes, cudaStream_t stream);

/* ---- K3 prune: histgnn/trainer.py:166-207 (prune_with_cache) for one block,
 * incl. graphs.py:123-127 (Csr2Graph.prune_many). counts_dev[0] = |compute_rows|,
 * counts_dev[1] = |layer_live|; global_ctr[2] += prune writes. */
long long hg_prune_scratch_bytes(long long n_src_max);
int hg_prune_block(const int32_t* n_dst_dev, long long n_dst_max, const int32_t* n_src_dev, long long n_src_max,
                   const uint8_t* live_dst, const uint8_t* inj_dst, const int32_t* start, int32_t* end,
                   const int32_t* col, uint8_t* keep, int32_t* compute_rows, int32_t* pos_of, uint8_t* src_mask,
                   int32_t* live_src, int32_t* counts_dev, long long* global_ctr, void* scratch,
                   long long scratch_bytes, cudaStream_t stream);

/* ---- K4 cache lookup: histgnn/cache.py:103-129 (_LayerCache.lookup) via
 * cache.py:269-285 (HistCache.lookup, layer >= 1). t_stale may be +inf;
 * the current iteration is read from it_dev. */
int hg_cache_lookup(const int32_t* n_live_dev, long long n_live_max, const int32_t* live, const int32_t* src_nodes,
                    long long n_src_max, int32_t* row_of, const int32_t* admit_iter, int32_t* row_owner,
                    const int32_t* it_dev, double t_stale, uint8_t* hit_flag, int32_t* hit_row, long long* layer_ctr,
                    cudaStream_t stream);

/* ---- K5 feature load: histgnn/trainer.py:326-343 (Trainer._load_input),
 * cache.py:274-284 (feature region), trainer.py:213-228 (FeatureSource.fetch).
 * feats may be a UVA pointer to pinned host memory. dtype 0 = fp32, 1 = fp16. */
long long hg_load_features_scratch_bytes(long long n_live_max);
/* scratch may be NULL (register gather); with it, fp32 rows are copied by TMA bulk copies */
int hg_load_features(const int32_t* n_live_dev, long long n_live_max, const int32_t* live, const int32_t* src_nodes,
                     const int32_t* feature_row_of, const void* region, const void* feats, int dim, int dtype,
                     float* h_out, long long* global_ctr, void* scratch, long long scratch_bytes,
                     cudaStream_t stream);

/* Sharded feature table: miss rows of node id are read from
 * shard o with bounds[o] <= id < bounds[o+1] at shard_ptrs[o] + (id - bounds[o])
 * * dim; shard_ptrs (device array [P], P <= 16) may hold CUDA-IPC mappings of
 * peer GPUs' shards (one-sided NVLink reads). Partition as
 * comms.py:329-337 (partition_features). Rows from shards != local_shard are
 * counted in global_ctr[3]. */
int hg_load_features_sharded(const int32_t* n_live_dev, long long n_live_max, const int32_t* live,
                             const int32_t* src_nodes, const int32_t* feature_row_of, const void* region,
                             const void* const* shard_ptrs, const long long* shard_bounds, int num_shards,
                             int local_shard, int dim, int dtype, float* h_out, long long* global_ctr,
                             long long* owner_rows, cudaStream_t stream);
/* owner_rows (int64[P] or NULL): rows read from each owner's shard, the
 * transfer sizes of comms.py:326-337 (requests_for_batch) taken from the real
 * reads; the accounting of comms.py:283-323 is derived from them on the host
 * (distributed.transfer_accounting).
 * shard allocation and CUDA IPC export/open/close of peer shards */
int hg_device_alloc(long long bytes, void** out);
int hg_device_free(void* p);
long long hg_ipc_handle_bytes(void);
int hg_ipc_export(void* p, void* handle_out);
int hg_ipc_open(const void* handle, void** out);
int hg_ipc_close(void* p);

/* ---- K6 block aggregation: histgnn/nn.py:101-128,142-156 (_gcn_matrix,
 * _mean_matrix, _layer_forward_ctx). kind 0 = GCN, 1 = SAGE_MEAN. */
int hg_aggregate_fwd(int kind, const int32_t* R_dev, long long R_max, const int32_t* rows, const int32_t* start,
                     const int32_t* end, const int32_t* col, const int32_t* dst_deg, const int32_t* src_deg,
                     const float* h_in, int d, void* A_ts, float* row_w, cudaStream_t stream);
/* K5 fused into K6 (layer 0): hg_resolve_feature_rows writes rowp[live[i]]
 * = the address of live source i's feature row (static region row, table row
 * or owner-shard row over NVLink; shard_ptrs NULL = unsharded `feats`) with
 * hg_load_features' accounting; hg_aggregate_fwd_rows aggregates layer 0
 * reading those rows in place (dtype 0 fp32 / 1 fp16, d = padded width), so
 * no fp32 copy of the input frontier is materialised. Bit-identical to
 * hg_load_features + hg_aggregate_fwd. */
int hg_resolve_feature_rows(const int32_t* n_live_dev, long long n_live_max, const int32_t* live,
                            const int32_t* src_nodes, const int32_t* feature_row_of, const void* region,
                            const void* feats, const void* const* shard_ptrs, const long long* shard_bounds,
                            int num_shards, int local_shard, int dim, int dtype, unsigned long long* rowp,
                            long long* global_ctr, long long* owner_rows, cudaStream_t stream);
/* hg_aggregate_fwd_rows: dtype 0 fp32 / 1 fp16 feature rows; dtype 2 = fp32
 * rows of a hidden layer (layer output + cache-hit rows, hg_resolve_hit_rows) */
int hg_aggregate_fwd_rows(int kind, const int32_t* R_dev, long long R_max, const int32_t* rows, const int32_t* start,
                          const int32_t* end, const int32_t* col, const int32_t* dst_deg, const int32_t* src_deg,
                          const unsigned long long* rowp, int dtype, int d, void* A_ts, float* row_w,
                          cudaStream_t stream);

/* ---- K7 on tcgen05 over TS operands (bf16 hi/lo core-matrix tiles in HBM, written by
 * hg_aggregate_fwd / hg_gather_dz / hg_ts_pack; layout in csrc/hg_ts.cuh). Each K-chunk
 * stage is one 4-D TMA box per operand (cp.async.bulk.tensor) into a 4-stage smem ring;
 * one thread issues tcgen05.mma; fp32 accumulators in TMEM (csrc/hg_tsgemm.cu).
 *   fwd:   h_out[rows[i]] = relu?(A_ts[i,:K1] . PT_ts^T),  PT_ts = TS(P^T)   nn.py:150,156,289
 *   dgrad: SG = dz_ts . W_ts^T,  W_ts = TS(P[:K])                           nn.py:171,175-176
 *   wgrad: dP = A_ts^T . dz_ts over the rows (split-K, fixed-order sum)       nn.py:170,173-174 */
long long hg_ts_bytes(long long rows, int cols);
/* pack X[rows x cols] (X(r,c) = transposed ? src[c*ld+r] : src[r*ld+c]) into a TS buffer sized for rows_alloc rows */
int hg_ts_pack(const float* src, long long ld, int transposed, int rows, int cols, long long rows_alloc, void* dst,
               cudaStream_t stream);
int hg_ts_linear_fwd(const int32_t* R_dev, long long R_max, const void* A_ts, int K1, const void* PT_ts, int N,
                     const int32_t* rows, int relu, float* h_out, cudaStream_t stream);
int hg_ts_linear_dgrad(const int32_t* R_dev, long long R_max, const void* dz_ts, int N, const void* W_ts, int K,
                       float* SG, cudaStream_t stream);
int hg_ts_linear_wgrad(const int32_t* R_dev, long long R_max, const void* A_ts, int K1, const void* dz_ts, int N,
                       float* dP, float* partial, int splits, cudaStream_t stream);

/* ---- GAT block layer (BASELINE config 5). No reference implementation exists
 * (histgnn/nn.py:28-30 has GCN / SAGE_MEAN only); the layer is defined by the CPU
 * restatement oracle/gat.py (layer_forward / layer_backward), which these follow:
 *   scores:    el[j,h] = <z_j,h , a_src,h>, er[j,h] = <z_j,h , a_dst,h> over the live rows
 *   aggregate: h_out[rows[r]] = relu?(sum_j softmax_j(leaky(el_j + er_i)) z_j + bias) over the
 *              surviving in-edges of i = rows[r] plus the self loop; mx / ssum [R x H] kept
 *   bwd_dst:   gz [R x HF] (ReLU-masked), cc = sum_j a da, der = sum_j ds        [R x H],
 *              per-CTA partials of d bias = sum gz and d a_dst = sum der z_i
 *   bwd_src:   dz_j (TS, compact over live) = sum_i a_ij gz_i + del_j a_src (+ der_j a_dst), del [n_live x H],
 *              per-CTA partials of d a_src = sum del z_j
 *   param_grads: d a_src, d a_dst, d bias (fixed-order column sums)
 *   scatter_norms: d_in[live[k]] = SG[k], fp64 norms (nn.py:346-349)
 * HF = d_out <= 512, H <= 8 heads, HF % H == 0. */
int hg_gat_scores(const int32_t* n_live_dev, long long n_live_max, const int32_t* live, const float* z, int HF, int H,
                  const float* att_src, const float* att_dst, float* el, float* er, cudaStream_t stream);
int hg_gat_aggregate(const int32_t* R_dev, long long R_max, const int32_t* rows, const int32_t* start,
                     const int32_t* end, const int32_t* col, const float* z, const float* el, const float* er, int HF,
                     int H, const float* bias, int relu, float* h_out, float* mx, float* ssum, cudaStream_t stream);
int hg_gat_bwd_dst(const int32_t* R_dev, long long R_max, const int32_t* rows, const int32_t* start,
                   const int32_t* end, const int32_t* col, const float* z, const float* el, const float* er,
                   const float* mx, const float* ssum, const float* d_h, const float* h_out, int relu, int HF, int H,
                   float* gz, float* cc, float* der, float* part, cudaStream_t stream);
int hg_gat_bwd_src(const int32_t* n_live_dev, long long n_live_max, const int32_t* live, const int32_t* seg_lo,
                   const int32_t* seg_hi, const unsigned* csc_pos, const int32_t* rows, const int32_t* n_dst_dev,
                   const int32_t* pos_of, const float* z, const float* el, const float* er, const float* mx,
                   const float* ssum, const float* gz, const float* cc, const float* der, const float* att_src,
                   const float* att_dst, int HF, int H, void* dz_ts, float* del, float* part, cudaStream_t stream);
long long hg_gat_param_scratch_bytes(int HF);
/* part buffers of bwd_dst ([grid][2][HF]: bias, a_dst) and bwd_src ([grid][HF]: a_src), summed in a fixed order */
int hg_gat_param_grads(long long R_max, long long n_live_max, int HF, const float* part_dst, const float* part_src,
                       float* d_att_src, float* d_att_dst, float* d_bias, cudaStream_t stream);
int hg_gat_scatter_norms(const int32_t* n_live_dev, long long n_live_max, const int32_t* live, const float* SG, int d,
                         float* d_in, double* norms, cudaStream_t stream);

/* ---- forward epilogue: nn.py:161-162,288-293 (ReLU, h_full[rows], injected rows) */
int hg_scatter_rows(const int32_t* R_dev, long long R_max, const int32_t* rows, const float* Z, int dout, int relu,
                    float* h_out, cudaStream_t stream);
int hg_inject_rows(const int32_t* n_dev, long long n_max, const uint8_t* flag, const int32_t* hit_row,
                   const float* table, int dim, float* h_out, cudaStream_t stream);
/* cache-hit rows read in place (the engine's alternative to hg_inject_rows for
 * layers >= 1): rowp[r] = flagged r ? address of its cache row (table row, or
 * with `tables` the owner ring row of owner << 26 | row) : h_out + r * dim;
 * the next layer's aggregation reads its sources through rowp
 * (hg_aggregate_fwd_rows, dtype 0), so no hit row is copied. */
int hg_resolve_hit_rows(const int32_t* n_dev, long long n_max, const uint8_t* flag, const int32_t* hit_row,
                        const float* table, const float* const* tables, int dim, const float* h_out,
                        unsigned long long* rowp, cudaStream_t stream);

/* ---- loss: nn.py:326-343 (cross_entropy, fp64) */
int hg_cross_entropy(const float* logits, const int32_t* labels, int B, int C, float* dlogits, double* row_logp,
                     double* loss, cudaStream_t stream);

/* ---- K8 backward: nn.py:166-177,300-320 (_layer_backward, backward) */
int hg_gather_dz(const int32_t* R_dev, long long R_max, const int32_t* rows, const float* d_h, const float* h_out,
                 int dout, int relu, void* dz_ts, cudaStream_t stream);
/* GAT layer-0 transform operand read in place: row k of A_ts (TS layout for
 * n_max rows) = the feature row at rowp[rows[k]] (dtype 0 fp32, 1 fp16 -> fp32),
 * for k < *n_dev; padding rows of the last tile zeroed. The fp32 copy of the
 * input frontier (hg_load_features) and its re-gather are not needed.
 * Reference: oracle/gat.py layer_forward (z = h_in[live] W). */
int hg_gather_rows_ts(const int32_t* n_dev, long long n_max, const int32_t* rows, const unsigned long long* rowp,
                      int dtype, int d, void* A_ts, cudaStream_t stream);
long long hg_csc_scratch_bytes(long long E_max, long long n_src_max);
int hg_build_csc(const int32_t* n_dst_dev, const int32_t* blk_off, const uint8_t* keep, const int32_t* pos_of,
                 const int32_t* col, long long E_max, long long n_src_max, unsigned* keys_sorted,
                 unsigned* vals_sorted, int32_t* seg_lo, int32_t* seg_hi, void* scratch, long long scratch_bytes,
                 cudaStream_t stream);
/* K8 + K9 fused: transposed aggregation + nn.py:346-349 (node_grad_norms) */
/* need_row (uint8 per source row, may be NULL): rows with 0 get their fp64
 * norm only, no gradient row (the next layer does not compute them);
 * row_w (SAGE, may be NULL): the per-compute-row mean weights 1/cnt written
 * by hg_aggregate_fwd[_rows] (row_w there, may be NULL);
 * dz_ts (may be NULL): instead of d_in rows, write the previous layer's dz
 * operand (hg_gather_dz fused): row pos_prev[c] = d_in[c] masked by
 * h_prev[c] > 0 when relu_prev, TS layout for R_prev_max rows, padding rows
 * of the last tile up to the device count *R_prev_dev zeroed */
int hg_transpose_agg(int kind, const int32_t* n_live_dev, long long n_live_max, const int32_t* live,
                     const int32_t* seg_lo, const int32_t* seg_hi, const unsigned* vals_sorted, const int32_t* rows,
                     const int32_t* start, const int32_t* end, const int32_t* dst_deg, const int32_t* src_deg,
                     const int32_t* n_dst_dev, const int32_t* pos_of, const float* SG, int ldSG, int d,
                     float* d_in, double* norms, const uint8_t* need_row, const float* row_w,
                     void* dz_ts, const int32_t* R_prev_dev, long long R_prev_max, const int32_t* pos_prev,
                     const float* h_prev, int relu_prev, cudaStream_t stream);
int hg_row_norms(const float* x, long long n, int d, double* out, cudaStream_t stream);

/* ---- K11 optimizer: nn.py:355-360 (sgd_step) */
int hg_sgd(float* params, const float* grads, long long n, float eta, cudaStream_t stream);
/* Data-parallel gradient average fused with SGD over NVLink peer memory, the
 * alternative to an NCCL all-reduce hook before hg_sgd (histgnn/trainer.py:423-433,
 * nn.py:355-360 with gradients averaged over P ranks). my_slots: this rank's
 * 2 x n float exchange area, my_flag: its u64 flag word (both CUDA-IPC
 * exported); slots[r] / flags[r]: device arrays with every rank's mapping;
 * state: 8 u64 words, zero except [4] = peer-wait timeout in ns (0 = 120 s);
 * a peer that misses it sets state[3] and the update is skipped (no trap; the
 * host checks state[3]). Two launches, no host sync; sums in rank order so
 * every rank applies identical bits. */
int hg_p2p_allreduce_sgd(float* params, const float* grads, long long n, float* my_slots,
                         unsigned long long* my_flag, const float* const* slots, unsigned long long* const* flags,
                         int P, unsigned long long* state, float eta, cudaStream_t stream);

/* ---- K10 cache update: histgnn/cache.py:188-204 (_LayerCache.update) via
 * cache.py:289-322 (HistCache.update_cache), with _write/_release/
 * _count_overwrites cache.py:131-186. Two stages so the host can size the
 * ring table on first use (cache.py:79-91) after reading n_write. In
 * hg_cache_write, `cap` is the number of ALLOCATED table rows (grid bound);
 * the logical ring capacity is read from layer_ctr[9] on the device, so the
 * doublings of cache.py:93-101 need no reallocation while it fits. */
long long hg_cache_update_scratch_bytes(long long n_max);
int hg_cache_rank(const int32_t* n_dev, int n_max, double p_grad, const int32_t* live, const int32_t* src_nodes,
                  const double* norms, const uint8_t* computed_flag, int32_t* row_of, int32_t* row_owner,
                  long long* layer_ctr, void* scratch, long long scratch_bytes, cudaStream_t stream);
int hg_cache_write(int n_max, int cap, int H, const int32_t* it_dev, double t_stale, int refresh_retained,
                   const int32_t* live, const float* emb, float* table, int32_t* row_of, int32_t* row_owner,
                   int32_t* admit_iter, long long* layer_ctr, void* scratch, long long scratch_bytes,
                   cudaStream_t stream);

/* ---- end-of-window sweep: histgnn/cache.py:206-211 (_LayerCache.sweep) on the
 * device: double the capacity (up to `limit`, rows already allocated) when the
 * window's forced overwrites exceed 1% of its admissions, then reset the window
 * counters and the ring header. No host read. */
int hg_cache_sweep(long long* layer_ctr, long long limit, cudaStream_t stream);

/* ---- owner-sharded cache (semantics: oracle/shardcache.py;
 * kernels: csrc/hg_shard_cache.cu). Node v is owned by o with
 * bounds[o] <= v < bounds[o+1] (comms.py:329-337); an owner's row_of /
 * admit_iter are indexed by v - bounds[o], its row_owner holds global ids.
 * Request area (the requesting rank's IPC-mapped memory): per rank position j
 * req_id, req_act, req_src and, for writes, the row req_emb[j]; header
 * int64[8]: [0] n, [1] k, [2] iteration, [3] expired count.
 *
 * hg_cache_request_reset: start of a step (hdr = {0, 0, *it_dev, 0}).
 * hg_cache_lookup_sharded: cache.py:103-129 as a pure read of every owner's
 *   state (pointer tables of P <= 32 entries, peer mappings over CUDA IPC);
 *   hit_row[loc] = owner << 26 | ring row, expired ids appended to exp_ids
 *   (not invalidated: the owners apply them at commit).
 * hg_inject_rows_sharded: h_out[r] = the owner ring row of every flagged r
 *   (tables = the P ring base pointers).
 * hg_cache_request: cache.py:188-191's admission rank of one batch as actions
 *   (0 evict-if-held, 1 write, 2 retained) in rank order; touches no state.
 * hg_cache_invalidate / hg_cache_apply: owner side of the commit: all ranks'
 *   expiries (cache.py:106-115), then one rank's request restricted to owned
 *   ids (cache.py:131-204) and that batch's end_iteration sweep (:206-211,
 *   :330-334). cap_fixed = ceil(capacity / P) or -1; n_owned / limit bound
 *   the first-use sizing and growth (cache.py:79-101).
 * hg_peer_signal / hg_peer_wait: device barrier over IPC-mapped u64 flags;
 *   state u64[4] = {epoch, timeout flag (sticky), timeout ns (0 = 120 s)}. */
int hg_cache_request_reset(long long* req_hdr, const int32_t* it_dev, cudaStream_t stream);
int hg_cache_lookup_sharded(const int32_t* n_live_dev, long long n_live_max, const int32_t* live,
                            const int32_t* src_nodes, long long n_src_max, int P, const long long* bounds,
                            const int32_t* const* row_of, const int32_t* const* admit_iter, const int32_t* it_dev,
                            double t_stale, uint8_t* hit_flag, int32_t* hit_row, int32_t* exp_ids, long long* req_hdr,
                            long long* layer_ctr, cudaStream_t stream);
int hg_inject_rows_sharded(const int32_t* n_dev, long long n_max, const uint8_t* flag, const int32_t* hit_row,
                           const float* const* tables, int dim, float* h_out, cudaStream_t stream);
int hg_cache_request(const int32_t* n_dev, int n_max, double p_grad, const int32_t* live, const int32_t* src_nodes,
                     const double* norms, const uint8_t* computed_flag, const float* emb, int row_words,
                     int32_t* req_id, uint8_t* req_act, int32_t* req_src, float* req_emb, long long* req_hdr,
                     void* scratch, long long scratch_bytes, cudaStream_t stream);
long long hg_cache_apply_scratch_bytes(long long n_max);
int hg_cache_invalidate(int P, const int32_t* const* exp_ids, const long long* const* req_hdrs, long long n_max,
                        long long lo, long long hi, int32_t* row_of, int32_t* row_owner, long long* layer_ctr,
                        cudaStream_t stream);
int hg_cache_apply(const long long* req_hdr, const int32_t* req_id, const uint8_t* req_act, const float* req_emb,
                   long long n_max, int row_words, long long lo, long long hi, double t_stale, int refresh_retained,
                   long long cap_fixed, long long n_owned, long long limit, float* table, int32_t* row_of,
                   int32_t* row_owner, int32_t* admit_iter, long long* layer_ctr, void* scratch,
                   long long scratch_bytes, cudaStream_t stream);
int hg_peer_signal(unsigned long long* my_flag, unsigned long long* state, cudaStream_t stream);
int hg_peer_wait(unsigned long long* const* flags, int P, unsigned long long* state, cudaStream_t stream);

/* ---- full-graph CSR2 on the device: histgnn/graphs.py:161-172 (build_csr2):
 * rows by destination, input edge order inside a row; counts + scan + atomic
 * placement + per-row sort of the edge indices (csrc/hg_graph.cu), no library
 * sort. src / dst int32 device arrays of E edges (N < 2^31, E < 2^32). */
long long hg_build_csr2_scratch_bytes(long long E, long long N);
int hg_build_csr2(const int32_t* src, const int32_t* dst, long long E, long long N, int64_t* start, int64_t* end,
                  int32_t* col, void* scratch, long long scratch_bytes, cudaStream_t stream);

/* ---- dataset ingest, host side (csrc/hg_ingest.cu):
 * multi-threaded parsers of the reference's text formats over a read-only
 * mapping of the file. Call once with out / src / dst = NULL to count, then
 * with arrays of *count entries. On bad input *err = kind (1 not an integer,
 * 2 negative, 3 out of range, 4 wrong field count) and *err_line = the first
 * offending line (1-based); the caller words the message like the reference.
 * hg_parse_int_lines: histgnn/data.py:109-129 (_read_int_lines); upper < 0 =
 *   unbounded; *err_val = the offending value.
 * hg_parse_edge_list: histgnn/graphs.py:186-218 (read_edge_list): "src dst"
 *   lines, '#' comments; ids parsed into int32 (device id width). */
int hg_parse_int_lines(const char* path, long long upper, int64_t* out, long long* count, int* err,
                       long long* err_line, long long* err_val, int nthreads);
int hg_parse_edge_list(const char* path, int32_t* src, int32_t* dst, long long* count, long long* max_src,
                       long long* max_dst, int* err, long long* err_line, int nthreads);

/* ---- static feature region: histgnn/cache.py:338-351 (backfill_features) */
long long hg_degree_order_scratch_bytes(long long n);
int hg_feature_region(const int64_t* g_start, const int64_t* g_end, long long n, long long k, int32_t* chosen,
                      int32_t* feature_row_of, void* scratch, long long scratch_bytes, cudaStream_t stream);

/* ---- native synthetic data: histgnn/data.py:243-270 (synth_power_law),
 * bit-identical to the reference for the same numpy Generator. pcg[6] in/out
 * is the Generator's PCG64 state (state hi/lo, inc hi/lo, has_uint32,
 * uinteger); it is advanced exactly as `rng.integers(len(pool))` would, so
 * numpy continues the stream for features, labels and the split. Host
 * function; writes 2*m*(n-m) edges into host int32 arrays; returns the edge
 * count or -1 for invalid (n, m). */
long long hg_synth_power_law(long long n, int m, unsigned long long* pcg, int32_t* src_out, int32_t* dst_out);

#ifdef __cplusplus
}
#endif

#endif /* HGB200_H_ */
