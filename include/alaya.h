/*
 * alaya.h -- C-ABI of the B200-native DIPR retrieval + sparse-attention path.
 *
 * This is the drop-in boundary under the reference's Python surface
 * (package ``sparsekv``, /root/reference/pkg/src/sparsekv). The reference has
 * no native code; each entry point below replaces one numeric stage of its
 * decode step, cited file:line:
 *
 *   alaya_dipr_attention   Session.attention on the DIPR/FLAT plan
 *                          (store.py:191-216 -> _head_attention :252-293,
 *                          _retrieve flat branch :336-337).
 *   alaya_dipr_attention_update  Session.update (store.py:160-189) + the above.
 *   alaya_scan             inner_products + scores.max()  (core.py:64-67,
 *                          dipr.py:63-64), batched over GQA groups.
 *   alaya_attend           mask s >= max - beta (dipr.py:64), setdiff with the
 *                          window ids (store.py:271-273, core.py:159-165),
 *                          PartialAttention.over(selected) and .over(window)
 *                          merged (attention.py:98-143) -> one (m,l,acc) state.
 *   alaya_merge_partials   PartialAttention.merge + finalize
 *                          (attention.py:128-152) across sequence shards.
 *   alaya_selected         dipr_bruteforce's id set (dipr.py:65-70) and the
 *                          Session.last_diagnostics lists (store.py:288-292).
 *   alaya_block_bounds_*   sound coarse block filter feeding the scan
 *                          (input: BlockIndex, index.py:195-243).
 *
 * Conventions: every pointer named d_* is DEVICE memory; descriptor arrays and
 * params are HOST memory read during the call. All work is stream-ordered on
 * ``stream``; no call synchronises the device. Return value 0 = ok, otherwise
 * an alaya_status code; alaya_last_error() gives a message (thread-local).
 * Entry points are reentrant; state lives only in the caller's workspace.
 */
#ifndef ALAYA_H_
#define ALAYA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ALAYA_OK = 0,
  ALAYA_ERR_ARG = 1,        /* maps to ValueError (store.py:175-178,200-204) */
  ALAYA_ERR_SHAPE = 2,      /* maps to ValueError */
  ALAYA_ERR_NONFINITE = 3,  /* maps to FloatingPointError (attention.py:150-151) */
  ALAYA_ERR_CUDA = 4,
  ALAYA_ERR_WORKSPACE = 5,
  ALAYA_ERR_UNSUPPORTED = 6
} alaya_status;

typedef enum { ALAYA_F32 = 0, ALAYA_BF16 = 1 } alaya_dtype;

typedef enum {
  ALAYA_SCAN_AUTO = 0,
  ALAYA_SCAN_CUDA_CORE = 1, /* warp-shuffle q.k on FP32 pipes */
  ALAYA_SCAN_TCGEN05 = 2    /* bf16 q.K^T on 5th-gen tensor cores (TMEM accum) */
} alaya_scan_kind;

/* One sequence (session) for one layer.
 * Base prefix keys of kv head h, token t (local row) live at
 *   k + (h * head_stride + t * dim) elements; same for v.
 * Session-window rows (Session.update, store.py:160-189) at
 *   wk + (h * w_head_stride + r * dim).
 * Sequence-sharded mode: this shard holds global rows
 *   [token_offset, token_offset + n) of a base prefix of prefix_len tokens;
 *   unsharded callers pass token_offset = 0, prefix_len = n. */
typedef struct {
  const void* k;
  const void* v;
  const void* wk;
  const void* wv;
  int64_t head_stride;
  int64_t w_head_stride;
  int64_t token_offset;
  int64_t prefix_len;
  int32_t n;
  int32_t w;
  /* Coarse block filter input (alaya_block_bounds output for this layer slab):
   * [Hkv][bounds_head_stride elements], per 128-token block [5][dim] in the K
   * dtype: min, max, mean, representative key, radius. NULL when
   * params.block_filter == 0. */
  const void* bounds;
  int64_t bounds_head_stride;
  /* Optional DEVICE window row count (CUDA-graph mode). When non-NULL the kernels
   * read the session-window row count from *d_w when they run, `w` is the ring
   * CAPACITY in rows, and alaya_window_append writes row *d_w and increments it
   * (rows beyond the capacity are dropped). A decode step captured once as a
   * CUDA graph then stays valid while the window grows. NULL: `w` is the count. */
  int32_t* d_w;
} alaya_seq;

typedef struct {
  int32_t n_query_heads;
  int32_t n_kv_heads;
  int32_t dim;           /* 16, 32, 64, 128 or 256 */
  int32_t dtype;         /* alaya_dtype of K/V (base and window) */
  float beta;            /* raw inner-product slack (dipr.py:47-70) */
  int32_t win_initial;   /* WindowConfig.initial (core.py:152) */
  int32_t win_last;      /* WindowConfig.last (core.py:153) */
  int32_t chunk;         /* tokens per work chunk; 0 = auto */
  int32_t scan_kind;     /* alaya_scan_kind */
  int32_t block_filter;  /* 1 = skip 128-token blocks whose sound upper bound
                          * sum_d max(q_d lo_d, q_d hi_d) is below LB - beta, LB
                          * = max score of the base-window tokens (a lower bound
                          * of the DIPR max). Exact: the DIPR set is unchanged. */
  /* Optional DEVICE call sequence number (CUDA-graph mode): a u64 the captured step
   * increments once per replay before its first layer. Inside a stream capture it
   * gives every captured call a per-replay identity, so the scan can start on prep's
   * published header (the eager fast path) in graphs too. NULL: calls captured in a
   * graph wait for prep's completion instead. */
  const unsigned long long* d_call_seq;
} alaya_params;

/* Coarse block index of one sequence's context (alaya_block_reps output):
 * reps + h*head_stride + (blk*r + i)*dim = representative i of block blk of
 * kv head h; the index was built over n_tokens tokens (the full imported
 * context; a reused prefix may be shorter, index.py:206-214 then clips). */
typedef struct {
  const void* reps;
  int64_t head_stride;
  int64_t n_tokens;
  int32_t n_blocks;
  int32_t r;
} alaya_block_index;

#ifndef ALAYA_MAX_BATCH
#define ALAYA_MAX_BATCH 32
#endif
#define ALAYA_PARTIAL_STRIDE(dim) ((dim) + 2) /* (m, l, acc[dim]) per query head */

const char* alaya_last_error(void);
int alaya_version(void);
/* Diagnostics only (not a reference interface): while d_buf is non-null, the
 * prep/scan/attend/combine kernels of every later call stamp %globaltimer per
 * CTA into d_buf as u64 [4 kinds][1024 CTAs][16 slots] (needs 512 KB). */
int alaya_debug_trace(void* d_buf, int64_t bytes);

/* Workspace bytes needed for a call on this batch. */
size_t alaya_workspace_bytes(const alaya_params* p, const alaya_seq* seqs, int batch);

/* Full single-GPU decode step for one layer over `batch` sequences.
 * d_q: [batch][Hq][dim] fp32.  d_out: [batch][Hq][dim] fp32. */
int alaya_dipr_attention(const alaya_params* p, const alaya_seq* seqs, int batch,
                         const float* d_q, float* d_out, void* d_ws, size_t ws_bytes,
                         void* stream);

/* Session.update followed by Session.attention for one layer of a batch
 * (store.py:160-189 then 191-216) in one call: the new K/V row of every
 * sequence (d_k_new/d_v_new [batch][Hkv][dim] fp32, rounded to the KV dtype)
 * is written as window row seqs[b].w - 1 -- seqs[b].w counts the windows rows
 * INCLUDING the new one -- by the call's first kernel, then the same step as
 * alaya_dipr_attention. Saves the separate alaya_window_append launch.
 * Not for device window counts (d_w). */
int alaya_dipr_attention_update(const alaya_params* p, const alaya_seq* seqs, int batch,
                                const float* d_k_new, const float* d_v_new, const float* d_q,
                                float* d_out, void* d_ws, size_t ws_bytes, void* stream);

/* Stage 1: score every base key of every query head, per-head max and the
 * candidate superset. Writes the local max per (seq, q head) to d_smax
 * ([batch][Hq] fp32, -inf where n == 0); d_smax may be NULL (scan only). */
int alaya_scan(const alaya_params* p, const alaya_seq* seqs, int batch, const float* d_q,
               float* d_smax, void* d_ws, size_t ws_bytes, void* stream);

/* Stage 2: exact filter at d_smax - beta (the GLOBAL max after an allreduce in
 * sharded mode), V gather + online softmax over the selection, merged with
 * the window rows this shard owns. Writes one partial state per query head:
 * d_part[(b*Hq+qh)*(dim+2) + {0:m, 1:l, 2..:acc}] (m = -inf, l = 0 if empty).
 * want_values = 0 skips the V gather (DIPR-only). */
int alaya_attend(const alaya_params* p, const alaya_seq* seqs, int batch, const float* d_q,
                 const float* d_smax, float* d_part, int want_values, void* d_ws,
                 size_t ws_bytes, void* stream);

/* Stages 1+2 fused for the sharded step (replaces scan -> allreduce(MAX) ->
 * attend of sharded.py; reference dipr.py:64 global max over all shards):
 * the CTA completing a (seq, kv head) group's scan stores the group's local
 * maxima straight into every rank's exchange buffer (bufs: the n_ranks
 * symmetric buffers of alaya_exch_alloc/open, NVLink P2P) and raises a
 * per-group flag to `epoch`; the attend kernel, running beside the scan, waits
 * for the n_ranks flags of each group it filters, takes the max over the
 * ranks' slots and filters at that global max - beta. Writes d_part as
 * alaya_attend does (d_part may be NULL when gather_epoch != 0); gather_epoch
 * != 0 also pushes the partials to every rank (see alaya_merge_exchanged), so
 * the layer needs no separate collective. Every rank calls it with the same epoch (the kind-0
 * epoch counter of alaya_exch: slots of parity epoch&1, kind 0). A rank that
 * never arrives sets *d_err = 1 after a bounded poll. ALAYA_ERR_UNSUPPORTED
 * when the call is not tcgen05-eligible (use the staged path). */
int alaya_sharded_step(const alaya_params* p, const alaya_seq* seqs, int batch, const float* d_q,
                       void* const* bufs, int n_ranks, int rank, int64_t cap_floats,
                       unsigned long long epoch, unsigned long long gather_epoch, float* d_part,
                       int* d_err, void* d_ws, size_t ws_bytes, void* stream);

/* Merge of the fused sharded step (replaces allgather -> merge of sharded.py;
 * reference attention.py:128-152): with gather_epoch != 0, alaya_sharded_step's
 * combine stores each row's partial straight into slot[rank] (kind 1) of every
 * rank's buffer and the last row raises this rank's kind-1 flag everywhere; this
 * kernel waits for the n_ranks flags of d_own_buf at `epoch` (= that
 * gather_epoch, the kind-1 epoch counter of alaya_exch), merges the ranks'
 * partials in rank order and finalizes to d_out [rows][dim]. Bounded poll:
 * *d_err = 1 if a rank never arrives. */
int alaya_merge_exchanged(void* d_own_buf, int n_ranks, int64_t cap_floats, unsigned long long epoch,
                          int rows, int dim, float* d_out, int* d_status, int* d_err, void* stream);

/* Stage 3: merge n_parts partial sets (d_parts: [n_parts][batch*Hq][dim+2]) in
 * order and finalize to d_out [batch*Hq][dim] fp32. Non-finite output sets
 * *d_status (device int) to ALAYA_ERR_NONFINITE. */
int alaya_merge_partials(const float* d_parts, int n_parts, int rows, int dim, float* d_out,
                         int* d_status, void* stream);

/* PartialAttention.merge without finalize (attention.py:128-143): merge
 * n_parts state sets in order into d_state [rows][dim+2]. */
int alaya_merge_states(const float* d_parts, int n_parts, int rows, int dim, float* d_state,
                       void* stream);

/* After alaya_attend on the same workspace: per (seq, q head) selected ids
 * (global; deterministic order, ascending within each scan sub-list -- sort
 * for the reference's sorted lists) into d_ids[(b*Hq+qh)*cap ...], counts into
 * d_selected[b*Hq+qh] and the retrieved count (including window ids) into
 * d_retrieved[b*Hq+qh]. cap must be >= max prefix rows per shard. */
int alaya_selected(const alaya_params* p, const alaya_seq* seqs, int batch, int64_t* d_ids,
                   int64_t cap, int32_t* d_selected, int32_t* d_retrieved, void* d_ws,
                   size_t ws_bytes, void* stream);

/* Session.update (store.py:160-189) for a batch: append one row per kv head to
 * every sequence's session window. Row seqs[b].w of wk/wv (head stride
 * w_head_stride) receives d_k/d_v[b][h][0..dim) (fp32, converted to p->dtype).
 * The caller owns window capacity; seqs[b].w is the row index written. */
int alaya_window_append(const alaya_params* p, const alaya_seq* seqs, int batch, const float* d_k,
                        const float* d_v, void* stream);

/* Coarse block index build (input of the block filter; the reference's
 * BlockIndex, index.py:195-243, ranks blocks by representatives -- a heuristic
 * -- while a filter that must keep the exact DIPR set needs a sound bound):
 * per kv head h and 128-token block i of d_k ([heads][head_stride] elements,
 * n rows), d_bounds[h*bounds_head_stride + i*5*dim + r*dim + e] with rows
 * r = 0 min, 1 max, 2 mean, 3 largest-norm key (the reference's
 * representative, index.py:217-228), 4 [e=0] radius max||k - mean|| (rounded up).
 * bounds_head_stride >= ceil(n/128)*5*dim. */
int alaya_block_bounds(const void* d_k, int dtype, int n_heads, int64_t head_stride, int n, int dim,
                       void* d_bounds, int64_t bounds_head_stride, void* stream);

/* TOP_K retrieval on the flat index (FlatIndex.top_k, index.py:60-66, as
 * Session._retrieve uses it, store.py:314-318): per (seq, q head) the k base
 * tokens of largest q.k (ties: smaller token id), as global ids in no
 * particular order, into d_ids[(b*Hq+qh)*cap ...] (their fp32 scores into
 * d_scores, nullable) with the count in d_count[b*Hq+qh] (= min(k, n)). Same workspace as alaya_dipr_attention
 * (beta and block_filter of *p are ignored). Unsharded sequences only. */
int alaya_topk(const alaya_params* p, const alaya_seq* seqs, int batch, const float* d_q, int k,
               int64_t* d_ids, float* d_scores, int64_t cap, int32_t* d_count, void* d_ws,
               size_t ws_bytes, void* stream);

/* BlockIndex build (build_block_index / select_representatives,
 * index.py:217-243): for kv head h and block blk = [blk*block_size, ...) of
 * d_k, the r keys of largest L2 norm (ties: smaller position) into
 * d_reps[h*reps_head_stride + (blk*r + i)*dim] (K dtype); a block with fewer
 * than r keys repeats its first representative. */
int alaya_block_reps(const void* d_k, int dtype, int n_heads, int64_t head_stride, int n, int dim,
                     int block_size, int r, void* d_reps, int64_t reps_head_stride, void* stream);

/* TOP_K over the coarse block index (Session._retrieve, store.py:305-312 with
 * BlockIndex.top_blocks, index.py:206-214): per (seq, q head) the k_blocks
 * blocks of largest max-representative score (ties: smaller start), their
 * token ranges clipped to the sequence's prefix, as global ids into
 * d_ids/d_count like alaya_topk; the chosen block numbers and scores (no
 * order) into d_blocks/d_block_scores [(b*Hq+qh)*k_blocks ...] (nullable).
 * bix: host array [batch]. */
int alaya_block_topk(const alaya_params* p, const alaya_seq* seqs, const alaya_block_index* bix,
                     int batch, int block_size, int k_blocks, const float* d_q, int64_t* d_ids,
                     int64_t cap, int32_t* d_count, int32_t* d_blocks, float* d_block_scores,
                     void* stream);

/* Sparse attention over explicit base ids (Session._head_attention after
 * retrieval, store.py:268-293): ids in the base window (core.py:159-165) are
 * dropped, PartialAttention.over(rest) is merged with the window partial
 * (base window ids + session rows) and finalized into d_out [batch*Hq][dim].
 * d_selected (nullable) receives the kept id count; a non-finite output sets
 * *d_status (nullable device int) to ALAYA_ERR_NONFINITE. */
int alaya_sparse_attention(const alaya_params* p, const alaya_seq* seqs, int batch,
                           const float* d_q, const int64_t* d_ids, int64_t cap,
                           const int32_t* d_count, float* d_out, int32_t* d_selected,
                           int32_t* d_status, void* stream);

/* ---- graph DIPRS (dipr.py:107-289) --------------------------------------- */

/* Proximity graph over one sequence's base prefix, per kv head h (CSR):
 * neighbours of node u = nbrs[h*nbrs_head_stride + offsets[h*offsets_head_stride + u] ...
 * offsets[... + u + 1]); entry[h] = entry point. n_nodes must equal the
 * sequence's n (the reference walks a graph only when p == index.n). */
typedef struct {
  const int64_t* offsets;
  const int32_t* nbrs;
  const int32_t* entry;
  int64_t offsets_head_stride;
  int64_t nbrs_head_stride;
  int32_t n_nodes;
  int32_t pad_;
} alaya_graph;

size_t alaya_diprs_workspace_bytes(const alaya_params* p, const alaya_seq* seqs,
                                   const alaya_graph* graphs, int batch);

/* diprs(index, q, entry, l0, beta, window_max) per (seq, q head): the
 * candidate-list walk of traverse() with the reference's acceptance rule, and
 * the final cut s >= max(best, floor) - beta. floor_mode 0: none; 1: the
 * window-cache maximum (Session._window_score_max, store.py:339-354: base
 * window ids + session rows); 2: d_floors[b*Hq+qh]. Ids (global, no order)
 * into d_ids[(b*Hq+qh)*cap ...], counts into d_count (-1: an adjacency list
 * exceeded the scratch), explored-node counts into d_explored (nullable).
 * graphs: host array [batch]. */
int alaya_diprs(const alaya_params* p, const alaya_seq* seqs, const alaya_graph* graphs, int batch,
                const float* d_q, int l0, int floor_mode, const float* d_floors, int64_t* d_ids,
                int64_t cap, int32_t* d_count, int32_t* d_explored, void* d_ws, size_t ws_bytes,
                void* stream);

/* ---- sequence-sharded exchange over peer memory -------------- */

/* Bytes of one rank's symmetric exchange buffer for n_ranks ranks and
 * messages of up to cap_floats floats (0 if out of range, n_ranks <= 16). */
size_t alaya_exch_bytes(int n_ranks, int64_t cap_floats);
/* cudaMalloc a zeroed exchange buffer and export its CUDA IPC handle
 * (ipc_handle: 64 bytes, cudaIpcMemHandle_t). */
int alaya_exch_alloc(size_t bytes, void** d_buf, void* ipc_handle);
/* Map a peer rank's exchange buffer (cudaIpcOpenMemHandle, lazy peer access). */
int alaya_exch_open(const void* ipc_handle, void** d_buf);
int alaya_exch_close(void* d_buf);
int alaya_exch_free(void* d_buf);
/* One exchange on `stream`: bufs[r] = rank r's buffer as mapped in this process.
 * kind 0: allreduce-max of d_local[count] into d_out (the global DIPR max,
 * replaces ncclAllReduce(max)); kind 1: allgather of d_local[count], read the
 * result in place at alaya_exch_slots(own buffer, ..., 1, epoch) as
 * [n_ranks][cap_floats] (replaces ncclAllGather). epoch: 1, 2, ... per kind,
 * the same sequence on every rank. A peer that never arrives sets *d_err. */
int alaya_exch(void* const* bufs, int n_ranks, int rank, int64_t cap_floats, int kind,
               const float* d_local, int64_t count, unsigned long long epoch, float* d_out, int* d_err,
               void* stream);
float* alaya_exch_slots(void* d_buf, int n_ranks, int64_t cap_floats, int kind, unsigned long long epoch);

/* ---- AVDB vector files (reference vfs.py, docs/file-format.md) ---------- */

typedef struct {
  uint32_t dim;
  uint32_t element_width;   /* 16 (IEEE half) or 32 */
  uint64_t n_vectors;
  uint32_t n_data_blocks;
  uint32_t n_index_blocks;  /* graph adjacency blocks (not loaded here) */
  uint32_t n_tombstones;    /* ids marked deleted (vectors still loaded, vfs.py:310-314) */
  uint32_t pad_;
  uint64_t file_bytes;
  uint64_t directory_offset;
  uint64_t index_head;
} alaya_avdb_info;

/* Header + directory chain of one file (read_header / read_directory,
 * vfs.py:247-286). Format errors -> ALAYA_ERR_ARG naming path and offset. */
int alaya_avdb_stat(const char* path, alaya_avdb_info* out);

/* write_vector_file (vfs.py:188-244) for a vector-only file: host fp32
 * vectors [n][dim], element_width 32 or 16 (half, round-to-nearest-even).
 * Byte-identical to the reference writer. Host only. */
int alaya_avdb_write(const char* path, const float* vectors, int64_t n, int dim, int element_width);

/* Graph index chain of a K file (vfs.py:126-145, 324-330): sizes, entry point
 * and max degree; fills degrees [n_nodes] / nbrs [n_edges] (host, nullable:
 * call once for the sizes). n_nodes = 0 when the file has no index. */
int alaya_avdb_graph(const char* path, int64_t* n_nodes, int64_t* n_edges, int32_t* entry_point,
                     int32_t* max_degree, int32_t* degrees, int32_t* nbrs);

/* Pinned staging bytes alaya_avdb_load needs for these files (0 on error). */
size_t alaya_avdb_staging_bytes(const char* const* paths, int n_files);

/* read_vector_file (vfs.py:289-338) of n_files files of n vectors x dim into
 * the device slab d_dst[f*dst_file_stride + row*dim + e] (dst_dtype F32:
 * exact widening, BF16: round to nearest even). Each file image is read into
 * h_staging (PINNED host memory, >= alaya_avdb_staging_bytes) and one
 * stream-ordered kernel unpacks the data blocks straight from it. h_staging
 * must stay untouched until the stream passes this call. */
int alaya_avdb_load(const char* const* paths, int n_files, int64_t n, int dim, int dst_dtype,
                    void* d_dst, int64_t dst_file_stride, void* h_staging, size_t staging_bytes,
                    void* stream);

/* Blocks kept / blocks considered by the block filter in the last scan on
 * this workspace: device pointer to two int32 (valid after the scan). */
int* alaya_ws_block_stats(const alaya_params* p, const alaya_seq* seqs, int batch, void* d_ws);

/* Diagnostics: candidate-superset sizes of the last scan on this workspace,
 * device pointer to int32 [total_chunks][G][4 scan sub-lists]. */
int* alaya_ws_candidate_counts(const alaya_params* p, const alaya_seq* seqs, int batch, void* d_ws);

/* Device status word of the last alaya_dipr_attention on this workspace
 * (ALAYA_OK or ALAYA_ERR_NONFINITE); pointer into d_ws. */
int* alaya_ws_status(void* d_ws);

#ifdef __cplusplus
}
#endif
#endif /* ALAYA_H_ */
