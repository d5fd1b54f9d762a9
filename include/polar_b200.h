/*
 * polar_b200.h -- C ABI of libpolar_b200.so, the B200 (sm_100a) kernels of
 * Polar Sparsity's batched-decode hot path.
 *
 * Conventions (every entry point):
 *   - stream-ordered: work is enqueued on `stream` (a cudaStream_t passed as
 *     void*; NULL = legacy default stream); nothing synchronises the host;
 *   - the library never allocates: outputs and workspaces are caller-owned
 *     device buffers whose sizes come from the *_workspace_bytes queries,
 *     which keeps every call CUDA-graph capturable;
 *   - data: bf16 activations/weights/KV (uint16 bit patterns), f32 logits
 *     and accumulators, int32 indices and lengths;
 *   - return value: PS_OK or a PS_ERR_* status (ps_status_string() names
 *     it).  Host-visible argument errors are detected before any launch.
 *
 * The reference (`sparsedecode`, /root/reference/pkg) has no FFI: its
 * operator API is the set of Python functions re-exported by
 * sparsedecode/__init__.py:18-75 and bound by name in engine.py:25-35.  Each
 * entry point below names the reference function it replaces; the Python
 * package paper_2505_14884_b200 mirrors those names on top of this ABI.
 */
#ifndef POLAR_B200_H
#define POLAR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map 1:1 onto the reference's exception types) ---- */
#define PS_OK               0
#define PS_ERR_VALUE        1  /* ValueError  (shapes, k range, scale <= 0) */
#define PS_ERR_INDEX        2  /* IndexError  (ids out of range)            */
#define PS_ERR_EMPTY_CACHE  3  /* EmptyCacheError (exceptions.py:4-5)       */
#define PS_ERR_CAPACITY     4  /* CapacityError   (exceptions.py:8-9)       */
#define PS_ERR_UNSUPPORTED  5  /* ValueError: shape not built for sm_100a   */
#define PS_ERR_WORKSPACE    6  /* ValueError: workspace too small           */
#define PS_ERR_CUDA         7  /* RuntimeError: CUDA launch/config failure  */

#define PS_DTYPE_F32  0
#define PS_DTYPE_BF16 1

#define PS_ACT_NONE 0
#define PS_ACT_RELU 1

int ps_version(void);
/* programmatic dependent launch of every kernel (default on); 0 disables */
void ps_set_pdl(int enable);
const char* ps_status_string(int status);
/* number of SMs of the current device (grid sizing helper) */
int ps_num_sms(void);

/* ======================================================================
 * Select-Head Attention (SHA) decode
 * Replaces sparsedecode.kernels.gqa_selective_attention_decode
 * (kernels.py:513-548 -> _attention_over_units 386-444) and, for G == 1,
 * selective_head_flash_attention_decode (kernels.py:464-510).
 *
 *   q       bf16 (B, H, d_h), row b at q + b*q_ld elements (q_ld >= H*d_h)
 *   k_cache bf16 (B, H_kv, cap, d_h) contiguous; v_cache likewise
 *   lengths int32 (B,): rows [0, lengths[b]) are valid; others never read
 *   sel     int32 (B, top_k): selected KV-group ids per sequence (distinct,
 *           in [0, H_kv); query heads g*G .. g*G+G-1, G = H/H_kv, attend)
 *   out     (B, H, d_h) f32 or bf16, row b at out + b*out_ld elements;
 *           heads of non-selected groups are written as exact 0.0
 *   group_base  tensor parallelism: this rank's cache/q/out hold global groups
 *           [group_base, group_base + H_kv); selected ids outside that range
 *           are skipped (0 without TP)
 *   num_splits  KV splits per (b, group) unit (FlashDecoding); 0 = auto
 *   max_len_hint  expected max_b lengths[b] (0 = cap); it only sizes the grid.
 *           The kernel reads the tile count from the device lengths, so
 *           the call (and a CUDA graph that captured it) stays exact for
 *           any lengths[b] <= cap
 *   ws      >= ps_sha_workspace_bytes(...) bytes; must be zero-filled
 *           before its first use (the kernel leaves it zeroed again)
 * ==================================================================== */
/* debug: 0 forces the CUDA-core SHA path (d_h = 128 otherwise runs on mma.sync) */
void ps_debug_sha_mma(int enable);
/* debug: per-CTA globaltimer stamps of ps_sha_decode's tensor-core kernel
 * (8 u64 per CTA: start, after the dependency wait, partition known, end); NULL = off */
void ps_debug_sha_trace(void* buf);
size_t ps_sha_workspace_bytes(int B, int H, int H_kv, int d_h, int top_k, int num_splits);
int ps_sha_auto_splits(int B, int H_kv, int d_h, int top_k, int max_len);
int ps_sha_decode(const void* q, int64_t q_ld,
                  const void* k_cache, const void* v_cache,
                  const int32_t* lengths, const int32_t* sel, int group_base,
                  int B, int H, int H_kv, int cap, int d_h, int top_k,
                  float scale, int num_splits, int max_len_hint,
                  void* out, int64_t out_ld, int out_dtype,
                  void* ws, size_t ws_bytes, void* stream);

/* ======================================================================
 * KV cache append for one decode step.
 * Replaces sparsedecode.tensors.KVCache.append_step (tensors.py:150-170):
 * writes k_new/v_new (B, H_kv, d_h) bf16 (row b at +b*src_ld elements) at
 * position lengths[b] and increments lengths[b].  A sequence already at
 * capacity is left untouched and err_flag (int32, may be NULL) is set to 1.
 * ==================================================================== */
int ps_kv_append(void* k_cache, void* v_cache, int32_t* lengths,
                 const void* k_new, const void* v_new, int64_t src_ld,
                 int B, int H_kv, int cap, int d_h, int32_t* err_flag, void* stream);

/* Paged KV cache (the reference cache is contiguous,
 * tensors.py:116-213).  K and V live in pools of `pool_pages` pages of
 * layout (page, H_kv, page_rows, d_h) bf16; logical row r of sequence b is
 * row r % page_rows of page block_table[b * table_ld + r / page_rows], so
 * the logical capacity is table_ld * page_rows.  page_rows must be a
 * multiple of the SHA tile (4096 / d_h rows; 32 at d_h = 128).  Every one
 * of a row's table_ld entries must be readable (entries past a sequence's
 * length are prefetched as hints and never dereferenced).
 * ps_sha_decode_paged: ps_sha_decode over the paged pools (same math, same
 *   workspace query, same error behaviour).
 * ps_kv_append_paged: ps_kv_append into the page holding lengths[b]
 *   (the caller maps that page before the step).  Unmapped pages hold -1 in
 *   block_table: an append whose row falls in one writes nothing, leaves
 *   lengths[b] as it was and sets err_flag to 2 (1 = capacity). */
int ps_sha_decode_paged(const void* q, int64_t q_ld, const void* k_pool, const void* v_pool,
                        int pool_pages, int page_rows, const int32_t* block_table, int64_t table_ld,
                        const int32_t* lengths, const int32_t* sel, int group_base,
                        int B, int H, int H_kv, int d_h, int top_k,
                        float scale, int num_splits, int max_len_hint,
                        void* out, int64_t out_ld, int out_dtype,
                        void* ws, size_t ws_bytes, void* stream);
int ps_kv_append_paged(void* k_pool, void* v_pool, int page_rows, const int32_t* block_table,
                       int64_t table_ld, int32_t* lengths, const void* k_new, const void* v_new,
                       int64_t src_ld, int B, int H_kv, int d_h, int32_t* err_flag, void* stream);

/* ======================================================================
 * Selection (bit-exact with the reference ordering: value descending,
 * ties -> lower index, -0.0 == +0.0, NaN below -inf).
 * ps_topk_rows replaces tensors.topk_indices_rows (tensors.py:65-73) and
 * BatchHeadIndex.from_logits (kernels.py:107-112); ids are written
 * ascending.  `bitmap` (may be NULL) additionally receives an atomic OR of
 * every selected id (bit i of word i/32) -- the union's first half.
 * ps_threshold_rows is the router's predict() (routers.py:188-190, logit >
 * thr) ORed into the bitmap.
 * ps_union_rows ORs an id matrix into the bitmap; ps_bitmap_compact
 * replaces union_neuron_indices (kernels.py:376-383): ascending ids of the
 * set bits in [lo, hi) minus lo (lo % 32 == 0; lo=0, hi=width for the whole
 * union, a neuron shard's range under tensor parallelism) and the
 * device-resident count, padding idx_out up to a multiple of `pad` with the
 * last id, and clearing the bitmap for the next call.  Bitmaps must be
 * zero-filled before first use; words = ceil(width/32).
 * ==================================================================== */
int ps_topk_rows(const float* logits, int rows, int cols, int64_t ld, int k,
                 int32_t* idx_out, uint32_t* bitmap, void* stream);
int ps_threshold_rows(const float* logits, int rows, int cols, int64_t ld, float thr,
                      uint32_t* bitmap, void* stream);
/* Fused per-row selection + union + compaction (one launch per layer): top-k
 * (k > 0) or threshold (k <= 0: logit > thr) per row; each row's selection
 * words are stored into the workspace, the last CTA of every 16-row group
 * ORs the group, and the last group compacts bits [lo, hi) into union_out /
 * count_out exactly as ps_bitmap_compact does.  No contended atomics.
 * bias: f32 (cols) added to every row before selection (the router's output
 * bias, routers.py:286-288), or NULL.  rows <= 1024.
 * ws >= ps_select_union_workspace_bytes(rows, cols), zero-filled before its
 * first use (its tickets self-reset; the bitmaps are fully rewritten). */
size_t ps_select_union_workspace_bytes(int rows, int cols);
int ps_select_union(const float* logits, const float* bias, int rows, int cols, int64_t ld, int k, float thr,
                    void* ws, size_t ws_bytes, int lo, int hi, int pad,
                    int32_t* union_out, int32_t* count_out, void* stream);
/* ps_select_union_bitmap -- union hand-off: the per-row top-k (k >= 1) or
 * threshold (k <= 0: logit > thr) sets are OR-ed into `bitmap` (ceil(cols/32)
 * uint32 words, zero on entry) and the launch ends there: no ticket, no
 * compaction.  The gathered GEMMs read the bitmap (PS_GG_BITMAP).  CTA 0
 * zeroes `clear` (the buffer of the previous layer; may be NULL), so two
 * buffers alternate layer by layer.  cols <= 36864. */
int ps_select_union_bitmap(const float* logits, const float* bias, int rows, int cols, int64_t ld, int k, float thr,
                           uint32_t* bitmap, uint32_t* clear, void* stream);
/* debug: per-CTA phase timestamps of the top-k kernel (16 x u64 per CTA), NULL = off */
void ps_debug_topk_trace(void* buf);
/* ps_select_union kernel: 1 = the low-latency row kernel (topk_union.cu,
 * default for cols <= 36864), 0 = the bracket/candidate kernel (select.cu). */
void ps_debug_topk_v2(int enable);
int ps_union_rows(const int32_t* rows_idx, int rows, int k, int width,
                  uint32_t* bitmap, void* stream);
int ps_bitmap_compact(uint32_t* bitmap, int width, int lo, int hi, int pad,
                      int32_t* idx_out, int32_t* count_out, void* stream);

/* ======================================================================
 * Head router fused with its top-k.
 * Replaces HeadRouter.decision_function (routers.py:324-325, 178-186)
 * followed by BatchHeadIndex.from_logits (kernels.py:107-112), as called
 * in engine.py:352-357.
 *   x      bf16 (B, d), row b at +b*x_ld;  w_t bf16 (H_kv, d) (= W^T);
 *   bias   f32 (H_kv) or NULL;  logits_out f32 (B, H_kv) or NULL;
 *   sel_out int32 (B, k) ascending.
 * ==================================================================== */
int ps_head_router_topk(const void* x, int64_t x_ld, const void* w_t, const float* bias,
                        int B, int d, int H_kv, int k,
                        float* logits_out, int32_t* sel_out, void* stream);
/* Same, fused with the step's KV append (ps_kv_append semantics: k_new /
 * v_new rows of H_cache heads written at lengths[b], then lengths[b]++; a
 * full sequence sets err_flag) -- one launch instead of two per layer. */
int ps_head_router_topk_append(const void* x, int64_t x_ld, const void* w_t, const float* bias,
                               int B, int d, int H_kv, int k, float* logits_out, int32_t* sel_out,
                               void* k_cache, void* v_cache, int32_t* lengths,
                               const void* k_new, const void* v_new, int64_t src_ld,
                               int H_cache, int cap, int d_h, int32_t* err_flag, void* stream);
/* Same, appending into a paged cache (ps_kv_append_paged layout). */
int ps_head_router_topk_append_paged(const void* x, int64_t x_ld, const void* w_t, const float* bias,
                                     int B, int d, int H_kv, int k, float* logits_out, int32_t* sel_out,
                                     void* k_pool, void* v_pool, int page_rows,
                                     const int32_t* block_table, int64_t table_ld, int32_t* lengths,
                                     const void* k_new, const void* v_new, int64_t src_ld,
                                     int H_cache, int d_h, int32_t* err_flag, void* stream);

/* ======================================================================
 * Gathered GEMM on tcgen05 tensor cores (TMEM accumulators).
 *
 * ps_gather_gemm  ("rows" form; replaces selective_gemm, kernels.py:268-291,
 * the up-projection half of sparse_mlp_forward 353-373, and -- with
 * idx == NULL -- the dense router layers routers.py:286-288):
 *   out[n, j] = act( sum_k w_rows[idx[j], k] * x[n, k] + bias[idx[j]] )
 *               (+ residual[n, j] if residual != NULL, added after act)
 *   for j < count (count = *count_dev if count_dev else M), n < N;
 *   columns j in [count, M_pad) of out are written as 0.
 *   w_rows bf16 (w_height, K) row-major (neuron-major);  x bf16 (N, K) row b at
 *   +b*x_ld;  out (N, M_pad) f32/bf16 row n at +n*out_ld.
 *
 * ps_gather_gemm_t ("contraction" form; replaces selective_gemm_t,
 * kernels.py:294-310, and the down-projection of sparse_mlp_forward):
 *   out[n, m] = sum_{j < count} h[n, j] * w_rows[idx[j], m] + bias[m]
 *               (+ residual[n, m] if residual != NULL)
 *   w_rows bf16 (w_height, M) row-major;  h bf16 (N, K_pad) row n at +n*h_ld
 *   with K_pad >= count rounded up to 64 and zero beyond count.
 *
 * idx is int32 (NULL = identity) with ids < w_height.  Operands are moved by
 * the TMA engine (2-D tiles; sm_100 tile::gather4 for gathered rows), so
 * rows must be 16-byte aligned: K % 8 == 0 (rows form), M % 8 == 0
 * (contraction form), x_ld / h_ld % 8 == 0.
 * ws >= ps_gather_gemm_workspace_bytes(...) and zero-filled before first use.
 * ==================================================================== */
/* debug / tuning hook: per-CTA globaltimer trace (8 x u64 per CTA) and
 * overrides of the pipeline depth and split-K CTA target (0 = default) */
void ps_debug_gemm_trace(void* buf, int stages, int target_ctas);
/* A-operand copy engine: 0 = TMA (tile / tile::gather4), 1 = cp.async loader
 * warps for gathered rows (default), 2 = cp.async loader warps always */
void ps_debug_gemm_lsu_mode(int mode);
/* small-batch path of ps_gather_gemm: N <= 4 (and no residual) runs a
 * CUDA-core gathered GEMV -- whole rows per warp, no split-K -- instead of the
 * tcgen05 tiles; 0 forces the tiles (default 1, env PS_GG_GEMV) */
void ps_debug_gemm_gemv(int enable);
/* flags: PS_GG_A_READY -- w_rows, idx and count_dev were written at least
 * two launches earlier in the stream (or are static): the A stream may start
 * before the immediately preceding kernel completes (programmatic dependent
 * launch).  Without it (or with idx == count_dev == NULL, i.e. static dense
 * weights, where it is implied) only static data is read early. */
#define PS_GG_A_READY 1
/* flags: PS_GG_BITMAP -- union hand-off: `idx` is the union BITMAP over the
 * w_height weight rows (ceil(w_height / 32) uint32 words, as written by
 * ps_select_union_bitmap) instead of a compacted id list; the kernel derives
 * the ids on the device (word-prefix popcounts).  UP writes the union size to
 * count_dev (may be NULL); DOWN ignores count_dev.  Tensor-core path only
 * (not the N <= 4 GEMV); w_height <= 32768. */
#define PS_GG_BITMAP 2
size_t ps_gather_gemm_workspace_bytes(int N, int M, int K, int splits);
int ps_gather_gemm_auto_splits(int N, int M, int K);
int ps_gather_gemm(const void* w_rows, int w_height, const int32_t* idx, const int32_t* count_dev,
                   const void* x, int64_t x_ld, const float* bias,
                   const float* residual, int64_t residual_ld,
                   int N, int M, int K, int act, int splits, int flags,
                   void* out, int64_t out_ld, int out_dtype,
                   void* ws, size_t ws_bytes, void* stream);
int ps_gather_gemm_t(const void* w_rows, int w_height, const int32_t* idx, const int32_t* count_dev,
                     const void* h, int64_t h_ld, const float* bias, const float* residual,
                     int64_t residual_ld, int N, int M, int K_max, int splits, int flags,
                     void* out, int64_t out_ld, int out_dtype,
                     void* ws, size_t ws_bytes, void* stream);

/* ps_sparse_mlp -- the whole selective MLP in ONE launch (replaces
 * sparse_mlp_forward, kernels.py:353-373, and the engine's per-layer MLP
 * block, engine.py:371-392):
 *   hidden[n, j] = relu( sum_k w1_rows[idx[j], k] x[n, k] + b1[idx[j]] )  (bf16, j < count;
 *                  columns [count, round_up(count, 128)) written as 0)
 *   out[n, m]   += sum_{j < count} hidden[n, j] w2_rows[idx[j], m] + b2[m]   (f32, ACCUMULATED:
 *                  out holds the residual stream, or zeros, on entry)
 *   count = *count_dev (idx == count_dev == NULL: every neuron, the dense MLP).
 *   w1_rows / w2_rows: bf16 (D, d) neuron-major (W1^T, W2^T); x bf16 (N, d); hidden bf16 (N, h_ld >= round_up(D,128));
 *   N <= 256.  One persistent CTA per SM, stream-K over both projections:
 *   split up-projection tiles are summed with f32 reductions and finished by
 *   their last piece; each down-projection K block waits only on the
 *   up-projection tile it reads (device flags) and adds its partial into out.
 *   No second launch, no grid barrier.  The f32 reductions make the last bits
 *   of out depend on arrival order (results agree to f32 rounding).
 *   ws: zero-initialised once, ps_sparse_mlp_workspace_bytes(N, D, d) bytes,
 *   self-resetting (CUDA-graph safe); one stream at a time per workspace. */
size_t ps_sparse_mlp_workspace_bytes(int N, int D, int d);
int ps_sparse_mlp(const void* w1_rows, const float* b1, const void* w2_rows, const float* b2, int D, int d,
                  const int32_t* idx, const int32_t* count_dev, const void* x, int64_t x_ld, int N,
                  void* hidden, int64_t h_ld, float* out, int64_t out_ld, void* ws, size_t ws_bytes, void* stream);

/* ps_router_mlp -- the two-layer neuron router in ONE launch (replaces
 * MlpRouter.decision_function, routers.py:286-288):
 *   hid = relu(x W_in + b_in) (bf16 (N, hid_ld)), logits = hid W_out + b_out (f32; b_out may be NULL,
 *   e.g. when ps_select_union adds it).  w_in_rows = W_in^T (h, d), w_out_rows = W_out^T (D, h), bf16. */
size_t ps_router_mlp_workspace_bytes(int N, int h, int D);
int ps_router_mlp(const void* w_in_rows, const float* b_in, const void* w_out_rows, const float* b_out,
                  int d, int h, int D, const void* x, int64_t x_ld, int N, void* hid, int64_t hid_ld,
                  float* logits, int64_t logits_ld, void* ws, size_t ws_bytes, void* stream);
void ps_debug_chain_stages(int stages);
void ps_debug_chain_trace(void* buf);

/* ps_router_mlp_fused -- the same router (routers.py:286-288) as one
 * persistent launch with a device grid barrier between its layers: one CTA
 * per 128 logit columns (D <= 128 * #SMs, all co-resident), W_in split over
 * the CTAs (<= 4 K-blocks each), both layers' static weights TMA-prefetched
 * before the dependency wait.  N <= 128, d % 64 == 0, h % 128 == 0; other
 * shapes return PS_ERR_UNSUPPORTED (callers fall back to ps_router_mlp or two
 * GEMMs).  ws: ps_router_mlp_fused_workspace_bytes(N, d, h, D) bytes,
 * zero-initialised once (monotonic barrier counter + f32 partials). */
size_t ps_router_mlp_fused_workspace_bytes(int N, int d, int h, int D);
int ps_router_mlp_fused(const void* w_in_rows, const float* b_in, const void* w_out_rows, const float* b_out,
                        int d, int h, int D, const void* x, int64_t x_ld, int N, void* hid, int64_t hid_ld,
                        float* logits, int64_t logits_ld, void* ws, size_t ws_bytes, void* stream);
void ps_debug_router_trace(void* buf);

/* ======================================================================
 * Tensor-parallel exchange.
 * ps_allreduce_add_bf16: x (f32 (B, d), row stride x_ld) += sum over the
 *   `world` ranks of their bf16 (B, d) partials, in ONE launch over peer
 *   memory -- replaces dist.all_reduce(partial) + x.add_(partial) after the
 *   O- and down-projections (parallel.py).  bufs / flags: device arrays of
 *   the ranks' partial buffers (this call's slot) and inbox addresses
 *   (CUDA IPC mappings); inbox: this rank's 8 uint32 flags; state: 2 uint32
 *   (device epoch, ticket), zero-initialised once.  Callers alternate two
 *   partial buffers from call to call (collective.P2PAllReduce).
 * ==================================================================== */
int ps_allreduce_add_bf16(const unsigned long long* bufs, const unsigned long long* flags, unsigned int* inbox,
                          unsigned int* state, int rank, int world, int B, int d, float* x, int64_t x_ld,
                          void* stream);

/* ======================================================================
 * Decode-step glue.
 * ps_layernorm: model.layernorm (model.py:168-175): x f32 (B, d) row b at
 *   +b*x_ld -> y bf16 (B, d), eps 1e-5, f32 statistics.
 * ps_embed: x[b] = embed[tokens[b]] + pos_embed[lengths[b]] (engine.py:342),
 *   f32 out, bf16 tables.
 * ==================================================================== */
int ps_layernorm(const float* x, int64_t x_ld, const float* gamma, const float* beta,
                 int B, int d, void* y, int64_t y_ld, void* stream);
/* ps_add_layernorm: x += add (f32 (d), may be NULL; written back -- the
 *   bias of the projection whose GEMM just accumulated into x, e.g. b_o of
 *   engine.py:368 or b2 of kernels.py:372), then y = layernorm(x) as above.
 *   d % 4 == 0, 16-byte aligned rows. */
int ps_add_layernorm(float* x, int64_t x_ld, const float* add, const float* gamma, const float* beta,
                     int B, int d, void* y, int64_t y_ld, void* stream);
/* ps_swiglu: the gated activation of swiglu_mlp_forward (kernels.py:335-350):
 *   h[b, j] = silu(gu[b, j]) * gu[b, D + j]   (bf16 in/out, f32 math)     */
int ps_swiglu(const void* gu, int64_t gu_ld, int B, int D, void* h, int64_t h_ld, void* stream);
int ps_embed(const int32_t* tokens, const int32_t* lengths, const void* embed,
             const void* pos_embed, int B, int d, float* x, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* POLAR_B200_H */
