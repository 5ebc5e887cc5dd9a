/*
 * dbk.h -- C-ABI of the B200-native decode hot path of arXiv 2503.05248
 * ("dynamic batching": memory-aware and SLA-constrained batch sizing).
 *
 * One continuous-batching decode iteration = paged KV-cache decode attention
 * over the active batch ("decoding latency ... increases with batch
 * size"; PAPER.md:71 PagedAttention) + the device-side batch telemetry that
 * feeds Algorithm 1 and Algorithm 2,
 * which run on the host in this library.  See DESIGN.md for the readings of
 * the paper (R1..R23) referenced below.
 *
 * Conventions (every entry point):
 *  - returns dbk_status, 0 = DBK_OK; never throws, never aborts;
 *  - on error, dbk_last_error() returns a thread-local message; the call has
 *    no effect unless stated otherwise;
 *  - "device" pointers are CUDA global-memory pointers on the pool's device
 *    (e.g. torch tensor data_ptr()); "host" pointers are CPU memory;
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  A pool, a
 *    scheduler and an engine are NOT thread-safe; use one host thread and one
 *    stream per pool (the library orders its own uploads on that stream);
 *  - the library never allocates KV storage: the caller passes the KV memory
 *    (ownership stays with the caller, who keeps it alive until destroy).  It
 *    allocates only small device metadata (block tables, work lists,
 *    split-K workspace, the stats record) with cudaMalloc;
 *  - there is no CPU fallback: without a usable CUDA device the GPU entry
 *    points fail with DBK_ECUDA.
 */
#ifndef DBK_H_
#define DBK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum dbk_status {
    DBK_OK = 0,
    DBK_EINVAL = 1,       /* bad argument / configuration                          */
    DBK_ECAP = 2,         /* would exceed the page cap; nothing changed (R8)       */
    DBK_ENOENT = 3,       /* unknown request id                                    */
    DBK_EINFEASIBLE = 4,  /* no b >= 1 meets the constraint                        */
    DBK_ECUDA = 5,        /* CUDA runtime error (message has the CUDA error text)  */
    DBK_ENCCL = 6,        /* NCCL error                                            */
    DBK_EFATAL = 7        /* a single request exceeds the cap alone        */
} dbk_status;

const char *dbk_last_error(void);
const char *dbk_version(void);

/* ------------------------------------------------------------------------ */
/* KV pool: paged KV cache + page allocator + request table                  */
/* ------------------------------------------------------------------------ */

/* Shapes of one GPU's share of the model (KV-head TP: pass the local heads and
 * kv_head_offset).
 * Device layout of the caller-provided KV memory:
 *   kv[layer][page][kv_head][2 (K,V)][page_size][head_dim], element kv_dtype.
 * Constraints: q_heads % kv_heads == 0, q_heads/kv_heads in {1,2,4,8},
 * head_dim in {64,128}, page_size == 16, kv_dtype 0 = fp16, 1 = bf16. */
typedef struct dbk_pool_config {
    int32_t layers, q_heads, kv_heads, head_dim, page_size, kv_dtype;
    int64_t cap_pages;          /* M_max in pages (R4)          */
    int32_t max_requests;       /* request slots (rows of the block table)   */
    int32_t max_pages_per_req;  /* block-table row width = ceil(L_max / P)   */
    int32_t device;             /* CUDA device ordinal                       */
    int32_t kv_head_offset;     /* KV-head TP: global index of this pool's
                                 * first kv head, rank * kv_heads for rank r of a TP-G job; its
                                 * q heads are kv_head_offset * (q_heads/kv_heads) + 0.. .  Only
                                 * the synthetic generator sees it (K/V/q values are keyed by the
                                 * GLOBAL head, so the G shards of a job hold disjoint slices of
                                 * the TP1 problem); 0 on one GPU.  >= 0 */
} dbk_pool_config;

typedef struct dbk_pool dbk_pool;

/* Bytes of KV memory the pool needs: layers*cap_pages*kv_heads*2*P*d*2. */
size_t dbk_kv_pool_bytes(const dbk_pool_config *cfg);

/* kv_mem: caller-owned device memory of >= dbk_kv_pool_bytes(cfg) bytes,
 * 256-byte aligned.  Contents need not be initialised (never-written slots
 * are masked).  EINVAL on bad shapes, ECUDA if the device is unusable. */
dbk_status dbk_kv_pool_create(const dbk_pool_config *cfg, void *kv_mem, size_t kv_bytes,
                              dbk_pool **out);
dbk_status dbk_kv_pool_destroy(dbk_pool *pool);

/* Register request req_id (>= 0) with prompt length l_in >= 1 and target
 * output length l_out >= 1 (l_in,i / l_out,i).  It holds 0
 * tokens and a free request slot.  EINVAL if it already exists or no slot
 * is free; EFATAL if ceil((l_in + l_out)/P) > cap_pages or > max_pages_per_req. */
dbk_status dbk_request_begin(dbk_pool *pool, int64_t req_id, int32_t l_in, int32_t l_out);

/* Append n_tok[i] tokens to request req_ids[i] (host arrays, batch order).
 * Pages come lowest-free-first in batch order (R7, R8); all-or-nothing:
 * DBK_ECAP if the batch needs more pages than are free, state unchanged.
 * k, v: device [sum(n_tok)][layers][kv_heads][head_dim] in kv_dtype, rows in
 * batch order; or both NULL = synthetic values from the seeded generator
 * (synth/hashgen.py, kinds K/V, pos = the token's position) with synth_seed.
 * Async on `stream`. */
dbk_status dbk_append_tokens(dbk_pool *pool, int32_t n_req, const int64_t *req_ids,
                             const int32_t *n_tok, const void *k, const void *v,
                             uint64_t synth_seed, void *stream);

/* Finish or preempt: all pages of each request return to the free set (R9),
 * the slot is freed and its device block-table row is cleared before the
 * next launch.  All-or-nothing: ENOENT on an unknown id, EINVAL on an id named twice, and
 * then nothing is released. */
dbk_status dbk_release(dbk_pool *pool, int32_t n_req, const int64_t *req_ids);

/* Swap space ("The swapping method involves
 * temporarily moving data from GPU memory to CPU memory when capacity is
 * exceeded.  The data are moved back to the GPU when space becomes
 * available").  host_mem: caller-owned PINNED host memory (cudaHostAlloc /
 * torch pin_memory; EINVAL otherwise) that outlives the pool; it holds
 * floor(bytes / (layers * kv_heads * 2*P*d*2)) swap pages laid out
 * [layer][swap_page][kv_head][2][P][head_dim] (layer-major, like the pool).
 * NULL detaches.  EINVAL while requests are swapped out. */
dbk_status dbk_swap_space_attach(dbk_pool *pool, void *host_mem, size_t bytes, int64_t *swap_pages_out);

/* Move each request's KV (all its pages, all layers) into swap pages taken
 * lowest-free-first in batch order, then release its device pages and slot
 * (as dbk_release); the request keeps its id, l_in, l_out and ctx.
 * All-or-nothing: ECAP if the swap space lacks pages, ENOENT on an unknown
 * or already swapped id, EINVAL on an id named twice (state unchanged).  The device-to-host copies are
 * copy-engine 2-D copies (one per run of consecutive pages) async on
 * `stream`, ordered before any later write to the released pages on it. */
dbk_status dbk_swap_out(dbk_pool *pool, int32_t n_req, const int64_t *req_ids, void *stream);

/* Bring swapped requests back: each gets a slot and ceil(ctx/P) device pages
 * lowest-free-first in batch order (exactly the pages an append of ctx tokens
 * would take, R7), its KV is copied host-to-device on `stream` and its swap
 * pages are freed.  All-or-nothing: ECAP if device pages are short, EINVAL if
 * slots are short or an id is named twice, ENOENT if an id is not swapped out.  dbk_release of a
 * swapped-out id frees its swap pages. */
dbk_status dbk_swap_in(dbk_pool *pool, int32_t n_req, const int64_t *req_ids, void *stream);

/* Swap pages in use / free, and the bytes moved by swap_out + swap_in so far. */
dbk_status dbk_swap_usage(dbk_pool *pool, int64_t *used_pages, int64_t *free_pages, int64_t *bytes_moved);

/* Host view of one request: ctx (tokens held), n_pages, slot, and up to
 * pages_cap page ids (logical order) into pages_out (nullable). */
dbk_status dbk_request_info(dbk_pool *pool, int64_t req_id, int32_t *ctx, int32_t *n_pages,
                            int32_t *slot, int32_t *pages_out, int32_t pages_cap);
dbk_status dbk_pool_usage(dbk_pool *pool, int64_t *used_pages, int64_t *free_pages);

/* Copy the device block table [max_requests][max_pages_per_req] int32
 * (-1 = empty) to host memory (synchronous on `stream`). */
dbk_status dbk_block_table_d2h(dbk_pool *pool, int32_t *host_out, void *stream);

/* Which decode kernel the pool launches and how: decode_path 1 = K1 (CUDA-core
 * FMA, MHA or GQA fallback), 2 = K2 (tensor-core GQA: TMA tensor tiles + mma);
 * ctas_per_sm = resident CTAs of that kernel; chunk_pages = pages per work item
 * of the last decode batch; launches = kernels this pool has launched. */
typedef struct dbk_pool_info {
    int32_t decode_path, ctas_per_sm, chunk_pages, work_items;
    int64_t launches, last_decode_bytes;
    int32_t tma_rank;   /* K2 tile fetch: 5 = one 5-D TMA box per page tile, 2 = 2-D boxes */
    int32_t _reserved;
} dbk_pool_info;
dbk_status dbk_pool_get_info(dbk_pool *pool, dbk_pool_info *out);

/* ------------------------------------------------------------------------ */
/* Decode step: paged decode attention (+ fused batch statistics)           */
/* ------------------------------------------------------------------------ */

typedef struct dbk_batch {
    int32_t n;             /* active requests (0 = no-op)                        */
    int32_t layer;         /* 0 .. layers-1                                       */
    int32_t fuse_stats;    /* 1: also produce the dbk_stats record (S4)           */
    int32_t chain;         /* 1: the previous operation on `stream` is this pool's *
                            * dbk_decode_step (same batch, another layer): launch  *
                            * as a programmatic dependent so it fills that launch's *
                            * tail (ignored with fuse_stats); 2: the previous      *
                            * operation is a KERNEL producing q / this step's K/V  *
                            * (e.g. the model's QKV GEMM): programmatic dependent  *
                            * launch that waits for it before reading anything;    *
                            * 0: plain stream order                                */
    const int64_t *req_ids;/* host [n], batch order                               */
} dbk_batch;

/* For each request i and q-head h (kv head g = h / (q_heads/kv_heads)):
 *   out[i][h][:] = sum_{j < ctx_i} softmax_j(q[i][h].K_{i,g,j} / sqrt(d)) V_{i,g,j}
 * over the request's paged KV of `layer` (R1, R2; oracle O1).  q: device
 * [n][q_heads][head_dim] kv_dtype; out: device [n][q_heads][head_dim] of
 * out_dtype (0 fp16, 1 bf16, 2 fp32).  fp32 accumulation.  With fuse_stats
 * the same launch reduces the batch statistics record (O3).  n = 0: no launch, q and out
 * untouched; with fuse_stats the record becomes the empty batch's (cap_pages = free_pages =
 * cap, every other field 0; R28).  DBK_ENOENT: an unknown request; DBK_EINVAL: a request
 * holding no tokens or named twice in the batch (nothing launched).  Async. */
dbk_status dbk_decode_step(dbk_pool *pool, const dbk_batch *batch, const void *q, void *out,
                           int32_t out_dtype, void *stream);

/* The same attention for layers [batch->layer, batch->layer + n_layers) of the batch in as few
 * persistent launches as the split-K workspace budget allows (all of them when it fits; the
 * attention-only step, where every layer's q exists before the first launch): a task is
 * (request chunk, kv head, layer), so the work queue spans the layers and no launch edge,
 * ramp or tail separates them.  q of layer batch->layer + l at q + l*q_layer_stride
 * elements, out at out + l*out_layer_stride elements (strides multiples of 8, >= 0).  With
 * fuse_stats the first launch also reduces the statistics record; chain as above for the
 * first launch (the later ones always chain).  launches_out (nullable): kernels launched.
 * Results are identical to n_layers calls of dbk_decode_step.  Async. */
dbk_status dbk_decode_step_layers(dbk_pool *pool, const dbk_batch *batch, int32_t n_layers, const void *q,
                                  int64_t q_layer_stride, void *out, int64_t out_layer_stride, int32_t out_dtype,
                                  void *stream, int32_t *launches_out);

/* Batch statistics of the last fused launch (oracle O3).
 * 16 x int64 = 128 bytes.  step_ns and n_waiting are filled by the host
 * (engine) -- zero from dbk_batch_stats. */
typedef struct dbk_stats {
    int64_t n_active, sum_ctx, sum_ctx_sq, max_ctx, sum_pages, cap_pages, free_pages, over_cap,
        table_mismatch, n_finished, fin_sum_lin, fin_sum_lin_sq, fin_sum_lout, fin_sum_lout_sq,
        step_ns, n_waiting;
} dbk_stats;

/* Copies the device record to host_out; synchronises `stream`. */
dbk_status dbk_batch_stats(dbk_pool *pool, dbk_stats *host_out, void *stream);

/* ------------------------------------------------------------------------ */
/* Chunked prefill (PD fusion)          */
/* ------------------------------------------------------------------------ */

/* One prefill chunk per request: query tokens at positions q_start[i] ..
 * q_start[i] + q_len[i] - 1 of request req_ids[i], whose K/V must already be
 * appended (ctx >= q_start + q_len).  Rows of q / out are the chunks
 * concatenated in batch order: row r = sum_{i' < i} q_len[i'] + j.            */
typedef struct dbk_prefill_batch {
    int32_t n;               /* chunks (0 = no-op)                               */
    int32_t layer;           /* 0 .. layers-1                                     */
    const int64_t *req_ids;  /* host [n]                                          */
    const int32_t *q_start;  /* host [n], >= 0                                    */
    const int32_t *q_len;    /* host [n], >= 1                                    */
} dbk_prefill_batch;

/* Causal paged attention of every chunk token (K7, tcgen05 tensor cores):
 *   out[r][h][:] = sum_{k <= p} softmax_k(q[r][h].K_{i,g,k} / sqrt(d)) V_{i,g,k},
 * p = q_start[i] + j the token's position, g = h / (q_heads / kv_heads) -- the
 * decode formula (R1, R2; oracle O1) with ctx = p + 1 per query row.
 * q: device [rows][q_heads][head_dim] kv_dtype, 16-B aligned; out: device
 * [rows][q_heads][head_dim] out_dtype (0 fp16, 1 bf16, 2 fp32).  fp32
 * accumulation.  EINVAL on a bad chunk or when the pool has no 5-D tensor map
 * (tile index >= 2^31); ENOENT on an unknown id.  Async on `stream`. */
dbk_status dbk_prefill_step(dbk_pool *pool, const dbk_prefill_batch *batch, const void *q, void *out,
                            int32_t out_dtype, void *stream);

/* ------------------------------------------------------------------------ */
/* Full decode step with synthetic weights           */
/* ------------------------------------------------------------------------ */

/* A Llama-2-shaped decoder over the pool's heads (readings R32-R35; oracle O8,
 * oracle/model.py): pre-norm RMSNorm, QKV projection, rotate-half RoPE, paged
 * decode attention (K1/K2 over the pool), O projection + residual, RMSNorm,
 * SwiGLU MLP + residual, final RMSNorm and LM head.  The paper does not
 * define the model; its decode latency is the whole model's ("the enlarged
 * matrix dimensions in the matrix multiplication operations required for
 * larger batches").  fp16 pools only. */
typedef struct dbk_model_config {
    int32_t hidden;        /* H, multiple of 128                                    */
    int32_t ffn;           /* F (SwiGLU inner size), multiple of 128                */
    int32_t vocab;         /* V, multiple of 4 (16-B rows of fp32 logits)           */
    int32_t max_pos;       /* RoPE table rows: positions 0 .. max_pos-1             */
    double rms_eps;        /* 1e-5 (Llama-2)                                        */
    double rope_theta;     /* 10000 (Llama-2)                                       */
    uint64_t weight_seed;  /* synthetic weights (synth/hashgen.py gen_matrix)       */
    uint64_t token_seed;   /* synthetic input token of (req, pos) (gen_token)       */
    int32_t tp_size;       /* tensor parallelism over KV heads and the FFN: 0 or 1 = one GPU;
                            * G > 1: this model holds rank tp_rank's slice (the pool's kv
                            * heads, kv_head_offset = tp_rank * kv_heads; hidden, ffn and vocab
                            * are the GLOBAL sizes) and needs dbk_model_attach_tp           */
    int32_t tp_rank;
} dbk_model_config;

typedef struct dbk_model dbk_model;

/* Bytes of fp16 weights: V*H (embedding) + L*(2H + (Hq+2Hkv)d*H + H*Hq*d +
 * 2F*H + H*F) + H + V*H (LM head), each tensor 256-B aligned. */
size_t dbk_model_weight_bytes(const dbk_pool_config *pool_cfg, const dbk_model_config *cfg);

/* weight_mem: caller-owned device memory of >= dbk_model_weight_bytes bytes,
 * 256-B aligned; the model fills it with the synthetic weights (device
 * generator, synchronous).  The model allocates its activation workspace for
 * the pool's max_requests rows (cudaMalloc).  Every projection runs on the
 * tensor-core GEMM (dbk_gemm_*) with the step's elementwise work fused into its
 * epilogue; the QKV and gate|up weights are stored with their rows permuted for
 * those epilogues (RoPE pairs adjacent, gate/up rows interleaved).  EINVAL on
 * bad shapes (kv_dtype must be fp16, head_dim must divide 128), ECUDA on CUDA
 * failures. */
dbk_status dbk_model_create(dbk_pool *pool, const dbk_model_config *cfg, void *weight_mem, size_t bytes,
                            dbk_model **out);
dbk_status dbk_model_destroy(dbk_model *model);

/* Like dbk_append_tokens but without writing KV: allocates the pages of
 * n_tok[i] more tokens per request (lowest-free-first, all-or-nothing, R7/R8)
 * and advances ctx; the caller (e.g. dbk_model_step) writes those slots
 * before any attention reads them. */
dbk_status dbk_reserve_tokens(dbk_pool *pool, int32_t n_req, const int64_t *req_ids, const int32_t *n_tok,
                              void *stream);

/* One decode step of the whole model for the batch: request i's decode
 * token sits at position p_i = ctx_i - 1 (reserved, not yet written), its input
 * token id is gen_token(token_seed, req_i, p_i).  Writes the token's K/V of
 * every layer into the pool and, if logits != NULL, logits [n][vocab] fp32
 * (device).  fuse_stats: layer 0's attention launch also produces the
 * dbk_stats record (S4).  Async on `stream`. */
dbk_status dbk_model_step(dbk_model *model, int32_t n, const int64_t *req_ids, int32_t fuse_stats,
                          void *logits, void *stream);

/* PD fusion through the model: the decode tokens of req_ids[0..n) (as dbk_model_step)
 * plus every token of each prefill chunk (chunks->req_ids[c], positions q_start[c] ..
 * q_start[c] + q_len[c] - 1, already reserved; chunks->layer is ignored) run as ONE batch
 * of n + sum(q_len) rows through the GEMMs; decode rows attend with K1/K2, chunk rows
 * causally with K7 (R24).  Token ids gen_token(token_seed, req, pos) for every row.
 * logits (nullable): device [n + sum(q_len)][vocab] fp32, rows in that order.  tokens
 * (nullable): device int32 [n], the decode rows' input token ids (e.g. the previous step's
 * samples; clamped into [0, vocab)) instead of gen_token.  sampled (nullable): device int32
 * [n + sum(q_len)], greedy sampling -- the lowest index of each row's largest logit.  EINVAL
 * if the rows exceed max_requests or a chunk lies outside the reserved tokens. */
dbk_status dbk_model_step_pd(dbk_model *model, int32_t n, const int64_t *req_ids, const dbk_prefill_batch *chunks,
                             int32_t fuse_stats, void *logits, const int32_t *tokens, int32_t *sampled,
                             void *stream);

/* Tensor-parallel residual stream ("TP model step").
 * With tp_size = G, the O and down projections of rank r produce partial sums; their GEMM
 * epilogue adds each 32-column chunk straight into the residual buffer of the rank that owns
 * those columns (rank o owns [o H/G, (o+1) H/G)) in THAT rank's memory (TMA reduce-add through
 * CUDA-IPC mappings: NVLink / NVSwitch peer memory across GPUs), a one-warp barrier publishes the
 * step (release / acquire at system scope), and the next RMSNorm reads every owner's slice:
 * the all-reduce's reduce-scatter runs inside the GEMM, its all-gather inside the norm.
 * dbk_tp_create allocates 3 rotating fp32 buffers [rows][hidden] + flags (one cudaMalloc) and
 * writes this rank's 64-byte IPC handle; the caller gathers every rank's handle (rank order)
 * for dbk_tp_open.  hidden % (32 * nranks) == 0, nranks <= 8.  Every rank must run the same
 * sequence of model steps on the same batch (the barriers pair up by count); a rank that never
 * arrives makes the others' barrier kernel trap after 20 s (the step then fails with ECUDA). */
typedef struct dbk_tp dbk_tp;
dbk_status dbk_tp_create(int32_t nranks, int32_t rank, int32_t device, int64_t rows, int32_t hidden,
                         void *handle_out_64, dbk_tp **out);
dbk_status dbk_tp_open(dbk_tp *t, const void *handles /* [nranks][64] */);
dbk_status dbk_tp_barrier(dbk_tp *t, void *stream);  /* a standalone barrier (async on stream) */
dbk_status dbk_tp_destroy(dbk_tp *t);
/* The model's residual stream becomes the communicator's buffers (rows >= max_requests,
 * same nranks / rank / hidden as the model's config, else EINVAL). */
dbk_status dbk_model_attach_tp(dbk_model *model, dbk_tp *tp);

/* Introspection (tests): device pointers of the activation workspace of the last
 * step, rows = batch order: [0] x fp32 [n][H] (residual stream), [1] h fp16 [n][H]
 * (last norm output), [2] NULL (the QKV output lives only in the GEMM epilogue),
 * [3] q fp16 [n][Hq][d] (after RoPE), [4] attention out fp16 [n][Hq*d], [5] NULL
 * (gate|up: fused into the SiLU epilogue), [6] act fp16 [n][F] -- all of the LAST
 * layer; [7] logits fp32 [n][V] (internal buffer). */
dbk_status dbk_model_buffers(dbk_model *model, void **ptrs_out_8);

/* Time split of the model steps since the last reset (CUDA events on the
 * step's stream): attention launches vs everything else (GEMMs, norms, RoPE). */
dbk_status dbk_model_timing(dbk_model *model, double *attn_ms, double *total_ms, int64_t *steps,
                            int32_t reset);

/* ------------------------------------------------------------------------ */
/* Tensor-core GEMM of the model projections (NEXT row 3)                    */
/* ------------------------------------------------------------------------ */

/* The model's projections Y = X W^T ("the enlarged matrix dimensions in the
 * matrix multiplication operations required for larger batches")
 * on the 5th-generation tensor cores (tcgen05.mma, TMEM accumulators, TMA),
 * persistent (gemm_tc.cu).  dbk_model_* runs the same kernel with the decode
 * step's elementwise work fused into its epilogue; this entry point exposes the
 * plain forms for tests and measurement.  cta_group: 1 = one SM per 128 weight
 * rows, 2 = CTA pairs (cta_group::2, 256 weight rows per pair).  A launch with
 * very few whole weight tiles (<= SMs / (8 * cta_group) at M <= 256) splits K:
 * fp32 partials go into a workspace the handle allocates at its first such
 * launch (M x N x 4 bytes, synchronous cudaMalloc: not inside a stream capture)
 * and keeps until destroy, so one handle's launches must be stream-ordered. */
typedef struct dbk_gemm dbk_gemm;
dbk_status dbk_gemm_create(int32_t device, int32_t cta_group, dbk_gemm **out);
/* x: device fp16 [M][ldx] row-major (activations), w: device fp16 [N][K]
 * row-major (weights, K contiguous), y: device [M][ldy] row-major;
 * mode 0: y (fp16) = x w^T; 1: y (fp32) = x w^T; 2: y (fp32) += x w^T
 * (stream-K: K is split over the SMs and each partial product is added into y
 * by the TMA unit, so the order of the fp32 additions varies run to run);
 * 4: SwiGLU, y (fp16) [M][N/2] with y[m][j] = silu(z[m][2j]) * z[m][2j+1],
 * z = x w^T (w's rows interleaved gate_j, up_j; N % (128 * cta_group) == 0).
 * fp32 accumulation.  Async on `stream`.  EINVAL unless K % 64 == 0, N >= 1,
 * ldx >= K, ldx % 8 == 0, ldy >= N, x, w and the rows of y 16-B aligned;
 * M == 0 is a no-op. */
dbk_status dbk_gemm_run(dbk_gemm *g, int32_t M, int32_t N, int32_t K, const void *x, int64_t ldx, const void *w,
                        void *y, int64_t ldy, int32_t mode, void *stream);
/* Measurement hook: trace = device uint64 [148][8] (or NULL = off); the following launches
 * stamp %globaltimer per CTA at start, after setup, first operands in shared memory, last
 * MMA issued, last accumulator ready, its first TMEM chunk loaded, epilogue done, exit
 * (slots 0-7).  mode 0 = normal; 1 = the operand pipeline without MMAs, 2 = the MMAs without
 * operand loads (both give garbage results: they time one side of the pipeline alone). */
dbk_status dbk_gemm_trace(dbk_gemm *g, void *trace, int32_t mode);
/* Measurement hook: bn > 0 fixes the activation tile width (rounded up to 32, <= 256) of the
 * following launches; 0 restores the cost model's choice. */
dbk_status dbk_gemm_force_tile(dbk_gemm *g, int32_t bn);
/* The tiling of the last dbk_gemm_run (measurement / tests): activation tile width bn and
 * units (tiles) in total; units_a < units when the last wave was re-tiled -- units [units_a,
 * units) use the narrower width bn_b.  split > 1: K was split that many ways.  Any out pointer
 * may be NULL. */
dbk_status dbk_gemm_last_plan(dbk_gemm *g, int32_t *bn, int32_t *bn_b, int32_t *units_a, int32_t *units,
                              int32_t *split);
dbk_status dbk_gemm_destroy(dbk_gemm *g);

/* ------------------------------------------------------------------------ */
/* Synthetic input generator (input side only; none of the method's math)  */
/* ------------------------------------------------------------------------ */

/* out[r][h][e] = value(seed, kind, req[r], pos[r], layer, h, e) * 2^scale_log2,
 * the generator of synth/hashgen.py, for r < n_rows, h < n_heads, e < d.
 * req, pos: host arrays [n_rows]; out: device, dtype 0 fp16 / 1 bf16 / 2 fp32. */
dbk_status dbk_synth_fill(uint64_t seed, int32_t kind, int32_t n_rows, const int64_t *req,
                          const int32_t *pos, int32_t layer, int32_t n_heads, int32_t d,
                          int32_t scale_log2, int32_t dtype, void *out, void *stream);

/* Measurement utility (not part of the method): read `bytes` (multiple of 16) of device
 * memory once with 16-byte streaming loads and return the kernel's CUDA-event time in
 * ms -- the read-only HBM bandwidth of this GPU, reported beside the attention
 * kernel's.  Synchronous on `stream`. */
dbk_status dbk_probe_read_bandwidth(const void *buf, size_t bytes, int32_t device, void *stream,
                                    double *ms_out);

/* Measurement utility (not part of the method): with DBK_TRACE_TASKS=N set when the pool is
 * created, every decode warp task (K1/K2) appends a record of 4 x u64 -- start and end
 * (%globaltimer ns), SM id << 32 | launch sequence, task << 32 | pages -- up to N records.
 * Copies min(count, cap) records to host (nullable) and their number to n_out (0 without
 * tracing); reset = 1 restarts the buffer.  Synchronises the device. */
dbk_status dbk_pool_trace_d2h(dbk_pool *pool, void *host, int64_t cap, int64_t *n_out, int32_t reset);

/* ------------------------------------------------------------------------ */
/* Scheduler: Algorithm 1 (memory), Algorithm 2 (SLA), min, static          */
/* ------------------------------------------------------------------------ */

enum { DBK_POLICY_STATIC = 0, DBK_POLICY_MEMORY = 1, DBK_POLICY_SLA = 2, DBK_POLICY_COMBINED = 3 };
enum { DBK_R_STATIC = 0, DBK_R_MEMORY = 1, DBK_R_SLA = 2, DBK_R_MIN = 3, DBK_R_CARRY = 4 };

typedef struct dbk_sched_config {
    int32_t policy;                 /* DBK_POLICY_*                                       */
    int32_t b_static;               /* static baseline b                    */
    int32_t b_min, b_max, b0;       /* B_min, B_max; b_0                    */
    int32_t alpha, delta;           /* Alg. 2 constants (R15)               */
    int32_t w_len;                  /* moments window, completed requests (R11)           */
    int32_t w_sla;                  /* SLA window, decode steps (R14)                     */
    int32_t refresh_steps;          /* L0 refresh period (R12)                            */
    int32_t page_size, _reserved;
    double eps_m;                   /* epsilon_M in (0, 0.5] (Eq. 2; R5)     */
    double d_sla_ms, eps_d_ms;      /* D_SLA, epsilon_D (Eq. 3)              */
    int64_t bytes_per_token;        /* beta: KV bytes per token, all layers, this GPU     */
    int64_t prior_n, prior_sum_lin, prior_sum_lin_sq, prior_sum_lout, prior_sum_lout_sq;
} dbk_sched_config;

typedef struct dbk_sched dbk_sched;

dbk_status dbk_sched_create(const dbk_sched_config *cfg, dbk_sched **out);
dbk_status dbk_sched_destroy(dbk_sched *s);

/* Consume the GLOBAL statistics of the decode step just finished (step_ns
 * filled) and return b_{t+1} (PAPER.md:219 b* = min{b_mem, b_SLA}).
 * mem_cap_bytes: M_max of the whole job (eta via R4); sla_ms > 0 overrides
 * cfg.d_sla_ms; n_prefill_waiting = N^p (R13).  rationale_out: DBK_R_*.
 * Integer-exact (R6); EINFEASIBLE is never returned here (b_quad = 0 gives
 * L0 = eta and b = N^d). */
dbk_status dbk_choose_batch_size(dbk_sched *s, const dbk_stats *global, int64_t mem_cap_bytes,
                                 double sla_ms, int32_t n_prefill_waiting, int32_t *b_out,
                                 int32_t *rationale_out);

typedef struct dbk_sched_state {
    int64_t t, eta, L0, b_quad, theta_q;
    int64_t win_n, win_S, win_V2;   /* window moments: n, S = sum(l_in+l_out), n^2 v */
    int32_t b, b_mem, b_sla, b_low, b_high, sla_count;
} dbk_sched_state;
dbk_status dbk_sched_get_state(dbk_sched *s, dbk_sched_state *out);

/* Pure helpers (host), exposed for tests: theta_q = floor(Theta^-1(1-eps)*2^24 + 1/2)
 * (Wichura AS241); b_quad = largest b with the R6 predicate true (0 if none). */
dbk_status dbk_theta_q(double eps_m, int64_t *theta_q_out);
dbk_status dbk_b_quad(int64_t n, int64_t S, int64_t V2, int64_t eta, int64_t theta_q,
                      int64_t *b_out);

/* ------------------------------------------------------------------------ */
/* Engine: one continuous-batching iteration per call (S1 -> S7, R17-R22)    */
/* ------------------------------------------------------------------------ */

typedef struct dbk_engine_config {
    int32_t n_requests;
    int32_t q_scale_log2;           /* synthetic q scale (peaked variant: 4)                */
    const int64_t *arrival_ns;      /* host [n_requests], non-decreasing (copied)          */
    const int32_t *l_in;            /* host [n_requests] (copied)                          */
    const int32_t *l_out;           /* host [n_requests] (copied)                          */
    const int64_t *req_ids;         /* host [n_requests] global ids, or NULL = 0..n-1      */
    int64_t mem_cap_bytes;          /* M_max of the WHOLE job (all ranks)                  */
    double sla_ms;                  /* <= 0: cfg value of the scheduler                    */
    uint64_t synth_seed;
    int32_t out_dtype;              /* 0 fp16, 1 bf16, 2 fp32                              */
    int32_t time_attention;         /* 1: CUDA events around each attention launch         */
    int32_t rank, world;            /* DP request shards (R21); 0, 1 for one GPU           */
    int32_t pd_fusion;              /* 1: PD fusion -- admitted prompts are prefilled in     *
                                     * chunks of c_t = max(0, b_t - N^d) tokens inside the    *
                                     * decode iteration (R25-R28; device-resident mode only)  */
    int32_t preempt_mode;           /* 0: recompute (R18); 1: swap a victim to the pool's   *
                                     * swap space when it has room, else recompute (R29-R31;*
                                     * needs dbk_swap_space_attach; not with pd_fusion)      */
    int32_t pd_token_budget;        /* PD fusion only.  0: the iteration's token budget is b_t *
                                     * (R25: c_t = b_t - N^d).  > 0: a fixed token budget per *
                                     * iteration (R36: c_t = budget - N^d) while b_t still     *
                                     * bounds running + prefilling requests                    */
    int32_t per_layer_launches;     /* device-resident decode-only steps: 0 = the layers go   *
                                     * through dbk_decode_step_layers (multi-layer launches); *
                                     * 1 = one PDL-chained launch per layer (as a model's     *
                                     * layer-by-layer step would issue them)                  */
} dbk_engine_config;

typedef struct dbk_engine dbk_engine;

/* Buffers of one step.  Device-resident mode: host_* all NULL; the engine
 * generates q (synthetic, pos = ctx-1) into q_dev and appends the decode
 * token's K/V with the synthetic generator.  With PD fusion the prefill
 * chunk's rows follow the decode rows in q_dev / out_dev: decode rows
 * [0, N^d), chunk rows [N^d, N^d + c_t) (c_t is clamped to max_requests - N^d).  End-to-end mode: host_q
 * [layers][n][q_heads][d], host_k / host_v [layers][n][kv_heads][d] (pinned
 * host, kv_dtype; layer-major, as a model produces them) are copied H2D into
 * q_dev / kv_dev layer by layer each step and out is copied D2H into host_out
 * [layers][n][q_heads][d] (out_dtype).
 * q_dev: [layers][max_requests][q_heads][d]; out_dev: same shape, out_dtype;
 * kv_dev: [2][layers][max_requests][kv_heads][d] (e2e only). */
typedef struct dbk_engine_buffers {
    void *q_dev, *out_dev, *kv_dev;
    const void *host_q, *host_k, *host_v;
    void *host_out;
    int32_t *host_tokens;  /* full-model mode, end to end: pinned host int32 [n_requests] indexed
                            * by trace index; each step reads the decode rows' input tokens
                            * from it (H2D) and writes their greedy samples back (D2H) */
} dbk_engine_buffers;

typedef struct dbk_step_record {
    int64_t t, clock_ns, step_ns, sum_ctx, used_pages, table_hash;
    int32_t b_t, b_next, n_admitted, n_preempted, n_decode, n_finished, rationale, n_waiting;
    int64_t h2d_bytes, d2h_bytes;
    int32_t launches;
    int32_t n_prefill;              /* PD fusion: prompt tokens prefilled this step (this rank) */
    int32_t n_swap_out, n_swap_in;  /* swap preemption: victims swapped out / readmitted by swap-in */
    int64_t swap_bytes;             /* bytes the swaps of this step moved (both directions)   */
} dbk_step_record;

/* The engine over a trace (arrivals sorted, lengths >= 1, request ids unique -- EINVAL
 * otherwise); DBK_EFATAL when one request alone cannot fit the cap. */
dbk_status dbk_engine_create(dbk_pool *pool, dbk_sched *sched, const dbk_engine_config *cfg,
                             dbk_engine **out);
dbk_status dbk_engine_destroy(dbk_engine *e);

/* Run one iteration (single GPU, or with a communicator attached).  Returns
 * DBK_ENOENT (and does nothing) when every request has finished. */
dbk_status dbk_engine_step(dbk_engine *e, const dbk_engine_buffers *bufs, void *stream,
                           dbk_step_record *rec);
/* Split form for multi-GPU with a caller-side exchange: launch the step and
 * return this rank's record (stream synchronised) ... */
dbk_status dbk_engine_step_launch(dbk_engine *e, const dbk_engine_buffers *bufs, void *stream,
                                  dbk_stats *local_out);
/* ... then finish it with the reduced global record (retire, windows, b_{t+1}). */
dbk_status dbk_engine_step_finish(dbk_engine *e, const dbk_stats *global, dbk_step_record *rec);

dbk_status dbk_engine_done(dbk_engine *e, int32_t *done);
/* The last step's decode batch: n, then req_ids[n], ctx[n] (host, cap entries). */
dbk_status dbk_engine_last_batch(dbk_engine *e, int32_t *n, int64_t *req_ids, int32_t *ctx,
                                 int32_t cap);
/* Full-model mode (NEXT row 3): every decode step runs dbk_model_step (QKV / O /
 * MLP / LM-head GEMMs + the attention) instead of the synthetic-q attention; the
 * decode token's KV is written by the model (dbk_reserve_tokens + RoPE epilogue).
 * Device-resident, non-PD engines only; NULL detaches.  EINVAL if the model was created on
 * another pool than the engine's. */
dbk_status dbk_engine_attach_model(dbk_engine *e, dbk_model *model);
/* Per-request timeline on the engine clock (ns), for trace index i < n (host
 * arrays, nullable): first_admit_ns[i] = clock of the step that first admitted
 * it, finish_ns[i] = end of the step that emitted its last token; -1 where it
 * has not happened yet or the request belongs to another DP rank.  Feeds the
 * scheduling-delay criterion of the capacity experiment. */
dbk_status dbk_engine_request_times(dbk_engine *e, int32_t n, int64_t *first_admit_ns, int64_t *finish_ns);
/* Attention timing accumulated with time_attention = 1: total ms of the
 * attention launches (CUDA events on the launching stream), their count (kernels:
 * a multi-layer launch counts once) and the algorithmic bytes they moved. */
dbk_status dbk_engine_attn_timing(dbk_engine *e, double *ms, int64_t *launches, int64_t *bytes,
                                  int32_t reset);

/* ------------------------------------------------------------------------ */
/* Multi-GPU statistics exchange (NCCL over NVLink)        */
/* ------------------------------------------------------------------------ */

enum { DBK_MODE_DP = 0, DBK_MODE_TP = 1 };
typedef struct dbk_comm dbk_comm;

/* 128-byte ncclUniqueId, produced on rank 0 and broadcast by the caller. */
dbk_status dbk_comm_unique_id(void *id_out_128);
dbk_status dbk_comm_create(int32_t nranks, int32_t rank, const void *id_128, int32_t device,
                           dbk_comm **out);
dbk_status dbk_comm_destroy(dbk_comm *c);
/* ncclAllGather of the 128-byte records, then dbk_stats_reduce. */
dbk_status dbk_stats_allgather(dbk_comm *c, const dbk_stats *local, dbk_stats *all,
                               dbk_stats *global, int32_t mode, void *stream);
/* Host reduction: DP = SUM (max_ctx MAX, over_cap OR); TP = all equal
 * (EINVAL otherwise); both: step_ns = MAX. */
dbk_status dbk_stats_reduce(const dbk_stats *all, int32_t nranks, int32_t mode, dbk_stats *global);
/* This communicator's size and rank as NCCL reports them (ncclCommCount, ncclCommUserRank). */
dbk_status dbk_comm_info(dbk_comm *c, int32_t *nranks, int32_t *rank);
/* dbk_engine_step then exchanges every step's record through `c`.  DP (request shards): the
 * communicator must have cfg.world ranks; TP (KV-head shards): the engine has world 1 and
 * every rank serves all requests.  EINVAL otherwise.  NULL detaches. */
dbk_status dbk_engine_attach_comm(dbk_engine *e, dbk_comm *c, int32_t mode);
/* The last exchange of dbk_engine_step: up to cap per-rank records in rank order (each with
 * that rank's own device-timed step_ns) into all (nullable), their count, the host time of
 * that exchange (us: H2D + all-gather + D2H + reduce) and the total / count since the last
 * reset.  nranks = 0 before the first exchange or without a communicator. */
dbk_status dbk_engine_last_exchange(dbk_engine *e, dbk_stats *all, int32_t cap, int32_t *nranks, double *us,
                                    double *us_total, int64_t *count, int32_t reset);

/* ------------------------------------------------------------------------ */
/* Mailbox exchange: the same records over peer memory, no collective launch  */
/* ------------------------------------------------------------------------ */

/* SURVEY.md §8(e) "B200-native v2".  Each rank owns a device mailbox (2 x nranks slots of
 * 256 B) exported with CUDA IPC; every peer maps it (P2P over NVLink/NVSwitch; the same
 * device when ranks share a GPU).  One single-warp kernel per step stores the rank's 128-B
 * record into every mailbox, waits (acquire loads) for the other ranks' records of the same
 * step and writes the gathered records into mapped pinned host memory -- no H2D, no NCCL
 * launch, no separate D2H.  1 <= nranks <= 32. */
typedef struct dbk_mbox dbk_mbox;

/* Allocate this rank's mailbox on `device`; handle_out_64 receives its 64-byte IPC handle,
 * which the caller gathers from every rank (rank order) for dbk_mbox_open. */
dbk_status dbk_mbox_create(int32_t nranks, int32_t rank, int32_t device, void *handle_out_64, dbk_mbox **out);
/* Map every peer's mailbox: handles = nranks x 64 bytes in rank order (own entry ignored).
 * ECUDA if a handle cannot be opened (e.g. no peer access). */
dbk_status dbk_mbox_open(dbk_mbox *m, const void *handles);
dbk_status dbk_mbox_destroy(dbk_mbox *m);
/* Standalone exchange of a host record (every rank calls it once per exchange, in the same
 * order): all = the nranks records (rank order), global = dbk_stats_reduce(all, mode).
 * Synchronous on `stream`; ECUDA if a peer's record does not arrive within 20 s. */
dbk_status dbk_mbox_exchange(dbk_mbox *m, const dbk_stats *local, dbk_stats *all, dbk_stats *global, int32_t mode,
                             void *stream);
/* dbk_engine_step then exchanges through the mailbox instead of a communicator: the step's
 * first kernel stamps %globaltimer, its last one builds the record from the device
 * statistics with step_ns = the device time between the two (S5), exchanges it and the host
 * reduces (DP: nranks = cfg.world; TP: engine world 1).  NULL detaches.  EINVAL on a size
 * mismatch or when a communicator is attached. */
dbk_status dbk_engine_attach_mbox(dbk_engine *e, dbk_mbox *m, int32_t mode);

#ifdef __cplusplus
}
#endif
#endif /* DBK_H_ */
