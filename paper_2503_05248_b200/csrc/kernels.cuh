// Device-side data structures and kernel launchers (internal to libdbk).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace dbk {

// Per-request metadata of one decode batch (uploaded once per batch change).
struct ReqMeta {
    int64_t req_id;
    int32_t slot;        // block-table row
    int32_t ctx;         // tokens in KV incl. this step's token
    int32_t l_in, l_out; // for the finishing statistics (O3)
    int32_t chunk_base;  // first split-K workspace row of this request (if nchunks > 1)
    int32_t nchunks;     // work items of this request
};
static_assert(sizeof(ReqMeta) == 32, "ReqMeta layout");

// One work item = a chunk of <= kItemPages pages of one request (the unit a warp task streams),
// with everything the decode kernels need to start it in ONE load; its physical page ids are
// read from the device block table, row `slot`, entries pg0 .. pg0 + n - 1.
struct ItemMeta {
    int32_t i;            // batch index
    int32_t c;            // chunk index within the request
    int32_t pg0, n;       // first logical page and page count
    int32_t ctx;          // tokens of the request (incl. this step's)
    int32_t chunk_base;   // first split-K workspace row of the request (if nchunks > 1)
    int32_t nchunks;      // work items of the request
    int32_t slot;         // block-table row (page ids, statistics)
};
static_assert(sizeof(ItemMeta) == 32, "ItemMeta layout");
constexpr int kItemPages = 64;

struct DecodeParams {
    const uint8_t *kv_layer;     // KV base of the first layer of this launch (`layer`)
    int64_t page_stride;         // bytes per (layer, page): kv_heads * tile_bytes
    const int32_t *block_table;  // [max_requests][bt_stride]
    int32_t bt_stride;
    int32_t n;                   // requests in the batch
    const ReqMeta *req;          // [n]
    const ItemMeta *items;       // [n_items], longest first
    int32_t n_items;
    int32_t chunk_pages;         // pages per work item
    const void *q;               // [n][q_heads][D]
    void *out;                   // [n][q_heads][D]
    int32_t out_dtype;           // 0 fp16, 1 bf16, 2 fp32
    int32_t q_heads;
    float scale_log2;            // log2(e) / sqrt(D)
    float *ws_o;                 // [n_items][q_heads][D] split-K partial numerators
    float2 *ws_ml;               // [n_items][q_heads] (running max in log2 units, denominator)
    int32_t *counters;           // [n][kv_heads] arrival counters (zero between launches)
    // fused batch statistics (S4)
    int32_t fuse_stats;
    int32_t max_pages_per_req;
    unsigned long long *stats;   // 16 x u64, zeroed before the launch
    int32_t *stats_done;         // zero between launches
    int64_t cap_pages;
    // K2 (tensor-core GQA) addressing through the pool-wide 2-D tensor map
    int32_t layer;               // first layer of this launch
    int32_t kv_heads;
    // one launch may stream n_layers consecutive layers (attention-only step: every layer's q is
    // ready before the first launch); task t = (l * n_items + item) * kv_heads + head
    int32_t n_layers;
    int64_t layer_stride;        // bytes between layers in the pool
    int64_t q_layer_stride;      // elements between layers of q
    int64_t out_layer_stride;    // elements between layers of out
    int32_t n_ws_rows;           // split-K workspace rows per layer (counters: n per layer)
    // persistent CTAs: tasks t = work_item * kv_heads + kv_head handed out by an atomic
    // counter; task_counter[0] = next task, [1] = exited CTAs (both reset by the last CTA)
    int32_t n_tasks;
    int32_t *task_counter;
    int32_t tma_rank;            // K2: 5 = one 5-D box per tile, 2 = 2-D boxes of 16 x 64
    int32_t half_boxes;          // K2: 1 = GqaMaps::half (8-token boxes) is valid: a last page
                                 //  holding <= 8 tokens moves only its first 8 K / V rows
    // 1: programmatic dependent launch after the previous decode launch on the stream (its
    // scratch -- split-K workspace, arrival and task counters -- is the other parity's);
    // 2: programmatic dependent launch after the kernel that wrote q / the new K/V: every warp
    // waits on the grid dependency before its first global read
    int32_t pdl;
    int32_t seq;                 // this decode launch's sequence number (>= 1, per pool)
    int32_t *done_seq;           // sequence number of the last decode grid whose scratch is reset
    // measurement only (DBK_TRACE_TASKS): per-task timeline records, null in production runs
    unsigned long long *trace;   // [0] = record counter, records of 4 x u64 from index 4
    int32_t trace_cap;           // records
    int32_t trace_seq;           // launch sequence number stamped into the records
};

// Launch with (pdl) or without the programmatic-stream-serialization attribute.
template <typename... KArgs, typename... Args>
cudaError_t launch_kernel(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                          Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<Args &&>(args)...);
}

struct AppendJob {
    int64_t req_id;
    int32_t pos0;     // position of the first token written by this job
    int32_t ntok;     // tokens in this job (all in one page)
    int32_t phys;     // physical page
    int32_t src_row;  // first source row (explicit K/V), -1 = synthetic
};
static_assert(sizeof(AppendJob) == 24, "AppendJob layout");

struct AppendParams {
    uint8_t *kv;                 // pool base
    int64_t layer_stride, page_stride, tile_bytes;
    const AppendJob *jobs;
    int32_t n_jobs, layers, kv_heads;
    const void *k_src, *v_src;   // [rows][layers][kv_heads][D] or null (synthetic); with
                                 // src_layer_rows > 0: [layers][src_layer_rows][kv_heads][D]
    int32_t src_layer_rows = 0;
    uint64_t seed;
    int32_t head0 = 0;           // global index of kv head 0 (KV-head TP shard) for the generator
    int32_t layer0 = 0;          // this launch writes layers [layer0, layer0 + n_launch_layers)
    int32_t n_launch_layers = 0; // 0 = all layers
};

struct BtDelta {
    int32_t slot, idx, val;
};

// K7 (chunked prefill): one tile = up to 128 / group query tokens of one request's chunk.
struct PrefTile {
    int32_t slot;      // block-table row
    int32_t q_start;   // position of the chunk's first token
    int32_t j0;        // first chunk token of this tile
    int32_t rows_tok;  // tokens in this tile
    int32_t q_row0;    // row of the chunk's first token in q / out ([rows][q_heads][D])
    int32_t _pad[3];
};
static_assert(sizeof(PrefTile) == 32, "PrefTile layout");

struct PrefillParams {
    const int32_t *block_table;
    int32_t bt_stride;
    int32_t layer;
    int64_t cap_pages;
    int32_t kv_heads, q_heads;
    const PrefTile *tiles;
    const void *q;       // [rows][q_heads][D], pool dtype
    void *out;           // [rows][q_heads][D]
    int32_t out_dtype;
    float scale_log2;
};

// K2's tensor maps over the pool: `full` moves one (page, kv head) tile (5-D: one box; 2-D: boxes
// of 16 rows x 64 elements), `half` boxes of 8 rows x 64 elements (2-D, 128B-swizzled: each lands
// on one 1024-byte swizzle atom of the full tile's layout) for a request's last page when it
// holds <= 8 tokens.
struct GqaMaps {
    CUtensorMap full;
    CUtensorMap half;
};

// launchers (return cudaGetLastError() of the launch)
// maps != nullptr and group >= 2 selects K2 (tensor cores); otherwise K1 (CUDA cores).
// Persistent launch of min(ctas, p.n_tasks) CTAs (ctas = SMs x resident CTAs per SM).
cudaError_t launch_decode(const DecodeParams &p, int kv_dtype, int head_dim, int group,
                          int ctas, const GqaMaps *maps, cudaStream_t s);
cudaError_t launch_decode_gqa(const DecodeParams &p, int kv_dtype, int head_dim, int group,
                              int ctas, const GqaMaps &maps, cudaStream_t s);
int decode_gqa_ctas_per_sm(int kv_dtype, int head_dim, int group);
cudaError_t launch_append(const AppendParams &p, int kv_dtype, int head_dim, cudaStream_t s);
cudaError_t launch_bt_apply(int32_t *bt, int32_t stride, const BtDelta *d, int32_t n,
                            cudaStream_t s);
cudaError_t launch_synth_rows(uint64_t seed, int kind, int n_rows, const int64_t *req,
                              const int32_t *pos, int layer, int n_heads, int d, int scale_log2,
                              int dtype, void *out, cudaStream_t s);
// out[l][row0 + r][h][:] = synth(seed, kind, req[r], pos[r], l, head0 + h) for all layers (device req/pos).
cudaError_t launch_synth_rows_layers(uint64_t seed, int kind, int n_rows, const int64_t *req, const int32_t *pos,
                                    int layers, int layer_rows, int row0, int n_heads, int head0, int d,
                                    int scale_log2, int dtype, void *out, cudaStream_t s);
// q[l][i][h][:] = synth(seed, q, req_i, ctx_i - 1, l, head0 + h) for all layers, layer stride layer_rows rows.
cudaError_t launch_synth_q(uint64_t seed, const ReqMeta *req, int n, int layers, int layer_rows,
                           int q_heads, int head0, int d, int scale_log2, int dtype, void *q, cudaStream_t s);
int decode_ctas_per_sm(int kv_dtype, int head_dim, int group);
// K7: grid (n_tiles, kv_heads); needs the pool's 5-D tensor map.
cudaError_t launch_prefill(const PrefillParams &p, int kv_dtype, int head_dim, int group, int n_tiles,
                           int kv_heads, const CUtensorMap &tmap, cudaStream_t s);
int prefill_rows_per_tile();
cudaError_t launch_read_probe(const void *buf, size_t bytes, uint32_t *sink, int sms, cudaStream_t s);

}  // namespace dbk
