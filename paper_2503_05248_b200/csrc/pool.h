// Internal definition of dbk_pool (host bookkeeping + device metadata).
#pragma once

#include <cstdint>
#include <functional>
#include <queue>
#include <unordered_map>
#include <vector>

#include "common.h"
#include "kernels.cuh"

namespace dbk {

// Free-page bitmap; take_lowest() returns the lowest-numbered free page (R7).
struct PageBitmap {
    std::vector<uint64_t> words;  // bit = 1: free
    int64_t free_count = 0;
    size_t hint = 0;              // no free page below word `hint`
    void init(int64_t cap);
    int64_t take_lowest();
    void give_back(int64_t page);
};

struct Request {
    int64_t id = 0;
    int32_t l_in = 0, l_out = 0, ctx = 0, slot = -1;
    std::vector<int32_t> pages;   // logical page -> physical page
};

// A request whose KV lives in the host swap space (swap preemption, NEXT row 4): no device
// pages and no slot; swap_pages[k] holds its logical page k.
struct SwappedRequest {
    int32_t l_in = 0, l_out = 0, ctx = 0;
    std::vector<int32_t> swap_pages;
};

dbk_status flush_deltas(dbk_pool *p, cudaStream_t s);
// layers_hint: layers one launch will stream (the chunk-size rule sizes tasks per launch)
dbk_status prepare_batch(dbk_pool *p, int32_t n, const int64_t *ids, cudaStream_t s, int32_t layers_hint = 1);
// dbk_append_tokens in two halves: bookkeeping + job upload, then per-layer-range KV writes
dbk_status append_plan(dbk_pool *p, int32_t n, const int64_t *ids, const int32_t *n_tok, bool explicit_rows,
                       cudaStream_t s, bool upload_jobs = true);
dbk_status append_launch(dbk_pool *p, const void *k, const void *v, uint64_t seed, int32_t layer0, int32_t nl,
                         cudaStream_t s, int32_t src_layer_rows = 0);

}  // namespace dbk

struct dbk_pool {
    dbk_pool_config cfg{};
    uint8_t *kv = nullptr;
    size_t kv_bytes = 0;
    int64_t elt = 2, tile_bytes = 0, page_stride = 0, layer_stride = 0;
    dbk::PageBitmap pages;
    std::unordered_map<int64_t, dbk::Request> reqs;
    // host swap space (caller-owned pinned memory, layout [layer][swap page][page_stride bytes])
    uint8_t *swap_host = nullptr;
    int64_t swap_cap = 0;
    dbk::PageBitmap swap_pages;
    std::unordered_map<int64_t, dbk::SwappedRequest> swapped;
    int64_t swap_bytes_moved = 0;             // bytes copied by swap_out + swap_in (counter)
    std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> free_slots;
    std::vector<int32_t> host_bt;             // mirror of the device table
    int32_t *d_bt = nullptr;
    std::vector<dbk::BtDelta> pending;        // device-table updates not yet applied
    std::vector<dbk::AppendJob> jobs;
    dbk::UploadBuffer up_delta, up_append, up_meta, up_rows;
    uint64_t epoch = 1;                       // bumped by every mutation
    // cached decode-batch metadata
    bool meta_valid = false;
    uint64_t meta_epoch = 0;
    std::vector<int64_t> meta_ids;
    std::vector<dbk::ReqMeta> meta_req;
    std::vector<uint8_t> slot_seen;  // prepare_batch: block-table slots named by the batch (repeat check)
    std::vector<int2> meta_work;
    std::vector<uint8_t> meta_blob;
    int32_t meta_items = 0, meta_chunk_pages = 0, meta_ws_rows = 0, meta_layers_hint = 1;
    int64_t ws_budget_bytes = 512ll << 20;   // split-K workspace per scratch parity (layer groups)
    int32_t max_layers_per_launch = 0;       // 0: as many as the workspace budget allows
    const dbk::ReqMeta *d_req = nullptr;
    const dbk::ItemMeta *d_items = nullptr;
    // split-K workspace, arrival counters, statistics record
    float *d_ws_o = nullptr;
    float2 *d_ws_ml = nullptr;
    size_t ws_cap = 0;
    int32_t *d_counters = nullptr;
    int64_t *d_stats = nullptr;
    int32_t *d_stats_done = nullptr;
    int32_t *d_task_counter = nullptr;        // persistent decode: [2 parities][next task, exited warps]
    int32_t *d_done_seq = nullptr;            // last decode grid whose scratch is reset (PDL trigger)
    int32_t decode_seq = 0;                   // decode launches so far (DecodeParams::seq)
    dbk_stats *h_stats = nullptr;
    int num_sms = 148, ctas_per_sm = 1;
    // pages per warp task: <= 64 (two page ids per lane); 32 measured best (profiles/r01_tune.txt)
    int64_t max_chunk_pages = 32, force_chunk_pages = 0;
    int64_t tasks_per_warp = 3;               // chunk size target: total tasks ~ tasks_per_warp x warps
    int64_t last_decode_bytes = 0;
    int64_t n_launches = 0;                   // kernels launched by this pool (gpu_launches)
    int launch_parity = 0;                    // scratch copy of the next decode launch
    bool pdl_enabled = true;
    unsigned long long *d_trace = nullptr;    // DBK_TRACE_TASKS=N: task timeline buffer (measurement)
    int32_t trace_cap = 0;
    // pool-wide 2-D tensor map (rows of head_dim elements, 16 x 64 boxes, 128B swizzle) for K2
    alignas(64) CUtensorMap tmap;
    bool has_tmap = false;
    alignas(64) CUtensorMap tmap_half;  // K2: 8-row boxes for last pages holding <= 8 tokens
    bool has_tmap_half = false;
    int tma_rank = 0;                         // 5: one box per tile; 2: 2*d/64 boxes per tile
    // K7 (chunked prefill, any group size): always the 5-D one-box-per-tile map
    alignas(64) CUtensorMap ptmap;
    bool has_ptmap = false;
    dbk::UploadBuffer up_pref;
    std::vector<dbk::PrefTile> pref_tiles;
    int64_t last_prefill_flops = 0;
    // cached tile list: the L per-layer launches of one step upload once
    bool pref_valid = false;
    uint64_t pref_epoch = 0;
    std::vector<int64_t> pref_ids;
    std::vector<int32_t> pref_s0, pref_len;
    int32_t pref_n_tiles = 0;
};
