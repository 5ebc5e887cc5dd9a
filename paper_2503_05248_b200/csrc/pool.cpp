// KV pool: page allocator (host source of truth), request table, device block
// tables and the decode / append launches.
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <new>
#include <queue>
#include <unordered_map>
#include <vector>

#include "common.h"
#include "kernels.cuh"
#include "pool.h"

namespace dbk {

thread_local std::string g_err;

void set_error(const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
}

dbk_status fail(dbk_status st, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

dbk_status UploadBuffer::reserve(size_t bytes) {
    if (bytes <= cap) return DBK_OK;
    if (pending) DBK_CUDA(cudaEventSynchronize(done));
    pending = false;
    release();
    size_t c = 4096;
    while (c < bytes) c *= 2;
    const auto t0 = std::chrono::steady_clock::now();
    DBK_CUDA(cudaMallocHost(&host, c));
    DBK_CUDA(cudaMalloc(&dev, c));
    if (!done) DBK_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    cap = c;
    if (std::getenv("DBK_DEBUG_ALLOC"))
        std::fprintf(stderr, "[dbk] upload buffer: %zu bytes in %.1f ms\n", c,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    return DBK_OK;
}

dbk_status UploadBuffer::upload(const void *src, size_t bytes, cudaStream_t s) {
    DBK_TRY(reserve(bytes));
    if (pending) DBK_CUDA(cudaEventSynchronize(done));
    std::memcpy(host, src, bytes);
    DBK_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, s));
    DBK_CUDA(cudaEventRecord(done, s));
    pending = true;
    return DBK_OK;
}

void UploadBuffer::release() {
    if (host) cudaFreeHost(host);
    if (dev) cudaFree(dev);
    host = dev = nullptr;
    cap = 0;
}

// ---------------------------------------------------------------- allocator (R7)
void PageBitmap::init(int64_t cap) {
    words.assign(static_cast<size_t>((cap + 63) / 64), ~0ULL);
    if (cap % 64) words.back() = (1ULL << (cap % 64)) - 1;
    free_count = cap;
    hint = 0;
}
int64_t PageBitmap::take_lowest() {
    for (size_t w = hint; w < words.size(); ++w) {
        if (words[w]) {
            const int b = __builtin_ctzll(words[w]);
            words[w] &= words[w] - 1;
            hint = w;
            --free_count;
            return static_cast<int64_t>(w) * 64 + b;
        }
    }
    return -1;
}
void PageBitmap::give_back(int64_t p) {
    const size_t w = static_cast<size_t>(p / 64);
    words[w] |= 1ULL << (p % 64);
    ++free_count;
    if (w < hint) hint = w;
}

}  // namespace dbk

using namespace dbk;

// K2's tensor map over the whole pool: a 2-D tensor of rows = layers*cap*kv_heads*2*16
// token rows x head_dim elements; one box = 16 rows x 64 elements with the 128-byte swizzle.
static bool make_pool_tmap(dbk_pool *p, bool try5, CUtensorMap *dst, int *rank, uint32_t box_rows = 16) {
    const dbk_pool_config &c = p->cfg;
    const uint64_t tiles = static_cast<uint64_t>(c.layers) * c.cap_pages * c.kv_heads;  // (layer, page, head)
    if (tiles * 2 * c.page_size >= (1ull << 31)) return false;  // int32 TMA coordinates
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
        q != cudaDriverEntryPointSuccess)
        return false;
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    const cuuint32_t halves = static_cast<cuuint32_t>(c.head_dim / 64);
    const cuuint64_t row = static_cast<cuuint64_t>(c.head_dim) * 2;  // one token row, bytes
    // Preferred: ONE 8 KiB box per (page, head) tile -- a 5-D view {64 elements, 16 tokens,
    // d/64 halves, K|V, tile} whose box lands in shared memory as [K|V][half][token][64],
    // i.e. 128-B rows with the token index as the swizzle row (conflict-free ldmatrix).
    if (try5) {
        const cuuint64_t gdim[5] = {64, static_cast<cuuint64_t>(c.page_size), halves, 2, tiles};
        const cuuint64_t gstride[4] = {row, 128, row * c.page_size, row * c.page_size * 2};
        // K7 (prefill) fetches each d-half of K and V separately: box {64, 16, 1, 1, 1}
        const bool split = dst == &p->ptmap;
        const cuuint32_t box[5] = {64, static_cast<cuuint32_t>(c.page_size), split ? 1u : halves, split ? 1u : 2u, 1};
        const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
        if (encode(dst, CU_TENSOR_MAP_DATA_TYPE_UINT16, 5, p->kv, gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
            *rank = 5;
            return true;
        }
        if (dst == &p->ptmap) return false;  // K7 needs the 5-D boxes
    }
    // Fallback: 2-D rows x d, boxes of 16 rows x 64 elements (2 * d/64 boxes per tile).
    const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(c.head_dim), tiles * 2 * c.page_size};
    const cuuint64_t gstride[1] = {row};
    const cuuint32_t box[2] = {64, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(dst, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, p->kv, gdim, gstride, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    *rank = 2;
    return r == CUDA_SUCCESS;
}

// split-K arrival counters of one scratch parity: one per (layer, request slot, kv head), so a
// launch may stream every layer (dbk_decode_step_layers)
static size_t counters_per_parity(const dbk_pool_config *c) {
    return static_cast<size_t>(c->layers) * c->max_requests * c->kv_heads;
}

static bool pool_cfg_ok(const dbk_pool_config *c) {
    if (!c) return false;
    if (c->layers < 1 || c->q_heads < 1 || c->kv_heads < 1 || c->q_heads % c->kv_heads) return false;
    const int g = c->q_heads / c->kv_heads;
    if (g != 1 && g != 2 && g != 4 && g != 8) return false;
    if (c->head_dim != 64 && c->head_dim != 128) return false;
    if (c->page_size != 16 || (c->kv_dtype != 0 && c->kv_dtype != 1)) return false;
    if (c->cap_pages < 1 || c->cap_pages > (1LL << 31) - 1 || c->max_requests < 1 ||
        c->max_pages_per_req < 1)
        return false;
    // generator key: head index in 12 bits (synth/hashgen.py)
    if (c->kv_head_offset < 0 || (c->kv_head_offset + c->kv_heads) * g > 4096) return false;
    return true;
}

extern "C" {

const char *dbk_last_error(void) { return dbk::g_err.c_str(); }
const char *dbk_version(void) { return "dbk 0.1 (sm_100a)"; }

size_t dbk_kv_pool_bytes(const dbk_pool_config *c) {
    if (!pool_cfg_ok(c)) return 0;
    return static_cast<size_t>(c->layers) * static_cast<size_t>(c->cap_pages) * c->kv_heads * 2 *
           c->page_size * c->head_dim * 2;
}

dbk_status dbk_kv_pool_create(const dbk_pool_config *cfg, void *kv_mem, size_t kv_bytes, dbk_pool **out) {
    if (!out) return fail(DBK_EINVAL, "pool_create: null output");
    if (!pool_cfg_ok(cfg))
        return fail(DBK_EINVAL, "pool_create: invalid config (heads, head_dim in {64,128}, page_size 16, dtype)");
    const size_t need = dbk_kv_pool_bytes(cfg);
    if (!kv_mem || kv_bytes < need || (reinterpret_cast<uintptr_t>(kv_mem) & 255))
        return fail(DBK_EINVAL, "pool_create: kv_mem must be 256-B aligned and >= %zu bytes", need);
    DBK_CUDA(cudaSetDevice(cfg->device));
    dbk_pool *p = new (std::nothrow) dbk_pool();
    if (!p) return fail(DBK_EINVAL, "out of host memory");
    p->cfg = *cfg;
    p->kv = static_cast<uint8_t *>(kv_mem);
    p->kv_bytes = kv_bytes;
    p->elt = 2;
    p->tile_bytes = 2LL * cfg->page_size * cfg->head_dim * p->elt;
    p->page_stride = p->tile_bytes * cfg->kv_heads;
    p->layer_stride = p->page_stride * cfg->cap_pages;
    p->pages.init(cfg->cap_pages);
    for (int s = 0; s < cfg->max_requests; ++s) p->free_slots.push(s);
    const size_t bt_n = static_cast<size_t>(cfg->max_requests) * cfg->max_pages_per_req;
    auto cleanup = [&](dbk_status st) {
        dbk_kv_pool_destroy(p);
        return st;
    };
    if (cudaMalloc(&p->d_bt, bt_n * sizeof(int32_t)) != cudaSuccess ||
        cudaMemset(p->d_bt, 0xFF, bt_n * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&p->d_counters, 2 * counters_per_parity(cfg) * sizeof(int32_t)) != cudaSuccess ||
        cudaMemset(p->d_counters, 0, 2 * counters_per_parity(cfg) * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&p->d_stats, 128 + 64) != cudaSuccess ||
        cudaMemset(p->d_stats, 0, 128 + 64) != cudaSuccess ||
        cudaMallocHost(&p->h_stats, sizeof(dbk_stats)) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess)
        return cleanup(fail(DBK_ECUDA, "pool_create: %s", cudaGetErrorString(cudaGetLastError())));
    p->d_stats_done = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(p->d_stats) + 128);
    p->d_task_counter = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(p->d_stats) + 160);
    p->d_done_seq = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(p->d_stats) + 176);
    p->host_bt.assign(bt_n, -1);
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, cfg->device);
    p->num_sms = dev_sms;
    if (const char *e = std::getenv("DBK_DECODE_SMS")) {  // measurement: attention on a subset of the SMs
        const int v = std::atoi(e);
        if (v >= 1 && v < dev_sms) p->num_sms = v;
    }
    const int group = cfg->q_heads / cfg->kv_heads;
    const char *cc = std::getenv("DBK_GQA_CUDA_CORE");  // 1: force K1 for GQA (comparison runs)
    const char *t2 = std::getenv("DBK_GQA_TMA2");  // 1: force the 2-D boxes (comparison runs)
    if (group >= 2 && !(cc && cc[0] == '1'))
        p->has_tmap = make_pool_tmap(p, !(t2 && t2[0] == '1'), &p->tmap, &p->tma_rank);
    if (p->has_tmap) {  // 4-row boxes for partly filled last pages (DBK_GQA_HALF=0: off, comparison runs)
        const char *hb = std::getenv("DBK_GQA_HALF");
        int r2 = 0;
        p->has_tmap_half = !(hb && hb[0] == '0') && make_pool_tmap(p, false, &p->tmap_half, &r2, 4);
    }
    int prank = 0;
    p->has_ptmap = make_pool_tmap(p, true, &p->ptmap, &prank);
    p->ctas_per_sm = p->has_tmap ? decode_gqa_ctas_per_sm(cfg->kv_dtype, cfg->head_dim, group)
                                 : decode_ctas_per_sm(cfg->kv_dtype, cfg->head_dim, group);
    if (const char *e = std::getenv("DBK_NO_PDL")) p->pdl_enabled = !(e[0] == '1');  // A/B runs
    if (const char *e = std::getenv("DBK_WS_BUDGET_MB")) {  // tuning override: layers per launch
        const long long v = std::atoll(e);
        if (v >= 1) p->ws_budget_bytes = v << 20;
    }
    if (const char *e = std::getenv("DBK_LAYERS_PER_LAUNCH")) {  // test / tuning cap on layers per launch
        const long long v = std::atoll(e);
        if (v >= 1) p->max_layers_per_launch = static_cast<int32_t>(v);
    }
    if (const char *e = std::getenv("DBK_TRACE_TASKS")) {  // measurement: task timeline records
        const long long v = std::atoll(e);
        if (v > 0 && v <= (1 << 24)) {
            const size_t bytes = static_cast<size_t>(v + 1) * 32;
            if (cudaMalloc(&p->d_trace, bytes) != cudaSuccess || cudaMemset(p->d_trace, 0, bytes) != cudaSuccess)
                return cleanup(fail(DBK_ECUDA, "pool_create: trace buffer"));
            p->trace_cap = static_cast<int32_t>(v);
        }
    }
    if (const char *e = std::getenv("DBK_TASKS_PER_WARP")) {  // tuning override
        const long long v = std::atoll(e);
        if (v >= 1 && v <= 16) p->tasks_per_warp = v;
    }
    if (const char *e = std::getenv("DBK_CHUNK_PAGES")) {  // tuning override (multiple of 4, <= 64)
        const long long v = std::atoll(e);
        if (v >= 4 && v <= 64 && v % 4 == 0) p->force_chunk_pages = v;
    }
    *out = p;
    return DBK_OK;
}

dbk_status dbk_kv_pool_destroy(dbk_pool *p) {
    if (!p) return DBK_OK;
    cudaSetDevice(p->cfg.device);
    cudaDeviceSynchronize();
    if (p->d_bt) cudaFree(p->d_bt);
    if (p->d_trace) cudaFree(p->d_trace);
    if (p->d_counters) cudaFree(p->d_counters);
    if (p->d_stats) cudaFree(p->d_stats);
    if (p->h_stats) cudaFreeHost(p->h_stats);
    if (p->d_ws_o) cudaFree(p->d_ws_o);
    if (p->d_ws_ml) cudaFree(p->d_ws_ml);
    p->up_delta.release();
    p->up_append.release();
    p->up_meta.release();
    p->up_rows.release();
    p->up_pref.release();
    if (p->up_pref.done) cudaEventDestroy(p->up_pref.done);
    if (p->up_delta.done) cudaEventDestroy(p->up_delta.done);
    if (p->up_append.done) cudaEventDestroy(p->up_append.done);
    if (p->up_meta.done) cudaEventDestroy(p->up_meta.done);
    if (p->up_rows.done) cudaEventDestroy(p->up_rows.done);
    delete p;
    return DBK_OK;
}

dbk_status dbk_request_begin(dbk_pool *p, int64_t id, int32_t l_in, int32_t l_out) {
    if (!p) return fail(DBK_EINVAL, "null pool");
    if (id < 0 || l_in < 1 || l_out < 1) return fail(DBK_EINVAL, "request_begin: need id >= 0, l_in >= 1, l_out >= 1");
    if (p->reqs.count(id) || p->swapped.count(id))
        return fail(DBK_EINVAL, "request %lld already active", static_cast<long long>(id));
    const int64_t P = p->cfg.page_size;
    const int64_t need = (static_cast<int64_t>(l_in) + l_out + P - 1) / P;
    if (need > p->cfg.cap_pages || need > p->cfg.max_pages_per_req)
        return fail(DBK_EFATAL, "request %lld needs %lld pages alone (cap %lld, row %d)", static_cast<long long>(id),
                    static_cast<long long>(need), static_cast<long long>(p->cfg.cap_pages), p->cfg.max_pages_per_req);
    if (p->free_slots.empty()) return fail(DBK_EINVAL, "no free request slot (max_requests = %d)", p->cfg.max_requests);
    Request r;
    r.id = id;
    r.l_in = l_in;
    r.l_out = l_out;
    r.ctx = 0;
    r.slot = p->free_slots.top();
    p->free_slots.pop();
    p->reqs.emplace(id, std::move(r));
    ++p->epoch;
    return DBK_OK;
}

}  // extern "C"

namespace dbk {
dbk_status flush_deltas(dbk_pool *p, cudaStream_t s) {
    if (p->pending.empty()) return DBK_OK;
    // The apply kernel writes deltas in parallel, so keep only the LAST delta per entry
    // (a slot released and reused before a flush has a clear followed by a new page).
    {
        std::unordered_map<int64_t, size_t> last;
        last.reserve(p->pending.size() * 2);
        for (size_t k = 0; k < p->pending.size(); ++k)
            last[static_cast<int64_t>(p->pending[k].slot) * p->cfg.max_pages_per_req + p->pending[k].idx] = k;
        if (last.size() != p->pending.size()) {
            std::vector<BtDelta> uniq;
            uniq.reserve(last.size());
            for (size_t k = 0; k < p->pending.size(); ++k)
                if (last[static_cast<int64_t>(p->pending[k].slot) * p->cfg.max_pages_per_req + p->pending[k].idx] == k)
                    uniq.push_back(p->pending[k]);
            p->pending.swap(uniq);
        }
    }
    DBK_TRY(p->up_delta.upload(p->pending.data(), p->pending.size() * sizeof(BtDelta), s));
    DBK_CUDA(launch_bt_apply(p->d_bt, p->cfg.max_pages_per_req, static_cast<const BtDelta *>(p->up_delta.dev),
                             static_cast<int32_t>(p->pending.size()), s));
    ++p->n_launches;
    p->pending.clear();
    return DBK_OK;
}
// Validates and performs the bookkeeping of an append (pages lowest-free-first, all-or-nothing,
// R7/R8), flushes the block-table deltas and uploads the job list; no KV is written yet.
// true when some id appears twice in ids[0, n) (list calls are all-or-nothing and name each
// request once)
bool has_duplicate_ids(int32_t n, const int64_t *ids) {
    std::vector<int64_t> sorted(ids, ids + n);
    std::sort(sorted.begin(), sorted.end());
    return std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end();
}

dbk_status append_plan(dbk_pool *p, int32_t n, const int64_t *ids, const int32_t *n_tok, bool explicit_rows,
                       cudaStream_t s, bool upload_jobs) {
    if (!p) return fail(DBK_EINVAL, "null pool");
    if (n < 0 || (n > 0 && (!ids || !n_tok))) return fail(DBK_EINVAL, "append_tokens: bad arrays");
    const int64_t P = p->cfg.page_size;
    // validate and count pages first: all-or-nothing (R8)
    std::vector<Request *> rs(n);
    int64_t need = 0;
    for (int i = 0; i < n; ++i) {
        auto it = p->reqs.find(ids[i]);
        if (it == p->reqs.end()) return fail(DBK_ENOENT, "append_tokens: unknown request %lld", static_cast<long long>(ids[i]));
        Request &r = it->second;
        if (n_tok[i] < 0) return fail(DBK_EINVAL, "append_tokens: negative token count");
        const int64_t nc = static_cast<int64_t>(r.ctx) + n_tok[i];
        const int64_t np = (nc + P - 1) / P;
        if (np > p->cfg.max_pages_per_req) return fail(DBK_EINVAL, "append_tokens: request %lld exceeds max_pages_per_req", static_cast<long long>(ids[i]));
        need += np - static_cast<int64_t>(r.pages.size());
        rs[i] = &r;
    }
    if (has_duplicate_ids(n, ids)) return fail(DBK_EINVAL, "append_tokens: duplicate request id in one call");
    if (need > p->pages.free_count)
        return fail(DBK_ECAP, "append_tokens: needs %lld pages, %lld free", static_cast<long long>(need),
                    static_cast<long long>(p->pages.free_count));
    DBK_CUDA(cudaSetDevice(p->cfg.device));
    p->jobs.clear();
    int32_t src_row = 0;
    for (int i = 0; i < n; ++i) {
        Request &r = *rs[i];
        const int32_t c0 = r.ctx, c1 = r.ctx + n_tok[i];
        while (static_cast<int64_t>(r.pages.size()) * P < c1) {
            const int64_t pg = p->pages.take_lowest();
            const int32_t idx = static_cast<int32_t>(r.pages.size());
            r.pages.push_back(static_cast<int32_t>(pg));
            p->host_bt[static_cast<size_t>(r.slot) * p->cfg.max_pages_per_req + idx] = static_cast<int32_t>(pg);
            p->pending.push_back({r.slot, idx, static_cast<int32_t>(pg)});
        }
        for (int32_t pos = c0; pos < c1;) {
            const int32_t in_page = static_cast<int32_t>(P - pos % P);
            const int32_t cnt = std::min(in_page, c1 - pos);
            AppendJob j;
            j.req_id = r.id;
            j.pos0 = pos;
            j.ntok = cnt;
            j.phys = r.pages[pos / P];
            j.src_row = explicit_rows ? src_row + (pos - c0) : -1;
            p->jobs.push_back(j);
            pos += cnt;
        }
        src_row += n_tok[i];
        r.ctx = c1;
    }
    ++p->epoch;
    DBK_TRY(flush_deltas(p, s));
    if (!upload_jobs) {
        p->jobs.clear();  // reserve only: nothing for append_launch to write
        return DBK_OK;
    }
    if (!p->jobs.empty())
        DBK_TRY(p->up_append.upload(p->jobs.data(), p->jobs.size() * sizeof(AppendJob), s));
    return DBK_OK;
}

// Writes layers [layer0, layer0 + nl) of the jobs planned by the last append_plan (whose job
// list is still in up_append's device buffer).
dbk_status append_launch(dbk_pool *p, const void *k, const void *v, uint64_t seed, int32_t layer0, int32_t nl,
                         cudaStream_t s, int32_t src_layer_rows) {
    if (p->jobs.empty() || nl <= 0) return DBK_OK;
    AppendParams ap;
    ap.kv = p->kv;
    ap.layer_stride = p->layer_stride;
    ap.page_stride = p->page_stride;
    ap.tile_bytes = p->tile_bytes;
    ap.jobs = static_cast<const AppendJob *>(p->up_append.dev);
    ap.n_jobs = static_cast<int32_t>(p->jobs.size());
    ap.layers = p->cfg.layers;
    ap.kv_heads = p->cfg.kv_heads;
    ap.k_src = k;
    ap.v_src = v;
    ap.seed = seed;
    ap.head0 = p->cfg.kv_head_offset;
    ap.layer0 = layer0;
    ap.n_launch_layers = nl;
    ap.src_layer_rows = src_layer_rows;
    DBK_CUDA(launch_append(ap, p->cfg.kv_dtype, p->cfg.head_dim, s));
    ++p->n_launches;
    return DBK_OK;
}

}  // namespace dbk

extern "C" {

dbk_status dbk_append_tokens(dbk_pool *p, int32_t n, const int64_t *ids, const int32_t *n_tok,
                             const void *k, const void *v, uint64_t seed, void *stream) {
    if (!p) return fail(DBK_EINVAL, "null pool");
    if ((k == nullptr) != (v == nullptr)) return fail(DBK_EINVAL, "append_tokens: k and v must both be given or both NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DBK_TRY(dbk::append_plan(p, n, ids, n_tok, k != nullptr, s));
    return dbk::append_launch(p, k, v, seed, 0, p->cfg.layers, s);
}

dbk_status dbk_reserve_tokens(dbk_pool *p, int32_t n, const int64_t *ids, const int32_t *n_tok, void *stream) {
    if (!p) return fail(DBK_EINVAL, "null pool");
    return dbk::append_plan(p, n, ids, n_tok, false, static_cast<cudaStream_t>(stream), false);
}

dbk_status dbk_release(dbk_pool *p, int32_t n, const int64_t *ids) {
    if (!p) return fail(DBK_EINVAL, "null pool");
    if (n < 0 || (n > 0 && !ids)) return fail(DBK_EINVAL, "release: bad arrays");
    // all-or-nothing like append_tokens: every id known (resident or swapped out), none twice
    for (int i = 0; i < n; ++i)
        if (!p->swapped.count(ids[i]) && !p->reqs.count(ids[i]))
            return fail(DBK_ENOENT, "release: unknown request %lld", static_cast<long long>(ids[i]));
    if (dbk::has_duplicate_ids(n, ids)) return fail(DBK_EINVAL, "release: duplicate request id in one call");
    for (int i = 0; i < n; ++i) {
        auto sw = p->swapped.find(ids[i]);
        if (sw != p->swapped.end()) {  // a swapped-out request: its swap pages go back
            for (int32_t h : sw->second.swap_pages) p->swap_pages.give_back(h);
            p->swapped.erase(sw);
            continue;
        }
        auto it = p->reqs.find(ids[i]);
        if (it == p->reqs.end()) return fail(DBK_ENOENT, "release: unknown request %lld", static_cast<long long>(ids[i]));
        Request &r = it->second;
        for (size_t x = 0; x < r.pages.size(); ++x) {
            p->pages.give_back(r.pages[x]);
            p->host_bt[static_cast<size_t>(r.slot) * p->cfg.max_pages_per_req + x] = -1;
            p->pending.push_back({r.slot, static_cast<int32_t>(x), -1});
        }
        p->free_slots.push(r.slot);
        p->reqs.erase(it);
    }
    ++p->epoch;
    return DBK_OK;
}

dbk_status dbk_swap_space_attach(dbk_pool *p, void *host_mem, size_t bytes, int64_t *swap_pages_out) {
    if (!p) return fail(DBK_EINVAL, "null pool");
    if (!p->swapped.empty()) return fail(DBK_EINVAL, "swap_space_attach: requests are swapped out");
    const size_t per_page = static_cast<size_t>(p->cfg.layers) * p->page_stride;
    const int64_t n = host_mem ? static_cast<int64_t>(bytes / per_page) : 0;
    if (host_mem) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, host_mem) != cudaSuccess || a.type != cudaMemoryTypeHost) {
            cudaGetLastError();
            return fail(DBK_EINVAL, "swap_space_attach: host_mem must be pinned host memory (cudaHostAlloc)");
        }
        if (n < 1) return fail(DBK_EINVAL, "swap_space_attach: %zu bytes hold no page (%zu B per page)", bytes, per_page);
    }
    p->swap_host = static_cast<uint8_t *>(host_mem);
    p->swap_cap = n;
    p->swap_pages.init(n);
    if (swap_pages_out) *swap_pages_out = n;
    return DBK_OK;
}

dbk_status dbk_swap_usage(dbk_pool *p, int64_t *used, int64_t *free_pages, int64_t *bytes_moved) {
    if (!p) return fail(DBK_EINVAL, "null pool");
    if (used) *used = p->swap_cap - p->swap_pages.free_count;
    if (free_pages) *free_pages = p->swap_pages.free_count;
    if (bytes_moved) *bytes_moved = p->swap_bytes_moved;
    return DBK_OK;
}

}  // extern "C"

namespace dbk {
// Copy engine transfers of one request's pages: maximal runs where the device page and the
// swap page both advance by one become ONE 2-D copy (rows = layers).
dbk_status swap_copy(dbk_pool *p, const std::vector<int32_t> &dev_pages, const std::vector<int32_t> &host_pages,
                     bool to_host, cudaStream_t s) {
    const size_t ps = static_cast<size_t>(p->page_stride);
    const size_t hpitch = static_cast<size_t>(p->swap_cap) * ps;
    const size_t dpitch = static_cast<size_t>(p->layer_stride);
    size_t k = 0;
    while (k < dev_pages.size()) {
        size_t run = 1;
        while (k + run < dev_pages.size() && dev_pages[k + run] == dev_pages[k] + static_cast<int32_t>(run) &&
               host_pages[k + run] == host_pages[k] + static_cast<int32_t>(run))
            ++run;
        uint8_t *dev = p->kv + static_cast<size_t>(dev_pages[k]) * ps;
        uint8_t *host = p->swap_host + static_cast<size_t>(host_pages[k]) * ps;
        if (to_host)
            DBK_CUDA(cudaMemcpy2DAsync(host, hpitch, dev, dpitch, run * ps, p->cfg.layers, cudaMemcpyDeviceToHost, s));
        else
            DBK_CUDA(cudaMemcpy2DAsync(dev, dpitch, host, hpitch, run * ps, p->cfg.layers, cudaMemcpyHostToDevice, s));
        p->swap_bytes_moved += static_cast<int64_t>(run * ps) * p->cfg.layers;
        k += run;
    }
    return DBK_OK;
}
}  // namespace dbk

extern "C" {

dbk_status dbk_swap_out(dbk_pool *p, int32_t n, const int64_t *ids, void *stream) {
    if (!p) return fail(DBK_EINVAL, "null pool");
    if (n < 0 || (n > 0 && !ids)) return fail(DBK_EINVAL, "swap_out: bad arrays");
    if (!p->swap_host) return fail(DBK_EINVAL, "swap_out: no swap space attached");
    if (dbk::has_duplicate_ids(n, ids)) return fail(DBK_EINVAL, "swap_out: duplicate request id in one call");
    int64_t need = 0;
    for (int i = 0; i < n; ++i) {
        auto it = p->reqs.find(ids[i]);
        if (it == p->reqs.end()) return fail(DBK_ENOENT, "swap_out: unknown request %lld", static_cast<long long>(ids[i]));
        need += static_cast<int64_t>(it->second.pages.size());
    }
    if (need > p->swap_pages.free_count)
        return fail(DBK_ECAP, "swap_out: needs %lld swap pages, %lld free", static_cast<long long>(need),
                    static_cast<long long>(p->swap_pages.free_count));
    DBK_CUDA(cudaSetDevice(p->cfg.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (int i = 0; i < n; ++i) {
        auto it = p->reqs.find(ids[i]);
        Request &r = it->second;
        SwappedRequest sr;
        sr.l_in = r.l_in;
        sr.l_out = r.l_out;
        sr.ctx = r.ctx;
        for (size_t x = 0; x < r.pages.size(); ++x) sr.swap_pages.push_back(static_cast<int32_t>(p->swap_pages.take_lowest()));
        // stream order: the D2H copies precede any later write to the released pages
        DBK_TRY(swap_copy(p, r.pages, sr.swap_pages, true, s));
        for (size_t x = 0; x < r.pages.size(); ++x) {
            p->pages.give_back(r.pages[x]);
            p->host_bt[static_cast<size_t>(r.slot) * p->cfg.max_pages_per_req + x] = -1;
            p->pending.push_back({r.slot, static_cast<int32_t>(x), -1});
        }
        p->free_slots.push(r.slot);
        p->swapped.emplace(ids[i], std::move(sr));
        p->reqs.erase(it);
    }
    ++p->epoch;
    return DBK_OK;
}

dbk_status dbk_swap_in(dbk_pool *p, int32_t n, const int64_t *ids, void *stream) {
    if (!p) return fail(DBK_EINVAL, "null pool");
    if (n < 0 || (n > 0 && !ids)) return fail(DBK_EINVAL, "swap_in: bad arrays");
    if (dbk::has_duplicate_ids(n, ids)) return fail(DBK_EINVAL, "swap_in: duplicate request id in one call");
    int64_t need = 0;
    for (int i = 0; i < n; ++i) {
        auto it = p->swapped.find(ids[i]);
        if (it == p->swapped.end()) return fail(DBK_ENOENT, "swap_in: request %lld is not swapped out", static_cast<long long>(ids[i]));
        need += static_cast<int64_t>(it->second.swap_pages.size());
    }
    if (need > p->pages.free_count)
        return fail(DBK_ECAP, "swap_in: needs %lld pages, %lld free", static_cast<long long>(need),
                    static_cast<long long>(p->pages.free_count));
    if (static_cast<size_t>(n) > p->free_slots.size()) return fail(DBK_EINVAL, "swap_in: no free request slot");
    DBK_CUDA(cudaSetDevice(p->cfg.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (int i = 0; i < n; ++i) {
        auto it = p->swapped.find(ids[i]);
        SwappedRequest &sr = it->second;
        Request r;
        r.id = ids[i];
        r.l_in = sr.l_in;
        r.l_out = sr.l_out;
        r.ctx = sr.ctx;
        r.slot = p->free_slots.top();
        p->free_slots.pop();
        for (size_t x = 0; x < sr.swap_pages.size(); ++x) {  // lowest-free-first, like an append (R7)
            const int32_t pg = static_cast<int32_t>(p->pages.take_lowest());
            r.pages.push_back(pg);
            p->host_bt[static_cast<size_t>(r.slot) * p->cfg.max_pages_per_req + x] = pg;
            p->pending.push_back({r.slot, static_cast<int32_t>(x), pg});
        }
        DBK_TRY(swap_copy(p, r.pages, sr.swap_pages, false, s));
        for (int32_t h : sr.swap_pages) p->swap_pages.give_back(h);
        p->reqs.emplace(r.id, std::move(r));
        p->swapped.erase(it);
    }
    ++p->epoch;
    DBK_TRY(flush_deltas(p, s));
    return DBK_OK;
}

dbk_status dbk_request_info(dbk_pool *p, int64_t id, int32_t *ctx, int32_t *n_pages, int32_t *slot,
                            int32_t *pages_out, int32_t pages_cap) {
    if (!p) return fail(DBK_EINVAL, "null pool");
    auto it = p->reqs.find(id);
    if (it == p->reqs.end()) return fail(DBK_ENOENT, "request_info: unknown request %lld", static_cast<long long>(id));
    const Request &r = it->second;
    if (ctx) *ctx = r.ctx;
    if (n_pages) *n_pages = static_cast<int32_t>(r.pages.size());
    if (slot) *slot = r.slot;
    if (pages_out)
        for (int32_t x = 0; x < pages_cap && x < static_cast<int32_t>(r.pages.size()); ++x) pages_out[x] = r.pages[x];
    return DBK_OK;
}

dbk_status dbk_pool_usage(dbk_pool *p, int64_t *used, int64_t *free_pages) {
    if (!p) return fail(DBK_EINVAL, "null pool");
    if (used) *used = p->cfg.cap_pages - p->pages.free_count;
    if (free_pages) *free_pages = p->pages.free_count;
    return DBK_OK;
}

dbk_status dbk_pool_get_info(dbk_pool *p, dbk_pool_info *o) {
    if (!p || !o) return fail(DBK_EINVAL, "pool_get_info: null argument");
    o->decode_path = p->has_tmap ? 2 : 1;
    o->ctas_per_sm = p->ctas_per_sm;
    o->chunk_pages = p->meta_chunk_pages;
    o->work_items = p->meta_items;
    o->launches = p->n_launches;
    o->last_decode_bytes = p->last_decode_bytes;
    o->tma_rank = p->has_tmap ? p->tma_rank : 0;
    o->_reserved = 0;
    return DBK_OK;
}

dbk_status dbk_block_table_d2h(dbk_pool *p, int32_t *host_out, void *stream) {
    if (!p || !host_out) return fail(DBK_EINVAL, "block_table_d2h: null argument");
    DBK_CUDA(cudaSetDevice(p->cfg.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DBK_TRY(flush_deltas(p, s));
    const size_t bytes = static_cast<size_t>(p->cfg.max_requests) * p->cfg.max_pages_per_req * sizeof(int32_t);
    DBK_CUDA(cudaMemcpyAsync(host_out, p->d_bt, bytes, cudaMemcpyDeviceToHost, s));
    DBK_CUDA(cudaStreamSynchronize(s));
    return DBK_OK;
}

}  // extern "C"

namespace dbk {

// Build (or reuse) the device metadata of a decode batch: per-request ReqMeta and
// the split-K work list.  Reused while the batch and the pool state are unchanged
// (the L per-layer launches of one step upload once).
dbk_status prepare_batch(dbk_pool *p, int32_t n, const int64_t *ids, cudaStream_t s, int32_t layers_hint) {
    if (p->meta_valid && p->meta_epoch == p->epoch && p->meta_ids.size() == static_cast<size_t>(n) &&
        p->meta_layers_hint == layers_hint && std::equal(p->meta_ids.begin(), p->meta_ids.end(), ids))
        return DBK_OK;
    const int64_t P = p->cfg.page_size;
    p->meta_valid = false;  // rebuilt below; a rejected batch leaves no half-built cache behind
    p->meta_req.resize(n);
    int64_t total_pages = 0;
    // a request decodes one token per step: a batch naming it twice is malformed (K4 would count
    // it twice); its block-table slot is unique, so a slot bitmap finds repeats in O(n)
    std::vector<uint8_t> &seen = p->slot_seen;
    seen.assign(static_cast<size_t>(p->cfg.max_requests), 0);
    for (int i = 0; i < n; ++i) {
        auto it = p->reqs.find(ids[i]);
        if (it == p->reqs.end()) return fail(DBK_ENOENT, "decode_step: unknown request %lld", static_cast<long long>(ids[i]));
        const Request &r = it->second;
        if (r.ctx < 1) return fail(DBK_EINVAL, "decode_step: request %lld holds no tokens", static_cast<long long>(ids[i]));
        if (seen[r.slot]++) return fail(DBK_EINVAL, "decode_step: request %lld appears twice in the batch", static_cast<long long>(ids[i]));
        ReqMeta &m = p->meta_req[i];
        m.req_id = r.id;
        m.slot = r.slot;
        m.ctx = r.ctx;
        m.l_in = r.l_in;
        m.l_out = r.l_out;
        total_pages += (r.ctx + P - 1) / P;
    }
    // chunk size (pages per warp task, 4..32): ~tasks_per_warp (3) tasks per resident warp of
    // ONE launch so the dynamic queue balances, but not below 12 pages while every warp still
    // gets a task: each task pays fixed costs (metadata, q, split-K partial + merge) -- measured
    // on the per-GPU shards of 70B KV-head TP (profiles/r01_tune_chunks.txt): 12 pages beat 6
    // by 13 % at TP8, 15 beat 12 by 4 % at TP4.  A launch streams layers_hint layers, so its
    // queue holds that many times the work: multi-layer launches take 32-page chunks, where
    // most requests are one task and need no split-K (profiles/r02_tune_chunks_ml.txt: TP8
    // 5.57 -> 6.66 TB/s from 12 to 32 pages)
    const int64_t warps = static_cast<int64_t>(p->num_sms) * p->ctas_per_sm * 4;
    const int64_t tpw = p->tasks_per_warp;
    const int64_t work = total_pages * p->cfg.kv_heads * std::max(layers_hint, 1);
    int64_t cp = (work + tpw * warps - 1) / (tpw * warps);
    cp = std::max<int64_t>(cp, std::min<int64_t>(12, (work + warps - 1) / warps));
    cp = std::max<int64_t>(4, std::min<int64_t>(p->max_chunk_pages, cp));
    if (p->force_chunk_pages > 0) cp = std::min<int64_t>(p->force_chunk_pages, p->max_chunk_pages);
    p->meta_work.clear();
    int32_t base = 0, ws_rows = 0;
    for (int i = 0; i < n; ++i) {
        ReqMeta &m = p->meta_req[i];
        const int32_t pages = static_cast<int32_t>((m.ctx + P - 1) / P);
        const int32_t nc = static_cast<int32_t>((pages + cp - 1) / cp);
        m.chunk_base = nc > 1 ? ws_rows : 0;  // split-K rows only for requests that are split
        m.nchunks = nc;
        for (int32_t c = 0; c < nc; ++c) p->meta_work.push_back(make_int2(i, c));
        base += nc;
        if (nc > 1) ws_rows += nc;
    }
    // longest task first: the dynamic queue then ends on short tasks (small tail)
    std::stable_sort(p->meta_work.begin(), p->meta_work.end(), [&](const int2 &a, const int2 &b) {
        const int64_t pa = std::min<int64_t>(cp, (p->meta_req[a.x].ctx + P - 1) / P - a.y * cp);
        const int64_t pb = std::min<int64_t>(cp, (p->meta_req[b.x].ctx + P - 1) / P - b.y * cp);
        return pa > pb;
    });
    p->meta_items = base;
    p->meta_ws_rows = ws_rows;
    p->meta_chunk_pages = static_cast<int32_t>(cp);
    // blob: ReqMeta[n] | ItemMeta[items]; the kernels take each item's page ids from the device
    // block table (row `slot`), which flush_deltas brings up to date before every launch
    const size_t rb = sizeof(ReqMeta) * static_cast<size_t>(n);
    const size_t ib = sizeof(ItemMeta) * static_cast<size_t>(base);
    p->meta_blob.resize(rb + ib);
    if (rb) std::memcpy(p->meta_blob.data(), p->meta_req.data(), rb);
    ItemMeta *im = reinterpret_cast<ItemMeta *>(p->meta_blob.data() + rb);
    for (int32_t w = 0; w < base; ++w) {
        const int2 wk = p->meta_work[w];
        const ReqMeta &m = p->meta_req[wk.x];
        const int32_t pages = static_cast<int32_t>((m.ctx + P - 1) / P);
        ItemMeta it;
        it.i = wk.x;
        it.c = wk.y;
        it.pg0 = static_cast<int32_t>(wk.y * cp);
        it.n = std::min<int32_t>(static_cast<int32_t>(cp), pages - it.pg0);
        it.ctx = m.ctx;
        it.chunk_base = m.chunk_base;
        it.nchunks = m.nchunks;
        it.slot = m.slot;
        im[w] = it;
    }
    DBK_TRY(p->up_meta.upload(p->meta_blob.data(), p->meta_blob.size(), s));
    p->d_req = static_cast<const ReqMeta *>(p->up_meta.dev);
    p->d_items = reinterpret_cast<const ItemMeta *>(static_cast<const uint8_t *>(p->up_meta.dev) + rb);
    p->meta_layers_hint = layers_hint;
    p->meta_ids.assign(ids, ids + n);
    p->meta_epoch = p->epoch;
    p->meta_valid = true;
    return DBK_OK;
}

int64_t decode_bytes(const dbk_pool *p, int out_dtype) {
    // algorithmic bytes of one decode launch
    const int64_t P = p->cfg.page_size, d = p->cfg.head_dim;
    int64_t ctx_sum = 0, pages = 0;
    for (const ReqMeta &m : p->meta_req) {
        ctx_sum += m.ctx;
        pages += (m.ctx + P - 1) / P;
    }
    const int64_t n = static_cast<int64_t>(p->meta_req.size());
    const int64_t eo = out_dtype == 2 ? 4 : 2;
    return ctx_sum * 2 * p->cfg.kv_heads * d * 2 + n * p->cfg.q_heads * d * 2 + n * p->cfg.q_heads * d * eo + pages * 4;
}

}  // namespace dbk

namespace dbk {

// Split-K workspace rows (of q_heads x (D fp32 + (m, l))) that fit the budget, capped by what the
// pool could ever use (every layer of the largest batch split into 4-page chunks).
static size_t ws_budget_rows(const dbk_pool *p) {
    const size_t row = static_cast<size_t>(p->cfg.head_dim) * sizeof(float) + sizeof(float2);
    const size_t most = static_cast<size_t>(p->cfg.layers) * p->cfg.max_requests *
                        ((p->cfg.max_pages_per_req + 3) / 4) * p->cfg.q_heads;
    return std::min(most, static_cast<size_t>(p->ws_budget_bytes) / row);
}

// Split-K workspace for nl layers of the prepared batch (two scratch parities).  Allocated once
// at the budget (never grown in steady state: a reallocation synchronises the device and, with
// the pool holding nearly all HBM, took ~0.4 s inside a timed step); the layers per launch
// adapt to it instead.
static dbk_status ensure_ws(dbk_pool *p, int32_t nl, cudaStream_t s) {
    const size_t need = static_cast<size_t>(std::max(p->meta_ws_rows, 1)) * nl * p->cfg.q_heads;
    if (need <= p->ws_cap) return DBK_OK;
    const size_t c = std::max<size_t>(need, ws_budget_rows(p));
    const auto t0 = std::chrono::steady_clock::now();
    DBK_CUDA(cudaStreamSynchronize(s));
    if (p->d_ws_o) cudaFree(p->d_ws_o);
    if (p->d_ws_ml) cudaFree(p->d_ws_ml);
    p->d_ws_o = nullptr;
    p->d_ws_ml = nullptr;
    p->ws_cap = 0;
    DBK_CUDA(cudaMalloc(&p->d_ws_o, 2 * c * p->cfg.head_dim * sizeof(float)));  // two parities
    DBK_CUDA(cudaMalloc(&p->d_ws_ml, 2 * c * sizeof(float2)));
    p->ws_cap = c;
    if (std::getenv("DBK_DEBUG_ALLOC"))
        std::fprintf(stderr, "[dbk] split-K workspace: %zu rows x 2 parities (%.1f MB) in %.1f ms\n", c,
                     2.0 * c * (p->cfg.head_dim * 4 + 8) / 1e6,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    return DBK_OK;
}

// One persistent launch over layers [layer0, layer0 + nl) of the prepared batch.
static dbk_status decode_launch(dbk_pool *p, int32_t n, int32_t layer0, int32_t nl, const void *q, int64_t q_ls,
                                void *out, int64_t o_ls, int32_t out_dtype, bool stats, int chain, cudaStream_t s) {
    DBK_TRY(ensure_ws(p, nl, s));
    DecodeParams dp;
    dp.kv_layer = p->kv + static_cast<size_t>(layer0) * p->layer_stride;
    dp.page_stride = p->page_stride;
    dp.block_table = p->d_bt;
    dp.bt_stride = p->cfg.max_pages_per_req;
    dp.n = n;
    dp.req = p->d_req;
    dp.items = p->d_items;
    dp.n_items = p->meta_items;
    dp.chunk_pages = p->meta_chunk_pages;
    dp.q = q;
    dp.out = out;
    dp.out_dtype = out_dtype;
    dp.q_heads = p->cfg.q_heads;
    dp.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(p->cfg.head_dim)));
    // consecutive launches alternate two copies of their scratch (programmatic dependent launch:
    // a chained launch may start while the previous one drains; kernels.cuh DecodeParams::pdl)
    const int par = p->launch_parity;
    dp.ws_o = p->d_ws_o + static_cast<size_t>(par) * p->ws_cap * p->cfg.head_dim;
    dp.ws_ml = p->d_ws_ml + static_cast<size_t>(par) * p->ws_cap;
    dp.counters = p->d_counters + static_cast<size_t>(par) * counters_per_parity(&p->cfg);
    dp.fuse_stats = stats ? 1 : 0;
    dp.max_pages_per_req = p->cfg.max_pages_per_req;
    dp.stats = reinterpret_cast<unsigned long long *>(p->d_stats);
    dp.stats_done = p->d_stats_done;
    dp.cap_pages = p->cfg.cap_pages;
    dp.layer = layer0;
    dp.kv_heads = p->cfg.kv_heads;
    dp.n_layers = nl;
    dp.layer_stride = p->layer_stride;
    dp.q_layer_stride = q_ls;
    dp.out_layer_stride = o_ls;
    dp.n_ws_rows = p->meta_ws_rows;
    dp.n_tasks = p->meta_items * p->cfg.kv_heads * nl;
    dp.task_counter = p->d_task_counter + 2 * par;
    dp.tma_rank = p->tma_rank;
    dp.half_boxes = p->has_tmap_half ? 1 : 0;
    dp.pdl = !p->pdl_enabled ? 0 : (chain == 2 ? 2 : ((chain == 1 && !stats) ? 1 : 0));
    dp.seq = ++p->decode_seq;
    dp.done_seq = p->d_done_seq;
    dp.trace = p->d_trace;
    dp.trace_cap = p->trace_cap;
    dp.trace_seq = static_cast<int32_t>(p->n_launches);
    // persistent grid: every resident CTA slot (4 warps each), or fewer for small batches
    const int ctas = std::max(1, std::min(p->num_sms * p->ctas_per_sm, (dp.n_tasks + 3) / 4));
    GqaMaps maps;
    if (p->has_tmap) {
        maps.full = p->tmap;
        maps.half = p->has_tmap_half ? p->tmap_half : p->tmap;
    }
    DBK_CUDA(launch_decode(dp, p->cfg.kv_dtype, p->cfg.head_dim, p->cfg.q_heads / p->cfg.kv_heads, ctas,
                           p->has_tmap ? &maps : nullptr, s));
    ++p->n_launches;
    p->launch_parity ^= 1;
    return DBK_OK;
}

static dbk_status decode_args_ok(dbk_pool *p, const dbk_batch *b, const void *q, void *out, int32_t out_dtype) {
    if (!p || !b) return fail(DBK_EINVAL, "decode_step: null argument");
    if (b->n < 0 || (b->n > 0 && (!b->req_ids || !q || !out))) return fail(DBK_EINVAL, "decode_step: bad arrays");
    if (b->layer < 0 || b->layer >= p->cfg.layers) return fail(DBK_EINVAL, "decode_step: layer out of range");
    if (b->chain < 0 || b->chain > 2) return fail(DBK_EINVAL, "decode_step: chain must be 0, 1 or 2");
    if (out_dtype < 0 || out_dtype > 2) return fail(DBK_EINVAL, "decode_step: out_dtype must be 0, 1 or 2");
    if (b->n > p->cfg.max_requests) return fail(DBK_EINVAL, "decode_step: n > max_requests");
    if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(out)) & 15)
        return fail(DBK_EINVAL, "decode_step: q and out must be 16-byte aligned");
    return DBK_OK;
}

}  // namespace dbk

// The stats record before a fused step: zero for K4 to accumulate into, or -- an empty batch,
// where no launch reduces it -- the empty batch's record (O3: cap_pages = free_pages = cap, R28).
static_assert(sizeof(dbk_stats) == 128, "dbk_stats is the 128-byte record K4 reduces into");
static dbk_status reset_stats(dbk_pool *p, int32_t n, cudaStream_t s) {
    if (n > 0) {
        DBK_CUDA(cudaMemsetAsync(p->d_stats, 0, sizeof(dbk_stats), s));
        return DBK_OK;
    }
    dbk_stats empty{};
    empty.cap_pages = p->cfg.cap_pages;
    empty.free_pages = p->cfg.cap_pages;
    // pageable source: staged before the call returns, so the stack record may go
    DBK_CUDA(cudaMemcpyAsync(p->d_stats, &empty, sizeof(dbk_stats), cudaMemcpyHostToDevice, s));
    return DBK_OK;
}

extern "C" dbk_status dbk_decode_step(dbk_pool *p, const dbk_batch *b, const void *q, void *out,
                                      int32_t out_dtype, void *stream) {
    DBK_TRY(decode_args_ok(p, b, q, out, out_dtype));
    DBK_CUDA(cudaSetDevice(p->cfg.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DBK_TRY(flush_deltas(p, s));
    // the batch is checked (prepare_batch) before the stats record is reset: a rejected call
    // leaves everything as it was
    if (b->n > 0) DBK_TRY(prepare_batch(p, b->n, b->req_ids, s));
    if (b->fuse_stats) DBK_TRY(reset_stats(p, b->n, s));
    if (b->n == 0) return DBK_OK;
    DBK_TRY(decode_launch(p, b->n, b->layer, 1, q, 0, out, 0, out_dtype, b->fuse_stats != 0, b->chain, s));
    p->last_decode_bytes = decode_bytes(p, out_dtype);
    return DBK_OK;
}

extern "C" dbk_status dbk_decode_step_layers(dbk_pool *p, const dbk_batch *b, int32_t n_layers, const void *q,
                                             int64_t q_layer_stride, void *out, int64_t out_layer_stride,
                                             int32_t out_dtype, void *stream, int32_t *launches_out) {
    DBK_TRY(decode_args_ok(p, b, q, out, out_dtype));
    if (n_layers < 1 || b->layer + n_layers > p->cfg.layers)
        return fail(DBK_EINVAL, "decode_step_layers: layers [%d, %d) out of range", b->layer, b->layer + n_layers);
    if (q_layer_stride < 0 || out_layer_stride < 0 || (q_layer_stride % 8) || (out_layer_stride % 8))
        return fail(DBK_EINVAL, "decode_step_layers: layer strides must be >= 0 and multiples of 8 elements");
    DBK_CUDA(cudaSetDevice(p->cfg.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DBK_TRY(flush_deltas(p, s));
    if (launches_out) *launches_out = 0;
    if (b->n > 0) DBK_TRY(prepare_batch(p, b->n, b->req_ids, s, n_layers));
    if (b->fuse_stats) DBK_TRY(reset_stats(p, b->n, s));
    if (b->n == 0) return DBK_OK;
    // layers per launch: as many as the split-K workspace budget holds (every layer of the step
    // in one launch when it fits)
    const int64_t per_layer_rows = static_cast<int64_t>(std::max(p->meta_ws_rows, 1)) * p->cfg.q_heads;
    const int64_t fit = static_cast<int64_t>(std::max(p->ws_cap, ws_budget_rows(p))) / per_layer_rows;
    int32_t group = static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(n_layers, fit)));
    if (p->max_layers_per_launch > 0) group = std::min(group, p->max_layers_per_launch);
    const int64_t eo = out_dtype == 2 ? 4 : 2;
    int32_t launched = 0;
    for (int32_t l0 = 0; l0 < n_layers; l0 += group) {
        const int32_t nl = std::min(group, n_layers - l0);
        const void *ql = static_cast<const uint8_t *>(q) + l0 * q_layer_stride * p->elt;
        void *ol = static_cast<uint8_t *>(out) + l0 * out_layer_stride * eo;
        const bool stats = b->fuse_stats && l0 == 0;
        DBK_TRY(decode_launch(p, b->n, b->layer + l0, nl, ql, q_layer_stride, ol, out_layer_stride, out_dtype, stats,
                              l0 > 0 ? 1 : b->chain, s));
        ++launched;
    }
    if (launches_out) *launches_out = launched;
    p->last_decode_bytes = decode_bytes(p, out_dtype);  // per layer
    return DBK_OK;
}

extern "C" dbk_status dbk_prefill_step(dbk_pool *p, const dbk_prefill_batch *b, const void *q, void *out,
                                       int32_t out_dtype, void *stream) {
    if (!p || !b) return fail(DBK_EINVAL, "prefill_step: null argument");
    if (b->n < 0 || (b->n > 0 && (!b->req_ids || !b->q_start || !b->q_len || !q || !out)))
        return fail(DBK_EINVAL, "prefill_step: bad arrays");
    if (b->layer < 0 || b->layer >= p->cfg.layers) return fail(DBK_EINVAL, "prefill_step: layer out of range");
    if (out_dtype < 0 || out_dtype > 2) return fail(DBK_EINVAL, "prefill_step: out_dtype must be 0, 1 or 2");
    if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(out)) & 15)
        return fail(DBK_EINVAL, "prefill_step: q and out must be 16-byte aligned");
    if (!p->has_ptmap) return fail(DBK_EINVAL, "prefill_step: pool has no 5-D tensor map");
    const int group = p->cfg.q_heads / p->cfg.kv_heads;
    const int qb = prefill_rows_per_tile() / group;  // chunk tokens per CTA (two 128-row tiles)
    const bool same = p->pref_valid && p->pref_epoch == p->epoch && p->pref_ids.size() == static_cast<size_t>(b->n) &&
                      std::equal(p->pref_ids.begin(), p->pref_ids.end(), b->req_ids) &&
                      std::equal(p->pref_s0.begin(), p->pref_s0.end(), b->q_start) &&
                      std::equal(p->pref_len.begin(), p->pref_len.end(), b->q_len);
    p->pref_tiles.clear();
    int64_t row = 0, flops = 0;
    for (int i = 0; i < b->n && !same; ++i) {
        auto it = p->reqs.find(b->req_ids[i]);
        if (it == p->reqs.end())
            return fail(DBK_ENOENT, "prefill_step: unknown request %lld", static_cast<long long>(b->req_ids[i]));
        const Request &r = it->second;
        const int32_t s0 = b->q_start[i], len = b->q_len[i];
        if (s0 < 0 || len < 1 || static_cast<int64_t>(s0) + len > r.ctx)
            return fail(DBK_EINVAL, "prefill_step: chunk %d [%d, %d) outside the %d tokens held", i, s0, s0 + len,
                        r.ctx);
        for (int32_t j0 = 0; j0 < len; j0 += qb) {
            PrefTile t{};
            t.slot = r.slot;
            t.q_start = s0;
            t.j0 = j0;
            t.rows_tok = std::min(qb, len - j0);
            t.q_row0 = static_cast<int32_t>(row);
            p->pref_tiles.push_back(t);
        }
        // algorithmic flops: QK^T and PV over the causal triangle, 4 d per (query head, key)
        for (int64_t j = 0; j < len; ++j) flops += 4LL * p->cfg.head_dim * p->cfg.q_heads * (s0 + j + 1);
        row += len;
    }
    if (row >= (1LL << 31) / p->cfg.q_heads) return fail(DBK_EINVAL, "prefill_step: too many rows");
    DBK_CUDA(cudaSetDevice(p->cfg.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DBK_TRY(flush_deltas(p, s));
    if (b->n == 0) return DBK_OK;
    if (!same) {
        // most keys first: the long causal tails start early, the grid ends on short CTAs
        std::stable_sort(p->pref_tiles.begin(), p->pref_tiles.end(), [](const PrefTile &x, const PrefTile &y) {
            return x.q_start + x.j0 + x.rows_tok > y.q_start + y.j0 + y.rows_tok;
        });
        DBK_TRY(p->up_pref.upload(p->pref_tiles.data(), p->pref_tiles.size() * sizeof(PrefTile), s));
        p->pref_ids.assign(b->req_ids, b->req_ids + b->n);
        p->pref_s0.assign(b->q_start, b->q_start + b->n);
        p->pref_len.assign(b->q_len, b->q_len + b->n);
        p->pref_epoch = p->epoch;
        p->pref_valid = true;
        p->pref_n_tiles = static_cast<int32_t>(p->pref_tiles.size());
        p->last_prefill_flops = flops;
    }
    PrefillParams pp;
    pp.block_table = p->d_bt;
    pp.bt_stride = p->cfg.max_pages_per_req;
    pp.layer = b->layer;
    pp.cap_pages = p->cfg.cap_pages;
    pp.kv_heads = p->cfg.kv_heads;
    pp.q_heads = p->cfg.q_heads;
    pp.tiles = static_cast<const PrefTile *>(p->up_pref.dev);
    pp.q = q;
    pp.out = out;
    pp.out_dtype = out_dtype;
    pp.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(p->cfg.head_dim)));
    DBK_CUDA(launch_prefill(pp, p->cfg.kv_dtype, p->cfg.head_dim, group, p->pref_n_tiles, p->cfg.kv_heads,
                            p->ptmap, s));
    ++p->n_launches;
    return DBK_OK;
}

extern "C" dbk_status dbk_batch_stats(dbk_pool *p, dbk_stats *host_out, void *stream) {
    if (!p || !host_out) return fail(DBK_EINVAL, "batch_stats: null argument");
    DBK_CUDA(cudaSetDevice(p->cfg.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DBK_CUDA(cudaMemcpyAsync(p->h_stats, p->d_stats, sizeof(dbk_stats), cudaMemcpyDeviceToHost, s));
    DBK_CUDA(cudaStreamSynchronize(s));
    *host_out = *p->h_stats;
    host_out->step_ns = 0;
    host_out->n_waiting = 0;
    return DBK_OK;
}

extern "C" dbk_status dbk_probe_read_bandwidth(const void *buf, size_t bytes, int32_t device, void *stream,
                                                double *ms_out) {
    if (!buf || !ms_out || bytes < 16 || bytes % 16) return fail(DBK_EINVAL, "probe_read_bandwidth: bad arguments");
    DBK_CUDA(cudaSetDevice(device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    uint32_t *sink = nullptr;
    cudaEvent_t a = nullptr, b = nullptr;
    DBK_CUDA(cudaMalloc(&sink, sizeof(uint32_t)));
    cudaError_t e = cudaEventCreate(&a);
    if (e == cudaSuccess) e = cudaEventCreate(&b);
    if (e == cudaSuccess) e = launch_read_probe(buf, bytes, sink, sms, s);  // warm-up
    if (e == cudaSuccess) e = cudaEventRecord(a, s);
    if (e == cudaSuccess) e = launch_read_probe(buf, bytes, sink, sms, s);
    if (e == cudaSuccess) e = cudaEventRecord(b, s);
    if (e == cudaSuccess) e = cudaEventSynchronize(b);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, a, b);
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
    cudaFree(sink);
    if (e != cudaSuccess) return fail(DBK_ECUDA, "probe_read_bandwidth: %s", cudaGetErrorString(e));
    *ms_out = ms;
    return DBK_OK;
}

extern "C" dbk_status dbk_synth_fill(uint64_t seed, int32_t kind, int32_t n_rows, const int64_t *req,
                                     const int32_t *pos, int32_t layer, int32_t n_heads, int32_t d,
                                     int32_t scale_log2, int32_t dtype, void *out, void *stream) {
    if (n_rows < 0 || (n_rows > 0 && (!req || !pos || !out)) || d % 8 || d < 8 || n_heads < 1 ||
        kind < 0 || kind > 2 || dtype < 0 || dtype > 2 || layer < 0)
        return fail(DBK_EINVAL, "synth_fill: bad arguments");
    if (n_rows == 0) return DBK_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::vector<uint8_t> blob(static_cast<size_t>(n_rows) * 12);
    std::memcpy(blob.data(), req, static_cast<size_t>(n_rows) * 8);
    std::memcpy(blob.data() + static_cast<size_t>(n_rows) * 8, pos, static_cast<size_t>(n_rows) * 4);
    int64_t *d_req = nullptr;
    DBK_CUDA(cudaMalloc(&d_req, blob.size()));
    cudaError_t e = cudaMemcpyAsync(d_req, blob.data(), blob.size(), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
        e = launch_synth_rows(seed, kind, n_rows, d_req, reinterpret_cast<const int32_t *>(d_req + n_rows), layer,
                              n_heads, d, scale_log2, dtype, out, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(d_req);
    if (e != cudaSuccess) return fail(DBK_ECUDA, "synth_fill: %s", cudaGetErrorString(e));
    return DBK_OK;
}

// Measurement utility: the decode kernels' task timeline (DBK_TRACE_TASKS=N at pool creation).
extern "C" dbk_status dbk_pool_trace_d2h(dbk_pool *p, void *host, int64_t cap, int64_t *n_out, int32_t reset) {
    if (!p || !n_out) return fail(DBK_EINVAL, "pool_trace_d2h: null argument");
    *n_out = 0;
    if (!p->d_trace) return DBK_OK;
    DBK_CUDA(cudaSetDevice(p->cfg.device));
    DBK_CUDA(cudaDeviceSynchronize());
    unsigned long long cnt = 0;
    DBK_CUDA(cudaMemcpy(&cnt, p->d_trace, 8, cudaMemcpyDeviceToHost));
    const int64_t n = std::min<int64_t>(static_cast<int64_t>(cnt), std::min<int64_t>(cap, p->trace_cap));
    if (host && n > 0) DBK_CUDA(cudaMemcpy(host, p->d_trace + 4, static_cast<size_t>(n) * 32, cudaMemcpyDeviceToHost));
    *n_out = n;
    if (reset) DBK_CUDA(cudaMemset(p->d_trace, 0, 8));
    return DBK_OK;
}
