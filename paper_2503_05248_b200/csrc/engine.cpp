// Engine: one continuous-batching decode iteration per call (SURVEY.md §8(a) S1-S7,
// DESIGN.md R17-R22).  The decode step's GPU work is timed with CUDA events; the
// measured latency feeds Algorithm 2 and advances the engine clock.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <deque>
#include <new>
#include <vector>

#include "common.h"
#include "kernels.cuh"
#include "mailbox.h"
#include "pool.h"

using namespace dbk;

struct dbk_engine {
    dbk_pool *pool = nullptr;
    dbk_sched *sched = nullptr;
    dbk_engine_config cfg{};
    // full (global) trace; this rank serves indices i with i % world == rank
    std::vector<int64_t> arrival, ids;
    std::vector<int32_t> l_in, l_out, gen;
    std::vector<int64_t> admit_ns, finish_ns;  // per trace index, -1 = not yet
    std::vector<uint8_t> swapped;     // per trace index: KV in the pool's swap space (R29)
    std::vector<int32_t> mine;        // local trace indices in arrival order
    size_t next_local = 0;            // next local index to release
    size_t next_global = 0;           // first global index with arrival > clock
    std::deque<int32_t> queue;        // local waiting (trace indices)
    std::vector<int32_t> running;     // local running, admission order
    // PD fusion (R25-R28): admitted requests still prefilling, admission order (all of them
    // were admitted after every running request: prefill is FCFS)
    struct Prefilling {
        int32_t r, done;
    };
    std::vector<Prefilling> prefilling;
    std::vector<int64_t> pf_ids;      // this step's chunk: request, first position, tokens
    std::vector<int32_t> pf_start, pf_len;
    std::vector<uint8_t> pf_rows;     // per chunk row: req id (int64) | position (int32)
    UploadBuffer up_pf;
    UploadBuffer tok_in, tok_out;     // full-model e2e: token ids (pinned staging + device)
    int32_t step_prefill = 0;
    int64_t clock = 0, t = 0;
    int32_t b = 1;
    int64_t fin_global = 0;           // cumulative finished (global)
    bool prev_known = false;
    int64_t prev_running_g = 0, prev_waiting_g = 0;
    // step state between launch and finish
    bool in_step = false;
    int64_t step_clock0 = 0;
    int32_t step_b = 0, step_adm = 0, step_pre = 0, step_launches = 0;
    int32_t step_swap_out = 0, step_swap_in = 0;
    int64_t step_swap_bytes = 0;
    uint64_t step_hash = 0;
    int64_t step_h2d = 0, step_d2h = 0;
    std::vector<int64_t> batch_ids;
    std::vector<int32_t> batch_ctx;
    dbk_stats local{};
    // events
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::vector<cudaEvent_t> att0, att1;
    double att_ms = 0;
    int64_t att_launches = 0, att_bytes = 0;  // attention kernels timed and their algorithmic bytes
    int32_t step_attn_kernels = 0;            // multi-layer launches of this step
    std::vector<int64_t> layer_bytes;
    dbk_comm *comm = nullptr;
    int32_t comm_mode = DBK_MODE_DP;
    int32_t comm_nranks = 1;
    dbk_mbox *mbox = nullptr;         // mailbox exchange (v2), instead of comm
    bool mbox_pending = false;        // this step's records are in x_all (gathered by the kernel)
    std::vector<dbk_stats> x_all;     // the last exchange: every rank's record, rank order
    double x_us = 0, x_us_total = 0;  // host time of the last exchange / since the last reset
    int64_t x_count = 0;
    dbk_model *model = nullptr;       // full-model mode (NEXT row 3)
    // end-to-end mode: host<->device copies on their own streams, ordered by events
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_d2h = nullptr, ev_up = nullptr;
    std::vector<cudaEvent_t> ev_q, ev_o;
    ~dbk_engine() {
        up_pf.release();
        if (up_pf.done) cudaEventDestroy(up_pf.done);
        tok_in.release();
        tok_out.release();
        if (tok_in.done) cudaEventDestroy(tok_in.done);
        if (tok_out.done) cudaEventDestroy(tok_out.done);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        for (auto e : att0) cudaEventDestroy(e);
        for (auto e : att1) cudaEventDestroy(e);
        for (auto e : ev_q) cudaEventDestroy(e);
        for (auto e : ev_o) cudaEventDestroy(e);
        if (ev_d2h) cudaEventDestroy(ev_d2h);
        if (ev_up) cudaEventDestroy(ev_up);
        if (h2d) cudaStreamDestroy(h2d);
        if (d2h) cudaStreamDestroy(d2h);
    }
};

namespace {

// R21: equal split of b_t, the remainder rotating with the step index t (a rank whose floor
// share is 0 when b_t < G still admits every G steps: liveness)
int32_t b_share(int32_t b, int32_t rank, int32_t world, int64_t t) {
    const int64_t k = ((static_cast<int64_t>(rank) - t) % world + world) % world;
    return b / world + (k < b % world ? 1 : 0);
}

void release_arrivals(dbk_engine *e) {
    while (e->next_local < e->mine.size() && e->arrival[e->mine[e->next_local]] <= e->clock)
        e->queue.push_back(e->mine[e->next_local++]);
    while (e->next_global < e->arrival.size() && e->arrival[e->next_global] <= e->clock) ++e->next_global;
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

dbk_status ensure_copy_streams(dbk_engine *e) {
    if (e->h2d) return DBK_OK;
    const int L = e->pool->cfg.layers;
    DBK_CUDA(cudaStreamCreateWithFlags(&e->h2d, cudaStreamNonBlocking));
    DBK_CUDA(cudaStreamCreateWithFlags(&e->d2h, cudaStreamNonBlocking));
    DBK_CUDA(cudaEventCreateWithFlags(&e->ev_d2h, cudaEventDisableTiming));
    DBK_CUDA(cudaEventCreateWithFlags(&e->ev_up, cudaEventDisableTiming));
    e->ev_q.assign(L, nullptr);
    e->ev_o.assign(L, nullptr);
    for (int l = 0; l < L; ++l) {
        DBK_CUDA(cudaEventCreateWithFlags(&e->ev_q[l], cudaEventDisableTiming));
        DBK_CUDA(cudaEventCreateWithFlags(&e->ev_o[l], cudaEventDisableTiming));
    }
    return DBK_OK;
}

}  // namespace

extern "C" {

dbk_status dbk_engine_create(dbk_pool *pool, dbk_sched *sched, const dbk_engine_config *cfg,
                             dbk_engine **out) {
    if (!pool || !sched || !cfg || !out) return fail(DBK_EINVAL, "engine_create: null argument");
    const dbk_engine_config &c = *cfg;
    if (c.n_requests < 0 || (c.n_requests > 0 && (!c.arrival_ns || !c.l_in || !c.l_out)))
        return fail(DBK_EINVAL, "engine_create: trace arrays missing");
    if (c.world < 1 || c.rank < 0 || c.rank >= c.world) return fail(DBK_EINVAL, "engine_create: bad rank/world");
    if (c.out_dtype < 0 || c.out_dtype > 2) return fail(DBK_EINVAL, "engine_create: bad out_dtype");
    if (c.pd_fusion != 0 && c.pd_fusion != 1) return fail(DBK_EINVAL, "engine_create: pd_fusion must be 0 or 1");
    if (c.pd_fusion && !pool->has_ptmap) return fail(DBK_EINVAL, "engine_create: PD fusion needs the pool's prefill tensor map");
    if (c.preempt_mode != 0 && c.preempt_mode != 1) return fail(DBK_EINVAL, "engine_create: preempt_mode must be 0 or 1");
    if (c.per_layer_launches != 0 && c.per_layer_launches != 1)
        return fail(DBK_EINVAL, "engine_create: per_layer_launches must be 0 or 1");
    if (c.pd_token_budget < 0 || (c.pd_token_budget > 0 && !c.pd_fusion))
        return fail(DBK_EINVAL, "engine_create: pd_token_budget needs pd_fusion and must be >= 0");
    if (c.preempt_mode == 1 && (c.pd_fusion || !pool->swap_host))
        return fail(DBK_EINVAL, "engine_create: swap preemption needs an attached swap space and pd_fusion = 0");
    if (c.req_ids) {  // the pool keys requests by id: a trace naming one twice would collide mid-run
        std::vector<int64_t> sorted(c.req_ids, c.req_ids + c.n_requests);
        std::sort(sorted.begin(), sorted.end());
        if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
            return fail(DBK_EINVAL, "engine_create: duplicate request id in the trace");
    }
    for (int i = 0; i < c.n_requests; ++i) {
        if (c.l_in[i] < 1 || c.l_out[i] < 1) return fail(DBK_EINVAL, "engine_create: lengths must be >= 1");
        if (i && c.arrival_ns[i] < c.arrival_ns[i - 1]) return fail(DBK_EINVAL, "engine_create: arrivals must be sorted");
        const int64_t need = ceil_div(static_cast<int64_t>(c.l_in[i]) + c.l_out[i], pool->cfg.page_size);
        if (need > pool->cfg.cap_pages || need > pool->cfg.max_pages_per_req)
            return fail(DBK_EFATAL, "engine_create: request %d cannot fit the cap alone", i);
    }
    dbk_engine *e = new (std::nothrow) dbk_engine();
    if (!e) return fail(DBK_EINVAL, "out of host memory");
    e->pool = pool;
    e->sched = sched;
    e->cfg = c;
    e->arrival.assign(c.arrival_ns, c.arrival_ns + c.n_requests);
    e->l_in.assign(c.l_in, c.l_in + c.n_requests);
    e->l_out.assign(c.l_out, c.l_out + c.n_requests);
    e->gen.assign(c.n_requests, 0);
    e->admit_ns.assign(c.n_requests, -1);
    e->finish_ns.assign(c.n_requests, -1);
    e->swapped.assign(c.n_requests, 0);
    e->ids.resize(c.n_requests);
    for (int i = 0; i < c.n_requests; ++i) e->ids[i] = c.req_ids ? c.req_ids[i] : i;
    for (int i = c.rank; i < c.n_requests; i += c.world) e->mine.push_back(i);
    dbk_sched_state st;
    dbk_sched_get_state(sched, &st);
    e->b = st.b;
    e->cfg.arrival_ns = nullptr;
    e->cfg.l_in = nullptr;
    e->cfg.l_out = nullptr;
    e->cfg.req_ids = nullptr;
    cudaSetDevice(pool->cfg.device);
    if (cudaEventCreate(&e->ev0) != cudaSuccess || cudaEventCreate(&e->ev1) != cudaSuccess) {
        delete e;
        return fail(DBK_ECUDA, "engine_create: cudaEventCreate failed");
    }
    const int L = pool->cfg.layers;
    e->att0.resize(L);
    e->att1.resize(L);
    for (int l = 0; l < L; ++l) {
        if (cudaEventCreate(&e->att0[l]) != cudaSuccess || cudaEventCreate(&e->att1[l]) != cudaSuccess) {
            delete e;
            return fail(DBK_ECUDA, "engine_create: cudaEventCreate failed");
        }
    }
    e->layer_bytes.assign(L, 0);
    *out = e;
    return DBK_OK;
}

dbk_status dbk_engine_destroy(dbk_engine *e) {
    delete e;
    return DBK_OK;
}

dbk_status dbk_engine_done(dbk_engine *e, int32_t *done) {
    if (!e || !done) return fail(DBK_EINVAL, "engine_done: null argument");
    *done = e->fin_global >= static_cast<int64_t>(e->arrival.size()) ? 1 : 0;
    return DBK_OK;
}

dbk_status dbk_engine_attach_model(dbk_engine *e, dbk_model *m) {
    if (!e) return fail(DBK_EINVAL, "attach_model: null engine");
    // the model's QKV epilogue writes the decode tokens' K/V into its own pool's pages, which
    // must be the pages this engine allocates
    if (m && model_pool(m) != e->pool) return fail(DBK_EINVAL, "attach_model: the model was created on another pool");
    e->model = m;
    return DBK_OK;
}

dbk_status dbk_engine_attach_comm(dbk_engine *e, dbk_comm *c, int32_t mode) {
    if (!e || (mode != DBK_MODE_DP && mode != DBK_MODE_TP)) return fail(DBK_EINVAL, "attach_comm: bad argument");
    if (c && e->mbox) return fail(DBK_EINVAL, "attach_comm: a mailbox is attached");
    int32_t n = 1;
    if (c) {
        DBK_TRY(dbk_comm_info(c, &n, nullptr));
        // DP: the engine serves request shard `rank` of `world`, the communicator must span the
        // same ranks; TP: every rank serves all requests (world 1), the communicator spans the
        // KV-head shards
        if (mode == DBK_MODE_DP && n != e->cfg.world)
            return fail(DBK_EINVAL, "attach_comm: DP communicator of %d ranks, engine world %d", n, e->cfg.world);
        if (mode == DBK_MODE_TP && e->cfg.world != 1)
            return fail(DBK_EINVAL, "attach_comm: TP mode needs an engine with world 1 (got %d)", e->cfg.world);
    }
    e->comm = c;
    e->comm_mode = mode;
    e->comm_nranks = n;
    return DBK_OK;
}

dbk_status dbk_engine_attach_mbox(dbk_engine *e, dbk_mbox *m, int32_t mode) {
    if (!e || (mode != DBK_MODE_DP && mode != DBK_MODE_TP)) return fail(DBK_EINVAL, "attach_mbox: bad argument");
    if (m && e->comm) return fail(DBK_EINVAL, "attach_mbox: a communicator is attached");
    const int32_t n = m ? mbox_nranks(m) : 1;
    if (m && mode == DBK_MODE_DP && n != e->cfg.world)
        return fail(DBK_EINVAL, "attach_mbox: DP mailbox of %d ranks, engine world %d", n, e->cfg.world);
    if (m && mode == DBK_MODE_TP && e->cfg.world != 1)
        return fail(DBK_EINVAL, "attach_mbox: TP mode needs an engine with world 1 (got %d)", e->cfg.world);
    e->mbox = m;
    e->comm_mode = mode;
    e->comm_nranks = n;
    return DBK_OK;
}

dbk_status dbk_engine_last_exchange(dbk_engine *e, dbk_stats *all, int32_t cap, int32_t *nranks, double *us,
                                    double *us_total, int64_t *count, int32_t reset) {
    if (!e) return fail(DBK_EINVAL, "engine_last_exchange: null engine");
    const int32_t n = static_cast<int32_t>(e->x_all.size());
    if (nranks) *nranks = n;
    for (int32_t r = 0; all && r < n && r < cap; ++r) all[r] = e->x_all[r];
    if (us) *us = e->x_us;
    if (us_total) *us_total = e->x_us_total;
    if (count) *count = e->x_count;
    if (reset) {
        e->x_us_total = 0;
        e->x_count = 0;
    }
    return DBK_OK;
}

dbk_status dbk_engine_step_launch(dbk_engine *e, const dbk_engine_buffers *bufs, void *stream,
                                  dbk_stats *local_out) {
    if (!e || !bufs || !local_out) return fail(DBK_EINVAL, "engine_step_launch: null argument");
    if (e->in_step) return fail(DBK_EINVAL, "engine_step_launch: previous step not finished");
    if (e->fin_global >= static_cast<int64_t>(e->arrival.size())) return fail(DBK_ENOENT, "engine: all requests finished");
    dbk_pool *p = e->pool;
    const dbk_pool_config &pc = p->cfg;
    const bool e2e = bufs->host_q != nullptr;
    const bool tok_io = bufs->host_tokens != nullptr;  // full-model end to end: token ids in, samples out
    if (!bufs->q_dev || !bufs->out_dev) return fail(DBK_EINVAL, "engine_step_launch: q_dev and out_dev are required");
    if (e2e && (!bufs->host_k || !bufs->host_v || !bufs->kv_dev))
        return fail(DBK_EINVAL, "engine_step_launch: end-to-end mode needs host_q, host_k, host_v and kv_dev");
    const bool pd = e->cfg.pd_fusion != 0;
    if (pd && e2e) return fail(DBK_EINVAL, "engine_step_launch: PD fusion runs in device-resident mode only");
    if (e->model && e2e) return fail(DBK_EINVAL, "engine_step_launch: full-model mode takes token ids (host_tokens), not q/K/V");
    if (tok_io && !e->model) return fail(DBK_EINVAL, "engine_step_launch: host_tokens needs an attached model");
    DBK_CUDA(cudaSetDevice(pc.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t P = pc.page_size;
    const int64_t launches0 = p->n_launches;

    // S1: arrivals, idle jump (global, R19)
    release_arrivals(e);
    const bool idle_g = e->prev_known ? (e->prev_running_g == 0 && e->prev_waiting_g == 0)
                                      : (e->next_global == 0);
    if (idle_g && e->next_global < e->arrival.size()) {
        e->clock = std::max(e->clock, e->arrival[e->next_global]);
        release_arrivals(e);
    }
    e->step_clock0 = e->clock;
    e->step_b = e->b;
    DBK_CUDA(cudaEventRecord(e->ev0, s));
    if (e->mbox) {  // S5 on the device clock: the exchange kernel subtracts this stamp
        DBK_TRY(mbox_stamp(e->mbox, s));
        ++p->n_launches;
    }

    // S1: FCFS admission with head-of-line blocking (R17); prefill = synthetic fill of T tokens,
    // a swapped-out request is swapped back in instead (R30).  Pages are taken in admission
    // order: pending fills are flushed before a swap-in.
    const int32_t share = b_share(e->b, e->cfg.rank, e->cfg.world, e->t);
    std::vector<int64_t> adm_ids;
    std::vector<int32_t> adm_tok;
    int64_t free_pages = p->pages.free_count;
    int32_t adm = 0, pre = 0;
    e->step_swap_out = e->step_swap_in = 0;
    const int64_t swap_bytes0 = p->swap_bytes_moved;
    auto flush_fills = [&]() -> dbk_status {
        if (!adm_ids.empty())
            DBK_TRY(dbk_append_tokens(p, static_cast<int32_t>(adm_ids.size()), adm_ids.data(), adm_tok.data(),
                                      nullptr, nullptr, e->cfg.synth_seed, s));
        adm_ids.clear();
        adm_tok.clear();
        return DBK_OK;
    };
    while (!pd && !e->queue.empty() && static_cast<int32_t>(e->running.size()) < share) {
        const int32_t r = e->queue.front();
        const int64_t T = static_cast<int64_t>(e->l_in[r]) + e->gen[r];
        if (free_pages < ceil_div(T + 1, P)) break;
        e->queue.pop_front();
        if (e->swapped[r]) {
            DBK_TRY(flush_fills());
            DBK_TRY(dbk_swap_in(p, 1, &e->ids[r], s));
            e->swapped[r] = 0;
            ++e->step_swap_in;
        } else {
            DBK_TRY(dbk_request_begin(p, e->ids[r], e->l_in[r], e->l_out[r]));
            adm_ids.push_back(e->ids[r]);
            adm_tok.push_back(static_cast<int32_t>(T));
        }
        free_pages -= ceil_div(T, P);
        e->running.push_back(r);
        if (e->admit_ns[r] < 0) e->admit_ns[r] = e->clock;
        ++adm;
    }
    DBK_TRY(flush_fills());

    // S1/S2: page growth for this step's decode token; LIFO preemption on overflow (R18)
    // a running request holds ctx = l_in + generated tokens; it needs a page iff ctx % P == 0.
    // PD fusion: the admission order is running ++ prefilling, so prefills are evicted first.
    // Swap mode (R29): a running victim goes to the swap space if it has room, else recompute.
    int64_t need = 0;
    for (int32_t r : e->running)
        if ((static_cast<int64_t>(e->l_in[r]) + e->gen[r]) % P == 0) ++need;
    while (need > p->pages.free_count) {
        int32_t victim;
        if (pd && !e->prefilling.empty()) {
            victim = e->prefilling.back().r;
            e->prefilling.pop_back();
        } else {
            victim = e->running.back();
            e->running.pop_back();
            if ((static_cast<int64_t>(e->l_in[victim]) + e->gen[victim]) % P == 0) --need;
        }
        const int64_t vid = e->ids[victim];
        const int64_t vpages = ceil_div(static_cast<int64_t>(e->l_in[victim]) + e->gen[victim], P);
        if (e->cfg.preempt_mode == 1 && vpages <= p->swap_pages.free_count) {
            DBK_TRY(dbk_swap_out(p, 1, &vid, s));
            e->swapped[victim] = 1;
            ++e->step_swap_out;
        } else {
            DBK_TRY(dbk_release(p, 1, &vid));
        }
        e->queue.push_front(victim);
        ++pre;
    }
    e->step_swap_bytes = p->swap_bytes_moved - swap_bytes0;
    const int32_t n = static_cast<int32_t>(e->running.size());
    e->batch_ids.resize(n);
    e->batch_ctx.resize(n);
    std::vector<int32_t> ones(n, 1);
    for (int32_t x = 0; x < n; ++x) e->batch_ids[x] = e->ids[e->running[x]];
    e->step_h2d = e->step_d2h = 0;
    const size_t qrow = static_cast<size_t>(pc.q_heads) * pc.head_dim * 2;
    const size_t kvrow = static_cast<size_t>(pc.layers) * pc.kv_heads * pc.head_dim * 2;
    const size_t orow = static_cast<size_t>(pc.q_heads) * pc.head_dim * (e->cfg.out_dtype == 2 ? 4 : 2);
    if (n > 0) {
        if (e2e) {  // the K/V rows arrive over PCIe below (after every small upload of this step)
            DBK_TRY(append_plan(p, n, e->batch_ids.data(), ones.data(), true, s));  // layers appended per layer
        } else if (e->model) {  // the model's QKV epilogue writes the decode token's K/V
            DBK_TRY(dbk_reserve_tokens(p, n, e->batch_ids.data(), ones.data(), s));
        } else {
            DBK_TRY(dbk_append_tokens(p, n, e->batch_ids.data(), ones.data(), nullptr, nullptr, e->cfg.synth_seed, s));
        }
    }
    // PD fusion (R25-R27): chunk budget c_t = max(0, b_share - N^d) prompt tokens, FCFS over the
    // in-progress prefills then new admissions; pages left after the decode growth
    e->pf_ids.clear();
    e->pf_start.clear();
    e->pf_len.clear();
    int32_t n_pf_rows = 0;
    if (pd) {
        // R25: the token budget is this rank's b_t; R36: a fixed budget, b_t bounding requests only
        const int64_t tokens = e->cfg.pd_token_budget > 0 ? e->cfg.pd_token_budget : share;
        int64_t budget = std::max<int64_t>(0, std::min<int64_t>(tokens, pc.max_requests) - n);
        int64_t freep = p->pages.free_count;
        size_t i = 0;
        while (budget > 0) {
            int32_t r, done;
            int64_t k;
            bool cut = false;
            if (i < e->prefilling.size()) {
                r = e->prefilling[i].r;
                done = e->prefilling[i].done;
                const int64_t T = static_cast<int64_t>(e->l_in[r]) + e->gen[r];
                k = std::min<int64_t>(T - done, budget);
                const int64_t room = (ceil_div(done, P) + freep) * P - done;
                if (room < k) {
                    cut = true;
                    k = room;
                }
                if (k <= 0) break;
                freep -= ceil_div(done + k, P) - ceil_div(done, P);
            } else if (!e->queue.empty() &&
                       static_cast<int64_t>(e->running.size() + e->prefilling.size()) < share) {
                r = e->queue.front();
                done = 0;
                const int64_t T = static_cast<int64_t>(e->l_in[r]) + e->gen[r];
                if (freep < ceil_div(T + 1, P)) break;
                e->queue.pop_front();
                DBK_TRY(dbk_request_begin(p, e->ids[r], e->l_in[r], e->l_out[r]));
                e->prefilling.push_back({r, 0});
                if (e->admit_ns[r] < 0) e->admit_ns[r] = e->clock;
                ++adm;
                k = std::min<int64_t>(T, budget);
                freep -= ceil_div(k, P);
            } else {
                break;
            }
            e->pf_ids.push_back(e->ids[r]);
            e->pf_start.push_back(done);
            e->pf_len.push_back(static_cast<int32_t>(k));
            e->prefilling[i].done += static_cast<int32_t>(k);
            n_pf_rows += static_cast<int32_t>(k);
            budget -= k;
            ++i;
            if (cut) break;
        }
        if (!e->pf_ids.empty() && e->model) {  // the model writes the chunk's K/V (real prefill)
            DBK_TRY(dbk_reserve_tokens(p, static_cast<int32_t>(e->pf_ids.size()), e->pf_ids.data(), e->pf_len.data(), s));
        } else if (!e->pf_ids.empty()) {
            DBK_TRY(dbk_append_tokens(p, static_cast<int32_t>(e->pf_ids.size()), e->pf_ids.data(), e->pf_len.data(),
                                      nullptr, nullptr, e->cfg.synth_seed, s));
            // the chunk's q rows (synthetic, all layers) follow the decode rows: (req, position)
            e->pf_rows.resize(static_cast<size_t>(n_pf_rows) * 12);
            int64_t *rq = reinterpret_cast<int64_t *>(e->pf_rows.data());
            int32_t *rp = reinterpret_cast<int32_t *>(e->pf_rows.data() + static_cast<size_t>(n_pf_rows) * 8);
            int32_t x = 0;
            for (size_t m = 0; m < e->pf_ids.size(); ++m)
                for (int32_t j = 0; j < e->pf_len[m]; ++j, ++x) {
                    rq[x] = e->pf_ids[m];
                    rp[x] = e->pf_start[m] + j;
                }
            DBK_TRY(e->up_pf.upload(e->pf_rows.data(), e->pf_rows.size(), s));
            const uint8_t *dev = static_cast<const uint8_t *>(e->up_pf.dev);
            DBK_CUDA(launch_synth_rows_layers(e->cfg.synth_seed, 0, n_pf_rows, reinterpret_cast<const int64_t *>(dev),
                                              reinterpret_cast<const int32_t *>(dev + static_cast<size_t>(n_pf_rows) * 8),
                                              pc.layers, pc.max_requests, n, pc.q_heads,
                                              pc.kv_head_offset * (pc.q_heads / pc.kv_heads), pc.head_dim,
                                              e->cfg.q_scale_log2, pc.kv_dtype, bufs->q_dev, s));
            ++p->n_launches;
        }
    }
    e->step_prefill = n_pf_rows;
    uint64_t h = kFnvOffset;
    for (int32_t x = 0; x < n; ++x) {
        const int32_t r = e->running[x];
        e->gen[r] += 1;
        const Request &rq = p->reqs.at(e->ids[r]);
        e->batch_ctx[x] = rq.ctx;
        h = fnv1a64(h, rq.id);
        h = fnv1a64(h, rq.ctx);
        h = fnv1a64(h, static_cast<int64_t>(rq.pages.size()));
        for (int32_t pg : rq.pages) h = fnv1a64(h, pg);
    }
    e->step_hash = h;

    // S3/S4: decode attention for every layer; statistics fused into layer 0
    dbk_batch bt;
    bt.n = n;
    bt.req_ids = e->batch_ids.data();
    // device-resident decode-only step: every layer's q exists before the first attention
    // launch, so the layers go through multi-layer launches unless per-layer ones were asked for
    // e2e steps chain their per-layer launches too: each layer's KV append runs on the copy
    // stream right behind that layer's inputs, so the compute stream holds only the decode
    // launches (an event wait each) and layer l+1's CTAs fill layer l's tail
    const bool chained = n_pf_rows == 0 && n > 0 && !e->model;
    const bool multi = chained && !e2e && !e->cfg.per_layer_launches;
    if (n > 0) DBK_TRY(prepare_batch(p, n, e->batch_ids.data(), s, multi ? pc.layers : 1));
    if (n > 0 && !e2e && !e->model) {  // synthetic q of all layers (stands in for the QKV projection), one launch
        DBK_CUDA(launch_synth_q(e->cfg.synth_seed, p->d_req, n, pc.layers, pc.max_requests, pc.q_heads,
                                pc.kv_head_offset * (pc.q_heads / pc.kv_heads), pc.head_dim, e->cfg.q_scale_log2, pc.kv_dtype, bufs->q_dev, s));
        ++p->n_launches;
    }
    if (e2e && n > 0) {
        // end-to-end: this step's new K/V rows and q come from pinned host memory on a copy
        // stream (inside the timed region: it waits on ev0), layer by layer: layer l's KV
        // append and attention wait only for layer l's K, V and q, so the PCIe transfers of
        // later layers overlap the attention of earlier ones.  Issued after this step's small
        // metadata uploads on `s`: host-to-device copies share the copy engine in issue order,
        // so an upload queued behind 400 MB of inputs would hold layer 0 back until they land.
        DBK_TRY(ensure_copy_streams(e));
        // K/V rows are layer-major on both sides ([layers][rows][kv_heads][d]): one contiguous
        // copy per layer (2-D copies of 2 KiB rows -- 70B shards -- ran far below PCIe speed)
        uint8_t *kd = static_cast<uint8_t *>(bufs->kv_dev);
        uint8_t *vd = kd + static_cast<size_t>(pc.max_requests) * kvrow;
        const size_t lrow = kvrow / pc.layers;  // one layer's K (or V) row of a request
        DBK_CUDA(cudaEventRecord(e->ev_up, s));
        DBK_CUDA(cudaStreamWaitEvent(e->h2d, e->ev_up, 0));
        for (int l = 0; l < pc.layers; ++l) {
            const size_t doff = static_cast<size_t>(l) * pc.max_requests * lrow, hoff = static_cast<size_t>(l) * n * lrow;
            DBK_CUDA(cudaMemcpyAsync(kd + doff, static_cast<const uint8_t *>(bufs->host_k) + hoff, n * lrow,
                                     cudaMemcpyHostToDevice, e->h2d));
            DBK_CUDA(cudaMemcpyAsync(vd + doff, static_cast<const uint8_t *>(bufs->host_v) + hoff, n * lrow,
                                     cudaMemcpyHostToDevice, e->h2d));
            uint8_t *qd = static_cast<uint8_t *>(bufs->q_dev) + static_cast<size_t>(l) * pc.max_requests * qrow;
            const uint8_t *qh = static_cast<const uint8_t *>(bufs->host_q) + static_cast<size_t>(l) * n * qrow;
            DBK_CUDA(cudaMemcpyAsync(qd, qh, n * qrow, cudaMemcpyHostToDevice, e->h2d));
            // the layer's new K/V rows into their page slots (K5), on the copy stream: after the
            // step's job list upload (ev_up) and every earlier launch on `s`, which ev_up covers
            DBK_TRY(append_launch(p, kd, vd, 0, l, 1, e->h2d, pc.max_requests));
            DBK_CUDA(cudaEventRecord(e->ev_q[l], e->h2d));
        }
        e->step_h2d += 2 * static_cast<int64_t>(n * kvrow) + static_cast<int64_t>(pc.layers) * n * qrow;
    }
    // device-resident decode-only steps chain the layer launches (programmatic dependent
    // launch: layer l+1's CTAs fill layer l's tail); then the attention time is one window
    const bool per_layer_ev = e->cfg.time_attention && n > 0 && !chained && !e->model;
    if (e->cfg.time_attention && chained) DBK_CUDA(cudaEventRecord(e->att0[0], s));
    if (e->model) {
        dbk_prefill_batch pb{};
        pb.n = static_cast<int32_t>(e->pf_ids.size());
        pb.req_ids = e->pf_ids.data();
        pb.q_start = e->pf_start.data();
        pb.q_len = e->pf_len.data();
        int32_t *tok_dev = nullptr, *smp_dev = nullptr;
        if (tok_io && n > 0) {  // this step's input tokens from the caller's array (pinned), H2D
            DBK_TRY(e->tok_in.reserve(static_cast<size_t>(n) * 4));
            int32_t *th = static_cast<int32_t *>(e->tok_in.host);
            if (e->tok_in.pending) DBK_CUDA(cudaEventSynchronize(e->tok_in.done));
            for (int32_t x = 0; x < n; ++x) th[x] = bufs->host_tokens[e->running[x]];
            DBK_CUDA(cudaMemcpyAsync(e->tok_in.dev, th, static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, s));
            DBK_CUDA(cudaEventRecord(e->tok_in.done, s));
            e->tok_in.pending = true;
            tok_dev = static_cast<int32_t *>(e->tok_in.dev);
            DBK_TRY(e->tok_out.reserve(static_cast<size_t>(pc.max_requests) * 4));
            smp_dev = static_cast<int32_t *>(e->tok_out.dev);
            e->step_h2d += static_cast<int64_t>(n) * 4;
        }
        DBK_TRY(dbk_model_step_pd(e->model, n, e->batch_ids.data(), pb.n > 0 ? &pb : nullptr, 1, nullptr, tok_dev,
                                  smp_dev, s));
        if (smp_dev) {  // the decode rows' samples back to pinned memory (scattered after the sync)
            DBK_CUDA(cudaMemcpyAsync(e->tok_out.host, smp_dev, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost, s));
            e->step_d2h += static_cast<int64_t>(n) * 4;
        }
    }
    if (multi) {
        bt.layer = 0;
        bt.fuse_stats = 1;
        bt.chain = 0;
        const int64_t ls = static_cast<int64_t>(pc.max_requests) * pc.q_heads * pc.head_dim;
        DBK_TRY(dbk_decode_step_layers(p, &bt, pc.layers, bufs->q_dev, ls, bufs->out_dev, ls, e->cfg.out_dtype, s,
                                       &e->step_attn_kernels));
        for (int l = 0; l < pc.layers; ++l) e->layer_bytes[l] = p->last_decode_bytes;
    }
    for (int l = 0; l < (e->model || multi ? 0 : pc.layers); ++l) {
        uint8_t *qd = static_cast<uint8_t *>(bufs->q_dev) + static_cast<size_t>(l) * pc.max_requests * qrow;
        uint8_t *od = static_cast<uint8_t *>(bufs->out_dev) + static_cast<size_t>(l) * pc.max_requests * orow;
        bt.layer = l;
        bt.fuse_stats = l == 0 ? 1 : 0;
        bt.chain = (chained && l > 0) ? 1 : 0;
        if (e2e && n > 0) DBK_CUDA(cudaStreamWaitEvent(s, e->ev_q[l], 0));  // q, K, V landed and appended
        if (per_layer_ev) DBK_CUDA(cudaEventRecord(e->att0[l], s));
        DBK_TRY(dbk_decode_step(p, &bt, qd, od, e->cfg.out_dtype, s));
        if (per_layer_ev) DBK_CUDA(cudaEventRecord(e->att1[l], s));
        e->layer_bytes[l] = p->last_decode_bytes;
        if (n_pf_rows > 0) {  // causal attention of the prefill chunk (K7, tensor cores)
            dbk_prefill_batch pb;
            pb.n = static_cast<int32_t>(e->pf_ids.size());
            pb.layer = l;
            pb.req_ids = e->pf_ids.data();
            pb.q_start = e->pf_start.data();
            pb.q_len = e->pf_len.data();
            DBK_TRY(dbk_prefill_step(p, &pb, qd + static_cast<size_t>(n) * qrow, od + static_cast<size_t>(n) * orow,
                                     e->cfg.out_dtype, s));
        }
        if (e2e && n > 0 && bufs->host_out) {  // layer l's output goes back while l+1 computes
            DBK_CUDA(cudaEventRecord(e->ev_o[l], s));
            DBK_CUDA(cudaStreamWaitEvent(e->d2h, e->ev_o[l], 0));
            uint8_t *oh = static_cast<uint8_t *>(bufs->host_out) + static_cast<size_t>(l) * n * orow;
            DBK_CUDA(cudaMemcpyAsync(oh, od, n * orow, cudaMemcpyDeviceToHost, e->d2h));
        }
    }
    if (e->cfg.time_attention && chained) DBK_CUDA(cudaEventRecord(e->att1[0], s));
    if (e2e && n > 0) {
        if (bufs->host_out) e->step_d2h += static_cast<int64_t>(pc.layers) * n * orow;
        DBK_CUDA(cudaEventRecord(e->ev_d2h, e->d2h));
        DBK_CUDA(cudaStreamWaitEvent(s, e->ev_d2h, 0));  // the step ends after the last copy
    }
    DBK_CUDA(cudaEventRecord(e->ev1, s));
    const int64_t n_waiting = static_cast<int64_t>(e->queue.size() + e->prefilling.size());
    if (e->mbox) {  // S6 fused: the record leaves for every peer's mailbox straight from the device
        DBK_TRY(mbox_launch(e->mbox, reinterpret_cast<const unsigned long long *>(p->d_stats), n == 0, pc.cap_pages,
                            n_waiting, true, nullptr, s));
        ++p->n_launches;
    }
    // S5: statistics record (synchronises the stream) and device-timed step latency
    DBK_TRY(dbk_batch_stats(p, &e->local, s));
    if (n == 0) {  // no decode launch reduced the record: the empty batch's record (O3)
        e->local = dbk_stats{};
        e->local.cap_pages = pc.cap_pages;
        e->local.free_pages = pc.cap_pages;
    }
    float ms = 0.f;
    DBK_CUDA(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
    e->local.step_ns = std::llround(static_cast<double>(ms) * 1e6);
    if (tok_io && n > 0) {  // the stream is synchronised: each decode row's sample -> its request's slot
        const int32_t *sh = static_cast<const int32_t *>(e->tok_out.host);
        for (int32_t x = 0; x < n; ++x) bufs->host_tokens[e->running[x]] = sh[x];
    }
    e->local.n_waiting = n_waiting;
    if (e->mbox) {  // the gathered records (mapped host memory); this rank's carries the device step time
        e->x_all.resize(static_cast<size_t>(e->comm_nranks));
        DBK_TRY(mbox_collect(e->mbox, e->x_all.data()));
        e->local = e->x_all[static_cast<size_t>(mbox_rank(e->mbox))];
        e->mbox_pending = true;
    }
    if (pd) {  // R27: completed prompts join the decode batch from the next step on
        size_t m = 0;
        while (m < e->prefilling.size() &&
               e->prefilling[m].done == e->l_in[e->prefilling[m].r] + e->gen[e->prefilling[m].r]) {
            e->running.push_back(e->prefilling[m].r);
            ++m;
        }
        e->prefilling.erase(e->prefilling.begin(), e->prefilling.begin() + static_cast<std::ptrdiff_t>(m));
    }
    if (e->cfg.time_attention && n > 0 && e->model) {  // the model's per-layer attention events
        double a = 0;
        DBK_TRY(dbk_model_timing(e->model, &a, nullptr, nullptr, 1));
        e->att_ms += a;
        e->att_bytes += static_cast<int64_t>(pc.layers) * p->last_decode_bytes;
        e->att_launches += pc.layers;
    }
    if (e->cfg.time_attention && n > 0 && !e->model) {
        for (int l = 0; l < pc.layers; ++l) {
            float a = 0.f;
            if (per_layer_ev) DBK_CUDA(cudaEventElapsedTime(&a, e->att0[l], e->att1[l]));
            else if (l == 0) DBK_CUDA(cudaEventElapsedTime(&a, e->att0[0], e->att1[0]));
            e->att_ms += a;
            e->att_bytes += e->layer_bytes[l];
            if (!multi) ++e->att_launches;
        }
        if (multi) e->att_launches += e->step_attn_kernels;  // kernels, each streaming several layers
    }
    e->step_adm = adm;
    e->step_pre = pre;
    e->step_launches = static_cast<int32_t>(p->n_launches - launches0);
    e->in_step = true;
    *local_out = e->local;
    return DBK_OK;
}

dbk_status dbk_engine_step_finish(dbk_engine *e, const dbk_stats *global, dbk_step_record *rec) {
    if (!e || !global) return fail(DBK_EINVAL, "engine_step_finish: null argument");
    if (!e->in_step) return fail(DBK_EINVAL, "engine_step_finish: no step in flight");
    dbk_pool *p = e->pool;
    // S5': retire finished requests (release their pages)
    std::vector<int32_t> keep;
    std::vector<int64_t> done_ids;
    keep.reserve(e->running.size());
    for (int32_t r : e->running) {
        if (e->gen[r] == e->l_out[r]) {
            done_ids.push_back(e->ids[r]);
            e->finish_ns[r] = e->clock + global->step_ns;
        } else {
            keep.push_back(r);
        }
    }
    if (!done_ids.empty()) DBK_TRY(dbk_release(p, static_cast<int32_t>(done_ids.size()), done_ids.data()));
    e->running.swap(keep);
    // S6: clock, arrivals, global N^p / N^d
    e->clock += global->step_ns;
    release_arrivals(e);
    e->fin_global += global->n_finished;
    const int64_t running_g = global->n_active - global->n_finished;
    const int64_t waiting_g = static_cast<int64_t>(e->next_global) - running_g - e->fin_global;
    dbk_stats g = *global;
    g.n_waiting = waiting_g;
    // S7: b_{t+1}
    int32_t b_next = e->b, why = DBK_R_CARRY;
    DBK_TRY(dbk_choose_batch_size(e->sched, &g, e->cfg.mem_cap_bytes, e->cfg.sla_ms,
                                  static_cast<int32_t>(waiting_g), &b_next, &why));
    if (rec) {
        std::memset(rec, 0, sizeof *rec);
        rec->t = e->t;
        rec->clock_ns = e->step_clock0;
        rec->step_ns = global->step_ns;
        rec->sum_ctx = global->sum_ctx;
        rec->used_pages = global->sum_pages;
        rec->table_hash = static_cast<int64_t>(e->step_hash);
        rec->b_t = e->step_b;
        rec->b_next = b_next;
        rec->n_admitted = e->step_adm;
        rec->n_preempted = e->step_pre;
        rec->n_decode = static_cast<int32_t>(global->n_active);
        rec->n_finished = static_cast<int32_t>(global->n_finished);
        rec->rationale = why;
        rec->n_waiting = static_cast<int32_t>(waiting_g);
        rec->h2d_bytes = e->step_h2d;
        rec->d2h_bytes = e->step_d2h;
        rec->launches = e->step_launches;
        rec->n_prefill = e->step_prefill;
        rec->n_swap_out = e->step_swap_out;
        rec->n_swap_in = e->step_swap_in;
        rec->swap_bytes = e->step_swap_bytes;
    }
    e->b = b_next;
    e->prev_known = true;
    e->prev_running_g = running_g;
    e->prev_waiting_g = waiting_g;
    e->t += 1;
    e->in_step = false;
    return DBK_OK;
}

dbk_status dbk_engine_step(dbk_engine *e, const dbk_engine_buffers *bufs, void *stream, dbk_step_record *rec) {
    if (!e) return fail(DBK_EINVAL, "engine_step: null engine");
    dbk_stats local;
    DBK_TRY(dbk_engine_step_launch(e, bufs, stream, &local));
    dbk_stats global = local;
    if (e->mbox) {  // gathered by the step's exchange kernel
        if (!e->mbox_pending) return fail(DBK_EINVAL, "engine_step: mailbox records missing");
        e->mbox_pending = false;
        DBK_TRY(dbk_stats_reduce(e->x_all.data(), e->comm_nranks, e->comm_mode, &global));
        ++e->x_count;
    } else if (e->comm) {  // the gather buffer holds one record per communicator rank
        e->x_all.resize(static_cast<size_t>(e->comm_nranks));
        const auto t0 = std::chrono::steady_clock::now();
        DBK_TRY(dbk_stats_allgather(e->comm, &local, e->x_all.data(), &global, e->comm_mode, stream));
        e->x_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        e->x_us_total += e->x_us;
        ++e->x_count;
    } else if (e->cfg.world != 1) {
        return fail(DBK_EINVAL, "engine_step: world > 1 needs a communicator (or use step_launch/finish)");
    }
    return dbk_engine_step_finish(e, &global, rec);
}

dbk_status dbk_engine_last_batch(dbk_engine *e, int32_t *n, int64_t *ids, int32_t *ctx, int32_t cap) {
    if (!e || !n) return fail(DBK_EINVAL, "engine_last_batch: null argument");
    *n = static_cast<int32_t>(e->batch_ids.size());
    for (int32_t x = 0; x < cap && x < *n; ++x) {
        if (ids) ids[x] = e->batch_ids[x];
        if (ctx) ctx[x] = e->batch_ctx[x];
    }
    return DBK_OK;
}

dbk_status dbk_engine_request_times(dbk_engine *e, int32_t n, int64_t *first_admit_ns, int64_t *finish_ns) {
    if (!e || n < 0) return fail(DBK_EINVAL, "engine_request_times: bad argument");
    for (int32_t i = 0; i < n; ++i) {
        const bool have = static_cast<size_t>(i) < e->admit_ns.size();
        if (first_admit_ns) first_admit_ns[i] = have ? e->admit_ns[i] : -1;
        if (finish_ns) finish_ns[i] = have ? e->finish_ns[i] : -1;
    }
    return DBK_OK;
}

dbk_status dbk_engine_attn_timing(dbk_engine *e, double *ms, int64_t *launches, int64_t *bytes, int32_t reset) {
    if (!e) return fail(DBK_EINVAL, "engine_attn_timing: null engine");
    if (ms) *ms = e->att_ms;
    if (launches) *launches = e->att_launches;
    if (bytes) *bytes = e->att_bytes;
    if (reset) {
        e->att_ms = 0;
        e->att_launches = 0;
        e->att_bytes = 0;
    }
    return DBK_OK;
}

}  // extern "C"
