// Cross-GPU statistics exchange: one ncclAllGather of the
// 128-byte dbk_stats record per rank per step over NVLink/NVSwitch, then a
// deterministic host reduction, so every rank takes the same b_{t+1}.
#include <nccl.h>

#include <cstring>
#include <new>
#include <vector>

#include "common.h"

struct dbk_comm {
    ncclComm_t nccl = nullptr;
    int nranks = 1, rank = 0, device = 0;
    dbk_stats *d_buf = nullptr;   // [1 + nranks] records: send, then gathered
    dbk_stats *h_buf = nullptr;   // pinned [nranks]
};

#define DBK_NCCL(call)                                                                          \
    do {                                                                                        \
        ncclResult_t r_ = (call);                                                               \
        if (r_ != ncclSuccess) return ::dbk::fail(DBK_ENCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
    } while (0)

extern "C" {

dbk_status dbk_stats_reduce(const dbk_stats *all, int32_t nranks, int32_t mode, dbk_stats *out) {
    if (!all || !out || nranks < 1) return dbk::fail(DBK_EINVAL, "stats_reduce: bad arguments");
    dbk_stats g;
    std::memset(&g, 0, sizeof g);
    if (mode == DBK_MODE_TP) {
        g = all[0];
        for (int r = 1; r < nranks; ++r) {
            dbk_stats a = all[r], b = all[0];
            a.step_ns = b.step_ns = 0;
            a.n_waiting = b.n_waiting = 0;
            if (std::memcmp(&a, &b, sizeof a) != 0)
                return dbk::fail(DBK_EINVAL, "stats_reduce: TP ranks disagree on batch statistics (rank %d)", r);
        }
    } else if (mode == DBK_MODE_DP) {
        for (int r = 0; r < nranks; ++r) {
            const dbk_stats &a = all[r];
            g.n_active += a.n_active;
            g.sum_ctx += a.sum_ctx;
            g.sum_ctx_sq += a.sum_ctx_sq;
            g.max_ctx = a.max_ctx > g.max_ctx ? a.max_ctx : g.max_ctx;
            g.sum_pages += a.sum_pages;
            g.cap_pages += a.cap_pages;
            g.free_pages += a.free_pages;
            g.over_cap |= a.over_cap;
            g.table_mismatch += a.table_mismatch;
            g.n_finished += a.n_finished;
            g.fin_sum_lin += a.fin_sum_lin;
            g.fin_sum_lin_sq += a.fin_sum_lin_sq;
            g.fin_sum_lout += a.fin_sum_lout;
            g.fin_sum_lout_sq += a.fin_sum_lout_sq;
            g.n_waiting += a.n_waiting;
        }
    } else {
        return dbk::fail(DBK_EINVAL, "stats_reduce: unknown mode %d", mode);
    }
    g.step_ns = 0;
    for (int r = 0; r < nranks; ++r) g.step_ns = all[r].step_ns > g.step_ns ? all[r].step_ns : g.step_ns;
    *out = g;
    return DBK_OK;
}

dbk_status dbk_comm_unique_id(void *id_out) {
    if (!id_out) return dbk::fail(DBK_EINVAL, "comm_unique_id: null output");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    DBK_NCCL(ncclGetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof id);
    return DBK_OK;
}

dbk_status dbk_comm_create(int32_t nranks, int32_t rank, const void *id_in, int32_t device, dbk_comm **out) {
    if (!id_in || !out || nranks < 1 || rank < 0 || rank >= nranks) return dbk::fail(DBK_EINVAL, "comm_create: bad arguments");
    DBK_CUDA(cudaSetDevice(device));
    dbk_comm *c = new (std::nothrow) dbk_comm();
    if (!c) return dbk::fail(DBK_EINVAL, "out of host memory");
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    ncclUniqueId id;
    std::memcpy(&id, id_in, sizeof id);
    ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return dbk::fail(DBK_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
    if (cudaMalloc(&c->d_buf, sizeof(dbk_stats) * (1 + nranks)) != cudaSuccess ||
        cudaMallocHost(&c->h_buf, sizeof(dbk_stats) * nranks) != cudaSuccess) {
        dbk_comm_destroy(c);
        return dbk::fail(DBK_ECUDA, "comm_create: allocation failed");
    }
    *out = c;
    return DBK_OK;
}

dbk_status dbk_comm_info(dbk_comm *c, int32_t *nranks, int32_t *rank) {
    if (!c) return dbk::fail(DBK_EINVAL, "comm_info: null communicator");
    int n = 0, r = 0;
    DBK_NCCL(ncclCommCount(c->nccl, &n));
    DBK_NCCL(ncclCommUserRank(c->nccl, &r));
    if (nranks) *nranks = n;
    if (rank) *rank = r;
    return DBK_OK;
}

dbk_status dbk_comm_destroy(dbk_comm *c) {
    if (!c) return DBK_OK;
    if (c->nccl) ncclCommDestroy(c->nccl);
    if (c->d_buf) cudaFree(c->d_buf);
    if (c->h_buf) cudaFreeHost(c->h_buf);
    delete c;
    return DBK_OK;
}

dbk_status dbk_stats_allgather(dbk_comm *c, const dbk_stats *local, dbk_stats *all, dbk_stats *global,
                               int32_t mode, void *stream) {
    if (!c || !local || !all || !global) return dbk::fail(DBK_EINVAL, "stats_allgather: null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DBK_CUDA(cudaSetDevice(c->device));
    DBK_CUDA(cudaMemcpyAsync(c->d_buf, local, sizeof(dbk_stats), cudaMemcpyHostToDevice, s));
    DBK_NCCL(ncclAllGather(c->d_buf, c->d_buf + 1, sizeof(dbk_stats) / sizeof(int64_t), ncclInt64, c->nccl, s));
    DBK_CUDA(cudaMemcpyAsync(c->h_buf, c->d_buf + 1, sizeof(dbk_stats) * c->nranks, cudaMemcpyDeviceToHost, s));
    DBK_CUDA(cudaStreamSynchronize(s));
    std::memcpy(all, c->h_buf, sizeof(dbk_stats) * c->nranks);
    return dbk_stats_reduce(all, c->nranks, mode, global);
}

}  // extern "C"
