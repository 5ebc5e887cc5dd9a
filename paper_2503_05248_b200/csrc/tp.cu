// Tensor-parallel residual stream of the full decode step ("TP O-proj
// allreduce fused over NVLink", the model's step latency).
//
// With the model's heads and FFN split over G ranks (dbk_model_config.tp_size), the O and down
// projections produce PARTIAL sums of the residual update.  The all-reduce is split into
//   reduce-scatter  inside the GEMM: every 32-column chunk of a partial tile is added by TMA
//                   (cp.reduce.async.bulk .add) straight into the residual slice of the rank that
//                   OWNS those columns (rank r owns columns [r H/G, (r+1) H/G)), in that rank's
//                   memory (CUDA-IPC mapping: NVLink/NVSwitch peer memory on a multi-GPU box);
//   barrier         one warp (this file): release this rank's arrival into every rank's flag
//                   array, acquire every rank's;
//   all-gather      inside the next RMSNorm, which reads the G owners' slices of its row.
// This object owns kTpBufs rotating residual buffers [rows][H] fp32 plus the flags, in one
// allocation exported with CUDA IPC, and maps every peer's.
#include <cstring>
#include <new>
#include <vector>

#include "common.h"
#include "device_common.cuh"
#include "tp.h"

namespace dbk {
namespace {
constexpr int kMaxTpRanks = 8;
}

}  // namespace dbk

struct dbk_tp {
    int nranks = 0, rank = 0, device = 0, hidden = 0;
    int64_t rows = 0;
    uint8_t *local = nullptr;                     // kTpBufs buffers, then the flags
    size_t buf_bytes = 0;
    std::vector<void *> opened;                   // peer mappings (cudaIpcOpenMemHandle)
    void *bufs[dbk::kTpBufs][dbk::kMaxTpRanks]{};  // host copies of every rank's buffer pointers
    float **d_bufs = nullptr;                     // device [kTpBufs][nranks]
    uint64_t **d_flag_ptrs = nullptr;             // device [nranks]: rank r's flag array
    uint64_t epoch = 0;
    bool ready = false;
};

namespace dbk {
namespace {

__global__ void __launch_bounds__(32) tp_barrier_kernel(uint64_t *const *flags, int nranks, int rank, uint64_t epoch,
                                                        uint64_t timeout_ns) {
    const int lane = threadIdx.x;
    // every write this rank's previous kernels made (the GEMM's reduce-adds into peer memory) is
    // complete at this point in the stream; publish them system-wide, then the arrival
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("fence.sc.sys;" ::: "memory");
    if (lane < nranks)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flags[lane] + rank), "l"(epoch) : "memory");
    if (lane < nranks) {
        const uint64_t *mine = flags[rank] + lane;
        const uint64_t t0 = dev::globaltimer_ns();
        for (;;) {
            uint64_t v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
            if (v >= epoch) break;
            if (dev::globaltimer_ns() - t0 > timeout_ns) __trap();  // a rank never arrived
            __nanosleep(64);
        }
    }
    __syncwarp();
    asm volatile("fence.acq_rel.sys;" ::: "memory");
}

}  // namespace

int32_t tp_nranks(const dbk_tp *t) { return t->nranks; }
int32_t tp_rank(const dbk_tp *t) { return t->rank; }
int64_t tp_rows(const dbk_tp *t) { return t->rows; }
int32_t tp_hidden(const dbk_tp *t) { return t->hidden; }
void *const *tp_bufs(const dbk_tp *t, int idx) { return t->bufs[((idx % kTpBufs) + kTpBufs) % kTpBufs]; }
float *const *tp_bufs_dev(const dbk_tp *t, int idx) {
    return t->d_bufs + static_cast<size_t>(((idx % kTpBufs) + kTpBufs) % kTpBufs) * t->nranks;
}

dbk_status tp_barrier(dbk_tp *t, cudaStream_t s) {
    if (!t->ready) return fail(DBK_EINVAL, "tp: not opened");
    ++t->epoch;
    tp_barrier_kernel<<<1, 32, 0, s>>>(t->d_flag_ptrs, t->nranks, t->rank, t->epoch, 20000000000ull);
    DBK_CUDA(cudaGetLastError());
    return DBK_OK;
}

}  // namespace dbk

extern "C" {

dbk_status dbk_tp_create(int32_t nranks, int32_t rank, int32_t device, int64_t rows, int32_t hidden,
                         void *handle_out_64, dbk_tp **out) {
    if (!out || !handle_out_64 || nranks < 1 || nranks > dbk::kMaxTpRanks || rank < 0 || rank >= nranks || rows < 1 ||
        hidden < 1 || hidden % (32 * nranks))
        return dbk::fail(DBK_EINVAL, "tp_create: need 1 <= nranks <= %d, 0 <= rank < nranks, rows >= 1, hidden a "
                                     "multiple of 32 * nranks", dbk::kMaxTpRanks);
    DBK_CUDA(cudaSetDevice(device));
    dbk_tp *t = new (std::nothrow) dbk_tp();
    if (!t) return dbk::fail(DBK_EINVAL, "out of host memory");
    t->nranks = nranks;
    t->rank = rank;
    t->device = device;
    t->rows = rows;
    t->hidden = hidden;
    t->buf_bytes = (static_cast<size_t>(rows) * hidden * sizeof(float) + 255) & ~static_cast<size_t>(255);
    const size_t bytes = dbk::kTpBufs * t->buf_bytes + dbk::kMaxTpRanks * sizeof(uint64_t);
    cudaIpcMemHandle_t h;
    if (cudaMalloc(&t->local, bytes) != cudaSuccess || cudaMemset(t->local, 0, bytes) != cudaSuccess ||
        cudaMalloc(&t->d_bufs, sizeof(float *) * dbk::kTpBufs * nranks) != cudaSuccess ||
        cudaMalloc(&t->d_flag_ptrs, sizeof(uint64_t *) * nranks) != cudaSuccess ||
        cudaIpcGetMemHandle(&h, t->local) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
        const cudaError_t e = cudaGetLastError();
        dbk_tp_destroy(t);
        return dbk::fail(DBK_ECUDA, "tp_create: %s", cudaGetErrorString(e));
    }
    std::memcpy(handle_out_64, &h, sizeof h);
    *out = t;
    return DBK_OK;
}

dbk_status dbk_tp_open(dbk_tp *t, const void *handles) {
    if (!t || !handles) return dbk::fail(DBK_EINVAL, "tp_open: null argument");
    if (t->ready) return dbk::fail(DBK_EINVAL, "tp_open: already open");
    DBK_CUDA(cudaSetDevice(t->device));
    std::vector<uint8_t *> base(static_cast<size_t>(t->nranks), nullptr);
    for (int r = 0; r < t->nranks; ++r) {
        if (r == t->rank) {
            base[r] = t->local;
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const uint8_t *>(handles) + 64 * static_cast<size_t>(r), sizeof h);
        void *ptr = nullptr;
        const cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            cudaGetLastError();
            // nothing stays mapped: a failed open leaves the handle as created (retry-able)
            for (void *q : t->opened) cudaIpcCloseMemHandle(q);
            t->opened.clear();
            return dbk::fail(DBK_ECUDA, "tp_open: cudaIpcOpenMemHandle(rank %d): %s", r, cudaGetErrorString(e));
        }
        t->opened.push_back(ptr);
        base[r] = static_cast<uint8_t *>(ptr);
    }
    std::vector<float *> db(static_cast<size_t>(dbk::kTpBufs) * t->nranks);
    std::vector<uint64_t *> fl(static_cast<size_t>(t->nranks));
    for (int r = 0; r < t->nranks; ++r) {
        for (int b = 0; b < dbk::kTpBufs; ++b) {
            t->bufs[b][r] = base[r] + b * t->buf_bytes;
            db[static_cast<size_t>(b) * t->nranks + r] = static_cast<float *>(t->bufs[b][r]);
        }
        fl[r] = reinterpret_cast<uint64_t *>(base[r] + dbk::kTpBufs * t->buf_bytes);
    }
    DBK_CUDA(cudaMemcpy(t->d_bufs, db.data(), sizeof(float *) * db.size(), cudaMemcpyHostToDevice));
    DBK_CUDA(cudaMemcpy(t->d_flag_ptrs, fl.data(), sizeof(uint64_t *) * fl.size(), cudaMemcpyHostToDevice));
    t->ready = true;
    return DBK_OK;
}

dbk_status dbk_tp_destroy(dbk_tp *t) {
    if (!t) return DBK_OK;
    cudaSetDevice(t->device);
    cudaDeviceSynchronize();
    for (void *p : t->opened) cudaIpcCloseMemHandle(p);
    if (t->local) cudaFree(t->local);
    if (t->d_bufs) cudaFree(t->d_bufs);
    if (t->d_flag_ptrs) cudaFree(t->d_flag_ptrs);
    delete t;
    return DBK_OK;
}

dbk_status dbk_tp_barrier(dbk_tp *t, void *stream) {
    if (!t) return dbk::fail(DBK_EINVAL, "tp_barrier: null handle");
    DBK_CUDA(cudaSetDevice(t->device));
    return dbk::tp_barrier(t, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
