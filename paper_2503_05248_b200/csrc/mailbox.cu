// Cross-GPU statistics exchange without a collective launch (SURVEY.md §8(e) "B200-native v2"):
// every rank owns a device MAILBOX of 256-byte slots, one per (parity, source rank), exported
// with CUDA IPC and mapped by every peer (over NVLink / NVSwitch on a multi-GPU box; the same
// device's memory when the ranks share one GPU in tests).  At the end of a step ONE single-warp
// kernel on the step's stream
//   1. builds this rank's 128-byte record from the batch statistics K4 reduced on the device
//      (plus the step's device-timed latency: %globaltimer now minus the stamp the step's first
//      kernel took, and the host's N^p count),
//   2. stores it into slot [parity][rank] of EVERY rank's mailbox (P2P stores) and publishes it
//      with a release store of the step's sequence number,
//   3. spins (acquire loads, lane r polls rank r's slot) until all G records of this step have
//      arrived, and
//   4. writes the G records straight into mapped pinned host memory,
// so the host's one stream synchronisation of the step returns the gathered records: no H2D of
// the record, no NCCL launch, no separate D2H.  The host reduction is the same deterministic
// dbk_stats_reduce as the NCCL path, so every rank takes the same b_{t+1}.
//
// Slot reuse is safe by construction: step t uses parity t & 1; a rank can write parity t & 1
// again only at step t + 2, which needs every rank's step t + 1 record, pushed by a kernel that
// its stream runs after the same rank's step t kernel finished reading.
#include <chrono>
#include <cstring>
#include <new>
#include <vector>

#include "common.h"
#include "device_common.cuh"
#include "mailbox.h"

namespace dbk {
namespace {

constexpr int kSlot = 256;          // bytes per slot: seq (8 B) at 0, the record (128 B) at 128
constexpr int kMaxRanks = 32;       // one polling lane per rank

struct MboxParams {
    uint8_t *const *peers;          // [nranks] mailbox bases (own included), device-visible
    int nranks, rank;
    int64_t seq;                    // this exchange's sequence number (>= 1)
    const unsigned long long *stats;  // device record reduced by K4, or null: use `rec`
    int empty;                      // no decode launch this step: the empty record (O3)
    int64_t cap_pages, n_waiting;
    const int64_t *t0;              // step start stamp (globaltimer), or null: keep rec.step_ns
    dbk_stats rec;                  // by-value record (standalone exchange)
    dbk_stats *host_all;            // mapped pinned [nranks]
    int32_t *host_err;              // mapped pinned error flag
    int64_t timeout_ns;
};

__global__ void mbox_stamp_kernel(int64_t *t0) { t0[0] = static_cast<int64_t>(dev::globaltimer_ns()); }

__global__ void __launch_bounds__(32) mbox_exchange_kernel(const MboxParams p) {
    const int lane = threadIdx.x;
    const int parity = static_cast<int>(p.seq & 1);
    // 1. this rank's record, field `lane` (16 int64 fields)
    int64_t v = 0;
    if (lane < 16) {
        if (p.stats == nullptr) {
            v = reinterpret_cast<const int64_t *>(&p.rec)[lane];
        } else if (p.empty) {
            v = (lane == 5 || lane == 6) ? p.cap_pages : 0;
        } else {
            v = static_cast<int64_t>(p.stats[lane]);
        }
        if (lane == 14 && p.t0) v = static_cast<int64_t>(dev::globaltimer_ns()) - p.t0[0];
        if (lane == 15 && p.stats) v = p.n_waiting;
    }
    // 2. push into every rank's slot [parity][rank]: the record, then the sequence number
    for (int r = 0; r < p.nranks; ++r) {
        uint8_t *slot = p.peers[r] + (static_cast<size_t>(parity) * p.nranks + p.rank) * kSlot;
        if (lane < 16)
            asm volatile("st.relaxed.sys.global.s64 [%0], %1;" ::"l"(slot + 128 + 8 * lane), "l"(v) : "memory");
        __syncwarp();
        if (lane == 0) {
            asm volatile("fence.acq_rel.sys;" ::: "memory");
            asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(slot), "l"(p.seq) : "memory");
        }
    }
    // 3. wait for every rank's record of this step in the own mailbox (lane r polls rank r)
    uint8_t *own = p.peers[p.rank] + static_cast<size_t>(parity) * p.nranks * kSlot;
    int ok = 1;
    if (lane < p.nranks) {
        const uint64_t start = dev::globaltimer_ns();
        int64_t s = 0;
        for (;;) {
            asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(s) : "l"(own + lane * kSlot) : "memory");
            if (s == p.seq) break;
            if (dev::globaltimer_ns() - start > static_cast<uint64_t>(p.timeout_ns)) {
                ok = 0;
                break;
            }
            __nanosleep(64);
        }
    }
    ok = __all_sync(0xffffffffu, ok);
    if (!ok) {
        if (lane == 0) *reinterpret_cast<volatile int32_t *>(p.host_err) = 1;
        return;
    }
    // 4. the G records -> mapped host memory (rank order)
    for (int r = 0; r < p.nranks; ++r) {
        if (lane < 16) {
            int64_t x;
            asm volatile("ld.relaxed.sys.global.s64 %0, [%1];" : "=l"(x) : "l"(own + r * kSlot + 128 + 8 * lane) : "memory");
            reinterpret_cast<volatile int64_t *>(p.host_all + r)[lane] = x;
        }
    }
    __threadfence_system();
}

}  // namespace
}  // namespace dbk

struct dbk_mbox {
    int nranks = 1, rank = 0, device = 0;
    uint8_t *d_local = nullptr;          // own mailbox [2][nranks] slots
    uint8_t **d_peers = nullptr;         // device array of mailbox bases
    std::vector<void *> opened;          // IPC-opened peer mailboxes (to close)
    int64_t *d_t0 = nullptr;
    dbk_stats *h_all = nullptr, *d_h_all = nullptr;  // mapped pinned [nranks]
    int32_t *h_err = nullptr, *d_h_err = nullptr;
    int64_t seq = 0;
    bool ready = false;
    int64_t timeout_ns = 20'000'000'000LL;
};

namespace dbk {

dbk_status mbox_stamp(dbk_mbox *m, cudaStream_t s) {
    mbox_stamp_kernel<<<1, 1, 0, s>>>(m->d_t0);
    DBK_CUDA(cudaGetLastError());
    return DBK_OK;
}

dbk_status mbox_launch(dbk_mbox *m, const unsigned long long *d_stats, bool empty, int64_t cap_pages,
                       int64_t n_waiting, bool stamped, const dbk_stats *rec, cudaStream_t s) {
    if (!m->ready) return fail(DBK_EINVAL, "mailbox: not opened (dbk_mbox_open)");
    MboxParams p{};
    p.peers = m->d_peers;
    p.nranks = m->nranks;
    p.rank = m->rank;
    p.seq = ++m->seq;
    p.stats = d_stats;
    p.empty = empty ? 1 : 0;
    p.cap_pages = cap_pages;
    p.n_waiting = n_waiting;
    p.t0 = stamped ? m->d_t0 : nullptr;
    if (rec) p.rec = *rec;
    p.host_all = m->d_h_all;
    p.host_err = m->d_h_err;
    p.timeout_ns = m->timeout_ns;
    *m->h_err = 0;
    mbox_exchange_kernel<<<1, 32, 0, s>>>(p);
    DBK_CUDA(cudaGetLastError());
    return DBK_OK;
}

dbk_status mbox_collect(dbk_mbox *m, dbk_stats *all) {
    if (*reinterpret_cast<volatile int32_t *>(m->h_err))
        return fail(DBK_ECUDA, "mailbox exchange: not every rank's record arrived within %.0f s (seq %lld)",
                    m->timeout_ns / 1e9, static_cast<long long>(m->seq));
    std::memcpy(all, m->h_all, sizeof(dbk_stats) * m->nranks);
    return DBK_OK;
}

int32_t mbox_nranks(const dbk_mbox *m) { return m->nranks; }
int32_t mbox_rank(const dbk_mbox *m) { return m->rank; }

}  // namespace dbk

extern "C" {

dbk_status dbk_mbox_create(int32_t nranks, int32_t rank, int32_t device, void *handle_out_64, dbk_mbox **out) {
    if (!out || !handle_out_64 || nranks < 1 || nranks > dbk::kMaxRanks || rank < 0 || rank >= nranks)
        return dbk::fail(DBK_EINVAL, "mbox_create: bad arguments (1 <= nranks <= %d)", dbk::kMaxRanks);
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
    DBK_CUDA(cudaSetDevice(device));
    dbk_mbox *m = new (std::nothrow) dbk_mbox();
    if (!m) return dbk::fail(DBK_EINVAL, "out of host memory");
    m->nranks = nranks;
    m->rank = rank;
    m->device = device;
    const size_t bytes = 2ull * nranks * dbk::kSlot;
    cudaIpcMemHandle_t h;
    if (cudaMalloc(&m->d_local, bytes) != cudaSuccess || cudaMemset(m->d_local, 0, bytes) != cudaSuccess ||
        cudaMalloc(&m->d_peers, sizeof(uint8_t *) * nranks) != cudaSuccess ||
        cudaMalloc(&m->d_t0, sizeof(int64_t)) != cudaSuccess ||
        cudaHostAlloc(&m->h_all, sizeof(dbk_stats) * nranks, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void **>(&m->d_h_all), m->h_all, 0) != cudaSuccess ||
        cudaHostAlloc(&m->h_err, sizeof(int32_t), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void **>(&m->d_h_err), m->h_err, 0) != cudaSuccess ||
        cudaIpcGetMemHandle(&h, m->d_local) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
        const cudaError_t e = cudaGetLastError();
        dbk_mbox_destroy(m);
        return dbk::fail(DBK_ECUDA, "mbox_create: %s", cudaGetErrorString(e));
    }
    *m->h_err = 0;
    std::memcpy(handle_out_64, &h, sizeof h);
    *out = m;
    return DBK_OK;
}

dbk_status dbk_mbox_open(dbk_mbox *m, const void *handles) {
    if (!m || !handles) return dbk::fail(DBK_EINVAL, "mbox_open: null argument");
    if (m->ready) return dbk::fail(DBK_EINVAL, "mbox_open: already open");
    DBK_CUDA(cudaSetDevice(m->device));
    std::vector<uint8_t *> bases(static_cast<size_t>(m->nranks), nullptr);
    for (int r = 0; r < m->nranks; ++r) {
        if (r == m->rank) {
            bases[r] = m->d_local;
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const uint8_t *>(handles) + 64 * static_cast<size_t>(r), sizeof h);
        void *ptr = nullptr;
        const cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            cudaGetLastError();
            // nothing stays mapped: a failed open leaves the mailbox as created (retry-able)
            for (void *q : m->opened) cudaIpcCloseMemHandle(q);
            m->opened.clear();
            return dbk::fail(DBK_ECUDA, "mbox_open: cudaIpcOpenMemHandle(rank %d): %s", r, cudaGetErrorString(e));
        }
        m->opened.push_back(ptr);
        bases[r] = static_cast<uint8_t *>(ptr);
    }
    DBK_CUDA(cudaMemcpy(m->d_peers, bases.data(), sizeof(uint8_t *) * m->nranks, cudaMemcpyHostToDevice));
    m->ready = true;
    return DBK_OK;
}

dbk_status dbk_mbox_destroy(dbk_mbox *m) {
    if (!m) return DBK_OK;
    cudaSetDevice(m->device);
    cudaDeviceSynchronize();
    for (void *p : m->opened) cudaIpcCloseMemHandle(p);
    if (m->d_local) cudaFree(m->d_local);
    if (m->d_peers) cudaFree(m->d_peers);
    if (m->d_t0) cudaFree(m->d_t0);
    if (m->h_all) cudaFreeHost(m->h_all);
    if (m->h_err) cudaFreeHost(m->h_err);
    delete m;
    return DBK_OK;
}

dbk_status dbk_mbox_exchange(dbk_mbox *m, const dbk_stats *local, dbk_stats *all, dbk_stats *global, int32_t mode,
                             void *stream) {
    if (!m || !local || !all || !global) return dbk::fail(DBK_EINVAL, "mbox_exchange: null argument");
    DBK_CUDA(cudaSetDevice(m->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DBK_TRY(dbk::mbox_launch(m, nullptr, false, 0, 0, false, local, s));
    DBK_CUDA(cudaStreamSynchronize(s));
    DBK_TRY(dbk::mbox_collect(m, all));
    return dbk_stats_reduce(all, m->nranks, mode, global);
}

}  // extern "C"
