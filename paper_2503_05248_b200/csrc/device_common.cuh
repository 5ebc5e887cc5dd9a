// Device helpers shared by the decode kernels (K1 CUDA-core, K2 tensor-core): PTX wrappers
// for mbarriers / TMA, element conversions, the synthetic generator, the fused batch
// statistics (K4) and the CTA epilogue with the split-K merge (K3).  Internal to libdbk.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "kernels.cuh"

namespace dbk {
namespace dev {

constexpr int kP = 16;          // tokens per page
constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D TMA (bulk copy) global -> shared, completion counted on `bar`; the KV
// stream is read once per step, so it is marked evict-first in L2.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// ------------------------------------------------------------------ element types
template <typename T>
struct Elt;
template <>
struct Elt<__half> {
    __device__ static float2 to_f2(uint32_t u) {
        return __half22float2(*reinterpret_cast<const __half2 *>(&u));
    }
    __device__ static uint32_t from_f2(float a, float b) {
        __half2 h = __floats2half2_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    }
    __device__ static void store(void *p, float x) { *reinterpret_cast<__half *>(p) = __float2half_rn(x); }
};
template <>
struct Elt<__nv_bfloat16> {
    __device__ static float2 to_f2(uint32_t u) {
        return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u));
    }
    __device__ static uint32_t from_f2(float a, float b) {
        __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    }
    __device__ static void store(void *p, float x) {
        *reinterpret_cast<__nv_bfloat16 *>(p) = __float2bfloat16_rn(x);
    }
};

template <typename T>
__device__ __forceinline__ void unpack8(const uint4 &u, float f[8]) {
    float2 a = Elt<T>::to_f2(u.x), b = Elt<T>::to_f2(u.y), c = Elt<T>::to_f2(u.z),
           d = Elt<T>::to_f2(u.w);
    f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
    f[4] = c.x; f[5] = c.y; f[6] = d.x; f[7] = d.y;
}
template <typename T>
__device__ __forceinline__ uint4 pack8(const float f[8]) {
    return make_uint4(Elt<T>::from_f2(f[0], f[1]), Elt<T>::from_f2(f[2], f[3]),
                      Elt<T>::from_f2(f[4], f[5]), Elt<T>::from_f2(f[6], f[7]));
}

__device__ __forceinline__ void store_out(void *out, size_t idx, int dtype, float x) {
    if (dtype == 2)
        reinterpret_cast<float *>(out)[idx] = x;
    else if (dtype == 0)
        reinterpret_cast<__half *>(out)[idx] = __float2half_rn(x);
    else
        reinterpret_cast<__nv_bfloat16 *>(out)[idx] = __float2bfloat16_rn(x);
}

// Two consecutive outputs (fp32 / fp16 / bf16) from registers, one store.
__device__ __forceinline__ void store2_out(void *out, size_t elem, int dtype, float a, float b) {
    if (dtype == 2) {
        *reinterpret_cast<float2 *>(reinterpret_cast<float *>(out) + elem) = make_float2(a, b);
    } else if (dtype == 0) {
        *reinterpret_cast<uint32_t *>(reinterpret_cast<__half *>(out) + elem) = Elt<__half>::from_f2(a, b);
    } else {
        *reinterpret_cast<uint32_t *>(reinterpret_cast<__nv_bfloat16 *>(out) + elem) =
            Elt<__nv_bfloat16>::from_f2(a, b);
    }
}

// ------------------------------------------------------------------ synthetic generator
// Same definition as synth/hashgen.py (input generation only).
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
// synth_key = synth_key2(synth_key1(seed, kind, req), pos, layer, head, g): kernels that generate
// many values of one (kind, request) hoist the first hash out of their loops
__device__ __forceinline__ uint64_t synth_key1(uint64_t seed, int kind, int64_t req) {
    return splitmix64(seed ^ (static_cast<uint64_t>(kind) << 56) ^ static_cast<uint64_t>(req));
}
__device__ __forceinline__ uint64_t synth_key2(uint64_t k1, int pos, int layer, int head, int g) {
    uint64_t w = (static_cast<uint64_t>(static_cast<uint32_t>(pos)) << 32) |
                 (static_cast<uint64_t>(layer) << 20) | (static_cast<uint64_t>(head) << 8) |
                 static_cast<uint64_t>(g);
    return splitmix64(k1 ^ w);
}
__device__ __forceinline__ uint64_t synth_key(uint64_t seed, int kind, int64_t req, int pos,
                                              int layer, int head, int g) {
    return synth_key2(synth_key1(seed, kind, req), pos, layer, head, g);
}
__device__ __forceinline__ void synth_vals(uint64_t key, float scale, float f[8]) {
#pragma unroll
    for (int b = 0; b < 8; ++b) f[b] = static_cast<float>(static_cast<int>((key >> (8 * b)) & 0xFF) - 128) * scale;
}

// ------------------------------------------------------------------ K4: fused batch statistics
// One warp per request (the CTA holding chunk 0 of kv-head 0).  Integer atomics:
// order-independent, bit-exact with the oracle O3.
__device__ __forceinline__ void batch_stats_warp(const DecodeParams &p, const ReqMeta &rm, int lane) {
    const int32_t *row = p.block_table + static_cast<size_t>(rm.slot) * p.bt_stride;
    int cnt = 0;
    for (int b = 0; b < p.max_pages_per_req; b += 32) {
        const bool v = (b + lane < p.max_pages_per_req) && __ldg(row + b + lane) >= 0;
        cnt += __popc(__ballot_sync(kFull, v));
    }
    if (lane == 0) {
        unsigned long long *st = p.stats;
        const unsigned long long c = static_cast<unsigned long long>(rm.ctx);
        atomicAdd(st + 0, 1ull);
        atomicAdd(st + 1, c);
        atomicAdd(st + 2, c * c);
        atomicMax(st + 3, c);
        atomicAdd(st + 4, static_cast<unsigned long long>(cnt));
        if (cnt != (rm.ctx + kP - 1) / kP) atomicAdd(st + 8, 1ull);
        if (rm.ctx == rm.l_in + rm.l_out) {
            const unsigned long long a = rm.l_in, b = rm.l_out;
            atomicAdd(st + 9, 1ull);
            atomicAdd(st + 10, a);
            atomicAdd(st + 11, a * a);
            atomicAdd(st + 12, b);
            atomicAdd(st + 13, b * b);
        }
        __threadfence();
        const int done = atomicAdd(p.stats_done, 1);
        if (done == p.n - 1) {  // last request: derived fields against the cap
            __threadfence();
            const long long pages = static_cast<long long>(atomicAdd(st + 4, 0ull));
            st[5] = static_cast<unsigned long long>(p.cap_pages);
            st[6] = static_cast<unsigned long long>(p.cap_pages - pages);
            st[7] = pages > p.cap_pages ? 1ull : 0ull;
            *p.stats_done = 0;
        }
    }
}

// ------------------------------------------------------------------ persistent warp tasks
// A task is (work item, kv head) = up to 32 pages of one request for one kv head, served
// by ONE warp from start to end (no CTA-wide barriers anywhere).  Tasks are handed out by
// an atomic counter in the order of the work list (the host sorts it longest-first).  A
// warp streams the concatenation of its current and next task's pages through its ring,
// so the DRAM stream does not pause at task boundaries (epilogue, q load, metadata).
struct Task {
    int task;        // >= n_tasks: no task
    int g;           // kv head
    int l;           // layer within the launch
    ItemMeta it;     // the work item (request chunk)
    int phys_lane;   // physical page of the chunk's k-th page, held by lane k (k < 32)
    int phys_lane2;  // ... of page 32 + k
};

// Physical page of the task's j-th page (j warp-uniform, j < 64).
__device__ __forceinline__ int page_of(const Task &t, int j) {
    return __shfl_sync(kFull, j < 32 ? t.phys_lane : t.phys_lane2, j & 31);
}

// ------------------------------------------------------------------ task timeline (measurement)
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// One record per finished task when p.trace is set (DBK_TRACE_TASKS): start / end (globaltimer
// ns), SM id | launch sequence, task | pages.  Lane 0 only; a no-op in production.
__device__ __forceinline__ void trace_task(const DecodeParams &p, uint64_t t0, int task, int pages, int lane) {
    if (p.trace == nullptr || lane != 0) return;
    const uint64_t t1 = globaltimer_ns();
    uint32_t smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    const unsigned long long k = atomicAdd(p.trace, 1ull);
    if (k >= static_cast<unsigned long long>(p.trace_cap)) return;
    unsigned long long *r = p.trace + 4 * (k + 1);
    r[0] = t0;
    r[1] = t1;
    r[2] = (static_cast<uint64_t>(smid) << 32) | static_cast<uint32_t>(p.trace_seq);
    r[3] = (static_cast<uint64_t>(static_cast<uint32_t>(task)) << 32) | static_cast<uint32_t>(pages);
}

// The item record, then its page ids straight from the device block table (the tables the
// allocator's deltas keep current; the single source of truth for every kernel that addresses
// the pool): issued one task ahead of use, so the dependent second load overlaps the current
// task's page stream (the ring holds STAGES tiles in flight meanwhile).
__device__ __forceinline__ Task load_task(const DecodeParams &p, int task, int lane) {
    Task t;
    t.task = task;
    t.phys_lane = 0;
    t.phys_lane2 = 0;
    t.g = 0;
    t.l = 0;
    if (task >= p.n_tasks) {
        t.task = p.n_tasks;
        t.it = ItemMeta{0, 0, 0, 0, 1, 0, 1, 0};
        return t;
    }
    // layer-major: the queue sweeps the layers one after the other (each longest-first), so the
    // pages in flight stay within ~one layer's slice of the pool (TLB reach, DRAM locality)
    const int per_layer = p.n_items * p.kv_heads;
    t.l = task / per_layer;
    const int ih = task - t.l * per_layer;
    const int item = ih / p.kv_heads;
    t.g = ih - item * p.kv_heads;
    const int4 *im = reinterpret_cast<const int4 *>(p.items + item);
    const int4 a = __ldg(im), b = __ldg(im + 1);
    t.it = ItemMeta{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    const int32_t *row = p.block_table + static_cast<size_t>(t.it.slot) * p.bt_stride + t.it.pg0;
    t.phys_lane = lane < t.it.n ? __ldg(row + lane) : 0;
    t.phys_lane2 = lane + 32 < t.it.n ? __ldg(row + 32 + lane) : 0;
    return t;
}

// Task assignment (the host sorts the work list longest-first): tasks are claimed from an
// atomic counter -- two at the start (the current one and the next, whose pages the ring
// streams across the boundary), then each further one only when the warp nears the end of its
// current task.  A warp never holds more than one unstarted task beyond the next: claiming
// three or four ahead (round 1) left a third of the warps without work when there are ~2
// tasks per warp (70B TP shards, task trace); static assignment instead stalls on the CTAs
// that become resident late under programmatic dependent launch.
struct TaskPlan {
    int nw;    // warps of the grid
};
__device__ __forceinline__ TaskPlan task_plan(const DecodeParams &, int nw) {
    TaskPlan t;
    t.nw = nw;
    return t;
}
// lane 0 claims the next task; the value is valid in lane 0 only (broadcast at use, so the
// atomic's latency hides behind the current task's pages)
__device__ __forceinline__ int task_claim(const DecodeParams &p, const TaskPlan &, int lane) {
    return lane == 0 ? atomicAdd(p.task_counter, 1) : 0;
}

// Programmatic dependent launch, released without blocking: the NEXT decode grid reuses the
// scratch parity (task counter, split-K workspace and arrival counters) of the PREVIOUS one,
// so this grid lets it launch once the previous grid's last warp has reset that scratch and
// published its sequence number in done_seq.  Polled at task boundaries (a warp never stalls
// for the previous grid while it has work); every grid's CTAs trigger or exit, and they exit
// only after griddepcontrol.wait (task_exit), so the chain is safe either way.
__device__ __forceinline__ bool pdl_try_release(const DecodeParams &p, int lane) {
    int ok = 0;
    if (lane == 0) {
        int v;
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p.done_seq) : "memory");
        ok = v >= p.seq - 1;
    }
    ok = __shfl_sync(kFull, ok, 0);
    if (ok) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    return ok != 0;
}

// A warp with no task left.  It first waits for the PREVIOUS decode grid to complete (a no-op
// without the launch attribute) -- a CTA's exit also releases the next grid, which must find
// the previous grid's scratch reset -- then counts itself out; the last warp resets the task
// counters and publishes this grid's sequence number (release) for the next grid's trigger.
__device__ __forceinline__ void task_exit(const DecodeParams &p, int lane, int total_warps) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (lane == 0) {
        __threadfence();
        const int e = atomicAdd(p.task_counter + 1, 1);
        if (e == total_warps - 1) {
            p.task_counter[0] = 0;
            p.task_counter[1] = 0;
            __threadfence();
            asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p.done_seq), "r"(p.seq) : "memory");
        }
    }
}

// Split-K bookkeeping after a warp wrote its chunk's partial: returns true in every lane
// of the warp whose chunk arrived last for (request, kv head); that warp merges.
// ci = the (layer, request, kv head) counter index.
__device__ __forceinline__ bool split_arrive_last(const DecodeParams &p, int ci, int nchunks, int lane) {
    // The warp's partial stores happen-before lane 0's acq_rel RMW (__syncwarp + cumulativity),
    // which releases them at gpu scope; the last arriver's acquire makes every chunk's partial
    // visible (read with ld.global.cg, which bypasses L1) -- no full fences / L1 invalidation.
    __syncwarp();
    int last = 0;
    if (lane == 0) {
        int prev;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                     : "=r"(prev)
                     : "l"(p.counters + ci)
                     : "memory");
        last = prev == nchunks - 1;
    }
    last = __shfl_sync(kFull, last, 0);
    return last != 0;
}

// The last warp merges the chunks' (m, l, O) of q-heads g*GQ .. g*GQ+GQ-1 (workspace rows
// wbase .. wbase+nchunks-1) and writes out at element obase + h*D (obase = the layer's and
// request's output row); ci = the arrival counter it resets.
template <int GQ, int D>
__device__ __forceinline__ void split_merge_warp(const DecodeParams &p, int wbase, int nchunks, size_t obase,
                                                 int g, int ci, int lane) {
    // Online merge over the chunks: lane owns dims lane*PL .. lane*PL+PL-1 of all GQ heads;
    // each chunk's loads (GQ (m, l) pairs + GQ x PL partial sums) are independent of the
    // running state, so they are in flight together.
    constexpr int PL = D / 32;
    float M[GQ], L[GQ], acc[GQ][PL];
#pragma unroll
    for (int t = 0; t < GQ; ++t) {
        M[t] = -INFINITY;
        L[t] = 0.f;
#pragma unroll
        for (int e = 0; e < PL; ++e) acc[t][e] = 0.f;
    }
    for (int x = 0; x < nchunks; ++x) {
        const size_t w0 = static_cast<size_t>(wbase + x) * p.q_heads + g * GQ;
        float2 ml[GQ];
        float v[GQ][PL];
#pragma unroll
        for (int t = 0; t < GQ; ++t) {
            ml[t] = __ldcg(&p.ws_ml[w0 + t]);  // same address in every lane: one broadcast load
            const float *src = p.ws_o + (w0 + t) * D + lane * PL;
#pragma unroll
            for (int e = 0; e < PL; ++e) v[t][e] = __ldcg(src + e);
        }
#pragma unroll
        for (int t = 0; t < GQ; ++t) {
            if (ml[t].x == -INFINITY) continue;
            const float Mn = fmaxf(M[t], ml[t].x);
            const float a = (M[t] == -INFINITY) ? 0.f : exp2f(M[t] - Mn), b = exp2f(ml[t].x - Mn);
            L[t] = L[t] * a + ml[t].y * b;
#pragma unroll
            for (int e = 0; e < PL; ++e) acc[t][e] = acc[t][e] * a + v[t][e] * b;
            M[t] = Mn;
        }
    }
#pragma unroll
    for (int t = 0; t < GQ; ++t) {
        const float inv = 1.f / L[t];
        const size_t ob = obase + static_cast<size_t>(g * GQ + t) * D + lane * PL;
#pragma unroll
        for (int e = 0; e < PL; e += 2) store2_out(p.out, ob + e, p.out_dtype, acc[t][e] * inv, acc[t][e + 1] * inv);
    }
    if (lane == 0) p.counters[ci] = 0;
}


// 8 consecutive outputs (fp32 / fp16 / bf16) from registers.
__device__ __forceinline__ void store8_out(void *out, size_t elem, int dtype, const float f[8]) {
    if (dtype == 2) {
        float4 *o = reinterpret_cast<float4 *>(reinterpret_cast<float *>(out) + elem);
        o[0] = make_float4(f[0], f[1], f[2], f[3]);
        o[1] = make_float4(f[4], f[5], f[6], f[7]);
    } else if (dtype == 0) {
        *reinterpret_cast<uint4 *>(reinterpret_cast<__half *>(out) + elem) = pack8<__half>(f);
    } else {
        *reinterpret_cast<uint4 *>(reinterpret_cast<__nv_bfloat16 *>(out) + elem) = pack8<__nv_bfloat16>(f);
    }
}

}  // namespace dev
}  // namespace dbk
