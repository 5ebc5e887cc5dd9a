// K1 (+K3, K4): paged decode attention on the CUDA cores -- MHA, and the GQA fallback.
//
// Persistent warps: the grid is SMs x resident CTAs; every warp takes tasks = (work item
// = (request, chunk of <= 32 pages), kv head g) from an atomic counter and serves the task's
// GQ q-heads by itself.  A warp streams the pages of its current and next task through
// its own STAGES-deep ring of (K,V) page tiles [2][16][D] (8 KiB at d = 128), each filled by
// ONE 1-D TMA bulk copy (cp.async.bulk, L2 evict-first) completing on an mbarrier; no
// CTA-wide barrier exists, so one warp's task epilogue never stalls the others' streams.
// Lane layout: LPT = D/8 lanes cover one token row (8 dims per lane, one conflict-free
// 16-byte ld.shared), TG = 32/LPT token groups; group grp owns tokens kk*TG + grp of each
// page with its own online-softmax state (log2 units); the groups merge with shuffles at
// the end of the task.  Chunks of one request merge through the split-K workspace, done
// by the warp that arrives last (K3).  The batch statistics (K4) ride in the layer-0
// launch: the warp that owns (request, chunk 0, kv head 0) reduces that request's row.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "device_common.cuh"
#include "kernels.cuh"

namespace dbk {
namespace {
using namespace dev;

template <typename T, int D, int GQ, int WARPS, int STAGES>
__global__ void __launch_bounds__(WARPS * 32)
decode_kernel(const DecodeParams p) {
    constexpr int LPT = D / 8;
    constexpr int TG = 32 / LPT;
    constexpr int KI = kP / TG;  // tokens per group per page (= LPT / 2)
    constexpr int TILE = 2 * kP * D * static_cast<int>(sizeof(T));
    static_assert(KI * 2 == LPT, "lane layout");

    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[WARPS][STAGES];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / LPT, dl = lane % LPT;
    uint8_t *wbuf = smem + warp * STAGES * TILE;
    const uint64_t pol = evict_first_policy();

    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[warp][s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    // launched right behind the producer of q / the step's K/V (the model's QKV GEMM): the CTA
    // is resident and set up by now; the data is not
    if (p.pdl == 2) asm volatile("griddepcontrol.wait;" ::: "memory");
    const TaskPlan plan = task_plan(p, static_cast<int>(gridDim.x) * WARPS);
    int f0 = task_claim(p, plan, lane), f1 = task_claim(p, plan, lane);
    f0 = __shfl_sync(kFull, f0, 0);
    f1 = __shfl_sync(kFull, f1, 0);
    Task cur = load_task(p, f0, lane), nxt = load_task(p, f1, lane);
    bool released = pdl_try_release(p, lane), drained = false;
    uint32_t seq_iss = 0, cur_start = 0;
    // keep STAGES tiles in flight along this warp's page sequence (current, then next task)
    auto top_up = [&](uint32_t seq_cons) {
        while (seq_iss < seq_cons + STAGES) {
            const int j = static_cast<int>(seq_iss - cur_start);
            int ph, g, lay, valid;
            if (j < cur.it.n) {
                ph = page_of(cur, j);
                g = cur.g;
                lay = cur.l;
                valid = cur.it.ctx - (cur.it.pg0 + j) * kP;
            } else if (j - cur.it.n < nxt.it.n) {
                ph = page_of(nxt, j - cur.it.n);
                g = nxt.g;
                lay = nxt.l;
                valid = nxt.it.ctx - (nxt.it.pg0 + j - cur.it.n) * kP;
            } else {
                break;
            }
            if (lane == 0) {
                const int s = seq_iss % STAGES;
                const uint8_t *src = p.kv_layer + static_cast<size_t>(lay) * p.layer_stride +
                                     static_cast<size_t>(g) * TILE + static_cast<size_t>(ph) * p.page_stride;
                fence_proxy_async();
                if (valid >= kP) {
                    mbar_expect_tx(&bars[warp][s], TILE);
                    bulk_g2s(wbuf + s * TILE, src, TILE, &bars[warp][s], pol);
                } else {
                    // a request's last, partly filled page: only its `valid` K rows and V rows
                    // (the slots past ctx are never read: their scores are masked, their V rows
                    // skipped), so no page padding crosses HBM -- ~2 % of the KV stream at the
                    // 7B trace's mean context
                    const uint32_t half = static_cast<uint32_t>(valid) * D * sizeof(T);
                    mbar_expect_tx(&bars[warp][s], 2 * half);
                    bulk_g2s(wbuf + s * TILE, src, half, &bars[warp][s], pol);
                    bulk_g2s(wbuf + s * TILE + TILE / 2, src + TILE / 2, half, &bars[warp][s], pol);
                }
            }
            ++seq_iss;
        }
    };
    top_up(0);
    // raw q of a task (lane holds dims dl*8 .. dl*8+7 of each q-head of the group)
    auto load_q = [&](const Task &t, uint4 (&qr)[GQ]) {
#pragma unroll
        for (int h = 0; h < GQ; ++h)
            qr[h] = __ldg(reinterpret_cast<const uint4 *>(
                reinterpret_cast<const T *>(p.q) + t.l * p.q_layer_stride +
                (static_cast<size_t>(t.it.i) * p.q_heads + t.g * GQ + h) * D + dl * 8));
    };
    uint4 qraw[GQ];
    load_q(cur, qraw);

    while (cur.task < p.n_tasks) {
        if (!released) released = pdl_try_release(p, lane);
        // the q of `nxt` (its metadata arrived during the previous task) is requested now and
        // used when it becomes current, so its latency hides behind this task
        uint4 qnext[GQ];
        load_q(nxt, qnext);
        const int i = cur.it.i, c = cur.it.c, g = cur.g, lay = cur.l;
        const uint64_t t_task0 = p.trace ? globaltimer_ns() : 0;
        if (p.fuse_stats && c == 0 && g == 0 && lay == 0) batch_stats_warp(p, p.req[i], lane);

        float q[GQ][8];  // pre-scaled to log2 units
#pragma unroll
        for (int t = 0; t < GQ; ++t) {
            unpack8<T>(qraw[t], q[t]);
#pragma unroll
            for (int e = 0; e < 8; ++e) q[t][e] *= p.scale_log2;
        }
        float m[GQ], l[GQ], acc[GQ][8];
#pragma unroll
        for (int t = 0; t < GQ; ++t) {
            m[t] = -INFINITY;
            l[t] = 0.f;
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[t][e] = 0.f;
        }

        int pend = 0;
        bool claimed = false;
        for (int k = 0; k < cur.it.n; ++k) {
            if (!claimed && k + 3 >= cur.it.n) {  // the task after `nxt`, three pages ahead of need
                if (!drained) pend = task_claim(p, plan, lane);
                claimed = true;
            }
            const uint32_t jseq = cur_start + k;
            const int s = jseq % STAGES;
            mbar_wait(&bars[warp][s], (jseq / STAGES) & 1);
            const T *Kt = reinterpret_cast<const T *>(wbuf + s * TILE);
            const T *Vt = Kt + kP * D;
            const int valid = cur.it.ctx - (cur.it.pg0 + k) * kP;  // >= 1; < 16 only on the last page
#pragma unroll
            for (int t = 0; t < GQ; ++t) {
                // scores: partial dot products over this lane's 8 dims for its KI tokens
                float v[KI];
#pragma unroll
                for (int kk = 0; kk < KI; ++kk) {
                    float kf[8];
                    unpack8<T>(*reinterpret_cast<const uint4 *>(Kt + (kk * TG + grp) * D + dl * 8), kf);
                    float a = 0.f;
#pragma unroll
                    for (int e = 0; e < 8; ++e) a = fmaf(q[t][e], kf[e], a);
                    v[kk] = a;
                }
                // transpose-reduce across the LPT lanes of the group: afterwards lane dl holds the
                // full score of token (dl >> 1) * TG + grp
#pragma unroll
                for (int o = LPT / 2, cnt = KI; o >= 1; o >>= 1) {
                    const bool upper = (dl & o) != 0;
                    if (cnt > 1) {
                        const int half = cnt / 2;
#pragma unroll
                        for (int x = 0; x < half; ++x) {
                            const float send = upper ? v[x] : v[x + half];
                            const float keep = upper ? v[x + half] : v[x];
                            v[x] = keep + __shfl_xor_sync(kFull, send, o);
                        }
                        cnt = half;
                    } else {
                        v[0] += __shfl_xor_sync(kFull, v[0], o);
                    }
                }
                float sc = v[0];
                if ((dl >> 1) * TG + grp >= valid) sc = -INFINITY;
                float mx = sc;
#pragma unroll
                for (int o = LPT / 2; o >= 2; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
                const float m_new = fmaxf(m[t], mx);
                const float alpha = (m[t] == -INFINITY) ? 0.f : exp2f(m[t] - m_new);
                const float pme = (sc == -INFINITY) ? 0.f : exp2f(sc - m_new);
                float pv[KI];
                float psum = 0.f;
#pragma unroll
                for (int kk = 0; kk < KI; ++kk) {
                    pv[kk] = __shfl_sync(kFull, pme, (lane & ~(LPT - 1)) + 2 * kk);
                    psum += pv[kk];
                }
                m[t] = m_new;
                l[t] = l[t] * alpha + psum;
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[t][e] *= alpha;
                if (valid >= kP) {
#pragma unroll
                    for (int kk = 0; kk < KI; ++kk) {
                        float vf[8];
                        unpack8<T>(*reinterpret_cast<const uint4 *>(Vt + (kk * TG + grp) * D + dl * 8), vf);
#pragma unroll
                        for (int e = 0; e < 8; ++e) acc[t][e] = fmaf(pv[kk], vf[e], acc[t][e]);
                    }
                } else {  // last page: slots >= valid were never written for this request
#pragma unroll
                    for (int kk = 0; kk < KI; ++kk) {
                        if (kk * TG + grp < valid) {
                            float vf[8];
                            unpack8<T>(*reinterpret_cast<const uint4 *>(Vt + (kk * TG + grp) * D + dl * 8), vf);
#pragma unroll
                            for (int e = 0; e < 8; ++e) acc[t][e] = fmaf(pv[kk], vf[e], acc[t][e]);
                        }
                    }
                }
            }
            __syncwarp();
            top_up(jseq + 1);
        }

        // ---- end of task: merge the TG token groups with shuffles, then store or split-K
        const bool split = cur.it.nchunks > 1;
        const size_t obase = lay * p.out_layer_stride + static_cast<size_t>(i) * p.q_heads * D;
        const int wb = lay * p.n_ws_rows + cur.it.chunk_base, ci = (lay * p.n + i) * p.kv_heads + g;
        const int wi = wb + c;
#pragma unroll
        for (int t = 0; t < GQ; ++t) {
            float M = m[t];
#pragma unroll
            for (int o = LPT; o < 32; o <<= 1) M = fmaxf(M, __shfl_xor_sync(kFull, M, o));
            const float f = (m[t] == -INFINITY) ? 0.f : exp2f(m[t] - M);
            float L = l[t] * f, a[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) a[e] = acc[t][e] * f;
#pragma unroll
            for (int o = LPT; o < 32; o <<= 1) {
                L += __shfl_xor_sync(kFull, L, o);
#pragma unroll
                for (int e = 0; e < 8; ++e) a[e] += __shfl_xor_sync(kFull, a[e], o);
            }
            const int h = g * GQ + t;
            if (grp == 0) {
                if (!split) {
                    const float inv = 1.f / L;
#pragma unroll
                    for (int e = 0; e < 8; ++e) a[e] *= inv;
                    store8_out(p.out, obase + static_cast<size_t>(h) * D + dl * 8, p.out_dtype, a);
                } else {
                    float4 *w = reinterpret_cast<float4 *>(p.ws_o + (static_cast<size_t>(wi) * p.q_heads + h) * D + dl * 8);
                    w[0] = make_float4(a[0], a[1], a[2], a[3]);
                    w[1] = make_float4(a[4], a[5], a[6], a[7]);
                    if (dl == 0) p.ws_ml[static_cast<size_t>(wi) * p.q_heads + h] = make_float2(M, L);
                }
            }
        }
        if (split && split_arrive_last(p, ci, cur.it.nchunks, lane))
            split_merge_warp<GQ, D>(p, wb, cur.it.nchunks, obase, g, ci, lane);
        trace_task(p, t_task0, cur.task, cur.it.n, lane);

        // the claimed task's metadata: it becomes `nxt` (its pages join the ring behind cur's)
        const int nn = drained ? p.n_tasks : __shfl_sync(kFull, pend, 0);
        drained = nn >= p.n_tasks;
        const Task nnx = load_task(p, nn, lane);
        cur_start += cur.it.n;
        cur = nxt;
        nxt = nnx;
#pragma unroll
        for (int t = 0; t < GQ; ++t) qraw[t] = qnext[t];
        if (cur.task >= p.n_tasks && nxt.task < p.n_tasks) {  // no static second task: the claim is next
            cur = nxt;
            nxt = load_task(p, p.n_tasks, lane);
            load_q(cur, qraw);
        }
        top_up(cur_start);
    }
    task_exit(p, lane, static_cast<int>(gridDim.x) * WARPS);
}

template <int D>
constexpr int stages_for() { return D == 128 ? 3 : 5; }
constexpr int kWarps = 4;

template <typename T, int D>
constexpr size_t decode_smem() {
    return static_cast<size_t>(kWarps) * stages_for<D>() * 2 * kP * D * sizeof(T);
}

template <typename T, int D, int GQ>
cudaError_t launch_t(const DecodeParams &p, int ctas, cudaStream_t s) {
    auto kern = decode_kernel<T, D, GQ, kWarps, stages_for<D>()>;
    constexpr size_t smem = decode_smem<T, D>();
    static bool configured = false;  // per instantiation
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    return launch_kernel(kern, dim3(ctas), dim3(kWarps * 32), smem, s, p.pdl != 0, p);
}

template <typename T, int D, int GQ>
int occ_t() {
    auto kern = decode_kernel<T, D, GQ, kWarps, stages_for<D>()>;
    constexpr size_t smem = decode_smem<T, D>();
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kWarps * 32, smem) != cudaSuccess) n = 1;
    return n > 0 ? n : 1;
}

template <typename T, int D>
cudaError_t by_group(const DecodeParams &p, int group, int ctas, cudaStream_t s) {
    switch (group) {
        case 1: return launch_t<T, D, 1>(p, ctas, s);
        case 2: return launch_t<T, D, 2>(p, ctas, s);
        case 4: return launch_t<T, D, 4>(p, ctas, s);
        case 8: return launch_t<T, D, 8>(p, ctas, s);
        default: return cudaErrorInvalidValue;
    }
}
template <typename T, int D>
int occ_by_group(int group) {
    switch (group) {
        case 1: return occ_t<T, D, 1>();
        case 2: return occ_t<T, D, 2>();
        case 4: return occ_t<T, D, 4>();
        case 8: return occ_t<T, D, 8>();
        default: return 1;
    }
}

}  // namespace

cudaError_t launch_decode(const DecodeParams &p, int kv_dtype, int head_dim, int group, int ctas,
                          const GqaMaps *maps, cudaStream_t s) {
    if (p.n_tasks <= 0) return cudaSuccess;
    if (maps && group >= 2) return launch_decode_gqa(p, kv_dtype, head_dim, group, ctas, *maps, s);
    if (kv_dtype == 0) {
        if (head_dim == 128) return by_group<__half, 128>(p, group, ctas, s);
        if (head_dim == 64) return by_group<__half, 64>(p, group, ctas, s);
    } else {
        if (head_dim == 128) return by_group<__nv_bfloat16, 128>(p, group, ctas, s);
        if (head_dim == 64) return by_group<__nv_bfloat16, 64>(p, group, ctas, s);
    }
    return cudaErrorInvalidValue;
}

int decode_ctas_per_sm(int kv_dtype, int head_dim, int group) {
    if (kv_dtype == 0) return head_dim == 128 ? occ_by_group<__half, 128>(group) : occ_by_group<__half, 64>(group);
    return head_dim == 128 ? occ_by_group<__nv_bfloat16, 128>(group) : occ_by_group<__nv_bfloat16, 64>(group);
}

}  // namespace dbk
