// K2: paged decode attention for grouped-query attention on the tensor cores (sm_100a).
//
// With GQA the GQ = q_heads/kv_heads query heads of a group share each K/V page, so the
// page is a real dense contraction: S = Q_g K^T (GQ x 16 tokens x d) and O_g += P V
// (GQ x d x 16 tokens) -- 8 flop/B at GQ = 8, more than the CUDA cores retire at HBM speed
// (SURVEY.md §7 "GQA is ALU-bound on CUDA cores").  Each page tile is fetched by 2-D TMA
// (cp.async.bulk.tensor) through a pool-wide tensor map with the 128-byte swizzle, so the
// ldmatrix fragment loads are bank-conflict free, and consumed by warp-level
// mma.sync.m16n8k16 (rows = the group's q-heads, padded to 16; fp32 accumulate).  The S
// accumulator fragment is re-used in registers as the A operand of P V.  bf16 KV keeps P
// to ~16 bits by splitting it into bf16 hi + lo parts (two MMAs); fp16 KV uses fp16 P
// (11 bits) -- both well inside the 2e-3 bar (R23).  Work decomposition
// (persistent warps, one task = (request chunk, kv head) per warp, rings that stream across
// task boundaries), the fused statistics and the split-K merge are the same as K1.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "device_common.cuh"
#include "kernels.cuh"

namespace dbk {
namespace {
using namespace dev;

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// One (page, kv head) tile through the 5-D view {64, 16 tokens, d/64 halves, K|V, tile}: the
// whole 2 x 16 x d tile in one TMA, landing as [K|V][half][token][64] with the 128B swizzle.
__device__ __forceinline__ void tma_load_tile5(void *dst, const CUtensorMap *map, int tile, uint64_t *bar,
                                               uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %2, %2, %2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(tile), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t r[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t r[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
// D(16x8) += A(16x16) B(16x8); A rows 8..15 are zero padding (a1 = a3 = 0).
template <typename T>
__device__ __forceinline__ void mma_pad(float d[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
    if constexpr (std::is_same<T, __half>::value) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
    } else {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
    }
}

constexpr int kBox = 16 * 128;  // one TMA box: 16 rows x 64 elements (128 B), 128B-swizzled
constexpr int kPartRows = 4;    // rows per box of the partial-page map (GqaMaps::half)

template <typename T, int D, int GQ, int WARPS, int STAGES>
__global__ void __launch_bounds__(WARPS * 32)
decode_gqa_kernel(const DecodeParams p, const __grid_constant__ GqaMaps tmap) {
    constexpr int NBOX = D / 64;            // boxes per K (or V) tile of one page
    constexpr int STAGE = 2 * NBOX * kBox;  // K boxes, then V boxes
    constexpr int KSTEPS = D / 16;
    constexpr int NT = D / 8;               // n-tiles of the output
    constexpr bool kBF16 = std::is_same<T, __nv_bfloat16>::value;
    static_assert(GQ >= 2 && GQ <= 8, "group size");

    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bars[WARPS][STAGES];
    // 128B swizzle atoms need 1024-byte aligned destinations
    const uint32_t raw_off = smem_u32(smem_raw);
    uint8_t *smem = smem_raw + ((1024u - (raw_off & 1023u)) & 1023u);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gq = lane >> 2, cq = lane & 3;   // mma fragment row (q-head) / column pair
    const int mtx = lane >> 3, mr = lane & 7;  // ldmatrix: this lane addresses row mr of matrix mtx
    uint8_t *wbuf = smem + warp * STAGES * STAGE;
    const uint64_t pol = evict_first_policy();
    // row of the pool-wide tensor map: [layer][page][kv_head][K|V][16 tokens] x D elements

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
                fence_proxy_async();
                const int64_t row_layer = static_cast<int64_t>(p.layer + lay) * p.cap_pages;
                const int tile = static_cast<int>((row_layer + ph) * p.kv_heads + g);
                if (valid <= kP - kPartRows && p.half_boxes) {
                    // a request's last, partly filled page: only its first ceil(valid / 4) x 4 K
                    // rows and V rows (4-row boxes of a second tensor map; the 128B swizzle is a
                    // function of the shared-memory address, so each box lands where the full
                    // tile would put those rows), so page padding stays off the HBM stream; rows
                    // >= valid are masked (K) and zeroed (V) below
                    const int nb = (valid + kPartRows - 1) / kPartRows;
                    mbar_expect_tx(&bars[warp][s], 2 * NBOX * nb * kPartRows * 128);
#pragma unroll
                    for (int kv = 0; kv < 2; ++kv)
#pragma unroll
                        for (int b = 0; b < NBOX; ++b)
                            for (int r = 0; r < nb; ++r)
                                tma_load_2d(wbuf + s * STAGE + (kv * NBOX + b) * kBox + r * kPartRows * 128, &tmap.half,
                                            b * 64, tile * 32 + kv * 16 + r * kPartRows, &bars[warp][s], pol);
                } else if (p.tma_rank == 5) {
                    mbar_expect_tx(&bars[warp][s], STAGE);
                    tma_load_tile5(wbuf + s * STAGE, &tmap.full, tile, &bars[warp][s], pol);
                } else {
                    mbar_expect_tx(&bars[warp][s], STAGE);
#pragma unroll
                    for (int kv = 0; kv < 2; ++kv)
#pragma unroll
                        for (int b = 0; b < NBOX; ++b)
                            tma_load_2d(wbuf + s * STAGE + (kv * NBOX + b) * kBox, &tmap.full, b * 64, tile * 32 + kv * 16,
                                        &bars[warp][s], pol);
                }
            }
            ++seq_iss;
        }
    };
    top_up(0);
    // Q fragments (A operand): row gq = q-head g*GQ+gq, columns = head dims
    auto load_q = [&](const Task &t, uint32_t (&qa)[KSTEPS][2]) {
        const T *qrow = reinterpret_cast<const T *>(p.q) + t.l * p.q_layer_stride +
                        (static_cast<size_t>(t.it.i) * p.q_heads + t.g * GQ + gq) * D;
#pragma unroll
        for (int kk = 0; kk < KSTEPS; ++kk) {
            qa[kk][0] = gq < GQ ? __ldg(reinterpret_cast<const uint32_t *>(qrow + 16 * kk + 2 * cq)) : 0u;
            qa[kk][1] = gq < GQ ? __ldg(reinterpret_cast<const uint32_t *>(qrow + 16 * kk + 8 + 2 * cq)) : 0u;
        }
    };
    uint32_t qa[KSTEPS][2];
    load_q(cur, qa);

    while (cur.task < p.n_tasks) {
        if (!released) released = pdl_try_release(p, lane);
        // the q of `nxt` (its metadata arrived during the previous task)
        uint32_t qn[KSTEPS][2];
        load_q(nxt, qn);
        const int i = cur.it.i, c = cur.it.c, g = cur.g, lay = cur.l;
        const uint64_t t_task0 = p.trace ? globaltimer_ns() : 0;
        if (p.fuse_stats && c == 0 && g == 0 && lay == 0) batch_stats_warp(p, p.req[i], lane);
        float o[NT][4];
#pragma unroll
        for (int j = 0; j < NT; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
        float m = -INFINITY, l = 0.f;

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
            uint8_t *st = wbuf + s * STAGE;
            const uint32_t kb_base = smem_u32(st), vb_base = smem_u32(st + NBOX * kBox);
            const int valid = cur.it.ctx - (cur.it.pg0 + k) * kP;
            if (valid < kP) {  // last page: never-written V slots may hold NaN; P = 0 there is not enough
                for (int x = lane; x < (kP - valid) * NBOX * 8; x += 32) {
                    const int row = valid + x / (NBOX * 8), rem = x % (NBOX * 8);
                    *reinterpret_cast<uint4 *>(st + NBOX * kBox + (rem >> 3) * kBox + row * 128 + (rem & 7) * 16) =
                        make_uint4(0u, 0u, 0u, 0u);
                }
                __syncwarp();
            }
            // S = Q K^T for tokens 0-7 (s0) and 8-15 (s1); even / odd k-steps accumulate in
            // separate registers so the two dependent MMA chains are half as long
            float s0[2][4] = {}, s1[2][4] = {};
#pragma unroll
            for (int kk = 0; kk < KSTEPS; ++kk) {
                const int tok = (mtx >> 1) * 8 + mr, ch = (kk & 3) * 2 + (mtx & 1);
                uint32_t kb[4];
                ldsm_x4(kb, kb_base + (kk >> 2) * kBox + tok * 128 + ((ch ^ (tok & 7)) << 4));
                mma_pad<T>(s0[kk & 1], qa[kk][0], qa[kk][1], kb[0], kb[1]);
                mma_pad<T>(s1[kk & 1], qa[kk][0], qa[kk][1], kb[2], kb[3]);
            }
            // online softmax for q-head gq over this lane's tokens 2cq, 2cq+1, 8+2cq, 9+2cq
            const int t0 = 2 * cq;
            float x[4] = {(s0[0][0] + s0[1][0]) * p.scale_log2, (s0[0][1] + s0[1][1]) * p.scale_log2,
                          (s1[0][0] + s1[1][0]) * p.scale_log2, (s1[0][1] + s1[1][1]) * p.scale_log2};
            if (t0 >= valid) x[0] = -INFINITY;
            if (t0 + 1 >= valid) x[1] = -INFINITY;
            if (t0 + 8 >= valid) x[2] = -INFINITY;
            if (t0 + 9 >= valid) x[3] = -INFINITY;
            float mx = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
            mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 2));
            const float m_new = fmaxf(m, mx);
            const float alpha = (m == -INFINITY) ? 0.f : exp2f(m - m_new);
            float pr[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) pr[j] = (x[j] == -INFINITY) ? 0.f : exp2f(x[j] - m_new);
            l = l * alpha + (pr[0] + pr[1]) + (pr[2] + pr[3]);
            m = m_new;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                o[j][0] *= alpha;
                o[j][1] *= alpha;
            }
            // P (A operand, straight from the S fragments) times V
            const uint32_t pa0 = Elt<T>::from_f2(pr[0], pr[1]), pa2 = Elt<T>::from_f2(pr[2], pr[3]);
            uint32_t pl0 = 0u, pl2 = 0u;
            if constexpr (kBF16) {
                const float2 h0 = Elt<T>::to_f2(pa0), h2 = Elt<T>::to_f2(pa2);
                pl0 = Elt<T>::from_f2(pr[0] - h0.x, pr[1] - h0.y);
                pl2 = Elt<T>::from_f2(pr[2] - h2.x, pr[3] - h2.y);
            }
#pragma unroll
            for (int pp = 0; pp < D / 16; ++pp) {
                const int tok = (mtx & 1) * 8 + mr, ch = (pp & 3) * 2 + (mtx >> 1);
                uint32_t vb[4];
                ldsm_x4_t(vb, vb_base + (pp >> 2) * kBox + tok * 128 + ((ch ^ (tok & 7)) << 4));
                mma_pad<T>(o[2 * pp], pa0, pa2, vb[0], vb[1]);
                mma_pad<T>(o[2 * pp + 1], pa0, pa2, vb[2], vb[3]);
                if constexpr (kBF16) {
                    mma_pad<T>(o[2 * pp], pl0, pl2, vb[0], vb[1]);
                    mma_pad<T>(o[2 * pp + 1], pl0, pl2, vb[2], vb[3]);
                }
            }
            __syncwarp();
            top_up(jseq + 1);
        }

        // ---- end of task (warp-local): normalise and store, or write the split-K partial
        l += __shfl_xor_sync(kFull, l, 1);
        l += __shfl_xor_sync(kFull, l, 2);
        const bool split = cur.it.nchunks > 1;
        const size_t obase = lay * p.out_layer_stride + static_cast<size_t>(i) * p.q_heads * D;
        const int wb = lay * p.n_ws_rows + cur.it.chunk_base, ci = (lay * p.n + i) * p.kv_heads + g;
        if (gq < GQ) {
            const int h = g * GQ + gq;
            if (!split) {
                const float inv = 1.f / l;
                const size_t base = obase + static_cast<size_t>(h) * D + 2 * cq;
#pragma unroll
                for (int j = 0; j < NT; ++j) store2_out(p.out, base + 8 * j, p.out_dtype, o[j][0] * inv, o[j][1] * inv);
            } else {
                const int wi = wb + c;
                float *w = p.ws_o + (static_cast<size_t>(wi) * p.q_heads + h) * D + 2 * cq;
#pragma unroll
                for (int j = 0; j < NT; ++j) *reinterpret_cast<float2 *>(w + 8 * j) = make_float2(o[j][0], o[j][1]);
                if (cq == 0) p.ws_ml[static_cast<size_t>(wi) * p.q_heads + h] = make_float2(m, l);
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
        for (int kk = 0; kk < KSTEPS; ++kk) {
            qa[kk][0] = qn[kk][0];
            qa[kk][1] = qn[kk][1];
        }
        if (cur.task >= p.n_tasks && nxt.task < p.n_tasks) {  // no static second task: the claim is next
            cur = nxt;
            nxt = load_task(p, p.n_tasks, lane);
            load_q(cur, qa);
        }
        top_up(cur_start);
    }
    task_exit(p, lane, static_cast<int>(gridDim.x) * WARPS);
}

constexpr int kWarps = 4;
template <int D>
constexpr int gqa_stages() { return D == 128 ? 3 : 5; }

template <typename T, int D>
constexpr size_t gqa_smem() {
    return static_cast<size_t>(kWarps) * gqa_stages<D>() * 2 * (D / 64) * kBox + 1024;
}

template <typename T, int D, int GQ>
cudaError_t launch_gqa_t(const DecodeParams &p, int ctas, const GqaMaps &tmap, cudaStream_t s) {
    auto kern = decode_gqa_kernel<T, D, GQ, kWarps, gqa_stages<D>()>;
    constexpr size_t smem = gqa_smem<T, D>();
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    return launch_kernel(kern, dim3(ctas), dim3(kWarps * 32), smem, s, p.pdl != 0, p, tmap);
}

template <typename T, int D, int GQ>
int gqa_occ_t() {
    auto kern = decode_gqa_kernel<T, D, GQ, kWarps, gqa_stages<D>()>;
    constexpr size_t smem = gqa_smem<T, D>();
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kWarps * 32, smem) != cudaSuccess) n = 1;
    return n > 0 ? n : 1;
}

// Tuning variants of the (warps per CTA, ring stages) trade-off for GQ = 8 (DBK_GQA_WS =
// "2x6" or "8x3"; default 4x3): same shared memory per SM, different warps vs depth.
template <typename T, int D, int GQ, int W, int S>
cudaError_t launch_gqa_v(const DecodeParams &p, const GqaMaps &tmap, cudaStream_t s) {
    auto kern = decode_gqa_kernel<T, D, GQ, W, S>;
    constexpr size_t smem = static_cast<size_t>(W) * S * 2 * (D / 64) * kBox + 1024;
    static int occ = -1, sms = 148;
    if (occ < 0) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, W * 32, smem) != cudaSuccess || n < 1) n = 1;
        occ = n;
    }
    const int ctas = std::max(1, std::min(sms * occ, (p.n_tasks + W - 1) / W));
    return launch_kernel(kern, dim3(ctas), dim3(W * 32), smem, s, p.pdl != 0, p, tmap);
}

int gqa_variant() {
    static int v = -1;
    if (v < 0) {
        const char *e = std::getenv("DBK_GQA_WS");
        v = 0;
        if (e && std::strcmp(e, "2x6") == 0) v = 1;
        if (e && std::strcmp(e, "8x3") == 0) v = 2;
        if (e && std::strcmp(e, "1x3") == 0) v = 3;
        if (e && std::strcmp(e, "2x3") == 0) v = 4;
        if (e && std::strcmp(e, "1x4") == 0) v = 5;
    }
    return v;
}

template <typename T, int D>
cudaError_t gqa_group(const DecodeParams &p, int group, int ctas, const GqaMaps &tmap, cudaStream_t s) {
    switch (group) {
        case 2: return launch_gqa_t<T, D, 2>(p, ctas, tmap, s);
        case 4: return launch_gqa_t<T, D, 4>(p, ctas, tmap, s);
        case 8:
            if (gqa_variant() == 1) return launch_gqa_v<T, D, 8, 2, 6>(p, tmap, s);
            if (gqa_variant() == 2) return launch_gqa_v<T, D, 8, 8, 3>(p, tmap, s);
            if (gqa_variant() == 3) return launch_gqa_v<T, D, 8, 1, 3>(p, tmap, s);
            if (gqa_variant() == 4) return launch_gqa_v<T, D, 8, 2, 3>(p, tmap, s);
            if (gqa_variant() == 5) return launch_gqa_v<T, D, 8, 1, 4>(p, tmap, s);
            return launch_gqa_t<T, D, 8>(p, ctas, tmap, s);
        default: return cudaErrorInvalidValue;
    }
}
template <typename T, int D>
int gqa_occ_group(int group) {
    switch (group) {
        case 2: return gqa_occ_t<T, D, 2>();
        case 4: return gqa_occ_t<T, D, 4>();
        case 8: return gqa_occ_t<T, D, 8>();
        default: return 1;
    }
}

}  // namespace

cudaError_t launch_decode_gqa(const DecodeParams &p, int kv_dtype, int head_dim, int group, int ctas,
                              const GqaMaps &tmap, cudaStream_t s) {
    if (kv_dtype == 0) {
        if (head_dim == 128) return gqa_group<__half, 128>(p, group, ctas, tmap, s);
        if (head_dim == 64) return gqa_group<__half, 64>(p, group, ctas, tmap, s);
    } else {
        if (head_dim == 128) return gqa_group<__nv_bfloat16, 128>(p, group, ctas, tmap, s);
        if (head_dim == 64) return gqa_group<__nv_bfloat16, 64>(p, group, ctas, tmap, s);
    }
    return cudaErrorInvalidValue;
}

int decode_gqa_ctas_per_sm(int kv_dtype, int head_dim, int group) {
    if (kv_dtype == 0) return head_dim == 128 ? gqa_occ_group<__half, 128>(group) : gqa_occ_group<__half, 64>(group);
    return head_dim == 128 ? gqa_occ_group<__nv_bfloat16, 128>(group) : gqa_occ_group<__nv_bfloat16, 64>(group);
}

}  // namespace dbk
