// sm_100a kernels of the decode hot path:
//   K1/K3/K4  decode_kernel   paged decode attention, split-K merge by the last-arriving
//                             CTA, batch statistics fused into the layer-0 launch
//   K5/K6     append_kernel   KV append (explicit rows or the synthetic generator)
//             bt_apply_kernel block-table deltas (new pages, cleared rows)
//             synth_*         input-side generator (synth/hashgen.py on the device)
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "device_common.cuh"
#include "kernels.cuh"

namespace dbk {
namespace {
using namespace dev;

// ------------------------------------------------------------------ K1/K3: paged decode attention
// CTA = (work item = (request, chunk of chunk_pages pages), kv head g); it serves the
// GQ q-heads g*GQ .. g*GQ+GQ-1.  Each warp streams pages pg0+warp, pg0+warp+WARPS, ...
// through its own STAGES-deep ring of (K,V) page tiles [2][16][D], filled by 1-D TMA
// bulk copies completing on an mbarrier.  Lane layout in a warp: LPT = D/8 lanes cover
// one token row (8 dims per lane, one 16-byte LDS), TG = 32/LPT token groups; group grp
// owns tokens kk*TG + grp of each page and keeps its own online-softmax state, merged
// at the end through shared memory (and across chunks by the last-arriving CTA).
template <typename T, int D, int GQ, int WARPS, int STAGES>
__global__ void __launch_bounds__(WARPS * 32)
decode_kernel(const DecodeParams p) {
    constexpr int LPT = D / 8;
    constexpr int TG = 32 / LPT;
    constexpr int KI = kP / TG;  // tokens per group per page (= LPT / 2)
    constexpr int TILE = 2 * kP * D * static_cast<int>(sizeof(T));
    constexpr int NG = WARPS * TG;
    static_assert(KI * 2 == LPT, "lane layout");

    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[WARPS][STAGES];
    __shared__ int s_last;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / LPT, dl = lane % LPT;
    const int2 item = p.work[blockIdx.x];
    const int i = item.x, c = item.y;
    const int g = blockIdx.y;
    const ReqMeta rm = p.req[i];
    const int npages = (rm.ctx + kP - 1) / kP;
    const int pg0 = c * p.chunk_pages;
    const int pg1 = min(pg0 + p.chunk_pages, npages);
    const int span = pg1 - pg0;
    const int my_n = span > warp ? (span - warp + WARPS - 1) / WARPS : 0;

    uint8_t *wbuf = smem + warp * STAGES * TILE;
    const int32_t *bt_row = p.block_table + static_cast<size_t>(rm.slot) * p.bt_stride;
    const uint8_t *kvg = p.kv_layer + static_cast<size_t>(g) * TILE;
    // physical page of this warp's k-th page, one per lane (my_n <= 32)
    const int phys_lane = lane < my_n ? __ldg(bt_row + pg0 + warp + lane * WARPS) : 0;
    const uint64_t pol = evict_first_policy();

    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[warp][s], 1);
        fence_mbar_init();
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
        const int ph = __shfl_sync(kFull, phys_lane, s);
        if (lane == 0 && s < my_n) {
            mbar_expect_tx(&bars[warp][s], TILE);
            bulk_g2s(wbuf + s * TILE, kvg + static_cast<size_t>(ph) * p.page_stride, TILE,
                     &bars[warp][s], pol);
        }
    }

    if (p.fuse_stats && c == 0 && g == 0 && warp == WARPS - 1) batch_stats_warp(p, rm, lane);

    // q (pre-scaled to log2 units): lane holds dims dl*8 .. dl*8+7 of each q-head of the group
    float q[GQ][8];
#pragma unroll
    for (int t = 0; t < GQ; ++t) {
        const uint4 u = __ldg(reinterpret_cast<const uint4 *>(
            reinterpret_cast<const T *>(p.q) + (static_cast<size_t>(i) * p.q_heads + g * GQ + t) * D + dl * 8));
        unpack8<T>(u, q[t]);
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

    for (int k = 0; k < my_n; ++k) {
        const int s = k % STAGES;
        mbar_wait(&bars[warp][s], (k / STAGES) & 1);
        const T *Kt = reinterpret_cast<const T *>(wbuf + s * TILE);
        const T *Vt = Kt + kP * D;
        const int valid = rm.ctx - (pg0 + warp + k * WARPS) * kP;  // >= 1; < 16 only on the last page
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
        const int ph = __shfl_sync(kFull, phys_lane, (k + STAGES) & 31);
        if (lane == 0 && k + STAGES < my_n) {
            fence_proxy_async();
            mbar_expect_tx(&bars[warp][s], TILE);
            bulk_g2s(wbuf + s * TILE, kvg + static_cast<size_t>(ph) * p.page_stride, TILE,
                     &bars[warp][s], pol);
        }
    }

    // ---- merge the NG group states of this CTA
    __syncthreads();
    float *sm_acc = reinterpret_cast<float *>(smem);  // [NG][GQ][D]
    float *sm_m = sm_acc + NG * GQ * D;                // [NG][GQ]
    float *sm_l = sm_m + NG * GQ;
    const int gid = warp * TG + grp;
#pragma unroll
    for (int t = 0; t < GQ; ++t) {
        float4 *dst = reinterpret_cast<float4 *>(sm_acc + (gid * GQ + t) * D + dl * 8);
        dst[0] = make_float4(acc[t][0], acc[t][1], acc[t][2], acc[t][3]);
        dst[1] = make_float4(acc[t][4], acc[t][5], acc[t][6], acc[t][7]);
        if (dl == 0) {
            sm_m[gid * GQ + t] = m[t];
            sm_l[gid * GQ + t] = l[t];
        }
    }
    __syncthreads();
    merge_and_store<GQ, D, NG, WARPS * 32>(p, rm, i, c, g, sm_acc, sm_m, sm_l, &s_last);
}

template <int D>
constexpr int stages_for() { return D == 128 ? 3 : 4; }
constexpr int kWarps = 4;

template <typename T, int D, int GQ>
size_t decode_smem() {
    constexpr int TILE = 2 * kP * D * static_cast<int>(sizeof(T));
    constexpr int NG = kWarps * (32 / (D / 8));
    const size_t stage = static_cast<size_t>(kWarps) * stages_for<D>() * TILE;
    const size_t merge = static_cast<size_t>(NG) * GQ * (D + 2) * sizeof(float);
    return stage > merge ? stage : merge;
}

template <typename T, int D, int GQ>
cudaError_t launch_decode_t(const DecodeParams &p, int kv_heads, cudaStream_t s) {
    auto kern = decode_kernel<T, D, GQ, kWarps, stages_for<D>()>;
    const size_t smem = decode_smem<T, D, GQ>();
    static bool configured = false;  // per instantiation
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    dim3 grid(p.n_items, kv_heads);
    kern<<<grid, kWarps * 32, smem, s>>>(p);
    return cudaGetLastError();
}

template <typename T, int D, int GQ>
int occupancy_t() {
    auto kern = decode_kernel<T, D, GQ, kWarps, stages_for<D>()>;
    const size_t smem = decode_smem<T, D, GQ>();
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kWarps * 32, smem) != cudaSuccess) n = 1;
    return n > 0 ? n : 1;
}

template <typename T, int D>
cudaError_t dispatch_group(const DecodeParams &p, int group, int kv_heads, cudaStream_t s) {
    switch (group) {
        case 1: return launch_decode_t<T, D, 1>(p, kv_heads, s);
        case 2: return launch_decode_t<T, D, 2>(p, kv_heads, s);
        case 4: return launch_decode_t<T, D, 4>(p, kv_heads, s);
        case 8: return launch_decode_t<T, D, 8>(p, kv_heads, s);
        default: return cudaErrorInvalidValue;
    }
}
template <typename T, int D>
int occ_group(int group) {
    switch (group) {
        case 1: return occupancy_t<T, D, 1>();
        case 2: return occupancy_t<T, D, 2>();
        case 4: return occupancy_t<T, D, 4>();
        case 8: return occupancy_t<T, D, 8>();
        default: return 1;
    }
}

// ------------------------------------------------------------------ K5/K6: KV append
template <typename T, int D>
__global__ void __launch_bounds__(256) append_kernel(const AppendParams p) {
    constexpr int VPR = D / 8;  // 16-byte vectors per row
    const AppendJob job = p.jobs[blockIdx.x];
    const int layer = blockIdx.y;
    const int rows_per_block = job.ntok;  // rows of one (head, K|V) tile this job writes
    const int total = p.kv_heads * 2 * rows_per_block * VPR;
    uint8_t *page = p.kv + static_cast<size_t>(layer) * p.layer_stride +
                    static_cast<size_t>(job.phys) * p.page_stride;
    const float scale = 1.0f / 128.0f;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const int v = idx % VPR;
        int r = idx / VPR;
        const int tok = r % rows_per_block;
        r /= rows_per_block;
        const int kv = r & 1, head = r >> 1;
        const int pos = job.pos0 + tok;
        T *dst = reinterpret_cast<T *>(page + static_cast<size_t>(head) * p.tile_bytes) +
                 (kv * kP + (pos % kP)) * D + v * 8;
        uint4 val;
        if (job.src_row < 0) {
            float f[8];
            synth_vals(synth_key(p.seed, 1 + kv, job.req_id, pos, layer, head, v), scale, f);
            val = pack8<T>(f);
        } else {
            const T *src = reinterpret_cast<const T *>(kv ? p.v_src : p.k_src) +
                           ((static_cast<size_t>(job.src_row + tok) * p.layers + layer) * p.kv_heads + head) * D +
                           v * 8;
            val = __ldg(reinterpret_cast<const uint4 *>(src));
        }
        *reinterpret_cast<uint4 *>(dst) = val;
    }
}

__global__ void bt_apply_kernel(int32_t *bt, int32_t stride, const BtDelta *d, int32_t n) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const BtDelta x = d[k];
        bt[static_cast<size_t>(x.slot) * stride + x.idx] = x.val;
    }
}

// ------------------------------------------------------------------ synthetic rows
__device__ __forceinline__ void store8(void *out, size_t elem, int dtype, const float f[8]) {
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

__global__ void synth_rows_kernel(uint64_t seed, int kind, int n_rows, const int64_t *req,
                                  const int32_t *pos, int layer, int n_heads, int d, float scale,
                                  int dtype, void *out) {
    const int vpr = d / 8;
    const long total = static_cast<long>(n_rows) * n_heads * vpr;
    for (long k = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; k < total;
         k += static_cast<long>(gridDim.x) * blockDim.x) {
        const int v = static_cast<int>(k % vpr);
        const long rh = k / vpr;
        const int h = static_cast<int>(rh % n_heads);
        const int r = static_cast<int>(rh / n_heads);
        float f[8];
        synth_vals(synth_key(seed, kind, req[r], pos[r], layer, h, v), scale, f);
        store8(out, static_cast<size_t>(rh) * d + v * 8, dtype, f);
    }
}

// q of every layer for the batch in `req`: q[l][i][h][:] = synth(seed, q, req_i, ctx_i - 1, l, h),
// layer l at q + l * layer_rows rows (one launch per step).
__global__ void synth_q_kernel(uint64_t seed, const ReqMeta *req, int n, int layers, int layer_rows,
                               int q_heads, int d, float scale, int dtype, void *q) {
    const int vpr = d / 8;
    const long per_layer = static_cast<long>(n) * q_heads * vpr;
    const long total = per_layer * layers;
    for (long k = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; k < total;
         k += static_cast<long>(gridDim.x) * blockDim.x) {
        const int l = static_cast<int>(k / per_layer);
        const long kk = k % per_layer;
        const int v = static_cast<int>(kk % vpr);
        const long rh = kk / vpr;
        const int h = static_cast<int>(rh % q_heads);
        const int r = static_cast<int>(rh / q_heads);
        const ReqMeta rm = req[r];
        float f[8];
        synth_vals(synth_key(seed, 0, rm.req_id, rm.ctx - 1, l, h, v), scale, f);
        store8(q, (static_cast<size_t>(l) * layer_rows * q_heads + rh) * d + v * 8, dtype, f);
    }
}

int grid_for(long work, int block) {
    long b = (work + block - 1) / block;
    if (b > 148L * 16) b = 148L * 16;
    return static_cast<int>(b < 1 ? 1 : b);
}

}  // namespace

cudaError_t launch_decode(const DecodeParams &p, int kv_dtype, int head_dim, int group,
                          int kv_heads, const CUtensorMap *tmap, cudaStream_t s) {
    if (p.n_items <= 0) return cudaSuccess;
    if (tmap && group >= 2) return launch_decode_gqa(p, kv_dtype, head_dim, group, kv_heads, *tmap, s);
    if (kv_dtype == 0) {
        if (head_dim == 128) return dispatch_group<__half, 128>(p, group, kv_heads, s);
        if (head_dim == 64) return dispatch_group<__half, 64>(p, group, kv_heads, s);
    } else {
        if (head_dim == 128) return dispatch_group<__nv_bfloat16, 128>(p, group, kv_heads, s);
        if (head_dim == 64) return dispatch_group<__nv_bfloat16, 64>(p, group, kv_heads, s);
    }
    return cudaErrorInvalidValue;
}

int decode_ctas_per_sm(int kv_dtype, int head_dim, int group) {
    if (kv_dtype == 0) return head_dim == 128 ? occ_group<__half, 128>(group) : occ_group<__half, 64>(group);
    return head_dim == 128 ? occ_group<__nv_bfloat16, 128>(group) : occ_group<__nv_bfloat16, 64>(group);
}

cudaError_t launch_append(const AppendParams &p, int kv_dtype, int head_dim, cudaStream_t s) {
    if (p.n_jobs <= 0) return cudaSuccess;
    dim3 grid(p.n_jobs, p.layers);
    if (kv_dtype == 0) {
        if (head_dim == 128) append_kernel<__half, 128><<<grid, 256, 0, s>>>(p);
        else append_kernel<__half, 64><<<grid, 256, 0, s>>>(p);
    } else {
        if (head_dim == 128) append_kernel<__nv_bfloat16, 128><<<grid, 256, 0, s>>>(p);
        else append_kernel<__nv_bfloat16, 64><<<grid, 256, 0, s>>>(p);
    }
    return cudaGetLastError();
}

cudaError_t launch_bt_apply(int32_t *bt, int32_t stride, const BtDelta *d, int32_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    bt_apply_kernel<<<grid_for(n, 256), 256, 0, s>>>(bt, stride, d, n);
    return cudaGetLastError();
}

cudaError_t launch_synth_rows(uint64_t seed, int kind, int n_rows, const int64_t *req,
                              const int32_t *pos, int layer, int n_heads, int d, int scale_log2,
                              int dtype, void *out, cudaStream_t s) {
    const long work = static_cast<long>(n_rows) * n_heads * (d / 8);
    if (work <= 0) return cudaSuccess;
    synth_rows_kernel<<<grid_for(work, 256), 256, 0, s>>>(seed, kind, n_rows, req, pos, layer, n_heads,
                                                          d, ldexpf(1.0f, scale_log2 - 7), dtype, out);
    return cudaGetLastError();
}

cudaError_t launch_synth_q(uint64_t seed, const ReqMeta *req, int n, int layers, int layer_rows,
                           int q_heads, int d, int scale_log2, int dtype, void *q, cudaStream_t s) {
    const long work = static_cast<long>(n) * layers * q_heads * (d / 8);
    if (work <= 0) return cudaSuccess;
    synth_q_kernel<<<grid_for(work, 256), 256, 0, s>>>(seed, req, n, layers, layer_rows, q_heads, d,
                                                       ldexpf(1.0f, scale_log2 - 7), dtype, q);
    return cudaGetLastError();
}

}  // namespace dbk
