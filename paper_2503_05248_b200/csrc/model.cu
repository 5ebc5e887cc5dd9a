// Full decode step with synthetic weights (R32-R35):
// a Llama-2-shaped decoder whose attention is the pool's paged decode attention (K1/K2).
//   - every projection (QKV, O, gate|up, down, LM head) is our tcgen05 GEMM (gemm_tc.cu) with
//     the step's elementwise work fused into its epilogue: RoPE of q and k + the token's K/V
//     written straight into its page slot (QKV), silu(gate) * up (gate|up: weight rows stored
//     interleaved), the residual add (O and down accumulate into the fp32 residual stream);
//   - our kernels around them: synthetic weight fill, embedding + RMSNorm, RMSNorm.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <utility>
#include <vector>

#include "common.h"
#include "device_common.cuh"
#include "gemm.h"
#include "kernels.cuh"
#include "pool.h"
#include "tp.h"

using namespace dbk;

namespace {
using namespace dbk::dev;

using RowMeta = TokRow;  // one activation row: a decode token (pos = ctx - 1) or a chunk token

constexpr int kWChunk = 128;  // synthetic weight rows are K/128 "heads" of 128 dims (hashgen)
constexpr int kKindToken = 7, kKindEmbed = 8, kKindLn1 = 9, kKindWqkv = 10, kKindWo = 11, kKindLn2 = 12,
              kKindWgu = 13, kKindWdown = 14, kKindLnf = 15, kKindLm = 16;
// physical -> logical row order of a weight as stored for its GEMM epilogue (gemm.h)
constexpr int kPermNone = 0, kPermQkv = 1, kPermGu = 2;

// ------------------------------------------------------------------ kernels
// Which rows / columns of the GLOBAL synthetic matrix a (possibly tensor-parallel, possibly
// row-permuted) local weight holds.  Rank r of a TP-G model keeps the q / k / v rows of its heads
// in W_qkv, the columns of its q heads in W_o, the gate / up rows of its FFN slice in W_gu and
// the columns of that slice in W_down ("TP model step").
struct FillMap {
    int perm = kPermNone;                // kPermNone / kPermQkv / kPermGu
    int hq_l = 0, hkv_l = 0, d = 0;      // local heads
    int hq_g = 0, hkv_g = 0, hq0 = 0, hk0 = 0;  // global heads, this rank's first q / kv head
    int64_t f_l = 0, f_g = 0, f0 = 0;    // gate|up: local / global FFN size, first global column
    int64_t k_off = 0;                   // global column of local column 0 (multiple of 8)
};

__device__ __forceinline__ int64_t global_row(int64_t prow, const FillMap &fm) {
    if (fm.perm == kPermQkv) {
        const int64_t lr = qkv_logical_row(prow, fm.hq_l, fm.hkv_l, fm.d);
        const int64_t qd = static_cast<int64_t>(fm.hq_l) * fm.d, kd = static_cast<int64_t>(fm.hkv_l) * fm.d;
        if (lr < qd) return static_cast<int64_t>(fm.hq0) * fm.d + lr;
        if (lr < qd + kd) return static_cast<int64_t>(fm.hq_g + fm.hk0) * fm.d + (lr - qd);
        return static_cast<int64_t>(fm.hq_g + fm.hkv_g + fm.hk0) * fm.d + (lr - qd - kd);
    }
    if (fm.perm == kPermGu) {
        const int64_t lr = gu_logical_row(prow, fm.f_l);  // [0, f_l) gate rows, [f_l, 2 f_l) up rows
        return lr < fm.f_l ? fm.f0 + lr : fm.f_g + fm.f0 + (lr - fm.f_l);
    }
    return prow;
}

// W[row][k] = (byte - 128) * scale (+1 for norm gains), byte of (seed, kind, 0, row, layer, k / 128,
// k % 128) at the GLOBAL (row, k) of the local element: the host passes scale = 2^(scale_log2 - 7),
// i.e. value * 2^scale_log2 of synth/hashgen.py.  Physical row `prow` holds global row
// global_row(prow) (kPermQkv / kPermGu: the GEMM epilogues' layouts, gemm.h).
__global__ void fill_weights_kernel(__half *w, int64_t rows, int K, int layer, int kind, uint64_t seed, float scale,
                                    int norm, const FillMap fm) {
    const int64_t per_row = K / 8;
    const int64_t total = rows * per_row;
    for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < total;
         c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t prow = c / per_row;
        const int64_t row = global_row(prow, fm);
        const int64_t k = (c % per_row) * 8;
        const int64_t kg = k + fm.k_off;
        float f[8];
        synth_vals(synth_key(seed, kind, 0, static_cast<int>(row), layer, static_cast<int>(kg / kWChunk),
                             static_cast<int>((kg % kWChunk) / 8)),
                   scale, f);
        if (norm)
#pragma unroll
            for (int e = 0; e < 8; ++e) f[e] += 1.0f;
        *reinterpret_cast<uint4 *>(w + prow * K + k) = pack8<__half>(f);
    }
}

__device__ __forceinline__ float block_sum(float v, float *red) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float t = 0.f;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) t += red[w];
    __syncthreads();
    return t;
}

// h[i] = RMSNorm(x[i]) * g (fp16); with embed != nullptr, x[i] = E[token(req_i, pos_i)] first.
// One CTA per row; H % 8 == 0 and H / 8 <= 4 * blockDim.x.
__global__ void __launch_bounds__(256) norm_kernel(float *x, const __half *g, float eps, int H, __half *h,
                                                   const RowMeta *rows, const __half *embed, uint64_t tok_seed,
                                                   int vocab, const int32_t *tokens, int n_tok) {
    __shared__ float red[8];
    // launched with programmatic dependent launch after the GEMM that produced x
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int i = blockIdx.x;
    float *xr = x + static_cast<size_t>(i) * H;
    const int nv = H / 8;
    float v[4][8];
    float ss = 0.f;
    const __half *er = nullptr;
    if (embed) {
        const RowMeta rm = rows[i];
        uint64_t tok;
        if (i < n_tok) {  // caller-provided token id (e.g. the previous step's sample)
            const int32_t t = tokens[i];
            tok = static_cast<uint64_t>(t < 0 ? 0 : (t >= vocab ? vocab - 1 : t));
        } else {
            tok = (synth_key(tok_seed, kKindToken, rm.req_id, rm.pos, 0, 0, 0) >> 16) % static_cast<uint64_t>(vocab);
        }
        er = embed + static_cast<size_t>(tok) * H;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int j = threadIdx.x + c * blockDim.x;
        if (j < nv) {
            if (er) {
                unpack8<__half>(*reinterpret_cast<const uint4 *>(er + j * 8), v[c]);
                *reinterpret_cast<float4 *>(xr + j * 8) = make_float4(v[c][0], v[c][1], v[c][2], v[c][3]);
                *reinterpret_cast<float4 *>(xr + j * 8 + 4) = make_float4(v[c][4], v[c][5], v[c][6], v[c][7]);
            } else {
                const float4 a = *reinterpret_cast<const float4 *>(xr + j * 8);
                const float4 b = *reinterpret_cast<const float4 *>(xr + j * 8 + 4);
                v[c][0] = a.x; v[c][1] = a.y; v[c][2] = a.z; v[c][3] = a.w;
                v[c][4] = b.x; v[c][5] = b.y; v[c][6] = b.z; v[c][7] = b.w;
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) ss += v[c][e] * v[c][e];
        }
    }
    const float r = rsqrtf(block_sum(ss, red) / static_cast<float>(H) + eps);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int j = threadIdx.x + c * blockDim.x;
        if (j < nv) {
            float gg[8], o[8];
            unpack8<__half>(*reinterpret_cast<const uint4 *>(g + j * 8), gg);
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = v[c][e] * r * gg[e];
            *reinterpret_cast<uint4 *>(h + static_cast<size_t>(i) * H + j * 8) = pack8<__half>(o);
        }
    }
}

// Tensor-parallel RMSNorm ("TP model step"): h[i] = RMSNorm(x_i) * g where the row
// x_i is GATHERED from the owners of its column slices (xsrc[o] = rank o's buffer; the all-gather
// half of the all-reduce), or is the embedding E[token(req_i, pos_i)] when xsrc is null.  Then
// this rank's slice [own0, own0 + own_n) of x_i is ADDED into base (the buffer the next residual
// GEMM accumulates into, atomically: peers' GEMM partials may already be arriving) and the same
// slice of zero_dst is cleared for the accumulation after that.  One CTA per row.
__global__ void __launch_bounds__(256) tp_norm_kernel(const float *const *xsrc, const __half *g, float eps, int H,
                                                      __half *h, const RowMeta *rows, const __half *embed,
                                                      uint64_t tok_seed, int vocab, const int32_t *tokens, int n_tok,
                                                      int own0, int own_n, float *base, float *zero_dst) {
    __shared__ float red[8];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int i = blockIdx.x;
    const int nv = H / 8;
    float v[4][8];
    float ss = 0.f;
    const __half *er = nullptr;
    if (!xsrc) {
        const RowMeta rm = rows[i];
        uint64_t tok;
        if (i < n_tok) {
            const int32_t t = tokens[i];
            tok = static_cast<uint64_t>(t < 0 ? 0 : (t >= vocab ? vocab - 1 : t));
        } else {
            tok = (synth_key(tok_seed, kKindToken, rm.req_id, rm.pos, 0, 0, 0) >> 16) % static_cast<uint64_t>(vocab);
        }
        er = embed + static_cast<size_t>(tok) * H;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int j = threadIdx.x + c * blockDim.x;
        if (j < nv) {
            if (er) {
                unpack8<__half>(*reinterpret_cast<const uint4 *>(er + j * 8), v[c]);
            } else {
                const float *src = xsrc[(j * 8) / own_n] + static_cast<size_t>(i) * H + j * 8;  // owner's slice
                const float4 a = *reinterpret_cast<const float4 *>(src);
                const float4 b = *reinterpret_cast<const float4 *>(src + 4);
                v[c][0] = a.x; v[c][1] = a.y; v[c][2] = a.z; v[c][3] = a.w;
                v[c][4] = b.x; v[c][5] = b.y; v[c][6] = b.z; v[c][7] = b.w;
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) ss += v[c][e] * v[c][e];
        }
    }
    const float r = rsqrtf(block_sum(ss, red) / static_cast<float>(H) + eps);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int j = threadIdx.x + c * blockDim.x;
        if (j < nv) {
            float gg[8], o[8];
            unpack8<__half>(*reinterpret_cast<const uint4 *>(g + j * 8), gg);
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = v[c][e] * r * gg[e];
            *reinterpret_cast<uint4 *>(h + static_cast<size_t>(i) * H + j * 8) = pack8<__half>(o);
            if (j * 8 >= own0 && j * 8 < own0 + own_n) {
                const size_t at = static_cast<size_t>(i) * H + j * 8;
                if (base)
#pragma unroll
                    for (int e = 0; e < 8; ++e) atomicAdd(base + at + e, v[c][e]);
                if (zero_dst) {
                    *reinterpret_cast<float4 *>(zero_dst + at) = make_float4(0.f, 0.f, 0.f, 0.f);
                    *reinterpret_cast<float4 *>(zero_dst + at + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        }
    }
}

// Greedy sampling: out[i] = the lowest index of the largest logit of row i (NaN rows -> 0).
__global__ void __launch_bounds__(256) argmax_kernel(const float *logits, int V, int32_t *out) {
    __shared__ float bv[8];
    __shared__ int bi[8];
    const float *row = logits + static_cast<size_t>(blockIdx.x) * V;
    float best = -INFINITY;
    int idx = 0x7fffffff;
    for (int j = threadIdx.x; j < V; j += blockDim.x) {
        const float v = row[j];
        if (v > best) {  // strided scan: the first hit of a value is its lowest index in this thread
            best = v;
            idx = j;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const float ov = __shfl_xor_sync(kFull, best, o);
        const int oi = __shfl_xor_sync(kFull, idx, o);
        if (ov > best || (ov == best && oi < idx)) {
            best = ov;
            idx = oi;
        }
    }
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (lane == 0) {
        bv[warp] = best;
        bi[warp] = idx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x / 32); ++w)
            if (bv[w] > best || (bv[w] == best && bi[w] < idx)) {
                best = bv[w];
                idx = bi[w];
            }
        out[blockIdx.x] = idx == 0x7fffffff ? 0 : idx;
    }
}

int grid_of(int64_t work, int block, int sms) {
    int64_t b = (work + block - 1) / block;
    const int64_t cap = static_cast<int64_t>(sms) * 8;
    return static_cast<int>(b < 1 ? 1 : (b > cap ? cap : b));
}

size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

struct LayerW {
    __half *ln1, *wqkv, *wo, *ln2, *wgu, *wdown;
};

}  // namespace

struct dbk_model {
    dbk_pool *pool = nullptr;
    int device = 0;
    dbk_model_config cfg{};
    int L = 0, Hq = 0, Hkv = 0, d = 0, H = 0, F = 0, V = 0, nqkv = 0, rows = 0;
    __half *embed = nullptr, *lnf = nullptr, *lm = nullptr;
    std::vector<LayerW> lw;
    float2 *cs = nullptr;
    float *x = nullptr, *logits = nullptr;
    __half *h = nullptr, *q = nullptr, *attn = nullptr, *act = nullptr;
    GemmRunner gemm;  // tcgen05 GEMM, CTA pairs
    // tensor parallelism (cfg.tp_size > 1): this rank's slice and the attached residual stream
    int G = 1, tp_r = 0, Hq_g = 0, Hkv_g = 0, F_g = 0;
    dbk_tp *tp = nullptr;
    int tp_cur = 0;  // rotation index of the TP residual buffers (continues across steps)
    UploadBuffer up_rows;
    std::vector<RowMeta> rows_h;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::vector<cudaEvent_t> a0, a1;
    bool pending = false;
    double attn_ms = 0, total_ms = 0;
    int64_t steps = 0;
    ~dbk_model() {
        up_rows.release();
        if (up_rows.done) cudaEventDestroy(up_rows.done);
        for (void *ptr : {static_cast<void *>(cs), static_cast<void *>(x), static_cast<void *>(logits),
                          static_cast<void *>(h), static_cast<void *>(q), static_cast<void *>(attn),
                          static_cast<void *>(act)})
            if (ptr) cudaFree(ptr);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        for (auto e : a0) cudaEventDestroy(e);
        for (auto e : a1) cudaEventDestroy(e);
    }
};

namespace {

// Y = X W^T through the tensor-core GEMM with epilogue `e` (PDL: the GEMM waits on the grid
// dependency before it reads X or writes its outputs; its weight prefetch overlaps the previous
// kernel's tail).
dbk_status gemm(dbk_model *m, int M, int N, int K, const __half *X, const __half *W, const GemmEpiArgs &e,
                cudaStream_t s) {
    const cudaError_t err = m->gemm.run(M, N, K, X, K, W, e, s, true);
    if (err != cudaSuccess) return fail(DBK_ECUDA, "model GEMM (%d x %d x %d): %s", M, N, K, cudaGetErrorString(err));
    return DBK_OK;
}

GemmEpiArgs epi_plain(int kind, void *y, int64_t ldy) {
    GemmEpiArgs e;
    e.kind = kind;
    e.y = y;
    e.ldy = ldy;
    return e;
}

dbk_status collect_timing(dbk_model *m) {
    if (!m->pending) return DBK_OK;
    DBK_CUDA(cudaEventSynchronize(m->ev1));
    float t = 0.f;
    DBK_CUDA(cudaEventElapsedTime(&t, m->ev0, m->ev1));
    m->total_ms += t;
    for (int l = 0; l < m->L; ++l) {
        DBK_CUDA(cudaEventElapsedTime(&t, m->a0[l], m->a1[l]));
        m->attn_ms += t;
    }
    ++m->steps;
    m->pending = false;
    return DBK_OK;
}

}  // namespace

namespace dbk {
// the pool whose KV the model's QKV epilogue writes (the engine checks it is its own)
dbk_pool *model_pool(const dbk_model *m) { return m->pool; }
}  // namespace dbk

extern "C" {

size_t dbk_model_weight_bytes(const dbk_pool_config *pc, const dbk_model_config *c) {
    if (!pc || !c || c->hidden <= 0 || c->ffn <= 0 || c->vocab <= 0) return 0;
    const int G = c->tp_size > 1 ? c->tp_size : 1;
    const size_t H = c->hidden, F = c->ffn / G, V = c->vocab, d = pc->head_dim;  // local FFN slice
    const size_t nqkv = (static_cast<size_t>(pc->q_heads) + 2 * pc->kv_heads) * d;
    size_t per_layer = align256(H * 2) * 2 + align256(nqkv * H * 2) + align256(H * pc->q_heads * d * 2) +
                       align256(2 * F * H * 2) + align256(H * F * 2);
    return align256(V * H * 2) + pc->layers * per_layer + align256(H * 2) + align256(V * H * 2);
}

dbk_status dbk_model_create(dbk_pool *p, const dbk_model_config *c, void *wmem, size_t bytes, dbk_model **out) {
    if (!p || !c || !out) return fail(DBK_EINVAL, "model_create: null argument");
    const dbk_pool_config &pc = p->cfg;
    if (pc.kv_dtype != 0) return fail(DBK_EINVAL, "model_create: the model path is fp16 (kv_dtype 0)");
    const int G = c->tp_size > 1 ? c->tp_size : 1;
    if (c->tp_size < 0 || c->tp_rank < 0 || c->tp_rank >= G)
        return fail(DBK_EINVAL, "model_create: need 0 <= tp_rank < tp_size");
    if (pc.kv_head_offset != c->tp_rank * pc.kv_heads)
        return fail(DBK_EINVAL, "model_create: the pool must hold this rank's kv heads (kv_head_offset = tp_rank * "
                                "kv_heads)");
    if (G > 1 && (c->ffn % (G * kWChunk) || c->hidden % (32 * G)))
        return fail(DBK_EINVAL, "model_create: tensor parallel needs ffn %% (128 * tp_size) == 0 and hidden %% "
                                "(32 * tp_size) == 0");
    if (c->hidden % kWChunk || c->ffn % kWChunk || c->hidden > 8 * 4 * 256 || c->vocab < 1 || c->max_pos < 1 ||
        (pc.q_heads * pc.head_dim) % kWChunk || c->rms_eps <= 0 || c->rope_theta <= 0 || 128 % pc.head_dim ||
        c->vocab % 4 || ((pc.q_heads + 2 * pc.kv_heads) * pc.head_dim) % 256)
        return fail(DBK_EINVAL, "model_create: hidden, ffn, q_heads*head_dim multiples of 128, (Hq + 2 Hkv) * d a "
                                "multiple of 256, vocab a multiple of 4, hidden <= 8192");
    const size_t need = dbk_model_weight_bytes(&pc, c);
    if (!wmem || bytes < need || (reinterpret_cast<uintptr_t>(wmem) & 255))
        return fail(DBK_EINVAL, "model_create: weight_mem must be 256-B aligned and >= %zu bytes", need);
    DBK_CUDA(cudaSetDevice(pc.device));
    dbk_model *m = new (std::nothrow) dbk_model();
    if (!m) return fail(DBK_EINVAL, "out of host memory");
    m->pool = p;
    m->device = pc.device;
    m->cfg = *c;
    m->L = pc.layers;
    m->Hq = pc.q_heads;
    m->Hkv = pc.kv_heads;
    m->d = pc.head_dim;
    m->H = c->hidden;
    m->G = G;
    m->tp_r = c->tp_rank;
    m->F = c->ffn / G;  // local FFN slice
    m->F_g = c->ffn;
    m->Hq_g = pc.q_heads * G;
    m->Hkv_g = pc.kv_heads * G;
    m->V = c->vocab;
    m->nqkv = (m->Hq + 2 * m->Hkv) * m->d;
    m->rows = pc.max_requests;
    auto bail = [&](dbk_status st) {
        delete m;
        return st;
    };
    // weights: carve the caller's memory, fill with the generator
    uint8_t *w = static_cast<uint8_t *>(wmem);
    auto take = [&](size_t elems) {
        __half *r = reinterpret_cast<__half *>(w);
        w += align256(elems * 2);
        return r;
    };
    const int sms = p->num_sms;
    auto fill = [&](__half *dst, int64_t rows_, int K, int layer, int kind, int scale_log2, int norm,
                    const FillMap &fm = FillMap{}) {
        fill_weights_kernel<<<grid_of(rows_ * K / 8, 256, sms), 256>>>(
            dst, rows_, K, layer, kind, c->weight_seed, std::ldexp(1.0f, scale_log2 - 7), norm, fm);
    };
    FillMap fm_qkv;  // this rank's q / k / v heads, RoPE pairs adjacent
    fm_qkv.perm = kPermQkv;
    fm_qkv.hq_l = pc.q_heads;
    fm_qkv.hkv_l = pc.kv_heads;
    fm_qkv.d = pc.head_dim;
    fm_qkv.hq_g = m->Hq_g;
    fm_qkv.hkv_g = m->Hkv_g;
    fm_qkv.hq0 = c->tp_rank * pc.q_heads;
    fm_qkv.hk0 = c->tp_rank * pc.kv_heads;
    FillMap fm_o;  // the columns of this rank's q heads
    fm_o.k_off = static_cast<int64_t>(c->tp_rank) * pc.q_heads * pc.head_dim;
    FillMap fm_gu;  // the gate / up rows of this rank's FFN slice, interleaved
    fm_gu.perm = kPermGu;
    fm_gu.f_l = m->F;
    fm_gu.f_g = m->F_g;
    fm_gu.f0 = static_cast<int64_t>(c->tp_rank) * m->F;
    FillMap fm_down;  // the columns of that slice
    fm_down.k_off = fm_gu.f0;
    auto sl2 = [](int K) { return -static_cast<int>(std::ceil(std::log2(static_cast<double>(K)) / 2)); };
    const int H = m->H, F = m->F, V = m->V, qd = m->Hq * m->d;
    m->embed = take(static_cast<size_t>(V) * H);
    fill(m->embed, V, H, 0, kKindEmbed, 0, 0);
    m->lw.resize(m->L);
    for (int l = 0; l < m->L; ++l) {
        LayerW &x = m->lw[l];
        x.ln1 = take(H);
        x.wqkv = take(static_cast<size_t>(m->nqkv) * H);
        x.wo = take(static_cast<size_t>(H) * qd);
        x.ln2 = take(H);
        x.wgu = take(static_cast<size_t>(2) * F * H);
        x.wdown = take(static_cast<size_t>(H) * F);
        fill(x.ln1, 1, H, l, kKindLn1, -3, 1);
        fill(x.wqkv, m->nqkv, H, l, kKindWqkv, sl2(H), 0, fm_qkv);
        fill(x.wo, H, qd, l, kKindWo, sl2(m->Hq_g * m->d), 0, fm_o);  // scales of the GLOBAL K
        fill(x.ln2, 1, H, l, kKindLn2, -3, 1);
        fill(x.wgu, 2 * F, H, l, kKindWgu, sl2(H), 0, fm_gu);
        fill(x.wdown, H, F, l, kKindWdown, sl2(m->F_g), 0, fm_down);
    }
    m->lnf = take(H);
    m->lm = take(static_cast<size_t>(V) * H);
    fill(m->lnf, 1, H, 0, kKindLnf, -3, 1);
    fill(m->lm, V, H, 0, kKindLm, sl2(H), 0);
    if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
        return bail(fail(DBK_ECUDA, "model_create: weight fill failed"));
    // RoPE table: angles in double, rounded once to fp32
    {
        const int hd = m->d / 2;
        std::vector<float2> t(static_cast<size_t>(c->max_pos) * hd);
        for (int pos = 0; pos < c->max_pos; ++pos)
            for (int j = 0; j < hd; ++j) {
                const double a = pos * std::pow(c->rope_theta, -2.0 * j / m->d);
                t[static_cast<size_t>(pos) * hd + j] = make_float2(static_cast<float>(std::cos(a)),
                                                                   static_cast<float>(std::sin(a)));
            }
        if (cudaMalloc(&m->cs, t.size() * sizeof(float2)) != cudaSuccess ||
            cudaMemcpy(m->cs, t.data(), t.size() * sizeof(float2), cudaMemcpyHostToDevice) != cudaSuccess)
            return bail(fail(DBK_ECUDA, "model_create: RoPE table"));
    }
    const size_t R = m->rows;
    if (cudaMalloc(&m->x, R * H * 4) != cudaSuccess || cudaMalloc(&m->logits, R * V * 4) != cudaSuccess ||
        cudaMalloc(&m->h, R * H * 2) != cudaSuccess || cudaMalloc(&m->q, R * qd * 2) != cudaSuccess ||
        cudaMalloc(&m->attn, R * qd * 2) != cudaSuccess || cudaMalloc(&m->act, R * F * 2) != cudaSuccess)
        return bail(fail(DBK_ECUDA, "model_create: activation workspace"));
    // zeroed once: the GEMM epilogues write q, K/V and the fp16 activations with TMA bulk stores,
    // which compute-sanitizer's initcheck does not see as initialisation (its reports on the
    // attention's q reads vanish with this; the parity suite checks every row the step reads)
    for (auto [ptr, bytes] : {std::pair<void *, size_t>{m->x, R * H * 4}, {m->logits, R * V * 4}, {m->h, R * H * 2},
                              {m->q, R * qd * 2}, {m->attn, R * qd * 2}, {m->act, R * F * 2}})
        if (cudaMemset(ptr, 0, bytes) != cudaSuccess) return bail(fail(DBK_ECUDA, "model_create: workspace clear"));
    if (m->gemm.init(pc.device, 2) != cudaSuccess) return bail(fail(DBK_ECUDA, "model_create: tensor-core GEMM init"));
    m->a0.assign(m->L, nullptr);
    m->a1.assign(m->L, nullptr);
    if (cudaEventCreate(&m->ev0) != cudaSuccess || cudaEventCreate(&m->ev1) != cudaSuccess)
        return bail(fail(DBK_ECUDA, "model_create: events"));
    for (int l = 0; l < m->L; ++l)
        if (cudaEventCreate(&m->a0[l]) != cudaSuccess || cudaEventCreate(&m->a1[l]) != cudaSuccess)
            return bail(fail(DBK_ECUDA, "model_create: events"));
    *out = m;
    return DBK_OK;
}

dbk_status dbk_model_destroy(dbk_model *m) {
    if (!m) return DBK_OK;
    cudaSetDevice(m->device);  // the pool may already be gone
    cudaDeviceSynchronize();
    delete m;
    return DBK_OK;
}

dbk_status dbk_model_step(dbk_model *m, int32_t n, const int64_t *ids, int32_t fuse_stats, void *logits,
                          void *stream) {
    return dbk_model_step_pd(m, n, ids, nullptr, fuse_stats, logits, nullptr, nullptr, stream);
}

dbk_status dbk_model_step_pd(dbk_model *m, int32_t n, const int64_t *ids, const dbk_prefill_batch *chunks,
                             int32_t fuse_stats, void *logits, const int32_t *tokens, int32_t *sampled,
                             void *stream) {
    if (!m) return fail(DBK_EINVAL, "model_step: null model");
    if (n < 0 || (n > 0 && !ids)) return fail(DBK_EINVAL, "model_step: bad batch");
    const int32_t nch = chunks ? chunks->n : 0;
    if (nch < 0 || (nch > 0 && (!chunks->req_ids || !chunks->q_start || !chunks->q_len)))
        return fail(DBK_EINVAL, "model_step: bad chunk arrays");
    dbk_pool *p = m->pool;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DBK_CUDA(cudaSetDevice(p->cfg.device));
    DBK_TRY(collect_timing(m));
    // activation rows: the decode tokens (batch order), then every chunk's tokens
    m->rows_h.clear();
    for (int32_t i = 0; i < n; ++i) {
        auto it = p->reqs.find(ids[i]);
        if (it == p->reqs.end()) return fail(DBK_ENOENT, "model_step: unknown request %lld", static_cast<long long>(ids[i]));
        if (it->second.ctx < 1) return fail(DBK_EINVAL, "model_step: request without a reserved decode token");
        m->rows_h.push_back({ids[i], it->second.slot, it->second.ctx - 1});
    }
    for (int32_t c = 0; c < nch; ++c) {
        auto it = p->reqs.find(chunks->req_ids[c]);
        if (it == p->reqs.end())
            return fail(DBK_ENOENT, "model_step: unknown request %lld", static_cast<long long>(chunks->req_ids[c]));
        const int32_t s0 = chunks->q_start[c], len = chunks->q_len[c];
        if (s0 < 0 || len < 1 || static_cast<int64_t>(s0) + len > it->second.ctx)
            return fail(DBK_EINVAL, "model_step: chunk %d outside the reserved tokens", c);
        for (int32_t j = 0; j < len; ++j) m->rows_h.push_back({chunks->req_ids[c], it->second.slot, s0 + j});
    }
    const int R = static_cast<int>(m->rows_h.size());
    if (R == 0) return DBK_OK;
    if (R > m->rows) return fail(DBK_EINVAL, "model_step: %d rows > max_requests (%d)", R, m->rows);
    for (const RowMeta &r : m->rows_h)
        if (r.pos >= m->cfg.max_pos) return fail(DBK_EINVAL, "model_step: position beyond max_pos");
    DBK_TRY(flush_deltas(p, s));
    if (n > 0) DBK_TRY(prepare_batch(p, n, ids, s));
    DBK_TRY(m->up_rows.upload(m->rows_h.data(), m->rows_h.size() * sizeof(RowMeta), s));
    const RowMeta *rows = static_cast<const RowMeta *>(m->up_rows.dev);
    const int H = m->H, F = m->F, qd = m->Hq * m->d;
    const float eps = static_cast<float>(m->cfg.rms_eps);
    const bool tp = m->tp != nullptr;
    if (m->G > 1 && !tp) return fail(DBK_EINVAL, "model_step: tensor-parallel model without dbk_model_attach_tp");
    const int own_n = H / m->G, own0 = m->tp_r * own_n;
    // RMSNorm of the residual stream into h.  One GPU: x in place.  Tensor parallel: buffer k of
    // the rotation is read from its owners, this rank's slice is added into buffer k + 1 (the next
    // residual GEMM's target) unless `last`, and buffer k + 2 is cleared.
    auto norm = [&](const __half *gain, bool embed, bool last) -> dbk_status {
        if (!tp) {
            if (embed) {
                norm_kernel<<<R, 256, 0, s>>>(m->x, gain, eps, H, m->h, rows, m->embed, m->cfg.token_seed, m->V, tokens,
                                              tokens ? n : 0);
                DBK_CUDA(cudaGetLastError());
                return DBK_OK;
            }
            DBK_CUDA(launch_kernel(norm_kernel, dim3(R), dim3(256), 0, s, true, m->x, gain, eps, H, m->h,
                                   static_cast<const RowMeta *>(nullptr), static_cast<const __half *>(nullptr),
                                   uint64_t{0}, 0, static_cast<const int32_t *>(nullptr), 0));
            return DBK_OK;
        }
        const int k = m->tp_cur;
        const float *const *src = embed ? nullptr : tp_bufs_dev(m->tp, k);
        float *base = last ? nullptr : static_cast<float *>(tp_bufs(m->tp, k + 1)[m->tp_r]);
        float *zero = static_cast<float *>(tp_bufs(m->tp, k + 2)[m->tp_r]);
        DBK_CUDA(launch_kernel(tp_norm_kernel, dim3(R), dim3(256), 0, s, !embed, src, gain, eps, H, m->h,
                               embed ? rows : static_cast<const RowMeta *>(nullptr), m->embed, m->cfg.token_seed, m->V,
                               tokens, embed && tokens ? n : 0, own0, own_n, base, zero));
        m->tp_cur = (k + 1) % kTpBufs;  // the next residual GEMM accumulates into buffer k + 1
        return DBK_OK;
    };
    // x += (.) W^T: one GPU in place; tensor parallel -- every partial goes to the owner of its
    // columns in the current target buffer, then all ranks meet at a barrier
    std::vector<void *> tp_y;
    auto residual = [&](const __half *X, int K, const __half *W) -> dbk_status {
        GemmEpiArgs e = epi_plain(kEpiAcc32, m->x, H);
        if (tp) {
            void *const *bufs = tp_bufs(m->tp, m->tp_cur);
            tp_y.assign(bufs, bufs + m->G);
            e.y = tp_y[m->tp_r];
            e.tp_size = m->G;
            e.tp_cols = own_n;
            e.tp_y = tp_y.data();
        }
        DBK_TRY(gemm(m, R, H, K, X, W, e, s));
        if (tp) {
            DBK_TRY(tp_barrier(m->tp, s));
            ++p->n_launches;
        }
        return DBK_OK;
    };
    DBK_CUDA(cudaEventRecord(m->ev0, s));
    DBK_TRY(norm(m->lw[0].ln1, true, false));
    dbk_batch bt{};
    bt.n = n;
    bt.req_ids = ids;
    bt.chain = 2;  // right behind the QKV GEMM that writes q and the new K/V (waits for it)
    dbk_prefill_batch pb{};
    if (nch > 0) pb = *chunks;
    GemmEpiArgs rope;  // QKV epilogue: RoPE + the token's K/V into its page slot, q -> m->q
    rope.kind = kEpiRopeKV;
    rope.rows = rows;
    rope.bt = p->d_bt;
    rope.bt_stride = p->cfg.max_pages_per_req;
    rope.page_stride = p->page_stride;
    rope.tile_bytes = p->tile_bytes;
    rope.cs = m->cs;
    rope.q_heads = m->Hq;
    rope.kv_heads = m->Hkv;
    rope.head_dim = m->d;
    rope.q_out = m->q;
    const GemmEpiArgs silu = epi_plain(kEpiSiluMul, m->act, F);    // act = silu(gate) * up
    for (int l = 0; l < m->L; ++l) {
        const LayerW &w = m->lw[l];
        rope.kv_layer = p->kv + static_cast<size_t>(l) * p->layer_stride;
        DBK_TRY(gemm(m, R, m->nqkv, H, m->h, w.wqkv, rope, s));
        DBK_CUDA(cudaEventRecord(m->a0[l], s));
        if (n > 0 || (fuse_stats && l == 0)) {
            bt.layer = l;
            bt.fuse_stats = (fuse_stats && l == 0) ? 1 : 0;
            DBK_TRY(dbk_decode_step(p, &bt, m->q, m->attn, 0, s));
        }
        if (nch > 0) {  // the chunk rows' causal attention (K7, tensor cores)
            pb.layer = l;
            DBK_TRY(dbk_prefill_step(p, &pb, m->q + static_cast<size_t>(n) * qd, m->attn + static_cast<size_t>(n) * qd,
                                     0, s));
        }
        DBK_CUDA(cudaEventRecord(m->a1[l], s));
        DBK_TRY(residual(m->attn, qd, w.wo));
        DBK_TRY(norm(w.ln2, false, false));
        DBK_TRY(gemm(m, R, 2 * F, H, m->h, w.wgu, silu, s));
        DBK_TRY(residual(m->act, F, w.wdown));
        const bool last = l + 1 == m->L;
        DBK_TRY(norm(last ? m->lnf : m->lw[l + 1].ln1, false, last));
        DBK_CUDA(cudaGetLastError());
        p->n_launches += 6;  // 4 GEMMs, 2 norms (attention counts itself)
    }
    float *lg = logits ? static_cast<float *>(logits) : m->logits;
    DBK_TRY(gemm(m, R, m->V, H, m->h, m->lm, epi_plain(kEpiF32, lg, m->V), s));
    p->n_launches += 1;
    if (sampled) {
        argmax_kernel<<<R, 256, 0, s>>>(lg, m->V, sampled);
        DBK_CUDA(cudaGetLastError());
        ++p->n_launches;
    }
    if (tp) {  // every rank has read the step's last residual buffer before the next step reuses it
        DBK_TRY(tp_barrier(m->tp, s));
        ++p->n_launches;
    }
    DBK_CUDA(cudaEventRecord(m->ev1, s));
    m->pending = true;
    p->n_launches += 1;  // the embedding + first norm
    return DBK_OK;
}

dbk_status dbk_model_attach_tp(dbk_model *m, dbk_tp *t) {
    if (!m || !t) return fail(DBK_EINVAL, "model_attach_tp: null argument");
    if (tp_nranks(t) != m->G || tp_rank(t) != m->tp_r || tp_hidden(t) != m->H || tp_rows(t) < m->rows)
        return fail(DBK_EINVAL, "model_attach_tp: communicator (%d ranks, rank %d, hidden %d, %lld rows) does not match "
                                "the model (tp_size %d, tp_rank %d, hidden %d, %d rows)",
                    tp_nranks(t), tp_rank(t), tp_hidden(t), static_cast<long long>(tp_rows(t)), m->G, m->tp_r, m->H,
                    m->rows);
    m->tp = t;
    m->tp_cur = 0;
    return DBK_OK;
}

dbk_status dbk_model_buffers(dbk_model *m, void **p) {
    if (!m || !p) return fail(DBK_EINVAL, "model_buffers: null argument");
    void *b[8] = {m->x, m->h, nullptr, m->q, m->attn, nullptr, m->act, m->logits};
    for (int k = 0; k < 8; ++k) p[k] = b[k];
    return DBK_OK;
}

dbk_status dbk_model_timing(dbk_model *m, double *attn_ms, double *total_ms, int64_t *steps, int32_t reset) {
    if (!m) return fail(DBK_EINVAL, "model_timing: null model");
    DBK_TRY(collect_timing(m));
    if (attn_ms) *attn_ms = m->attn_ms;
    if (total_ms) *total_ms = m->total_ms;
    if (steps) *steps = m->steps;
    if (reset) {
        m->attn_ms = m->total_ms = 0;
        m->steps = 0;
    }
    return DBK_OK;
}

}  // extern "C"
