// sm_100a kernels of the decode hot path:
//   (K1 lives in decode_mha.cu, K2 in decode_gqa.cu)
//   K5/K6     append_kernel   KV append (explicit rows or the synthetic generator)
//             bt_apply_kernel block-table deltas (new pages, cleared rows)
//             synth_*         input-side generator (synth/hashgen.py on the device)
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>

#include "device_common.cuh"
#include "kernels.cuh"

namespace dbk {
namespace {
using namespace dev;

// ------------------------------------------------------------------ K5/K6: KV append
template <typename T, int D>
__global__ void __launch_bounds__(256) append_kernel(const AppendParams p) {
    constexpr int VPR = D / 8;  // 16-byte vectors per row
    const AppendJob job = p.jobs[blockIdx.x];
    const int layer = p.layer0 + blockIdx.y;
    const int rows_per_block = job.ntok;  // rows of one (head, K|V) tile this job writes
    const int total = p.kv_heads * 2 * rows_per_block * VPR;
    uint8_t *page = p.kv + static_cast<size_t>(layer) * p.layer_stride +
                    static_cast<size_t>(job.phys) * p.page_stride;
    const float scale = 1.0f / 128.0f;
    // the request's first hash of K (kind 1) and V (kind 2), once per thread
    const uint64_t k1k = job.src_row < 0 ? synth_key1(p.seed, 1, job.req_id) : 0;
    const uint64_t k1v = job.src_row < 0 ? synth_key1(p.seed, 2, job.req_id) : 0;
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
            synth_vals(synth_key2(kv ? k1v : k1k, pos, layer, p.head0 + head, v), scale, f);
            val = pack8<T>(f);
        } else {
            const size_t srow = p.src_layer_rows > 0
                                    ? static_cast<size_t>(layer) * p.src_layer_rows + job.src_row + tok
                                    : static_cast<size_t>(job.src_row + tok) * p.layers + layer;
            const T *src = reinterpret_cast<const T *>(kv ? p.v_src : p.k_src) +
                           (srow * p.kv_heads + head) * D +
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
// block (row chunk, layer): the chunk's rows one after the other, the threads over (head, 8-value
// group) -- no 64-bit index divisions, and the request's first hash once per row
__global__ void __launch_bounds__(256) synth_q_kernel(uint64_t seed, const ReqMeta *req, int n, int rows_per_block,
                                                      int layer_rows, int q_heads, int head0, int vshift, float scale,
                                                      int dtype, void *q) {
    const int l = blockIdx.y;
    const int hv = q_heads << vshift, d = 8 << vshift;
    const int r1 = min(n, (static_cast<int>(blockIdx.x) + 1) * rows_per_block);
    for (int r = blockIdx.x * rows_per_block; r < r1; ++r) {
        const ReqMeta rm = req[r];
        const uint64_t k1 = synth_key1(seed, 0, rm.req_id);
        for (int t = threadIdx.x; t < hv; t += blockDim.x) {
            const int h = t >> vshift, v = t & ((1 << vshift) - 1);
            float f[8];
            synth_vals(synth_key2(k1, rm.ctx - 1, l, head0 + h, v), scale, f);
            store8(q, ((static_cast<size_t>(l) * layer_rows + r) * q_heads + h) * d + v * 8, dtype, f);
        }
    }
}

// rows of every layer: out[l][row0 + r][h][:] = synth(seed, kind, req[r], pos[r], l, h), layer l at
// out + l * layer_rows rows (PD fusion: the prefill chunk's q, one launch per step).
__global__ void synth_rows_layers_kernel(uint64_t seed, int kind, int n_rows, const int64_t *req, const int32_t *pos,
                                         int layers, int layer_rows, int row0, int n_heads, int head0, int d,
                                         float scale, int dtype, void *out) {
    const int vpr = d / 8;
    const long per_layer = static_cast<long>(n_rows) * n_heads * vpr;
    const long total = per_layer * layers;
    for (long k = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; k < total;
         k += static_cast<long>(gridDim.x) * blockDim.x) {
        const int l = static_cast<int>(k / per_layer);
        const long kk = k % per_layer;
        const int v = static_cast<int>(kk % vpr);
        const long rh = kk / vpr;
        const int h = static_cast<int>(rh % n_heads);
        const int r = static_cast<int>(rh / n_heads);
        float f[8];
        synth_vals(synth_key(seed, kind, req[r], pos[r], l, head0 + h, v), scale, f);
        store8(out, ((static_cast<size_t>(l) * layer_rows + row0) * n_heads + rh) * d + v * 8, dtype, f);
    }
}

int grid_for(long work, int block) {
    long b = (work + block - 1) / block;
    if (b > 148L * 16) b = 148L * 16;
    return static_cast<int>(b < 1 ? 1 : b);
}

}  // namespace

cudaError_t launch_append(const AppendParams &p, int kv_dtype, int head_dim, cudaStream_t s) {
    if (p.n_jobs <= 0) return cudaSuccess;
    dim3 grid(p.n_jobs, p.n_launch_layers > 0 ? p.n_launch_layers : p.layers);
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

cudaError_t launch_synth_rows_layers(uint64_t seed, int kind, int n_rows, const int64_t *req, const int32_t *pos,
                                    int layers, int layer_rows, int row0, int n_heads, int head0, int d,
                                    int scale_log2, int dtype, void *out, cudaStream_t s) {
    const long work = static_cast<long>(n_rows) * layers * n_heads * (d / 8);
    if (work <= 0) return cudaSuccess;
    synth_rows_layers_kernel<<<grid_for(work, 256), 256, 0, s>>>(seed, kind, n_rows, req, pos, layers, layer_rows,
                                                                 row0, n_heads, head0, d, ldexpf(1.0f, scale_log2 - 7),
                                                                 dtype, out);
    return cudaGetLastError();
}

cudaError_t launch_synth_q(uint64_t seed, const ReqMeta *req, int n, int layers, int layer_rows,
                           int q_heads, int head0, int d, int scale_log2, int dtype, void *q, cudaStream_t s) {
    if (n <= 0 || layers <= 0) return cudaSuccess;
    if (d != 64 && d != 128) return cudaErrorInvalidValue;
    const int vshift = d == 128 ? 4 : 3;
    // ~4 row blocks per SM over all layers, at least one row each
    const int rows_per_block = std::max(1, std::min(n, (n * layers + 148 * 4 - 1) / (148 * 4)));
    const dim3 grid((n + rows_per_block - 1) / rows_per_block, layers);
    synth_q_kernel<<<grid, 256, 0, s>>>(seed, req, n, rows_per_block, layer_rows, q_heads, head0, vshift,
                                        ldexpf(1.0f, scale_log2 - 7), dtype, q);
    return cudaGetLastError();
}

// Read-only streaming probe (measurement utility, not part of the method): every byte of
// `buf` is read once with 16-byte non-allocating loads, 8 independent loads in flight per
// thread, grid = SMs x 8 CTAs; the XOR of the data goes to `sink` so nothing is elided.
__global__ void __launch_bounds__(512) read_probe_kernel(const uint4 *__restrict__ buf, size_t n16, uint32_t *sink) {
    uint32_t x = 0;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    for (; k + 7 * stride < n16; k += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                         : "l"(buf + k + u * stride));
#pragma unroll
        for (int u = 0; u < 8; ++u) x ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; k < n16; k += stride) {
        const uint4 v = buf[k];
        x ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (x == 0x9E3779B9u) sink[0] = x;  // practically never taken; keeps the loads live
}

cudaError_t launch_read_probe(const void *buf, size_t bytes, uint32_t *sink, int sms, cudaStream_t s) {
    read_probe_kernel<<<sms * 4, 512, 0, s>>>(static_cast<const uint4 *>(buf), bytes / 16, sink);
    return cudaGetLastError();
}

}  // namespace dbk
