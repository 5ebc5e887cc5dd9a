// K7: paged chunked-prefill attention on the 5th-generation tensor cores (tcgen05 + TMEM)
// -- the dense contraction of PD fusion ("our method is also valid for
// determining chunk size").
//
// Query token j of a request's prefill chunk sits at position p = q_start + j and attends
// causally to keys 0..p of that request's paged KV (the chunk's own K/V already appended).
// CTA = (tile of 128 query rows, kv head g); a row is (chunk token, q-head of the group),
// token-major, so GQA groups share every K/V page.  Warp roles (192 threads):
//   warp 4      TMA producer: one 5-D tensor-map box per (page, kv head) tile into a ring
//   warp 5      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 0..3  softmax / O correction / epilogue, thread t <-> TMEM lane t <-> query row t
// Per block of 4 pages (64 keys): S = Q K^T (M = 128, N = 16 per page, K = d) lands in TMEM
// (double buffered); the softmax threads read their row with tcgen05.ld, keep a per-row
// running max in log2 units (O is rescaled in TMEM only when the max grows by > 2^8, so P
// stays <= 256), write P to shared memory in the canonical no-swizzle K-major layout, and
// O += P V runs as M = 128, N = d, K = 16 per page with V as an MN-major 128B-swizzled
// operand straight from the TMA tile.  bf16 keeps P to ~16 bits with a hi + lo split.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <type_traits>

#include "device_common.cuh"
#include "kernels.cuh"

namespace dbk {
namespace {
using namespace dev;

constexpr int kRows = 128;     // MMA M: query rows per tile
constexpr int kNB = 4;         // pages per softmax block (64 keys)
constexpr int kStages = 12;    // page-tile ring depth (>= 2 blocks in flight)
constexpr int kThreads = 192;  // 4 softmax warps + producer + MMA

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return static_cast<uint64_t>((addr & 0x3FFFFu) >> 4) | (static_cast<uint64_t>(lbo >> 4) << 16) |
           (static_cast<uint64_t>(sbo >> 4) << 32) | (1ull << 46) | (static_cast<uint64_t>(layout) << 61);
}
// kind::f16 instruction descriptor: fp32 accumulate, A/B format (0 f16, 1 bf16), B major.
__host__ __device__ constexpr uint32_t idesc_f16(uint32_t fmt, uint32_t b_mn_major, uint32_t m, uint32_t n) {
    return (1u << 4) | (fmt << 7) | (fmt << 10) | (b_mn_major << 16) | ((n >> 3) << 17) | ((m >> 4) << 24);
}
__device__ __forceinline__ void umma_ss(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(r[k]);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])),
        "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])),
        "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
        "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])),
        "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31])));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tma_tile5(void *dst, const CUtensorMap *map, int tile, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %2, %2, %2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(tile), "r"(smem_u32(bar))
        : "memory");
}

template <typename T, int D, int GQ>
__global__ void __launch_bounds__(kThreads, 1)
prefill_tc_kernel(const PrefillParams p, const __grid_constant__ CUtensorMap tmap) {
    constexpr int NBOX = D / 64;
    constexpr int TILE = 2 * NBOX * 2048;            // K | V of one (page, kv head)
    constexpr int QBYTES = NBOX * kRows * 128;       // Q tile, [half][row][128 B], 128B swizzle
    constexpr int PSLICE = kRows * 16 * 2;           // P of one page: 128 rows x 16 keys
    constexpr bool kBF16 = std::is_same<T, __nv_bfloat16>::value;
    constexpr int NPBUF = kBF16 ? 2 : 1;             // hi (+ lo) parts of P
    constexpr int KSTEPS = D / 16;
    constexpr uint32_t kFmt = kBF16 ? 1u : 0u;
    constexpr uint32_t ID_S = idesc_f16(kFmt, 0, kRows, 16);  // S = Q K^T per page
    constexpr uint32_t ID_O = idesc_f16(kFmt, 1, kRows, D);   // O += P V per page (V MN-major)
    constexpr int S_COLS = kNB * 16;                // TMEM columns per S buffer
    constexpr uint32_t TM_COLS = (2 * S_COLS + D) <= 256 ? 256 : 512;

    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    __shared__ __align__(8) uint64_t s_full[2], s_free[2], p_full, pv_done[2], q_ready;
    __shared__ uint32_t tmem_base_sh;

    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *q_s = smem;
    uint8_t *ring = smem + QBYTES;
    uint8_t *p_s = ring + kStages * TILE;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const PrefTile tl = p.tiles[blockIdx.x];
    const int g = blockIdx.y;
    const int p_last = tl.q_start + tl.j0 + tl.rows_tok - 1;  // last query position of the tile
    const int n_keys = p_last + 1;
    const int n_pages = (n_keys + kP - 1) / kP;
    const int n_blk = (n_pages + kNB - 1) / kNB;
    const int32_t *bt_row = p.block_table + static_cast<size_t>(tl.slot) * p.bt_stride;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(&s_full[k], 1);
            mbar_init(&s_free[k], kRows);
            mbar_init(&pv_done[k], 1);
        }
        mbar_init(&p_full, kRows);
        mbar_init(&q_ready, kRows);
        fence_mbar_init();
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(TM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    const uint32_t tm_s = tmem, tm_o = tmem + 2 * S_COLS;

    if (warp == 4) {
        // ---------------- TMA producer
        const int64_t tile_layer = static_cast<int64_t>(p.layer) * p.cap_pages;
        for (int base = 0; base < n_pages; base += 32) {
            const int ph_lane = base + lane < n_pages ? __ldg(bt_row + base + lane) : 0;
            const int cnt = min(32, n_pages - base);
            for (int k = 0; k < cnt; ++k) {
                const int gi = base + k;
                const int ph = __shfl_sync(kFull, ph_lane, k);
                if (lane == 0) {
                    const int st = gi % kStages;
                    if (gi >= kStages) mbar_wait(&empty[st], ((gi / kStages) - 1) & 1);
                    mbar_expect_tx(&full[st], TILE);
                    tma_tile5(ring + st * TILE, &tmap, static_cast<int>((tile_layer + ph) * p.kv_heads + g), &full[st]);
                }
            }
        }
    } else if (warp == 5) {
        // ---------------- MMA issuer (one thread)
        if (lane == 0) {
            mbar_wait(&q_ready, 0);
            tc_fence_after();
            const uint32_t q_addr = smem_u32(q_s), ring_addr = smem_u32(ring), p_addr = smem_u32(p_s);
            auto issue_pv = [&](int c) {
                mbar_wait(&p_full, c & 1);
                tc_fence_after();
                const int np = min(kNB, n_pages - c * kNB);
                for (int pj = 0; pj < np; ++pj) {
                    const int gi = c * kNB + pj, st = gi % kStages;
                    const uint64_t vdesc = smem_desc(ring_addr + st * TILE + NBOX * 2048, 2048, 1024, 2);
#pragma unroll
                    for (int h = 0; h < NPBUF; ++h) {
                        const uint64_t pdesc = smem_desc(p_addr + (h * kNB + pj) * PSLICE, 128, 256, 0);
                        umma_ss(tm_o, pdesc, vdesc, ID_O, (c > 0 || pj > 0 || h > 0) ? 1u : 0u);
                    }
                    umma_commit(&empty[st]);
                }
                umma_commit(&pv_done[c & 1]);
            };
            for (int b = 0; b < n_blk; ++b) {
                if (b >= 2) mbar_wait(&s_free[b & 1], ((b >> 1) - 1) & 1);
                tc_fence_after();
                const int np = min(kNB, n_pages - b * kNB);
                for (int pj = 0; pj < np; ++pj) {
                    const int gi = b * kNB + pj, st = gi % kStages;
                    mbar_wait(&full[st], (gi / kStages) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < KSTEPS; ++kk) {
                        const uint32_t half = kk >> 2, koff = (kk & 3) * 32;
                        const uint64_t qdesc = smem_desc(q_addr + half * (kRows * 128) + koff, 16, 1024, 2);
                        const uint64_t kdesc = smem_desc(ring_addr + st * TILE + half * 2048 + koff, 16, 1024, 2);
                        umma_ss(tm_s + (b & 1) * S_COLS + pj * 16, qdesc, kdesc, ID_S, kk > 0 ? 1u : 0u);
                    }
                }
                umma_commit(&s_full[b & 1]);
                if (b >= 1) issue_pv(b - 1);
            }
            issue_pv(n_blk - 1);
        }
        __syncwarp();
    } else {
        // ---------------- softmax / correction / epilogue: thread t owns query row t
        const int r = threadIdx.x;
        const int jt = r / GQ;                     // token of this row within the tile
        const bool row_ok = jt < tl.rows_tok;
        const int p_row = tl.q_start + tl.j0 + jt;
        const int h = g * GQ + r % GQ;
        // Q row -> shared memory, 128B-swizzled K-major (rows of the A operand)
        {
            const T *src = reinterpret_cast<const T *>(p.q) +
                           (static_cast<size_t>(tl.q_row0 + tl.j0 + (row_ok ? jt : 0)) * p.q_heads + h) * D;
#pragma unroll
            for (int c = 0; c < D / 8; ++c) {
                uint4 v = row_ok ? __ldg(reinterpret_cast<const uint4 *>(src) + c) : make_uint4(0u, 0u, 0u, 0u);
                const int half = c >> 3, ch = c & 7;
                *reinterpret_cast<uint4 *>(q_s + half * (kRows * 128) + r * 128 + ((ch ^ (r & 7)) << 4)) = v;
            }
            fence_proxy_async();
            mbar_arrive(&q_ready);
        }
        const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
        float M = -INFINITY, L = 0.f;
        for (int b = 0; b < n_blk; ++b) {
            mbar_wait(&s_full[b & 1], (b >> 1) & 1);
            tc_fence_after();
            float s[S_COLS];
            tmem_ld32(tm_s + lane_base + (b & 1) * S_COLS, *reinterpret_cast<float(*)[32]>(s));
            tmem_ld32(tm_s + lane_base + (b & 1) * S_COLS + 32, *reinterpret_cast<float(*)[32]>(s + 32));
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&s_free[b & 1]);
            float bmax = -INFINITY;
#pragma unroll
            for (int c = 0; c < S_COLS; ++c) {
                const int key = b * S_COLS + c;
                s[c] = (row_ok && key <= p_row) ? s[c] * p.scale_log2 : -INFINITY;
                bmax = fmaxf(bmax, s[c]);
            }
            if (b > 0) {  // PV of the previous block done: P buffer free, O stable
                mbar_wait(&pv_done[(b - 1) & 1], ((b - 1) >> 1) & 1);
                tc_fence_after();
            }
            const float m_new = fmaxf(M, bmax);
            const bool grow = m_new > M + 8.f;  // rescale only when the max grows by > 2^8
            const float f = grow ? ((M == -INFINITY) ? 0.f : exp2f(M - m_new)) : 1.f;
            if (b > 0 && __any_sync(kFull, grow)) {
#pragma unroll
                for (int c0 = 0; c0 < D; c0 += 32) {
                    float o[32];
                    tmem_ld32(tm_o + lane_base + c0, o);
                    tmem_ld_wait();
#pragma unroll
                    for (int k = 0; k < 32; ++k) o[k] *= f;
                    tmem_st32(tm_o + lane_base + c0, o);
                }
                tmem_st_wait();
            }
            if (grow) {
                L *= f;
                M = m_new;
            }
            // P = exp2(s - M) (<= 2^8), stored per page as [16 row groups][2 k-halves][8 rows][16 B]
#pragma unroll
            for (int pj = 0; pj < kNB; ++pj) {
                float pv[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const float x = s[pj * 16 + k];
                    pv[k] = (x == -INFINITY) ? 0.f : exp2f(x - M);
                    L += pv[k];
                }
#pragma unroll
                for (int kh = 0; kh < 2; ++kh) {
                    float hi[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) hi[k] = pv[kh * 8 + k];
                    const uint4 ph = pack8<T>(hi);
                    uint8_t *dst = p_s + pj * PSLICE + (r >> 3) * 256 + kh * 128 + (r & 7) * 16;
                    *reinterpret_cast<uint4 *>(dst) = ph;
                    if constexpr (kBF16) {
                        float lo[8], ht[8];
                        unpack8<T>(ph, ht);
#pragma unroll
                        for (int k = 0; k < 8; ++k) lo[k] = hi[k] - ht[k];
                        *reinterpret_cast<uint4 *>(dst + kNB * PSLICE) = pack8<T>(lo);
                    }
                }
            }
            // never-written V slots of a partial last page could hold NaN: zero them (P = 0 there)
            if (b == n_blk - 1 && (n_keys & (kP - 1))) {
                const int gi = n_pages - 1, st = gi % kStages, v0 = n_keys & (kP - 1);
                uint8_t *vt = ring + st * TILE + NBOX * 2048;
                for (int x = r; x < (kP - v0) * NBOX * 8; x += kRows) {
                    const int row = v0 + x / (NBOX * 8), rem = x % (NBOX * 8);
                    *reinterpret_cast<uint4 *>(vt + (rem >> 3) * 2048 + row * 128 + (rem & 7) * 16) = make_uint4(0u, 0u, 0u, 0u);
                }
            }
            fence_proxy_async();
            tc_fence_before();
            mbar_arrive(&p_full);
        }
        // epilogue: O / L for this row
        mbar_wait(&pv_done[(n_blk - 1) & 1], ((n_blk - 1) >> 1) & 1);
        tc_fence_after();
        const float inv = 1.f / L;
        const size_t ob = (static_cast<size_t>(tl.q_row0 + tl.j0 + jt) * p.q_heads + h) * D;
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 32) {
            float o[32];
            tmem_ld32(tm_o + lane_base + c0, o);
            tmem_ld_wait();
            if (row_ok) {
#pragma unroll
                for (int k = 0; k < 32; k += 8) {
                    float v8[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) v8[e] = o[k + e] * inv;
                    store8_out(p.out, ob + c0 + k, p.out_dtype, v8);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TM_COLS));
    }
}

template <typename T, int D>
constexpr size_t prefill_smem() {
    return static_cast<size_t>(D / 64) * kRows * 128 + static_cast<size_t>(kStages) * 2 * (D / 64) * 2048 +
           (std::is_same<T, __nv_bfloat16>::value ? 2 : 1) * kNB * kRows * 32 + 1024;
}

template <typename T, int D, int GQ>
cudaError_t launch_prefill_t(const PrefillParams &p, int n_tiles, int kv_heads, const CUtensorMap &tmap,
                             cudaStream_t s) {
    auto kern = prefill_tc_kernel<T, D, GQ>;
    constexpr size_t smem = prefill_smem<T, D>();
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    kern<<<dim3(n_tiles, kv_heads), kThreads, smem, s>>>(p, tmap);
    return cudaGetLastError();
}

template <typename T, int D>
cudaError_t prefill_group(const PrefillParams &p, int group, int n_tiles, int kv_heads, const CUtensorMap &tmap,
                          cudaStream_t s) {
    switch (group) {
        case 1: return launch_prefill_t<T, D, 1>(p, n_tiles, kv_heads, tmap, s);
        case 2: return launch_prefill_t<T, D, 2>(p, n_tiles, kv_heads, tmap, s);
        case 4: return launch_prefill_t<T, D, 4>(p, n_tiles, kv_heads, tmap, s);
        case 8: return launch_prefill_t<T, D, 8>(p, n_tiles, kv_heads, tmap, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

int prefill_rows_per_tile() { return kRows; }

cudaError_t launch_prefill(const PrefillParams &p, int kv_dtype, int head_dim, int group, int n_tiles,
                           int kv_heads, const CUtensorMap &tmap, cudaStream_t s) {
    if (n_tiles <= 0) return cudaSuccess;
    if (kv_dtype == 0) {
        if (head_dim == 128) return prefill_group<__half, 128>(p, group, n_tiles, kv_heads, tmap, s);
        if (head_dim == 64) return prefill_group<__half, 64>(p, group, n_tiles, kv_heads, tmap, s);
    } else {
        if (head_dim == 128) return prefill_group<__nv_bfloat16, 128>(p, group, n_tiles, kv_heads, tmap, s);
        if (head_dim == 64) return prefill_group<__nv_bfloat16, 64>(p, group, n_tiles, kv_heads, tmap, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace dbk
