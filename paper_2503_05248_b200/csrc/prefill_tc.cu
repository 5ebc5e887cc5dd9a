// K7: paged chunked-prefill attention on the 5th-generation tensor cores (tcgen05 + TMEM)
// -- the dense contraction of PD fusion ("our method is also valid for
// determining chunk size").
//
// Query token j of a request's prefill chunk sits at position p = q_start + j and attends
// causally to keys 0..p of that request's paged KV (the chunk's own K/V already appended).
// A row is (chunk token, q-head of the kv group), token-major, so the GQA group shares every
// K/V page.  CTA = (pair of 128-row tiles A, B of one chunk, kv head g): both tiles consume
// the same K/V blocks (half the shared-memory traffic per flop of a single tile).
//   warp 8       TMA producer: 64-key blocks (4 pages) into a ring of block stages laid out
//                [K|V][d/64][64 keys][128 B] (128B swizzle), 4 boxes per page
//   warp 9       TMEM allocator (all 512 columns) + tcgen05.mma issuer (elected lane)
//   warps 0..3   softmax / correction / epilogue of tile A (thread t <-> TMEM lane t <-> row)
//   warps 4..7   the same for tile B
// Per 64-key block b and tile: S = Q K^T (M = 128, N = 64, K = d) lands in TMEM (double
// buffered); the softmax threads read their row with tcgen05.ld, keep a running max in log2
// units (O is rescaled in TMEM only when the max grows by > 2^8, so P <= 256), and write P
// back over S as packed 16-bit pairs; O += P V then takes A = P straight from TMEM
// (tcgen05.mma ... [tmem_a]) and B = V as an MN-major 128B-swizzled operand.  bf16 keeps P
// to ~16 bits with a hi + lo split (two PV MMAs per 16 keys).  S(b+2) reuses the columns of
// P(b): tcgen05.mma ops execute in issue order, so PV(b) has read P(b) before S(b+2) writes.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <type_traits>

#include "device_common.cuh"
#include "kernels.cuh"
#include "tc_common.cuh"

namespace dbk {
namespace {
using namespace dev;
using namespace tc;

constexpr int kRows = 128;      // MMA M: query rows per tile
constexpr int kBK = 64;         // keys per block (4 pages)
constexpr int kThreads = 320;   // 2 x 4 softmax warps + producer + MMA
constexpr int kTileCols = 256;  // TMEM columns per tile: S0 | S1 (64 each) | O (d <= 128)

// 2^x on the SFU (flush-to-zero; -inf -> +0)
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// Packed fp32 pairs (sm_100 FFMA2 / FADD2): one instruction for two lanes of work.
__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t r, float &a, float &b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
// one {64 elements x 16 tokens} box (2 KiB) of the (page, kv head) tile: d-half h of K or V
__device__ __forceinline__ void tma_box(void *dst, const CUtensorMap *map, int h, int kv, int tile, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(h), "r"(kv), "r"(tile), "r"(smem_u32(bar))
        : "memory");
}

template <typename T, int D, int GQ, int STG>
__global__ void __launch_bounds__(kThreads, 1)
prefill_tc_kernel(const PrefillParams p, const __grid_constant__ CUtensorMap tmap) {
    constexpr int NBOX = D / 64;
    constexpr int HALF = kBK * 128;                  // one d-half of K or V of a block: 8 KiB
    constexpr int STAGE = 2 * NBOX * HALF;           // K | V of a 64-key block
    constexpr int QT = NBOX * kRows * 128;           // Q of one tile, [half][row][128 B]
    constexpr bool kBF16 = std::is_same<T, __nv_bfloat16>::value;
    constexpr int KSTEPS = D / 16;
    constexpr uint32_t kFmt = kBF16 ? 1u : 0u;
    constexpr uint32_t ID_S = idesc_f16(kFmt, 0, kRows, kBK);  // S = Q K^T per block
    constexpr uint32_t ID_O = idesc_f16(kFmt, 1, kRows, D);    // O += P V per 16 keys
    constexpr int QB = kRows / GQ;                            // chunk tokens per tile

    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t kv_full[STG], kv_empty[STG];
    __shared__ __align__(8) uint64_t s_full[2][2], p_full[2][2], o_done[2], q_ready;
    __shared__ uint32_t tmem_base_sh;

    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *q_s = smem;                 // [tile][half][row][128 B]
    uint8_t *ring = smem + 2 * QT;       // [stage][K|V][half][key][128 B]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const PrefTile tl = p.tiles[blockIdx.x];
    const int g = blockIdx.y;
    const int pos0 = tl.q_start + tl.j0;              // position of the pair's first token
    const int n_keys = pos0 + tl.rows_tok;            // keys seen by the pair's last token
    const int n_pages = (n_keys + kP - 1) / kP;
    const int n_blk = (n_keys + kBK - 1) / kBK;
    const bool has_b = tl.rows_tok > QB;
    const int nblk_a = (pos0 + min(QB, tl.rows_tok) - 1) / kBK + 1;
    const int32_t *bt_row = p.block_table + static_cast<size_t>(tl.slot) * p.bt_stride;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STG; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        for (int t = 0; t < 2; ++t) {
            for (int k = 0; k < 2; ++k) {
                mbar_init(&s_full[t][k], 1);
                mbar_init(&p_full[t][k], kRows);
            }
            mbar_init(&o_done[t], 1);  // one phase: the tile's last PV
        }
        mbar_init(&q_ready, 2 * kRows);
        fence_mbar_init();
    }
    if (warp == 9) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    if (warp == 8) {
        // ---------------- TMA producer: block b = pages 4b .. 4b+3 into stage b % STG
        const int64_t tile_layer = static_cast<int64_t>(p.layer) * p.cap_pages;
        for (int b = 0; b < n_blk; ++b) {
            const int np = min(4, n_pages - 4 * b);
            const int ph = lane < np ? __ldg(bt_row + 4 * b + lane) : 0;
            const int st = b % STG;
            if (lane == 0) {
                if (b >= STG) mbar_wait(&kv_empty[st], ((b / STG) - 1) & 1);
                mbar_expect_tx(&kv_full[st], np * 2 * NBOX * 2048);
            }
            __syncwarp();
            if (lane < np) {
                const int tile = static_cast<int>((tile_layer + ph) * p.kv_heads + g);
                uint8_t *sb = ring + st * STAGE + lane * 2048;
#pragma unroll
                for (int kv = 0; kv < 2; ++kv)
#pragma unroll
                    for (int h = 0; h < NBOX; ++h) tma_box(sb + (kv * NBOX + h) * HALF, &tmap, h, kv, tile, &kv_full[st]);
            }
        }
    } else if (warp == 9) {
        // ---------------- MMA issuer: the whole warp runs the schedule (warp-uniform
        // descriptor math on the uniform datapath), one elected lane issues each tcgen05 op
        {
            mbar_wait(&q_ready, 0);
            tc_fence_after();
            const uint32_t q_addr = smem_u32(q_s), ring_addr = smem_u32(ring);
            auto issue_pv = [&](int c) {
                const int st = c % STG;
                for (int t = 0; t < 2; ++t) {
                    if (t == 0 ? c >= nblk_a : !has_b) continue;
                    mbar_wait(&p_full[t][c & 1], (c >> 1) & 1);
                    tc_fence_after();
                    const uint32_t tp = tmem + t * kTileCols + (c & 1) * 64, to = tmem + t * kTileCols + 128;
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        const uint64_t vdesc = smem_desc(ring_addr + st * STAGE + NBOX * HALF + kk * 2048, HALF, 1024, 2);
                        umma_ts(to, tp + kk * 8, vdesc, ID_O, (c > 0 || kk > 0) ? 1u : 0u);
                        if constexpr (kBF16) umma_ts(to, tp + 32 + kk * 8, vdesc, ID_O, 1u);
                    }
                    // the tile's O is final after its last PV: one commit, one phase (the
                    // epilogue's only wait on it)
                    if (c == (t == 0 ? nblk_a : n_blk) - 1) umma_commit(&o_done[t]);
                }
                // every phase of kv_empty is observed by the producer before the next one
                // completes; the softmax threads also wait on it to know PV(c) is done
                umma_commit(&kv_empty[st]);
            };
            for (int b = 0; b < n_blk; ++b) {
                const int st = b % STG;
                mbar_wait(&kv_full[st], (b / STG) & 1);
                tc_fence_after();
                for (int t = 0; t < 2; ++t) {
                    if (t == 0 ? b >= nblk_a : !has_b) continue;
                    // S(b) overwrites P(b-2) in TMEM with no wait: tcgen05.mma ops of a CTA
                    // execute in issue order (scratch/umma_war.cu: 0 of 3.8e7 rows corrupted)
                    const uint32_t ts = tmem + t * kTileCols + (b & 1) * 64;
#pragma unroll
                    for (int kk = 0; kk < KSTEPS; ++kk) {
                        const uint32_t half = kk >> 2, koff = (kk & 3) * 32;
                        const uint64_t qdesc = smem_desc(q_addr + t * QT + half * (kRows * 128) + koff, 16, 1024, 2);
                        const uint64_t kdesc = smem_desc(ring_addr + st * STAGE + half * HALF + koff, 16, 1024, 2);
                        umma_ss(ts, qdesc, kdesc, ID_S, kk > 0 ? 1u : 0u);
                    }
                    umma_commit(&s_full[t][b & 1]);
                }
                if (b >= 1) issue_pv(b - 1);
            }
            issue_pv(n_blk - 1);
        }
    } else {
        // ---------------- softmax / correction / epilogue: thread owns row r of tile t
        const int t = warp >> 2;
        const int r = threadIdx.x & 127;
        const int jt = t * QB + r / GQ;            // token of this row within the pair
        const bool row_ok = jt < tl.rows_tok;
        const int p_row = pos0 + jt;
        const int h = g * GQ + r % GQ;
        {   // Q row -> shared memory, 128B-swizzled K-major (rows of the A operand)
            const T *src = reinterpret_cast<const T *>(p.q) +
                           (static_cast<size_t>(tl.q_row0 + tl.j0 + (row_ok ? jt : 0)) * p.q_heads + h) * D;
            uint8_t *qt = q_s + t * QT;
#pragma unroll
            for (int c = 0; c < D / 8; ++c) {
                uint4 v = row_ok ? __ldg(reinterpret_cast<const uint4 *>(src) + c) : make_uint4(0u, 0u, 0u, 0u);
                const int half = c >> 3, ch = c & 7;
                *reinterpret_cast<uint4 *>(qt + half * (kRows * 128) + r * 128 + ((ch ^ (r & 7)) << 4)) = v;
            }
            fence_proxy_async();
            mbar_arrive(&q_ready);
        }
        const int my_blk = t == 0 ? nblk_a : (has_b ? n_blk : 0);
        // the tile that processes the last block zeroes its never-valid V rows (P = 0 there,
        // but 0 * NaN from never-written pool slots or stale shared memory would poison O)
        const bool zero_tail = ((t == 0) == (nblk_a == n_blk)) && (n_keys & (kBK - 1)) != 0;
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t tm = tmem + t * kTileCols + lane_base;
        const float c_log2 = p.scale_log2;
        float M = -INFINITY, L = 0.f;
        for (int b = 0; b < my_blk; ++b) {
            mbar_wait(&s_full[t][b & 1], (b >> 1) & 1);
            tc_fence_after();
            const uint32_t ts = tm + (b & 1) * 64;
            uint32_t u[64];
            tmem_ld32(ts, *reinterpret_cast<uint32_t(*)[32]>(u));
            tmem_ld32(ts + 32, *reinterpret_cast<uint32_t(*)[32]>(u + 32));
            tmem_ld_wait();
            float s[64];
            float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
            const int vis = row_ok ? p_row - b * kBK : -1;  // keys k <= vis of this block are visible
            if (vis >= kBK - 1) {
#pragma unroll
                for (int k = 0; k < 64; ++k) s[k] = __uint_as_float(u[k]);
            } else {
#pragma unroll
                for (int k = 0; k < 64; ++k) s[k] = k <= vis ? __uint_as_float(u[k]) : -INFINITY;
            }
#pragma unroll
            for (int k = 0; k < 64; k += 2) mx[(k >> 1) & 3] = fmax3(mx[(k >> 1) & 3], s[k], s[k + 1]);
            const float bmax = fmaxf(fmax3(mx[0], mx[1], mx[2]), mx[3]);
            const float m_new = fmaxf(M, bmax * c_log2);
            const bool grow = m_new > M + 8.f;  // rescale only when the max grows by > 2^8
            if (b > 0 && __any_sync(kFull, grow)) {
                const float f = grow ? exp2f(M - m_new) : 1.f;
                // O holds blocks < b: wait for PV(b-1) through the commit onto kv_empty of
                // block b-1's stage (phase (b-1)/STG).  Valid parity wait: that barrier's
                // previous phase (block b-1-STG <= b-2) is complete -- the commit behind S(b)
                // covers the earlier-issued PV(b-2) -- and its next one (block b-1+STG) needs
                // this thread's own P(b-1+STG), so it cannot have completed yet.
                mbar_wait(&kv_empty[(b - 1) % STG], ((b - 1) / STG) & 1);
                tc_fence_after();
#pragma unroll
                for (int c0 = 0; c0 < D; c0 += 32) {
                    uint32_t o[32];
                    tmem_ld32(tm + 128 + c0, o);
                    tmem_ld_wait();
#pragma unroll
                    for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * f);
                    tmem_st32(tm + 128 + c0, o);
                }
                if (grow) L *= f;
            }
            if (grow) M = m_new;
            // P = exp2(s c - M) <= 2^8 as packed 16-bit pairs over S: hi in columns 0..31, lo in
            // 32..63.  bf16: hi = P truncated to its top 16 bits (one byte permute per pair),
            // lo = the exact fp32 remainder rounded to bf16 -- ~17 significant bits in all.
            const float nm = (M == -INFINITY) ? 0.f : -M;
            const uint64_t c2 = f2_pack(c_log2, c_log2), nm2 = f2_pack(nm, nm);
            uint64_t L2 = f2_pack(0.f, 0.f);
#pragma unroll
            for (int k0 = 0; k0 < 64; k0 += 32) {
                uint32_t hi[16], lo[16];
#pragma unroll
                for (int k = 0; k < 32; k += 2) {
                    float x0, x1, p0, p1;
                    f2_unpack(ffma2(f2_pack(s[k0 + k], s[k0 + k + 1]), c2, nm2), x0, x1);
                    p0 = ex2_approx(x0);
                    p1 = ex2_approx(x1);
                    const uint64_t pp = f2_pack(p0, p1);
                    L2 = fadd2(L2, pp);
                    if constexpr (kBF16) {
                        const uint32_t u0 = __float_as_uint(p0), u1 = __float_as_uint(p1);
                        hi[k >> 1] = __byte_perm(u0, u1, 0x7632);
                        float r0, r1;
                        f2_unpack(fadd2(pp, f2_pack(-__uint_as_float(u0 & 0xFFFF0000u), -__uint_as_float(u1 & 0xFFFF0000u))),
                                  r0, r1);
                        lo[k >> 1] = Elt<T>::from_f2(r0, r1);
                    } else {
                        hi[k >> 1] = Elt<T>::from_f2(p0, p1);
                    }
                }
                tmem_st16(ts + (k0 >> 1), hi);
                if constexpr (kBF16) tmem_st16(ts + 32 + (k0 >> 1), lo);
            }
            float La, Lb;
            f2_unpack(L2, La, Lb);
            if (zero_tail && b == n_blk - 1) {
                uint8_t *vt = ring + (b % STG) * STAGE + NBOX * HALF;
                const int v0 = n_keys & (kBK - 1);
                for (int x = r; x < (kBK - v0) * NBOX * 8; x += kRows) {
                    const int row = v0 + x / (NBOX * 8), rem = x % (NBOX * 8);
                    *reinterpret_cast<uint4 *>(vt + (rem >> 3) * HALF + row * 128 + (rem & 7) * 16) = make_uint4(0u, 0u, 0u, 0u);
                }
                fence_proxy_async();
            }
            L += La + Lb;
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&p_full[t][b & 1]);
        }
        if (my_blk > 0) {
            // epilogue: O / L for this row, once the tile's last PV has completed (o_done has
            // exactly one phase)
            mbar_wait(&o_done[t], 0);
            tc_fence_after();
            const float inv = 1.f / L;
            const size_t ob = (static_cast<size_t>(tl.q_row0 + tl.j0 + jt) * p.q_heads + h) * D;
#pragma unroll
            for (int c0 = 0; c0 < D; c0 += 32) {
                uint32_t o[32];
                tmem_ld32(tm + 128 + c0, o);
                tmem_ld_wait();
                if (row_ok) {
#pragma unroll
                    for (int k = 0; k < 32; k += 8) {
                        float v8[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) v8[e] = __uint_as_float(o[k + e]) * inv;
                        store8_out(p.out, ob + c0 + k, p.out_dtype, v8);
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

template <int D>
constexpr int prefill_stages() {
    return D == 128 ? 4 : 6;
}
template <int D>
constexpr size_t prefill_smem() {
    return 2 * static_cast<size_t>(D / 64) * kRows * 128 +
           static_cast<size_t>(prefill_stages<D>()) * 2 * (D / 64) * kBK * 128 + 1024;
}

template <typename T, int D, int GQ>
cudaError_t launch_prefill_t(const PrefillParams &p, int n_tiles, int kv_heads, const CUtensorMap &tmap,
                             cudaStream_t s) {
    auto kern = prefill_tc_kernel<T, D, GQ, prefill_stages<D>()>;
    constexpr size_t smem = prefill_smem<D>();
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

int prefill_rows_per_tile() { return 2 * kRows; }

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
