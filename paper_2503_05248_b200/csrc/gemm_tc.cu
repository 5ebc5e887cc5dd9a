// Model GEMMs on the 5th-generation tensor cores (the decode step's
// QKV / O / gate-up / down / LM-head projections, "enlarged matrix dimensions in the
// matrix multiplication operations required for larger batches").
//
//   Y[M][N] = X[M][K] W[N][K]^T,  X = activations (M = batch rows <= a few hundred), W = weights.
//
// Swap-AB: the weight rows are the MMA's M side (128 per CTA, 256 per CTA pair with
// cta_group::2) and the activation rows its N side (BN <= 256), so the decode batch never pads
// an M = 128 tile.  D lives in TMEM: lane = weight row, column = activation row.
//   warp 0      TMA producer: 128B-swizzled {64 K x 128 weight rows} and {64 K x BN/CG act rows}
//               boxes into a ring of stages (CTA pairs: each CTA loads its half of both operands,
//               completion counted on the leader's barrier); the weight boxes of the first stages
//               are requested before the grid-dependency wait (weights never depend on the
//               previous kernel)
//   warp 1      TMEM owner (2 x BN columns: double-buffered accumulator) and, in the leader CTA,
//               the tcgen05.mma issuer (4 x K=16 MMAs per stage)
//   warps 2-5   epilogue, 32 activation rows at a time: tcgen05.ld of the thread's TMEM lane,
//               the fused elementwise op, the result transposed into a shared-memory chunk image
//               and written by TMA, double-buffered so the next chunk overlaps the store: per
//               warp ([32 m][32 n], bulk tensor store / reduce-add, no cross-warp barrier) or, for
//               RoPE, per CTA ([32 m][128], per-row bulk copies into q and the KV pages).
//               (Per-thread strided st.global of the accumulator columns cost ~1.4 us per 32 rows
//               whatever the element size: profiles/r02_gemm_trace.log.)
// Scheduling (persistent): GEMMs that ACCUMULATE into an fp32 output (the residual stream: O and
// down projections) are stream-K -- the (tile x k-block) iterations are split evenly over the CTA
// groups and every partial tile is added into the output by the TMA unit (cp.reduce.async.bulk
// .add), so no wave is partly idle and no CTA waits for another; the other GEMMs run whole tiles
// (no K split) round-robin, with the activation tile width BN chosen from a cost model of wave
// count x per-k-block time (MMA time vs the operand traffic, fitted as ~50 B/clk/SM; at M = 512
// the binding resource is the SM's shared-memory port -- every operand byte is written by TMA and
// read by the MMA -- which the two-pair activation multicast (NP = 2, opt-in) does not relieve).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <new>

#include "common.h"
#include "device_common.cuh"
#include "gemm.h"
#include "tc_common.cuh"

#ifndef OUTBUFS
#define OUTBUFS 2
#endif

namespace dbk {
namespace {
using namespace dev;
using namespace tc;

constexpr int kBM = 128;          // weight rows per CTA = TMEM lanes
constexpr int kBK = 64;           // K elements per stage: one 128-byte swizzled row
constexpr int kThreads = 192;     // warp 0 TMA, warp 1 TMEM + MMA, warps 2-5 epilogue
constexpr int kMaxStages = 8;
constexpr int kMaxTp = 8;         // tensor-parallel ranks a residual GEMM can route to
constexpr int kMaxBN = 256;
constexpr int kChunk = 32;                      // activation rows per epilogue chunk
constexpr int kStageOut = kChunk * kBM * 4;     // one chunk of fp32 outputs: 16 KiB
constexpr int kOutBufs = OUTBUFS;               // chunk images in flight (1: +1 operand stage)
constexpr int kDynSmem = 227 * 1024 - 4096;     // dynamic shared memory per CTA (static ~3.3 KiB)
constexpr int kRingBudget = kDynSmem - 1024 - kOutBufs * kStageOut;

// Output tensor maps: [0] the output; with tensor-parallel routing (GemmEpiArgs::tp_size > 1)
// [r] = rank r's residual stream, the owner of columns [r H/G, (r+1) H/G).
struct OutMaps {
    CUtensorMap m[kMaxTp];
};

struct KParams {
    int32_t M, N, K, BN, m_tiles, kb, groups, stages;
    int32_t units;
    int32_t stream_k;   // 1: contiguous iteration ranges (partial tiles reduce-added); 0: whole tiles
    int64_t T;          // units * kb
    uint64_t *trace;    // optional [CTA][8] %globaltimer phase stamps (experiments/gemm_bench.py --trace)
    int32_t dbg;        // measurement only: 1 = no MMAs (operand stream alone), 2 = no operand loads
    int32_t split;      // whole tiles, K split S ways (S > 1): segment = (unit, k-range); partials
                        // reduce-added into ws, the tile's last segment applies the epilogue
    int32_t ldw;        // ws row stride (= N)
    float *ws;
    int32_t *cnt;       // [units][CG] arrival counters (zero between launches)
    // whole tiles, last wave re-tiled (units_a < units): units [0, units_a) are (BN, m_tiles)
    // tiles of weight tiles [0, n_a); units [units_a, units) cover weight tiles [n_a, ...) with the
    // narrower activation tile BN_b (m_tiles_b per weight tile), so the wave that would run on a
    // fraction of the CTA groups at BN runs on more of them at BN_b
    int32_t units_a, n_a, BN_b, m_tiles_b;
    GemmEpiArgs e;
};

struct Seg {
    int32_t unit, k0, k1;
    int32_t j;  // split-K: this segment's K range index (0 otherwise)
};
// The next segment (one unit's k-block range) of group g.  Stream-K: the group's iteration range
// [it, it1); whole tiles: units g, g + G, g + 2G, ... (it counts the group's units).
__device__ __forceinline__ bool next_seg(const KParams &p, int g, int64_t &it, int64_t it1, Seg &s) {
    if (p.stream_k) {
        if (it >= it1) return false;
        s.unit = static_cast<int32_t>(it / p.kb);
        s.j = 0;
        s.k0 = static_cast<int32_t>(it % p.kb);
        s.k1 = static_cast<int32_t>(min(static_cast<int64_t>(p.kb), s.k0 + (it1 - it)));
        it += s.k1 - s.k0;
        return true;
    }
    if (p.split > 1) {
        const int64_t sx = g + it * p.groups;
        if (sx >= static_cast<int64_t>(p.units) * p.split) return false;
        const int j = static_cast<int>(sx % p.split);
        s.unit = static_cast<int32_t>(sx / p.split);
        s.j = j;
        s.k0 = j * p.kb / p.split;
        s.k1 = (j + 1) * p.kb / p.split;
        ++it;
        return true;
    }
    const int64_t u = g + it * p.groups;
    if (u >= p.units) return false;
    s.unit = static_cast<int32_t>(u);
    s.j = 0;
    s.k0 = 0;
    s.k1 = p.kb;
    ++it;
    return true;
}

template <int CG>
__device__ __forceinline__ void tma_load2d(void *dst, const CUtensorMap *map, int c0, int c1, uint32_t bar) {
    if constexpr (CG == 1) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
            : "memory");
    } else {
        asm volatile(
            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
            : "memory");
    }
}
// CTA-pair load multicast to the CTAs of `mask` (same shared-memory offset in each); completion is
// counted on the barrier at `bar`'s offset in the leader CTA of each destination's pair.
__device__ __forceinline__ void tma_load2d_mc(void *dst, const CUtensorMap *map, int c0, int c1, uint32_t bar,
                                              uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void tma_store2d(const CUtensorMap *map, const void *src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void tma_reduce_add2d(const CUtensorMap *map, const void *src, int c0, int c1) {
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(smem_u32(src))
                 : "memory");
}
// contiguous shared -> global bulk copy (16-B aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most kOutBufs - 1 of this thread's bulk groups still read shared memory
__device__ __forceinline__ void bulk_wait_read_buf() {
    if constexpr (kOutBufs == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Elementwise part of the epilogue.  Plain / SiLU / residual kinds: each epilogue warp owns its 32
// TMEM lanes (weight rows) and writes a private [32 m][32 n] chunk image (SiLU: [32 m][16 act
// columns]) that its lane 0 stores with one TMA op -- no cross-warp barrier.  RoPE: the four
// warps write one [32 m][128] image holding each head in logical order (per-row bulk copies).
template <int EPI>
__device__ __forceinline__ void epi_to_smem(const KParams &p, const float (&v)[32], int r, int n,
                                            const float2 (&cs)[32], uint8_t *so, int lane) {
    if constexpr (EPI == kEpiF32 || EPI == kEpiAcc32) {
        float *s = reinterpret_cast<float *>(so);
#pragma unroll
        for (int j = 0; j < kChunk; ++j) s[j * 32 + lane] = v[j];
    } else if constexpr (EPI == kEpiF16) {
        __half *s = reinterpret_cast<__half *>(so);
#pragma unroll
        for (int j = 0; j < kChunk; ++j) s[j * 32 + lane] = __float2half_rn(v[j]);
    } else if constexpr (EPI == kEpiSiluMul) {
        // rows interleaved (gate_j, up_j): the even lane of each pair owns act column lane / 2
        __half *s = reinterpret_cast<__half *>(so);
#pragma unroll
        for (int j = 0; j < kChunk; ++j) {
            const float up = __shfl_xor_sync(kFull, v[j], 1);
            const float gt = v[j];
            // silu(g) = g / (1 + e^-g): fast divide (MUFU.RCP; g -> -inf gives 0), no IEEE slow path
            const float a = __fdividef(gt, 1.0f + __expf(-gt)) * up;
            if (!(lane & 1)) s[j * 16 + (lane >> 1)] = __float2half_rn(a);
        }
    } else if constexpr (EPI == kEpiRopeKV) {
        // rotate-half pair i = (x[i], x[i + d/2]) of a q or k head sits in rows (2i, 2i + 1); the
        // chunk image holds each head in logical order
        const GemmEpiArgs &e = p.e;
        const int d = e.head_dim;
        const int hh = n / d, rr = n % d;
        __half *s = reinterpret_cast<__half *>(so);
        const int col0 = r - rr;  // the head's first row within the tile
        if (hh < e.q_heads + e.kv_heads) {
            const int i = rr >> 1, hd = d >> 1;
            const bool odd = rr & 1;
            const int col = col0 + (odd ? i + hd : i);
            const float sgn = odd ? 1.f : -1.f;
#pragma unroll
            for (int j = 0; j < kChunk; ++j) {
                const float other = __shfl_xor_sync(kFull, v[j], 1);
                s[j * kBM + col] = __float2half_rn(fmaf(sgn * other, cs[j].y, v[j] * cs[j].x));
            }
        } else {
#pragma unroll
            for (int j = 0; j < kChunk; ++j) s[j * kBM + r] = __float2half_rn(v[j]);
        }
    }
}

// Issue the global writes of a chunk image: RoPE -- epilogue warp 0, one bulk copy per (token,
// head), each lane commits its own bulk group; the others -- lane 0 of the owning warp, one TMA
// op for its 32 weight rows starting at nrow0.
template <int EPI>
__device__ __forceinline__ void epi_issue(const KParams &p, const OutMaps *ty, const uint8_t *so, int nrow0,
                                          int m, const int64_t *m_off, int cb, int lane) {
    if constexpr (EPI == kEpiRopeKV) {
        // lane j: token m + j; one contiguous d-element row per head of the tile
        const GemmEpiArgs &e = p.e;
        const int d = e.head_dim;
        if (m + lane < p.M) {
            for (int h0 = 0; h0 < kBM; h0 += d) {
                const int hh = (nrow0 + h0) / d;
                const uint8_t *src = so + (lane * kBM + h0) * 2;
                uint8_t *dst;
                if (hh < e.q_heads) {
                    dst = reinterpret_cast<uint8_t *>(e.q_out + (static_cast<int64_t>(m + lane) * e.q_heads + hh) * d);
                } else if (hh < e.q_heads + e.kv_heads) {
                    dst = e.kv_layer + m_off[cb + lane] + (hh - e.q_heads) * e.tile_bytes;
                } else {
                    dst = e.kv_layer + m_off[cb + lane] + (hh - e.q_heads - e.kv_heads) * e.tile_bytes +
                          static_cast<int64_t>(kP) * d * 2;
                }
                bulk_s2g(dst, src, d * 2);
            }
        }
        bulk_commit();
    } else if (lane == 0) {
        if constexpr (EPI == kEpiAcc32) {
            // tensor parallel: these 32 columns belong to one rank's slice of the residual stream;
            // the partial goes straight into that rank's memory (reduce-scatter fused into the GEMM)
            const int owner = p.e.tp_size > 1 ? nrow0 / p.e.tp_cols : 0;
            tma_reduce_add2d(&ty->m[owner], so, nrow0, m);
        } else if constexpr (EPI == kEpiSiluMul) {
            tma_store2d(&ty->m[0], so, nrow0 / 2, m);
        } else {
            tma_store2d(&ty->m[0], so, nrow0, m);
        }
        bulk_commit();
    }
}

// Weight tile (nt) and activation tile (mt) of work unit `unit` for pair `pair` of the cluster:
// with NP = 2 pairs per cluster a unit is a super-unit of NP adjacent weight tiles sharing one
// activation tile, pair j taking weight tile NP * (unit / m_tiles) + j.
template <int NP>
__device__ __forceinline__ void unit_tiles(const KParams &p, int unit, int pair, int &nt, int &mt) {
    nt = (unit / p.m_tiles) * NP + pair;
    mt = unit % p.m_tiles;
}
// weight tile, first activation row and activation tile width of a unit (re-tiled last wave:
// KParams::units_a)
template <int NP>
__device__ __forceinline__ void unit_geom(const KParams &p, int unit, int pair, int &nt, int &m0, int &bn) {
    if (NP == 1 && unit >= p.units_a) {
        const int u2 = unit - p.units_a;
        nt = p.n_a + u2 / p.m_tiles_b;
        m0 = (u2 % p.m_tiles_b) * p.BN_b;
        bn = p.BN_b;
        return;
    }
    int mt;
    unit_tiles<NP>(p, unit, pair, nt, mt);
    m0 = mt * p.BN;
    bn = p.BN;
}

// NP = CTA pairs per cluster.  NP = 2 (CG = 2 only): the two pairs of a 4-CTA cluster compute
// adjacent weight tiles against the same activation tile in lockstep, and each CTA loads HALF of
// its activation box and multicasts it to the same-rank CTA of the other pair -- the activation
// operand crosses L2 -> SM once per cluster instead of once per pair (the M = 512 GEMMs stream
// their operands at the chip's L2 throughput).  A stage is refilled only after BOTH
// pairs' MMAs have consumed it (the empty barrier counts the two leaders' commits).
template <int CG, int NP, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tx,
               const __grid_constant__ CUtensorMap txb, const __grid_constant__ OutMaps ty, const KParams p) {
    static_assert(NP == 1 || (NP == 2 && CG == 2), "multicast pairs need CTA pairs");
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages], tfull[2], tempty[2];
    __shared__ uint32_t tmem_base_sh;
    __shared__ int32_t m_pos[EPI == kEpiRopeKV ? kMaxBN : 1];
    __shared__ int64_t m_off[EPI == kEpiRopeKV ? kMaxBN : 1];

    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int BNc = p.BN / CG;  // activation rows this CTA loads per stage
    const uint32_t a_bytes = kBM * 128, stage_bytes = a_bytes + BNc * 128;
    uint8_t *outbuf = smem + p.stages * stage_bytes;  // kOutBufs chunk images
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = CG == 2 ? cluster_rank() : 0u;
    const uint32_t rank = crank & (CG - 1);          // rank within the pair (0 = the MMA leader)
    const uint32_t lead = crank - rank;              // the pair leader's rank in the cluster
    const int pair = static_cast<int>(crank >> 1) & (NP - 1);
    const int BNh = BNc / NP;                        // activation rows this CTA loads (and multicasts)
    const int g = static_cast<int>(blockIdx.x) / (CG * NP);
    const int64_t it0 = p.stream_k ? g * p.T / p.groups : 0;
    const int64_t it1 = p.stream_k ? (g + 1) * p.T / p.groups : 0;
    uint32_t tcols = 32;
    while (tcols < static_cast<uint32_t>(2 * p.BN)) tcols <<= 1;
    uint64_t *tr = p.trace ? p.trace + blockIdx.x * 8 : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = global_ns();

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NP);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], CG * 4);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        if constexpr (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                         "r"(tcols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                         "r"(tcols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        }
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    if (tr && threadIdx.x == 0) tr[1] = global_ns();

    if (warp == 0) {
        // ---------------- TMA producer
        const uint32_t full_lead = CG == 2 ? cluster_addr(&full[0], lead) : smem_u32(&full[0]);
        const uint16_t mc_mask = static_cast<uint16_t>((1u << rank) | (1u << (rank + 2)));
        // the first ring's weight boxes go out before the grid-dependency wait: weights never
        // depend on the previous kernel, the activations (and the outputs' readers) do
        int pre = 0;
        {
            int64_t it_p = it0;
            Seg s0;
            if (lane == 0 && p.dbg != 2 && next_seg(p, g, it_p, it1, s0)) {
                int nt0, mt0;
                unit_tiles<NP>(p, s0.unit, pair, nt0, mt0);
                const int wrow = nt0 * kBM * CG + static_cast<int>(rank) * kBM;
                pre = min(p.stages, s0.k1 - s0.k0);
                for (int s = 0; s < pre; ++s) {
                    if (rank == 0) mbar_expect_tx(&full[s], CG * stage_bytes);
                    tma_load2d<CG>(smem + s * stage_bytes, &tw, (s0.k0 + s) * kBK, wrow, full_lead + s * 8);
                }
            }
            pre = __shfl_sync(kFull, pre, 0);
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");
        int stage = 0, done = 0;
        uint32_t phase = 0;
        int64_t it = it0;
        Seg sg;
        while (next_seg(p, g, it, it1, sg)) {
            int nt, m0, bn;
            unit_geom<NP>(p, sg.unit, pair, nt, m0, bn);
            const int wrow = nt * kBM * CG + static_cast<int>(rank) * kBM;
            const int xrow = m0 + static_cast<int>(rank) * (bn / CG);
            const uint32_t unit_stage_tx = CG * (a_bytes + (bn / CG) * 128);
            const CUtensorMap *txu = bn == p.BN ? &tx : &txb;
            for (int kb = sg.k0; kb < sg.k1; ++kb, ++done) {
                if (lane == 0) {
                    uint8_t *sa = smem + stage * stage_bytes;
                    const uint32_t fb = full_lead + stage * 8;
                    if (p.dbg == 2) {  // measurement: the ring cycles without operand traffic
                        mbar_wait(&empty[stage], phase ^ 1);
                        if (rank == 0) mbar_arrive(&full[stage]);
                    } else {
                        if (done >= pre) {
                            mbar_wait(&empty[stage], phase ^ 1);
                            if (rank == 0) mbar_expect_tx(&full[stage], unit_stage_tx);
                            tma_load2d<CG>(sa, &tw, kb * kBK, wrow, fb);
                        }
                        if constexpr (NP == 2)
                            tma_load2d_mc(sa + a_bytes + pair * BNh * 128, &tx, kb * kBK, xrow + pair * BNh, fb,
                                          mc_mask);
                        else
                            tma_load2d<CG>(sa + a_bytes, txu, kb * kBK, xrow, fb);
                    }
                }
                __syncwarp();
                if (++stage == p.stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    } else if (warp == 1) {
        // ---------------- MMA issuer (the leader CTA of a pair issues for both)
        if (rank == 0) {
            const uint32_t idesc_a = idesc_f16(0, 0, kBM * CG, p.BN), idesc_b = idesc_f16(0, 0, kBM * CG, p.BN_b);
            const uint32_t base = smem_u32(smem);
            int stage = 0, acc = 0;
            uint32_t phase = 0, aph = 0;
            int64_t it = it0;
            Seg sg;
            bool first = true;
            while (next_seg(p, g, it, it1, sg)) {
                mbar_wait(&tempty[acc], aph ^ 1);
                tc_fence_after();
                const uint32_t td = tmem + acc * p.BN;
                const uint32_t idesc = (NP == 1 && sg.unit >= p.units_a) ? idesc_b : idesc_a;
                for (int kb = sg.k0; kb < sg.k1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (tr && first && lane == 0) tr[2] = global_ns();
                    first = false;
                    const uint32_t sa = base + stage * stage_bytes, sb = sa + a_bytes;
#pragma unroll
                    for (int kk = 0; kk < (p.dbg == 1 ? 0 : kBK / 16); ++kk) {
                        const uint64_t ad = smem_desc(sa + kk * 32, 16, 1024, 2);
                        const uint64_t bd = smem_desc(sb + kk * 32, 16, 1024, 2);
                        const uint32_t accum = (kb > sg.k0 || kk > 0) ? 1u : 0u;
                        if constexpr (CG == 2) umma_ss_pair(td, ad, bd, idesc, accum);
                        else umma_ss(td, ad, bd, idesc, accum);
                    }
                    if constexpr (CG == 2) umma_commit_pair(&empty[stage], NP == 2 ? 0xF : 3);
                    else umma_commit(&empty[stage]);
                    if (++stage == p.stages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if constexpr (CG == 2) umma_commit_pair(&tfull[acc], static_cast<uint16_t>(3u << lead));
                else umma_commit(&tfull[acc]);
                if (tr && lane == 0) tr[3] = global_ns();
                if (++acc == 2) {
                    acc = 0;
                    aph ^= 1;
                }
            }
        }
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    } else {
        // ---------------- epilogue: thread <-> TMEM lane (weight row) of its warp's quarter
        asm volatile("griddepcontrol.wait;" ::: "memory");
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const int et = threadIdx.x - 64;
        const bool issuer = et < 32;  // epilogue warp 0 writes the chunks out
        const uint32_t tempty_lead = CG == 2 ? cluster_addr(&tempty[0], lead) : smem_u32(&tempty[0]);
        int acc = 0, chunk = 0;
        uint32_t aph = 0;
        int64_t it = it0;
        Seg sg;
        while (next_seg(p, g, it, it1, sg)) {
            int nt, m0, bn;
            unit_geom<NP>(p, sg.unit, pair, nt, m0, bn);
            const int nrow0 = nt * kBM * CG + static_cast<int>(rank) * kBM;  // this CTA's first weight row
            if constexpr (EPI == kEpiRopeKV) {
                epi_bar();  // the previous unit is done with m_pos / m_off
                for (int i = et; i < bn; i += 128) {
                    const int m = m0 + i;
                    if (m < p.M) {
                        const TokRow tk = p.e.rows[m];
                        const int32_t page = p.e.bt[static_cast<int64_t>(tk.slot) * p.e.bt_stride + tk.pos / kP];
                        m_pos[i] = tk.pos;
                        m_off[i] = page * p.e.page_stride + static_cast<int64_t>(tk.pos % kP) * p.e.head_dim * 2;
                    } else {
                        m_pos[i] = 0;
                        m_off[i] = 0;
                    }
                }
                epi_bar();
            }
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
            if (tr && et == 0) tr[4] = global_ns();
            const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + acc * p.BN;
            const int cmax = min(bn, p.M - m0);  // activation rows of this tile (>= 1)
            const int ncol = nrow0 + row;           // this thread's output column (weight row)
            // the kind's epilogue of one chunk: v = the chunk's 32 accumulator values of this row
            auto emit = [&](int c0, const float (&v)[32]) {
                // RoPE: this chunk's (cos, sin) pairs
                float2 cs[kChunk];
                if constexpr (EPI == kEpiRopeKV) {
                    const int rr_ = ncol % p.e.head_dim;
                    const int hd = p.e.head_dim >> 1;
#pragma unroll
                    for (int j = 0; j < kChunk; ++j)
                        cs[j] = __ldg(p.e.cs + static_cast<int64_t>(m_pos[c0 + j]) * hd + (rr_ >> 1));
                }
                if constexpr (EPI == kEpiRopeKV) {
                    uint8_t *so = outbuf + (chunk % kOutBufs) * kStageOut;
                    // the writes issued from this buffer two chunks ago have finished reading it
                    if (issuer) bulk_wait_read_buf();
                    epi_bar();
                    epi_to_smem<EPI>(p, v, row, ncol, cs, so, lane);
                    fence_proxy_async();
                    epi_bar();
                    if (issuer) epi_issue<EPI>(p, &ty, so, nrow0, m0 + c0, m_off, c0, lane);
                } else {
                    // this warp's private pair of 4-KiB chunk images
                    uint8_t *so = outbuf + (q * kOutBufs + (chunk % kOutBufs)) * (kStageOut / 4);
                    if (lane == 0) bulk_wait_read_buf();
                    __syncwarp();
                    epi_to_smem<EPI>(p, v, row, ncol, cs, so, lane);
                    fence_proxy_async();
                    __syncwarp();
                    epi_issue<EPI>(p, &ty, so, nrow0 + q * 32, m0 + c0, m_off, c0, lane);
                }
                ++chunk;
            };
            const bool split = EPI != kEpiAcc32 && p.split > 1;
            for (int c0 = 0; c0 < cmax; c0 += kChunk) {
                uint32_t rr[32];
                tmem_ld32(ta + c0, rr);
                tmem_ld_wait();
                if (tr && et == 0 && c0 == 0) tr[5] = global_ns();
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[j]);
                if (c0 + kChunk >= cmax) {
                    // the tile's accumulator is in registers: release it to the next tile's MMAs
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(tempty_lead + acc * 8);
                }
                if (split) {
                    // this K range's partial: a private [32 m][32 n] fp32 image per warp, reduce-added
                    // into the workspace by the TMA unit (the sums happen in L2)
                    uint8_t *so = outbuf + (q * kOutBufs + (chunk % kOutBufs)) * (kStageOut / 4);
                    if (lane == 0) bulk_wait_read_buf();
                    __syncwarp();
                    float *sf = reinterpret_cast<float *>(so);
#pragma unroll
                    for (int j = 0; j < kChunk; ++j) sf[j * 32 + lane] = v[j];
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        tma_reduce_add2d(&ty.m[1], so, nrow0 + q * 32, m0 + c0);
                        bulk_commit();
                    }
                    ++chunk;
                } else {
                    emit(c0, v);
                }
            }
            if (split) {
                // every partial of this segment has been added into the workspace; once all S
                // segments of the tile have (arrival counter; they are co-resident: units x S <=
                // the resident CTA groups), segment j reads back the tile's chunks j, j + S, ...,
                // clears them and runs the epilogue on them; the last to leave resets the counters
                if (lane == 0) {
                    bulk_wait_all();
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                }
                __syncwarp();
                epi_bar();
                int32_t *cnt = p.cnt + 2 * (sg.unit * CG + static_cast<int>(rank));
                if (et == 0) {
                    __threadfence();
                    atomicAdd(cnt, 1);
                    int a;
                    while (true) {
                        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(a) : "l"(cnt) : "memory");
                        if (a >= p.split) break;
                        __nanosleep(64);
                    }
                }
                epi_bar();
                __threadfence();
                for (int c0 = sg.j * kChunk; c0 < cmax; c0 += p.split * kChunk) {
                    float v[32];
                    float *w = p.ws + static_cast<int64_t>(m0 + c0) * p.ldw + ncol;
#pragma unroll
                    for (int r = 0; r < kChunk; ++r) {
                        const bool in = m0 + c0 + r < p.M && ncol < p.N;
                        v[r] = in ? __ldcg(w + static_cast<int64_t>(r) * p.ldw) : 0.f;
                    }
#pragma unroll
                    for (int r = 0; r < kChunk; ++r)
                        if (m0 + c0 + r < p.M && ncol < p.N) __stcg(w + static_cast<int64_t>(r) * p.ldw, 0.f);
                    emit(c0, v);
                }
                epi_bar();
                if (et == 0 && atomicAdd(cnt + 1, 1) == p.split - 1) {  // every segment is past the wait
                    cnt[0] = 0;
                    cnt[1] = 0;
                }
            }
            if (++acc == 2) {
                acc = 0;
                aph ^= 1;
            }
        }
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        if (issuer || lane == 0) bulk_wait_all();
        if (tr && et == 0) tr[6] = global_ns();
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        if constexpr (CG == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols));
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols));
        if (tr && lane == 0) tr[7] = global_ns();
    }
}

using KernFn = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, OutMaps, KParams);

template <int CG, int NP = 1>
KernFn kernel_for(int epi) {
    switch (epi) {
        case kEpiF16: return gemm_tc_kernel<CG, NP, kEpiF16>;
        case kEpiF32: return gemm_tc_kernel<CG, NP, kEpiF32>;
        case kEpiAcc32: return gemm_tc_kernel<CG, NP, kEpiAcc32>;
        case kEpiRopeKV: return gemm_tc_kernel<CG, NP, kEpiRopeKV>;
        case kEpiSiluMul: return gemm_tc_kernel<CG, NP, kEpiSiluMul>;
        default: return nullptr;
    }
}

bool encode_2d(void *fn, CUtensorMap *map, CUtensorMapDataType dt, int esize, const void *base, uint64_t inner,
               uint64_t rows, uint64_t ld_elems, uint32_t box_inner, uint32_t box_rows, bool swizzle) {
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    const cuuint64_t gdim[2] = {inner, rows};
    const cuuint64_t gstride[1] = {ld_elems * esize};
    const cuuint32_t box[2] = {box_inner, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return encode(map, dt, 2, const_cast<void *>(base), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Activation tile width for whole-tile GEMMs: the multiple of 32 that minimises
// waves x per-k-block time, per-k-block time = max(MMA: 2 BN clk, operand traffic at ~50 B/clk
// per SM: (128 + BN/(CG NP)) x 128 B / 50) + a fixed ~40 clk (profiles/r02_gemm_trace.log); NP = 2:
// the activation box is multicast to two pairs, each SM fetches half of its share.
double per_kblock_clk(int bn, int cg, int np = 1) {
    return std::max(2.0 * bn, (128.0 + static_cast<double>(bn) / (cg * np)) * 128.0 / 50.0) + 40.0;
}

// returns the estimate (clocks per k-block x waves) of the chosen tiling
double choose_tiles(int M, int n_tiles, int groups, int cg, int *BN, int *m_tiles, int np = 1) {
    double best = 1e300;
    *m_tiles = (M + kMaxBN - 1) / kMaxBN;
    *BN = ((M + *m_tiles - 1) / *m_tiles + 31) / 32 * 32;
    for (int mt = *m_tiles; mt <= std::max(1, (M + 31) / 32); ++mt) {
        const int bn = ((M + mt - 1) / mt + 31) / 32 * 32;
        if ((M + bn - 1) / bn != mt) continue;
        const int64_t units = static_cast<int64_t>(n_tiles) * mt;
        const int64_t waves = (units + groups - 1) / groups;
        const double t = static_cast<double>(waves) * per_kblock_clk(bn, cg, np);
        if (t < best * 0.999) {
            best = t;
            *BN = bn;
            *m_tiles = mt;
        }
    }
    return best;
}

}  // namespace

// measurement: DBK_GEMM_NP = 1 / 2 forces the pairs per cluster (unset: the cost model decides)
static int np_env() {
    static const int v = [] {
        const char *e = std::getenv("DBK_GEMM_NP");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

// measurement: DBK_GEMM_HET=0 never re-tiles the last wave
static bool het_env_ok() {
    static const bool ok = [] {
        const char *e = std::getenv("DBK_GEMM_HET");
        return !(e && e[0] == '0');
    }();
    return ok;
}

static bool split_env_ok() {
    static const bool ok = [] {
        const char *e = std::getenv("DBK_GEMM_SPLIT");  // measurement: 0 = never split K
        return !(e && e[0] == '0');
    }();
    return ok;
}

GemmRunner::~GemmRunner() {
    if (ws_) cudaFree(ws_);
    if (cnt_) cudaFree(cnt_);
}

cudaError_t GemmRunner::init(int device, int cta_group) {
    if (cta_group != 1 && cta_group != 2) return cudaErrorInvalidValue;
    device_ = device;
    cg_ = cta_group;
    cudaError_t e = cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    cudaDriverEntryPointQueryResult q;
    if ((e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &encode_, cudaEnableDefault, &q)) != cudaSuccess)
        return e;
    if (!encode_ || q != cudaDriverEntryPointSuccess) return cudaErrorNotSupported;
    for (int epi = kEpiF16; epi <= kEpiSiluMul; ++epi) {
        KernFn k = cg_ == 2 ? kernel_for<2>(epi) : kernel_for<1>(epi);
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmem)) != cudaSuccess)
            return e;
    }
    if (cg_ == 1) {
        max_groups_ = sms_;
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * sms_);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = kDynSmem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int clusters = 0;
        if ((e = cudaOccupancyMaxActiveClusters(&clusters, kernel_for<2>(kEpiF16), &cfg)) != cudaSuccess) return e;
        max_groups_ = std::min(clusters, sms_ / 2);
        if (max_groups_ < 1) return cudaErrorNotSupported;
        // 4-CTA clusters (two pairs sharing the activation operand by multicast)
        for (int epi = kEpiF16; epi <= kEpiSiluMul; ++epi) {
            if ((e = cudaFuncSetAttribute(kernel_for<2, 2>(epi), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          kDynSmem)) != cudaSuccess)
                return e;
        }
        attr[0].val.clusterDim.x = 4;
        cfg.gridDim = dim3(4 * (sms_ / 4));
        int c4 = 0;
        if (cudaOccupancyMaxActiveClusters(&c4, kernel_for<2, 2>(kEpiF16), &cfg) != cudaSuccess) {
            (void)cudaGetLastError();
            c4 = 0;
        }
        max_clusters4_ = std::min(c4, sms_ / 4);
    }
    if (const char *v = std::getenv("DBK_GEMM_SMS")) {  // measurement: the GEMM on a subset of the SMs
        const int n = std::atoi(v) / cg_;
        if (n >= 1) max_groups_ = std::min(max_groups_, n);
        if (n >= 1) max_clusters4_ = std::min(max_clusters4_, n / 2);
    }
    return cudaSuccess;
}

cudaError_t GemmRunner::run(int M, int N, int K, const __half *X, int64_t ldx, const __half *W, const GemmEpiArgs &e,
                            cudaStream_t s, bool pdl) {
    if (M == 0) return cudaSuccess;
    if (M < 0 || K <= 0 || K % kBK || N <= 0 || ldx < K || ldx % 8 || (reinterpret_cast<uintptr_t>(X) & 15) ||
        (reinterpret_cast<uintptr_t>(W) & 15) || !encode_)
        return cudaErrorInvalidValue;
    // fused epilogues address whole weight tiles (rows past N would be zero-filled operands)
    if ((e.kind == kEpiRopeKV || e.kind == kEpiSiluMul) && N % (kBM * cg_)) return cudaErrorInvalidValue;
    if (e.kind == kEpiRopeKV && (e.head_dim <= 0 || kBM % e.head_dim)) return cudaErrorInvalidValue;
    KParams p{};
    p.M = M;
    p.N = N;
    p.K = K;
    p.kb = K / kBK;
    const int n_tiles = (N + kBM * cg_ - 1) / (kBM * cg_);  // a ragged last tile: TMA zero-fills
                                                            // its weight rows, clips its stores
    p.stream_k = e.kind == kEpiAcc32 ? 1 : 0;
    double whole_clk = 1e300;  // the cost model's whole-tile estimate (whole-tile kinds)
    if (p.stream_k) {
        p.m_tiles = (M + kMaxBN - 1) / kMaxBN;
        p.BN = ((M + p.m_tiles - 1) / p.m_tiles + 31) / 32 * 32;
    } else {
        whole_clk = choose_tiles(M, n_tiles, max_groups_, cg_, &p.BN, &p.m_tiles) * p.kb;
    }
    if (force_bn_ > 0) {  // measurement: a fixed activation tile width
        p.BN = std::min(kMaxBN, (force_bn_ + 31) / 32 * 32);
        p.m_tiles = (M + p.BN - 1) / p.BN;
    }
    p.split = 1;
    if (!p.stream_k && force_bn_ <= 0 && split_ok_ && split_env_ok()) {
        // split K when the whole tiles cannot keep the CTA groups busy (a 70B-TP8 QKV slice:
        // N = 1280 is 5 tiles for 74 pairs; the 7B / 13B down projections at small batches):
        // full-width tiles, K cut S ways, every K range's fp32 partial reduce-added into a
        // workspace by TMA, then the tile's S segments (co-resident: units x S <= groups) each
        // read back and finish a share of its 32-row chunks.  Taken when the cost model says
        // <= 0.9 x the best whole-tile tiling: S-way k-blocks at the widest tile plus the
        // reduction, fitted on the final build as ~4 us + 0.6 us per MB reduce-added
        // (profiles/r02_gemm_split.json: TP8 QKV 32 -> 14-21 us, 7B down at M <= 256 44 -> 26-32 us)
        const int mt0 = (M + kMaxBN - 1) / kMaxBN;
        const int bn0 = ((M + mt0 - 1) / mt0 + 31) / 32 * 32;
        const int units0 = n_tiles * mt0;
        const int S = std::min(max_groups_ / std::max(units0, 1), p.kb / 4);
        if (units0 * 2 <= max_groups_ && S >= 2) {
            const double clk_per_us = 1800.0;
            const double mb = static_cast<double>(units0) * S * (kBM * cg_) * bn0 * 4.0 / 1e6;
            const double split_clk = per_kblock_clk(bn0, cg_) * ((p.kb + S - 1) / S) + (4.0 + 0.6 * mb) * clk_per_us;
            if (split_clk < 0.9 * whole_clk) {
                p.m_tiles = mt0;
                p.BN = bn0;
                p.split = S;
            }
        }
    }
    // Two pairs per cluster sharing the activation operand by multicast (an even number of weight
    // tiles, no K split): measured and NOT taken by default -- 0.97-1.27 x the time of one pair per
    // cluster on the 7B / 13B / 70B-TP8 shapes (profiles/r02_gemm_multicast.json): the M = 512
    // GEMMs are bound by the SM's shared-memory port (every operand byte is written by TMA and read
    // by the MMA), which multicast does not relieve.  DBK_GEMM_NP=2 forces it (measurement).
    int np = 1;
    if (cg_ == 2 && max_clusters4_ >= 1 && p.split == 1 && n_tiles % 2 == 0 && np_env() == 2) {
        np = 2;
        if (!p.stream_k && force_bn_ <= 0) {
            int bn2 = p.BN, mt2 = p.m_tiles;
            choose_tiles(M, n_tiles / 2, max_clusters4_, cg_, &bn2, &mt2, 2);
            p.BN = bn2;
            p.m_tiles = mt2;
        }
    }
    p.units = (n_tiles / np) * p.m_tiles;
    p.units_a = p.units;
    p.n_a = n_tiles;
    p.BN_b = p.BN;
    p.m_tiles_b = p.m_tiles;
    if (!p.stream_k && p.split == 1 && np == 1 && force_bn_ <= 0 && het_env_ok() && p.BN >= 128) {
        // Re-tile a mostly idle last wave (gate/up at M = 512: 172 units of BN = 256 on 74 CTA
        // pairs, the third wave on 24 of them): the full waves keep BN, the weight tiles left over
        // run at half the activation width -- twice the units, each at ~0.75 of the time per
        // k-block -- when the cost model says >= 5 % sooner (DBK_GEMM_HET=0: never)
        const int G = max_groups_;
        const int64_t waves = (static_cast<int64_t>(p.units) + G - 1) / G;
        const int64_t rem = p.units - (waves - 1) * G;
        const int n_a = static_cast<int>(((waves - 1) * G) / p.m_tiles);
        if (waves >= 2 && rem * 2 < G && n_a * p.m_tiles >= G && n_a < n_tiles) {
            const int mt_b = 2 * p.m_tiles;
            const int bn_b = ((M + mt_b - 1) / mt_b + 31) / 32 * 32;
            const int64_t units_b = static_cast<int64_t>(n_tiles - n_a) * ((M + bn_b - 1) / bn_b);
            const int64_t units_a = static_cast<int64_t>(n_a) * p.m_tiles;
            const double t_whole = static_cast<double>(waves) * per_kblock_clk(p.BN, cg_);
            const double t_het = static_cast<double>((units_a + G - 1) / G) * per_kblock_clk(p.BN, cg_) +
                                 static_cast<double>((units_b + G - 1) / G) * per_kblock_clk(bn_b, cg_);
            if (bn_b < p.BN && t_het < 0.95 * t_whole) {
                p.units_a = static_cast<int32_t>(units_a);
                p.n_a = n_a;
                p.BN_b = bn_b;
                p.m_tiles_b = (M + bn_b - 1) / bn_b;
                p.units = static_cast<int32_t>(units_a + units_b);
            }
        }
    }
    p.T = static_cast<int64_t>(p.units) * p.kb;
    const int maxg = np == 2 ? max_clusters4_ : max_groups_;
    if (p.stream_k) {
        // >= 4 k-blocks per group: a partial tile's reduce-add (BN x 128 x 4 B) stays small next to
        // the operand traffic of its k-blocks
        p.groups = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(maxg, p.T / 4)));
    } else {
        p.groups = std::min<int64_t>(maxg, static_cast<int64_t>(p.units) * p.split);
    }
    p.ldw = N;
    p.ws = nullptr;
    p.cnt = nullptr;
    if (p.split > 1) {
        const size_t need = static_cast<size_t>(M) * N;  // fp32 [M][N], zero between launches
        const int ncnt = 2 * p.units * cg_;                         // arrivals, departures per (tile, CTA)
        if (need > ws_elems_ || ncnt > cnt_cap_) {  // first use of a shape: grows once (synchronous)
            if (ws_) cudaFree(ws_);
            if (cnt_) cudaFree(cnt_);
            ws_ = nullptr;
            cnt_ = nullptr;
            ws_elems_ = std::max(need, ws_elems_);
            cnt_cap_ = std::max(ncnt, cnt_cap_);
            cudaError_t err;
            if ((err = cudaMalloc(&ws_, ws_elems_ * sizeof(float))) != cudaSuccess) return err;
            if ((err = cudaMalloc(&cnt_, static_cast<size_t>(cnt_cap_) * sizeof(int32_t))) != cudaSuccess) return err;
            if ((err = cudaMemset(ws_, 0, ws_elems_ * sizeof(float))) != cudaSuccess) return err;
            if ((err = cudaMemset(cnt_, 0, static_cast<size_t>(cnt_cap_) * sizeof(int32_t))) != cudaSuccess) return err;
        }
        p.ws = ws_;
        p.cnt = cnt_;
    }
    const int stage_bytes = kBM * 128 + (p.BN / cg_) * 128;
    p.stages = std::min(kMaxStages, kRingBudget / stage_bytes);
    p.trace = trace_;
    p.dbg = dbg_;
    p.e = e;
    CUtensorMap tw, tx;
    OutMaps ty;
    CUtensorMap txb;
    if (!encode_2d(encode_, &tw, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, W, K, N, K, kBK, kBM, true) ||
        !encode_2d(encode_, &tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, X, K, M, ldx, kBK, p.BN / (cg_ * np), true) ||
        !encode_2d(encode_, &txb, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, X, K, M, ldx, kBK, p.BN_b / (cg_ * np), true))
        return cudaErrorInvalidValue;
    bool ok = true;
    switch (e.kind) {
        case kEpiF16:  // per-warp boxes: 32 weight rows x 32 activation rows
            ok = encode_2d(encode_, &ty.m[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, e.y, N, M, e.ldy, 32, kChunk, false);
            break;
        case kEpiF32:
            ok = encode_2d(encode_, &ty.m[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, e.y, N, M, e.ldy, 32, kChunk, false);
            break;
        case kEpiAcc32:
            if (e.tp_size > 1) {
                // every rank's residual stream (peer memory); each GEMM column goes to its owner
                if (e.tp_size > kMaxTp || !e.tp_y || e.tp_cols * e.tp_size != N || e.tp_cols % 32) return cudaErrorInvalidValue;
                for (int r = 0; r < e.tp_size && ok; ++r)
                    ok = encode_2d(encode_, &ty.m[r], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, e.tp_y[r], N, M, e.ldy, 32,
                                   kChunk, false);
            } else {
                ok = encode_2d(encode_, &ty.m[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, e.y, N, M, e.ldy, 32, kChunk,
                               false);
            }
            break;
        case kEpiSiluMul:
            ok = encode_2d(encode_, &ty.m[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, e.y, N / 2, M, e.ldy, 16, kChunk,
                           false);
            break;
        default:
            ty.m[0] = tw;  // unused by the RoPE / KV epilogue (per-row bulk copies)
    }
    if (ok && p.split > 1)  // the split-K workspace [M][N] fp32, per-warp 32 x 32 reduce-add boxes
        ok = encode_2d(encode_, &ty.m[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, p.ws, N, M, N, 32, kChunk, false);
    if (!ok) return cudaErrorInvalidValue;
    KernFn k = cg_ == 2 ? (np == 2 ? kernel_for<2, 2>(e.kind) : kernel_for<2>(e.kind)) : kernel_for<1>(e.kind);
    if (!k) return cudaErrorInvalidValue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.groups * cg_ * np);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = static_cast<size_t>(p.stages) * stage_bytes + kOutBufs * kStageOut + 1024;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cg_ * np;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    ++launches_;
    last_np_ = np;
    last_het_ = p.units_a < p.units;
    plan_[0] = p.BN;
    plan_[1] = p.BN_b;
    plan_[2] = p.units_a;
    plan_[3] = p.units;
    plan_[4] = p.split;
    return cudaLaunchKernelEx(&cfg, k, tw, tx, txb, ty, p);
}

}  // namespace dbk

// ------------------------------------------------------------------ C-ABI
using namespace dbk;

struct dbk_gemm {
    GemmRunner run;
};

extern "C" {

dbk_status dbk_gemm_create(int32_t device, int32_t cta_group, dbk_gemm **out) {
    if (!out) return fail(DBK_EINVAL, "gemm_create: null out");
    if (cta_group != 1 && cta_group != 2) return fail(DBK_EINVAL, "gemm_create: cta_group must be 1 or 2");
    DBK_CUDA(cudaSetDevice(device));
    dbk_gemm *g = new (std::nothrow) dbk_gemm();
    if (!g) return fail(DBK_EINVAL, "out of host memory");
    const cudaError_t e = g->run.init(device, cta_group);
    if (e != cudaSuccess) {
        delete g;
        return fail(DBK_ECUDA, "gemm_create: %s", cudaGetErrorString(e));
    }
    *out = g;
    return DBK_OK;
}

dbk_status dbk_gemm_run(dbk_gemm *g, int32_t M, int32_t N, int32_t K, const void *x, int64_t ldx, const void *w,
                        void *y, int64_t ldy, int32_t mode, void *stream) {
    if (!g || (M > 0 && (!x || !w || !y))) return fail(DBK_EINVAL, "gemm_run: null argument");
    if (mode != kEpiF16 && mode != kEpiF32 && mode != kEpiAcc32 && mode != kEpiSiluMul)
        return fail(DBK_EINVAL, "gemm_run: mode must be 0 (fp16), 1 (fp32), 2 (fp32 +=) or 4 (silu * up)");
    const int esz = (mode == kEpiF16 || mode == kEpiSiluMul) ? 2 : 4;
    const int64_t ncols = mode == kEpiSiluMul ? N / 2 : N;
    if (ldy < ncols || (ldy * esz) % 16 || (reinterpret_cast<uintptr_t>(y) & 15))
        return fail(DBK_EINVAL, "gemm_run: need ldy >= N (N/2 for mode 4) and 16-B aligned rows of y");
    if (mode == kEpiSiluMul && N % (kBM * g->run.cta_group()))
        return fail(DBK_EINVAL, "gemm_run: mode 4 needs N %% %d == 0", kBM * g->run.cta_group());
    if (M < 0 || K <= 0 || K % kBK || N <= 0 || ldx < K || ldx % 8)
        return fail(DBK_EINVAL, "gemm_run: need K %% 64 == 0, N >= 1, ldx >= K, ldx %% 8 == 0");
    GemmEpiArgs e;
    e.kind = mode;
    e.y = y;
    e.ldy = ldy;
    const cudaError_t st = g->run.run(M, N, K, static_cast<const __half *>(x), ldx, static_cast<const __half *>(w), e,
                                      static_cast<cudaStream_t>(stream), false);
    if (st != cudaSuccess) return fail(DBK_ECUDA, "gemm_run: %s", cudaGetErrorString(st));
    return DBK_OK;
}

dbk_status dbk_gemm_trace(dbk_gemm *g, void *trace, int32_t mode) {
    if (!g) return fail(DBK_EINVAL, "gemm_trace: null handle");
    if (mode < 0 || mode > 2) return fail(DBK_EINVAL, "gemm_trace: mode 0, 1 or 2");
    g->run.set_trace(static_cast<uint64_t *>(trace));
    g->run.set_debug(mode);
    return DBK_OK;
}

dbk_status dbk_gemm_force_tile(dbk_gemm *g, int32_t bn) {
    if (!g || bn < 0 || bn > 256) return fail(DBK_EINVAL, "gemm_force_tile: bn in 0 (automatic) .. 256");
    g->run.force_bn(bn);
    return DBK_OK;
}

dbk_status dbk_gemm_last_plan(dbk_gemm *g, int32_t *bn, int32_t *bn_b, int32_t *units_a, int32_t *units,
                              int32_t *split) {
    if (!g) return fail(DBK_EINVAL, "gemm_last_plan: null handle");
    int32_t v[5];
    g->run.last_plan(v);
    if (bn) *bn = v[0];
    if (bn_b) *bn_b = v[1];
    if (units_a) *units_a = v[2];
    if (units) *units = v[3];
    if (split) *split = v[4];
    return DBK_OK;
}

dbk_status dbk_gemm_destroy(dbk_gemm *g) {
    delete g;
    return DBK_OK;
}

}  // extern "C"
