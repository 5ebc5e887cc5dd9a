// Model GEMMs on the 5th-generation tensor cores (gemm_tc.cu): Y[M][N] = X[M][K] W[N][K]^T with
// the decode step's elementwise work fused into the epilogue.  Internal to libdbk.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace dbk {

// One activation row of a model step: a decode token (pos = ctx - 1) or a prefill-chunk token.
struct TokRow {
    int64_t req_id;
    int32_t slot;  // block-table row
    int32_t pos;   // token position
};
static_assert(sizeof(TokRow) == 16, "TokRow layout");

enum GemmEpi : int32_t {
    kEpiF16 = 0,    // Y (fp16) = acc
    kEpiF32 = 1,    // Y (fp32) = acc
    kEpiAcc32 = 2,  // Y (fp32) += acc            (residual stream: O and down projections; split-K
                    //  partial tiles are added by TMA reduce-add, so the order of the adds varies)
    kEpiRopeKV = 3, // QKV projection: RoPE on q and k, q -> q_out, k and v -> the token's page slot
    kEpiSiluMul = 4 // gate|up projection (rows interleaved gate_j, up_j): act[m][j] = silu(gate) * up
};

// Epilogue operands (fields a given epilogue does not use are ignored).
struct GemmEpiArgs {
    int32_t kind = kEpiF16;
    void *y = nullptr;        // kinds 0-2: Y; kind 4: act [M][ldy] fp16
    int64_t ldy = 0;          // row stride of Y / act (elements)
    // kind 3 (RoPE + KV write), rows of the weight are permuted so that a RoPE pair (j, j + d/2) of
    // a q or k head sits in adjacent rows (2j, 2j + 1); v rows are in natural order
    const TokRow *rows = nullptr;  // [M]
    const int32_t *bt = nullptr;   // device block table
    int32_t bt_stride = 0;
    uint8_t *kv_layer = nullptr;   // this layer's slice of the pool
    int64_t page_stride = 0, tile_bytes = 0;
    const float2 *cs = nullptr;    // (cos, sin)[pos][d/2]
    int32_t q_heads = 0, kv_heads = 0, head_dim = 0;
    __half *q_out = nullptr;       // [M][q_heads][head_dim]
    // kind 2 under tensor parallelism: the output's columns are split over tp_size ranks in slices
    // of tp_cols; the partial product of slice r is reduce-added into tp_y[r] (rank r's residual
    // stream, peer memory), so the GEMM performs the all-reduce's reduce-scatter
    int32_t tp_size = 1, tp_cols = 0;
    void *const *tp_y = nullptr;   // host array [tp_size] of device pointers, same layout as y
};

// Persistent tcgen05 GEMM (stream-K for the accumulating epilogue, whole tiles otherwise).
class GemmRunner {
public:
    // cta_group 1 (one SM per 128 weight rows) or 2 (CTA pairs, 256 rows).
    cudaError_t init(int device, int cta_group);
    // X: fp16 [M][ldx] (ldx >= K, K % 64 == 0), W: fp16 [N][K] row-major, N % (128 * cta_group) == 0.
    // pdl: programmatic dependent launch after the previous kernel on the stream.
    cudaError_t run(int M, int N, int K, const __half *X, int64_t ldx, const __half *W, const GemmEpiArgs &e,
                    cudaStream_t s, bool pdl);
    int cta_group() const { return cg_; }
    // debug: per-CTA %globaltimer phase stamps [CTA][8] of the following launches (nullptr = off)
    void set_trace(uint64_t *t) { trace_ = t; }
    // measurement only: 1 = skip the MMAs, 2 = skip the operand loads (results are garbage)
    void set_debug(int mode) { dbg_ = mode; }
    // measurement: activation tile width (0 = the cost model's choice)
    void force_bn(int bn) { force_bn_ = bn; }
    int64_t launches() const { return launches_; }
    int last_pairs_per_cluster() const { return last_np_; }  // 2: the last launch multicast its activations
    // the last launch's tiling: BN, BN_b, units_a, units, split (dbk_gemm_last_plan)
    void last_plan(int32_t *out5) const {
        for (int i = 0; i < 5; ++i) out5[i] = plan_[i];
    }
    // measurement: 0 = never split K for the whole-tile epilogues (DBK_GEMM_SPLIT=0 does the same)
    void allow_split(bool on) { split_ok_ = on; }
    GemmRunner() = default;
    GemmRunner(const GemmRunner &) = delete;  // owns the split-K workspace
    GemmRunner &operator=(const GemmRunner &) = delete;
    ~GemmRunner();

private:
    int device_ = 0, cg_ = 1, sms_ = 0, max_groups_ = 0;
    int max_clusters4_ = 0, last_np_ = 1;  // co-resident 4-CTA clusters (two pairs; 0 = not available)
    bool last_het_ = false;                // the last launch re-tiled its last wave (KParams::units_a)
    int32_t plan_[5] = {0, 0, 0, 0, 0};    // last launch: BN, BN_b, units_a, units, split
    uint64_t *trace_ = nullptr;
    int dbg_ = 0, force_bn_ = 0;
    bool split_ok_ = true;
    int64_t launches_ = 0;
    void *encode_ = nullptr;  // cuTensorMapEncodeTiled
    // split-K of the whole-tile epilogues: fp32 partial sums [M][N] reduce-added here (zero between
    // launches: the last segment of a tile reads its tile back and clears it) and one arrival
    // counter per (tile, CTA of the pair)
    float *ws_ = nullptr;
    size_t ws_elems_ = 0;
    int32_t *cnt_ = nullptr;
    int cnt_cap_ = 0;
};

// Rows of a weight matrix as stored for the fused epilogues: physical row -> logical row.
// QKV (kEpiRopeKV): within each q / k head, physical 2i -> i, 2i + 1 -> i + d/2; v rows unchanged.
__host__ __device__ inline int64_t qkv_logical_row(int64_t phys, int q_heads, int kv_heads, int d) {
    const int64_t h = phys / d, r = phys % d;
    if (h >= q_heads + kv_heads) return phys;
    return h * d + ((r & 1) ? (r >> 1) + d / 2 : (r >> 1));
}
// gate|up (kEpiSiluMul): physical 2j -> gate row j, 2j + 1 -> up row F + j.
__host__ __device__ inline int64_t gu_logical_row(int64_t phys, int64_t F) {
    return (phys & 1) ? F + (phys >> 1) : (phys >> 1);
}

}  // namespace dbk
