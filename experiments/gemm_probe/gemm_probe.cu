// Probe: how far is cuBLASLt's top heuristic from the best of its top-8 candidates on the
// model step's GEMM shapes (Y[M][N] = X[M][K] W[N][K]^T, fp16 in, fp32 accumulate)?
#include <cublasLt.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <vector>
int main() {
    cublasLtHandle_t lt; cublasLtCreate(&lt);
    size_t ws_bytes = 32u << 20; void *ws; cudaMalloc(&ws, ws_bytes);
    struct S { int M, N, K; bool f32; } shapes[] = {
        {512, 12288, 4096, false}, {512, 4096, 4096, true}, {512, 22016, 4096, false}, {512, 4096, 11008, true},
        {512, 32000, 4096, true}, {256, 12288, 4096, false}, {256, 4096, 4096, true}, {256, 22016, 4096, false},
        {256, 4096, 11008, true}, {128, 4096, 11008, true}, {300, 15360, 5120, false}, {300, 5120, 13824, true}};
    void *X, *W, *Y; cudaMalloc(&X, 512ull * 11008 * 2); cudaMalloc(&W, 32000ull * 11008 * 2); cudaMalloc(&Y, 512ull * 32000 * 4);
    cudaMemset(X, 0, 512ull * 11008 * 2); cudaMemset(W, 0, 32000ull * 11008 * 2);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (auto &sh : shapes) {
        cublasLtMatmulDesc_t op; cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F);
        cublasOperation_t tA = CUBLAS_OP_T, tB = CUBLAS_OP_N;
        cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &tA, sizeof tA);
        cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tB, sizeof tB);
        cublasLtMatrixLayout_t a, b, c;
        cublasLtMatrixLayoutCreate(&a, CUDA_R_16F, sh.K, sh.N, sh.K);
        cublasLtMatrixLayoutCreate(&b, CUDA_R_16F, sh.K, sh.M, sh.K);
        cublasLtMatrixLayoutCreate(&c, sh.f32 ? CUDA_R_32F : CUDA_R_16F, sh.N, sh.M, sh.N);
        cublasLtMatmulPreference_t pref; cublasLtMatmulPreferenceCreate(&pref);
        cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws_bytes, sizeof ws_bytes);
        cublasLtMatmulHeuristicResult_t res[8]; int found = 0;
        cublasLtMatmulAlgoGetHeuristic(lt, op, a, b, c, c, pref, 8, res, &found);
        const float alpha = 1.f, beta = sh.f32 ? 1.f : 0.f;
        std::vector<float> t(found);
        for (int i = 0; i < found; ++i) {
            for (int w = 0; w < 3; ++w) cublasLtMatmul(lt, op, &alpha, W, a, X, b, &beta, Y, c, Y, c, &res[i].algo, ws, ws_bytes, 0);
            cudaEventRecord(e0);
            for (int r = 0; r < 20; ++r) cublasLtMatmul(lt, op, &alpha, W, a, X, b, &beta, Y, c, Y, c, &res[i].algo, ws, ws_bytes, 0);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); t[i] = ms / 20 * 1e3f;
        }
        int best = 0; for (int i = 1; i < found; ++i) if (t[i] < t[best]) best = i;
        double fl = 2.0 * sh.M * sh.N * sh.K;
        printf("M %d N %d K %d f32 %d: %d candidates, top-1 %.1f us (%.0f TF), best #%d %.1f us (%.0f TF), gain %.1f%%\n",
               sh.M, sh.N, sh.K, sh.f32, found, t[0], fl / t[0] / 1e6, best, t[best], fl / t[best] / 1e6,
               (t[0] / t[best] - 1) * 100);
    }
    return 0;
}
