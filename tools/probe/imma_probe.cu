// Probe: cuBLASLt int8 x int8 -> int32 GEMM ("TN", column-major) on sm_100a at the
// a0 shapes (m = Dp outputs per row, n = queries, k = (l-1) Dp), exactness and speed.
#include <cublasLt.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#define CK(x) do { auto e = (x); if (e != 0) { printf("err %d at %s:%d\n", (int)e, __FILE__, __LINE__); exit(1); } } while (0)
int main(int argc, char **argv) {
    int m = 960, n = 10000, kmax = 7 * 960;
    cublasLtHandle_t h; CK(cublasLtCreate(&h));
    std::vector<int8_t> A((size_t)kmax * m), B((size_t)kmax * n);
    srand(1);
    for (auto &v : A) v = (int8_t)(rand() % 129 - 64);
    for (auto &v : B) v = (int8_t)(rand() % 129 - 64);
    int8_t *dA, *dB; int32_t *dC; void *ws; size_t wsb = 64 << 20;
    CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dC, (size_t)m * n * 4)); CK(cudaMalloc(&ws, wsb));
    CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice)); CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int l = 2; l <= 8; l++) {
        int k = (l - 1) * 960, lda = kmax, ldb = kmax;
        cublasLtMatmulDesc_t op; CK(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32I, CUDA_R_32I));
        cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
        CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)));
        CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)));
        cublasLtMatrixLayout_t la, lb, lc;
        CK(cublasLtMatrixLayoutCreate(&la, CUDA_R_8I, k, m, lda));
        CK(cublasLtMatrixLayoutCreate(&lb, CUDA_R_8I, k, n, ldb));
        CK(cublasLtMatrixLayoutCreate(&lc, CUDA_R_32I, m, n, m));
        cublasLtMatmulPreference_t pref; CK(cublasLtMatmulPreferenceCreate(&pref));
        CK(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof(wsb)));
        cublasLtMatmulHeuristicResult_t res[4]; int nres = 0;
        CK(cublasLtMatmulAlgoGetHeuristic(h, op, la, lb, lc, lc, pref, 4, res, &nres));
        if (nres == 0) { printf("l=%d no algo\n", l); return 1; }
        int32_t alpha = 1, beta = 0;
        const int8_t *Ap = dA + (size_t)(8 - l) * 960;  // suffix of the concatenated row
        for (int it = 0; it < 3; it++)
            CK(cublasLtMatmul(h, op, &alpha, Ap, la, dB, lb, &beta, dC, lc, dC, lc, &res[0].algo, ws, wsb, 0));
        cudaEventRecord(e0);
        int R = 10;
        for (int it = 0; it < R; it++)
            CK(cublasLtMatmul(h, op, &alpha, Ap, la, dB, lb, &beta, dC, lc, dC, lc, &res[0].algo, ws, wsb, 0));
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= R;
        std::vector<int32_t> C((size_t)m * n);
        CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
        int bad = 0;
        for (int t = 0; t < 200; t++) {
            int i = rand() % m, j = rand() % n;
            long long s = 0;
            for (int kk = 0; kk < k; kk++) s += (long long)A[(size_t)i * lda + (8 - l) * 960 + kk] * B[(size_t)j * ldb + kk];
            if (s != C[(size_t)j * m + i]) bad++;
        }
        printf("l=%d k=%d ms=%.4f TOPS=%.1f bad=%d algos=%d\n", l, k, ms, 2.0 * m * n * k / ms / 1e9, bad, nres);
    }
    return 0;
}
