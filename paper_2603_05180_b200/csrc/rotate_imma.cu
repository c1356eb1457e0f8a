// rotate_imma.cu -- a0 (q' = fl32(q R)) on the int8 tensor cores,
// exact by certification.
//
// The oracle's q'_n is fl32(y_n), y_n the sequential fp64 chain
// s = fma(q_k, R_kn, s), k ascending from +0.  Here:
//  1. Each query row is scaled by 2^-e (|u_k| = |q_k| 2^-e < 1/4), rounded to
//     the fixed point U_k = rint(u_k 2^56) (|u_k - U_k 2^-56| <= 2^-57) and U_k
//     is written in S = 8 balanced base-128 digits, U_k 2^-56 = sum_s a_ks 2^-7s
//     (|a| <= 64, integer arithmetic); each column n of R likewise with 2^-f_n,
//     digits b_knt.
//  2. For every level l = 2..9 one int8 x int8 -> int32 GEMM (cuBLASLt, the
//     tensor cores) computes C_l[m][n] = sum_{s+t=l} sum_k a_mks b_knt exactly:
//     the slices of a level are concatenated along k (K' = (l-1) Dp).
//  3. yhat = 2^(e+f_n) sum_l 2^-7l C_l (fp64, ascending l) differs from the
//     exact sum S of the products by at most 2^(e+f_n) (Dp 2^-53 + 2^-50
//     sum_l |2^-7l C_l|): the dropped digit pairs s+t > 9 and the fixed-point
//     roundings (< 2^-54 per term), the 8-term fp64 sum.  The oracle's y_n
//     differs from S by at most gamma_Dp ||q|| ||R_n|| (recursive summation,
//     exact products).  If [yhat - b, yhat + b] lies strictly inside the fp32
//     rounding cell of fl32(yhat), then fl32(y_n) = fl32(yhat): certified.
//     Otherwise (~0.02% of outputs at cfg2) k_recompute runs the sequential
//     chain for that output.
// The R slices, exponents and column norms are computed once per index.
#include <cublasLt.h>

#include <cmath>
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>

#include "crisp_internal.cuh"

namespace crisp {

namespace {

constexpr int SL = 8;  // slices per operand
constexpr int LV = 9;  // levels 2..LV (slice pairs s + t <= LV)

std::mutex g_mu;
cublasLtHandle_t g_lt = nullptr;
std::map<int, void *> g_ws;  // cuBLASLt workspace per device
constexpr size_t WS_BYTES = 32u << 20;

#define CRISP_LT(call)                                                                  \
    do {                                                                                \
        cublasStatus_t st_ = (call);                                                    \
        if (st_ != CUBLAS_STATUS_SUCCESS) {                                             \
            ::crisp::set_error(std::string(#call) + ": cublasLt status " + std::to_string((int)st_)); \
            throw ::crisp::Err{CRISP_ECUDA};                                            \
        }                                                                               \
    } while (0)

// 2^e as a double (normal range), exact
__device__ __forceinline__ double pow2(int e) {
    return (e >= -1022 && e <= 1023) ? __longlong_as_double((long long)(1023 + e) << 52) : ldexp(1.0, e);
}

// one row (warp): exponent, 2-norm, digits a_1..a_8 of u = x 2^-e into out[(s-1) Dpk + k]
__device__ __forceinline__ void slice_vec(const float *__restrict__ x, int64_t xstride, int Dp, int Dpk,
                                          int8_t *__restrict__ out, int32_t *e_out, double *n2_out, int lane) {
    float mx = 0.f;
    double ss = 0.0;
    for (int k = lane; k < Dp; k += 32) {
        const float v = x[(int64_t)k * xstride];
        mx = fmaxf(mx, fabsf(v));
        ss = fma((double)v, (double)v, ss);
    }
    for (int off = 16; off; off >>= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        ss += __shfl_xor_sync(0xffffffffu, ss, off);
    }
    const int e = mx > 0.f ? ilogbf(mx) + 3 : 0;  // |x| 2^-e < 1/4: the top digit stays in [-64, 63]
    if (lane == 0) {
        *e_out = e;
        *n2_out = sqrt(ss) * 1.01;
    }
    const double sc = pow2(56 - e);  // exact scaling
    for (int k4 = lane * 4; k4 < Dpk; k4 += 128) {
        // U = rint(x 2^(56-e)), |U| < 2^54; balanced base-128 digits, least significant
        // first; 4 consecutive k per lane, one 4-byte store per digit
        long long U[4];
#pragma unroll
        for (int j = 0; j < 4; j++)
            U[j] = k4 + j < Dp ? __double2ll_rn((double)x[(int64_t)(k4 + j) * xstride] * sc) : 0;
#pragma unroll
        for (int s = SL; s >= 1; s--) {
            uint32_t packed = 0;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const long long d = ((U[j] + 64) & 127) - 64;  // in [-64, 63]
                U[j] = (U[j] - d) >> 7;                         // exact
                packed |= ((uint32_t)d & 0xffu) << (8 * j);
            }
            *(uint32_t *)(out + (int64_t)(s - 1) * Dpk + k4) = packed;
        }
    }
}

// queries: Qcat[m][(s-1) Dpk + k] = a_s (ascending slices)
__global__ void k_slice_rows(const float *__restrict__ X, int64_t rows, int Dp, int64_t ldx, int Dpk,
                             int8_t *__restrict__ Qcat, int32_t *__restrict__ qe, double *__restrict__ qn2) {
    const int64_t m = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (m >= rows) return;
    slice_vec(X + m * ldx, 1, Dp, Dpk, Qcat + m * (int64_t)SL * Dpk, qe + m, qn2 + m, threadIdx.x & 31);
}

// R columns: Rrev[n][(SL-t) Dpk + k] = b_t (descending slices), so that the
// level-l operand [b_{l-1} .. b_1] is the row suffix from (LV-l) Dpk
__global__ void k_slice_cols(const float *__restrict__ R, int Dp, int Dpk, int8_t *__restrict__ tmp,
                             int8_t *__restrict__ Rrev, int32_t *__restrict__ re, double *__restrict__ rn2) {
    const int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (n >= Dp) return;
    const int lane = threadIdx.x & 31;
    int8_t *t = tmp + (int64_t)n * SL * Dpk;
    slice_vec(R + n, Dp, Dp, Dpk, t, re + n, rn2 + n, lane);
    __syncwarp();
    for (int i = lane; i < SL * Dpk; i += 32) {
        const int s = i / Dpk + 1, k = i % Dpk;
        Rrev[(int64_t)n * SL * Dpk + (int64_t)(SL - s) * Dpk + k] = t[i];
    }
}

__global__ void k_certify(const int32_t *__restrict__ C, int64_t rows, int Dp, int Dpk, const int32_t *__restrict__ qe,
                          const double *__restrict__ qn2, const int32_t *__restrict__ re,
                          const double *__restrict__ rn2, float *__restrict__ Y, int64_t ldy,
                          unsigned long long *__restrict__ nfall, int64_t *__restrict__ flist) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t m = blockIdx.y;
    if (n >= Dp || m >= rows) return;
    const int64_t plane = rows * (int64_t)Dpk;
    int32_t c[LV - 1];
#pragma unroll
    for (int l = 2; l <= LV; l++) c[l - 2] = C[(int64_t)(l - 2) * plane + m * Dpk + n];
    double acc = 0.0, mag = 0.0;
#pragma unroll
    for (int l = LV; l >= 2; l--) {  // ascending magnitude; 2^-7l exact
        const double t = (double)c[l - 2] * pow2(-7 * l);
        acc += t;
        mag += fabs(t);
    }
    const double p2 = pow2(qe[m] + re[n]);  // exact (|exponents| small)
    const double y = acc * p2;
    const double b = ((double)Dp * 0x1p-53 + mag * 0x1p-50) * p2 + (double)Dp * 0x1p-53 * 1.01 * qn2[m] * rn2[n];
    const float f = (float)y;
    // neighbours of f (bit steps; f = 0 -> the smallest subnormals)
    const int fb = __float_as_int(f);
    const float fdn = f == 0.f ? -1.4e-45f : __int_as_float(f > 0.f ? fb - 1 : fb + 1);
    const float fup = f == 0.f ? 1.4e-45f : __int_as_float(f > 0.f ? fb + 1 : fb - 1);
    const double lo = 0.5 * ((double)f + (double)fdn);
    const double hi = 0.5 * ((double)f + (double)fup);
    Y[m * ldy + n] = f;
    if (!(y - b > lo && y + b < hi)) flist[atomicAdd(nfall, 1ull)] = m * Dp + n;  // k_recompute
}

// the uncertified outputs: the sequential chain itself, a thread per output,
// reading q' s row and R's column n (Rt: R transposed) as float4 streams with
// 32 terms in flight ahead of their fma's
__global__ void __launch_bounds__(128) k_recompute(const unsigned long long *__restrict__ nfall,
                                                   const int64_t *__restrict__ flist, int Dp,
                                                   const float *__restrict__ X, int64_t ldx,
                                                   const float *__restrict__ Rt, float *__restrict__ Y,
                                                   int64_t ldy) {
    const int64_t nf = (int64_t)*nfall;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t mn = flist[i], m = mn / Dp;
        const int n = (int)(mn - m * Dp);
        const float *xr = X + m * ldx, *rr = Rt + (int64_t)n * Dp;
        double s = 0.0;
        int k = 0;
        if (((ldx | Dp) & 3) == 0) {
            const float4 *x4 = (const float4 *)xr, *r4 = (const float4 *)rr;
            const int nv = Dp / 4;
            float4 xa[8], ra[8];
#pragma unroll
            for (int j = 0; j < 8; j++) {
                xa[j] = j < nv ? __ldg(x4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
                ra[j] = j < nv ? __ldg(r4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            for (int v0 = 0; v0 < nv; v0 += 8) {
                float4 xb[8], rb[8];
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const int v = v0 + 8 + j;
                    xb[j] = v < nv ? __ldg(x4 + v) : make_float4(0.f, 0.f, 0.f, 0.f);
                    rb[j] = v < nv ? __ldg(r4 + v) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int j = 0; j < 8; j++)
                    if (v0 + j < nv) {
                        s = __fma_rn((double)xa[j].x, (double)ra[j].x, s);
                        s = __fma_rn((double)xa[j].y, (double)ra[j].y, s);
                        s = __fma_rn((double)xa[j].z, (double)ra[j].z, s);
                        s = __fma_rn((double)xa[j].w, (double)ra[j].w, s);
                    }
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    xa[j] = xb[j];
                    ra[j] = rb[j];
                }
            }
            k = nv * 4;
        }
        for (; k < Dp; k++) s = __fma_rn((double)xr[k], (double)rr[k], s);
        Y[m * ldy + n] = (float)s;
    }
}

// Rt = R^T (fp32), the recompute's contiguous columns
__global__ void k_transpose(const float *__restrict__ R, int Dp, float *__restrict__ Rt) {
    __shared__ float t[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int r = by + j, c = bx + threadIdx.x;
        t[j][threadIdx.x] = (r < Dp && c < Dp) ? R[(int64_t)r * Dp + c] : 0.f;
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int r = bx + j, c = by + threadIdx.x;
        if (r < Dp && c < Dp) Rt[(int64_t)r * Dp + c] = t[threadIdx.x][j];
    }
}

struct Plan {
    cublasLtMatmulDesc_t op = nullptr;
    cublasLtMatrixLayout_t la[LV + 1] = {}, lb[LV + 1] = {}, lc = nullptr;
    cublasLtMatmulAlgo_t algo[LV + 1];
};
std::map<std::tuple<int, int, int64_t>, Plan> g_plans;  // (Dp, Dpk, rows)

void *ensure_lt(int device) {
    if (!g_lt) CRISP_LT(cublasLtCreate(&g_lt));
    void *&ws = g_ws[device];
    if (!ws) CRISP_CUDA(cudaMalloc(&ws, WS_BYTES));
    return ws;
}

const Plan &plan_for(int Dp, int Dpk, int64_t rows) {
    auto key = std::make_tuple(Dp, Dpk, rows);
    auto it = g_plans.find(key);
    if (it != g_plans.end()) return it->second;
    Plan p;
    CRISP_LT(cublasLtMatmulDescCreate(&p.op, CUBLAS_COMPUTE_32I, CUDA_R_32I));
    const cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
    CRISP_LT(cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)));
    CRISP_LT(cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)));
    // column-major: D (Dpk x rows) = A^T (Dpk x K') B (K' x rows); A = R slices (row n
    // of Rsl, ld SL Dpk), B = query slices (row m of Qcat, ld SL Dpk)
    CRISP_LT(cublasLtMatrixLayoutCreate(&p.lc, CUDA_R_32I, Dpk, rows, Dpk));  // outputs padded to Dpk (aligned)
    cublasLtMatmulPreference_t pref;
    CRISP_LT(cublasLtMatmulPreferenceCreate(&pref));
    size_t wsb = WS_BYTES;
    CRISP_LT(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof(wsb)));
    for (int l = 2; l <= LV; l++) {
        const uint64_t K = (uint64_t)(l - 1) * Dpk;
        CRISP_LT(cublasLtMatrixLayoutCreate(&p.la[l], CUDA_R_8I, K, Dpk, (int64_t)SL * Dpk));
        CRISP_LT(cublasLtMatrixLayoutCreate(&p.lb[l], CUDA_R_8I, K, rows, (int64_t)SL * Dpk));
        cublasLtMatmulHeuristicResult_t res;
        int nres = 0;
        CRISP_LT(cublasLtMatmulAlgoGetHeuristic(g_lt, p.op, p.la[l], p.lb[l], p.lc, p.lc, pref, 1, &res, &nres));
        if (nres == 0) {
            cublasLtMatmulPreferenceDestroy(pref);
            set_error("cublasLt: no int8 GEMM algorithm for the rotation");
            throw Err{CRISP_ECUDA};
        }
        p.algo[l] = res.algo;
    }
    cublasLtMatmulPreferenceDestroy(pref);
    if (g_plans.size() > 64) g_plans.clear();  // (descriptors of dropped plans are leaked: bounded)
    return g_plans.emplace(key, p).first->second;
}

}  // namespace

int rotation_slices_k(int Dp) { return (Dp + 15) / 16 * 16; }

void prepare_rotation_slices(crisp_index *ix, cudaStream_t s) {
    if (!ix->R || ix->Rsl) return;
    const int Dp = ix->Dp, Dpk = rotation_slices_k(Dp);
    int8_t *tmp = nullptr;
    CRISP_CUDA(cudaMalloc(&ix->Rsl, (size_t)Dpk * SL * Dpk));  // rows n >= Dp stay zero
    CRISP_CUDA(cudaMemsetAsync(ix->Rsl, 0, (size_t)Dpk * SL * Dpk, s));
    CRISP_CUDA(cudaMalloc(&ix->Rexp, (size_t)Dp * 4));
    CRISP_CUDA(cudaMalloc(&ix->Rn2, (size_t)Dp * 8));
    CRISP_CUDA(cudaMalloc(&ix->Rt, (size_t)Dp * Dp * 4));
    ix->hbm_bytes += (int64_t)Dpk * SL * Dpk + (int64_t)Dp * 12 + (int64_t)Dp * Dp * 4;
    k_transpose<<<dim3((Dp + 31) / 32, (Dp + 31) / 32), dim3(32, 8), 0, s>>>(ix->R, Dp, ix->Rt);
    CRISP_LAUNCH();
    CRISP_CUDA(cudaMallocAsync(&tmp, (size_t)Dp * SL * Dpk, s));
    k_slice_cols<<<(Dp + 7) / 8, 256, 0, s>>>(ix->R, Dp, Dpk, tmp, ix->Rsl, ix->Rexp, ix->Rn2);
    CRISP_LAUNCH();
    CRISP_CUDA(cudaFreeAsync(tmp, s));
}

bool rotate_imma_enabled() {
    static const bool on = getenv("CRISP_ROTATE_IMMA") ? atoi(getenv("CRISP_ROTATE_IMMA")) != 0 : true;
    return on;
}

// Y (rows x ldy) = fl32(X R) for X rows (ldx, zero beyond D), certified (see top)
void rotate_rows_imma(const crisp_index *ix, const float *X, int64_t rows, int64_t ldx, float *Y, int64_t ldy,
                      cudaStream_t s, unsigned long long *nfall) {
    if (rows <= 0) return;
    const int Dp = ix->Dp, Dpk = rotation_slices_k(Dp);
    std::lock_guard<std::mutex> lk(g_mu);
    void *ws = ensure_lt(ix->device);
    const Plan &p = plan_for(Dp, Dpk, rows);
    // scratch: Qcat (rows x SL Dpk int8) | C (LV-1 levels x rows x Dp int32) | qn2 | qe
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t qbytes = up((size_t)rows * SL * Dpk), cbytes = up((size_t)(LV - 1) * rows * Dpk * 4);
    char *buf = nullptr;
    CRISP_CUDA(cudaMallocAsync(&buf, qbytes + cbytes + up((size_t)rows * 8) + up((size_t)rows * 4), s));
    int8_t *Qcat = (int8_t *)buf;
    int32_t *C = (int32_t *)(buf + qbytes);
    double *qn2 = (double *)(buf + qbytes + cbytes);
    int32_t *qe = (int32_t *)(buf + qbytes + cbytes + up((size_t)rows * 8));
    k_slice_rows<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(X, rows, Dp, ldx, Dpk, Qcat, qe, qn2);
    CRISP_LAUNCH();
    const int32_t alpha = 1, beta = 0;
    for (int l = 2; l <= LV; l++) {
        const int8_t *A = ix->Rsl + (size_t)(LV - l) * Dpk;  // [b_{l-1} .. b_1]
        int32_t *Cl = C + (size_t)(l - 2) * rows * Dpk;
        CRISP_LT(cublasLtMatmul(g_lt, p.op, &alpha, A, p.la[l], Qcat, p.lb[l], &beta, Cl, p.lc, Cl, p.lc, &p.algo[l],
                                ws, WS_BYTES, s));
    }
    // uncertified outputs: counter + list (at most rows x Dp entries)
    unsigned long long *cnt = nullptr;
    int64_t *flist = nullptr;
    const size_t fcap = (size_t)rows * Dp;
    CRISP_CUDA(cudaMallocAsync(&cnt, 8 + fcap * 8, s));
    flist = (int64_t *)(cnt + 1);
    CRISP_CUDA(cudaMemsetAsync(cnt, 0, 8, s));
    dim3 g((Dp + 127) / 128, (unsigned)rows);
    k_certify<<<g, 128, 0, s>>>(C, rows, Dp, Dpk, qe, qn2, ix->Rexp, ix->Rn2, Y, ldy, cnt, flist);
    CRISP_LAUNCH();
    k_recompute<<<148 * 8, 128, 0, s>>>(cnt, flist, Dp, X, ldx, ix->Rt, Y, ldy);
    CRISP_LAUNCH();
    if (nfall) CRISP_CUDA(cudaMemcpyAsync(nfall, cnt, 8, cudaMemcpyDeviceToDevice, s));
    // CRISP_IMMA_STATS=1: report the uncertified outputs on stderr (diagnostics; syncs)
    static const bool stats = getenv("CRISP_IMMA_STATS") && atoi(getenv("CRISP_IMMA_STATS")) != 0;
    if (stats) {
        unsigned long long h = 0;
        CRISP_CUDA(cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, s));
        CRISP_CUDA(cudaStreamSynchronize(s));
        fprintf(stderr, "crisp imma: %llu of %lld outputs recomputed\n", h, (long long)(rows * Dp));
    }
    CRISP_CUDA(cudaFreeAsync(cnt, s));
    CRISP_CUDA(cudaFreeAsync(buf, s));
}

// a0 for rows of X: the certified int8 path when enabled and available for
// this D' (cuBLASLt has an int8 kernel for the shapes), else the fp64 FMA
// kernel; both give the oracle's fl32 of the sequential chain
void rotate_rows(crisp_index *ix, const float *X, int64_t rows, int64_t ldx, float *Y, int64_t ldy, cudaStream_t s) {
    static std::mutex mu;
    static std::map<int, bool> unavailable;  // D' values cuBLASLt rejected
    bool imma = rotate_imma_enabled();
    if (imma) {
        std::lock_guard<std::mutex> lk(mu);
        imma = !unavailable.count(ix->Dp);
    }
    if (imma) {
        try {
            prepare_rotation_slices(ix, s);
            rotate_rows_imma(ix, X, rows, ldx, Y, ldy, s, nullptr);
            return;
        } catch (Err &) {
            std::lock_guard<std::mutex> lk(mu);
            unavailable[ix->Dp] = true;
        }
    }
    rotate_rows_f64(X, rows, ix->Dp, ldx, ix->R, Y, ldy, s);
}

}  // namespace crisp
