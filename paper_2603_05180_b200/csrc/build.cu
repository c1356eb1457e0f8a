// build.cu -- crisp_build on the GPU (P:L249-256 phases 1-2).
//
// Every step that decides an integer (sample choice, cell assignment, CSR
// order) or feeds the search (X', codebooks) is computed in a fixed, sequential
// fp64 order per output element so that, given the same inputs, it reproduces
// the oracle's values exactly.  Only the eigenvalues (cuSOLVER
// syevd) and the QR factor (cuSOLVER geqrf/orgqr) use a library with its own
// summation order; they feed a threshold decision (CEV > 0.85) and R, which
// parity tests inject (crisp_build_with) or check by property.
#include <cub/cub.cuh>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "crisp_internal.cuh"

namespace crisp {

#define CRISP_SOLVER(call)                                                                      \
    do {                                                                                        \
        cusolverStatus_t s_ = (call);                                                           \
        if (s_ != CUSOLVER_STATUS_SUCCESS) {                                                    \
            set_error(std::string(#call) + ": cusolver status " + std::to_string((int)s_));     \
            throw Err{CRISP_ECUDA};                                                             \
        }                                                                                       \
    } while (0)

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// RAII device scratch for the build (freed when the build step returns)
struct Scratch {
    std::vector<void *> ptrs;
    void *get(size_t bytes) {
        void *p = nullptr;
        CRISP_CUDA(cudaMalloc(&p, bytes ? bytes : 16));
        ptrs.push_back(p);
        return p;
    }
    template <class T>
    T *alloc(size_t n) { return (T *)get(n * sizeof(T)); }
    ~Scratch() {
        for (void *p : ptrs) cudaFree(p);
    }
};

// ---------------------------------------------------------------------------
// fp64 sequential-order GEMM: C[m][n] = sum_k fma(a(m,k), b(k,n), s) with k
// ascending from s = +0.  64x64 tile per CTA, 16x16 threads, 4x4 outputs each.
// ---------------------------------------------------------------------------
template <class LA, class LB, class ST>
__global__ void __launch_bounds__(256) k_gemm_seq(int64_t Mr, int Nc, int Kd, LA la, LB lb, ST st) {
    __shared__ double As[16][64];
    __shared__ double Bs[16][64];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t m0 = (int64_t)blockIdx.y * 64;
    const int n0 = blockIdx.x * 64;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = 0.0;
    for (int k0 = 0; k0 < Kd; k0 += 16) {
        for (int e = threadIdx.x; e < 1024; e += 256) {
            int mm = e >> 4, kk = e & 15;
            As[kk][mm] = (m0 + mm < Mr && k0 + kk < Kd) ? la(m0 + mm, k0 + kk) : 0.0;
        }
        for (int e = threadIdx.x; e < 1024; e += 256) {
            int kk = e >> 6, nn = e & 63;
            Bs[kk][nn] = (k0 + kk < Kd && n0 + nn < Nc) ? lb(k0 + kk, n0 + nn) : 0.0;
        }
        __syncthreads();
        const int kmax = min(16, Kd - k0);
        for (int kk = 0; kk < kmax; kk++) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; i++) a[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; j++) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = __fma_rn(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) {
            int64_t m = m0 + ty + 16 * i;
            int n = n0 + tx + 16 * j;
            if (m < Mr && n < Nc) st(m, n, acc[i][j]);
        }
}

struct LoadRowF32 {  // a(m,k) = X[m*ld + k]
    const float *X;
    int64_t ld;
    __device__ double operator()(int64_t m, int k) const { return (double)X[m * ld + k]; }
};
struct LoadMatF32 {  // b(k,n) = R[k*ld + n]
    const float *R;
    int ld;
    __device__ double operator()(int k, int n) const { return (double)R[(int64_t)k * ld + n]; }
};
struct StoreF32 {
    float *Y;
    int64_t ld;
    __device__ void operator()(int64_t m, int n, double v) const { Y[m * ld + n] = (float)v; }
};
// covariance: a(i, r) = S[r][i] - mu[i], b(r, j) = S[r][j] - mu[j]
struct LoadCentT {
    const float *S;
    const double *mu;
    int D;
    __device__ double operator()(int64_t i, int r) const {
        return __dsub_rn((double)S[(int64_t)r * D + i], mu[i]);
    }
};
struct LoadCent {
    const float *S;
    const double *mu;
    int D;
    __device__ double operator()(int r, int j) const {
        return __dsub_rn((double)S[(int64_t)r * D + j], mu[j]);
    }
};
struct StoreCov {
    double *C;
    int D;
    double inv;  // 1/(n-1) applied as a division below
    double nm1;
    __device__ void operator()(int64_t i, int j, double v) const { C[i * D + j] = v / nm1; }
};

// ---------------------------------------------------------------------------
// Rotation Y = fl32(X . R), the same sequential fp64 order per
// output as k_gemm_seq (k ascending from +0; padded k contribute fma(0, 0, s) =
// s exactly), with a larger register tile: 128x64 outputs per CTA, 8x4 per
// thread, k-tiles of 32 staged as doubles in shared memory, double-buffered:
// the global loads of tile t+1 are in registers while tile t is multiplied.
// ---------------------------------------------------------------------------
constexpr int RT_BM = 128, RT_BN = 64, RT_BK = 32;
constexpr int RT_AV = RT_BM * (RT_BK / 4) / 256;  // float4s of A per thread per tile (4)
constexpr int RT_BV = RT_BK * RT_BN / 256;        // floats of B per thread per tile (8)
struct RotTile {
    float4 a[RT_AV];
    float b[RT_BV];
};
__device__ __forceinline__ void rot_load(RotTile &t, int64_t Mr, int Dp, const float *__restrict__ X, int64_t ldx,
                                         const float *__restrict__ R, int64_t m0, int n0, int k0, bool vecA, int tid) {
#pragma unroll
    for (int u = 0; u < RT_AV; u++) {
        const int e = tid + u * 256;
        const int r = e >> 3, kq = (e & 7) * 4;
        const int64_t m = m0 + r;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (m < Mr) {
            const float *src = X + m * ldx + k0 + kq;
            if (vecA && k0 + kq + 3 < Dp) v = __ldg((const float4 *)src);
            else {
                v.x = k0 + kq < Dp ? src[0] : 0.f;
                v.y = k0 + kq + 1 < Dp ? src[1] : 0.f;
                v.z = k0 + kq + 2 < Dp ? src[2] : 0.f;
                v.w = k0 + kq + 3 < Dp ? src[3] : 0.f;
            }
        }
        t.a[u] = v;
    }
#pragma unroll
    for (int u = 0; u < RT_BV; u++) {
        const int e = tid + u * 256;
        const int kk = e >> 6, nn = e & 63;
        const int k = k0 + kk, n = n0 + nn;
        t.b[u] = (k < Dp && n < Dp) ? __ldg(R + (int64_t)k * Dp + n) : 0.f;
    }
}
__device__ __forceinline__ void rot_store(const RotTile &t, double *As, double *Bs, int tid) {
#pragma unroll
    for (int u = 0; u < RT_AV; u++) {
        const int e = tid + u * 256;
        const int r = e >> 3, kq = (e & 7) * 4;
        As[(kq + 0) * RT_BM + r] = (double)t.a[u].x;
        As[(kq + 1) * RT_BM + r] = (double)t.a[u].y;
        As[(kq + 2) * RT_BM + r] = (double)t.a[u].z;
        As[(kq + 3) * RT_BM + r] = (double)t.a[u].w;
    }
#pragma unroll
    for (int u = 0; u < RT_BV; u++) {
        const int e = tid + u * 256;
        Bs[(e >> 6) * RT_BN + (e & 63)] = (double)t.b[u];
    }
}
__global__ void __launch_bounds__(256, 2) k_rotate_f64(int64_t Mr, int Dp, const float *__restrict__ X, int64_t ldx,
                                                        const float *__restrict__ R, float *__restrict__ Y,
                                                        int64_t ldy) {
    extern __shared__ __align__(16) double rsm[];
    constexpr int TS = RT_BK * RT_BM + RT_BK * RT_BN;  // doubles per stage
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t m0 = (int64_t)blockIdx.y * RT_BM;
    const int n0 = blockIdx.x * RT_BN;
    double acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = 0.0;
    const bool vecA = (ldx & 3) == 0;
    RotTile t;
    rot_load(t, Mr, Dp, X, ldx, R, m0, n0, 0, vecA, tid);
    rot_store(t, rsm, rsm + RT_BK * RT_BM, tid);
    __syncthreads();
    int stage = 0;
    for (int k0 = 0; k0 < Dp; k0 += RT_BK) {
        const bool more = k0 + RT_BK < Dp;
        if (more) rot_load(t, Mr, Dp, X, ldx, R, m0, n0, k0 + RT_BK, vecA, tid);
        const double *As = rsm + stage * TS, *Bs = As + RT_BK * RT_BM;
#pragma unroll 4
        for (int kk = 0; kk < RT_BK; kk++) {
            double a[8], b[4];
#pragma unroll
            for (int i = 0; i < 8; i++) a[i] = As[kk * RT_BM + ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; j++) b[j] = Bs[kk * RT_BN + tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = __fma_rn(a[i], b[j], acc[i][j]);
        }
        if (more) {
            double *An = rsm + (stage ^ 1) * TS;
            rot_store(t, An, An + RT_BK * RT_BM, tid);  // the other stage: last read before the previous barrier
        }
        __syncthreads();
        stage ^= 1;
    }
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int64_t m = m0 + ty + 16 * i;
            const int n = n0 + tx + 16 * j;
            if (m < Mr && n < Dp) Y[m * ldy + n] = (float)acc[i][j];
        }
}

void rotate_rows_f64(const float *X, int64_t rows, int32_t Dp, int64_t ldx, const float *R, float *Y, int64_t ldy,
                     cudaStream_t s) {
    if (rows <= 0) return;
    static bool attr = false;
    const int smem = 2 * (RT_BK * RT_BM + RT_BK * RT_BN) * 8;
    if (!attr) {
        CRISP_CUDA(cudaFuncSetAttribute(k_rotate_f64, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr = true;
    }
    dim3 grid(nblk(Dp, RT_BN), (unsigned)((rows + RT_BM - 1) / RT_BM));
    k_rotate_f64<<<grid, 256, smem, s>>>(rows, Dp, X, ldx, R, Y, ldy);
    CRISP_LAUNCH();
}

// ---------------------------------------------------------------------------
// sampling: n rows of smallest (philox key, index)
// ---------------------------------------------------------------------------
__global__ void k_sample_keys(int64_t N, uint64_t seed, uint32_t stream, uint64_t *keys, int32_t *idx) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    uint32_t o[4];
    draw(seed, stream, (uint64_t)i, 0, o);
    keys[i] = ((uint64_t)o[0] << 32) | o[1];
    idx[i] = (int32_t)i;
}

static void sample_rows(int64_t N, int64_t n, uint64_t seed, uint32_t stream, int32_t *rows_out, cudaStream_t s) {
    Scratch sc;
    uint64_t *k1 = sc.alloc<uint64_t>(N), *k2 = sc.alloc<uint64_t>(N);
    int32_t *i1 = sc.alloc<int32_t>(N), *i2 = sc.alloc<int32_t>(N);
    k_sample_keys<<<nblk(N, 256), 256, 0, s>>>(N, seed, stream, k1, i1);
    CRISP_LAUNCH();
    size_t tb = 0;
    CRISP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k1, k2, i1, i2, (int)N, 0, 64, s));
    void *tmp = sc.get(tb);
    // stable radix sort: equal keys keep ascending index order
    CRISP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k1, k2, i1, i2, (int)N, 0, 64, s));
    size_t tb2 = 0;
    CRISP_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb2, i2, rows_out, (int)n, 0, 32, s));
    void *tmp2 = sc.get(tb2);
    CRISP_CUDA(cub::DeviceRadixSort::SortKeys(tmp2, tb2, i2, rows_out, (int)n, 0, 32, s));
    CRISP_CUDA(cudaStreamSynchronize(s));
}

__global__ void k_gather_rows(const float *X, int64_t ld, const int32_t *rows, int64_t n, int D, float *out) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * D) return;
    int64_t r = e / D;
    int c = (int)(e % D);
    out[e] = X[(int64_t)rows[r] * ld + c];
}

// ---------------------------------------------------------------------------
// CEV
// ---------------------------------------------------------------------------
__global__ void k_colmean(const float *S, int64_t n, int D, double *mu) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= D) return;
    double s = 0.0;
    for (int64_t r = 0; r < n; r++) s = __dadd_rn(s, (double)S[r * D + i]);
    mu[i] = s / (double)n;
}

// CEV sample size (Z16): ceil(min(0.1 N, 1e5)), all rows if N <= 10
int64_t cev_sample_size(int64_t N) { return (N <= 10) ? N : std::min<int64_t>((N + 9) / 10, 100000); }

// rows of the sample of size n (ascending index): all rows when n == N
static void sample_or_all(int64_t N, int64_t n, uint64_t seed, uint32_t stream, int32_t *rows, cudaStream_t s) {
    if (n == N) {
        std::vector<int32_t> h(n);
        for (int64_t i = 0; i < n; i++) h[i] = (int32_t)i;
        CRISP_CUDA(cudaMemcpy(rows, h.data(), n * 4, cudaMemcpyHostToDevice));
    } else {
        sample_rows(N, n, seed, stream, rows, s);
    }
}

void sample_row_ids(int64_t N, int64_t n, uint64_t seed, uint32_t stream, int32_t *rows_dev, cudaStream_t s) {
    sample_or_all(N, n, seed, stream, rows_dev, s);
}

static double cev_of_rows(const float *S, int64_t n, int D, cudaStream_t s, std::vector<double> *var = nullptr);

// the CEV of the dataset's sample; var (optional) receives the sample's per-dimension
// variances (the covariance diagonal), zeros if the sample has fewer than 2 rows
static double compute_cev(const float *X, int64_t N, int64_t ld, int D, uint64_t seed, cudaStream_t s,
                          std::vector<double> *var = nullptr) {
    const int64_t n = cev_sample_size(N);
    if (var) var->assign(D, 0.0);
    if (n < 2) return 0.0;
    Scratch sc;
    int32_t *rows = sc.alloc<int32_t>(n);
    sample_or_all(N, n, seed, STREAM_CEV_SAMPLE, rows, s);
    float *S = sc.alloc<float>((size_t)n * D);
    k_gather_rows<<<nblk(n * D, 256), 256, 0, s>>>(X, ld, rows, n, D, S);
    CRISP_LAUNCH();
    return cev_of_rows(S, n, D, s, var);
}

// CEV of the sample rows S (n x D, packed, ascending global index): covariance with
// divisor n-1 in the sequential fp64 order, eigenvalues, top floor(0.2 D) share
static double cev_of_rows(const float *S, int64_t n, int D, cudaStream_t s, std::vector<double> *var) {
    if (var) var->assign(D, 0.0);
    if (n < 2) return 0.0;
    Scratch sc;
    double *mu = sc.alloc<double>(D);
    k_colmean<<<nblk(D, 128), 128, 0, s>>>(S, n, D, mu);
    CRISP_LAUNCH();
    double *Cm = sc.alloc<double>((size_t)D * D);
    dim3 grid(nblk(D, 64), nblk(D, 64));
    k_gemm_seq<<<grid, 256, 0, s>>>((int64_t)D, D, (int)n, LoadCentT{S, mu, D}, LoadCent{S, mu, D},
                                    StoreCov{Cm, D, 0.0, (double)(n - 1)});
    CRISP_LAUNCH();
    if (var) {  // the per-dimension variances (block-wise rotation, R16), before the solver overwrites Cm
        CRISP_CUDA(cudaMemcpy2DAsync(var->data(), 8, Cm, (size_t)(D + 1) * 8, 8, D, cudaMemcpyDeviceToHost, s));
        CRISP_CUDA(cudaStreamSynchronize(s));
    }
    // eigenvalues only (symmetric; layout irrelevant)
    cusolverDnHandle_t h;
    CRISP_SOLVER(cusolverDnCreate(&h));
    struct HG {
        cusolverDnHandle_t h;
        ~HG() { cusolverDnDestroy(h); }
    } hg{h};
    CRISP_SOLVER(cusolverDnSetStream(h, s));
    double *w = sc.alloc<double>(D);
    int lw = 0;
    CRISP_SOLVER(cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_LOWER, D, Cm, D, w, &lw));
    double *work = sc.alloc<double>(lw);
    int *info = sc.alloc<int>(1);
    CRISP_SOLVER(cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_LOWER, D, Cm, D, w, work, lw, info));
    std::vector<double> hw(D);
    int hinfo = 0;
    CRISP_CUDA(cudaMemcpyAsync(hw.data(), w, D * 8, cudaMemcpyDeviceToHost, s));
    CRISP_CUDA(cudaMemcpyAsync(&hinfo, info, 4, cudaMemcpyDeviceToHost, s));
    CRISP_CUDA(cudaStreamSynchronize(s));
    CRISP_CHECK(hinfo == 0, "eigensolver failed to converge");
    // CEV = sum of the top floor(0.2 D) eigenvalues / sum, negatives clamped
    std::sort(hw.begin(), hw.end(), [](double a, double b) { return a > b; });
    int kk = std::max(1, D / 5);
    double top = 0.0, tot = 0.0;
    for (int i = 0; i < D; i++) {
        double l = hw[i] > 0.0 ? hw[i] : 0.0;
        tot += l;
        if (i < kk) top += l;
    }
    return tot < 1e-12 ? 0.0 : top / tot;
}

// ---------------------------------------------------------------------------
// rotation: G ~ N(0,1) by Philox + Box-Muller, QR, sign fix
// ---------------------------------------------------------------------------
__global__ void k_gaussian_colmajor(int D, uint64_t seed, double *Gcm) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // e = i*D + j (row-major index)
    if (e >= (int64_t)D * D) return;
    int64_t i = e / D, j = e % D;
    uint32_t o[4];
    draw(seed, STREAM_ROTATION, (uint64_t)e, 0, o);
    double u1 = 1.0 - u53(o[0], o[1]);
    double u2 = u53(o[2], o[3]);
    Gcm[j * D + i] = sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}
__global__ void k_diag(const double *A, int D, double *d) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < D) d[i] = A[(int64_t)i * D + i];
}
// R[i][j] (row-major fp32) = Q(i,j) * sign(R'_jj); Q column-major
__global__ void k_q_to_R(const double *Qcm, const double *diag, int D, float *R) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)D * D) return;
    int64_t i = e / D, j = e % D;
    double q = Qcm[j * D + i];
    if (diag[j] < 0.0) q = -q;
    R[e] = (float)q;
}

static void make_rotation(int D, uint64_t seed, float *R, cudaStream_t s) {
    Scratch sc;
    double *A = sc.alloc<double>((size_t)D * D);
    k_gaussian_colmajor<<<nblk((int64_t)D * D, 256), 256, 0, s>>>(D, seed, A);
    CRISP_LAUNCH();
    cusolverDnHandle_t h;
    CRISP_SOLVER(cusolverDnCreate(&h));
    struct HG {
        cusolverDnHandle_t h;
        ~HG() { cusolverDnDestroy(h); }
    } hg{h};
    CRISP_SOLVER(cusolverDnSetStream(h, s));
    double *tau = sc.alloc<double>(D);
    int *info = sc.alloc<int>(1);
    int lw1 = 0, lw2 = 0;
    CRISP_SOLVER(cusolverDnDgeqrf_bufferSize(h, D, D, A, D, &lw1));
    CRISP_SOLVER(cusolverDnDorgqr_bufferSize(h, D, D, D, A, D, tau, &lw2));
    double *work = sc.alloc<double>(std::max(lw1, lw2));
    CRISP_SOLVER(cusolverDnDgeqrf(h, D, D, A, D, tau, work, lw1, info));
    double *dg = sc.alloc<double>(D);
    k_diag<<<nblk(D, 128), 128, 0, s>>>(A, D, dg);
    CRISP_LAUNCH();
    CRISP_SOLVER(cusolverDnDorgqr(h, D, D, D, A, D, tau, work, lw2, info));
    k_q_to_R<<<nblk((int64_t)D * D, 256), 256, 0, s>>>(A, dg, D, R);
    CRISP_LAUNCH();
    int hinfo = 0;
    CRISP_CUDA(cudaMemcpyAsync(&hinfo, info, 4, cudaMemcpyDeviceToHost, s));
    CRISP_CUDA(cudaStreamSynchronize(s));
    CRISP_CHECK(hinfo == 0, "QR failed");
}

// In-place X' = X R over row chunks with one scratch tile.
static void rotate_in_place(crisp_index *ix, cudaStream_t s) {
    const int64_t rowbytes = (int64_t)ix->pitch * 4;
    int64_t rc = std::max<int64_t>(64, std::min<int64_t>(ix->N, (512LL << 20) / rowbytes));
    rc = std::min<int64_t>(rc, 32768);  // the certify grid and the level scratch per tile (rotate_imma.cu)
    Scratch sc;
    float *tile = sc.alloc<float>((size_t)rc * ix->pitch);
    for (int64_t r0 = 0; r0 < ix->N; r0 += rc) {
        int64_t rows = std::min(rc, ix->N - r0);
        rotate_rows(ix, ix->X + r0 * ix->pitch, rows, ix->pitch, tile, ix->pitch, s);
        CRISP_CUDA(cudaMemcpy2DAsync(ix->X + r0 * ix->pitch, rowbytes, tile, rowbytes, (size_t)ix->Dp * 4, rows,
                                     cudaMemcpyDeviceToDevice, s));
    }
    CRISP_CUDA(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------------------
// k-means per half-subspace (details S:L221), all 2M halves
// at once.  S: n x Dp sample (row pitch Dp); half h covers dims [h*dh,(h+1)*dh).
// ---------------------------------------------------------------------------
__global__ void k_kpp_first(const float *S, int64_t n, int Dp, int dh, int K, int nh, uint64_t seed, float *C) {
    int h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= nh) return;
    double u = uniform(seed, STREAM_KM_INIT, 0, (uint32_t)h);
    int64_t p0 = (int64_t)(u * (double)n);
    if (p0 >= n) p0 = n - 1;
    for (int t = 0; t < dh; t++) C[((int64_t)h * K + 0) * dh + t] = S[p0 * Dp + (int64_t)h * dh + t];
}
__global__ void k_kpp_d2(const float *S, int64_t n, int Dp, int dh, int K, int nh, const float *C, int c,
                         double *D2) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * nh) return;
    int h = (int)(e / n);
    int64_t p = e % n;
    double d = dist64(S + p * Dp + (int64_t)h * dh, C + ((int64_t)h * K + c) * dh, dh);
    if (c == 0 || d < D2[e]) D2[e] = d;
}
// k-means++ pick: the sequential fp64 sums of the oracle (total,
// then the running sum up to the first position above u * total), one CTA per
// half-subspace: the CTA stages D2 through shared memory in chunks, one thread
// keeps the sums in the oracle's order (the loads are no longer on its chain)
constexpr int KPP_CH = 2048;  // doubles per staged chunk
__global__ void __launch_bounds__(256) k_kpp_pick(const float *S, int64_t n, int Dp, int dh, int K, int nh,
                                                  uint64_t seed, int c, const double *D2, float *C) {
    __shared__ double buf[2][KPP_CH];
    __shared__ int64_t s_pick;
    __shared__ int s_stop;
    const int h = blockIdx.x;
    const double *d = D2 + (int64_t)h * n;
    const int tid = threadIdx.x;
    // pass 1: total; pass 2: the running sum against the target
    double tot = 0.0, target = 0.0, cum = 0.0;
    int64_t lastpos = 0, pick = -1;
    const double uc = uniform(seed, STREAM_KM_INIT, (uint64_t)c, (uint32_t)h);
    for (int pass = 0; pass < 2; pass++) {
        if (pass == 1) {
            if (tid == 0) s_stop = !(tot > 0.0);
            __syncthreads();
            if (s_stop) break;
            target = uc * tot;
        }
        int b = 0;
        for (int64_t p0 = 0; p0 < n; p0 += KPP_CH, b ^= 1) {
            // the other threads load chunk i+1 while thread 0 sums chunk i (one barrier
            // per chunk: chunk i+2 reuses chunk i's buffer only after thread 0 passed it)
            const int cn = (int)(n - p0 < KPP_CH ? n - p0 : KPP_CH);
            for (int i = tid; i < cn; i += blockDim.x) buf[b][i] = d[p0 + i];
            __syncthreads();
            if (pass == 1 && s_stop) break;
            if (tid == 0) {
                const double *x = buf[b];
                if (pass == 0) {
                    int i = 0;
                    for (; i + 8 <= cn; i += 8) {  // eight loads ahead of the adds
                        double v[8];
#pragma unroll
                        for (int u = 0; u < 8; u++) v[u] = x[i + u];
#pragma unroll
                        for (int u = 0; u < 8; u++) tot = __dadd_rn(tot, v[u]);
                    }
                    for (; i < cn; i++) tot = __dadd_rn(tot, x[i]);
                } else if (pick < 0) {
                    for (int i0 = 0; i0 < cn && pick < 0; i0 += 8) {
                        double v[8];
#pragma unroll
                        for (int u = 0; u < 8; u++) v[u] = i0 + u < cn ? x[i0 + u] : 0.0;
#pragma unroll
                        for (int u = 0; u < 8; u++) {
                            if (i0 + u < cn && pick < 0) {
                                if (v[u] > 0.0) lastpos = p0 + i0 + u;
                                cum = __dadd_rn(cum, v[u]);
                                if (cum > target) pick = p0 + i0 + u;
                            }
                        }
                    }
                    s_stop = pick >= 0;
                }
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        if (tot > 0.0) {
            if (pick < 0) pick = lastpos;
        } else {
            pick = (int64_t)(uc * (double)n);
            if (pick >= n) pick = n - 1;
        }
        s_pick = pick;
    }
    __syncthreads();
    const int64_t pk = s_pick;
    for (int t = tid; t < dh; t += blockDim.x) C[((int64_t)h * K + c) * dh + t] = S[pk * Dp + (int64_t)h * dh + t];
}
// k-means++ pick, certified parallel form.  All D2 >= 0, so any summation
// order of a prefix is within gamma = (n + 64) u of the exact prefix E(p); the
// oracle's sequential running sums cum(p) and total are too.  A thread sums
// its contiguous segment, a block scan gives the segment offsets, and from the
// parallel prefixes Ep and the certified interval [T_lo, T_hi] of the oracle's
// target u_c * total, the first p with certainly cum(p) > target is the pick
// when no earlier p possibly exceeds it; when nothing can exceed it the pick is
// the last positive position.  Any other case (a prefix within ~2e-11 of the
// target) takes the oracle's sequential rule in thread 0.
constexpr int KPP_T = 1024;
__global__ void __launch_bounds__(KPP_T) k_kpp_pick_par(const float *S, int64_t n, int Dp, int dh, int K,
                                                         uint64_t seed, int c, const double *D2, float *C) {
    __shared__ double wsum[KPP_T / 32];
    __shared__ int64_t s_first_sure, s_first_maybe, s_last;
    __shared__ int64_t s_pick;
    const int h = blockIdx.x;
    const double *d = D2 + (int64_t)h * n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t per = (n + KPP_T - 1) / KPP_T, lo = min(n, tid * per), hi = min(n, lo + per);
    double seg = 0.0;
    int64_t lastpos = -1;
    for (int64_t p = lo; p < hi; p++) {
        const double v = d[p];
        seg += v;
        if (v > 0.0) lastpos = p;
    }
    // exclusive block scan of the segment sums (warp scan + warp totals)
    double inc = seg;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += t;
    }
    if (lane == 31) wsum[warp] = inc;
    if (tid == 0) {
        s_first_sure = INT64_MAX;
        s_first_maybe = INT64_MAX;
        s_last = -1;
    }
    __syncthreads();
    if (warp == 0) {
        double w = wsum[lane];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, w, off);
            if (lane >= off) w += t;
        }
        wsum[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const double total = wsum[KPP_T / 32 - 1];
    double run = (warp ? wsum[warp - 1] : 0.0) + inc - seg;  // exclusive prefix of this segment
    atomicMax((unsigned long long *)&s_last, (unsigned long long)(lastpos + 1));  // +1: -1 -> 0
    const double uc = uniform(seed, STREAM_KM_INIT, (uint64_t)c, (uint32_t)h);
    const double g = ((double)n + 64.0) * 0x1p-53 * 1.01;  // any-order prefix vs exact
    const double g2 = 2.0 * g + 0x1p-50;                    // cum (or target) vs the parallel prefix (+ roundings)
    const double t_lo = uc * total * (1.0 - g2), t_hi = uc * total * (1.0 + g2);
    for (int64_t p = lo; p < hi; p++) {
        run += d[p];
        if (run * (1.0 - g2) > t_hi) {
            atomicMin((unsigned long long *)&s_first_sure, (unsigned long long)p);
            break;
        }
        if (run * (1.0 + g2) > t_lo) atomicMin((unsigned long long *)&s_first_maybe, (unsigned long long)p);
    }
    __syncthreads();
    if (tid == 0) {
        const int64_t last = s_last - 1;
        int64_t pick = -1;
        bool sure = false;
        if (!(total > 0.0)) {  // all D2 == 0 (exactly: non-negative terms)
            pick = (int64_t)(uc * (double)n);
            if (pick >= n) pick = n - 1;
            sure = true;
        } else if (s_first_sure != INT64_MAX) {
            // no earlier position may exceed the target
            if (s_first_maybe == INT64_MAX || s_first_maybe >= s_first_sure) {
                pick = s_first_sure;
                sure = true;
            }
        } else if (s_first_maybe == INT64_MAX) {
            pick = last;  // no position can exceed the target
            sure = true;
        }
        if (!sure) {  // the oracle's sequential rule
            double tot = 0.0;
            for (int64_t p = 0; p < n; p++) tot = __dadd_rn(tot, d[p]);
            const double target = uc * tot;
            double cum = 0.0;
            int64_t lp = 0;
            pick = -1;
            for (int64_t p = 0; p < n; p++) {
                if (d[p] > 0.0) lp = p;
                cum = __dadd_rn(cum, d[p]);
                if (cum > target) {
                    pick = p;
                    break;
                }
            }
            if (pick < 0) pick = lp;
        }
        s_pick = pick;
    }
    __syncthreads();
    const int64_t pk = s_pick;
    for (int t = tid; t < dh; t += KPP_T) C[((int64_t)h * K + c) * dh + t] = S[pk * Dp + (int64_t)h * dh + t];
}
// argmin over the K centroids of one half-subspace h for 128 points per CTA
// (Alg. "assign" S:L220): the centroids staged as doubles and the
// points' h-th half staged transposed (Xs[d][pt], pitch 129: conflict-free), so
// a thread reads its point and every lane the same centroid (broadcast).  Two
// centroids per pass share the point's conversion; each distance is dist64's
// sequential chain and ties keep the first centroid.
constexpr int AS_T = 128;
__global__ void __launch_bounds__(AS_T) k_argmin_staged(const float *__restrict__ P, int64_t n, int64_t ldp, int dh,
                                                        int K, const float *__restrict__ C,
                                                        const int *__restrict__ done, int32_t *__restrict__ a,
                                                        double *__restrict__ dmin, const int32_t *__restrict__ hoff) {
    extern __shared__ __align__(16) double ssm[];
    const int h = blockIdx.y;
    if (done && done[h]) return;
    double *Cs = ssm;                    // K x dh
    float *Xs = (float *)(Cs + K * dh);  // dh x (AS_T + 1)
    const int tid = threadIdx.x;
    const int64_t p0 = (int64_t)blockIdx.x * AS_T;
    const float *Ch = C + (int64_t)h * K * dh;
    for (int i = tid; i < K * dh; i += AS_T) Cs[i] = (double)Ch[i];
    const int np = (int)(n - p0 < AS_T ? n - p0 : AS_T);
    // half h's dims (hoff: [hoff[h], hoff[h+1]), R18), zero beyond its width up to dh: the
    // zero terms of the centroids' padded rows add exact zeros to each dist64 chain
    const int64_t ho = hoff ? hoff[h] : (int64_t)h * dh;
    const int hw = hoff ? hoff[h + 1] - hoff[h] : dh;
    for (int i = tid; i < np * dh; i += AS_T) {
        const int pt = i / dh, d = i - pt * dh;
        Xs[d * (AS_T + 1) + pt] = d < hw ? P[(p0 + pt) * ldp + ho + d] : 0.0f;
    }
    __syncthreads();
    if (tid >= np) return;
    double bd = 0.0;
    int best = 0;
    for (int c = 0; c < K; c += 2) {
        const double *c0 = Cs + c * dh, *c1 = c0 + dh;
        const bool two = c + 1 < K;
        double s0 = 0.0, s1 = 0.0;
        for (int d = 0; d < dh; d++) {
            const double xd = (double)Xs[d * (AS_T + 1) + tid];
            const double t0 = __dsub_rn(xd, c0[d]);
            s0 = __fma_rn(t0, t0, s0);
            if (two) {
                const double t1 = __dsub_rn(xd, c1[d]);
                s1 = __fma_rn(t1, t1, s1);
            }
        }
        if (c == 0 || s0 < bd) {
            bd = s0;
            best = c;
        }
        if (two && s1 < bd) {
            bd = s1;
            best = c + 1;
        }
    }
    a[(int64_t)h * n + p0 + tid] = best;
    if (dmin) dmin[(int64_t)h * n + p0 + tid] = bd;
}
__global__ void k_cells_from_halves(const int32_t *__restrict__ ah, int64_t N, int M, int K, int32_t *__restrict__ cells) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // e = m*N + p
    if (e >= N * M) return;
    const int64_t m = e / N, p = e - m * N;
    cells[e] = ah[(2 * m) * N + p] * K + ah[(2 * m + 1) * N + p];
}
static int argmin_smem(int K, int dh) { return K * dh * 8 + dh * (AS_T + 1) * 4; }
static void argmin_staged(const float *P, int64_t n, int64_t ldp, int dh, int K, int nh, const float *C,
                          const int *done, int32_t *a, double *dmin, cudaStream_t s,
                          const int32_t *hoff = nullptr) {
    const int sm = argmin_smem(K, dh);
    static int attr = 0;
    if (sm > attr) {
        CRISP_CUDA(cudaFuncSetAttribute(k_argmin_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        attr = sm;
    }
    dim3 g((unsigned)((n + AS_T - 1) / AS_T), (unsigned)nh);
    k_argmin_staged<<<g, AS_T, sm, s>>>(P, n, ldp, dh, K, C, done, a, dmin, hoff);
    CRISP_LAUNCH();
}
__global__ void k_km_compare(int64_t n, int nh, const int32_t *a, const int32_t *aold, const int *done, int *diff) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * nh) return;
    int h = (int)(e / n);
    if (!done[h] && a[e] != aold[e]) diff[h] = 1;
}
__global__ void k_km_converge(int nh, int it, const int *diff, int *done, int *active) {
    int h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= nh) return;
    if (!done[h] && it > 0 && diff[h] == 0) done[h] = 1;  // no assignment changed: stop
    active[h] = !done[h];
}
// thread per (h, c, t): mean over members in ascending point order
// k-means update: the members of each (h, c) listed in ascending point
// order (a stable radix sort of (h K + a, p)): a thread per (h, c, t) sums only
// its members in ascending p (the oracle's order)
__global__ void k_km_keys(int64_t n, int nh, int K, const int32_t *a, int32_t *key, int32_t *val) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * nh) return;
    const int h = (int)(e / n);
    key[e] = h * K + a[e];
    val[e] = (int32_t)(e - (int64_t)h * n);
}
__global__ void k_km_bins(const int32_t *skey, int64_t tot, int nb, int64_t *off) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;  // lower bound of bin b, b <= nb
    if (b > nb) return;
    int64_t lo = 0, hi = tot;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (skey[mid] < b) lo = mid + 1;
        else hi = mid;
    }
    off[b] = lo;
}
__global__ void k_km_update_sorted(const float *S, int Dp, int dh, int K, int nh, const int32_t *pts,
                                   const int64_t *off, const int *active, float *C, int64_t *cnt) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)nh * K * dh) return;
    const int t = (int)(e % dh);
    const int c = (int)((e / dh) % K);
    const int h = (int)(e / ((int64_t)dh * K));
    if (!active[h]) return;
    const int64_t j0 = off[(int64_t)h * K + c], j1 = off[(int64_t)h * K + c + 1];
    const float *col = S + (int64_t)h * dh + t;
    double sum = 0.0;
    int64_t j = j0;
    for (; j + 8 <= j1; j += 8) {  // eight loads ahead of their adds
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) v[u] = col[(int64_t)pts[j + u] * Dp];
#pragma unroll
        for (int u = 0; u < 8; u++) sum = __dadd_rn(sum, (double)v[u]);
    }
    for (; j < j1; j++) sum = __dadd_rn(sum, (double)col[(int64_t)pts[j] * Dp]);
    const int64_t k = j1 - j0;
    if (k > 0) C[((int64_t)h * K + c) * dh + t] = (float)(sum / (double)k);
    if (t == 0) cnt[(int64_t)h * K + c] = k;
}
// empty clusters, ascending c: farthest untaken point (by its assignment distance)
__global__ void k_km_reseed(const float *S, int64_t n, int Dp, int dh, int K, int nh, const int *active,
                            const int64_t *cnt, const double *dmin, unsigned char *taken, float *C) {
    int h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= nh || !active[h]) return;
    bool any = false;
    for (int c = 0; c < K; c++) any |= (cnt[(int64_t)h * K + c] == 0);
    if (!any) return;
    unsigned char *tk = taken + (int64_t)h * n;
    const double *dm = dmin + (int64_t)h * n;
    for (int64_t p = 0; p < n; p++) tk[p] = 0;
    for (int c = 0; c < K; c++) {
        if (cnt[(int64_t)h * K + c] != 0) continue;
        int64_t best = -1;
        double bd = -1.0;
        for (int64_t p = 0; p < n; p++)
            if (!tk[p] && dm[p] > bd) {
                bd = dm[p];
                best = p;
            }
        if (best < 0) best = 0;
        tk[best] = 1;
        for (int t = 0; t < dh; t++) C[((int64_t)h * K + c) * dh + t] = S[best * Dp + (int64_t)h * dh + t];
    }
}
__global__ void k_km_copy(int64_t n, int nh, const int *active, const int32_t *a, int32_t *aold) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * nh) return;
    if (active[e / n]) aold[e] = a[e];
}

// the k-means sample of an adaptive split (R18): row r holds half h's dims in [h dh, h dh + w_h),
// zeros after, so every k-means kernel runs on equal dh-wide halves (zero dims add exact zeros)
__global__ void k_gather_halves(const float *__restrict__ X, int64_t ld, const int32_t *__restrict__ rows, int64_t n,
                                const int32_t *__restrict__ hoff, int nh, int dh, float *__restrict__ S) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t rw = (int64_t)nh * dh;
    if (e >= n * rw) return;
    const int64_t r = e / rw;
    const int c = (int)(e - r * rw), h = c / dh, t = c - h * dh;
    S[e] = t < hoff[h + 1] - hoff[h] ? X[(int64_t)rows[r] * ld + hoff[h] + t] : 0.0f;
}

static void train_codebooks(crisp_index *ix, int64_t kmeans_sample, int iters, uint64_t seed, cudaStream_t s) {
    const int64_t N = ix->N;
    const int dh = ix->dh, K = ix->K, nh = 2 * ix->M;
    const int Dp = ix->hoff ? nh * dh : ix->Dp;  // sample row width
    int64_t n = std::min<int64_t>(N, std::max<int64_t>(1, kmeans_sample));
    Scratch sc;
    int32_t *rows = sc.alloc<int32_t>(n);
    sample_or_all(N, n, seed, STREAM_KM_SAMPLE, rows, s);
    float *S = sc.alloc<float>((size_t)n * Dp);
    // gather with pitch Dp (the padded dims of X are zero)
    {
        struct G {
        };
        if (ix->hoff)
            k_gather_halves<<<nblk(n * Dp, 256), 256, 0, s>>>(ix->X, ix->pitch, rows, n, ix->hoff, nh, dh, S);
        else
            k_gather_rows<<<nblk(n * Dp, 256), 256, 0, s>>>(ix->X, ix->pitch, rows, n, Dp, S);
        CRISP_LAUNCH();
    }
    float *C = ix->cb;
    double *D2 = sc.alloc<double>((size_t)n * nh);
    k_kpp_first<<<nblk(nh, 64), 64, 0, s>>>(S, n, Dp, dh, K, nh, seed, C);
    CRISP_LAUNCH();
    k_kpp_d2<<<nblk(n * nh, 256), 256, 0, s>>>(S, n, Dp, dh, K, nh, C, 0, D2);
    CRISP_LAUNCH();
    for (int c = 1; c < K; c++) {
        if (getenv("CRISP_KPP_SEQ")) k_kpp_pick<<<nh, 256, 0, s>>>(S, n, Dp, dh, K, nh, seed, c, D2, C);
        else k_kpp_pick_par<<<nh, KPP_T, 0, s>>>(S, n, Dp, dh, K, seed, c, D2, C);
        CRISP_LAUNCH();
        k_kpp_d2<<<nblk(n * nh, 256), 256, 0, s>>>(S, n, Dp, dh, K, nh, C, c, D2);
        CRISP_LAUNCH();
    }
    int32_t *a = sc.alloc<int32_t>((size_t)n * nh), *aold = sc.alloc<int32_t>((size_t)n * nh);
    double *dmin = sc.alloc<double>((size_t)n * nh);
    int *done = sc.alloc<int>(nh), *diff = sc.alloc<int>(nh), *active = sc.alloc<int>(nh);
    int64_t *cnt = sc.alloc<int64_t>((size_t)nh * K);
    unsigned char *taken = sc.alloc<unsigned char>((size_t)n * nh);
    CRISP_CUDA(cudaMemsetAsync(done, 0, nh * 4, s));
    // member lists for the update: keys h K + a, values p, stably sorted
    const int64_t tot = n * nh;
    int32_t *key = sc.alloc<int32_t>(tot), *val = sc.alloc<int32_t>(tot), *skey = sc.alloc<int32_t>(tot),
            *sval = sc.alloc<int32_t>(tot);
    int64_t *boff = sc.alloc<int64_t>((size_t)nh * K + 1);
    int kbits = 1;
    while ((1LL << kbits) < (long long)nh * K) kbits++;
    size_t stb = 0;
    CRISP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, stb, key, skey, val, sval, (int)tot, 0, kbits, s));
    void *stmp = sc.get(stb);
    for (int it = 0; it < iters; it++) {
        argmin_staged(S, n, Dp, dh, K, nh, C, done, a, dmin, s);
        CRISP_CUDA(cudaMemsetAsync(diff, 0, nh * 4, s));
        if (it > 0) {
            k_km_compare<<<nblk(n * nh, 256), 256, 0, s>>>(n, nh, a, aold, done, diff);
            CRISP_LAUNCH();
        }
        k_km_converge<<<nblk(nh, 64), 64, 0, s>>>(nh, it, diff, done, active);
        CRISP_LAUNCH();
        k_km_keys<<<nblk(tot, 256), 256, 0, s>>>(n, nh, K, a, key, val);
        CRISP_LAUNCH();
        CRISP_CUDA(cub::DeviceRadixSort::SortPairs(stmp, stb, key, skey, val, sval, (int)tot, 0, kbits, s));
        k_km_bins<<<nblk((int64_t)nh * K + 1, 256), 256, 0, s>>>(skey, tot, nh * K, boff);
        CRISP_LAUNCH();
        k_km_update_sorted<<<nblk((int64_t)nh * K * dh, 128), 128, 0, s>>>(S, Dp, dh, K, nh, sval, boff, active, C,
                                                                            cnt);
        CRISP_LAUNCH();
        k_km_reseed<<<nblk(nh, 32), 32, 0, s>>>(S, n, Dp, dh, K, nh, active, cnt, dmin, taken, C);
        CRISP_LAUNCH();
        k_km_copy<<<nblk(n * nh, 256), 256, 0, s>>>(n, nh, active, a, aold);
        CRISP_LAUNCH();
    }
    CRISP_CUDA(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------------------
// cell assignment, CSR, codes
// ---------------------------------------------------------------------------
__global__ void k_iota(int32_t *v, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (int32_t)i;
}
__global__ void k_hist2(const int32_t *cells, int64_t N, int M, int KK, int BS, int NB, int32_t *cnt) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= N * M) return;
    int m = (int)(e / N);
    int64_t p = e % N;
    int c = cells[e];
    atomicAdd(&cnt[((int64_t)m * KK + c) * NB + p / BS], 1);
}
// off2[(m*KK+c)*(NB+1)+b] from the per-m exclusive scan over (c, b)
__global__ void k_off2(const int32_t *scan, int64_t N, int M, int KK, int NB, int32_t *off2, int32_t *gsize) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // over M*KK*(NB+1)
    if (e >= (int64_t)M * KK * (NB + 1)) return;
    int b = (int)(e % (NB + 1));
    int64_t mc = e / (NB + 1);
    int m = (int)(mc / KK), c = (int)(mc % KK);
    int32_t v;
    if (b < NB) v = scan[mc * NB + b];
    else v = (c + 1 < KK) ? scan[(mc + 1) * NB] : (int32_t)N;
    off2[e] = v;
    if (b == NB) gsize[mc] = v - scan[mc * NB];
    (void)m;
}
__global__ void k_codes(const float *X, int64_t N, int64_t pitch, int Dp, int W, uint32_t *codes32) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // over N * W*64
    int64_t span = (int64_t)W * 64;
    bool bit = false;
    int64_t p = e / span;
    int i = (int)(e % span);
    if (e < N * span) bit = (i < Dp) && (X[p * pitch + i] > 0.0f);
    unsigned v = __ballot_sync(0xffffffffu, bit);
    if (e < N * span && (threadIdx.x & 31) == 0) codes32[p * (2 * W) + i / 32] = v;
}

void finish_csr(crisp_index *ix, cudaStream_t s) {
    const int64_t N = ix->N;
    const int M = ix->M, KK = ix->K * ix->K, NB = ix->NB, BS = ix->BS;
    Scratch sc;
    int32_t *iota = sc.alloc<int32_t>(N), *kout = sc.alloc<int32_t>(N);
    k_iota<<<nblk(N, 256), 256, 0, s>>>(iota, N);
    CRISP_LAUNCH();
    int bits = 1;
    while ((1 << bits) < KK) bits++;
    size_t tb = 0;
    CRISP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, ix->cells, kout, iota, ix->ids, (int)N, 0, bits, s));
    void *tmp = sc.get(tb);
    for (int m = 0; m < M; m++) {
        // stable: ids ascending inside a cell (Z18)
        CRISP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, ix->cells + (int64_t)m * N, kout, iota,
                                                   ix->ids + (int64_t)m * N, (int)N, 0, bits, s));
    }
    // block offsets (off2, BS ids) and warp sub-block offsets (off2w, SBW ids)
    for (int level = 0; level < 2; level++) {
        const int nb = level == 0 ? NB : ix->NBW, bs = level == 0 ? BS : ix->SBW;
        int32_t *dst = level == 0 ? ix->off2 : ix->off2w;
        const int64_t ne = (int64_t)KK * nb;
        int32_t *cnt = sc.alloc<int32_t>((size_t)M * ne), *scan = sc.alloc<int32_t>((size_t)M * ne);
        CRISP_CUDA(cudaMemsetAsync(cnt, 0, (size_t)M * ne * 4, s));
        k_hist2<<<nblk(N * M, 256), 256, 0, s>>>(ix->cells, N, M, KK, bs, nb, cnt);
        CRISP_LAUNCH();
        size_t tb2 = 0;
        CRISP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, cnt, scan, (int)ne, s));
        void *tmp2 = sc.get(tb2);
        for (int m = 0; m < M; m++)
            CRISP_CUDA(
                cub::DeviceScan::ExclusiveSum(tmp2, tb2, cnt + (int64_t)m * ne, scan + (int64_t)m * ne, (int)ne, s));
        k_off2<<<nblk((int64_t)M * KK * (nb + 1), 256), 256, 0, s>>>(scan, N, M, KK, nb, dst, ix->gsize);
        CRISP_LAUNCH();
    }
    {
        std::vector<int32_t> h((size_t)M * KK);
        CRISP_CUDA(cudaMemcpyAsync(h.data(), ix->gsize, h.size() * 4, cudaMemcpyDeviceToHost, s));
        CRISP_CUDA(cudaStreamSynchronize(s));
        ix->slice_hint = slice_hint_of(h.data(), M, KK, ix->N_global, ix->SBW);
        cell_size_maxima(ix, h.data());
    }
    CRISP_CUDA(cudaStreamSynchronize(s));
}

void cell_size_maxima(crisp_index *ix, const int32_t *sizes) {
    const int64_t KK = (int64_t)ix->K * ix->K;
    int64_t tot = 0;
    for (int m = 0; m < ix->M; m++) {
        int32_t mx = 0;
        for (int64_t c = 0; c < KK; c++) mx = std::max(mx, sizes[m * KK + c]);
        tot += mx;
    }
    ix->maxcell_sum = tot;
}

double slice_hint_of(const int32_t *sizes, int M, int64_t KK, int64_t N_global, int SBW) {
    double acc = 0.0;
    for (int m = 0; m < M; m++)
        for (int64_t c = 0; c < KK; c++) acc += (double)sizes[m * KK + c] * (double)sizes[m * KK + c];
    const double es = acc / ((double)M * (double)std::max<int64_t>(1, N_global));
    return es * (double)SBW / (double)std::max<int64_t>(1, N_global);
}

__global__ void k_check_finite(const float *X, int64_t N, int64_t pitch, int D, int *bad) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= N * D) return;
    float v = X[(e / D) * pitch + e % D];
    if (!isfinite(v)) *bad = 1;
}

// ---------------------------------------------------------------------------
// Block-wise variance redistribution (reading R16): R = I except on the dimensions
// of the rot_block subspaces of largest variance energy E_m (the sum of their 2 d_h
// per-dimension sample variances, ascending dimension, fp64; ties to the smaller m), where
// it is the rotation of P:L225 of that size (Q of QR of a Philox Gaussian, seed)
static void make_block_rotation(crisp_index *ix, const std::vector<double> &var, uint64_t seed, cudaStream_t s) {
    const int Dp = ix->Dp, M = ix->M, w = Dp / M, b = std::min(ix->rot_block, M);
    std::vector<double> E(M, 0.0);
    for (int m = 0; m < M; m++) {
        double e = 0.0;
        for (int i = m * w; i < (m + 1) * w; i++) e += i < (int)var.size() ? var[i] : 0.0;
        E[m] = e;
    }
    std::vector<int> order(M);
    for (int m = 0; m < M; m++) order[m] = m;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return E[x] > E[y]; });
    std::vector<int> top(order.begin(), order.begin() + b);
    std::sort(top.begin(), top.end());
    std::vector<int> blk;
    for (int m : top)
        for (int i = m * w; i < (m + 1) * w; i++) blk.push_back(i);
    const int ds = (int)blk.size();
    Scratch sc;
    float *Rs = sc.alloc<float>((size_t)ds * ds);
    make_rotation(ds, seed, Rs, s);
    std::vector<float> hs((size_t)ds * ds), hR((size_t)Dp * Dp, 0.0f);
    CRISP_CUDA(cudaMemcpyAsync(hs.data(), Rs, hs.size() * 4, cudaMemcpyDeviceToHost, s));
    CRISP_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < Dp; i++) hR[(size_t)i * Dp + i] = 1.0f;
    for (int i = 0; i < ds; i++)
        for (int j = 0; j < ds; j++) hR[(size_t)blk[i] * Dp + blk[j]] = hs[(size_t)i * ds + j];
    CRISP_CUDA(cudaMemcpyAsync(ix->R, hR.data(), hR.size() * 4, cudaMemcpyHostToDevice, s));
    CRISP_CUDA(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------------------
// Adaptive subspace decomposition (reading R18).  With S(e) the sum of the
// per-dimension variances v_i for i < e (ascending, fp64) and T = S(Dp), cut j (1 <= j < M)
// is the smallest even e in [c_{j-1} + 2, Dp - 2 (M - j)] with S(e) >= T j / M, else the
// upper end; the widths c_j - c_{j-1} put few dimensions where the variance is high.
std::vector<int32_t> adaptive_widths(const std::vector<double> &var, int M, int Dp) {
    std::vector<double> S((size_t)Dp + 1, 0.0);
    for (int i = 0; i < Dp; i++) S[i + 1] = S[i] + (i < (int)var.size() ? var[i] : 0.0);
    const double T = S[Dp];
    std::vector<int32_t> w;
    int prev = 0;
    for (int j = 1; j < M; j++) {
        const int hi = Dp - 2 * (M - j);
        const double target = (T * j) / M;
        int e = prev + 2;
        while (e < hi && S[e] < target) e += 2;
        w.push_back(e - prev);
        prev = e;
    }
    w.push_back(Dp - prev);
    return w;
}

void set_subspace_widths(crisp_index *ix, const int32_t *widths) {
    const int M = ix->M;
    int64_t sum = 0;
    int wmax = 0;
    bool equal = true;
    for (int m = 0; m < M; m++) {
        CRISP_CHECK(widths[m] >= 2 && widths[m] % 2 == 0, "subspace widths must be even and >= 2");
        sum += widths[m];
        wmax = std::max(wmax, (int)widths[m]);
        equal = equal && widths[m] == widths[0];
    }
    CRISP_CHECK(sum == ix->Dp, "subspace widths must sum to padded_D");
    cudaFree(ix->hoff);
    ix->hoff = nullptr;
    ix->hoff_h.clear();
    if (equal) return;  // the equal split: dh = Dp / 2M as set
    ix->hoff_h.resize((size_t)2 * M + 1);
    int o = 0;
    for (int m = 0; m < M; m++) {
        ix->hoff_h[2 * m] = o;
        ix->hoff_h[2 * m + 1] = o + widths[m] / 2;
        o += widths[m];
    }
    ix->hoff_h[2 * M] = o;
    ix->dh = wmax / 2;
    CRISP_CUDA(cudaMalloc(&ix->hoff, ix->hoff_h.size() * 4));
    CRISP_CUDA(cudaMemcpy(ix->hoff, ix->hoff_h.data(), ix->hoff_h.size() * 4, cudaMemcpyHostToDevice));
    ix->hbm_bytes += (int64_t)ix->hoff_h.size() * 4;
}

void build_index(crisp_index *ix, const float *data_dev, const float *R_inj, const float *cb_inj,
                 int64_t kmeans_sample, int32_t kmeans_iters, int32_t rotation_mode, float tau_cev, uint64_t seed,
                 cudaStream_t s, const double *cev_given, const std::vector<double> *var_given) {
    const int64_t N = ix->N;
    // X <- data, zero padded to pitch
    CRISP_CUDA(cudaMemsetAsync(ix->X, 0, (size_t)N * ix->pitch * 4, s));
    CRISP_CUDA(cudaMemcpy2DAsync(ix->X, (size_t)ix->pitch * 4, data_dev, (size_t)ix->D * 4, (size_t)ix->D * 4, N,
                                 cudaMemcpyDeviceToDevice, s));
    {
        Scratch sc;
        int *bad = sc.alloc<int>(1);
        CRISP_CUDA(cudaMemsetAsync(bad, 0, 4, s));
        k_check_finite<<<nblk(N * ix->D, 256), 256, 0, s>>>(ix->X, N, ix->pitch, ix->D, bad);
        CRISP_LAUNCH();
        int hb = 0;
        CRISP_CUDA(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, s));
        CRISP_CUDA(cudaStreamSynchronize(s));
        CRISP_CHECK(hb == 0, "data contains non-finite values");
    }
    // spectral check on the original D columns; a model build over a
    // gathered sample (build_model) supplies the global sample's CEV instead
    std::vector<double> var;
    if (cev_given) {
        ix->cev = *cev_given;
        if (var_given) var = *var_given;
    } else {
        ix->cev = compute_cev(ix->X, N, ix->pitch, ix->D, seed, s, &var);
    }
    bool rotate;
    if (R_inj) rotate = true;
    else if (cb_inj) rotate = false;  // injected build without R: no rotation
    else rotate = rotation_mode < 0 ? (ix->cev > (double)tau_cev) : (rotation_mode != 0);  // strict >
    if (rotate) {
        CRISP_CUDA(cudaMalloc(&ix->R, (size_t)ix->Dp * ix->Dp * 4));
        ix->hbm_bytes += (int64_t)ix->Dp * ix->Dp * 4;
        if (R_inj)
            CRISP_CUDA(cudaMemcpyAsync(ix->R, R_inj, (size_t)ix->Dp * ix->Dp * 4, cudaMemcpyDefault, s));
        else if (ix->rot_block > 0)
            make_block_rotation(ix, var, seed, s);
        else
            make_rotation(ix->Dp, seed, ix->R, s);
        rotate_in_place(ix, s);
        ix->rotated = 1;
    }
    if (ix->adaptive_req) {
        // R18: widths from the per-dimension variances of the stored vectors on the CEV sample
        // (those of X when not rotated, zero on the padding; else recomputed on X')
        std::vector<double> v2;
        if (ix->rotated) compute_cev(ix->X, N, ix->pitch, ix->Dp, seed, s, &v2);
        const std::vector<int32_t> w = adaptive_widths(ix->rotated ? v2 : var, ix->M, ix->Dp);
        set_subspace_widths(ix, w.data());
        ix->adaptive_req = 0;
        ix->cb = (float *)nullptr;
        CRISP_CUDA(cudaMalloc(&ix->cb, (size_t)ix->M * 2 * ix->K * ix->dh * 4));
        ix->hbm_bytes += (int64_t)ix->M * 2 * ix->K * ix->dh * 4;
    }
    if (cb_inj) {
        CRISP_CUDA(cudaMemcpyAsync(ix->cb, cb_inj, (size_t)ix->M * 2 * ix->K * ix->dh * 4, cudaMemcpyDefault, s));
    } else {
        train_codebooks(ix, kmeans_sample, kmeans_iters, seed, s);
    }
    {
        int32_t *ah = nullptr;  // per half-subspace argmin, then cells = i K + j
        CRISP_CUDA(cudaMallocAsync(&ah, (size_t)N * 2 * ix->M * 4, s));
        argmin_staged(ix->X, N, ix->pitch, ix->dh, ix->K, 2 * ix->M, ix->cb, nullptr, ah, nullptr, s, ix->hoff);
        k_cells_from_halves<<<nblk(N * ix->M, 256), 256, 0, s>>>(ah, N, ix->M, ix->K, ix->cells);
        CRISP_LAUNCH();
        CRISP_CUDA(cudaFreeAsync(ah, s));
    }
    CRISP_LAUNCH();
    finish_csr(ix, s);
    k_codes<<<nblk(N * (int64_t)ix->Wp * 64, 256), 256, 0, s>>>(ix->X, N, ix->pitch, ix->Dp, ix->Wp,
                                                                  (uint32_t *)ix->codes);
    CRISP_LAUNCH();
    if (ix->vfilter) build_verify_filter(ix, s);
    CRISP_CUDA(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------------------
// Verification filter (DESIGN R17).  mu = column means (fp64 sums in a fixed
// order, rounded to fp32); per row, y = x - mu (fp64, exact up to 2^-53
// relative), e with max |y_i| < 2^(e+7), c_i = clamp(rint(y_i 2^-e), +-127),
// the integer c.c, and rho = ||y - 2^e c|| (fp64 sum, rounded up with a 1e-9
// relative and a 1e-15 ||y|| absolute margin).  The search bounds
// ||q' - x|| from these (search.cu, filt_bounds) and reads the fp32 row only
// when the bound cannot exclude it.
// ---------------------------------------------------------------------------
constexpr int MU_CHUNKS = 512;
__global__ void k_mu_partial(const float *__restrict__ X, int64_t N, int pitch, double *__restrict__ part) {
    // block (32 columns x 8 row lanes), chunk blockIdx.y of the rows
    const int col = blockIdx.x * 32 + (threadIdx.x & 31), rl = threadIdx.x >> 5;
    const int64_t r0 = N * blockIdx.y / MU_CHUNKS, r1 = N * (blockIdx.y + 1) / MU_CHUNKS;
    __shared__ double sh[8][32];
    double a = 0.0;
    if (col < pitch)
        for (int64_t r = r0 + rl; r < r1; r += 8) a += (double)X[r * pitch + col];
    sh[rl][threadIdx.x & 31] = a;
    __syncthreads();
    if (rl == 0 && col < pitch) {
        double t = 0.0;
        for (int i = 0; i < 8; i++) t += sh[i][threadIdx.x & 31];
        part[(int64_t)blockIdx.y * pitch + col] = t;
    }
}
__global__ void k_mu_final(const double *__restrict__ part, int pitch, int64_t N, float *__restrict__ mu) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= pitch) return;
    double t = 0.0;
    for (int c = 0; c < MU_CHUNKS; c++) t += part[(int64_t)c * pitch + col];
    mu[col] = (float)(t / (double)N);
}

__global__ void k_int8_copy(const float *__restrict__ X, int64_t N, int pitch, int c8pitch,
                            const float *__restrict__ mu, int8_t *__restrict__ C8, int4 *__restrict__ meta) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= N) return;
    const float *x = X + row * pitch;
    double m = 0.0, n2 = 0.0;
    for (int i = lane; i < pitch; i += 32) {
        const double y = (double)x[i] - (double)mu[i];
        m = fmax(m, fabs(y));
        n2 = fma(y, y, n2);
    }
    for (int o = 16; o; o >>= 1) {
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        n2 += __shfl_xor_sync(0xffffffffu, n2, o);
    }
    int e = 0;
    if (m > 0.0) {
        frexp(m, &e);  // m < 2^e
        e -= 7;        // |y_i 2^-e| < 128
    }
    const double up = ldexp(1.0, -e), dn = ldexp(1.0, e);
    int8_t *c = C8 + row * c8pitch;
    double r2 = 0.0;
    int cc = 0;
    for (int i = lane; i < c8pitch; i += 32) {
        const double y = i < pitch ? (double)x[i] - (double)mu[i] : 0.0;
        const double v = fmin(127.0, fmax(-127.0, rint(y * up)));
        c[i] = (int8_t)v;
        cc += (int)v * (int)v;
        const double r = y - v * dn;
        r2 = fma(r, r, r2);
    }
    for (int o = 16; o; o >>= 1) {
        r2 += __shfl_xor_sync(0xffffffffu, r2, o);
        cc += __shfl_xor_sync(0xffffffffu, cc, o);
    }
    if (lane == 0) {
        const float rho = __double2float_ru(sqrt(r2) * (1.0 + 1e-9) + 1e-15 * sqrt(n2));
        meta[row] = make_int4(cc, e, __float_as_int(rho), 0);
    }
}

void build_verify_filter(crisp_index *ix, cudaStream_t s) {
    const int64_t N = ix->N;
    const int pitch = ix->pitch;
    ix->c8pitch = (pitch + 15) / 16 * 16;
    if (!ix->C8) {
        CRISP_CUDA(cudaMalloc(&ix->C8, (size_t)N * ix->c8pitch + 64));
        CRISP_CUDA(cudaMalloc(&ix->c8meta, (size_t)N * 16 + 16));
        CRISP_CUDA(cudaMalloc(&ix->mu, (size_t)pitch * 4 + 16));
        ix->hbm_bytes += N * (int64_t)ix->c8pitch + N * 16 + (int64_t)pitch * 4;
    }
    Scratch sc;
    double *part = sc.alloc<double>((size_t)MU_CHUNKS * pitch);
    k_mu_partial<<<dim3(nblk(pitch, 32), MU_CHUNKS), 256, 0, s>>>(ix->X, N, pitch, part);
    CRISP_LAUNCH();
    k_mu_final<<<nblk(pitch, 128), 128, 0, s>>>(part, pitch, N, ix->mu);
    CRISP_LAUNCH();
    k_int8_copy<<<nblk(N, 8), 256, 0, s>>>(ix->X, N, pitch, ix->c8pitch, ix->mu, ix->C8, (int4 *)ix->c8meta);
    CRISP_LAUNCH();
    CRISP_CUDA(cudaStreamSynchronize(s));  // the scratch is freed on return
}

}  // namespace crisp

namespace crisp {
double cev_of_sample(const float *S_dev, int64_t n, int D, cudaStream_t s, std::vector<double> *var) {
    return cev_of_rows(S_dev, n, D, s, var);
}
}  // namespace crisp
