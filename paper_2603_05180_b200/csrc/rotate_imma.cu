// rotate_imma.cu -- a0 (q' = fl32(q R)) on the int8 tensor cores,
// exact by certification.
//
// The oracle's q'_n is fl32(y_n), y_n the sequential fp64 chain
// s = fma(q_k, R_kn, s), k ascending from +0.  Here:
//  1. Each query row is scaled by 2^-e (|u_k| = |q_k| 2^-e < 1/4), rounded to
//     the fixed point U_k = rint(u_k 2^56) (|u_k - U_k 2^-56| <= 2^-57) and U_k
//     is written in S = 7 balanced base-256 digits, U_k 2^-56 = sum_s a_ks 2^-8s
//     (a in [-128, 127], integer arithmetic); each column n of R likewise with
//     2^-f_n, digits b_knt.
//  2. For every level l = 2..8 the exact int32 sum C_l[m][n] = sum_{s+t=l}
//     sum_k a_mks b_knt (|C_l| <= 7 Dp 2^14 < 2^31 for Dp < 18724) on the
//     int8 tensor cores: k_rot_tc (hand-written tcgen05, below) or, with
//     CRISP_ROTATE_GEMM=cublaslt, one cuBLASLt GEMM per level (the slices of a
//     level concatenated along k, K' = (l-1) Dp).
//  3. yhat = 2^(e+f_n) sum_l 2^-8l C_l (fp64, ascending l) differs from the
//     exact sum S of the products by at most 2^(e+f_n) (Dp 2^-53 + 2^-50
//     sum_l |2^-8l C_l|): the dropped digit pairs s+t > 8 (< 7 2^14 2^-72 per
//     term) and the fixed-point roundings (< 2^-58), together < 2^-54 per
//     term; the 7-term fp64 sum.  The oracle's y_n
//     differs from S by at most gamma_Dp ||q|| ||R_n|| (recursive summation,
//     exact products).  If [yhat - b, yhat + b] lies strictly inside the fp32
//     rounding cell of fl32(yhat), then fl32(y_n) = fl32(yhat): certified.
//     Otherwise (~0.02% of outputs at cfg2) k_recompute runs the sequential
//     chain for that output.
// The R slices, exponents and column norms are computed once per index.
#include <cublasLt.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>

#include "crisp_internal.cuh"
#include "tc_util.cuh"

namespace crisp {

namespace {

constexpr int SL = 7;  // slices (balanced base-256 digits) per operand
constexpr int LV = 8;  // levels 2..LV (slice pairs s + t <= LV)
constexpr int DB = 8;  // bits per digit

std::mutex g_mu;
cublasLtHandle_t g_lt = nullptr;
constexpr size_t WS_BYTES = 32u << 20;  // cuBLASLt workspace, allocated per call (stream-ordered)

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
    const int e = mx > 0.f ? ilogbf(mx) + 3 : 0;  // |x| 2^-e < 1/4: |U| < 2^54, the top digit in [-64, 64]
    if (lane == 0) {
        *e_out = e;
        *n2_out = sqrt(ss) * 1.01;
    }
    const double sc = pow2(56 - e);  // exact scaling
    for (int k4 = lane * 4; k4 < Dpk; k4 += 128) {
        // U = rint(x 2^(56-e)), |U| < 2^54; balanced base-256 digits, least significant
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
                const long long d = ((U[j] + 128) & 255) - 128;  // in [-128, 127]
                U[j] = (U[j] - d) >> DB;                          // exact
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

// The certificate of one output from its level sums c[l-2] = C_l (l = 2..LV):
// yhat = 2^(e_q + f_n) sum_l 2^-8l C_l and its bound b (see the top); returns
// fl32(yhat) and, if [yhat - b, yhat + b] is not strictly inside the fp32
// rounding cell of fl32(yhat), lists the output for k_recompute.
// uncertified outputs: total count, then per query row (up to RCAP columns per row; a row's
// list is recomputed by one warp sharing the row in shared memory), the rest in a flat list
constexpr int RCAP = 32;
struct FallLists {
    unsigned long long *nfall;  // [0] all uncertified outputs, [1] those in the flat list
    int64_t *flist;             // m Dp + n
    int32_t *rowcnt;            // rows
    int32_t *rowlist;           // rows x RCAP columns n
};
__device__ __forceinline__ float certify_one(const int32_t (&c)[LV - 1], int32_t e_q, double n_q, int32_t e_n,
                                             double n_n, int Dp, int64_t m, int n, const FallLists &fl) {
    double acc = 0.0, mag = 0.0;
#pragma unroll
    for (int l = LV; l >= 2; l--) {  // ascending magnitude; 2^-8l exact
        const double t = (double)c[l - 2] * pow2(-DB * l);
        acc += t;
        mag += fabs(t);
    }
    const double p2 = pow2(e_q + e_n);  // exact (|exponents| small)
    const double y = acc * p2;
    const double b = ((double)Dp * 0x1p-53 + mag * 0x1p-50) * p2 + (double)Dp * 0x1p-53 * 1.01 * n_q * n_n;
    const float f = (float)y;
    // neighbours of f (bit steps; f = 0 -> the smallest subnormals)
    const int fb = __float_as_int(f);
    const float fdn = f == 0.f ? -1.4e-45f : __int_as_float(f > 0.f ? fb - 1 : fb + 1);
    const float fup = f == 0.f ? 1.4e-45f : __int_as_float(f > 0.f ? fb + 1 : fb - 1);
    const double lo = 0.5 * ((double)f + (double)fdn);
    const double hi = 0.5 * ((double)f + (double)fup);
    if (!(y - b > lo && y + b < hi)) {  // k_recompute_rows / k_recompute
        atomicAdd(fl.nfall, 1ull);
        const int slot = atomicAdd(fl.rowcnt + m, 1);
        if (slot < RCAP) fl.rowlist[m * RCAP + slot] = n;
        else fl.flist[atomicAdd(fl.nfall + 1, 1ull)] = m * Dp + n;
    }
    return f;
}

__global__ void k_certify(const int32_t *__restrict__ C, int64_t rows, int Dp, int Dpk, const int32_t *__restrict__ qe,
                          const double *__restrict__ qn2, const int32_t *__restrict__ re,
                          const double *__restrict__ rn2, float *__restrict__ Y, int64_t ldy, FallLists fl) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t m = blockIdx.y;
    if (n >= Dp || m >= rows) return;
    const int64_t plane = rows * (int64_t)Dpk;
    int32_t c[LV - 1];
#pragma unroll
    for (int l = 2; l <= LV; l++) c[l - 2] = C[(int64_t)(l - 2) * plane + m * Dpk + n];
    Y[m * ldy + n] = certify_one(c, qe[m], qn2[m], re[n], rn2[n], Dp, m, n, fl);
}

// ---------------------------------------------------------------------------
// The level GEMMs and the certificate in one hand-written sm_100a kernel (the
// 5th-generation tensor cores: tcgen05.mma kind::i8 with int32 accumulators in
// tensor memory, operands staged by TMA).  A CTA owns a tile of 128 query rows x
// 64 columns n of R and keeps the seven level sums C_l (l = 2..8) of its tile in
// TMEM: level l at columns [64 (l-2), 64 (l-2) + 64) of a 512-column allocation
// (128 lanes = the tile's rows).  Per k-block of 128 it loads the seven query
// digit planes a_s (128 x 128 int8 each) and the seven R digit planes b_t (64 x
// 128 each) with TMA (128-byte swizzle, K-major), and one elected thread issues
// the 28 products a_s b_t^T with s + t <= 8 (4 MMAs of K = 32 each, M = 128,
// N = 64) into the accumulator of level s + t.  The epilogue warps read the
// seven levels of each output back (tcgen05.ld) and run the certificate of
// k_certify on them directly: C never goes to HBM.
// ---------------------------------------------------------------------------
namespace tc {

constexpr int BM = 128, BN = 64, BK = 128;                     // tile rows, columns, k-block (bytes)
constexpr int A_TILE = BM * BK, B_TILE = BN * BK;              // 16 KB, 8 KB
constexpr int NA = 4;                                          // A ring: digit-plane tiles in flight
constexpr int SMEM_TILES = 2 * SL * B_TILE + NA * A_TILE;      // B double-buffered (2 x 56 KB) + A ring (64 KB)
constexpr int THREADS_TC = 128;                                // warp 0: TMA, warp 1: MMA issue; all 4: epilogue

using tcu::mbar_expect_tx;
using tcu::mbar_init;
using tcu::mbar_wait;
using tcu::mma_commit;
using tcu::smem_u32;
using tcu::sw128_desc;
using tcu::tma_load_2d;
// instruction descriptor: s8 x s8 -> s32, K-major A and B, M = 128, N = 64
constexpr uint32_t IDESC = tcu::idesc(2u, 1u, BM, BN);
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
    tcu::mma<0>(d_tmem, a, b, IDESC, accumulate);
}

// Pipeline: per k-block the seven R planes b_1..b_7 go to one of two B buffers and
// the seven query planes a_1..a_7 stream through a ring of NA A tiles; the MMA
// thread consumes a_s with b_1..b_{8-s} (accumulating into levels s+1..8) and
// releases its ring slot (and, after a_7, the B buffer) with tcgen05.commit, so
// the TMA thread loads k-block kb+1 while the tensor cores work on kb.
__global__ void __launch_bounds__(THREADS_TC, 1)
    k_rot_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int64_t rows, int Dp,
             int Dpk, const int32_t *__restrict__ qe, const double *__restrict__ qn2, const int32_t *__restrict__ re,
             const double *__restrict__ rn2, float *__restrict__ Y, int64_t ldy, FallLists fl) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    // 1024-byte aligned (the 128-byte swizzle atoms), keeping the shared-memory provenance
    unsigned char *base = smraw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smraw) & 1023u)) & 1023u);
    unsigned char *Bs = base;                          // 2 x SL tiles of B_TILE
    unsigned char *As = base + 2 * SL * B_TILE;        // NA tiles of A_TILE
    __shared__ __align__(8) uint64_t fullB[2], emptyB[2], fullA[NA], emptyA[NA], done;
    __shared__ uint32_t tmem_base;
    __shared__ int32_t s_re[BN];
    __shared__ double s_rn2[BN];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t m0 = (int64_t)blockIdx.y * BM;
    const int n0 = blockIdx.x * BN;
    if (tid == 0) {
        for (int i = 0; i < 2; i++) {
            mbar_init(&fullB[i], 1);
            mbar_init(&emptyB[i], 1);
        }
        for (int i = 0; i < NA; i++) {
            mbar_init(&fullA[i], 1);
            mbar_init(&emptyA[i], 1);
        }
        mbar_init(&done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mapA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mapB) : "memory");
    }
    if (warp == 1) {  // the whole TMEM of the SM: 7 levels x 64 int32 columns (+64 unused; one CTA per SM)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    for (int i = tid; i < BN; i += THREADS_TC) {
        const int n = n0 + i;
        s_re[i] = n < Dp ? re[n] : 0;
        s_rn2[i] = n < Dp ? rn2[n] : 0.0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base;
    const int nkb = Dpk / BK;
    if (warp == 0 && lane == 0) {
        // TMA producer
        for (int kb = 0; kb < nkb; kb++) {
            const int bb = kb & 1;
            mbar_wait(&emptyB[bb], ((kb >> 1) & 1) ^ 1);
            mbar_expect_tx(&fullB[bb], (uint32_t)(SL * B_TILE));
            for (int t = 1; t <= SL; t++)  // R digit plane b_t (stored descending: plane SL - t of Rsl)
                tma_load_2d(Bs + (bb * SL + t - 1) * B_TILE, &mapB, (SL - t) * Dpk + kb * BK, n0, &fullB[bb]);
            for (int s = 1; s <= SL; s++) {
                const int i = kb * SL + s - 1, slot = i % NA;
                mbar_wait(&emptyA[slot], ((i / NA) & 1) ^ 1);
                mbar_expect_tx(&fullA[slot], (uint32_t)A_TILE);
                // query digit plane a_s: bytes [(s-1) Dpk + kb BK, +BK) of rows [m0, m0+BM)
                tma_load_2d(As + slot * A_TILE, &mapA, (s - 1) * Dpk + kb * BK, (int)m0, &fullA[slot]);
            }
        }
    } else if (warp == 1) {
        // MMA issuer (the whole warp waits; one elected lane issues): a_s b_t into the accumulator of level s + t (s + t <= LV).  The
        // descriptors are formed once per tile; the k-steps of 32 bytes advance the start
        // address field (16-byte units) by 2 (the 128-byte swizzle is a function of the
        // address bits, and tiles are 1024-byte aligned)
        const uint64_t dB0 = sw128_desc(smem_u32(Bs));
        const uint64_t dA0 = sw128_desc(smem_u32(As));
        for (int kb = 0; kb < nkb; kb++) {
            const int bb = kb & 1;
            mbar_wait(&fullB[bb], (kb >> 1) & 1);
            const uint64_t dBb = dB0 + (uint64_t)((bb * SL * B_TILE) >> 4);
            for (int s = 1; s <= SL; s++) {
                const int i = kb * SL + s - 1, slot = i % NA;
                mbar_wait(&fullA[slot], (i / NA) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint64_t da = dA0 + (uint64_t)((slot * A_TILE) >> 4);
                const uint32_t first = (kb == 0 && s == 1) ? 0u : 1u;  // the first product of a level overwrites
                for (int t = 1; s + t <= LV; t++) {
                    const uint32_t d = tmem + (uint32_t)(BN * (s + t - 2));
                    const uint64_t db = dBb + (uint64_t)(((t - 1) * B_TILE) >> 4);
                    mma_i8(d, da, db, first);
                    mma_i8(d, da + 2, db + 2, 1u);
                    mma_i8(d, da + 4, db + 4, 1u);
                    mma_i8(d, da + 6, db + 6, 1u);
                }
                mma_commit(&emptyA[slot]);  // the ring slot is free once these MMAs have read it
            }
            mma_commit(&emptyB[bb]);
        }
        mma_commit(&done);
    }
    __syncwarp();
    mbar_wait(&done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // epilogue: thread (warp w, lane) owns TMEM lane 32 w + lane = row m0 + 32 w + lane
    const int64_t m = m0 + warp * 32 + lane;
    const bool live = m < rows;
    const int32_t e_q = live ? qe[m] : 0;
    const double n_q = live ? qn2[m] : 0.0;
    const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c8 = 0; c8 < BN; c8 += 8) {
        uint32_t v[LV - 1][8];
#pragma unroll
        for (int l = 2; l <= LV; l++)
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                : "=r"(v[l - 2][0]), "=r"(v[l - 2][1]), "=r"(v[l - 2][2]), "=r"(v[l - 2][3]), "=r"(v[l - 2][4]),
                  "=r"(v[l - 2][5]), "=r"(v[l - 2][6]), "=r"(v[l - 2][7])
                : "r"(trow + (uint32_t)(BN * (l - 2) + c8)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (!live) continue;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int n = n0 + c8 + j;
            if (n >= Dp) continue;
            int32_t c[LV - 1];
#pragma unroll
            for (int l = 2; l <= LV; l++) c[l - 2] = (int32_t)v[l - 2][j];
            Y[m * ldy + n] = certify_one(c, e_q, n_q, s_re[c8 + j], s_rn2[c8 + j], Dp, m, n, fl);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

}  // namespace tc

// the uncertified outputs: the sequential chain itself, a thread per output,
// reading q' s row and R's column n (Rt: R transposed) as float4 streams with
// 32 terms in flight ahead of their fma's (per-row lists: k_recompute_rows;
// the flat overflow list: k_recompute)
// one output's chain from a query row (global or shared) and R's column n (Rt row n)
__device__ __forceinline__ double chain_one(const float *__restrict__ xr, const float *__restrict__ rr, int Dp,
                                            bool vec) {
    double s = 0.0;
    int k = 0;
    if (vec) {
        const float4 *x4 = (const float4 *)xr, *r4 = (const float4 *)rr;
        const int nv = Dp / 4;
        float4 xa[8], ra[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            xa[j] = j < nv ? x4[j] : make_float4(0.f, 0.f, 0.f, 0.f);
            ra[j] = j < nv ? __ldg(r4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        for (int v0 = 0; v0 < nv; v0 += 8) {
            float4 xb[8], rb[8];
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int v = v0 + 8 + j;
                xb[j] = v < nv ? x4[v] : make_float4(0.f, 0.f, 0.f, 0.f);
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
    return s;
}

// the per-row lists: a warp per query row, the row staged once in shared memory, a lane per
// listed output (the rows' X reads are no longer repeated per output; R's columns come
// from L2)
__global__ void __launch_bounds__(32) k_recompute_rows(const int32_t *__restrict__ rowcnt,
                                                       const int32_t *__restrict__ rowlist, int64_t rows, int Dp,
                                                       const float *__restrict__ X, int64_t ldx,
                                                       const float *__restrict__ Rt, float *__restrict__ Y,
                                                       int64_t ldy) {
    extern __shared__ __align__(16) float xs[];  // Dp
    const int64_t m = blockIdx.x;
    const int cnt = min(rowcnt[m], RCAP);
    if (cnt == 0) return;
    const int lane = threadIdx.x;
    const float *xr = X + m * ldx;
    for (int k = lane; k < Dp; k += 32) xs[k] = xr[k];
    __syncwarp();
    if (lane < cnt) {
        const int n = rowlist[m * RCAP + lane];
        Y[m * ldy + n] = (float)chain_one(xs, Rt + (int64_t)n * Dp, Dp, (Dp & 3) == 0);
    }
}

__global__ void __launch_bounds__(128) k_recompute(const unsigned long long *__restrict__ nfall,
                                                   const int64_t *__restrict__ flist, int Dp,
                                                   const float *__restrict__ X, int64_t ldx,
                                                   const float *__restrict__ Rt, float *__restrict__ Y,
                                                   int64_t ldy) {
    const int64_t nf = (int64_t)*nfall;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t mn = flist[i], m = mn / Dp;
        const int n = (int)(mn - m * Dp);
        Y[m * ldy + n] = (float)chain_one(X + m * ldx, Rt + (int64_t)n * Dp, Dp, ((ldx | Dp) & 3) == 0);
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

void ensure_lt() {
    if (!g_lt) CRISP_LT(cublasLtCreate(&g_lt));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        CRISP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) {
            set_error("cuTensorMapEncodeTiled unavailable");
            throw Err{CRISP_ECUDA};
        }
        fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

// 2-D uint8 tensor map over rows of `width` bytes (row stride = width), box (box_x bytes, box_y rows),
// 128-byte swizzle
CUtensorMap make_map_u8(const void *base, uint64_t width, uint64_t rows, uint32_t box_x, uint32_t box_y) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {width, rows};
    const cuuint64_t strides[1] = {width};
    const cuuint32_t box[2] = {box_x, box_y};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(base), dims, strides,
                                            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
        throw Err{CRISP_ECUDA};
    }
    return m;
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

// slice row length: D' rounded up to the tensor-core kernel's k-block (128) and
// n-tile (64); the padding digits are zero
int rotation_slices_k(int Dp) { return (Dp + 127) / 128 * 128; }

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
    // CRISP_ROTATE_GEMM=cublaslt: the level GEMMs as cuBLASLt int8 GEMMs + k_certify
    // (the earlier design, kept for comparison); default: k_rot_tc
    const bool use_lt = getenv("CRISP_ROTATE_GEMM") && std::string(getenv("CRISP_ROTATE_GEMM")) == "cublaslt";
    // scratch: Qcat (rows x SL Dpk int8) | C (LV-1 levels x rows x Dp int32) | qn2 | qe
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t qbytes = up((size_t)rows * SL * Dpk), cbytes = use_lt ? up((size_t)(LV - 1) * rows * Dpk * 4) : 0;
    char *buf = nullptr;
    CRISP_CUDA(cudaMallocAsync(&buf, qbytes + cbytes + up((size_t)rows * 8) + up((size_t)rows * 4), s));
    int8_t *Qcat = (int8_t *)buf;
    int32_t *C = (int32_t *)(buf + qbytes);
    double *qn2 = (double *)(buf + qbytes + cbytes);
    int32_t *qe = (int32_t *)(buf + qbytes + cbytes + up((size_t)rows * 8));
    k_slice_rows<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(X, rows, Dp, ldx, Dpk, Qcat, qe, qn2);
    CRISP_LAUNCH();
    // uncertified outputs: counters, per-row lists (RCAP columns) and the flat overflow list
    // (at most rows x Dp entries)
    unsigned long long *cnt = nullptr;
    const size_t fcap = (size_t)rows * Dp;
    const size_t lbytes = up(16) + up(fcap * 8) + up((size_t)rows * 4) + up((size_t)rows * RCAP * 4);
    CRISP_CUDA(cudaMallocAsync(&cnt, lbytes, s));
    FallLists fl;
    fl.nfall = cnt;
    fl.flist = (int64_t *)((char *)cnt + up(16));
    fl.rowcnt = (int32_t *)((char *)fl.flist + up(fcap * 8));
    fl.rowlist = fl.rowcnt + up((size_t)rows * 4) / 4;
    CRISP_CUDA(cudaMemsetAsync(cnt, 0, 16, s));
    CRISP_CUDA(cudaMemsetAsync(fl.rowcnt, 0, (size_t)rows * 4, s));
    if (use_lt) {
        std::lock_guard<std::mutex> lk(g_mu);
        ensure_lt();
        const Plan &p = plan_for(Dp, Dpk, rows);
        void *ws = nullptr;  // per call: concurrent searches on other streams never share it
        CRISP_CUDA(cudaMallocAsync(&ws, WS_BYTES, s));
        const int32_t alpha = 1, beta = 0;
        for (int l = 2; l <= LV; l++) {
            const int8_t *A = ix->Rsl + (size_t)(LV - l) * Dpk;  // [b_{l-1} .. b_1]
            int32_t *Cl = C + (size_t)(l - 2) * rows * Dpk;
            CRISP_LT(cublasLtMatmul(g_lt, p.op, &alpha, A, p.la[l], Qcat, p.lb[l], &beta, Cl, p.lc, Cl, p.lc,
                                    &p.algo[l], ws, WS_BYTES, s));
        }
        CRISP_CUDA(cudaFreeAsync(ws, s));
        dim3 g((Dp + 127) / 128, (unsigned)rows);
        k_certify<<<g, 128, 0, s>>>(C, rows, Dp, Dpk, qe, qn2, ix->Rexp, ix->Rn2, Y, ldy, fl);
        CRISP_LAUNCH();
    } else {
        static std::mutex amu;
        static std::map<int, bool> attr;  // per device
        const int smem = tc::SMEM_TILES + 1024;
        {
            std::lock_guard<std::mutex> lk(amu);
            if (!attr[ix->device]) {
                CRISP_CUDA(cudaFuncSetAttribute(tc::k_rot_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                attr[ix->device] = true;
            }
        }
        const CUtensorMap mA = make_map_u8(Qcat, (uint64_t)SL * Dpk, (uint64_t)rows, tc::BK, tc::BM);
        const CUtensorMap mB = make_map_u8(ix->Rsl, (uint64_t)SL * Dpk, (uint64_t)Dpk, tc::BK, tc::BN);
        dim3 g((unsigned)(Dpk / tc::BN), (unsigned)((rows + tc::BM - 1) / tc::BM));
        tc::k_rot_tc<<<g, tc::THREADS_TC, smem, s>>>(mA, mB, rows, Dp, Dpk, qe, qn2, ix->Rexp, ix->Rn2, Y, ldy, fl);
        CRISP_LAUNCH();
    }
    {
        const int xsm = Dp * 4;
        if (xsm > 48 * 1024) {
            static std::mutex rmu;
            std::lock_guard<std::mutex> lk(rmu);
            CRISP_CUDA(cudaFuncSetAttribute(k_recompute_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, xsm));
        }
        k_recompute_rows<<<(unsigned)rows, 32, xsm, s>>>(fl.rowcnt, fl.rowlist, rows, Dp, X, ldx, ix->Rt, Y, ldy);
        CRISP_LAUNCH();
    }
    k_recompute<<<148 * 8, 128, 0, s>>>(cnt + 1, fl.flist, Dp, X, ldx, ix->Rt, Y, ldy);
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
