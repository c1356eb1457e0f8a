// probe_tc.cu -- a1's query x centroid contraction on the tensor cores (the
// "dense query x centroid contraction" of the north star; Alg. 1 l.4):
// a certified SCREEN of the half distances, which k_probe then resolves exactly.
//
// For every half-subspace (m, h) and a tile of 128 queries, one tcgen05.mma
// chain (kind::tf32, M = 128 queries, N = 64 >= K centroids, fp32 accumulators
// in TMEM; operands staged by TMA with the 128-byte swizzle) forms the dot
// products <q'_{m,h}, C_{m,h,c}>.  The epilogue turns them into an interval
// [lo_c, hi_c] that provably contains dist64(q'_{m,h}, C_{m,h,c}) (App. A.1):
//   s~  = |q|^2 + |c|^2 - 2 dot~   (norms in fp64 from the fp32 inputs)
//   |dot~ - dot| <= (2^-9 + (dh + 2) 2^-23) |q| |c|   (tf32 inputs: relative
//        error <= 2^-10 each, even truncated; products exact in fp32; an
//        fp32 accumulation of dh terms, even truncating, <= dh 2^-23 sum|q_i c_i|)
//   |dist64 - exact| <= (dh + 4) 2^-52 (|q|^2 + |c|^2)   (recursive fp64 sum of
//        non-negative terms of exactly formed differences)
// lo/hi are rounded outward to fp32.  k_probe computes dist64 only for the
// centroids whose interval can reach the R smallest, and takes every ordering
// decision on those exact values (the tie orders (delta, c) and (cost, i, j) of
// App. A.2 are decided on dist64 values only).
#include "crisp_internal.cuh"
#include "tc_util.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>

namespace crisp {

namespace {

constexpr int SB_M = 128, SB_N = 64;  // queries per tile, centroids (K <= 64)
constexpr int SB_THREADS = 128;

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        CRISP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        CRISP_CHECK(q == cudaDriverEntryPointSuccess && p, "cuTensorMapEncodeTiled unavailable");
        fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

// 2-D fp32 map: rows of `width` floats at a stride of `stride` floats, box (32 floats, box_y rows)
CUtensorMap map_f32(const void *base, uint64_t width, uint64_t rows, uint64_t stride, uint32_t box_y) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {width, rows};
    const cuuint64_t strides[1] = {stride * 4};
    const cuuint32_t box[2] = {32, box_y};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(base), dims, strides, box,
                                 es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled (screen) failed: " + std::to_string((int)r));
        throw Err{CRISP_ECUDA};
    }
    return m;
}

// padded codebooks: row (2m+h)*64 + c holds C_{m,h,c} in its first dh floats, zeros
// elsewhere (c >= K rows and dims >= dh are zero: the over-read query dims of a
// k-block beyond dh contribute 0)
__global__ void k_pad_codebooks(const float *__restrict__ cb, int M, int K, int dh, int DHP,
                                float *__restrict__ cbp, double *__restrict__ cn2) {
    const int row = blockIdx.x, t = threadIdx.x;  // row = (2m+h)*64 + c
    const int hs = row / SB_N, c = row % SB_N;
    for (int j = t; j < DHP; j += blockDim.x)
        cbp[(int64_t)row * DHP + j] = (c < K && j < dh) ? cb[((int64_t)hs * K + c) * dh + j] : 0.0f;
    if (t == 0 && c < K) {
        double s = 0.0;
        for (int j = 0; j < dh; j++) {
            const double v = (double)cb[((int64_t)hs * K + c) * dh + j];
            s = __fma_rn(v, v, s);
        }
        cn2[hs * K + c] = s;
    }
}

template <int NKB>
__global__ void __launch_bounds__(SB_THREADS) k_screen_tc(const __grid_constant__ CUtensorMap mapQ,
                                                          const __grid_constant__ CUtensorMap mapC,
                                                          const float *__restrict__ qrot, int pitch, int64_t q0,
                                                          int64_t Qc, int K, int dh, int nhalf,
                                                          const double *__restrict__ cn2,
                                                          ScreenOut *__restrict__ scr, int RQ, int dbg,
                                                          const int32_t *__restrict__ hoff) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    // 1024-byte aligned (the 128-byte swizzle atoms), keeping the shared-memory provenance
    unsigned char *base = smraw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smraw) & 1023u)) & 1023u);
    unsigned char *As = base;                        // NKB tiles of 128 rows x 128 B
    unsigned char *Bs = base + NKB * SB_M * 128;     // NKB tiles of 64 rows x 128 B
    __shared__ __align__(8) uint64_t full, done;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int hs = blockIdx.x;                       // half-subspace 2m + h
    const int64_t m0 = q0 + (int64_t)blockIdx.y * SB_M;
    // the half's dims: [hoff[hs], hoff[hs] + hw) (R18), else [hs dh, (hs + 1) dh); query dims read
    // past hw meet zero codebook entries (exact zero products)
    const int ho = hoff ? hoff[hs] : hs * dh, hw = hoff ? hoff[hs + 1] - hoff[hs] : dh;
    if (tid == 0) {
        tcu::mbar_init(&full, 1);
        tcu::mbar_init(&done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
                         tcu::smem_u32(&tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base;
    if (tid == 0 && !(dbg & 4)) {
        tcu::mbar_expect_tx(&full, (uint32_t)(NKB * (SB_M + SB_N) * 128));
        for (int kb = 0; kb < NKB; kb++) {
            tcu::tma_load_2d(As + kb * SB_M * 128, &mapQ, ho + kb * 32, (int)m0, &full);
            tcu::tma_load_2d(Bs + kb * SB_N * 128, &mapC, kb * 32, hs * SB_N, &full);
        }
    }
    if (warp == 0) {
        if (!(dbg & 4)) tcu::mbar_wait(&full, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        constexpr uint32_t ID = tcu::idesc(1u, 2u, SB_M, SB_N);  // tf32 x tf32 -> f32
        const uint64_t da = tcu::sw128_desc(tcu::smem_u32(As)), db = tcu::sw128_desc(tcu::smem_u32(Bs));
#pragma unroll
        for (int kb = 0; kb < NKB; kb++)
#pragma unroll
            for (int kk = 0; kk < 4; kk++)  // 8 tf32 = 32 bytes per MMA
                if (!(dbg & 1))
                tcu::mma<1>(tmem, da + (uint64_t)((kb * SB_M * 128) >> 4) + 2 * kk,
                            db + (uint64_t)((kb * SB_N * 128) >> 4) + 2 * kk, ID, (kb | kk) ? 1u : 0u);
        tcu::mma_commit(&done);
    }
    __syncwarp();
    tcu::mbar_wait(&done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // epilogue: thread = query row m0 + tid (TMEM lane), columns = centroids.  The
    // intervals go to shared memory (the operand tiles are no longer needed), then the
    // thread selects for its (query, half): t = the RQ-th smallest upper bound, and the
    // mask of the centroids whose lower bound is <= t (the only ones that can be among
    // the RQ smallest dist64 values)
    const int64_t q = m0 + warp * 32 + lane;
    const bool live = q < Qc;
    double nq = 0.0;
    if (live) {
        const float *qr = qrot + q * pitch + ho;
        for (int j = 0; j < hw; j++) {
            const double v = (double)qr[j];
            nq = __fma_rn(v, v, nq);
        }
    }
    const double sq = sqrt(nq);
    const double eps_dot = (0x1p-9 + (double)(dh + 2) * 0x1p-23) * (1.0 + 0x1p-20);
    const double eps_sum = (double)(dh + 4) * 0x1p-52;
    float *los = (float *)base + tid, *his = (float *)base + SB_THREADS * SB_N + tid;  // [c * SB_THREADS + tid]
    const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c0 = 0; c0 < SB_N; c0 += 16) {
        uint32_t v[16] = {};
        if (!(dbg & 2))
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(trow + (uint32_t)c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const int c = c0 + j;
            float lo = INFINITY, hi = INFINITY;
            if (c < K) {
                const double nc = cn2[hs * K + c];
                const double dot = (double)__uint_as_float(v[j]);
                const double sv = nq + nc - 2.0 * dot;
                const double e = 2.0 * eps_dot * sq * sqrt(nc) * (1.0 + 0x1p-40) + eps_sum * (nq + nc) +
                                 0x1p-50 * (nq + nc + 2.0 * fabs(dot));  // the fp64 evaluation of sv and e
                lo = __double2float_rd(fmax(0.0, sv - e));
                hi = __double2float_ru(sv + e);
                if (!(lo <= hi)) lo = -INFINITY, hi = INFINITY;  // NaN: no information
            }
            los[c * SB_THREADS] = lo;
            his[c * SB_THREADS] = hi;
        }
    }
    if (live) {
        // t: any value works for exactness (k_probe certifies the prefix of members with
        // dist64 <= t and redoes a walk that goes past it); aim at the RQ-th smallest upper
        // bound by bisection over [min hi, max hi]: after the steps, t = the bracket's top,
        // with at least RQ upper bounds <= t
        const int R = min(RQ, K);
        float lo_t = INFINITY, hi_t = -INFINITY;
        for (int c = 0; c < K; c++) {
            lo_t = fminf(lo_t, his[c * SB_THREADS]);
            hi_t = fmaxf(hi_t, his[c * SB_THREADS]);
        }
        float t = hi_t;
        if (isfinite(lo_t) && isfinite(hi_t))
            for (int it = 0; it < 10; it++) {
                const float mid = 0.5f * (lo_t + t);
                int n = 0;
                for (int c = 0; c < K; c++) n += his[c * SB_THREADS] <= mid;
                if (n >= R) t = mid;
                else lo_t = mid;
            }
        else
            t = INFINITY;
        unsigned long long mask = 0ull;
        for (int c = 0; c < K; c++) mask |= (unsigned long long)(los[c * SB_THREADS] <= t) << c;
        scr[(q - q0) * nhalf + hs] = ScreenOut{t, 0, mask};
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
}

}  // namespace

// the padded codebooks and centroid norms of the screen, once per index
void prepare_screen(crisp_index *ix, cudaStream_t s) {
    if (ix->cbp) return;
    const int DHP = (ix->dh + 31) / 32 * 32, nh = 2 * ix->M;
    CRISP_CUDA(cudaMalloc(&ix->cbp, (size_t)nh * SB_N * DHP * 4));
    CRISP_CUDA(cudaMalloc(&ix->cn2, (size_t)nh * ix->K * 8));
    ix->hbm_bytes += (int64_t)nh * SB_N * DHP * 4 + (int64_t)nh * ix->K * 8;
    k_pad_codebooks<<<nh * SB_N, 64, 0, s>>>(ix->cb, ix->M, ix->K, ix->dh, DHP, ix->cbp, ix->cn2);
    CRISP_LAUNCH();
}

bool screen_supported(const crisp_index *ix) {
    // K <= 64 centroids per half (one N = 64 tile), d_h <= 128 (four 32-float k-blocks), a
    // 16-byte row pitch (TMA strides)
    // and 16-byte-aligned half-subspace slices (d_h a multiple of 4: TMA box starts)
    bool ok = ix->K <= SB_N && ix->dh <= 128 && (ix->dh % 4) == 0 && (ix->pitch % 4) == 0;
    for (int32_t o : ix->hoff_h) ok = ok && (o % 4) == 0;  // adaptive widths (R18): aligned half starts
    return ok;
}

// intervals [lo, hi] of dist64(q'_{m,h}, C_{m,h,c}) for queries [q0, q1) of qrot:
// scr[((q - q0) * 2M + 2m + h) * K + c]
void screen_halves(crisp_index *ix, const float *qrot, int64_t q0, int64_t q1, ScreenOut *scr, int RQ,
                   cudaStream_t s) {
    if (q1 <= q0) return;
    prepare_screen(ix, s);
    const int DHP = (ix->dh + 31) / 32 * 32, NKB = DHP / 32, nh = 2 * ix->M;
    const CUtensorMap mQ = map_f32(qrot, (uint64_t)ix->pitch, (uint64_t)q1, (uint64_t)ix->pitch, SB_M);
    const CUtensorMap mC = map_f32(ix->cbp, (uint64_t)DHP, (uint64_t)nh * SB_N, (uint64_t)DHP, SB_N);
    // operand tiles, reused afterwards for the intervals of the tile (128 x 64 x 8 bytes)
    const int smem = std::max(NKB * (SB_M + SB_N) * 128, SB_M * SB_N * 8) + 1024;
    static std::mutex mu;
    static std::map<int, bool> attr;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!attr[ix->device]) {
            CRISP_CUDA(cudaFuncSetAttribute(k_screen_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 192 * 128 + 1024));
            CRISP_CUDA(cudaFuncSetAttribute(k_screen_tc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 192 * 128 + 1024));
            CRISP_CUDA(cudaFuncSetAttribute(k_screen_tc<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 192 * 128 + 1024));
            CRISP_CUDA(cudaFuncSetAttribute(k_screen_tc<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 192 * 128 + 1024));
            attr[ix->device] = true;
        }
    }
    dim3 g((unsigned)nh, (unsigned)((q1 - q0 + SB_M - 1) / SB_M));
    const int dbg = getenv("CRISP_SCREEN_DEBUG") ? atoi(getenv("CRISP_SCREEN_DEBUG")) : 0;  // bisection knobs
#define CRISP_SCR(NK)                                                                                              \
    k_screen_tc<NK><<<g, SB_THREADS, smem, s>>>(mQ, mC, qrot, ix->pitch, q0, q1, ix->K, ix->dh, nh, ix->cn2, scr, RQ, dbg, \
                                                ix->hoff)
    if (NKB == 1) CRISP_SCR(1);
    else if (NKB == 2) CRISP_SCR(2);
    else if (NKB == 3) CRISP_SCR(3);
    else CRISP_SCR(4);
#undef CRISP_SCR
    CRISP_LAUNCH();
}

}  // namespace crisp
