// crisp_internal.cuh -- internal declarations of libcrisp (CUDA path only).
// Shares nothing with oracle/ (the CPU checker).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/crisp.h"

// ---------------------------------------------------------------------------
// Error plumbing: every CUDA status is mapped to a crisp_status with a
// thread-local message (crisp_last_error).
// ---------------------------------------------------------------------------
namespace crisp {

void set_error(const std::string &msg);

struct Err {
    crisp_status st;
};

#define CRISP_CUDA(call)                                                                                 \
    do {                                                                                                 \
        cudaError_t e_ = (call);                                                                         \
        if (e_ != cudaSuccess) {                                                                         \
            ::crisp::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                      \
            throw ::crisp::Err{e_ == cudaErrorMemoryAllocation ? CRISP_ENOMEM : CRISP_ECUDA};            \
        }                                                                                                \
    } while (0)

#define CRISP_CHECK(cond, msg)                                                                           \
    do {                                                                                                 \
        if (!(cond)) {                                                                                   \
            ::crisp::set_error(msg);                                                                     \
            throw ::crisp::Err{CRISP_EINVAL};                                                            \
        }                                                                                                \
    } while (0)

#define CRISP_LAUNCH() CRISP_CUDA(cudaGetLastError())

// Method randomness streams (same numbering as DESIGN.md "Method randomness").
constexpr uint32_t STREAM_CEV_SAMPLE = 1u;
constexpr uint32_t STREAM_ROTATION = 2u;
constexpr uint32_t STREAM_KM_SAMPLE = 3u;
constexpr uint32_t STREAM_KM_INIT = 4u;

constexpr int MAX_M = 127;   // byte counters hold V <= 2M
constexpr int MAX_K = 255;
constexpr int MAX_TOPK = 1024;

}  // namespace crisp

// ---------------------------------------------------------------------------
// The index: everything lives in HBM (device pointers) except scalars.
// ---------------------------------------------------------------------------
struct crisp_index {
    int device = 0;
    int64_t N = 0, N_global = 0, gid_base = 0;
    int32_t D = 0, Dp = 0, pitch = 0, M = 0, K = 0, dh = 0, W = 0;
    int32_t Wp = 0;            // code row stride in words: W rounded up to 8 (64-B rows, 16-B loads)
    int32_t rotated = 0;       // 1: global rotation; 2: block-wise (R16)
    int32_t rot_block = 0;     // block-wise rotation over this many subspaces (0: global)
    // adaptive subspace decomposition (R18): half h covers dims [hoff_h[h], hoff_h[h+1]);
    // empty = the equal split (half h at h*dh).  dh is then the largest half width (the codebook
    // row stride; rows are zero beyond their half's width)
    std::vector<int32_t> hoff_h;
    int32_t *hoff = nullptr;   // device copy of hoff_h (nullptr: equal split)
    int32_t adaptive_req = 0;  // widths from the variance rule, chosen during the build
    double cev = 0.0;
    float *X = nullptr;        // N x pitch, stored (rotated) vectors, zero padded
    float *R = nullptr;        // Dp x Dp row-major (rotated only)
    int8_t *Rsl = nullptr;     // Dp x 7 Dpk: int8 slices of R's columns, descending (rotate_imma.cu)
    int32_t *Rexp = nullptr;   // Dp: column scale exponents of the slices
    double *Rn2 = nullptr;     // Dp: column 2-norms (x 1.01)
    float *Rt = nullptr;       // Dp x Dp: R transposed (the certified rotation's exact recompute)
    float *cb = nullptr;       // M x 2 x K x dh
    float *cbp = nullptr;      // 2M x 64 x DHP: codebooks padded for the a1 screen (probe_tc.cu)
    double *cn2 = nullptr;     // 2M x K: centroid squared norms (fp64) for the screen
    int32_t *cells = nullptr;  // M x N
    int32_t *ids = nullptr;    // M x N CSR ids
    int32_t *off2 = nullptr;   // M x K^2 x (NB+1): start of ids >= b*BS inside cell c
    int32_t *off2w = nullptr;  // M x K^2 x (NBW+1): the same at warp sub-block granularity SBW = BS/8
    int32_t *gsize = nullptr;  // M x K^2 sizes for the budget walk (local or global)
    uint64_t *codes = nullptr; // N x W
    // verification filter (DESIGN R17): rows centred on the column means and quantised per
    // row to int8 (x - mu ~ 2^e c), with c.c, e and rho >= ||(x - mu) - 2^e c|| per row;
    // certified bounds of the exact distances from a D-byte read
    int8_t *C8 = nullptr;      // N x c8pitch codes (null: filter off)
    int32_t *c8meta = nullptr; // N x 4: {c.c, e, rho (float bits), 0}
    float *mu = nullptr;       // pitch: column means (fp32)
    int32_t c8pitch = 0;       // code row stride (pitch rounded up to 16)
    int32_t vfilter = 1;       // build (and use) the filter
    int32_t BS = 0, NB = 0;    // on-chip counter block: ids per block, number of blocks
    int32_t SBW = 0, NBW = 0;  // warp sub-block: ids per sub-block (BS/8), number of sub-blocks (8*NB)
    double slice_hint = 0.0;   // expected ids of a query's activated slice per warp sub-block (count kernel choice)
    int64_t budget = 0;
    double beta = 0.0;         // the ratio the budget came from (0: given as an integer)
    int64_t maxcell_sum = 0;   // sum over subspaces of the largest (global) cell size: bounds R_qm - B
    int32_t tau = 1, patience_factor = 40;
    int32_t ad_on = 0, ad_stride = 32;  // Optimized Mode ADSampling (crisp_set_adsampling)
    double ad_eps0 = 2.1;
    int64_t workspace_bytes = 0;
    int64_t hbm_bytes = 0;
};

namespace crisp {

// expected slice length per warp sub-block from cell sizes (M x K^2, host):
// the size of the cell holding a random point, E[s] = sum s^2 / N, scaled to SBW
double slice_hint_of(const int32_t *sizes_host, int M, int64_t KK, int64_t N_global, int SBW);

// helpers implemented in api.cu
void *dmalloc(size_t bytes, crisp_index *ix);
bool is_device_ptr(const void *p);
int64_t decimal_ceil(double ratio, int64_t n);
// per-subspace largest cell size (global sizes, host M x K^2) -> ix->maxcell (exact candidate bound)
void cell_size_maxima(crisp_index *ix, const int32_t *sizes_host);

// build steps (build.cu)
// adaptive subspace decomposition (R18): validate M even widths summing to Dp and
// set the half offsets (an equal split leaves the index on the equal-split path)
void set_subspace_widths(crisp_index *ix, const int32_t *widths);
// the width rule on per-dimension variances (zero beyond var.size())
std::vector<int32_t> adaptive_widths(const std::vector<double> &var, int M, int Dp);
void build_index(crisp_index *ix, const float *data_dev, const float *R_inj, const float *cb_inj, int64_t kmeans_sample,
                 int32_t kmeans_iters, int32_t rotation_mode, float tau_cev, uint64_t seed, cudaStream_t s,
                 const double *cev_given = nullptr, const std::vector<double> *var_given = nullptr);
int64_t cev_sample_size(int64_t N);
void sample_row_ids(int64_t N, int64_t n, uint64_t seed, uint32_t stream, int32_t *rows_dev, cudaStream_t s);
double cev_of_sample(const float *S_dev, int64_t n, int D, cudaStream_t s, std::vector<double> *var = nullptr);
void finish_csr(crisp_index *ix, cudaStream_t s);
// the verification filter's int8 copy of the centred rows (build.cu; R17)
void build_verify_filter(crisp_index *ix, cudaStream_t s);

// fp64 sequential-order GEMM: Y(rows x Dp, pitch ldy) = fl32(X(rows x Dp, pitch ldx) . R(Dp x Dp))
// a0 on the int8 tensor cores, certified (rotate_imma.cu)
void prepare_rotation_slices(crisp_index *ix, cudaStream_t s);
bool rotate_imma_enabled();
void rotate_rows_imma(const crisp_index *ix, const float *X, int64_t rows, int64_t ldx, float *Y, int64_t ldy,
                      cudaStream_t s, unsigned long long *nfall);
void rotate_rows(crisp_index *ix, const float *X, int64_t rows, int64_t ldx, float *Y, int64_t ldy, cudaStream_t s);
void rotate_rows_f64(const float *X, int64_t rows, int32_t Dp, int64_t ldx, const float *R, float *Y, int64_t ldy,
                     cudaStream_t s);

// a1 screen on the tensor cores (probe_tc.cu): per (query, half-subspace) the
// threshold t (the RQ-th smallest certified upper bound of dist64) and the mask
// of the centroids whose certified lower bound is <= t
struct ScreenOut {
    float t;
    int32_t pad;
    unsigned long long mask;
};
bool screen_supported(const crisp_index *ix);
void screen_halves(crisp_index *ix, const float *qrot, int64_t q0, int64_t q1, ScreenOut *scr, int RQ,
                   cudaStream_t s);

// search (search.cu)
struct SearchOut {
    int64_t *ids;      // Q x k global ids (device)
    float *d32;        // Q x k fp32 (device) or null
    double *d64;       // Q x k fp64 (device) or null
};
struct TraceDev;  // device-side trace buffers (search.cu)
// queries_host: when not null, queries_dev is an uninitialised device staging
// buffer that the search fills from it (H2D overlapped with the query transform)
void search(const crisp_index *ix, const float *queries_dev, int64_t Q, int32_t k, int mode, SearchOut out,
            cudaStream_t s, const crisp_trace_t *host_trace, const float *queries_host = nullptr);
void merge_topk(const double *d, const int64_t *ids, int32_t G, int64_t Q, int32_t k, double *out_d64, float *out_d,
                int64_t *out_ids, cudaStream_t s);
crisp_session *session_begin(const crisp_index *ix, const float *queries, int64_t Q, int32_t k, int mode,
                             int32_t *local_counts, cudaStream_t s, bool transformed = false);
void transform_queries(const crisp_index *ix, const float *queries, int64_t Q, float *qrot, cudaStream_t s);
void session_hist(crisp_session *ss, const int32_t *gcount, int32_t *lhist, cudaStream_t s);
void session_finish(crisp_session *ss, const int32_t *gcount, const int32_t *allhist, int32_t G, int32_t rank,
                    int64_t *out_ids, double *out_d64, cudaStream_t s);
void session_free(crisp_session *ss);
// exact global patience over G shards (phi=1; search.cu)
void session_gp_order(crisp_session *ss, const int32_t *gcount, const int32_t *allhist, int32_t G, int32_t rank,
                      int32_t *local_hh, cudaStream_t s);
void session_gp_prepare(crisp_session *ss, const int32_t *all_hh, int32_t G, int32_t rank, const int64_t *gid_bases,
                        cudaStream_t s);
void session_gp_round(crisp_session *ss, int64_t *n_entries, cudaStream_t s);
void session_gp_fetch(crisp_session *ss, void *entries, int32_t *counts, cudaStream_t s);
void session_gp_replay(crisp_session *ss, const int32_t *all_cnt, const void *all_ent, int64_t stride, int32_t G,
                       int32_t *running, cudaStream_t s);
void session_gp_result(crisp_session *ss, int64_t *out_ids, double *out_d64, cudaStream_t s);

// stage timing
bool stage_timing_on();

}  // namespace crisp

// ---------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------
namespace crisp {

// Philox4x32-10 (Salmon et al. SC'11); same generator as the oracle writes on
// its own.
__host__ __device__ inline void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                               uint32_t k1, uint32_t out[4]) {
#pragma unroll
    for (int r = 0; r < 10; r++) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

__host__ __device__ inline void draw(uint64_t seed, uint32_t stream, uint64_t idx, uint32_t sub, uint32_t o[4]) {
    philox4x32_10((uint32_t)idx, (uint32_t)(idx >> 32), stream, sub, (uint32_t)seed, (uint32_t)(seed >> 32), o);
}

__host__ __device__ inline double u53(uint32_t a, uint32_t b) {
    uint64_t v = (((uint64_t)a << 32) | (uint64_t)b) >> 11;
    return (double)v * (1.0 / 9007199254740992.0);
}

__host__ __device__ inline double uniform(uint64_t seed, uint32_t stream, uint64_t idx, uint32_t sub) {
    uint32_t o[4];
    draw(seed, stream, idx, sub, o);
    return u53(o[0], o[1]);
}

// dist64 over n floats: d = (double)a - (double)b, s = fma(d, d, s), ascending i.
__device__ __forceinline__ double dist64(const float *__restrict__ a, const float *__restrict__ b, int n) {
    double s = 0.0;
    for (int i = 0; i < n; i++) {
        double d = __dsub_rn((double)a[i], (double)b[i]);
        s = __fma_rn(d, d, s);
    }
    return s;
}

}  // namespace crisp
