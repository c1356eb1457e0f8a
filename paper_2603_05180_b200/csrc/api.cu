// api.cu -- extern "C" entry points of libcrisp.so (see include/crisp.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <map>
#include <vector>

#include "crisp_internal.cuh"

namespace crisp {

static thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }

bool is_device_ptr(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ceil(ratio * n) with ratio read as the decimal it was written as (SURVEY
// 8(c) O1: B = ceil(beta N), tau = ceil(alpha M) "computed exactly: parse beta and
// alpha as decimal rationals").  The decimal is the shortest one that rounds to
// the given double (the repr a user types and a language prints: 0.035, not
// 0.035000000000000003), found by trying 1..17 significant digits; then
// ceil(mant * 10^e10 * n) in 128-bit integers.  0.035 * 20000 -> 700 and
// 0.07 * 100 -> 7, where the binary product rounds to 701 and 8.
int64_t decimal_ceil(double ratio, int64_t n) {
    if (!(ratio > 0.0) || !std::isfinite(ratio) || n <= 0) return 0;
    char buf[64];
    int prec = 1;
    for (; prec <= 17; prec++) {
        snprintf(buf, sizeof buf, "%.*e", prec - 1, ratio);
        if (strtod(buf, nullptr) == ratio) break;
    }
    // buf = d.ddd...e[+-]XX : mantissa digits and the decimal exponent
    __int128 mant = 0;
    int ndig = 0, e10 = 0;
    const char *c = buf;
    for (; *c && *c != 'e'; c++)
        if (*c >= '0' && *c <= '9') {
            mant = mant * 10 + (*c - '0');
            ndig++;
        }
    if (*c == 'e') e10 = atoi(c + 1);
    int scale = e10 - (ndig - 1);  // ratio = mant * 10^scale
    __int128 num = mant * (__int128)n;
    if (scale >= 0) {
        for (int i = 0; i < scale; i++) num *= 10;
        return (int64_t)num;
    }
    __int128 den = 1;
    for (int i = 0; i < -scale; i++) den *= 10;
    return (int64_t)((num + den - 1) / den);
}

static void apply_knobs(crisp_index *ix, double beta, int64_t budget, double alpha, int32_t tau, int32_t pf) {
    if (budget > 0) {
        ix->budget = budget;
        ix->beta = 0.0;
    } else {
        CRISP_CHECK(beta > 0.0 && beta <= 1.0, "budget_ratio must be in (0, 1]");
        ix->beta = beta;  // re-derived when the global cell sizes (N_global) change
        ix->budget = std::max<int64_t>(1, decimal_ceil(beta, ix->N_global));
    }
    if (tau > 0) ix->tau = tau;
    else {
        CRISP_CHECK(alpha > 0.0 && alpha <= 1.0, "min_collision_ratio must be in (0, 1]");
        ix->tau = (int32_t)std::max<int64_t>(1, decimal_ceil(alpha, ix->M));
    }
    CRISP_CHECK(pf >= 0, "patience_factor must be >= 0");
    ix->patience_factor = pf;
}

// ids per on-chip counter block: a power of two in [4096, 32768] (the count
// kernel gives each of its 8 warps BS/8 <= 4096 counters)
static int block_ids_for(int64_t N) {
    int cap = 32768;
    if (const char *v = getenv("CRISP_BLOCK_IDS")) cap = std::max(4096, std::min(32768, atoi(v)));
    int bs = 4096;
    while (bs < cap && bs < N) bs <<= 1;
    while (bs > cap) bs >>= 1;
    return std::max(4096, bs);
}

template <class T>
static T *dalloc(crisp_index *ix, size_t n) {
    void *p = nullptr;
    CRISP_CUDA(cudaMalloc(&p, std::max<size_t>(n * sizeof(T), 16)));
    ix->hbm_bytes += (int64_t)(n * sizeof(T));
    return (T *)p;
}

static void free_index(crisp_index *ix) {
    if (!ix) return;
    cudaSetDevice(ix->device);
    cudaFree(ix->X);
    cudaFree(ix->R);
    cudaFree(ix->Rsl);
    cudaFree(ix->Rexp);
    cudaFree(ix->Rn2);
    cudaFree(ix->Rt);
    cudaFree(ix->cb);
    cudaFree(ix->cbp);
    cudaFree(ix->cn2);
    cudaFree(ix->cells);
    cudaFree(ix->ids);
    cudaFree(ix->off2);
    cudaFree(ix->off2w);
    cudaFree(ix->gsize);
    cudaFree(ix->codes);
    cudaFree(ix->C8);
    cudaFree(ix->c8meta);
    cudaFree(ix->mu);
    cudaFree(ix->hoff);
    delete ix;
}

static crisp_index *new_index(int64_t N, int32_t D, const crisp_params *p) {
    CRISP_CHECK(p != nullptr, "params is NULL");
    CRISP_CHECK(N >= 1, "N must be >= 1");
    CRISP_CHECK(D >= 1, "D must be >= 1");
    CRISP_CHECK(p->M >= 1 && p->M <= MAX_M, "M must be in [1, 127]");
    CRISP_CHECK(p->K >= 1 && p->K <= MAX_K, "K must be in [1, 255]");
    CRISP_CHECK((int64_t)p->M * N < (1LL << 31), "M*N must be < 2^31");
    int ndev = 0;
    CRISP_CUDA(cudaGetDeviceCount(&ndev));
    CRISP_CHECK(p->device >= 0 && p->device < ndev, "invalid device ordinal");
    CRISP_CUDA(cudaSetDevice(p->device));
    {
        // keep freed search scratch in the pool (no OS round trips per search)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, p->device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    crisp_index *ix = new crisp_index();
    ix->device = p->device;
    ix->N = N;
    ix->N_global = N;
    ix->D = D;
    ix->M = p->M;
    ix->K = p->K;
    ix->Dp = ((D + 2 * p->M - 1) / (2 * p->M)) * (2 * p->M);
    ix->dh = ix->Dp / (2 * p->M);
    ix->pitch = ((ix->Dp + 3) / 4) * 4;
    ix->W = (ix->Dp + 63) / 64;
    ix->Wp = (ix->W + 7) / 8 * 8;
    CRISP_CHECK(p->rotation_block >= 0 && p->rotation_block <= p->M, "rotation_block must be in [0, M]");
    ix->rot_block = p->rotation_block;
    if (p->subspace_widths) set_subspace_widths(ix, p->subspace_widths);
    else ix->adaptive_req = p->adaptive_subspaces != 0;
    CRISP_CHECK(!(ix->rot_block > 0 && (ix->adaptive_req || !ix->hoff_h.empty())),
                "rotation_block with adaptive subspaces is not supported");
    ix->BS = block_ids_for(N);
    ix->NB = (int32_t)((N + ix->BS - 1) / ix->BS);
    ix->SBW = ix->BS / 8;
    ix->NBW = ix->NB * 8;
    ix->workspace_bytes = p->workspace_bytes;
    {
        const char *e = getenv("CRISP_VERIFY_FILTER");  // build-time default of crisp_set_verify_filter
        ix->vfilter = (e && *e) ? (atoi(e) != 0) : 1;
    }
    try {
        const int64_t KK = (int64_t)ix->K * ix->K;
        ix->X = dalloc<float>(ix, (size_t)N * ix->pitch);
        if (!ix->adaptive_req) ix->cb = dalloc<float>(ix, (size_t)ix->M * 2 * ix->K * ix->dh);  // else: in the build
        ix->cells = dalloc<int32_t>(ix, (size_t)ix->M * N);
        ix->ids = dalloc<int32_t>(ix, (size_t)ix->M * N + 4);  // +4: k_count_frag's 16-byte loads of the last quad
        ix->off2 = dalloc<int32_t>(ix, (size_t)ix->M * KK * (ix->NB + 1));
        ix->off2w = dalloc<int32_t>(ix, (size_t)ix->M * KK * (ix->NBW + 1));
        ix->gsize = dalloc<int32_t>(ix, (size_t)ix->M * KK);
        ix->codes = dalloc<uint64_t>(ix, (size_t)N * ix->Wp);
    } catch (...) {
        free_index(ix);
        throw;
    }
    return ix;
}

static const float *to_device(const float *src, size_t n, std::vector<void *> &tmp) {
    if (is_device_ptr(src)) return src;
    void *p = nullptr;
    CRISP_CUDA(cudaMalloc(&p, n * sizeof(float)));
    tmp.push_back(p);
    CRISP_CUDA(cudaMemcpy(p, src, n * sizeof(float), cudaMemcpyHostToDevice));
    return (const float *)p;
}

struct TmpFree {
    std::vector<void *> v;
    ~TmpFree() {
        for (void *p : v) cudaFree(p);
    }
};

static crisp_status build_common(const float *data, int64_t N, int64_t gid_base, int32_t D, const crisp_params *p,
                                 const float *R, const float *cb, bool inject, crisp_index **out) {
    crisp_index *ix = nullptr;
    try {
        CRISP_CHECK(out != nullptr, "out is NULL");
        CRISP_CHECK(data != nullptr, "data is NULL");
        if (inject) CRISP_CHECK(cb != nullptr, "codebooks are NULL");
        CRISP_CHECK(!(inject && p->adaptive_subspaces && !p->subspace_widths),
                    "injected codebooks of an adaptive split need subspace_widths");
        ix = new_index(N, D, p);
        ix->gid_base = gid_base;
        // device inputs may still be in flight on the caller's streams (the build
        // runs on its own non-blocking stream): order the build after all of it
        CRISP_CUDA(cudaDeviceSynchronize());
        TmpFree tf;
        const float *dd = to_device(data, (size_t)N * D, tf.v);
        const float *Rd = R ? to_device(R, (size_t)ix->Dp * ix->Dp, tf.v) : nullptr;
        const float *cbd = inject ? to_device(cb, (size_t)ix->M * 2 * ix->K * ix->dh, tf.v) : nullptr;
        cudaStream_t s;
        CRISP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct SG {
            cudaStream_t s;
            ~SG() { cudaStreamDestroy(s); }
        } sg{s};
        build_index(ix, dd, Rd, cbd, p->kmeans_sample > 0 ? p->kmeans_sample : 100000,
                    p->kmeans_iters > 0 ? p->kmeans_iters : 20, inject ? 0 : p->rotation, p->tau_cev, p->seed, s);
        apply_knobs(ix, p->budget_ratio, p->budget, p->min_collision_ratio, p->tau, p->patience_factor);
        *out = ix;
        return CRISP_OK;
    } catch (Err &e) {
        free_index(ix);
        return e.st;
    } catch (std::exception &e) {
        set_error(e.what());
        free_index(ix);
        return CRISP_ECUDA;
    }
}

}  // namespace crisp

using namespace crisp;

extern "C" {

const char *crisp_last_error(void) { return g_err.c_str(); }
const char *crisp_version(void) { return "crisp-b200 0.2 (sm_100a)"; }

int64_t crisp_exact_ceil(double ratio, int64_t n) { return decimal_ceil(ratio, n); }

crisp_status crisp_default_params(crisp_params *p) {
    if (!p) {
        set_error("params is NULL");
        return CRISP_EINVAL;
    }
    memset(p, 0, sizeof(*p));
    p->M = 16;
    p->K = 50;
    p->tau_cev = 0.85f;
    p->rotation = -1;
    p->kmeans_iters = 20;
    p->kmeans_sample = 100000;
    p->seed = 0;
    p->device = 0;
    p->budget_ratio = 0.01;
    p->budget = 0;
    p->min_collision_ratio = 0.3;
    p->tau = 0;
    p->patience_factor = 40;
    p->workspace_bytes = 0;
    return CRISP_OK;
}

crisp_status crisp_build(const float *data, int64_t N, int32_t D, const crisp_params *p, crisp_index **out) {
    return build_common(data, N, 0, D, p, nullptr, nullptr, false, out);
}

crisp_status crisp_build_with(const float *data, int64_t N, int32_t D, const crisp_params *p, const float *R,
                              const float *codebooks, crisp_index **out) {
    return build_common(data, N, 0, D, p, R, codebooks, true, out);
}

int64_t crisp_cev_sample_size(int64_t N) { return N < 0 ? 0 : cev_sample_size(N); }

crisp_status crisp_sample_rows(int64_t N, int64_t n, uint64_t seed, uint32_t stream, int32_t *rows_out) {
    try {
        CRISP_CHECK(rows_out != nullptr, "rows_out is NULL");
        CRISP_CHECK(N >= 1 && n >= 0 && n <= N && N < (1LL << 31), "need 0 <= n <= N < 2^31");
        if (n == 0) return CRISP_OK;
        int dev = 0;
        CRISP_CUDA(cudaGetDevice(&dev));
        const bool on_dev = is_device_ptr(rows_out);
        int32_t *d = rows_out;
        if (!on_dev) CRISP_CUDA(cudaMalloc(&d, (size_t)n * 4));
        struct F {
            int32_t *p;
            bool own;
            ~F() {
                if (own) cudaFree(p);
            }
        } f{d, !on_dev};
        sample_row_ids(N, n, seed, stream, d, 0);
        CRISP_CUDA(cudaDeviceSynchronize());
        if (!on_dev) CRISP_CUDA(cudaMemcpy(rows_out, d, (size_t)n * 4, cudaMemcpyDeviceToHost));
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_build_model(const float *cev_rows, int64_t n_cev, const float *km_rows, int64_t n_km, int32_t D,
                               const crisp_params *p, float *R_out, float *codebooks_out, int32_t *rotated_out,
                               double *cev_out) {
    crisp_index *ix = nullptr;
    try {
        CRISP_CHECK(p && km_rows && codebooks_out && rotated_out, "NULL argument");
        CRISP_CHECK(n_km >= 1 && n_cev >= 0 && D >= 1, "bad sizes");
        CRISP_CHECK(!p->adaptive_subspaces && !p->subspace_widths, "crisp_build_model takes the equal split only");
        CRISP_CHECK(n_cev < 2 || cev_rows != nullptr, "cev_rows is NULL");
        ix = new_index(n_km, D, p);
        CRISP_CUDA(cudaDeviceSynchronize());
        TmpFree tf;
        double cev = 0.0;
        cudaStream_t s;
        CRISP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct SG {
            cudaStream_t s;
            ~SG() { cudaStreamDestroy(s); }
        } sg{s};
        std::vector<double> var(D, 0.0);
        if (n_cev >= 2) {
            const float *cd = to_device(cev_rows, (size_t)n_cev * D, tf.v);
            cev = cev_of_sample(cd, n_cev, D, s, &var);
        }
        const float *kd = to_device(km_rows, (size_t)n_km * D, tf.v);
        // an index over the k-means sample: the same rotation (seed; a block rotation from the
        // CEV sample's variances) and k-means (every row of the sample, ascending global id) as
        // a build over the whole dataset
        build_index(ix, kd, nullptr, nullptr, n_km, p->kmeans_iters > 0 ? p->kmeans_iters : 20, p->rotation,
                    p->tau_cev, p->seed, s, &cev, &var);
        *rotated_out = ix->rotated;
        if (cev_out) *cev_out = cev;
        if (ix->rotated && R_out)
            CRISP_CUDA(cudaMemcpy(R_out, ix->R, (size_t)ix->Dp * ix->Dp * 4, cudaMemcpyDefault));
        CRISP_CUDA(cudaMemcpy(codebooks_out, ix->cb, (size_t)ix->M * 2 * ix->K * ix->dh * 4, cudaMemcpyDefault));
        free_index(ix);
        return CRISP_OK;
    } catch (Err &e) {
        free_index(ix);
        return e.st;
    } catch (std::exception &e) {
        set_error(e.what());
        free_index(ix);
        return CRISP_ECUDA;
    }
}

crisp_status crisp_build_shard(const float *shard, int64_t N_local, int64_t gid_base, int32_t D, const crisp_params *p,
                               const float *R, const float *codebooks, crisp_index **out) {
    return build_common(shard, N_local, gid_base, D, p, R, codebooks, true, out);
}

void crisp_free(crisp_index *idx) { free_index(idx); }

crisp_status crisp_local_cell_sizes(const crisp_index *ix, int64_t *sizes) {
    try {
        CRISP_CHECK(ix && sizes, "NULL argument");
        CRISP_CUDA(cudaSetDevice(ix->device));
        const int64_t KK = (int64_t)ix->K * ix->K;
        std::vector<int32_t> off((size_t)ix->M * KK * (ix->NB + 1));
        CRISP_CUDA(cudaMemcpy(off.data(), ix->off2, off.size() * 4, cudaMemcpyDeviceToHost));
        for (int m = 0; m < ix->M; m++)
            for (int64_t c = 0; c < KK; c++) {
                const int32_t *o = off.data() + ((int64_t)m * KK + c) * (ix->NB + 1);
                sizes[m * KK + c] = o[ix->NB] - o[0];
            }
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_set_global_cell_sizes(crisp_index *ix, const int64_t *sizes) {
    try {
        CRISP_CHECK(ix && sizes, "NULL argument");
        CRISP_CUDA(cudaSetDevice(ix->device));
        const int64_t KK = (int64_t)ix->K * ix->K;
        std::vector<int32_t> h((size_t)ix->M * KK);
        int64_t n0 = 0;
        for (int64_t c = 0; c < KK; c++) n0 += sizes[c];
        for (int m = 0; m < ix->M; m++) {
            int64_t nm = 0;
            for (int64_t c = 0; c < KK; c++) {
                CRISP_CHECK(sizes[m * KK + c] >= 0 && sizes[m * KK + c] < (1LL << 31), "bad cell size");
                h[m * KK + c] = (int32_t)sizes[m * KK + c];
                nm += sizes[m * KK + c];
            }
            CRISP_CHECK(nm == n0, "cell sizes must sum to the same N in every subspace");
        }
        CRISP_CHECK(n0 >= ix->N, "global sizes smaller than the local shard");
        CRISP_CUDA(cudaMemcpy(ix->gsize, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
        ix->N_global = n0;
        ix->slice_hint = slice_hint_of(h.data(), ix->M, KK, n0, ix->SBW);
        cell_size_maxima(ix, h.data());
        // a budget given as a ratio follows N_global (B = ceil(beta N_global), O1)
        if (ix->beta > 0.0) ix->budget = std::max<int64_t>(1, decimal_ceil(ix->beta, ix->N_global));
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_set_adsampling(crisp_index *ix, int32_t enable, double eps0, int32_t stride) {
    try {
        CRISP_CHECK(ix != nullptr, "index is NULL");
        CRISP_CHECK(!enable || (stride >= 4 && stride % 4 == 0 && 128 % stride == 0),
                    "ADSampling stride must be a multiple of 4 that divides 128");
        CRISP_CHECK(!enable || (eps0 >= 0.0 && std::isfinite(eps0)), "ADSampling eps0 must be finite and >= 0");
        ix->ad_on = enable ? 1 : 0;
        if (enable) {
            ix->ad_eps0 = eps0;
            ix->ad_stride = stride;
        }
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_set_verify_filter(crisp_index *ix, int32_t enable) {
    try {
        CRISP_CHECK(ix != nullptr, "index is NULL");
        CRISP_CUDA(cudaSetDevice(ix->device));
        CRISP_CUDA(cudaDeviceSynchronize());  // searches in flight may read the copy
        if (enable && !ix->C8) {
            cudaStream_t s;
            CRISP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            try {
                crisp::build_verify_filter(ix, s);
                CRISP_CUDA(cudaStreamSynchronize(s));
            } catch (...) {
                cudaStreamDestroy(s);
                throw;
            }
            cudaStreamDestroy(s);
        } else if (!enable && ix->C8) {
            cudaFree(ix->C8);
            cudaFree(ix->c8meta);
            cudaFree(ix->mu);
            ix->C8 = nullptr;
            ix->c8meta = nullptr;
            ix->mu = nullptr;
            ix->hbm_bytes -= ix->N * (int64_t)ix->c8pitch + ix->N * 16 + (int64_t)ix->pitch * 4;
        }
        ix->vfilter = enable ? 1 : 0;
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_set_search_params(crisp_index *ix, double beta, int64_t budget, double alpha, int32_t tau,
                                     int32_t patience_factor) {
    try {
        CRISP_CHECK(ix != nullptr, "index is NULL");
        apply_knobs(ix, beta, budget, alpha, tau, patience_factor);
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_index_info(const crisp_index *ix, crisp_index_info_t *o) {
    if (!ix || !o) {
        set_error("NULL argument");
        return CRISP_EINVAL;
    }
    o->N = ix->N;
    o->N_global = ix->N_global;
    o->gid_base = ix->gid_base;
    o->D = ix->D;
    o->padded_D = ix->Dp;
    o->pitch = ix->pitch;
    o->slice_hint = ix->slice_hint;
    o->M = ix->M;
    o->K = ix->K;
    o->dh = ix->dh;
    o->rotated = ix->rotated;
    o->cev = ix->cev;
    o->budget = ix->budget;
    o->tau = ix->tau;
    o->patience_factor = ix->patience_factor;
    o->block_ids = ix->BS;
    o->n_blocks = ix->NB;
    o->hbm_bytes = ix->hbm_bytes;
    o->rotation_block = ix->rotated ? ix->rot_block : 0;
    o->adaptive = ix->hoff_h.empty() ? 0 : 1;
    const int64_t KK = (int64_t)ix->K * ix->K;
    o->logical_bytes = 4 * ix->N * ix->Dp + 4 * (int64_t)ix->M * ix->N + 8 * (int64_t)ix->M * (KK + 1) +
                       4 * (int64_t)ix->M * 2 * ix->K * ix->dh + 8 * (int64_t)ix->W * ix->N +
                       (ix->rotated ? 4 * (int64_t)ix->Dp * ix->Dp : 0);
    return CRISP_OK;
}

static crisp_status search_impl(const crisp_index *ix, const float *queries, int64_t Q, int32_t k, crisp_mode mode,
                                int64_t *out_ids, float *out_d, double *out_d64, cudaStream_t s, bool sync_host,
                                const crisp_trace_t *tr) {
    try {
        CRISP_CHECK(ix != nullptr, "index is NULL");
        CRISP_CHECK(Q >= 0, "Q must be >= 0");
        CRISP_CHECK(k >= 1 && k <= MAX_TOPK, "k must be in [1, 1024]");
        CRISP_CHECK(k <= ix->N_global, "k > N");
        CRISP_CHECK(mode == CRISP_GUARANTEED || mode == CRISP_OPTIMIZED, "bad mode");
        CRISP_CHECK(out_ids != nullptr, "out_ids is NULL");
        CRISP_CUDA(cudaSetDevice(ix->device));
        if (Q == 0) return CRISP_OK;
        CRISP_CHECK(queries != nullptr, "queries is NULL");
        if (!sync_host) {
            CRISP_CHECK(is_device_ptr(queries) && is_device_ptr(out_ids), "async search needs device pointers");
            SearchOut so{out_ids, out_d, out_d64};
            search(ix, queries, Q, k, (int)mode, so, s, tr);
            return CRISP_OK;
        }
        // synchronous call: device arguments may still be written by work the
        // caller queued on any stream (the search runs on its own non-blocking
        // stream), so order it after all of it, as crisp_build does
        if (is_device_ptr(queries) || is_device_ptr(out_ids) || (out_d && is_device_ptr(out_d)))
            CRISP_CUDA(cudaDeviceSynchronize());
        // host buffers: stream-ordered device staging (H2D in, D2H out) on this host thread's
        // own stream for the device (kept for the thread's lifetime: the pool then reuses the
        // previous call's scratch on the same stream; measured with a fresh stream per call:
        // occasional 10-15 ms calls at cfg4)
        static thread_local std::map<int, cudaStream_t> tl_streams;
        cudaStream_t &st = tl_streams[ix->device];
        if (!st) CRISP_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        struct SG {
            cudaStream_t s;
            std::vector<void *> v;
            ~SG() {
                for (void *p : v) cudaFreeAsync(p, s);
                cudaStreamSynchronize(s);
            }
        } sg{st, {}};
        auto stage = [&](size_t bytes) {
            void *p = nullptr;
            CRISP_CUDA(cudaMallocAsync(&p, std::max<size_t>(bytes, 16), st));
            sg.v.push_back(p);
            return p;
        };
        const float *qd = queries, *qh = nullptr;
        if (!is_device_ptr(queries)) {  // staged: the search copies it in parts, overlapped with a0
            qd = (const float *)stage((size_t)Q * ix->D * 4);
            qh = queries;
        }
        bool ids_dev = is_device_ptr(out_ids), d_dev = out_d ? is_device_ptr(out_d) : true;
        int64_t *oi = ids_dev ? out_ids : (int64_t *)stage((size_t)Q * k * 8);
        float *od = (out_d && !d_dev) ? (float *)stage((size_t)Q * k * 4) : out_d;
        SearchOut so{oi, od, out_d64};
        search(ix, qd, Q, k, (int)mode, so, st, tr, qh);
        if (!ids_dev) CRISP_CUDA(cudaMemcpyAsync(out_ids, oi, (size_t)Q * k * 8, cudaMemcpyDeviceToHost, st));
        if (out_d && !d_dev) CRISP_CUDA(cudaMemcpyAsync(out_d, od, (size_t)Q * k * 4, cudaMemcpyDeviceToHost, st));
        CRISP_CUDA(cudaStreamSynchronize(st));
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    } catch (std::exception &e) {
        set_error(e.what());
        return CRISP_ECUDA;
    }
}

crisp_status crisp_search(const crisp_index *ix, const float *queries, int64_t Q, int32_t k, crisp_mode mode,
                          int64_t *out_ids, float *out_dist2) {
    return search_impl(ix, queries, Q, k, mode, out_ids, out_dist2, nullptr, nullptr, true, nullptr);
}

crisp_status crisp_search_async(const crisp_index *ix, const float *queries, int64_t Q, int32_t k, crisp_mode mode,
                                int64_t *out_ids, float *out_dist2, void *stream) {
    return search_impl(ix, queries, Q, k, mode, out_ids, out_dist2, nullptr, (cudaStream_t)stream, false, nullptr);
}

crisp_status crisp_search_shard_async(const crisp_index *ix, const float *queries, int64_t Q, int32_t k,
                                      crisp_mode mode, int64_t *out_ids, double *out_dist64, void *stream) {
    return search_impl(ix, queries, Q, k, mode, out_ids, nullptr, out_dist64, (cudaStream_t)stream, false, nullptr);
}

crisp_status crisp_search_trace(const crisp_index *ix, const float *queries, int64_t Q, int32_t k, crisp_mode mode,
                                int64_t *out_ids, float *out_dist2, crisp_trace_t *trace) {
    return search_impl(ix, queries, Q, k, mode, out_ids, out_dist2, nullptr, nullptr, true, trace);
}

crisp_status crisp_merge_topk(const double *d, const int64_t *ids, int32_t G, int64_t Q, int32_t k, double *out_d64,
                              float *out_d, int64_t *out_ids, void *stream) {
    try {
        CRISP_CHECK(d && ids && out_ids, "NULL argument");
        CRISP_CHECK(G >= 1 && k >= 1 && Q >= 0, "bad sizes");
        CRISP_CHECK(is_device_ptr(d) && is_device_ptr(ids) && is_device_ptr(out_ids), "device pointers required");
        merge_topk(d, ids, G, Q, k, out_d64, out_d, out_ids, (cudaStream_t)stream);
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_shard_search_begin(const crisp_index *ix, const float *queries, int64_t Q, int32_t k,
                                      crisp_mode mode, int32_t *local_counts, crisp_session **out, void *stream) {
    try {
        CRISP_CHECK(ix && queries && local_counts && out, "NULL argument");
        CRISP_CHECK(Q >= 1, "Q must be >= 1");
        CRISP_CHECK(k >= 1 && k <= MAX_TOPK && k <= ix->N_global, "bad k");
        CRISP_CHECK(mode == CRISP_GUARANTEED || mode == CRISP_OPTIMIZED, "bad mode");
        CRISP_CHECK(is_device_ptr(queries) && is_device_ptr(local_counts), "device pointers required");
        CRISP_CUDA(cudaSetDevice(ix->device));
        *out = session_begin(ix, queries, Q, k, (int)mode, local_counts, (cudaStream_t)stream);
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_transform_queries_async(const crisp_index *ix, const float *queries, int64_t Q, float *qrot,
                                           void *stream) {
    try {
        CRISP_CHECK(ix && queries && qrot, "NULL argument");
        CRISP_CHECK(Q >= 0, "Q must be >= 0");
        CRISP_CHECK(is_device_ptr(queries) && is_device_ptr(qrot), "device pointers required");
        CRISP_CUDA(cudaSetDevice(ix->device));
        transform_queries(ix, queries, Q, qrot, (cudaStream_t)stream);
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_shard_search_begin_transformed(const crisp_index *ix, const float *qrot, int64_t Q, int32_t k,
                                                  crisp_mode mode, int32_t *local_counts, crisp_session **out,
                                                  void *stream) {
    try {
        CRISP_CHECK(ix && qrot && local_counts && out, "NULL argument");
        CRISP_CHECK(Q >= 1, "Q must be >= 1");
        CRISP_CHECK(k >= 1 && k <= MAX_TOPK && k <= ix->N_global, "bad k");
        CRISP_CHECK(mode == CRISP_GUARANTEED || mode == CRISP_OPTIMIZED, "bad mode");
        CRISP_CHECK(is_device_ptr(qrot) && is_device_ptr(local_counts), "device pointers required");
        CRISP_CUDA(cudaSetDevice(ix->device));
        *out = session_begin(ix, qrot, Q, k, (int)mode, local_counts, (cudaStream_t)stream, true);
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_shard_search_hist(crisp_session *s, const int32_t *global_counts, int32_t *local_hist,
                                     void *stream) {
    try {
        CRISP_CHECK(s && global_counts && local_hist, "NULL argument");
        session_hist(s, global_counts, local_hist, (cudaStream_t)stream);
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_shard_search_finish(crisp_session *s, const int32_t *global_counts, const int32_t *all_hist,
                                       int32_t G, int32_t rank, int64_t *out_ids, double *out_dist64, void *stream) {
    try {
        CRISP_CHECK(s && global_counts && all_hist && out_ids && out_dist64, "NULL argument");
        CRISP_CHECK(G >= 1 && rank >= 0 && rank < G, "bad G / rank");
        session_finish(s, global_counts, all_hist, G, rank, out_ids, out_dist64, (cudaStream_t)stream);
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_shard_gp_order(crisp_session *s, const int32_t *global_counts, const int32_t *all_hist, int32_t G,
                                  int32_t rank, int32_t *local_hhist, void *stream) {
    try {
        CRISP_CHECK(s && global_counts && all_hist && local_hhist, "NULL argument");
        CRISP_CHECK(G >= 1 && G <= 32 && rank >= 0 && rank < G, "bad G / rank (G <= 32)");
        CRISP_CHECK(is_device_ptr(local_hhist), "device pointers required");
        session_gp_order(s, global_counts, all_hist, G, rank, local_hhist, (cudaStream_t)stream);
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_shard_gp_prepare(crisp_session *s, const int32_t *all_hhist, int32_t G, int32_t rank,
                                    const int64_t *gid_bases, void *stream) {
    try {
        CRISP_CHECK(s && all_hhist && gid_bases, "NULL argument");
        CRISP_CHECK(G >= 1 && G <= 32 && rank >= 0 && rank < G, "bad G / rank (G <= 32)");
        CRISP_CHECK(is_device_ptr(all_hhist), "device pointers required");
        session_gp_prepare(s, all_hhist, G, rank, gid_bases, (cudaStream_t)stream);
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_shard_gp_round(crisp_session *s, int64_t *n_entries, void *stream) {
    try {
        CRISP_CHECK(s && n_entries, "NULL argument");
        session_gp_round(s, n_entries, (cudaStream_t)stream);
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_shard_gp_fetch(crisp_session *s, void *entries, int32_t *counts, void *stream) {
    try {
        CRISP_CHECK(s && entries && counts, "NULL argument");
        CRISP_CHECK(is_device_ptr(entries) && is_device_ptr(counts), "device pointers required");
        session_gp_fetch(s, entries, counts, (cudaStream_t)stream);
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_shard_gp_replay(crisp_session *s, const int32_t *all_counts, const void *all_entries, int64_t stride,
                                   int32_t G, int32_t *running, void *stream) {
    try {
        CRISP_CHECK(s && all_counts && all_entries && running, "NULL argument");
        CRISP_CHECK(stride >= 0, "bad stride");
        session_gp_replay(s, all_counts, all_entries, stride, G, running, (cudaStream_t)stream);
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

crisp_status crisp_shard_gp_result(crisp_session *s, int64_t *out_ids, double *out_dist64, void *stream) {
    try {
        CRISP_CHECK(s && out_ids && out_dist64, "NULL argument");
        session_gp_result(s, out_ids, out_dist64, (cudaStream_t)stream);
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

void crisp_shard_search_free(crisp_session *s) { session_free(s); }

crisp_status crisp_export(const crisp_index *ix, crisp_export_t *o) {
    try {
        CRISP_CHECK(ix && o, "NULL argument");
        CRISP_CUDA(cudaSetDevice(ix->device));
        const int64_t N = ix->N, KK = (int64_t)ix->K * ix->K;
        if (o->R && ix->rotated)
            CRISP_CUDA(cudaMemcpy(o->R, ix->R, (size_t)ix->Dp * ix->Dp * 4, cudaMemcpyDeviceToHost));
        if (o->X)
            CRISP_CUDA(cudaMemcpy2D(o->X, (size_t)ix->Dp * 4, ix->X, (size_t)ix->pitch * 4, (size_t)ix->Dp * 4, N,
                                    cudaMemcpyDeviceToHost));
        if (o->codebooks)
            CRISP_CUDA(cudaMemcpy(o->codebooks, ix->cb, (size_t)ix->M * 2 * ix->K * ix->dh * 4, cudaMemcpyDeviceToHost));
        if (o->cells) CRISP_CUDA(cudaMemcpy(o->cells, ix->cells, (size_t)ix->M * N * 4, cudaMemcpyDeviceToHost));
        if (o->ids) CRISP_CUDA(cudaMemcpy(o->ids, ix->ids, (size_t)ix->M * N * 4, cudaMemcpyDeviceToHost));
        if (o->codes)
            CRISP_CUDA(cudaMemcpy2D(o->codes, (size_t)ix->W * 8, ix->codes, (size_t)ix->Wp * 8, (size_t)ix->W * 8, N,
                                    cudaMemcpyDeviceToHost));
        if (o->offsets) {
            std::vector<int32_t> off((size_t)ix->M * KK * (ix->NB + 1));
            CRISP_CUDA(cudaMemcpy(off.data(), ix->off2, off.size() * 4, cudaMemcpyDeviceToHost));
            for (int m = 0; m < ix->M; m++) {
                for (int64_t c = 0; c < KK; c++) o->offsets[m * (KK + 1) + c] = off[((int64_t)m * KK + c) * (ix->NB + 1)];
                o->offsets[m * (KK + 1) + KK] = N;
            }
        }
        if (o->cell_sizes) {
            std::vector<int32_t> g((size_t)ix->M * KK);
            CRISP_CUDA(cudaMemcpy(g.data(), ix->gsize, g.size() * 4, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < g.size(); i++) o->cell_sizes[i] = g[i];
        }
        if (o->subspace_widths)
            for (int m = 0; m < ix->M; m++)
                o->subspace_widths[m] = ix->hoff_h.empty() ? 2 * ix->dh : ix->hoff_h[2 * m + 2] - ix->hoff_h[2 * m];
        return CRISP_OK;
    } catch (Err &e) {
        return e.st;
    }
}

}  // extern "C"
