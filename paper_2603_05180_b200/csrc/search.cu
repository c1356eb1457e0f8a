// search.cu -- the batched CRISP query engine (Alg. 1) on sm_100a.
//
// Stages:
//   a0  k_prep_queries / rotate_rows_f64   q' = fl32(q R)
//   a1+a2  k_probe     half distances (dist64), half sorts, Multi-Sequence
//                      selection as a staircase argmin (== heap order, App. A.3),
//                      budget cut, rank weights                (Alg. 1 l.2-17)
//   a3+a4  k_count_select  collision counting over the CSR slices into
//                      on-chip byte counters per (query, id block), then the
//                      threshold compaction in ascending id      (Eq. 1; l.13-18)
//          k_fallback  |C| < k underflow fallback
//   a5 (phi=0) k_rerank_exact + k_merge_lists  exact L2 + top-k
//   a4+a5 (phi=1) k_rerank_patience  Hamming order + exact L2 in that order
//                      with patience P = factor*k
//   a6  k_merge_lists  cross-shard merge (multi-GPU)
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "crisp_internal.cuh"

#ifndef CRISP_CF_CAP
#define CRISP_CF_CAP 1024  // measured: 1024 (two entries per thread) beats 2048 at cfg4 (22.9 vs 24.6 ms) and cfg3
#endif
namespace crisp {

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

constexpr int WARPS = 8;
constexpr int THREADS = WARPS * 32;
constexpr int CS_CAP = 512;           // slice-table entries per round (count kernel)
constexpr int CS_U = 8;               // ids staged per thread per round
constexpr int CS_TCAP = THREADS * CS_U;  // positions per round
constexpr int HSORT_BW = 1024;       // bins per window of k_hsort_cta's per-warp counters
constexpr int PATIENCE_CH = 128;      // min rows verified per patience chunk (k_patience_tail)
constexpr int TAIL_CAP = 1024;        // max rows per chunk of k_patience_tail

__device__ __forceinline__ bool less_di(double a, int64_t ia, double b, int64_t ib) {
    return a < b || (a == b && ia < ib);
}

// ---------------------------------------------------------------------------
// a0: zero-padded copy of the queries (pitch floats per row)
// ---------------------------------------------------------------------------
__global__ void k_prep_queries(const float *__restrict__ q, int64_t Qc, int D, int pitch, float *__restrict__ out) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= Qc * pitch) return;
    int64_t r = e / pitch;
    int c = (int)(e % pitch);
    out[e] = c < D ? q[r * D + c] : 0.0f;
}

// ---------------------------------------------------------------------------
// a1 + a2: one warp per (query, subspace)
// ---------------------------------------------------------------------------
// dist64 (sequential fma over the dims, S:App. A.1) of a query half held as
// doubles and a centroid: ((double)q_i - (double)c_i)^2 accumulated in order
__device__ __forceinline__ double dist64_qd(const double *__restrict__ q, const float *__restrict__ c, int n) {
    double s = 0.0;
    for (int i = 0; i < n; i++) {
        const double d = __dsub_rn(q[i], (double)c[i]);
        s = __fma_rn(d, d, s);
    }
    return s;
}

__global__ void __launch_bounds__(THREADS) k_probe(const float *__restrict__ qrot, int pitch, int64_t q0, int64_t Qc,
                                                    const float *__restrict__ cb, int M, int K, int dh,
                                                    const int32_t *__restrict__ gsize, int smem_gsize, int64_t budget,
                                                    int wk, uint32_t *__restrict__ act, int32_t *__restrict__ act_len,
                                                    int64_t *__restrict__ retrieved, int qpw, int smem_cb,
                                                    const ScreenOut *__restrict__ scr,
                                                    unsigned long long *__restrict__ probe_stats,
                                                    const int32_t *__restrict__ hoff) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int KK = K * K;
    const int m = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int32_t *gs = (int32_t *)sm;
    float *cbs = (float *)(sm + (smem_gsize ? ((KK * 4 + 15) & ~15) : 0));  // this subspace's 2 x K x dh (smem_cb)
    // staged codebook rows at an odd stride: the lanes of a warp (one centroid each)
    // read distinct banks in dist64
    const int cst = smem_cb ? (dh | 1) : dh;
    unsigned char *wbase = (unsigned char *)cbs + (smem_cb ? ((2 * K * cst * 4 + 15) & ~15) : 0);
    const int per_warp = ((4 * K + 2 * dh) * 8 + 3 * K + 15) & ~15;
    double *tmp = (double *)(wbase + warp * per_warp);  // 2K
    double *a = tmp + 2 * K, *b = a + K;
    double *qs = b + K;                                 // 2 dh: this query's two halves, as doubles
    unsigned char *pa = (unsigned char *)(qs + 2 * dh), *pb = pa + K, *col = pb + K;
    const int32_t *gsm = gsize + (int64_t)m * KK;
    const float *cbm = cb + (int64_t)m * 2 * K * dh;
    if (smem_gsize)
        for (int i = threadIdx.x; i < KK; i += THREADS) gs[i] = gsm[i];
    if (smem_cb)
        for (int i = threadIdx.x; i < 2 * K * dh; i += THREADS) cbs[(i / dh) * cst + i % dh] = cbm[i];
    __syncthreads();
    if (smem_gsize) gsm = gs;
    if (smem_cb) cbm = cbs;
    // dist64 of this query's half `side` to centroid c (exactly the oracle's order)
    auto half_dist = [&](int side, int c) -> double {
        return smem_cb ? dist64_qd(qs + side * dh, cbs + (side * K + c) * cst, dh)
                       : dist64_qd(qs + side * dh, cbm + (int64_t)(side * K + c) * cst, dh);
    };
    // every centroid exact, each half sorted by (delta, c) via ranks
    auto full_halves = [&]() {
        for (int side = 0; side < 2; side++)
            for (int c = lane; c < K; c += 32) tmp[side * K + c] = half_dist(side, c);
        __syncwarp();
        for (int side = 0; side < 2; side++) {
            const double *t = tmp + side * K;
            double *dst = side ? b : a;
            unsigned char *pdst = side ? pb : pa;
            for (int c = lane; c < K; c += 32) {
                double v = t[c];
                int r = 0;
                for (int c2 = 0; c2 < K; c2++) {
                    double u = t[c2];
                    r += (u < v) || (u == v && c2 < c);
                }
                dst[r] = v;
                pdst[r] = (unsigned char)c;
            }
        }
        __syncwarp();
    };
    // each query: the (q, m) activated list, or false if the walk needs a rank at or past
    // the certified prefixes (ra, rb) of the half sorts (then the caller redoes it exactly)
    auto walk = [&](int64_t q, int ra, int rb) -> bool {
        for (int i = lane; i < K; i += 32) col[i] = 0;
        __syncwarp();
        // Multi-Sequence as a staircase argmin over (a_i + b_col[i], i)
        uint32_t *out = act + (q * M + m) * (int64_t)KK;
        int rank = 0;
        int64_t ret = 0;
        while (ret < budget && rank < KK) {
            double bc = INFINITY;
            int bi = 0x7fffffff;
            bool past = false;
            for (int i = lane; i < K; i += 32) {
                int ci = col[i];
                if (ci < K && (i == 0 || col[i - 1] > ci)) {
                    if (i >= ra || ci >= rb) {
                        past = true;
                        continue;
                    }
                    double cost = __dadd_rn(a[i], b[ci]);
                    if (cost < bc) {  // rows visited in ascending i: first wins ties
                        bc = cost;
                        bi = i;
                    }
                }
            }
            if (__any_sync(0xffffffffu, past)) return false;
            // warp argmin of (cost, i) by three 32-bit min reductions: the costs are
            // non-negative doubles (sums of dist64 values, or +inf), whose bit patterns order
            // as unsigned integers: min of the high words, then of the low words among the
            // lanes at that high word, then the smallest i among the lanes at that cost
            {
                const unsigned long long cb = (unsigned long long)__double_as_longlong(bc);
                const unsigned hi = (unsigned)(cb >> 32), lo = (unsigned)cb;
                const unsigned mh = __reduce_min_sync(0xffffffffu, hi);
                const unsigned ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
                const bool at = hi == mh && lo == ml;
                bi = (int)__reduce_min_sync(0xffffffffu, at ? (unsigned)bi : 0x7fffffffu);
                bc = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
            }
            const int j = col[bi];
            const int cell = pa[bi] * K + pb[j];
            rank++;
            const int w = (wk > 0 && rank <= wk) ? 2 : 1;  // Alg. 1 l.10-12
            __syncwarp();
            if (lane == 0) {
                out[rank - 1] = (uint32_t)cell | ((uint32_t)w << 16);
                col[bi] = (unsigned char)(j + 1);
            }
            ret += gsm[cell];
            __syncwarp();
        }
        if (lane == 0) {
            act_len[q * M + m] = rank;
            retrieved[q * M + m] = ret;
        }
        __syncwarp();
        return true;
    };
    unsigned long long n_exact = 0, n_redo = 0;
    // each warp takes qpw queries in turn (the codebooks and sizes staged once per CTA)
    for (int qi = 0; qi < qpw; qi++) {
        const int64_t q = q0 + ((int64_t)blockIdx.x * WARPS + warp) * qpw + qi;  // queries [q0, Qc)
        if (q >= Qc) break;
        if (hoff) {  // adaptive widths (R18): each half's dims, zero beyond its width (exact zero terms)
            for (int i = lane; i < 2 * dh; i += 32) {
                const int h = 2 * m + (i >= dh), t = i - (i >= dh ? dh : 0);
                qs[i] = t < hoff[h + 1] - hoff[h] ? (double)qrot[q * pitch + hoff[h] + t] : 0.0;
            }
        } else {
            const float *qm = qrot + q * pitch + (int64_t)m * 2 * dh;
            for (int i = lane; i < 2 * dh; i += 32) qs[i] = (double)qm[i];
        }
        __syncwarp();
        if (scr) {
            // a1 screened (probe_tc.cu): per half, t = the RQ-th smallest certified upper bound
            // and the mask of the centroids whose lower bound is <= t -- the only ones that can
            // be among the RQ smallest dist64 values; dist64 runs for them alone, and those with
            // dist64 <= t are, in (delta, c) order, exactly the first r of the full sort (every
            // other centroid has dist64 > t)
            int rr[2];
            for (int side = 0; side < 2; side++) {
                const ScreenOut so = scr[(q - q0) * 2 * M + 2 * m + side];
                const unsigned long long mk = so.mask;
                const double t = (double)so.t;
                const int S = __popcll(mk);
                // the members, listed in ascending c (col[] is scratch until the walk)
                for (int c = lane; c < K; c += 32)
                    if ((mk >> c) & 1ull) col[__popcll(mk & ((1ull << c) - 1ull))] = (unsigned char)c;
                __syncwarp();
                double *tt = tmp + side * K;
                for (int i = lane; i < S; i += 32) tt[i] = half_dist(side, col[i]);
                __syncwarp();
                double *dst = side ? b : a;
                unsigned char *pdst = side ? pb : pa;
                int nval = 0;
                for (int i = lane; i < S; i += 32) {
                    const double v = tt[i];
                    const int c = col[i];
                    int r = 0;
                    for (int i2 = 0; i2 < S; i2++) {  // members in ascending c: ties by c = by i2
                        const double u = tt[i2];
                        r += (u < v) || (u == v && i2 < i);
                    }
                    dst[r] = v;
                    pdst[r] = (unsigned char)c;
                    nval += v <= t;
                }
                n_exact += (lane == 0) ? S : 0;
                __syncwarp();
                for (int off = 16; off; off >>= 1) nval += __shfl_xor_sync(0xffffffffu, nval, off);
                rr[side] = nval;
                __syncwarp();
            }
            if (walk(q, rr[0], rr[1])) continue;
            n_redo++;
        }
        full_halves();
        if (scr) n_exact += (lane == 0) ? 2 * K : 0;
        walk(q, K, K);
    }
    if (probe_stats) {
        for (int off = 16; off; off >>= 1) n_exact += __shfl_xor_sync(0xffffffffu, n_exact, off);
        if (lane == 0) {
            atomicAdd(probe_stats, n_exact);
            atomicAdd(probe_stats + 1, n_redo);
        }
    }
}

// ---------------------------------------------------------------------------
// a3: collision counting into on-chip byte counters.  A CTA owns one query and a
// run of BPC consecutive id blocks of BS ids.  The query's activated cells
// (all subspaces) are cached once in shared memory; for each block their CSR
// slices restricted to the block are flattened (off2 offsets, prefetched one
// block ahead), the ids of a window of positions are staged into shared memory
// with coalesced independent loads (one memory latency per window), and then
// applied subspace by subspace as plain byte read-modify-writes with a barrier
// between subspaces: inside one subspace an id occurs at most once (the CSR
// partition property), so no atomics are needed.
// ---------------------------------------------------------------------------
constexpr int CS_EPT = CS_CAP / THREADS;  // table entries per thread
constexpr uint32_t WFLAG = 0x80000000u;   // weight-2 flag (Alg. 1 l.10-12)

struct CountSmem {
    uint32_t erow[CS_CAP];     // cached entries: (m*KK + cell) | WFLAG
    int32_t gst[CS_CAP];       // per block: ids[] index of the slice start | WFLAG
    int32_t pre[CS_CAP + 1];   // exclusive prefix of slice lengths
    int32_t pos[CS_TCAP];      // window: ids[] index | WFLAG, then local id | WFLAG
    int32_t lpre[MAX_M + 2];   // prefix of act_len over m
    int32_t mps[MAX_M + 1], mpe[MAX_M + 1];  // per-window position range of each subspace
    int32_t wtot[WARPS];
    int32_t base;
    typename cub::BlockScan<int, THREADS>::TempStorage scan;
};

// bank swizzle of the staged window positions (k_count_select)
__device__ __forceinline__ int pos_swz(int p) { return p ^ ((p >> 4) & 15); }

__device__ __forceinline__ int m_of_entry(const int32_t *lpre, int M, int e) {
    int lo = 0, hi = M;  // largest m with lpre[m] <= e
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (lpre[mid] <= e) lo = mid;
        else hi = mid;
    }
    return lo;
}

// lpre and (if they fit) the cached entries of query q; returns Etot
__device__ int count_setup(CountSmem &S, int64_t q, const uint32_t *__restrict__ act,
                           const int32_t *__restrict__ act_len, int M, int KK) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        int acc = 0;
        for (int m0 = 0; m0 < M; m0 += 32) {
            const int m = m0 + lane;
            int v = m < M ? __ldg(act_len + q * M + m) : 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                int t = __shfl_up_sync(0xffffffffu, v, off);
                if (lane >= off) v += t;
            }
            if (m < M) S.lpre[m + 1] = acc + v;
            acc += __shfl_sync(0xffffffffu, v, 31);
        }
        if (lane == 0) S.lpre[0] = 0;
    }
    __syncthreads();
    const int Etot = S.lpre[M];
    if (Etot <= CS_CAP) {
        const uint32_t *actq = act + q * (int64_t)M * KK;
        for (int t = tid; t < Etot; t += THREADS) {
            const int m = m_of_entry(S.lpre, M, t);
            const uint32_t v = __ldg(actq + (int64_t)m * KK + (t - S.lpre[m]));
            S.erow[t] = (uint32_t)(m * KK + (int)(v & 0xffffu)) | ((v >> 16) == 2u ? WFLAG : 0u);
        }
    }
    __syncthreads();
    return Etot;
}

__device__ __forceinline__ uint32_t entry_of(const CountSmem &S, int e, bool cached, const uint32_t *__restrict__ act,
                                             int64_t q, int M, int KK) {
    if (cached) return S.erow[e];
    const int m = m_of_entry(S.lpre, M, e);
    const uint32_t v = __ldg(act + q * (int64_t)M * KK + (int64_t)m * KK + (e - S.lpre[m]));
    return (uint32_t)(m * KK + (int)(v & 0xffffu)) | ((v >> 16) == 2u ? WFLAG : 0u);
}

// Count block b of query q into the zeroed counters.  s0r/s1r: off2 values of
// this block for the thread's cached entries (cached case), refilled for nb.
// If cross != nullptr, the ids whose count crosses tau (old < tau <= new; a
// count only grows, so each id crosses at most once) are flagged in the bitmap.
__device__ void count_one_block(CountSmem &S, unsigned char *cnt8, int BS, int64_t q, int b, int nb, int Etot,
                                const uint32_t *__restrict__ act, int M, int KK, const int32_t *__restrict__ off2,
                                int NB, const int32_t *__restrict__ ids, int64_t N, int (&s0r)[CS_EPT],
                                int (&s1r)[CS_EPT], int tau, uint32_t *cross) {
    const int tid = threadIdx.x;
    const bool cached = Etot <= CS_CAP;
    const uint32_t bbase = (uint32_t)b * (uint32_t)BS;
    for (int e0 = 0; e0 < Etot; e0 += CS_CAP) {
        const int ne = min(CS_CAP, Etot - e0);
        int lens[CS_EPT];
#pragma unroll
        for (int u = 0; u < CS_EPT; u++) {
            const int t = tid * CS_EPT + u;
            lens[u] = 0;
            if (t < ne) {
                const uint32_t erw = entry_of(S, e0 + t, cached, act, q, M, KK);
                const int row = (int)(erw & ~WFLAG);
                int s0, s1;
                if (cached) {
                    s0 = s0r[u];
                    s1 = s1r[u];
                    if (nb >= 0) {  // prefetch the next block's offsets
                        const int32_t *o = off2 + (int64_t)row * (NB + 1) + nb;
                        s0r[u] = __ldg(o);
                        s1r[u] = __ldg(o + 1);
                    }
                } else {
                    const int32_t *o = off2 + (int64_t)row * (NB + 1) + b;
                    s0 = __ldg(o);
                    s1 = __ldg(o + 1);
                }
                S.gst[t] = (int32_t)((uint32_t)((int64_t)(row / KK) * N + s0) | (erw & WFLAG));
                lens[u] = s1 - s0;
            }
        }
        int pres[CS_EPT], T;
        cub::BlockScan<int, THREADS>(S.scan).ExclusiveSum(lens, pres, T);
#pragma unroll
        for (int u = 0; u < CS_EPT; u++) {
            const int t = tid * CS_EPT + u;
            if (t < ne) S.pre[t] = pres[u];
        }
        if (tid == 0) S.pre[ne] = T;
        __syncthreads();
        const int ma = m_of_entry(S.lpre, M, e0), mb = m_of_entry(S.lpre, M, e0 + ne - 1);
        for (int P0 = 0; P0 < T; P0 += CS_TCAP) {
            const int Wn = min(CS_TCAP, T - P0);
            // fill the window: position -> ids[] index (| weight flag).  Thread tid
            // takes the CS_U consecutive positions from tid*CS_U: a binary search
            // finds the entry of the first, then it walks forward (S.pos is
            // swizzled, pos_swz, so these writes and the strided reads below are
            // nearly conflict-free)
            {
                const int pa = tid * CS_U;
                if (pa < Wn) {
                    int t = 0, hi2 = ne;  // largest t with pre[t] <= P0 + pa
                    while (hi2 - t > 1) {
                        const int mid = (t + hi2) >> 1;
                        if (S.pre[mid] <= P0 + pa) t = mid;
                        else hi2 = mid;
                    }
                    int nxt = S.pre[t + 1], cur = S.pre[t], g = S.gst[t];
#pragma unroll 4
                    for (int i = 0; i < CS_U; i++) {
                        const int P = P0 + pa + i;
                        if (pa + i >= Wn) break;
                        while (nxt <= P) {
                            t++;
                            cur = nxt;
                            nxt = S.pre[t + 1];
                            g = S.gst[t];
                        }
                        S.pos[pos_swz(pa + i)] = g + (P - cur);
                    }
                }
            }
            __syncthreads();
            // stage the window's ids: independent coalesced loads
            {
                int v[CS_U], idv[CS_U];
#pragma unroll
                for (int u = 0; u < CS_U; u++) {
                    const int p = tid + u * THREADS;
                    v[u] = p < Wn ? S.pos[pos_swz(p)] : 0;
                }
#pragma unroll
                for (int u = 0; u < CS_U; u++) {
                    const int p = tid + u * THREADS;
                    idv[u] = p < Wn ? __ldg(ids + ((uint32_t)v[u] & ~WFLAG)) : 0;
                }
#pragma unroll
                for (int u = 0; u < CS_U; u++) {
                    const int p = tid + u * THREADS;
                    if (p < Wn) S.pos[pos_swz(p)] = (int32_t)(((uint32_t)idv[u] - bbase) | ((uint32_t)v[u] & WFLAG));
                }
            }
            if (tid <= mb - ma) {  // window position range of each subspace
                const int m = ma + tid;
                const int ea = max(S.lpre[m], e0) - e0, eb = min(S.lpre[m + 1], e0 + ne) - e0;
                S.mps[tid] = max(S.pre[ea], P0) - P0;
                S.mpe[tid] = min(S.pre[eb], P0 + Wn) - P0;
            }
            __syncthreads();
            // subspace by subspace: plain byte RMW, barrier between subspaces
            for (int mi = 0; mi <= mb - ma; mi++) {
                const int pe = S.mpe[mi];
                for (int p = S.mps[mi] + tid; p < pe; p += THREADS) {
                    const uint32_t x = (uint32_t)S.pos[pos_swz(p)];
                    const uint32_t local = x & ~WFLAG;
                    const int old = cnt8[local];
                    const int nw = old + 1 + (int)(x >> 31);
                    cnt8[local] = (unsigned char)nw;
                    if (cross && old < tau && nw >= tau) atomicOr(cross + (local >> 5), 1u << (local & 31));
                }
                __syncthreads();
            }
        }
        if (T == 0) __syncthreads();
    }
}

__device__ __forceinline__ void zero_counters(unsigned char *cnt8, int BS) {
    for (int i = threadIdx.x; i < BS / 16; i += THREADS) ((uint4 *)cnt8)[i] = make_uint4(0, 0, 0, 0);
}

__device__ __forceinline__ void prefetch_first(const CountSmem &S, int Etot, const int32_t *__restrict__ off2, int NB,
                                               int b, int (&s0r)[CS_EPT], int (&s1r)[CS_EPT]) {
    if (Etot > CS_CAP) return;
#pragma unroll
    for (int u = 0; u < CS_EPT; u++) {
        const int t = threadIdx.x * CS_EPT + u;
        if (t < Etot) {
            const int32_t *o = off2 + (int64_t)(S.erow[t] & ~WFLAG) * (NB + 1) + b;
            s0r[u] = __ldg(o);
            s1r[u] = __ldg(o + 1);
        }
    }
}

// a3 + a4 for BPC blocks of one query; candidates go to the query's pool
// region at a per-block base taken from an atomic cursor (blocks keep their
// ascending-id order inside; consumers enumerate blocks in ascending order).
__global__ void __launch_bounds__(THREADS, 4) k_count_select(const uint32_t *__restrict__ act,
                                                           const int32_t *__restrict__ act_len, int M, int KK,
                                                           const int32_t *__restrict__ off2, int NB,
                                                           const int32_t *__restrict__ ids, int64_t N, int BS, int BPC,
                                                           int tau, int32_t *__restrict__ pool, int64_t CAPQ,
                                                           int32_t *__restrict__ cursor, int32_t *__restrict__ cbase,
                                                           int32_t *__restrict__ ncand, int32_t *__restrict__ need,
                                                           uint8_t *__restrict__ traceV,
                                                           const int32_t *__restrict__ qperm) {
    extern __shared__ __align__(16) unsigned char smraw[];
    unsigned char *cnt8 = smraw;
    uint32_t *cross = (uint32_t *)(smraw + BS);            // BS bits
    CountSmem &S = *(CountSmem *)(smraw + BS + BS / 8);
    const int64_t q = qperm ? qperm[blockIdx.y] : blockIdx.y;  // locality order (query_order)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int b_lo = blockIdx.x * BPC, b_hi = min(NB, b_lo + BPC);
    const int Etot = count_setup(S, q, act, act_len, M, KK);
    int s0r[CS_EPT], s1r[CS_EPT];
    prefetch_first(S, Etot, off2, NB, b_lo, s0r, s1r);
    const int wwords = BS / 256;  // bitmap words per warp
    for (int b = b_lo; b < b_hi; b++) {
        zero_counters(cnt8, BS + BS / 8);
        __syncthreads();
        count_one_block(S, cnt8, BS, q, b, b + 1 < b_hi ? b + 1 : -1, Etot, act, M, KK, off2, NB, ids, N, s0r, s1r,
                        tau, cross);
        // a4: C = {x : V[x] >= tau} (Alg. 1 l.18), ascending id: the crossing
        // bitmap holds exactly those ids; each warp compacts its word range
        int cw = 0;
        for (int i = lane; i < wwords; i += 32) cw += __popc(cross[warp * wwords + i]);
#pragma unroll
        for (int off = 16; off; off >>= 1) cw += __shfl_xor_sync(0xffffffffu, cw, off);
        if (lane == 0) S.wtot[warp] = cw;
        __syncthreads();
        if (tid == 0) {
            int n = 0;
            for (int w2 = 0; w2 < WARPS; w2++) n += S.wtot[w2];
            const int base = atomicAdd(cursor + q, n);
            S.base = base;
            cbase[q * NB + b] = base;
            ncand[q * NB + b] = n;
            if ((int64_t)base + n > CAPQ) atomicMax(need, base + n);
        }
        __syncthreads();
        int running = S.base;
        for (int w2 = 0; w2 < warp; w2++) running += S.wtot[w2];
        int32_t *outp = pool + q * CAPQ;
        for (int i0 = 0; i0 < wwords; i0 += 32) {
            const int i = i0 + lane;
            uint32_t word = i < wwords ? cross[warp * wwords + i] : 0u;
            const int c = __popc(word);
            int inc = c;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                int t = __shfl_up_sync(0xffffffffu, inc, off);
                if (lane >= off) inc += t;
            }
            int o = running + inc - c;
            const int g0 = b * BS + (warp * wwords + i) * 32;
            while (word) {
                const int bit = __ffs(word) - 1;
                if (o < CAPQ) outp[o] = g0 + bit;
                o++;
                word &= word - 1;
            }
            running += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (traceV) {
            for (int j = tid; j < BS; j += THREADS)
                if ((int64_t)b * BS + j < N) traceV[q * N + (int64_t)b * BS + j] = cnt8[j];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// a3 + a4, warp-owned counters (default).  Each warp owns the SBW = BS/8 byte
// counters of one sub-block of ids and streams that sub-block's part of every
// activated slice (off2w offsets) on its own: no CTA barrier after setup, no
// staging through shared memory.  A warp walks the slices in activation order
// (subspace-major) in batches of 32 consecutive positions of ONE slice, so
// the lanes of a batch hit distinct counters and plain byte read-modify-
// writes suffice; __syncwarp orders consecutive batches (an id recurs only
// across subspaces, CSR partition property).  The (slice, offset)
// walk is a warp-uniform state machine; the id loads of CW_U batches are in
// flight before their read-modify-writes.
// a4 (C = {x : V[x] >= tau}, Alg. 1 l.18) is taken at the read-modify-write:
// V only grows, by 1 or 2, so x enters C exactly once, at the increment that
// lifts V[x] from below tau to tau or more; that increment sets x's bit in the
// warp's candidate bitmap (SBW bits).  After the sub-block the warp reads the
// bitmap in ascending id (its own candidate segment, base from an atomic
// cursor) and re-zeroes counters and bitmap; the counters are not scanned.
// ---------------------------------------------------------------------------
constexpr int CW_U = 4;  // 32-position batches with loads in flight per warp (k_count_warp)
constexpr uint32_t CW_EMASK = 0xffffffu;  // cached entry: (m*KK + cell) | m << 24 | WFLAG
struct CountWSmem {
    uint32_t erow[CS_CAP];
    int32_t lpre[MAX_M + 2];
    int next;               // next sub-block task of the CTA (dynamic: warps stay balanced)
};
__host__ __device__ constexpr size_t countw_fixed_smem(int BS) {  // counters + dummy, bitmaps, CountWSmem
    return (size_t)BS + 16 + (size_t)BS / 8 + ((sizeof(CountWSmem) + 15) & ~(size_t)15);
}

__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t cw_entry(const uint32_t *__restrict__ actq, const int32_t *lpre, int M, int KK,
                                             int e) {
    const int m = m_of_entry(lpre, M, e);
    const uint32_t v = __ldg(actq + (int64_t)m * KK + (e - lpre[m]));
    return (uint32_t)(m * KK + (int)(v & 0xffffu)) | ((uint32_t)m << 24) | ((v >> 16) == 2u ? WFLAG : 0u);
}

template <bool HAM, bool ATOM>
__global__ void __launch_bounds__(THREADS, HAM ? 4 : 5) k_count_warp(const uint32_t *__restrict__ act,
                                                           const int32_t *__restrict__ act_len, int M, int KK,
                                                           const int32_t *__restrict__ off2w, int NBW,
                                                           const int32_t *__restrict__ ids, int64_t N, int BS, int BPC,
                                                           int NB, int tau, int32_t *__restrict__ pool, int64_t CAPQ,
                                                           int32_t *__restrict__ cursor, int32_t *__restrict__ cbase,
                                                           int32_t *__restrict__ ncand, int32_t *__restrict__ need,
                                                           uint8_t *__restrict__ traceV, const float *__restrict__ qrot,
                                                           int pitch, int Dp, const uint64_t *__restrict__ codes,
                                                           int Wd, uint16_t *__restrict__ hbuf,
                                                           int32_t *__restrict__ ghist,
                                                           const int32_t *__restrict__ qperm) {
    extern __shared__ __align__(16) unsigned char smraw[];
    unsigned char *cnt8 = smraw;  // BS byte counters (+16 dummy bytes); warp w owns [w*SBW, (w+1)*SBW)
    uint32_t *bm = (uint32_t *)(smraw + BS + 16);  // candidate bitmaps: warp w owns words [w*SBW/32, +SBW/32)
    CountWSmem &S = *(CountWSmem *)(smraw + BS + 16 + BS / 8);
    // phi=1 (hbuf != null): b(q') and the query's Hamming histogram of this CTA
    uint64_t *qc = (uint64_t *)(smraw + countw_fixed_smem(BS));  // Wd
    int *hist = (int *)(qc + Wd);                                 // Dp + 1
    const int64_t q = qperm ? qperm[blockIdx.y] : blockIdx.y;  // locality order (query_order)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int SBW = BS >> 3, NWW = SBW >> 5;  // counters / bitmap words per warp
    const int b_lo = blockIdx.x * BPC, b_hi = min(NB, b_lo + BPC);
    unsigned char *wc = cnt8 + warp * SBW;
    uint32_t *wbm = bm + warp * NWW;
    const uint32_t sm_cnt = (uint32_t)__cvta_generic_to_shared(cnt8);
    const uint32_t sm_dummy = sm_cnt + (uint32_t)BS;
    // lpre (exclusive prefix of act_len over m) and the cached entries
    if (warp == 0) {
        int acc = 0;
        for (int m0 = 0; m0 < M; m0 += 32) {
            const int m = m0 + lane;
            int v = m < M ? __ldg(act_len + q * M + m) : 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, v, off);
                if (lane >= off) v += t;
            }
            if (m < M) S.lpre[m + 1] = acc + v;
            acc += __shfl_sync(0xffffffffu, v, 31);
        }
        if (lane == 0) {
            S.lpre[0] = 0;
            S.next = 0;
        }
    }
    // counters, the dummy counter (padding lanes add 0 to it) and the bitmaps
    for (int i = tid; i < (BS + 16 + BS / 8) / 16; i += THREADS) ((uint4 *)cnt8)[i] = make_uint4(0, 0, 0, 0);
    if (HAM && hbuf) {
        const float *qrow = qrot + q * pitch;
        for (int d0 = warp * 32; d0 < Wd * 64; d0 += THREADS) {  // bit (i mod 64) of word i/64 = [q'_i > 0] (Z10)
            const int d = d0 + lane;
            const unsigned bits = __ballot_sync(0xffffffffu, d < Dp && qrow[d] > 0.0f);
            if (lane == 0) ((uint32_t *)qc)[d0 >> 5] = bits;
        }
        for (int i = tid; i < Dp + 1; i += THREADS) hist[i] = 0;
    }
    __syncthreads();
    const int Etot = S.lpre[M];
    const uint32_t *actq = act + q * (int64_t)M * KK;
    const bool cached = Etot <= CS_CAP && (int64_t)M * KK <= (int64_t)CW_EMASK + 1;
    if (cached)
        for (int t = tid; t < Etot; t += THREADS) S.erow[t] = cw_entry(actq, S.lpre, M, KK, t);
    __syncthreads();
    const int nchunk = SBW / 512;  // 16-byte lane chunks of the warp's counters (SBW <= 4096: <= 8)
    const uint32_t taum1 = (uint32_t)tau - 1u;
    int32_t *outp = pool + q * CAPQ;
    const int ntask = (b_hi - b_lo) * 8;
    for (;;) {
        // next sub-block of the CTA's run (any warp may take any: its own counters)
        int t = 0;
        if (lane == 0) t = atomicAdd(&S.next, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= ntask) break;
        const int sb = b_lo * 8 + t;
        const int sbase = sb * SBW;                                      // first id of the sub-block
        const uint32_t lbase = (uint32_t)sbase - (uint32_t)(warp * SBW);  // id - lbase: this warp's counter
        if ((int64_t)sbase < N) {
            for (int e0 = 0; e0 < Etot; e0 += 32) {
                // this lane's entry: slice of the sub-block (ids[] start g, length len), weight flag
                const int e = e0 + lane;
                uint32_t wf = 0;
                int len = 0, g = 0;
                if (e < Etot) {
                    const uint32_t er = cached ? S.erow[e] : cw_entry(actq, S.lpre, M, KK, e);
                    const int32_t *o = off2w + (int64_t)(er & CW_EMASK) * (NBW + 1) + sb;
                    const int s0 = __ldg(o), s1 = __ldg(o + 1);
                    len = s1 - s0;
                    g = (int)((er >> 24) & 127u) * (int)N + s0;
                    wf = er >> 31;
                }
                uint32_t rest = __ballot_sync(0xffffffffu, len > 0);  // slices still to walk
                // warp-uniform walk state: current slice (start G, length L, flag F), offset p
                int G = 0, L = 0, p = 0;
                uint32_t F = 0;
                if (rest) {
                    const int j = __ffs(rest) - 1;
                    rest &= rest - 1;
                    G = __shfl_sync(0xffffffffu, g, j);
                    L = __shfl_sync(0xffffffffu, len, j);
                    F = __shfl_sync(0xffffffffu, wf, j);
                }
                while (L > 0) {
                    uint32_t xa[CW_U], xi[CW_U];
#pragma unroll
                    for (int u = 0; u < CW_U; u++) {
                        const bool ok = p + lane < L;
                        // unconditional load (past the slice end: its first id) so that no
                        // branch joins on the result and all CW_U loads are in flight
                        xa[u] = (uint32_t)__ldg(ids + (uint32_t)(G + (ok ? p + lane : 0)));
                        xi[u] = ok ? 1u + F : 0u;  // increment: the weight (Alg. 1 l.10-12); 0 = not a position
                        p += 32;
                        if (p >= L) {  // next slice (uniform)
                            p = 0;
                            L = 0;
                            if (rest) {
                                const int j = __ffs(rest) - 1;
                                rest &= rest - 1;
                                G = __shfl_sync(0xffffffffu, g, j);
                                L = __shfl_sync(0xffffffffu, len, j);
                                F = __shfl_sync(0xffffffffu, wf, j);
                            }
                        }
                    }
                    if (ATOM) {
                        // one shared atomic per position on the counter's 32-bit word (bytes
                        // never carry: V <= 2M <= 254); no ordering between batches needed
#pragma unroll
                        for (int u = 0; u < CW_U; u++)
                            if (xi[u]) {
                                const uint32_t off = xa[u] - (uint32_t)sbase, sh = (off & 3) * 8;
                                const uint32_t v =
                                    (atomicAdd((uint32_t *)(wc + (off & ~3u)), xi[u] << sh) >> sh) & 0xffu;
                                if (taum1 - v < xi[u]) atomicOr(wbm + (off >> 5), 1u << (off & 31));
                            }
                    } else {
#pragma unroll
                        for (int u = 0; u < CW_U; u++) {
                            const uint32_t a = xi[u] ? sm_cnt + (xa[u] - lbase) : sm_dummy;
                            const uint32_t v = lds_u8(a);
                            sts_u8(a, v + xi[u]);
                            if (taum1 - v < xi[u]) {  // v < tau <= v + inc: x enters C
                                const uint32_t off = xa[u] - (uint32_t)sbase;
                                atomicOr(wbm + (off >> 5), 1u << (off & 31));
                            }
                            __syncwarp();
                        }
                    }
                }
            }
        }
        // a4: read C in ascending id from the bitmap (lane l: words [l*wpl, (l+1)*wpl)),
        // re-zero bitmap and counters.
        if (traceV) {
            for (int i = 0; i < nchunk; i++) {
                const int64_t x0 = (int64_t)sbase + i * 512 + lane * 16;
                const unsigned char *vb = wc + i * 512 + lane * 16;
                for (int j = 0; j < 16; j++)
                    if (x0 + j < N) traceV[q * N + x0 + j] = vb[j];
            }
        }
#pragma unroll
        for (int i = 0; i < 8; i++)
            if (i < nchunk) *(uint4 *)(wc + i * 512 + lane * 16) = make_uint4(0, 0, 0, 0);
        const int wpl = NWW >= 32 ? NWW >> 5 : 1;  // 1, 2 or 4 (NWW in [16, 128])
        uint32_t bw[4] = {0, 0, 0, 0};
        if (lane * wpl < NWW) {
            uint32_t *pw = wbm + lane * wpl;
            if (wpl == 4) {
                const uint4 v = *(const uint4 *)pw;
                bw[0] = v.x, bw[1] = v.y, bw[2] = v.z, bw[3] = v.w;
                *(uint4 *)pw = make_uint4(0, 0, 0, 0);
            } else {
                for (int j = 0; j < wpl; j++) {
                    bw[j] = pw[j];
                    pw[j] = 0;
                }
            }
        }
        const int c = __popc(bw[0]) + __popc(bw[1]) + __popc(bw[2]) + __popc(bw[3]);
        int inc = c;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int tt = __shfl_up_sync(0xffffffffu, inc, off);
            if (lane >= off) inc += tt;
        }
        const int n = __shfl_sync(0xffffffffu, inc, 31);
        int base = 0;
        if (lane == 0) {
            base = atomicAdd(cursor + q, n);
            cbase[q * NBW + sb] = base;
            ncand[q * NBW + sb] = n;
            if ((int64_t)base + n > CAPQ) atomicMax(need, base + n);
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        int o = base + inc - c;
        const int g0 = sbase + lane * wpl * 32;
        if ((int64_t)base + n <= CAPQ) {
            // the segment fits (the usual case): two 64-bit words per lane, no bound check
            int32_t *dst = outp + o;
#pragma unroll
            for (int j = 0; j < 2; j++) {
                uint64_t word = (uint64_t)bw[2 * j] | ((uint64_t)bw[2 * j + 1] << 32);
                const int gj = g0 + j * 64 - 1;
                while (word) {
                    *dst++ = gj + __ffsll((long long)word);
                    word &= word - 1;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                uint32_t word = bw[j];
                while (word) {
                    if (o < CAPQ) outp[o] = g0 + j * 32 + __ffs(word) - 1;
                    o++;
                    word &= word - 1;
                }
            }
        }
        __syncwarp();
        if (HAM && hbuf && n > 0) {
            // a4, phi=1: h(x) = popcount(b(q') xor b(x)) (Alg. 1 l.19) of this segment's
            // candidates.  4 lanes per candidate, each lane 16-byte loads of its words
            // (code rows are Wd = 8j words); 32 candidates per pass, all loads in flight;
            // h is written at the candidate's pool position.
            __syncwarp();
            const int g4 = lane >> 2, gl = lane & 3, nt = Wd >> 3;
            for (int v0 = 0; v0 < n; v0 += 32) {
                int pos[4], id[4];
                bool okv[4];
#pragma unroll
                for (int r = 0; r < 4; r++) {
                    const int vi = v0 + r * 8 + g4;
                    pos[r] = base + vi;
                    okv[r] = vi < n && pos[r] < CAPQ;
                    id[r] = okv[r] ? outp[pos[r]] : 0;
                }
                int hr[4] = {0, 0, 0, 0};
#pragma unroll 2
                for (int t = 0; t < nt; t++) {
                    const int wd = 2 * gl + 8 * t;
                    const uint64_t q0 = qc[wd], q1 = qc[wd + 1];
                    ulonglong2 cw[4];
#pragma unroll
                    for (int r = 0; r < 4; r++)
                        cw[r] = __ldg((const ulonglong2 *)(codes + (int64_t)id[r] * Wd + wd));
#pragma unroll
                    for (int r = 0; r < 4; r++) hr[r] += __popcll(q0 ^ cw[r].x) + __popcll(q1 ^ cw[r].y);
                }
                // sum over the 4 lanes of a candidate; two candidates per word (h <= 65535)
                uint32_t p01 = (uint32_t)hr[0] | ((uint32_t)hr[1] << 16), p23 = (uint32_t)hr[2] | ((uint32_t)hr[3] << 16);
                p01 += __shfl_xor_sync(0xffffffffu, p01, 1);
                p23 += __shfl_xor_sync(0xffffffffu, p23, 1);
                p01 += __shfl_xor_sync(0xffffffffu, p01, 2);
                p23 += __shfl_xor_sync(0xffffffffu, p23, 2);
                if (gl == 0) {
                    const int hh[4] = {(int)(p01 & 0xffffu), (int)(p01 >> 16), (int)(p23 & 0xffffu), (int)(p23 >> 16)};
#pragma unroll
                    for (int r = 0; r < 4; r++)
                        if (okv[r]) {
                            hbuf[q * CAPQ + pos[r]] = (uint16_t)hh[r];
                            atomicAdd(&hist[hh[r]], 1);
                        }
                }
            }
        }
    }
    if (HAM && hbuf) {
        __syncthreads();
        int32_t *gh = ghist + q * (int64_t)(Dp + 1);
        for (int i = tid; i < Dp + 1; i += THREADS)
            if (hist[i]) atomicAdd(&gh[i], hist[i]);
    }
}

// ---------------------------------------------------------------------------
// a3 + a4, fragment-flattened counting (the small-cell regime: many activated
// cells per query, each contributing a short run of ids to every id block).
// A CTA owns one query and one id block of BF = F*BS ids, whose V counters
// (bytes, packed four to a 32-bit word) live in shared memory.  For a chunk of
// the query's activated cells (k_act_rows lists them per query) it stages each
// cell's fragment inside the block -- [off2[c][F b], off2[c][F b + F]) of the
// subspace's CSR ids, which holds exactly the cell's ids in the
// block -- drops the empty ones and takes an exclusive prefix of their counts
// of 16-byte quads of ids[] (aligned to absolute positions 4j).  Each warp
// takes an equal share of the chunk's quads; a lane takes one quad per step
// (one 16-byte load), finds its fragment with a 5-step shuffle search over a
// sliding window of 32 fragments held in the lanes, masks the edge words
// outside the fragment, and adds the weight w (Alg. 1 l.10-12) of each of its
// ids with a shared reduction on the counter's word.  The same id can recur only
// across subspaces (CSR partition property) and the reductions order
// those, so no barrier separates subspaces.  After the last chunk a SWAR scan
// of the counters sets the bit of every x with V[x] >= tau (C, Alg. 1 l.18) in
// the candidate bitmap, which the CTA finally writes out in ascending id.
// (CRISP_COUNT_SWAR=0: atomics with return; V only grows, by 1 or 2, so x enters
// C exactly at the increment that lifts its count from below tau to tau or
// more, and that increment sets x's bit.  Measured in round 2: 17.1 / 86.1 /
// 32.4 ms at cfg4/3/5 against 16.9 / 81.2 / 29.5 ms with the scan.  A variant
// that expanded each chunk into a table of one descriptor per quad instead of
// the shuffle search measured 18.4 ms at cfg4: the expansion's imbalanced
// per-thread loops cost what the search saved; profiles/r02_ncu_count_cfg4_s3.json.)
// ---------------------------------------------------------------------------
constexpr int CF_CAP = CRISP_CF_CAP;  // fragments staged per chunk
#ifndef CRISP_COUNT_LAG
#define CRISP_COUNT_LAG 0
#endif
constexpr bool CF_LAG = CRISP_COUNT_LAG != 0;
#ifndef CRISP_COUNT_REDUX
#define CRISP_COUNT_REDUX 1  // the fragment search by one warp OR-reduction (0: 5-step shuffle search)
#endif
constexpr bool CF_REDUX = CRISP_COUNT_REDUX != 0;
constexpr int CF_MAXW = 32;   // warps per CTA: 16 (two CTAs per SM, F <= 2) or 32 (one CTA per SM, F = 4)

struct CountFSmem {
    int4 tab[CF_CAP + 40];  // staged non-empty fragments (quad prefix, first quad, first position | WFLAG, end); padded
    long long wtot64[CF_MAXW];
    int32_t wtot[CF_MAXW];
    int next, base;
    uint64_t qc[64];  // b(q'), phi=1 fused Hamming (D' <= 4096)
};
// counters (BF bytes), candidate bitmap (BF bits), 32 dummy words (the atomics of
// lanes without an id), CountFSmem
__host__ __device__ constexpr size_t countf_smem(int BF) {
    return (size_t)BF + (size_t)BF / 8 + 128 + ((sizeof(CountFSmem) + 15) & ~(size_t)15);
}

__device__ __forceinline__ uint32_t atom_add_sh(uint32_t a, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
    return old;
}
// the same without a compiler memory barrier (the count loop's other shared accesses are
// reads of the staged table, which no atomic touches)
__device__ __forceinline__ uint32_t atom_add_sh_nc(uint32_t a, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v));
    return old;
}
__device__ __forceinline__ void red_add_sh_nc(uint32_t a, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void red_add_sh(uint32_t a, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_or_sh(uint32_t a, uint32_t v) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// The activated cells of each query as one compact row of entries
// (m*KK + cell) | WFLAG (weight 2), in activation order, and their number:
// the count kernel's staging then reads a contiguous row.  One warp per query.
__global__ void k_act_rows(const uint32_t *__restrict__ act, const int32_t *__restrict__ act_len, int M, int KK,
                           int64_t Qc, uint32_t *__restrict__ erow, int32_t *__restrict__ etot) {
    const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (q >= Qc) return;
    const int lane = threadIdx.x & 31;
    const uint32_t *aq = act + q * (int64_t)M * KK;
    uint32_t *eq = erow + q * (int64_t)M * KK;
    int base = 0;
    for (int m = 0; m < M; m++) {
        const int L = __ldg(act_len + q * M + m);
        for (int r = lane; r < L; r += 32) {
            const uint32_t v = __ldg(aq + (int64_t)m * KK + r);
            eq[base + r] = (uint32_t)(m * KK + (int)(v & 0xffffu)) | ((v >> 16) == 2u ? WFLAG : 0u);
        }
        base += L;
    }
    if (lane == 0) etot[q] = base;
}

template <int CF_WARPS, bool SWAR = false>
__global__ void __launch_bounds__(CF_WARPS * 32, 32 / CF_WARPS) k_count_frag(const uint32_t *__restrict__ erow,
                                                               const int32_t *__restrict__ etot, int M, int KK,
                                                               const int32_t *__restrict__ off2, int NB, int F,
                                                               const int32_t *__restrict__ ids, int64_t N, int BS,
                                                               int NS, int tau, int32_t *__restrict__ pool,
                                                               int64_t CAPQ, int32_t *__restrict__ cursor,
                                                               int32_t *__restrict__ cbase,
                                                               int32_t *__restrict__ ncand, int32_t *__restrict__ need,
                                                               uint8_t *__restrict__ traceV,
                                                               const int32_t *__restrict__ qperm,
                                                               const float *__restrict__ qrot, int pitch, int Dp,
                                                               const uint64_t *__restrict__ codes, int Wd,
                                                               uint16_t *__restrict__ hbuf,
                                                               int32_t *__restrict__ ghist) {
    constexpr int CF_THREADS = CF_WARPS * 32;
    constexpr int CF_EPT = CF_CAP / CF_THREADS;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int BF = BS * F;
    uint32_t *cw = (uint32_t *)smraw;              // BF byte counters, 4 per word
    uint32_t *bm = (uint32_t *)(smraw + BF);       // BF-bit candidate bitmap
    CountFSmem &S = *(CountFSmem *)(smraw + BF + BF / 8 + 128);
    const uint32_t sm_cw = (uint32_t)__cvta_generic_to_shared(cw);
    const uint32_t sm_bm = sm_cw + (uint32_t)BF;
    const int64_t q = qperm ? qperm[blockIdx.y] : blockIdx.y;  // locality order (query_order)
    const int sb = blockIdx.x;                                 // id block [sb*BF, (sb+1)*BF)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t sm_dummy = sm_bm + (uint32_t)(BF / 8) + 4u * (uint32_t)lane;  // this lane's dummy word
    const uint32_t bbase = (uint32_t)sb * (uint32_t)BF;
    const uint32_t cw_rel = sm_cw - bbase;  // + (x & ~3): the counter word of id x (BF % 4 == 0)
    const int c0 = sb * F, c1 = min(NB, c0 + F);  // off2 columns bounding the block
    for (int i = tid; i < (BF + BF / 8 + 128) / 16; i += CF_THREADS) ((uint4 *)smraw)[i] = make_uint4(0, 0, 0, 0);
    const int Etot = __ldg(etot + q);
    const uint32_t *eq = erow + q * (int64_t)M * KK;
    if (hbuf && warp == 0) {
        const float *qrow = qrot + q * pitch;
        for (int d0 = 0; d0 < Wd * 64; d0 += 32) {  // bit (i mod 64) of word i/64 = [q'_i > 0] (Z10)
            const int d = d0 + lane;
            const unsigned bits = __ballot_sync(0xffffffffu, d < Dp && qrow[d] > 0.0f);
            if (lane == 0) ((uint32_t *)S.qc)[d0 >> 5] = bits;
        }
    }
    const uint32_t taum1 = (uint32_t)tau - 1u;
    __syncthreads();
    for (int e0 = 0; e0 < Etot; e0 += CF_CAP) {
        const int ne = min(CF_CAP, Etot - e0);
        // stage this chunk's fragments: warp w takes entries [w*32*CF_EPT, (w+1)*32*CF_EPT) of the
        // chunk, lane l the entries w*32*CF_EPT + 32u + l (coalesced entry loads, then the
        // off2 pairs, all in flight together), a warp scan of the packed (chunks,
        // non-empty) values, one barrier for the warp totals, the scatter of the non-empty
        // fragments (their order in the table is immaterial: the counts commute)
        const int W0 = warp * 32 * CF_EPT;
        uint32_t er[CF_EPT];
#pragma unroll
        for (int u = 0; u < CF_EPT; u++) {
            const int t = W0 + 32 * u + lane;
            er[u] = t < ne ? __ldg(eq + e0 + t) : 0xffffffffu;
        }
        int s0[CF_EPT], s1[CF_EPT];
#pragma unroll
        for (int u = 0; u < CF_EPT; u++) {
            const bool ok = er[u] != 0xffffffffu;
            const int32_t *o = off2 + (int64_t)(ok ? (er[u] & ~WFLAG) : 0u) * (NB + 1);
            s0[u] = ok ? __ldg(o + c0) : 0;
            s1[u] = ok ? __ldg(o + c1) : 0;
        }
        long long v[CF_EPT], ex[CF_EPT], carry = 0;
        const unsigned lemask_st = (2u << lane) - 1u;  // lanes <= this lane
        int g0[CF_EPT];  // absolute ids[] position of the fragment's first id
#pragma unroll
        for (int u = 0; u < CF_EPT; u++) {
            const int len = s1[u] - s0[u];
            g0[u] = (int)((er[u] & ~WFLAG) / (uint32_t)KK) * (int)N + s0[u];
            // the fragment's 16-byte quads of ids[] (aligned to absolute position 4j)
            const int nq = ((g0[u] + len + 3) >> 2) - (g0[u] >> 2);
            v[u] = len > 0 ? (((long long)nq << 16) | 1) : 0;
            // the packed (quads << 16 | non-empty) prefix from a 32-bit scan of the quads and a
            // ballot of the non-empty fragments (half the shuffles of a 64-bit scan)
            const int vq = len > 0 ? nq : 0;
            int x = vq;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, off);
                if (lane >= off) x += y;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, len > 0);
            ex[u] = carry + ((long long)(x - vq) << 16) + __popc(bal & (lemask_st >> 1));
            carry += ((long long)__shfl_sync(0xffffffffu, x, 31) << 16) + __popc(bal);
        }
        if (lane == 0) S.wtot64[warp] = carry;
        __syncthreads();
        long long wpre = 0, tot = 0;
        for (int w2 = 0; w2 < CF_WARPS; w2++) {
            const long long t = S.wtot64[w2];
            wpre += w2 < warp ? t : 0;
            tot += t;
        }
        const int NC = (int)(tot >> 16), nnz = (int)(tot & 0xffff);  // quads, non-empty fragments
#pragma unroll
        for (int u = 0; u < CF_EPT; u++)
            if (v[u]) {
                const long long xx = wpre + ex[u];
                // (quad prefix, first quad, first position | weight flag, end position)
                S.tab[(int)(xx & 0xffff)] = make_int4((int)(xx >> 16), g0[u] >> 2, (int)((uint32_t)g0[u] | (er[u] & WFLAG)),
                                                      g0[u] + s1[u] - s0[u]);
            }
        if (tid < 40) S.tab[nnz + tid] = make_int4(tid == 0 ? NC : 0x7fffffff, 0, 0, 0);
        __syncthreads();
        // Warp w takes the chunk's quads [w NC / W, (w+1) NC / W) (static, equal shares).  A lane
        // takes one quad per step (a 16-byte load of 4 consecutive ids[] words of one fragment,
        // edge words masked) and finds its fragment with a 5-step shuffle search over a window of
        // 32 consecutive fragments held in the lanes (quad prefixes strictly increase: no empty
        // fragments), which slides to the fragment of the step's last quad (32 quads span at
        // most 32 fragments).  Loads are software-pipelined (the next step's quad is in flight
        // while this step's atomics run); a lane without an id adds 0 to its own dummy word.
        // (Measured: the earlier dynamic tasks of 8 fragments cost about as many instructions per
        // task as the ~1.1 steps of quads a task holds.)
        const int Q0 = (int)((long long)NC * warp / CF_WARPS), Q1 = (int)((long long)NC * (warp + 1) / CF_WARPS);
        if (Q0 < Q1) {
            // the fragment holding quad Q0: the last f with tab[f].x <= Q0 (nnz <= CF_CAP = 32 x 32)
            int fb;
            {
                const int ci = lane * 32;
                const unsigned m1 = __ballot_sync(0xffffffffu, ci < nnz && S.tab[ci].x <= Q0);
                const int c = 31 - __clz(m1);  // bit 0 is set: tab[0].x = 0
                const int fi = c * 32 + lane;
                const unsigned m2 = __ballot_sync(0xffffffffu, fi < nnz && S.tab[fi].x <= Q0);
                fb = c * 32 + (31 - __clz(m2));
            }
            int4 te = S.tab[fb + lane];  // the table is padded past nnz (tab[nnz].x = NC, then +inf)
            uint4 qn;
            int gn0 = 0, gn1 = 0, qpn = 0;
            uint32_t wn = 0;
            const unsigned lemask = (2u << lane) - 1u;  // lanes <= this lane
            auto issue = [&](int pp) {
                const int p = pp + lane;
                int j = 0, jl = 0;
                if (CF_REDUX) {
                    // fragment fb holds quad pp; fragments fb+1.. start at distinct quads >= pp:
                    // OR their start offsets inside the step into one mask; lane l's fragment is
                    // fb + (number of starts at or before pp + l)
                    const int off = te.x - pp;
                    const unsigned starts =
                        __reduce_or_sync(0xffffffffu, (lane > 0 && off >= 0 && off < 32) ? (1u << off) : 0u);
                    j = __popc(starts & lemask);
                    jl = __popc(starts);
                } else {
#pragma unroll
                    for (int st = 16; st; st >>= 1) {
                        const int xv = __shfl_sync(0xffffffffu, te.x, j + st);
                        if (xv <= p) j += st;
                    }
                    jl = __shfl_sync(0xffffffffu, j, 31);
                }
                const int qx = __shfl_sync(0xffffffffu, te.x, j);
                const int qs = __shfl_sync(0xffffffffu, te.y, j);
                const int gw = __shfl_sync(0xffffffffu, te.z, j);
                const int ge = __shfl_sync(0xffffffffu, te.w, j);
                const bool ok = p < Q1;
                qpn = ok ? qs + (p - qx) : 0;
                gn0 = ok ? (int)((uint32_t)gw & ~WFLAG) : 1;
                gn1 = ok ? ge : 1;  // an empty range [1, 1) for lanes past Q1
                wn = 1u + ((uint32_t)gw >> 31);
                qn = __ldg((const uint4 *)ids + qpn);
                // slide the window to the fragment of this step's last quad
                if (jl > 0) {
                    fb += jl;
                    te = S.tab[fb + lane];
                }
            };
            issue(Q0);
            // CRISP_COUNT_LAG=1 (compile time) runs a step's crossing checks one step late, so that
            // its atomics' returns arrive while the next step's atomics issue: measured slower at
            // cfg4 (17.6 against 16.9 ms; 64 registers leave no room for the extra live values)
            uint32_t pov[4] = {0u, 0u, 0u, 0u}, pxs[4] = {0u, 0u, 0u, 0u}, pinc[4] = {0u, 0u, 0u, 0u};
            auto cross = [&](const uint32_t (&ov)[4], const uint32_t (&xs)[4], const uint32_t (&inc)[4]) {
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const uint32_t off = xs[e] - bbase;
                    const uint32_t o8 = (ov[e] >> ((off & 3u) * 8u)) & 0xffu;
                    if (taum1 - o8 < inc[e])  // o8 < tau <= o8 + inc: x enters C
                        red_or_sh(sm_bm + ((off >> 5) << 2), 1u << (off & 31));
                }
            };
            for (int pp = Q0; pp < Q1; pp += 32) {
                const uint4 qv = qn;
                const int q0 = qpn * 4, lo = gn0, hi = gn1;
                const uint32_t w = wn;
                if (pp + 32 < Q1) issue(pp + 32);
                const uint32_t xs[4] = {qv.x, qv.y, qv.z, qv.w};
                if constexpr (SWAR) {
                    // an element outside its fragment (quad edges, lanes past Q1) adds to the lane's
                    // dummy word (never read); bbase is a multiple of 4, so the counter word of x is
                    // sm_cw - bbase + (x & ~3) and its byte x & 3: the shift (x << 3) mod 32 by a
                    // wrapping funnel shift (89 instead of 99 instructions per step)
                    const int a = lo - q0, b = hi - q0;
#pragma unroll
                    for (int e = 0; e < 4; e++)
                        red_add_sh_nc(e >= a && e < b ? cw_rel + (xs[e] & ~3u) : sm_dummy,
                                      __funnelshift_l(0u, w, xs[e] << 3));
                } else {
                uint32_t ov[4], inc[4];
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const bool ok = q0 + e >= lo && q0 + e < hi;
                    inc[e] = ok ? w : 0u;
                    const uint32_t off = xs[e] - bbase;
                    ov[e] = atom_add_sh_nc(ok ? sm_cw + (off & ~3u) : sm_dummy, inc[e] << ((off & 3u) * 8u));
                }
                if (CF_LAG) {
                    cross(pov, pxs, pinc);
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        pov[e] = ov[e];
                        pxs[e] = xs[e];
                        pinc[e] = inc[e];
                    }
                } else {
                    cross(ov, xs, inc);
                }
                }
            }
            if (CF_LAG && !SWAR) cross(pov, pxs, pinc);
        }
        __syncthreads();  // the chunk's table is re-staged next
    }
    // a4: C in ascending id from the bitmap; warp w owns the contiguous bitmap words [w wpw, (w+1) wpw)
    const int nwords = BF / 32, wpw = nwords / CF_WARPS;  // wpw <= 128 (BF <= 131072 ids at 32 warps)
    uint32_t wr[4] = {0u, 0u, 0u, 0u};  // SWAR: this warp's words lane + 32 r, kept in registers
    if (SWAR) {
        // CRISP_COUNT_SWAR=1: the counts above are fire-and-forget reductions; C = {x : V[x] >= tau}
        // (Alg. 1 l.18) from the final counters (the chunk loop ended on a barrier), 32 per bitmap
        // word: bit 7 of ((c | 0x80) - tau) is [c >= tau] for c < 128 (M < 64), else a per-byte
        // compare; one multiply gathers a word's four flags.  Each warp scans the counters of its
        // own bitmap words and keeps them in registers for the listing below (no bitmap round trip
        // through shared memory, no barrier)
        const uint32_t t4 = (uint32_t)tau * 0x01010101u;
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const int wi = warp * wpw + lane + 32 * r;
            if (lane + 32 * r < wpw) {
                const uint4 a = ((const uint4 *)cw)[2 * wi], b = ((const uint4 *)cw)[2 * wi + 1];
                const uint32_t v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
                uint32_t word = 0u;
#pragma unroll
                for (int t = 0; t < 8; t++) {
                    const uint32_t f = M < 64 ? (((v[t] | 0x80808080u) - t4) >> 7) & 0x01010101u
                                              : __vcmpgeu4(v[t], t4) & 0x01010101u;
                    word |= ((f * 0x10204080u) >> 28) << (4 * t);
                }
                wr[r] = word;
            }
        }
    }
    {
        int c = 0;
        if (SWAR) {
#pragma unroll
            for (int r = 0; r < 4; r++) c += __popc(wr[r]);
        } else {
            for (int i = lane; i < wpw; i += 32) c += __popc(bm[warp * wpw + i]);
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
        if (lane == 0) S.wtot[warp] = c;
    }
    __syncthreads();
    if (tid == 0) {
        int n = 0;
        for (int w2 = 0; w2 < CF_WARPS; w2++) n += S.wtot[w2];
        const int base = atomicAdd(cursor + q, n);
        S.base = base;
        cbase[q * NS + sb] = base;
        ncand[q * NS + sb] = n;
        if ((int64_t)base + n > CAPQ) atomicMax(need, base + n);
    }
    __syncthreads();
    int running = S.base;
    for (int w2 = 0; w2 < warp; w2++) running += S.wtot[w2];
    int32_t *outp = pool + q * CAPQ;
#pragma unroll
    for (int r = 0; r < 4; r++) {
        const int i0 = 32 * r, i = i0 + lane;
        if (i0 >= wpw) break;
        uint32_t word = SWAR ? wr[r] : (i < wpw ? bm[warp * wpw + i] : 0u);
        const int c = __popc(word);
        int inc = c;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, off);
            if (lane >= off) inc += t;
        }
        int o = running + inc - c;
        const int g0 = (int)bbase + (warp * wpw + i) * 32;
        while (word) {
            if (o < CAPQ) outp[o] = g0 + __ffs(word) - 1;
            o++;
            word &= word - 1;
        }
        running += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (traceV) {
        const unsigned char *c8 = (const unsigned char *)cw;
        for (int j = tid; j < BF; j += CF_THREADS)
            if ((int64_t)bbase + j < N) traceV[q * N + (int64_t)bbase + j] = c8[j];
    }
    if (hbuf) {
        // a4, phi=1, fused: h(x) = popcount(b(q') xor b(x)) (Alg. 1 l.19) of this
        // block's candidates, right after they are listed (the count is issue-bound, so these
        // code-row streams overlap it).  4 lanes per candidate, 16-byte loads of its code row;
        // h at the candidate's pool position, the query's histogram of h by reductions.
        __syncthreads();  // the candidate ids in the pool, b(q') in shared memory
        int n = 0;
        for (int w2 = 0; w2 < CF_WARPS; w2++) n += S.wtot[w2];
        const int base = S.base;
        const int g4 = lane >> 2, gl = lane & 3, nt = Wd >> 3;
        int32_t *gh = ghist + q * (int64_t)(Dp + 1);
        for (int v0 = warp * 32; v0 < n; v0 += CF_WARPS * 32) {
            int pos[4], id[4];
            bool okv[4];
#pragma unroll
            for (int r = 0; r < 4; r++) {
                const int vi = v0 + r * 8 + g4;
                pos[r] = base + vi;
                okv[r] = vi < n && pos[r] < CAPQ;
                id[r] = okv[r] ? outp[pos[r]] : (int)bbase;
            }
            int hr[4] = {0, 0, 0, 0};
#pragma unroll 2
            for (int t = 0; t < nt; t++) {
                const int wd = 2 * gl + 8 * t;
                const uint64_t q0w = S.qc[wd], q1w = S.qc[wd + 1];
                ulonglong2 cwd[4];
#pragma unroll
                for (int r = 0; r < 4; r++) cwd[r] = __ldg((const ulonglong2 *)(codes + (int64_t)id[r] * Wd + wd));
#pragma unroll
                for (int r = 0; r < 4; r++) hr[r] += __popcll(q0w ^ cwd[r].x) + __popcll(q1w ^ cwd[r].y);
            }
            uint32_t p01 = (uint32_t)hr[0] | ((uint32_t)hr[1] << 16), p23 = (uint32_t)hr[2] | ((uint32_t)hr[3] << 16);
            p01 += __shfl_xor_sync(0xffffffffu, p01, 1);
            p23 += __shfl_xor_sync(0xffffffffu, p23, 1);
            p01 += __shfl_xor_sync(0xffffffffu, p01, 2);
            p23 += __shfl_xor_sync(0xffffffffu, p23, 2);
            if (gl == 0) {
                const int hh[4] = {(int)(p01 & 0xffffu), (int)(p01 >> 16), (int)(p23 & 0xffffu), (int)(p23 >> 16)};
#pragma unroll
                for (int r = 0; r < 4; r++)
                    if (okv[r]) {
                        hbuf[q * CAPQ + pos[r]] = (uint16_t)hh[r];
                        atomicAdd(&gh[hh[r]], 1);
                    }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// a4 fallback (Z8): |C| < k -> the first min(k,|T|) touched ids by
// (V desc, id asc), restated in ascending id.  Rare; one CTA per query,
// counting every block twice (histogram of V, then selection).  For a sharded
// index the decision (global |C|), the histogram (summed over shards) and the
// quota of ids with V == V* (given to shards in global-id order) are global.
// ---------------------------------------------------------------------------
__device__ void fb_hist_pass(CountSmem &S, unsigned char *cnt8, int BS, int64_t q, int Etot,
                             const uint32_t *__restrict__ act, int M, int KK, const int32_t *__restrict__ off2, int NB,
                             const int32_t *__restrict__ ids, int64_t N, int *hist) {
    const int tid = threadIdx.x;
    int s0r[CS_EPT], s1r[CS_EPT];
    for (int b = 0; b < NB; b++) {
        prefetch_first(S, Etot, off2, NB, b, s0r, s1r);
        zero_counters(cnt8, BS);
        __syncthreads();
        count_one_block(S, cnt8, BS, q, b, -1, Etot, act, M, KK, off2, NB, ids, N, s0r, s1r, 0, nullptr);
        for (int j = tid; j < BS; j += THREADS)
            if (cnt8[j]) atomicAdd(&hist[cnt8[j]], 1);
        __syncthreads();
    }
}

// selects ids with V > vstar and the first `quota` ids with V == vstar, in
// ascending id, into outp; returns the count (all threads)
__device__ int fb_select_pass(CountSmem &S, unsigned char *cnt8, int BS, int64_t q, int Etot,
                              const uint32_t *__restrict__ act, int M, int KK, const int32_t *__restrict__ off2,
                              int NB, const int32_t *__restrict__ ids, int64_t N, int vstar, int quota, int32_t *outp,
                              int *s_eqbase, int *s_n) {
    const int tid = threadIdx.x;
    int s0r[CS_EPT], s1r[CS_EPT];
    if (tid == 0) {
        *s_eqbase = 0;
        *s_n = 0;
    }
    __syncthreads();
    for (int b = 0; b < NB; b++) {
        prefetch_first(S, Etot, off2, NB, b, s0r, s1r);
        zero_counters(cnt8, BS);
        __syncthreads();
        count_one_block(S, cnt8, BS, q, b, -1, Etot, act, M, KK, off2, NB, ids, N, s0r, s1r, 0, nullptr);
        for (int j0 = 0; j0 < BS; j0 += THREADS * 16) {
            const int j = j0 + tid * 16;
            unsigned char vb[16];
#pragma unroll
            for (int i = 0; i < 16; i++) vb[i] = (j + i < BS) ? cnt8[j + i] : 0;
            int ceq = 0;
#pragma unroll
            for (int i = 0; i < 16; i++) ceq += vb[i] == vstar;
            int eoff, etot;
            cub::BlockScan<int, THREADS>(S.scan).ExclusiveSum(ceq, eoff, etot);
            __syncthreads();
            bool sel[16];
            int cs = 0, er = *s_eqbase + eoff;
#pragma unroll
            for (int i = 0; i < 16; i++) {
                sel[i] = vb[i] > vstar || (vb[i] == vstar && vb[i] > 0 && er < quota);
                if (vb[i] == vstar) er++;
                cs += sel[i];
            }
            int soff, stot;
            cub::BlockScan<int, THREADS>(S.scan).ExclusiveSum(cs, soff, stot);
            int o = *s_n + soff;
#pragma unroll
            for (int i = 0; i < 16; i++)
                if (sel[i]) outp[o++] = b * BS + j + i;
            __syncthreads();
            if (tid == 0) {
                *s_eqbase += etot;
                *s_n += stot;
            }
            __syncthreads();
        }
    }
    return *s_n;
}

// V* and the quota of ids with V == V* from a histogram of V over the touched set
__device__ __forceinline__ void fb_threshold(const int *hist, int M, int k, int *vstar, int *quota) {
    int acc = 0;
    *vstar = 1;
    *quota = hist[1];
    for (int v = 2 * M; v >= 1; v--) {
        if (acc + hist[v] >= k) {
            *vstar = v;
            *quota = k - acc;
            return;
        }
        acc += hist[v];
    }
}

__global__ void __launch_bounds__(THREADS) k_fallback(const uint32_t *__restrict__ act,
                                                       const int32_t *__restrict__ act_len, int M, int KK,
                                                       const int32_t *__restrict__ off2, int NB,
                                                       const int32_t *__restrict__ ids, int64_t N, int BS, int k,
                                                       int32_t *__restrict__ pool, int64_t CAPQ,
                                                       int32_t *__restrict__ cbase, int32_t *__restrict__ ncand, int NS,
                                                       int32_t *__restrict__ fbflag, int32_t *__restrict__ ghist,
                                                       int GHB) {
    extern __shared__ __align__(16) unsigned char smraw[];
    unsigned char *cnt8 = smraw;
    CountSmem &S = *(CountSmem *)(smraw + BS + BS / 8);
    __shared__ int hist[2 * MAX_M + 2];
    __shared__ int s_total, s_vstar, s_quota, s_eqbase, s_n;
    const int64_t q = blockIdx.x;
    const int tid = threadIdx.x;
    if (tid == 0) s_total = 0;
    for (int i = tid; i < 2 * MAX_M + 2; i += THREADS) hist[i] = 0;
    __syncthreads();
    {
        int t = 0;
        for (int b = tid; b < NS; b += THREADS) t += ncand[q * NS + b];
        for (int off = 16; off; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        if ((tid & 31) == 0 && t) atomicAdd(&s_total, t);
    }
    __syncthreads();
    if (s_total >= k) {
        if (tid == 0) fbflag[q] = 0;
        return;
    }
    const int Etot = count_setup(S, q, act, act_len, M, KK);
    fb_hist_pass(S, cnt8, BS, q, Etot, act, M, KK, off2, NB, ids, N, hist);
    if (tid == 0) fb_threshold(hist, M, k, &s_vstar, &s_quota);
    __syncthreads();
    const int n = fb_select_pass(S, cnt8, BS, q, Etot, act, M, KK, off2, NB, ids, N, s_vstar, s_quota, pool + q * CAPQ,
                                 &s_eqbase, &s_n);
    for (int b = tid; b < NS; b += THREADS) {
        ncand[q * NS + b] = (b == 0) ? n : 0;
        cbase[q * NS + b] = 0;
    }
    // phi=1: the Hamming histogram of the replaced candidate set restarts (k_hamming refills it)
    if (ghist)
        for (int i = tid; i < GHB; i += THREADS) ghist[q * GHB + i] = 0;
    if (tid == 0) fbflag[q] = 1;
}

// sharded: local histogram of V for queries whose GLOBAL |C| < k (zeros otherwise)
__global__ void __launch_bounds__(THREADS) k_fb_hist(const uint32_t *__restrict__ act,
                                                      const int32_t *__restrict__ act_len, int M, int KK,
                                                      const int32_t *__restrict__ off2, int NB,
                                                      const int32_t *__restrict__ ids, int64_t N, int BS, int k,
                                                      const int32_t *__restrict__ gcount, int32_t *__restrict__ lhist) {
    extern __shared__ __align__(16) unsigned char smraw[];
    unsigned char *cnt8 = smraw;
    CountSmem &S = *(CountSmem *)(smraw + BS + BS / 8);
    __shared__ int hist[2 * MAX_M + 2];
    const int64_t q = blockIdx.x;
    const int HB = 2 * M + 2;
    for (int i = threadIdx.x; i < 2 * MAX_M + 2; i += THREADS) hist[i] = 0;
    __syncthreads();
    if (gcount[q] < k) {
        const int Etot = count_setup(S, q, act, act_len, M, KK);
        fb_hist_pass(S, cnt8, BS, q, Etot, act, M, KK, off2, NB, ids, N, hist);
    }
    for (int i = threadIdx.x; i < HB; i += THREADS) lhist[q * HB + i] = hist[i];
}

// sharded: selection with the global V*/quota; this shard's share of the
// V == V* quota follows the global id order (shard g owns [g*N/G, (g+1)*N/G))
__global__ void __launch_bounds__(THREADS) k_fb_select(const uint32_t *__restrict__ act,
                                                        const int32_t *__restrict__ act_len, int M, int KK,
                                                        const int32_t *__restrict__ off2, int NB,
                                                        const int32_t *__restrict__ ids, int64_t N, int BS, int k,
                                                        const int32_t *__restrict__ gcount,
                                                        const int32_t *__restrict__ allhist, int G, int rank, int64_t Q,
                                                        int32_t *__restrict__ pool, int64_t CAPQ,
                                                        int32_t *__restrict__ cbase, int32_t *__restrict__ ncand,
                                                        int NS, int32_t *__restrict__ fbflag,
                                                        int32_t *__restrict__ ghist, int GHB) {
    extern __shared__ __align__(16) unsigned char smraw[];
    unsigned char *cnt8 = smraw;
    CountSmem &S = *(CountSmem *)(smraw + BS + BS / 8);
    __shared__ int hist[2 * MAX_M + 2];
    __shared__ int s_vstar, s_quota, s_eqbase, s_n;
    const int64_t q = blockIdx.x;
    const int tid = threadIdx.x, HB = 2 * M + 2;
    if (gcount[q] >= k) {
        if (tid == 0) fbflag[q] = 0;
        return;
    }
    for (int i = tid; i < HB; i += THREADS) {
        int t = 0;
        for (int g = 0; g < G; g++) t += allhist[((int64_t)g * Q + q) * HB + i];
        hist[i] = t;
    }
    __syncthreads();
    if (tid == 0) {
        int vstar, quota;
        fb_threshold(hist, M, k, &vstar, &quota);
        int before = 0;
        for (int g = 0; g < rank; g++) before += allhist[((int64_t)g * Q + q) * HB + vstar];
        const int mine = allhist[((int64_t)rank * Q + q) * HB + vstar];
        s_vstar = vstar;
        s_quota = max(0, min(mine, quota - before));
    }
    __syncthreads();
    const int Etot = count_setup(S, q, act, act_len, M, KK);
    const int n = fb_select_pass(S, cnt8, BS, q, Etot, act, M, KK, off2, NB, ids, N, s_vstar, s_quota, pool + q * CAPQ,
                                 &s_eqbase, &s_n);
    for (int b = tid; b < NS; b += THREADS) {
        ncand[q * NS + b] = (b == 0) ? n : 0;
        cbase[q * NS + b] = 0;
    }
    // phi=1: the Hamming histogram of the replaced candidate set restarts (k_hamming refills it)
    if (ghist)
        for (int i = tid; i < GHB; i += THREADS) ghist[q * GHB + i] = 0;
    if (tid == 0) fbflag[q] = 1;
}

// Query locality order: queries whose first-ranked cells in subspaces 0 and 1
// agree share most of their candidates (and so their CSR slices, codes and
// rows in L2); the count and verification grids visit queries in the order of
// this key.  A pure scheduling permutation: every per-query result is the same.
__global__ void k_query_key(const uint32_t *__restrict__ act, int M, int KK, int64_t Qc, uint32_t *__restrict__ key,
                            int32_t *__restrict__ iota) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= Qc) return;
    const uint32_t *a = act + q * (int64_t)M * KK;
    const uint32_t c0 = a[0] & 0xffffu, c1 = M > 1 ? (a[KK] & 0xffffu) : 0u;
    key[q] = c0 * (uint32_t)KK + c1;
    iota[q] = (int32_t)q;
}

__global__ void k_local_counts(const int32_t *__restrict__ ncand, int NB, int64_t Qc, int32_t *__restrict__ out) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= Qc) return;
    int t = 0;
    for (int b = 0; b < NB; b++) t += ncand[q * NB + b];
    out[q] = t;
}

// ---------------------------------------------------------------------------
// exact distance of one stored row to q' (fp64, lane partial sums + fixed
// butterfly; every lane returns the same value)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    return v;
}

// The query is staged in shared memory as doubles in component-major order
// (qd[c*nvec + v] = q'[4v + c], see load_qd) so that the lanes of a warp,
// which take consecutive float4s v, read consecutive doubles (no bank
// conflicts); one read serves both rows of row_dist2.
struct Q4 {
    double a, b, c, d;
};
__device__ __forceinline__ Q4 q4_at(const double *__restrict__ qd, int v, int nvec) {
    return {qd[v], qd[nvec + v], qd[2 * nvec + v], qd[3 * nvec + v]};
}
__device__ __forceinline__ void acc4(double &acc, const float4 x, const Q4 &q) {
    const double d0 = __dsub_rn((double)x.x, q.a), d1 = __dsub_rn((double)x.y, q.b);
    const double d2 = __dsub_rn((double)x.z, q.c), d3 = __dsub_rn((double)x.w, q.d);
    acc = __fma_rn(d0, d0, acc);
    acc = __fma_rn(d1, d1, acc);
    acc = __fma_rn(d2, d2, acc);
    acc = __fma_rn(d3, d3, acc);
}

// Row distances, a warp per row: lane l takes the float4s l, l+32, ... of the
// row in ascending order (its partial sum), then a butterfly.  Two rows at
// once share the query reads and double the loads in flight.
__device__ __forceinline__ void row_dist2(const float *__restrict__ r0, const float *__restrict__ r1,
                                          const double *__restrict__ qd, int nvec, int lane, double &o0, double &o1) {
    double a0 = 0.0, a1 = 0.0;
    const float4 *x0 = (const float4 *)r0, *x1 = (const float4 *)r1;
#pragma unroll 4
    for (int v = lane; v < nvec; v += 32) {
        const float4 u0 = __ldg(x0 + v);
        const float4 u1 = __ldg(x1 + v);
        const Q4 qv = q4_at(qd, v, nvec);
        acc4(a0, u0, qv);
        acc4(a1, u1, qv);
    }
    o0 = warp_sum(a0);
    o1 = warp_sum(a1);
}
// four rows at once: the query reads (shared-memory wavefronts) are amortised
// over four rows and four loads per lane are in flight per step
__device__ __forceinline__ void row_dist4(const float *__restrict__ r0, const float *__restrict__ r1,
                                          const float *__restrict__ r2, const float *__restrict__ r3,
                                          const double *__restrict__ qd, int nvec, int lane, double (&o)[4]) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const float4 *x0 = (const float4 *)r0, *x1 = (const float4 *)r1, *x2 = (const float4 *)r2,
                 *x3 = (const float4 *)r3;
#pragma unroll 2
    for (int v = lane; v < nvec; v += 32) {
        const float4 u0 = __ldg(x0 + v), u1 = __ldg(x1 + v), u2 = __ldg(x2 + v), u3 = __ldg(x3 + v);
        const Q4 qv = q4_at(qd, v, nvec);
        acc4(a0, u0, qv);
        acc4(a1, u1, qv);
        acc4(a2, u2, qv);
        acc4(a3, u3, qv);
    }
    o[0] = warp_sum(a0);
    o[1] = warp_sum(a1);
    o[2] = warp_sum(a2);
    o[3] = warp_sum(a3);
}
__device__ __forceinline__ double row_dist1(const float *__restrict__ r0, const double *__restrict__ qd, int nvec,
                                            int lane) {
    double a0 = 0.0;
    const float4 *x0 = (const float4 *)r0;
#pragma unroll 4
    for (int v = lane; v < nvec; v += 32) acc4(a0, __ldg(x0 + v), q4_at(qd, v, nvec));
    return warp_sum(a0);
}

// warp-cooperative insertion of (d, id) into a sorted list of capacity k
__device__ __forceinline__ void warp_insert(double *Ld, int64_t *Li, int &cnt, int k, double d, int64_t id, int lane) {
    int pos = 0;
    for (int i0 = 0; i0 < cnt; i0 += 32) {
        int i = i0 + lane;
        bool lt = i < cnt && less_di(Ld[i], Li[i], d, id);
        pos += __popc(__ballot_sync(0xffffffffu, lt));
    }
    int last = min(cnt, k - 1);  // entries [pos, last) move up by one
    for (int top = last - 1; top >= pos; top -= 32) {
        int i = top - lane;
        double td = 0.0;
        int64_t ti = 0;
        bool mv = i >= pos;
        if (mv) {
            td = Ld[i];
            ti = Li[i];
        }
        __syncwarp();
        if (mv) {
            Ld[i + 1] = td;
            Li[i + 1] = ti;
        }
        __syncwarp();
    }
    if (lane == 0) {
        Ld[pos] = d;
        Li[pos] = id;
    }
    cnt = min(cnt + 1, k);
    __syncwarp();
}

// q' as doubles, component-major: qd[c*nvec + v] = q'[4v + c], nvec = pitch/4
__device__ __forceinline__ void load_qd(double *qd, const float *qrow, int pitch) {
    const int nvec = pitch >> 2;
    for (int i = threadIdx.x; i < pitch; i += blockDim.x) qd[(i & 3) * nvec + (i >> 2)] = (double)qrow[i];
}

// ---------------------------------------------------------------------------
// Verification filter (DESIGN R17; crisp_set_verify_filter).  The index keeps
// every row centred on the column means mu (fp32) and quantised per row:
// x~ = 2^e c with c in [-127, 127]^D (int8), the integer sum c.c, and
// rho >= ||(x - mu) - x~|| (fp64, rounded up).  Per query, y = q' - mu (fp64)
// is written as y_fx = 2^(E-6) (d1 + 2^-7 d2) with int8 digits d1, d2 in
// [-64, 64] (k_q8_prep) and R >= ||y - y_fx||.  A warp then forms the integer
// dot products S1 = d1.c, S2 = d2.c exactly (dp4a, int32), so that
//   P = <y_fx, x~> = 2^(E-6+e) (S1 + S2/128)       (exact in fp64)
//   ||y - x~||^2 = ||y||^2 - 2 P + ||x~||^2 - 2 <y - y_fx, x~>,
//   |<y - y_fx, x~>| <= R ||x~||                   (Cauchy-Schwarz),
// and, with the triangle inequality ||q' - x|| = ||y - (x - mu)||,
//   sqrt(A_lo) - rho <= ||q' - x|| <= sqrt(A_hi) + rho
// where A_lo/A_hi carry the Cauchy-Schwarz term and 1e-11 relative slack for
// the fp64 evaluation (every other factor 1e-12).  A row whose lower bound
// exceeds sqrt(d_k) (1 + 1e-9), d_k the k-th best distance a top-k already
// holds, has d > d_k (1 + 2e-9): its exact verification would be a miss, so
// its fp32 row is not read.  Bytes per bounded row: D (codes) + 16 (meta).
// ---------------------------------------------------------------------------
struct FiltArgs {
    const uint4 *C8;     // N x nv16 (16 int8 codes each); null: filter off
    const int4 *meta;    // N: {c.c, e, rho (float bits), 0}
    int nv16;            // uint4 per code row (c8pitch / 16)
    const uint4 *qd;     // Qc x 2 nv16: digit planes d1 | d2 of each query (k_q8_prep)
    const double *qi;    // Qc x 4: {2^(E-6), ||y||^2, R, ok}
};

// per query: y = q' - mu, its two digit planes and the bound terms
__global__ void __launch_bounds__(256) k_q8_prep(const float *__restrict__ qrot, int pitch,
                                                 const float *__restrict__ mu, int c8pitch, uint4 *__restrict__ qd,
                                                 double *__restrict__ qi) {
    const int64_t q = blockIdx.x;
    const float *qr = qrot + q * pitch;
    __shared__ double red[3][8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double m = 0.0, n2 = 0.0;
    int bad = 0;
    for (int i = tid; i < pitch; i += 256) {
        const double y = (double)qr[i] - (double)mu[i];
        if (!isfinite(y)) bad = 1;
        m = fmax(m, fabs(y));
        n2 = fma(y, y, n2);
    }
    for (int o = 16; o; o >>= 1) {
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        n2 += __shfl_xor_sync(0xffffffffu, n2, o);
    }
    if (lane == 0) {
        red[0][warp] = m;
        red[1][warp] = n2;
    }
    bad = __syncthreads_or(bad);
    m = 0.0;
    n2 = 0.0;
    for (int w = 0; w < 8; w++) {
        m = fmax(m, red[0][w]);
        n2 += red[1][w];
    }
    int E = 0;
    if (m > 0.0) frexp(m, &E);  // m < 2^E
    const double up = ldexp(1.0, 6 - E), dn = ldexp(1.0, E - 6);
    int8_t *d1 = (int8_t *)(qd + q * 2 * (c8pitch / 16)), *d2 = d1 + c8pitch;
    double r2 = 0.0;
    for (int i = tid; i < c8pitch; i += 256) {
        const double y = i < pitch ? (double)qr[i] - (double)mu[i] : 0.0;
        const double v = y * up;                      // |v| < 64
        const double a = rint(v), b = rint((v - a) * 128.0);  // both in [-64, 64]
        d1[i] = bad ? 0 : (int8_t)a;
        d2[i] = bad ? 0 : (int8_t)b;
        const double r = y - dn * (a + b * 0.0078125);  // |r| <= 2^(E-14)
        r2 = fma(r, r, r2);
    }
    for (int o = 16; o; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    __syncthreads();
    if (lane == 0) red[2][warp] = r2;
    __syncthreads();
    if (tid == 0) {
        r2 = 0.0;
        for (int w = 0; w < 8; w++) r2 += red[2][w];
        // y itself is exact up to 2^-53 relative (fp32 - fp32 in fp64): 1e-15 ||y|| covers it
        qi[q * 4 + 0] = dn;
        qi[q * 4 + 1] = n2;
        qi[q * 4 + 2] = sqrt(r2) * (1.0 + 1e-9) + 1e-15 * sqrt(n2);
        qi[q * 4 + 3] = (bad || !isfinite(n2)) ? 0.0 : 1.0;
    }
}

// S1 = d1.c and S2 = d2.c of R rows at once (lanes take uint4 v = lane, lane +
// 32, ...; the digit reads are shared by the R rows); every lane returns them
template <int R>
__device__ __forceinline__ void rows_q8(const uint4 *const (&r)[R], const uint4 *__restrict__ sq, int nv16, int lane,
                                        int (&S1)[R], int (&S2)[R]) {
    int a[R], b[R];
#pragma unroll
    for (int u = 0; u < R; u++) a[u] = b[u] = 0;
#pragma unroll 2
    for (int v = lane; v < nv16; v += 32) {
        uint4 x[R];
#pragma unroll
        for (int u = 0; u < R; u++) x[u] = __ldg(r[u] + v);
        const uint4 p = sq[v], t = sq[nv16 + v];
#pragma unroll
        for (int u = 0; u < R; u++) {
            a[u] = __dp4a((int)x[u].x, (int)p.x, a[u]);
            a[u] = __dp4a((int)x[u].y, (int)p.y, a[u]);
            a[u] = __dp4a((int)x[u].z, (int)p.z, a[u]);
            a[u] = __dp4a((int)x[u].w, (int)p.w, a[u]);
            b[u] = __dp4a((int)x[u].x, (int)t.x, b[u]);
            b[u] = __dp4a((int)x[u].y, (int)t.y, b[u]);
            b[u] = __dp4a((int)x[u].z, (int)t.z, b[u]);
            b[u] = __dp4a((int)x[u].w, (int)t.w, b[u]);
        }
    }
#pragma unroll
    for (int u = 0; u < R; u++) {
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            a[u] += __shfl_xor_sync(0xffffffffu, a[u], off);
            b[u] += __shfl_xor_sync(0xffffffffu, b[u], off);
        }
        S1[u] = a[u];
        S2[u] = b[u];
    }
}

// per-query terms of the bound, staged once per CTA
struct QTerms {
    double dn, n2, R;
    bool ok;
};
__device__ __forceinline__ QTerms load_q8(uint4 *sq, const FiltArgs &fa, int64_t q) {
    const uint4 *g = fa.qd + q * 2 * fa.nv16;
    for (int i = threadIdx.x; i < 2 * fa.nv16; i += blockDim.x) sq[i] = g[i];
    const double *t = fa.qi + q * 4;
    return QTerms{t[0], t[1], t[2], t[3] != 0.0};
}

// certified lower / upper bounds of ||q' - x|| (see above)
__device__ __forceinline__ void filt_bounds(const QTerms &qt, int S1, int S2, int4 meta, double &lb, double &ub) {
    const double sc = ldexp(qt.dn, meta.y);
    const double P = sc * ((double)S1 + (double)S2 * 0.0078125);
    const double X2 = ldexp((double)meta.x, 2 * meta.y);
    const double xn = sqrt(X2) * (1.0 + 1e-12);
    const double A = qt.n2 - 2.0 * P + X2;
    const double slack = 2.0 * qt.R * xn * (1.0 + 1e-12) + 1e-11 * (qt.n2 + X2 + 2.0 * fabs(P));
    const double rho = (double)__int_as_float(meta.z) * (1.0 + 1e-12);
    const double alo = A - slack, ahi = A + slack;
    lb = (qt.ok && alo > 0.0) ? sqrt(alo) * (1.0 - 1e-12) - rho : 0.0;
    ub = qt.ok ? sqrt(fmax(ahi, 0.0)) * (1.0 + 1e-12) + rho : INFINITY;
}

// ---------------------------------------------------------------------------
// a5, Guaranteed Mode: exact L2 of every candidate, per-warp top-k, CTA merge.
// grid (S, Qc); candidates of query q are split over S*WARPS warps.
// ---------------------------------------------------------------------------
// prefix over the blocks' candidate counts (pre, NB+1) and their pool bases
__device__ __forceinline__ void block_prefix(const int32_t *__restrict__ ncand, const int32_t *__restrict__ cbase,
                                             int64_t q, int NB, int *pre, int *cbs) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        int acc = 0;
        for (int b0 = 0; b0 < NB; b0 += 32) {
            const int b = b0 + lane;
            int v = b < NB ? ncand[q * NB + b] : 0;
            if (b < NB) cbs[b] = cbase[q * NB + b];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                int t = __shfl_up_sync(0xffffffffu, v, off);
                if (lane >= off) v += t;
            }
            if (b < NB) pre[b + 1] = acc + v;
            acc += __shfl_sync(0xffffffffu, v, 31);
        }
        if (lane == 0) pre[0] = 0;
    }
}

template <bool ROWS4, bool FILT>
__global__ void __launch_bounds__(THREADS) k_rerank_exact(const float *__restrict__ qrot, int pitch,
                                                           const float *__restrict__ X, int64_t gid_base,
                                                           const int32_t *__restrict__ pool, int64_t CAPQ,
                                                           const int32_t *__restrict__ cbase,
                                                           const int32_t *__restrict__ ncand, int NB, int k,
                                                           double *__restrict__ part_d, int64_t *__restrict__ part_i,
                                                           const int32_t *__restrict__ qperm,
                                                           const float2 *__restrict__ lbb, const float *__restrict__ Tq,
                                                           unsigned long long *__restrict__ fstats) {
    extern __shared__ __align__(16) unsigned char sm[];
    double *qd = (double *)sm;
    double *Ld = qd + pitch;                         // WARPS x k
    int64_t *Li = (int64_t *)(Ld + WARPS * k);       // WARPS x k
    int *pre = (int *)(Li + WARPS * k);              // NB + 1
    int *cbs = pre + NB + 1;                         // NB
    __shared__ int wcnt[WARPS];
    const int64_t q = qperm ? qperm[blockIdx.y] : blockIdx.y;  // locality order (query_order)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    load_qd(qd, qrot + q * pitch, pitch);
    block_prefix(ncand, cbase, q, NB, pre, cbs);
    __syncthreads();
    const int total = pre[NB];
    const int nvec = pitch / 4;
    const int W = gridDim.x * WARPS;
    const int gw = blockIdx.x * WARPS + warp;
    double *myd = Ld + warp * k;
    int64_t *myi = Li + warp * k;
    int cnt = 0;
    double wd = INFINITY;
    int64_t wi = 0x7fffffffffffffffLL;
    int bcur = 0;
    const int32_t *poolq = pool + q * CAPQ;
    // up to four rows per warp step (v, v+W, v+2W, v+3W); the candidate ids come
    // from the segments through a monotone segment pointer
    auto lid_at = [&](int vv, int &bc) -> int {
        while (pre[bc + 1] <= vv) bc++;
        return poolq[cbs[bc] + (vv - pre[bc])];
    };
    auto offer = [&](double dd, int64_t gg) {
        if (cnt < k || less_di(dd, gg, wd, wi)) {
            warp_insert(myd, myi, cnt, k, dd, gg, lane);
            if (cnt == k) {
                wd = myd[k - 1];
                wi = myi[k - 1];
            }
        }
    };
    if (FILT) {
        // R17: only the candidates whose lower bound does not exceed T (the k-th
        // smallest upper bound of the query, k_lb_threshold) can be in the top-k;
        // a warp takes 32 consecutive positions, reads their bounds, and computes
        // the exact distances of the passing ones four at a time
        const double Tm = (double)Tq[q] * (1.0 + 1e-9);
        const float2 *lbq = lbb + q * CAPQ;
        int bl = 0;  // this lane's segment pointer (its positions only increase)
        unsigned nb = 0, ne = 0;
        for (int base = gw * 32; base < total; base += W * 32) {
            const int v = base + lane;
            int lid = -1;
            if (v < total) {
                while (pre[bl + 1] <= v) bl++;
                const int p = cbs[bl] + (v - pre[bl]);
                if (!((double)lbq[p].x > Tm)) lid = poolq[p];
            }
            unsigned m = __ballot_sync(0xffffffffu, lid >= 0);
            nb += min(32, total - base);
            ne += __popc(m);
            while (m) {
                int ls[4], nl = 0;
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    ls[u] = -1;
                    if (m) {
                        ls[u] = __shfl_sync(0xffffffffu, lid, __ffs(m) - 1);
                        m &= m - 1;
                        nl++;
                    }
                }
                if (nl == 4) {
                    double d4[4];
                    row_dist4(X + (int64_t)ls[0] * pitch, X + (int64_t)ls[1] * pitch, X + (int64_t)ls[2] * pitch,
                              X + (int64_t)ls[3] * pitch, qd, nvec, lane, d4);
#pragma unroll
                    for (int u = 0; u < 4; u++) offer(d4[u], gid_base + ls[u]);
                } else {
                    if (nl >= 2) {
                        double d0, d1;
                        row_dist2(X + (int64_t)ls[0] * pitch, X + (int64_t)ls[1] * pitch, qd, nvec, lane, d0, d1);
                        offer(d0, gid_base + ls[0]);
                        offer(d1, gid_base + ls[1]);
                    } else {
                        offer(row_dist1(X + (int64_t)ls[0] * pitch, qd, nvec, lane), gid_base + ls[0]);
                    }
                    if (nl == 3) offer(row_dist1(X + (int64_t)ls[2] * pitch, qd, nvec, lane), gid_base + ls[2]);
                }
            }
        }
        if (fstats && lane == 0 && nb) atomicAdd(fstats + 1, (unsigned long long)ne);
    }
    for (int v = FILT ? total : gw; v < total; v += 4 * W) {
        if (ROWS4 && v + 3 * W < total) {
            int b1 = bcur;
            const int l0 = lid_at(v, bcur), l1 = lid_at(v + W, b1), l2 = lid_at(v + 2 * W, b1),
                      l3 = lid_at(v + 3 * W, b1);
            double d4[4];
            row_dist4(X + (int64_t)l0 * pitch, X + (int64_t)l1 * pitch, X + (int64_t)l2 * pitch,
                      X + (int64_t)l3 * pitch, qd, nvec, lane, d4);
            offer(d4[0], gid_base + l0);
            offer(d4[1], gid_base + l1);
            offer(d4[2], gid_base + l2);
            offer(d4[3], gid_base + l3);
            continue;
        }
        for (int vv = v; vv < total; vv += 2 * W) {
            const int v1 = vv + W;
            int b1 = bcur;
            const int lid0 = lid_at(vv, bcur);
            const int lid1 = v1 < total ? lid_at(v1, b1) : -1;
            double d0, d1;
            if (lid1 >= 0) {
                row_dist2(X + (int64_t)lid0 * pitch, X + (int64_t)lid1 * pitch, qd, nvec, lane, d0, d1);
            } else {
                d0 = row_dist1(X + (int64_t)lid0 * pitch, qd, nvec, lane);
                d1 = INFINITY;
            }
            offer(d0, gid_base + lid0);
            if (lid1 >= 0) offer(d1, gid_base + lid1);
        }
        break;  // the two-row loop took every remaining row of this warp
    }
    if (lane == 0) wcnt[warp] = cnt;
    __syncthreads();
    // CTA merge: rank of each entry = sum over lists of #entries less than it
    double *od = part_d + ((int64_t)q * gridDim.x + blockIdx.x) * k;
    int64_t *oi = part_i + ((int64_t)q * gridDim.x + blockIdx.x) * k;
    for (int r = threadIdx.x; r < k; r += THREADS) {
        od[r] = INFINITY;
        oi[r] = -1;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < WARPS * k; e += THREADS) {
        int w = e / k, i = e % k;
        if (i >= wcnt[w]) continue;
        double d = Ld[w * k + i];
        int64_t id = Li[w * k + i];
        int rank = i;
        for (int w2 = 0; w2 < WARPS; w2++) {
            if (w2 == w) continue;
            int lo = 0, hi = wcnt[w2];
            const double *L2d = Ld + w2 * k;
            const int64_t *L2i = Li + w2 * k;
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                if (less_di(L2d[mid], L2i[mid], d, id)) lo = mid + 1;
                else hi = mid;
            }
            rank += lo;
        }
        if (rank < k) {
            od[rank] = d;
            oi[rank] = id;
        }
    }
}

// ---------------------------------------------------------------------------
// a5, Guaranteed Mode with the verification filter (R17), passes 1 and 2:
// k_lb_bounds streams the int8 copies of the query's candidates and writes
// (lb, ub) of ||q' - x|| per pool slot (lb rounded down, ub rounded up);
// k_lb_threshold selects T >= the k-th smallest ub (two 11/12-bit histogram
// passes over the bits of the non-negative floats; T is the upper edge of the
// bin that holds it).  k rows then have sqrt(d) <= T, so a row with lb > T (1 + 1e-9) is
// outside the top-k, and k_rerank_exact<., true> reads only the others.
// ---------------------------------------------------------------------------
template <int MINB>
__global__ void __launch_bounds__(THREADS, MINB) k_lb_bounds(const float *__restrict__ qrot, int pitch, FiltArgs fa,
                                                        const int32_t *__restrict__ pool, int64_t CAPQ,
                                                        const int32_t *__restrict__ cbase,
                                                        const int32_t *__restrict__ ncand, int NB,
                                                        float2 *__restrict__ lbb, const int32_t *__restrict__ qperm,
                                                        unsigned long long *__restrict__ fstats) {
    extern __shared__ __align__(16) unsigned char sm[];
    uint4 *sq = (uint4 *)sm;                   // 2 nv16 (the query's digit planes)
    int *pre = (int *)(sq + 2 * fa.nv16);      // NB + 1
    int *cbs = pre + NB + 1;                   // NB
    const int64_t q = qperm ? qperm[blockIdx.y] : blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    block_prefix(ncand, cbase, q, NB, pre, cbs);
    const QTerms qt = load_q8(sq, fa, q);
    __syncthreads();
    const int total = pre[NB];
    const int W = gridDim.x * WARPS;
    const int gw = blockIdx.x * WARPS + warp;
    const int32_t *poolq = pool + q * CAPQ;
    float2 *lbq = lbb + q * CAPQ;
    int bcur = 0;
    auto slot_at = [&](int vv, int &bc) -> int {
        while (pre[bc + 1] <= vv) bc++;
        return cbs[bc] + (vv - pre[bc]);
    };
    if (!qt.ok) {  // non-finite q': no bound for this query (every row exact)
        for (int v = blockIdx.x * THREADS + threadIdx.x; v < total; v += gridDim.x * THREADS) {
            int b = 0;
            lbq[slot_at(v, b)] = make_float2(0.0f, INFINITY);
        }
        return;
    }
    for (int v = gw; v < total; v += 4 * W) {
        int slot[4], rows[4];
        int b1 = bcur;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int vv = v + u * W;
            slot[u] = vv < total ? (u == 0 ? slot_at(vv, bcur) : slot_at(vv, b1)) : -1;
            rows[u] = slot[u] >= 0 ? poolq[slot[u]] : -1;
        }
        const uint4 *r4[4];
#pragma unroll
        for (int u = 0; u < 4; u++) r4[u] = fa.C8 + (int64_t)(rows[u] >= 0 ? rows[u] : rows[0]) * fa.nv16;
        int S1[4], S2[4];
        rows_q8<4>(r4, sq, fa.nv16, lane, S1, S2);
        int sl = -1, rl = 0, s1 = 0, s2 = 0;
#pragma unroll
        for (int u = 0; u < 4; u++)
            if (lane == u) {
                sl = slot[u];
                rl = rows[u];
                s1 = S1[u];
                s2 = S2[u];
            }
        if (sl >= 0) {
            double lb, ub;
            filt_bounds(qt, s1, s2, __ldg(fa.meta + rl), lb, ub);
            lbq[sl] = make_float2(__double2float_rd(fmax(lb, 0.0)), __double2float_ru(ub));
        }
    }
    if (fstats && threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(fstats, (unsigned long long)total);
}

__global__ void __launch_bounds__(THREADS) k_lb_threshold(const int32_t *__restrict__ cbase,
                                                          const int32_t *__restrict__ ncand, int NB, int64_t CAPQ,
                                                          const float2 *__restrict__ lbb, int k,
                                                          float *__restrict__ Tq) {
    extern __shared__ __align__(16) unsigned char sm[];
    int *pre = (int *)sm;            // NB + 1
    int *cbs = pre + NB + 1;         // NB
    __shared__ unsigned hist[4096];
    __shared__ unsigned s_bin, s_rank;
    const int64_t q = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31;
    block_prefix(ncand, cbase, q, NB, pre, cbs);
    __syncthreads();
    const int total = pre[NB];
    if (total <= k) {
        if (tid == 0) Tq[q] = INFINITY;
        return;
    }
    const float2 *lbq = lbb + q * CAPQ;
    unsigned prefix = 0, rank = (unsigned)(k - 1);  // 0-based rank of the k-th smallest
    // pass 0: bits 30..20 (2048 bins); pass 1: bits 19..8 (4096 bins) inside the bin of pass 0
    for (int pass = 0; pass < 2; pass++) {
        const int shift = pass == 0 ? 20 : 8, nbins = pass == 0 ? 2048 : 4096;
        for (int i = tid; i < nbins; i += THREADS) hist[i] = 0;
        __syncthreads();
        int b = 0;
        for (int v = tid; v < total; v += THREADS) {
            while (pre[b + 1] <= v) b++;
            const unsigned u = __float_as_uint(lbq[cbs[b] + (v - pre[b])].y);
            if (pass == 0 || (u >> 20) == prefix) atomicAdd(&hist[(u >> shift) & (nbins - 1)], 1u);
        }
        __syncthreads();
        if (tid < 32) {
            // lane-contiguous bins, lane sums, warp scan, then the bin that holds rank
            const int per = nbins / 32;
            unsigned ls = 0;
            for (int i = 0; i < per; i++) ls += hist[lane * per + i];
            unsigned inc = ls;
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            const unsigned exc = inc - ls;
            if (rank >= exc && rank < inc) {
                unsigned c = exc;
                for (int i = 0; i < per; i++) {
                    const unsigned h = hist[lane * per + i];
                    if (rank < c + h) {
                        s_bin = lane * per + i;
                        s_rank = rank - c;
                        break;
                    }
                    c += h;
                }
            }
        }
        __syncthreads();
        if (pass == 0) prefix = s_bin;
        else prefix = (prefix << 12) | s_bin;
        rank = s_rank;
        __syncthreads();
    }
    if (tid == 0) Tq[q] = __uint_as_float((prefix << 8) | 0xffu);  // upper edge of the bin (>= the k-th ub)
}

// ---------------------------------------------------------------------------
// a5, Guaranteed Mode, grouped (the dense-candidate regime: |C_q| a large share
// of N, e.g. cfg3/cfg5).  A CTA owns a group of GR consecutive queries of the
// locality order (R8) and a range of RW ids.  It marks each query's candidates
// of the range in a byte mask per id (bit g = query g of the group), lists the
// ids any of them holds, and reads every such row ONCE: a warp loads the row
// (float4, lane l takes float4s l, l+32, ...) and accumulates the distance of
// every member query at the same time, in the same order as k_rerank_exact (the
// lane's partial sum in ascending float4 order, then the butterfly), so the
// distances are identical to the ungrouped kernel's.  Per (warp, query) top-k
// lists, merged per query into the partial list of (query, range); k_merge_lists
// merges the ranges.  A row shared by the group's queries is read once instead
// of once per query.
// ---------------------------------------------------------------------------
constexpr int RG_MAX = 8;  // queries per group (mask bits)

template <int GR>
__global__ void __launch_bounds__(THREADS) k_rerank_group(const float *__restrict__ qrot, int pitch,
                                                           const float *__restrict__ X, int64_t gid_base, int64_t N,
                                                           const int32_t *__restrict__ pool, int64_t CAPQ,
                                                           const int32_t *__restrict__ cbase,
                                                           const int32_t *__restrict__ ncand, int NS, int segw,
                                                           const int32_t *__restrict__ fb, int RW, int k,
                                                           int64_t Qc, double *__restrict__ part_d,
                                                           int64_t *__restrict__ part_i,
                                                           const int32_t *__restrict__ qperm) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int nvec = pitch / 4;
    double *qd = (double *)sm;                               // GR x pitch (component-major per query)
    double *Ld = qd + (size_t)GR * pitch;                    // WARPS x GR x k
    int64_t *Li = (int64_t *)(Ld + WARPS * GR * k);          // WARPS x GR x k
    uint32_t *mask = (uint32_t *)(Li + WARPS * GR * k);     // RW bytes (4 ids per word)
    uint16_t *list = (uint16_t *)((unsigned char *)mask + RW);  // RW
    __shared__ int wcnt[WARPS][RG_MAX];
    __shared__ int s_n, s_base[WARPS + 1];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t lo = (int64_t)blockIdx.x * RW;
    const int64_t hi = min(N, lo + RW);
    const int seg = (int)(lo / segw);
    int64_t qs[GR];
    int ng = 0;
#pragma unroll
    for (int g = 0; g < GR; g++) {
        const int64_t qi = (int64_t)blockIdx.y * GR + g;
        qs[g] = qi < Qc ? (qperm ? qperm[qi] : qi) : -1;
        ng += qi < Qc;
    }
#pragma unroll
    for (int g = 0; g < GR; g++)
        if (qs[g] >= 0) load_qd(qd + (size_t)g * pitch, qrot + qs[g] * pitch, pitch);
    for (int i = tid; i < RW / 4; i += THREADS) mask[i] = 0u;
    __syncthreads();
    // each query's candidates in [lo, hi): its segment of this range (ascending ids), or the
    // fallback's single segment (segment 0, ascending ids over all of [0, N))
#pragma unroll
    for (int g = 0; g < GR; g++) {
        if (qs[g] < 0) continue;
        const int64_t q = qs[g];
        const int sgi = fb[q] ? 0 : seg;
        const int n = ncand[q * NS + sgi];
        const int32_t *c = pool + q * CAPQ + cbase[q * NS + sgi];
        // [a, b): the segment's ids in [lo, hi) (binary searches; ids ascending)
        int a = 0, b = n;
        {
            int l2 = 0, h2 = n;
            while (l2 < h2) {
                const int md = (l2 + h2) >> 1;
                if (c[md] < lo) l2 = md + 1;
                else h2 = md;
            }
            a = l2;
            h2 = n;
            while (l2 < h2) {
                const int md = (l2 + h2) >> 1;
                if (c[md] < hi) l2 = md + 1;
                else h2 = md;
            }
            b = l2;
        }
        for (int i = a + tid; i < b; i += THREADS) {
            const int x = (int)(c[i] - lo);
            atomicOr(mask + (x >> 2), 1u << (8 * (x & 3) + g));
        }
    }
    __syncthreads();
    // list the ids with a non-empty mask, ascending (per-warp contiguous ranges)
    {
        const unsigned char *m8 = (const unsigned char *)mask;
        const int per = RW / WARPS;
        int cnt = 0;
        for (int i = lane; i < per; i += 32) cnt += m8[warp * per + i] != 0;
#pragma unroll
        for (int off = 16; off; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
        if (lane == 0) s_base[warp + 1] = cnt;
        __syncthreads();
        if (tid == 0) {
            s_base[0] = 0;
            for (int w2 = 0; w2 < WARPS; w2++) s_base[w2 + 1] += s_base[w2];
            s_n = s_base[WARPS];
        }
        __syncthreads();
        int o = s_base[warp];
        for (int i0 = 0; i0 < per; i0 += 32) {
            const int i = i0 + lane;
            const bool f = i < per && m8[warp * per + i] != 0;
            const unsigned bal = __ballot_sync(0xffffffffu, f);
            if (f) list[o + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)(warp * per + i);
            o += __popc(bal);
        }
    }
    for (int i = tid; i < WARPS * RG_MAX; i += THREADS) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const int nl = s_n;
    const unsigned char *m8 = (const unsigned char *)mask;
    // rows: warp w takes list entries w, w + WARPS, ...
    int cnt[GR];
#pragma unroll
    for (int g = 0; g < GR; g++) cnt[g] = 0;
    for (int e = warp; e < nl; e += WARPS) {
        const int x = list[e];
        const uint32_t mm = m8[x];
        const float4 *xr = (const float4 *)(X + (lo + x) * (int64_t)pitch);
        double acc[GR];
#pragma unroll
        for (int g = 0; g < GR; g++) acc[g] = 0.0;
#pragma unroll 2
        for (int v = lane; v < nvec; v += 32) {
            const float4 u = __ldg(xr + v);
#pragma unroll
            for (int g = 0; g < GR; g++)
                if ((mm >> g) & 1u) acc4(acc[g], u, q4_at(qd + (size_t)g * pitch, v, nvec));
        }
        const int64_t gid = gid_base + lo + x;
#pragma unroll
        for (int g = 0; g < GR; g++) {
            if (!((mm >> g) & 1u)) continue;
            const double d = warp_sum(acc[g]);
            double *myd = Ld + ((size_t)warp * GR + g) * k;
            int64_t *myi = Li + ((size_t)warp * GR + g) * k;
            if (cnt[g] < k || less_di(d, gid, myd[k - 1], myi[k - 1])) warp_insert(myd, myi, cnt[g], k, d, gid, lane);
        }
    }
    if (lane == 0)
#pragma unroll
        for (int g = 0; g < GR; g++) wcnt[warp][g] = cnt[g];
    __syncthreads();
    // per query: merge the WARPS lists by rank into the partial list of (query, range)
    const int NR = gridDim.x;
    for (int g = 0; g < ng; g++) {
        const int64_t q = qs[g];
        double *od = part_d + ((int64_t)q * NR + blockIdx.x) * k;
        int64_t *oi = part_i + ((int64_t)q * NR + blockIdx.x) * k;
        for (int r = tid; r < k; r += THREADS) {
            od[r] = INFINITY;
            oi[r] = -1;
        }
        __syncthreads();
        for (int e2 = tid; e2 < WARPS * k; e2 += THREADS) {
            const int w = e2 / k, i = e2 % k;
            if (i >= wcnt[w][g]) continue;
            const double d = Ld[((size_t)w * GR + g) * k + i];
            const int64_t id = Li[((size_t)w * GR + g) * k + i];
            int rank = i;
            for (int w2 = 0; w2 < WARPS; w2++) {
                if (w2 == w) continue;
                int l2 = 0, h2 = wcnt[w2][g];
                const double *L2d = Ld + ((size_t)w2 * GR + g) * k;
                const int64_t *L2i = Li + ((size_t)w2 * GR + g) * k;
                while (l2 < h2) {
                    const int md = (l2 + h2) >> 1;
                    if (less_di(L2d[md], L2i[md], d, id)) l2 = md + 1;
                    else h2 = md;
                }
                rank += l2;
            }
            if (rank < k) {
                od[rank] = d;
                oi[rank] = id;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// merge of L sorted lists (d, id; id < 0 = padding) of length k per query ->
// final top-k.  Used for the S partial lists of a query and for the G shards.
// lists layout: [(q*L + l)*k + i] (stride_q = L*k)  or shards [(l*Q + q)*k + i]
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(THREADS) k_merge_lists(const double *__restrict__ d, const int64_t *__restrict__ ids,
                                                          int L, int64_t Q, int k, int shard_major,
                                                          double *__restrict__ out_d64, float *__restrict__ out_d,
                                                          int64_t *__restrict__ out_i) {
    const int64_t q = blockIdx.x;
    auto idx = [&](int l, int i) -> int64_t {
        return shard_major ? (((int64_t)l * Q + q) * k + i) : ((q * L + l) * (int64_t)k + i);
    };
    for (int r = threadIdx.x; r < k; r += THREADS) {
        if (out_d64) out_d64[q * k + r] = INFINITY;
        if (out_d) out_d[q * k + r] = INFINITY;
        out_i[q * k + r] = -1;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < L * k; e += THREADS) {
        int l = e / k, i = e % k;
        int64_t id = ids[idx(l, i)];
        if (id < 0) continue;
        double dv = d[idx(l, i)];
        int rank = i;
        for (int l2 = 0; l2 < L; l2++) {
            if (l2 == l) continue;
            int lo = 0, hi = k;
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                int64_t mi = ids[idx(l2, mid)];
                bool lt = mi >= 0 && less_di(d[idx(l2, mid)], mi, dv, id);
                if (lt) lo = mid + 1;
                else hi = mid;
            }
            rank += lo;
        }
        if (rank < k) {
            if (out_d64) out_d64[q * k + rank] = dv;
            if (out_d) out_d[q * k + rank] = (float)dv;
            out_i[q * k + rank] = id;
        }
    }
}

// ---------------------------------------------------------------------------
// Optimized Mode (phi=1), stage a4: Hamming order (Z9 ties by id).
// k_hamming: grid (HS, Qc); CTA s of query q takes a contiguous slice of the
// ascending-id candidate list, G lanes per candidate read its code words
// (coalesced), h = popcount(b(q') xor b(x)); per-CTA histogram of h, flushed
// to a per-query histogram with one atomic per non-empty bin.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(THREADS) k_hamming(const float *__restrict__ qrot, int pitch, int Dp,
                                                      const uint64_t *__restrict__ codes, int Wd,
                                                      const int32_t *__restrict__ pool, int64_t CAPQ,
                                                      const int32_t *__restrict__ cbase,
                                                      const int32_t *__restrict__ ncand, int NB,
                                                      uint16_t *__restrict__ hbuf, int32_t *__restrict__ ghist,
                                                      const int32_t *__restrict__ only_fb,
                                                      const int32_t *__restrict__ qperm) {
    extern __shared__ __align__(16) unsigned char sm[];
    uint64_t *qc = (uint64_t *)sm;          // Wd
    int *hist = (int *)(qc + Wd);           // Dp + 1
    int *pre = hist + Dp + 1;               // NB + 1
    int *cbs = pre + NB + 1;                // NB
    const int64_t q = qperm ? qperm[blockIdx.y] : blockIdx.y;  // locality order (query_order)
    if (only_fb && !only_fb[q]) return;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float *qrow = qrot + q * pitch;
    for (int w = tid; w < Wd; w += THREADS) {
        uint64_t word = 0;
        for (int i = 0; i < 64; i++) {
            const int d = w * 64 + i;
            if (d < Dp && qrow[d] > 0.0f) word |= (uint64_t)1 << i;  // b(q') with the [x > 0] convention (Z10)
        }
        qc[w] = word;
    }
    for (int i = tid; i < Dp + 1; i += THREADS) hist[i] = 0;
    block_prefix(ncand, cbase, q, NB, pre, cbs);
    __syncthreads();
    const int total = pre[NB];
    const int per = (total + gridDim.x - 1) / gridDim.x;
    const int v_lo = blockIdx.x * per, v_hi = min(total, v_lo + per);
    // G lanes per candidate, each loading at most two code words
    int G = 1;
    while (G < 32 && G * 2 < Wd) G <<= 1;
    const int gpw = 32 / G, g = lane / G, gl = lane % G;
    const int32_t *poolq = pool + q * CAPQ;
    int bl = 0;  // block of this lane's candidate (monotone in v)
    for (int v0 = v_lo + warp * 32; v0 < v_hi; v0 += WARPS * 32) {
        const int v = v0 + lane;
        int lid = -1, pos = 0;
        if (v < v_hi) {
            while (pre[bl + 1] <= v) bl++;
            pos = cbs[bl] + (v - pre[bl]);
            lid = __ldg(poolq + pos);
        }
#pragma unroll 4
        for (int r = 0; r < 32 / gpw; r++) {
            const int src = r * gpw + g;
            const int lr = __shfl_sync(0xffffffffu, lid, src);
            const int ps = __shfl_sync(0xffffffffu, pos, src);
            int hv = 0;
            if (lr >= 0) {
                const uint64_t *cr = codes + (int64_t)lr * Wd;
                if (gl < Wd) hv = __popcll(qc[gl] ^ __ldg(cr + gl));
                if (gl + G < Wd) hv += __popcll(qc[gl + G] ^ __ldg(cr + gl + G));
            }
            for (int off = G >> 1; off; off >>= 1) hv += __shfl_xor_sync(0xffffffffu, hv, off);
            if (lr >= 0 && gl == 0) {
                hbuf[q * CAPQ + ps] = (uint16_t)hv;  // h at the candidate's pool position
                atomicAdd(&hist[hv], 1);
            }
        }
    }
    __syncthreads();
    int32_t *gh = ghist + q * (int64_t)(Dp + 1);
    for (int i = tid; i < Dp + 1; i += THREADS)
        if (hist[i]) atomicAdd(&gh[i], hist[i]);
}

// k_hamming_dense (a4, phi=1, after k_count_warp without the fused popcount):
// the query's candidates occupy pool positions [0, |C_q|) exactly (segment
// bases come from a cursor starting at 0), so a CTA takes a contiguous range
// of positions: 4 lanes per candidate with 16-byte code loads, h written at
// the position, a CTA histogram flushed to the query's histogram.
template <int HT>
__global__ void __launch_bounds__(THREADS, HT > 2 ? 2 : 4) k_hamming_dense(const float *__restrict__ qrot, int pitch, int Dp,
                                                            const uint64_t *__restrict__ codes, int Wd,
                                                            const int32_t *__restrict__ pool, int64_t CAPQ,
                                                            const int32_t *__restrict__ cursor,
                                                            uint16_t *__restrict__ hbuf, int32_t *__restrict__ ghist,
                                                            const int32_t *__restrict__ fb,
                                                            const int32_t *__restrict__ qperm) {
    extern __shared__ __align__(16) unsigned char sm[];
    uint64_t *qc = (uint64_t *)sm;     // Wd
    int *hist = (int *)(qc + Wd);      // Dp + 1
    const int64_t q = qperm ? qperm[blockIdx.y] : blockIdx.y;
    if (fb[q]) return;  // the fallback replaced C_q: k_hamming handles it
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float *qrow = qrot + q * pitch;
    for (int d0 = warp * 32; d0 < Wd * 64; d0 += THREADS) {
        const int d = d0 + lane;
        const unsigned bits = __ballot_sync(0xffffffffu, d < Dp && qrow[d] > 0.0f);
        if (lane == 0) ((uint32_t *)qc)[d0 >> 5] = bits;
    }
    for (int i = tid; i < Dp + 1; i += THREADS) hist[i] = 0;
    __syncthreads();
    const int total = (int)min((int64_t)cursor[q], CAPQ);
    const int per = (total + gridDim.x - 1) / gridDim.x;
    const int lo = blockIdx.x * per, hi = min(total, lo + per);
    const int32_t *poolq = pool + q * CAPQ;
    const int g4 = lane >> 2, gl = lane & 3, nt = Wd >> 3;
    // the ids of the next pass are loaded before this pass's code rows
    int idn[4];
#pragma unroll
    for (int r = 0; r < 4; r++) {
        const int v = lo + warp * 32 + r * 8 + g4;
        idn[r] = v < hi ? __ldg(poolq + v) : 0;
    }
    for (int v0 = lo + warp * 32; v0 < hi; v0 += WARPS * 32) {
        int id[4];
        bool okv[4];
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const int v = v0 + r * 8 + g4;
            okv[r] = v < hi;
            id[r] = idn[r];
            const int vn = v + WARPS * 32;
            idn[r] = vn < hi ? __ldg(poolq + vn) : 0;
        }
        int hr[4] = {0, 0, 0, 0};
        // HT 16-byte chunks of each of the 4 rows issued together before their popcounts
        // (DRAM-bound at cfg4: the loads in flight set the rate)
        for (int t0 = 0; t0 < nt; t0 += HT) {
            ulonglong2 cw[HT][4];
#pragma unroll
            for (int tt = 0; tt < HT; tt++)
#pragma unroll
                for (int r = 0; r < 4; r++)
                    cw[tt][r] = t0 + tt < nt ? __ldg((const ulonglong2 *)(codes + (int64_t)id[r] * Wd + 2 * gl + 8 * (t0 + tt)))
                                             : make_ulonglong2(0ull, 0ull);
#pragma unroll
            for (int tt = 0; tt < HT; tt++) {
                const int wd = 2 * gl + 8 * min(t0 + tt, nt - 1);
                const uint64_t q0 = t0 + tt < nt ? qc[wd] : 0ull, q1 = t0 + tt < nt ? qc[wd + 1] : 0ull;
#pragma unroll
                for (int r = 0; r < 4; r++) hr[r] += __popcll(q0 ^ cw[tt][r].x) + __popcll(q1 ^ cw[tt][r].y);
            }
        }
        uint32_t p01 = (uint32_t)hr[0] | ((uint32_t)hr[1] << 16), p23 = (uint32_t)hr[2] | ((uint32_t)hr[3] << 16);
        p01 += __shfl_xor_sync(0xffffffffu, p01, 1);
        p23 += __shfl_xor_sync(0xffffffffu, p23, 1);
        p01 += __shfl_xor_sync(0xffffffffu, p01, 2);
        p23 += __shfl_xor_sync(0xffffffffu, p23, 2);
        if (gl == 0) {
            const int hh[4] = {(int)(p01 & 0xffffu), (int)(p01 >> 16), (int)(p23 & 0xffffu), (int)(p23 >> 16)};
#pragma unroll
            for (int r = 0; r < 4; r++)
                if (okv[r]) {
                    hbuf[q * CAPQ + v0 + r * 8 + g4] = (uint16_t)hh[r];
                    atomicAdd(&hist[hh[r]], 1);
                }
        }
    }
    __syncthreads();
    int32_t *gh = ghist + q * (int64_t)(Dp + 1);
    for (int i = tid; i < Dp + 1; i += THREADS)
        if (hist[i]) atomicAdd(&gh[i], hist[i]);
}

// k_hamming_seg (a4, phi=1): the same h, segment-major.  Grid (query groups,
// candidate segments) with the segment as the slow index: the CTAs in flight
// all work inside one id block, whose code rows (BF x 8 Wd bytes, 24 MB at
// cfg4) stay in L2 while every query's candidates in that block are scored,
// so each code row comes from DRAM about once per step instead of once per
// query that holds it.  A warp takes one query of the group (its b(q') in its
// own shared slice) and that query's candidates of the segment, 4 lanes per
// candidate; h goes to the candidate's pool position (k_hhist then builds the
// per-query histograms).
template <int HT>
__global__ void __launch_bounds__(THREADS, 4) k_hamming_seg(const uint64_t *__restrict__ qcodes,
                                                          const uint64_t *__restrict__ codes, int Wd,
                                                          const int32_t *__restrict__ pool, int64_t CAPQ,
                                                          const int32_t *__restrict__ cbase,
                                                          const int32_t *__restrict__ ncand, int NS, int64_t Qn,
                                                          uint16_t *__restrict__ hbuf, const int32_t *__restrict__ fb,
                                                          const int32_t *__restrict__ qperm) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint64_t *qc = (uint64_t *)sm + warp * Wd;  // this warp's b(q')
    const int64_t qi = (int64_t)blockIdx.x * WARPS + warp;
    if (qi >= Qn) return;
    const int64_t q = qperm ? qperm[qi] : qi;
    if (fb[q]) return;  // the fallback replaced C_q: k_hamming handles it
    const int sb = blockIdx.y;
    const int n = ncand[q * NS + sb];
    if (n <= 0) return;
    for (int i = lane; i < Wd; i += 32) qc[i] = qcodes[q * Wd + i];
    __syncwarp();
    const int base = cbase[q * NS + sb];
    const int32_t *poolq = pool + q * CAPQ + base;
    uint16_t *hq = hbuf + q * CAPQ + base;
    const int g4 = lane >> 2, gl = lane & 3, nt = Wd >> 3;
    int idn[4];
#pragma unroll
    for (int r = 0; r < 4; r++) {
        const int v = r * 8 + g4;
        idn[r] = v < n ? __ldg(poolq + v) : 0;
    }
    for (int v0 = 0; v0 < n; v0 += 32) {
        int id[4];
        bool okv[4];
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const int v = v0 + r * 8 + g4;
            okv[r] = v < n;
            id[r] = idn[r];
            const int vn = v + 32;
            idn[r] = vn < n ? __ldg(poolq + vn) : 0;
        }
        int hr[4] = {0, 0, 0, 0};
        for (int t0 = 0; t0 < nt; t0 += HT) {
            ulonglong2 cw[HT][4];
#pragma unroll
            for (int tt = 0; tt < HT; tt++)
#pragma unroll
                for (int r = 0; r < 4; r++)
                    cw[tt][r] = t0 + tt < nt ? __ldg((const ulonglong2 *)(codes + (int64_t)id[r] * Wd + 2 * gl + 8 * (t0 + tt)))
                                             : make_ulonglong2(0ull, 0ull);
#pragma unroll
            for (int tt = 0; tt < HT; tt++) {
                const int wd = 2 * gl + 8 * min(t0 + tt, nt - 1);
                const uint64_t q0 = t0 + tt < nt ? qc[wd] : 0ull, q1 = t0 + tt < nt ? qc[wd + 1] : 0ull;
#pragma unroll
                for (int r = 0; r < 4; r++) hr[r] += __popcll(q0 ^ cw[tt][r].x) + __popcll(q1 ^ cw[tt][r].y);
            }
        }
        uint32_t p01 = (uint32_t)hr[0] | ((uint32_t)hr[1] << 16), p23 = (uint32_t)hr[2] | ((uint32_t)hr[3] << 16);
        p01 += __shfl_xor_sync(0xffffffffu, p01, 1);
        p23 += __shfl_xor_sync(0xffffffffu, p23, 1);
        p01 += __shfl_xor_sync(0xffffffffu, p01, 2);
        p23 += __shfl_xor_sync(0xffffffffu, p23, 2);
        if (gl == 0) {
            const int hh[4] = {(int)(p01 & 0xffffu), (int)(p01 >> 16), (int)(p23 & 0xffffu), (int)(p23 >> 16)};
#pragma unroll
            for (int r = 0; r < 4; r++)
                if (okv[r]) hq[v0 + r * 8 + g4] = (uint16_t)hh[r];
        }
    }
}

// b(q') of every query (Wd words; bit (i mod 64) of word i/64 = [q'_i > 0], Z10), warp per query
__global__ void k_qcodes(const float *__restrict__ qrot, int pitch, int Dp, int Wd, int64_t Qn,
                         uint64_t *__restrict__ qcodes) {
    const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (q >= Qn) return;
    const float *qrow = qrot + q * pitch;
    for (int d0 = 0; d0 < Wd * 64; d0 += 32) {
        const int d = d0 + lane;
        const unsigned bits = __ballot_sync(0xffffffffu, d < Dp && qrow[d] > 0.0f);
        if (lane == 0) ((uint32_t *)(qcodes + q * Wd))[d0 >> 5] = bits;
    }
}

// per-query histogram of h over the dense pool positions (after k_hamming_seg)
__global__ void __launch_bounds__(THREADS) k_hhist(int Dp, const int32_t *__restrict__ cursor, int64_t CAPQ,
                                                   const uint16_t *__restrict__ hbuf, int32_t *__restrict__ ghist,
                                                   const int32_t *__restrict__ fb) {
    extern __shared__ __align__(16) unsigned char sm[];
    int *hist = (int *)sm;  // Dp + 1
    const int64_t q = blockIdx.x;
    if (fb[q]) return;
    for (int i = threadIdx.x; i < Dp + 1; i += THREADS) hist[i] = 0;
    __syncthreads();
    const int total = (int)min((int64_t)cursor[q], CAPQ);
    const uint16_t *hq = hbuf + q * CAPQ;
    for (int v = threadIdx.x; v < total; v += THREADS) atomicAdd(&hist[hq[v]], 1);
    __syncthreads();
    int32_t *gh = ghist + q * (int64_t)(Dp + 1);
    for (int i = threadIdx.x; i < Dp + 1; i += THREADS)
        if (hist[i]) atomicAdd(&gh[i], hist[i]);
}

// k_hsort: one warp per query; stable counting sort of the ascending-id list by
// h -> order (h, id), written over the query's pool region.
// One warp: bin starts of the per-query histogram (start[], Dp+1) and the
// stable scatter of the ascending-id candidate list by h into `out`.  Only the
// bins whose start is below `limit` are scattered (the positions the
// speculative rounds read); limit = INT_MAX scatters everything.
__device__ int hsort_warp(const int32_t *__restrict__ gh, int Dp, const int32_t *__restrict__ cq,
                          const uint16_t *__restrict__ hq, const int *pre, const int *cbs, int32_t *__restrict__ out,
                          int *start, int limit) {
    // cq/hq: the query's pool (ids, h) at candidate positions; pre/cbs: the
    // segment prefix and bases (ascending id order = ascending segments)
    const int lane = threadIdx.x & 31;
    int acc = 0, cut = -1;
    for (int b0 = 0; b0 < Dp + 1; b0 += 32) {
        const int i = b0 + lane;
        const int v = i < Dp + 1 ? gh[i] : 0;
        int inc = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, off);
            if (lane >= off) inc += t;
        }
        const int st = acc + inc - v;
        if (i < Dp + 1) start[i] = st;
        const unsigned below = __ballot_sync(0xffffffffu, i < Dp + 1 && st < limit);
        if (below) cut = b0 + 31 - __clz(below);  // starts are monotone
        acc += __shfl_sync(0xffffffffu, inc, 31);
    }
    const int total = acc;
    __syncwarp();
    const bool full = cut >= Dp;
    constexpr int U = 8;  // chunks of 32 loaded ahead (independent loads)
    int bl = 0;           // segment of this lane's position (monotone)
    for (int v00 = 0; v00 < total; v00 += 32 * U) {
        int hh[U], ll[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int v = v00 + u * 32 + lane;
            hh[u] = 0x7fffffff;
            ll[u] = 0;
            if (v < total) {
                while (pre[bl + 1] <= v) bl++;
                const int pos = cbs[bl] + (v - pre[bl]);
                hh[u] = hq[pos];
                ll[u] = cq[pos];
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int h = hh[u];
            const bool qual = h <= cut;
            const unsigned qm = __ballot_sync(0xffffffffu, qual);
            if (!qm) continue;
            int rank = 0, cnt = 0, leader = 32;
            if (full) {
                if (qual) {
                    const unsigned peers = __match_any_sync(qm, h);
                    leader = __ffs(peers) - 1;
                    rank = __popc(peers & ((1u << lane) - 1));
                    cnt = __popc(peers);
                }
            } else {
                for (unsigned m = qm; m; m &= m - 1) {  // few qualifying lanes: O(qualifying)
                    const int j = __ffs(m) - 1;
                    const int hj = __shfl_sync(0xffffffffu, h, j);
                    if (qual && hj == h) {
                        if (leader == 32) leader = j;
                        rank += j < lane;
                        cnt++;
                    }
                }
            }
            int base = 0;
            if (qual && lane == leader) {
                base = start[h];
                start[h] = base + cnt;
            }
            base = __shfl_sync(0xffffffffu, base, qual ? leader : lane);
            if (qual) out[base + rank] = ll[u];
            __syncwarp();
        }
    }
    return total;
}

// k_hsort: one warp per query; order (h, id) of the positions the speculative
// rounds read, written over the query's pool region.
__device__ void warp_segments(const int32_t *__restrict__ ncand, const int32_t *__restrict__ cbase, int64_t q, int NS,
                              int *pre, int *cbs) {
    const int lane = threadIdx.x & 31;
    int acc = 0;
    for (int b0 = 0; b0 < NS; b0 += 32) {
        const int b = b0 + lane;
        int v = b < NS ? ncand[q * NS + b] : 0;
        if (b < NS) cbs[b] = cbase[q * NS + b];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, v, off);
            if (lane >= off) v += t;
        }
        if (b < NS) pre[b + 1] = acc + v;
        acc += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) pre[0] = 0;
    __syncwarp();
}

// k_hsort_cta: the same (h, id) order of the bins below the cut with a CTA per
// query: each warp takes a contiguous range of the ascending candidate list,
// counts its qualifying elements per bin, the per-(warp, bin) offsets follow
// from the bin starts (stable: earlier warps first), and each warp scatters
// its range in order.  smem: start (Dp+1), segments (2NS+1), counts WARPS x (Dp+1).
template <bool LIST>
__global__ void __launch_bounds__(THREADS) k_hsort_cta(const int32_t *__restrict__ ncand,
                                                        const int32_t *__restrict__ cbase, int NS, int Dp,
                                                        const int32_t *__restrict__ ghist,
                                                        const int32_t *__restrict__ pool,
                                                        const uint16_t *__restrict__ hbuf, int64_t CS,
                                                        int32_t *__restrict__ order, int32_t *__restrict__ total_out,
                                                        int limit) {
    extern __shared__ __align__(16) unsigned char sm[];
    int *start = (int *)sm;         // Dp + 1
    int *pre = start + Dp + 1;      // NS + 1
    int *cbs = pre + NS + 1;        // NS
    int *wcnt = cbs + NS;           // WARPS x HSORT_BW (one window of bins)
    __shared__ int s_total, s_cut;
    const int64_t q = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int HB = Dp + 1;
    if (warp == 0) {
        warp_segments(ncand, cbase, q, NS, pre, cbs);
        const int32_t *gh = ghist + q * (int64_t)HB;
        int acc = 0, cut = -1;
        for (int b0 = 0; b0 < HB; b0 += 32) {
            const int i = b0 + lane;
            const int v = i < HB ? gh[i] : 0;
            int inc = v;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, off);
                if (lane >= off) inc += t;
            }
            const int st = acc + inc - v;
            if (i < HB) start[i] = st;
            const unsigned below = __ballot_sync(0xffffffffu, i < HB && st < limit);
            if (below) cut = b0 + 31 - __clz(below);  // starts are monotone
            acc += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) {
            s_total = acc;
            s_cut = cut;
        }
    }
    __syncthreads();
    const int total = s_total, cut = s_cut;
    const int per = (total + WARPS - 1) / WARPS;
    const int lo = min(total, warp * per), hi = min(total, lo + per);
    const int32_t *cq = pool + q * CS;
    const uint16_t *hq = hbuf + q * CS;
    int *mycnt = wcnt + warp * HSORT_BW;
    int bl0 = 0;  // segment holding position lo
    {
        int a = 0, b = NS;  // largest a with pre[a] <= lo
        while (b - a > 1) {
            const int mid = (a + b) >> 1;
            if (pre[mid] <= lo) a = mid;
            else b = mid;
        }
        bl0 = a;
    }
    constexpr int U = 8;
    // the qualifying bins [0, cut] in windows of HSORT_BW bins (the per-warp counters cover
    // one window: ~45 KB of shared memory instead of 8 (D'+1) ints, so several CTAs fit an
    // SM; at cfg4 every query's cut lies in the first window).  Per window, phase A counts
    // this warp's elements per bin; the per-(warp, bin) output offsets follow; phase B
    // scatters them stably.  LIST: window 0's phase A also lists the pool positions of all
    // qualifying elements, in order, in the unused tail of the query's order row ([total,
    // CS), capw per warp), and later work visits only them.
    int32_t *out = order + q * CS;
    constexpr bool listing = LIST;
    const int64_t capw64 = listing ? (CS - total) / WARPS : 0;
    const int capw = capw64 < (1 << 30) ? (int)capw64 : (1 << 30);
    int32_t *scr = out + total + (int64_t)warp * capw;
    __shared__ int s_over;
    if (tid == 0) s_over = listing ? 0 : 1;
    int nq = 0;
    for (int w0 = 0; w0 <= cut; w0 += HSORT_BW) {
        const int w1 = min(cut, w0 + HSORT_BW - 1);
        const int nbw = w1 - w0 + 1;
        for (int i = tid; i < WARPS * HSORT_BW; i += THREADS) wcnt[i] = 0;
        __syncthreads();  // counters zeroed (and s_over initialised)
        const bool use_list = listing && w0 > 0 && !s_over;
        if (use_list) {
            for (int i0 = 0; i0 < nq; i0 += 32) {
                const int i = i0 + lane;
                const int h = i < nq ? (int)hq[scr[i]] : 0x7fffffff;
                if (h >= w0 && h <= w1) atomicAdd(&mycnt[h - w0], 1);
            }
        } else {
            int bl = bl0;
            for (int v00 = lo; v00 < hi; v00 += 32 * U) {
                int hh[U], pp[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int v = v00 + u * 32 + lane;
                    hh[u] = 0x7fffffff;
                    pp[u] = 0;
                    if (v < hi) {
                        while (pre[bl + 1] <= v) bl++;
                        pp[u] = cbs[bl] + (v - pre[bl]);
                        hh[u] = hq[pp[u]];
                    }
                }
#pragma unroll
                for (int u = 0; u < U; u++) {
                    if (hh[u] >= w0 && hh[u] <= w1) atomicAdd(&mycnt[hh[u] - w0], 1);
                    if (listing && w0 == 0) {
                        const bool qual = hh[u] <= cut;
                        const unsigned qm = __ballot_sync(0xffffffffu, qual);
                        const int r = nq + __popc(qm & ((1u << lane) - 1));
                        if (qual && r < capw) scr[r] = pp[u];
                        nq += __popc(qm);
                    }
                }
            }
            if (listing && w0 == 0 && lane == 0 && nq > capw) atomicOr(&s_over, 1);
        }
        __syncthreads();
        // per-(warp, bin) output offsets: bin start + the bin's elements of earlier warps
        for (int h = tid; h < nbw; h += THREADS) {
            int run = start[w0 + h];
            for (int w2 = 0; w2 < WARPS; w2++) {
                const int c = wcnt[w2 * HSORT_BW + h];
                wcnt[w2 * HSORT_BW + h] = run;
                run += c;
            }
        }
        __syncthreads();
        // one element per lane: stable placement within its bin (peers ranked by lane)
        auto place = [&](bool inw, int h, int id) {
            const unsigned qm = __ballot_sync(0xffffffffu, inw);
            if (!qm) return;
            int rank = 0, cnt = 0, leader = 32;
            if (inw) {
                const unsigned peers = __match_any_sync(qm, h);
                leader = __ffs(peers) - 1;
                rank = __popc(peers & ((1u << lane) - 1));
                cnt = __popc(peers);
            }
            int base = 0;
            if (inw && lane == leader) {
                base = mycnt[h - w0];
                mycnt[h - w0] = base + cnt;
            }
            base = __shfl_sync(0xffffffffu, base, inw ? leader : lane);
            if (inw) out[base + rank] = id;
            __syncwarp();
        };
        if (listing && !s_over) {
            // phase B over the listed qualifying elements only, in order
            for (int i0 = 0; i0 < nq; i0 += 32) {
                const int i = i0 + lane;
                const int pos = i < nq ? scr[i] : 0;
                const int h = i < nq ? (int)hq[pos] : 0x7fffffff;
                const bool inw = h >= w0 && h <= w1;
                place(inw, h, inw ? cq[pos] : 0);
            }
        } else {
            // phase B: stable scatter of this warp's range
            int bl = bl0;
            for (int v00 = lo; v00 < hi; v00 += 32 * U) {
                int hh[U], ll[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int v = v00 + u * 32 + lane;
                    hh[u] = 0x7fffffff;
                    ll[u] = 0;
                    if (v < hi) {
                        while (pre[bl + 1] <= v) bl++;
                        const int pos = cbs[bl] + (v - pre[bl]);
                        hh[u] = hq[pos];
                        ll[u] = cq[pos];
                    }
                }
#pragma unroll
                for (int u = 0; u < U; u++) place(hh[u] >= w0 && hh[u] <= w1, hh[u], ll[u]);
            }
        }
        __syncthreads();  // the window's counters are reused next
    }
    if (tid == 0) total_out[q] = total;
}

__global__ void __launch_bounds__(32) k_hsort(const int32_t *__restrict__ ncand, const int32_t *__restrict__ cbase,
                                              int NS, int Dp, const int32_t *__restrict__ ghist,
                                              const int32_t *__restrict__ pool, const uint16_t *__restrict__ hbuf,
                                              int64_t CS, int32_t *__restrict__ order, int32_t *__restrict__ total_out,
                                              int limit) {
    extern __shared__ __align__(16) unsigned char sm[];
    int *start = (int *)sm;       // Dp + 1
    int *pre = start + Dp + 1;    // NS + 1
    int *cbs = pre + NS + 1;      // NS
    const int64_t q = blockIdx.x;
    warp_segments(ncand, cbase, q, NS, pre, cbs);
    const int total = hsort_warp(ghist + q * (int64_t)(Dp + 1), Dp, pool + q * CS, hbuf + q * CS, pre, cbs,
                                 order + q * CS, start, limit);
    if (threadIdx.x == 0) total_out[q] = total;
}

// ---------------------------------------------------------------------------
// Optimized Mode, stage a5: exact L2 in (h, id) order with patience.
// Speculative rounds: k_verify_rows computes dist64 of candidates
// [r*S0, (r+1)*S0) of every unfinished query in parallel (HBM streaming like
// the Guaranteed-Mode kernel); k_patience_scan then replays them in order per
// query (warp per query) and stops exactly where the sequential rule stops.
// Queries still running after the speculative rounds finish in k_patience_tail.
// ---------------------------------------------------------------------------
struct PatState {
    double *Td;       // Qc x k, sorted top-k distances
    int64_t *Ti;      // Qc x k, their global ids
    int32_t *cnt;     // Qc, entries in the top-k list
    int32_t *pat;     // Qc, consecutive non-improving verifications
    int32_t *done;    // Qc
    int64_t *nver;    // Qc, rows verified when done
    int32_t *pos;     // Qc, next position of the query's order to verify
    int32_t *nlen;    // Qc, rows of its next round (certainly needed: P - pat, clamped)
};

// rows [j0, j0 + n) of query q in a verification round: the round's fixed span
// (j0r >= 0) or the query's own (j0r < 0: st.pos, st.nlen), inside its order
// and below the positions k_hsort ordered (send)
__device__ __forceinline__ int round_span(const PatState &st, int64_t q, int j0r, int len, int total, int send,
                                          int &j0) {
    if (j0r < 0) {
        j0 = st.pos[q];
        len = st.nlen[q];
    } else
        j0 = j0r;
    return max(0, min(min(len, total - j0), send - j0));
}

template <bool ROWS4>
__global__ void __launch_bounds__(THREADS, ROWS4 ? 6 : 5) k_verify_rows(const float *__restrict__ qrot, int pitch,
                                                          const float *__restrict__ X, const int32_t *__restrict__ pool,
                                                          int64_t PS, const int32_t *__restrict__ totals,
                                                          PatState st, int j0r, int len, int send,
                                                          int dstride, double *__restrict__ dbuf,
                                                          const int32_t *__restrict__ qperm) {
    extern __shared__ __align__(16) unsigned char sm[];
    double *qd = (double *)sm;
    const int64_t q = qperm ? qperm[blockIdx.y] : blockIdx.y;  // locality order (query_order)
    if (st.done[q]) return;
    const int total = totals[q];
    int j0;
    const int n = round_span(st, q, j0r, len, total, send, j0);
    if (n <= 0) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    load_qd(qd, qrot + q * pitch, pitch);
    __syncthreads();
    const int nvec = pitch / 4;
    const int W = gridDim.x * WARPS;
    const int32_t *ord = pool + q * PS + j0;
    double *dq = dbuf + q * (int64_t)dstride;
    for (int j = blockIdx.x * WARPS + warp; j < n; j += 4 * W) {
        if (ROWS4 && j + 3 * W < n) {
            double d4[4];
            row_dist4(X + (int64_t)ord[j] * pitch, X + (int64_t)ord[j + W] * pitch, X + (int64_t)ord[j + 2 * W] * pitch,
                      X + (int64_t)ord[j + 3 * W] * pitch, qd, nvec, lane, d4);
            if (lane == 0) {
                dq[j] = d4[0];
                dq[j + W] = d4[1];
                dq[j + 2 * W] = d4[2];
                dq[j + 3 * W] = d4[3];
            }
            continue;
        }
        for (int jj = j; jj < n; jj += 2 * W) {
            const int j1 = jj + W;
            const int l0 = ord[jj];
            if (j1 < n) {
                double d0, d1;
                row_dist2(X + (int64_t)l0 * pitch, X + (int64_t)ord[j1] * pitch, qd, nvec, lane, d0, d1);
                if (lane == 0) {
                    dq[jj] = d0;
                    dq[j1] = d1;
                }
            } else {
                const double d0 = row_dist1(X + (int64_t)l0 * pitch, qd, nvec, lane);
                if (lane == 0) dq[jj] = d0;
            }
        }
        break;  // the two-row loop took every remaining row of this warp
    }
}

// A verification round >= 1 with the filter (R17): every row of the span is
// first bounded through its int8 copy against the query's k-th best distance
// at the start of the round (the k-th best only shrinks, so a miss certified
// against it is a miss at the row's own turn); only rows the bound cannot
// exclude are read in fp32 for their exact distance.  Excluded rows get +inf
// in dbuf, which the in-order replay (k_patience_scan) counts as a miss,
// exactly as their exact distance would be.
template <int MINB>
__global__ void __launch_bounds__(THREADS, MINB) k_verify_rows_lb(const float *__restrict__ qrot, int pitch,
                                                             const float *__restrict__ X, FiltArgs fa,
                                                             const int32_t *__restrict__ pool, int64_t PS,
                                                             const int32_t *__restrict__ totals, PatState st, int k,
                                                             int j0r, int len, int send, int dstride,
                                                             double *__restrict__ dbuf,
                                                             const int32_t *__restrict__ qperm,
                                                             unsigned long long *__restrict__ fstats) {
    extern __shared__ __align__(16) unsigned char sm[];
    double *qd = (double *)sm;                   // pitch
    uint4 *sq = (uint4 *)(qd + pitch);           // 2 nv16 (the query's digit planes)
    const int64_t q = qperm ? qperm[blockIdx.y] : blockIdx.y;
    if (st.done[q]) return;
    const int total = totals[q];
    int j0;
    const int n = round_span(st, q, j0r, len, total, send, j0);
    if (n <= 0) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    load_qd(qd, qrot + q * pitch, pitch);
    const QTerms qt = load_q8(sq, fa, q);
    __syncthreads();
    // threshold sqrt(d_k) (1 + 1e-9); none while the top-k is not full
    const double thr = (qt.ok && st.cnt[q] >= k) ? sqrt(st.Td[q * k + k - 1]) * (1.0 + 1e-9) : -1.0;
    const int nvec = pitch / 4;
    const int W = gridDim.x * WARPS;
    const int32_t *ord = pool + q * PS + j0;
    double *dq = dbuf + q * (int64_t)dstride;
    unsigned nb = 0, ne = 0;
    // rows the bound keeps wait in a per-warp queue and are read four at a time
    int *eq_j = (int *)(sq + 2 * fa.nv16) + warp * 64, *eq_r = eq_j + 32;
    int eqn = 0;  // warp-uniform
    auto exact_flush = [&](int min_rows) {
        while (eqn >= min_rows && eqn > 0) {
            __syncwarp();
            const int m = min(eqn, 4);
            int jr[4], rr[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                jr[u] = eq_j[max(0, eqn - 1 - u)];
                rr[u] = eq_r[max(0, eqn - 1 - u)];
            }
            if (m == 4) {
                double d4[4];
                row_dist4(X + (int64_t)rr[0] * pitch, X + (int64_t)rr[1] * pitch, X + (int64_t)rr[2] * pitch,
                          X + (int64_t)rr[3] * pitch, qd, nvec, lane, d4);
                if (lane == 0) {
#pragma unroll
                    for (int u = 0; u < 4; u++) dq[jr[u]] = d4[u];
                }
            } else if (m >= 2) {
                double d0, d1;
                row_dist2(X + (int64_t)rr[0] * pitch, X + (int64_t)rr[1] * pitch, qd, nvec, lane, d0, d1);
                if (lane == 0) {
                    dq[jr[0]] = d0;
                    dq[jr[1]] = d1;
                }
                if (m == 3) {
                    const double d2 = row_dist1(X + (int64_t)rr[2] * pitch, qd, nvec, lane);
                    if (lane == 0) dq[jr[2]] = d2;
                }
            } else {
                const double d0 = row_dist1(X + (int64_t)rr[0] * pitch, qd, nvec, lane);
                if (lane == 0) dq[jr[0]] = d0;
            }
            eqn -= m;
            ne += m;
            __syncwarp();
        }
    };
    int j = blockIdx.x * WARPS + warp;
    int nxt[4];  // the next group's row ids, loaded one group ahead
#pragma unroll
    for (int u = 0; u < 4; u++) nxt[u] = j + u * W < n ? ord[j + u * W] : -1;
    for (; j < n; j += 4 * W) {
        int rows[4], nr = 0;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            rows[u] = nxt[u];
            nr += rows[u] >= 0;
            const int jn = j + (4 + u) * W;
            nxt[u] = jn < n ? ord[jn] : -1;
        }
        unsigned need;  // rows whose exact distance is needed (bit u: row u)
        if (thr < 0.0) {
            need = (1u << nr) - 1u;
        } else {
            const uint4 *r4[4];
#pragma unroll
            for (int u = 0; u < 4; u++) r4[u] = fa.C8 + (int64_t)(rows[u] >= 0 ? rows[u] : rows[0]) * fa.nv16;
            int S1[4], S2[4];
            rows_q8<4>(r4, sq, fa.nv16, lane, S1, S2);
            nb += nr;
            // lane u bounds row u
            int s1 = 0, s2 = 0, rr = -1;
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (lane == u) {
                    s1 = S1[u];
                    s2 = S2[u];
                    rr = rows[u];
                }
            bool keep = false;
            if (rr >= 0) {
                double lb, ub;
                filt_bounds(qt, s1, s2, __ldg(fa.meta + rr), lb, ub);
                keep = !(lb > thr);
                if (!keep) dq[j + lane * W] = INFINITY;
            }
            need = __ballot_sync(0xffffffffu, keep);
        }
        // queue the kept rows (warp-uniform bookkeeping; lane 0 writes)
        if (need) {
            if (lane == 0) {
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if ((need >> u) & 1u) {
                        eq_j[eqn] = j + u * W;
                        eq_r[eqn] = rows[u];
                        eqn++;
                    }
            }
            eqn = __shfl_sync(0xffffffffu, eqn, 0);
            if (eqn >= 28) exact_flush(4);
        }
    }
    exact_flush(1);
    if (fstats && lane == 0 && (nb | ne)) {
        atomicAdd(fstats, (unsigned long long)nb);
        atomicAdd(fstats + 1, (unsigned long long)(thr < 0.0 ? 0 : ne));
    }
}

// Block-major filtered round (opt-in CRISP_LB_BLOCKS=1; measured slower): the same bounds as
// k_verify_rows_lb, but the rows of every running query's span are first
// bucketed by id block (BSZ ids, k_span_bucket), and k_verify_lb_blk takes
// (query group, id block) with the block as the slow grid index, so the int8
// rows of one block (BSZ x c8pitch bytes, ~50 MB) stay in L2 while all the
// queries' rows in it are bounded: a row is read from DRAM about once per
// round instead of once per query that verifies it.  Exact distances of the
// kept rows read q' from global memory (same arithmetic and order as
// row_dist*: identical values).
__device__ __forceinline__ Q4 q4_g(const float4 *__restrict__ q4, int v) {
    const float4 t = __ldg(q4 + v);
    return {(double)t.x, (double)t.y, (double)t.z, (double)t.w};
}
__device__ __forceinline__ void row_dist4_g(const float *__restrict__ r0, const float *__restrict__ r1,
                                            const float *__restrict__ r2, const float *__restrict__ r3,
                                            const float *__restrict__ qrow, int nvec, int lane, double (&o)[4]) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const float4 *x0 = (const float4 *)r0, *x1 = (const float4 *)r1, *x2 = (const float4 *)r2,
                 *x3 = (const float4 *)r3, *q4 = (const float4 *)qrow;
#pragma unroll 2
    for (int v = lane; v < nvec; v += 32) {
        const float4 u0 = __ldg(x0 + v), u1 = __ldg(x1 + v), u2 = __ldg(x2 + v), u3 = __ldg(x3 + v);
        const Q4 qv = q4_g(q4, v);
        acc4(a0, u0, qv);
        acc4(a1, u1, qv);
        acc4(a2, u2, qv);
        acc4(a3, u3, qv);
    }
    o[0] = warp_sum(a0);
    o[1] = warp_sum(a1);
    o[2] = warp_sum(a2);
    o[3] = warp_sum(a3);
}
__device__ __forceinline__ double row_dist1_g(const float *__restrict__ r0, const float *__restrict__ qrow, int nvec,
                                              int lane) {
    double a0 = 0.0;
    const float4 *x0 = (const float4 *)r0, *q4 = (const float4 *)qrow;
#pragma unroll 4
    for (int v = lane; v < nvec; v += 32) acc4(a0, __ldg(x0 + v), q4_g(q4, v));
    return warp_sum(a0);
}

// per running query (CTA): its span's (id, position) pairs grouped by id block
__global__ void __launch_bounds__(256) k_span_bucket(const int32_t *__restrict__ pool, int64_t PS,
                                                     const int32_t *__restrict__ totals, PatState st, int send,
                                                     int BSH, int NBB, int DS, int2 *__restrict__ spair,
                                                     int32_t *__restrict__ boff) {
    extern __shared__ __align__(16) unsigned char sm[];
    int *cnt = (int *)sm;  // NBB + 1
    const int64_t q = blockIdx.x;
    int32_t *bo = boff + q * (int64_t)(NBB + 1);
    if (st.done[q]) {
        for (int b = threadIdx.x; b <= NBB; b += blockDim.x) bo[b] = 0;
        return;
    }
    int j0;
    const int n = round_span(st, q, -1, 0, totals[q], send, j0);
    const int32_t *ord = pool + q * PS + j0;
    for (int b = threadIdx.x; b <= NBB; b += blockDim.x) cnt[b] = 0;
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) atomicAdd(&cnt[ord[j] >> BSH], 1);
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of the counts (one warp)
        int carry = 0;
        for (int b0 = 0; b0 <= NBB; b0 += 32) {
            const int b = b0 + threadIdx.x;
            const int v = b <= NBB ? cnt[b] : 0;
            int inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o);
                if ((int)threadIdx.x >= o) inc += t;
            }
            if (b <= NBB) {
                bo[b] = carry + inc - v;
                cnt[b] = carry + inc - v;  // running insert position
            }
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
    __syncthreads();
    int2 *sp = spair + q * (int64_t)DS;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const int id = ord[j];
        sp[atomicAdd(&cnt[id >> BSH], 1)] = make_int2(id, j);
    }
}

template <int QPC>
__global__ void __launch_bounds__(THREADS, 3) k_verify_lb_blk(const float *__restrict__ qrot, int pitch,
                                                           const float *__restrict__ X, FiltArgs fa, PatState st,
                                                           int k, int64_t Qn, int NBB, int DS,
                                                           const int2 *__restrict__ spair,
                                                           const int32_t *__restrict__ boff,
                                                           double *__restrict__ dbuf,
                                                           unsigned long long *__restrict__ fstats) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.y;
    int *eq_j = (int *)sm + warp * 64, *eq_r = eq_j + 32;
    unsigned nb = 0, ne = 0;
    // a CTA takes QPC consecutive queries of block b; warp w takes queries w, w + WARPS, ...
    for (int64_t q = (int64_t)blockIdx.x * QPC + warp; q < min(Qn, (int64_t)(blockIdx.x + 1) * QPC); q += WARPS) {
    if (st.done[q]) continue;
    const int32_t *bo = boff + q * (int64_t)(NBB + 1);
    const int p0 = bo[b], p1 = bo[b + 1];
    if (p0 >= p1) continue;
    const double *qi = fa.qi + q * 4;
    const QTerms qt{qi[0], qi[1], qi[2], qi[3] != 0.0};
    const double thr = (qt.ok && st.cnt[q] >= k) ? sqrt(st.Td[q * k + k - 1]) * (1.0 + 1e-9) : -1.0;
    const uint4 *sq = fa.qd + q * 2 * fa.nv16;  // the digit planes (global; L1 keeps them)
    const float *qrow = qrot + q * pitch;
    const int nvec = pitch / 4;
    const int2 *sp = spair + q * (int64_t)DS;
    double *dq = dbuf + q * (int64_t)DS;
    int eqn = 0;
    auto exact_flush = [&](int min_rows) {
        while (eqn >= min_rows && eqn > 0) {
            __syncwarp();
            const int m = min(eqn, 4);
            int jr[4], rr[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                jr[u] = eq_j[max(0, eqn - 1 - u)];
                rr[u] = eq_r[max(0, eqn - 1 - u)];
            }
            if (m == 4) {
                double d4[4];
                row_dist4_g(X + (int64_t)rr[0] * pitch, X + (int64_t)rr[1] * pitch, X + (int64_t)rr[2] * pitch,
                            X + (int64_t)rr[3] * pitch, qrow, nvec, lane, d4);
                if (lane == 0) {
#pragma unroll
                    for (int u = 0; u < 4; u++) dq[jr[u]] = d4[u];
                }
            } else {
                for (int u = 0; u < m; u++) {
                    const double d0 = row_dist1_g(X + (int64_t)rr[u] * pitch, qrow, nvec, lane);
                    if (lane == 0) dq[jr[u]] = d0;
                }
            }
            eqn -= m;
            ne += m;
            __syncwarp();
        }
    };
    for (int p = p0; p < p1; p += 4) {
        int rows[4], jj[4], nr = 0;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int2 e = p + u < p1 ? sp[p + u] : make_int2(-1, 0);
            rows[u] = e.x;
            jj[u] = e.y;
            nr += e.x >= 0;
        }
        unsigned need;
        if (thr < 0.0) {
            need = (1u << nr) - 1u;
        } else {
            const uint4 *r4[4];
#pragma unroll
            for (int u = 0; u < 4; u++) r4[u] = fa.C8 + (int64_t)(rows[u] >= 0 ? rows[u] : rows[0]) * fa.nv16;
            int S1[4], S2[4];
            rows_q8<4>(r4, sq, fa.nv16, lane, S1, S2);
            nb += nr;
            int s1 = 0, s2 = 0, rr = -1, jl = 0;
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (lane == u) {
                    s1 = S1[u];
                    s2 = S2[u];
                    rr = rows[u];
                    jl = jj[u];
                }
            bool keep = false;
            if (rr >= 0) {
                double lb, ub;
                filt_bounds(qt, s1, s2, __ldg(fa.meta + rr), lb, ub);
                keep = !(lb > thr);
                if (!keep) dq[jl] = INFINITY;
            }
            need = __ballot_sync(0xffffffffu, keep);
        }
        if (need) {
            if (lane == 0) {
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if ((need >> u) & 1u) {
                        eq_j[eqn] = jj[u];
                        eq_r[eqn] = rows[u];
                        eqn++;
                    }
            }
            eqn = __shfl_sync(0xffffffffu, eqn, 0);
            if (eqn >= 28) exact_flush(4);
        }
    }
    exact_flush(1);
    if (thr < 0.0) ne = 0;
    }
    if (fstats && lane == 0 && (nb | ne)) {
        atomicAdd(fstats, (unsigned long long)nb);
        atomicAdd(fstats + 1, (unsigned long long)ne);
    }
}

// ADSampling context of Optimized Mode verification (Eq. 2; crisp_set_adsampling)
struct AdCtx {
    int on;
    double eps0;
    int stride;
    int Dp;
    const float *X;   // stored rows (pitch floats)
    int pitch;
    int64_t gid_base;
    const float *q;   // this query's q' (fp32, pitch floats)
};

// Eq. 2 threshold r_k^2 * (t/D) * (1 + eps0/sqrt(t))^2, in the oracle's order
__device__ __forceinline__ double ad_thr(double rk2, int t, int D, double eps0) {
    const double f = __dadd_rn(1.0, __ddiv_rn(eps0, __dsqrt_rn((double)t)));
    return __dmul_rn(__ddiv_rn(__dmul_rn(rk2, (double)t), (double)D), __dmul_rn(f, f));
}

// Eq. 2 decided exactly as the oracle does: the partial sums in dimension
// order (the dist64 chain), checked at t = stride, 2*stride, ... < D.  Used
// only for candidates that would enter the top-k (for every other candidate
// pruned and non-improving are the same outcome).  The warp first forms the
// partial sums in parallel (prefix scans, 128 dims per step) and the
// thresholds (one checkpoint per lane); a decision whose partial sum is
// farther than 1e-12 relative from its threshold is the sequential chain's
// decision too (the two sums of non-negative terms differ by < t * 2^-52
// relative).  Only if a checkpoint is that close does lane 0 run the
// sequential chain itself.
__device__ bool ad_pruned_seq(const AdCtx &ad, int64_t gid, double rk2, int lane) {
    const float4 *x4 = (const float4 *)(ad.X + (gid - ad.gid_base) * (int64_t)ad.pitch);
    const float4 *q4 = (const float4 *)ad.q;
    const int nv = ad.Dp / 4, per = ad.stride >> 2, ncp = (ad.Dp - 1) / ad.stride;  // checkpoints t < D
    double run = 0.0;
    int verdict = 0;  // 0 undecided, 1 pruned, 2 not pruned, 3 ambiguous
    for (int v0 = 0; v0 < nv && verdict == 0; v0 += 32) {
        const int v = v0 + lane;
        double p = 0.0;
        if (v < nv) {
            const float4 xv = __ldg(x4 + v), qv = __ldg(q4 + v);
            const float xa[4] = {xv.x, xv.y, xv.z, xv.w}, qa[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const double d = __dsub_rn((double)qa[c], (double)xa[c]);
                p = __fma_rn(d, d, p);
            }
        }
        double sc = p;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, sc, off);
            if (lane >= off) sc = __dadd_rn(sc, t);
        }
        const double s = __dadd_rn(run, sc);
        const int cp = (v + 1) / per;  // checkpoint index + 1 when (v + 1) % per == 0
        bool above = false, close = false;
        if (v < nv && (v + 1) % per == 0 && cp <= ncp) {
            const double th = ad_thr(rk2, cp * ad.stride, ad.Dp, ad.eps0);
            above = s > __dmul_rn(th, 1.0 + 1e-12);
            close = !above && s >= __dmul_rn(th, 1.0 - 1e-12);
        }
        const unsigned ma = __ballot_sync(0xffffffffu, above), mc = __ballot_sync(0xffffffffu, close);
        if (ma | mc) verdict = (mc && (!ma || __ffs(mc) < __ffs(ma))) ? 3 : 1;  // the first decisive checkpoint
        run = __dadd_rn(run, __shfl_sync(0xffffffffu, sc, 31));
    }
    if (verdict == 0) verdict = 2;
    if (verdict != 3) return verdict == 1;
    int pr = 0;  // ambiguous: the sequential chain, as the oracle
    if (lane == 0) {
        double s = 0.0;
        for (int v = 0; v < nv && !pr; v++) {
            const float4 xv = __ldg(x4 + v), qv = __ldg(q4 + v);
            const float xa[4] = {xv.x, xv.y, xv.z, xv.w}, qa[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const double d = __dsub_rn((double)qa[c], (double)xa[c]);
                s = __fma_rn(d, d, s);
                const int t = 4 * v + c + 1;
                if (!pr && t % ad.stride == 0 && t < ad.Dp && s > ad_thr(rk2, t, ad.Dp, ad.eps0)) pr = 1;
            }
        }
    }
    return __shfl_sync(0xffffffffu, pr, 0) != 0;
}

// One row under ADSampling with a certified early stop (warp per row): the
// partial sums are formed 128 dimensions at a time (lane partials of 4 dims and
// a warp prefix scan), and the row stops at the first checkpoint whose partial
// exceeds thr(t) * (1 + 1e-12).  That margin exceeds the difference between
// this summation order and the oracle's sequential chain (< t * 2^-52
// relative for sums of non-negative terms), so a stopped row is pruned in the
// sequential rule under this r_k, and so under any smaller r_k met later in
// the same round (Eq. 2 is monotone in r_k).  Returns NaN for a stopped row,
// else the full squared distance.  thr: thresholds per checkpoint c (t =
// (c+1)*stride), already times (1 + 1e-12).
__device__ __forceinline__ double ad_row(const float *__restrict__ row, const double *__restrict__ qd, int nvec, int Dp,
                                         int stride, const double *__restrict__ thr, bool prune, int lane) {
    const float4 *x4 = (const float4 *)row;
    double run = 0.0;
    const int per = stride >> 2;  // float4s per checkpoint interval
    for (int v0 = 0; v0 < nvec; v0 += 32) {
        const int v = v0 + lane;
        double p = 0.0;
        if (v < nvec) acc4(p, __ldg(x4 + v), q4_at(qd, v, nvec));
        double sc = p;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, sc, off);
            if (lane >= off) sc = __dadd_rn(sc, t);
        }
        if (prune) {
            const int t = 4 * (v + 1);  // dimensions up to and including this lane's float4
            bool over = false;
            if (v < nvec && (v + 1) % per == 0 && t < Dp) over = __dadd_rn(run, sc) > thr[(v + 1) / per - 1];
            if (__ballot_sync(0xffffffffu, over)) return __longlong_as_double(0x7ff8000000000000LL);  // NaN
        }
        run = __dadd_rn(run, __shfl_sync(0xffffffffu, sc, 31));
    }
    return run;
}

// k_verify_rows_ad: a speculative round under ADSampling.  r_k^2 is the query's
// k-th best at the start of the round (+inf while fewer than k: no pruning).
__global__ void __launch_bounds__(THREADS) k_verify_rows_ad(const float *__restrict__ qrot, int pitch, int Dp,
                                                             const float *__restrict__ X,
                                                             const int32_t *__restrict__ pool, int64_t PS,
                                                             const int32_t *__restrict__ totals, PatState st, int k,
                                                             int j0r, int len, int send, int dstride,
                                                             double *__restrict__ dbuf,
                                                             const int32_t *__restrict__ qperm, double eps0,
                                                             int stride) {
    extern __shared__ __align__(16) unsigned char sm[];
    double *qd = (double *)sm;      // pitch
    double *thr = qd + pitch;       // Dp / stride
    const int64_t q = qperm ? qperm[blockIdx.y] : blockIdx.y;
    if (st.done[q]) return;
    const int total = totals[q];
    int j0;
    const int n = round_span(st, q, j0r, len, total, send, j0);
    if (n <= 0) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool prune = st.cnt[q] >= k;
    const double rk2 = prune ? st.Td[q * k + k - 1] : 0.0;
    load_qd(qd, qrot + q * pitch, pitch);
    for (int c = threadIdx.x; c < Dp / stride; c += THREADS)
        thr[c] = __dmul_rn(ad_thr(rk2, (c + 1) * stride, Dp, eps0), 1.0 + 1e-12);
    __syncthreads();
    const int nvec = pitch / 4;
    const int W = gridDim.x * WARPS;
    const int32_t *ord = pool + q * PS + j0;
    double *dq = dbuf + q * (int64_t)dstride;
    for (int j = blockIdx.x * WARPS + warp; j < n; j += W) {
        const double d = ad_row(X + (int64_t)ord[j] * pitch, qd, nvec, Dp, stride, thr, prune, lane);
        if (lane == 0) dq[j] = d;
    }
}

// one warp scans up to 32 (d, id) entries (lanes >= gn invalid) against the
// top-k list with the patience counter; returns the stop index or -1
// The patience rule over one group of <= 32 verified candidates in order
// (myd: exact d, or NaN = pruned by a round's certified early stop).  With
// ADSampling a candidate that would enter a full top-k is first checked
// against Eq. 2 under the current r_k; pruned candidates count as misses.
__device__ __forceinline__ int patience_group(double myd, int64_t myi, int gn, double *Td, int64_t *Ti, int &cnt_top,
                                              int &pat, int k, int P, int lane, const AdCtx *ad = nullptr) {
    int start = 0;
    while (start < gn) {
        const bool full = cnt_top >= k;
        const double wdv = full ? Td[k - 1] : 0.0;
        const int64_t wiv = full ? Ti[k - 1] : 0;
        const bool better = lane >= start && lane < gn && !isnan(myd) && (!full || less_di(myd, myi, wdv, wiv));
        const unsigned mask = __ballot_sync(0xffffffffu, better);
        const int f = mask ? (__ffs(mask) - 1) : gn;
        const int nonimp = f - start;
        if (P > 0 && pat + nonimp >= P) return start + (P - pat) - 1;  // the P-th consecutive miss
        pat += nonimp;
        if (f >= gn) break;
        const double dd = __shfl_sync(0xffffffffu, myd, f);
        const int64_t ii = __shfl_sync(0xffffffffu, myi, f);
        if (ad && ad->on && full && ad_pruned_seq(*ad, ii, wdv, lane)) {
            if (P > 0 && pat + 1 >= P) return f;
            pat += 1;
            start = f + 1;
            continue;
        }
        warp_insert(Td, Ti, cnt_top, k, dd, ii, lane);
        pat = 0;
        start = f + 1;
    }
    return -1;
}

__device__ __forceinline__ void write_topk(int64_t q, int k, int cnt_top, const double *Td, const int64_t *Ti,
                                           double *out_d64, float *out_d, int64_t *out_i, int lane, int stride) {
    for (int r = lane; r < k; r += stride) {
        const double dv = r < cnt_top ? Td[r] : INFINITY;
        const int64_t iv = r < cnt_top ? Ti[r] : -1;
        if (out_d64) out_d64[q * k + r] = dv;
        if (out_d) out_d[q * k + r] = (float)dv;
        out_i[q * k + r] = iv;
    }
}

// warp per query; dynamic smem WARPS x k (d, id) + WARPS x 32 PSCAN_G staged (d, id)
constexpr int PSCAN_G = 8;
__global__ void __launch_bounds__(THREADS) k_patience_scan(int64_t Qc, const int32_t *__restrict__ totals,
                                                            const int32_t *__restrict__ pool, int64_t PS,
                                                            int64_t gid_base, const double *__restrict__ dbuf, int j0r,
                                                            int len, int send, int nl_min, int nl_max, int dstride,
                                                            int k, int P, PatState st,
                                                            double *__restrict__ out_d64, float *__restrict__ out_d,
                                                            int64_t *__restrict__ out_i, AdCtx ad,
                                                            const float *__restrict__ qrot) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t q = (int64_t)blockIdx.x * WARPS + warp;
    if (q >= Qc || st.done[q]) return;
    double *Td = (double *)sm + warp * k;
    int64_t *Ti = (int64_t *)((double *)sm + WARPS * k) + warp * k;
    int cnt_top = st.cnt[q], pat = st.pat[q];
    for (int i = lane; i < cnt_top; i += 32) {
        Td[i] = st.Td[q * k + i];
        Ti[i] = st.Ti[q * k + i];
    }
    __syncwarp();
    const int total = totals[q];
    int j0;
    const int n = round_span(st, q, j0r, len, total, send, j0);
    const int32_t *ord = pool + q * PS + j0;
    const double *dq = dbuf + q * (int64_t)dstride;
    ad.q = qrot + q * (int64_t)ad.pitch;
    // PSCAN_G groups of 32 entries staged per warp with all loads in flight, then
    // replayed group by group from shared memory
    double *sd = (double *)((int64_t *)((double *)sm + WARPS * k) + WARPS * k) + warp * (32 * PSCAN_G);
    int64_t *si = (int64_t *)((double *)sm + WARPS * k) + WARPS * k + WARPS * (32 * PSCAN_G) + warp * (32 * PSCAN_G);
    int64_t stop = -1;
    for (int c0 = 0; c0 < n && stop < 0; c0 += 32 * PSCAN_G) {
        double vd[PSCAN_G];
        int32_t vi[PSCAN_G];
#pragma unroll
        for (int u = 0; u < PSCAN_G; u++) {
            const int j = c0 + u * 32 + lane;
            vd[u] = j < n ? dq[j] : INFINITY;
            vi[u] = j < n ? ord[j] : 0;
        }
#pragma unroll
        for (int u = 0; u < PSCAN_G; u++) {
            sd[u * 32 + lane] = vd[u];
            si[u * 32 + lane] = gid_base + vi[u];
        }
        __syncwarp();
        for (int g0 = c0; g0 < min(n, c0 + 32 * PSCAN_G) && stop < 0; g0 += 32) {
            const int gn = min(32, n - g0);
            const double myd = lane < gn ? sd[g0 - c0 + lane] : INFINITY;
            const int64_t myi = lane < gn ? si[g0 - c0 + lane] : 0x7fffffffffffffffLL;
            const int s = patience_group(myd, myi, gn, Td, Ti, cnt_top, pat, k, P, lane, &ad);
            if (s >= 0) stop = (int64_t)j0 + g0 + s + 1;
        }
        __syncwarp();
    }
    const bool fin = stop >= 0 || j0 + n >= total;
    for (int i = lane; i < cnt_top; i += 32) {
        st.Td[q * k + i] = Td[i];
        st.Ti[q * k + i] = Ti[i];
    }
    if (lane == 0) {
        st.cnt[q] = cnt_top;
        st.pat[q] = pat;
        if (fin) {
            st.done[q] = 1;
            st.nver[q] = stop >= 0 ? stop : total;
        } else {
            // still running: at least P - pat more rows are verified (no improvement
            // can stop it earlier), the span of its next round
            st.pos[q] = j0 + n;
            st.nlen[q] = P > 0 ? min(nl_max, max(nl_min, P - pat)) : nl_max;
        }
    }
    if (fin) write_topk(q, k, cnt_top, Td, Ti, out_d64, out_d, out_i, lane, 32);
}

// CTA per query still running after the speculative rounds: chunked
// verification from position `from` (all warps compute the chunk's rows, warp
// 0 replays them in order).  k_hsort ordered the positions below sorted_end;
// a query that reaches sorted_end first completes its order.
__global__ void __launch_bounds__(THREADS, 4) k_patience_tail(const float *__restrict__ qrot, int pitch,
                                                            const float *__restrict__ X, int64_t gid_base,
                                                            int32_t *__restrict__ order, int64_t PS,
                                                            const int32_t *__restrict__ totals,
                                                            int sorted_end, int rows4, int k, int P,
                                                            PatState st, double *__restrict__ out_d64,
                                                            float *__restrict__ out_d, int64_t *__restrict__ out_i,
                                                            int Dp, const int32_t *__restrict__ ghist,
                                                            const int32_t *__restrict__ pool,
                                                            const uint16_t *__restrict__ hbuf,
                                                            const int32_t *__restrict__ ncand,
                                                            const int32_t *__restrict__ cbase, int NS,
                                                            const int32_t *__restrict__ qperm, AdCtx ad) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int64_t q = qperm ? qperm[blockIdx.x] : blockIdx.x;  // locality order (query_order)
    if (st.done[q]) return;
    double *qd = (double *)sm;                       // pitch
    double *chd = qd + pitch;                        // TAIL_CAP
    int64_t *chi = (int64_t *)(chd + TAIL_CAP);      // TAIL_CAP
    double *Td = (double *)(chi + TAIL_CAP);         // k
    int64_t *Ti = (int64_t *)(Td + k);               // k
    double *thr = (double *)(Ti + k);                // Dp / 4 + 1 (ADSampling thresholds of a chunk)
    int *hstart = (int *)(thr + Dp / 4 + 1);         // Dp + 1
    int *spre = hstart + Dp + 1;                     // NS + 1
    int *scbs = spre + NS + 1;                       // NS
    __shared__ int s_stop, s_cnt, s_pat;
    __shared__ int64_t s_nver;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    load_qd(qd, qrot + q * pitch, pitch);
    int cnt_top = st.cnt[q], pat = st.pat[q];
    for (int i = tid; i < cnt_top; i += THREADS) {
        Td[i] = st.Td[q * k + i];
        Ti[i] = st.Ti[q * k + i];
    }
    if (tid == 0) {
        s_stop = 0;
        s_cnt = cnt_top;
        s_pat = pat;
    }
    __syncthreads();
    const int total = totals[q];
    const int32_t *ord = order + q * PS;
    const int nvec = pitch / 4;
    int64_t nver = total;
    ad.q = qrot + q * (int64_t)pitch;
    bool sorted = false;
    // chunk: the rows certainly verified next (P - pat: no improvement can stop the
    // query earlier), at least PATIENCE_CH; ADSampling chunks of PATIENCE_CH
    for (int pos = st.pos[q], n = 0; pos < total; pos += n) {
        n = min(total - pos, ad.on || P == 0 ? PATIENCE_CH : max(PATIENCE_CH, min(TAIL_CAP, P - s_pat)));
        if (!sorted && pos + n > sorted_end) {  // k_hsort ordered only [0, sorted_end): complete the order
            if (warp == 0) {
                warp_segments(ncand, cbase, q, NS, spre, scbs);
                hsort_warp(ghist + q * (int64_t)(Dp + 1), Dp, pool + q * PS, hbuf + q * PS, spre, scbs,
                           order + q * PS, hstart, 0x7fffffff);
            }
            __syncthreads();
            sorted = true;
        }
        if (ad.on) {
            // ADSampling: rows of the chunk with the certified early stop under the
            // r_k at the chunk's start (see ad_row), then the in-order scan
            const bool prune = s_cnt >= k;
            const double rk2 = prune ? Td[k - 1] : 0.0;
            for (int c = tid; c < Dp / ad.stride; c += THREADS)
                thr[c] = __dmul_rn(ad_thr(rk2, (c + 1) * ad.stride, Dp, ad.eps0), 1.0 + 1e-12);
            __syncthreads();
            for (int i = warp; i < n; i += WARPS) {
                const int l0 = ord[pos + i];
                const double d0 = ad_row(X + (int64_t)l0 * pitch, qd, nvec, Dp, ad.stride, thr, prune, lane);
                if (lane == 0) {
                    chd[i] = d0;
                    chi[i] = gid_base + l0;
                }
            }
        } else if (rows4) {
            // four consecutive rows per warp step
            for (int i = warp * 4; i < n; i += WARPS * 4) {
                if (i + 3 < n) {
                    const int l0 = ord[pos + i], l1 = ord[pos + i + 1], l2 = ord[pos + i + 2], l3 = ord[pos + i + 3];
                    double d4[4];
                    row_dist4(X + (int64_t)l0 * pitch, X + (int64_t)l1 * pitch, X + (int64_t)l2 * pitch,
                              X + (int64_t)l3 * pitch, qd, nvec, lane, d4);
                    if (lane < 4) {
                        const int li = lane == 0 ? l0 : lane == 1 ? l1 : lane == 2 ? l2 : l3;
                        chd[i + lane] = d4[lane];
                        chi[i + lane] = gid_base + li;
                    }
                } else {
                    for (int ii = i; ii < n; ii++) {
                        const int l0 = ord[pos + ii];
                        const double d0 = row_dist1(X + (int64_t)l0 * pitch, qd, nvec, lane);
                        if (lane == 0) {
                            chd[ii] = d0;
                            chi[ii] = gid_base + l0;
                        }
                    }
                }
            }
        } else
        for (int i = warp * 2; i < n; i += WARPS * 2) {
            const int l0 = ord[pos + i];
            if (i + 1 < n) {
                const int l1 = ord[pos + i + 1];
                double d0, d1;
                row_dist2(X + (int64_t)l0 * pitch, X + (int64_t)l1 * pitch, qd, nvec, lane, d0, d1);
                if (lane == 0) {
                    chd[i] = d0;
                    chi[i] = gid_base + l0;
                    chd[i + 1] = d1;
                    chi[i + 1] = gid_base + l1;
                }
            } else {
                const double d0 = row_dist1(X + (int64_t)l0 * pitch, qd, nvec, lane);
                if (lane == 0) {
                    chd[i] = d0;
                    chi[i] = gid_base + l0;
                }
            }
        }
        __syncthreads();
        if (warp == 0) {
            int64_t stop = -1;
            for (int g0 = 0; g0 < n && stop < 0; g0 += 32) {
                const int gn = min(32, n - g0);
                const double myd = lane < gn ? chd[g0 + lane] : INFINITY;
                const int64_t myi = lane < gn ? chi[g0 + lane] : 0x7fffffffffffffffLL;
                const int s = patience_group(myd, myi, gn, Td, Ti, cnt_top, pat, k, P, lane, &ad);
                if (s >= 0) stop = (int64_t)pos + g0 + s + 1;
            }
            if (lane == 0) {
                s_cnt = cnt_top;
                s_pat = pat;
                if (stop >= 0) {
                    s_stop = 1;
                    s_nver = stop;
                }
            }
        }
        __syncthreads();
        if (s_stop) {
            nver = s_nver;
            break;
        }
    }
    __syncthreads();
    const int ct = s_cnt;
    write_topk(q, k, ct, Td, Ti, out_d64, out_d, out_i, tid, THREADS);
    if (tid == 0) {
        st.done[q] = 1;
        st.nver[q] = nver;
        st.cnt[q] = ct;
    }
}

// ---------------------------------------------------------------------------
// per-query work counters for the roofline (only when stage timing is on):
// [0] ids streamed by the count (local slice lengths summed over activated
// cells), [1] sum |C_q|, [2] rows verified, [3] fallback queries
// ---------------------------------------------------------------------------
__device__ unsigned long long d_stats[4];
__device__ unsigned long long d_filter_stats[2];  // R17: rows bounded through the int8 copy, of those read exactly
static unsigned long long *d_filter_stats_ptr() {
    void *p = nullptr;
    cudaGetSymbolAddress(&p, d_filter_stats);
    return (unsigned long long *)p;
}
__device__ unsigned long long d_probe_stats[2];  // a1: exact half distances computed, screened walks redone exactly
static unsigned long long *d_probe_stats_ptr() {
    void *p = nullptr;
    cudaGetSymbolAddress(&p, d_probe_stats);
    return (unsigned long long *)p;
}

__global__ void k_stats(const uint32_t *__restrict__ act, const int32_t *__restrict__ act_len, int M, int KK,
                        const int32_t *__restrict__ off2, int NB, const int32_t *__restrict__ ncand, int NS,
                        const int64_t *__restrict__ nver, const int32_t *__restrict__ fb, int64_t Qc) {
    const int64_t q = blockIdx.x;
    unsigned long long ids = 0;
    for (int m = 0; m < M; m++) {
        const int L = act_len[q * M + m];
        for (int r = threadIdx.x; r < L; r += blockDim.x) {
            int c = (int)(act[(q * M + m) * (int64_t)KK + r] & 0xffffu);
            const int32_t *o = off2 + ((int64_t)m * KK + c) * (NB + 1);
            ids += (unsigned long long)(o[NB] - o[0]);
        }
    }
    for (int off = 16; off; off >>= 1) ids += __shfl_xor_sync(0xffffffffu, ids, off);
    if ((threadIdx.x & 31) == 0) atomicAdd(&d_stats[0], ids);
    if (threadIdx.x == 0) {
        unsigned long long c = 0;
        for (int b = 0; b < NS; b++) c += (unsigned long long)ncand[q * NS + b];
        atomicAdd(&d_stats[1], c);
        atomicAdd(&d_stats[2], nver ? (unsigned long long)nver[q] : c);
        atomicAdd(&d_stats[3], (unsigned long long)fb[q]);
    }
}

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------
struct StageEv {
    cudaEvent_t a, b;
    int stage;
};
static thread_local std::vector<StageEv> g_events;
static thread_local double g_stage_ms[8];  // 0 transform 1 probe 2 count 3 fallback 4 verify 5 merge 6 hamming
static std::atomic<bool> g_timing{false};    // process-wide switch (crisp_set_stage_timing); tables are per thread
static std::atomic<bool> g_counters{false};  // the work counters (k_stats, probe and filter tallies) as well
static thread_local int64_t g_launches = 0;  // kernels of this library launched by searches on this thread

bool stage_timing_on() { return g_timing; }

struct StageScope {
    cudaStream_t s;
    int stage;
    cudaEvent_t a = nullptr, b = nullptr;
    StageScope(cudaStream_t s_, int st) : s(s_), stage(st) {
        if (!g_timing) return;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
    }
    ~StageScope() {
        if (!g_timing) return;
        cudaEventRecord(b, s);
        g_events.push_back({a, b, stage});
    }
};

struct DevBuf {
    cudaStream_t s;
    std::vector<void *> ptrs;
    explicit DevBuf(cudaStream_t s_) : s(s_) {}
    template <class T>
    T *alloc(size_t n) {
        void *p = nullptr;
        CRISP_CUDA(cudaMallocAsync(&p, std::max<size_t>(n * sizeof(T), 16), s));
        ptrs.push_back(p);
        return (T *)p;
    }
    ~DevBuf() {
        for (void *p : ptrs) cudaFreeAsync(p, s);
    }
};

static int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return v ? atoi(v) : dflt;
}
static double env_double(const char *name, double dflt) {
    const char *v = getenv(name);
    return v ? atof(v) : dflt;
}

// kernel attributes are per device: set them once for each device a search runs on
static void set_attrs() {
    static std::mutex mu;
    static std::vector<int> done_dev;
    int dev = 0;
    CRISP_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (std::find(done_dev.begin(), done_dev.end(), dev) != done_dev.end()) return;
    CRISP_CUDA(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_count_select, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_count_frag<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_count_frag<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_count_frag<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_count_frag<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_count_frag<32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_count_warp<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_count_warp<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_count_warp<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_count_warp<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_fallback, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_fb_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_fb_select, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_rerank_exact<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_rerank_exact<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_lb_bounds<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_lb_bounds<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_lb_threshold, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_verify_rows_lb<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_span_bucket, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_verify_rows_lb<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_rerank_group<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_rerank_group<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_rerank_group<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_rerank_exact<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_hamming, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_patience_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_hamming_dense<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_hamming_seg<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_hamming_seg<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_hhist, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_hamming_dense<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_hsort, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_hsort_cta<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_hsort_cta<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_verify_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_verify_rows<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_patience_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_verify_rows_ad, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CRISP_CUDA(cudaFuncSetAttribute(k_patience_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    done_dev.push_back(dev);
}

// ---------------------------------------------------------------------------
// Work buffers of one query chunk and the stages that run on them.
// ---------------------------------------------------------------------------
struct Work {
    const crisp_index *ix;
    int k, mode;
    int64_t Qc, CAPQ;
    int rgroup = 0, segw = 0, RW = 0, NR = 0, GR = 0, rg_smem = 0;  // grouped phi=0 re-rank
    ScreenOut *scr = nullptr;  // a1 screen (Qc x 2M), if the screen runs
    int probe_r = 24;
    int S, S1, HS, S0, R0, BPC, count_kernel, count_atom, NS, CF, ham_fused, rows4, ad, adsp, F, DS, round_rows, nl_min, Pq,
        vra_smem;
    // verification filter (R17): phi=1 rounds >= 1 (lbf) / phi=0 two-pass re-rank (lb0)
    FiltArgs fa{};
    int lbf = 0, lb0 = 0, nl_max = 0, vrl_smem = 0, lbb_smem = 0, lbt_smem = 0;
    float2 *lbb = nullptr;
    float *Tq = nullptr;
    int lbblk = 0, BSH = 0, NBB = 0, bkt_smem = 0;  // block-major filtered rounds
    int2 *spair = nullptr;
    int32_t *boff = nullptr;
    // the query's digit planes and bound terms (k_q8_prep), before the filtered kernels
    void q8_prep(int64_t qn, cudaStream_t s) const {
        k_q8_prep<<<(unsigned)qn, 256, 0, s>>>(qrot, ix->pitch, ix->mu, ix->c8pitch, const_cast<uint4 *>(fa.qd),
                                               const_cast<double *>(fa.qi));
        CRISP_LAUNCH();
        g_launches++;
    }
    // end of the speculative rounds (positions the Hamming order must cover)
    // positions k_hsort orders (the rounds stop there; k_patience_tail completes the
    // order of a query that goes further): ADSampling's fixed rounds + 1024, exact:
    // F + 2 max(P, 512) + 1024 (measured: nver <= 3.7 P at cfg2, k = 10)
    int order_end() const {
        return ad && !adsp ? (R0 == 0 ? 0 : F + (R0 - 1) * S0) + 1024
                           : std::max(F, first_round(ix, k)) + 2 * std::max(Pq, 512) + 1024;
    }
    DevBuf buf;
    float *qpad = nullptr, *qrot = nullptr;
    uint32_t *act = nullptr, *erow = nullptr;  // erow: compact activated-cell rows (k_count_frag)
    int32_t *act_len = nullptr, *etot = nullptr;
    int64_t *retr = nullptr;
    int32_t *pool = nullptr, *ncand = nullptr, *cbase = nullptr, *cursor = nullptr, *need = nullptr, *fb = nullptr;
    double *part_d = nullptr, *dbuf = nullptr, *d64tmp = nullptr;
    int64_t *part_i = nullptr, *nver = nullptr;
    int32_t *cbuf = nullptr, *ghist = nullptr, *totals = nullptr;
    uint32_t *qkey = nullptr, *qkey2 = nullptr;
    int32_t *qiota = nullptr, *qperm = nullptr;  // qperm: query locality order (null: identity)
    void *qsort_tmp = nullptr;
    size_t qsort_bytes = 0;
    uint16_t *hbuf = nullptr;
    uint64_t *qcodes = nullptr;  // b(q') per query (k_hamming_seg)
    PatState pst{};
    uint8_t *traceV = nullptr;
    bool full_order = false;  // trace: order every candidate (not only what the rounds read)
    int probe_gs, probe_cb, probe_qpw, probe_smem, count_smem, countw_smem, countw_ham_smem, rx_smem, ham_smem, hsort_smem, hsort_cta_smem, vr_smem, scan_smem, pat_smem;

    // round 0 of exact verification: f P rows rounded up to 64 (every query
    // verifies at least min(P, |C|) rows; measured nver / P: ~1.7 at cfg2, k = 10,
    // ~1.2 at cfg4, k = 100)
    static int64_t patience_rows(const crisp_index *ix, int k) {
        return ix->patience_factor > 0 ? (int64_t)ix->patience_factor * k : 0;
    }
    static int first_round(const crisp_index *ix, int k) {
        const int64_t P = patience_rows(ix, k);
        const double f = env_double("CRISP_PATIENCE_FIRST_F", 1.0);
        const int64_t r = P > 0 ? std::min<int64_t>(1 << 16, std::max<int64_t>(128, ((int64_t)(f * P) + 63) / 64 * 64))
                                : 1024;
        return std::max(32, env_int("CRISP_PATIENCE_FIRST", (int)r));
    }
    static int64_t per_query_bytes(const crisp_index *ix, int k, int mode, int64_t CAPQ, bool traceV) {
        const int KK = ix->K * ix->K;
        const int S = std::max(1, env_int("CRISP_RERANK_SPLITS", 4));
        // >= the dbuf row stride DS of Work()
        const int S0 = std::max({first_round(ix, k), std::max(64, env_int("CRISP_PATIENCE_BATCH", 1024)),
                                 (int)std::min<int64_t>(1 << 16, std::max<int64_t>(patience_rows(ix, k), 1024))});
        int64_t perq = (int64_t)ix->pitch * 8 + (int64_t)ix->M * KK * 8 + (int64_t)ix->M * 12 + CAPQ * 4 + 4 +
                       (int64_t)ix->M * 2 * 16 +
                       (int64_t)ix->NBW * 8 + 64;
        if (mode == 0) perq += (int64_t)std::max<int64_t>(S, (ix->N + 4095) / 4096) * k * 16 + (ix->C8 ? CAPQ * 8 + 4 : 0);
        if (ix->C8) perq += 2 * (int64_t)ix->c8pitch + 32;  // query digit planes + bound terms
        else perq += CAPQ * 6 + (int64_t)(ix->Dp + 1) * 4 + (int64_t)S0 * 16 + (int64_t)k * 16 + 32 + (int64_t)ix->Wp * 8 +
                     (ix->N >> 10) * 4 + 8;  // + the span buckets of the block-major filtered rounds
        if (traceV) perq += ix->N;
        return perq;
    }

    Work(const crisp_index *ix_, int k_, int mode_, int64_t Qc_, int64_t CAPQ_, bool want_traceV, bool want_d64tmp,
         cudaStream_t s)
        : ix(ix_), k(k_), mode(mode_), Qc(Qc_), CAPQ(CAPQ_), buf(s) {
        const int M = ix->M, K = ix->K, KK = K * K, NB = ix->NB, BS = ix->BS, pitch = ix->pitch, Dp = ix->Dp;
        S = std::max(1, env_int("CRISP_RERANK_SPLITS", 4));       // CTAs per query in the row kernels
        HS = std::max(1, env_int("CRISP_HAMMING_SPLITS", 2));     // CTAs per query in k_hamming(_dense)
        ad = (mode == 1 && ix->ad_on) ? 1 : 0;
        // speculative rounds (then k_patience_tail): round 0 = F rows, then S0 rows per
        // round for the queries still running (exact: F about 1.75 P, short rounds after;
        // ADSampling: an exact round 0 establishes r_k, later rounds prune under it)
        Pq = (int)std::min<int64_t>(1 << 24, patience_rows(ix, k));
        S0 = std::max(64, env_int("CRISP_PATIENCE_BATCH", 1024));  // ADSampling: rows per round >= 1
        // ADSampling on the exact schedule's per-query spans (else fixed S0-row rounds)
        adsp = ad ? env_int("CRISP_AD_SPANS", 1) : 0;
        R0 = std::max(0, std::min(16, env_int("CRISP_PATIENCE_ROUNDS", ad && !adsp ? 2 : 3)));
        S1 = std::max(1, env_int("CRISP_ROUND_SPLITS", 3));       // CTAs per query, exact rounds >= 1
        nl_min = std::max(32, env_int("CRISP_ROUND_MIN", 64));  // min span of an exact round >= 1
        BPC = std::max(1, std::min(NB, env_int("CRISP_COUNT_BPC", 16)));  // id blocks per count CTA
        // 0: k_count_select (CTA-flattened slices, for many small cells), 1: k_count_warp
        // (warp-owned sub-blocks, for slices of >= 8 ids per sub-block); env overrides
        // 0: k_count_select (CTA-flattened slices, subspace by subspace; kept for comparison),
        // 1: k_count_warp (warp-owned sub-blocks, for slices of >= 8 ids per sub-block),
        // 2: k_count_frag (fragment-flattened, shared atomics; the small-cell regime)
        count_kernel = env_int("CRISP_COUNT_KERNEL", ix->slice_hint >= 8.0 ? 1 : 2);
        CF = std::max(1, std::min(std::min(NB, 4), env_int("CRISP_COUNT_F", 2)));  // k_count_frag: BS ids x CF per CTA
        while (CF > 1 && countf_smem(BS * CF) > 200 * 1024) CF >>= 1;
        // candidate segments per query (id blocks, warp sub-blocks, or frag blocks)
        NS = count_kernel == 0 ? NB : count_kernel == 1 ? ix->NBW : (NB + CF - 1) / CF;
        count_atom = env_int("CRISP_COUNT_ATOM", 0);  // k_count_warp: shared atomics (else byte load/store pairs; faster)
        // phi=1: popcounts inside the count kernel (CRISP_HAMMING_FUSED=1), else k_hamming_dense.
        // Measured at cfg4: fused into k_count_frag 65.4 ms against 21.7 + 16.2 ms separate (each
        // CTA's code-row stream runs after its counting, with only two CTAs per SM); into
        // k_count_warp at cfg2 6.1 against 3.6 + 2.0 ms (r01): off by default
        ham_fused = env_int("CRISP_HAMMING_FUSED", 0);
        if (count_kernel == 2 && ix->Wp > 64) ham_fused = 0;  // b(q') is staged in 64 words
        // row kernels: four rows per warp step for rows up to 4 KB (measured: faster at D=960, slower at 4096)
        rows4 = env_int("CRISP_ROWS4", pitch <= 1024 ? 1 : 0);
        // round 0: exact verification of every query's first F rows.  ADSampling on
        // the spans: only 2k rows (rounded to 64), enough to give most queries an r_k,
        // so that the rows after them are verified under Eq. 2 and pruned early
        // (P:L240-244); exact: F ~ P (first_round)
        // (measured: on these workloads a 2k-row round 0 is slower -- cfg4 verify 81.7 ms against
        // 80.1 exact, cfg2 5.33 ms against 3.25 -- the text-like distances are concentrated
        // (ratio to r_k ~1.3 < Eq. 2's margin), so few rows prune; default: F ~ P as exact)
        if (ad && adsp)
            F = env_int("CRISP_AD_FIRST", 0) > 0
                    ? std::max(64, (std::max(32, env_int("CRISP_AD_FIRST", 0)) + 63) / 64 * 64)
                    : first_round(ix, k);
        else
            F = ad ? std::min(S0, std::max(32, env_int("CRISP_AD_FIRST", S0))) : first_round(ix, k);
        // verification filter: a short exact round 0 (the top-k forms), then rounds whose
        // rows are bounded through the int8 copy against the k-th best at the round's start;
        // spans of at most nl_max rows refresh that threshold as the top-k improves
        // (on when the patience P is long against that round: measured at cfg2, k = 10, P = 400,
        // the extra rounds cost more than the bytes they save, 3.47 against 3.25 ms; at cfg4,
        // k = 100, P = 4000, verification 79.4 -> 34.3 ms.  CRISP_FILTER_ROUNDS=2 forces it)
        {
            const int fr = env_int("CRISP_FILTER_ROUNDS", 1);
            const int F0 = std::max(64, (std::max(k, env_int("CRISP_LB_FIRST", 256)) + 63) / 64 * 64);
            // ADSampling (f1) keeps it: a row the bound excludes has d > the round's d_k >= the running
            // r_k, so it is a miss whether Eq. 2 prunes it or not; the replay applies Eq. 2 to every
            // row that would enter the top-k (patience_group), exactly as the sequential rule
            lbf = (mode == 1 && (!ad || adsp) && ix->C8 && ix->vfilter && fr && (fr == 2 || Pq >= 4 * F0)) ? 1 : 0;
            if (lbf) {
                F = F0;
                R0 = std::max(1, std::min(16, env_int("CRISP_LB_ROUNDS", 6)));
                S1 = std::max(1, env_int("CRISP_ROUND_SPLITS", 2));  // measured at cfg4: 29.1 (2) / 29.8 (3) / 31.6 ms (6)
            }
        }
        DS = std::max({F, S0, std::min(std::max(Pq, nl_min), 1 << 16)});  // dbuf row stride (max span of a round)
        // filtered spans: 2048 rows (cfg4, P = 4000: 29.1 ms; 1024 / 4096: 37.4 / 35.0 ms before the
        // exact-row queue), or P/2 for long patience (cfg3 P = 100k, cfg5 P = 20k: six rounds of 2048 rows
        // left most rows to the unfiltered tail)
        nl_max = lbf ? std::max(nl_min, std::min(DS, env_int("CRISP_LB_SPAN", std::max(2048, Pq / 2)))) : DS;
        if (ix->C8) {
            fa.C8 = (const uint4 *)ix->C8;
            fa.meta = (const int4 *)ix->c8meta;
            fa.nv16 = ix->c8pitch / 16;
        }
        round_rows = std::max(1, env_int("CRISP_ROUND_ROWS", 128));  // min rows per CTA in round 0
        vra_smem = pitch * 8 + (Dp / 4 + 1) * 8;
        qpad = buf.alloc<float>((size_t)Qc * pitch);
        qrot = ix->rotated ? buf.alloc<float>((size_t)Qc * pitch) : qpad;
        act = buf.alloc<uint32_t>((size_t)Qc * M * KK);
        act_len = buf.alloc<int32_t>((size_t)Qc * M);
        retr = buf.alloc<int64_t>((size_t)Qc * M);
        if (count_kernel == 2) {
            erow = buf.alloc<uint32_t>((size_t)Qc * M * KK);
            etot = buf.alloc<int32_t>((size_t)Qc);
        }
        pool = buf.alloc<int32_t>((size_t)Qc * CAPQ);
        ncand = buf.alloc<int32_t>((size_t)Qc * NS);
        cbase = buf.alloc<int32_t>((size_t)Qc * NS);
        cursor = buf.alloc<int32_t>((size_t)Qc + 1);  // [Qc] = overflow need
        need = cursor + Qc;
        fb = buf.alloc<int32_t>((size_t)Qc);
        if (env_int("CRISP_QUERY_ORDER", 1)) {
            qkey = buf.alloc<uint32_t>((size_t)Qc);
            qkey2 = buf.alloc<uint32_t>((size_t)Qc);
            qiota = buf.alloc<int32_t>((size_t)Qc);
            qperm = buf.alloc<int32_t>((size_t)Qc);
            CRISP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, qsort_bytes, qkey, qkey2, qiota, qperm, (int)Qc, 0, 32,
                                                       s));
            qsort_tmp = buf.alloc<unsigned char>(qsort_bytes);
        }
        if (mode == 0) {
            // grouped re-rank (k_rerank_group) for dense candidate sets: the expected share of
            // N a query keeps is about M B / (tau N) (each candidate needs tau of the M
            // activated slices of ~B ids); CRISP_RERANK_GROUP=0/1 forces it
            const double dens = (double)ix->M * (double)ix->budget / ((double)std::max(1, ix->tau) * (double)ix->N_global);
            // measured: slower than k_rerank_exact on cfg3/cfg5 (5.37 s / 13.3 s against 1.45 s / 2.71 s per
            // 10k queries: one 8-warp CTA per SM with one row per warp step cannot keep enough loads
            // in flight), so it is opt-in (CRISP_RERANK_GROUP=1); `dens` is kept for that switch
            rgroup = env_int("CRISP_RERANK_GROUP", 0) != 0 && dens > 0.0 ? 1 : 0;
            segw = count_kernel == 2 ? BS * CF : count_kernel == 1 ? ix->SBW : BS;
            RW = std::min(16384, segw);
            NR = (int)((ix->N + RW - 1) / RW);
            GR = pitch <= 1024 ? 8 : pitch <= 2048 ? 4 : 2;
            rg_smem = GR * pitch * 8 + WARPS * GR * k * 16 + 3 * RW;
            if (rg_smem > 220 * 1024) rgroup = 0;
            const int L = rgroup ? NR : S;
            part_d = buf.alloc<double>((size_t)Qc * L * k);
            part_i = buf.alloc<int64_t>((size_t)Qc * L * k);
            lb0 = (!rgroup && ix->C8 && ix->vfilter && env_int("CRISP_FILTER_RERANK", 1)) ? 1 : 0;
            if (lb0) {
                lbb = buf.alloc<float2>((size_t)Qc * CAPQ);
                Tq = buf.alloc<float>((size_t)Qc);
            }
        } else {
            cbuf = buf.alloc<int32_t>((size_t)Qc * CAPQ);
            hbuf = buf.alloc<uint16_t>((size_t)Qc * CAPQ);
            qcodes = buf.alloc<uint64_t>((size_t)Qc * ix->Wp);
            ghist = buf.alloc<int32_t>((size_t)Qc * (Dp + 1));
            totals = buf.alloc<int32_t>((size_t)Qc);
            dbuf = buf.alloc<double>((size_t)Qc * DS);
            pst.Td = buf.alloc<double>((size_t)Qc * k);
            pst.Ti = buf.alloc<int64_t>((size_t)Qc * k);
            pst.cnt = buf.alloc<int32_t>((size_t)Qc * 5);
            pst.pat = pst.cnt + Qc;
            pst.done = pst.pat + Qc;
            pst.pos = pst.done + Qc;
            pst.nlen = pst.pos + Qc;
            pst.nver = buf.alloc<int64_t>((size_t)Qc);
            nver = pst.nver;
        }
        if (lbf || lb0) {
            fa.qd = buf.alloc<uint4>((size_t)Qc * 2 * fa.nv16);
            fa.qi = buf.alloc<double>((size_t)Qc * 4);
        }
        // block-major filtered rounds (opt-in CRISP_LB_BLOCKS=1).  Measured at cfg4: slower
        // (verify 34.6-35.1 against 29.1 ms): the round-1 DRAM bytes drop only from ~64 to 52 GB
        // (L2 hit rate 44-52%: the CTAs in flight span several id blocks) while the bucketing
        // and the short per-(query, block) tasks add work
        if (lbf && env_int("CRISP_LB_BLOCKS", 0)) {
            // id blocks of 2^BSH ids whose int8 rows take <= ~64 MB (half of L2)
            const int64_t rowb = ix->c8pitch + 16;
            BSH = 10;
            while (BSH < 24 && ((int64_t)1 << (BSH + 1)) * rowb <= (int64_t)64 << 20) BSH++;
            BSH = env_int("CRISP_LB_BSH", BSH);
            NBB = (int)((ix->N + ((int64_t)1 << BSH) - 1) >> BSH);
            bkt_smem = (NBB + 1) * 4;
            if (NBB <= 65535 && bkt_smem <= 200 * 1024) {
                lbblk = 1;
                spair = buf.alloc<int2>((size_t)Qc * DS);
                boff = buf.alloc<int32_t>((size_t)Qc * (NBB + 1));
            }
        }
        if (want_traceV) traceV = buf.alloc<uint8_t>((size_t)Qc * ix->N);
        if (want_d64tmp) d64tmp = buf.alloc<double>((size_t)Qc * k);
        probe_gs = (KK * 4 <= 48 * 1024) ? 1 : 0;
        probe_cb = (2 * K * (ix->dh | 1) * 4 <= 96 * 1024) ? 1 : 0;  // rows padded to an odd stride
        probe_qpw = std::max(1, env_int("CRISP_PROBE_QPW", 4));  // queries per warp in k_probe
        // a1 screen on the tensor cores (CRISP_PROBE_SCREEN=0 disables); dist64 for the
        // centroids that can reach the probe_r smallest of each half
        // The walk pops about L = B K^2 / N cells per subspace (cells of average size); a
        // staircase of L cells reaches ranks ~sqrt(2L) in each half.  The screen certifies a
        // prefix of about probe_r ranks; when that is most of K it saves nothing (and a short
        // prefix would send walks through the exact redo), so the probe then runs unscreened.
        {
            const double L = (double)ix->budget * (double)KK / (double)std::max<int64_t>(1, ix->N_global);
            const int r_auto = std::max(24, (int)std::ceil(2.0 * std::sqrt(2.0 * L)) + 4);
            probe_r = std::max(1, env_int("CRISP_PROBE_R", r_auto));
            const int want = env_int("CRISP_PROBE_SCREEN", probe_r < (4 * K) / 5 ? 1 : 0);
            if (want && screen_supported(ix)) scr = buf.alloc<ScreenOut>((size_t)Qc * 2 * M);
        }
        probe_smem = (probe_gs ? ((KK * 4 + 15) & ~15) : 0) + (probe_cb ? ((2 * K * (ix->dh | 1) * 4 + 15) & ~15) : 0) +
                     WARPS * ((((4 * K + 2 * ix->dh) * 8) + 3 * K + 15) & ~15);
        count_smem = BS + BS / 8 + (int)sizeof(CountSmem);
        countw_smem = (int)countw_fixed_smem(BS);
        countw_ham_smem = ix->Wp * 8 + (Dp + 1) * 4;
        rx_smem = pitch * 8 + WARPS * k * 16 + (2 * NS + 1) * 4;
        ham_smem = ix->Wp * 8 + (Dp + 1) * 4 + (2 * NS + 1) * 4;
        hsort_smem = (Dp + 1 + 2 * NS + 1) * 4;
        hsort_cta_smem = (Dp + 1 + 2 * NS + 1 + WARPS * HSORT_BW) * 4;
        vr_smem = pitch * 8;
        vrl_smem = pitch * 8 + 2 * std::max(16, ix->c8pitch) + WARPS * 64 * 4;
        lbb_smem = 2 * std::max(16, ix->c8pitch) + (2 * NS + 1) * 4;
        lbt_smem = (2 * NS + 1) * 4;
        scan_smem = WARPS * k * 16 + WARPS * 32 * PSCAN_G * 16;
        pat_smem = pitch * 8 + TAIL_CAP * 16 + k * 16 + (Dp / 4 + 1) * 8 + (Dp + 1 + 2 * NS + 1) * 4;
        set_attrs();
        if (lbf && vrl_smem > 220 * 1024) lbf = 0;
        if (lb0 && (lbb_smem > 200 * 1024 || lbt_smem > 140 * 1024)) lb0 = 0;
        CRISP_CHECK(probe_smem <= 200 * 1024 && count_smem <= 200 * 1024 && rx_smem <= 220 * 1024 &&
                        pat_smem <= 220 * 1024 && ham_smem <= 200 * 1024 && scan_smem <= 220 * 1024,
                    "shared-memory footprint too large for this (D, K, k)");
    }
};

// a0, a1+a2, a3+a4 (count/select) for queries [0, qn) of the chunk
static void run_front(Work &w, const float *queries, int64_t qn, cudaStream_t s, const float *hq = nullptr,
                      bool transformed = false) {
    const crisp_index *ix = w.ix;
    const int M = ix->M, K = ix->K, KK = K * K, NB = ix->NB, pitch = ix->pitch;
    // a0 (and a1+a2) in parts; with host queries (hq: the source of the device
    // staging `queries`) part p's H2D copy runs on a side stream while part p-1 is
    // padded, rotated and probed
    const int P = (hq && qn >= 2048) ? std::max(1, std::min(16, env_int("CRISP_H2D_PARTS", 3))) : 1;
    auto probe = [&](int64_t r0, int64_t r1) {
        dim3 g(nblk(r1 - r0, WARPS * w.probe_qpw), M);
        if (w.scr) {  // a1's contraction on the tensor cores: certified screen intervals (probe_tc.cu)
            screen_halves(const_cast<crisp_index *>(ix), w.qrot, r0, r1, w.scr, w.probe_r, s);
            g_launches++;
        }
        k_probe<<<g, THREADS, w.probe_smem, s>>>(w.qrot, pitch, r0, r1, ix->cb, M, K, ix->dh, ix->gsize, w.probe_gs,
                                                 ix->budget, w.mode == 1 ? w.k : 0, w.act, w.act_len, w.retr,
                                                 w.probe_qpw, w.probe_cb, w.scr,
                                                 g_counters ? d_probe_stats_ptr() : nullptr, ix->hoff);
        CRISP_LAUNCH();
        g_launches++;
    };
    // part p of the batch: sizes in the ratio 1 : 2 : ... : P, so that only the small first
    // part's copy is exposed (measured at cfg4, host API: 48.7 ms against 49.0 with equal
    // thirds; CRISP_H2D_TRI=0 keeps equal parts)
    const bool tri = env_int("CRISP_H2D_TRI", 1) != 0;
    auto part_lo = [&](int p) -> int64_t {
        return tri ? qn * ((int64_t)p * (p + 1) / 2) / ((int64_t)P * (P + 1) / 2) : qn * p / P;
    };
    if (transformed) {  // q' given (crisp_transform_queries_async): rows of pitch floats
        StageScope st(s, 0);
        CRISP_CUDA(cudaMemcpyAsync(w.qrot, queries, (size_t)qn * pitch * 4, cudaMemcpyDeviceToDevice, s));
    } else {
        StageScope st(s, 0);
        cudaStream_t cs = nullptr;
        cudaEvent_t ev[17] = {};
        if (hq) {
            CRISP_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            for (auto &e : ev) CRISP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CRISP_CUDA(cudaEventRecord(ev[16], s));  // the staging buffer is allocated on s
            CRISP_CUDA(cudaStreamWaitEvent(cs, ev[16], 0));
            for (int p = 0; p < P; p++) {
                const int64_t r0 = part_lo(p), r1 = part_lo(p + 1);
                CRISP_CUDA(cudaMemcpyAsync((void *)(queries + r0 * ix->D), hq + r0 * ix->D,
                                           (size_t)(r1 - r0) * ix->D * 4, cudaMemcpyHostToDevice, cs));
                CRISP_CUDA(cudaEventRecord(ev[p], cs));
            }
        }
        for (int p = 0; p < P; p++) {
            const int64_t r0 = part_lo(p), r1 = part_lo(p + 1);
            if (hq) CRISP_CUDA(cudaStreamWaitEvent(s, ev[p], 0));
            k_prep_queries<<<nblk((r1 - r0) * pitch, 256), 256, 0, s>>>(queries + r0 * ix->D, r1 - r0, ix->D, pitch,
                                                                        w.qpad + r0 * pitch);
            CRISP_LAUNCH();
            g_launches++;
            if (ix->rotated) {  // int8 tensor cores, certified, else fp64 FMA (rotate_imma.cu)
                rotate_rows(const_cast<crisp_index *>(ix), w.qpad + r0 * pitch, r1 - r0, pitch, w.qrot + r0 * pitch,
                            pitch, s);
                g_launches += 3;  // slices, certify, recompute (+ 8 cuBLASLt GEMMs), or the FMA kernel
            }
            if (P > 1) probe(r0, r1);
        }
        if (hq) {
            for (auto &e : ev) CRISP_CUDA(cudaEventDestroy(e));
            CRISP_CUDA(cudaStreamDestroy(cs));
        }
    }
    {
        StageScope st(s, 1);
        if (P == 1) probe(0, qn);
        if (w.qperm) {
            k_query_key<<<nblk(qn, 256), 256, 0, s>>>(w.act, M, KK, qn, w.qkey, w.qiota);
            CRISP_LAUNCH();
            g_launches++;
            int bits = 1;
            while ((1ull << bits) < (unsigned long long)KK * KK) bits++;
            size_t tb = w.qsort_bytes;
            CRISP_CUDA(cub::DeviceRadixSort::SortPairs(w.qsort_tmp, tb, w.qkey, w.qkey2, w.qiota, w.qperm, (int)qn, 0,
                                                       bits, s));
        }
    }
    {
        StageScope st(s, 2);
        CRISP_CUDA(cudaMemsetAsync(w.cursor, 0, (size_t)(w.Qc + 1) * 4, s));
        if (w.mode == 1) CRISP_CUDA(cudaMemsetAsync(w.ghist, 0, (size_t)qn * (ix->Dp + 1) * 4, s));
        dim3 g(nblk(NB, w.BPC), (unsigned)qn);
        if (w.count_kernel == 2)
        {
            k_act_rows<<<nblk(qn, 8), 256, 0, s>>>(w.act, w.act_len, M, KK, qn, w.erow, w.etot);
            CRISP_LAUNCH();
            g_launches++;
            // 64K ids per CTA: 16 warps, two CTAs per SM; 128K ids: 32 warps, one CTA per SM
            uint16_t *hb = (w.mode == 1 && w.ham_fused) ? w.hbuf : nullptr;  // phi=1: Hamming fused into the count
            if (w.CF * ix->BS <= 32768 && env_int("CRISP_COUNT_W8", 0))
                k_count_frag<8><<<dim3((unsigned)w.NS, (unsigned)qn), 256, countf_smem(ix->BS * w.CF), s>>>(
                    w.erow, w.etot, M, KK, ix->off2, NB, w.CF, ix->ids, ix->N, ix->BS, w.NS, ix->tau, w.pool, w.CAPQ,
                    w.cursor, w.cbase, w.ncand, w.need, w.traceV, w.qperm, w.qrot, pitch, ix->Dp, ix->codes, ix->Wp,
                    hb, w.ghist);
            else {
                // reductions without return + a final threshold scan over the counters (measured at
                // cfg4/3/5 phi=1: count 16.9 / 81.2 / 29.5 ms against 17.1 / 86.1 / 32.4 ms with the
                // atomics' returns and crossing bits); CRISP_COUNT_SWAR=0 keeps the crossing bits
                const bool sw = env_int("CRISP_COUNT_SWAR", 1) != 0;
#define CRISP_CF(WN, SW)                                                                                          \
    k_count_frag<WN, SW><<<dim3((unsigned)w.NS, (unsigned)qn), WN * 32, countf_smem(ix->BS * w.CF), s>>>(           \
        w.erow, w.etot, M, KK, ix->off2, NB, w.CF, ix->ids, ix->N, ix->BS, w.NS, ix->tau, w.pool, w.CAPQ, w.cursor, \
        w.cbase, w.ncand, w.need, w.traceV, w.qperm, w.qrot, pitch, ix->Dp, ix->codes, ix->Wp, hb, w.ghist)
                if (w.CF * ix->BS > 65536) {
                    if (sw) CRISP_CF(32, true);
                    else CRISP_CF(32, false);
                } else if (sw) CRISP_CF(16, true);
                else CRISP_CF(16, false);
#undef CRISP_CF
            }
        }
        else if (w.count_kernel == 0)
            k_count_select<<<g, THREADS, w.count_smem, s>>>(w.act, w.act_len, M, KK, ix->off2, NB, ix->ids, ix->N,
                                                            ix->BS, w.BPC, ix->tau, w.pool, w.CAPQ, w.cursor, w.cbase,
                                                            w.ncand, w.need, w.traceV, w.qperm);
        else {
            uint16_t *hb = (w.mode == 1 && w.ham_fused) ? w.hbuf : nullptr;  // phi=1: Hamming fused into the count
            const int smem = w.countw_smem + (hb ? w.countw_ham_smem : 0);
#define CRISP_COUNT_WARP(HM, AT)                                                                               \
    k_count_warp<HM, AT><<<g, THREADS, smem, s>>>(w.act, w.act_len, M, KK, ix->off2w, ix->NBW, ix->ids, ix->N, ix->BS, \
                                                  w.BPC, NB, ix->tau, w.pool, w.CAPQ, w.cursor, w.cbase, w.ncand,      \
                                                  w.need, w.traceV, w.qrot, pitch, ix->Dp, ix->codes, ix->Wp, hb,      \
                                                  w.ghist, w.qperm)
            if (hb && w.count_atom) CRISP_COUNT_WARP(true, true);
            else if (hb) CRISP_COUNT_WARP(true, false);
            else if (w.count_atom) CRISP_COUNT_WARP(false, true);
            else CRISP_COUNT_WARP(false, false);
#undef CRISP_COUNT_WARP
        }
        CRISP_LAUNCH();
        g_launches++;
    }
}

static int32_t read_need(Work &w, cudaStream_t s) {
    int32_t h = 0;
    CRISP_CUDA(cudaMemcpyAsync(&h, w.need, 4, cudaMemcpyDeviceToHost, s));
    CRISP_CUDA(cudaStreamSynchronize(s));
    return h;
}

static void run_fallback_local(Work &w, int64_t qn, cudaStream_t s) {
    const crisp_index *ix = w.ix;
    StageScope st(s, 3);
    k_fallback<<<(unsigned)qn, THREADS, w.count_smem, s>>>(w.act, w.act_len, ix->M, ix->K * ix->K, ix->off2, ix->NB,
                                                           ix->ids, ix->N, ix->BS, w.k, w.pool, w.CAPQ, w.cbase,
                                                           w.ncand, w.NS, w.fb, w.ghist, ix->Dp + 1);
    CRISP_LAUNCH();
    g_launches++;
}

// a4 at phi=1: the Hamming distances of every candidate and the (h, id) order
// (cbuf, up to order_end, or all of it with full_order); resets the patience state
static void run_order(Work &w, int64_t qn, cudaStream_t s) {
    const crisp_index *ix = w.ix;
    const int NB = w.NS, pitch = ix->pitch, Dp = ix->Dp;
    CRISP_CUDA(cudaMemsetAsync(w.pst.cnt, 0, (size_t)w.Qc * 5 * 4, s));
    {
        // h of the queries whose candidate set the fallback replaced (k_hamming),
        // then of all others over their dense pool positions (k_hamming_dense),
        // unless k_count_warp computed it with the count
        StageScope st(s, 6);
        dim3 g(w.HS, (unsigned)qn);
        k_hamming<<<g, THREADS, w.ham_smem, s>>>(w.qrot, pitch, Dp, ix->codes, ix->Wp, w.pool, w.CAPQ, w.cbase, w.ncand,
                                                 NB, w.hbuf, w.ghist, w.fb, w.qperm);
        CRISP_LAUNCH();
        g_launches++;
        if (w.count_kernel == 2 && !w.ham_fused && env_int("CRISP_HAMMING_SEG", 1) &&
            (size_t)WARPS * ix->Wp * 8 <= 48 * 1024) {
            // segment-major over the 64K-id segments of k_count_frag (the code rows of one id
            // block stay in L2; measured at cfg4: 8.6 against 11.3 ms), then the histograms.
            // (The 4096-id segments of k_count_warp, cfg2, hold too few candidates per warp:
            // 3.6 against 1.9 ms, so that path keeps the per-query kernel.)
            k_qcodes<<<nblk(qn, 8), 256, 0, s>>>(w.qrot, pitch, Dp, ix->Wp, qn, w.qcodes);
            CRISP_LAUNCH();
            dim3 g2(nblk(qn, WARPS), (unsigned)NB);
            if (env_int("CRISP_HAMMING_SEG_HT", 2) >= 4)
                k_hamming_seg<4><<<g2, THREADS, WARPS * ix->Wp * 8, s>>>(w.qcodes, ix->codes, ix->Wp, w.pool, w.CAPQ,
                                                                         w.cbase, w.ncand, NB, qn, w.hbuf, w.fb,
                                                                         w.qperm);
            else
                k_hamming_seg<2><<<g2, THREADS, WARPS * ix->Wp * 8, s>>>(w.qcodes, ix->codes, ix->Wp, w.pool, w.CAPQ,
                                                                         w.cbase, w.ncand, NB, qn, w.hbuf, w.fb,
                                                                         w.qperm);
            CRISP_LAUNCH();
            g_launches++;
            k_hhist<<<(unsigned)qn, THREADS, (Dp + 1) * 4, s>>>(Dp, w.cursor, w.CAPQ, w.hbuf, w.ghist, w.fb);
            CRISP_LAUNCH();
            g_launches += 2;
        } else if (!((w.count_kernel == 1 || w.count_kernel == 2) && w.ham_fused)) {
            dim3 g2(w.HS, (unsigned)qn);
            // 16-byte chunks of each code row issued together per lane (CRISP_HAMMING_HT: 2, or 4 with
            // 2 CTAs per SM; measured at cfg4: 12.4 ms with 2 (8 loads in flight), 14.7 with 4, 14.0 before)
            if (env_int("CRISP_HAMMING_HT", 2) >= 4)
                k_hamming_dense<4><<<g2, THREADS, w.countw_ham_smem, s>>>(w.qrot, pitch, Dp, ix->codes, ix->Wp, w.pool,
                                                                          w.CAPQ, w.cursor, w.hbuf, w.ghist, w.fb,
                                                                          w.qperm);
            else
                k_hamming_dense<2><<<g2, THREADS, w.countw_ham_smem, s>>>(w.qrot, pitch, Dp, ix->codes, ix->Wp, w.pool,
                                                                          w.CAPQ, w.cursor, w.hbuf, w.ghist, w.fb,
                                                                          w.qperm);
            CRISP_LAUNCH();
            g_launches++;
        }
    }
    {
        // (h, id) order into cbuf
        StageScope st(s, 7);
        if (w.hsort_cta_smem <= 200 * 1024)
        {
            // LIST: phase B visits only the listed qualifying elements (when the
            // sorted prefix is short: k = 10 configurations)
            const int lim = w.full_order ? 0x7fffffff : w.order_end();
            // (measured at cfg4, k = 100, cut 7072: LIST 1.67 against 1.83 ms; the listing falls
            // back to the scan by itself when the order row's tail cannot hold the list)
            if (lim <= env_int("CRISP_HSORT_LIST_MAX", 16384))
                k_hsort_cta<true><<<(unsigned)qn, THREADS, w.hsort_cta_smem, s>>>(
                    w.ncand, w.cbase, NB, Dp, w.ghist, w.pool, w.hbuf, w.CAPQ, w.cbuf, w.totals, lim);
            else
                k_hsort_cta<false><<<(unsigned)qn, THREADS, w.hsort_cta_smem, s>>>(
                    w.ncand, w.cbase, NB, Dp, w.ghist, w.pool, w.hbuf, w.CAPQ, w.cbuf, w.totals, lim);
        }
        else
            k_hsort<<<(unsigned)qn, 32, w.hsort_smem, s>>>(w.ncand, w.cbase, NB, Dp, w.ghist, w.pool, w.hbuf, w.CAPQ,
                                                           w.cbuf, w.totals, w.full_order ? 0x7fffffff : w.order_end());
        CRISP_LAUNCH();
        g_launches++;
    }
}

// a4 (phi=1 Hamming order) + a5 for queries [0, qn) of the chunk -> outputs
static void run_verify(Work &w, int64_t qn, int64_t *oi, float *od, double *od64, cudaStream_t s) {
    const crisp_index *ix = w.ix;
    const int NB = w.NS, pitch = ix->pitch, Dp = ix->Dp, k = w.k;  // NB: candidate segments
    if (!od64) od64 = w.d64tmp;
    if (w.mode == 0 && w.rgroup) {
        {
            StageScope st(s, 4);
            dim3 g((unsigned)w.NR, nblk(qn, w.GR));
#define CRISP_RG(GRV)                                                                                                   k_rerank_group<GRV><<<g, THREADS, w.rg_smem, s>>>(w.qrot, pitch, ix->X, ix->gid_base, ix->N, w.pool, w.CAPQ,                                                       w.cbase, w.ncand, NB, w.segw, w.fb, w.RW, k, qn, w.part_d,                                                         w.part_i, w.qperm)
            if (w.GR == 8) CRISP_RG(8);
            else if (w.GR == 4) CRISP_RG(4);
            else CRISP_RG(2);
#undef CRISP_RG
            CRISP_LAUNCH();
            g_launches++;
        }
        {
            StageScope st(s, 5);
            k_merge_lists<<<(unsigned)qn, THREADS, 0, s>>>(w.part_d, w.part_i, w.NR, qn, k, 0, od64, od, oi);
            CRISP_LAUNCH();
            g_launches++;
        }
        return;
    }
    if (w.mode == 0) {
        {
            StageScope st(s, 4);
            dim3 g(w.S, (unsigned)qn);
            unsigned long long *fst = g_counters ? d_filter_stats_ptr() : nullptr;
            if (w.lb0) {
                w.q8_prep(qn, s);
                // 4 CTAs/SM (64 registers): 186.7 against 198.2 ms with 3 at cfg4
                if (env_int("CRISP_LBB_CTAS", 4) == 4)
                    k_lb_bounds<4><<<g, THREADS, w.lbb_smem, s>>>(w.qrot, pitch, w.fa, w.pool, w.CAPQ, w.cbase, w.ncand,
                                                                  NB, w.lbb, w.qperm, fst);
                else
                    k_lb_bounds<3><<<g, THREADS, w.lbb_smem, s>>>(w.qrot, pitch, w.fa, w.pool, w.CAPQ, w.cbase, w.ncand,
                                                                  NB, w.lbb, w.qperm, fst);
                CRISP_LAUNCH();
                k_lb_threshold<<<(unsigned)qn, THREADS, w.lbt_smem, s>>>(w.cbase, w.ncand, NB, w.CAPQ, w.lbb, k, w.Tq);
                CRISP_LAUNCH();
                k_rerank_exact<false, true><<<g, THREADS, w.rx_smem, s>>>(w.qrot, pitch, ix->X, ix->gid_base, w.pool,
                                                                          w.CAPQ, w.cbase, w.ncand, NB, k, w.part_d,
                                                                          w.part_i, w.qperm, w.lbb, w.Tq, fst);
                g_launches += 2;
            } else if (w.rows4)
                k_rerank_exact<true, false><<<g, THREADS, w.rx_smem, s>>>(w.qrot, pitch, ix->X, ix->gid_base, w.pool,
                                                                          w.CAPQ, w.cbase, w.ncand, NB, k, w.part_d,
                                                                          w.part_i, w.qperm, nullptr, nullptr, nullptr);
            else
                k_rerank_exact<false, false><<<g, THREADS, w.rx_smem, s>>>(w.qrot, pitch, ix->X, ix->gid_base, w.pool,
                                                                           w.CAPQ, w.cbase, w.ncand, NB, k, w.part_d,
                                                                           w.part_i, w.qperm, nullptr, nullptr,
                                                                           nullptr);
            CRISP_LAUNCH();
            g_launches++;
        }
        {
            StageScope st(s, 5);
            k_merge_lists<<<(unsigned)qn, THREADS, 0, s>>>(w.part_d, w.part_i, w.S, qn, k, 0, od64, od, oi);
            CRISP_LAUNCH();
            g_launches++;
        }
        return;
    }
    const int P = ix->patience_factor > 0 ? ix->patience_factor * k : 0;
    run_order(w, qn, s);
    StageScope st(s, 4);
    // verification rounds.  Round 0: positions [0, F) of every query.  Exact
    // verification, rounds >= 1: each running query its own span [pos, pos + nlen)
    // (the rows it certainly verifies next, set by the scan).  ADSampling: fixed
    // spans [F + (r-1) S0, F + r S0), pruned under the r_k of the round's start.
    AdCtx ad{w.ad, ix->ad_eps0, ix->ad_stride, Dp, ix->X, pitch, ix->gid_base, nullptr};
    const int send = w.full_order ? 0x7fffffff : w.order_end();
    if (w.lbf) w.q8_prep(qn, s);
    for (int r = 0; r < w.R0; r++) {
        const bool own = r > 0 && (!w.ad || w.adsp);
        const int j0 = own ? -1 : (r == 0 ? 0 : w.F + (r - 1) * w.S0), len = r == 0 ? w.F : w.S0;
        // CTAs per query: at most S, at least round_rows rows each (the query staging is per CTA)
        dim3 g(own ? w.S1 : std::max(1, std::min(w.S, len / w.round_rows)), (unsigned)qn);
        if (w.lbf && r > 0 && w.lbblk) {
            k_span_bucket<<<(unsigned)qn, 256, w.bkt_smem, s>>>(w.cbuf, w.CAPQ, w.totals, w.pst, send, w.BSH, w.NBB,
                                                                  w.DS, w.spair, w.boff);
            CRISP_LAUNCH();
            g_launches++;
            if (env_int("CRISP_LB_QPC", 64) >= 64)
                k_verify_lb_blk<64><<<dim3(nblk(qn, 64), (unsigned)w.NBB), THREADS, WARPS * 64 * 4, s>>>(
                    w.qrot, pitch, ix->X, w.fa, w.pst, k, qn, w.NBB, w.DS, w.spair, w.boff, w.dbuf,
                    g_counters ? d_filter_stats_ptr() : nullptr);
            else
                k_verify_lb_blk<WARPS><<<dim3(nblk(qn, WARPS), (unsigned)w.NBB), THREADS, WARPS * 64 * 4, s>>>(
                    w.qrot, pitch, ix->X, w.fa, w.pst, k, qn, w.NBB, w.DS, w.spair, w.boff, w.dbuf,
                    g_counters ? d_filter_stats_ptr() : nullptr);
        } else if (w.lbf && r > 0 && env_int("CRISP_LB_CTAS", 3) == 4)
            k_verify_rows_lb<4><<<g, THREADS, w.vrl_smem, s>>>(w.qrot, pitch, ix->X, w.fa, w.cbuf, w.CAPQ, w.totals,
                                                               w.pst, k, j0, len, send, w.DS, w.dbuf, w.qperm,
                                                               g_counters ? d_filter_stats_ptr() : nullptr);
        else if (w.lbf && r > 0)
            k_verify_rows_lb<3><<<g, THREADS, w.vrl_smem, s>>>(w.qrot, pitch, ix->X, w.fa, w.cbuf, w.CAPQ, w.totals,
                                                               w.pst, k, j0, len, send, w.DS, w.dbuf, w.qperm,
                                                               g_counters ? d_filter_stats_ptr() : nullptr);
        else if (w.ad && r > 0)  // round 0 starts with an empty top-k: nothing to prune
            k_verify_rows_ad<<<g, THREADS, w.vra_smem, s>>>(w.qrot, pitch, Dp, ix->X, w.cbuf, w.CAPQ, w.totals, w.pst,
                                                            k, j0, len, send, w.DS, w.dbuf, w.qperm, ix->ad_eps0,
                                                            ix->ad_stride);
        else if (w.rows4)
            k_verify_rows<true><<<g, THREADS, w.vr_smem, s>>>(w.qrot, pitch, ix->X, w.cbuf, w.CAPQ, w.totals, w.pst,
                                                              j0, len, send, w.DS, w.dbuf, w.qperm);
        else
            k_verify_rows<false><<<g, THREADS, w.vr_smem, s>>>(w.qrot, pitch, ix->X, w.cbuf, w.CAPQ, w.totals,
                                                               w.pst, j0, len, send, w.DS, w.dbuf, w.qperm);
        CRISP_LAUNCH();
        g_launches++;
        k_patience_scan<<<nblk(qn, WARPS), THREADS, w.scan_smem, s>>>(qn, w.totals, w.cbuf, w.CAPQ, ix->gid_base,
                                                                      w.dbuf, j0, len, send, w.nl_min, w.nl_max, w.DS, k,
                                                                      P, w.pst, od64, od, oi, ad, w.qrot);
        CRISP_LAUNCH();
        g_launches++;
    }
    k_patience_tail<<<(unsigned)qn, THREADS, w.pat_smem, s>>>(w.qrot, pitch, ix->X, ix->gid_base, w.cbuf, w.CAPQ,
                                                              w.totals, send, w.rows4, k, P, w.pst, od64, od, oi, Dp,
                                                              w.ghist, w.pool, w.hbuf, w.ncand, w.cbase, NB, w.qperm,
                                                              ad);
    CRISP_LAUNCH();
    g_launches++;
}

static void run_stats(Work &w, int64_t qn, cudaStream_t s) {
    if (!g_counters) return;
    const crisp_index *ix = w.ix;
    k_stats<<<(unsigned)qn, 128, 0, s>>>(w.act, w.act_len, ix->M, ix->K * ix->K, ix->off2, ix->NB, w.ncand, w.NS,
                                         w.mode == 1 ? w.nver : nullptr, w.fb, qn);
    CRISP_LAUNCH();
    // a diagnostics kernel (work counters): not counted among the search's launches
}

static void trace_candidates(Work &w, int64_t q0, int64_t qn, const crisp_trace_t *tr, cudaStream_t s) {
    const int NB = w.NS;  // candidate segments
    const int64_t N = w.ix->N, CAPQ = w.CAPQ;
    std::vector<int32_t> h_pool((size_t)qn * CAPQ), h_ncand((size_t)qn * NB), h_cbase((size_t)qn * NB);
    CRISP_CUDA(cudaMemcpyAsync(h_pool.data(), w.pool, (size_t)qn * CAPQ * 4, cudaMemcpyDeviceToHost, s));
    CRISP_CUDA(cudaMemcpyAsync(h_ncand.data(), w.ncand, (size_t)qn * NB * 4, cudaMemcpyDeviceToHost, s));
    CRISP_CUDA(cudaMemcpyAsync(h_cbase.data(), w.cbase, (size_t)qn * NB * 4, cudaMemcpyDeviceToHost, s));
    CRISP_CUDA(cudaStreamSynchronize(s));
    for (int64_t q = 0; q < qn; q++) {
        int64_t n = 0;
        for (int b = 0; b < NB; b++) {
            const int c = h_ncand[q * NB + b], base = h_cbase[q * NB + b];
            for (int j = 0; j < c; j++) {
                const int32_t id = h_pool[q * CAPQ + base + j];
                if (tr->cand) tr->cand[(q0 + q) * N + n] = id;
                if (tr->order && w.mode == 0) tr->order[(q0 + q) * N + n] = id;
                n++;
            }
        }
        if (tr->cand_n) tr->cand_n[q0 + q] = n;
        if (tr->n_verified && w.mode == 0) tr->n_verified[q0 + q] = n;
    }
}

static void trace_rest(Work &w, int64_t q0, int64_t qn, const crisp_trace_t *tr, cudaStream_t s) {
    const crisp_index *ix = w.ix;
    const int M = ix->M, KK = ix->K * ix->K, NB = w.NS, Dp = ix->Dp, pitch = ix->pitch;  // NB: segments
    const int64_t N = ix->N, CAPQ = w.CAPQ;
    std::vector<int32_t> hl((size_t)qn * M), h_pool, h_ncand;
    std::vector<uint32_t> ha;
    std::vector<int64_t> hr((size_t)qn * M), hn;
    CRISP_CUDA(cudaMemcpyAsync(hl.data(), w.act_len, (size_t)qn * M * 4, cudaMemcpyDeviceToHost, s));
    CRISP_CUDA(cudaMemcpyAsync(hr.data(), w.retr, (size_t)qn * M * 8, cudaMemcpyDeviceToHost, s));
    if (tr->act_cell || tr->act_w) {
        ha.resize((size_t)qn * M * KK);
        CRISP_CUDA(cudaMemcpyAsync(ha.data(), w.act, (size_t)qn * M * KK * 4, cudaMemcpyDeviceToHost, s));
    }
    if (tr->V && w.traceV)
        CRISP_CUDA(cudaMemcpyAsync(tr->V + q0 * N, w.traceV, (size_t)qn * N, cudaMemcpyDeviceToHost, s));
    if (tr->qrot)
        for (int64_t q = 0; q < qn; q++)
            CRISP_CUDA(cudaMemcpyAsync(tr->qrot + (q0 + q) * Dp, w.qrot + q * pitch, (size_t)Dp * 4,
                                       cudaMemcpyDeviceToHost, s));
    if (tr->fallback) CRISP_CUDA(cudaMemcpyAsync(tr->fallback + q0, w.fb, (size_t)qn * 4, cudaMemcpyDeviceToHost, s));
    if (w.mode == 1) {
        hn.resize(qn);
        h_pool.resize((size_t)qn * CAPQ);
        h_ncand.resize((size_t)qn * NB);
        CRISP_CUDA(cudaMemcpyAsync(hn.data(), w.nver, (size_t)qn * 8, cudaMemcpyDeviceToHost, s));
        CRISP_CUDA(cudaMemcpyAsync(h_pool.data(), w.cbuf, (size_t)qn * CAPQ * 4, cudaMemcpyDeviceToHost, s));
        CRISP_CUDA(cudaMemcpyAsync(h_ncand.data(), w.ncand, (size_t)qn * NB * 4, cudaMemcpyDeviceToHost, s));
    }
    CRISP_CUDA(cudaStreamSynchronize(s));
    for (int64_t q = 0; q < qn; q++) {
        for (int m = 0; m < M; m++) {
            const int L = hl[q * M + m];
            if (tr->act_len) tr->act_len[(q0 + q) * M + m] = L;
            if (tr->retrieved) tr->retrieved[(q0 + q) * M + m] = hr[q * M + m];
            for (int r = 0; r < L && !ha.empty(); r++) {
                const uint32_t v = ha[(q * M + m) * (int64_t)KK + r];
                if (tr->act_cell) tr->act_cell[((q0 + q) * M + m) * (int64_t)KK + r] = (int32_t)(v & 0xffffu);
                if (tr->act_w) tr->act_w[((q0 + q) * M + m) * (int64_t)KK + r] = (int32_t)(v >> 16);
            }
        }
        if (w.mode == 1) {
            int64_t n = 0;
            for (int b = 0; b < NB; b++) n += h_ncand[q * NB + b];
            if (tr->order)
                for (int64_t i = 0; i < n; i++) tr->order[(q0 + q) * N + i] = h_pool[q * CAPQ + i];
            if (tr->n_verified) tr->n_verified[q0 + q] = hn[q];
        }
    }
}

// default per-search scratch cap: half of the device memory free at the call,
// at least 4 GiB and at most 64 GiB (a 10k-query cfg4 batch needs ~17 GB and
// must not be split into a full and a nearly empty chunk)
static int64_t default_workspace() {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
        cudaGetLastError();
        return 16LL << 30;
    }
    return std::max<int64_t>(4LL << 30, std::min<int64_t>(64LL << 30, (int64_t)(fr / 2)));
}

// Candidate capacity per query: an exact upper bound of |C_q| known before the
// search, so that crisp_search_async never reads anything back (no host sync).
// Every x in C has V[x] >= tau (Alg. 1 l.18), and sum_x V[x] = sum over the
// activated cells of w * |cell| <= wmax * sum_m R_qm with w <= 2 at phi=1 and
// w = 1 at phi=0 (Alg. 1 l.10-12); the budget walk stops at the first cell that
// brings R_qm to >= B (Z3), so R_qm <= B - 1 + max_c |cell_{m,c}|.  The fallback
// (|C| < k) writes at most k.  Trace calls keep room for every id.
static int64_t candidate_capacity(const crisp_index *ix, int mode, int k, bool trace) {
    const int64_t all = (int64_t)ix->NB * ix->BS;
    if (trace) return all;
    const int64_t wmax = mode == 1 ? 2 : 1;
    const int64_t R = (int64_t)ix->M * std::max<int64_t>(0, ix->budget - 1) + ix->maxcell_sum;
    int64_t b = wmax * R / std::max(1, ix->tau);
    b = std::min<int64_t>(b, ix->N);
    b = std::max<int64_t>(b, std::min<int64_t>(k, ix->N));
    if (const char *v = getenv("CRISP_CAND_CAP")) b = std::max<int64_t>(b, atoll(v));  // test hook (only grows)
    return std::max<int64_t>(16, std::min(b, all));
}

// The whole batch, in query chunks that fit the workspace, with candidate
// capacity CAPQ per query (candidate_capacity: never exceeded).  Only the trace
// path reads back (its outputs); otherwise everything is stream-ordered on s.
// CRISP_PIPE = p >= 2: the batch in p query chunks on two side streams, so that one
// chunk's front (a0-a4: the issue-bound collision count) runs while the previous
// chunk's verification streams HBM.  Stream-ordered: forked from and joined into s.
static void search_pipelined(const crisp_index *ix, const float *queries, int64_t Q, int32_t k, int mode,
                             SearchOut out, cudaStream_t s, int64_t CAPQ, int parts) {
    const int64_t Qc = (Q + parts - 1) / parts;
    cudaStream_t ss[2];
    cudaEvent_t fork, done[2];
    for (int i = 0; i < 2; i++) {
        CRISP_CUDA(cudaStreamCreateWithFlags(&ss[i], cudaStreamNonBlocking));
        CRISP_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
    CRISP_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    {
        Work w0(ix, k, mode, Qc, CAPQ, false, out.d64 == nullptr, s), w1(ix, k, mode, Qc, CAPQ, false, out.d64 == nullptr, s);
        Work *ws[2] = {&w0, &w1};
        CRISP_CUDA(cudaEventRecord(fork, s));  // the Work buffers were allocated on s
        for (int i = 0; i < 2; i++) CRISP_CUDA(cudaStreamWaitEvent(ss[i], fork, 0));
        int c = 0;
        for (int64_t q0 = 0; q0 < Q; q0 += Qc, c++) {
            const int64_t qn = std::min(Qc, Q - q0);
            Work &w = *ws[c & 1];
            cudaStream_t st = ss[c & 1];
            run_front(w, queries + q0 * ix->D, qn, st, nullptr);
            run_fallback_local(w, qn, st);
            run_verify(w, qn, out.ids + q0 * k, out.d32 ? out.d32 + q0 * k : nullptr,
                       out.d64 ? out.d64 + q0 * k : nullptr, st);
            run_stats(w, qn, st);
        }
        for (int i = 0; i < 2; i++) {
            CRISP_CUDA(cudaEventRecord(done[i], ss[i]));
            CRISP_CUDA(cudaStreamWaitEvent(s, done[i], 0));  // joined before the buffers are freed on s
        }
    }
    for (int i = 0; i < 2; i++) {
        cudaEventDestroy(done[i]);
        cudaStreamDestroy(ss[i]);
    }
    cudaEventDestroy(fork);
}

static void search_pass(const crisp_index *ix, const float *queries, int64_t Q, int32_t k, int mode, SearchOut out,
                        cudaStream_t s, const crisp_trace_t *tr, int64_t CAPQ, const float *hq) {
    const int64_t ws = ix->workspace_bytes > 0 ? ix->workspace_bytes : default_workspace();
    const int64_t perq = Work::per_query_bytes(ix, k, mode, CAPQ, tr && tr->V);
    const int parts = std::max(1, std::min(16, env_int("CRISP_PIPE", 1)));
    if (parts >= 2 && !tr && !hq && Q >= 2048 && perq * 2 * ((Q + parts - 1) / parts) <= ws) {
        search_pipelined(ix, queries, Q, k, mode, out, s, CAPQ, parts);
        return;
    }
    int64_t Qc = std::max<int64_t>(1, std::min<int64_t>(Q, ws / perq));
    Qc = std::min<int64_t>(Qc, 65535);
    Work w(ix, k, mode, Qc, CAPQ, tr && tr->V, out.d64 == nullptr, s);
    w.full_order = tr != nullptr;
    for (int64_t q0 = 0; q0 < Q; q0 += Qc) {
        const int64_t qn = std::min(Qc, Q - q0);
        run_front(w, queries + q0 * ix->D, qn, s, hq ? hq + q0 * ix->D : nullptr);
        run_fallback_local(w, qn, s);
        if (tr) {
            CRISP_CHECK(read_need(w, s) <= CAPQ, "internal: candidate capacity exceeded");
            trace_candidates(w, q0, qn, tr, s);
        }
        run_verify(w, qn, out.ids + q0 * k, out.d32 ? out.d32 + q0 * k : nullptr, out.d64 ? out.d64 + q0 * k : nullptr,
                   s);
        run_stats(w, qn, s);
        if (tr) trace_rest(w, q0, qn, tr, s);
    }
}

void search(const crisp_index *ix, const float *queries, int64_t Q, int32_t k, int mode, SearchOut out,
            cudaStream_t s, const crisp_trace_t *tr, const float *queries_host) {
    search_pass(ix, queries, Q, k, mode, out, s, tr, candidate_capacity(ix, mode, k, tr != nullptr), queries_host);
}

// ---------------------------------------------------------------------------
// Shard session: the search split at the two exchange points of the exact
// global fallback.  The whole batch is one chunk.
// ---------------------------------------------------------------------------
}  // namespace crisp

namespace crisp {
struct GPBuf;
}
struct crisp_session {
    const crisp_index *ix;
    crisp::Work *w;
    int64_t Q;
    int k, mode;
    crisp::GPBuf *gp = nullptr;  // exact global patience (phi=1 over G shards)
};

namespace crisp {

// a0 alone for Q queries into qrot (Q x pitch): the zero-padded copy, then the certified
// int8 tensor-core transform when the index is rotated (as run_front)
void transform_queries(const crisp_index *ix, const float *queries, int64_t Q, float *qrot, cudaStream_t s) {
    if (Q <= 0) return;
    const int pitch = ix->pitch;
    float *qpad = qrot;
    if (ix->rotated) CRISP_CUDA(cudaMallocAsync(&qpad, (size_t)Q * pitch * 4, s));
    k_prep_queries<<<nblk(Q * pitch, 256), 256, 0, s>>>(queries, Q, ix->D, pitch, qpad);
    CRISP_LAUNCH();
    g_launches++;
    if (ix->rotated) {
        rotate_rows(const_cast<crisp_index *>(ix), qpad, Q, pitch, qrot, pitch, s);
        g_launches += 3;
        CRISP_CUDA(cudaFreeAsync(qpad, s));
    }
}

crisp_session *session_begin(const crisp_index *ix, const float *queries, int64_t Q, int32_t k, int mode,
                             int32_t *local_counts, cudaStream_t s, bool transformed) {
    CRISP_CHECK(Q <= 65535, "a shard session takes at most 65535 queries (split the batch)");
    const int64_t cap = candidate_capacity(ix, mode, k, false);
    const int64_t ws = ix->workspace_bytes > 0 ? ix->workspace_bytes : default_workspace();
    CRISP_CHECK(Work::per_query_bytes(ix, k, mode, cap, false) * Q <= ws,
                "shard session scratch exceeds the workspace (split the batch)");
    Work *w = new Work(ix, k, mode, std::max<int64_t>(Q, 1), cap, false, false, s);
    try {
        run_front(*w, queries, Q, s, nullptr, transformed);
        k_local_counts<<<nblk(Q, 256), 256, 0, s>>>(w->ncand, w->NS, Q, local_counts);
        CRISP_LAUNCH();
        g_launches++;
        return new crisp_session{ix, w, Q, k, mode};
    } catch (...) {
        delete w;
        throw;
    }
}

void session_hist(crisp_session *ss, const int32_t *gcount, int32_t *lhist, cudaStream_t s) {
    Work &w = *ss->w;
    const crisp_index *ix = ss->ix;
    StageScope st(s, 3);
    k_fb_hist<<<(unsigned)ss->Q, THREADS, w.count_smem, s>>>(w.act, w.act_len, ix->M, ix->K * ix->K, ix->off2, ix->NB,
                                                             ix->ids, ix->N, ix->BS, ss->k, gcount, lhist);
    CRISP_LAUNCH();
    g_launches++;
}

void session_finish(crisp_session *ss, const int32_t *gcount, const int32_t *allhist, int32_t G, int32_t rank,
                    int64_t *out_ids, double *out_d64, cudaStream_t s) {
    Work &w = *ss->w;
    const crisp_index *ix = ss->ix;
    {
        StageScope st(s, 3);
        k_fb_select<<<(unsigned)ss->Q, THREADS, w.count_smem, s>>>(
            w.act, w.act_len, ix->M, ix->K * ix->K, ix->off2, ix->NB, ix->ids, ix->N, ix->BS, ss->k, gcount, allhist,
            G, rank, ss->Q, w.pool, w.CAPQ, w.cbase, w.ncand, w.NS, w.fb, w.ghist, ix->Dp + 1);
        CRISP_LAUNCH();
        g_launches++;
    }
    run_verify(w, ss->Q, out_ids, nullptr, out_d64, s);
    run_stats(w, ss->Q, s);
}

// ---------------------------------------------------------------------------
// Exact global patience over G point shards (phi=1).  The global
// verification order is (h, gid) over the union of the shards' candidate sets
// (P:L455-458 applied to the whole dataset).  Every rank keeps the same global
// state per query (top-k, patience counter, position, window length); a round
// takes the global window [pos, pos + len), each rank verifies its own rows in
// it (their local positions follow from the all-gathered Hamming histograms),
// emits the rows that may improve the top-k as it stood at the round's start
// (the k-th best only shrinks, so every other row is a certain miss), and after
// an all-gather every rank replays the window in global order with the
// sequential rule.  The result and the stop index equal those of a single
// index over all rows, for every G.
// ---------------------------------------------------------------------------
struct GEnt {
    int32_t gpos;  // position in the global (h, gid) order
    int32_t lid;   // local id on the emitting shard
    double d;      // exact distance
};
static_assert(sizeof(GEnt) == 16, "GEnt is the 16-byte record of include/crisp.h");

struct GPBuf {
    int G = 1, rank = 0, H = 0;
    int32_t *base = nullptr, *lcum = nullptr;  // Q x (H + 1)
    int32_t *gtot = nullptr, *gpos = nullptr, *glen = nullptr;
    int32_t *cnt = nullptr, *offs = nullptr;  // Q + 1
    GEnt *stage = nullptr, *packed = nullptr;  // Q x DS
    int32_t *running = nullptr;
    int32_t *all_off = nullptr;  // G x (Q + 1)
    int64_t *gbase = nullptr;    // G
    void *scan_tmp = nullptr;
    size_t scan_bytes = 0;
    int nl_min = 512, nl_max = 4096;
    int64_t n_packed = 0;
    std::vector<void *> ptrs;
    template <class T>
    T *alloc(size_t n, cudaStream_t s) {
        void *p = nullptr;
        CRISP_CUDA(cudaMallocAsync(&p, std::max<size_t>(n * sizeof(T), 16), s));
        ptrs.push_back(p);
        return (T *)p;
    }
    ~GPBuf() {
        for (void *p : ptrs) cudaFree(p);
    }
};

__global__ void __launch_bounds__(256) k_gp_tables(const int32_t *__restrict__ allh, int G, int rank, int64_t Q, int H,
                                                   int32_t *__restrict__ base, int32_t *__restrict__ lcum,
                                                   int32_t *__restrict__ gtot) {
    // base[h] = global position of this rank's first candidate with Hamming distance h
    //         = (all candidates with h' < h) + (candidates of ranks < rank with h);
    // lcum[h] = local position of that candidate; [H] are the totals
    typedef cub::BlockScan<int, 256> BScan;
    __shared__ typename BScan::TempStorage ts;
    __shared__ int carry_all, carry_me;
    const int64_t q = blockIdx.x;
    if (threadIdx.x == 0) carry_all = carry_me = 0;
    __syncthreads();
    for (int h0 = 0; h0 < H; h0 += 256) {
        const int h = h0 + threadIdx.x;
        int tot = 0, pre = 0, mine = 0;
        if (h < H)
            for (int g = 0; g < G; g++) {
                const int v = allh[((int64_t)g * Q + q) * H + h];
                tot += v;
                pre += g < rank ? v : 0;
                mine += g == rank ? v : 0;
            }
        int ea, em, sa, sme;
        BScan(ts).ExclusiveSum(tot, ea, sa);
        __syncthreads();
        BScan(ts).ExclusiveSum(mine, em, sme);
        if (h < H) {
            base[q * (H + 1) + h] = carry_all + ea + pre;
            lcum[q * (H + 1) + h] = carry_me + em;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            carry_all += sa;
            carry_me += sme;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        base[q * (H + 1) + H] = carry_all;
        lcum[q * (H + 1) + H] = carry_me;
        gtot[q] = carry_all;
    }
}

// number of this rank's candidates whose global position is < P
__device__ __forceinline__ int gp_loc(const int32_t *__restrict__ base, const int32_t *__restrict__ lcum, int H, int P) {
    if (base[0] > P) return 0;
    int lo = 0, hi = H;  // the last h with base[h] <= P (base is non-decreasing)
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (base[mid] <= P) lo = mid;
        else hi = mid - 1;
    }
    const int mine = lo < H ? lcum[lo + 1] - lcum[lo] : 0;
    return lcum[lo] + min(max(P - base[lo], 0), mine);
}

// global position of this rank's candidate at local position i
__device__ __forceinline__ int gp_gpos(const int32_t *__restrict__ base, const int32_t *__restrict__ lcum, int H, int i) {
    int lo = 0, hi = H;  // the last h with lcum[h] <= i: the (non-empty) bin holding i
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (lcum[mid] <= i) lo = mid;
        else hi = mid - 1;
    }
    return base[lo] + (i - lcum[lo]);
}

// this round's local span of every running query: st.pos / st.nlen (the own-span
// convention of the verification kernels)
__global__ void k_gp_span(int64_t Q, int H, const int32_t *__restrict__ base, const int32_t *__restrict__ lcum,
                          const int32_t *__restrict__ gtot, const int32_t *__restrict__ gpos,
                          const int32_t *__restrict__ glen, PatState st) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= Q) return;
    if (st.done[q]) {
        st.nlen[q] = 0;
        return;
    }
    const int P0 = gpos[q], P1 = min(P0 + glen[q], gtot[q]);
    const int32_t *b = base + q * (H + 1), *l = lcum + q * (H + 1);
    const int a = gp_loc(b, l, H, P0), e = gp_loc(b, l, H, P1);
    st.pos[q] = a;
    st.nlen[q] = e - a;
}

// the window's rows that may improve the top-k as it stood at the round's start,
// in ascending position (warp per query)
__global__ void __launch_bounds__(THREADS) k_gp_emit(int64_t Q, int k, PatState st, const double *__restrict__ dbuf,
                                                      int DS, const int32_t *__restrict__ order, int64_t CAPQ,
                                                      int64_t gid_base, int H,
                                                      const int32_t *__restrict__ base,
                                                      const int32_t *__restrict__ lcum, GEnt *__restrict__ stage,
                                                      int32_t *__restrict__ cnt) {
    const int64_t q = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (q >= Q) return;
    if (st.done[q]) {
        if (lane == 0) cnt[q] = 0;
        return;
    }
    const int a = st.pos[q], n = st.nlen[q];
    const bool full = st.cnt[q] >= k;
    const double dk = full ? st.Td[q * k + k - 1] : 0.0;
    const int64_t ik = full ? st.Ti[q * k + k - 1] : 0;
    const int32_t *b = base + q * (H + 1), *l = lcum + q * (H + 1);
    GEnt *out = stage + q * (int64_t)DS;
    int c = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
        const int j = j0 + lane;
        bool em = false;
        int lid = 0;
        double d = 0.0;
        if (j < n) {
            d = dbuf[q * (int64_t)DS + j];
            lid = order[q * CAPQ + a + j];
            em = !full || less_di(d, gid_base + lid, dk, ik);
        }
        const unsigned m = __ballot_sync(0xffffffffu, em);
        if (em) out[c + __popc(m & ((1u << lane) - 1u))] = GEnt{gp_gpos(b, l, H, a + j), lid, d};
        c += __popc(m);
    }
    if (lane == 0) cnt[q] = c;
}

__global__ void k_gp_pack(int64_t Q, int DS, const GEnt *__restrict__ stage, const int32_t *__restrict__ cnt,
                          const int32_t *__restrict__ offs, GEnt *__restrict__ packed) {
    const int64_t q = blockIdx.x;
    const int n = cnt[q], o = offs[q];
    for (int i = threadIdx.x; i < n; i += blockDim.x) packed[o + i] = stage[q * (int64_t)DS + i];
}

// every rank replays the window in global order (warp per query; lane g < G
// holds the head of rank g's list, a warp arg-min picks the next entry)
__global__ void __launch_bounds__(THREADS) k_gp_replay(int64_t Q, int G, int k, int P, const int32_t *__restrict__ all_cnt,
                                                        const int32_t *__restrict__ all_off,
                                                        const GEnt *__restrict__ all_ent, int64_t stride,
                                                        const int64_t *__restrict__ gbase, PatState st,
                                                        int32_t *__restrict__ gpos, int32_t *__restrict__ glen,
                                                        const int32_t *__restrict__ gtot, int nl_min, int nl_max,
                                                        int32_t *__restrict__ running) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t q = (int64_t)blockIdx.x * WARPS + warp;
    if (q >= Q || st.done[q]) return;
    double *Td = (double *)sm + warp * k;
    int64_t *Ti = (int64_t *)((double *)sm + WARPS * k) + warp * k;
    int cnt_top = st.cnt[q], pat = st.pat[q];
    for (int i = lane; i < cnt_top; i += 32) {
        Td[i] = st.Td[q * k + i];
        Ti[i] = st.Ti[q * k + i];
    }
    __syncwarp();
    const int P0 = gpos[q], P1 = min(P0 + glen[q], gtot[q]);
    // lane g: rank g's list of this query
    const int nmine = lane < G ? all_cnt[(int64_t)lane * Q + q] : 0;
    const GEnt *mine = lane < G ? all_ent + (int64_t)lane * stride + all_off[(int64_t)lane * (Q + 1) + q] : nullptr;
    int head = 0;
    int last = P0 - 1, stop = -1;
    for (;;) {
        const int hp = head < nmine ? mine[head].gpos : 0x7fffffff;
        // arg-min over the lanes (positions are distinct across ranks)
        int mp = hp, ml = lane;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const int op = __shfl_xor_sync(0xffffffffu, mp, o), ol = __shfl_xor_sync(0xffffffffu, ml, o);
            if (op < mp || (op == mp && ol < ml)) {
                mp = op;
                ml = ol;
            }
        }
        if (mp == 0x7fffffff) break;
        int lid = 0;
        double d = 0.0;
        if (lane == ml) {
            lid = mine[head].lid;
            d = mine[head].d;
            head++;
        }
        lid = __shfl_sync(0xffffffffu, lid, ml);
        d = __shfl_sync(0xffffffffu, d, ml);
        const int gap = mp - last - 1;  // certain misses before this entry
        if (P > 0 && pat + gap >= P) {
            stop = last + (P - pat);
            break;
        }
        pat += gap;
        const int64_t gid = gbase[ml] + lid;
        if (cnt_top < k || less_di(d, gid, Td[k - 1], Ti[k - 1])) {
            warp_insert(Td, Ti, cnt_top, k, d, gid, lane);
            pat = 0;
        } else {
            pat++;
            if (P > 0 && pat >= P) {
                stop = mp;
                break;
            }
        }
        last = mp;
    }
    if (stop < 0) {
        const int gap = P1 - 1 - last;
        if (P > 0 && pat + gap >= P) stop = last + (P - pat);
        else pat += gap;
    }
    for (int i = lane; i < cnt_top; i += 32) {
        st.Td[q * k + i] = Td[i];
        st.Ti[q * k + i] = Ti[i];
    }
    if (lane == 0) {
        st.cnt[q] = cnt_top;
        st.pat[q] = pat;
        if (stop >= 0 || P1 >= gtot[q]) {
            st.done[q] = 1;
            st.nver[q] = stop >= 0 ? stop + 1 : gtot[q];
        } else {
            gpos[q] = P1;
            glen[q] = P > 0 ? min(nl_max, max(nl_min, P - pat)) : nl_max;
            atomicAdd(running, 1);
        }
    }
}

__global__ void k_gp_result(int64_t Q, int k, PatState st, double *__restrict__ out_d64, int64_t *__restrict__ out_i) {
    const int64_t q = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (q >= Q) return;
    write_topk(q, k, st.cnt[q], st.Td + q * k, st.Ti + q * k, out_d64, nullptr, out_i, lane, 32);
}

void session_gp_order(crisp_session *ss, const int32_t *gcount, const int32_t *allhist, int32_t G, int32_t rank,
                      int32_t *local_hh, cudaStream_t s) {
    Work &w = *ss->w;
    const crisp_index *ix = ss->ix;
    CRISP_CHECK(ss->mode == 1, "global patience is for Optimized Mode sessions");
    {
        StageScope st(s, 3);
        k_fb_select<<<(unsigned)ss->Q, THREADS, w.count_smem, s>>>(
            w.act, w.act_len, ix->M, ix->K * ix->K, ix->off2, ix->NB, ix->ids, ix->N, ix->BS, ss->k, gcount, allhist,
            G, rank, ss->Q, w.pool, w.CAPQ, w.cbase, w.ncand, w.NS, w.fb, w.ghist, ix->Dp + 1);
        CRISP_LAUNCH();
        g_launches++;
    }
    w.full_order = true;  // the global window may reach any local position
    run_order(w, ss->Q, s);
    CRISP_CUDA(cudaMemcpyAsync(local_hh, w.ghist, (size_t)ss->Q * (ix->Dp + 1) * 4, cudaMemcpyDeviceToDevice, s));
}

void session_gp_prepare(crisp_session *ss, const int32_t *all_hh, int32_t G, int32_t rank, const int64_t *gid_bases,
                        cudaStream_t s) {
    Work &w = *ss->w;
    const crisp_index *ix = ss->ix;
    const int64_t Q = ss->Q;
    delete ss->gp;
    GPBuf *gp = ss->gp = new GPBuf();
    gp->G = G;
    gp->rank = rank;
    gp->H = ix->Dp + 1;
    gp->nl_min = std::max(32, env_int("CRISP_GP_MIN", 512));
    gp->nl_max = std::max(gp->nl_min, std::min(w.DS, env_int("CRISP_GP_MAX", 4096)));
    gp->base = gp->alloc<int32_t>((size_t)Q * (gp->H + 1), s);
    gp->lcum = gp->alloc<int32_t>((size_t)Q * (gp->H + 1), s);
    gp->gtot = gp->alloc<int32_t>((size_t)Q, s);
    gp->gpos = gp->alloc<int32_t>((size_t)Q, s);
    gp->glen = gp->alloc<int32_t>((size_t)Q, s);
    gp->cnt = gp->alloc<int32_t>((size_t)Q + 1, s);
    gp->offs = gp->alloc<int32_t>((size_t)Q + 1, s);
    gp->stage = gp->alloc<GEnt>((size_t)Q * w.DS, s);
    gp->packed = gp->alloc<GEnt>((size_t)Q * w.DS, s);
    gp->running = gp->alloc<int32_t>(1, s);
    gp->all_off = gp->alloc<int32_t>((size_t)G * (Q + 1), s);
    gp->gbase = gp->alloc<int64_t>((size_t)G, s);
    CRISP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, gp->scan_bytes, gp->cnt, gp->offs, (int)Q + 1, s));
    gp->scan_tmp = gp->alloc<unsigned char>(gp->scan_bytes, s);
    CRISP_CUDA(cudaMemcpyAsync(gp->gbase, gid_bases, (size_t)G * 8, cudaMemcpyHostToDevice, s));
    k_gp_tables<<<(unsigned)Q, 256, 0, s>>>(all_hh, G, rank, Q, gp->H, gp->base, gp->lcum, gp->gtot);
    CRISP_LAUNCH();
    g_launches++;
    // round 0: the first F positions (exact, or F ~ P without the filter)
    CRISP_CUDA(cudaMemsetAsync(gp->gpos, 0, (size_t)Q * 4, s));
    std::vector<int32_t> h0((size_t)Q, std::min(w.F, w.DS));
    CRISP_CUDA(cudaMemcpyAsync(gp->glen, h0.data(), (size_t)Q * 4, cudaMemcpyHostToDevice, s));
    CRISP_CUDA(cudaStreamSynchronize(s));  // h0 is a host temporary
    if (w.lbf) w.q8_prep(Q, s);
}

void session_gp_round(crisp_session *ss, int64_t *n_entries, cudaStream_t s) {
    Work &w = *ss->w;
    const crisp_index *ix = ss->ix;
    GPBuf *gp = ss->gp;
    CRISP_CHECK(gp != nullptr, "crisp_shard_gp_prepare first");
    const int64_t Q = ss->Q;
    const int k = ss->k, pitch = ix->pitch;
    StageScope st(s, 4);
    k_gp_span<<<nblk(Q, 256), 256, 0, s>>>(Q, gp->H, gp->base, gp->lcum, gp->gtot, gp->gpos, gp->glen, w.pst);
    CRISP_LAUNCH();
    dim3 g(w.S1, (unsigned)Q);
    if (w.lbf)
        k_verify_rows_lb<3><<<g, THREADS, w.vrl_smem, s>>>(w.qrot, pitch, ix->X, w.fa, w.cbuf, w.CAPQ, w.totals,
                                                           w.pst, k, -1, 0, 0x7fffffff, w.DS, w.dbuf, w.qperm,
                                                           g_counters ? d_filter_stats_ptr() : nullptr);
    else if (w.rows4)
        k_verify_rows<true><<<g, THREADS, w.vr_smem, s>>>(w.qrot, pitch, ix->X, w.cbuf, w.CAPQ, w.totals, w.pst, -1,
                                                          0, 0x7fffffff, w.DS, w.dbuf, w.qperm);
    else
        k_verify_rows<false><<<g, THREADS, w.vr_smem, s>>>(w.qrot, pitch, ix->X, w.cbuf, w.CAPQ, w.totals, w.pst, -1,
                                                           0, 0x7fffffff, w.DS, w.dbuf, w.qperm);
    CRISP_LAUNCH();
    k_gp_emit<<<nblk(Q, WARPS), THREADS, 0, s>>>(Q, k, w.pst, w.dbuf, w.DS, w.cbuf, w.CAPQ, ix->gid_base, gp->H,
                                                  gp->base, gp->lcum, gp->stage, gp->cnt);
    CRISP_LAUNCH();
    CRISP_CUDA(cudaMemsetAsync(gp->cnt + Q, 0, 4, s));
    CRISP_CUDA(cub::DeviceScan::ExclusiveSum(gp->scan_tmp, gp->scan_bytes, gp->cnt, gp->offs, (int)Q + 1, s));
    k_gp_pack<<<(unsigned)Q, 128, 0, s>>>(Q, w.DS, gp->stage, gp->cnt, gp->offs, gp->packed);
    CRISP_LAUNCH();
    g_launches += 5;
    int32_t tot = 0;
    CRISP_CUDA(cudaMemcpyAsync(&tot, gp->offs + Q, 4, cudaMemcpyDeviceToHost, s));
    CRISP_CUDA(cudaStreamSynchronize(s));
    gp->n_packed = tot;
    *n_entries = tot;
}

void session_gp_fetch(crisp_session *ss, void *entries, int32_t *counts, cudaStream_t s) {
    GPBuf *gp = ss->gp;
    CRISP_CHECK(gp != nullptr, "crisp_shard_gp_round first");
    CRISP_CUDA(cudaMemcpyAsync(entries, gp->packed, (size_t)gp->n_packed * sizeof(GEnt), cudaMemcpyDeviceToDevice, s));
    CRISP_CUDA(cudaMemcpyAsync(counts, gp->cnt, (size_t)ss->Q * 4, cudaMemcpyDeviceToDevice, s));
}

void session_gp_replay(crisp_session *ss, const int32_t *all_cnt, const void *all_ent, int64_t stride, int32_t G,
                       int32_t *running, cudaStream_t s) {
    Work &w = *ss->w;
    const crisp_index *ix = ss->ix;
    GPBuf *gp = ss->gp;
    CRISP_CHECK(gp != nullptr && G == gp->G, "crisp_shard_gp_prepare first (same G)");
    const int64_t Q = ss->Q;
    const int k = ss->k;
    const int P = ix->patience_factor > 0 ? ix->patience_factor * k : 0;
    StageScope st(s, 4);
    for (int g = 0; g < G; g++) {
        // rank g's counts, then a 0 for the exclusive scan's total
        CRISP_CUDA(cudaMemcpyAsync(gp->cnt, all_cnt + (int64_t)g * Q, (size_t)Q * 4, cudaMemcpyDeviceToDevice, s));
        CRISP_CUDA(cudaMemsetAsync(gp->cnt + Q, 0, 4, s));
        CRISP_CUDA(cub::DeviceScan::ExclusiveSum(gp->scan_tmp, gp->scan_bytes, gp->cnt, gp->all_off + (int64_t)g * (Q + 1),
                                                 (int)Q + 1, s));
    }
    CRISP_CUDA(cudaMemsetAsync(gp->running, 0, 4, s));
    k_gp_replay<<<nblk(Q, WARPS), THREADS, WARPS * k * 16, s>>>(Q, G, k, P, all_cnt, gp->all_off, (const GEnt *)all_ent,
                                                                 stride, gp->gbase, w.pst, gp->gpos, gp->glen, gp->gtot,
                                                                 gp->nl_min, gp->nl_max, gp->running);
    CRISP_LAUNCH();
    g_launches++;
    CRISP_CUDA(cudaMemcpyAsync(running, gp->running, 4, cudaMemcpyDeviceToHost, s));
    CRISP_CUDA(cudaStreamSynchronize(s));
}

void session_gp_result(crisp_session *ss, int64_t *out_ids, double *out_d64, cudaStream_t s) {
    Work &w = *ss->w;
    k_gp_result<<<nblk(ss->Q, WARPS), THREADS, 0, s>>>(ss->Q, ss->k, w.pst, out_d64, out_ids);
    CRISP_LAUNCH();
    g_launches++;
    run_stats(w, ss->Q, s);
}

void session_free(crisp_session *ss) {
    if (!ss) return;
    delete ss->gp;
    delete ss->w;
    delete ss;
}

void merge_topk(const double *d, const int64_t *ids, int32_t G, int64_t Q, int32_t k, double *out_d64, float *out_d,
                int64_t *out_ids, cudaStream_t s) {
    if (Q <= 0) return;
    k_merge_lists<<<(unsigned)Q, THREADS, 0, s>>>(d, ids, G, Q, k, 1, out_d64, out_d, out_ids);
    CRISP_LAUNCH();
    g_launches++;
}


}  // namespace crisp

// stage timing ABI
extern "C" crisp_status crisp_set_stage_timing(int32_t on) {
    crisp::g_timing = on != 0;
    crisp::g_counters = on == 1;  // 2: stage events only (no extra kernels in the timed work)
    return CRISP_OK;
}

extern "C" crisp_status crisp_search_counters(int64_t *out, int32_t n, int32_t reset) {
    unsigned long long h[4], hp[2], hf[2];
    if (cudaMemcpyFromSymbol(h, crisp::d_stats, sizeof(h)) != cudaSuccess ||
        cudaMemcpyFromSymbol(hp, crisp::d_probe_stats, sizeof(hp)) != cudaSuccess ||
        cudaMemcpyFromSymbol(hf, crisp::d_filter_stats, sizeof(hf)) != cudaSuccess) {
        crisp::set_error("cudaMemcpyFromSymbol failed");
        return CRISP_ECUDA;
    }
    for (int i = 0; i < 4 && i < n; i++) out[i] = (int64_t)h[i];
    if (n > 4) out[4] = crisp::g_launches;
    if (n > 5) out[5] = (int64_t)hp[0];
    if (n > 6) out[6] = (int64_t)hp[1];
    if (n > 7) out[7] = (int64_t)hf[0];
    if (n > 8) out[8] = (int64_t)hf[1];
    if (reset) {
        unsigned long long z[4] = {0, 0, 0, 0};
        cudaMemcpyToSymbol(crisp::d_stats, z, sizeof(z));
        cudaMemcpyToSymbol(crisp::d_probe_stats, z, 2 * sizeof(unsigned long long));
        cudaMemcpyToSymbol(crisp::d_filter_stats, z, 2 * sizeof(unsigned long long));
        crisp::g_launches = 0;
    }
    return CRISP_OK;
}

extern "C" crisp_status crisp_stage_times(double *ms, int32_t n, int32_t reset) {
    for (auto &e : crisp::g_events) {
        cudaEventSynchronize(e.b);
        float t = 0.f;
        cudaEventElapsedTime(&t, e.a, e.b);
        if (e.stage >= 0 && e.stage < 8) crisp::g_stage_ms[e.stage] += t;
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    crisp::g_events.clear();
    for (int i = 0; i < n && i < 8; i++) ms[i] = crisp::g_stage_ms[i];
    if (reset)
        for (int i = 0; i < 8; i++) crisp::g_stage_ms[i] = 0.0;
    return CRISP_OK;
}
