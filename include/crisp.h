/*
 * crisp.h -- C ABI of the B200-native CRISP query engine (libcrisp.so).
 *
 * CRISP: Correlation-Resilient Indexing via Subspace Partitioning (arXiv
 * 2603.05180).  Citations "P:Lnnn" are lines of the paper's LaTeX source
 * (PAPER.md), "S:Lnnn" lines of SPEC.md.  The problem is kNN under L2 over
 * X in R^{N x D}; results are squared L2 distances.
 *
 * Conventions for every call:
 *  - Ownership: the caller owns every input and output buffer.  Builds copy the
 *    data into HBM and never keep a caller pointer; an index owns all its device
 *    memory until crisp_free.
 *  - Pointers: "host or device" arguments are classified with
 *    cudaPointerGetAttributes; *_async calls require device pointers and run on
 *    the given cudaStream_t (passed as void*; NULL = legacy default stream).
 *  - Layout: row-major, fp32 vectors, int64 ids, Q x k results ascending by
 *    (distance, id), padded with (-1, +inf) when fewer than k candidates exist.
 *  - Errors: every call returns a crisp_status; crisp_last_error() returns a
 *    thread-local message for the last non-OK status of the calling thread.
 *    CRISP_EINVAL: bad argument (k < 1 or k > N, non-finite data, M < 1, K < 1,
 *    M > 127, K > 255, NULL pointer).  CRISP_ECUDA / CRISP_ENOMEM pass through
 *    the CUDA failure (message holds cudaGetErrorString).  There is no CPU
 *    fallback: without a working CUDA device every compute call fails.
 *  - Thread safety: an index is read-only during search; concurrent searches
 *    on different streams are allowed (scratch is per call).  Parameter setters
 *    must not race with searches.
 */
#ifndef CRISP_H
#define CRISP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CRISP_OK = 0,
    CRISP_EINVAL = 1,
    CRISP_EIO = 2,
    CRISP_ENOMEM = 3,
    CRISP_ECUDA = 4,
    CRISP_ENCCL = 5,
    CRISP_EUNSUPPORTED = 6
} crisp_status;

/* Execution flag phi (Table 1; Sec. 4.3.2). */
typedef enum {
    CRISP_GUARANTEED = 0, /* binary scoring, exhaustive exact-L2 verification */
    CRISP_OPTIMIZED = 1   /* rank-weighted scoring, Hamming order, patience */
} crisp_mode;

typedef struct crisp_index crisp_index;     /* opaque; owns HBM */
typedef struct crisp_session crisp_session; /* opaque; one phased shard search (owns its scratch) */

typedef struct {
    int32_t M;                 /* subspaces (required, no paper default) */
    int32_t K;                 /* centroids per half-subspace, default 50 */
    float tau_cev;             /* CEV gate, default 0.85; rotate iff CEV > tau_cev */
    int32_t rotation;          /* -1 auto (gate), 0 force off, 1 force on */
    int32_t kmeans_iters;      /* Lloyd iterations, default 20 */
    int64_t kmeans_sample;     /* k-means training rows, default 100000 */
    uint64_t seed;             /* drives every random draw of the method (Philox4x32-10) */
    int32_t device;            /* CUDA device ordinal */
    double budget_ratio;       /* beta: per-subspace retrieved fraction (range 0.001-0.06 P:L525) */
    int64_t budget;            /* if > 0 overrides beta: B ids per subspace (exact integer) */
    double min_collision_ratio;/* alpha: tau = ceil(alpha*M) (range 0.1-0.6 P:L525) */
    int32_t tau;               /* if > 0 overrides alpha: integer collision threshold */
    int32_t patience_factor;   /* P = patience_factor * k (default 40); 0 = disabled */
    int64_t workspace_bytes;   /* per-search scratch cap (query chunking); 0 = default: half the free device memory, in [4, 64] GiB */
    int32_t rotation_block;    /* 0: global rotation when it applies; b > 0: block-wise variance
                                  redistribution (DESIGN R16): rotate only the dimensions of the b
                                  subspaces of largest sample variance, R = I elsewhere */
    int32_t adaptive_subspaces; /* 0: M equal subspaces; 1: adaptive subspace decomposition
                                   (DESIGN R18): contiguous even widths cut where the stored
                                   vectors' running per-dimension variance (CEV sample) first reaches
                                   j/M of the total, halves of equal width; ignored if subspace_widths */
    const int32_t *subspace_widths; /* NULL, or M even widths >= 2 summing to padded_D (host memory,
                                   read during the build call only): subspace m covers dims
                                   [sum_{j<m} w_j, sum_{j<=m} w_j), halves of w_m / 2; required with
                                   injected codebooks of a non-equal split.  Codebook rows keep the
                                   stride dh = max w_m / 2, zero beyond the half's width.  Not
                                   supported by crisp_build_model (equal split only). */
} crisp_params;

typedef struct {
    int64_t N;          /* points held by this index (shard-local) */
    int64_t N_global;   /* points of the whole dataset (budget base) */
    int64_t gid_base;   /* global id of local point 0 */
    int32_t D;          /* input dimensionality */
    int32_t padded_D;   /* D zero-padded to a multiple of 2M */
    int32_t pitch;      /* row pitch of the stored vectors in floats (multiple of 4) */
    int32_t M, K, dh;   /* dh = padded_D / (2M) */
    int32_t rotated;    /* 1 if X' = XR was applied */
    double cev;         /* measured CEV */
    int64_t budget;     /* B ids per subspace in effect */
    int32_t tau;        /* collision threshold in effect */
    int32_t patience_factor;
    int32_t block_ids;  /* ids per on-chip counter block */
    int32_t n_blocks;
    int64_t hbm_bytes;  /* device bytes owned by the index */
    int64_t logical_bytes; /* 4ND + 4MN + 8M(K^2+1) + codebooks + 8*ceil(D/64)*N + 4D^2 if rotated */
    double slice_hint;  /* expected ids per activated slice and 4096-id warp sub-block: >= 8 selects the
                           warp-owned collision-count kernel, else the CTA-flattened one (env CRISP_COUNT_KERNEL) */
    int32_t rotation_block; /* subspaces of a block-wise rotation (0: global or none) */
    int32_t adaptive;       /* 1 if the subspace widths are not the equal split (R18) */
} crisp_index_info_t;

/* Host buffers filled by crisp_export (any may be NULL to skip). */
typedef struct {
    float *R;          /* padded_D x padded_D (only if rotated) */
    float *X;          /* N x padded_D stored vectors (rotated if applied) */
    float *codebooks;  /* M x 2 x K x dh */
    int32_t *cells;    /* M x N cell ids */
    int64_t *offsets;  /* M x (K^2+1) CSR Offsets */
    int32_t *ids;      /* M x N CSR ids, local */
    uint64_t *codes;   /* N x ceil(padded_D/64) binary codes */
    int64_t *cell_sizes; /* M x K^2 sizes used for budgets (global after crisp_set_global_cell_sizes) */
    int32_t *subspace_widths; /* M: the subspace widths in effect (equal: 2 dh each) */
} crisp_export_t;

/* Host buffers filled by crisp_search_trace (any may be NULL).  Stage outputs of
 * Alg. 1 for parity checks. */
typedef struct {
    int32_t *act_len;    /* Q x M: activated cells per (q,m) (a2) */
    int32_t *act_cell;   /* Q x M x K^2: activated cells in pop order (a2) */
    int32_t *act_w;      /* Q x M x K^2: their weights 1/2 (a2, Alg. 1 l.10-12) */
    int64_t *retrieved;  /* Q x M: ids retrieved, budget counting (Alg. 1 l.16) */
    uint8_t *V;          /* Q x N: collision scores (a3, Eq. 1) */
    int64_t *cand_n;     /* Q: |C_q| (a4) */
    int32_t *cand;       /* Q x N: C_q local ids ascending (a4, Alg. 1 l.18) */
    int32_t *order;      /* Q x N: verification order (phi=1: Hamming (h,id); phi=0: C_q) */
    int64_t *n_verified; /* Q: candidates verified (phi=1: patience stop) */
    int32_t *fallback;   /* Q: 1 if the underflow fallback fired */
    float *qrot;         /* Q x padded_D: transformed query q' (a0) */
} crisp_trace_t;

/* Fill p with the paper's defaults (K=50, tau_cev=0.85, 20 Lloyd iterations,
 * 1e5 k-means rows, beta=0.01, alpha=0.3, P=40k). */
crisp_status crisp_default_params(crisp_params *p);

/* Build (P:L249-256 phases 1-2): spectral check on a min(0.1N,1e5) sample
 * (P:L264-268), adaptive rotation X' = XR in place, 2M k-means
 * codebooks, cell assignment, per-subspace CSR Offsets/IDs
 * (P:L363-369), binary codes.  data: N x D fp32 row-major, host or
 * device; a device buffer may still be being written on any stream: the call
 * synchronizes the device first.  On success *out owns the index. */
crisp_status crisp_build(const float *data, int64_t N, int32_t D, const crisp_params *p, crisp_index **out);

/* Same, with the rotation R (padded_D x padded_D fp32 row-major, or NULL for
 * no rotation) and the codebooks (M x 2 x K x dh fp32) injected instead of
 * computed; used for parity ("given the same seeded inputs and codebooks"). */
crisp_status crisp_build_with(const float *data, int64_t N, int32_t D, const crisp_params *p, const float *R_or_null,
                              const float *codebooks, crisp_index **out);

/* One shard of a point-sharded index: local rows with global ids
 * gid_base..gid_base+N_local-1, shared R and codebooks (both injected; R may be
 * NULL).  Budgets use local sizes until crisp_set_global_cell_sizes. */
crisp_status crisp_build_shard(const float *shard, int64_t N_local, int64_t gid_base, int32_t D, const crisp_params *p,
                               const float *R_or_null, const float *codebooks, crisp_index **out);

/* Local cell sizes, M x K^2 int64 host buffer (for the allreduce of N3). */
crisp_status crisp_local_cell_sizes(const crisp_index *idx, int64_t *sizes);

/* Install summed (global) cell sizes, M x K^2 int64 host buffer: the budget
 * walk of a2 then activates exactly the cells a single global index would. */
crisp_status crisp_set_global_cell_sizes(crisp_index *idx, const int64_t *sizes);

/* Set search knobs.  beta/alpha are used only when budget/tau <= 0:
 * B = max(1, ceil(beta*N_global)) ("retrieve beta of the dataset per
 * subspace"; Z1/Z3) and tau = max(1, ceil(alpha*M)) (Thm 1's
 * threshold alpha*M; R1), both computed exactly as crisp_exact_ceil does.  A
 * budget given as beta follows N_global when crisp_set_global_cell_sizes
 * changes it; an integer budget is kept as given.  EINVAL: beta or alpha
 * outside (0, 1] when used, patience_factor < 0. */
crisp_status crisp_set_search_params(crisp_index *idx, double beta, int64_t budget, double alpha, int32_t tau,
                                     int32_t patience_factor);

/* Optimized Mode verification by ADSampling (Eq. 2; SURVEY 8(f)
 * row f1): a candidate is pruned at the first t = stride, 2*stride, ... < D at
 * which its partial squared distance over the first t stored dimensions
 * exceeds r_k^2 * (t/D) * (1 + eps0/sqrt(t))^2, r_k^2 being the current k-th
 * best squared distance (+inf until k results exist); a pruned candidate counts
 * as a non-improving verification for the patience rule.  enable = 0
 * restores exact verification.  The paper's values are eps0 = 2.1 and
 * stride = 32.  stride must divide 128 and be a multiple of 4; eps0
 * must be >= 0.  Applies to searches with mode CRISP_OPTIMIZED only. */
crisp_status crisp_set_adsampling(crisp_index *idx, int32_t enable, double eps0, int32_t stride);

/* Verification filter (a5 of both modes; DESIGN R17).  The exact re-rank
 * (Alg. 1 l.22-27) only needs the exact distance of a candidate
 * that can enter the current top-k.  With the filter on, the index keeps every
 * stored row centred on the column means and quantised per row to int8
 * (x - mu ~ 2^e c), with c.c, e and a rounded-up residual norm per row; a
 * search first bounds ||q' - x|| from below through that copy (exact integer
 * dot products with two int8 digit planes of q' - mu, Cauchy-Schwarz and the
 * triangle inequality, certified fp64 rounding) and reads the fp32 row only
 * when the bound does not exceed the current k-th best distance.  A candidate
 * skipped this way is one the exact rule would verify without improving the
 * top-k, so ids, distances and patience stops are unchanged.  enable = 1
 * builds the copy (N x padded_D bytes + 16 B per row of HBM) if absent;
 * enable = 0 frees it.  Indexes are built with the filter on unless the
 * environment sets CRISP_VERIFY_FILTER=0.  Blocks until searches in flight on
 * the index's device have finished. */
crisp_status crisp_set_verify_filter(crisp_index *idx, int32_t enable);

crisp_status crisp_index_info(const crisp_index *idx, crisp_index_info_t *out);

/* Batched search, Alg. 1: a0 query transform, a1 half distances,
 * a2 Multi-Sequence cell selection under the budget, a3 collision counting
 * over the CSR lists, a4 threshold + fallback (+ Hamming order if phi=1), a5
 * exact L2 verification (+ patience if phi=1) and top-k.  queries: Q x D fp32
 * (host or device); out_ids: Q x k int64 global ids; out_dist2: Q x k fp32
 * squared L2 (host or device).  Synchronous. */
crisp_status crisp_search(const crisp_index *idx, const float *queries, int64_t Q, int32_t k, crisp_mode mode,
                          int64_t *out_ids, float *out_dist2);

/* Stream-ordered search on device pointers; returns after enqueueing. */
crisp_status crisp_search_async(const crisp_index *idx, const float *queries, int64_t Q, int32_t k, crisp_mode mode,
                                int64_t *out_ids, float *out_dist2, void *stream);

/* Shard search for multi-GPU merging: like crisp_search_async but returns
 * fp64 distances (out_dist64, Q x k) so the cross-shard merge orders by the
 * same dist64 values as a single index (SURVEY App. A.1, A.2 "Merge"). */
crisp_status crisp_search_shard_async(const crisp_index *idx, const float *queries, int64_t Q, int32_t k,
                                      crisp_mode mode, int64_t *out_ids, double *out_dist64, void *stream);

/* Global top-k by (d, gid) over G per-shard lists (device pointers, G x Q x k
 * each, ids < 0 are padding) -> Q x k (a6). */
crisp_status crisp_merge_topk(const double *d, const int64_t *ids, int32_t G, int64_t Q, int32_t k, double *out_d64,
                              float *out_d, int64_t *out_ids, void *stream);

/* Phased shard search with the EXACT global underflow fallback (P:L449 applied
 * to the whole point-sharded dataset).  All pointers are device
 * pointers on `stream`; the caller runs the collectives in between:
 *   1. begin: a0..a4 without the fallback; local_counts[q] = local |C_q|.
 *   2. caller: all-reduce(SUM) local_counts -> global_counts.
 *   3. hist: for queries with global |C_q| < k, local_hist[q][v] = number of
 *      touched local ids with score v (v = 0..2M; Q x (2M+2) int32).
 *   4. caller: all-gather local_hist over the G ranks -> all_hist (G x Q x (2M+2)).
 *   5. finish: fallback queries take the global top-k touched ids by
 *      (V desc, gid asc) -- this rank keeps ids with V > V* and its share of the
 *      V == V* quota in rank (= global id) order -- then a5 verification;
 *      out_ids / out_dist64 are this shard's Q x k top-k by (d, gid).
 * The batch is processed as one chunk.  free releases the session. */
crisp_status crisp_shard_search_begin(const crisp_index *idx, const float *queries, int64_t Q, int32_t k,
                                      crisp_mode mode, int32_t *local_counts, crisp_session **out, void *stream);
crisp_status crisp_shard_search_hist(crisp_session *s, const int32_t *global_counts, int32_t *local_hist,
                                     void *stream);
crisp_status crisp_shard_search_finish(crisp_session *s, const int32_t *global_counts, const int32_t *all_hist,
                                       int32_t G, int32_t rank, int64_t *out_ids, double *out_dist64, void *stream);
void crisp_shard_search_free(crisp_session *s);

/* a0 alone: qrot[q][0..pitch) = fl32(q R) zero-padded (the
 * queries themselves, padded, when the index is not rotated), pitch = the
 * stored row pitch of crisp_index_info_t.  queries: Q x D, qrot: Q x pitch
 * fp32, both device memory; stream-ordered.  With
 * crisp_shard_search_begin_transformed a sharded search transforms each
 * rank's slice of the batch once and all-gathers q' instead of
 * every rank transforming every query; the results are identical. */
crisp_status crisp_transform_queries_async(const crisp_index *idx, const float *queries, int64_t Q, float *qrot,
                                           void *stream);
/* crisp_shard_search_begin with the queries already transformed (qrot: Q x
 * pitch fp32 device memory as written by crisp_transform_queries_async). */
crisp_status crisp_shard_search_begin_transformed(const crisp_index *idx, const float *qrot, int64_t Q, int32_t k,
                                                  crisp_mode mode, int32_t *local_counts, crisp_session **out,
                                                  void *stream);

/* Exact global patience for Optimized Mode over G point shards (Alg. 1
 * l.22-27 with the patience rule of P:L458 applied to the union of the shards'
 * candidates, in the global (h, gid) order).  Instead
 * of crisp_shard_search_finish, an Optimized-Mode session continues with:
 *   1. gp_order: the fallback selection (as finish), then the Hamming
 *      distances and the full local (h, gid) order; local_hhist[q][h] = number
 *      of this shard's candidates of query q at Hamming distance h
 *      (Q x (padded_D + 1) int32, device).
 *   2. caller: all-gather local_hhist -> all_hhist (G x Q x (padded_D + 1)).
 *   3. gp_prepare: position tables (the global position of every local
 *      candidate follows from all_hhist), round 0's window; gid_bases (host,
 *      G int64) are the shards' first global ids.
 *   4. rounds, until *running == 0:
 *      gp_round: verifies this shard's candidates in every running query's
 *        global window and keeps the ones that may improve the query's top-k
 *        (all others are certain misses) as 16-byte records
 *        {int32 global position, int32 local id, double exact distance},
 *        packed by query in ascending query and position; *n_entries (host)
 *        = how many;
 *      gp_fetch: copies them to entries (>= n_entries x 16 B, device) and
 *        their number per query to counts (Q int32, device);
 *      caller: all-gather counts -> all_counts (G x Q) and entries, each
 *        rank's padded to `stride` records -> all_entries (G x stride);
 *      gp_replay: every rank replays the windows in global order with the
 *        sequential rule (identical state on every rank); *running (host) =
 *        queries still running.
 *   5. gp_result: out_ids / out_dist64 (Q x k, device) = the global top-k by
 *      (d, gid), identical on every rank and to a single index over all rows.
 * G <= 32.  Host-synchronising (the sizes of the all-gathers). */
crisp_status crisp_shard_gp_order(crisp_session *s, const int32_t *global_counts, const int32_t *all_hist, int32_t G,
                                  int32_t rank, int32_t *local_hhist, void *stream);
crisp_status crisp_shard_gp_prepare(crisp_session *s, const int32_t *all_hhist, int32_t G, int32_t rank,
                                    const int64_t *gid_bases, void *stream);
crisp_status crisp_shard_gp_round(crisp_session *s, int64_t *n_entries, void *stream);
crisp_status crisp_shard_gp_fetch(crisp_session *s, void *entries, int32_t *counts, void *stream);
crisp_status crisp_shard_gp_replay(crisp_session *s, const int32_t *all_counts, const void *all_entries, int64_t stride,
                                   int32_t G, int32_t *running, void *stream);
crisp_status crisp_shard_gp_result(crisp_session *s, int64_t *out_ids, double *out_dist64, void *stream);

/* Search with stage outputs copied to host buffers (parity / tracing). */
crisp_status crisp_search_trace(const crisp_index *idx, const float *queries, int64_t Q, int32_t k, crisp_mode mode,
                                int64_t *out_ids, float *out_dist2, crisp_trace_t *trace);

/* Copy the index contents to host buffers. */
crisp_status crisp_export(const crisp_index *idx, crisp_export_t *out);

/* Stage timing: when enabled, every crisp_search* records CUDA events around
 * each stage on its stream and accumulates the device time per stage (ms) into
 * a per-thread table; crisp_stage_times synchronises on those events, copies up
 * to n entries (stage order: 0 transform, 1 probe a1+a2, 2 count+select a3+a4,
 * 3 fallback, 4 hamming+verify a4/a5, 5 merge) and, if reset != 0, clears it.
 * on = 1 also accumulates the work counters of crisp_search_counters (extra
 * tally kernels in the searched stream); on = 2 records the stage events only;
 * 0 turns both off. */
crisp_status crisp_set_stage_timing(int32_t on);
crisp_status crisp_stage_times(double *ms, int32_t n, int32_t reset);

/* Work counters accumulated over the searches run while stage timing is on
 * (current device), for algorithmic-byte accounting: out[0] ids streamed by
 * the collision count (a3), out[1] sum of |C_q| (a4), out[2] rows verified
 * (a5), out[3] queries that took the fallback, out[4] kernels of this library
 * launched by searches/merges on the calling thread (counted always), out[5]
 * exact half distances (dist64) the a1 probe computed, out[6] (query,
 * subspace) walks whose tensor-core screen did not cover the ranks the walk
 * reached and were redone on exact half sorts, out[7] candidate rows whose
 * distance bound the verification filter computed (crisp_set_verify_filter),
 * out[8] of those, rows whose fp32 row was read for the exact distance because
 * the bound could not exclude them.  Up to n entries are written;
 * reset != 0 clears them. */
crisp_status crisp_search_counters(int64_t *out, int32_t n, int32_t reset);

/* Distributed model build (SURVEY 8(e) N1/N2 without a full index on one rank).
 * The build's randomness is counter-based (Philox keyed by seed, streams per
 * use; DESIGN R3), so the CEV sample and the k-means sample of a dataset of
 * N_global rows are fixed sets of global row ids:
 *   crisp_cev_sample_size(N) = ceil(min(0.1 N, 1e5)) (all rows if N <= 10; P:L264,
 *     S:L117), the CEV sample's size;
 *   crisp_sample_rows(N, n, seed, stream, rows_out): the n sampled row ids in
 *     ascending order (the n rows of smallest (Philox key, id)); stream 1 = CEV
 *     sample, stream 3 = k-means sample (n = min(N, kmeans_sample));
 *     rows_out host or device, n int32.
 * Each rank contributes its rows of both samples; with the rows gathered in
 * ascending global id, crisp_build_model returns exactly the rotation (Dp x Dp
 * fp32 into R_out, written only if *rotated_out = 1), the codebooks (M x 2 x K
 * x dh into codebooks_out) and the CEV that crisp_build over all N_global rows
 * would use (spectral check P:L262-271, rotation P:L225, k-means S:L221).
 * cev_rows: n_cev x D fp32 (n_cev = crisp_cev_sample_size(N_global)); km_rows:
 * n_km x D fp32.  Buffers host or device; the caller owns all of them. */
int64_t crisp_cev_sample_size(int64_t N);
crisp_status crisp_sample_rows(int64_t N, int64_t n, uint64_t seed, uint32_t stream, int32_t *rows_out);
crisp_status crisp_build_model(const float *cev_rows, int64_t n_cev, const float *km_rows, int64_t n_km, int32_t D,
                               const crisp_params *p, float *R_out, float *codebooks_out, int32_t *rotated_out,
                               double *cev_out);

/* ceil(ratio * n) with ratio read as the decimal it was written as: the
 * shortest decimal string that rounds to `ratio` (what printf("%.17g")-free
 * languages print, e.g. 0.035), multiplied exactly in 128-bit integers
 * (floating ceil(0.035*20000) = 701, exact 700; ceil(0.07*100)
 * = 8, exact 7).  Returns 0 for ratio <= 0, a non-finite ratio or n <= 0.
 * Host-only; no device needed. */
int64_t crisp_exact_ceil(double ratio, int64_t n);

void crisp_free(crisp_index *idx);
const char *crisp_last_error(void);
const char *crisp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CRISP_H */
