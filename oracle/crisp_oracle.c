/*
 * oracle/crisp_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of CRISP
 * (Correlation-Resilient Indexing via Subspace Partitioning, arXiv 2603.05180),
 * written from PAPER.md.  It exists to check the CUDA path; it is never part of
 * the product.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  It shares no code, header,
 * table or constant with paper_2603_05180_b200/ (the CUDA path), and neither
 * side includes or imports the other.
 *
 * Citations: "P:Lnnn" = line nnn of PAPER.md (LaTeX source of the paper),
 * "S:Lnnn" = line of SPEC.md.  Readings of ambiguous passages are numbered
 * Z1..Z24 as in SURVEY.md 8(c) and listed in DESIGN.md.
 *
 * Arithmetic contract: every distance that decides an order
 * is dist64 = sum_i fma(d_i, d_i, s), d_i = (double)a_i - (double)b_i, summed in
 * ascending i from +0.0.  Compiled with -O2 -ffp-contract=off (no fast-math).
 *
 * Parity status: every exported function below is
 * pinned by a -m "not gpu" test except or_eig_sym_jacobi's convergence
 * tolerance (pinned by closed forms/trace identity only, not bit-exact).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------- */
/* Counter-based generator for the random numbers the METHOD draws: the CEV   */
/* sample, the Gaussian G of the rotation and the k-means   */
/* sample / k-means++ draws.  Philox4x32-10 (Salmon et al., SC'11).  The CUDA */
/* side implements the same generator independently.                          */
/* ------------------------------------------------------------------------- */
void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; r++) {
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        if (r < 9) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* stream ids */
#define OR_STREAM_CEV_SAMPLE 1u
#define OR_STREAM_ROTATION   2u
#define OR_STREAM_KM_SAMPLE  3u
#define OR_STREAM_KM_INIT    4u

static void draw(uint64_t seed, uint32_t stream, uint64_t idx, uint32_t sub, uint32_t out[4])
{
    uint32_t ctr[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), stream, sub};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    or_philox4x32_10(ctr, key, out);
}

/* 53-bit uniform in [0,1) from two words */
static double u53(uint32_t a, uint32_t b)
{
    uint64_t v = (((uint64_t)a << 32) | (uint64_t)b) >> 11;
    return (double)v * (1.0 / 9007199254740992.0);
}

double or_uniform(uint64_t seed, uint32_t stream, uint64_t idx, uint32_t sub)
{
    uint32_t o[4];
    draw(seed, stream, idx, sub, o);
    return u53(o[0], o[1]);
}

/* Standard normal by Box-Muller (one normal per counter). */
double or_normal(uint64_t seed, uint32_t stream, uint64_t idx, uint32_t sub)
{
    uint32_t o[4];
    draw(seed, stream, idx, sub, o);
    double u1 = 1.0 - u53(o[0], o[1]); /* (0,1] */
    double u2 = u53(o[2], o[3]);       /* [0,1) */
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

/* ------------------------------------------------------------------------- */
/* dist64                                                    */
/* ------------------------------------------------------------------------- */
double or_dist64(const float *a, const float *b, int64_t n)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) {
        double d = (double)a[i] - (double)b[i];
        s = fma(d, d, s);
    }
    return s;
}

/* ------------------------------------------------------------------------- */
/* Bounded sample without replacement ("bounded random sample ... of    */
/* size min(0.1N, 10^5)").  Uniform without replacement realised as:  */
/* every row i gets the 64-bit Philox key of counter i; the sample is the n   */
/* rows of smallest (key, i), returned in ascending row order.                */
/* ------------------------------------------------------------------------- */
typedef struct { uint64_t key; int64_t idx; } keyidx;

static int cmp_keyidx(const void *a, const void *b)
{
    const keyidx *x = (const keyidx *)a, *y = (const keyidx *)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}
static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return x < y ? -1 : (x > y);
}

void or_sample_rows(int64_t N, int64_t n, uint64_t seed, uint32_t stream, int64_t *out)
{
    keyidx *t = (keyidx *)malloc(sizeof(keyidx) * (size_t)(N > 0 ? N : 1));
    for (int64_t i = 0; i < N; i++) {
        uint32_t o[4];
        draw(seed, stream, (uint64_t)i, 0, o);
        t[i].key = ((uint64_t)o[0] << 32) | o[1];
        t[i].idx = i;
    }
    qsort(t, (size_t)N, sizeof(keyidx), cmp_keyidx);
    for (int64_t i = 0; i < n; i++) out[i] = t[i].idx;
    qsort(out, (size_t)n, sizeof(int64_t), cmp_i64);
    free(t);
}

/* n = ceil(min(0.1 N, 1e5)), all rows when N <= 10 (Z16) */
int64_t or_cev_sample_size(int64_t N)
{
    if (N <= 10) return N;
    int64_t n = (N + 9) / 10;
    return n < 100000 ? n : 100000;
}

/* ------------------------------------------------------------------------- */
/* Spectral correlation check: covariance of the sample (divisor */
/* n-1), symmetric eigenvalues, CEV = sum of top floor(0.2 D) / sum.  */
/* ------------------------------------------------------------------------- */
void or_covariance(const float *X, int64_t ld, const int64_t *rows, int64_t n, int32_t D, double *C)
{
    double *mu = (double *)calloc((size_t)D, sizeof(double));
    for (int32_t i = 0; i < D; i++) {
        double s = 0.0;
        for (int64_t r = 0; r < n; r++) s += (double)X[rows[r] * ld + i];
        mu[i] = s / (double)n;
    }
    /* C_ij = sum_r fma(d_ri, d_rj, .) over r ascending, d = x - mu (divisor n-1).
     * Rows are visited in blocks (r still ascending for every output) so each
     * block stays in cache; threads own disjoint output rows i. */
    for (int64_t e = 0; e < (int64_t)D * D; e++) C[e] = 0.0;
    const int64_t RB = 64;
    double *dblk = (double *)malloc(sizeof(double) * (size_t)RB * D);
    for (int64_t r0 = 0; r0 < n; r0 += RB) {
        int64_t rn = n - r0 < RB ? n - r0 : RB;
        for (int64_t r = 0; r < rn; r++)
            for (int32_t i = 0; i < D; i++) dblk[r * D + i] = (double)X[rows[r0 + r] * ld + i] - mu[i];
#pragma omp parallel for schedule(dynamic, 8)
        for (int32_t i = 0; i < D; i++) {
            double *ci = C + (int64_t)i * D;
            for (int64_t r = 0; r < rn; r++) {
                const double *dr = dblk + r * D;
                double di = dr[i];
                for (int32_t j = 0; j <= i; j++) ci[j] = fma(di, dr[j], ci[j]);
            }
        }
    }
    for (int32_t i = 0; i < D; i++)
        for (int32_t j = 0; j <= i; j++) {
            double v = C[(int64_t)i * D + j] / (double)(n - 1);
            C[(int64_t)i * D + j] = v;
            C[(int64_t)j * D + i] = v;
        }
    free(dblk);
    free(mu);
}

/* Cyclic Jacobi eigenvalue iteration for a symmetric D x D matrix (in place).
 * Eigenvalues are left on the diagonal and copied to w (unsorted). */
void or_eig_sym_jacobi(double *A, int32_t D, double *w)
{
    for (int sweep = 0; sweep < 100; sweep++) {
        double off = 0.0, tot = 0.0;
        for (int32_t p = 0; p < D; p++)
            for (int32_t q = 0; q < D; q++) {
                double a = A[(int64_t)p * D + q];
                tot += a * a;
                if (p != q) off += a * a;
            }
        if (off <= 1e-30 * tot || off == 0.0) break;
        for (int32_t p = 0; p < D - 1; p++) {
            for (int32_t q = p + 1; q < D; q++) {
                double apq = A[(int64_t)p * D + q];
                if (apq == 0.0) continue;
                double app = A[(int64_t)p * D + p], aqq = A[(int64_t)q * D + q];
                double theta = (aqq - app) / (2.0 * apq);
                double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int32_t r = 0; r < D; r++) {
                    double arp = A[(int64_t)r * D + p], arq = A[(int64_t)r * D + q];
                    A[(int64_t)r * D + p] = c * arp - s * arq;
                    A[(int64_t)r * D + q] = s * arp + c * arq;
                }
                for (int32_t r = 0; r < D; r++) {
                    double apr = A[(int64_t)p * D + r], aqr = A[(int64_t)q * D + r];
                    A[(int64_t)p * D + r] = c * apr - s * aqr;
                    A[(int64_t)q * D + r] = s * apr + c * aqr;
                }
                A[(int64_t)p * D + q] = 0.0;
                A[(int64_t)q * D + p] = 0.0;
            }
        }
    }
    for (int32_t i = 0; i < D; i++) w[i] = A[(int64_t)i * D + i];
}

static int cmp_desc_double(const void *a, const void *b)
{
    double x = *(const double *)a, y = *(const double *)b;
    return x > y ? -1 : (x < y);
}

/* CEV from eigenvalues: sort descending, clamp negatives to 0
 * (S:L127), k = floor(0.2 D) (at least 1), total < 1e-12 -> 0. */
double or_cev_from_eigs(double *w, int32_t D)
{
    qsort(w, (size_t)D, sizeof(double), cmp_desc_double);
    int32_t kk = D / 5;
    if (kk < 1) kk = 1;
    double top = 0.0, tot = 0.0;
    for (int32_t i = 0; i < D; i++) {
        double l = w[i] > 0.0 ? w[i] : 0.0;
        tot += l;
        if (i < kk) top += l;
    }
    if (tot < 1e-12) return 0.0;
    return top / tot;
}

/* Full spectral check on the first D columns of X (row pitch ld). */
double or_cev(const float *X, int64_t N, int64_t ld, int32_t D, uint64_t seed)
{
    int64_t n = or_cev_sample_size(N);
    if (n < 2) return 0.0;
    int64_t *rows = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    or_sample_rows(N, n, seed, OR_STREAM_CEV_SAMPLE, rows);
    double *C = (double *)malloc(sizeof(double) * (size_t)D * (size_t)D);
    double *w = (double *)malloc(sizeof(double) * (size_t)D);
    or_covariance(X, ld, rows, n, D, C);
    or_eig_sym_jacobi(C, D, w);
    double cev = or_cev_from_eigs(w, D);
    free(rows); free(C); free(w);
    return cev;
}

/* ------------------------------------------------------------------------- */
/* Randomized orthogonal rotation: G_ij ~ N(0,1), G = Q R', R <- Q,   */
/* with diag(R') > 0.  Householder QR in fp64.                        */
/* G[i][j] = normal(seed, ROTATION, i*D + j).                                  */
/* ------------------------------------------------------------------------- */
void or_gaussian_matrix(int32_t D, uint64_t seed, double *G)
{
    for (int64_t e = 0; e < (int64_t)D * D; e++) G[e] = or_normal(seed, OR_STREAM_ROTATION, (uint64_t)e, 0);
}

/* Householder QR of A (D x D row-major, overwritten).  Q (D x D) returned with
 * columns sign-fixed so that R' has a positive diagonal.  Rdiag gets diag(R')
 * after the sign fix (all >= 0). */
void or_qr_householder(double *A, int32_t D, double *Qout, double *Rdiag)
{
    double *V = (double *)calloc((size_t)D * D, sizeof(double)); /* column k holds v_k */
    double *beta = (double *)calloc((size_t)D, sizeof(double));
    double *diag = (double *)calloc((size_t)D, sizeof(double));
    for (int32_t k = 0; k < D; k++) {
        double nrm = 0.0;
        for (int32_t i = k; i < D; i++) nrm = fma(A[(int64_t)i * D + k], A[(int64_t)i * D + k], nrm);
        nrm = sqrt(nrm);
        double x0 = A[(int64_t)k * D + k];
        double alpha = (x0 >= 0.0) ? -nrm : nrm; /* reflect x onto alpha e1 */
        /* v = x - alpha e1 */
        double vnorm2 = 0.0;
        for (int32_t i = k; i < D; i++) {
            double v = A[(int64_t)i * D + k] - (i == k ? alpha : 0.0);
            V[(int64_t)i * D + k] = v;
            vnorm2 = fma(v, v, vnorm2);
        }
        diag[k] = alpha;
        if (vnorm2 == 0.0) { beta[k] = 0.0; continue; }
        beta[k] = 2.0 / vnorm2;
        /* A[k:, j] -= beta v (v^T A[k:, j]) for j >= k */
        for (int32_t j = k; j < D; j++) {
            double s = 0.0;
            for (int32_t i = k; i < D; i++) s = fma(V[(int64_t)i * D + k], A[(int64_t)i * D + j], s);
            s *= beta[k];
            for (int32_t i = k; i < D; i++) A[(int64_t)i * D + j] -= s * V[(int64_t)i * D + k];
        }
    }
    /* Q = H_0 H_1 ... H_{D-1} : backward accumulation on the identity */
    for (int64_t e = 0; e < (int64_t)D * D; e++) Qout[e] = 0.0;
    for (int32_t i = 0; i < D; i++) Qout[(int64_t)i * D + i] = 1.0;
    for (int32_t k = D - 1; k >= 0; k--) {
        if (beta[k] == 0.0) continue;
        for (int32_t j = 0; j < D; j++) {
            double s = 0.0;
            for (int32_t i = k; i < D; i++) s = fma(V[(int64_t)i * D + k], Qout[(int64_t)i * D + j], s);
            s *= beta[k];
            for (int32_t i = k; i < D; i++) Qout[(int64_t)i * D + j] -= s * V[(int64_t)i * D + k];
        }
    }
    /* sign fix: column k of Q times sign(R'_kk) so that diag(R') > 0 */
    for (int32_t k = 0; k < D; k++) {
        double sg = diag[k] < 0.0 ? -1.0 : 1.0;
        if (sg < 0.0)
            for (int32_t i = 0; i < D; i++) Qout[(int64_t)i * D + k] = -Qout[(int64_t)i * D + k];
        Rdiag[k] = fabs(diag[k]);
    }
    free(V); free(beta); free(diag);
}

/* R (fp32, D x D row-major) = fl32(Q) of the sign-fixed QR of G(seed). */
void or_rotation(int32_t D, uint64_t seed, float *R32, double *R64_or_null)
{
    double *G = (double *)malloc(sizeof(double) * (size_t)D * D);
    double *Q = (double *)malloc(sizeof(double) * (size_t)D * D);
    double *rd = (double *)malloc(sizeof(double) * (size_t)D);
    or_gaussian_matrix(D, seed, G);
    or_qr_householder(G, D, Q, rd);
    for (int64_t e = 0; e < (int64_t)D * D; e++) {
        R32[e] = (float)Q[e];
        if (R64_or_null) R64_or_null[e] = Q[e];
    }
    free(G); free(Q); free(rd);
}

/* x' = fl32(x R), each output an fp64 fma chain over i ascending (P:L271
 * "X' = XR"; P:L283 row-by-row with a D-float buffer; Z14). In = out allowed. */
void or_rotate_rows(const float *X, int64_t n, int32_t D, int64_t ld, const float *R, float *Y, int64_t ldy)
{
#pragma omp parallel
    {
        double *acc = (double *)malloc(sizeof(double) * (size_t)D); /* the D-entry buffer of P:L283 */
#pragma omp for schedule(static)
        for (int64_t r = 0; r < n; r++) {
            const float *x = X + r * ld;
            for (int32_t j = 0; j < D; j++) acc[j] = 0.0;
            /* every output j accumulates fma(x_i, R_ij, .) with i ascending */
            for (int32_t i = 0; i < D; i++) {
                double xi = (double)x[i];
                const float *Ri = R + (int64_t)i * D;
                for (int32_t j = 0; j < D; j++) acc[j] = fma(xi, (double)Ri[j], acc[j]);
            }
            for (int32_t j = 0; j < D; j++) Y[r * ldy + j] = (float)acc[j];
        }
        free(acc);
    }
}

/* ------------------------------------------------------------------------- */
/* k-means per half-subspace ("learning a codebook of K centroids per  */
/* half via k-means"; K=50 P:L363).  Details are SPEC's:     */
/* k-means++ init, Lloyd iterations with early stop when no assignment        */
/* changes, empty clusters re-seeded from the farthest point, ties to lowest  */
/* centroid id.                                                               */
/* pts: n rows of dh floats (pitch ldp).  C: K x dh output.  obj (optional):  */
/* objective after each assignment step, length iters (unused entries = -1).  */
/* ------------------------------------------------------------------------- */
int32_t or_argmin_centroid(const float *x, const float *C, int32_t K, int32_t dh, double *dmin)
{
    int32_t best = 0;
    double bd = or_dist64(x, C, dh);
    for (int32_t c = 1; c < K; c++) {
        double d = or_dist64(x, C + (int64_t)c * dh, dh);
        if (d < bd) { bd = d; best = c; }
    }
    if (dmin) *dmin = bd;
    return best;
}

/* Half-subspace h covers dims [hoff[h], hoff[h+1]) of the stored vectors.
 * Equal widths: hoff[h] = h*dh (hoff == NULL).  Adaptive subspace
 * decomposition (reading R18): any even widths w_m = hoff[2m+2] -
 * hoff[2m] with equal halves; codebook rows keep the stride dh = max half
 * width, zero beyond the half's own width. */
static int64_t half_off(const int32_t *hoff, int32_t h, int32_t dh) { return hoff ? hoff[h] : (int64_t)h * dh; }
static int32_t half_w(const int32_t *hoff, int32_t h, int32_t dh) { return hoff ? hoff[h + 1] - hoff[h] : dh; }

/* nearest of K centroids (rows of `stride` floats, first w used) by (dist64, c) */
static int32_t argmin_centroid_w(const float *x, const float *C, int32_t K, int32_t w, int32_t stride)
{
    int32_t best = 0;
    double bd = or_dist64(x, C, w);
    for (int32_t c = 1; c < K; c++) {
        double d = or_dist64(x, C + (int64_t)c * stride, w);
        if (d < bd) { bd = d; best = c; }
    }
    return best;
}

void or_kmeans(const float *pts, int64_t n, int64_t ldp, int32_t dh, int32_t K, int32_t iters,
               uint64_t seed, uint32_t half, float *C, double *obj)
{
    double *D2 = (double *)malloc(sizeof(double) * (size_t)n);
    int32_t *a = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t *aold = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    double *dmin = (double *)malloc(sizeof(double) * (size_t)n);
    double *sum = (double *)malloc(sizeof(double) * (size_t)dh);
    unsigned char *taken = (unsigned char *)calloc((size_t)n, 1);
    if (obj) for (int32_t i = 0; i < iters; i++) obj[i] = -1.0;

    /* k-means++ seeding */
    {
        double u = or_uniform(seed, OR_STREAM_KM_INIT, 0, half);
        int64_t p0 = (int64_t)(u * (double)n);
        if (p0 >= n) p0 = n - 1;
        memcpy(C, pts + p0 * ldp, sizeof(float) * (size_t)dh);
        for (int64_t p = 0; p < n; p++) D2[p] = or_dist64(pts + p * ldp, C, dh);
        for (int32_t c = 1; c < K; c++) {
            double tot = 0.0;
            for (int64_t p = 0; p < n; p++) tot += D2[p];
            double uc = or_uniform(seed, OR_STREAM_KM_INIT, (uint64_t)c, half);
            int64_t pick;
            if (tot > 0.0) {
                double target = uc * tot, cum = 0.0;
                pick = -1;
                int64_t lastpos = 0;
                for (int64_t p = 0; p < n; p++) {
                    if (D2[p] > 0.0) lastpos = p;
                    cum += D2[p];
                    if (cum > target) { pick = p; break; }
                }
                if (pick < 0) pick = lastpos;
            } else {
                pick = (int64_t)(uc * (double)n);
                if (pick >= n) pick = n - 1;
            }
            float *cc = C + (int64_t)c * dh;
            memcpy(cc, pts + pick * ldp, sizeof(float) * (size_t)dh);
            for (int64_t p = 0; p < n; p++) {
                double d = or_dist64(pts + p * ldp, cc, dh);
                if (d < D2[p]) D2[p] = d;
            }
        }
    }
    /* Lloyd */
    for (int32_t it = 0; it < iters; it++) {
        double o = 0.0;
        for (int64_t p = 0; p < n; p++) {
            a[p] = or_argmin_centroid(pts + p * ldp, C, K, dh, &dmin[p]);
            o += dmin[p];
        }
        if (obj) obj[it] = o;
        if (it > 0) {
            int same = 1;
            for (int64_t p = 0; p < n; p++) if (a[p] != aold[p]) { same = 0; break; }
            if (same) break;
        }
        memset(taken, 0, (size_t)n);
        for (int32_t c = 0; c < K; c++) {
            int64_t cnt = 0;
            for (int32_t t = 0; t < dh; t++) sum[t] = 0.0;
            for (int64_t p = 0; p < n; p++) {
                if (a[p] != c) continue;
                cnt++;
                for (int32_t t = 0; t < dh; t++) sum[t] += (double)pts[p * ldp + t];
            }
            float *cc = C + (int64_t)c * dh;
            if (cnt > 0) {
                for (int32_t t = 0; t < dh; t++) cc[t] = (float)(sum[t] / (double)cnt);
            } else {
                /* re-seed from the point farthest from its centroid */
                int64_t best = -1;
                double bd = -1.0;
                for (int64_t p = 0; p < n; p++)
                    if (!taken[p] && dmin[p] > bd) { bd = dmin[p]; best = p; }
                if (best < 0) best = 0;
                taken[best] = 1;
                memcpy(cc, pts + best * ldp, sizeof(float) * (size_t)dh);
            }
        }
        memcpy(aold, a, sizeof(int32_t) * (size_t)n);
    }
    free(D2); free(a); free(aold); free(dmin); free(sum); free(taken);
}

/* Codebooks for all 2M halves from the k-means sample (min(N, 1e5)
 * rows, drawn with stream KM_SAMPLE).  Layout cb[((m*2+side)*K + c)*dh + t].
 * Subspace m covers dims [m*2dh, (m+1)*2dh); left = first dh, right = next dh
 * (Z17 for padding); with hoff (R18) half h covers [hoff[h], hoff[h+1])
 * and its centroids fill the first hoff[h+1]-hoff[h] floats of their rows. */
void or_train_codebooks(const float *X, int64_t N, int64_t ld, int32_t M, int32_t K, int32_t dh,
                        int32_t iters, int64_t sample, uint64_t seed, const int32_t *hoff, float *cb)
{
    int64_t n = sample < N ? sample : N;
    int64_t *rows = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    or_sample_rows(N, n, seed, OR_STREAM_KM_SAMPLE, rows);
#pragma omp parallel for schedule(dynamic)
    for (int32_t h = 0; h < 2 * M; h++) {
        const int32_t w = half_w(hoff, h, dh);
        const int64_t o = half_off(hoff, h, dh);
        float *pts = (float *)malloc(sizeof(float) * (size_t)n * w);
        float *Cw = (float *)malloc(sizeof(float) * (size_t)K * w);
        for (int64_t r = 0; r < n; r++)
            memcpy(pts + r * w, X + rows[r] * ld + o, sizeof(float) * (size_t)w);
        or_kmeans(pts, n, w, w, K, iters, seed, (uint32_t)h, Cw, NULL);
        float *ch = cb + (int64_t)h * K * dh;
        for (int32_t c = 0; c < K; c++)
            for (int32_t t = 0; t < dh; t++) ch[(int64_t)c * dh + t] = t < w ? Cw[(int64_t)c * w + t] : 0.0f;
        free(pts); free(Cw);
    }
    free(rows);
}

/* ------------------------------------------------------------------------- */
/* Cell assignment: cell_m(x) = i*K + j, i/j = nearest   */
/* left/right centroid by (dist64, c).  cells: M x N (row m contiguous).      */
/* ------------------------------------------------------------------------- */
void or_assign(const float *X, int64_t N, int64_t ld, int32_t M, int32_t K, int32_t dh,
               const int32_t *hoff, const float *cb, int32_t *cells)
{
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < N; p++) {
        for (int32_t m = 0; m < M; m++) {
            const int32_t hl = 2 * m, hr = 2 * m + 1;
            int32_t i = argmin_centroid_w(X + p * ld + half_off(hoff, hl, dh), cb + ((int64_t)hl * K) * dh, K,
                                          half_w(hoff, hl, dh), dh);
            int32_t j = argmin_centroid_w(X + p * ld + half_off(hoff, hr, dh), cb + ((int64_t)hr * K) * dh, K,
                                          half_w(hoff, hr, dh), dh);
            cells[(int64_t)m * N + p] = i * K + j;
        }
    }
}

/* CSR: per subspace, ids sorted by cell (counting sort, ids     */
/* ascending inside a cell, Z18); off has K^2+1 entries, off[0]=0, off[K^2]=N.*/
void or_csr(const int32_t *cells, int64_t N, int32_t M, int32_t K, int64_t *off, int32_t *ids)
{
    int64_t KK = (int64_t)K * K;
    for (int32_t m = 0; m < M; m++) {
        int64_t *o = off + (int64_t)m * (KK + 1);
        for (int64_t c = 0; c <= KK; c++) o[c] = 0;
        for (int64_t p = 0; p < N; p++) o[cells[(int64_t)m * N + p] + 1]++;
        for (int64_t c = 0; c < KK; c++) o[c + 1] += o[c];
        int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)KK);
        memcpy(cur, o, sizeof(int64_t) * (size_t)KK);
        for (int64_t p = 0; p < N; p++) {
            int32_t c = cells[(int64_t)m * N + p];
            ids[(int64_t)m * N + cur[c]++] = (int32_t)p;
        }
        free(cur);
    }
}

/* Binary codes: bit (i mod 64) of word i/64 is [x_i > 0] (Z10). */
void or_codes(const float *X, int64_t N, int64_t ld, int32_t D, uint64_t *codes)
{
    int32_t W = (D + 63) / 64;
    for (int64_t p = 0; p < N; p++) {
        for (int32_t w = 0; w < W; w++) codes[p * W + w] = 0;
        for (int32_t i = 0; i < D; i++)
            if (X[p * ld + i] > 0.0f) codes[p * W + i / 64] |= (uint64_t)1 << (i % 64);
    }
}

/* ------------------------------------------------------------------------- */
/* Search (Alg. 1).                                               */
/* ------------------------------------------------------------------------- */
typedef struct { double d; int64_t id; } dist_id;
typedef struct { double d; int32_t c; } dist_c;
typedef struct { double cost; int32_t i, j; } heap_ent;
typedef struct { int32_t h; int32_t id; } ham_id;

static int cmp_dist_c(const void *a, const void *b)
{
    const dist_c *x = (const dist_c *)a, *y = (const dist_c *)b;
    if (x->d != y->d) return x->d < y->d ? -1 : 1;
    return x->c < y->c ? -1 : (x->c > y->c);
}
static int less_dist_id(dist_id x, dist_id y) { return x.d < y.d || (x.d == y.d && x.id < y.id); }
static int cmp_dist_id(const void *a, const void *b)
{
    dist_id x = *(const dist_id *)a, y = *(const dist_id *)b;
    return less_dist_id(x, y) ? -1 : (less_dist_id(y, x) ? 1 : 0);
}
static int cmp_ham_id(const void *a, const void *b)
{
    const ham_id *x = (const ham_id *)a, *y = (const ham_id *)b;
    if (x->h != y->h) return x->h < y->h ? -1 : 1;
    return x->id < y->id ? -1 : (x->id > y->id);
}
static int heap_less(heap_ent x, heap_ent y)
{
    if (x.cost != y.cost) return x.cost < y.cost;
    if (x.i != y.i) return x.i < y.i;
    return x.j < y.j;
}
static void heap_push(heap_ent *h, int32_t *n, heap_ent e)
{
    int32_t i = (*n)++;
    h[i] = e;
    while (i > 0) {
        int32_t p = (i - 1) / 2;
        if (!heap_less(h[i], h[p])) break;
        heap_ent t = h[i]; h[i] = h[p]; h[p] = t; i = p;
    }
}
static heap_ent heap_pop(heap_ent *h, int32_t *n)
{
    heap_ent top = h[0];
    h[0] = h[--(*n)];
    int32_t i = 0;
    for (;;) {
        int32_t l = 2 * i + 1, r = l + 1, s = i;
        if (l < *n && heap_less(h[l], h[s])) s = l;
        if (r < *n && heap_less(h[r], h[s])) s = r;
        if (s == i) break;
        heap_ent t = h[i]; h[i] = h[s]; h[s] = t; i = s;
    }
    return top;
}

void or_half_sorted_w(const float *qh, const float *Ch, int32_t K, int32_t w, int32_t stride, double *dist,
                      int32_t *perm);
/* Sorted partial distances of one half (Alg. 1 line 4; Z4). */
void or_half_sorted(const float *qh, const float *Ch, int32_t K, int32_t dh, double *dist, int32_t *perm)
{
    or_half_sorted_w(qh, Ch, K, dh, dh, dist, perm);
}

/* the same over the first w floats of centroid rows of `stride` floats (R18) */
void or_half_sorted_w(const float *qh, const float *Ch, int32_t K, int32_t w, int32_t stride, double *dist,
                      int32_t *perm)
{
    dist_c *t = (dist_c *)malloc(sizeof(dist_c) * (size_t)K);
    for (int32_t c = 0; c < K; c++) { t[c].d = or_dist64(qh, Ch + (int64_t)c * stride, w); t[c].c = c; }
    qsort(t, (size_t)K, sizeof(dist_c), cmp_dist_c);
    for (int32_t r = 0; r < K; r++) { dist[r] = t[r].d; perm[r] = t[r].c; }
    free(t);
}

/* Multi-Sequence traversal of one subspace with a real priority queue and a
 * visited set (Alg. 1 lines 5-17).  Emits the activated cells
 * in pop order with their weights; returns the number popped.  gsize: K^2 cell
 * sizes used for the budget (global sizes for sharded indexes, Z23). */
int32_t or_multisequence(const double *a, const int32_t *pa, const double *b, const int32_t *pb,
                         int32_t K, const int64_t *gsize, int64_t budget, int32_t wmode_k,
                         int32_t *out_cell, int32_t *out_w, int64_t *out_retrieved)
{
    int64_t KK = (int64_t)K * K;
    heap_ent *h = (heap_ent *)malloc(sizeof(heap_ent) * (size_t)(KK + 1));
    unsigned char *vis = (unsigned char *)calloc((size_t)KK, 1);
    int32_t hn = 0, rank = 0;
    int64_t retrieved = 0;
    heap_ent e0 = {a[0] + b[0], 0, 0};
    heap_push(h, &hn, e0);
    vis[0] = 1;
    while (retrieved < budget && hn > 0) {
        heap_ent e = heap_pop(h, &hn);
        int32_t cell = pa[e.i] * K + pb[e.j];
        rank++;
        int32_t w = (wmode_k > 0 && rank <= wmode_k) ? 2 : 1; /* Alg. 1 lines 10-12 */
        out_cell[rank - 1] = cell;
        out_w[rank - 1] = w;
        retrieved += gsize[cell];
        if (e.i + 1 < K && !vis[(int64_t)(e.i + 1) * K + e.j]) {
            vis[(int64_t)(e.i + 1) * K + e.j] = 1;
            heap_ent n1 = {a[e.i + 1] + b[e.j], e.i + 1, e.j};
            heap_push(h, &hn, n1);
        }
        if (e.j + 1 < K && !vis[(int64_t)e.i * K + e.j + 1]) {
            vis[(int64_t)e.i * K + e.j + 1] = 1;
            heap_ent n2 = {a[e.i] + b[e.j + 1], e.i, e.j + 1};
            heap_push(h, &hn, n2);
        }
    }
    free(h); free(vis);
    if (out_retrieved) *out_retrieved = retrieved;
    return rank;
}

typedef struct {
    /* index */
    int64_t N;            /* local points */
    int64_t gid_base;     /* global id of local point 0 (shards) */
    int32_t D;            /* stored (padded) dimensionality Dp, = 2*M*dh */
    int32_t M, K, dh;     /* dh: codebook row stride = the (largest) half width */
    const int32_t *hoff;  /* 2M+1 half offsets (R18), NULL = equal halves of dh */
    const float *X;       /* N x D stored (rotated if applicable) */
    const float *R;       /* D x D or NULL */
    const float *cb;      /* M x 2 x K x dh */
    const int64_t *off;   /* M x (K^2+1) */
    const int32_t *ids;   /* M x N */
    const uint64_t *codes;/* N x ceil(D/64) */
    const int64_t *gsize; /* M x K^2 (budget sizes) */
    /* search parameters */
    int64_t budget;       /* B ids per subspace (exact integer, O1) */
    int32_t tau;          /* integer threshold (exact, O1) */
    int32_t patience;     /* P = factor*k, 0 = disabled */
    int32_t ad_on;        /* phi=1 verification by ADSampling (Eq. 2) */
    double ad_eps0;       /* its safety margin epsilon_0 (2.1) */
    int32_t ad_stride;    /* checks every ad_stride dimensions (32) */
    int32_t fb_mode;      /* 0: underflow fallback; 1: none (sharded protocol, first phase) */
    const int32_t *ext_cand; /* Q x N external candidate lists (ascending local ids) or NULL */
    const int64_t *ext_n;    /* Q: length of the external list, < 0 = compute C normally */
} or_index;

typedef struct {
    int32_t *act_len;     /* Q x M                 (or NULL) */
    int32_t *act_cell;    /* Q x M x K^2 pop order (or NULL) */
    int32_t *act_w;       /* Q x M x K^2           (or NULL) */
    int64_t *retrieved;   /* Q x M                 (or NULL) */
    uint16_t *V;          /* Q x N                 (or NULL) */
    int64_t *cand_n;      /* Q                     (or NULL) */
    int32_t *cand;        /* Q x N local ids, ascending (or NULL) */
    int32_t *order;       /* Q x N local ids in verification order (or NULL) */
    int64_t *n_verified;  /* Q                     (or NULL) */
    int32_t *fallback;    /* Q flag                (or NULL) */
    float *qrot;          /* Q x D rotated query   (or NULL) */
} or_trace;

/* ADSampling (Eq. 2; SPEC adsampling_verify): the pruning
 * threshold r_k^2 * (t/D) * (1 + eps0/sqrt(t))^2, evaluated in this order. */
double or_adsampling_threshold(double rk2, int32_t t, int32_t D, double eps0)
{
    const double f = 1.0 + eps0 / sqrt((double)t);
    return ((rk2 * (double)t) / (double)D) * (f * f);
}

/* Accumulate (q_i - x_i)^2 in dimension order (the dist64 chain); at every
 * multiple t of stride with t < D, prune if the partial sum exceeds the
 * threshold.  Returns 1 (pruned, *out = the partial sum at the pruning t) or
 * 0 (*out = the exact dist64).  rk2 = +inf never prunes.  A check at t = D is
 * not made: it could only prune a candidate whose exact distance exceeds r_k,
 * which is non-improving either way. */
int32_t or_adsampling_verify(const float *q, const float *x, int32_t D, double rk2, double eps0, int32_t stride,
                             double *out)
{
    double s = 0.0;
    for (int32_t i = 0; i < D; i++) {
        double d = (double)q[i] - (double)x[i];
        s = fma(d, d, s);
        const int32_t t = i + 1;
        if (stride > 0 && t % stride == 0 && t < D && s > or_adsampling_threshold(rk2, t, D, eps0)) {
            *out = s;
            return 1;
        }
    }
    *out = s;
    return 0;
}

static void search_one(const or_index *ix, const float *q_in, int32_t k, int32_t mode,
                       int64_t qi, int64_t *out_id, double *out_d, const or_trace *tr)
{
    const int32_t D = ix->D, M = ix->M, K = ix->K, dh = ix->dh;
    const int64_t N = ix->N, KK = (int64_t)K * K;
    float *q = (float *)malloc(sizeof(float) * (size_t)D);
    /* a0: q' = q R when the index is rotated, fp64 chain -> fp32 */
    if (ix->R) {
        for (int32_t j = 0; j < D; j++) {
            double s = 0.0;
            for (int32_t i = 0; i < D; i++) s = fma((double)q_in[i], (double)ix->R[(int64_t)i * D + j], s);
            q[j] = (float)s;
        }
    } else {
        memcpy(q, q_in, sizeof(float) * (size_t)D);
    }
    if (tr && tr->qrot) memcpy(tr->qrot + qi * D, q, sizeof(float) * (size_t)D);

    uint16_t *V = (uint16_t *)calloc((size_t)(N > 0 ? N : 1), sizeof(uint16_t)); /* Alg. 1 line 1 */
    double *a = (double *)malloc(sizeof(double) * (size_t)K), *b = (double *)malloc(sizeof(double) * (size_t)K);
    int32_t *pa = (int32_t *)malloc(sizeof(int32_t) * (size_t)K), *pb = (int32_t *)malloc(sizeof(int32_t) * (size_t)K);
    int32_t *cl = (int32_t *)malloc(sizeof(int32_t) * (size_t)KK), *wl = (int32_t *)malloc(sizeof(int32_t) * (size_t)KK);
    int32_t wk = (mode == 1) ? k : 0;
    for (int32_t m = 0; m < M; m++) {
        /* a1: Dist(q_left, C_left), Dist(q_right, C_right), sorted (Alg. 1 l.3-4) */
        or_half_sorted_w(q + half_off(ix->hoff, 2 * m, dh), ix->cb + ((int64_t)(m * 2 + 0) * K) * dh, K,
                         half_w(ix->hoff, 2 * m, dh), dh, a, pa);
        or_half_sorted_w(q + half_off(ix->hoff, 2 * m + 1, dh), ix->cb + ((int64_t)(m * 2 + 1) * K) * dh, K,
                         half_w(ix->hoff, 2 * m + 1, dh), dh, b, pb);
        /* a2: Multi-Sequence traversal under the budget (Alg. 1 l.5-17) */
        int64_t ret = 0;
        int32_t L = or_multisequence(a, pa, b, pb, K, ix->gsize + (int64_t)m * KK, ix->budget, wk, cl, wl, &ret);
        /* a3: V[id] += w over each activated cell's CSR slice (Alg. 1 l.13-16, Eq. 1) */
        for (int32_t r = 0; r < L; r++) {
            const int64_t *o = ix->off + (int64_t)m * (KK + 1);
            for (int64_t p = o[cl[r]]; p < o[cl[r] + 1]; p++) V[ix->ids[(int64_t)m * N + p]] += (uint16_t)wl[r];
        }
        if (tr && tr->act_len) tr->act_len[qi * M + m] = L;
        if (tr && tr->retrieved) tr->retrieved[qi * M + m] = ret;
        if (tr && tr->act_cell)
            for (int32_t r = 0; r < L; r++) {
                tr->act_cell[(qi * M + m) * KK + r] = cl[r];
                tr->act_w[(qi * M + m) * KK + r] = wl[r];
            }
    }
    if (tr && tr->V) memcpy(tr->V + qi * N, V, sizeof(uint16_t) * (size_t)N);

    /* a4: C = {x : V[x] >= tau} in ascending id (Alg. 1 l.18) */
    int32_t *C = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1));
    int64_t nc = 0;
    int32_t fb = 0;
    const int ext = ix->ext_n && ix->ext_n[qi] >= 0;
    if (ext) {  /* candidate set decided outside (sharded global fallback) */
        nc = ix->ext_n[qi];
        memcpy(C, ix->ext_cand + qi * N, sizeof(int32_t) * (size_t)nc);
    } else {
        for (int64_t x = 0; x < N; x++) if (V[x] >= ix->tau) C[nc++] = (int32_t)x;
    }
    if (!ext && ix->fb_mode == 0 && nc < k) {
        /* fallback (Z8): first min(k,|T|) touched ids by (V desc, id asc),
         * then restated in ascending id */
        fb = 1;
        nc = 0;
        for (int32_t v = 2 * M; v >= 1 && nc < k; v--)
            for (int64_t x = 0; x < N && nc < k; x++)
                if (V[x] == v) C[nc++] = (int32_t)x;
    }
    if (fb) {
        /* ascending id (simple insertion sort, nc <= k) */
        for (int64_t i = 1; i < nc; i++) {
            int32_t v = C[i];
            int64_t j = i - 1;
            while (j >= 0 && C[j] > v) { C[j + 1] = C[j]; j--; }
            C[j + 1] = v;
        }
    }
    if (tr && tr->fallback) tr->fallback[qi] = fb;
    if (tr && tr->cand_n) tr->cand_n[qi] = nc;
    if (tr && tr->cand) memcpy(tr->cand + qi * N, C, sizeof(int32_t) * (size_t)nc);

    dist_id *best = (dist_id *)malloc(sizeof(dist_id) * (size_t)(k + 1));
    int32_t nb = 0;
    int64_t nver = 0;
    if (mode == 0) {
        /* a5, Guaranteed Mode: exact L2 for every x in C, top-k by (d, id) */
        dist_id *all = (dist_id *)malloc(sizeof(dist_id) * (size_t)(nc > 0 ? nc : 1));
        for (int64_t i = 0; i < nc; i++) {
            all[i].d = or_dist64(q, ix->X + (int64_t)C[i] * D, D);
            all[i].id = ix->gid_base + C[i];
        }
        qsort(all, (size_t)nc, sizeof(dist_id), cmp_dist_id);
        nb = (int32_t)(nc < k ? nc : k);
        for (int32_t i = 0; i < nb; i++) best[i] = all[i];
        nver = nc;
        free(all);
        if (tr && tr->order) memcpy(tr->order + qi * N, C, sizeof(int32_t) * (size_t)nc);
    } else {
        /* a4 (phi=1): order C by Hamming distance (Z9: (h, id)) */
        int32_t W = (D + 63) / 64;
        uint64_t *qc = (uint64_t *)calloc((size_t)W, sizeof(uint64_t));
        for (int32_t i = 0; i < D; i++) if (q[i] > 0.0f) qc[i / 64] |= (uint64_t)1 << (i % 64);
        ham_id *hs = (ham_id *)malloc(sizeof(ham_id) * (size_t)(nc > 0 ? nc : 1));
        for (int64_t i = 0; i < nc; i++) {
            int32_t h = 0;
            for (int32_t w = 0; w < W; w++) h += __builtin_popcountll(qc[w] ^ ix->codes[(int64_t)C[i] * W + w]);
            hs[i].h = h; hs[i].id = C[i];
        }
        qsort(hs, (size_t)nc, sizeof(ham_id), cmp_ham_id);
        if (tr && tr->order) for (int64_t i = 0; i < nc; i++) tr->order[qi * N + i] = hs[i].id;
        /* a5 (phi=1): exact L2 in that order with patience (Z11, Z12),
         * or ADSampling (Eq. 2) when ad_on: r_k^2 = +inf until k results exist, and a
         * pruned candidate counts as a non-improving verification */
        int64_t cnt = 0;
        for (int64_t i = 0; i < nc; i++) {
            dist_id e;
            e.id = ix->gid_base + hs[i].id;
            nver++;
            if (ix->ad_on) {
                const double rk2 = nb < k ? INFINITY : best[nb - 1].d;
                if (or_adsampling_verify(q, ix->X + (int64_t)hs[i].id * D, D, rk2, ix->ad_eps0, ix->ad_stride,
                                         &e.d)) {
                    cnt++;
                    if (ix->patience > 0 && cnt == ix->patience) break;
                    continue;
                }
            } else {
                e.d = or_dist64(q, ix->X + (int64_t)hs[i].id * D, D);
            }
            if (nb < k || less_dist_id(e, best[nb - 1])) {
                /* insert into the sorted top-k, evicting the worst when full */
                int32_t pos = nb < k ? nb : k - 1;
                if (nb < k) nb++;
                while (pos > 0 && less_dist_id(e, best[pos - 1])) { best[pos] = best[pos - 1]; pos--; }
                best[pos] = e;
                cnt = 0;
            } else {
                cnt++;
            }
            if (ix->patience > 0 && cnt == ix->patience) break;
        }
        free(qc); free(hs);
    }
    if (tr && tr->n_verified) tr->n_verified[qi] = nver;
    /* O16: ascending (d, id), padded with (-1, +inf) (Z21) */
    for (int32_t i = 0; i < k; i++) {
        if (i < nb) { out_id[i] = best[i].id; out_d[i] = best[i].d; }
        else { out_id[i] = -1; out_d[i] = INFINITY; }
    }
    free(q); free(V); free(a); free(b); free(pa); free(pb); free(cl); free(wl); free(C); free(best);
}

void or_search(int64_t N, int64_t gid_base, int32_t D, int32_t M, int32_t K, int32_t dh, const int32_t *hoff,
               const float *X, const float *R, const float *cb, const int64_t *off, const int32_t *ids,
               const uint64_t *codes, const int64_t *gsize, int64_t budget, int32_t tau, int32_t patience,
               int32_t ad_on, double ad_eps0, int32_t ad_stride,
               int32_t fb_mode, const int32_t *ext_cand, const int64_t *ext_n,
               const float *queries, int64_t Q, int32_t k, int32_t mode, int32_t nthreads,
               int64_t *out_ids, double *out_d,
               int32_t *t_act_len, int32_t *t_act_cell, int32_t *t_act_w, int64_t *t_retrieved,
               uint16_t *t_V, int64_t *t_cand_n, int32_t *t_cand, int32_t *t_order, int64_t *t_nver,
               int32_t *t_fallback, float *t_qrot)
{
    or_index ix = {N, gid_base, D, M, K, dh, hoff, X, R, cb, off, ids, codes, gsize, budget, tau, patience,
                   ad_on, ad_eps0, ad_stride, fb_mode, ext_cand, ext_n};
    or_trace tr = {t_act_len, t_act_cell, t_act_w, t_retrieved, t_V, t_cand_n, t_cand, t_order, t_nver,
                   t_fallback, t_qrot};
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(dynamic)
    for (int64_t qi = 0; qi < Q; qi++)
        search_one(&ix, queries + qi * D, k, mode, qi, out_ids + qi * k, out_d + qi * k, &tr);
}

int32_t or_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------- */
/* Checkers used to pin the oracle (not part of the method).                  */
/* ------------------------------------------------------------------------- */

/* Exact kNN by brute force: first k by (dist64, id). */
void or_bruteforce_knn(const float *X, int64_t N, int32_t D, const float *Qv, int64_t Q, int32_t k,
                       int64_t *out_ids, double *out_d)
{
#pragma omp parallel for schedule(dynamic)
    for (int64_t qi = 0; qi < Q; qi++) {
        dist_id *all = (dist_id *)malloc(sizeof(dist_id) * (size_t)N);
        for (int64_t x = 0; x < N; x++) { all[x].d = or_dist64(Qv + qi * D, X + x * D, D); all[x].id = x; }
        qsort(all, (size_t)N, sizeof(dist_id), cmp_dist_id);
        for (int32_t i = 0; i < k; i++) {
            if (i < N) { out_ids[qi * k + i] = all[i].id; out_d[qi * k + i] = all[i].d; }
            else { out_ids[qi * k + i] = -1; out_d[qi * k + i] = INFINITY; }
        }
        free(all);
    }
}

/* Brute-force collision scores without CSR and without a heap:
 * A_qm = shortest prefix of ALL K^2 cells fully sorted by (a_i+b_j, i, j)
 * whose sizes (counted directly from cells[]) reach the budget; then
 * S(x) = sum_m w * [cell_m(x) in A_qm].  qrot: already-rotated queries. */
typedef struct { double cost; int32_t i, j; } cost_ij;
static int cmp_cost_ij(const void *a, const void *b)
{
    const cost_ij *x = (const cost_ij *)a, *y = (const cost_ij *)b;
    if (x->cost != y->cost) return x->cost < y->cost ? -1 : 1;
    if (x->i != y->i) return x->i < y->i ? -1 : 1;
    return x->j < y->j ? -1 : (x->j > y->j);
}
void or_bruteforce_scores(const int32_t *cells, int64_t N, int32_t D, int32_t M, int32_t K, int32_t dh,
                          const int32_t *hoff, const float *cb, const float *qrot, int64_t Q, int64_t budget, int32_t wk,
                          uint16_t *S)
{
    int64_t KK = (int64_t)K * K;
#pragma omp parallel for schedule(dynamic)
    for (int64_t qi = 0; qi < Q; qi++) {
        int64_t *size = (int64_t *)malloc(sizeof(int64_t) * (size_t)KK);
        int32_t *wcell = (int32_t *)malloc(sizeof(int32_t) * (size_t)KK);
        cost_ij *all = (cost_ij *)malloc(sizeof(cost_ij) * (size_t)KK);
        double *a = (double *)malloc(sizeof(double) * (size_t)K), *b = (double *)malloc(sizeof(double) * (size_t)K);
        int32_t *pa = (int32_t *)malloc(sizeof(int32_t) * (size_t)K), *pb = (int32_t *)malloc(sizeof(int32_t) * (size_t)K);
        for (int64_t x = 0; x < N; x++) S[qi * N + x] = 0;
        for (int32_t m = 0; m < M; m++) {
            const float *q = qrot + qi * D;
            for (int64_t c = 0; c < KK; c++) { size[c] = 0; wcell[c] = 0; }
            for (int64_t x = 0; x < N; x++) size[cells[(int64_t)m * N + x]]++;
            /* sorted halves by a plain selection sort on (dist64, c) */
            for (int32_t side = 0; side < 2; side++) {
                double *dd = side ? b : a;
                int32_t *pp = side ? pb : pa;
                const float *Ch = cb + ((int64_t)(m * 2 + side) * K) * dh;
                const int32_t h = 2 * m + side;
                for (int32_t c = 0; c < K; c++) {
                    dd[c] = or_dist64(q + half_off(hoff, h, dh), Ch + (int64_t)c * dh, half_w(hoff, h, dh));
                    pp[c] = c;
                }
                for (int32_t r = 0; r < K; r++) {
                    int32_t mi = r;
                    for (int32_t s = r + 1; s < K; s++)
                        if (dd[s] < dd[mi] || (dd[s] == dd[mi] && pp[s] < pp[mi])) mi = s;
                    double td = dd[r]; dd[r] = dd[mi]; dd[mi] = td;
                    int32_t tp = pp[r]; pp[r] = pp[mi]; pp[mi] = tp;
                }
            }
            for (int32_t i = 0; i < K; i++)
                for (int32_t j = 0; j < K; j++) { all[i * K + j].cost = a[i] + b[j]; all[i * K + j].i = i; all[i * K + j].j = j; }
            qsort(all, (size_t)KK, sizeof(cost_ij), cmp_cost_ij);
            int64_t got = 0;
            for (int64_t r = 0; r < KK && got < budget; r++) {
                int32_t cell = pa[all[r].i] * K + pb[all[r].j];
                wcell[cell] = (wk > 0 && r + 1 <= wk) ? 2 : 1;
                got += size[cell];
            }
            for (int64_t x = 0; x < N; x++) S[qi * N + x] += (uint16_t)wcell[cells[(int64_t)m * N + x]];
        }
        free(size); free(wcell); free(all); free(a); free(b); free(pa); free(pb);
    }
}

/* Merge of per-shard top-k lists by (d, gid) (Z23). */
void or_merge_topk(const double *d, const int64_t *ids, int32_t G, int64_t Q, int32_t k,
                   double *out_d, int64_t *out_ids)
{
    for (int64_t qi = 0; qi < Q; qi++) {
        dist_id *all = (dist_id *)malloc(sizeof(dist_id) * (size_t)G * k);
        int64_t n = 0;
        for (int32_t g = 0; g < G; g++)
            for (int32_t i = 0; i < k; i++) {
                int64_t id = ids[((int64_t)g * Q + qi) * k + i];
                if (id < 0) continue;
                all[n].d = d[((int64_t)g * Q + qi) * k + i];
                all[n].id = id;
                n++;
            }
        qsort(all, (size_t)n, sizeof(dist_id), cmp_dist_id);
        for (int32_t i = 0; i < k; i++) {
            if (i < n) { out_d[qi * k + i] = all[i].d; out_ids[qi * k + i] = all[i].id; }
            else { out_d[qi * k + i] = INFINITY; out_ids[qi * k + i] = -1; }
        }
        free(all);
    }
}

/* Theorem 1. */
double or_hoeffding_bound(int32_t M, double pstar, double tau)
{
    double mu = (double)M * pstar;
    if (!(mu > tau)) return NAN; /* vacuous */
    double t = mu - tau;
    return 1.0 - exp(-2.0 * t * t / (double)M);
}

/* P(S < tau), S ~ Binomial(M, p): exact summation. */
double or_binomial_failure(int32_t M, double p, int32_t tau)
{
    double tot = 0.0;
    for (int32_t s = 0; s < tau && s <= M; s++) {
        double lc = lgamma((double)M + 1) - lgamma((double)s + 1) - lgamma((double)(M - s) + 1);
        double term;
        if (p == 0.0) term = (s == 0) ? 1.0 : 0.0;
        else if (p == 1.0) term = (s == M) ? 1.0 : 0.0;
        else term = exp(lc + s * log(p) + (M - s) * log1p(-p));
        tot += term;
    }
    return tot;
}
