/*
 * oracle/rii_ref.c -- plain, slow, single-threaded CPU oracle for the hot path of
 * Rii (Reconfigurable Inverted Index; Matsui, Hinami, Satoh, ACM MM 2018,
 * arXiv 1808.03969).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` legs may load, call or execute this library.
 * The product path (paper_1808_03969_b200/) never imports or links it, and this
 * file shares no code, header, table or constant generator with that path.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC (see
 * oracle/build.sh).  x86-64 SSE arithmetic, no FMA contraction, so every float
 * operation below is one IEEE-754 binary32 (or binary64) round-to-nearest op.
 *
 * Citation keys: "P:n" = /root/reference/PAPER.md line n, with the section,
 * equation or algorithm named; "S:n" = SPEC.md line n; "R#" / "CA#" / "O-xxx" =
 * the readings listed in DESIGN.md section "Readings of the paper".
 *
 * Pins: every function here is checked by tests/test_oracle_*.py against
 * closed forms, invariants, brute force on tiny inputs and the paper's printed
 * memory figures.  Parity unpinned: the value of the
 * threshold theta (machine-dependent) -- only the rule
 * |S| < theta is pinned (via path_used).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* status codes (same numeric meaning as the product ABI, defined independently) */
#define REF_OK 0
#define REF_ERR_ARG 1
#define REF_ERR_STATE 2
#define REF_ERR_OOM 3
#define REF_ERR_TRAIN 6

#define REF_PATH_AUTO 0
#define REF_PATH_LINEAR 1
#define REF_PATH_IVF 2

/* ------------------------------------------------------------------------- */
/* Instrumentation (test infrastructure only): how many times the empty-cluster
 * re-seeding branches ran -- [0] code-book training (R8), [1] PQk-means
 * (R9) -- so that the pins can show those branches are exercised.  Reading
 * them changes nothing the oracle computes.  Not thread-safe (the oracle is
 * single-threaded per call; the counters are only read by serial pin tests). */
static int64_t g_reseeds[2];
int64_t rref_reseed_count(int which) { return which >= 0 && which < 2 ? g_reseeds[which] : -1; }
void rref_reseed_reset(void) { g_reseeds[0] = g_reseeds[1] = 0; }

/* ------------------------------------------------------------------------- */
/* Counter-based hash used for every seeded choice (R8, R10).                 */
/* splitmix64 finaliser (Steele, Lea, Flood 2014); a bijection on 64 bits.     */
uint64_t rref_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* ------------------------------------------------------------------------- */
/* CA1: squared Euclidean distance between a ds-dim sub-vector and a code word, */
/* t = u_j - c_j; acc = acc + t*t, j ascending, fp32 ("A(m,z) is the */
/* squared Euclidean distance between the mth part of q and zth code word").   */
static float ca1(const float *u, const float *c, int ds) {
    float acc = 0.0f;
    for (int j = 0; j < ds; ++j) {
        float t = u[j] - c[j];
        acc = acc + t * t;
    }
    return acc;
}

/* The same distance evaluated in fp64 from the fp32 inputs (CA3). */
static double ca1_64(const float *u, const float *c, int ds) {
    double acc = 0.0;
    for (int j = 0; j < ds; ++j) {
        double t = (double)u[j] - (double)c[j];
        acc = acc + t * t;
    }
    return acc;
}

/* Codebook layout: cb[(m*Z + z)*ds + j], D = M*ds  (Sec. 3). */

/* Eq. 1: x -> xbar, xbar^m = argmin_z || x_m - c_{m,z} ||^2,
 * ties to the lowest z (CA4 / S:72). */
int rref_encode(const float *cb, int D, int M, int Z, const float *x, int64_t n, uint8_t *codes) {
    if (M <= 0 || D % M != 0 || Z < 1 || Z > 256) return REF_ERR_ARG;
    int ds = D / M;
    for (int64_t i = 0; i < n; ++i) {
        for (int m = 0; m < M; ++m) {
            const float *u = x + i * D + m * ds;
            float best = INFINITY;
            int bz = 0;
            for (int z = 0; z < Z; ++z) {
                float d = ca1(u, cb + ((int64_t)m * Z + z) * ds, ds);
                if (d < best) { best = d; bz = z; }
            }
            codes[i * M + m] = (uint8_t)bz;
        }
    }
    return REF_OK;
}

/* Reconstruction: concatenation of the selected code words. */
void rref_decode(const float *cb, int D, int M, int Z, const uint8_t *codes, int64_t n, float *x) {
    int ds = D / M;
    for (int64_t i = 0; i < n; ++i)
        for (int m = 0; m < M; ++m)
            for (int j = 0; j < ds; ++j)
                x[i * D + m * ds + j] = cb[((int64_t)m * Z + codes[i * M + m]) * ds + j];
}

/* OPQ rotation (Rii-OPQ: "an input vector is first rotated with the
 * matrix.  The remaining process is exactly the same as PQ"): y = R x for n rows,
 * R row-major D x D.  Canonical order CR: y_i = ((0 + R_i0 x_0) +
 * R_i1 x_1) + ..., j ascending, one fp32 multiply and one fp32 add per term. */
void rref_rotate(const float *R, int D, const float *x, int64_t n, float *y) {
    for (int64_t v = 0; v < n; ++v)
        for (int i = 0; i < D; ++i) {
            float acc = 0.0f;
            for (int j = 0; j < D; ++j) {
                float t = R[(int64_t)i * D + j] * x[v * D + j];
                acc = acc + t;
            }
            y[v * D + i] = acc;
        }
}

/* Distance table A in R^{M x Z} (Alg. 1 L1 "CompareCodewords"). */
void rref_lut(const float *cb, int D, int M, int Z, const float *q, float *A) {
    int ds = D / M;
    for (int m = 0; m < M; ++m)
        for (int z = 0; z < Z; ++z)
            A[m * Z + z] = ca1(q + m * ds, cb + ((int64_t)m * Z + z) * ds, ds);
}

void rref_lut64(const float *cb, int D, int M, int Z, const float *q, double *A) {
    int ds = D / M;
    for (int m = 0; m < M; ++m)
        for (int z = 0; z < Z; ++z)
            A[m * Z + z] = ca1_64(q + m * ds, cb + ((int64_t)m * Z + z) * ds, ds);
}

/* CA2 / Eq. 2: d_A(q, xbar)^2 = sum_m A(m, xbar^m), fp32, m ascending. */
float rref_adc(const float *A, int M, int Z, const uint8_t *code) {
    float d = 0.0f;
    for (int m = 0; m < M; ++m) d = d + A[m * Z + code[m]];
    return d;
}

double rref_adc64(const double *A, int M, int Z, const uint8_t *code) {
    double d = 0.0;
    for (int m = 0; m < M; ++m) d = d + A[m * Z + code[m]];
    return d;
}

/* Symmetric distance tables (d_S): T[m][i][j] = CA1(c_{m,i}, c_{m,j}). */
void rref_sdc_tables(const float *cb, int D, int M, int Z, float *T) {
    int ds = D / M;
    for (int m = 0; m < M; ++m)
        for (int i = 0; i < Z; ++i)
            for (int j = 0; j < Z; ++j)
                T[((int64_t)m * Z + i) * Z + j] =
                    ca1(cb + ((int64_t)m * Z + i) * ds, cb + ((int64_t)m * Z + j) * ds, ds);
}

/* d_S(a, b) = sum_m T_m[a_m][b_m] in CA2 order. */
float rref_sdc(const float *T, int M, int Z, const uint8_t *a, const uint8_t *b) {
    float d = 0.0f;
    for (int m = 0; m < M; ++m) d = d + T[((int64_t)m * Z + a[m]) * Z + b[m]];
    return d;
}

/* ------------------------------------------------------------------------- */
/* Result array U with PartialSort + Take (Alg. 1 L2, L5-L7).  The
 * paper's partial_sort keeps the R best; here a sorted array of at most R
 * (dist, id) tuples, ordered lexicographically (CA4: ties to the lowest id). */
typedef struct {
    int R, count;
    float *d;
    int64_t *id;
} topr_t;

static int topr_less(float da, int64_t ia, float db, int64_t ib) {
    return da < db || (da == db && ia < ib);
}

static void topr_push(topr_t *t, float d, int64_t id) {
    if (t->count == t->R && !topr_less(d, id, t->d[t->R - 1], t->id[t->R - 1])) return;
    int pos = t->count < t->R ? t->count : t->R - 1;
    while (pos > 0 && topr_less(d, id, t->d[pos - 1], t->id[pos - 1])) {
        t->d[pos] = t->d[pos - 1];
        t->id[pos] = t->id[pos - 1];
        --pos;
    }
    t->d[pos] = d;
    t->id[pos] = id;
    if (t->count < t->R) t->count++;
}

/* Take(U, R), padded with (id -1, +inf) when fewer than R candidates exist (R18). */
static void topr_take(const topr_t *t, int64_t *out_ids, float *out_dist) {
    for (int r = 0; r < t->R; ++r) {
        if (r < t->count) { out_ids[r] = t->id[r]; out_dist[r] = t->d[r]; }
        else { out_ids[r] = -1; out_dist[r] = INFINITY; }
    }
}

static int check_targets(const int64_t *S, int64_t nS, int64_t N) {
    for (int64_t i = 0; i < nS; ++i) {
        if (S[i] < 0 || S[i] >= N) return REF_ERR_ARG;
        if (i > 0 && S[i] <= S[i - 1]) return REF_ERR_ARG; /* R6: strictly ascending */
    }
    return REF_OK;
}

/* Alg. 1 PQLinearScan: for s in S: d = sum_m A(m, xbar_s^m);
 * PushBack; PartialSort(U, R); Take(U, R).  S == NULL means S = {0..N-1}. */
int rref_linear(const float *cb, int D, int M, int Z, const uint8_t *codes, int64_t N,
                const float *q, int64_t nq, int topk, const int64_t *S, int64_t nS,
                int64_t *out_ids, float *out_dist) {
    if (topk < 1) return REF_ERR_ARG;
    if (S && check_targets(S, nS, N) != REF_OK) return REF_ERR_ARG;
    float *A = (float *)malloc(sizeof(float) * M * Z);
    topr_t t = {topk, 0, (float *)malloc(sizeof(float) * topk), (int64_t *)malloc(sizeof(int64_t) * topk)};
    if (!A || !t.d || !t.id) { free(A); free(t.d); free(t.id); return REF_ERR_OOM; }
    int64_t ns = S ? nS : N;
    for (int64_t qi = 0; qi < nq; ++qi) {
        rref_lut(cb, D, M, Z, q + qi * D, A);                 /* L1 */
        t.count = 0;                                          /* L2 */
        for (int64_t i = 0; i < ns; ++i) {                    /* L3 */
            int64_t s = S ? S[i] : i;
            float d = rref_adc(A, M, Z, codes + s * M);       /* L4 */
            topr_push(&t, d, s);                              /* L5-L6 */
        }
        topr_take(&t, out_ids + qi * topk, out_dist + qi * topk); /* L7 */
    }
    free(A); free(t.d); free(t.id);
    return REF_OK;
}

typedef struct { float d; int64_t k; } dk_t;
static int dk_cmp(const void *a, const void *b) {
    const dk_t *x = (const dk_t *)a, *y = (const dk_t *)b;
    if (x->d < y->d) return -1;
    if (x->d > y->d) return 1;
    return (x->k > y->k) - (x->k < y->k);
}

static int is_member(const int64_t *S, int64_t nS, int64_t n) { /* binary search */
    int64_t lo = 0, hi = nS;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (S[mid] < n) lo = mid + 1; else hi = mid;
    }
    return lo < nS && S[lo] == n;
}

/* Number of posting lists to traverse (reading R1):
 * S = ALL -> min(L, K); otherwise min(K, ceil(L*N/|S|)). */
int64_t rref_num_probe(int64_t N, int64_t K, int64_t nS, int has_S, int64_t L) {
    if (!has_S) return L < K ? L : K;
    if (nS <= 0) return 0;
    int64_t p = (L * N + nS - 1) / nS;
    return p < K ? p : K;
}

/* Alg. 2 InvertedIndex under readings R1 (L = lists) and R2 mode A
 * (every S-member of the P nearest lists is evaluated; no mid-list stop). */
int rref_ivf(const float *cb, int D, int M, int Z, const uint8_t *codes, int64_t N,
             const uint8_t *centers, int64_t K, const int64_t *offsets, const int64_t *ids,
             const float *q, int64_t nq, int topk, const int64_t *S, int64_t nS, int64_t L,
             int64_t *out_ids, float *out_dist) {
    if (topk < 1 || K < 1 || L < 1) return REF_ERR_ARG;
    if (S && check_targets(S, nS, N) != REF_OK) return REF_ERR_ARG;
    float *A = (float *)malloc(sizeof(float) * M * Z);
    dk_t *T = (dk_t *)malloc(sizeof(dk_t) * K);
    topr_t t = {topk, 0, (float *)malloc(sizeof(float) * topk), (int64_t *)malloc(sizeof(int64_t) * topk)};
    if (!A || !T || !t.d || !t.id) { free(A); free(T); free(t.d); free(t.id); return REF_ERR_OOM; }
    int64_t P = rref_num_probe(N, K, nS, S != NULL, L);
    for (int64_t qi = 0; qi < nq; ++qi) {
        rref_lut(cb, D, M, Z, q + qi * D, A);                         /* L1 */
        for (int64_t k = 0; k < K; ++k) {                             /* L3-L5 */
            T[k].d = rref_adc(A, M, Z, centers + k * M);
            T[k].k = k;
        }
        qsort(T, (size_t)K, sizeof(dk_t), dk_cmp);                    /* L6 (full sort; first P used) */
        t.count = 0;                                                  /* L7 */
        for (int64_t r = 0; r < P; ++r) {                             /* L8 */
            int64_t k = T[r].k;
            for (int64_t p = offsets[k]; p < offsets[k + 1]; ++p) {   /* L9 */
                int64_t n = ids[p];
                if (S && !is_member(S, nS, n)) continue;              /* L10-L11 (skipped for S=ALL) */
                float d = rref_adc(A, M, Z, codes + n * M);           /* L12 */
                topr_push(&t, d, n);                                  /* L13 */
            }
        }
        topr_take(&t, out_ids + qi * topk, out_dist + qi * topk);     /* L14-L16 */
    }
    free(A); free(T); free(t.d); free(t.id);
    return REF_OK;
}

/* Alg. 2 InvertedIndex exactly as printed (reading R2 mode B, "paper"):
 * L is the number of candidates.  The ceil(K L / |S|) (capped at K, P:492-502;
 * |S| = N for S = ALL) nearest lists by (d0, k) are traversed in that order, ids
 * ascending inside a list (R11), non-members of S skipped (L10-11), and the
 * traversal returns as soon as |U| = L (L14-16); if the lists run out first, what
 * was collected is returned. */
int rref_ivf_paper(const float *cb, int D, int M, int Z, const uint8_t *codes, int64_t N,
                   const uint8_t *centers, int64_t K, const int64_t *offsets, const int64_t *ids,
                   const float *q, int64_t nq, int topk, const int64_t *S, int64_t nS, int64_t L,
                   int64_t *out_ids, float *out_dist) {
    if (topk < 1 || K < 1 || L < 1) return REF_ERR_ARG;
    if (S && check_targets(S, nS, N) != REF_OK) return REF_ERR_ARG;
    float *A = (float *)malloc(sizeof(float) * M * Z);
    dk_t *T = (dk_t *)malloc(sizeof(dk_t) * K);
    topr_t t = {topk, 0, (float *)malloc(sizeof(float) * topk), (int64_t *)malloc(sizeof(int64_t) * topk)};
    if (!A || !T || !t.d || !t.id) { free(A); free(T); free(t.d); free(t.id); return REF_ERR_OOM; }
    int64_t ns = S ? nS : N;
    int64_t P = ns > 0 ? (K * L + ns - 1) / ns : K;
    if (P > K) P = K;
    for (int64_t qi = 0; qi < nq; ++qi) {
        rref_lut(cb, D, M, Z, q + qi * D, A);                         /* L1 */
        for (int64_t k = 0; k < K; ++k) {                             /* L3-L5 */
            T[k].d = rref_adc(A, M, Z, centers + k * M);
            T[k].k = k;
        }
        qsort(T, (size_t)K, sizeof(dk_t), dk_cmp);                    /* L6 */
        t.count = 0;                                                  /* L7 */
        int64_t got = 0;
        for (int64_t r = 0; r < P && got < L; ++r) {                  /* L8 */
            int64_t k = T[r].k;
            for (int64_t p = offsets[k]; p < offsets[k + 1] && got < L; ++p) {  /* L9 */
                int64_t n = ids[p];
                if (S && !is_member(S, nS, n)) continue;              /* L10-L11 */
                float d = rref_adc(A, M, Z, codes + n * M);           /* L12 */
                topr_push(&t, d, n);                                  /* L13 */
                ++got;                                                /* L14: stop at |U| = L */
            }
        }
        topr_take(&t, out_ids + qi * topk, out_dist + qi * topk);     /* L15-L16 */
    }
    free(A); free(T); free(t.d); free(t.id);
    return REF_OK;
}

/* Default threshold (reading R3): theta(L) = ceil(L*N/K) + K. */
int64_t rref_default_theta(int64_t N, int64_t K, int64_t L) {
    if (K <= 0) return INT64_MAX;
    return (L * N + K - 1) / K + K;
}

/* Alg. 3 Query: |S| < theta -> PQLinearScan, else InvertedIndex.
 * theta < 0 -> default (R3).  K == 0 forces the linear scan. */
int rref_query(const float *cb, int D, int M, int Z, const uint8_t *codes, int64_t N,
               const uint8_t *centers, int64_t K, const int64_t *offsets, const int64_t *ids,
               const float *q, int64_t nq, int topk, const int64_t *S, int64_t nS, int64_t L,
               int64_t theta, int path, int64_t *out_ids, float *out_dist, int *path_used) {
    int64_t ns = S ? nS : N;
    int use = path;
    if (K <= 0) {
        if (path == REF_PATH_IVF) return REF_ERR_STATE;
        use = REF_PATH_LINEAR;
    } else if (path == REF_PATH_AUTO) {
        int64_t th = theta >= 0 ? theta : rref_default_theta(N, K, L);
        use = ns < th ? REF_PATH_LINEAR : REF_PATH_IVF;   /* L1 */
    }
    if (path_used) *path_used = use;
    if (use == REF_PATH_LINEAR)
        return rref_linear(cb, D, M, Z, codes, N, q, nq, topk, S, nS, out_ids, out_dist);
    return rref_ivf(cb, D, M, Z, codes, N, centers, K, offsets, ids, q, nq, topk, S, nS, L,
                    out_ids, out_dist);
}

/* ------------------------------------------------------------------------- */
/* Assignment a(n) = argmin_k d_S(xbar_n, cbar_k), CA2 order, ties
 * to the lowest k (CA4).  dist_out (optional) receives the fp32 minimum. */
int rref_assign(const float *T, int M, int Z, const uint8_t *codes, int64_t n,
                const uint8_t *centers, int64_t K, int32_t *assign_out, float *dist_out) {
    if (K < 1) return REF_ERR_ARG;
    for (int64_t i = 0; i < n; ++i) {
        float best = INFINITY;
        int64_t bk = 0;
        for (int64_t k = 0; k < K; ++k) {
            float d = rref_sdc(T, M, Z, codes + i * M, centers + k * M);
            if (d < best) { best = d; bk = k; }
        }
        assign_out[i] = (int32_t)bk;
        if (dist_out) dist_out[i] = best;
    }
    return REF_OK;
}

/* Posting lists W_k = {n | a(n) = k} (Eq. 4), ids ascending (R11),
 * stored as CSR: offsets[K+1], ids[N]. */
int rref_build_postings(const int32_t *assign, int64_t N, int64_t K, int64_t *offsets, int64_t *ids) {
    for (int64_t k = 0; k <= K; ++k) offsets[k] = 0;
    for (int64_t n = 0; n < N; ++n) {
        if (assign[n] < 0 || assign[n] >= K) return REF_ERR_ARG;
        offsets[assign[n] + 1]++;
    }
    for (int64_t k = 0; k < K; ++k) offsets[k + 1] += offsets[k];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (K > 0 ? K : 1));
    if (!fill) return REF_ERR_OOM;
    for (int64_t k = 0; k < K; ++k) fill[k] = offsets[k];
    for (int64_t n = 0; n < N; ++n) ids[fill[assign[n]]++] = n;
    free(fill);
    return REF_OK;
}

/* ------------------------------------------------------------------------- */
/* Reconfigure sample (reading R10): the n_s = min(N, 100 K') ids
 * with the smallest splitmix64(seed ^ id), returned in ascending key order. */
typedef struct { uint64_t key; int64_t id; } kid_t;
static int kid_cmp(const void *a, const void *b) {
    const kid_t *x = (const kid_t *)a, *y = (const kid_t *)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

int rref_sample_ids(int64_t N, int64_t ns, uint64_t seed, int64_t *out) {
    if (ns > N || ns < 0) return REF_ERR_ARG;
    kid_t *a = (kid_t *)malloc(sizeof(kid_t) * (N > 0 ? N : 1));
    if (!a) return REF_ERR_OOM;
    for (int64_t i = 0; i < N; ++i) { a[i].key = rref_splitmix64(seed ^ (uint64_t)i); a[i].id = i; }
    qsort(a, (size_t)N, sizeof(kid_t), kid_cmp);
    for (int64_t i = 0; i < ns; ++i) out[i] = a[i].id;
    free(a);
    return REF_OK;
}

/* PQk-means (P:674-675, P:697 cite the PQk-means paper; update rule = reading R9):
 *  init     : the first K distinct codes of the sample, in sample order;
 *  iterate  : assign (CA2 argmin, ties lowest k) -> histogram h[k][m][z'] ->
 *             new cbar_k^m = argmin_z sum_{z'} h[k][m][z'] * (double)T_m[z][z'] (fp64,
 *             z' ascending, ties lowest z) -> empty clusters, k ascending, take the
 *             not-yet-used member of the currently largest cluster (ties lowest k)
 *             farthest (fp32 assignment distance; ties lowest sample index) from its
 *             centre; that member's code becomes cbar_k and moves to k.
 * objective (optional, n_iter + 1 values): fp64 sum over the sample of the fp64
 * SDC to the assigned centre, after each assignment step and after the final one. */
int rref_pqkmeans(const float *T, int M, int Z, const uint8_t *X, int64_t ns, int64_t K,
                  int n_iter, uint8_t *C, double *objective) {
    if (K < 1 || K > ns || n_iter < 0) return REF_ERR_ARG;
    /* init: first K pairwise-distinct codes in sample order */
    int64_t got = 0;
    for (int64_t i = 0; i < ns && got < K; ++i) {
        int dup = 0;
        for (int64_t k = 0; k < got && !dup; ++k)
            if (memcmp(C + k * M, X + i * M, (size_t)M) == 0) dup = 1;
        if (!dup) { memcpy(C + got * M, X + i * M, (size_t)M); ++got; }
    }
    if (got < K) return REF_ERR_ARG;

    int32_t *a = (int32_t *)malloc(sizeof(int32_t) * ns);
    float *dist = (float *)malloc(sizeof(float) * ns);
    int64_t *size = (int64_t *)malloc(sizeof(int64_t) * K);
    int64_t *h = (int64_t *)malloc(sizeof(int64_t) * M * Z);
    char *used = (char *)malloc((size_t)ns);
    if (!a || !dist || !size || !h || !used) {
        free(a); free(dist); free(size); free(h); free(used);
        return REF_ERR_OOM;
    }
    for (int it = 0; it <= n_iter; ++it) {
        rref_assign(T, M, Z, X, ns, C, K, a, dist);
        if (objective) {
            double obj = 0.0;
            for (int64_t i = 0; i < ns; ++i) {
                double s = 0.0;
                for (int m = 0; m < M; ++m)
                    s = s + (double)T[((int64_t)m * Z + X[i * M + m]) * Z + C[(int64_t)a[i] * M + m]];
                obj = obj + s;
            }
            objective[it] = obj;
        }
        if (it == n_iter) break;
        for (int64_t k = 0; k < K; ++k) size[k] = 0;
        for (int64_t i = 0; i < ns; ++i) size[a[i]]++;
        /* update step: per cluster k with members, per subspace m */
        for (int64_t k = 0; k < K; ++k) {
            if (size[k] == 0) continue;
            for (int64_t j = 0; j < (int64_t)M * Z; ++j) h[j] = 0;
            for (int64_t i = 0; i < ns; ++i)
                if (a[i] == k)
                    for (int m = 0; m < M; ++m) h[m * Z + X[i * M + m]]++;
            for (int m = 0; m < M; ++m) {
                double best = INFINITY;
                int bz = 0;
                for (int z = 0; z < Z; ++z) {
                    double s = 0.0;
                    for (int zp = 0; zp < Z; ++zp)
                        s = s + (double)h[m * Z + zp] * (double)T[((int64_t)m * Z + z) * Z + zp];
                    if (s < best) { best = s; bz = z; }
                }
                C[k * M + m] = (uint8_t)bz;
            }
        }
        /* re-seed empty clusters */
        memset(used, 0, (size_t)ns);
        for (int64_t k = 0; k < K; ++k) {
            if (size[k] != 0) continue;
            int64_t g = 0;
            for (int64_t j = 1; j < K; ++j) if (size[j] > size[g]) g = j;
            int64_t bi = -1;
            for (int64_t i = 0; i < ns; ++i) {
                if (a[i] != g || used[i]) continue;
                if (bi < 0 || dist[i] > dist[bi]) bi = i;
            }
            if (bi < 0) continue; /* unreachable while K <= ns */
            g_reseeds[1]++;
            memcpy(C + k * M, X + bi * M, (size_t)M);
            used[bi] = 1;
            a[bi] = (int32_t)k;
            size[g]--;
            size[k] = 1;
        }
    }
    free(a); free(dist); free(size); free(h); free(used);
    return REF_OK;
}

/* Alg. 4 Reconfigure: Cbar <- PQkmeans(sample of min(N, 100K') codes,
 * K'); W_k <- {n | a(n) = k} over all N codes.  Outputs centers[K*M], assign[N],
 * offsets[K+1], ids[N]. */
int rref_reconfigure(const float *cb, int D, int M, int Z, const uint8_t *codes, int64_t N,
                     int64_t K, int n_iter, uint64_t seed, uint8_t *centers, int32_t *assign,
                     int64_t *offsets, int64_t *ids, double *objective) {
    if (K < 1 || K > N) return REF_ERR_ARG;
    int64_t ns = 100 * K < N ? 100 * K : N;
    float *T = (float *)malloc(sizeof(float) * (size_t)M * Z * Z);
    int64_t *sid = (int64_t *)malloc(sizeof(int64_t) * ns);
    uint8_t *X = (uint8_t *)malloc((size_t)ns * M);
    if (!T || !sid || !X) { free(T); free(sid); free(X); return REF_ERR_OOM; }
    rref_sdc_tables(cb, D, M, Z, T);
    int st = rref_sample_ids(N, ns, seed, sid);
    if (st == REF_OK) {
        for (int64_t i = 0; i < ns; ++i) memcpy(X + i * M, codes + sid[i] * M, (size_t)M);
        st = rref_pqkmeans(T, M, Z, X, ns, K, n_iter, centers, objective);
    }
    if (st == REF_OK) st = rref_assign(T, M, Z, codes, N, centers, K, assign, NULL);
    if (st == REF_OK) st = rref_build_postings(assign, N, K, offsets, ids);
    free(T); free(sid); free(X);
    return st;
}

/* ------------------------------------------------------------------------- */
/* Code-book training (reading R8; the paper only says "preliminarily trained",
 * P:777): per subspace m, Lloyd k-means with
 *  init   : the Z rows with the smallest splitmix64(seed ^ (m << 40) ^ row) whose
 *           sub-vectors are pairwise distinct (key order);
 *  assign : CA1 argmin, ties lowest z; d_i = that fp32 minimum;
 *  update : member sums in int64 fixed point llrint((double)v * 2^32), mean =
 *           (float)(((double)sum / 2^32) / (double)count);
 *  empty  : z ascending, the not-yet-used row with the largest d_i (ties lowest row).
 * Requires n >= Z and n * max|v| < 2^31 (fixed-point range). */
int rref_train(const float *x, int64_t n, int D, int M, int Z, int n_iter, uint64_t seed, float *cb) {
    if (M <= 0 || D % M != 0 || Z < 1 || Z > 256 || n_iter < 0) return REF_ERR_ARG;
    if (n < Z) return REF_ERR_TRAIN;
    int ds = D / M;
    double amax = 0.0;
    for (int64_t i = 0; i < n * D; ++i) { double v = fabs((double)x[i]); if (v > amax) amax = v; }
    if (amax * (double)n >= 2147483648.0) return REF_ERR_ARG;

    kid_t *ord = (kid_t *)malloc(sizeof(kid_t) * n);
    int32_t *a = (int32_t *)malloc(sizeof(int32_t) * n);
    float *d = (float *)malloc(sizeof(float) * n);
    int64_t *sum = (int64_t *)malloc(sizeof(int64_t) * Z * ds);
    int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * Z);
    char *used = (char *)malloc((size_t)n);
    int st = REF_OK;
    if (!ord || !a || !d || !sum || !cnt || !used) { st = REF_ERR_OOM; goto done; }

    for (int m = 0; m < M && st == REF_OK; ++m) {
        float *c = cb + (int64_t)m * Z * ds;
        for (int64_t i = 0; i < n; ++i) {
            ord[i].key = rref_splitmix64(seed ^ ((uint64_t)m << 40) ^ (uint64_t)i);
            ord[i].id = i;
        }
        qsort(ord, (size_t)n, sizeof(kid_t), kid_cmp);
        int got = 0;
        for (int64_t r = 0; r < n && got < Z; ++r) {
            const float *u = x + ord[r].id * D + m * ds;
            int dup = 0;
            for (int z = 0; z < got && !dup; ++z) {
                int eq = 1;
                for (int j = 0; j < ds; ++j) if (c[z * ds + j] != u[j]) { eq = 0; break; }
                dup = eq;
            }
            if (!dup) { for (int j = 0; j < ds; ++j) c[got * ds + j] = u[j]; ++got; }
        }
        if (got < Z) { st = REF_ERR_TRAIN; break; }

        for (int it = 0; it < n_iter; ++it) {
            for (int64_t i = 0; i < n; ++i) {
                const float *u = x + i * D + m * ds;
                float best = INFINITY;
                int bz = 0;
                for (int z = 0; z < Z; ++z) {
                    float dd = ca1(u, c + z * ds, ds);
                    if (dd < best) { best = dd; bz = z; }
                }
                a[i] = bz;
                d[i] = best;
            }
            for (int64_t j = 0; j < (int64_t)Z * ds; ++j) sum[j] = 0;
            for (int z = 0; z < Z; ++z) cnt[z] = 0;
            for (int64_t i = 0; i < n; ++i) {
                cnt[a[i]]++;
                for (int j = 0; j < ds; ++j)
                    sum[a[i] * ds + j] += llrint((double)x[i * D + m * ds + j] * 4294967296.0);
            }
            for (int z = 0; z < Z; ++z) {
                if (cnt[z] == 0) continue;
                for (int j = 0; j < ds; ++j)
                    c[z * ds + j] = (float)(((double)sum[z * ds + j] / 4294967296.0) / (double)cnt[z]);
            }
            memset(used, 0, (size_t)n);
            for (int z = 0; z < Z; ++z) {
                if (cnt[z] != 0) continue;
                int64_t bi = -1;
                for (int64_t i = 0; i < n; ++i) {
                    if (used[i]) continue;
                    if (bi < 0 || d[i] > d[bi]) bi = i;
                }
                used[bi] = 1;
                g_reseeds[0]++;
                for (int j = 0; j < ds; ++j) c[z * ds + j] = x[bi * D + m * ds + j];
            }
        }
    }
done:
    free(ord); free(a); free(d); free(sum); free(cnt); free(used);
    return st;
}
