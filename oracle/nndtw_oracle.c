/*
 * nndtw_oracle.c -- plain, slow, fp64 CPU oracle for exact 1-NN search under windowed DTW
 * pruned by LB_Kim -> LB_Enhanced^V (arxiv 1808.09617).
 *
 * TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load or call this library.  The CUDA product path shares no code,
 * header, table or helper with it, and must never route through it.
 *
 * Citations: "P:<line>" = /root/reference/PAPER.md line, "S:<line>" = SPEC.md line,
 * "Cn" = the reading numbered n in DESIGN.md ("Readings of the paper").
 *
 * Arithmetic: fp64 throughout; inputs are fp32 arrays promoted to double.  Build with
 * -O2 -ffp-contract=off and without -ffast-math so that every operation below is one IEEE
 * rounding (the per-cell contract of DESIGN.md: d = a-b; delta = d*d; D = delta + min).
 * Indices in comments follow the paper (1-based); code is 0-based.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_INF (1.0 / 0.0)

/* delta(a,b) = (a-b)^2.  P:143 calls it "the L2-norm of A_i and B_j"; Eq. 2 takes the
 * square root of the accumulated sum, so the cost is the squared difference (reading C1). */
static double delta(double a, double b) {
    double d = a - b;
    return d * d;
}

static double min2(double x, double y) { return y < x ? y : x; }

static int clamp_w(int L, int w) {
    /* C3: w >= L-1 is unconstrained ("DTW_L is equivalent to unconstrained DTW"). */
    if (w > L - 1) w = L - 1;
    return w;
}

/* ---------------------------------------------------------------------------------------
 * DTW_W (Eq. 1; window P:164-171), two rolling rows.  Boundary conditions
 * (reading C2): D(0,0)=0, D(i,0)=D(0,j)=+inf, cells with |i-j|>W are +inf.
 * Returns D(L,L) (squared domain); DTW = sqrt of it (Eq. 2).
 * If cutoff is finite, abandons when every in-window cell of a row exceeds cutoff (row-min
 * test, reading C14; a row is a cut of every warping path) and returns +inf with
 * *abandoned = 1.
 * ------------------------------------------------------------------------------------- */
double oracle_dtw_cut(const float *A, const float *B, int L, int w, double cutoff,
                      int *abandoned, int64_t *cells) {
    w = clamp_w(L, w);
    double *prev = (double *)malloc(sizeof(double) * (size_t)(L + 1));
    double *cur = (double *)malloc(sizeof(double) * (size_t)(L + 1));
    for (int j = 0; j <= L; ++j) prev[j] = ORACLE_INF;
    prev[0] = 0.0; /* D(0,0) = 0 */
    if (abandoned) *abandoned = 0;
    int64_t ncell = 0;
    for (int i = 1; i <= L; ++i) {
        for (int j = 0; j <= L; ++j) cur[j] = ORACLE_INF;
        int jlo = i - w < 1 ? 1 : i - w;
        int jhi = i + w > L ? L : i + w;
        double rowmin = ORACLE_INF;
        for (int j = jlo; j <= jhi; ++j) {
            /* Eq. 1: D(i,j) = delta(A_i,B_j) + min{D(i-1,j-1), D(i,j-1), D(i-1,j)} */
            double m = min2(min2(prev[j - 1], cur[j - 1]), prev[j]);
            double dij = delta((double)A[i - 1], (double)B[j - 1]) + m;
            cur[j] = dij;
            rowmin = min2(rowmin, dij);
            ++ncell;
        }
        double *t = prev; prev = cur; cur = t;
        if (rowmin > cutoff) {
            if (abandoned) *abandoned = 1;
            free(prev); free(cur);
            if (cells) *cells += ncell;
            return ORACLE_INF;
        }
    }
    double r = prev[L];
    free(prev); free(cur);
    if (cells) *cells += ncell;
    return r;
}

double oracle_dtw(const float *A, const float *B, int L, int w) {
    return oracle_dtw_cut(A, B, L, w, ORACLE_INF, NULL, NULL);
}

/* Squared Euclidean distance, the candidate-ordering key of P:567-570 (and DTW_0). */
double oracle_sqed(const float *A, const float *B, int L) {
    double s = 0.0;
    for (int i = 0; i < L; ++i) s = s + delta((double)A[i], (double)B[i]);
    return s;
}

/* ---------------------------------------------------------------------------------------
 * Envelopes, Eq. 3-4, naive scan:
 *   U_i = max_{max(1,i-W) <= j <= min(L,i+W)} B_j ,  L_i = min over the same range.
 * min/max of fp32 values are exact, so the outputs are fp32.
 * ------------------------------------------------------------------------------------- */
void oracle_envelope(const float *B, int L, int w, float *U, float *Lo) {
    w = clamp_w(L, w);
    for (int i = 1; i <= L; ++i) {
        int lo = i - w < 1 ? 1 : i - w;
        int hi = i + w > L ? L : i + w;
        float u = B[lo - 1], l = B[lo - 1];
        for (int j = lo; j <= hi; ++j) {
            if (B[j - 1] > u) u = B[j - 1];
            if (B[j - 1] < l) l = B[j - 1];
        }
        U[i - 1] = u;
        Lo[i - 1] = l;
    }
}

/* ---------------------------------------------------------------------------------------
 * LB_Kim, sum variant "without repetitions" (§4.2), reading C7:
 * features first, last, min, max in that order; a feature is dropped if its index in A or
 * its index in B was already used by an admitted feature; argmin/argmax ties -> lowest index.
 * ------------------------------------------------------------------------------------- */
static void argminmax(const float *X, int L, int *amin, int *amax) {
    int mn = 0, mx = 0;
    for (int i = 1; i < L; ++i) {
        if (X[i] < X[mn]) mn = i;
        if (X[i] > X[mx]) mx = i;
    }
    *amin = mn;
    *amax = mx;
}

double oracle_lb_kim_sum(const float *A, const float *B, int L) {
    int amin, amax, bmin, bmax;
    argminmax(A, L, &amin, &amax);
    argminmax(B, L, &bmin, &bmax);
    int ia[4] = {0, L - 1, amin, amax};
    int ib[4] = {0, L - 1, bmin, bmax};
    int usedA[4], usedB[4], nused = 0;
    double s = 0.0;
    for (int f = 0; f < 4; ++f) {
        int clash = 0;
        for (int u = 0; u < nused; ++u)
            if (usedA[u] == ia[f] || usedB[u] == ib[f]) clash = 1;
        if (clash) continue;
        s = s + delta((double)A[ia[f]], (double)B[ib[f]]);
        usedA[nused] = ia[f];
        usedB[nused] = ib[f];
        ++nused;
    }
    return s;
}

/* LB_Keogh terms summed over 1-based columns from..to inclusive (reading C6). */
double oracle_lb_keogh_range(const float *A, const float *U, const float *Lo, int from, int to) {
    double res = 0.0;
    for (int i = from; i <= to; ++i) {
        double a = (double)A[i - 1];
        if (a > (double)U[i - 1]) res = res + delta(a, (double)U[i - 1]);
        else if (a < (double)Lo[i - 1]) res = res + delta(a, (double)Lo[i - 1]);
    }
    return res;
}

double oracle_lb_keogh(const float *A, const float *U, const float *Lo, int L) {
    return oracle_lb_keogh_range(A, U, Lo, 1, L);
}

/* ---------------------------------------------------------------------------------------
 * LB_Enhanced^V_W, Algorithm 1, line by line.  D is the current distance to the
 * NN; the abort of line 12 ("if res >= D return inf") fires, per reading C12, only when
 * res > D*(1+margin) so that an exact tie is never pruned (margin = 0 gives Alg. 1's test
 * up to the >= / > distinction).  n_bands = min(floor(L/2), V) (reading C10).
 * Returns +inf and *aborted = 1 when line 12 fires.  L >= 2 (reading C11).
 * ------------------------------------------------------------------------------------- */
double oracle_lb_enhanced(const float *A, const float *B, const float *U, const float *Lo,
                          int L, int W, int V, double D, double margin, int *aborted) {
    W = clamp_w(L, W);
#define Ax(i) ((double)A[(i) - 1])
#define Bx(i) ((double)B[(i) - 1])
    if (aborted) *aborted = 0;
    /* line 1 */
    double res = delta(Ax(1), Bx(1)) + delta(Ax(L), Bx(L));
    /* line 2 */
    int n_bands = L / 2 < V ? L / 2 : V;
    /* lines 3-11: left bands L_i and right bands R_{L-i+1} */
    for (int i = 2; i <= n_bands; ++i) {
        double minL = delta(Ax(i), Bx(i));                           /* line 4 */
        double minR = delta(Ax(L - i + 1), Bx(L - i + 1));           /* line 5 */
        int j0 = i - W > 1 ? i - W : 1;
        for (int j = j0; j <= i - 1; ++j) {                           /* line 6 */
            minL = min2(minL, delta(Ax(i), Bx(j)));                   /* line 7 */
            minL = min2(minL, delta(Ax(j), Bx(i)));                   /* line 8 */
            minR = min2(minR, delta(Ax(L - i + 1), Bx(L - j + 1)));   /* line 9 */
            minR = min2(minR, delta(Ax(L - j + 1), Bx(L - i + 1)));   /* line 10 */
        }
        res = res + minL + minR;                                      /* line 11 */
    }
    /* line 12 */
    if (res > D * (1.0 + margin)) {
        if (aborted) *aborted = 1;
        return ORACLE_INF;
    }
    /* lines 13-15: LB_Keogh bridge over columns n_bands+1 .. L-n_bands */
    for (int i = n_bands + 1; i <= L - n_bands; ++i) {
        if (Ax(i) > (double)U[i - 1]) res = res + delta(Ax(i), (double)U[i - 1]);
        else if (Ax(i) < (double)Lo[i - 1]) res = res + delta(Ax(i), (double)Lo[i - 1]);
    }
    return res;
#undef Ax
#undef Bx
}

/* ---------------------------------------------------------------------------------------
 * LB_Improved_W (Lemire; §2.3.3 "Improved Lower Bound"): LB_Keogh(A, env B) plus
 * LB_Keogh(B, env A'), A' the projection of A onto the envelope of B (Eq. "projection",
 * P:261-268).  UB/LB = envelope of B (Eq. 3-4).  The envelope of A' is the naive scan.
 * (SURVEY §8(f) NEXT-4.)
 * ------------------------------------------------------------------------------------- */
double oracle_lb_improved(const float *A, const float *B, const float *UB, const float *LB,
                          int L, int W) {
    W = clamp_w(L, W);
    float *Ap = (float *)malloc(sizeof(float) * (size_t)L);
    float *Ua = (float *)malloc(sizeof(float) * (size_t)L);
    float *La = (float *)malloc(sizeof(float) * (size_t)L);
    for (int i = 0; i < L; ++i) {
        if (A[i] > UB[i]) Ap[i] = UB[i];
        else if (A[i] < LB[i]) Ap[i] = LB[i];
        else Ap[i] = A[i];
    }
    oracle_envelope(Ap, L, W, Ua, La);
    double res = oracle_lb_keogh(A, UB, LB, L) + oracle_lb_keogh(B, Ua, La, L);
    free(Ap); free(Ua); free(La);
    return res;
}

/* ---------------------------------------------------------------------------------------
 * LB_New_W (Shen et al.; §2.3.4 "New Lower Bound"):
 *   delta(A_1,B_1) + delta(A_L,B_L) + sum_{i=2}^{L-1} min_{j in [max(1,i-W), min(L,i+W)]}
 *   delta(A_i, B_j).
 * For L = 1 the two boundary terms are the same cell; the value is delta(A_1,B_1) (as C11).
 * ------------------------------------------------------------------------------------- */
double oracle_lb_new(const float *A, const float *B, int L, int W) {
    W = clamp_w(L, W);
    if (L == 1) return delta((double)A[0], (double)B[0]);
    double res = delta((double)A[0], (double)B[0]) + delta((double)A[L - 1], (double)B[L - 1]);
    for (int i = 2; i <= L - 1; ++i) {
        int lo = i - W < 1 ? 1 : i - W;
        int hi = i + W > L ? L : i + W;
        double m = ORACLE_INF;
        for (int j = lo; j <= hi; ++j) m = min2(m, delta((double)A[i - 1], (double)B[j - 1]));
        res = res + m;
    }
    return res;
}

/* Symmetric LB_Enhanced: max(LB_Enh(A,B), LB_Enh(B,A)); UB/LB
 * = envelope of B, UA/LA = envelope of A.  Both are admissible (Thm 2 with the roles of A and
 * B exchanged; DTW is symmetric), so their max is. */
double oracle_lb_enhanced_sym(const float *A, const float *B, const float *UA, const float *LA,
                              const float *UB, const float *LB, int L, int W, int V) {
    double x = oracle_lb_enhanced(A, B, UB, LB, L, W, V, ORACLE_INF, 0.0, NULL);
    double y = oracle_lb_enhanced(B, A, UA, LA, L, W, V, ORACLE_INF, 0.0, NULL);
    return x > y ? x : y;
}

/* ---------------------------------------------------------------------------------------
 * LB_Enhanced^V with the LB_Improved bridge ("replace LB_Keogh by LB_Improved within
 * LB_Enhanced"), reading C21:
 *   LB_Enhanced^V_W(A,B)  [bands + LB_Keogh bridge over rows n_bands+1 .. L-n_bands]
 *   + sum over the bridge columns j = n_bands+1 .. L-n_bands (1-based) of the LB_Keogh term of
 *     B_j against the envelope (Eq. 3-4, naive scan) of A', the projection of A onto the
 *     envelope of B (Eq. "projection").
 * Admissible: a cell (i,j) with |i-j| <= W has B_j in [L_i, U_i], so (A_i-B_j)^2 >=
 * (A_i-A'_i)^2 + (A'_i-B_j)^2; the first parts are counted once per bridge row (the LB_Keogh
 * terms), the second once per bridge column, and no cell of a bridge column lies in a band
 * (band cells have max(i,j) <= n_bands or min(i,j) > L-n_bands) -- LB_Improved's argument
 * next to Theorem 2's bands.
 * ------------------------------------------------------------------------------------- */
double oracle_lb_enhanced_improved(const float *A, const float *B, const float *UB,
                                   const float *LB, int L, int W, int V) {
    W = clamp_w(L, W);
    double res = oracle_lb_enhanced(A, B, UB, LB, L, W, V, ORACLE_INF, 0.0, NULL);
    int n_bands = L / 2 < V ? L / 2 : V;
    float *Ap = (float *)malloc(sizeof(float) * (size_t)L);
    float *Ua = (float *)malloc(sizeof(float) * (size_t)L);
    float *La = (float *)malloc(sizeof(float) * (size_t)L);
    for (int i = 0; i < L; ++i) {
        if (A[i] > UB[i]) Ap[i] = UB[i];
        else if (A[i] < LB[i]) Ap[i] = LB[i];
        else Ap[i] = A[i];
    }
    oracle_envelope(Ap, L, W, Ua, La);
    res = res + oracle_lb_keogh_range(B, Ua, La, n_bands + 1, L - n_bands);
    free(Ap); free(Ua); free(La);
    return res;
}

/* The cascade value used by the search (P:299-304 cascading, P:619-621 Kim):
 * max(LB_Kim_sum, LB_Enhanced) with no abort. */
double oracle_lb_cascade(const float *A, const float *B, const float *U, const float *Lo,
                         int L, int W, int V) {
    double k = oracle_lb_kim_sum(A, B, L);
    double e = oracle_lb_enhanced(A, B, U, Lo, L, W, V, ORACLE_INF, 0.0, NULL);
    return k > e ? k : e;
}

/* ---------------------------------------------------------------------------------------
 * Nearest-neighbour search.  Result per query: the train index
 * n minimising (D_n, n) lexicographically (reading C13: ties -> lowest index), its squared
 * distance, and counters.
 * ------------------------------------------------------------------------------------- */
typedef struct {
    int64_t lb_calls, pruned_kim, pruned_enh, dtw_calls, dtw_abandoned, cells;
} oracle_counts;

/* Mode (i): exhaustive.  exclude >= 0 skips that train index (LOOCV self-exclusion). */
static void nn_exhaustive_one(const float *q, const float *T, int64_t nt, int L, int w,
                              int64_t exclude, int64_t *idx, double *dist, oracle_counts *c) {
    double best = ORACLE_INF;
    int64_t bi = -1;
    for (int64_t n = 0; n < nt; ++n) {
        if (n == exclude) continue;
        double d = oracle_dtw_cut(q, T + n * (int64_t)L, L, w, ORACLE_INF, NULL,
                                  c ? &c->cells : NULL);
        if (c) c->dtw_calls++;
        if (d < best || bi < 0) { best = d; bi = n; }
    }
    *idx = bi;
    *dist = best;
}

/* Mode (ii): the paper's sequential pruned search.  Visit train series in ascending squared
 * Euclidean distance to the query, ties by index; prune by LB_Kim then by Algorithm 1
 * with the current D; DTW with row-min abandoning at D; update on (d < D) or (d == D and
 * n < nn) (reading C13).  Prune tests use D*(1+(3L+8)*2^-53) (reading C12) so an fp64 LB
 * that equals DTW mathematically (W=0) cannot prune a tie by one ulp. */
typedef struct { double key; int64_t n; } ed_pair;
static int cmp_ed(const void *x, const void *y) {
    const ed_pair *a = (const ed_pair *)x, *b = (const ed_pair *)y;
    if (a->key < b->key) return -1;
    if (a->key > b->key) return 1;
    return (a->n > b->n) - (a->n < b->n);
}

static void nn_pruned_one(const float *q, const float *T, const float *U, const float *Lo,
                          int64_t nt, int L, int w, int V, int64_t exclude, int64_t *idx,
                          double *dist, oracle_counts *c) {
    ed_pair *ord = (ed_pair *)malloc(sizeof(ed_pair) * (size_t)(nt > 0 ? nt : 1));
    int64_t m = 0;
    for (int64_t n = 0; n < nt; ++n) {
        if (n == exclude) continue;
        ord[m].key = oracle_sqed(q, T + n * (int64_t)L, L);
        ord[m].n = n;
        ++m;
    }
    qsort(ord, (size_t)m, sizeof(ed_pair), cmp_ed);
    double margin = (3.0 * L + 8.0) * 0x1p-53;
    double D = ORACLE_INF;
    int64_t nn = -1;
    for (int64_t k = 0; k < m; ++k) {
        int64_t n = ord[k].n;
        const float *B = T + n * (int64_t)L;
        if (c) c->lb_calls++;
        double lk = oracle_lb_kim_sum(q, B, L);
        if (lk > D * (1.0 + margin)) { if (c) c->pruned_kim++; continue; }
        int ab = 0;
        double le = oracle_lb_enhanced(q, B, U + n * (int64_t)L, Lo + n * (int64_t)L, L, w, V,
                                       D, margin, &ab);
        if (ab || le > D * (1.0 + margin)) { if (c) c->pruned_enh++; continue; }
        int abandoned = 0;
        if (c) c->dtw_calls++;
        double d = oracle_dtw_cut(q, B, L, w, D, &abandoned, c ? &c->cells : NULL);
        if (abandoned) { if (c) c->dtw_abandoned++; continue; }
        if (d < D || (d == D && n < nn) || nn < 0) { D = d; nn = n; }
    }
    free(ord);
    *idx = nn;
    *dist = D;
}

/* ---- thread pool over queries -------------------------------------------------------- */
typedef struct {
    const float *Q, *T, *U, *Lo;
    int64_t nq, nt;
    int L, w, V, mode;
    int64_t self_base; /* >= 0: query q excludes train index self_base+q (LOOCV) */
    int64_t *idx;
    double *dist;
    oracle_counts *counts; /* per query, nullable */
    int64_t next;
} nn_job;

static void *nn_worker(void *arg) {
    nn_job *J = (nn_job *)arg;
    for (;;) {
        int64_t q = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
        if (q >= J->nq) break;
        oracle_counts c;
        memset(&c, 0, sizeof c);
        int64_t ex = J->self_base >= 0 ? J->self_base + q : -1;
        if (J->mode == 0)
            nn_exhaustive_one(J->Q + q * (int64_t)J->L, J->T, J->nt, J->L, J->w, ex,
                              &J->idx[q], &J->dist[q], &c);
        else
            nn_pruned_one(J->Q + q * (int64_t)J->L, J->T, J->U, J->Lo, J->nt, J->L, J->w,
                          J->V, ex, &J->idx[q], &J->dist[q], &c);
        if (J->counts) J->counts[q] = c;
    }
    return NULL;
}

static void run_pool(nn_job *J, int threads) {
    if (threads < 1) threads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)threads);
    J->next = 0;
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, nn_worker, J);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
}

/* mode 0 = exhaustive (i), 1 = paper's pruned search (ii).  U/Lo are the train envelopes at w
 * (only read in mode 1).  counts: nullable array of nq records. */
void oracle_nn(const float *Q, int64_t nq, const float *T, const float *U, const float *Lo,
               int64_t nt, int L, int w, int V, int mode, int threads, int64_t *idx,
               double *dist, oracle_counts *counts) {
    nn_job J = {Q, T, U, Lo, nq, nt, L, w, V, mode, -1, idx, dist, counts, 0};
    run_pool(&J, threads);
}

/* Envelopes for a set of series (training-time precomputation). */
void oracle_envelopes(const float *X, int64_t n, int L, int w, float *U, float *Lo) {
    for (int64_t i = 0; i < n; ++i)
        oracle_envelope(X + i * (int64_t)L, L, w, U + i * (int64_t)L, Lo + i * (int64_t)L);
}

/* ---------------------------------------------------------------------------------------
 * Leave-one-out warping-window search (reading C17): for each window w_p and each
 * held-out series i in [q_begin, q_end), the NN over j != i; errors[p] counts label
 * mismatches.  nn_out (nullable) receives [nw][q_end-q_begin] NN indices.
 * ------------------------------------------------------------------------------------- */
void oracle_loocv(const float *X, const int32_t *labels, int64_t n, int L,
                  const int32_t *windows, int nw, int V, int64_t q_begin, int64_t q_end,
                  int mode, int threads, int64_t *errors, int64_t *nn_out) {
    int64_t nq = q_end - q_begin;
    float *U = (float *)malloc(sizeof(float) * (size_t)(n * L));
    float *Lo = (float *)malloc(sizeof(float) * (size_t)(n * L));
    int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nq > 0 ? nq : 1));
    double *dist = (double *)malloc(sizeof(double) * (size_t)(nq > 0 ? nq : 1));
    for (int p = 0; p < nw; ++p) {
        int w = windows[p];
        oracle_envelopes(X, n, L, w, U, Lo);
        nn_job J = {X + q_begin * (int64_t)L, X, U, Lo, nq, n, L, w, V, mode, q_begin,
                    idx, dist, NULL, 0};
        run_pool(&J, threads);
        int64_t e = 0;
        for (int64_t q = 0; q < nq; ++q) {
            /* no other series (n = 1): no neighbour, counted as an error (C17) */
            if (idx[q] < 0 || labels[idx[q]] != labels[q_begin + q]) ++e;
            if (nn_out) nn_out[(int64_t)p * nq + q] = idx[q];
        }
        errors[p] = e;
    }
    free(U); free(Lo); free(idx); free(dist);
}
