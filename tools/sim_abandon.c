// sim_abandon.c -- planning tool (not product, not oracle): how many DP cells does early
// abandoning evaluate on the survivors of a query if the abandon test adds the LB_Keogh
// suffix of the rows not yet reached (UCR-suite style) versus the plain row minimum?
//
//   gcc -O2 -fopenmp -o /tmp/sim tools/sim_abandon.c -lm
//   /tmp/sim train.f32 test.f32 N Q L w
//
// Survivors = pairs with LB_Keogh <= d* (d* = the query's exact NN distance, i.e. the final
// best-so-far); abandon threshold = d*.  Prints total cells evaluated both ways.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

static float *load(const char *path, long n) {
    float *x = malloc(n * sizeof(float));
    FILE *f = fopen(path, "rb");
    if (!f || fread(x, sizeof(float), n, f) != (size_t)n) {
        fprintf(stderr, "read %s\n", path);
        exit(1);
    }
    fclose(f);
    return x;
}

// row-major DTW with row-min abandoning; suffix (nullable) adds S[i+1] to the row minimum.
static double dtw(const float *a, const float *b, int L, int w, double thr, const double *suf,
                  long *cells) {
    double *prev = malloc((L + 1) * sizeof(double)), *cur = malloc((L + 1) * sizeof(double));
    for (int j = 0; j <= L; ++j) prev[j] = INFINITY;
    prev[0] = 0;
    long c = 0;
    double res = INFINITY;
    for (int i = 1; i <= L; ++i) {
        for (int j = 0; j <= L; ++j) cur[j] = INFINITY;
        int jl = i - w > 1 ? i - w : 1, jh = i + w < L ? i + w : L;
        double rmin = INFINITY;
        for (int j = jl; j <= jh; ++j) {
            double d = (double)a[i - 1] - b[j - 1];
            double m = prev[j - 1];
            if (prev[j] < m) m = prev[j];
            if (cur[j - 1] < m) m = cur[j - 1];
            cur[j] = d * d + m;
            if (cur[j] < rmin) rmin = cur[j];
            ++c;
        }
        double extra = suf ? suf[i] : 0.0;  // rows i+1..L (1-based) = suffix from index i
        if (rmin + extra > thr) {
            res = INFINITY;
            goto out;
        }
        double *t = prev;
        prev = cur;
        cur = t;
    }
    res = prev[L];
out:
    free(prev);
    free(cur);
    *cells += c;
    return res;
}

int main(int argc, char **argv) {
    if (argc < 7) return 1;
    long N = atol(argv[3]), Q = atol(argv[4]);
    int L = atoi(argv[5]), w = atoi(argv[6]);
    float *T = load(argv[1], N * L), *X = load(argv[2], Q * L);
    float *U = malloc(N * L * sizeof(float)), *Lo = malloc(N * L * sizeof(float));
    for (long n = 0; n < N; ++n)
        for (int i = 0; i < L; ++i) {
            float u = -INFINITY, l = INFINITY;
            for (int j = i - w < 0 ? 0 : i - w; j <= (i + w < L - 1 ? i + w : L - 1); ++j) {
                float v = T[n * L + j];
                if (v > u) u = v;
                if (v < l) l = v;
            }
            U[n * L + i] = u;
            Lo[n * L + i] = l;
        }
    long tot_a = 0, tot_b = 0, nsurv = 0, full = 0;
#pragma omp parallel for reduction(+ : tot_a, tot_b, nsurv, full) schedule(dynamic)
    for (long q = 0; q < Q; ++q) {
        const float *a = X + q * L;
        double *lb = malloc(N * sizeof(double));
        double *suf = malloc((L + 1) * sizeof(double));
        for (long n = 0; n < N; ++n) {
            double s = 0;
            for (int i = 0; i < L; ++i) {
                double t = 0, x = a[i];
                if (x > U[n * L + i]) t = x - U[n * L + i];
                else if (x < Lo[n * L + i]) t = Lo[n * L + i] - x;
                s += t * t;
            }
            lb[n] = s;
        }
        // exact NN: visit in LB order (selection of the min repeatedly is slow; use the
        // argmin seed, then all with lb <= bsf)
        long am = 0;
        for (long n = 1; n < N; ++n)
            if (lb[n] < lb[am]) am = n;
        long dummy = 0;
        double bsf = dtw(a, T + am * L, L, w, INFINITY, NULL, &dummy);
        for (long n = 0; n < N; ++n)
            if (lb[n] <= bsf) {
                double d = dtw(a, T + n * L, L, w, bsf, NULL, &dummy);
                if (d < bsf) bsf = d;
            }
        for (long n = 0; n < N; ++n) {
            if (!(lb[n] <= bsf)) continue;
            nsurv++;
            suf[L] = 0;
            for (int i = L - 1; i >= 0; --i) {
                double t = 0, x = a[i];
                if (x > U[n * L + i]) t = x - U[n * L + i];
                else if (x < Lo[n * L + i]) t = Lo[n * L + i] - x;
                suf[i] = suf[i + 1] + t * t;
            }
            long ca = 0, cb = 0;
            dtw(a, T + n * L, L, w, bsf, NULL, &ca);
            dtw(a, T + n * L, L, w, bsf, suf, &cb);
            tot_a += ca;
            tot_b += cb;
            if (cb == (long)L * (2 * w + 1) - (long)w * (w + 1)) full++;
        }
        free(lb);
        free(suf);
    }
    printf("survivors %ld  cells plain %ld  cells with suffix %ld  ratio %.3f  full %ld\n", nsurv,
           tot_a, tot_b, (double)tot_b / tot_a, full);
    return 0;
}
