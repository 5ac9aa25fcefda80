// search.cu -- S3 (seed, prune, compaction), S5 (per-query argmin decode), S7 (fp64 near-tie
// re-rank) and S8 bookkeeping kernels.
#include <cstdlib>

#include "launchers.cuh"

namespace nndtw {

// ---- fills -----------------------------------------------------------------------------------
__global__ void k_fill_u64(unsigned long long *p, int64_t n, unsigned long long v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

int launch_fill_u64(unsigned long long *p, int64_t n, unsigned long long v, cudaStream_t st) {
    if (n <= 0) return 0;
    int64_t grid = (n + 255) / 256;
    if (grid > 4096) grid = 4096;
    k_fill_u64<<<(unsigned)grid, 256, 0, st>>>(p, n, v);
    count_launch(1, __func__);
    return 0;
}

// ---- classify call initialisation: every per-query slot and the counters in one launch --------
// key = (+inf, none), minkey = none, f64key = resolve_out = kNone64, overflow = tiecnt = 0,
// counters = 0, survivor-bucket counts = 0 (config-1-sized calls are a chain of small
// launches; this replaces seven)
__global__ void k_classify_init(int64_t nq, unsigned long long *key,
                                unsigned long long *minkey, unsigned long long *f64key,
                                unsigned long long *resolve_out, unsigned *overflow,
                                unsigned *tiecnt, unsigned long long *counters, int ncounters,
                                unsigned long long *bucket_count) {
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i0 < ncounters) counters[i0] = 0ull;
    if (i0 < NBUCKET) bucket_count[i0] = 0ull;
    for (int64_t i = i0; i < nq; i += (int64_t)gridDim.x * blockDim.x) {
        key[i] = kKeyInit;
        minkey[i] = kNone;
        f64key[i] = kNone64;
        resolve_out[i] = kNone64;
        overflow[i] = 0u;
        tiecnt[i] = 0u;
    }
}

int launch_classify_init(int64_t nq, unsigned long long *key, unsigned long long *minkey,
                         unsigned long long *f64key, unsigned long long *resolve_out,
                         unsigned *overflow, unsigned *tiecnt, unsigned long long *counters,
                         int ncounters, unsigned long long *bucket_count, cudaStream_t st) {
    int64_t grid = (nq + 255) / 256;
    if (grid < 1) grid = 1;
    if (grid > 4096) grid = 4096;
    k_classify_init<<<(unsigned)grid, 256, 0, st>>>(nq, key, minkey, f64key, resolve_out, overflow,
                                                    tiecnt, counters, ncounters, bucket_count);
    count_launch(1, __func__);
    return 0;
}

// ---- S3 seeds: the argmin-LB candidate of every query (and optionally a second candidate) -----
__global__ void k_seed_items(const unsigned long long *minkey, const int32_t *seed2, int64_t nq,
                             int64_t nt, Item *items, unsigned long long *count) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    unsigned long long k = minkey[q];
    unsigned n1 = (unsigned)(k & 0xffffffffull);
    if (k != kNone && n1 < (unsigned)nt) {
        unsigned long long pos = atomicAdd(count, 1ull);
        items[pos] = Item{(unsigned)q, n1, 0.0f};
    }
    if (seed2 != nullptr) {
        int n2 = seed2[q];
        if (n2 >= 0 && n2 < nt && (unsigned)n2 != n1) {
            unsigned long long pos = atomicAdd(count, 1ull);
            items[pos] = Item{(unsigned)q, (unsigned)n2, 0.0f};
        }
    }
}

// the train index of a packed key, or -1 (no candidate)
__global__ void k_key_index(const unsigned long long *key, int64_t nq, int64_t nt, int32_t *idx) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const unsigned long long k = key[q];
    const unsigned n = (unsigned)(k & 0xffffffffull);
    idx[q] = (k != kNone && n < (unsigned)nt) ? (int32_t)n : -1;
}

int launch_key_index(const unsigned long long *key, int64_t nq, int64_t nt, int32_t *idx,
                     cudaStream_t st) {
    if (nq == 0) return 0;
    k_key_index<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(key, nq, nt, idx);
    count_launch(1, __func__);
    return 0;
}

int launch_seed_items(const unsigned long long *minkey, const int32_t *seed2, int64_t nq,
                      int64_t nt, Item *items, unsigned long long *count, cudaStream_t st) {
    if (nq == 0) return 0;
    k_seed_items<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(minkey, seed2, nq, nt, items,
                                                               count);
    count_launch(1, __func__);
    return 0;
}

// ---- S3 compaction: surviving pairs LB <= bsf*(1+eps_p), in LB-bucket order -------------------
// One CTA-tile = (query q, CT_N consecutive train indices), 16 consecutive ones per thread (4
// float4 loads).  A survivor's bucket is floor(NBUCKET * LB / thr) (thr = the query's seeded
// best-so-far with the prune margin).  PASS 0 counts survivors per bucket (a shared-memory
// histogram per tile, one global atomic per bucket and tile); k_bucket_scan turns the counts
// into bucket offsets; PASS 1 reserves a contiguous run per bucket and tile and scatters the
// items, so the item list is bucket-major (and query-major inside a bucket): every query's
// lowest-bound candidates are processed first, across all queries at once.
constexpr int CT_N = 4096;

template <int PASS>
__global__ void __launch_bounds__(256) k_compact(const float *__restrict__ lb, int64_t ldlb,
                                                 int64_t nq, int64_t nt,
                                                 const unsigned long long *__restrict__ key,
                                                 const unsigned long long *__restrict__ minkey,
                                                 const int32_t *__restrict__ seed2, float eps_p,
                                                 Item *__restrict__ items,
                                                 unsigned long long *bucket_count,
                                                 const unsigned long long *bucket_base,
                                                 unsigned long long *bucket_fill,
                                                 unsigned long long capacity, int one_bucket) {
    __shared__ unsigned hist[NBUCKET];
    __shared__ unsigned long long base[NBUCKET];
    const int64_t tiles_per_row = (nt + CT_N - 1) / CT_N;
    const int64_t ntiles = tiles_per_row * nq;
    const bool vec = (ldlb & 3) == 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        if (threadIdx.x < NBUCKET) hist[threadIdx.x] = 0u;
        __syncthreads();
        const int64_t q = tile / tiles_per_row;
        const int64_t nbase = (tile % tiles_per_row) * CT_N;
        const float thr = key_dist(key[q]) * (1.0f + eps_p);
        const float scale = (thr > 0.0f && !one_bucket) ? (float)NBUCKET / thr : 0.0f;
        const unsigned s1 = (unsigned)(minkey[q] & 0xffffffffull);
        const unsigned s2 = seed2 ? (unsigned)seed2[q] : 0xffffffffu;
        const float *row = lb + q * ldlb;
        float v[16];
        unsigned flags = 0;  // bit e: element nbase + 16*tid + e survives
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t n0 = nbase + 16 * threadIdx.x + 4 * k;
            if (vec && n0 + 3 < nt) {
                const float4 f = *reinterpret_cast<const float4 *>(row + n0);
                v[4 * k] = f.x; v[4 * k + 1] = f.y; v[4 * k + 2] = f.z; v[4 * k + 3] = f.w;
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) v[4 * k + e] = (n0 + e < nt) ? row[n0 + e] : kInf;
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const unsigned n = (unsigned)(n0 + e);
                const bool ok = (n0 + e < nt) && v[4 * k + e] <= thr && n != s1 && n != s2;
                flags |= (ok ? 1u : 0u) << (4 * k + e);
            }
        }
        auto bucket_of = [&](float x) {
            const int b = (int)(x * scale);
            return b < 0 ? 0 : (b >= NBUCKET ? NBUCKET - 1 : b);
        };
        if (PASS == 0) {
#pragma unroll
            for (int e = 0; e < 16; ++e)
                if ((flags >> e) & 1u) atomicAdd(&hist[bucket_of(v[e])], 1u);
            __syncthreads();
            if (threadIdx.x < NBUCKET && hist[threadIdx.x])
                atomicAdd(bucket_count + threadIdx.x, (unsigned long long)hist[threadIdx.x]);
        } else {
            unsigned slot[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
                slot[e] = ((flags >> e) & 1u) ? atomicAdd(&hist[bucket_of(v[e])], 1u) : 0u;
            __syncthreads();
            if (threadIdx.x < NBUCKET) {
                const unsigned c = hist[threadIdx.x];
                base[threadIdx.x] = c ? bucket_base[threadIdx.x] +
                                            atomicAdd(bucket_fill + threadIdx.x, (unsigned long long)c)
                                      : 0ull;
            }
            __syncthreads();
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                if ((flags >> e) & 1u) {
                    const unsigned long long pos = base[bucket_of(v[e])] + slot[e];
                    if (pos < capacity)
                        items[pos] = Item{(unsigned)q, (unsigned)(nbase + 16 * threadIdx.x + e), v[e]};
                }
            }
        }
        __syncthreads();  // hist / base are reused by the next tile
    }
}

// bucket counts -> offsets; the total is the survivor count the DTW kernel reads
// (a capped workspace: survivors beyond `capacity` are not stored -- the overflow word is set
// and the call's answer is invalid; nndtw_classify_overflowed reports it to the caller)
__global__ void k_bucket_scan(const unsigned long long *count, unsigned long long *base,
                              unsigned long long *fill, unsigned long long *total,
                              unsigned long long capacity, unsigned long long *cap_overflow) {
    if (threadIdx.x == 0) {
        unsigned long long run = 0;
        for (int b = 0; b < NBUCKET; ++b) {
            base[b] = run;
            fill[b] = 0ull;
            run += count[b];
        }
        *total = run;
        if (run > capacity && cap_overflow) *cap_overflow = 1ull;
    }
}

int launch_compact(const float *lb, int64_t ldlb, int64_t nq, int64_t nt,
                   const unsigned long long *key, const unsigned long long *minkey,
                   const int32_t *seed2, float eps_p, Item *items, unsigned long long *count,
                   unsigned long long *buckets, unsigned long long capacity,
                   unsigned long long *cap_overflow, int num_sms, cudaStream_t st) {
    if (nq == 0 || nt == 0) return 0;
    // buckets: [count | base | fill] x NBUCKET; the counts were zeroed by k_classify_init
    unsigned long long *bcount = buckets, *bbase = buckets + NBUCKET, *bfill = buckets + 2 * NBUCKET;
    int64_t ntiles = ((nt + CT_N - 1) / CT_N) * nq;
    int64_t grid = ntiles < (int64_t)num_sms * 8 ? ntiles : (int64_t)num_sms * 8;
    static const char *ob = getenv("NNDTW_ONE_BUCKET");  // experiments: q-major order
    const int one = ob && ob[0] == '1';
    k_compact<0><<<(unsigned)grid, 256, 0, st>>>(lb, ldlb, nq, nt, key, minkey, seed2, eps_p,
                                                  items, bcount, bbase, bfill, capacity, one);
    k_bucket_scan<<<1, 32, 0, st>>>(bcount, bbase, bfill, count, capacity, cap_overflow);
    k_compact<1><<<(unsigned)grid, 256, 0, st>>>(lb, ldlb, nq, nt, key, minkey, seed2, eps_p,
                                                  items, bcount, bbase, bfill, capacity, one);
    count_launch(3, __func__);
    return 0;
}

// ---- S3 compaction from the two-stage S2's lists (lb_sparse.cu) --------------------------------
// After the two-stage S2 every pair that can survive is on a per-train-series list (its partial
// cascade value passed bsf1*(1+eps_p) >= the final threshold) with its full cascade value next to
// it, so the survivors are compacted from the lists instead of from the whole bound matrix: the
// same test (value <= thr, not a seed), the same LB buckets.  A tile = LC_W train series, one
// warp per series, lanes over the series' entries (coalesced list reads); PASS 1 runs the tile
// twice -- count, reserve a run per bucket (one global atomic per bucket and tile), scatter --
// so no per-thread slot storage is needed for lists of any length.  Inside a bucket the items are
// train-major (a query's candidates of one bucket are spread over the round).
constexpr int LC_W = 8;

template <int PASS>
__global__ void __launch_bounds__(32 * LC_W) k_list_compact(
    const long long *__restrict__ col_off, const int32_t *__restrict__ blist,
    const float *__restrict__ bval, int64_t nt, const unsigned long long *__restrict__ key,
    const unsigned long long *__restrict__ minkey, const int32_t *__restrict__ seed2, float eps_p,
    Item *__restrict__ items, unsigned long long *bucket_count,
    const unsigned long long *bucket_base, unsigned long long *bucket_fill,
    unsigned long long capacity, int one_bucket) {
    __shared__ unsigned hist[NBUCKET];
    __shared__ unsigned long long base[NBUCKET];
    const int lane = threadIdx.x & 31;
    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);
    const int64_t ntiles = (nt + LC_W - 1) / LC_W;
    // the bucket of a kept entry, or -1
    auto classify = [&](int64_t n, long long e) -> int {
        const int32_t q = blist[e];
        const float v = bval[e];
        const float thr = key_dist(key[q]) * (1.0f + eps_p);
        const unsigned s1 = (unsigned)(minkey[q] & 0xffffffffull);
        const unsigned s2 = seed2 ? (unsigned)seed2[q] : 0xffffffffu;
        if (!(v <= thr) || (unsigned)n == s1 || (unsigned)n == s2) return -1;
        const float scale = (thr > 0.0f && !one_bucket) ? (float)NBUCKET / thr : 0.0f;
        const int b = (int)(v * scale);
        return b < 0 ? 0 : (b >= NBUCKET ? NBUCKET - 1 : b);
    };
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        if (threadIdx.x < NBUCKET) hist[threadIdx.x] = 0u;
        __syncthreads();
        const int64_t n = tile * LC_W + warp;
        const long long beg = n < nt ? col_off[n] : 0, end = n < nt ? col_off[n + 1] : 0;
        for (long long e = beg + lane; e < end; e += 32) {
            const int b = classify(n, e);
            if (b >= 0) atomicAdd(&hist[b], 1u);
        }
        __syncthreads();
        if (PASS == 0) {
            if (threadIdx.x < NBUCKET && hist[threadIdx.x])
                atomicAdd(bucket_count + threadIdx.x, (unsigned long long)hist[threadIdx.x]);
        } else {
            if (threadIdx.x < NBUCKET) {
                const unsigned c = hist[threadIdx.x];
                base[threadIdx.x] = c ? bucket_base[threadIdx.x] +
                                            atomicAdd(bucket_fill + threadIdx.x, (unsigned long long)c)
                                      : 0ull;
                hist[threadIdx.x] = 0u;
            }
            __syncthreads();
            for (long long e = beg + lane; e < end; e += 32) {
                const int b = classify(n, e);
                if (b < 0) continue;
                const unsigned long long pos = base[b] + atomicAdd(&hist[b], 1u);
                if (pos < capacity) items[pos] = Item{(unsigned)blist[e], (unsigned)n, bval[e]};
            }
        }
        __syncthreads();  // hist / base are reused by the next tile
    }
}

int launch_list_compact(const long long *col_off, const int32_t *blist, const float *bval,
                        int64_t nt, const unsigned long long *key,
                        const unsigned long long *minkey, const int32_t *seed2, float eps_p,
                        Item *items, unsigned long long *count, unsigned long long *buckets,
                        unsigned long long capacity, unsigned long long *cap_overflow,
                        int num_sms, cudaStream_t st) {
    if (nt == 0) return 0;
    unsigned long long *bcount = buckets, *bbase = buckets + NBUCKET, *bfill = buckets + 2 * NBUCKET;
    const int64_t ntiles = (nt + LC_W - 1) / LC_W;
    const int64_t grid = ntiles < (int64_t)num_sms * 8 ? ntiles : (int64_t)num_sms * 8;
    static const char *ob = getenv("NNDTW_ONE_BUCKET");
    const int one = ob && ob[0] == '1';
    k_list_compact<0><<<(unsigned)grid, 32 * LC_W, 0, st>>>(col_off, blist, bval, nt, key, minkey,
                                                            seed2, eps_p, items, bcount, bbase,
                                                            bfill, capacity, one);
    k_bucket_scan<<<1, 32, 0, st>>>(bcount, bbase, bfill, count, capacity, cap_overflow);
    k_list_compact<1><<<(unsigned)grid, 32 * LC_W, 0, st>>>(col_off, blist, bval, nt, key, minkey,
                                                            seed2, eps_p, items, bcount, bbase,
                                                            bfill, capacity, one);
    count_launch(3, __func__);
    return 0;
}

// ---- in-band cells per anti-diagonal, prefix-summed (GCUPS bookkeeping) ----------------------
__global__ void k_cells_prefix(int L, int w, long long *prefix) {
    __shared__ long long tot[1024];
    const int nk = 2 * L - 1;
    const int per = (nk + blockDim.x - 1) / blockDim.x;
    const int k0 = threadIdx.x * per;
    long long s = 0;
    for (int k = k0; k < k0 + per && k < nk; ++k) {
        int lo = k - (L - 1) > 0 ? k - (L - 1) : 0;
        int t = (k - w + 1) >> 1;  // ceil((k-w)/2) for any sign
        if (t > lo) lo = t;
        int hi = k < L - 1 ? k : L - 1;
        int t2 = (k + w) >> 1;
        if (t2 < hi) hi = t2;
        s += hi >= lo ? hi - lo + 1 : 0;
    }
    tot[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long run = 0;
        for (int i = 0; i < (int)blockDim.x; ++i) {
            long long v = tot[i];
            tot[i] = run;
            run += v;
        }
    }
    __syncthreads();
    long long run = tot[threadIdx.x];
    for (int k = k0; k < k0 + per && k < nk; ++k) {
        int lo = k - (L - 1) > 0 ? k - (L - 1) : 0;
        int t = (k - w + 1) >> 1;
        if (t > lo) lo = t;
        int hi = k < L - 1 ? k : L - 1;
        int t2 = (k + w) >> 1;
        if (t2 < hi) hi = t2;
        run += hi >= lo ? hi - lo + 1 : 0;
        prefix[k] = run;
    }
}

int launch_cells_prefix(int L, int w, long long *prefix, cudaStream_t st) {
    if (w > L - 1) w = L - 1;
    k_cells_prefix<<<1, 1024, 0, st>>>(L, w, prefix);
    count_launch(1, __func__);
    return 0;
}

// ---- S7: fp64 DTW with the oracle's per-cell operation sequence --------------------------------
// d = a - b; delta = d*d; m = min(diag, left, up) (exact); D = delta + m; D(0,0) = delta;
// out-of-band cells are +inf.  Evaluation order does not change any cell's value, so the result
// is bit-identical to the oracle's row-by-row evaluation with the same operations.
// One warp per pair, row strips of 32*RR64 rows: lane l owns RR64 consecutive rows and sweeps the
// columns with a one-lane skew; the row above a lane's top row arrives by shuffle (lane l-1's
// bottom row one step earlier) or, for lane 0, from the previous strip's bottom row kept in
// shared memory (buf: L+1 doubles; buf[1+j] = D(row above, j), buf[0] = D(row above, -1)).
constexpr int RR64 = 8;

__device__ double dtw64_warp(const float *__restrict__ a, const float *__restrict__ b, int L,
                             int w, double *buf) {
    const int lane = threadIdx.x & 31;
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    const int H = 32 * RR64;
    for (int j = lane; j < L; j += 32) buf[1 + j] = INF;  // D(-1, j) = +inf
    if (lane == 0) buf[0] = 0.0;                           // D(-1,-1) = 0
    __syncwarp();
    double result = INF;
    for (int i0s = 0; i0s < L; i0s += H) {
        const int i0 = i0s + lane * RR64;
        double av[RR64], Dl[RR64];
#pragma unroll
        for (int r = 0; r < RR64; ++r) {
            av[r] = (i0 + r < L) ? (double)a[i0 + r] : 0.0;
            Dl[r] = INF;  // D(i, -1)
        }
        double up_prev = (lane == 0) ? buf[0] : INF;
        double bot = INF;
        for (int s = 0; s < L + 31; ++s) {
            const int j = s - lane;
            const double from_up = __shfl_up_sync(0xffffffffu, bot, 1);
            const bool jin = j >= 0 && j < L;
            const double bj = jin ? (double)b[j] : 0.0;
            const double rbv = (lane == 0 && jin) ? buf[1 + j] : INF;
            const double up = (lane == 0) ? rbv : from_up;
            double dgv = up_prev, upv = up;
#pragma unroll
            for (int r = 0; r < RR64; ++r) {
                const int i = i0 + r;
                const double old = Dl[r];
                double nv = INF;
                if (jin && i < L && i - j <= w && j - i <= w) {
                    const double dd = __dsub_rn(av[r], bj);
                    const double delta = __dmul_rn(dd, dd);
                    const double m = (i == 0 && j == 0) ? 0.0 : fmin(fmin(dgv, old), upv);
                    nv = __dadd_rn(delta, m);
                }
                if (jin) Dl[r] = nv;
                dgv = old;
                upv = jin ? nv : INF;
            }
            up_prev = up;
            bot = jin ? Dl[RR64 - 1] : INF;
            if (lane == 31 && jin) buf[1 + j] = bot;
            if (j == L - 1 && L - 1 >= i0 && L - 1 < i0 + RR64) {
#pragma unroll
                for (int r = 0; r < RR64; ++r)
                    if (i0 + r == L - 1) result = Dl[r];
            }
        }
        __syncwarp();
        if (lane == 0) buf[0] = INF;  // D(row above, -1) for later strips
        __syncwarp();
    }
    const int owner = ((L - 1) % H) / RR64;
    return __shfl_sync(0xffffffffu, result, owner);
}

// The same fp64 DTW by a CTA of nstrips = ceil(L / (32 RR64)) warps, warp k on strip k (rows
// 256k .. 256k+255), pipelined: warp k reads the row above its strip from rows[k] as warp k-1
// writes it (lane 31, column by column; published every 32 columns through prog[k], a
// shared-memory counter behind a block fence), and writes its own bottom row to rows[k+1].
// The cells and their operations are dtw64_warp's (bit-identical results); long series no
// longer run on one warp alone: config 4's 16 near-tie pairs (L = 2048) took 8 ms on 16 warps.
// rows: (nstrips + 1) x (L + 1) doubles; prog: nstrips ints; every thread gets the result.
__device__ double dtw64_cta(const float *__restrict__ a, const float *__restrict__ b, int L,
                            int w, double *rows, volatile int *prog, double *res) {
    const int lane = threadIdx.x & 31;
    const int k = threadIdx.x >> 5;           // strip
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    const int H = 32 * RR64;
    const int nstrips = (L + H - 1) / H;
    const int ld = L + 1;
    if (k == 0) {  // rows[0]: D(-1, j) = +inf, D(-1, -1) = 0
        for (int j = lane; j < L; j += 32) rows[1 + j] = INF;
        if (lane == 0) rows[0] = 0.0;
    }
    if (lane == 0) {
        prog[k] = (k == 0) ? L : 0;            // strip 0's row above is complete
        rows[(size_t)(k + 1) * ld] = INF;      // D(row above, -1) of strip k+1
    }
    __syncthreads();
    const double *above = rows + (size_t)k * ld;
    double *below = rows + (size_t)(k + 1) * ld;
    const int i0 = k * H + lane * RR64;
    double av[RR64], Dl[RR64];
#pragma unroll
    for (int r = 0; r < RR64; ++r) {
        av[r] = (i0 + r < L) ? (double)a[i0 + r] : 0.0;
        Dl[r] = INF;
    }
    double up_prev = (lane == 0) ? above[0] : INF;
    double bot = INF;
    double result = INF;
    int ready = 0;  // lane 0: columns of the row above known to be written
    for (int s = 0; s < L + 31; ++s) {
        const int j = s - lane;
        if (lane == 0 && j < L && j >= ready) {  // wait for warp k-1's next 32 columns
            const int need = (j + 32 < L) ? j + 32 : L;
            while (prog[k] < need) {
            }
            ready = need;
            __threadfence_block();
        }
        __syncwarp();
        const double from_up = __shfl_up_sync(0xffffffffu, bot, 1);
        const bool jin = j >= 0 && j < L;
        const double bj = jin ? (double)b[j] : 0.0;
        const double rbv = (lane == 0 && jin) ? above[1 + j] : INF;
        const double up = (lane == 0) ? rbv : from_up;
        double dgv = up_prev, upv = up;
#pragma unroll
        for (int r = 0; r < RR64; ++r) {
            const int i = i0 + r;
            const double old = Dl[r];
            double nv = INF;
            if (jin && i < L && i - j <= w && j - i <= w) {
                const double dd = __dsub_rn(av[r], bj);
                const double delta = __dmul_rn(dd, dd);
                const double m = (i == 0 && j == 0) ? 0.0 : fmin(fmin(dgv, old), upv);
                nv = __dadd_rn(delta, m);
            }
            if (jin) Dl[r] = nv;
            dgv = old;
            upv = jin ? nv : INF;
        }
        up_prev = up;
        bot = jin ? Dl[RR64 - 1] : INF;
        if (lane == 31 && jin) {
            below[1 + j] = bot;
            if (k + 1 < nstrips && ((j & 31) == 31 || j == L - 1)) {
                __threadfence_block();
                prog[k + 1] = j + 1;
            }
        }
        if (j == L - 1 && L - 1 >= i0 && L - 1 < i0 + RR64) {
#pragma unroll
            for (int r = 0; r < RR64; ++r)
                if (i0 + r == L - 1) result = Dl[r];
        }
    }
    const int owner = (L - 1) / H;  // the strip holding row L-1
    const int olane = ((L - 1) % H) / RR64;
    if (k == owner && lane == olane) *res = result;
    __syncthreads();
    const double out = *res;
    __syncthreads();  // (rows / prog / res are reused by the next pair)
    return out;
}

// Near-tie set sizes (single-shard EXACT mode): a query whose band holds one candidate needs no
// fp64 re-rank -- that candidate is the unique minimum.
__global__ void k_tie_count(const TieEntry *e, const unsigned long long *count,
                            unsigned long long cap, const unsigned long long *gkey, float eps_t,
                            unsigned *tiecnt) {
    unsigned long long n = *count;
    if (n > cap) n = cap;
    for (unsigned long long x = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (unsigned long long)gridDim.x * blockDim.x) {
        TieEntry t = e[x];
        if (t.d32 <= key_dist(gkey[t.q]) * (1.0f + eps_t)) atomicAdd(tiecnt + t.q, 1u);
    }
}

int launch_tie_count(const TieEntry *e, const unsigned long long *count, unsigned long long cap,
                     const unsigned long long *gkey, float eps_t, unsigned *tiecnt, int num_sms,
                     cudaStream_t st) {
    k_tie_count<<<num_sms * 2, 256, 0, st>>>(e, count, cap, gkey, eps_t, tiecnt);
    count_launch(1, __func__);
    return 0;
}

__global__ void k_refine(TieEntry *e, const unsigned long long *count, unsigned long long cap,
                         const float *__restrict__ A, const float *__restrict__ B, int L, int w,
                         const unsigned long long *__restrict__ gkey, float eps_t,
                         unsigned long long *f64key, unsigned long long *counters,
                         const unsigned *tiecnt, const unsigned *overflow) {
    extern __shared__ double dbuf[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    double *buf = dbuf + (size_t)warp * (L + 1);
    unsigned long long n = *count;
    if (n > cap) n = cap;
    for (unsigned long long x = (unsigned long long)blockIdx.x * wpb + warp; x < n;
         x += (unsigned long long)gridDim.x * wpb) {
        TieEntry t = e[x];
        float gb = key_dist(gkey[t.q]);
        if (t.d32 <= gb * (1.0f + eps_t)) {
            if (tiecnt != nullptr && tiecnt[t.q] == 1u && !overflow[t.q]) {
                if (lane == 0) {  // singleton band: the candidate is the answer
                    e[x].d64 = 0.0;
                    atomicMin(f64key + t.q, 0ull);
                }
                __syncwarp();
                continue;
            }
            double d = dtw64_warp(A + (int64_t)t.q * L, B + (int64_t)t.n * L, L, w, buf);
            if (lane == 0) {
                e[x].d64 = d;
                atomicMin(f64key + t.q, (unsigned long long)__double_as_longlong(d));
                if (counters) atomicAdd(counters + CNT_TIES, 1ull);
            }
        } else if (lane == 0) {
            e[x].d64 = -1.0;
        }
        __syncwarp();
    }
}

// k_refine with one CTA per entry (dtw64_cta): blockDim = 32 * nstrips
__global__ void k_refine_cta(TieEntry *e, const unsigned long long *count, unsigned long long cap,
                             const float *__restrict__ A, const float *__restrict__ B, int L,
                             int w, const unsigned long long *__restrict__ gkey, float eps_t,
                             unsigned long long *f64key, unsigned long long *counters,
                             const unsigned *tiecnt, const unsigned *overflow) {
    extern __shared__ double dsh[];
    const int nstrips = blockDim.x >> 5;
    double *rows = dsh;
    double *res = dsh + (size_t)(nstrips + 1) * (L + 1);
    volatile int *prog = (volatile int *)(res + 1);
    unsigned long long n = *count;
    if (n > cap) n = cap;
    for (unsigned long long x = blockIdx.x; x < n; x += gridDim.x) {
        TieEntry t = e[x];
        const float gb = key_dist(gkey[t.q]);
        if (t.d32 <= gb * (1.0f + eps_t)) {
            if (tiecnt != nullptr && tiecnt[t.q] == 1u && !overflow[t.q]) {
                if (threadIdx.x == 0) {  // singleton band: the candidate is the answer
                    e[x].d64 = 0.0;
                    atomicMin(f64key + t.q, 0ull);
                }
                continue;
            }
            const double d = dtw64_cta(A + (int64_t)t.q * L, B + (int64_t)t.n * L, L, w, rows,
                                       prog, res);
            if (threadIdx.x == 0) {
                e[x].d64 = d;
                atomicMin(f64key + t.q, (unsigned long long)__double_as_longlong(d));
                if (counters) atomicAdd(counters + CNT_TIES, 1ull);
            }
        } else if (threadIdx.x == 0) {
            e[x].d64 = -1.0;
        }
    }
}

// Overflowed queries (the tie log dropped an entry): every pair that survived the cascade at
// the global best is re-ranked in fp64 (rare, slow, exact).  pass 0: min fp64 -> f64key;
// pass 1: lowest index with fp64 == gf64 -> out.
__global__ void k_refine_overflow(const unsigned long long *log_count, unsigned long long log_cap,
                                  const unsigned *overflow, int64_t nq, const float *lb,
                                  int64_t ldlb, int64_t nt, const float *__restrict__ A,
                                  const float *__restrict__ B, int L, int w,
                                  const unsigned long long *gkey, float eps_p, int pass,
                                  unsigned long long *f64key, const unsigned long long *gf64,
                                  int64_t index_base, unsigned long long *out) {
    extern __shared__ double dbuf[];
    if (*log_count <= log_cap) return;  // no entry was dropped: nothing to re-rank here
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    double *buf = dbuf + (size_t)warp * (L + 1);
    for (int64_t q = 0; q < nq; ++q) {
        if (!overflow[q]) continue;
        float thr = key_dist(gkey[q]) * (1.0f + eps_p);
        for (int64_t n = (int64_t)blockIdx.x * wpb + warp; n < nt;
             n += (int64_t)gridDim.x * wpb) {
            if (!(lb[q * ldlb + n] <= thr)) continue;
            double d = dtw64_warp(A + q * L, B + n * L, L, w, buf);
            if (lane == 0) {
                unsigned long long bits = (unsigned long long)__double_as_longlong(d);
                if (pass == 0) {
                    atomicMin(f64key + q, bits);
                } else if (bits == gf64[q]) {
                    atomicMin(out + q, ((unsigned long long)(index_base + n) << 32) |
                                           (unsigned long long)__float_as_uint((float)d));
                }
            }
            __syncwarp();
        }
    }
}

static int refine_block(int L, size_t *smem) {
    int wpb = 4;
    while (wpb > 1 && (size_t)wpb * (L + 1) * sizeof(double) > 200 * 1024) wpb >>= 1;
    *smem = (size_t)wpb * (L + 1) * sizeof(double);
    return wpb * 32;
}

int launch_refine(TieEntry *e, const unsigned long long *count, unsigned long long cap,
                  const float *A, const float *B, int L, int w, const unsigned long long *gkey,
                  float eps_t, unsigned long long *f64key, unsigned long long *counters,
                  const unsigned *tiecnt, const unsigned *overflow, int num_sms,
                  cudaStream_t st) {
    if (w > L - 1) w = L - 1;
    // a CTA of one warp per 256-row strip per entry where its row buffers fit (L <= 2048-ish):
    // long series in parallel over their strips; else (or NNDTW_REFINE_CTA=0) one warp per entry
    const int nstrips = (L + 32 * RR64 - 1) / (32 * RR64);
    const size_t csmem = (size_t)(nstrips + 1) * (L + 1) * sizeof(double) + sizeof(double) +
                         (size_t)nstrips * sizeof(int);
    static const bool cta_on = [] {
        const char *e = getenv("NNDTW_REFINE_CTA");
        return !(e && e[0] == '0');
    }();
    if (cta_on && nstrips >= 2 && nstrips <= 16 && csmem <= 200 * 1024) {
        cudaFuncSetAttribute(k_refine_cta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)csmem);
        k_refine_cta<<<num_sms * 2, 32 * nstrips, csmem, st>>>(e, count, cap, A, B, L, w, gkey,
                                                                eps_t, f64key, counters, tiecnt,
                                                                overflow);
        count_launch(1, __func__);
        return 0;
    }
    size_t smem;
    int block = refine_block(L, &smem);
    cudaFuncSetAttribute(k_refine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_refine<<<num_sms * 2, block, smem, st>>>(e, count, cap, A, B, L, w, gkey, eps_t, f64key,
                                               counters, tiecnt, overflow);
    count_launch(1, __func__);
    return 0;
}

int launch_refine_overflow(const unsigned long long *log_count, unsigned long long log_cap,
                           const unsigned *overflow, int64_t nq, const float *lb, int64_t ldlb,
                           int64_t nt, const float *A, const float *B, int L, int w,
                           const unsigned long long *gkey, float eps_p, int pass,
                           unsigned long long *f64key, const unsigned long long *gf64,
                           int64_t index_base, unsigned long long *out, int num_sms,
                           cudaStream_t st) {
    if (w > L - 1) w = L - 1;
    size_t smem;
    int block = refine_block(L, &smem);
    cudaFuncSetAttribute(k_refine_overflow, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    k_refine_overflow<<<num_sms, block, smem, st>>>(log_count, log_cap, overflow, nq, lb, ldlb,
                                                    nt, A, B, L, w,
                                                    gkey, eps_p, pass, f64key, gf64,
                                                    index_base, out);
    count_launch(1, __func__);
    return 0;
}

// S7 step 2: lowest index among local candidates whose fp64 value equals the global minimum.
__global__ void k_resolve(const TieEntry *e, const unsigned long long *count,
                          unsigned long long cap, const unsigned long long *gf64,
                          int64_t index_base, unsigned long long *out) {
    unsigned long long n = *count;
    if (n > cap) n = cap;
    for (unsigned long long x = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (unsigned long long)gridDim.x * blockDim.x) {
        TieEntry t = e[x];
        if (t.d64 < 0.0) continue;
        if ((unsigned long long)__double_as_longlong(t.d64) == gf64[t.q])
            atomicMin(out + t.q, ((unsigned long long)(index_base + t.n) << 32) |
                                     (unsigned long long)__float_as_uint(t.d32));
    }
}

int launch_resolve(const TieEntry *e, const unsigned long long *count, unsigned long long cap,
                   const unsigned long long *gf64, int64_t index_base, unsigned long long *out,
                   int num_sms, cudaStream_t st) {
    k_resolve<<<num_sms * 2, 256, 0, st>>>(e, count, cap, gf64, index_base, out);
    count_launch(1, __func__);
    return 0;
}

// (idx << 32 | f32) -> (f32 << 32 | idx); keys with no candidate stay kKeyInit.
__global__ void k_swap_key(const unsigned long long *in, int64_t nq, unsigned long long *out) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    unsigned long long k = in[q];
    out[q] = (k == kNone64) ? kKeyInit : ((k << 32) | (k >> 32));
}

int launch_swap_key(const unsigned long long *in, int64_t nq, unsigned long long *out,
                    cudaStream_t st) {
    if (nq == 0) return 0;
    k_swap_key<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(in, nq, out);
    count_launch(1, __func__);
    return 0;
}

// ---- S5 decode -----------------------------------------------------------------------------
__global__ void k_finalize(const unsigned long long *key, int64_t nq, int fmt,
                           const int32_t *labels, int64_t nlabels, int64_t *idx_out,
                           int32_t *label_out, float *dist_out) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    unsigned long long k = key[q];
    unsigned idx = fmt == 0 ? (unsigned)(k & 0xffffffffull) : (unsigned)(k >> 32);
    unsigned db = fmt == 0 ? (unsigned)(k >> 32) : (unsigned)(k & 0xffffffffull);
    bool ok = (int64_t)idx < nlabels && idx != 0xffffffffu;
    if (idx_out) idx_out[q] = ok ? (int64_t)idx : -1;
    if (label_out) label_out[q] = (ok && labels) ? labels[idx] : -1;
    if (dist_out) dist_out[q] = __uint_as_float(db);
}

int launch_finalize(const unsigned long long *key, int64_t nq, int fmt, const int32_t *labels,
                    int64_t nlabels, int64_t *idx_out, int32_t *label_out, float *dist_out,
                    cudaStream_t st) {
    if (nq == 0) return 0;
    k_finalize<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(key, nq, fmt, labels, nlabels,
                                                             idx_out, label_out, dist_out);
    count_launch(1, __func__);
    return 0;
}

// ---- S8: LOOCV error count for one window ----------------------------------------------------
__global__ void k_count_errors(const unsigned long long *key, int64_t nq, const int32_t *labels,
                               int64_t q_begin, int64_t *errors, int32_t *nn_out,
                               int32_t *prev_nn) {
    __shared__ int cnt;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q < nq) {
        unsigned idx = (unsigned)(key[q] & 0xffffffffull);
        int wrong = (idx == 0xffffffffu) ? 1 : (labels[idx] != labels[q_begin + q]);
        if (wrong) atomicAdd(&cnt, 1);
        if (nn_out) nn_out[q] = (int32_t)idx;
        if (prev_nn) prev_nn[q] = (int32_t)idx;
    }
    __syncthreads();
    if (threadIdx.x == 0 && cnt) atomicAdd((unsigned long long *)errors, (unsigned long long)cnt);
}

int launch_count_errors(const unsigned long long *key, int64_t nq, const int32_t *labels,
                        int64_t q_begin, int64_t *errors, int32_t *nn_out, int32_t *prev_nn,
                        cudaStream_t st) {
    if (nq == 0) return 0;
    k_count_errors<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(key, nq, labels, q_begin,
                                                                 errors, nn_out, prev_nn);
    count_launch(1, __func__);
    return 0;
}

}  // namespace nndtw
