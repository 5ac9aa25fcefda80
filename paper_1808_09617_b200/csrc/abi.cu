// abi.cu -- host orchestration behind the C ABI of include/nndtw.h.
//
// No host synchronisation on the search path: every stage reads its work counts from device
// memory (persistent DTW grids), so nndtw_classify is a fixed sequence of kernel launches on
// the caller's stream (CUDA-graph capturable when stats == NULL).
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>

#include <cstdlib>

#include "launchers.cuh"

namespace nndtw {

static std::atomic<int64_t> g_launches{0};
void count_launch(int n, const char *who) {
    g_launches.fetch_add(n, std::memory_order_relaxed);
#ifdef NNDTW_DEBUG
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "NNDTW_DEBUG: %s -> %s\n", who ? who : "?", cudaGetErrorString(e));
        fflush(stderr);
    }
#else
    (void)who;
#endif
}
int64_t launches_total() { return g_launches.load(std::memory_order_relaxed); }

// ---- finite check (input validation for the Python layer) -----------------------------------
// Flags NaN, +-inf and |x| >= 2^36: the DTW kernels' out-of-matrix pads (+-2^64*k, see
// dtw_band.cu) must square to +inf against every real value, which holds for |x| < 2^36.
__global__ void k_check_finite(const float *x, int64_t n, int32_t *bad) {
    int found = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (!(fabsf(x[i]) < 0x1p36f)) found = 1;
    if (__any_sync(0xffffffffu, found) && (threadIdx.x & 31) == 0) *bad = 1;
}

int launch_check_finite(const float *x, int64_t n, int32_t *bad, cudaStream_t st) {
    if (n <= 0) return 0;
    int64_t grid = (n + 255) / 256;
    if (grid > 2048) grid = 2048;
    k_check_finite<<<(unsigned)grid, 256, 0, st>>>(x, n, bad);
    count_launch(1, __func__);
    return 0;
}

}  // namespace nndtw

using namespace nndtw;

static thread_local std::string g_err;

static int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

static int cuda_fail(const char *where) {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return NNDTW_OK;
    return fail(NNDTW_E_CUDA, std::string(where) + ": " + cudaGetErrorName(e) + " (" +
                                  cudaGetErrorString(e) + ")");
}

static int device_sms(int *sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cuda_fail("cudaGetDevice");
    static std::mutex mu;
    static int cache_dev = -1, cache_sms = 0, cache_ok = 0;
    std::lock_guard<std::mutex> lk(mu);
    if (cache_dev != dev) {
        int major = 0, minor = 0, n = 0;
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cache_dev = dev;
        cache_sms = n;
        cache_ok = (major == 10 && minor == 0);
    }
    *sms = cache_sms;
    if (!cache_ok) return fail(NNDTW_E_ARCH, "libnndtw is built for sm_100a (B200) only");
    return NNDTW_OK;
}

static inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// ---- classify workspace layout -----------------------------------------------------------
struct ClassifyWs {
    unsigned long long *counters;  // CNT_N + 4 (seed count, item count, log count, overflow)
    unsigned long long *seed_count, *main_count, *log_count;
    unsigned long long *cap_overflow;  // set when a survivor or list count exceeded item_cap
    unsigned long long *fb_count;      // S4 band-limited passes: items appended per level [2]
    nndtw_kim *qkim;
    unsigned long long *minkey, *f64key, *resolve_out;
    unsigned *overflow;
    unsigned *tiecnt;
    float *lb;
    int64_t ldlb;
    unsigned long long *buckets;  // survivor-order buckets: count | base | fill
    unsigned long long *split_count;  // SEARCH_B: survivors in the buckets after the split
    Item *seed_items;
    Item *items;
    unsigned long long item_cap;
    TieEntry *log;
    unsigned long long log_cap;
    long long *cells_prefix;
    long long *cells_prefix2;  // in-band cells of the band-limited pass's window
    long long *cells_prefix3;  // ... of the second band-limited pass (full windows)
    float *qU, *qL;  // query envelopes (symmetric bound)
    // two-stage S2 (lb_sparse.cu): per-train-series lists of the queries left after stage A
    long long *col_count, *col_off, *col_fill;
    float *apad;     // the band kernel's padded query rows (survivor round, GA variant)
    int64_t apad_cap;
    unsigned *colmask;  // two-stage lists: live bits per (32-query tile, train series)
    void *ed_scratch;   // ED seed (ed_seed.cu): bf16 operand images and norms
    size_t ed_bytes;
    unsigned long long *edkey;  // [nq] the ED argmin as a packed key
    int32_t *edseed;            // [nq] its train index (the first seed round's extra seed)
    int32_t *blist;  // the listed queries, train-series-major (col_off)
    float *bval;     // their full cascade values (S3 compacts from these lists)
    unsigned long long *minkey2;  // argmin of the full cascade value (second seed)
    size_t bytes;
};

static unsigned long long full_pair_cap(int64_t nq, int64_t nt) {
    return (unsigned long long)nq * (unsigned long long)nt + 1;
}

// pair_cap: entries of the survivor list and of the two-stage pair lists (full = nq*nt + 1)
static ClassifyWs classify_layout(void *base, int64_t nq, int64_t nt, int L,
                                  unsigned long long pair_cap) {
    ClassifyWs W;
    size_t off = 0;
    char *b = (char *)base;
    auto take = [&](size_t bytes) -> char * {
        char *p = b ? b + off : nullptr;
        off = align256(off + bytes);
        return p;
    };
    const size_t q1 = (size_t)(nq > 0 ? nq : 1);
    W.counters = (unsigned long long *)take(sizeof(unsigned long long) * (CNT_N + 6));
    W.seed_count = W.counters ? W.counters + CNT_N : nullptr;
    W.main_count = W.counters ? W.counters + CNT_N + 1 : nullptr;
    W.log_count = W.counters ? W.counters + CNT_N + 2 : nullptr;
    W.cap_overflow = W.counters ? W.counters + CNT_N + 3 : nullptr;
    W.fb_count = W.counters ? W.counters + CNT_N + 4 : nullptr;
    W.qkim = (nndtw_kim *)take(sizeof(nndtw_kim) * q1);
    W.minkey = (unsigned long long *)take(8 * q1);
    W.f64key = (unsigned long long *)take(8 * q1);
    W.resolve_out = (unsigned long long *)take(8 * q1);
    W.overflow = (unsigned *)take(4 * q1);
    W.tiecnt = (unsigned *)take(4 * q1);
    W.ldlb = (nt + 3) / 4 * 4;
    W.lb = (float *)take(sizeof(float) * (size_t)nq * (size_t)W.ldlb);
    W.buckets = (unsigned long long *)take(sizeof(unsigned long long) * 3 * NBUCKET);
    W.split_count = (unsigned long long *)take(sizeof(unsigned long long));
    W.seed_items = (Item *)take(sizeof(Item) * (2 * q1 + 1));
    W.item_cap = pair_cap;
    W.items = (Item *)take(sizeof(Item) * (size_t)W.item_cap);
    W.log_cap = (unsigned long long)(64 * nq > 65536 ? 64 * nq : 65536);
    if (const char *cap = getenv("NNDTW_TIE_LOG_CAP")) {  // tests: force the overflow path
        const long long c = atoll(cap);
        if (c > 0 && (unsigned long long)c < W.log_cap) W.log_cap = (unsigned long long)c;
    }
    W.log = (TieEntry *)take(sizeof(TieEntry) * (size_t)W.log_cap);
    W.cells_prefix = (long long *)take(sizeof(long long) * (size_t)(2 * L));
    W.cells_prefix2 = (long long *)take(sizeof(long long) * (size_t)(2 * L));
    W.cells_prefix3 = (long long *)take(sizeof(long long) * (size_t)(2 * L));
    W.qU = (float *)take(sizeof(float) * q1 * (size_t)L);  // symmetric bound: query envelopes
    W.qL = (float *)take(sizeof(float) * q1 * (size_t)L);
    const size_t t1 = (size_t)(nt > 0 ? nt : 1);
    W.col_count = (long long *)take(sizeof(long long) * t1);
    W.col_off = (long long *)take(sizeof(long long) * (t1 + 1));
    W.col_fill = (long long *)take(sizeof(long long) * t1);
    W.minkey2 = (unsigned long long *)take(8 * q1);
    W.apad_cap = (int64_t)q1 * band_apad_row_floats(L);
    W.apad = (float *)take(sizeof(float) * (size_t)W.apad_cap);
    W.colmask = (unsigned *)take(sizeof(unsigned) * ((q1 + 31) / 32) * t1);
    W.ed_bytes = ed_seed_supported(L) ? ed_seed_scratch_bytes((int64_t)q1, (int64_t)t1, L) : 0;
    W.ed_scratch = take(W.ed_bytes);
    W.edkey = (unsigned long long *)take(8 * q1);
    W.edseed = (int32_t *)take(4 * q1);
    W.blist = (int32_t *)take(sizeof(int32_t) * (size_t)W.item_cap);
    W.bval = (float *)take(sizeof(float) * (size_t)W.item_cap);
    W.bytes = off;
    return W;
}

static ClassifyWs classify_layout(void *base, int64_t nq, int64_t nt, int L) {
    return classify_layout(base, nq, nt, L, full_pair_cap(nq, nt));
}

// The layout a workspace of ws_bytes holds: the full one (every pair can be a survivor) when it
// fits, else the largest pair capacity that does (nndtw_classify_workspace_bytes_capped).  A
// call whose survivors or listed pairs exceed the capacity sets the overflow word
// (nndtw_classify_overflowed); its keys are then not valid and the caller reruns it with more.
static ClassifyWs classify_layout_for(void *base, int64_t nq, int64_t nt, int L, size_t ws_bytes) {
    const unsigned long long full = full_pair_cap(nq, nt);
    ClassifyWs W = classify_layout(base, nq, nt, L, full);
    if (ws_bytes >= W.bytes) return W;
    const size_t fixed = classify_layout(nullptr, nq, nt, L, 0).bytes;
    const size_t per_pair = sizeof(Item) + sizeof(int32_t) + sizeof(float);
    if (ws_bytes <= fixed) return W;  // too small for any capacity: reported by the caller
    // the largest capacity that fits (alignment: each of the three arrays rounds up to 256 B,
    // so this starts at most a few dozen above it; the layout size grows with the capacity)
    unsigned long long cap = (unsigned long long)((ws_bytes - fixed) / per_pair);
    if (cap >= full) cap = full - 1;
    while (cap > 0 && classify_layout(nullptr, nq, nt, L, cap).bytes > ws_bytes) --cap;
    if (cap < 2ull * (unsigned long long)nq + 2ull) return W;  // (not even the seed rounds)
    return classify_layout(base, nq, nt, L, cap);
}

static int check_common(int64_t n, int L, int w) {
    if (n < 0) return fail(NNDTW_E_ARG, "negative count");
    if (L < 2) return fail(NNDTW_E_LENGTH, "L must be >= 2 (Algorithm 1 needs L >= 2)");
    if (L > 8192) return fail(NNDTW_E_LENGTH, "L > 8192 is not supported");
    if (w < 0) return fail(NNDTW_E_WINDOW, "w must be >= 0");
    return NNDTW_OK;
}

static int dtw_fail(int rc, int L, int w) {
    if (rc == 0) return NNDTW_OK;
    return fail(NNDTW_E_WINDOW, "no DTW kernel for L=" + std::to_string(L) +
                                    " w=" + std::to_string(w));
}

struct StageTimer {
    bool on;
    cudaStream_t st;
    cudaEvent_t ev[8];
    int n = 0;
    StageTimer(bool on_, cudaStream_t s) : on(on_), st(s) {
        if (on)
            for (auto &e : ev) cudaEventCreate(&e);
    }
    void mark() {
        if (on && n < 8) cudaEventRecord(ev[n++], st);
    }
    float ms(int a, int b) {
        float m = 0;
        if (on && b < n) cudaEventElapsedTime(&m, ev[a], ev[b]);
        return m;
    }
    ~StageTimer() {
        if (on)
            for (auto &e : ev) cudaEventDestroy(e);
    }
};

// S7 for one shard whose local best is the global best (single GPU, LOOCV).
static void exact_local(ClassifyWs &W, const float *q, int64_t nq, const float *t, int64_t nt,
                        int L, int w, int64_t index_base, unsigned long long *key,
                        unsigned long long *cnt, int sms, cudaStream_t st) {
    const float eps_p = eps_prune(L), eps_t = eps_tie(L);
    launch_tie_count(W.log, W.log_count, W.log_cap, key, eps_t, W.tiecnt, sms, st);
    launch_refine(W.log, W.log_count, W.log_cap, q, t, L, w, key, eps_t, W.f64key, cnt,
                  W.tiecnt, W.overflow, sms, st);
    launch_refine_overflow(W.log_count, W.log_cap, W.overflow, nq, W.lb, W.ldlb, nt, q, t, L, w, key, eps_p, 0,
                           W.f64key, nullptr, index_base, nullptr, sms, st);
    launch_resolve(W.log, W.log_count, W.log_cap, W.f64key, index_base, W.resolve_out, sms, st);
    launch_refine_overflow(W.log_count, W.log_cap, W.overflow, nq, W.lb, W.ldlb, nt, q, t, L, w, key, eps_p, 1,
                           W.f64key, W.f64key, index_base, W.resolve_out, sms, st);
    launch_swap_key(W.resolve_out, nq, key, st);
}

// The band-limited S4 pass in front of the row-strip kernel (full windows, band wb <= w / 8):
// on where that band is at least 103 offsets wide (long series: config 4, L = 2048, wb = 207:
// 11.7 k -> 14.0 k queries/s); at L = 256 (config 1, wb = 25) it was slower (1.03 -> 0.94 M
// queries/s at w = 255).  NNDTW_ADAPT_FULL=0/1 forces it off/on.
static bool second_band_level() {  // experiments: NNDTW_ADAPT_LEVELS=2
    const char *e = getenv("NNDTW_ADAPT_LEVELS");
    return e && e[0] == '2';
}

static int full_window_band(int L, int w) {
    const int wb = band_adapt_window(L, w, true);
    const char *e = getenv("NNDTW_ADAPT_FULL");
    if (e) return e[0] == '1' ? wb : -1;
    return wb >= 103 ? wb : -1;
}

// Core of nndtw_classify (also used per window by nndtw_loocv_window).
static int classify_impl(const float *q, int64_t nq, const float *t, const float *U,
                         const float *Lo, const nndtw_kim *tkim, int64_t nt, int64_t index_base,
                         int64_t self_offset, int L, int w, int v, uint32_t flags,
                         const int32_t *seed2_in, void *ws, size_t ws_bytes,
                         unsigned long long *key, nndtw_stats *stats, cudaStream_t st,
                         StageTimer *outer_tm = nullptr) {
    int sms = 0;
    int rc = device_sms(&sms);
    if (rc) return rc;
    if ((rc = check_common(nq, L, w))) return rc;
    if (nt < 0) return fail(NNDTW_E_ARG, "negative nt");
    if (v < 1) return fail(NNDTW_E_V, "V must be >= 1");
    if (w > L - 1) w = L - 1;
    if (nq > 0 && (!q || !key || !ws)) return fail(NNDTW_E_ARG, "null pointer argument");
    if (nt > 0 && (!t || !U || !Lo || !tkim)) return fail(NNDTW_E_ARG, "null pointer argument");
    if (index_base < 0 || index_base + nt > 0x7fffffffll)
        return fail(NNDTW_E_INDEX, "global train indices must be < 2^31 (signed int64 shard "
                                   "combine of (index << 32) keys)");
    ClassifyWs W = classify_layout_for(ws, nq, nt, L, ws_bytes);
    if (ws_bytes < W.bytes) return fail(NNDTW_E_WORKSPACE, "workspace too small");
    if (nq == 0) return NNDTW_OK;
    const int64_t launches0 = launches_total();
    StageTimer tm(stats != nullptr && outer_tm == nullptr, st);
    const float eps_p = eps_prune(L), eps_t = eps_tie(L);

    // Phases (sharded search, dist.py): SEED = init + S2 bound + S3 seed round, leaving the state
    // in ws; SEARCH = S3 compaction + S4/S5 survivors against the key passed in (the MIN over
    // shards of the seed keys), or the same in two halves SEARCH_A (compaction + the survivors
    // of buckets < split) and SEARCH_B (the rest), with another MIN over shards in between.
    // No phase flag: everything, in one call.
    const unsigned phases = flags & (NNDTW_CLASSIFY_PHASE_SEED | NNDTW_CLASSIFY_PHASE_SEARCH |
                                     NNDTW_CLASSIFY_PHASE_SEARCH_A | NNDTW_CLASSIFY_PHASE_SEARCH_B);
    const bool all = phases == 0;
    const bool do_seed = all || (flags & NNDTW_CLASSIFY_PHASE_SEED);
    const bool whole = all || (flags & NNDTW_CLASSIFY_PHASE_SEARCH) ||
                       ((flags & NNDTW_CLASSIFY_PHASE_SEARCH_A) && (flags & NNDTW_CLASSIFY_PHASE_SEARCH_B));
    const bool do_compact = whole || (flags & NNDTW_CLASSIFY_PHASE_SEARCH_A);
    const bool dtw_a = !whole && (flags & NNDTW_CLASSIFY_PHASE_SEARCH_A);
    const bool dtw_b = !whole && (flags & NNDTW_CLASSIFY_PHASE_SEARCH_B);
    const bool do_finish = whole || dtw_b;              // S5/S7 after the last survivors
    static const int split_b = [] {
        const char *e = getenv("NNDTW_SPLIT_BUCKET");  // experiments: the SEARCH_A/B split
        const int b = e ? atoi(e) : NBUCKET / 4;
        return b < 0 ? 0 : (b > NBUCKET ? NBUCKET : b);
    }();
    const int keogh = (flags & NNDTW_CLASSIFY_BOUND_KEOGH) ? 1 : 0;
    const bool sym = (flags & NNDTW_CLASSIFY_BOUND_SYMMETRIC) != 0;
    // alternative S2 bounds (NEXT-1 / NEXT-4): assembled outside the tile kernel, then finished
    const uint32_t alt = flags & (NNDTW_CLASSIFY_BOUND_IMPROVED | NNDTW_CLASSIFY_BOUND_NEW |
                                  NNDTW_CLASSIFY_BOUND_ENHANCED_IMPROVED |
                                  NNDTW_CLASSIFY_BOUND_NONE);
    if (alt & (alt - 1)) return fail(NNDTW_E_ARG, "more than one alternative bound flag");
    if (alt && (keogh || sym))
        return fail(NNDTW_E_ARG, "an alternative bound cannot be combined with KEOGH/SYMMETRIC");
    const bool alt_none = (alt & NNDTW_CLASSIFY_BOUND_NONE) != 0;
    // cascade levels for the level counters: band level only where Algorithm 1's bands exist
    const int count_no_bands = (keogh || (alt && !(alt & NNDTW_CLASSIFY_BOUND_ENHANCED_IMPROVED)))
                                   ? 1 : 0;
    // Two-stage S2 for the default cascade (lb_sparse.cu): stage A = LB_Kim + Algorithm 1's
    // bands for all pairs, a seed round, stage B = the bridge only for the pairs the partial
    // cascade kept, a second seed round.
    // Used where it pays: enough bridge work (nq*nt*(L - 2nb) >= 2^33 pair-columns, ~0.7 ms
    // of the one-stage tile kernel) to cover its extra seed round and lists, and rows that fit
    // the sparse kernel's register path (L <= 1024).  NNDTW_S2_STAGES=1 / =2 forces one / two
    // stages (tests, experiments; read per call -- keep it fixed across the phases of one
    // sharded classify: the search phase compacts from the seed phase's lists).
    const int nb_ = (L / 2) < v ? (L / 2) : v;
    bool two_stage = !alt && !sym && !keogh && nb_ >= 1 && nb_ <= 16 && L <= 1024 &&
                     (double)nq * (double)nt * (double)(L - 2 * nb_) >= 8589934592.0;
    if (const char *e = getenv("NNDTW_S2_STAGES")) {
        if (e[0] == '1') two_stage = false;
        if (e[0] == '2') two_stage = !alt && !sym && !keogh && nb_ >= 1 && nb_ <= 16;
    }
    // Euclidean-nearest first seed (ed_seed.cu; the paper's candidate order): in the
    // two-stage path, when the caller gives no seed of its own (LOOCV passes the previous
    // window's neighbour), there is no leave-one-out self pair (the ED argmin would be the
    // held-out series itself) and the rows fit the tensor-core kernel.  NNDTW_ED_SEED=0 disables
    // it (experiments; read per call -- keep it fixed across the phases of one sharded classify).
    bool ed_seed = two_stage && seed2_in == nullptr && self_offset < 0 && ed_seed_supported(L) &&
                   nt > 0;
    if (const char *e = getenv("NNDTW_ED_SEED"))
        if (e[0] == '0') ed_seed = false;
    const int32_t *seed2 = ed_seed ? W.edseed : seed2_in;
    TieLog log{W.log, W.log_count, W.log_cap, W.overflow};
    unsigned long long *cnt = stats ? W.counters : nullptr;

    tm.mark();  // 0
    if (do_seed) {
        launch_classify_init(nq, key, W.minkey, W.f64key, W.resolve_out, W.overflow, W.tiecnt,
                             W.counters, CNT_N + 6, W.buckets, st);
        launch_cells_prefix(L, w, W.cells_prefix, st);
    }
    tm.mark();  // 1
    if (do_seed) {  // query-side S1: Kim features (+ envelopes for the symmetric bound)
        launch_series_stats(q, nq, L, W.qkim, st);
        if (nt > 0 && sym) launch_envelopes(q, nq, L, w, W.qU, W.qL, nullptr, st);
    }
    tm.mark();  // 2
    if (do_seed && nt > 0 && alt) {
        // S2 with an alternative bound: matrix, then max with LB_Kim / self pair / argmin seed
        int lrc = 0;
        if (alt & NNDTW_CLASSIFY_BOUND_IMPROVED) {
            lrc = launch_lb(q, nq, nullptr, t, U, Lo, nullptr, nt, L, w, v, 0, -1, W.lb, W.ldlb,
                            nullptr, st, 1) ||
                  launch_lb_improved_pass(q, nq, t, U, Lo, nt, L, w, 0, L, W.lb, W.ldlb, sms, st);
        } else if (alt & NNDTW_CLASSIFY_BOUND_ENHANCED_IMPROVED) {
            const int nb = (L / 2) < v ? (L / 2) : v;
            lrc = launch_lb(q, nq, nullptr, t, U, Lo, nullptr, nt, L, w, v, 0, -1, W.lb, W.ldlb,
                            nullptr, st, 0) ||
                  launch_lb_improved_pass(q, nq, t, U, Lo, nt, L, w, nb, L - nb, W.lb, W.ldlb, sms,
                                          st);
        } else if (alt & NNDTW_CLASSIFY_BOUND_NEW) {
            lrc = launch_lb_pairs(0, q, nq, t, nullptr, nullptr, nt, L, w, W.lb, W.ldlb, st);
        } else {  // BOUND_NONE: the bound is 0 for every pair
            cudaMemsetAsync(W.lb, 0, sizeof(float) * (size_t)nq * (size_t)W.ldlb, st);
        }
        if (lrc) return fail(NNDTW_E_ARG, "bound kernel launch failed (shape)");
        launch_bound_finish(W.lb, W.ldlb, nq, nt, q, t, alt_none ? nullptr : W.qkim, tkim, L,
                            self_offset, W.minkey, st);
    }
    // (level counters read the full cascade values from the bound matrix: with them on, the
    // two-stage S2 writes those there too -- pass the flag to the seed phase as well)
    const bool level_stats = stats != nullptr && (flags & NNDTW_CLASSIFY_LEVEL_STATS) != 0;
    StageTimer bridge_tm(stats != nullptr && outer_tm == nullptr && two_stage, st);
    long long bridge_pairs_h = 0;
    if (do_seed && two_stage && nt > 0) {
        if (ed_seed) {  // the ED argmin joins the first seed round
            cudaMemsetAsync(W.edkey, 0xff, 8 * (size_t)nq, st);
            if (launch_ed_seed(q, nq, t, nt, L, W.ed_scratch, W.edkey, sms, st))
                return fail(NNDTW_E_ARG, "ED seed launch failed");
            launch_key_index(W.edkey, nq, nt, W.edseed, st);
        }
        // stage A: max(LB_Kim, boundary + bands) for all pairs + its argmin (first seed)
        if (launch_lb(q, nq, W.qkim, t, U, Lo, tkim, nt, L, w, v, 1, self_offset, W.lb, W.ldlb,
                      W.minkey, st, 0, 0, 1))
            return fail(NNDTW_E_ARG, "too many train series for one launch");
        // first seed round -> best-so-far bsf1 in key
        launch_seed_items(W.minkey, seed2, nq, nt, W.seed_items, W.seed_count, st);
        rc = dispatch_dtw(q, t, nq, nt, W.seed_items, W.seed_count, 2 * (unsigned long long)nq + 1,
                          nullptr, nullptr, 0, L, w, 0, key, index_base, eps_t, log, nullptr,
                          W.cells_prefix, nullptr, nullptr, st, sms);
        if ((rc = dtw_fail(rc, L, w))) return rc;
        // stage B: the pairs Algorithm 1's line-12 test keeps (P <= bsf1*(1+eps_p)), per train
        // series, and the full cascade value for them (+ its argmin: the second seed)
        launch_col_compact(W.lb, W.ldlb, nq, nt, key, eps_p, W.col_count, W.col_off, W.col_fill,
                           W.blist, W.item_cap, W.colmask, W.cap_overflow, sms, st);
        cudaMemsetAsync(W.minkey2, 0xff, 8 * (size_t)nq, st);
        if (bridge_tm.on) cudaEventRecord(bridge_tm.ev[0], st);
        if (launch_lb_sparse(q, W.qkim, nq, t, U, Lo, tkim, nt, L, w, v, W.col_off,
                             W.blist, W.bval, level_stats ? W.lb : nullptr, W.ldlb, W.minkey2,
                             sms, st))
            return fail(NNDTW_E_ARG, "sparse bridge launch failed");
        if (bridge_tm.on) {
            cudaEventRecord(bridge_tm.ev[1], st);
            bridge_tm.n = 2;
        }
        if (stats) cudaMemcpyAsync(&bridge_pairs_h, W.col_off + nt, 8, cudaMemcpyDeviceToHost, st);
        // second seed round: the full-cascade argmin where it differs from the first seeds
        launch_seed_items2(W.minkey2, W.minkey, seed2, nq, nt, W.seed_items,
                           W.counters + CNT_SEED2, st);
        rc = dispatch_dtw(q, t, nq, nt, W.seed_items, W.counters + CNT_SEED2,
                          2 * (unsigned long long)nq + 1, nullptr, nullptr, 0, L, w, 0, key,
                          index_base, eps_t, log, nullptr, W.cells_prefix, nullptr, nullptr, st,
                          sms);
        if ((rc = dtw_fail(rc, L, w))) return rc;
        // the compaction and the level counters exclude the full-cascade argmin (and seed2)
        cudaMemcpyAsync(W.minkey, W.minkey2, 8 * (size_t)nq, cudaMemcpyDeviceToDevice, st);
    }
    if (do_seed && !alt && !two_stage) {
        // S2: cascade bound for all pairs + per-query argmin-LB candidate
        if (nt > 0 && launch_lb(q, nq, W.qkim, t, U, Lo, tkim, nt, L, w, v, 1, self_offset,
                                W.lb, W.ldlb, sym ? nullptr : W.minkey, st, keogh))
            return fail(NNDTW_E_ARG, "too many train series for one launch");
        if (nt > 0 && sym) {  // second direction of the symmetric bound, then the seed argmin
            if (launch_lb(t, nt, nullptr, q, W.qU, W.qL, nullptr, nq, L, w, v, 0, -1, W.lb,
                          W.ldlb, nullptr, st, keogh, 1))
                return fail(NNDTW_E_ARG, "too many queries for one launch");
            launch_row_argmin(W.lb, W.ldlb, nq, nt, W.minkey, st);
        }
    }
    tm.mark();  // 3
    if ((rc = cuda_fail("lb"))) return rc;
    if (nt > 0 && do_seed && !two_stage) {
        // S3: seed round (argmin-LB candidate, plus seed2 if given)
        launch_seed_items(W.minkey, seed2, nq, nt, W.seed_items, W.seed_count, st);
        rc = dispatch_dtw(q, t, nq, nt, W.seed_items, W.seed_count, 2 * (unsigned long long)nq + 1,
                          nullptr, nullptr, 0, L, w, 0, key, index_base, eps_t, log, nullptr,
                          W.cells_prefix, nullptr, nullptr, st, sms);
        if ((rc = dtw_fail(rc, L, w))) return rc;
    }
    if (nt > 0 && do_compact && level_stats) {
        // stats: pairs pruned per cascade level against the same threshold as the compaction
        launch_lb_level_counts(q, nq, W.qkim, t, tkim, nt, L, w, v, alt_none ? 0 : 1,
                               count_no_bands, self_offset, W.lb, W.ldlb, key, W.minkey, seed2,
                               eps_p, W.counters + CNT_PRUNED_KIM, st);
    }
    if (nt > 0 && do_compact && two_stage) {
        // S3 from the two-stage lists (every possible survivor is listed, with its full value)
        launch_list_compact(W.col_off, W.blist, W.bval, nt, key, W.minkey, seed2, eps_p, W.items,
                            W.main_count, W.buckets, W.item_cap, W.cap_overflow, sms, st);
    } else if (nt > 0 && do_compact) {
        // S3: prune + compact the survivors against the seeded best-so-far
        launch_compact(W.lb, W.ldlb, nq, nt, key, W.minkey, seed2, eps_p, W.items,
                       W.main_count, W.buckets, W.item_cap, W.cap_overflow, sms, st);
    }
    tm.mark();  // 4
    if (nt > 0 && whole) {
        // S4/S5: DTW with early abandoning on the survivors.  Wide windows first run the
        // band-limited pass (window wb < w): exact for every
        // item whose band edges stay above the threshold; the others are appended after the
        // survivors and rerun with the full window below.
        // (not for the no-bound baseline: every pair is a survivor there, against a loose
        // early best-so-far, and a tenth of them fell back -- 96 -> 195 ms on config 2)
        const int kind = dtw_kernel_kind(L, w);
        const int wb = alt_none ? -1
                                : kind == 1 ? band_adapt_window(L, w)
                                            : kind == 2 ? full_window_band(L, w) : -1;
        int levels = 0;
        if (wb >= 0) {
            launch_cells_prefix(L, wb, W.cells_prefix2, st);
            cudaMemsetAsync(W.fb_count, 0, 2 * sizeof(unsigned long long), st);
            if (dispatch_dtw(q, t, nq, nt, W.items, W.main_count, W.item_cap, nullptr, nullptr, 0,
                             L, w, 0, key, index_base, eps_t, log, cnt, W.cells_prefix2, nullptr,
                             nullptr, st, sms, W.apad, W.apad_cap, wb, W.items, W.fb_count,
                             0) == 0)
                levels = 1;
            // full windows: a second band, twice as wide, for the items the first sends back
            const int wb2 = 2 * wb + 1;
            if (levels == 1 && kind == 2 && second_band_level() && wb2 < w) {
                launch_cells_prefix(L, wb2, W.cells_prefix3, st);
                if (dispatch_dtw(q, t, nq, nt, W.items, W.main_count, W.item_cap, nullptr,
                                 nullptr, 0, L, w, 0, key, index_base, eps_t, log, cnt,
                                 W.cells_prefix3, nullptr, nullptr, st, sms, W.apad, W.apad_cap,
                                 wb2, W.items, W.fb_count, 1) == 0)
                    levels = 2;
            }
        }
        rc = dispatch_dtw(q, t, nq, nt, W.items, W.main_count, W.item_cap, nullptr, nullptr, 0, L, w, 0,
                          key, index_base, eps_t, log, cnt, W.cells_prefix, nullptr, nullptr,
                          st, sms, W.apad, W.apad_cap, -1, nullptr,
                          levels ? W.fb_count : nullptr, levels);
        if ((rc = dtw_fail(rc, L, w))) return rc;
    } else if (nt > 0 && dtw_a) {
        // the survivors of buckets < split_b: items [0, base[split_b]) (the bucket-major list)
        const unsigned long long *na = split_b < NBUCKET ? W.buckets + NBUCKET + split_b
                                                         : W.main_count;
        rc = dispatch_dtw(q, t, nq, nt, W.items, na, W.item_cap, nullptr, nullptr, 0, L, w, 0,
                          key, index_base, eps_t, log, cnt, W.cells_prefix, nullptr, nullptr,
                          st, sms, W.apad, W.apad_cap);
        if ((rc = dtw_fail(rc, L, w))) return rc;
    } else if (nt > 0 && dtw_b) {
        // the rest: items [base[split_b], total) -- the offset is read on the host
        unsigned long long h[2] = {0ull, 0ull};
        if (split_b < NBUCKET)
            cudaMemcpyAsync(&h[0], W.buckets + NBUCKET + split_b, 8, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(&h[1], W.main_count, 8, cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_fail("classify split sync");
        unsigned long long total = h[1] < W.item_cap ? h[1] : W.item_cap;
        const unsigned long long a = split_b < NBUCKET ? (h[0] < total ? h[0] : total) : total;
        const unsigned long long nbrest = total - a;
        cudaMemcpyAsync(W.split_count, &nbrest, 8, cudaMemcpyHostToDevice, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_fail("classify split sync");
        if (nbrest > 0) {
            rc = dispatch_dtw(q, t, nq, nt, W.items + a, W.split_count, W.item_cap - a, nullptr,
                              nullptr, 0, L, w, 0, key, index_base, eps_t, log, cnt,
                              W.cells_prefix, nullptr, nullptr, st, sms, W.apad, W.apad_cap);
            if ((rc = dtw_fail(rc, L, w))) return rc;
        }
    }
    tm.mark();  // 5
    if ((rc = cuda_fail("dtw"))) return rc;
    if ((flags & NNDTW_CLASSIFY_EXACT) && nt > 0 && do_finish)
        exact_local(W, q, nq, t, nt, L, w, index_base, key, cnt, sms, st);
    tm.mark();  // 6
    if ((rc = cuda_fail("classify"))) return rc;
    if (stats) {
        unsigned long long h[CNT_N + 3];
        cudaMemcpyAsync(h, W.counters, sizeof h, cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_fail("classify sync");
        if (do_seed) {
            stats->lb_pairs += nq * nt;
            stats->rounds += 1;
        }
        // (the counters accumulate from the seed phase on: the call that finishes the survivor
        // round reports them once)
        if (do_compact) stats->survivors += (int64_t)h[CNT_N + 1];
        if (do_seed) stats->bridge_pairs += two_stage ? (int64_t)bridge_pairs_h : nq * nt;
#ifdef NNDTW_PROFILE_SETUP
        if (do_finish)
            fprintf(stderr, "NNDTW_PROFILE_SETUP setup_cycles %llu warp_cycles %llu share %.4f\n",
                    h[6], h[7], h[7] ? (double)h[6] / (double)h[7] : 0.0);
#endif
        if (do_compact && level_stats) {
            stats->pruned_kim = (stats->pruned_kim < 0 ? 0 : stats->pruned_kim) + (int64_t)h[CNT_PRUNED_KIM];
            stats->pruned_bands = (stats->pruned_bands < 0 ? 0 : stats->pruned_bands) + (int64_t)h[CNT_PRUNED_BANDS];
            stats->pruned_keogh = (stats->pruned_keogh < 0 ? 0 : stats->pruned_keogh) + (int64_t)h[CNT_PRUNED_KEOGH];
        }
        if (do_finish) {
            stats->dtw_calls += (int64_t)h[CNT_ITEMS] + (int64_t)h[CNT_N] +
                                (int64_t)h[CNT_SEED2];  // main + seed items (both rounds)
            stats->dtw_abandoned += (int64_t)h[CNT_ABANDONED];
            stats->cells += (int64_t)h[CNT_CELLS];
            stats->near_tie_pairs += (int64_t)h[CNT_TIES];
            stats->dtw_fallback += (int64_t)h[CNT_FALLBACK];
            stats->rounds += 1;
        }
        stats->launches += (int32_t)(launches_total() - launches0);
        if (outer_tm == nullptr) {
            stats->ms_envelopes += tm.ms(1, 2);
            stats->ms_lb += tm.ms(2, 3);
            stats->ms_dtw += tm.ms(4, 5);
            stats->ms_other += tm.ms(0, 1) + tm.ms(3, 4) + tm.ms(5, 6);
            stats->ms_lb_bridge += bridge_tm.ms(0, 1);
        }
    }
    return NNDTW_OK;
}

// ---- LOOCV workspace ---------------------------------------------------------------------
struct LoocvWs {
    float *U, *Lo;
    nndtw_kim *kim;
    int32_t *prev_nn;
    unsigned long long *key;
    void *cws;
    size_t cws_bytes;
    size_t bytes;
};

static LoocvWs loocv_layout(void *base, int64_t n, int L, int64_t nq) {
    LoocvWs W;
    size_t off = 0;
    char *b = (char *)base;
    auto take = [&](size_t bytes) -> char * {
        char *p = b ? b + off : nullptr;
        off = align256(off + bytes);
        return p;
    };
    const size_t q1 = (size_t)(nq > 0 ? nq : 1);
    W.U = (float *)take(sizeof(float) * (size_t)n * L);
    W.Lo = (float *)take(sizeof(float) * (size_t)n * L);
    W.kim = (nndtw_kim *)take(sizeof(nndtw_kim) * (size_t)(n > 0 ? n : 1));
    W.prev_nn = (int32_t *)take(4 * q1);
    W.key = (unsigned long long *)take(8 * q1);
    W.cws_bytes = classify_layout(nullptr, nq, n, L).bytes;
    W.cws = take(W.cws_bytes);
    W.bytes = off;
    return W;
}

extern "C" {

const char *nndtw_last_error(void) { return g_err.c_str(); }
int nndtw_version(void) { return 2; }

const char *nndtw_dtw_kernel_name(int32_t L, int32_t w) {
    if (L < 2 || w < 0) return "";
    static const char *names[3] = {"k_dtw_w0", "k_dtw_band", "k_dtw_strip"};
    return names[dtw_kernel_kind(L, w)];
}
int32_t nndtw_band_limited_window(int32_t L, int32_t w) {
    if (L < 2 || w < 0) return -1;
    if (w > L - 1) w = L - 1;
    const int kind = dtw_kernel_kind(L, w);
    return kind == 1 ? band_adapt_window(L, w) : kind == 2 ? full_window_band(L, w) : -1;
}
int64_t nndtw_launch_count(void) { return launches_total(); }

int nndtw_check_device(void) {
    int sms;
    return device_sms(&sms);
}

int nndtw_check_finite(const float *x, int64_t n, int32_t *bad, void *stream) {
    int sms, rc;
    if ((rc = device_sms(&sms))) return rc;
    if (n < 0 || (n > 0 && (!x || !bad))) return fail(NNDTW_E_ARG, "bad arguments");
    launch_check_finite(x, n, bad, (cudaStream_t)stream);
    return cuda_fail("nndtw_check_finite");
}

int nndtw_envelopes(const float *x, int64_t n, int32_t L, int32_t w, float *upper,
                    float *lower, nndtw_kim *kim, void *stream) {
    int sms, rc;
    if ((rc = device_sms(&sms))) return rc;
    if (n < 0) return fail(NNDTW_E_ARG, "negative count");
    if (L < 1 || L > 8192) return fail(NNDTW_E_LENGTH, "L must be in [1, 8192]");
    if (w < 0) return fail(NNDTW_E_WINDOW, "w must be >= 0");
    if (n > 0 && (!x || !upper || !lower)) return fail(NNDTW_E_ARG, "null pointer argument");
    if (launch_envelopes(x, n, L, w, upper, lower, kim, (cudaStream_t)stream))
        return fail(NNDTW_E_LENGTH, "unsupported envelope shape");
    return cuda_fail("nndtw_envelopes");
}

int nndtw_series_stats(const float *x, int64_t n, int32_t L, nndtw_kim *kim, void *stream) {
    int sms, rc;
    if ((rc = device_sms(&sms))) return rc;
    if (n < 0 || (n > 0 && (!x || !kim))) return fail(NNDTW_E_ARG, "bad arguments");
    if (L < 1) return fail(NNDTW_E_LENGTH, "L must be >= 1");
    launch_series_stats(x, n, L, kim, (cudaStream_t)stream);
    return cuda_fail("nndtw_series_stats");
}

int nndtw_lb_enhanced(const float *q, int64_t nq, const nndtw_kim *qkim, const float *t,
                      const float *upper, const float *lower, const nndtw_kim *tkim,
                      int64_t nt, int32_t L, int32_t w, int32_t v, uint32_t flags, float *lb,
                      int64_t ldlb, void *stream) {
    int sms, rc;
    if ((rc = device_sms(&sms))) return rc;
    if ((rc = check_common(nq, L, w))) return rc;
    if (nt < 0) return fail(NNDTW_E_ARG, "negative nt");
    if (v < 1) return fail(NNDTW_E_V, "V must be >= 1");
    if (ldlb < nt) return fail(NNDTW_E_ARG, "ldlb < nt");
    bool kim = (flags & NNDTW_LB_WITH_KIM) != 0;
    if (nq > 0 && nt > 0 && (!q || !t || !upper || !lower || !lb || (kim && (!qkim || !tkim))))
        return fail(NNDTW_E_ARG, "null pointer argument");
    const int partial = (flags & NNDTW_LB_PARTIAL) ? 1 : 0;
    if (partial && (flags & NNDTW_LB_KEOGH))
        return fail(NNDTW_E_ARG, "NNDTW_LB_PARTIAL cannot be combined with NNDTW_LB_KEOGH");
    if (launch_lb(q, nq, qkim, t, upper, lower, tkim, nt, L, w, v, kim ? 1 : 0, -1, lb, ldlb,
                  nullptr, (cudaStream_t)stream, (flags & NNDTW_LB_KEOGH) ? 1 : 0, 0, partial))
        return fail(NNDTW_E_ARG, "too many train series for one launch");
    return cuda_fail("nndtw_lb_enhanced");
}

int nndtw_lb_enhanced_symmetric(const float *q, const float *q_upper, const float *q_lower,
                                const nndtw_kim *qkim, int64_t nq, const float *t,
                                const float *t_upper, const float *t_lower,
                                const nndtw_kim *tkim, int64_t nt, int32_t L, int32_t w,
                                int32_t v, uint32_t flags, float *lb, int64_t ldlb,
                                void *stream) {
    int sms, rc;
    if ((rc = device_sms(&sms))) return rc;
    if ((rc = check_common(nq, L, w))) return rc;
    if (nt < 0) return fail(NNDTW_E_ARG, "negative nt");
    if (v < 1) return fail(NNDTW_E_V, "V must be >= 1");
    if (ldlb < nt) return fail(NNDTW_E_ARG, "ldlb < nt");
    bool kim = (flags & NNDTW_LB_WITH_KIM) != 0;
    if (nq > 0 && nt > 0 && (!q || !q_upper || !q_lower || !t || !t_upper || !t_lower || !lb ||
                             (kim && (!qkim || !tkim))))
        return fail(NNDTW_E_ARG, "null pointer argument");
    const int keogh = (flags & NNDTW_LB_KEOGH) ? 1 : 0;
    cudaStream_t st = (cudaStream_t)stream;
    if (launch_lb(q, nq, qkim, t, t_upper, t_lower, tkim, nt, L, w, v, kim ? 1 : 0, -1, lb,
                  ldlb, nullptr, st, keogh) ||
        launch_lb(t, nt, nullptr, q, q_upper, q_lower, nullptr, nq, L, w, v, 0, -1, lb, ldlb,
                  nullptr, st, keogh, 1))
        return fail(NNDTW_E_ARG, "too many series for one launch");
    return cuda_fail("nndtw_lb_enhanced_symmetric");
}

int nndtw_lb_improved(const float *q, int64_t nq, const float *t, const float *t_upper,
                      const float *t_lower, int64_t nt, int32_t L, int32_t w, float *lb,
                      int64_t ldlb, void *stream) {
    int sms, rc;
    if ((rc = device_sms(&sms))) return rc;
    if ((rc = check_common(nq, L, w))) return rc;
    if (nt < 0) return fail(NNDTW_E_ARG, "negative nt");
    if (ldlb < nt) return fail(NNDTW_E_ARG, "ldlb < nt");
    if (nq > 0 && nt > 0 && (!q || !t || !t_upper || !t_lower || !lb))
        return fail(NNDTW_E_ARG, "null pointer argument");
    cudaStream_t st = (cudaStream_t)stream;
    // first pass LB_Keogh(q, env t) over all columns (tile kernel), then LB_Keogh(t, env q')
    if (launch_lb(q, nq, nullptr, t, t_upper, t_lower, nullptr, nt, L, w, 1, 0, -1, lb, ldlb,
                  nullptr, st, 1) ||
        launch_lb_improved_pass(q, nq, t, t_upper, t_lower, nt, L, w, 0, L, lb, ldlb, sms, st))
        return fail(NNDTW_E_ARG, "too many series for one launch");
    return cuda_fail("nndtw_lb_improved");
}

int nndtw_lb_enhanced_improved(const float *q, int64_t nq, const float *t, const float *t_upper,
                               const float *t_lower, int64_t nt, int32_t L, int32_t w, int32_t v,
                               float *lb, int64_t ldlb, void *stream) {
    int sms, rc;
    if ((rc = device_sms(&sms))) return rc;
    if ((rc = check_common(nq, L, w))) return rc;
    if (nt < 0) return fail(NNDTW_E_ARG, "negative nt");
    if (v < 1) return fail(NNDTW_E_V, "V must be >= 1");
    if (ldlb < nt) return fail(NNDTW_E_ARG, "ldlb < nt");
    if (nq > 0 && nt > 0 && (!q || !t || !t_upper || !t_lower || !lb))
        return fail(NNDTW_E_ARG, "null pointer argument");
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = (L / 2) < v ? (L / 2) : v;
    if (launch_lb(q, nq, nullptr, t, t_upper, t_lower, nullptr, nt, L, w, v, 0, -1, lb, ldlb,
                  nullptr, st, 0) ||
        launch_lb_improved_pass(q, nq, t, t_upper, t_lower, nt, L, w, nb, L - nb, lb, ldlb, sms,
                                st))
        return fail(NNDTW_E_ARG, "too many series for one launch");
    return cuda_fail("nndtw_lb_enhanced_improved");
}

int nndtw_lb_new(const float *q, int64_t nq, const float *t, int64_t nt, int32_t L, int32_t w,
                 float *lb, int64_t ldlb, void *stream) {
    int sms, rc;
    if ((rc = device_sms(&sms))) return rc;
    if ((rc = check_common(nq, L, w))) return rc;
    if (nt < 0) return fail(NNDTW_E_ARG, "negative nt");
    if (ldlb < nt) return fail(NNDTW_E_ARG, "ldlb < nt");
    if (nq > 0 && nt > 0 && (!q || !t || !lb)) return fail(NNDTW_E_ARG, "null pointer argument");
    if (launch_lb_pairs(0, q, nq, t, nullptr, nullptr, nt, L, w, lb, ldlb, (cudaStream_t)stream))
        return fail(NNDTW_E_LENGTH, "L too long for the LB_New kernel's shared memory");
    return cuda_fail("nndtw_lb_new");
}

size_t nndtw_ed_seed_workspace_bytes(int64_t nq, int64_t nt, int32_t L) {
    if (nq < 0 || nt < 0 || L < 1) return 0;
    return ed_seed_scratch_bytes(nq, nt, L);
}

int nndtw_ed_seed(const float *q, int64_t nq, const float *t, int64_t nt, int32_t L, void *ws,
                  size_t ws_bytes, uint64_t *key, void *stream) {
    int sms, rc;
    if ((rc = device_sms(&sms))) return rc;
    if (nq < 0 || nt < 0) return fail(NNDTW_E_ARG, "negative count");
    if (L < 1) return fail(NNDTW_E_LENGTH, "L must be >= 1");
    if (!ed_seed_supported(L)) return fail(NNDTW_E_LENGTH, "L must be >= 1");
    if (nq > 0 && nt > 0 && (!q || !t || !key || !ws)) return fail(NNDTW_E_ARG, "null pointer argument");
    if (ws_bytes < ed_seed_scratch_bytes(nq, nt, L)) return fail(NNDTW_E_WORKSPACE, "ws too small");
    if (launch_ed_seed(q, nq, t, nt, L, ws, (unsigned long long *)key, sms, (cudaStream_t)stream))
        return fail(NNDTW_E_ARG, "ed seed launch failed");
    return cuda_fail("nndtw_ed_seed");
}

int nndtw_tightness(const float *lb, const float *dtw, int64_t n, double *sum, uint64_t *count,
                    uint32_t *max_bits, void *stream) {
    int sms, rc;
    if ((rc = device_sms(&sms))) return rc;
    if (n < 0) return fail(NNDTW_E_ARG, "negative count");
    if (n > 0 && (!lb || !dtw || !sum || !count || !max_bits))
        return fail(NNDTW_E_ARG, "null pointer argument");
    launch_tightness(lb, dtw, n, sum, (unsigned long long *)count, max_bits, sms,
                     (cudaStream_t)stream);
    return cuda_fail("nndtw_tightness");
}

int nndtw_dtw_batch(const float *a, const float *b, const int32_t *ia, const int32_t *ib,
                    int64_t npairs, int32_t L, int32_t w, const float *cutoff, float *out,
                    void *stream) {
    int sms, rc;
    if ((rc = device_sms(&sms))) return rc;
    if ((rc = check_common(npairs, L, w))) return rc;
    if (npairs == 0) return NNDTW_OK;
    if (!a || !b || !out) return fail(NNDTW_E_ARG, "null pointer argument");
    if (w > L - 1) w = L - 1;
    TieLog log{nullptr, nullptr, 0, nullptr};
    rc = dispatch_dtw(a, b, INT64_MAX, INT64_MAX, nullptr, nullptr, 0, ia, ib, npairs, L, w, 1, nullptr, 0,
                      eps_tie(L), log, nullptr, nullptr, cutoff, out, (cudaStream_t)stream, sms);
    if ((rc = dtw_fail(rc, L, w))) return rc;
    return cuda_fail("nndtw_dtw_batch");
}

size_t nndtw_classify_workspace_bytes(int64_t nq, int64_t nt, int32_t L, int32_t w) {
    (void)w;
    return classify_layout(nullptr, nq, nt, L).bytes;
}

size_t nndtw_classify_workspace_bytes_capped(int64_t nq, int64_t nt, int32_t L, int32_t w,
                                             int64_t max_pairs) {
    (void)w;
    const unsigned long long full = full_pair_cap(nq, nt);
    const unsigned long long lo = 2ull * (unsigned long long)(nq > 0 ? nq : 0) + 2ull;
    unsigned long long cap = max_pairs < 0 ? full : (unsigned long long)max_pairs;
    if (cap < lo) cap = lo;
    if (cap >= full) return classify_layout(nullptr, nq, nt, L).bytes;
    return classify_layout(nullptr, nq, nt, L, cap).bytes;
}

int nndtw_classify_overflowed(const void *ws, size_t ws_bytes, int64_t nq, int64_t nt, int32_t L,
                              int32_t *overflowed, void *stream) {
    if (!ws || !overflowed) return fail(NNDTW_E_ARG, "null pointer argument");
    if (nq < 0 || nt < 0 || L < 2) return fail(NNDTW_E_ARG, "bad shape");
    ClassifyWs W = classify_layout_for(const_cast<void *>(ws), nq, nt, L, ws_bytes);
    if (ws_bytes < W.bytes) return fail(NNDTW_E_WORKSPACE, "workspace too small");
    *overflowed = 0;
    if (nq == 0) return NNDTW_OK;
    unsigned long long h = 0;
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemcpyAsync(&h, W.cap_overflow, sizeof h, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_fail("overflow check");
    *overflowed = h != 0ull ? 1 : 0;
    return NNDTW_OK;
}

int nndtw_classify(const float *q, int64_t nq, const float *t, const float *upper,
                   const float *lower, const nndtw_kim *tkim, int64_t nt, int64_t index_base,
                   int64_t self_offset, int32_t L, int32_t w, int32_t v, uint32_t flags,
                   void *ws, size_t ws_bytes, uint64_t *key, nndtw_stats *stats, void *stream) {
    if (stats) {
        std::memset(stats, 0, sizeof *stats);
        stats->pruned_kim = stats->pruned_bands = stats->pruned_keogh = -1;
    }
    return classify_impl(q, nq, t, upper, lower, tkim, nt, index_base, self_offset, L, w, v,
                         flags, nullptr, ws, ws_bytes, (unsigned long long *)key, stats,
                         (cudaStream_t)stream);
}

int nndtw_classify_refine(void *ws, size_t ws_bytes, const float *q, int64_t nq,
                          const float *t, int64_t nt, int32_t L, int32_t w,
                          const uint64_t *gkey, uint64_t *f64key, void *stream) {
    int sms, rc;
    if ((rc = device_sms(&sms))) return rc;
    if ((rc = check_common(nq, L, w))) return rc;
    if (w > L - 1) w = L - 1;
    ClassifyWs W = classify_layout_for(ws, nq, nt, L, ws_bytes);
    if (!ws || ws_bytes < W.bytes) return fail(NNDTW_E_WORKSPACE, "workspace too small");
    if (nq == 0) return NNDTW_OK;
    cudaStream_t st = (cudaStream_t)stream;
    launch_fill_u64((unsigned long long *)f64key, nq, kNone64, st);
    if (nt > 0) {
        launch_refine(W.log, W.log_count, W.log_cap, q, t, L, w,
                      (const unsigned long long *)gkey, eps_tie(L),
                      (unsigned long long *)f64key, nullptr, nullptr, W.overflow, sms, st);
        launch_refine_overflow(W.log_count, W.log_cap, W.overflow, nq, W.lb, W.ldlb, nt, q, t, L, w,
                               (const unsigned long long *)gkey, eps_prune(L), 0,
                               (unsigned long long *)f64key, nullptr, 0, nullptr, sms, st);
    }
    return cuda_fail("nndtw_classify_refine");
}

int nndtw_classify_resolve(void *ws, size_t ws_bytes, const float *q, int64_t nq,
                           const float *t, int64_t nt, int32_t L, int32_t w,
                           int64_t index_base, const uint64_t *gkey, const uint64_t *gf64,
                           uint64_t *out, void *stream) {
    int sms, rc;
    if ((rc = device_sms(&sms))) return rc;
    if ((rc = check_common(nq, L, w))) return rc;
    if (w > L - 1) w = L - 1;
    ClassifyWs W = classify_layout_for(ws, nq, nt, L, ws_bytes);
    if (!ws || ws_bytes < W.bytes) return fail(NNDTW_E_WORKSPACE, "workspace too small");
    if (nq == 0) return NNDTW_OK;
    cudaStream_t st = (cudaStream_t)stream;
    launch_fill_u64((unsigned long long *)out, nq, kNone64, st);
    if (nt > 0) {
        launch_resolve(W.log, W.log_count, W.log_cap, (const unsigned long long *)gf64,
                       index_base, (unsigned long long *)out, sms, st);
        launch_refine_overflow(W.log_count, W.log_cap, W.overflow, nq, W.lb, W.ldlb, nt, q, t, L, w,
                               (const unsigned long long *)gkey, eps_prune(L), 1, nullptr,
                               (const unsigned long long *)gf64, index_base,
                               (unsigned long long *)out, sms, st);
    }
    return cuda_fail("nndtw_classify_resolve");
}

int nndtw_finalize(const uint64_t *key, int64_t nq, int32_t key_format, const int32_t *labels,
                   int64_t nlabels, int64_t *idx_out, int32_t *label_out, float *dist_out,
                   void *stream) {
    int sms, rc;
    if ((rc = device_sms(&sms))) return rc;
    if (nq < 0 || (nq > 0 && !key) || (key_format != 0 && key_format != 1))
        return fail(NNDTW_E_ARG, "bad arguments");
    launch_finalize((const unsigned long long *)key, nq, key_format, labels, nlabels, idx_out,
                    label_out, dist_out, (cudaStream_t)stream);
    return cuda_fail("nndtw_finalize");
}

size_t nndtw_loocv_workspace_bytes(int64_t n, int32_t L, int64_t q_begin, int64_t q_end) {
    return loocv_layout(nullptr, n, L, q_end - q_begin).bytes;
}

int nndtw_loocv_window(const float *x, const int32_t *labels, int64_t n, int32_t L,
                       const int32_t *windows, int32_t nw, int32_t v, int64_t q_begin,
                       int64_t q_end, void *ws, size_t ws_bytes, int64_t *errors,
                       int32_t *nn_out, nndtw_stats *stats, void *stream) {
    int sms, rc;
    if ((rc = device_sms(&sms))) return rc;
    if ((rc = check_common(n, L, 0))) return rc;
    if (v < 1) return fail(NNDTW_E_V, "V must be >= 1");
    if (nw < 0 || (nw > 0 && !windows)) return fail(NNDTW_E_ARG, "bad window list");
    if (q_begin < 0 || q_end < q_begin || q_end > n)
        return fail(NNDTW_E_ARG, "query range outside [0, n]");
    if (n > 0 && nw > 0 && (!x || !labels || !errors || !ws))
        return fail(NNDTW_E_ARG, "null pointer");
    for (int p = 0; p < nw; ++p)
        if (windows[p] < 0) return fail(NNDTW_E_WINDOW, "w must be >= 0");
    const int64_t nq = q_end - q_begin;
    LoocvWs W = loocv_layout(ws, n, L, nq);
    if (ws_bytes < W.bytes) return fail(NNDTW_E_WORKSPACE, "workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    if (stats) {
        std::memset(stats, 0, sizeof *stats);
        stats->pruned_kim = stats->pruned_bands = stats->pruned_keogh = -1;
    }
    if (nq == 0 || nw == 0) return NNDTW_OK;
    const float *qx = x + q_begin * (int64_t)L;
    cudaEvent_t e0, e1, e2;
    if (stats) {
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventCreate(&e2);
    }
    float ms_env = 0, ms_rest = 0;
    for (int p = 0; p < nw; ++p) {
        int w = windows[p] > L - 1 ? L - 1 : windows[p];
        if (stats) cudaEventRecord(e0, st);
        launch_envelopes(x, n, L, w, W.U, W.Lo, p == 0 ? W.kim : nullptr, st);
        if (stats) cudaEventRecord(e1, st);
        rc = classify_impl(qx, nq, x, W.U, W.Lo, W.kim, n, 0, q_begin, L, w, v,
                           NNDTW_CLASSIFY_EXACT, p == 0 ? nullptr : W.prev_nn, W.cws,
                           W.cws_bytes, W.key, stats, st, nullptr);
        if (rc) return rc;
        launch_count_errors(W.key, nq, labels, q_begin, errors + p,
                            nn_out ? nn_out + (int64_t)p * nq : nullptr, W.prev_nn, st);
        if (stats) {
            cudaEventRecord(e2, st);
            cudaEventSynchronize(e2);
            float a = 0, b = 0;
            cudaEventElapsedTime(&a, e0, e1);
            cudaEventElapsedTime(&b, e1, e2);
            ms_env += a;
            ms_rest += b;
        }
    }
    if (stats) {
        stats->ms_envelopes = ms_env;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaEventDestroy(e2);
    }
    return cuda_fail("nndtw_loocv_window");
}

}  // extern "C"
