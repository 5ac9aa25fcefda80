/*
 * nndtw.h -- C ABI of libnndtw.so: exact 1-NN search under windowed DTW pruned by the
 * LB_Kim -> LB_Enhanced^V cascade of arxiv 1808.09617, as hand-written CUDA for sm_100a (B200).
 *
 * Citations: "P:<line>" = PAPER.md line (section / equation / algorithm given alongside),
 * "Cn" = reading n of DESIGN.md ("Readings of the paper").
 *
 * Conventions (all entry points):
 *  - Every float/int array argument is a DEVICE pointer unless marked "host".  Arrays are
 *    caller-owned, row-major and contiguous; series are float32 [n][L].  The library never
 *    allocates device memory, never frees or retains a caller pointer past the call; scratch
 *    comes from the caller's `ws` (size from the matching *_workspace_bytes function).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Calls are
 *    asynchronous on `stream` unless stated; a call that fills a host-side nndtw_stats
 *    synchronises `stream` before returning.
 *  - Distances are SQUARED (the accumulated cost D(L,L) of Eq. 1); DTW itself is
 *    its square root (Eq. 2).  delta(a,b) = (a-b)^2 (reading C1).
 *  - The window w is absolute (reading C4 resolves fractions); w >= L-1 is clamped to L-1,
 *    which is unconstrained DTW (reading C3).  w = 0 is the squared Euclidean distance.
 *  - Return value: NNDTW_OK or an NNDTW_E_* code; nndtw_last_error() gives a thread-local
 *    message.  No C++ exception crosses the ABI.  Inputs must be finite with |x| < 2^36
 *    (nndtw_check_finite; the Python layer checks: NaN would silently be dropped by fminf and
 *    larger magnitudes break the DTW kernels' +inf pads).
 */
#ifndef NNDTW_H
#define NNDTW_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define NNDTW_API __attribute__((visibility("default")))
#else
#define NNDTW_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define NNDTW_OK 0
#define NNDTW_E_ARG 1        /* null pointer, negative count, misaligned pointer */
#define NNDTW_E_LENGTH 2     /* L < 2 (Algorithm 1 is not admissible at L = 1, reading C11) */
#define NNDTW_E_WINDOW 3     /* w < 0 */
#define NNDTW_E_V 4          /* V < 1 */
#define NNDTW_E_WORKSPACE 5  /* ws too small */
#define NNDTW_E_CUDA 6       /* a CUDA runtime error (message has the name) */
#define NNDTW_E_ARCH 7       /* the current device is not sm_100 */
#define NNDTW_E_INDEX 8      /* a global train index is >= 2^31 (index_base + nt > 2^31 - 1) */

/* Per-series LB_Kim features (sum variant P:619-621, reading C7):
 * min / max value and their lowest indices (ties -> lowest index).  First and last values are
 * read from the series itself.  16 bytes, naturally aligned. */
typedef struct {
    float vmin, vmax;
    int32_t imin, imax;
} nndtw_kim;

/* Host-side counters, filled (after a stream synchronisation) when a non-NULL pointer is
 * passed.  All counts are exact integers. */
typedef struct {
    int64_t lb_pairs;       /* (query, train) pairs whose cascade bound was computed */
    int64_t survivors;      /* pairs with LB <= bsf*(1+eps_p) after the seed round */
    /* Pairs pruned by each level of the cascade against the seeded best-so-far
     * bsf*(1+eps_p): LB_Kim already exceeds it; else the boundary terms + bands of
     * Algorithm 1 exceed it (its line-12 abort); else the full bound with
     * the LB_Keogh bridge does.  Seed pairs and the leave-one-out self pair are not counted, so
     * lb_pairs = pruned_kim + pruned_bands + pruned_keogh + survivors + seeds (+ self pairs).
     * Filled only under NNDTW_CLASSIFY_LEVEL_STATS (an extra bands-only pass over the pairs,
     * timed in ms_other); -1 otherwise. */
    int64_t pruned_kim, pruned_bands, pruned_keogh;
    /* Two-stage S2 (the default cascade): pairs whose LB_Keogh bridge was computed, i.e. kept by
     * LB_Kim and Algorithm 1's bands against the first seed's best-so-far (line-12 test);
     * lb_pairs for the one-stage bounds. */
    int64_t bridge_pairs;
    int64_t dtw_calls;      /* DTW work items started (seeds + survivors) */
    int64_t dtw_abandoned;  /* survivor items stopped by early abandoning */
    int64_t cells;          /* in-band DP cells on the diagonals the survivor round processed */
    int64_t near_tie_pairs; /* pairs re-ranked in fp64 (reading C16) */
    int32_t rounds;         /* DTW rounds run (seed round included) */
    int32_t launches;       /* kernel launches issued by the call */
    /* CUDA-event stage times on the call's stream: ms_envelopes = the query-side S1 work (Kim
     * features, and the queries' envelopes for the symmetric bound; the train envelopes are
     * built before the call), ms_lb = the LB cascade kernel(s) (two-stage S2: stage A,
     * the first seed round, the bridge lists and kernel, the second seed round), ms_dtw = the
     * survivor-round DTW kernel, ms_other = everything else (compaction, S7). */
    float ms_envelopes, ms_lb, ms_dtw, ms_other;
    /* the part of ms_lb spent in the sparse bridge kernel (two-stage S2; 0 otherwise) */
    float ms_lb_bridge;
    /* S4 band-limited pass (wide windows): survivors whose
     * band-edge cells came within the threshold and were rerun with the full window */
    int64_t dtw_fallback;
} nndtw_stats;

/* Library identity and introspection. */
NNDTW_API const char *nndtw_last_error(void);
NNDTW_API int nndtw_version(void);
/* Number of kernels this library has launched in the process so far (bench bookkeeping). */
NNDTW_API int64_t nndtw_launch_count(void);
/* Name of the S4 kernel nndtw_dtw_batch / nndtw_classify run for (L, w): "k_dtw_w0" (w = 0,
 * squared ED), "k_dtw_band" (anti-diagonal band wavefront) or "k_dtw_strip" (row strips, long
 * windows); "" for invalid arguments.  Host-only (bench / profiling bookkeeping). */
NNDTW_API const char *nndtw_dtw_kernel_name(int32_t L, int32_t w);
/* The band window wb of the band-limited S4 pass nndtw_classify's survivor round runs first for
 * (L, w), or -1 when it runs the full window directly.
 * Band-kernel windows: wb = 13G - 1 <= w/2 for w >= 64; full windows (the row-strip kernel):
 * wb <= w/8 where that is >= 103; -1 for L % 4 != 0 or NNDTW_ADAPT=0.  Host-only. */
NNDTW_API int32_t nndtw_band_limited_window(int32_t L, int32_t w);
/* NNDTW_OK if the current device is sm_100 (B200); NNDTW_E_ARCH otherwise. */
NNDTW_API int nndtw_check_device(void);
/* *bad (device int32, caller-zeroed) is set to 1 if x [n] holds a NaN, an infinity or a value
 * with |x| >= 2^36.  Input precondition of every DTW entry point: the kernels' out-of-matrix
 * shared-memory pads (+-2^64*k) rely on (pad - x)^2 overflowing to +inf. */
NNDTW_API int nndtw_check_finite(const float *x, int64_t n, int32_t *bad, void *stream);

/*
 * S1 -- envelopes, Eq. 3-4:
 *   upper[i][k] = max_{max(0,k-w) <= j <= min(L-1,k+w)} x[i][j],  lower = min over the same.
 * x: [n][L]; upper, lower: [n][L] outputs (bit-exact: min/max of floats are exact); the
 * outputs must not overlap x (series are staged through shared memory by persistent CTAs, so
 * one series' output can be written before another's input is read).
 * kim: [n] output, nullable: the LB_Kim features of each series (nndtw_kim).
 * Precomputed "at training time".  Errors: E_ARG, E_LENGTH (L < 1), E_WINDOW.
 */
NNDTW_API int nndtw_envelopes(const float *x, int64_t n, int32_t L, int32_t w, float *upper,
                    float *lower, nndtw_kim *kim, void *stream);

/* LB_Kim features only (query side): kim[i] for x [n][L]. */
NNDTW_API int nndtw_series_stats(const float *x, int64_t n, int32_t L, nndtw_kim *kim, void *stream);

/*
 * S2 -- batched cascade bound over all (query, train) pairs:
 *   lb[i*ldlb + j] = LB_Enhanced^V_W(q_i, t_j)                   (flags & 1 == 0)
 *                  = max(LB_Kim_sum(q_i,t_j), LB_Enhanced^V_W)     (flags & NNDTW_LB_WITH_KIM)
 * LB_Enhanced is Eq. 7 computed as Algorithm 1 without the line-12
 * abort (the bound is wanted for every pair): boundary terms, n_bands = min(floor(L/2), V)
 * left/right bands (readings C8-C10) and the LB_Keogh bridge over
 * columns n_bands+1 .. L-n_bands against t_j's envelopes.
 * q: [nq][L]; t, upper, lower: [nt][L]; qkim: [nq], tkim: [nt] (both required with WITH_KIM,
 * else nullable); lb: [nq][ldlb], ldlb >= nt.  fp32 arithmetic.
 */
#define NNDTW_LB_WITH_KIM 1u
/* flags & NNDTW_LB_KEOGH: LB_Keogh (m = L, reading C6) over all L columns in place of
 * LB_Enhanced -- the paper's comparison bound (Fig. 9 normalises by it). */
#define NNDTW_LB_KEOGH 2u
/* flags & NNDTW_LB_PARTIAL: Algorithm 1 up to its line-12 test only -- the boundary terms and the
 * bands (lines 1-11), no LB_Keogh bridge (max with LB_Kim under WITH_KIM): the value
 * the two-stage S2 compares with the best-so-far before it computes the bridge.  A lower bound of
 * the full value (every bridge term is >= 0).  Not combinable with NNDTW_LB_KEOGH. */
#define NNDTW_LB_PARTIAL 4u
NNDTW_API int nndtw_lb_enhanced(const float *q, int64_t nq, const nndtw_kim *qkim, const float *t,
                      const float *upper, const float *lower, const nndtw_kim *tkim,
                      int64_t nt, int32_t L, int32_t w, int32_t v, uint32_t flags, float *lb,
                      int64_t ldlb, void *stream);

/*
 * S2, symmetric variant:
 *   lb[i*ldlb + j] = max(LB(q_i, t_j), LB(t_j, q_i))  [then max with LB_Kim under WITH_KIM]
 * with LB = LB_Enhanced^V_W (or LB_Keogh under NNDTW_LB_KEOGH).  The boundary terms and the
 * bands of Algorithm 1 are symmetric in (A, B), so only the LB_Keogh bridge differs: the
 * second pass runs the tile kernel with the roles exchanged (queries' envelopes q_upper /
 * q_lower, from nndtw_envelopes on q) and folds its value in with max.  Admissible: DTW is
 * symmetric and each direction is a lower bound (Thm 2).  Same layouts as nndtw_lb_enhanced;
 * q_upper, q_lower: [nq][L].  Cost: twice the bridge work.
 */
NNDTW_API int nndtw_lb_enhanced_symmetric(const float *q, const float *q_upper,
                                          const float *q_lower, const nndtw_kim *qkim,
                                          int64_t nq, const float *t, const float *t_upper,
                                          const float *t_lower, const nndtw_kim *tkim,
                                          int64_t nt, int32_t L, int32_t w, int32_t v,
                                          uint32_t flags, float *lb, int64_t ldlb,
                                          void *stream);

/*
 * Comparison bounds of the paper's evaluation, all pairs
 * (q: [nq][L]; t: [nt][L]; lb: [nq][ldlb] out, ldlb >= nt; fp32; asynchronous):
 * nndtw_lb_improved: LB_Improved_W(q_i, t_j) = LB_Keogh(q_i, env t_j) + LB_Keogh(t_j, env q')
 *   (§2.3.3), q' the projection of q_i onto t_j's envelope; env q' by the O(L)
 *   van Herk sliding max/min per pair ("the optimised algorithm to compute the projection
 *   envelopes").  t_upper / t_lower: t's envelopes (nndtw_envelopes, same w).
 * nndtw_lb_enhanced_improved: LB_Enhanced^V_W with the LB_Improved bridge (reading
 *   C21): nndtw_lb_enhanced's value plus, over the bridge columns n_bands+1 .. L-n_bands, the
 *   LB_Keogh terms of t_j against the envelope of q'.  Admissible; >= LB_Enhanced^V.
 * nndtw_lb_new: LB_New_W(q_i, t_j) = delta(first) + delta(last) + sum over the inner i of the
 *   minimum delta(q_i, t_j') over the window (§2.3.4); O(L*w) per pair, as defined.
 */
NNDTW_API int nndtw_lb_improved(const float *q, int64_t nq, const float *t,
                                const float *t_upper, const float *t_lower, int64_t nt,
                                int32_t L, int32_t w, float *lb, int64_t ldlb, void *stream);
NNDTW_API int nndtw_lb_enhanced_improved(const float *q, int64_t nq, const float *t,
                                         const float *t_upper, const float *t_lower, int64_t nt,
                                         int32_t L, int32_t w, int32_t v, float *lb,
                                         int64_t ldlb, void *stream);
NNDTW_API int nndtw_lb_new(const float *q, int64_t nq, const float *t, int64_t nt, int32_t L,
                           int32_t w, float *lb, int64_t ldlb, void *stream);

/*
 * Euclidean-nearest candidate of every query (the paper's candidate order; the ED is
 * DTW_0), on piecewise-aggregate approximations: x -> the means over f consecutive points
 * (the last segment zero-padded), f the smallest power of two with ceil(L/f) <= 128.
 * key[i] = min over j of ((bits of f32 ED(paa(q_i), paa(t_j))) << 32 | j), ED squared, computed
 * from bf16-rounded PAAs with fp32 accumulation on the tensor cores (tcgen05), so the chosen j is
 * nearest up to that approximation -- it serves as a seed (any candidate's exact DTW is a valid
 * best-so-far), not as a distance.  key must hold 0xFFFF...FF on entry (it is min-ed into).
 * q: [nq][L], t: [nt][L] device fp32, L >= 1; ws: device scratch of
 * nndtw_ed_seed_workspace_bytes(nq, nt, L) bytes.
 */
NNDTW_API size_t nndtw_ed_seed_workspace_bytes(int64_t nq, int64_t nt, int32_t L);
NNDTW_API int nndtw_ed_seed(const float *q, int64_t nq, const float *t, int64_t nt, int32_t L,
                            void *ws, size_t ws_bytes, uint64_t *key, void *stream);

/*
 * Tightness (reading C20): over the n pairs with 0 < dtw[p] <
 * +inf, accumulate sum[0] += sum of sqrt(lb[p] / dtw[p]) (fp64), count[0] += #pairs and
 * max_bits[0] = max(max_bits[0], float bits of the largest ratio).  lb and dtw are squared
 * values (fp32 device arrays [n]); sum (double[1]), count (uint64[1]) and max_bits
 * (uint32[1]) are device pointers the caller zeroes.  Asynchronous.
 */
NNDTW_API int nndtw_tightness(const float *lb, const float *dtw, int64_t n, double *sum,
                              uint64_t *count, uint32_t *max_bits, void *stream);

/*
 * S4 -- batched windowed DTW, Eq. 1 inside |i-j| <= w, with early
 * abandoning.  Pair p compares a[ia[p]] with b[ib[p]] (ia/ib nullable = p).
 * cutoff: [npairs] squared cutoffs, nullable (= +inf).  out[p] = squared DTW in fp32, or +inf
 * when abandoned; abandoning happens only when the minimum over a cut of the DP (two
 * consecutive anti-diagonals, reading C14) exceeds cutoff*(1+(4L+8)*2^-24), which guarantees
 * the exact value exceeds cutoff.  a: [*][L], b: [*][L].
 */
NNDTW_API int nndtw_dtw_batch(const float *a, const float *b, const int32_t *ia, const int32_t *ib,
                    int64_t npairs, int32_t L, int32_t w, const float *cutoff, float *out,
                    void *stream);

/*
 * S2-S7 -- 1-NN search of every query against one train shard.
 * Key format: key[i] = (float bits of the squared distance << 32) | global train index;
 * global index = index_base + local index (< 2^31, else NNDTW_E_INDEX: format-1 keys put the
 * index in the high half and must stay non-negative as int64).  Non-negative floats order like their
 * bits, so an unsigned (or signed int64: bit 63 is 0) MIN over keys gives the smallest
 * distance with ties to the lowest index (reading C13) -- the shard combine of S6.
 * Stages: LB cascade for all pairs (S2); seed = DTW to the argmin-LB candidate (S3); prune
 * pairs with LB > bsf*(1+eps_p), eps_p = (3L+8)*2^-24 (reading C16); DTW with early abandon
 * against the live per-query best on the survivors, atomicMin on the key (S4/S5).
 * flags & NNDTW_CLASSIFY_EXACT: also run the fp64 near-tie re-rank locally (S7; only valid
 * for a single shard) so that key is final: the candidate chosen is the one the fp64 oracle
 * chooses, its fp32 distance in the high half.
 * Without EXACT the caller combines shards with MIN over keys, then calls
 * nndtw_classify_refine and nndtw_classify_resolve with the same ws (see dist.py).
 * q: [nq][L]; t, upper, lower: [nt][L]; tkim: [nt] (from nndtw_envelopes); key: [nq] out.
 * self_offset >= 0 excludes train index (local) i + self_offset for query i (leave-one-out);
 * pass -1 otherwise.  stats: host, nullable (non-NULL synchronises).
 */
#define NNDTW_CLASSIFY_EXACT 1u
/* flags & NNDTW_CLASSIFY_BOUND_KEOGH: prune with max(LB_Kim, LB_Keogh) instead of
 * max(LB_Kim, LB_Enhanced^V) (same exact answer; a baseline for the V-sweep). */
#define NNDTW_CLASSIFY_BOUND_KEOGH 2u
/* flags & NNDTW_CLASSIFY_BOUND_SYMMETRIC: prune with the symmetric bound max(LB(q,t), LB(t,q))
 * (see nndtw_lb_enhanced_symmetric); the queries' envelopes are built in ws.
 * Same exact answer; tighter bound, twice the bridge work. */
#define NNDTW_CLASSIFY_BOUND_SYMMETRIC 4u
/* Two-phase call for a sharded search (dist.py): PHASE_SEED runs the initialisation, the S2
 * bound and the S3 seed round and returns the seed keys in key (state kept in ws); the caller
 * MIN-reduces key over the shards; PHASE_SEARCH (same ws, q, t, flags otherwise) takes that
 * key as the starting best-so-far -- a valid upper bound on every query's global NN distance,
 * so each shard prunes against the global seed instead of its own -- and runs S3 compaction
 * and S4/S5.  Neither flag: both phases in one call.  The answer does not change. */
#define NNDTW_CLASSIFY_PHASE_SEED 8u
#define NNDTW_CLASSIFY_PHASE_SEARCH 16u
/* PHASE_SEARCH in two halves, so that shards can exchange their best-so-far in between:
 * SEARCH_A runs S3 compaction and S4 on the survivors of the lowest-bound buckets (LB below a
 * fixed fraction of the seeded best-so-far); the caller MIN-reduces key over the
 * shards; SEARCH_B (same ws) takes that key and runs S4/S5 on the remaining survivors.  The
 * union is PHASE_SEARCH's work; the answer does not change.  SEARCH_B synchronises the stream
 * once (it reads the split point). */
#define NNDTW_CLASSIFY_PHASE_SEARCH_A 32u
#define NNDTW_CLASSIFY_PHASE_SEARCH_B 64u
/* flags & NNDTW_CLASSIFY_LEVEL_STATS (with non-NULL stats): fill the per-level prune counters
 * pruned_kim / pruned_bands / pruned_keogh (one extra bands-only pass, no bridge).  In a
 * phased (sharded) classify, set it on the SEED call as well: with the two-stage S2 the seed
 * phase then also stores the full cascade values the counters read. */
#define NNDTW_CLASSIFY_LEVEL_STATS 128u
/* Alternative S2 bounds (the paper's NN-DTW time per bound,
 * Fig. 9-11).  At most one of them, not with BOUND_KEOGH / BOUND_SYMMETRIC; the
 * answer never changes (every bound is admissible, Thm 2):
 *   BOUND_IMPROVED           max(LB_Kim, LB_Improved)
 *   BOUND_NEW                max(LB_Kim, LB_New)
 *   BOUND_ENHANCED_IMPROVED  max(LB_Kim, LB_Enhanced^V with the LB_Improved bridge)
 *   BOUND_NONE               no lower bound: every pair is a survivor, DTW with early
 *                            abandoning only (the no-LB baseline).
 * With LEVEL_STATS the bridge-level counter pruned_keogh counts the pairs pruned by the full
 * bound (pruned_bands is 0 except for BOUND_ENHANCED_IMPROVED). */
#define NNDTW_CLASSIFY_BOUND_IMPROVED 256u
#define NNDTW_CLASSIFY_BOUND_NEW 512u
#define NNDTW_CLASSIFY_BOUND_ENHANCED_IMPROVED 1024u
#define NNDTW_CLASSIFY_BOUND_NONE 2048u
/* Workspace.  nndtw_classify_workspace_bytes: the full layout, room for every (query, train)
 * pair as a survivor and as a two-stage list entry (24 bytes per pair with the 4-byte bound
 * matrix).  nndtw_classify_workspace_bytes_capped: room for at most max_pairs survivors and
 * max_pairs list entries (4 + 20*max_pairs/(nq*nt) bytes per pair; >= 2*nq + 2); classify
 * infers the capacity from ws_bytes (the full layout whenever ws_bytes holds it).  A call whose
 * survivors or listed pairs exceed the capacity stores only what fits and sets an overflow word
 * in ws: its keys are then NOT valid.  nndtw_classify_overflowed synchronises `stream`, and sets
 * *overflowed = 1 if the last classify on ws overflowed (else 0); the caller reruns that call
 * with a larger (e.g. the full) workspace.  The answer of a call that did not overflow is the
 * full layout's. */
NNDTW_API size_t nndtw_classify_workspace_bytes(int64_t nq, int64_t nt, int32_t L, int32_t w);
NNDTW_API size_t nndtw_classify_workspace_bytes_capped(int64_t nq, int64_t nt, int32_t L,
                                                       int32_t w, int64_t max_pairs);
NNDTW_API int nndtw_classify_overflowed(const void *ws, size_t ws_bytes, int64_t nq, int64_t nt,
                                        int32_t L, int32_t *overflowed, void *stream);
NNDTW_API int nndtw_classify(const float *q, int64_t nq, const float *t, const float *upper,
                   const float *lower, const nndtw_kim *tkim, int64_t nt, int64_t index_base,
                   int64_t self_offset, int32_t L, int32_t w, int32_t v, uint32_t flags,
                   void *ws, size_t ws_bytes, uint64_t *key, nndtw_stats *stats, void *stream);

/*
 * S7 (sharded) -- near-tie re-rank, step 1.  gkey: [nq] the MIN of all shards' keys.  For
 * every locally completed candidate whose fp32 distance is within gkey*(1+eps_t) of the global
 * best, recompute DTW in fp64 with the oracle's per-cell operation sequence (DESIGN.md
 * "fp64 re-rank"); f64key[i] = bits of the smallest such fp64 value (INT64_MAX if none: keys stay < 2^63 so a signed int64 MIN
 * reduction combines them).
 * Requires the ws of the preceding nndtw_classify call (same q, t).
 */
NNDTW_API int nndtw_classify_refine(void *ws, size_t ws_bytes, const float *q, int64_t nq,
                          const float *t, int64_t nt, int32_t L, int32_t w,
                          const uint64_t *gkey, uint64_t *f64key, void *stream);
/* S7 step 2.  gf64: [nq] MIN over shards of f64key; gkey as for refine.  out[i] = (global
 * index << 32) | fp32 bits of the local candidate with fp64 value == gf64[i] and the lowest
 * index (INT64_MAX if none); a MIN over shards gives the final answer (key_format 1).
 * Same ws and arguments as the preceding refine call. */
NNDTW_API int nndtw_classify_resolve(void *ws, size_t ws_bytes, const float *q, int64_t nq,
                           const float *t, int64_t nt, int32_t L, int32_t w,
                           int64_t index_base, const uint64_t *gkey, const uint64_t *gf64,
                           uint64_t *out, void *stream);

/*
 * Decode keys: key_format 0 = (f32 bits << 32) | idx (nndtw_classify), 1 = (idx << 32) | f32
 * bits (nndtw_classify_resolve).  idx_out [nq] int64, label_out [nq] int32 (labels[idx]),
 * dist_out [nq] float (squared distance); each nullable.  labels: [nlabels] (global ids).
 */
NNDTW_API int nndtw_finalize(const uint64_t *key, int64_t nq, int32_t key_format, const int32_t *labels,
                   int64_t nlabels, int64_t *idx_out, int32_t *label_out, float *dist_out,
                   void *stream);

/*
 * S8 -- leave-one-out warping-window search (reading C17).  For every window
 * windows[p] (host array, absolute w, any order) and every held-out series i in
 * [q_begin, q_end): the exact 1-NN of x[i] among x[j], j != i, under DTW_{w_p}
 * (ties -> lowest j, fp64-exact via the local re-rank).  errors[p] += #{i: labels[nn] !=
 * labels[i]} (device int64 [nw], accumulated -- zero it first); nn_out: [nw][q_end-q_begin]
 * int32, nullable.  The train set is all n series (replicated); shard the held-out range
 * across ranks and SUM errors.  Windows are processed in the given order and each window is
 * seeded with the previous window's neighbour (DTW is monotone in w).
 */
NNDTW_API size_t nndtw_loocv_workspace_bytes(int64_t n, int32_t L, int64_t q_begin, int64_t q_end);
NNDTW_API int nndtw_loocv_window(const float *x, const int32_t *labels, int64_t n, int32_t L,
                       const int32_t *windows, int32_t nw, int32_t v, int64_t q_begin,
                       int64_t q_end, void *ws, size_t ws_bytes, int64_t *errors,
                       int32_t *nn_out, nndtw_stats *stats, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* NNDTW_H */
