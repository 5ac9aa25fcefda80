// launchers.cuh -- host launch functions of the kernels (internal to libnndtw.so).
#pragma once
#include "common.cuh"

namespace nndtw {

int launch_envelopes(const float *x, int64_t n, int L, int w, float *U, float *Lo,
                     nndtw_kim *kim, cudaStream_t st);
int launch_series_stats(const float *x, int64_t n, int L, nndtw_kim *kim, cudaStream_t st);
int launch_check_finite(const float *x, int64_t n, int32_t *bad, cudaStream_t st);
int launch_lb(const float *q, int64_t nq, const nndtw_kim *qkim, const float *t,
              const float *U, const float *Lo, const nndtw_kim *tkim, int64_t nt, int L, int w,
              int v, int with_kim, int64_t self_offset, float *lb, int64_t ldlb,
              unsigned long long *minkey, cudaStream_t st, int keogh = 0, int transposed = 0,
              int no_bridge = 0);
// Two-stage S2 (lb_sparse.cu): after stage A (launch_lb with no_bridge) and the first seed
// round, the LB_Keogh bridge only for the pairs the partial cascade did not prune.
int launch_col_compact(const float *lb, int64_t ldlb, int64_t nq, int64_t nt,
                       const unsigned long long *key, float eps_p, long long *col_count,
                       long long *col_off, long long *col_fill, int32_t *qlist,
                       unsigned long long qlist_cap, unsigned *colmask,
                       unsigned long long *cap_overflow, int num_sms, cudaStream_t st);
int launch_lb_sparse(const float *q, const nndtw_kim *qkim, int64_t nq, const float *t,
                     const float *U, const float *Lo, const nndtw_kim *tkim, int64_t nt, int L,
                     int w, int v, const long long *col_off, const int32_t *qlist, float *bval,
                     float *lb, int64_t ldlb, unsigned long long *minkey2, int num_sms,
                     cudaStream_t st);
int launch_seed_items2(const unsigned long long *minkey2, const unsigned long long *minkey1,
                       const int32_t *seed2, int64_t nq, int64_t nt, Item *items,
                       unsigned long long *count, cudaStream_t st);
// S3 prune counters per cascade level (stats; lb.cu k_lb_tile in level-count mode)
int launch_lb_level_counts(const float *q, int64_t nq, const nndtw_kim *qkim, const float *t,
                           const nndtw_kim *tkim, int64_t nt, int L, int w, int v, int with_kim,
                           int keogh, int64_t self_offset, const float *lb, int64_t ldlb,
                           const unsigned long long *key, const unsigned long long *minkey,
                           const int32_t *seed2, float eps_p, unsigned long long *level_cnt,
                           cudaStream_t st);
// NEXT-4 (bounds_improved.cu): lb[q][n] += sum over columns [c_lo, c_hi) of the LB_Keogh term of
// t_n against the envelope of q's projection onto t_n's envelope (LB_Improved's second pass, O(L))
int launch_lb_improved_pass(const float *q, int64_t nq, const float *t, const float *U,
                            const float *Lo, int64_t nt, int L, int w, int c_lo, int c_hi,
                            float *lb, int64_t ldlb, int num_sms, cudaStream_t st);
// S2 finish for bounds assembled outside the tile kernel: max with LB_Kim (qkim non-null), the
// leave-one-out self pair -> NaN, per-query argmin key (atomicMin into minkey, pre-filled kNone)
int launch_bound_finish(float *lb, int64_t ldlb, int64_t nq, int64_t nt, const float *q,
                        const float *t, const nndtw_kim *qkim, const nndtw_kim *tkim, int L,
                        int64_t self_offset, unsigned long long *minkey, cudaStream_t st);
// S2 extras (bounds_next.cu): LB_New, all pairs (kind 0; O(L*w) per pair as the bound is defined)
int launch_lb_pairs(int kind, const float *q, int64_t nq, const float *t, const float *U,
                    const float *Lo, int64_t nt, int L, int w, float *lb, int64_t ldlb,
                    cudaStream_t st);
int launch_row_argmin(const float *lb, int64_t ldlb, int64_t nq, int64_t nt,
                      unsigned long long *minkey, cudaStream_t st);
int launch_tightness(const float *lb, const float *d, int64_t n, double *sum,
                     unsigned long long *count, unsigned *max_bits, int num_sms,
                     cudaStream_t st);
int launch_fill_u64(unsigned long long *p, int64_t n, unsigned long long v, cudaStream_t st);
int launch_classify_init(int64_t nq, unsigned long long *key, unsigned long long *minkey,
                         unsigned long long *f64key, unsigned long long *resolve_out,
                         unsigned *overflow, unsigned *tiecnt, unsigned long long *counters,
                         int ncounters, unsigned long long *bucket_count, cudaStream_t st);
int launch_seed_items(const unsigned long long *minkey, const int32_t *seed2, int64_t nq,
                      int64_t nt, Item *items, unsigned long long *count, cudaStream_t st);
int launch_list_compact(const long long *col_off, const int32_t *blist, const float *bval,
                        int64_t nt, const unsigned long long *key,
                        const unsigned long long *minkey, const int32_t *seed2, float eps_p,
                        Item *items, unsigned long long *count, unsigned long long *buckets,
                        unsigned long long capacity, unsigned long long *cap_overflow,
                        int num_sms, cudaStream_t st);
int launch_compact(const float *lb, int64_t ldlb, int64_t nq, int64_t nt,
                   const unsigned long long *key, const unsigned long long *minkey,
                   const int32_t *seed2, float eps_p, Item *items, unsigned long long *count,
                   unsigned long long *buckets, unsigned long long capacity,
                   unsigned long long *cap_overflow, int num_sms, cudaStream_t st);
int launch_cells_prefix(int L, int w, long long *prefix, cudaStream_t st);
int launch_refine(TieEntry *e, const unsigned long long *count, unsigned long long cap,
                  const float *A, const float *B, int L, int w, const unsigned long long *gkey,
                  float eps_t, unsigned long long *f64key, unsigned long long *counters,
                  const unsigned *tiecnt, const unsigned *overflow, int num_sms,
                  cudaStream_t st);
int launch_tie_count(const TieEntry *e, const unsigned long long *count, unsigned long long cap,
                     const unsigned long long *gkey, float eps_t, unsigned *tiecnt, int num_sms,
                     cudaStream_t st);
int launch_refine_overflow(const unsigned long long *log_count, unsigned long long log_cap,
                           const unsigned *overflow, int64_t nq, const float *lb, int64_t ldlb,
                           int64_t nt, const float *A, const float *B, int L, int w,
                           const unsigned long long *gkey, float eps_p, int pass,
                           unsigned long long *f64key, const unsigned long long *gf64,
                           int64_t index_base, unsigned long long *out, int num_sms,
                           cudaStream_t st);
int launch_resolve(const TieEntry *e, const unsigned long long *count, unsigned long long cap,
                   const unsigned long long *gf64, int64_t index_base, unsigned long long *out,
                   int num_sms, cudaStream_t st);
int launch_swap_key(const unsigned long long *in, int64_t nq, unsigned long long *out,
                    cudaStream_t st);
int launch_finalize(const unsigned long long *key, int64_t nq, int fmt, const int32_t *labels,
                    int64_t nlabels, int64_t *idx_out, int32_t *label_out, float *dist_out,
                    cudaStream_t st);
int launch_count_errors(const unsigned long long *key, int64_t nq, const int32_t *labels,
                        int64_t q_begin, int64_t *errors, int32_t *nn_out, int32_t *prev_nn,
                        cudaStream_t st);

// S4 dispatch: picks the band-wavefront kernel (2w+2 <= 32*32 slots) or the row-strip kernel
// (long windows).  mode 0 = search (items + device count, atomicMin into key, tie log),
// mode 1 = batch (ia/ib/cutoff/out, nitems_host pairs).  Returns 0 or an NNDTW_E_* code.
// S4 band-limited pass (dtw_band.cu): its window for a distance window w, or -1
int band_adapt_window(int L, int w, bool full_window = false);
int dispatch_dtw(const float *A, const float *B, int64_t na, int64_t nb, const Item *items,
                 const unsigned long long *nitems_dev, unsigned long long item_cap,
                 const int32_t *ia, const int32_t *ib, int64_t nitems_host, int L, int w,
                 int mode, unsigned long long *key, int64_t index_base, float eps_t, TieLog log,
                 unsigned long long *counters, const long long *cells_prefix,
                 const float *cutoff, float *out, cudaStream_t st, int num_sms,
                 float *apad_ws = nullptr, int64_t apad_cap = 0, int adapt_w = -1,
                 Item *fb_items = nullptr, unsigned long long *fb_count = nullptr,
                 int fbsel = 0);
// floats per query row of the band kernel's padded A copy (an upper bound of its row length
// seglen for any window: padl + L + padr <= L + w + R + 48)
inline int64_t band_apad_row_floats(int L) { return 2 * (int64_t)L + 128; }

int launch_key_index(const unsigned long long *key, int64_t nq, int64_t nt, int32_t *idx,
                     cudaStream_t st);
// ed_seed.cu: per-query argmin of the Euclidean distance over all train series (tensor cores)
int ed_seed_supported(int L);
size_t ed_seed_scratch_bytes(int64_t nq, int64_t nt, int L);
int launch_ed_seed(const float *q, int64_t nq, const float *t, int64_t nt, int L, void *scratch,
                   unsigned long long *key, int num_sms, cudaStream_t st);

int dtw_kernel_kind(int L, int w);  // 0 = k_dtw_w0, 1 = k_dtw_band, 2 = k_dtw_strip
int strip_rows_per_lane(int L);
int launch_dtw_strip(const float *A, const float *B, const Item *items,
                     const unsigned long long *nitems_dev, unsigned long long item_cap,
                     const int32_t *ia, const int32_t *ib, int64_t nitems_host, int L, int w,
                     int mode, unsigned long long *key, int64_t index_base, float eps_t,
                     TieLog log, unsigned long long *counters, const long long *cells_prefix,
                     const float *cutoff, float *out, cudaStream_t st, int num_sms,
                     const unsigned long long *fb_count = nullptr, int fbsel = 0);

}  // namespace nndtw
