// dtw_strip.cu -- S4 for long windows (w too wide for the band-register layout, e.g.
// BJ:configs[4], L = 2048, w = L-1): windowed DTW (Eq. 1) by row strips.
//
// B200 design.  One warp per (query, train) pair.  The matrix is
// cut into strips of H = 32*RR rows; lane l owns rows i0 + l*RR .. i0 + l*RR + RR-1, split into
// KS sub-blocks of RB = RR/KS rows, and sweeps the columns with a staggered skew: on step s,
// sub-block k of lane l is at column j = s - l*KS - k.  Then every cell's inputs were produced
// on an earlier step -- the row above a sub-block is the previous sub-block's bottom row one
// step earlier (one register; across lanes one warp shuffle), the diagonal two steps earlier --
// so the KS sub-blocks of a step are independent dependency chains (a lane evaluating its RR
// rows top-down at one column is one serial chain of RR fused cells, which left the SM issue
// mostly waiting on the previous cell: KS = 4 cuts that chain 4x).  Inside a sub-block:
//     D(i,j) = (A_i - B_j)^2 + min(D(i,j-1), D(i-1,j-1), D(i-1,j))
// The bottom row of a strip is written to shared memory (the next strip's "row above") and its
// minimum -- a complete row, hence a cut of every warping path (reading C14) -- decides early
// abandoning against the live best-so-far.  B and the strip rows live in shared memory; padded
// B values (+/-2^64) make out-of-range columns +inf.  When w < L-1, cells with |i-j| > w are
// masked to +inf (MASK variant).
#include <cstdlib>
#include <type_traits>

#include "launchers.cuh"

namespace nndtw {

constexpr int STRIP_PAD = 136;  // B pads on each side (>= 32*KS skew steps, KS <= 4)

struct StripParams {
    const float *A, *B;
    const Item *items;
    const unsigned long long *nitems_dev;
    unsigned long long item_cap;
    const int32_t *ia, *ib;
    int64_t nitems_host;
    int L, w, mode;
    unsigned long long *key;
    int64_t index_base;
    float eps_t;
    float eps_p;  // search mode: skip items with lb > bsf*(1+eps_p)
    TieLog log;
    unsigned long long *counters;
    const long long *cells_prefix;
    const float *cutoff;
    float *out;
    int rowlen;  // floats per warp region: (L + 2*PAD) for B, L + 32*KS + 1 for the row
                 // buffer, then ceil(L/32) block suffix minima of the row buffer
    int ks;      // sub-blocks per lane (the template KS; sizes rowlen)
    // full-window pass after the band-limited one (dtw_band.cu): run the items appended after
    // the survivors (fb_count of them), or every survivor again if they did not all fit
    const unsigned long long *fb_count;  // nullable: the band-limited passes' append counts
    int fbsel;                           // which level's appended items to run (>= 1)
};

template <int RR, int KS, bool MASK>
__global__ void __launch_bounds__(128) k_dtw_strip(StripParams p) {
    static_assert(RR % KS == 0, "sub-blocks split the lane's rows evenly");
    constexpr int RB = RR / KS;
    extern __shared__ __align__(16) float smem_s[];
    const int lane = threadIdx.x & 31;
    // warp index through a shuffle and every data-dependent branch through a vote: the loop
    // bounds and exits are then provably warp-uniform, and the per-step shuffles compile to
    // plain SHFLs instead of divergence-safe WARPSYNC / collective sequences
    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);
    const int L = p.L, w = p.w;
    float *sB = smem_s + (size_t)warp * p.rowlen;           // B[j] at sB[PAD + j]
    float *bsuf = sB + (L + 2 * STRIP_PAD) + (L + 32 * KS + 1);  // [ceil(L/32)]
    float *rb = sB + (L + 2 * STRIP_PAD);                    // rb[1 + j] = row above, column j
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    int64_t nitems = p.nitems_host;
    int64_t ioff = 0;
    if (p.mode == 0) {
        unsigned long long c = *p.nitems_dev;
        nitems = (int64_t)(c < p.item_cap ? c : p.item_cap);
        if (p.fb_count != nullptr && p.fbsel >= 1) {  // the items level fbsel - 1 appended
            const unsigned long long f0 = p.fb_count[0];
            const unsigned long long off = c + (p.fbsel >= 2 ? f0 : 0ull);
            const unsigned long long n = p.fb_count[p.fbsel - 1];
            if (off + n <= p.item_cap) {
                ioff = (int64_t)off;
                nitems = (int64_t)n;
            }  // else: every survivor again
        }
    }
    // B pads: -2^64*(k+1) before, +2^64*(k+1) after (distinct from the A pad below)
    for (int x = lane; x < STRIP_PAD; x += 32) {
        sB[STRIP_PAD - 1 - x] = -0x1p64f * (float)(x + 1);
        sB[STRIP_PAD + L + x] = 0x1p64f * (float)(x + 1);
    }
    const int H = 32 * RR;
    const int nstrips = (L + H - 1) / H;
    const int nsteps = L + 32 * KS - 1;
    long long my_items = 0, my_aband = 0, my_cells = 0, my_skipped = 0;

    for (int64_t it = gw; it < nitems; it += nwarps) {
        unsigned a_idx, b_idx;
        float thr_batch = kInf;
        if (p.mode == 0) {
            Item itm = p.items[ioff + it];
            a_idx = itm.q;
            b_idx = itm.n;
            float live = key_dist(ld_relaxed_u64(p.key + a_idx));
            live = __shfl_sync(0xffffffffu, live, 0);
            if (__any_sync(0xffffffffu, itm.lb > live * (1.0f + p.eps_p))) {  // pruned by the live best-so-far
                ++my_skipped;
                continue;
            }
        } else {
            a_idx = p.ia ? (unsigned)p.ia[it] : (unsigned)it;
            b_idx = p.ib ? (unsigned)p.ib[it] : (unsigned)it;
            thr_batch = p.cutoff ? p.cutoff[it] * (1.0f + p.eps_t) : kInf;
        }
        const float *ga = p.A + (int64_t)a_idx * L;
        const float *gb = p.B + (int64_t)b_idx * L;
        __syncwarp();
        for (int x = lane; x < L; x += 32) cp_async4(sB + STRIP_PAD + x, gb + x);
        for (int x = lane; x < L + 32 * KS; x += 32) rb[1 + x] = kInf;  // D(-1, j) = +inf; pads
        if (lane == 0) rb[0] = 0.0f;                          // D(-1,-1) = 0
        cp_async_wait_all();
        __syncwarp();

        float res = kInf;
        bool abandoned = false;
        int strips_done = 0;
        long long partial_cells = 0;  // cells of a strip left at a mid-strip checkpoint
        for (int st = 0; st < nstrips; ++st) {
            const int i0 = st * H + lane * RR;  // first row of this lane
            float a[RR], Dl[RR];
#pragma unroll
            for (int r = 0; r < RR; ++r) {
                const int i = i0 + r;
                a[r] = i < L ? __ldg(ga + i) : 0x1p64f * 3.0f;  // rows past the end: +inf cells
                Dl[r] = kInf;                                    // D(i, -1) = +inf
            }
            // rows of a sub-block in aligned register pairs: the differences of two rows against
            // the sub-block's one column value are one FADD2 with a broadcast operand
            // (a_R - b, a_R+1 - b) -- bit-identical to two FADDs, half the issue slots
            unsigned long long ap[RR / 2 > 0 ? RR / 2 : 1];
#pragma unroll
            for (int m = 0; m < RR / 2; ++m) ap[m] = f2_pack(a[2 * m], a[2 * m + 1]);
            // Block suffix minima of the row above (the previous strip's bottom row):
            // bsuf[m] = min over columns >= 32m.  With the lanes' frontier they form a cut of
            // every warping path at any step of the strip (see the checkpoint below).
            {
                const int nblk = (L + 31) >> 5;
                float carry = kInf;
                for (int k0 = ((nblk - 1) >> 5) << 5; k0 >= 0; k0 -= 32) {
                    const int m = k0 + lane;
                    float bm = kInf;
                    if (m < nblk)
                        for (int j = 32 * m; j < 32 * m + 32 && j < L; ++j) bm = fminf(bm, rb[1 + j]);
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        const float o = __shfl_down_sync(0xffffffffu, bm, off);
                        if (lane + off < 32) bm = fminf(bm, o);
                    }
                    bm = fminf(bm, carry);
                    if (m < nblk) bsuf[m] = bm;
                    carry = __shfl_sync(0xffffffffu, bm, 0);
                }
                __syncwarp();
            }
            // the live best-so-far, used for the abandon tests of this strip
            float thr = thr_batch;
            if (p.mode == 0) thr = key_dist(ld_relaxed_u64(p.key + a_idx)) * (1.0f + p.eps_t);
            float up_prev = (lane == 0) ? rb[0] : kInf;  // diagonal input of the top row
            float pb2[KS];  // bottom of sub-block k two steps ago (diagonal input of k+1)
#pragma unroll
            for (int k = 0; k < KS; ++k) pb2[k] = kInf;
            float rowmin = kInf;
            const bool last = (st == nstrips - 1);
            // One step: sub-block k of this lane at column s - lane*KS - k.  CHECK: ramp-up /
            // ramp-down steps where some column is outside [0, L) (range-checked); steady steps
            // need no checks.
            // bw: nullptr -> each sub-block loads its B value; else bw[-k] is sub-block k's value
            // (the 4-step groups below fetch them as two aligned float4 per group)
            auto step = [&](int s, auto check_tag, const float *bw) {
                constexpr bool CHECK = decltype(check_tag)::value;
                // the lane above's last sub-block bottom, one step ago, at this lane's column
                const float from_up = __shfl_up_sync(0xffffffffu, Dl[RR - 1], 1);
                const float rbv = rb[1 + s];        // lane 0's column; rb padded with +inf
                const float up = (lane == 0) ? rbv : from_up;
                float nb2[KS];
#pragma unroll
                for (int k = KS - 1; k >= 0; --k) {  // descending: k reads k-1's old bottom
                    const int j = s - lane * KS - k;
                    const float b = bw ? bw[-k] : sB[STRIP_PAD + j];  // pads: +inf cells
                    float dgv = (k == 0) ? up_prev : pb2[k - 1];
                    float upv = (k == 0) ? up : Dl[k * RB - 1];
                    nb2[k] = Dl[k * RB + RB - 1];
                    float tt[RB];
#pragma unroll
                    for (int r = 0; r < RB; ++r) {
                        const int R = k * RB + r;
                        if ((RB % 2) == 0 && (r % 2) == 0) {
                            f2_unpack(f2_sub(ap[R / 2], f2_pack(b, b)), tt[r], tt[r + 1]);
                        } else if ((RB % 2) != 0) {
                            tt[r] = a[R] - b;
                        }
                    }
#pragma unroll
                    for (int r = 0; r < RB; ++r) {
                        const int R = k * RB + r;
                        const float t = tt[r];
                        const float old = Dl[R];
                        float nv = fmaf(t, t, fminf(fminf(old, dgv), upv));
                        if (MASK) {
                            const int i = i0 + R;
                            if (j - i > w || i - j > w) nv = kInf;
                        }
                        Dl[R] = nv;
                        dgv = old;
                        upv = nv;
                    }
                }
#pragma unroll
                for (int k = 0; k < KS; ++k) pb2[k] = nb2[k];
                up_prev = up;
                const int jb = s - lane * KS - (KS - 1);  // the bottom row's column
                const bool jin = !CHECK || (jb >= 0 && jb < L);
                if (lane == 31 && jin) {
                    rb[1 + jb] = Dl[RR - 1];
                    rowmin = fminf(rowmin, Dl[RR - 1]);
                }
            };
            // steady phase: every column in [0, L-1) <=> 32KS-1 <= s < L-1 (no sub-block reaches
            // the last column, where the result is captured); the rest is range-checked
            const bool has_steady = L >= 32 * KS + 1;
            const int s_lo = has_steady ? 32 * KS - 1 : nsteps, s_hi = has_steady ? L - 1 : nsteps;
            for (int s = 0; s < s_lo; ++s) step(s, std::true_type{}, nullptr);
            int s = s_lo;
            bool cut_abandon = false;
            for (; s + 3 < s_hi; s += 4) {
                if ((s & 31) == 31 && s > 32 * KS) {
                    // Checkpoint: the computed cells of this strip form a staircase (row by row
                    // the last column is non-increasing, by one between consecutive sub-blocks
                    // and lanes).  Every warping path leaves it through a frontier cell: the
                    // last cell of each row (Dl), the cell left of it in the bottom row of each
                    // sub-block or lane above (pb2, up_prev: their diagonal successor is not
                    // computed), the bottom row of the strip so far (lane 31's rowmin), or the
                    // previous strip's bottom row from column s-1 on (bsuf[s/32] covers columns
                    // >= s-31, a superset).  D is non-decreasing along paths, so the minimum is a
                    // lower bound of the distance (reading C14).
                    float mv = up_prev;
#pragma unroll
                    for (int r = 0; r < RR; ++r) mv = fminf(mv, Dl[r]);
#pragma unroll
                    for (int k = 0; k < KS; ++k) mv = fminf(mv, pb2[k]);
                    if (lane == 31) mv = fminf(mv, rowmin);
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1)
                        mv = fminf(mv, __shfl_xor_sync(0xffffffffu, mv, off));
                    mv = fminf(mv, bsuf[s >> 5]);
                    float th = thr_batch;
                    if (p.mode == 0) th = key_dist(ld_relaxed_u64(p.key + a_idx)) * (1.0f + p.eps_t);
                    th = __shfl_sync(0xffffffffu, th, 0);  // one view of the live best per warp
                    if (__any_sync(0xffffffffu, !(mv <= th))) {
                        cut_abandon = true;
                        break;
                    }
                }
                if constexpr (KS == 4) {
                    // the group's B values: columns x0-3 .. x0+3 of this lane, x0 = s - 4*lane;
                    // PAD + s = 3 (mod 4) at every group start (s_lo = 127, PAD = 136), so they
                    // are two aligned float4 -- 2 loads per 4 steps, and the 32 lanes' float4
                    // are contiguous (no bank conflicts), instead of 4 stride-4 loads per step
                    static_assert((STRIP_PAD + 32 * KS - 1) % 4 == 3, "group alignment");
                    const float *bp = sB + STRIP_PAD + s - 4 * lane - 3;
                    const float4 lo = *reinterpret_cast<const float4 *>(bp);
                    const float4 hi = *reinterpret_cast<const float4 *>(bp + 4);
                    const float bw[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
                    // step s+m, sub-block k: column x0 + m - k = bw[3 + m - k]
                    step(s, std::false_type{}, bw + 3);
                    step(s + 1, std::false_type{}, bw + 4);
                    step(s + 2, std::false_type{}, bw + 5);
                    step(s + 3, std::false_type{}, bw + 6);
                } else {
                    step(s, std::false_type{}, nullptr);
                    step(s + 1, std::false_type{}, nullptr);
                    step(s + 2, std::false_type{}, nullptr);
                    step(s + 3, std::false_type{}, nullptr);
                }
            }
            if (cut_abandon) {
                // in-band cells of the complete strips plus this strip's computed columns
                if (p.counters) {
                    long long c = 0;
#pragma unroll
                    for (int r = 0; r < RR; ++r) {
                        const int i = i0 + r;
                        const int jmax = s - 1 - lane * KS - r / RB;  // last column computed
                        if (i < L && jmax >= 0) {
                            const int lo = i - w > 0 ? i - w : 0;
                            int hi = i + w < L - 1 ? i + w : L - 1;
                            hi = hi < jmax ? hi : jmax;
                            c += hi >= lo ? hi - lo + 1 : 0;
                        }
                    }
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
                    partial_cells = c;
                }
                abandoned = true;
                break;
            }
            for (; s < s_hi; ++s) step(s, std::false_type{}, nullptr);
            // ramp-down; row L-1 (last strip) reaches column L-1 on step s_star, uniform
            const int own_l = ((L - 1) % H) / RR, own_r = (L - 1) - (st * H + own_l * RR);
            const int s_star = (L - 1) + own_l * KS + own_r / RB;
            for (s = s_hi; s < nsteps; ++s) {
                step(s, std::true_type{}, nullptr);
                if (last && s == s_star && lane == own_l) {
#pragma unroll
                    for (int r = 0; r < RR; ++r)
                        if (r == own_r) res = Dl[r];
                }
            }
            __syncwarp();
            // column -1 of the next strip's row above is +inf (only row -1 has the 0 corner)
            if (lane == 0) rb[0] = kInf;
            ++strips_done;
            if (!last) {
                const float rm = __shfl_sync(0xffffffffu, rowmin, 31);
                if (__any_sync(0xffffffffu, !(rm <= thr))) {
                    abandoned = true;
                    break;
                }
            }
            __syncwarp();
        }
        // the lane that owned row L-1 holds the result
        const int owner = ((L - 1) % H) / RR;
        res = __shfl_sync(0xffffffffu, res, owner);
        if (lane == 0) {
            if (p.mode == 0) {
                if (!abandoned) {
                    unsigned gidx = (unsigned)(p.index_base + b_idx);
                    unsigned long long old = atomicMin(p.key + a_idx, make_key(res, gidx));
                    float best = fminf(res, key_dist(old));
                    if (res <= best * (1.0f + p.eps_t)) {
                        unsigned long long slot = atomicAdd(p.log.count, 1ull);
                        if (slot < p.log.capacity) {
                            TieEntry e;
                            e.q = a_idx;
                            e.n = b_idx;
                            e.d32 = res;
                            e.pad = 0.0f;
                            e.d64 = 0.0;
                            p.log.e[slot] = e;
                        } else {
                            p.log.overflow[a_idx] = 1u;
                        }
                    }
                }
            } else {
                p.out[it] = abandoned ? kInf : res;
            }
            if (p.counters) {
                my_items += 1;
                my_aband += abandoned ? 1 : 0;
                // in-band cells of the completed rows (strips are row ranges), closed form
                long long c;
                if (!abandoned) {
                    c = p.cells_prefix[2 * L - 2];
                } else {
                    const long long R = strips_done * H < L ? strips_done * H : L;
                    long long t = L - w;  // rows i with i + w <= L-1
                    t = t < 0 ? 0 : (t > R ? R : t);
                    long long s1 = t * (t - 1) / 2 + t * (long long)w + (R - t) * (L - 1);
                    long long m = R - 1 - w;
                    long long s2 = m > 0 ? m * (m + 1) / 2 : 0;
                    c = s1 - s2 + R + partial_cells;
                }
                my_cells += c;
            }
        }
    }
    if (p.counters && lane == 0 && my_skipped > 0)
        atomicAdd(p.counters + CNT_SKIPPED, (unsigned long long)my_skipped);
    if (p.counters && lane == 0 && my_items > 0) {
        atomicAdd(p.counters + CNT_ITEMS, (unsigned long long)my_items);
        atomicAdd(p.counters + CNT_ABANDONED, (unsigned long long)my_aband);
        atomicAdd(p.counters + CNT_CELLS, (unsigned long long)my_cells);
    }
}

// Rows per lane: the strips cover ceil(L / 32RR) * 32RR rows; take the RR in {32, 16, 12, 10, 8}
// that wastes the fewest rows (ties: the larger RR, fewer strips).  RR = 32 (8 rows per
// sub-block at KS = 4) amortises the per-step overhead (the cross-lane shuffle, the row-above
// read, the bottom-row store and minimum, register rotation) over twice the cells: raw rate at
// L = 2048, full window, 7.24 -> 8.07 Tcells/s; config 4 6.20 -> 6.64 Tcells/s in search mode
// (167 registers; 12 warps/SM, as the shared-memory rows allow anyway).
int strip_rows_per_lane(int L) {
    static const char *rre = getenv("NNDTW_STRIP_RR");  // experiments: force 32/16/12/10/8
    if (rre) {
        const int r = atoi(rre);
        if (r == 32 || r == 16 || r == 12 || r == 10 || r == 8) return r;
    }
    int best = 8;
    long long best_rows = -1;
    for (int RR : {32, 16, 12, 10, 8}) {
        const long long H = 32LL * RR;
        const long long rows = (L + H - 1) / H * H;
        if (best_rows < 0 || rows < best_rows) {
            best_rows = rows;
            best = RR;
        }
    }
    return best;
}

template <int RR, int KS, bool MASK>
static int launch_strip_t(StripParams &p, cudaStream_t st, int num_sms) {
    auto kern = k_dtw_strip<RR, KS, MASK>;
    // up to 4 warps per CTA, fewer when the rows are long (L up to 8192: 66 KB per warp)
    int warps = (int)((220 * 1024) / ((size_t)p.rowlen * sizeof(float)));
    if (warps > 4) warps = 4;
    if (warps < 1) return -2;
    size_t smem = (size_t)warps * p.rowlen * sizeof(float);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, warps * 32, smem);
    if (occ < 1) occ = 1;
    int64_t grid = (int64_t)num_sms * occ;
    if (p.mode == 1) {
        int64_t need = (p.nitems_host + warps - 1) / warps;
        if (need < grid) grid = need > 0 ? need : 1;
    }
    kern<<<(unsigned)grid, warps * 32, smem, st>>>(p);
    count_launch(1, __func__);
    return 0;
}

int launch_dtw_strip(const float *A, const float *B, const Item *items,
                     const unsigned long long *nitems_dev, unsigned long long item_cap,
                     const int32_t *ia, const int32_t *ib, int64_t nitems_host, int L, int w,
                     int mode, unsigned long long *key, int64_t index_base, float eps_t,
                     TieLog log, unsigned long long *counters, const long long *cells_prefix,
                     const float *cutoff, float *out, cudaStream_t st, int num_sms,
                     const unsigned long long *fb_count, int fbsel) {
    StripParams p;
    p.fb_count = fb_count;
    p.fbsel = fbsel;
    p.A = A;
    p.B = B;
    p.items = items;
    p.nitems_dev = nitems_dev;
    p.item_cap = item_cap;
    p.ia = ia;
    p.ib = ib;
    p.nitems_host = nitems_host;
    p.L = L;
    p.w = w;
    p.mode = mode;
    p.key = key;
    p.index_base = index_base;
    p.eps_t = eps_t;
    p.eps_p = eps_prune(L);
    p.log = log;
    p.counters = counters;
    p.cells_prefix = cells_prefix;
    p.cutoff = cutoff;
    p.out = out;
    const bool mask = w < L - 1;
    const int RR = strip_rows_per_lane(L);
    // sub-blocks per lane: the stagger costs 32*KS-1 ramp steps per strip of L + 32*KS - 1, so
    // short rows keep fewer sub-blocks (L = 256: KS = 4 would add 50 % steps); KS divides RR
    int ks = L >= 1024 ? 4 : (L >= 512 ? 2 : 1);
    // search mode with 32-row lanes: most items are abandoned inside the first strip, where
    // the 127 ramp steps of KS = 4 weigh more than the shorter chains cost (config 4: 6.60 ->
    // 6.76 Tcells/s; raw full matrices prefer KS = 4: 8.07 vs 7.95)
    if (mode == 0 && RR == 32 && ks == 4) ks = 2;
    if (RR % ks != 0) ks = 2;
    static const char *kse = getenv("NNDTW_STRIP_KS");  // experiments: force 1, 2 or 4
    if (kse && RR % atoi(kse) == 0) ks = atoi(kse);
    p.ks = ks;
    p.rowlen = (L + 2 * STRIP_PAD) + (L + 32 * p.ks + 1) + (L + 31) / 32;
    p.rowlen = (p.rowlen + 3) / 4 * 4;
#define STRIP_KS(RRv)                                                                             \
    if (RR == RRv) {                                                                              \
        if (ks == 4)                                                                              \
            return mask ? launch_strip_t<RRv, (RRv % 4 == 0 ? 4 : 2), true>(p, st, num_sms)      \
                        : launch_strip_t<RRv, (RRv % 4 == 0 ? 4 : 2), false>(p, st, num_sms);    \
        if (ks == 2)                                                                              \
            return mask ? launch_strip_t<RRv, 2, true>(p, st, num_sms)                            \
                        : launch_strip_t<RRv, 2, false>(p, st, num_sms);                          \
        return mask ? launch_strip_t<RRv, 1, true>(p, st, num_sms)                                \
                    : launch_strip_t<RRv, 1, false>(p, st, num_sms);                              \
    }
    STRIP_KS(32)
    STRIP_KS(16)
    STRIP_KS(12)
    STRIP_KS(10)
    STRIP_KS(8)
#undef STRIP_KS
    return -1;
}

}  // namespace nndtw
