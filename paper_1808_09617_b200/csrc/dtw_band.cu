// dtw_band.cu -- S4: windowed DTW (Eq. 1; Sakoe-Chiba band P:164-171) on a list of
// (query, train) work items, with early abandoning against a per-query best-so-far.
//
// B200 design.  A group of G lanes owns one DP matrix; lane g
// holds R (even) consecutive band offsets d = j - i, slots s = g*R + r <-> d = s - w, in
// registers D[r].  The matrix is swept by anti-diagonals k = i + j: cell (k, d) depends on
// (k-2, d) [diagonal move], (k-1, d-1) [left] and (k-1, d+1) [up], so one register per offset
// suffices -- on diagonal k only offsets with d = k (mod 2) exist and they read neighbours of
// the other parity, last written on diagonal k-1:
//     D[r] <- (A_i*sc_r - B_j)^2 + min(D[r], D[r-1], D[r+1])    (FFMA, FMNMX3, FFMA)
// Neighbours across lanes: one warp shuffle per diagonal (shfl_up of D[R-1] on even-phase
// diagonals, shfl_down of D[0] on odd ones).  A and B sit in shared memory with index-dependent
// pads (+-2^64*k, distinct per index) so that cells outside the matrix get +inf (their squared
// difference overflows) while the cells (x, x) outside it get 0 -- this makes D(-1,-1) = 0 the
// start condition and carries D(L-1,L-1) unchanged to the end of the last unrolled period, so
// the R-diagonal period is fully unrolled with no boundary tests.  The band edge d = w+1 is a
// "kill" slot whose A value is scaled by +inf (NaN/inf results, ignored by fminf); slots
// beyond it stay +inf.  Early abandoning (reading C14): after every period the registers hold
// two consecutive anti-diagonals, a cut of every warping path; the group abandons when every
// lane's minimum exceeds bsf*(1+eps_t) (one warp ballot).  GA variant (config 2's layout): the
// query rows come through L1 from a padded copy in the classify workspace (k_pad_rows) and only
// the train row is staged, which halves the shared memory per group (16 warps/SM instead of 8).
#include <cstdlib>

#include "launchers.cuh"

namespace nndtw {

struct BandParams {
    const float *A, *B;
    const Item *items;                    // search mode: (q, n)
    const unsigned long long *nitems_dev; // search mode: device count
    unsigned long long item_cap;          // search mode: capacity of items
    const int32_t *ia, *ib;               // batch mode (nullable = identity)
    int64_t nitems_host;                  // batch mode count
    int L, w, G, gpw, nper, k0, padl, seglen, vec4;
    int mode;                             // 0 search, 1 batch
    unsigned long long *key;
    int64_t index_base;
    float eps_t;
    float eps_p;                          // search mode: skip items with lb > bsf*(1+eps_p)
    TieLog log;
    unsigned long long *counters;         // nullable
    const long long *cells_prefix;        // [2L-1], nullable iff counters null
    const float *cutoff;                  // batch, nullable
    float *out;                           // batch
    int64_t dbg_na, dbg_nb;               // row counts of A and B (debug asserts)
    const float *Apad;                    // GA variant: A rows with their pads, [na][seglen]
    float *apad_ws;                       // search mode, nullable: room for Apad
    int64_t apad_cap;                     // floats available at apad_ws
    // Band-limited pass (ADAPT, search mode): the layout's window w is narrower than the
    // distance's; an item whose band-edge cells come within the threshold is appended to the
    // item array after the items it reads (level fbsel appends at fb_count[fbsel]) for the next
    // pass.  fbsel >= 1: run the items level fbsel - 1 appended -- or, if they
    // did not all fit below item_cap, every survivor again.
    Item *fb_items;
    unsigned long long *fb_count;
    int fbsel;
};

// An opaque copy: the compiler cannot rematerialise the value (it would otherwise recompute
// the per-slot kill scales with ISETP+FSEL inside the unrolled period).
__device__ __forceinline__ float pin_reg(float v) {
    float r;
    asm volatile("mov.b32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}

// KM (kill mode): 0 = general (kill slot anywhere: per-slot scale registers, edge masks);
// 1 = aligned, G*R = 2w+2 (kill slot is the top lane's last register: one scale register,
// edge masks); 2 = aligned and gpw*G = 32 (every lane used: rotating shuffles deliver the
// neighbouring group's kill slot, so no edge masks are needed at all).
// A 128-register cap (launch bounds asking for two CTAs of 8 warps) where it costs no spills
// (R <= 24, or R = 26 in the aligned layouts).  Shared memory still holds the SM to one CTA on
// config 2 (8 groups x 2 padded rows = 164 KB), but the capped allocation schedules better:
// 130 -> 126 registers, DTW 206.6 -> 198.2 ms (profiles/round1k_full.md).
template <int R, int KM>
constexpr int band_min_blocks() {
    return (R <= 24 || (R == 26 && KM >= 1)) ? 2 : 1;
}

template <int R, int KM, bool PACK, bool GA = false, bool ADAPT = false>
__global__ void __launch_bounds__(256, band_min_blocks<R, KM>()) k_dtw_band(BandParams p) {
    constexpr bool ALIGNED = KM >= 1;
    constexpr bool NOMASK = KM == 2;
    extern __shared__ __align__(16) float smem_f[];
    constexpr int H = R / 2;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int G = p.G, gpw = p.gpw, L = p.L, w = p.w;
    const int gw = lane / G;
    const int g = lane - gw * G;
    const bool valid_lane = gw < gpw;
    const int warps_per_block = blockDim.x >> 5;
    const int64_t gid = ((int64_t)blockIdx.x * warps_per_block + warp) * gpw + gw;
    const int64_t ngroups = (int64_t)gridDim.x * warps_per_block * gpw;
    const unsigned gbits = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gw * G));

    // GA: the A (query) rows are read from a padded global copy through L1 and only B is
    // staged -- half the shared memory per group, twice the resident warps
    float *sA = smem_f + (size_t)(warp * gpw + (valid_lane ? gw : 0)) * (GA ? 1 : 2) * p.seglen;
    float *sB = GA ? sA : sA + p.seglen;

    // index-dependent pads, written once (they never change)
    if (valid_lane) {
        for (int x = g; x < p.seglen; x += G) {
            int idx = x - p.padl;
            if (idx < 0 || idx >= L) {
                float v = idx < 0 ? 0x1p64f * (float)idx : 0x1p64f * (float)(idx - L + 1);
                if (!GA) sA[x] = v;
                sB[x] = v;
            }
        }
    }

    // slot bookkeeping
    const int g0 = w / R, r0 = w - (w / R) * R;     // slot of d = 0 (result)
    const int skill = 2 * w + 1;                     // kill slot d = w+1
    float sc[ALIGNED ? 1 : R];
    if (ALIGNED) {
        sc[0] = pin_reg((g * R + R - 1 == skill) ? kInf : 1.0f);
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) sc[r] = pin_reg((g * R + r == skill) ? kInf : 1.0f);
    }
    // general layout, packed: negated per-slot scales in pairs (2m, 2m+1) for the FFMA2 form
    unsigned long long scn[(!ALIGNED && PACK) ? R / 2 : 1];
    if (!ALIGNED && PACK) {
#pragma unroll
        for (int m = 0; m < R / 2; ++m) scn[m] = f2_pack(-sc[2 * m], -sc[2 * m + 1]);
    }
    const float nbmask_lo = (g == 0) ? kInf : 0.0f;        // selects +inf at group edges
    const float nbmask_hi = (g == G - 1) ? kInf : 0.0f;

    int64_t nitems = p.nitems_host;
    int64_t ioff = 0;  // fbsel: the appended items start after the survivors
    if (p.mode == 0) {
        unsigned long long c = *p.nitems_dev;
        nitems = (int64_t)(c < p.item_cap ? c : p.item_cap);
        if (p.fbsel) {  // level fbsel: the items level fbsel - 1 appended
            const unsigned long long f0 = p.fb_count[0];
            const unsigned long long off = c + (p.fbsel >= 2 ? f0 : 0ull);
            const unsigned long long n = p.fb_count[p.fbsel - 1];
            if (off + n <= p.item_cap) {
                ioff = (int64_t)off;
                nitems = (int64_t)n;
            } else if (ADAPT) {
                nitems = 0;  // not all were stored: the last, full-window pass reruns everything
            }  // else: every survivor again (exact, slower)
        }
    }
    int64_t it = gid;
    bool active = valid_lane && it < nitems;

    float D[R];
#pragma unroll
    for (int r = 0; r < R; ++r) D[r] = kInf;  // idle lanes too (their values feed shuffles)
    int per = 0;
    unsigned qcur = 0, ncur = 0;
    float thr_batch = kInf;
    long long my_items = 0, my_aband = 0, my_cells = 0;

    // Search mode: an item whose bound exceeds its query's live best-so-far (prune margin as
    // in S3) is skipped -- survivors arrive in LB-bucket order, so later ones often meet a
    // best-so-far already tightened by the earlier (lower-bound) candidates of their query.
    // The best-so-far load overlaps the row copies; a skipped item starts with an all-+inf
    // state, so the period's cut test retires it after one period (no extra control flow in
    // the hot loop).
    bool skipping = false;
    long long my_skipped = 0;
    float e0 = kInf, e1 = kInf;             // ADAPT: band-edge minima over the period
    unsigned long long kstart = 0;
#ifdef NNDTW_PROFILE_SETUP
    // instrumentation build only (tools/setup_share.sh): cycles spent waiting for item setups
    long long prof_setup = 0;
    const long long prof_t0 = clock64();
#endif
    auto setup = [&]() {
#ifdef NNDTW_PROFILE_SETUP
        const long long ps0 = clock64();
#endif
        unsigned a_idx, b_idx;
        float ilb = 0.0f;
        if (p.mode == 0) {
            Item itm = p.items[ioff + it];
            a_idx = itm.q;
            b_idx = itm.n;
            ilb = itm.lb;
        } else {
            a_idx = p.ia ? (unsigned)p.ia[it] : (unsigned)it;
            b_idx = p.ib ? (unsigned)p.ib[it] : (unsigned)it;
            thr_batch = p.cutoff ? p.cutoff[it] * (1.0f + p.eps_t) : kInf;
        }
        NNDTW_ASSERT(a_idx < (unsigned)p.dbg_na && b_idx < (unsigned)p.dbg_nb,
                     "band item oob: it=%lld a=%u b=%u na=%lld nb=%lld", (long long)it, a_idx,
                     b_idx, (long long)p.dbg_na, (long long)p.dbg_nb);
        qcur = a_idx;
        ncur = b_idx;
        const float *ga = p.A + (int64_t)a_idx * L;
        const float *gb = p.B + (int64_t)b_idx * L;
        // all copies in flight at once (cp.async), one wait: the rows arrive in about one
        // memory round trip instead of L/G dependent load->store steps
        if (p.vec4) {
#pragma unroll 4
            for (int x = 4 * g; x < L; x += 4 * G) {
                if (!GA) cp_async16(sA + p.padl + x, ga + x);
                cp_async16(sB + p.padl + x, gb + x);
            }
        } else {
            for (int x = g; x < L; x += G) {
                if (!GA) cp_async4(sA + p.padl + x, ga + x);
                cp_async4(sB + p.padl + x, gb + x);
            }
        }
        // warm L2 with the train row of this group's NEXT item (one bulk prefetch): its
        // setup then waits on an L2 hit instead of HBM (train rows are 205 MB on config 2)
        if (p.mode == 0 && g == 0 && p.vec4) {
            const int64_t nx = it + ngroups;
            if (nx < nitems) {
                const unsigned nb = p.items[ioff + nx].n;
                bulk_prefetch_l2(p.B + (int64_t)nb * L, (unsigned)L * 4u);
            }
        }
        if (p.mode == 0) kstart = ld_relaxed_u64(p.key + a_idx);
        cp_async_wait_all();
#ifdef NNDTW_PROFILE_SETUP
        prof_setup += clock64() - ps0;  // (no __syncwarp here: setup runs in divergent code)
#endif
        skipping = false;
        if (p.mode == 0) {
            // (all lanes of the group read the same address in one instruction)
            skipping = ilb > key_dist(kstart) * (1.0f + p.eps_p);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) D[r] = (!skipping && g == g0 && r == r0) ? 0.0f : kInf;
        per = 0;
    };

    if (active) setup();
    __syncwarp();

    // live best-so-far of the group's query, read one period ahead (the abandon test uses the
    // value loaded during the previous period: never tighter than the true live value)
    unsigned long long kprev = kstart;
    while (__any_sync(0xffffffffu, active)) {
        unsigned long long knext = 0;
        if (p.mode == 0 && active) knext = ld_relaxed_u64(p.key + qcur);

        // ---- one period: R anti-diagonals, fully unrolled ----------------------------
        const int kp = p.k0 + per * R;
        const int I0 = (kp + w - g * R) >> 1;   // kp + w is even by construction
        const int J0 = (kp - w + g * R) >> 1;
        const float *pa = (GA ? p.Apad + (size_t)qcur * p.seglen : sA) + p.padl + I0 - (H - 1);
        const float *pb = sB + p.padl + J0;
        NNDTW_ASSERT(p.padl + I0 - (H - 1) >= 0 && p.padl + I0 + H - 1 < p.seglen &&
                         p.padl + J0 >= 0 && p.padl + J0 + R - 1 < p.seglen,
                     "band smem oob: g=%d per=%d I0=%d J0=%d padl=%d seglen=%d", g, per, I0,
                     J0, p.padl, p.seglen);
        float aw[R - 1];
#pragma unroll
        for (int x = 0; x < R - 1; ++x) aw[x] = GA ? __ldg(pa + x) : pa[x];
        if (PACK) {
            // Half-packed cells: on an even diagonal t, cell m reads (a[t/2-m+H-1], b[t/2+m]);
            // on t+1 the same slot index m reads the same a and b one further.  One FADD2 with
            // a broadcast operand gives both differences: (a, a) - (b[y], b[y+1]).  The b pairs
            // come in two register copies -- pairs starting at even y (be) and at odd y (bo) --
            // loaded separately so that every pair is an aligned 64-bit register pair.  In the
            // general layout (kill slot anywhere) the pair is one FFMA2 instead:
            // (b[y], b[y+1]) - (a, a) * (sc[2m], sc[2m+1]) -- same square, kill scale folded in.
            unsigned long long be[H], bo[H > 1 ? H - 1 : 1];
#pragma unroll
            for (int k = 0; k < H; ++k) be[k] = f2_pack(pb[2 * k], pb[2 * k + 1]);
#pragma unroll
            for (int k = 0; k < H - 1; ++k)
                bo[k] = f2_pack(lds_distinct(pb + 2 * k + 1), lds_distinct(pb + 2 * k + 2));
#pragma unroll
            for (int t = 0; t < R; t += 2) {
                unsigned long long T[H];
#pragma unroll
                for (int m = 0; m < H; ++m) {
                    const float a = aw[(t >> 1) - m + H - 1];
                    const int y = (t >> 1) + m;
                    const unsigned long long bp = (y & 1) ? bo[y >> 1] : be[y >> 1];
                    if (ALIGNED) T[m] = f2_sub(f2_pack(a, a), bp);
                    else T[m] = f2_fma(f2_pack(a, a), scn[m], bp);
                }
                {  // diagonal t (even offsets r = 2m)
                    float nlo;
                    if (NOMASK) nlo = __shfl_sync(0xffffffffu, D[R - 1], (lane + 31) & 31);
                    else nlo = __shfl_up_sync(0xffffffffu, D[R - 1], 1) + nbmask_lo;
#pragma unroll
                    for (int m = 0; m < H; ++m) {
                        const int r = 2 * m;
                        float t0, t1;
                        f2_unpack(T[m], t0, t1);
                        const float lo = (r == 0) ? nlo : D[r - 1];
                        D[r] = fmaf(t0, t0, fminf(fminf(D[r], lo), D[r + 1]));
                    }
                    if (ADAPT) {  // band edges d = -w (lane 0, slot 0) and d = +w (top lane, R-2)
                        e0 = fminf(e0, D[0]);
                        e1 = fminf(e1, D[R - 2]);
                    }
                }
                {  // diagonal t+1 (odd offsets r = 2m+1); r = R-1 carries the kill scale
                    float nhi;
                    if (NOMASK) nhi = __shfl_sync(0xffffffffu, D[0], (lane + 1) & 31);
                    else nhi = __shfl_down_sync(0xffffffffu, D[0], 1) + nbmask_hi;
#pragma unroll
                    for (int m = 0; m < H; ++m) {
                        const int r = 2 * m + 1;
                        float t0, t1;
                        f2_unpack(T[m], t0, t1);
                        const float hi = (r == R - 1) ? nhi : D[r + 1];
                        const float v = fmaf(t1, t1, fminf(fminf(D[r], D[r - 1]), hi));
                        D[r] = (ALIGNED && r == R - 1) ? v * sc[0] : v;
                    }
                }
            }
        } else {
            float bw[R];
#pragma unroll
            for (int y = 0; y < R; ++y) bw[y] = pb[y];
#pragma unroll
            for (int t = 0; t < R; ++t) {
                const int phi = t & 1;
                float nlo = 0.0f, nhi = 0.0f;
                if (phi == 0) nlo = __shfl_up_sync(0xffffffffu, D[R - 1], 1) + nbmask_lo;
                else nhi = __shfl_down_sync(0xffffffffu, D[0], 1) + nbmask_hi;
#pragma unroll
                for (int m = 0; m < H; ++m) {
                    const int r = phi + 2 * m;
                    const float a = aw[(t >> 1) - m + H - 1];
                    const float b = bw[((t + 1) >> 1) + m];
                    float sr;
                    if (ALIGNED) sr = (r == R - 1) ? sc[0] : 1.0f;
                    else sr = sc[r];
                    const float tt = (ALIGNED && r != R - 1) ? (a - b) : fmaf(a, sr, -b);
                    const float lo = (r == 0) ? nlo : D[r - 1];
                    const float hi = (r == R - 1) ? nhi : D[r + 1];
                    D[r] = fmaf(tt, tt, fminf(fminf(D[r], lo), hi));
                }
                if (ADAPT && phi == 0) {  // band edges d = -w (lane 0, slot 0), +w (top, R-2)
                    e0 = fminf(e0, D[0]);
                    e1 = fminf(e1, D[R - 2]);
                }
            }
        }
        per = active ? per + 1 : 0;  // idle groups replay period 0 (stay in bounds)

        // ---- events: completion / early abandon --------------------------------------
        float lmin = D[0];
#pragma unroll
        for (int r = 1; r < R; ++r) lmin = fminf(lmin, D[r]);
        // (the freshest observed best-so-far: the key loaded at this period's start, when this
        // group's item was already running then -- keys only decrease)
        const unsigned long long kuse = (p.mode == 0 && active && knext != 0ull && knext < kprev)
                                            ? knext : kprev;
        float thr = p.mode == 0 ? key_dist(kuse) * (1.0f + p.eps_t) : thr_batch;
        kprev = knext;
        bool vote = !(lmin <= thr);
        unsigned ballot = __ballot_sync(0xffffffffu, vote);
        bool done = active && per == p.nper;
        bool abandon = active && !done && ((ballot & gbits) == gbits);
        bool fired = false;
        if (ADAPT) {
            // an edge cell within the threshold: a path leaving the band might be cheaper than
            // the band's value, so the item goes to the full-
            // window pass; otherwise every out-of-band cell exceeds the threshold and the
            // band's values, abandon and result are the full window's
            const bool near = (g == 0 && e0 <= thr) || (g == G - 1 && e1 <= thr);
            const unsigned fb = __ballot_sync(0xffffffffu, near);
            fired = active && !skipping && (fb & gbits) != 0u;
            done = done && !fired;
            abandon = abandon && !fired;
            e0 = kInf;
            e1 = kInf;
        }
#ifdef NNDTW_TRACE
        if (active && p.mode == 0 && blockIdx.x == 0 && warp == 0 && lane < 2)
            printf("TRACE lane=%d it=%lld q=%u n=%u per=%d/%d lmin=%g thr=%g D0=%g done=%d ab=%d\n",
                   lane, (long long)it, qcur, ncur, per, p.nper, lmin, thr, D[0], (int)done,
                   (int)abandon);
#endif
        if (__any_sync(0xffffffffu, done || abandon || fired)) {  // rare: once per item per group
            if (ADAPT && fired && g == 0) {
                const unsigned long long k = atomicAdd(p.fb_count + p.fbsel, 1ull);
                const unsigned long long pos = (unsigned long long)(ioff + nitems) + k;
                if (pos < p.item_cap) p.fb_items[pos] = Item{qcur, ncur, p.items[ioff + it].lb};
                if (p.counters != nullptr) {
                    atomicAdd(p.counters + CNT_FALLBACK, 1ull);
                    int klast = p.k0 + per * R - 1;
                    if (klast > 2 * L - 2) klast = 2 * L - 2;
                    my_cells += klast >= 0 ? p.cells_prefix[klast] : 0;
                }
            }
            if (done && g == g0) {  // (most items end abandoned: the result slot only here)
                float res = D[0];
#pragma unroll
                for (int r = 1; r < R; ++r)
                    if (r == r0) res = D[r];
                if (p.mode == 0) {
                    unsigned gidx = (unsigned)(p.index_base + ncur);
                    unsigned long long old = atomicMin(p.key + qcur, make_key(res, gidx));
                    float best = fminf(res, key_dist(old));
                    if (res <= best * (1.0f + p.eps_t)) {
                        unsigned long long slot = atomicAdd(p.log.count, 1ull);
                        if (slot < p.log.capacity) {
                            TieEntry e;
                            e.q = qcur;
                            e.n = ncur;
                            e.d32 = res;
                            e.pad = 0.0f;
                            e.d64 = 0.0;
                            p.log.e[slot] = e;
                        } else {
                            p.log.overflow[qcur] = 1u;
                        }
                    }
                } else {
                    p.out[it] = res;
                }
            }
            if (abandon && p.mode == 1 && g == 0) p.out[it] = kInf;
            if (done || abandon || fired) {
                if (!fired && g == 0 && p.counters != nullptr) {
                    if (skipping) {
                        my_skipped += 1;
                    } else {
                        int klast = p.k0 + per * R - 1;
                        if (klast > 2 * L - 2) klast = 2 * L - 2;
                        my_items += 1;
                        my_aband += abandon ? 1 : 0;
                        my_cells += klast >= 0 ? p.cells_prefix[klast] : 0;
                    }
                }
                it += ngroups;
                active = it < nitems;
                if (active) {
                    setup();
                    kprev = kstart;
                } else {
                    per = 0;  // idle groups replay period 0 (stay in bounds)
                }
            }
        }
        __syncwarp();
    }
#ifdef NNDTW_PROFILE_SETUP
    if (p.counters != nullptr) {  // per warp: setup cycles summed over its groups, warp cycles
        unsigned long long ws = (valid_lane && g == 0) ? (unsigned long long)prof_setup : 0ull;
        for (int off = 1; off < 32; off <<= 1) ws += __shfl_xor_sync(0xffffffffu, ws, off);
        if (lane == 0) {
            atomicAdd(p.counters + 6, ws);
            atomicAdd(p.counters + 7, (unsigned long long)(clock64() - prof_t0));
        }
    }
#endif
    if (p.counters != nullptr && valid_lane && g == 0 && my_skipped > 0)
        atomicAdd(p.counters + CNT_SKIPPED, (unsigned long long)my_skipped);
    if (p.counters != nullptr && valid_lane && g == 0 && (my_items > 0 || my_cells > 0)) {
        atomicAdd(p.counters + CNT_ITEMS, (unsigned long long)my_items);
        atomicAdd(p.counters + CNT_ABANDONED, (unsigned long long)my_aband);
        atomicAdd(p.counters + CNT_CELLS, (unsigned long long)my_cells);
    }
}

// ---- host-side selection and launch ----------------------------------------------------------
struct BandChoice {
    int R, G, gpw, warps;   // warps per CTA
    int km;                 // kill mode (see k_dtw_band)
    int ctas;               // resident CTAs per SM (model)
    bool pack;              // half-packed FADD2 cells (aligned layouts only)
    int k0, nper, padl, seglen;
};

// Geometry of the padded shared-memory rows for slot width R and G lanes per group.
static void band_geometry(int R, int G, int L, int w, BandChoice &c) {
    const int H = R / 2;
    c.k0 = (w & 1) ? -1 : 0;  // period starts satisfy (k + w) even
    c.nper = (2 * L - 1 - c.k0 + R - 1) / R;
    const int kp_last = c.k0 + (c.nper - 1) * R;
    const int amin = ((c.k0 + w - (G - 1) * R) >> 1) - (H - 1);
    const int amax = ((kp_last + w) >> 1) + H - 1 + 1;
    const int bmin = (c.k0 - w) >> 1;
    const int bmax = ((kp_last - w + (G - 1) * R) >> 1) + R - 1 + 1;
    const int lo = amin < bmin ? amin : bmin;
    const int hi = amax > bmax ? amax : bmax;
    c.padl = ((lo < 0 ? -lo : 0) + 1 + 3) / 4 * 4;  // 16-byte aligned row start
    const int padr = (hi > L - 1 ? hi - (L - 1) : 0) + 1;
    const int seg = c.padl + L + padr;
    // Lanes of a group read with stride R/2 words (distinct banks when R/2 is odd); the
    // groups of a warp sit 2*seglen words apart -- make that 32/gpw' (mod 32) so that the
    // groups' bank sets interleave instead of colliding (gpw' = gpw rounded up to 2^k).
    int gpw = 32 / G, gp2 = 1;
    while (gp2 < gpw) gp2 <<= 1;
    const int want = (32 / gp2) / 2;  // seglen mod 16 (2*seglen mod 32 = 32/gp2)
    int sl = seg;
    while ((sl & 15) != (want & 15)) ++sl;
    c.seglen = sl;
}

// Model: per period a lane issues 1.5R^2 cell ops,
// 2R-1 LDS, R shuffles (+R edge-mask adds unless KM=2) and ~20 bookkeeping instructions; the
// edge-cell chain (shuffle + min + fma, ~38 cycles) bounds a warp to >= 38R cycles per
// period.  Useful cells per SMSP-cycle = wps*gpw*R*(w+1/2)*slot_util / max(wps*issue, 38R),
// wps = resident warps per scheduler (shared memory / register limited).
static BandChoice choose_band_pass(int w, int L, bool all_widths);

static BandChoice choose_band(int w, int L) {
    BandChoice c = choose_band_pass(w, L, false);
    // R = 16 / 32 are excluded only while another width fits: at 2w+2 = 1024 (w = 511) the
    // aligned R = 32, G = 32 layout is the only band layout
    if (c.R == 0) c = choose_band_pass(w, L, true);
    return c;
}

static BandChoice choose_band_pass(int w, int L, bool all_widths) {
    BandChoice best{};
    best.R = 0;
    double bt = 0;
    static const char *force = getenv("NNDTW_BAND_R");  // experiments: force the slot width
    const int rforce = force ? atoi(force) : 0;
    for (int R = 2; R <= 32; R += 2) {
        if (rforce && R != rforce) continue;
        int G = (2 * w + 2 + R - 1) / R;
        if (G > 32) continue;
        bool aligned = (G * R == 2 * w + 2);
        // Measured pruning of the candidate list (profiles/round1l_band_layout_check_L300.txt,
        // band_sweep_r1i.txt): R = 16 and R = 32 are the slowest widths in every sweep; general
        // (unaligned) layouts wider than R = 24 pay for their per-slot scale registers and win
        // only where no R <= 24 layout fits two groups in a warp (2w+2 > 16*24): w = 192..234
        // at L = 300 go from one group per warp (2.2-3.9 Tcells/s) to two (4.3-4.5).
        static const int gmax = [] {  // experiments: widest general (unaligned) layout
            const char *e = getenv("NNDTW_BAND_GENERAL_MAX");
            return e ? atoi(e) : 30;
        }();
        if (!rforce && !all_widths && (R == 16 || R == 32)) continue;
        if (!aligned && R > gmax) continue;  // register budget of the general variant
        if (!aligned && R > 24 && !rforce && (2 * w + 2 + 23) / 24 <= 16) continue;
        BandChoice c{};
        c.R = R;
        c.G = G;
        c.gpw = 32 / G;
        c.km = aligned ? ((c.gpw * G == 32) ? 2 : 1) : 0;
        band_geometry(R, G, L, w, c);
        const double warp_smem = (double)c.gpw * 2 * c.seglen * sizeof(float);
        static const char *wcap_env = getenv("NNDTW_BAND_WARPS");  // experiments
        int wcap = wcap_env ? atoi(wcap_env) : 8;
        if (wcap > 8) wcap = 8;  // __launch_bounds__(256, ...)
        int warps = (int)((226.0 * 1024) / warp_smem);
        if (warps < 1) continue;
        if (warps > wcap) warps = wcap;
        c.warps = warps;
        const int ctas_smem = (int)((227.0 * 1024) / (warps * warp_smem));
        const int regs = c.km >= 1 ? 48 + 2 * R : 48 + 3 * R;
        const int ctas_regs = 65536 / (regs * 32 * warps);
        int ctas = ctas_smem < ctas_regs ? ctas_smem : ctas_regs;
        if (ctas < 1) continue;
        c.ctas = ctas;
        int wsm = ctas * warps;
        if (wsm > 48) wsm = 48;
        const double wps = wsm / 4.0;
        const double issue = 1.5 * R * R + (2.0 * R - 1) + R + (c.km == 2 ? 0 : R) + 20.0 +
                             (((R / 2) & 1) ? 0.0 : 0.15 * R * R);  // even R/2: bank conflicts
        const double chain = 38.0 * R;
        const double util = (double)(2 * w + 1) / (double)(G * R);
        const double thr = wps * c.gpw * R * (w + 0.5) * util /
                           (wps * issue > chain ? wps * issue : chain);
        if (thr > bt) {
            bt = thr;
            best = c;
        }
    }
    return best;
}

bool band_supported(int w, int L) { return choose_band(w, L).R != 0; }

// A rows with the kernel's index-dependent pads (GA variant): out[r][x] = A[r][x - padl] inside,
// the +-2^64 pad values outside
__global__ void k_pad_rows(const float *__restrict__ A, int64_t na, int L, int padl, int seglen,
                           float *__restrict__ out) {
    const int64_t n = na * (int64_t)seglen;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / seglen;
        const int x = (int)(e - r * seglen), idx = x - padl;
        out[e] = (idx < 0) ? 0x1p64f * (float)idx
                           : (idx >= L ? 0x1p64f * (float)(idx - L + 1) : A[r * L + idx]);
    }
}

template <int R, int KM, bool PACK, bool GA = false, bool ADAPT = false>
static int launch_band_t(BandParams &p, const BandChoice &c, cudaStream_t st, int num_sms) {
    auto kern = k_dtw_band<R, KM, PACK, GA, ADAPT>;
    const int block = 32 * c.warps;
    size_t smem = (size_t)c.warps * p.gpw * (GA ? 1 : 2) * p.seglen * sizeof(float);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem);
    if (occ < 1) occ = 1;
    int64_t groups_per_block = (int64_t)c.warps * p.gpw;
    int64_t want = (int64_t)num_sms * occ;
    if (p.mode == 1) {
        int64_t need = (p.nitems_host + groups_per_block - 1) / groups_per_block;
        if (need < want) want = need > 0 ? need : 1;
    }
    kern<<<(unsigned)want, block, smem, st>>>(p);
    count_launch(1, __func__);
    return 0;
}

#define BAND_CASE(RR)                                                                   \
    case RR:                                                                            \
        return c.km == 2   ? (c.pack ? launch_band_t<RR, 2, true>(p, c, st, num_sms)    \
                                     : launch_band_t<RR, 2, false>(p, c, st, num_sms))  \
               : c.km == 1 ? (c.pack ? launch_band_t<RR, 1, true>(p, c, st, num_sms)    \
                                     : launch_band_t<RR, 1, false>(p, c, st, num_sms))  \
                           : (c.pack ? launch_band_t<RR, 0, true>(p, c, st, num_sms)    \
                                     : launch_band_t<RR, 0, false>(p, c, st, num_sms));

int launch_dtw_band(BandParams p, cudaStream_t st, int num_sms) {
    BandChoice c = choose_band(p.w, p.L);
    if (c.R == 0) return -1;
    {
        // Half-packed cells (FADD2, or FFMA2 with the kill scale in the general layout): a
        // measured choice (tools/pack_sweep.sh, tools/band_sweep.sh; profiles/pack_sweep_b200.txt,
        // profiles/band_sweep_r1i.txt): in the aligned layouts faster at R = 20, 22, 26 (config
        // 2's R=26: 6.6 -> 7.3 Tcells/s), slower at R = 16; in the general layout (per-slot
        // kill scales, FFMA2 form) 3-15 % slower at every R with two CTAs per SM.
        static const char *pk = getenv("NNDTW_PACK");
        const bool rule = c.km >= 1 && (c.R == 20 || c.R == 22 || c.R == 26);
        c.pack = pk ? pk[0] == '1' : rule;
    }
    static const bool verbose = getenv("NNDTW_VERBOSE") != nullptr;
    if (verbose)
        fprintf(stderr,
                "nndtw band: L=%d w=%d -> R=%d G=%d gpw=%d km=%d pack=%d warps/cta=%d seglen=%d\n",
                p.L, p.w, c.R, c.G, c.gpw, c.km, (int)c.pack, c.warps, c.seglen);
    p.G = c.G;
    p.gpw = c.gpw;
    p.k0 = c.k0;
    p.nper = c.nper;
    p.padl = c.padl;
    p.seglen = c.seglen;
    p.vec4 = (p.L % 4 == 0 && c.seglen % 4 == 0 && c.padl % 4 == 0 &&
              ((uintptr_t)p.A % 16) == 0 && ((uintptr_t)p.B % 16) == 0) ? 1 : 0;
    {
        // Global A rows (GA) for the config-2 layout (R = 26, full warp, half-packed): there two
        // padded rows per group hold the SM to 8 warps; with the query rows read through L1
        // from a padded copy (k_pad_rows, once per launch) only B is staged and 16 warps fit
        // -- the survivor round 198 -> 190 ms.  Other layouts keep both rows in shared memory:
        // forced on for every layout, config 3's LOOCV went 424 -> 434 ms and config 1's
        // survivor rounds 9.10 -> 9.34 ms (their bands leave room for two CTAs, or the L1
        // reads cost more than the residency gains).  NNDTW_BAND_GA=0 disables it.
        static const char *ga = getenv("NNDTW_BAND_GA");
        const bool ga_on = !(ga && ga[0] == '0');
        if (ga_on && p.mode == 0 && p.apad_ws != nullptr && c.R == 26 && c.km == 2 && c.pack &&
            p.vec4 && p.dbg_na > 0 && p.dbg_na * (int64_t)c.seglen <= p.apad_cap) {
            const int64_t n = p.dbg_na * (int64_t)c.seglen;
            const int64_t blocks = (n + 255) / 256 < 4 * num_sms ? (n + 255) / 256 : 4 * num_sms;
            k_pad_rows<<<(unsigned)blocks, 256, 0, st>>>(p.A, p.dbg_na, p.L, p.padl, p.seglen,
                                                         p.apad_ws);
            count_launch(1, "k_pad_rows");
            p.Apad = p.apad_ws;
            return launch_band_t<26, 2, true, true>(p, c, st, num_sms);
        }
    }
    switch (c.R) {
        BAND_CASE(2)
        BAND_CASE(4)
        BAND_CASE(6)
        BAND_CASE(8)
        BAND_CASE(10)
        BAND_CASE(12)
        BAND_CASE(14)
        BAND_CASE(16)
        BAND_CASE(18)
        BAND_CASE(20)
        BAND_CASE(22)
        BAND_CASE(24)
        BAND_CASE(26)
        BAND_CASE(28)
        BAND_CASE(30)
        BAND_CASE(32)
        default:
            return -1;
    }
}

// ---- band-limited pass ------------------------------------
// The window wb of the band-limited pass for a distance window w, or -1: the R = 26 full-warp
// aligned layout (the GA variant, 2wb + 2 = 26 G with G * gpw = 32) with the largest
// wb <= w / 2.  Measured on config 2 (queries/s): R = 26, wb = 51 (G = 4): 57.6 k (13 % of the
// survivors fall back); R = 20, wb = 79 and R = 22, wb = 87 (G = 8, four groups per warp,
// hardly any fall back): 49.7 k / 50.1 k; R = 26, wb = 25: 41.1 k; unpacked R = 14, wb = 55:
// 53.2 k; R = 12, wb = 47: 48.9 k; no pass: 47.9 k.  NNDTW_ADAPT_R (20 / 22 / 26) and
// NNDTW_ADAPT_FRAC (wb <= frac * w) select others for experiments.
static int band_adapt_r() {  // experiments: NNDTW_ADAPT_R = 20 / 22 / 26 (default)
    const char *e = getenv("NNDTW_ADAPT_R");
    const int r = e ? atoi(e) : 26;
    return (r == 20 || r == 22) ? r : 26;
}

int band_adapt_window(int L, int w, bool full_window) {
    const char *ee = getenv("NNDTW_ADAPT");  // 0 = off; an integer > 1 forces that wb
    const int env = ee ? atoi(ee) : -1;
    if (w > L - 1) w = L - 1;
    if (env == 0 || L % 4 != 0) return -1;
    const int R = band_adapt_r();
    // experiments: wb <= w * frac (default 0.5; 1/8 in front of the row-strip kernel: config 4
    // at wb = 207 / 415 / 103: 14.0 k / 12.6 k / 11.3 k queries/s, 11.7 k without the pass)
    const char *ef = getenv("NNDTW_ADAPT_FRAC");
    const double frac = ef ? atof(ef) : (full_window ? 0.125 : 0.5);
    int best = -1;
    for (int G = 1; G <= 32; G <<= 1) {
        const int wb = (R / 2) * G - 1;
        if (env > 1 ? wb == env : wb <= frac * w) best = wb > best ? wb : best;
    }
    if (best < 0 || best >= w) return -1;
    const char *em = getenv("NNDTW_ADAPT_MINW");  // experiments: the smallest w (default 64)
    if (env < 0 && w < (em ? atoi(em) : 64)) return -1;  // default: wide windows only
    return best;
}

// Launch the band-limited pass: p.w = wb (band_adapt_window), search mode, p.fb_items /
// p.fb_count set.  -1 if the layout cannot run (the caller then runs the full window only).
int launch_dtw_band_adapt(BandParams p, cudaStream_t st, int num_sms) {
    if (p.mode != 0 || p.apad_ws == nullptr || p.fb_count == nullptr || p.fb_items == nullptr)
        return -1;
    const int R = band_adapt_r();
    const int G = (2 * p.w + 2) / R;
    if (G * R != 2 * p.w + 2 || G < 1 || G > 32 || (32 % G) != 0) return -1;
    BandChoice c{};
    c.R = R;
    c.G = G;
    c.gpw = 32 / G;
    c.km = 2;
    c.pack = true;
    band_geometry(R, G, p.L, p.w, c);
    // GA rows must be 16-byte aligned (cp.async16, the padded query copy); one staged row per
    // group, so consecutive groups sit seglen words apart: seglen = 4 (mod 32) staggers up to 8
    // groups of a warp over distinct bank quads
    while (c.seglen % 32 != 4) ++c.seglen;
    // CTA size: the most resident warps (one staged row per group; at most 16 warps per SM
    // at the 128-register cap)
    const double warp_smem = (double)c.gpw * c.seglen * sizeof(float);
    int bestw = 0, best_res = 0;
    for (int wv = 1; wv <= 8; ++wv) {
        int ctas = (int)((227.0 * 1024) / (wv * warp_smem));
        if (ctas > 16 / wv) ctas = 16 / wv;
        if (ctas * wv >= best_res && ctas > 0) {
            best_res = ctas * wv;
            bestw = wv;
        }
    }
    if (bestw < 1) return -1;
    c.warps = bestw;
    p.G = c.G;
    p.gpw = c.gpw;
    p.k0 = c.k0;
    p.nper = c.nper;
    p.padl = c.padl;
    p.seglen = c.seglen;
    p.vec4 = (p.L % 4 == 0 && c.seglen % 4 == 0 && c.padl % 4 == 0 &&
              ((uintptr_t)p.A % 16) == 0 && ((uintptr_t)p.B % 16) == 0) ? 1 : 0;
    if (!p.vec4 || p.dbg_na <= 0 || p.dbg_na * (int64_t)c.seglen > p.apad_cap) return -1;
    const int64_t n = p.dbg_na * (int64_t)c.seglen;
    const int64_t blocks = (n + 255) / 256 < 4 * num_sms ? (n + 255) / 256 : 4 * num_sms;
    k_pad_rows<<<(unsigned)blocks, 256, 0, st>>>(p.A, p.dbg_na, p.L, p.padl, p.seglen, p.apad_ws);
    count_launch(1, "k_pad_rows");
    p.Apad = p.apad_ws;
    if (R == 20) return launch_band_t<20, 2, true, true, true>(p, c, st, num_sms);
    if (R == 22) return launch_band_t<22, 2, true, true, true>(p, c, st, num_sms);
    return launch_band_t<26, 2, true, true, true>(p, c, st, num_sms);
}

// ---- w = 0: DTW_0 is the squared Euclidean distance; one warp per item -------------
__global__ void __launch_bounds__(256) k_dtw_w0(BandParams p) {
    const int lane = threadIdx.x & 31;
    // warp id through a shuffle and the skip test through a vote: provably warp-uniform loop
    // control, so the reduction's shuffles need no divergence handling
    const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) +
                        __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int64_t nitems = p.nitems_host;
    if (p.mode == 0) {
        unsigned long long c = *p.nitems_dev;
        nitems = (int64_t)(c < p.item_cap ? c : p.item_cap);
    }
    for (int64_t it = wid; it < nitems; it += nw) {
        unsigned a_idx, b_idx;
        if (p.mode == 0) {
            Item itm = p.items[it];
            a_idx = itm.q;
            b_idx = itm.n;
            float live = key_dist(ld_relaxed_u64(p.key + a_idx));
            live = __shfl_sync(0xffffffffu, live, 0);
            if (__any_sync(0xffffffffu, itm.lb > live * (1.0f + p.eps_p))) {  // pruned by the live best
                if (lane == 0 && p.counters) atomicAdd(p.counters + CNT_SKIPPED, 1ull);
                continue;
            }
        } else {
            a_idx = p.ia ? (unsigned)p.ia[it] : (unsigned)it;
            b_idx = p.ib ? (unsigned)p.ib[it] : (unsigned)it;
        }
        const float *ga = p.A + (int64_t)a_idx * p.L;
        const float *gb = p.B + (int64_t)b_idx * p.L;
        float s = 0.0f;
        for (int i = lane; i < p.L; i += 32) {
            float t = __ldg(ga + i) - __ldg(gb + i);
            s = fmaf(t, t, s);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) {
            if (p.mode == 0) {
                unsigned long long old =
                    atomicMin(p.key + a_idx, make_key(s, (unsigned)(p.index_base + b_idx)));
                float best = fminf(s, key_dist(old));
                if (s <= best * (1.0f + p.eps_t)) {
                    unsigned long long slot = atomicAdd(p.log.count, 1ull);
                    if (slot < p.log.capacity) {
                        TieEntry e;
                        e.q = a_idx;
                        e.n = b_idx;
                        e.d32 = s;
                        e.pad = 0.0f;
                        e.d64 = 0.0;
                        p.log.e[slot] = e;
                    } else {
                        p.log.overflow[a_idx] = 1u;
                    }
                }
                if (p.counters) {
                    atomicAdd(p.counters + CNT_ITEMS, 1ull);
                    atomicAdd(p.counters + CNT_CELLS, (unsigned long long)p.L);
                }
            } else {
                p.out[it] = s;
            }
        }
    }
}

static int launch_dtw_w0(BandParams &p, cudaStream_t st, int num_sms) {
    int64_t grid = (int64_t)num_sms * 8;
    if (p.mode == 1) {
        int64_t need = (p.nitems_host + 7) / 8;
        if (need < grid) grid = need > 0 ? need : 1;
    }
    k_dtw_w0<<<(unsigned)grid, 256, 0, st>>>(p);
    count_launch(1, __func__);
    return 0;
}

// Which S4 kernel runs for (L, w): 0 = k_dtw_w0, 1 = k_dtw_band, 2 = k_dtw_strip.
int dtw_kernel_kind(int L, int w) {
    if (w > L - 1) w = L - 1;
    if (w == 0) return 0;
    // Full window (w = L-1): the band sweeps (w+1)(2L-1) slot-cells for L^2 cells (50% useful)
    // while the row-strip kernel computes L^2 unmasked cells, so it wins when its strips are
    // nearly full (measured: L=256, w=255: 1.9 -> 4.4 Tcells/s; L=300: 3.6 -> 4.4; L=384: 2.8 -> 5.1;
    // L=128 (one half-empty strip): 2.6 -> 1.9, so the band stays there).
    static const char *fs = getenv("NNDTW_FORCE_STRIP");  // experiments: 1 = strip, 0 = band
    bool strip = false;
    if (w >= L - 1) {
        const int H = 32 * strip_rows_per_lane(L);
        strip = (long long)((L + H - 1) / H) * H * 100 <= (long long)L * 112;  // <= 12% idle rows
    }
    if (fs) strip = fs[0] == '1';
    return (band_supported(w, L) && !strip) ? 1 : 2;
}

int dispatch_dtw(const float *A, const float *B, int64_t na, int64_t nb, const Item *items,
                 const unsigned long long *nitems_dev, unsigned long long item_cap,
                 const int32_t *ia, const int32_t *ib, int64_t nitems_host, int L, int w,
                 int mode, unsigned long long *key, int64_t index_base, float eps_t, TieLog log,
                 unsigned long long *counters, const long long *cells_prefix,
                 const float *cutoff, float *out, cudaStream_t st, int num_sms,
                 float *apad_ws, int64_t apad_cap, int adapt_w, Item *fb_items,
                 unsigned long long *fb_count, int fbsel) {
    if (w > L - 1) w = L - 1;
    BandParams p;
    p.fb_items = fb_items;
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
    {
        static const char *ns = getenv("NNDTW_NO_SKIP");  // experiments: no live-bsf skip
        if (ns && ns[0] == '1') p.eps_p = kInf;
    }
    p.log = log;
    p.counters = counters;
    p.cells_prefix = cells_prefix;
    p.cutoff = cutoff;
    p.out = out;
    p.dbg_na = na;
    p.dbg_nb = nb;
    p.Apad = nullptr;
    p.apad_ws = apad_ws;
    p.apad_cap = apad_cap;
    if (adapt_w >= 0) {  // the band-limited pass (its caller checked band_adapt_window)
        p.w = adapt_w;
        return launch_dtw_band_adapt(p, st, num_sms);
    }
    const int kind = dtw_kernel_kind(L, w);
    if (kind == 0) return launch_dtw_w0(p, st, num_sms);
    if (kind == 1) {
        int rc = launch_dtw_band(p, st, num_sms);
        if (rc == 0) return 0;
    }
    return launch_dtw_strip(A, B, items, nitems_dev, item_cap, ia, ib, nitems_host, L, w, mode,
                            key, index_base, eps_t, log, counters, cells_prefix, cutoff, out, st,
                            num_sms, fbsel ? fb_count : nullptr, fbsel);
}

}  // namespace nndtw
