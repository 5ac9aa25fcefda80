// bounds_improved.cu -- SURVEY §8(f) NEXT-4: LB_Improved with the O(L) projection envelope, the
// LB_Improved bridge inside LB_Enhanced, and the bound "finish" pass that turns any all-pairs
// bound matrix into classify's S2 output (Kim cascade, leave-one-out self pair, argmin seed).
//
// LB_Improved_W(A,B) = LB_Keogh(A, env B) + LB_Keogh(B, env A'),  A'_i = clamp(A_i, L^B_i, U^B_i)
// (§2.3.3).  The paper times it with "the optimised algorithm to compute the
// projection envelopes", i.e. an O(L) sliding max/min of A' per pair.  Here one warp
// owns a pair and computes env A' with the van Herk / Gil-Werman scheme: the padded row
// (-inf / +inf outside [0, L), reading C5's clipping) is cut into blocks of K = 2w+1 aligned at
// index -w; g = prefix max (min) inside each block, h = suffix max (min); then
//   U'_j = max(h[j-w], g[j+w])                       (one block boundary inside the window)
// with h[j-w] = h[0] for j-w < 0 (the pads of block 0 are -inf) and g[j+w] = g[L-1] when j+w
// lies past the end in L-1's block, -inf when it lies in a later block (h[j-w] then already
// covers [j-w, L-1]).  The projection of the whole row is computed first (all of its loads in
// flight at once, float4 where aligned) into shared memory; the prefix / suffix scans are
// warp-segmented scans (resets at block starts / ends) over chunks of 32*CE elements with a
// carry across chunks: O(1) work per element, independent of w.
//
// The kernel computes only the SECOND pass, sum over columns j in [c_lo, c_hi) of
// keogh(B_j, L'_j, U'_j), and ADDS it to lb[q][n]; the first pass is the LB tile kernel
// (lb.cu):
//   * LB_Improved           = tile kernel in LB_Keogh mode            + pass over [0, L)
//   * LB_Enhanced^V with the LB_Improved bridge (reading C21)
//                           = tile kernel (bands + LB_Keogh bridge)   + pass over the bridge
//                             columns [nb, L - nb).
// Both stay admissible: for a path cell (i, j) with |i-j| <= w, B_j is inside [L^B_i, U^B_i],
// so (A_i - B_j)^2 >= (A_i - A'_i)^2 + (A'_i - B_j)^2 (the cross term is >= 0); the first
// parts are counted once per (bridge) row -- the Keogh terms --, the second once per column of
// the range, and no cell of a bridge column lies in one of Algorithm 1's bands (DESIGN.md
// reading C21).
#include "launchers.cuh"

namespace nndtw {

constexpr int IMP_CE = 8;                 // elements per lane per chunk
constexpr int IMP_CH = 32 * IMP_CE;       // elements per chunk

struct MaxMin {
    float mx, mn;
};

// warp segmented inclusive scan in the direction of increasing lane (UP) or decreasing lane:
// (f, v): f = the lane's elements contain a reset; combine(a, b) = b.f ? b : (a.f | b.f, a v b)
template <bool UP>
__device__ __forceinline__ void seg_scan(int &f, MaxMin &v, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int of = UP ? __shfl_up_sync(0xffffffffu, f, off) : __shfl_down_sync(0xffffffffu, f, off);
        const float ox = UP ? __shfl_up_sync(0xffffffffu, v.mx, off) : __shfl_down_sync(0xffffffffu, v.mx, off);
        const float on = UP ? __shfl_up_sync(0xffffffffu, v.mn, off) : __shfl_down_sync(0xffffffffu, v.mn, off);
        // branch-free (selects): no divergent control flow between the shuffles, so the
        // compiler emits plain SHFLs instead of WARPSYNC/ENDCOLLECTIVE sequences
        const bool take = (UP ? lane >= off : lane + off < 32) && !f;
        v.mx = take ? fmaxf(v.mx, ox) : v.mx;
        v.mn = take ? fminf(v.mn, on) : v.mn;
        f = take ? of : f;
    }
}

// 8 consecutive floats of a row (vectorised when the row is 16-byte aligned)
template <bool VEC>
__device__ __forceinline__ void load8(const float *p, int j0, int L, float (&x)[IMP_CE]) {
    if (VEC && j0 + IMP_CE <= L) {
        const float4 lo = __ldg(reinterpret_cast<const float4 *>(p + j0));
        const float4 hi = __ldg(reinterpret_cast<const float4 *>(p + j0 + 4));
        x[0] = lo.x; x[1] = lo.y; x[2] = lo.z; x[3] = lo.w;
        x[4] = hi.x; x[5] = hi.y; x[6] = hi.z; x[7] = hi.w;
    } else {
#pragma unroll
        for (int e = 0; e < IMP_CE; ++e) x[e] = j0 + e < L ? __ldg(p + j0 + e) : 0.0f;
    }
}

// 8 consecutive shared-memory floats of a lane as two 16-byte accesses: a warp's 32 lanes then
// touch 1 KB contiguously (4 wavefronts) instead of 8-way bank conflicts at stride 8 words
__device__ __forceinline__ void lds8(const float *p, float (&x)[IMP_CE]) {
    const float4 lo = *reinterpret_cast<const float4 *>(p);
    const float4 hi = *reinterpret_cast<const float4 *>(p + 4);
    x[0] = lo.x; x[1] = lo.y; x[2] = lo.z; x[3] = lo.w;
    x[4] = hi.x; x[5] = hi.y; x[6] = hi.z; x[7] = hi.w;
}
__device__ __forceinline__ void sts8(float *p, const float (&x)[IMP_CE]) {
    *reinterpret_cast<float4 *>(p) = make_float4(x[0], x[1], x[2], x[3]);
    *reinterpret_cast<float4 *>(p + 4) = make_float4(x[4], x[5], x[6], x[7]);
}

template <bool VEC>
__global__ void __launch_bounds__(256) k_lb_improved_pass(const float *__restrict__ q, int64_t nq,
                                                          const float *__restrict__ t,
                                                          const float *__restrict__ U,
                                                          const float *__restrict__ Lo,
                                                          int64_t nt, int L, int w, int c_lo,
                                                          int c_hi, float *lb, int64_t ldlb,
                                                          int rows_per_warp) {
    extern __shared__ __align__(16) float imp_smem[];
    // warp index through a shuffle: provably warp-uniform, so the pair loop's bounds are too and
    // the shuffles below need no divergence handling (WARPSYNC / collective sequences)
    const int lane = threadIdx.x & 31, warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);
    const int nwarps = blockDim.x >> 5;
    const int Lp = (L + IMP_CH - 1) / IMP_CH * IMP_CH;  // rows padded to whole chunks
    float *ap = imp_smem + (size_t)warp * 6 * Lp;      // A' [Lp]
    float *gx = ap + Lp, *gn = gx + Lp, *hx = gn + Lp, *hn = hx + Lp, *bs = hn + Lp;
    const int K = 2 * w + 1;
    const int nch = Lp / IMP_CH;
    const int64_t npairs = nq * nt;
    // last index of the block holding L-1: g[j+w] for j+w in L-1..blast_end is g[L-1]
    const int blast_end = ((L - 1 + w) / K + 1) * K - w - 1;
    const int64_t pr0 = ((int64_t)blockIdx.x * nwarps + warp) * rows_per_warp;
    const int64_t pe = pr0 + rows_per_warp < npairs ? pr0 + rows_per_warp : npairs;
    // the next pair's first chunk is loaded while this pair is scanned (software pipeline: the
    // per-pair chain of load -> scans -> gather is latency-bound otherwise)
    float na[IMP_CE], nl[IMP_CE], nu[IMP_CE], nb[IMP_CE];
    auto load_chunk0 = [&](int64_t pr) {
        // train-major pair order: a warp's consecutive pairs share the train series (its
        // envelope and row stay in L1/L2 across queries; the queries are the small set)
        const int64_t ni = pr / nq, qi = pr - ni * nq;
        const int j0 = lane * IMP_CE;
        load8<VEC>(q + qi * L, j0, L, na);
        load8<VEC>(Lo + ni * L, j0, L, nl);
        load8<VEC>(U + ni * L, j0, L, nu);
        load8<VEC>(t + ni * L, j0, L, nb);
    };
    if (pr0 < pe) load_chunk0(pr0);
    for (int64_t pr = pr0; pr < pe; ++pr) {
        // train-major pair order: a warp's consecutive pairs share the train series (its
        // envelope and row stay in L1/L2 across queries; the queries are the small set)
        const int64_t ni = pr / nq, qi = pr - ni * nq;
        const float *a = q + qi * L, *b = t + ni * L, *u = U + ni * L, *lo = Lo + ni * L;
        // ---- projection A' (and the row of B) into shared memory ---------------------------
        {
            const int j0 = lane * IMP_CE;
            float xp[IMP_CE];
#pragma unroll
            for (int e = 0; e < IMP_CE; ++e) xp[e] = fminf(fmaxf(na[e], nl[e]), nu[e]);
            sts8(ap + j0, xp);
            sts8(bs + j0, nb);
        }
#pragma unroll 2
        for (int c = 1; c < nch; ++c) {
            const int j0 = c * IMP_CH + lane * IMP_CE;
            float xa[IMP_CE], xl[IMP_CE], xu[IMP_CE], xb[IMP_CE];
            load8<VEC>(a, j0, L, xa);
            load8<VEC>(lo, j0, L, xl);
            load8<VEC>(u, j0, L, xu);
            load8<VEC>(b, j0, L, xb);
            float xp[IMP_CE];
#pragma unroll
            for (int e = 0; e < IMP_CE; ++e) xp[e] = fminf(fmaxf(xa[e], xl[e]), xu[e]);
            sts8(ap + j0, xp);
            sts8(bs + j0, xb);
        }
        if (pr + 1 < pe) load_chunk0(pr + 1);
        __syncwarp();
        // ---- forward (prefix) segmented scan: resets at block starts (j + w) % K == 0 ------
        MaxMin carry{-kInf, kInf};
        for (int c = 0; c < nch; ++c) {
            const int j0 = c * IMP_CH + lane * IMP_CE;
            float x[IMP_CE];
            bool rs[IMP_CE];
            lds8(ap + j0, x);
            int pos = (j0 + w) % K;
#pragma unroll
            for (int e = 0; e < IMP_CE; ++e) {
                rs[e] = pos == 0 && j0 + e < L;
                pos = pos + 1 == K ? 0 : pos + 1;
            }
            MaxMin run{-kInf, kInf};
            int f = 0;
#pragma unroll
            for (int e = 0; e < IMP_CE; ++e) {
                run.mx = fmaxf(rs[e] ? -kInf : run.mx, x[e]);
                run.mn = fminf(rs[e] ? kInf : run.mn, x[e]);
                f |= rs[e] ? 1 : 0;
            }
            MaxMin inc = run;
            int fi = f;
            seg_scan<true>(fi, inc, lane);
            // carry into this lane = inclusive result of lane-1 (combined with the chunk carry)
            MaxMin cin;
            cin.mx = __shfl_up_sync(0xffffffffu, inc.mx, 1);
            cin.mn = __shfl_up_sync(0xffffffffu, inc.mn, 1);
            const int fprev = __shfl_up_sync(0xffffffffu, fi, 1);
            {
                const bool first = lane == 0, addc = lane == 0 || !fprev;
                cin.mx = first ? carry.mx : (addc ? fmaxf(cin.mx, carry.mx) : cin.mx);
                cin.mn = first ? carry.mn : (addc ? fminf(cin.mn, carry.mn) : cin.mn);
            }
            MaxMin r = cin;  // the carry applies until the lane's first reset
            float vx[IMP_CE], vn[IMP_CE];
#pragma unroll
            for (int e = 0; e < IMP_CE; ++e) {
                r.mx = fmaxf(rs[e] ? -kInf : r.mx, x[e]);
                r.mn = fminf(rs[e] ? kInf : r.mn, x[e]);
                vx[e] = r.mx;
                vn[e] = r.mn;
            }
            sts8(gx + j0, vx);
            sts8(gn + j0, vn);
            carry.mx = __shfl_sync(0xffffffffu, r.mx, 31);
            carry.mn = __shfl_sync(0xffffffffu, r.mn, 31);
        }
        // ---- backward (suffix) segmented scan: resets at block ends (j + w + 1) % K == 0 ---
        // (elements past L-1 are the +-inf pads: identities, never resets)
        carry = MaxMin{-kInf, kInf};
        for (int c = nch - 1; c >= 0; --c) {
            const int j0 = c * IMP_CH + lane * IMP_CE;
            float x[IMP_CE];
            bool re[IMP_CE];
            lds8(ap + j0, x);
            int pos = (j0 + w) % K;
#pragma unroll
            for (int e = 0; e < IMP_CE; ++e) {
                re[e] = pos == K - 1 && j0 + e < L;
                pos = pos + 1 == K ? 0 : pos + 1;
            }
            MaxMin run{-kInf, kInf};
            int f = 0;
#pragma unroll
            for (int e = IMP_CE - 1; e >= 0; --e) {
                // past L-1: the pads (identities), never resets
                const float xv = j0 + e < L ? x[e] : -kInf, xn = j0 + e < L ? x[e] : kInf;
                run.mx = fmaxf(re[e] ? -kInf : run.mx, xv);
                run.mn = fminf(re[e] ? kInf : run.mn, xn);
                f |= re[e] ? 1 : 0;
            }
            MaxMin inc = run;
            int fi = f;
            seg_scan<false>(fi, inc, lane);
            MaxMin cin;
            cin.mx = __shfl_down_sync(0xffffffffu, inc.mx, 1);
            cin.mn = __shfl_down_sync(0xffffffffu, inc.mn, 1);
            const int fnext = __shfl_down_sync(0xffffffffu, fi, 1);
            {
                const bool first = lane == 31, addc = lane == 31 || !fnext;
                cin.mx = first ? carry.mx : (addc ? fmaxf(cin.mx, carry.mx) : cin.mx);
                cin.mn = first ? carry.mn : (addc ? fminf(cin.mn, carry.mn) : cin.mn);
            }
            MaxMin r = cin;
            float vx[IMP_CE], vn[IMP_CE];
#pragma unroll
            for (int e = IMP_CE - 1; e >= 0; --e) {
                const float xv = j0 + e < L ? x[e] : -kInf, xn = j0 + e < L ? x[e] : kInf;
                r.mx = fmaxf(re[e] ? -kInf : r.mx, xv);
                r.mn = fminf(re[e] ? kInf : r.mn, xn);
                vx[e] = r.mx;
                vn[e] = r.mn;
            }
            sts8(hx + j0, vx);
            sts8(hn + j0, vn);
            carry.mx = __shfl_sync(0xffffffffu, r.mx, 0);
            carry.mn = __shfl_sync(0xffffffffu, r.mn, 0);
        }
        __syncwarp();
        // ---- envelope of A' at column j and the LB_Keogh(B, env A') terms ---------------
        float acc = 0.0f;
#pragma unroll 4
        for (int j = c_lo + lane; j < c_hi; j += 32) {
            const int jl = j - w < 0 ? 0 : j - w;
            const int jr = j + w;
            const int jg = jr < L - 1 ? jr : L - 1;  // past L-1 in L-1's block: g[L-1]
            const bool gok = jr <= blast_end;         // in a later block: -inf (no term)
            const float gxv = gx[jg], gnv = gn[jg];
            const float ux = fmaxf(hx[jl], gok ? gxv : -kInf);
            const float un = fminf(hn[jl], gok ? gnv : kInf);
            const float bj = bs[j];
            const float d = fmaxf(fmaxf(bj - ux, un - bj), 0.0f);
            acc = fmaf(d, d, acc);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) lb[qi * ldlb + ni] += acc;
        __syncwarp();
    }
}

int launch_lb_improved_pass(const float *q, int64_t nq, const float *t, const float *U,
                            const float *Lo, int64_t nt, int L, int w, int c_lo, int c_hi,
                            float *lb, int64_t ldlb, int num_sms, cudaStream_t st) {
    if (nq == 0 || nt == 0) return 0;
    if (w > L - 1) w = L - 1;
    if (c_lo < 0) c_lo = 0;
    if (c_hi > L) c_hi = L;
    if (c_hi <= c_lo) return 0;
    const int Lp = (L + IMP_CH - 1) / IMP_CH * IMP_CH;
    const size_t warp_bytes = (size_t)6 * Lp * sizeof(float);
    int warps = (int)((110 * 1024) / warp_bytes);  // two CTAs per SM
    if (warps < 1) warps = (int)((220 * 1024) / warp_bytes);
    if (warps < 1) return -1;  // L > 9216
    if (warps > 8) warps = 8;
    const size_t smem = warps * warp_bytes;
    const int64_t npairs = nq * nt;
    const int64_t want = (int64_t)num_sms * 2 * warps;  // warps resident
    int rows = (int)((npairs + want * 4 - 1) / (want * 4));  // ~4 waves of pairs per warp slot
    if (rows < 1) rows = 1;
    const int64_t grid = (npairs + (int64_t)warps * rows - 1) / ((int64_t)warps * rows);
    const bool vec = (L % 4) == 0 && ((uintptr_t)q % 16) == 0 && ((uintptr_t)U % 16) == 0 &&
                     ((uintptr_t)Lo % 16) == 0;
    if (vec) {
        cudaFuncSetAttribute(k_lb_improved_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        k_lb_improved_pass<true><<<(unsigned)grid, 32 * warps, smem, st>>>(
            q, nq, t, U, Lo, nt, L, w, c_lo, c_hi, lb, ldlb, rows);
    } else {
        cudaFuncSetAttribute(k_lb_improved_pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        k_lb_improved_pass<false><<<(unsigned)grid, 32 * warps, smem, st>>>(
            q, nq, t, U, Lo, nt, L, w, c_lo, c_hi, lb, ldlb, rows);
    }
    count_launch(1, __func__);
    return 0;
}

// ---- bound finish pass (classify S2 with a bound assembled outside the tile kernel) -----------
// v = lb[q][n]; with_kim: v = max(v, LB_Kim) (the cascade's first level); the
// leave-one-out self pair becomes NaN (never compacted, never the seed); minkey[q] = the
// smallest (v bits << 32 | n) -- the argmin-LB seed candidate of S3, lowest index on ties.
__global__ void __launch_bounds__(256) k_bound_finish(float *lb, int64_t ldlb, int64_t nq,
                                                      int64_t nt, const float *__restrict__ q,
                                                      const float *__restrict__ t,
                                                      const nndtw_kim *__restrict__ qkim,
                                                      const nndtw_kim *__restrict__ tkim, int L,
                                                      int64_t self_offset,
                                                      unsigned long long *minkey) {
    const int64_t qi = blockIdx.x;
    if (qi >= nq) return;
    unsigned long long best = kNone;
    const float qf = q[qi * L], ql = q[qi * L + L - 1];
    for (int64_t n = threadIdx.x; n < nt; n += blockDim.x) {
        float v = lb[qi * ldlb + n];
        if (qkim != nullptr)
            v = fmaxf(v, kim_sum(qf, ql, t[n * L], t[n * L + L - 1], qkim[qi], tkim[n], L));
        const bool self = self_offset >= 0 && n == qi + self_offset;
        if (self) v = __int_as_float(0x7fffffff);
        lb[qi * ldlb + n] = v;
        const unsigned long long k = make_key(v, (unsigned)n);
        if (!self) best = k < best ? k : best;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, off);
        best = o < best ? o : best;
    }
    __shared__ unsigned long long red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) best = red[i] < best ? red[i] : best;
        if (best != kNone && minkey != nullptr) atomicMin(minkey + qi, best);
    }
}

int launch_bound_finish(float *lb, int64_t ldlb, int64_t nq, int64_t nt, const float *q,
                        const float *t, const nndtw_kim *qkim, const nndtw_kim *tkim, int L,
                        int64_t self_offset, unsigned long long *minkey, cudaStream_t st) {
    if (nq == 0 || nt == 0) return 0;
    if (nq > 0x7fffffffll) return -1;
    k_bound_finish<<<(unsigned)nq, 256, 0, st>>>(lb, ldlb, nq, nt, q, t, qkim, tkim, L,
                                                 self_offset, minkey);
    count_launch(1, __func__);
    return 0;
}

}  // namespace nndtw
