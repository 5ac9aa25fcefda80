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
// covers [j-w, L-1]).  The prefix / suffix scans are warp-segmented scans (resets at block
// starts / ends) over chunks of 32*CE elements with a carry across chunks: O(1) work per
// element, independent of w.
//
// The kernel computes only the SECOND pass, sum over columns j in [c_lo, c_hi) of
// keogh(B_j, L'_j, U'_j), and ADDS it to lb[q][n]; the first pass is the LB tile kernel
// (lb.cu):
//   * LB_Improved           = tile kernel in LB_Keogh mode            + pass over [0, L)
//   * LB_Enhanced^V with the LB_Improved bridge (reading C21)
//                           = tile kernel (bands + LB_Keogh bridge)   + pass over
//                             [nb + w, L - nb - w), the columns whose window lies inside the
//                             bridge rows [nb, L - nb).
// Both stay admissible: for a path cell (i, j) with |i-j| <= w, B_j is inside [L^B_i, U^B_i],
// so (A_i - B_j)^2 >= (A_i - A'_i)^2 + (A'_i - B_j)^2 (the cross term is >= 0); the first
// terms are counted once per row (the Keogh terms), the second once per column of the range
// (every path visits each such column in some bridge row), reading C21.
#include "launchers.cuh"

namespace nndtw {

constexpr int IMP_CE = 4;                 // elements per lane per chunk
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
        const bool in = UP ? lane >= off : lane + off < 32;
        if (in && !f) {
            v.mx = fmaxf(v.mx, ox);
            v.mn = fminf(v.mn, on);
            f = of;
        }
    }
}

__global__ void __launch_bounds__(256) k_lb_improved_pass(const float *__restrict__ q, int64_t nq,
                                                          const float *__restrict__ t,
                                                          const float *__restrict__ U,
                                                          const float *__restrict__ Lo,
                                                          int64_t nt, int L, int w, int c_lo,
                                                          int c_hi, float *lb, int64_t ldlb,
                                                          int rows_per_warp) {
    extern __shared__ float imp_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    float *ap = imp_smem + (size_t)warp * 5 * L;  // A' [L]
    float *gx = ap + L, *gn = gx + L, *hx = gn + L, *hn = hx + L;
    const int K = 2 * w + 1;
    const int nch = (L + IMP_CH - 1) / IMP_CH;
    const int64_t npairs = nq * nt;
    for (int64_t pr = ((int64_t)blockIdx.x * nwarps + warp) * rows_per_warp, pe = pr + rows_per_warp;
         pr < pe && pr < npairs; ++pr) {
        const int64_t qi = pr / nt, ni = pr - qi * nt;
        const float *a = q + qi * L, *b = t + ni * L, *u = U + ni * L, *lo = Lo + ni * L;
        // ---- projection A' and the forward (prefix) segmented scan ----------------------
        MaxMin carry{-kInf, kInf};
        for (int c = 0; c < nch; ++c) {
            const int j0 = c * IMP_CH + lane * IMP_CE;
            float x[IMP_CE];
            MaxMin run{-kInf, kInf};
            int f = 0;
#pragma unroll
            for (int e = 0; e < IMP_CE; ++e) {
                const int j = j0 + e;
                float v = 0.0f;
                if (j < L) v = fminf(fmaxf(__ldg(a + j), __ldg(lo + j)), __ldg(u + j));
                x[e] = v;
                if (j < L) ap[j] = v;
                const bool reset = ((j + w) % K) == 0;
                if (j < L) {
                    if (reset) { run.mx = v; run.mn = v; f = 1; }
                    else { run.mx = fmaxf(run.mx, v); run.mn = fminf(run.mn, v); }
                }
            }
            MaxMin inc = run;
            int fi = f;
            seg_scan<true>(fi, inc, lane);
            // carry into this lane = inclusive result of lane-1 (combined with the chunk carry)
            MaxMin cin;
            int fprev;
            cin.mx = __shfl_up_sync(0xffffffffu, inc.mx, 1);
            cin.mn = __shfl_up_sync(0xffffffffu, inc.mn, 1);
            fprev = __shfl_up_sync(0xffffffffu, fi, 1);
            if (lane == 0) { cin = carry; fprev = 1; }
            else if (!fprev) { cin.mx = fmaxf(cin.mx, carry.mx); cin.mn = fminf(cin.mn, carry.mn); }
            // rewrite this lane's prefix values: carry applies until the lane's first reset
            MaxMin r = cin;
#pragma unroll
            for (int e = 0; e < IMP_CE; ++e) {
                const int j = j0 + e;
                if (j < L) {
                    if (((j + w) % K) == 0) { r.mx = x[e]; r.mn = x[e]; }
                    else { r.mx = fmaxf(r.mx, x[e]); r.mn = fminf(r.mn, x[e]); }
                    gx[j] = r.mx;
                    gn[j] = r.mn;
                }
            }
            // chunk carry = value after the last element of the chunk (lane 31)
            carry.mx = __shfl_sync(0xffffffffu, r.mx, 31);
            carry.mn = __shfl_sync(0xffffffffu, r.mn, 31);
        }
        __syncwarp();
        // ---- backward (suffix) segmented scan: resets at block ends ---------------------
        carry = MaxMin{-kInf, kInf};
        for (int c = nch - 1; c >= 0; --c) {
            const int j0 = c * IMP_CH + lane * IMP_CE;
            float x[IMP_CE];
            MaxMin run{-kInf, kInf};
            int f = 0;
#pragma unroll
            for (int e = IMP_CE - 1; e >= 0; --e) {
                const int j = j0 + e;
                x[e] = j < L ? ap[j] : 0.0f;
                const bool reset = ((j + w + 1) % K) == 0;  // j is the last index of its block
                if (j < L) {
                    if (reset) { run.mx = x[e]; run.mn = x[e]; f = 1; }
                    else { run.mx = fmaxf(run.mx, x[e]); run.mn = fminf(run.mn, x[e]); }
                }
            }
            MaxMin inc = run;
            int fi = f;
            seg_scan<false>(fi, inc, lane);
            MaxMin cin;
            int fnext;
            cin.mx = __shfl_down_sync(0xffffffffu, inc.mx, 1);
            cin.mn = __shfl_down_sync(0xffffffffu, inc.mn, 1);
            fnext = __shfl_down_sync(0xffffffffu, fi, 1);
            if (lane == 31) { cin = carry; fnext = 1; }
            else if (!fnext) { cin.mx = fmaxf(cin.mx, carry.mx); cin.mn = fminf(cin.mn, carry.mn); }
            MaxMin r = cin;
#pragma unroll
            for (int e = IMP_CE - 1; e >= 0; --e) {
                const int j = j0 + e;
                if (j < L) {
                    if (((j + w + 1) % K) == 0) { r.mx = x[e]; r.mn = x[e]; }
                    else { r.mx = fmaxf(r.mx, x[e]); r.mn = fminf(r.mn, x[e]); }
                    hx[j] = r.mx;
                    hn[j] = r.mn;
                }
            }
            carry.mx = __shfl_sync(0xffffffffu, r.mx, 0);
            carry.mn = __shfl_sync(0xffffffffu, r.mn, 0);
        }
        __syncwarp();
        // ---- envelope of A' at column j and the LB_Keogh(B, env A') terms ---------------
        const int blast = (L - 1 + w) / K;  // block of index L-1
        float acc = 0.0f;
        for (int j = c_lo + lane; j < c_hi; j += 32) {
            const int jl = j - w < 0 ? 0 : j - w;
            const int jr = j + w;
            float ux = hx[jl], un = hn[jl];
            if (jr <= L - 1) {
                ux = fmaxf(ux, gx[jr]);
                un = fminf(un, gn[jr]);
            } else if ((jr + w) / K == blast) {
                ux = fmaxf(ux, gx[L - 1]);
                un = fminf(un, gn[L - 1]);
            }
            const float bj = __ldg(b + j);
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
    const size_t warp_bytes = (size_t)5 * L * sizeof(float);
    int warps = (int)((200 * 1024) / warp_bytes);
    if (warps < 1) return -1;  // L > 10240
    if (warps > 8) warps = 8;
    const size_t smem = warps * warp_bytes;
    const int64_t npairs = nq * nt;
    int64_t want = (int64_t)num_sms * 8 * warps;  // warps in flight
    int rows = (int)((npairs + want - 1) / want);
    if (rows < 1) rows = 1;
    const int64_t grid = (npairs + (int64_t)warps * rows - 1) / ((int64_t)warps * rows);
    cudaFuncSetAttribute(k_lb_improved_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_lb_improved_pass<<<(unsigned)grid, 32 * warps, smem, st>>>(q, nq, t, U, Lo, nt, L, w, c_lo,
                                                                  c_hi, lb, ldlb, rows);
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
