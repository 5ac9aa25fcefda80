// envelopes.cu -- S1: upper/lower warping envelopes (Eq. 3-4) and LB_Kim features.
//
// Design: O(1) work per element independent of w, HBM-bound.  The clipped
// window [i-w, i+w] has length k = 2w+1 in "padded" coordinates; cutting the padded axis into
// segments of length k aligned at position -w (seg(p) = (p+w)/k), every window is the union of
// a suffix of one segment and a prefix of the next (van Herk / Gil-Werman).  Each thread owns
// E consecutive elements in registers; the segmented prefix (g) and suffix (h) max/min are
// computed with a register scan + warp-shuffle segmented scan + cross-warp carry, staged in
// shared memory, and combined as
//   U_i = max(h[max(i-w,0)], seg(i+w) == seg(min(i+w,L-1)) ? g[min(i+w,L-1)] : -inf).
// One "series group" of TPS = 32*ceil(L/(32E)) threads handles one series; several groups
// share a CTA when L is short.
#include "launchers.cuh"

namespace nndtw {

template <int E>
struct EnvCfg {
    static constexpr int kBlock = 256;
};

struct MaxMin {
    float mx, mn;
};

__device__ __forceinline__ MaxMin mm_op(MaxMin a, MaxMin b) {
    return {fmaxf(a.mx, b.mx), fminf(a.mn, b.mn)};
}

// Segmented inclusive scan over the TPS threads of a series group, forward (DIR=+1, thread t
// combines with t-1, t-2, ...) or backward (DIR=-1).  `pass` = this element does not start a
// segment (so it absorbs the running value of its predecessor in scan order).
template <int DIR>
__device__ __forceinline__ MaxMin seg_scan(MaxMin v, bool pass, int lane, int wig, int nwarps,
                                           MaxMin *s_val, int *s_pass) {
    // warp level: predecessor in scan order is lane-1 (forward) or lane+1 (backward)
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        float pmx, pmn;
        int ppass;
        if (DIR > 0) {
            pmx = __shfl_up_sync(0xffffffffu, v.mx, off);
            pmn = __shfl_up_sync(0xffffffffu, v.mn, off);
            ppass = __shfl_up_sync(0xffffffffu, (int)pass, off);
        } else {
            pmx = __shfl_down_sync(0xffffffffu, v.mx, off);
            pmn = __shfl_down_sync(0xffffffffu, v.mn, off);
            ppass = __shfl_down_sync(0xffffffffu, (int)pass, off);
        }
        bool valid = DIR > 0 ? (lane >= off) : (lane + off < 32);
        if (valid) {
            if (pass) v = mm_op(v, {pmx, pmn});
            pass = pass && ppass;
        }
    }
    if (nwarps > 1) {
        // warp totals (last element in scan order) -> smem, sequential combine by one thread
        int last_lane = DIR > 0 ? 31 : 0;
        if (lane == last_lane) {
            s_val[wig] = v;
            s_pass[wig] = pass;
        }
        __syncthreads();
        if (lane == 0 && wig == 0) {
            // exclusive prefix over warps in scan order, stored back in place
            MaxMin run = {-kInf, kInf};
            bool have = false;
            for (int s = 0; s < nwarps; ++s) {
                int wi = DIR > 0 ? s : nwarps - 1 - s;
                MaxMin tot = s_val[wi];
                int tp = s_pass[wi];
                s_val[wi] = run;          // carry INTO warp wi
                s_pass[wi] = have;
                // running value after warp wi: if wi is all-pass, combine with previous
                if (tp && have) run = mm_op(run, tot);
                else run = tot;
                have = true;
            }
        }
        __syncthreads();
        MaxMin carry = s_val[wig];
        bool has = s_pass[wig];
        // elements of this warp that are still "passing" at the warp start absorb the carry
        if (has && pass) v = mm_op(v, carry);
        __syncthreads();
    }
    return v;
}

template <int E>
__global__ void __launch_bounds__(256) k_envelopes(const float *__restrict__ x, int64_t n,
                                                   int L, int w, int tps, float *__restrict__ U,
                                                   float *__restrict__ Lo,
                                                   nndtw_kim *__restrict__ kim) {
    extern __shared__ float smem[];
    const int groups = blockDim.x / tps;
    const int grp = threadIdx.x / tps;
    const int t = threadIdx.x % tps;
    const int lane = threadIdx.x & 31;
    const int wig = t >> 5;             // warp within group
    const int nwarps = tps >> 5;
    const int64_t s = (int64_t)blockIdx.x * groups + grp;
    const bool live = s < n;
    const int k = 2 * w + 1;

    float *gmx = smem + (size_t)grp * 4 * L;
    float *gmn = gmx + L;
    float *hmx = gmn + L;
    float *hmn = hmx + L;
    // scan scratch after the 4*L*groups floats
    MaxMin *s_val = reinterpret_cast<MaxMin *>(smem + (size_t)groups * 4 * L) + grp * 32;
    int *s_pass = reinterpret_cast<int *>(smem + (size_t)groups * 4 * L + groups * 64) + grp * 32;

    const float *xs = x + (live ? s : 0) * (int64_t)L;
    float v[E];
    const int p0 = t * E;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        int p = p0 + e;
        v[e] = (live && p < L) ? __ldg(xs + p) : 0.0f;
    }
    auto seg = [&](int p) { return (p + w) / k; };

    // ---- forward (prefix within segment) --------------------------------------------
    float fmx[E], fmn[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        int p = p0 + e;
        bool in = p < L;
        float vx = in ? v[e] : -kInf, vn = in ? v[e] : kInf;
        if (e > 0 && seg(p) == seg(p - 1)) {
            fmx[e] = fmaxf(fmx[e - 1], vx);
            fmn[e] = fminf(fmn[e - 1], vn);
        } else {
            fmx[e] = vx;
            fmn[e] = vn;
        }
    }
    {
        bool pass = (t > 0) && seg(p0 - 1) == seg(p0 + E - 1);
        MaxMin agg = seg_scan<1>({fmx[E - 1], fmn[E - 1]}, pass, lane, wig, nwarps, s_val,
                                 s_pass);
        // carry = inclusive result of thread t-1
        float cmx = __shfl_up_sync(0xffffffffu, agg.mx, 1);
        float cmn = __shfl_up_sync(0xffffffffu, agg.mn, 1);
        if (nwarps > 1) {
            // lane 0 needs the last lane of the previous warp
            if (lane == 31) {
                s_val[wig] = agg;
            }
            __syncthreads();
            if (lane == 0 && wig > 0) {
                cmx = s_val[wig - 1].mx;
                cmn = s_val[wig - 1].mn;
            }
            __syncthreads();
        }
        bool carry_in = (t > 0) && seg(p0 - 1) == seg(p0);
        if (carry_in) {
            int s0 = seg(p0);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                if (seg(p0 + e) == s0) {
                    fmx[e] = fmaxf(fmx[e], cmx);
                    fmn[e] = fminf(fmn[e], cmn);
                }
            }
        }
    }
    // ---- backward (suffix within segment) -------------------------------------------
    float bmx[E], bmn[E];
#pragma unroll
    for (int e = E - 1; e >= 0; --e) {
        int p = p0 + e;
        bool in = p < L;
        float vx = in ? v[e] : -kInf, vn = in ? v[e] : kInf;
        if (e < E - 1 && seg(p) == seg(p + 1)) {
            bmx[e] = fmaxf(bmx[e + 1], vx);
            bmn[e] = fminf(bmn[e + 1], vn);
        } else {
            bmx[e] = vx;
            bmn[e] = vn;
        }
    }
    {
        bool pass = (t < tps - 1) && seg(p0) == seg(p0 + E);
        MaxMin agg = seg_scan<-1>({bmx[0], bmn[0]}, pass, lane, wig, nwarps, s_val, s_pass);
        float cmx = __shfl_down_sync(0xffffffffu, agg.mx, 1);
        float cmn = __shfl_down_sync(0xffffffffu, agg.mn, 1);
        if (nwarps > 1) {
            if (lane == 0) s_val[wig] = agg;
            __syncthreads();
            if (lane == 31 && wig < nwarps - 1) {
                cmx = s_val[wig + 1].mx;
                cmn = s_val[wig + 1].mn;
            }
            __syncthreads();
        }
        bool carry_in = (t < tps - 1) && seg(p0 + E - 1) == seg(p0 + E);
        if (carry_in) {
            int s1 = seg(p0 + E - 1);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                if (seg(p0 + e) == s1) {
                    bmx[e] = fmaxf(bmx[e], cmx);
                    bmn[e] = fminf(bmn[e], cmn);
                }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        int p = p0 + e;
        if (p < L) {
            gmx[p] = fmx[e];
            gmn[p] = fmn[e];
            hmx[p] = bmx[e];
            hmn[p] = bmn[e];
        }
    }
    __syncthreads();
    if (live) {
        float *Us = U + s * (int64_t)L;
        float *Ls = Lo + s * (int64_t)L;
        for (int i = t; i < L; i += tps) {
            int lo = i - w < 0 ? 0 : i - w;
            int hi = i + w;
            int hc = hi < L - 1 ? hi : L - 1;
            float u = hmx[lo], l = hmn[lo];
            if (seg(hi) == seg(hc)) {
                u = fmaxf(u, gmx[hc]);
                l = fminf(l, gmn[hc]);
            }
            Us[i] = u;
            Ls[i] = l;
        }
    }
    if (kim != nullptr) {
        // LB_Kim features: min/max with the lowest index on ties (reading C7)
        float mn = kInf, mx = -kInf;
        int imn = 0x7fffffff, imx = 0x7fffffff;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            int p = p0 + e;
            if (p < L) {
                if (v[e] < mn) { mn = v[e]; imn = p; }
                if (v[e] > mx) { mx = v[e]; imx = p; }
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            float omn = __shfl_down_sync(0xffffffffu, mn, off);
            int oimn = __shfl_down_sync(0xffffffffu, imn, off);
            float omx = __shfl_down_sync(0xffffffffu, mx, off);
            int oimx = __shfl_down_sync(0xffffffffu, imx, off);
            if (omn < mn || (omn == mn && oimn < imn)) { mn = omn; imn = oimn; }
            if (omx > mx || (omx == mx && oimx < imx)) { mx = omx; imx = oimx; }
        }
        __syncthreads();
        float *red = gmx;  // reuse (envelope outputs already written)
        if (lane == 0) {
            red[wig * 4 + 0] = mn;
            red[wig * 4 + 1] = __int_as_float(imn);
            red[wig * 4 + 2] = mx;
            red[wig * 4 + 3] = __int_as_float(imx);
        }
        __syncthreads();
        if (t == 0 && live) {
            for (int q = 1; q < nwarps; ++q) {
                float omn = red[q * 4 + 0], omx = red[q * 4 + 2];
                int oimn = __float_as_int(red[q * 4 + 1]), oimx = __float_as_int(red[q * 4 + 3]);
                if (omn < mn || (omn == mn && oimn < imn)) { mn = omn; imn = oimn; }
                if (omx > mx || (omx == mx && oimx < imx)) { mx = omx; imx = oimx; }
            }
            nndtw_kim r;
            r.vmin = mn;
            r.vmax = mx;
            r.imin = imn;
            r.imax = imx;
            kim[s] = r;
        }
    }
}

// Kim features only (query side).  One warp per series.
__global__ void k_series_stats(const float *__restrict__ x, int64_t n, int L,
                               nndtw_kim *__restrict__ kim) {
    int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (s >= n) return;
    const float *xs = x + s * (int64_t)L;
    float mn = kInf, mx = -kInf;
    int imn = 0x7fffffff, imx = 0x7fffffff;
    for (int p = lane; p < L; p += 32) {
        float v = __ldg(xs + p);
        if (v < mn) { mn = v; imn = p; }
        if (v > mx) { mx = v; imx = p; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        float omn = __shfl_down_sync(0xffffffffu, mn, off);
        int oimn = __shfl_down_sync(0xffffffffu, imn, off);
        float omx = __shfl_down_sync(0xffffffffu, mx, off);
        int oimx = __shfl_down_sync(0xffffffffu, imx, off);
        if (omn < mn || (omn == mn && oimn < imn)) { mn = omn; imn = oimn; }
        if (omx > mx || (omx == mx && oimx < imx)) { mx = omx; imx = oimx; }
    }
    if (lane == 0) {
        nndtw_kim r;
        r.vmin = mn;
        r.vmax = mx;
        r.imin = imn;
        r.imax = imx;
        kim[s] = r;
    }
}

// ---- launchers ---------------------------------------------------------------------------
int launch_envelopes(const float *x, int64_t n, int L, int w, float *U, float *Lo,
                     nndtw_kim *kim, cudaStream_t st) {
    if (n == 0) return 0;
    if (w > L - 1) w = L - 1;
    const int E = 8;
    int tps = ((L + E - 1) / E + 31) / 32 * 32;
    int block = tps >= 256 ? tps : 256 / tps * tps;
    int groups = block / tps;
    size_t smem = (size_t)groups * 4 * L * sizeof(float) + (size_t)groups * 64 * sizeof(float) +
                  (size_t)groups * 32 * sizeof(int);
    if (block > 1024 || smem > 200 * 1024) return -1;
    int64_t grid = (n + groups - 1) / groups;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_envelopes<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    k_envelopes<8><<<(unsigned)grid, block, smem, st>>>(x, n, L, w, tps, U, Lo, kim);
    count_launch(1, __func__);
    return 0;
}

int launch_series_stats(const float *x, int64_t n, int L, nndtw_kim *kim, cudaStream_t st) {
    if (n == 0) return 0;
    int64_t threads = n * 32;
    int64_t grid = (threads + 255) / 256;
    k_series_stats<<<(unsigned)grid, 256, 0, st>>>(x, n, L, kim);
    count_launch(1, __func__);
    return 0;
}

}  // namespace nndtw
