// envelopes.cu -- S1: upper/lower warping envelopes (Eq. 3-4) and LB_Kim features.
//
// Design: O(1) work per element independent of w, so the kernel is HBM-bound
// (12 B per element: read x, write U and L).  Van Herk / Gil-Werman: in padded coordinates the
// clipped window [i-w, i+w] has length k = 2w+1; cutting the axis into segments of length k
// aligned at padded position 0 (position p starts a segment iff (p+w) mod k == 0), every
// window is a suffix of one segment plus a prefix of the next, so
//   U_i = max(h[max(i-w,0)], (i+w <= L-1 || i < T) ? g[min(i+w,L-1)] : -inf),
// g = prefix max within the segment, h = suffix max, T = (seg(L-1)+1)*k - 2w (the window's
// right part lies in the same segment as L-1).  Likewise L_i with min.
//
// A group of TPS = 32*ceil(L/(32E)) threads owns one series; thread t holds the E contiguous
// elements [tE, tE+E) in registers (float4 loads).  Segment starts inside a chunk are a bit
// mask computed once per thread (one modulo per thread, none per element); the in-register
// prefix/suffix runs are completed across threads by one segmented warp scan per direction
// (shuffles) plus a carry over the group's warps.  g and h go to shared memory for the
// windowed gather; U and L leave as float4 stores.  The Kim features (min/max and their
// lowest indices) come from the same registers.
#include <cstdlib>

#include "launchers.cuh"

namespace nndtw {

struct Seg {  // running segmented value: (max, min) and "a segment boundary was crossed"
    float mx, mn;
    int f;
};

__device__ __forceinline__ Seg seg_shfl_up(Seg v, int off) {
    return {__shfl_up_sync(0xffffffffu, v.mx, off), __shfl_up_sync(0xffffffffu, v.mn, off),
            __shfl_up_sync(0xffffffffu, v.f, off)};
}
__device__ __forceinline__ Seg seg_shfl_down(Seg v, int off) {
    return {__shfl_down_sync(0xffffffffu, v.mx, off), __shfl_down_sync(0xffffffffu, v.mn, off),
            __shfl_down_sync(0xffffffffu, v.f, off)};
}
// a then b in scan order: b restarts the segment if it crossed a boundary
__device__ __forceinline__ Seg seg_cat(Seg a, Seg b) {
    if (b.f) return b;
    return {fmaxf(a.mx, b.mx), fminf(a.mn, b.mn), a.f};
}

template <int E>
__global__ void __launch_bounds__(512) k_envelopes(const float *__restrict__ x, int64_t n,
                                                   int L, int w, int tps, int vec, int T,
                                                   float *__restrict__ U,
                                                   float *__restrict__ Lo,
                                                   nndtw_kim *__restrict__ kim) {
    extern __shared__ __align__(16) unsigned char env_smem[];
    const int groups = blockDim.x / tps;
    const int grp = threadIdx.x / tps;
    const int t = threadIdx.x - grp * tps;
    const int lane = threadIdx.x & 31;
    const int wig = t >> 5;
    const int nw = tps >> 5;
    const int k = 2 * w + 1;
    const int span = tps * E;
    const int pspan = span + (span >> 4) + 1;  // one pad slot per 16: thread-strided access
    auto pad = [](int q) { return q + (q >> 4); };  // is bank-conflict free

    float2 *G = reinterpret_cast<float2 *>(env_smem) + (size_t)grp * 2 * pspan;
    float2 *H = G + pspan;
    Seg *tot = reinterpret_cast<Seg *>(reinterpret_cast<float2 *>(env_smem) +
                                       (size_t)groups * 2 * pspan) + grp * 32;  // [0,16) fwd, [16,32) bwd
    const int p0 = t * E;
    const int64_t s = (int64_t)blockIdx.x * groups + grp;
    const bool live = s < n;

    // ---- load E contiguous elements -------------------------------------------------------
    const float *xs = x + (live ? s : 0) * (int64_t)L;
    float v[E];
    if (vec) {
#pragma unroll
        for (int j = 0; j < E / 4; ++j) {
            float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
            if (live && p0 + 4 * j < L) f = __ldg(reinterpret_cast<const float4 *>(xs + p0) + j);
            v[4 * j] = f.x;
            v[4 * j + 1] = f.y;
            v[4 * j + 2] = f.z;
            v[4 * j + 3] = f.w;
        }
    } else {
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = (live && p0 + e < L) ? __ldg(xs + p0 + e) : 0.0f;
    }
    const int nvalid = L - p0;  // elements e < nvalid are real

    // ---- segment starts inside [p0, p0+E]: bit e set iff (p0+e+w) mod k == 0; position L
    // also starts one (so no scan ever mixes padding into a real position) ----------------------
    unsigned m = 0;
    {
        const int r0 = (p0 + w) % k;
        for (int q = (r0 == 0) ? 0 : k - r0; q <= E; q += k) m |= 1u << q;
        if (nvalid >= 0 && nvalid <= E) m |= 1u << nvalid;
    }

    // ---- forward: g = running max/min from the segment start ------------------------------------
    float gx[E], gn[E];
    gx[0] = v[0];
    gn[0] = v[0];
#pragma unroll
    for (int e = 1; e < E; ++e) {
        const bool st = (m >> e) & 1u;
        gx[e] = st ? v[e] : fmaxf(gx[e - 1], v[e]);
        gn[e] = st ? v[e] : fminf(gn[e - 1], v[e]);
    }
    // ---- backward: h = running max/min to the segment end ---------------------------------------
    float hx[E], hn[E];
    hx[E - 1] = v[E - 1];
    hn[E - 1] = v[E - 1];
#pragma unroll
    for (int e = E - 2; e >= 0; --e) {
        const bool en = (m >> (e + 1)) & 1u;
        hx[e] = en ? v[e] : fmaxf(hx[e + 1], v[e]);
        hn[e] = en ? v[e] : fminf(hn[e + 1], v[e]);
    }

    // ---- cross-thread completion: segmented scans (forward over t ascending, backward
    // descending); a thread's aggregate restarts if its chunk contains a boundary ------------
    const unsigned mfwd = m & ((1u << E) - 1u);   // starts at e in [0, E)
    const unsigned mbwd = m >> 1;                 // ends at e in [0, E)
    Seg af{gx[E - 1], gn[E - 1], mfwd != 0u};
    Seg ab{hx[0], hn[0], mbwd != 0u};
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        Seg pf = seg_shfl_up(af, off);
        Seg pb = seg_shfl_down(ab, off);
        if (lane >= off) af = seg_cat(pf, af);
        if (lane + off < 32) ab = seg_cat(pb, ab);
    }
    Seg cf{-kInf, kInf, 1}, cb{-kInf, kInf, 1};  // carries from earlier warps ("f=1": none)
    if (nw > 1) {
        if (lane == 31) tot[wig] = af;
        if (lane == 0) tot[16 + wig] = ab;
        __syncthreads();
        for (int j = 0; j < wig; ++j) cf = (j == 0) ? tot[j] : seg_cat(cf, tot[j]);
        for (int j = nw - 1; j > wig; --j) cb = (j == nw - 1) ? tot[16 + j] : seg_cat(cb, tot[16 + j]);
        af = seg_cat(cf, af);
        ab = seg_cat(cb, ab);
    }
    // exclusive carry into this thread = inclusive value of the previous thread in scan order
    Seg inf{__shfl_up_sync(0xffffffffu, af.mx, 1), __shfl_up_sync(0xffffffffu, af.mn, 1), 0};
    Seg inb{__shfl_down_sync(0xffffffffu, ab.mx, 1), __shfl_down_sync(0xffffffffu, ab.mn, 1), 0};
    if (lane == 0) inf = {cf.mx, cf.mn, 0};   // identity when wig == 0
    if (lane == 31) inb = {cb.mx, cb.mn, 0};
    const int bf = mfwd ? __ffs(mfwd) - 1 : E;            // elements e < bf continue a segment
    const int bb = mbwd ? 31 - __clz(mbwd) : -1;          // elements e > bb continue one
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (e < bf) {
            gx[e] = fmaxf(gx[e], inf.mx);
            gn[e] = fminf(gn[e], inf.mn);
        }
        if (e > bb) {
            hx[e] = fmaxf(hx[e], inb.mx);
            hn[e] = fminf(hn[e], inb.mn);
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        G[pad(p0 + e)] = make_float2(gx[e], gn[e]);
        H[pad(p0 + e)] = make_float2(hx[e], hn[e]);
    }
    __syncthreads();

    // ---- gather the window extremes for this thread's own elements ------------------------------
    // U_p = max(h[max(p-w,0)], g[min(p+w,L-1)] if p < Tg), Tg = max(L-w, T)
    const int Tg = (L - w > T) ? L - w : T;
    float ux[E], ln[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int p = p0 + e;
        const int lo = max(p - w, 0);
        const int hc = min(p + w, L - 1);
        const float2 hv = H[pad(lo)];
        const float2 gv = G[pad(hc)];
        const bool useg = p < Tg;
        ux[e] = useg ? fmaxf(hv.x, gv.x) : hv.x;
        ln[e] = useg ? fminf(hv.y, gv.y) : hv.y;
    }
    if (live) {
        float *Us = U + s * (int64_t)L;
        float *Ls = Lo + s * (int64_t)L;
        if (vec) {
#pragma unroll
            for (int j = 0; j < E / 4; ++j) {
                if (p0 + 4 * j < L) {
                    reinterpret_cast<float4 *>(Us + p0)[j] =
                        make_float4(ux[4 * j], ux[4 * j + 1], ux[4 * j + 2], ux[4 * j + 3]);
                    reinterpret_cast<float4 *>(Ls + p0)[j] =
                        make_float4(ln[4 * j], ln[4 * j + 1], ln[4 * j + 2], ln[4 * j + 3]);
                }
            }
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e)
                if (e < nvalid) {
                    Us[p0 + e] = ux[e];
                    Ls[p0 + e] = ln[e];
                }
        }
    }

    // ---- LB_Kim features: min / max and their lowest indices (reading C7) ----------------------
    if (kim != nullptr) {
        float mn = kInf, mx = -kInf;
        int imn = 0x7fffffff, imx = 0x7fffffff;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (e < nvalid) {
                if (v[e] < mn) { mn = v[e]; imn = p0 + e; }
                if (v[e] > mx) { mx = v[e]; imx = p0 + e; }
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
        if (nw > 1) {
            __syncthreads();  // tot[] reuse
            float4 *red = reinterpret_cast<float4 *>(tot);
            if (lane == 0) red[wig] = make_float4(mn, __int_as_float(imn), mx, __int_as_float(imx));
            __syncthreads();
            if (t == 0) {
                for (int q = 1; q < nw; ++q) {
                    float4 r = red[q];
                    float omn = r.x, omx = r.z;
                    int oimn = __float_as_int(r.y), oimx = __float_as_int(r.w);
                    if (omn < mn || (omn == mn && oimn < imn)) { mn = omn; imn = oimn; }
                    if (omx > mx || (omx == mx && oimx < imx)) { mx = omx; imx = oimx; }
                }
            }
        }
        if (t == 0 && live) {
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
    static const char *ef = getenv("NNDTW_ENV_E");  // experiments: force elements per thread
    int E = L <= 128 ? 4 : (L <= 256 ? 8 : 16);
    if (ef) E = atoi(ef);
    const int tps = (L + 32 * E - 1) / (32 * E) * 32;
    if (tps > 512) return -1;  // L > 8192
    const int block = tps >= 256 ? tps : 256;
    const int groups = block / tps;
    const int span = tps * E;
    const int pspan = span + (span >> 4) + 1;
    const size_t smem = (size_t)groups * 2 * pspan * sizeof(float2) + (size_t)groups * 32 * 16;
    const int k = 2 * w + 1;
    const int T = ((L - 1 + w) / k + 1) * k - 2 * w;
    const int vec = (L % 4 == 0 && ((uintptr_t)x % 16) == 0 && ((uintptr_t)U % 16) == 0 &&
                     ((uintptr_t)Lo % 16) == 0) ? 1 : 0;
    const int64_t grid = (n + groups - 1) / groups;
    if (grid > 0x7fffffffll) return -1;
#define ENV_LAUNCH(EE)                                                                            \
    do {                                                                                          \
        if (smem > 48 * 1024)                                                                     \
            cudaFuncSetAttribute(k_envelopes<EE>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                 (int)smem);                                                      \
        k_envelopes<EE><<<(unsigned)grid, block, smem, st>>>(x, n, L, w, tps, vec, T, U, Lo, kim); \
    } while (0)
    if (E == 4) ENV_LAUNCH(4);
    else if (E == 8) ENV_LAUNCH(8);
    else ENV_LAUNCH(16);
#undef ENV_LAUNCH
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
