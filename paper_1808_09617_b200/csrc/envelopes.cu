// envelopes.cu -- S1: upper/lower warping envelopes (Eq. 3-4) and LB_Kim features.
//
// Design: O(1) work per element independent of w, so the kernels are HBM-bound
// (12 B per element: read x, write U and L).  Two kernels: k_env_direct (w >= 16; chunk
// prefix/suffix + a sparse table over chunk extremes, further below) and the van Herk kernel
// k_envelopes (w < 16, L <= 256, or padded rows too large for shared memory), described here.
// Van Herk / Gil-Werman: in padded coordinates the
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
#include <algorithm>
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

    // ---- LB_Kim features, thread and warp part (reading C7): values first (min/max only), then
    // the lowest index of the warp's extreme, searched only by the threads that hold it.  Done
    // before the scans so that v[] dies early (registers bound this kernel's occupancy) ---------
    float kmn = kInf, kmx = -kInf;
    unsigned kimn = 0x7fffffffu, kimx = 0x7fffffffu;
    if (kim != nullptr) {
        if (nvalid >= E) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                kmn = fminf(kmn, v[e]);
                kmx = fmaxf(kmx, v[e]);
            }
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                kmn = fminf(kmn, e < nvalid ? v[e] : kInf);
                kmx = fmaxf(kmx, e < nvalid ? v[e] : -kInf);
            }
        }
        const float tmn = kmn, tmx = kmx;  // this thread's own extremes
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            kmn = fminf(kmn, __shfl_xor_sync(0xffffffffu, kmn, off));
            kmx = fmaxf(kmx, __shfl_xor_sync(0xffffffffu, kmx, off));
        }
        if (tmn == kmn) {
            for (int e = E - 1; e >= 0; --e)
                if (e < nvalid && v[e] == kmn) kimn = p0 + e;
        }
        if (tmx == kmx) {
            for (int e = E - 1; e >= 0; --e)
                if (e < nvalid && v[e] == kmx) kimx = p0 + e;
        }
        kimn = __reduce_min_sync(0xffffffffu, kimn);
        kimx = __reduce_min_sync(0xffffffffu, kimx);
    }

    // ---- forward: g = running max/min from the segment start, completed across threads by a
    // segmented scan over t ascending (a thread's aggregate restarts if its chunk holds a
    // boundary); one direction at a time, again for register pressure --------------------------
    {
        const unsigned mfwd = m & ((1u << E) - 1u);  // starts at e in [0, E)
        float gx[E], gn[E];
        gx[0] = v[0];
        gn[0] = v[0];
#pragma unroll
        for (int e = 1; e < E; ++e) {
            const bool st = (m >> e) & 1u;
            gx[e] = st ? v[e] : fmaxf(gx[e - 1], v[e]);
            gn[e] = st ? v[e] : fminf(gn[e - 1], v[e]);
        }
        Seg af{gx[E - 1], gn[E - 1], mfwd != 0u};
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            Seg pf = seg_shfl_up(af, off);
            if (lane >= off) af = seg_cat(pf, af);
        }
        Seg cf{-kInf, kInf, 1};  // carry from earlier warps ("f=1": none)
        if (nw > 1) {
            if (lane == 31) tot[wig] = af;
            __syncthreads();
            for (int j = 0; j < wig; ++j) cf = (j == 0) ? tot[j] : seg_cat(cf, tot[j]);
            af = seg_cat(cf, af);
        }
        // exclusive carry into this thread = inclusive value of the previous thread
        float cmx = __shfl_up_sync(0xffffffffu, af.mx, 1);
        float cmn = __shfl_up_sync(0xffffffffu, af.mn, 1);
        if (lane == 0) { cmx = cf.mx; cmn = cf.mn; }  // identity when wig == 0
        const int bf = mfwd ? __ffs(mfwd) - 1 : E;    // elements e < bf continue a segment
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (e < bf) {
                gx[e] = fmaxf(gx[e], cmx);
                gn[e] = fminf(gn[e], cmn);
            }
            G[pad(p0 + e)] = make_float2(gx[e], gn[e]);
        }
    }
    // ---- backward: h = running max/min to the segment end (scan over t descending) -----------
    {
        const unsigned mbwd = m >> 1;  // ends at e in [0, E)
        float hx[E], hn[E];
        hx[E - 1] = v[E - 1];
        hn[E - 1] = v[E - 1];
#pragma unroll
        for (int e = E - 2; e >= 0; --e) {
            const bool en = (m >> (e + 1)) & 1u;
            hx[e] = en ? v[e] : fmaxf(hx[e + 1], v[e]);
            hn[e] = en ? v[e] : fminf(hn[e + 1], v[e]);
        }
        Seg ab{hx[0], hn[0], mbwd != 0u};
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            Seg pb = seg_shfl_down(ab, off);
            if (lane + off < 32) ab = seg_cat(pb, ab);
        }
        Seg cb{-kInf, kInf, 1};
        if (nw > 1) {
            if (lane == 0) tot[16 + wig] = ab;
            __syncthreads();
            for (int j = nw - 1; j > wig; --j)
                cb = (j == nw - 1) ? tot[16 + j] : seg_cat(cb, tot[16 + j]);
            ab = seg_cat(cb, ab);
        }
        float cmx = __shfl_down_sync(0xffffffffu, ab.mx, 1);
        float cmn = __shfl_down_sync(0xffffffffu, ab.mn, 1);
        if (lane == 31) { cmx = cb.mx; cmn = cb.mn; }
        const int bb = mbwd ? 31 - __clz(mbwd) : -1;  // elements e > bb continue a segment
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (e > bb) {
                hx[e] = fmaxf(hx[e], cmx);
                hn[e] = fminf(hn[e], cmn);
            }
            H[pad(p0 + e)] = make_float2(hx[e], hn[e]);
        }
    }
    __syncthreads();

    // ---- gather the window extremes for this thread's own elements ------------------------------
    // U_p = max(h[max(p-w,0)], g[min(p+w,L-1)] if p < Tg), Tg = max(L-w, T)
    const int Tg = (L - w > T) ? L - w : T;
    float ux[E], ln[E];
    if constexpr (E == 16) {
        // p0 = 16t, so pad(p0 + e + d) = 17t + (e+d) + floor((e+d)/16): a per-thread base plus an
        // offset that is uniform over the block (w is), and pad(max(q,0)) = max(pad(q),0),
        // pad(min(q,L-1)) = min(pad(q),pad(L-1)) since pad is monotone with pad(0) = 0
        const int b17 = 17 * t;
        const int pl = pad(L - 1);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int dh = e - w, dg = e + w;
            const float2 hv = H[max(b17 + dh + (dh >> 4), 0)];
            const float2 gv = G[min(b17 + dg + (dg >> 4), pl)];
            const bool useg = p0 + e < Tg;
            ux[e] = useg ? fmaxf(hv.x, gv.x) : hv.x;
            ln[e] = useg ? fminf(hv.y, gv.y) : hv.y;
        }
    } else {
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

    // ---- LB_Kim features: cross-warp part and store ------------------------------------------
    if (kim != nullptr) {
        float mn = kmn, mx = kmx;
        unsigned imn = kimn, imx = kimx;
        if (nw > 1) {
            __syncthreads();  // tot[] reuse
            float4 *red = reinterpret_cast<float4 *>(tot);
            if (lane == 0) red[wig] = make_float4(mn, __uint_as_float(imn), mx, __uint_as_float(imx));
            __syncthreads();
            if (t == 0) {
                for (int q = 1; q < nw; ++q) {
                    float4 r = red[q];
                    float omn = r.x, omx = r.z;
                    unsigned oimn = __float_as_uint(r.y), oimx = __float_as_uint(r.w);
                    if (omn < mn || (omn == mn && oimn < imn)) { mn = omn; imn = oimn; }
                    if (omx > mx || (omx == mx && oimx < imx)) { mx = omx; imx = oimx; }
                }
            }
        }
        if (t == 0 && live) {
            nndtw_kim r;
            r.vmin = mn;
            r.vmax = mx;
            r.imin = (int)imn;
            r.imax = (int)imx;
            kim[s] = r;
        }
    }
}

// ---- S1, direct form for w >= 16 ------------------------------------------
// Chunks of 16 elements, one per thread (p0 = 16t).  With w = 16q + R the window [i-w, i+w] of
// element i = 16t + e is: the suffix of chunk cl = t-q-(e<R) from i-w, the whole chunks
// cl+1 .. ch-1, and the prefix of chunk ch = t+q+(e+R>=16) up to i+w.  The middle always
// contains the core t-q+1 .. t+q-1 (2q-1 chunks, one sparse-table query), plus chunk t-q when
// e < R and chunk t+q when e+R >= 16.  So per element: two shared-memory reads (suffix, prefix)
// and a 3-input max / min with one of four per-thread middle values -- which one, and every
// shared-memory offset, is a compile-time function of (e, R) with R a template parameter.
// Positions outside [0, L) hold the identities (-inf for max, +inf for min): the series is
// padded, which is exactly the clipping of Eq. 3-4.  No segment scans, no cross-thread carries.
constexpr int ENV_DIRECT_THREADS = 256;

template <int R>
__global__ void __launch_bounds__(ENV_DIRECT_THREADS, 3)
    k_env_direct(const float *__restrict__ x, int64_t n, int L, int w, int tps, int vec, int kc,
                 float *__restrict__ U, float *__restrict__ Lo, nndtw_kim *__restrict__ kim) {
    constexpr int E = 16;
    extern __shared__ __align__(16) unsigned char env_smem[];
    const int groups = blockDim.x / tps;
    const int grp = threadIdx.x / tps;
    const int t = threadIdx.x - grp * tps;
    const int lane = threadIdx.x & 31;
    const int wig = t >> 5;
    const int nw = tps >> 5;
    const int q = w >> 4;             // w = 16q + R, q >= 1
    const int offc = q + 1;           // padding chunks on each side of the element arrays
    const int plen = (17 * (2 * offc + tps) + 1) & ~1;  // pad(q) = q + q/16; even (16 B)
    const int padc = q + 1;           // padding entries on each side of the chunk arrays
    const int zlen = tps + 2 * padc;
    const int zall = (3 * zlen + 1) & ~1;
    float4 *red = reinterpret_cast<float4 *>(env_smem) + grp * 16;  // kim, per warp
    float2 *base = reinterpret_cast<float2 *>(reinterpret_cast<float4 *>(env_smem) + groups * 16);
    float2 *P = base + (size_t)grp * 2 * plen;  // chunk prefix (max, min)
    float2 *S = P + plen;                       // chunk suffix (max, min)
    float2 *Z = base + (size_t)groups * 2 * plen + (size_t)grp * zall;  // chunk extremes
    float2 *X0 = Z + zlen, *X1 = X0 + zlen;     // sparse-table levels >= 1, ping-pong
    // input staging, two sets in flight, float4 slot i stored at swz(i): conflict-free both for
    // the coalesced side (8 consecutive slots) and for the per-thread side (slots 4t..4t+3);
    // global reads and writes stay warp-coalesced (a thread owning 64 contiguous bytes would
    // cost ~40% of HBM throughput, tools/rw_roof.cu)
    auto swz = [](int i) { return (i & ~7) | ((i & 7) ^ ((i >> 3) & 3)); };
    const int slen = 16 * tps;
    int mys[4];  // this thread's own four slots
#pragma unroll
    for (int j = 0; j < 4; ++j) mys[j] = swz(4 * t + j);
    float *XS = reinterpret_cast<float *>(base + (size_t)groups * (2 * plen + zall)) +
                (size_t)grp * 2 * slen;
    const float2 ident = make_float2(-kInf, kInf);
    // identities in the padding, once per block (data sets never write there)
    for (int j = t; j < 17 * offc; j += tps) {
        P[j] = ident;
        S[j] = ident;
        P[plen - 1 - j] = ident;
        S[plen - 1 - j] = ident;
    }
    for (int j = t; j < padc; j += tps) {
        Z[j] = X0[j] = X1[j] = ident;
        Z[zlen - 1 - j] = X0[zlen - 1 - j] = X1[zlen - 1 - j] = ident;
    }
    const int p0 = t * E;
    const int nvalid = L - p0;
    const int own = 17 * (offc + t);          // padded index of this thread's element 0
    const int sb = 17 * (offc + t - q);       // ... of chunk t-q, element 0
    const int hb = 17 * (offc + t + q);       // ... of chunk t+q, element 0
    const int64_t nsets = (n + groups - 1) / groups;
    auto stage = [&](int64_t set, int buf) {  // coalesced copies of one set into XS[buf]
        const int64_t ss = set * groups + grp;
        if (set < nsets && ss < n) {
            const float *xs = x + ss * (int64_t)L;
            float *d = XS + buf * slen;
            if (vec) {
#pragma unroll 1
                for (int f = t; 4 * f < L; f += tps) cp_async16(d + 4 * swz(f), xs + 4 * f);
            } else {
#pragma unroll 1
                for (int p = t; p < L; p += tps) cp_async4(d + 4 * swz(p >> 2) + (p & 3), xs + p);
            }
        }
        cp_async_commit();
    };
    stage(blockIdx.x, 0);
    int buf = 0;
    for (int64_t set = blockIdx.x; set < nsets; set += gridDim.x, buf ^= 1) {
        const int64_t s = set * groups + grp;
        const bool live = s < n;
        cp_async_wait_all();
        __syncthreads();  // every thread's copies of this set have landed
        float v[E];
        {
            const float4 *src = reinterpret_cast<const float4 *>(XS + buf * slen);
#pragma unroll
            for (int j = 0; j < E / 4; ++j) {
                const float4 f = src[mys[j]];  // elements past L are never read as data (nvalid)
                v[4 * j] = f.x;
                v[4 * j + 1] = f.y;
                v[4 * j + 2] = f.z;
                v[4 * j + 3] = f.w;
            }
        }
        stage(set + gridDim.x, buf ^ 1);  // next set's copies overlap this set's work

        // ---- LB_Kim, thread and warp part (reading C7) --------------------------------------
        float kmn = kInf, kmx = -kInf;
        unsigned kimn = 0x7fffffffu, kimx = 0x7fffffffu;
        // ---- chunk prefix / suffix extremes -> P, S; chunk extremes -> Z ---------------------
        float2 agg;  // this chunk's (max, min)
        if (nvalid >= E) {
            float ax = v[0], an = v[0];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                ax = fmaxf(ax, v[e]);
                an = fminf(an, v[e]);
                P[own + e] = make_float2(ax, an);
            }
            agg = make_float2(ax, an);
            kmn = an;
            kmx = ax;
            ax = an = v[E - 1];
#pragma unroll
            for (int e = E - 1; e >= 0; --e) {
                ax = fmaxf(ax, v[e]);
                an = fminf(an, v[e]);
                S[own + e] = make_float2(ax, an);
            }
        } else {  // the chunk holding L-1, and chunks past it: identities beyond L-1
            float ax = -kInf, an = kInf;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                ax = fmaxf(ax, e < nvalid ? v[e] : -kInf);
                an = fminf(an, e < nvalid ? v[e] : kInf);
                P[own + e] = make_float2(ax, an);
            }
            agg = make_float2(ax, an);
            kmn = an;
            kmx = ax;
            ax = -kInf;
            an = kInf;
#pragma unroll
            for (int e = E - 1; e >= 0; --e) {
                ax = fmaxf(ax, e < nvalid ? v[e] : -kInf);
                an = fminf(an, e < nvalid ? v[e] : kInf);
                S[own + e] = make_float2(ax, an);
            }
        }
        Z[padc + t] = agg;
        if (kim != nullptr) {
            const float tmn = kmn, tmx = kmx;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                kmn = fminf(kmn, __shfl_xor_sync(0xffffffffu, kmn, off));
                kmx = fmaxf(kmx, __shfl_xor_sync(0xffffffffu, kmx, off));
            }
            if (tmn == kmn) {
                for (int e = E - 1; e >= 0; --e)
                    if (e < nvalid && v[e] == kmn) kimn = p0 + e;
            }
            if (tmx == kmx) {
                for (int e = E - 1; e >= 0; --e)
                    if (e < nvalid && v[e] == kmx) kimx = p0 + e;
            }
            kimn = __reduce_min_sync(0xffffffffu, kimn);
            kimx = __reduce_min_sync(0xffffffffu, kimx);
            if (nw > 1 && lane == 0)
                red[wig] = make_float4(kmn, __uint_as_float(kimn), kmx, __uint_as_float(kimx));
        }
        __syncthreads();

        // ---- sparse table over chunk extremes up to level kc = floor(log2(2q-1)) -------------
        // (entry j of level k covers chunks j .. j+2^k-1, so the left padding entries are real
        // values too; the right padding stays identity at every level)
        for (int k = 1; k <= kc; ++k) {
            const float2 *src = (k == 1) ? Z : ((k & 1) ? X0 : X1);
            float2 *dst = (k & 1) ? X1 : X0;
            for (int j = t; j < padc + tps; j += tps) {
                const float2 a = src[j], b = src[j + (1 << (k - 1))];
                dst[j] = make_float2(fmaxf(a.x, b.x), fminf(a.y, b.y));
            }
            __syncthreads();
        }
        const float2 *lev = (kc == 0) ? Z : ((kc & 1) ? X1 : X0);
        const float2 ca = lev[padc + t - q + 1];
        const float2 cb = lev[padc + t + q - (1 << kc)];
        const float2 ml = Z[padc + t - q];
        const float2 mr = Z[padc + t + q];
        const float cx = fmaxf(ca.x, cb.x), cn = fminf(ca.y, cb.y);           // core
        const float lx = fmaxf(cx, ml.x), ln_ = fminf(cn, ml.y);               // + chunk t-q
        const float rx = fmaxf(cx, mr.x), rn = fminf(cn, mr.y);                // + chunk t+q
        const float bx = fmaxf(lx, mr.x), bn = fminf(ln_, mr.y);               // + both

        // ---- gather: U_i = max(suffix(i-w), middle, prefix(i+w)) ------------------------------
        float ux[E], lw[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int cs = (e - R) + ((e - R) < 0 ? -1 : 0);   // pad offset of e-R in chunk t-q
            const int cp = (e + R) + ((e + R) >= 16 ? 1 : 0);  // pad offset of e+R in chunk t+q
            const float2 sv = S[sb + cs];
            const float2 pv = P[hb + cp];
            const bool lft = e < R, rgt = e + R >= 16;
            const float mx = lft ? (rgt ? bx : lx) : (rgt ? rx : cx);
            const float mn = lft ? (rgt ? bn : ln_) : (rgt ? rn : cn);
            ux[e] = fmaxf(fmaxf(sv.x, pv.x), mx);
            lw[e] = fminf(fminf(sv.y, pv.y), mn);
        }
        // ---- out through shared memory: the data parts of P, S are free once every gather is
        // done (their identity padding must survive: the staging starts past it) -------------
        const int ds = (17 * offc + 1) & ~1;
        __syncthreads();
        {
            float4 *ou = reinterpret_cast<float4 *>(P + ds);
            float4 *ol = reinterpret_cast<float4 *>(S + ds);
#pragma unroll
            for (int j = 0; j < E / 4; ++j) {
                const int i = mys[j];
                ou[i] = make_float4(ux[4 * j], ux[4 * j + 1], ux[4 * j + 2], ux[4 * j + 3]);
                ol[i] = make_float4(lw[4 * j], lw[4 * j + 1], lw[4 * j + 2], lw[4 * j + 3]);
            }
        }
        __syncthreads();
        if (live) {
            float *Us = U + s * (int64_t)L;
            float *Ls = Lo + s * (int64_t)L;
            const float *ou = reinterpret_cast<const float *>(P + ds);
            const float *ol = reinterpret_cast<const float *>(S + ds);
            if (vec) {
#pragma unroll 1
                for (int f = t; 4 * f < L; f += tps) {
                    const int o = 4 * swz(f);
                    reinterpret_cast<float4 *>(Us)[f] = *reinterpret_cast<const float4 *>(ou + o);
                    reinterpret_cast<float4 *>(Ls)[f] = *reinterpret_cast<const float4 *>(ol + o);
                }
            } else {
#pragma unroll 1
                for (int p = t; p < L; p += tps) {
                    Us[p] = ou[4 * swz(p >> 2) + (p & 3)];
                    Ls[p] = ol[4 * swz(p >> 2) + (p & 3)];
                }
            }
        }
        if (kim != nullptr && t == 0) {
            float mn = kmn, mx = kmx;
            unsigned imn = kimn, imx = kimx;
            for (int j = 1; j < nw; ++j) {
                const float4 r = red[j];
                const unsigned oimn = __float_as_uint(r.y), oimx = __float_as_uint(r.w);
                if (r.x < mn || (r.x == mn && oimn < imn)) { mn = r.x; imn = oimn; }
                if (r.z > mx || (r.z == mx && oimx < imx)) { mx = r.z; imx = oimx; }
            }
            if (live) {
                nndtw_kim o;
                o.vmin = mn;
                o.vmax = mx;
                o.imin = (int)imn;
                o.imax = (int)imx;
                kim[s] = o;
            }
        }
        __syncthreads();  // P, S, Z, levels and red[] are rewritten by the next set
    }
}

size_t env_direct_smem(int tps, int groups, int w) {
    const int q = w >> 4;
    const size_t plen = (17 * (size_t)(2 * (q + 1) + tps) + 1) & ~(size_t)1;
    const size_t zlen = tps + 2 * (size_t)(q + 1);
    const size_t zall = (3 * zlen + 1) & ~(size_t)1;
    return (size_t)groups * ((2 * plen + zall) * sizeof(float2) + 16 * sizeof(float4) +
                             2 * 16 * (size_t)tps * sizeof(float));
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
    static const char *ed = getenv("NNDTW_ENV_DIRECT");  // experiments: 0 = van Herk only
    if (E == 16 && w >= 16 && tps <= ENV_DIRECT_THREADS && !(ed && atoi(ed) == 0)) {
        static const char *eb = getenv("NNDTW_ENV_DBLOCK");  // experiments: block size
        int dblock = eb ? atoi(eb) : 64;  // 2 series per block at L <= 512: measured best
        if (dblock < tps) dblock = tps;
        if (dblock > ENV_DIRECT_THREADS) dblock = ENV_DIRECT_THREADS;
        dblock = dblock / tps * tps;
        const int dgroups = dblock / tps;
        const size_t dsmem = env_direct_smem(tps, dgroups, w);
        if (dsmem <= 112 * 1024) {
            const int q = w >> 4;
            int kc = 0;
            while ((2 << kc) <= 2 * q - 1) ++kc;  // floor(log2(2q - 1))
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            const int64_t nsets = (n + dgroups - 1) / dgroups;
#define ENV_DIRECT(RR)                                                                             \
    case RR: {                                                                                     \
        cudaFuncSetAttribute(k_env_direct<RR>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                             (int)dsmem);                                                          \
        int occ = 1;                                                                               \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_env_direct<RR>,                     \
                                                      dblock, dsmem);                              \
        if (occ < 1) occ = 1;                                                                      \
        const int64_t g = std::min<int64_t>(nsets, (int64_t)sms * occ);                            \
        k_env_direct<RR><<<(unsigned)g, dblock, dsmem, st>>>(x, n, L, w, tps, vec, kc,             \
                                                                          U, Lo, kim);             \
    } break;
            switch (w & 15) {
                ENV_DIRECT(0) ENV_DIRECT(1) ENV_DIRECT(2) ENV_DIRECT(3)
                ENV_DIRECT(4) ENV_DIRECT(5) ENV_DIRECT(6) ENV_DIRECT(7)
                ENV_DIRECT(8) ENV_DIRECT(9) ENV_DIRECT(10) ENV_DIRECT(11)
                ENV_DIRECT(12) ENV_DIRECT(13) ENV_DIRECT(14) ENV_DIRECT(15)
            }
#undef ENV_DIRECT
            count_launch(1, __func__);
            return 0;
        }
    }
#define ENV_LAUNCH(EE)                                                                            \
    do {                                                                                          \
        if (smem > 48 * 1024)                                                                     \
            cudaFuncSetAttribute(k_envelopes<EE>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                 (int)smem);                                                      \
        k_envelopes<EE><<<(unsigned)grid, block, smem, st>>>(x, n, L, w, tps, vec, T, U, Lo, kim);    \
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
