// lb_sparse.cu -- S2 in two stages, in the cascade order of the paper: LB_Kim, then
// Algorithm 1's boundary terms and bands with the line-12 abort, then the LB_Keogh bridge
// (lines 13-15) only for the pairs that survived.
//
//   stage A  k_lb_tile in no-bridge mode (lb.cu): P = max(LB_Kim, boundary + bands) for every
//            pair, and the per-query argmin of P -> first seed; the seed's DTW (S3 seed round)
//            gives a best-so-far bsf1 per query.
//   lists    k_col_compact: the pairs with P <= bsf1*(1+eps_p) (the others are pruned: Algorithm
//            1 returns "infinity" at line 12) as per-train-series lists of queries.
//   stage B  k_lb_sparse: one warp per train series computes the full cascade value
//            max(LB_Kim, boundary + bands + bridge) for its listed queries, stores it next to
//            the list entry, and the per-query argmin of the full value -> second seed (another
//            S3 seed round).
// Afterwards every pair that can survive is listed with its full cascade value (the others have
// P > bsf1 >= the final best-so-far), so S3's compaction (k_list_compact, search.cu) keeps the
// pairs the one-stage path keeps, up to the rounding order of the bridge sum.  On config 2 the
// partial cascade leaves 7.3 % of the pairs to the O(L) bridge.
//
// B200 design.  Column lists: tiles of 32 queries x 1024 train series read the bound matrix
// coalesced (float4), count per (tile, series) in registers and reserve with one atomic per
// (tile, series) -- two passes (count, scatter) around a one-block scan; the count pass stores
// the 32-bit live mask per (tile, series), so the scatter pass reads 1/32 of the matrix's bytes.
// Sparse bridge (k_lb_sparse below): the series' envelope over the bridge columns in registers,
// the listed queries' rows streamed through a per-warp cp.async ring (the 20 MB of queries stay
// in L2), column pairs in f32x2, groups of 8 queries reduced with one transposing shuffle tree;
// then each lane finishes its own query of the 32-query batch: boundary terms and bands from the
// query's head/tail values (staged once per batch), LB_Kim, max.
#include "launchers.cuh"

namespace nndtw {

constexpr int CC_Q = 32;     // queries per column-compaction tile
constexpr int CC_N = 1024;   // train series per tile (256 threads x 4)

// PASS 0 reads the bound matrix, counts per (tile, series) and stores the tile's live bits per
// series (colmask[q-tile][n], 32 bits: 1/8 byte per pair); PASS 1 scatters from the masks
// alone, so the 4 GB matrix is streamed once, not twice.
template <int PASS>
__global__ void __launch_bounds__(256) k_col_compact(const float *__restrict__ lb, int64_t ldlb,
                                                     int64_t nq, int64_t nt,
                                                     const unsigned long long *__restrict__ key,
                                                     float eps_p, long long *col_count,
                                                     const long long *__restrict__ col_off,
                                                     long long *col_fill, int32_t *qlist,
                                                     unsigned long long qlist_cap,
                                                     unsigned *colmask) {
    const int64_t ntq = (nq + CC_Q - 1) / CC_Q, ntn = (nt + CC_N - 1) / CC_N;
    const bool vec = (ldlb & 3) == 0;
    for (int64_t tile = blockIdx.x; tile < ntq * ntn; tile += gridDim.x) {
        const int64_t tq = tile / ntn;
        const int64_t q0 = tq * CC_Q;
        const int64_t n0 = (tile % ntn) * CC_N + 4 * threadIdx.x;
        unsigned live[4] = {0u, 0u, 0u, 0u};  // bit qq: query q0+qq keeps series n0+e
        unsigned *mrow = colmask + tq * nt;
        if (PASS == 0) {
#pragma unroll 16
            for (int qq = 0; qq < CC_Q; ++qq) {  // (16 rows' loads in flight per thread)
                const int64_t q = q0 + qq;
                if (q >= nq) break;
                const float thr = key_dist(key[q]) * (1.0f + eps_p);
                const float *row = lb + q * ldlb;
                float v[4];
                if (vec && n0 + 3 < nt) {
                    const float4 f = *reinterpret_cast<const float4 *>(row + n0);
                    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[e] = n0 + e < nt ? row[n0 + e] : kInf;
                }
#pragma unroll
                for (int e = 0; e < 4; ++e)  // (NaN -- the leave-one-out self pair -- is never kept)
                    live[e] |= (n0 + e < nt && v[e] <= thr) ? (1u << qq) : 0u;
            }
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (n0 + e < nt) mrow[n0 + e] = live[e];
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) live[e] = n0 + e < nt ? mrow[n0 + e] : 0u;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int c = __popc(live[e]);
            if (c == 0) continue;
            const int64_t n = n0 + e;
            if (PASS == 0) {
                atomicAdd((unsigned long long *)(col_count + n), (unsigned long long)c);
            } else {
                long long pos = col_off[n] +
                                (long long)atomicAdd((unsigned long long *)(col_fill + n),
                                                     (unsigned long long)c);
                unsigned m = live[e];
                while (m) {
                    const int qq = __ffs(m) - 1;
                    m &= m - 1;
                    if ((unsigned long long)pos < qlist_cap) qlist[pos] = (int32_t)(q0 + qq);
                    ++pos;
                }
            }
        }
    }
}

// counts -> offsets (col_off[n] = sum of counts before n; col_off[nt] = total), fill = 0.
// A capped workspace (total > cap): the offsets are clamped to cap -- the lists past it are
// empty, so every reader stays inside the arrays -- and the overflow word is set (the call's
// answer is invalid; nndtw_classify_overflowed reports it).
__global__ void __launch_bounds__(1024) k_col_scan(const long long *count, long long *off,
                                                   long long *fill, int64_t nt,
                                                   long long cap,
                                                   unsigned long long *cap_overflow) {
    __shared__ long long part[1024];
    const int64_t per = (nt + blockDim.x - 1) / blockDim.x;
    const int64_t b = threadIdx.x * per, e = b + per < nt ? b + per : nt;
    long long s = 0;
    for (int64_t i = b; i < e; ++i) s += count[i];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long run = 0;
        for (int i = 0; i < (int)blockDim.x; ++i) {
            const long long v = part[i];
            part[i] = run;
            run += v;
        }
        off[nt] = run < cap ? run : cap;
        if (run > cap && cap_overflow) *cap_overflow = 1ull;
    }
    __syncthreads();
    long long run = part[threadIdx.x];
    for (int64_t i = b; i < e; ++i) {
        off[i] = run < cap ? run : cap;
        run += count[i];
        fill[i] = 0;
    }
}

int launch_col_compact(const float *lb, int64_t ldlb, int64_t nq, int64_t nt,
                       const unsigned long long *key, float eps_p, long long *col_count,
                       long long *col_off, long long *col_fill, int32_t *qlist,
                       unsigned long long qlist_cap, unsigned *colmask,
                       unsigned long long *cap_overflow, int num_sms, cudaStream_t st) {
    if (nq == 0 || nt == 0) return 0;
    cudaMemsetAsync(col_count, 0, sizeof(long long) * (size_t)nt, st);
    const int64_t ntiles = ((nq + CC_Q - 1) / CC_Q) * ((nt + CC_N - 1) / CC_N);
    const int64_t grid = ntiles < (int64_t)num_sms * 8 ? ntiles : (int64_t)num_sms * 8;
    k_col_compact<0><<<(unsigned)grid, 256, 0, st>>>(lb, ldlb, nq, nt, key, eps_p, col_count,
                                                     col_off, col_fill, qlist, qlist_cap,
                                                     colmask);
    k_col_scan<<<1, 1024, 0, st>>>(col_count, col_off, col_fill, nt, (long long)qlist_cap,
                                    cap_overflow);
    k_col_compact<1><<<(unsigned)grid, 256, 0, st>>>(lb, ldlb, nq, nt, key, eps_p, col_count,
                                                     col_off, col_fill, qlist, qlist_cap,
                                                     colmask);
    count_launch(3, __func__);
    return 0;
}

constexpr int SP_NBMAX = 16;  // bands per side held by lanes (2*nb - 1 <= 31 lanes)
constexpr int SP_D = 4;       // query-row ring depth (register path): D-1 rows in flight

__host__ __device__ inline int sparse_row_len(int L, int nch) {
    const int lp = (L + 127) / 128 * 128;
    return nch > 0 && 128 * nch > lp ? 128 * nch : lp;
}

// shared memory per warp (floats): NCH > 0 the query-row ring + the series' head / tail values,
// NCH == 0 the masked envelope rows + head / tail
__host__ __device__ inline int sparse_warp_floats(int L, int nch) {
    const int Lp = sparse_row_len(L, nch);
    // (NCH > 0: after a batch's bridge the ring holds the 32 queries' head / tail pairs)
    const int ring = SP_D * Lp > 32 * (2 * SP_NBMAX + 2) ? SP_D * Lp : 32 * (2 * SP_NBMAX + 2);
    return (nch > 0 ? ring : 2 * Lp) + 2 * SP_NBMAX;
}

// Batches of 32 listed queries: the warp computes each query's bridge (lanes over the columns),
// lane p keeps query p's bridge sum; then every lane finishes its own query -- Algorithm 1's
// boundary terms and bands (lines 1-11) and LB_Kim -- so that this O(V*w) tail runs once per 32
// pairs of issue slots.
// NCH > 0 (L <= 128*NCH, L % 4 == 0): the series' envelope over the bridge columns sits in
// registers (NCH float4 of U and of L per lane, band columns masked to (+inf, -inf)); the listed
// queries' rows stream through a per-warp shared-memory ring of SP_D rows by cp.async (16 B per
// lane and chunk; a lane reads back only what it copied, so no warp barrier), SP_D-1 rows in
// flight.  Groups of 8 queries: per-lane partial sums, one transposing warp reduction (10
// shuffles for 8 sums).
// NCH == 0: generic scalar path (envelope rows in shared memory, one warp sum per query).
template <int NCH>
__global__ void __launch_bounds__(256) k_lb_sparse(const float *__restrict__ q,
                                                   const nndtw_kim *__restrict__ qkim,
                                                   const float *__restrict__ t,
                                                   const float *__restrict__ U,
                                                   const float *__restrict__ Lo,
                                                   const nndtw_kim *__restrict__ tkim,
                                                   int64_t nt, int L, int w, int nb,
                                                   const long long *__restrict__ col_off,
                                                   const int32_t *__restrict__ qlist,
                                                   float *__restrict__ bval, float *lb,
                                                   int64_t ldlb, unsigned long long *minkey2) {
    extern __shared__ __align__(16) float sp_smem[];
    const int lane = threadIdx.x & 31;
    // warp index through a shuffle: provably warp-uniform loop control (plain SHFL reductions)
    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);
    const int Lp = sparse_row_len(L, NCH);
    float *wbase = sp_smem + (size_t)warp * sparse_warp_floats(L, NCH);
    float *ring = wbase;                          // NCH > 0: SP_D query rows
    float *sU = wbase, *sL = wbase + Lp;          // NCH == 0: masked envelope rows
    // the series' (t[x], t[L-1-x]) pairs, x < nb (Algorithm 1's left and right bands together)
    float2 *th2 = reinterpret_cast<float2 *>(wbase + sparse_warp_floats(L, NCH) - 2 * SP_NBMAX);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    if (NCH > 0) {  // the ring's columns past L are never copied: finite from the start
        for (int i = lane; i < sparse_warp_floats(L, NCH) - 2 * SP_NBMAX; i += 32) ring[i] = 0.0f;
        __syncwarp();
    }
    for (int64_t n = gw; n < nt; n += nw) {
        const long long beg = col_off[n], cnt = col_off[n + 1] - beg;
        if (cnt == 0) continue;
        const float *un = U + n * L, *ln = Lo + n * L, *tn = t + n * L;
        // the series' envelope over the bridge columns [nb, L-nb); other columns (+inf, -inf)
        float4 ur[NCH > 0 ? NCH : 1], lr[NCH > 0 ? NCH : 1];
        if (NCH > 0) {
#pragma unroll
            for (int h = 0; h < NCH; ++h) {
                const int c = 128 * h + 4 * lane;
                float4 u4 = make_float4(kInf, kInf, kInf, kInf);
                float4 l4 = make_float4(-kInf, -kInf, -kInf, -kInf);
                if (c < L) {
                    u4 = __ldg(reinterpret_cast<const float4 *>(un + c));
                    l4 = __ldg(reinterpret_cast<const float4 *>(ln + c));
                }
                float *uu = reinterpret_cast<float *>(&u4), *ll = reinterpret_cast<float *>(&l4);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const bool br = c + e >= nb && c + e < L - nb;
                    uu[e] = br ? uu[e] : kInf;
                    ll[e] = br ? ll[e] : -kInf;
                }
                ur[h] = u4;
                lr[h] = l4;
            }
        } else {
            for (int c = lane; c < Lp; c += 32) {
                const bool br = c >= nb && c < L - nb;
                sU[c] = br ? __ldg(un + c) : kInf;
                sL[c] = br ? __ldg(ln + c) : -kInf;
            }
        }
        if (lane < nb) th2[lane] = make_float2(__ldg(tn + lane), __ldg(tn + (L - 1 - lane)));
        const nndtw_kim kb = tkim[n];
        const float t0 = __ldg(tn), tl = __ldg(tn + L - 1);
        __syncwarp();
        for (long long kb0 = 0; kb0 < cnt; kb0 += 32) {
            const int nbatch = (int)(cnt - kb0 < 32 ? cnt - kb0 : 32);
            const int myq = lane < nbatch ? qlist[beg + kb0 + lane] : 0;  // coalesced
            float mybridge = 0.0f;
            if (NCH > 0) {
                // query row pp of the batch -> ring slot pp % SP_D (this lane's 16-byte pieces)
                static_assert(8 % SP_D == 0, "ring slots must repeat within a group of 8");
                auto issue = [&](int pp, int slot) {
                    const float *a = q + (int64_t)__shfl_sync(0xffffffffu, myq, pp) * L;
                    float *dst = ring + slot * Lp;
#pragma unroll
                    for (int h = 0; h < NCH; ++h) {
                        const int c = 128 * h + 4 * lane;
                        if (c < L) cp_async16(dst + c, a + c);
                    }
                };
#pragma unroll
                for (int pp = 0; pp < SP_D - 1; ++pp) {
                    if (pp < nbatch) issue(pp, pp);
                    cp_async_commit();
                }
                // groups of 8 queries (a 32-way unrolled body overflowed the instruction cache)
#pragma unroll 1
                for (int g = 0; g < 4; ++g) {
                    if (8 * g >= nbatch) break;
                    float part[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int pp = 8 * g + i;
                        if (pp + SP_D - 1 < nbatch) issue(pp + SP_D - 1, (i + SP_D - 1) % SP_D);
                        cp_async_commit();
                        cp_async_wait_group<SP_D - 1>();  // row pp has landed (this lane's part)
                        float acc = 0.0f;
                        if (pp < nbatch) {
                            const float *src = ring + (i % SP_D) * Lp;
                            // column pairs in f32x2: a - U and L - a as FADD2, the square-sum
                            // as FFMA2 (two accumulators, added at the end)
                            unsigned long long acc2 = 0ull;
#pragma unroll
                            for (int h = 0; h < NCH; ++h) {
                                const int c = 128 * h + 4 * lane;
                                // (columns past L: stale ring data against (+inf, -inf): 0)
                                const float4 a4 = *reinterpret_cast<const float4 *>(src + c);
                                const float4 u4 = ur[h], l4 = lr[h];
#pragma unroll
                                for (int hf = 0; hf < 2; ++hf) {
                                    const unsigned long long av =
                                        hf ? f2_pack(a4.z, a4.w) : f2_pack(a4.x, a4.y);
                                    const unsigned long long uv =
                                        hf ? f2_pack(u4.z, u4.w) : f2_pack(u4.x, u4.y);
                                    const unsigned long long lv =
                                        hf ? f2_pack(l4.z, l4.w) : f2_pack(l4.x, l4.y);
                                    float p0, p1, m0, m1;
                                    f2_unpack(f2_sub(av, uv), p0, p1);
                                    f2_unpack(f2_sub(lv, av), m0, m1);
                                    const float d0 = fmaxf(fmaxf(p0, m0), 0.0f);
                                    const float d1 = fmaxf(fmaxf(p1, m1), 0.0f);
                                    const unsigned long long dv = f2_pack(d0, d1);
                                    acc2 = f2_fma(dv, dv, acc2);
                                }
                            }
                            float s0, s1;
                            f2_unpack(acc2, s0, s1);
                            acc = s0 + s1;
                        }
                        part[i] = acc;
                    }
                    // transposing reduction over lane bits 4, 3, 2 (8 -> 1 value per lane), then
                    // a butterfly over bits 1, 0: lanes 4i .. 4i+3 hold query 8g+i's bridge
#pragma unroll
                    for (int o = 16, nv = 4; o >= 4; o >>= 1, nv >>= 1) {
                        const bool up = (lane & o) != 0;
#pragma unroll
                        for (int k = 0; k < nv; ++k) {
                            const float send = up ? part[k] : part[k + nv];
                            const float keep = up ? part[k + nv] : part[k];
                            part[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                        }
                    }
                    part[0] += __shfl_xor_sync(0xffffffffu, part[0], 2);
                    part[0] += __shfl_xor_sync(0xffffffffu, part[0], 1);
                    const float r = __shfl_sync(0xffffffffu, part[0], 4 * (lane & 7));
                    if ((lane >> 3) == g) mybridge = r;
                }
            } else {
                for (int pp = 0; pp < nbatch; ++pp) {
                    const int qi = __shfl_sync(0xffffffffu, myq, pp);
                    const float *a = q + (int64_t)qi * L;
                    float acc = 0.0f;
                    for (int c = lane; c < L; c += 32) {
                        const float av = __ldg(a + c);
                        const float d = fmaxf(fmaxf(av - sU[c], sL[c] - av), 0.0f);
                        acc = fmaf(d, d, acc);
                    }
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1)
                        acc += __shfl_xor_sync(0xffffffffu, acc, off);
                    mybridge = lane == pp ? acc : mybridge;
                }
            }
            // every lane finishes its own query: boundary terms + bands (Algorithm 1 lines 1-11,
            // the band minimum over |differences| squared once, in the tile kernel's order),
            // LB_Kim.  The left band of the series and the right band (the left band of the
            // reversed series) run together as f32x2 pairs (a[x], a[L-1-x]) - (t[y], t[L-1-y]).
            // NCH > 0: the query's pairs are first copied into the (now free) ring in one round
            // trip (read one by one from L2 they were a chain of dependent misses).
            const int s2 = (nb % 2 == 0) ? nb + 1 : nb + 2;  // pairs per lane row (odd: banks)
            if (NCH > 0) {
                __syncwarp();  // every lane's ring reads of this batch are done
                // per copy instruction 32 / (2nb) queries, 2nb lanes each (lane x < nb: a[x],
                // else a[L-1-(x-nb)]): few rows per instruction, not 32 scattered ones
                const int per = 32 / (2 * nb), k = lane / (2 * nb), x = lane % (2 * nb);
                const int side = x < nb ? 0 : 1, xx = x < nb ? x : x - nb;
                for (int p0 = 0; p0 < nbatch; p0 += per) {
                    const int p = p0 + k;
                    const int qi = __shfl_sync(0xffffffffu, myq, p & 31);
                    if (k < per && p < nbatch)
                        cp_async4(ring + 2 * (p * s2 + xx) + side,
                                  q + (int64_t)qi * L + (side ? L - 1 - xx : xx));
                }
                cp_async_commit();
                cp_async_wait_group<0>();
                __syncwarp();  // the pair rows were written by other lanes
            }
            if (lane < nbatch) {
                const float *a = q + (int64_t)myq * L;
                const float2 *hd2 = reinterpret_cast<const float2 *>(ring) + lane * s2;
                auto qa = [&](int x) {  // (a[x], a[L-1-x])
                    if (NCH > 0) {
                        const float2 v = hd2[x];
                        return f2_pack(v.x, v.y);
                    }
                    return f2_pack(__ldg(a + x), __ldg(a + (L - 1 - x)));
                };
                auto tb = [&](int x) {  // (t[x], t[L-1-x])
                    const float2 v = th2[x];
                    return f2_pack(v.x, v.y);
                };
                float a0, al;
                f2_unpack(qa(0), a0, al);
                float bands = boundary_terms(a0, al, t0, tl);
                for (int i = 1; i < nb; ++i) {
                    const unsigned long long ai = qa(i), bi = tb(i);
                    float m0, m1;
                    f2_unpack(f2_sub(ai, bi), m0, m1);
                    m0 = fabsf(m0);
                    m1 = fabsf(m1);
                    for (int jj = i - w > 0 ? i - w : 0; jj < i; ++jj) {
                        float x0, x1, y0, y1;
                        f2_unpack(f2_sub(ai, tb(jj)), x0, x1);  // a_i - b_jj
                        f2_unpack(f2_sub(qa(jj), bi), y0, y1);  // a_jj - b_i
                        m0 = fminf(m0, fminf(fabsf(x0), fabsf(y0)));
                        m1 = fminf(m1, fminf(fabsf(x1), fabsf(y1)));
                    }
                    bands = fmaf(m0, m0, bands);  // left band, then right: the tile kernel's order
                    bands = fmaf(m1, m1, bands);
                }
                const float kim = kim_sum(a0, al, t0, tl, qkim[myq], kb, L);
                const float full = fmaxf(kim, bands + mybridge);
                bval[beg + kb0 + lane] = full;  // next to its list entry (coalesced)
                if (lb) lb[(int64_t)myq * ldlb + n] = full;  // level counters only
                atomicMin(minkey2 + myq, make_key(full, (unsigned)n));
            }
            __syncwarp();  // the next batch's row copies overwrite the pair rows
        }
        __syncwarp();  // the next series overwrites th2 (and, NCH == 0, sU / sL)
    }
}

int launch_lb_sparse(const float *q, const nndtw_kim *qkim, int64_t nq, const float *t,
                     const float *U, const float *Lo, const nndtw_kim *tkim, int64_t nt, int L,
                     int w, int v, const long long *col_off, const int32_t *qlist, float *bval,
                     float *lb, int64_t ldlb, unsigned long long *minkey2, int num_sms,
                     cudaStream_t st) {
    if (nq == 0 || nt == 0) return 0;
    if (w > L - 1) w = L - 1;
    const int nb = (L / 2) < v ? (L / 2) : v;
    if (nb < 1 || nb > SP_NBMAX) return -1;  // (L = 1: the one-stage path)
    // the register path needs 16-byte rows: L % 4 == 0 and aligned q, U, L bases
    const bool vec_ = (L % 4) == 0 && ((uintptr_t)q % 16) == 0 && ((uintptr_t)U % 16) == 0 &&
                      ((uintptr_t)Lo % 16) == 0;
    const int nch = !vec_ ? 0 : L <= 128 ? 1 : L <= 256 ? 2 : L <= 512 ? 4 : L <= 1024 ? 8 : 0;
    const size_t warp_bytes = (size_t)sparse_warp_floats(L, nch) * sizeof(float);
    int warps = (int)((200 * 1024) / warp_bytes);
    if (warps < 1) warps = 1;
    if (warps > 8) warps = 8;
    const size_t smem = warps * warp_bytes;
    auto kern = k_lb_sparse<0>;
    if (nch == 1) kern = k_lb_sparse<1>;
    else if (nch == 2) kern = k_lb_sparse<2>;
    else if (nch == 4) kern = k_lb_sparse<4>;
    else if (nch == 8) kern = k_lb_sparse<8>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // persistent warps, as many as fit
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * warps, smem);
    if (occ < 1) occ = 1;
    int64_t grid = (int64_t)num_sms * occ;
    const int64_t need = (nt + warps - 1) / warps;
    if (need < grid) grid = need;
    kern<<<(unsigned)grid, 32 * warps, smem, st>>>(q, qkim, t, U, Lo, tkim, nt, L, w, nb,
                                                   col_off, qlist, bval, lb, ldlb, minkey2);
    count_launch(1, __func__);
    return 0;
}

// the second seed round's items: the argmin of the full cascade value, where it differs from the
// first round's candidates (the partial-cascade argmin and the caller's extra seed)
__global__ void k_seed_items2(const unsigned long long *minkey2, const unsigned long long *minkey1,
                              const int32_t *seed2, int64_t nq, int64_t nt, Item *items,
                              unsigned long long *count) {
    const int64_t qi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (qi >= nq) return;
    const unsigned long long k2 = minkey2[qi];
    if (k2 == kNone) return;
    const unsigned n2 = (unsigned)(k2 & 0xffffffffull);
    const unsigned n1 = (unsigned)(minkey1[qi] & 0xffffffffull);
    const unsigned s2 = seed2 ? (unsigned)seed2[qi] : 0xffffffffu;
    if (n2 >= (unsigned)nt || n2 == n1 || n2 == s2) return;
    const unsigned long long pos = atomicAdd(count, 1ull);
    items[pos] = Item{(unsigned)qi, n2, 0.0f};
}

int launch_seed_items2(const unsigned long long *minkey2, const unsigned long long *minkey1,
                       const int32_t *seed2, int64_t nq, int64_t nt, Item *items,
                       unsigned long long *count, cudaStream_t st) {
    if (nq == 0) return 0;
    k_seed_items2<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(minkey2, minkey1, seed2, nq, nt,
                                                                items, count);
    count_launch(1, __func__);
    return 0;
}

}  // namespace nndtw
