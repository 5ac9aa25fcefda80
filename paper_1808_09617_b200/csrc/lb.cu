// lb.cu -- S2: batched LB_Kim -> LB_Enhanced^V cascade over all (query, train) pairs.
//
// LB_Enhanced is Eq. 7 in the order of Algorithm 1: boundary terms
// (line 1), n_bands = min(floor(L/2), V) (line 2, reading C10), the left band L_i and the right
// band R_{L-i+1} minima for i = 2..n_bands (lines 3-11; the right band is the left band of the
// reversed series, reading C9), then the LB_Keogh bridge (lines 13-15) over columns
// n_bands+1..L-n_bands.  One stage: every pair's full bound is produced (north_star "over all
// query x train pairs"); pruning happens against the best-so-far later.  Two stages (large
// inputs, lb_sparse.cu): this kernel in no-bridge mode is stage A -- the line-12 abort is then
// taken against the first seed's best-so-far by the column lists, and the bridge runs only for
// the pairs they keep.
// LB_Kim is the sum variant "without repetitions" (reading C7).
//
// B200 design: the bridge is the O(L) part.  A CTA computes a 64-query x
// 128-train tile; each thread owns 8 queries x 4 train series (32 accumulators), so per column
// it reads 8 query values (2 broadcast LDS.128) and 4 (U,L) pairs (4 conflict-free LDS.64)
// for 32 pair-updates
//   t = max(a-U, L-a, 0);  acc += t*t   (t > 0 only when a is outside [L, U]).
// Two queries share one train column: (a_q, a_q') - (U, U) and (L, L) - (a_q, a_q') are one
// packed FADD2 each, U and L entering as broadcast scalar operands (measured: FADD2 issues
// at half rate but halves the issue slots; 9.8 -> 7.8 ms for 1000 x 100000 pairs), then
// FMNMX3 with 0 and FFMA per pair -- 3 issue slots per pair-column instead of 4, with results
// bit-identical to the scalar sequence.
// Columns are staged through shared memory in chunks of 16, double-buffered with register
// prefetch.  Grid x runs over query tiles so CTAs resident together share one train tile
// (the 400 MB of envelopes of config 2 are read once from HBM; the queries stay in L2).
#include "launchers.cuh"

namespace nndtw {

constexpr int LB_TQ = 64, LB_TN = 128, LB_CC = 16, LB_QPT = 8, LB_NPT = 4;
constexpr int LB_NBMAX = 16;
constexpr int LB_SA_STRIDE = LB_TQ + 4;   // floats (keeps 16-byte alignment of float4 reads)
constexpr int LB_SE_STRIDE = LB_TN + 1;   // float2 units (conflict-free chunk stores)

struct LbParams {
    const float *q;
    int64_t nq;
    const nndtw_kim *qkim;
    const float *t, *U, *Lo;
    const nndtw_kim *tkim;
    int64_t nt;
    int L, w, nb, with_kim;
    int keogh;  // 1: LB_Keogh over all L columns instead of LB_Enhanced
    int transposed;  // 1: q/t roles exchanged -- write lb[t-row][q-col] = max(existing, value)
                     // (second pass of the symmetric bound)
    int64_t self_offset;
    float *lb;
    int64_t ldlb;
    unsigned long long *minkey;
    // Level-count mode (stats): no bridge, no output; lb holds
    // the finished cascade values, count_key the seeded best-so-far keys.  Each pair outside
    // the seeds / self pair with cascade value > bsf*(1+count_eps) is counted at the first level
    // of the cascade that already exceeds the threshold: Kim, the
    // boundary + band part of Algorithm 1 (its line-12 abort), or the full bound with the
    // LB_Keogh bridge.  level_cnt[0..2] += those counts.
    // 1: no LB_Keogh bridge -- write max(LB_Kim, boundary + bands) (Algorithm 1 up to its
    // line-12 abort test) and its per-query argmin key: stage A of the two-stage cascade
    int no_bridge;
    const unsigned long long *count_key;
    const unsigned long long *seed_minkey;
    const int32_t *seed2;
    float count_eps;
    unsigned long long *level_cnt;
};

struct LbSmem {
    float a[2][LB_CC][LB_SA_STRIDE];
    float2 e[2][LB_CC][LB_SE_STRIDE];  // (U, L)
    // query head / tail values transposed: qh[i][r] = x_r[i], qh[NBMAX + i][r] = x_r[L-1-i] --
    // a warp's 8 queries are two broadcast LDS.128 into aligned register pairs (FADD2 operands)
    float qh[2 * LB_NBMAX][LB_TQ];
    float th[LB_TN][2 * LB_NBMAX + 1];  // odd row stride: lane-indexed reads are conflict-free
    KimF qk[LB_TQ];
    KimF tk[LB_TN];
};

template <bool SMEM_BANDS>
__global__ void __launch_bounds__(256, 2) k_lb_tile(LbParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LbSmem &S = *reinterpret_cast<LbSmem *>(smem_raw);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int tq = tid >> 5;  // warp index: queries tq*8 .. tq*8+7 of the tile
    const int64_t q0 = (int64_t)blockIdx.x * LB_TQ;
    const int64_t n0 = (int64_t)blockIdx.y * LB_TN;
    const int L = p.L, w = p.w;
    // bands use nb; the bridge covers [nbb, L - nbb): all columns for LB_Keogh
    const int nb = p.nb, nbb = p.keogh ? 0 : p.nb;

    // ---- stage band values and Kim features -------------------------------------------
    if (SMEM_BANDS) {
        for (int e = tid; e < LB_TQ * nb; e += 256) {
            int r = e / nb, i = e % nb;
            int64_t qq = q0 + r;
            const float *src = p.q + (qq < p.nq ? qq : 0) * (int64_t)L;
            S.qh[i][r] = src[i];
            S.qh[LB_NBMAX + i][r] = src[L - 1 - i];
        }
        for (int e = tid; e < LB_TN * nb; e += 256) {
            int r = e / nb, i = e % nb;
            int64_t nn = n0 + r;
            const float *src = p.t + (nn < p.nt ? nn : 0) * (int64_t)L;
            S.th[r][i] = src[i];
            S.th[r][LB_NBMAX + i] = src[L - 1 - i];
        }
    }
    if (p.with_kim) {
        for (int e = tid; e < LB_TQ; e += 256) {
            int64_t qq = q0 + e;
            S.qk[e] = kim_f(p.qkim[qq < p.nq ? qq : 0], L);
        }
        for (int e = tid; e < LB_TN; e += 256) {
            int64_t nn = n0 + e;
            S.tk[e] = kim_f(p.tkim[nn < p.nt ? nn : 0], L);
        }
    }

    // ---- column-chunk loader (register prefetch) ------------------------------------------
    const int ch_begin = nbb / LB_CC;
    const int ch_end = (p.count_key || p.no_bridge) ? ch_begin
                                                    : (L - nbb + LB_CC - 1) / LB_CC;  // exclusive
    float ra[4];
    float2 re[8];
    // load slot k of this thread: tile row (tid >> 4) + 16k, column c0 + (tid & 15) -- the same
    // column for every k, so the column test is one per chunk; row pointers are hoisted and
    // full tiles skip the row tests
    const int lr = tid >> 4, lc = tid & 15;
    const bool qfull = q0 + LB_TQ <= p.nq, nfull = n0 + LB_TN <= p.nt;
    const int64_t rs16 = 16 * (int64_t)L;
    const float *qrow = p.q + (q0 + lr < p.nq ? q0 + lr : 0) * (int64_t)L + lc;
    const int64_t erow = (n0 + lr < p.nt ? n0 + lr : 0) * (int64_t)L + lc;
    const float *urow = p.U + erow, *lrow = p.Lo + erow;
    auto load_chunk = [&](int ch) {
        const int c0 = ch * LB_CC;
        const bool cok = c0 + lc >= nbb && c0 + lc < L - nbb;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const bool ok = cok && (qfull || q0 + lr + 16 * k < p.nq);
            ra[k] = ok ? __ldg(qrow + k * rs16 + c0) : 0.0f;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const bool ok = cok && (nfull || n0 + lr + 16 * k < p.nt);
            re[k] = ok ? make_float2(__ldg(urow + k * rs16 + c0), __ldg(lrow + k * rs16 + c0))
                       : make_float2(kInf, -kInf);
        }
    };
    auto store_chunk = [&](int buf) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            int e = tid + 256 * k;
            S.a[buf][e & 15][e >> 4] = ra[k];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            int e = tid + 256 * k;
            S.e[buf][e & 15][e >> 4] = re[k];
        }
    };

    if (ch_begin < ch_end) {
        load_chunk(ch_begin);
        store_chunk(0);
    }
    __syncthreads();

    // ---- boundary terms + bands (Alg. 1 lines 1-11) --------------------------------------
    float acc[LB_QPT][LB_NPT];
    auto qhv = [&](int qi, int i) -> float {   // head value x[i] of query tq*8+qi
        if (SMEM_BANDS) return S.qh[i][tq * LB_QPT + qi];
        int64_t qq = q0 + tq * LB_QPT + qi;
        return __ldg(p.q + (qq < p.nq ? qq : 0) * (int64_t)L + i);
    };
    auto qtv = [&](int qi, int i) -> float {   // tail value x[L-1-i]
        if (SMEM_BANDS) return S.qh[LB_NBMAX + i][tq * LB_QPT + qi];
        int64_t qq = q0 + tq * LB_QPT + qi;
        return __ldg(p.q + (qq < p.nq ? qq : 0) * (int64_t)L + (L - 1 - i));
    };
    auto thv = [&](int j, int i) -> float {
        if (SMEM_BANDS) return S.th[lane + 32 * j][i];
        int64_t nn = n0 + lane + 32 * j;
        return __ldg(p.t + (nn < p.nt ? nn : 0) * (int64_t)L + i);
    };
    auto ttv = [&](int j, int i) -> float {
        if (SMEM_BANDS) return S.th[lane + 32 * j][LB_NBMAX + i];
        int64_t nn = n0 + lane + 32 * j;
        return __ldg(p.t + (nn < p.nt ? nn : 0) * (int64_t)L + (L - 1 - i));
    };
#pragma unroll
    for (int qi = 0; qi < LB_QPT; ++qi)
#pragma unroll
        for (int j = 0; j < LB_NPT; ++j)
            acc[qi][j] = p.keogh ? 0.0f : boundary_terms(qhv(qi, 0), qtv(qi, 0), thv(j, 0),
                                                          ttv(j, 0));

    // 8 query values (side 0: x[i], side 1: x[L-1-i]) as four f32x2 pairs (queries 2k, 2k+1)
    auto q8 = [&](int side, int i, unsigned long long (&v)[LB_QPT / 2]) {
        if (SMEM_BANDS) {
            const float *r = &S.qh[side * LB_NBMAX + i][tq * LB_QPT];
            const float4 x0 = *reinterpret_cast<const float4 *>(r);
            const float4 x1 = *reinterpret_cast<const float4 *>(r + 4);
            v[0] = f2_pack(x0.x, x0.y); v[1] = f2_pack(x0.z, x0.w);
            v[2] = f2_pack(x1.x, x1.y); v[3] = f2_pack(x1.z, x1.w);
        } else {
#pragma unroll
            for (int k = 0; k < LB_QPT / 2; ++k)
                v[k] = side ? f2_pack(qtv(2 * k, i), qtv(2 * k + 1, i))
                            : f2_pack(qhv(2 * k, i), qhv(2 * k + 1, i));
        }
    };
    for (int i = 1; i < (p.keogh ? 0 : nb); ++i) {
        const int jlo = i - w > 0 ? i - w : 0;
#pragma unroll
        for (int side = 0; side < 2; ++side) {
            float m[LB_QPT][LB_NPT];
            unsigned long long ai[LB_QPT / 2];
            float bi[LB_NPT];
            q8(side, i, ai);
#pragma unroll
            for (int j = 0; j < LB_NPT; ++j) bi[j] = side ? ttv(j, i) : thv(j, i);
            // min over the band of (x-y)^2 = (min |x-y|)^2 exactly (rounding is monotone in
            // |x-y|): the band minimum runs on |differences| (FMNMX3 with |.| operands, ALU pipe)
            // and squares once; the differences of two queries against one train value are one
            // FADD2 (bit-identical to two FADDs).  The cell (i, i) joins the first band step's
            // FMNMX3 (its |.| is then an operand modifier, not an instruction).
            auto band_step = [&](int jj, bool first) {
                unsigned long long aj[LB_QPT / 2];
                float bj[LB_NPT];
                q8(side, jj, aj);
#pragma unroll
                for (int j = 0; j < LB_NPT; ++j) bj[j] = side ? ttv(j, jj) : thv(j, jj);
#pragma unroll
                for (int qp = 0; qp < LB_QPT / 2; ++qp)
#pragma unroll
                    for (int j = 0; j < LB_NPT; ++j) {
                        float x0, x1, y0, y1;
                        f2_unpack(f2_sub(ai[qp], f2_pack(bj[j], bj[j])), x0, x1);  // a_i - b_jj
                        f2_unpack(f2_sub(aj[qp], f2_pack(bi[j], bi[j])), y0, y1);  // a_jj - b_i
                        if (first) {
                            float d0, d1;
                            f2_unpack(f2_sub(ai[qp], f2_pack(bi[j], bi[j])), d0, d1);  // a_i - b_i
                            m[2 * qp][j] = fminf(fabsf(d0), fminf(fabsf(x0), fabsf(y0)));
                            m[2 * qp + 1][j] = fminf(fabsf(d1), fminf(fabsf(x1), fabsf(y1)));
                        } else {
                            m[2 * qp][j] = fminf(m[2 * qp][j], fminf(fabsf(x0), fabsf(y0)));
                            m[2 * qp + 1][j] =
                                fminf(m[2 * qp + 1][j], fminf(fabsf(x1), fabsf(y1)));
                        }
                    }
            };
            if (jlo < i) {
                band_step(i - 1, true);
                for (int jj = jlo; jj < i - 1; ++jj) band_step(jj, false);
            } else {  // w = 0: the band is the cell (i, i) alone
#pragma unroll
                for (int qp = 0; qp < LB_QPT / 2; ++qp)
#pragma unroll
                    for (int j = 0; j < LB_NPT; ++j) {
                        float d0, d1;
                        f2_unpack(f2_sub(ai[qp], f2_pack(bi[j], bi[j])), d0, d1);
                        m[2 * qp][j] = fabsf(d0);
                        m[2 * qp + 1][j] = fabsf(d1);
                    }
            }
#pragma unroll
            for (int qi = 0; qi < LB_QPT; ++qi)
#pragma unroll
                for (int j = 0; j < LB_NPT; ++j)  // band term: m^2 added with one rounding
                    acc[qi][j] = fmaf(m[qi][j], m[qi][j], acc[qi][j]);
        }
    }

    // ---- LB_Keogh bridge (Alg. 1 lines 13-15) ---------------------------------------------
    for (int ch = ch_begin; ch < ch_end; ++ch) {
        const int buf = (ch - ch_begin) & 1;
        const bool more = ch + 1 < ch_end;
        if (more) load_chunk(ch + 1);
#pragma unroll
        for (int c = 0; c < LB_CC; ++c) {
            const float4 a0 = *reinterpret_cast<const float4 *>(&S.a[buf][c][tq * LB_QPT]);
            const float4 a1 = *reinterpret_cast<const float4 *>(&S.a[buf][c][tq * LB_QPT + 4]);
#ifdef NNDTW_LB_SCALAR
            const float av[LB_QPT] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
            for (int j = 0; j < LB_NPT; ++j) {
                const float2 e2 = S.e[buf][c][lane + 32 * j];
#pragma unroll
                for (int qi = 0; qi < LB_QPT; ++qi) {
                    float t = fmaxf(fmaxf(av[qi] - e2.x, e2.y - av[qi]), 0.0f);
                    acc[qi][j] = fmaf(t, t, acc[qi][j]);
                }
            }
#else
            const unsigned long long ap[LB_QPT / 2] = {f2_pack(a0.x, a0.y), f2_pack(a0.z, a0.w),
                                                       f2_pack(a1.x, a1.y), f2_pack(a1.z, a1.w)};
#pragma unroll
            for (int j = 0; j < LB_NPT; ++j) {
                const float2 e2 = S.e[buf][c][lane + 32 * j];
                // (U, U) and (L, L): FADD2 takes a broadcast scalar operand (no register copy)
                const unsigned long long uu = f2_pack(e2.x, e2.x), ll = f2_pack(e2.y, e2.y);
#pragma unroll
                for (int qp = 0; qp < LB_QPT / 2; ++qp) {
                    float u0, u1, l0, l1;
                    f2_unpack(f2_sub(ap[qp], uu), u0, u1);  // a - U   (two queries)
                    f2_unpack(f2_sub(ll, ap[qp]), l0, l1);  // L - a
                    const float t0 = fmaxf(fmaxf(u0, l0), 0.0f);
                    const float t1 = fmaxf(fmaxf(u1, l1), 0.0f);
                    // (FFMA2 here measured no faster: same FMA-pipe cycles)
                    acc[2 * qp][j] = fmaf(t0, t0, acc[2 * qp][j]);
                    acc[2 * qp + 1][j] = fmaf(t1, t1, acc[2 * qp + 1][j]);
                }
            }
#endif
        }
        if (more) store_chunk(buf ^ 1);
        __syncthreads();
    }

    if (p.count_key) {  // level-count mode (see LbParams)
        unsigned long long c0 = 0, c1 = 0, c2 = 0;
#pragma unroll
        for (int qi = 0; qi < LB_QPT; ++qi) {
            const int rq = tq * LB_QPT + qi;
            const int64_t qq = q0 + rq;
            const bool qok = qq < p.nq;
            const float thr = qok ? key_dist(p.count_key[qq]) * (1.0f + p.count_eps) : 0.0f;
            const unsigned s1 = qok ? (unsigned)(p.seed_minkey[qq] & 0xffffffffull) : 0u;
            const unsigned s2 = (qok && p.seed2) ? (unsigned)p.seed2[qq] : 0xffffffffu;
#pragma unroll
            for (int j = 0; j < LB_NPT; ++j) {
                const int rn = lane + 32 * j;
                const int64_t nn = n0 + rn;
                if (!qok || nn >= p.nt || (p.self_offset >= 0 && nn == qq + p.self_offset) ||
                    (unsigned)nn == s1 || (unsigned)nn == s2)
                    continue;
                const float full = p.lb[qq * p.ldlb + nn];
                const float kim = p.with_kim ? kim_sum_f(qhv(qi, 0), qtv(qi, 0), thv(j, 0),
                                                         ttv(j, 0), S.qk[rq], S.tk[rn])
                                             : 0.0f;
                if (kim > thr) c0 += 1;
                else if (full > thr) {
                    if (acc[qi][j] > thr) c1 += 1;
                    else c2 += 1;
                }
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            c0 += __shfl_xor_sync(0xffffffffu, c0, off);
            c1 += __shfl_xor_sync(0xffffffffu, c1, off);
            c2 += __shfl_xor_sync(0xffffffffu, c2, off);
        }
        if (lane == 0) {
            if (c0) atomicAdd(p.level_cnt + 0, c0);
            if (c1) atomicAdd(p.level_cnt + 1, c1);
            if (c2) atomicAdd(p.level_cnt + 2, c2);
        }
        return;
    }

    // ---- Kim cascade, self exclusion, output, per-query argmin key --------------------------
#pragma unroll
    for (int qi = 0; qi < LB_QPT; ++qi) {
        const int rq = tq * LB_QPT + qi;
        const int64_t qq = q0 + rq;
        unsigned long long best = kNone;
#pragma unroll
        for (int j = 0; j < LB_NPT; ++j) {
            const int rn = lane + 32 * j;
            const int64_t nn = n0 + rn;
            float v = acc[qi][j];
            if (p.with_kim)
                v = fmaxf(v, kim_sum_f(qhv(qi, 0), qtv(qi, 0), thv(j, 0), ttv(j, 0), S.qk[rq],
                                       S.tk[rn]));
            if (p.transposed) {
                if (qq < p.nq && nn < p.nt) {
                    float *dst = p.lb + nn * p.ldlb + qq;
                    *dst = fmaxf(*dst, v);
                }
                continue;
            }
            // the leave-one-out self pair: NaN (fails every "lb <= threshold" test, so it is never
            // compacted nor re-ranked) and never the argmin seed
            const bool self = p.self_offset >= 0 && nn == qq + p.self_offset;
            if (self) v = __int_as_float(0x7fffffff);
            if (qq < p.nq && nn < p.nt) {
                p.lb[qq * p.ldlb + nn] = v;
                unsigned long long k = make_key(v, (unsigned)nn);
                if (!self) best = k < best ? k : best;
            }
        }
        if (p.minkey != nullptr) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                unsigned long long o = __shfl_xor_sync(0xffffffffu, best, off);
                best = o < best ? o : best;
            }
            if (lane == 0 && qq < p.nq && best != kNone) atomicMin(p.minkey + qq, best);
        }
    }
}

static int launch_lb_params(LbParams &p, cudaStream_t st);

int launch_lb(const float *q, int64_t nq, const nndtw_kim *qkim, const float *t,
              const float *U, const float *Lo, const nndtw_kim *tkim, int64_t nt, int L, int w,
              int v, int with_kim, int64_t self_offset, float *lb, int64_t ldlb,
              unsigned long long *minkey, cudaStream_t st, int keogh, int transposed,
              int no_bridge) {
    if (nq == 0 || nt == 0) return 0;
    if (w > L - 1) w = L - 1;
    LbParams p;
    p.no_bridge = no_bridge;
    p.q = q;
    p.nq = nq;
    p.qkim = qkim;
    p.t = t;
    p.U = U;
    p.Lo = Lo;
    p.tkim = tkim;
    p.nt = nt;
    p.L = L;
    p.w = w;
    p.nb = (L / 2) < v ? (L / 2) : v;
    p.with_kim = with_kim;
    p.keogh = keogh;
    p.transposed = transposed;
    if (transposed) {
        with_kim = 0;
        p.with_kim = 0;
        minkey = nullptr;
    }
    p.self_offset = self_offset;
    p.lb = lb;
    p.ldlb = ldlb;
    p.minkey = minkey;
    p.count_key = nullptr;
    p.seed_minkey = nullptr;
    p.seed2 = nullptr;
    p.count_eps = 0.0f;
    p.level_cnt = nullptr;
    return launch_lb_params(p, st);
}

int launch_lb_level_counts(const float *q, int64_t nq, const nndtw_kim *qkim, const float *t,
                           const nndtw_kim *tkim, int64_t nt, int L, int w, int v, int with_kim,
                           int keogh, int64_t self_offset, const float *lb, int64_t ldlb,
                           const unsigned long long *key, const unsigned long long *minkey,
                           const int32_t *seed2, float eps_p, unsigned long long *level_cnt,
                           cudaStream_t st) {
    if (nq == 0 || nt == 0) return 0;
    if (w > L - 1) w = L - 1;
    LbParams p;
    p.no_bridge = 0;
    p.q = q;
    p.nq = nq;
    p.qkim = qkim;
    p.t = t;
    p.U = nullptr;
    p.Lo = nullptr;
    p.tkim = tkim;
    p.nt = nt;
    p.L = L;
    p.w = w;
    p.nb = (L / 2) < v ? (L / 2) : v;
    p.with_kim = with_kim;
    p.keogh = keogh;
    p.transposed = 0;
    p.self_offset = self_offset;
    p.lb = const_cast<float *>(lb);
    p.ldlb = ldlb;
    p.minkey = nullptr;
    p.count_key = key;
    p.seed_minkey = minkey;
    p.seed2 = seed2;
    p.count_eps = eps_p;
    p.level_cnt = level_cnt;
    return launch_lb_params(p, st);
}

static int launch_lb_params(LbParams &p, cudaStream_t st) {
    const int64_t nq = p.nq, nt = p.nt;
    dim3 grid((unsigned)((nq + LB_TQ - 1) / LB_TQ), (unsigned)((nt + LB_TN - 1) / LB_TN));
    if (grid.y > 65535u) return -1;
    size_t smem = sizeof(LbSmem);
    if (p.nb <= LB_NBMAX) {
        cudaFuncSetAttribute(k_lb_tile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        k_lb_tile<true><<<grid, 256, smem, st>>>(p);
    } else {
        cudaFuncSetAttribute(k_lb_tile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        k_lb_tile<false><<<grid, 256, smem, st>>>(p);
    }
    count_launch(1, __func__);
    return 0;
}

}  // namespace nndtw
