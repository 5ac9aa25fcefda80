// ed_seed.cu -- a first seed for every query from the paper's own candidate order: the train
// series nearest in Euclidean distance (P:567-570 -- the sequential search visits candidates in
// ED order; DTW_0 = ED).  Any candidate's exact DTW is a valid best-so-far, so the seed
// only has to be good, not exact: its DTW on config 2 is 1.34x the final NN distance on average,
// against 2.73x for the argmin of the partial cascade value (tools/seed_study.py), which shortens
// the two-stage S2's lists and starts the survivor round closer to its end point.
//
// All-pairs ED is a dense contraction: ED(q, t) = |q|^2 + |t|^2 - 2 q.t, so the work is the GEMM
// Q T^T (nq x nt x L) on the 5th-generation tensor cores, in bf16 with fp32 accumulation, and
// the per-query argmin is fused into the epilogue -- the nq x nt scores never reach memory.
//
// B200 design (k_ed_argmin).  A CTA owns 128 queries (UMMA M = 128): their bf16 PAA rows, K-major,
// sit in shared memory for the whole unit (<= 2 K-chunks x 16 KB, the 128-byte-swizzled canonical
// layout), and it sweeps a range of train tiles of 256 series (UMMA N = 256): per tile the
// K-chunks of the train rows arrive by bulk copies (pre-swizzled images, one cp.async.bulk per
// 32 KB chunk on an mbarrier) into a six-stage ring; one elected thread issues tcgen05.mma
// (kind::f16, 4 x K = 16 per chunk) into one of two 128 x 256 fp32 accumulators in TMEM and
// commits each chunk to its stage's mbarrier (which frees the stage); four epilogue warps read
// their 32 TMEM lanes (tcgen05.ld 32x32b) and update a per-row running argmin of |t|^2 - 2 q.t
// while the next tile accumulates.  One atomicMin per query and unit at the end.
#include "launchers.cuh"

#include <cuda_bf16.h>

namespace nndtw {

constexpr int ED_M = 128, ED_N = 256, ED_KC = 64;  // bf16 per K-chunk row: 128 bytes
constexpr int ED_A_CHUNK = ED_M * ED_KC * 2;       // 16 KB
constexpr int ED_B_CHUNK = ED_N * ED_KC * 2;       // 32 KB
constexpr int ED_MAX_LK = 128;                     // PAA length cap: A resident in 32 KB
constexpr int ED_STAGES = 6;                       // B ring: 6 x 32 KB (with A: 224 KB)

// The seed is chosen on piecewise-aggregate approximations (means over f consecutive points,
// f the smallest power of two with ceil(L / f) <= 128): on config 2 (f = 4) the PAA-ED argmin's
// DTW is 1.336x the final distance, the full ED argmin's 1.341x (tools/seed_study.py) -- the
// seed quality is the same at a quarter of the bytes and MMA work.
__host__ __device__ inline int ed_f(int L) {
    int f = 1;
    while ((L + f - 1) / f > ED_MAX_LK) f <<= 1;
    return f;
}
__host__ __device__ inline int ed_lk(int L) {
    const int f = ed_f(L), Lr = (L + f - 1) / f;
    return (Lr + ED_KC - 1) / ED_KC * ED_KC;
}

// Rows to their PAA (means over f points; the last segment zero-padded) in bf16, in the operand
// image the tensor cores read: per tile of `rows` rows and K-chunk of 64 columns a contiguous
// block, row r at (r / 8) * 1024 + (r % 8) * 128 bytes, its 16-byte chunk c at c ^ (r % 8) (the
// 128-byte swizzle), so every block is one bulk copy into shared memory.  Rows past n and columns
// past the PAA length are zero.  |PAA|^2 in fp32.
__global__ void k_ed_prep(const float *__restrict__ x, int64_t n, int L, int f, int Lk, int rows,
                          __nv_bfloat16 *__restrict__ img, float *__restrict__ norm) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int nkc = Lk / ED_KC;
    const int64_t nrows = (n + rows - 1) / rows * rows;
    for (int64_t r = wid; r < nrows; r += nw) {
        const int64_t tile = r / rows;
        const int rr = (int)(r - tile * rows);
        uint8_t *base = reinterpret_cast<uint8_t *>(img) + tile * (int64_t)nkc * rows * 128 +
                        (rr >> 3) * 1024 + (rr & 7) * 128;
        float s = 0.0f;
        for (int c = lane; c < Lk; c += 32) {
            float v = 0.0f;
            if (r < n)
                for (int e = 0; e < f; ++e) v += (c * f + e < L) ? x[r * L + c * f + e] : 0.0f;
            v *= 1.0f / (float)f;
            s = fmaf(v, v, s);
            const int kc = c / ED_KC, kk = c % ED_KC, ch = kk >> 3, e = kk & 7;
            __nv_bfloat16 *dst = reinterpret_cast<__nv_bfloat16 *>(
                base + (int64_t)kc * rows * 128 + ((ch ^ (rr & 7)) << 4) + e * 2);
            *dst = __float2bfloat16_rn(v);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0 && r < n) norm[r] = s;
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// K-major, 128-byte-swizzled canonical UMMA operand: rows of 128 bytes, 8-row groups 1024 bytes
// apart (SBO), 16-byte chunk c of row r stored at chunk c ^ (r % 8)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFFu);   // start address (16-byte units)
    d |= (uint64_t)1 << 16;                   // leading byte offset (unused when swizzled)
    d |= (uint64_t)(1024 >> 4) << 32;         // stride byte offset: 8-row groups
    d |= (uint64_t)1 << 46;                   // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                   // layout: SWIZZLE_128B
    return d;
}

__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// one bulk copy global -> shared, completing `bytes` on the mbarrier (armed by expect_tx)
__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes,
                                          uint32_t bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
        : "memory");
}

// Warp-specialised: warp 4 (one elected lane) loads and issues the MMAs, warps 0-3 run the
// epilogue on their TMEM lane quarters.  Two 256-column accumulators (all 512 TMEM columns): the
// epilogue of one tile overlaps the MMAs of the next.  Work unit = (128-query block, range of
// train tiles); the query block's operand image (nkc x 16 KB) is one bulk copy per unit.
__global__ void __launch_bounds__(160, 1)
    k_ed_argmin(const __nv_bfloat16 *__restrict__ qimg, const __nv_bfloat16 *__restrict__ timg,
                const float *__restrict__ qn, const float *__restrict__ tn, int64_t nq,
                int64_t nt, int Lk, int nsplit, unsigned long long *key) {
    extern __shared__ __align__(1024) uint8_t ed_smem[];
    const int tid = threadIdx.x, lane = tid & 31;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
    const int nkc = Lk / ED_KC;
    // 1024-byte aligned base (the 128-byte swizzle pattern repeats every 1024 bytes)
    uint8_t *smA = ed_smem + ((1024u - (smem_u32(ed_smem) & 1023u)) & 1023u);
    uint8_t *smB = smA + nkc * ED_A_CHUNK;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smB + ED_STAGES * ED_B_CHUNK);
    // bars: full[S], empty[S], afull[2], aempty[2], abar
    uint32_t *tslot = reinterpret_cast<uint32_t *>(bars + 2 * ED_STAGES + 5);
    const uint32_t b_full = smem_u32(bars), b_empty = b_full + 8 * ED_STAGES;
    const uint32_t b_afull = b_empty + 8 * ED_STAGES, b_aempty = b_afull + 16;
    const uint32_t b_a = b_aempty + 16;
    if (tid == 0) {
        for (int i = 0; i < ED_STAGES; ++i) {
            mbar_init(b_full + 8 * i, 1);
            mbar_init(b_empty + 8 * i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(b_afull + 8 * i, 1);
            mbar_init(b_aempty + 8 * i, 128);
        }
        mbar_init(b_a, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tslot)),
                     "n"(2 * ED_N)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t taddr = *tslot;

    const int64_t nmb = (nq + ED_M - 1) / ED_M;
    const int64_t ntile = (nt + ED_N - 1) / ED_N;
    const int64_t units = nmb * nsplit;

    if (warp == 4) {
        if (lane == 0) {
            // ---- producer + MMA issuer -------------------------------------------------------
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) |
                                   ((uint32_t)(ED_N >> 3) << 17) | ((uint32_t)(ED_M >> 4) << 24);
            const uint32_t aA = smem_u32(smA), aB = smem_u32(smB);
            uint32_t ph_full[ED_STAGES], ph_empty[ED_STAGES];
            bool used[ED_STAGES];
            for (int i = 0; i < ED_STAGES; ++i) {
                ph_full[i] = ph_empty[i] = 0u;
                used[i] = false;
            }
            uint32_t ph_aempty[2] = {0u, 0u}, ph_a = 0u;
            bool aused[2] = {false, false};
            int buf = 0;
            uint64_t gload = 0, gcons = 0;  // chunk counters (load / consume)
            bool a_pending = false;
            for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
                const int64_t mb = u / nsplit;
                const int sp = (int)(u % nsplit);
                const int64_t t_beg = ntile * sp / nsplit, t_end = ntile * (sp + 1) / nsplit;
                if (t_beg >= t_end) continue;
                // A: every MMA of the previous unit must be done reading it
                if (a_pending) {
                    for (int st = 0; st < ED_STAGES; ++st)
                        if (used[st]) {
                            mbar_wait(b_empty + 8 * st, ph_empty[st]);
                            ph_empty[st] ^= 1u;
                            used[st] = false;
                        }
                }
                bulk_load(aA, qimg + mb * (int64_t)nkc * ED_M * ED_KC,
                          (uint32_t)(nkc * ED_A_CHUNK), b_a);
                a_pending = true;
                const int64_t nchunks = (t_end - t_beg) * nkc;
                auto load_chunk = [&](int64_t c) {  // chunk c of this unit -> its ring stage
                    const int st = (int)(gload % ED_STAGES);
                    if (used[st]) {  // the MMAs that read this stage before are done
                        mbar_wait(b_empty + 8 * st, ph_empty[st]);
                        ph_empty[st] ^= 1u;
                    }
                    const int64_t tile = t_beg + c / nkc;
                    const int kc = (int)(c % nkc);
                    bulk_load(aB + st * ED_B_CHUNK,
                              timg + (tile * nkc + kc) * (int64_t)ED_N * ED_KC,
                              (uint32_t)ED_B_CHUNK, b_full + 8 * st);
                    used[st] = true;
                    ++gload;
                };
                const int64_t pre = nchunks < ED_STAGES - 1 ? nchunks : ED_STAGES - 1;
                for (int64_t c = 0; c < pre; ++c) load_chunk(c);
                mbar_wait(b_a, ph_a);
                ph_a ^= 1u;
                for (int64_t c = 0; c < nchunks; ++c) {
                    const int st = (int)(gcons % ED_STAGES);
                    const int kc = (int)(c % nkc);
                    if (kc == 0 && aused[buf]) {  // the epilogue is done with this accumulator
                        mbar_wait(b_aempty + 8 * buf, ph_aempty[buf]);
                        ph_aempty[buf] ^= 1u;
                    }
                    mbar_wait(b_full + 8 * st, ph_full[st]);
                    ph_full[st] ^= 1u;
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t dtm = taddr + (uint32_t)(buf * ED_N);
#pragma unroll
                    for (int k = 0; k < ED_KC / 16; ++k) {
                        const uint64_t da = umma_desc_sw128(aA + kc * ED_A_CHUNK + k * 32);
                        const uint64_t db = umma_desc_sw128(aB + st * ED_B_CHUNK + k * 32);
                        const uint32_t acc = (kc | k) != 0 ? 1u : 0u;
                        asm volatile(
                            "{\n\t.reg .pred p;\n\t"
                            "setp.ne.b32 p, %4, 0;\n\t"
                            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(
                                dtm),
                            "l"(da), "l"(db), "r"(idesc), "r"(acc)
                            : "memory");
                    }
                    umma_commit(b_empty + 8 * st);  // frees the stage when these MMAs finish
                    ++gcons;
                    if (kc == nkc - 1) {            // tile complete -> its accumulator is ready
                        umma_commit(b_afull + 8 * buf);
                        aused[buf] = true;
                        buf ^= 1;
                    }
                    if (c + ED_STAGES - 1 < nchunks) load_chunk(c + ED_STAGES - 1);
                }
            }
        }
    } else {
        // ---- epilogue: warps 0-3, TMEM lanes 32w .. 32w+31 = this thread's query -------------
        uint32_t ph_afull[2] = {0u, 0u};
        int buf = 0;
        for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
            const int64_t mb = u / nsplit;
            const int sp = (int)(u % nsplit);
            const int64_t t_beg = ntile * sp / nsplit, t_end = ntile * (sp + 1) / nsplit;
            if (t_beg >= t_end) continue;
            const int64_t row = mb * ED_M + 32 * warp + lane;
            const float qrow = row < nq ? qn[row] : 0.0f;
            float bestv = kInf;
            int64_t besti = -1;
            for (int64_t tt = t_beg; tt < t_end; ++tt) {
                mbar_wait(b_afull + 8 * buf, ph_afull[buf]);
                ph_afull[buf] ^= 1u;
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const int64_t n0 = tt * ED_N;
                // 4 blocks of 64 columns: the block's |t|^2 (16 float4, the same addresses for
                // every lane: L1 broadcasts) and accumulator columns (4 x tcgen05.ld x16) are all
                // requested before the first compare -- one latency per block, not per column
#pragma unroll 1
                for (int blk = 0; blk < ED_N / 64; ++blk) {
                    const int64_t nb0 = n0 + blk * 64;
                    float tv[64];
                    const float4 *tp = reinterpret_cast<const float4 *>(tn + nb0);
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float4 f = __ldg(tp + k);
                        tv[4 * k] = f.x; tv[4 * k + 1] = f.y; tv[4 * k + 2] = f.z; tv[4 * k + 3] = f.w;
                    }
                    uint32_t v[64];
#pragma unroll
                    for (int cb = 0; cb < 4; ++cb)
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, "
                            "%7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
                            : "=r"(v[16 * cb + 0]), "=r"(v[16 * cb + 1]), "=r"(v[16 * cb + 2]),
                              "=r"(v[16 * cb + 3]), "=r"(v[16 * cb + 4]), "=r"(v[16 * cb + 5]),
                              "=r"(v[16 * cb + 6]), "=r"(v[16 * cb + 7]), "=r"(v[16 * cb + 8]),
                              "=r"(v[16 * cb + 9]), "=r"(v[16 * cb + 10]), "=r"(v[16 * cb + 11]),
                              "=r"(v[16 * cb + 12]), "=r"(v[16 * cb + 13]), "=r"(v[16 * cb + 14]),
                              "=r"(v[16 * cb + 15])
                            : "r"(taddr + ((uint32_t)(32 * warp) << 16) +
                                  (uint32_t)(buf * ED_N + blk * 64 + cb * 16)));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    // score' = |t|^2 - 2 q.t (|q|^2 is added once per row); the block minimum
                    // by a min tree, the index only when the row's best improves (rare once a
                    // few tiles are done)
                    float sc[64];
#pragma unroll
                    for (int j = 0; j < 64; ++j) sc[j] = fmaf(-2.0f, __uint_as_float(v[j]), tv[j]);
                    if (nb0 + 64 > nt) {  // the last tile's columns past nt (warp-uniform)
#pragma unroll
                        for (int j = 0; j < 64; ++j) sc[j] = nb0 + j < nt ? sc[j] : kInf;
                    }
                    float m = sc[0];
#pragma unroll
                    for (int j = 1; j < 64; j += 2) m = fminf(m, fminf(sc[j], j + 1 < 64 ? sc[j + 1] : kInf));
                    if (m + qrow < bestv) {
                        int jj = 0;
#pragma unroll
                        for (int j = 63; j >= 0; --j) jj = sc[j] == m ? j : jj;  // first minimum
                        bestv = m + qrow;
                        besti = nb0 + jj;
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(b_aempty + 8 * buf);  // this thread is done with the accumulator
                buf ^= 1;
            }
            if (row < nq && besti >= 0)
                atomicMin(key + row, make_key(fmaxf(bestv, 0.0f), (unsigned)besti));
        }
    }
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr),
                     "n"(2 * ED_N)
                     : "memory");
}

int ed_seed_supported(int L) { return L >= 1; }

size_t ed_seed_scratch_bytes(int64_t nq, int64_t nt, int L) {
    const int64_t Lk = ed_lk(L);
    const int64_t qrows = (nq + ED_M - 1) / ED_M * ED_M, trows = (nt + ED_N - 1) / ED_N * ED_N;
    return (size_t)(qrows + trows) * (size_t)Lk * 2 + (size_t)((nq + 3) / 4 * 4 + trows) * 4 +
           1024;
}

// q [nq][L], t [nt][L] fp32 -> key[q] = min over n of ((ED(q, t_n) as f32 bits) << 32 | n),
// computed in bf16 / fp32 on the tensor cores (key must hold kNone on entry).  scratch: the bf16
// operand images and norms, ed_seed_scratch_bytes.
int launch_ed_seed(const float *q, int64_t nq, const float *t, int64_t nt, int L, void *scratch,
                   unsigned long long *key, int num_sms, cudaStream_t st) {
    if (nq == 0 || nt == 0) return 0;
    if (!ed_seed_supported(L)) return -1;
    const int Lk = ed_lk(L);
    const int64_t qrows = (nq + ED_M - 1) / ED_M * ED_M, trows = (nt + ED_N - 1) / ED_N * ED_N;
    __nv_bfloat16 *qimg = reinterpret_cast<__nv_bfloat16 *>(scratch);
    __nv_bfloat16 *timg = qimg + qrows * Lk;
    float *qn = reinterpret_cast<float *>(timg + trows * Lk);
    float *tn = qn + (nq + 3) / 4 * 4;  // 16-byte aligned: the epilogue reads it as float4
    const int f = ed_f(L);
    k_ed_prep<<<num_sms * 8, 256, 0, st>>>(q, nq, L, f, Lk, ED_M, qimg, qn);
    k_ed_prep<<<num_sms * 8, 256, 0, st>>>(t, nt, L, f, Lk, ED_N, timg, tn);
    const int nkc = Lk / ED_KC;
    const size_t smem = (size_t)nkc * ED_A_CHUNK + ED_STAGES * ED_B_CHUNK + 256 + 1024;
    cudaFuncSetAttribute(k_ed_argmin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t nmb = (nq + ED_M - 1) / ED_M;
    const int64_t ntile = (nt + ED_N - 1) / ED_N;
    // about four units per SM (balance), each long enough to amortise its A load
    int nsplit = (int)((4 * (int64_t)num_sms + nmb - 1) / nmb);
    if (nsplit > ntile) nsplit = (int)ntile;
    if (nsplit < 1) nsplit = 1;
    const int64_t units = nmb * nsplit;
    const int grid = (int)(units < num_sms ? units : num_sms);
    k_ed_argmin<<<grid, 160, smem, st>>>(qimg, timg, qn, tn, nq, nt, Lk, nsplit, key);
    count_launch(3, __func__);
    return 0;
}

}  // namespace nndtw
