// common.cuh -- internal helpers shared by the libnndtw.so translation units (not part of
// the ABI).  Nothing here is shared with oracle/ (DESIGN.md "Oracle independence").
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>

#include "../../include/nndtw.h"

#ifdef NNDTW_DEBUG
#define NNDTW_ASSERT(cond, ...)                                                        \
    do {                                                                               \
        if (!(cond)) {                                                                 \
            printf("NNDTW_ASSERT %s:%d %s | ", __FILE__, __LINE__, #cond);             \
            printf(__VA_ARGS__);                                                       \
            printf("\n");                                                              \
            __trap();                                                                  \
        }                                                                              \
    } while (0)
#else
#define NNDTW_ASSERT(cond, ...) \
    do {                        \
    } while (0)
#endif

namespace nndtw {

constexpr float kInf = __builtin_huge_valf();
constexpr unsigned long long kKeyInit = 0x7F800000FFFFFFFFull;  // (+inf bits << 32) | ~0
constexpr unsigned long long kNone = ~0ull;
// "no candidate" in keys exchanged between ranks: the largest signed int64, so that a signed
// MIN reduction (NCCL / gloo on int64) treats it as +inf.
constexpr unsigned long long kNone64 = 0x7FFFFFFFFFFFFFFFull;

// Rounding-error margins of reading C16 (u = 2^-24, fp32 storage and accumulation):
//  prune a pair only if LB > bsf*(1+eps_p), eps_p = (3L+8)u;
//  abandon / near-tie band at bsf*(1+eps_t), eps_t = (4L+8)u.
inline float eps_prune(int L) { return (3.0f * (float)L + 8.0f) * 0x1p-24f; }
inline float eps_tie(int L) { return (4.0f * (float)L + 8.0f) * 0x1p-24f; }

// process-wide launch counter (bench bookkeeping; incremented by every launcher)
void count_launch(int n = 1, const char *who = nullptr);
int64_t launches_total();

struct CudaCheck {
    static int last(const char *where);
};

// ---- small device helpers ----------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

// GPU-scope relaxed load: sees other SMs' atomics (L2 is the coherence point) without the
// system-scope cost of ld.volatile.
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ float key_dist(unsigned long long k) {
    return __uint_as_float((unsigned)(k >> 32));
}

__device__ __forceinline__ unsigned long long make_key(float d, unsigned idx) {
    return ((unsigned long long)__float_as_uint(d) << 32) | (unsigned long long)idx;
}

__device__ __forceinline__ float sq(float x) { return x * x; }

// ---- packed fp32 pairs (sm_100 FADD2): two IEEE round-to-nearest subtractions in one
// instruction, bit-identical to two scalar FADDs.  Operands are 64-bit register pairs
// (lo, hi); the pack/unpack moves vanish when the halves already sit in an aligned pair.
__device__ __forceinline__ unsigned long long f2_pack(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_unpack(unsigned long long v, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
// shared-memory load the compiler may not merge with another load of the same address (used to
// fill two differently aligned register-pair copies of one row without register moves)
__device__ __forceinline__ float lds_distinct(const float *p) {
    float v;
    asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
}
__device__ __forceinline__ unsigned long long f2_sub(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b,
                                                     unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// cp.async global -> shared (LDGSTS), 4 or 16 bytes, and the wait for all of a thread's copies
__device__ __forceinline__ void cp_async4(float *dst, const float *src) {
    unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(float *dst, const float *src) {
    unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}
// TMA bulk prefetch of [src, src+bytes) into L2 (16-byte aligned, multiple of 16 bytes)
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
// all but the most recently committed group of this thread's copies have landed
__device__ __forceinline__ void cp_async_wait_group1() {
    asm volatile("cp.async.wait_group 1;" ::: "memory");
}
// all but the N most recently committed groups of this thread's copies have landed
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---- LB_Kim, sum variant "without repetitions" (reading C7) -----------------------
// features first, last, min, max in that order; a feature is dropped if its index in either
// series is already used (first/last indices are 0 and L-1); ties -> lowest index (the
// nndtw_kim features).  qf/ql, tf/tl = first/last values of the two series.
// Branch-free form: per series the usable-feature flags (bit 0: the min index is interior,
// bit 1: the max index is interior, bit 2: min and max share an index), then per pair
//   okmin = both mins interior, okmax = both maxes interior and not (okmin and a shared index)
// and the feature terms are added by select after an FFMA -- the same roundings in the same
// order for every caller (tile kernel, sparse bridge, bound finish), so their values agree.
struct KimF {
    float vmin, vmax;
    unsigned flags;
};
__device__ __forceinline__ KimF kim_f(const nndtw_kim &k, int L) {
    KimF f;
    f.vmin = k.vmin;
    f.vmax = k.vmax;
    f.flags = (k.imin != 0 && k.imin != L - 1 ? 1u : 0u) |
              (k.imax != 0 && k.imax != L - 1 ? 2u : 0u) | (k.imax == k.imin ? 4u : 0u);
    return f;
}
__device__ __forceinline__ float kim_sum_f(float qf, float ql, float tf, float tl, const KimF &a,
                                           const KimF &b) {
    const float dl = ql - tl, df = qf - tf;
    float kim = fmaf(df, df, __fmul_rn(dl, dl));
    const unsigned both = a.flags & b.flags, any = a.flags | b.flags;
    const bool okmin = (both & 1u) != 0;
    const bool okmax = (both & 2u) != 0 && !(okmin && (any & 4u) != 0);
    const float dmn = a.vmin - b.vmin, dmx = a.vmax - b.vmax;
    const float k1 = fmaf(dmn, dmn, kim);
    kim = okmin ? k1 : kim;
    const float k2 = fmaf(dmx, dmx, kim);
    return okmax ? k2 : kim;
}
__device__ __forceinline__ float kim_sum(float qf, float ql, float tf, float tl,
                                         const nndtw_kim &ka, const nndtw_kim &kb, int L) {
    return kim_sum_f(qf, ql, tf, tl, kim_f(ka, L), kim_f(kb, L));
}

// Algorithm 1 line 1: delta(A_1, B_1) + delta(A_L, B_L), one rounding order for every
// kernel that computes it (tile, sparse bridge), so their band sums agree bit for bit
__device__ __forceinline__ float boundary_terms(float qf, float ql, float tf, float tl) {
    const float df = qf - tf, dl = ql - tl;
    return fmaf(df, df, __fmul_rn(dl, dl));
}

// ---- work items ---------------------------------------------------------------------------
// A DTW work item: query (row of A), train (row of B), local indices, and the pair's cascade
// bound (survivor items are skipped at fetch time when it exceeds the live best-so-far).
struct Item {
    unsigned q, n;
    float lb;
};

// Survivor order (S3/S4): LB / bsf_seed buckets, visited in ascending order so that every query's
// most promising candidates run first and later ones meet a tightened best-so-far.
constexpr int NBUCKET = 64;

// near-tie log entry (S7): completed candidate within the band of the live best at the time
struct TieEntry {
    unsigned q, n;
    float d32;
    float pad;
    double d64;
};

struct TieLog {
    TieEntry *e;
    unsigned long long *count;   // appended entries (may exceed capacity: overflow)
    unsigned long long capacity;
    unsigned *overflow;          // [nq] 1 if an entry of query q was dropped
};

// Per-call device counters (stats); index meaning below.
enum { CNT_ITEMS = 0, CNT_ABANDONED = 1, CNT_CELLS = 2, CNT_SURVIVORS = 3, CNT_TIES = 4,
       CNT_SKIPPED = 5, CNT_PRUNED_KIM = 8, CNT_PRUNED_BANDS = 9, CNT_PRUNED_KEOGH = 10,
       CNT_SEED2 = 11, CNT_FALLBACK = 12, CNT_N = 13 };

}  // namespace nndtw
