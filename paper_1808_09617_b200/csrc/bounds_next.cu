// bounds_next.cu -- SURVEY §8(f) next rows: LB_New (a comparison bound of the paper's
// evaluation), the symmetric-bound helpers, and the tightness reduction.  LB_Improved is
// in bounds_improved.cu.
//
// LB_New_W(A,B) = delta(A_1,B_1) + delta(A_L,B_L) + sum_{i=2}^{L-1} min_{j in win(i)} delta(A_i,B_j)
//   (§2.3.4).  min_j (a-b_j)^2 is taken as (min_j |a-b_j|)^2: squaring a rounded
//   non-negative difference is monotone, so the fp32 result is the same as the minimum of the
//   fp32 squares.
//
// Evaluated for all (query, train) pairs: a CTA stages 8 query rows and 16 train rows in shared
// memory (odd row stride, conflict-free) and each thread owns one pair.  The windowed minima are
// direct scans of the 2w+1 window, O(L*w) per pair: the bound's definition takes a minimum over
// every cell of the window (no sliding-window shortcut applies to a min of |a_i - b_j|), the cost
// LB_Enhanced avoids.
#include "launchers.cuh"

namespace nndtw {

constexpr int NB_TQ = 8, NB_TN = 16;  // 128 pairs per CTA, one per thread

// kind 0: LB_New (the only kind; the template parameter is kept for the launcher's switch)
template <int KIND>
__global__ void __launch_bounds__(128) k_lb_pairs(const float *__restrict__ q, int64_t nq,
                                                  const float *__restrict__ t,
                                                  const float *__restrict__ U,
                                                  const float *__restrict__ Lo, int64_t nt,
                                                  int L, int w, float *__restrict__ lb,
                                                  int64_t ldlb) {
    extern __shared__ float nb_smem[];
    const int stride = L + 1;
    float *sA = nb_smem;                    // [NB_TQ][stride]
    float *sB = sA + NB_TQ * stride;        // [NB_TN][stride]
    const int64_t q0 = (int64_t)blockIdx.x * NB_TQ, n0 = (int64_t)blockIdx.y * NB_TN;
    for (int e = threadIdx.x; e < NB_TQ * L; e += blockDim.x) {
        const int r = e / L, c = e - r * L;
        const int64_t qq = q0 + r < nq ? q0 + r : nq - 1;
        sA[r * stride + c] = q[qq * L + c];
    }
    for (int e = threadIdx.x; e < NB_TN * L; e += blockDim.x) {
        const int r = e / L, c = e - r * L;
        const int64_t nn = n0 + r < nt ? n0 + r : nt - 1;
        sB[r * stride + c] = t[nn * L + c];
    }
    __syncthreads();
    const int qi = threadIdx.x / NB_TN, ni = threadIdx.x % NB_TN;
    const float *a = sA + qi * stride, *b = sB + ni * stride;
    float res = sq(a[0] - b[0]);
    if (L > 1) res += sq(a[L - 1] - b[L - 1]);
    for (int i = 1; i < L - 1; ++i) {
        const float ai = a[i];
        const int lo = i - w > 0 ? i - w : 0, hi = i + w < L - 1 ? i + w : L - 1;
        float m = kInf;
        for (int j = lo; j <= hi; ++j) m = fminf(m, fabsf(ai - b[j]));
        res += m * m;
    }
    const int64_t qq = q0 + qi, nn = n0 + ni;
    if (qq < nq && nn < nt) lb[qq * ldlb + nn] = res;
}

int launch_lb_pairs(int kind, const float *q, int64_t nq, const float *t, const float *U,
                    const float *Lo, int64_t nt, int L, int w, float *lb, int64_t ldlb,
                    cudaStream_t st) {
    if (nq == 0 || nt == 0) return 0;
    if (w > L - 1) w = L - 1;
    if (kind != 0) return -1;
    const size_t rows = NB_TQ + NB_TN;
    const size_t smem = rows * (size_t)(L + 1) * sizeof(float);
    if (smem > 227 * 1024) return -1;
    dim3 grid((unsigned)((nq + NB_TQ - 1) / NB_TQ), (unsigned)((nt + NB_TN - 1) / NB_TN));
    if (grid.y > 65535u) return -1;
    cudaFuncSetAttribute(k_lb_pairs<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_lb_pairs<0><<<grid, 128, smem, st>>>(q, nq, t, U, Lo, nt, L, w, lb, ldlb);
    count_launch(1, __func__);
    return 0;
}

// ---- per-row argmin key of a bound matrix (the seed candidate when the bound is assembled in
// several passes, e.g. the symmetric LB_Enhanced) -------------------------------------------------
__global__ void __launch_bounds__(256) k_row_argmin(const float *__restrict__ lb, int64_t ldlb,
                                                    int64_t nq, int64_t nt,
                                                    unsigned long long *minkey) {
    const int64_t q = blockIdx.x;
    if (q >= nq) return;
    unsigned long long best = kNone;
    for (int64_t n = threadIdx.x; n < nt; n += blockDim.x) {
        const unsigned long long k = make_key(lb[q * ldlb + n], (unsigned)n);
        best = k < best ? k : best;
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
        red[0] = best;
        if (best != kNone) minkey[q] = best;
    }
}

int launch_row_argmin(const float *lb, int64_t ldlb, int64_t nq, int64_t nt,
                      unsigned long long *minkey, cudaStream_t st) {
    if (nq == 0 || nt == 0) return 0;
    if (nq > 0x7fffffffll) return -1;
    k_row_argmin<<<(unsigned)nq, 256, 0, st>>>(lb, ldlb, nq, nt, minkey);
    count_launch(1, __func__);
    return 0;
}

// ---- tightness: sum over pairs with DTW > 0 of sqrt(LB / DTW^2) in fp64, the pair count,
// and the largest ratio (an admissible bound keeps it <= 1 up to rounding) ------------------------
__global__ void __launch_bounds__(256) k_tightness(const float *__restrict__ lb,
                                                   const float *__restrict__ d, int64_t n,
                                                   double *sum, unsigned long long *count,
                                                   unsigned *max_bits) {
    double s = 0.0;
    unsigned long long c = 0;
    float mx = 0.0f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float di = d[i];
        if (di > 0.0f && di < kInf) {
            const double r = sqrt((double)lb[i] / (double)di);
            s += r;
            c += 1;
            mx = fmaxf(mx, (float)r);
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, off);
        c += __shfl_xor_sync(0xffffffffu, c, off);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    }
    if ((threadIdx.x & 31) == 0 && c > 0) {
        atomicAdd(sum, s);
        atomicAdd(count, c);
        atomicMax(max_bits, __float_as_uint(mx));
    }
}

int launch_tightness(const float *lb, const float *d, int64_t n, double *sum,
                     unsigned long long *count, unsigned *max_bits, int num_sms,
                     cudaStream_t st) {
    if (n <= 0) return 0;
    int64_t grid = (n + 255) / 256;
    if (grid > (int64_t)num_sms * 8) grid = (int64_t)num_sms * 8;
    k_tightness<<<(unsigned)grid, 256, 0, st>>>(lb, d, n, sum, count, max_bits);
    count_launch(1, __func__);
    return 0;
}

}  // namespace nndtw
