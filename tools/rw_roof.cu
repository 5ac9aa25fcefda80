// HBM roof for the envelope kernel's traffic mix: read x once, write two arrays of the same size
// (12 B per element), float4, grid-stride, 148 x k CTAs.  Also a plain copy (8 B per element)
// for comparison with MEASURED_PEAKS.json.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_rw2(const float4 *__restrict__ x, size_t n4, float4 *__restrict__ a,
                      float4 *__restrict__ b) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
         i += (size_t)gridDim.x * blockDim.x) {
        float4 v = __ldg(x + i);
        a[i] = v;
        b[i] = make_float4(-v.x, -v.y, -v.z, -v.w);
    }
}
// the envelope kernels' pattern: each thread owns 16 contiguous floats (4 float4, 64 B)
__global__ void k_rw2_chunk(const float4 *__restrict__ x, size_t n4, float4 *__restrict__ a,
                            float4 *__restrict__ b) {
    for (size_t c = blockIdx.x * (size_t)blockDim.x + threadIdx.x; c < n4 / 4;
         c += (size_t)gridDim.x * blockDim.x) {
        float4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = __ldg(x + 4 * c + j);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            a[4 * c + j] = v[j];
            b[4 * c + j] = make_float4(-v[j].x, -v[j].y, -v[j].z, -v[j].w);
        }
    }
}
__global__ void k_copy(const float4 *__restrict__ x, size_t n4, float4 *__restrict__ a) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
         i += (size_t)gridDim.x * blockDim.x)
        a[i] = __ldg(x + i);
}

int main() {
    const size_t n = 100000ull * 512;  // config 2's train set
    const size_t n4 = n / 4;
    float4 *x, *a, *b;
    cudaMalloc(&x, n * 4);
    cudaMalloc(&a, n * 4);
    cudaMalloc(&b, n * 4);
    cudaMemset(x, 0, n * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int blocks : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
        for (int kind = 0; kind < 3; ++kind) {
            auto go = [&]() {
                if (kind == 1) k_copy<<<blocks, 256>>>(x, n4, a);
                else if (kind == 0) k_rw2<<<blocks, 256>>>(x, n4, a, b);
                else k_rw2_chunk<<<blocks, 256>>>(x, n4, a, b);
            };
            for (int r = 0; r < 3; ++r) go();
            cudaEventRecord(e0);
            const int reps = 20;
            for (int r = 0; r < reps; ++r) go();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            ms /= reps;
            const double bytes = kind == 1 ? 8.0 * n : 12.0 * n;
            const char *nm[3] = {"read1-write2 (12 B/elt)", "copy (8 B/elt)",
                                 "read1-write2, 64 B per thread"};
            printf("%s blocks=%d: %.4f ms  %.0f GB/s\n", nm[kind],
                   blocks, ms, bytes / ms / 1e6);
        }
    }
    return 0;
}
