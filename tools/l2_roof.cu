// L2 -> SM read roof for the sparse bridge's access pattern (k_lb_sparse): warps read whole
// 2 KB rows (float4 per lane, 4 per row) picked pseudo-randomly from a 20 MB L2-resident set
// (config 2's 10,000 query rows of L = 512), and fold them into a register sum.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_roof tools/l2_roof.cu
//   tools/l2_roof [rows_in_flight_per_warp]
// Prints GB/s for warps/SM in {8, 16, 32} and 1, 2, 4 rows in flight per warp.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int INFL>
__global__ void rd(const float4 *__restrict__ x, int nrows, int row4, long long iters,
                   float *out) {
    const int lane = threadIdx.x & 31;
    const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    unsigned h = (unsigned)gw * 2654435761u + 12345u;
    float acc = 0.f;
    for (long long it = 0; it < iters; it += INFL) {
        float4 v[INFL][4];
#pragma unroll
        for (int k = 0; k < INFL; ++k) {
            h = h * 1664525u + 1013904223u;
            const int r = (int)((h >> 8) % (unsigned)nrows);
#pragma unroll
            for (int c = 0; c < 4; ++c) v[k][c] = __ldg(x + (long long)r * row4 + 32 * c + lane);
        }
#pragma unroll
        for (int k = 0; k < INFL; ++k)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc += v[k][c].x + v[k][c].y + v[k][c].z + v[k][c].w;
    }
    if (acc == 12345.f) out[0] = acc;
}

template <int INFL>
void run(const float4 *x, int nrows, float *out, int sms, int wpsm) {
    const int bs = 256, blocks = sms * wpsm / 8;
    const long long iters = 4096;
    rd<INFL><<<blocks, bs>>>(x, nrows, 128, iters, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) rd<INFL><<<blocks, bs>>>(x, nrows, 128, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 5.0 * blocks * 8 * (double)iters * 2048.0;
    printf("warps/SM %2d  rows in flight %d  %.0f GB/s\n", wpsm, INFL, bytes / (ms * 1e6));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int nrows = 10000;
    float4 *x;
    float *out;
    cudaMalloc(&x, (size_t)nrows * 2048);
    cudaMalloc(&out, 4);
    cudaMemset(x, 0, (size_t)nrows * 2048);
    for (int w : {8, 16, 32}) {
        run<1>(x, nrows, out, sms, w);
        run<2>(x, nrows, out, sms, w);
        run<4>(x, nrows, out, sms, w);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
