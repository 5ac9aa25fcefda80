// pipebench.cu -- issue/pipe throughput of the DTW cell instruction mixes on sm_100a.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pipebench tools/pipebench.cu
//
// Each variant runs NCH independent chains per thread so latency is hidden; one CTA of 512
// threads per SM (4 warps per scheduler).  Reports warp-instructions per SMSP-cycle and, for
// the cell mixes, DP cells per SM-cycle.  Used to choose between the scalar cell
// (FADD, FMNMX3, FFMA) and the packed cell (FADD2 + FFMA2 over two cells, 2x FMNMX3).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NCH = 8;
constexpr int ITERS = 4096;

__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk(unsigned long long v, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}

template <int V>
__global__ void __launch_bounds__(512) k(float *out, long long *cyc, float seed) {
    float x[NCH], y[NCH], z[NCH];
    unsigned long long px[NCH], py[NCH], pz[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        x[c] = seed * (c + 1) + threadIdx.x;
        y[c] = seed - c;
        z[c] = seed + 0.5f * c;
        px[c] = pk(x[c], x[c] + 1.f);
        py[c] = pk(y[c], y[c] - 1.f);
        pz[c] = pk(z[c], z[c] * 2.f);
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            if (V == 0) {  // FFMA 3-reg
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(y[c]), "f"(z[c]));
            } else if (V == 1) {  // FADD
                asm volatile("add.f32 %0, %0, %1;" : "+f"(x[c]) : "f"(y[c]));
            } else if (V == 2) {  // FMNMX3
                asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(y[c]), "f"(z[c]));
            } else if (V == 3) {  // FMNMX 2-input
                asm volatile("min.f32 %0, %0, %1;" : "+f"(x[c]) : "f"(y[c]));
            } else if (V == 4) {  // FFMA2
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(px[c]) : "l"(py[c]), "l"(pz[c]));
            } else if (V == 5) {  // FADD2
                asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(px[c]) : "l"(py[c]));
            } else if (V == 6) {  // scalar cell: t = a - b; D = t*t + min3(D, lo, hi)
                float t;
                asm volatile("sub.f32 %0, %1, %2;" : "=f"(t) : "f"(y[c]), "f"(z[c]));
                float m;
                asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(m) : "f"(x[c]), "f"(y[c]), "f"(z[(c + 1) % NCH]));
                asm volatile("fma.rn.f32 %0, %1, %1, %2;" : "=f"(x[c]) : "f"(t), "f"(m));
            } else if (V == 7) {  // packed cell pair: FADD2, 2x FMNMX3, FFMA2
                unsigned long long t;
                asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(py[c]), "l"(pz[c]));
                float d0, d1;
                upk(px[c], d0, d1);
                float m0, m1;
                asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(m0) : "f"(d0), "f"(y[c]), "f"(z[c]));
                asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(m1) : "f"(d1), "f"(z[c]), "f"(y[c]));
                unsigned long long m = pk(m0, m1);
                asm volatile("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(px[c]) : "l"(t), "l"(m));
            } else if (V == 8) {  // FFMA imm form (one register source + immediates)
                asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3F000000;" : "+f"(x[c]));
            } else if (V == 9) {  // FFMA2 with one repeated operand
                asm volatile("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(px[c]) : "l"(py[c]));
            } else if (V == 10) {  // LB bridge scalar: u=a-U, l=L-a, t=max(u,l,0), acc+=t*t
                float u, l, t;
                const float a = x[(c + 1) % NCH];
                asm volatile("sub.f32 %0, %1, %2;" : "=f"(u) : "f"(a), "f"(z[c]));
                asm volatile("sub.f32 %0, %1, %2;" : "=f"(l) : "f"(y[c]), "f"(a));
                asm volatile("max.f32 %0, %1, %2, 0f00000000;" : "=f"(t) : "f"(u), "f"(l));
                asm volatile("fma.rn.f32 %0, %1, %1, %0;" : "+f"(x[c]) : "f"(t));
            } else if (V == 11) {  // LB bridge packed over two pairs
                unsigned long long u, l;
                const unsigned long long a2 = px[(c + 1) % NCH];
                asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(u) : "l"(a2), "l"(pk(z[c], z[c])));
                asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(l) : "l"(pk(y[c], y[c])), "l"(a2));
                float u0, u1, l0, l1, t0, t1;
                upk(u, u0, u1);
                upk(l, l0, l1);
                asm volatile("max.f32 %0, %1, %2, 0f00000000;" : "=f"(t0) : "f"(u0), "f"(l0));
                asm volatile("max.f32 %0, %1, %2, 0f00000000;" : "=f"(t1) : "f"(u1), "f"(l1));
                unsigned long long t = pk(t0, t1);
                asm volatile("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(px[c]) : "l"(t));
            } else if (V == 12) {  // DTW half-packed: FADD2, 2x FMNMX3, 2x FFMA
                unsigned long long t;
                asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(py[c]), "l"(pz[c]));
                float t0, t1;
                upk(t, t0, t1);
                float d0, d1;
                upk(px[c], d0, d1);
                float m0, m1;
                asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(m0) : "f"(d0), "f"(y[c]), "f"(z[c]));
                asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(m1) : "f"(d1), "f"(z[c]), "f"(y[c]));
                asm volatile("fma.rn.f32 %0, %1, %1, %2;" : "=f"(d0) : "f"(t0), "f"(m0));
                asm volatile("fma.rn.f32 %0, %1, %1, %2;" : "=f"(d1) : "f"(t1), "f"(m1));
                px[c] = pk(d0, d1);
            } else if (V == 13) {  // DTW cell with two 2-input FMNMX
                float t;
                asm volatile("sub.f32 %0, %1, %2;" : "=f"(t) : "f"(y[c]), "f"(z[c]));
                float m;
                asm volatile("min.f32 %0, %1, %2;" : "=f"(m) : "f"(x[c]), "f"(y[c]));
                asm volatile("min.f32 %0, %0, %1;" : "+f"(m) : "f"(z[(c + 1) % NCH]));
                asm volatile("fma.rn.f32 %0, %1, %1, %2;" : "=f"(x[c]) : "f"(t), "f"(m));
            } else if (V == 14) {  // FMNMX3 with an immediate zero
                asm volatile("max.f32 %0, %0, %1, 0f00000000;" : "+f"(x[c]) : "f"(y[c]));
            } else if (V == 15) {  // FFMA + FMNMX3 alternating (pipe overlap test)
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(y[c]), "f"(z[c]));
                asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(z[c]) : "f"(y[c]), "f"(x[(c + 1) % NCH]));
            } else if (V == 17) {  // LB packed with scalar FFMA accumulation
                unsigned long long u, l;
                const unsigned long long a2 = px[(c + 1) % NCH];
                asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(u) : "l"(a2), "l"(pk(z[c], z[c])));
                asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(l) : "l"(pk(y[c], y[c])), "l"(a2));
                float u0, u1, l0, l1, t0, t1, p0, p1;
                upk(u, u0, u1);
                upk(l, l0, l1);
                asm volatile("max.f32 %0, %1, %2, 0f00000000;" : "=f"(t0) : "f"(u0), "f"(l0));
                asm volatile("max.f32 %0, %1, %2, 0f00000000;" : "=f"(t1) : "f"(u1), "f"(l1));
                upk(px[c], p0, p1);
                asm volatile("fma.rn.f32 %0, %1, %1, %0;" : "+f"(p0) : "f"(t0));
                asm volatile("fma.rn.f32 %0, %1, %1, %0;" : "+f"(p1) : "f"(t1));
                px[c] = pk(p0, p1);
            } else if (V == 18) {  // LB: u scalar FADD, l scalar FADD, FMNMX x2 (2-input), FFMA via max(t,0)*t
                float u, l, t, r;
                const float a = x[(c + 1) % NCH];
                asm volatile("sub.f32 %0, %1, %2;" : "=f"(u) : "f"(a), "f"(z[c]));
                asm volatile("sub.f32 %0, %1, %2;" : "=f"(l) : "f"(y[c]), "f"(a));
                asm volatile("max.f32 %0, %1, %2;" : "=f"(t) : "f"(u), "f"(l));
                asm volatile("max.f32 %0, %1, 0f00000000;" : "=f"(r) : "f"(t));
                asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(x[c]) : "f"(t), "f"(r));
            } else if (V == 19) {  // FADD2 + FFMA alternating (do they share a sub-pipe?)
                asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(px[c]) : "l"(py[c]));
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(y[c]), "f"(z[c]));
            } else if (V == 20) {  // FADD2 + FFMA + FMNMX3
                asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(px[c]) : "l"(py[c]));
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(y[c]), "f"(z[c]));
                asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(z[c]) : "f"(y[c]), "f"(x[(c + 1) % NCH]));
            } else if (V == 21) {  // FADD + FFMA alternating
                asm volatile("add.f32 %0, %0, %1;" : "+f"(y[c]) : "f"(z[c]));
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(y[c]), "f"(z[c]));
            } else if (V == 22) {  // FADD2 + FMNMX3
                asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(px[c]) : "l"(py[c]));
                asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(z[c]) : "f"(y[c]), "f"(x[(c + 1) % NCH]));
            } else if (V == 23) {  // FADD2 with a broadcast scalar operand
                asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(px[c]) : "l"(pk(y[c], y[c])));
            } else if (V == 16) {  // FFMA + FMNMX (2-in) alternating
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(y[c]), "f"(z[c]));
                asm volatile("min.f32 %0, %0, %1;" : "+f"(z[c]) : "f"(x[(c + 1) % NCH]));
            }
        }
    }
    long long t1 = clock64();
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        float a, b;
        upk(px[c], a, b);
        acc += x[c] + a + b;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
void run(const char *name, int instr_per_chain_iter, double cells_per_chain_iter, int nsm,
         float *out, long long *cyc) {
    k<V><<<nsm, 512>>>(out, cyc, 1.0001f);
    cudaDeviceSynchronize();
    k<V><<<nsm, 512>>>(out, cyc, 1.0001f);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("%s: %s\n", name, cudaGetErrorString(e));
        return;
    }
    long long h[1024];
    cudaMemcpy(h, cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < nsm; ++i) s += (double)h[i];
    double cycles = s / nsm;
    double warp_instr_per_smsp = 4.0 * ITERS * NCH * instr_per_chain_iter;  // 16 warps / 4 SMSPs
    double ipc = warp_instr_per_smsp / cycles;
    double cells_sm = 16.0 * 32 * ITERS * NCH * cells_per_chain_iter / cycles;
    printf("%-34s warp-instr/SMSP/clk = %.3f   cells/SM/clk = %.1f\n", name, ipc, cells_sm);
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    long long *cyc;
    cudaMalloc(&out, (size_t)nsm * 512 * sizeof(float));
    cudaMalloc(&cyc, (size_t)nsm * sizeof(long long));
    run<0>("FFMA (3 reg)", 1, 0, nsm, out, cyc);
    run<1>("FADD", 1, 0, nsm, out, cyc);
    run<2>("FMNMX3", 1, 0, nsm, out, cyc);
    run<3>("FMNMX (2 in)", 1, 0, nsm, out, cyc);
    run<4>("FFMA2 (f32x2, 3 reg)", 1, 0, nsm, out, cyc);
    run<5>("FADD2 (f32x2)", 1, 0, nsm, out, cyc);
    run<8>("FFMA imm", 1, 0, nsm, out, cyc);
    run<9>("FFMA2 (a*a+d)", 1, 0, nsm, out, cyc);
    run<6>("scalar cell FADD+FMNMX3+FFMA", 3, 1, nsm, out, cyc);
    run<7>("packed cell FADD2+2FMNMX3+FFMA2", 4, 2, nsm, out, cyc);
    run<12>("half-packed FADD2+2FMNMX3+2FFMA", 5, 2, nsm, out, cyc);
    run<13>("cell FADD+2FMNMX+FFMA", 4, 1, nsm, out, cyc);
    run<10>("LB scalar FADD,FADD,FMNMX3,FFMA", 4, 1, nsm, out, cyc);
    run<11>("LB packed 2FADD2,2FMNMX3,FFMA2", 5, 2, nsm, out, cyc);
    run<17>("LB packed 2FADD2,2FMNMX3,2FFMA", 6, 2, nsm, out, cyc);
    run<18>("LB FADD,FADD,FMNMX,FMNMX,FFMA", 5, 1, nsm, out, cyc);
    run<14>("FMNMX3 imm 0", 1, 0, nsm, out, cyc);
    run<19>("FADD2+FFMA", 2, 0, nsm, out, cyc);
    run<20>("FADD2+FFMA+FMNMX3", 3, 0, nsm, out, cyc);
    run<21>("FADD+FFMA", 2, 0, nsm, out, cyc);
    run<22>("FADD2+FMNMX3", 2, 0, nsm, out, cyc);
    run<23>("FADD2 broadcast", 1, 0, nsm, out, cyc);
    run<15>("FFMA+FMNMX3", 2, 0, nsm, out, cyc);
    run<16>("FFMA+FMNMX", 2, 0, nsm, out, cyc);
    return 0;
}
