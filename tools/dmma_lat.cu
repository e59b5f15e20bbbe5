// DMMA m8n8k4 f64 latency / throughput probe: one CTA per SM, W warps, each
// warp runs C independent accumulator chains of dependent DMMAs.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int C>
__global__ void k(int iters, double* out, long long* cyc) {
    double c[C][2];
    for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-9;
    const double a = 1.0000001, b = 0.9999999;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < C; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int C>
void run(int warps) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    const int iters = 4096;
    k<C><<<148, warps * 32>>>(iters, out, cyc);
    k<C><<<148, warps * 32>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double per_warp_dmma = double(h) / (iters * C);
    printf("chains/warp %d warps/SM %2d: %.2f cycles per DMMA per warp, SM rate %.3f DMMA/clk (peak 0.25)\n", C, warps,
           per_warp_dmma, warps / per_warp_dmma);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run<1>(1);
    run<2>(1);
    run<4>(1);
    run<8>(1);
    run<1>(4);
    run<2>(4);
    run<4>(4);
    run<1>(8);
    run<2>(8);
    run<4>(8);
    run<1>(16);
    run<2>(16);
    run<4>(16);
    run<8>(16);
    return 0;
}
