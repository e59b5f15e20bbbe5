// DMMA m8n8k4 throughput vs independent accumulator chains per warp and warps
// per SMSP (the orbit-FFT base change runs 3 warps x 2 chains per SMSP).
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void k(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
    double c[ILP][2];
#pragma unroll
    for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}
template <int ILP>
void run(int warps_per_sm, int sms, double* d) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    k<ILP><<<sms, 32 * warps_per_sm>>>(d, 100);
    cudaEventRecord(e0);
    k<ILP><<<sms, 32 * warps_per_sm>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * ILP * (double)iters * sms * warps_per_sm;
    printf("chains/warp %d warps/SM %2d (per SMSP %d): %.2f TFLOP/s\n", ILP, warps_per_sm, warps_per_sm / 4, fl / ms / 1e9);
}
int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d; cudaMalloc(&d, 1 << 20);
    for (int w : {4, 8, 12, 16}) { run<1>(w, sms, d); run<2>(w, sms, d); run<4>(w, sms, d); }
    return 0;
}
