// Microbenchmark: FP64 DFMA, FP64 DMMA (mma.sync.m8n8k4.f64), FP32 FFMA peaks
// on B200 (the roofline denominators MEASURED_PEAKS.json does not carry).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double acc[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += acc[i];
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <int ILP>
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
    float acc[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) acc[i] = fmaf(acc[i], a, b);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += acc[i];
    if (s == 12345.678f) out[threadIdx.x] = s;
}

template <int ILP>
__global__ void dmma_kernel(double* out, int iters) {
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
__global__ void dmma16_kernel(double* out, int iters) {
    double a0 = 1.0 + threadIdx.x * 1e-6, a1 = 0.5, b = 0.999;
    double c[ILP][4];
#pragma unroll
    for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i)
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <int ILP>
__global__ void hmma_tf32_kernel(float* out, int iters) {
    // mma.sync.m16n8k8 tf32 (legacy warp-level tensor op on sm_100a)
    uint32_t a0 = __float_as_uint(1.0f + threadIdx.x * 1e-6f), a1 = __float_as_uint(0.5f), a2 = a0, a3 = a1;
    uint32_t b0 = __float_as_uint(0.999f), b1 = b0;
    float c[ILP][4];
#pragma unroll
    for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.678f) out[threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    cudaMalloc(&d, 1 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int blocksPerSM : {2, 4, 8}) {
        const int grid = sms * blocksPerSM, threads = 256;
        float ms;
        dfma_kernel<8><<<grid, threads>>>(d, 100, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        dfma_kernel<8><<<grid, threads>>>(d, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * iters * (double)grid * threads;
        printf("DFMA  bps=%d: %.2f TFLOP/s\n", blocksPerSM, flops / ms / 1e9);

        ffma_kernel<8><<<grid, threads>>>((float*)d, 100, 1.0000001f, 1e-9f);
        cudaEventRecord(e0);
        ffma_kernel<8><<<grid, threads>>>((float*)d, iters, 1.0000001f, 1e-9f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("FFMA  bps=%d: %.2f TFLOP/s\n", blocksPerSM, flops / ms / 1e9);

        dmma_kernel<4><<<grid, threads>>>(d, 100);
        cudaEventRecord(e0);
        dmma_kernel<4><<<grid, threads>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double mflops = 2.0 * 256 * 4 * (double)iters * grid * (threads / 32);
        printf("DMMA m8n8k4 bps=%d: %.2f TFLOP/s\n", blocksPerSM, mflops / ms / 1e9);

        dmma16_kernel<4><<<grid, threads>>>(d, 100);
        cudaEventRecord(e0);
        dmma16_kernel<4><<<grid, threads>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        mflops = 2.0 * 512 * 4 * (double)iters * grid * (threads / 32);
        printf("DMMA m16n8k4 bps=%d: %.2f TFLOP/s\n", blocksPerSM, mflops / ms / 1e9);

        hmma_tf32_kernel<4><<<grid, threads>>>((float*)d, 100);
        cudaEventRecord(e0);
        hmma_tf32_kernel<4><<<grid, threads>>>((float*)d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        mflops = 2.0 * 16 * 8 * 8 * 4 * (double)iters * grid * (threads / 32);
        printf("HMMA m16n8k8 tf32 bps=%d: %.2f TFLOP/s\n", blocksPerSM, mflops / ms / 1e9);
    }
    cudaError_t err = cudaGetLastError();
    printf("err=%s\n", cudaGetErrorString(err));
    return 0;
}
