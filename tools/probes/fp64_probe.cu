// FP64 throughput probe: DFMA (vector pipe) against DMMA (mma.sync m8n8k4
// f64, the tensor pipe), to decide how the high-order M2L contraction is
// issued.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_probe(int iters, const double *in, double *sink) {
    const double m = in[0], c = in[1];
    double a[16];
#pragma unroll
    for (int k = 0; k < 16; k++) a[k] = threadIdx.x * 1e-3 + k;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 16; k++) a[k] = fma(a[k], m, c);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 16; k++) s += a[k];
    if (s == 12345.678) sink[blockIdx.x] = s;
}

// CH independent accumulator tiles per warp
template <int CH>
__global__ void dmma_probe(int iters, const double *in, double *sink) {
    double a = in[0] + threadIdx.x * 1e-9, b = in[1] - threadIdx.x * 1e-9;
    double c[CH][2];
#pragma unroll
    for (int k = 0; k < CH; k++) c[k][0] = c[k][1] = k;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < CH; k++)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(c[k][0]), "+d"(c[k][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < CH; k++) s += c[k][0] + c[k][1];
    if (s == 12345.678) sink[blockIdx.x] = s;
}

// DFMA and DMMA interleaved: do the two pipes overlap?
template <int CH>
__global__ void mixed_probe(int iters, const double *in, double *sink) {
    const double m = in[0], cc = in[1];
    double a = in[0] + threadIdx.x * 1e-9, b = in[1] - threadIdx.x * 1e-9;
    double c[CH][2], f[16];
#pragma unroll
    for (int k = 0; k < CH; k++) c[k][0] = c[k][1] = k;
#pragma unroll
    for (int k = 0; k < 16; k++) f[k] = threadIdx.x * 1e-3 + k;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < CH; k++)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(c[k][0]), "+d"(c[k][1])
                         : "d"(a), "d"(b));
#pragma unroll
        for (int k = 0; k < 16; k++) f[k] = fma(f[k], m, cc);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < CH; k++) s += c[k][0] + c[k][1];
#pragma unroll
    for (int k = 0; k < 16; k++) s += f[k];
    if (s == 12345.678) sink[blockIdx.x] = s;
}

template <class K>
float timeit(K kern, int blocks, int threads, int iters, const double *in, double *sink) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<blocks, threads>>>(iters, in, sink);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(iters, in, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main() {
    double h[2] = {0.9999999, 1e-9};
    double *in, *sink;
    cudaMalloc(&in, 64);
    cudaMalloc(&sink, 1 << 20);
    cudaMemcpy(in, h, 16, cudaMemcpyHostToDevice);
    int blocks = 148 * 8, it = 4096;
    float ms = timeit(dfma_probe, blocks, 256, it, in, sink);
    printf("DFMA  %.2f TFLOP/s\n", 2.0 * 16 * it * blocks * 256.0 / (ms * 1e-3) / 1e12);
    ms = timeit(dmma_probe<4>, blocks, 256, it, in, sink);
    printf("DMMA4 %.2f TFLOP/s\n", 2.0 * 256 * 4 * it * blocks * 8.0 / (ms * 1e-3) / 1e12);
    ms = timeit(dmma_probe<8>, blocks, 256, it, in, sink);
    printf("DMMA8 %.2f TFLOP/s\n", 2.0 * 256 * 8 * it * blocks * 8.0 / (ms * 1e-3) / 1e12);
    ms = timeit(dmma_probe<2>, blocks, 256, it, in, sink);
    printf("DMMA2 %.2f TFLOP/s\n", 2.0 * 256 * 2 * it * blocks * 8.0 / (ms * 1e-3) / 1e12);
    // per iteration: CH DMMAs (CH * 512 flops per warp) and 16 DFMAs per thread (32 flops)
    ms = timeit(mixed_probe<2>, blocks, 256, it, in, sink);
    printf("mixed(2 DMMA + 16 DFMA per thread-iter): total %.2f TFLOP/s (dmma part %.2f, dfma part %.2f)\n",
           (2.0 * 256 * 2 * 8 + 2.0 * 16 * 256) * it * blocks / (ms * 1e-3) / 1e12,
           2.0 * 256 * 2 * 8 * it * blocks / (ms * 1e-3) / 1e12, 2.0 * 16 * 256 * it * blocks / (ms * 1e-3) / 1e12);
    ms = timeit(mixed_probe<4>, blocks, 256, it, in, sink);
    printf("mixed(4 DMMA + 16 DFMA per thread-iter): total %.2f TFLOP/s (dmma part %.2f, dfma part %.2f)\n",
           (2.0 * 256 * 4 * 8 + 2.0 * 16 * 256) * it * blocks / (ms * 1e-3) / 1e12,
           2.0 * 256 * 4 * 8 * it * blocks / (ms * 1e-3) / 1e12, 2.0 * 16 * 256 * it * blocks / (ms * 1e-3) / 1e12);
    return 0;
}
