// FP32 packed-op throughput probe: FFMA2 vs FADD2 vs FMUL2 and the P2P mix.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe pipe_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f2;
#define FMA(d, a, b, c) asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c))
#define ADD(d, a, b) asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b))
#define MUL(d, a, b) asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b))
__device__ f2 pk(float a, float b) { f2 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
template <int MODE>
__global__ void probe(int iters, const float *in, float *sink) {
    const float m0 = in[0], c0 = in[1], z0 = in[2];
    const f2 m = pk(m0, m0), c = pk(c0, c0), z = pk(z0, z0);
    f2 a[13];
#pragma unroll
    for (int k = 0; k < 13; k++) a[k] = pk(threadIdx.x * 1e-3f + k, k * 0.5f);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 13; k++) {
            if (MODE == 0) FMA(a[k], a[k], m, c);
            if (MODE == 1) ADD(a[k], a[k], c);
            if (MODE == 2) MUL(a[k], a[k], m);
            if (MODE == 3) FMA(a[k], a[k], m, z);     // mul as fma(+0) (z read from memory)
            if (MODE == 4) { if (k < 4) ADD(a[k], a[k], c); else if (k < 8) MUL(a[k], a[k], m); else FMA(a[k], a[k], m, c); }
            if (MODE == 5) { if (k < 4) FMA(a[k], c, m, a[k]); else if (k < 8) FMA(a[k], a[k], m, z); else FMA(a[k], a[k], m, c); }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 13; k++) { float lo, hi; asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[k])); s += lo + hi; }
    if (s == 12345.678f) sink[blockIdx.x] = s;
}
template <int MODE> float run(int iters, const float *in, float *sink, int blocks) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    probe<MODE><<<blocks, 256>>>(iters, in, sink);
    cudaEventRecord(e0);
    probe<MODE><<<blocks, 256>>>(iters, in, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double lane_ops = 2.0 * 13 * iters * (double)blocks * 256;
    return (float)(lane_ops / (ms * 1e-3) / 1e12);  // T lane-ops/s
}
int main() {
    float h[3] = {0.999999f, 1e-7f, 0.0f}; float *in, *sink;
    cudaMalloc(&in, 64); cudaMalloc(&sink, 1 << 20); cudaMemcpy(in, h, 12, cudaMemcpyHostToDevice);
    int blocks = 148 * 8, it = 4096;
    printf("T lane-ops/s: ffma2 %.1f fadd2 %.1f fmul2 %.1f fma2(+0) %.1f mix(4add,4mul,5fma) %.1f allfma %.1f\n",
           run<0>(it, in, sink, blocks), run<1>(it, in, sink, blocks), run<2>(it, in, sink, blocks),
           run<3>(it, in, sink, blocks), run<4>(it, in, sink, blocks), run<5>(it, in, sink, blocks));
    return 0;
}
