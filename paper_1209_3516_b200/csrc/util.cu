// util.cu -- direct-sum checker on the device, result combine, and the
// FP32 FMA throughput probe used as the roofline denominator.
#include "fmm_common.cuh"

namespace fmm {

// Direct sums onto sampled targets (src/_taylor.py:496-528): one block per
// target, threads stride the sources, fixed-order tree reduction.
__global__ void direct_kernel(int64_t n, const double *__restrict__ x, const double *__restrict__ y,
                              const double *__restrict__ z, const double *__restrict__ q, int64_t nt,
                              const int64_t *__restrict__ tidx, double *phi, double *fx, double *fy,
                              double *fz) {
    __shared__ double red[4][256];
    for (int64_t t = blockIdx.x; t < nt; t += gridDim.x) {
        const int64_t i = tidx[t];
        const double xi = x[i], yi = y[i], zi = z[i];
        double pot = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
        for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
            if (j == i) continue;
            const double dx = xi - x[j], dy = yi - y[j], dz = zi - z[j];
            const double r2 = dx * dx + dy * dy + dz * dz;
            if (r2 == 0.0) continue;
            const double rinv = 1.0 / sqrt(r2);
            const double qr = q[j] * rinv;
            const double qr3 = qr * rinv * rinv;
            pot += qr;
            gx += qr3 * dx;
            gy += qr3 * dy;
            gz += qr3 * dz;
        }
        red[0][threadIdx.x] = pot;
        red[1][threadIdx.x] = gx;
        red[2][threadIdx.x] = gy;
        red[3][threadIdx.x] = gz;
        __syncthreads();
        for (int h = blockDim.x / 2; h > 0; h >>= 1) {
            if (threadIdx.x < h)
                for (int c = 0; c < 4; c++) red[c][threadIdx.x] += red[c][threadIdx.x + h];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            phi[t] = red[0][0];
            fx[t] = red[1][0];
            fy[t] = red[2][0];
            fz[t] = red[3][0];
        }
        __syncthreads();
    }
}

__global__ void combine_kernel(int64_t n, const double *a0, const double *a1, const double *a2,
                               const double *a3, double *b0, double *b1, double *b2, double *b3) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        b0[i] += a0[i];
        b1[i] += a1[i];
        b2[i] += a2[i];
        b3[i] += a3[i];
    }
}

// 16 independent FFMA chains per thread: enough ILP to saturate the pipe.
__global__ void ffma_probe_kernel(int iters, float *sink) {
    float a[16];
#pragma unroll
    for (int k = 0; k < 16; k++) a[k] = threadIdx.x * 1e-3f + k;
    const float m = 0.999999f, c = 1e-7f;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 16; k++) a[k] = fmaf(a[k], m, c);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 16; k++) s += a[k];
    if (s == 12345.678f) sink[blockIdx.x] = s;  // keep the chains alive
}

// packed f32x2 FMA (FFMA2 on sm_100a): 8 chains x 2 lanes
__global__ void ffma2_probe_kernel(int iters, float *sink) {
    unsigned long long a[8];
    const float m = 0.999999f, c = 1e-7f;
    unsigned long long mm, cc;
    asm("mov.b64 %0, {%1, %2};" : "=l"(mm) : "f"(m), "f"(m));
    asm("mov.b64 %0, {%1, %2};" : "=l"(cc) : "f"(c), "f"(c));
#pragma unroll
    for (int k = 0; k < 8; k++) {
        float lo = threadIdx.x * 1e-3f + k, hi = lo + 0.5f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(a[k]) : "f"(lo), "f"(hi));
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[k]) : "l"(mm), "l"(cc));
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[k]));
        s += lo + hi;
    }
    if (s == 12345.678f) sink[blockIdx.x] = s;
}

}  // namespace fmm

using namespace fmm;

extern "C" {

int fmm_direct(int64_t n, const double *x, const double *y, const double *z, const double *q, int64_t nt,
               const int64_t *tidx, double *phi, double *fx, double *fy, double *fz, void *stream) {
    if (nt <= 0) return FMM_OK;
    direct_kernel<<<grid_for(nt, 1, 148 * 8), 256, 0, as_stream(stream)>>>(n, x, y, z, q, nt, tidx, phi, fx,
                                                                          fy, fz);
    FMM_CUDA_CHECK("fmm_direct");
    return FMM_OK;
}

int fmm_combine(int64_t n, const double *a_phi, const double *a_fx, const double *a_fy, const double *a_fz,
                double *phi, double *fx, double *fy, double *fz, void *stream) {
    combine_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, a_phi, a_fx, a_fy, a_fz, phi, fx, fy,
                                                                   fz);
    FMM_CUDA_CHECK("fmm_combine");
    return FMM_OK;
}

int fmm_ffma_probe(int packed, int blocks, int iters, float *sink, double *host_flops, void *stream) {
    cudaStream_t s = as_stream(stream);
    if (packed)
        ffma2_probe_kernel<<<blocks, 256, 0, s>>>(iters, sink);
    else
        ffma_probe_kernel<<<blocks, 256, 0, s>>>(iters, sink);
    *host_flops = 2.0 * 16.0 * (double)iters * 256.0 * (double)blocks;
    FMM_CUDA_CHECK("fmm_ffma_probe");
    return FMM_OK;
}

}  // extern "C"
