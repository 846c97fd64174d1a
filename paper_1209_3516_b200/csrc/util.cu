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

__global__ void unpermute_kernel(const int32_t *__restrict__ perm, int64_t n, const double *a0, const double *a1,
                                 const double *a2, const double *a3, double *b0, double *b1, double *b2,
                                 double *b3) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t o = perm[i];
        b0[o] = a0[i];
        b1[o] = a1[i];
        b2[o] = a2[i];
        b3[o] = a3[i];
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

// FP32 pipe probes.  mode 0: FFMA with immediate operands; 1: FFMA2 (packed
// f32x2); 2: FFMA with all-register operands; 3: FFMA2 all-register;
// 4: FMUL/FADD register pairs.  16 independent chains per thread.
template <int MODE>
__global__ void fp32_probe_kernel(int iters, float *sink) {
    float m = 0.999999f, c = 1e-7f;
    if (MODE >= 2) {  // defeat immediate folding: operands come from memory
        m = sink[gridDim.x * 2 + 0] + 0.999999f;
        c = sink[gridDim.x * 2 + 1] + 1e-7f;
    }
    if (MODE == 1 || MODE == 3) {
        unsigned long long a[8], mm, cc;
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
        return;
    }
    float a[16];
#pragma unroll
    for (int k = 0; k < 16; k++) a[k] = threadIdx.x * 1e-3f + k;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 16; k++) {
            if (MODE == 4) a[k] = (k & 1) ? a[k] * m : a[k] + c;
            else a[k] = fmaf(a[k], m, c);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 16; k++) s += a[k];
    if (s == 12345.678f) sink[blockIdx.x] = s;
}

// mode 5..7: the P2P pair math with sources generated in registers (no
// memory): the compute-only ceiling of the near-field instruction mix.
// 5: exact P2P mix (rsqrt.approx); 6: same without the MUFU (rinv = r2);
// 7: mix with FFMA2-packed pairs (two targets per f32x2 lane pair).
template <int MODE>
__global__ void p2p_probe_kernel(int iters, float *sink) {
    constexpr int K = 8;
    float tx[K], ty[K], tz[K], ap[K], ax[K], ay[K], az[K];
    const float base = sink[gridDim.x * 2 + 1];  // runtime value: no immediate folding
#pragma unroll
    for (int u = 0; u < K; u++) {
        tx[u] = base + 0.1f * u + threadIdx.x * 1e-4f; ty[u] = base + 0.2f + 0.01f * u;
        tz[u] = base + 0.3f - 0.02f * u;
        ap[u] = ax[u] = ay[u] = az[u] = 0.f;
    }
    float4 s = make_float4(sink[gridDim.x * 2] + 1.5f, 2.5f, 3.5f, 1.0f);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < K; u++) {
            const float dx = tx[u] - s.x, dy = ty[u] - s.y, dz = tz[u] - s.z;
            const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
            float rinv;
            if (MODE == 6) rinv = r2;
            else asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rinv) : "f"(r2));
            const float qr = s.w * rinv;
            const float qr3 = qr * rinv * rinv;
            ap[u] += qr;
            ax[u] = fmaf(qr3, dx, ax[u]);
            ay[u] = fmaf(qr3, dy, ay[u]);
            az[u] = fmaf(qr3, dz, az[u]);
        }
        s.x += 1e-3f;
    }
    float acc = 0.f;
#pragma unroll
    for (int u = 0; u < K; u++) acc += ap[u] + ax[u] + ay[u] + az[u];
    if (acc == 12345.678f) sink[blockIdx.x] = acc;
}

typedef unsigned long long pf2;
#define PF2_PACK(r, lo, hi) asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi))
#define PF2_UNPACK(v, lo, hi) asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v))

// mode 7: the packed (FFMA2/FADD2/FMUL2) pair math on register sources.
__global__ void p2p_probe_packed_kernel(int iters, float *sink) {
    constexpr int K = 8;
    pf2 tx[K / 2], ty[K / 2], tz[K / 2], ap[K / 2], ax[K / 2], ay[K / 2], az[K / 2];
    const float base = sink[gridDim.x * 2 + 1];
#pragma unroll
    for (int v = 0; v < K / 2; v++) {
        PF2_PACK(tx[v], base + 0.1f * v + threadIdx.x * 1e-4f, base + 0.05f * v);
        PF2_PACK(ty[v], base + 0.2f + 0.01f * v, base + 0.3f);
        PF2_PACK(tz[v], base + 0.3f - 0.02f * v, base + 0.1f);
        ap[v] = ax[v] = ay[v] = az[v] = 0ull;
    }
    float sx = sink[gridDim.x * 2] + 1.5f, sy = 2.5f, sz = 3.5f, sq = 1.0f;
    for (int it = 0; it < iters; it++) {
        pf2 bx, by, bz, bq;
        PF2_PACK(bx, sx, sx); PF2_PACK(by, sy, sy); PF2_PACK(bz, sz, sz); PF2_PACK(bq, sq, sq);
#pragma unroll
        for (int v = 0; v < K / 2; v++) {
            pf2 dx, dy, dz, r2, rinv, qr, rr, qr3;
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dx) : "l"(tx[v]), "l"(bx));
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dy) : "l"(ty[v]), "l"(by));
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dz) : "l"(tz[v]), "l"(bz));
            asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(r2) : "l"(dx));
            asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(r2) : "l"(dy));
            asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(r2) : "l"(dz));
            float a, b;
            PF2_UNPACK(r2, a, b);
            asm("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(a));
            asm("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(b));
            PF2_PACK(rinv, a, b);
            asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(qr) : "l"(rinv), "l"(bq));
            asm("add.rn.f32x2 %0, %0, %1;" : "+l"(ap[v]) : "l"(qr));
            asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(rr) : "l"(rinv));
            asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(qr3) : "l"(qr), "l"(rr));
            asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(ax[v]) : "l"(qr3), "l"(dx));
            asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(ay[v]) : "l"(qr3), "l"(dy));
            asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(az[v]) : "l"(qr3), "l"(dz));
        }
        sx += 1e-3f;
    }
    float acc = 0.f;
#pragma unroll
    for (int v = 0; v < K / 2; v++) {
        float a, b, c, d;
        PF2_UNPACK(ap[v], a, b);
        PF2_UNPACK(ax[v], c, d);
        acc += a + b + c + d;
    }
    if (acc == 12345.678f) sink[blockIdx.x] = acc;
}

}  // namespace fmm

using namespace fmm;

extern "C" {

int fmm_direct(int64_t n, const double *x, const double *y, const double *z, const double *q, int64_t nt,
               const int64_t *tidx, double *phi, double *fx, double *fy, double *fz, void *stream) {
    if (nt <= 0) return FMM_OK;
    direct_kernel<<<grid_for(nt, 1, 148 * 8), 256, 0, as_stream(stream)>>>(n, x, y, z, q, nt, tidx, phi, fx,
                                                                          fy, fz); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_direct");
    return FMM_OK;
}

int fmm_unpermute(const int32_t *perm, int64_t n, const double *a0, const double *a1, const double *a2,
                  const double *a3, double *b0, double *b1, double *b2, double *b3, void *stream) {
    unpermute_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(perm, n, a0, a1, a2, a3, b0, b1, b2, b3); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_unpermute");
    return FMM_OK;
}

int fmm_combine(int64_t n, const double *a_phi, const double *a_fx, const double *a_fy, const double *a_fz,
                double *phi, double *fx, double *fy, double *fz, void *stream) {
    combine_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, a_phi, a_fx, a_fy, a_fz, phi, fx, fy,
                                                                   fz); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_combine");
    return FMM_OK;
}

int fmm_ffma_probe(int mode, int blocks, int iters, float *sink, double *host_flops, void *stream) {
    cudaStream_t s = as_stream(stream);
    switch (mode) {
        case 0: fp32_probe_kernel<0><<<blocks, 256, 0, s>>>(iters, sink); fmm::note_launch(); break;
        case 1: fp32_probe_kernel<1><<<blocks, 256, 0, s>>>(iters, sink); fmm::note_launch(); break;
        case 2: fp32_probe_kernel<2><<<blocks, 256, 0, s>>>(iters, sink); fmm::note_launch(); break;
        case 3: fp32_probe_kernel<3><<<blocks, 256, 0, s>>>(iters, sink); fmm::note_launch(); break;
        case 4: fp32_probe_kernel<4><<<blocks, 256, 0, s>>>(iters, sink); fmm::note_launch(); break;
        case 5: p2p_probe_kernel<5><<<blocks, 256, 0, s>>>(iters, sink); fmm::note_launch(); break;
        case 6: p2p_probe_kernel<6><<<blocks, 256, 0, s>>>(iters, sink); fmm::note_launch(); break;
        case 7: p2p_probe_packed_kernel<<<blocks, 256, 0, s>>>(iters, sink); fmm::note_launch(); break;
        default: set_error("bad probe mode %d", mode); return FMM_ERR_INVALID;
    }
    // flops: FFMA = 2 per lane-op, FMUL/FADD = 1 (mode 4 counts 1 per op);
    // modes 5/6 report 20 flops per pair (8 pairs per iteration)
    if (mode >= 5) *host_flops = 20.0 * 8.0 * (double)iters * 256.0 * (double)blocks;
    else *host_flops = (mode == 4 ? 1.0 : 2.0) * 16.0 * (double)iters * 256.0 * (double)blocks;
    FMM_CUDA_CHECK("fmm_ffma_probe");
    return FMM_OK;
}

}  // extern "C"
