// p2p.cu -- near-field particle-particle sums over the P2P plan
// (src/traversal.py:531-548 -> src/_taylor.py:366-407).
//
//   phi_i = sum_j q_j / r_ij,   f_i = sum_j q_j (x_i - x_j) / r_ij^3  (= -grad phi)
//
// Decomposition (B200-first): one CTA per target leaf row.
// Targets are register-blocked K per lane (every lane holds the same K
// targets), LANES RUN OVER SOURCES, so lane utilisation does not depend on
// the leaf size; sources stream as contiguous Morton body runs read with
// coalesced float4 (x, y, z, q) loads (L2-resident at C2; the CTA's warps
// share them through L1).  When a leaf has fewer target blocks than the CTA
// has warps, the remaining warps split the source runs and the partial sums
// are folded through shared memory in a fixed order (deterministic).
// Each warp folds its 32 per-lane partial sums with shuffles at row end.
//
// FP32 fast path per pair: 3 FADD, FMUL + 2 FFMA (r2), MUFU.RSQ, FMUL
// (q*rinv), FADD (phi), 2 FMUL (q*rinv^3), 3 FFMA (force) = 13 FP32-pipe
// instructions + 1 SFU; 20 flops under the reference's cost model.  The
// guarded variant (i != j, r2 > 0) is used only for the self run.
#include "fmm_common.cuh"

namespace fmm {

__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

constexpr int kP2PWarps = 4;

// Anchor of a row: sources are re-expressed as (hi - a_hi) + (lo - a_lo),
// accurate to the leaf scale when the float64 inputs are not float32-exact.
struct Anchor {
    float hx, hy, hz, lx, ly, lz;
};

template <int K, bool GUARD, bool ANCHOR>
__device__ __forceinline__ void p2p_f32_span(int32_t j0, int32_t j1, int step, const float4 *__restrict__ b,
                                             const float4 *__restrict__ blo, const Anchor &an,
                                             const float (&tx)[K], const float (&ty)[K],
                                             const float (&tz)[K], const int32_t (&ti)[K], float (&ap)[K],
                                             float (&ax)[K], float (&ay)[K], float (&az)[K]) {
    for (int32_t j = j0; j < j1; j += step) {
        float4 s = __ldg(&b[j]);
        if (ANCHOR) {
            const float4 l = __ldg(&blo[j]);
            s.x = (s.x - an.hx) + (l.x - an.lx);
            s.y = (s.y - an.hy) + (l.y - an.ly);
            s.z = (s.z - an.hz) + (l.z - an.lz);
        }
#pragma unroll
        for (int u = 0; u < K; u++) {
            const float dx = tx[u] - s.x;
            const float dy = ty[u] - s.y;
            const float dz = tz[u] - s.z;
            const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
            float rinv = rsqrt_approx(r2);
            if (GUARD) rinv = (r2 > 0.0f && j != ti[u]) ? rinv : 0.0f;
            const float qr = s.w * rinv;
            const float qr3 = qr * rinv * rinv;
            ap[u] += qr;
            ax[u] = fmaf(qr3, dx, ax[u]);
            ay[u] = fmaf(qr3, dy, ay[u]);
            az[u] = fmaf(qr3, dz, az[u]);
        }
    }
}

template <int K, bool SAFE, bool ANCHOR>
__global__ void __launch_bounds__(kP2PWarps * 32) p2p_f32_kernel(
    int32_t nrows, const int32_t *__restrict__ leaf_rows, const int32_t *__restrict__ start,
    const int32_t *__restrict__ end, const int64_t *__restrict__ run_off, const int4 *__restrict__ runs,
    const float4 *__restrict__ b, const float4 *__restrict__ blo, double *phi, double *fx, double *fy,
    double *fz, int *flag) {
    __shared__ float red[kP2PWarps][4 * K];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int row = blockIdx.x; row < nrows; row += gridDim.x) {
        const int32_t t = leaf_rows[row];
        const int32_t ts = start[t], cnt = end[t] - ts;
        const int nblk = (cnt + K - 1) / K;
        const int nparts = nblk >= kP2PWarps ? 1 : kP2PWarps / nblk;
        const int64_t r0 = run_off[row], r1 = run_off[row + 1];
        const int rounds = (nblk + kP2PWarps - 1) / kP2PWarps;  // nparts == 1 case
        for (int rd = 0; rd < (nparts > 1 ? 1 : rounds); rd++) {
            int tb, part;
            if (nparts > 1) { tb = w % nblk; part = w / nblk; }
            else { tb = rd * kP2PWarps + w; part = 0; }
            const bool active = (nparts > 1) ? (part < nparts) : (tb < nblk);
            float tx[K], ty[K], tz[K], ap[K], ax[K], ay[K], az[K];
            int32_t ti[K];
            if (active) {
                Anchor an{};
                if (ANCHOR) {
                    const float4 h = __ldg(&b[ts]), l = __ldg(&blo[ts]);
                    an = Anchor{h.x, h.y, h.z, l.x, l.y, l.z};
                }
#pragma unroll
                for (int u = 0; u < K; u++) {
                    int32_t i = ts + min(tb * K + u, cnt - 1);
                    float4 v = __ldg(&b[i]);
                    if (ANCHOR) {
                        const float4 l = __ldg(&blo[i]);
                        v.x = (v.x - an.hx) + (l.x - an.lx);
                        v.y = (v.y - an.hy) + (l.y - an.ly);
                        v.z = (v.z - an.hz) + (l.z - an.lz);
                    }
                    tx[u] = v.x; ty[u] = v.y; tz[u] = v.z;
                    ti[u] = i;
                    ap[u] = ax[u] = ay[u] = az[u] = 0.0f;
                }
                const int step = 32 * nparts;
                for (int64_t r = r0; r < r1; r++) {
                    const int4 run = __ldg(&runs[r]);
                    const int32_t j0 = run.x + part * 32 + lane;
                    if (SAFE || run.z)
                        p2p_f32_span<K, true, ANCHOR>(j0, run.y, step, b, blo, an, tx, ty, tz, ti, ap, ax, ay, az);
                    else
                        p2p_f32_span<K, false, ANCHOR>(j0, run.y, step, b, blo, an, tx, ty, tz, ti, ap, ax, ay, az);
                }
#pragma unroll
                for (int u = 0; u < K; u++) {
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        ap[u] += __shfl_xor_sync(0xffffffffu, ap[u], o);
                        ax[u] += __shfl_xor_sync(0xffffffffu, ax[u], o);
                        ay[u] += __shfl_xor_sync(0xffffffffu, ay[u], o);
                        az[u] += __shfl_xor_sync(0xffffffffu, az[u], o);
                    }
                }
            }
            if (nparts > 1) {
                if (active && lane == 0) {
#pragma unroll
                    for (int u = 0; u < K; u++) {
                        red[w][u] = ap[u];
                        red[w][K + u] = ax[u];
                        red[w][2 * K + u] = ay[u];
                        red[w][3 * K + u] = az[u];
                    }
                }
                __syncthreads();
                if (active && part == 0) {
                    // fold parts in fixed order; lane u finalises target u
#pragma unroll
                    for (int u = 0; u < K; u++) {
                        float p_ = 0.f, x_ = 0.f, y_ = 0.f, z_ = 0.f;
                        for (int q = 0; q < nparts; q++) {
                            const int ww = q * nblk + tb;
                            p_ += red[ww][u];
                            x_ += red[ww][K + u];
                            y_ += red[ww][2 * K + u];
                            z_ += red[ww][3 * K + u];
                        }
                        ap[u] = p_; ax[u] = x_; ay[u] = y_; az[u] = z_;
                    }
                }
                __syncthreads();
            }
            if (active && part == 0) {
#pragma unroll
                for (int u = 0; u < K; u++) {
                    if (lane == u && tb * K + u < cnt) {
                        const int32_t i = ts + tb * K + u;
                        phi[i] = (double)ap[u];
                        fx[i] = (double)ax[u];
                        fy[i] = (double)ay[u];
                        fz[i] = (double)az[u];
                        if (!(isfinite(ap[u]) && isfinite(ax[u]) && isfinite(ay[u]) && isfinite(az[u])))
                            atomicOr(flag, 1);
                    }
                }
            }
        }
    }
}

// ---- FP64 variant (parity mode) ------------------------------------------
template <int K>
__global__ void __launch_bounds__(kP2PWarps * 32) p2p_f64_kernel(
    int32_t nrows, const int32_t *__restrict__ leaf_rows, const int32_t *__restrict__ start,
    const int32_t *__restrict__ end, const int64_t *__restrict__ run_off, const int4 *__restrict__ runs,
    const double *__restrict__ xs, const double *__restrict__ ys, const double *__restrict__ zs,
    const double *__restrict__ qs, int use_rsqrt, double *phi, double *fx, double *fy, double *fz) {
    __shared__ double red[kP2PWarps][4 * K];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int row = blockIdx.x; row < nrows; row += gridDim.x) {
        const int32_t t = leaf_rows[row];
        const int32_t ts = start[t], cnt = end[t] - ts;
        const int nblk = (cnt + K - 1) / K;
        const int nparts = nblk >= kP2PWarps ? 1 : kP2PWarps / nblk;
        const int64_t r0 = run_off[row], r1 = run_off[row + 1];
        const int rounds = (nblk + kP2PWarps - 1) / kP2PWarps;
        for (int rd = 0; rd < (nparts > 1 ? 1 : rounds); rd++) {
            int tb, part;
            if (nparts > 1) { tb = w % nblk; part = w / nblk; }
            else { tb = rd * kP2PWarps + w; part = 0; }
            const bool active = (nparts > 1) ? (part < nparts) : (tb < nblk);
            double tx[K], ty[K], tz[K], ap[K], ax[K], ay[K], az[K];
            int32_t ti[K];
            if (active) {
#pragma unroll
                for (int u = 0; u < K; u++) {
                    int32_t i = ts + min(tb * K + u, cnt - 1);
                    tx[u] = xs[i]; ty[u] = ys[i]; tz[u] = zs[i];
                    ti[u] = i;
                    ap[u] = ax[u] = ay[u] = az[u] = 0.0;
                }
                const int step = 32 * nparts;
                for (int64_t r = r0; r < r1; r++) {
                    const int4 run = __ldg(&runs[r]);
                    for (int32_t j = run.x + part * 32 + lane; j < run.y; j += step) {
                        const double sx = xs[j], sy = ys[j], sz = zs[j], sq = qs[j];
#pragma unroll
                        for (int u = 0; u < K; u++) {
                            const double dx = tx[u] - sx, dy = ty[u] - sy, dz = tz[u] - sz;
                            const double r2 = dx * dx + dy * dy + dz * dz;
                            double rinv = use_rsqrt ? (double)(1.0f / sqrtf((float)r2)) : 1.0 / sqrt(r2);
                            rinv = (r2 > 0.0 && j != ti[u]) ? rinv : 0.0;
                            const double qr = sq * rinv;
                            const double qr3 = qr * rinv * rinv;
                            ap[u] += qr;
                            ax[u] += qr3 * dx;
                            ay[u] += qr3 * dy;
                            az[u] += qr3 * dz;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < K; u++) {
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        ap[u] += __shfl_xor_sync(0xffffffffu, ap[u], o);
                        ax[u] += __shfl_xor_sync(0xffffffffu, ax[u], o);
                        ay[u] += __shfl_xor_sync(0xffffffffu, ay[u], o);
                        az[u] += __shfl_xor_sync(0xffffffffu, az[u], o);
                    }
                }
            }
            if (nparts > 1) {
                if (active && lane == 0) {
#pragma unroll
                    for (int u = 0; u < K; u++) {
                        red[w][u] = ap[u];
                        red[w][K + u] = ax[u];
                        red[w][2 * K + u] = ay[u];
                        red[w][3 * K + u] = az[u];
                    }
                }
                __syncthreads();
                if (active && part == 0) {
#pragma unroll
                    for (int u = 0; u < K; u++) {
                        double p_ = 0, x_ = 0, y_ = 0, z_ = 0;
                        for (int q = 0; q < nparts; q++) {
                            const int ww = q * nblk + tb;
                            p_ += red[ww][u];
                            x_ += red[ww][K + u];
                            y_ += red[ww][2 * K + u];
                            z_ += red[ww][3 * K + u];
                        }
                        ap[u] = p_; ax[u] = x_; ay[u] = y_; az[u] = z_;
                    }
                }
                __syncthreads();
            }
            if (active && part == 0) {
#pragma unroll
                for (int u = 0; u < K; u++) {
                    if (lane == u && tb * K + u < cnt) {
                        const int32_t i = ts + tb * K + u;
                        phi[i] = ap[u];
                        fx[i] = ax[u];
                        fy[i] = ay[u];
                        fz[i] = az[u];
                    }
                }
            }
        }
    }
}

}  // namespace fmm

using namespace fmm;

extern "C" int fmm_p2p(int precision, int safe, int use_rsqrt, int32_t nrows, const int32_t *leaf_rows,
                       const int32_t *start, const int32_t *end, const int64_t *run_off, const void *runs,
                       const double *xs, const double *ys, const double *zs, const double *qs,
                       const void *b32, const void *b32lo, double *phi, double *fx, double *fy, double *fz,
                       int *dev_flag, void *stream) {
    if (nrows <= 0) return FMM_OK;
    cudaStream_t s = as_stream(stream);
    const int grid = nrows;
    if (precision == FMM_PREC_FP32 || precision == FMM_PREC_FP32_ANCHORED) {
        if (!b32) { set_error("fp32 P2P needs the float4 body copy"); return FMM_ERR_INVALID; }
        const bool anch = precision == FMM_PREC_FP32_ANCHORED;
        if (anch && !b32lo) { set_error("anchored fp32 P2P needs the float4 residual copy"); return FMM_ERR_INVALID; }
        auto kern = anch ? (safe ? p2p_f32_kernel<8, true, true> : p2p_f32_kernel<8, false, true>)
                         : (safe ? p2p_f32_kernel<8, true, false> : p2p_f32_kernel<8, false, false>);
        kern<<<grid, kP2PWarps * 32, 0, s>>>(nrows, leaf_rows, start, end, run_off, (const int4 *)runs,
                                             (const float4 *)b32, (const float4 *)b32lo, phi, fx, fy, fz,
                                             dev_flag);
    } else if (precision == FMM_PREC_FP64) {
        p2p_f64_kernel<4><<<grid, kP2PWarps * 32, 0, s>>>(nrows, leaf_rows, start, end, run_off,
                                                          (const int4 *)runs, xs, ys, zs, qs, use_rsqrt, phi,
                                                          fx, fy, fz);
    } else {
        set_error("bad precision %d", precision);
        return FMM_ERR_INVALID;
    }
    FMM_CUDA_CHECK("fmm_p2p");
    return FMM_OK;
}
