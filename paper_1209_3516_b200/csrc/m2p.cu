// m2p.cu -- treecode far field: source-cell multipoles evaluated directly at
// the bodies of each target leaf (src/traversal.py:520-528 ->
// src/_taylor.py:272-307), over the target-sorted CSR M2P list.
//
//   phi(y) += sum_{|m| < p} (-1)^|m| M_m D_m(y - c)
//   f_i(y) -= sum_{|m| < p} (-1)^|m| M_m D_{m+e_i}(y - c)      (f = -grad phi)
//
// with D_k = d^k (1/|r|) for |k| <= p from the reference's recurrence.  A
// body exactly at the cell center is skipped, as in the reference.  Float64,
// or (precision="fp32", p <= 6) float32 D, moments and per-source sums: the
// shift is formed in float64 and rounded once, the running sums stay
// float64.
//
// One warp per target row, one LANE per body (rows of more than 32 bodies
// take several passes); the warp walks the row's source cells together, so
// each source's center and moments are one broadcast load per warp.  Per
// (body, source) the lane forms the source's contribution from zero and
// adds it to its running sums, the reference's per-call `phi[j] += pot`.
//  * m2p_reg<P> (P <= 6): D and the multi-indices at compile time (taylor.cuh).
//  * m2p_gen (any p <= 12): the same recurrence from the runtime tables.
#include <type_traits>

#include "taylor.cuh"

namespace fmm {

template <int P, typename T = double>
__global__ void __launch_bounds__(128) m2p_reg(int32_t ncells, const int64_t *__restrict__ rows,
                                               const int32_t *__restrict__ src,
                                               const int32_t *__restrict__ start,
                                               const int32_t *__restrict__ end,
                                               const double *__restrict__ ctr, const double *__restrict__ M,
                                               const double *__restrict__ x, const double *__restrict__ y,
                                               const double *__restrict__ z, double *phi, double *fx,
                                               double *fy, double *fz) {
    constexpr int NC = ncoef(P);
    constexpr int ND = ncoef(P + 1);  // D up to degree P
    constexpr bool kF32 = std::is_same_v<T, float>;
    // float32 terms: each source's signed moments are converted once per
    // warp into shared memory (lane m converts moment m), not by every lane
    __shared__ float msm[kF32 ? 4 : 1][kF32 ? NC : 1];
    const int lane = threadIdx.x & 31;
    float *mw = msm[kF32 ? (threadIdx.x >> 5) : 0];
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ncells;
         t += (gridDim.x * blockDim.x) >> 5) {
        const int64_t k0 = rows[t], k1 = rows[t + 1];
        if (k0 == k1) continue;
        for (int32_t b0 = start[t]; b0 < end[t]; b0 += 32) {
            const int32_t i = b0 + lane;
            const bool valid = i < end[t];
            const double bx = valid ? x[i] : 0.0, by = valid ? y[i] : 0.0, bz = valid ? z[i] : 0.0;
            double ap = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
            // one source's contribution (zero for a body at its center)
            auto term = [&](int32_t s, double cx, double cy, double cz, T &pot, T &gx, T &gy, T &gz) {
                pot = gx = gy = gz = T(0);
                const double rx = bx - cx, ry = by - cy, rz = bz - cz;
                if (!valid || rx * rx + ry * ry + rz * rz == 0.0) return false;
                T D[ND];
                d_tensors_reg<P + 1, T>(T(rx), T(ry), T(rz), D);
                const double *Ms = M + (int64_t)s * NC;
                static_for<0, NC>([&](auto Im) {
                    constexpr int m = decltype(Im)::value;
                    constexpr int mx = kTab.mi[m][0], my = kTab.mi[m][1], mz = kTab.mi[m][2];
                    constexpr bool odd = kTab.deg[m] & 1;
                    T mm;
                    if constexpr (kF32) mm = mw[m];
                    else mm = odd ? -__ldg(&Ms[m]) : __ldg(&Ms[m]);
                    pot += mm * D[m];
                    gx += mm * D[IX(mx + 1, my, mz)];
                    gy += mm * D[IX(mx, my + 1, mz)];
                    gz += mm * D[IX(mx, my, mz + 1)];
                });
                return true;
            };
            auto add = [&](T pot, T gx, T gy, T gz) {
                ap += (double)pot;
                ax -= (double)gx;
                ay -= (double)gy;
                az -= (double)gz;
            };
            // the next source's id and center are fetched one iteration
            // ahead, off the dependent chain of the current one
            int32_t sn = src[k0];
            double cxn = ctr[sn * 3], cyn = ctr[sn * 3 + 1], czn = ctr[sn * 3 + 2];
            for (int64_t k = k0; k < k1; k++) {
                const int32_t s = sn;
                const double cx = cxn, cy = cyn, cz = czn;
                if constexpr (kF32) {
                    __syncwarp();  // the previous source's moments are consumed
                    for (int m = lane; m < NC; m += 32) {
                        const double v = __ldg(&M[(int64_t)s * NC + m]);
                        mw[m] = (float)((d_tab.deg[m] & 1) ? -v : v);
                    }
                    __syncwarp();
                }
                if (k + 1 < k1) {
                    sn = src[k + 1];
                    cxn = ctr[sn * 3];
                    cyn = ctr[sn * 3 + 1];
                    czn = ctr[sn * 3 + 2];
                }
                T p0, x0, y0, z0;
                if (term(s, cx, cy, cz, p0, x0, y0, z0)) add(p0, x0, y0, z0);
            }
            if (valid) {
                phi[i] += ap;
                fx[i] += ax;
                fy[i] += ay;
                fz[i] += az;
            }
        }
    }
}

// Runtime-table recurrence (src/_taylor.py:57-95) into a per-thread array.
__device__ void d_tensors_rt(double rx, double ry, double rz, int deg, double *D) {
    const double r2 = rx * rx + ry * ry + rz * rz;
    const double inv_r2 = 1.0 / r2;
    D[0] = sqrt(inv_r2);
    const int nd = ncoef(deg + 1);
    for (int idx = 1; idx < nd; idx++) {
        const int kx = d_tab.mi[idx][0], ky = d_tab.mi[idx][1], kz = d_tab.mi[idx][2];
        double acc = 0.0;
        if (kx > 0) {
            acc -= (2.0 * kx - 1.0) * rx * D[d_tab.idx3[kx - 1][ky][kz]];
            if (kx > 1) acc -= (kx - 1.0) * (kx - 1.0) * D[d_tab.idx3[kx - 2][ky][kz]];
            if (ky > 0) {
                acc -= 2.0 * ky * ry * D[d_tab.idx3[kx][ky - 1][kz]];
                if (ky > 1) acc -= ky * (ky - 1.0) * D[d_tab.idx3[kx][ky - 2][kz]];
            }
            if (kz > 0) {
                acc -= 2.0 * kz * rz * D[d_tab.idx3[kx][ky][kz - 1]];
                if (kz > 1) acc -= kz * (kz - 1.0) * D[d_tab.idx3[kx][ky][kz - 2]];
            }
        } else if (ky > 0) {
            acc -= (2.0 * ky - 1.0) * ry * D[d_tab.idx3[kx][ky - 1][kz]];
            if (ky > 1) acc -= (ky - 1.0) * (ky - 1.0) * D[d_tab.idx3[kx][ky - 2][kz]];
            if (kz > 0) {
                acc -= 2.0 * kz * rz * D[d_tab.idx3[kx][ky][kz - 1]];
                if (kz > 1) acc -= kz * (kz - 1.0) * D[d_tab.idx3[kx][ky][kz - 2]];
            }
        } else {
            acc -= (2.0 * kz - 1.0) * rz * D[d_tab.idx3[kx][ky][kz - 1]];
            if (kz > 1) acc -= (kz - 1.0) * (kz - 1.0) * D[d_tab.idx3[kx][ky][kz - 2]];
        }
        D[idx] = acc * inv_r2;
    }
}

__global__ void __launch_bounds__(128) m2p_gen(int p, int32_t ncells, const int64_t *__restrict__ rows,
                                               const int32_t *__restrict__ src, const int32_t *__restrict__ start,
                                               const int32_t *__restrict__ end, const double *__restrict__ ctr,
                                               const double *__restrict__ M, const double *__restrict__ x,
                                               const double *__restrict__ y, const double *__restrict__ z,
                                               double *phi, double *fx, double *fy, double *fz) {
    const int nc = ncoef(p);
    const int lane = threadIdx.x & 31;
    double D[NMI];
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ncells;
         t += (gridDim.x * blockDim.x) >> 5) {
        const int64_t k0 = rows[t], k1 = rows[t + 1];
        if (k0 == k1) continue;
        for (int32_t b0 = start[t]; b0 < end[t]; b0 += 32) {
            const int32_t i = b0 + lane;
            const bool valid = i < end[t];
            const double bx = valid ? x[i] : 0.0, by = valid ? y[i] : 0.0, bz = valid ? z[i] : 0.0;
            double ap = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
            for (int64_t k = k0; k < k1; k++) {
                const int32_t s = src[k];
                const double rx = bx - ctr[s * 3], ry = by - ctr[s * 3 + 1], rz = bz - ctr[s * 3 + 2];
                if (!valid || rx * rx + ry * ry + rz * rz == 0.0) continue;
                d_tensors_rt(rx, ry, rz, p, D);
                const double *Ms = M + (int64_t)s * nc;
                double pot = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
                for (int m = 0; m < nc; m++) {
                    const int mx = d_tab.mi[m][0], my = d_tab.mi[m][1], mz = d_tab.mi[m][2];
                    const double mm = (d_tab.deg[m] & 1) ? -__ldg(&Ms[m]) : __ldg(&Ms[m]);
                    pot += mm * D[m];
                    gx += mm * D[d_tab.idx3[mx + 1][my][mz]];
                    gy += mm * D[d_tab.idx3[mx][my + 1][mz]];
                    gz += mm * D[d_tab.idx3[mx][my][mz + 1]];
                }
                ap += pot;
                ax -= gx;
                ay -= gy;
                az -= gz;
            }
            if (valid) {
                phi[i] += ap;
                fx[i] += ax;
                fy[i] += ay;
                fz[i] += az;
            }
        }
    }
}

}  // namespace fmm

using namespace fmm;

extern "C" int fmm_m2p_csr(int p, int precision, int32_t ncells, const int64_t *rows, const int32_t *src, const int32_t *start,
                           const int32_t *end, const double *ctr, const double *M, const double *x,
                           const double *y, const double *z, double *phi, double *fx, double *fy, double *fz,
                           void *stream) {
    if (p < 1 || p > TMAX) {
        set_error("m2p: p must be in [1, %d], got %d", TMAX, p);
        return FMM_ERR_INVALID;
    }
    if (ncells <= 0) return FMM_OK;
    cudaStream_t s = as_stream(stream);
    const int grid = grid_for((int64_t)ncells * 32, 128, 148 * 16);
#define M2P_REG(PP)                                                                                           \
    case PP:                                                                                                  \
        if (precision == FMM_PREC_FP32)                                                                       \
            m2p_reg<PP, float><<<grid, 128, 0, s>>>(ncells, rows, src, start, end, ctr, M, x, y, z, phi, fx, fy, \
                                                    fz);                                                      \
        else                                                                                                  \
            m2p_reg<PP><<<grid, 128, 0, s>>>(ncells, rows, src, start, end, ctr, M, x, y, z, phi, fx, fy, fz); \
        break;
    switch (p) {
        M2P_REG(1)
        M2P_REG(2)
        M2P_REG(3)
        M2P_REG(4)
        M2P_REG(5)
        M2P_REG(6)
        default:
            m2p_gen<<<grid, 128, 0, s>>>(p, ncells, rows, src, start, end, ctr, M, x, y, z, phi, fx, fy, fz);
    }
#undef M2P_REG
    fmm::note_launch();
    FMM_CUDA_CHECK("fmm_m2p_csr");
    return FMM_OK;
}
