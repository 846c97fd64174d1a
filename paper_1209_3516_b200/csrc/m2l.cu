// m2l.cu -- multipole-to-local conversion over the target-sorted CSR list
// (src/traversal.py:500-517 -> src/_taylor.py:169-188, :57-95).
//
//   L_n += (1/n!) sum_{|m| < p-|n|} (-1)^|m| M_m D_{m+n}(r),  r = c_t - c_s
//
// with D_k = d^k (1/|r|) generated per pair by the reference's degree-by-
// degree recurrence (no stored translation operators).  Float64.
//
// Two kernels:
//  * m2l_reg<P> (P <= 5): one warp per target row, one LANE per (t, s) pair;
//    D, M_s and the per-lane L partial sums live in registers, every
//    multi-index resolves at compile time; the 32 partial sums are folded
//    with shuffles at row end and added once to L_t.
//  * m2l_warp (any p <= 12): one warp per target row, the warp handles one
//    pair at a time -- lanes split each degree of the D recurrence, then
//    lanes own output coefficients; D and M_s staged in shared memory.
#include <type_traits>

#include "fmm_common.cuh"

namespace fmm {

// ---- register kernel, compile-time multi-indices ------------------------
// static_for hands each iteration its index as a type, so every table
// lookup below is a constant expression and D / M / L stay in registers.
template <int B, int E, class F>
__device__ __forceinline__ void static_for(F &&f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + 1, E>(f);
    }
}

#define IX(a, b, c) (std::integral_constant<int, kTab.idx3[a][b][c]>::value)

template <int P>
__device__ __forceinline__ void d_tensors_reg(double rx, double ry, double rz, double (&D)[ncoef(P)]) {
    const double r2 = rx * rx + ry * ry + rz * rz;
    const double inv_r2 = 1.0 / r2;
    D[0] = sqrt(inv_r2);
    static_for<1, ncoef(P)>([&](auto I) {
        constexpr int idx = decltype(I)::value;
        constexpr int kx = kTab.mi[idx][0], ky = kTab.mi[idx][1], kz = kTab.mi[idx][2];
        double acc = 0.0;
        if constexpr (kx > 0) {
            acc -= (2.0 * kx - 1.0) * rx * D[IX(kx - 1, ky, kz)];
            if constexpr (kx > 1) acc -= (kx - 1.0) * (kx - 1.0) * D[IX(kx - 2, ky, kz)];
            if constexpr (ky > 0) {
                acc -= 2.0 * ky * ry * D[IX(kx, ky - 1, kz)];
                if constexpr (ky > 1) acc -= ky * (ky - 1.0) * D[IX(kx, ky - 2, kz)];
            }
            if constexpr (kz > 0) {
                acc -= 2.0 * kz * rz * D[IX(kx, ky, kz - 1)];
                if constexpr (kz > 1) acc -= kz * (kz - 1.0) * D[IX(kx, ky, kz - 2)];
            }
        } else if constexpr (ky > 0) {
            acc -= (2.0 * ky - 1.0) * ry * D[IX(kx, ky - 1, kz)];
            if constexpr (ky > 1) acc -= (ky - 1.0) * (ky - 1.0) * D[IX(kx, ky - 2, kz)];
            if constexpr (kz > 0) {
                acc -= 2.0 * kz * rz * D[IX(kx, ky, kz - 1)];
                if constexpr (kz > 1) acc -= kz * (kz - 1.0) * D[IX(kx, ky, kz - 2)];
            }
        } else {
            acc -= (2.0 * kz - 1.0) * rz * D[IX(kx, ky, kz - 1)];
            if constexpr (kz > 1) acc -= (kz - 1.0) * (kz - 1.0) * D[IX(kx, ky, kz - 2)];
        }
        D[idx] = acc * inv_r2;
    });
}

template <int P>
__global__ void __launch_bounds__(128) m2l_reg(int32_t ncells, const int64_t *__restrict__ rows,
                                               const int32_t *__restrict__ src,
                                               const double *__restrict__ ctr,
                                               const double *__restrict__ M, double *L) {
    constexpr int NC = ncoef(P);
    const int lane = threadIdx.x & 31;
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ncells;
         t += (gridDim.x * blockDim.x) >> 5) {
        const int64_t k0 = rows[t], k1 = rows[t + 1];
        if (k0 == k1) continue;
        const double cx = ctr[t * 3], cy = ctr[t * 3 + 1], cz = ctr[t * 3 + 2];
        double acc[NC];
#pragma unroll
        for (int n = 0; n < NC; n++) acc[n] = 0.0;
        for (int64_t k = k0 + lane; k < k1; k += 32) {
            const int32_t s = src[k];
            double D[NC];
            d_tensors_reg<P>(cx - ctr[s * 3], cy - ctr[s * 3 + 1], cz - ctr[s * 3 + 2], D);
            double Ms[NC];
#pragma unroll
            for (int m = 0; m < NC; m++) Ms[m] = __ldg(&M[(int64_t)s * NC + m]);
            static_for<0, NC>([&](auto In) {
                constexpr int n = decltype(In)::value;
                double a = 0.0;
                static_for<0, ncoef(P - kTab.deg[n])>([&](auto Im) {
                    constexpr int m = decltype(Im)::value;
                    constexpr int j = kTab.idx3[kTab.mi[n][0] + kTab.mi[m][0]][kTab.mi[n][1] + kTab.mi[m][1]]
                                               [kTab.mi[n][2] + kTab.mi[m][2]];
                    if constexpr (kTab.deg[m] & 1) a -= Ms[m] * D[j];
                    else a += Ms[m] * D[j];
                });
                acc[n] += a;
            });
        }
#pragma unroll
        for (int n = 0; n < NC; n++) {
            double v = acc[n];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            acc[n] = v;
        }
        if (lane == 0) {
            static_for<0, NC>([&](auto In) {
                constexpr int n = decltype(In)::value;
                constexpr double inv = 1.0 / kTab.mfact[n];
                L[(int64_t)t * NC + n] += acc[n] * inv;
            });
        }
    }
}

// ---- generic warp kernel ------------------------------------------------
constexpr int kM2LWarps = 4;
constexpr int kMaxSlots = (NMI + 31) / 32;

__global__ void __launch_bounds__(kM2LWarps * 32) m2l_warp(int p, int32_t ncells,
                                                           const int64_t *__restrict__ rows,
                                                           const int32_t *__restrict__ src,
                                                           const double *__restrict__ ctr,
                                                           const double *__restrict__ M, double *L) {
    __shared__ double sD[kM2LWarps][NMI];
    __shared__ double sM[kM2LWarps][NMI];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nc = ncoef(p);
    double *D = sD[w];
    double *Ms = sM[w];
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ncells;
         t += (gridDim.x * blockDim.x) >> 5) {
        const int64_t k0 = rows[t], k1 = rows[t + 1];
        if (k0 == k1) continue;
        const double cx = ctr[t * 3], cy = ctr[t * 3 + 1], cz = ctr[t * 3 + 2];
        double acc[kMaxSlots];
#pragma unroll
        for (int q = 0; q < kMaxSlots; q++) acc[q] = 0.0;
        for (int64_t k = k0; k < k1; k++) {
            const int32_t s = src[k];
            const double rx = cx - ctr[s * 3], ry = cy - ctr[s * 3 + 1], rz = cz - ctr[s * 3 + 2];
            const double r2 = rx * rx + ry * ry + rz * rz;
            const double inv_r2 = 1.0 / r2;
            __syncwarp();
            for (int m = lane; m < nc; m += 32) Ms[m] = M[(int64_t)s * nc + m];
            if (lane == 0) D[0] = sqrt(inv_r2);
            __syncwarp();
            for (int d = 1; d < p; d++) {
                for (int idx = ncoef(d) + lane; idx < ncoef(d + 1); idx += 32) {
                    const int kx = d_tab.mi[idx][0], ky = d_tab.mi[idx][1], kz = d_tab.mi[idx][2];
                    double a = 0.0;
                    if (kx > 0) {
                        a -= (2.0 * kx - 1.0) * rx * D[d_tab.idx3[kx - 1][ky][kz]];
                        if (kx > 1) a -= (kx - 1.0) * (kx - 1.0) * D[d_tab.idx3[kx - 2][ky][kz]];
                        if (ky > 0) {
                            a -= 2.0 * ky * ry * D[d_tab.idx3[kx][ky - 1][kz]];
                            if (ky > 1) a -= ky * (ky - 1.0) * D[d_tab.idx3[kx][ky - 2][kz]];
                        }
                        if (kz > 0) {
                            a -= 2.0 * kz * rz * D[d_tab.idx3[kx][ky][kz - 1]];
                            if (kz > 1) a -= kz * (kz - 1.0) * D[d_tab.idx3[kx][ky][kz - 2]];
                        }
                    } else if (ky > 0) {
                        a -= (2.0 * ky - 1.0) * ry * D[d_tab.idx3[kx][ky - 1][kz]];
                        if (ky > 1) a -= (ky - 1.0) * (ky - 1.0) * D[d_tab.idx3[kx][ky - 2][kz]];
                        if (kz > 0) {
                            a -= 2.0 * kz * rz * D[d_tab.idx3[kx][ky][kz - 1]];
                            if (kz > 1) a -= kz * (kz - 1.0) * D[d_tab.idx3[kx][ky][kz - 2]];
                        }
                    } else {
                        a -= (2.0 * kz - 1.0) * rz * D[d_tab.idx3[kx][ky][kz - 1]];
                        if (kz > 1) a -= (kz - 1.0) * (kz - 1.0) * D[d_tab.idx3[kx][ky][kz - 2]];
                    }
                    D[idx] = a * inv_r2;
                }
                __syncwarp();
            }
#pragma unroll
            for (int q = 0; q < kMaxSlots; q++) {
                const int n = lane + 32 * q;
                if (n < nc) {
                    const int nx = d_tab.mi[n][0], ny = d_tab.mi[n][1], nz = d_tab.mi[n][2];
                    const int lim = ncoef(p - d_tab.deg[n]);
                    double a = 0.0;
                    for (int m = 0; m < lim; m++) {
                        const double term =
                            Ms[m] * D[d_tab.idx3[nx + d_tab.mi[m][0]][ny + d_tab.mi[m][1]][nz + d_tab.mi[m][2]]];
                        if (d_tab.deg[m] & 1) a -= term;
                        else a += term;
                    }
                    acc[q] += a;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < kMaxSlots; q++) {
            const int n = lane + 32 * q;
            if (n < nc) L[(int64_t)t * nc + n] += acc[q] / d_tab.mfact[n];
        }
    }
}

}  // namespace fmm

using namespace fmm;

extern "C" int fmm_m2l_csr(int p, int32_t ncells, const int64_t *rows, const int32_t *src,
                           const double *ctr, const double *M, double *L, void *stream) {
    if (p < 1 || p > TMAX) { set_error("expansion order %d outside supported range 1..%d", p, TMAX); return FMM_ERR_INVALID; }
    cudaStream_t s = as_stream(stream);
    const int grid = grid_for((int64_t)ncells * 32, 128, 148 * 16);
    switch (p) {
        case 1: m2l_reg<1><<<grid, 128, 0, s>>>(ncells, rows, src, ctr, M, L); fmm::note_launch(); break;
        case 2: m2l_reg<2><<<grid, 128, 0, s>>>(ncells, rows, src, ctr, M, L); fmm::note_launch(); break;
        case 3: m2l_reg<3><<<grid, 128, 0, s>>>(ncells, rows, src, ctr, M, L); fmm::note_launch(); break;
        case 4: m2l_reg<4><<<grid, 128, 0, s>>>(ncells, rows, src, ctr, M, L); fmm::note_launch(); break;
        case 5: m2l_reg<5><<<grid, 128, 0, s>>>(ncells, rows, src, ctr, M, L); fmm::note_launch(); break;
        default:
            m2l_warp<<<grid_for((int64_t)ncells * 32, kM2LWarps * 32, 148 * 16), kM2LWarps * 32, 0, s>>>(
                p, ncells, rows, src, ctr, M, L); fmm::note_launch();
    }
    FMM_CUDA_CHECK("fmm_m2l_csr");
    return FMM_OK;
}
