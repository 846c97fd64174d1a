// m2l.cu -- multipole-to-local conversion over the target-sorted CSR list
// (src/traversal.py:500-517 -> src/_taylor.py:169-188, :57-95).
//
//   L_n += (1/n!) sum_{|m| < p-|n|} (-1)^|m| M_m D_{m+n}(r),  r = c_t - c_s
//
// with D_k = d^k (1/|r|) generated per pair by the reference's degree-by-
// degree recurrence (no stored translation operators).  Float64.
//
// Two kernels:
//  * m2l_reg<P> (P <= 7): one warp per target row, one LANE per (t, s) pair;
//    D and the per-lane L partial sums live in registers (for P >= 5 the
//    source moments stream through, P <= 4 keeps them in registers too),
//    every multi-index resolves at compile time; the 32 partial sums are
//    folded with shuffles at row end and added once to L_t.
//  * m2l_smem<8>: lane per pair with D in a thread-private shared-memory
//    row and the outputs in two register passes (below).
//  * m2l_lanes<P> (9 <= P <= 12): one block per target row, one WARP per
//    pair; lanes split each degree of the D recurrence (a shared-memory
//    recipe per entry), then own output coefficients and walk contiguous
//    (|m|, m_x) term rows -- see below.
// For 8 <= P <= 10 on lattice trees the evaluation takes the offset-grouped
// tensor-pipe form instead (m2l_grouped.cu, fmm_m2l_grouped).
#include "taylor.cuh"

#ifndef FMM_M2L_VEC
#define FMM_M2L_VEC 1
#endif



namespace fmm {

// ---- register kernel, compile-time multi-indices (taylor.cuh) -----------
// L partial sums += the pair's contraction (src/_taylor.py:169-188), all
// multi-indices compile-time.  Moments-outer streams the source's moments
// one at a time (fewer live registers); outputs-outer keeps them in registers.
template <int P>
__device__ __forceinline__ void m2l_contract_mouter(const double *__restrict__ Mrow, const double (&D)[ncoef(P)],
                                                    double (&acc)[ncoef(P)]) {
#if FMM_M2L_VEC
    // 16 B loads from the row's 16 B-aligned window (an odd-length row starts
    // 8 B into it for odd cells): element m is window element m + odd
    const bool odd = (reinterpret_cast<uintptr_t>(Mrow) & 15u) != 0;
    const double2 *win = reinterpret_cast<const double2 *>(Mrow - (odd ? 1 : 0));
#endif
    static_for<0, ncoef(P)>([&](auto Im) {
        constexpr int m = decltype(Im)::value;
#if FMM_M2L_VEC
        const double2 we = __ldg(&win[m >> 1]), wo = __ldg(&win[(m + 1) >> 1]);
        const double me = (m & 1) ? we.y : we.x, mo = ((m + 1) & 1) ? wo.y : wo.x;
        const double raw = odd ? mo : me;
        const double mm = (kTab.deg[m] & 1) ? -raw : raw;
#else
        const double mm = (kTab.deg[m] & 1) ? -__ldg(&Mrow[m]) : __ldg(&Mrow[m]);
#endif
        static_for<0, ncoef(P - kTab.deg[m])>([&](auto In) {
            constexpr int n = decltype(In)::value;
            constexpr int j = kTab.idx3[kTab.mi[n][0] + kTab.mi[m][0]][kTab.mi[n][1] + kTab.mi[m][1]]
                                       [kTab.mi[n][2] + kTab.mi[m][2]];
            acc[n] = fma(mm, D[j], acc[n]);
        });
    });
}

template <int P>
__device__ __forceinline__ void m2l_contract_nouter(const double *__restrict__ Mrow, const double (&D)[ncoef(P)],
                                                    double (&acc)[ncoef(P)]) {
    constexpr int NC = ncoef(P);
    double Ms[NC];
#if FMM_M2L_VEC
    if constexpr (NC % 2 == 0) {  // rows of an even count are 16 B aligned: LDG.128
        const double2 *r2 = reinterpret_cast<const double2 *>(Mrow);
#pragma unroll
        for (int q = 0; q < NC / 2; q++) {
            const double2 v = __ldg(&r2[q]);
            Ms[2 * q] = v.x;
            Ms[2 * q + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int m = 0; m < NC; m++) Ms[m] = __ldg(&Mrow[m]);
    }
#else
#pragma unroll
    for (int m = 0; m < NC; m++) Ms[m] = __ldg(&Mrow[m]);
#endif
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

// P = 5 streams the moments (moments-outer order: ~170 registers instead of
// 254); P <= 4 keeps the row of moments in registers (moments-outer was 13 %
// slower there).  Every lane reads its own source's row, so the L1 sees 32
// cache lines per load instruction (90 % L1 throughput at C3,
// profiles/r02_m2l5_ncu_c3.json): the rows are read as 16 B pairs from their
// 16 B-aligned window (odd-length rows of odd cells start 8 B into it), which
// halves the load instructions -- C2 p=4 0.346 -> 0.291 ms, C3 p=5 2.56 ->
// 2.41 ms (FMM_M2L_VEC=0 keeps 8 B loads).
template <int P>
__device__ __forceinline__ void m2l_reg_body(int32_t ncells, const int64_t *__restrict__ rows,
                                             const int32_t *__restrict__ src, const double *__restrict__ ctr,
                                             const double *__restrict__ cs, const double *__restrict__ M,
                                             double *L) {
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
            d_tensors_reg<P>(cx - cs[s * 3], cy - cs[s * 3 + 1], cz - cs[s * 3 + 2], D);
            if constexpr (P >= 5) m2l_contract_mouter<P>(M + (int64_t)s * NC, D, acc);
            else m2l_contract_nouter<P>(M + (int64_t)s * NC, D, acc);
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

template <int P>
__global__ void __launch_bounds__(128) m2l_reg(int32_t ncells, const int64_t *__restrict__ rows,
                                               const int32_t *__restrict__ src, const double *__restrict__ ctr,
                                               const double *__restrict__ cs, const double *__restrict__ M,
                                               double *L) {
    m2l_reg_body<P>(ncells, rows, src, ctr, cs, M, L);
}

#ifndef FMM_M2L_REG5_MINB
#define FMM_M2L_REG5_MINB 1
#endif
__global__ void __launch_bounds__(128, FMM_M2L_REG5_MINB) m2l_reg5(int32_t ncells, const int64_t *__restrict__ rows,
                                                                  const int32_t *__restrict__ src,
                                                                  const double *__restrict__ ctr,
                                                                  const double *__restrict__ cs,
                                                                  const double *__restrict__ M, double *L) {
    m2l_reg_body<5>(ncells, rows, src, ctr, cs, M, L);
}

// ---- p >= 8: lane per pair, D in shared memory, outputs in G passes -------
// The register kernel's per-lane state (D and every output's sum) outgrows
// the register file from p = 8.  Here each lane keeps its pair's D in a
// thread-private shared-memory row (odd stride: conflict-free) and the
// target row is swept G times, each pass owning one slice of the outputs
// in registers and recomputing D per pair (the recurrence is ~1/5 of the
// contraction's work at p = 10).
__host__ __device__ constexpr int m2l_smem_groups(int P) { return (ncoef(P) + 59) / 60; }  // 60 outputs per pass
__host__ __device__ constexpr int m2l_smem_stride(int P) { return ncoef(P) | 1; }
constexpr int kM2LSmemThreads = 64;

template <int P, int N0, int N1, int M>
__host__ __device__ constexpr bool m2l_group_uses(void) {
    for (int n = N0; n < N1; n++)
        if (kTab.deg[n] + kTab.deg[M] <= P - 1) return true;
    return false;
}

template <int P>
__global__ void __launch_bounds__(kM2LSmemThreads) m2l_smem(int32_t ncells, const int64_t *__restrict__ rows,
                                                            const int32_t *__restrict__ src,
                                                            const double *__restrict__ ctr,
                                                            const double *__restrict__ cs,
                                                            const double *__restrict__ M, double *L) {
    constexpr int NC = ncoef(P), S = m2l_smem_stride(P), G = m2l_smem_groups(P);
    extern __shared__ double dsm[];
    double *D = dsm + threadIdx.x * S;
    const int lane = threadIdx.x & 31;
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ncells; t += (gridDim.x * blockDim.x) >> 5) {
        const int64_t k0 = rows[t], k1 = rows[t + 1];
        if (k0 == k1) continue;
        const double cx = ctr[t * 3], cy = ctr[t * 3 + 1], cz = ctr[t * 3 + 2];
        static_for<0, G>([&](auto Ig) {
            constexpr int g = decltype(Ig)::value;
            constexpr int n0 = g * NC / G, n1 = (g + 1) * NC / G;
            double acc[n1 - n0];
#pragma unroll
            for (int i = 0; i < n1 - n0; i++) acc[i] = 0.0;
            for (int64_t k = k0 + lane; k < k1; k += 32) {
                const int32_t s = src[k];
                d_tensors_ptr<P>(cx - cs[s * 3], cy - cs[s * 3 + 1], cz - cs[s * 3 + 2], D);
                const double *Mrow = M + (int64_t)s * NC;
                static_for<0, NC>([&](auto Im) {
                    constexpr int m = decltype(Im)::value;
                    if constexpr (m2l_group_uses<P, n0, n1, m>()) {
                        const double mm = (kTab.deg[m] & 1) ? -__ldg(&Mrow[m]) : __ldg(&Mrow[m]);
                        static_for<n0, n1>([&](auto In) {
                            constexpr int n = decltype(In)::value;
                            if constexpr (kTab.deg[n] + kTab.deg[m] <= P - 1) {
                                constexpr int j = kTab.idx3[kTab.mi[n][0] + kTab.mi[m][0]]
                                                           [kTab.mi[n][1] + kTab.mi[m][1]]
                                                           [kTab.mi[n][2] + kTab.mi[m][2]];
                                acc[n - n0] = fma(mm, D[j], acc[n - n0]);
                            }
                        });
                    }
                });
            }
            static_for<n0, n1>([&](auto In) {
                constexpr int n = decltype(In)::value;
                double v = acc[n - n0];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                constexpr double inv = 1.0 / kTab.mfact[n];
                if (lane == 0) L[(int64_t)t * NC + n] += v * inv;
            });
        });
    }
}

// ---- high orders (P >= 6): lanes own outputs ------------------------------
// One CTA (4 warps) per target row; warp w takes the row's pairs w, w+4, ...
// Per pair the warp stages the parity-signed moments and D (degrees < P,
// the reference's recurrence, src/_taylor.py:57-95) in its shared-memory
// slice.  Lane l owns the outputs n = l + 32 i (graded-lex order, so one
// slot i spans few degrees) and accumulates them over all its pairs in
// registers.  For output n the terms group into rows of fixed (|m|, m_x):
// along a row m steps (m_x, |m|-m_x-t, t) and n + m steps (n_x+m_x, ., n_z+t),
// so both operands are CONTIGUOUS runs -- idx(v) = ncoef(|v|) + tri(|v| -
// v_x) + v_z -- and the M run is the same for every lane (broadcast).  Rows
// and run lengths are compile-time; only each lane's D offset is computed.
// The four warps' partials are folded in a fixed order: deterministic.
__host__ __device__ constexpr int tri(int a) { return a * (a + 1) / 2; }

#ifndef FMM_M2L_WARPS
#define FMM_M2L_WARPS 8
#endif
#ifndef FMM_M2L_ACC
#define FMM_M2L_ACC 1
#endif
constexpr int kM2LAcc = FMM_M2L_ACC;  // independent FMA chains per output
// warps per row CTA: FMM_M2L_WARPS while three NC-double slices per warp fit
// the 48 KB of static shared memory, else 4
__host__ __device__ constexpr int m2l_warps(int P) {
    return ncoef(P) * 3 * 8 * FMM_M2L_WARPS <= 44000 ? FMM_M2L_WARPS : 4;
}

template <int P, int kM2LWarps = m2l_warps(P)>
__global__ void __launch_bounds__(kM2LWarps * 32) m2l_lanes(int32_t ncells, const int64_t *__restrict__ rows,
                                                 const int32_t *__restrict__ src, const double *__restrict__ ctr,
                                                 const double *__restrict__ cs, const double *__restrict__ M,
                                                 double *L) {
    constexpr int NC = ncoef(P);
    constexpr int NS = (NC + 31) / 32;
    __shared__ double sM[kM2LWarps][NC];
    __shared__ double sD[kM2LWarps][NC];
    __shared__ double red[kM2LWarps][NC];
    __shared__ DRecipe rec[NC];
    __shared__ double sgn[NC];
    for (int i = threadIdx.x; i < NC; i += blockDim.x) {
        rec[i] = make_recipe(i);
        sgn[i] = (d_tab.deg[i] & 1) ? -1.0 : 1.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double *Ms = sM[w], *D = sD[w];
    for (int32_t t = blockIdx.x; t < ncells; t += gridDim.x) {
        const int64_t k0 = rows[t], k1 = rows[t + 1];
        if (k0 == k1) continue;
        const double cx = ctr[t * 3], cy = ctr[t * 3 + 1], cz = ctr[t * 3 + 2];
        double acc[NS];
#pragma unroll
        for (int i = 0; i < NS; i++) acc[i] = 0.0;
        for (int64_t k = k0 + w; k < k1; k += kM2LWarps) {
            const int32_t s = src[k];
            for (int m = lane; m < NC; m += 32) Ms[m] = sgn[m] * __ldg(&M[(int64_t)s * NC + m]);
            const double r[3] = {cx - cs[s * 3], cy - cs[s * 3 + 1], cz - cs[s * 3 + 2]};
            const double inv_r2 = 1.0 / (r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
            if (lane == 0) D[0] = sqrt(inv_r2);
            __syncwarp();
#pragma unroll
            for (int d = 1; d < P; d++) {
                for (int idx = ncoef(d) + lane; idx < ncoef(d + 1); idx += 32) {
                    const DRecipe q = rec[idx];
                    const int pv = q.pivot;
                    double a = 0.0;
#pragma unroll
                    for (int ax = 0; ax < 3; ax++) {
                        if (q.i1[ax] < 0) continue;
                        const double kk = (double)q.k[ax];
                        a -= (ax == pv ? 2.0 * kk - 1.0 : 2.0 * kk) * r[ax] * D[q.i1[ax]];
                        if (q.i2[ax] >= 0) a -= (ax == pv ? (kk - 1.0) * (kk - 1.0) : kk * (kk - 1.0)) * D[q.i2[ax]];
                    }
                    D[idx] = a * inv_r2;
                }
                __syncwarp();
            }
#pragma unroll 1
            for (int i = 0; i < NS; i++) {
                const int n = 32 * i + lane;
                const bool valid = n < NC;
                const int nn = valid ? n : 0;
                const DRecipe qn = rec[nn];
                const int nx = qn.k[0], nz = qn.k[2];
                const int dn = valid ? qn.k[0] + qn.k[1] + qn.k[2] : P;
                double a[kM2LAcc];
#pragma unroll
                for (int c = 0; c < kM2LAcc; c++) a[c] = 0.0;
                static_for<0, P>([&](auto Idm) {
                    constexpr int dm = decltype(Idm)::value;
                    if (dn + dm <= P - 1) {
                        const int dv = dn + dm;
                        static_for<0, dm + 1>([&](auto Imx) {
                            constexpr int mx = decltype(Imx)::value;
                            constexpr int bm = ncoef(dm) + tri(dm - mx), len = dm - mx + 1;
                            const int bd = dv * (dv + 1) * (dv + 2) / 6 + tri(dv - nx - mx) + nz;
#pragma unroll
                            for (int u = 0; u < len; u++) {
                                constexpr int c0 = (tri(dm) + mx) % kM2LAcc;  // rows rotate over the chains
                                double &ac = a[(c0 + u) % kM2LAcc];
                                ac = fma(Ms[bm + u], D[bd + u], ac);
                            }
                        });
                    }
                });
                double sum = a[0];
#pragma unroll
                for (int c = 1; c < kM2LAcc; c++) sum += a[c];
                acc[i] += sum;
            }
            __syncwarp();  // the warp's slices are rewritten by its next pair
        }
#pragma unroll
        for (int i = 0; i < NS; i++)
            if (32 * i + lane < NC) red[w][32 * i + lane] = acc[i];
        __syncthreads();
        for (int n = threadIdx.x; n < NC; n += blockDim.x) {
            double v = red[0][n];
#pragma unroll
            for (int q = 1; q < kM2LWarps; q++) v += red[q][n];  // fixed order: deterministic
            L[(int64_t)t * NC + n] += v / d_tab.mfact[n];
        }
        __syncthreads();  // red is rewritten by the next row
    }
}


}  // namespace fmm

using namespace fmm;

extern "C" int fmm_m2l_csr(int p, int32_t ncells, const int64_t *rows, const int32_t *src,
                           const double *ctr, const double *ctr_src, const double *M, double *L, void *stream) {
    if (!ctr_src) ctr_src = ctr;  // one tree
    if (p < 1 || p > TMAX) { set_error("expansion order %d outside supported range 1..%d", p, TMAX); return FMM_ERR_INVALID; }
    cudaStream_t s = as_stream(stream);
    const int grid = grid_for((int64_t)ncells * 32, 128, 148 * 16);
    switch (p) {
        case 1: m2l_reg<1><<<grid, 128, 0, s>>>(ncells, rows, src, ctr, ctr_src, M, L); fmm::note_launch(); break;
        case 2: m2l_reg<2><<<grid, 128, 0, s>>>(ncells, rows, src, ctr, ctr_src, M, L); fmm::note_launch(); break;
        case 3: m2l_reg<3><<<grid, 128, 0, s>>>(ncells, rows, src, ctr, ctr_src, M, L); fmm::note_launch(); break;
        case 4: m2l_reg<4><<<grid, 128, 0, s>>>(ncells, rows, src, ctr, ctr_src, M, L); fmm::note_launch(); break;
        case 5: m2l_reg5<<<grid, 128, 0, s>>>(ncells, rows, src, ctr, ctr_src, M, L); fmm::note_launch(); break;
        // p = 6, 7: the register kernel too (moments streamed; D and the sums
        // fill the 255 registers, a few spill to L1): C4 p = 6, theta = 0.3
        // M2L 19.3 -> 1.6 ms, p = 7 13.3 -> 1.9 ms at C2 against m2l_lanes.
        // From p = 8 the register arrays spill wholesale (tens of KB of local
        // memory per thread) and m2l_lanes is 4-6x faster.
        case 6: m2l_reg<6><<<grid, 128, 0, s>>>(ncells, rows, src, ctr, ctr_src, M, L); fmm::note_launch(); break;
        case 7: m2l_reg<7><<<grid, 128, 0, s>>>(ncells, rows, src, ctr, ctr_src, M, L); fmm::note_launch(); break;
#define M2L_LANES(PP)                                                                                 \
    case PP:                                                                                          \
        m2l_lanes<PP><<<grid_for(ncells, 1, 148 * 8), m2l_warps(PP) * 32, 0, s>>>(ncells, rows, src, ctr, ctr_src, M, L); \
        fmm::note_launch();                                                                           \
        break;
        // p = 8: lane per pair with D in shared memory, two output passes
        // (C4 theta = 0.4: 18.4 -> 7.9 ms against m2l_lanes); at p = 10 the
        // per-pass D recurrences cost more than they save (36.6 -> 60-91 ms
        // for 4-9 passes), so p >= 9 stays on m2l_lanes
        case 8: {
            const int shm = kM2LSmemThreads * m2l_smem_stride(8) * (int)sizeof(double);
            cudaFuncSetAttribute(m2l_smem<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, shm);
            m2l_smem<8><<<grid_for((int64_t)ncells * 32, kM2LSmemThreads, 148 * 16), kM2LSmemThreads, shm, s>>>(
                ncells, rows, src, ctr, ctr_src, M, L);
            fmm::note_launch();
            break;
        }
        M2L_LANES(9)
        M2L_LANES(10)
        M2L_LANES(11)
        M2L_LANES(12)
#undef M2L_LANES
        default:
            set_error("expansion order %d outside supported range 1..%d", p, TMAX);
            return FMM_ERR_INVALID;
    }
    FMM_CUDA_CHECK("fmm_m2l_csr");
    return FMM_OK;
}
