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
#include <stdlib.h>

#include "taylor.cuh"

namespace fmm {

// ---- register kernel, compile-time multi-indices (taylor.cuh) -----------
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

// ---- block kernel for high orders (p >= 6) -------------------------------
// The contraction L_n += sum_m (-1)^|m| M_m D_{n+m} has C(p+5, 6) terms
// (5005 at p = 10).  They are listed n-major, cut into chunks of kChunk
// terms that never straddle two outputs n, and dealt round-robin to the
// block's threads: every thread owns a fixed set of chunks, so the work is
// balanced whatever the output's term count.  Per batch of kWarps pairs,
// warp g builds pair g's parity-signed moments and D tensor in shared
// memory; then every thread runs its chunks over the whole batch.  At row
// end the chunk partials are folded per output in a fixed order
// (deterministic) and added to L_t once.
constexpr int kChunk = 8;
constexpr int kMaxTerms = 12376 + NMI * kChunk;     // C(17,6) + padding, p = 12
constexpr int kMaxChunks = kMaxTerms / kChunk;
constexpr int kBlkWarps = 4;

struct TermTable {
    int p, nchunks, nterms;
    uint32_t term[kMaxTerms];     // m | (j << 16), chunk-major
    uint16_t chunk_n[kMaxChunks];  // output of each chunk
    uint16_t first_chunk[NMI + 1]; // chunks of output n: [first_chunk[n], first_chunk[n+1])
};

static __device__ TermTable d_terms;

static int build_term_table(int p, TermTable &t) {
    const Tables &T = kTab;
    const int nc = ncoef(p);
    int nt = 0, ch = 0;
    t.p = p;
    for (int n = 0; n < nc; n++) {
        t.first_chunk[n] = (uint16_t)ch;
        const int lim = ncoef(p - T.deg[n]);
        int k = 0;
        for (int m = 0; m < lim; m++) {
            const int j = T.idx3[T.mi[n][0] + T.mi[m][0]][T.mi[n][1] + T.mi[m][1]][T.mi[n][2] + T.mi[m][2]];
            t.term[nt++] = (uint32_t)m | ((uint32_t)j << 16);
            if (++k == kChunk) {
                t.chunk_n[ch++] = (uint16_t)n;
                k = 0;
            }
        }
        if (k) {  // pad the last chunk of this output with (m = 0, j = zero slot)
            for (; k < kChunk; k++) t.term[nt++] = 0u | (0xFFFFu << 16);
            t.chunk_n[ch++] = (uint16_t)n;
        }
    }
    t.first_chunk[nc] = (uint16_t)ch;
    t.nchunks = ch;
    t.nterms = nt;
    return ch;
}

template <int NT>
__global__ void __launch_bounds__(NT) m2l_block(int p, int32_t ncells, const int64_t *__restrict__ rows,
                                                const int32_t *__restrict__ src, const double *__restrict__ ctr,
                                                const double *__restrict__ M, double *L) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int G = NT / 32;
    const int nc = ncoef(p);
    const int nch = d_terms.nchunks;
    uint32_t *sterm = (uint32_t *)smem_raw;                    // nch * kChunk
    double *sD = (double *)(sterm + ((nch * kChunk + 1) & ~1)); // G * (nc + 1); slot nc is the zero
    double *sM = sD + G * (nc + 1);                            // G * nc
    double *spart = sM + G * nc;                               // nch
    for (int i = threadIdx.x; i < nch * kChunk; i += NT) {
        uint32_t v = d_terms.term[i];
        if ((v >> 16) == 0xFFFFu) v = (v & 0xFFFFu) | ((uint32_t)nc << 16);  // -> zero slot
        sterm[i] = v;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nslot = (nch + NT - 1) / NT;  // chunks per thread (<= kMaxChunks / NT)
    for (int t = blockIdx.x; t < ncells; t += gridDim.x) {
        const int64_t k0 = rows[t], k1 = rows[t + 1];
        if (k0 == k1) continue;
        const double cx = ctr[t * 3], cy = ctr[t * 3 + 1], cz = ctr[t * 3 + 2];
        double acc[(kMaxChunks + NT - 1) / NT];
#pragma unroll
        for (int q = 0; q < (kMaxChunks + NT - 1) / NT; q++) acc[q] = 0.0;
        for (int64_t kb = k0; kb < k1; kb += G) {
            __syncthreads();  // previous batch consumed (and srec / sterm loaded)
            const int gcount = (int)min((int64_t)G, k1 - kb);
            {   // warp w builds pair w's parity-signed moments and D tensor
                const int64_t k = kb + w;
                double *Ms = sM + w * nc;
                double *D = sD + w * (nc + 1);
                if (w < gcount) {
                    const int32_t s = src[k];
                    for (int m = lane; m < nc; m += 32) {
                        const double v = M[(int64_t)s * nc + m];
                        Ms[m] = (d_tab.deg[m] & 1) ? -v : v;
                    }
                    const double rx = cx - ctr[s * 3], ry = cy - ctr[s * 3 + 1], rz = cz - ctr[s * 3 + 2];
                    const double r2 = rx * rx + ry * ry + rz * rz;
                    const double inv_r2 = 1.0 / r2;
                    if (lane == 0) {
                        D[0] = sqrt(inv_r2);
                        D[nc] = 0.0;
                    }
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
                } else {
                    for (int m = lane; m < nc; m += 32) Ms[m] = 0.0;
                    for (int m = lane; m <= nc; m += 32) D[m] = 0.0;
                }
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < (kMaxChunks + NT - 1) / NT; q++) {
                const int c = threadIdx.x + q * NT;
                if (q < nslot && c < nch) {
                    const uint32_t *tt = sterm + c * kChunk;
                    double a = acc[q];
                    for (int g = 0; g < gcount; g++) {
                        const double *D = sD + g * (nc + 1);
                        const double *Ms = sM + g * nc;
#pragma unroll
                        for (int e = 0; e < kChunk; e++) {
                            const uint32_t v = tt[e];
                            a = fma(Ms[v & 0xFFFFu], D[v >> 16], a);
                        }
                    }
                    acc[q] = a;
                }
            }
        }
        // fold chunk partials per output in a fixed order; one add per L_n
        __syncthreads();
#pragma unroll
        for (int q = 0; q < (kMaxChunks + NT - 1) / NT; q++) {
            const int c = threadIdx.x + q * NT;
            if (q < nslot && c < nch) spart[c] = acc[q];
        }
        __syncthreads();
        for (int n = threadIdx.x; n < nc; n += NT) {
            double v = 0.0;
            for (int c = d_terms.first_chunk[n]; c < d_terms.first_chunk[n + 1]; c++) v += spart[c];
            L[(int64_t)t * nc + n] += v / d_tab.mfact[n];
        }
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

template <int P>
__global__ void __launch_bounds__(128) m2l_lanes(int32_t ncells, const int64_t *__restrict__ rows,
                                                 const int32_t *__restrict__ src, const double *__restrict__ ctr,
                                                 const double *__restrict__ M, double *L) {
    constexpr int NC = ncoef(P);
    constexpr int NS = (NC + 31) / 32;
    __shared__ double sM[4][NC];
    __shared__ double sD[4][NC];
    __shared__ double red[4][NC];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double *Ms = sM[w], *D = sD[w];
    for (int32_t t = blockIdx.x; t < ncells; t += gridDim.x) {
        const int64_t k0 = rows[t], k1 = rows[t + 1];
        if (k0 == k1) continue;
        const double cx = ctr[t * 3], cy = ctr[t * 3 + 1], cz = ctr[t * 3 + 2];
        double acc[NS];
#pragma unroll
        for (int i = 0; i < NS; i++) acc[i] = 0.0;
        for (int64_t k = k0 + w; k < k1; k += 4) {
            const int32_t s = src[k];
            for (int m = lane; m < NC; m += 32) {
                const double v = __ldg(&M[(int64_t)s * NC + m]);
                Ms[m] = (d_tab.deg[m] & 1) ? -v : v;
            }
            const double rx = cx - ctr[s * 3], ry = cy - ctr[s * 3 + 1], rz = cz - ctr[s * 3 + 2];
            const double inv_r2 = 1.0 / (rx * rx + ry * ry + rz * rz);
            if (lane == 0) D[0] = sqrt(inv_r2);
            __syncwarp();
            for (int d = 1; d < P; d++) {
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
#pragma unroll 1
            for (int i = 0; i < NS; i++) {
                const int n = 32 * i + lane;
                const bool valid = n < NC;
                const int nn = valid ? n : 0;
                const int nx = d_tab.mi[nn][0], nz = d_tab.mi[nn][2], dn = valid ? d_tab.deg[nn] : P;
                double a = 0.0;
                static_for<0, P>([&](auto Idm) {
                    constexpr int dm = decltype(Idm)::value;
                    if (dn + dm <= P - 1) {
                        const int dv = dn + dm;
                        static_for<0, dm + 1>([&](auto Imx) {
                            constexpr int mx = decltype(Imx)::value;
                            constexpr int bm = ncoef(dm) + tri(dm - mx), len = dm - mx + 1;
                            const int bd = dv * (dv + 1) * (dv + 2) / 6 + tri(dv - nx - mx) + nz;
#pragma unroll
                            for (int u = 0; u < len; u++) a = fma(Ms[bm + u], D[bd + u], a);
                        });
                    }
                });
                acc[i] += a;
            }
            __syncwarp();  // the warp's slices are rewritten by its next pair
        }
#pragma unroll
        for (int i = 0; i < NS; i++)
            if (32 * i + lane < NC) red[w][32 * i + lane] = acc[i];
        __syncthreads();
        for (int n = threadIdx.x; n < NC; n += blockDim.x)
            L[(int64_t)t * NC + n] += (((red[0][n] + red[1][n]) + red[2][n]) + red[3][n]) / d_tab.mfact[n];
        __syncthreads();  // red is rewritten by the next row
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
#define M2L_LANES(PP)                                                                                   \
    case PP:                                                                                            \
        if (PP >= 8 && !getenv("FMM_B200_M2L_BLOCK")) {                                                 \
            m2l_lanes<PP><<<grid_for(ncells, 1, 148 * 8), 128, 0, s>>>(ncells, rows, src, ctr, M, L);    \
            fmm::note_launch();                                                                         \
            break;                                                                                      \
        }                                                                                               \
        [[fallthrough]];
        M2L_LANES(6)
        M2L_LANES(7)
        M2L_LANES(8)
        M2L_LANES(9)
        M2L_LANES(10)
        M2L_LANES(11)
        M2L_LANES(12)
#undef M2L_LANES
        default: {
            // high orders: block kernel over a load-balanced term table
            static int table_p[64];  // per device: the table is a device symbol
            static bool init = false;
            static TermTable host_tab;
            if (!init) {
                for (int i = 0; i < 64; i++) table_p[i] = -1;
                init = true;
            }
            int dev = 0;
            cudaGetDevice(&dev);
            dev &= 63;
            build_term_table(p, host_tab);
            if (table_p[dev] != p) {
                if (cudaMemcpyToSymbolAsync(d_terms, &host_tab, sizeof(TermTable), 0, cudaMemcpyHostToDevice, s) !=
                    cudaSuccess)
                    return cuda_status("fmm_m2l_csr table");
                if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_status("fmm_m2l_csr table sync");
                table_p[dev] = p;
            }
            constexpr int NT = kBlkWarps * 32;
            const int nc = ncoef(p), nch = host_tab.nchunks;
            const size_t smem = (size_t)((nch * kChunk + 1) & ~1) * 4 +
                                (size_t)kBlkWarps * (2 * nc + 1) * 8 + (size_t)nch * 8;
            static size_t smem_set[64] = {};  // the attribute is per device
            if (smem > smem_set[dev]) {
                cudaFuncSetAttribute(m2l_block<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                smem_set[dev] = smem;
            }
            m2l_block<NT><<<grid_for(ncells, 1, 148 * 4), NT, smem, s>>>(p, ncells, rows, src, ctr, M, L);
            fmm::note_launch();
        }
    }
    FMM_CUDA_CHECK("fmm_m2l_csr");
    return FMM_OK;
}
