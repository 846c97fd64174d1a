// m2l_sym.cu -- symmetric M2L over UNORDERED cell pairs.
//
// Replaces the reference's _m2l_mutual (src/_taylor.py:191-217): one
// derivative tensor D(r), r = c_a - c_b, serves both directions of the pair
// (a, b) through D_k(-r) = (-1)^|k| D_k(r):
//
//   L_a[n] += (1/n!)          sum_{|m| < p-|n|} (-1)^|m| M_b[m] D_{m+n}
//   L_b[n] += (1/n!) (-1)^|n| sum_{|m| < p-|n|}          M_a[m] D_{m+n}
//
// Deterministic without float atomics, like the symmetric P2P (p2p_sym.cu):
// a warp owns a FIRST member a (rows_a/src_a: CSR of the pairs by first
// member), one lane per pair; the sums for a stay in the lanes' registers
// and are folded once per row, the finished coefficients for b (the
// "reaction") are stored in the pair's slot of a scratch buffer, and a second
// kernel, one warp per cell, adds the cell's slots in ascending order of the
// first member.  Register form with compile-time multi-indices (taylor.cuh),
// orders p <= 7: from p = 8 the far field takes the offset-grouped tensor
// kernel (m2l_grouped.cu), which shares one D over a whole lattice group
// rather than over the two directions of a pair.
#include "taylor.cuh"

namespace fmm {

namespace {

constexpr int kSymM2LWarps = 4;

template <int P>
__global__ void __launch_bounds__(kSymM2LWarps * 32) m2l_sym_kernel(
    int32_t a_lo, int32_t a_hi, const int64_t *__restrict__ rowsA, const int32_t *__restrict__ srcA,
    int64_t slot_base, const double *__restrict__ ctr, const double *__restrict__ M, double *__restrict__ react,
    double *L) {
    constexpr int NC = ncoef(P);
    __shared__ double Ma[kSymM2LWarps][NC];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int32_t a = a_lo + (int32_t)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); a < a_hi;
         a += (int32_t)((gridDim.x * blockDim.x) >> 5)) {
        const int64_t k0 = rowsA[a], k1 = rowsA[a + 1];
        if (k0 == k1) continue;
        __syncwarp();
        for (int n = lane; n < NC; n += 32) Ma[warp][n] = M[(int64_t)a * NC + n];
        __syncwarp();
        const double cx = ctr[a * 3], cy = ctr[a * 3 + 1], cz = ctr[a * 3 + 2];
        double acc[NC];
#pragma unroll
        for (int n = 0; n < NC; n++) acc[n] = 0.0;
        for (int64_t k = k0 + lane; k < k1; k += 32) {
            const int32_t b = srcA[k];
            double D[NC];
            d_tensors_reg<P>(cx - ctr[b * 3], cy - ctr[b * 3 + 1], cz - ctr[b * 3 + 2], D);
            // first member: the directed conversion b -> a, moments streamed
            const double *__restrict__ Mb = M + (int64_t)b * NC;
            static_for<0, NC>([&](auto Im) {
                constexpr int m = decltype(Im)::value;
                const double raw = __ldg(&Mb[m]);
                const double mm = (kTab.deg[m] & 1) ? -raw : raw;
                static_for<0, ncoef(P - kTab.deg[m])>([&](auto In) {
                    constexpr int n = decltype(In)::value;
                    constexpr int j = kTab.idx3[kTab.mi[n][0] + kTab.mi[m][0]][kTab.mi[n][1] + kTab.mi[m][1]]
                                               [kTab.mi[n][2] + kTab.mi[m][2]];
                    acc[n] = fma(mm, D[j], acc[n]);
                });
            });
            // second member: finished coefficients into the pair's slot
            double *__restrict__ out = react + (k - slot_base) * NC;
            static_for<0, NC>([&](auto In) {
                constexpr int n = decltype(In)::value;
                double s = 0.0;
                static_for<0, ncoef(P - kTab.deg[n])>([&](auto Im) {
                    constexpr int m = decltype(Im)::value;
                    constexpr int j = kTab.idx3[kTab.mi[n][0] + kTab.mi[m][0]][kTab.mi[n][1] + kTab.mi[m][1]]
                                               [kTab.mi[n][2] + kTab.mi[m][2]];
                    s = fma(Ma[warp][m], D[j], s);
                });
                constexpr double inv = ((kTab.deg[n] & 1) ? -1.0 : 1.0) / kTab.mfact[n];
                out[n] = s * inv;
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
                L[(int64_t)a * NC + n] += acc[n] * inv;
            });
        }
    }
}

// Position of b in the ascending row [lo, hi) of srcA (it is there).
__device__ __forceinline__ int64_t sym_row_find(const int32_t *__restrict__ src, int64_t lo, int64_t hi, int32_t b) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (src[mid] < b) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Second members: a warp per cell b adds its slots in ascending order of the
// first member (rows_b/src_b: CSR of the pairs by second member), lanes over
// the coefficients.
template <int P>
__global__ void __launch_bounds__(128) m2l_sym_reduce_kernel(
    int32_t ncells, int32_t a_lo, int32_t a_hi, const int64_t *__restrict__ rowsB, const int32_t *__restrict__ srcB,
    const int64_t *__restrict__ rowsA, const int32_t *__restrict__ srcA, int64_t slot_base,
    const double *__restrict__ react, double *L) {
    constexpr int NC = ncoef(P), NS = (NC + 31) / 32;
    const int lane = threadIdx.x & 31;
    for (int32_t b = (int32_t)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); b < ncells;
         b += (int32_t)((gridDim.x * blockDim.x) >> 5)) {
        const int64_t e0 = rowsB[b], e1 = rowsB[b + 1];
        if (e0 == e1) continue;
        double s[NS];
#pragma unroll
        for (int i = 0; i < NS; i++) s[i] = 0.0;
        bool any = false;
        for (int64_t eb = e0; eb < e1; eb += 32) {
            const int64_t e = eb + lane;
            int64_t mine = -1;
            if (e < e1) {
                const int32_t a = srcB[e];
                if (a >= a_lo && a < a_hi) mine = sym_row_find(srcA, rowsA[a], rowsA[a + 1], b) - slot_base;
            }
            const int ne = (int)min((int64_t)32, e1 - eb);
            for (int q = 0; q < ne; q++) {
                const int64_t slot = __shfl_sync(0xffffffffu, mine, q);
                if (slot < 0) continue;
                any = true;
                const double *__restrict__ row = react + slot * NC;
#pragma unroll
                for (int i = 0; i < NS; i++)
                    if (32 * i + lane < NC) s[i] += row[32 * i + lane];
            }
        }
        if (any) {
#pragma unroll
            for (int i = 0; i < NS; i++)
                if (32 * i + lane < NC) L[(int64_t)b * NC + 32 * i + lane] += s[i];
        }
    }
}

template <int P>
void launch_m2l_sym(int32_t ncells, int32_t a_lo, int32_t a_hi, const int64_t *rows_a, const int32_t *src_a,
                    const int64_t *rows_b, const int32_t *src_b, int64_t slot_base, const double *ctr,
                    const double *M, double *react, double *L, cudaStream_t st) {
    m2l_sym_kernel<P><<<grid_for((int64_t)(a_hi - a_lo) * 32, kSymM2LWarps * 32, 148 * 16), kSymM2LWarps * 32, 0, st>>>(
        a_lo, a_hi, rows_a, src_a, slot_base, ctr, M, react, L);
    fmm::note_launch();
    m2l_sym_reduce_kernel<P><<<grid_for((int64_t)ncells * 32, 128, 148 * 16), 128, 0, st>>>(
        ncells, a_lo, a_hi, rows_b, src_b, rows_a, src_a, slot_base, react, L);
    fmm::note_launch();
}

}  // namespace

}  // namespace fmm

using namespace fmm;

extern "C" int fmm_m2l_sym(int p, int32_t ncells, int32_t a_lo, int32_t a_hi, const int64_t *rows_a,
                           const int32_t *src_a, const int64_t *rows_b, const int32_t *src_b, int64_t slot_base,
                           const double *ctr, const double *M, double *react, double *L, void *stream) {
    if (ncells <= 0 || a_hi <= a_lo) return FMM_OK;
    if (a_lo < 0 || a_hi > ncells) { set_error("first-member range [%d, %d) outside the cells", a_lo, a_hi); return FMM_ERR_INVALID; }
    if (!react) { set_error("symmetric M2L needs the reaction buffer"); return FMM_ERR_INVALID; }
    if (p < 1 || p > FMM_M2L_SYM_MAX_P) {
        set_error("symmetric M2L: expansion order %d outside 1..%d (higher orders run directed)", p, FMM_M2L_SYM_MAX_P);
        return FMM_ERR_INVALID;
    }
    cudaStream_t st = as_stream(stream);
    switch (p) {
#define M2L_SYM(PP)                                                                                              \
    case PP:                                                                                                     \
        launch_m2l_sym<PP>(ncells, a_lo, a_hi, rows_a, src_a, rows_b, src_b, slot_base, ctr, M, react, L, st);   \
        break;
        M2L_SYM(1) M2L_SYM(2) M2L_SYM(3) M2L_SYM(4) M2L_SYM(5) M2L_SYM(6) M2L_SYM(7)
#undef M2L_SYM
    }
    FMM_CUDA_CHECK("fmm_m2l_sym");
    return FMM_OK;
}
