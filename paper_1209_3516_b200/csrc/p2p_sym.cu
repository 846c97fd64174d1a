// p2p_sym.cu -- symmetric near field over UNORDERED leaf pairs, and the
// symmetric M2L over unordered cell pairs.
//
// Replaces the reference's mutual kernels: _p2p_mutual
// (src/_taylor.py:410-449: one 1/r per body pair, added to both bodies) and
// _m2l_mutual (src/_taylor.py:191-217: one derivative tensor per cell pair,
// contracted in both directions).  A mutual self pair (_p2p_mutual_self,
// :452-493) stays with the directed kernel as the leaf's guarded self run.
//
// Both kernels are deterministic without float atomics: the sums a pair adds
// to its FIRST member stay in the registers of the CTA owning that row and
// are added by it; the sums for the SECOND member (the "reaction") go to a
// per-pair slot of a scratch buffer, and a second kernel, one CTA per cell,
// adds the cell's slots in ascending order of the first member.
//
// P2P pair kernel: a CTA per first leaf a, its partners' bodies dealt to 4
// warps as one stream.  A warp keeps up to 2 targets of a per lane (64 per
// sweep) and takes the stream's sources 32 at a time; in step k lane l meets source slot (l + k) mod 32, whose
// position comes from the warp's shared-memory copy and whose four reaction
// sums travel round the warp by one shuffle each per step, so that after 32
// steps every lane holds the finished sums of its own slot and stores them
// coalesced.  The pair costs 20 operations for both directions (3 sub, 3
// r2, 1 guard, 2 r^-3, 3 g = d r^-3, 4 + 4 accumulations) against 2 x 13.
#include "fmm_common.cuh"

namespace fmm {

namespace {

constexpr int kSymWarps = 4;

template <typename T> struct V4 {};
template <> struct V4<float> { using type = float4; };
template <> struct V4<double> { using type = double4; };

__device__ __forceinline__ float sym_rsqrt(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// MUFU.RSQ64H seed + one third-order step (as the streamed FP64 P2P)
__device__ __forceinline__ double sym_rsqrt(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-(x * y), y, 1.0);
    return fma(y * e, fma(0.375, e, 0.5), y);
}

template <typename T, typename B>
__device__ __forceinline__ void sym_pair(const B &t, const B &s, T (&acc)[4], T &rp, T &rx, T &ry, T &rz) {
    const T dx = t.x - s.x, dy = t.y - s.y, dz = t.z - s.z;
    const T r2 = fma(dz, dz, fma(dy, dy, dx * dx));
    T rinv = sym_rsqrt(r2);
    rinv = r2 > T(0) ? rinv : T(0);
    const T r3 = rinv * rinv * rinv;
    const T gx = dx * r3, gy = dy * r3, gz = dz * r3;
    acc[0] = fma(s.w, rinv, acc[0]);
    acc[1] = fma(s.w, gx, acc[1]);
    acc[2] = fma(s.w, gy, acc[2]);
    acc[3] = fma(s.w, gz, acc[3]);
    rp = fma(t.w, rinv, rp);
    rx = fma(t.w, gx, rx);
    ry = fma(t.w, gy, ry);
    rz = fma(t.w, gz, rz);
}

// One 32-source chunk against the lane's targets: in step k lane l meets
// source slot (l + k) mod 32; the slot's four reaction sums travel with it.
template <typename T, typename B, bool TWO>
__device__ __forceinline__ void sym_chunk(const B *__restrict__ sb, int lane, const B &t0, const B &t1, T (&acc0)[4],
                                          T (&acc1)[4], T &rp, T &rx, T &ry, T &rz) {
    const int nxt = (lane + 1) & 31;
#pragma unroll 4
    for (int st = 0; st < 32; st++) {
        const B sv = sb[(lane + st) & 31];
        sym_pair<T>(t0, sv, acc0, rp, rx, ry, rz);
        if constexpr (TWO) sym_pair<T>(t1, sv, acc1, rp, rx, ry, rz);
        rp = __shfl_sync(0xffffffffu, rp, nxt);
        rx = __shfl_sync(0xffffffffu, rx, nxt);
        ry = __shfl_sync(0xffffffffu, ry, nxt);
        rz = __shfl_sync(0xffffffffu, rz, nxt);
    }
}

// rowsA/srcA: CSR of the unordered pairs by first leaf (sources ascending);
// slot_off[k] = first reaction slot of pair k (slots = bodies of srcA[k]).
// Only first leaves in [a_lo, a_hi) (one chunk of a bounded react buffer).
//
// The partners of a first leaf are swept as ONE source stream: the reaction
// slots of a row are consecutive (slot_off is a prefix sum over the row's
// partner sizes), so stream position i is slot i, body
// cstart[srcA[k]] + i - slot_off[k] of the partner k covering it.  The
// warps take the stream 32 positions at a time, each lane walking its own
// partner cursor forward; only the row's last chunk is padded.  A sweep
// whose targets fit one per lane skips the second target's arithmetic.
template <typename T>
__global__ void __launch_bounds__(kSymWarps * 32) p2p_sym_kernel(
    int32_t a_lo, int32_t a_hi, const int64_t *__restrict__ rowsA, const int32_t *__restrict__ srcA,
    const int64_t *__restrict__ slot_off, int64_t slot_base, const int32_t *__restrict__ cstart,
    const int32_t *__restrict__ cend, const typename V4<T>::type *__restrict__ bodies,
    typename V4<T>::type *__restrict__ react, double *__restrict__ phi, double *__restrict__ fx,
    double *__restrict__ fy, double *__restrict__ fz) {
    using B = typename V4<T>::type;
    const int32_t a = a_lo + (int32_t)blockIdx.x;
    if (a >= a_hi) return;
    const int64_t k0 = rowsA[a], k1 = rowsA[a + 1];
    if (k0 == k1) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t as = cstart[a], na = cend[a] - as;
    const int64_t s0 = slot_off[k0], s1 = slot_off[k1];
    __shared__ B sbuf[kSymWarps][32];
    __shared__ T fold[kSymWarps][64][4];
    for (int32_t tb = 0; tb < na; tb += 64) {
        const bool two = na - tb > 32;
        const int32_t i0 = tb + lane, i1 = tb + 32 + lane;
        B t0 = bodies[as + min(i0, na - 1)], t1 = bodies[as + min(i1, na - 1)];
        if (i0 >= na) t0.w = T(0);
        if (i1 >= na) t1.w = T(0);
        T acc0[4] = {T(0), T(0), T(0), T(0)}, acc1[4] = {T(0), T(0), T(0), T(0)};
        int64_t kc = k0;  // the lane's partner cursor (stream positions only grow)
        for (int64_t cb = s0 + warp * 32; cb < s1; cb += kSymWarps * 32) {
            const int64_t i = cb + lane;
            const bool valid = i < s1;
            const int64_t ii = valid ? i : s1 - 1;
            while (slot_off[kc + 1] <= ii) kc++;
            B s = bodies[cstart[srcA[kc]] + (int32_t)(ii - slot_off[kc])];
            if (!valid) s.w = T(0);
            __syncwarp();
            sbuf[warp][lane] = s;
            __syncwarp();
            T rp = T(0), rx = T(0), ry = T(0), rz = T(0);
            if (two) sym_chunk<T, B, true>(sbuf[warp], lane, t0, t1, acc0, acc1, rp, rx, ry, rz);
            else sym_chunk<T, B, false>(sbuf[warp], lane, t0, t1, acc0, acc1, rp, rx, ry, rz);
            if (valid) {
                B out;
                out.x = rp; out.y = -rx; out.z = -ry; out.w = -rz;  // (phi, fx, fy, fz)
                if (tb > 0) {
                    const B old = react[i - slot_base];
                    out.x += old.x; out.y += old.y; out.z += old.z; out.w += old.w;
                }
                react[i - slot_base] = out;
            }
        }
#pragma unroll
        for (int c = 0; c < 4; c++) {
            fold[warp][lane][c] = acc0[c];
            fold[warp][32 + lane][c] = acc1[c];
        }
        __syncthreads();
        if (threadIdx.x < 64 && tb + (int32_t)threadIdx.x < na) {
            double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int w = 0; w < kSymWarps; w++)
#pragma unroll
                for (int c = 0; c < 4; c++) s[c] += (double)fold[w][threadIdx.x][c];
            const int64_t i = (int64_t)as + tb + threadIdx.x;
            phi[i] += s[0];
            fx[i] += s[1];
            fy[i] += s[2];
            fz[i] += s[3];
        }
        __syncthreads();
    }
}

// Position of b in the ascending row [lo, hi) of srcA (it is there).
__device__ __forceinline__ int64_t row_find(const int32_t *__restrict__ src, int64_t lo, int64_t hi, int32_t b) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (src[mid] < b) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Second members: a CTA per leaf b adds its reaction slots in ascending
// order of the first member (rowsB/srcB: CSR of the pairs by second leaf).
template <typename T>
__global__ void __launch_bounds__(64) p2p_sym_reduce_kernel(
    int32_t ncells, int32_t a_lo, int32_t a_hi, const int64_t *__restrict__ rowsB, const int32_t *__restrict__ srcB,
    const int64_t *__restrict__ rowsA, const int32_t *__restrict__ srcA, const int64_t *__restrict__ slot_off,
    int64_t slot_base, const int32_t *__restrict__ cstart, const int32_t *__restrict__ cend,
    const typename V4<T>::type *__restrict__ react, double *__restrict__ phi, double *__restrict__ fx,
    double *__restrict__ fy, double *__restrict__ fz) {
    using B = typename V4<T>::type;
    const int32_t b = blockIdx.x;
    if (b >= ncells) return;
    const int64_t e0 = rowsB[b], e1 = rowsB[b + 1];
    if (e0 == e1) return;
    const int32_t bs = cstart[b], nb = cend[b] - bs;
    __shared__ int64_t slots[64];
    double s[4][4];  // up to 4 bodies per thread per sweep (ncrit <= 256 in one sweep)
    for (int32_t jb = 0; jb < nb; jb += 256) {
#pragma unroll
        for (int u = 0; u < 4; u++) s[u][0] = s[u][1] = s[u][2] = s[u][3] = 0.0;
        for (int64_t eb = e0; eb < e1; eb += 64) {
            const int64_t e = eb + threadIdx.x;
            int64_t sl = -1;
            if (e < e1) {
                const int32_t a = srcB[e];
                if (a >= a_lo && a < a_hi) sl = slot_off[row_find(srcA, rowsA[a], rowsA[a + 1], b)] - slot_base;
            }
            __syncthreads();
            slots[threadIdx.x] = sl;
            __syncthreads();
            const int ne = (int)min((int64_t)64, e1 - eb);
            for (int q = 0; q < ne; q++) {
                const int64_t base = slots[q];
                if (base < 0) continue;
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int32_t j = jb + u * 64 + threadIdx.x;
                    if (j < nb) {
                        const B v = react[base + j];
                        s[u][0] += (double)v.x; s[u][1] += (double)v.y; s[u][2] += (double)v.z; s[u][3] += (double)v.w;
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int32_t j = jb + u * 64 + threadIdx.x;
            if (j < nb) {
                const int64_t i = (int64_t)bs + j;
                phi[i] += s[u][0];
                fx[i] += s[u][1];
                fy[i] += s[u][2];
                fz[i] += s[u][3];
            }
        }
    }
}

}  // namespace

}  // namespace fmm

using namespace fmm;

template <typename T>
static void launch_p2p_sym(int32_t ncells, int32_t a_lo, int32_t a_hi, const int64_t *rows_a, const int32_t *src_a,
                           const int64_t *rows_b, const int32_t *src_b, const int64_t *slot_off, int64_t slot_base,
                           const int32_t *start, const int32_t *end, const void *bodies4, void *react, double *phi,
                           double *fx, double *fy, double *fz, cudaStream_t st) {
    using B = typename V4<T>::type;
    p2p_sym_kernel<T><<<a_hi - a_lo, kSymWarps * 32, 0, st>>>(a_lo, a_hi, rows_a, src_a, slot_off, slot_base, start, end,
                                                             (const B *)bodies4, (B *)react, phi, fx, fy, fz);
    fmm::note_launch();
    p2p_sym_reduce_kernel<T><<<ncells, 64, 0, st>>>(ncells, a_lo, a_hi, rows_b, src_b, rows_a, src_a, slot_off,
                                                    slot_base, start, end, (const B *)react, phi, fx, fy, fz);
    fmm::note_launch();
}

extern "C" int fmm_p2p_sym(int precision, int32_t ncells, int32_t a_lo, int32_t a_hi, const int64_t *rows_a,
                           const int32_t *src_a, const int64_t *rows_b, const int32_t *src_b, const int64_t *slot_off,
                           int64_t slot_base, const int32_t *start, const int32_t *end, const void *bodies4,
                           void *react, double *phi, double *fx, double *fy, double *fz, void *stream) {
    if (ncells <= 0 || a_hi <= a_lo) return FMM_OK;
    if (a_lo < 0 || a_hi > ncells) { set_error("first-leaf range [%d, %d) outside the cells", a_lo, a_hi); return FMM_ERR_INVALID; }
    if (!bodies4 || !react) { set_error("symmetric P2P needs the packed body copy and the reaction buffer"); return FMM_ERR_INVALID; }
    cudaStream_t st = as_stream(stream);
    if (precision == FMM_PREC_FP32)
        launch_p2p_sym<float>(ncells, a_lo, a_hi, rows_a, src_a, rows_b, src_b, slot_off, slot_base, start, end,
                              bodies4, react, phi, fx, fy, fz, st);
    else if (precision == FMM_PREC_FP64)
        launch_p2p_sym<double>(ncells, a_lo, a_hi, rows_a, src_a, rows_b, src_b, slot_off, slot_base, start, end,
                               bodies4, react, phi, fx, fy, fz, st);
    else { set_error("symmetric P2P: precision %d (FMM_PREC_FP32 or FMM_PREC_FP64)", precision); return FMM_ERR_INVALID; }
    FMM_CUDA_CHECK("fmm_p2p_sym");
    return FMM_OK;
}
