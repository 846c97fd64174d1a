// passes.cu -- vertical FMM passes on the GPU (src/tree.py:163-189,
// src/_taylor.py:102-269): P2M at the leaves, M2M bottom-up and L2L
// top-down level-synchronously (one launch per level over that level's
// cells, gather/pull form, so no atomics), L2P per body.
//
// Float64 throughout (these passes are <1% of the flops; they keep the
// reference's 1e-12 agreement).  For p <= 5 (the BASELINE orders) M2M, L2L
// and L2P are compiled per order with every multi-index a constant and a
// thread owning a whole cell or body; for higher orders a warp applies each
// M2M / L2L shift as three separable 1-D passes (m2m_sep / l2l_sep) and a
// thread owns a body's L2P.  Every write is private.
#include "taylor.cuh"

namespace fmm {

// ---- P2M: warp per leaf, lane per coefficient ---------------------------
// M_m = sum_j q_j (x_j - c)^m / m!  (src/_taylor.py:134-143).  The warp
// takes the leaf's bodies 32 at a time: lane j tabulates its body's scaled
// powers dx^a / a!, dy^b / b!, dz^c / c! (a, b, c < p) and charge in the
// warp's shared slab, then lane m accumulates q_j * px[a_m] * py[b_m] *
// pz[c_m] over the chunk -- three shared loads and three FP64 ops per body
// and coefficient, no per-lane monomial loops.
constexpr int kMaxSlots = (NMI + 31) / 32;
constexpr int kP2MWarps = 4;

template <int NS>  // coefficient slots per lane: ceil(ncoef(p) / 32)
__global__ void __launch_bounds__(kP2MWarps * 32) p2m_kernel(
    int p, const int32_t *__restrict__ cells, int32_t ncells, const uint8_t *__restrict__ leaf,
    const int32_t *__restrict__ start, const int32_t *__restrict__ end, const double *__restrict__ ctr,
    const double *__restrict__ xs, const double *__restrict__ ys, const double *__restrict__ zs,
    const double *__restrict__ qs, double *M) {
    __shared__ double pw_all[kP2MWarps][32][3 * TMAX + 1];  // [body][axis * TMAX + power | charge]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double (*pw)[3 * TMAX + 1] = pw_all[w];
    const int nc = ncoef(p);
    int ia[NS], ib[NS], ic[NS];
#pragma unroll
    for (int k = 0; k < NS; k++) {
        const int m = min(lane + 32 * k, nc - 1);
        ia[k] = d_tab.mi[m][0];
        ib[k] = TMAX + d_tab.mi[m][1];
        ic[k] = 2 * TMAX + d_tab.mi[m][2];
    }
    for (int ci = blockIdx.x * kP2MWarps + w; ci < ncells; ci += gridDim.x * kP2MWarps) {
        const int32_t c = cells[ci];
        if (!leaf[c]) continue;
        const double cx = ctr[c * 3], cy = ctr[c * 3 + 1], cz = ctr[c * 3 + 2];
        const int32_t s = start[c], e = end[c];
        double acc[NS];
#pragma unroll
        for (int k = 0; k < NS; k++) acc[k] = 0.0;
        for (int32_t b0 = s; b0 < e; b0 += 32) {
            const int cnt = min(32, e - b0);
            if (lane < cnt) {
                const double dx = xs[b0 + lane] - cx, dy = ys[b0 + lane] - cy, dz = zs[b0 + lane] - cz;
                double vx = 1.0, vy = 1.0, vz = 1.0;
                for (int a = 0; a < p; a++) {
                    pw[lane][a] = vx;
                    pw[lane][TMAX + a] = vy;
                    pw[lane][2 * TMAX + a] = vz;
                    const double r = d_tab.rcp[a + 1];
                    vx = vx * dx * r;
                    vy = vy * dy * r;
                    vz = vz * dz * r;
                }
                pw[lane][3 * TMAX] = qs[b0 + lane];
            }
            __syncwarp();
            for (int j = 0; j < cnt; j++) {
                const double q = pw[j][3 * TMAX];
#pragma unroll
                for (int k = 0; k < NS; k++) acc[k] += q * (pw[j][ia[k]] * pw[j][ib[k]] * pw[j][ic[k]]);
            }
            __syncwarp();
        }
#pragma unroll
        for (int k = 0; k < NS; k++) {
            const int m = lane + 32 * k;
            if (m < nc) M[(int64_t)c * nc + m] = acc[k];
        }
    }
}

// ---- P >= 6: warp per cell, separable translation passes ----------------
// The shift operators factor over the axes: t^(m-k)/(m-k)! and the L2L
// weight C(n,k) t^(n-k) are products of one factor per axis, so a warp
// applies a translation as three 1-D passes over the expansion (z, then y,
// then x), each staying inside the |m| < p index set: ~3 x 220 x 3.3 FMAs
// per child link at p = 10 instead of the 5005 terms x 3 flops of the
// direct sum the runtime kernels above walk per coefficient.  Same terms,
// summed in another order (multipoles / locals agree to rounding).
__host__ __device__ constexpr int sep_idx(int x, int y, int z) {  // graded-lex index of (x, y, z)
    return (x + y + z) * (x + y + z + 1) * (x + y + z + 2) / 6 + (y + z) * (y + z + 1) / 2 + z;
}
constexpr int kSepWarps = 4;
__constant__ double c_binom[TMAX + 1][TMAX + 1];

__global__ void __launch_bounds__(kSepWarps * 32) m2m_sep(int p, const int32_t *__restrict__ cells, int32_t count,
                                                         const uint8_t *__restrict__ leaf,
                                                         const int32_t *__restrict__ children,
                                                         const double *__restrict__ ctr, double *M) {
    extern __shared__ double sep_sm[];
    const int nc = ncoef(p), lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double *b0 = sep_sm + w * (2 * nc + 3 * (TMAX + 1)), *b1 = b0 + nc, *pw = b1 + nc;  // pw[3][TMAX+1]
    constexpr int NS = (ncoef(TMAX) + 31) / 32;
    for (int32_t wi = blockIdx.x * kSepWarps + w; wi < count; wi += gridDim.x * kSepWarps) {
        const int32_t c = cells[wi];
        if (leaf[c]) continue;
        double acc[NS];
#pragma unroll
        for (int j = 0; j < NS; j++) acc[j] = 0.0;
        for (int o = 0; o < 8; o++) {
            const int32_t ch = children[c * 8 + o];
            if (ch < 0) continue;
            for (int q = lane; q < nc; q += 32) b0[q] = M[(int64_t)ch * nc + q];
            if (lane < 3) {  // t_a^j / j!, as the runtime kernel forms them
                const double t = ctr[ch * 3 + lane] - ctr[c * 3 + lane];
                double f = 1.0;
                for (int j = 0; j < p; j++) {
                    pw[lane * (TMAX + 1) + j] = f;
                    f = f * t * d_tab.rcp[j + 1];
                }
            }
            __syncwarp();
            for (int q = lane; q < nc; q += 32) {  // z: (x, y, kz) -> (x, y, mz)
                const int x = d_tab.mi[q][0], y = d_tab.mi[q][1], z = d_tab.mi[q][2];
                double a = 0.0;
                for (int k = 0; k <= z; k++) a = fma(b0[sep_idx(x, y, k)], pw[2 * (TMAX + 1) + z - k], a);
                b1[q] = a;
            }
            __syncwarp();
            for (int q = lane; q < nc; q += 32) {  // y
                const int x = d_tab.mi[q][0], y = d_tab.mi[q][1], z = d_tab.mi[q][2];
                double a = 0.0;
                for (int k = 0; k <= y; k++) a = fma(b1[sep_idx(x, k, z)], pw[(TMAX + 1) + y - k], a);
                b0[q] = a;
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < NS; j++) {  // x, into the lane's outputs
                const int q = lane + 32 * j;
                if (q < nc) {
                    const int x = d_tab.mi[q][0], y = d_tab.mi[q][1], z = d_tab.mi[q][2];
                    double a = acc[j];
                    for (int k = 0; k <= x; k++) a = fma(b0[sep_idx(k, y, z)], pw[x - k], a);
                    acc[j] = a;
                }
            }
            __syncwarp();  // b0 / pw are rewritten by the next child
        }
#pragma unroll
        for (int j = 0; j < NS; j++) {
            const int q = lane + 32 * j;
            if (q < nc) M[(int64_t)c * nc + q] += acc[j];
        }
    }
}

__global__ void __launch_bounds__(kSepWarps * 32) l2l_sep(int p, const int32_t *__restrict__ cells, int32_t count,
                                                         const int32_t *__restrict__ parent,
                                                         const double *__restrict__ ctr, double *L) {
    extern __shared__ double sep_sm[];
    const int nc = ncoef(p), lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double *b0 = sep_sm + w * (2 * nc + 3 * (TMAX + 1)), *b1 = b0 + nc, *pw = b1 + nc;
    for (int32_t wi = blockIdx.x * kSepWarps + w; wi < count; wi += gridDim.x * kSepWarps) {
        const int32_t c = cells[wi];
        const int32_t pa = parent[c];
        if (pa < 0) continue;
        for (int q = lane; q < nc; q += 32) b0[q] = L[(int64_t)pa * nc + q];
        if (lane < 3) {  // t_a^j
            const double t = ctr[c * 3 + lane] - ctr[pa * 3 + lane];
            double f = 1.0;
            for (int j = 0; j < p; j++) {
                pw[lane * (TMAX + 1) + j] = f;
                f *= t;
            }
        }
        __syncwarp();
        for (int q = lane; q < nc; q += 32) {  // z: (x, y, nz) -> (x, y, kz), sum over nz >= kz
            const int x = d_tab.mi[q][0], y = d_tab.mi[q][1], k = d_tab.mi[q][2];
            double a = 0.0;
            for (int n = k; n < p - x - y; n++) a = fma(b0[sep_idx(x, y, n)], c_binom[n][k] * pw[2 * (TMAX + 1) + n - k], a);
            b1[q] = a;
        }
        __syncwarp();
        for (int q = lane; q < nc; q += 32) {  // y
            const int x = d_tab.mi[q][0], k = d_tab.mi[q][1], z = d_tab.mi[q][2];
            double a = 0.0;
            for (int n = k; n < p - x - z; n++) a = fma(b1[sep_idx(x, n, z)], c_binom[n][k] * pw[(TMAX + 1) + n - k], a);
            b0[q] = a;
        }
        __syncwarp();
        for (int q = lane; q < nc; q += 32) {  // x, added to the child's locals
            const int k = d_tab.mi[q][0], y = d_tab.mi[q][1], z = d_tab.mi[q][2];
            double a = 0.0;
            for (int n = k; n < p - y - z; n++) a = fma(b0[sep_idx(n, y, z)], c_binom[n][k] * pw[n - k], a);
            L[(int64_t)c * nc + q] += a;
        }
        __syncwarp();  // b0 / b1 / pw are rewritten by the next cell
    }
}

static int sep_smem(int p) { return kSepWarps * (2 * ncoef(p) + 3 * (TMAX + 1)) * (int)sizeof(double); }

static void sep_tables() {  // binomials up to TMAX, once per device
    static bool done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && done[dev]) return;
    double b[TMAX + 1][TMAX + 1] = {};
    for (int n = 0; n <= TMAX; n++) {
        b[n][0] = 1.0;
        for (int k = 1; k <= n; k++) b[n][k] = b[n - 1][k - 1] + (k <= n - 1 ? b[n - 1][k] : 0.0);
    }
    cudaMemcpyToSymbol(c_binom, b, sizeof(b));
    if (dev < 64) done[dev] = true;
}

// ---- P <= 5: thread per cell, every multi-index compile-time -------------
// The runtime-order kernels above walk term loops with table lookups per
// term; for the orders the BASELINE runs use (P = 4, 5) a thread owns a
// whole cell instead: per child (M2M) or from the parent (L2L) it builds
// the shift's scaled powers once and adds every term with compile-time
// indices, the expansions in registers.
template <int P>
__global__ void __launch_bounds__(128) m2m_cell_kernel(const int32_t *__restrict__ cells, int32_t count,
                                                       const uint8_t *__restrict__ leaf,
                                                       const int32_t *__restrict__ children,
                                                       const double *__restrict__ ctr, double *M) {
    constexpr int NC = ncoef(P);
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        const int32_t c = cells[i];
        if (leaf[c]) continue;
        double acc[NC];
#pragma unroll
        for (int m = 0; m < NC; m++) acc[m] = 0.0;
        for (int o = 0; o < 8; o++) {
            const int32_t ch = children[c * 8 + o];
            if (ch < 0) continue;
            const double t[3] = {ctr[ch * 3] - ctr[c * 3], ctr[ch * 3 + 1] - ctr[c * 3 + 1],
                                 ctr[ch * 3 + 2] - ctr[c * 3 + 2]};
            double pw[3][P];  // t_d^a / a!
#pragma unroll
            for (int d = 0; d < 3; d++) {
                pw[d][0] = 1.0;
#pragma unroll
                for (int a = 1; a < P; a++) pw[d][a] = pw[d][a - 1] * t[d] * (1.0 / a);
            }
            double Mc[NC];
#pragma unroll
            for (int k = 0; k < NC; k++) Mc[k] = M[(int64_t)ch * NC + k];
            static_for<0, NC>([&](auto Im) {
                constexpr int m = decltype(Im)::value;
                constexpr int mx = kTab.mi[m][0], my = kTab.mi[m][1], mz = kTab.mi[m][2];
                double a = 0.0;
                static_for<0, m + 1>([&](auto Ik) {  // graded-lex: k <= m componentwise implies index(k) <= m
                    constexpr int k = decltype(Ik)::value;
                    constexpr int kx = kTab.mi[k][0], ky = kTab.mi[k][1], kz = kTab.mi[k][2];
                    if constexpr (kx <= mx && ky <= my && kz <= mz)
                        a = fma(Mc[k], pw[0][mx - kx] * pw[1][my - ky] * pw[2][mz - kz], a);
                });
                acc[m] += a;
            });
        }
#pragma unroll
        for (int m = 0; m < NC; m++) M[(int64_t)c * NC + m] += acc[m];
    }
}

template <int P>
__global__ void __launch_bounds__(128) l2l_cell_kernel(const int32_t *__restrict__ cells, int32_t count,
                                                       const int32_t *__restrict__ parent,
                                                       const double *__restrict__ ctr, double *L) {
    constexpr int NC = ncoef(P);
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        const int32_t c = cells[i];
        const int32_t pa = parent[c];
        if (pa < 0) continue;
        const double t[3] = {ctr[c * 3] - ctr[pa * 3], ctr[c * 3 + 1] - ctr[pa * 3 + 1],
                             ctr[c * 3 + 2] - ctr[pa * 3 + 2]};
        double pw[3][P];  // t_d^a / a!
#pragma unroll
        for (int d = 0; d < 3; d++) {
            pw[d][0] = 1.0;
#pragma unroll
            for (int a = 1; a < P; a++) pw[d][a] = pw[d][a - 1] * t[d] * (1.0 / a);
        }
        double Lp[NC];  // L_n n!
        static_for<0, NC>([&](auto In) {
            constexpr int n = decltype(In)::value;
            constexpr double f = kTab.mfact[n];
            Lp[n] = L[(int64_t)pa * NC + n] * f;
        });
        static_for<0, NC>([&](auto Ik) {
            constexpr int k = decltype(Ik)::value;
            constexpr int kx = kTab.mi[k][0], ky = kTab.mi[k][1], kz = kTab.mi[k][2];
            double a = 0.0;
            static_for<k, NC>([&](auto In) {  // n >= k componentwise implies index(n) >= k
                constexpr int n = decltype(In)::value;
                constexpr int nx = kTab.mi[n][0], ny = kTab.mi[n][1], nz = kTab.mi[n][2];
                if constexpr (nx >= kx && ny >= ky && nz >= kz)
                    a = fma(Lp[n], pw[0][nx - kx] * pw[1][ny - ky] * pw[2][nz - kz], a);
            });
            constexpr double inv = 1.0 / kTab.mfact[k];
            L[(int64_t)c * NC + k] += a * inv;
        });
    }
}

// ---- L2P: thread per body (src/_taylor.py:243-269); f = -grad phi -------
__global__ void l2p_kernel(int p, int64_t b0, int64_t n, const int32_t *__restrict__ body_leaf,
                           const double *__restrict__ ctr, const double *__restrict__ xs,
                           const double *__restrict__ ys, const double *__restrict__ zs,
                           const double *__restrict__ L, double *phi, double *fx, double *fy,
                           double *fz) {
    const int nc = ncoef(p);
    for (int64_t i = b0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = body_leaf[i];
        const double ux = xs[i] - ctr[c * 3], uy = ys[i] - ctr[c * 3 + 1], uz = zs[i] - ctr[c * 3 + 2];
        const double *Lc = L + (int64_t)c * nc;
        double pot = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
        // walk the graded-lex multi-indices with running powers: for each
        // (a, b) the z-exponent runs 0..p-1-a-b, u^k = ux^a uy^b uz^c
        double pa_ = 1.0, pa1 = 0.0;  // ux^a, a*ux^(a-1)
        for (int a = 0; a < p; a++) {
            double pb = 1.0, pb1 = 0.0;
            for (int b = 0; a + b < p; b++) {
                double pc = 1.0, pc1 = 0.0;
                for (int g = 0; a + b + g < p; g++) {
                    const double lk = Lc[d_tab.idx3[a][b][g]];
                    pot += lk * (pa_ * pb * pc);
                    gx += lk * (pa1 * pb * pc);
                    gy += lk * (pa_ * pb1 * pc);
                    gz += lk * (pa_ * pb * pc1);
                    pc1 = pc1 * uz + pc;  // d/duz of uz^(g+1) = (g+1) uz^g
                    pc = pc * uz;
                }
                pb1 = pb1 * uy + pb;
                pb = pb * uy;
            }
            pa1 = pa1 * ux + pa_;
            pa_ = pa_ * ux;
        }
        phi[i] += pot;
        fx[i] -= gx;
        fy[i] -= gy;
        fz[i] -= gz;
    }
}

// P2M for p <= 5: a thread per leaf walks its bodies; per body the scaled
// powers u_d^a / a! once, then every moment an FMA with constant indices.
template <int P>
__global__ void __launch_bounds__(128) p2m_leaf_kernel(const int32_t *__restrict__ cells, int32_t ncells,
                                                       const uint8_t *__restrict__ leaf,
                                                       const int32_t *__restrict__ start,
                                                       const int32_t *__restrict__ end, const double *__restrict__ ctr,
                                                       const double *__restrict__ xs, const double *__restrict__ ys,
                                                       const double *__restrict__ zs, const double *__restrict__ qs,
                                                       double *M) {
    constexpr int NC = ncoef(P);
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ncells; i += gridDim.x * blockDim.x) {
        const int32_t c = cells[i];
        if (!leaf[c]) continue;
        const double cc[3] = {ctr[c * 3], ctr[c * 3 + 1], ctr[c * 3 + 2]};
        double acc[NC];
#pragma unroll
        for (int m = 0; m < NC; m++) acc[m] = 0.0;
        for (int32_t j = start[c]; j < end[c]; j++) {
            const double u[3] = {xs[j] - cc[0], ys[j] - cc[1], zs[j] - cc[2]};
            const double q = qs[j];
            double pw[3][P];
#pragma unroll
            for (int d = 0; d < 3; d++) {
                pw[d][0] = 1.0;
#pragma unroll
                for (int a = 1; a < P; a++) pw[d][a] = pw[d][a - 1] * u[d] * (1.0 / a);
            }
            static_for<0, NC>([&](auto Im) {
                constexpr int m = decltype(Im)::value;
                constexpr int a = kTab.mi[m][0], b = kTab.mi[m][1], g = kTab.mi[m][2];
                acc[m] = fma(q, pw[0][a] * (pw[1][b] * pw[2][g]), acc[m]);
            });
        }
#pragma unroll
        for (int m = 0; m < NC; m++) M[(int64_t)c * NC + m] = acc[m];
    }
}

// L2P for p <= 5 with compile-time multi-indices: the body's powers
// u_d^a and their derivatives a u_d^(a-1) are built once, every term of
// phi = sum L_k u^k and of its gradient is an FMA with constant indices.
template <int P>
__global__ void __launch_bounds__(128) l2p_body_kernel(int64_t b0, int64_t n, const int32_t *__restrict__ body_leaf,
                                                       const double *__restrict__ ctr, const double *__restrict__ xs,
                                                       const double *__restrict__ ys, const double *__restrict__ zs,
                                                       const double *__restrict__ L, double *phi, double *fx,
                                                       double *fy, double *fz) {
    constexpr int NC = ncoef(P);
    for (int64_t i = b0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = body_leaf[i];
        const double u[3] = {xs[i] - ctr[c * 3], ys[i] - ctr[c * 3 + 1], zs[i] - ctr[c * 3 + 2]};
        double pw[3][P], dp[3][P];  // u_d^a, a u_d^(a-1)
#pragma unroll
        for (int d = 0; d < 3; d++) {
            pw[d][0] = 1.0;
            dp[d][0] = 0.0;
#pragma unroll
            for (int a = 1; a < P; a++) {
                dp[d][a] = dp[d][a - 1] * u[d] + pw[d][a - 1];
                pw[d][a] = pw[d][a - 1] * u[d];
            }
        }
        const double *Lc = L + (int64_t)c * NC;
        double pot = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
        static_for<0, NC>([&](auto Ik) {
            constexpr int k = decltype(Ik)::value;
            constexpr int a = kTab.mi[k][0], b = kTab.mi[k][1], g = kTab.mi[k][2];
            const double lk = Lc[k];
            const double yz = pw[1][b] * pw[2][g];
            pot = fma(lk, pw[0][a] * yz, pot);
            gx = fma(lk, dp[0][a] * yz, gx);
            gy = fma(lk, pw[0][a] * (dp[1][b] * pw[2][g]), gy);
            gz = fma(lk, pw[0][a] * (pw[1][b] * dp[2][g]), gz);
        });
        phi[i] += pot;
        fx[i] -= gx;
        fy[i] -= gy;
        fz[i] -= gz;
    }
}

}  // namespace fmm

using namespace fmm;

extern "C" {

int fmm_upward(int p, int32_t ncells, const int32_t *children, const int32_t *start, const int32_t *end,
               const uint8_t *leaf, const double *ctr, const double *xs, const double *ys,
               const double *zs, const double *qs, const int32_t *cells_by_level,
               const int32_t *host_level_off, int nlev, double *M, void *stream) {
    if (p < 1 || p > TMAX) { set_error("expansion order %d outside supported range 1..%d", p, TMAX); return FMM_ERR_INVALID; }
    cudaStream_t s = as_stream(stream);
    const int nc = ncoef(p);
    const int32_t total = host_level_off[nlev];
    if (total > 0 && p <= 5) {
        const int g = grid_for(total, 128);
        switch (p) {
#define P2M_LEAF(PP)                                                                                                \
    case PP:                                                                                                        \
        p2m_leaf_kernel<PP><<<g, 128, 0, s>>>(cells_by_level, total, leaf, start, end, ctr, xs, ys, zs, qs, M); \
        break;
            P2M_LEAF(1) P2M_LEAF(2) P2M_LEAF(3) P2M_LEAF(4) P2M_LEAF(5)
#undef P2M_LEAF
        }
        fmm::note_launch();
    } else if (total > 0) {
        const int g = grid_for(total, kP2MWarps, 148 * 16);
        const int ns = (nc + 31) / 32;
        if (ns <= 1)
            p2m_kernel<1><<<g, kP2MWarps * 32, 0, s>>>(p, cells_by_level, total, leaf, start, end, ctr, xs, ys, zs, qs, M);
        else if (ns <= 2)
            p2m_kernel<2><<<g, kP2MWarps * 32, 0, s>>>(p, cells_by_level, total, leaf, start, end, ctr, xs, ys, zs, qs, M);
        else if (ns <= 4)
            p2m_kernel<4><<<g, kP2MWarps * 32, 0, s>>>(p, cells_by_level, total, leaf, start, end, ctr, xs, ys, zs, qs, M);
        else if (ns <= 8)
            p2m_kernel<8><<<g, kP2MWarps * 32, 0, s>>>(p, cells_by_level, total, leaf, start, end, ctr, xs, ys, zs, qs, M);
        else
            p2m_kernel<kMaxSlots><<<g, kP2MWarps * 32, 0, s>>>(p, cells_by_level, total, leaf, start, end, ctr, xs, ys, zs, qs,
                                                   M);
        fmm::note_launch();
    }
    for (int L = nlev - 2; L >= 0; L--) {
        int32_t off = host_level_off[L], cnt = host_level_off[L + 1] - off;
        if (cnt <= 0) continue;
        switch (p) {
#define M2M_CELL(PP)                                                                                          \
    case PP:                                                                                                  \
        m2m_cell_kernel<PP><<<grid_for(cnt, 128), 128, 0, s>>>(cells_by_level + off, cnt, leaf, children, ctr, M); \
        break;
            M2M_CELL(1) M2M_CELL(2) M2M_CELL(3) M2M_CELL(4) M2M_CELL(5)
#undef M2M_CELL
            default:
                m2m_sep<<<grid_for(cnt, kSepWarps, 148 * 16), kSepWarps * 32, sep_smem(p), s>>>(
                    p, cells_by_level + off, cnt, leaf, children, ctr, M);
        }
        fmm::note_launch();
    }
    FMM_CUDA_CHECK("fmm_upward");
    return FMM_OK;
}

int fmm_downward(int p, int32_t ncells, const int32_t *parent, const uint8_t *leaf, const double *ctr,
                 const int32_t *cells_by_level, const int32_t *host_level_off, int nlev, int64_t body_lo,
                 int64_t body_hi, const int32_t *body_leaf, const double *xs, const double *ys, const double *zs,
                 double *L, double *phi, double *fx, double *fy, double *fz, void *stream) {
    if (p < 1 || p > TMAX) { set_error("expansion order %d outside supported range 1..%d", p, TMAX); return FMM_ERR_INVALID; }
    cudaStream_t s = as_stream(stream);
    const int nc = ncoef(p);
    for (int Lv = 1; Lv < nlev; Lv++) {
        int32_t off = host_level_off[Lv], cnt = host_level_off[Lv + 1] - off;
        if (cnt <= 0) continue;
        switch (p) {
#define L2L_CELL(PP)                                                                                      \
    case PP:                                                                                              \
        l2l_cell_kernel<PP><<<grid_for(cnt, 128), 128, 0, s>>>(cells_by_level + off, cnt, parent, ctr, L); \
        break;
            L2L_CELL(1) L2L_CELL(2) L2L_CELL(3) L2L_CELL(4) L2L_CELL(5)
#undef L2L_CELL
            default:
                sep_tables();
                l2l_sep<<<grid_for(cnt, kSepWarps, 148 * 16), kSepWarps * 32, sep_smem(p), s>>>(
                    p, cells_by_level + off, cnt, parent, ctr, L);
        }
        fmm::note_launch();
    }
    if (body_hi > body_lo) {
        const int g = grid_for(body_hi - body_lo, 128);
        switch (p) {
#define L2P_BODY(PP)                                                                                         \
    case PP:                                                                                                 \
        l2p_body_kernel<PP><<<g, 128, 0, s>>>(body_lo, body_hi, body_leaf, ctr, xs, ys, zs, L, phi, fx, fy, fz); \
        break;
            L2P_BODY(1) L2P_BODY(2) L2P_BODY(3) L2P_BODY(4) L2P_BODY(5)
#undef L2P_BODY
            default:
                l2p_kernel<<<g, 128, 0, s>>>(p, body_lo, body_hi, body_leaf, ctr, xs, ys, zs, L, phi, fx, fy, fz);
        }
        fmm::note_launch();
    }
    FMM_CUDA_CHECK("fmm_downward");
    return FMM_OK;
}

}  // extern "C"
