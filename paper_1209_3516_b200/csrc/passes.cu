// passes.cu -- vertical FMM passes on the GPU (src/tree.py:163-189,
// src/_taylor.py:102-269): P2M at the leaves, M2M bottom-up and L2L
// top-down level-synchronously (one launch per level over that level's
// cells, gather/pull form, so no atomics), L2P per body.
//
// Float64 throughout (these passes are <1% of the flops; they keep the
// reference's 1e-12 agreement).  Expansion order p is a runtime value
// (1..12); a thread owns one (cell, coefficient) so every write is private.
#include "fmm_common.cuh"

namespace fmm {

// x^a / a! for a = 0..deg (recurrence of src/_taylor.py:102-115 per axis)
__device__ inline void pow_fact_axis(double d, int deg, double *out) {
    out[0] = 1.0;
    for (int a = 1; a <= deg; a++) out[a] = out[a - 1] * d / a;
}

__device__ inline void pow_axis(double d, int deg, double *out) {
    out[0] = 1.0;
    for (int a = 1; a <= deg; a++) out[a] = out[a - 1] * d;
}

// ---- P2M: block per leaf, thread per coefficient; bodies staged in smem --
constexpr int kP2MTile = 64;

__global__ void p2m_kernel(int p, const int32_t *__restrict__ cells, int32_t ncells,
                           const uint8_t *__restrict__ leaf,
                           const int32_t *__restrict__ start, const int32_t *__restrict__ end,
                           const double *__restrict__ ctr, const double *__restrict__ xs,
                           const double *__restrict__ ys, const double *__restrict__ zs,
                           const double *__restrict__ qs, double *M) {
    __shared__ double sp[kP2MTile][3][TMAX];
    __shared__ double sq[kP2MTile];
    const int nc = ncoef(p);
    for (int ci = blockIdx.x; ci < ncells; ci += gridDim.x) {
        const int32_t c = cells[ci];
        if (!leaf[c]) continue;
        const double cx = ctr[c * 3], cy = ctr[c * 3 + 1], cz = ctr[c * 3 + 2];
        const int32_t s = start[c], e = end[c];
        int mx = 0, my = 0, mz = 0;
        if (threadIdx.x < nc) {
            mx = d_tab.mi[threadIdx.x][0];
            my = d_tab.mi[threadIdx.x][1];
            mz = d_tab.mi[threadIdx.x][2];
        }
        double acc = 0.0;
        for (int32_t b0 = s; b0 < e; b0 += kP2MTile) {
            int cnt = min(kP2MTile, e - b0);
            __syncthreads();
            for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
                pow_fact_axis(xs[b0 + t] - cx, p - 1, sp[t][0]);
                pow_fact_axis(ys[b0 + t] - cy, p - 1, sp[t][1]);
                pow_fact_axis(zs[b0 + t] - cz, p - 1, sp[t][2]);
                sq[t] = qs[b0 + t];
            }
            __syncthreads();
            if (threadIdx.x < nc)
                for (int t = 0; t < cnt; t++) acc += sq[t] * (sp[t][0][mx] * sp[t][1][my] * sp[t][2][mz]);
        }
        if (threadIdx.x < nc) M[(int64_t)c * nc + threadIdx.x] = acc;
        __syncthreads();
    }
}

// ---- M2M: thread per (internal cell of this level, coefficient m) --------
// Mdst[m] += sum_child sum_{k<=m} Msrc[k] t^{m-k}/(m-k)!, t = c_child - c_parent
__global__ void m2m_level(int p, const int32_t *__restrict__ cells, int32_t count,
                          const uint8_t *__restrict__ leaf, const int32_t *__restrict__ children,
                          const double *__restrict__ ctr, double *M) {
    const int nc = ncoef(p);
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < (int64_t)count * nc;
         it += (int64_t)gridDim.x * blockDim.x) {
        int32_t c = cells[it / nc];
        int m = (int)(it % nc);
        if (leaf[c]) continue;
        const int mx = d_tab.mi[m][0], my = d_tab.mi[m][1], mz = d_tab.mi[m][2];
        double total = 0.0;
        for (int o = 0; o < 8; o++) {
            int32_t ch = children[c * 8 + o];
            if (ch < 0) continue;
            double px[TMAX], py[TMAX], pz[TMAX];
            pow_fact_axis(ctr[ch * 3] - ctr[c * 3], mx, px);
            pow_fact_axis(ctr[ch * 3 + 1] - ctr[c * 3 + 1], my, py);
            pow_fact_axis(ctr[ch * 3 + 2] - ctr[c * 3 + 2], mz, pz);
            const double *Ms = M + (int64_t)ch * nc;
            double acc = 0.0;
            for (int kx = 0; kx <= mx; kx++)
                for (int ky = 0; ky <= my; ky++)
                    for (int kz = 0; kz <= mz; kz++)
                        acc += Ms[d_tab.idx3[kx][ky][kz]] * (px[mx - kx] * py[my - ky] * pz[mz - kz]);
            total += acc;
        }
        M[(int64_t)c * nc + m] += total;
    }
}

// ---- L2L: thread per (cell of this level, coefficient k), pull from parent
// Ldst[k] += (1/k!) sum_{n>=k} Lsrc[n] n! t^{n-k}/(n-k)!,  t = c_child - c_parent
__global__ void l2l_level(int p, const int32_t *__restrict__ cells, int32_t count,
                          const int32_t *__restrict__ parent, const double *__restrict__ ctr,
                          double *L) {
    const int nc = ncoef(p);
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < (int64_t)count * nc;
         it += (int64_t)gridDim.x * blockDim.x) {
        int32_t c = cells[it / nc];
        int k = (int)(it % nc);
        int32_t pa = parent[c];
        if (pa < 0) continue;
        const int kx = d_tab.mi[k][0], ky = d_tab.mi[k][1], kz = d_tab.mi[k][2];
        const int rem = p - 1 - (kx + ky + kz);  // max degree of n-k
        double px[TMAX], py[TMAX], pz[TMAX];
        pow_fact_axis(ctr[c * 3] - ctr[pa * 3], rem, px);
        pow_fact_axis(ctr[c * 3 + 1] - ctr[pa * 3 + 1], rem, py);
        pow_fact_axis(ctr[c * 3 + 2] - ctr[pa * 3 + 2], rem, pz);
        const double *Ls = L + (int64_t)pa * nc;
        double acc = 0.0;
        for (int ax = 0; ax <= rem; ax++)
            for (int ay = 0; ay <= rem - ax; ay++)
                for (int az = 0; az <= rem - ax - ay; az++) {
                    int n = d_tab.idx3[kx + ax][ky + ay][kz + az];
                    acc += Ls[n] * d_tab.mfact[n] * (px[ax] * py[ay] * pz[az]);
                }
        L[(int64_t)c * nc + k] += acc / d_tab.mfact[k];
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
        int32_t c = body_leaf[i];
        double ux[TMAX], uy[TMAX], uz[TMAX];
        pow_axis(xs[i] - ctr[c * 3], p - 1, ux);
        pow_axis(ys[i] - ctr[c * 3 + 1], p - 1, uy);
        pow_axis(zs[i] - ctr[c * 3 + 2], p - 1, uz);
        const double *Lc = L + (int64_t)c * nc;
        double pot = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
        for (int k = 0; k < nc; k++) {
            const int a = d_tab.mi[k][0], b = d_tab.mi[k][1], e = d_tab.mi[k][2];
            double lk = Lc[k];
            pot += lk * (ux[a] * uy[b] * uz[e]);
            if (a > 0) gx += lk * a * (ux[a - 1] * uy[b] * uz[e]);
            if (b > 0) gy += lk * b * (ux[a] * uy[b - 1] * uz[e]);
            if (e > 0) gz += lk * e * (ux[a] * uy[b] * uz[e - 1]);
        }
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
    int blk = nc <= 32 ? 32 : (nc <= 64 ? 64 : (nc <= 128 ? 128 : (nc <= 256 ? 256 : 384)));
    const int32_t total = host_level_off[nlev];
    if (total > 0)
        p2m_kernel<<<grid_for(total, 1, 148 * 32), blk, 0, s>>>(p, cells_by_level, total, leaf, start, end, ctr,
                                                               xs, ys, zs, qs, M); fmm::note_launch();
    for (int L = nlev - 2; L >= 0; L--) {
        int32_t off = host_level_off[L], cnt = host_level_off[L + 1] - off;
        if (cnt <= 0) continue;
        m2m_level<<<grid_for((int64_t)cnt * nc, 128), 128, 0, s>>>(p, cells_by_level + off, cnt, leaf,
                                                                  children, ctr, M); fmm::note_launch();
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
        l2l_level<<<grid_for((int64_t)cnt * nc, 128), 128, 0, s>>>(p, cells_by_level + off, cnt, parent,
                                                                  ctr, L); fmm::note_launch();
    }
    if (body_hi > body_lo)
        l2p_kernel<<<grid_for(body_hi - body_lo, 128), 128, 0, s>>>(p, body_lo, body_hi, body_leaf, ctr, xs, ys,
                                                                    zs, L, phi, fx, fy, fz); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_downward");
    return FMM_OK;
}

}  // extern "C"
