// tree_build.cu -- Morton-key tree construction on the GPU, bit-exact with
// the reference (src/geometry.py:134-206, src/tree.py:43-160, :370-454).
//
// Compiled with --fmad=false: the reference (numba, no fastmath) never fuses
// a*b+c, and keys, centers, bmax and rmax must match it bit for bit.
//
// Layout: bodies are float64 SoA in Morton order (plus a float4 copy for
// the FP32 P2P path); cells are SoA int32/uint64/double arrays indexed by
// the reference's pre-order cell id.  The carve is a single pass over the
// sorted keys (see "single-pass carve" below): pre-order is the order by
// (start, level) -- a cell precedes its descendants (same start, lower
// level) and every later sibling subtree (larger start) -- so one scan of
// per-body cell counts numbers every cell.
#include <cub/cub.cuh>
#include <atomic>
#include <stdarg.h>
#include <stdio.h>

#include "fmm_common.cuh"

namespace fmm {

static thread_local char g_err[512] = "";
static std::atomic<long long> g_launches{0};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_status(const char *where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", where, cudaGetErrorString(e));
        return FMM_ERR_CUDA;
    }
    return FMM_OK;
}

// ---------------------------------------------------------------------------
// ingest + bounds
// ---------------------------------------------------------------------------
constexpr int kBoundsBlocks = 592;  // 4 x 148 SMs

template <class T>
__global__ void ingest_bounds_partial(const T *__restrict__ x, const T *__restrict__ y,
                                      const T *__restrict__ z, const T *__restrict__ q, int64_t n,
                                      double *x64, double *y64, double *z64, double *q64,
                                      bool copy, double *partial) {
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double a = (double)x[i], b = (double)y[i], c = (double)z[i];
        if (copy) {
            x64[i] = a;
            y64[i] = b;
            z64[i] = c;
            q64[i] = (double)q[i];
        }
        mn[0] = fmin(mn[0], a); mx[0] = fmax(mx[0], a);
        mn[1] = fmin(mn[1], b); mx[1] = fmax(mx[1], b);
        mn[2] = fmin(mn[2], c); mx[2] = fmax(mx[2], c);
    }
    __shared__ double s[6][32];
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int d = 0; d < 3; d++) {
        double a = mn[d], b = mx[d];
        for (int o = 16; o > 0; o >>= 1) {
            a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if (lane == 0) { s[d][w] = a; s[3 + d][w] = b; }
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        int nw = blockDim.x >> 5;
        double v = s[threadIdx.x][0];
        for (int k = 1; k < nw; k++)
            v = threadIdx.x < 3 ? fmin(v, s[threadIdx.x][k]) : fmax(v, s[threadIdx.x][k]);
        partial[blockIdx.x * 6 + threadIdx.x] = v;
    }
}

__global__ void bounds_final(const double *partial, int nb, double *root) {
    // one warp: lane-strided over the block partials, then shuffles
    const int lane = threadIdx.x & 31;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int b = lane; b < nb; b += 32)
        for (int d = 0; d < 3; d++) {
            lo[d] = fmin(lo[d], partial[b * 6 + d]);
            hi[d] = fmax(hi[d], partial[b * 6 + 3 + d]);
        }
    for (int d = 0; d < 3; d++)
        for (int o = 16; o > 0; o >>= 1) {
            lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
            hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
        }
    if (lane != 0) return;
    // size = max extent; 0 -> 1.0 (src/tree.py:388-392); extents in x, y, z order
    double size = hi[0] - lo[0];
    double e1 = hi[1] - lo[1], e2 = hi[2] - lo[2];
    if (e1 > size) size = e1;
    if (e2 > size) size = e2;
    if (size == 0.0) size = 1.0;
    root[0] = lo[0];
    root[1] = lo[1];
    root[2] = lo[2];
    root[3] = size;
    root[4] = (double)(1 << MAX_LEVEL) / size;
    root[5] = hi[0];
    root[6] = hi[1];
    root[7] = hi[2];
}

// ---------------------------------------------------------------------------
// Morton keys (src/geometry.py:134-161)
// ---------------------------------------------------------------------------
__global__ void morton_kernel(const double *__restrict__ x, const double *__restrict__ y,
                              const double *__restrict__ z, int64_t n, const double *__restrict__ root,
                              uint64_t *keys, int32_t *iota) {
    const double lo0 = root[0], lo1 = root[1], lo2 = root[2], inv_h = root[4];
    const int64_t top = (1ll << MAX_LEVEL) - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t ix = (int64_t)((x[i] - lo0) * inv_h);
        int64_t iy = (int64_t)((y[i] - lo1) * inv_h);
        int64_t iz = (int64_t)((z[i] - lo2) * inv_h);
        ix = ix < 0 ? 0 : (ix > top ? top : ix);
        iy = iy < 0 ? 0 : (iy > top ? top : iy);
        iz = iz < 0 ? 0 : (iz > top ? top : iz);
        keys[i] = spread21((uint64_t)ix) | spread21((uint64_t)iy) << 1 | spread21((uint64_t)iz) << 2;
        if (iota) iota[i] = (int32_t)i;
    }
}

__global__ void permute_kernel(const int32_t *__restrict__ perm, const double *__restrict__ x,
                               const double *__restrict__ y, const double *__restrict__ z,
                               const double *__restrict__ q, int64_t n, double *xs, double *ys,
                               double *zs, double *qs, float4 *b32, float4 *b32lo, int *inexact) {
    bool any = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t o = perm[i];
        double a = x[o], b = y[o], c = z[o], d = q[o];
        xs[i] = a;
        ys[i] = b;
        zs[i] = c;
        qs[i] = d;
        if (b32) {
            float4 h = make_float4((float)a, (float)b, (float)c, (float)d);
            b32[i] = h;
            float4 l = make_float4((float)(a - (double)h.x), (float)(b - (double)h.y),
                                   (float)(c - (double)h.z), 0.0f);
            if (b32lo) b32lo[i] = l;
            any |= (l.x != 0.0f) | (l.y != 0.0f) | (l.z != 0.0f);
        }
    }
    if (inexact && __syncthreads_or(any) && threadIdx.x == 0) atomicOr(inexact, 1);
}

// ---------------------------------------------------------------------------
// single-pass carve (replaces the level loop): for sorted keys, body i's leaf
// level l(i) is the first level whose cell around i holds <= ncrit bodies
// (or 21); i starts a cell at every level in [ldiff(i), l(i)], where
// ldiff(i) is the first level at which key i differs from key i-1.  An
// exclusive scan of the per-body counts numbers the cells in (start, level)
// order -- exactly the reference's pre-order (src/tree.py:43-77).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int first_diff_level(const uint64_t *keys, int64_t i) {
    if (i == 0) return 0;
    const uint64_t x = keys[i] ^ keys[i - 1];
    if (x == 0) return MAX_LEVEL + 1;  // same depth-21 cell: starts nothing
    const int b = 63 - __clzll((long long)x);
    return MAX_LEVEL - b / 3;
}

// size of the run of equal level-L prefix around i, clipped to the window
// [i - ncrit, i + ncrit]: <= ncrit exactly when the true cell holds <= ncrit
__device__ __forceinline__ int64_t run_in_window(const uint64_t *keys, int64_t n, int64_t i, int L, int ncrit) {
    const int sh = 3 * (MAX_LEVEL - L);
    const uint64_t pre = sh >= 64 ? 0 : keys[i] >> sh;
    int64_t wl = i - ncrit < 0 ? 0 : i - ncrit;
    int64_t wh = i + ncrit + 1 > n ? n : i + ncrit + 1;
    int64_t a = wl, b = i;  // first index in [wl, i] with the prefix
    while (a < b) {
        const int64_t m = (a + b) >> 1;
        if ((sh >= 64 ? 0 : keys[m] >> sh) < pre) a = m + 1;
        else b = m;
    }
    const int64_t lo = a;
    a = i + 1;
    b = wh;  // first index in (i, wh) past the prefix
    while (a < b) {
        const int64_t m = (a + b) >> 1;
        if ((sh >= 64 ? 0 : keys[m] >> sh) <= pre) a = m + 1;
        else b = m;
    }
    return a - lo;
}

__global__ void carve_count(const uint64_t *__restrict__ keys, int64_t n, int ncrit, int allow_big,
                            int32_t *ccount, int8_t *leaf_level, int32_t *level_hist, int *err) {
    __shared__ int32_t hist[MAX_LEVEL + 2];
    for (int k = threadIdx.x; k < MAX_LEVEL + 2; k += blockDim.x) hist[k] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        // smallest L in [0, 21] with run <= ncrit (monotone in L), else 21
        int lo = 0, hi = MAX_LEVEL;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (run_in_window(keys, n, i, mid, ncrit) <= ncrit) hi = mid;
            else lo = mid + 1;
        }
        const int leafL = lo;
        if (leafL == MAX_LEVEL && !allow_big && run_in_window(keys, n, i, MAX_LEVEL, ncrit) > ncrit)
            atomicExch(err, 1);
        const int ld = first_diff_level(keys, i);
        const int c = leafL >= ld ? leafL - ld + 1 : 0;
        ccount[i] = c;
        leaf_level[i] = (int8_t)leafL;
        for (int L = ld; L <= leafL; L++) atomicAdd(&hist[L], 1);
        if (c > 0) atomicAdd(&hist[MAX_LEVEL + 1], 1);  // body starts a leaf
    }
    __syncthreads();
    for (int k = threadIdx.x; k < MAX_LEVEL + 2; k += blockDim.x)
        if (hist[k]) atomicAdd(&level_hist[k], hist[k]);
}

__global__ void carve_emit(const uint64_t *__restrict__ keys, int64_t n, const int32_t *__restrict__ cbase,
                           const int8_t *__restrict__ leaf_level, int32_t *level_cursor, int32_t *children,
                           int32_t *parent, int8_t *level, uint64_t *key, int32_t *start, int32_t *end,
                           uint8_t *leaf, int32_t *cells_by_level) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int ld = first_diff_level(keys, i);
        const int leafL = leaf_level[i];
        for (int L = ld; L <= leafL; L++) {
            const int32_t c = cbase[i] + (L - ld);
            const int sh = 3 * (MAX_LEVEL - L);
            const uint64_t pre = sh >= 64 ? 0 : keys[i] >> sh;
            int64_t e = n;
            if (L > 0) {  // first body past this cell's prefix
                const uint64_t lim = (pre + 1) << sh;
                int64_t a = i + 1, b = n;
                while (a < b) {
                    const int64_t m = (a + b) >> 1;
                    if (keys[m] < lim) a = m + 1;
                    else b = m;
                }
                e = a;
            }
            start[c] = (int32_t)i;
            end[c] = (int32_t)e;
            level[c] = (int8_t)L;
            key[c] = pre;
            leaf[c] = L == leafL ? 1 : 0;
            int32_t pc = -1;
            if (L > 0) {
                if (L - 1 >= ld) {
                    pc = c - 1;  // the parent starts at the same body
                } else {     // the parent starts at the first body of the level-(L-1) prefix
                    const int psh = 3 * (MAX_LEVEL - (L - 1));
                    const uint64_t ppre = keys[i] >> psh;
                    int64_t a = 0, b = i;
                    while (a < b) {
                        const int64_t m = (a + b) >> 1;
                        if ((keys[m] >> psh) < ppre) a = m + 1;
                        else b = m;
                    }
                    pc = cbase[a] + (L - 1 - first_diff_level(keys, a));
                }
                children[pc * 8 + (int)(pre & 7ull)] = c;
            }
            parent[c] = pc;
            cells_by_level[atomicAdd(&level_cursor[L], 1)] = c;
        }
    }
}

__global__ void carve_links(int32_t ncells, const int32_t *__restrict__ start, const int32_t *__restrict__ end,
                            int32_t *sub_end) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ncells; j += gridDim.x * blockDim.x) {
        const int32_t e = end[j];
        int lo = j + 1, hi = ncells;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (start[mid] < e) lo = mid + 1;
            else hi = mid;
        }
        sub_end[j] = lo;
    }
}

__global__ void body_leaf_kernel(int32_t ncells, const uint8_t *leaf, const int32_t *start,
                                 const int32_t *end, int32_t *body_leaf) {
    // one warp per cell; leaves write their body range
    int lane = threadIdx.x & 31;
    for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < ncells;
         c += (gridDim.x * blockDim.x) >> 5) {
        if (!leaf[c]) continue;
        for (int32_t i = start[c] + lane; i < end[c]; i += 32) body_leaf[i] = c;
    }
}

// ---------------------------------------------------------------------------
// cell geometry (src/tree.py:80-160, cubic + geometric)
// ---------------------------------------------------------------------------
constexpr int kChunk = 1024;  // bodies per bmax work item

__global__ void geometry_cells(int32_t ncells, const int8_t *__restrict__ level,
                               const uint64_t *__restrict__ key, const int32_t *__restrict__ start,
                               const int32_t *__restrict__ end, const double *__restrict__ root,
                               double *lo, double *hi, double *ctr, double *rmax,
                               unsigned long long *b2, int32_t *nchunk) {
    const double r[3] = {root[0], root[1], root[2]};
    const double root_size = root[3];
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncells; c += gridDim.x * blockDim.x) {
        int lvl = level[c];
        double size = root_size / (double)(1ll << lvl);
        uint64_t full = key[c] << (3 * (MAX_LEVEL - lvl));
        double idx[3] = {(double)(compact21(full) >> (MAX_LEVEL - lvl)),
                         (double)(compact21(full >> 1) >> (MAX_LEVEL - lvl)),
                         (double)(compact21(full >> 2) >> (MAX_LEVEL - lvl))};
        double a[3];
        for (int d = 0; d < 3; d++) {
            double l = r[d] + idx[d] * size;
            double h = l + size;
            double m = 0.5 * (l + h);
            lo[c * 3 + d] = l;
            hi[c * 3 + d] = h;
            ctr[c * 3 + d] = m;
            double u = fabs(l - m), v = fabs(h - m);
            a[d] = (v > u) ? v : u;
        }
        rmax[c] = sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
        b2[c] = 0ull;
        nchunk[c] = (end[c] - start[c] + kChunk - 1) / kChunk;
    }
}

// rect and/or center-of-mass cells (src/tree.py:101-141): the tight box of
// the cell's bodies and the charge-weighted center, in the reference's
// sequential body order (bit-exact sums; one thread per cell -- a
// non-default mode, bounded by the root's N-body chain), then rmax again.
__global__ void geometry_rect_com(int32_t ncells, const int32_t *__restrict__ start,
                                  const int32_t *__restrict__ end, const double *__restrict__ xs,
                                  const double *__restrict__ ys, const double *__restrict__ zs,
                                  const double *__restrict__ qs, int rect, int com, double *lo, double *hi,
                                  double *ctr, double *rmax) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncells; c += gridDim.x * blockDim.x) {
        const int32_t s = start[c], e = end[c];
        if (rect) {
            double x0 = xs[s], x1 = xs[s], y0 = ys[s], y1 = ys[s], z0 = zs[s], z1 = zs[s];
            for (int32_t j = s + 1; j < e; j++) {
                const double x = xs[j], y = ys[j], z = zs[j];
                if (x < x0) x0 = x;
                if (x > x1) x1 = x;
                if (y < y0) y0 = y;
                if (y > y1) y1 = y;
                if (z < z0) z0 = z;
                if (z > z1) z1 = z;
            }
            lo[c * 3] = x0; lo[c * 3 + 1] = y0; lo[c * 3 + 2] = z0;
            hi[c * 3] = x1; hi[c * 3 + 1] = y1; hi[c * 3 + 2] = z1;
        }
        double m[3];
        bool mid = true;
        if (com) {
            double q = 0.0, cx = 0.0, cy = 0.0, cz = 0.0;
            for (int32_t j = s; j < e; j++) {
                const double qj = qs[j];
                q += qj;
                cx += qj * xs[j];
                cy += qj * ys[j];
                cz += qj * zs[j];
            }
            if (q != 0.0) {
                m[0] = cx / q;
                m[1] = cy / q;
                m[2] = cz / q;
                mid = false;
            }
        }
        double a[3];
        for (int d = 0; d < 3; d++) {
            const double l = lo[c * 3 + d], h = hi[c * 3 + d];
            if (mid) m[d] = 0.5 * (l + h);
            ctr[c * 3 + d] = m[d];
            const double u = fabs(l - m[d]), v = fabs(h - m[d]);
            a[d] = (v > u) ? v : u;
        }
        rmax[c] = sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
    }
}

__device__ inline int upper_bound_i32(const int32_t *a, int n, int32_t v) {
    int lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] <= v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// bmax accumulators and chunk counts alone (fmm_cell_bmax_range)
__global__ void bmax_chunks(int32_t ncells, const int32_t *__restrict__ start, const int32_t *__restrict__ end,
                            unsigned long long *b2, int32_t *nchunk) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncells; c += gridDim.x * blockDim.x) {
        b2[c] = 0ull;
        nchunk[c] = (end[c] - start[c] + kChunk - 1) / kChunk;
    }
}

__global__ void geometry_bmax(int32_t ncells, const int32_t *__restrict__ choff,
                              const int32_t *__restrict__ nchunk, const int32_t *__restrict__ start,
                              const int32_t *__restrict__ end, const double *__restrict__ ctr,
                              const double *__restrict__ xs, const double *__restrict__ ys,
                              const double *__restrict__ zs, unsigned long long *b2, int32_t body_lo = 0,
                              int32_t body_hi = 0x7fffffff) {
    const int lane = threadIdx.x & 31;
    const int total = choff[ncells - 1] + nchunk[ncells - 1];
    for (int it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < total;
         it += (gridDim.x * blockDim.x) >> 5) {
        int c = upper_bound_i32(choff, ncells, it) - 1;
        int k = it - choff[c];
        int32_t s = start[c] + k * kChunk;
        int32_t e = min(end[c], s + kChunk);
        s = max(s, body_lo);  // only the resident bodies (a rank's share, fmm_cell_bmax_range)
        e = min(e, body_hi);
        const double cx = ctr[c * 3], cy = ctr[c * 3 + 1], cz = ctr[c * 3 + 2];
        double best = 0.0;
        for (int32_t j = s + lane; j < e; j += 32) {
            double dx = xs[j] - cx, dy = ys[j] - cy, dz = zs[j] - cz;
            double d2 = dx * dx + dy * dy + dz * dz;
            if (d2 > best) best = d2;
        }
        for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0 && best > 0.0) atomicMax(&b2[c], (unsigned long long)__double_as_longlong(best));
    }
}

__global__ void geometry_finish(int32_t ncells, const unsigned long long *b2, double *bmax) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncells; c += gridDim.x * blockDim.x)
        bmax[c] = sqrt(__longlong_as_double((long long)b2[c]));
}

constexpr int kCarveStage = 3 + MAX_LEVEL + 2;

// Cell count (last exclusive-scan entry + its count) and the caller's flag
// into the staging block read back in one copy.
__global__ void carve_stage(const int32_t *__restrict__ cbase, const int32_t *__restrict__ ccount, int64_t n,
                            const int32_t *__restrict__ flag, int32_t *stage) {
    if (threadIdx.x == 0) {
        stage[0] = cbase[n - 1] + ccount[n - 1];
        stage[2] = flag ? *flag : 0;
    }
}

static size_t sort_temp_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, n, 0, 64);
    return bytes;
}

static size_t sortkeys_temp_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, bytes, (const uint64_t *)nullptr, (uint64_t *)nullptr, n, 0,
                                   64);
    return bytes;
}

static size_t scan_temp_bytes(int64_t n) {
    size_t a = 0, b = 0;
    cub::DeviceScan::InclusiveSum(nullptr, a, (const int32_t *)nullptr, (int32_t *)nullptr, n);
    cub::DeviceScan::ExclusiveSum(nullptr, b, (const int64_t *)nullptr, (int64_t *)nullptr, n);
    return a > b ? a : b;
}

size_t workspace_bytes(int64_t n) {
    int64_t m = n < 1024 ? 1024 : n;
    size_t s = sort_temp_bytes(m);
    size_t k = sortkeys_temp_bytes(m);
    size_t c = scan_temp_bytes(m);
    size_t t = s > k ? s : k;
    t = t > c ? t : c;
    // + two int32 arrays of m, one uint64 array of m, one int64 array of m, slack
    return t + (size_t)m * (4 + 4 + 8 + 8 + 8) + (1 << 20);
}

}  // namespace fmm

using namespace fmm;

extern "C" {

int fmm_abi_version(void) { return 1; }

const char *fmm_last_error(void) { return fmm::g_err; }

long long fmm_launch_count(void) { return fmm::g_launches.load(std::memory_order_relaxed); }

int fmm_device_sm_count(void) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return sms;
}

int fmm_workspace_bytes(int64_t n, size_t *host_bytes) {
    *host_bytes = fmm::workspace_bytes(n);
    return FMM_OK;
}

int fmm_ingest_bounds(const void *x, const void *y, const void *z, const void *q, int dtype, int64_t n,
                      double *x64, double *y64, double *z64, double *q64, double *root, void *ws,
                      size_t ws_bytes, void *stream) {
    if (n <= 0) { set_error("empty particle set"); return FMM_ERR_INVALID; }
    Arena ar(ws, ws_bytes);
    double *partial = ar.take<double>(kBoundsBlocks * 6);
    if (!partial) { set_error("workspace too small"); return FMM_ERR_INVALID; }
    cudaStream_t s = as_stream(stream);
    int nb = grid_for(n, 256, kBoundsBlocks);
    if (dtype == FMM_DTYPE_F64) {
        bool copy = (x != (const void *)x64);
        ingest_bounds_partial<double><<<nb, 256, 0, s>>>((const double *)x, (const double *)y,
                                                         (const double *)z, (const double *)q, n, x64,
                                                         y64, z64, q64, copy, partial); fmm::note_launch();
    } else if (dtype == FMM_DTYPE_F32) {
        ingest_bounds_partial<float><<<nb, 256, 0, s>>>((const float *)x, (const float *)y,
                                                        (const float *)z, (const float *)q, n, x64, y64,
                                                        z64, q64, true, partial); fmm::note_launch();
    } else {
        set_error("bad dtype %d", dtype);
        return FMM_ERR_INVALID;
    }
    bounds_final<<<1, 32, 0, s>>>(partial, nb, root); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_ingest_bounds");
    return FMM_OK;
}

int fmm_morton_keys(const double *x, const double *y, const double *z, int64_t n, const double *root,
                    uint64_t *keys, int32_t *iota, void *stream) {
    morton_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(x, y, z, n, root, keys, iota); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_morton_keys");
    return FMM_OK;
}

int fmm_sort_pairs_u64(const uint64_t *keys_in, const int32_t *vals_in, uint64_t *keys_out,
                       int32_t *vals_out, int64_t n, int end_bit, void *ws, size_t ws_bytes,
                       void *stream) {
    size_t need = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, keys_in, keys_out, vals_in, vals_out, n, 0, end_bit,
                                    as_stream(stream));
    if (need > ws_bytes) { set_error("sort workspace %zu > %zu", need, ws_bytes); return FMM_ERR_INVALID; }
    cub::DeviceRadixSort::SortPairs(ws, need, keys_in, keys_out, vals_in, vals_out, n, 0, end_bit,
                                    as_stream(stream));
    FMM_CUDA_CHECK("fmm_sort_pairs_u64");
    return FMM_OK;
}

int fmm_permute_bodies(const int32_t *perm, const double *x, const double *y, const double *z,
                       const double *q, int64_t n, double *xs, double *ys, double *zs, double *qs,
                       void *b32, void *b32lo, int *dev_inexact, void *stream) {
    permute_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(perm, x, y, z, q, n, xs, ys, zs, qs,
                                                                    (float4 *)b32, (float4 *)b32lo,
                                                                    dev_inexact); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_permute_bodies");
    return FMM_OK;
}

int fmm_carve_count(const uint64_t *keys, int64_t n, int32_t ncrit, int allow_big, int32_t *cbase,
                    int8_t *leaf_level, int32_t *host_level_hist, int32_t *host_ncells, const int32_t *dev_flag,
                    int32_t *host_flag, void *ws, size_t ws_bytes, void *stream) {
    cudaStream_t s = as_stream(stream);
    Arena ar(ws, ws_bytes);
    int32_t *ccount = ar.take<int32_t>(n);
    // staging for the one host read: {cell count, error, flag, hist[23]}
    int32_t *stage = ar.take<int32_t>(kCarveStage);
    if (!ccount || !stage) { set_error("workspace too small"); return FMM_ERR_INVALID; }
    int32_t *hist = stage + 3;
    cudaMemsetAsync(stage, 0, sizeof(int32_t) * kCarveStage, s);
    carve_count<<<grid_for(n, 256), 256, 0, s>>>(keys, n, ncrit, allow_big, ccount, leaf_level, hist, stage + 1); fmm::note_launch();
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, ccount, cbase, n, s);
    if (need > ar.left()) { set_error("scan workspace"); return FMM_ERR_INVALID; }
    cub::DeviceScan::ExclusiveSum(ar.rest(), need, ccount, cbase, n, s);
    carve_stage<<<1, 32, 0, s>>>(cbase, ccount, n, dev_flag, stage); fmm::note_launch();
    static thread_local int32_t *pinned = nullptr;
    if (!pinned && cudaMallocHost((void **)&pinned, sizeof(int32_t) * kCarveStage) != cudaSuccess)
        return cuda_status("fmm_carve_count pinned buffer");
    cudaMemcpyAsync(pinned, stage, sizeof(int32_t) * kCarveStage, cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_status("fmm_carve_count sync");
    *host_ncells = pinned[0];
    for (int L = 0; L < MAX_LEVEL + 2; L++) host_level_hist[L] = pinned[3 + L];
    if (host_flag) *host_flag = pinned[2];
    if (pinned[1]) {
        set_error("max depth exceeded: more than ncrit=%d bodies share one depth-%d grid cell "
                  "(pass allow_oversized_leaves=True to keep them in one leaf)",
                  ncrit, MAX_LEVEL);
        return FMM_ERR_MAX_DEPTH;
    }
    FMM_CUDA_CHECK("fmm_carve_count");
    return FMM_OK;
}

int fmm_carve_emit(const uint64_t *keys, int64_t n, const int32_t *cbase, const int8_t *leaf_level,
                   int32_t ncells, const int32_t *host_level_off, int32_t *children, int32_t *parent,
                   int8_t *level, uint64_t *key, int32_t *start, int32_t *end, int32_t *sub_end, uint8_t *leaf,
                   int32_t *cells_by_level, int32_t *body_leaf, void *ws, size_t ws_bytes, void *stream) {
    cudaStream_t s = as_stream(stream);
    Arena ar(ws, ws_bytes);
    int32_t *cursor = ar.take<int32_t>(MAX_LEVEL + 2);
    if (!cursor) { set_error("workspace too small"); return FMM_ERR_INVALID; }
    cudaMemcpyAsync(cursor, host_level_off, sizeof(int32_t) * (MAX_LEVEL + 2), cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(children, 0xFF, sizeof(int32_t) * 8 * (size_t)ncells, s);  // -1
    carve_emit<<<grid_for(n, 256), 256, 0, s>>>(keys, n, cbase, leaf_level, cursor, children, parent, level, key,
                                                start, end, leaf, cells_by_level); fmm::note_launch();
    carve_links<<<grid_for(ncells, 256), 256, 0, s>>>(ncells, start, end, sub_end); fmm::note_launch();
    body_leaf_kernel<<<grid_for((int64_t)ncells * 32, 256), 256, 0, s>>>(ncells, leaf, start, end, body_leaf); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_carve_emit");
    return FMM_OK;
}

int fmm_cell_geometry(int32_t ncells, const int8_t *level, const uint64_t *key, const int32_t *start,
                      const int32_t *end, const double *xs, const double *ys, const double *zs,
                      const double *qs, int rect, int com, const double *root, double *lo, double *hi,
                      double *ctr, double *bmax, double *rmax, void *ws, size_t ws_bytes, void *stream) {
    cudaStream_t s = as_stream(stream);
    Arena ar(ws, ws_bytes);
    unsigned long long *b2 = ar.take<unsigned long long>(ncells);
    int32_t *nchunk = ar.take<int32_t>(ncells);
    int32_t *choff = ar.take<int32_t>(ncells);
    if (!b2 || !nchunk || !choff) { set_error("workspace too small"); return FMM_ERR_INVALID; }
    int g = grid_for(ncells, 256);
    geometry_cells<<<g, 256, 0, s>>>(ncells, level, key, start, end, root, lo, hi, ctr, rmax, b2, nchunk); fmm::note_launch();
    if (rect || com) {
        if (com && !qs) { set_error("center_mode com needs the charges"); return FMM_ERR_INVALID; }
        geometry_rect_com<<<grid_for(ncells, 64), 64, 0, s>>>(ncells, start, end, xs, ys, zs, qs, rect, com, lo, hi,
                                                             ctr, rmax); fmm::note_launch();
    }
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, nchunk, choff, ncells, s);
    if (need > ar.left()) { set_error("scan workspace"); return FMM_ERR_INVALID; }
    cub::DeviceScan::ExclusiveSum(ar.rest(), need, nchunk, choff, ncells, s);
    geometry_bmax<<<148 * 8, 256, 0, s>>>(ncells, choff, nchunk, start, end, ctr, xs, ys, zs, b2); fmm::note_launch();
    geometry_finish<<<g, 256, 0, s>>>(ncells, b2, bmax); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_cell_geometry");
    return FMM_OK;
}


int fmm_cell_bmax_range(int32_t ncells, const int32_t *start, const int32_t *end, const double *ctr,
                        const double *xs, const double *ys, const double *zs, int32_t body_lo, int32_t body_hi,
                        double *bmax, void *ws, size_t ws_bytes, void *stream) {
    cudaStream_t s = as_stream(stream);
    Arena ar(ws, ws_bytes);
    unsigned long long *b2 = ar.take<unsigned long long>(ncells);
    int32_t *nchunk = ar.take<int32_t>(ncells);
    int32_t *choff = ar.take<int32_t>(ncells);
    if (!b2 || !nchunk || !choff) { set_error("workspace too small"); return FMM_ERR_INVALID; }
    int g = grid_for(ncells, 256);
    bmax_chunks<<<g, 256, 0, s>>>(ncells, start, end, b2, nchunk); fmm::note_launch();
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, nchunk, choff, ncells, s);
    if (need > ar.left()) { set_error("scan workspace"); return FMM_ERR_INVALID; }
    cub::DeviceScan::ExclusiveSum(ar.rest(), need, nchunk, choff, ncells, s);
    geometry_bmax<<<148 * 8, 256, 0, s>>>(ncells, choff, nchunk, start, end, ctr, xs, ys, zs, b2, body_lo, body_hi);
    fmm::note_launch();
    geometry_finish<<<g, 256, 0, s>>>(ncells, b2, bmax); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_cell_bmax_range");
    return FMM_OK;
}

}  // extern "C"
