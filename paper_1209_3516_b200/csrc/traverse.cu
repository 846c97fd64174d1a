// traverse.cu -- dual-tree traversal to CSR interaction lists
// (src/traversal.py:144-262, directed, one shared tree, MAC "fmm").
//
// The reference pops (a, b) pairs off a DFS stack; each pair's fate depends
// only on (a, b): both leaves -> P2P (tested BEFORE the MAC, so (a, a)
// leaf pairs are always P2P); else MAC accepted -> M2L; else open one
// side (a leaf -> open b; b leaf -> open a; rmax[a] >= rmax[b] -> open a;
// else open b) and push its non-empty children.  The emitted SETS are
// therefore independent of visiting order, and a breadth-first frontier
// over int32 pairs reproduces them exactly.  Compiled with --fmad=false so
// r2 and the squared MAC match the reference bit for bit.
//
// Emission uses warp-aggregated atomics on 64-bit counters that keep
// counting past capacity (the reference's overflow-and-retry contract,
// src/traversal.py:166-168); order is then fixed by a radix sort on
// (target, source), so the CSR output is deterministic.
#include <cub/cub.cuh>

#include "fmm_common.cuh"
#include "rowsort.cuh"

namespace fmm {

__device__ inline unsigned long long warp_reserve(unsigned long long *counter, int want, int lane,
                                                  int *my_off) {
    // inclusive scan of `want` over the warp, one atomic by the last lane
    int incl = want;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    int total = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && total > 0) base = atomicAdd(counter, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 31);
    *my_off = incl - want;
    return base;
}

// Fate of a pair (src/traversal.py:185-211): 1 = P2P (both leaves, tested
// before the MAC), 2 = M2L (MAC accepted), 3 = split.
// One tree's cell arrays as the traversals read them: the target tree A
// and the source tree B are the same arrays for a one-tree evaluation.
struct Cells {
    const int32_t *children;
    const uint8_t *leaf;
    const double *ctr, *bmax, *rmax;
};

// _mac_ok (src/traversal.py:144-156) for target a of A, source b of B:
// 0 = bh, 1 = bmax, 2 = fmm; r2 == 0 rejects.
__device__ __forceinline__ bool mac_accept(int32_t a, int32_t b, const Cells &A, const Cells &B, int kind_mac,
                                           double th2) {
    const double dx = A.ctr[a * 3] - B.ctr[b * 3];
    const double dy = A.ctr[a * 3 + 1] - B.ctr[b * 3 + 1];
    const double dz = A.ctr[a * 3 + 2] - B.ctr[b * 3 + 2];
    const double r2 = dx * dx + dy * dy + dz * dz;
    if (r2 == 0.0) return false;
    const double s = kind_mac == 2 ? A.bmax[a] + B.bmax[b] : (kind_mac == 1 ? B.bmax[b] : 2.0 * B.rmax[b]);
    return s * s < th2 * r2;
}

__device__ __forceinline__ int pair_fate(int32_t a, int32_t b, const Cells &A, const Cells &B, int kind_mac,
                                         double th2) {
    if (A.leaf[a] && B.leaf[b]) return 1;
    return mac_accept(a, b, A, B, kind_mac, th2) ? 2 : 3;
}

// One breadth-first step.  Every frontier pair is a pair already known to
// split; its children pairs are classified right here, so P2P and M2L
// pairs are emitted directly and only pairs that split again reach the
// next frontier (the root pair (0, 0) is classified by the first step,
// which the host launches with `classify_self = 1`).
__global__ void traverse_step_kernel(const int32_t *__restrict__ fa, const int32_t *__restrict__ fb,
                                     int64_t nfront_host, const unsigned long long *__restrict__ nfront_dev,
                                     int64_t cap_front, int classify_self, Cells A, Cells B,
                                     const int32_t *__restrict__ cstart, const int32_t *__restrict__ cend,
                                     int32_t blo, int32_t bhi, const uint8_t *__restrict__ tmask, int m2l_owner,
                                     int kind_mac, double th2, int32_t *p2p_t,
                                     int32_t *p2p_s, int64_t cap_p2p,
                                     int32_t *m2l_t, int32_t *m2l_s, int64_t cap_m2l, int32_t *na,
                                     int32_t *nb, int64_t cap_next, unsigned long long *cnt_p2p,
                                     unsigned long long *cnt_m2l, unsigned long long *cnt_next) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // the frontier size comes from the host or from the previous step's
    // counter on the device (sync-free chains of steps); entries past the
    // buffer capacity were never written
    int64_t nfront = nfront_dev ? (int64_t)*nfront_dev : nfront_host;
    if (nfront > cap_front) nfront = cap_front;
    // a range that covers the root's bodies filters nothing: skip the loads
    const bool ranged = blo > cstart[0] || bhi < cend[0];
    // iterate in warp-uniform trip counts so the shuffles see full warps
    const int64_t nround = (nfront + stride - 1) / stride;
    for (int64_t r = 0; r < nround; r++) {
        const int64_t k = r * stride + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        // children in their octant slots (absent ones flagged, not
        // compacted: a runtime slot index would turn every register array
        // access into a select chain)
        int32_t ca[8], cb[8];
        bool ok[8];
        int fate[8];
#pragma unroll
        for (int o = 0; o < 8; o++) ok[o] = false;
        // the side of the pair that is not opened is the same for all its
        // children: its leaf flag, centre and radius are read once
        bool open_a = false, lfix = false;
        double fx = 0.0, fy = 0.0, fz = 0.0, fbm = 0.0, frm = 0.0;
        if (k < nfront) {
            const int32_t a = fa[k], b = fb[k];
            if (classify_self) {
                ca[0] = a;
                cb[0] = b;
                ok[0] = true;
            } else {
                const bool la = A.leaf[a], lb = B.leaf[b];
                open_a = la ? false : (lb ? true : (A.rmax[a] >= B.rmax[b]));
                const Cells &F = open_a ? B : A;
                const int32_t f = open_a ? b : a;
                lfix = open_a ? lb : la;
                fx = F.ctr[f * 3];
                fy = F.ctr[f * 3 + 1];
                fz = F.ctr[f * 3 + 2];
                fbm = F.bmax[f];
                frm = F.rmax[f];
                const int32_t *kids = open_a ? A.children + a * 8 : B.children + b * 8;
#pragma unroll
                for (int o = 0; o < 8; o++) {
                    const int32_t ch = kids[o];
                    ok[o] = ch >= 0;
                    ca[o] = open_a ? ch : a;
                    cb[o] = open_a ? b : ch;
                }
            }
        }
        // pair_fate with the fixed side's values (same operations and order)
        auto fate_of = [&](int32_t a, int32_t b) {
            if (classify_self) return pair_fate(a, b, A, B, kind_mac, th2);
            const Cells &O = open_a ? A : B;
            const int32_t c = open_a ? a : b;  // the opened side's child
            if (lfix && O.leaf[c]) return 1;
            const double ax = open_a ? O.ctr[c * 3] : fx, ay = open_a ? O.ctr[c * 3 + 1] : fy,
                         az = open_a ? O.ctr[c * 3 + 2] : fz;
            const double bx = open_a ? fx : O.ctr[c * 3], by = open_a ? fy : O.ctr[c * 3 + 1],
                         bz = open_a ? fz : O.ctr[c * 3 + 2];
            const double dx = ax - bx, dy = ay - by, dz = az - bz;
            const double r2 = dx * dx + dy * dy + dz * dz;
            if (r2 == 0.0) return 3;
            const double bma = open_a ? O.bmax[c] : fbm, bmb = open_a ? fbm : O.bmax[c];
            const double rmb = open_a ? frm : O.rmax[c];
            const double sz = kind_mac == 2 ? bma + bmb : (kind_mac == 1 ? bmb : 2.0 * rmb);
            return sz * sz < th2 * r2 ? 2 : 3;
        };
        int np = 0, nm = 0, nn = 0;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            fate[q] = 0;
            if (ok[q]) {
                // multi-GPU: only targets whose body range meets [blo, bhi)
                if (ranged && (cend[ca[q]] <= blo || cstart[ca[q]] >= bhi)) continue;
                // target subset (sampled evaluations): only flagged target cells
                if (tmask && !tmask[ca[q]]) continue;
                fate[q] = fate_of(ca[q], cb[q]);
                // chunked single-GPU runs: an M2L pair belongs to the chunk
                // holding its target's first body (no pair is emitted twice)
                if (fate[q] == 2 && m2l_owner && (cstart[ca[q]] < blo || cstart[ca[q]] >= bhi)) fate[q] = 0;
                np += fate[q] == 1;
                nm += fate[q] == 2;
                nn += fate[q] == 3;
            }
        }
        int op, om, on;
        const unsigned long long bp = warp_reserve(cnt_p2p, np, lane, &op);
        const unsigned long long bm = warp_reserve(cnt_m2l, nm, lane, &om);
        const unsigned long long bn = warp_reserve(cnt_next, nn, lane, &on);
        unsigned long long ip = bp + op, im = bm + om, in = bn + on;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            if (fate[q] == 1) {
                if (ip < (unsigned long long)cap_p2p) { p2p_t[ip] = ca[q]; p2p_s[ip] = cb[q]; }
                ip++;
            } else if (fate[q] == 2) {
                if (im < (unsigned long long)cap_m2l) { m2l_t[im] = ca[q]; m2l_s[im] = cb[q]; }
                im++;
            } else if (fate[q] == 3) {
                if (in < (unsigned long long)cap_next) { na[in] = ca[q]; nb[in] = cb[q]; }
                in++;
            }
        }
    }
}

// ---- CSR by counting (sync-free) -------------------------------------------
// Row sizes by atomic counting, an exclusive scan, an atomic scatter and a
// segmented sort of every row's sources: the same (target, source)-sorted
// CSR as the radix path, but the pair count is read on the device, so the
// host never waits for the traversal.
// A thread's emitted pairs are contiguous and often share their target, so
// the warp groups equal targets (match_any) and one lane per group issues
// the atomic.  Trip counts are warp-uniform so the match sees full warps.
__global__ void row_count_kernel(const int32_t *__restrict__ t, const unsigned long long *__restrict__ dev_n,
                                 int64_t cap, unsigned long long *cnt) {
    int64_t n = (int64_t)*dev_n;
    if (n > cap) n = cap;
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t nround = (n + stride - 1) / stride;
    for (int64_t r = 0; r < nround; r++) {
        const int64_t k = r * stride + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        const int32_t key = k < n ? t[k] : -1;
        const unsigned grp = __match_any_sync(0xffffffffu, key);
        if (key >= 0 && lane == __ffs(grp) - 1) atomicAdd(&cnt[key], (unsigned long long)__popc(grp));
    }
}

__global__ void row_scatter_kernel(const int32_t *__restrict__ t, const int32_t *__restrict__ s,
                                   const unsigned long long *__restrict__ dev_n, int64_t cap,
                                   unsigned long long *cursor, int32_t *out) {
    int64_t n = (int64_t)*dev_n;
    if (n > cap) n = cap;
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t nround = (n + stride - 1) / stride;
    for (int64_t r = 0; r < nround; r++) {
        const int64_t k = r * stride + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        const int32_t key = k < n ? t[k] : -1;
        const unsigned grp = __match_any_sync(0xffffffffu, key);
        const int leader = __ffs(grp) - 1;
        unsigned long long base = 0;
        if (key >= 0 && lane == leader) base = atomicAdd(&cursor[key], (unsigned long long)__popc(grp));
        base = __shfl_sync(grp, base, leader);
        if (key >= 0) out[base + __popc(grp & ((1u << lane) - 1u))] = s[k];
    }
}

// Per-row sort of the scattered sources (a row's sources are distinct, so
// stability is moot): one CTA per row, the row in registers, a block radix
// sort over the source-id bits.  Rows longer than the tile are queued for
// the large-tile kernel (and, past its tile, the in-memory bitonic one).
constexpr int kRowSmallThreads = 256, kRowSmallItems = 4;    // 1024 keys
constexpr int kRowLargeThreads = 512, kRowLargeItems = 16;   // 8192 keys

template <int THREADS, int ITEMS>
__device__ __forceinline__ void row_sort_tile(const int32_t *in, int32_t *out, int64_t len, int nbits,
                                              typename cub::BlockRadixSort<int32_t, THREADS, ITEMS>::TempStorage &tmp) {
    int32_t keys[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        const int64_t k = (int64_t)i * THREADS + threadIdx.x;  // striped load
        keys[i] = k < len ? in[k] : (int32_t)((1u << nbits) - 1u);
    }
    // ids are below 2^nbits, so the all-ones pads sort last (a pad equal to
    // an id is indistinguishable from it in the output)
    cub::BlockRadixSort<int32_t, THREADS, ITEMS>(tmp).SortBlockedToStriped(keys, 0, nbits);
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        const int64_t k = (int64_t)i * THREADS + threadIdx.x;
        if (k < len) out[k] = keys[i];
    }
}

__global__ void __launch_bounds__(kRowSmallThreads) row_sort_small_kernel(
    int32_t ncells, const int64_t *__restrict__ rows, const int32_t *__restrict__ in, int32_t *out, int nbits,
    int32_t *long_rows, unsigned long long *nlong) {
    __shared__ typename cub::BlockRadixSort<int32_t, kRowSmallThreads, kRowSmallItems>::TempStorage tmp;
    for (int32_t r = blockIdx.x; r < ncells; r += gridDim.x) {
        const int64_t b = rows[r], len = rows[r + 1] - b;
        if (len <= 1) {
            if (len == 1 && threadIdx.x == 0) out[b] = in[b];
            continue;
        }
        if (len > (int64_t)kRowSmallThreads * kRowSmallItems) {
            if (threadIdx.x == 0) long_rows[atomicAdd(nlong, 1ull)] = r;
            continue;
        }
        row_sort_tile<kRowSmallThreads, kRowSmallItems>(in + b, out + b, len, nbits, tmp);
        __syncthreads();  // tmp is reused by the next row
    }
}

__global__ void __launch_bounds__(kRowLargeThreads) row_sort_large_kernel(
    const int64_t *__restrict__ rows, const int32_t *__restrict__ in, int32_t *out, int nbits,
    const int32_t *__restrict__ long_rows, const unsigned long long *__restrict__ nlong, int32_t *huge_rows,
    unsigned long long *nhuge) {
    __shared__ typename cub::BlockRadixSort<int32_t, kRowLargeThreads, kRowLargeItems>::TempStorage tmp;
    const int64_t n = (int64_t)*nlong;
    for (int64_t k = blockIdx.x; k < n; k += gridDim.x) {
        const int32_t r = long_rows[k];
        const int64_t b = rows[r], len = rows[r + 1] - b;
        if (len > (int64_t)kRowLargeThreads * kRowLargeItems) {
            if (threadIdx.x == 0) huge_rows[atomicAdd(nhuge, 1ull)] = r;
            continue;
        }
        row_sort_tile<kRowLargeThreads, kRowLargeItems>(in + b, out + b, len, nbits, tmp);
        __syncthreads();
    }
}

// Bitmap sort (rowsort.cuh): one warp per row.
constexpr int kRowBitmapWarps = 8;
constexpr int kRowSparseWarps = 4;
#ifndef FMM_SORT_MINB
#define FMM_SORT_MINB 8
#endif

// Rows whose ids fit one bitmap pass (or are too long to stage) are sorted
// here; wide rows of up to kSparseMax ids are queued for the sparse kernel,
// which stages them in shared memory and visits only their non-empty
// windows.
__global__ void __launch_bounds__(kRowBitmapWarps * 32) row_sort_bitmap_kernel(
    int32_t ncells, const int64_t *__restrict__ rows, const int32_t *__restrict__ in, int32_t *out,
    int32_t *wide_rows, unsigned long long *nwide) {
    __shared__ uint32_t bm_all[kRowBitmapWarps][kSortSegWords];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int32_t r = blockIdx.x * kRowBitmapWarps + w; r < ncells; r += gridDim.x * kRowBitmapWarps) {
        const int64_t k0 = rows[r], k1 = rows[r + 1];
        if (k1 - k0 <= kSparseMax && row_is_wide(in, k0, k1, lane)) {
            if (lane == 0) wide_rows[atomicAdd(nwide, 1ull)] = r;
            continue;
        }
        warp_bitmap_sort(in, out, k0, k1, bm_all[w], lane);
    }
}

__global__ void __launch_bounds__(kRowSparseWarps * 32, FMM_SORT_MINB) row_sort_sparse_kernel(const int64_t *__restrict__ rows,
                                                                             const int32_t *__restrict__ in,
                                                                             int32_t *out,
                                                                             const int32_t *__restrict__ wide_rows,
                                                                             const unsigned long long *__restrict__ nwide) {
    __shared__ uint32_t bm_all[kRowSparseWarps][kSortSegWords];
    __shared__ uint32_t ent_all[kRowSparseWarps][kSparseMax];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int x = lane; x < kSortSegWords; x += 32) bm_all[w][x] = 0u;
    __syncwarp();
    const int64_t n = (int64_t)*nwide;
    for (int64_t k = (int64_t)blockIdx.x * kRowSparseWarps + w; k < n; k += (int64_t)gridDim.x * kRowSparseWarps) {
        const int32_t r = wide_rows[k];
        warp_bitmap_sort_sparse(in, out, rows[r], rows[r + 1] - rows[r], bm_all[w], ent_all[w], lane);
    }
}

static int sort_rows_launch(int32_t ncells, const int64_t *rows, const int32_t *in, int32_t *out, int32_t *wide_rows,
                            unsigned long long *nwide, cudaStream_t st) {
    cudaMemsetAsync(nwide, 0, sizeof(unsigned long long), st);
    row_sort_bitmap_kernel<<<grid_for(ncells, kRowBitmapWarps, 148 * 8), kRowBitmapWarps * 32, 0, st>>>(
        ncells, rows, in, out, wide_rows, nwide); fmm::note_launch();
    row_sort_sparse_kernel<<<148 * (FMM_SORT_MINB > 6 ? FMM_SORT_MINB : 6), kRowSparseWarps * 32, 0, st>>>(rows, in, out, wide_rows, nwide); fmm::note_launch();
    return FMM_OK;
}

// Rows past the large tile: copy, then an all-ascending bitonic sort in
// global memory by one CTA (a mirrored compare opens every merge, so the
// virtual +inf entries past the row never move and need no storage).
__global__ void __launch_bounds__(1024) row_sort_huge_kernel(const int64_t *__restrict__ rows,
                                                             const int32_t *__restrict__ in, int32_t *out,
                                                             const int32_t *__restrict__ huge_rows,
                                                             const unsigned long long *__restrict__ nhuge) {
    const int64_t n = (int64_t)*nhuge;
    for (int64_t k = blockIdx.x; k < n; k += gridDim.x) {
        const int32_t r = huge_rows[k];
        const int64_t b = rows[r], len = rows[r + 1] - b;
        int32_t *v = out + b;
        for (int64_t i = threadIdx.x; i < len; i += blockDim.x) v[i] = in[b + i];
        int64_t p2 = 1;
        while (p2 < len) p2 <<= 1;
        __syncthreads();
        for (int64_t size = 2; size <= p2; size <<= 1) {
            const int64_t half = size >> 1;
            for (int64_t i = threadIdx.x; i < p2 / 2; i += blockDim.x) {
                const int64_t lo = (i / half) * size + (i % half), hi = (i / half) * size + size - 1 - (i % half);
                if (hi < len) {
                    const int32_t x = v[lo], y = v[hi];
                    if (x > y) { v[lo] = y; v[hi] = x; }
                }
            }
            __syncthreads();
            for (int64_t stride = half >> 1; stride > 0; stride >>= 1) {
                for (int64_t i = threadIdx.x; i < p2 / 2; i += blockDim.x) {
                    const int64_t lo = (i / stride) * stride * 2 + (i % stride), hi = lo + stride;
                    if (hi < len) {
                        const int32_t x = v[lo], y = v[hi];
                        if (x > y) { v[lo] = y; v[hi] = x; }
                    }
                }
                __syncthreads();
            }
        }
        __syncthreads();
    }
}

// ---- CSR ----------------------------------------------------------------
// ---- treecode (src/traversal.py:265-313) ----------------------------------
// Per target leaf t the reference walks the source tree from the root and
// classifies each (t, c) it pops: MAC accepted -> M2P (tested FIRST, so a
// leaf source far enough away is M2P); else c a leaf -> P2P; else push c's
// non-empty children.  The sets are independent of visiting order, so a
// breadth-first frontier over (t, c) pairs -- one source level per step --
// reproduces them.  The seed frontier is every leaf whose bodies meet
// [blo, bhi), paired with the root.
__global__ void treecode_seed_flags(int32_t ncells, const uint8_t *__restrict__ leaf,
                                    const int32_t *__restrict__ cstart, const int32_t *__restrict__ cend,
                                    int32_t blo, int32_t bhi, uint8_t *flag, int32_t *fb) {
    for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < ncells; c += gridDim.x * blockDim.x) {
        flag[c] = leaf[c] && cend[c] > blo && cstart[c] < bhi;
        fb[c] = 0;  // every seed pair starts at the root
    }
}

__global__ void treecode_step_kernel(const int32_t *__restrict__ fa, const int32_t *__restrict__ fb,
                                     const unsigned long long *__restrict__ nfront_dev, int64_t cap_front, Cells A,
                                     Cells B, int kind_mac, double th2,
                                     int32_t *m2p_t, int32_t *m2p_s, int64_t cap_m2p, int32_t *p2p_t,
                                     int32_t *p2p_s, int64_t cap_p2p, int32_t *na, int32_t *nb, int64_t cap_next,
                                     unsigned long long *cnt_p2p, unsigned long long *cnt_m2p,
                                     unsigned long long *cnt_next) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t nfront = (int64_t)*nfront_dev;
    if (nfront > cap_front) nfront = cap_front;
    const int64_t nround = (nfront + stride - 1) / stride;
    for (int64_t r = 0; r < nround; r++) {
        const int64_t k = r * stride + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        int fate = 0;  // 1 = P2P, 2 = M2P, 3 = open the source
        int32_t t = 0, c = 0;
        int nch = 0;
        if (k < nfront) {
            t = fa[k];
            c = fb[k];
            if (mac_accept(t, c, A, B, kind_mac, th2)) fate = 2;
            else if (B.leaf[c]) fate = 1;
            else {
                fate = 3;
#pragma unroll
                for (int o = 0; o < 8; o++) nch += B.children[c * 8 + o] >= 0;
            }
        }
        int op, om, on;
        const unsigned long long bp = warp_reserve(cnt_p2p, fate == 1, lane, &op);
        const unsigned long long bm = warp_reserve(cnt_m2p, fate == 2, lane, &om);
        const unsigned long long bn = warp_reserve(cnt_next, nch, lane, &on);
        if (fate == 1) {
            const unsigned long long ip = bp + op;
            if (ip < (unsigned long long)cap_p2p) { p2p_t[ip] = t; p2p_s[ip] = c; }
        } else if (fate == 2) {
            const unsigned long long im = bm + om;
            if (im < (unsigned long long)cap_m2p) { m2p_t[im] = t; m2p_s[im] = c; }
        } else if (fate == 3) {
            unsigned long long in = bn + on;
#pragma unroll
            for (int o = 0; o < 8; o++) {
                const int32_t ch = B.children[c * 8 + o];
                if (ch >= 0) {
                    if (in < (unsigned long long)cap_next) { na[in] = t; nb[in] = ch; }
                    in++;
                }
            }
        }
    }
}

// ---- listfmm (src/traversal.py:314-497) ---------------
// Level-wise lists on the cubic tree, theta-free.  V list: for every cell
// c, the children of the parent's 3x3x3 neighbourhood that are not adjacent
// to c (M2L).  U list: for every leaf t, its own-level neighbourhood (a leaf
// neighbour itself, an internal one all its descendant leaves, swept over
// the contiguous pre-order subtree) plus the leaf cells of every coarser
// ancestor's neighbourhood (P2P).  Same-level neighbours are found by binary
// search in the (level, key) table: the pre-order ids stably sorted by level
// list each level in pre-order, which is key order.
// Every thread walks its target twice: count, one warp-aggregated reserve,
// then write -- the emitted SETS are the reference's.
__device__ __forceinline__ int64_t level_lookup(const uint64_t *__restrict__ skeys, int64_t lo, int64_t hi,
                                                uint64_t key) {
    const int64_t hi0 = hi;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (skeys[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return (lo < hi0 && skeys[lo] == key) ? lo : -1;
}

__device__ __forceinline__ uint64_t interleave3(int64_t ix, int64_t iy, int64_t iz) {
    return spread21((uint64_t)ix) | (spread21((uint64_t)iy) << 1) | (spread21((uint64_t)iz) << 2);
}

struct LevelTable {
    const int32_t *cells;  // cells_by_level
    const uint64_t *keys;  // key[cells_by_level]
    const int64_t *off;    // level offsets (depth + 2)
};

__global__ void fill_iota(int32_t *a, int32_t n) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

__global__ void gather_keys(int32_t n, const int32_t *__restrict__ cells, const uint64_t *__restrict__ key,
                            uint64_t *out) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = key[cells[i]];
}

// V list of cell c: calls f(ch) for every well-separated child of the
// parent's neighbourhood, in the reference's (z, y, x, octant) order.
template <class F>
__device__ __forceinline__ void vlist_walk(int32_t c, const int8_t *__restrict__ level,
                                           const uint64_t *__restrict__ key, const int32_t *__restrict__ parent,
                                           const int32_t *__restrict__ children, const LevelTable &tab, F &&f) {
    const int lvl = level[c];
    if (lvl == 0) return;
    const uint64_t k = key[c];
    const int64_t ix = (int64_t)compact21(k), iy = (int64_t)compact21(k >> 1), iz = (int64_t)compact21(k >> 2);
    const uint64_t pk = key[parent[c]];
    const int64_t px = (int64_t)compact21(pk), py = (int64_t)compact21(pk >> 1), pz = (int64_t)compact21(pk >> 2);
    const int plvl = lvl - 1;
    const int64_t ng = (int64_t)1 << plvl;
    for (int dz = -1; dz <= 1; dz++) {
        const int64_t jz = pz + dz;
        if (jz < 0 || jz >= ng) continue;
        for (int dy = -1; dy <= 1; dy++) {
            const int64_t jy = py + dy;
            if (jy < 0 || jy >= ng) continue;
            for (int dx = -1; dx <= 1; dx++) {
                const int64_t jx = px + dx;
                if (jx < 0 || jx >= ng) continue;
                const int64_t pos = level_lookup(tab.keys, tab.off[plvl], tab.off[plvl + 1], interleave3(jx, jy, jz));
                if (pos < 0) continue;
                const int32_t nc = tab.cells[pos];
                for (int o = 0; o < 8; o++) {
                    const int32_t ch = children[nc * 8 + o];
                    if (ch < 0) continue;
                    const uint64_t ck = key[ch];
                    const int64_t ddx = (int64_t)compact21(ck) - ix, ddy = (int64_t)compact21(ck >> 1) - iy,
                                  ddz = (int64_t)compact21(ck >> 2) - iz;
                    if (ddx >= -1 && ddx <= 1 && ddy >= -1 && ddy <= 1 && ddz >= -1 && ddz <= 1) continue;
                    f(ch);
                }
            }
        }
    }
}

// U list of leaf t: calls f(s) for every near-field source leaf.
template <class F>
__device__ __forceinline__ void ulist_walk(int32_t t, const int8_t *__restrict__ level,
                                           const uint64_t *__restrict__ key, const uint8_t *__restrict__ leaf,
                                           const int32_t *__restrict__ sub_end, const LevelTable &tab, F &&f) {
    const int lvl = level[t];
    const uint64_t k = key[t];
    const int64_t ix = (int64_t)compact21(k), iy = (int64_t)compact21(k >> 1), iz = (int64_t)compact21(k >> 2);
    const int64_t ng = (int64_t)1 << lvl;
    for (int dz = -1; dz <= 1; dz++) {
        const int64_t jz = iz + dz;
        if (jz < 0 || jz >= ng) continue;
        for (int dy = -1; dy <= 1; dy++) {
            const int64_t jy = iy + dy;
            if (jy < 0 || jy >= ng) continue;
            for (int dx = -1; dx <= 1; dx++) {
                const int64_t jx = ix + dx;
                if (jx < 0 || jx >= ng) continue;
                const int64_t pos = level_lookup(tab.keys, tab.off[lvl], tab.off[lvl + 1], interleave3(jx, jy, jz));
                if (pos < 0) continue;
                const int32_t c = tab.cells[pos];
                if (leaf[c]) f(c);
                else
                    for (int32_t d = c; d < sub_end[c]; d++)
                        if (leaf[d]) f(d);
            }
        }
    }
    uint64_t ak = k;
    for (int lv = lvl - 1; lv > 0; lv--) {
        ak >>= 3;
        const int64_t ax = (int64_t)compact21(ak), ay = (int64_t)compact21(ak >> 1), az = (int64_t)compact21(ak >> 2);
        const int64_t ngl = (int64_t)1 << lv;
        for (int dz = -1; dz <= 1; dz++) {
            const int64_t jz = az + dz;
            if (jz < 0 || jz >= ngl) continue;
            for (int dy = -1; dy <= 1; dy++) {
                const int64_t jy = ay + dy;
                if (jy < 0 || jy >= ngl) continue;
                for (int dx = -1; dx <= 1; dx++) {
                    if (dx == 0 && dy == 0 && dz == 0) continue;  // the ancestor itself
                    const int64_t jx = ax + dx;
                    if (jx < 0 || jx >= ngl) continue;
                    const int64_t pos =
                        level_lookup(tab.keys, tab.off[lv], tab.off[lv + 1], interleave3(jx, jy, jz));
                    if (pos < 0) continue;
                    const int32_t c = tab.cells[pos];
                    if (leaf[c]) f(c);
                }
            }
        }
    }
}

__global__ void listfmm_kernel(int32_t ncells, const int8_t *__restrict__ level, const uint64_t *__restrict__ key,
                               const int32_t *__restrict__ parent, const int32_t *__restrict__ children,
                               const uint8_t *__restrict__ leaf, const int32_t *__restrict__ sub_end,
                               const int32_t *__restrict__ cstart, const int32_t *__restrict__ cend, int32_t blo,
                               int32_t bhi, LevelTable tab, int32_t *m2l_t, int32_t *m2l_s, int64_t cap_m2l,
                               int32_t *p2p_t, int32_t *p2p_s, int64_t cap_p2p, unsigned long long *cnt_p2p,
                               unsigned long long *cnt_m2l) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t nround = (ncells + stride - 1) / stride;
    for (int64_t r = 0; r < nround; r++) {
        const int64_t k = r * stride + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        const bool mine = k < ncells && cend[k] > blo && cstart[k] < bhi;
        const int32_t c = (int32_t)k;
        int nv = 0, nu = 0;
        if (mine) {
            vlist_walk(c, level, key, parent, children, tab, [&](int32_t) { nv++; });
            if (leaf[c]) ulist_walk(c, level, key, leaf, sub_end, tab, [&](int32_t) { nu++; });
        }
        int ov, ou;
        unsigned long long iv = warp_reserve(cnt_m2l, nv, lane, &ov) + ov;
        unsigned long long iu = warp_reserve(cnt_p2p, nu, lane, &ou) + ou;
        if (mine) {
            vlist_walk(c, level, key, parent, children, tab, [&](int32_t s) {
                if (iv < (unsigned long long)cap_m2l) { m2l_t[iv] = c; m2l_s[iv] = s; }
                iv++;
            });
            if (leaf[c])
                ulist_walk(c, level, key, leaf, sub_end, tab, [&](int32_t s) {
                    if (iu < (unsigned long long)cap_p2p) { p2p_t[iu] = c; p2p_s[iu] = s; }
                    iu++;
                });
        }
    }
}

__global__ void pack_pairs(const int32_t *t, const int32_t *s, int64_t n, int sbits, uint64_t *keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        keys[i] = ((uint64_t)(uint32_t)t[i] << sbits) | (uint64_t)(uint32_t)s[i];
}

__global__ void unpack_rows(const uint64_t *keys, int64_t n, int sbits, int32_t ncells, int32_t *src,
                            int64_t *rows) {
    const uint64_t mask = (1ull << sbits) - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = keys[i];
        src[i] = (int32_t)(k & mask);
        int32_t t = (int32_t)(k >> sbits);
        int32_t tprev = i > 0 ? (int32_t)(keys[i - 1] >> sbits) : -1;
        // rows[c] for every c in (tprev, t] starts at i
        for (int32_t c = tprev + 1; c <= t; c++) rows[c] = i;
        if (i == n - 1)
            for (int32_t c = t + 1; c <= ncells; c++) rows[c] = n;
    }
}

// 32-bit variant when (target, source) fit in 32 bits: half the sort traffic
__global__ void pack_pairs32(const int32_t *t, const int32_t *s, int64_t n, int sbits, uint32_t *keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        keys[i] = ((uint32_t)t[i] << sbits) | (uint32_t)s[i];
}

__global__ void unpack_rows32(const uint32_t *keys, int64_t n, int sbits, int32_t ncells, int32_t *src,
                              int64_t *rows) {
    const uint32_t mask = (1u << sbits) - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        src[i] = (int32_t)(k & mask);
        const int32_t t = (int32_t)(k >> sbits);
        const int32_t tprev = i > 0 ? (int32_t)(keys[i - 1] >> sbits) : -1;
        for (int32_t c = tprev + 1; c <= t; c++) rows[c] = i;
        if (i == n - 1)
            for (int32_t c = t + 1; c <= ncells; c++) rows[c] = n;
    }
}

__global__ void fill_i64(int64_t *a, int64_t n, int64_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        a[i] = v;
}

}  // namespace fmm

using namespace fmm;

// The source tree's arrays default to the target tree's (one-tree evaluation).
// ---- mutual traversal ---------------------------------
// Partition owner (src/traversal.py:621-640): the reference's partition
// roots are the maximal subtrees holding fewer than `grain` bodies (leaves
// included), so a cell is unowned (-1) iff it is internal with >= grain
// bodies, and otherwise owned by its highest ancestor-or-self whose parent
// is unowned.
__global__ void partition_owner_kernel(int32_t ncells, const int32_t *__restrict__ parent,
                                       const uint8_t *__restrict__ leaf, const int32_t *__restrict__ cstart,
                                       const int32_t *__restrict__ cend, int64_t grain, int32_t *owner) {
    for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < ncells; c += gridDim.x * blockDim.x) {
        int32_t r = -1;
        if (leaf[c] || (int64_t)(cend[c] - cstart[c]) < grain) {
            r = c;
            while (r != 0) {
                const int32_t up = parent[r];
                if ((int64_t)(cend[up] - cstart[up]) >= grain) break;
                r = up;
            }
        }
        owner[c] = r;
    }
}

// Children pairs of an unresolved pair (src/traversal.py:222-256): a leaf
// -> b's children; b leaf -> a's; a mutual self pair -> (ci, ci) and
// (ci, cj), i < j; else the larger rmax opens (ties: the target).
template <class F>
__device__ __forceinline__ void for_split(int32_t a, int32_t b, int m, const Cells &C, F &&f) {
    const int32_t *ka = C.children + (int64_t)a * 8, *kb = C.children + (int64_t)b * 8;
    if (C.leaf[a]) {
        for (int o = 0; o < 8; o++) if (kb[o] >= 0) f(a, kb[o]);
    } else if (C.leaf[b]) {
        for (int o = 0; o < 8; o++) if (ka[o] >= 0) f(ka[o], b);
    } else if (m && a == b) {
        for (int i = 0; i < 8; i++) {
            const int32_t ci = ka[i];
            if (ci < 0) continue;
            f(ci, ci);
            for (int j = i + 1; j < 8; j++) if (ka[j] >= 0) f(ci, ka[j]);
        }
    } else if (C.rmax[a] >= C.rmax[b]) {
        for (int o = 0; o < 8; o++) if (ka[o] >= 0) f(ka[o], b);
    } else {
        for (int o = 0; o < 8; o++) if (kb[o] >= 0) f(a, kb[o]);
    }
}

// One breadth-first step of the mutual traversal.  Frontier entries are
// (a, b, mut) pairs that must be SPLIT (mut in bit 31 of fb); step 0 holds
// the unclassified seed (classify_self).  Each child pair of a split is
// first demoted when mutual and its cells have different partition owners
// -- the directed pairs (x, y) and (y, x), the reference's driver
// (src/traversal.py:727-738) -- and every resulting item is classified
// with the unit rules on the spot (both leaves -> P2P; MAC, both
// directions when mutual -> M2L; else it enters the next frontier), so
// P2P and M2L pairs never pass through the frontier buffers (C2: 1.47 ->
// ~0.6 ms for the 12 steps).  Emitted lists are DIRECTED: a mutual entry
// (a, b) is written as (a, b) and, when a != b, (b, a) -- the reference's
// trace expansion (src/traversal.py:644-650) -- so the directed M2L / P2P
// executors run them unchanged.  Only targets whose bodies meet [blo, bhi)
// are emitted.
__global__ void mutual_step_kernel(const int32_t *__restrict__ fa, const int32_t *__restrict__ fb,
                                   const unsigned long long *__restrict__ nfront_dev, int64_t cap_front,
                                   int classify_self, Cells C, const int32_t *__restrict__ owner,
                                   const int32_t *__restrict__ cstart, const int32_t *__restrict__ cend, int32_t blo,
                                   int32_t bhi, int kind_mac, double th2, int32_t *p2p_t, int32_t *p2p_s,
                                   int64_t cap_p2p, int32_t *m2l_t, int32_t *m2l_s, int64_t cap_m2l, int32_t *na,
                                   int32_t *nb, int64_t cap_next, unsigned long long *cnt_p2p,
                                   unsigned long long *cnt_m2l, unsigned long long *cnt_next, int32_t *sp_a,
                                   int32_t *sp_b, int64_t cap_sp, int32_t *sm_a, int32_t *sm_b, int64_t cap_sm,
                                   unsigned long long *cnt_sym) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t nfront = (int64_t)*nfront_dev;
    if (nfront > cap_front) nfront = cap_front;
    const int64_t nround = (nfront + stride - 1) / stride;
    auto keep = [&](int32_t c) { return cend[c] > blo && cstart[c] < bhi; };
    // a mutual entry whose two members are both kept stays UNORDERED when
    // the caller gave a symmetric list for its kind (fmm_traverse_mutual_sym)
    auto sym_p2p = [&](int32_t x, int32_t y, int mm) { return sp_a && mm && x != y && keep(x) && keep(y); };
    auto sym_m2l = [&](int32_t x, int32_t y, int mm) { return sm_a && mm && x != y && keep(x) && keep(y); };
    // an item's fate: 1 P2P, 2 M2L, 3 split
    auto fate_of = [&](int32_t x, int32_t y, int m) {
        if (C.leaf[x] && C.leaf[y]) return 1;
        if (mac_accept(x, y, C, C, kind_mac, th2) && (!m || mac_accept(y, x, C, C, kind_mac, th2))) return 2;
        return 3;
    };
    // the items of a pair entering classification (demotion of a mutual
    // pair across partition owners), each handed to g(x, y, m)
    auto items = [&](int32_t x, int32_t y, int m, auto &&g) {
        if (m && owner[x] >= 0 && owner[y] >= 0 && owner[x] != owner[y]) {
            g(x, y, 0);
            g(y, x, 0);
        } else {
            g(x, y, m);
        }
    };
    auto children = [&](int32_t a, int32_t b, int m, auto &&g) {
        if (classify_self) items(a, b, m, g);
        else for_split(a, b, m, C, [&](int32_t x, int32_t y) { items(x, y, m, g); });
    };
    for (int64_t r = 0; r < nround; r++) {
        const int64_t k = r * stride + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        int32_t a = 0, b = 0;
        int m = 0;
        const bool live = k < nfront;
        if (live) {
            a = fa[k];
            b = fb[k] & 0x7fffffff;
            m = (int)((uint32_t)fb[k] >> 31);
        }
        // the fates of the first 32 items are kept (2 bits each) for the
        // write pass; only a mutual self split has more (36 children)
        int np = 0, nm = 0, nn = 0, nit = 0, nsp = 0, nsm = 0;
        uint64_t fbits = 0;
        if (live)
            children(a, b, m, [&](int32_t x, int32_t y, int mm) {
                const int ft = fate_of(x, y, mm);
                if (nit < 32) fbits |= (uint64_t)ft << (2 * nit);
                nit++;
                if (ft == 1) {
                    if (sym_p2p(x, y, mm)) nsp++;
                    else np += keep(x) + (mm && x != y && keep(y));
                } else if (ft == 2) {
                    if (sym_m2l(x, y, mm)) nsm++;
                    else nm += keep(x) + (mm && keep(y));
                } else {
                    nn += keep(x) || (mm && keep(y));
                }
            });
        int op, om, on, osp = 0, osm = 0;
        const unsigned long long bp = warp_reserve(cnt_p2p, np, lane, &op);
        const unsigned long long bm = warp_reserve(cnt_m2l, nm, lane, &om);
        const unsigned long long bn = warp_reserve(cnt_next, nn, lane, &on);
        const unsigned long long bsp = sp_a ? warp_reserve(cnt_sym, nsp, lane, &osp) : 0ull;
        const unsigned long long bsm = sm_a ? warp_reserve(cnt_sym + 1, nsm, lane, &osm) : 0ull;
        unsigned long long ip = bp + op, im = bm + om, in = bn + on, isp = bsp + osp, ism = bsm + osm;
        int it = 0;
        if (live)
            children(a, b, m, [&](int32_t x, int32_t y, int mm) {
                const int ft = it < 32 ? (int)((fbits >> (2 * it)) & 3u) : fate_of(x, y, mm);
                it++;
                if (ft == 1 && sym_p2p(x, y, mm)) {
                    if (isp < (unsigned long long)cap_sp) { sp_a[isp] = min(x, y); sp_b[isp] = max(x, y); }
                    isp++;
                } else if (ft == 2 && sym_m2l(x, y, mm)) {
                    if (ism < (unsigned long long)cap_sm) { sm_a[ism] = min(x, y); sm_b[ism] = max(x, y); }
                    ism++;
                } else if (ft == 1 || ft == 2) {
                    int32_t *tt = ft == 1 ? p2p_t : m2l_t, *ss = ft == 1 ? p2p_s : m2l_s;
                    const unsigned long long cap = (unsigned long long)(ft == 1 ? cap_p2p : cap_m2l);
                    unsigned long long &at = ft == 1 ? ip : im;
                    if (keep(x)) {
                        if (at < cap) { tt[at] = x; ss[at] = y; }
                        at++;
                    }
                    if (mm && (ft == 2 || x != y) && keep(y)) {
                        if (at < cap) { tt[at] = y; ss[at] = x; }
                        at++;
                    }
                } else if (keep(x) || (mm && keep(y))) {
                    if (in < (unsigned long long)cap_next) {
                        na[in] = x;
                        nb[in] = y | (mm ? (int32_t)0x80000000u : 0);
                    }
                    in++;
                }
            });
    }
}

// The traversal's seed in one launch (no host-to-device copies): the log
// zeroed with one root pair entering step 0, the frontier (0, root_b).
__global__ void traverse_seed(unsigned long long *log, int nlog, int32_t *fa, int32_t *fb, int32_t root_b) {
    for (int i = threadIdx.x; i < nlog; i += blockDim.x) log[i] = i == 2 ? 1ull : 0ull;
    if (threadIdx.x == 0) {
        fa[0] = 0;
        fb[0] = root_b;
    }
}

static Cells cells_of(const int32_t *children, const uint8_t *leaf, const double *ctr, const double *bmax,
                      const double *rmax) {
    return Cells{children, leaf, ctr, bmax, rmax};
}
static Cells source_cells(const Cells &A, const int32_t *children_b, const uint8_t *leaf_b, const double *ctr_b,
                          const double *bmax_b, const double *rmax_b) {
    return children_b ? Cells{children_b, leaf_b, ctr_b, bmax_b, rmax_b} : A;
}

extern "C" {

int fmm_traverse_step(const int32_t *fa, const int32_t *fb, int64_t nfront, int classify_self,
                      const int32_t *children,
                      const uint8_t *leaf, const double *ctr, const double *bmax, const double *rmax,
                      const int32_t *children_b, const uint8_t *leaf_b, const double *ctr_b, const double *bmax_b,
                      const double *rmax_b,
                      const int32_t *start, const int32_t *end, int32_t body_lo, int32_t body_hi,
                      int m2l_owner_only, int kind, double th2, int32_t *p2p_t, int32_t *p2p_s, int64_t cap_p2p,
                      int32_t *m2l_t,
                      int32_t *m2l_s, int64_t cap_m2l, int32_t *na, int32_t *nb, int64_t cap_next,
                      unsigned long long *dev_counts, void *stream) {
    if (nfront <= 0) return FMM_OK;
    const Cells A = cells_of(children, leaf, ctr, bmax, rmax);
    const Cells B = source_cells(A, children_b, leaf_b, ctr_b, bmax_b, rmax_b);
    traverse_step_kernel<<<grid_for(nfront, 256, 148 * 16), 256, 0, as_stream(stream)>>>(
        fa, fb, nfront, nullptr, nfront, classify_self, A, B, start, end, body_lo,
        body_hi, nullptr, m2l_owner_only, kind, th2, p2p_t, p2p_s, cap_p2p, m2l_t, m2l_s, cap_m2l,
        na, nb, cap_next, dev_counts, dev_counts + 1, dev_counts + 2); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_traverse_step");
    return FMM_OK;
}

int fmm_traverse(int32_t *front_a0, int32_t *front_b0, int32_t *front_a1, int32_t *front_b1, int64_t cap_front,
                 int nsteps, const int32_t *children, const uint8_t *leaf, const double *ctr,
                 const double *bmax, const double *rmax, const int32_t *children_b, const uint8_t *leaf_b,
                 const double *ctr_b, const double *bmax_b, const double *rmax_b, const int32_t *start, const int32_t *end,
                 int32_t body_lo, int32_t body_hi, const uint8_t *tmask, int m2l_owner_only, int kind, double th2,
                 int32_t *p2p_t, int32_t *p2p_s, int64_t cap_p2p, int32_t *m2l_t, int32_t *m2l_s, int64_t cap_m2l,
                 unsigned long long *dev_log, void *stream) {
    cudaStream_t st = as_stream(stream);
    const Cells A = cells_of(children, leaf, ctr, bmax, rmax);
    const Cells B = source_cells(A, children_b, leaf_b, ctr_b, bmax_b, rmax_b);
    // dev_log[0] = n_p2p, [1] = n_m2l, [2 + s] = frontier entering step s
    traverse_seed<<<1, 32, 0, st>>>(dev_log, nsteps + 3, front_a0, front_b0, 0); fmm::note_launch();
    const int grid = 148 * 8;
    for (int sidx = 0; sidx < nsteps; sidx++) {
        const bool even = (sidx & 1) == 0;
        traverse_step_kernel<<<grid, 256, 0, st>>>(
            even ? front_a0 : front_a1, even ? front_b0 : front_b1, 0, dev_log + 2 + sidx, cap_front, sidx == 0,
            A, B, start, end, body_lo, body_hi, tmask, m2l_owner_only, kind, th2, p2p_t,
            p2p_s, cap_p2p,
            m2l_t, m2l_s, cap_m2l, even ? front_a1 : front_a0, even ? front_b1 : front_b0, cap_front,
            dev_log, dev_log + 1, dev_log + 3 + sidx); fmm::note_launch();
    }
    FMM_CUDA_CHECK("fmm_traverse");
    return FMM_OK;
}

int fmm_treecode_traverse(int32_t *front_a0, int32_t *front_b0, int32_t *front_a1, int32_t *front_b1,
                          int64_t cap_front, int nsteps, int32_t ncells, const int32_t *children,
                          const uint8_t *leaf, const double *ctr, const double *bmax, const double *rmax,
                          const int32_t *children_b, const uint8_t *leaf_b, const double *ctr_b,
                          const double *bmax_b, const double *rmax_b,
                          const int32_t *start, const int32_t *end, int32_t body_lo, int32_t body_hi, int kind,
                          double th2, int32_t *m2p_t, int32_t *m2p_s, int64_t cap_m2p, int32_t *p2p_t,
                          int32_t *p2p_s, int64_t cap_p2p, unsigned long long *dev_log, void *ws,
                          size_t ws_bytes, void *stream) {
    cudaStream_t st = as_stream(stream);
    const Cells A = cells_of(children, leaf, ctr, bmax, rmax);
    const Cells B = source_cells(A, children_b, leaf_b, ctr_b, bmax_b, rmax_b);
    if (cap_front < ncells) {
        set_error("treecode frontier capacity %lld < ncells %d", (long long)cap_front, ncells);
        return FMM_ERR_INVALID;
    }
    Arena ar(ws, ws_bytes);
    uint8_t *flag = ar.take<uint8_t>((size_t)ncells);
    if (!flag) { set_error("workspace too small"); return FMM_ERR_INVALID; }
    // dev_log[0] = n_p2p, [1] = n_m2p, [2 + s] = frontier entering step s
    cudaMemsetAsync(dev_log, 0, sizeof(unsigned long long) * (nsteps + 3), st);
    treecode_seed_flags<<<grid_for(ncells, 256), 256, 0, st>>>(ncells, leaf, start, end, body_lo, body_hi, flag,
                                                                front_b0); fmm::note_launch();
    size_t need = 0;
    cub::CountingInputIterator<int32_t> it(0);
    cub::DeviceSelect::Flagged(nullptr, need, it, flag, front_a0, dev_log + 2, ncells, st);
    if (need > ar.left()) { set_error("select workspace"); return FMM_ERR_INVALID; }
    cub::DeviceSelect::Flagged(ar.rest(), need, it, flag, front_a0, dev_log + 2, ncells, st);
    const int grid = 148 * 8;
    for (int sidx = 0; sidx < nsteps; sidx++) {
        const bool even = (sidx & 1) == 0;
        treecode_step_kernel<<<grid, 256, 0, st>>>(
            even ? front_a0 : front_a1, even ? front_b0 : front_b1, dev_log + 2 + sidx, cap_front, A, B,
            kind, th2, m2p_t, m2p_s, cap_m2p, p2p_t, p2p_s, cap_p2p, even ? front_a1 : front_a0,
            even ? front_b1 : front_b0, cap_front, dev_log, dev_log + 1, dev_log + 3 + sidx); fmm::note_launch();
    }
    FMM_CUDA_CHECK("fmm_treecode_traverse");
    return FMM_OK;
}

int fmm_partition_owner(int32_t ncells, const int32_t *parent, const uint8_t *leaf, const int32_t *start,
                        const int32_t *end, int64_t grain, int32_t *owner, void *stream) {
    if (grain < 1) { set_error("task_grain must be >= 1, got %lld", (long long)grain); return FMM_ERR_INVALID; }
    partition_owner_kernel<<<grid_for(ncells, 256), 256, 0, as_stream(stream)>>>(ncells, parent, leaf, start, end,
                                                                                grain, owner); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_partition_owner");
    return FMM_OK;
}

static int traverse_mutual_impl(int32_t *front_a0, int32_t *front_b0, int32_t *front_a1, int32_t *front_b1,
                                int64_t cap_front, int nsteps, const int32_t *children, const uint8_t *leaf,
                                const double *ctr, const double *bmax, const double *rmax, const int32_t *owner,
                                const int32_t *start, const int32_t *end, int32_t body_lo, int32_t body_hi, int kind,
                                double th2, int32_t *p2p_t, int32_t *p2p_s, int64_t cap_p2p, int32_t *m2l_t,
                                int32_t *m2l_s, int64_t cap_m2l, unsigned long long *dev_log, int32_t *sp_a,
                                int32_t *sp_b, int64_t cap_sp, int32_t *sm_a, int32_t *sm_b, int64_t cap_sm,
                                unsigned long long *dev_sym, const char *who, void *stream) {
    cudaStream_t st = as_stream(stream);
    if (cap_front < 1) { set_error("frontier capacity must be >= 1"); return FMM_ERR_INVALID; }
    if ((sp_a || sm_a) && !dev_sym) { set_error("symmetric lists need their device counters"); return FMM_ERR_INVALID; }
    const Cells C = cells_of(children, leaf, ctr, bmax, rmax);
    // dev_log[0] = n_p2p, [1] = n_m2l, [2 + s] = frontier entering step s;
    // the seed is the unclassified mutual root pair (0, 0)
    traverse_seed<<<1, 32, 0, st>>>(dev_log, nsteps + 3, front_a0, front_b0, (int32_t)0x80000000u); fmm::note_launch();
    if (dev_sym) cudaMemsetAsync(dev_sym, 0, 2 * sizeof(unsigned long long), st);
    const int grid = 148 * 8;
    for (int sidx = 0; sidx < nsteps; sidx++) {
        const bool even = (sidx & 1) == 0;
        mutual_step_kernel<<<grid, 256, 0, st>>>(
            even ? front_a0 : front_a1, even ? front_b0 : front_b1, dev_log + 2 + sidx, cap_front, sidx == 0, C,
            owner, start,
            end, body_lo, body_hi, kind, th2, p2p_t, p2p_s, cap_p2p, m2l_t, m2l_s, cap_m2l,
            even ? front_a1 : front_a0, even ? front_b1 : front_b0, cap_front, dev_log, dev_log + 1,
            dev_log + 3 + sidx, sp_a, sp_b, cap_sp, sm_a, sm_b, cap_sm, dev_sym); fmm::note_launch();
    }
    FMM_CUDA_CHECK(who);
    return FMM_OK;
}

int fmm_traverse_mutual(int32_t *front_a0, int32_t *front_b0, int32_t *front_a1, int32_t *front_b1,
                        int64_t cap_front, int nsteps, const int32_t *children, const uint8_t *leaf,
                        const double *ctr, const double *bmax, const double *rmax, const int32_t *owner,
                        const int32_t *start, const int32_t *end, int32_t body_lo, int32_t body_hi, int kind,
                        double th2, int32_t *p2p_t, int32_t *p2p_s, int64_t cap_p2p, int32_t *m2l_t,
                        int32_t *m2l_s, int64_t cap_m2l, unsigned long long *dev_log, void *stream) {
    return traverse_mutual_impl(front_a0, front_b0, front_a1, front_b1, cap_front, nsteps, children, leaf, ctr, bmax,
                                rmax, owner, start, end, body_lo, body_hi, kind, th2, p2p_t, p2p_s, cap_p2p, m2l_t,
                                m2l_s, cap_m2l, dev_log, nullptr, nullptr, 0, nullptr, nullptr, 0, nullptr,
                                "fmm_traverse_mutual", stream);
}

int fmm_traverse_mutual_sym(int32_t *front_a0, int32_t *front_b0, int32_t *front_a1, int32_t *front_b1,
                            int64_t cap_front, int nsteps, const int32_t *children, const uint8_t *leaf,
                            const double *ctr, const double *bmax, const double *rmax, const int32_t *owner,
                            const int32_t *start, const int32_t *end, int32_t body_lo, int32_t body_hi, int kind,
                            double th2, int32_t *p2p_t, int32_t *p2p_s, int64_t cap_p2p, int32_t *m2l_t,
                            int32_t *m2l_s, int64_t cap_m2l, unsigned long long *dev_log, int32_t *sym_p2p_a,
                            int32_t *sym_p2p_b, int64_t cap_sym_p2p, int32_t *sym_m2l_a, int32_t *sym_m2l_b,
                            int64_t cap_sym_m2l, unsigned long long *dev_sym, void *stream) {
    return traverse_mutual_impl(front_a0, front_b0, front_a1, front_b1, cap_front, nsteps, children, leaf, ctr, bmax,
                                rmax, owner, start, end, body_lo, body_hi, kind, th2, p2p_t, p2p_s, cap_p2p, m2l_t,
                                m2l_s, cap_m2l, dev_log, sym_p2p_a, sym_p2p_b, cap_sym_p2p, sym_m2l_a, sym_m2l_b,
                                cap_sym_m2l, dev_sym, "fmm_traverse_mutual_sym", stream);
}

int fmm_listfmm_lists(int32_t ncells, int depth, const int64_t *level_off, const int8_t *level,
                      const uint64_t *key, const int32_t *parent, const int32_t *children, const uint8_t *leaf,
                      const int32_t *sub_end, const int32_t *start, const int32_t *end,
                      int32_t body_lo, int32_t body_hi, int32_t *m2l_t,
                      int32_t *m2l_s, int64_t cap_m2l, int32_t *p2p_t, int32_t *p2p_s, int64_t cap_p2p,
                      unsigned long long *dev_counts, void *ws, size_t ws_bytes, void *stream) {
    cudaStream_t st = as_stream(stream);
    if (depth < 0 || depth > MAX_LEVEL) { set_error("bad depth %d", depth); return FMM_ERR_INVALID; }
    Arena ar(ws, ws_bytes);
    uint64_t *skeys = ar.take<uint64_t>((size_t)ncells);
    int64_t *doff = ar.take<int64_t>((size_t)depth + 2);
    int32_t *iota = ar.take<int32_t>((size_t)ncells);
    int32_t *bylevel = ar.take<int32_t>((size_t)ncells);
    uint8_t *lv_sorted = ar.take<uint8_t>((size_t)ncells);
    if (!skeys || !doff || !iota || !bylevel || !lv_sorted) { set_error("workspace too small"); return FMM_ERR_INVALID; }
    cudaMemcpyAsync(doff, level_off, sizeof(int64_t) * ((size_t)depth + 2), cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(dev_counts, 0, 2 * sizeof(unsigned long long), st);
    // (level, key) table: a stable sort of the pre-order ids by level keeps
    // pre-order, i.e. key order, within each level
    fill_iota<<<grid_for(ncells, 256), 256, 0, st>>>(iota, ncells); fmm::note_launch();
    size_t need = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, (const uint8_t *)level, lv_sorted, iota, bylevel, ncells, 0, 8, st);
    if (need > ar.left()) { set_error("sort workspace"); return FMM_ERR_INVALID; }
    cub::DeviceRadixSort::SortPairs(ar.rest(), need, (const uint8_t *)level, lv_sorted, iota, bylevel, ncells, 0, 8,
                                    st);
    gather_keys<<<grid_for(ncells, 256), 256, 0, st>>>(ncells, bylevel, key, skeys); fmm::note_launch();
    LevelTable tab{bylevel, skeys, doff};
    listfmm_kernel<<<grid_for(ncells, 128, 148 * 16), 128, 0, st>>>(
        ncells, level, key, parent, children, leaf, sub_end, start, end, body_lo, body_hi, tab, m2l_t, m2l_s,
        cap_m2l, p2p_t, p2p_s, cap_p2p, dev_counts, dev_counts + 1); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_listfmm_lists");
    return FMM_OK;
}

int fmm_sort_rows(int32_t ncells, const int64_t *rows, const int32_t *in, int32_t *out, void *ws, size_t ws_bytes,
                  void *stream) {
    Arena ar(ws, ws_bytes);
    int32_t *wide_rows = ar.take<int32_t>((size_t)ncells + 1);
    unsigned long long *nwide = ar.take<unsigned long long>(1);
    if (!wide_rows || !nwide) { set_error("workspace too small"); return FMM_ERR_INVALID; }
    sort_rows_launch(ncells, rows, in, out, wide_rows, nwide, as_stream(stream));
    FMM_CUDA_CHECK("fmm_sort_rows");
    return FMM_OK;
}

int fmm_pairs_to_rows(const int32_t *t, const int32_t *s, const unsigned long long *dev_npairs, int64_t cap,
                      int32_t ncells, int32_t nsrc, int sort_rows, int32_t *src_sorted, int64_t *rows, void *ws,
                      size_t ws_bytes, void *stream) {
    cudaStream_t st = as_stream(stream);
    if (nsrc <= 0) nsrc = ncells;
    int nbits = 1;
    while ((1ll << nbits) < (int64_t)nsrc) nbits++;
    Arena ar(ws, ws_bytes);
    unsigned long long *cursor = ar.take<unsigned long long>((size_t)ncells + 1);
    int32_t *unsorted = ar.take<int32_t>((size_t)(cap > 0 ? cap : 1));
    int32_t *long_rows = ar.take<int32_t>((size_t)ncells);
    unsigned long long *nlong = ar.take<unsigned long long>(2);
    if (!cursor || !unsorted || !long_rows || !nlong) {
        set_error("workspace too small for %lld pairs", (long long)cap);
        return FMM_ERR_INVALID;
    }
    cudaMemsetAsync(cursor, 0, sizeof(unsigned long long) * ((size_t)ncells + 1), st);
    cudaMemsetAsync(nlong, 0, 2 * sizeof(unsigned long long), st);
    const int grid = 148 * 8;
    row_count_kernel<<<grid, 256, 0, st>>>(t, dev_npairs, cap, cursor); fmm::note_launch();
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, (const int64_t *)cursor, rows, ncells + 1, st);
    if (need > ar.left()) { set_error("scan workspace"); return FMM_ERR_INVALID; }
    cub::DeviceScan::ExclusiveSum(ar.rest(), need, (const int64_t *)cursor, rows, ncells + 1, st);
    cudaMemcpyAsync(cursor, rows, sizeof(int64_t) * ((size_t)ncells + 1), cudaMemcpyDeviceToDevice, st);
    if (!sort_rows) {  // grouped rows straight into the output
        row_scatter_kernel<<<grid, 256, 0, st>>>(t, s, dev_npairs, cap, cursor, src_sorted); fmm::note_launch();
        FMM_CUDA_CHECK("fmm_pairs_to_rows");
        return FMM_OK;
    }
    row_scatter_kernel<<<grid, 256, 0, st>>>(t, s, dev_npairs, cap, cursor, unsorted); fmm::note_launch();
    // the bitmap sort handles any id range (one 32768-id window per pass);
    // the block radix tiles remain as a cross-check (FMM_B200_ROWSORT_RADIX=1)
    if (!getenv("FMM_B200_ROWSORT_RADIX")) {
        sort_rows_launch(ncells, rows, unsorted, src_sorted, long_rows, nlong, st);
        FMM_CUDA_CHECK("fmm_pairs_to_rows");
        return FMM_OK;
    }
    int32_t *huge_rows = (int32_t *)cursor;
    row_sort_small_kernel<<<grid_for(ncells, 1, 148 * 16), kRowSmallThreads, 0, st>>>(
        ncells, rows, unsorted, src_sorted, nbits, long_rows, nlong); fmm::note_launch();
    row_sort_large_kernel<<<148, kRowLargeThreads, 0, st>>>(rows, unsorted, src_sorted, nbits, long_rows, nlong,
                                                            huge_rows, nlong + 1); fmm::note_launch();
    row_sort_huge_kernel<<<148, 1024, 0, st>>>(rows, unsorted, src_sorted, huge_rows, nlong + 1); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_pairs_to_rows");
    return FMM_OK;
}

int fmm_pairs_to_csr(const int32_t *t, const int32_t *s, int64_t npairs, int32_t ncells,
                     int32_t *src_sorted, int64_t *rows, void *ws, size_t ws_bytes, void *stream) {
    cudaStream_t st = as_stream(stream);
    if (npairs == 0) {
        fill_i64<<<grid_for(ncells + 1, 256), 256, 0, st>>>(rows, ncells + 1, 0); fmm::note_launch();
        FMM_CUDA_CHECK("fmm_pairs_to_csr");
        return FMM_OK;
    }
    int sbits = 1;
    while ((1ll << sbits) < (int64_t)ncells) sbits++;
    Arena ar(ws, ws_bytes);
    if (2 * sbits <= 32) {
        uint32_t *k0 = ar.take<uint32_t>(npairs);
        uint32_t *k1 = ar.take<uint32_t>(npairs);
        if (!k0 || !k1) { set_error("workspace too small for %lld pairs", (long long)npairs); return FMM_ERR_INVALID; }
        pack_pairs32<<<grid_for(npairs, 256), 256, 0, st>>>(t, s, npairs, sbits, k0); fmm::note_launch();
        size_t need = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, need, k0, k1, npairs, 0, 2 * sbits, st);
        if (need > ar.left()) { set_error("sort workspace"); return FMM_ERR_INVALID; }
        cub::DeviceRadixSort::SortKeys(ar.rest(), need, k0, k1, npairs, 0, 2 * sbits, st);
        unpack_rows32<<<grid_for(npairs, 256), 256, 0, st>>>(k1, npairs, sbits, ncells, src_sorted, rows); fmm::note_launch();
        FMM_CUDA_CHECK("fmm_pairs_to_csr");
        return FMM_OK;
    }
    uint64_t *k0 = ar.take<uint64_t>(npairs);
    uint64_t *k1 = ar.take<uint64_t>(npairs);
    if (!k0 || !k1) { set_error("workspace too small for %lld pairs", (long long)npairs); return FMM_ERR_INVALID; }
    pack_pairs<<<grid_for(npairs, 256), 256, 0, st>>>(t, s, npairs, sbits, k0); fmm::note_launch();
    size_t need = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, need, k0, k1, npairs, 0, 2 * sbits, st);
    if (need > ar.left()) { set_error("sort workspace"); return FMM_ERR_INVALID; }
    cub::DeviceRadixSort::SortKeys(ar.rest(), need, k0, k1, npairs, 0, 2 * sbits, st);
    unpack_rows<<<grid_for(npairs, 256), 256, 0, st>>>(k1, npairs, sbits, ncells, src_sorted, rows); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_pairs_to_csr");
    return FMM_OK;
}

}  // extern "C"
