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

__global__ void traverse_step_kernel(const int32_t *__restrict__ fa, const int32_t *__restrict__ fb,
                                     int64_t nfront, const int32_t *__restrict__ children,
                                     const uint8_t *__restrict__ leaf, const double *__restrict__ ctr,
                                     const double *__restrict__ bmax, const double *__restrict__ rmax,
                                     const int32_t *__restrict__ cstart, const int32_t *__restrict__ cend,
                                     int32_t blo, int32_t bhi, int kind_mac, double th2, int32_t *p2p_t,
                                     int32_t *p2p_s, int64_t cap_p2p,
                                     int32_t *m2l_t, int32_t *m2l_s, int64_t cap_m2l, int32_t *na,
                                     int32_t *nb, int64_t cap_next, unsigned long long *counts) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // iterate in warp-uniform trip counts so the shuffles see full warps
    const int64_t nround = (nfront + stride - 1) / stride;
    for (int64_t r = 0; r < nround; r++) {
        int64_t k = r * stride + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        bool valid = k < nfront;
        int32_t a = 0, b = 0;
        int kind = 0;  // 0 none, 1 p2p, 2 m2l, 3 expand
        int nkids = 0;
        int32_t kids[8];
        bool open_a = false;
        if (valid) {
            a = fa[k];
            b = fb[k];
            // multi-GPU: only targets whose body range meets [blo, bhi)
            if (cend[a] <= blo || cstart[a] >= bhi) valid = false;
        }
        if (valid) {
            bool la = leaf[a], lb = leaf[b];
            if (la && lb) {
                kind = 1;
            } else {
                double dx = ctr[a * 3] - ctr[b * 3];
                double dy = ctr[a * 3 + 1] - ctr[b * 3 + 1];
                double dz = ctr[a * 3 + 2] - ctr[b * 3 + 2];
                double r2 = dx * dx + dy * dy + dz * dz;
                bool ok = false;
                if (r2 != 0.0) {
                    // src/traversal.py:144-156: 0 = bh, 1 = bmax, 2 = fmm
                    double s = kind_mac == 2 ? bmax[a] + bmax[b] : (kind_mac == 1 ? bmax[b] : 2.0 * rmax[b]);
                    ok = s * s < th2 * r2;
                }
                if (ok) {
                    kind = 2;
                } else {
                    kind = 3;
                    open_a = la ? false : (lb ? true : (rmax[a] >= rmax[b]));
                    int32_t who = open_a ? a : b;
#pragma unroll
                    for (int o = 0; o < 8; o++) {
                        int32_t ch = children[who * 8 + o];
                        if (ch >= 0) kids[nkids++] = ch;
                    }
                }
            }
        }
        int off;
        unsigned long long base = warp_reserve(&counts[0], kind == 1 ? 1 : 0, lane, &off);
        if (kind == 1) {
            unsigned long long at = base + off;
            if (at < (unsigned long long)cap_p2p) { p2p_t[at] = a; p2p_s[at] = b; }
        }
        base = warp_reserve(&counts[1], kind == 2 ? 1 : 0, lane, &off);
        if (kind == 2) {
            unsigned long long at = base + off;
            if (at < (unsigned long long)cap_m2l) { m2l_t[at] = a; m2l_s[at] = b; }
        }
        base = warp_reserve(&counts[2], nkids, lane, &off);
        for (int q = 0; q < nkids; q++) {
            unsigned long long at = base + off + q;
            if (at < (unsigned long long)cap_next) {
                na[at] = open_a ? kids[q] : a;
                nb[at] = open_a ? b : kids[q];
            }
        }
    }
}

// ---- CSR ----------------------------------------------------------------
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

__global__ void fill_i64(int64_t *a, int64_t n, int64_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        a[i] = v;
}

}  // namespace fmm

using namespace fmm;

extern "C" {

int fmm_traverse_step(const int32_t *fa, const int32_t *fb, int64_t nfront, const int32_t *children,
                      const uint8_t *leaf, const double *ctr, const double *bmax, const double *rmax,
                      const int32_t *start, const int32_t *end, int32_t body_lo, int32_t body_hi,
                      int kind, double th2, int32_t *p2p_t, int32_t *p2p_s, int64_t cap_p2p, int32_t *m2l_t,
                      int32_t *m2l_s, int64_t cap_m2l, int32_t *na, int32_t *nb, int64_t cap_next,
                      unsigned long long *dev_counts, void *stream) {
    if (nfront <= 0) return FMM_OK;
    traverse_step_kernel<<<grid_for(nfront, 256, 148 * 16), 256, 0, as_stream(stream)>>>(
        fa, fb, nfront, children, leaf, ctr, bmax, rmax, start, end, body_lo, body_hi, kind, th2, p2p_t, p2p_s, cap_p2p, m2l_t, m2l_s, cap_m2l,
        na, nb, cap_next, dev_counts);
    FMM_CUDA_CHECK("fmm_traverse_step");
    return FMM_OK;
}

int fmm_pairs_to_csr(const int32_t *t, const int32_t *s, int64_t npairs, int32_t ncells,
                     int32_t *src_sorted, int64_t *rows, void *ws, size_t ws_bytes, void *stream) {
    cudaStream_t st = as_stream(stream);
    if (npairs == 0) {
        fill_i64<<<grid_for(ncells + 1, 256), 256, 0, st>>>(rows, ncells + 1, 0);
        FMM_CUDA_CHECK("fmm_pairs_to_csr");
        return FMM_OK;
    }
    int sbits = 1;
    while ((1ll << sbits) < (int64_t)ncells) sbits++;
    Arena ar(ws, ws_bytes);
    uint64_t *k0 = ar.take<uint64_t>(npairs);
    uint64_t *k1 = ar.take<uint64_t>(npairs);
    if (!k0 || !k1) { set_error("workspace too small for %lld pairs", (long long)npairs); return FMM_ERR_INVALID; }
    pack_pairs<<<grid_for(npairs, 256), 256, 0, st>>>(t, s, npairs, sbits, k0);
    size_t need = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, need, k0, k1, npairs, 0, 2 * sbits, st);
    if (need > ar.left()) { set_error("sort workspace"); return FMM_ERR_INVALID; }
    cub::DeviceRadixSort::SortKeys(ar.rest(), need, k0, k1, npairs, 0, 2 * sbits, st);
    unpack_rows<<<grid_for(npairs, 256), 256, 0, st>>>(k1, npairs, sbits, ncells, src_sorted, rows);
    FMM_CUDA_CHECK("fmm_pairs_to_csr");
    return FMM_OK;
}

}  // extern "C"
