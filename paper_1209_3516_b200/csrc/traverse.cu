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

// Fate of a pair (src/traversal.py:185-211): 1 = P2P (both leaves, tested
// before the MAC), 2 = M2L (MAC accepted), 3 = split.
// _mac_ok (src/traversal.py:144-156) for target a, source b: 0 = bh,
// 1 = bmax, 2 = fmm; r2 == 0 rejects.
__device__ __forceinline__ bool mac_accept(int32_t a, int32_t b, const double *__restrict__ ctr,
                                           const double *__restrict__ bmax, const double *__restrict__ rmax,
                                           int kind_mac, double th2) {
    const double dx = ctr[a * 3] - ctr[b * 3];
    const double dy = ctr[a * 3 + 1] - ctr[b * 3 + 1];
    const double dz = ctr[a * 3 + 2] - ctr[b * 3 + 2];
    const double r2 = dx * dx + dy * dy + dz * dz;
    if (r2 == 0.0) return false;
    const double s = kind_mac == 2 ? bmax[a] + bmax[b] : (kind_mac == 1 ? bmax[b] : 2.0 * rmax[b]);
    return s * s < th2 * r2;
}

__device__ __forceinline__ int pair_fate(int32_t a, int32_t b, const uint8_t *__restrict__ leaf,
                                         const double *__restrict__ ctr, const double *__restrict__ bmax,
                                         const double *__restrict__ rmax, int kind_mac, double th2) {
    if (leaf[a] && leaf[b]) return 1;
    return mac_accept(a, b, ctr, bmax, rmax, kind_mac, th2) ? 2 : 3;
}

// One breadth-first step.  Every frontier pair is a pair already known to
// split; its children pairs are classified right here, so P2P and M2L
// pairs are emitted directly and only pairs that split again reach the
// next frontier (the root pair (0, 0) is classified by the first step,
// which the host launches with `classify_self = 1`).
__global__ void traverse_step_kernel(const int32_t *__restrict__ fa, const int32_t *__restrict__ fb,
                                     int64_t nfront_host, const unsigned long long *__restrict__ nfront_dev,
                                     int64_t cap_front, int classify_self, const int32_t *__restrict__ children,
                                     const uint8_t *__restrict__ leaf, const double *__restrict__ ctr,
                                     const double *__restrict__ bmax, const double *__restrict__ rmax,
                                     const int32_t *__restrict__ cstart, const int32_t *__restrict__ cend,
                                     int32_t blo, int32_t bhi, int m2l_owner, int kind_mac, double th2,
                                     int32_t *p2p_t,
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
    // iterate in warp-uniform trip counts so the shuffles see full warps
    const int64_t nround = (nfront + stride - 1) / stride;
    for (int64_t r = 0; r < nround; r++) {
        const int64_t k = r * stride + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        int32_t ca[8], cb[8];
        int fate[8];
        int n = 0;
        if (k < nfront) {
            const int32_t a = fa[k], b = fb[k];
            if (classify_self) {
                ca[0] = a;
                cb[0] = b;
                n = 1;
            } else {
                const bool la = leaf[a], lb = leaf[b];
                const bool open_a = la ? false : (lb ? true : (rmax[a] >= rmax[b]));
                const int32_t who = open_a ? a : b;
#pragma unroll
                for (int o = 0; o < 8; o++) {
                    const int32_t ch = children[who * 8 + o];
                    if (ch >= 0) {
                        ca[n] = open_a ? ch : a;
                        cb[n] = open_a ? b : ch;
                        n++;
                    }
                }
            }
        }
        int np = 0, nm = 0, nn = 0;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            fate[q] = 0;
            if (q < n) {
                // multi-GPU: only targets whose body range meets [blo, bhi)
                if (cend[ca[q]] <= blo || cstart[ca[q]] >= bhi) continue;
                fate[q] = pair_fate(ca[q], cb[q], leaf, ctr, bmax, rmax, kind_mac, th2);
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
                                     const unsigned long long *__restrict__ nfront_dev, int64_t cap_front,
                                     const int32_t *__restrict__ children, const uint8_t *__restrict__ leaf,
                                     const double *__restrict__ ctr, const double *__restrict__ bmax,
                                     const double *__restrict__ rmax, int kind_mac, double th2,
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
            if (mac_accept(t, c, ctr, bmax, rmax, kind_mac, th2)) fate = 2;
            else if (leaf[c]) fate = 1;
            else {
                fate = 3;
#pragma unroll
                for (int o = 0; o < 8; o++) nch += children[c * 8 + o] >= 0;
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
                const int32_t ch = children[c * 8 + o];
                if (ch >= 0) {
                    if (in < (unsigned long long)cap_next) { na[in] = t; nb[in] = ch; }
                    in++;
                }
            }
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

extern "C" {

int fmm_traverse_step(const int32_t *fa, const int32_t *fb, int64_t nfront, int classify_self,
                      const int32_t *children,
                      const uint8_t *leaf, const double *ctr, const double *bmax, const double *rmax,
                      const int32_t *start, const int32_t *end, int32_t body_lo, int32_t body_hi,
                      int m2l_owner_only, int kind, double th2, int32_t *p2p_t, int32_t *p2p_s, int64_t cap_p2p,
                      int32_t *m2l_t,
                      int32_t *m2l_s, int64_t cap_m2l, int32_t *na, int32_t *nb, int64_t cap_next,
                      unsigned long long *dev_counts, void *stream) {
    if (nfront <= 0) return FMM_OK;
    traverse_step_kernel<<<grid_for(nfront, 256, 148 * 16), 256, 0, as_stream(stream)>>>(
        fa, fb, nfront, nullptr, nfront, classify_self, children, leaf, ctr, bmax, rmax, start, end, body_lo,
        body_hi, m2l_owner_only, kind, th2, p2p_t, p2p_s, cap_p2p, m2l_t, m2l_s, cap_m2l,
        na, nb, cap_next, dev_counts, dev_counts + 1, dev_counts + 2); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_traverse_step");
    return FMM_OK;
}

int fmm_traverse(int32_t *front_a0, int32_t *front_b0, int32_t *front_a1, int32_t *front_b1, int64_t cap_front,
                 int nsteps, const int32_t *children, const uint8_t *leaf, const double *ctr,
                 const double *bmax, const double *rmax, const int32_t *start, const int32_t *end,
                 int32_t body_lo, int32_t body_hi, int m2l_owner_only, int kind, double th2, int32_t *p2p_t,
                 int32_t *p2p_s, int64_t cap_p2p, int32_t *m2l_t, int32_t *m2l_s, int64_t cap_m2l,
                 unsigned long long *dev_log, void *stream) {
    cudaStream_t st = as_stream(stream);
    // dev_log[0] = n_p2p, [1] = n_m2l, [2 + s] = frontier entering step s
    cudaMemsetAsync(dev_log, 0, sizeof(unsigned long long) * (nsteps + 3), st);
    const unsigned long long one = 1;
    cudaMemcpyAsync(dev_log + 2, &one, sizeof(one), cudaMemcpyHostToDevice, st);
    const int32_t zero = 0;
    cudaMemcpyAsync(front_a0, &zero, sizeof(zero), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(front_b0, &zero, sizeof(zero), cudaMemcpyHostToDevice, st);
    const int grid = 148 * 8;
    for (int sidx = 0; sidx < nsteps; sidx++) {
        const bool even = (sidx & 1) == 0;
        traverse_step_kernel<<<grid, 256, 0, st>>>(
            even ? front_a0 : front_a1, even ? front_b0 : front_b1, 0, dev_log + 2 + sidx, cap_front, sidx == 0,
            children, leaf, ctr, bmax, rmax, start, end, body_lo, body_hi, m2l_owner_only, kind, th2, p2p_t,
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
                          const int32_t *start, const int32_t *end, int32_t body_lo, int32_t body_hi, int kind,
                          double th2, int32_t *m2p_t, int32_t *m2p_s, int64_t cap_m2p, int32_t *p2p_t,
                          int32_t *p2p_s, int64_t cap_p2p, unsigned long long *dev_log, void *ws,
                          size_t ws_bytes, void *stream) {
    cudaStream_t st = as_stream(stream);
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
            even ? front_a0 : front_a1, even ? front_b0 : front_b1, dev_log + 2 + sidx, cap_front, children, leaf,
            ctr, bmax, rmax, kind, th2, m2p_t, m2p_s, cap_m2p, p2p_t, p2p_s, cap_p2p, even ? front_a1 : front_a0,
            even ? front_b1 : front_b0, cap_front, dev_log, dev_log + 1, dev_log + 3 + sidx); fmm::note_launch();
    }
    FMM_CUDA_CHECK("fmm_treecode_traverse");
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
