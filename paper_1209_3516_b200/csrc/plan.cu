// plan.cu -- P2P work decomposition and the reference's pair counters.
//
// The P2P list from the traversal (leaf pairs, src/traversal.py:185-195) is
// CSR over target leaves with ascending source-leaf ids.  Leaves in
// pre-order own consecutive body ranges, so Morton-adjacent source leaves
// of a row merge into one contiguous body run (664 source
// leaves per row collapse to ~28 runs of ~770 bodies at C2).  The target
// leaf's own bodies always form a separate "self" run, the only place the
// kernel needs the i != j / r2 > 0 guards.
//
// Counters follow src/_taylor.py:366-407: pairs = sum |t||s| - sum_self |t|
// - skipped, skipped = ordered i != j pairs of one leaf with r2 == 0.0 in
// float64 (coincident bodies always share a leaf: equal positions give
// equal depth-21 keys).  Compiled with --fmad=false so r2 matches.
#include <cub/cub.cuh>

#include "fmm_common.cuh"

namespace fmm {

// One warp per target row does the whole plan.  Source leaves are handled
// as leaf ORDINALS (rank among the source tree's leaves in pre-order):
// leaves in pre-order own consecutive body ranges, so two sources share a
// body run exactly when their ordinals are consecutive.  The warp marks the
// row's ordinals in a shared-memory bitmap (the row's sources are
// distinct) and reads the runs straight off the bitmap with word-level bit
// operations -- run starts are set bits whose predecessor bit is clear,
// run ends set bits whose successor is clear, the self leaf a run of its
// own -- each lane owning a contiguous block of words, so the sorted row is
// never materialised.  Runs are stored row-locally at the row's own CSR
// offset (runs <= pairs), in ascending source order.  The pair counters
// follow the reference: pairs = sum |t| |s| - self |t| - coincident, where
// the coincident ordered pairs (r2 == 0.0 in float64) can only occur inside
// the target leaf itself, and only between bodies with equal depth-21 keys
// -- with the sorted keys given, leaves without two equal adjacent keys
// skip the O(|t|^2) scan.
constexpr int kPlanWarps = 4;
#ifndef FMM_PLAN_SEG_SHIFT
#define FMM_PLAN_SEG_SHIFT 14
#endif
#ifndef FMM_PLAN_WIDE
#define FMM_PLAN_WIDE 512
#endif
#ifndef FMM_PLAN_MINB
#define FMM_PLAN_MINB 8
#endif
constexpr int kSegShift = FMM_PLAN_SEG_SHIFT;             // log2(ordinals per bitmap pass)
constexpr uint32_t kSegOrd = 1u << kSegShift;             // 16384 ordinals per bitmap pass
constexpr int kPlanSegWords = 1 << (kSegShift - 5);       // 512 words (2 KB per warp)
constexpr int kWideMax = FMM_PLAN_WIDE;  // longest row staged in shared memory (longer ones gather per pass)

// A row's coincident-pair scan, counters and run range (one warp).
__device__ __forceinline__ void plan_row_finish(int32_t r, int32_t t, int64_t k0, int64_t nrun, long long blocks,
                                                bool self, int32_t ts, int32_t te, const double *__restrict__ xs,
                                                const double *__restrict__ ys, const double *__restrict__ zs,
                                                const uint64_t *__restrict__ keys, int64_t *run_rng,
                                                unsigned long long *stats, unsigned long long *nruns_total, int lane) {
    // coincident pairs inside the target leaf (only if the self pair is listed)
    unsigned long long skipped = 0;
    self = __any_sync(0xffffffffu, self);
    bool dup = keys == nullptr;
    if (self && !dup)
        for (int32_t i = ts + lane; i + 1 < te && !dup; i += 32) dup = keys[i] == keys[i + 1];
    if (self && __any_sync(0xffffffffu, dup)) {
        for (int64_t i = ts + lane; i < te; i += 32) {
            for (int64_t j = ts; j < te; j++) {
                if (j == i) continue;
                const double dx = xs[i] - xs[j], dy = ys[i] - ys[j], dz = zs[i] - zs[j];
                const double r2 = dx * dx + dy * dy + dz * dz;
                if (r2 == 0.0) skipped++;
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        blocks += __shfl_xor_sync(0xffffffffu, blocks, o);
        skipped += __shfl_xor_sync(0xffffffffu, skipped, o);
    }
    if (lane == 0) {
        run_rng[2 * (int64_t)r] = k0;
        run_rng[2 * (int64_t)r + 1] = k0 + nrun;
        if (stats) {
            atomicAdd(&stats[0], (unsigned long long)blocks - skipped);
            atomicAdd(&stats[1], skipped);
            atomicAdd(nruns_total, (unsigned long long)nrun);
        }
    }
}

// Runs of one bitmap pass.  bm (the warp's window, bm[-1] and
// bm[kPlanSegWords] zero) holds the row's ordinals in [seg << kSegShift, (seg + 1)
// << 15); words [wa, wb] are the touched ones.  prev_top: is ordinal
// (seg << kSegShift) - 1 in the row; next_first: is (seg + 1) << 15.  Appends the
// pass's runs after the row's first nrun, updates the counters, clears the
// window and returns bit 31 of the pass's last word (the next pass's
// prev_top when that pass is seg + 1).
__device__ __forceinline__ uint32_t plan_pass(uint32_t *bm, uint32_t seg, uint32_t wa, uint32_t wb, uint32_t prev_top,
                                              bool next_first, int32_t ot, int64_t k0, int64_t nt, int64_t &nrun,
                                              long long &blocks, bool &self, const int32_t *__restrict__ s_bstart,
                                              const int32_t *__restrict__ s_bend, int32_t soff, int4 *runs, int lane) {
    const uint32_t sbase = seg << kSegShift;
    // the pass's word window, split into contiguous per-lane blocks
    const uint32_t nw = wb - wa + 1, per = (nw + 31) / 32;
    const uint32_t w0 = wa + min(lane * per, nw), w1 = wa + min(lane * per + per, nw);
    const int32_t self_word = (ot >= 0 && ((uint32_t)ot >> kSegShift) == seg) ? (int32_t)(((uint32_t)ot >> 5) & (kPlanSegWords - 1)) : -2;
    const int32_t prev_self = (ot >= 0 && (uint32_t)ot + 1u == sbase) ? 1 : 0;  // self just before this pass
    const int32_t next_self = (ot >= 0 && (uint32_t)ot == sbase + kSegOrd) ? 1 : 0;
    // masks of run starts / ends in word x
    auto masks = [&](uint32_t x, uint32_t &st, uint32_t &en) {
        const uint32_t W = bm[x];
        const uint32_t P = (x == 0) ? (prev_top << 31) : bm[x - 1];
        const uint32_t N = (x == kPlanSegWords - 1) ? (next_first ? 1u : 0u) : bm[x + 1];
        uint32_t Bs = 0u, Be = 0u;  // forced starts / ends around the self leaf
        if ((int32_t)x == self_word) {
            const uint32_t M = 1u << ((uint32_t)ot & 31u);
            Bs |= M | (M << 1);
            Be |= M | (M >> 1);
        }
        if ((int32_t)x - 1 == self_word && ((uint32_t)ot & 31u) == 31u) Bs |= 1u;
        if ((int32_t)x + 1 == self_word && ((uint32_t)ot & 31u) == 0u) Be |= 1u << 31;
        if (x == 0 && prev_self) Bs |= 1u;
        if (x == kPlanSegWords - 1 && next_self) Be |= 1u << 31;
        st = W & (~((W << 1) | (P >> 31)) | Bs);
        en = W & (~((W >> 1) | (N << 31)) | Be);
    };
    int cnt = 0;
    for (uint32_t x = w0; x < w1; x++) {
        uint32_t st, en;
        masks(x, st, en);
        cnt += __popc(st);
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    int64_t idx = k0 + nrun + (incl - cnt) - 1;  // run holding the entry before this lane's block
    for (uint32_t x = w0; x < w1; x++) {
        uint32_t st, en;
        masks(x, st, en);
        for (uint32_t m = st | en; m; m &= m - 1u) {
            const uint32_t bit = (uint32_t)__ffs(m) - 1u, b = 1u << bit;
            const uint32_t o = sbase + (x << 5) + bit;
            if (st & b) {
                ++idx;
                const int32_t b0 = s_bstart[o];
                // component stores: the run's end may be written by
                // another lane (a run crossing lane blocks)
                runs[idx].x = b0 + soff;
                runs[idx].z = (int32_t)o == ot ? 1 : 0;
                runs[idx].w = 0;
                blocks -= (long long)nt * b0;
            }
            if (en & b) {
                const int32_t b1 = s_bend[o];
                runs[idx].y = b1 + soff;
                blocks += (long long)nt * b1;
            }
        }
        if ((int32_t)x == self_word && (bm[x] >> ((uint32_t)ot & 31u) & 1u)) {
            blocks -= (long long)nt;
            self = true;
        }
    }
    nrun += __shfl_sync(0xffffffffu, incl, 31);
    __syncwarp();  // every lane read its neighbours' words
    const uint32_t top = bm[kPlanSegWords - 1] >> 31;
    __syncwarp();
    for (uint32_t x = w0; x < w1; x++) bm[x] = 0u;
    __syncwarp();
    return top;
}

// Rows of up to kWideMax sources: the ordinals were staged in the warp's
// shared slab `ent` while their range was found, and the passes visit only
// the bitmap windows that hold some -- a row of leaf neighbours in an
// adaptive tree clusters into a few dense groups of ordinals far apart --
// each pass scanning only the words between its smallest and largest
// ordinal, with no second gather of the row.
__device__ __forceinline__ void plan_row_staged(int32_t r, int32_t t, int64_t k0, int n, uint32_t seg, uint32_t *bm,
                                                const uint32_t *ent, const int32_t *__restrict__ start,
                                                const int32_t *__restrict__ end, const int32_t *__restrict__ t_ord,
                                                const int32_t *__restrict__ s_bstart,
                                                const int32_t *__restrict__ s_bend, int cross, int32_t soff,
                                                const double *__restrict__ xs, const double *__restrict__ ys,
                                                const double *__restrict__ zs, const uint64_t *__restrict__ keys,
                                                int64_t *run_rng, int4 *runs, unsigned long long *stats,
                                                unsigned long long *nruns_total, int lane) {
    constexpr uint32_t kNone = 0xffffffffu;
    const int32_t ts = start[t], te = end[t];
    const int64_t nt = te - ts;
    const int32_t ot = cross ? -1 : t_ord[t];
    long long blocks = 0;
    bool self = false;
    int64_t nrun = 0;
    uint32_t prev_seg = kNone, prev_top = 0u;
    while (n > 0 && seg != kNone) {
        const uint32_t sbase = seg << kSegShift;
        uint32_t wa = kNone, wb = 0u, nseg = kNone;
        bool next_first = false;
        for (int e = lane; e < n; e += 32) {
            const uint32_t v = ent[e], g = v >> kSegShift;
            if (g == seg) {
                const uint32_t wd = (v >> 5) & (kPlanSegWords - 1);
                atomicOr(&bm[wd], 1u << (v & 31u));
                wa = min(wa, wd);
                wb = max(wb, wd);
            } else if (g > seg) {
                nseg = min(nseg, g);
            }
            next_first |= v == sbase + kSegOrd;
        }
        wa = __reduce_min_sync(0xffffffffu, wa);
        wb = __reduce_max_sync(0xffffffffu, wb);
        nseg = __reduce_min_sync(0xffffffffu, nseg);
        next_first = __any_sync(0xffffffffu, next_first);
        __syncwarp();
        const uint32_t top = plan_pass(bm, seg, wa, wb, prev_seg + 1u == seg ? prev_top : 0u, next_first, ot, k0, nt,
                                       nrun, blocks, self, s_bstart, s_bend, soff, runs, lane);
        prev_seg = seg;
        prev_top = top;
        seg = nseg;
    }
    plan_row_finish(r, t, k0, nrun, blocks, self, ts, te, xs, ys, zs, keys, run_rng, stats, nruns_total, lane);
    __syncwarp();  // ent is rewritten by the warp's next row
}

__global__ void __launch_bounds__(kPlanWarps * 32, FMM_PLAN_MINB) plan_rows_kernel(
    const int32_t *__restrict__ nrows_dev, const int32_t *__restrict__ leaf_rows, const int64_t *__restrict__ rows,
    const int32_t *__restrict__ src, const int32_t *__restrict__ start, const int32_t *__restrict__ end,
    const int32_t *__restrict__ t_ord, const int32_t *__restrict__ s_ord, const int32_t *__restrict__ s_bstart,
    const int32_t *__restrict__ s_bend, int cross, int32_t soff, const double *__restrict__ xs,
    const double *__restrict__ ys, const double *__restrict__ zs, const uint64_t *__restrict__ keys,
    int64_t *run_rng, int4 *runs, int64_t cap_runs, unsigned long long *stats, unsigned long long *nruns_total,
    unsigned long long *runs_needed) {
    __shared__ uint32_t bm_all[kPlanWarps][kPlanSegWords + 2];
    __shared__ uint32_t ent_all[kPlanWarps][kWideMax];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *ent = ent_all[wid];
    uint32_t *bm = bm_all[wid] + 1;  // bm[-1] and bm[kPlanSegWords] stay 0: neighbour words of the edges
    for (int x = lane; x < kPlanSegWords + 2; x += 32) bm_all[wid][x] = 0u;
    __syncwarp();
    const int32_t nrows = *nrows_dev;
    for (int32_t r = blockIdx.x * kPlanWarps + wid; r < nrows; r += gridDim.x * kPlanWarps) {
        const int32_t t = leaf_rows[r];
        const int64_t k0 = rows[t], k1 = rows[t + 1];
        const int32_t ts = start[t], te = end[t];
        const int64_t nt = te - ts;
        const int32_t ot = cross ? -1 : t_ord[t];  // the self leaf's ordinal
        if (k1 > cap_runs) {  // runs are row-local (k0 + run < k1): the buffer is short
            if (lane == 0) {
                run_rng[2 * (int64_t)r] = run_rng[2 * (int64_t)r + 1] = k0;
                atomicMax(runs_needed, (unsigned long long)k1);
            }
            continue;
        }
        const bool staged = k1 - k0 <= kWideMax;
        uint32_t lo = 0xffffffffu, hi = 0u;
        for (int64_t k = k0 + lane; k < k1; k += 32) {
            const uint32_t v = (uint32_t)s_ord[src[k]];
            if (staged) ent[k - k0] = v;
            lo = min(lo, v);
            hi = max(hi, v);
        }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        if (staged) {  // one gather of the row, non-empty windows only
            __syncwarp();
            plan_row_staged(r, t, k0, (int)(k1 - k0), lo >> kSegShift, bm, ent, start, end, t_ord, s_bstart, s_bend, cross,
                            soff, xs, ys, zs, keys, run_rng, runs, stats, nruns_total, lane);
            continue;
        }
        long long blocks = 0;
        bool self = false;
        int64_t nrun = 0;        // runs so far in this row (warp-uniform)
        uint32_t prev_top = 0u;  // bit 31 of the word before the current pass
        for (uint32_t seg = lo >> kSegShift; k1 > k0 && seg <= (hi >> kSegShift); seg++) {
            const uint32_t sbase = seg << kSegShift;
            bool next_first = false;  // is ordinal sbase + 32768 (next pass) set?
            for (int64_t k = k0 + lane; k < k1; k += 32) {
                const uint32_t v = (uint32_t)s_ord[src[k]];
                if ((v >> kSegShift) == seg) atomicOr(&bm[(v >> 5) & (kPlanSegWords - 1)], 1u << (v & 31u));
                next_first |= v == sbase + kSegOrd;
            }
            next_first = __any_sync(0xffffffffu, next_first);
            __syncwarp();
            const uint32_t wa = (seg == (lo >> kSegShift)) ? ((lo >> 5) & (kPlanSegWords - 1)) : 0u;
            const uint32_t wb = (seg == (hi >> kSegShift)) ? ((hi >> 5) & (kPlanSegWords - 1)) : kPlanSegWords - 1;
            prev_top = plan_pass(bm, seg, wa, wb, prev_top, next_first, ot, k0, nt, nrun, blocks, self, s_bstart,
                                 s_bend, soff, runs, lane);
        }
        plan_row_finish(r, t, k0, nrun, blocks, self, ts, te, xs, ys, zs, keys, run_rng, stats, nruns_total, lane);
    }
}

// Leaf ordinals: ord[c] = number of leaves before c in pre-order (an
// exclusive scan of the leaf flags), cell[ord[c]] = c for leaves.
__global__ void leaf_cells_kernel(int32_t ncells, const uint8_t *__restrict__ leaf, const int32_t *__restrict__ ord,
                                  const int32_t *__restrict__ start, const int32_t *__restrict__ end,
                                  int32_t *bstart, int32_t *bend) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncells; c += gridDim.x * blockDim.x)
        if (leaf[c]) {
            bstart[ord[c]] = start[c];
            bend[ord[c]] = end[c];
        }
}

struct LeafFlag {
    __host__ __device__ __forceinline__ int32_t operator()(uint8_t v) const { return v ? 1 : 0; }
};

static int leaf_ordinals(int32_t ncells, const uint8_t *leaf, const int32_t *start, const int32_t *end,
                         int32_t *ord, int32_t *bstart, int32_t *bend, Arena &ar, cudaStream_t s) {
    cub::TransformInputIterator<int32_t, LeafFlag, const uint8_t *> flags(leaf, LeafFlag());
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, flags, ord, ncells, s);
    if (need > ar.left()) { set_error("scan workspace"); return FMM_ERR_INVALID; }
    cub::DeviceScan::ExclusiveSum(ar.rest(), need, flags, ord, ncells, s);
    leaf_cells_kernel<<<grid_for(ncells, 256), 256, 0, s>>>(ncells, leaf, ord, start, end, bstart, bend); fmm::note_launch();
    return FMM_OK;
}

__global__ void leaf_in_range(int32_t ncells, const uint8_t *leaf, const int32_t *start, int32_t lo, int32_t hi,
                              const uint8_t *tmask, uint8_t *flag) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncells; c += gridDim.x * blockDim.x)
        flag[c] = leaf[c] && start[c] >= lo && start[c] < hi && (!tmask || tmask[c]);
}

}  // namespace fmm

using namespace fmm;


extern "C" int fmm_p2p_plan(int32_t ncells, const uint8_t *leaf, const int32_t *start, const int32_t *end,
                            int32_t body_lo, int32_t body_hi, const uint8_t *tmask, const int64_t *rows,
                            const int32_t *src,
                            const double *xs, const double *ys, const double *zs,
                            const uint64_t *keys, const uint8_t *src_leaf, int32_t src_ncells,
                            const int32_t *src_start, const int32_t *src_end, int32_t src_offset, int32_t *leaf_rows,
                            int64_t *run_rng, void *runs, int64_t cap_runs, int64_t *host_nruns,
                            int32_t *host_nleaf_rows, int32_t *dev_nrows, unsigned long long *dev_stats, void *ws,
                            size_t ws_bytes, void *stream) {
    cudaStream_t s = as_stream(stream);
    const int cross = src_start != nullptr;
    if (cross && (!src_end || !src_leaf || src_ncells <= 0)) {
        set_error("cross-tree plan needs the source tree's leaf flags, starts, ends and cell count");
        return FMM_ERR_INVALID;
    }
    Arena ar(ws, ws_bytes);
    int32_t *nsel_ws = ar.take<int32_t>(1);
    unsigned long long *st3 = ar.take<unsigned long long>(4);  // {pairs, skipped, runs, -}
    uint8_t *flag = ar.take<uint8_t>((size_t)ncells);
    int32_t *t_ord = ar.take<int32_t>((size_t)ncells);
    int32_t *t_bs = ar.take<int32_t>((size_t)ncells);
    int32_t *t_be = ar.take<int32_t>((size_t)ncells);
    int32_t *s_ord = cross ? ar.take<int32_t>((size_t)src_ncells) : t_ord;
    int32_t *s_bs = cross ? ar.take<int32_t>((size_t)src_ncells) : t_bs;
    int32_t *s_be = cross ? ar.take<int32_t>((size_t)src_ncells) : t_be;
    if (!nsel_ws || !st3 || !flag || !t_ord || !t_bs || !t_be || !s_ord || !s_bs || !s_be) {
        set_error("workspace too small");
        return FMM_ERR_INVALID;
    }
    int rc = leaf_ordinals(ncells, leaf, start, end, t_ord, t_bs, t_be, ar, s);
    if (rc == FMM_OK && cross) rc = leaf_ordinals(src_ncells, src_leaf, src_start, src_end, s_ord, s_bs, s_be, ar, s);
    if (rc != FMM_OK) return rc;
    // the row count and the counters go straight to the caller's buffers
    int32_t *nsel = dev_nrows ? dev_nrows : nsel_ws;
    unsigned long long *stats = dev_stats ? dev_stats : st3;
    unsigned long long *runs_need = dev_stats ? dev_stats + 2 : st3 + 3;  // 0, or the runs capacity required
    leaf_in_range<<<grid_for(ncells, 256), 256, 0, s>>>(ncells, leaf, start, body_lo, body_hi, tmask, flag); fmm::note_launch();
    size_t need = 0;
    cub::CountingInputIterator<int32_t> it(0);
    cub::DeviceSelect::Flagged(nullptr, need, it, flag, leaf_rows, nsel, ncells, s);
    if (need > ar.left()) { set_error("select workspace"); return FMM_ERR_INVALID; }
    cub::DeviceSelect::Flagged(ar.rest(), need, it, flag, leaf_rows, nsel, ncells, s);
    cudaMemsetAsync(st3, 0, 4 * sizeof(unsigned long long), s);
    if (dev_stats) cudaMemsetAsync(dev_stats, 0, 3 * sizeof(unsigned long long), s);
    // leaf_rows is sized ncells: the kernel reads the row count on the device
    plan_rows_kernel<<<grid_for(ncells, kPlanWarps, 148 * 8), kPlanWarps * 32, 0, s>>>(
        nsel, leaf_rows, rows, src, start, end, t_ord, s_ord, s_bs, s_be, cross, cross ? src_offset : 0, xs, ys, zs,
        keys, run_rng, (int4 *)runs, cap_runs, stats, st3 + 2, runs_need); fmm::note_launch();
    if (host_nleaf_rows || host_nruns) {  // optional host view (synchronises)
        int32_t nrows = 0;
        unsigned long long total = 0, needed = 0;
        cudaMemcpyAsync(&nrows, nsel, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(&total, st3 + 2, sizeof(total), cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(&needed, runs_need, sizeof(needed), cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_status("fmm_p2p_plan sync");
        if (host_nleaf_rows) *host_nleaf_rows = nrows;
        if (needed) {  // grow-and-retry: the exact capacity comes back in *host_nruns
            if (host_nruns) *host_nruns = (int64_t)needed;
            set_error("P2P runs buffer too small: %lld entries needed, cap_runs %lld", (long long)needed,
                      (long long)cap_runs);
            return FMM_ERR_CAPACITY;
        }
        if (host_nruns) *host_nruns = (int64_t)total;
    }
    FMM_CUDA_CHECK("fmm_p2p_plan");
    return FMM_OK;
}
