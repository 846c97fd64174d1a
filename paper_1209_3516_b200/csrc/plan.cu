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

// Source leaves of a target row merge into one body run when adjacent; in
// a one-tree evaluation the target's own leaf always stands alone (self).
// cross: sources belong to another tree (no self leaf).
__device__ inline bool run_start(const int32_t *src, int64_t k, int64_t k0, int32_t t,
                                 const int32_t *sstart, const int32_t *send, int cross) {
    if (k == k0) return true;
    int32_t s = src[k], sp = src[k - 1];
    return (!cross && (s == t || sp == t)) || sstart[s] != send[sp];
}

// Runs per row (nr) and the reference's pair counters in one pass over the
// row's sources: pairs = sum |t| |s| - self |t| - coincident, where the
// coincident ordered pairs (r2 == 0.0 in float64) can only occur inside the
// target leaf itself, and only between bodies with equal depth-21 keys --
// with the sorted keys given, leaves without two equal adjacent keys skip
// the O(|t|^2) scan.
__global__ void plan_count(const int32_t *__restrict__ nrows_dev, int32_t ncells, const int32_t *__restrict__ leaf_rows,
                           const int64_t *__restrict__ rows, const int32_t *__restrict__ src,
                           const int32_t *__restrict__ start, const int32_t *__restrict__ end,
                           const int32_t *__restrict__ sstart, const int32_t *__restrict__ send, int cross,
                           const double *__restrict__ xs, const double *__restrict__ ys,
                           const double *__restrict__ zs, const uint64_t *__restrict__ keys, int64_t *nr,
                           unsigned long long *stats) {
    const int lane = threadIdx.x & 31;
    const int32_t nrows = *nrows_dev;
    // rows past the device count get 0 so one scan over ncells + 1 works
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < ncells;
         r += (gridDim.x * blockDim.x) >> 5) {
        if (r >= nrows) {
            if (lane == 0) nr[r] = 0;
            continue;
        }
        const int32_t t = leaf_rows[r];
        const int64_t k0 = rows[t], k1 = rows[t + 1];
        const int32_t ts = start[t], te = end[t];
        const int64_t nt = te - ts;
        int64_t cnt = 0;
        unsigned long long blocks = 0, skipped = 0;
        bool self = false;
        for (int64_t kb = k0; kb < k1; kb += 32) {
            const int64_t k = kb + lane;
            const bool valid = k < k1;
            const bool f = valid && run_start(src, k, k0, t, sstart, send, cross);
            cnt += __popc(__ballot_sync(0xffffffffu, f));
            if (valid) {
                const int32_t s = src[k];
                blocks += (unsigned long long)(nt * (send[s] - sstart[s]));
                if (!cross && s == t) {
                    blocks -= (unsigned long long)nt;
                    self = true;
                }
            }
        }
        // coincident pairs inside the target leaf (only if the self pair is listed)
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
            nr[r] = cnt;
            if (stats) {
                atomicAdd(&stats[0], blocks - skipped);
                atomicAdd(&stats[1], skipped);
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) nr[ncells] = 0;
}

__global__ void plan_write(const int32_t *__restrict__ nrows_dev, const int32_t *__restrict__ leaf_rows,
                           const int64_t *__restrict__ rows, const int32_t *__restrict__ src,
                           const int32_t *__restrict__ sstart, const int32_t *__restrict__ send, int cross,
                           int32_t soff, const int64_t *__restrict__ run_off, int4 *runs) {
    const int lane = threadIdx.x & 31;
    const int32_t nrows = *nrows_dev;
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nrows;
         r += (gridDim.x * blockDim.x) >> 5) {
        const int32_t t = leaf_rows[r];
        const int64_t k0 = rows[t], k1 = rows[t + 1];
        int64_t base = run_off[r] - 1;  // index of the run holding the previous entry
        for (int64_t kb = k0; kb < k1; kb += 32) {
            int64_t k = kb + lane;
            bool valid = k < k1;
            bool f = valid && run_start(src, k, k0, t, sstart, send, cross);
            bool last = valid && (k + 1 == k1 || run_start(src, k + 1, k0, t, sstart, send, cross));
            unsigned m = __ballot_sync(0xffffffffu, f);
            int64_t idx = base + __popc(m & ((2u << lane) - 1u));
            if (f) {
                int32_t s = src[k];
                runs[idx].x = sstart[s] + soff;
                runs[idx].z = (!cross && s == t) ? 1 : 0;
                runs[idx].w = 0;
            }
            if (last) runs[idx].y = send[src[k]] + soff;
            base += __popc(m);
        }
    }
}

__global__ void leaf_in_range(int32_t ncells, const uint8_t *leaf, const int32_t *start, int32_t lo, int32_t hi,
                              uint8_t *flag) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncells; c += gridDim.x * blockDim.x)
        flag[c] = leaf[c] && start[c] >= lo && start[c] < hi;
}

}  // namespace fmm

using namespace fmm;


extern "C" int fmm_p2p_plan(int32_t ncells, const uint8_t *leaf, const int32_t *start, const int32_t *end,
                            int32_t body_lo, int32_t body_hi,
                            const int64_t *rows, const int32_t *src_sorted, const double *xs,
                            const double *ys, const double *zs, const uint64_t *keys, const int32_t *src_start,
                            const int32_t *src_end, int32_t src_offset, int32_t *leaf_rows, int64_t *run_off,
                            void *runs, int64_t cap_runs, int64_t *host_nruns, int32_t *host_nleaf_rows,
                            int32_t *dev_nrows, unsigned long long *dev_stats, void *ws, size_t ws_bytes,
                            void *stream) {
    cudaStream_t s = as_stream(stream);
    Arena ar(ws, ws_bytes);
    int32_t *nsel = ar.take<int32_t>(1);
    int64_t *nr = ar.take<int64_t>((size_t)ncells + 1);
    uint8_t *flag = ar.take<uint8_t>((size_t)ncells);
    if (!nsel || !nr || !flag) { set_error("workspace too small"); return FMM_ERR_INVALID; }
    leaf_in_range<<<grid_for(ncells, 256), 256, 0, s>>>(ncells, leaf, start, body_lo, body_hi, flag); fmm::note_launch();
    size_t need = 0;
    cub::CountingInputIterator<int32_t> it(0);
    cub::DeviceSelect::Flagged(nullptr, need, it, flag, leaf_rows, nsel, ncells, s);
    if (need > ar.left()) { set_error("select workspace"); return FMM_ERR_INVALID; }
    cub::DeviceSelect::Flagged(ar.rest(), need, it, flag, leaf_rows, nsel, ncells, s);
    // leaf_rows is sized ncells: the kernels read the row count on the device
    const int g = grid_for((int64_t)ncells * 32, 256, 148 * 16);
    if (dev_stats) cudaMemsetAsync(dev_stats, 0, 2 * sizeof(unsigned long long), s);
    const int cross = src_start != nullptr;
    const int32_t *ss = cross ? src_start : start, *se = cross ? src_end : end;
    plan_count<<<g, 256, 0, s>>>(nsel, ncells, leaf_rows, rows, src_sorted, start, end, ss, se, cross, xs, ys, zs,
                                 keys, nr, dev_stats); fmm::note_launch();
    need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, nr, run_off, ncells + 1, s);
    if (need > ar.left()) { set_error("scan workspace"); return FMM_ERR_INVALID; }
    cub::DeviceScan::ExclusiveSum(ar.rest(), need, nr, run_off, ncells + 1, s);
    if (host_nleaf_rows || host_nruns) {  // optional host view (synchronises)
        int32_t nrows = 0;
        int64_t total = 0;
        cudaMemcpyAsync(&nrows, nsel, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(&total, run_off + ncells, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_status("fmm_p2p_plan sync");
        if (host_nleaf_rows) *host_nleaf_rows = nrows;
        if (host_nruns) *host_nruns = total;
        if (total > cap_runs) { set_error("run capacity %lld < %lld", (long long)cap_runs, (long long)total); return FMM_ERR_CAPACITY; }
    }
    if (dev_nrows) cudaMemcpyAsync(dev_nrows, nsel, sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
    plan_write<<<g, 256, 0, s>>>(nsel, leaf_rows, rows, src_sorted, ss, se, cross, cross ? src_offset : 0, run_off,
                                 (int4 *)runs); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_p2p_plan");
    return FMM_OK;
}
