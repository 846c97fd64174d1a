// partition.cu -- one rank's share of the tree for the Morton-partitioned
// multi-GPU evaluation (paper_1209_3516_b200/distributed.py, SURVEY.md
// §8(e); the reference's target ownership, src/traversal.py:19-26,
// :621-639), in four launches and one small device-to-host copy:
//
//  * cuts: body cut points on leaf boundaries -- cut r is the start of the
//    leaf holding body r n / world, made non-decreasing (a running max);
//  * chunks: the pre-order cells whose first body lies in each rank's range
//    (cell starts are non-decreasing in pre-order: a lower bound);
//  * the level-grouped lists of this rank's OWN cells (body range inside its
//    range) and of the SHARED cells (straddling an interior cut), in the
//    order of cells_by_level, with per-(group, level) counts.
#include <cub/cub.cuh>

#include "fmm_common.cuh"

namespace fmm {

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t *a, int64_t n, int64_t v) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// one warp: lane r the cut of rank boundary r (a warp max-scan makes them
// non-decreasing), then lane r the chunk bound of cut r (world <= 31 per
// pass; more ranks loop)
__global__ void plan_cuts(int32_t ncells, int64_t n, int world, const int32_t *__restrict__ start,
                          const int32_t *__restrict__ body_leaf, int64_t *cuts, int64_t *chunks) {
    const int lane = threadIdx.x & 31;
    int64_t carry = 0;
    for (int r0 = 0; r0 <= world; r0 += 32) {
        const int r = r0 + lane;
        int64_t c = 0;
        if (r >= 1 && r < world) c = start[body_leaf[(int64_t)r * n / world]];
        if (r == world) c = n;
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t v = __shfl_up_sync(0xffffffffu, c, o);
            if (lane >= o && v > c) c = v;
        }
        if (carry > c) c = carry;
        if (r <= world) cuts[r] = c;
        carry = __shfl_sync(0xffffffffu, c, 31);
    }
    __syncwarp();
    for (int r = lane; r <= world; r += 32) chunks[r] = lower_bound_i32(start, ncells, cuts[r]);
}

// per position of cells_by_level: own / shared flags and the per-(group,
// level) counts (block histogram, then one atomic per bin)
__global__ void plan_groups(int32_t ncells, int world, int rank, const int32_t *__restrict__ bfs,
                            const int32_t *__restrict__ start, const int32_t *__restrict__ end,
                            const int8_t *__restrict__ level, const int64_t *__restrict__ cuts, uint8_t *own,
                            uint8_t *shared, int64_t *counts) {
    __shared__ int hist[3 * 32];
    for (int k = threadIdx.x; k < 3 * 32; k += blockDim.x) hist[k] = 0;
    __syncthreads();
    const int64_t lo = cuts[rank], hi = cuts[rank + 1];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ncells; i += gridDim.x * blockDim.x) {
        const int c = bfs[i];
        const int64_t s = start[c], e = end[c];
        const bool o = s >= lo && e <= hi;
        // an interior cut strictly inside (s, e): the first cut above s
        int a = 1, b = world;  // search cuts[1 .. world-1]
        while (a < b) {
            const int m = (a + b) >> 1;
            if (cuts[m] <= s) a = m + 1;
            else b = m;
        }
        const bool sh = a < world && cuts[a] < e;
        own[i] = o;
        shared[i] = sh && !o;
        atomicAdd(&hist[(o ? 0 : (sh ? 1 : 2)) * 32 + level[c]], 1);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < 3 * 32; k += blockDim.x)
        if (hist[k]) atomicAdd((unsigned long long *)&counts[k], (unsigned long long)hist[k]);
}

}  // namespace fmm

using namespace fmm;

extern "C" int fmm_partition_plan(int32_t ncells, int64_t n, int world, int rank, const int32_t *start,
                                  const int32_t *end, const int32_t *body_leaf, const int32_t *cells_by_level,
                                  const int8_t *level, int32_t *own_cells, int32_t *shared_cells, int64_t *host_out,
                                  void *ws, size_t ws_bytes, void *stream) {
    if (world < 1 || rank < 0 || rank >= world) {
        set_error("bad rank %d of %d", rank, world);
        return FMM_ERR_INVALID;
    }
    cudaStream_t s = as_stream(stream);
    const int nout = 2 * (world + 1) + 3 * 32 + 2;
    Arena ar(ws, ws_bytes);
    int64_t *out = ar.take<int64_t>((size_t)nout);
    uint8_t *own = ar.take<uint8_t>((size_t)ncells);
    uint8_t *shared = ar.take<uint8_t>((size_t)ncells);
    int *nsel = ar.take<int>(2);
    if (!out || !own || !shared || !nsel) { set_error("workspace too small"); return FMM_ERR_INVALID; }
    int64_t *cuts = out, *chunks = out + world + 1, *counts = out + 2 * (world + 1);
    cudaMemsetAsync(out, 0, sizeof(int64_t) * nout, s);
    plan_cuts<<<1, 32, 0, s>>>(ncells, n, world, start, body_leaf, cuts, chunks);
    fmm::note_launch();
    plan_groups<<<grid_for(ncells, 256, 148 * 4), 256, 0, s>>>(ncells, world, rank, cells_by_level, start, end,
                                                               level, cuts, own, shared, counts);
    fmm::note_launch();
    size_t need = 0;
    cub::DeviceSelect::Flagged(nullptr, need, cells_by_level, own, own_cells, nsel, ncells, s);
    if (need > ar.left()) { set_error("select workspace"); return FMM_ERR_INVALID; }
    cub::DeviceSelect::Flagged(ar.rest(), need, cells_by_level, own, own_cells, nsel, ncells, s);
    cub::DeviceSelect::Flagged(ar.rest(), need, cells_by_level, shared, shared_cells, nsel + 1, ncells, s);
    // the selected counts ride along with the rest (they equal the count sums)
    static thread_local int64_t *pinned = nullptr;
    static thread_local int pinned_n = 0;
    if (pinned_n < nout) {
        if (pinned) cudaFreeHost(pinned);
        if (cudaMallocHost((void **)&pinned, sizeof(int64_t) * nout) != cudaSuccess) {
            pinned = nullptr;
            pinned_n = 0;
            return cuda_status("fmm_partition_plan pinned buffer");
        }
        pinned_n = nout;
    }
    cudaMemcpyAsync(pinned, out, sizeof(int64_t) * (nout - 2), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_status("fmm_partition_plan sync");
    for (int k = 0; k < nout - 2; k++) host_out[k] = pinned[k];
    FMM_CUDA_CHECK("fmm_partition_plan");
    return FMM_OK;
}
