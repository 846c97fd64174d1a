// rowsort.cuh -- warp-cooperative sort of one CSR row of DISTINCT ids.
//
// A row of an interaction list holds each source cell at most once, so the
// row is sorted by marking its ids in a warp-private shared-memory bitmap
// over the row's [min, max] window (kSortSegWords * 32 ids per pass) and
// compacting the set bits in order: no comparisons, no block barriers --
// one warp per row keeps many rows in flight, which is what bounds these
// latency-limited passes.
#pragma once

#include <cstdint>

namespace fmm {

#ifndef FMM_SORT_SHIFT
#define FMM_SORT_SHIFT 14
#endif
constexpr int kSortShift = FMM_SORT_SHIFT;              // log2(ids per bitmap pass)
constexpr int kSortSegWords = 1 << (kSortShift - 5);    // 512 words: 16384 ids per pass

// Sorts in[k0..k1) (distinct ids) into out[k0..k1).
__device__ __forceinline__ void warp_bitmap_sort(const int32_t *__restrict__ in, int32_t *out, int64_t k0, int64_t k1,
                                                 uint32_t *bm, int lane) {
    uint32_t lo = 0xffffffffu, hi = 0u;
    for (int64_t k = k0 + lane; k < k1; k += 32) {
        const uint32_t v = (uint32_t)in[k];
        lo = min(lo, v);
        hi = max(hi, v);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    int64_t pos = k0;
    for (uint32_t seg = lo >> 5; k1 > k0 && seg <= (hi >> 5); seg += kSortSegWords) {
        const uint32_t seg_end = min(seg + (uint32_t)kSortSegWords, (hi >> 5) + 1u), nw = seg_end - seg;
        for (uint32_t x = lane; x < nw; x += 32) bm[x] = 0u;
        __syncwarp();
        for (int64_t k = k0 + lane; k < k1; k += 32) {
            const uint32_t v = (uint32_t)in[k], word = v >> 5;
            if (word >= seg && word < seg_end) atomicOr(&bm[word - seg], 1u << (v & 31u));
        }
        __syncwarp();
        // every lane compacts a contiguous block of words, in order
        const uint32_t per = (nw + 31) / 32, w0 = min(lane * per, nw), w1 = min(w0 + per, nw);
        int cnt = 0;
        for (uint32_t x = w0; x < w1; x++) cnt += __popc(bm[x]);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        int64_t at = pos + incl - cnt;
        for (uint32_t x = w0; x < w1; x++) {
            for (uint32_t bits = bm[x]; bits; bits &= bits - 1u)
                out[at++] = (int32_t)(((seg + x) << 5) + (uint32_t)(__ffs(bits) - 1));
        }
        pos += __shfl_sync(0xffffffffu, incl, 31);
        __syncwarp();  // bm is rewritten by the next pass; out is read after return
    }
}

// ---- rows of <= kSparseMax ids spread over several windows -----------------
// The ids are staged once in the warp's shared slab `ent`; each pass marks
// one NON-EMPTY 32768-id window (the rows of an adaptive tree cluster into a
// few dense groups far apart) and compacts only the words between its
// smallest and largest id.  `bm` (kSortSegWords words) is zero on entry and
// on return.
constexpr int kSparseMax = 1024;

__device__ __forceinline__ void warp_bitmap_sort_sparse(const int32_t *__restrict__ in, int32_t *out, int64_t k0,
                                                        int64_t len, uint32_t *bm, uint32_t *ent, int lane) {
    constexpr uint32_t kNone = 0xffffffffu;
    const int n = (int)len;
    uint32_t seg = kNone;
    for (int e = lane; e < n; e += 32) {
        const uint32_t v = (uint32_t)in[k0 + e];
        ent[e] = v;
        seg = min(seg, v >> kSortShift);
    }
    seg = __reduce_min_sync(0xffffffffu, seg);
    __syncwarp();
    int64_t pos = k0;
    while (seg != kNone) {
        uint32_t wa = kNone, wb = 0u, nseg = kNone;
        for (int e = lane; e < n; e += 32) {
            const uint32_t v = ent[e], g = v >> kSortShift;
            if (g == seg) {
                const uint32_t wd = (v >> 5) & (kSortSegWords - 1);
                atomicOr(&bm[wd], 1u << (v & 31u));
                wa = min(wa, wd);
                wb = max(wb, wd);
            } else if (g > seg) {
                nseg = min(nseg, g);
            }
        }
        wa = __reduce_min_sync(0xffffffffu, wa);
        wb = __reduce_max_sync(0xffffffffu, wb);
        nseg = __reduce_min_sync(0xffffffffu, nseg);
        __syncwarp();
        const uint32_t nw = wb - wa + 1, per = (nw + 31) / 32;
        const uint32_t w0 = wa + min(lane * per, nw), w1 = wa + min(lane * per + per, nw);
        int cnt = 0;
        for (uint32_t x = w0; x < w1; x++) cnt += __popc(bm[x]);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        int64_t at = pos + incl - cnt;
        for (uint32_t x = w0; x < w1; x++) {
            for (uint32_t bits = bm[x]; bits; bits &= bits - 1u)
                out[at++] = (int32_t)((seg << kSortShift) + (x << 5) + (uint32_t)(__ffs(bits) - 1));
            bm[x] = 0u;
        }
        pos += __shfl_sync(0xffffffffu, incl, 31);
        __syncwarp();
        seg = nseg;
    }
    __syncwarp();  // ent is rewritten by the warp's next row
}

// True when the row's ids [lo, hi] need more than one bitmap pass.
__device__ __forceinline__ bool row_is_wide(const int32_t *__restrict__ in, int64_t k0, int64_t k1, int lane) {
    uint32_t lo = 0xffffffffu, hi = 0u;
    for (int64_t k = k0 + lane; k < k1; k += 32) {
        const uint32_t v = (uint32_t)in[k];
        lo = min(lo, v);
        hi = max(hi, v);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    return k1 > k0 && (hi >> 5) - (lo >> 5) >= (uint32_t)kSortSegWords;
}

}  // namespace fmm
