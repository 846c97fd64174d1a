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

constexpr int kSortSegWords = 1024;  // 32768 ids per pass

struct IdentityIds {
    __device__ __forceinline__ uint32_t operator()(int32_t v) const { return (uint32_t)v; }
};

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

// ---- rows spread over several bitmap passes: sort in registers -----------
// Bitonic network over N = 32 * ITEMS keys held lane-major (lane l owns
// elements [l * ITEMS, (l + 1) * ITEMS)); pads are 0xffffffff.  Its cost
// does not depend on the id window, which is what makes it the choice when
// a row's ids spread over several 32768-id bitmap passes.
template <int ITEMS>
__device__ __forceinline__ void warp_bitonic_sort(uint32_t (&v)[ITEMS], int lane) {
    constexpr int N = 32 * ITEMS;
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= ITEMS) {  // partner in lane ^ (j / ITEMS), same slot
                const int lm = j / ITEMS;
                const bool lower = (lane & lm) == 0;
#pragma unroll
                for (int i = 0; i < ITEMS; i++) {
                    const bool asc = ((lane * ITEMS + i) & k) == 0;
                    const uint32_t o = __shfl_xor_sync(0xffffffffu, v[i], lm);
                    v[i] = (lower == asc) ? min(v[i], o) : max(v[i], o);
                }
            } else {  // partner in this lane's registers
#pragma unroll
                for (int i = 0; i < ITEMS; i++) {
                    if ((i & j) == 0) {
                        const bool asc = ((lane * ITEMS + i) & k) == 0;
                        const uint32_t a = v[i], b = v[i | j];
                        v[i] = asc ? min(a, b) : max(a, b);
                        v[i | j] = asc ? max(a, b) : min(a, b);
                    }
                }
            }
        }
    }
}

// Load row [k0, k1) (len <= 32 * ITEMS) lane-major through `map`, sort.
template <int ITEMS, class Map>
__device__ __forceinline__ void warp_bitonic_load_sort(const int32_t *__restrict__ in, int64_t k0, int64_t len,
                                                       uint32_t (&v)[ITEMS], int lane, Map map) {
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        const int64_t e = (int64_t)lane * ITEMS + i;
        v[i] = e < len ? map(in[k0 + e]) : 0xffffffffu;
    }
    warp_bitonic_sort<ITEMS>(v, lane);
}

template <int ITEMS>
__device__ __forceinline__ void warp_bitonic_row(const int32_t *__restrict__ in, int32_t *out, int64_t k0, int64_t len,
                                                 int lane) {
    uint32_t v[ITEMS];
    warp_bitonic_load_sort<ITEMS>(in, k0, len, v, lane, IdentityIds());
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        const int64_t e = (int64_t)lane * ITEMS + i;
        if (e < len) out[k0 + e] = (int32_t)v[i];
    }
}

// Row [k0, k1) of up to 1024 ids, in registers, dispatched on its length.
__device__ __forceinline__ void warp_bitonic_any(const int32_t *__restrict__ in, int32_t *out, int64_t k0, int64_t len,
                                                 int lane) {
    if (len <= 128) warp_bitonic_row<4>(in, out, k0, len, lane);
    else if (len <= 256) warp_bitonic_row<8>(in, out, k0, len, lane);
    else if (len <= 512) warp_bitonic_row<16>(in, out, k0, len, lane);
    else warp_bitonic_row<32>(in, out, k0, len, lane);
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
