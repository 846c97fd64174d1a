// fmm_common.cuh -- shared definitions for the B200 FMM kernels.
//
// Cartesian Taylor multi-index tables (graded-lex order: ascending degree,
// within a degree descending mx then my; src/_taylor.py:1-45) are built at
// compile time so templated kernels resolve every index to an immediate.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fmm_b200.h"

namespace fmm {

constexpr int MAX_LEVEL = 21;
constexpr int TMAX = 12;                                     // src/_taylor.py:23
constexpr int NMI = (TMAX + 1) * (TMAX + 2) * (TMAX + 3) / 6;  // |m| <= TMAX

__host__ __device__ constexpr int ncoef(int p) { return p * (p + 1) * (p + 2) / 6; }

struct Tables {
    int mi[NMI][3];
    int deg[NMI];
    double mfact[NMI];
    double ifact[TMAX + 2];                 // 1/k!
    double rcp[TMAX + 2];                   // 1/k (rcp[0] unused)
    short idx3[TMAX + 2][TMAX + 2][TMAX + 2];
};

constexpr Tables make_tables() {
    Tables t{};
    for (int a = 0; a < TMAX + 2; a++)
        for (int b = 0; b < TMAX + 2; b++)
            for (int c = 0; c < TMAX + 2; c++) t.idx3[a][b][c] = -1;
    int n = 0;
    for (int d = 0; d <= TMAX; d++)
        for (int mx = d; mx >= 0; mx--)
            for (int my = d - mx; my >= 0; my--) {
                t.mi[n][0] = mx;
                t.mi[n][1] = my;
                t.mi[n][2] = d - mx - my;
                t.idx3[mx][my][d - mx - my] = (short)n;
                t.deg[n] = d;
                n++;
            }
    double fact[TMAX + 2] = {};
    fact[0] = 1.0;
    for (int d = 1; d < TMAX + 2; d++) fact[d] = fact[d - 1] * d;
    for (int d = 0; d < TMAX + 2; d++) t.ifact[d] = 1.0 / fact[d];
    t.rcp[0] = 0.0;
    for (int d = 1; d < TMAX + 2; d++) t.rcp[d] = 1.0 / d;
    for (int i = 0; i < n; i++) t.mfact[i] = fact[t.mi[i][0]] * fact[t.mi[i][1]] * fact[t.mi[i][2]];
    return t;
}

constexpr Tables kTab = make_tables();

// Runtime-indexed copy in global memory, one per translation unit (device
// symbols do not link across units without -rdc).
static __device__ Tables d_tab = kTab;

// Spread / compact the low 21 bits to every third bit (src/geometry.py:112-131).
__host__ __device__ inline uint64_t spread21(uint64_t v) {
    v &= 0x1FFFFFull;
    v = (v | v << 32) & 0x1F00000000FFFFull;
    v = (v | v << 16) & 0x1F0000FF0000FFull;
    v = (v | v << 8) & 0x100F00F00F00F00Full;
    v = (v | v << 4) & 0x10C30C30C30C30C3ull;
    v = (v | v << 2) & 0x1249249249249249ull;
    return v;
}

__host__ __device__ inline uint64_t compact21(uint64_t v) {
    v &= 0x1249249249249249ull;
    v = (v ^ (v >> 2)) & 0x10C30C30C30C30C3ull;
    v = (v ^ (v >> 4)) & 0x100F00F00F00F00Full;
    v = (v ^ (v >> 8)) & 0x1F0000FF0000FFull;
    v = (v ^ (v >> 16)) & 0x1F00000000FFFFull;
    v = (v ^ (v >> 32)) & 0x1FFFFFull;
    return v;
}

// Launch accounting: every kernel launch site of the library calls this
// (CUB's internal kernels are not counted); read by fmm_launch_count().
void note_launch();

// Error plumbing ----------------------------------------------------------
void set_error(const char *fmt, ...);
int cuda_status(const char *where);

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline int grid_for(int64_t n, int block, int64_t cap = 148 * 64) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

// Workspace carving: aligned bump allocator over a caller buffer.
struct Arena {
    char *base;
    size_t size, used;
    __host__ Arena(void *b, size_t s) : base((char *)b), size(s), used(0) {}
    template <class T>
    __host__ T *take(size_t count) {
        size_t off = (used + 255) & ~(size_t)255;
        size_t bytes = count * sizeof(T);
        if (off + bytes > size) return nullptr;
        used = off + bytes;
        return reinterpret_cast<T *>(base + off);
    }
    __host__ size_t left() const { return size > used ? size - ((used + 255) & ~(size_t)255) : 0; }
    __host__ void *rest() { size_t off = (used + 255) & ~(size_t)255; return base + off; }
};

}  // namespace fmm

#define FMM_CUDA_CHECK(where)                              \
    do {                                                   \
        int _st = fmm::cuda_status(where);                 \
        if (_st != FMM_OK) return _st;                     \
    } while (0)
