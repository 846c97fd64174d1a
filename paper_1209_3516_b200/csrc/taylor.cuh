// taylor.cuh -- compile-time Cartesian Taylor machinery shared by the
// M2L and M2P kernels: D_k = d^k (1/|r|) by the reference's degree-by-degree
// recurrence (src/_taylor.py:57-95) with every multi-index resolved at
// compile time, so D stays in registers.
#pragma once

#include <type_traits>
#include <utility>

#include "fmm_common.cuh"

namespace fmm {

// static_for hands each iteration its index as a type, so every table
// lookup below is a constant expression and D / M / L stay in registers.
template <int B, class F, int... I>
__device__ __forceinline__ void static_for_seq(F &&f, std::integer_sequence<int, I...>) {
    (f(std::integral_constant<int, B + I>{}), ...);  // a fold: no recursion depth limit
}

template <int B, int E, class F>
__device__ __forceinline__ void static_for(F &&f) {
    if constexpr (B < E) static_for_seq<B>(f, std::make_integer_sequence<int, E - B>{});
}

#define IX(a, b, c) (std::integral_constant<int, kTab.idx3[a][b][c]>::value)

template <int P, typename T = double>
__device__ __forceinline__ void d_tensors_reg(T rx, T ry, T rz, T (&D)[ncoef(P)]) {
    const T r2 = rx * rx + ry * ry + rz * rz;
    T inv_r2;
    if constexpr (std::is_same_v<T, float>) {  // float32 terms: MUFU.RSQ (~2^-22.9) in place of IEEE div + sqrt
        float d0;
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(d0) : "f"(r2));
        D[0] = d0;
        inv_r2 = d0 * d0;
    } else {
        inv_r2 = T(1) / r2;
        D[0] = sqrt(inv_r2);
    }
    static_for<1, ncoef(P)>([&](auto I) {
        constexpr int idx = decltype(I)::value;
        constexpr int kx = kTab.mi[idx][0], ky = kTab.mi[idx][1], kz = kTab.mi[idx][2];
        T acc = T(0);
        if constexpr (kx > 0) {
            acc -= T(2.0 * kx - 1.0) * rx * D[IX(kx - 1, ky, kz)];
            if constexpr (kx > 1) acc -= T((kx - 1.0) * (kx - 1.0)) * D[IX(kx - 2, ky, kz)];
            if constexpr (ky > 0) {
                acc -= T(2.0 * ky) * ry * D[IX(kx, ky - 1, kz)];
                if constexpr (ky > 1) acc -= T(ky * (ky - 1.0)) * D[IX(kx, ky - 2, kz)];
            }
            if constexpr (kz > 0) {
                acc -= T(2.0 * kz) * rz * D[IX(kx, ky, kz - 1)];
                if constexpr (kz > 1) acc -= T(kz * (kz - 1.0)) * D[IX(kx, ky, kz - 2)];
            }
        } else if constexpr (ky > 0) {
            acc -= T(2.0 * ky - 1.0) * ry * D[IX(kx, ky - 1, kz)];
            if constexpr (ky > 1) acc -= T((ky - 1.0) * (ky - 1.0)) * D[IX(kx, ky - 2, kz)];
            if constexpr (kz > 0) {
                acc -= T(2.0 * kz) * rz * D[IX(kx, ky, kz - 1)];
                if constexpr (kz > 1) acc -= T(kz * (kz - 1.0)) * D[IX(kx, ky, kz - 2)];
            }
        } else {
            acc -= T(2.0 * kz - 1.0) * rz * D[IX(kx, ky, kz - 1)];
            if constexpr (kz > 1) acc -= T((kz - 1.0) * (kz - 1.0)) * D[IX(kx, ky, kz - 2)];
        }
        D[idx] = acc * inv_r2;
    });
}

// The same recurrence into a thread-private array in shared memory (orders
// whose D does not fit the register file).
template <int P>
__device__ __forceinline__ void d_tensors_ptr(double rx, double ry, double rz, double *D) {
    const double r2 = rx * rx + ry * ry + rz * rz;
    const double inv_r2 = 1.0 / r2;
    D[0] = sqrt(inv_r2);
    static_for<1, ncoef(P)>([&](auto I) {
        constexpr int idx = decltype(I)::value;
        constexpr int kx = kTab.mi[idx][0], ky = kTab.mi[idx][1], kz = kTab.mi[idx][2];
        double acc = 0.0;
        if constexpr (kx > 0) {
            acc -= (2.0 * kx - 1.0) * rx * D[IX(kx - 1, ky, kz)];
            if constexpr (kx > 1) acc -= ((kx - 1.0) * (kx - 1.0)) * D[IX(kx - 2, ky, kz)];
            if constexpr (ky > 0) {
                acc -= (2.0 * ky) * ry * D[IX(kx, ky - 1, kz)];
                if constexpr (ky > 1) acc -= (ky * (ky - 1.0)) * D[IX(kx, ky - 2, kz)];
            }
            if constexpr (kz > 0) {
                acc -= (2.0 * kz) * rz * D[IX(kx, ky, kz - 1)];
                if constexpr (kz > 1) acc -= (kz * (kz - 1.0)) * D[IX(kx, ky, kz - 2)];
            }
        } else if constexpr (ky > 0) {
            acc -= (2.0 * ky - 1.0) * ry * D[IX(kx, ky - 1, kz)];
            if constexpr (ky > 1) acc -= ((ky - 1.0) * (ky - 1.0)) * D[IX(kx, ky - 2, kz)];
            if constexpr (kz > 0) {
                acc -= (2.0 * kz) * rz * D[IX(kx, ky, kz - 1)];
                if constexpr (kz > 1) acc -= (kz * (kz - 1.0)) * D[IX(kx, ky, kz - 2)];
            }
        } else {
            acc -= (2.0 * kz - 1.0) * rz * D[IX(kx, ky, kz - 1)];
            if constexpr (kz > 1) acc -= ((kz - 1.0) * (kz - 1.0)) * D[IX(kx, ky, kz - 2)];
        }
        D[idx] = acc * inv_r2;
    });
}

// One D-recurrence step (src/_taylor.py:57-95) as data: the entry's
// multi-index and the indices of the D values it reads (-1 = term absent),
// pivot first -- D_k = -(1/r^2) [(2k_p - 1) r_p D_{k-e_p} + (k_p - 1)^2
// D_{k-2e_p} + sum over the later axes a: 2 k_a r_a D_{k-e_a} + k_a (k_a - 1)
// D_{k-2e_a}].
struct __align__(16) DRecipe {
    int16_t i1[3], i2[3];  // per axis: k - e_a, k - 2 e_a (pivot axis and later axes only)
    int8_t k[3], pivot;
};
static_assert(sizeof(DRecipe) == 16, "one LDS.128 per recurrence entry");

__device__ inline DRecipe make_recipe(int idx) {
    DRecipe r;
    const int k[3] = {d_tab.mi[idx][0], d_tab.mi[idx][1], d_tab.mi[idx][2]};
    const int pivot = k[0] > 0 ? 0 : (k[1] > 0 ? 1 : 2);
    for (int a = 0; a < 3; a++) {
        r.k[a] = (int8_t)k[a];
        r.i1[a] = r.i2[a] = -1;
        if (a < pivot || k[a] == 0) continue;
        int km[3] = {k[0], k[1], k[2]};
        km[a] -= 1;
        r.i1[a] = d_tab.idx3[km[0]][km[1]][km[2]];
        if (k[a] > 1) {
            km[a] -= 1;
            r.i2[a] = d_tab.idx3[km[0]][km[1]][km[2]];
        }
    }
    r.pivot = (int8_t)pivot;
    return r;
}

}  // namespace fmm
