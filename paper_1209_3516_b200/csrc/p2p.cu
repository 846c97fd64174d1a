// p2p.cu -- near-field particle-particle sums over the P2P plan
// (src/traversal.py:531-548 -> src/_taylor.py:366-407).
//
//   phi_i = sum_j q_j / r_ij,   f_i = sum_j q_j (x_i - x_j) / r_ij^3  (= -grad phi)
//
// Decomposition (B200-first): one CTA per target leaf row.
// Targets are register-blocked K per lane (every lane holds the same K
// targets), LANES RUN OVER SOURCES, so lane utilisation does not depend on
// the leaf size; sources stream as contiguous Morton body runs read with
// coalesced float4 (x, y, z, q) loads (L2-resident at C2; the CTA's warps
// share them through L1).  When a leaf has fewer target blocks than the CTA
// has warps, the remaining warps split the source runs and the partial sums
// are folded through shared memory in a fixed order (deterministic).
// Each warp folds its 32 per-lane partial sums with shuffles at row end.
//
// FP32 fast path per pair: 3 FADD, FMUL + 2 FFMA (r2), MUFU.RSQ, FMUL
// (q*rinv), FADD (phi), 2 FMUL (q*rinv^3), 3 FFMA (force) = 13 FP32-pipe
// instructions + 1 SFU; 20 flops under the reference's cost model.  The
// guarded variant (i != j, r2 > 0) is used only for the self run.
#include <type_traits>

#include "bulk.cuh"
#include "fmm_common.cuh"

namespace fmm {

__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

constexpr int kP2PWarps = 4;

// FMM_PREC_FP32_ACC64 knobs: chunks between float64 flushes (1 measured no
// more accurate than 4 at the C4 corner, and 5 % slower); a Newton step on
// MUFU.RSQ (measured: no accuracy gain there -- the float32 SUMS set the
// floor, not the approximate 1/sqrt -- and 15 % slower, so off)
#ifndef FMM_P2P_FLUSH
#define FMM_P2P_FLUSH 4
#endif
constexpr int kFlush = FMM_P2P_FLUSH;
#ifndef FMM_P2P_ACC_REFINE
#define FMM_P2P_ACC_REFINE 0
#endif
constexpr bool kAccRefine = FMM_P2P_ACC_REFINE;

// Anchor of a row: sources are re-expressed as (hi - a_hi) + (lo - a_lo),
// accurate to the leaf scale when the float64 inputs are not float32-exact.
struct Anchor {
    float hx, hy, hz, lx, ly, lz;
};

// Non-coherent 128-bit load issued where it is written (volatile: the
// compiler may not sink it next to its use, which defeats the prefetch).
__device__ __forceinline__ float4 ldg_pinned(const float4 *p) {
    float4 v;
    asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

template <bool ANCHOR>
__device__ __forceinline__ float4 load_body(const float4 *__restrict__ b, const float4 *__restrict__ blo,
                                            const Anchor &an, int32_t j) {
    float4 s = ldg_pinned(&b[j]);
    if (ANCHOR) {
        const float4 l = __ldg(&blo[j]);
        s.x = (s.x - an.hx) + (l.x - an.lx);
        s.y = (s.y - an.hy) + (l.y - an.ly);
        s.z = (s.z - an.hz) + (l.z - an.lz);
    }
    return s;
}

// K target-source interactions for one source s (13 FP32 ops + 1 MUFU each).
template <int K, bool GUARD>
__device__ __forceinline__ void p2p_f32_pairs(const float4 &s, int32_t rel, const float (&tx)[K],
                                              const float (&ty)[K], const float (&tz)[K], float (&ap)[K],
                                              float (&ax)[K], float (&ay)[K], float (&az)[K]) {
#pragma unroll
    for (int u = 0; u < K; u++) {
        const float dx = tx[u] - s.x;
        const float dy = ty[u] - s.y;
        const float dz = tz[u] - s.z;
        const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        float rinv = rsqrt_approx(r2);
        if (GUARD) rinv = (r2 > 0.0f && rel != u) ? rinv : 0.0f;
        const float qr = s.w * rinv;
        const float qr3 = qr * rinv * rinv;
        ap[u] += qr;
        ax[u] = fmaf(qr3, dx, ax[u]);
        ay[u] = fmaf(qr3, dy, ay[u]);
        az[u] = fmaf(qr3, dz, az[u]);
    }
}

// Packed variant: targets (u, u+1) share one f32x2 register pair, the
// source is a scalar broadcast operand (SASS `Rn.F32`), so one FADD2 /
// FMUL2 / FFMA2 does two pairs' work: 13 packed ops + 2 MUFU per 2 pairs.
// The FP32 lanes (128/clk/SM) become the bound instead of issue slots.
typedef unsigned long long f2_t;

__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
    f2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_unpack(f2_t v, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
// Re-materialise a packed value through a real FADD2 (+0): the result is
// born in an aligned register pair, so ptxas stops re-pairing its halves
// with two MOVs before every packed use.
__device__ __forceinline__ f2_t f2_fresh(f2_t a) {
    f2_t r, z = 0ull;
    asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(z));
    return r;
}
__device__ __forceinline__ f2_t f2_sub_s(f2_t a, float s) {  // a - {s, s}
    f2_t r, b = f2_pack(s, s);
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b) {
    f2_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t f2_mul_s(f2_t a, float s) {
    return f2_mul(a, f2_pack(s, s));
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b) {
    f2_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
    f2_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

template <int K, bool GUARD, bool REFINE = false>
__device__ __forceinline__ void p2p_f32x2_pairs(const float4 &s, int32_t rel, const f2_t (&tx)[K / 2],
                                                const f2_t (&ty)[K / 2], const f2_t (&tz)[K / 2], f2_t (&ap)[K / 2],
                                                f2_t (&ax)[K / 2], f2_t (&ay)[K / 2], f2_t (&az)[K / 2]) {
    // stage-major order: every step runs for all K/2 target pairs before the
    // next, so K/2 independent chains sit between dependent instructions
    constexpr int V = K / 2;
    f2_t dx[V], dy[V], dz[V], r2[V], rinv[V];
#pragma unroll
    for (int v = 0; v < V; v++) dx[v] = f2_sub_s(tx[v], s.x);
#pragma unroll
    for (int v = 0; v < V; v++) dy[v] = f2_sub_s(ty[v], s.y);
#pragma unroll
    for (int v = 0; v < V; v++) dz[v] = f2_sub_s(tz[v], s.z);
#pragma unroll
    for (int v = 0; v < V; v++) r2[v] = f2_mul(dx[v], dx[v]);
#pragma unroll
    for (int v = 0; v < V; v++) r2[v] = f2_fma(dy[v], dy[v], r2[v]);
#pragma unroll
    for (int v = 0; v < V; v++) r2[v] = f2_fma(dz[v], dz[v], r2[v]);
#pragma unroll
    for (int v = 0; v < V; v++) {
        float r2l, r2h;
        f2_unpack(r2[v], r2l, r2h);
        float rl = rsqrt_approx(r2l), rh = rsqrt_approx(r2h);
        if (GUARD) {
            rl = (r2l > 0.0f && rel != 2 * v) ? rl : 0.0f;
            rh = (r2h > 0.0f && rel != 2 * v + 1) ? rh : 0.0f;
        }
        rinv[v] = f2_pack(rl, rh);
    }
    if (REFINE) {  // one Newton step, y (3/2 - r2/2 y^2): MUFU.RSQ's ~2^-22.9 to float32 rounding
        const f2_t mhalf = f2_pack(-0.5f, -0.5f), three_half = f2_pack(1.5f, 1.5f);
#pragma unroll
        for (int v = 0; v < V; v++) {
            const f2_t h = f2_mul(r2[v], mhalf);
            const f2_t yy = f2_mul(rinv[v], rinv[v]);
            rinv[v] = f2_mul(rinv[v], f2_fma(h, yy, three_half));
        }
    }
    f2_t qr[V], rr[V];
#pragma unroll
    for (int v = 0; v < V; v++) qr[v] = f2_mul_s(rinv[v], s.w);
#pragma unroll
    for (int v = 0; v < V; v++) rr[v] = f2_mul(rinv[v], rinv[v]);
#pragma unroll
    for (int v = 0; v < V; v++) ap[v] = f2_add(ap[v], qr[v]);
#pragma unroll
    for (int v = 0; v < V; v++) rr[v] = f2_mul(qr[v], rr[v]);
#pragma unroll
    for (int v = 0; v < V; v++) ax[v] = f2_fma(rr[v], dx[v], ax[v]);
#pragma unroll
    for (int v = 0; v < V; v++) ay[v] = f2_fma(rr[v], dy[v], ay[v]);
#pragma unroll
    for (int v = 0; v < V; v++) az[v] = f2_fma(rr[v], dz[v], az[v]);
}

// cp.async (LDGSTS) helpers: each lane streams ITS OWN sources through a
// private ring of kStages 16-byte slots in shared memory, so no cross-lane
// synchronisation is needed; wait_group(kStages - 2) leaves the next
// kStages - 2 fetches in flight while the current source is consumed.
constexpr int kStages = 4;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// One lane-strided sweep over sources [j0, j1) for K register targets.
// Non-anchored: sources stream through the lane's cp.async ring `ring`.
// Anchored: register loads (the extra residual makes the ring twice as big).
// GUARD (self run only): skip j == own index (rel == u) and r2 == 0.
template <int K, bool GUARD, bool ANCHOR, bool REFINE = false>
__device__ __forceinline__ void p2p_f32_span(int32_t j0, int32_t j1, int step, const float4 *__restrict__ b,
                                             const float4 *__restrict__ blo, const Anchor &an, int32_t i0,
                                             float4 *ring, const f2_t (&tx)[K / 2], const f2_t (&ty)[K / 2],
                                             const f2_t (&tz)[K / 2], f2_t (&ap)[K / 2], f2_t (&ax)[K / 2],
                                             f2_t (&ay)[K / 2], f2_t (&az)[K / 2]) {
    if (j0 >= j1) return;
    if (ANCHOR) {
        for (int32_t j = j0; j < j1; j += step)
            p2p_f32x2_pairs<K, GUARD, REFINE>(load_body<ANCHOR>(b, blo, an, j), j - i0, tx, ty, tz, ap, ax, ay, az);
        return;
    }
    const int32_t nit = (j1 - j0 + step - 1) / step;
    const float4 *gp = b + j0;
#pragma unroll
    for (int k = 0; k < kStages - 1; k++) {
        if (k < nit) cp_async16(&ring[k * 32], gp + k * step);
        cp_async_commit();
    }
    const float4 *gnext = gp + (kStages - 1) * step;
    int32_t it = 0;
    // steady state, unrolled by the ring depth: slots are compile-time and
    // every fetch is in range (no predicate, no modulo)
    if (it + 2 * kStages - 1 <= nit) {
        // the LDS of the next slot is issued before the current slot's math
        cp_async_wait<kStages - 2>();
        float4 cur = ring[0];
        for (; it + 2 * kStages - 1 <= nit; it += kStages) {
#pragma unroll
            for (int q = 0; q < kStages; q++) {
                cp_async16(&ring[((q + kStages - 1) % kStages) * 32], gnext);
                gnext += step;
                cp_async_commit();
                cp_async_wait<kStages - 2>();
                const float4 nxt = ring[((q + 1) % kStages) * 32];
                p2p_f32x2_pairs<K, GUARD, REFINE>(cur, j0 + (it + q) * step - i0, tx, ty, tz, ap, ax, ay, az);
                cur = nxt;
            }
        }
    }
    for (; it < nit; it++) {
        const int32_t nx = it + kStages - 1;
        if (nx < nit) cp_async16(&ring[(nx % kStages) * 32], gnext);
        gnext += step;
        cp_async_commit();
        cp_async_wait<kStages - 1>();
        const float4 s = ring[(it % kStages) * 32];
        p2p_f32x2_pairs<K, GUARD, REFINE>(s, j0 + it * step - i0, tx, ty, tz, ap, ax, ay, az);
    }
}

// Fold the warp's 4*KB per-lane partial sums (phi, fx, fy, fz of KB targets)
// over the 32 lanes by recursive halving: at each step a lane keeps half of
// its values and receives its partner's copy of that half, so the whole fold
// takes 4*KB - 1 shuffles (not 4*KB*5).  Lane l ends holding value index
// l mod 4*KB, i.e. quantity (l mod 4*KB) / KB of target l mod KB.
template <int KB>
__device__ __forceinline__ float warp_fold(const f2_t (&ap)[KB / 2], const f2_t (&ax)[KB / 2],
                                           const f2_t (&ay)[KB / 2], const f2_t (&az)[KB / 2], int lane) {
    constexpr int N = 4 * KB;
    float v[N];
#pragma unroll
    for (int w = 0; w < KB / 2; w++) {
        f2_unpack(ap[w], v[0 * KB + 2 * w], v[0 * KB + 2 * w + 1]);
        f2_unpack(ax[w], v[1 * KB + 2 * w], v[1 * KB + 2 * w + 1]);
        f2_unpack(ay[w], v[2 * KB + 2 * w], v[2 * KB + 2 * w + 1]);
        f2_unpack(az[w], v[3 * KB + 2 * w], v[3 * KB + 2 * w + 1]);
    }
#pragma unroll
    for (int n = N; n > 1; n >>= 1) {
        const int o = n >> 1;  // lane bit that picks the half this lane keeps
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int k = 0; k < n / 2; k++) {
            const float keep = up ? v[k + n / 2] : v[k];
            const float send = up ? v[k] : v[k + n / 2];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
#pragma unroll
    for (int o = N; o < 32; o <<= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    return v[0];
}

// Block of KB consecutive targets starting at i0 (padded with the last
// valid target), all runs of the row, folded over the warp (warp_fold).
// ACC64: the FP32 partials are folded into a float64 sum after every run.
template <int KB, bool SAFE, bool ANCHOR, bool ACC64 = false>
__device__ __forceinline__ std::conditional_t<ACC64, double, float> p2p_f32_block(
    int32_t i0, int32_t ilast, int64_t r0, int64_t r1, int part, int nparts, int lane,
    const int4 *__restrict__ runs, const float4 *__restrict__ b, const float4 *__restrict__ blo, const Anchor &an,
    float4 *ring) {
    f2_t tx[KB / 2], ty[KB / 2], tz[KB / 2], ap[KB / 2], ax[KB / 2], ay[KB / 2], az[KB / 2];
#pragma unroll
    for (int v = 0; v < KB / 2; v++) {
        const float4 e = load_body<ANCHOR>(b, blo, an, min(i0 + 2 * v, ilast));
        const float4 o = load_body<ANCHOR>(b, blo, an, min(i0 + 2 * v + 1, ilast));
        tx[v] = f2_fresh(f2_pack(e.x, o.x));
        ty[v] = f2_fresh(f2_pack(e.y, o.y));
        tz[v] = f2_fresh(f2_pack(e.z, o.z));
        ap[v] = ax[v] = ay[v] = az[v] = 0ull;
    }
    double acc64 = 0.0;
    const int step = 32 * nparts;
    for (int64_t r = r0; r < r1; r++) {
        const int4 run = __ldg(&runs[r]);
        const int32_t j0 = run.x + part * 32 + lane;
        if (SAFE || run.z)
            p2p_f32_span<KB, true, ANCHOR, ACC64 && kAccRefine>(j0, run.y, step, b, blo, an, i0, ring, tx, ty, tz, ap, ax, ay, az);
        else
            p2p_f32_span<KB, false, ANCHOR, ACC64 && kAccRefine>(j0, run.y, step, b, blo, an, i0, ring, tx, ty, tz, ap, ax, ay, az);
        if constexpr (ACC64) {
            acc64 += (double)warp_fold<KB>(ap, ax, ay, az, lane);
#pragma unroll
            for (int v = 0; v < KB / 2; v++) ap[v] = ax[v] = ay[v] = az[v] = 0ull;
        }
    }
    if constexpr (ACC64) return acc64;
    else return warp_fold<KB>(ap, ax, ay, az, lane);
}

// Streamed rows (the fast path): all non-self runs of the row form ONE
// source sequence (the run table sits in shared memory).  A unit (target
// block tb, part p of P) takes the p-th of P equal contiguous shares of the
// sequence, in chunks of kChunk = 32 * kSPL consecutive sources.  Each warp streams its chunks
// through a private ring of kWStages shared-memory stages: lane 0 copies a
// chunk in with one cp.async.bulk per run segment (UBLKCP: one instruction
// moves up to the whole chunk) that completes on the stage's mbarrier, and
// the lanes read it back with one LDS.128 per source.  Per source and lane
// this leaves the LDS next to the 13 * KB / 2 packed FP32 ops -- the
// per-lane address, run-seek and cp.async bookkeeping of a lane-private
// stream are gone -- and the warps stay independent of each other.
// The target leaf's own bodies are swept first in a short guarded pass (the
// only place i == j or r2 == 0 can occur for float32-exact inputs).
constexpr int kMaxRuns = 512;
#ifndef FMM_P2P_SPL
#define FMM_P2P_SPL 8
#endif
#ifndef FMM_P2P_WSTAGES
#define FMM_P2P_WSTAGES 2
#endif
constexpr int kSPL = FMM_P2P_SPL;          // sources per lane per chunk
constexpr int kWStages = FMM_P2P_WSTAGES;  // chunks in flight per warp
constexpr int kChunk = 32 * kSPL;          // sources per chunk

// Lane 0's cursor into the run table: run r starts at sequence position rpos.
struct RunCursor {
    int r;
    int32_t rpos;
};

// Copy sequence positions [p0, p0 + need) into `dst` (lane 0 only): walk
// the cursor forward to p0, then one bulk copy per run segment.
template <typename T>
__device__ __forceinline__ void chunk_produce(T *dst, uint64_t *bar, int32_t p0, int32_t need, RunCursor &c,
                                              const int2 *srun, const T *__restrict__ b) {
    // (no proxy fence: every LDS of this stage has returned -- its values were
    // consumed by the math -- before the __syncwarp that precedes us)
    constexpr uint32_t kBytes = sizeof(T);
    mbar_expect_tx(bar, (uint32_t)need * kBytes);
    int2 run = srun[c.r];
    while (c.rpos + (run.y - run.x) <= p0) {
        c.rpos += run.y - run.x;
        run = srun[++c.r];
    }
    int32_t off = p0 - c.rpos;
    while (need > 0) {
        const int32_t take = min(run.y - run.x - off, need);
        if (take > 0) bulk_g2s(dst, b + run.x + off, (uint32_t)take * kBytes, bar);
        dst += take;
        need -= take;
        if (need > 0) {
            c.rpos += run.y - run.x;
            run = srun[++c.r];
            off = 0;
        }
    }
}

// One unit of a streamed row: KB targets from i0 (padded with the last
// valid target) against sources [s0, s1) of the block's source line, which
// is the target leaf's own cnt bodies (positions [0, cnt), guarded sweep)
// followed by the run sequence (positions cnt + [0, total)).  `ring` is the
// warp's kWStages * kChunk stage buffer, `bars` its barriers, `phase` their
// parity bits (one per stage).
// ACC64 (precision FMM_PREC_FP32_ACC64): pair terms in float32, the lanes'
// float32 partials folded into a float64 sum every kFlush chunks (and after
// the self sweep), so the rounding of long float32 sums never builds up:
// at the C4 corner the near field's error floor drops from ~5.5e-7 to
// ~1.1e-7 relative for 5-7 % more time.

template <int KB, bool ACC64 = false>
__device__ __forceinline__ std::conditional_t<ACC64, double, float> p2p_f32_stream_unit(
    int32_t i0, int32_t ilast, int32_t ts, int32_t cnt, int32_t s0, int32_t s1, int lane,
    const float4 *__restrict__ b, float4 *ring, uint64_t *bars, uint32_t &phase, const int2 *srun) {
    f2_t tx[KB / 2], ty[KB / 2], tz[KB / 2], ap[KB / 2], ax[KB / 2], ay[KB / 2], az[KB / 2];
    // the stream share [lo, hi), cut into chunks from lo; the first chunks
    // are requested before anything else so they land during the self sweep
    const int32_t lo = max(s0, cnt) - cnt, hi = max(s1, cnt) - cnt;
    const int nk = (hi - lo + kChunk - 1) / kChunk;
    RunCursor cur{0, 0};
    if (lane == 0)
        for (int k = 0; k < min(nk, kWStages); k++) {
            const int32_t p0 = lo + k * kChunk;
            chunk_produce(ring + k * kChunk, &bars[k], p0, min(kChunk, hi - p0), cur, srun, b);
        }
#pragma unroll
    for (int v = 0; v < KB / 2; v++) {
        const float4 e = __ldg(&b[min(i0 + 2 * v, ilast)]);
        const float4 o = __ldg(&b[min(i0 + 2 * v + 1, ilast)]);
        tx[v] = f2_fresh(f2_pack(e.x, o.x));
        ty[v] = f2_fresh(f2_pack(e.y, o.y));
        tz[v] = f2_fresh(f2_pack(e.z, o.z));
        ap[v] = ax[v] = ay[v] = az[v] = 0ull;
    }
    double acc64 = 0.0;
    auto flush = [&]() {
        if constexpr (ACC64) {
            acc64 += (double)warp_fold<KB>(ap, ax, ay, az, lane);
#pragma unroll
            for (int v = 0; v < KB / 2; v++) ap[v] = ax[v] = ay[v] = az[v] = 0ull;
        }
    };
    // 1) the self share, guarded
    for (int32_t j = ts + s0 + lane; j < ts + min(s1, cnt); j += 32)
        p2p_f32x2_pairs<KB, true, ACC64 && kAccRefine>(__ldg(&b[j]), j - i0, tx, ty, tz, ap, ax, ay, az);
    flush();
    // 2) the chunks
    int st = 0;
    for (int k = 0; k < nk; k++) {
        if (k > 0 && lane == 0 && k - 1 + kWStages < nk) {  // refill the stage consumed last iteration
            const int sp = st == 0 ? kWStages - 1 : st - 1;
            const int32_t p0 = lo + (k - 1 + kWStages) * kChunk;
            chunk_produce(ring + sp * kChunk, &bars[sp], p0, min(kChunk, hi - p0), cur, srun, b);
        }
        __syncwarp();
        mbar_wait(&bars[st], (phase >> st) & 1u);
        phase ^= 1u << st;
        const float4 *src = ring + st * kChunk + lane;
        const int32_t valid = hi - (lo + k * kChunk);
        if (valid >= kChunk) {
            float4 s = src[0];
#pragma unroll
            for (int q = 0; q < kSPL; q++) {
                const float4 nxt = src[((q + 1) % kSPL) * 32];
                p2p_f32x2_pairs<KB, false, ACC64 && kAccRefine>(s, 0, tx, ty, tz, ap, ax, ay, az);
                s = nxt;
            }
        } else {
#pragma unroll 1
            for (int q = 0; q < kSPL; q++)
                if (q * 32 + lane < valid)
                    p2p_f32x2_pairs<KB, false, ACC64 && kAccRefine>(src[q * 32], 0, tx, ty, tz, ap, ax, ay, az);
        }
        __syncwarp();  // every lane is done with stage st before lane 0 refills it
        if (++st == kWStages) st = 0;
        if (ACC64 && (k % kFlush == kFlush - 1 || k == nk - 1)) flush();
    }
    if constexpr (ACC64) return acc64;
    else return warp_fold<KB>(ap, ax, ay, az, lane);
}

// Target blocks of a leaf: cnt / 8 blocks of 8, then the remainder as one
// block of 4 (r <= 4) or 8 -- at most 3 padded slots per leaf.
__device__ __forceinline__ int gcd_small(int a, int b) {
    while (b) {
        const int t = a % b;
        a = b;
        b = t;
    }
    return a;
}

// Work units of a row: every target block's source stream is split into P
// interleaved parts with P = W / gcd(nblk, W), so the nblk * P units divide
// evenly over the W warps of the CTA (no warp idles at the row barrier).
// Partial sums of the parts are folded through shared memory in a fixed
// order (deterministic).  Leaves too large for the fold buffer (oversized
// leaves) fall back to P = 1 with direct stores.
// FMM_P2P_BLK = 8 (default): blocks of 8 targets per lane, the last block
// of a leaf 4 or 8; = 4: every block 4 targets (fewer registers, more
// resident warps: an occupancy experiment)
#ifndef FMM_P2P_BLK
#define FMM_P2P_BLK 8
#endif
constexpr int kBlk = FMM_P2P_BLK;
constexpr bool kK4Only = kBlk == 4;
constexpr int kMaxUnits = kK4Only ? 128 : 64;

template <bool SAFE, bool ANCHOR>
constexpr int p2p_f32_pool_bytes() {
    return (!SAFE && !ANCHOR ? kP2PWarps * kWStages * kChunk : kP2PWarps * kStages * 32) * (int)sizeof(float4);
}

#ifndef FMM_P2P_MINB
#define FMM_P2P_MINB 4  // resident CTAs per SM the register budget is cut for
#endif
template <bool SAFE, bool ANCHOR, bool ACC64 = false>
__global__ void __launch_bounds__(kP2PWarps * 32, FMM_P2P_MINB) p2p_f32_kernel(
    int32_t nrows_host, const int32_t *__restrict__ nrows_dev, const int32_t *__restrict__ leaf_rows, const int32_t *__restrict__ start,
    const int32_t *__restrict__ end, const int64_t *__restrict__ run_off, const int4 *__restrict__ runs,
    const float4 *__restrict__ b, const float4 *__restrict__ blo, double *phi, double *fx, double *fy,
    double *fz, int *flag, int cross) {
    constexpr bool kStream = !SAFE && !ANCHOR;
    // the tile ring (streamed rows) and the lane rings (run-by-run rows) share
    // one pool: a row uses one or the other
    extern __shared__ __align__(128) float4 pool[];  // p2p_f32_pool_bytes<SAFE, ANCHOR>()
    using acc_t = std::conditional_t<ACC64, double, float>;
    __shared__ acc_t red[kMaxUnits][4][kBlk];
    __shared__ int2 srun[kMaxRuns];
    __shared__ int32_t stotal;
    __shared__ uint64_t wbars[kP2PWarps][kWStages];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float4 *ring = &pool[w * kStages * 32 + lane];
    if (kStream && lane == 0) {
        for (int k = 0; k < kWStages; k++) mbar_init(&wbars[w][k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    float4 *wring = pool + w * kWStages * kChunk;
    uint32_t phase = 0;  // parity of each of this warp's stage barriers
    const int32_t nrows = nrows_dev ? *nrows_dev : nrows_host;
    for (int row = blockIdx.x; row < nrows; row += gridDim.x) {
        const int32_t t = leaf_rows[row];
        const int32_t ts = start[t], cnt = end[t] - ts;
        const int rem = cnt & (kBlk - 1);
        const int nblk = cnt / kBlk + (rem ? 1 : 0);
        const bool small_last = !kK4Only && rem != 0 && rem <= 4;
        const int64_t r0 = run_off[2 * (int64_t)row], r1 = run_off[2 * (int64_t)row + 1];
        const int nr = (int)(r1 - r0);
        // streamed rows split every block's source line over the warps by
        // weight (P = kP2PWarps partials per block, folded below)
        const bool streamed = kStream && nr <= kMaxRuns && nblk * kP2PWarps <= kMaxUnits;
        int P = streamed ? kP2PWarps : kP2PWarps / gcd_small(nblk, kP2PWarps);
        const bool fold = nblk * P <= kMaxUnits;
        if (!fold) P = 1;
        const int nunits = nblk * P;
        Anchor an{};
        if (ANCHOR) {
            const float4 h = __ldg(&b[ts]), l = __ldg(&blo[ts]);
            an = Anchor{h.x, h.y, h.z, l.x, l.y, l.z};
        }
        if (streamed) {
            if (threadIdx.x == 0) stotal = 0;
            for (int k = threadIdx.x; k < nunits * 4 * kBlk; k += blockDim.x) (&red[0][0][0])[k] = acc_t(0);
            __syncthreads();
            int32_t len = 0;
            for (int k = threadIdx.x; k < nr; k += blockDim.x) {
                const int4 rr = __ldg(&runs[r0 + k]);
                const int2 v = rr.z ? make_int2(rr.x, rr.x) : make_int2(rr.x, rr.y);  // self run: empty
                srun[k] = v;
                len += v.y - v.x;
            }
            for (int o = 16; o > 0; o >>= 1) len += __shfl_xor_sync(0xffffffffu, len, o);
            if (lane == 0) atomicAdd(&stotal, len);
            __syncthreads();
        }
        // a unit's folded sums: lane l holds quantity q of target uu
        auto emit = [&](int u, int tb, int32_t i0, bool k4, acc_t val) {
            const int q = k4 ? (lane >> 2) & 3 : lane >> 3;
            const int uu = k4 ? lane & 3 : lane & 7;
            if (fold) {
                if (lane < (k4 ? 16 : 32)) red[u][q][uu] = val;
            } else if (lane < (k4 ? 16 : 32) && tb * kBlk + uu < cnt) {
                double *out = q == 0 ? phi : q == 1 ? fx : q == 2 ? fy : fz;
                out[i0 + uu] = (double)val;
                if (!isfinite(val)) atomicOr(flag, 1);
            }
        };
        if (streamed) {
            // block tb's line: cnt self sources + total stream sources, weight
            // 2 per source (K8) or 1 (the K4 last block); warp w takes the
            // w-th quarter of the concatenated weighted lines
            const int32_t scnt = cross ? 0 : cnt;  // cross-tree rows have no self leaf
            const int64_t L = (int64_t)scnt + stotal;
            constexpr int64_t bw = kK4Only ? 1 : 2;  // weight per source of a full block
            const int64_t Wl = L * (bw * nblk - (small_last ? 1 : 0));
            const int64_t A = Wl * w / kP2PWarps, B = Wl * (w + 1) / kP2PWarps;
            for (int tb = (int)(A / (bw * L)); tb < nblk && bw * L * tb < B; tb++) {
                const bool k4 = kK4Only || (tb == nblk - 1 && small_last);
                const int64_t Sb = bw * L * tb, sc = k4 ? 1 : 2;
                const int32_t s0 = (int32_t)((max(A, Sb) - Sb) / sc);
                const int32_t s1 = (int32_t)((min(B, Sb + sc * L) - Sb) / sc);
                if (s1 <= s0) continue;
                const int32_t i0 = ts + tb * kBlk;
                const acc_t val =
                    k4 ? p2p_f32_stream_unit<4, ACC64>(i0, ts + cnt - 1, ts, scnt, s0, s1, lane, b, wring, wbars[w],
                                                       phase, srun)
                       : p2p_f32_stream_unit<8, ACC64>(i0, ts + cnt - 1, ts, scnt, s0, s1, lane, b, wring, wbars[w],
                                                       phase, srun);
                emit(tb * kP2PWarps + w, tb, i0, k4, val);
            }
        } else {
            for (int u = w; u < nunits; u += kP2PWarps) {
                const int tb = u / P, part = u % P;
                const int32_t i0 = ts + tb * kBlk;
                const bool k4 = kK4Only || (tb == nblk - 1 && small_last);
                const acc_t val =
                    k4 ? p2p_f32_block<4, SAFE, ANCHOR, ACC64>(i0, ts + cnt - 1, r0, r1, part, P, lane, runs, b, blo,
                                                               an, ring)
                       : p2p_f32_block<8, SAFE, ANCHOR, ACC64>(i0, ts + cnt - 1, r0, r1, part, P, lane, runs, b, blo,
                                                               an, ring);
                emit(u, tb, i0, k4, val);
            }
        }
        __syncthreads();  // partial sums complete; srun / pool may be rewritten after this
        if (fold) {
            for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
                const int tb = k / kBlk, l = k % kBlk;
                acc_t p_ = 0, x_ = 0, y_ = 0, z_ = 0;
                for (int q = 0; q < P; q++) {  // fixed order: deterministic
                    const int uu = tb * P + q;
                    p_ += red[uu][0][l];
                    x_ += red[uu][1][l];
                    y_ += red[uu][2][l];
                    z_ += red[uu][3][l];
                }
                const int32_t i = ts + k;
                phi[i] = (double)p_;
                fx[i] = (double)x_;
                fy[i] = (double)y_;
                fz[i] = (double)z_;
                if (!(isfinite(p_) && isfinite(x_) && isfinite(y_) && isfinite(z_))) atomicOr(flag, 1);
            }
            __syncthreads();  // red is rewritten by the next row
        }
    }
}

// ---- FP64 streamed variant (parity mode, and the promoted near field of
// precision="fp32" at the high-order corner) -------------------------------
//
// Same decomposition as the FP32 streamed rows: one CTA per target leaf row,
// 4 warps, every target block's source line (self leaf guarded, then the
// row's non-self run sequence) split over the warps by weight, the run
// sequence streamed per warp through a 2-stage ring of double4 chunks filled
// by cp.async.bulk on mbarriers.  Targets are register-blocked 4 per lane.
// 1/sqrt(r2) is MUFU.RSQ64H (rsqrt.approx.f64, ~2^-23 relative) refined by
// one third-order step, y + y e (1/2 + 3/8 e) with e = 1 - r2 y^2 (error
// O(e^3), below float64 rounding), instead of IEEE div + sqrt: 5 FP64 ops
// against 2 Newton steps' 8.  Each lane's sums are float64 throughout.
constexpr int kK64 = 4;                 // targets per lane
constexpr int kSPL64 = 4;               // sources per lane per chunk
constexpr int kChunk64 = 32 * kSPL64;   // sources per chunk
constexpr int kMaxUnits64 = 128;        // 4 parts x 32 blocks (ncrit <= 128 folds)

__device__ __forceinline__ double rsqrt_f64(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-(x * y), y, 1.0);
    return fma(y * e, fma(0.375, e, 0.5), y);
}

template <bool GUARD>
__device__ __forceinline__ void p2p_f64_pairs(const double4 &s, int32_t rel, const double (&tx)[kK64],
                                              const double (&ty)[kK64], const double (&tz)[kK64], double (&ap)[kK64],
                                              double (&ax)[kK64], double (&ay)[kK64], double (&az)[kK64]) {
#pragma unroll
    for (int u = 0; u < kK64; u++) {
        const double dx = tx[u] - s.x, dy = ty[u] - s.y, dz = tz[u] - s.z;
        const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
        double rinv = rsqrt_f64(r2);
        if (GUARD) rinv = (r2 > 0.0 && rel != u) ? rinv : 0.0;
        const double qr = s.w * rinv;
        const double qr3 = qr * rinv * rinv;
        ap[u] += qr;
        ax[u] = fma(qr3, dx, ax[u]);
        ay[u] = fma(qr3, dy, ay[u]);
        az[u] = fma(qr3, dz, az[u]);
    }
}

// warp_fold for the 16 float64 sums of a 4-target block: lane l ends holding
// value index l mod 16 = quantity (l mod 16) / 4 of target l mod 4.
__device__ __forceinline__ double warp_fold_f64(const double (&ap)[kK64], const double (&ax)[kK64],
                                                const double (&ay)[kK64], const double (&az)[kK64], int lane) {
    constexpr int N = 4 * kK64;
    double v[N];
#pragma unroll
    for (int u = 0; u < kK64; u++) {
        v[u] = ap[u];
        v[kK64 + u] = ax[u];
        v[2 * kK64 + u] = ay[u];
        v[3 * kK64 + u] = az[u];
    }
#pragma unroll
    for (int n = N; n > 1; n >>= 1) {
        const int o = n >> 1;
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int k = 0; k < n / 2; k++) {
            const double keep = up ? v[k + n / 2] : v[k];
            const double send = up ? v[k] : v[k + n / 2];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
#pragma unroll
    for (int o = N; o < 32; o <<= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    return v[0];
}

// One unit of a streamed FP64 row (see p2p_f32_stream_unit).  GUARD_ALL
// (cross-tree rows) guards every source against r2 == 0.
template <bool GUARD_ALL>
__device__ __forceinline__ double p2p_f64_stream_unit(int32_t i0, int32_t ilast, int32_t ts, int32_t cnt, int32_t s0,
                                                      int32_t s1, int lane, const double4 *__restrict__ b,
                                                      double4 *ring, uint64_t *bars, uint32_t &phase,
                                                      const int2 *srun) {
    double tx[kK64], ty[kK64], tz[kK64], ap[kK64], ax[kK64], ay[kK64], az[kK64];
    const int32_t lo = max(s0, cnt) - cnt, hi = max(s1, cnt) - cnt;
    const int nk = (hi - lo + kChunk64 - 1) / kChunk64;
    RunCursor cur{0, 0};
    if (lane == 0)
        for (int k = 0; k < min(nk, kWStages); k++) {
            const int32_t p0 = lo + k * kChunk64;
            chunk_produce(ring + k * kChunk64, &bars[k], p0, min(kChunk64, hi - p0), cur, srun, b);
        }
#pragma unroll
    for (int u = 0; u < kK64; u++) {
        const double4 t = b[min(i0 + u, ilast)];
        tx[u] = t.x;
        ty[u] = t.y;
        tz[u] = t.z;
        ap[u] = ax[u] = ay[u] = az[u] = 0.0;
    }
    for (int32_t j = ts + s0 + lane; j < ts + min(s1, cnt); j += 32)
        p2p_f64_pairs<true>(b[j], j - i0, tx, ty, tz, ap, ax, ay, az);
    int st = 0;
    for (int k = 0; k < nk; k++) {
        if (k > 0 && lane == 0 && k - 1 + kWStages < nk) {
            const int sp = st == 0 ? kWStages - 1 : st - 1;
            const int32_t p0 = lo + (k - 1 + kWStages) * kChunk64;
            chunk_produce(ring + sp * kChunk64, &bars[sp], p0, min(kChunk64, hi - p0), cur, srun, b);
        }
        __syncwarp();
        mbar_wait(&bars[st], (phase >> st) & 1u);
        phase ^= 1u << st;
        const double4 *src = ring + st * kChunk64 + lane;
        const int32_t valid = hi - (lo + k * kChunk64);
        if (valid >= kChunk64) {
            double4 s = src[0];
#pragma unroll
            for (int q = 0; q < kSPL64; q++) {
                const double4 nxt = src[((q + 1) % kSPL64) * 32];
                p2p_f64_pairs<GUARD_ALL>(s, -1, tx, ty, tz, ap, ax, ay, az);
                s = nxt;
            }
        } else {
#pragma unroll 1
            for (int q = 0; q < kSPL64; q++)
                if (q * 32 + lane < valid) p2p_f64_pairs<GUARD_ALL>(src[q * 32], -1, tx, ty, tz, ap, ax, ay, az);
        }
        __syncwarp();
        if (++st == kWStages) st = 0;
    }
    return warp_fold_f64(ap, ax, ay, az, lane);
}

// One unit of a row that does not stream (more than kMaxRuns runs): block tb
// against every run, part `part` of P lane-interleaved parts, from global.
__device__ __forceinline__ double p2p_f64_runs_unit(int32_t i0, int32_t ilast, int64_t r0, int64_t r1, int part,
                                                    int P, int lane, bool guard_all, const int4 *__restrict__ runs,
                                                    const double4 *__restrict__ b) {
    double tx[kK64], ty[kK64], tz[kK64], ap[kK64], ax[kK64], ay[kK64], az[kK64];
#pragma unroll
    for (int u = 0; u < kK64; u++) {
        const double4 t = b[min(i0 + u, ilast)];
        tx[u] = t.x;
        ty[u] = t.y;
        tz[u] = t.z;
        ap[u] = ax[u] = ay[u] = az[u] = 0.0;
    }
    const int step = 32 * P;
    for (int64_t r = r0; r < r1; r++) {
        const int4 run = __ldg(&runs[r]);
        if (run.z || guard_all) {
            for (int32_t j = run.x + part * 32 + lane; j < run.y; j += step)
                p2p_f64_pairs<true>(b[j], j - i0, tx, ty, tz, ap, ax, ay, az);
        } else {
            for (int32_t j = run.x + part * 32 + lane; j < run.y; j += step)
                p2p_f64_pairs<false>(b[j], -1, tx, ty, tz, ap, ax, ay, az);
        }
    }
    return warp_fold_f64(ap, ax, ay, az, lane);
}

#ifndef FMM_P2P64_MINB
#define FMM_P2P64_MINB 4
#endif
template <bool CROSS>
__global__ void __launch_bounds__(kP2PWarps * 32, FMM_P2P64_MINB) p2p_f64s_kernel(
    int32_t nrows_host, const int32_t *__restrict__ nrows_dev, const int32_t *__restrict__ leaf_rows,
    const int32_t *__restrict__ start, const int32_t *__restrict__ end, const int64_t *__restrict__ run_off,
    const int4 *__restrict__ runs, const double4 *__restrict__ b, double *phi, double *fx, double *fy, double *fz) {
    extern __shared__ __align__(128) double4 pool64[];  // kP2PWarps * kWStages * kChunk64
    __shared__ double red[kMaxUnits64][4][kK64];
    __shared__ int2 srun[kMaxRuns];
    __shared__ int32_t stotal;
    __shared__ uint64_t wbars[kP2PWarps][kWStages];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        for (int k = 0; k < kWStages; k++) mbar_init(&wbars[w][k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    double4 *wring = pool64 + w * kWStages * kChunk64;
    uint32_t phase = 0;
    const int32_t nrows = nrows_dev ? *nrows_dev : nrows_host;
    for (int row = blockIdx.x; row < nrows; row += gridDim.x) {
        const int32_t t = leaf_rows[row];
        const int32_t ts = start[t], cnt = end[t] - ts;
        const int nblk = (cnt + kK64 - 1) / kK64;
        const int64_t r0 = run_off[2 * (int64_t)row], r1 = run_off[2 * (int64_t)row + 1];
        const int nr = (int)(r1 - r0);
        const bool fold = nblk * kP2PWarps <= kMaxUnits64;
        const bool streamed = fold && nr <= kMaxRuns;
        if (streamed) {
            if (threadIdx.x == 0) stotal = 0;
            __syncthreads();
            int32_t len = 0;
            for (int k = threadIdx.x; k < nr; k += blockDim.x) {
                const int4 rr = __ldg(&runs[r0 + k]);
                const int2 v = rr.z ? make_int2(rr.x, rr.x) : make_int2(rr.x, rr.y);  // self run: swept apart
                srun[k] = v;
                len += v.y - v.x;
            }
            for (int o = 16; o > 0; o >>= 1) len += __shfl_xor_sync(0xffffffffu, len, o);
            if (lane == 0) atomicAdd(&stotal, len);
        }
        if (fold)
            for (int k = threadIdx.x; k < nblk * kP2PWarps * 4 * kK64; k += blockDim.x) (&red[0][0][0])[k] = 0.0;
        __syncthreads();
        // lane l holds quantity (l >> 2) & 3 of target l & 3
        auto emit = [&](int u, int tb, double val) {
            const int q = (lane >> 2) & 3, uu = lane & 3;
            if (lane >= 16) return;
            if (fold) {
                red[u][q][uu] = val;
            } else if (tb * kK64 + uu < cnt) {
                double *out = q == 0 ? phi : q == 1 ? fx : q == 2 ? fy : fz;
                out[ts + tb * kK64 + uu] = val;
            }
        };
        if (streamed) {
            const int32_t scnt = CROSS ? 0 : cnt;
            const int64_t L = (int64_t)scnt + stotal;
            const int64_t Wl = L * nblk;
            const int64_t A = Wl * w / kP2PWarps, B = Wl * (w + 1) / kP2PWarps;
            for (int tb = (int)(L > 0 ? A / L : nblk); tb < nblk && L * tb < B; tb++) {
                const int64_t Sb = L * tb;
                const int32_t s0 = (int32_t)(max(A, Sb) - Sb), s1 = (int32_t)(min(B, Sb + L) - Sb);
                if (s1 <= s0) continue;
                const double val = p2p_f64_stream_unit<CROSS>(ts + tb * kK64, ts + cnt - 1, ts, scnt, s0, s1, lane,
                                                             b, wring, wbars[w], phase, srun);
                emit(tb * kP2PWarps + w, tb, val);
            }
        } else {
            const int P = fold ? kP2PWarps : 1;
            for (int u = w; u < nblk * P; u += kP2PWarps) {
                const int tb = u / P, part = u % P;
                const double val =
                    p2p_f64_runs_unit(ts + tb * kK64, ts + cnt - 1, r0, r1, part, P, lane, CROSS, runs, b);
                emit(tb * kP2PWarps + part, tb, val);
            }
        }
        __syncthreads();
        if (fold) {
            for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
                const int tb = k / kK64, l = k % kK64;
                double p_ = 0.0, x_ = 0.0, y_ = 0.0, z_ = 0.0;
                for (int q = 0; q < kP2PWarps; q++) {  // fixed order: deterministic
                    const int uu = tb * kP2PWarps + q;
                    p_ += red[uu][0][l];
                    x_ += red[uu][1][l];
                    y_ += red[uu][2][l];
                    z_ += red[uu][3][l];
                }
                const int32_t i = ts + k;
                phi[i] = p_;
                fx[i] = x_;
                fy[i] = y_;
                fz[i] = z_;
            }
            __syncthreads();
        }
    }
}

__global__ void pack_b64_kernel(int64_t n, const double *__restrict__ xs, const double *__restrict__ ys,
                                const double *__restrict__ zs, const double *__restrict__ qs, double4 *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = make_double4(xs[i], ys[i], zs[i], qs[i]);
}

// ---- FP64 variant (use_rsqrt: the reference's float32 1/sqrt, FP64 sums) --
template <int K>
__global__ void __launch_bounds__(kP2PWarps * 32) p2p_f64_kernel(
    int32_t nrows_host, const int32_t *__restrict__ nrows_dev, const int32_t *__restrict__ leaf_rows, const int32_t *__restrict__ start,
    const int32_t *__restrict__ end, const int64_t *__restrict__ run_off, const int4 *__restrict__ runs,
    const double *__restrict__ xs, const double *__restrict__ ys, const double *__restrict__ zs,
    const double *__restrict__ qs, int use_rsqrt, double *phi, double *fx, double *fy, double *fz) {
    __shared__ double red[kP2PWarps][4 * K];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int32_t nrows = nrows_dev ? *nrows_dev : nrows_host;
    for (int row = blockIdx.x; row < nrows; row += gridDim.x) {
        const int32_t t = leaf_rows[row];
        const int32_t ts = start[t], cnt = end[t] - ts;
        const int nblk = (cnt + K - 1) / K;
        const int nparts = nblk >= kP2PWarps ? 1 : kP2PWarps / nblk;
        const int64_t r0 = run_off[2 * (int64_t)row], r1 = run_off[2 * (int64_t)row + 1];
        const int rounds = (nblk + kP2PWarps - 1) / kP2PWarps;
        for (int rd = 0; rd < (nparts > 1 ? 1 : rounds); rd++) {
            int tb, part;
            if (nparts > 1) { tb = w % nblk; part = w / nblk; }
            else { tb = rd * kP2PWarps + w; part = 0; }
            const bool active = (nparts > 1) ? (part < nparts) : (tb < nblk);
            double tx[K], ty[K], tz[K], ap[K], ax[K], ay[K], az[K];
            int32_t ti[K];
            if (active) {
#pragma unroll
                for (int u = 0; u < K; u++) {
                    int32_t i = ts + min(tb * K + u, cnt - 1);
                    tx[u] = xs[i]; ty[u] = ys[i]; tz[u] = zs[i];
                    ti[u] = i;
                    ap[u] = ax[u] = ay[u] = az[u] = 0.0;
                }
                const int step = 32 * nparts;
                for (int64_t r = r0; r < r1; r++) {
                    const int4 run = __ldg(&runs[r]);
                    for (int32_t j = run.x + part * 32 + lane; j < run.y; j += step) {
                        const double sx = xs[j], sy = ys[j], sz = zs[j], sq = qs[j];
#pragma unroll
                        for (int u = 0; u < K; u++) {
                            const double dx = tx[u] - sx, dy = ty[u] - sy, dz = tz[u] - sz;
                            const double r2 = dx * dx + dy * dy + dz * dz;
                            double rinv = use_rsqrt ? (double)(1.0f / sqrtf((float)r2)) : 1.0 / sqrt(r2);
                            rinv = (r2 > 0.0 && j != ti[u]) ? rinv : 0.0;
                            const double qr = sq * rinv;
                            const double qr3 = qr * rinv * rinv;
                            ap[u] += qr;
                            ax[u] += qr3 * dx;
                            ay[u] += qr3 * dy;
                            az[u] += qr3 * dz;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < K; u++) {
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        ap[u] += __shfl_xor_sync(0xffffffffu, ap[u], o);
                        ax[u] += __shfl_xor_sync(0xffffffffu, ax[u], o);
                        ay[u] += __shfl_xor_sync(0xffffffffu, ay[u], o);
                        az[u] += __shfl_xor_sync(0xffffffffu, az[u], o);
                    }
                }
            }
            if (nparts > 1) {
                if (active && lane == 0) {
#pragma unroll
                    for (int u = 0; u < K; u++) {
                        red[w][u] = ap[u];
                        red[w][K + u] = ax[u];
                        red[w][2 * K + u] = ay[u];
                        red[w][3 * K + u] = az[u];
                    }
                }
                __syncthreads();
                if (active && part == 0) {
#pragma unroll
                    for (int u = 0; u < K; u++) {
                        double p_ = 0, x_ = 0, y_ = 0, z_ = 0;
                        for (int q = 0; q < nparts; q++) {
                            const int ww = q * nblk + tb;
                            p_ += red[ww][u];
                            x_ += red[ww][K + u];
                            y_ += red[ww][2 * K + u];
                            z_ += red[ww][3 * K + u];
                        }
                        ap[u] = p_; ax[u] = x_; ay[u] = y_; az[u] = z_;
                    }
                }
                __syncthreads();
            }
            if (active && part == 0) {
#pragma unroll
                for (int u = 0; u < K; u++) {
                    if (lane == u && tb * K + u < cnt) {
                        const int32_t i = ts + tb * K + u;
                        phi[i] = ap[u];
                        fx[i] = ax[u];
                        fy[i] = ay[u];
                        fz[i] = az[u];
                    }
                }
            }
        }
    }
}

// Coincident (target, source) pairs of a cross-tree plan: r2 == 0.0 in
// float64 -- the reference skips and counts them (src/traversal.py:552-597).
// A block per row, threads over the row's (target, source) pairs.
__global__ void p2p_coincident_kernel(int32_t nrows_host, const int32_t *__restrict__ nrows_dev,
                                      const int32_t *__restrict__ leaf_rows, const int32_t *__restrict__ start,
                                      const int32_t *__restrict__ end, const int64_t *__restrict__ run_off,
                                      const int4 *__restrict__ runs, const double *__restrict__ xs,
                                      const double *__restrict__ ys, const double *__restrict__ zs,
                                      unsigned long long *count) {
    const int32_t nrows = nrows_dev ? *nrows_dev : nrows_host;
    unsigned long long local = 0;
    for (int row = blockIdx.x; row < nrows; row += gridDim.x) {
        const int32_t t = leaf_rows[row];
        const int32_t ts = start[t], cnt = end[t] - ts;
        for (int64_t r = run_off[2 * (int64_t)row]; r < run_off[2 * (int64_t)row + 1]; r++) {
            const int4 run = runs[r];
            const int64_t len = run.y - run.x, tot = len * cnt;
            for (int64_t k = threadIdx.x; k < tot; k += blockDim.x) {
                const int32_t i = ts + (int32_t)(k / len), j = run.x + (int32_t)(k % len);
                const double dx = __dsub_rn(xs[i], xs[j]), dy = __dsub_rn(ys[i], ys[j]), dz = __dsub_rn(zs[i], zs[j]);
                const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
                local += r2 == 0.0;
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

}  // namespace fmm

using namespace fmm;

extern "C" int fmm_p2p(int precision, int safe, int use_rsqrt, int cross, int32_t nrows, const int32_t *dev_nrows,
                       const int32_t *leaf_rows,
                       const int32_t *start, const int32_t *end, const int64_t *run_off, const void *runs,
                       const double *xs, const double *ys, const double *zs, const double *qs,
                       const void *b32, const void *b32lo, double *phi, double *fx, double *fy, double *fz,
                       int *dev_flag, void *stream) {
    if (nrows <= 0) return FMM_OK;
    cudaStream_t s = as_stream(stream);
    const int grid = nrows;
    if (precision == FMM_PREC_FP32 || precision == FMM_PREC_FP32_ANCHORED || precision == FMM_PREC_FP32_ACC64) {
        if (!b32) { set_error("fp32 P2P needs the float4 body copy"); return FMM_ERR_INVALID; }
        const bool acc64 = precision == FMM_PREC_FP32_ACC64;
        if (acc64 && safe) { set_error("fp32-acc64 P2P has no guarded redo (use fp64)"); return FMM_ERR_INVALID; }
        const bool anch = precision == FMM_PREC_FP32_ANCHORED;
        if (anch && !b32lo) { set_error("anchored fp32 P2P needs the float4 residual copy"); return FMM_ERR_INVALID; }
        auto kern = anch ? (safe ? p2p_f32_kernel<true, true> : p2p_f32_kernel<false, true>)
                         : (safe ? p2p_f32_kernel<true, false> : p2p_f32_kernel<false, false>);
        if (acc64) kern = p2p_f32_kernel<false, false, true>;
        const int pool = anch ? (safe ? p2p_f32_pool_bytes<true, true>() : p2p_f32_pool_bytes<false, true>())
                              : (safe ? p2p_f32_pool_bytes<true, false>() : p2p_f32_pool_bytes<false, false>());
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pool);
        kern<<<grid, kP2PWarps * 32, pool, s>>>(nrows, dev_nrows, leaf_rows, start, end, run_off, (const int4 *)runs,
                                             (const float4 *)b32, (const float4 *)b32lo, phi, fx, fy, fz,
                                             dev_flag, cross); fmm::note_launch();
    } else if (precision == FMM_PREC_FP64 && b32 && !use_rsqrt) {
        // streamed rows over the double4 body copy (fmm_pack_bodies_f64)
        auto kern = cross ? p2p_f64s_kernel<true> : p2p_f64s_kernel<false>;
        const int pool = kP2PWarps * kWStages * kChunk64 * (int)sizeof(double4);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pool);
        kern<<<grid, kP2PWarps * 32, pool, s>>>(nrows, dev_nrows, leaf_rows, start, end, run_off, (const int4 *)runs,
                                                (const double4 *)b32, phi, fx, fy, fz); fmm::note_launch();
    } else if (precision == FMM_PREC_FP64) {
        p2p_f64_kernel<4><<<grid, kP2PWarps * 32, 0, s>>>(nrows, dev_nrows, leaf_rows, start, end, run_off,
                                                          (const int4 *)runs, xs, ys, zs, qs, use_rsqrt, phi,
                                                          fx, fy, fz); fmm::note_launch();
    } else {
        set_error("bad precision %d", precision);
        return FMM_ERR_INVALID;
    }
    FMM_CUDA_CHECK("fmm_p2p");
    return FMM_OK;
}

extern "C" int fmm_p2p_coincident(int32_t nrows, const int32_t *dev_nrows, const int32_t *leaf_rows,
                                  const int32_t *start, const int32_t *end, const int64_t *run_off, const void *runs,
                                  const double *xs, const double *ys, const double *zs, unsigned long long *count,
                                  void *stream) {
    if (nrows <= 0) return FMM_OK;
    p2p_coincident_kernel<<<grid_for(nrows, 1, 148 * 8), 256, 0, as_stream(stream)>>>(
        nrows, dev_nrows, leaf_rows, start, end, run_off, (const int4 *)runs, xs, ys, zs, count); fmm::note_launch();
    FMM_CUDA_CHECK("fmm_p2p_coincident");
    return FMM_OK;
}

extern "C" int fmm_pack_bodies_f64(int64_t n, const double *xs, const double *ys, const double *zs, const double *qs,
                                   void *out, void *stream) {
    if (n <= 0) return FMM_OK;
    pack_b64_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, xs, ys, zs, qs, (double4 *)out);
    fmm::note_launch();
    FMM_CUDA_CHECK("fmm_pack_bodies_f64");
    return FMM_OK;
}
