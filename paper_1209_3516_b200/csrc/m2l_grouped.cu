// m2l_grouped.cu -- M2L by lattice-offset group on the FP64 tensor pipe
// (fmm_m2l_grouped): the reference's contraction (src/traversal.py:500-517
// -> src/_taylor.py:169-188, D by the recurrence of :57-95) regrouped so
// that pairs sharing one D tensor become a matrix product.
#include <cub/cub.cuh>

#include "bulk.cuh"
#include "taylor.cuh"

namespace fmm {

// ---- offset-grouped M2L on the FP64 tensor pipe (DMMA), p >= 6 -----------
// With cubic cells and geometric centres every M2L vector is a lattice
// vector: r = o * u, u = root_size / 2^(L+1) for L = max(level_t, level_s),
// o an integer triple (C4 at theta = 0.3: 11.7M pairs, 14,128 distinct
// (level_t, level_s, o)).  Pairs that share (level_t, level_s, o) share D,
// so the contraction L_n += sum_m T_nm M_m with T_nm = (-1)^|m| D_{n+m}
// becomes a matrix product once targets are batched: a CTA owns a BATCH of
// up to 8 target cells of one level at the same octant of Morton-consecutive
// parents (their lists are near-translates: 72 % of the 8 columns filled
// at C4), walks the union of their groups in key order and, per group, applies
// the (NC x NC, block-triangular) T to the 8 source moment columns with
// mma.m8n8k4.f64 (tile (n-tile i, m-tile j) is needed iff deg(8i) + deg(4j)
// <= p-1: 197 DMMAs per group at p = 10, 79 % of their MACs useful).
// Measured on B200: DMMA 37 TFLOP/s, DFMA 34 (tools/probes/fp64_probe.cu),
// and one DMMA is 256 FMAs per warp instruction, which leaves the issue
// slots to the operand loads.
//
// D per distinct group is computed once (a device hash of the group keys,
// the reference's recurrence src/_taylor.py:57-95 per table row, stored
// with its negation so the A fragment's (-1)^|m| is an index).  One
// producer warp streams each group's D row and the batch's source moment
// rows into a STAGES-deep shared-memory ring with cp.async.bulk on
// mbarriers; the consumer warps own fixed n-tiles and keep the batch's
// 8 x NC local expansions in DMMA accumulators until the batch ends, then
// add them to L once -- no atomics, and the order is fixed by the sort
// (deterministic).  Pairs off the lattice (centres rounded away from it,
// e.g. a cloud far from the origin) become single-pair groups whose D the
// producer computes from their own r.
template <int P>
struct MG {
    static constexpr int NC = ncoef(P);
    static constexpr int NT = (NC + 7) / 8;  // n-tiles (8 outputs)
    static constexpr int MT = (NC + 3) / 4;  // m-tiles (4 moments)
    static constexpr int NCP = MT * 4;
    // moment row stride (doubles): room for a one-element alignment shift,
    // and 2 RS = 8 mod 32 banks so the B fragment's 4 slots x 4 moments of
    // a half warp hit distinct banks
    static constexpr int RS = (NCP + 1) + (((4 - (NCP + 1) % 16) % 16) + 16) % 16;
    static constexpr int DS = 2 * NC + 2;  // D, 0, -D, 0
    static constexpr int NW = 4;           // consumer warps
    static constexpr int STAGES = P >= 9 ? 3 : 4;
};

// Tile schedule of one order, evaluated once.  The NW consumer warps form
// an NG x KG grid: n-tiles go to the NG row groups (LPT over J[i], the
// number of m-tiles paired with n-tile i -- a prefix, deg(4j) grows with
// j), and within a row group the m-tiles go to its KG warps (LPT over the
// tiles they carry).  Each B fragment (moment column j) is then loaded by
// NG warps instead of all NW, and the KG warps of a row group sum their
// accumulators once per batch.  slot[i][j] is tile (i, j)'s place in its
// owner's per-lane index array.
// KG = 2 from p = 9 (C4: p = 9 3.44 -> 3.28 ms, p = 10 8.29 -> 8.18), 1 at
// p = 8 (4.82 against 5.28 ms); KG = 4 doubles the accumulators and drops
// to 2 CTAs per SM (p = 10 14.2 ms).  FMM_MG_KG overrides (experiments).
#ifdef FMM_MG_KG
constexpr int mg_kg(int) { return FMM_MG_KG; }
#else
constexpr int mg_kg(int p) { return p >= 9 ? 2 : 1; }
#endif
template <int P>
struct MGSched {
    static constexpr int KG = mg_kg(P), NG = MG<P>::NW / KG;
    int J[MG<P>::NT];
    int ng[MG<P>::NT];
    int owner[MG<P>::NT][MG<P>::MT];
    int slot[MG<P>::NT][MG<P>::MT];
    int count[MG<P>::NW];
    bool col_used[MG<P>::NW][MG<P>::MT];
    int maxcount;
};

template <int P>
constexpr MGSched<P> make_mg_sched() {
    using G = MG<P>;
    using S = MGSched<P>;
    MGSched<P> s{};
    for (int i = 0; i < G::NT; i++) {
        s.J[i] = 0;
        const int dn = 8 * i < G::NC ? kTab.deg[8 * i] : 99;
        for (int j = 0; j < G::MT; j++)
            if (dn + kTab.deg[4 * j] <= P - 1) s.J[i]++;
    }
    int gload[S::NG] = {};
    for (int i = 0; i < G::NT; i++) {
        int g = 0;
        for (int q = 1; q < S::NG; q++)
            if (gload[q] < gload[g]) g = q;
        gload[g] += s.J[i];
        s.ng[i] = g;
    }
    for (int i = 0; i < G::NT; i++)
        for (int j = 0; j < G::MT; j++) s.owner[i][j] = s.slot[i][j] = -1;
    for (int g = 0; g < S::NG; g++) {
        int kload[S::KG] = {};
        for (int j = 0; j < G::MT; j++) {
            int c = 0;
            for (int i = 0; i < G::NT; i++)
                if (s.ng[i] == g && j < s.J[i]) c++;
            if (!c) continue;
            int k = 0;
            for (int q = 1; q < S::KG; q++)
                if (kload[q] < kload[k]) k = q;
            kload[k] += c;
            for (int i = 0; i < G::NT; i++)
                if (s.ng[i] == g && j < s.J[i]) s.owner[i][j] = g * S::KG + k;
        }
    }
    for (int w = 0; w < G::NW; w++) {
        s.count[w] = 0;
        for (int j = 0; j < G::MT; j++) s.col_used[w][j] = false;
    }
    for (int i = 0; i < G::NT; i++)
        for (int j = 0; j < G::MT; j++)
            if (s.owner[i][j] >= 0) {
                s.slot[i][j] = s.count[s.owner[i][j]]++;
                s.col_used[s.owner[i][j]][j] = true;
            }
    s.maxcount = 1;
    for (int w = 0; w < G::NW; w++) s.maxcount = s.count[w] > s.maxcount ? s.count[w] : s.maxcount;
    return s;
}

template <int P>
inline constexpr MGSched<P> kMGS = make_mg_sched<P>();

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// A-fragment source for lane `lane` of tile (i, j): index into the signed D
// row (DS entries) -- (-1)^|m| D_{n+m}, or a zero slot.
template <int P>
__device__ __forceinline__ int mg_tile_index(int i, int j, int lane) {
    using G = MG<P>;
    const int n = 8 * i + (lane >> 2), m = 4 * j + (lane & 3);
    if (n >= G::NC || m >= G::NC) return G::NC;
    const int dn = d_tab.deg[n], dm = d_tab.deg[m];
    if (dn + dm > P - 1) return G::NC;
    const int v = d_tab.idx3[d_tab.mi[n][0] + d_tab.mi[m][0]][d_tab.mi[n][1] + d_tab.mi[m][1]]
                            [d_tab.mi[n][2] + d_tab.mi[m][2]];
    return (dm & 1) ? G::NC + 1 + v : v;
}

// D_k(r), deg k < P, by the reference's recurrence into a signed row
// (D, 0, -D, 0) -- one thread (the group table) ...
template <int P>
__device__ __forceinline__ void mg_d_row_thread(double rx, double ry, double rz, double *row) {
    constexpr int NC = ncoef(P);
    double D[NC];
    d_tensors_reg<P>(rx, ry, rz, D);
#pragma unroll
    for (int i = 0; i < NC; i++) {
        row[i] = D[i];
        row[NC + 1 + i] = -D[i];
    }
    row[NC] = 0.0;
    row[2 * NC + 1] = 0.0;
}

// ... or one warp, degree by degree (the producer's off-lattice groups)
template <int P>
__device__ __forceinline__ void mg_d_row_warp(const double (&r)[3], const DRecipe *rec, double *D, int lane) {
    constexpr int NC = ncoef(P);
    double *Dn = D + NC + 1;
    const double inv_r2 = 1.0 / (r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    if (lane == 0) {
        const double d0 = sqrt(inv_r2);
        D[0] = d0;
        Dn[0] = -d0;
        D[NC] = 0.0;
        Dn[NC] = 0.0;
    }
    __syncwarp();
#pragma unroll 1
    for (int d = 1; d < P; d++) {
        for (int idx = ncoef(d) + lane; idx < ncoef(d + 1); idx += 32) {
            const DRecipe q = rec[idx];
            const int pv = q.pivot;
            double a = 0.0;
#pragma unroll
            for (int ax = 0; ax < 3; ax++) {
                if (q.i1[ax] < 0) continue;
                const double kk = (double)q.k[ax];
                a -= (ax == pv ? 2.0 * kk - 1.0 : 2.0 * kk) * r[ax] * D[q.i1[ax]];
                if (q.i2[ax] >= 0) a -= (ax == pv ? (kk - 1.0) * (kk - 1.0) : kk * (kk - 1.0)) * D[q.i2[ax]];
            }
            a *= inv_r2;
            D[idx] = a;
            Dn[idx] = -a;
        }
        __syncwarp();
    }
}

template <int P, int W>
__device__ __forceinline__ void mg_consume(const double *__restrict__ sD, const double *__restrict__ brow,
                                           const int (&tix)[kMGS<P>.maxcount], double (&acc)[MG<P>::NT][2]) {
    using G = MG<P>;
    static_for<0, G::MT>([&](auto Ij) {
        constexpr int j = decltype(Ij)::value;
        if constexpr (kMGS<P>.col_used[W][j]) {
            const double b = brow[4 * j];
            static_for<0, G::NT>([&](auto Ii) {
                constexpr int i = decltype(Ii)::value;
                if constexpr (kMGS<P>.owner[i][j] == W) {
                    constexpr int sl = kMGS<P>.slot[i][j];
                    dmma884(acc[i], sD[tix[sl]], b);
                }
            });
        }
    });
}

template <int P>
struct MGSmem {
    static constexpr int KG = MGSched<P>::KG;
    double D[MG<P>::STAGES][MG<P>::DS];
    union {
        double M[MG<P>::STAGES][8 * MG<P>::RS];
        double red[KG > 1 ? KG - 1 : 1][MG<P>::NT][64];  // the batch-end sum of a row group's KG warps
    };
    double zero[MG<P>::NCP];
    uint64_t full[MG<P>::STAGES], empty[MG<P>::STAGES];
    int rowoff[MG<P>::STAGES][8];
    DRecipe rec[MG<P>::NC];
    int tcell[8];
    double tctr[8][3];
};

template <int P, int W>
__device__ __forceinline__ void mg_consumer(int32_t e0, int32_t e1, MGSmem<P> &sm, double *L) {
    using G = MG<P>;
    using S = MGSched<P>;
    constexpr int g = W / S::KG, kq = W % S::KG;
    const int lane = threadIdx.x & 31;
    int tix[kMGS<P>.maxcount];
    static_for<0, G::NT>([&](auto Ii) {
        constexpr int i = decltype(Ii)::value;
        static_for<0, G::MT>([&](auto Ij) {
            constexpr int j = decltype(Ij)::value;
            if constexpr (kMGS<P>.owner[i][j] == W) {
                constexpr int sl = kMGS<P>.slot[i][j];
                tix[sl] = mg_tile_index<P>(i, j, lane);
            }
        });
    });
    double acc[G::NT][2];
#pragma unroll
    for (int i = 0; i < G::NT; i++) acc[i][0] = acc[i][1] = 0.0;
    for (int32_t e = e0; e < e1; e++) {
        const int u = e - e0, st = u % G::STAGES;
        mbar_wait(&sm.full[st], (u / G::STAGES) & 1);
        const int ro = sm.rowoff[st][lane >> 2];
        const double *brow = (ro >= 0 ? &sm.M[st][ro] : sm.zero) + (lane & 3);
        mg_consume<P, W>(sm.D[st], brow, tix, acc);
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[st]);
    }
    if constexpr (S::KG > 1) {
        // every group is consumed (all bulk copies landed): the stage ring
        // is free for the row groups' fold, in a fixed order (deterministic)
        asm volatile("bar.sync 1, %0;" ::"n"(G::NW * 32) : "memory");
        if constexpr (kq > 0)
            static_for<0, G::NT>([&](auto Ii) {
                constexpr int i = decltype(Ii)::value;
                if constexpr (kMGS<P>.ng[i] == g) {
                    sm.red[kq - 1][i][2 * lane] = acc[i][0];
                    sm.red[kq - 1][i][2 * lane + 1] = acc[i][1];
                }
            });
        asm volatile("bar.sync 1, %0;" ::"n"(G::NW * 32) : "memory");
        if constexpr (kq > 0) return;
        static_for<0, G::NT>([&](auto Ii) {
            constexpr int i = decltype(Ii)::value;
            if constexpr (kMGS<P>.ng[i] == g) {
#pragma unroll
                for (int q = 0; q < S::KG - 1; q++) {
                    acc[i][0] += sm.red[q][i][2 * lane];
                    acc[i][1] += sm.red[q][i][2 * lane + 1];
                }
            }
        });
    }
    // C fragment: row n = 8 i + lane/4, columns (target slots) 2 (lane%4) + {0, 1}
    static_for<0, G::NT>([&](auto Ii) {
        constexpr int i = decltype(Ii)::value;
        if constexpr (kMGS<P>.ng[i] == g) {
            const int n = 8 * i + (lane >> 2);
            if (n < G::NC) {
                const double inv = 1.0 / d_tab.mfact[n];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int t = sm.tcell[2 * (lane & 3) + h];
                    if (t >= 0) L[(int64_t)t * G::NC + n] += acc[i][h] * inv;
                }
            }
        }
    });
}

// producer: entry e's D row and moment rows into stage st (lane roles:
// lanes 0..7 one slot each, lane 8 the D row)
template <int P>
__device__ __forceinline__ void mg_produce(int32_t e, int st, MGSmem<P> &sm, const int32_t *__restrict__ ent_start,
                                           const int32_t *__restrict__ ent_gid, const uint64_t *__restrict__ gkey,
                                           const int32_t *__restrict__ gsrc, const double *__restrict__ Dtab,
                                           const double *__restrict__ ctr, const double *__restrict__ M, int lane) {
    using G = MG<P>;
    constexpr int NC = G::NC;
    const int32_t k0 = ent_start[e], k1 = ent_start[e + 1];
    const int32_t gid = ent_gid[e];
    const int32_t k = k0 + lane;
    const bool valid = lane < 8 && k < k1;
    const int myslot = valid ? (int)(gkey[k] & 7) : 0;
    const int mysrc = valid ? gsrc[k] : -1;
    const unsigned smask = __reduce_or_sync(0xffffffffu, valid ? 1u << myslot : 0u);
    // slot l's source sits at lane popc(smask below l) (slots ascend within a group)
    const int lsl = lane & 7;
    const int from = __popc(smask & ((1u << lsl) - 1u));
    const int s_l = __shfl_sync(0xffffffffu, mysrc, from);
    const bool present = lane < 8 && ((smask >> lane) & 1u);
    int64_t start = 0;
    uint32_t bytes_l = 0;
    if (present) {
        start = (int64_t)s_l * NC;
        const int64_t a0 = (start + 1) & ~1ll, b0 = (start + NC) & ~1ll;  // 16 B-aligned interior
        double *row = &sm.M[st][lane * G::RS + (int)(start & 1)];
        if (a0 > start) row[0] = __ldg(&M[start]);
        if (b0 < start + NC) row[NC - 1] = __ldg(&M[start + NC - 1]);
        bytes_l = (uint32_t)((b0 - a0) * 8);
        sm.rowoff[st][lane] = lane * G::RS + (int)(start & 1);
    } else if (lane < 8) {
        sm.rowoff[st][lane] = -1;
    }
    if (gid < 0) {  // off the lattice (or past the table): D from the group's own r
        const int slot0 = __shfl_sync(0xffffffffu, myslot, 0), src0 = __shfl_sync(0xffffffffu, mysrc, 0);
        const double r[3] = {sm.tctr[slot0][0] - ctr[src0 * 3], sm.tctr[slot0][1] - ctr[src0 * 3 + 1],
                             sm.tctr[slot0][2] - ctr[src0 * 3 + 2]};
        mg_d_row_warp<P>(r, sm.rec, sm.D[st], lane);
    }
    uint32_t bytes = bytes_l;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
    if (gid >= 0) bytes += (uint32_t)(G::DS * 8);
    __syncwarp();
    if (lane == 0) mbar_expect_tx(&sm.full[st], bytes);  // the stage's one arrival
    __syncwarp();
    if (present && bytes_l) {
        const int64_t a0 = (start + 1) & ~1ll;
        bulk_g2s(&sm.M[st][lane * G::RS + (int)(start & 1) + (int)(a0 - start)], M + a0, bytes_l, &sm.full[st]);
    }
    if (lane == 8 && gid >= 0) bulk_g2s(sm.D[st], Dtab + (int64_t)gid * G::DS, G::DS * 8, &sm.full[st]);
}

template <int P>
__global__ void __launch_bounds__((MG<P>::NW + 1) * 32) m2l_dmma(
    const uint64_t *__restrict__ gkey, const int32_t *__restrict__ gsrc, const int32_t *__restrict__ ent_start,
    const int32_t *__restrict__ ent_gid, const int32_t *__restrict__ bent, const int32_t *__restrict__ bent_end,
    const int32_t *__restrict__ batch_cells, int32_t nbatch_max, const double *__restrict__ Dtab,
    const double *__restrict__ ctr, const double *__restrict__ M, double *L) {
    using G = MG<P>;
    constexpr int NC = G::NC;
    extern __shared__ __align__(16) unsigned char mg_smem_raw[];
    MGSmem<P> &sm = *reinterpret_cast<MGSmem<P> *>(mg_smem_raw);
    const int b = blockIdx.x;
    if (b >= nbatch_max) return;
    const int32_t e0 = bent[b], e1 = bent_end[b];
    if (e0 >= e1) return;
    for (int i = threadIdx.x; i < NC; i += blockDim.x) sm.rec[i] = make_recipe(i);
    for (int i = threadIdx.x; i < G::STAGES * 8 * G::RS; i += blockDim.x) (&sm.M[0][0])[i] = 0.0;  // finite padding
    for (int i = threadIdx.x; i < G::NCP; i += blockDim.x) sm.zero[i] = 0.0;
    if (threadIdx.x < 8) {
        const int t = batch_cells[b * 8 + threadIdx.x];
        sm.tcell[threadIdx.x] = t;
        for (int a = 0; a < 3; a++) sm.tctr[threadIdx.x][a] = t >= 0 ? ctr[t * 3 + a] : 0.0;
    }
    if (threadIdx.x == 0) {
        for (int q = 0; q < G::STAGES; q++) {
            mbar_init(&sm.full[q], 1);
            mbar_init(&sm.empty[q], G::NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < G::NW) {
        switch (warp) {
            case 0: mg_consumer<P, 0>(e0, e1, sm, L); break;
            case 1: mg_consumer<P, 1>(e0, e1, sm, L); break;
            case 2: mg_consumer<P, 2>(e0, e1, sm, L); break;
            default: mg_consumer<P, 3>(e0, e1, sm, L); break;
        }
        return;
    }
    for (int32_t e = e0; e < e1; e++) {
        const int u = e - e0, st = u % G::STAGES;
        if (u >= G::STAGES) mbar_wait(&sm.empty[st], ((u / G::STAGES) - 1) & 1);
        mg_produce<P>(e, st, sm, ent_start, ent_gid, gkey, gsrc, Dtab, ctr, M, lane);
    }
}

// ---- grouping pre-pass ----------------------------------------------------
constexpr uint64_t kMgNone = ~0ull;
// D-key table: 2^20 slots; up to kMgDCap groups get a D row (C4 at theta =
// 0.3: 14,128 groups; the adaptive C3 tree: 22,129 at 0.5, 166,647 at 0.3).
// Groups past the cap keep their batching, and the producer forms their D.
constexpr int kMgHashBits = 20;
constexpr int kMgDCap = 131072;

__device__ __forceinline__ uint32_t mg_hash(uint64_t k) {
    return (uint32_t)((k * 0x9E3779B97F4A7C15ull) >> (64 - kMgHashBits));
}

// batch order of the target cells: (level, octant in the parent, the
// parent's key) -- cells of one level at one relative position in Morton-
// consecutive parents, whose lists are near-translates (C4 theta = 0.3: 72 %
// of the batch columns filled; the octant of the last two levels: 62 %)
__global__ void mg_cell_keys(int32_t ncells, const int64_t *__restrict__ rows, const int8_t *__restrict__ level,
                             const uint64_t *__restrict__ ckey, uint64_t *out, int32_t *iota) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncells; c += gridDim.x * blockDim.x) {
        iota[c] = c;
        if (rows[c + 1] <= rows[c]) {
            out[c] = kMgNone;
            continue;
        }
        const int l = level[c];
        const uint64_t k = ckey[c];
        const uint64_t low = k & 7ull, high = k >> 3;
        const int hb = 3 * l - 3;
        const uint64_t h55 = hb > 55 ? high >> (hb - 55) : high;
        out[c] = ((uint64_t)l << 58) | (low << 55) | h55;
    }
}

__global__ void mg_level_segments(int32_t ncells, const uint64_t *__restrict__ skey, int32_t *seg /* [2][32] */) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ncells; i += gridDim.x * blockDim.x) {
        if (skey[i] == kMgNone) continue;
        const int l = (int)(skey[i] >> 58);
        if (i == 0 || (int)(skey[i - 1] >> 58) != l) seg[l] = i;
        if (i == ncells - 1 || skey[i + 1] == kMgNone || (int)(skey[i + 1] >> 58) != l) seg[32 + l] = i + 1;
    }
}

__global__ void mg_assign(int32_t ncells, const uint64_t *__restrict__ skey, const int32_t *__restrict__ scell,
                          const int32_t *__restrict__ seg, int32_t *cell_tag, int32_t *batch_cells) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ncells; i += gridDim.x * blockDim.x) {
        if (skey[i] == kMgNone) continue;
        const int l = (int)(skey[i] >> 58);
        int base = 0;
        for (int q = 0; q < l; q++) base += (seg[32 + q] - seg[q] + 7) >> 3;
        const int j = i - seg[l];
        const int b = base + (j >> 3), slot = j & 7;
        const int c = scell[i];
        cell_tag[c] = b * 8 + slot;
        batch_cells[b * 8 + slot] = c;
    }
}

// D-key of a lattice group: (level_t, level_s - level_t, o) + 1 (0 = empty slot)
__device__ __forceinline__ uint64_t mg_dkey(int lt, uint64_t gcode) { return (((uint64_t)lt << 35) | gcode) + 1; }

// one warp per target row: pair key = batch << 40 | group << 3 | slot, the
// group a lattice code (level delta, o) or (1 << 36 | slot | source id)
// off the lattice; lattice D-keys are inserted into the hash table
__global__ void mg_pair_keys(int32_t ncells, const int64_t *__restrict__ rows, const int32_t *__restrict__ src,
                             const int8_t *__restrict__ level, const double *__restrict__ ctr,
                             const double *__restrict__ root, const int32_t *__restrict__ cell_tag, int64_t cap,
                             unsigned long long *htab, uint64_t *key, int32_t *val) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    const double size = root[3];
    for (int64_t t = wid; t < ncells; t += nw) {
        const int64_t k0 = rows[t], k1 = rows[t + 1];
        if (k0 == k1) continue;
        const int tag = cell_tag[t], lt = level[t];
        const double cx = ctr[t * 3], cy = ctr[t * 3 + 1], cz = ctr[t * 3 + 2];
        for (int64_t k = k0 + lane; k < k1; k += 32) {
            const int s = src[k], ls = level[s];
            const int L = lt > ls ? lt : ls;
            const double u = ldexp(size, -(L + 1));
            const double r[3] = {cx - ctr[s * 3], cy - ctr[s * 3 + 1], cz - ctr[s * 3 + 2]};
            // on the lattice to float64 rounding of the centres (D from o u is then the
            // per-pair D to ~1e-13 relative)
            bool lat = (ls - lt) >= -15 && (ls - lt) <= 15;
            uint64_t g = (uint64_t)(ls - lt + 16) << 30;
#pragma unroll
            for (int a = 0; a < 3; a++) {
                const double o = rint(r[a] / u);
                lat = lat && fabs(o) <= 511.0 && fabs(o * u - r[a]) <= 0x1p-45 * u;
                g |= (uint64_t)(((int)o + 512) & 1023) << (20 - 10 * a);
            }
            if (lat) {  // insert the D-key (linear probing); a full table leaves the pair off the lattice
                const unsigned long long dk = mg_dkey(lt, g);
                uint32_t h = mg_hash(dk);
                bool done = false;
                for (int probe = 0; probe < 64 && !done; probe++, h = (h + 1) & ((1u << kMgHashBits) - 1)) {
                    const unsigned long long cur = htab[h];
                    if (cur == dk) done = true;
                    else if (cur == 0ull) {
                        const unsigned long long prev = atomicCAS(&htab[h], 0ull, dk);
                        done = prev == 0ull || prev == dk;
                    }
                }
                lat = done;
            }
            if (!lat) g = (1ull << 36) | ((uint64_t)(tag & 7) << 30) | (uint64_t)s;  // one pair per group
            key[k] = ((uint64_t)(tag >> 3) << 40) | (g << 3) | (uint64_t)(tag & 7);
            val[k] = s;
        }
    }
    // capacity padding sorts last
    const int64_t n = rows[ncells];
    for (int64_t k = n + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < cap; k += gridDim.x * (int64_t)blockDim.x)
        key[k] = kMgNone;
}

// dense ids for the table's D-keys and their signed D rows (thread per slot)
template <int P>
__global__ void mg_table_rows(const unsigned long long *__restrict__ htab, const double *__restrict__ root,
                              int32_t *hid, int32_t *ngroups, double *Dtab, int64_t dcap) {
    const double size = root[3];
    for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < (1 << kMgHashBits); h += gridDim.x * blockDim.x) {
        const unsigned long long dk1 = htab[h];
        if (!dk1) continue;
        const int id = atomicAdd(ngroups, 1);
        hid[h] = id < dcap ? id : -1;
        if (id >= dcap) continue;
        const uint64_t dk = dk1 - 1;
        const int lt = (int)(dk >> 35), dl = (int)((dk >> 30) & 31) - 16;
        const int L = dl > 0 ? lt + dl : lt;
        const double u = ldexp(size, -(L + 1));
        double r[3];
#pragma unroll
        for (int a = 0; a < 3; a++) r[a] = (double)((int)((dk >> (20 - 10 * a)) & 1023) - 512) * u;
        mg_d_row_thread<P>(r[0], r[1], r[2], Dtab + (int64_t)id * MG<P>::DS);
    }
}

__global__ void mg_entry_flags(const int64_t *__restrict__ rows, int32_t ncells, int64_t cap,
                               const uint64_t *__restrict__ key, int32_t *flag) {
    const int64_t n = rows[ncells];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap; i += gridDim.x * (int64_t)blockDim.x)
        flag[i] = i < n && (i == 0 || (key[i] >> 3) != (key[i - 1] >> 3));
}

// per group entry: its first pair, its D row (-1: the producer computes D),
// and each batch's entry range
__global__ void mg_entries(const int64_t *__restrict__ rows, int32_t ncells, const uint64_t *__restrict__ key,
                           const int32_t *__restrict__ flag, const int32_t *__restrict__ eidx,
                           const int8_t *__restrict__ level, const int32_t *__restrict__ batch_cells,
                           const unsigned long long *__restrict__ htab, const int32_t *__restrict__ hid,
                           int32_t *ent_start, int32_t *ent_gid, int32_t *bent, int32_t *bent_end) {
    const int64_t n = rows[ncells];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (int64_t)blockDim.x) {
        const int32_t e = eidx[i] + flag[i] - 1;  // the entry holding pair i
        const uint64_t b = key[i] >> 40;
        if (flag[i]) {
            ent_start[e] = (int32_t)i;
            const uint64_t g = (key[i] >> 3) & ((1ull << 37) - 1);
            int32_t gid = -1;
            if (!(g >> 36)) {
                const int lt = level[batch_cells[b * 8]];
                const unsigned long long dk = mg_dkey(lt, g);
                uint32_t h = mg_hash(dk);
                for (int probe = 0; probe < 64; probe++, h = (h + 1) & ((1u << kMgHashBits) - 1))
                    if (htab[h] == dk) {
                        gid = hid[h];
                        break;
                    }
            }
            ent_gid[e] = gid;
        }
        if (i == 0 || (key[i - 1] >> 40) != b) bent[b] = e;
        if (i == n - 1 || (key[i + 1] >> 40) != b) bent_end[b] = e + 1;
        if (i == n - 1) ent_start[e + 1] = (int32_t)n;
    }
}

}  // namespace fmm

using namespace fmm;

// ---- grouped M2L entry points ---------------------------------------------
namespace {
struct MgLayout {
    uint64_t *ckey[2], *pkey[2];
    int32_t *iota, *scell, *seg, *cell_tag, *batch_cells, *pval[2], *flag, *eidx, *ent_start, *ent_gid, *bent,
        *bent_end, *hid, *ngroups;
    unsigned long long *htab;
    double *Dtab;
    void *tmp;
    size_t tmp_bytes;
    int64_t dcap;
    int32_t nbmax;
    int end_bit;
};

size_t mg_tmp_bytes(int32_t ncells, int64_t cap, int end_bit) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, (int)ncells, 0, 64);
    cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, cap, 0, end_bit);
    cub::DeviceScan::ExclusiveSum(nullptr, c, (const int32_t *)nullptr, (int32_t *)nullptr, cap);
    return a > b ? (a > c ? a : c) : (b > c ? b : c);
}

// bytes used (the layout is filled when ws is given and large enough)
size_t mg_layout(int p, int32_t ncells, int64_t cap, void *ws, size_t ws_bytes, MgLayout *lay) {
    MgLayout l{};
    l.nbmax = ncells / 8 + 23;
    int kb = 1;
    while ((1ll << kb) <= l.nbmax) kb++;
    l.end_bit = 40 + kb;
    int64_t dcap = cap < kMgDCap ? cap : kMgDCap;
    const int64_t dmem = ((int64_t)512 << 20) / ((2 * ncoef(p) + 2) * 8);  // <= 512 MB of D rows
    if (dcap > dmem) dcap = dmem;
    l.dcap = dcap;
    Arena A(ws, ws ? ws_bytes : ~(size_t)0 >> 2);
    l.ckey[0] = A.take<uint64_t>(ncells);
    l.ckey[1] = A.take<uint64_t>(ncells);
    l.iota = A.take<int32_t>(ncells);
    l.scell = A.take<int32_t>(ncells);
    l.seg = A.take<int32_t>(64);
    l.ngroups = A.take<int32_t>(1);
    l.cell_tag = A.take<int32_t>(ncells);
    l.batch_cells = A.take<int32_t>((size_t)l.nbmax * 8);
    l.bent = A.take<int32_t>(l.nbmax);
    l.bent_end = A.take<int32_t>(l.nbmax);
    l.htab = A.take<unsigned long long>((size_t)1 << kMgHashBits);
    l.hid = A.take<int32_t>((size_t)1 << kMgHashBits);
    l.Dtab = A.take<double>((size_t)dcap * (2 * ncoef(p) + 2));
    for (int q = 0; q < 2; q++) {
        l.pkey[q] = A.take<uint64_t>(cap);
        l.pval[q] = A.take<int32_t>(cap);
    }
    l.flag = A.take<int32_t>(cap);
    l.eidx = A.take<int32_t>(cap);
    l.ent_start = A.take<int32_t>(cap + 1);
    l.ent_gid = A.take<int32_t>(cap);
    l.tmp_bytes = mg_tmp_bytes(ncells, cap, l.end_bit);
    void *tmp = A.take<char>(l.tmp_bytes);
    l.tmp = tmp;
    if (lay) *lay = l;
    if (ws && !tmp) return 0;  // does not fit
    return A.used + 256;
}

template <int P>
int mg_launch(const MgLayout &l, const double *root, const double *ctr, const double *M, double *L, cudaStream_t s) {
    mg_table_rows<P><<<grid_for((int64_t)1 << kMgHashBits, 128, 148 * 8), 128, 0, s>>>(l.htab, root, l.hid,
                                                                                       l.ngroups, l.Dtab, l.dcap);
    fmm::note_launch();
    return 0;
}

template <int P>
int mg_main(const MgLayout &l, const double *ctr, const double *M, double *L, cudaStream_t s) {
    const int shm = (int)sizeof(MGSmem<P>);
    cudaFuncSetAttribute(m2l_dmma<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, shm);
    m2l_dmma<P><<<l.nbmax, (MG<P>::NW + 1) * 32, shm, s>>>(l.pkey[1], l.pval[1], l.ent_start, l.ent_gid, l.bent,
                                                           l.bent_end, l.batch_cells, l.nbmax, l.Dtab, ctr, M, L);
    fmm::note_launch();
    return 0;
}
}  // namespace

extern "C" int fmm_m2l_grouped_bytes(int p, int32_t ncells, int64_t cap_pairs, size_t *host_bytes) {
    if (!host_bytes) { set_error("fmm_m2l_grouped_bytes: null output"); return FMM_ERR_INVALID; }
    if (p < 6 || p > 10) { set_error("fmm_m2l_grouped: order %d outside 6..10", p); return FMM_ERR_INVALID; }
    *host_bytes = mg_layout(p, ncells, cap_pairs < 1 ? 1 : cap_pairs, nullptr, 0, nullptr);
    return FMM_OK;
}

extern "C" int fmm_m2l_grouped(int p, int32_t ncells, const int64_t *rows, const int32_t *src, int64_t cap_pairs,
                               const int8_t *level, const uint64_t *cell_key, const double *ctr, const double *root,
                               const double *M, double *L, void *ws, size_t ws_bytes, void *stream) {
    if (p < 6 || p > 10) { set_error("fmm_m2l_grouped: order %d outside 6..10", p); return FMM_ERR_INVALID; }
    if (cap_pairs < 1) cap_pairs = 1;
    if (ncells >= (1 << 30)) { set_error("fmm_m2l_grouped: %d cells exceed the 30-bit source field", ncells); return FMM_ERR_INVALID; }
    if (cap_pairs >= (1ll << 31)) { set_error("fmm_m2l_grouped: %lld pairs exceed int32 indexing", (long long)cap_pairs); return FMM_ERR_INVALID; }
    MgLayout l;
    const size_t need = mg_layout(p, ncells, cap_pairs, nullptr, 0, nullptr);
    if (ws_bytes < need || !mg_layout(p, ncells, cap_pairs, ws, ws_bytes, &l)) {
        set_error("fmm_m2l_grouped: workspace of %zu bytes, %zu needed", ws_bytes, need);
        return FMM_ERR_CAPACITY;
    }
    cudaStream_t s = as_stream(stream);
    const int gc = grid_for(ncells, 256, 148 * 8);
    // target batches
    mg_cell_keys<<<gc, 256, 0, s>>>(ncells, rows, level, cell_key, l.ckey[0], l.iota);
    fmm::note_launch();
    size_t tb = l.tmp_bytes;
    cub::DeviceRadixSort::SortPairs(l.tmp, tb, l.ckey[0], l.ckey[1], l.iota, l.scell, (int)ncells, 0, 64, s);
    cudaMemsetAsync(l.seg, 0, 65 * sizeof(int32_t), s);  // seg + ngroups
    cudaMemsetAsync(l.batch_cells, 0xFF, (size_t)l.nbmax * 8 * sizeof(int32_t), s);
    cudaMemsetAsync(l.bent, 0, (size_t)l.nbmax * sizeof(int32_t), s);
    cudaMemsetAsync(l.bent_end, 0, (size_t)l.nbmax * sizeof(int32_t), s);
    cudaMemsetAsync(l.htab, 0, sizeof(unsigned long long) << kMgHashBits, s);
    mg_level_segments<<<gc, 256, 0, s>>>(ncells, l.ckey[1], l.seg);
    fmm::note_launch();
    mg_assign<<<gc, 256, 0, s>>>(ncells, l.ckey[1], l.scell, l.seg, l.cell_tag, l.batch_cells);
    fmm::note_launch();
    // pair keys, the D-key table and its rows
    mg_pair_keys<<<grid_for((int64_t)ncells * 32, 256, 148 * 16), 256, 0, s>>>(
        ncells, rows, src, level, ctr, root, l.cell_tag, cap_pairs, l.htab, l.pkey[0], l.pval[0]);
    fmm::note_launch();
    switch (p) {
        case 6: mg_launch<6>(l, root, ctr, M, L, s); break;
        case 7: mg_launch<7>(l, root, ctr, M, L, s); break;
        case 8: mg_launch<8>(l, root, ctr, M, L, s); break;
        case 9: mg_launch<9>(l, root, ctr, M, L, s); break;
        default: mg_launch<10>(l, root, ctr, M, L, s); break;
    }
    // (batch, group, slot) order, group entries, batch ranges
    tb = l.tmp_bytes;
    cub::DeviceRadixSort::SortPairs(l.tmp, tb, l.pkey[0], l.pkey[1], l.pval[0], l.pval[1], cap_pairs, 0, l.end_bit,
                                    s);
    const int gp = grid_for(cap_pairs, 256, 148 * 16);
    mg_entry_flags<<<gp, 256, 0, s>>>(rows, ncells, cap_pairs, l.pkey[1], l.flag);
    fmm::note_launch();
    tb = l.tmp_bytes;
    cub::DeviceScan::ExclusiveSum(l.tmp, tb, l.flag, l.eidx, cap_pairs, s);
    mg_entries<<<gp, 256, 0, s>>>(rows, ncells, l.pkey[1], l.flag, l.eidx, level, l.batch_cells, l.htab, l.hid,
                                  l.ent_start, l.ent_gid, l.bent, l.bent_end);
    fmm::note_launch();
    switch (p) {
        case 6: mg_main<6>(l, ctr, M, L, s); break;
        case 7: mg_main<7>(l, ctr, M, L, s); break;
        case 8: mg_main<8>(l, ctr, M, L, s); break;
        case 9: mg_main<9>(l, ctr, M, L, s); break;
        default: mg_main<10>(l, ctr, M, L, s); break;
    }
    FMM_CUDA_CHECK("fmm_m2l_grouped");
    return FMM_OK;
}
