/*
 * fmm_b200.h -- C ABI of libfmm_b200.so, the B200 (sm_100a) Laplace FMM
 * hot path: Morton-key tree build, vertical passes, dual-tree traversal to
 * CSR lists, M2L and P2P.
 *
 * Conventions (mirroring the reference's numba-core seam):
 *  - every pointer is a DEVICE pointer (cudaMalloc / torch.Tensor.data_ptr())
 *    unless named host_*; outputs are preallocated by the caller and filled
 *    or accumulated in place;
 *  - the library allocates nothing persistent; scratch space is a
 *    caller-owned workspace whose size is obtained from a *_workspace_bytes
 *    query;
 *  - the last argument is the cudaStream_t (as void*); calls are
 *    asynchronous on that stream unless they return counts through host_*
 *    pointers (those synchronise the stream);
 *  - return value: FMM_OK, or an error code.  FMM_ERR_CAPACITY means an
 *    output array was too small; the exact required size is returned through
 *    the documented out-parameter and the call may be repeated with bigger
 *    buffers (the reference's grow-and-retry contract, src/tree.py:400-418,
 *    src/traversal.py:806-828).  FMM_ERR_MAX_DEPTH mirrors the reference's
 *    "max depth exceeded" ValueError (src/tree.py:419-423).
 *
 * Index widths: bodies and cells are int32 (N < 2^31), keys uint64.
 * Reference paths: src/ = fmmkit/ (/root/reference/pkg/src/fmmkit/).
 */
#ifndef FMM_B200_H
#define FMM_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FMM_API __attribute__((visibility("default")))
#else
#define FMM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define FMM_OK 0
#define FMM_ERR_CAPACITY 1
#define FMM_ERR_MAX_DEPTH 2
#define FMM_ERR_INVALID 3
#define FMM_ERR_CUDA 4

#define FMM_DTYPE_F64 0
#define FMM_DTYPE_F32 1

#define FMM_PREC_FP64 0
#define FMM_PREC_FP32 1
/* FP32 near field on offsets from a per-row anchor, with sources split
 * into float32 hi + lo parts: for float64 inputs that float32 cannot
 * represent (tight clusters), keeps dx accurate to the leaf scale. */
#define FMM_PREC_FP32_ANCHORED 2
/* FP32 pair terms summed in float64: the lanes' float32 partials are folded
 * into float64 every few source chunks, so the near field's error floor is
 * ~1e-7 relative instead of the ~5e-7 of long float32 sums (float32-exact
 * inputs only; no guarded redo: a non-finite sum is redone in FP64). */
#define FMM_PREC_FP32_ACC64 3

FMM_API int fmm_abi_version(void);
/* Message of the last error on the calling thread ("" when none). */
FMM_API const char *fmm_last_error(void);
/* Kernels launched by this library so far (its own kernels; CUB's internal
 * sort/scan kernels are not counted). */
FMM_API long long fmm_launch_count(void);
/* Number of SMs of the current device (grid sizing). */
FMM_API int fmm_device_sm_count(void);

/* ---- tree build (replaces src/tree.py:370-454 and src/geometry.py:134-206) */

/* Scratch bytes needed by every call below for n bodies (or cells/pairs). */
FMM_API int fmm_workspace_bytes(int64_t n, size_t *host_bytes);

/* Upcast x,y,z,q (FMM_DTYPE_*) into float64 SoA and compute the root cube
 * (compute_bounds + cubic root, src/geometry.py:200-206, src/tree.py:387-392).
 * root[8] = {lo0, lo1, lo2, size, inv_h, hi0, hi1, hi2} on the device. */
FMM_API int fmm_ingest_bounds(const void *x, const void *y, const void *z, const void *q, int dtype,
                      int64_t n, double *x64, double *y64, double *z64, double *q64, double *root,
                      void *ws, size_t ws_bytes, void *stream);

/* Depth-21 Morton keys (src/geometry.py:134-161) and iota values. */
FMM_API int fmm_morton_keys(const double *x, const double *y, const double *z, int64_t n, const double *root,
                    uint64_t *keys, int32_t *iota, void *stream);

/* Stable radix sort of (key, value) pairs over key bits [0, end_bit)
 * (np.argsort(kind="stable"), src/tree.py:395). */
FMM_API int fmm_sort_pairs_u64(const uint64_t *keys_in, const int32_t *vals_in, uint64_t *keys_out,
                       int32_t *vals_out, int64_t n, int end_bit, void *ws, size_t ws_bytes,
                       void *stream);

/* Gather bodies into Morton order: float64 SoA plus a float4 (x,y,z,q)
 * copy for the FP32 P2P path (src/tree.py:396-398) and its float4
 * residual (x - fp32(x), ...); dev_inexact[0] is set when any residual
 * is non-zero (inputs not representable in float32). */
FMM_API int fmm_permute_bodies(const int32_t *perm, const double *x, const double *y, const double *z,
                       const double *q, int64_t n, double *xs, double *ys, double *zs, double *qs,
                       void *b32, void *b32lo, int *dev_inexact, void *stream);

/* Single-pass carve, step 1 (replaces the fmm_build_level loop): per body,
 * its leaf level and the number of cells it starts; cbase = exclusive scan
 * of those counts = pre-order id of the first cell starting at that body.
 * host_level_hist[23] receives cells per level 0..21 and, in slot 22, the
 * number of leaves; host_ncells the total; host_flag (optional) a copy of
 * the device int *dev_flag read in the same transfer (the build passes
 * fmm_permute_bodies' float32-inexact flag).  Synchronises once, with one
 * pinned copy.  FMM_ERR_MAX_DEPTH when a depth-21 cell holds more than
 * ncrit bodies and !allow_big (src/tree.py:419-423). */
FMM_API int fmm_carve_count(const uint64_t *keys, int64_t n, int32_t ncrit, int allow_big, int32_t *cbase,
                    int8_t *leaf_level, int32_t *host_level_hist, int32_t *host_ncells, const int32_t *dev_flag,
                    int32_t *host_flag, void *ws, size_t ws_bytes, void *stream);

/* Single-pass carve, step 2: writes every cell array in the reference's
 * pre-order (children by octant, -1 when empty), cells_by_level grouped by
 * level using host_level_off[23] (exclusive offsets from the histogram),
 * and the per-body leaf index. */
FMM_API int fmm_carve_emit(const uint64_t *keys, int64_t n, const int32_t *cbase, const int8_t *leaf_level,
                   int32_t ncells, const int32_t *host_level_off, int32_t *children, int32_t *parent,
                   int8_t *level, uint64_t *key, int32_t *start, int32_t *end, int32_t *sub_end, uint8_t *leaf,
                   int32_t *cells_by_level, int32_t *body_leaf, void *ws, size_t ws_bytes, void *stream);

/* Cubic/geometric cell geometry, bit-exact (src/tree.py:80-160). */
FMM_API int fmm_cell_geometry(int32_t ncells, const int8_t *level, const uint64_t *key, const int32_t *start,
                      const int32_t *end, const double *xs, const double *ys, const double *zs,
                      const double *qs, int rect, int com, const double *root, double *lo, double *hi,
                      double *ctr, double *bmax, double *rmax, void *ws, size_t ws_bytes, void *stream);

/* bmax over the bodies in [body_lo, body_hi) only (0 for cells without
 * any): a rank of a sharded build holds just its own bodies, and the
 * ranks' values are combined with a MAX all-reduce -- max and sqrt
 * commute, so the result equals fmm_cell_geometry's bit for bit. */
FMM_API int fmm_cell_bmax_range(int32_t ncells, const int32_t *start, const int32_t *end, const double *ctr,
                        const double *xs, const double *ys, const double *zs, int32_t body_lo, int32_t body_hi,
                        double *bmax, void *ws, size_t ws_bytes, void *stream);

/* ---- vertical passes (src/tree.py:163-189, src/_taylor.py:102-269) ------ */

/* P2M at every listed leaf, then M2M bottom-up level by level over the
 * listed internal cells (their M rows must be zero on entry).
 * cells_by_level lists pre-order cell ids grouped by level;
 * host_level_off[L]..host_level_off[L+1] is level L (host array, nlev+1).
 * Passing every cell gives the reference's upward pass; a multi-GPU rank
 * passes the cells it owns, then the shared top cells. */
FMM_API int fmm_upward(int p, int32_t ncells, const int32_t *children, const int32_t *start, const int32_t *end,
               const uint8_t *leaf, const double *ctr, const double *xs, const double *ys,
               const double *zs, const double *qs, const int32_t *cells_by_level,
               const int32_t *host_level_off, int nlev, double *M, void *stream);

/* L2L top-down over the listed cells, then L2P for bodies [body_lo,
 * body_hi); phi/f are ACCUMULATED (f -= grad). */
FMM_API int fmm_downward(int p, int32_t ncells, const int32_t *parent, const uint8_t *leaf, const double *ctr,
                 const int32_t *cells_by_level, const int32_t *host_level_off, int nlev,
                 int64_t body_lo, int64_t body_hi, const int32_t *body_leaf, const double *xs, const double *ys,
                 const double *zs, double *L, double *phi, double *fx, double *fy, double *fz,
                 void *stream);

/* ---- dual traversal (src/traversal.py:144-262, directed, MAC "fmm") ---- */

/* One breadth-first step over frontier pairs (fa[k], fb[k]), each a pair
 * known to split (classify_self = 1 classifies the frontier pairs
 * themselves instead -- used for the root pair).  The children pairs are
 * classified on the spot: P2P and M2L pairs are appended to their lists,
 * pairs that split again to the next frontier; counters live in
 * dev_counts[3] = {n_p2p, n_m2l, n_next} and keep counting past capacity.
 * kind: MAC kind code (0 bh, 1 bmax, 2 fmm; src/mac.py:21-22); th2 = theta*theta
 * computed by the caller exactly as the reference.  Pairs whose target
 * cell's body range misses [body_lo, body_hi) are dropped (a multi-GPU rank
 * keeps only its own targets; [0, n) keeps everything).  With
 * m2l_owner_only, an M2L pair is emitted only if its target's FIRST body
 * lies in [body_lo, body_hi), so chunks of one GPU's targets, cut on leaf
 * boundaries, partition the M2L list as well as the P2P list. */
FMM_API int fmm_traverse_step(const int32_t *fa, const int32_t *fb, int64_t nfront, int classify_self,
                      const int32_t *children,
                      const uint8_t *leaf, const double *ctr, const double *bmax, const double *rmax,
                      const int32_t *children_b, const uint8_t *leaf_b, const double *ctr_b, const double *bmax_b,
                      const double *rmax_b,
                      const int32_t *start, const int32_t *end, int32_t body_lo, int32_t body_hi,
                      int m2l_owner_only, int kind, double th2, int32_t *p2p_t, int32_t *p2p_s, int64_t cap_p2p,
                      int32_t *m2l_t,
                      int32_t *m2l_s, int64_t cap_m2l, int32_t *na, int32_t *nb, int64_t cap_next,
                      unsigned long long *dev_counts, void *stream);

/* The whole traversal without host round trips: nsteps breadth-first steps
 * chained on the device (each step reads its frontier size from the
 * previous one), frontiers ping-ponging between buffers 0 and 1 (capacity
 * cap_front each).  dev_log (nsteps + 3 entries) receives {n_p2p, n_m2l,
 * frontier size entering step 0, 1, ..., nsteps}; the caller reads it once:
 * a non-zero last entry means nsteps was too small, and any count above its
 * capacity means buffers must grow (the lists are then incomplete; rerun).
 * tmask (optional, one byte per target cell) keeps only pairs whose target
 * cell is flagged: a sampled evaluation flags the cells holding the sample
 * bodies (leaves and their ancestors), and every kept target's row is the
 * same as in the full lists. */
FMM_API int fmm_traverse(int32_t *front_a0, int32_t *front_b0, int32_t *front_a1, int32_t *front_b1,
                 int64_t cap_front, int nsteps, const int32_t *children, const uint8_t *leaf,
                 const double *ctr, const double *bmax, const double *rmax, const int32_t *children_b,
                 const uint8_t *leaf_b, const double *ctr_b, const double *bmax_b, const double *rmax_b,
                 const int32_t *start,
                 const int32_t *end, int32_t body_lo, int32_t body_hi, const uint8_t *tmask, int m2l_owner_only,
                 int kind,
                 double th2, int32_t *p2p_t, int32_t *p2p_s, int64_t cap_p2p, int32_t *m2l_t, int32_t *m2l_s,
                 int64_t cap_m2l, unsigned long long *dev_log, void *stream);

/* Partition owners of the mutual traversal (replaces _partition_roots +
 * _owner_map, src/traversal.py:621-640): owner[c] = the partition root
 * (maximal subtree with < grain bodies, leaves included) holding cell c,
 * -1 above the partition.  grain >= 1 (EvalConfig.task_grain). */
/* One rank's share of the tree for the Morton-partitioned evaluation
 * (paper_1209_3516_b200/distributed.py; the reference's target ownership,
 * src/traversal.py:19-26, :621-639): body cuts on leaf boundaries (cut r =
 * the start of the leaf holding body r*n/world, made non-decreasing), the
 * cells whose first body lies in each rank's range (chunks), and the
 * level-grouped lists of this rank's own cells (body range inside its own)
 * and of the cells straddling an interior cut, in cells_by_level order.
 * host_out (2*(world+1) + 96 int64) receives {cuts[world+1], chunks[world+1],
 * counts[3][32]} (counts by (own, shared, other) x level) in ONE copy; the
 * call synchronises.  own_cells / shared_cells hold ncells each. */
FMM_API int fmm_partition_plan(int32_t ncells, int64_t n, int world, int rank, const int32_t *start,
                       const int32_t *end, const int32_t *body_leaf, const int32_t *cells_by_level,
                       const int8_t *level, int32_t *own_cells, int32_t *shared_cells, int64_t *host_out,
                       void *ws, size_t ws_bytes, void *stream);

FMM_API int fmm_partition_owner(int32_t ncells, const int32_t *parent, const uint8_t *leaf, const int32_t *start,
                        const int32_t *end, int64_t grain, int32_t *owner, void *stream);

/* Mutual dual traversal (replaces _dual_driver + _collect_units with mutual
 * units, src/traversal.py:159-262, :704-791, and their retries): from the
 * mutual root pair, a mutual pair straddling two owners is demoted to the
 * directed pairs (a, b) and (b, a); pairs are classified with the unit
 * rules (MAC in both directions when mutual; a mutual self pair splits
 * into (ci, ci) and (ci, cj), i < j).  The lists are written DIRECTED:
 * a mutual entry (a, b) as (a, b) and, for a != b, (b, a) (the reference's
 * trace expansion), for the directed M2L/P2P executors; only targets whose
 * bodies meet [body_lo, body_hi).  Frontier and dev_log as fmm_traverse
 * (2 * depth + 2 steps suffice). */
FMM_API int fmm_traverse_mutual(int32_t *front_a0, int32_t *front_b0, int32_t *front_a1, int32_t *front_b1,
                        int64_t cap_front, int nsteps, const int32_t *children, const uint8_t *leaf,
                        const double *ctr, const double *bmax, const double *rmax, const int32_t *owner,
                        const int32_t *start, const int32_t *end, int32_t body_lo, int32_t body_hi, int kind,
                        double th2, int32_t *p2p_t, int32_t *p2p_s, int64_t cap_p2p, int32_t *m2l_t,
                        int32_t *m2l_s, int64_t cap_m2l, unsigned long long *dev_log, void *stream);

/* fmm_traverse_mutual keeping mutual entries UNORDERED for the symmetric
 * executors (fmm_p2p_sym, fmm_m2l_sym; the reference's _p2p_mutual /
 * _m2l_mutual, src/_taylor.py:191-217, :410-449): a mutual P2P (M2L) entry
 * of two distinct cells whose bodies both meet [body_lo, body_hi) is written
 * once, as (min, max), to sym_p2p_* (sym_m2l_*) when that list is given
 * (NULL: written directed, as fmm_traverse_mutual); demoted pairs, mutual
 * self pairs and entries with one member outside the range stay directed.
 * dev_sym[0], dev_sym[1] receive the symmetric P2P and M2L counts (grow and
 * rerun when one exceeds its capacity). */
FMM_API int fmm_traverse_mutual_sym(int32_t *front_a0, int32_t *front_b0, int32_t *front_a1, int32_t *front_b1,
                            int64_t cap_front, int nsteps, const int32_t *children, const uint8_t *leaf,
                            const double *ctr, const double *bmax, const double *rmax, const int32_t *owner,
                            const int32_t *start, const int32_t *end, int32_t body_lo, int32_t body_hi, int kind,
                            double th2, int32_t *p2p_t, int32_t *p2p_s, int64_t cap_p2p, int32_t *m2l_t,
                            int32_t *m2l_s, int64_t cap_m2l, unsigned long long *dev_log, int32_t *sym_p2p_a,
                            int32_t *sym_p2p_b, int64_t cap_sym_p2p, int32_t *sym_m2l_a, int32_t *sym_m2l_b,
                            int64_t cap_sym_m2l, unsigned long long *dev_sym, void *stream);

/* Treecode lists (replaces _collect_treecode, src/traversal.py:265-313, with
 * its capacity retry, :944-966): every leaf whose bodies meet
 * [body_lo, body_hi) walks the source tree from the root; a pair (t, c)
 * with the MAC accepted is M2P (tested first), else a leaf c is P2P, else
 * c's children are visited.  Breadth-first, nsteps steps chained on the
 * device (one source level per step; depth + 1 suffice).  Frontier buffers
 * hold cap_front >= ncells pairs each; ws holds ncells bytes plus a CUB
 * select.  dev_log (nsteps + 3 entries) receives {n_p2p, n_m2p, frontier
 * size entering step 0, ..., nsteps}: read it once, grow and rerun on any
 * count above its capacity or a non-zero last entry. */
FMM_API int fmm_treecode_traverse(int32_t *front_a0, int32_t *front_b0, int32_t *front_a1, int32_t *front_b1,
                          int64_t cap_front, int nsteps, int32_t ncells, const int32_t *children,
                          const uint8_t *leaf, const double *ctr, const double *bmax, const double *rmax,
                          const int32_t *children_b, const uint8_t *leaf_b, const double *ctr_b,
                          const double *bmax_b, const double *rmax_b,
                          const int32_t *start, const int32_t *end, int32_t body_lo, int32_t body_hi, int kind,
                          double th2, int32_t *m2p_t, int32_t *m2p_s, int64_t cap_m2p, int32_t *p2p_t,
                          int32_t *p2p_s, int64_t cap_p2p, unsigned long long *dev_log, void *ws,
                          size_t ws_bytes, void *stream);

/* listfmm lists (replaces _collect_vlist / _collect_ulist,
 * src/traversal.py:341-497, with their capacity retry, :1061-1118): the
 * V list (M2L: children of the parent's 3x3x3 neighbourhood not adjacent
 * to the target) of every cell and the U list (P2P: own-level neighbours,
 * or their descendant leaves, plus leaf cells adjacent to a coarser
 * ancestor) of every leaf whose bodies meet [body_lo, body_hi).
 * level_off is a HOST array of the depth + 2 cell-count offsets per level.
 * dev_counts[2] = {n_p2p, n_m2l}, counting past capacity (grow and rerun).
 * ws holds the (level, key) table (~25 B per cell) and a CUB sort. */
FMM_API int fmm_listfmm_lists(int32_t ncells, int depth, const int64_t *level_off, const int8_t *level,
                      const uint64_t *key, const int32_t *parent, const int32_t *children, const uint8_t *leaf,
                      const int32_t *sub_end, const int32_t *start, const int32_t *end,
                      int32_t body_lo, int32_t body_hi, int32_t *m2l_t,
                      int32_t *m2l_s, int64_t cap_m2l, int32_t *p2p_t, int32_t *p2p_s, int64_t cap_p2p,
                      unsigned long long *dev_counts, void *ws, size_t ws_bytes, void *stream);

/* Sort every CSR row's ids ascending (rows of distinct ids, e.g. a grouped
 * interaction list): out[rows[c]..rows[c+1]) = sorted in[...].  One warp
 * per row: a shared-memory bitmap when the row's ids fit one 32768-id
 * window, a register bitonic sort for wider rows of up to 1024 ids.  ws
 * holds fmm_workspace_bytes(ncells + 1). */
FMM_API int fmm_sort_rows(int32_t ncells, const int64_t *rows, const int32_t *in, int32_t *out, void *ws,
                  size_t ws_bytes, void *stream);

/* The same CSR as fmm_pairs_to_csr without a host pair count: *dev_npairs
 * (a traversal's device counter, clamped to cap) pairs are counted per
 * target, scattered, and each row's sources sorted by one CTA (block radix
 * sort; long rows by a larger tile or an in-memory bitonic sort), so a
 * traversal and its CSR chain on the stream with no host round trip.
 * Sources are ids below nsrc (<= 0: ncells).  sort_rows = 0 skips the
 * row sort (rows grouped, order within a row free: fmm_p2p_plan sorts its
 * rows itself).  ws holds
 * fmm_workspace_bytes(max(cap, ncells + 1)). */
FMM_API int fmm_pairs_to_rows(const int32_t *t, const int32_t *s, const unsigned long long *dev_npairs, int64_t cap,
                      int32_t ncells, int32_t nsrc, int sort_rows, int32_t *src_sorted, int64_t *rows, void *ws,
                      size_t ws_bytes, void *stream);

/* Sort (t, s) pairs by target then source and build row offsets over all
 * cells: rows[c]..rows[c+1] are the sources of target c (ascending). */
FMM_API int fmm_pairs_to_csr(const int32_t *t, const int32_t *s, int64_t npairs, int32_t ncells,
                     int32_t *src_sorted, int64_t *rows, void *ws, size_t ws_bytes, void *stream);

/* P2P work decomposition: merge every target-leaf row's Morton-adjacent
 * source leaves into contiguous body runs (ascending) and split off the
 * self leaf.  Rows are the leaves whose bodies lie in [body_lo, body_hi).
 * Input: the P2P list grouped by target (rows[t]..rows[t+1] index src; the
 * order within a row is free -- fmm_pairs_to_rows with sort_rows = 0).
 * One warp per row marks the row's source-leaf ordinals in a bitmap and
 * reads the runs off it (fmm_sort_rows gives the sorted row when wanted).
 * Outputs: the leaf rows (leaf_rows[r] = target leaf, sized ncells),
 * run_rng[2r], run_rng[2r+1] (the row's runs, stored row-locally at the
 * row's own CSR offset, so runs is sized like src: cap_runs >= the pair
 * count), runs as int4 {bstart, bend, self_flag, 0}.  The call never
 * synchronises unless host_nruns / host_nleaf_rows are given; the row
 * count is written to dev_nrows for fmm_p2p.
 * Also computes the reference's pair counters (p2p_pairs, p2p_skipped)
 * into dev_stats[0..1] (src/_taylor.py:366-407 accounting); dev_stats[2]
 * is 0, or -- when a row's runs would pass cap_runs (rows are then left
 * empty) -- the runs capacity required.  With host_nruns the call then
 * returns FMM_ERR_CAPACITY and *host_nruns holds that capacity
 * (grow-and-retry); async callers read dev_stats[2].  keys (the sorted
 * body keys, optional) let leaves without two equal keys skip the
 * coincident-pair scan (coincident bodies share a key); NULL scans all.
 * Cross-tree plans (src_start given, with src_leaf, src_end, src_ncells):
 * the sources are the source tree's leaves, their body runs shifted by
 * src_offset (where the source bodies sit in the P2P body arrays); no self
 * leaf, no coincident scan (see fmm_p2p_coincident).  tmask (optional)
 * plans only the flagged target leaves (as fmm_traverse). */
FMM_API int fmm_p2p_plan(int32_t ncells, const uint8_t *leaf, const int32_t *start, const int32_t *end,
                 int32_t body_lo, int32_t body_hi, const uint8_t *tmask, const int64_t *rows, const int32_t *src,
                 const double *xs, const double *ys, const double *zs,
                 const uint64_t *keys, const uint8_t *src_leaf, int32_t src_ncells, const int32_t *src_start,
                 const int32_t *src_end, int32_t src_offset, int32_t *leaf_rows, int64_t *run_rng, void *runs,
                 int64_t cap_runs,
                 int64_t *host_nruns, int32_t *host_nleaf_rows, int32_t *dev_nrows,
                 unsigned long long *dev_stats, void *ws, size_t ws_bytes, void *stream);

/* ---- executors (src/traversal.py:500-548) ------------------------------ */

/* L[t] += sum over row sources of M2L(M[s], ctr[t]-ctr_src[s]) (src/_taylor.py:169-188).
 * ctr_src and M are the source tree's (a cross-tree evaluation); ctr_src
 * NULL means the same tree. */
FMM_API int fmm_m2l_csr(int p, int32_t ncells, const int64_t *rows, const int32_t *src, const double *ctr,
                const double *ctr_src, const double *M, double *L, void *stream);

/* The same M2L (same tree, cubic cells, geometric centres), evaluated by
 * offset group on the FP64 tensor pipe: pairs sharing (level_t, level_s,
 * lattice offset) share one D tensor, targets are batched 8 per CTA, and
 * each group is one block-triangular matrix product (mma.m8n8k4.f64) over
 * the batch's source moments.  rows/src: the M2L CSR (any order within a
 * row; rows[ncells] is the pair count, read on the device), cap_pairs >=
 * that count (the src buffer's size); level/cell_key: the tree's cell
 * arrays; root: the device root record (root[3] = root size).  Results are
 * deterministic (a radix sort fixes the order) and equal fmm_m2l_csr's to
 * float64 rounding.  6 <= p <= 10.  ws: fmm_m2l_grouped_bytes. */
FMM_API int fmm_m2l_grouped_bytes(int p, int32_t ncells, int64_t cap_pairs, size_t *host_bytes);
FMM_API int fmm_m2l_grouped(int p, int32_t ncells, const int64_t *rows, const int32_t *src, int64_t cap_pairs,
                    const int8_t *level, const uint64_t *cell_key, const double *ctr, const double *root,
                    const double *M, double *L, void *ws, size_t ws_bytes, void *stream);

/* Treecode far field (replaces _exec_m2p, src/traversal.py:520-528 ->
 * _m2p, src/_taylor.py:272-307): for every target leaf row t of the CSR M2P
 * list and every body j of t, phi[j] += sum (-1)^|m| M_m D_m(x_j - c_s) and
 * f[j] -= the gradient terms (f = -grad phi); bodies at a cell center are
 * skipped.  Accumulates (+=) into phi/fx/fy/fz; 1 <= p <= 12.  precision
 * FMM_PREC_FP64 is the reference's arithmetic; FMM_PREC_FP32 (p <= 6; higher
 * orders stay float64) forms D, the moments and each source's contribution in
 * float32 and accumulates them in float64. */
FMM_API int fmm_m2p_csr(int p, int precision, int32_t ncells, const int64_t *rows, const int32_t *src,
                const int32_t *start, const int32_t *end, const double *ctr, const double *M, const double *x, const double *y,
                const double *z, double *phi, double *fx, double *fy, double *fz, void *stream);

/* Near field over the P2P plan.  precision FMM_PREC_FP32 reads the float4
 * body copy b32; FMM_PREC_FP64 reads, when b32 is given, the double4 body
 * copy written by fmm_pack_bodies_f64 (streamed rows, rsqrt.approx.f64 +
 * Newton), else the float64 SoA.  Results are STORED
 * (not accumulated) into phi/fx/fy/fz for every body of a planned leaf row.
 * use_rsqrt (FP64 only) mirrors src/_taylor.py:318-323.
 * nrows bounds the grid; when dev_nrows is given the kernels stop at the
 * device-side row count (written by fmm_p2p_plan) -- no host round trip.
 * dev_flag[0] is set when a non-finite sum was produced (FP32 collision of
 * distinct bodies); the caller reruns with safe=1.
 * cross: the sources are another tree's bodies (src/traversal.py:552-597),
 * appended after the targets in the body arrays (the plan's runs point
 * there): the target leaf's own bodies are then not swept as sources. */
FMM_API int fmm_p2p(int precision, int safe, int use_rsqrt, int cross, int32_t nrows, const int32_t *dev_nrows,
            const int32_t *leaf_rows,
            const int32_t *start, const int32_t *end, const int64_t *run_rng, const void *runs,
            const double *xs, const double *ys, const double *zs, const double *qs, const void *b32,
            const void *b32lo, double *phi, double *fx, double *fy, double *fz, int *dev_flag, void *stream);

/* Symmetric near field over UNORDERED leaf pairs (replaces _p2p_mutual,
 * src/_taylor.py:410-449: one 1/r per body pair, added to both bodies; the
 * reference's mutual self pair, :452-493, stays the directed kernel's
 * guarded self run).  rows_a/src_a: CSR of the pairs (a, b) by first leaf,
 * each row ascending; rows_b/src_b: the same pairs by second leaf, ascending
 * first leaves; slot_off[k] = the first reaction slot of pair k of src_a
 * (one slot per body of src_a[k]; exclusive prefix sums).  Only first leaves
 * in [a_lo, a_hi) are evaluated, their slots addressed relative to
 * slot_base, so a caller can bound react (float4 / double4 per slot) and
 * sweep the rows in chunks.  The pair kernel ADDS the first members' sums
 * to phi/fx/fy/fz and stores the second members' sums in react; a second
 * kernel adds each leaf's slots in ascending order of the first member:
 * deterministic, no atomics.  precision FMM_PREC_FP32 reads the float4 body
 * copy, FMM_PREC_FP64 the double4 copy (fmm_pack_bodies_f64). */
FMM_API int fmm_p2p_sym(int precision, int32_t ncells, int32_t a_lo, int32_t a_hi, const int64_t *rows_a,
                const int32_t *src_a, const int64_t *rows_b, const int32_t *src_b, const int64_t *slot_off,
                int64_t slot_base, const int32_t *start, const int32_t *end, const void *bodies4, void *react,
                double *phi, double *fx, double *fy, double *fz, void *stream);

/* Symmetric M2L over UNORDERED cell pairs (replaces _m2l_mutual,
 * src/_taylor.py:191-217: one derivative tensor D(c_a - c_b) per pair,
 * contracted in both directions through D_k(-r) = (-1)^|k| D_k(r)).
 * rows_a/src_a: CSR of the pairs (a, b) by first member, each row ascending;
 * rows_b/src_b: the same pairs by second member, ascending first members.
 * Pair k of src_a owns the slot k - slot_base of react (ncoef(p) doubles per
 * slot); only first members in [a_lo, a_hi) are evaluated, so a caller can
 * bound react and sweep the rows in chunks (slot_base = rows_a[a_lo]).  The
 * pair kernel ADDS the first members' sums to L and stores the second
 * members' finished coefficients in react; a second kernel adds each cell's
 * slots in ascending order of the first member: deterministic, no atomics.
 * Orders 1..FMM_M2L_SYM_MAX_P (higher orders: keep the pairs directed, the
 * offset-grouped fmm_m2l_grouped shares D over whole lattice groups). */
#define FMM_M2L_SYM_MAX_P 7
FMM_API int fmm_m2l_sym(int p, int32_t ncells, int32_t a_lo, int32_t a_hi, const int64_t *rows_a,
                const int32_t *src_a, const int64_t *rows_b, const int32_t *src_b, int64_t slot_base,
                const double *ctr, const double *M, double *react, double *L, void *stream);

/* Pack the float64 SoA bodies into the double4 (x, y, z, q) copy the
 * streamed FP64 P2P reads (32 B per body). */
FMM_API int fmm_pack_bodies_f64(int64_t n, const double *xs, const double *ys, const double *zs, const double *qs,
                                void *out, void *stream);

/* Coincident (target, source) pairs of a cross-tree P2P plan (r2 == 0.0 in
 * float64, which the reference skips and counts as p2p_skipped,
 * src/traversal.py:552-597), added into *count. */
FMM_API int fmm_p2p_coincident(int32_t nrows, const int32_t *dev_nrows, const int32_t *leaf_rows,
                       const int32_t *start, const int32_t *end, const int64_t *run_rng, const void *runs,
                       const double *xs, const double *ys, const double *zs, unsigned long long *count,
                       void *stream);

/* Scatter four Morton-ordered arrays back to input order:
 * b_k[perm[i]] = a_k[i] (Tree.results_in_input_order, src/tree.py:344-348). */
FMM_API int fmm_unpermute(const int32_t *perm, int64_t n, const double *a0, const double *a1, const double *a2,
                  const double *a3, double *b0, double *b1, double *b2, double *b3, void *stream);

/* Final combine: out = p2p + far (phi, f) for all n bodies. */
FMM_API int fmm_combine(int64_t n, const double *a_phi, const double *a_fx, const double *a_fy,
                const double *a_fz, double *phi, double *fx, double *fy, double *fz, void *stream);

/* ---- oracle-free utilities --------------------------------------------- */

/* Direct O(S*N) sums onto target indices tidx (src/_taylor.py:496-528). */
FMM_API int fmm_direct(int64_t n, const double *x, const double *y, const double *z, const double *q,
               int64_t nt, const int64_t *tidx, double *phi, double *fx, double *fy, double *fz,
               void *stream);

/* FP32 pipe throughput probe over `blocks` x 256 threads, 16 independent
 * chains per thread, `iters` iterations: mode 0 FFMA (immediate operands),
 * 1 FFMA2 (packed f32x2), 2 FFMA (register operands), 3 FFMA2 (register
 * operands), 4 FMUL/FADD (register operands), 5 the P2P pair math on
 * register sources (20 flops/pair), 6 the same without MUFU.  sink needs blocks*2+2
 * floats (zeroed).  The caller times it with events; host_flops = flops
 * per launch (2 per FMA lane-op, 1 per FMUL/FADD). */
FMM_API int fmm_ffma_probe(int mode, int blocks, int iters, float *sink, double *host_flops, void *stream);

#ifdef __cplusplus
}
#endif
#endif
