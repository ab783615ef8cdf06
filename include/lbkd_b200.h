/*
 * lbkd_b200.h -- C ABI of the B200-native left-balanced k-d tree builder
 * (arXiv 2211.00120).  Plain pointers and sizes only; every pointer named
 * d_* is a device pointer on the context's device; `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream).
 *
 * Each entry point replaces one interface of the reference package `lbkd`
 * (/root/reference/pkg/src/lbkd):
 *
 *   lbkd_build_rr        builder.build_round_robin       builder.py:200-236
 *   lbkd_build_widest    widest.build_widest             widest.py:134-191
 *   lbkd_update_tags_rr  kernels_*.update_tags_round_robin
 *                        (accel plugin seam)             kernels_numba.py:21-46,
 *                                                        accel.py:48-58
 *   lbkd_update_tags_widest  kernels_*.update_tags_widest kernels_numba.py:49-110
 *   lbkd_num_levels      treemath.num_levels             treemath.py:57-61
 *   lbkd_strerror        the ValueError texts of ingest  builder.py:117-141,
 *                        and the widest capacity check   widest.py:147-156
 *
 * Output contract of the build calls (KdTree, builder.py:26-60):
 *   d_points_out[s*k + c]  coordinate c of the point stored at node s
 *                          (level order, children of s at 2s+1, 2s+2)
 *   d_perm[s]              input row of that point (KdTree.payload for the
 *                          default arange payload); may be NULL
 *   d_split_dims[s]        widest only: split dimension of node s
 * The permutation is bit-identical to the reference's on the same float32
 * input, ties included (stable w.r.t. current order, -0.0 == +0.0).
 * d_points_out may alias d_points (in-place reordering, as in the paper).
 *
 * Threading: a context is used by one host thread at a time; work is
 * enqueued on `stream`.  The build calls end with one stream
 * synchronisation to read back the non-finite flag (disable with
 * lbkd_set_check(ctx, 0) to keep a build fully asynchronous).  A build
 * whose input holds a NaN or +-inf stops on the device right after its
 * input pass (every later kernel returns at once) and reports
 * LBKD_ENONFINITE; its outputs are then undefined.
 */
#ifndef LBKD_B200_H
#define LBKD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum lbkd_status {
    LBKD_OK = 0,
    LBKD_EINVAL_SHAPE = 1,   /* k < 1, k > LBKD_MAX_K, n < 0, bad pointers */
    LBKD_ENONFINITE = 2,     /* a coordinate is NaN or +-inf (builder.py:134-135) */
    LBKD_ECAPACITY = 3,      /* n > 2^31-1, or n << dim_bits > 2^31-1 (widest) */
    LBKD_ECUDA = 4,          /* CUDA runtime error (see lbkd_last_cuda_error) */
    LBKD_ENOPEER = 5,        /* multi-device: no peer access */
    LBKD_ENOMEM = 6,         /* device allocation failed */
    LBKD_EUNSUPPORTED = 7    /* e.g. trace requested for a multi-CTA build */
};

#define LBKD_MAX_K 16

typedef struct lbkd_ctx lbkd_ctx;

int lbkd_create(lbkd_ctx **out, int device);
void lbkd_destroy(lbkd_ctx *ctx);
void lbkd_set_check(lbkd_ctx *ctx, int check_nonfinite);

/* builder.build_round_robin(points, k) -- builder.py:200-236 */
int lbkd_build_rr(lbkd_ctx *ctx, const float *d_points, float *d_points_out, int64_t n, int k,
                  uint32_t *d_perm, void *stream);

/* widest.build_widest(points, k) -- widest.py:134-191 */
int lbkd_build_widest(lbkd_ctx *ctx, const float *d_points, float *d_points_out, int64_t n, int k,
                      uint32_t *d_perm, uint8_t *d_split_dims, void *stream);

/* float64 input -- the reference's own coordinate dtype (ingest promotes
 * every input to float64, builder.py:131-133).  Same contract as
 * lbkd_build_rr / lbkd_build_widest with n x k float64 rows in and out; the
 * permutation and split dims are bit-identical to the reference's on the
 * same float64 input.  The device computes each dimension's dense ranks
 * (-0.0 == +0.0), builds on the rank codes and gathers the float64 rows;
 * widest widths are float64 differences of the original values.  Ends with
 * k + 1 stream synchronisations (distinct-value counts, non-finite flag). */
int lbkd_build_rr_f64(lbkd_ctx *ctx, const double *d_points, double *d_points_out, int64_t n, int k,
                      uint32_t *d_perm, void *stream);
int lbkd_build_widest_f64(lbkd_ctx *ctx, const double *d_points, double *d_points_out, int64_t n, int k,
                          uint32_t *d_perm, uint8_t *d_split_dims, void *stream);
int lbkd_build_rr_f64_trace(lbkd_ctx *ctx, const double *d_points, double *d_points_out, int64_t n, int k,
                            uint32_t *d_perm, uint32_t *d_trace, void *stream);
int lbkd_build_widest_f64_trace(lbkd_ctx *ctx, const double *d_points, double *d_points_out, int64_t n, int k,
                                uint32_t *d_perm, uint8_t *d_split_dims, uint32_t *d_trace, void *stream);

/* Round-robin build that also records, for every sort level l, the order of
 * the not-yet-final points after the sort: d_trace[l*n + p] = index (into
 * d_points) of the point at working position p (the reference's array with
 * the finalized prefix cut off).  This is what BuildRecorder(capture=True)
 * needs (builder.py:63-105).  Only for n <= lbkd_single_cta_capacity(k). */
int lbkd_build_rr_trace(lbkd_ctx *ctx, const float *d_points, float *d_points_out, int64_t n, int k,
                        uint32_t *d_perm, uint32_t *d_trace, void *stream);
int lbkd_build_widest_trace(lbkd_ctx *ctx, const float *d_points, float *d_points_out, int64_t n, int k,
                            uint32_t *d_perm, uint8_t *d_split_dims, uint32_t *d_trace, void *stream);

/* Pipelined builds from / to HOST memory (pinned for overlap): the same
 * contract as lbkd_build_rr / lbkd_build_widest with host pointers.  Each
 * call enqueues H2D -> build -> D2H on three internal streams forked from
 * `stream` and returns; consecutive calls overlap (two device buffer sets
 * alternate).  Host buffers of a call must stay untouched until
 * lbkd_host_join, which makes `stream` wait for every outstanding call and,
 * with sync != 0, waits on the host and returns LBKD_ENONFINITE if any input
 * since the last join held a NaN or infinity. */
int lbkd_build_rr_host(lbkd_ctx *ctx, const float *h_points, float *h_points_out, int64_t n, int k,
                       uint32_t *h_perm, void *stream);
int lbkd_build_widest_host(lbkd_ctx *ctx, const float *h_points, float *h_points_out, int64_t n, int k,
                           uint32_t *h_perm, uint8_t *h_split_dims, void *stream);
int lbkd_host_join(lbkd_ctx *ctx, void *stream, int sync);

/* Multi-device sharding (no reference counterpart -- the
 * reference is single-process).  After the top `top_levels` levels the
 * 2^top_levels subtrees are independent:
 *  - lbkd_build_rr_top: on the device holding the input, build levels
 *    0..top_levels-1 (nodes written to d_out/d_perm at their global slots) and
 *    pack subtree j's points into d_sub: array c (c < k: coordinate c as
 *    float bits, c == k: input row) at d_sub + c*sub_stride + off_j, where
 *    off_j = segment_begin(F(top)+j) - F(top) (treemath.py:108-126), in the
 *    order the reference's sort leaves them (needed for its tie-break).
 *  - lbkd_build_rr_sub: on any device, finish the subtree rooted at
 *    (root_level, root_index) of an n_total-point tree from its packed
 *    points; nodes land at their global level-order slots of the full-size
 *    d_out / d_perm.  When sub_stride is a multiple of 4 and d_sub is 16-byte
 *    aligned, d_sub itself is the working set (no copy; its contents are
 *    undefined afterwards).
 * Results are bit-identical to lbkd_build_rr. */
int lbkd_build_rr_top(lbkd_ctx *ctx, const float *d_points, int64_t n, int k, int top_levels, float *d_out,
                      uint32_t *d_perm, uint32_t *d_sub, int64_t sub_stride, void *stream);
int lbkd_build_rr_sub(lbkd_ctx *ctx, uint32_t *d_sub, int64_t sub_stride, int64_t n_total, int k,
                      int root_level, int64_t root_index, float *d_out, uint32_t *d_perm, void *stream);
/* Recursive halving of the top levels (multigpu.py): build ONE level of the
 * subtree rooted at (root_level, root_index) -- from the raw points d_points
 * (n_total x k float32) at the root (d_sub unused; stride must then be
 * ceil4(n_total)), else from its packed points d_sub (layout of
 * lbkd_build_rr_top, `stride` words between the k + 1 arrays), which is read
 * in place.  d_next (same stride) receives the next level's working set in
 * in-order layout: the left child's points at [0, subtree_size(2s+1)), one
 * unused slot (the node), then the right child's points -- each child ready
 * to be split again or finished with lbkd_build_rr_sub, without copies.
 * stride: a multiple of 4 >= the subtree size; d_sub / d_next 16-byte
 * aligned.  The node goes to d_out / d_perm. */
int lbkd_build_rr_split(lbkd_ctx *ctx, const float *d_points, uint32_t *d_sub, int64_t stride, int64_t n_total,
                        int k, int root_level, int64_t root_index, float *d_out, uint32_t *d_perm,
                        uint32_t *d_next, void *stream);

/* The accel plugin seam (accel.py:48-58): in-place tag refinement. */
int lbkd_update_tags_rr(uint32_t *d_tags, int64_t n, int levels, int l, void *stream);
int lbkd_update_tags_widest(uint32_t *d_tags, const double *d_coords, int k, uint8_t *d_split_dims,
                            const double *d_world_lo, const double *d_world_hi, int64_t n, int levels,
                            int l, int dim_bits, void *stream);

int lbkd_num_levels(int64_t n);
int64_t lbkd_single_cta_capacity(int k, int widest);
/* Geometry chosen for (n, k, mode): subtree bits b (M = 2^b - 1 points per
 * CTA), first in-CTA level lam0, number of global levels. */
int lbkd_plan_info(int64_t n, int k, int widest, int *b, int *lam0);
/* Kernel launches enqueued by the last build on this context. */
int64_t lbkd_last_launch_count(const lbkd_ctx *ctx);
/* Profiling: with lbkd_set_profile(ctx, 1) every digit-pass launch of the
 * next builds is bracketed by CUDA events on the build stream and counts the
 * points it reorders; lbkd_profile_read() returns, for the LAST build, the
 * number of digit-pass launches, their summed device time and their
 * algorithmic bytes (each reordered point reads and writes its k coordinates
 * and its index once).  Synchronises on the events. */
void lbkd_set_profile(lbkd_ctx *ctx, int on);
int lbkd_profile_read(lbkd_ctx *ctx, int *n_pass_launches, double *pass_ms, double *pass_bytes);
/* Per kernel class of the last profiled build (cls = -1: all launches):
 * 0 init, 1 hist, 2 pick, 3 filter, 4 select, 5 partition, 6 subtree,
 * 7 sort-path digit pass, 8 other.  Same units as lbkd_profile_read. */
int lbkd_profile_kernel(lbkd_ctx *ctx, int cls, int *n_launches, double *ms, double *bytes);
/* Global-level algorithm: 0 = pivot selection + stable 3-way partition per
 * level (default), 1 = the literal per-level segmented LSD radix sort
 * (onesweep digit passes).  Both are bit-exact; env LBKD_ALGO=sort selects 1
 * at context creation.  lbkd_profile_read reports the partition (0) or the
 * digit pass (1) kernel. */
int lbkd_set_algorithm(lbkd_ctx *ctx, int algo);
int lbkd_get_algorithm(const lbkd_ctx *ctx);
/* Round-robin select path: 1 = the global levels two per partition pass
 * (the second level selected in the first's layout, one 4-way partition;
 * default), 0 = one level per pass.  Env LBKD_PAIR=0 at context creation.
 * Both are bit-exact. */
int lbkd_set_level_pairs(lbkd_ctx *ctx, int on);
/* In-CTA phase (the last levels, one CTA per subtree): -1 = default per
 * split rule (round-robin: presorted chain lists; widest: per-level
 * selection), 0 = presorted lists, 1 = selection.  Env LBKD_SUBTREE=lists|sel
 * at context creation.  Both are bit-exact. */
int lbkd_set_subtree_kernel(lbkd_ctx *ctx, int which);
/* ---- Queries over a built tree -------------------
 * Replace lbkd.kernels_numpy.knn_search / radius_search
 * (/root/reference/pkg/src/lbkd/kernels_numpy.py:114-196 and :199-245; the
 * plugin seam accel.get_kernels(), accel.py:48-58) for a BATCH of queries;
 * the reference answers one query per call.  All pointers are device
 * pointers.  d_tree: the build's level-order output, n x k float32 rows;
 * d_split_dims: u8[n] of a widest tree, or NULL for round-robin (dim =
 * level(s) mod k).  d_queries: nq x k float64.  Distances are float64 squared
 * euclidean, bit-identical to the reference's (same accumulation order, no
 * FMA contraction).
 *
 * lbkd_knn: for every query the min(m, n) = m nearest nodes (1 <= m <= n)
 * ordered by (dist2, node index), into row q of d_out_idx / d_out_d2 (nq x m,
 * int64 / float64) -- queries.knn (queries.py:41-62) per row. */
int lbkd_knn(const float *d_tree, int64_t n, int k, const uint8_t *d_split_dims, const double *d_queries,
             int64_t nq, int m, int64_t *d_out_idx, double *d_out_d2, void *stream);
/* Radius search in two calls (queries.radius_query, queries.py:65-77):
 * lbkd_radius_count writes per-query hit counts (dist2 <= r2, boundary
 * included) to d_counts[nq] and their exclusive prefix sums to
 * d_offsets[nq + 1] (d_offsets[nq] = total hits); d_scratch holds
 * lbkd_radius_scratch_len(nq) int64.  After sizing d_out_idx to the total,
 * lbkd_radius_fill writes every query's hits to d_out_idx[d_offsets[q] ..
 * d_offsets[q + 1]) sorted ascending. */
int lbkd_radius_count(const float *d_tree, int64_t n, int k, const uint8_t *d_split_dims, const double *d_queries,
                      int64_t nq, double r2, int64_t *d_counts, int64_t *d_offsets, int64_t *d_scratch,
                      void *stream);
int64_t lbkd_radius_scratch_len(int64_t nq);
int lbkd_radius_fill(const float *d_tree, int64_t n, int k, const uint8_t *d_split_dims, const double *d_queries,
                     int64_t nq, double r2, const int64_t *d_offsets, int64_t *d_out_idx, void *stream);
/* ---- Validation over a built tree ---------------
 * lbkd_check_valid replaces verify.check_valid (verify.py:195-245): every node
 * against every ancestor's split plane, closed on both sides.  Writes
 * d_witness[3] = {descendant, ancestor, dim} of the first violation (lowest
 * descendant, then nearest ancestor) or {-1, -1, -1} for a valid tree;
 * d_scratch: one uint64.  lbkd_subtree_boxes replaces
 * verify.brute_subtree_boxes (verify.py:347-374): d_lo / d_hi (n x k
 * float64) = world bounds clipped by every ancestor plane (a zero extreme of
 * the world bounds is reported as +0.0). */
int lbkd_check_valid(const float *d_tree, int64_t n, int k, const uint8_t *d_split_dims, int64_t *d_witness,
                     uint64_t *d_scratch, void *stream);
int lbkd_subtree_boxes(const float *d_tree, int64_t n, int k, const uint8_t *d_split_dims, double *d_lo,
                       double *d_hi, void *stream);
/* The same four calls on float64 level-order rows (trees built from float64
 * input by lbkd_build_*_f64). */
int lbkd_knn_f64(const double *d_tree, int64_t n, int k, const uint8_t *d_split_dims, const double *d_queries,
                 int64_t nq, int m, int64_t *d_out_idx, double *d_out_d2, void *stream);
int lbkd_radius_count_f64(const double *d_tree, int64_t n, int k, const uint8_t *d_split_dims,
                          const double *d_queries, int64_t nq, double r2, int64_t *d_counts, int64_t *d_offsets,
                          int64_t *d_scratch, void *stream);
int lbkd_radius_fill_f64(const double *d_tree, int64_t n, int k, const uint8_t *d_split_dims,
                         const double *d_queries, int64_t nq, double r2, const int64_t *d_offsets,
                         int64_t *d_out_idx, void *stream);
int lbkd_check_valid_f64(const double *d_tree, int64_t n, int k, const uint8_t *d_split_dims, int64_t *d_witness,
                         uint64_t *d_scratch, void *stream);
int lbkd_subtree_boxes_f64(const double *d_tree, int64_t n, int k, const uint8_t *d_split_dims, double *d_lo,
                           double *d_hi, void *stream);
const char *lbkd_strerror(int code);
const char *lbkd_last_cuda_error(void);

#ifdef __cplusplus
}
#endif
#endif
