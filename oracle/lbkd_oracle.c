/*
 * lbkd_oracle.c -- CPU restatement of the reference tag-and-sort k-d tree
 * build.  TEST INFRASTRUCTURE ONLY: this file is the checker the CUDA path
 * is compared against (tests/, __graft_entry__.smoke(), bench.py's
 * cpu_baseline / --impl reference leg).  Nothing in the product path links
 * or calls it.
 *
 * It restates, phase for phase, the reference package `lbkd`:
 *   build_round_robin   /root/reference/pkg/src/lbkd/builder.py:200-236
 *   sort_phase          /root/reference/pkg/src/lbkd/builder.py:165-181
 *       np.lexsort((coords[:, l % k], tags)) -- an indirect STABLE sort by
 *       (tag, coordinate); restated here as a stable bottom-up merge sort
 *       with the same comparison (float compare, so -0.0 == +0.0 exactly as
 *       numpy compares the float64-promoted values).
 *   update_tags_round_robin  kernels_numpy.py:21-48 / kernels_numba.py:21-46
 *   final_sort          builder.py:194-197 (argsort of a permutation)
 *   build_widest        widest.py:134-191
 *   sort_phase_widest   widest.py:119-131
 *   update_tags_widest  kernels_numpy.py:51-111 / kernels_numba.py:49-110
 *   world_bounds / widest_dim  widest.py:84-93
 *
 * Inputs are float32 AoS points (n x k); the reference promotes to float64,
 * which is exact and order preserving, so comparing the float32 values is
 * the same ordering.  Widths for the widest variant are float64 differences
 * of the promoted values with a first-max argmax (np.argmax semantics).
 *
 * Output: perm[s] = input row of the point stored at node s
 * (KdTree.payload with the default arange payload), and for widest
 * split_dims[s].
 *
 * Parity pin: tests/test_oracle.py checks this file against the golden
 * vectors in tests/golden/ produced by running the reference itself
 * (tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    uint32_t tag;
    float key;
    uint32_t idx;
} rec_t;

static int bit_length_u64(uint64_t v) {
    int b = 0;
    while (v) { b++; v >>= 1; }
    return b;
}

/* treemath.num_levels (treemath.py:57-61) */
int oracle_num_levels(uint64_t n) { return bit_length_u64(n); }

static inline int rec_less(const rec_t *a, const rec_t *b) {
    /* builder.less (builder.py:158-162): tag first, then the coordinate */
    if (a->tag != b->tag) return a->tag < b->tag;
    return a->key < b->key;
}

/* Stable bottom-up merge sort (np.lexsort is documented stable). */
static void stable_sort(rec_t *a, rec_t *tmp, int64_t n) {
    /* insertion sort runs of 32 */
    const int64_t RUN = 32;
    for (int64_t lo = 0; lo < n; lo += RUN) {
        int64_t hi = lo + RUN < n ? lo + RUN : n;
        for (int64_t i = lo + 1; i < hi; i++) {
            rec_t x = a[i];
            int64_t j = i - 1;
            while (j >= lo && rec_less(&x, &a[j])) { a[j + 1] = a[j]; j--; }
            a[j + 1] = x;
        }
    }
    rec_t *src = a, *dst = tmp;
    for (int64_t w = RUN; w < n; w *= 2) {
        for (int64_t lo = 0; lo < n; lo += 2 * w) {
            int64_t mid = lo + w < n ? lo + w : n;
            int64_t hi = lo + 2 * w < n ? lo + 2 * w : n;
            int64_t i = lo, j = mid, o = lo;
            if (mid >= hi || !rec_less(&src[mid], &src[mid - 1])) {
                memcpy(dst + lo, src + lo, (size_t)(hi - lo) * sizeof(rec_t));
                continue;
            }
            while (i < mid && j < hi) {
                /* take from the right only when strictly less: stable */
                if (rec_less(&src[j], &src[i])) dst[o++] = src[j++];
                else dst[o++] = src[i++];
            }
            while (i < mid) dst[o++] = src[i++];
            while (j < hi) dst[o++] = src[j++];
        }
        rec_t *t = src; src = dst; dst = t;
    }
    if (src != a) memcpy(a, src, (size_t)n * sizeof(rec_t));
}

/* kernels_numpy._pivot_positions (kernels_numpy.py:21-38), scalar form */
static inline int64_t pivot_pos(int64_t s, int64_t n, int levels, int l) {
    int shift = levels - l - 1;
    int64_t top = ((int64_t)1 << l) - 1;
    int64_t nls = s - top;
    int64_t bottom_have = n - (((int64_t)1 << (levels - 1)) - 1);
    int64_t low = nls << shift;
    if (low > bottom_have) low = bottom_have;
    int64_t begin = top + nls * (((int64_t)1 << shift) - 1) + low;
    int cshift = shift - 1;
    int64_t first = ((2 * s + 2) << cshift) - 1;
    int64_t on_bottom = n - first;
    int64_t cw = (int64_t)1 << cshift;
    if (on_bottom < 0) on_bottom = 0;
    if (on_bottom > cw) on_bottom = cw;
    return begin + cw - 1 + on_bottom;
}

static int nthreads_used = 1;
int oracle_threads(void) { return nthreads_used; }

/*
 * Round-robin build (builder.py:200-236).  pts: n*k float32 AoS.
 * perm_out[s] = input row at node s.  Returns 0.
 * If trace_tags/trace_idx are non-null they receive, per phase, the tag and
 * index arrays (phase order: init, sort0, update0, ..., final) -- the
 * BuildRecorder(capture=True) sequence (builder.py:219-235); each phase
 * occupies n entries.
 */
int oracle_build_rr(const float *pts, int64_t n, int k, uint32_t *perm_out,
                    uint32_t *trace_tags, uint32_t *trace_idx) {
    if (n <= 0) return 0;
    rec_t *a = (rec_t *)malloc((size_t)n * sizeof(rec_t));
    rec_t *tmp = (rec_t *)malloc((size_t)n * sizeof(rec_t));
    if (!a || !tmp) { free(a); free(tmp); return -1; }
    for (int64_t i = 0; i < n; i++) { a[i].tag = 0; a[i].idx = (uint32_t)i; }
    int phase = 0;
#define TRACE()                                                              \
    do {                                                                     \
        if (trace_tags) {                                                    \
            for (int64_t i_ = 0; i_ < n; i_++) {                             \
                trace_tags[(int64_t)phase * n + i_] = a[i_].tag;             \
                trace_idx[(int64_t)phase * n + i_] = a[i_].idx;              \
            }                                                                \
        }                                                                    \
        phase++;                                                             \
    } while (0)
    TRACE();
    int levels = oracle_num_levels((uint64_t)n);
    for (int l = 0; l < levels - 1; l++) {
        int dim = l % k;
        for (int64_t i = 0; i < n; i++) a[i].key = pts[(int64_t)a[i].idx * k + dim];
        stable_sort(a, tmp, n);                             /* builder.py:178 */
        TRACE();
        int64_t top = ((int64_t)1 << l) - 1;                /* kernels_numba.py:23 */
#pragma omp parallel for schedule(static)
        for (int64_t i = top; i < n; i++) {
            int64_t s = a[i].tag;
            int64_t p = pivot_pos(s, n, levels, l);
            if (i < p) a[i].tag = (uint32_t)(2 * s + 1);
            else if (i > p) a[i].tag = (uint32_t)(2 * s + 2);
        }
        TRACE();
    }
    /* final_sort: tags are a permutation of 0..n-1 (builder.py:194-197) */
    for (int64_t i = 0; i < n; i++) perm_out[a[i].tag] = a[i].idx;
    if (trace_tags) {
        for (int64_t i = 0; i < n; i++) {
            trace_tags[(int64_t)phase * n + i] = (uint32_t)i;
            trace_idx[(int64_t)phase * n + i] = perm_out[i];
        }
    }
#undef TRACE
    free(a);
    free(tmp);
    return 0;
}

/* widest.dim_bits_for (widest.py:66-70) */
int oracle_dim_bits_for(int k) { return bit_length_u64((uint64_t)(k - 1)); }

/*
 * Widest-dimension build (widest.py:134-191, kernels_numba.py:49-110).
 * split_dims_out[s] = split dimension of node s.
 */
int oracle_build_widest(const float *pts, int64_t n, int k, uint32_t *perm_out,
                        uint8_t *split_dims_out) {
    if (n <= 0) return 0;
    int db = oracle_dim_bits_for(k);
    uint32_t mask = (1u << db) - 1u;
    rec_t *a = (rec_t *)malloc((size_t)n * sizeof(rec_t));
    rec_t *tmp = (rec_t *)malloc((size_t)n * sizeof(rec_t));
    double *wlo = (double *)malloc(sizeof(double) * k);
    double *whi = (double *)malloc(sizeof(double) * k);
    if (!a || !tmp || !wlo || !whi) { free(a); free(tmp); free(wlo); free(whi); return -1; }
    /* world_bounds (widest.py:84-88) */
    for (int d = 0; d < k; d++) { wlo[d] = pts[d]; whi[d] = pts[d]; }
    for (int64_t i = 1; i < n; i++)
        for (int d = 0; d < k; d++) {
            double v = pts[i * k + d];
            if (v < wlo[d]) wlo[d] = v;
            if (v > whi[d]) whi[d] = v;
        }
    /* widest_dim: first argmax of f64 widths (widest.py:91-93) */
    int root = 0;
    for (int d = 1; d < k; d++)
        if (whi[d] - wlo[d] > whi[root] - wlo[root]) root = d;
    memset(split_dims_out, 0, (size_t)n);
    for (int64_t i = 0; i < n; i++) { a[i].tag = (uint32_t)root; a[i].idx = (uint32_t)i; }
    int levels = oracle_num_levels((uint64_t)n);
    for (int l = 0; l < levels - 1; l++) {
        /* sort_phase_widest: minor key = own coordinate in the tag's dim */
        for (int64_t i = 0; i < n; i++)
            a[i].key = pts[(int64_t)a[i].idx * k + (a[i].tag & mask)];
        stable_sort(a, tmp, n);
        int64_t top = ((int64_t)1 << l) - 1;
        /* pivot elements first: they record split_dims (kernels_numba.py:75-76);
         * everything else only reads finalized ancestors (< top) and the
         * pivot coordinates, so doing it in two sweeps is equivalent. */
        for (int64_t i = top; i < n; i++) {
            int64_t s = a[i].tag >> db;
            if (pivot_pos(s, n, levels, l) == i) split_dims_out[s] = (uint8_t)(a[i].tag & mask);
        }
#pragma omp parallel
        {
            double lo[64], hi[64];
#pragma omp for schedule(static)
            for (int64_t i = top; i < n; i++) {
                uint32_t packed = a[i].tag;
                int64_t s = packed >> db;
                int d = (int)(packed & mask);
                int64_t p = pivot_pos(s, n, levels, l);
                if (i == p) continue;
                for (int j = 0; j < k; j++) { lo[j] = wlo[j]; hi[j] = whi[j]; }
                double plane = pts[(int64_t)a[p].idx * k + d];
                int64_t child;
                if (i < p) { if (plane < hi[d]) hi[d] = plane; child = 2 * s + 1; }
                else { if (plane > lo[d]) lo[d] = plane; child = 2 * s + 2; }
                int64_t anc = s;
                while (anc > 0) {                               /* kernels_numba.py:91-102 */
                    int64_t q = (anc - 1) >> 1;
                    int dq = split_dims_out[q];
                    double cp = pts[(int64_t)a[q].idx * k + dq];  /* node q sits at position q */
                    if (anc & 1) { if (cp < hi[dq]) hi[dq] = cp; }
                    else { if (cp > lo[dq]) lo[dq] = cp; }
                    anc = q;
                }
                int nd = 0;
                double best = hi[0] - lo[0];
                for (int j = 1; j < k; j++) {
                    double w = hi[j] - lo[j];
                    if (w > best) { best = w; nd = j; }
                }
                a[i].tag = (uint32_t)((child << db) | nd);
            }
        }
    }
    for (int64_t i = 0; i < n; i++) perm_out[a[i].tag >> db] = a[i].idx;
    int64_t bottom = ((int64_t)1 << (levels - 1)) - 1;          /* widest.py:187-190 */
    for (int64_t i = 0; i < n; i++) {
        int64_t s = a[i].tag >> db;
        if (s >= bottom) split_dims_out[s] = (uint8_t)(a[i].tag & mask);
    }
    free(a); free(tmp); free(wlo); free(whi);
    return 0;
}

void oracle_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
    nthreads_used = omp_get_max_threads();
#else
    (void)t;
    nthreads_used = 1;
#endif
}
