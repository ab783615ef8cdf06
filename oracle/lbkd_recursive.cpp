/*
 * lbkd_recursive.cpp -- threaded CPU restatement of the reference's
 * RECURSIVE oracle.  TEST INFRASTRUCTURE ONLY: the checker the CUDA path is
 * compared against (tests/, __graft_entry__.smoke(), bench.py's
 * cpu_baseline / --impl reference leg).  Nothing in the product path links
 * or calls it.
 *
 * It restates verify.reference_build
 *   /root/reference/pkg/src/lbkd/verify.py:121-168
 * ("sorts each subtree's points along its split dimension, places the element
 * whose rank equals the left subtree's size at the node, and recurses"):
 *   place(node, idx, box):
 *     dim  = widest ? widest_dim(box) : level(node) % k        (:141-145)
 *     idx  = idx[argsort(coords[idx, dim], kind="stable")]     (:147)
 *     off  = subtree_size(2 node + 1, n) if 2 node + 1 < n else 0  (:148-149)
 *     node <- idx[off]; recurse left on idx[:off], right on idx[off+1:]
 *     widest: children's boxes = box clipped by the plane     (:153-165)
 * with
 *   treemath.level / subtree_size     treemath.py:46-54, 85-98
 *   widest.world_bounds / widest_dim  widest.py:84-93 (first-max argmax of
 *                                     the float64 widths)
 *
 * The stable argsort is std::stable_sort over records (k coordinates + the
 * input row) with the comparison `a < b` on the coordinate, so -0.0 == +0.0
 * ties keep their current order exactly like numpy's stable sort of the
 * float64-promoted values.  Coordinates are float32 (promotion to float64 is
 * exact and order preserving) or float64 (the reference's own dtype).
 *
 * This is a second oracle, structurally independent of the tag-and-sort
 * restatement in lbkd_oracle.c (the two agree,
 * ties included).  It is the one that scales to N = 1B: subtrees are
 * independent, so after the top levels (sorted with libstdc++'s parallel
 * stable sort) the subtrees run as parallel tasks over the host cores.
 *
 * Parity pin: tests/test_oracle.py checks it against the reference-run
 * golden vectors (tests/golden/) and against lbkd_oracle.c.
 */
#include <parallel/algorithm>
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <omp.h>

namespace {

inline int bit_length(uint64_t v) {
    int b = 0;
    while (v) { ++b; v >>= 1; }
    return b;
}

// treemath.level (treemath.py:46-54)
inline int level_of(uint64_t s) { return bit_length(s + 1) - 1; }

// treemath.subtree_size (treemath.py:85-98)
inline uint64_t subtree_size(uint64_t s, uint64_t n) {
    const int L = bit_length(n);
    const int l = level_of(s);
    const int sh = L - l - 1;
    const uint64_t j = s - ((1ull << l) - 1);
    const uint64_t B = n - ((1ull << (L - 1)) - 1);
    const uint64_t w = 1ull << sh;
    const uint64_t lo = j << sh;
    uint64_t on = B > lo ? B - lo : 0;
    if (on > w) on = w;
    return w - 1 + on;
}

template <typename T, int K>
struct Rec {
    T c[K];
    uint32_t idx;
};

struct Box {
    double lo[16], hi[16];
};

// widest.widest_dim: np.argmax of the float64 widths (first maximum)
inline int widest_dim(const Box& b, int k) {
    int best = 0;
    double bw = b.hi[0] - b.lo[0];
    for (int d = 1; d < k; ++d) {
        const double w = b.hi[d] - b.lo[d];
        if (w > bw) { bw = w; best = d; }
    }
    return best;
}

template <typename T, int K>
struct Builder {
    using R = Rec<T, K>;
    R* a;
    uint64_t n;
    int widest;
    uint32_t* perm;
    uint8_t* dims;

    int dim_of(uint64_t node, const Box& box) const { return widest ? widest_dim(box, K) : level_of(node) % K; }

    void sort_slice(uint64_t lo, uint64_t hi, int d, bool parallel) {
        auto less = [d](const R& x, const R& y) { return x.c[d] < y.c[d]; };
        if (parallel)
            __gnu_parallel::stable_sort(a + lo, a + hi, less);
        else
            std::stable_sort(a + lo, a + hi, less);
    }

    // one node: sort its slice, place rank `off`; returns the plane
    double place_node(uint64_t node, uint64_t lo, uint64_t hi, int d, bool parallel) {
        sort_slice(lo, hi, d, parallel);
        const uint64_t lc = 2 * node + 1;
        const uint64_t off = lc < n ? subtree_size(lc, n) : 0;
        perm[node] = a[lo + off].idx;
        if (dims) dims[node] = (uint8_t)d;
        return (double)a[lo + off].c[d];
    }

    void rec(uint64_t node, uint64_t lo, uint64_t hi, Box box) {
        // iterative on the right child, recursive on the left (depth <= 31)
        while (true) {
            const int d = dim_of(node, box);
            const double plane = place_node(node, lo, hi, d, false);
            const uint64_t lc = 2 * node + 1;
            const uint64_t off = lc < n ? subtree_size(lc, n) : 0;
            if (lc < n) {
                Box lb = box;
                if (widest) lb.hi[d] = std::min(lb.hi[d], plane);
                rec(lc, lo, lo + off, lb);
            }
            if (lc + 1 >= n) return;
            if (widest) box.lo[d] = std::max(box.lo[d], plane);
            node = lc + 1;
            lo = lo + off + 1;
        }
    }

    struct Task {
        uint64_t node, lo, hi;
        Box box;
    };

    void run(const Box& world, int threads) {
        // top levels breadth first with the parallel stable sort, until
        // there are enough independent subtrees for the host threads
        std::vector<Task> cur{{0, 0, n, world}}, next;
        const size_t want = (size_t)threads * 8;
        while (!cur.empty() && cur.size() < want) {
            next.clear();
            for (const Task& t : cur) {
                const int d = dim_of(t.node, t.box);
                const double plane = place_node(t.node, t.lo, t.hi, d, threads > 1);
                const uint64_t lc = 2 * t.node + 1;
                const uint64_t off = lc < n ? subtree_size(lc, n) : 0;
                if (lc < n) {
                    Task l{lc, t.lo, t.lo + off, t.box};
                    if (widest) l.box.hi[d] = std::min(l.box.hi[d], plane);
                    next.push_back(l);
                }
                if (lc + 1 < n) {
                    Task r{lc + 1, t.lo + off + 1, t.hi, t.box};
                    if (widest) r.box.lo[d] = std::max(r.box.lo[d], plane);
                    next.push_back(r);
                }
            }
            cur.swap(next);
        }
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
        for (long i = 0; i < (long)cur.size(); ++i) rec(cur[i].node, cur[i].lo, cur[i].hi, cur[i].box);
    }
};

template <typename T, int K>
int build_k(const T* pts, uint64_t n, int widest, uint32_t* perm, uint8_t* dims, int threads) {
    using R = Rec<T, K>;
    R* a = (R*)malloc(n * sizeof(R));
    if (!a) return -1;
    Box world;
    for (int d = 0; d < K; ++d) {
        world.lo[d] = INFINITY;
        world.hi[d] = -INFINITY;
    }
#pragma omp parallel num_threads(threads)
    {
        Box loc;
        for (int d = 0; d < K; ++d) {
            loc.lo[d] = INFINITY;
            loc.hi[d] = -INFINITY;
        }
#pragma omp for schedule(static)
        for (long i = 0; i < (long)n; ++i) {
            for (int d = 0; d < K; ++d) {
                const T v = pts[(uint64_t)i * K + d];
                a[i].c[d] = v;
                loc.lo[d] = std::min(loc.lo[d], (double)v);
                loc.hi[d] = std::max(loc.hi[d], (double)v);
            }
            a[i].idx = (uint32_t)i;
        }
#pragma omp critical
        for (int d = 0; d < K; ++d) {
            world.lo[d] = std::min(world.lo[d], loc.lo[d]);
            world.hi[d] = std::max(world.hi[d], loc.hi[d]);
        }
    }
    Builder<T, K> b{a, n, widest, perm, dims};
    b.run(world, threads);
    free(a);
    return 0;
}

template <typename T>
int build_t(const T* pts, int64_t n, int k, int widest, uint32_t* perm, uint8_t* dims, int threads) {
    if (n <= 0) return 0;
    if (threads <= 0) threads = omp_get_num_procs();
    omp_set_num_threads(threads);  // also the parallel stable sort's team
    const uint64_t un = (uint64_t)n;
    switch (k) {
        case 1: return build_k<T, 1>(pts, un, widest, perm, dims, threads);
        case 2: return build_k<T, 2>(pts, un, widest, perm, dims, threads);
        case 3: return build_k<T, 3>(pts, un, widest, perm, dims, threads);
        case 4: return build_k<T, 4>(pts, un, widest, perm, dims, threads);
        case 5: return build_k<T, 5>(pts, un, widest, perm, dims, threads);
        case 6: return build_k<T, 6>(pts, un, widest, perm, dims, threads);
        case 7: return build_k<T, 7>(pts, un, widest, perm, dims, threads);
        case 8: return build_k<T, 8>(pts, un, widest, perm, dims, threads);
        case 9: return build_k<T, 9>(pts, un, widest, perm, dims, threads);
        case 10: return build_k<T, 10>(pts, un, widest, perm, dims, threads);
        case 11: return build_k<T, 11>(pts, un, widest, perm, dims, threads);
        case 12: return build_k<T, 12>(pts, un, widest, perm, dims, threads);
        case 13: return build_k<T, 13>(pts, un, widest, perm, dims, threads);
        case 14: return build_k<T, 14>(pts, un, widest, perm, dims, threads);
        case 15: return build_k<T, 15>(pts, un, widest, perm, dims, threads);
        case 16: return build_k<T, 16>(pts, un, widest, perm, dims, threads);
        default: return -2;
    }
}

}  // namespace

extern "C" {

/* Recursive median placement (verify.py:121-168) on float32 AoS points.
 * perm[s] = input row at node s; dims (widest, may be null for RR) = split
 * dimension of node s.  threads <= 0: all host threads.  Returns 0. */
int oracle_rec_build_f32(const float* pts, int64_t n, int k, int widest, uint32_t* perm, uint8_t* dims,
                         int threads) {
    return build_t<float>(pts, n, k, widest, perm, dims, threads);
}

/* The same on float64 AoS points (the reference's own coordinate dtype). */
int oracle_rec_build_f64(const double* pts, int64_t n, int k, int widest, uint32_t* perm, uint8_t* dims,
                         int threads) {
    return build_t<double>(pts, n, k, widest, perm, dims, threads);
}

}  // extern "C"
