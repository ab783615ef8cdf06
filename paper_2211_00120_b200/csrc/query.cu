// Batched nearest-neighbour and radius queries over a built level-order tree
// (SURVEY.md section 8(f) rank 1).
//
// Reference: lbkd.kernels_numpy.knn_search / radius_search
// (/root/reference/pkg/src/lbkd/kernels_numpy.py:114-245) behind
// lbkd.queries.knn / radius_query (queries.py:41-77).  The reference answers
// one query per call on the host; here one thread answers one query of a
// batch, reading the tree straight from the build's output (level-order
// float32 or float64 AoS rows; node s has children 2s+1 and 2s+2, its split plane is its
// own coordinate in dim level(s) mod k, or split_dims[s] for widest trees).
//
// Exactness: the reference computes in float64 (on float64 copies of
// float32 points, which widen exactly; float64 trees are read as they are), and the distance is
// accumulated in the same order with separately rounded multiply and add
// (__dmul_rn / __dadd_rn: no FMA contraction), so squared distances are
// bit-identical.  The kNN answer is the unique m smallest (dist2, node) pairs
// -- the keep-list insertion and the pruning rule (skip a far side only when
// the list is full and its plane distance exceeds the worst kept distance;
// equal is visited) are the reference's, so the result does not depend on
// the traversal order.  Radius results are sorted ascending per query like
// queries.radius_query (queries.py:77).
#include <math_constants.h>
#include "../../include/lbkd_b200.h"
#include "common.cuh"

namespace lbkd {
void note_cuda_error(cudaError_t e);  // capi.cu: lbkd_last_cuda_error text
namespace {

constexpr int kStack = 32;  // far-side stack: depth <= levels <= 31

__device__ __forceinline__ int node_dim(const uint8_t* split_dims, u32 node, int k) {
    if (split_dims) return split_dims[node];
    const int lvl = 31 - __clz(node + 1);  // level(s) = floor(log2(s + 1))
    return lvl % k;
}

template <typename T>
__device__ __forceinline__ double dist2(const T* row, const double* q, int k) {
    double d2 = 0.0;
    for (int j = 0; j < k; ++j) {
        const double t = __dsub_rn(q[j], (double)row[j]);
        d2 = __dadd_rn(d2, __dmul_rn(t, t));
    }
    return d2;
}

// Keep-list in local memory (MCAP > 0) or in the caller's output row
// (MCAP == 0, any m).  HEAP = false: the reference's sorted insertion (cheap
// for small m); HEAP = true: a max-heap on (dist2, node), O(log m) per take,
// heap-sorted at the end.  Both keep exactly the m smallest (dist2, node)
// pairs, so the answer is the same.
template <typename T, int MCAP, bool HEAP>
__global__ void __launch_bounds__(128) knn_kernel(const T* __restrict__ tree, u32 n, int k,
                                                  const uint8_t* __restrict__ split_dims,
                                                  const double* __restrict__ queries, u64 nq, int m,
                                                  int64_t* __restrict__ out_idx, double* __restrict__ out_d2) {
    const u64 qi = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (qi >= nq) return;
    double q[LBKD_MAX_K];
    for (int j = 0; j < k; ++j) q[j] = queries[qi * k + j];
    int64_t* oi = out_idx + qi * (u64)m;
    double* od = out_d2 + qi * (u64)m;
    u32 lidx[MCAP > 0 ? MCAP : 1];
    double ld2[MCAP > 0 ? MCAP : 1];
    auto IDX = [&](int p) -> u32 { return MCAP > 0 ? lidx[p] : (u32)oi[p]; };
    auto D2 = [&](int p) -> double { return MCAP > 0 ? ld2[p] : od[p]; };
    auto SET = [&](int p, u32 i, double d) {
        if (MCAP > 0) { lidx[p] = i; ld2[p] = d; }
        else { oi[p] = i; od[p] = d; }
    };
    // (d, i) after (pd, pi) in the (dist2, node) order
    auto after = [](double d, u32 i, double pd, u32 pi) { return d > pd || (d == pd && i > pi); };
    auto sift_down = [&](int p, int len, u32 i, double d) {  // place (d, i) from slot p down
        while (true) {
            int c = 2 * p + 1;
            if (c >= len) break;
            if (c + 1 < len && after(D2(c + 1), IDX(c + 1), D2(c), IDX(c))) ++c;
            if (!after(D2(c), IDX(c), d, i)) break;
            SET(p, IDX(c), D2(c));
            p = c;
        }
        SET(p, i, d);
    };
    u32 st_node[kStack];
    double st_d2[kStack];
    int top = 0, count = 0;
    double worst = CUDART_INF;
    u32 node = 0;
    while (true) {
        if (node < n) {
            const T* row = tree + (u64)node * k;
            const double d2 = dist2(row, q, k);
            if (HEAP) {
                if (count < m) {
                    int p = count++;
                    while (p > 0) {  // sift up
                        const int par = (p - 1) >> 1;
                        if (!after(d2, node, D2(par), IDX(par))) break;
                        SET(p, IDX(par), D2(par));
                        p = par;
                    }
                    SET(p, node, d2);
                    if (count == m) worst = D2(0);
                } else if (!after(d2, node, D2(0), IDX(0))) {  // beats the worst kept
                    sift_down(0, m, node, d2);
                    worst = D2(0);
                }
            } else {
                bool take;
                if (count < m) take = true;
                else if (d2 < worst) take = true;
                else take = d2 == worst && node < IDX(count - 1);
                if (take) {
                    int pos;
                    if (count < m) pos = count++;
                    else pos = m - 1;
                    while (pos > 0) {
                        const double pd = D2(pos - 1);
                        const u32 pi = IDX(pos - 1);
                        if (!after(pd, pi, d2, node)) break;
                        SET(pos, pi, pd);
                        --pos;
                    }
                    SET(pos, node, d2);
                    if (count == m) worst = D2(m - 1);
                }
            }
            const int dim = node_dim(split_dims, node, k);
            const double delta = __dsub_rn(q[dim], (double)row[dim]);
            const u32 left = 2 * node + 1;
            u32 nearc, farc;
            if (delta <= 0.0) { nearc = left; farc = left + 1; }
            else { farc = left; nearc = left + 1; }
            st_node[top] = farc;
            st_d2[top] = __dmul_rn(delta, delta);
            ++top;
            node = nearc;
        } else {
            bool found = false;
            while (top > 0) {
                --top;
                if (count < m || st_d2[top] <= worst) {
                    node = st_node[top];
                    found = true;
                    break;
                }
            }
            if (!found) break;
        }
    }
    if (HEAP) {  // heap sort: the max goes to the end, ascending result
        for (int e = count - 1; e > 0; --e) {
            const u32 i = IDX(e);
            const double d = D2(e);
            SET(e, IDX(0), D2(0));
            sift_down(0, e, i, d);
        }
    }
    if (MCAP > 0)
        for (int p = 0; p < count; ++p) { oi[p] = lidx[p]; od[p] = ld2[p]; }
}

// Radius traversal.  FILL = false: count the hits; FILL = true: write them
// from out_idx[offsets[qi]] in traversal order.
template <typename T, bool FILL>
__global__ void __launch_bounds__(128) radius_kernel(const T* __restrict__ tree, u32 n, int k,
                                                     const uint8_t* __restrict__ split_dims,
                                                     const double* __restrict__ queries, u64 nq, double r2,
                                                     int64_t* __restrict__ counts,
                                                     const int64_t* __restrict__ offsets,
                                                     int64_t* __restrict__ out_idx) {
    const u64 qi = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (qi >= nq) return;
    double q[LBKD_MAX_K];
    for (int j = 0; j < k; ++j) q[j] = queries[qi * k + j];
    int64_t* dst = FILL ? out_idx + offsets[qi] : nullptr;
    u32 st_node[kStack];
    int top = 0;
    int64_t count = 0;
    u32 node = 0;
    while (true) {
        if (node < n) {
            const T* row = tree + (u64)node * k;
            if (dist2(row, q, k) <= r2) {
                if (FILL) dst[count] = node;
                ++count;
            }
            const int dim = node_dim(split_dims, node, k);
            const double delta = __dsub_rn(q[dim], (double)row[dim]);
            const u32 left = 2 * node + 1;
            u32 nearc, farc;
            if (delta <= 0.0) { nearc = left; farc = left + 1; }
            else { farc = left; nearc = left + 1; }
            if (__dmul_rn(delta, delta) <= r2) st_node[top++] = farc;
            node = nearc;
        } else {
            if (top == 0) break;
            node = st_node[--top];
        }
    }
    if (!FILL) counts[qi] = count;
}

// Exclusive scan of nq int64 counts into offsets[0..nq] (offsets[nq] =
// total): per-CTA sums, one CTA scans the sums, per-CTA rescan.
constexpr int kScanT = 1024;

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* sh, int64_t& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(kFullMask, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (w == 0) {
        int64_t s = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(kFullMask, s, o);
            if (lane >= o) s += y;
        }
        sh[32 + lane] = s;
    }
    __syncthreads();
    total = sh[32 + (blockDim.x >> 5) - 1];
    const int64_t r = x - v + (w ? sh[32 + w - 1] : 0);
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kScanT) scan_sums_kernel(const int64_t* counts, u64 nq, int64_t* sums) {
    __shared__ int64_t sh[64];
    const u64 i = (u64)blockIdx.x * kScanT + threadIdx.x;
    int64_t tot;
    block_excl_scan(i < nq ? counts[i] : 0, sh, tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanT) scan_top_kernel(int64_t* sums, u64 nb) {
    __shared__ int64_t sh[64];
    int64_t carry = 0;
    for (u64 b0 = 0; b0 < nb; b0 += kScanT) {
        const u64 i = b0 + threadIdx.x;
        int64_t tot;
        const int64_t e = block_excl_scan(i < nb ? sums[i] : 0, sh, tot);
        if (i < nb) sums[i] = carry + e;
        carry += tot;
    }
    if (threadIdx.x == 0) sums[nb] = carry;
}

__global__ void __launch_bounds__(kScanT) scan_apply_kernel(const int64_t* counts, u64 nq, const int64_t* sums,
                                                            u64 nb, int64_t* offsets) {
    __shared__ int64_t sh[64];
    const u64 i = (u64)blockIdx.x * kScanT + threadIdx.x;
    int64_t tot;
    const int64_t e = block_excl_scan(i < nq ? counts[i] : 0, sh, tot);
    if (i < nq) offsets[i] = sums[blockIdx.x] + e;
    if (blockIdx.x == 0 && threadIdx.x == 0) offsets[nq] = sums[nb];
}

// Ascending sort of each query's hits, one CTA per query.  Direction-free
// bitonic network (each merge starts with a flip stage), so a length that is
// not a power of two needs no padding: pairs whose upper element lies past
// the end are skipped (virtual +inf there never moves).  Segments up to
// kSortSmem sort in shared memory, longer ones in place in global memory.
constexpr int kSortT = 256;
constexpr int kSortSmem = 4096;

template <typename Arr>
__device__ __forceinline__ void bitonic_sort(Arr v, u32 len) {
    u32 P = 1;
    while (P < len) P <<= 1;
    for (u32 size = 2; size <= P; size <<= 1) {
        const u32 h = size >> 1;
        for (u32 i = threadIdx.x; i < P / 2; i += blockDim.x) {
            const u32 blk = i / h, off = i % h;
            const u32 a = blk * size + off, b = blk * size + size - 1 - off;
            if (b < len) {
                const int64_t x = v[a], y = v[b];
                if (x > y) { v[a] = y; v[b] = x; }
            }
        }
        __syncthreads();
        for (u32 hh = h >> 1; hh >= 1; hh >>= 1) {
            for (u32 i = threadIdx.x; i < P / 2; i += blockDim.x) {
                const u32 a = (i / hh) * 2 * hh + i % hh, b = a + hh;
                if (b < len) {
                    const int64_t x = v[a], y = v[b];
                    if (x > y) { v[a] = y; v[b] = x; }
                }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(kSortT) radius_sort_kernel(const int64_t* offsets, int64_t* out_idx) {
    __shared__ int64_t sv[kSortSmem];
    const int64_t b = offsets[blockIdx.x], e = offsets[blockIdx.x + 1];
    const u32 len = (u32)(e - b);
    if (len < 2) return;
    int64_t* g = out_idx + b;
    if (len <= (u32)kSortSmem) {
        for (u32 i = threadIdx.x; i < len; i += blockDim.x) sv[i] = g[i];
        __syncthreads();
        bitonic_sort(sv, len);
        for (u32 i = threadIdx.x; i < len; i += blockDim.x) g[i] = sv[i];
    } else {
        volatile int64_t* vg = g;  // global network: every stage reads the previous one's writes
        bitonic_sort(vg, len);
    }
}

cudaError_t finish(void) { return cudaGetLastError(); }

}  // namespace
}  // namespace lbkd

using namespace lbkd;

namespace {
int query_args_ok(const void* tree, int64_t n, int k, const double* q, int64_t nq) {
    if (n < 0 || n > (int64_t)0x7fffffff || k < 1 || k > LBKD_MAX_K || nq < 0) return 0;
    if ((n > 0 && !tree) || (nq > 0 && !q)) return 0;
    return 1;
}
int rc_of(cudaError_t e) {
    if (e == cudaSuccess) return LBKD_OK;
    note_cuda_error(e);
    return LBKD_ECUDA;
}
}  // namespace

namespace {

template <typename T>
int knn_impl(const T* d_tree, int64_t n, int k, const uint8_t* d_split_dims, const double* d_queries,
             int64_t nq, int m, int64_t* d_out_idx, double* d_out_d2, void* stream) {
    if (!query_args_ok(d_tree, n, k, d_queries, nq) || m < 1 || m > n || (nq > 0 && (!d_out_idx || !d_out_d2)))
        return LBKD_EINVAL_SHAPE;
    if (nq == 0 || n == 0) return LBKD_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned grid = (unsigned)((nq + 127) / 128);
    const u32 un = (u32)n;
    const u64 unq = (u64)nq;
#define LBKD_KNN(C, H) \
    knn_kernel<T, C, H><<<grid, 128, 0, st>>>(d_tree, un, k, d_split_dims, d_queries, unq, m, d_out_idx, d_out_d2)
    if (m <= 1) LBKD_KNN(1, false);
    else if (m <= 4) LBKD_KNN(4, false);
    else if (m <= 8) LBKD_KNN(8, false);
    else if (m <= 16) LBKD_KNN(16, true);
    else if (m <= 32) LBKD_KNN(32, true);
    else if (m <= 64) LBKD_KNN(64, true);
    else if (m <= 128) LBKD_KNN(128, true);
    else LBKD_KNN(0, true);
#undef LBKD_KNN
    return rc_of(finish());
}

template <typename T>
int radius_count_impl(const T* d_tree, int64_t n, int k, const uint8_t* d_split_dims, const double* d_queries,
                      int64_t nq, double r2, int64_t* d_counts, int64_t* d_offsets, int64_t* d_scratch,
                      void* stream) {
    if (!query_args_ok(d_tree, n, k, d_queries, nq) || !(r2 >= 0.0) || !d_offsets || (nq > 0 && !d_counts))
        return LBKD_EINVAL_SHAPE;
    cudaStream_t st = (cudaStream_t)stream;
    if (nq == 0) return rc_of(cudaMemsetAsync(d_offsets, 0, sizeof(int64_t), st));
    if (n == 0) {
        cudaMemsetAsync(d_counts, 0, sizeof(int64_t) * nq, st);
        return rc_of(cudaMemsetAsync(d_offsets, 0, sizeof(int64_t) * (nq + 1), st));
    }
    if (!d_scratch) return LBKD_EINVAL_SHAPE;
    const unsigned grid = (unsigned)((nq + 127) / 128);
    radius_kernel<T, false><<<grid, 128, 0, st>>>(d_tree, (u32)n, k, d_split_dims, d_queries, (u64)nq, r2, d_counts,
                                                nullptr, nullptr);
    const u64 nb = ((u64)nq + kScanT - 1) / kScanT;
    scan_sums_kernel<<<(unsigned)nb, kScanT, 0, st>>>(d_counts, (u64)nq, d_scratch);
    scan_top_kernel<<<1, kScanT, 0, st>>>(d_scratch, nb);
    scan_apply_kernel<<<(unsigned)nb, kScanT, 0, st>>>(d_counts, (u64)nq, d_scratch, nb, d_offsets);
    return rc_of(finish());
}

template <typename T>
int radius_fill_impl(const T* d_tree, int64_t n, int k, const uint8_t* d_split_dims, const double* d_queries,
                     int64_t nq, double r2, const int64_t* d_offsets, int64_t* d_out_idx, void* stream) {
    if (!query_args_ok(d_tree, n, k, d_queries, nq) || !(r2 >= 0.0) || (nq > 0 && !d_offsets))
        return LBKD_EINVAL_SHAPE;
    if (nq == 0 || n == 0) return LBKD_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned grid = (unsigned)((nq + 127) / 128);
    radius_kernel<T, true><<<grid, 128, 0, st>>>(d_tree, (u32)n, k, d_split_dims, d_queries, (u64)nq, r2, nullptr,
                                               d_offsets, d_out_idx);
    radius_sort_kernel<<<(unsigned)nq, kSortT, 0, st>>>(d_offsets, d_out_idx);
    return rc_of(finish());
}

}  // namespace

extern "C" {

int lbkd_knn(const float* d_tree, int64_t n, int k, const uint8_t* d_split_dims, const double* d_queries,
             int64_t nq, int m, int64_t* d_out_idx, double* d_out_d2, void* stream) {
    return knn_impl(d_tree, n, k, d_split_dims, d_queries, nq, m, d_out_idx, d_out_d2, stream);
}

int lbkd_knn_f64(const double* d_tree, int64_t n, int k, const uint8_t* d_split_dims, const double* d_queries,
                 int64_t nq, int m, int64_t* d_out_idx, double* d_out_d2, void* stream) {
    return knn_impl(d_tree, n, k, d_split_dims, d_queries, nq, m, d_out_idx, d_out_d2, stream);
}

int lbkd_radius_count(const float* d_tree, int64_t n, int k, const uint8_t* d_split_dims, const double* d_queries,
                      int64_t nq, double r2, int64_t* d_counts, int64_t* d_offsets, int64_t* d_scratch,
                      void* stream) {
    return radius_count_impl(d_tree, n, k, d_split_dims, d_queries, nq, r2, d_counts, d_offsets, d_scratch, stream);
}

int lbkd_radius_count_f64(const double* d_tree, int64_t n, int k, const uint8_t* d_split_dims,
                          const double* d_queries, int64_t nq, double r2, int64_t* d_counts, int64_t* d_offsets,
                          int64_t* d_scratch, void* stream) {
    return radius_count_impl(d_tree, n, k, d_split_dims, d_queries, nq, r2, d_counts, d_offsets, d_scratch, stream);
}

int64_t lbkd_radius_scratch_len(int64_t nq) { return nq <= 0 ? 1 : (nq + kScanT - 1) / kScanT + 1; }

int lbkd_radius_fill(const float* d_tree, int64_t n, int k, const uint8_t* d_split_dims, const double* d_queries,
                     int64_t nq, double r2, const int64_t* d_offsets, int64_t* d_out_idx, void* stream) {
    return radius_fill_impl(d_tree, n, k, d_split_dims, d_queries, nq, r2, d_offsets, d_out_idx, stream);
}

int lbkd_radius_fill_f64(const double* d_tree, int64_t n, int k, const uint8_t* d_split_dims,
                         const double* d_queries, int64_t nq, double r2, const int64_t* d_offsets,
                         int64_t* d_out_idx, void* stream) {
    return radius_fill_impl(d_tree, n, k, d_split_dims, d_queries, nq, r2, d_offsets, d_out_idx, stream);
}

}  // extern "C"
