// Whole-tree validation and subtree boxes on the GPU.
//
// lbkd_check_valid replaces verify.check_valid
// (/root/reference/pkg/src/lbkd/verify.py:195-245): node d violates the
// ordering if, for an ancestor p reached through child a, d's coordinate in
// p's split dim lies on the wrong side of p's plane (left: own > plane,
// right: own < plane; closed on both sides).  One thread per node walks its
// ancestors nearest first; the witness is the lowest violating node and, for
// it, the nearest violated ancestor -- the reference's deterministic rescan
// order (:226-243).
//
// lbkd_subtree_boxes replaces verify.brute_subtree_boxes (verify.py:347-374):
// box(s) = world bounds clipped by the plane of every ancestor (left child:
// hi[d] = min(hi[d], plane); right child: lo[d] = max(lo[d], plane)).  The
// reference applies the clips top-down with Python's min / max, which keep
// the EARLIER operand on ties; walking up from the node we keep the latest
// (= top-most) of equal values, so even the sign of a zero matches.
#include "../../include/lbkd_b200.h"
#include "common.cuh"

namespace lbkd {
void note_cuda_error(cudaError_t e);
namespace {

__device__ __forceinline__ int vdim(const uint8_t* dims, u64 s, int k) {
    if (dims) return dims[s];
    return (63 - __clzll(s + 1)) % k;  // level(s) mod k
}

template <typename T>
__global__ void check_valid_kernel(const T* __restrict__ tree, u64 n, int k, const uint8_t* __restrict__ dims,
                                   unsigned long long* __restrict__ best) {
    for (u64 d = (u64)blockIdx.x * blockDim.x + threadIdx.x; d < n; d += (u64)gridDim.x * blockDim.x) {
        u64 a = d;
        while (a > 0) {
            const u64 p = (a - 1) >> 1;
            const int dp = vdim(dims, p, k);
            const T own = tree[d * k + dp], plane = tree[p * k + dp];
            if ((a & 1) ? own > plane : own < plane) {
                atomicMin(best, (unsigned long long)d);
                break;
            }
            a = p;
        }
    }
}

// witness fields of the lowest violating node: [descendant, ancestor, dim],
// -1s when the tree is valid
template <typename T>
__global__ void witness_kernel(const T* __restrict__ tree, u64 n, int k, const uint8_t* __restrict__ dims,
                               const unsigned long long* __restrict__ best, int64_t* __restrict__ out) {
    const unsigned long long d = *best;
    out[0] = out[1] = out[2] = -1;
    if (d >= n) return;
    u64 a = d;
    while (a > 0) {
        const u64 p = (a - 1) >> 1;
        const int dp = vdim(dims, p, k);
        const T own = tree[d * k + dp], plane = tree[p * k + dp];
        if ((a & 1) ? own > plane : own < plane) {
            out[0] = (int64_t)d;
            out[1] = (int64_t)p;
            out[2] = dp;
            return;
        }
        a = p;
    }
}

// world bounds into row 0 of lo / hi: order-preserving u64 keys of the
// float64 values (float32 widens exactly) reduced with atomics in the row-0
// slots, then decoded
__device__ __forceinline__ unsigned long long flip64(double x) {
    unsigned long long u = (unsigned long long)__double_as_longlong(x);
    if (u == 0x8000000000000000ull) u = 0ull;  // -0.0 == +0.0
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void bounds_init_kernel(double* lo, double* hi, int k) {
    const int j = threadIdx.x;
    if (j < k) {
        reinterpret_cast<unsigned long long*>(lo)[j] = ~0ull;
        reinterpret_cast<unsigned long long*>(hi)[j] = 0ull;
    }
}

template <typename T>
__global__ void bounds_kernel(const T* __restrict__ tree, u64 n, int k, double* lo, double* hi) {
    const int j = blockIdx.y;
    unsigned long long mn = ~0ull, mx = 0ull;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const unsigned long long key = flip64((double)tree[i * k + j]);
        mn = key < mn ? key : mn;
        mx = key > mx ? key : mx;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(kFullMask, mn, o), b = __shfl_xor_sync(kFullMask, mx, o);
        mn = a < mn ? a : mn;
        mx = b > mx ? b : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(reinterpret_cast<unsigned long long*>(lo) + j, mn);
        atomicMax(reinterpret_cast<unsigned long long*>(hi) + j, mx);
    }
}

__global__ void bounds_finish_kernel(double* lo, double* hi, int k) {
    const int j = threadIdx.x;
    if (j < k) {
        // coords.min / max (axis=0) of finite values; -0.0 and 0.0 compare
        // equal and numpy's reduction may return either -- a zero extreme is
        // reported as +0.0 here (flip64 folds -0.0 into +0.0)
        for (int side = 0; side < 2; ++side) {
            double* v = side ? hi : lo;
            const unsigned long long key = reinterpret_cast<unsigned long long*>(v)[j];
            const unsigned long long u = (key >> 63) ? (key & 0x7fffffffffffffffull) : ~key;
            v[j] = __longlong_as_double((long long)u);
        }
    }
}

template <typename T>
__global__ void boxes_kernel(const T* __restrict__ tree, u64 n, int k, const uint8_t* __restrict__ dims,
                             double* __restrict__ lo, double* __restrict__ hi) {
    for (u64 s = 1 + (u64)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (u64)gridDim.x * blockDim.x) {
        T l[LBKD_MAX_K], h[LBKD_MAX_K];
        bool hl[LBKD_MAX_K], hh[LBKD_MAX_K];
        for (int j = 0; j < k; ++j) hl[j] = hh[j] = false;
        u64 a = s;
        while (a > 0) {  // nearest ancestor first; ties keep the top-most
            const u64 p = (a - 1) >> 1;
            const int dp = vdim(dims, p, k);
            const T plane = tree[p * k + dp];
            if (a & 1) {
                if (!hh[dp] || plane <= h[dp]) { h[dp] = plane; hh[dp] = true; }
            } else {
                if (!hl[dp] || plane >= l[dp]) { l[dp] = plane; hl[dp] = true; }
            }
            a = p;
        }
        for (int j = 0; j < k; ++j) {
            const double wl = lo[j], wh = hi[j];  // world (row 0) comes first top-down
            lo[s * k + j] = (hl[j] && (double)l[j] > wl) ? (double)l[j] : wl;
            hi[s * k + j] = (hh[j] && (double)h[j] < wh) ? (double)h[j] : wh;
        }
    }
}

int rc_of(cudaError_t e) {
    if (e == cudaSuccess) return LBKD_OK;
    note_cuda_error(e);
    return LBKD_ECUDA;
}

unsigned grid_for(u64 n) {
    u64 g = (n + 255) / 256;
    return (unsigned)(g < 148ull * 16 ? (g ? g : 1) : 148ull * 16);
}

}  // namespace
}  // namespace lbkd

using namespace lbkd;

namespace {

template <typename T>
int check_valid_impl(const T* d_tree, int64_t n, int k, const uint8_t* d_split_dims, int64_t* d_witness,
                     uint64_t* d_scratch, void* stream) {
    if (n < 0 || k < 1 || k > LBKD_MAX_K || !d_witness || !d_scratch || (n > 0 && !d_tree)) return LBKD_EINVAL_SHAPE;
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(d_scratch, 0xff, sizeof(uint64_t), st);
    if (n > 1)
        check_valid_kernel<T><<<grid_for((u64)n), 256, 0, st>>>(d_tree, (u64)n, k, d_split_dims,
                                                                 reinterpret_cast<unsigned long long*>(d_scratch));
    witness_kernel<T><<<1, 1, 0, st>>>(d_tree, (u64)n, k, d_split_dims,
                                       reinterpret_cast<const unsigned long long*>(d_scratch), d_witness);
    return rc_of(cudaGetLastError());
}

template <typename T>
int subtree_boxes_impl(const T* d_tree, int64_t n, int k, const uint8_t* d_split_dims, double* d_lo, double* d_hi,
                       void* stream) {
    if (n < 0 || k < 1 || k > LBKD_MAX_K || (n > 0 && (!d_tree || !d_lo || !d_hi))) return LBKD_EINVAL_SHAPE;
    if (n == 0) return LBKD_OK;
    cudaStream_t st = (cudaStream_t)stream;
    bounds_init_kernel<<<1, 32, 0, st>>>(d_lo, d_hi, k);
    const unsigned g = grid_for((u64)n) < 296 ? grid_for((u64)n) : 296;
    bounds_kernel<T><<<dim3(g, k), 256, 0, st>>>(d_tree, (u64)n, k, d_lo, d_hi);
    bounds_finish_kernel<<<1, 32, 0, st>>>(d_lo, d_hi, k);
    if (n > 1) boxes_kernel<T><<<grid_for((u64)n), 256, 0, st>>>(d_tree, (u64)n, k, d_split_dims, d_lo, d_hi);
    return rc_of(cudaGetLastError());
}

}  // namespace

extern "C" {

int lbkd_check_valid(const float* d_tree, int64_t n, int k, const uint8_t* d_split_dims, int64_t* d_witness,
                     uint64_t* d_scratch, void* stream) {
    return check_valid_impl(d_tree, n, k, d_split_dims, d_witness, d_scratch, stream);
}

int lbkd_check_valid_f64(const double* d_tree, int64_t n, int k, const uint8_t* d_split_dims, int64_t* d_witness,
                         uint64_t* d_scratch, void* stream) {
    return check_valid_impl(d_tree, n, k, d_split_dims, d_witness, d_scratch, stream);
}

int lbkd_subtree_boxes(const float* d_tree, int64_t n, int k, const uint8_t* d_split_dims, double* d_lo,
                       double* d_hi, void* stream) {
    return subtree_boxes_impl(d_tree, n, k, d_split_dims, d_lo, d_hi, stream);
}

int lbkd_subtree_boxes_f64(const double* d_tree, int64_t n, int k, const uint8_t* d_split_dims, double* d_lo,
                           double* d_hi, void* stream) {
    return subtree_boxes_impl(d_tree, n, k, d_split_dims, d_lo, d_hi, stream);
}

}  // extern "C"
