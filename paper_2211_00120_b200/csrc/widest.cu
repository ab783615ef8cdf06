// widest.cu -- per-node work of the widest-dimension variant on the global
// levels (widest.py:84-93, kernels_numba.py:49-110).
//
// The reference re-derives each element's child box by walking the
// finalized ancestors (O(l) per element per level).  Only two results exist
// per level-l node (its two children), so here one thread per child node
// clips its parent's stored box by the parent's plane and takes the first
// argmax of the float64 widths; the rekey kernel then reads the split dim
// of each element's node.  Clipping is min/max over a set of planes, so the
// top-down result equals the reference's bottom-up walk.
#include "kernels.cuh"

namespace lbkd {

constexpr int kMaxKW = 16;

// world_bounds (widest.py:84-88): per-dimension min/max as order-flipped
// uint32 so plain atomicMin/atomicMax are exact.  d_minmax: [k] min, [k] max.
__global__ void world_bounds_kernel(const float* __restrict__ pts, u64 n, int k, u32* d_minmax) {
    __shared__ u32 smin[kMaxKW], smax[kMaxKW];
    if (threadIdx.x < kMaxKW) { smin[threadIdx.x] = 0xffffffffu; smax[threadIdx.x] = 0u; }
    __syncthreads();
    u32 mn[kMaxKW], mx[kMaxKW];
    for (int d = 0; d < k; ++d) { mn[d] = 0xffffffffu; mx[d] = 0u; }
    u64 total = n * (u64)k;
    // walk the flat array; element e belongs to dim e % k
    for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < total; e += (u64)gridDim.x * blockDim.x) {
        u32 f = flip_key(__ldg(pts + e));
        int d = (int)(e % (u64)k);
        for (int c = 0; c < k; ++c)
            if (c == d) { mn[c] = min(mn[c], f); mx[c] = max(mx[c], f); }
    }
    for (int d = 0; d < k; ++d) {
        u32 a = __reduce_min_sync(kFullMask, mn[d]);
        u32 b = __reduce_max_sync(kFullMask, mx[d]);
        if ((threadIdx.x & 31) == 0) { atomicMin(&smin[d], a); atomicMax(&smax[d], b); }
    }
    __syncthreads();
    if (threadIdx.x < (unsigned)k) {
        atomicMin(&d_minmax[threadIdx.x], smin[threadIdx.x]);
        atomicMax(&d_minmax[k + threadIdx.x], smax[threadIdx.x]);
    }
}

void launch_world_bounds(const BuildParams& bp, u32* d_minmax, cudaStream_t st) {
    u64 total = bp.n * (u64)bp.k;
    u64 blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    world_bounds_kernel<<<(unsigned)blocks, 256, 0, st>>>(bp.pts, bp.n, bp.k, d_minmax);
}

__device__ __forceinline__ int first_argmax_width(const float* lo, const float* hi, int k, const WidthTab& wt) {
    int best = 0;
    double bw = coord_width(wt, 0, lo[0], hi[0]);
    for (int d = 1; d < k; ++d) {
        double w = coord_width(wt, d, lo[d], hi[d]);
        if (w > bw) { bw = w; best = d; }
    }
    return best;
}

// root: box = world, dim = widest_dim(world) (widest.py:91-93, :164-166)
__global__ void widest_root_kernel(const u32* d_minmax, int k, float* box0, uint8_t* split_dims, WidthTab wt) {
    if (threadIdx.x != 0) return;
    float lo[kMaxKW], hi[kMaxKW];
    for (int d = 0; d < k; ++d) {
        lo[d] = unflip_key(d_minmax[d]);
        hi[d] = unflip_key(d_minmax[k + d]);
        box0[d] = lo[d];
        box0[k + d] = hi[d];
    }
    split_dims[0] = (uint8_t)first_argmax_width(lo, hi, k, wt);
}

void launch_widest_root(const BuildParams& bp, const u32* d_minmax, float* box0, cudaStream_t st) {
    widest_root_kernel<<<1, 32, 0, st>>>(d_minmax, bp.k, box0, bp.split_dims, bp.wt);
}

// children of level-lp nodes: box_c = box_parent clipped by the parent's
// plane (left: hi, right: lo), dim_c = first argmax of f64 widths
__global__ void widest_nodes_kernel(u64 n, int lp, const float* __restrict__ boxes_in, float* boxes_out,
                                    uint8_t* split_dims, const float* __restrict__ out_pts, int k, WidthTab wt) {
    u64 nchild = 2ull << lp;
    u64 c = blockIdx.x * (u64)blockDim.x + threadIdx.x;
    if (c >= nchild) return;
    u64 Fp = (1ull << lp) - 1ull, Fc = (2ull << lp) - 1ull;
    u64 node = Fc + c;
    if (node >= n) return;
    u64 pj = c >> 1;
    u64 s = Fp + pj;
    int d = split_dims[s];
    float plane = out_pts[s * k + d];  // the parent's point, just placed
    float lo[kMaxKW], hi[kMaxKW];
    for (int q = 0; q < k; ++q) { lo[q] = boxes_in[pj * 2 * k + q]; hi[q] = boxes_in[pj * 2 * k + k + q]; }
    if ((c & 1ull) == 0) { if (plane < hi[d]) hi[d] = plane; }   // left child
    else { if (plane > lo[d]) lo[d] = plane; }                     // right child
    for (int q = 0; q < k; ++q) { boxes_out[c * 2 * k + q] = lo[q]; boxes_out[c * 2 * k + k + q] = hi[q]; }
    split_dims[node] = (uint8_t)first_argmax_width(lo, hi, k, wt);
}

void launch_widest_nodes(const BuildParams& bp, int parent_level, const float* boxes_in, float* boxes_out,
                         cudaStream_t st) {
    u64 nchild = 2ull << parent_level;
    unsigned blocks = (unsigned)((nchild + 255) / 256);
    widest_nodes_kernel<<<blocks, 256, 0, st>>>(bp.n, parent_level, boxes_in, boxes_out, bp.split_dims,
                                                bp.out_pts, bp.k, bp.wt);
}

}  // namespace lbkd
