// update_tags.cu -- the reference's kernel-plugin seam on the GPU.
//
// The reference dispatches its per-element tag refinement through
// accel.get_kernels() (/root/reference/pkg/src/lbkd/accel.py:48-58), whose
// modules export
//   update_tags_round_robin(tags, n, levels, l)            kernels_numba.py:21-46
//   update_tags_widest(tags, coords, split_dims, world_lo,
//                      world_hi, n, levels, l, dim_bits)   kernels_numba.py:49-110
// These are the same trivially parallel kernels over device arrays, one
// thread per element, exposed through the C-ABI (lbkd_update_tags_rr /
// lbkd_update_tags_widest) so a caller that keeps the reference's own sort
// can still drop in the GPU update.  The fused build path does not call them:
// there the update is the epilogue of the last digit pass (global_sort.cu)
// and of each in-CTA level (subtree.cu).
#include "kernels.cuh"

namespace lbkd {

__device__ __forceinline__ long long pivot_pos_ll(long long s, long long n, int levels, int l) {
    int shift = levels - l - 1;
    long long top = (1ll << l) - 1;
    long long nls = s - top;
    long long bottom_have = n - ((1ll << (levels - 1)) - 1);
    long long low = nls << shift;
    if (low > bottom_have) low = bottom_have;
    long long begin = top + nls * ((1ll << shift) - 1) + low;
    int cshift = shift - 1;
    long long first = ((2 * s + 2) << cshift) - 1;
    long long on_bottom = n - first;
    long long cw = 1ll << cshift;
    if (on_bottom < 0) on_bottom = 0;
    if (on_bottom > cw) on_bottom = cw;
    return begin + cw - 1 + on_bottom;
}

__global__ void update_tags_rr_kernel(u32* tags, long long n, int levels, int l) {
    long long top = (1ll << l) - 1;
    for (long long i = top + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        long long s = tags[i];
        long long p = pivot_pos_ll(s, n, levels, l);
        if (i < p) tags[i] = (u32)(2 * s + 1);
        else if (i > p) tags[i] = (u32)(2 * s + 2);
    }
}

__global__ void update_tags_widest_kernel(u32* tags, const double* coords, int k, uint8_t* split_dims,
                                          const double* wlo, const double* whi, long long n, int levels, int l,
                                          int dim_bits) {
    long long top = (1ll << l) - 1;
    u32 mask = (1u << dim_bits) - 1u;
    for (long long i = top + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        u32 packed = tags[i];
        long long s = packed >> dim_bits;
        int d = (int)(packed & mask);
        long long p = pivot_pos_ll(s, n, levels, l);
        if (i == p) {
            split_dims[s] = (uint8_t)d;  // the unique writer of node s's slot
            continue;
        }
        double lo[16], hi[16];
        for (int q = 0; q < k; ++q) { lo[q] = wlo[q]; hi[q] = whi[q]; }
        double plane = coords[p * k + d];
        long long child;
        if (i < p) { hi[d] = fmin(hi[d], plane); child = 2 * s + 1; }
        else { lo[d] = fmax(lo[d], plane); child = 2 * s + 2; }
        long long a = s;
        while (a > 0) {  // finalized ancestors sit at their own index
            long long q = (a - 1) >> 1;
            int dq = split_dims[q];
            double cp = coords[q * k + dq];
            if (a & 1) hi[dq] = fmin(hi[dq], cp);
            else lo[dq] = fmax(lo[dq], cp);
            a = q;
        }
        int nd = 0;
        double best = hi[0] - lo[0];
        for (int q = 1; q < k; ++q) {
            double w = hi[q] - lo[q];
            if (w > best) { best = w; nd = q; }
        }
        tags[i] = (u32)((child << dim_bits) | nd);
    }
}

void launch_update_tags_rr(u32* tags, long long n, int levels, int l, cudaStream_t st) {
    long long work = n - ((1ll << l) - 1);
    if (work <= 0) return;
    long long blocks = (work + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    update_tags_rr_kernel<<<(unsigned)blocks, 256, 0, st>>>(tags, n, levels, l);
}

void launch_update_tags_widest(u32* tags, const double* coords, int k, uint8_t* split_dims, const double* wlo,
                               const double* whi, long long n, int levels, int l, int dim_bits, cudaStream_t st) {
    long long work = n - ((1ll << l) - 1);
    if (work <= 0) return;
    long long blocks = (work + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    update_tags_widest_kernel<<<(unsigned)blocks, 256, 0, st>>>(tags, coords, k, split_dims, wlo, whi, n, levels,
                                                                l, dim_bits);
}

}  // namespace lbkd
