// kernels.cuh -- launch-side declarations shared by the .cu translation units.
#pragma once
#include <cstdint>
#include "common.cuh"

namespace lbkd {

enum Mode { kRoundRobin = 0, kWidest = 1 };

// Working set of the global levels.
// Points travel with their sort: W[buf] holds k coordinate arrays and one
// index array (SoA, `stride` u32 each) in IN-ORDER layout -- the level-l
// segment of node F(l)+j occupies [ib(j), ib(j) + ss(j)), and every finished
// node stays at its own in-order slot, so splitting a segment moves nothing.
// Each segment's data lives in W[parity] and flips buffer only on the digit
// passes that actually reorder it.
struct Buffers {
    u32* w[2];
    u64 stride;
    u32* hist;        // [nseg][4][256] digit counts of the level's keys
    u32* seg_and;     // [nseg] AND of keys  \  digit d of segment j is constant
    u32* seg_or;      // [nseg] OR of keys   /  iff ((and ^ or) >> 8d) & 255 == 0
    uint8_t* state[2];  // per level (l & 1): parity_in << 4 | mask of passes to run
    u64* status;      // [tiles][256] decoupled-lookback words
    u32* tile_ctr;    // one counter per pass launch
    u64* moved;       // per pass launch: points the launch reordered (profiling)
    u32* err;         // [0] non-finite flag
    float* boxes[2];  // widest: boxes of the level's nodes [nseg][2k]
};

struct BuildParams {
    u64 n;
    int k;
    int mode;
    int b;            // subtree capacity bits: M = 2^b - 1, tile T = 2^(b-1)
    const float* pts;
    float* out_pts;
    u32* perm;
    uint8_t* split_dims;   // widest only
    u32* dbg;              // optional per-level trace (single-subtree builds)
    int lroot = 0;         // sub-build: root node (level, index) of the view;
    u64 jroot = 0;         // the whole tree is (0, 0)
};

inline LevelGeom view_of(const BuildParams& bp, int l) { return make_view(bp.n, l, bp.lroot, bp.jroot); }

__device__ __host__ __forceinline__ u32* warr(const Buffers& bf, u32 buf, int a) {
    return bf.w[buf] + (u64)a * bf.stride;
}

// global_sort.cu
void launch_init(const BuildParams& bp, const Buffers& bf, cudaStream_t st);
void launch_hist(const BuildParams& bp, const Buffers& bf, int l, cudaStream_t st);
void launch_plan(const BuildParams& bp, const Buffers& bf, int l, cudaStream_t st);
void launch_pass(const BuildParams& bp, const Buffers& bf, int l, int pass, u32 epoch,
                 u32* tile_ctr, u64* moved, cudaStream_t st);
void launch_pivots(const BuildParams& bp, const Buffers& bf, int l, cudaStream_t st);
void launch_extract(const BuildParams& bp, const Buffers& bf, int top, u32* d_sub, u64 sub_stride,
                    cudaStream_t st);

// subtree.cu
size_t subtree_smem_bytes(int b, int k, int mode);
size_t subtree_rr_smem_bytes(int b, int k);
void launch_subtree(const BuildParams& bp, const Buffers& bf, int lam0, cudaStream_t st);

// widest.cu
void launch_world_bounds(const BuildParams& bp, u32* d_minmax, cudaStream_t st);
void launch_widest_root(const BuildParams& bp, const u32* d_minmax, float* box0, cudaStream_t st);
void launch_widest_nodes(const BuildParams& bp, int parent_level, const float* boxes_in,
                         float* boxes_out, cudaStream_t st);

}  // namespace lbkd
