// kernels.cuh -- launch-side declarations shared by the .cu translation units.
#pragma once
#include <cstdint>
#include "common.cuh"

namespace lbkd {

// Device-resident per-level plan, written by plan_kernel, read by the pass
// kernels, the next level's rekey and the subtree kernel.  Keeping it on the
// device lets a whole build be enqueued without host round trips.
struct LevelPlan {
    u32 skip[4];      // digit pass p is the identity for every segment
    u32 src[4];       // ping-pong buffer the pass reads
    u32 final_pass;   // pass that places pivots and partitions children
    u32 next_sel;     // buffer holding W_{l+1} after the level (W_0: 0)
    u32 pad[2];
};

enum Mode { kRoundRobin = 0, kWidest = 1 };

struct Buffers {
    u32* keys[2];
    u32* vals[2];
    u32* hist;        // [nseg][4][256]
    u32* seg_and;     // [nseg]
    u32* seg_or;      // [nseg]
    u64* status;      // [tiles][256] decoupled-lookback words
    u32* tile_ctr;    // one counter per pass launch
    LevelPlan* plan;
    u32* err;         // [0] non-finite flag
    float* boxes[2];  // widest: per-level node boxes [nseg][2k] (lo..., hi...)
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
};

// global_sort.cu
int global_items_for_bits(int b);
void launch_rekey_hist(const BuildParams& bp, const Buffers& bf, int l, cudaStream_t st);
void launch_plan(const BuildParams& bp, const Buffers& bf, int l, cudaStream_t st);
void launch_pass(const BuildParams& bp, const Buffers& bf, int l, int pass, u32 epoch,
                 u32* tile_ctr, cudaStream_t st);

// subtree.cu
size_t subtree_smem_bytes(int b, int k, int mode);
void launch_subtree(const BuildParams& bp, const Buffers& bf, int lam0, cudaStream_t st);

// widest.cu
void launch_world_bounds(const BuildParams& bp, u32* d_minmax, cudaStream_t st);
void launch_widest_root(const BuildParams& bp, const u32* d_minmax, float* box0, cudaStream_t st);
void launch_widest_nodes(const BuildParams& bp, int parent_level, const float* boxes_in,
                         float* boxes_out, cudaStream_t st);

}  // namespace lbkd
