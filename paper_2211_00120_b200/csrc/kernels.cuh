// kernels.cuh -- launch-side declarations shared by the .cu translation units.
#pragma once
#include <cstdint>
#include "common.cuh"
#include "lbkd_b200.h"

namespace lbkd {

enum Mode { kRoundRobin = 0, kWidest = 1 };

// Fields of a node's within-node order T(s) (select.cu): m dimensions, most
// significant first, then the input index.
struct Chain {
    u32 m;
    uint8_t d[LBKD_MAX_K];
};
constexpr int kChainWords = sizeof(Chain) / 4;

// RR: dims l, l-1, ..., max(0, l-k+1) (mod k)
__host__ __device__ inline void rr_chain(int l, int k, Chain& c) {
    int m = l + 1 < k ? l + 1 : k;
    c.m = (u32)m;
    for (int i = 0; i < m; ++i) c.d[i] = (uint8_t)((l - i) % k);
}

// widest: node s and its ancestors' split dims, most recent first, repeats
// dropped (the reference's stable sorts nest: widest.py:119-131)
__device__ inline void widest_chain(u64 s, int k, const uint8_t* split_dims, Chain& c) {
    c.m = 0;
    u32 seen = 0;
    u64 a = s;
    while (true) {
        const int d = split_dims[a];
        if (!((seen >> d) & 1u)) {
            seen |= 1u << d;
            c.d[c.m++] = (uint8_t)d;
            if ((int)c.m == k) break;
        }
        if (a == 0) break;
        a = (a - 1) >> 1;
    }
}

// per-segment pick record of the select path
enum { kSelLo = 0, kSelShift, kSelB, kSelR, kSelC, kSelOff, kSelFill, kSelMode, kSelW = 8 };
// sel[kSelB] of a segment whose node box is a single point: the node is the
// element at in-order position sel[kSelLo] (pick / filter, select.cu)
constexpr u32 kSelPositional = 0xffffffffu;

// Working set of the global levels.
// Points travel with their sort: W[buf] holds k coordinate arrays and one
// index array (SoA, `stride` u32 each) in IN-ORDER layout -- the level-l
// segment of node F(l)+j occupies [ib(j), ib(j) + ss(j)), and every finished
// node stays at its own in-order slot, so splitting a segment moves nothing.
// Sort path: each segment's data lives in W[parity] and flips buffer only on the digit
// passes that actually reorder it; select path: level l lives in
// W[(l - lfirst) & 1].
struct Buffers {
    u32* w[2];
    u64 stride;
    // select path (select.cu)
    u32* sel;         // [nseg][kSelW]
    u32* cand;        // candidate records [n][k+1]
    u32* cand2;       // compaction buffer  [n][k+1]
    u32* cand_ctr;    // [1]
    u32* piv;         // [nseg][k+1] pivot records (coordinate bits + index)
    Chain* chains;    // [nseg]
    u32* tile_lt;     // [tiles][2] per (tile, segment part) counts below the pivot
    u32* sub_lt;      // [subtiles][2] the same per 256-position warp subtile
    u32* ppos;        // [nseg] pivot positions
    u32* hist;        // [nseg][4][256] digit counts of the level's keys
    u32* seg_and;     // [nseg] AND of keys  \  digit d of segment j is constant
    u32* seg_or;      // [nseg] OR of keys   /  iff ((and ^ or) >> 8d) & 255 == 0
    uint8_t* state[2];  // per level (l & 1): parity_in << 4 | mask of passes to run
    u64* status;      // [tiles][256] decoupled-lookback words
    u32* tile_ctr;    // one counter per pass launch
    u64* moved;       // per pass launch: points the launch reordered (profiling)
    u32* err;         // [0] non-finite flag (sticky over pipelined host builds), [1] this build's abort word
    float* boxes[2];  // widest: boxes of the level's nodes [nseg][2k]
    uint8_t* bmode[2];  // bucket mode of the level's nodes (0 value-linear, 1 key-linear)
    // level pairs (select.cu, "two levels per partition"): the second
    // level's pivot records / chains / positions and its below-pivot counts
    // per child side ([2][tiles][2], [2][subtiles][2]) beside the first's
    u32* piv2;
    Chain* chains2;
    u32* ppos2;
    u32* tile_lt2;
    u32* sub_lt2;
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
    int subtree_sel = 1;   // in-CTA levels by selection (subtree_sel.cu) or by presorted lists
    int lroot = 0;         // sub-build: root node (level, index) of the view;
    u64 jroot = 0;         // the whole tree is (0, 0)
    WidthTab wt{};         // float64 builds: rank-coded coordinates' value table (else wt.v == null)
    int pair = 0;          // round robin: global levels two per partition pass (select.cu)
};

inline LevelGeom view_of(const BuildParams& bp, int l) { return make_view(bp.n, l, bp.lroot, bp.jroot); }

__device__ __host__ __forceinline__ u32* warr(const Buffers& bf, u32 buf, int a) {
    return bf.w[buf] + (u64)a * bf.stride;
}

// select.cu
struct SelArgs {
    LevelGeom g;
    int k, mode, D;
    Buffers bf;
    u32 par;               // W[par] holds the level's data
    u32* hist;             // [nseg][2^D]
    u32* sel;
    u32* cand;
    u32* cand2;
    u32* cand_ctr;
    u32* piv;
    Chain* chains;
    uint8_t* split_dims;
    u32* perm;
    float* out_pts;
    const float* boxes_in;  // widest: boxes of the level's segments
    float* boxes_out;       //         boxes of their children
    const uint8_t* bmode_in;  // bucket mode of the level's segments
    uint8_t* bmode_out;       //   and of their children (select.cu)
    u32* tile_lt;          // [tiles][2] below-pivot counts -> exclusive prefixes
    u32* sub_lt;           // [subtiles][2] below-pivot counts per 256-position warp subtile
    u32* ppos;             // [nseg] in-order position of each segment's pivot
    u32* hist_next;        // partition: the next level's histogram (D = kFuseD), or null
    int hflush_every;      // partition: flush the warp-private 16-bit bins every this many subtiles (<= 255)
    int tiles_per_cta;
    u64 ntiles;
    WidthTab wt;           // widths of rank-coded (float64) builds
    // level pairs: the second level of a pair (a.g = the children, level
    // l + 1) still in its parents' layout (g0 = level l): parents' pivot
    // records, chains, positions and below counts; side strides of the
    // children's count arrays (tile_lt / sub_lt = [2][...][2])
    int pair;
    LevelGeom g0;
    const u32* piv0;
    const Chain* chains0;
    const u32* ppos0;
    const u32* tile_lt0;
    const u32* sub_lt0;
    u64 lt_tstride, lt_sstride;
    int fuse_d;            // pair partition: bins of its fused histogram (2^fuse_d per grandchild)
};
int sel_digit_bits(u64 nseg);
void launch_init_stats(const BuildParams& bp, const Buffers& bf, u32* minmax, cudaStream_t st);
void launch_check_finite(const float* pts, u64 total, u32* err, cudaStream_t st);
void launch_view_minmax(const BuildParams& bp, const Buffers& bf, u32* minmax, u64 m, cudaStream_t st);
void launch_root(const BuildParams& bp, const Buffers& bf, const u32* minmax, cudaStream_t st);
void launch_sel_hist(const SelArgs& a, int b, cudaStream_t st);
void launch_sel_pick(const SelArgs& a, cudaStream_t st);
void launch_sel_filter(const SelArgs& a, int b, cudaStream_t st);
void launch_sel_select(const SelArgs& a, int b, cudaStream_t st);
int sel_items(int b);
int sel_tile(int b);
void launch_sel_part(const SelArgs& a, int b, cudaStream_t st);
void launch_sel_child_hist(const SelArgs& a, int b, cudaStream_t st);
void launch_sel_filter_pair(const SelArgs& a, int b, cudaStream_t st);
void launch_sel_part_pair(const SelArgs& a, int b, cudaStream_t st);

// global_sort.cu
void launch_init(const BuildParams& bp, const Buffers& bf, cudaStream_t st);
void launch_hist(const BuildParams& bp, const Buffers& bf, int l, cudaStream_t st);
void launch_plan(const BuildParams& bp, const Buffers& bf, int l, cudaStream_t st);
void launch_pass(const BuildParams& bp, const Buffers& bf, int l, int pass, u32 epoch,
                 u32* tile_ctr, u64* moved, cudaStream_t st);
void launch_pivots(const BuildParams& bp, const Buffers& bf, int l, cudaStream_t st);
void launch_extract(const BuildParams& bp, const Buffers& bf, int top, u32* d_sub, u64 sub_stride, int src_par,
                    cudaStream_t st);

// subtree.cu / subtree_sel.cu
struct SubtreeArgs {
    u64 n;
    int L, lam0, k, mode, M;
    const u32* w[2];          // global-level working set (SoA, in-order)
    u64 stride;
    const uint8_t* prev_state;  // plan state of level lam0-1
    const float* pts;
    float* out_pts;
    u32* perm;
    uint8_t* split_dims;
    const float* boxes0;  // widest: boxes of level-lam0 nodes [nseg][2k]
    u32* dbg;
    u64 jbase;    // global index (level lam0) of the view's first subtree
    u64 pbase;    // global in-order position of the view's first point
    int lfirst;   // root level of the view
    int from_pts; // single-CTA whole-tree build straight from the input
    int entry_sorted;  // sort path: each subtree arrives in the reference's
                       // order T(parent); select path: in input order
    int src_par;       // select path: W[src_par] holds the subtree (else prev_state)
    int bucket_lists;  // RR list kernel: chain orders by one bucket pass each (env LBKD_BUCKET=0: radix passes)
    const u32* abort_word;  // non-null and set: non-finite input, return at once
    WidthTab wt;       // widths of rank-coded (float64) builds
};

size_t subtree_smem_bytes(int b, int k, int mode);
size_t subtree_rr_smem_bytes(int b, int k);
void launch_subtree(const BuildParams& bp, const Buffers& bf, int lam0, int entry_sorted, int src_par,
                    cudaStream_t st);
size_t subtree_sel_smem_bytes(int b, int k);
void launch_subtree_sel(const SubtreeArgs& a, unsigned grid, int b, cudaStream_t st);

// rank64.cu (float64 input: per-dimension dense ranks, see the file header)
void note_cuda_error(cudaError_t e);
size_t rank_scratch_words(u64 n);
int rank_sort_dim(const double* pts, u64 n, int k, int d, u32* scratch, u32* err, cudaStream_t st);
const u32* rank_count_word(const u32* scratch, u64 n);
int rank_assign_dim(u64 n, int k, int d, u32 center, int wide, float* codes, double* table, u32* scratch,
                    cudaStream_t st);
void launch_gather_rows_f64(const double* pts, const u32* perm, u64 n, int k, double* out, cudaStream_t st);

// widest.cu
void launch_world_bounds(const BuildParams& bp, u32* d_minmax, cudaStream_t st);
void launch_widest_root(const BuildParams& bp, const u32* d_minmax, float* box0, cudaStream_t st);
void launch_widest_nodes(const BuildParams& bp, int parent_level, const float* boxes_in,
                         float* boxes_out, cudaStream_t st);

}  // namespace lbkd
