// capi.cu -- C ABI and host orchestration (see include/lbkd_b200.h).
//
// One build = the reference's loop (builder.py:224-232) re-cut for B200:
//   prologue                     AoS -> SoA working set W[0], non-finite flag,
//                                world box / root dim (init_stats + root)
//   global levels 0 .. lam0-1    per level (select.cu): hist -> pick ->
//                                filter -> select -> stable 3-way partition
//                                (segments larger than one CTA can hold)
//   in-CTA levels lam0 .. L-1    one CTA per level-lam0 subtree finishes it in
//                                shared memory (subtree.cu / subtree_sel.cu)
// LBKD_ALGO=sort swaps the global levels for the literal per-level segmented
// radix sort (global_sort.cu).  Everything is enqueued on the caller's stream
// with device-side plans and replayed as a CUDA graph when repeated; the
// only host synchronisation is the final non-finite check.  Builds on one
// context are ordered by an event (they share its scratch).  Float64 input
// goes through rank64.cu first (lbkd_build_*_f64).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>
#include "../../include/lbkd_b200.h"
#include "kernels.cuh"

using namespace lbkd;

namespace {
thread_local char g_cuda_err[256] = "";

void note_cuda(cudaError_t e) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
}

}  // namespace

namespace lbkd {
void note_cuda_error(cudaError_t e) { note_cuda(e); }
void launch_update_tags_rr(u32* tags, long long n, int levels, int l, cudaStream_t st);
void launch_update_tags_widest(u32* tags, const double* coords, int k, uint8_t* split_dims, const double* wlo,
                               const double* whi, long long n, int levels, int l, int dim_bits, cudaStream_t st);
}

struct lbkd_ctx {
    int device = 0;
    int check = 1;
    u32 epoch = 1;
    int ctr = 0;
    int64_t launches = 0;
    int algo = 0;      // 0: select + partition (default), 1: per-level sort
    int subtree_sel = -1;  // in-CTA phase: -1 default per mode, 1 selection (subtree_sel.cu), 0 lists
    // CUDA graph of the last build (select path, no profiling / trace):
    // replayed when the same build is requested again (no launch gaps)
    int use_graph = 1;
    cudaStream_t cap_stream = nullptr;
    cudaEvent_t cap_fork = nullptr, cap_join = nullptr;
    struct GraphKey {
        const void* pts;
        const void* out;
        const void* perm;
        const void* dims;
        const void* err;
        int64_t n;
        int k, mode, algo, sub, check, profile;
        bool operator==(const GraphKey& o) const {
            return pts == o.pts && out == o.out && perm == o.perm && dims == o.dims && err == o.err && n == o.n && k == o.k &&
                   mode == o.mode && algo == o.algo && sub == o.sub && check == o.check && profile == o.profile;
        }
    };
    // a few instantiated graphs (the pipelined host builds alternate two
    // buffer slots, so two keys are live at once); least recently used evicted
    struct GraphEntry {
        GraphKey key{};
        cudaGraphExec_t exec = nullptr;
        int64_t launches = 0;
        int n_ev = 0;  // profiling events recorded by the captured build
        u64 used = 0;
    };
    static constexpr int kGraphSlots = 4;
    GraphEntry graphs[kGraphSlots];
    u64 graph_tick = 0;
    int err_sticky = 0;  // set while a pipelined host build is enqueued: its flag accumulates until lbkd_host_join
    u32* err_host = nullptr;  // the pipelined host builds' own non-finite flag (device builds use bf.err)
    // every build on this context (device or host, any stream) uses the same
    // scratch buffers: each build's stream first waits for the previous
    // build's completion event, so builds on one context never overlap
    cudaEvent_t done_ev = nullptr;
    // pipelined host-buffer builds (lbkd_build_*_host): two device buffer
    // sets alternate, H2D / build / D2H run on three streams
    struct HostPipe {
        float* d_in[2] = {nullptr, nullptr};
        float* d_out[2] = {nullptr, nullptr};
        u32* d_perm[2] = {nullptr, nullptr};
        uint8_t* d_dims[2] = {nullptr, nullptr};
        size_t cap = 0;    // capacity of d_in / d_out in floats (n * k)
        size_t cap_n = 0;  // capacity of d_perm / d_dims in points
        cudaStream_t s_h2d = nullptr, s_build = nullptr, s_d2h = nullptr;
        cudaEvent_t start = nullptr, h2d_done[2], build_done[2], d2h_done[2];
        int slot = 0, pending = 0;
    } hp;
    size_t cap_cand = 0, cap_ptiles = 0, cap_piv = 0;
    int pair_levels = 1;  // round robin: global levels two per partition (LBKD_PAIR=0: one)
    int w_par_end = 0;  // W buffer holding the data after the global levels (level pairs shift it)
    // grow-only device allocations
    size_t cap_n = 0, cap_seg = 0, cap_tiles = 0, cap_w = 0, cap_copy = 0;
    Buffers bf{};
    float* pts_copy = nullptr;
    u32* perm_scratch = nullptr;
    uint8_t* dims_scratch = nullptr;
    u32* minmax = nullptr;
    u32* h_err = nullptr;  // pinned
    // profiling (lbkd_set_profile): CUDA events around every kernel launch
    // of a build, its kernel class and its algorithmic HBM bytes
    int profile = 0;
    std::vector<cudaEvent_t> ev;
    std::vector<int> ev_cls;
    std::vector<double> ev_bytes;
    int n_ev_used = 0;
    u64* d_moved = nullptr;
    int k_last = 0;
    // float64 builds (rank64.cu): rank scratch, rank-coded points, the float32
    // build's output, the widest value table; cur_wt is handed to build()
    u32* rank_scratch = nullptr;
    size_t cap_rank = 0;
    float* codes = nullptr;
    float* out32 = nullptr;
    size_t cap_codes = 0;
    double* vtab = nullptr;
    size_t cap_vtab = 0;
    double* out64_tmp = nullptr;
    size_t cap_out64 = 0;
    u32* f64_err = nullptr;
    WidthTab cur_wt{};
};

// kernel classes of the profile (lbkd_profile_kernel)
enum { kPInit = 0, kPHist, kPPick, kPFilter, kPSelect, kPPart, kPSubtree, kPSortPass, kPOther, kPClasses };

static void prof_record(cudaEvent_t e, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
    else cudaEventRecord(e, st);
}

// open / close a profiled launch: events on the build stream around it
static int prof_begin(lbkd_ctx* c, cudaStream_t st) {
    if (!c->profile) return 0;
    while ((int)c->ev.size() < c->n_ev_used + 2) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return 1;
        c->ev.push_back(e);
    }
    // external record: inside a stream capture the event becomes a real
    // event-record node of the graph, so a replayed graph times its kernels
    // back to back (no host launch gaps inside the brackets); the flag is
    // only legal while capturing (ungraphed builds: sort path, value tables)
    prof_record(c->ev[c->n_ev_used], st);
    return 0;
}
static void prof_end(lbkd_ctx* c, cudaStream_t st, int cls, double bytes) {
    c->launches += 1;
    if (!c->profile) return;
    prof_record(c->ev[c->n_ev_used + 1], st);
    const int i = c->n_ev_used / 2;
    if ((int)c->ev_cls.size() <= i) {
        c->ev_cls.resize(i + 1);
        c->ev_bytes.resize(i + 1);
    }
    c->ev_cls[i] = cls;
    c->ev_bytes[i] = bytes;
    c->n_ev_used += 2;
}

static int choose_bits_default(int k, int mode);

// subtree capacity bits: M = 2^b - 1 points per CTA (lam0 = L - b); env
// LBKD_SUBTREE_BITS lowers it (tuning experiments)
static int choose_bits(int k, int mode) {
    int b = choose_bits_default(k, mode);
    const char* e = getenv("LBKD_SUBTREE_BITS");
    if (e && b > 0) {
        const int want = atoi(e);
        if (want >= 9 && want < b) b = want;
    }
    return b;
}

static int choose_bits_default(int k, int mode) {
    const size_t limit = 227 * 1024 - 256;  // one CTA per SM (general / trace kernel)
    const size_t two = 113 * 1024;           // two CTAs per SM
    const size_t four = 56 * 1024;           // four CTAs per SM
    // round-robin: presorted-list kernel, 2 CTAs/SM (b <= 12); widest k <= 4:
    // selection kernel, 4 CTAs/SM (b <= 11); widest k > 4: general kernel.
    // Every kernel that may run for (b, k, mode) must fit.
    const bool wsel = mode == kWidest && k <= 4;
    for (int b = wsel ? 11 : 12; b >= 9; --b) {
        if (subtree_smem_bytes(b, k, mode) > limit) continue;
        if (mode == kRoundRobin && subtree_rr_smem_bytes(b, k) > two) continue;
        if (subtree_sel_smem_bytes(b, k) > (wsel ? four : limit)) continue;
        return b;
    }
    return -1;
}

#define CK(x)                                  \
    do {                                       \
        cudaError_t e_ = (x);                  \
        if (e_ != cudaSuccess) {               \
            note_cuda(e_);                     \
            return LBKD_ECUDA;                 \
        }                                      \
    } while (0)

static void drop_graph(lbkd_ctx* c);
static thread_local lbkd_ctx* g_grow_ctx = nullptr;  // the context whose buffers grow() reallocates

template <typename T>
static int grow(T*& p, size_t& cap_unused, size_t count) {
    (void)cap_unused;
    if (g_grow_ctx) drop_graph(g_grow_ctx);  // captured graphs point at the old buffers
    if (p) cudaFree(p);
    p = nullptr;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T) + 256);
    if (e != cudaSuccess) {
        note_cuda(e);
        p = nullptr;
        return LBKD_ENOMEM;
    }
    return LBKD_OK;
}

static void drop_graph(lbkd_ctx* c) {
    for (auto& e : c->graphs) {
        if (e.exec) cudaGraphExecDestroy(e.exec);
        e = lbkd_ctx::GraphEntry{};
    }
}

// need_w = false: the caller supplies both working-set buffers (build_split)
static int ensure(lbkd_ctx* c, u64 n, int k, int b, int lam0, bool need_w_bufs = true) {
    g_grow_ctx = c;
    size_t dummy = 0;
    int rc;
    // W[2] holds k+1 SoA arrays of n words each (only when global levels run)
    const size_t stride = (n + 3) & ~(size_t)3;  // 16-byte aligned arrays
    size_t need_w = lam0 > 0 && need_w_bufs ? (size_t)(k + 1) * stride : 0;
    if (need_w > c->cap_w) {
        for (int i = 0; i < 2; ++i)
            if ((rc = grow(c->bf.w[i], dummy, need_w))) return rc;
        c->cap_w = need_w;
    }
    c->bf.stride = stride;
    if (n > c->cap_n) {
        if ((rc = grow(c->perm_scratch, dummy, n))) return rc;
        if ((rc = grow(c->dims_scratch, dummy, n))) return rc;
        c->cap_n = n;
    }
    size_t nseg = (size_t)1 << (lam0 > 0 ? lam0 : 0);
    if (nseg > c->cap_seg) {
        if ((rc = grow(c->bf.hist, dummy, nseg * 1024))) return rc;
        if ((rc = grow(c->bf.seg_and, dummy, nseg))) return rc;
        if ((rc = grow(c->bf.seg_or, dummy, nseg))) return rc;
        for (int i = 0; i < 2; ++i) {
            if ((rc = grow(c->bf.boxes[i], dummy, nseg * 2 * (size_t)LBKD_MAX_K))) return rc;
            if ((rc = grow(c->bf.bmode[i], dummy, nseg))) return rc;
            if ((rc = grow(c->bf.state[i], dummy, nseg))) return rc;
        }
        c->cap_seg = nseg;
    }
    if (lam0 > 0 && c->algo == 0) {
        const size_t rec = (size_t)(k + 2) * n;
        if (rec > c->cap_cand) {
            if ((rc = grow(c->bf.cand, dummy, rec))) return rc;
            if ((rc = grow(c->bf.cand2, dummy, rec))) return rc;
            c->cap_cand = rec;
        }
        const size_t pv = nseg * (size_t)(LBKD_MAX_K + 1);
        if (pv > c->cap_piv) {
            if ((rc = grow(c->bf.piv, dummy, pv))) return rc;
            if ((rc = grow(c->bf.chains, dummy, nseg))) return rc;
            if ((rc = grow(c->bf.sel, dummy, nseg * kSelW))) return rc;
            if ((rc = grow(c->bf.ppos, dummy, nseg))) return rc;
            if ((rc = grow(c->bf.piv2, dummy, pv))) return rc;
            if ((rc = grow(c->bf.chains2, dummy, nseg))) return rc;
            if ((rc = grow(c->bf.ppos2, dummy, nseg))) return rc;
            c->cap_piv = pv;
        }
        const size_t pt = 2 * (n / 256 + 16);  // per 256-position subtile (tiles are coarser)
        if (pt > c->cap_ptiles) {
            if ((rc = grow(c->bf.tile_lt, dummy, pt))) return rc;
            if ((rc = grow(c->bf.sub_lt, dummy, pt))) return rc;
            if ((rc = grow(c->bf.tile_lt2, dummy, 2 * pt))) return rc;
            if ((rc = grow(c->bf.sub_lt2, dummy, 2 * pt))) return rc;
            c->cap_ptiles = pt;
        }
    }
    size_t T = (size_t)1 << (b - 1);
    size_t tiles = (n + T - 1) / T + 1;
    if (tiles > c->cap_tiles) {
        if ((rc = grow(c->bf.status, dummy, tiles * 256))) return rc;
        // status words are epoch-tagged; zero once so no stale word can match
        CK(cudaMemset(c->bf.status, 0, tiles * 256 * sizeof(u64)));
        c->cap_tiles = tiles;
    }
    if (!c->bf.tile_ctr) {
        if ((rc = grow(c->bf.tile_ctr, dummy, 4 * 64))) return rc;
        if ((rc = grow(c->d_moved, dummy, 256))) return rc;
        if ((rc = grow(c->bf.err, dummy, 4))) return rc;
        if ((rc = grow(c->err_host, dummy, 4))) return rc;
        CK(cudaMemset(c->err_host, 0, 4 * sizeof(u32)));
        if ((rc = grow(c->bf.cand_ctr, dummy, 4))) return rc;
        if ((rc = grow(c->minmax, dummy, 2 * LBKD_MAX_K))) return rc;
        if (!c->h_err) CK(cudaMallocHost(&c->h_err, sizeof(u32) * 4));
    }
    return LBKD_OK;
}

// number of points in the segments of level l of the view (the view minus
// the finished nodes between its segments)
static u64 level_points(const BuildParams& bp, int l) {
    const LevelGeom g = view_of(bp, l);
    return g.nview - (g.nseg - 1);
}

// sort path: the global levels [lfrom, lto) of the view bp (hist -> plan ->
// up to four digit passes -> pivots [-> widest child dims])
static int run_levels_sort(lbkd_ctx* c, const BuildParams& bp, int lfrom, int lto, cudaStream_t st) {
    Buffers& bf = c->bf;
    for (int l = lfrom; l < lto; ++l) {
        const u64 nseg = 1ull << (l - bp.lroot);
        const double pts = (double)level_points(bp, l);
        CK(cudaMemsetAsync(bf.hist, 0, nseg * 1024 * sizeof(u32), st));
        CK(cudaMemsetAsync(bf.seg_and, 0xff, nseg * sizeof(u32), st));
        CK(cudaMemsetAsync(bf.seg_or, 0, nseg * sizeof(u32), st));
        if (prof_begin(c, st)) return LBKD_ECUDA;
        launch_hist(bp, bf, l, st);
        prof_end(c, st, kPHist, 4.0 * pts);
        if (prof_begin(c, st)) return LBKD_ECUDA;
        launch_plan(bp, bf, l, st);
        prof_end(c, st, kPOther, 0.0);
        for (int p = 0; p < 4; ++p) {
            if (prof_begin(c, st)) return LBKD_ECUDA;
            const int slot = c->ctr % 256;
            launch_pass(bp, bf, l, p, c->epoch, bf.tile_ctr + slot, c->profile ? c->d_moved + slot : nullptr, st);
            ++c->ctr;
            // bytes: each reordered point reads + writes k coords + index,
            // counted on the device (resolved in lbkd_profile_read)
            prof_end(c, st, kPSortPass, -1.0 - slot);
            c->epoch = (c->epoch + 1) & 0x3fffffffu;
            if (c->epoch == 0) c->epoch = 1;
        }
        if (prof_begin(c, st)) return LBKD_ECUDA;
        launch_pivots(bp, bf, l, st);
        prof_end(c, st, kPOther, 0.0);
        if (bp.mode == kWidest) {
            if (prof_begin(c, st)) return LBKD_ECUDA;
            launch_widest_nodes(bp, l, bf.boxes[l & 1], bf.boxes[(l + 1) & 1], st);
            prof_end(c, st, kPOther, 0.0);
        }
    }
    return LBKD_OK;
}

// select path: the global levels [lfrom, lto) of the view bp -- per level
// hist -> pick -> filter -> select -> partition (select.cu).  Level pairs
// (bp.pair: round robin, 2 <= k <= 4): after level l's select, its children
// are selected in the level-l layout (child hist -> pick -> filter pair ->
// select) and ONE partition pass moves every point to its grandchild's run.
static int run_levels_select(lbkd_ctx* c, const BuildParams& bp, int lfrom, int lto, cudaStream_t st) {
    Buffers& bf = c->bf;
    const int k = bp.k;
    const double A = 4.0 * (k + 1);
    // from level kFuseFrom on (k <= 4) each level's histogram (D = 9; 8 after
    // a pair) is accumulated by the previous partition kernel (widest: binned
    // in each child's own split dim, written by the select kernel)
    const int kFuseFrom = 6;
    const bool fusable = k <= 4 && (bp.mode == kRoundRobin || getenv("LBKD_FUSE_WIDEST") == nullptr ||
                                    getenv("LBKD_FUSE_WIDEST")[0] != '0');
    // (widest pairs are exact too -- the kernels take each node's split dim --
    // but measured slower on config 5: 34.7 vs 33.3 ms, LBKD_PAIR_WIDEST=1)
    static const bool pair_widest = getenv("LBKD_PAIR_WIDEST") && getenv("LBKD_PAIR_WIDEST")[0] == '1';
    const bool pairs = bp.pair && k >= 2 && k <= 4 && (bp.mode == kRoundRobin || (pair_widest && fusable));
    u32 wpar = 0;       // W[wpar] holds level l's data
    int fused_D = 0;    // D of the histogram the previous partition fused (0: none)
    const u64 T = (u64)sel_tile(bp.b);
    auto base_args = [&](const LevelGeom& g, int D, u32 bpar) {
        SelArgs a;
        memset(&a, 0, sizeof(a));
        a.g = g;
        a.k = k;
        a.mode = bp.mode;
        a.wt = bp.wt;
        a.D = D;
        a.bf = bf;
        a.par = wpar;
        a.hist = bf.hist;
        a.sel = bf.sel;
        a.cand = bf.cand;
        a.cand2 = bf.cand2;
        a.cand_ctr = bf.cand_ctr;
        a.piv = bf.piv;
        a.chains = bf.chains;
        a.split_dims = bp.split_dims;
        a.perm = bp.perm;
        a.out_pts = bp.out_pts;
        a.boxes_in = bf.boxes[bpar];
        a.boxes_out = bf.boxes[bpar ^ 1];
        a.bmode_in = bf.bmode[bpar];
        a.bmode_out = bf.bmode[bpar ^ 1];
        a.tile_lt = bf.tile_lt;
        a.sub_lt = bf.sub_lt;
        a.ppos = bf.ppos;
        return a;
    };
    for (int l = lfrom; l < lto;) {
        const LevelGeom g = view_of(bp, l);
        const u64 nseg = g.nseg;
        const bool pair = pairs && l + 1 < lto;
        const int lnext = l + (pair ? 2 : 1);
        static const bool pair_nofuse = getenv("LBKD_PAIR_NOFUSE") && getenv("LBKD_PAIR_NOFUSE")[0] == '1';
        const bool fuse_next = fusable && lnext < lto && lnext >= kFuseFrom && !(pair && pair_nofuse);
        const int D = fused_D ? fused_D : sel_digit_bits(nseg);
        const u32 bpar = (u32)((l - bp.lroot) & 1);  // boxes / bucket modes alternate per level
        const double pts = (double)level_points(bp, l);
        if (!fused_D) CK(cudaMemsetAsync(bf.hist, 0, (nseg << D) * sizeof(u32), st));
        CK(cudaMemsetAsync(bf.cand_ctr, 0, sizeof(u32), st));
        const u64 ntl = (g.nview + T - 1) / T;  // per-tile below-pivot counts accumulate atomically in the filter
        CK(cudaMemsetAsync(bf.tile_lt, 0, 2 * ntl * sizeof(u32), st));
        SelArgs a = base_args(g, D, bpar);
        if (l == lfrom) CK(cudaMemsetAsync(bf.bmode[bpar], 0, nseg, st));  // the view root: value-linear
        if (!fused_D) {
            if (prof_begin(c, st)) return LBKD_ECUDA;
            launch_sel_hist(a, bp.b, st);
            prof_end(c, st, kPHist, 4.0 * pts);
        }
        if (prof_begin(c, st)) return LBKD_ECUDA;
        launch_sel_pick(a, st);
        prof_end(c, st, kPPick, 4.0 * (double)(nseg << D));
        if (prof_begin(c, st)) return LBKD_ECUDA;
        launch_sel_filter(a, bp.b, st);
        prof_end(c, st, kPFilter, 4.0 * pts);
        if (prof_begin(c, st)) return LBKD_ECUDA;
        launch_sel_select(a, bp.b, st);
        prof_end(c, st, kPSelect, 0.0);
        if (!pair) {
            a.hist_next = nullptr;
            if (fuse_next) {  // this level's histogram has been read by pick
                CK(cudaMemsetAsync(bf.hist, 0, (2 * nseg * 512) * sizeof(u32), st));  // 2 children x 2^kFuseD
                a.hist_next = bf.hist;
            }
            if (prof_begin(c, st)) return LBKD_ECUDA;
            launch_sel_part(a, bp.b, st);
            // reads every point of the level, writes all but the nodes
            prof_end(c, st, kPPart, A * (2.0 * pts - (double)nseg));
            fused_D = fuse_next ? 9 : 0;  // 9 = kFuseD (select.cu)
        } else {
            // ---- level l + 1, its segments still in the level-l layout ----
            const LevelGeom g1 = view_of(bp, l + 1);
            const int D1 = sel_digit_bits(g1.nseg) > 9 ? sel_digit_bits(g1.nseg) : 9;
            SelArgs b = base_args(g1, D1, bpar ^ 1);
            b.pair = 1;
            b.g0 = g;
            b.piv = bf.piv2;
            b.chains = bf.chains2;
            b.ppos = bf.ppos2;
            b.piv0 = bf.piv;
            b.chains0 = bf.chains;
            b.ppos0 = bf.ppos;
            b.tile_lt = bf.tile_lt2;
            b.sub_lt = bf.sub_lt2;
            b.lt_tstride = 2 * ntl;
            b.lt_sstride = 2 * ntl * (T / 256);  // 256-position warp subtiles (select.cu kSub)
            b.tile_lt0 = bf.tile_lt;
            b.sub_lt0 = bf.sub_lt;
            CK(cudaMemsetAsync(bf.hist, 0, (g1.nseg << D1) * sizeof(u32), st));
            CK(cudaMemsetAsync(bf.cand_ctr, 0, sizeof(u32), st));
            CK(cudaMemsetAsync(bf.tile_lt2, 0, 2 * b.lt_tstride * sizeof(u32), st));
            if (prof_begin(c, st)) return LBKD_ECUDA;
            launch_sel_child_hist(b, bp.b, st);
            prof_end(c, st, kPHist, 8.0 * pts);
            if (prof_begin(c, st)) return LBKD_ECUDA;
            launch_sel_pick(b, st);
            prof_end(c, st, kPPick, 4.0 * (double)(g1.nseg << D1));
            if (prof_begin(c, st)) return LBKD_ECUDA;
            launch_sel_filter_pair(b, bp.b, st);
            prof_end(c, st, kPFilter, 8.0 * pts);
            if (prof_begin(c, st)) return LBKD_ECUDA;
            launch_sel_select(b, bp.b, st);
            prof_end(c, st, kPSelect, 0.0);
            b.hist_next = nullptr;
            // the fused level-(l+2) histogram: 2^fd bins per grandchild (9:
            // the partition's ring has 2 stages so the bins fit; LBKD_PAIR_FD)
            static const int pair_fd = [] {
                const char* e = getenv("LBKD_PAIR_FD");
                return e && atoi(e) == 8 ? 8 : 9;
            }();
            b.fuse_d = pair_fd;
            if (fuse_next) {  // 4 grandchildren x 2^fd per parent
                CK(cudaMemsetAsync(bf.hist, 0, (4 * nseg << pair_fd) * sizeof(u32), st));
                b.hist_next = bf.hist;
            }
            if (prof_begin(c, st)) return LBKD_ECUDA;
            launch_sel_part_pair(b, bp.b, st);
            // reads every point of level l, writes all but its nodes and their children's
            prof_end(c, st, kPPart, A * (2.0 * pts - 3.0 * (double)nseg));
            fused_D = fuse_next ? pair_fd : 0;
        }
        wpar ^= 1u;
        l = lnext;
    }
    c->w_par_end = (int)wpar;
    return LBKD_OK;
}

static int run_levels(lbkd_ctx* c, const BuildParams& bp, int lfrom, int lto, cudaStream_t st) {
    // the digit-pass tiles (512 x items) need segments of >= 2^9 - 1 points
    if (c->algo != 0 && lto > lfrom && bp.b < 10) return LBKD_EUNSUPPORTED;
    return c->algo == 0 ? run_levels_select(c, bp, lfrom, lto, st) : run_levels_sort(c, bp, lfrom, lto, st);
}

// the in-CTA levels from lam0 on
static int run_subtrees(lbkd_ctx* c, const BuildParams& bp, int lam0, cudaStream_t st) {
    if (prof_begin(c, st)) return LBKD_ECUDA;
    const int entry_sorted = c->algo != 0 || lam0 == 0;
    const int src_par = c->algo != 0 ? -1 : (bp.pair ? c->w_par_end : ((lam0 - bp.lroot) & 1));
    launch_subtree(bp, c->bf, lam0, entry_sorted, src_par, st);
    // each point of the subtrees is read once (k coords + index) and written
    // once to its level-order slot (k coords + perm)
    const u64 pts = lam0 == 0 ? bp.n : level_points(bp, lam0);
    prof_end(c, st, kPSubtree, 8.0 * (bp.k + 1) * (double)pts);
    return LBKD_OK;
}

static int begin_build(lbkd_ctx* c, int k, cudaStream_t st) {
    Buffers& bf = c->bf;
    CK(cudaMemsetAsync(bf.tile_ctr, 0, sizeof(u32) * 4 * 64, st));
    if (c->profile) {
        CK(cudaMemsetAsync(c->d_moved, 0, sizeof(u64) * 256, st));
        c->n_ev_used = 0;
    }
    c->k_last = k;
    c->ctr = 0;
    if (!c->err_sticky) CK(cudaMemsetAsync(bf.err, 0, sizeof(u32) * 4, st));
    else CK(cudaMemsetAsync(bf.err + 1, 0, sizeof(u32), st));  // (the abort word is per build)
    return LBKD_OK;
}

// order this build after the previous one on the context (shared scratch)
static int begin_order(lbkd_ctx* c, cudaStream_t st) {
    if (!c->done_ev) CK(cudaEventCreateWithFlags(&c->done_ev, cudaEventDisableTiming));
    else CK(cudaStreamWaitEvent(st, c->done_ev, 0));
    return LBKD_OK;
}

static int end_build(lbkd_ctx* c, cudaStream_t st) {
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->done_ev, st));
    if (c->check) {
        CK(cudaMemcpyAsync(c->h_err, c->bf.err, sizeof(u32), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (c->h_err[0]) return LBKD_ENONFINITE;
    }
    return LBKD_OK;
}

static int check_args(lbkd_ctx* c, int64_t n_in, int k, int mode) {
    if (!c || n_in < 0 || k < 1 || k > LBKD_MAX_K) return LBKD_EINVAL_SHAPE;
    if (n_in > 0x7fffffffll) return LBKD_ECAPACITY;
    if (mode == kWidest) {
        int db = bit_length((u64)(k - 1));
        if ((n_in << db) > 0x7fffffffll) return LBKD_ECAPACITY;
    }
    return LBKD_OK;
}

// input -> working set W[0] (global levels) and the root's key range /
// widest world box and root dim
static int prologue(lbkd_ctx* c, const BuildParams& bp, int lam0, cudaStream_t st) {
    const int k = bp.k;
    const double pts = (double)bp.n;
    if (lam0 > 0 && c->algo == 0) {
        CK(cudaMemsetAsync(c->minmax, 0xff, sizeof(u32) * k, st));
        CK(cudaMemsetAsync(c->minmax + k, 0, sizeof(u32) * k, st));
        if (prof_begin(c, st)) return LBKD_ECUDA;
        launch_init_stats(bp, c->bf, c->minmax, st);
        prof_end(c, st, kPInit, pts * (4.0 * k + 4.0 * (k + 1)));
        if (prof_begin(c, st)) return LBKD_ECUDA;
        launch_root(bp, c->bf, c->minmax, st);
        prof_end(c, st, kPOther, 0.0);
        return LBKD_OK;
    }
    if (lam0 == 0) {  // no init pass: check the caller's array directly
        if (prof_begin(c, st)) return LBKD_ECUDA;
        launch_check_finite(bp.pts, bp.n * (u64)k, c->bf.err, st);
        prof_end(c, st, kPOther, pts * 4.0 * k);
    }
    if (bp.mode == kWidest) {
        CK(cudaMemsetAsync(c->minmax, 0xff, sizeof(u32) * k, st));
        CK(cudaMemsetAsync(c->minmax + k, 0, sizeof(u32) * k, st));
        if (prof_begin(c, st)) return LBKD_ECUDA;
        launch_world_bounds(bp, c->minmax, st);
        prof_end(c, st, kPOther, pts * 4.0 * k);
        if (prof_begin(c, st)) return LBKD_ECUDA;
        launch_widest_root(bp, c->minmax, c->bf.boxes[0], st);
        prof_end(c, st, kPOther, 0.0);
    }
    if (lam0 > 0) {
        if (prof_begin(c, st)) return LBKD_ECUDA;
        launch_init(bp, c->bf, st);
        prof_end(c, st, kPInit, pts * (4.0 * k + 4.0 * (k + 1)));
    }
    return LBKD_OK;
}

static int build(lbkd_ctx* c, const float* d_points, float* d_out, int64_t n_in, int k, u32* d_perm,
                 uint8_t* d_dims, u32* d_trace, int mode, cudaStream_t st) {
    int rc = check_args(c, n_in, k, mode);
    if (rc) return rc;
    c->launches = 0;
    if (n_in == 0) return LBKD_OK;
    if (!d_points || !d_out) return LBKD_EINVAL_SHAPE;
    CK(cudaSetDevice(c->device));
    const u64 n = (u64)n_in;
    const int b = choose_bits(k, mode);
    if (b < 0) return LBKD_EINVAL_SHAPE;
    const int L = bit_length(n);
    const int lam0 = L - b > 0 ? L - b : 0;
    if (d_trace && lam0 > 0) return LBKD_EUNSUPPORTED;
    const bool inplace = (const void*)d_points == (const void*)d_out;
    rc = ensure(c, n, k, b, lam0);
    if (rc) return rc;
    if ((rc = begin_order(c, st))) return rc;

    BuildParams bp;
    bp.n = n;
    bp.k = k;
    bp.mode = mode;
    bp.b = b;
    bp.pts = d_points;
    // the global levels read the input only in init (into W), so in-place
    // reordering needs a private copy only for single-CTA builds
    if (inplace && lam0 == 0) {
        if ((u64)k * n > c->cap_copy) {
            size_t dummy = 0;
            if ((rc = grow(c->pts_copy, dummy, (size_t)k * n))) return rc;
            c->cap_copy = (u64)k * n;
        }
        CK(cudaMemcpyAsync(c->pts_copy, d_points, n * (u64)k * sizeof(float), cudaMemcpyDeviceToDevice, st));
        bp.pts = c->pts_copy;
    }
    bp.out_pts = d_out;
    bp.perm = d_perm ? d_perm : c->perm_scratch;
    bp.split_dims = d_dims ? d_dims : c->dims_scratch;
    bp.dbg = d_trace;
    bp.wt = c->cur_wt;
    bp.subtree_sel = c->subtree_sel >= 0 ? c->subtree_sel : (mode == kWidest ? 1 : 0);
    bp.pair = c->pair_levels && c->algo == 0 && !d_trace;
    // the select path is a fixed, host-sync-free sequence for given buffers:
    // capture it once into a CUDA graph and replay it (the sort path carries
    // per-launch lookback epochs and is always launched directly)
    // (value-table builds carry their table in the kernel arguments: never graphed)
    // (profiled builds are graphed too: their event brackets are event-record
    // nodes, and a replay times the kernels of THAT replay)
    const bool graphable = c->use_graph && c->algo == 0 && !d_trace && bp.pts == d_points && !bp.wt.v;
    lbkd_ctx::GraphKey key{d_points, d_out, d_perm, d_dims, c->bf.err, n_in, k, mode, c->algo, bp.subtree_sel, c->check,
                           c->profile};
    lbkd_ctx::GraphEntry* hit = nullptr;
    lbkd_ctx::GraphEntry* victim = &c->graphs[0];
    for (auto& e : c->graphs) {
        if (e.exec && e.key == key) hit = &e;
        if (!e.exec || (victim->exec && e.used < victim->used)) victim = &e;
    }
    if (graphable && hit) {
        hit->used = ++c->graph_tick;
        CK(cudaGraphLaunch(hit->exec, st));
        c->launches = hit->launches;
        c->n_ev_used = hit->n_ev;
        c->k_last = k;
        return end_build(c, st);
    }
    if (graphable) {
        if (!c->cap_stream) {
            CK(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&c->cap_fork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->cap_join, cudaEventDisableTiming));
        }
        if (victim->exec) {
            cudaGraphExecDestroy(victim->exec);
            *victim = lbkd_ctx::GraphEntry{};
        }
        cudaGraph_t graph = nullptr;
        CK(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
        int r2 = begin_build(c, k, c->cap_stream);
        if (!r2) r2 = prologue(c, bp, lam0, c->cap_stream);
        if (!r2) r2 = run_levels(c, bp, 0, lam0, c->cap_stream);
        if (!r2) r2 = run_subtrees(c, bp, lam0, c->cap_stream);
        const cudaError_t ce = cudaStreamEndCapture(c->cap_stream, &graph);
        if (r2) {
            if (graph) cudaGraphDestroy(graph);
            return r2;
        }
        CK(ce);
        const cudaError_t ie = cudaGraphInstantiate(&victim->exec, graph, 0);
        cudaGraphDestroy(graph);
        CK(ie);
        victim->key = key;
        victim->launches = c->launches;
        victim->n_ev = c->n_ev_used;
        victim->used = ++c->graph_tick;
        CK(cudaGraphLaunch(victim->exec, st));
        return end_build(c, st);
    }
    if ((rc = begin_build(c, k, st))) return rc;
    if ((rc = prologue(c, bp, lam0, st))) return rc;
    if ((rc = run_levels(c, bp, 0, lam0, st))) return rc;
    if ((rc = run_subtrees(c, bp, lam0, st))) return rc;
    return end_build(c, st);
}

// float64 input (rank64.cu): per-dimension dense ranks coded as float32,
// the float32 build, then the float64 rows gathered by the permutation
static int build_f64(lbkd_ctx* c, const double* d_points, double* d_out, int64_t n_in, int k, u32* d_perm,
                     uint8_t* d_dims, u32* d_trace, int mode, cudaStream_t st) {
    int rc = check_args(c, n_in, k, mode);
    if (rc) return rc;
    c->launches = 0;
    if (n_in == 0) return LBKD_OK;
    if (!d_points || !d_out) return LBKD_EINVAL_SHAPE;
    CK(cudaSetDevice(c->device));
    const u64 n = (u64)n_in;
    g_grow_ctx = c;
    size_t dummy = 0;
    const size_t rw = rank_scratch_words(n);
    if (rw > c->cap_rank) {
        if ((rc = grow(c->rank_scratch, dummy, rw))) return rc;
        c->cap_rank = rw;
    }
    if (n * (u64)k > c->cap_codes) {
        if ((rc = grow(c->codes, dummy, n * (size_t)k))) return rc;
        if ((rc = grow(c->out32, dummy, n * (size_t)k))) return rc;
        c->cap_codes = n * (size_t)k;
    }
    if (mode == kWidest && n * (u64)k > c->cap_vtab) {
        if ((rc = grow(c->vtab, dummy, n * (size_t)k))) return rc;
        c->cap_vtab = n * (size_t)k;
    }
    if (!c->f64_err && (rc = grow(c->f64_err, dummy, 4))) return rc;
    if (!c->h_err) CK(cudaMallocHost(&c->h_err, sizeof(u32) * 4));
    if ((rc = begin_order(c, st))) return rc;
    CK(cudaMemsetAsync(c->f64_err, 0, 4 * sizeof(u32), st));
    WidthTab wt{};
    wt.stride = n;
    wt.v = mode == kWidest ? c->vtab : nullptr;
    for (int d = 0; d < k; ++d) {
        if ((rc = rank_sort_dim(d_points, n, k, d, c->rank_scratch, c->f64_err, st))) return rc;
        u32* hc = c->h_err + 1;  // pinned
        CK(cudaMemcpyAsync(hc, rank_count_word(c->rank_scratch, n), sizeof(u32), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const u64 distinct = (u64)*hc + 1;
        const int wide = distinct > 2ull * kRankSide - 1;
        wt.wide |= (u32)wide << d;
        wt.center[d] = wide ? 0u : (u32)(distinct / 2);
        if ((rc = rank_assign_dim(n, k, d, wt.center[d], wide, c->codes, wt.v ? c->vtab + (u64)d * n : nullptr,
                                  c->rank_scratch, st)))
            return rc;
    }
    CK(cudaMemcpyAsync(c->h_err, c->f64_err, sizeof(u32), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (c->h_err[0]) return LBKD_ENONFINITE;
    c->cur_wt = wt;
    rc = build(c, c->codes, c->out32, n_in, k, d_perm, d_dims, d_trace, mode, st);
    c->cur_wt = WidthTab{};
    if (rc) return rc;
    const u32* perm = d_perm ? d_perm : c->perm_scratch;
    if ((const void*)d_out == (const void*)d_points) {
        if (n * (u64)k > c->cap_out64) {
            if ((rc = grow(c->out64_tmp, dummy, n * (size_t)k))) return rc;
            c->cap_out64 = n * (size_t)k;
        }
        launch_gather_rows_f64(d_points, perm, n, k, c->out64_tmp, st);
        CK(cudaMemcpyAsync(d_out, c->out64_tmp, n * (size_t)k * sizeof(double), cudaMemcpyDeviceToDevice, st));
    } else {
        launch_gather_rows_f64(d_points, perm, n, k, d_out, st);
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->done_ev, st));
    return LBKD_OK;
}

// multi-device, rank 0: the top `top` levels of the whole tree, then the
// 2^top subtrees' points (k coordinate arrays + index array, in the
// reference's entry order) packed back to back into d_sub
static int build_top(lbkd_ctx* c, const float* d_points, int64_t n_in, int k, int top, float* d_out, u32* d_perm,
                     u32* d_sub, int64_t sub_stride, cudaStream_t st) {
    int rc = check_args(c, n_in, k, kRoundRobin);
    if (rc) return rc;
    c->launches = 0;
    if (!d_points || !d_out || !d_perm || !d_sub || top < 1) return LBKD_EINVAL_SHAPE;
    CK(cudaSetDevice(c->device));
    const u64 n = (u64)n_in;
    const int b = choose_bits(k, kRoundRobin);
    const int L = bit_length(n);
    const int lam0 = L - b > 0 ? L - b : 0;
    if (top > lam0) return LBKD_EUNSUPPORTED;  // tree too small to shard
    if ((u64)sub_stride < n) return LBKD_EINVAL_SHAPE;
    rc = ensure(c, n, k, b, lam0);
    if (rc) return rc;
    BuildParams bp;
    bp.n = n;
    bp.k = k;
    bp.mode = kRoundRobin;
    bp.b = b;
    bp.pts = d_points;
    bp.out_pts = d_out;
    bp.perm = d_perm;
    bp.split_dims = c->dims_scratch;
    bp.dbg = nullptr;
    if ((rc = begin_order(c, st))) return rc;
    if ((rc = begin_build(c, k, st))) return rc;
    if ((rc = prologue(c, bp, lam0, st))) return rc;
    if ((rc = run_levels(c, bp, 0, top, st))) return rc;
    if (prof_begin(c, st)) return LBKD_ECUDA;
    launch_extract(bp, c->bf, top, d_sub, (u64)sub_stride, c->algo == 0 ? (top & 1) : -1, st);  // lroot = 0
    prof_end(c, st, kPOther, 8.0 * (k + 1) * (double)level_points(bp, top));
    return end_build(c, st);
}

// multi-device, rank j: finish the subtree rooted at (root_level, root_index)
// of an n_total-point tree from its points in d_sub (as packed by build_top);
// nodes land at their global level-order slots of d_out / d_perm
// A packed SoA buffer (k + 1 arrays, `stride` words apart) can serve as the
// working set itself when the stride is a multiple of 4 words and the base is
// 16-byte aligned (the bulk copies and 16-byte loads of the global levels)
static bool aliasable(const void* p, int64_t stride) {
    return p && (stride % 4) == 0 && ((uintptr_t)p & 15u) == 0;
}

// Finish the subtree rooted at (root_level, root_index) from its packed
// points (aliased as W[0] -- then overwritten -- when aliasable, else copied)
static int build_sub(lbkd_ctx* c, u32* d_sub, int64_t sub_stride, int64_t n_total, int k, int root_level,
                     int64_t root_index, float* d_out, u32* d_perm, cudaStream_t st) {
    int rc = check_args(c, n_total, k, kRoundRobin);
    if (rc) return rc;
    c->launches = 0;
    if (!d_sub || !d_out || !d_perm || root_level < 0) return LBKD_EINVAL_SHAPE;
    CK(cudaSetDevice(c->device));
    const u64 n = (u64)n_total;
    const int L = bit_length(n);
    if (root_level > L - 1 || (u64)root_index >= (1ull << root_level)) return LBKD_EINVAL_SHAPE;
    const int b = choose_bits(k, kRoundRobin);
    int lam0 = L - b > 0 ? L - b : 0;
    if (lam0 < root_level) lam0 = root_level;
    const LevelGeom gr = make_geom(n, root_level);
    const u64 nview = seg_size(gr, (u64)root_index);
    if ((u64)sub_stride < nview) return LBKD_EINVAL_SHAPE;
    const bool alias = c->algo == 0 && lam0 > root_level && aliasable(d_sub, sub_stride);
    // aliased: the context's W[1] takes the caller's stride
    rc = ensure(c, alias ? (u64)sub_stride : nview, k, b, lam0 - root_level + 1);
    if (rc) return rc;
    BuildParams bp;
    bp.n = n;
    bp.k = k;
    bp.mode = kRoundRobin;
    bp.b = b;
    bp.pts = nullptr;
    bp.out_pts = d_out;
    bp.perm = d_perm;
    bp.split_dims = c->dims_scratch;
    bp.dbg = nullptr;
    bp.lroot = root_level;
    bp.subtree_sel = c->subtree_sel >= 0 ? c->subtree_sel : 0;
    bp.jroot = (u64)root_index;
    bp.pair = c->pair_levels && c->algo == 0;  // (the sub-build's own global levels, two per pass)
    if ((rc = begin_order(c, st))) return rc;
    if ((rc = begin_build(c, k, st))) return rc;
    u32* const own_w0 = c->bf.w[0];
    if (alias) c->bf.w[0] = d_sub;
    else
        CK(cudaMemcpy2DAsync(c->bf.w[0], c->bf.stride * sizeof(u32), d_sub, (size_t)sub_stride * sizeof(u32),
                             nview * sizeof(u32), (size_t)k + 1, cudaMemcpyDeviceToDevice, st));
    struct Restore {
        lbkd_ctx* c;
        u32* w0;
        ~Restore() { c->bf.w[0] = w0; }
    } restore{c, own_w0};
    if (c->algo == 0 && lam0 > root_level) {
        CK(cudaMemsetAsync(c->minmax, 0xff, sizeof(u32) * k, st));
        CK(cudaMemsetAsync(c->minmax + k, 0, sizeof(u32) * k, st));
        if (prof_begin(c, st)) return LBKD_ECUDA;
        launch_view_minmax(bp, c->bf, c->minmax, nview, st);
        prof_end(c, st, kPOther, 4.0 * k * (double)nview);
        if (prof_begin(c, st)) return LBKD_ECUDA;
        launch_root(bp, c->bf, c->minmax, st);
        prof_end(c, st, kPOther, 0.0);
    }
    if ((rc = run_levels(c, bp, root_level, lam0, st))) return rc;
    if ((rc = run_subtrees(c, bp, lam0, st))) return rc;
    return end_build(c, st);
}

// Recursive halving step (multi-device): ONE level of the subtree rooted at
// (root_level, root_index) -- from the raw AoS input at the root, else from
// its packed points used in place as W[0] -- with d_next as W[1]: after it,
// d_next holds the next level's working set in in-order layout, the left
// child's points at [0, ss(2s+1)), the right child's after the node's slot.
// No copies besides the level's own partition.
static int build_split(lbkd_ctx* c, const float* d_points, u32* d_sub, int64_t stride, int64_t n_total, int k,
                       int root_level, int64_t root_index, float* d_out, u32* d_perm, u32* d_next, cudaStream_t st) {
    int rc = check_args(c, n_total, k, kRoundRobin);
    if (rc) return rc;
    c->launches = 0;
    if (!d_out || !d_perm || !d_next || root_level < 0 || c->algo != 0) return LBKD_EINVAL_SHAPE;
    if (root_level == 0 ? !d_points : !d_sub) return LBKD_EINVAL_SHAPE;
    CK(cudaSetDevice(c->device));
    const u64 n = (u64)n_total;
    const int L = bit_length(n);
    if (root_level > L - 1 || (u64)root_index >= (1ull << root_level)) return LBKD_EINVAL_SHAPE;
    const int b = choose_bits(k, kRoundRobin);
    const int lam0 = L - b > 0 ? L - b : 0;
    if (root_level + 1 > lam0) return LBKD_EUNSUPPORTED;  // global levels only
    const u64 nview = seg_size(make_geom(n, root_level), (u64)root_index);
    if ((u64)stride < nview || !aliasable(d_next, stride) || (root_level > 0 && !aliasable(d_sub, stride)))
        return LBKD_EINVAL_SHAPE;
    rc = ensure(c, root_level == 0 ? n : (u64)stride, k, b, lam0 - root_level + 1, root_level == 0);
    if (rc) return rc;
    if (c->bf.stride != (u64)stride) return LBKD_EINVAL_SHAPE;  // root: stride must be ceil4(n)
    BuildParams bp;
    bp.n = n;
    bp.k = k;
    bp.mode = kRoundRobin;
    bp.b = b;
    bp.pts = d_points;
    bp.out_pts = d_out;
    bp.perm = d_perm;
    bp.split_dims = c->dims_scratch;
    bp.dbg = nullptr;
    bp.lroot = root_level;
    bp.jroot = (u64)root_index;
    if ((rc = begin_order(c, st))) return rc;
    if ((rc = begin_build(c, k, st))) return rc;
    struct Restore {
        lbkd_ctx* c;
        u32* w0;
        u32* w1;
        ~Restore() {
            c->bf.w[0] = w0;
            c->bf.w[1] = w1;
        }
    } restore{c, c->bf.w[0], c->bf.w[1]};
    c->bf.w[1] = d_next;
    if (root_level == 0) {
        if ((rc = prologue(c, bp, lam0, st))) return rc;  // AoS -> W[0], root box
    } else {
        c->bf.w[0] = d_sub;
        CK(cudaMemsetAsync(c->minmax, 0xff, sizeof(u32) * k, st));
        CK(cudaMemsetAsync(c->minmax + k, 0, sizeof(u32) * k, st));
        if (prof_begin(c, st)) return LBKD_ECUDA;
        launch_view_minmax(bp, c->bf, c->minmax, nview, st);
        prof_end(c, st, kPOther, 4.0 * k * (double)nview);
        if (prof_begin(c, st)) return LBKD_ECUDA;
        launch_root(bp, c->bf, c->minmax, st);
        prof_end(c, st, kPOther, 0.0);
    }
    if ((rc = run_levels(c, bp, root_level, root_level + 1, st))) return rc;
    return end_build(c, st);
}

// ---------------------------------------------------------------------------
// pipelined builds from / to HOST buffers (pinned for overlap): call i's
// H2D runs while build i-1 computes and D2H of call i-1 drains while build i
// computes; a build only waits for the buffers it reuses
// ---------------------------------------------------------------------------
static int host_pipe_ensure(lbkd_ctx* c, size_t n, int k) {
    auto& h = c->hp;
    g_grow_ctx = c;
    if (!h.s_h2d) {
        CK(cudaStreamCreateWithFlags(&h.s_h2d, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&h.s_build, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&h.s_d2h, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&h.start, cudaEventDisableTiming));
        for (int i = 0; i < 2; ++i) {
            CK(cudaEventCreateWithFlags(&h.h2d_done[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&h.build_done[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&h.d2h_done[i], cudaEventDisableTiming));
            CK(cudaEventRecord(h.build_done[i], h.s_build));
            CK(cudaEventRecord(h.d2h_done[i], h.s_d2h));
        }
    }
    // point buffers grow on n * k, perm / split-dim buffers on n (a later
    // call may have more points and fewer dimensions)
    const size_t need = n * (size_t)k;
    if (need > h.cap || n > h.cap_n) {
        CK(cudaDeviceSynchronize());
        size_t dummy = 0;
        int rc;
        for (int i = 0; i < 2; ++i) {
            if (need > h.cap) {
                if ((rc = grow(h.d_in[i], dummy, need))) return rc;
                if ((rc = grow(h.d_out[i], dummy, need))) return rc;
            }
            if (n > h.cap_n) {
                if ((rc = grow(h.d_perm[i], dummy, n))) return rc;
                if ((rc = grow(h.d_dims[i], dummy, n))) return rc;
            }
        }
        if (need > h.cap) h.cap = need;
        if (n > h.cap_n) h.cap_n = n;
    }
    return LBKD_OK;
}

static int build(lbkd_ctx* c, const float* d_points, float* d_out, int64_t n_in, int k, u32* d_perm,
                 uint8_t* d_dims, u32* d_trace, int mode, cudaStream_t st);

static int build_host(lbkd_ctx* c, const float* h_points, float* h_out, int64_t n_in, int k, u32* h_perm,
                      uint8_t* h_dims, int mode, cudaStream_t st) {
    int rc = check_args(c, n_in, k, mode);
    if (rc) return rc;
    if (n_in == 0) return LBKD_OK;
    if (!h_points || !h_out) return LBKD_EINVAL_SHAPE;
    CK(cudaSetDevice(c->device));
    const size_t n = (size_t)n_in;
    if ((rc = host_pipe_ensure(c, n, k))) return rc;
    auto& h = c->hp;
    const int s = h.slot;
    h.slot ^= 1;
    // fork from the caller's stream
    CK(cudaEventRecord(h.start, st));
    CK(cudaStreamWaitEvent(h.s_h2d, h.start, 0));
    // d_in[s] is free once the build that read it (two calls ago) is done
    CK(cudaStreamWaitEvent(h.s_h2d, h.build_done[s], 0));
    CK(cudaMemcpyAsync(h.d_in[s], h_points, n * k * sizeof(float), cudaMemcpyHostToDevice, h.s_h2d));
    CK(cudaEventRecord(h.h2d_done[s], h.s_h2d));
    CK(cudaStreamWaitEvent(h.s_build, h.h2d_done[s], 0));
    CK(cudaStreamWaitEvent(h.s_build, h.d2h_done[s], 0));  // d_out[s] drained
    // the build writes the pipeline's own non-finite flag, which accumulates
    // until lbkd_host_join (device builds keep theirs in bf.err)
    if (!c->err_host) {
        size_t dummy = 0;
        if ((rc = grow(c->err_host, dummy, 4))) return rc;
        CK(cudaMemset(c->err_host, 0, 4 * sizeof(u32)));
    }
    const int check = c->check;
    u32* const dev_err = c->bf.err;
    c->check = 0;
    c->err_sticky = 1;
    c->bf.err = c->err_host;
    rc = build(c, h.d_in[s], h.d_out[s], n_in, k, h.d_perm[s], h.d_dims[s], nullptr, mode, h.s_build);
    c->bf.err = dev_err;
    c->err_sticky = 0;
    c->check = check;
    if (rc) return rc;
    CK(cudaEventRecord(h.build_done[s], h.s_build));
    CK(cudaStreamWaitEvent(h.s_d2h, h.build_done[s], 0));
    CK(cudaMemcpyAsync(h_out, h.d_out[s], n * k * sizeof(float), cudaMemcpyDeviceToHost, h.s_d2h));
    if (h_perm) CK(cudaMemcpyAsync(h_perm, h.d_perm[s], n * sizeof(u32), cudaMemcpyDeviceToHost, h.s_d2h));
    if (h_dims && mode == kWidest)
        CK(cudaMemcpyAsync(h_dims, h.d_dims[s], n * sizeof(uint8_t), cudaMemcpyDeviceToHost, h.s_d2h));
    CK(cudaEventRecord(h.d2h_done[s], h.s_d2h));
    h.pending = 1;
    return LBKD_OK;
}

// join: the caller's stream waits for every pipelined build; with sync != 0
// also waits on the host and reports non-finite input seen since the last join
static int host_join(lbkd_ctx* c, cudaStream_t st, int sync) {
    auto& h = c->hp;
    if (!h.s_h2d) return LBKD_OK;
    CK(cudaSetDevice(c->device));
    for (int i = 0; i < 2; ++i) CK(cudaStreamWaitEvent(st, h.d2h_done[i], 0));
    if (!sync) return LBKD_OK;
    CK(cudaMemcpyAsync(c->h_err, c->err_host, sizeof(u32), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const u32 e = c->h_err[0];
    CK(cudaMemsetAsync(c->err_host, 0, sizeof(u32) * 4, st));
    CK(cudaStreamSynchronize(st));
    h.pending = 0;
    return e ? LBKD_ENONFINITE : LBKD_OK;
}

extern "C" {

int lbkd_build_rr_host(lbkd_ctx* c, const float* h_points, float* h_out, int64_t n, int k, uint32_t* h_perm,
                       void* stream) {
    return build_host(c, h_points, h_out, n, k, h_perm, nullptr, kRoundRobin, (cudaStream_t)stream);
}

int lbkd_build_widest_host(lbkd_ctx* c, const float* h_points, float* h_out, int64_t n, int k, uint32_t* h_perm,
                           uint8_t* h_split_dims, void* stream) {
    return build_host(c, h_points, h_out, n, k, h_perm, h_split_dims, kWidest, (cudaStream_t)stream);
}

int lbkd_host_join(lbkd_ctx* c, void* stream, int sync) { return c ? host_join(c, (cudaStream_t)stream, sync) : LBKD_EINVAL_SHAPE; }

int lbkd_create(lbkd_ctx** out, int device) {
    if (!out) return LBKD_EINVAL_SHAPE;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        note_cuda(e);
        return LBKD_ECUDA;
    }
    // Random 4-byte gathers (rekey, subtree load) otherwise pull 128-byte
    // lines from HBM; 32 bytes is one sector.  Streaming kernels are fully
    // coalesced, so the smaller fetch granularity costs them nothing.
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 32);
    lbkd_ctx* c = new lbkd_ctx();
    c->device = device;
    if (const char* e = getenv("LBKD_PAIR")) c->pair_levels = e[0] != '0';
    const char* algo = getenv("LBKD_ALGO");
    if (algo && strcmp(algo, "sort") == 0) c->algo = 1;
    const char* gr = getenv("LBKD_GRAPH");
    if (gr && strcmp(gr, "0") == 0) c->use_graph = 0;
    const char* sub = getenv("LBKD_SUBTREE");
    if (sub && strcmp(sub, "lists") == 0) c->subtree_sel = 0;
    if (sub && strcmp(sub, "sel") == 0) c->subtree_sel = 1;
    *out = c;
    return LBKD_OK;
}

void lbkd_destroy(lbkd_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    for (auto& e : c->graphs)
        if (e.exec) cudaGraphExecDestroy(e.exec);
    if (c->cap_stream) {
        cudaStreamDestroy(c->cap_stream);
        cudaEventDestroy(c->cap_fork);
        cudaEventDestroy(c->cap_join);
    }
    if (c->hp.s_h2d) {
        cudaDeviceSynchronize();
        for (int i = 0; i < 2; ++i) {
            cudaFree(c->hp.d_in[i]);
            cudaFree(c->hp.d_out[i]);
            cudaFree(c->hp.d_perm[i]);
            cudaFree(c->hp.d_dims[i]);
            cudaEventDestroy(c->hp.h2d_done[i]);
            cudaEventDestroy(c->hp.build_done[i]);
            cudaEventDestroy(c->hp.d2h_done[i]);
        }
        cudaEventDestroy(c->hp.start);
        cudaStreamDestroy(c->hp.s_h2d);
        cudaStreamDestroy(c->hp.s_build);
        cudaStreamDestroy(c->hp.s_d2h);
    }
    for (int i = 0; i < 2; ++i) {
        cudaFree(c->bf.w[i]);
        cudaFree(c->bf.boxes[i]);
        cudaFree(c->bf.bmode[i]);
        cudaFree(c->bf.state[i]);
    }
    cudaFree(c->bf.hist);
    cudaFree(c->bf.sel);
    cudaFree(c->bf.cand);
    cudaFree(c->bf.cand2);
    cudaFree(c->bf.cand_ctr);
    cudaFree(c->bf.piv);
    cudaFree(c->bf.chains);
    cudaFree(c->bf.tile_lt);
    cudaFree(c->bf.sub_lt);
    cudaFree(c->bf.ppos);
    cudaFree(c->bf.piv2);
    cudaFree(c->bf.chains2);
    cudaFree(c->bf.ppos2);
    cudaFree(c->bf.tile_lt2);
    cudaFree(c->bf.sub_lt2);
    cudaFree(c->bf.seg_and);
    cudaFree(c->bf.seg_or);
    cudaFree(c->bf.status);
    cudaFree(c->bf.tile_ctr);
    cudaFree(c->bf.err);
    cudaFree(c->err_host);
    if (c->done_ev) cudaEventDestroy(c->done_ev);
    cudaFree(c->pts_copy);
    cudaFree(c->perm_scratch);
    cudaFree(c->dims_scratch);
    cudaFree(c->minmax);
    cudaFree(c->d_moved);
    cudaFree(c->rank_scratch);
    cudaFree(c->codes);
    cudaFree(c->out32);
    cudaFree(c->vtab);
    cudaFree(c->out64_tmp);
    cudaFree(c->f64_err);
    for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
    if (c->h_err) cudaFreeHost(c->h_err);
    delete c;
}

void lbkd_set_check(lbkd_ctx* c, int check) {
    if (c) c->check = check ? 1 : 0;
}

int lbkd_build_rr(lbkd_ctx* c, const float* d_points, float* d_out, int64_t n, int k, uint32_t* d_perm,
                  void* stream) {
    return build(c, d_points, d_out, n, k, d_perm, nullptr, nullptr, kRoundRobin, (cudaStream_t)stream);
}

int lbkd_build_widest(lbkd_ctx* c, const float* d_points, float* d_out, int64_t n, int k, uint32_t* d_perm,
                      uint8_t* d_dims, void* stream) {
    return build(c, d_points, d_out, n, k, d_perm, d_dims, nullptr, kWidest, (cudaStream_t)stream);
}

int lbkd_build_rr_f64(lbkd_ctx* c, const double* d_points, double* d_out, int64_t n, int k, uint32_t* d_perm,
                      void* stream) {
    return build_f64(c, d_points, d_out, n, k, d_perm, nullptr, nullptr, kRoundRobin, (cudaStream_t)stream);
}

int lbkd_build_widest_f64(lbkd_ctx* c, const double* d_points, double* d_out, int64_t n, int k, uint32_t* d_perm,
                          uint8_t* d_dims, void* stream) {
    return build_f64(c, d_points, d_out, n, k, d_perm, d_dims, nullptr, kWidest, (cudaStream_t)stream);
}

int lbkd_build_rr_f64_trace(lbkd_ctx* c, const double* d_points, double* d_out, int64_t n, int k,
                            uint32_t* d_perm, uint32_t* d_trace, void* stream) {
    if (!d_trace) return LBKD_EINVAL_SHAPE;
    return build_f64(c, d_points, d_out, n, k, d_perm, nullptr, d_trace, kRoundRobin, (cudaStream_t)stream);
}

int lbkd_build_widest_f64_trace(lbkd_ctx* c, const double* d_points, double* d_out, int64_t n, int k,
                                uint32_t* d_perm, uint8_t* d_dims, uint32_t* d_trace, void* stream) {
    if (!d_trace) return LBKD_EINVAL_SHAPE;
    return build_f64(c, d_points, d_out, n, k, d_perm, d_dims, d_trace, kWidest, (cudaStream_t)stream);
}

int lbkd_build_rr_trace(lbkd_ctx* c, const float* d_points, float* d_out, int64_t n, int k, uint32_t* d_perm,
                        uint32_t* d_trace, void* stream) {
    if (!d_trace) return LBKD_EINVAL_SHAPE;
    return build(c, d_points, d_out, n, k, d_perm, nullptr, d_trace, kRoundRobin, (cudaStream_t)stream);
}

int lbkd_build_widest_trace(lbkd_ctx* c, const float* d_points, float* d_out, int64_t n, int k,
                            uint32_t* d_perm, uint8_t* d_dims, uint32_t* d_trace, void* stream) {
    if (!d_trace) return LBKD_EINVAL_SHAPE;
    return build(c, d_points, d_out, n, k, d_perm, d_dims, d_trace, kWidest, (cudaStream_t)stream);
}

int lbkd_build_rr_top(lbkd_ctx* c, const float* d_points, int64_t n, int k, int top_levels, float* d_out,
                      uint32_t* d_perm, uint32_t* d_sub, int64_t sub_stride, void* stream) {
    return build_top(c, d_points, n, k, top_levels, d_out, d_perm, d_sub, sub_stride, (cudaStream_t)stream);
}

int lbkd_build_rr_sub(lbkd_ctx* c, uint32_t* d_sub, int64_t sub_stride, int64_t n_total, int k,
                      int root_level, int64_t root_index, float* d_out, uint32_t* d_perm, void* stream) {
    return build_sub(c, d_sub, sub_stride, n_total, k, root_level, root_index, d_out, d_perm, (cudaStream_t)stream);
}

int lbkd_build_rr_split(lbkd_ctx* c, const float* d_points, uint32_t* d_sub, int64_t stride, int64_t n_total, int k,
                        int root_level, int64_t root_index, float* d_out, uint32_t* d_perm, uint32_t* d_next,
                        void* stream) {
    return build_split(c, d_points, d_sub, stride, n_total, k, root_level, root_index, d_out, d_perm, d_next,
                       (cudaStream_t)stream);
}

int lbkd_update_tags_rr(uint32_t* d_tags, int64_t n, int levels, int l, void* stream) {
    if (!d_tags || n < 1 || l < 0 || l > levels - 2) return LBKD_EINVAL_SHAPE;
    launch_update_tags_rr(d_tags, n, levels, l, (cudaStream_t)stream);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        note_cuda(e);
        return LBKD_ECUDA;
    }
    return LBKD_OK;
}

int lbkd_update_tags_widest(uint32_t* d_tags, const double* d_coords, int k, uint8_t* d_split_dims,
                            const double* d_world_lo, const double* d_world_hi, int64_t n, int levels, int l,
                            int dim_bits, void* stream) {
    if (!d_tags || !d_coords || !d_split_dims || n < 1 || k < 1 || k > LBKD_MAX_K || l < 0 || l > levels - 2)
        return LBKD_EINVAL_SHAPE;
    launch_update_tags_widest(d_tags, d_coords, k, d_split_dims, d_world_lo, d_world_hi, n, levels, l, dim_bits,
                              (cudaStream_t)stream);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        note_cuda(e);
        return LBKD_ECUDA;
    }
    return LBKD_OK;
}

int lbkd_num_levels(int64_t n) { return n > 0 ? bit_length((u64)n) : 0; }

int64_t lbkd_single_cta_capacity(int k, int widest) {
    int b = choose_bits(k, widest ? kWidest : kRoundRobin);
    return b < 0 ? 0 : ((int64_t)1 << b) - 1;
}

int lbkd_plan_info(int64_t n, int k, int widest, int* b_out, int* lam0_out) {
    if (k < 1 || k > LBKD_MAX_K || n < 0) return LBKD_EINVAL_SHAPE;
    int b = choose_bits(k, widest ? kWidest : kRoundRobin);
    int L = n > 0 ? bit_length((u64)n) : 0;
    if (b_out) *b_out = b;
    if (lam0_out) *lam0_out = L - b > 0 ? L - b : 0;
    return LBKD_OK;
}

int64_t lbkd_last_launch_count(const lbkd_ctx* c) { return c ? c->launches : 0; }

void lbkd_set_profile(lbkd_ctx* c, int on) {
    if (c) c->profile = on ? 1 : 0;
}

// per-class totals of the last profiled build (device time from the events,
// algorithmic bytes from the launch geometry or the device counters)
static int profile_class(lbkd_ctx* c, int cls, int* n_out, double* ms_out, double* bytes_out) {
    if (!c) return LBKD_EINVAL_SHAPE;
    const int n = c->n_ev_used / 2;
    int cnt = 0;
    double ms = 0.0, bytes = 0.0;
    if (n > 0) {
        CK(cudaSetDevice(c->device));
        std::vector<u64> moved(256, 0);
        CK(cudaMemcpy(moved.data(), c->d_moved, sizeof(u64) * 256, cudaMemcpyDeviceToHost));
        for (int i = 0; i < n; ++i) {
            if (cls >= 0 && c->ev_cls[i] != cls) continue;
            float t = 0.f;
            CK(cudaEventSynchronize(c->ev[2 * i + 1]));
            CK(cudaEventElapsedTime(&t, c->ev[2 * i], c->ev[2 * i + 1]));
            ms += t;
            ++cnt;
            const double b = c->ev_bytes[i];
            // sort path digit passes: every reordered point reads and writes
            // its k coordinates and its index once
            bytes += b >= 0.0 ? b : (double)moved[(int)(-b - 1.0)] * 2.0 * 4.0 * (double)(c->k_last + 1);
        }
    }
    if (n_out) *n_out = cnt;
    if (ms_out) *ms_out = ms;
    if (bytes_out) *bytes_out = bytes;
    return LBKD_OK;
}

int lbkd_profile_read(lbkd_ctx* c, int* n_pass_launches, double* pass_ms, double* pass_bytes) {
    if (!c) return LBKD_EINVAL_SHAPE;
    return profile_class(c, c->algo == 0 ? kPPart : kPSortPass, n_pass_launches, pass_ms, pass_bytes);
}

int lbkd_profile_kernel(lbkd_ctx* c, int cls, int* n_launches, double* ms, double* bytes) {
    if (cls < -1 || cls >= kPClasses) return LBKD_EINVAL_SHAPE;
    return profile_class(c, cls, n_launches, ms, bytes);
}

int lbkd_set_algorithm(lbkd_ctx* c, int algo) {
    if (!c || algo < 0 || algo > 1) return LBKD_EINVAL_SHAPE;
    c->algo = algo;
    return LBKD_OK;
}

int lbkd_get_algorithm(const lbkd_ctx* c) { return c ? c->algo : -1; }

int lbkd_set_level_pairs(lbkd_ctx* c, int on) {
    if (!c || on < 0 || on > 1) return LBKD_EINVAL_SHAPE;
    if (c->pair_levels != on) drop_graph(c);  // (the cached graphs hold the other schedule)
    c->pair_levels = on;
    return LBKD_OK;
}

int lbkd_set_subtree_kernel(lbkd_ctx* c, int which) {
    if (!c || which < -1 || which > 1) return LBKD_EINVAL_SHAPE;
    c->subtree_sel = which;
    return LBKD_OK;
}

const char* lbkd_strerror(int code) {
    switch (code) {
        case LBKD_OK: return "ok";
        case LBKD_EINVAL_SHAPE: return "invalid shape or argument";
        case LBKD_ENONFINITE: return "coordinates must be finite (no NaN or infinity)";
        case LBKD_ECAPACITY: return "points exceed the 32-bit tag capacity";
        case LBKD_ECUDA: return "CUDA error";
        case LBKD_ENOPEER: return "peer access unavailable";
        case LBKD_ENOMEM: return "device allocation failed";
        case LBKD_EUNSUPPORTED: return "unsupported request";
        default: return "unknown error";
    }
}

const char* lbkd_last_cuda_error(void) { return g_cuda_err; }

}  // extern "C"
