// select.cu -- the global (large-segment) levels as pivot SELECTION plus one
// stable 3-way PARTITION per level, instead of a full per-level sort.
//
// Why this is bit-exact: the reference sorts every level
// stably by (tag, coord[dim]) (builder.py:165-181 / widest.py:119-131), so
// inside a level-l node the order it leaves is a FIXED total order
//     T(s) = (c[dim(s)], c[dim(parent)], ..., c[dim(root)], input index)
// (later repeats of a dimension dropped; RR: dims l, l-1, ..., l-k+1 mod k).
// The node's point is the element of rank pivot_off(s) under T(s)
// (kernels_numba.py:21-46 arithmetic); the left child gets every element
// below it, the right child every element above it.  Nothing else about the
// reference's arrangement is observable: the next level orders its nodes by
// a total order of its own.  So one level is
//   hist   : per-segment histogram of the key c[dim] in 2^D equal-width
//            buckets over the node's box (levels < 6; from level 6 on it is
//            fused into the previous level's partition)   (HBM read 4 B/pt)
//   pick   : bucket holding rank pivot_off, rank inside it     (per segment)
//   filter : the elements of that bucket -> candidate records, per-tile and
//            per-subtile counts of the elements below it      (4 B/pt)
//   select : radix select over the candidates' composite key (chain coords +
//            index) -> the node's point, written to its level-order slot;
//            the tile counts become per-segment exclusive prefixes.  The top
//            levels run each segment on a thread-block CLUSTER (DSMEM
//            merges), so millions of candidates (tie-heavy / wide-range
//            data) do not serialise on one SM
//   part   : stable 3-way partition of every segment around its pivot
//            (read + write k coords + index = 8(k+1) B/pt through a TMA-fed
//            shared-memory ring per warp; destinations from the select's
//            prefixes, no lookback), fused with the next level's histogram
// The partition is stable, so every segment keeps the INPUT order of its
// points; the in-CTA phase (subtree.cu) derives its chain orders from that.
//
// Layout: in-order SoA as in global_sort.cu -- segment j of level l occupies
// [ib(j), ib(j) + ss(j)) of W[(l - lfirst) & 1]; finished nodes leave a hole.
#include "kernels.cuh"

#include <cooperative_groups.h>

#include <cstdlib>

namespace lbkd {

// Round-robin: the dimension a level-l node's points are bucketed by -- the
// first dimension of its chain (l, l-1, ... mod k, truncated near the root)
// in which its box is not a single value.  Every point of the node ties on
// the chain dims before it (they lie in the box), so the node's order is the
// same order without them; bucketing a pinned dim would put the whole node
// into one bucket.  -1: every chain dim is pinned (the order is the input
// order: pick makes the segment positional).
__device__ __forceinline__ int rr_key_dim(const float* box, int k, int l) {
    const int m = l + 1 < k ? l + 1 : k;
    for (int i = 0; i < m; ++i) {
        const int d = (l - i) % k;
        if (box[d] < box[k + d]) return d;
    }
    return -1;
}

// the key dimension of segment t of the level (widest: the node's split dim,
// pinned only when the whole box is a point)
__device__ __forceinline__ int seg_key_dim(const SelArgs& a, u64 t) {
    if (a.mode == kRoundRobin) {
        const int d = rr_key_dim(a.boxes_in + t * 2ull * a.k, a.k, a.g.l);
        return d >= 0 ? d : a.g.l % a.k;
    }
    return (int)a.split_dims[a.g.Fl + a.g.sbase + t];
}

__device__ __forceinline__ int bitlen32(u32 v) { return v ? 32 - __clz(v) : 0; }

// equal-width buckets of [lo, hi]: shift such that (hi - lo) >> shift < 2^D
__device__ __forceinline__ u32 bucket_shift(u32 lo, u32 hi, int D) {
    int b = bitlen32(hi - lo) - D;
    return b > 0 ? (u32)b : 0u;
}

// Equal-width buckets of a segment's VALUE range [lo, hi] in its split
// dimension: its node's box (the world box clipped by the ancestors' planes,
// a valid bound of every point of the node).  Float keys are exponential in their bits, so
// equal widths in key space would put half of a [0, 1) segment into the few
// buckets of [0.5, 1); equal widths in value space split it evenly.  The map
// is monotone (IEEE subtraction, multiplication by a positive scale and the
// truncation are monotone) and identical in hist and filter, which is all
// the selection needs.  -0.0 and +0.0 land in the same bucket.
//
// KEY-linear mode (mode 1): equal widths of the order-flipped key range --
// right for data spread over many binades (log-like, e.g. 1e-30..1e30),
// where value-linear buckets put almost the whole node into its lowest
// bucket.  A node's mode is set by its parent's selection (select kernel):
// once a pivot bucket held more than 1/32 of its node, the children use key
// buckets (and pass that on).  Uniform data never triggers it.
struct Bucketer {
    float hlo, scale;  // value mode: halves (no overflow of hi - lo); key mode: scale < 0,
    u32 top;           //   hlo = the flipped key of lo, -scale - 1 = the shift
};

__device__ __forceinline__ Bucketer make_bucketer(float lo, float hi, int D, int mode = 0) {
    Bucketer b;
    b.top = (1u << D) - 1u;
    if (mode) {
        const u32 klo = flip_key(lo), khi = flip_key(hi);
        u32 sh = 0;
        while (((khi - klo) >> sh) > b.top) ++sh;
        b.hlo = __uint_as_float(klo);
        b.scale = -(float)(sh + 1u);
        return b;
    }
    b.hlo = 0.5f * lo;
    const float w = 0.5f * hi - b.hlo;
    b.scale = w > 0.0f ? __fdiv_rn((float)(1u << D), w) : 0.0f;
    return b;
}

__device__ __forceinline__ u32 bucket_key(const Bucketer& b, u32 bits) {  // key mode: a shift of the flipped key
    const u32 r = (flip_key(__uint_as_float(bits)) - __float_as_uint(b.hlo)) >> ((u32)(-b.scale) - 1u);
    return r < b.top ? r : b.top;
}

__device__ __forceinline__ u32 bucket_val(const Bucketer& b, u32 bits) {
    // fp32, round-to-nearest each step: monotone in the key
    const float x = __fmul_rn(__fsub_rn(0.5f * __uint_as_float(bits), b.hlo), b.scale);
    return x < (float)b.top ? (u32)x : b.top;  // NaN (non-finite input, reported later) -> top
}

__device__ __forceinline__ bool key_mode(const Bucketer& b) { return b.scale < 0.0f; }

__device__ __forceinline__ u32 bucket_of(const Bucketer& b, u32 bits) {
    return key_mode(b) ? bucket_key(b, bits) : bucket_val(b, bits);
}

// Incremental segment cursor over the view's in-order positions for a CTA
// that walks consecutive tiles (each tile <= the smallest segment, so a tile
// holds at most two segment parts); 64-bit geometry only at segment changes.
struct SegCursor {
    u64 cur, sb, se;  // current segment and its [sb, se) positions
    __device__ void init(const LevelGeom& g, u64 p) {
        cur = v_seg_of(g, p);
        sb = v_ibegin(g, cur);
        se = sb + v_size(g, cur);
    }
    // parts of tile [ts, ts + cnt): [r0a, r0b) of cur, [r1a, r1b) of cur + 1
    __device__ void parts(const LevelGeom& g, u64 ts, u64 cnt, u32& r0a, u32& r0b, u32& r1a, u32& r1b, bool& has1) {
        while (se + 1 <= ts && cur + 1 < g.nseg) {  // past cur and the finished node after it
            ++cur;
            sb = se + 1;
            se = sb + v_size(g, cur);
        }
        r0a = sb > ts ? (u32)(sb - ts) : 0u;
        r0b = se > ts ? (u32)((se - ts < cnt) ? se - ts : cnt) : 0u;
        if (r0b < r0a) r0b = r0a;
        has1 = cur + 1 < g.nseg && se + 1 < ts + cnt;
        r1a = r1b = (u32)cnt;
        if (has1) {
            r1a = (u32)(se + 1 - ts);
            const u64 e1 = se + 1 + v_size(g, cur + 1);
            r1b = (u32)((e1 - ts < cnt) ? e1 - ts : cnt);
        }
    }
};

// tile -> (first segment part, second segment part) of the view; a tile
// holds at most two segment parts (tile <= smallest segment)
struct TileParts {
    u64 j0;
    u32 r0a, r0b, r1a, r1b;  // tile-relative [a, b) of the parts
    bool has1;
    u64 ib0, ib1;            // in-order (view) begins of segments j0, j0+1
};

__device__ __forceinline__ TileParts tile_parts(const LevelGeom& g, u64 ts, u64 cnt) {
    TileParts p;
    p.j0 = v_seg_of(g, ts);
    const u64 s0b = v_ibegin(g, p.j0), s0e = s0b + v_size(g, p.j0);
    p.ib0 = s0b;
    p.r0a = s0b > ts ? (u32)(s0b - ts) : 0u;
    p.r0b = s0e > ts ? (u32)((s0e - ts < cnt) ? s0e - ts : cnt) : 0u;
    if (p.r0b < p.r0a) p.r0b = p.r0a;
    p.has1 = false;
    p.r1a = p.r1b = (u32)cnt;
    p.ib1 = 0;
    if (p.j0 + 1 < g.nseg) {
        const u64 s1b = v_ibegin(g, p.j0 + 1);
        if (s1b < ts + cnt) {
            p.has1 = true;
            p.ib1 = s1b;
            p.r1a = (u32)(s1b - ts);
            const u64 s1e = s1b + v_size(g, p.j0 + 1);
            p.r1b = (u32)((s1e - ts < cnt) ? s1e - ts : cnt);
        }
    }
    return p;
}

// ---------------------------------------------------------------------------
// init: AoS float32 input -> W[0] SoA (k coordinate arrays + index array),
// the non-finite check of builder.py:134-135 and the per-dimension min/max
// (world_bounds, widest.py:84-88; the root's key range) as order-flipped
// u32 so plain atomics are exact.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) init_stats_kernel(const float* __restrict__ pts, u64 n, int k, u32* w0,
                                                         u64 stride, u32* err, u32* minmax) {
    __shared__ u32 smn[LBKD_MAX_K], smx[LBKD_MAX_K];
    if (threadIdx.x < LBKD_MAX_K) { smn[threadIdx.x] = 0xffffffffu; smx[threadIdx.x] = 0u; }
    __syncthreads();
    u32 mn[LBKD_MAX_K], mx[LBKD_MAX_K];
#pragma unroll
    for (int c = 0; c < LBKD_MAX_K; ++c) { mn[c] = 0xffffffffu; mx[c] = 0u; }
    bool bad = false;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const float* q = pts + i * k;
#pragma unroll
        for (int c = 0; c < LBKD_MAX_K; ++c) {
            if (c < k) {
                const float f = __ldg(q + c);
                bad |= !isfinite(f);
                const u32 key = flip_key(f);
                mn[c] = min(mn[c], key);
                mx[c] = max(mx[c], key);
                w0[c * stride + i] = __float_as_uint(f);
            }
        }
        w0[(u64)k * stride + i] = (u32)i;
    }
    if (__any_sync(kFullMask, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
#pragma unroll
    for (int c = 0; c < LBKD_MAX_K; ++c) {
        if (c < k) {
            const u32 a = __reduce_min_sync(kFullMask, mn[c]);
            const u32 b = __reduce_max_sync(kFullMask, mx[c]);
            if ((threadIdx.x & 31) == 0) { atomicMin(&smn[c], a); atomicMax(&smx[c], b); }
        }
    }
    __syncthreads();
    if (threadIdx.x < (unsigned)k) {
        atomicMin(&minmax[threadIdx.x], smn[threadIdx.x]);
        atomicMax(&minmax[k + threadIdx.x], smx[threadIdx.x]);
    }
}

void launch_init_stats(const BuildParams& bp, const Buffers& bf, u32* minmax, cudaStream_t st) {
    u64 blocks = (bp.n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    init_stats_kernel<<<(unsigned)blocks, 256, 0, st>>>(bp.pts, bp.n, bp.k, bf.w[0], bf.stride, bf.err, minmax);
}

// non-finite check of builder.py:134-135 for builds without global levels
// (single-CTA trees read the input straight from the caller's array)
__global__ void check_finite_kernel(const float* __restrict__ pts, u64 total, u32* err) {
    bool bad = false;
    for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < total; e += (u64)gridDim.x * blockDim.x)
        bad |= !isfinite(__ldg(pts + e));
    if (__any_sync(kFullMask, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

void launch_check_finite(const float* pts, u64 total, u32* err, cudaStream_t st) {
    u64 blocks = (total + 255) / 256;
    if (blocks > 148 * 4) blocks = 148 * 4;
    if (blocks < 1) blocks = 1;
    check_finite_kernel<<<(unsigned)blocks, 256, 0, st>>>(pts, total, err);
}

// bounding box of a sub-build's points (W[0], blockIdx.y = dimension): the
// view root's box (any valid bound of its points works)
__global__ void view_minmax_kernel(const u32* __restrict__ w0, u64 stride, u64 m, int k, u32* minmax) {
    const int d = blockIdx.y;
    const u32* keys = w0 + (u64)d * stride;
    u32 mn = 0xffffffffu, mx = 0u;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x) {
        const u32 key = flip_key(__uint_as_float(keys[i]));
        mn = min(mn, key);
        mx = max(mx, key);
    }
    mn = __reduce_min_sync(kFullMask, mn);
    mx = __reduce_max_sync(kFullMask, mx);
    if ((threadIdx.x & 31) == 0) { atomicMin(&minmax[d], mn); atomicMax(&minmax[k + d], mx); }
}

void launch_view_minmax(const BuildParams& bp, const Buffers& bf, u32* minmax, u64 m, cudaStream_t st) {
    u64 blocks = (m + 255) / 256;
    if (blocks > 148 * 2) blocks = 148 * 2;
    if (blocks < 1) blocks = 1;
    view_minmax_kernel<<<dim3((unsigned)blocks, (unsigned)bp.k), 256, 0, st>>>(bf.w[0], bf.stride, m, bp.k, minmax);
}

// root box = world box (widest.py:84-88); widest: root dim = first argmax
// of the float64 widths (widest.py:91-93, :164-166)
__global__ void root_kernel(const u32* minmax, int k, int mode, float* box0, uint8_t* split_dims, WidthTab wt) {
    if (threadIdx.x != 0) return;
    int d0 = 0;
    double bw = 0.0;
    for (int d = 0; d < k; ++d) {
        const float lo = unflip_key(minmax[d]), hi = unflip_key(minmax[k + d]);
        box0[d] = lo;
        box0[k + d] = hi;
        const double w = coord_width(wt, d, lo, hi);
        if (d == 0 || w > bw) { bw = w; d0 = d; }
    }
    if (mode == kWidest) split_dims[0] = (uint8_t)d0;
}

void launch_root(const BuildParams& bp, const Buffers& bf, const u32* minmax, cudaStream_t st) {
    root_kernel<<<1, 32, 0, st>>>(minmax, bp.k, bp.mode, bf.boxes[0], bp.split_dims, bp.wt);
}

__device__ __forceinline__ Bucketer seg_bucketer(const SelArgs& a, u64 t, int d) {
    const float* box = a.boxes_in + t * 2ull * a.k;
    return make_bucketer(box[d], box[a.k + d], a.D, a.bmode_in[t]);
}

// ---------------------------------------------------------------------------
// hist: per segment, 2^D equal-width buckets of the key over [min, max].
// Each CTA walks a contiguous run of tiles and flushes its shared histogram
// when the segment changes (global atomics O(#CTAs + #segments) x 2^D).
// ---------------------------------------------------------------------------
constexpr int kHThreads = 256;

template <int ITEMS>
__global__ void __launch_bounds__(kHThreads) sel_hist_kernel(SelArgs a) {
    extern __shared__ u32 h[];
    constexpr int T = kHThreads * ITEMS;
    const int nb = 1 << a.D;
    const LevelGeom& g = a.g;
    for (int i = threadIdx.x; i < nb; i += kHThreads) h[i] = 0u;
    const u64 t0 = (u64)blockIdx.x * a.tiles_per_cta;
    u64 t1 = t0 + a.tiles_per_cta;
    if (t1 > a.ntiles) t1 = a.ntiles;
    SegCursor sc;
    sc.init(g, t0 * T);
    u64 cur = sc.cur;  // segment the shared histogram currently counts
    __syncthreads();
    auto flush = [&](u64 seg) {
        __syncthreads();
        u32* gh = a.hist + seg * (u64)nb;
        for (int i = threadIdx.x; i < nb; i += kHThreads) {
            const u32 v = h[i];
            if (v) { atomicAdd(&gh[i], v); h[i] = 0u; }
        }
        __syncthreads();
    };
    const u32* W = a.bf.w[a.par];
    int dk = -1, dk1 = -1;
    u64 nseg_c = ~0ull;  // segment whose key dim dk1 holds
    Bucketer bk{};
    const u32* kp = nullptr;
    for (u64 t = t0; t < t1; ++t) {
        const u64 ts = t * T;
        const u64 cnt = g.nview - ts < (u64)T ? g.nview - ts : (u64)T;
        u32 r0a, r0b, r1a, r1b;
        bool has1;
        sc.parts(g, ts, cnt, r0a, r0b, r1a, r1b, has1);
        if (sc.cur != cur) {  // the previous tile ended exactly at a segment end
            flush(cur);
            cur = sc.cur;
            dk = -1;
        }
        if (dk < 0) {
            dk = seg_key_dim(a, cur);
            bk = seg_bucketer(a, cur, dk);
            kp = W + (u64)dk * a.bf.stride;
        }
        u32 key[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            // only the tile's segment parts (the finished nodes between
            // segments hold no data in this buffer)
            const u32 r = (u32)(i * kHThreads + threadIdx.x);
            const bool use = (r >= r0a && r < r0b) || (has1 && r >= r1a && r < r1b);
            key[i] = use ? kp[ts + r] : 0u;
        }
        if (has1 && nseg_c != cur + 1) {  // the next segment's key dim, once per segment
            nseg_c = cur + 1;
            dk1 = seg_key_dim(a, cur + 1);
        }
        if (has1 && dk1 != dk) {  // the next segment is keyed by another dim
            const u32* k1 = W + (u64)dk1 * a.bf.stride;
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const u32 r = (u32)(i * kHThreads + threadIdx.x);
                if (r >= r1a && r < r1b) key[i] = k1[ts + r];
            }
        }
        // (the bucket mode hoisted out of the per-key loops)
        auto bin = [&](u32 ra, u32 rb) {
            if (key_mode(bk)) {
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const u32 r = (u32)(i * kHThreads + threadIdx.x);
                    if (r >= ra && r < rb) atomicAdd(&h[bucket_key(bk, key[i])], 1u);
                }
            } else {
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const u32 r = (u32)(i * kHThreads + threadIdx.x);
                    if (r >= ra && r < rb) atomicAdd(&h[bucket_val(bk, key[i])], 1u);
                }
            }
        };
        bin(r0a, r0b);
        if (has1) {
            flush(cur);
            cur = cur + 1;
            dk = dk1;
            bk = seg_bucketer(a, cur, dk);
            kp = W + (u64)dk * a.bf.stride;
            bin(r1a, r1b);
        }
    }
    flush(cur);
}

// ---------------------------------------------------------------------------
// pick: one CTA per segment -- the bucket b* holding rank pivot_off and the
// rank r inside it; reserves the segment's candidate range.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) sel_pick_kernel(SelArgs a) {
    __shared__ u32 wtot[32];
    const u64 j = blockIdx.x;
    // a node box that is a single point (every coordinate of every point of
    // the segment equal): the within-node order is the input order, which is
    // the segment's order in W (stable partitions) -- the node is the element
    // at in-order offset pivot_off, no histogram and no candidates to sort
    {
        const float* box = a.boxes_in + j * 2ull * a.k;
        bool point = true;
        if (a.mode == kRoundRobin) {
            point = rr_key_dim(box, a.k, a.g.l) < 0;  // every chain dim pinned
        } else {
            for (int d = 0; d < a.k; ++d) point &= box[d] == box[a.k + d];
        }
        if (point) {
            if (threadIdx.x == 0) {
                u32* sel = a.sel + j * kSelW;
                sel[kSelLo] = (u32)(v_ibegin(a.g, j) + v_pivot(a.g, j));  // the node's position
                sel[kSelB] = kSelPositional;
                sel[kSelR] = 0u;
                sel[kSelC] = 1u;
                sel[kSelOff] = atomicAdd(a.cand_ctr, 1u);
                sel[kSelFill] = 0u;
            }
            return;
        }
    }
    const int nb = 1 << a.D;
    const int per = nb / 256;
    const u32* h = a.hist + j * (u64)nb;
    const u32 po = (u32)v_pivot(a.g, j);
    u32 s = 0;
    for (int i = 0; i < per; ++i) s += h[threadIdx.x * per + i];
    const u32 ex = block_exclusive_scan<u32>(s, wtot, nullptr);
    if (po >= ex && po < ex + s) {
        u32 cum = ex;
        int b = threadIdx.x * per;
        while (cum + h[b] <= po) { cum += h[b]; ++b; }
        u32* sel = a.sel + j * kSelW;
        const u32 C = h[b];
        const int d = seg_key_dim(a, j);
        const float* box = a.boxes_in + j * 2ull * a.k;
        sel[kSelLo] = __float_as_uint(box[d]);  // the filter rebuilds the bucketer
        sel[kSelShift] = __float_as_uint(box[a.k + d]);
        sel[kSelMode] = a.bmode_in[j];
        sel[kSelB] = (u32)b;
        sel[kSelR] = po - cum;
        sel[kSelC] = C;
        sel[kSelOff] = atomicAdd(a.cand_ctr, C);
        sel[kSelFill] = 0u;
    }
}

// ---------------------------------------------------------------------------
// filter: per (tile, part) and per (warp subtile, part) the number of
// elements in buckets below b*, and every element of bucket b* -> a
// candidate record (k coordinate bits, input index, in-order position) in
// the segment's candidate range.  A tile is T = 8 x blockDim positions, a
// warp subtile kSub = 256 positions (8 per thread, thread-contiguous); the
// part index of both is relative to the TILE's first segment.
// ---------------------------------------------------------------------------
constexpr int kSub = 256;  // positions per warp subtile (32 lanes x 8 rows)
constexpr int kFCap = 256;  // filter: candidate records staged per CTA

template <int THREADS>
__global__ void __launch_bounds__(THREADS, 2048 / THREADS) sel_filter_kernel(SelArgs a) {
    // CTA = a contiguous run of tiles; per tile every warp owns one 256-
    // position subtile (8 items per thread, thread-contiguous).  Counts of
    // elements below b*: per (subtile, part) one plain store by the warp,
    // per (tile, part) one global atomic per warp (tile_lt is zeroed per
    // level).  The rare hits (1 / 2^D of the points) are staged in the CTA's
    // shared memory (shared-atomic slots) and appended to their segments'
    // candidate ranges once, at the end, one global atomic per segment per
    // 32 records (the per-warp global atomic on ONE fill counter per segment
    // serialised at the top levels); a full staging area falls back to
    // per-warp global reservations.  Two block barriers (start, end).
    constexpr int ITEMS = 8;
    constexpr int T = THREADS * ITEMS;
    constexpr int NSUB = T / kSub;
    const LevelGeom& g = a.g;
    const u32* W = a.bf.w[a.par];
    const int k = a.k, R = k + 2;
    extern __shared__ u32 fsm[];  // [0] staged count, [kFCap] segment ids, [kFCap * R] records
    u32* const s_seg = fsm + 1;
    u32* const s_rec = s_seg + kFCap;
    for (int e = threadIdx.x; e < kFCap; e += THREADS) s_seg[e] = ~0u;
    if (threadIdx.x == 0) fsm[0] = 0u;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const u32 ltm = lanemask_lt();
    const u64 t0 = (u64)blockIdx.x * a.tiles_per_cta;
    u64 t1 = t0 + a.tiles_per_cta;
    if (t1 > a.ntiles) t1 = a.ntiles;
    if (t0 >= t1) return;  // (the whole CTA)
    SegCursor sc;
    sc.init(g, t0 * T);
    u64 cj = ~0ull;
    Bucketer cbk{};
    u32 cbs = 0;
    int cdk = 0;
    for (u64 t = t0; t < t1; ++t) {
        const u64 ts = t * T;
        const u64 cnt = g.nview - ts < (u64)T ? g.nview - ts : (u64)T;
        u32 r0a, r0b, r1a, r1b;
        bool has1;
        sc.parts(g, ts, cnt, r0a, r0b, r1a, r1b, has1);
        const u64 s = t * NSUB + warp;
        u32 nlt_s[2] = {0u, 0u};
#pragma unroll
        for (int part = 0; part < 2; ++part) {
            const u64 j = sc.cur + part;
            const u32 ra = part ? r1a : r0a, rb = part ? r1b : r0b;
            if (!((part == 0 || has1) && ra < rb)) continue;
            u32* sel = a.sel + j * kSelW;
            if (j != cj) {  // the segment's bucketer and key dim, kept while tiles stay in it
                cj = j;
                cbk = make_bucketer(__uint_as_float(sel[kSelLo]), __uint_as_float(sel[kSelShift]), a.D,
                                    (int)sel[kSelMode]);
                cbs = sel[kSelB];
                cdk = seg_key_dim(a, j);
            }
            const Bucketer bk = cbk;
            const u32 bs = cbs;
            const u32* kp = W + (u64)cdk * a.bf.stride + ts;
            u32 hits = 0, nlt = 0;
            const u32 r0 = (u32)threadIdx.x * ITEMS;
            if (bs == kSelPositional) {  // (pick: a point box) the node is at in-order position sel[kSelLo]
                const u32 npos = sel[kSelLo];
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const u32 r = r0 + (u32)i;
                    if (r >= ra && r < rb) {
                        const u32 p = (u32)(ts + r);
                        if (p == npos) hits |= 1u << i;
                        nlt += p < npos ? 1u : 0u;
                    }
                }
            } else if (r0 >= ra && r0 + ITEMS <= rb) {
                // the thread's 8 keys lie in this part: two 16-byte loads (the
                // SoA columns are 16-byte aligned and tiles start at multiples
                // of T words)
                const uint4 q0 = *reinterpret_cast<const uint4*>(kp + r0);
                const uint4 q1 = *reinterpret_cast<const uint4*>(kp + r0 + 4);
                const u32 key[ITEMS] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
                if (key_mode(bk)) {
#pragma unroll
                    for (int i = 0; i < ITEMS; ++i) {
                        const u32 b = bucket_key(bk, key[i]);
                        if (b == bs) hits |= 1u << i;
                        nlt += b < bs ? 1u : 0u;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < ITEMS; ++i) {
                        const u32 b = bucket_val(bk, key[i]);
                        if (b == bs) hits |= 1u << i;
                        nlt += b < bs ? 1u : 0u;
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const u32 r = r0 + (u32)i;
                    if (r >= ra && r < rb) {
                        const u32 b = bucket_of(bk, kp[r]);
                        if (b == bs) hits |= 1u << i;
                        nlt += b < bs ? 1u : 0u;
                    }
                }
            }
            nlt = __reduce_add_sync(kFullMask, nlt);
            nlt_s[part] = nlt;
            if (lane == 0 && nlt) atomicAdd(&a.tile_lt[t * 2 + part], nlt);
            // candidates: warp-aggregated slot reservation
            const u32 nh = (u32)__popc(hits);
            const u32 wtot = __reduce_add_sync(kFullMask, nh);  // usually 0: skip the scan
            if (wtot) {
                u32 x = nh;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const u32 y = __shfl_up_sync(kFullMask, x, o);
                    if (lane >= o) x += y;
                }
                u32 pos = 0;
                if (lane == 31) pos = atomicAdd(&fsm[0], wtot);
                pos = __shfl_sync(kFullMask, pos, 31);
                if (pos + wtot <= (u32)kFCap) {  // staged in shared memory
                    u32 q = pos + x - nh;
                    while (hits) {
                        const int i = __ffs(hits) - 1;
                        hits &= hits - 1;
                        const u32 r = (u32)(threadIdx.x * ITEMS + i);
                        u32* rec = s_rec + q * R;
                        for (int c = 0; c <= k; ++c) rec[c] = W[(u64)c * a.bf.stride + ts + r];
                        rec[k + 1] = (u32)(ts + r);
                        s_seg[q] = (u32)j;
                        ++q;
                    }
                } else {  // staging full (tie-heavy data): reserve in the segment directly
                    u32 base = 0;
                    if (lane == 31) base = atomicAdd(&sel[kSelFill], wtot);
                    base = __shfl_sync(kFullMask, base, 31);
                    u32 slot = sel[kSelOff] + base + x - nh;
                    while (hits) {
                        const int i = __ffs(hits) - 1;
                        hits &= hits - 1;
                        const u32 r = (u32)(threadIdx.x * ITEMS + i);
                        u32* rec = a.cand + (u64)slot * R;
                        for (int c = 0; c <= k; ++c) rec[c] = W[(u64)c * a.bf.stride + ts + r];
                        rec[k + 1] = (u32)(ts + r);
                        ++slot;
                    }
                }
            }
        }
        if (lane == 0) {
            a.sub_lt[s * 2] = nlt_s[0];
            a.sub_lt[s * 2 + 1] = nlt_s[1];
        }
        (void)ltm;
    }
    // the staged candidates -> their segments' ranges: per 32 records one
    // global reservation per distinct segment (peers by __match_any_sync)
    __syncthreads();
    const u32 nst = min(fsm[0], (u32)kFCap);
    for (u32 e0 = (u32)warp * 32u; e0 < nst; e0 += (u32)THREADS) {
        const u32 e = e0 + (u32)lane;
        const u32 js = e < nst ? s_seg[e] : ~0u;  // ~0: a slot of an overflowed reservation, never written
        const u32 peers = __match_any_sync(kFullMask, js);
        const int leader = __ffs(peers) - 1;
        u32 base = 0;
        if (js != ~0u && lane == leader) base = atomicAdd(&a.sel[(u64)js * kSelW + kSelFill], (u32)__popc(peers));
        base = __shfl_sync(kFullMask, base, leader);
        if (js != ~0u) {
            const u32 slot = a.sel[(u64)js * kSelW + kSelOff] + base + (u32)__popc(peers & ltm);
            const u32* src = s_rec + e * R;
            u32* rec = a.cand + (u64)slot * R;
            for (int c = 0; c < R; ++c) rec[c] = src[c];
        }
    }
}

// ---------------------------------------------------------------------------
// select: one CTA per segment.  Radix select of rank r among the segment's
// candidates under the composite key (chain coords order-flipped, then the
// input index): per field, equal-width buckets over the live [min, max],
// narrowing until one candidate is left.  Every candidate that falls below
// the narrowing bucket is below the pivot: it is added to its tile's count,
// after which the segment's per-tile counts are turned into exclusive
// prefixes (the partition's destinations, no lookback).  Writes the node
// (level-order output), the pivot record / position / chain the partition
// compares against, and for widest the children's boxes and split dims
// (kernels_numba.py:80-110).
// ---------------------------------------------------------------------------
constexpr int kSThreads = 256;

__device__ __forceinline__ u32 rec_field(const u32* rec, const Chain& ch, int f, int k) {
    return f < (int)ch.m ? flip_key(__uint_as_float(rec[ch.d[f]])) : rec[k];
}

// CS > 1: a thread-block cluster of CS CTAs per segment (top levels, where a
// few segments can hold millions of candidates -- tie-heavy or wide-range
// data): every CTA scans 1/CS of the candidates; ranges and histograms are
// combined in the rank-0 CTA's shared memory (DSMEM), one cluster barrier
// per phase, and rank 0 alone writes the segment's results.
template <int NT, int CS>
__global__ void __launch_bounds__(NT) sel_select_kernel(SelArgs a, int T) {
    namespace cg = cooperative_groups;
    __shared__ u32 hist[256];
    __shared__ u32 red[2][32];
    __shared__ u32 s_misc[4];
    __shared__ u32 wtot[32];
    // rank 0: every CTA's candidate range, double-buffered by round: a round
    // that ends right after reading it (constant field -> break) has no
    // further cluster barrier, so a fast CTA's next write must not land in
    // the buffer a slow CTA is still reading
    __shared__ u32 c_mm[2][2][CS];
    int mm_buf = 0;
    __shared__ Chain s_ch;
    // the hardware's rank inside the cluster and the cluster's index (a 1-D
    // grid of 1-D clusters: cluster c holds blocks c * CS .. c * CS + CS - 1)
    u32 crank = 0u;
    u64 j = blockIdx.x;
    if constexpr (CS > 1) {
        crank = cg::this_cluster().block_rank();
        u32 cid;
        asm("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
        j = cid;
    }
    const int k = a.k, R = k + 2, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto csync = [&]() {
        if constexpr (CS > 1) cg::this_cluster().sync();
    };
    // rank 0's copy of a shared variable (DSMEM)
    auto r0 = [&](auto* p) {
        if constexpr (CS > 1) return cg::this_cluster().map_shared_rank(p, 0);
        else return p;
    };
    const LevelGeom& g = a.g;
    const u64 node = g.Fl + g.sbase + j;
    u32* sel = a.sel + j * kSelW;
    if (tid == 0) {
        if (a.mode == kRoundRobin) rr_chain(g.l, k, s_ch);
        else widest_chain(node, k, a.split_dims, s_ch);
    }
    // (clusters: every CTA must have started before any touches another's
    // shared memory)
    if constexpr (CS > 1) csync();
    else __syncthreads();
    const Chain ch = s_ch;
    // the segment's tiles: the first one holds it as part 1 unless the
    // segment starts exactly at the tile start
    const u64 ib = v_ibegin(g, j);
    const u64 tfirst = ib / (u64)T;
    const u64 tlast = (ib + v_size(g, j) - 1) / (u64)T;
    const u32 pfirst = (ib == tfirst * (u64)T) ? 0u : 1u;
    auto count_below = [&](const u32* rec) {
        const u64 pos = rec[k + 1];
        const u64 t = pos / (u64)T;
        const u32 pt = t == tfirst ? pfirst : 0u;
        atomicAdd(&a.tile_lt[t * 2 + pt], 1u);
        atomicAdd(&a.sub_lt[(pos / (u64)kSub) * 2 + pt], 1u);
    };
    u32 n = sel[kSelC];
    u32 r = sel[kSelR];
    const u64 off = sel[kSelOff];
    const u32* src = a.cand + off * R;
    u32* bufs[2] = {a.cand2 + off * R, a.cand + off * R};
    int nb_flip = 0;
    for (int f = 0; f <= (int)ch.m && n > 1; ++f) {
        while (n > 1) {
            // live range of field f
            u32 mn = 0xffffffffu, mx = 0u;
            for (u32 i = tid + crank * NT; i < n; i += NT * CS) {
                const u32 v = rec_field(src + (u64)i * R, ch, f, k);
                mn = min(mn, v);
                mx = max(mx, v);
            }
            mn = __reduce_min_sync(kFullMask, mn);
            mx = __reduce_max_sync(kFullMask, mx);
            if (lane == 0) { red[0][warp] = mn; red[1][warp] = mx; }
            for (int i = tid; i < 256; i += NT) hist[i] = 0u;
            __syncthreads();
            if (warp == 0) {  // the block's range: one reduction over the warps' values
                const u32 a0 = __reduce_min_sync(kFullMask, lane < NT / 32 ? red[0][lane] : 0xffffffffu);
                const u32 b0 = __reduce_max_sync(kFullMask, lane < NT / 32 ? red[1][lane] : 0u);
                if (lane == 0) {
                    if constexpr (CS > 1) {
                        r0(&c_mm[mm_buf][0][0])[crank] = a0;
                        r0(&c_mm[mm_buf][1][0])[crank] = b0;
                    } else {
                        s_misc[0] = a0;
                        s_misc[1] = b0;
                    }
                }
            }
            if constexpr (CS > 1) {
                csync();
                mn = 0xffffffffu;
                mx = 0u;
#pragma unroll
                for (int q = 0; q < CS; ++q) {
                    mn = min(mn, r0(&c_mm[mm_buf][0][0])[q]);
                    mx = max(mx, r0(&c_mm[mm_buf][1][0])[q]);
                }
                mm_buf ^= 1;
            } else {
                __syncthreads();
                mn = s_misc[0];
                mx = s_misc[1];
            }
            if (mn == mx) break;  // field constant over the candidates
            const u32 sh = bucket_shift(mn, mx, 8);
            for (u32 i = tid + crank * NT; i < n; i += NT * CS)
                atomicAdd(&hist[(rec_field(src + (u64)i * R, ch, f, k) - mn) >> sh], 1u);
            if constexpr (CS > 1) csync();  // every CTA's histogram is complete
            else __syncthreads();
            if (warp == 0 && crank == 0) {
                // bucket holding rank r: 8 bins per lane, a warp scan of the
                // lane sums, then the one lane whose range holds r walks its bins
                u32 c[8];
                u32 sum = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    c[q] = hist[lane * 8 + q];
                    if constexpr (CS > 1) {
                        auto cl = cg::this_cluster();
                        for (int rr = 1; rr < CS; ++rr) c[q] += cl.map_shared_rank(hist, rr)[lane * 8 + q];
                    }
                    sum += c[q];
                }
                u32 x = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const u32 y = __shfl_up_sync(kFullMask, x, o);
                    if (lane >= o) x += y;
                }
                u32 cum = x - sum;
                if (r >= cum && r < x) {
                    int bsel = -1;
                    u32 bcnt = 0;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        if (bsel < 0) {
                            if (cum + c[q] > r) {
                                bsel = lane * 8 + q;
                                bcnt = c[q];
                            } else {
                                cum += c[q];
                            }
                        }
                    }
                    s_misc[2] = (u32)bsel;
                    s_misc[3] = cum;
                    s_misc[1] = bcnt;  // the bucket's count over every CTA of the cluster
                    s_misc[0] = 0u;  // compaction counter
                }
            }
            if constexpr (CS > 1) csync();  // rank 0 picked the bucket
            else __syncthreads();
            const u32 bsel = *r0(&s_misc[2]);
            r -= *r0(&s_misc[3]);
            const u32 cnt = *r0(&s_misc[1]);
            u32* dst = bufs[nb_flip];
            u32* ctr = r0(&s_misc[0]);
            for (u32 i0 = crank * NT; i0 < n; i0 += NT * CS) {
                const u32 i = i0 + tid;
                bool hit = false;
                if (i < n) {
                    const u32 b = (rec_field(src + (u64)i * R, ch, f, k) - mn) >> sh;
                    hit = b == bsel;
                    if (b < bsel) count_below(src + (u64)i * R);
                }
                const u32 m = __ballot_sync(kFullMask, hit);
                if (m) {
                    const int leader = __ffs(m) - 1;
                    u32 base = 0;
                    if (lane == leader) base = atomicAdd(ctr, (u32)__popc(m));
                    base = __shfl_sync(kFullMask, base, leader);
                    if (hit) {
                        const u32* s = src + (u64)i * R;
                        u32* d = dst + (u64)(base + __popc(m & lanemask_lt())) * R;
                        for (int c = 0; c < R; ++c) d[c] = s[c];
                    }
                }
            }
            if constexpr (CS > 1) csync();  // the compacted candidates are complete
            else __syncthreads();
            src = dst;
            nb_flip ^= 1;
            n = cnt;
        }
    }
    if constexpr (CS > 1) {
        // every CTA's below-pivot counts are in; rank 0 finishes the segment
        csync();
        if (crank != 0) return;
    }
    // src[0] is the node's point
    if (tid <= k) a.piv[j * (k + 1) + tid] = src[tid];
    if (tid == 0) {
        for (int c = 0; c < kChainWords; ++c) reinterpret_cast<u32*>(a.chains + j)[c] = reinterpret_cast<const u32*>(&ch)[c];
        a.perm[node] = src[k];
        a.ppos[j] = src[k + 1];
    }
    if (tid < k) a.out_pts[node * k + tid] = __uint_as_float(src[tid]);
    if (tid < 2) {
        // child tid of node: box = node box clipped by the node's plane (the
        // next level's bucket range; widest: its split dim)
        const int d = ch.d[0];
        const float plane = __uint_as_float(src[d]);
        const float* bin = a.boxes_in + j * 2ull * k;
        float lo[LBKD_MAX_K], hi[LBKD_MAX_K];
        for (int q = 0; q < k; ++q) { lo[q] = bin[q]; hi[q] = bin[k + q]; }
        if (tid == 0) { if (plane < hi[d]) hi[d] = plane; }
        else { if (plane > lo[d]) lo[d] = plane; }
        const u64 c = 2 * j + tid;
        float* bout = a.boxes_out + c * 2ull * k;
        int best = 0;
        double bw = 0.0;
        for (int q = 0; q < k; ++q) {
            bout[q] = lo[q];
            bout[k + q] = hi[q];
            const double w = coord_width(a.wt, q, lo[q], hi[q]);
            if (q == 0 || w > bw) { bw = w; best = q; }
        }
        const u64 cnode = 2 * node + 1 + tid;
        if (a.mode == kWidest && cnode < g.n) a.split_dims[cnode] = (uint8_t)best;
        // the children's bucket mode: key-linear once a pivot bucket held more
        // than 1/32 of its node (value-linear buckets failing: log-like data)
        const bool crowded = (u64)sel[kSelC] * 32ull > v_size(g, j);
        a.bmode_out[c] = (a.bmode_in[j] || crowded) ? 1u : 0u;
    }
    // per-tile counts below the pivot -> exclusive prefixes in tile order
    __syncthreads();
    u32 carry = 0;
    for (u64 t0 = tfirst; t0 <= tlast; t0 += NT) {
        const u64 t = t0 + tid;
        u32* slot = t <= tlast ? &a.tile_lt[t * 2 + (t == tfirst ? pfirst : 0u)] : nullptr;
        const u32 v = slot ? *slot : 0u;
        const u32 ex = block_exclusive_scan<u32>(v, wtot, nullptr);
        if (slot) *slot = carry + ex;
        // chunk total: last thread's inclusive value
        if (tid == NT - 1) s_misc[1] = ex + v;
        __syncthreads();
        carry += s_misc[1];
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// part: stable 3-way partition of every segment around its pivot.  Each
// warp owns one 256-position subtile at a time and needs no other warp:
// the number of elements below the pivot in everything before its subtile
// comes from select (per-tile exclusive prefix) plus the filter's counts of
// the earlier subtiles of the same tile.  The warp loads its subtile's k+1
// arrays with coalesced loads (all rows in flight at once), classifies
// against the pivot (chain fields only on a tie), ranks with warp ballots
// and stores every element straight from registers into its child run --
// no shared-memory staging and no block barrier.  Stability: rows in
// position order, lanes in order inside a row.
// ---------------------------------------------------------------------------
constexpr int kPThreads = 256;
constexpr int kPRows = kSub / 32;

// equal leading coordinates: compare the rest of the node's chain, then the
// input row (rare; re-reads the point from the source arrays)
__device__ __noinline__ int part_tie_side(const SelArgs& a, u64 j, u64 pos) {
    const int k = a.k, A = k + 1;
    const u32* W = a.bf.w[a.par];
    const Chain* ch = a.chains + j;
    const u32* pv = a.piv + j * A;
    const u32 mm = ch->m;
    for (u32 f = 1; f < mm; ++f) {
        const int d = ch->d[f];
        const u32 xx = flip_key(__uint_as_float(W[(u64)d * a.bf.stride + pos]));
        const u32 yy = flip_key(__uint_as_float(pv[d]));
        if (xx != yy) return xx < yy ? 0 : 1;
    }
    const u32 xx = W[(u64)k * a.bf.stride + pos], yy = pv[k];
    return xx < yy ? 0 : (xx > yy ? 1 : 2);
}

// D0 >= 0: every segment's leading key is coordinate D0 (round-robin): full
// single-part subtiles take a lean path (float compares, no part masks)
template <int KMAX, int D0>
__global__ void __launch_bounds__(kPThreads, KMAX <= 4 ? 2 : 1) sel_part_kernel(SelArgs a, int T) {
    const int lane = threadIdx.x & 31;
    const int k = a.k, A = k + 1;
    const LevelGeom& g = a.g;
    const u32* Wsrc = a.bf.w[a.par];
    u32* Wdst = a.bf.w[a.par ^ 1u];
    const u64 stride = a.bf.stride;
    const u64 nsub = (g.nview + kSub - 1) / kSub;
    const int nsub_tile = T / kSub;
    const u32 lt = lanemask_lt();
    const u64 sstep = (u64)gridDim.x * (kPThreads / 32);
    // software pipeline: the next subtile's loads are in flight while this
    // one is split (the kernel is load-latency bound otherwise)
    u32 vn[KMAX + 1][kPRows];
    auto load_sub = [&](u64 s2) {
        const u64 ss2 = s2 * kSub;
        const u64 cnt2 = g.nview - ss2 < (u64)kSub ? g.nview - ss2 : (u64)kSub;
#pragma unroll
        for (int c = 0; c <= KMAX; ++c) {
            if (c < A) {
                const u32* src = Wsrc + (u64)c * stride + ss2 + lane;
                if (cnt2 == (u64)kSub) {
#pragma unroll
                    for (int i = 0; i < kPRows; ++i) vn[c][i] = src[i * 32];
                } else {
#pragma unroll
                    for (int i = 0; i < kPRows; ++i) vn[c][i] = (u32)(i * 32 + lane) < cnt2 ? src[i * 32] : 0u;
                }
            }
        }
    };
    u64 s = (u64)blockIdx.x * (kPThreads / 32) + (threadIdx.x >> 5);
    if (s < nsub) load_sub(s);
    for (; s < nsub; s += sstep) {
        const u64 ss = s * kSub;
        const u64 cnt = g.nview - ss < (u64)kSub ? g.nview - ss : (u64)kSub;
        const bool full = cnt == (u64)kSub;
        u32 v[KMAX + 1][kPRows];
#pragma unroll
        for (int c = 0; c <= KMAX; ++c)
#pragma unroll
            for (int i = 0; i < kPRows; ++i) v[c][i] = vn[c][i];
        if (s + sstep < nsub) load_sub(s + sstep);
        // geometry (warp-uniform)
        const TileParts tp = tile_parts(g, ss, cnt);
        const u64 t = ss / (u64)T;
        const u64 j0t = v_seg_of(g, t * (u64)T);  // the tile's first segment
        const int sin = (int)(s - t * (u64)nsub_tile);  // subtile inside the tile
        long long bL0 = 0, bR0 = 0, bL1 = 0, bR1 = 0;
        int d00 = 0, d01 = 0;
        u32 y00 = 0, y01 = 0;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            if (p == 1 && !tp.has1) continue;
            const u64 j = tp.j0 + p;
            const u32 pt = j == j0t ? 0u : 1u;
            // below-pivot elements of segment j before this subtile
            u32 below = lane < sin ? a.sub_lt[(t * (u64)nsub_tile + lane) * 2 + pt] : 0u;
            below = __reduce_add_sync(kFullMask, below) + a.tile_lt[t * 2 + pt];
            const u64 ib = p ? tp.ib1 : tp.ib0;
            const u64 before = ss > ib ? ss - ib : 0ull;
            const u64 pb = (before > 0 && a.ppos[j] < ss) ? 1ull : 0ull;
            const long long l = (long long)(ib + below);
            const long long rr = (long long)(ib + v_pivot(g, j) + 1 + (before - below - pb));
            const int d = a.chains[j].d[0];
            const u32 y = flip_key(__uint_as_float(a.piv[j * A + d]));
            if (p == 0) { bL0 = l; bR0 = rr; d00 = d; y00 = y; }
            else { bL1 = l; bR1 = rr; d01 = d; y01 = y; }
        }
        const u32 r0a = tp.r0a, r0b = tp.r0b, r1a = tp.r1a, r1b = tp.r1b;
        if (D0 >= 0 && full && !tp.has1 && r0a == 0 && r0b == (u32)kSub) {
            // lean path: one segment part covers the whole subtile
            const float yf = __uint_as_float(a.piv[tp.j0 * A + (D0 >= 0 ? D0 : 0)]);
            u32 bl = (u32)bL0, br = (u32)bR0;
            u32* dbase = Wdst + lane * 0;
#pragma unroll
            for (int i = 0; i < kPRows; ++i) {
                const float xf = __uint_as_float(v[D0 >= 0 ? D0 : 0][i]);
                int side = xf < yf ? 0 : (xf > yf ? 1 : 2);  // -0.0 == +0.0 like numpy
                if (side == 2) side = part_tie_side(a, tp.j0, ss + (u64)(i * 32 + lane));
                const u32 ml = __ballot_sync(kFullMask, side == 0);
                const u32 mr = __ballot_sync(kFullMask, side == 1);
                const u32 dst = side == 0 ? bl + __popc(ml & lt) : br + __popc(mr & lt);
                bl += __popc(ml);
                br += __popc(mr);
                if (side < 2) {
#pragma unroll
                    for (int c = 0; c <= KMAX; ++c)
                        if (c < A) dbase[(u64)c * stride + dst] = v[c][i];
                }
            }
            continue;
        }
#pragma unroll
        for (int i = 0; i < kPRows; ++i) {
            const u32 r = (u32)(i * 32 + lane);
            const bool in0 = r >= r0a && r < r0b, in1 = r >= r1a && r < r1b;
            int side = 2;  // 2: pivot or outside the parts
            if (in0 || in1) {
                const int dd = in1 ? d01 : d00;
                u32 x = 0;
#pragma unroll
                for (int c = 0; c < KMAX; ++c)
                    if (c == dd) x = v[c][i];
                x = flip_key(__uint_as_float(x));
                const u32 y = in1 ? y01 : y00;
                if (x != y) {
                    side = x < y ? 0 : 1;
                } else {  // tie in the leading field: the rest of the chain, then the index
                    const u64 j = tp.j0 + (in1 ? 1 : 0);
                    const Chain* ch = a.chains + j;
                    const u32* pv = a.piv + j * A;
                    const u32 mm = ch->m;
                    for (u32 f = 1; f < mm && side == 2; ++f) {
                        const int d = ch->d[f];
                        u32 xx = 0;
#pragma unroll
                        for (int c = 0; c < KMAX; ++c)
                            if (c == d) xx = v[c][i];
                        xx = flip_key(__uint_as_float(xx));
                        const u32 yy = flip_key(__uint_as_float(pv[d]));
                        if (xx != yy) side = xx < yy ? 0 : 1;
                    }
                    if (side == 2) {
                        u32 xx = 0;
#pragma unroll
                        for (int c = 0; c <= KMAX; ++c)
                            if (c == k) xx = v[c][i];
                        const u32 yy = pv[k];
                        side = xx < yy ? 0 : (xx > yy ? 1 : 2);
                    }
                }
            }
            const u32 ml = __ballot_sync(kFullMask, side == 0);
            const u32 mr = __ballot_sync(kFullMask, side == 1);
            const u32 pm = __ballot_sync(kFullMask, in1);
            long long dst = -1;
            if (side < 2) {
                const u32 m = (side == 0 ? ml : mr) & (in1 ? pm : ~pm);
                const long long base = side == 0 ? (in1 ? bL1 : bL0) : (in1 ? bR1 : bR0);
                dst = base + __popc(m & lt);
            }
            // advance the four run bases by this row's counts
            bL0 += __popc(ml & ~pm);
            bR0 += __popc(mr & ~pm);
            bL1 += __popc(ml & pm);
            bR1 += __popc(mr & pm);
            if (dst >= 0) {
#pragma unroll
                for (int c = 0; c <= KMAX; ++c)
                    if (c < A) Wdst[(u64)c * stride + (u64)dst] = v[c][i];
            }
        }
    }
}

// Bulk-copy variant (k <= 4): every warp streams its subtiles through a
// private 3-stage shared-memory ring filled by cp.async.bulk (the TMA engine)
// with one mbarrier per stage -- two subtiles in flight per warp without
// holding them in registers.
constexpr int kPStages = 3;
// bulk partition smem: [mbarriers][per-warp fused histograms][per-warp rings]
constexpr size_t kPHistOff = 128 * ((kPThreads / 32) * kPStages * 8 / 128 + 1);
// fused next-level histogram: 2^kFuseD bins per child; warp-private copies
// hold two 16-bit bins per word (flushed at least every 255 subtiles, so a
// bin never exceeds 255 x 256 < 2^16 between flushes)
constexpr int kFuseD = 9;
constexpr int kFuseBins = 1 << kFuseD;
constexpr size_t kPRingOff = kPHistOff + sizeof(u32) * (kPThreads / 32) * 512;

struct PHdr {
    u32 sl[2], tl[2], pp[2], y[2], d[2];  // d: the part's split dim (widest)
};

// NST ring stages, MINB CTAs per SM (occupancy variants, LBKD_PART_CFG)
template <int KMAX, int D0, int NST = kPStages, int MINB = 2>
__global__ void __launch_bounds__(kPThreads, MINB) sel_part_bulk_kernel(SelArgs a, int T) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int kPStages = NST;
    const int lane = threadIdx.x & 31;
    const int k = a.k, A = k + 1;
    const LevelGeom& g = a.g;
    const u32* Wsrc = a.bf.w[a.par];
    u32* Wdst = a.bf.w[a.par ^ 1u];
    const u64 stride = a.bf.stride;
    const u64 nsub = (g.nview + kSub - 1) / kSub;
    const int nsub_tile = T / kSub;
    const u32 lt = lanemask_lt();
    const u64 sstep = (u64)gridDim.x * (kPThreads / 32);
    const int warp = threadIdx.x >> 5;
    u64* bars = reinterpret_cast<u64*>(smem_raw) + warp * kPStages;
    u32* ring = reinterpret_cast<u32*>(smem_raw + kPRingOff) + (size_t)warp * kPStages * (KMAX + 1) * kSub;
    if (lane == 0) {
        for (int st = 0; st < kPStages; ++st) mbar_init(&bars[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](u64 s2, int st) {  // lane 0
        const u64 ss2 = s2 * kSub;
        const u64 cnt2 = g.nview - ss2 < (u64)kSub ? g.nview - ss2 : (u64)kSub;
        const u32 bytes = (u32)(((cnt2 + 3) & ~3ull) * 4);  // arrays padded to 4 words
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier reads of the stage
        mbar_expect_tx(&bars[st], bytes * (u32)A);
        for (int c = 0; c < A; ++c)
            bulk_g2s(ring + ((size_t)st * (KMAX + 1) + c) * kSub, Wsrc + (u64)c * stride + ss2, bytes, &bars[st]);
    };
    // each warp owns a contiguous run of subtiles (the fused histogram of the
    // next level then changes segment rarely; interleaving the warps of a CTA
    // over one run measured 10% slower)
    const u64 nw = (u64)gridDim.x * (kPThreads / 32);
    const u64 chunk = (nsub + nw - 1) / nw;
    u64 s = ((u64)blockIdx.x * (kPThreads / 32) + warp) * chunk;
    const u64 s_end = s + chunk < nsub ? s + chunk : nsub;
    constexpr u64 sd = 1;
    if (lane == 0) {
        for (int q = 0; q < kPStages - 1; ++q)
            if (s + q * sd < s_end) issue(s + q * sd, q);
    }
    // fused histogram of the next level (its two children of one segment,
    // warp-private 2 x 256 bins), flushed when the segment changes
    u32* wh = reinterpret_cast<u32*>(smem_raw + kPHistOff) + warp * 512;
    const bool fuse = a.hist_next != nullptr;
    u64 hseg = ~0ull;
    Bucketer hb0{}, hb1{};
    const int dn = (g.l + 1) % k;
    int hdn0 = dn, hdn1 = dn;  // the children's dims (widest: per segment)
    int hcnt = 0;  // subtiles binned since the last flush
    auto hflush = [&]() {
        if (hseg != ~0ull) {
            for (int i = lane; i < 512; i += 32) {
                const u32 v = wh[i];
                if (v) {
                    u32* gh = a.hist_next + (2 * hseg + (i >> 8)) * (u64)kFuseBins + 2 * (i & 255);
                    if (v & 0xffffu) atomicAdd(gh, v & 0xffffu);
                    if (v >> 16) atomicAdd(gh + 1, v >> 16);
                    wh[i] = 0u;
                }
            }
        }
        hcnt = 0;
        __syncwarp();
    };
    if (fuse) {
        for (int i = lane; i < 512; i += 32) wh[i] = 0u;
        __syncwarp();
    }
    // per-subtile header: per segment part the lane's sub_lt word, the
    // tile_lt prefix, the pivot position and the pivot's key
    const int tsh = 31 - __clz(T);  // T is a power of two
    auto hdr_load = [&](u64 s2, PHdr& h2) {
        const u64 ss2 = s2 * kSub;
        const u64 cnt2 = g.nview - ss2 < (u64)kSub ? g.nview - ss2 : (u64)kSub;
        const TileParts tp2 = tile_parts(g, ss2, cnt2);
        const u64 t2 = ss2 >> tsh;
        const u64 j0t = v_seg_of(g, t2 << tsh);  // the tile's first segment
        const int sin = (int)(s2 - t2 * (u64)nsub_tile);  // subtile inside the tile
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            h2.sl[p] = 0u; h2.tl[p] = 0u; h2.pp[p] = 0u; h2.y[p] = 0u; h2.d[p] = D0 >= 0 ? (u32)D0 : 0u;
            if (p == 1 && !tp2.has1) continue;
            const u64 j = tp2.j0 + p;
            const u32 pt = j == j0t ? 0u : 1u;
            h2.sl[p] = lane < sin ? a.sub_lt[(t2 * (u64)nsub_tile + lane) * 2 + pt] : 0u;
            h2.tl[p] = a.tile_lt[t2 * 2 + pt];
            h2.pp[p] = a.ppos[j];
            if (D0 < 0) h2.d[p] = (u32)a.split_dims[g.Fl + g.sbase + j];  // widest: the segment's dim
            h2.y[p] = a.piv[j * A + h2.d[p]];
        }
    };
    PHdr hn;
    if (s < s_end) hdr_load(s, hn);
    // per-column destination bases (the stores then need one 32-bit-offset
    // address add each instead of a 64-bit column*stride product per row)
    u32* dcol[KMAX + 1];
#pragma unroll
    for (int c = 0; c <= KMAX; ++c) dcol[c] = Wdst + (u64)(c < A ? c : 0) * stride;
    u32 phases = 0u;
    int stage = 0;
    for (; s < s_end; s += sd) {
        const u64 ss = s * kSub;
        const u64 cnt = g.nview - ss < (u64)kSub ? g.nview - ss : (u64)kSub;
        const bool full = cnt == (u64)kSub;
        if (lane == 0 && s + (kPStages - 1) * sd < s_end)
            issue(s + (kPStages - 1) * sd, (stage + kPStages - 1) % kPStages);
        mbar_wait(&bars[stage], (phases >> stage) & 1u);
        phases ^= 1u << stage;
        const u32* sv = ring + (size_t)stage * (KMAX + 1) * kSub + lane;
#define V(c, i) (sv[(c) * kSub + (i) * 32])
        // geometry (warp-uniform); the header words were loaded one subtile
        // ahead (hdr_load) so their L2 latency overlaps the previous subtile
        const TileParts tp = tile_parts(g, ss, cnt);
        const PHdr h = hn;
        if (s + sd < s_end) hdr_load(s + sd, hn);
        long long bL0 = 0, bR0 = 0, bL1 = 0, bR1 = 0;
        const int d00 = (int)h.d[0], d01 = (int)h.d[1];  // round robin: D0 for every segment
        u32 y00 = 0, y01 = 0;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            if (p == 1 && !tp.has1) continue;
            const u64 j = tp.j0 + p;
            // below-pivot elements of segment j before this subtile
            const u32 below = __reduce_add_sync(kFullMask, h.sl[p]) + h.tl[p];
            const u64 ib = p ? tp.ib1 : tp.ib0;
            const u64 before = ss > ib ? ss - ib : 0ull;
            const u64 pb = (before > 0 && h.pp[p] < ss) ? 1ull : 0ull;
            const long long l = (long long)(ib + below);
            const long long rr = (long long)(ib + v_pivot(g, j) + 1 + (before - below - pb));
            const u32 y = flip_key(__uint_as_float(h.y[p]));
            if (p == 0) { bL0 = l; bR0 = rr; y00 = y; }
            else { bL1 = l; bR1 = rr; y01 = y; }
        }
        const u32 r0a = tp.r0a, r0b = tp.r0b, r1a = tp.r1a, r1b = tp.r1b;
        if (full && !tp.has1 && r0a == 0 && r0b == (u32)kSub) {
            // lean path: one segment part covers the whole subtile
            const int dl0 = D0 >= 0 ? D0 : d00;
            const float yf = __uint_as_float(a.piv[tp.j0 * A + dl0]);
            u32 bl = (u32)bL0, br = (u32)bR0;
            if (fuse && tp.j0 != hseg) {
                hflush();
                hseg = tp.j0;
                const float* c0 = a.boxes_out + (2 * hseg) * 2ull * k;
                const float* c1 = c0 + 2 * k;
                if (D0 < 0) {  // widest: the children's own split dims (written by select)
                    const u64 cn = 2 * (g.Fl + g.sbase + hseg) + 1;
                    hdn0 = cn < g.n ? (int)a.split_dims[cn] : 0;
                    hdn1 = cn + 1 < g.n ? (int)a.split_dims[cn + 1] : 0;
                } else {  // round-robin: the children's key dims at level l + 1 (rr_key_dim)
                    const int e0 = rr_key_dim(c0, k, g.l + 1), e1 = rr_key_dim(c1, k, g.l + 1);
                    hdn0 = e0 >= 0 ? e0 : dn;
                    hdn1 = e1 >= 0 ? e1 : dn;
                }
                hb0 = make_bucketer(c0[hdn0], c0[k + hdn0], kFuseD, a.bmode_out[2 * hseg]);
                hb1 = make_bucketer(c1[hdn1], c1[k + hdn1], kFuseD, a.bmode_out[2 * hseg + 1]);
            }
            if (fuse) {
                if (hcnt >= a.hflush_every) hflush();  // 16-bit bins: flush before they could overflow
                ++hcnt;
            }
            // (1) every row's side by one float compare, 2 bits per row; (2)
            // the rare ties (-> chain, index) in a separate pass, so the
            // call does not split the rows' instruction streams; (3) ranks,
            // fused histogram and stores, the bucket mode hoisted out
            u32 sides = 0;
#pragma unroll
            for (int i = 0; i < kPRows; ++i) {
                const float xf = __uint_as_float(V(dl0, i));
                const u32 sd = xf < yf ? 0u : (xf > yf ? 1u : 2u);  // -0.0 == +0.0 like numpy
                sides |= sd << (2 * i);
            }
            if (__any_sync(kFullMask, (sides & 0xAAAAu) != 0u)) {
                for (int i = 0; i < kPRows; ++i) {
                    if (((sides >> (2 * i)) & 3u) == 2u) {
                        const u32 sd = (u32)part_tie_side(a, tp.j0, ss + (u64)(i * 32 + lane));
                        sides = (sides & ~(3u << (2 * i))) | (sd << (2 * i));
                    }
                }
            }
            auto rows = [&](auto bucket_fn) {
#pragma unroll
                for (int i = 0; i < kPRows; ++i) {
                    const int side = (int)((sides >> (2 * i)) & 3u);
                    const u32 ml = __ballot_sync(kFullMask, side == 0);
                    const u32 mr = __ballot_sync(kFullMask, side == 1);
                    const u32 dst = side == 0 ? bl + __popc(ml & lt) : br + __popc(mr & lt);
                    bl += __popc(ml);
                    br += __popc(mr);
                    if (fuse && side < 2) {
                        const u32 kn = V(side ? hdn1 : hdn0, i);
                        const u32 hbk = bucket_fn(side ? hb1 : hb0, kn);
                        atomicAdd(&wh[side * 256 + (hbk >> 1)], (hbk & 1u) ? 0x10000u : 1u);
                    }
                    if (side < 2) {
#pragma unroll
                        for (int c = 0; c <= KMAX; ++c)
                            if (c < A) dcol[c][dst] = V(c, i);
                    }
                }
            };
            // (both children of a node share their bucket mode: select.cu)
            if (fuse && key_mode(hb0)) rows([](const Bucketer& b, u32 x) { return bucket_key(b, x); });
            else rows([](const Bucketer& b, u32 x) { return bucket_val(b, x); });
        } else {
#pragma unroll
        for (int i = 0; i < kPRows; ++i) {
            const u32 r = (u32)(i * 32 + lane);
            const bool in0 = r >= r0a && r < r0b, in1 = r >= r1a && r < r1b;
            int side = 2;  // 2: pivot or outside the parts
            if (in0 || in1) {
                const int dd = in1 ? d01 : d00;
                u32 x = 0;
#pragma unroll
                for (int c = 0; c < KMAX; ++c)
                    if (c == dd) x = V(c, i);
                x = flip_key(__uint_as_float(x));
                const u32 y = in1 ? y01 : y00;
                if (x != y) {
                    side = x < y ? 0 : 1;
                } else {  // tie in the leading field: the rest of the chain, then the index
                    const u64 j = tp.j0 + (in1 ? 1 : 0);
                    const Chain* ch = a.chains + j;
                    const u32* pv = a.piv + j * A;
                    const u32 mm = ch->m;
                    for (u32 f = 1; f < mm && side == 2; ++f) {
                        const int d = ch->d[f];
                        u32 xx = 0;
#pragma unroll
                        for (int c = 0; c < KMAX; ++c)
                            if (c == d) xx = V(c, i);
                        xx = flip_key(__uint_as_float(xx));
                        const u32 yy = flip_key(__uint_as_float(pv[d]));
                        if (xx != yy) side = xx < yy ? 0 : 1;
                    }
                    if (side == 2) {
                        u32 xx = 0;
#pragma unroll
                        for (int c = 0; c <= KMAX; ++c)
                            if (c == k) xx = V(c, i);
                        const u32 yy = pv[k];
                        side = xx < yy ? 0 : (xx > yy ? 1 : 2);
                    }
                }
            }
            if (fuse && side < 2) {
                const u64 j = tp.j0 + (in1 ? 1 : 0);
                const float* cb = a.boxes_out + (2 * j + side) * 2ull * k;
                const u64 cn = 2 * (g.Fl + g.sbase + j) + 1 + side;
                int dnc = D0 >= 0 ? dn : (cn < g.n ? (int)a.split_dims[cn] : 0);
                if (D0 >= 0) {
                    const int e = rr_key_dim(cb, k, g.l + 1);
                    if (e >= 0) dnc = e;
                }
                const Bucketer hb = make_bucketer(cb[dnc], cb[k + dnc], kFuseD, a.bmode_out[2 * j + side]);
                atomicAdd(&a.hist_next[(2 * j + side) * (u64)kFuseBins + bucket_of(hb, V(dnc, i))], 1u);
            }
            const u32 ml = __ballot_sync(kFullMask, side == 0);
            const u32 mr = __ballot_sync(kFullMask, side == 1);
            const u32 pm = __ballot_sync(kFullMask, in1);
            long long dst = -1;
            if (side < 2) {
                const u32 m = (side == 0 ? ml : mr) & (in1 ? pm : ~pm);
                const long long base = side == 0 ? (in1 ? bL1 : bL0) : (in1 ? bR1 : bR0);
                dst = base + __popc(m & lt);
            }
            // advance the four run bases by this row's counts
            bL0 += __popc(ml & ~pm);
            bR0 += __popc(mr & ~pm);
            bL1 += __popc(ml & pm);
            bR1 += __popc(mr & pm);
            if (dst >= 0) {
#pragma unroll
                for (int c = 0; c <= KMAX; ++c)
                    if (c < A) dcol[c][dst] = V(c, i);
            }
        }
        }
#undef V
        __syncwarp();  // every lane is done with this stage before it is refilled
        stage = stage + 1 == kPStages ? 0 : stage + 1;
    }
    if (fuse) hflush();
}


// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
int sel_items(int b) {
    int items = (1 << (b - 1)) / 256;
    return items > 8 ? 8 : items;
}

// tile of the filter / select scan: at most two segment parts per tile
int sel_tile(int b) { return 256 * sel_items(b); }

int sel_digit_bits(u64 nseg) {
    int lg = 0;
    while ((1ull << lg) < nseg) ++lg;
    int D = 20 - lg;
    return D < 8 ? 8 : (D > 11 ? 11 : D);
}

void launch_sel_hist(const SelArgs& a0, int b, cudaStream_t st) {
    SelArgs a = a0;
    int items = (1 << (b - 1)) / kHThreads;
    if (items > 8) items = 8;
    const u64 T = (u64)kHThreads * items;
    a.ntiles = (a.g.nview + T - 1) / T;
    // CTAs per SM (LBKD_HIST_CTAS_PER_SM): measured 16 > 8 > 4 > 2 -- the
    // per-CTA flush of up to 2^D global atomics costs less than lost
    // parallelism (0.66 / 0.74 / 0.74 / 1.16 ms per build at 100M)
    u64 per_sm = 16;
    if (const char* e = getenv("LBKD_HIST_CTAS_PER_SM")) {
        const int v = atoi(e);
        if (v >= 1 && v <= 32) per_sm = (u64)v;
    }
    const u64 target = 148 * per_sm;
    u64 tpc = (a.ntiles + target - 1) / target;
    if (tpc < 1) tpc = 1;
    a.tiles_per_cta = (int)tpc;
    const unsigned grid = (unsigned)((a.ntiles + tpc - 1) / tpc);
    const size_t sm = sizeof(u32) << a.D;
    // tile <= 2^(b-1) <= the smallest segment: at most two parts per tile
    switch (items) {
        case 8: sel_hist_kernel<8><<<grid, kHThreads, sm, st>>>(a); break;
        case 4: sel_hist_kernel<4><<<grid, kHThreads, sm, st>>>(a); break;
        case 2: sel_hist_kernel<2><<<grid, kHThreads, sm, st>>>(a); break;
        default: sel_hist_kernel<1><<<grid, kHThreads, sm, st>>>(a); break;
    }
}

void launch_sel_pick(const SelArgs& a, cudaStream_t st) {
    sel_pick_kernel<<<(unsigned)a.g.nseg, 256, 0, st>>>(a);
}

void launch_sel_filter(const SelArgs& a0, int b, cudaStream_t st) {
    SelArgs a = a0;
    const int T = sel_tile(b);
    a.ntiles = (a.g.nview + T - 1) / T;
    const u64 grid = a.ntiles < 148 * 8 ? a.ntiles : 148 * 8;
    // contiguous runs of tiles per CTA (the segment cursor advances locally);
    // CTAs per SM (LBKD_FILTER_CTAS_PER_SM): measured at 100M, 2048-point
    // tiles (RR) best at 32 (2.30 ms vs 2.38 at 16), 1024-point tiles
    // (widest) at 64 (2.87 vs 3.10)
    u64 per_sm = T >= 2048 ? 32 : 64;
    if (const char* e = getenv("LBKD_FILTER_CTAS_PER_SM")) {
        const int v = atoi(e);
        if (v >= 1 && v <= 64) per_sm = (u64)v;
    }
    const u64 target = 148 * per_sm;
    u64 tpc = (a.ntiles + target - 1) / target;
    if (tpc < 1) tpc = 1;
    a.tiles_per_cta = (int)tpc;
    const unsigned g2 = (unsigned)((a.ntiles + tpc - 1) / tpc);
    (void)grid;
    const size_t sm = sizeof(u32) * (1 + (size_t)kFCap * (1 + a.k + 2));  // count, segment ids, records
    auto go = [&](auto kern, int nt) {
        if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        kern<<<g2, nt, sm, st>>>(a);
    };
    switch (T) {
        case 2048: go(sel_filter_kernel<256>, 256); break;
        case 1024: go(sel_filter_kernel<128>, 128); break;
        case 512: go(sel_filter_kernel<64>, 64); break;
        default: go(sel_filter_kernel<32>, 32); break;
    }
}

void launch_sel_select(const SelArgs& a, int b, cudaStream_t st) {
    // few segments with many candidates (top levels): wide CTAs; many
    // segments with a few candidates (deep levels): narrow CTAs
    // (the top levels' segments as clusters of CTAs: a segment can hold
    // millions of candidates on tie-heavy or wide-range data)
    const unsigned g = (unsigned)a.g.nseg;
    auto cluster_go = [&](auto kern, int nt, int cs) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(g * (unsigned)cs);
        cfg.blockDim = dim3((unsigned)nt);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, a, sel_tile(b));
    };
    // LBKD_SELECT_CLUSTER (default 10): at nseg <= 16 clusters of 8 (bit 3)
    // or 4 (bit 2) CTAs of 1024 threads; at nseg <= 128 clusters of 8 (bit 4)
    // or 4 (bit 1) CTAs of 256; 0 = one CTA per segment everywhere
    static const int csel = [] {
        const char* e = getenv("LBKD_SELECT_CLUSTER");
        return e ? atoi(e) : 10;
    }();
    if (a.g.nseg <= 16) {
        if (csel & 8) cluster_go(sel_select_kernel<1024, 8>, 1024, 8);
        else if (csel & 4) cluster_go(sel_select_kernel<1024, 4>, 1024, 4);
        else sel_select_kernel<1024, 1><<<g, 1024, 0, st>>>(a, sel_tile(b));
    } else if (a.g.nseg <= 128 && (csel & 16)) {
        cluster_go(sel_select_kernel<256, 8>, 256, 8);
    } else if (a.g.nseg <= 128 && (csel & 2)) {
        cluster_go(sel_select_kernel<256, 4>, 256, 4);
    } else if (a.g.nseg >= 2048) {
        sel_select_kernel<64, 1><<<g, 64, 0, st>>>(a, sel_tile(b));
    } else {
        sel_select_kernel<256, 1><<<g, 256, 0, st>>>(a, sel_tile(b));
    }
}

void launch_sel_part(const SelArgs& a0, int b, cudaStream_t st) {
    SelArgs a = a0;
    // the fused histogram's 16-bit warp bins take <= 255 subtiles x 256
    // points between flushes; LBKD_HFLUSH_EVERY lowers it (tests of the
    // flush path at small sizes)
    a.hflush_every = 255;
    if (const char* e = getenv("LBKD_HFLUSH_EVERY")) {
        const int v = atoi(e);
        if (v >= 1 && v < 255) a.hflush_every = v;
    }
    const int T = sel_tile(b);
    const u64 nsub = (a.g.nview + kSub - 1) / kSub;
    const u64 per_cta = kPThreads / 32;
    u64 grid = (nsub + per_cta - 1) / per_cta;
    const u64 cap = 148ull * 8;
    if (grid > cap) grid = cap;
    // register-resident subtile: (KMAX + 1) x 8 words per lane
    const int d0 = a.mode == kRoundRobin ? a.g.l % a.k : -1;  // RR: every segment splits dim l mod k
    auto bulk_go = [&](auto kern, int KM, int nst = kPStages, int minb = 2) {
        const size_t sm = kPRingOff + sizeof(u32) * (size_t)(kPThreads / 32) * nst * (KM + 1) * kSub;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        u64 g2 = (nsub + per_cta - 1) / per_cta;
        if (g2 > 148ull * minb) g2 = 148ull * minb;  // persistent: minb CTAs per SM
        kern<<<(unsigned)g2, kPThreads, sm, st>>>(a, T);
    };
#define LBKD_PART_D(KM, D) bulk_go(sel_part_bulk_kernel<KM, D>, KM)
#define LBKD_PART(KM)                                                                          \
    switch (d0) {                                                                              \
        case 0: LBKD_PART_D(KM, 0); break;                                                     \
        case 1: LBKD_PART_D(KM, (KM > 1 ? 1 : 0)); break;                                      \
        case 2: LBKD_PART_D(KM, (KM > 2 ? 2 : 0)); break;                                      \
        case 3: LBKD_PART_D(KM, (KM > 3 ? 3 : 0)); break;                                      \
        default: LBKD_PART_D(KM, -1); break; /* widest: per-segment dims */                    \
    }
    switch (a.k) {
        case 1: LBKD_PART(1); break;
        case 2: LBKD_PART(2); break;
        case 3: LBKD_PART(3); break;
        case 4: LBKD_PART(4); break;
        default:
            if (a.k <= 8) sel_part_kernel<8, -1><<<(unsigned)grid, kPThreads, 0, st>>>(a, T);
            else sel_part_kernel<16, -1><<<(unsigned)grid, kPThreads, 0, st>>>(a, T);
            break;
    }
#undef LBKD_PART
#undef LBKD_PART_D
}

}  // namespace lbkd
