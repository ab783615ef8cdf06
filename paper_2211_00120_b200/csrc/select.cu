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
// Round robin (k = 2..4) runs the levels in PAIRS: after level l's select,
// level l+1 is selected in level l's layout (child hist, pick, filter pair,
// select with per-side counts) and one stable 4-way partition moves every
// point to its grandchild's run -- see "Level pairs" below and DESIGN.md §2.
//
// Layout: in-order SoA as in global_sort.cu -- segment j of level l occupies
// [ib(j), ib(j) + ss(j)) of W[(l - lfirst) & 1]; finished nodes leave a hole.
#include "kernels.cuh"

#include <cooperative_groups.h>

#include <cstdlib>
#include <type_traits>

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

// Level pairs: the key of a level-(l+1) child that still lies in its
// parent's layout.  rr_key_dim as usual; a child whose chain dims are all
// pinned (its order is the input order) is keyed by its INDEX column (k),
// key-linear over [0, n) -- an index is a nonnegative u32, so its float
// bits' flipped key is the index plus 2^31, monotone -- instead of being
// made positional (its in-order slot is not known before the split).
struct PairKey {
    int d;
    float lo, hi;
    int mode;
};

__device__ __forceinline__ PairKey pair_child_key(const float* box, uint8_t bmode, int k, int l1, u64 n,
                                                  int wd = -1) {
    PairKey p;
    // round robin: rr_key_dim; widest (wd = the child's split dim): that dim
    // unless the box is a single point
    int d;
    if (wd < 0) {
        d = rr_key_dim(box, k, l1);
    } else {
        bool point = true;
        for (int c = 0; c < k; ++c) point &= box[c] == box[k + c];
        d = point ? -1 : wd;
    }
    if (d >= 0) {
        p.d = d;
        p.lo = box[d];
        p.hi = box[k + d];
        p.mode = bmode;
    } else {
        p.d = k;
        p.lo = __uint_as_float(0u);
        p.hi = __uint_as_float((u32)n);
        p.mode = 1;
    }
    return p;
}

// the key of view segment c of level a.g.l (a pair's second level); widest:
// the split dim the first level's select wrote for that node
__device__ __forceinline__ PairKey pair_key_of(const SelArgs& a, u64 c) {
    const int wd = a.mode == kWidest ? (int)a.split_dims[a.g.Fl + a.g.sbase + c] : -1;
    return pair_child_key(a.boxes_in + c * 2ull * a.k, a.bmode_in[c], a.k, a.g.l, a.g.n, wd);
}

// side of the point at layout position pos against a pivot whose leading
// coordinate it ties: the rest of the node's chain, then the input row
// (0 below, 1 above, 2 the pivot itself)
__device__ __noinline__ int tie_side_of(const u32* W, u64 stride, int k, const Chain* ch, const u32* pv, u64 pos) {
    const u32 mm = ch->m;
    for (u32 f = 1; f < mm; ++f) {
        const int d = ch->d[f];
        const u32 xx = flip_key(__uint_as_float(W[(u64)d * stride + pos]));
        const u32 yy = flip_key(__uint_as_float(pv[d]));
        if (xx != yy) return xx < yy ? 0 : 1;
    }
    const u32 xx = W[(u64)k * stride + pos], yy = pv[k];
    return xx < yy ? 0 : (xx > yy ? 1 : 2);
}

// the same, skipping the chain fields whose dim the node's box pins (every
// point of the node ties there: identical / tie-heavy data)
__device__ __noinline__ int tie_side_pinned(const u32* W, u64 stride, int k, const Chain* ch, const u32* pv, u64 pos,
                                            u32 pinned) {
    const u32 mm = ch->m;
    for (u32 f = 1; f < mm; ++f) {
        if ((pinned >> f) & 1u) continue;
        const int d = ch->d[f];
        const u32 xx = flip_key(__uint_as_float(W[(u64)d * stride + pos]));
        const u32 yy = flip_key(__uint_as_float(pv[d]));
        if (xx != yy) return xx < yy ? 0 : 1;
    }
    const u32 xx = W[(u64)k * stride + pos], yy = pv[k];
    return xx < yy ? 0 : (xx > yy ? 1 : 2);
}

// chain fields (bit f) whose dim a box pins
__device__ __forceinline__ u32 pinned_fields(const Chain* ch, const float* box, int k) {
    u32 m = 0;
    for (u32 f = 1; f < ch->m; ++f) {
        const int d = ch->d[f];
        if (box[d] == box[k + d]) m |= 1u << f;  // (== : a NaN bound from non-finite input pins nothing)
    }
    return m;
}

// the same, for a row of a partition subtile staged in shared memory (the
// warp's TMA ring: column c of row i at sv[c * 256 + i * 32], sv = the
// lane's base) -- no global re-reads on tie-heavy data
__device__ __forceinline__ u32 tie_side_ring(const u32* sv, int i, int k, const Chain* ch, const u32* pv) {
    const u32 mm = ch->m;
    for (u32 f = 1; f < mm; ++f) {
        const int d = ch->d[f];
        const u32 xx = flip_key(__uint_as_float(sv[d * 256 + i * 32]));
        const u32 yy = flip_key(__uint_as_float(pv[d]));
        if (xx != yy) return xx < yy ? 0u : 1u;
    }
    const u32 xx = sv[k * 256 + i * 32], yy = pv[k];
    return xx < yy ? 0u : (xx > yy ? 1u : 2u);
}

// the build's abort word (Buffers::err[1], set with the non-finite flag by
// the init / check kernels): every later kernel of the build returns at
// once, so NaN / inf input never drives the selection's invariants (the
// counts of one kernel against the compares of the next) out of range
__device__ __forceinline__ bool aborted(const SelArgs& a) { return a.bf.err && a.bf.err[1] != 0u; }

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

// field-wise select of two bucketers (a conditional on the structs would
// take their addresses: local memory)
__device__ __forceinline__ Bucketer bsel2(bool second, const Bucketer& b0, const Bucketer& b1) {
    Bucketer b;
    b.hlo = second ? b1.hlo : b0.hlo;
    b.scale = second ? b1.scale : b0.scale;
    b.top = second ? b1.top : b0.top;
    return b;
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
    if (__any_sync(kFullMask, bad) && (threadIdx.x & 31) == 0) {
        atomicOr(err, 1u);
        atomicOr(err + 1, 1u);  // this build's abort word (kernels after init return at once)
    }
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

// k = 3, 16-byte aligned input: four points per thread step -- three
// 16-byte loads of 12 floats, one 16-byte store per SoA column
__global__ void __launch_bounds__(256) init_stats3_kernel(const float4* __restrict__ pts4, u64 n, u32* w0, u64 stride,
                                                          u32* err, u32* minmax) {
    __shared__ u32 smn[3], smx[3];
    if (threadIdx.x < 3) { smn[threadIdx.x] = 0xffffffffu; smx[threadIdx.x] = 0u; }
    __syncthreads();
    u32 mn[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, mx[3] = {0u, 0u, 0u};
    bool bad = false;
    auto one = [&](int c, float f) {
        bad |= !isfinite(f);
        const u32 key = flip_key(f);
        mn[c] = min(mn[c], key);
        mx[c] = max(mx[c], key);
    };
    const u64 ng = n / 4;
    for (u64 g = blockIdx.x * (u64)blockDim.x + threadIdx.x; g < ng; g += (u64)gridDim.x * blockDim.x) {
        const float4 a = __ldg(pts4 + 3 * g), b = __ldg(pts4 + 3 * g + 1), c = __ldg(pts4 + 3 * g + 2);
        const float x[4] = {a.x, a.w, b.z, c.y}, y[4] = {a.y, b.x, b.w, c.z}, z[4] = {a.z, b.y, c.x, c.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) { one(0, x[i]); one(1, y[i]); one(2, z[i]); }
        const u64 p = 4 * g;
        *reinterpret_cast<uint4*>(w0 + p) = make_uint4(__float_as_uint(x[0]), __float_as_uint(x[1]), __float_as_uint(x[2]), __float_as_uint(x[3]));
        *reinterpret_cast<uint4*>(w0 + stride + p) = make_uint4(__float_as_uint(y[0]), __float_as_uint(y[1]), __float_as_uint(y[2]), __float_as_uint(y[3]));
        *reinterpret_cast<uint4*>(w0 + 2 * stride + p) = make_uint4(__float_as_uint(z[0]), __float_as_uint(z[1]), __float_as_uint(z[2]), __float_as_uint(z[3]));
        *reinterpret_cast<uint4*>(w0 + 3 * stride + p) = make_uint4((u32)p, (u32)p + 1u, (u32)p + 2u, (u32)p + 3u);
    }
    if (blockIdx.x == 0 && threadIdx.x < n - 4 * ng) {  // the last n mod 4 points
        const u64 i = 4 * ng + threadIdx.x;
        const float* q = reinterpret_cast<const float*>(pts4) + 3 * i;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float f = __ldg(q + c);
            one(c, f);
            w0[c * stride + i] = __float_as_uint(f);
        }
        w0[3 * stride + i] = (u32)i;
    }
    if (__any_sync(kFullMask, bad) && (threadIdx.x & 31) == 0) {
        atomicOr(err, 1u);
        atomicOr(err + 1, 1u);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const u32 a = __reduce_min_sync(kFullMask, mn[c]);
        const u32 b = __reduce_max_sync(kFullMask, mx[c]);
        if ((threadIdx.x & 31) == 0) { atomicMin(&smn[c], a); atomicMax(&smx[c], b); }
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        atomicMin(&minmax[threadIdx.x], smn[threadIdx.x]);
        atomicMax(&minmax[3 + threadIdx.x], smx[threadIdx.x]);
    }
}

void launch_init_stats(const BuildParams& bp, const Buffers& bf, u32* minmax, cudaStream_t st) {
    if (bp.k == 3 && ((uintptr_t)bp.pts & 15u) == 0 && (bf.stride & 3u) == 0 && !getenv("LBKD_INIT_SCALAR")) {
        u64 blocks = (bp.n / 4 + 255) / 256;
        if (blocks > 148 * 8) blocks = 148 * 8;
        if (blocks < 1) blocks = 1;
        init_stats3_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(bp.pts), bp.n, bf.w[0],
                                                             bf.stride, bf.err, minmax);
        return;
    }
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
    if (__any_sync(kFullMask, bad) && (threadIdx.x & 31) == 0) {
        atomicOr(err, 1u);
        atomicOr(err + 1, 1u);
    }
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
    if (aborted(a)) return;  // non-finite input: the build is reported, not run
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
        // ITEMS consecutive positions per thread
        const u32 rb0 = (u32)threadIdx.x * ITEMS;
        u32 key[ITEMS];
        // (vector loads only inside one part: the finished nodes' slots
        // between segments are never written in this buffer)
        if (ITEMS % 4 == 0 && ((rb0 >= r0a && rb0 + ITEMS <= r0b) || (has1 && rb0 >= r1a && rb0 + ITEMS <= r1b))) {
#pragma unroll
            for (int i = 0; i < ITEMS; i += 4) {
                const uint4 q = *reinterpret_cast<const uint4*>(kp + ts + rb0 + i);
                key[i] = q.x; key[i + 1] = q.y; key[i + 2] = q.z; key[i + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const u32 r = rb0 + (u32)i;
                const bool use = (r >= r0a && r < r0b) || (has1 && r >= r1a && r < r1b);
                key[i] = use ? kp[ts + r] : 0u;
            }
        }
        if (has1 && nseg_c != cur + 1) {  // the next segment's key dim, once per segment
            nseg_c = cur + 1;
            dk1 = seg_key_dim(a, cur + 1);
        }
        if (has1 && dk1 != dk) {  // the next segment is keyed by another dim
            const u32* k1 = W + (u64)dk1 * a.bf.stride;
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const u32 r = rb0 + (u32)i;
                if (r >= r1a && r < r1b) key[i] = k1[ts + r];
            }
        }
        // (the bucket mode hoisted out of the per-key loops)
        auto bin = [&](u32 ra, u32 rb) {
            if (key_mode(bk)) {
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const u32 r = rb0 + (u32)i;
                    if (r >= ra && r < rb) atomicAdd(&h[bucket_key(bk, key[i])], 1u);
                }
            } else {
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const u32 r = rb0 + (u32)i;
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
    if (aborted(a)) return;  // non-finite input: the build is reported, not run
    __shared__ u32 wtot[32];
    const u64 j = blockIdx.x;
    // a node box that is a single point (every coordinate of every point of
    // the segment equal): the within-node order is the input order, which is
    // the segment's order in W (stable partitions) -- the node is the element
    // at in-order offset pivot_off, no histogram and no candidates to sort
    if (!a.pair) {  // (level pairs: such a child is keyed by its index column, pair_child_key)
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
        const float* box = a.boxes_in + j * 2ull * a.k;
        if (a.pair) {
            const PairKey pk = pair_key_of(a, j);
            sel[kSelLo] = __float_as_uint(pk.lo);
            sel[kSelShift] = __float_as_uint(pk.hi);
            sel[kSelMode] = (u32)pk.mode;
        } else {
            const int d = seg_key_dim(a, j);
            sel[kSelLo] = __float_as_uint(box[d]);  // the filter rebuilds the bucketer
            sel[kSelShift] = __float_as_uint(box[a.k + d]);
            sel[kSelMode] = a.bmode_in[j];
        }
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
    if (aborted(a)) return;  // non-finite input: the build is reported, not run
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
    if (aborted(a)) return;  // non-finite input: the build is reported, not run
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
    // (level pairs: the candidates' positions and the count slots are those
    // of the PARENT's layout, one count array per child side)
    const u64 jl = a.pair ? (j >> 1) : j;
    const LevelGeom& gl = a.pair ? a.g0 : g;
    u32* const tlt = a.tile_lt + (a.pair ? (j & 1) * a.lt_tstride : 0ull);
    u32* const slt = a.sub_lt + (a.pair ? (j & 1) * a.lt_sstride : 0ull);
    const u64 ib = v_ibegin(gl, jl);
    const u64 tfirst = ib / (u64)T;
    const u64 tlast = (ib + v_size(gl, jl) - 1) / (u64)T;
    const u32 pfirst = (ib == tfirst * (u64)T) ? 0u : 1u;
    auto count_below = [&](const u32* rec) {
        const u64 pos = rec[k + 1];
        const u64 t = pos / (u64)T;
        const u32 pt = t == tfirst ? pfirst : 0u;
        atomicAdd(&tlt[t * 2 + pt], 1u);
        atomicAdd(&slt[(pos / (u64)kSub) * 2 + pt], 1u);
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
        u32* slot = t <= tlast ? &tlt[t * 2 + (t == tfirst ? pfirst : 0u)] : nullptr;
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
__device__ __forceinline__ int part_tie_side(const SelArgs& a, u64 j, u64 pos) {
    return tie_side_of(a.bf.w[a.par], a.bf.stride, a.k, a.chains + j, a.piv + j * (a.k + 1), pos);
}

// D0 >= 0: every segment's leading key is coordinate D0 (round-robin): full
// single-part subtiles take a lean path (float compares, no part masks)
template <int KMAX, int D0>
__global__ void __launch_bounds__(kPThreads, KMAX <= 4 ? 2 : 1) sel_part_kernel(SelArgs a, int T) {
    if (aborted(a)) return;  // non-finite input: the build is reported, not run
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
    if (aborted(a)) return;  // non-finite input: the build is reported, not run
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
                const Chain* tch = a.chains + tp.j0;
                const u32* tpv = a.piv + tp.j0 * A;
#pragma unroll 1
                for (int i = 0; i < kPRows; ++i) {
                    if (((sides >> (2 * i)) & 3u) == 2u) {
                        const u32 sd = tie_side_ring(sv, i, k, tch, tpv);
                        sides = (sides & ~(3u << (2 * i))) | (sd << (2 * i));
                    }
                }
            }
            // in phases so the rows' dependency chains overlap: all ballots,
            // then the destinations (two running sums), then histogram + stores
            auto rows = [&](auto bucket_fn) {
                u32 ml[kPRows], mr[kPRows], dsts[kPRows];
#pragma unroll
                for (int i = 0; i < kPRows; ++i) {
                    const u32 sd = (sides >> (2 * i)) & 3u;
                    ml[i] = __ballot_sync(kFullMask, sd == 0u);
                    mr[i] = __ballot_sync(kFullMask, sd == 1u);
                }
#pragma unroll
                for (int i = 0; i < kPRows; ++i) {
                    const u32 sd = (sides >> (2 * i)) & 3u;
                    dsts[i] = sd == 0u ? bl + __popc(ml[i] & lt) : br + __popc(mr[i] & lt);
                    bl += __popc(ml[i]);
                    br += __popc(mr[i]);
                }
#pragma unroll
                for (int i = 0; i < kPRows; ++i) {
                    const int side = (int)((sides >> (2 * i)) & 3u);
                    const u32 dst = dsts[i];
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


// ===========================================================================
// Level pairs (round robin, k <= 4): two global levels per partition pass.
// Level l runs hist -> pick -> filter -> select as above; its children (level
// l + 1) are then selected while still in the level-l layout:
//   child hist  : every point's side against its parent's pivot (chain on
//                 ties), its child's key binned                 (8 B/pt)
//   pick        : as above, keys by pair_child_key
//   filter pair : the same sides, per (subtile, parent part, child side)
//                 counts below b* and the candidates              (8 B/pt)
//   select      : as above, count slots of the parent's layout per side
//   part pair   : ONE stable 4-way partition of every parent into its four
//                 grandchild runs (the three pivots are already written),
//                 fused with the level-(l+2) histogram of the grandchildren
// -- 16 B/pt of key reads replace one whole 8(k+1) B/pt partition pass and a
// filter pass per pair of levels.
// ===========================================================================

// level-(l+1) histogram of the children of every level-l segment (2^D bins
// per child, D = a.D); one CTA walks a contiguous run of tiles and flushes
// its shared bins when the parent changes
template <int ITEMS>
__global__ void __launch_bounds__(kHThreads, 4) sel_child_hist_kernel(SelArgs a) {
    if (aborted(a)) return;  // non-finite input: the build is reported, not run
    extern __shared__ u32 h[];  // [2][2^D]
    constexpr int T = kHThreads * ITEMS;
    const int nb = 1 << a.D;
    const LevelGeom& g0 = a.g0;
    const int k = a.k, A = k + 1;
    const u64 stride = a.bf.stride;
    const u32* W = a.bf.w[a.par];
    for (int i = threadIdx.x; i < 2 * nb; i += kHThreads) h[i] = 0u;
    const u64 t0 = (u64)blockIdx.x * a.tiles_per_cta;
    u64 t1 = t0 + a.tiles_per_cta;
    if (t1 > a.ntiles) t1 = a.ntiles;
    SegCursor sc;
    sc.init(g0, t0 * T);
    u64 cur = ~0ull;  // the parent whose children's bins are in h
    __syncthreads();
    auto flush = [&]() {
        __syncthreads();
        if (cur != ~0ull) {
            u32* gh = a.hist + 2 * cur * (u64)nb;
            for (int i = threadIdx.x; i < 2 * nb; i += kHThreads) {
                const u32 v = h[i];
                if (v) {
                    atomicAdd(&gh[i], v);
                    h[i] = 0u;
                }
            }
        }
        __syncthreads();
    };
    int dl = 0, dk0 = 0, dk1 = 0;
    u32 pinm = 0;
    float y = 0.f;
    Bucketer b0{}, b1{};
    for (u64 t = t0; t < t1; ++t) {
        const u64 ts = t * T;
        const u64 cnt = g0.nview - ts < (u64)T ? g0.nview - ts : (u64)T;
        u32 r0a, r0b, r1a, r1b;
        bool has1;
        sc.parts(g0, ts, cnt, r0a, r0b, r1a, r1b, has1);
#pragma unroll 1
        for (int p = 0; p < 2; ++p) {
            if (p == 1 && !has1) break;
            const u64 j = sc.cur + p;
            const u32 ra = p ? r1a : r0a, rb = p ? r1b : r0b;
            if (ra >= rb) continue;
            if (j != cur) {
                flush();
                cur = j;
                dl = a.chains0[j].d[0];
                y = __uint_as_float(a.piv0[j * A + dl]);
                // (the children's boxes pin what the parent's does in every
                // chain dim but its split dim)
                pinm = pinned_fields(a.chains0 + j, a.boxes_in + (2 * j) * 2ull * k, k);
                const PairKey p0 = pair_key_of(a, 2 * j);
                const PairKey p1 = pair_key_of(a, 2 * j + 1);
                dk0 = p0.d;
                dk1 = p1.d;
                b0 = make_bucketer(p0.lo, p0.hi, a.D, p0.mode);
                b1 = make_bucketer(p1.lo, p1.hi, a.D, p1.mode);
            }
            // ITEMS consecutive positions per thread: both key columns
            // loaded up front (16-byte loads) when the children share their
            // key dim, so the loads do not wait on the side compares
            const u32 r0 = (u32)threadIdx.x * ITEMS;
            const bool same = dk0 == dk1;
            u32 xk[ITEMS], kv[ITEMS];
            const u32* kl = W + (u64)dl * stride + ts + r0;
            const u32* kc = W + (u64)dk0 * stride + ts + r0;
            if (ITEMS % 4 == 0 && r0 >= ra && r0 + ITEMS <= rb) {
#pragma unroll
                for (int i = 0; i < ITEMS; i += 4) {
                    const uint4 q = *reinterpret_cast<const uint4*>(kl + i);
                    xk[i] = q.x; xk[i + 1] = q.y; xk[i + 2] = q.z; xk[i + 3] = q.w;
                }
                if (same) {
#pragma unroll
                    for (int i = 0; i < ITEMS; i += 4) {
                        const uint4 q = *reinterpret_cast<const uint4*>(kc + i);
                        kv[i] = q.x; kv[i + 1] = q.y; kv[i + 2] = q.z; kv[i + 3] = q.w;
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const u32 r = r0 + (u32)i;
                    const bool in = r >= ra && r < rb;
                    xk[i] = in ? kl[i] : 0u;
                    kv[i] = (in && same) ? kc[i] : 0u;
                }
            }
            const bool ub = same && b0.hlo == b1.hlo && b0.scale == b1.scale && b0.top == b1.top;
            if (ub && r0 >= ra && r0 + ITEMS <= rb) {
                // common case: one key column and one bucketer for both
                // children; sides by float compares, the rare ties apart
                u32 sides = 0;
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const float x = __uint_as_float(xk[i]);
                    sides |= (x < y ? 0u : (x > y ? 1u : 2u)) << (2 * i);
                }
                if (sides & 0xAAAAu) {
                    for (int i = 0; i < ITEMS; ++i)
                        if (((sides >> (2 * i)) & 3u) == 2u) {
                            const u32 sd = (u32)tie_side_pinned(W, stride, k, a.chains0 + j, a.piv0 + j * A,
                                                            ts + r0 + (u32)i, pinm);
                            sides = (sides & ~(3u << (2 * i))) | (sd << (2 * i));
                        }
                }
                auto items = [&](auto bucket_fn) {
#pragma unroll
                    for (int i = 0; i < ITEMS; ++i) {
                        const u32 sd = (sides >> (2 * i)) & 3u;
                        if (sd < 2u)
                            atomicAdd(&h[(int)sd * nb + (int)bucket_fn(b0, kv[i])], 1u);
                    }
                };
                if (key_mode(b0)) items([](const Bucketer& bb, u32 x) { return bucket_key(bb, x); });
                else items([](const Bucketer& bb, u32 x) { return bucket_val(bb, x); });
                continue;
            }
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const u32 r = r0 + (u32)i;
                if (r >= ra && r < rb) {
                    const float x = __uint_as_float(xk[i]);
                    int side = x < y ? 0 : (x > y ? 1 : 2);  // -0.0 == +0.0 like numpy
                    if (side == 2) side = tie_side_pinned(W, stride, k, a.chains0 + j, a.piv0 + j * A, ts + r, pinm);
                    if (side < 2) {
                        const u32 key = same ? kv[i] : W[(u64)(side ? dk1 : dk0) * stride + ts + r];
                        const u32 b = bucket_of(bsel2(side != 0, b0, b1), key);
                        atomicAdd(&h[side * nb + (int)b], 1u);
                    }
                }
            }
        }
    }
    flush();
}

// filter of the second level of a pair: per tile (parent parts as in the
// filter above) every point's child side, then its child's bucket against
// that child's b*: counts below b* per (subtile, part, side) and (tile,
// part, side), and the hits as candidate records (position = the parent
// layout's) staged per CTA like the filter above
template <int THREADS>
__global__ void __launch_bounds__(THREADS) sel_filter_pair_kernel(SelArgs a) {
    if (aborted(a)) return;  // non-finite input: the build is reported, not run
    constexpr int ITEMS = 8;
    constexpr int T = THREADS * ITEMS;
    constexpr int NSUB = T / kSub;
    const LevelGeom& g0 = a.g0;
    const u32* W = a.bf.w[a.par];
    const u64 stride = a.bf.stride;
    const int k = a.k, A = k + 1, R = k + 2;
    extern __shared__ u32 fsm[];  // [0] staged count, [kFCap] segment ids, [kFCap * R] records
    u32* const s_seg = fsm + 1;
    u32* const s_rec = s_seg + kFCap;
    for (int e = threadIdx.x; e < kFCap; e += THREADS) s_seg[e] = ~0u;
    if (threadIdx.x == 0) fsm[0] = 0u;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const u64 t0 = (u64)blockIdx.x * a.tiles_per_cta;
    u64 t1 = t0 + a.tiles_per_cta;
    if (t1 > a.ntiles) t1 = a.ntiles;
    if (t0 < t1) {
        SegCursor sc;
        sc.init(g0, t0 * T);
        u64 cj = ~0ull;
        int dl = 0, dk0 = 0, dk1 = 0;
        u32 pinm = 0;
        float y = 0.f;
        Bucketer bk0{}, bk1{};
        u32 bs0 = 0u, bs1 = 0u;
        bool ub = false;  // the two children's bucketers are equal
        for (u64 t = t0; t < t1; ++t) {
            const u64 ts = t * T;
            const u64 cnt = g0.nview - ts < (u64)T ? g0.nview - ts : (u64)T;
            u32 r0a, r0b, r1a, r1b;
            bool has1;
            sc.parts(g0, ts, cnt, r0a, r0b, r1a, r1b, has1);
            const u64 s = t * NSUB + warp;
            u32 n00 = 0u, n01 = 0u, n10 = 0u, n11 = 0u;  // below counts [part][side]
#pragma unroll 1
            for (int part = 0; part < 2; ++part) {
                const u64 j = sc.cur + part;
                const u32 ra = part ? r1a : r0a, rb = part ? r1b : r0b;
                if (!((part == 0 || has1) && ra < rb)) continue;
                if (j != cj) {  // the parent's pivot and its children's picks, kept while tiles stay in it
                    cj = j;
                    dl = a.chains0[j].d[0];
                    y = __uint_as_float(a.piv0[j * A + dl]);
                    pinm = pinned_fields(a.chains0 + j, a.boxes_in + (2 * j) * 2ull * k, k);
                    const u32* sl0 = a.sel + (2 * j) * kSelW;
                    const u32* sl1 = sl0 + kSelW;
                    bk0 = make_bucketer(__uint_as_float(sl0[kSelLo]), __uint_as_float(sl0[kSelShift]), a.D,
                                        (int)sl0[kSelMode]);
                    bk1 = make_bucketer(__uint_as_float(sl1[kSelLo]), __uint_as_float(sl1[kSelShift]), a.D,
                                        (int)sl1[kSelMode]);
                    bs0 = sl0[kSelB];
                    bs1 = sl1[kSelB];
                    dk0 = pair_key_of(a, 2 * j).d;
                    dk1 = pair_key_of(a, 2 * j + 1).d;
                    ub = bk0.hlo == bk1.hlo && bk0.scale == bk1.scale && bk0.top == bk1.top;
                }
                const u32 r0 = (u32)threadIdx.x * ITEMS;
                u32 key[ITEMS];
                if (r0 >= ra && r0 + ITEMS <= rb) {
                    const u32* kp = W + (u64)dl * stride + ts + r0;
                    const uint4 q0 = *reinterpret_cast<const uint4*>(kp);
                    const uint4 q1 = *reinterpret_cast<const uint4*>(kp + 4);
                    key[0] = q0.x; key[1] = q0.y; key[2] = q0.z; key[3] = q0.w;
                    key[4] = q1.x; key[5] = q1.y; key[6] = q1.z; key[7] = q1.w;
                } else {
#pragma unroll
                    for (int i = 0; i < ITEMS; ++i) {
                        const u32 r = r0 + (u32)i;
                        key[i] = (r >= ra && r < rb) ? W[(u64)dl * stride + ts + r] : 0u;
                    }
                }
                // the children's key column up front when they share it
                const bool same = dk0 == dk1;
                u32 ck[ITEMS];
                {
                    const u32* kc = W + (u64)dk0 * stride + ts + r0;
                    if (same && r0 >= ra && r0 + ITEMS <= rb) {
                        const uint4 q0 = *reinterpret_cast<const uint4*>(kc);
                        const uint4 q1 = *reinterpret_cast<const uint4*>(kc + 4);
                        ck[0] = q0.x; ck[1] = q0.y; ck[2] = q0.z; ck[3] = q0.w;
                        ck[4] = q1.x; ck[5] = q1.y; ck[6] = q1.z; ck[7] = q1.w;
                    } else {
#pragma unroll
                        for (int i = 0; i < ITEMS; ++i) {
                            const u32 r = r0 + (u32)i;
                            ck[i] = (same && r >= ra && r < rb) ? kc[i] : 0u;
                        }
                    }
                }
                u32 hits = 0, hside = 0, nlt0 = 0, nlt1 = 0;
                const bool inside = r0 >= ra && r0 + ITEMS <= rb;
                if (inside && same && ub) {
                    // common case: all 8 items in the part, both children keyed
                    // by one column and one bucketer (their box ranges in the
                    // key dim are the parent's): sides by float compares, the
                    // rare ties apart, then one bucket per item
                    u32 sides = 0;
#pragma unroll
                    for (int i = 0; i < ITEMS; ++i) {
                        const float x = __uint_as_float(key[i]);
                        sides |= (x < y ? 0u : (x > y ? 1u : 2u)) << (2 * i);
                    }
                    if (sides & 0xAAAAu) {
                        for (int i = 0; i < ITEMS; ++i)
                            if (((sides >> (2 * i)) & 3u) == 2u) {
                                const u32 sd = (u32)tie_side_pinned(W, stride, k, a.chains0 + j, a.piv0 + j * A,
                                                                ts + r0 + (u32)i, pinm);
                                sides = (sides & ~(3u << (2 * i))) | (sd << (2 * i));
                            }
                    }
                    u32 cnt = 0;  // below b*: side 0 low half, side 1 high half
                    auto items = [&](auto bucket_fn) {
#pragma unroll
                        for (int i = 0; i < ITEMS; ++i) {
                            const u32 sd = (sides >> (2 * i)) & 3u;
                            const u32 b = bucket_fn(bk0, ck[i]);
                            const u32 bsel = sd ? bs1 : bs0;
                            const bool in = sd < 2u;
                            hits |= (in && b == bsel ? 1u : 0u) << i;
                            hside |= (sd & 1u) << i;
                            cnt += (in && b < bsel) ? (sd ? 0x10000u : 1u) : 0u;
                        }
                    };
                    if (key_mode(bk0)) items([](const Bucketer& bb, u32 x) { return bucket_key(bb, x); });
                    else items([](const Bucketer& bb, u32 x) { return bucket_val(bb, x); });
                    nlt0 = cnt & 0xffffu;
                    nlt1 = cnt >> 16;
                } else {
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const u32 r = r0 + (u32)i;
                    if (r >= ra && r < rb) {
                        const float x = __uint_as_float(key[i]);
                        int side = x < y ? 0 : (x > y ? 1 : 2);
                        if (side == 2) side = tie_side_pinned(W, stride, k, a.chains0 + j, a.piv0 + j * A, ts + r, pinm);
                        if (side < 2) {
                            const u32 kv = same ? ck[i] : W[(u64)(side ? dk1 : dk0) * stride + ts + r];
                            const u32 b = bucket_of(bsel2(side != 0, bk0, bk1), kv);
                            const u32 bsel = side ? bs1 : bs0;
                            if (b == bsel) {
                                hits |= 1u << i;
                                hside |= (u32)side << i;
                            }
                            if (b < bsel) {
                                if (side) ++nlt1;
                                else ++nlt0;
                            }
                        }
                    }
                }
                }
                nlt0 = __reduce_add_sync(kFullMask, nlt0);
                nlt1 = __reduce_add_sync(kFullMask, nlt1);
                if (part) { n10 = nlt0; n11 = nlt1; }
                else { n00 = nlt0; n01 = nlt1; }
                if (lane == 0) {
                    if (nlt0) atomicAdd(&a.tile_lt[t * 2 + part], nlt0);
                    if (nlt1) atomicAdd(&a.tile_lt[a.lt_tstride + t * 2 + part], nlt1);
                }
                const u32 nh = (u32)__popc(hits);
                const u32 wtot = __reduce_add_sync(kFullMask, nh);
                if (wtot) {
                    u32 x = nh;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const u32 yv = __shfl_up_sync(kFullMask, x, o);
                        if (lane >= o) x += yv;
                    }
                    u32 pos = 0;
                    if (lane == 31) pos = atomicAdd(&fsm[0], wtot);
                    pos = __shfl_sync(kFullMask, pos, 31);
                    const bool staged = pos + wtot <= (u32)kFCap;  // (warp-uniform)
                    if (staged) {  // staged in shared memory
                        u32 q = pos + x - nh;
                        while (hits) {
                            const int i = __ffs(hits) - 1;
                            hits &= hits - 1;
                            const u32 r = r0 + (u32)i;
                            u32* rec = s_rec + q * R;
                            s_seg[q] = (u32)(2 * j) + ((hside >> i) & 1u);
                            ++q;
                            for (int cc = 0; cc < A; ++cc) rec[cc] = W[(u64)cc * stride + ts + r];
                            rec[k + 1] = (u32)(ts + r);
                        }
                    } else {
                        // staging full (tie-heavy data): slots of the children's
                        // ranges directly, one reservation per child side per warp
                        const u32 hL = hits & ~hside, hR = hits & hside;
                        const u32 nL = (u32)__popc(hL), nR = (u32)__popc(hR);
                        u32 xl = nL, xr = nR;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const u32 yl = __shfl_up_sync(kFullMask, xl, o);
                            const u32 yr = __shfl_up_sync(kFullMask, xr, o);
                            if (lane >= o) { xl += yl; xr += yr; }
                        }
                        u32* const selL = a.sel + (2 * j) * kSelW;
                        u32* const selR = selL + kSelW;
                        u32 bL = 0, bR = 0;
                        if (lane == 31) {
                            if (xl) bL = selL[kSelOff] + atomicAdd(&selL[kSelFill], xl);
                            if (xr) bR = selR[kSelOff] + atomicAdd(&selR[kSelFill], xr);
                        }
                        bL = __shfl_sync(kFullMask, bL, 31) + xl - nL;
                        bR = __shfl_sync(kFullMask, bR, 31) + xr - nR;
                        while (hits) {
                            const int i = __ffs(hits) - 1;
                            hits &= hits - 1;
                            const u32 r = r0 + (u32)i;
                            const u32 slot = ((hside >> i) & 1u) ? bR++ : bL++;
                            u32* rec = a.cand + (u64)slot * R;
                            for (int cc = 0; cc < A; ++cc) rec[cc] = W[(u64)cc * stride + ts + r];
                            rec[k + 1] = (u32)(ts + r);
                        }
                    }
                }
            }
            if (lane == 0) {
                a.sub_lt[s * 2] = n00;
                a.sub_lt[s * 2 + 1] = n10;
                a.sub_lt[a.lt_sstride + s * 2] = n01;
                a.sub_lt[a.lt_sstride + s * 2 + 1] = n11;
            }
        }
    }
    // the staged candidates -> their children's ranges (as in the filter above)
    __syncthreads();
    const u32 ltm = lanemask_lt();
    const u32 nst = min(fsm[0], (u32)kFCap);
    for (u32 e0 = (u32)warp * 32u; e0 < nst; e0 += (u32)THREADS) {
        const u32 e = e0 + (u32)lane;
        const u32 js = e < nst ? s_seg[e] : ~0u;
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

// the pair partition: every parent segment -> its four grandchild runs
//   LL [ib, ib + poL)          LR [ib + poL + 1, ib + po)
//   RL [ib + po + 1, + poR)    RR [ib + po + 1 + poR + 1, ib + size)
// (po, poL, poR: the parent's and the children's pivot offsets; their slots
// stay holes).  A point's destination is its run's begin plus the number of
// its run's points before it: per subtile from the two levels' below-pivot
// prefixes (L before = level-l count; LL / RL before = level-(l+1) counts;
// LR / RR by difference), inside the subtile by warp ballots.  Same TMA ring
// and warp-owned subtile runs as sel_part_bulk_kernel; the fused histogram
// bins the four grandchildren (2^FD bins each, 16-bit warp bins).
struct PHdr2 {
    u32 sl[3], tl[3];  // a part's lane sub count words (level l, L side, R side) and tile prefixes
};
// a parent's geometry and its three pivots (positions, leading coordinates)
struct PPar {
    u64 j;
    u32 ib, ie, po, poL, poR, pp0, ppL, ppR;
    int dl, dlL, dlR;  // the split dims of the parent and its children
    float y, yL, yR;
};

template <int KMAX, int NST, int FD>
__global__ void __launch_bounds__(kPThreads, 2) sel_part_pair_kernel(SelArgs a, int T) {
    if (aborted(a)) return;  // non-finite input: the build is reported, not run
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int kGB = 1 << FD;  // bins per grandchild
    constexpr int kWW = 2 * kGB;  // words of a warp's bins (4 grandchildren, two 16-bit bins per word)
    const int lane = threadIdx.x & 31;
    const int k = a.k, A = k + 1;
    const LevelGeom& g0 = a.g0;  // parents: the layout
    const LevelGeom& g1 = a.g;   // children
    const bool wide = a.mode == kWidest;
    const u32* Wsrc = a.bf.w[a.par];
    u32* Wdst = a.bf.w[a.par ^ 1u];
    const u64 stride = a.bf.stride;
    const u64 nsub = (g0.nview + kSub - 1) / kSub;
    const int nsub_tile = T / kSub;
    const u32 lt = lanemask_lt();
    const int warp = threadIdx.x >> 5;
    u64* bars = reinterpret_cast<u64*>(smem_raw) + warp * NST;
    u32* ring = reinterpret_cast<u32*>(smem_raw + kPHistOff + sizeof(u32) * (kPThreads / 32) * kWW) +
                (size_t)warp * NST * (KMAX + 1) * kSub;
    if (lane == 0) {
        for (int st = 0; st < NST; ++st) mbar_init(&bars[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](u64 s2, int st) {  // lane 0
        const u64 ss2 = s2 * kSub;
        const u64 cnt2 = g0.nview - ss2 < (u64)kSub ? g0.nview - ss2 : (u64)kSub;
        const u32 bytes = (u32)(((cnt2 + 3) & ~3ull) * 4);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bars[st], bytes * (u32)A);
        for (int c = 0; c < A; ++c)
            bulk_g2s(ring + ((size_t)st * (KMAX + 1) + c) * kSub, Wsrc + (u64)c * stride + ss2, bytes, &bars[st]);
    };
    const u64 nw = (u64)gridDim.x * (kPThreads / 32);
    const u64 chunk = (nsub + nw - 1) / nw;
    u64 s = ((u64)blockIdx.x * (kPThreads / 32) + warp) * chunk;
    const u64 s_end = s + chunk < nsub ? s + chunk : nsub;
    if (lane == 0) {
        for (int q = 0; q < NST - 1; ++q)
            if (s + q < s_end) issue(s + q, q);
    }
    // fused level-(l+2) histogram: the four grandchildren of one parent
    u32* wh = reinterpret_cast<u32*>(smem_raw + kPHistOff) + warp * kWW;
    const bool fuse = a.hist_next != nullptr;
    u64 hseg = ~0ull;
    Bucketer hb0{}, hb1{}, hb2{}, hb3{};
    int hd0 = 0, hd1 = 0, hd2 = 0, hd3 = 0;
    bool hsides = false, hall = false;
    int hmode = 4;  // 0: both sides value-linear, 3: both key-linear, else mixed / per grandchild
    const int dn2 = (g1.l + 1) % k;
    // a grandchild's key dim for the fused histogram: round robin
    // rr_key_dim (-1: pinned, the level's dim); widest its split dim
    auto gdim = [&](u64 c, const float* cb) -> int {
        if (!wide) return rr_key_dim(cb, k, g1.l + 1);
        const u64 node = ((2ull << g1.l) - 1ull) + (g1.sbase << 1) + c;
        return node < g1.n ? (int)a.split_dims[node] : 0;
    };
    int hcnt = 0;
    auto hflush = [&]() {
        if (hseg != ~0ull) {
            for (int i = lane; i < kWW; i += 32) {
                const u32 v = wh[i];
                if (v) {
                    u32* gh = a.hist_next + (4 * hseg + i / (kGB / 2)) * (u64)kGB + 2 * (i % (kGB / 2));
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
        for (int i = lane; i < kWW; i += 32) wh[i] = 0u;
        __syncwarp();
    }
    const int tsh = 31 - __clz(T);
    // split dims: round robin by level; widest per node (written by the selects)
    auto sdim = [&](const LevelGeom& gg, u64 t, int rr_dim) -> int {
        return wide ? (int)a.split_dims[gg.Fl + gg.sbase + t] : rr_dim;
    };
    auto load_par = [&](u64 j) {
        PPar p;
        p.j = j;
        const u64 ib = v_ibegin(g0, j);
        p.ib = (u32)ib;
        p.ie = (u32)(ib + v_size(g0, j));
        p.po = (u32)v_pivot(g0, j);
        p.poL = (u32)v_pivot(g1, 2 * j);
        p.poR = (u32)v_pivot(g1, 2 * j + 1);
        p.pp0 = a.ppos0[j];
        p.ppL = a.ppos[2 * j];
        p.ppR = a.ppos[2 * j + 1];
        p.dl = sdim(g0, j, g0.l % k);
        p.dlL = sdim(g1, 2 * j, g1.l % k);
        p.dlR = sdim(g1, 2 * j + 1, g1.l % k);
        p.y = __uint_as_float(a.piv0[j * A + p.dl]);
        p.yL = __uint_as_float(a.piv[(2 * j) * A + p.dlL]);
        p.yR = __uint_as_float(a.piv[(2 * j + 1) * A + p.dlR]);
        return p;
    };
    // the parent of the last lean subtile: subtiles inside it skip the
    // 64-bit geometry (tile_parts, v_seg_of, v_pivot) and the pivot loads
    PPar cp;
    cp.j = ~0ull;
    cp.ib = cp.ie = 0u;
    // part p's count words of subtile s2 whose part p is segment j (j == ~0:
    // the subtile's first segment)
    auto hdr_load = [&](u64 s2, u64 j, PHdr2& h2) {
        const u64 ss2 = s2 * kSub;
        const u64 t2 = ss2 >> tsh;
        const u64 tstart = t2 << tsh;
        u32 pt;
        if (j == ~0ull && ss2 >= cp.ib && ss2 < cp.ie) {
            pt = tstart >= cp.ib ? 0u : 1u;  // (the tile starts inside the cached parent, or before it)
        } else {
            if (j == ~0ull) j = v_seg_of(g0, ss2);
            pt = j == v_seg_of(g0, tstart) ? 0u : 1u;
        }
        const int sin = (int)(s2 - t2 * (u64)nsub_tile);
        const u64 w = (t2 * (u64)nsub_tile + lane) * 2 + pt;
        h2.sl[0] = lane < sin ? a.sub_lt0[w] : 0u;
        h2.sl[1] = lane < sin ? a.sub_lt[w] : 0u;
        h2.sl[2] = lane < sin ? a.sub_lt[a.lt_sstride + w] : 0u;
        h2.tl[0] = a.tile_lt0[t2 * 2 + pt];
        h2.tl[1] = a.tile_lt[t2 * 2 + pt];
        h2.tl[2] = a.tile_lt[a.lt_tstride + t2 * 2 + pt];
    };
    // the four run bases of a parent at subtile start ss
    auto bases = [&](const PHdr2& h, const PPar& p, u64 ss, u32* b) {
        const u32 nL = __reduce_add_sync(kFullMask, h.sl[0]) + h.tl[0];
        const u32 nLL = __reduce_add_sync(kFullMask, h.sl[1]) + h.tl[1];
        const u32 nRL = __reduce_add_sync(kFullMask, h.sl[2]) + h.tl[2];
        const u32 s32 = (u32)ss;
        const u32 before = s32 > p.ib ? s32 - p.ib : 0u;
        const u32 pb = (before > 0 && p.pp0 < s32) ? 1u : 0u;
        const u32 pLb = p.ppL < s32 ? 1u : 0u;
        const u32 pRb = p.ppR < s32 ? 1u : 0u;
        const u32 nR = before - nL - pb;
        b[0] = p.ib + nLL;
        b[1] = p.ib + p.poL + 1u + (nL - nLL - pLb);
        b[2] = p.ib + p.po + 1u + nRL;
        b[3] = p.ib + p.po + 1u + p.poR + 1u + (nR - nRL - pRb);
    };
    PHdr2 hn;
    if (s < s_end) hdr_load(s, ~0ull, hn);
    u32* dcol[KMAX + 1];
#pragma unroll
    for (int c = 0; c <= KMAX; ++c) dcol[c] = Wdst + (u64)(c < A ? c : 0) * stride;
    u32 phases = 0u;
    int stage = 0;
    for (; s < s_end; ++s) {
        const u64 ss = s * kSub;
        const u64 cnt = g0.nview - ss < (u64)kSub ? g0.nview - ss : (u64)kSub;
        const bool full = cnt == (u64)kSub;
        if (lane == 0 && s + (NST - 1) < s_end) issue(s + (NST - 1), (stage + NST - 1) % NST);
        mbar_wait(&bars[stage], (phases >> stage) & 1u);
        phases ^= 1u << stage;
        const u32* sv = ring + (size_t)stage * (KMAX + 1) * kSub + lane;
#define V(c, i) (sv[(c) * kSub + (i) * 32])
        bool lean = full && ss >= cp.ib && ss + kSub <= cp.ie;
        TileParts tp;
        if (!lean) {
            tp = tile_parts(g0, ss, cnt);
            if (full && !tp.has1 && tp.r0a == 0 && tp.r0b == (u32)kSub) {
                cp = load_par(tp.j0);
                lean = true;
            }
        }
        const PHdr2 h = hn;
        if (s + 1 < s_end) hdr_load(s + 1, ~0ull, hn);
        if (lean) {
            // lean path: one parent covers the whole subtile
            const u64 j0 = cp.j;
            u32 b[4];
            bases(h, cp, ss, b);
            const float y = cp.y, yL = cp.yL, yR = cp.yR;
            if (fuse && j0 != hseg) {
                hflush();
                hseg = j0;
                auto gset = [&](int q, int& hd, Bucketer& hbq) {
                    const u64 c = 4 * hseg + q;
                    const float* cb = a.boxes_out + c * 2ull * k;
                    const int e = gdim(c, cb);
                    hd = e >= 0 ? e : dn2;
                    hbq = make_bucketer(cb[hd], cb[k + hd], FD, a.bmode_out[c]);
                };
                gset(0, hd0, hb0);
                gset(1, hd1, hb1);
                gset(2, hd2, hb2);
                gset(3, hd3, hb3);
                // the two grandchildren of a child share their key range and
                // mode unless the child's own plane cut that key dim (k == 1
                // or a pinned chain): then one bucketer per child side
                auto same = [](const Bucketer& x, int dx, const Bucketer& z, int dz) {
                    return dx == dz && x.hlo == z.hlo && x.scale == z.scale && x.top == z.top;
                };
                hsides = same(hb0, hd0, hb1, hd1) && same(hb2, hd2, hb3, hd3);
                hall = hsides && same(hb0, hd0, hb2, hd2);  // k >= 3: one range for all four
                hmode = hsides ? ((key_mode(hb0) ? 1 : 0) | (key_mode(hb2) ? 2 : 0)) : 4;
            }
            if (fuse) {
                if (hcnt >= a.hflush_every) hflush();
                ++hcnt;
            }
            // sides against the parent (2 bits per row), ties separately
            u32 s1 = 0;
#pragma unroll
            for (int i = 0; i < kPRows; ++i) {
                const float x = __uint_as_float(V(cp.dl, i));
                s1 |= (x < y ? 0u : (x > y ? 1u : 2u)) << (2 * i);
            }
            if (__any_sync(kFullMask, (s1 & 0xAAAAu) != 0u)) {
#pragma unroll 1
                for (int i = 0; i < kPRows; ++i) {
                    if (((s1 >> (2 * i)) & 3u) == 2u) {
                        const u32 sd = tie_side_ring(sv, i, k, a.chains0 + j0, a.piv0 + j0 * A);
                        s1 = (s1 & ~(3u << (2 * i))) | (sd << (2 * i));
                    }
                }
            }
            // sides against the child's pivot (3: the parent's pivot row)
            u32 s2 = 0;
#pragma unroll
            for (int i = 0; i < kPRows; ++i) {
                const u32 a1 = (s1 >> (2 * i)) & 3u;
                u32 sd = 3u;
                if (a1 < 2u) {
                    const float x = __uint_as_float(V(a1 ? cp.dlR : cp.dlL, i));
                    const float yy = a1 ? yR : yL;
                    sd = x < yy ? 0u : (x > yy ? 1u : 2u);
                }
                s2 |= sd << (2 * i);
            }
            if (__any_sync(kFullMask, (s2 & 0xAAAAu & ~(s2 << 1)) != 0u)) {  // some row == 2 (not 3)
#pragma unroll 1
                for (int i = 0; i < kPRows; ++i) {
                    if (((s2 >> (2 * i)) & 3u) == 2u) {
                        const u64 c = 2 * j0 + ((s1 >> (2 * i)) & 1u);
                        const u32 sd = tie_side_ring(sv, i, k, a.chains + c, a.piv + c * A);
                        s2 = (s2 & ~(3u << (2 * i))) | (sd << (2 * i));
                    }
                }
            }
            // rows without any of the three pivots (all but <= 3 rows of a
            // parent): two ballots, counts by difference
            const bool allv = !__any_sync(kFullMask, ((s1 | s2) & 0xAAAAu) != 0u);
            auto rows = [&](auto bucket_fn, auto av_tag) {
                constexpr bool AV = decltype(av_tag)::value;
#pragma unroll
            for (int i = 0; i < kPRows; ++i) {
                const u32 a1 = (s1 >> (2 * i)) & 3u, a2 = (s2 >> (2 * i)) & 3u;
                const bool valid = AV || (a1 < 2u && a2 < 2u);
                const u32 q = 2u * a1 + a2;  // grandchild (when valid)
                const u32 mv = AV ? kFullMask : __ballot_sync(kFullMask, valid);
                const u32 m1 = __ballot_sync(kFullMask, valid && a1 == 1u);
                const u32 m2 = __ballot_sync(kFullMask, valid && a2 == 1u);
                const u32 mine = mv & (a1 ? m1 : ~m1) & (a2 ? m2 : ~m2);
                const u32 base = q == 0u ? b[0] : (q == 1u ? b[1] : (q == 2u ? b[2] : b[3]));
                const u32 dst = base + (u32)__popc(mine & lt);
                if (AV) {
                    const u32 n11 = (u32)__popc(m1 & m2), c1 = (u32)__popc(m1), c2 = (u32)__popc(m2);
                    b[0] += 32u - c1 - c2 + n11;
                    b[1] += c2 - n11;
                    b[2] += c1 - n11;
                    b[3] += n11;
                } else {
                    b[0] += (u32)__popc(mv & ~m1 & ~m2);
                    b[1] += (u32)__popc(mv & ~m1 & m2);
                    b[2] += (u32)__popc(mv & m1 & ~m2);
                    b[3] += (u32)__popc(mv & m1 & m2);
                }
                if (valid) {
                    if (fuse) {
                        u32 hbk;
                        if (hall) {
                            hbk = bucket_fn(hb0, V(hd0, i));
                        } else if (hsides) {  // one bucketer per child side
                            hbk = bucket_fn(bsel2(a1 != 0u, hb0, hb2), V(a1 ? hd2 : hd0, i));
                        } else {
                            const int hd = q == 0u ? hd0 : (q == 1u ? hd1 : (q == 2u ? hd2 : hd3));
                            const Bucketer hbq = bsel2(q >= 2u, bsel2(q == 1u, hb0, hb1), bsel2(q == 3u, hb2, hb3));
                            hbk = bucket_of(hbq, V(hd, i));
                        }
                        atomicAdd(&wh[q * (kGB / 2) + (hbk >> 1)], (hbk & 1u) ? 0x10000u : 1u);
                    }
#pragma unroll
                    for (int c = 0; c <= KMAX; ++c)
                        if (c < A) dcol[c][dst] = V(c, i);
                }
            }
            };
            auto bv = [](const Bucketer& bb, u32 x) { return bucket_val(bb, x); };
            auto bkk = [](const Bucketer& bb, u32 x) { return bucket_key(bb, x); };
            auto bo = [](const Bucketer& bb, u32 x) { return bucket_of(bb, x); };
            // rows without pivots, in phases so the rows' dependency chains
            // overlap: all ballots, then the destinations (a 4-wide running
            // sum), then the histogram and the stores
            auto rows_av = [&](auto bucket_fn) {
                u32 m1[kPRows], m2[kPRows], dsts[kPRows];
#pragma unroll
                for (int i = 0; i < kPRows; ++i) {
                    m1[i] = __ballot_sync(kFullMask, (s1 >> (2 * i)) & 1u);
                    m2[i] = __ballot_sync(kFullMask, (s2 >> (2 * i)) & 1u);
                }
#pragma unroll
                for (int i = 0; i < kPRows; ++i) {
                    const u32 a1 = (s1 >> (2 * i)) & 1u, a2 = (s2 >> (2 * i)) & 1u;
                    const u32 q = 2u * a1 + a2;
                    const u32 mine = (a1 ? m1[i] : ~m1[i]) & (a2 ? m2[i] : ~m2[i]);
                    const u32 base = q == 0u ? b[0] : (q == 1u ? b[1] : (q == 2u ? b[2] : b[3]));
                    dsts[i] = base + (u32)__popc(mine & lt);
                    const u32 n11 = (u32)__popc(m1[i] & m2[i]), c1 = (u32)__popc(m1[i]), c2 = (u32)__popc(m2[i]);
                    b[0] += 32u - c1 - c2 + n11;
                    b[1] += c2 - n11;
                    b[2] += c1 - n11;
                    b[3] += n11;
                }
#pragma unroll
                for (int i = 0; i < kPRows; ++i) {
                    const u32 a1 = (s1 >> (2 * i)) & 1u, a2 = (s2 >> (2 * i)) & 1u;
                    const u32 q = 2u * a1 + a2;
                    if (fuse) {  // (hall: one bucketer for the four grandchildren)
                        const u32 hbk = bucket_fn(hb0, V(hd0, i));
                        atomicAdd(&wh[q * (kGB / 2) + (hbk >> 1)], (hbk & 1u) ? 0x10000u : 1u);
                    }
#pragma unroll
                    for (int c = 0; c <= KMAX; ++c)
                        if (c < A) dcol[c][dsts[i]] = V(c, i);
                }
            };
            // (two compact variants of the hot loop: instruction-cache misses
            // measured expensive; everything else takes the generic rows)
            if (allv && (!fuse || (hall && hmode == 0))) {
                rows_av(bv);
            } else if (allv && hall && hmode == 3) {
                rows_av(bkk);
            } else {
                rows(bo, std::false_type{});
            }
        } else {
            // general path (a parent boundary inside the subtile, or the
            // view's last partial subtile): runs (part, grandchild), ranks by
            // match_any, the fused histogram by global atomics
            const u64 j0 = tp.j0;
            u32 b[2][4];
            const PPar P0 = load_par(j0);
            {
                PHdr2 h0;  // (the prefetched header may have used the cache)
                hdr_load(s, j0, h0);
                bases(h0, P0, ss, b[0]);
            }
            PPar P1 = P0;
            if (tp.has1) {
                PHdr2 h1;  // the second parent's header (its tile part index)
                hdr_load(s, j0 + 1, h1);
                P1 = load_par(j0 + 1);
                bases(h1, P1, ss, b[1]);
            } else {
                b[1][0] = b[1][1] = b[1][2] = b[1][3] = 0u;
            }
#pragma unroll 1
            for (int i = 0; i < kPRows; ++i) {
                const u32 r = (u32)(i * 32 + lane);
                const bool in0 = r >= tp.r0a && r < tp.r0b, in1 = r >= tp.r1a && r < tp.r1b;
                u32 run = 8u;  // 8: no run (outside the parts, or one of the three pivots)
                if (in0 || in1) {
                    const u64 j = j0 + (in1 ? 1 : 0);
                    const PPar& P = in1 ? P1 : P0;
                    const u64 pos = ss + r;
                    const float x = __uint_as_float(V(P.dl, i));
                    const float yv = P.y;
                    int a1 = x < yv ? 0 : (x > yv ? 1 : 2);
                    if (a1 == 2) a1 = tie_side_of(Wsrc, stride, k, a.chains0 + j, a.piv0 + j * A, pos);
                    if (a1 < 2) {
                        const u64 c = 2 * j + a1;
                        const float x2 = __uint_as_float(V(a1 ? P.dlR : P.dlL, i));
                        const float y2 = a1 ? P.yR : P.yL;
                        int a2 = x2 < y2 ? 0 : (x2 > y2 ? 1 : 2);
                        if (a2 == 2) a2 = tie_side_of(Wsrc, stride, k, a.chains + c, a.piv + c * A, pos);
                        if (a2 < 2) {
                            const u32 q = 2u * (u32)a1 + (u32)a2;
                            run = (in1 ? 4u : 0u) + q;
                            if (fuse) {
                                const u64 gc = 4 * j + q;
                                const float* cb = a.boxes_out + gc * 2ull * k;
                                const int e = gdim(gc, cb);
                                const int dnc = e >= 0 ? e : dn2;
                                const Bucketer hbq = make_bucketer(cb[dnc], cb[k + dnc], FD, a.bmode_out[gc]);
                                atomicAdd(&a.hist_next[gc * (u64)kGB + bucket_of(hbq, V(dnc, i))], 1u);
                            }
                        }
                    }
                }
                const u32 peers = __match_any_sync(kFullMask, run);
                u32 dst = 0;
#pragma unroll
                for (int rr = 0; rr < 8; ++rr)
                    if (run == (u32)rr) dst = b[rr >> 2][rr & 3];
                dst += (u32)__popc(peers & lt);
#pragma unroll
                for (int rr = 0; rr < 8; ++rr) b[rr >> 2][rr & 3] += (u32)__popc(__ballot_sync(kFullMask, run == (u32)rr));
                if (run < 8u) {
#pragma unroll
                    for (int c = 0; c <= KMAX; ++c)
                        if (c < A) dcol[c][dst] = V(c, i);
                }
            }
        }
#undef V
        __syncwarp();
        stage = stage + 1 == NST ? 0 : stage + 1;
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

void launch_sel_child_hist(const SelArgs& a0, int b, cudaStream_t st) {
    SelArgs a = a0;
    int items = (1 << (b - 1)) / kHThreads;
    if (items > 8) items = 8;
    const u64 T = (u64)kHThreads * items;
    a.ntiles = (a.g0.nview + T - 1) / T;
    const u64 target = 148 * 16;
    u64 tpc = (a.ntiles + target - 1) / target;
    if (tpc < 1) tpc = 1;
    a.tiles_per_cta = (int)tpc;
    const unsigned grid = (unsigned)((a.ntiles + tpc - 1) / tpc);
    const size_t sm = sizeof(u32) * 2 << a.D;
    auto go = [&](auto kern) {
        if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        kern<<<grid, kHThreads, sm, st>>>(a);
    };
    switch (items) {
        case 8: go(sel_child_hist_kernel<8>); break;
        case 4: go(sel_child_hist_kernel<4>); break;
        case 2: go(sel_child_hist_kernel<2>); break;
        default: go(sel_child_hist_kernel<1>); break;
    }
}

void launch_sel_filter_pair(const SelArgs& a0, int b, cudaStream_t st) {
    SelArgs a = a0;
    const int T = sel_tile(b);
    a.ntiles = (a.g0.nview + T - 1) / T;
    const u64 per_sm = T >= 2048 ? 32 : 64;
    const u64 target = 148 * per_sm;
    u64 tpc = (a.ntiles + target - 1) / target;
    if (tpc < 1) tpc = 1;
    a.tiles_per_cta = (int)tpc;
    const unsigned g2 = (unsigned)((a.ntiles + tpc - 1) / tpc);
    const size_t sm = sizeof(u32) * (1 + (size_t)kFCap * (1 + a.k + 2));
    auto go = [&](auto kern, int nt) {
        if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        kern<<<g2, nt, sm, st>>>(a);
    };
    switch (T) {
        case 2048: go(sel_filter_pair_kernel<256>, 256); break;
        case 1024: go(sel_filter_pair_kernel<128>, 128); break;
        case 512: go(sel_filter_pair_kernel<64>, 64); break;
        default: go(sel_filter_pair_kernel<32>, 32); break;
    }
}

void launch_sel_part_pair(const SelArgs& a0, int b, cudaStream_t st) {
    SelArgs a = a0;
    a.hflush_every = 255;
    if (const char* e = getenv("LBKD_HFLUSH_EVERY")) {
        const int v = atoi(e);
        if (v >= 1 && v < 255) a.hflush_every = v;
    }
    const int T = sel_tile(b);
    const u64 nsub = (a.g0.nview + kSub - 1) / kSub;
    const u64 per_cta = kPThreads / 32;
    auto go = [&](auto kern, int KM, int nst, int fd) {
        const size_t sm = kPHistOff + sizeof(u32) * (size_t)(kPThreads / 32) * (2u << fd) +
                          sizeof(u32) * (size_t)(kPThreads / 32) * nst * (KM + 1) * kSub;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        u64 g2 = (nsub + per_cta - 1) / per_cta;
        if (g2 > 148ull * 2) g2 = 148ull * 2;
        kern<<<(unsigned)g2, kPThreads, sm, st>>>(a, T);
    };
    // a.fuse_d: 8 (3-stage ring) or 9 (2-stage ring: the 4 KB warp bins fit)
#define LBKD_PP(KM)                                                              \
    if (a.fuse_d >= 9) go(sel_part_pair_kernel<KM, 2, 9>, KM, 2, 9);             \
    else go(sel_part_pair_kernel<KM, kPStages, 8>, KM, kPStages, 8);
    switch (a.k) {
        case 2: LBKD_PP(2); break;
        case 3: LBKD_PP(3); break;
        default: LBKD_PP(4); break;
    }
#undef LBKD_PP
}

}  // namespace lbkd
