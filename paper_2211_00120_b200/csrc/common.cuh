// common.cuh -- shared device helpers for the B200 k-d tree builder.
//
// Implicit-tree arithmetic restated from the reference
//   /root/reference/pkg/src/lbkd/treemath.py:46-140 (level, num_levels,
//   subtree_size, segment_begin, pivot_pos) and the fused pivot formula of
//   kernels_numpy._pivot_positions (kernels_numpy.py:21-38).
//
// Working-array convention: at level l
// the working array W_l holds only the N - F(l) points that are not yet
// final (F(l) = 2^l - 1), grouped by level-l node.  Segment j (node
// F(l) + j) starts at bw(j) = segment_begin(F(l)+j) - F(l); finalized nodes
// are written straight to the output, so W_l is the reference's array with
// the finalized prefix cut off.
#pragma once
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

namespace lbkd {

typedef unsigned long long u64;
typedef unsigned int u32;

constexpr u32 kFullMask = 0xffffffffu;

// Order-preserving map float32 -> uint32 with -0.0 canonicalised to +0.0.
// numpy compares the float64-promoted values, for which -0.0 == +0.0 and the
// stable sort keeps such pairs in current order.
__host__ __device__ __forceinline__ u32 float_bits(float f) {
#ifdef __CUDA_ARCH__
    return __float_as_uint(f);
#else
    u32 u;
    memcpy(&u, &f, 4);
    return u;
#endif
}

__host__ __device__ __forceinline__ float bits_float(u32 u) {
#ifdef __CUDA_ARCH__
    return __uint_as_float(u);
#else
    float f;
    memcpy(&f, &u, 4);
    return f;
#endif
}

__host__ __device__ __forceinline__ u32 flip_key(float f) {
    u32 u = float_bits(f);
    if (u == 0x80000000u) u = 0u;
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__host__ __device__ __forceinline__ float unflip_key(u32 k) {
    u32 u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    return bits_float(u);
}

// ---- rank-coded coordinates (float64 inputs) ---------------------------------
// A float64 build (lbkd_build_*_f64, rank64.cu) replaces every coordinate by
// its dense rank among the distinct values of its dimension (-0.0 == +0.0,
// exactly numpy's ordering of the values) and codes the rank as a float32,
// strictly increasing in the rank.  Every comparison of the build then gives
// the float64 answer; the only arithmetic on coordinate VALUES -- the widest
// variant's float64 widths (widest.py:91-93) -- looks the values up again in
// a per-dimension table of the distinct values (WidthTab).
//
// Code: v = rank - center[d]; |v| < 2^24 -> (float)v exactly; beyond that
// the float32 bit pattern keeps counting (0x4B800000 = 2^24 plus |v| - 2^24
// ulps), so values stay nearly linear in the rank (the selection's value-
// linear buckets stay balanced) and each side holds 889M ranks.  The wide
// code (a dimension with more distinct values than that, only possible above
// 1.7G points) counts through the whole order-flipped float range instead.
constexpr u32 kRankLin = 1u << 24;
constexpr u32 kRankSide = 0x7F7FFFFFu - 0x4B800000u + (1u << 24);  // ranks per side in the linear code

struct WidthTab {
    const double* v;      // [k][stride] distinct values of each dim in rank order; null: plain float32 input
    u64 stride;
    u32 wide;             // bit d: dimension d uses the wide code
    u32 center[16];
};

__host__ __device__ __forceinline__ float rank_code(u32 r, u32 center, int wide) {
    if (wide) {
        u32 key = 0x00800000u + r;
        if (key >= 0x7FFFFFFFu) key += 1u;  // skip the -0.0 key
        return unflip_key(key);
    }
    const bool neg = r < center;
    const u32 m = neg ? center - r : r - center;
    const u32 bits = m < kRankLin ? float_bits((float)m) : 0x4B800000u + (m - kRankLin);
    return bits_float(bits | (neg ? 0x80000000u : 0u));
}

__host__ __device__ __forceinline__ u32 rank_decode(float f, u32 center, int wide) {
    if (wide) {
        const u32 key = flip_key(f);
        return key - 0x00800000u - (key > 0x7FFFFFFFu ? 1u : 0u);
    }
    const u32 b = float_bits(f);
    const u32 mb = b & 0x7FFFFFFFu;
    const u32 m = mb < 0x4B800000u ? (u32)bits_float(mb) : mb - 0x4B800000u + kRankLin;
    return (b >> 31) ? center - m : center + m;
}

// float64 width hi - lo of dimension d (the widest variant's argmax key)
__host__ __device__ __forceinline__ double coord_width(const WidthTab& t, int d, float lo, float hi) {
    if (!t.v) return (double)hi - (double)lo;
    const double* v = t.v + (u64)d * t.stride;
    const int wide = (int)((t.wide >> d) & 1u);
    return v[rank_decode(hi, t.center[d], wide)] - v[rank_decode(lo, t.center[d], wide)];
}

// Geometry of one level of the implicit left-balanced tree.
struct LevelGeom {
    int l;        // level being split
    int L;        // num_levels(N) = bit_length(N)
    int sh;       // L - l - 1 (log2 of bottom-level slots per level-l subtree)
    u64 n;        // N
    u64 B;        // bottom_have = N - F(L-1)
    u64 Fl;       // F(l) = 2^l - 1 (finalized nodes before level l)
    u64 nl;       // N - F(l): elements in W_l
    u64 nseg;     // segments in the view (2^l for the whole tree)
    // view of a subtree (multi-GPU shard / sub-build); the whole tree is the
    // view rooted at level 0.  Local segment t is global segment sbase + t,
    // local in-order position p is global position pbase + p.
    u64 sbase;
    u64 pbase;
    u64 nview;    // points in the view
    int lfirst;   // root level of the view (buffers start at parity 0 there)
};

__host__ __device__ inline int bit_length(u64 v) {
    int b = 0;
    while (v) { ++b; v >>= 1; }
    return b;
}

__host__ __device__ inline LevelGeom make_geom(u64 n, int l) {
    LevelGeom g;
    g.n = n;
    g.L = bit_length(n);
    g.l = l;
    g.sh = g.L - l - 1;
    g.B = n - ((1ull << (g.L - 1)) - 1ull);
    g.Fl = (1ull << l) - 1ull;
    g.nl = n - g.Fl;
    g.nseg = 1ull << l;
    g.sbase = 0;
    g.pbase = 0;
    g.nview = n;
    g.lfirst = 0;
    return g;
}

// size of segment j (treemath.subtree_size, treemath.py:85-98)
__host__ __device__ __forceinline__ u64 seg_size(const LevelGeom& g, u64 j) {
    u64 w = 1ull << g.sh;
    u64 lo = j << g.sh;
    u64 on = g.B > lo ? g.B - lo : 0ull;
    if (on > w) on = w;
    return w - 1ull + on;
}

// begin of segment j inside W_l (treemath.segment_begin, treemath.py:108-126,
// minus the F(l) finalized prefix)
__host__ __device__ __forceinline__ u64 seg_begin(const LevelGeom& g, u64 j) {
    u64 lo = j << g.sh;
    return j * ((1ull << g.sh) - 1ull) + (lo < g.B ? lo : g.B);
}

// offset of the pivot inside segment j = size of the left child's subtree
// (treemath.pivot_pos, treemath.py:129-140; kernels_numpy.py:33-38)
__host__ __device__ __forceinline__ u64 pivot_off(const LevelGeom& g, u64 j) {
    if (g.sh <= 0) return 0ull;
    u64 cw = 1ull << (g.sh - 1);
    u64 lo = (2ull * j) * cw;
    u64 on = g.B > lo ? g.B - lo : 0ull;
    if (on > cw) on = cw;
    return cw - 1ull + on;
}

// In-order layout (global levels): segment j of level l begins at
// ib(j) = bw(j) + j -- the compacted begin plus one finished ancestor node
// between consecutive segments -- which simplifies to
// min(j * 2^(sh+1), j * 2^sh + B).
__host__ __device__ __forceinline__ u64 seg_ibegin(const LevelGeom& g, u64 j) {
    u64 lo = j << g.sh;
    return lo + (lo < g.B ? lo : g.B);
}

// segment whose in-order range starts at or before position p (p may be the
// finished node just after it); inverse of the piecewise-linear ib(j)
__host__ __device__ __forceinline__ u64 seg_of_inorder(const LevelGeom& g, u64 p) {
    u64 ja = p >> (g.sh + 1);
    u64 jb = p >= g.B ? (p - g.B) >> g.sh : 0ull;
    u64 j = ja > jb ? ja : jb;
    const u64 all = 1ull << g.l;
    return j < all ? j : all - 1;
}

// View of the subtree rooted at node (level lroot, index jroot) at level l.
__host__ __device__ inline LevelGeom make_view(u64 n, int l, int lroot, u64 jroot) {
    LevelGeom g = make_geom(n, l);
    LevelGeom gr = make_geom(n, lroot);
    g.nseg = 1ull << (l - lroot);
    g.sbase = jroot << (l - lroot);
    g.pbase = seg_ibegin(gr, jroot);
    g.nview = seg_size(gr, jroot);
    g.lfirst = lroot;
    return g;
}

// local (view) forms of the in-order helpers
__host__ __device__ __forceinline__ u64 v_ibegin(const LevelGeom& g, u64 t) {
    return seg_ibegin(g, g.sbase + t) - g.pbase;
}
__host__ __device__ __forceinline__ u64 v_size(const LevelGeom& g, u64 t) { return seg_size(g, g.sbase + t); }
__host__ __device__ __forceinline__ u64 v_pivot(const LevelGeom& g, u64 t) { return pivot_off(g, g.sbase + t); }
__host__ __device__ __forceinline__ u64 v_seg_of(const LevelGeom& g, u64 p) {
    u64 j = seg_of_inorder(g, g.pbase + p);
    j = j > g.sbase ? j - g.sbase : 0ull;
    return j < g.nseg ? j : g.nseg - 1;
}

// segment containing W_l position p (inverse of seg_begin); O(1) with two
// integer divisions -- evaluated once per tile, not per element.
__host__ __device__ inline u64 seg_of(const LevelGeom& g, u64 p) {
    u64 full = (2ull << g.sh) - 1ull;
    u64 nf = g.B >> g.sh;
    if (nf > (1ull << g.l)) nf = 1ull << g.l;
    u64 p1 = nf * full;
    if (p < p1) return p / full;
    u64 rem = g.B - (nf << g.sh);
    u64 small = (1ull << g.sh) - 1ull;
    u64 ps = small + rem;
    u64 q = p - p1;
    if (q < ps || small == 0) return nf;
    return nf + 1ull + (q - ps) / small;
}

// Lanes of the warp holding the same NBITS-bit value (the set of "peers"),
// built from one ballot per bit.  MATCH.ANY runs on the B200's low-rate ADU
// pipe (measured: the pipe saturates at ~40 cycles per instruction, see
// DESIGN.md), while VOTE/LOP3 issue at full rate, so the bit-sliced form is
// several times faster for 8-9 bit digits.  Invalid lanes match only
// themselves.
template <int NBITS>
__device__ __forceinline__ u32 warp_peers(u32 v, bool valid) {
    u32 m = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < NBITS; ++b) {
        const bool bit = (v >> b) & 1u;
        const u32 bal = __ballot_sync(0xffffffffu, bit);
        m &= bit ? bal : ~bal;
    }
    return valid ? m : (1u << (threadIdx.x & 31u));
}

// warp_peers for a warp whose 32 lanes are all valid (no validity ballot)
template <int NBITS>
__device__ __forceinline__ u32 warp_peers_full(u32 v) {
    u32 m = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < NBITS; ++b) {
        const u32 bal = __ballot_sync(0xffffffffu, (v >> b) & 1u);
        m &= ((v >> b) & 1u) ? bal : ~bal;
    }
    return m;
}

// ---- PTX helpers -----------------------------------------------------------
__device__ __forceinline__ u32 lanemask_lt() {
    u32 r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

__device__ __forceinline__ u64 ld_relaxed_u64(const u64* p) {
    u64 v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_u64(u64* p, u64 v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// L2-only (32-byte sector) loads for random gathers: the default LDG path
// promotes a miss to a full 128-byte line, quadrupling DRAM traffic for
// scattered 4-byte reads.
__device__ __forceinline__ float ld_cg_f32(const float* p) {
    float v;
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ u32 ld_cg_u32(const u32* p) {
    u32 v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// ---- bulk async copies (TMA engine, 1-D) completing on an mbarrier --------
__device__ __forceinline__ u32 smem_addr(const void* p) { return (u32)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
// global -> shared, `bytes` a multiple of 16, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}

// Decoupled-lookback status word: [63:34] epoch, [33:32] flag, [31:0] count
constexpr u64 kFlagAgg = 1ull;
constexpr u64 kFlagInc = 2ull;
__device__ __forceinline__ u64 pack_status(u32 epoch, u64 flag, u32 count) {
    return ((u64)epoch << 34) | (flag << 32) | (u64)count;
}

// Exclusive block scan over blockDim.x values (blockDim.x multiple of 32,
// at most 1024).  `warp_tot` must hold 32 entries.
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* warp_tot, T* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(kFullMask, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        T t = lane < nw ? warp_tot[lane] : T(0);
        T s = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(kFullMask, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) warp_tot[lane] = s - t;
        if (lane == 31 && total) *total = s;
    }
    __syncthreads();
    T r = x - v + warp_tot[warp];
    __syncthreads();
    return r;
}

// Exclusive block scan with ONE barrier: warp scans, lane 31 publishes its
// warp's total into buf[warp], one barrier, then every thread adds the totals
// of the warps before its own (broadcast loads).  buf (32 entries) must not
// be written again before the caller's next barrier.
template <typename T>
__device__ __forceinline__ T block_exclusive_scan_1b(T v, T* buf) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(kFullMask, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) buf[warp] = x;
    __syncthreads();
    T pre = T(0);
    for (int w = 0; w < warp; ++w) pre += buf[w];
    return pre + x - v;
}

}  // namespace lbkd
