// global_sort.cu -- the per-level sort phase of the top (large-segment)
// levels: a segmented, stable, onesweep LSD radix sort of every level-l
// segment by its split coordinate, with the points travelling as payload.
//
// Reference semantics (bit-exact):
//   sort_phase   /root/reference/pkg/src/lbkd/builder.py:165-181
//       np.lexsort((coords[:, l % k], tags)): stable by (tag, coordinate)
//   update_tags_round_robin  kernels_numba.py:21-46 (pivot arithmetic)
//   sort_phase_widest        widest.py:119-131 (minor key = own coordinate in
//                            the tag's split dimension)
//
// Why segmented: after update pass l-1 the tags along the array are already
// ascending (children 2s+1 < 2s+2 < 2(s+1)+1) and each level-l node owns one
// contiguous segment, so the (tag, coord) sort never moves a point across
// segments: the tag digits of the packed 64-bit key are provably in order
// and their digit passes are skipped.  What remains is a stable sort of each
// segment by its 32-bit order-flipped coordinate.
//
// Why in-order layout: the reference moves each finished node to the front
// (its final tag order).  Here every node stays at its in-order slot; the
// left child's segment is then exactly the part before the pivot and the
// right child's the part after it, so updateTags moves nothing -- the pivot
// is read off in place (pivot kernel) and the children inherit the parent's
// buffer.  A digit pass runs only for segments whose digit actually varies
// (per-segment AND/OR), and skipped segments are not touched at all.
//
// Why payload: a random 4-byte gather on B200 costs a 128-byte line and is
// limited to ~50 G gathers/s (measured, tools/micro/gather.cu), so the points
// move with their keys as SoA arrays and no kernel ever gathers.
#include "kernels.cuh"

namespace lbkd {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kBuckets = 512;  // 2 segments x 256 digits per tile

static int items_for_bits(int b) { return (1 << (b - 1)) / kThreads; }

__device__ __forceinline__ u32 parity_out(uint8_t st) {
    return ((st >> 4) ^ (u32)__popc(st & 15u)) & 1u;
}

// split dimension of level-l segment j
__device__ __forceinline__ int seg_dim(int mode, const uint8_t* split_dims, const LevelGeom& g, int k, u64 j) {
    return mode == kRoundRobin ? (g.l % k) : (int)split_dims[g.Fl + g.sbase + j];
}

// parity (buffer) holding level-l (local) segment j at the start of the
// level: its parent's final buffer (sbase is even below the view's root)
__device__ __forceinline__ u32 seg_parity_in(const uint8_t* prev_state, const LevelGeom& g, u64 j) {
    return g.l == g.lfirst ? 0u : parity_out(prev_state[j >> 1]);
}

// ---------------------------------------------------------------------------
// init: AoS float32 input -> W[0] SoA (k coordinate arrays + index array),
// and the non-finite check of builder.py:134-135.
// ---------------------------------------------------------------------------
__global__ void init_kernel(const float* __restrict__ pts, u64 n, int k, u32* w0, u64 stride, u32* err) {
    bool bad = false;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const float* q = pts + i * k;
        for (int c = 0; c < k; ++c) {
            float f = __ldg(q + c);
            bad |= !isfinite(f);
            w0[c * stride + i] = __float_as_uint(f);
        }
        w0[(u64)k * stride + i] = (u32)i;
    }
    if (__any_sync(kFullMask, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

void launch_init(const BuildParams& bp, const Buffers& bf, cudaStream_t st) {
    u64 blocks = (bp.n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    init_kernel<<<(unsigned)blocks, 256, 0, st>>>(bp.pts, bp.n, bp.k, bf.w[0], bf.stride, bf.err);
}

// ---------------------------------------------------------------------------
// hist: per-(segment, digit pass, digit) counts of the level's keys and the
// per-segment AND/OR that drive digit-pass skipping.  Each CTA walks a
// contiguous run of tiles and flushes its shared histogram only when the
// segment changes, so global atomics stay O(#CTAs + #segments).
// ---------------------------------------------------------------------------
struct HistArgs {
    LevelGeom g;
    int k, mode, tiles_per_cta;
    u64 ntiles;
    Buffers bf;
    const uint8_t* prev_state;
    const uint8_t* split_dims;
};

constexpr int kHistThreads = 256;

// warp-private bins, bumped by each match group's highest lane with a plain
// read-modify-write (the groups of one instruction hit distinct bins, and
// consecutive rounds are ordered by __syncwarp) -- shared atomics cost
// ~2 cycles per lane on B200, this costs one bank-conflicted LDS/STS pair
// All four digit histograms of one warp row: 32 bit ballots give the peer
// masks of every digit; `full` (warp-uniform) skips the validity ballot.
__device__ __forceinline__ void hist_round(u32* h, u32 key, bool inc, bool full) {
    const u32 lane = threadIdx.x & 31u;
    const u32 v = full ? 0xffffffffu : __ballot_sync(kFullMask, inc);
    u32 m[4] = {v, v, v, v};
#pragma unroll
    for (int b = 0; b < 8; ++b) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const u32 bit = (key >> (8 * q + b)) & 1u;
            const u32 bal = __ballot_sync(kFullMask, bit);
            m[q] &= bit ? bal : ~bal;
        }
    }
    if (inc) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (lane == 31u - __clz(m[q])) h[q * 256 + ((key >> (8 * q)) & 255u)] += (u32)__popc(m[q]);
    }
    __syncwarp();
}

template <int ITEMS>
__global__ void __launch_bounds__(kHistThreads) hist_kernel(HistArgs a) {
    constexpr int kW = kHistThreads / 32;
    __shared__ u32 h[kW][4 * 256];
    __shared__ u32 s_and[kW], s_or[kW];
    constexpr int T = kHistThreads * ITEMS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const LevelGeom& g = a.g;
    for (int i = threadIdx.x; i < kW * 4 * 256; i += kHistThreads) (&h[0][0])[i] = 0;
    u64 t0 = (u64)blockIdx.x * a.tiles_per_cta;
    u64 t1 = t0 + a.tiles_per_cta;
    if (t1 > a.ntiles) t1 = a.ntiles;
    u64 cur = v_seg_of(g, t0 * T);
    u32 acc_and = 0xffffffffu, acc_or = 0u;
    u32* hw = h[warp];
    __syncthreads();

    auto flush = [&](u64 seg) {
        u32 wa = __reduce_and_sync(kFullMask, acc_and);
        u32 wo = __reduce_or_sync(kFullMask, acc_or);
        if (lane == 0) { s_and[warp] = wa; s_or[warp] = wo; }
        __syncthreads();
        u32* gh = a.bf.hist + seg * 1024ull;
        for (int i = threadIdx.x; i < 1024; i += kHistThreads) {
            u32 v = 0;
#pragma unroll
            for (int w = 0; w < kW; ++w) { v += h[w][i]; h[w][i] = 0; }
            if (v) atomicAdd(&gh[i], v);
        }
        if (threadIdx.x == 0) {
            u32 A = 0xffffffffu, O = 0u;
            for (int w = 0; w < kW; ++w) { A &= s_and[w]; O |= s_or[w]; }
            atomicAnd(&a.bf.seg_and[seg], A);
            atomicOr(&a.bf.seg_or[seg], O);
        }
        acc_and = 0xffffffffu;
        acc_or = 0u;
        __syncthreads();
    };

    for (u64 t = t0; t < t1; ++t) {
        const u64 ts = t * T;
        const u64 cnt = g.nview - ts < (u64)T ? g.nview - ts : (u64)T;
        // segment `cur` occupies [sb, e0); a finished node sits at e0 and
        // segment cur+1 starts at e0 + 1
        const u64 sb = v_ibegin(g, cur);
        const u64 e0 = sb + v_size(g, cur);
        const bool has_next = cur + 1 < g.nseg && e0 + 1 < ts + cnt;
        const u32 r0a = sb > ts ? (u32)(sb - ts) : 0u;
        const u32 r0b = e0 > ts ? (u32)((e0 - ts < cnt) ? e0 - ts : cnt) : 0u;
        const u32 r1a = has_next ? (u32)(e0 + 1 - ts) : (u32)cnt;
        const u32* k0 = warr(a.bf, seg_parity_in(a.prev_state, g, cur), seg_dim(a.mode, a.split_dims, g, a.k, cur));
        const u32* k1 = has_next ? warr(a.bf, seg_parity_in(a.prev_state, g, cur + 1),
                                        seg_dim(a.mode, a.split_dims, g, a.k, cur + 1))
                                 : k0;
        u32 key[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            u32 r = (u32)(warp * ITEMS * 32 + i * 32 + lane);
            key[i] = 0;
            if (r >= r0a && r < r0b) key[i] = flip_key(__uint_as_float(k0[ts + r]));
            else if (r >= r1a && r < cnt) key[i] = flip_key(__uint_as_float(k1[ts + r]));
        }
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const u32 row = (u32)(warp * ITEMS * 32 + i * 32);
            u32 r = row + lane;
            bool inc = r >= r0a && r < r0b;
            if (inc) { acc_and &= key[i]; acc_or |= key[i]; }
            const bool full = row >= r0a && row + 32 <= r0b;
            if (__any_sync(kFullMask, inc)) hist_round(hw, key[i], inc, full);
        }
        if (has_next) {
            __syncthreads();
            flush(cur);
            ++cur;
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const u32 row = (u32)(warp * ITEMS * 32 + i * 32);
                u32 r = row + lane;
                bool inc = r >= r1a && r < cnt;
                if (inc) { acc_and &= key[i]; acc_or |= key[i]; }
                const bool full = row >= r1a && row + 32 <= cnt;
                if (__any_sync(kFullMask, inc)) hist_round(hw, key[i], inc, full);
            }
        }
    }
    __syncthreads();
    flush(cur);
}

void launch_hist(const BuildParams& bp, const Buffers& bf, int l, cudaStream_t st) {
    HistArgs a;
    a.g = view_of(bp, l);
    a.k = bp.k;
    a.mode = bp.mode;
    int items = (1 << (bp.b - 1)) / kHistThreads;  // tile <= smallest segment
    if (items > 8) items = 8;
    const u64 T = (u64)kHistThreads * items;
    a.ntiles = (a.g.nview + T - 1) / T;
    u64 target = 148 * 8;
    u64 tpc = (a.ntiles + target - 1) / target;
    if (tpc < 1) tpc = 1;
    a.tiles_per_cta = (int)tpc;
    a.bf = bf;
    a.prev_state = bf.state[(l + 1) & 1];
    a.split_dims = bp.split_dims;
    unsigned grid = (unsigned)((a.ntiles + tpc - 1) / tpc);
    switch (items) {
        case 8: hist_kernel<8><<<grid, kHistThreads, 0, st>>>(a); break;
        case 4: hist_kernel<4><<<grid, kHistThreads, 0, st>>>(a); break;
        default: hist_kernel<2><<<grid, kHistThreads, 0, st>>>(a); break;
    }
}

// ---------------------------------------------------------------------------
// plan: per segment, which digit passes reorder it (digit not constant) and
// which buffer it starts in (its parent's final buffer).
// ---------------------------------------------------------------------------
__global__ void plan_kernel(LevelGeom g, const u32* seg_and, const u32* seg_or, const uint8_t* prev_state,
                            uint8_t* state) {
    u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x;
    if (j >= g.nseg) return;
    u32 vary = seg_and[j] ^ seg_or[j];
    u32 mask = 0;
    for (int p = 0; p < 4; ++p)
        if ((vary >> (8 * p)) & 255u) mask |= 1u << p;
    u32 par = seg_parity_in(prev_state, g, j);
    state[j] = (uint8_t)((par << 4) | mask);
}

void launch_plan(const BuildParams& bp, const Buffers& bf, int l, cudaStream_t st) {
    LevelGeom g = view_of(bp, l);
    unsigned blocks = (unsigned)((g.nseg + 255) / 256);
    plan_kernel<<<blocks, 256, 0, st>>>(g, bf.seg_and, bf.seg_or, bf.state[(l + 1) & 1], bf.state[l & 1]);
}

// ---------------------------------------------------------------------------
// onesweep digit pass
// ---------------------------------------------------------------------------
struct PassArgs {
    LevelGeom g;
    int pass, k, mode;
    u32 epoch;
    Buffers bf;
    const uint8_t* state;
    const uint8_t* split_dims;
    u32* tile_ctr;
    u64* moved;
};

template <int ITEMS>
struct PassSmem {
    static constexpr int T = kThreads * ITEMS;
    unsigned short cnt[kWarps][kBuckets];  // per-warp counts, then warp prefixes
    u32 bstart[kBuckets];                  // tile-local start of each bucket
    u32 gdelta[kBuckets];                  // offset-in-segment = gdelta[b] + slot
    u32 dstoff[T];                         // destination of sorted slot i
    unsigned short inv[T];                 // tile position of sorted slot i
    u64 scan_tmp[32];
    u64 info[16];
    // followed by raw[k+1][T] u32 (payload staged by cp.async)
};

__device__ __forceinline__ void cp_async4(u32* smem_dst, const u32* gsrc) {
    u32 s = (u32)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(u32* smem_dst, const u32* gsrc) {
    u32 s = (u32)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int ITEMS>
__global__ void __launch_bounds__(kThreads, 2) pass_kernel(PassArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PassSmem<ITEMS>& S = *reinterpret_cast<PassSmem<ITEMS>*>(smem_raw);
    constexpr int T = PassSmem<ITEMS>::T;
    u32* raw = reinterpret_cast<u32*>(smem_raw + sizeof(PassSmem<ITEMS>));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
    const LevelGeom& g = a.g;
    const int p = a.pass;
    const int shift = 8 * p;
    const int A = a.k + 1;

    if (tid == 0) {
        u64 tile = atomicAdd(a.tile_ctr, 1u);
        u64 ts = tile * T;
        u64 cnt = g.nview - ts < (u64)T ? g.nview - ts : (u64)T;
        u64 j0 = v_seg_of(g, ts);
        u64 s0b = v_ibegin(g, j0), s0e = s0b + v_size(g, j0);
        uint8_t st0 = a.state[j0];
        u64 r0a = s0b > ts ? s0b - ts : 0ull;
        u64 r0b = s0e > ts ? ((s0e - ts < cnt) ? s0e - ts : cnt) : 0ull;
        bool act0 = ((st0 >> p) & 1u) && r0a < r0b;
        u64 r1a = cnt, r1b = cnt;
        bool has1 = false, act1 = false;
        uint8_t st1 = 0;
        if (j0 + 1 < g.nseg) {
            u64 s1b = v_ibegin(g, j0 + 1);
            if (s1b < ts + cnt) {
                has1 = true;
                st1 = a.state[j0 + 1];
                act1 = (st1 >> p) & 1u;
                r1a = s1b - ts;
                u64 s1e = s1b + v_size(g, j0 + 1);
                r1b = (s1e - ts < cnt) ? s1e - ts : cnt;
            }
        }
        u32 src0 = ((st0 >> 4) ^ (u32)__popc(st0 & ((1u << p) - 1u))) & 1u;
        u32 src1 = ((st1 >> 4) ^ (u32)__popc(st1 & ((1u << p) - 1u))) & 1u;
        S.info[0] = tile;
        S.info[1] = ts;
        S.info[2] = act0 ? r0a : 0;
        S.info[3] = act0 ? r0b : 0;
        S.info[4] = act1 ? r1a : cnt;
        S.info[5] = act1 ? r1b : cnt;
        S.info[6] = j0;
        S.info[7] = (act0 ? 1u : 0u) | (act1 ? 2u : 0u) | (has1 ? 4u : 0u) | ((act0 && s0b < ts) ? 8u : 0u) |
                    (src0 << 4) | (src1 << 5);
        S.info[9] = s0b;
        S.info[10] = has1 ? s0e + 1 : 0;  // in-order begin of segment j0+1
        u64 nact = (act0 ? r0b - r0a : 0) + (act1 ? r1b - r1a : 0);
        if (nact && a.moved) atomicAdd(a.moved, nact);
        S.info[11] = (u64)seg_dim(a.mode, a.split_dims, g, a.k, j0) |
                     ((u64)(has1 ? seg_dim(a.mode, a.split_dims, g, a.k, j0 + 1) : 0) << 8);
    }
    for (int i = tid; i < kWarps * kBuckets / 2; i += kThreads) reinterpret_cast<u32*>(&S.cnt[0][0])[i] = 0u;
    __syncthreads();
    const u32 flags = (u32)S.info[7];
    if ((flags & 3u) == 0) return;  // neither segment reorders in this pass
    const u64 tile = S.info[0], ts = S.info[1];
    const u32 r0a = (u32)S.info[2], r0b = (u32)S.info[3], r1a = (u32)S.info[4], r1b = (u32)S.info[5];
    const u64 j0 = S.info[6];
    const bool act0 = flags & 1u, act1 = flags & 2u, need_lb = flags & 8u;
    const u32 src0 = (flags >> 4) & 1u, src1 = (flags >> 5) & 1u;
    const int d0 = (int)(S.info[11] & 255u), d1 = (int)((S.info[11] >> 8) & 255u);

    // --- stage the payload of the active elements (all k+1 arrays) with
    // cp.async while the keys are ranked
    // 16-byte chunks (stride is a multiple of 4 words); only a chunk that
    // straddles a part boundary falls back to per-word copies
#pragma unroll
    for (u32 chunk = tid; chunk < (u32)T / 4u; chunk += kThreads) {
        const u32 r = chunk * 4u;
        const bool all0 = r >= r0a && r + 4 <= r0b, all1 = r >= r1a && r + 4 <= r1b;
        const bool any0 = r < r0b && r + 4 > r0a, any1 = r < r1b && r + 4 > r1a;
        if (all0 || all1) {
            const u32* g = a.bf.w[all1 ? src1 : src0] + ts + r;
            for (int c = 0; c < A; ++c) cp_async16(raw + c * T + r, g + (u64)c * a.bf.stride);
        } else if (any0 || any1) {
            for (u32 q = r; q < r + 4; ++q) {
                const bool in0 = q >= r0a && q < r0b, in1 = q >= r1a && q < r1b;
                if (!(in0 || in1)) continue;
                const u32* g = a.bf.w[in1 ? src1 : src0] + ts + q;
                for (int c = 0; c < A; ++c) cp_async4(raw + c * T + q, g + (u64)c * a.bf.stride);
            }
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");

    u32 key[ITEMS];
    const u32* k0p = a.bf.w[src0] + (u64)d0 * a.bf.stride + ts;
    const u32* k1p = a.bf.w[src1] + (u64)d1 * a.bf.stride + ts;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        u32 r = (u32)(warp * ITEMS * 32 + i * 32 + lane);
        bool in0 = r >= r0a && r < r0b, in1 = r >= r1a && r < r1b;
        key[i] = 0u;
        if (in0) key[i] = k0p[r];
        else if (in1) key[i] = k1p[r];
    }
    // --- warp-level stable ranking: peers of each element's bucket from
    // bit-sliced ballots, then the per-round counter bumps by each group's
    // highest lane
    u32 br[ITEMS];  // bucket << 16 | warp-local rank
    u32 peers[ITEMS];
    const u32 lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const u32 row = (u32)(warp * ITEMS * 32 + i * 32);
        u32 r = row + lane;
        bool in0 = r >= r0a && r < r0b, in1 = r >= r1a && r < r1b;
        u32 dg = (flip_key(__uint_as_float(key[i])) >> shift) & 255u;
        u32 b = in0 ? dg : (in1 ? (dg | 256u) : (0x1000u | lane));
        br[i] = b;
        // a row entirely inside one active part (the common case) needs only
        // the 8 digit bits; otherwise the segment bit and validity join in
        const bool full = (row >= r0a && row + 32 <= r0b) || (row >= r1a && row + 32 <= r1b);
        peers[i] = full ? warp_peers_full<8>(dg) : warp_peers<9>(b, in0 || in1);
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const u32 b = br[i];
        const int leader = 31 - __clz(peers[i]);
        u32 c = 0;
        if (lane == leader && b < 1024u) {
            c = S.cnt[warp][b];
            S.cnt[warp][b] = (unsigned short)(c + __popc(peers[i]));
        }
        c = __shfl_sync(kFullMask, c, leader);
        br[i] = ((b & 0xffffu) << 16) | (c + __popc(peers[i] & lt));
        __syncwarp();
    }
    __syncthreads();

    // --- thread t owns bucket t: warp prefixes and the tile count
    u32 tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        u32 c = S.cnt[w][tid];
        S.cnt[w][tid] = (unsigned short)tot;
        tot += c;
    }
    // --- publish the counts of this tile's LAST segment (if it reorders)
    u64* my_status = a.bf.status + tile * 256ull;
    const bool has1 = flags & 4u;
    if (tid < 256) {
        if (!has1 && act0) st_relaxed_u64(my_status + tid, pack_status(a.epoch, need_lb ? kFlagAgg : kFlagInc, tot));
    } else if (act1) {
        st_relaxed_u64(my_status + (tid - 256), pack_status(a.epoch, kFlagInc, tot));
    }
    // --- one scan: tile-local bucket starts (low) + per-segment digit bases
    // from the level histogram (high)
    u32 hv = 0;
    if (tid < 256) { if (act0) hv = a.bf.hist[(j0 * 4ull + p) * 256ull + tid]; }
    else if (act1) hv = a.bf.hist[((j0 + 1) * 4ull + p) * 256ull + (tid - 256)];
    u64 ex = block_exclusive_scan<u64>((u64)tot | ((u64)hv << 32), S.scan_tmp, nullptr);
    const u32 bstart = (u32)(ex & 0xffffffffu);
    u32 base = (u32)(ex >> 32);
    if (tid == 256) S.info[8] = ex >> 32;  // histogram total of segment j0
    S.bstart[tid] = bstart;
    __syncthreads();
    if (tid >= 256) base -= (u32)S.info[8];

    // --- decoupled lookback for segment j0 (digit = tid), four predecessors
    // per round trip
    u32 prefix = 0;
    if (tid < 256 && need_lb) {
        long long t = (long long)tile - 1;
        while (true) {
            u64 w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                w[q] = (t - q >= 0) ? ld_relaxed_u64(a.bf.status + (u64)(t - q) * 256ull + tid) : 0ull;
            int q = 0;
            bool done = false;
#pragma unroll
            for (; q < 4; ++q) {
                u64 fl = (w[q] >> 32) & 3ull;
                if ((u32)(w[q] >> 34) != a.epoch || fl == 0) break;
                prefix += (u32)(w[q] & 0xffffffffu);
                if (fl == kFlagInc) { done = true; break; }
            }
            if (done) break;
            if (q == 0) __nanosleep(100);  // predecessor not ready: yield issue slots
            t -= q;
        }
        if (!has1) st_relaxed_u64(my_status + tid, pack_status(a.epoch, kFlagInc, prefix + tot));
    }
    S.gdelta[tid] = base + prefix - bstart;
    __syncthreads();

    // --- sorted slot -> (tile position, destination)
    const u64 ib0 = S.info[9], ib1 = S.info[10];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const u32 b = br[i] >> 16;
        if (b < 1024u) {
            u32 r = (u32)(warp * ITEMS * 32 + i * 32 + lane);
            u32 slot = S.bstart[b] + S.cnt[warp][b] + (br[i] & 0xffffu);
            S.inv[slot] = (unsigned short)r;
            S.dstoff[slot] = (u32)((b & 256u) ? ib1 : ib0) + S.gdelta[b] + slot;
        }
    }
    cp_async_wait_all();
    __syncthreads();

    // --- coalesced write-out of every array (runs of one bucket are contiguous)
    const u32 nact = (r0b - r0a) + (r1b - r1a);
    const u32 split1 = S.bstart[256];
    u32* dst0 = a.bf.w[src0 ^ 1u];
    u32* dst1 = a.bf.w[src1 ^ 1u];
    const u64 stride = a.bf.stride;
    for (u32 i = tid; i < nact; i += kThreads) {
        const u32* rp = raw + S.inv[i];
        u32* d = ((i >= split1) ? dst1 : dst0) + S.dstoff[i];
        for (int c = 0; c < A; ++c) {
            *d = rp[c * T];
            d += stride;
        }
    }
}

template <int ITEMS>
static void launch_pass_t(const PassArgs& a, unsigned grid, cudaStream_t st) {
    size_t sm = sizeof(PassSmem<ITEMS>) + (size_t)(a.k + 1) * PassSmem<ITEMS>::T * sizeof(u32);
    cudaFuncSetAttribute(pass_kernel<ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    pass_kernel<ITEMS><<<grid, kThreads, sm, st>>>(a);
}

void launch_pass(const BuildParams& bp, const Buffers& bf, int l, int pass, u32 epoch, u32* tile_ctr,
                 u64* moved, cudaStream_t st) {
    PassArgs a;
    a.g = view_of(bp, l);
    a.pass = pass;
    a.k = bp.k;
    a.mode = bp.mode;
    a.epoch = epoch;
    a.bf = bf;
    a.state = bf.state[l & 1];
    a.split_dims = bp.split_dims;
    a.tile_ctr = tile_ctr;
    a.moved = moved;
    int items = items_for_bits(bp.b);
    const u64 T = (u64)kThreads * items;
    unsigned grid = (unsigned)((a.g.nview + T - 1) / T);
    switch (items) {  // the sort path requires b >= 10 (capi.cu)
        case 8: launch_pass_t<8>(a, grid, st); break;
        case 4: launch_pass_t<4>(a, grid, st); break;
        case 2: launch_pass_t<2>(a, grid, st); break;
        default: launch_pass_t<1>(a, grid, st); break;
    }
}

// ---------------------------------------------------------------------------
// pivots: after the level's passes every segment is sorted in place; its
// pivot (kernels_numba.py:21-46 arithmetic) is node F(l)+j.  One thread per
// node copies index and point to the level-order output.
// ---------------------------------------------------------------------------
__global__ void pivot_kernel(LevelGeom g, int k, Buffers bf, const uint8_t* state, u32* perm, float* out) {
    u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x;
    if (j >= g.nseg) return;
    u32 par = parity_out(state[j]);
    u64 pos = v_ibegin(g, j) + v_pivot(g, j);
    u64 node = g.Fl + g.sbase + j;
    const u32* w = bf.w[par];
    perm[node] = w[(u64)k * bf.stride + pos];
    for (int c = 0; c < k; ++c) out[node * k + c] = __uint_as_float(w[(u64)c * bf.stride + pos]);
}

// ---------------------------------------------------------------------------
// extract (multi-device rank 0): after the top levels, subtree j of level
// `top` is one contiguous in-order range of every SoA array; copy it to the
// packed send buffer at offset seg_begin(j) (the compacted begin = the sum of
// the sizes of the subtrees before it).
// ---------------------------------------------------------------------------
__global__ void extract_kernel(LevelGeom g, int k, Buffers bf, const uint8_t* prev_state, int src_par, u32* d_sub,
                               u64 sub_stride) {
    // local segment t of the view (global segment sbase + t)
    const u64 t = blockIdx.y / (u64)(k + 1);
    const int c = (int)(blockIdx.y % (u64)(k + 1));
    const u32 par = src_par >= 0 ? (u32)src_par : parity_out(prev_state[t >> 1]);
    const u32* src = bf.w[par] + (u64)c * bf.stride + v_ibegin(g, t);
    // packed: the sizes of the view's earlier segments
    u32* dst = d_sub + (u64)c * sub_stride + (seg_begin(g, g.sbase + t) - seg_begin(g, g.sbase));
    const u64 m = v_size(g, t);
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// the view's level-`top` subtrees (whole tree: lroot = 0)
void launch_extract(const BuildParams& bp, const Buffers& bf, int top, u32* d_sub, u64 sub_stride, int src_par,
                    cudaStream_t st) {
    LevelGeom g = view_of(bp, top);
    dim3 grid(148 * 2, (unsigned)(g.nseg * (u64)(bp.k + 1)));
    extract_kernel<<<grid, 256, 0, st>>>(g, bp.k, bf, bf.state[(top - 1) & 1], src_par, d_sub, sub_stride);
}

void launch_pivots(const BuildParams& bp, const Buffers& bf, int l, cudaStream_t st) {
    LevelGeom g = view_of(bp, l);
    unsigned blocks = (unsigned)((g.nseg + 255) / 256);
    pivot_kernel<<<blocks, 256, 0, st>>>(g, bp.k, bf, bf.state[l & 1], bp.perm, bp.out_pts);
}

}  // namespace lbkd
