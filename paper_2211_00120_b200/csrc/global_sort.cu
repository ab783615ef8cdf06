// global_sort.cu -- the per-level "sort phase" of the top (large-segment)
// levels: a segmented, stable, onesweep LSD radix sort of W_l by the split
// coordinate, with the updateTags refinement fused into its last digit pass.
//
// Reference semantics (what must come out bit-exact):
//   sort_phase   /root/reference/pkg/src/lbkd/builder.py:165-181
//       np.lexsort((coords[:, l % k], tags)): stable by (tag, coordinate)
//   update_tags_round_robin  kernels_numba.py:21-46 (pivot arithmetic)
//   sort_phase_widest        widest.py:119-131 (minor key = own coord in the
//                            tag's dimension)
//
// Why segmented: after update pass l-1 every element carries the tag of the
// level-l node whose contiguous segment it sits in, and tags are already in
// ascending order along the array (children 2s+1 < 2s+2 < 2(s+1)+1).  The
// (tag, coord) sort therefore never moves an element across segments: the
// tag digits of the packed 64-bit key are provably constant-order and their
// digit passes are skipped entirely; what remains is a stable sort of each
// segment by its 32-bit order-flipped coordinate.  Segment boundaries come
// from O(1) treemath arithmetic, not from stored tags.
//
// Each digit pass is one onesweep kernel: per-tile warp-match ranking into
// shared memory, decoupled lookback across the tiles of a segment, and a
// shared-memory-staged coalesced scatter.  Tiles (T = 2^(b-1) keys) are never
// larger than the smallest segment on the global levels, so a tile spans at
// most two segments; only the first can have started in an earlier tile.
#include "kernels.cuh"

namespace lbkd {

constexpr int kPassThreads = 256;
constexpr int kBuckets = 512;  // 2 segments x 256 digits per tile

int global_items_for_bits(int b) { return (1 << (b - 1)) / kPassThreads; }

// ---------------------------------------------------------------------------
// rekey + histogram: keys[p] = flip(coord of point vals[p] in the split dim of
// p's segment); per-(segment, digit-pass, digit) counts; per-segment AND/OR of
// the keys (digit-pass skipping).  Level 0 reads the points sequentially,
// writes vals = identity and checks every coordinate is finite.
// ---------------------------------------------------------------------------
struct RekeyArgs {
    LevelGeom g;
    int k, mode, level0, items, tiles_per_cta;
    u64 ntiles;
    const float* pts;
    const uint8_t* split_dims;
    u32* keys[2];
    u32* vals[2];
    const LevelPlan* plan;
    u32* hist;
    u32* seg_and;
    u32* seg_or;
    u32* err;
};

__device__ __forceinline__ void hist_add(u32* h, u32 d, bool inc) {
    u32 v = inc ? d : (0x10000u | threadIdx.x);
    u32 peers = __match_any_sync(kFullMask, v);
    int leader = __ffs(peers) - 1;
    if (inc && (int)(threadIdx.x & 31) == leader) atomicAdd(&h[d], (u32)__popc(peers));
}

template <int ITEMS>
__global__ void __launch_bounds__(kPassThreads) rekey_hist_kernel(RekeyArgs a) {
    __shared__ u32 h[4 * 256];
    __shared__ u32 s_and[kPassThreads / 32], s_or[kPassThreads / 32];
    constexpr int T = kPassThreads * ITEMS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const LevelGeom& g = a.g;
    const u32 sel = a.level0 ? 0u : a.plan->next_sel;
    const u32* vin = a.vals[sel];
    u32* kout = a.keys[sel];
    u32* vout = a.vals[sel];
    for (int i = threadIdx.x; i < 4 * 256; i += kPassThreads) h[i] = 0;

    u64 t0 = (u64)blockIdx.x * a.tiles_per_cta;
    u64 t1 = t0 + a.tiles_per_cta;
    if (t1 > a.ntiles) t1 = a.ntiles;
    if (t0 >= t1) return;
    u64 cur = seg_of(g, t0 * T);
    u32 acc_and = 0xffffffffu, acc_or = 0u;
    bool bad = false;
    int dim_rr = g.l % a.k;
    __syncthreads();

    auto flush = [&](u64 seg) {
        u32 wa = __reduce_and_sync(kFullMask, acc_and);
        u32 wo = __reduce_or_sync(kFullMask, acc_or);
        if (lane == 0) { s_and[warp] = wa; s_or[warp] = wo; }
        __syncthreads();
        u32* gh = a.hist + seg * 1024ull;
        for (int i = threadIdx.x; i < 1024; i += kPassThreads) {
            u32 v = h[i];
            if (v) { atomicAdd(&gh[i], v); h[i] = 0; }
        }
        if (threadIdx.x == 0) {
            u32 A = 0xffffffffu, O = 0u;
            for (int w = 0; w < kPassThreads / 32; ++w) { A &= s_and[w]; O |= s_or[w]; }
            atomicAnd(&a.seg_and[seg], A);
            atomicOr(&a.seg_or[seg], O);
        }
        acc_and = 0xffffffffu;
        acc_or = 0u;
        __syncthreads();
    };

    for (u64 t = t0; t < t1; ++t) {
        u64 ts = t * T;
        u64 cnt = g.nl - ts < (u64)T ? g.nl - ts : (u64)T;
        u64 nb = (cur + 1 < g.nseg) ? seg_begin(g, cur + 1) : ~0ull;
        u64 bnd = (nb >= ts && nb < ts + cnt) ? nb - ts : cnt;  // first pos of next seg
        u32 key[ITEMS];
        u32 rel[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            u32 r = (u32)(warp * ITEMS * 32 + i * 32 + lane);
            rel[i] = r;
            key[i] = 0;
            if (r < cnt) {
                u64 p = ts + r;
                u32 idx;
                int d;
                if (a.level0) {
                    idx = (u32)p;
                    vout[p] = idx;
                    const float* q = a.pts + (u64)idx * a.k;
                    for (int c = 0; c < a.k; ++c) {
                        float f = q[c];
                        if (!isfinite(f)) bad = true;
                    }
                } else {
                    idx = vin[p];
                }
                if (a.mode == kRoundRobin) {
                    d = dim_rr;
                } else {
                    u64 seg = (r < bnd) ? cur : cur + 1;
                    d = a.split_dims[g.Fl + seg];
                }
                key[i] = flip_key(__ldg(a.pts + (u64)idx * a.k + d));
                kout[p] = key[i];
            }
        }
        // phase A: elements of segment `cur`
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            bool inc = rel[i] < bnd;
            if (inc) { acc_and &= key[i]; acc_or |= key[i]; }
#pragma unroll
            for (int q = 0; q < 4; ++q) hist_add(h + q * 256, (key[i] >> (8 * q)) & 255u, inc);
        }
        if (bnd < cnt) {
            __syncthreads();
            flush(cur);
            ++cur;
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                bool inc = rel[i] >= bnd && rel[i] < cnt;
                if (inc) { acc_and &= key[i]; acc_or |= key[i]; }
#pragma unroll
                for (int q = 0; q < 4; ++q) hist_add(h + q * 256, (key[i] >> (8 * q)) & 255u, inc);
            }
        }
    }
    __syncthreads();
    flush(cur);
    if (bad) atomicOr(a.err, 1u);
}

void launch_rekey_hist(const BuildParams& bp, const Buffers& bf, int l, cudaStream_t st) {
    RekeyArgs a;
    a.g = make_geom(bp.n, l);
    a.k = bp.k;
    a.mode = bp.mode;
    a.level0 = (l == 0);
    a.items = global_items_for_bits(bp.b);
    const u64 T = (u64)kPassThreads * a.items;
    a.ntiles = (a.g.nl + T - 1) / T;
    // persistent-ish: ~8 CTAs per SM, each a contiguous run of tiles, so the
    // per-segment histogram flushes stay O(#CTAs + #segments)
    u64 target = 148 * 8;
    u64 tpc = (a.ntiles + target - 1) / target;
    if (tpc < 1) tpc = 1;
    a.tiles_per_cta = (int)tpc;
    a.pts = bp.pts;
    a.split_dims = bp.split_dims;
    for (int i = 0; i < 2; ++i) { a.keys[i] = bf.keys[i]; a.vals[i] = bf.vals[i]; }
    a.plan = bf.plan;
    a.hist = bf.hist;
    a.seg_and = bf.seg_and;
    a.seg_or = bf.seg_or;
    a.err = bf.err;
    unsigned grid = (unsigned)((a.ntiles + tpc - 1) / tpc);
    switch (a.items) {
        case 16: rekey_hist_kernel<16><<<grid, kPassThreads, 0, st>>>(a); break;
        case 8: rekey_hist_kernel<8><<<grid, kPassThreads, 0, st>>>(a); break;
        default: rekey_hist_kernel<4><<<grid, kPassThreads, 0, st>>>(a); break;
    }
}

// ---------------------------------------------------------------------------
// plan: which digit passes are identities (digit constant inside every
// segment), which pass is last (it carries the updateTags epilogue), and the
// ping-pong buffer each pass reads.  One CTA.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) plan_kernel(LevelPlan* plan, const u32* seg_and,
                                                    const u32* seg_or, u64 nseg) {
    __shared__ u32 s_red[32];
    u32 x = 0;
    for (u64 s = threadIdx.x; s < nseg; s += blockDim.x) x |= seg_and[s] ^ seg_or[s];
    x = __reduce_or_sync(kFullMask, x);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        u32 v = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v |= s_red[w];
        u32 nontriv[4];
        for (int p = 0; p < 4; ++p) nontriv[p] = ((v >> (8 * p)) & 255u) != 0;
        int fin = 0;
        for (int p = 0; p < 4; ++p)
            if (nontriv[p]) fin = p;
        u32 cur = plan->next_sel;
        LevelPlan np;
        for (int p = 0; p < 4; ++p) {
            bool run = (p == fin) || (p < fin && nontriv[p]);
            np.skip[p] = run ? 0u : 1u;
            np.src[p] = cur;
            if (run) cur ^= 1u;
        }
        np.final_pass = (u32)fin;
        np.next_sel = cur;
        np.pad[0] = np.pad[1] = 0;
        *plan = np;
    }
}

void launch_plan(const BuildParams& bp, const Buffers& bf, int l, cudaStream_t st) {
    LevelGeom g = make_geom(bp.n, l);
    plan_kernel<<<1, 1024, 0, st>>>(bf.plan, bf.seg_and, bf.seg_or, g.nseg);
}

// ---------------------------------------------------------------------------
// onesweep digit pass
// ---------------------------------------------------------------------------
struct PassArgs {
    LevelGeom g, gn;  // this level, next level
    int pass, k;
    u32 epoch;
    u64 ntiles;
    u32* keys[2];
    u32* vals[2];
    const u32* hist;
    u64* status;
    u32* tile_ctr;
    const LevelPlan* plan;
    const float* pts;
    float* out_pts;
    u32* perm;
};

template <int ITEMS>
struct PassSmem {
    static constexpr int T = kPassThreads * ITEMS;
    u32 keys[T];
    u32 vals[T];
    unsigned short cnt[kPassThreads / 32][kBuckets];
    u32 bstart[kBuckets + 1];
    u32 gdelta[kBuckets];
    u64 scan_tmp[32];
    u64 info[16];
};

__device__ __forceinline__ void write_node(const PassArgs& a, u64 node, u32 idx) {
    a.perm[node] = idx;
    const float* src = a.pts + (u64)idx * a.k;
    float* dst = a.out_pts + node * a.k;
    for (int c = 0; c < a.k; ++c) dst[c] = src[c];
}

template <int ITEMS>
__global__ void __launch_bounds__(kPassThreads) onesweep_pass_kernel(PassArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PassSmem<ITEMS>& S = *reinterpret_cast<PassSmem<ITEMS>*>(smem_raw);
    constexpr int T = PassSmem<ITEMS>::T;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
    const LevelPlan plan = *a.plan;
    if (plan.skip[a.pass]) return;
    const bool fin = (u32)a.pass == plan.final_pass;
    const u32 src = plan.src[a.pass];
    const u32* kin = a.keys[src];
    const u32* vin = a.vals[src];
    u32* kout = a.keys[src ^ 1u];
    u32* vout = a.vals[src ^ 1u];
    const LevelGeom& g = a.g;
    const int shift = 8 * a.pass;

    // --- tile acquisition (in launch order: lookback only waits on earlier
    // tiles, which are already resident) and segment geometry of the tile
    if (tid == 0) {
        u64 tile = atomicAdd(a.tile_ctr, 1u);
        u64 ts = tile * T;
        u64 cnt = g.nl - ts < (u64)T ? g.nl - ts : (u64)T;
        u64 j0 = seg_of(g, ts);
        u64 b0 = seg_begin(g, j0);
        u64 b1 = (j0 + 1 < g.nseg) ? seg_begin(g, j0 + 1) : g.nl;
        u64 bnd = (b1 < ts + cnt) ? b1 - ts : cnt;
        S.info[0] = tile;
        S.info[1] = ts;
        S.info[2] = cnt;
        S.info[3] = j0;
        S.info[4] = b0;
        S.info[5] = b1;
        S.info[6] = bnd;
        S.info[7] = (b0 < ts) ? 1ull : 0ull;  // first segment continues from earlier tiles
    }
    for (int i = tid; i < (kPassThreads / 32) * kBuckets / 2; i += kPassThreads)
        reinterpret_cast<u32*>(&S.cnt[0][0])[i] = 0u;
    __syncthreads();
    const u64 tile = S.info[0], ts = S.info[1];
    const u32 cnt = (u32)S.info[2];
    const u64 j0 = S.info[3];
    const u32 bnd = (u32)S.info[6];
    const bool need_lb = S.info[7] != 0;
    const bool has1 = bnd < cnt;

    // --- load (warp-striped, coalesced) and rank within the warp
    u32 key[ITEMS], val[ITEMS];
    unsigned short bkt[ITEMS], rnk[ITEMS];
    const u32 lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        u32 r = (u32)(warp * ITEMS * 32 + i * 32 + lane);
        bool valid = r < cnt;
        key[i] = valid ? kin[ts + r] : 0u;
        val[i] = valid ? vin[ts + r] : 0u;
        u32 b = valid ? (((key[i] >> shift) & 255u) | (r >= bnd ? 256u : 0u)) : (0x1000u | lane);
        u32 peers = __match_any_sync(kFullMask, b);
        int leader = __ffs(peers) - 1;
        u32 c = 0;
        if (lane == leader && valid) {
            c = S.cnt[warp][b];
            S.cnt[warp][b] = (unsigned short)(c + __popc(peers));
        }
        c = __shfl_sync(kFullMask, c, leader);
        bkt[i] = (unsigned short)(b & 1023u);
        rnk[i] = (unsigned short)(c + __popc(peers & lt));
        __syncwarp();
    }
    __syncthreads();

    // --- per-bucket warp prefixes and tile totals (thread t: buckets t, t+256)
    u32 tot0 = 0, tot1 = 0;
#pragma unroll
    for (int w = 0; w < kPassThreads / 32; ++w) {
        u32 c0 = S.cnt[w][tid], c1 = S.cnt[w][tid + 256];
        S.cnt[w][tid] = (unsigned short)tot0;
        S.cnt[w][tid + 256] = (unsigned short)tot1;
        tot0 += c0;
        tot1 += c1;
    }
    u64 packed_tot;
    u64 ex = block_exclusive_scan<u64>((u64)tot0 | ((u64)tot1 << 32), S.scan_tmp, &S.info[8]);
    const u32 seg0_count = (u32)(S.info[8] & 0xffffffffu);
    S.bstart[tid] = (u32)(ex & 0xffffffffu);
    S.bstart[tid + 256] = seg0_count + (u32)(ex >> 32);
    (void)packed_tot;

    // --- per-segment global digit offsets from the level histogram
    const u32* h0 = a.hist + (j0 * 4ull + a.pass) * 256ull;
    u64 hv = (u64)h0[tid];
    if (has1) hv |= (u64)h0[1024 + tid] << 32;  // segment j0+1 is the next 1024 words
    u64 base = block_exclusive_scan<u64>(hv, S.scan_tmp, nullptr);
    u32 base0 = (u32)(base & 0xffffffffu), base1 = (u32)(base >> 32);

    // --- decoupled lookback (only the first segment can span earlier tiles)
    u64* my_status = a.status + tile * 256ull;
    if (has1) {
        st_relaxed_u64(my_status + tid, pack_status(a.epoch, kFlagInc, tot1));
    } else if (!need_lb) {
        st_relaxed_u64(my_status + tid, pack_status(a.epoch, kFlagInc, tot0));
    } else {
        st_relaxed_u64(my_status + tid, pack_status(a.epoch, kFlagAgg, tot0));
    }
    u32 prefix = 0;
    if (need_lb) {
        u64 t = tile - 1;
        while (true) {
            u64 w = ld_relaxed_u64(a.status + t * 256ull + tid);
            u32 ep = (u32)(w >> 34);
            u64 fl = (w >> 32) & 3ull;
            if (ep != a.epoch || fl == 0) continue;
            prefix += (u32)(w & 0xffffffffu);
            if (fl == kFlagInc) break;
            --t;
        }
        if (!has1) st_relaxed_u64(my_status + tid, pack_status(a.epoch, kFlagInc, prefix + tot0));
    }
    // offset-in-segment of sorted tile slot i is gdelta[bucket] + i
    S.gdelta[tid] = base0 + prefix - S.bstart[tid];
    S.gdelta[tid + 256] = base1 - S.bstart[tid + 256];
    __syncthreads();

    // --- scatter into shared memory in tile-sorted order
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        u32 r = (u32)(warp * ITEMS * 32 + i * 32 + lane);
        if (r < cnt) {
            u32 b = bkt[i];
            u32 slot = S.bstart[b] + S.cnt[warp][b] + rnk[i];
            S.keys[slot] = key[i];
            S.vals[slot] = val[i];
        }
    }
    __syncthreads();

    // --- coalesced global write-out
    const u64 sb0 = S.info[4], sb1 = S.info[5];
    const u32 split1 = S.bstart[256];
    if (!fin) {
#pragma unroll 4
        for (u32 i = tid; i < cnt; i += kPassThreads) {
            u32 k = S.keys[i];
            u32 seg1 = i >= split1 ? 1u : 0u;
            u32 b = ((k >> shift) & 255u) | (seg1 << 8);
            u64 dst = (seg1 ? sb1 : sb0) + (u32)(S.gdelta[b] + i);
            kout[dst] = k;
            vout[dst] = S.vals[i];
        }
        return;
    }
    // final pass: fused updateTags (kernels_numba.py:21-46): the element at
    // the pivot offset becomes node F(l)+j and is written out; the others move
    // to their child's segment of W_{l+1} (pivots compacted away).
    const u64 po0 = pivot_off(g, j0);
    const u64 po1 = has1 ? pivot_off(g, j0 + 1) : 0ull;
    const bool last = (g.l == g.L - 2);
    for (u32 i = tid; i < cnt; i += kPassThreads) {
        u32 k = S.keys[i];
        u32 v = S.vals[i];
        u32 seg1 = i >= split1 ? 1u : 0u;
        u32 b = ((k >> shift) & 255u) | (seg1 << 8);
        u64 o = (u32)(S.gdelta[b] + i);
        u64 j = j0 + seg1;
        u64 po = seg1 ? po1 : po0;
        if (o == po) {
            write_node(a, g.Fl + j, v);
            continue;
        }
        u64 right = o > po ? 1ull : 0ull;
        u64 child = 2ull * j + right;
        if (last) {
            write_node(a, a.gn.Fl + child, v);
            continue;
        }
        u64 off = right ? o - po - 1ull : o;
        vout[seg_begin(a.gn, child) + off] = v;
    }
}

void launch_pass(const BuildParams& bp, const Buffers& bf, int l, int pass, u32 epoch,
                 u32* tile_ctr, cudaStream_t st) {
    PassArgs a;
    a.g = make_geom(bp.n, l);
    a.gn = make_geom(bp.n, l + 1);
    a.pass = pass;
    a.k = bp.k;
    a.epoch = epoch;
    int items = global_items_for_bits(bp.b);
    const u64 T = (u64)kPassThreads * items;
    a.ntiles = (a.g.nl + T - 1) / T;
    for (int i = 0; i < 2; ++i) { a.keys[i] = bf.keys[i]; a.vals[i] = bf.vals[i]; }
    a.hist = bf.hist;
    a.status = bf.status;
    a.tile_ctr = tile_ctr;
    a.plan = bf.plan;
    a.pts = bp.pts;
    a.out_pts = bp.out_pts;
    a.perm = bp.perm;
    unsigned grid = (unsigned)a.ntiles;
    switch (items) {
        case 16: {
            size_t sm = sizeof(PassSmem<16>);
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(onesweep_pass_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                attr = true;
            }
            onesweep_pass_kernel<16><<<grid, kPassThreads, sm, st>>>(a);
            break;
        }
        case 8: {
            size_t sm = sizeof(PassSmem<8>);
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(onesweep_pass_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                attr = true;
            }
            onesweep_pass_kernel<8><<<grid, kPassThreads, sm, st>>>(a);
            break;
        }
        default: {
            size_t sm = sizeof(PassSmem<4>);
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(onesweep_pass_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                attr = true;
            }
            onesweep_pass_kernel<4><<<grid, kPassThreads, sm, st>>>(a);
            break;
        }
    }
}

}  // namespace lbkd
