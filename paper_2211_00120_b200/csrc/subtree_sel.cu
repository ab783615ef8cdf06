// subtree_sel.cu -- the in-CTA levels (lam0 .. L-1) of every level-lam0
// subtree as per-level pivot SELECTION inside one CTA's shared memory, for
// both split rules.  Same argument as the global levels (select.cu, DESIGN.md
// §2): a node's point is the element of rank pivot_off(s) under the node's
// fixed within-node order T(s) = (c[dim(s)], c[dim(parent)], ..., input
// index); where its children's points sit is unobservable.  So no list is
// ever sorted:
//
// block phase (segments > 31 points), per level, all threads:
//   setup   per segment: size, pivot offset (kernels_numba.py:21-46), split
//           dim (RR: l mod k; widest: first f64 argmax of the node box,
//           kernels_numba.py:80-110), NB equal-width buckets of the box
//   hist    every live point -> its segment's bucket (shared atomics)
//   pick    warp per segment: bucket b* holding rank pivot_off
//   gather  points of b* -> the segment's candidate list
//   resolve warp per segment: rank of every candidate under T(s) by
//           comparison (chain fields and the input index only on ties)
//           -> the node; children boxes = box clipped by the node's plane
//   split   every live point -> left / right child by one comparison
// warp phase (segments <= 31 points): one warp per segment holds its points
// in registers and finishes the segment's subtree: each level a point's rank
// inside its node is a 32-lane comparison count.
// Finally the nodes of each level (one contiguous range of the level-order
// output) are written coalesced.
#include "kernels.cuh"

namespace lbkd {

constexpr int kSelThreads = 256;  // four CTAs per SM (b = 11: <= 2047 points each)
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kSelPerSM = 4;
constexpr int kNB = 64;              // buckets per segment (block phase)
constexpr int kWarpSegMax = 31;      // warp phase once segments hold <= 31 points
constexpr int kBoxK = 4;             // widest: per-lane boxes in the warp phase (k <= 4)

struct SelLayout {
    int Mp, nsb, nsw;  // padded capacity, max segments in block / warp phase
    size_t off_P, off_seg, off_cand, off_ntab, off_hist, off_box0, off_box1, off_segv, off_ndim, off_wpv, off_wrk,
        total;
};

// per-segment scalar arrays (u32 each): size, po, dim, bstar, rank, coff,
// ccnt, cfill, piv, lo bits, hi bits -> 11 words
constexpr int kSegWords = 12;

__host__ __device__ inline SelLayout sel_layout(int b, int k) {
    SelLayout s;
    const int M = (1 << b) - 1;
    s.Mp = (M + 8) & ~7;
    s.nsb = b >= 7 ? 1 << (b - 6) : 1;  // segments of the deepest block level
    s.nsw = b >= 6 ? 1 << (b - 5) : 1;  // segments when the warp phase starts
    size_t o = 0;
    s.off_P = o;
    o += sizeof(float) * (size_t)k * s.Mp;
    s.off_seg = o;
    o += 2 * (size_t)s.Mp;
    s.off_cand = o;
    o += 2 * (size_t)s.Mp;
    s.off_ntab = o;
    o += 2 * (size_t)s.Mp;
    o = (o + 15) & ~(size_t)15;
    s.off_hist = o;
    o += sizeof(u32) * (size_t)s.nsb * (kNB / 2);
    s.off_box0 = o;
    o += sizeof(float) * 2 * (size_t)k * s.nsw;
    s.off_box1 = o;
    o += sizeof(float) * 2 * (size_t)k * s.nsw;
    s.off_segv = o;
    o += sizeof(u32) * kSegWords * (size_t)s.nsw;
    s.off_ndim = o;  // widest: split dim of every subtree node (heap order)
    o += (size_t)s.Mp;
    o = (o + 15) & ~(size_t)15;
    s.off_wpv = o;   // warp phase: per warp, pivot plane + dim of each node
    o += (sizeof(float) + sizeof(u32)) * 32 * kSelWarps;
    s.off_wrk = o;   // warp phase: per warp, [k][32] ranks
    o += (size_t)k * 32 * kSelWarps;
    s.total = (o + 127) & ~(size_t)127;
    return s;
}

size_t subtree_sel_smem_bytes(int b, int k) { return sel_layout(b, k).total; }

// kSgLo / kSgHi: bucketer (half lo, scale); kSgDeg: the node box is a point
// (every coordinate of every point in it is equal: the order is the input order)
enum { kSgSize = 0, kSgPo, kSgDim, kSgB, kSgR, kSgOff, kSgCnt, kSgFill, kSgPiv, kSgLo, kSgHi, kSgDeg };
// candidate sets above this size are resolved by a CTA-wide radix select
// instead of all-pairs comparison (O(C^2): the tie-heavy widest cliff)
constexpr u32 kBigCand = 128;

// block-phase bucket of coordinate v in a segment (fp32, round-to-nearest
// each step: monotone in v; NaN -> the top bucket)
__device__ __forceinline__ u32 seg_bucket(const u32* s, float v, u32 top) {
    const float x = __fmul_rn(__fsub_rn(0.5f * v, __uint_as_float(s[kSgLo])), __uint_as_float(s[kSgHi]));
    return x < (float)top ? (u32)x : top;
}

// CTA-wide radix select of rank r among C candidates (local ids in cs) under
// the composite key (chain coordinates flipped, then the row: rowv[x], or x
// when local ids are in row order); losers are overwritten with 0xffff.  Out
// of line: only tie-heavy candidate sets take it (kBigCand).
__device__ __noinline__ void big_select(unsigned short* cs, u32 C, u32 r, const float* P, int Mp, const Chain& wch,
                                        const u32* rowv, u32* hist, u32* piv) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    u32* rh = hist;        // 256 bins
    u32* rr = hist + 256;  // [2][warps] reductions, [3] pick
    u32 n = C;
    auto field = [&](int f, u32 x) -> u32 {
        return f < (int)wch.m ? flip_key(P[(int)wch.d[f] * Mp + x]) : (rowv ? rowv[x] : x);
    };
    for (int f = 0; f <= (int)wch.m && n > 1; ++f) {
        while (n > 1) {
            u32 mn = 0xffffffffu, mx = 0u;
            for (u32 q = tid; q < C; q += kSelThreads) {
                const u32 x = cs[q];
                if (x == 0xffffu) continue;
                const u32 v = field(f, x);
                mn = min(mn, v);
                mx = max(mx, v);
            }
            mn = __reduce_min_sync(kFullMask, mn);
            mx = __reduce_max_sync(kFullMask, mx);
            if (lane == 0) { rr[warp] = mn; rr[kSelWarps + warp] = mx; }
            for (int i = tid; i < 256; i += kSelThreads) rh[i] = 0u;
            __syncthreads();
            mn = 0xffffffffu;
            mx = 0u;
            for (int w = 0; w < kSelWarps; ++w) { mn = min(mn, rr[w]); mx = max(mx, rr[kSelWarps + w]); }
            if (mn == mx) {  // field constant over the live set
                __syncthreads();
                break;
            }
            u32 sh = 0;
            while (((mx - mn) >> sh) > 255u) ++sh;
            for (u32 q = tid; q < C; q += kSelThreads) {
                const u32 x = cs[q];
                if (x != 0xffffu) atomicAdd(&rh[(field(f, x) - mn) >> sh], 1u);
            }
            __syncthreads();
            if (warp == 0) {  // bucket holding rank r: 8 bins per lane
                u32 c8[8], sum = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) { c8[q] = rh[lane * 8 + q]; sum += c8[q]; }
                u32 xs = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const u32 y = __shfl_up_sync(kFullMask, xs, o);
                    if (lane >= o) xs += y;
                }
                u32 cum = xs - sum;
                if (r >= cum && r < xs) {
                    int bsel = 0;
                    for (int q = 0; q < 8; ++q) {
                        if (cum + c8[q] > r) { bsel = lane * 8 + q; break; }
                        cum += c8[q];
                    }
                    rr[2 * kSelWarps] = (u32)bsel;
                    rr[2 * kSelWarps + 1] = cum;
                    rr[2 * kSelWarps + 2] = rh[bsel];
                }
            }
            __syncthreads();
            const u32 bsel = rr[2 * kSelWarps];
            r -= rr[2 * kSelWarps + 1];
            n = rr[2 * kSelWarps + 2];
            for (u32 q = tid; q < C; q += kSelThreads) {
                const u32 x = cs[q];
                if (x != 0xffffu && ((field(f, x) - mn) >> sh) != bsel) cs[q] = 0xffffu;
            }
            __syncthreads();
        }
    }
    for (u32 q = tid; q < C; q += kSelThreads)
        if (cs[q] != 0xffffu) *piv = cs[q];  // the one live candidate
    __syncthreads();
}

template <int KT>
__global__ void __launch_bounds__(kSelThreads, kSelPerSM) subtree_sel_kernel(SubtreeArgs a, int b) {
    if (a.abort_word && *a.abort_word) return;  // non-finite input (select.cu aborted)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ uint8_t s_outer[LBKD_MAX_K];  // widest: distinct dims of the subtree root's ancestors
    __shared__ int s_nouter;
    typedef unsigned short u16;
    const int k = KT ? KT : a.k;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const SelLayout Ly = sel_layout(b, k);
    const int Mp = Ly.Mp;
    float* P = reinterpret_cast<float*>(smem_raw + Ly.off_P);
    u16* seg = reinterpret_cast<u16*>(smem_raw + Ly.off_seg);
    u16* cand = reinterpret_cast<u16*>(smem_raw + Ly.off_cand);
    u16* ntab = reinterpret_cast<u16*>(smem_raw + Ly.off_ntab);
    u32* hist = reinterpret_cast<u32*>(smem_raw + Ly.off_hist);
    float* boxA = reinterpret_cast<float*>(smem_raw + Ly.off_box0);
    float* boxB = reinterpret_cast<float*>(smem_raw + Ly.off_box1);
    u32* sv = reinterpret_cast<u32*>(smem_raw + Ly.off_segv);
    uint8_t* ndim = reinterpret_cast<uint8_t*>(smem_raw + Ly.off_ndim);
    float* wplane = reinterpret_cast<float*>(smem_raw + Ly.off_wpv) + warp * 32;
    u32* wpdim = reinterpret_cast<u32*>(smem_raw + Ly.off_wpv + sizeof(float) * 32 * kSelWarps) + warp * 32;
    const u16 kFin = 0xffffu;

    const int L = a.L;
    const u64 j = a.jbase + blockIdx.x;  // global index of the subtree root at level lam0
    const u64 Bn = a.n - ((1ull << (L - 1)) - 1ull);
    auto seg_size_l = [&](int sh, u64 J) -> u32 {
        const u64 w = 1ull << sh, lo = J << sh;
        u64 on = Bn > lo ? Bn - lo : 0ull;
        if (on > w) on = w;
        return (u32)(w - 1ull + on);
    };
    auto pivot_off_l = [&](int sh, u64 J) -> u32 {
        if (sh <= 0) return 0u;
        const u64 cw = 1ull << (sh - 1), lo = (2ull * J) * cw;
        u64 on = Bn > lo ? Bn - lo : 0ull;
        if (on > cw) on = cw;
        return (u32)(cw - 1ull + on);
    };
    const int lam0 = a.lam0;
    const int m = (int)(a.from_pts ? a.n : seg_size_l(L - lam0 - 1, j));

    // ---- load the subtree's points (coalesced; input order = local id order)
    const u32* src = nullptr;
    const u32* vin = nullptr;
    if (!a.from_pts) {
        u32 par = 0;
        if (a.src_par >= 0) {
            par = (u32)a.src_par;
        } else if (lam0 != a.lfirst) {
            const uint8_t st = a.prev_state[blockIdx.x >> 1];
            par = ((st >> 4) ^ (u32)__popc(st & 15u)) & 1u;
        }
        const LevelGeom g0 = make_geom(a.n, lam0);
        src = a.w[par] + (seg_ibegin(g0, j) - a.pbase);
        vin = src + (u64)k * a.stride;
    }
    if (src) {
        // all loads in flight at once: 4-byte cp.async straight into shared
        // memory (the subtree's slice starts at an arbitrary word)
        for (int c = 0; c < k; ++c) {
            const u32* g = src + (u64)c * a.stride;
            for (int lid = tid; lid < m; lid += kSelThreads) {
                const u32 sa = (u32)__cvta_generic_to_shared(P + c * Mp + lid);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(g + lid) : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int lid = tid; lid < m; lid += kSelThreads) {
        if (!src) {
            const float* q = a.pts + (u64)lid * k;
            for (int c = 0; c < k; ++c) P[c * Mp + lid] = q[c];
        }
        seg[lid] = 0;
    }
    if (src) asm volatile("cp.async.wait_all;" ::: "memory");
    if (tid == 0) {  // (the chains' tail above the subtree: widest_chain_of)
        int no = 0;
        if (a.mode == kWidest && lam0 > 0) {
            u32 seen = 0;
            u64 s = ((1ull << (lam0 - 1)) - 1ull) + (j >> 1);  // parent of the subtree root
            while (true) {
                const int d = a.split_dims[s];
                if (!((seen >> d) & 1u)) {
                    seen |= 1u << d;
                    s_outer[no++] = (uint8_t)d;
                    if (no == k) break;
                }
                if (s == 0) break;
                s = (s - 1) >> 1;
            }
        }
        s_nouter = no;
    }
    // input row of a local id (the final tie-break of every chain)
    auto idx_of = [&](u32 lid) -> u32 { return vin ? vin[lid] : lid; };
    // input-row order of two local ids: a subtree that arrives in input order
    // (select path, single-CTA builds) has local ids in input-row order
    // already -- no global load of the rows
    const bool lid_is_row_order = !a.entry_sorted || !vin;
    auto row_less = [&](u32 x, u32 y) -> bool { return lid_is_row_order ? x < y : idx_of(x) < idx_of(y); };
    // subtree root box (global phase: boxes of level lam0; single-CTA build:
    // reduced here) and, for widest, the dims of the ancestors above the root
    if (a.from_pts) {
        // world box of the whole input (widest.py:84-88)
        for (int c = 0; c < k; ++c) {
            float lo = INFINITY, hi = -INFINITY;
            for (int p = tid; p < m; p += kSelThreads) {
                const float v = P[c * Mp + p];
                lo = fminf(lo, v);
                hi = fmaxf(hi, v);
            }
            // fminf/fmaxf ignore NaN; non-finite input is reported elsewhere
            for (int o = 16; o > 0; o >>= 1) {
                lo = fminf(lo, __shfl_xor_sync(kFullMask, lo, o));
                hi = fmaxf(hi, __shfl_xor_sync(kFullMask, hi, o));
            }
            if (lane == 0) {
                reinterpret_cast<float*>(cand)[2 * warp] = lo;  // cand is free until the first gather
                reinterpret_cast<float*>(cand)[2 * warp + 1] = hi;
            }
            __syncthreads();
            if (tid == 0) {
                float l2 = INFINITY, h2 = -INFINITY;
                for (int w = 0; w < kSelWarps; ++w) {
                    l2 = fminf(l2, reinterpret_cast<float*>(cand)[2 * w]);
                    h2 = fmaxf(h2, reinterpret_cast<float*>(cand)[2 * w + 1]);
                }
                boxA[c] = l2;
                boxA[k + c] = h2;
            }
            __syncthreads();
        }
    } else if (tid < 2 * k) {
        boxA[tid] = a.boxes0[blockIdx.x * 2ull * k + tid];
    }
    __syncthreads();

    // composite order of the chain of a node: c[d0], then the chain fields,
    // then the input row.  chain_at(i) gives the i-th chain dim (i >= 1).
    auto less_tie = [&](u32 x, u32 y, int nchain, auto chain_at) -> bool {
        for (int f = 1; f < nchain; ++f) {
            const int d = chain_at(f);
            const u32 kx = flip_key(P[d * Mp + x]), ky = flip_key(P[d * Mp + y]);
            if (kx != ky) return kx < ky;
        }
        return row_less(x, y);
    };
    // widest: chain of a node = its dim, then its ancestors' dims (repeats
    // dropped).  Ancestors inside the subtree come from ndim (heap order),
    // above it from the global split dims.
    // own_dim >= 0: the node's own dim (not yet stored in ndim)
    auto widest_chain_of = [&](u32 heap, int depth, Chain& ch, int own_dim = -1) {
        ch.m = 0;
        u32 seen = 0;
        u32 h = heap;
        int dd = depth;
        while (true) {
            const int d = (h == heap && own_dim >= 0) ? own_dim : ndim[h];
            if (!((seen >> d) & 1u)) {
                seen |= 1u << d;
                ch.d[ch.m++] = (uint8_t)d;
                if ((int)ch.m == k) return;
            }
            if (dd == 0) break;
            h = (h - 1) >> 1;
            --dd;
        }
        // above the subtree: its ancestors' distinct dims in walk order,
        // gathered once per CTA (s_outer) instead of a global walk per call
        for (int q = 0; q < s_nouter; ++q) {
            const int d = s_outer[q];
            if (!((seen >> d) & 1u)) {
                seen |= 1u << d;
                ch.d[ch.m++] = (uint8_t)d;
                if ((int)ch.m == k) return;
            }
        }
    };
    auto first_argmax = [&](const float* box) -> int {
        int best = 0;
        double bw = coord_width(a.wt, 0, box[0], box[k]);
        for (int d = 1; d < k; ++d) {
            const double w = coord_width(a.wt, d, box[d], box[k + d]);
            if (w > bw) { bw = w; best = d; }
        }
        return best;
    };

    int lam = lam0;
    // ======================= block phase =======================
    for (; lam <= L - 1 && (L - lam - 1) >= 5; ++lam) {
        const int sh = L - lam - 1;
        const int dl = lam - lam0;
        const int nloc = 1 << dl;
        const u64 J0 = j << dl;
        const u32 hbase = (1u << dl) - 1u;  // heap index of segment 0
        // buckets per segment: the whole histogram (nsb * kNB bins) split
        // over this level's nloc <= nsb segments -- 2048 at the in-CTA root
        // for b = 11, so the pivot's bucket holds a handful of candidates
        const int nbw = max(kNB / 2, (Ly.nsb * (kNB / 2)) >> dl);  // 32-bit words (2 bins) per segment
        const u32 nbtop = 2u * (u32)nbw - 1u;
        // ---- setup
        for (int t = tid; t < nloc; t += kSelThreads) {
            u32* s = sv + t * kSegWords;
            const float* box = boxA + t * 2 * k;
            const int d = a.mode == kRoundRobin ? lam % k : first_argmax(box);
            if (a.mode == kWidest) {
                ndim[hbase + t] = (uint8_t)d;
                const u64 node = ((1ull << lam) - 1ull) + J0 + t;
                if (node < a.n) a.split_dims[node] = (uint8_t)d;
            }
            s[kSgSize] = seg_size_l(sh, J0 + t);
            s[kSgPo] = pivot_off_l(sh, J0 + t);
            s[kSgDim] = (u32)d;
            // value-linear buckets of the node box in fp32 (halves: no
            // overflow of hi - lo for any finite box); the same function in
            // hist and gather, monotone in the coordinate
            const float hlo = 0.5f * box[d];
            const float w = 0.5f * box[k + d] - hlo;
            s[kSgLo] = __float_as_uint(hlo);
            s[kSgHi] = __float_as_uint(w > 0.0f ? __fdiv_rn((float)(2 * nbw), w) : 0.0f);
            s[kSgFill] = 0u;
            u32 deg = 1u;
            for (int c = 0; c < k; ++c) deg &= box[c] == box[k + c] ? 1u : 0u;
            s[kSgDeg] = deg;
        }
        for (int i = tid; i < nloc * nbw; i += kSelThreads) hist[i] = 0u;
        __syncthreads();
        // ---- hist (two 16-bit bins per word)
        for (int p = tid; p < m; p += kSelThreads) {
            const u32 t = seg[p];
            if (t == kFin) continue;
            const u32* s = sv + t * kSegWords;
            const u32 bk = seg_bucket(s, P[(int)s[kSgDim] * Mp + p], nbtop);
            atomicAdd(&hist[t * nbw + (bk >> 1)], (bk & 1u) ? 0x10000u : 1u);
        }
        __syncthreads();
        // ---- pick: warp per segment
        for (int t = warp; t < nloc; t += kSelWarps) {
            u32* s = sv + t * kSegWords;
            const u32 po = s[kSgPo];
            u32 base = 0;  // elements in the buckets before this 64-bucket chunk
            int bs = 0;
            u32 cum = 0, cnt = 0;
            for (int w0 = 0; w0 < nbw; w0 += 32) {
                const u32 hw = hist[t * nbw + w0 + lane];  // one word (two bins) per lane
                const u32 c0 = hw & 0xffffu, c1 = hw >> 16;
                u32 x = c0 + c1;
                for (int o = 1; o < 32; o <<= 1) {
                    const u32 y = __shfl_up_sync(kFullMask, x, o);
                    if (lane >= o) x += y;
                }
                const u32 ex = base + x - c0 - c1;  // elements before bucket 2*(w0+lane)
                int bsel = -1;
                u32 cu = 0, cn = 0;
                if (po >= ex && po < ex + c0) { bsel = 2 * (w0 + lane); cu = ex; cn = c0; }
                else if (po >= ex + c0 && po < ex + c0 + c1) { bsel = 2 * (w0 + lane) + 1; cu = ex + c0; cn = c1; }
                const u32 who = __ballot_sync(kFullMask, bsel >= 0);
                if (who) {
                    const int src_l = __ffs(who) - 1;
                    bs = __shfl_sync(kFullMask, bsel, src_l);
                    cum = __shfl_sync(kFullMask, cu, src_l);
                    cnt = __shfl_sync(kFullMask, cn, src_l);
                    break;
                }
                base += __shfl_sync(kFullMask, x, 31);
            }
            if (lane == 0) {
                s[kSgB] = (u32)bs;
                s[kSgR] = po - cum;
                s[kSgCnt] = cnt;
            }
        }
        __syncthreads();
        // candidate ranges: exclusive scan of the counts (warp 0, 32 segments
        // per step)
        if (warp == 0) {
            u32 base = 0;
            for (int t0 = 0; t0 < nloc; t0 += 32) {
                const int t = t0 + lane;
                const u32 c = t < nloc ? sv[t * kSegWords + kSgCnt] : 0u;
                u32 x = c;
                for (int o = 1; o < 32; o <<= 1) {
                    const u32 y = __shfl_up_sync(kFullMask, x, o);
                    if (lane >= o) x += y;
                }
                if (t < nloc) sv[t * kSegWords + kSgOff] = base + x - c;
                base += __shfl_sync(kFullMask, x, 31);
            }
        }
        __syncthreads();
        // ---- gather the candidates
        for (int p = tid; p < m; p += kSelThreads) {
            const u32 t = seg[p];
            if (t == kFin) continue;
            u32* s = sv + t * kSegWords;
            const u32 bk = seg_bucket(s, P[(int)s[kSgDim] * Mp + p], nbtop);
            if (bk == s[kSgB]) cand[s[kSgOff] + atomicAdd(&s[kSgFill], 1u)] = (u16)p;
        }
        __syncthreads();
        // ---- big candidate sets (tie-heavy / identical / sorted data: the
        // pivot's bucket can hold most of a node): radix select over the
        // composite key (chain coordinates, then the row), the whole CTA on
        // one segment at a time -- per round the live range, 256 buckets,
        // the bucket holding rank r; losers are marked dead in place
        for (int t = 0; t < nloc; ++t) {
            u32* s = sv + t * kSegWords;
            const u32 C = s[kSgCnt];
            if (C <= kBigCand) continue;  // (CTA-uniform)
            u16* cs = cand + s[kSgOff];
            Chain wch;
            if (a.mode == kWidest) widest_chain_of(hbase + t, dl, wch);
            else rr_chain(lam, k, wch);
            big_select(cs, C, s[kSgR], P, Mp, wch, lid_is_row_order ? nullptr : vin, hist, &s[kSgPiv]);
        }
        // ---- resolve: rank of each candidate inside its segment by
        // comparison, one thread per candidate over the whole CTA (a warp per
        // segment left most warps idle at the top levels, where one or two
        // segments hold all candidates); the chain is built only on a tie
        {
            const u32* sl = sv + (nloc - 1) * kSegWords;
            const u32 total = sl[kSgOff] + sl[kSgCnt];
            for (u32 q = tid; q < total; q += kSelThreads) {
                // segment of candidate q: offsets strictly increase (every
                // segment's pivot bucket holds its pivot)
                int lo = 0, hi = nloc - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (sv[mid * kSegWords + kSgOff] <= q) lo = mid;
                    else hi = mid - 1;
                }
                const int t = lo;
                u32* s = sv + t * kSegWords;
                const u32 C = s[kSgCnt], off = s[kSgOff];
                if (C > kBigCand) continue;  // (selected above)
                const int d = (int)s[kSgDim];
                const u32 ci = cand[q];
                const float ki = P[d * Mp + ci];  // finite: float order == flipped-key order
                Chain wch;
                bool have = false;
                u32 rank = 0;
                if (s[kSgDeg]) {  // identical points: the input order decides
                    for (u32 jj = 0; jj < C; ++jj) rank += row_less(cand[off + jj], ci) ? 1u : 0u;
                    if (rank == s[kSgR]) s[kSgPiv] = ci;
                    continue;
                }
                for (u32 jj = 0; jj < C; ++jj) {
                    const u32 cj = cand[off + jj];
                    const float kj = P[d * Mp + cj];
                    bool lt = kj < ki;
                    if (kj == ki && cj != ci) {
                        if (!have) {
                            if (a.mode == kWidest) widest_chain_of(hbase + t, dl, wch);
                            else rr_chain(lam, k, wch);
                            have = true;
                        }
                        lt = less_tie(cj, ci, (int)wch.m, [&](int f) -> int { return wch.d[f]; });
                    }
                    rank += lt ? 1u : 0u;
                }
                if (rank == s[kSgR]) s[kSgPiv] = ci;
            }
        }
        __syncthreads();
        // children boxes, nodes
        for (int t = tid; t < nloc; t += kSelThreads) {
            const u32* s = sv + t * kSegWords;
            const u32 piv = s[kSgPiv];
            const int d = (int)s[kSgDim];
            ntab[hbase + t] = (u16)piv;
            const float plane = P[d * Mp + piv];
            const float* box = boxA + t * 2 * k;
            float* bl = boxB + (2 * t) * 2 * k;
            float* br = boxB + (2 * t + 1) * 2 * k;
            for (int c = 0; c < 2 * k; ++c) { bl[c] = box[c]; br[c] = box[c]; }
            if (plane < bl[k + d]) bl[k + d] = plane;  // left child: hi = min(hi, plane)
            if (plane > br[d]) br[d] = plane;          // right child: lo = max(lo, plane)
        }
        // ---- split: every live point -> left / right child
        for (int p = tid; p < m; p += kSelThreads) {
            const u32 t = seg[p];
            if (t == kFin) continue;
            const u32* s = sv + t * kSegWords;
            const u32 piv = s[kSgPiv];
            if ((u32)p == piv) {
                seg[p] = kFin;
                continue;
            }
            const int d = (int)s[kSgDim];
            const float kp = P[d * Mp + p], kv = P[d * Mp + piv];  // finite: float order == flipped-key order
            bool lt;
            if (kp != kv) {
                lt = kp < kv;
            } else if (s[kSgDeg]) {
                lt = row_less((u32)p, piv);
            } else {
                Chain wch;
                if (a.mode == kWidest) widest_chain_of(hbase + t, dl, wch);
                else rr_chain(lam, k, wch);
                lt = less_tie((u32)p, piv, (int)wch.m, [&](int f) -> int { return wch.d[f]; });
            }
            seg[p] = (u16)(2 * t + (lt ? 0u : 1u));
        }
        __syncthreads();
        float* tb = boxA;
        boxA = boxB;
        boxB = tb;
    }

    // ======================= warp phase =======================
    if (lam <= L - 1) {
        const int dl = lam - lam0;
        const int nloc = 1 << dl;
        const u64 J0 = j << dl;
        const int sh = L - lam - 1;
        // per-segment lists (any order): counts, offsets, scatter
        for (int t = tid; t < nloc; t += kSelThreads) {
            sv[t * kSegWords + kSgCnt] = 0u;
            sv[t * kSegWords + kSgFill] = 0u;
        }
        __syncthreads();
        for (int p = tid; p < m; p += kSelThreads) {
            const u32 t = seg[p];
            if (t != kFin) atomicAdd(&sv[t * kSegWords + kSgCnt], 1u);
        }
        __syncthreads();
        if (warp == 0) {  // segment offsets: warp scan, 32 segments per step
            u32 base = 0;
            for (int t0 = 0; t0 < nloc; t0 += 32) {
                const int t = t0 + lane;
                const u32 c = t < nloc ? sv[t * kSegWords + kSgCnt] : 0u;
                u32 x = c;
                for (int o = 1; o < 32; o <<= 1) {
                    const u32 y = __shfl_up_sync(kFullMask, x, o);
                    if (lane >= o) x += y;
                }
                if (t < nloc) sv[t * kSegWords + kSgOff] = base + x - c;
                base += __shfl_sync(kFullMask, x, 31);
            }
        }
        __syncthreads();
        for (int p = tid; p < m; p += kSelThreads) {
            const u32 t = seg[p];
            if (t == kFin) continue;
            u32* s = sv + t * kSegWords;
            cand[s[kSgOff] + atomicAdd(&s[kSgFill], 1u)] = (u16)p;
        }
        __syncthreads();
        uint8_t* wrk = reinterpret_cast<uint8_t*>(smem_raw + Ly.off_wrk) + warp * 32 * k;  // [k][32] ranks
        for (int t = warp; t < nloc; t += kSelWarps) {
            const u64 Jt = J0 + t;
            const u32* s = sv + t * kSegWords;
            const u32 sz = s[kSgCnt];
            bool act = (u32)lane < sz;
            const u32 lid = act ? cand[s[kSgOff] + lane] : 0u;
            const u32 actm = __ballot_sync(kFullMask, act);
            // ---- rank of every point of the segment under each dimension's
            // order, once: RR: the full chain T_d (exact for every level of
            // the warp phase when lam >= k-1); widest: (c[d], input row),
            // with a per-dim flag for equal coordinates (then the level falls
            // back to full chain comparisons)
            const bool rr_exact = a.mode == kRoundRobin && lam >= k - 1;
            u32 tiemask = 0;  // widest: dims with equal coordinates in the segment
            for (int d = 0; d < k; ++d) {
                const u32 key = act ? flip_key(P[d * Mp + lid]) : 0u;
                // bitonic sort of (key, lane) over the warp: lane p ends with
                // the p-th smallest point, i.e. the rank of point bid is p
                u32 bk = act ? key : 0xffffffffu, bid = (u32)lane;
#pragma unroll
                for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
                    for (int stride = size >> 1; stride > 0; stride >>= 1) {
                        const u32 ok = __shfl_xor_sync(kFullMask, bk, stride);
                        const u32 oi = __shfl_xor_sync(kFullMask, bid, stride);
                        const bool asc = (lane & size) == 0;
                        const bool lower = (lane & stride) == 0;
                        const bool psmall = ok < bk || (ok == bk && oi < bid);
                        if ((lower == asc) == psmall) { bk = ok; bid = oi; }
                    }
                }
                const u32 nk = __shfl_down_sync(kFullMask, bk, 1);
                const u32 tiem = __ballot_sync(kFullMask, lane + 1 < (int)sz && nk == bk);
                u32 rank = 0;
                if (!tiem) {
                    wrk[d * 32 + bid] = (uint8_t)lane;
                    __syncwarp();
                    rank = wrk[d * 32 + lane];
                } else {
                    // equal coordinates: exact ranks by comparison (chain on ties)
                    bool tie = false;
                    for (int i = 0; i < 32; ++i) {
                        const u32 ok = __shfl_sync(kFullMask, key, i);
                        if (((actm >> i) & 1u) && i != lane) {
                            rank += ok < key ? 1u : 0u;
                            tie |= ok == key;
                        }
                    }
                    tiemask |= 1u << d;
                    Chain ch;
                    if (rr_exact) rr_chain(d + ((lam - d + k - 1) / k) * k, k, ch);  // a level with dim d
                    for (int i = 0; i < 32; ++i) {
                        const u32 ok = __shfl_sync(kFullMask, key, i);
                        const u32 ol = __shfl_sync(kFullMask, lid, i);
                        if (act && tie && ((actm >> i) & 1u) && i != lane && ok == key) {
                            const bool lt = rr_exact ? less_tie(ol, lid, (int)ch.m, [&](int f) -> int { return ch.d[f]; })
                                                     : row_less(ol, lid);
                            rank += lt ? 1u : 0u;
                        }
                    }
                }
                __syncwarp();
                wrk[d * 32 + lane] = (uint8_t)rank;
            }
            __syncwarp();
            u32 nd = 0;  // heap index of the point's node inside the segment's subtree (< 31)
            // widest: the point's node box (k <= kBoxK)
            float blo[kBoxK], bhi[kBoxK];
            if (a.mode == kWidest) {
                for (int c = 0; c < kBoxK; ++c)
                    if (c < k) { blo[c] = boxA[t * 2 * k + c]; bhi[c] = boxA[t * 2 * k + k + c]; }
            }
            // lanes of my node (the same mask on every active lane of a node):
            // the segment's lanes, narrowed to my side after every level
            u32 eqn = __ballot_sync(kFullMask, act);
            for (int l2 = lam; l2 <= L - 1; ++l2) {
                const int dd = l2 - lam;
                const int sh2 = L - l2 - 1;
                const u32 off = nd + 1u - (1u << dd);  // node's index among its level inside the segment
                const u64 J = (Jt << dd) + off;
                const u32 heap = (1u << (dl + dd)) - 1u + ((u32)t << dd) + off;  // heap index in the subtree
                int d = l2 % k;
                if (a.mode == kWidest && act) {
                    int best = 0;
                    double bw = coord_width(a.wt, 0, blo[0], bhi[0]);
                    for (int c = 1; c < kBoxK; ++c) {
                        if (c < k) {
                            const double w = coord_width(a.wt, c, blo[c], bhi[c]);
                            if (w > bw) { bw = w; best = c; }
                        }
                    }
                    d = best;
                }
                u32 rank;
                const bool exact = rr_exact || !__any_sync(kFullMask, act && ((tiemask >> d) & 1u));
                if (exact) {
                    // lanes of my node, then those with a smaller precomputed
                    // rank (5 rank bits)
                    const u32 key = act ? (u32)wrk[d * 32 + lane] : 0u;
                    const u32 eq = eqn;
                    // ranks (< 31) present in my node as a bit set: one
                    // segmented OR over each node's lanes
                    rank = 0;
                    if (act) {
                        const u32 keys = __reduce_or_sync(eq, 1u << key);
                        rank = (u32)__popc(keys & ((1u << key) - 1u));
                    }
                } else {
                    // widest with equal coordinates in this dim: full chain comparisons
                    const u32 key = act ? flip_key(P[d * Mp + lid]) : 0u;
                    Chain ch;
                    if (a.mode == kRoundRobin) {
                        rr_chain(l2, k, ch);  // (tiny trees: truncated chains near the root)
                    } else if (act) {
                        widest_chain_of(heap, dl + dd, ch, d);  // the node's own dim heads its chain
                    }
                    rank = 0;
                    for (int i = 0; i < 32; ++i) {
                        const u32 ok = __shfl_sync(kFullMask, key, i);
                        const u32 on = __shfl_sync(kFullMask, act ? nd : 0xffffffffu, i);
                        const u32 ol = __shfl_sync(kFullMask, lid, i);
                        if (act && on == nd && i != lane) {
                            if (ok < key) ++rank;
                            else if (ok == key && less_tie(ol, lid, (int)ch.m, [&](int f) -> int { return ch.d[f]; }))
                                ++rank;
                        }
                    }
                }
                const u32 po = pivot_off_l(sh2, J);
                const bool is_piv = act && rank == po;
                if (is_piv) {
                    ntab[heap] = (u16)lid;
                    if (a.mode == kWidest) {
                        ndim[heap] = (uint8_t)d;
                        const u64 node = ((1ull << l2) - 1ull) + J;
                        if (node < a.n) a.split_dims[node] = (uint8_t)d;
                        wplane[nd] = P[d * Mp + lid];
                        wpdim[nd] = (u32)d;
                    }
                }
                __syncwarp();
                bool right = false;
                if (act && !is_piv) {
                    right = rank > po;
                    if (a.mode == kWidest) {
                        const float pl = wplane[nd];
                        const int pd = (int)wpdim[nd];
                        for (int c = 0; c < kBoxK; ++c) {
                            if (c == pd) {
                                if (right) { if (pl > blo[c]) blo[c] = pl; }
                                else { if (pl < bhi[c]) bhi[c] = pl; }
                            }
                        }
                    }
                    nd = 2u * nd + 1u + (right ? 1u : 0u);
                }
                act = act && !is_piv;
                __syncwarp();
                const u32 live = __ballot_sync(kFullMask, act);
                if (!live) break;
                const u32 rb = __ballot_sync(kFullMask, right);
                eqn &= live & (right ? rb : ~rb);
            }
            __syncwarp();
        }
        (void)sh;
    }

    // ======================= output =======================
    __syncthreads();
    for (int dl = 0; lam0 + dl <= L - 1; ++dl) {
        const int l2 = lam0 + dl;
        const u64 first = ((1ull << l2) - 1ull) + (j << dl);
        if (first >= a.n) break;
        u64 cntn = 1ull << dl;
        if (first + cntn > a.n) cntn = a.n - first;
        const u32 h0 = (1u << dl) - 1u;
        for (u32 i = tid; i < (u32)cntn; i += kSelThreads) a.perm[first + i] = idx_of(ntab[h0 + i]);
        float* dst = a.out_pts + first * (u64)k;
        for (u32 i = tid; i < (u32)cntn * (u32)k; i += kSelThreads) {
            const u32 t = i / (u32)k, c = i - t * (u32)k;
            dst[i] = P[c * Mp + ntab[h0 + t]];
        }
    }
}

void launch_subtree_sel(const SubtreeArgs& a, unsigned grid, int b, cudaStream_t st) {
    const size_t sm = subtree_sel_smem_bytes(b, a.k);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        kern<<<grid, kSelThreads, sm, st>>>(a, b);
    };
    switch (a.k) {
        case 2: go(subtree_sel_kernel<2>); break;
        case 3: go(subtree_sel_kernel<3>); break;
        case 4: go(subtree_sel_kernel<4>); break;
        default: go(subtree_sel_kernel<0>); break;
    }
}

}  // namespace lbkd
