// subtree.cu -- finish every level-lam0 subtree inside one CTA's shared
// memory.  Once a subtree holds at most M = 2^b - 1 points (b = 13 for k <= 4)
// all of its remaining levels (lam0 .. L-2) run without touching HBM: the
// points are gathered once into shared memory, every level runs the same
// stable (segment, coordinate) sort + updateTags split as the global levels
// (builder.py:224-232 / widest.py:172-183), and each finished node is written
// to its level-order slot exactly once.
//
// Per level, per CTA:
//   keys: order-flipped coordinate in the split dimension of the element's
//         node (RR: l mod k; widest: that node's dims, computed below)
//   sort: LSD 8-bit digit passes over the key (digits constant across the
//         whole subtree are skipped), then over the local segment id, each a
//         stable block-wide pass ranked with warp match/ballot counters
//   split: the element at each segment's pivot offset (kernels_numba.py:
//         21-46 arithmetic) is the node; the rest move, compacted, into the
//         child segments
//   widest: child split dims = first argmax of the float64 widths of the
//         clipped domain box (kernels_numba.py:80-110), by walking the
//         in-CTA ancestors' (dim, plane) pairs up to the subtree root box
#include "kernels.cuh"

#include <cstdlib>

namespace lbkd {

constexpr int kSubThreads = 1024;  // general kernel (widest, small trees)
constexpr int kSubWarps = kSubThreads / 32;
constexpr int kRRThreads = 512;    // round-robin kernel: two CTAs per SM
constexpr int kRRWarps = kRRThreads / 32;
constexpr int kMaxRounds = 8;  // M <= 8 x threads -> at most 8 rounds
constexpr int kMaxK = 16;


size_t subtree_smem_bytes(int b, int k, int mode) {
    size_t M = ((size_t)1 << b) - 1;
    size_t bytes = 0;
    bytes += sizeof(float) * (size_t)k * M;           // P (SoA)
    bytes += 2 * sizeof(u32) * M;                       // E0, E1
    bytes += sizeof(unsigned short) * kSubWarps * 256;  // per-warp counters
    bytes += sizeof(u32) * 4 * 256;                     // group sums
    bytes += sizeof(u32) * 64;                          // scratch
    if (mode == kWidest) bytes += M * (sizeof(float) + 1) + 2 * kMaxK * sizeof(float);
    return (bytes + 15) & ~(size_t)15;
}

// One stable block-wide counting pass: Eout[rank(e)] = e for the m elements
// of Ein, ranked by digit(e) in 0..255 with ties kept in Ein order.
template <int NT, typename ET, typename DigitFn>
__device__ __forceinline__ void block_pass(const ET* __restrict__ Ein, ET* __restrict__ Eout, int m,
                                           DigitFn digit, unsigned short (*cnt)[256], u32 (*gsum)[256],
                                           u32* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
    const int C = ((m + NT - 1) / NT) * 32;  // per-warp chunk
    const int R = C / 32;
    for (int i = tid; i < (NT / 32) * 256 / 2; i += NT) reinterpret_cast<u32*>(&cnt[0][0])[i] = 0u;
    __syncthreads();
    const u32 lt = lanemask_lt();
    u32 ev[kMaxRounds];
    u32 dr[kMaxRounds];  // digit << 16 | warp-local rank
#pragma unroll
    for (int r = 0; r < kMaxRounds; ++r) {
        if (r < R) {
            int p = warp * C + r * 32 + lane;
            bool valid = p < m;
            u32 e = valid ? (u32)Ein[p] : 0u;
            u32 d = valid ? digit(e) : (0x1000u | lane);
            u32 peers = warp_peers<8>(d, valid);
            int leader = __ffs(peers) - 1;
            u32 c = 0;
            if (lane == leader && valid) {
                c = cnt[warp][d];
                cnt[warp][d] = (unsigned short)(c + __popc(peers));
            }
            c = __shfl_sync(kFullMask, c, leader);
            ev[r] = e;
            dr[r] = ((d & 255u) << 16) | (c + __popc(peers & lt));
            __syncwarp();
        }
    }
    __syncthreads();
    // warp prefixes per digit: 4 groups of 8 warps walk the counter columns
    {
        const int d = tid & 255, grp = tid >> 8;
        u32 s = 0;
#pragma unroll
        for (int w = grp * 8; w < grp * 8 + 8; ++w) {
            u32 c = cnt[w][d];
            cnt[w][d] = (unsigned short)s;
            s += c;
        }
        gsum[grp][d] = s;
    }
    __syncthreads();
    if (tid < 256) {
        // NT / 256 groups (the unused ones count zero)
        constexpr int NG = NT / 256;
        u32 g0 = gsum[0][tid], g1 = NG > 1 ? gsum[1][tid] : 0u, g2 = NG > 2 ? gsum[2][tid] : 0u,
            g3 = NG > 3 ? gsum[3][tid] : 0u;
        u32 tot = g0 + g1 + g2 + g3;
        // exclusive scan over 256 digit totals within the first 8 warps
        u32 x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u32 y = __shfl_up_sync(kFullMask, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) scratch[warp] = x;
        asm volatile("bar.sync 1, 256;");
        u32 wpre = 0;
        for (int w = 0; w < warp; ++w) wpre += scratch[w];
        u32 base = wpre + x - tot;
        gsum[0][tid] = base;
        gsum[1][tid] = base + g0;
        gsum[2][tid] = base + g0 + g1;
        gsum[3][tid] = base + g0 + g1 + g2;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kMaxRounds; ++r) {
        if (r < R) {
            int p = warp * C + r * 32 + lane;
            if (p < m) {
                u32 d = dr[r] >> 16;
                u32 slot = gsum[warp >> 3][d] + cnt[warp][d] + (dr[r] & 0xffffu);
                Eout[slot] = (ET)ev[r];
            }
        }
    }
    __syncthreads();
}

// Stable sort of the list in buf[cur] (m entries, local id in the low 16
// bits) by the coordinate array Pd, ping-ponging between buf0 and buf1;
// digits constant over the list are skipped.  Returns the new cur.
template <int NT, typename ET>
__device__ __forceinline__ int list_sort_dim(ET* buf0, ET* buf1, int cur, int m, const float* Pd, unsigned short (*cnt)[256],
                             u32 (*gsum)[256], u32* scratch) {
    const int tid = threadIdx.x;
    u32 x_and = 0xffffffffu, x_or = 0u;
    for (int p = tid; p < m; p += NT) {
        const u32 kk = flip_key(Pd[p]);
        x_and &= kk;
        x_or |= kk;
    }
    x_and = __reduce_and_sync(kFullMask, x_and);
    x_or = __reduce_or_sync(kFullMask, x_or);
    scratch[32 + (tid >> 5)] = x_and ^ x_or;  // every lane stores the warp-uniform value: a
    // lane-0 guard here was miscompiled by NVVM 12.9 (it reused the guarded
    // (tid >> 3) == 4 * warp for every lane in the next cnt[warp] address)
    __syncthreads();
    u32 vary = 0;
    for (int w = 0; w < (NT / 32); ++w) vary |= scratch[32 + w];
    __syncthreads();
    for (int q = 0; q < 4; ++q) {
        if (((vary >> (8 * q)) & 255u) == 0) continue;
        const int sh = 8 * q;
        block_pass<NT>(cur ? buf1 : buf0, cur ? buf0 : buf1, m,
                   [&](u32 e) { return (flip_key(Pd[e & 0xffffu]) >> sh) & 255u; }, cnt, gsum, scratch);
        cur ^= 1;
    }
    return cur;
}

// One round-robin chain order T_d = (c[d], c[d-1], ..., c[d-k+1], local id)
// of the m points of P, written to out as local ids, by ONE value-linear
// bucket pass instead of 3-4 radix passes: 2 NB equal-width buckets over the
// points' [min, max] in dim d (monotone in the key, so buckets are ordered),
// shared-atomic counts, a block scan, an atomic scatter, then every bucket
// is put in T_d order by insertion sort under the full chain comparator (the
// scatter's order inside a bucket does not matter).  Local ids compare like
// the input order (ids follow input order, or T_e order -- which agrees with
// the input order on points that tie in all k coordinates).  Returns false,
// leaving out undefined, if some bucket holds more than kBucketRun points
// (tie-heavy data): the caller then runs the radix passes.
constexpr int kBucketRun = 24;

template <int NT, int KT>
__device__ __noinline__ bool bucket_list(unsigned short* __restrict__ out, int m, const float* __restrict__ P, int Mp,
                                         int d, int kk, int NB, u32* __restrict__ hist, u32* __restrict__ scratch) {
    const int k = KT ? KT : kk;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* Pd = P + d * Mp;
    float fmn = __int_as_float(0x7f800000), fmx = -__int_as_float(0x7f800000);
    for (int p = tid; p < m; p += NT) {
        const float x = Pd[p];
        fmn = fminf(fmn, x);
        fmx = fmaxf(fmx, x);
    }
    u32 kmin = flip_key(fmn), kmax = flip_key(fmx);
    for (int b = tid; b < NB; b += NT) hist[b] = 0u;
    kmin = __reduce_min_sync(kFullMask, kmin);
    kmax = __reduce_max_sync(kFullMask, kmax);
    scratch[warp] = kmin;  // every lane stores the warp-uniform value (NVVM 12.9, list_sort_dim)
    scratch[32 + warp] = kmax;
    __syncthreads();
    kmin = 0xffffffffu;
    kmax = 0u;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        kmin = min(kmin, scratch[w]);
        kmax = max(kmax, scratch[32 + w]);
    }
    // 2 NB buckets as 16-bit halves of the NB shared words (counts, then
    // starts, then ends; every value <= m < 2^16, so no half carries)
    const u32 NBK = 2u * (u32)NB;
    const float lo = unflip_key(kmin);
    const float range = __fsub_rn(unflip_key(kmax), lo);
    float scale = range > 0.f ? __fdiv_rn((float)NBK, range) : 0.f;
    if (!(scale <= 3.0e38f)) scale = 0.f;  // overflowing range / denormal width: one bucket -> radix
    auto bucket = [&](float x) -> u32 {
        const u32 b = (u32)__fmul_rn(__fsub_rn(x, lo), scale);  // NaN-free: x >= lo, finite
        return b < NBK ? b : NBK - 1u;
    };
    for (int p = tid; p < m; p += NT) {
        const u32 b = bucket(Pd[p]);
        atomicAdd(&hist[b >> 1], (b & 1u) ? 0x10000u : 1u);
    }
    __syncthreads();
    // exclusive scan over the 2 NB counts, NB / NT consecutive words per
    // thread, and the largest bucket
    const int per = NB / NT;  // a multiple of 4 (NB = Mp >= 4 NT): 16-byte shared loads / stores
    uint4* const h4 = reinterpret_cast<uint4*>(hist) + tid * (per / 4);
    u32 s = 0, big = 0;
    auto acc = [&](u32 c) {
        s += (c & 0xffffu) + (c >> 16);
        big = max(big, max(c & 0xffffu, c >> 16));
    };
    for (int i = 0; i < per / 4; ++i) {
        const uint4 c = h4[i];
        acc(c.x);
        acc(c.y);
        acc(c.z);
        acc(c.w);
    }
    big = __reduce_max_sync(kFullMask, big);
    const u32 ex = block_exclusive_scan_1b<u32>(s, scratch);
    scratch[32 + warp] = big;
    u32 run = ex;
    auto starts = [&](u32 c) -> u32 {
        const u32 s0 = run;
        run += c & 0xffffu;
        const u32 s1 = run;
        run += c >> 16;
        return s0 | (s1 << 16);
    };
    for (int i = 0; i < per / 4; ++i) {
        const uint4 c = h4[i];
        uint4 o;
        o.x = starts(c.x);
        o.y = starts(c.y);
        o.z = starts(c.z);
        o.w = starts(c.w);
        h4[i] = o;
    }
    __syncthreads();
    big = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) big = max(big, scratch[32 + w]);
    if (big > (u32)kBucketRun) {
        __syncthreads();
        return false;
    }
    for (int p = tid; p < m; p += NT) {
        const u32 b = bucket(Pd[p]);
        const u32 old = atomicAdd(&hist[b >> 1], (b & 1u) ? 0x10000u : 1u);
        out[(b & 1u) ? old >> 16 : old & 0xffffu] = (unsigned short)p;
    }
    __syncthreads();
    // the halves now hold the buckets' ends; order each bucket under T_d
    auto isort = [&](int st, int e) {
        for (int i = st + 1; i < e; ++i) {
            // finite coordinates: float order == flipped-key order (-0 == +0)
            const u32 v = out[i];
            const float kv = Pd[v];
            int t = i - 1;
            while (t >= st) {
                const u32 w = out[t];
                const float kw = Pd[w];
                bool less = kv < kw;
                if (kv == kw) {
                    less = v < w;
                    for (int f = 1; f < k; ++f) {
                        const int dd = (d - f + k) % k;
                        const float x = P[dd * Mp + v], y = P[dd * Mp + w];
                        if (x != y) {
                            less = x < y;
                            break;
                        }
                    }
                }
                if (!less) break;
                out[t + 1] = (unsigned short)w;
                --t;
            }
            out[t + 1] = (unsigned short)v;
        }
    };
    for (int w = tid; w < NB; w += NT) {
        const u32 c = hist[w];
        const int e0 = (int)(c & 0xffffu), e1 = (int)(c >> 16);
        const int st0 = w ? (int)(hist[w - 1] >> 16) : 0;
        if (e0 - st0 > 1) isort(st0, e0);
        if (e1 - e0 > 1) isort(e0, e1);
    }
    __syncthreads();
    return true;
}

// Entry order of a subtree that arrives in INPUT order (select path): the
// reference's order inside the subtree root's parent, i.e. the lexicographic
// order of (c[ch.d[0]], ..., c[ch.d[m-1]], input index).  One stable sort by
// the leading field leaves every run of equal leading keys in input order;
// runs of at most kTieRun elements (float data: almost always pairs) are then
// re-ordered by the remaining fields in place, one thread per run (insertion
// sort).  Only when a longer run exists are the remaining fields sorted in
// LSD order from the input order again.  buf0 holds the identity on entry;
// returns the buffer (0/1) holding the result.
constexpr int kTieRun = 32;

__device__ __forceinline__ bool chain_less(u32 a, u32 b, const float* P, int ldP, const Chain& ch) {
    for (u32 f = 1; f < ch.m; ++f) {
        const float* Pd = P + (size_t)ch.d[f] * ldP;
        const u32 x = flip_key(Pd[a]), y = flip_key(Pd[b]);
        if (x != y) return x < y;
    }
    return a < b;  // local ids are in input order
}

template <int NT, typename ET>
__device__ __forceinline__ int entry_order(ET* buf0, ET* buf1, int m, const float* P, int ldP, const Chain& ch,
                           unsigned short (*cnt)[256], u32 (*gsum)[256], u32* scratch) {
    if (ch.m == 0) return 0;
    const float* P0 = P + (size_t)ch.d[0] * ldP;
    int cur = list_sort_dim<NT>(buf0, buf1, 0, m, P0, cnt, gsum, scratch);
    if (ch.m == 1) return cur;
    ET* L = cur ? buf1 : buf0;
    int longrun = 0;
    for (int p = threadIdx.x; p + 1 < m; p += NT) {
        const u32 kp = flip_key(P0[L[p] & 0xffffu]);
        if (flip_key(P0[L[p + 1] & 0xffffu]) != kp) continue;           // no tie at p
        if (p > 0 && flip_key(P0[L[p - 1] & 0xffffu]) == kp) continue;  // not the run's start
        int q = p + 2;
        while (q < m && q - p <= kTieRun && flip_key(P0[L[q] & 0xffffu]) == kp) ++q;
        if (q - p > kTieRun) {
            longrun = 1;
            continue;
        }
        for (int i = p + 1; i < q; ++i) {  // insertion sort of L[p, q)
            const ET v = L[i];
            int t = i - 1;
            while (t >= p && chain_less((u32)v & 0xffffu, (u32)L[t] & 0xffffu, P, ldP, ch)) {
                L[t + 1] = L[t];
                --t;
            }
            L[t + 1] = v;
        }
    }
    if (!__syncthreads_or(longrun)) return cur;
    for (int p = threadIdx.x; p < m; p += NT) buf0[p] = (ET)p;
    __syncthreads();
    cur = 0;
    for (int f = (int)ch.m - 1; f >= 0; --f)
        cur = list_sort_dim<NT>(buf0, buf1, cur, m, P + (size_t)ch.d[f] * ldP, cnt, gsum, scratch);
    return cur;
}

__global__ void __launch_bounds__(kSubThreads, 1) subtree_kernel(SubtreeArgs a) {
    if (a.abort_word && *a.abort_word) return;  // non-finite input (select.cu aborted)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int M = a.M, k = a.k, tid = threadIdx.x;
    unsigned char* sp = smem_raw;
    float* P = reinterpret_cast<float*>(sp);
    sp += sizeof(float) * (size_t)k * M;
    u32* E[2];
    E[0] = reinterpret_cast<u32*>(sp);
    sp += sizeof(u32) * M;
    E[1] = reinterpret_cast<u32*>(sp);
    sp += sizeof(u32) * M;
    unsigned short(*cnt)[256] = reinterpret_cast<unsigned short(*)[256]>(sp);
    sp += sizeof(unsigned short) * kSubWarps * 256;
    u32(*gsum)[256] = reinterpret_cast<u32(*)[256]>(sp);
    sp += sizeof(u32) * 4 * 256;
    u32* scratch = reinterpret_cast<u32*>(sp);
    sp += sizeof(u32) * 64;
    float* nplane = nullptr;
    float* rootbox = nullptr;
    unsigned char* ndim = nullptr;
    if (a.mode == kWidest) {
        nplane = reinterpret_cast<float*>(sp);
        sp += sizeof(float) * M;
        rootbox = reinterpret_cast<float*>(sp);
        sp += sizeof(float) * 2 * kMaxK;
        ndim = sp;
    }

    const u64 jl = blockIdx.x;      // subtree within the view
    const u64 j = a.jbase + jl;     // global index at level lam0
    const LevelGeom g0 = make_geom(a.n, a.lam0);
    const int m = (int)(a.from_pts ? a.n : seg_size(g0, j));
    // the subtree's points: the whole input for a single-CTA build, else its
    // in-order range of the global levels' working set (contiguous, so the
    // load is coalesced -- no gather)
    const u32* src = nullptr;
    const u32* vin = nullptr;
    if (!a.from_pts) {
        u32 par = 0;
        if (a.src_par >= 0) {
            par = (u32)a.src_par;
        } else if (a.lam0 != a.lfirst) {
            const uint8_t st = a.prev_state[jl >> 1];
            par = ((st >> 4) ^ (u32)__popc(st & 15u)) & 1u;
        }
        src = a.w[par] + (seg_ibegin(g0, j) - a.pbase);
        vin = src + (u64)k * a.stride;
    }
    for (int lid = tid; lid < m; lid += kSubThreads) {
        if (src) {
            for (int c = 0; c < k; ++c) P[c * M + lid] = __uint_as_float(src[(u64)c * a.stride + lid]);
        } else {
            const float* q = a.pts + (u64)lid * k;
            for (int c = 0; c < k; ++c) P[c * M + lid] = q[c];
        }
        E[0][lid] = (u32)lid;
    }
    if (a.mode == kWidest) {
        if (tid < 2 * k) rootbox[tid] = a.boxes0[jl * 2ull * k + tid];
        if (tid == 0) ndim[0] = a.split_dims[g0.Fl + j];
    }
    __syncthreads();

    auto write_node = [&](u64 node, u32 lid) {
        a.perm[node] = vin ? vin[lid] : lid;
        float* dst = a.out_pts + node * (u64)k;
        for (int c = 0; c < k; ++c) dst[c] = P[c * M + lid];
    };

    int cur = 0;
    if (!a.entry_sorted && !a.from_pts && a.lam0 > 0) {
        // input order -> the reference's order inside the subtree's parent
        // (no static shared memory here: it would misalign the dynamic
        // region, so every thread derives the chain itself)
        Chain ch;
        if (a.mode == kRoundRobin) rr_chain(a.lam0 - 1, k, ch);
        else widest_chain(make_geom(a.n, a.lam0 - 1).Fl + (j >> 1), k, a.split_dims, ch);
        cur = entry_order<kSubThreads>(E[0], E[1], m, P, M, ch, cnt, gsum, scratch);
    }
    for (int lam = a.lam0; lam <= a.L - 2; ++lam) {
        const LevelGeom g = make_geom(a.n, lam);
        const int dl = lam - a.lam0;
        const u64 nloc = 1ull << dl;
        const u64 J0 = j << dl;
        const u64 lb0 = seg_begin(g, J0);
        const int mc = m - (int)(nloc - 1);
        const int dim_rr = lam % k;
        const u32 nb = (u32)(nloc - 1);  // local node index of segment 0

        auto key_of = [&](u32 e) -> u32 {
            u32 lid = e & 0xffffu;
            int d = (a.mode == kWidest) ? (int)ndim[nb + (e >> 16)] : dim_rr;
            return flip_key(P[d * M + lid]);
        };

        // digits constant over the whole subtree are skipped
        u32 x_and = 0xffffffffu, x_or = 0u;
        for (int p = tid; p < mc; p += kSubThreads) {
            u32 kk = key_of(E[cur][p]);
            x_and &= kk;
            x_or |= kk;
        }
        x_and = __reduce_and_sync(kFullMask, x_and);
        x_or = __reduce_or_sync(kFullMask, x_or);
        scratch[32 + (tid >> 5)] = x_and ^ x_or;  // all lanes: same value
        __syncthreads();
        u32 vary = 0;
        for (int w = 0; w < kSubWarps; ++w) vary |= scratch[32 + w];
        __syncthreads();

        bool moved = false;
        for (int q = 0; q < 4; ++q) {
            if (((vary >> (8 * q)) & 255u) == 0) continue;
            const int sh = 8 * q;
            block_pass<kSubThreads>(E[cur], E[cur ^ 1], mc, [&](u32 e) { return (key_of(e) >> sh) & 255u; }, cnt, gsum,
                       scratch);
            cur ^= 1;
            moved = true;
        }
        if (moved && dl > 0) {
            for (int q = 0; q * 8 < dl; ++q) {
                const int sh = 16 + 8 * q;
                block_pass<kSubThreads>(E[cur], E[cur ^ 1], mc, [&](u32 e) { return (e >> sh) & 255u; }, cnt, gsum, scratch);
                cur ^= 1;
            }
        }
        if (a.dbg) {
            for (int p = tid; p < mc; p += kSubThreads) a.dbg[(u64)lam * a.n + lb0 + p] = E[cur][p] & 0xffffu;
        }

        // split: pivots become nodes, the rest move into the child segments
        const bool last = (lam == a.L - 2);
        const LevelGeom gn = make_geom(a.n, lam + 1);
        for (int p = tid; p < mc; p += kSubThreads) {
            u32 e = E[cur][p];
            u32 t = e >> 16, lid = e & 0xffffu;
            u64 J = J0 + t;
            u64 o = lb0 + (u64)p - seg_begin(g, J);
            u64 po = pivot_off(g, J);
            if (o == po) {
                write_node(g.Fl + J, lid);
                if (a.mode == kWidest) nplane[nb + t] = P[(int)ndim[nb + t] * M + lid];
                continue;
            }
            u32 right = o > po ? 1u : 0u;
            if (last) {
                write_node(gn.Fl + 2 * J + right, lid);
                continue;
            }
            E[cur ^ 1][p - (int)t - (int)right] = ((2u * t + right) << 16) | lid;
        }
        cur ^= 1;
        __syncthreads();

        if (a.mode == kWidest) {
            // split dims of the children (level lam+1 nodes of this subtree)
            const u32 nch = (u32)(2 * nloc);
            const u32 cb = (u32)(2 * nloc - 1);  // local index of the first child
            for (u32 c = tid; c < nch; c += kSubThreads) {
                u64 gnode = gn.Fl + 2 * J0 + c;
                if (gnode >= a.n) continue;
                float lo[kMaxK], hi[kMaxK];
                for (int d = 0; d < k; ++d) { lo[d] = rootbox[d]; hi[d] = rootbox[k + d]; }
                u32 u = cb + c;
                while (u > 0) {
                    u32 par = (u - 1) >> 1;
                    int dp = ndim[par];
                    float pl = nplane[par];
                    if (u & 1u) { if (pl < hi[dp]) hi[dp] = pl; }
                    else { if (pl > lo[dp]) lo[dp] = pl; }
                    u = par;
                }
                int best = 0;
                double bw = coord_width(a.wt, 0, lo[0], hi[0]);
                for (int d = 1; d < k; ++d) {
                    double w = coord_width(a.wt, d, lo[d], hi[d]);
                    if (w > bw) { bw = w; best = d; }
                }
                ndim[cb + c] = (unsigned char)best;
                a.split_dims[gnode] = (uint8_t)best;
            }
            __syncthreads();
        }
    }
    if (a.lam0 > a.L - 2) {
        // the subtree root is a bottom-level node (only when L - 1 == lam0)
        if (tid == 0 && m == 1) write_node(g0.Fl + j, 0u);
    }
}

// ===========================================================================
// Round-robin fast path: presorted lists instead of per-level sorts.
//
// Within a subtree entered at level lam0 >= k, the order the reference's
// stable sorts leave inside every node at level l is a FIXED total order
//     T_d = (c[d], c[d-1], ..., c[d-k+1], input index),  d = l mod k
// (each level's stable sort by c[d] starts from the previous level's
// order, and after k levels all coordinates are in the chain; further
// repeats of a coordinate never decide a comparison).  The entry order is
// T_{(lam0-1) mod k}; T_d = stable_sort(T_{d-1}, c[d]), so k-1 block radix
// sorts give all k orders as lists of local ids.
//
// Block phase (segments > 31 points), per level:
//   (1) the active list T_{l mod k}: the element at each segment's pivot
//       offset (kernels_numba.py:21-46) is the node; every element records
//       (child segment, side) in one packed state word; the list itself
//       splits without a scan (left part precedes the pivot);
//   (2) every other list still needed later is split stably into the child
//       segments -- up to two lists share ONE block scan of packed
//       (right, pivot) counts; destinations come from per-segment tables
//       (right elements of the earlier segments: one scan per level).
// Warp phase (segments <= 31 points, the last <= 5 levels): the position of
// every point in each list is its rank under T_d; one warp per segment
// finishes the segment's subtree in registers -- each level a point's rank
// inside its node is a count over the warp's lanes -- without barriers.
// ===========================================================================
constexpr int kWarpSegBits = 5;  // warp phase once segments hold <= 2^5 - 1 points

size_t subtree_rr_smem_bytes(int b, int k) {
    size_t M = ((size_t)1 << b) - 1;
    size_t Mp = (M + 8) & ~(size_t)7;  // 16-byte aligned u16 arrays
    size_t bytes = sizeof(float) * (size_t)k * Mp;   // P
    bytes += sizeof(unsigned short) * Mp * (k + 2);   // k lists + two partition targets
    bytes += sizeof(unsigned short) * Mp;             // packed state of each point
    size_t nloc = ((size_t)1 << (b - 2));             // segments at the deepest block level
    // level tables + node table (after the chain sorts) alias the sort scratch
    size_t tables = sizeof(u32) * 2 * (nloc + 8) + sizeof(unsigned short) * Mp;
    size_t sortscr = sizeof(unsigned short) * kRRWarps * 256 + sizeof(u32) * 4 * 256;
    bytes += tables > sortscr ? tables : sortscr;
    bytes += sizeof(u64) * 64;
    return (bytes + 15) & ~(size_t)15;
}

// KT, MPT: compile-time k and padded capacity for the common shapes (all
// shared-memory offsets become immediates); 0 = taken from the arguments
template <int KT, int MPT>
__global__ void __launch_bounds__(kRRThreads, 2) subtree_rr_kernel(SubtreeArgs a) {
    if (a.abort_word && *a.abort_word) return;  // non-finite input (select.cu aborted)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    typedef unsigned short u16;
    const int M = MPT ? MPT - 1 : a.M, k = KT ? KT : a.k, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int Mp = MPT ? MPT : (M + 8) & ~7;
    unsigned char* sp = smem_raw;
    float* P = reinterpret_cast<float*>(sp);
    sp += sizeof(float) * (size_t)k * Mp;
    // the k + 2 lists as offsets from one shared base: pointers kept in a
    // local array would lose their address space (generic LD/ST)
    u16* const LB = reinterpret_cast<u16*>(sp);
    int Lo[kMaxK + 2];
    for (int d = 0; d <= k + 1; ++d) Lo[d] = d * Mp;
    sp += sizeof(u16) * Mp * (k + 2);
    u16* state = reinterpret_cast<u16*>(sp);  // (next-level segment << 2) | side (0 L, 1 R, 2 node)
    sp += sizeof(u16) * Mp;
    sp = smem_raw + (((size_t)(sp - smem_raw) + 15) & ~(size_t)15);  // keep the shared base (no uintptr_t round trip)
    // per-level tables alias the radix-sort scratch (chain sorts)
    const int nmax = (M + 1) / 4;  // 2^(b-2) segments at the deepest block level
    // per segment t: lp[t] = begin in the lists | pivot offset << 16;
    //               rp[t] = right elements of the earlier segments | begin of
    //               its right child in the next lists minus those << 16
    u32* lp = reinterpret_cast<u32*>(sp);
    u32* rp = lp + nmax + 8;
    u16* ntab = reinterpret_cast<u16*>(rp + nmax + 8);  // local id of the point of every node, heap order
    unsigned short(*cnt)[256] = reinterpret_cast<unsigned short(*)[256]>(sp);
    u32(*gsum)[256] = reinterpret_cast<u32(*)[256]>(sp + sizeof(unsigned short) * kRRWarps * 256);
    size_t tables = sizeof(u32) * 2 * ((size_t)nmax + 8) + sizeof(u16) * Mp;
    size_t sortscr = sizeof(unsigned short) * kRRWarps * 256 + sizeof(u32) * 4 * 256;
    u32* scratch = reinterpret_cast<u32*>(sp + (tables > sortscr ? tables : sortscr));
    u64* scratch64 = reinterpret_cast<u64*>(scratch);

    const u64 jl = blockIdx.x;      // subtree within the view
    const u64 j = a.jbase + jl;     // global index at level lam0
    const LevelGeom g0 = make_geom(a.n, a.lam0);
    const int m = (int)seg_size(g0, j);
    u32 par = 0;
    if (a.src_par >= 0) {
        par = (u32)a.src_par;
    } else if (a.lam0 != a.lfirst) {
        const uint8_t st = a.prev_state[jl >> 1];
        par = ((st >> 4) ^ (u32)__popc(st & 15u)) & 1u;
    }
    const u32* src = a.w[par] + (seg_ibegin(g0, j) - a.pbase);
    const u32* vin = src + (u64)k * a.stride;
    const int e = (a.lam0 - 1) % k;  // dimension of the entry order
    u16* ident = LB + (a.entry_sorted ? Lo[e] : Lo[0]);
    for (int lid = tid; lid < m; lid += kRRThreads) {
        for (int c = 0; c < k; ++c) P[c * Mp + lid] = __uint_as_float(src[(u64)c * a.stride + lid]);
        ident[lid] = (u16)lid;
        state[lid] = 0;
    }
    __syncthreads();
    // the k chain orders by one bucket pass each (tie-heavy subtrees fall
    // back to the radix passes below)
    bool listed = a.bucket_lists && (Mp % (4 * kRRThreads)) == 0;
    if (listed) {
        u32* hist = reinterpret_cast<u32*>(sp);  // the tables / sort-scratch region holds >= 4 Mp bytes
        for (int d = 0; d < k && listed; ++d) {
            if (a.entry_sorted && d == e) continue;
            listed = bucket_list<kRRThreads, KT>(LB + Lo[d], m, P, Mp, d, k, Mp, hist, scratch);
        }
        if (!listed) {
            for (int lid = tid; lid < m; lid += kRRThreads) ident[lid] = (u16)lid;
            __syncthreads();
        }
    }
    if (!listed && !a.entry_sorted) {
        // input order -> T_e (full chain: lam0 >= k), then hand the other
        // buffers out as the remaining lists and the spares
        Chain ch;
        rr_chain(a.lam0 - 1, k, ch);
        const int r = entry_order<kRRThreads>(LB + Lo[0], LB + Lo[1], m, P, Mp, ch, cnt, gsum, scratch);
        const int res = r * Mp;  // list buffers are still in order here
        int q = 0;
        for (int d = 0; d <= k + 1; ++d) {
            if (d == e) { Lo[d] = res; continue; }
            if (q * Mp == res) ++q;
            Lo[d] = (q++) * Mp;
        }
    }

    // ---- chain sorts: T_d = stable_sort(T_{d-1}, c[d]) for the k-1 other dims
    for (int q = 1; q < k && !listed; ++q) {
        const int d = (e + q) % k;
        const int dprev = (e + q - 1) % k;
        const float* Pd = P + d * Mp;
        u32 x_and = 0xffffffffu, x_or = 0u;
        for (int p = tid; p < m; p += kRRThreads) {
            u32 kk = flip_key(Pd[p]);
            x_and &= kk;
            x_or |= kk;
        }
        x_and = __reduce_and_sync(kFullMask, x_and);
        x_or = __reduce_or_sync(kFullMask, x_or);
        scratch[32 + (tid >> 5)] = x_and ^ x_or;  // every lane stores the warp-uniform value (NVVM 12.9, above)
        __syncthreads();
        u32 vary = 0;
        for (int w = 0; w < kRRWarps; ++w) vary |= scratch[32 + w];
        __syncthreads();
        const u16* in = LB + Lo[dprev];
        u16* outA = LB + Lo[d];
        u16* outB = LB + Lo[k];  // spare
        int npass = 0;
        for (int b = 0; b < 4; ++b) {
            if (((vary >> (8 * b)) & 255u) == 0) continue;
            u16* out = (npass & 1) ? outB : outA;
            const int sh = 8 * b;
            block_pass<kRRThreads>(in, out, m, [&](u32 lid) { return (flip_key(Pd[lid]) >> sh) & 255u; }, cnt, gsum, scratch);
            in = out;
            ++npass;
        }
        if (npass == 0) {
            for (int p = tid; p < m; p += kRRThreads) outA[p] = in[p];
            __syncthreads();
        } else if (npass & 1) {
            // result in outA == Lst[d]
        } else {
            // result in the spare list: swap roles
            const int t = Lo[k];
            Lo[k] = Lo[d];
            Lo[d] = t;
        }
    }

    // geometry without per-level bit_length loops: B = bottom slots in use
    const int L = a.L;
    const u64 Bn = a.n - ((1ull << (L - 1)) - 1ull);
    auto seg_size_l = [&](int sh, u64 J) -> u32 {
        const u64 w = 1ull << sh, lo = J << sh;
        u64 on = Bn > lo ? Bn - lo : 0ull;
        if (on > w) on = w;
        return (u32)(w - 1ull + on);
    };
    auto seg_begin_l = [&](int sh, u64 J) -> u64 {
        const u64 lo = J << sh;
        return J * ((1ull << sh) - 1ull) + (lo < Bn ? lo : Bn);
    };
    auto pivot_off_l = [&](int sh, u64 J) -> u32 {
        if (sh <= 0) return 0u;
        const u64 cw = 1ull << (sh - 1), lo = (2ull * J) * cw;
        u64 on = Bn > lo ? Bn - lo : 0ull;
        if (on > cw) on = cw;
        return (u32)(cw - 1ull + on);
    };

    int lam = a.lam0;
    // ================= block phase =================
    for (; lam <= L - 2 && (L - lam - 1) > kWarpSegBits - 1; ++lam) {
        const int sh = L - lam - 1;
        const int dl = lam - a.lam0;
        const int nloc = 1 << dl;
        const u64 J0 = j << dl;
        const u64 lb0 = seg_begin_l(sh, J0);
        const int mc = m - (nloc - 1);
        const int ad = lam % k;
        const u64 Fl = (1ull << lam) - 1ull;
        const bool last = (lam == L - 2);
        // tables + right elements of the earlier segments (one scan)
        {
            u32 v = 0;
            const int per = (nloc + kRRThreads - 1) / kRRThreads;  // <= 2
            u32 rs[2] = {0u, 0u}, lb2[2] = {0u, 0u}, po2[2] = {0u, 0u};
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int t = tid * per + i;
                if (i < per && t < nloc) {
                    const u32 sz = seg_size_l(sh, J0 + t);
                    po2[i] = pivot_off_l(sh, J0 + t);
                    lb2[i] = (u32)(seg_begin_l(sh, J0 + t) - lb0);
                    lp[t] = lb2[i] | (po2[i] << 16);
                    rs[i] = sz - po2[i] - 1u;
                    v += rs[i];
                }
            }
            u32 ex;
            if (nloc <= 32) {  // every segment is in warp 0: a warp scan, no block barriers
                if (warp == 0) {
                    u32 x = v;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const u32 y = __shfl_up_sync(kFullMask, x, o);
                        if (lane >= o) x += y;
                    }
                    ex = x - v;
                } else {
                    ex = 0u;  // (no segments on the other warps)
                }
            } else {
                ex = block_exclusive_scan_1b<u32>(v, scratch);
            }
            u32 run = ex;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int t = tid * per + i;
                if (i < per && t < nloc) {
                    rp[t] = run | ((lb2[i] - (u32)t + po2[i] - run) << 16);
                    run += rs[i];
                }
            }
        }
        __syncthreads();

        // (1) the active list: nodes, sides, child segments; its own split
        u16* A = LB + Lo[ad];
        u16* tmpA = LB + Lo[k];
        for (int p = tid; p < mc; p += kRRThreads) {
            const u32 lid = A[p];
            const u32 t = state[lid] >> 2;
            const u32 lpt = lp[t];
            const u32 lb = lpt & 0xffffu;
            const u32 o = (u32)p - lb;
            const u32 po = lpt >> 16;
            if (o == po) {
                state[lid] = (u16)(((2u * t) << 2) | 2u);
                ntab[nloc - 1 + t] = (u16)lid;
                continue;
            }
            const u32 r = o > po ? 1u : 0u;
            state[lid] = (u16)(((2u * t + r) << 2) | r);
            if (last) ntab[2 * nloc - 1 + 2 * t + r] = (u16)lid;
            else tmpA[lb - t + o - r] = (u16)lid;
        }
        __syncthreads();
        if (last) {  // (only for tiny subtrees) the bottom level is written too
            lam = L;
            break;
        }
        {
            const int t = Lo[k];
            Lo[k] = Lo[ad];
            Lo[ad] = t;
        }

        // (2) the passive lists still needed later, two per block scan
        int todo[kMaxK];
        int nt = 0;
        for (int d = 0; d < k; ++d) {
            if (d == ad) continue;
            const int next_use = lam + ((d - ad + k) % k);
            if (next_use <= L - 2) todo[nt++] = d;
        }
        for (int i0 = 0; i0 < nt; i0 += 2) {
            const int dA = todo[i0];
            const int dB = i0 + 1 < nt ? todo[i0 + 1] : -1;
            const u16* XA = LB + Lo[dA];
            const bool hasB = dB >= 0;
            const u16* XB = LB + (hasB ? Lo[dB] : Lo[dA]);
            u16* YA = LB + Lo[k];
            u16* YB = LB + Lo[k + 1];
            // 8 consecutive positions per thread, one 16-byte load per list;
            // per list the counts (right | pivot << 16) of the thread's
            // positions, both lists scanned in one 64-bit block scan
            const int p0 = tid * 8;
            u32 la[8], lb8[8], sa[8], sb[8];
            u32 va = 0, vb = 0;
            if (p0 < mc) {
                const uint4 qa = *reinterpret_cast<const uint4*>(XA + p0);
                const u32 wa[4] = {qa.x, qa.y, qa.z, qa.w};
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    la[i] = (wa[i >> 1] >> (16 * (i & 1))) & 0xffffu;
                    sa[i] = p0 + i < mc ? (u32)state[la[i]] : 3u;
                }
                if (hasB) {
                    const uint4 qb = *reinterpret_cast<const uint4*>(XB + p0);
                    const u32 wb[4] = {qb.x, qb.y, qb.z, qb.w};
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        lb8[i] = (wb[i >> 1] >> (16 * (i & 1))) & 0xffffu;
                        sb[i] = p0 + i < mc ? (u32)state[lb8[i]] : 3u;
                    }
                }
                // state & 3: 0 left, 1 right, 2 node, 3 past the end
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const u32 ca = sa[i] & 3u;
                    va += ca == 1u ? 1u : (ca == 2u ? 0x10000u : 0u);
                    if (hasB) {
                        const u32 cb = sb[i] & 3u;
                        vb += cb == 1u ? 1u : (cb == 2u ? 0x10000u : 0u);
                    }
                }
            }
            const u64 ex64 = block_exclusive_scan_1b<u64>((u64)va | ((u64)vb << 32), scratch64);
            if (p0 < mc) {
                u32 exa = (u32)ex64, exb = (u32)(ex64 >> 32);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int p = p0 + i;
                    const u32 ca = sa[i] & 3u;
                    if (ca < 2u) {
                        const u32 rpt = rp[sa[i] >> 3];
                        const u32 Rex = exa & 0xffffu, Pex = exa >> 16;
                        const u32 dst = ca ? (rpt >> 16) + Rex : (u32)p - Rex - Pex + (rpt & 0xffffu);
                        YA[dst] = (u16)la[i];
                    }
                    exa += ca == 1u ? 1u : (ca == 2u ? 0x10000u : 0u);
                    if (hasB) {
                        const u32 cb = sb[i] & 3u;
                        if (cb < 2u) {
                            const u32 rpt = rp[sb[i] >> 3];
                            const u32 Rex = exb & 0xffffu, Pex = exb >> 16;
                            const u32 dst = cb ? (rpt >> 16) + Rex : (u32)p - Rex - Pex + (rpt & 0xffffu);
                            YB[dst] = (u16)lb8[i];
                        }
                        exb += cb == 1u ? 1u : (cb == 2u ? 0x10000u : 0u);
                    }
                }
            }
            __syncthreads();
            {
                const int t = Lo[k];
                Lo[k] = Lo[dA];
                Lo[dA] = t;
            }
            if (hasB) {
                const int t = Lo[k + 1];
                Lo[k + 1] = Lo[dB];
                Lo[dB] = t;
            }
        }
    }

    // ================= warp phase =================
    if (lam <= L - 1) {
        const int dl = lam - a.lam0;
        const int nloc = 1 << dl;
        const u64 J0 = j << dl;
        const int sh = L - lam - 1;
        const u64 lb0 = seg_begin_l(sh, J0);
        // rank of every point in each list that is used again = its rank
        // under T_d inside its segment; the spare buffers receive them
        int rko[kMaxK];
        int freeb[kMaxK + 2];
        int nfree = 0;
        freeb[nfree++] = Lo[k];
        freeb[nfree++] = Lo[k + 1];
        const int memo = Lo[lam % k];
        const u16* member = LB + memo;
        for (int d = 0; d < k; ++d) {
            rko[d] = -1;
            const int first_use = lam + ((d - lam % k + k) % k);
            if (first_use > L - 2) continue;
            const int dsto = freeb[--nfree];
            u16* dst = LB + dsto;
            const u16* X = LB + Lo[d];
            for (int p = tid; p < m - (nloc - 1); p += kRRThreads) dst[X[p]] = (u16)p;
            rko[d] = dsto;
            if (Lo[d] != memo) freeb[nfree++] = Lo[d];
            __syncthreads();
        }
        for (int t = warp; t < nloc; t += kRRWarps) {
            const u64 Jt = J0 + t;
            const u32 sb = (u32)(seg_begin_l(sh, Jt) - lb0);
            const u32 sz = seg_size_l(sh, Jt);
            bool act = (u32)lane < sz;
            const u32 lid = act ? member[sb + lane] : 0u;
            u32 nd = 0;  // heap index of the point's node inside segment t's subtree (< 31)
            // lanes of my node (every active lane of a node holds the same
            // mask): the segment's lanes, then per level narrowed to my side
            u32 eq = __ballot_sync(kFullMask, act);
            for (int l2 = lam; l2 <= L - 1; ++l2) {
                const int dd = l2 - lam;
                const int sh2 = L - l2 - 1;
                // local rank under T_d inside the segment (< 31): the segment
                // begins at sb in every list
                const u32 key = (act && l2 <= L - 2) ? (u32)LB[rko[l2 % k] + lid] - sb : 0u;
                // the keys (segment-local ranks < 31) present in my node as
                // a bit set: one segmented OR over the node's lanes (measured
                // faster than a bit-serial compare over warp-wide ballots)
                u32 rank = 0;
                if (act) {
                    const u32 keys = __reduce_or_sync(eq, 1u << key);
                    rank = (u32)__popc(keys & ((1u << key) - 1u));
                }
                bool right = false;
                if (act) {
                    const u32 off = nd + 1u - (1u << dd);  // node's index among depth dd
                    const u64 J = (Jt << dd) + off;
                    // 32-bit: J << sh2 <= 2^(L-1) and B < 2^31 for n < 2^31
                    u32 po = 0;
                    if (sh2 > 0) {
                        const u32 cw = 1u << (sh2 - 1), lo = (u32)J << sh2;
                        u32 on = (u32)Bn > lo ? (u32)Bn - lo : 0u;
                        po = cw - 1u + (on < cw ? on : cw);
                    }
                    if (rank == po) {
                        ntab[(1u << (dl + dd)) - 1u + ((u32)t << dd) + off] = (u16)lid;
                        act = false;
                    } else {
                        right = rank > po;
                        nd = 2u * nd + 1u + (right ? 1u : 0u);
                    }
                }
                const u32 live = __ballot_sync(kFullMask, act);
                if (!live) break;
                const u32 rb = __ballot_sync(kFullMask, right);
                eq &= live & (right ? rb : ~rb);
            }
        }
    }

    // ================= output =================
    // each level's nodes of this subtree are one contiguous range of the
    // level-order arrays: coalesced stores of points and input rows
    __syncthreads();
    // the input rows, staged once (coalesced) in the dead list buffers
    u32* const vs = reinterpret_cast<u32*>(LB);
    for (int lid = tid; lid < m; lid += kRRThreads) vs[lid] = vin[lid];
    __syncthreads();
    for (int dl = 0; a.lam0 + dl <= L - 1; ++dl) {
        const int l2 = a.lam0 + dl;
        const u64 first = ((1ull << l2) - 1ull) + (j << dl);
        if (first >= a.n) break;
        u64 cntn = 1ull << dl;
        if (first + cntn > a.n) cntn = a.n - first;
        const u32 h0 = (1u << dl) - 1u;
        for (u32 i = tid; i < (u32)cntn; i += kRRThreads) a.perm[first + i] = vs[ntab[h0 + i]];
        float* dst = a.out_pts + first * (u64)k;
        for (u32 i = tid; i < (u32)cntn * (u32)k; i += kRRThreads) {
            const u32 t = i / (u32)k, c = i - t * (u32)k;
            dst[i] = P[c * Mp + ntab[h0 + t]];
        }
    }
}

void launch_subtree(const BuildParams& bp, const Buffers& bf, int lam0, int entry_sorted, int src_par,
                    cudaStream_t st) {
    SubtreeArgs a;
    a.n = bp.n;
    a.L = bit_length(bp.n);
    a.lam0 = lam0;
    a.k = bp.k;
    a.mode = bp.mode;
    a.wt = bp.wt;
    a.M = (1 << bp.b) - 1;
    a.w[0] = bf.w[0];
    a.w[1] = bf.w[1];
    a.stride = bf.stride;
    a.prev_state = bf.state[(lam0 + 1) & 1];
    a.pts = bp.pts;
    a.out_pts = bp.out_pts;
    a.perm = bp.perm;
    a.split_dims = bp.split_dims;
    a.boxes0 = bf.boxes[lam0 & 1];
    a.dbg = bp.dbg;
    a.abort_word = bf.err ? bf.err + 1 : nullptr;
    a.jbase = bp.jroot << (lam0 - bp.lroot);
    a.pbase = seg_ibegin(make_geom(bp.n, bp.lroot), bp.jroot);
    a.lfirst = bp.lroot;
    a.from_pts = lam0 == 0 ? 1 : 0;
    a.entry_sorted = entry_sorted;
    a.src_par = src_par;
    {
        const char* e = getenv("LBKD_BUCKET");
        a.bucket_lists = !(e && e[0] == '0');
    }
    unsigned grid = (unsigned)(1ull << (lam0 - bp.lroot));
    const bool sel_ok = !bp.dbg && (bp.mode == kRoundRobin || bp.k <= 4);
    if (sel_ok && (bp.subtree_sel || (bp.mode == kRoundRobin && lam0 < bp.k))) {
        // per-level selection in shared memory (subtree_sel.cu): any entry order
        launch_subtree_sel(a, grid, bp.b, st);
        return;
    }
    if (bp.mode == kRoundRobin && lam0 >= bp.k) {
        size_t sm = subtree_rr_smem_bytes(bp.b, bp.k);
        const int Mp = (a.M + 8) & ~7;
        auto go = [&](auto kern) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            kern<<<grid, kRRThreads, sm, st>>>(a);
        };
        if (bp.k == 3 && Mp == 4096) go(subtree_rr_kernel<3, 4096>);
        else if (bp.k == 2 && Mp == 4096) go(subtree_rr_kernel<2, 4096>);
        else if (bp.k == 4 && Mp == 2048) go(subtree_rr_kernel<4, 2048>);
        else go(subtree_rr_kernel<0, 0>);
        return;
    }
    size_t sm = subtree_smem_bytes(bp.b, bp.k, bp.mode);
    cudaFuncSetAttribute(subtree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    subtree_kernel<<<grid, kSubThreads, sm, st>>>(a);
}

}  // namespace lbkd
