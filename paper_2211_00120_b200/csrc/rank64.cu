// rank64.cu -- float64 input (the reference's own dtype, builder.py:131-133).
//
// The build only ever COMPARES coordinates (less(), builder.py:158-162; the
// stable lexsort), except for the widest variant's float64 widths
// (widest.py:91-93).  So a float64 build is the float32 build of the points'
// per-dimension dense ranks: replace x[i][d] by the rank of its value among
// the distinct values of dimension d (-0.0 == +0.0, numpy's ordering), code
// the rank as a strictly increasing float32 (rank_code, common.cuh), build,
// and gather the float64 rows by the resulting permutation.  The widths come
// from a per-dimension table of the distinct values (WidthTab).
//
// Ranks come from a hand-written LSD radix sort of (order-flipped float64
// bits, row) pairs, 8-bit digits:
//   rs_keys      key = flip64(canon(x)), row index; non-finite flag
//   per pass:  rs_hist (per 2048-item tile digit counts, digit-major)
//              scan_u32 (exclusive scan -> every (digit, tile) output offset)
//              rs_skip  (a digit holding every key: the pass is skipped)
//              rs_scatter (stable: warp-ordered ranks from bit-sliced
//                          ballots, per-warp digit bases in shared memory)
//              rs_flip  (ping-pong parity kept on the device)
//   rs_flags     flag[i] = key[i] != key[i-1];  scan_u32 -> ranks, count
//   rs_assign    codes[row][d] = rank_code(rank), table[d][rank] = value
// A pass moves 12 B per point each way; constant digits (e.g. the exponent
// bytes of data in [0, 1)) cost only their histogram.
#include "kernels.cuh"

namespace lbkd {

namespace {

constexpr int kRsThreads = 256;
constexpr int kRsTile = 2048;  // 8 warps x 8 rounds x 32 lanes
constexpr int kScanItems = 8;
constexpr int kScanTile = kRsThreads * kScanItems;

__device__ __forceinline__ u64 flip64(double x) {
    u64 u = (u64)__double_as_longlong(x);
    if (u == 0x8000000000000000ull) u = 0ull;  // -0.0 == +0.0
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ double unflip64(u64 k) {
    const u64 u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)u);
}

__global__ void rs_keys(const double* __restrict__ pts, u64 n, int k, int d, u64* key, u32* val, u32* err) {
    bool bad = false;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const double x = __ldg(pts + i * k + d);
        bad |= !isfinite(x);
        key[i] = flip64(x);
        val[i] = (u32)i;
    }
    if (__any_sync(kFullMask, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

__global__ void __launch_bounds__(kRsThreads) rs_hist(const u64* key0, const u64* key1, const u32* par, u64 n,
                                                     u64 ntiles, int shift, u32* hist) {
    __shared__ u32 h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const u64* key = *par ? key1 : key0;
    const u64 base = blockIdx.x * (u64)kRsTile;
    for (int i = threadIdx.x; i < kRsTile; i += kRsThreads) {
        const u64 p = base + i;
        if (p < n) atomicAdd(&h[(u32)(key[p] >> shift) & 255u], 1u);
    }
    __syncthreads();
    hist[(u64)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// a digit that holds every key leaves the order unchanged: skip the pass
__global__ void rs_skip(const u32* offs, u64 ntiles, u64 n, u32* skip) {
    const u32 d = threadIdx.x;
    const u64 lo = offs[(u64)d * ntiles];
    const u64 hi = d == 255 ? n : offs[(u64)(d + 1) * ntiles];
    const bool all = hi - lo == n;
    const bool any = __syncthreads_or(all);
    if (d == 0) *skip = any ? 1u : 0u;
}

__global__ void __launch_bounds__(kRsThreads) rs_scatter(u64* key0, u64* key1, u32* val0, u32* val1,
                                                        const u32* par, const u32* skip, u64 n, u64 ntiles,
                                                        int shift, const u32* offs) {
    if (*skip) return;
    const u32 p = *par;
    const u64* kin = p ? key1 : key0;
    const u32* vin = p ? val1 : val0;
    u64* kout = p ? key0 : key1;
    u32* vout = p ? val0 : val1;
    __shared__ u32 cnt[8][256];
    __shared__ u32 tbase[256];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 8 * 256; i += kRsThreads) (&cnt[0][0])[i] = 0;
    tbase[threadIdx.x] = offs[(u64)threadIdx.x * ntiles + blockIdx.x];
    __syncthreads();
    const u64 base = blockIdx.x * (u64)kRsTile + (u64)w * 256;
    u64 kk[8];
    u32 vv[8];
    u32 dg[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const u64 i = base + r * 32 + lane;
        const bool ok = i < n;
        kk[r] = ok ? kin[i] : 0ull;
        vv[r] = ok ? vin[i] : 0u;
        dg[r] = (u32)(kk[r] >> shift) & 255u;
        const u32 peers = warp_peers<8>(dg[r], ok);
        // the highest lane of each digit group counts it
        if (ok && (peers >> lane) == 1u) cnt[w][dg[r]] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {  // per digit: exclusive base of each warp (warp order = item order)
        const int d = threadIdx.x;
        u32 run = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const u32 c = cnt[q][d];
            cnt[q][d] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const u64 i = base + r * 32 + lane;
        const bool ok = i < n;
        const u32 peers = warp_peers<8>(dg[r], ok);
        if (ok) {
            const u32 pos = tbase[dg[r]] + cnt[w][dg[r]] + __popc(peers & lanemask_lt());
            kout[pos] = kk[r];
            vout[pos] = vv[r];
        }
        __syncwarp();
        if (ok && (peers >> lane) == 1u) cnt[w][dg[r]] += __popc(peers);
        __syncwarp();
    }
}

__global__ void rs_flip(u32* par, const u32* skip) {
    if (!*skip) *par ^= 1u;
}

// ---- exclusive scan of u32 (reduce, scan of the partials, scan) -----------
__global__ void __launch_bounds__(kRsThreads) scan_reduce(const u32* in, u64 m, u32* part) {
    const u64 base = blockIdx.x * (u64)kScanTile;
    u32 s = 0;
    for (int i = threadIdx.x; i < kScanTile; i += kRsThreads) {
        const u64 p = base + i;
        if (p < m) s += in[p];
    }
    s = __reduce_add_sync(kFullMask, s);
    __shared__ u32 ws[8];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        u32 t = 0;
        for (int q = 0; q < 8; ++q) t += ws[q];
        part[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(1024) scan_partials(u32* part, u64 np, u32* total) {
    __shared__ u32 wt[32];
    __shared__ u32 tot;
    u32 carry = 0;
    for (u64 b = 0; b < np; b += 1024) {
        const u64 i = b + threadIdx.x;
        const u32 v = i < np ? part[i] : 0u;
        const u32 ex = block_exclusive_scan<u32>(v, wt, &tot);
        if (i < np) part[i] = carry + ex;
        __syncthreads();
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void __launch_bounds__(kRsThreads) scan_apply(const u32* in, u64 m, const u32* part, u32* out) {
    __shared__ u32 wt[32];
    const u64 base = blockIdx.x * (u64)kScanTile + (u64)threadIdx.x * kScanItems;
    u32 v[kScanItems];
    u32 s = 0;
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) {
        v[q] = base + q < m ? in[base + q] : 0u;
        s += v[q];
    }
    u32 run = block_exclusive_scan<u32>(s, wt, (u32*)nullptr) + part[blockIdx.x];
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) {
        if (base + q < m) out[base + q] = run;
        run += v[q];
    }
}

void scan_u32(const u32* in, u32* out, u64 m, u32* part, u32* total, cudaStream_t st) {
    const u64 nb = (m + kScanTile - 1) / kScanTile;
    scan_reduce<<<(unsigned)nb, kRsThreads, 0, st>>>(in, m, part);
    scan_partials<<<1, 1024, 0, st>>>(part, nb, total);
    scan_apply<<<(unsigned)nb, kRsThreads, 0, st>>>(in, m, part, out);
}

__global__ void rs_flags(const u64* key0, const u64* key1, const u32* par, u64 n, u32* flag) {
    const u64* key = *par ? key1 : key0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        flag[i] = (i > 0 && key[i] != key[i - 1]) ? 1u : 0u;
}

__global__ void rs_assign(const u64* key0, const u64* key1, const u32* val0, const u32* val1, const u32* par,
                          const u32* flag, const u32* excl, u64 n, int k, int d, u32 center, int wide, float* codes,
                          double* table) {
    const u32 p = *par;
    const u64* key = p ? key1 : key0;
    const u32* val = p ? val1 : val0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u32 f = flag[i];
        const u32 r = excl[i] + f;
        codes[(u64)val[i] * k + d] = rank_code(r, center, wide);
        if (table && (i == 0 || f)) table[r] = unflip64(key[i]);
    }
}

unsigned grid_for(u64 n, unsigned per_sm) {
    u64 b = (n + 255) / 256;
    if (b > 148ull * per_sm) b = 148ull * per_sm;
    return b < 1 ? 1u : (unsigned)b;
}

}  // namespace

size_t rank_scratch_words(u64 n) {
    // keys 2n u64, vals 2n, flags n, excl n, hist + offs 2 x 256 x tiles,
    // partials, par / skip / count words (in u32 units, 16-byte padded)
    const u64 ntiles = (n + kRsTile - 1) / kRsTile;
    const u64 m = 256 * ntiles;
    const u64 np = (m > n ? m : n) / kScanTile + 2;
    auto pad = [](u64 w) { return (w + 3) & ~3ull; };
    return pad(4 * n) + pad(2 * n) + pad(n) + pad(n) + pad(m) + pad(m) + pad(np) + 16;
}

// Sorts dimension d of the float64 AoS points and writes, on the device,
// the number of distinct values to *d_count.  Then rank_assign_dim writes
// the codes (after the caller chose the centre from that count).
int rank_sort_dim(const double* pts, u64 n, int k, int d, u32* scratch, u32* err, cudaStream_t st) {
    const u64 ntiles = (n + kRsTile - 1) / kRsTile;
    const u64 m = 256 * ntiles;
    auto pad = [](u64 w) { return (w + 3) & ~3ull; };
    u32* p = scratch;
    u64* key0 = (u64*)p;
    u64* key1 = key0 + n;
    p += pad(4 * n);
    u32* val0 = p;
    u32* val1 = p + n;
    p += pad(2 * n);
    u32* flag = p;
    p += pad(n);
    u32* excl = p;
    p += pad(n);
    u32* hist = p;
    p += pad(m);
    u32* offs = p;
    p += pad(m);
    u32* part = p;
    p += pad((m > n ? m : n) / kScanTile + 2);
    u32* par = p;
    u32* skip = p + 1;
    u32* count = p + 2;
    cudaMemsetAsync(par, 0, 4 * sizeof(u32), st);
    rs_keys<<<grid_for(n, 8), 256, 0, st>>>(pts, n, k, d, key0, val0, err);
    for (int pass = 0; pass < 8; ++pass) {
        const int shift = 8 * pass;
        rs_hist<<<(unsigned)ntiles, kRsThreads, 0, st>>>(key0, key1, par, n, ntiles, shift, hist);
        scan_u32(hist, offs, m, part, nullptr, st);
        rs_skip<<<1, 256, 0, st>>>(offs, ntiles, n, skip);
        rs_scatter<<<(unsigned)ntiles, kRsThreads, 0, st>>>(key0, key1, val0, val1, par, skip, n, ntiles, shift,
                                                            offs);
        rs_flip<<<1, 1, 0, st>>>(par, skip);
    }
    rs_flags<<<grid_for(n, 8), 256, 0, st>>>(key0, key1, par, n, flag);
    scan_u32(flag, excl, n, part, count, st);  // count = distinct values - 1
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : (note_cuda_error(e), 4);
}

int rank_assign_dim(u64 n, int k, int d, u32 center, int wide, float* codes, double* table, u32* scratch,
                    cudaStream_t st) {
    const u64 ntiles = (n + kRsTile - 1) / kRsTile;
    const u64 m = 256 * ntiles;
    auto pad = [](u64 w) { return (w + 3) & ~3ull; };
    u32* p = scratch;
    u64* key0 = (u64*)p;
    u64* key1 = key0 + n;
    p += pad(4 * n);
    u32* val0 = p;
    u32* val1 = p + n;
    p += pad(2 * n);
    u32* flag = p;
    p += pad(n);
    u32* excl = p;
    p += pad(n);
    p += pad(m) + pad(m) + pad((m > n ? m : n) / kScanTile + 2);
    u32* par = p;
    rs_assign<<<grid_for(n, 8), 256, 0, st>>>(key0, key1, val0, val1, par, flag, excl, n, k, d, center, wide, codes,
                                            table);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : (note_cuda_error(e), 4);
}

// the count word written by rank_sort_dim (distinct values - 1)
const u32* rank_count_word(const u32* scratch, u64 n) {
    const u64 ntiles = (n + kRsTile - 1) / kRsTile;
    const u64 m = 256 * ntiles;
    auto pad = [](u64 w) { return (w + 3) & ~3ull; };
    return scratch + pad(4 * n) + pad(2 * n) + pad(n) + pad(n) + pad(m) + pad(m) +
           pad((m > n ? m : n) / kScanTile + 2) + 2;
}

// out[s][c] = pts[perm[s]][c] (float64 rows in level order)
__global__ void gather_rows_f64(const double* __restrict__ pts, const u32* __restrict__ perm, u64 n, int k,
                                double* out) {
    for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < n * (u64)k; e += (u64)gridDim.x * blockDim.x) {
        const u64 s = e / (u64)k;
        const int c = (int)(e - s * k);
        out[e] = pts[(u64)perm[s] * k + c];
    }
}

void launch_gather_rows_f64(const double* pts, const u32* perm, u64 n, int k, double* out, cudaStream_t st) {
    gather_rows_f64<<<grid_for(n * (u64)k, 16), 256, 0, st>>>(pts, perm, n, k, out);
}

}  // namespace lbkd
