// Micro-benchmark: DRAM bytes moved by random 4-byte gathers under different
// load flavours and L2 fetch-granularity limits (run under ncu).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_plain(const float* __restrict__ src, const uint32_t* __restrict__ idx, float* out, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = src[idx[i]];
}
__global__ void k_cg(const float* __restrict__ src, const uint32_t* __restrict__ idx, float* out, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) { float v; asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(src + idx[i])); out[i] = v; }
}
__global__ void k_nc_na(const float* __restrict__ src, const uint32_t* __restrict__ idx, float* out, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) { float v; asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(src + idx[i])); out[i] = v; }
}
__global__ void k_cv(const float* __restrict__ src, const uint32_t* __restrict__ idx, float* out, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) { float v; asm volatile("ld.global.cv.f32 %0, [%1];" : "=f"(v) : "l"(src + idx[i])); out[i] = v; }
}
__global__ void k_l2_64(const float* __restrict__ src, const uint32_t* __restrict__ idx, float* out, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) { float v; asm volatile("ld.global.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(src + idx[i])); out[i] = v; }
}
__global__ void k_relaxed(const float* __restrict__ src, const uint32_t* __restrict__ idx, float* out, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) { float v; asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(src + idx[i])); out[i] = v; }
}
__global__ void k_fill(uint32_t* idx, size_t n, size_t range, uint32_t seed) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) { uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed; x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29; idx[i] = (uint32_t)(x % range); }
}

int main() {
    size_t n = 100000000, range = 300000000;
    float* src; uint32_t* idx; float* out;
    cudaMalloc(&src, range * 4); cudaMalloc(&idx, n * 4); cudaMalloc(&out, n * 4);
    cudaMemset(src, 0, range * 4);
    unsigned g = (unsigned)((n + 255) / 256);
    k_fill<<<g, 256>>>(idx, n, range, 1234);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const char* names[] = {"plain", "cg", "nc_na", "cv", "l2_64", "relaxed"};
    for (int lim : {0, 32, 128}) {
        cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, lim);
        size_t got = 0; cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
        for (int v = 0; v < 6; ++v) {
            float best = 1e9;
            for (int r = 0; r < 3; ++r) {
                cudaEventRecord(a);
                switch (v) {
                    case 0: k_plain<<<g, 256>>>(src, idx, out, n); break;
                    case 1: k_cg<<<g, 256>>>(src, idx, out, n); break;
                    case 2: k_nc_na<<<g, 256>>>(src, idx, out, n); break;
                    case 3: k_cv<<<g, 256>>>(src, idx, out, n); break;
                    case 4: k_l2_64<<<g, 256>>>(src, idx, out, n); break;
                    case 5: k_relaxed<<<g, 256>>>(src, idx, out, n); break;
                }
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
            }
            printf("limit=%d (set rc=%d got=%zu) %-8s %.3f ms  %.1f Gidx/s\n", lim, (int)e, got, names[v], best, n / best / 1e6);
        }
    }
    return 0;
}
