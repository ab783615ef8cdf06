// Throughput of warp peer detection on B200: __match_any_sync vs 8 bit-sliced
// ballots (the form the sort passes use).  One launch per variant, 148 x 8
// CTAs of 512 threads, ITER rounds each; prints ns per warp-round per SM.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITER = 4096;
__global__ void k_match(unsigned* out, unsigned seed) {
    unsigned v = (threadIdx.x * 2654435761u) ^ seed, acc = 0;
    for (int i = 0; i < ITER; ++i) {
        v = v * 1664525u + 1013904223u;
        acc += __match_any_sync(0xffffffffu, (v >> 24) & 255u);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_ballot(unsigned* out, unsigned seed) {
    unsigned v = (threadIdx.x * 2654435761u) ^ seed, acc = 0;
    for (int i = 0; i < ITER; ++i) {
        v = v * 1664525u + 1013904223u;
        const unsigned d = (v >> 24) & 255u;
        unsigned m = 0xffffffffu;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const unsigned bit = (d >> b) & 1u;
            const unsigned bal = __ballot_sync(0xffffffffu, bit);
            m &= bit ? bal : ~bal;
        }
        acc += m;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_base(unsigned* out, unsigned seed) {
    unsigned v = (threadIdx.x * 2654435761u) ^ seed, acc = 0;
    for (int i = 0; i < ITER; ++i) {
        v = v * 1664525u + 1013904223u;
        acc += (v >> 24) & 255u;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    unsigned* out;
    const int blocks = 148 * 4, threads = 512;
    cudaMalloc(&out, sizeof(unsigned) * blocks * threads);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[3] = {"base", "match_any", "ballot8"};
    for (int rep = 0; rep < 2; ++rep)
        for (int v = 0; v < 3; ++v) {
            cudaEventRecord(a);
            if (v == 0) k_base<<<blocks, threads>>>(out, 1);
            if (v == 1) k_match<<<blocks, threads>>>(out, 1);
            if (v == 2) k_ballot<<<blocks, threads>>>(out, 1);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double rounds_per_sm = (double)blocks * threads / 32 * ITER / 148;
            if (rep) printf("%-10s %8.3f ms  %6.2f ns per warp-round per SM  (%.1f SM cycles @1.965GHz)\n", names[v], ms,
                            ms * 1e6 / rounds_per_sm, ms * 1e6 / rounds_per_sm * 1.965);
        }
    return 0;
}
