// tools/icache.cu — cost of executing N straight-line instructions ONCE per warp (cold
// instruction cache) versus the same code in a loop (warm).  One warp per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int N>
__global__ void k_line(uint32_t *out, int reps, long long *cyc) {
    uint32_t a = threadIdx.x, b = blockIdx.x * 7 + 3, c = 11;
    const long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int i = 0; i < N; ++i) {  // independent-ish integer ops, no loads
            a = a * 0x9E3779B9u + b;
            b ^= a >> 7;
            c += a ^ b;
        }
    }
    const long long c1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c;
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}

template <int N>
void run(uint32_t *out, long long *cyc) {
    long long h[148];
    for (int reps : {1, 2, 8}) {
        k_line<N><<<148, 32>>>(out, reps, cyc);  // first launch: cold
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
        double m = 0;
        for (int i = 0; i < 148; ++i) m += h[i];
        printf("N=%5d instrs/iter~%5d reps %d: %.0f cycles per warp (%.1f cycles per iteration-instruction)\n", N, N * 4, reps,
               m / 148, m / 148 / (reps * N * 4.0));
    }
}

int main() {
    uint32_t *out;
    long long *cyc;
    cudaMalloc(&out, 148 * 32 * 4);
    cudaMalloc(&cyc, 148 * 8);
    run<64>(out, cyc);
    run<256>(out, cyc);
    run<1024>(out, cyc);
    run<2048>(out, cyc);
    return 0;
}
