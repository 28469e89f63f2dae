// tools/bm_cold.cu — cost of an fp64 Box-Muller (Philox + log + sqrt + sincos) executed once
// per thread in a fresh kernel (cold instruction cache) versus in a loop.  Not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint4 philox(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}
__device__ __forceinline__ void bm(uint32_t a, uint32_t b, double &za, double &zb) {
    const double u1 = ((double)a + 1.0) * 2.3283064365386963e-10, u2 = (double)b * 2.3283064365386963e-10;
    const double r = sqrt(-2.0 * log(u1)), th = 6.283185307179586 * u2;
    double s, c;
    sincos(th, &s, &c);
    za = r * c;
    zb = r * s;
}
__global__ void k_once(float *out, int reps) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0.0;
    for (int i = 0; i < reps; ++i) {
        const uint4 d = philox(make_uint4(i, g, 7, 5), 1u, 2u);
        double za, zb;
        bm(d.x, d.y, za, zb);
        acc += za + zb;
    }
    out[g] = (float)acc;
}
__global__ void k_philox_only(float *out, int reps) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int i = 0; i < reps; ++i) acc += philox(make_uint4(i, g, 7, 5), 1u, 2u).x;
    out[g] = (float)acc;
}
__global__ void k_empty(float *out) { out[blockIdx.x * blockDim.x + threadIdx.x] = 1.f; }

__global__ void k_read(const float4 *a, size_t n, float *sink) {
    float acc = 0.f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) acc += a[i].x;
    if (acc == 12345.f) *sink = acc;
}

int main() {
    float *out;
    CK(cudaMalloc(&out, 148 * 512 * 4 * 4));
    void *fl;
    const size_t FL = 256u << 20;
    CK(cudaMalloc(&fl, FL));
    auto flush = [&]() {
        cudaMemsetAsync(fl, 0, FL);
        k_read<<<148 * 4, 512>>>((const float4 *)fl, FL / 16, out);
    };
    cudaEvent_t a0, b0;
    cudaEventCreate(&a0);
    cudaEventCreate(&b0);
    for (int mode = 0; mode < 2; ++mode) {
        for (int reps : {1, 4}) {
            float sum_bm = 0.f, sum_e = 0.f;
            const int N = 20;
            for (int it = 0; it < N; ++it) {
                if (mode) flush();
                cudaEventRecord(a0);
                k_once<<<148, 512>>>(out, reps);
                cudaEventRecord(b0);
                cudaEventSynchronize(b0);
                float ms;
                cudaEventElapsedTime(&ms, a0, b0);
                sum_bm += ms;
                if (mode) flush();
                cudaEventRecord(a0);
                k_empty<<<148, 512>>>(out);
                cudaEventRecord(b0);
                cudaEventSynchronize(b0);
                cudaEventElapsedTime(&ms, a0, b0);
                sum_e += ms;
            }
            printf("%s reps %d: box-muller kernel %.2f us, empty %.2f us (mean of %d)\n", mode ? "L2 flushed" : "warm L2   ",
                   reps, sum_bm / N * 1e3, sum_e / N * 1e3, N);
        }
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int round = 0; round < 2; ++round) {
        for (int reps : {1, 2, 4, 16}) {
            float best = 1e9, bestp = 1e9, beste = 1e9;
            for (int it = 0; it < 20; ++it) {
                cudaEventRecord(a);
                k_once<<<148, 512>>>(out, reps);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
                cudaEventRecord(a);
                k_philox_only<<<148, 512>>>(out, reps);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms, a, b);
                if (ms < bestp) bestp = ms;
                cudaEventRecord(a);
                k_empty<<<148, 512>>>(out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms, a, b);
                if (ms < beste) beste = ms;
            }
            printf("reps %2d: box-muller kernel %.2f us, philox-only %.2f us, empty %.2f us\n", reps, best * 1e3,
                   bestp * 1e3, beste * 1e3);
        }
    }
    return 0;
}
