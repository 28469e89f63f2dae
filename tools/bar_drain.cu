// tools/bar_drain.cu — what makes a release/acquire grid barrier slow after a phase?
// A cooperative 148 x 512 kernel runs n iterations of {variant work; grid barrier} and
// reports microseconds per iteration.  Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__device__ __forceinline__ void grid_sync_ra(unsigned long long *ctr, unsigned long long &target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        unsigned long long cur;
        asm volatile("atom.add.release.gpu.u64 %0, [%1], 1;" : "=l"(cur) : "l"(ctr) : "memory");
        cur += 1;
        while (cur < target) asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(cur) : "l"(ctr) : "memory");
    }
    __syncthreads();
}

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

__global__ void k_var(int variant, int n, unsigned long long *ctr, unsigned long long base, uint32_t *plane,
                      uint32_t *dst, unsigned long long *acc, unsigned long long *out) {
    unsigned long long target = base;
    const size_t gtid = ((size_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x) * 32 + (threadIdx.x & 31);
    const size_t half = (size_t)gridDim.x * blockDim.x / 2;
    const int items = 2600;
    uint64_t t0 = gt();
    for (int it = 0; it < n; ++it) {
        if (gtid >= half) {
            const size_t k = gtid - half;
            switch (variant) {
                case 1:
                    if (k < items) dst[k] = (uint32_t)it;
                    break;
                case 2: {  // per-warp atomic on one address (all warps of the half)
                    if ((threadIdx.x & 31) == 0) atomicAdd(acc, 1ull);
                    break;
                }
                case 3:
                case 6: {
                    if (k < items) {
                        uint32_t s = 0;
#pragma unroll
                        for (int j = 0; j < 15; ++j) {
                            const size_t a = (k + j * 13) % items;
                            s += variant == 3 ? *reinterpret_cast<volatile uint32_t *>(plane + a) : __ldcg(plane + a);
                        }
                        dst[k] = s;
                    }
                    break;
                }
                case 4: {
                    if (k < items) {
                        uint32_t s = 0;
#pragma unroll
                        for (int g = 0; g < 8; ++g) s += philox(make_uint4(g, (uint32_t)k, it, 4), 1u, 0u).x;
                        dst[k] = s;
                    }
                    break;
                }
                case 5: {  // warp-aggregated atomic for the first 81 warps only
                    if (k < items && (threadIdx.x & 31) == 0) atomicAdd(acc, 1ull);
                    break;
                }
                case 7: {  // regrow-like: volatile loads + philox + store + warp atomic
                    if (k < items) {
                        uint32_t s = 0;
#pragma unroll
                        for (int j = 0; j < 15; ++j)
                            s += *reinterpret_cast<volatile uint32_t *>(plane + (k + j * 13) % items);
#pragma unroll
                        for (int g = 0; g < 8; ++g) s += philox(make_uint4(g, (uint32_t)k, it, 4), s, 0u).x;
                        dst[k] = s;
                        if ((threadIdx.x & 31) == 0) atomicAdd(acc, (unsigned long long)s & 7);
                    }
                    break;
                }
                default:
                    break;
            }
        }
        grid_sync_ra(ctr, target);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = gt() - t0;
}

int main() {
    unsigned long long *ctr, *acc, *out;
    uint32_t *plane, *dst;
    CK(cudaMalloc(&ctr, 8));
    CK(cudaMemset(ctr, 0, 8));
    CK(cudaMalloc(&acc, 8));
    CK(cudaMalloc(&out, 8));
    CK(cudaMalloc(&plane, 1 << 20));
    CK(cudaMemset(plane, 1, 1 << 20));
    CK(cudaMalloc(&dst, 1 << 20));
    unsigned long long base = 0;
    int n = 2000;
    const char *names[] = {"empty", "2600 stores", "1184 warp atomics, one address", "15 volatile loads + store",
                           "8 philox + store", "81 warp atomics, one address", "15 ldcg loads + store",
                           "regrow-like (loads, philox, store, 81 warp atomics)"};
    for (int v = 0; v < 8; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            void *args[] = {&v, &n, &ctr, &base, &plane, &dst, &acc, &out};
            CK(cudaLaunchCooperativeKernel((void *)k_var, 148, 512, args, 0, 0));
            CK(cudaDeviceSynchronize());
            base += 148ull * n;
        }
        unsigned long long o;
        CK(cudaMemcpy(&o, out, 8, cudaMemcpyDeviceToHost));
        printf("variant %d %-55s %.3f us per iteration\n", v, names[v], o / 1000.0 / n);
    }
    return 0;
}
