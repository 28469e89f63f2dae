// tools/microbench.cu — measures the primitives the step's latency-bound phases are made
// of on the B200 at hand: grid-barrier cost, dependent-load latency (L2 / DRAM), an fp64
// Box-Muller chain and same-address atomic throughput.  Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ void grid_sync(unsigned int *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int *vgen = bar + 1;
        const unsigned int gen = *vgen;
        __threadfence();
        const unsigned int nblocks = gridDim.x;
        if (atomicAdd(bar, 1u) == nblocks - 1) {
            bar[0] = 0u;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*vgen == gen) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

// release/acquire variant: arrival = atom.add.release.gpu on a monotonically increasing
// counter, wait = ld.acquire.gpu until it reaches the target (no separate reset, no SC fences)
__device__ __forceinline__ void grid_sync_ra(unsigned int *ctr, unsigned int &target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        unsigned int old;
        asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
        unsigned int cur = old + 1;
        while (cur < target) asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(ctr) : "memory");
    }
    __syncthreads();
}

__global__ void k_barriers(unsigned int *bar, int n, unsigned long long *out) {
    uint64_t t0 = gt();
    for (int i = 0; i < n; ++i) grid_sync(bar);
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = gt() - t0;
}

__global__ void k_barriers_ra(unsigned int *ctr, unsigned int base, int n, unsigned long long *out) {
    unsigned int target = base;
    uint64_t t0 = gt();
    for (int i = 0; i < n; ++i) grid_sync_ra(ctr, target);
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = gt() - t0;
}

__global__ void k_chain(const int *next, int n, int start, unsigned long long *out, int *sink) {
    int j = start;
    uint64_t t0 = gt();
    for (int i = 0; i < n; ++i) j = *(volatile const int *)(next + j);
    out[0] = gt() - t0;
    sink[0] = j;
}

__global__ void k_bm(int n, unsigned long long *out, double *sink) {
    uint64_t t0 = gt();
    double acc = 0;
    uint32_t wa = 12345u + threadIdx.x, wb = 777u;
    for (int i = 0; i < n; ++i) {
        const double u1 = ((double)wa + 1.0) * 2.3283064365386963e-10;
        const double u2 = (double)wb * 2.3283064365386963e-10;
        const double r = sqrt(-2.0 * log(u1));
        const double th = 6.283185307179586 * u2;
        acc += r * cos(th) + r * sin(th);
        wa = wa * 1664525u + (uint32_t)acc;
        wb ^= wa;
    }
    if (threadIdx.x == 0) out[0] = gt() - t0;
    sink[threadIdx.x] = acc;
}

__global__ void k_atomics(unsigned long long *ctr, int per_thread) {
    for (int i = 0; i < per_thread; ++i) atomicAdd(ctr, 1ull);
}

int main() {
    unsigned int *bar;
    unsigned long long *out;
    CK(cudaMalloc(&bar, 8));
    CK(cudaMemset(bar, 0, 8));
    CK(cudaMallocManaged(&out, 64));
    for (int threads : {256, 512, 1024}) {
        void *args[] = {&bar, nullptr, &out};
        int n = 1000;
        args[1] = &n;
        CK(cudaLaunchCooperativeKernel((void *)k_barriers, 148, threads, args, 0, 0));
        CK(cudaDeviceSynchronize());
        CK(cudaLaunchCooperativeKernel((void *)k_barriers, 148, threads, args, 0, 0));
        CK(cudaDeviceSynchronize());
        printf("grid barrier, 148 x %d threads: %.3f us per barrier\n", threads, out[0] / 1000.0 / n);
    }
    {
        unsigned int *ctr;
        CK(cudaMalloc(&ctr, 4));
        CK(cudaMemset(ctr, 0, 4));
        unsigned int base = 0;
        int n = 1000;
        for (int rep = 0; rep < 2; ++rep) {
            void *args[] = {&ctr, &base, &n, &out};
            CK(cudaLaunchCooperativeKernel((void *)k_barriers_ra, 148, 512, args, 0, 0));
            CK(cudaDeviceSynchronize());
            base += 148u * n;
        }
        printf("release/acquire grid barrier, 148 x 512: %.3f us per barrier\n", out[0] / 1000.0 / n);
    }
    // dependent load chain: small (L2) and large (DRAM) random permutations
    for (size_t nelem : {(size_t)1 << 14, (size_t)1 << 27}) {
        int *h = (int *)malloc(nelem * 4), *d, *sink;
        // random cycle with a large stride
        for (size_t i = 0; i < nelem; ++i) h[i] = (int)((i + 7919 * 64 + 1) % nelem);
        CK(cudaMalloc(&d, nelem * 4));
        CK(cudaMalloc(&sink, 4));
        CK(cudaMemcpy(d, h, nelem * 4, cudaMemcpyHostToDevice));
        int n = 2000;
        k_chain<<<1, 1>>>(d, n, 0, out, sink);
        CK(cudaDeviceSynchronize());
        k_chain<<<1, 1>>>(d, n, 0, out, sink);
        CK(cudaDeviceSynchronize());
        printf("dependent load chain over %zu MB: %.1f ns per load\n", nelem * 4 >> 20, (double)out[0] / n);
        cudaFree(d);
        free(h);
    }
    {
        double *sink;
        CK(cudaMalloc(&sink, 8 * 1024));
        int n = 200;
        k_bm<<<1, 32>>>(n, out, sink);
        CK(cudaDeviceSynchronize());
        k_bm<<<1, 32>>>(n, out, sink);
        CK(cudaDeviceSynchronize());
        printf("fp64 Box-Muller chain (1 warp): %.1f ns per pair\n", (double)out[0] / n);
        k_bm<<<148 * 4, 256>>>(n, out, sink);
        CK(cudaDeviceSynchronize());
        printf("fp64 Box-Muller chain (148x4x256 threads): %.1f ns per pair per thread\n", (double)out[0] / n);
    }
    {
        unsigned long long *ctr;
        CK(cudaMalloc(&ctr, 8));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        k_atomics<<<148, 256>>>(ctr, 1);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        k_atomics<<<148, 256>>>(ctr, 10);
        cudaEventRecord(b);
        CK(cudaDeviceSynchronize());
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("same-address atomicAdd: %.2f ns per atomic (%d atomics)\n", ms * 1e6 / (148 * 256 * 10), 148 * 256 * 10);
    }
    {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        void *args[] = {&bar, nullptr, &out};
        int n = 0;
        args[1] = &n;
        CK(cudaLaunchCooperativeKernel((void *)k_barriers, 148, 512, args, 0, 0));
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        for (int i = 0; i < 100; ++i) CK(cudaLaunchCooperativeKernel((void *)k_barriers, 148, 512, args, 0, 0));
        cudaEventRecord(b);
        CK(cudaDeviceSynchronize());
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("empty cooperative launch 148x512: %.2f us each (stream, back to back)\n", ms * 1000 / 100);
    }
    return 0;
}
