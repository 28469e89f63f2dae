// tools/bw_chunks.cu — achievable HBM read bandwidth for warp-granular random chunk reads
// (the policy kernel's access pattern: per-agent 512-B input columns scattered inside a
// 68-KB agent record, agents spread over a 555-MB array), versus chunk size.  Not product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ float4 ldnc(const float *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

// each warp reads `nchunks` chunks of `chunk_floats` floats at pseudo-random agent records
template <int UNROLL>
__global__ void k_read(const float *base, size_t n_agents, int agent_floats, int chunk_floats, int nchunks,
                       int iters, float *sink) {
    const int lane = threadIdx.x & 31;
    const size_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    float acc = 0.f;
    uint32_t s = (uint32_t)warp * 2654435761u + 12345u;
    for (int it = 0; it < iters; ++it) {
        s = s * 1664525u + 1013904223u;
        const size_t agent = s % n_agents;
        const float *a = base + agent * agent_floats;
        for (int c = 0; c < nchunks; c += UNROLL) {
            float4 v[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                uint32_t h = (s >> 7) + (uint32_t)(c + u) * 40503u;
                const int ncol = agent_floats / chunk_floats;
                const float *p = a + (size_t)(h % ncol) * chunk_floats;
                v[u] = (c + u < nchunks) ? ldnc(p + lane * 4 % chunk_floats + 0) : make_float4(0, 0, 0, 0);
                if (chunk_floats > 128) {
                    // larger chunks: each lane reads several float4
                    for (int off = 128; off < chunk_floats; off += 128) {
                        float4 w = ldnc(p + off + lane * 4);
                        v[u].x += w.x;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
        }
    }
    if (acc == 123.456f) sink[0] = acc;
}

int main() {
    const size_t n_agents = 8192;
    const int agent_floats = 16960;
    float *base, *sink;
    CK(cudaMalloc(&base, n_agents * agent_floats * 4));
    CK(cudaMemset(base, 0, n_agents * agent_floats * 4));
    CK(cudaMalloc(&sink, 4));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int blocks = 148 * 3, threads = 256;
    for (int chunk : {128, 256, 512, 1024}) {
        for (int nchunks : {32, 64}) {
            const int iters = 8;
            k_read<8><<<blocks, threads>>>(base, n_agents, agent_floats, chunk, nchunks, iters, sink);
            CK(cudaDeviceSynchronize());
            cudaEventRecord(a);
            k_read<8><<<blocks, threads>>>(base, n_agents, agent_floats, chunk, nchunks, iters, sink);
            cudaEventRecord(b);
            CK(cudaDeviceSynchronize());
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double bytes = (double)blocks * threads / 32 * iters * nchunks * chunk * 4;
            printf("chunk %5d B, %2d chunks/agent, 24 warps/SM: %.0f GB/s\n", chunk * 4, nchunks, bytes / ms / 1e6);
        }
    }
    // occupancy sweep for 512-B chunks
    for (int bps : {2, 4, 8}) {
        blocks = 148 * bps;
        const int iters = 8, chunk = 128, nchunks = 32;
        k_read<8><<<blocks, threads>>>(base, n_agents, agent_floats, chunk, nchunks, iters, sink);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        k_read<8><<<blocks, threads>>>(base, n_agents, agent_floats, chunk, nchunks, iters, sink);
        cudaEventRecord(b);
        CK(cudaDeviceSynchronize());
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)blocks * threads / 32 * iters * nchunks * chunk * 4;
        printf("chunk 512 B, %d x 8 warps/SM: %.0f GB/s\n", bps, bytes / ms / 1e6);
    }
    // sequential copy reference
    {
        float *dst;
        CK(cudaMalloc(&dst, n_agents * agent_floats * 4));
        cudaEventRecord(a);
        CK(cudaMemcpy(dst, base, n_agents * agent_floats * 4, cudaMemcpyDeviceToDevice));
        cudaEventRecord(b);
        CK(cudaDeviceSynchronize());
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("D2D memcpy 555 MB: %.0f GB/s (read+write)\n", 2.0 * n_agents * agent_floats * 4 / ms / 1e6);
    }
    return 0;
}
