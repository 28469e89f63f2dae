// Does an L2 persisting access-policy window survive a 512 MiB streaming flush on B200?
// A pointer chase over an 8 MiB buffer (one dependent load per 4 KB page, 2048 hops) after
// the buffer was touched by a kernel carrying the window, then a memset + read flush.
// Modes: none, stream attribute, graph kernel-node attribute.  Prints ns per hop.
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

__global__ void touch(unsigned *buf, size_t n) {
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) buf[i] += 0u;
}
__global__ void chase(const unsigned *buf, int hops, unsigned long long *out) {
    unsigned idx = 0;
    unsigned long long t0 = clock64();
    for (int h = 0; h < hops; ++h) idx = buf[idx];
    unsigned long long t1 = clock64();
    out[0] = t1 - t0;
    out[1] = idx;
}
__global__ void flush_read(const float4 *f, size_t n, float *sink) {
    float acc = 0.f;
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) acc += f[i].x;
    if (acc == 12345.f) *sink = acc;
}

int main() {
    const size_t bytes = 8 << 20, n = bytes / 4, stride = 1024;  // 4 KB hops
    unsigned *buf;
    cudaMalloc(&buf, bytes);
    std::vector<unsigned> h(n);
    const int hops = (int)(n / stride);
    for (int k = 0; k < hops; ++k) h[(size_t)k * stride] = (unsigned)(((size_t)((k * 7 + 3) % hops)) * stride);
    cudaMemcpy(buf, h.data(), bytes, cudaMemcpyHostToDevice);
    size_t fb = (size_t)512 << 20;
    void *flush;
    cudaMalloc(&flush, fb);
    float *sink;
    cudaMalloc(&sink, 4);
    unsigned long long *out;
    cudaMallocManaged(&out, 16);
    int maxp = 0;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
    printf("max persisting L2 %d bytes\n", maxp);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes < (size_t)maxp ? bytes : (size_t)maxp);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaAccessPolicyWindow win{};
    win.base_ptr = buf;
    win.num_bytes = bytes;
    win.hitRatio = 1.0f;
    win.hitProp = cudaAccessPropertyPersisting;
    win.missProp = cudaAccessPropertyStreaming;
    for (int mode = 0; mode < 3; ++mode) {
        cudaCtxResetPersistingL2Cache();
        cudaStreamAttrValue sv{};
        if (mode == 1) sv.accessPolicyWindow = win;
        cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &sv);
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        touch<<<148, 256, 0, s>>>(buf, n);
        chase<<<1, 1, 0, s>>>(buf, hops, out);
        cudaStreamEndCapture(s, &g);
        if (mode == 2) {
            size_t nn = 0;
            cudaGraphGetNodes(g, nullptr, &nn);
            std::vector<cudaGraphNode_t> nodes(nn);
            cudaGraphGetNodes(g, nodes.data(), &nn);
            cudaKernelNodeAttrValue v{};
            v.accessPolicyWindow = win;
            for (auto nd : nodes) cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributeAccessPolicyWindow, &v);
        }
        cudaGraphInstantiate(&ge, g, 0);
        double tot_warm = 0, tot_cold = 0;
        for (int it = 0; it < 5; ++it) {
            cudaGraphLaunch(ge, s);  // touch + chase (warm)
            cudaStreamSynchronize(s);
            tot_warm += (double)out[0] / hops;
            cudaMemsetAsync(flush, 1, fb, s);
            flush_read<<<148 * 4, 256, 0, s>>>((const float4 *)flush, fb / 16, sink);
            chase<<<1, 1, 0, s>>>(buf, hops, out);  // after the flush (no window on this launch)
            cudaStreamSynchronize(s);
            tot_cold += (double)out[0] / hops;
        }
        printf("mode %s: warm %.0f cycles/hop, after flush %.0f cycles/hop (%s)\n",
               mode == 0 ? "none" : mode == 1 ? "stream-attr" : "graph-node-attr", tot_warm / 5, tot_cold / 5,
               cudaGetErrorString(cudaGetLastError()));
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
    }
    return 0;
}
