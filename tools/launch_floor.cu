// The event-timed floor of one step's launches after an L2 flush, by launch method:
// (a) a CUDA graph of {plain kernel, cooperative kernel with a programmatic edge} — what
// sim_step(1) launches — against (b) the same two kernels launched directly on the stream,
// (c) one cooperative kernel alone (graph and direct), (d) two events with nothing between,
// (e) the graphs of (a) and (c) without the cooperative attribute on the 148 x 768 kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/launch_floor tools/launch_floor.cu
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess) {                                                   \
            printf("%s: %s\n", #x, cudaGetErrorString(e_));                        \
            return 1;                                                              \
        }                                                                          \
    } while (0)

__global__ void k_a(int *x) {
    if (blockIdx.x == 0 && threadIdx.x == 0) x[0] += 1;
}
__global__ void k_b(int *x) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (blockIdx.x == 0 && threadIdx.x == 0) x[1] += x[0];
}
__global__ void k_flush(const float4 *src, float *out, size_t n) {
    float acc = 0.f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const float4 v = src[i];
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 123.456f) out[0] = acc;
}

static bool g_no_coop = false;  // the second kernel without the cooperative attribute (same grid)
static cudaError_t launch_pair(cudaStream_t s, int *x, bool coop_only) {
    cudaError_t e = cudaSuccess;
    if (!coop_only) {
        k_a<<<148 * 4, 256, 0, s>>>(x);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(768);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = coop_only ? 1 : 2;
    if (g_no_coop) {  // only the programmatic edge (or no attribute at all)
        at[0] = at[1];
        cfg.numAttrs = coop_only ? 0 : 1;
    }
    return cudaLaunchKernelEx(&cfg, k_b, x);
}

int main() {
    const size_t FL = 256u << 20;
    const int K = 300;
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int *x;
    CK(cudaMalloc(&x, 64));
    CK(cudaMemset(x, 0, 64));
    char *fb;
    float *fo;
    CK(cudaMalloc(&fb, FL));
    CK(cudaMalloc(&fo, 4));
    std::vector<cudaEvent_t> e0(K), e1(K);
    for (int i = 0; i < K; ++i) {
        CK(cudaEventCreate(&e0[i]));
        CK(cudaEventCreate(&e1[i]));
    }
    cudaGraph_t g[4];
    cudaGraphExec_t ge[4];
    for (int c = 0; c < 4; ++c) {
        g_no_coop = c >= 2;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        CK(launch_pair(s, x, (c & 1) == 1));
        CK(cudaStreamEndCapture(s, &g[c]));
        CK(cudaGraphInstantiate(&ge[c], g[c], 0));
        CK(cudaGraphUpload(ge[c], s));
    }
    g_no_coop = false;
    const char *names[] = {"graph {plain, coop+PDL}", "direct {plain, coop+PDL}", "graph {coop}", "direct {coop}", "nothing",
                           "graph {plain, big+PDL}", "graph {big}"};
    for (int flush = 1; flush >= 0; --flush)
        for (int m = 0; m < 7; ++m) {
            for (int i = 0; i < K; ++i) {
                if (flush) {
                    CK(cudaMemsetAsync(fb, i & 1, FL, s));
                    k_flush<<<148 * 8, 256, 0, s>>>(reinterpret_cast<const float4 *>(fb), fo, FL / 16);
                }
                CK(cudaEventRecord(e0[i], s));
                if (m == 0) CK(cudaGraphLaunch(ge[0], s));
                if (m == 1) CK(launch_pair(s, x, false));
                if (m == 2) CK(cudaGraphLaunch(ge[1], s));
                if (m == 3) CK(launch_pair(s, x, true));
                if (m == 5) CK(cudaGraphLaunch(ge[2], s));
                if (m == 6) CK(cudaGraphLaunch(ge[3], s));
                CK(cudaEventRecord(e1[i], s));
            }
            CK(cudaStreamSynchronize(s));
            std::vector<float> t(K);
            for (int i = 0; i < K; ++i) CK(cudaEventElapsedTime(&t[i], e0[i], e1[i]));
            std::sort(t.begin(), t.end());
            printf("flush=%d %-26s median %.2f us  min %.2f  p90 %.2f\n", flush, names[m], t[K / 2] * 1e3, t[0] * 1e3,
                   t[K * 9 / 10] * 1e3);
        }
    return 0;
}
