// world.cu — world initialisation (K0), the occupancy/list rebuild used by create and
// set_state, and the canonical <-> device state conversions.
#include <cub/device/device_radix_sort.cuh>

#include "block_scan.cuh"
#include "sim_internal.cuh"

namespace eco {

// ---------------------------------------------------------------- K0 initialisation
// R[cell] = philox(INIT_RES, 0, cell>>2)[cell&3] < floor(rho * 2^32)
__global__ void k_init_resources(DevParams p) {
    const int wx = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int w = blockIdx.z;
    if (wx >= p.WW) return;
    uint32_t bits = 0u;
    const int x_base = wx << 5;
    for (int g = 0; g < 8; ++g) {
        const int x0 = x_base + 4 * g;
        if (x0 >= p.W) break;
        const uint4 d = draw4(p.seeds[w], PURPOSE_INIT_RES, 0u, (uint32_t)(((int64_t)y * p.W + x0) >> 2), 0u);
#pragma unroll
        for (int m = 0; m < 4; ++m)
            if (word_of(d, m) < p.init_res_thr) bits |= 1u << (4 * g + m);
    }
    p.plane0[(size_t)w * plane_words(p) + (size_t)y * p.WW + wx] = bits;
}

// placement keys: (draw(INIT_PLACE, 0, cell) << 32 | cell) for empty cells, ~0 for full
__global__ void k_place_keys(DevParams p, int w, unsigned long long *keys) {
    const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t HW = (int64_t)p.H * p.W;
    if (cell >= HW) return;
    const uint32_t *R = p.plane0 + (size_t)w * plane_words(p);
    unsigned long long k = ~0ull;
    if (!get_bit(R, p, (int)cell)) {
        const uint4 d = draw4(p.seeds[w], PURPOSE_INIT_PLACE, 0u, (uint32_t)(cell >> 2), 0u);
        k = ((unsigned long long)word_of(d, (int)(cell & 3)) << 32) | (unsigned long long)(uint32_t)cell;
    }
    keys[cell] = k;
}

// slot i < N0 takes the i-th smallest key; everything else is dead
__global__ void k_init_agents(DevParams p, int w, int n_initial, const unsigned long long *sorted) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.S) return;
    const size_t gs = (size_t)w * p.S + i;
    const bool live = i < n_initial;
    p.alive[gs] = live ? 1 : 0;
    p.cell[gs] = live ? (int32_t)(uint32_t)(sorted[i] & 0xffffffffull) : 0;
    p.energy[gs] = live ? p.e_init : 0;
    p.age[gs] = 0;
    p.repr[gs] = 0;
    p.last_action[gs] = 0;
    p.ate[gs] = 0;
    p.gr_seen[gs] = p.gr_ate[gs] = 0;
    p.gr_T[gs] = p.gr_C[gs] = 0;
}

// initial weights w_j = (float)(std * z_j), z from INIT_W keyed by the initial cell
__global__ void k_init_weights(DevParams p, int w, int n_initial) {
    const int groups = (p.P + 3) >> 2;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    for (int i = blockIdx.y; i < n_initial; i += gridDim.y) {
        if (q >= groups) continue;
        const size_t gs = (size_t)w * p.S + i;
        const uint4 d = draw4(p.seeds[w], PURPOSE_INIT_W, 0u, (uint32_t)p.cell[gs], (uint32_t)q);
        double z[4];
        box_muller(d.x, d.y, z[0], z[1]);
        box_muller(d.z, d.w, z[2], z[3]);
        float *wd = p.weights + gs * (size_t)p.Pd;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int j = 4 * q + m;
            if (j >= p.P) break;
            wd[canon_to_dev(p, j)] =
                __double2float_rn(__dmul_rn(p.init_weight_std, z[m]));
        }
    }
}

cudaError_t launch_init_resources(const DevParams &p, cudaStream_t s) {
    dim3 g1((p.WW + 127) / 128, p.H, p.n_worlds);
    k_init_resources<<<g1, 128, 0, s>>>(p);
    return cudaGetLastError();
}

size_t init_agents_scratch_bytes(const DevParams &p) {
    const int64_t HW = (int64_t)p.H * p.W;
    size_t need = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, need, (unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                   (int)HW, 0, 64);
    return 2 * sizeof(unsigned long long) * (size_t)HW + need + 256;
}

cudaError_t launch_init_agents(const DevParams &p, int n_initial, cudaStream_t s, void *scratch,
                               size_t scratch_bytes, const BandParams *band, int32_t *n_own_dev) {
    if (p.S == 0) return cudaSuccess;
    const int64_t HW = (int64_t)p.H * p.W;
    unsigned long long *keys_in = static_cast<unsigned long long *>(scratch);
    unsigned long long *keys_out = keys_in + HW;
    void *tmp = keys_out + HW;
    const size_t tmp_bytes = scratch_bytes - 2 * sizeof(unsigned long long) * (size_t)HW;
    cudaError_t e;
    for (int w = 0; w < p.n_worlds; ++w) {
        k_place_keys<<<(unsigned)((HW + 255) / 256), 256, 0, s>>>(p, w, keys_in);
        size_t need = 0;
        e = cub::DeviceRadixSort::SortKeys(nullptr, need, keys_in, keys_out, (int)HW, 0, 64, s);
        if (e != cudaSuccess) return e;
        if (need > tmp_bytes) return cudaErrorMemoryAllocation;
        e = cub::DeviceRadixSort::SortKeys(tmp, need, keys_in, keys_out, (int)HW, 0, 64, s);
        if (e != cudaSuccess) return e;
        int n_agents = n_initial;
        if (band) {  // one band of a banded world: its rows' agents in local slots 0..
            if ((e = band_init_agents(p, *band, n_initial, keys_out, n_own_dev, s)) != cudaSuccess) return e;
            int32_t n_own = 0;
            if ((e = cudaMemcpyAsync(&n_own, n_own_dev, 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
            if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
            n_agents = n_own < p.S ? n_own : p.S;
        } else {
            k_init_agents<<<(p.S + 255) / 256, 256, 0, s>>>(p, w, n_initial, keys_out);
        }
        if (n_agents > 0) {
            const int groups = (p.P + 3) >> 2;
            dim3 g((groups + 127) / 128, n_agents < 4096 ? n_agents : 4096);
            k_init_weights<<<g, 128, 0, s>>>(p, w, n_agents);
        }
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// ------------------------------------------------------- rebuild (create / set_state)
// One CTA per world: O from (alive, cell); ascending alive list; resource count.
__global__ void __launch_bounds__(1024) k_rebuild(DevParams p) {
    __shared__ uint32_t scratch[33];
    __shared__ unsigned long long res_acc;
    const int w = blockIdx.x;
    uint32_t *O = p.occ + (size_t)w * plane_words(p);
    const uint32_t *R = plane_cur(p, p.t[w]) + (size_t)w * plane_words(p);
    if (threadIdx.x == 0) res_acc = 0ull;
    unsigned long long local = 0ull;
    for (size_t i = threadIdx.x; i < plane_words(p); i += blockDim.x) {
        O[i] = 0u;
        const int y = (int)(i / p.WW);
        if (y >= p.row_lo && y < p.row_hi) local += __popc(R[i]);  // the rows this handle owns
    }
    if (p.coloc)  // co-location: agents per cell, counted below
        for (size_t i = threadIdx.x; i < (size_t)p.H * p.W; i += blockDim.x) p.ncount[(size_t)w * p.H * p.W + i] = 0;
    atomicAdd(&res_acc, local);
    __syncthreads();
    uint32_t base = 0u;
    const int64_t t = p.t[w];
    int32_t *list = list_of(p, t, w);
    for (int i0 = 0; i0 < p.S; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        const size_t gs = (size_t)w * p.S + i;
        const uint32_t a = (i < p.S && p.alive[gs]) ? 1u : 0u;
        if (a) {
            uint32_t bit;
            uint32_t *wp = word_ptr(O, p, p.cell[gs], bit);
            atomicOr(wp, bit);
            if (p.coloc) atomicAdd(p.ncount + (size_t)w * p.H * p.W + p.cell[gs], 1);
        }
        const uint32_t word = __ballot_sync(0xffffffffu, a != 0u);
        if ((threadIdx.x & 31) == 0 && i < p.S) p.alive_bits[(size_t)w * p.SW + (i >> 5)] = word;
        uint32_t tot;
        const uint32_t ex = block_exclusive_scan<1024>(a, scratch, tot);
        if (a) {
            list[base + ex] = i;
            list_cell_of(p, t, w)[base + ex] = p.cell[gs];
        }
        if (i < p.S) {  // movement windows: a run (re)started at a window start measures it
            p.mv_cell[gs] = a ? p.cell[gs] : 0;
            p.mv_inv[gs] = (a && t % SIM_MOVE_WINDOW == 0) ? p.age[gs] - (int32_t)t : -(1 << 29);
        }
        base += tot;
    }
    for (int k = threadIdx.x; k < p.mv_cap * SIM_MOVE_BINS; k += blockDim.x)
        p.mv_hist[(size_t)w * p.mv_cap * SIM_MOVE_BINS + k] = 0;
    if (threadIdx.x == 0) {
        *count_of(p, t, w) = (int32_t)base;
        *count_of(p, t + 1, w) = 0;
        p.n_win[w] = 0;
        p.n_cand[w] = 0;
        p.n_births[w] = 0;
        p.res_count[w] = (int64_t)res_acc;
    }
}

cudaError_t launch_rebuild(const DevParams &p, cudaStream_t s) {
    k_rebuild<<<p.n_worlds, 1024, 0, s>>>(p);
    return cudaGetLastError();
}

// ------------------------------------------------------------- plane <-> bytes
__global__ void k_pack_resources(DevParams p, const uint8_t *bytes) {
    const int wx = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y, w = blockIdx.z;
    if (wx >= p.WW) return;
    uint32_t bits = 0u;
    for (int b = 0; b < 32; ++b) {
        const int x = (wx << 5) + b;
        if (x < p.W && bytes[((size_t)w * p.H + y) * p.W + x]) bits |= 1u << b;
    }
    uint32_t *R = plane_cur(p, p.t[w]) + (size_t)w * plane_words(p);
    R[(size_t)y * p.WW + wx] = bits;
}

__global__ void k_unpack_resources(DevParams p, uint8_t *bytes) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y, w = blockIdx.z;
    if (x >= p.W) return;
    const uint32_t *R = plane_cur(p, p.t[w]) + (size_t)w * plane_words(p);
    bytes[((size_t)w * p.H + y) * p.W + x] = (R[(size_t)y * p.WW + (x >> 5)] >> (x & 31)) & 1u;
}

cudaError_t launch_pack_resources(const DevParams &p, const uint8_t *bytes, cudaStream_t s) {
    k_pack_resources<<<dim3((p.WW + 127) / 128, p.H, p.n_worlds), 128, 0, s>>>(p, bytes);
    return cudaGetLastError();
}

cudaError_t launch_unpack_resources(const DevParams &p, uint8_t *bytes, cudaStream_t s) {
    k_unpack_resources<<<dim3((p.W + 255) / 256, p.H, p.n_worlds), 256, 0, s>>>(p, bytes);
    return cudaGetLastError();
}

// logits: canonical [n][5] <-> device [n][LOGIT_STRIDE] (one contiguous copy and this kernel
// instead of a pitched copy of 20-byte rows, which moves a few bytes per DMA row)
__global__ void k_logits_restride(float *dst, int dst_stride, const float *src, int src_stride, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * 5) return;
    const size_t a = i / 5;
    const int k = (int)(i - a * 5);
    dst[a * dst_stride + k] = src[a * src_stride + k];
}

cudaError_t launch_logits_restride(float *dst, int dst_stride, const float *src, int src_stride, size_t n,
                                   cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_logits_restride<<<(unsigned)((n * 5 + 255) / 256), 256, 0, s>>>(dst, dst_stride, src, src_stride, n);
    return cudaGetLastError();
}

// --------------------------------------------------- weights canonical <-> device
__global__ void k_weights_to_device(DevParams p, const float *canon, size_t first, size_t n) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * (size_t)p.P) return;
    const size_t a = idx / p.P;
    const int j = (int)(idx - a * p.P);
    p.weights[(first + a) * p.Pd + canon_to_dev(p, j)] = canon[idx];
}

__global__ void k_weights_to_canon(DevParams p, float *canon, size_t first, size_t n) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * (size_t)p.P) return;
    const size_t a = idx / p.P;
    const int j = (int)(idx - a * p.P);
    canon[idx] = p.weights[(first + a) * p.Pd + canon_to_dev(p, j)];
}

cudaError_t launch_weights_to_device(const DevParams &p, const float *canon, size_t first, size_t n, cudaStream_t s) {
    const size_t tot = n * (size_t)p.P;
    if (!tot) return cudaSuccess;
    k_weights_to_device<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(p, canon, first, n);
    return cudaGetLastError();
}

cudaError_t launch_weights_to_canon(const DevParams &p, float *canon, size_t first, size_t n, cudaStream_t s) {
    const size_t tot = n * (size_t)p.P;
    if (!tot) return cudaSuccess;
    k_weights_to_canon<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(p, canon, first, n);
    return cudaGetLastError();
}

// ------------------------------------------- set_state: the live agents' weights only
// sim_set_state imports the weights of LIVE slots only (a dead slot's fields are unspecified,
// sim.h): live[k] = w*S + slot for k < n_live.  Gather: canonical row k of the source (row
// live[k] when by_slot, i.e. the caller's whole [n_worlds*S][P] array read in place from
// mapped host memory; row k of a compacted device copy otherwise) -> device-layout row k of
// `stage`, and any non-finite value sets *bad (the handle's weights are not touched yet).
// Scatter (after the host saw *bad == 0): stage row k -> the weights of live[k].
__global__ void k_weights_gather(DevParams p, const float *src, int by_slot, const int32_t *live, int n_live,
                                 float *stage, int32_t *bad) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= p.P) return;
    const int d = canon_to_dev(p, j);
    int nonfin = 0;
    for (int k = blockIdx.y; k < n_live; k += gridDim.y) {
        const size_t row = by_slot ? (size_t)live[k] : (size_t)k;
        const float v = src[row * p.P + j];
        nonfin |= !isfinite(v);
        stage[(size_t)k * p.Pd + d] = v;
    }
    if (nonfin) atomicOr(bad, 1);
}

__global__ void k_weights_scatter(DevParams p, const float4 *stage, const int32_t *live, int n_live) {
    const int q4 = p.Pd >> 2;  // float4 per row (Pd is a multiple of 32 floats)
    for (int k = blockIdx.y; k < n_live; k += gridDim.y) {
        float4 *dst = reinterpret_cast<float4 *>(p.weights + (size_t)live[k] * p.Pd);
        for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < q4; q += gridDim.x * blockDim.x)
            dst[q] = stage[(size_t)k * q4 + q];
    }
}

__global__ void k_weights_to_canon_list(DevParams p, const int32_t *list, int n, float *canon) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= p.P) return;
    const int d = canon_to_dev(p, j);
    for (int k = blockIdx.y; k < n; k += gridDim.y) canon[(size_t)k * p.P + j] = p.weights[(size_t)list[k] * p.Pd + d];
}

cudaError_t launch_weights_to_canon_list(const DevParams &p, const int32_t *list, int n, float *canon, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    dim3 g((unsigned)((p.P + 255) / 256), (unsigned)(n < 8192 ? n : 8192));
    k_weights_to_canon_list<<<g, 256, 0, s>>>(p, list, n, canon);
    return cudaGetLastError();
}

cudaError_t launch_weights_gather(const DevParams &p, const float *src, bool by_slot, const int32_t *live, int n_live,
                                  float *stage, int32_t *bad, cudaStream_t s) {
    if (n_live <= 0) return cudaSuccess;
    dim3 g((unsigned)((p.P + 255) / 256), (unsigned)(n_live < 8192 ? n_live : 8192));
    k_weights_gather<<<g, 256, 0, s>>>(p, src, by_slot ? 1 : 0, live, n_live, stage, bad);
    return cudaGetLastError();
}

cudaError_t launch_weights_scatter(const DevParams &p, const float *stage, const int32_t *live, int n_live,
                                   cudaStream_t s) {
    if (n_live <= 0) return cudaSuccess;
    dim3 g((unsigned)((p.Pd / 4 + 255) / 256), (unsigned)(n_live < 8192 ? n_live : 8192));
    k_weights_scatter<<<g, 256, 0, s>>>(p, reinterpret_cast<const float4 *>(stage), live, n_live);
    return cudaGetLastError();
}

}  // namespace eco
