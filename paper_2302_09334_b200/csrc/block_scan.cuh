// block_scan.cuh — warp-shuffle block-wide exclusive scan used by the slot/birth
// compaction kernels (K4) and the state rebuild.
#pragma once
#include <cstdint>

namespace eco {

// Exclusive scan of one uint32 per thread over a block of NT threads.  `warp_tot` is
// shared scratch of NT/32 words.  Returns the exclusive prefix; `total` gets the sum.
template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t *warp_tot, uint32_t &total) {
    static_assert(NT % 32 == 0 && NT <= 1024, "block size");
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t n = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += n;
    }
    if (lane == 31) warp_tot[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        uint32_t wv = lane < NW ? warp_tot[lane] : 0u;
        uint32_t winc = wv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t n = __shfl_up_sync(0xffffffffu, winc, o);
            if (lane >= o) winc += n;
        }
        if (lane < NW) warp_tot[lane] = winc - wv;  // exclusive warp offsets
        if (lane == NW - 1) warp_tot[NW] = winc;    // block total
    }
    __syncthreads();
    const uint32_t res = warp_tot[wid] + inc - v;
    total = warp_tot[NW];
    __syncthreads();  // scratch may be reused right after
    return res;
}

}  // namespace eco
