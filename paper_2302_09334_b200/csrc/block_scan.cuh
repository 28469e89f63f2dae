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

// Two independent exclusive scans (a and b) sharing the block barriers.  `warp_tot` holds
// 2 * (NT/32 + 1) words.
template <int NT>
__device__ __forceinline__ uint2 block_exclusive_scan2(uint2 v, uint32_t *warp_tot, uint2 &total) {
    static_assert(NT % 32 == 0 && NT <= 1024, "block size");
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t ia = v.x, ib = v.y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t na = __shfl_up_sync(0xffffffffu, ia, o), nb = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) {
            ia += na;
            ib += nb;
        }
    }
    uint32_t *ta = warp_tot, *tb = warp_tot + NW + 1;
    if (lane == 31) {
        ta[wid] = ia;
        tb[wid] = ib;
    }
    __syncthreads();
    if (wid == 0) {
        const uint32_t wa = lane < NW ? ta[lane] : 0u, wb = lane < NW ? tb[lane] : 0u;
        uint32_t xa = wa, xb = wb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t na = __shfl_up_sync(0xffffffffu, xa, o), nb = __shfl_up_sync(0xffffffffu, xb, o);
            if (lane >= o) {
                xa += na;
                xb += nb;
            }
        }
        if (lane < NW) {
            ta[lane] = xa - wa;
            tb[lane] = xb - wb;
        }
        if (lane == NW - 1) {
            ta[NW] = xa;
            tb[NW] = xb;
        }
    }
    __syncthreads();
    const uint2 res = make_uint2(ta[wid] + ia - v.x, tb[wid] + ib - v.y);
    total = make_uint2(ta[NW], tb[NW]);
    __syncthreads();
    return res;
}

}  // namespace eco
