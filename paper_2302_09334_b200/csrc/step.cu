// step.cu — the kernels of one world step (sm_100a).
//
// Graph mode (sim_step): two cooperative launches per step,
//   k_policy  [mutation of the previous step's children] + a2 observation + a3 per-agent
//             LSTM/head/argmax + the claim half of a4
//   k_post    a4 move/consume/physiology/death | grid barrier | a1 regrowth of step t+1 +
//             a5 birth candidates | grid barrier | a5 rank/winners/placement, t += 1
// (the first step after create/set_state is preceded by a standalone k_regrow; state
// export first completes any pending mutation with the standalone k_mutate).
// Instrumented mode (sim_step_timed): the same phases as separate kernels, timed one by one.
#include "phases.cuh"

namespace eco {

__device__ __constant__ int kDY[5] = {0, -1, 1, 0, 0};  // stay, N, S, E, W (R13)
__device__ __constant__ int kDX[5] = {0, 0, 0, 1, -1};

// streaming 16-B load of per-agent weights: read once per step, no reuse inside the
// step, so keep them out of L1 (L2 still serves re-reads across steps when they fit).
// `fresh` weights (a child written earlier in the same kernel) take the coherent L2 path.
__device__ __forceinline__ float4 ld_weights4(const float *ptr, bool fresh) {
    float4 v;
    if (fresh)
        asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "l"(ptr));
    else
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "l"(ptr));
    return v;
}

__device__ __forceinline__ float ld_weight(const float *ptr, bool fresh) {
    float v;
    if (fresh) asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(ptr));
    else asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(ptr));
    return v;
}

__device__ __forceinline__ float sigmoidf_acc(float z) { return 1.0f / (1.0f + expf(-z)); }

__device__ __forceinline__ void flush_counters(const DevParams &p, int w, unsigned long long nnz,
                                               unsigned long long ties) {
    if (w < 0) return;
    sim_step_record *rec = record_of(p, p.t[w], w);
    if (nnz) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->obs_nnz), nnz);
    if (ties) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->near_ties), ties);
}

// ------------------------------------------------------------------------- K2 policy
// Lane group of HD lanes per live agent (warp per agent at Hd = 32); lane k owns hidden
// unit k and its four gate rows (i, f, g, o).
//   x    : the (2r+1)^2 x 2 window of (R', O_t) as a bitmask in registers
//   z    = sum over ACTIVE inputs j of W_ih^T[j][k][:]  +  sum_j h_j W_hh^T[j][k][:]  + b[k][:]
//          (x is binary, so only the columns with x_j = 1 are read: the algorithmic bytes)
//   c'   = f*c + i*g,  h' = o*tanh(c'),  logits = W_out h' + b_out
//   a    = argmax, lowest index on ties; margin < 1e-4 counted as a near-tie (R28)
// then the move claim of a4: a valid non-stay move posts (MOVE draw << 32 | ~cell) with
// atomicMax on claim[target] (R14).
//
// with_mutation: the children placed by the previous step's rank phase get their weights
// here first (every warp runs its share of the mutation items before any agent); a warp
// whose agent is such a child waits for that child's items (mut_done) before reading its
// weights, through the coherent L2 path.  Requires a cooperative launch (co-residency).
template <int HD>
__global__ void __launch_bounds__(256, 3) k_policy(DevParams p, int with_mutation) {
    constexpr int G = HD;
    constexpr int AG = 32 / HD;  // agents per warp
    constexpr int U = 8;         // sparse columns in flight per lane
    constexpr int UH = HD < 8 ? HD : 8;
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int k = lane & (G - 1);
    const int grp = lane / G;
    const int wib = threadIdx.x >> 5;
    const int warps_per_block = blockDim.x >> 5;
    const long total = (long)p.n_worlds * p.S;
    const long per_round = (long)gridDim.x * warps_per_block * AG;
    const size_t HW = (size_t)p.H * p.W;

    // housekeeping for the later phases of this step: the survivor list of step t+1, the
    // winner counters and the record of step t+1 (whose regrowth runs early, inside this
    // step's k_post) start at 0; the birth bitmap of parity t+1 (used by step t-1) is
    // cleared for step t+1.
    {
        const size_t gtid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
        const size_t gthreads = (size_t)gridDim.x * blockDim.x;
        const size_t pw = plane_words(p);
        for (size_t k = gtid; k < (size_t)p.n_worlds * pw; k += gthreads) {
            const int w = (int)(k / pw);
            bbits_of(p, p.t[w] + 1, w)[k - (size_t)w * pw] = 0u;
        }
        for (size_t k = gtid; k < (size_t)p.n_worlds * p.H; k += gthreads) {
            const int w = (int)(k / p.H);
            rows_of(p, p.t[w] + 1, w)[k - (size_t)w * p.H] = 0;
        }
        for (size_t w = gtid; w < (size_t)p.n_worlds; w += gthreads) {
            const int64_t tw = p.t[w];
            *count_of(p, tw + 1, (int)w) = 0;
            p.n_win[w] = 0;
            sim_step_record *nxt = record_of(p, tw + 1, (int)w);
            *nxt = sim_step_record{};
            nxt->t = tw + 1;
        }
    }
    if (with_mutation) mutate_phase(p, interleaved_gtid(), (size_t)gridDim.x * blockDim.x);

    int acc_w = -1;
    unsigned long long acc_nnz = 0ull, acc_ties = 0ull;
    for (long base = 0; base < total; base += per_round) {
        // consecutive agents go to different CTAs so a small population spreads over all SMs
        const long v = base + (long)(wib * AG + grp) * gridDim.x + blockIdx.x;
        const bool in_range = v < total;
        const int w = in_range ? (int)(v / p.S) : 0;
        const int i = in_range ? (int)(v - (long)w * p.S) : 0;
        const int64_t t = p.t[w];
        const bool active = in_range && i < *count_of(p, t, w);
        if (!__any_sync(FULL, active)) continue;
        const int slot = active ? list_of(p, t, w)[i] : 0;
        const size_t gs = (size_t)w * p.S + slot;
        // a child of the previous step whose weights are being written in this kernel
        bool fresh = false;
        if (with_mutation && active && p.mut_pending[w]) {
            const int b = i - p.newborn_base[w];
            if (b >= 0 && b < p.n_births[w]) {
                fresh = true;
                if (k == 0) mutate_wait(p, w, b);
            }
        }
        __syncwarp();

        // ---- a2: observation bitmask (channel 0 = R' after regrowth, 1 = O_t incl. self)
        uint64_t m_lo = 0ull, m_hi = 0ull;
        int cellv = 0, y = 0, x = 0;
        if (active) {
            cellv = p.cell[gs];
            y = cellv / p.W;
            x = cellv - y * p.W;
            const uint32_t *Rn = plane_next(p, t) + (size_t)w * plane_words(p);
            const uint32_t *O = p.occ + (size_t)w * plane_words(p);
            const int wd = 2 * p.r + 1;
            for (int ch = 0; ch < 2; ++ch) {
                const uint32_t *pl = ch ? O : Rn;
                for (int row = 0; row < wd; ++row) {
                    const int yy = y - p.r + row;
                    if (yy < 0 || yy >= p.H) continue;
                    const uint64_t bits = row_bits(pl + (size_t)yy * p.WW, p.WW, x - p.r, wd);
                    const int pos = ch * wd * wd + row * wd;
                    if (pos < 64) {
                        m_lo |= bits << pos;
                        if (pos + wd > 64) m_hi |= bits >> (64 - pos);
                    } else {
                        m_hi |= bits << (pos - 64);
                    }
                }
            }
        }

        // ---- a3: LSTM
        const float *Wa = p.weights + gs * (size_t)p.Pd;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        uint64_t r_lo = m_lo, r_hi = m_hi;
        while (__any_sync(FULL, (r_lo | r_hi) != 0ull)) {
            float4 vv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int idx = -1;
                if (r_lo) {
                    idx = __ffsll((long long)r_lo) - 1;
                    r_lo &= r_lo - 1;
                } else if (r_hi) {
                    idx = 64 + __ffsll((long long)r_hi) - 1;
                    r_hi &= r_hi - 1;
                }
                vv[u] = idx >= 0 ? ld_weights4(Wa + ((size_t)idx * HD + k) * 4, fresh) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc.x += vv[u].x;
                acc.y += vv[u].y;
                acc.z += vv[u].z;
                acc.w += vv[u].w;
            }
        }
        const float hk = active ? p.h[gs * HD + k] : 0.f;
        const float ck = active ? p.c[gs * HD + k] : 0.f;
        const float *Whh = Wa + p.off_hh;
#pragma unroll
        for (int j0 = 0; j0 < HD; j0 += UH) {
            float4 vv[UH];
#pragma unroll
            for (int u = 0; u < UH; ++u)
                vv[u] = active ? ld_weights4(Whh + ((j0 + u) * HD + k) * 4, fresh) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < UH; ++u) {
                const float hj = __shfl_sync(FULL, hk, j0 + u, G);
                acc.x = fmaf(hj, vv[u].x, acc.x);
                acc.y = fmaf(hj, vv[u].y, acc.y);
                acc.z = fmaf(hj, vv[u].z, acc.z);
                acc.w = fmaf(hj, vv[u].w, acc.w);
            }
        }
        const float4 bb = active ? ld_weights4(Wa + p.off_b + k * 4, fresh) : make_float4(0.f, 0.f, 0.f, 0.f);
        acc.x += bb.x;
        acc.y += bb.y;
        acc.z += bb.z;
        acc.w += bb.w;
        const float ig = sigmoidf_acc(acc.x);
        const float fg = sigmoidf_acc(acc.y);
        const float gg = tanhf(acc.z);
        const float og = sigmoidf_acc(acc.w);
        const float cn = fg * ck + ig * gg;
        const float hn = og * tanhf(cn);

        // linear head: 5 group reductions
        float lg[5];
#pragma unroll
        for (int a = 0; a < 5; ++a) {
            float s = active ? ld_weight(Wa + p.off_out + a * HD + k, fresh) * hn : 0.f;
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o, G);
            lg[a] = s + (active ? ld_weight(Wa + p.off_bout + a, fresh) : 0.f);
        }

        if (active) {
            p.h[gs * HD + k] = hn;
            p.c[gs * HD + k] = cn;
            bool bad = !isfinite(hn) || !isfinite(cn);
            if (k == 0) {
                int best = 0;
                float bestv = lg[0];
#pragma unroll
                for (int a = 1; a < 5; ++a)
                    if (lg[a] > bestv) {
                        bestv = lg[a];
                        best = a;
                    }
                double second = -INFINITY;
#pragma unroll
                for (int a = 0; a < 5; ++a) {
                    if (a != best && (double)lg[a] > second) second = (double)lg[a];
                    bad = bad || !isfinite(lg[a]);
                    p.logits[gs * LOGIT_STRIDE + a] = lg[a];
                }
                // per-lane accumulation of the world's counters, flushed on world change
                if (w != acc_w) {
                    flush_counters(p, acc_w, acc_nnz, acc_ties);
                    acc_w = w;
                }
                acc_ties += ((double)bestv - second < 1e-4) ? 1ull : 0ull;
                acc_nnz += (unsigned long long)(__popcll(m_lo) + __popcll(m_hi));
                int act = best;
                if (*p.forced_on) {
                    const uint8_t f = p.forced[gs];
                    if (f != 255) act = f;
                }
                p.last_action[gs] = (uint8_t)act;
                int tg = -1;
                unsigned long long key = 0ull;
                if (act != 0) {
                    const int ty = y + kDY[act], tx = x + kDX[act];
                    if (ty >= 0 && ty < p.H && tx >= 0 && tx < p.W) {
                        const int tc = ty * p.W + tx;
                        const uint32_t *O = p.occ + (size_t)w * plane_words(p);
                        if (!get_bit(O, p, tc)) {
                            const uint4 d = draw4(p.seeds[w], PURPOSE_MOVE, (uint32_t)t, (uint32_t)cellv, 0u);
                            key = ((unsigned long long)d.x << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)cellv);
                            atomicMax(p.claim + (size_t)w * HW + tc, key);
                            tg = tc;
                        }
                    }
                }
                p.mrec[(size_t)w * p.S + i] = make_int4(slot, cellv, tg, (int)(uint32_t)(key >> 32));
            }
            if (bad) *reinterpret_cast<volatile int32_t *>(p.nonfinite) = 1;
        }
    }
    flush_counters(p, acc_w, acc_nnz, acc_ties);
}

cudaError_t policy_occupancy(int hidden, int threads, int *blocks_per_sm) {
    switch (hidden) {
        case 4: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_policy<4>, threads, 0);
        case 8: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_policy<8>, threads, 0);
        case 16: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_policy<16>, threads, 0);
        case 32: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_policy<32>, threads, 0);
        default: return cudaErrorInvalidValue;
    }
}

template <typename Kernel, typename... Args>
cudaError_t launch_coop(Kernel kernel, int blocks, int threads, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

cudaError_t launch_policy(const DevParams &p, const LaunchCfg &lc, int with_mutation, cudaStream_t s) {
    switch (p.Hd) {
        case 4: return launch_coop(k_policy<4>, lc.policy_blocks, lc.policy_threads, s, p, with_mutation);
        case 8: return launch_coop(k_policy<8>, lc.policy_blocks, lc.policy_threads, s, p, with_mutation);
        case 16: return launch_coop(k_policy<16>, lc.policy_blocks, lc.policy_threads, s, p, with_mutation);
        case 32: return launch_coop(k_policy<32>, lc.policy_blocks, lc.policy_threads, s, p, with_mutation);
        default: return cudaErrorInvalidValue;
    }
}

// ----------------------------------------------------------- standalone phase kernels
__global__ void __launch_bounds__(256) k_regrow(DevParams p, int ahead) {
    regrow_phase(p, ahead, interleaved_gtid(), (size_t)gridDim.x * blockDim.x);
}

__global__ void __launch_bounds__(256) k_move(DevParams p) {
    move_phase(p, interleaved_gtid(), (size_t)gridDim.x * blockDim.x);
}

__global__ void __launch_bounds__(256) k_birth_claim(DevParams p) {
    birth_claim_phase(p, interleaved_gtid(), (size_t)gridDim.x * blockDim.x);
}

constexpr int RANK_THREADS = 1024;
__global__ void __launch_bounds__(RANK_THREADS) k_birth_rank(DevParams p) {
    __shared__ uint32_t scratch[RANK_THREADS / 32 + 1];
    __shared__ int2 rowq[RANK_THREADS];
    for (int w = blockIdx.x; w < p.n_worlds; w += gridDim.x) birth_rank_world<RANK_THREADS>(p, w, scratch, rowq);
}

__global__ void __launch_bounds__(256) k_mutate(DevParams p) {
    mutate_phase(p, interleaved_gtid(), (size_t)gridDim.x * blockDim.x);
}

__global__ void k_clear_pending(DevParams p) {
    for (int w = threadIdx.x; w < p.n_worlds; w += blockDim.x) p.mut_pending[w] = 0;
}

// ------------------------------------------------------------------------ k_post
// a4 move/consume/physiology/death | barrier | a1 regrowth of step t+1 (needs only R'' of
// step t) + a5 birth candidates and claimed cells | barrier | a5 rank, winners, placement,
// counters, t += 1.  (The children's weights are written by the next k_policy.)
constexpr int POST_THREADS = 512;
constexpr int POST_BARRIERS = 2;
__global__ void __launch_bounds__(POST_THREADS) k_post(DevParams p, unsigned long long *bar) {
    __shared__ uint32_t scratch[POST_THREADS / 32 + 1];
    __shared__ int2 rowq[POST_THREADS];
    // warp-interleaved global index: consecutive warps of work land on different blocks
    // (SMs), so the per-item dependency chains of every phase run on all 148 SMs at once
    const size_t gtid = interleaved_gtid();
    const size_t gthreads = (size_t)gridDim.x * blockDim.x;
    unsigned long long target = grid_sync_base(bar, POST_BARRIERS);
    // phase clock: block 0 accumulates the time between barriers (as seen by block 0)
    const bool clk = blockIdx.x == 0 && threadIdx.x == 0;
    uint64_t t0 = clk ? globaltimer_ns() : 0ull, t1;
    move_phase(p, gtid, gthreads);
    grid_sync(bar, target);
    if (clk) { t1 = globaltimer_ns(); atomicAdd(p.phase_ns + 0, t1 - t0); t0 = t1; }
    regrow_phase(p, 1, gtid, gthreads);
    birth_claim_phase(p, gtid, gthreads);
    grid_sync(bar, target);
    if (clk) { t1 = globaltimer_ns(); atomicAdd(p.phase_ns + 1, t1 - t0); t0 = t1; }
    for (int w = blockIdx.x; w < p.n_worlds; w += gridDim.x) birth_rank_world<POST_THREADS>(p, w, scratch, rowq);
    if (clk) {
        t1 = globaltimer_ns();
        atomicAdd(p.phase_ns + 2, t1 - t0);
        grid_sync_done(bar);
    }
}

// --------------------------------------------------------------------------- launchers
cudaError_t launch_regrow(const DevParams &p, int ahead, cudaStream_t s) {
    const int real_words = (p.W + 31) >> 5;
    const size_t items = (size_t)p.H * real_words * p.n_worlds;
    size_t blocks = (items + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_regrow<<<(unsigned)blocks, 256, 0, s>>>(p, ahead);
    return cudaGetLastError();
}

cudaError_t launch_move(const DevParams &p, const LaunchCfg &lc, cudaStream_t s) {
    if (p.S == 0) return cudaSuccess;
    k_move<<<lc.agent_blocks, lc.agent_threads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_birth_claim(const DevParams &p, const LaunchCfg &lc, cudaStream_t s) {
    if (p.S == 0) return cudaSuccess;
    k_birth_claim<<<lc.agent_blocks, lc.agent_threads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_birth_rank(const DevParams &p, cudaStream_t s) {
    k_birth_rank<<<p.n_worlds, RANK_THREADS, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_mutate(const DevParams &p, const LaunchCfg &lc, cudaStream_t s) {
    if (p.S == 0) return cudaSuccess;
    k_mutate<<<lc.post_blocks, 256, 0, s>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_clear_pending<<<1, 64, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t post_occupancy(int *blocks_per_sm) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_post, POST_THREADS, 0);
}

cudaError_t launch_post(const DevParams &p, const LaunchCfg &lc, unsigned long long *bar, cudaStream_t s) {
    return launch_coop(k_post, lc.post_blocks, POST_THREADS, s, p, bar);
}

}  // namespace eco
