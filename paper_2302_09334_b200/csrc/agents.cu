// agents.cu — per-agent kernels of the world step:
//   K2 k_policy      observation gather + per-agent LSTM + linear head + argmax + move claim
//                    (step rows a2, a3 and the claim half of a4)
//   K3 k_move        claim resolution, movement, consumption, physiology, death (a4, a5)
//   K3b k_birth_claim lazy claim reset, birth candidate cell and birth claim (a5)
#include "sim_internal.cuh"

namespace eco {

__device__ __constant__ int kDY[5] = {0, -1, 1, 0, 0};  // stay, N, S, E, W (R13)
__device__ __constant__ int kDX[5] = {0, 0, 0, 1, -1};

// streaming 16-B load of per-agent weights: read once per step, no reuse inside the
// step, so keep them out of L1 (L2 still serves re-reads across steps when they fit).
__device__ __forceinline__ float4 ld_weights4(const float *ptr) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(ptr));
    return v;
}

__device__ __forceinline__ float sigmoidf_acc(float z) { return 1.0f / (1.0f + expf(-z)); }

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
template <int HD>
__global__ void __launch_bounds__(256) k_policy(DevParams p) {
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

    // housekeeping for the later phases of this step: the survivor list of step t+1 and
    // the winner counters start at 0; the birth bitmap of parity t+1 (used by step t-1)
    // is cleared for step t+1.
    {
        const size_t gtid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
        const size_t gthreads = (size_t)gridDim.x * blockDim.x;
        const size_t pw = plane_words(p);
        for (size_t k = gtid; k < (size_t)p.n_worlds * pw; k += gthreads) {
            const int w = (int)(k / pw);
            bbits_of(p, p.t[w] + 1, w)[k - (size_t)w * pw] = 0u;
        }
        for (size_t w = gtid; w < (size_t)p.n_worlds; w += gthreads) {
            *count_of(p, p.t[w] + 1, (int)w) = 0;
            p.n_win[w] = 0;
        }
    }

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
                vv[u] = idx >= 0 ? ld_weights4(Wa + ((size_t)idx * HD + k) * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
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
                vv[u] = active ? ld_weights4(Whh + ((j0 + u) * HD + k) * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < UH; ++u) {
                const float hj = __shfl_sync(FULL, hk, j0 + u, G);
                acc.x = fmaf(hj, vv[u].x, acc.x);
                acc.y = fmaf(hj, vv[u].y, acc.y);
                acc.z = fmaf(hj, vv[u].z, acc.z);
                acc.w = fmaf(hj, vv[u].w, acc.w);
            }
        }
        const float4 bb = active ? ld_weights4(Wa + p.off_b + k * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
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
            float s = active ? __ldg(Wa + p.off_out + a * HD + k) * hn : 0.f;
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o, G);
            lg[a] = s + (active ? __ldg(Wa + p.off_bout + a) : 0.f);
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
                sim_step_record *rec = record_of(p, t, w);
                if ((double)bestv - second < 1e-4)
                    atomicAdd(reinterpret_cast<unsigned long long *>(&rec->near_ties), 1ull);
                atomicAdd(reinterpret_cast<unsigned long long *>(&rec->obs_nnz),
                          (unsigned long long)(__popcll(m_lo) + __popcll(m_hi)));
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
                p.target[gs] = tg;
                p.mkey[gs] = key;
            }
            if (bad) *reinterpret_cast<volatile int32_t *>(p.nonfinite) = 1;
        }
    }
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

cudaError_t launch_policy(const DevParams &p, const LaunchCfg &lc, cudaStream_t s) {
    if (p.S == 0) return cudaSuccess;
    switch (p.Hd) {
        case 4: k_policy<4><<<lc.policy_blocks, lc.policy_threads, 0, s>>>(p); break;
        case 8: k_policy<8><<<lc.policy_blocks, lc.policy_threads, 0, s>>>(p); break;
        case 16: k_policy<16><<<lc.policy_blocks, lc.policy_threads, 0, s>>>(p); break;
        case 32: k_policy<32><<<lc.policy_blocks, lc.policy_threads, 0, s>>>(p); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// --------------------------------------------------------------------------- K3 move
// a4 + a5 (death): an agent moves iff it holds the max key on its target (R14); every
// live agent eats the resource under its final cell; fixed-point energy
// e += gain*ate - decay, age += 1, repr = e > thr ? repr+1 : 0 (R16, R17, R19); death
// iff e <= 0 (cause energy) or age > max_age (cause age) (R18).  O is updated in place
// (moves, deaths) with bit atomics; distinct agents touch distinct bits.  Survivors are
// appended to the step-(t+1) list (order is irrelevant to every result).
__device__ __forceinline__ void warp_count_add(unsigned long long *dst, bool flag) {
    const unsigned m = __ballot_sync(0xffffffffu, flag);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(dst, (unsigned long long)__popc(m));
}

// iteration helper: virtual index v over [0, n_worlds*S) -> (world, list position)
struct AgentIter {
    int w, i;
    bool in_range;
};
__device__ __forceinline__ AgentIter agent_at(const DevParams &p, long v) {
    AgentIter a;
    a.in_range = v < (long)p.n_worlds * p.S;
    a.w = a.in_range ? (int)(v / p.S) : 0;
    a.i = a.in_range ? (int)(v - (long)a.w * p.S) : 0;
    return a;
}

__global__ void __launch_bounds__(256) k_move(DevParams p) {
    const long total = (long)p.n_worlds * p.S;
    const long stride = (long)gridDim.x * blockDim.x;
    const size_t HW = (size_t)p.H * p.W;
    const unsigned lane = threadIdx.x & 31;
    for (long base = (long)blockIdx.x * blockDim.x; base < total; base += stride) {
        const AgentIter it = agent_at(p, base + threadIdx.x);
        const int w = it.w;
        const int64_t t = p.t[w];
        const bool active = it.in_range && it.i < *count_of(p, t, w);
        bool ate = false, died_e = false, died_a = false, survive = false;
        int slot = 0;
        if (active) {
            slot = list_of(p, t, w)[it.i];
            const size_t gs = (size_t)w * p.S + slot;
            uint32_t *O = p.occ + (size_t)w * plane_words(p);
            uint32_t *Rn = plane_next(p, t) + (size_t)w * plane_words(p);
            int cellv = p.cell[gs];
            const int tg = p.target[gs];
            uint32_t bit;
            if (tg >= 0 && p.claim[(size_t)w * HW + tg] == p.mkey[gs]) {
                atomicAnd(word_ptr(O, p, cellv, bit), ~bit);
                atomicOr(word_ptr(O, p, tg, bit), bit);
                cellv = tg;
                p.cell[gs] = tg;
            }
            uint32_t *rw = word_ptr(Rn, p, cellv, bit);
            if (*reinterpret_cast<volatile uint32_t *>(rw) & bit) {
                atomicAnd(rw, ~bit);
                ate = true;
            }
            p.ate[gs] = ate ? 1 : 0;
            long long e = (long long)p.energy[gs] + (ate ? (long long)p.e_gain : 0ll) - (long long)p.e_decay;
            if (p.e_max != 0x7fffffff && e > p.e_max) e = p.e_max;
            const int en = (int)e;
            const int ag = p.age[gs] + 1;
            p.energy[gs] = en;
            p.age[gs] = ag;
            p.repr[gs] = en > p.e_repr_gt ? p.repr[gs] + 1 : 0;
            if (en <= p.e_death_le) died_e = true;
            else if (ag > p.max_age) died_a = true;
            if (died_e || died_a) {
                p.alive[gs] = 0;
                atomicAnd(word_ptr(O, p, cellv, bit), ~bit);
                atomicAnd(p.alive_bits + (size_t)w * p.SW + (slot >> 5), ~(1u << (slot & 31)));
            } else {
                survive = true;
            }
        }
        const int w0 = __shfl_sync(0xffffffffu, w, 0);
        if (__all_sync(0xffffffffu, w == w0)) {
            sim_step_record *rec = record_of(p, p.t[w0], w0);
            warp_count_add(reinterpret_cast<unsigned long long *>(&rec->eaten), ate);
            warp_count_add(reinterpret_cast<unsigned long long *>(&rec->deaths_energy), died_e);
            warp_count_add(reinterpret_cast<unsigned long long *>(&rec->deaths_age), died_a);
            const unsigned m = __ballot_sync(0xffffffffu, survive);
            int pos0 = 0;
            if (lane == 0 && m) pos0 = atomicAdd(count_of(p, p.t[w0] + 1, w0), __popc(m));
            pos0 = __shfl_sync(0xffffffffu, pos0, 0);
            if (survive) list_of(p, t + 1, w)[pos0 + __popc(m & ((1u << lane) - 1u))] = slot;
        } else {
            sim_step_record *rec = record_of(p, t, w);
            if (ate) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->eaten), 1ull);
            if (died_e) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deaths_energy), 1ull);
            if (died_a) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deaths_age), 1ull);
            if (survive) list_of(p, t + 1, w)[atomicAdd(count_of(p, t + 1, w), 1)] = slot;
        }
    }
}

cudaError_t launch_move(const DevParams &p, const LaunchCfg &lc, cudaStream_t s) {
    if (p.S == 0) return cudaSuccess;
    k_move<<<lc.agent_blocks, lc.agent_threads, 0, s>>>(p);
    return cudaGetLastError();
}

// -------------------------------------------------------------------- K3b birth claim
// Lazy reset of this step's move claims (every claimant clears its own target; safe
// because K3 has finished reading them).  Then every live parent with repr >= T_repr
// picks the first cell of a Philox-rotated (N, S, E, W) order that is
// in-grid, agent-free after moves/deaths (O'') and resource-free after consumption (R'')
// (R21), and records the direction on its own cell (bdir; NO_DIR when it has none).
__global__ void __launch_bounds__(256) k_birth_claim(DevParams p) {
    const long total = (long)p.n_worlds * p.S;
    const long stride = (long)gridDim.x * blockDim.x;
    const size_t HW = (size_t)p.H * p.W;
    for (long base = (long)blockIdx.x * blockDim.x; base < total; base += stride) {
        const AgentIter it = agent_at(p, base + threadIdx.x);
        const int w = it.w;
        const int64_t t = p.t[w];
        const bool active = it.in_range && it.i < *count_of(p, t, w);
        bool no_cell = false;
        if (active) {
            const int slot = list_of(p, t, w)[it.i];
            const size_t gs = (size_t)w * p.S + slot;
            const int tg = p.target[gs];
            if (tg >= 0) p.claim[(size_t)w * HW + tg] = 0ull;
            if (p.alive[gs]) {
                const int cellv = p.cell[gs];
                uint8_t dir = NO_DIR;
                if (p.repr[gs] >= p.repr_steps) {
                    const uint32_t *O = p.occ + (size_t)w * plane_words(p);
                    const uint32_t *Rn = plane_next(p, t) + (size_t)w * plane_words(p);
                    const int y = cellv / p.W, x = cellv - y * p.W;
                    const uint4 d = draw4(p.seeds[w], PURPOSE_BIRTH, (uint32_t)t, (uint32_t)cellv, 0u);
                    const int s0 = (int)(d.x & 3u);
                    for (int kk = 0; kk < 4; ++kk) {
                        const int dd = (s0 + kk) & 3;
                        const int cy = y + dir_dy(dd), cx = x + dir_dx(dd);
                        if (cy < 0 || cy >= p.H || cx < 0 || cx >= p.W) continue;
                        const int c = cy * p.W + cx;
                        if (get_bit(O, p, c) || get_bit(Rn, p, c)) continue;
                        dir = (uint8_t)dd;
                        break;
                    }
                    no_cell = dir == NO_DIR;
                }
                p.bdir[(size_t)w * HW + cellv] = dir;
            }
        }
        if (no_cell)
            atomicAdd(reinterpret_cast<unsigned long long *>(&record_of(p, t, w)->deferred_no_cell), 1ull);
    }
}

cudaError_t launch_birth_claim(const DevParams &p, const LaunchCfg &lc, cudaStream_t s) {
    if (p.S == 0) return cudaSuccess;
    k_birth_claim<<<lc.agent_blocks, lc.agent_threads, 0, s>>>(p);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------- K3c birth win
// Claim resolution without atomics: the parent on cell p whose candidate is c wins iff
// its key (BIRTH w1 << 32 | ~p) exceeds the key of every other live parent adjacent to c
// that chose c (read from bdir of c's other neighbours, valid where O'' is set).  The
// winner marks c in the birth bitmap and records itself as c's parent.
__device__ __forceinline__ unsigned long long birth_key(uint64_t seed, int64_t t, int cellv) {
    const uint4 d = draw4(seed, PURPOSE_BIRTH, (uint32_t)t, (uint32_t)cellv, 0u);
    return ((unsigned long long)d.y << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)cellv);
}

__global__ void __launch_bounds__(256) k_birth_win(DevParams p) {
    const long total = (long)p.n_worlds * p.S;
    const long stride = (long)gridDim.x * blockDim.x;
    const size_t HW = (size_t)p.H * p.W;
    for (long base = (long)blockIdx.x * blockDim.x; base < total; base += stride) {
        const AgentIter it = agent_at(p, base + threadIdx.x);
        const int w = it.w;
        const int64_t t = p.t[w];
        const bool active = it.in_range && it.i < *count_of(p, t, w);
        bool win = false, lost = false;
        if (active) {
            const int slot = list_of(p, t, w)[it.i];
            const size_t gs = (size_t)w * p.S + slot;
            if (p.alive[gs]) {
                const int pc = p.cell[gs];
                const uint8_t *bd = p.bdir + (size_t)w * HW;
                const int d = bd[pc];
                if (d != NO_DIR) {
                    const uint32_t *O = p.occ + (size_t)w * plane_words(p);
                    const int py = pc / p.W, px = pc - py * p.W;
                    const int cy = py + dir_dy(d), cx = px + dir_dx(d);
                    const int c = cy * p.W + cx;
                    const uint64_t seed = p.seeds[w];
                    const unsigned long long kp = birth_key(seed, t, pc);
                    win = true;
                    for (int dq = 0; dq < 4 && win; ++dq) {
                        const int qy = cy + dir_dy(dq), qx = cx + dir_dx(dq);
                        if (qy < 0 || qy >= p.H || qx < 0 || qx >= p.W) continue;
                        const int q = qy * p.W + qx;
                        if (q == pc || !get_bit(O, p, q) || bd[q] != (uint8_t)(dq ^ 1)) continue;
                        if (birth_key(seed, t, q) > kp) win = false;
                    }
                    if (win) {
                        uint32_t bit;
                        atomicOr(word_ptr(bbits_of(p, t, w), p, c, bit), bit);
                        p.bparent[(size_t)w * HW + c] = slot;
                    } else {
                        lost = true;
                    }
                }
            }
        }
        const int w0 = __shfl_sync(0xffffffffu, w, 0);
        if (__all_sync(0xffffffffu, w == w0)) {
            const unsigned m = __ballot_sync(0xffffffffu, win);
            if ((threadIdx.x & 31) == 0 && m) atomicAdd(p.n_win + w0, __popc(m));
            warp_count_add(reinterpret_cast<unsigned long long *>(&record_of(p, p.t[w0], w0)->deferred_claim), lost);
        } else {
            if (win) atomicAdd(p.n_win + w, 1);
            if (lost) atomicAdd(reinterpret_cast<unsigned long long *>(&record_of(p, t, w)->deferred_claim), 1ull);
        }
    }
}

cudaError_t launch_birth_win(const DevParams &p, const LaunchCfg &lc, cudaStream_t s) {
    if (p.S == 0) return cudaSuccess;
    k_birth_win<<<lc.agent_blocks, lc.agent_threads, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace eco
