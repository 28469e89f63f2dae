// step.cu — the kernels of one world step (sm_100a).
//
// Graph mode (sim_step): two launches per step,
//   k_policy_half (Hd = 32)  a2 observation + a3 per-agent LSTM/head/argmax + the claim
//                 half of a4; one agent per half-warp, its weights streamed as 512-B
//                 chunks through a per-agent cp.async ring in shared memory
//   k_policy_reg  (Hd = 4, 8, 16) the same step with register loads, lane groups of Hd
//   k_post        cooperative: a4 move/consume/physiology/death | grid barrier | a5 birth
//                 candidates | barrier | a5 rank (every block), winners, placement and
//                 counters (block 0), a1 regrowth of step t+1, a5 mutation, t += 1
// (the first step after create/set_state is preceded by a standalone k_regrow).
// Instrumented mode (sim_step_timed): the same phases as separate kernels, timed one by one.
#include <type_traits>

#include "phases.cuh"

// The Hd = 32 policy kernel is k_policy_half.  Discarded variants (a per-warp TMA/cp.async
// pipeline, register streaming, one warp per agent with a 12-chunk ring, persistent warps
// streaming across agents) are recorded with their timings in DESIGN.md §6 and git history.
// k_policy_half: bulk L2 prefetch of each agent's W_hh|b|W_out block and active columns
// (1), of the block only (2), none (0: measured fastest, 34 vs 43 us with 1)
#ifndef ECO_POLICY_PREFETCH
#define ECO_POLICY_PREFETCH 0
#endif

namespace eco {


__device__ __constant__ int kDY[5] = {0, -1, 1, 0, 0};  // stay, N, S, E, W (R13)
__device__ __constant__ int kDX[5] = {0, 0, 0, 1, -1};

__device__ __forceinline__ float sigmoidf_acc(float z) { return 1.0f / (1.0f + expf(-z)); }

template <bool SHARD = false>
__device__ __forceinline__ void flush_counters(const DevParams &p, int w, unsigned long long nnz,
                                               unsigned long long ties) {
    if (w < 0) return;
    if (SHARD) {  // sharded: summed over the ranks by the exchange, added in k_post
        if (nnz) atomicAdd(p.pol_ctr, nnz);
        if (ties) atomicAdd(p.pol_ctr + 1, ties);
        return;
    }
    sim_step_record *rec = record_of(p, p.t[w], w);
    if (nnz) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->obs_nnz), nnz);
    if (ties) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->near_ties), ties);
}

// Per-lane accumulation of the policy counters of a world (flushed on world change/end).
struct PolicyCounters {
    int w = -1;
    unsigned long long nnz = 0ull, ties = 0ull;
    __device__ __forceinline__ void add(const DevParams &p, int ww, unsigned long long n, bool tie) {
        if (ww != w) {
            flush_counters(p, w, nnz, ties);
            w = ww;
            nnz = ties = 0ull;
        }
        nnz += n;
        ties += tie ? 1ull : 0ull;
    }
    __device__ __forceinline__ void flush(const DevParams &p) { flush_counters(p, w, nnz, ties); }
};

// ------------------------------------------------------------- a2 observation mask
// The (2r+1)^2 x 2 window of (R' after regrowth, O_t incl. self) around (y, x) as a
// bitmask: input index ch*(2r+1)^2 + row*(2r+1) + col (R10, R11).
// Lane l < 2(2r+1) fetches one row of one channel; the rows are OR-reduced over the
// warp (or the lane group `gmask`), so every lane of the group ends with the full mask.
__device__ __forceinline__ void obs_mask(const DevParams &p, int w, int64_t t, int y, int x, int l, int stride,
                                         unsigned gmask, uint64_t &m_lo, uint64_t &m_hi) {
    const int wd = 2 * p.r + 1;
    uint64_t lo = 0ull, hi = 0ull;
    for (int q = l; q < 2 * wd; q += stride) {
        const int ch = q / wd, row = q - ch * wd;
        const int yy = y - p.r + row;
        if (yy < 0 || yy >= p.H) continue;
        const uint32_t *pl = ch ? p.occ + (size_t)w * plane_words(p) : plane_next(p, t) + (size_t)w * plane_words(p);
        const uint64_t bits = row_bits(pl + (size_t)yy * p.WW, p.WW, x - p.r, wd);
        const int pos = ch * wd * wd + row * wd;
        if (pos < 64) {
            lo |= bits << pos;
            if (pos + wd > 64) hi |= bits >> (64 - pos);
        } else {
            hi |= bits << (pos - 64);
        }
    }
    const uint32_t a0 = __reduce_or_sync(gmask, (uint32_t)lo), a1 = __reduce_or_sync(gmask, (uint32_t)(lo >> 32));
    const uint32_t a2 = __reduce_or_sync(gmask, (uint32_t)hi), a3 = __reduce_or_sync(gmask, (uint32_t)(hi >> 32));
    m_lo = ((uint64_t)a1 << 32) | a0;
    m_hi = ((uint64_t)a3 << 32) | a2;
}

// The action (the policy's, or the forced one of the test hook), last_action, and the move
// claim of a4: a valid non-stay move posts (MOVE w0 << 32 | ~cell) with atomicMax on
// claim[target] (R14); a move off the grid is blocked (R15) or marks the lethal wall.
// occ_in_window(act) answers "is the target in O_t" from the policy's own window (r >= 1).
template <bool SHARD = false, typename OccFn>
__device__ __forceinline__ void agent_commit(const DevParams &p, int w, int i, int slot, size_t gs, int64_t t,
                                             int cellv, int act, int forced_on, OccFn occ_in_window) {
    if (forced_on) {
        p.own_act[gs] = (uint8_t)act;  // test hook (sim_get_policy_actions)
        const uint8_t f = p.forced[gs];
        if (f != 255) act = f;
    }
    p.last_action[gs] = (uint8_t)act;
    int tg = -1;
    unsigned long long key = 0ull;
    if (act != 0) {
        const int y = row_of(p, cellv), x = cellv - y * p.W;
        const int ty = y + kDY[act], tx = x + kDX[act];
        if (p.lethal_walls && !(ty >= 0 && ty < p.H && tx >= 0 && tx < p.W)) tg = WALL_TARGET;
        if (p.coloc) {  // co-location (R43): an in-grid move always succeeds, no claim
            if (ty >= 0 && ty < p.H && tx >= 0 && tx < p.W) tg = ty * p.W + tx;
        } else if (ty >= 0 && ty < p.H && tx >= 0 && tx < p.W) {
            const int tc = ty * p.W + tx;
            const bool occupied = p.r >= 1 ? occ_in_window(act)
                                           : get_bit(p.occ + (size_t)w * plane_words(p), p, tc) != 0u;
            if (!occupied) {
                const uint4 d = draw4(p.seeds[w], PURPOSE_MOVE, (uint32_t)t, (uint32_t)cellv, 0u);
                key = ((unsigned long long)d.x << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)cellv);
                if (!SHARD) atomicMax(p.claim + (size_t)w * p.H * p.W + tc, key);  // sharded: in k_post
                tg = tc;
            }
        }
    }
    const int4 mr = make_int4(slot, cellv, tg, (int)(uint32_t)(key >> 32));
    if (SHARD) p.mrec_slot[slot] = mr;  // sharded: exchanged by slot, listed in k_post
    else p.mrec[(size_t)w * p.S + i] = mr;
}

// ------------------------------------------------------------ agent epilogue (a3, a4)
// argmax (lowest index on exact ties), near-tie flag (margin < 1e-4, R28), forced action,
// stored logits/action, and the move claim of a4: a valid non-stay move posts
// (MOVE w0 << 32 | ~cell) with atomicMax on claim[target] (R14).  Called by the agent's
// group leader only.
template <bool SHARD = false>
__device__ __forceinline__ void agent_epilogue(const DevParams &p, int w, int i, int slot, size_t gs, int64_t t,
                                               int cellv, const float lg[5], uint64_t m_lo, uint64_t m_hi,
                                               int forced_on, PolicyCounters &ctr, bool &bad) {
    const unsigned nnz = (unsigned)(__popcll(m_lo) + __popcll(m_hi));
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
    ctr.add(p, w, nnz, (double)bestv - second < 1e-4);
#if ECO_GREED
    {  // greediness: a resource in the field of view (the window's resource channel, R10/R11)
        const int wd2 = (2 * p.r + 1) * (2 * p.r + 1);  // <= 49
        if (m_lo & ((1ull << wd2) - 1ull)) p.gr_seen[gs] = 1;
    }
#endif
    agent_commit<SHARD>(p, w, i, slot, gs, t, cellv, best, forced_on, [&](int act) {
        // O_t of the target: the agent channel of the window already holds it (r >= 1)
        const int wd = 2 * p.r + 1;
        const int bi = wd * wd + (p.r + kDY[act]) * wd + (p.r + kDX[act]);
        return ((bi < 64 ? (m_lo >> bi) : (m_hi >> (bi - 64))) & 1ull) != 0ull;
    });
}

// housekeeping for the later phases of this step (any policy kernel runs it): the survivor
// list of step t+1, the winner counters and the record of step t+1 (whose regrowth runs
// early, inside this step's k_post) start at 0; the claimed-cell bitmap of parity t+1
// (used by step t-1) is cleared for step t+1.
// (one thread per world: the counters and the record of step t+1)
__device__ __forceinline__ void housekeeping_world(const DevParams &p, int w) {
    const int64_t tw = p.t[w];
    *count_of(p, tw + 1, w) = 0;
    p.n_win[w] = 0;
    p.n_cand[w] = 0;
    if (p.n_ranks > 1 && w == 0) p.own_count[(tw + 1) & 1] = 0;
    sim_step_record *nxt = record_of(p, tw + 1, w);
    *nxt = sim_step_record{};
    nxt->t = tw + 1;
    if (tw % SIM_MOVE_WINDOW == SIM_MOVE_WINDOW - 1) {  // this step ends window tw/50: its bins from 0
        int32_t *hist = p.mv_hist + ((size_t)w * p.mv_cap + (size_t)((tw / SIM_MOVE_WINDOW) & (p.mv_cap - 1))) * SIM_MOVE_BINS;
        for (int b = 0; b < SIM_MOVE_BINS; ++b) hist[b] = 0;
    }
}
__device__ __forceinline__ void step_housekeeping(const DevParams &p) {
    const size_t gtid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t gthreads = (size_t)gridDim.x * blockDim.x;
    const size_t pw = plane_words(p);
    for (size_t k = gtid; k < (size_t)p.n_worlds * pw; k += gthreads) {
        const int w = (int)(k / pw);
        uint32_t *wp = bbits_of(p, p.t[w] + 1, w) + (k - (size_t)w * pw);
        uint32_t v = *wp;
        if (v) {  // the claimed cells of step t-1: clear their birth keys too
            *wp = 0u;
            const int kk = (int)(k - (size_t)w * pw), y = kk / p.WW, wx = kk - y * p.WW;
            while (v) {
                const int b = __ffs(v) - 1;
                v &= v - 1u;
                p.bkey[(size_t)w * p.H * p.W + (size_t)y * p.W + wx * 32 + b] = 0ull;
            }
        }
    }
    for (size_t w = gtid; w < (size_t)p.n_worlds; w += gthreads) housekeeping_world(p, (int)w);
}

// ------------------------------------------------------------- cp.async helpers
__device__ __forceinline__ uint32_t smem_addr(const void *ptr) {
    return (uint32_t)__cvta_generic_to_shared(ptr);
}
// 16-B global -> shared copy (LDGSTS), default L2 policy (a .L2::cache_hint operand raised
// "illegal instruction" on the B200 pool, driver 580.159)
__device__ __forceinline__ void cp_async16(void *dst, const void *src, uint64_t policy) {
    (void)policy;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}


// ============================================================ k_policy_reg (Hd < 32)
// The same step with register loads; a lane group of HD lanes per agent.
template <int HD>
__global__ void __launch_bounds__(256) k_policy_reg(DevParams p) {
    constexpr int G = HD;
    constexpr int AG = 32 / HD;
    constexpr int U = 8;
    constexpr int UH = HD < 8 ? HD : 8;
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int k = lane & (G - 1);
    const int grp = lane / G;
    const unsigned gmask = (G == 32) ? FULL : (((1u << G) - 1u) << (grp * G));
    const int wib = threadIdx.x >> 5;
    const int warps_per_block = blockDim.x >> 5;
    const long total = (long)p.n_worlds * p.S;
    const long per_round = (long)gridDim.x * warps_per_block * AG;
    step_housekeeping(p);
    PolicyCounters ctr;
    for (long base = 0; base < total; base += per_round) {
        const long v = base + (long)(wib * AG + grp) * gridDim.x + blockIdx.x;
        const bool in_range = v < total;
        const int w = in_range ? (int)(v / p.S) : 0;
        const int i = in_range ? (int)(v - (long)w * p.S) : 0;
        const int64_t t = p.t[w];
        const bool active = in_range && i < *count_of(p, t, w);
        if (!__any_sync(FULL, active)) continue;
        const int slot = active ? list_of(p, t, w)[i] : 0;
        const size_t gs = (size_t)w * p.S + slot;
        uint64_t m_lo = 0ull, m_hi = 0ull;
        int cellv = 0;
        if (active) cellv = p.cell[gs];
        {
            const int y = row_of(p, cellv), x = cellv - y * p.W;
            uint64_t lo, hi;
            obs_mask(p, w, t, y, x, active ? k : 1 << 20, G, gmask, lo, hi);
            if (active) {
                m_lo = lo;
                m_hi = hi;
            }
        }
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
                vv[u] = idx >= 0 ? __ldg(reinterpret_cast<const float4 *>(Wa + ((size_t)idx * HD + k) * 4))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
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
                vv[u] = active ? __ldg(reinterpret_cast<const float4 *>(Whh + ((j0 + u) * HD + k) * 4))
                               : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < UH; ++u) {
                const float hj = __shfl_sync(FULL, hk, j0 + u, G);
                acc.x = fmaf(hj, vv[u].x, acc.x);
                acc.y = fmaf(hj, vv[u].y, acc.y);
                acc.z = fmaf(hj, vv[u].z, acc.z);
                acc.w = fmaf(hj, vv[u].w, acc.w);
            }
        }
        const float4 bb = active ? __ldg(reinterpret_cast<const float4 *>(Wa + p.off_b + k * 4))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
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
            if (k == 0) agent_epilogue(p, w, i, slot, gs, t, cellv, lg, m_lo, m_hi, *p.forced_on, ctr, bad);
            if (bad) *reinterpret_cast<volatile int32_t *>(p.nonfinite) = 1;
        }
    }
    if (k == 0) ctr.flush(p);
}

// ------------------------------------------------------------- cp.async groups
constexpr int RING_COLS = 128;  // >= I = 2(2r+1)^2 for r <= 3 (98): compacted active-column list

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}


// ============================================================ k_policy_half (Hd = 32)
// One agent per HALF-warp, so that a launch keeps every live agent of the
// paper-scale world resident at once (4 blocks x 16 agents per SM = 9,472 >= 8,192 slots):
// no second wave, the tail is one agent's own latency.  Half-lane h owns hidden units h and
// h+16 (two float4 gate accumulators) and copies/reads their 2 x 16 B of every 512-B chunk.
// Ring: HALF_DEPTH chunks per agent (3 KB) in flight; 16 agents per block interleaved over
// the blocks (agent v = a * gridDim + block).  Column indices are compacted to bytes.
#ifndef ECO_POST_PDL
#define ECO_POST_PDL 1  // measured: 48.0 -> 47.45 us per step (2, the policy triggering early: 48.65)
#endif
#ifndef ECO_POLICY_DEEP
#define ECO_POLICY_DEEP 1
#endif
#ifndef ECO_HALF_FULLGRID
#define ECO_HALF_FULLGRID 1  // 4 blocks on every SM (592 at 8 warps): 48.0 -> 47.4 us per step
#endif
#ifndef ECO_HALF_WARPS
#define ECO_HALF_WARPS 8
#endif
constexpr int HALF_WARPS = ECO_HALF_WARPS;
constexpr int HALF_THREADS = HALF_WARPS * 32;
constexpr int HALF_AGENTS = 2 * HALF_WARPS;  // per block (16 at 8 warps)
#ifndef ECO_HALF_DEPTH
#define ECO_HALF_DEPTH 6
#endif
constexpr int HALF_DEPTH = ECO_HALF_DEPTH;
#ifndef ECO_POL_COMPACT_TILE
#define ECO_POL_COMPACT_TILE 2  // live list positions per tile of the compacted policy (2: one warp's; 16: one block's)
#endif
#ifndef ECO_POL_COMPACT_WAVES
#define ECO_POL_COMPACT_WAVES 4  // the compacted policy's grid, in waves of resident blocks
#endif
constexpr int CPT_TILE = ECO_POL_COMPACT_TILE;
static_assert(CPT_TILE >= 2 && CPT_TILE % 2 == 0 && HALF_AGENTS % CPT_TILE == 0, "whole warps per tile");
constexpr int POLICY_COMPACT_WORLDS = 512;  // worlds whose tile prefix fits the block's shared array
constexpr int HALF_SMEM = HALF_AGENTS * HALF_DEPTH * 32 * 16;  // 48 KB at depth 6 and 8 warps
// blocks per SM the smem allows (32 resident warps at depth <= 6)
constexpr int HALF_BPS = (HALF_DEPTH <= 6 ? 32 : HALF_DEPTH <= 8 ? 24 : 16) / HALF_WARPS > 0
                             ? (HALF_DEPTH <= 6 ? 32 : HALF_DEPTH <= 8 ? 24 : 16) / HALF_WARPS
                             : 1;

// P[slot] = W_hh h + b (Hd = 32) for list positions [0, n) of `list`, one agent per
// half-warp context (ctx of nctx; both halves of a warp call it together), through the same
// per-lane cp.async ring as the policy (`ring` = this context's R slots).  The sum is formed
// in the policy's order (the 32 W_hh rows by FMA, then b), so that a policy starting from P
// produces exactly the gates of one streaming W_hh itself.
// The ring runs on ACROSS a context's agents (ECO_HH_PIPE, default): an agent's 33 chunks
// are followed at once by the first chunks of the context's next agent (its slot read one
// agent ahead, its h while the current agent's last R chunks land), so R chunks stay in
// flight from the first agent's first chunk to the last agent's last — no drain, no
// dependent list -> slot -> row round trip between agents.  (Before: each agent drained the
// ring and began with that round trip, ~6.5 round trips per agent instead of 33 / R.)
#ifndef ECO_HH_PIPE
#define ECO_HH_PIPE 1
#endif
template <int R>
__device__ __forceinline__ void hh_pass(const DevParams &p, const int32_t *list, int n, int ctx, int nctx,
                                        float4 *ring) {
    constexpr int HD = 32, NHH = 32, NCH = NHH + 1;  // an agent's chunks: the 32 W_hh rows, then b
    static_assert(R >= 1 && R <= NCH, "ring depth");
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, hl = lane & 15;
    float4 *rg = ring + hl;  // slot s, unit hl: rg[s * 32]; unit hl+16: rg[s * 32 + 16]
#if ECO_HH_PIPE
    int i = ctx;
    bool active = i < n;
    if (!__any_sync(FULL, active)) return;
    auto issue = [&](int s_, const float *src, bool on) {
        if (on) {
            cp_async16(rg + s_ * 32, src, 0ull);
            cp_async16(rg + s_ * 32 + 16, src + 64, 0ull);
        }
        cp_commit();
    };
    // chunk q of the row at Wl: W_hh row q, or b
    auto chunk = [&](const float *Wl, int q) { return q < NHH ? Wl + p.off_hh + q * HD * 4 : Wl + p.off_b; };
    int slot = active ? list[i] : 0;
    bool nact = i + nctx < n;
    int nslot = nact ? list[i + nctx] : 0;
    const float *Wl = p.weights + (size_t)slot * p.Pd + hl * 4;
#pragma unroll
    for (int q = 0; q < R; ++q) issue(q, chunk(Wl, q), active);
    float hk0 = active ? p.h[(size_t)slot * HD + hl] : 0.f;
    float hk1 = active ? p.h[(size_t)slot * HD + hl + 16] : 0.f;
    int s = 0;  // the ring slot of the current agent's next chunk
    for (;;) {
        const float *Wn = p.weights + (size_t)nslot * p.Pd + hl * 4;
        float hn0 = 0.f, hn1 = 0.f;
        float4 acc0 = make_float4(0.f, 0.f, 0.f, 0.f), acc1 = acc0;
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
            cp_wait<R - 1>();
            const float4 c0 = rg[s * 32], c1 = rg[s * 32 + 16];
            if (k < NHH) {
                const float hj = __shfl_sync(FULL, k < 16 ? hk0 : hk1, k & 15, 16);
                acc0.x = fmaf(hj, c0.x, acc0.x);
                acc0.y = fmaf(hj, c0.y, acc0.y);
                acc0.z = fmaf(hj, c0.z, acc0.z);
                acc0.w = fmaf(hj, c0.w, acc0.w);
                acc1.x = fmaf(hj, c1.x, acc1.x);
                acc1.y = fmaf(hj, c1.y, acc1.y);
                acc1.z = fmaf(hj, c1.z, acc1.z);
                acc1.w = fmaf(hj, c1.w, acc1.w);
            } else {  // the bias
                acc0.x += c0.x;
                acc0.y += c0.y;
                acc0.z += c0.z;
                acc0.w += c0.w;
                acc1.x += c1.x;
                acc1.y += c1.y;
                acc1.z += c1.z;
                acc1.w += c1.w;
            }
            // refill the slot just read: this agent's chunk k + R, else the next agent's first ones
            if (k + R < NCH) issue(s, chunk(Wl, k + R), active);
            else issue(s, chunk(Wn, k + R - NCH), nact);
            if (k == NCH - R && nact) {  // the next agent's h, landing beside its first chunks
                hn0 = p.h[(size_t)nslot * HD + hl];
                hn1 = p.h[(size_t)nslot * HD + hl + 16];
            }
            s = s + 1 == R ? 0 : s + 1;
        }
        if (active) {
            float4 *P = reinterpret_cast<float4 *>(p.Pbuf + (size_t)slot * HD * 4);
            P[hl] = acc0;
            P[hl + 16] = acc1;
        }
        i += nctx;
        active = nact;
        slot = nslot;
        Wl = Wn;
        hk0 = hn0;
        hk1 = hn1;
        if (!__any_sync(FULL, active)) break;
        nact = i + nctx < n;
        nslot = nact ? list[i + nctx] : 0;  // needed NCH - R chunks from here
    }
    cp_wait<0>();
    __syncwarp();
#else
    for (int r0 = 0; r0 < n; r0 += nctx) {
        const int i = r0 + ctx;
        const bool active = i < n;
        if (!__any_sync(FULL, active)) break;
        const int slot = active ? list[i] : 0;
        const float *Wl = p.weights + (size_t)slot * p.Pd + hl * 4;
        const float *Whh = Wl + p.off_hh;
        auto issue = [&](int s_, const float *src) {
            if (active) {
                cp_async16(rg + s_ * 32, src, 0ull);
                cp_async16(rg + s_ * 32 + 16, src + 64, 0ull);
            }
            cp_commit();
        };
#pragma unroll
        for (int q = 0; q < R; ++q) issue(q, Whh + q * HD * 4);
        const float hk0 = active ? p.h[(size_t)slot * HD + hl] : 0.f;
        const float hk1 = active ? p.h[(size_t)slot * HD + hl + 16] : 0.f;
        float4 acc0 = make_float4(0.f, 0.f, 0.f, 0.f), acc1 = acc0;
#pragma unroll
        for (int k = 0; k < NHH; ++k) {
            cp_wait<R - 1>();
            const float4 c0 = rg[(k % R) * 32], c1 = rg[(k % R) * 32 + 16];
            const float hj = __shfl_sync(FULL, k < 16 ? hk0 : hk1, k & 15, 16);
            acc0.x = fmaf(hj, c0.x, acc0.x);
            acc0.y = fmaf(hj, c0.y, acc0.y);
            acc0.z = fmaf(hj, c0.z, acc0.z);
            acc0.w = fmaf(hj, c0.w, acc0.w);
            acc1.x = fmaf(hj, c1.x, acc1.x);
            acc1.y = fmaf(hj, c1.y, acc1.y);
            acc1.z = fmaf(hj, c1.z, acc1.z);
            acc1.w = fmaf(hj, c1.w, acc1.w);
            if (k + R < NHH) issue(k % R, Whh + (k + R) * HD * 4);
            else if (k + R == NHH) issue(k % R, Wl + p.off_b);
            else cp_commit();
        }
        cp_wait<R - 1>();  // the bias (chunk NHH, slot NHH % R)
        {
            const float4 c0 = rg[(NHH % R) * 32], c1 = rg[(NHH % R) * 32 + 16];
            acc0.x += c0.x;
            acc0.y += c0.y;
            acc0.z += c0.z;
            acc0.w += c0.w;
            acc1.x += c1.x;
            acc1.y += c1.y;
            acc1.z += c1.z;
            acc1.w += c1.w;
        }
        cp_wait<0>();
        if (active) {
            float4 *P = reinterpret_cast<float4 *>(p.Pbuf + (size_t)slot * HD * 4);
            P[hl] = acc0;
            P[hl + 16] = acc1;
        }
        __syncwarp();
    }
#endif
}

// P of every live agent of step t (after create / set_state / instrumented steps), one
// half-warp per agent; no children pending afterwards.
__global__ void __launch_bounds__(HALF_THREADS, HALF_BPS) k_prepare_p(DevParams p) {
    extern __shared__ __align__(1024) float4 half_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ag = warp * 2 + (lane >> 4);
    const int64_t t = p.t[0];
    hh_pass<HALF_DEPTH>(p, list_of(p, t, 0), *count_of(p, t, 0), ag * gridDim.x + blockIdx.x, gridDim.x * HALF_AGENTS,
            half_smem + (ag * HALF_DEPTH) * 32);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *p.p_children = 0;
        *p.own_surv = 0x7fffffff;  // sharded: every own agent has its P row
    }
}

// Banded mode: P rows of list_of(snap[0])[0, snap[1]) — the agents of the step in progress,
// snapshotted right after the band's policy (band_snap0) — on a second stream while
// the rest of the step runs; the children placed later have none (p_children, set by the rank).
__global__ void __launch_bounds__(HALF_THREADS, HALF_BPS) k_prepare_p_snap(DevParams p, const int64_t *snap) {
    extern __shared__ __align__(1024) float4 half_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ag = warp * 2 + (lane >> 4);
    hh_pass<HALF_DEPTH>(p, list_of(p, snap[0], 0), (int)snap[1], ag * gridDim.x + blockIdx.x, gridDim.x * HALF_AGENTS,
                        half_smem + (ag * HALF_DEPTH) * 32);
}

// Banded mode: P rows of the slots list[0, *n) (the step's arrivals from the neighbour bands)
__global__ void __launch_bounds__(HALF_THREADS, HALF_BPS) k_prepare_p_list(DevParams p, const int32_t *list,
                                                                           const int32_t *n) {
    extern __shared__ __align__(1024) float4 half_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ag = warp * 2 + (lane >> 4);
    hh_pass<HALF_DEPTH>(p, list, *n, ag * gridDim.x + blockIdx.x, gridDim.x * HALF_AGENTS, half_smem + (ag * HALF_DEPTH) * 32);
}

#ifdef ECO_TIMELINE
// diagnostic build: per step t (ring of 1024), the policy's first block start and last block
// end and k_post's, as globaltimer ns in phase_ns[16 + (t % 1024) * 4 + {0..3}] (starts
// stored inverted: atomicMax of ~x keeps the earliest); the host zeroes the ring
__device__ __forceinline__ void timeline_mark(const DevParams &p, int k, unsigned long long v, int64_t t = -1) {
    if (t < 0) t = p.t[0];
    atomicMax(p.phase_ns + 16 + (size_t)(t & 1023) * 4 + k, v);
}
#endif

// SHARD = false compiles the sharding branches out, so the unsharded kernels keep their code
// (a local DevParams copy to fold n_ranks costs 3 us in this kernel: measured).
template <bool SHARD, bool SPLIT = false, bool COMPACT = false>
__global__ void __launch_bounds__(HALF_THREADS, HALF_BPS) k_policy_half(DevParams p) {
    static_assert(!(SHARD && COMPACT), "the compacted mapping is for unsharded handles");
    constexpr int HD = 32, NHH = 32, QB = 32, Q0 = 33, R = HALF_DEPTH;
    constexpr unsigned FULL = 0xffffffffu;
    extern __shared__ __align__(1024) float4 half_smem[];  // [HALF_AGENTS][R][32 units]
    __shared__ uint8_t s_col[HALF_AGENTS][RING_COLS];
    __shared__ int s_w[HALF_AGENTS];
    __shared__ unsigned long long s_nnz[HALF_AGENTS], s_ties[HALF_AGENTS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int half = lane >> 4, hl = lane & 15;
    const int ag = warp * 2 + half;                 // agent of this half-warp within the block
    const unsigned hmask = 0xffffu << (16 * half);  // this half's lanes
#ifdef ECO_TIMELINE
    if (threadIdx.x == 0) timeline_mark(p, 0, ~globaltimer_ns());
#endif
#if ECO_POST_PDL >= 2
    asm volatile("griddepcontrol.launch_dependents;");  // k_post may be scheduled as blocks drain
#endif
#if ECO_STEP2_PDL
    // the second policy of a two-step graph is a programmatic dependent of k_post: wait for
    // it (a no-op for an ordinary launch)
    if (SPLIT && !SHARD) asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    step_housekeeping(p);
    const long total = (long)p.n_worlds * p.S;
    // COMPACT (p.pol_compact: more slots than one wave of blocks holds — several worlds, a
    // large world, a band; unsharded handles): every warp loops over tiles of CPT_TILE consecutive
    // LIVE list positions of the worlds — s_tile0[w] = the tiles of the worlds before w, from
    // the worlds' counts, made by warp 0 — so no block is launched for the empty tail of a
    // world's slot pool, and a warp goes on to its next tile without waiting for the block's
    // other agents (all worlds share t).  The compiled-out variant keeps the one-tile code.
    __shared__ int s_tile0[COMPACT ? POLICY_COMPACT_WORLDS + 1 : 1];
    int n_tiles = 1;
    if (COMPACT) {
        if (warp == 0) {
            const int par = (int)(p.t[0] & 1);
            int run = 0;
            for (int w0 = 0; w0 < p.n_worlds; w0 += 32) {
                const int wl = w0 + lane;
                const int cnt = wl < p.n_worlds ? p.n_alive[par * p.n_worlds + wl] : 0;
                const int tl = (cnt + CPT_TILE - 1) / CPT_TILE;
                int inc = tl;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int up = __shfl_up_sync(FULL, inc, o);
                    if (lane >= o) inc += up;
                }
                if (wl < p.n_worlds) s_tile0[wl] = run + inc - tl;
                run += __shfl_sync(FULL, inc, 31);
            }
            if (lane == 0) s_tile0[p.n_worlds] = run;
        }
        __syncthreads();
        n_tiles = s_tile0[p.n_worlds];
    }
    // (COMPACT) this context's counters of its current world, flushed when the world changes
    unsigned long long acc_nnz = 0ull, acc_ties = 0ull;
    int acc_w = -1;
    constexpr int CPT_PER_BLOCK = HALF_AGENTS / CPT_TILE;  // tiles a block works on at a time
    for (int tile = COMPACT ? (int)blockIdx.x * CPT_PER_BLOCK + ag / CPT_TILE : 0; tile < n_tiles;
         tile += COMPACT ? (int)gridDim.x * CPT_PER_BLOCK : 1) {
    // one world: contexts interleaved over the blocks (few agents spread over every SM);
    // sharded: block-major, so this rank's agents (a fraction of the slots) fill whole blocks
    // (more blocks than one wave: block-major too, p.pol_bmajor)
    long v = (SHARD || p.pol_bmajor) ? (long)blockIdx.x * HALF_AGENTS + ag : (long)ag * gridDim.x + blockIdx.x;
    if (COMPACT) {
        int lo = 0, hi = p.n_worlds;  // s_tile0[lo] <= tile < s_tile0[hi]: the last such lo owns the tile
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_tile0[mid] <= tile) lo = mid;
            else hi = mid;
        }
        const int ii = (tile - s_tile0[lo]) * CPT_TILE + ag % CPT_TILE;
        v = ii < p.S ? (long)lo * p.S + ii : total;
    }
    const bool in_range = v < total;
    const int w = in_range ? (int)(v / p.S) : 0;
    const int i = in_range ? (int)(v - (long)w * p.S) : 0;
    const int64_t t = p.t[w];
    // unsharded: both parities' count, slot and cell of list position i load beside t (one
    // round trip instead of t -> count -> slot -> cell; entries past a count are stale, unused)
    int n_list = 0, slot = 0, cell_l = 0, n_ch = 0, own_surv = 0;
    if (SHARD && SPLIT && in_range) own_surv = *p.own_surv;
    const int forced_on = in_range ? *p.forced_on : 0;  // loaded now, used by the epilogue
    if (!SHARD && in_range) {
        if (SPLIT) n_ch = *p.p_children;
        const size_t o0 = (size_t)w * p.S + i, o1 = ((size_t)p.n_worlds + w) * p.S + i;
        const int n0 = p.n_alive[w], n1 = p.n_alive[p.n_worlds + w];
        const int s0 = p.alive_list[o0], s1 = p.alive_list[o1];
        const int c0 = p.list_cell[o0], c1 = p.list_cell[o1];
        const bool odd = (t & 1) != 0;
        n_list = odd ? n1 : n0;
        slot = odd ? s1 : s0;
        cell_l = odd ? c1 : c0;
    }
    // sharded: the contexts walk this rank's own live slots instead of the whole list
    bool active = in_range && i < (SHARD ? p.own_count[t & 1] : n_list);
    unsigned long long nnz_a = 0ull, tie_a = 0ull;
#ifdef ECO_POLICY_TRACE
    // diagnostic build: per agent (kernel entry, mask ready, end, nnz) of the last launch
    unsigned long long *trace = p.phase_ns + 16 + 4 * (size_t)(v & 8191);
    const uint64_t t_entry = globaltimer_ns();
#endif
    if (SHARD) slot = active ? p.own_list[(t & 1) * p.S + i] : 0;
    if (__any_sync(FULL, active)) {  // both halves stay converged for the warp-wide intrinsics
        int cellv = 0;
        size_t gs = 0;
        const float *Wl = p.weights;  // + hl * 4: unit hl of a chunk; unit hl + 16 at + 64 floats
        if (active) {
            gs = (size_t)w * p.S + slot;
            Wl = p.weights + gs * (size_t)p.Pd + hl * 4;
        }
#if ECO_POLICY_PREFETCH && ECO_POLICY_PREFETCH != 2
        // the agent's contiguous W_hh | b | W_out | b_out block (17.7 KB at Hd = 32) streams into
        // L2 as one bulk prefetch: DRAM serves it sequentially, the ring then hits L2
        if (active && hl == 0) {
            const float *blk = p.weights + gs * (size_t)p.Pd + p.off_hh;
            const uint32_t bytes = (uint32_t)(p.Pd - p.off_hh) * 4u;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(blk), "r"(bytes) : "memory");
        }
#endif
        float4 *rg = half_smem + (ag * R) * 32 + hl;  // slot s, unit hl: rg[s * 32]; unit hl+16: rg[s * 32 + 16]
        const float *Whh = Wl + p.off_hh;
        auto issue = [&](int slot_, const float *src) {
            if (active) {
                cp_async16(rg + slot_ * 32, src, 0ull);
                cp_async16(rg + slot_ * 32 + 16, src + 64, 0ull);
            }
        };
        // split: the first chunk is P = W_hh h + b (k_post made it), or the bias of a child
        const bool child = SPLIT && active && (SHARD ? i >= own_surv : i >= n_list - n_ch);
        if (SPLIT) {
            issue(0, child ? Wl + p.off_b : p.Pbuf + (size_t)slot * HD * 4 + hl * 4);
            cp_commit();
        } else {
#pragma unroll
            for (int q = 0; q < R; ++q) {  // prologue: W_hh rows 0..R-1
                issue(q, Whh + q * HD * 4);
                cp_commit();
            }
        }
        float hk0 = 0.f, hk1 = 0.f, ck0 = 0.f, ck1 = 0.f;
        float wo0[5], wo1[5], bo[5];
        if (active) {
            hk0 = p.h[gs * HD + hl];
            hk1 = p.h[gs * HD + hl + 16];
            ck0 = p.c[gs * HD + hl];
            ck1 = p.c[gs * HD + hl + 16];
            cellv = SHARD ? p.cell[gs] : cell_l;
        }
        const float *Wo = Wl - hl * 4;
#pragma unroll
        for (int a = 0; a < 5; ++a) {
            wo0[a] = active ? __ldg(Wo + p.off_out + a * HD + hl) : 0.f;
            wo1[a] = active ? __ldg(Wo + p.off_out + a * HD + hl + 16) : 0.f;
            bo[a] = active ? __ldg(Wo + p.off_bout + a) : 0.f;
        }
        // observation mask: half-lane q < 2(2r+1) loads row q; OR over the half
        uint64_t m_lo = 0ull, m_hi = 0ull;
        {
            uint64_t lo = 0ull, hi = 0ull;
            const int wd = 2 * p.r + 1;
            if (active && hl < 2 * wd) {
                const int y = row_of(p, cellv), x = cellv - y * p.W;
                const int ch = hl / wd, row = hl - ch * wd;
                const int yy = y - p.r + row;
                if (yy >= 0 && yy < p.H) {
                    const uint32_t *pl =
                        ch ? p.occ + (size_t)w * plane_words(p) : plane_next(p, t) + (size_t)w * plane_words(p);
                    const uint64_t bits = row_bits(pl + (size_t)yy * p.WW, p.WW, x - p.r, wd);
                    const int pos = ch * wd * wd + row * wd;
                    if (pos < 64) {
                        lo = bits << pos;
                        if (pos + wd > 64) hi = bits >> (64 - pos);
                    } else {
                        hi = bits << (pos - 64);
                    }
                }
            }
            const uint32_t a0 = __reduce_or_sync(hmask, (uint32_t)lo), a1 = __reduce_or_sync(hmask, (uint32_t)(lo >> 32));
            const uint32_t a2 = __reduce_or_sync(hmask, (uint32_t)hi), a3 = __reduce_or_sync(hmask, (uint32_t)(hi >> 32));
            m_lo = ((uint64_t)a1 << 32) | a0;
            m_hi = ((uint64_t)a3 << 32) | a2;
        }
        // compacted ascending column indices (bytes)
        uint8_t *cols = s_col[ag];
        int nnz = 0;
#pragma unroll
        for (int part = 0; part < 8; ++part) {
            const int bit = part * 16 + hl;
            const uint64_t word = part < 4 ? m_lo : m_hi;
            const bool on = ((word >> (bit & 63)) & 1ull) != 0ull;
            const unsigned bal = (__ballot_sync(FULL, on) >> (16 * half)) & 0xffffu;
            if (on) cols[nnz + __popc(bal & ((1u << hl) - 1u))] = (uint8_t)bit;
            nnz += __popc(bal);
        }
        __syncwarp();
#if ECO_POLICY_PREFETCH == 1
        if (active)  // every active column (512 B) requested at once
            for (int q = hl; q < nnz; q += 16)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.weights + gs * (size_t)p.Pd +
                                                                                  (size_t)cols[q] * HD * 4),
                             "r"(HD * 16)
                             : "memory");
#endif
#ifdef ECO_POLICY_TRACE
        if (active && hl == 0) {
            trace[0] = t_entry;
            trace[1] = globaltimer_ns();
            trace[3] = nnz;
        }
#endif
        float4 acc0 = make_float4(0.f, 0.f, 0.f, 0.f), acc1 = acc0;
        if (SPLIT) {
            // chunk 0 = P (or b), chunks 1.. = the active columns; D ticks per round from 0.
            // An agent of a block's first half whose partner context (agent ag + HALF_AGENTS/2)
            // holds no agent this step also uses the partner's ring: 2R chunks in flight, so
            // the ~10 columns of a typical agent arrive in one round trip instead of two.
            const int N1 = 1 + nnz;
            const int Nw1 = __reduce_max_sync(FULL, active ? N1 : 0);
            auto stream = [&](auto DC) {
                constexpr int D = decltype(DC)::value;
                auto at = [&](int s_) { return rg + (s_ < R ? s_ : s_ + (HALF_AGENTS / 2 - 1) * R) * 32; };
                auto issue_at = [&](int s_, const float *src) {
                    if (active) {
                        cp_async16(at(s_), src, 0ull);
                        cp_async16(at(s_) + 16, src + 64, 0ull);
                    }
                };
#pragma unroll
                for (int q = 1; q < D; ++q) {
                    if (q < N1) issue_at(q, Wl + (int)cols[q - 1] * HD * 4);
                    cp_commit();
                }
                for (int k0 = 0; k0 < Nw1; k0 += D) {
#pragma unroll
                    for (int s2 = 0; s2 < D; ++s2) {
                        const int k = k0 + s2;
                        cp_wait<D - 1>();
                        if (k < N1) {
                            const float4 c0 = at(s2)[0], c1 = at(s2)[16];
                            if (k == 0) {
                                acc0 = c0;
                                acc1 = c1;
                            } else {
                                acc0.x += c0.x;
                                acc0.y += c0.y;
                                acc0.z += c0.z;
                                acc0.w += c0.w;
                                acc1.x += c1.x;
                                acc1.y += c1.y;
                                acc1.z += c1.z;
                                acc1.w += c1.w;
                            }
                        }
                        const int kn = k + D;
                        if (kn < N1) issue_at(s2, Wl + (int)cols[kn - 1] * HD * 4);
                        cp_commit();
                    }
                }
            };
#if ECO_POLICY_DEEP
            // per warp: its agents' partners (agents 2w + HALF_AGENTS/2 and the next, list
            // positions further on) hold no agent this step, so their rings are free
            const long pv = p.pol_bmajor ? (long)blockIdx.x * HALF_AGENTS + 2 * warp + HALF_AGENTS / 2
                                         : (long)(2 * warp + HALF_AGENTS / 2) * gridDim.x + blockIdx.x;
            // (COMPACT: the partner warp works on its own tiles)
            const bool deep = !SHARD && !COMPACT && warp < HALF_WARPS / 2 && pv >= (long)n_list;
            if (deep) stream(std::integral_constant<int, 2 * R>{});
            else stream(std::integral_constant<int, R>{});
#else
            stream(std::integral_constant<int, R>{});
#endif
        } else {
        const int N = Q0 + nnz;
        const int Nw = __reduce_max_sync(FULL, active ? N : 0);  // the warp runs the longer sequence
        auto refill = [&](int kn, int slot_) {
            if (kn < N) issue(slot_, kn < NHH ? Whh + kn * HD * 4 : (kn == QB ? Wl + p.off_b : Wl + (int)cols[kn - Q0] * HD * 4));
            cp_commit();
        };
#pragma unroll
        for (int k = 0; k < NHH; ++k) {  // W_hh rows
            cp_wait<R - 1>();
            const float4 c0 = rg[(k % R) * 32], c1 = rg[(k % R) * 32 + 16];
            const float hj = __shfl_sync(FULL, k < 16 ? hk0 : hk1, k & 15, 16);
            acc0.x = fmaf(hj, c0.x, acc0.x);
            acc0.y = fmaf(hj, c0.y, acc0.y);
            acc0.z = fmaf(hj, c0.z, acc0.z);
            acc0.w = fmaf(hj, c0.w, acc0.w);
            acc1.x = fmaf(hj, c1.x, acc1.x);
            acc1.y = fmaf(hj, c1.y, acc1.y);
            acc1.z = fmaf(hj, c1.z, acc1.z);
            acc1.w = fmaf(hj, c1.w, acc1.w);
            if (k + R < NHH) {
                issue(k % R, Whh + (k + R) * HD * 4);
                cp_commit();
            } else if (k + R == QB) {
                issue(k % R, Wl + p.off_b);
                cp_commit();
            } else {
                refill(k + R, k % R);
            }
        }
        // ticks QB.. : the bias, then the columns; R ticks per round from QB so slots are static
        for (int k0 = QB; k0 < Nw; k0 += R) {
#pragma unroll
            for (int s2 = 0; s2 < R; ++s2) {
                const int k = k0 + s2;
                constexpr int base = QB % R;
                const int rs = (base + s2) % R;
                cp_wait<R - 1>();
                if (k < N) {
                    const float4 c0 = rg[rs * 32], c1 = rg[rs * 32 + 16];
                    acc0.x += c0.x;
                    acc0.y += c0.y;
                    acc0.z += c0.z;
                    acc0.w += c0.w;
                    acc1.x += c1.x;
                    acc1.y += c1.y;
                    acc1.z += c1.z;
                    acc1.w += c1.w;
                }
                refill(k + R, rs);
            }
        }
        }  // !SPLIT
        cp_wait<0>();
#if defined(ECO_POLICY_TRACE) && defined(ECO_POLICY_TRACE_STREAM)
        if (active && hl == 0) trace[3] = globaltimer_ns();  // the chunks are in: the gates and epilogue follow
#endif
        const float cn0 = sigmoidf_acc(acc0.y) * ck0 + sigmoidf_acc(acc0.x) * tanhf(acc0.z);
        const float hn0 = sigmoidf_acc(acc0.w) * tanhf(cn0);
        const float cn1 = sigmoidf_acc(acc1.y) * ck1 + sigmoidf_acc(acc1.x) * tanhf(acc1.z);
        const float hn1 = sigmoidf_acc(acc1.w) * tanhf(cn1);
        float lg[5];
#pragma unroll
        for (int a = 0; a < 5; ++a) {
            float sm = wo0[a] * hn0 + wo1[a] * hn1;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) sm += __shfl_xor_sync(FULL, sm, o, 16);
            lg[a] = sm + bo[a];
        }
        if (active) {
            p.h[gs * HD + hl] = hn0;
            p.h[gs * HD + hl + 16] = hn1;
            p.c[gs * HD + hl] = cn0;
            p.c[gs * HD + hl + 16] = cn1;
            bool bad = !isfinite(hn0) || !isfinite(cn0) || !isfinite(hn1) || !isfinite(cn1);
            if (hl == 0) {
                PolicyCounters one;
                agent_epilogue<SHARD>(p, w, i, slot, gs, t, cellv, lg, m_lo, m_hi, forced_on, one, bad);
                nnz_a = one.nnz;
                tie_a = one.ties;
            }
            if (bad) *reinterpret_cast<volatile int32_t *>(p.nonfinite) = 1;
#ifdef ECO_POLICY_TRACE
            if (hl == 0) trace[2] = globaltimer_ns();
#endif
        }
    }
    if (COMPACT) {
        if (hl == 0 && active) {
            if (w != acc_w) {
                if (acc_w >= 0) flush_counters<SHARD>(p, acc_w, acc_nnz, acc_ties);
                acc_w = w;
                acc_nnz = acc_ties = 0ull;
            }
            acc_nnz += nnz_a;
            acc_ties += tie_a;
        }
        __syncwarp();  // the warp's next tile rewrites its s_col rows
        continue;
    }
    acc_w = active ? w : -1;
    acc_nnz = nnz_a;
    acc_ties = tie_a;
    }  // tiles
    if (hl == 0) {
        s_w[ag] = acc_w;
        s_nnz[ag] = acc_nnz;
        s_ties[ag] = acc_ties;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // runs of equal worlds (one world: a single flush per block)
        int wc = -1;
        unsigned long long a = 0ull, b = 0ull;
        for (int k = 0; k < HALF_AGENTS; ++k) {
            if (s_w[k] < 0) continue;
            if (s_w[k] != wc) {
                flush_counters<SHARD>(p, wc, a, b);
                wc = s_w[k];
                a = b = 0ull;
            }
            a += s_nnz[k];
            b += s_ties[k];
        }
        flush_counters<SHARD>(p, wc, a, b);
#ifdef ECO_TIMELINE
        timeline_mark(p, 1, globaltimer_ns());
#endif
    }
}

#include "policy_cnn.cuh"

cudaError_t policy_occupancy(int hidden, int net, int *blocks_per_sm, int *threads_out) {
    const int threads = net == 1 ? CNN_BLK_THREADS : 256;
    *threads_out = threads;
    if (net == 1)
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_policy_cnn_blk, CNN_BLK_THREADS, CNN_BLK_SMEM);
    switch (hidden) {
        case 4: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_policy_reg<4>, threads, 0);
        case 8: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_policy_reg<8>, threads, 0);
        case 16: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_policy_reg<16>, threads, 0);
        case 32: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_policy_half<false>, HALF_THREADS, HALF_SMEM);
        default: return cudaErrorInvalidValue;
    }
}

int policy_compact_worlds() { return POLICY_COMPACT_WORLDS; }

cudaError_t policy_prepare() {
    cudaError_t e = set_dyn_smem(k_policy_half<true>, HALF_SMEM);
    if (e != cudaSuccess) return e;
    e = set_dyn_smem(k_policy_cnn_blk, CNN_BLK_SMEM);
    if (e != cudaSuccess) return e;
    e = set_dyn_smem(k_policy_half<false, true>, HALF_SMEM);
    if (e != cudaSuccess) return e;
    e = set_dyn_smem(k_policy_half<true, true>, HALF_SMEM);
    if (e != cudaSuccess) return e;
    e = set_dyn_smem(k_policy_half<false, true, true>, HALF_SMEM);
    if (e != cudaSuccess) return e;
    e = set_dyn_smem(k_policy_half<false, false, true>, HALF_SMEM);
    if (e != cudaSuccess) return e;
    e = set_dyn_smem(k_prepare_p, HALF_SMEM);
    if (e != cudaSuccess) return e;
    e = set_dyn_smem(k_prepare_p_snap, HALF_SMEM);
    if (e != cudaSuccess) return e;
    e = set_dyn_smem(k_prepare_p_list, HALF_SMEM);
    if (e != cudaSuccess) return e;
    return set_dyn_smem(k_policy_half<false>, HALF_SMEM);
}

cudaError_t launch_policy(const DevParams &p, const LaunchCfg &lc, cudaStream_t s, bool pdl) {
    if (p.net == 1) {
#if ECO_STEP2_PDL
        if (pdl && p.n_ranks == 1) {  // a programmatic dependent of the previous step's post-policy kernel
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(lc.policy_blocks);
            cfg.blockDim = dim3(CNN_BLK_THREADS);
            cfg.dynamicSmemBytes = CNN_BLK_SMEM;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            return cudaLaunchKernelEx(&cfg, k_policy_cnn_blk, p);
        }
#endif
        k_policy_cnn_blk<<<lc.policy_blocks, CNN_BLK_THREADS, CNN_BLK_SMEM, s>>>(p);
        return cudaGetLastError();
    }
    switch (p.Hd) {
        case 4: k_policy_reg<4><<<lc.policy_blocks, lc.policy_threads, 0, s>>>(p); break;
        case 8: k_policy_reg<8><<<lc.policy_blocks, lc.policy_threads, 0, s>>>(p); break;
        case 16: k_policy_reg<16><<<lc.policy_blocks, lc.policy_threads, 0, s>>>(p); break;
        case 32: {
            // one half-warp per slot; at least enough blocks for the housekeeping's clear of
            // the claimed-cell bitmap (a large grid with few slots)
            const long slots = (long)p.n_worlds * p.S;
            long blocks = (slots + HALF_AGENTS - 1) / HALF_AGENTS;
            const long hk = ((long)p.n_worlds * plane_words(p) + 255) / 256;
            const long hk_cap = (long)lc.sms * 4;
            if (blocks < (hk < hk_cap ? hk : hk_cap)) blocks = hk < hk_cap ? hk : hk_cap;
#if ECO_HALF_FULLGRID
            if (blocks < (long)lc.sms * HALF_BPS) blocks = (long)lc.sms * HALF_BPS;  // every SM the same
#endif
            // compacted tiles: resident blocks loop over the live tiles
            if (p.pol_compact && p.n_ranks == 1 && blocks > (long)lc.sms * HALF_BPS * ECO_POL_COMPACT_WAVES)
                blocks = (long)lc.sms * HALF_BPS * ECO_POL_COMPACT_WAVES;
            const bool cpt = p.pol_compact && p.n_ranks == 1;
            if (p.n_ranks > 1 && p.split) k_policy_half<true, true><<<(unsigned)(blocks > 0 ? blocks : 1), HALF_THREADS, HALF_SMEM, s>>>(p);
            else if (p.n_ranks > 1) k_policy_half<true><<<(unsigned)(blocks > 0 ? blocks : 1), HALF_THREADS, HALF_SMEM, s>>>(p);
            else if (p.split && pdl) {  // a programmatic dependent of the previous k_post
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3((unsigned)(blocks > 0 ? blocks : 1));
                cfg.blockDim = dim3(HALF_THREADS);
                cfg.dynamicSmemBytes = HALF_SMEM;
                cfg.stream = s;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                return cpt ? cudaLaunchKernelEx(&cfg, k_policy_half<false, true, true>, p)
                           : cudaLaunchKernelEx(&cfg, k_policy_half<false, true>, p);
            }
            else if (p.split && cpt) k_policy_half<false, true, true><<<(unsigned)(blocks > 0 ? blocks : 1), HALF_THREADS, HALF_SMEM, s>>>(p);
            else if (p.split) k_policy_half<false, true><<<(unsigned)(blocks > 0 ? blocks : 1), HALF_THREADS, HALF_SMEM, s>>>(p);
            else if (cpt) k_policy_half<false, false, true><<<(unsigned)(blocks > 0 ? blocks : 1), HALF_THREADS, HALF_SMEM, s>>>(p);
            else k_policy_half<false><<<(unsigned)(blocks > 0 ? blocks : 1), HALF_THREADS, HALF_SMEM, s>>>(p);
            break;
        }
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ----------------------------------------------------------- standalone phase kernels
__global__ void __launch_bounds__(256) k_regrow(DevParams p, int ahead) {
    regrow_phase(p, p.t[0] + ahead, interleaved_gtid(), (size_t)gridDim.x * blockDim.x);
}

template <bool PAPER>
__global__ void __launch_bounds__(256) k_move(DevParams p) {
    move_phase<PAPER>(p, interleaved_gtid(), (size_t)gridDim.x * blockDim.x);
}

__global__ void __launch_bounds__(256) k_mv_pass(DevParams p) {  // one block per world, after the rank
    __shared__ int s_mv[SIM_MOVE_BINS];
    const int64_t T = p.t[blockIdx.x] - 1;  // the rank advanced t
#if ECO_METRICS & 2
    if (mv_window_end(T)) mv_pass_part(p, T, blockIdx.x, 0, p.S, threadIdx.x, blockDim.x, s_mv);
#endif
    if (gr_window_end(T)) greed_pass_part(p, blockIdx.x, 0, p.S, threadIdx.x, blockDim.x);
}

__global__ void __launch_bounds__(256) k_birth_claim(DevParams p) {
    birth_claim_phase(p, interleaved_gtid(), (size_t)gridDim.x * blockDim.x);
}

constexpr int RANK_THREADS = 1024;
__global__ void __launch_bounds__(RANK_THREADS) k_birth_rank(DevParams p) {
    __shared__ uint32_t scratch[2 * (RANK_THREADS / 32 + 1)];
    __shared__ int s_free[RANK_SMEM_CAP], s_bcell[RANK_SMEM_CAP], s_par[RANK_SMEM_CAP];
    for (int w = blockIdx.x; w < p.n_worlds; w += gridDim.x)
        birth_rank_world<RANK_THREADS>(p, w, scratch, s_free, s_bcell, s_par);
}

__global__ void __launch_bounds__(256) k_mutate(DevParams p) {
    __shared__ int s_cum[RANK_SMEM_CAP];  // several worlds: the children prefixed over the worlds
    mutate_phase(p, interleaved_gtid(), (size_t)gridDim.x * blockDim.x, s_cum, RANK_SMEM_CAP);
}

// ------------------------------------------------------------------------ k_post
// a4 move/consume/physiology/death | barrier | a5 birth candidates and claimed cells |
// barrier | a5 rank + winners (redundantly in every block), placement and counters (block
// 0), a1 regrowth of step t+1 (needs only R'' of step t), a5 mutation of the children,
// t += 1.  With several worlds (or > RANK_SMEM_CAP births) the rank runs one block per world
// and a third barrier precedes the mutation.  A phase that ends in a barrier pays for its
// writes in the barrier's release fence; the regrowth's plane writes (measured: +3..6 us of
// fence when they preceded a barrier) go last, where only the kernel's end waits for them.
#ifndef ECO_POST_THREADS
// 24 warps per block (4 P warps + 20 dynamics warps at paper scale): fewer idle warps in every
// block barrier of the latency-bound phases.  Measured (round 2): 1024 -> 768 threads: the
// driver's t = 5..25 33.2 -> 31.7 us, 10,000 steps 48.4 -> 46.7 us, large world 1.522 ->
// 1.514 ms; 512 / 640 / 896 no better overall
#define ECO_POST_THREADS 768
#endif
constexpr int POST_THREADS = ECO_POST_THREADS;
#ifndef ECO_MUT_WARM
#define ECO_MUT_WARM 1  // measured: 48.8 -> 48.0 us per step
#endif
#ifndef ECO_HH_WARPS
#define ECO_HH_WARPS 4  // split: the P warps of blocks 1.. (measured: 2..16 warps, depth 6..16)
#endif
#ifndef ECO_HH_WARPS_BIG
#define ECO_HH_WARPS_BIG 16  // ... above HH_BIG_AGENTS live agents the P stream is the longer part
#endif
#ifndef ECO_HH_BIG_AGENTS
#define ECO_HH_BIG_AGENTS 32768
#endif
#ifndef ECO_RANK_SHARE
#define ECO_RANK_SHARE 4  // several worlds: a ranking block's share of the regrowth, in eighths of a free block's (64-world ensemble, rank + regrowth: 0 -> 35.4, 4 -> 26.2, 6 -> 30.1, 8 -> 30.7 us)
#endif
#ifndef ECO_CLAIMS_MAX
#define ECO_CLAIMS_MAX 1024  // measured: 1024 and 2048 beat 4096 at the population cap
#endif
constexpr int CLAIMS_BLOCK_MAX = ECO_CLAIMS_MAX;
#ifndef ECO_HH_DEPTH
#define ECO_HH_DEPTH 8  // split: 512-B chunks in flight per P context (<= 33: W_hh rows + b)
#endif
#ifndef ECO_HH_DEPTH_BIG
#define ECO_HH_DEPTH_BIG 8  // ... in the many-slot variant
#endif
constexpr int HH_DEPTH = ECO_HH_DEPTH, HH_DEPTH_BIG = ECO_HH_DEPTH_BIG;
static_assert(HH_DEPTH <= 33 && HH_DEPTH_BIG <= 33, "a P context streams 33 chunks");
constexpr int HH_RING_SMALL = 2 * ECO_HH_WARPS * HH_DEPTH * 32 * 16, HH_RING_BIG = 2 * ECO_HH_WARPS_BIG * HH_DEPTH_BIG * 32 * 16;
constexpr int POST_SMEM = HH_RING_SMALL > HH_RING_BIG ? HH_RING_SMALL : HH_RING_BIG;  // split: the P rings (max)
constexpr int POST_SMEM_SMALL = HH_RING_SMALL;  // worlds that never exceed the threshold
// worlds with more slots than the threshold run k_post<., true>: 16 P warps per block (the
// P stream is the longer part of the step there: large world 1.71 -> 1.52 ms per step)
inline bool post_big(const DevParams &p) { return p.split && p.S > ECO_HH_BIG_AGENTS; }
inline int post_smem_bytes(const DevParams &p) { return !p.split ? 0 : post_big(p) ? POST_SMEM : POST_SMEM_SMALL; }
#ifdef ECO_BLOCK_CLOCK
// diagnostic build: per block and barrier k, summed own-work and barrier-wait durations in
// phase_ns[ECO_BLOCK_CLOCK_BASE + (k * gridDim + block) * 3 + {0, 1, 2}] (2: an explicit
// fence.acq_rel.gpu before the arrival, timed alone)
constexpr int ECO_BLOCK_CLOCK_BASE = 16;
#define POST_SYNC(k)                                                                              \
    do {                                                                                          \
        asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");                                  \
        const uint64_t a_ = globaltimer_ns();                                                     \
        uint64_t f_ = a_;                                                                         \
        if (threadIdx.x == 0) {                                                                   \
            asm volatile("fence.acq_rel.gpu;" ::: "memory");                                     \
            f_ = globaltimer_ns();                                                                \
        }                                                                                         \
        grid_sync(bar, target, nthr);                                                             \
        const uint64_t e_ = globaltimer_ns();                                                     \
        if (threadIdx.x == 0) {                                                                   \
            unsigned long long *q_ = p.phase_ns + ECO_BLOCK_CLOCK_BASE + ((k) * gridDim.x + blockIdx.x) * 3; \
            q_[0] += a_ - bt_;                                                                    \
            q_[1] += e_ - a_;                                                                     \
            q_[2] += f_ - a_;                                                                     \
        }                                                                                         \
        bt_ = e_;                                                                                 \
    } while (0)
#else
#define POST_SYNC(k) grid_sync(bar, target, nthr)
#endif

// MULTI: several worlds in the handle (the launcher's choice: p.n_worlds > 1), compiled as its
// own variant so that the one-world kernels carry none of its code (the one-shot phases are
// sensitive to code size and layout: as runtime branches the several-world paths cost the
// paper-scale step 0.8 us, measured)
template <bool SHARD, bool BIG = false, bool PAPER = false, bool MULTI = false>
__global__ void __launch_bounds__(POST_THREADS) k_post(DevParams p_, unsigned long long *bar) {
    static_assert(!(MULTI && (SHARD || BIG)), "several worlds: unsharded, no split policy");
    DevParams p = p_;
    if (!SHARD) p.n_ranks = 1;
    __shared__ uint32_t scratch[2 * (POST_THREADS / 32 + 1)];
    __shared__ int s_free[RANK_SMEM_CAP], s_bcell[RANK_SMEM_CAP], s_par[RANK_SMEM_CAP];
    __shared__ int s_mv[SIM_MOVE_BINS];  // a window end's movement histogram of this block
    extern __shared__ __align__(1024) float4 post_smem[];  // split: the P rings, 2 HH_WARPS contexts x HH_DEPTH
#if ECO_POST_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the policy grid has completed
#endif
    unsigned long long target = grid_sync_base(bar);
    const int64_t T = p.t[0];  // the step this launch completes (all worlds share t)
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef ECO_TIMELINE
    if (threadIdx.x == 0) timeline_mark(p, 2, ~globaltimer_ns());
#endif
    // split policy (one world): the last HH_WARPS warps of blocks 1.. make P = W_hh h + b of
    // every agent alive at the start of step T (the next step's survivors among them) from
    // the kernel's first cycle, streaming beside the latency-bound dynamics of the other
    // warps; they take part in no barrier.  The rows of the agents that die are never read
    // (a child placed in such a slot starts from its bias).
    constexpr int HH_WARPS = BIG ? ECO_HH_WARPS_BIG : ECO_HH_WARPS;  // compile-time: the roles need no load
    constexpr int DYN_WARPS = POST_THREADS / 32 - HH_WARPS;
    const bool hh_split = !MULTI && p.split && p.n_worlds == 1 && gridDim.x > 1;
#ifdef ECO_END_CLOCK
    // diagnostic build: per launch, the latest end of the P warps and of the other warps
    // after block 0's start, summed over the launches in phase_ns[4] and [5]
    unsigned long long *ec = reinterpret_cast<unsigned long long *>(p.phase_ns) + 10 + 3 * (T & 1);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long *pe = reinterpret_cast<unsigned long long *>(p.phase_ns) + 10 + 3 * ((T + 1) & 1);
        if (pe[0]) {
            p.phase_ns[4] += pe[1] - pe[0];
            p.phase_ns[5] += pe[2] - pe[0];
        }
        pe[0] = pe[1] = pe[2] = 0ull;
        ec[0] = globaltimer_ns();
    }
#define END_CLOCK(k) \
    if (lane == 0) atomicMax(ec + (k), (unsigned long long)globaltimer_ns())
#else
#define END_CLOCK(k)
#endif
    if (hh_split && blockIdx.x > 0 && wid >= DYN_WARPS) {
        const unsigned nb = gridDim.x - 1, b = blockIdx.x - 1;
        const int ag = (wid - DYN_WARPS) * 2 + (lane >> 4);
        // (sharded: this rank's own agents only)
        const int32_t *hl_ = SHARD ? p.own_list + (size_t)(T & 1) * p.S : list_of(p, T, 0);
        const int hn_ = SHARD ? p.own_count[T & 1] : *count_of(p, T, 0);
        constexpr int DEPTH = BIG ? HH_DEPTH_BIG : HH_DEPTH;
        hh_pass<DEPTH>(p, hl_, hn_, ag * (int)nb + (int)b, (int)nb * HH_WARPS * 2, post_smem + (ag * DEPTH) * 32);
        END_CLOCK(1);
#ifdef ECO_TIMELINE
        if (lane == 0) timeline_mark(p, 3, globaltimer_ns(), T);
#endif
        return;
    }
    // warp-interleaved global index: consecutive warps of work land on different blocks
    // (SMs), so the per-item dependency chains of every phase run on all 148 SMs at once;
    // with the split, over the dynamics warps (all of block 0's, DYN_WARPS of the others)
    size_t gtid = interleaved_gtid(), gthreads = (size_t)gridDim.x * blockDim.x;
    int nthr = blockDim.x;  // threads of this block in the barriers
    if (hh_split) {
        const size_t nb = gridDim.x - 1;
        gthreads = nb * DYN_WARPS * 32 + blockDim.x;
        gtid = blockIdx.x == 0 ? nb * DYN_WARPS * 32 + threadIdx.x : ((size_t)wid * nb + blockIdx.x - 1) * 32 + lane;
        if (blockIdx.x > 0) nthr = DYN_WARPS * 32;
    }
    // phase clock: block 0 accumulates the time between barriers (as seen by block 0)
    const bool clk = blockIdx.x == 0 && threadIdx.x == 0;
    uint64_t t0 = clk ? globaltimer_ns() : 0ull, t1;
    auto lap = [&](int k) {
        if (clk) {
            t1 = globaltimer_ns();
            atomicAdd(p.phase_ns + k, t1 - t0);
            t0 = t1;
        }
    };
#ifdef ECO_BLOCK_CLOCK
    uint64_t bt_ = globaltimer_ns();
#endif
    if (p.n_ranks > 1) {
        // sharded: the ranks' policies left their move records (summed over the ranks) but no
        // claims; post every agent's claim here, then resolve them after a barrier
        const int n = *count_of(p, T, 0);
        if (gtid == 0) {  // the ranks' policy counters, summed by the exchange; then reset
            sim_step_record *rec = record_of(p, T, 0);
            rec->obs_nnz += (int64_t)p.pol_ctr[0];
            rec->near_ties += (int64_t)p.pol_ctr[1];
            p.pol_ctr[0] = p.pol_ctr[1] = 0ull;
        }
        for (size_t k = gtid; k < (size_t)n; k += gthreads) {
            const int sl = list_of(p, T, 0)[k];
            const int4 mr = p.mrec_slot[sl];  // summed over the ranks; listed in this rank's order
            p.mrec[k] = mr;
            p.mrec_slot[sl] = make_int4(0, 0, 0, 0);  // zero again for the next exchange
            if (mr.z >= 0)
                atomicMax(p.claim + mr.z, ((unsigned long long)(uint32_t)mr.w << 32) |
                                              (unsigned long long)(0xFFFFFFFFu - (uint32_t)mr.y));
        }
        grid_sync(bar, target, nthr);
    }
    // several worlds: the move and claim phases visit the worlds' live list positions only
    const int *live_cum = nullptr;
    if (MULTI && p.n_worlds < RANK_SMEM_CAP) {
        live_prefix(p, T, s_free);  // (s_free: free until the rank)
        live_cum = s_free;
    }
    move_phase<PAPER>(p, gtid, gthreads, live_cum);
    POST_SYNC(0);
    lap(0);
    // sharded + split: this rank's survivors lead its next list; its children (appended by
    // the placement) follow and have no P row
    if (SHARD && p.split && blockIdx.x == 0 && threadIdx.x == 0)
        *p.own_surv = *reinterpret_cast<volatile int32_t *>(p.own_count + ((T + 1) & 1));
    if (MULTI) {
        // birth candidates on every thread
        const uint64_t h0 = blockIdx.x == 0 ? globaltimer_ns() : 0ull;
        birth_claim_phase(p, gtid, gthreads, live_cum);
        if (blockIdx.x == 0 && (threadIdx.x & 31) == 0)  // summed warp durations of block 0
            atomicAdd(p.phase_ns + 8, globaltimer_ns() - h0);
        POST_SYNC(1);
        lap(1);
    }
    if (!MULTI) {
        // one world: block 0 ranks the births and resolves their winners, publishes the
        // birth lists with a release flag, then places the children and writes the counters
        // (t += 1).  The other blocks regrow the grid of step T+1 meanwhile (it needs only R''
        // of step T), wait for the flag and mutate the children's weights: no grid barrier
        // between the rank and the mutation, and the placement overlaps the mutation.
        unsigned long long *flag = bar + 2;
        // many eligible parents (a large world at its cap): claims on every thread and a grid
        // barrier; otherwise block 0 makes them itself, saving the barrier
        const bool claims_grid = *reinterpret_cast<volatile int32_t *>(p.n_cand) > CLAIMS_BLOCK_MAX;
        if (claims_grid) {
            birth_claims_grid(p, T, gtid, gthreads);
            grid_sync(bar, target, nthr);
        }
        if (blockIdx.x == 0) {
            if (gridDim.x == 1) move_claim_reset(p, T, threadIdx.x, blockDim.x);  // no other block
            if (!claims_grid) birth_claims_block<POST_THREADS>(p, T);  // the listed eligible parents
            lap(1);
            const RankCounts k = rank_counts(p, 0, T);
            rank_publish<POST_THREADS>(p, 0, T, k, scratch, s_free, s_bcell, s_par);
            if (threadIdx.x == 0) {
                // unique per launch (monotonic), with the number of births in the low 24 bits
                const unsigned long long v = ((target + 1) << 24) | (unsigned long long)k.n_place;
                asm volatile("st.release.gpu.u64 [%0], %1;" ::"l"(flag), "l"(v) : "memory");
            }
            lap(2);
            rank_place<POST_THREADS>(p, 0, T, k, s_free, s_bcell, s_par);
            if (threadIdx.x == 0) *p.p_children = p.split ? k.n_place : 0;  // the new children have no P row
#if ECO_METRICS & 2
            // the end of a movement window: block 0, idle after placing the children, closes it
            // (every live agent of step T+1 is final here; off the critical path)
            if (mv_window_end(T)) mv_pass_part(p, T, 0, 0, p.S, threadIdx.x, blockDim.x, s_mv);
#endif
            if (gr_window_end(T)) greed_pass_part(p, 0, 0, p.S, threadIdx.x, blockDim.x);  // greediness windows
            if (gridDim.x == 1) mutate_world(p, 0, T, k.n_place, threadIdx.x, blockDim.x);  // no other block
        } else {
            const unsigned nb = gridDim.x - 1, b = blockIdx.x - 1;
            const int gw = hh_split ? DYN_WARPS : POST_THREADS / 32;  // the regrowth and mutation warps
            const size_t btid = ((size_t)wid * nb + b) * 32 + lane;
            const size_t bthr = (size_t)nb * gw * 32;
            const uint64_t r0 = b == 0 ? globaltimer_ns() : 0ull;
            move_claim_reset(p, T, btid, bthr);
            if (!p.regrow_split) regrow_phase(p, T + 1, btid, bthr);
            if (b == 0 && lane == 0) atomicAdd(p.phase_ns + 9, globaltimer_ns() - r0);
#if ECO_MUT_WARM
            const MutArgs ma = mut_args(p);
            // warm the mutation's instruction lines on this SM's four sub-partitions (dry:
            // one item of a stale birth entry, no stores)
            if (wid >= 1 && wid <= 4) mutate_world_nl(ma, T, p.seeds[0], 1, lane, (size_t)1 << 30, 1);
#endif
            __shared__ int s_nb;
            if (threadIdx.x == 0) {
                unsigned long long cur;
                do {
                    asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(cur) : "l"(flag) : "memory");
                } while (cur < ((target + 1) << 24));
                s_nb = (int)(cur & 0xFFFFFFull);  // the births, carried by the flag itself
            }
            asm volatile("bar.sync 1, %0;" ::"r"(gw * 32) : "memory");
            const int n_b = s_nb;
#if ECO_MUT_WARM
            if (n_b > 0) mutate_world_nl(ma, T, p.seeds[0], n_b, btid, bthr, 0);
#else
            if (n_b > 0) mutate_world(p, 0, T, n_b, btid, bthr);
#endif
        }
    } else {
        // several worlds: one block per world ranks, places and counts them (t += 1); the
        // blocks without a world regrow step T+1; a barrier; then the mutation
        // (the blocks without a world take the first share of the regrowth's words, the ranking
        // blocks the rest once their world is ranked: a ranking block counts as ECO_RANK_SHARE
        // / 8 of a free one)
        const size_t rg_all = regrow_words(p);
        const size_t nfree = (int)gridDim.x > p.n_worlds ? gridDim.x - p.n_worlds : 0;
        const size_t rg_split = nfree ? rg_all * (8 * nfree) / (8 * nfree + (size_t)ECO_RANK_SHARE * p.n_worlds) : 0;
        if ((int)blockIdx.x < p.n_worlds) {
            for (int w = blockIdx.x; w < p.n_worlds; w += gridDim.x)
                birth_rank_world<POST_THREADS>(p, w, scratch, s_free, s_bcell, s_par);
            if (nfree && rg_split < rg_all) {
                const unsigned nb = p.n_worlds, b = blockIdx.x;
                const size_t btid = ((size_t)(threadIdx.x >> 5) * nb + b) * 32 + (threadIdx.x & 31);
                regrow_phase(p, T + 1, btid, (size_t)nb * blockDim.x, rg_split, rg_all);
            }
        } else {
            const unsigned nb = gridDim.x - p.n_worlds, b = blockIdx.x - p.n_worlds;
            const size_t btid = ((size_t)(threadIdx.x >> 5) * nb + b) * 32 + (threadIdx.x & 31);
            regrow_phase(p, T + 1, btid, (size_t)nb * blockDim.x, 0, rg_split);
        }
        POST_SYNC(2);
        lap(2);
#if ECO_METRICS & 2
        if (mv_window_end(T))  // movement windows: one block per world, after every placement
            for (int w = blockIdx.x; w < p.n_worlds; w += gridDim.x)
                mv_pass_part(p, T, w, 0, p.S, threadIdx.x, blockDim.x, s_mv);
#endif
        if (gr_window_end(T))  // greediness windows
            for (int w = blockIdx.x; w < p.n_worlds; w += gridDim.x)
                greed_pass_part(p, w, 0, p.S, threadIdx.x, blockDim.x);
        if (p.n_worlds >= (int)gridDim.x) {  // no block was free: the regrowth goes beside the mutation
            const size_t half = gthreads / 2;  // a multiple of 32: halves are whole warps
            if (gtid >= half) regrow_phase(p, T + 1, gtid - half, gthreads - half);
        }
        mutate_phase(p, gtid, gthreads, s_free, RANK_SMEM_CAP);  // (the rank's lists are consumed: s_free is free)
    }
#ifdef ECO_BLOCK_CLOCK
    __syncthreads();
    if (threadIdx.x == 0) p.phase_ns[ECO_BLOCK_CLOCK_BASE + (3 * gridDim.x + blockIdx.x) * 3] += globaltimer_ns() - bt_;
#endif
#ifdef ECO_END_CLOCK
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
    if (threadIdx.x == 0) atomicMax(ec + 2, (unsigned long long)globaltimer_ns());
#endif
#ifdef ECO_TIMELINE
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
    if (threadIdx.x == 0) timeline_mark(p, 3, globaltimer_ns(), T);
#endif
    if (clk) {
        lap(3);
        grid_sync_done(bar, target);
    }
}

// --------------------------------------------------------------------------- launchers
// ------------------------------------------------ a1, large grids: shared-memory tiles
// PAPER.md:255-267 as regrow_window, for grids of many words (the configs[2] benchmark
// grids, the first step of a large world).  A tile is RG_TH rows x RG_TW words; its window
// rows y0-2 .. y0+RG_TH+1 and words wx0-4 .. wx0+RG_TW+3 are staged in shared memory by
// 16-B cp.async copies (zero-filled off the grid) through an RG_STAGES-deep ring, so every
// block keeps RG_STAGES-1 tiles of loads in flight while it computes one (one HBM read per
// word; the halo re-reads of neighbouring tiles hit L2).  Each thread owns 4 consecutive
// words of a row (one 128-bit vector in and out).  The work of a tile is balanced over its
// 256 threads instead of one word per lane (which diverges as soon as one word of a warp
// needs its count or a draw): (1) the words holding an empty cell are listed, (2) one
// thread per listed word forms its bit-sliced count and a 2-bit class per cell and lists
// its 4-cell groups holding an empty cell, (3) one thread per listed group draws the Philox
// block and ORs the grown bits into the word, (4) each thread stores its 4 words (all-full
// words unchanged).  The grown count is summed per block and added once per world.
constexpr int RG_TW = 32, RG_TH = 32;            // 1024 words (32,768 cells) per tile
constexpr int RG_THREADS = 256;                  // one 4-word vector per thread
constexpr int RG_VW = (RG_TW + 8) / 4;           // uint4 per staged row (4-word halo each side)
constexpr int RG_SROWS = RG_TH + 4;
constexpr int RG_LOADS = RG_SROWS * RG_VW;       // 360 vectors per tile
#ifndef ECO_RG_STAGES
#define ECO_RG_STAGES 3
#endif
constexpr int RG_STAGES = ECO_RG_STAGES;
#ifndef ECO_RG_BPS
#define ECO_RG_BPS 4  // resident blocks per SM the tiled regrowth is compiled for (registers per thread)
#endif
constexpr int RG_WORDS = RG_TW * RG_TH;
static_assert(RG_WORDS == 4 * RG_THREADS, "one 4-word vector per thread");

// the tile's window (RG_LOADS vectors) and, after it, the thresholds of its RG_TH rows (one
// 16-B vector per row, zero past the handle's rows): staged together, so a tile waits on
// no dependent global load
constexpr int RG_STAGE_VECS = RG_LOADS + RG_TH;
constexpr int RG_DYN_SMEM = RG_STAGES * RG_STAGE_VECS * 16;
// (ro: this thread's one or two window vectors as word offsets from the tile's origin, made
// once per launch — a tile whose window lies inside the grid needs no bounds test and no
// index arithmetic per vector: the staging was 40 % of the full-grid kernel's instructions)
struct RgOff {
    int off0, off1;
    bool has1;
};
__device__ __forceinline__ RgOff rg_offsets(const DevParams &p) {
    RgOff o;
    const int k0 = threadIdx.x, k1 = threadIdx.x + RG_THREADS;
    static_assert(RG_LOADS > RG_THREADS && RG_LOADS <= 2 * RG_THREADS, "one or two window vectors per thread");
    o.off0 = (k0 / RG_VW - 2) * p.WW + 4 * (k0 % RG_VW) - 4;
    o.has1 = k1 < RG_LOADS;
    o.off1 = (k1 / RG_VW - 2) * p.WW + 4 * (k1 % RG_VW) - 4;
    return o;
}
__device__ __forceinline__ void rg_issue(const DevParams &p, const uint32_t *src, int y0, int wx0, uint4 *stage,
                                         const RgOff &ro) {
    if (y0 >= 2 && y0 + RG_TH + 2 <= p.H && y0 + RG_TH <= p.row_hi && wx0 >= 4 && wx0 + RG_TW + 4 <= p.WW) {
        if (threadIdx.x < RG_TH)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(stage + RG_LOADS + threadIdx.x)),
                         "l"(p.T + (size_t)(y0 + (int)threadIdx.x) * 4)
                         : "memory");
        const uint32_t *base = src + (size_t)y0 * p.WW + wx0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(stage + threadIdx.x)), "l"(base + ro.off0)
                     : "memory");
        if (ro.has1)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(stage + threadIdx.x + RG_THREADS)),
                         "l"(base + ro.off1)
                         : "memory");
        return;
    }
    for (int k = threadIdx.x; k < RG_TH; k += RG_THREADS) {
        const int y = y0 + k;
        const bool in = y < p.row_hi;
        const uint32_t *g = in ? p.T + (size_t)y * 4 : p.T;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(stage + RG_LOADS + k)), "l"(g),
                     "r"(in ? 16 : 0)
                     : "memory");
    }
    for (int k = threadIdx.x; k < RG_LOADS; k += RG_THREADS) {
        const int r = k / RG_VW, q = k - r * RG_VW;
        const int yy = y0 - 2 + r, ww = wx0 - 4 + 4 * q;  // ww, WW multiples of 4: aligned, in-row
        const bool in = yy >= 0 && yy < p.H && ww >= 0 && ww < p.WW;
        const uint32_t *g = in ? src + (size_t)yy * p.WW + ww : src;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(stage + k)), "l"(g),
                     "r"(in ? 16 : 0)
                     : "memory");
    }
}

__device__ __forceinline__ void rg_flush(const DevParams &p, int64_t tstep, int w, unsigned long long acc,
                                         unsigned long long *s_red) {
    acc = __reduce_add_sync(0xffffffffu, (unsigned)acc);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long sum = 0;
        for (int i = 0; i < RG_THREADS / 32; ++i) sum += s_red[i];
        if (sum) atomicAdd(reinterpret_cast<unsigned long long *>(&record_of(p, tstep, w)->grown), sum);
    }
    __syncthreads();
}

// 16 bits -> every other bit of 32 (bit i -> bit 2i)
__device__ __forceinline__ uint32_t spread16(uint32_t x) {
    x &= 0xFFFFu;
    x = (x | (x << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}

__global__ void __launch_bounds__(RG_THREADS, ECO_RG_BPS) k_regrow_tiled(DevParams p, int ahead) {
    extern __shared__ __align__(1024) uint4 rg_dyn[];  // the stage ring [RG_STAGES][RG_STAGE_VECS]
    uint4 (*s_ring)[RG_STAGE_VECS] = reinterpret_cast<uint4 (*)[RG_STAGE_VECS]>(rg_dyn);
    __shared__ uint32_t s_code[2][RG_WORDS];     // listed words: 2-bit class per cell (cells 0-15, 16-31)
#if ECO_STEP2_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");  // (a programmatic dependent in the agent-free step's graphs)
#endif
    __shared__ uint32_t s_grow[RG_WORDS];        // grown bits by tile word
    __shared__ uint16_t s_need[RG_WORDS];        // listed words (tile word index)
    __shared__ uint16_t s_item[RG_WORDS * 8];    // listed groups (list index << 3 | group)
    __shared__ int s_nneed, s_nitem;
    __shared__ unsigned long long s_red[RG_THREADS / 32];
    const int64_t tstep = p.t[0] + ahead;
    const int real_words = (p.W + 31) >> 5;
    const int ntx = (real_words + RG_TW - 1) / RG_TW, nty = (p.row_hi - p.row_lo + RG_TH - 1) / RG_TH;
    const int per_world = ntx * nty;
    const int ntiles = per_world * p.n_worlds;  // validated: n_worlds * H * words < 2^31
    const int lane = threadIdx.x & 31;
    const size_t pw = plane_words(p);
    constexpr int RS = RG_VW * 4;  // words per staged row
    // tile coordinates walked incrementally (block b visits tiles b, b + gridDim, ...): one
    // division per block instead of two per tile
    struct TileAt {
        int w, ty, tx;
    };
    auto decompose = [&](int tile) {
        TileAt a;
        a.w = tile / per_world;
        const int r = tile - a.w * per_world;
        a.ty = r / ntx;
        a.tx = r - a.ty * ntx;
        return a;
    };
    const TileAt stride = decompose((int)gridDim.x);
    auto advance = [&](TileAt &a) {
        a.tx += stride.tx;
        if (a.tx >= ntx) {
            a.tx -= ntx;
            ++a.ty;
        }
        a.ty += stride.ty;
        if (a.ty >= nty) {
            a.ty -= nty;
            ++a.w;
        }
        a.w += stride.w;
    };
    TileAt at_issue = decompose((int)blockIdx.x), at = at_issue;
    const RgOff ro = rg_offsets(p);
    auto issue = [&](int j) {  // the block's j-th tile into stage j % RG_STAGES (an empty group past the end)
        const int tile = blockIdx.x + j * gridDim.x;
        if (tile < ntiles)
            rg_issue(p, plane_cur(p, tstep) + (size_t)at_issue.w * pw, p.row_lo + at_issue.ty * RG_TH,
                     at_issue.tx * RG_TW, s_ring[j % RG_STAGES], ro);
        advance(at_issue);
        cp_commit();
    };
#pragma unroll
    for (int j = 0; j < RG_STAGES - 1; ++j) issue(j);
    // this thread's vector: row tr, words tq*4 .. tq*4+3 of the tile
    const int tr = threadIdx.x >> 3, tq = threadIdx.x & 7;
    unsigned long long acc = 0;
    int acc_w = -1;
    for (int j = 0;; ++j, advance(at)) {
        const int tile = blockIdx.x + j * gridDim.x;
        if (tile >= ntiles) break;
        const int w = at.w, y0 = p.row_lo + at.ty * RG_TH, wx0 = at.tx * RG_TW;
        if (w != acc_w) {  // block-uniform
            if (acc_w >= 0) rg_flush(p, tstep, acc_w, acc, s_red);
            acc_w = w;
            acc = 0;
        }
        cp_wait<RG_STAGES - 2>();
        if (threadIdx.x == 0) s_nneed = s_nitem = 0;
        __syncthreads();  // tile j staged for every thread; the previous tile's reads are done
        issue(j + RG_STAGES - 1);
        const uint32_t *sw = reinterpret_cast<const uint32_t *>(s_ring[j % RG_STAGES]);
        const uint32_t *sT = reinterpret_cast<const uint32_t *>(s_ring[j % RG_STAGES] + RG_LOADS);  // [RG_TH][4]
        const int y = y0 + tr, wxv = wx0 + 4 * tq;
        const bool row_ok = y < p.row_hi;
        const uint4 cur4 = *reinterpret_cast<const uint4 *>(sw + (tr + 2) * RS + 4 * tq + 4);
        // (0) a tile none of whose vectors holds a zero bit (the filled grid: nearly every tile
        // from t ~ 300 on) is copied through — no lists, no counts, no draws, one vote instead
        // of the scan and the second barrier (the all-full step executed 93 instructions per
        // word, 18 us for a 33.5 MB copy: instruction-bound)
        const bool in_tile = row_ok && wxv < real_words;
        const bool has_zero = (cur4.x & cur4.y & cur4.z & cur4.w) != 0xFFFFFFFFu;
        if (!__syncthreads_or(in_tile && has_zero)) {
            if (in_tile) {
                uint32_t *dst = plane_next(p, tstep) + (size_t)w * pw + (size_t)y * p.WW + wxv;
                if (wxv + 4 <= real_words) {
                    *reinterpret_cast<uint4 *>(dst) = cur4;
                } else {
                    const uint32_t ov[4] = {cur4.x, cur4.y, cur4.z, cur4.w};
                    for (int u = 0; wxv + u < real_words; ++u) dst[u] = ov[u];
                }
            }
            continue;
        }
        // (1) words holding an empty cell, listed
        uint32_t needm = 0u;
        {
            const uint32_t cw[4] = {cur4.x, cur4.y, cur4.z, cur4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (row_ok && wxv + u < real_words && !word_full(p, wxv + u, cw[u])) needm |= 1u << u;
        }
        *reinterpret_cast<uint4 *>(s_grow + 4 * threadIdx.x) = make_uint4(0u, 0u, 0u, 0u);
        {
            const int n = __popc(needm);
            int incl = n;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            int base = 0;
            if (lane == 31 && incl) base = atomicAdd(&s_nneed, incl);
            base = __shfl_sync(0xffffffffu, base, 31) + incl - n;
            while (needm) {
                const int u = __ffs(needm) - 1;
                needm &= needm - 1u;
                s_need[base++] = (uint16_t)(4 * threadIdx.x + u);
            }
        }
        __syncthreads();
        // (2) counts and 2-bit classes of the listed words, and their groups to draw (a tile
        // whose words are all full -- the saturated grid -- skips (2) and (3): block-uniform)
        const int nneed = s_nneed;
        if (nneed > 0) {
        for (int k = threadIdx.x; k < nneed; k += RG_THREADS) {
            const int tw = s_need[k];
            const int r = tw / RG_TW, col = tw - r * RG_TW;
            const int wx = wx0 + col;
            uint32_t win[5][3];
#pragma unroll
            for (int dr = 0; dr < 5; ++dr)
#pragma unroll
                for (int dw = 0; dw < 3; ++dw) win[dr][dw] = sw[(r + dr) * RS + col + 3 + dw];
            const uint32_t cur = win[2][1];
            uint32_t c[5] = {0u, 0u, 0u, 0u, 0u};
            auto add = [&](uint32_t cy) {  // bit-sliced counter += cy
                uint32_t tt;
                tt = c[0] & cy; c[0] ^= cy; cy = tt;
                tt = c[1] & cy; c[1] ^= cy; cy = tt;
                tt = c[2] & cy; c[2] ^= cy; cy = tt;
                tt = c[3] & cy; c[3] ^= cy; cy = tt;
                c[4] ^= cy;
            };
            if (p.disc12) {  // BASELINE's 12-cell disc, offsets compile-time (R4)
#pragma unroll
                for (int dr = 0; dr < 5; ++dr) {
                    const int m = dr == 2 ? 2 : (dr == 1 || dr == 3) ? 1 : 0;
#pragma unroll
                    for (int dx = -m; dx <= m; ++dx)
                        if (!(dr == 2 && dx == 0)) add(shifted_word(win[dr][0], win[dr][1], win[dr][2], dx));
                }
            } else {
#pragma unroll
                for (int dr = 0; dr < 5; ++dr) {
                    const int m = p.row_dx[dr];
#pragma unroll 1
                    for (int dx = -m; dx <= m; ++dx) {
                        if (dr == 2 && dx == 0) continue;
                        add(shifted_word(win[dr][0], win[dr][1], win[dr][2], dx));
                    }
                }
            }
            // class(k) = [k >= k1] + [k >= k2] + [k >= k3] (nested masks): low bit g1^g2^g3,
            // high bit g2; interleaved into 2 bits per cell
            const uint32_t g1 = ge_const(c, p.cls_k1), g2 = ge_const(c, p.cls_k2), g3 = ge_const(c, p.cls_k3);
            const uint32_t lo = g1 ^ g2 ^ g3, hi = g2;
            s_code[0][k] = spread16(lo) | (spread16(hi) << 1);
            s_code[1][k] = spread16(lo >> 16) | (spread16(hi >> 16) << 1);
            const int nv = p.W - (wx << 5);  // valid cells of the word
            const uint32_t empty = ~cur & (nv >= 32 ? 0xffffffffu : ((1u << nv) - 1u));
            uint32_t gm = 0u;
#pragma unroll
            for (int g = 0; g < 8; ++g) gm |= ((empty >> (4 * g)) & 0xFu) ? (1u << g) : 0u;
            int pos = atomicAdd(&s_nitem, __popc(gm));
            while (gm) {
                const int g = __ffs(gm) - 1;
                gm &= gm - 1u;
                s_item[pos++] = (uint16_t)((k << 3) | g);
            }
        }
        __syncthreads();
        // (3) one Philox block per listed group (the draw is keyed by the cell: exact)
        const int nitem = s_nitem;
        const uint64_t seed = p.seeds[w];
        for (int i = threadIdx.x; i < nitem; i += RG_THREADS) {
            const int it = s_item[i];
            const int k = it >> 3, g = it & 7;
            const int tw = s_need[k];
            const int r = tw >> 5, col = tw & 31;  // RG_TW = 32
            const int yy = y0 + r, x0 = ((wx0 + col) << 5) + 4 * g;
            const uint32_t cur = sw[(r + 2) * RS + col + 4];
            const uint32_t code = s_code[g >> 2][k] >> (8 * (g & 3));  // 2 bits per cell of the group
            const uint4 d = draw4(seed, PURPOSE_REGROW, (uint32_t)tstep, (uint32_t)(((int64_t)yy * p.W + x0) >> 2), 0u);
            const int nv = p.W - x0;
            const uint32_t empty4 = (~cur >> (4 * g)) & (nv >= 4 ? 0xFu : ((1u << nv) - 1u));
            const uint32_t *Tr = sT + 4 * r;
            uint32_t bits = 0u;
            bits |= (d.x < Tr[code & 3u]) ? 1u : 0u;
            bits |= (d.y < Tr[(code >> 2) & 3u]) ? 2u : 0u;
            bits |= (d.z < Tr[(code >> 4) & 3u]) ? 4u : 0u;
            bits |= (d.w < Tr[(code >> 6) & 3u]) ? 8u : 0u;
            bits &= empty4;
            if (bits) atomicOr(&s_grow[tw], bits << (4 * g));
        }
        __syncthreads();
        }  // nneed > 0
        // (4) this thread's 4 words (128-bit store when the whole vector is in the row)
        if (row_ok && wxv < real_words) {
            const uint4 g4 = *reinterpret_cast<const uint4 *>(s_grow + 4 * threadIdx.x);
            const uint4 o = make_uint4(cur4.x | g4.x, cur4.y | g4.y, cur4.z | g4.z, cur4.w | g4.w);
            uint32_t *dst = plane_next(p, tstep) + (size_t)w * pw + (size_t)y * p.WW + wxv;
            if (wxv + 4 <= real_words) {
                *reinterpret_cast<uint4 *>(dst) = o;
            } else {
                const uint32_t ov[4] = {o.x, o.y, o.z, o.w};
                for (int u = 0; wxv + u < real_words; ++u) dst[u] = ov[u];
            }
            acc += (unsigned long long)(__popc(g4.x) + __popc(g4.y) + __popc(g4.z) + __popc(g4.w));
        }
    }
    cp_wait<0>();
    if (acc_w >= 0) rg_flush(p, tstep, acc_w, acc, s_red);
}

// words of all worlds from which the tiled kernel is used (the per-word gather path keeps
// small grids on up to 8 lanes per word, shorter Philox chains)
constexpr size_t RG_TILED_MIN_WORDS = 65536;

// An agent-free world (no slots: the configs[2] regrowth grids): a step is the regrowth kernel
// and this bookkeeping — the record and counters of step t+1 from zero, step t's record
// (resources += grown, as the rank's last thread writes it), t += 1 — one thread per world;
// no policy launch and no k_post (which would sweep a 16.8 MB claimed-cell bitmap and run
// five empty phases: 47 of the 94 us per step at 8192x16384).
__global__ void __launch_bounds__(256) k_advance_empty(DevParams p) {
#if ECO_STEP2_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous regrowth's counts are complete
#endif
    for (int w = threadIdx.x; w < p.n_worlds; w += blockDim.x) {
        const int64_t t = p.t[w];
        housekeeping_world(p, w);
        rank_finalize(p, w, t, 0, 0, 0, 0);
        p.t[w] = t + 1;
    }
}
cudaError_t launch_advance_empty(const DevParams &p, cudaStream_t s) {
#if ECO_STEP2_PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_advance_empty, p);
#else
    k_advance_empty<<<1, 256, 0, s>>>(p);
    return cudaGetLastError();
#endif
}

bool regrow_tiled(const DevParams &p) {
    const int real_words = (p.W + 31) >> 5;
    return (size_t)(p.row_hi - p.row_lo) * real_words * p.n_worlds >= RG_TILED_MIN_WORDS;
}

cudaError_t launch_regrow(const DevParams &p, int ahead, cudaStream_t s) {
    const int real_words = (p.W + 31) >> 5;
    const size_t items = (size_t)(p.row_hi - p.row_lo) * real_words * p.n_worlds;
    if (regrow_tiled(p)) {
        static int bps = 0;
        if (bps == 0) {
            set_dyn_smem(k_regrow_tiled, RG_DYN_SMEM);
            cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_regrow_tiled, RG_THREADS, RG_DYN_SMEM);
            if (e != cudaSuccess || bps < 1) bps = 4;
        }
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const size_t ntiles =
            (size_t)p.n_worlds * ((p.row_hi - p.row_lo + RG_TH - 1) / RG_TH) * ((real_words + RG_TW - 1) / RG_TW);
        size_t blocks = (size_t)sms * bps;
        if (blocks > ntiles) blocks = ntiles;
#if ECO_STEP2_PDL
        if (p.S == 0 && p.regrow_split) {  // the agent-free step: a programmatic dependent of k_advance_empty
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)blocks);
            cfg.blockDim = dim3(RG_THREADS);
            cfg.dynamicSmemBytes = RG_DYN_SMEM;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            return cudaLaunchKernelEx(&cfg, k_regrow_tiled, p, ahead);
        }
#endif
        k_regrow_tiled<<<(unsigned)blocks, RG_THREADS, RG_DYN_SMEM, s>>>(p, ahead);
        return cudaGetLastError();
    }
    size_t blocks = (items + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_regrow<<<(unsigned)blocks, 256, 0, s>>>(p, ahead);
    return cudaGetLastError();
}

#include "coloc.cuh"

cudaError_t launch_move(const DevParams &p, const LaunchCfg &lc, cudaStream_t s) {
    if (p.S == 0) return cudaSuccess;
    if (p.coloc) {  // co-location: the move (and lottery keys), then consumption .. death
        k_co_move<<<lc.agent_blocks, lc.agent_threads, 0, s>>>(p);
        k_co_live<<<lc.agent_blocks, lc.agent_threads, 0, s>>>(p);
        return cudaGetLastError();
    }
    if (paper_rules(p)) k_move<true><<<lc.agent_blocks, lc.agent_threads, 0, s>>>(p);
    else k_move<false><<<lc.agent_blocks, lc.agent_threads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_birth_claim(const DevParams &p, const LaunchCfg &lc, cudaStream_t s) {
    if (p.S == 0 || p.coloc) return cudaSuccess;  // (co-location: no birth claims)
    k_birth_claim<<<lc.agent_blocks, lc.agent_threads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_birth_rank(const DevParams &p, cudaStream_t s) {
    if (p.coloc) {  // (the regrowth of step t+1 is graph mode's: launch_post)
        k_co_rank<<<p.n_worlds, CO_THREADS, 0, s>>>(p);
        return cudaGetLastError();
    }
    k_birth_rank<<<p.n_worlds, RANK_THREADS, 0, s>>>(p);
    k_mv_pass<<<p.n_worlds, 256, 0, s>>>(p);  // movement / greediness windows ending here (after placement)
    return cudaGetLastError();
}

cudaError_t launch_mv_pass(const DevParams &p, cudaStream_t s) {
    k_mv_pass<<<p.n_worlds, 256, 0, s>>>(p);  // movement / greediness windows ending here
    return cudaGetLastError();
}

bool policy_supports_shard() { return true; }  // k_policy_half honours ownership

cudaError_t launch_prepare_p_snap(const DevParams &p, const int64_t *snap, cudaStream_t s) {
    if (!p.split) return cudaSuccess;
    const unsigned blocks = (unsigned)((p.S + HALF_AGENTS - 1) / HALF_AGENTS);
    k_prepare_p_snap<<<blocks > 0 ? blocks : 1, HALF_THREADS, HALF_SMEM, s>>>(p, snap);
    return cudaGetLastError();
}

cudaError_t launch_prepare_p_list(const DevParams &p, const int32_t *list, const int32_t *n, int sms, cudaStream_t s) {
    if (!p.split) return cudaSuccess;
    k_prepare_p_list<<<sms > 0 ? sms : 1, HALF_THREADS, HALF_SMEM, s>>>(p, list, n);
    return cudaGetLastError();
}

cudaError_t launch_prepare_p(const DevParams &p, const LaunchCfg &lc, cudaStream_t s) {
    if (!p.split) return cudaSuccess;
    const unsigned blocks = (unsigned)((p.S + HALF_AGENTS - 1) / HALF_AGENTS);
    k_prepare_p<<<blocks > 0 ? blocks : 1, HALF_THREADS, HALF_SMEM, s>>>(p);
    return cudaGetLastError();
}

__global__ void k_set_owner(DevParams p) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < p.S; k += gridDim.x * blockDim.x) {
        p.owner[k] = (uint8_t)(k % p.n_ranks);
        p.mrec_slot[k] = make_int4(0, 0, 0, 0);
    }
}

// this rank's own live slots of step t (one block: order is irrelevant to every result)
__global__ void k_build_own(DevParams p) {
    const int64_t t = p.t[0];
    const int n = *count_of(p, t, 0);
    __shared__ int cnt;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const int slot = list_of(p, t, 0)[k];
        if (p.owner[slot] == p.rank) p.own_list[(t & 1) * p.S + atomicAdd(&cnt, 1)] = slot;
    }
    __syncthreads();
    if (threadIdx.x == 0) p.own_count[t & 1] = cnt;
}

cudaError_t launch_set_owner(const DevParams &p, cudaStream_t s) {
    if (p.S == 0 || !p.owner) return cudaSuccess;
    k_set_owner<<<256, 256, 0, s>>>(p);
    if (p.n_ranks > 1 && p.n_worlds == 1) k_build_own<<<1, 1024, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_mutate(const DevParams &p, const LaunchCfg &lc, cudaStream_t s) {
    if (p.S == 0) return cudaSuccess;
    k_mutate<<<lc.sms * 8, 256, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t post_occupancy(int *blocks_per_sm) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_post<false, true>, POST_THREADS, POST_SMEM);
}

cudaError_t post_prepare() {
    cudaError_t e = set_dyn_smem(k_post_co, 0);
    if (e != cudaSuccess) return e;
    e = set_dyn_smem(k_post<true>, POST_SMEM_SMALL);
    if (e != cudaSuccess) return e;
    e = set_dyn_smem(k_post<false, true>, POST_SMEM);
    if (e != cudaSuccess) return e;
    e = set_dyn_smem(k_post<true, true>, POST_SMEM);
    if (e != cudaSuccess) return e;
    e = set_dyn_smem(k_post<false, false, true>, POST_SMEM_SMALL);
    if (e != cudaSuccess) return e;
    e = set_dyn_smem(k_post<false, false, false, true>, POST_SMEM_SMALL);
    if (e != cudaSuccess) return e;
    e = set_dyn_smem(k_post<false, false, true, true>, POST_SMEM_SMALL);
    if (e != cudaSuccess) return e;
    e = set_dyn_smem(k_post<false, true, true>, POST_SMEM);
    if (e != cudaSuccess) return e;
    return set_dyn_smem(k_post<false>, POST_SMEM_SMALL);
}

cudaError_t launch_post(const DevParams &p, const LaunchCfg &lc, unsigned long long *bar, cudaStream_t s) {
    if (p.coloc) {  // co-location (coloc.cuh): one cooperative launch, the phases split by grid barriers
        if (p.S == 0) return launch_regrow(p, 0, s);
        cudaLaunchConfig_t cc = {};
        cc.gridDim = dim3(lc.post_blocks);
        cc.blockDim = dim3(CO_THREADS);
        cc.stream = s;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cc.attrs = at;
        cc.numAttrs = 1;
#if ECO_POST_PDL
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // scheduled while the policy drains
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cc.numAttrs = 2;
#endif
        return cudaLaunchKernelEx(&cc, k_post_co, p, bar);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(lc.post_blocks);
    cfg.blockDim = dim3(POST_THREADS);
    cfg.dynamicSmemBytes = post_smem_bytes(p);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
#if ECO_POST_PDL
    // programmatic dependent launch: k_post's blocks are scheduled while the policy drains;
    // every thread waits (griddepcontrol.wait) for the policy grid's completion first
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 2;
#endif
    if (p.n_ranks > 1 && paper_rules(p)) return cudaErrorInvalidValue;  // (sim_shard refuses the paper rules)
    if (p.n_ranks > 1) return cudaLaunchKernelEx(&cfg, post_big(p) ? k_post<true, true> : k_post<true>, p, bar);
    if (p.n_worlds > 1)  // (post_big needs the split policy, i.e. one world)
        return cudaLaunchKernelEx(&cfg, paper_rules(p) ? k_post<false, false, true, true> : k_post<false, false, false, true>, p, bar);
    if (paper_rules(p))
        return cudaLaunchKernelEx(&cfg, post_big(p) ? k_post<false, true, true> : k_post<false, false, true>, p, bar);
    if (post_big(p)) return cudaLaunchKernelEx(&cfg, k_post<false, true>, p, bar);
    return cudaLaunchKernelEx(&cfg, k_post<false>, p, bar);
}

}  // namespace eco
