// phases.cuh — the phases of one world step as device functions, shared by the standalone
// kernels (instrumented mode) and the fused kernels of graph mode.
//
//   regrow_phase       a1  grid regrowth of a step, 1..8 lanes per 32-cell word
//   move_phase         a4  claim resolution, movement, consumption, physiology, death
//   birth_claim_phase  a5  lazy move-claim reset, birth candidate, claimed-cell dedup
//   birth_rank_world   a5  (one block per world) free slots, claimed cells in row-major
//                          order, claim winners, placement, counters, t += 1
//   mutate_phase       a5  children's weights (coalesced, one device weight per item)
//
// Data written by one phase and read by a later phase of the same kernel is read with
// plain (coherent) loads, never through the read-only path.
#pragma once
#include "block_scan.cuh"
#include "sim_internal.cuh"

namespace eco {

// ------------------------------------------------------------------ grid barrier
// Release/acquire barrier over all blocks of a cooperatively launched grid (co-residency
// guaranteed by the cooperative launch).  bar[0] counts arrivals monotonically across
// launches; `target` starts at grid_sync_base() and grows by gridDim per barrier.
__device__ __forceinline__ void grid_sync(unsigned long long *bar, unsigned long long &target, int nthr) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
    target += gridDim.x;
    if (threadIdx.x == 0) {
        unsigned long long cur;
        asm volatile("atom.add.release.gpu.u64 %0, [%1], 1;" : "=l"(cur) : "l"(bar) : "memory");
        cur += 1;
        while (cur < target) asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(cur) : "l"(bar) : "memory");
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
}
__device__ __forceinline__ void grid_sync(unsigned long long *bar, unsigned long long &target) {
    grid_sync(bar, target, blockDim.x);
}

// bar[1] holds the arrival count after the previous launch's last barrier (the launches
// may differ in their number of barriers); every block reads it before its first arrival.
__device__ __forceinline__ unsigned long long grid_sync_base(const unsigned long long *bar) {
    return *reinterpret_cast<const volatile unsigned long long *>(bar + 1);
}

// called once per launch after its last barrier by one thread of block 0
__device__ __forceinline__ void grid_sync_done(unsigned long long *bar, unsigned long long target) {
    *reinterpret_cast<volatile unsigned long long *>(bar + 1) = target;
}

__device__ __forceinline__ uint32_t ld_plain(const uint32_t *p) { return *reinterpret_cast<const volatile uint32_t *>(p); }

// Warp-interleaved global thread index (a permutation of [0, gridDim*blockDim)): warp k of
// the work goes to block k % gridDim, so short phases spread over every SM.
__device__ __forceinline__ size_t interleaved_gtid() {
    return ((size_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x) * 32 + (threadIdx.x & 31);
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Warp-aggregated "+v per lane" on a per-world counter (one atomic per warp when the
// warp's lanes share a world, which holds whenever S is a multiple of 32).
template <typename T, typename AddrOf>
__device__ __forceinline__ void warp_world_add(T v, int w, AddrOf addr_of) {
    const unsigned lane = threadIdx.x & 31;
    const int w0 = __shfl_sync(0xffffffffu, w, 0);
    if (__all_sync(0xffffffffu, w == w0)) {
        T s = v;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0 && s) atomicAdd(addr_of(w0), s);
    } else if (v) {
        atomicAdd(addr_of(w), v);
    }
}

// ----------------------------------------------------------------------- a1 regrow
// each empty cell grows with p = lat(y)*f(k) + c, k = resources in the
// Euclidean radius-r disc (centre excluded) of the START-of-step grid (synchronous),
// drawn as philox(REGROW, t, cell>>2)[cell&3] < T[y][class(k)].  Full cells stay full.
// The 12 (generally <= 24) neighbour bit-vectors are funnel-shifted words of rows y-2..y+2;
// k is accumulated bit-sliced (5 planes), ~10 logic ops per neighbour per 32 cells.  Philox runs only for 4-cell groups holding an empty cell (exact: draws are keyed
// by cell, not by sequence).
__device__ __forceinline__ uint32_t shifted_word(uint32_t prv, uint32_t cur, uint32_t nxt, int dx) {
    if (dx > 0) return __funnelshift_r(cur, nxt, dx);
    if (dx < 0) return __funnelshift_l(prv, cur, -dx);
    return cur;
}

__device__ __forceinline__ uint32_t ge_const(const uint32_t c[5], int m) {
    if (m <= 0) return 0xffffffffu;
    if (m >= 32) return 0u;
    uint32_t gt = 0u, eq = 0xffffffffu;
#pragma unroll
    for (int i = 4; i >= 0; --i) {
        if ((m >> i) & 1) {
            eq &= c[i];
        } else {
            gt |= eq & c[i];
            eq &= ~c[i];
        }
    }
    return gt | eq;
}

// The grown bits of groups [g0, g0 + ng) (4 cells each) of word (y, wx) of world w for step
// `t`, given its window win[dy + 2][dw + 1] = word (y + dy, wx + dw) of R_t (0 off-grid) and
// cur = win[2][1].  Shared by the L2-gather path below and the shared-memory-tiled kernel.
__device__ __forceinline__ uint32_t regrow_window(const DevParams &p, int w, int y, int wx, int64_t t, int g0, int ng,
                                                  const uint32_t (&win)[5][3], uint32_t cur) {
    uint32_t c[5] = {0u, 0u, 0u, 0u, 0u};
#pragma unroll
    for (int r = 0; r < 5; ++r) {  // disc row dy = r - 2: offsets dx = -m..m (compact loop)
        const int m = p.row_dx[r];
        const uint32_t prv = win[r][0], cen = win[r][1], nxt = win[r][2];
#pragma unroll 1
        for (int dx = -m; dx <= m; ++dx) {
            if (r == 2 && dx == 0) continue;
            uint32_t cy = shifted_word(prv, cen, nxt, dx), tt;
            tt = c[0] & cy; c[0] ^= cy; cy = tt;
            tt = c[1] & cy; c[1] ^= cy; cy = tt;
            tt = c[2] & cy; c[2] ^= cy; cy = tt;
            tt = c[3] & cy; c[3] ^= cy; cy = tt;
            c[4] ^= cy;
        }
    }
    const uint32_t ge1 = ge_const(c, p.cls_k1), ge2 = ge_const(c, p.cls_k2), ge3 = ge_const(c, p.cls_k3);
    const uint4 Trow = *reinterpret_cast<const uint4 *>(p.T + (size_t)y * 4);
    const uint64_t seed = p.seeds[w];
    const int x_base = wx << 5;
    uint32_t grow = 0u;
#pragma unroll 1
    for (int g = g0; g < g0 + ng; ++g) {
        const int x0 = x_base + 4 * g;
        if (x0 >= p.W) break;
        if (((cur >> (4 * g)) & 0xFu) == 0xFu) continue;  // all four cells full: no draw needed
        const uint32_t entity = (uint32_t)(((int64_t)y * p.W + x0) >> 2);
        const uint4 d = draw4(seed, PURPOSE_REGROW, (uint32_t)t, entity, 0u);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int b = 4 * g + m;
            if ((cur >> b) & 1u) continue;
            const int cls = (int)((ge1 >> b) & 1u) + (int)((ge2 >> b) & 1u) + (int)((ge3 >> b) & 1u);
            const uint32_t thr = cls == 0 ? Trow.x : cls == 1 ? Trow.y : cls == 2 ? Trow.z : Trow.w;
            if (word_of(d, m) < thr) grow |= 1u << b;
        }
    }
    return grow;
}

// a word whose real cells are all full cannot grow: no window, no count, no draw
__device__ __forceinline__ bool word_full(const DevParams &p, int wx, uint32_t cur) {
    const int nv = p.W - (wx << 5);  // valid cells in the word
    const uint32_t pad = nv >= 32 ? 0u : ~((1u << nv) - 1u);
    return (cur | pad) == 0xFFFFFFFFu;
}

// Regrow groups [g0, g0 + ng) of word (y, wx) of world w for step `t`, the window gathered
// from src = plane_cur(t) with coherent loads (inside the cooperative kernel the plane was
// written earlier in the same launch).  Returns the grown bits (the caller ORs the lanes of
// the word and stores cur | grow into plane_next(t)); `cur` gets the word's current bits.
__device__ __forceinline__ uint32_t regrow_groups(const DevParams &p, int w, int y, int wx, int64_t t, int g0, int ng,
                                                  uint32_t &cur) {
    const uint32_t *src = plane_cur(p, t) + (size_t)w * plane_words(p);
    cur = ld_plain(src + (size_t)y * p.WW + wx);
    if (word_full(p, wx, cur)) return 0u;
    uint32_t win[5][3];
#pragma unroll
    for (int dy = -2; dy <= 2; ++dy) {
        const int yy = y + dy;
#pragma unroll
        for (int dw = -1; dw <= 1; ++dw) {
            const int ww = wx + dw;
            win[dy + 2][dw + 1] =
                (yy >= 0 && yy < p.H && ww >= 0 && ww < p.WW) ? ld_plain(src + (size_t)yy * p.WW + ww) : 0u;
        }
    }
    return regrow_window(p, w, y, wx, t, g0, ng, win, cur);
}

// Grid-stride regrowth of every world for step `tstep` (all worlds share t).  A word's 8
// four-cell groups are split over L = 1..8 consecutive lanes (as many as the threads allow:
// a small grid gets 8 short chains per word instead of one long one); the lanes of a word
// OR their grown bits and the first stores the word.  One atomic per warp on the world's
// record of that step.  Must be called by all 32 lanes of a warp.
// (k_lo, k_hi: the words [k_lo, min(k_hi, all)) of the world-major word sequence only — two
// groups of blocks sharing one regrowth.)
__device__ __forceinline__ size_t regrow_words(const DevParams &p) {
    return (size_t)(p.row_hi - p.row_lo) * ((p.W + 31) >> 5) * p.n_worlds;
}
__device__ __forceinline__ void regrow_phase(const DevParams &p, int64_t tstep, size_t gtid, size_t gthreads,
                                             size_t k_lo = 0, size_t k_hi = ~(size_t)0) {
    const int real_words = (p.W + 31) >> 5;
    const int rows = p.row_hi - p.row_lo;  // the rows this handle owns (all H unless banded)
    const size_t per_world = (size_t)rows * real_words;
    const size_t all = per_world * p.n_worlds;
    if (k_hi > all) k_hi = all;
    if (k_lo >= k_hi) return;
    const size_t total = k_hi - k_lo;
    int lsh = 0;  // L = 1 << lsh lanes per word
    while (lsh < 3 && (total << (lsh + 1)) <= gthreads) ++lsh;
    const int L = 1 << lsh, ng = 8 >> lsh;
    const size_t items = total << lsh;
    const unsigned lane = gtid & 31;
    for (size_t base = gtid - lane; base < items; base += gthreads) {
        const size_t it = base + lane;
        const size_t k = k_lo + (it >> lsh);
        const int sub = (int)(it & (L - 1));
        int w = 0, y = 0, wx = 0;
        uint32_t grow = 0u, cur = 0u;
        if (it < items) {  // 32-bit index arithmetic (validated: H * words * worlds < 2^32)
            const uint32_t k32 = (uint32_t)k, pw32 = (uint32_t)per_world;
            w = (int)(k32 / pw32);
            const uint32_t r = k32 - (uint32_t)w * pw32;
            y = (int)(r / (uint32_t)real_words);
            wx = (int)(r - (uint32_t)y * (uint32_t)real_words);
            y += p.row_lo;
            grow = regrow_groups(p, w, y, wx, tstep, sub * ng, ng, cur);
        }
        for (int o = 1; o < L; o <<= 1) grow |= __shfl_xor_sync(0xffffffffu, grow, o);
        unsigned long long cnt = 0;
        if (it < items && sub == 0) {
            plane_next(p, tstep)[(size_t)w * plane_words(p) + (size_t)y * p.WW + wx] = cur | grow;
            cnt = (unsigned long long)__popc(grow);
        }
        warp_world_add<unsigned long long>(cnt, w, [&](int ww) {
            return reinterpret_cast<unsigned long long *>(&record_of(p, tstep, ww)->grown);
        });
    }
}

// ------------------------------------------------------------------- agent iteration
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

// Several worlds: the LIVE list positions of step t of all worlds as one world-major sequence
// (a world holds ~1,100 agents in 8,192 slots: a thread striding over every slot of every
// world runs 4-5 dependent iterations, most of them on empty positions).  live_prefix makes
// cum[w] = the live positions of the worlds before w (cum[n_worlds] = all) in the block's
// shared array (warp 0; every thread of the block calls it; ends with a block barrier).
__device__ __forceinline__ void live_prefix(const DevParams &p, int64_t t, int *cum) {
    if (threadIdx.x < 32) {
        const int lane = (int)threadIdx.x, par = (int)(t & 1);
        int run = 0;
        for (int w0 = 0; w0 < p.n_worlds; w0 += 32) {
            const int wl = w0 + lane;
            const int cnt = wl < p.n_worlds ? p.n_alive[par * p.n_worlds + wl] : 0;
            int inc = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int up = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += up;
            }
            if (wl < p.n_worlds) cum[wl] = run + inc - cnt;
            run += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) cum[p.n_worlds] = run;
    }
    __syncthreads();
}
__device__ __forceinline__ AgentIter agent_at_live(const DevParams &p, const int *cum, long g) {
    AgentIter a;
    a.in_range = g < (long)cum[p.n_worlds];
    int lo = 0, hi = p.n_worlds;  // cum[lo] <= g < cum[hi]: the last such lo
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if ((long)cum[mid] <= g) lo = mid;
        else hi = mid;
    }
    a.w = a.in_range ? lo : 0;
    a.i = a.in_range ? (int)(g - cum[lo]) : 0;
    return a;
}

// ------------------------------------------------- Appendix C movement metrics (NEXT-3)
#ifndef ECO_METRICS
#define ECO_METRICS 3  // bit 0: ages at death, bit 1: movement histograms (diagnostic switch)
#endif
// Each slot keeps (cell, inv) from the start of its current 50-step window, inv = age - 50k
// for window k: an agent alive through window k has the same inv at the start of window k+1,
// and nothing else does (a newborn's or a reused slot's inv is smaller), so no per-slot flag
// has to be cleared when agents die or are born.  mv_pass runs at the end of window k (step
// T = 50k+49, after the children of that step are placed, so every live slot is final):
// every live slot whose inv is unchanged gets the bin of the Manhattan distance between the
// two cells, and every live slot (a newborn too, at age 0) starts window k+1.
constexpr int32_t MV_INVALID = -(1 << 29);
__device__ __forceinline__ bool mv_window_end(int64_t T) { return (uint32_t)T % SIM_MOVE_WINDOW == SIM_MOVE_WINDOW - 1; }

// Slots [lo, hi) of world w by `nthr` threads of one block (thread index tid; named barrier 1
// over exactly those threads), counted in a shared histogram, then one global atomic per
// non-empty bin (a grid-wide per-warp scheme serialises thousands of same-address atomics).
__device__ __forceinline__ void mv_pass_part(const DevParams &p, int64_t T, int w, int lo, int hi, int tid, int nthr,
                                             int *s_hist, int bar_id = 1) {
    const uint32_t k = (uint32_t)T / SIM_MOVE_WINDOW;
    for (int b = tid; b < SIM_MOVE_BINS; b += nthr) s_hist[b] = 0;
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthr) : "memory");
    for (int i = lo + tid; i < hi; i += nthr) {
        const size_t gs = (size_t)w * p.S + i;
        if (!p.alive[gs]) continue;
        const int c1 = p.cell[gs];
        const int32_t inv = p.age[gs] - SIM_MOVE_WINDOW * (int32_t)(k + 1);
        if (p.mv_inv[gs] == inv) {
            const int c0 = p.mv_cell[gs];
            const int y0 = row_of(p, c0), y1 = row_of(p, c1);
            const int d = abs(y1 - y0) + abs((c1 - y1 * p.W) - (c0 - y0 * p.W));
            atomicAdd(s_hist + min(d / 3, SIM_MOVE_BINS - 1), 1);
        }
        p.mv_cell[gs] = c1;
        p.mv_inv[gs] = inv;
    }
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthr) : "memory");
    int32_t *hist = p.mv_hist + ((size_t)w * p.mv_cap + (size_t)(k & (p.mv_cap - 1))) * SIM_MOVE_BINS;
    for (int b = tid; b < SIM_MOVE_BINS; b += nthr)
        if (s_hist[b]) atomicAdd(hist + b, s_hist[b]);
}

// ----------------------------------------------------------------------- a4 move
// An agent moves iff it holds the max key on its target (R14); every live agent eats the
// resource under its final cell; fixed-point energy e += gain*ate - decay,
// age += 1, repr = e > thr ? repr+1 : 0 (R16, R17, R19); death iff e <= 0 (cause energy)
// or age > max_age (cause age) (R18).  O is updated in place with bit atomics; distinct
// agents touch distinct bits.  Survivors are appended to the step-(t+1) list (order is
// irrelevant to every result).  Must be called by all 32 lanes of a warp.
// PAPER: the paper world's death timer and lethal walls (death_steps > 0 or lethal_walls),
// compiled into separate kernels so BASELINE's move phase keeps its code (measured: the
// runtime checks cost 6 us per capped paper-scale step).
// live_cum: live_prefix's array (several worlds: only live list positions are visited), or null.
template <bool PAPER = false>
__device__ __forceinline__ void move_phase(const DevParams &p, size_t gtid, size_t gthreads,
                                           const int *live_cum = nullptr) {
    const long total = live_cum ? (long)live_cum[p.n_worlds] : (long)p.n_worlds * p.S;
    const size_t HW = (size_t)p.H * p.W;
    const unsigned lane = gtid & 31;
    for (long base = (long)(gtid - lane); base < total; base += (long)gthreads) {
        const AgentIter it = live_cum ? agent_at_live(p, live_cum, base + lane) : agent_at(p, base + lane);
        const int w = it.w;
        // t, both parities' counts and the move record of list position i load together
        // (entries past the count are stale and unused)
        int64_t t = 0;
        int n_list = 0;
        int4 mr = make_int4(0, 0, -1, 0);
        if (it.in_range) {
            t = p.t[w];
            const int n0 = p.n_alive[w], n1 = p.n_alive[p.n_worlds + w];
            mr = p.mrec[(size_t)w * p.S + it.i];  // (slot, cell, target, key hi) from the policy
            n_list = (t & 1) ? n1 : n0;
        }
        const bool active = it.in_range && it.i < n_list;
        bool ate = false, died_e = false, died_a = false, died_w = false, survive = false, cand = false;
        int cand_cell = 0;
        int slot = 0;
        int dage = 0;  // metrics: age at death
        if (PAPER && active && mr.z == WALL_TARGET) {  // walked into a lethal wall: dies before eating
            slot = mr.x;
            const size_t gs = (size_t)w * p.S + slot;
            uint32_t bit;
            p.alive[gs] = 0;
            p.ate[gs] = 0;
            greed_update(p, gs, t, false);
            atomicAnd(word_ptr(p.occ + (size_t)w * plane_words(p), p, mr.y, bit), ~bit);
            atomicAnd(p.alive_bits + (size_t)w * p.SW + (slot >> 5), ~(1u << (slot & 31)));
            died_w = true;
#if ECO_METRICS & 1
            dage = p.age[gs] + 1;
#endif
        } else if (active) {
            slot = mr.x;
            ECO_CHECK(slot >= 0 && slot < p.S && (mr.z < 0 || (int64_t)mr.z < (int64_t)p.H * p.W));
            const size_t gs = (size_t)w * p.S + slot;
            uint32_t *O = p.occ + (size_t)w * plane_words(p);
            uint32_t *Rn = plane_next(p, t) + (size_t)w * plane_words(p);
            int cellv = mr.y;
            const int tg = mr.z;
            const unsigned long long key =
                ((unsigned long long)(uint32_t)mr.w << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)cellv);
            // independent loads issued together: the SoA fields, the target's claim and the
            // R'' words of both possible final cells (only this agent consumes its final cell)
            int en0 = p.energy[gs], ag0 = p.age[gs], rp0 = p.repr[gs];
            uint32_t bit, bit_t = 0u;
            uint32_t *rw = word_ptr(Rn, p, cellv, bit), *rw_t = nullptr;
            const unsigned long long ck = tg >= 0 ? p.claim[(size_t)w * HW + tg] : 0ull;  // (tg -2: never here)
            uint32_t r_c = ld_plain(rw), r_t = 0u;
            if (tg >= 0) {
                rw_t = word_ptr(Rn, p, tg, bit_t);
                r_t = ld_plain(rw_t);
            }
            if (tg >= 0 && ck == key) {
                uint32_t ob;
                atomicAnd(word_ptr(O, p, cellv, ob), ~ob);
                atomicOr(word_ptr(O, p, tg, ob), ob);
                cellv = tg;
                p.cell[gs] = tg;
                rw = rw_t;
                bit = bit_t;
                r_c = r_t;
            }
            if (r_c & bit) {
                atomicAnd(rw, ~bit);
                ate = true;
            }
            p.ate[gs] = ate ? 1 : 0;
            greed_update(p, gs, t, ate);
            long long e = (long long)en0 + (ate ? (long long)p.e_gain : 0ll) - (long long)p.e_decay;
            if (p.e_max != 0x7fffffff && e > p.e_max) e = p.e_max;
            const int en = (int)e;
            const int ag = ag0 + 1;
            p.energy[gs] = en;
            p.age[gs] = ag;
            p.repr[gs] = en > p.e_repr_gt ? rp0 + 1 : 0;
            if (PAPER ? starves(p, gs, en) : en <= p.e_death_le) died_e = true;
            else if (ag > p.max_age) died_a = true;
            if (died_e || died_a) {
                p.alive[gs] = 0;
                atomicAnd(word_ptr(O, p, cellv, bit), ~bit);
                atomicAnd(p.alive_bits + (size_t)w * p.SW + (slot >> 5), ~(1u << (slot & 31)));
#if ECO_METRICS & 1
                dage = ag;
#endif
            } else {
                survive = true;
                cand = p.n_worlds == 1 && p.repr[gs] >= p.repr_steps;
                cand_cell = cellv;
            }
        }
        const int w0 = __shfl_sync(0xffffffffu, w, 0);
        if (__all_sync(0xffffffffu, w == w0)) {
            const int64_t t0 = __shfl_sync(0xffffffffu, t, 0);  // lane 0 is in range here
            sim_step_record *rec = record_of(p, t0, w0);
            const unsigned me = __ballot_sync(0xffffffffu, ate), md = __ballot_sync(0xffffffffu, died_e),
                           ma = __ballot_sync(0xffffffffu, died_a), m = __ballot_sync(0xffffffffu, survive),
                           mw = __ballot_sync(0xffffffffu, died_w);
            // eligible parents (R19) for the single-world claims in k_post; both list appends'
            // atomics are in flight together
            const unsigned mc = p.n_worlds == 1 ? __ballot_sync(0xffffffffu, cand) : 0u;
            int pos0 = 0, c0 = 0;
            if (lane == 0) {
                if (mc) c0 = atomicAdd(p.n_cand, __popc(mc));
                if (m) pos0 = atomicAdd(count_of(p, t0 + 1, w0), __popc(m));
                if (me) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->eaten), (unsigned long long)__popc(me));
                if (md) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deaths_energy), (unsigned long long)__popc(md));
                if (ma) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deaths_age), (unsigned long long)__popc(ma));
                if (mw) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deaths_wall), (unsigned long long)__popc(mw));
            }
            c0 = __shfl_sync(0xffffffffu, c0, 0);
            ECO_CHECK(!cand || c0 + __popc(mc & ((1u << lane) - 1u)) < p.S);
            if (cand) p.cand[c0 + __popc(mc & ((1u << lane) - 1u))] = make_int2(slot, cand_cell);
            // metrics: the deaths' ages, and at a window end the movement bins (warp sums)
#if ECO_METRICS & 1
            if (md | ma | mw) {
                const int dsum = __reduce_add_sync(0xffffffffu, dage);
                if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->death_age_sum), (unsigned long long)dsum);
            }
#endif

            pos0 = __shfl_sync(0xffffffffu, pos0, 0);
            if (survive) {
                const int q = pos0 + __popc(m & ((1u << lane) - 1u));
                ECO_CHECK(q < p.S && slot >= 0 && slot < p.S);
                list_of(p, t + 1, w)[q] = slot;
                list_cell_of(p, t + 1, w)[q] = cand_cell;  // survivors: cand_cell is the cell
            }
            if (p.n_ranks > 1) {  // sharded: this rank's own survivors, the next policy's work
                const bool mine = survive && p.owner[slot] == p.rank;
                const unsigned mo = __ballot_sync(0xffffffffu, mine);
                int o0 = 0;
                if (lane == 0 && mo) o0 = atomicAdd(p.own_count + ((t0 + 1) & 1), __popc(mo));
                o0 = __shfl_sync(0xffffffffu, o0, 0);
                if (mine) p.own_list[((t0 + 1) & 1) * p.S + o0 + __popc(mo & ((1u << lane) - 1u))] = slot;
            }
        } else {
            sim_step_record *rec = record_of(p, t, w);
            if (dage) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->death_age_sum), (unsigned long long)dage);
            if (ate) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->eaten), 1ull);
            if (died_e) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deaths_energy), 1ull);
            if (died_a) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deaths_age), 1ull);
            if (died_w) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deaths_wall), 1ull);
            if (survive) {
                const int q = atomicAdd(count_of(p, t + 1, w), 1);
                ECO_CHECK(q < p.S);
                list_of(p, t + 1, w)[q] = slot;
                list_cell_of(p, t + 1, w)[q] = cand_cell;
            }
        }
    }
}

// ----------------------------------------------------------------- a5 birth claim
// Lazy reset of this step's move claims (every claimant clears its own target; safe
// because the move phase has finished reading them).  Then every live parent with repr >=
// T_repr picks the first cell of a Philox-rotated (N, S, E, W) order that is
// in-grid, agent-free after moves/deaths (O'') and resource-free after consumption (R'')
// (R21), records its slot on its own cell, posts its claim key (BIRTH w1 << 32 | ~cell) on
// the candidate cell by atomicMax (the max is the winner) and marks the cell in the step's
// claimed-cell bitmap.  Distinct claimed cells are counted per world; deferred-claim losers
// are (candidates - claimed cells).  Must be called by all 32 lanes.
__device__ __forceinline__ void birth_claim_phase(const DevParams &p, size_t gtid, size_t gthreads,
                                                  const int *live_cum = nullptr) {
    const long total = live_cum ? (long)live_cum[p.n_worlds] : (long)p.n_worlds * p.S;
    const size_t HW = (size_t)p.H * p.W;
    const unsigned lane = gtid & 31;
    for (long base = (long)(gtid - lane); base < total; base += (long)gthreads) {
        const AgentIter it = live_cum ? agent_at_live(p, live_cum, base + lane) : agent_at(p, base + lane);
        const int w = it.w;
        const int64_t t = p.t[w];
        unsigned long long no_cell = 0, cand = 0;
        int new_cell = 0;
        if (it.in_range && it.i < *count_of(p, t, w)) {
            const int4 mr = p.mrec[(size_t)w * p.S + it.i];
            const int slot = mr.x;
            const size_t gs = (size_t)w * p.S + slot;
            const int tg = mr.z;
            if (tg >= 0) p.claim[(size_t)w * HW + tg] = 0ull;  // (-1 no move, -2 lethal wall)
            if (p.alive[gs]) {
                const int cellv = p.cell[gs];
                uint8_t dir = NO_DIR;
                if (p.repr[gs] >= p.repr_steps) {
                    const uint32_t *O = p.occ + (size_t)w * plane_words(p);
                    const uint32_t *Rn = plane_next(p, t) + (size_t)w * plane_words(p);
                    const int y = row_of(p, cellv), x = cellv - y * p.W;
                    // the four neighbours' O'' and R'' bits, loaded together (no dependent chain)
                    uint32_t freem = 0u;  // bit dd: neighbour dd is a candidate
#pragma unroll
                    for (int dd = 0; dd < 4; ++dd) {
                        const int cy = y + dir_dy(dd), cx = x + dir_dx(dd);
                        const bool in = cy >= 0 && cy < p.H && cx >= 0 && cx < p.W;
                        const int c = in ? cy * p.W + cx : cellv;
                        const uint32_t ob = get_bit(O, p, c), rb = get_bit(Rn, p, c);
                        if (in && !ob && !rb) freem |= 1u << dd;
                    }
                    const uint4 d = draw4(p.seeds[w], PURPOSE_BIRTH, (uint32_t)t, (uint32_t)cellv, 0u);
                    const int s0 = (int)(d.x & 3u);
                    // first candidate of the order s0, s0+1, s0+2, s0+3 (mod 4)
                    const uint32_t rot = ((freem >> s0) | (freem << (4 - s0))) & 0xFu;
                    if (rot) dir = (uint8_t)((s0 + __ffs(rot) - 1) & 3);
                    if (dir != NO_DIR) {
                        const int cy = y + dir_dy(dir), c = cy * p.W + x + dir_dx(dir);
                        uint32_t bit;
                        const uint32_t old = atomicOr(word_ptr(bbits_of(p, t, w), p, c, bit), bit);
                        if (!(old & bit)) new_cell = 1;
                        // the claim key (BIRTH w1, -parent cell): the cell's winner is the max
                        atomicMax(p.bkey + (size_t)w * HW + c,
                                  ((unsigned long long)d.y << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)cellv));
                        p.bslot[(size_t)w * HW + cellv] = slot;
                    }
                    if (dir == NO_DIR) no_cell = 1;
                    else cand = 1;
                }
            }
        }
        warp_world_add<unsigned long long>(no_cell, w, [&](int ww) {
            return reinterpret_cast<unsigned long long *>(&record_of(p, p.t[ww], ww)->deferred_no_cell);
        });
        // deferred_claim accumulates the candidates here; the rank phase subtracts the winners
        warp_world_add<unsigned long long>(cand, w, [&](int ww) {
            return reinterpret_cast<unsigned long long *>(&record_of(p, p.t[ww], ww)->deferred_claim);
        });
        warp_world_add<int>(new_cell, w, [&](int ww) { return p.n_win + ww; });
    }
}


// The candidate cell of the eligible parent on cellv (single world), or -1: the first of
// the Philox-rotated (N, S, E, W) neighbours that is in-grid, agent-free in O'' and
// resource-free in R'' (R21).  `key` gets its claim key (BIRTH w1 << 32 | ~cellv).
__device__ __forceinline__ int birth_target(const DevParams &p, int64_t t, int cellv, unsigned long long &key) {
    const uint32_t *O = p.occ;
    const uint32_t *Rn = plane_next(p, t);
    const int y = row_of(p, cellv), x = cellv - y * p.W;
    uint32_t freem = 0u;
#pragma unroll
    for (int dd = 0; dd < 4; ++dd) {
        const int cy = y + dir_dy(dd), cx = x + dir_dx(dd);
        const bool in = cy >= 0 && cy < p.H && cx >= 0 && cx < p.W;
        const int c = in ? cy * p.W + cx : cellv;
        const uint32_t ob = get_bit(O, p, c), rb = get_bit(Rn, p, c);
        if (in && !ob && !rb) freem |= 1u << dd;
    }
    const uint4 d = draw4(p.seeds[0], PURPOSE_BIRTH, (uint32_t)t, (uint32_t)cellv, 0u);
    key = ((unsigned long long)d.y << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)cellv);
    const int s0 = (int)(d.x & 3u);
    const uint32_t rot = ((freem >> s0) | (freem << (4 - s0))) & 0xFu;
    if (!rot) return -1;
    const int dir = (s0 + __ffs(rot) - 1) & 3;
    return (y + dir_dy(dir)) * p.W + x + dir_dx(dir);
}

// Single world: the claims of the eligible parents the move phase listed, by one block
// (NT threads): the same decision as birth_claim_phase (first Philox-rotated (N, S, E, W)
// neighbour that is in-grid, agent-free in O'' and resource-free in R''; slot on the own
// cell; atomicMax of the claim key on the candidate cell; the claimed-cell bitmap), so the
// rank can follow after a block barrier instead of a grid barrier.
#ifndef ECO_CLAIMS_B
#define ECO_CLAIMS_B 2  // measured: 1 -> 49.9, 2 -> 49.7, 4 -> 52.8 us per step (code size)
#endif
template <int NT>
__device__ void birth_claims_block(const DevParams &p, int64_t t) {
    constexpr int B = ECO_CLAIMS_B;  // candidates per thread in flight: their loads overlap
    const int nc = *reinterpret_cast<volatile int32_t *>(p.n_cand);
    int no_cell = 0, n_cand = 0, new_cells = 0;
    for (int r0 = 0; r0 < nc; r0 += NT * B) {
        int2 sc[B];
        int c[B];
        unsigned long long key[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int r = r0 + u * NT + (int)threadIdx.x;
            sc[u] = r < nc ? p.cand[r] : make_int2(-1, 0);
        }
#pragma unroll
        for (int u = 0; u < B; ++u) c[u] = sc[u].x >= 0 ? birth_target(p, t, sc[u].y, key[u]) : -2;
#pragma unroll
        for (int u = 0; u < B; ++u) {
            if (c[u] == -2) continue;
            if (c[u] < 0) {
                ++no_cell;
                continue;
            }
            uint32_t bit;
            const uint32_t old = atomicOr(word_ptr(bbits_of(p, t, 0), p, c[u], bit), bit);
            if (!(old & bit)) ++new_cells;
            atomicMax(p.bkey + c[u], key[u]);
            p.bslot[sc[u].y] = sc[u].x;
            ++n_cand;
        }
    }
    // warp sums first: one atomic per warp and counter, not one per thread
    no_cell = __reduce_add_sync(0xffffffffu, no_cell);
    n_cand = __reduce_add_sync(0xffffffffu, n_cand);
    new_cells = __reduce_add_sync(0xffffffffu, new_cells);
    if ((threadIdx.x & 31) == 0) {
        sim_step_record *rec = record_of(p, t, 0);
        if (no_cell) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deferred_no_cell), (unsigned long long)no_cell);
        // deferred_claim accumulates the candidates here; the rank subtracts the claimed cells
        if (n_cand) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deferred_claim), (unsigned long long)n_cand);
        if (new_cells) atomicAdd(p.n_win, new_cells);
    }
    __syncthreads();
}

// Single world with many eligible parents (a large world at its cap): the same claims as
// birth_claims_block, spread over every thread of the grid (a grid barrier follows).
__device__ __forceinline__ void birth_claims_grid(const DevParams &p, int64_t t, size_t gtid, size_t gthreads) {
    const int nc = *reinterpret_cast<volatile int32_t *>(p.n_cand);
    const unsigned lane = gtid & 31;
    for (size_t base = gtid - lane; base < (size_t)nc; base += gthreads) {
        const size_t r = base + lane;
        int no_cell = 0, cand = 0, new_cell = 0;
        if (r < (size_t)nc) {
            const int2 sc = p.cand[r];
            unsigned long long key;
            const int c = birth_target(p, t, sc.y, key);
            if (c < 0) {
                no_cell = 1;
            } else {
                uint32_t bit;
                const uint32_t old = atomicOr(word_ptr(bbits_of(p, t, 0), p, c, bit), bit);
                if (!(old & bit)) new_cell = 1;
                atomicMax(p.bkey + c, key);
                p.bslot[sc.y] = sc.x;
                cand = 1;
            }
        }
        const int a = __reduce_add_sync(0xffffffffu, no_cell), b = __reduce_add_sync(0xffffffffu, cand),
                  c = __reduce_add_sync(0xffffffffu, new_cell);
        if (lane == 0) {
            sim_step_record *rec = record_of(p, t, 0);
            if (a) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deferred_no_cell), (unsigned long long)a);
            if (b) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deferred_claim), (unsigned long long)b);
            if (c) atomicAdd(p.n_win, c);
        }
    }
}

// Single world, the blocks without the claims: the lazy reset of this step's move claims
// (each mover's target; the move phase has finished reading them).
__device__ __forceinline__ void move_claim_reset(const DevParams &p, int64_t t, size_t gtid, size_t gthreads) {
    const int n = *count_of(p, t, 0);
    for (size_t k = gtid; k < (size_t)n; k += gthreads) {
        const int tg = p.mrec[k].z;
        if (tg >= 0) p.claim[tg] = 0ull;
    }
}

// ------------------------------------------------------------------ a5 birth rank
// Each claimed cell c has exactly one winner: the live parent q adjacent to c that chose c
// with the largest key (BIRTH w1 << 32 | ~q).  n_place = min(claimed cells, free slots).
// (1) The first n_place free slots in ascending order (prefix scan of the alive bitmap) and
// (2) the first n_place claimed cells in row-major order (prefix scan of the claimed-cell
// bitmap) are found together, in chunks of NT alive words and NT*RANK_K bitmap words loaded
// at once (one memory round trip per chunk; the 200x400 world is one chunk).  (3) Rank r
// resolves the winner of cell c_r and places the child in free slot F[r] (R22); every later
// claimed cell is deferred for capacity.  Then the step's counters and the next alive count.
constexpr int RANK_SMEM_CAP = 1024;  // births ranked in shared memory (more spill to global)
constexpr int RANK_K = 8;            // claimed-cell bitmap words per thread per chunk

// Parent slot of claimed cell c: the claimant with the max key (BIRTH w1 << 32 | ~cell),
// posted by atomicMax during the claims (R21), then the slot recorded on its cell.
__device__ __forceinline__ int birth_parent_of(const DevParams &p, int w, int64_t t, int c) {
    (void)t;
    const size_t HW = (size_t)p.H * p.W;
    const unsigned long long k = *reinterpret_cast<const volatile unsigned long long *>(p.bkey + (size_t)w * HW + c);
    const int q = (int)(0xFFFFFFFFu - (uint32_t)k);
    return *reinterpret_cast<const volatile int32_t *>(p.bslot + (size_t)w * HW + q);
}

// child state of birth r in slot `child` on cell c; parent's repr reset; birth lists
__device__ __forceinline__ void place_child(const DevParams &p, int w, int64_t t, int c, int r, int n_surv, int child,
                                            int parent) {
    ECO_CHECK(child >= 0 && child < p.S && parent >= 0 && parent < p.S && n_surv + r < p.S);
    const size_t cs = (size_t)w * p.S + child;
    p.alive[cs] = 1;
    atomicOr(p.alive_bits + (size_t)w * p.SW + (child >> 5), 1u << (child & 31));
    p.cell[cs] = c;
    p.energy[cs] = p.e_init;
    p.age[cs] = 0;
    p.repr[cs] = 0;
    p.last_action[cs] = 0;
    p.ate[cs] = 0;
    p.gr_seen[cs] = 0;
    p.gr_ate[cs] = 0;
    p.gr_T[cs] = 0;
    p.gr_C[cs] = 0;
    p.low[cs] = 0;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);  // Hd in {4, 8, 16, 32}: rows are float4-aligned
    for (int k = 0; k < p.Hd; k += 4) {
        *reinterpret_cast<float4 *>(p.h + cs * p.Hd + k) = z4;
        *reinterpret_cast<float4 *>(p.c + cs * p.Hd + k) = z4;
    }
#pragma unroll
    for (int a = 0; a < LOGIT_STRIDE; a += 4) *reinterpret_cast<float4 *>(p.logits + cs * LOGIT_STRIDE + a) = z4;
    uint32_t bit;
    atomicOr(word_ptr(p.occ + (size_t)w * plane_words(p), p, c, bit), bit);
    p.repr[(size_t)w * p.S + parent] = 0;
    if (p.n_ranks > 1) {  // sharded: the child's weights stay on the parent's rank
        p.owner[child] = p.owner[parent];
        if (p.owner[parent] == p.rank) p.own_list[((t + 1) & 1) * p.S + atomicAdd(p.own_count + ((t + 1) & 1), 1)] = child;
    }
    list_of(p, t + 1, w)[n_surv + r] = child;
    list_cell_of(p, t + 1, w)[n_surv + r] = c;
}

// (1) + (2): free slots and claimed cells of ranks r < n_place into s_free / s_bcell (r <
// RANK_SMEM_CAP) or g_free / g_bcell (larger r).  All NT threads; `scratch` holds
// 2 * (NT/32 + 1) words.
// (Banded mode: only the claimed cells of bitmap words [bw_lo, bw_hi), the band's own rows.)
template <int NT>
__device__ void rank_lists(const DevParams &p, int w, int64_t t, int n_place, uint32_t *scratch, int *s_free,
                           int *s_bcell, int32_t *g_free, int32_t *g_bcell, size_t bw_lo = 0,
                           size_t bw_hi = ~(size_t)0) {
    const int tid = threadIdx.x;
    const uint32_t *ab = p.alive_bits + (size_t)w * p.SW;
    const uint32_t *bb = bbits_of(p, t, w);
    const size_t nbw = bw_hi < (size_t)p.H * p.WW ? bw_hi : (size_t)p.H * p.WW;
    uint32_t run_f = 0u, run_c = 0u;
    for (size_t j = 0;; ++j) {
        const bool need_f = run_f < (uint32_t)n_place, need_c = run_c < (uint32_t)n_place;  // block-uniform
        if (!need_f && !need_c) break;
        // all loads of the chunk first (independent), then one dual scan
        const size_t fi = j * NT + tid;
        uint32_t fr = 0u;
        if (need_f && fi < (size_t)p.SW) {
            const int nbits = p.S - (int)fi * 32;
            const uint32_t valid = nbits >= 32 ? 0xffffffffu : ((1u << nbits) - 1u);
            fr = ~ld_plain(ab + fi) & valid;
        }
        const size_t bi0 = bw_lo + (j * NT + tid) * RANK_K;
        uint32_t wd[RANK_K];
#pragma unroll
        for (int u = 0; u < RANK_K; ++u) wd[u] = (need_c && bi0 + u < nbw) ? ld_plain(bb + bi0 + u) : 0u;
        uint32_t cc = 0u;
#pragma unroll
        for (int u = 0; u < RANK_K; ++u) cc += (uint32_t)__popc(wd[u]);
        uint2 tot;
        const uint2 ex = block_exclusive_scan2<NT>(make_uint2((uint32_t)__popc(fr), cc), scratch, tot);
        uint32_t r = run_f + ex.x;
        while (fr && r < (uint32_t)n_place) {
            const int b = __ffs(fr) - 1;
            fr &= fr - 1u;
            const int slot = (int)fi * 32 + b;
            if (r < RANK_SMEM_CAP) s_free[r] = slot;
            else g_free[r] = slot;
            ++r;
        }
        uint32_t rc = run_c + ex.y;
        if (cc && rc < (uint32_t)n_place) {
            int y = (int)(bi0 / (size_t)p.WW), wx = (int)(bi0 - (size_t)y * p.WW);
#pragma unroll
            for (int u = 0; u < RANK_K; ++u) {
                uint32_t word = wd[u];
                while (word && rc < (uint32_t)n_place) {
                    const int b = __ffs(word) - 1;
                    word &= word - 1u;
                    const int c = y * p.W + wx * 32 + b;
                    if (rc < RANK_SMEM_CAP) s_bcell[rc] = c;
                    else g_bcell[rc] = c;
                    ++rc;
                }
                if (++wx == p.WW) {
                    wx = 0;
                    ++y;
                }
            }
        }
        run_f += tot.x;
        run_c += tot.y;
    }
    __syncthreads();
}

// step t's record, counters and the next alive count (one thread)
__device__ __forceinline__ void rank_finalize(const DevParams &p, int w, int64_t t, int n_start, int n_surv,
                                              int n_win, int n_place) {
    volatile sim_step_record *rec = record_of(p, t, w);
    const int64_t de = rec->deaths_energy, da = rec->deaths_age + rec->deaths_wall, grown = rec->grown,
                  eaten = rec->eaten, dc = rec->deferred_claim;
    const int64_t res = p.res_count[w] + grown - eaten;
    p.res_count[w] = res;
    rec->t = t;
    rec->agents_at_start = n_start;
    rec->births = n_place;
    rec->deferred_claim = dc - n_win;  // candidates - claimed cells
    rec->deferred_capacity = n_win - n_place;
    rec->population = n_surv + n_place;
    rec->resources = res;
    life_window_add(p, w, t, de + da, rec->death_age_sum);  // (da includes the wall deaths)
    *count_of(p, t + 1, w) = n_surv + n_place;
    p.n_births[w] = n_place;
    unsigned long long *tot = p.totals;
    if (w == 0) atomicAdd(tot + 0, 1ull);
    atomicAdd(tot + 1, (unsigned long long)n_start);
    atomicAdd(tot + 2, (unsigned long long)((size_t)p.H * p.W));
    atomicAdd(tot + 3, (unsigned long long)n_place);
    atomicAdd(tot + 4, (unsigned long long)(de + da));
    atomicAdd(tot + 5, (unsigned long long)eaten);
    atomicAdd(tot + 6, (unsigned long long)grown);
    if (p.rec_mirror) {  // the complete record, straight into the caller's mapped host buffer
        const volatile int64_t *src = reinterpret_cast<const volatile int64_t *>(rec);
        volatile int64_t *dst = reinterpret_cast<volatile int64_t *>(
            p.rec_mirror + (size_t)(t & (p.mirror_cap - 1)) * p.n_worlds + w);
        constexpr int NF = (int)(sizeof(sim_step_record) / sizeof(int64_t));
#pragma unroll
        for (int f = 0; f < NF; ++f) dst[f] = src[f];
    }
}

struct RankCounts {
    int n_start, n_surv, n_win, n_place;
};
__device__ __forceinline__ RankCounts rank_counts(const DevParams &p, int w, int64_t t) {
    RankCounts k;
    k.n_start = *reinterpret_cast<volatile int32_t *>(count_of(p, t, w));
    k.n_surv = *reinterpret_cast<volatile int32_t *>(count_of(p, t + 1, w));
    k.n_win = *reinterpret_cast<volatile int32_t *>(p.n_win + w);
    const int n_free = p.S - k.n_surv;
    k.n_place = k.n_win < n_free ? k.n_win : n_free;
    return k;
}

// Rank world w's births and resolve their winners: the birth lists (child slot, parent
// slot, cell) of ranks r < n_place go to global memory (all r) and shared memory (r <
// RANK_SMEM_CAP), n_births[w] = n_place.  All NT threads; ends with a block barrier.
template <int NT>
__device__ void rank_publish(const DevParams &p, int w, int64_t t, const RankCounts &k, uint32_t *scratch,
                             int *s_free, int *s_bcell, int *s_par) {
    int32_t *g_free = p.free_list + (size_t)w * p.S, *g_bcell = p.birth_cell + (size_t)w * p.S;
    if (k.n_place > 0) {
        rank_lists<NT>(p, w, t, k.n_place, scratch, s_free, s_bcell, g_free, g_bcell);
        for (int r = threadIdx.x; r < k.n_place; r += NT) {  // one birth per thread
            const int c = r < RANK_SMEM_CAP ? s_bcell[r] : *reinterpret_cast<volatile int32_t *>(g_bcell + r);
            const int child = r < RANK_SMEM_CAP ? s_free[r] : *reinterpret_cast<volatile int32_t *>(g_free + r);
            const int par = birth_parent_of(p, w, t, c);
            if (r < RANK_SMEM_CAP) s_par[r] = par;
            p.birth_child[(size_t)w * p.S + r] = child;
            p.birth_parent[(size_t)w * p.S + r] = par;
            g_bcell[r] = c;
        }
    }
    if (threadIdx.x == 0) p.n_births[w] = k.n_place;
    __syncthreads();
}

// Place the published births (children's state, occupancy, lists), then the step's
// counters and t += 1.  All NT threads of the block that ran rank_publish.
template <int NT>
__device__ void rank_place(const DevParams &p, int w, int64_t t, const RankCounts &k, const int *s_free,
                           const int *s_bcell, const int *s_par) {
    const size_t ws = (size_t)w * p.S;
    for (int r = threadIdx.x; r < k.n_place; r += NT) {
        const bool sm = r < RANK_SMEM_CAP;
        const int c = sm ? s_bcell[r] : p.birth_cell[ws + r];
        const int child = sm ? s_free[r] : p.birth_child[ws + r];
        const int par = sm ? s_par[r] : p.birth_parent[ws + r];
        place_child(p, w, t, c, r, k.n_surv, child, par);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        rank_finalize(p, w, t, k.n_start, k.n_surv, k.n_win, k.n_place);
        p.t[w] = t + 1;
    }
    __syncthreads();
}

// One block ranks and places world w's births, then t += 1.
template <int NT>
__device__ void birth_rank_world(const DevParams &p, int w, uint32_t *scratch, int *s_free, int *s_bcell,
                                 int *s_par) {
    const int64_t t = p.t[w];
    const RankCounts k = rank_counts(p, w, t);
    rank_publish<NT>(p, w, t, k, scratch, s_free, s_bcell, s_par);
    rank_place<NT>(p, w, t, k, s_free, s_bcell, s_par);
}

// ------------------------------------------------------------------- a5 mutation
// "an agent's weights are mutated by adding noise sampled from N(0, sigma)",
// sigma = 0.02 a standard deviation (R23).  The noise of canonical weight j comes from the
// Philox block (MUTATE, birth step, child cell, q = j >> 2): words (w0,w1) give z[4q],
// z[4q+1], (w2,w3) give z[4q+2], z[4q+3] via fp64 Box-Muller.  One item = one Box-Muller
// PAIR (canonical j even, j+1) of one child: one log, one sqrt and one sincos for two
// weights.  In the device layout the partner of j sits HD4 floats later (W_ih^T, W_hh^T:
// next column), 4 floats later (b: next unit of the same gate) or 1 float later (W_out,
// b_out), so consecutive items still touch consecutive addresses.  Runs after the rank
// phase advanced t, so the birth step is p.t[w] - 1.

// pair items per child: (I + Hd)/2 column pairs x HD4 rows, 2Hd bias pairs, ceil((5Hd+5)/2)
// (network 1: its device row is the canonical row, so pair it = weights 2it, 2it + 1)
template <typename PP>
__device__ __forceinline__ int mutate_items_per_child(const PP &p) {
    if (p.net == 1) return (p.P + 1) >> 1;
    return ((p.I + p.Hd) >> 1) * (p.Hd * 4) + 2 * p.Hd + (5 * p.Hd + 6) / 2;
}

// pair item -> device index d0 of its first weight, device stride of the partner (0 when
// the pair is a singleton: the last b_out entry), canonical index j0 (even)
template <typename PP>
__device__ __forceinline__ void mutate_item(const PP &p, int it, int &d0, int &dstep, int &j0) {
    if (p.net == 1) {
        d0 = j0 = 2 * it;
        dstep = 2 * it + 1 < p.P ? 1 : 0;
        return;
    }
    const int Hd = p.Hd, G = 4 * Hd, HD4 = Hd * 4;
    const int nA = ((p.I + Hd) >> 1) * HD4;
    if (it < nA) {
        const int s4 = p.hd_shift + 2;  // HD4 = 1 << s4
        const int pc = it >> s4, rem = it & (HD4 - 1), col = 2 * pc;
        const int row = ((rem & 3) << p.hd_shift) + (rem >> 2);
        d0 = (col << s4) + rem;  // W_hh^T follows W_ih^T contiguously (off_hh = I * HD4)
        dstep = HD4;
        j0 = col < p.I ? row * p.I + col : G * p.I + row * Hd + (col - p.I);
        return;
    }
    it -= nA;
    if (it < 2 * Hd) {  // b: it = kp*4 + gate, units 2kp and 2kp+1
        const int kp = it >> 2, gate = it & 3;
        d0 = p.off_b + (2 * kp) * 4 + gate;
        dstep = 4;
        j0 = G * p.I + G * Hd + gate * Hd + 2 * kp;
        return;
    }
    it -= 2 * Hd;  // W_out[5][Hd] then b_out[5], identical order in both layouts
    const int e = 2 * it, n_tail = 5 * Hd + 5;
    d0 = p.off_out + e;
    dstep = e + 1 < n_tail ? 1 : 0;
    j0 = G * p.I + G * Hd + G + e;
}

// (z[j0], z[j0+1]) for (step t, child cell): bit-identical to box_muller()'s (za, zb).
// Not inlined: one copy of the Philox + log + sincos code serves every call site (the
// one-shot phases of k_post are bound by instruction fetch, not by call overhead).
static __device__ __noinline__ double2 gauss_pair_nl(uint64_t seed, int64_t t, int cellc, int j0);
__device__ __forceinline__ void gauss_pair(uint64_t seed, int64_t t, int cellc, int j0, double &za, double &zb) {
    const double2 z = gauss_pair_nl(seed, t, cellc, j0);
    za = z.x;
    zb = z.y;
}
__device__ __forceinline__ double2 gauss_pair_body(uint64_t seed, int64_t t, int cellc, int j0) {
    double za, zb;
    const uint4 d = draw4(seed, PURPOSE_MUTATE, (uint32_t)t, (uint32_t)cellc, (uint32_t)(j0 >> 2));
    const bool lo = (j0 & 3) == 0;
    const uint32_t wa = lo ? d.x : d.z, wb = lo ? d.y : d.w;
    const double two_m32 = 2.3283064365386963e-10;
    const double u1 = __dmul_rn(__dadd_rn((double)wa, 1.0), two_m32);
    const double u2 = __dmul_rn((double)wb, two_m32);
    const double rad = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
    const double th = __dmul_rn(6.283185307179586, u2);
    double sn, cs;
    sincos(th, &sn, &cs);
    za = __dmul_rn(rad, cs);
    zb = __dmul_rn(rad, sn);
    return make_double2(za, zb);
}
static __device__ __noinline__ double2 gauss_pair_nl(uint64_t seed, int64_t t, int cellc, int j0) {
    return gauss_pair_body(seed, t, cellc, j0);
}

// U independent items per thread: all loads, then all Philox/log/sincos chains, then all
// stores (stores last, so no child store can alias an input the compiler must re-order).
// Item u is pair `iu[u]` of birth `bu[u]` (skipped unless ok[u]); birth(b, child, parent,
// cell) gives birth b's slots and cell.
template <int U, bool INL = false, typename PP, typename Birth>  // INL: the Gaussian pairs inlined (U chains interleave)
__device__ __forceinline__ void mutate_batch(const PP &p, int w, int64_t t, uint64_t seed, const uint32_t *bu,
                                             const uint32_t *iu, const bool *ok, Birth birth, bool dry = false) {
    float pa[U], pb[U];
    int cellc[U], d0[U], dstep[U], j0[U];
    float *dst[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        dst[u] = nullptr;
        if (!ok[u]) continue;
        mutate_item(p, (int)iu[u], d0[u], dstep[u], j0[u]);
        int child, parent;
        birth((int)bu[u], child, parent, cellc[u]);
        ECO_CHECK(child >= 0 && child < p.S && parent >= 0 && parent < p.S);
        // sharded: mutated on the child's owner = the parent's (placement sets owner[child]
        // concurrently with this phase, so read the parent's, which is stable)
        if (p.n_ranks > 1 && p.owner[parent] != p.rank) continue;
        const float *wp = p.weights + ((size_t)w * p.S + parent) * p.Pd + d0[u];
        pa[u] = wp[0];
        pb[u] = dstep[u] ? wp[dstep[u]] : 0.f;
        dst[u] = p.weights + ((size_t)w * p.S + child) * p.Pd + d0[u];
    }
    double za[U], zb[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (dst[u]) {
            if (INL) {
                const double2 z = gauss_pair_body(seed, t, cellc[u], j0[u]);
                za[u] = z.x;
                zb[u] = z.y;
            } else {
                gauss_pair(seed, t, cellc[u], j0[u], za[u], zb[u]);
            }
        }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (!dst[u] || dry) continue;
        dst[u][0] = __fadd_rn(pa[u], __double2float_rn(__dmul_rn(p.mutation_std, za[u])));
        if (dstep[u]) dst[u][dstep[u]] = __fadd_rn(pb[u], __double2float_rn(__dmul_rn(p.mutation_std, zb[u])));
    }
}

#ifndef ECO_MUTATE_U
#define ECO_MUTATE_U 1  // measured: 1 -> 48.9, 2 -> 49.5, 4 -> 51.0 us per step (instruction fetch)
#endif
// the nb children of world w born at step t, from the global birth lists.  Items k = gtid,
// gtid + gthreads, ... of nb * Q pairs; (birth, pair) = divmod(k, Q) is advanced
// incrementally (one division per thread).
// U: independent items in flight per thread; INL: inlined Gaussian pairs and 32-bit index
// divisions where the operands fit (the several-world path; the one-world path keeps its
// compact code: it is bound by instruction fetch)
template <int U = ECO_MUTATE_U, bool INL = false, typename PP>
__device__ __forceinline__ size_t mutate_world_impl(const PP &p, int w, int64_t t, uint64_t seed, int nb, size_t gtid,
                                                    size_t gthreads, bool dry) {
    const uint32_t Q = (uint32_t)mutate_items_per_child(p);
    const size_t n = (size_t)nb * Q;
    if (gtid >= n) return gtid;
    const size_t ws = (size_t)w * p.S;
    auto birth = [&](int b, int &child, int &parent, int &cell) {
        child = p.birth_child[ws + b];
        parent = p.birth_parent[ws + b];
        cell = p.birth_cell[ws + b];
    };
    // (INL) 32-bit divisions where the operands allow: a 64-bit one is ~100 instructions
    uint32_t sb, si, b, it;
    if (INL && gthreads <= 0xFFFFFFFFull) {
        sb = (uint32_t)gthreads / Q;
        si = (uint32_t)gthreads - sb * Q;
    } else {
        sb = (uint32_t)(gthreads / Q);
        si = (uint32_t)(gthreads % Q);
    }
    if (INL && gtid <= 0xFFFFFFFFull) {
        b = (uint32_t)gtid / Q;
        it = (uint32_t)gtid - b * Q;
    } else {
        b = (uint32_t)(gtid / Q);
        it = (uint32_t)(gtid % Q);
    }
    auto adv = [&](uint32_t &b_, uint32_t &i_) {
        i_ += si;
        b_ += sb;
        if (i_ >= Q) {
            i_ -= Q;
            ++b_;
        }
    };
    size_t k = gtid;
    for (; k < n; k += U * gthreads) {
        uint32_t bu[U], iu[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            bu[u] = b;
            iu[u] = it;
            ok[u] = k + u * gthreads < n;
            adv(b, it);
        }
        mutate_batch<U, INL>(p, w, t, seed, bu, iu, ok, birth, dry);
    }
    // the first index >= n of this thread's stride (gtid + m * gthreads): the last batch may
    // have ended on skipped items
#pragma unroll
    for (int u = 1; u < U; ++u)
        if (k > gtid && k - gthreads >= n) k -= gthreads;
    return k;
}
__device__ __forceinline__ void mutate_world(const DevParams &p, int w, int64_t t, int nb, size_t gtid,
                                             size_t gthreads) {
    mutate_world_impl(p, w, t, p.seeds[w], nb, gtid, gthreads, false);
}

// The single-world mutation as ONE out-of-line copy (the fields it needs by value, so the
// caller's parameters stay in registers): k_post's dynamics warps first run it `dry` (no
// stores) on one item while they wait for block 0's births, which loads its instruction
// lines into this SM's caches before the real call (the one-shot phases are bound by
// instruction fetch).
struct MutArgs {
    float *weights;
    const int32_t *birth_child, *birth_parent, *birth_cell;
    const uint8_t *owner;
    double mutation_std;
    int S, Pd, I, Hd, hd_shift, off_b, off_out, n_ranks, rank;
    int net, P;
};
__device__ __forceinline__ MutArgs mut_args(const DevParams &p) {
    MutArgs a;
    a.weights = p.weights;
    a.birth_child = p.birth_child;
    a.birth_parent = p.birth_parent;
    a.birth_cell = p.birth_cell;
    a.owner = p.owner;
    a.mutation_std = p.mutation_std;
    a.S = p.S;
    a.Pd = p.Pd;
    a.net = p.net;
    a.P = p.P;
    a.I = p.I;
    a.Hd = p.Hd;
    a.hd_shift = p.hd_shift;
    a.off_b = p.off_b;
    a.off_out = p.off_out;
    a.n_ranks = p.n_ranks;
    a.rank = p.rank;
    return a;
}
static __device__ __noinline__ void mutate_world_nl(MutArgs a, int64_t t, uint64_t seed, int nb, size_t gtid, size_t gthreads,
                                             int dry) {
    mutate_world_impl(a, 0, t, seed, nb, gtid, gthreads, dry != 0);
}

// all worlds, after the rank advanced t.  Several worlds: their pair items form ONE
// world-major sequence strided over the grid's threads (thread gtid takes items gtid, gtid +
// gthreads, ... of the concatenation), so every thread has work whatever a single world's
// births are; the worlds' birth counts are read 32 at a time, one per lane.  (One pass per
// world — a world's ~10 children are 43,000 items for 113,664 threads, 64 dependent passes —
// took 157 of the 64-world ensemble's 664 us per step.)  Whole warps call this together.
#ifndef ECO_MUTATE_INL_MULTI
#define ECO_MUTATE_INL_MULTI 1  // the Gaussian pair inlined in the several-world path (throughput, not fetch, bound)
#endif
#ifndef ECO_MUTATE_U_MULTI
#define ECO_MUTATE_U_MULTI 1  // measured (64-world ensemble, mutation phase): 1 -> 80.3, 2 -> 82.9, 3 -> 85.3, 4 -> 104 us
#endif
// Several worlds, their children prefixed over the worlds in the block's shared array s_cum
// [n_worlds + 1] (made here by warp 0; every thread of the block calls this): thread gtid
// takes pair items gtid, gtid + gthreads, ... of the world-major sequence of all children, U
// of them at a time — independent chains (loads, Philox, log, sincos, stores) of different
// children, usually of different worlds, interleaved by the compiler.
template <int U>
__device__ __forceinline__ void mutate_multi(const DevParams &p, size_t gtid, size_t gthreads, int *s_cum) {
    const int lane = (int)(threadIdx.x & 31u);
    if (threadIdx.x < 32) {
        int run = 0;
        for (int w0 = 0; w0 < p.n_worlds; w0 += 32) {
            const int wl = w0 + lane;
            const int nb = wl < p.n_worlds ? *reinterpret_cast<volatile int32_t *>(p.n_births + wl) : 0;
            int inc = nb;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int up = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += up;
            }
            if (wl < p.n_worlds) s_cum[wl] = run + inc - nb;
            run += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) s_cum[p.n_worlds] = run;
    }
    __syncthreads();
    const uint32_t Q = (uint32_t)mutate_items_per_child(p);
    const uint32_t C = (uint32_t)s_cum[p.n_worlds];
    const size_t n = (size_t)C * Q;
    if (gtid >= n) return;
    // (child, pair) of this thread's next item; gtid < n <= 2^31 * Q, gthreads < 2^32
    uint32_t c = (uint32_t)(gtid / Q), it = (uint32_t)(gtid - (size_t)c * Q);
    const uint32_t sb = (uint32_t)gthreads / Q, si = (uint32_t)gthreads - sb * Q;
    int w = 0;  // the world of child c (children are world-major: w only grows)
    for (size_t k = gtid; k < n; k += U * gthreads) {
        float pa[U], pb[U];
        int cellc[U], dstep[U], j0[U];
        int64_t tb[U];
        uint64_t seed[U];
        float *dst[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            dst[u] = nullptr;
            if (k + u * gthreads < n) {
                while (c >= (uint32_t)s_cum[w + 1]) ++w;
                const size_t bi = (size_t)w * p.S + (c - (uint32_t)s_cum[w]);
                const int child = p.birth_child[bi], parent = p.birth_parent[bi];
                cellc[u] = p.birth_cell[bi];
                tb[u] = p.t[w] - 1;
                seed[u] = p.seeds[w];
                ECO_CHECK(child >= 0 && child < p.S && parent >= 0 && parent < p.S);
                int d0;
                mutate_item(p, (int)it, d0, dstep[u], j0[u]);
                const float *wp = p.weights + ((size_t)w * p.S + parent) * p.Pd + d0;
                pa[u] = wp[0];
                pb[u] = dstep[u] ? wp[dstep[u]] : 0.f;
                dst[u] = p.weights + ((size_t)w * p.S + child) * p.Pd + d0;
            }
            it += si;
            c += sb;
            if (it >= Q) {
                it -= Q;
                ++c;
            }
        }
        double2 z[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (dst[u]) z[u] = gauss_pair_body(seed[u], tb[u], cellc[u], j0[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!dst[u]) continue;
            dst[u][0] = __fadd_rn(pa[u], __double2float_rn(__dmul_rn(p.mutation_std, z[u].x)));
            if (dstep[u]) dst[u][dstep[u]] = __fadd_rn(pb[u], __double2float_rn(__dmul_rn(p.mutation_std, z[u].y)));
        }
    }
}

// `s_cum`: a shared array of the block with room for n_worlds + 1 ints (s_cum_cap entries),
// or nullptr; with it (and every thread of the block calling) several worlds take the
// interleaved path above.
__device__ __forceinline__ void mutate_phase(const DevParams &p, size_t gtid, size_t gthreads, int *s_cum = nullptr,
                                             int s_cum_cap = 0) {
    if (p.n_worlds == 1) {
        const int nb = *reinterpret_cast<volatile int32_t *>(p.n_births);
        if (nb > 0) mutate_world(p, 0, p.t[0] - 1, nb, gtid, gthreads);
        return;
    }
    if (s_cum && p.n_worlds < s_cum_cap && ECO_MUTATE_U_MULTI > 0) {
        mutate_multi<(ECO_MUTATE_U_MULTI > 0 ? ECO_MUTATE_U_MULTI : 1)>(p, gtid, gthreads, s_cum);
        return;
    }
    const uint32_t Q = (uint32_t)mutate_items_per_child(p);
    const int lane = (int)(threadIdx.x & 31u);
    size_t g = gtid, base = 0;  // this thread's next item and the current world's first, in the concatenation
    for (int w0 = 0; w0 < p.n_worlds; w0 += 32) {
        const int wl = w0 + lane;
        const int nbl = wl < p.n_worlds ? *reinterpret_cast<volatile int32_t *>(p.n_births + wl) : 0;
        const int wn = p.n_worlds - w0 < 32 ? p.n_worlds - w0 : 32;
        for (int j = 0; j < wn; ++j) {
            const int nb = __shfl_sync(0xffffffffu, nbl, j);
            const size_t n = (size_t)nb * Q;
            if (g < base + n) {
                const int w = w0 + j;
                const size_t r0 = g - base;
                g = base + mutate_world_impl<1, ECO_MUTATE_INL_MULTI != 0>(p, w, p.t[w] - 1, p.seeds[w], nb,
                                                                                            r0, gthreads, false);
            }
            base += n;
        }
    }
}

}  // namespace eco
