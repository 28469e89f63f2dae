// sim_internal.cuh — device-side layout and helpers of libsim.so (sm_100a).
//
// Device layout:
//  * resource plane R and occupancy plane O: one bit per cell, rows padded to WW 32-bit
//    words (WW = ceil(W/32) rounded up to a multiple of 4 words = 16 B); bit b of word
//    (y, wx) is column 32*wx + b; padding bits are always 0.  R is double-buffered by
//    step parity: plane[t&1] = R_t, plane[(t+1)&1] = R' (post-regrowth) which becomes
//    R_{t+1} after consumption.
//  * agents: structure of arrays [world][slot]; weights [world][slot][Pd] in the
//    GEMV-friendly order W_ih^T[I][Hd][4], W_hh^T[Hd][Hd][4], b[Hd][4], W_out[5][Hd],
//    b_out[5], padded to Pd (multiple of 32 floats = 128 B).  Lane k of an agent's lane
//    group reads its unit's four gate weights (i,f,g,o) with one 16-B load.
//  * alive slots: a u8 flag per slot plus a bitmap [world][SW]; the live agents of step t
//    are listed (any order: no result depends on it) in alive_list[t&1].
//  * reproduction: per claimed cell the max birth-claim key bkey (BIRTH w1 << 32 | ~parent
//    cell, 0 = none), per parent cell its slot bslot, and a claimed-cell bitmap bbits[t&1]
//    over cells (plane layout).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/sim.h"

// sim_step(n >= 2) launches two-step graphs in which the second policy is a programmatic
// dependent of the first k_post (griddepcontrol.wait in the policy).  Defined once here so
// the host launch (api.cu) and the device wait (step.cu) always agree.
// Diagnostic build (-DECO_CHECKS=1, libsim_checked.so): device asserts on every cell, slot,
// list position and outbox index the kernels compute (compute-sanitizer is not available
// on the GPU pool; tests/test_gpu_checks.py runs the checked build).
#ifndef ECO_CHECKS
#define ECO_CHECKS 0
#endif
#if ECO_CHECKS
#include <cassert>
#define ECO_CHECK(cond) assert(cond)
#else
#define ECO_CHECK(cond) ((void)0)
#endif

#ifndef ECO_GRAPH_STEPS
#define ECO_GRAPH_STEPS 8  // (measured, sim_step(10000) at paper scale: 2 -> 41.16, 4 -> 40.25, 8 -> 39.79, 16 -> 39.60 us per step) steps per graph of sim_step(n >= this): every policy after the first a programmatic dependent
#endif
#ifndef ECO_GRAPH_ALL
#define ECO_GRAPH_ALL 1  // multi-step graphs for every unsharded handle (0: the split policy's only)
#endif
#ifndef ECO_STEP2_PDL
#define ECO_STEP2_PDL 1
#endif

// The step kernels' preferred shared-memory carveout (percent of the unified L1/shared
// array; -1 = the driver's choice).  One value for every kernel of a step, so consecutive
// kernels never make an SM drain and reconfigure between them.
#ifndef ECO_CARVEOUT
#define ECO_CARVEOUT -1
#endif

namespace eco {

// dynamic shared memory limit and the common carveout (ECO_CARVEOUT) of a kernel
template <class K>
inline cudaError_t set_dyn_smem(K k, int bytes) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess || ECO_CARVEOUT < 0) return e;
    return cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, ECO_CARVEOUT);
}

constexpr uint32_t PURPOSE_INIT_RES = 1, PURPOSE_INIT_PLACE = 2, PURPOSE_INIT_W = 3, PURPOSE_REGROW = 4,
                   PURPOSE_MOVE = 5, PURPOSE_BIRTH = 6, PURPOSE_MUTATE = 7,
                   PURPOSE_ACTION = 8,   // the sampled action of network 1 (R38)
                   PURPOSE_CONSUME = 9;  // co-location: the lottery on a resource cell (R45)
constexpr int LOGIT_STRIDE = 8;
constexpr uint8_t NO_DIR = 0xFF;

// Everything a kernel needs, passed by value (fixed for the handle's lifetime, so one
// captured CUDA graph serves every step; the step index lives in device memory).
struct DevParams {
    int H, W, WW, S, SW, Hd, I, P, Pd, n_worlds, r, log_cap;
    int net;             // 0: LSTM + linear head, argmax; 1: the paper's CNN-LSTM, sampled (NEXT-2)
    int coloc;           // 1: co-location (NEXT-1, R43-R47): ncount / elig_bits below, no claims
    int row_lo, row_hi;  // rows this handle owns: [0, H) unless it is one latitude band (banded mode)
    int regrow_split;    // 1: k_post leaves the regrowth of step t+1 to k_regrow_tiled, launched after
                         // it (agent-free worlds of many words: the configs[2] benchmark grids)
    int hd_shift;  // Hd = 1 << hd_shift
    double invW;   // 1 / W (cell -> row without an integer division)
    int repr_steps, max_age;
    int e_init, e_decay, e_gain, e_repr_gt, e_death_le, e_max;
    int death_steps;   // > 0: the death timer T_death, else immediate death
    int lethal_walls;  // 1: a move off the grid kills; the policy marks target -2
    int cls_k1, cls_k2, cls_k3;  // class thresholds f_class_min_k[1..3]
    int row_dx[5];  // regrowth disc: offsets (dy, dx) with |dx| <= row_dx[dy + 2], centre excluded
    int disc12;     // 1: the disc is BASELINE's radius-2 disc (row_dx = 0,1,2,1,0: 12 cells)
    int t_monotone; // 1: T[y][c] is non-decreasing in the class c on every row
    int off_hh, off_b, off_out, off_bout;  // offsets inside one agent's device weights
    double mutation_std, init_weight_std;
    uint32_t init_res_thr;
    const uint64_t *seeds;    // [n_worlds]
    int64_t *t;               // [n_worlds] step index (all equal)
    uint32_t *plane0, *plane1;// R double buffer [n_worlds][H][WW]
    uint32_t *occ;            // O [n_worlds][H][WW]
    uint32_t *bbits;          // birth bitmaps [2][n_worlds][H][WW] (by step parity)
    const uint32_t *T;        // [H][4] Bernoulli thresholds
    unsigned long long *claim;   // [n_worlds][H*W] move claims (0 = none)
    unsigned long long *bkey;    // [n_worlds][H*W] max birth-claim key on a claimed cell (0 = none)
    int32_t *bslot;              // [n_worlds][H*W] slot of the parent standing on the cell
    uint8_t *alive, *last_action, *ate;
    uint32_t *alive_bits;        // [n_worlds][SW]
    int32_t *cell, *energy, *age, *repr;
    int32_t *low;                // [n_worlds][S] consecutive steps with energy <= e_death_le
    float *h, *c, *logits, *weights;
    int4 *mrec;                  // [n_worlds][S] per list position: (slot, cell, target or -1, MOVE w0)
    int32_t *alive_list;         // [2][n_worlds][S]
    int32_t *list_cell;          // [2][n_worlds][S] the cell of each listed agent (= cell[slot])
    int32_t *n_alive;            // [2][n_worlds]
    int32_t *n_win;              // [n_worlds] birth-claim winners this step
    int32_t *free_list;          // [n_worlds][S] scratch (first n_place entries used)
    // Agent-sharded mode (one world over n_ranks GPUs, sim_shard): every rank holds the whole
    // world and runs the integer dynamics identically; the policy of a slot runs only on its
    // owner (owner[slot] == rank), whose memory alone holds that agent's weights, h and c.
    int32_t n_ranks, rank;
    uint8_t *owner;              // [S] owning rank of each slot (children inherit the parent's)
    unsigned long long *pol_ctr; // [2] sharded: this rank's policy counters (active inputs, near ties)
    int4 *mrec_slot;             // [S] sharded: move records by SLOT (the list order differs by rank)
    int32_t *own_list;           // [2][S] sharded: this rank's live slots of step t (by parity)
    int32_t *own_count;          // [2]
    int32_t *own_surv;           // sharded + split: own list positions below hold survivors (P rows)
    // Split policy (one unsharded world, Hd = 32, graph mode): P[slot] = W_hh h + b for the
    // NEXT step is computed by k_post for the survivors (off the policy's critical path,
    // beside the latency-bound phases); the policy then streams only P and the active W_ih
    // columns.  Children (the last *p_children list positions) start from their bias.
    int32_t split;
    // Hd = 32, one world whose slots need more than one wave of policy blocks (a large world, a
    // band): contexts block-major (full blocks, then empty ones) instead of interleaved
    int32_t pol_bmajor;
    // Hd = 32, several worlds (unsplit policy): the policy's blocks loop over the 16-agent
    // tiles of the worlds' LIVE list positions only (a per-block prefix over the worlds' counts)
    // instead of one block per 16 slots (the 64-world ensemble: 28,000 of 32,768 blocks empty)
    int32_t pol_compact;
    float *Pbuf;                 // [S][Hd*4] device order [k][4], like b
    // movement-histogram metrics (sim.h: sim_get_move_hist): each slot's cell and age at the
    // start of the current 50-step window, and the per-window histograms (a ring)
    int32_t *mv_cell, *mv_inv;   // [n_worlds][S]: cell and age - 50 k at the start of window k
    int32_t *mv_hist;            // [n_worlds][mv_cap][17]
    int mv_cap;                  // windows kept (a power of two)
    // greediness (§3.3 lab set-up, "non-overlapping fixed windows of 20 timesteps"):
    // per slot, flags of the current window (a resource was in the field of view / the agent
    // ate) and the counts T_r, C_r of the closed windows; G = C_r / T_r
    uint8_t *gr_seen, *gr_ate;   // [n_worlds][S]
    int32_t *gr_T, *gr_C;        // [n_worlds][S]
    // life expectancy (Appendix C, 500-step windows): per window, deaths and the
    // summed ages at death ([n_worlds][le_cap][2], a ring of windows aligned to 500 t)
    unsigned long long *le;
    int le_cap;
    int32_t *p_children;         // list positions at the end of step t's list without a P row
    int2 *cand;                  // [n_worlds][S] single world: this step's eligible parents (slot, cell)
    int32_t *n_cand;             // [n_worlds] their count
    int32_t *birth_child, *birth_parent, *birth_cell, *n_births;  // by birth rank
    int64_t *res_count;          // [n_worlds] resources at step start
    sim_step_record *log;        // [log_cap][n_worlds]
    sim_step_record *rec_mirror; // optional mapped host ring [mirror_cap][n_worlds] (sim_set_record_mirror)
    int32_t mirror_cap;          // a power of two
    unsigned long long *totals;  // [7] sim_totals order
    unsigned long long *phase_ns;  // [SIM_NUM_POST_PHASES] k_post phase clock (block 0)
    const uint8_t *forced;       // [n_worlds][S]
    uint8_t *own_act;            // [n_worlds][S] test hook: the policy's own action while forcing is on
    int32_t *ncount;             // co-location: [n_worlds][H*W] agents per cell
    uint32_t *elig_bits;         // co-location: [n_worlds][SW] eligible parents of the step (by slot)
    const int32_t *forced_on;    // device flag
    int32_t *nonfinite;          // host-mapped flag
};

// Banded mode (band.cu): the buffers of another band that a band's
// pull kernels read (a band of this process, or peer memory mapped from another GPU).
struct BandPeer {
    const uint32_t *plane0, *plane1, *occ, *bbits;
    const unsigned long long *claim, *bkey;
    const int32_t *mig, *nb;   // migrant and newborn outboxes ([2 directions][count + records])
};
constexpr int BAND_MAX = 32;
struct BandParams {
    int b, G, y0, y1;          // band b of G owns rows [y0, y1)
    int S_global;              // the world's population cap (R22 is global)
    int N0;                    // the world's initial agents (C.2 is global)
    int cap;                   // records per outbox direction: min(W, local slots)
    int32_t *mig_out, *nb_out; // this band's outboxes (pulled by the neighbours)
    int64_t *counts;           // [2 parities][4]: claimed cells in the own rows, survivors
    int32_t *plist, *n_plist;  // agents of this step after the move (stayers, then arrivals)
    int32_t *arr_slot;         // [2 cap] the arrivals' local slots
    int32_t *cslot;            // [H*W] local slot of a child whose parent is in a neighbour band
    int4 *hcand;               // [2 cap] own parents claiming a cell in a neighbour's row:
                               // (parent slot, parent cell, claimed cell, claim key hi)
    int32_t *n_hcand;
    int64_t *snap;             // [4] (step t + 1, survivors) after P5 (the global cap's input); split policy: [2..3] =
                               // (step t, its list's count) after the policy, for the P rows on the second stream
    int32_t *flags;            // [0] bit 0: local slot pool exhausted; [1] arrivals placed
    BandPeer up, down;         // bands b-1 and b+1 (plane0 == nullptr: none)
    const int64_t *all_counts[BAND_MAX];  // every band's counts
};

// ------------------------------------------------------------------ Philox4x32-10
// Salmon et al. SC'11.  Counter (c0 = sub, c1 = entity, c2 = step, c3 = purpose),
// key (seed lo, seed hi) — the RNG contract of DESIGN.md §3 (C.1).
// Rounds fully unrolled (measured after k_post's one-shot paths were made compact: 58.8 vs
// 59.4 us per paper-scale step rolled, and 10 % faster regrowth while the grid fills).
#ifndef ECO_PHILOX_UNROLL
#define ECO_PHILOX_UNROLL 10
#endif
constexpr int kPhiloxUnroll = ECO_PHILOX_UNROLL;
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll kPhiloxUnroll
    for (int round = 0; round < 10; ++round) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

__device__ __forceinline__ uint4 draw4(uint64_t seed, uint32_t purpose, uint32_t step, uint32_t entity,
                                       uint32_t sub) {
    return philox4x32_10(make_uint4(sub, entity, step, purpose), (uint32_t)seed, (uint32_t)(seed >> 32));
}

__device__ __forceinline__ uint32_t word_of(uint4 v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// fp64 Box-Muller of one word pair; products explicitly rounded (no contraction).
__device__ __forceinline__ void box_muller(uint32_t wa, uint32_t wb, double &za, double &zb) {
    const double two_m32 = 2.3283064365386963e-10;
    const double u1 = __dmul_rn(__dadd_rn((double)wa, 1.0), two_m32);
    const double u2 = __dmul_rn((double)wb, two_m32);
    const double rad = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
    const double th = __dmul_rn(6.283185307179586, u2);
    za = __dmul_rn(rad, cos(th));
    zb = __dmul_rn(rad, sin(th));
}

// canonical weight index j -> device index (see the layout note above); network 1 keeps
// the canonical order (its device row is the canonical row padded to Pd)
__device__ __forceinline__ int canon_to_dev(int j, int I, int Hd, int off_hh, int off_b, int off_out,
                                            int off_bout);
__device__ __forceinline__ int canon_to_dev(const DevParams &p, int j) {
    return p.net == 1 ? j : canon_to_dev(j, p.I, p.Hd, p.off_hh, p.off_b, p.off_out, p.off_bout);
}
__device__ __forceinline__ int canon_to_dev(int j, int I, int Hd, int off_hh, int off_b, int off_out,
                                            int off_bout) {
    const int G = 4 * Hd;
    if (j < G * I) {
        const int r = j / I, col = j - r * I;
        const int g = r / Hd, k = r - g * Hd;
        return (col * Hd + k) * 4 + g;
    }
    j -= G * I;
    if (j < G * Hd) {
        const int r = j / Hd, col = j - r * Hd;
        const int g = r / Hd, k = r - g * Hd;
        return off_hh + (col * Hd + k) * 4 + g;
    }
    j -= G * Hd;
    if (j < G) {
        const int g = j / Hd, k = j - g * Hd;
        return off_b + k * 4 + g;
    }
    j -= G;
    if (j < 5 * Hd) return off_out + j;
    j -= 5 * Hd;
    return off_bout + j;
}

// ------------------------------------------------------------------- bit planes
__host__ __device__ __forceinline__ size_t plane_words(const DevParams &p) { return (size_t)p.H * p.WW; }

// row of a cell (cell / W) without an integer division: a double multiply (relative error
// < 2^-52, so the truncation is at most one below for cells < 2^31) plus one correction
__device__ __forceinline__ int row_of(const DevParams &p, int cell) {
    ECO_CHECK(cell >= 0 && (int64_t)cell < (int64_t)p.H * p.W);
    int y = __double2int_rz((double)cell * p.invW);
    y += (cell - y * p.W >= p.W) ? 1 : 0;
    return y;
}

__device__ __forceinline__ uint32_t get_bit(const uint32_t *plane, const DevParams &p, int cell) {
    const int y = row_of(p, cell), x = cell - y * p.W;
    return (plane[(size_t)y * p.WW + (x >> 5)] >> (x & 31)) & 1u;
}

__device__ __forceinline__ uint32_t *word_ptr(uint32_t *plane, const DevParams &p, int cell, uint32_t &bit) {
    const int y = row_of(p, cell), x = cell - y * p.W;
    bit = 1u << (x & 31);
    return plane + (size_t)y * p.WW + (x >> 5);
}

// n (<= 31) bits of row `row` starting at column x0 (may be negative / past the row);
// out-of-row bits read 0.
__device__ __forceinline__ uint32_t row_bits(const uint32_t *row, int WW, int x0, int n) {
    const int w0 = x0 >> 5;  // arithmetic shift: floor division
    const int b0 = x0 & 31;
    const uint32_t lo = (w0 >= 0 && w0 < WW) ? __ldg(row + w0) : 0u;
    const uint32_t hi = (w0 + 1 >= 0 && w0 + 1 < WW) ? __ldg(row + w0 + 1) : 0u;
    return __funnelshift_r(lo, hi, b0) & ((1u << n) - 1u);
}

__device__ __forceinline__ uint32_t *plane_cur(const DevParams &p, int64_t t) {
    return (t & 1) ? p.plane1 : p.plane0;
}
__device__ __forceinline__ uint32_t *plane_next(const DevParams &p, int64_t t) {
    return (t & 1) ? p.plane0 : p.plane1;
}
__device__ __forceinline__ uint32_t *bbits_of(const DevParams &p, int64_t t, int w) {
    return p.bbits + ((size_t)(t & 1) * p.n_worlds + w) * plane_words(p);
}
__device__ __forceinline__ int32_t *list_of(const DevParams &p, int64_t t, int w) {
    return p.alive_list + ((size_t)(t & 1) * p.n_worlds + w) * p.S;
}
__device__ __forceinline__ int32_t *list_cell_of(const DevParams &p, int64_t t, int w) {
    return p.list_cell + ((size_t)(t & 1) * p.n_worlds + w) * p.S;
}
__device__ __forceinline__ int32_t *count_of(const DevParams &p, int64_t t, int w) {
    return p.n_alive + (size_t)(t & 1) * p.n_worlds + w;
}

__device__ __forceinline__ sim_step_record *record_of(const DevParams &p, int64_t t, int w) {
    return p.log + (size_t)(t & (p.log_cap - 1)) * p.n_worlds + w;  // log_cap: a power of two
}

constexpr int GR_WINDOW = 20;   // sim.h SIM_GREED_WINDOW
constexpr int LE_WINDOW = 500;  // sim.h SIM_LIFE_WINDOW
__device__ __forceinline__ bool gr_window_end(int64_t t) { return (uint32_t)t % GR_WINDOW == GR_WINDOW - 1; }
// the greediness flag of one agent that ate in step t (the window's counts are closed after
// the window's last step by greed_pass_part, off the move phase's critical path)
#ifndef ECO_GREED
#define ECO_GREED 1  // diagnostic switch (0: no greediness bookkeeping)
#endif
__device__ __forceinline__ void greed_update(const DevParams &p, size_t gs, int64_t t, bool ate) {
    (void)t;
#if ECO_GREED
    if (ate) p.gr_ate[gs] = 1;
#endif
}
// Close greediness window T / 20 for world w's slots [lo, hi) (after the step's placement):
// every live agent adds its flags (a newborn of step T has none) and starts the next window.
__device__ __forceinline__ void greed_pass_part(const DevParams &p, int w, int lo, int hi, int tid, int nthr) {
    for (int i = lo + tid; i < hi; i += nthr) {
        const size_t gs = (size_t)w * p.S + i;
        if (!p.alive[gs]) continue;
        p.gr_T[gs] += p.gr_seen[gs];
        p.gr_C[gs] += p.gr_ate[gs];
        p.gr_seen[gs] = 0;
        p.gr_ate[gs] = 0;
    }
}

// energy <= e_death_le: immediately (BASELINE, R18) or after death_steps consecutive steps
// (the paper's timer); `low` is the agent's counter (updated here)
__device__ __forceinline__ bool starves(const DevParams &p, size_t gs, int en) {
    const bool below = en <= p.e_death_le;
    if (p.death_steps <= 0) return below;
    const int32_t l = below ? p.low[gs] + 1 : 0;
    p.low[gs] = l;
    return l >= p.death_steps;
}
constexpr int WALL_TARGET = -2;  // move record target of an agent walking into a lethal wall
__host__ __device__ __forceinline__ bool paper_rules(const DevParams &p) { return p.death_steps > 0 || p.lethal_walls; }

// the step's deaths into its 500-step window (one thread per world, after the step's counts)
__device__ __forceinline__ void life_window_add(const DevParams &p, int w, int64_t t, int64_t deaths, int64_t age_sum) {
    if (!deaths) return;
    unsigned long long *e = p.le + ((size_t)w * p.le_cap + (size_t)((t / LE_WINDOW) & (p.le_cap - 1))) * 2;
    atomicAdd(e, (unsigned long long)deaths);
    atomicAdd(e + 1, (unsigned long long)age_sum);
}

// N, S, E, W (R13 order for moves is stay, N, S, E, W; births use N, S, E, W = 0..3)
__device__ __forceinline__ int dir_dy(int d) { return d == 0 ? -1 : d == 1 ? 1 : 0; }
__device__ __forceinline__ int dir_dx(int d) { return d == 2 ? 1 : d == 3 ? -1 : 0; }

// ----------------------------------------------------------------- host launchers
struct LaunchCfg {
    int policy_blocks, policy_threads;
    int agent_blocks, agent_threads;
    int post_blocks;  // co-resident blocks of the cooperative k_post
    int sms;          // multiprocessors
};

cudaError_t launch_init_resources(const DevParams &p, cudaStream_t s);
size_t init_agents_scratch_bytes(const DevParams &p);
// band != nullptr: only the initial agents in the band's rows, in local slots 0.. (*n_own)
cudaError_t launch_init_agents(const DevParams &p, int n_initial, cudaStream_t s, void *scratch, size_t scratch_bytes,
                               const BandParams *band = nullptr, int32_t *n_own_dev = nullptr);
cudaError_t launch_rebuild(const DevParams &p, cudaStream_t s);
cudaError_t launch_regrow(const DevParams &p, int ahead, cudaStream_t s);
bool regrow_tiled(const DevParams &p);  // launch_regrow uses the shared-memory-tiled kernel
cudaError_t policy_prepare();  // kernel attributes (dynamic shared memory of k_policy_half)
// pdl: launched as a programmatic dependent of the preceding k_post (two-step graphs)
cudaError_t launch_policy(const DevParams &p, const LaunchCfg &lc, cudaStream_t s, bool pdl = false);
cudaError_t launch_move(const DevParams &p, const LaunchCfg &lc, cudaStream_t s);
cudaError_t launch_birth_claim(const DevParams &p, const LaunchCfg &lc, cudaStream_t s);
cudaError_t launch_birth_rank(const DevParams &p, cudaStream_t s);
cudaError_t launch_mutate(const DevParams &p, const LaunchCfg &lc, cudaStream_t s);
cudaError_t policy_occupancy(int hidden, int net, int *blocks_per_sm, int *threads);
cudaError_t post_occupancy(int *blocks_per_sm);
cudaError_t launch_post(const DevParams &p, const LaunchCfg &lc, unsigned long long *bar, cudaStream_t s);
cudaError_t launch_set_owner(const DevParams &p, cudaStream_t s);  // owner[slot] = slot % n_ranks,
                                                                  // own list of step t, zero records
bool policy_supports_shard();  // the Hd = 32 policy kernel of this build honours ownership
int policy_compact_worlds();  // most worlds the compacted policy mapping (pol_compact) supports
cudaError_t launch_prepare_p(const DevParams &p, const LaunchCfg &lc, cudaStream_t s);  // P of step t
cudaError_t launch_prepare_p_snap(const DevParams &p, const int64_t *snap, cudaStream_t s);  // banded
cudaError_t band_snap(const DevParams &p, const BandParams &bp, cudaStream_t s);
cudaError_t launch_advance_empty(const DevParams &p, cudaStream_t s);  // an agent-free world's step bookkeeping
cudaError_t band_snap0(const DevParams &p, const BandParams &bp, cudaStream_t s);
cudaError_t launch_prepare_p_list(const DevParams &p, const int32_t *list, const int32_t *n, int sms, cudaStream_t s);  // banded
cudaError_t post_prepare();  // kernel attributes of k_post (dynamic shared memory)

// banded mode (band.cu); kinds: halo 0 = X1, 1 = X4a; merge 0 = X2, 1 = X4b
cudaError_t band_halo(const DevParams &p, const BandParams &bp, int kind, cudaStream_t s);
cudaError_t band_merge(const DevParams &p, const BandParams &bp, int kind, cudaStream_t s);
cudaError_t band_move(const DevParams &p, const BandParams &bp, int sms, cudaStream_t s);
cudaError_t band_arrive(const DevParams &p, const BandParams &bp, int sms, cudaStream_t s);
cudaError_t band_live(const DevParams &p, const BandParams &bp, int sms, cudaStream_t s);
cudaError_t band_claims(const DevParams &p, const BandParams &bp, int sms, cudaStream_t s);
cudaError_t band_rank(const DevParams &p, const BandParams &bp, cudaStream_t s);
cudaError_t band_mutate(const DevParams &p, const BandParams &bp, int sms, cudaStream_t s);
cudaError_t band_newborns(const DevParams &p, const BandParams &bp, int sms, cudaStream_t s);
cudaError_t band_init_agents(const DevParams &p, const BandParams &bp, int n_initial, const unsigned long long *sorted,
                             int32_t *n_own, cudaStream_t s);
size_t band_box_words(int W, int S, int Hd, int Pd, bool newborn);
cudaError_t launch_mv_pass(const DevParams &p, cudaStream_t s);  // movement histograms at a window end

// state conversion (canonical <-> device)
cudaError_t launch_pack_resources(const DevParams &p, const uint8_t *bytes, cudaStream_t s);
cudaError_t launch_unpack_resources(const DevParams &p, uint8_t *bytes, cudaStream_t s);
cudaError_t launch_logits_restride(float *dst, int dst_stride, const float *src, int src_stride, size_t n,
                                   cudaStream_t s);
cudaError_t launch_weights_to_device(const DevParams &p, const float *canon, size_t first_agent, size_t n_agents,
                                     cudaStream_t s);
cudaError_t launch_weights_gather(const DevParams &p, const float *src, bool by_slot, const int32_t *live, int n_live,
                                  float *stage, int32_t *bad, cudaStream_t s);
cudaError_t launch_weights_scatter(const DevParams &p, const float *stage, const int32_t *live, int n_live,
                                   cudaStream_t s);
// device-layout weights of slots list[k] (k < n) -> canonical rows k of `canon`
cudaError_t launch_weights_to_canon_list(const DevParams &p, const int32_t *list, int n, float *canon, cudaStream_t s);
cudaError_t launch_weights_to_canon(const DevParams &p, float *canon, size_t first_agent, size_t n_agents,
                                    cudaStream_t s);

}  // namespace eco
