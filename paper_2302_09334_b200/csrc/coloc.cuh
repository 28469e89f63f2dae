// coloc.cuh — the co-location step (readings R43-R47): the paper's
// own reproduction, "the off-spring appears on the same cell as its parent",
// with any number of agents per cell (the agent channel counts them).
// Included by step.cu inside namespace eco.  Used with network 1 (k_policy_cnn_blk), which
// reads the per-cell counts `ncount` for its agent channel and posts no move claims.
//
//   k_co_move   a4: every in-grid move succeeds (no collision exclusion, R43); a lethal wall
//               kills; counts follow the agents; an agent on a cell holding a resource
//               posts its lottery key (CONSUME draw of its slot << 32 | ~slot) with
//               atomicMax on the cell's claim word (R45)
//   k_co_live   a4: the key holder of a resource cell eats (exactly one per cell,
//               SPEC.md:273); energy, age, timers, death; survivors listed for t+1; the
//               eligible parents marked in a slot bitmap (R46)
//   k_co_rank   a5, one block per world: the eligible parents in slot order take the free
//               slots in ascending order (a dual prefix scan of the alive and eligible
//               bitmaps), each child on its parent's cell, the lottery words reset, the
//               step's counters, t += 1; the birth lists carry the child SLOT as the
//               mutation's Philox entity (R47: co-located children share a cell)
//               (and the metrics windows ending here)
// then k_mutate and k_regrow of step t+1.

#ifndef ECO_CO_THREADS
#define ECO_CO_THREADS 384  // threads per block of k_co_rank and k_post_co (measured: 1024 34.4, 768 32.6, 512 31.0, 384 30.8, 256 32.7 us per step)
#endif
constexpr int CO_THREADS = ECO_CO_THREADS;

__device__ __forceinline__ void co_move_phase(const DevParams &p, size_t gtid, size_t gthreads) {
    const long total = (long)p.n_worlds * p.S;
    const size_t HW = (size_t)p.H * p.W;
    for (long v = (long)gtid; v < total; v += (long)gthreads) {
        const AgentIter it = agent_at(p, v);
        const int w = it.w;
        const int64_t t = p.t[w];
        if (it.i >= *count_of(p, t, w)) continue;
        int4 mr = p.mrec[(size_t)w * p.S + it.i];
        const int slot = mr.x;
        ECO_CHECK(slot >= 0 && slot < p.S);
        const size_t gs = (size_t)w * p.S + slot;
        int cellv = mr.y;
        int32_t *cnt = p.ncount + (size_t)w * HW;
        if (mr.z == WALL_TARGET) {  // walked into a lethal wall: dies before eating (R36)
            p.alive[gs] = 0;
            p.ate[gs] = 0;
            greed_update(p, gs, t, false);
            atomicSub(cnt + cellv, 1);
            atomicAnd(p.alive_bits + (size_t)w * p.SW + (slot >> 5), ~(1u << (slot & 31)));
            sim_step_record *rec = record_of(p, t, w);
            atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deaths_wall), 1ull);
#if ECO_METRICS & 1
            atomicAdd(reinterpret_cast<unsigned long long *>(&rec->death_age_sum), (unsigned long long)(p.age[gs] + 1));
#endif
            continue;
        }
        if (mr.z >= 0) {  // R43: the move always succeeds
            atomicSub(cnt + cellv, 1);
            atomicAdd(cnt + mr.z, 1);
            cellv = mr.z;
            p.cell[gs] = cellv;
        }
        mr.w = cellv;  // the final cell (k_co_live, the lottery reset in k_co_rank)
        p.mrec[(size_t)w * p.S + it.i] = mr;
        uint32_t bit;
        const uint32_t *rw = word_ptr(plane_next(p, t) + (size_t)w * plane_words(p), p, cellv, bit);
        if (ld_plain(rw) & bit) {
            const uint4 d = draw4(p.seeds[w], PURPOSE_CONSUME, (uint32_t)t, (uint32_t)slot, 0u);
            atomicMax(p.claim + (size_t)w * HW + cellv,
                      ((unsigned long long)d.x << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)slot));
        }
    }
}

__device__ __forceinline__ void co_live_phase(const DevParams &p, size_t gtid, size_t gthreads) {
    const long total = (long)p.n_worlds * p.S;
    const size_t HW = (size_t)p.H * p.W;
    for (long v = (long)gtid; v < total; v += (long)gthreads) {
        const AgentIter it = agent_at(p, v);
        const int w = it.w;
        const int64_t t = p.t[w];
        if (it.i >= *count_of(p, t, w)) continue;
        const int4 mr = p.mrec[(size_t)w * p.S + it.i];
        if (mr.z == WALL_TARGET) continue;
        const int slot = mr.x, cellv = mr.w;
        const size_t gs = (size_t)w * p.S + slot;
        sim_step_record *rec = record_of(p, t, w);
        uint32_t bit;
        uint32_t *rw = word_ptr(plane_next(p, t) + (size_t)w * plane_words(p), p, cellv, bit);
        bool ate = false;
        if (ld_plain(rw) & bit) {  // the lottery (R45): only the key holder eats
            const uint4 d = draw4(p.seeds[w], PURPOSE_CONSUME, (uint32_t)t, (uint32_t)slot, 0u);
            const unsigned long long key =
                ((unsigned long long)d.x << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)slot);
            ate = p.claim[(size_t)w * HW + cellv] == key;
        }
        if (ate) {
            atomicAnd(rw, ~bit);
            atomicAdd(reinterpret_cast<unsigned long long *>(&rec->eaten), 1ull);
        }
        p.ate[gs] = ate ? 1 : 0;
        greed_update(p, gs, t, ate);
        long long e = (long long)p.energy[gs] + (ate ? (long long)p.e_gain : 0ll) - (long long)p.e_decay;
        if (p.e_max != 0x7fffffff && e > p.e_max) e = p.e_max;
        const int en = (int)e, ag = p.age[gs] + 1;
        p.energy[gs] = en;
        p.age[gs] = ag;
        const int rp = en > p.e_repr_gt ? p.repr[gs] + 1 : 0;
        p.repr[gs] = rp;
        const bool died_e = starves(p, gs, en), died_a = !died_e && ag > p.max_age;
        if (died_e || died_a) {
            p.alive[gs] = 0;
            atomicSub(p.ncount + (size_t)w * HW + cellv, 1);
            atomicAnd(p.alive_bits + (size_t)w * p.SW + (slot >> 5), ~(1u << (slot & 31)));
            atomicAdd(reinterpret_cast<unsigned long long *>(died_e ? &rec->deaths_energy : &rec->deaths_age), 1ull);
#if ECO_METRICS & 1
            atomicAdd(reinterpret_cast<unsigned long long *>(&rec->death_age_sum), (unsigned long long)ag);
#endif
            continue;
        }
        const int q = atomicAdd(count_of(p, t + 1, w), 1);
        ECO_CHECK(q < p.S);
        list_of(p, t + 1, w)[q] = slot;
        list_cell_of(p, t + 1, w)[q] = cellv;
        if (rp >= p.repr_steps) {  // an eligible parent (R19, R46)
            atomicOr(p.elig_bits + (size_t)w * p.SW + (slot >> 5), 1u << (slot & 31));
            atomicAdd(p.n_win + w, 1);
            atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deferred_claim), 1ull);  // candidates
        }
    }
}

// The free slots (alive bitmap zeros) and the eligible parents (elig_bits ones) of ranks
// r < n_place, both in ascending slot order, into s_free / s_par (r < RANK_SMEM_CAP) or the
// global lists; chunks of NT words scanned together.
template <int NT>
__device__ void co_rank_lists(const DevParams &p, int w, int n_place, uint32_t *scratch, int *s_free, int *s_par,
                              int32_t *g_free, int32_t *g_par) {
    const int tid = threadIdx.x;
    const uint32_t *ab = p.alive_bits + (size_t)w * p.SW, *eb = p.elig_bits + (size_t)w * p.SW;
    uint32_t run_f = 0u, run_e = 0u;
    for (size_t j = 0; (run_f < (uint32_t)n_place || run_e < (uint32_t)n_place) && j * NT < (size_t)p.SW; ++j) {
        const size_t wi = j * NT + tid;
        uint32_t fr = 0u, el = 0u;
        if (wi < (size_t)p.SW) {
            const int nbits = p.S - (int)wi * 32;
            const uint32_t valid = nbits >= 32 ? 0xffffffffu : ((1u << nbits) - 1u);
            fr = ~ld_plain(ab + wi) & valid;
            el = ld_plain(eb + wi);
        }
        uint2 tot;
        const uint2 ex = block_exclusive_scan2<NT>(make_uint2((uint32_t)__popc(fr), (uint32_t)__popc(el)), scratch, tot);
        uint32_t r = run_f + ex.x;
        for (; fr && r < (uint32_t)n_place; fr &= fr - 1u, ++r) {
            const int slot = (int)wi * 32 + __ffs(fr) - 1;
            if (r < RANK_SMEM_CAP) s_free[r] = slot;
            else g_free[r] = slot;
        }
        r = run_e + ex.y;
        for (; el && r < (uint32_t)n_place; el &= el - 1u, ++r) {
            const int slot = (int)wi * 32 + __ffs(el) - 1;
            if (r < RANK_SMEM_CAP) s_par[r] = slot;
            else g_par[r] = slot;
        }
        run_f += tot.x;
        run_e += tot.y;
    }
    __syncthreads();
}

// World w's rank, placement, counters, t += 1, then its movement / greediness windows ending
// here; all CO_THREADS threads of one block.
__device__ __forceinline__ void co_rank_world(const DevParams &p, int w, uint32_t *scratch, int *s_free, int *s_par,
                                              int *s_mv) {
    const size_t HW = (size_t)p.H * p.W;
    const int64_t t = p.t[w];
    const RankCounts k = rank_counts(p, w, t);  // n_win = eligible parents (k_co_live)
    const size_t ws = (size_t)w * p.S;
    int32_t *g_free = p.free_list + ws, *g_par = p.birth_parent + ws;
    if (k.n_place > 0) co_rank_lists<CO_THREADS>(p, w, k.n_place, scratch, s_free, s_par, g_free, g_par);
    for (int r = threadIdx.x; r < k.n_place; r += CO_THREADS) {
        const bool sm = r < RANK_SMEM_CAP;
        const int child = sm ? s_free[r] : *reinterpret_cast<volatile int32_t *>(g_free + r);
        const int par = sm ? s_par[r] : *reinterpret_cast<volatile int32_t *>(g_par + r);
        const int c = p.cell[ws + par];  // R46: the parent's cell
        place_child(p, w, t, c, r, k.n_surv, child, par);
        atomicAdd(p.ncount + (size_t)w * HW + c, 1);
        p.birth_child[ws + r] = child;
        p.birth_parent[ws + r] = par;
        p.birth_cell[ws + r] = child;  // the mutation's Philox entity: the child's slot (R47)
    }
    // the lottery words of this step's cells, and the eligible bitmap, back to zero
    for (int i = threadIdx.x; i < k.n_start; i += CO_THREADS) {
        const int4 mr = p.mrec[ws + i];
        if (mr.z != WALL_TARGET) p.claim[(size_t)w * HW + mr.w] = 0ull;
    }
    for (int j = threadIdx.x; j < p.SW; j += CO_THREADS) p.elig_bits[(size_t)w * p.SW + j] = 0u;
    __syncthreads();
    if (threadIdx.x == 0) {
        p.n_births[w] = k.n_place;
        rank_finalize(p, w, t, k.n_start, k.n_surv, k.n_win, k.n_place);
        p.t[w] = t + 1;
    }
    __syncthreads();
#if ECO_METRICS & 2
    if (mv_window_end(t)) mv_pass_part(p, t, w, 0, p.S, threadIdx.x, blockDim.x, s_mv);
#endif
    if (gr_window_end(t)) greed_pass_part(p, w, 0, p.S, threadIdx.x, blockDim.x);
}

// One block per world.  (The regrowth of step t+1 is a separate launch in the instrumented
// path: a block regrowing beside this one could start after t advanced; k_post_co reads t
// first and keeps every block resident.)
__global__ void __launch_bounds__(CO_THREADS) k_co_rank(DevParams p) {
    __shared__ uint32_t scratch[2 * (CO_THREADS / 32 + 1)];
    __shared__ int s_free[RANK_SMEM_CAP], s_par[RANK_SMEM_CAP];
    __shared__ int s_mv[SIM_MOVE_BINS];
    for (int w = blockIdx.x; w < p.n_worlds; w += gridDim.x) co_rank_world(p, w, scratch, s_free, s_par, s_mv);
}

__global__ void __launch_bounds__(256) k_co_move(DevParams p) {
    co_move_phase(p, (size_t)blockIdx.x * blockDim.x + threadIdx.x, (size_t)gridDim.x * blockDim.x);
}
__global__ void __launch_bounds__(256) k_co_live(DevParams p) {
    co_live_phase(p, (size_t)blockIdx.x * blockDim.x + threadIdx.x, (size_t)gridDim.x * blockDim.x);
}

// Graph mode: the whole post-policy step in one cooperative launch (one block per SM), the
// phases separated by grid barriers instead of kernel boundaries: move | live | rank (one
// block per world) beside the regrowth of step t+1 (the other blocks; t read before any
// block advances it) | mutation.
__global__ void __launch_bounds__(CO_THREADS) k_post_co(DevParams p, unsigned long long *bar) {
    __shared__ uint32_t scratch[2 * (CO_THREADS / 32 + 1)];
    __shared__ int s_free[RANK_SMEM_CAP], s_par[RANK_SMEM_CAP];
    __shared__ int s_mv[SIM_MOVE_BINS];
#if ECO_POST_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the policy grid has completed (programmatic dependent)
#endif
    unsigned long long target = grid_sync_base(bar);
    const int64_t T = p.t[0];  // (all worlds share t)
    const size_t gtid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, gthreads = (size_t)gridDim.x * blockDim.x;
    co_move_phase(p, gtid, gthreads);
    grid_sync(bar, target);
    co_live_phase(p, gtid, gthreads);
    grid_sync(bar, target);
    const bool spare = (int)gridDim.x > p.n_worlds;  // blocks left over for the regrowth
    if ((int)blockIdx.x < p.n_worlds) {
        for (int w = blockIdx.x; w < p.n_worlds; w += gridDim.x) co_rank_world(p, w, scratch, s_free, s_par, s_mv);
    } else {
        const size_t b = blockIdx.x - p.n_worlds, nb = gridDim.x - p.n_worlds;
        regrow_phase(p, T + 1, b * blockDim.x + threadIdx.x, nb * blockDim.x);
    }
    grid_sync(bar, target);
    mutate_phase(p, gtid, gthreads, s_free, RANK_SMEM_CAP);  // (the rank's lists are consumed: s_free is free)
    if (!spare) regrow_phase(p, T + 1, gtid, gthreads);
    if (blockIdx.x == 0 && threadIdx.x == 0) grid_sync_done(bar, target);
}
