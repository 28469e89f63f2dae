// births.cu — reproduction half of step row a5:
//   K4 k_birth_rank  winners of the birth claims, free-slot and alive-list compaction
//                    (prefix scans), rank of every winner by child cell (prefix scan of
//                    the birth bitmap, stopped as soon as every free slot is assigned),
//                    slot assignment / capacity deferral, per-step counters, t += 1.
//   K5 k_mutate      child weights = parent weights + (float)(sigma * z), z ~ N(0,1) from
//                    fp64 Box-Muller on Philox (MUTATE, t, child cell, j >> 2).
#include "block_scan.cuh"
#include "sim_internal.cuh"

namespace eco {

constexpr int RANK_THREADS = 1024;

__global__ void __launch_bounds__(RANK_THREADS) k_birth_rank(DevParams p) {
    __shared__ uint32_t scratch[RANK_THREADS / 32 + 1];
    __shared__ unsigned s_win, s_lost;
    __shared__ uint32_t s_limit;
    const int w = blockIdx.x;
    const int tid = threadIdx.x;
    const int64_t t = p.t[w];
    const int n_start = p.n_alive[w];
    const int n_cand = p.n_cand[w];
    const size_t HW = (size_t)p.H * p.W;
    const size_t pw = plane_words(p);
    uint32_t *bb = p.bbits + (size_t)w * pw;
    uint32_t *O = p.occ + (size_t)w * pw;
    if (tid == 0) {
        s_win = 0u;
        s_lost = 0u;
    }
    __syncthreads();

    // 1. winners: the parent holding the max key on its candidate cell
    unsigned my_win = 0u, my_lost = 0u;
    for (int i = tid; i < n_cand; i += RANK_THREADS) {
        const int slot = p.cand_list[(size_t)w * p.S + i];
        const size_t gs = (size_t)w * p.S + slot;
        const int c = p.bcand[gs];
        const bool win = p.bclaim[(size_t)w * HW + c] == p.bkey[gs];
        p.bwin[gs] = win ? 1 : 0;
        if (win) {
            uint32_t bit;
            uint32_t *wp = word_ptr(bb, p, c, bit);
            atomicOr(wp, bit);
            ++my_win;
        } else {
            ++my_lost;
        }
    }
    if (my_win) atomicAdd(&s_win, my_win);
    if (my_lost) atomicAdd(&s_lost, my_lost);
    __syncthreads();
    const int n_win = (int)s_win;

    // 2. lazy reset of the birth claims (all reads above are done)
    for (int i = tid; i < n_cand; i += RANK_THREADS) {
        const int slot = p.cand_list[(size_t)w * p.S + i];
        p.bclaim[(size_t)w * HW + p.bcand[(size_t)w * p.S + slot]] = 0ull;
    }

    // 3. one pass over the slots after deaths: ascending free list F and alive list
    uint32_t base_alive = 0u, base_free = 0u;
    for (int i0 = 0; i0 < p.S; i0 += RANK_THREADS * 4) {
        const int i = i0 + tid * 4;
        uint32_t fl = 0u;  // bit m = alive flag of slot i+m (4 = valid marker)
        uint32_t na = 0u, nf = 0u;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            if (i + m < p.S) {
                const bool a = p.alive[(size_t)w * p.S + i + m] != 0;
                fl |= (a ? 1u : 0u) << m;
                na += a ? 1u : 0u;
                nf += a ? 0u : 1u;
            }
        }
        uint32_t tot;
        const uint32_t ex = block_exclusive_scan<RANK_THREADS>(na | (nf << 16), scratch, tot);
        uint32_t oa = base_alive + (ex & 0xffffu), of = base_free + (ex >> 16);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            if (i + m < p.S) {
                if ((fl >> m) & 1u) p.alive_list[(size_t)w * p.S + (oa++)] = i + m;
                else p.free_list[(size_t)w * p.S + (of++)] = i + m;
            }
        }
        base_alive += tot & 0xffffu;
        base_free += tot >> 16;
    }
    const int n_free = (int)base_free;
    const int n_alive_ad = (int)base_alive;
    const int n_place = n_win < n_free ? n_win : n_free;

    // 4. rank = number of winning child cells before this one in row-major order: scan
    //    the birth bitmap, stopping once n_place winners are covered (later winners are
    //    deferred for capacity whatever their exact rank).
    uint32_t running = 0u, limit = 0u;
    if (n_place > 0) {
        for (size_t w0 = 0; w0 < pw; w0 += RANK_THREADS) {
            const size_t wi = w0 + tid;
            const uint32_t val = wi < pw ? (uint32_t)__popc(bb[wi]) : 0u;
            uint32_t tot;
            const uint32_t ex = block_exclusive_scan<RANK_THREADS>(val, scratch, tot);
            if (wi < pw) p.bprefix[(size_t)w * pw + wi] = running + ex;
            running += tot;
            limit = (uint32_t)((w0 + RANK_THREADS < pw) ? w0 + RANK_THREADS : pw);
            if (running >= (uint32_t)n_place) break;
        }
    }
    if (tid == 0) s_limit = limit;
    __syncthreads();
    limit = s_limit;

    // 5. placement: rank r < |F| takes free slot F[r] (R22); the child starts fresh
    for (int i = tid; i < n_cand; i += RANK_THREADS) {
        const int slot = p.cand_list[(size_t)w * p.S + i];
        const size_t gs = (size_t)w * p.S + slot;
        if (!p.bwin[gs]) continue;
        const int c = p.bcand[gs];
        const int y = c / p.W, x = c - y * p.W;
        const size_t wi = (size_t)y * p.WW + (x >> 5);
        const uint32_t below = (1u << (x & 31)) - 1u;
        int rank = 0x7fffffff;
        if (wi < limit) rank = (int)(p.bprefix[(size_t)w * pw + wi] + __popc(bb[wi] & below));
        if (rank < n_place) {
            const int child = p.free_list[(size_t)w * p.S + rank];
            const size_t cs = (size_t)w * p.S + child;
            p.alive[cs] = 1;
            p.cell[cs] = c;
            p.energy[cs] = p.e_init;
            p.age[cs] = 0;
            p.repr[cs] = 0;
            p.last_action[cs] = 0;
            p.ate[cs] = 0;
            for (int k = 0; k < p.Hd; ++k) {
                p.h[cs * p.Hd + k] = 0.f;
                p.c[cs * p.Hd + k] = 0.f;
            }
            for (int a = 0; a < LOGIT_STRIDE; ++a) p.logits[cs * LOGIT_STRIDE + a] = 0.f;
            p.target[cs] = -1;
            p.bcand[cs] = -1;
            uint32_t bit;
            atomicOr(word_ptr(O, p, c, bit), bit);
            p.repr[gs] = 0;
            p.birth_child[(size_t)w * p.S + rank] = child;
            p.birth_parent[(size_t)w * p.S + rank] = slot;
            p.alive_list[(size_t)w * p.S + n_alive_ad + rank] = child;
        }
    }
    __syncthreads();

    // 6. clear the birth bitmap
    for (int i = tid; i < n_cand; i += RANK_THREADS) {
        const int slot = p.cand_list[(size_t)w * p.S + i];
        const size_t gs = (size_t)w * p.S + slot;
        if (!p.bwin[gs]) continue;
        uint32_t bit;
        *word_ptr(bb, p, p.bcand[gs], bit) = 0u;
    }

    // 7. counters, lists, t += 1
    if (tid == 0) {
        sim_step_record *rec = record_of(p, t, w);
        const int64_t deaths = rec->deaths_energy + rec->deaths_age;
        p.res_count[w] += rec->grown - rec->eaten;
        rec->t = t;
        rec->agents_at_start = n_start;
        rec->births = n_place;
        rec->deferred_claim = (int64_t)s_lost;
        rec->deferred_capacity = n_win - n_place;
        rec->population = n_alive_ad + n_place;
        rec->resources = p.res_count[w];
        p.n_alive[w] = n_alive_ad + n_place;
        p.n_births[w] = n_place;
        p.n_cand[w] = 0;
        unsigned long long *tot = p.totals;
        if (w == 0) atomicAdd(tot + 0, 1ull);
        atomicAdd(tot + 1, (unsigned long long)n_start);
        atomicAdd(tot + 2, (unsigned long long)HW);
        atomicAdd(tot + 3, (unsigned long long)n_place);
        atomicAdd(tot + 4, (unsigned long long)deaths);
        atomicAdd(tot + 5, (unsigned long long)rec->eaten);
        atomicAdd(tot + 6, (unsigned long long)rec->grown);
        sim_step_record *nxt = record_of(p, t + 1, w);
        *nxt = sim_step_record{};
        nxt->t = t + 1;
        p.t[w] = t + 1;
    }
}

cudaError_t launch_birth_rank(const DevParams &p, cudaStream_t s) {
    k_birth_rank<<<p.n_worlds, RANK_THREADS, 0, s>>>(p);
    return cudaGetLastError();
}

// ----------------------------------------------------------------------- K5 mutate
// "an agent's weights are mutated by adding noise sampled from N(0, sigma)",
// sigma = 0.02 a standard deviation (R23).  One thread per canonical group q = j >> 2:
// one Philox call, two Box-Muller pairs, four weights.
__global__ void __launch_bounds__(128) k_mutate(DevParams p) {
    const int groups = (p.P + 3) >> 2;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= groups) return;
    for (int w = 0; w < p.n_worlds; ++w) {
        const int nb = p.n_births[w];
        if (nb == 0) continue;
        const int64_t t = p.t[w] - 1;  // K4 already advanced the step index
        const uint64_t seed = p.seeds[w];
        for (int b = blockIdx.y; b < nb; b += gridDim.y) {
            const int child = p.birth_child[(size_t)w * p.S + b];
            const int parent = p.birth_parent[(size_t)w * p.S + b];
            const size_t cs = (size_t)w * p.S + child, ps = (size_t)w * p.S + parent;
            const uint4 d = draw4(seed, PURPOSE_MUTATE, (uint32_t)t, (uint32_t)p.cell[cs], (uint32_t)q);
            double z[4];
            box_muller(d.x, d.y, z[0], z[1]);
            box_muller(d.z, d.w, z[2], z[3]);
            const float *wp = p.weights + ps * (size_t)p.Pd;
            float *wc = p.weights + cs * (size_t)p.Pd;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int j = 4 * q + m;
                if (j >= p.P) break;
                const int dd = canon_to_dev(j, p.I, p.Hd, p.off_hh, p.off_b, p.off_out, p.off_bout);
                wc[dd] = __fadd_rn(wp[dd], __double2float_rn(__dmul_rn(p.mutation_std, z[m])));
            }
        }
    }
}

cudaError_t launch_mutate(const DevParams &p, const LaunchCfg &lc, cudaStream_t s) {
    if (p.S == 0) return cudaSuccess;
    const int groups = (p.P + 3) >> 2;
    dim3 grid((groups + 127) / 128, lc.mutate_blocks_y);
    k_mutate<<<grid, 128, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace eco
