// births.cu — reproduction half of step row a5:
//   K4 k_birth_rank  one CTA per world: the first n_place = min(winners, free slots) free
//                    slots in ascending order (prefix scan of the alive bitmap) and the first
//                    n_place winning child cells in row-major order (prefix scan of the birth
//                    bitmap); both scans stop as soon as n_place entries are found.  Rank r
//                    gets free slot F[r] (R22); every later winner is deferred for capacity.
//                    Then the step's counters, the next alive list and t += 1.
//   K5 k_mutate      child weights = parent weights + (float)(sigma * z), z ~ N(0,1) from
//                    fp64 Box-Muller on Philox (MUTATE, t, child cell, j >> 2).
#include "block_scan.cuh"
#include "sim_internal.cuh"

namespace eco {

constexpr int RANK_THREADS = 1024;

__global__ void __launch_bounds__(RANK_THREADS) k_birth_rank(DevParams p) {
    __shared__ uint32_t scratch[RANK_THREADS / 32 + 1];
    const int w = blockIdx.x;
    const int tid = threadIdx.x;
    const int64_t t = p.t[w];
    const size_t HW = (size_t)p.H * p.W;
    const size_t pw = plane_words(p);
    const int n_start = *count_of(p, t, w);
    const int n_surv = *count_of(p, t + 1, w);  // survivors appended by K3
    const int n_win = p.n_win[w];
    const int n_free = p.S - n_surv;
    const int n_place = n_win < n_free ? n_win : n_free;
    uint32_t *O = p.occ + (size_t)w * pw;
    int32_t *next_list = list_of(p, t + 1, w);

    if (n_place > 0) {
        // 1. the first n_place free slots, ascending
        uint32_t running = 0u;
        for (int w0 = 0; w0 < p.SW; w0 += RANK_THREADS) {
            const int wi = w0 + tid;
            uint32_t fr = 0u;
            if (wi < p.SW) {
                const int nbits = p.S - wi * 32;
                const uint32_t valid = nbits >= 32 ? 0xffffffffu : ((1u << nbits) - 1u);
                fr = ~p.alive_bits[(size_t)w * p.SW + wi] & valid;
            }
            uint32_t tot;
            const uint32_t ex = block_exclusive_scan<RANK_THREADS>((uint32_t)__popc(fr), scratch, tot);
            uint32_t r = running + ex;
            while (fr && r < (uint32_t)n_place) {
                const int b = __ffs(fr) - 1;
                fr &= fr - 1u;
                p.free_list[(size_t)w * p.S + r] = wi * 32 + b;
                ++r;
            }
            running += tot;
            if (running >= (uint32_t)n_place) break;
        }
        __syncthreads();
        // 2. the first n_place winning child cells in row-major order, placed
        const uint32_t *bb = bbits_of(p, t, w);
        running = 0u;
        for (size_t w0 = 0; w0 < pw; w0 += RANK_THREADS) {
            const size_t wi = w0 + tid;
            uint32_t word = wi < pw ? bb[wi] : 0u;
            uint32_t tot;
            const uint32_t ex = block_exclusive_scan<RANK_THREADS>((uint32_t)__popc(word), scratch, tot);
            uint32_t r = running + ex;
            while (word && r < (uint32_t)n_place) {
                const int b = __ffs(word) - 1;
                word &= word - 1u;
                const int y = (int)(wi / p.WW), x = (int)(wi - (size_t)y * p.WW) * 32 + b;
                const int c = y * p.W + x;
                const int parent = p.bparent[(size_t)w * HW + c];
                const int child = p.free_list[(size_t)w * p.S + r];
                const size_t cs = (size_t)w * p.S + child;
                p.alive[cs] = 1;
                atomicOr(p.alive_bits + (size_t)w * p.SW + (child >> 5), 1u << (child & 31));
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
                uint32_t bit;
                atomicOr(word_ptr(O, p, c, bit), bit);
                p.repr[(size_t)w * p.S + parent] = 0;
                p.birth_child[(size_t)w * p.S + r] = child;
                p.birth_parent[(size_t)w * p.S + r] = parent;
                next_list[n_surv + r] = child;
                ++r;
            }
            running += tot;
            if (running >= (uint32_t)n_place) break;
        }
    }
    __syncthreads();

    // 3. counters, next alive count, t += 1
    if (tid == 0) {
        sim_step_record *rec = record_of(p, t, w);
        const int64_t deaths = rec->deaths_energy + rec->deaths_age;
        p.res_count[w] += rec->grown - rec->eaten;
        rec->t = t;
        rec->agents_at_start = n_start;
        rec->births = n_place;
        rec->deferred_capacity = n_win - n_place;
        rec->population = n_surv + n_place;
        rec->resources = p.res_count[w];
        *count_of(p, t + 1, w) = n_surv + n_place;
        p.n_births[w] = n_place;
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
