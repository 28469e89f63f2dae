// band.cu — one world split into latitude bands (BASELINE configs[3]).
//
// Band b of G owns the grid rows [y0, y1) and the agents standing in them; every band keeps
// the GLOBAL coordinate system (planes and per-cell buffers of the whole H x W grid, cells
// y*W + x), so every draw is keyed by the global cell exactly as in the unsharded world
// (R9) and a band computes bit for bit what the unsharded step computes for its rows.  A
// band reads nothing of the grid outside its rows except halo rows copied from its two
// neighbours.  One world step t of every band (sim_step on a banded handle, api.cu):
//
//   X1  halo: R'_t rows [y0-3, y0) and [y1, y1+3) and O_t rows of the same ranges from the
//       neighbours (the observation radius r <= 3; R' is already regrown there, so no
//       redundant halo regrowth is needed)
//   P1  policy of the own agents (the unsharded kernel: observation, LSTM, argmax, move
//       claims by atomicMax into the per-cell claim buffer, halo targets included)
//   X2  the claims on the boundary rows {y0-1, y0} and {y1-1, y1}: max-merged both ways, so
//       both bands hold the same winner for every cell a move can contest across the edge
//   P3  move resolution (R14): an own agent whose winning target lies in a neighbour's row
//       leaves (its whole state and weights packed into the outbox towards that neighbour)
//   X3  arrivals: the neighbours' migrants towards this band take the first free local
//       slots (ascending) and join the agents processed next
//   P5  consumption, physiology, death of the band's agents (stayers and arrivals)
//   X4a R'' = R_{t+1} rows [y0-2, y0), [y1, y1+2) and O'' rows y0-1, y1 from the neighbours
//   P7  birth candidates and claims of the own eligible parents (R21; halo cells included)
//   X4b the birth-claim keys and claimed-cell bits of the boundary rows, max/OR-merged
//   P9  counts (kept by P5, P7 and X4b): claimed cells in the own rows, survivors; ALL
//       bands' counts are read (the capacity rule R22 is global: claimed cells are ranked
//       row-major over the whole grid, i.e. band order then local order, and the first
//       S - A_total are placed)
//   P10 rank and placement of the children in the own rows (first free local slots); a
//       parent whose child's cell lies in a neighbour's row computes the child's global rank
//       itself (from the merged boundary-row bits and the counts), so both sides take the
//       same capacity decision; such a parent's mutated child weights go to the neighbour
//   P11 mutation (children of local parents, and the outgoing newborns' weights)
//   P13 regrowth of step t+1 on the own rows (R_{t+1} rows y0-2 .. y1+1 are present)
//   X5  incoming newborns' weights into the child slots placed in P10, pulled with the next
//       step's X1 (before the children's first policy; sim_get_state pulls them too)
//
// Exchanges are PULLS: a band's kernel reads its neighbour's buffers (device pointers of
// another band of this process, or peer memory mapped from another GPU).  Between a
// producing phase and the pulling phase every band passes a barrier (a no-op when all bands
// run in order on one stream; stream-ordered NCCL tokens across GPUs).  A buffer a
// neighbour pulls after barrier Xk is modified by its owner only after barrier X(k+1), so
// no pull races a write; max/OR merges are idempotent, so the two directions of a merge may
// interleave freely.
#include "phases.cuh"

namespace eco {

// ------------------------------------------------------------------ record layouts
// migrant record (int32 words): [0] cell (the new one), [1] energy, [2] age, [3] repr,
// [4] last_action, [5] ate, [6] mv_cell, [7] mv_inv, [8] source slot, [9] greediness T_r,
// [10] C_r, [11] the window's flags (seen | ate << 1), [12] the death timer, [16..24) logits,
// [24, 24+Hd) h, [24+Hd, 24+2Hd) c, [24+2Hd, +Pd) weights in the device layout.
// newborn record: [0] cell, [1] parent slot, [4, 4+Pd) weights (device layout, mutated).
// An outbox direction: [0] count, records from word 4.  dir 0 = towards band b-1 (up),
// dir 1 = towards b+1 (down).
constexpr int MIG_HDR = 24, NB_HDR = 4, BOX_HDR = 4;

__host__ __device__ __forceinline__ int mig_stride(int Hd, int Pd) { return MIG_HDR + 2 * Hd + Pd; }
__host__ __device__ __forceinline__ int nb_stride(int Pd) { return NB_HDR + Pd; }

__device__ __forceinline__ int32_t *box_dir(int32_t *box, int dir, int cap, int stride) {
    return box + (size_t)dir * (BOX_HDR + (size_t)cap * stride);
}
__device__ __forceinline__ const int32_t *box_dir(const int32_t *box, int dir, int cap, int stride) {
    return box + (size_t)dir * (BOX_HDR + (size_t)cap * stride);
}

__device__ __forceinline__ const uint32_t *peer_plane_next(const BandPeer &q, int64_t t) {
    return (t & 1) ? q.plane0 : q.plane1;
}

__device__ __forceinline__ bool own_row(const BandParams &bp, int y) { return y >= bp.y0 && y < bp.y1; }

// ------------------------------------------------------------------- X1 / X4a halo
// kind 0 (X1): R' = plane_next(t) and O rows, 3 each side; kind 1 (X4a): R'' (plane_next(t))
// 2 rows each side, O'' 1 row each side.  Rows are copied word for word (global rows).
__global__ void k_band_newborns(DevParams p, BandParams bp);
__global__ void k_band_halo(DevParams p, BandParams bp, int kind) {
    const int64_t t = p.t[0];
    const int nr = kind == 0 ? 3 : 2, no = kind == 0 ? 3 : 1;
    uint32_t *R = plane_next(p, t);
    const int WW = p.WW;
    // item: (side, plane, row k, word) flattened
    const int per_side = (nr + no) * WW;
    for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < 2 * per_side; it += gridDim.x * blockDim.x) {
        const int side = it / per_side;  // 0: up neighbour, 1: down neighbour
        int r = it - side * per_side;
        const bool is_r = r < nr * WW;
        if (!is_r) r -= nr * WW;
        const int k = r / WW, wx = r - k * WW;
        const BandPeer &q = side == 0 ? bp.up : bp.down;
        if (!q.plane0) continue;  // no neighbour on this side
        const int y = side == 0 ? bp.y0 - (is_r ? nr : no) + k : bp.y1 + k;
        if (y < 0 || y >= p.H) continue;
        const size_t off = (size_t)y * WW + wx;
        if (is_r) R[off] = peer_plane_next(q, t)[off];
        else p.occ[off] = q.occ[off];
    }
}

// ------------------------------------------------------------ X2 / X4b claim merges
// kind 0 (X2): move claims; kind 1 (X4b): birth-claim keys and the claimed-cell bits of
// step t.  Rows {y0-1, y0} with the up neighbour, {y1-1, y1} with the down neighbour.
__global__ void k_band_merge(DevParams p, BandParams bp, int kind) {
    const int64_t t = p.t[0];
    const int W = p.W;
    for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < 4 * W; it += gridDim.x * blockDim.x) {
        const int side = it / (2 * W);
        const int r = it - side * 2 * W;
        const int k = r / W, x = r - k * W;
        const BandPeer &q = side == 0 ? bp.up : bp.down;
        if (!q.plane0) continue;
        const int y = side == 0 ? bp.y0 - 1 + k : bp.y1 - 1 + k;
        if (y < 0 || y >= p.H) continue;
        const size_t c = (size_t)y * W + x;
        if (kind == 0) {
            const unsigned long long v = q.claim[c];
            if (v) atomicMax(p.claim + c, v);
        } else {
            const unsigned long long v = q.bkey[c];
            if (v) atomicMax(p.bkey + c, v);
        }
    }
    if (kind == 1) {  // claimed-cell bits of parity t, the same rows, word by word
        const int WW = p.WW;
        const uint32_t *mine = bbits_of(p, t, 0);
        for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < 4 * WW; it += gridDim.x * blockDim.x) {
            const int side = it / (2 * WW);
            const int r = it - side * 2 * WW;
            const int k = r / WW, wx = r - k * WW;
            const BandPeer &q = side == 0 ? bp.up : bp.down;
            if (!q.plane0) continue;
            const int y = side == 0 ? bp.y0 - 1 + k : bp.y1 - 1 + k;
            if (y < 0 || y >= p.H) continue;
            const size_t off = (size_t)y * WW + wx;
            const uint32_t v = q.bbits[(size_t)(t & 1) * plane_words(p) + off];
            if (v) {
                const uint32_t old = atomicOr(const_cast<uint32_t *>(mine) + off, v);
                const int fresh = __popc(v & ~old);  // cells claimed only from the neighbour's side
                if (fresh && own_row(bp, y))
                    atomicAdd(reinterpret_cast<unsigned long long *>(bp.counts + (t & 1) * 4), (unsigned long long)fresh);
            }
        }
    }
}

// ---------------------------------------------------------------------- P3 move
// R14 exactly as move_phase: an agent moves iff it holds the max key on its target.  A
// mover whose target row belongs to a neighbour leaves: its state goes to the outbox (the
// weights follow in k_band_pack), its slot and occupancy bit are freed.  Everyone else is
// listed for P5.
__global__ void k_band_move(DevParams p, BandParams bp) {
    const int64_t t = p.t[0];
    const int n_list = *count_of(p, t, 0);
    const int ms = mig_stride(p.Hd, p.Pd);
    const int lane = threadIdx.x & 31;
    for (int base = blockIdx.x * blockDim.x + threadIdx.x - lane; base < n_list; base += gridDim.x * blockDim.x) {
        const int i = base + lane;
        bool stay = false;
        int slot = 0;
        if (i < n_list) {
            const int4 mr = p.mrec[i];
            slot = mr.x;
            int cellv = mr.y;
            const int tg = mr.z;
            const unsigned long long key =
                ((unsigned long long)(uint32_t)mr.w << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)cellv);
            stay = true;
            if (tg == WALL_TARGET) {  // walked into a lethal wall: dies before eating
                stay = false;
                uint32_t ob;
                p.alive[slot] = 0;
                p.ate[slot] = 0;
                greed_update(p, slot, t, false);
                atomicAnd(word_ptr(p.occ, p, cellv, ob), ~ob);
                atomicAnd(p.alive_bits + (slot >> 5), ~(1u << (slot & 31)));
                sim_step_record *rec = record_of(p, t, 0);
                atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deaths_wall), 1ull);
#if ECO_METRICS & 1
                atomicAdd(reinterpret_cast<unsigned long long *>(&rec->death_age_sum), (unsigned long long)(p.age[slot] + 1));
#endif
            } else if (tg >= 0 && p.claim[tg] == key) {
                uint32_t ob;
                atomicAnd(word_ptr(p.occ, p, cellv, ob), ~ob);
                const int ty = row_of(p, tg);
                if (own_row(bp, ty)) {
                    atomicOr(word_ptr(p.occ, p, tg, ob), ob);
                    p.cell[slot] = tg;
                } else {  // leaves for the neighbour band
                    stay = false;
                    const int dir = ty < bp.y0 ? 0 : 1;
                    int32_t *box = box_dir(bp.mig_out, dir, bp.cap, ms);
                    const int k = atomicAdd(box, 1);
                    ECO_CHECK(k < bp.cap);
                    int32_t *rec = box + BOX_HDR + (size_t)k * ms;
                    rec[0] = tg;
                    rec[1] = p.energy[slot];
                    rec[2] = p.age[slot];
                    rec[3] = p.repr[slot];
                    rec[4] = p.last_action[slot];
                    rec[5] = p.ate[slot];
                    rec[6] = p.mv_cell[slot];
                    rec[7] = p.mv_inv[slot];
                    rec[8] = slot;
                    rec[9] = p.gr_T[slot];
                    rec[10] = p.gr_C[slot];
                    rec[11] = p.gr_seen[slot] | (p.gr_ate[slot] << 1);
                    rec[12] = p.low[slot];
                    p.alive[slot] = 0;
                    atomicAnd(p.alive_bits + (slot >> 5), ~(1u << (slot & 31)));
                }
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, stay);
        int q0 = 0;
        if (lane == 0 && m) q0 = atomicAdd(bp.n_plist, __popc(m));
        q0 = __shfl_sync(0xffffffffu, q0, 0);
        ECO_CHECK(!stay || (q0 + __popc(m & ((1u << lane) - 1u)) < p.S && slot < p.S));
        if (stay) bp.plist[q0 + __popc(m & ((1u << lane) - 1u))] = slot;
    }
}

// the departing agents' float state and weights into their outbox records: every thread
// of the grid copies 16-B vectors of any record (a record is ~17 KB at Hd = 32; one warp per
// record left each warp a chain of dependent 512-B copies: measured 117 us per step)
__device__ __forceinline__ void copy_agent_vecs(const DevParams &p, size_t q, const float *logits, const float *h,
                                                const float *c, const float *w, float *lo, float *ho, float *co,
                                                float *wo) {
    // vector q of an agent's float state: [0, 2) logits, then h, c (Hd/4 each), then Pd/4 weights
    const int nh = p.Hd >> 2;
    if (q < 2) {
        reinterpret_cast<float4 *>(lo)[q] = reinterpret_cast<const float4 *>(logits)[q];
    } else if (q < 2 + (size_t)nh) {
        reinterpret_cast<float4 *>(ho)[q - 2] = reinterpret_cast<const float4 *>(h)[q - 2];
    } else if (q < 2 + 2 * (size_t)nh) {
        reinterpret_cast<float4 *>(co)[q - 2 - nh] = reinterpret_cast<const float4 *>(c)[q - 2 - nh];
    } else {
        const size_t k = q - 2 - 2 * nh;
        reinterpret_cast<float4 *>(wo)[k] = reinterpret_cast<const float4 *>(w)[k];
    }
}

__global__ void k_band_pack(DevParams p, BandParams bp) {
    const int ms = mig_stride(p.Hd, p.Pd);
    const size_t per = 2 + 2 * (size_t)(p.Hd >> 2) + (size_t)(p.Pd >> 2);  // vectors per agent
    const int n0 = *box_dir(bp.mig_out, 0, bp.cap, ms), n1 = *box_dir(bp.mig_out, 1, bp.cap, ms);
    const size_t n = (size_t)(n0 + n1) * per;
    for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(v / per);
        const size_t q = v - (size_t)k * per;
        int32_t *rec = k < n0 ? box_dir(bp.mig_out, 0, bp.cap, ms) + BOX_HDR + (size_t)k * ms
                              : box_dir(bp.mig_out, 1, bp.cap, ms) + BOX_HDR + (size_t)(k - n0) * ms;
        const int slot = rec[8];
        float *f = reinterpret_cast<float *>(rec);
        copy_agent_vecs(p, q, p.logits + (size_t)slot * LOGIT_STRIDE, p.h + (size_t)slot * p.Hd,
                        p.c + (size_t)slot * p.Hd, p.weights + (size_t)slot * p.Pd, f + 16, f + MIG_HDR,
                        f + MIG_HDR + p.Hd, f + MIG_HDR + 2 * p.Hd);
    }
}

// ------------------------------------------------------------------- X3 arrivals
// One block: the neighbours' migrants towards this band take the first free local slots in
// ascending order (alive bitmap scan); slots, alive flags and the P5 list are written here,
// the records are copied by k_band_arrive_copy.
#ifndef ECO_BAND_NT
#define ECO_BAND_NT 1024  // threads of the one-block band kernels (arrivals, rank)
#endif
constexpr int BAND_NT = ECO_BAND_NT;
__global__ void __launch_bounds__(BAND_NT) k_band_arrive(DevParams p, BandParams bp) {
    __shared__ uint32_t scratch[2 * (BAND_NT / 32 + 1)];
    const int ms = mig_stride(p.Hd, p.Pd);
    const int n_up = bp.up.plane0 ? *box_dir(bp.up.mig, 1, bp.cap, ms) : 0;
    const int n_dn = bp.down.plane0 ? *box_dir(bp.down.mig, 0, bp.cap, ms) : 0;
    const int n = n_up + n_dn;
    if (threadIdx.x == 0) bp.flags[1] = n;
    if (n == 0) return;
    const int n_pl = *bp.n_plist;
    uint32_t run = 0u;
    for (int j0 = 0; j0 < p.SW && run < (uint32_t)n; j0 += BAND_NT) {
        const int j = j0 + threadIdx.x;
        uint32_t fr = 0u;
        if (j < p.SW) {
            const int nbits = p.S - j * 32;
            const uint32_t valid = nbits >= 32 ? 0xffffffffu : ((1u << nbits) - 1u);
            fr = ~p.alive_bits[j] & valid;
        }
        uint32_t tot;
        uint32_t r = run + block_exclusive_scan<BAND_NT>((uint32_t)__popc(fr), scratch, tot);
        uint32_t take = 0u;
        while (fr && r < (uint32_t)n) {
            const int b = __ffs(fr) - 1;
            fr &= fr - 1u;
            const int slot = j * 32 + b;
            bp.arr_slot[r] = slot;
            bp.plist[n_pl + r] = slot;
            p.alive[slot] = 1;
            take |= 1u << b;
            ++r;
        }
        if (take) p.alive_bits[j] |= take;  // one thread per word
        run += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int got = run < (uint32_t)n ? (int)run : n;
        if (got < n) atomicOr(bp.flags, 1);  // local slot pool exhausted (band_slots < slots)
        *bp.n_plist = n_pl + got;
        bp.flags[1] = got;
    }
}

__global__ void k_band_arrive_copy(DevParams p, BandParams bp) {
    const int ms = mig_stride(p.Hd, p.Pd);
    const int n_up = bp.up.plane0 ? *box_dir(bp.up.mig, 1, bp.cap, ms) : 0;
    const int got = bp.flags[1];
    const size_t per = 2 + 2 * (size_t)(p.Hd >> 2) + (size_t)(p.Pd >> 2);
    auto rec_of = [&](int k) {
        return k < n_up ? box_dir(bp.up.mig, 1, bp.cap, ms) + BOX_HDR + (size_t)k * ms
                        : box_dir(bp.down.mig, 0, bp.cap, ms) + BOX_HDR + (size_t)(k - n_up) * ms;
    };
    const size_t gtid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, gthr = (size_t)gridDim.x * blockDim.x;
    for (size_t k = gtid; k < (size_t)got; k += gthr) {  // scalar state and occupancy
        const int32_t *rec = rec_of((int)k);
        const int slot = bp.arr_slot[k];
        ECO_CHECK(slot >= 0 && slot < p.S && (int)k < 2 * bp.cap);
        const int cell = rec[0];
        p.cell[slot] = cell;
        p.energy[slot] = rec[1];
        p.age[slot] = rec[2];
        p.repr[slot] = rec[3];
        p.last_action[slot] = (uint8_t)rec[4];
        p.ate[slot] = (uint8_t)rec[5];
        p.mv_cell[slot] = rec[6];
        p.mv_inv[slot] = rec[7];
        p.gr_T[slot] = rec[9];
        p.gr_C[slot] = rec[10];
        p.gr_seen[slot] = (uint8_t)(rec[11] & 1);
        p.gr_ate[slot] = (uint8_t)(rec[11] >> 1);
        p.low[slot] = rec[12];
        uint32_t ob;
        atomicOr(word_ptr(p.occ, p, cell, ob), ob);
    }
    for (size_t v = gtid; v < (size_t)got * per; v += gthr) {  // logits, h, c, weights
        const int k = (int)(v / per);
        const size_t q = v - (size_t)k * per;
        const float *f = reinterpret_cast<const float *>(rec_of(k));
        const int slot = bp.arr_slot[k];
        copy_agent_vecs(p, q, f + 16, f + MIG_HDR, f + MIG_HDR + p.Hd, f + MIG_HDR + 2 * p.Hd,
                        p.logits + (size_t)slot * LOGIT_STRIDE, p.h + (size_t)slot * p.Hd, p.c + (size_t)slot * p.Hd,
                        p.weights + (size_t)slot * p.Pd);
    }
}

// ------------------------------------------------------- P5 consume, physiology, death
// move_phase's arithmetic after the move (R16-R19) for the listed agents:
// eat the resource under the final cell, e += gain*ate - decay, age += 1, repr, death by
// energy (precedence) or age; survivors into the step-(t+1) list, eligible parents into the
// candidate list; the step's counters.
__global__ void k_band_live(DevParams p, BandParams bp) {
    const int64_t t = p.t[0];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *bp.n_hcand = 0;                      // (P7 lists this step's)
        bp.counts[(t & 1) * 4] = 0;           // own-row claimed cells, counted by P7 and X4b
    }
    const int n = *bp.n_plist;
    const int lane = threadIdx.x & 31;
    uint32_t *Rn = plane_next(p, t);
    sim_step_record *rec = record_of(p, t, 0);
    for (int base = blockIdx.x * blockDim.x + threadIdx.x - lane; base < n; base += gridDim.x * blockDim.x) {
        const int i = base + lane;
        bool ate = false, died_e = false, died_a = false, survive = false, cand = false;
        int slot = 0, cellv = 0, dage = 0;
        if (i < n) {
            slot = bp.plist[i];
            ECO_CHECK(slot >= 0 && slot < p.S && i < p.S);
            cellv = p.cell[slot];
            uint32_t bit;
            uint32_t *rw = word_ptr(Rn, p, cellv, bit);
            if (ld_plain(rw) & bit) {
                atomicAnd(rw, ~bit);
                ate = true;
            }
            p.ate[slot] = ate ? 1 : 0;
            greed_update(p, slot, t, ate);
            long long e = (long long)p.energy[slot] + (ate ? (long long)p.e_gain : 0ll) - (long long)p.e_decay;
            if (p.e_max != 0x7fffffff && e > p.e_max) e = p.e_max;
            const int en = (int)e, ag = p.age[slot] + 1;
            p.energy[slot] = en;
            p.age[slot] = ag;
            const int rp = en > p.e_repr_gt ? p.repr[slot] + 1 : 0;
            p.repr[slot] = rp;
            if (starves(p, slot, en)) died_e = true;
            else if (ag > p.max_age) died_a = true;
            if (died_e || died_a) {
                p.alive[slot] = 0;
                atomicAnd(word_ptr(p.occ, p, cellv, bit), ~bit);
                atomicAnd(p.alive_bits + (slot >> 5), ~(1u << (slot & 31)));
#if ECO_METRICS & 1
                dage = ag;
#endif
            } else {
                survive = true;
                cand = rp >= p.repr_steps;
            }
        }
        const unsigned me = __ballot_sync(0xffffffffu, ate), md = __ballot_sync(0xffffffffu, died_e),
                       ma = __ballot_sync(0xffffffffu, died_a), m = __ballot_sync(0xffffffffu, survive),
                       mc = __ballot_sync(0xffffffffu, cand);
        const int dsum = __reduce_add_sync(0xffffffffu, dage);
        int pos0 = 0, c0 = 0;
        if (lane == 0) {
            if (mc) c0 = atomicAdd(p.n_cand, __popc(mc));
            if (m) pos0 = atomicAdd(count_of(p, t + 1, 0), __popc(m));
            if (me) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->eaten), (unsigned long long)__popc(me));
            if (md) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deaths_energy), (unsigned long long)__popc(md));
            if (ma) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deaths_age), (unsigned long long)__popc(ma));
            if (dsum) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->death_age_sum), (unsigned long long)dsum);
        }
        c0 = __shfl_sync(0xffffffffu, c0, 0);
        pos0 = __shfl_sync(0xffffffffu, pos0, 0);
        if (cand) p.cand[c0 + __popc(mc & ((1u << lane) - 1u))] = make_int2(slot, cellv);
        if (survive) {
            const int q = pos0 + __popc(m & ((1u << lane) - 1u));
            list_of(p, t + 1, 0)[q] = slot;
            list_cell_of(p, t + 1, 0)[q] = cellv;
        }
    }
}

// --------------------------------------------------------------------- P7 claims
// Lazy reset of this step's move claims (the own claimants' targets and the four merged
// boundary rows), the outbox counters of this step (the neighbours pulled them before
// barrier X4a) and the P5 list, then the birth claims of the own eligible parents (birth_target: first free
// Philox-rotated neighbour in O'' / R'', halo rows included; R21).  Each candidate's target
// and claim key are kept for P10.
__global__ void k_band_claims(DevParams p, BandParams bp) {
    const int64_t t = p.t[0];
    const size_t gtid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, gthr = (size_t)gridDim.x * blockDim.x;
    const int n_list = *count_of(p, t, 0);
    for (size_t k = gtid; k < (size_t)n_list; k += gthr) {
        const int tg = p.mrec[k].z;
        if (tg >= 0) p.claim[tg] = 0ull;
    }
    for (size_t k = gtid; k < (size_t)4 * p.W; k += gthr) {
        const int side = (int)(k / (2 * p.W)), r = (int)(k - (size_t)side * 2 * p.W);
        const int y = (side == 0 ? bp.y0 - 1 : bp.y1 - 1) + r / p.W;
        if (y >= 0 && y < p.H) p.claim[(size_t)y * p.W + r % p.W] = 0ull;
    }
    if (gtid == 0) {
        const int ms = mig_stride(p.Hd, p.Pd), ns = nb_stride(p.Pd);
        *box_dir(bp.mig_out, 0, bp.cap, ms) = 0;
        *box_dir(bp.mig_out, 1, bp.cap, ms) = 0;
        *box_dir(bp.nb_out, 0, bp.cap, ns) = 0;
        *box_dir(bp.nb_out, 1, bp.cap, ns) = 0;
        *bp.n_plist = 0;  // (P5 consumed the list)
    }
    const int nc = *p.n_cand;
    const unsigned lane = threadIdx.x & 31;
    for (size_t base = gtid - lane; base < (size_t)nc; base += gthr) {
        const size_t r = base + lane;
        int no_cell = 0, is_cand = 0, new_own = 0;
        if (r < (size_t)nc) {
            const int2 sc = p.cand[r];
            unsigned long long key;
            const int c = birth_target(p, t, sc.y, key);
            if (c < 0) {
                no_cell = 1;
            } else {
                uint32_t bit;
                const uint32_t old = atomicOr(word_ptr(bbits_of(p, t, 0), p, c, bit), bit);
                atomicMax(p.bkey + c, key);
                p.bslot[sc.y] = sc.x;
                const bool own = own_row(bp, row_of(p, c));
                if (own && !(old & bit)) new_own = 1;  // a distinct claimed cell of the own rows
                if (!own) {  // a cell of a neighbour's row: P10 decides it here too
                    const int k = atomicAdd(bp.n_hcand, 1);
                    ECO_CHECK(k < 2 * bp.cap);
                    bp.hcand[k] = make_int4(sc.x, sc.y, c, (int)(uint32_t)(key >> 32));
                }
                is_cand = 1;
            }
        }
        const int a = __reduce_add_sync(0xffffffffu, no_cell), b = __reduce_add_sync(0xffffffffu, is_cand),
                  n_own = __reduce_add_sync(0xffffffffu, new_own);
        if (lane == 0) {
            sim_step_record *rec = record_of(p, t, 0);
            if (a) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deferred_no_cell), (unsigned long long)a);
            if (b) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->deferred_claim), (unsigned long long)b);
            if (n_own) atomicAdd(reinterpret_cast<unsigned long long *>(bp.counts + (t & 1) * 4), (unsigned long long)n_own);
        }
    }
}

// ----------------------------------------------------------------- P10 rank, place
// Global capacity (R22): claimed cells ranked row-major over the whole grid = band order
// then the band's row-major order; the first S - A_total (A_total = all survivors) are
// placed.  This band's claimed cells have global ranks C_lt + r (C_lt: claimed cells of the
// bands above), so its first n_place = clamp(S - A_total - C_lt, 0, c_own) are placed, in
// its first n_place free local slots.  A child whose winning parent stands in a neighbour's
// row gets its weights in X5 (cslot[cell] = its slot).  A local parent whose child's cell
// lies in a neighbour's boundary row computes that cell's global rank from the merged
// claimed-cell bits of the row and the counts, resets its repr when the child is placed and
// queues the child's weights for the neighbour.
__device__ __forceinline__ int row_popc_range(const uint32_t *row, int x0, int x1) {  // bits [x0, x1) of a row
    int n = 0;
    for (int x = x0; x < x1;) {
        const int wx = x >> 5, b = x & 31;
        const int hi = (x1 - (wx << 5)) < 32 ? (x1 - (wx << 5)) : 32;
        uint32_t m = row[wx] >> b;
        if (hi - b < 32) m &= (1u << (hi - b)) - 1u;
        n += __popc(m);
        x = (wx << 5) + hi;
    }
    return n;
}

constexpr int BAND_ROW_WORDS = 2048;  // boundary-row prefix counts kept in shared memory (W <= 65,536)
__global__ void __launch_bounds__(BAND_NT) k_band_rank(DevParams p, BandParams bp) {
    __shared__ uint32_t scratch[2 * (BAND_NT / 32 + 1)];
    __shared__ int s_free[RANK_SMEM_CAP], s_bcell[RANK_SMEM_CAP];
    __shared__ uint16_t s_pre[2][BAND_ROW_WORDS];  // exclusive prefix popcounts of rows y0-1 and y1
    __shared__ long long s_clt, s_atot;
    const int64_t t = p.t[0];
    const int par_t = (int)(t & 1);
    if (threadIdx.x == 0) {
        long long clt = 0, at = 0;
        for (int b = 0; b < bp.G; ++b) {
            const int64_t *cnt = bp.all_counts[b] + par_t * 4;
            const long long c = *reinterpret_cast<const volatile long long *>(cnt);
            const long long a = *reinterpret_cast<const volatile long long *>(cnt + 1);
            if (b < bp.b) clt += c;
            at += a;
        }
        s_clt = clt;
        s_atot = at;
    }
    __syncthreads();
    const long long clt = s_clt, cap = (long long)bp.S_global - s_atot;
    const int c_own = (int)bp.counts[par_t * 4];
    const int n_surv = *count_of(p, t + 1, 0);
    long long np = cap - clt;
    if (np < 0) np = 0;
    if (np > c_own) np = c_own;
    int n_place = (int)np;
    if (n_place > p.S - n_surv) {  // local slot pool exhausted (band_slots < slots)
        if (threadIdx.x == 0) atomicOr(bp.flags, 1);
        n_place = p.S - n_surv;
    }
    int32_t *g_free = p.free_list, *g_bcell = p.birth_cell;
    if (n_place > 0)
        rank_lists<BAND_NT>(p, 0, t, n_place, scratch, s_free, s_bcell, g_free, g_bcell, (size_t)bp.y0 * p.WW,
                                 (size_t)bp.y1 * p.WW);
    const int ns = nb_stride(p.Pd);
    for (int r = threadIdx.x; r < n_place; r += BAND_NT) {
        const int c = r < RANK_SMEM_CAP ? s_bcell[r] : g_bcell[r];
        const int child = r < RANK_SMEM_CAP ? s_free[r] : g_free[r];
        const unsigned long long k = p.bkey[c];
        const int q = (int)(0xFFFFFFFFu - (uint32_t)k);  // the winning parent's cell
        const int par = own_row(bp, row_of(p, q)) ? p.bslot[q] : -1;
        ECO_CHECK(child >= 0 && child < p.S && par < p.S && n_surv + r < p.S);
        p.alive[child] = 1;
        atomicOr(p.alive_bits + (child >> 5), 1u << (child & 31));
        p.cell[child] = c;
        p.energy[child] = p.e_init;
        p.age[child] = 0;
        p.repr[child] = 0;
        p.last_action[child] = 0;
        p.ate[child] = 0;
        p.gr_seen[child] = 0;
        p.gr_ate[child] = 0;
        p.gr_T[child] = 0;
        p.gr_C[child] = 0;
        p.low[child] = 0;
        for (int j = 0; j < p.Hd; ++j) {
            p.h[(size_t)child * p.Hd + j] = 0.f;
            p.c[(size_t)child * p.Hd + j] = 0.f;
        }
        for (int a = 0; a < LOGIT_STRIDE; ++a) p.logits[(size_t)child * LOGIT_STRIDE + a] = 0.f;
        uint32_t bit;
        atomicOr(word_ptr(p.occ, p, c, bit), bit);
        if (par >= 0) p.repr[par] = 0;
        else bp.cslot[c] = child;
        list_of(p, t + 1, 0)[n_surv + r] = child;
        list_cell_of(p, t + 1, 0)[n_surv + r] = c;
        p.birth_child[r] = child;
        p.birth_parent[r] = par;
        p.birth_cell[r] = c;
    }
    // local parents of children in a neighbour's boundary row (listed by the claims); the
    // claimed cells of those two rows ranked with prefix popcounts (one block scan per row)
    const int nc = *bp.n_hcand;
    const uint32_t *bb = bbits_of(p, t, 0);
    const bool pre_ok = p.WW <= BAND_ROW_WORDS;
    if (nc > 0 && pre_ok) {  // (block-uniform)
        for (int side = 0; side < 2; ++side) {
            const int y = side == 0 ? bp.y0 - 1 : bp.y1;
            const bool ex = y >= 0 && y < p.H;
            uint32_t run = 0u;
            for (int w0 = 0; w0 < p.WW; w0 += BAND_NT) {
                const int wx = w0 + (int)threadIdx.x;
                const uint32_t v = (ex && wx < p.WW) ? (uint32_t)__popc(bb[(size_t)y * p.WW + wx]) : 0u;
                uint32_t tot;
                const uint32_t e = run + block_exclusive_scan<BAND_NT>(v, scratch, tot);
                if (wx < p.WW) s_pre[side][wx] = (uint16_t)e;
                run += tot;
                __syncthreads();
            }
        }
        __syncthreads();
    }
    for (int k = threadIdx.x; k < nc; k += BAND_NT) {
        const int4 hc = bp.hcand[k];
        const int2 tg = make_int2(hc.z, hc.w), sc = make_int2(hc.x, hc.y);
        const int ty = row_of(p, tg.x);
        const unsigned long long key =
            ((unsigned long long)(uint32_t)tg.y << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)sc.y);
        if (p.bkey[tg.x] != key) continue;  // lost the claim
        const int tx = tg.x - ty * p.W;
        const uint32_t *row = bb + (size_t)ty * p.WW;
        long long g;
        int dir;
        // claimed cells of the row before tx (prefix of whole words + the partial word)
        const int wx = tx >> 5;
        const int before = pre_ok ? (int)s_pre[ty < bp.y0 ? 0 : 1][wx] + __popc(row[wx] & ((1u << (tx & 31)) - 1u))
                                  : row_popc_range(row, 0, tx);
        if (ty < bp.y0) {  // the up neighbour's last row: its claimed cells at x' >= tx rank after it
            const int total = pre_ok ? (int)s_pre[0][p.WW - 1] + __popc(row[p.WW - 1]) : row_popc_range(row, 0, p.W);
            g = clt - (total - before);
            dir = 0;
        } else {  // the down neighbour's first row
            g = clt + c_own + before;
            dir = 1;
        }
        if (g < cap) {
            p.repr[sc.x] = 0;
            int32_t *box = box_dir(bp.nb_out, dir, bp.cap, ns);
            const int kk = atomicAdd(box, 1);
            ECO_CHECK(kk < bp.cap);
            int32_t *rec = box + BOX_HDR + (size_t)kk * ns;
            rec[0] = tg.x;
            rec[1] = sc.x;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // the step's record (rank_finalize's arithmetic with the band's own counts)
        volatile sim_step_record *rec = record_of(p, t, 0);
        const int64_t grown = rec->grown, eaten = rec->eaten, dc = rec->deferred_claim;
        const int64_t res = p.res_count[0] + grown - eaten;
        p.res_count[0] = res;
        rec->t = t;
        rec->agents_at_start = *count_of(p, t, 0);
        rec->births = n_place;
        rec->deferred_claim = dc - c_own;
        rec->deferred_capacity = c_own - n_place;
        rec->population = n_surv + n_place;
        rec->resources = res;
        life_window_add(p, 0, t, rec->deaths_energy + rec->deaths_age + rec->deaths_wall, rec->death_age_sum);
        *count_of(p, t + 1, 0) = n_surv + n_place;
        p.n_births[0] = n_place;
        *p.p_children = n_place;  // split policy: the children (list end) start from their bias
        unsigned long long *tot = p.totals;
        atomicAdd(tot + 0, 1ull);
        atomicAdd(tot + 1, (unsigned long long)rec->agents_at_start);
        atomicAdd(tot + 2, (unsigned long long)((size_t)(bp.y1 - bp.y0) * p.W));
        atomicAdd(tot + 3, (unsigned long long)n_place);
        atomicAdd(tot + 4, (unsigned long long)(rec->deaths_energy + rec->deaths_age + rec->deaths_wall));
        atomicAdd(tot + 5, (unsigned long long)eaten);
        atomicAdd(tot + 6, (unsigned long long)grown);
        p.t[0] = t + 1;
    }
}

// --------------------------------------------------------------------- P11 mutate
// The children of local parents (birth lists; parent -1 = foreign, weights come in X5) and
// the outgoing newborns of both directions, one Box-Muller pair per item as mutate_world
// (MUTATE keyed by (birth step, child cell), R23, R29).
__global__ void k_band_mutate(DevParams p, BandParams bp) {
    const int64_t T = p.t[0] - 1;  // the rank advanced t
    const int ns = nb_stride(p.Pd);
    const int nl = p.n_births[0];
    int32_t *box0 = box_dir(bp.nb_out, 0, bp.cap, ns), *box1 = box_dir(bp.nb_out, 1, bp.cap, ns);
    const int n0 = *box0, n1 = *box1;
    const int nb = nl + n0 + n1;
    const uint32_t Q = (uint32_t)mutate_items_per_child(p);
    const uint64_t seed = p.seeds[0];
    const size_t n = (size_t)nb * Q;
    for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) {
        const int b = (int)(k / Q), it = (int)(k - (size_t)b * Q);
        int parent, cellc;
        float *dstw;
        if (b < nl) {
            parent = p.birth_parent[b];
            if (parent < 0) continue;
            cellc = p.birth_cell[b];
            dstw = p.weights + (size_t)p.birth_child[b] * p.Pd;
        } else {
            const int kk = b - nl;
            int32_t *rec = kk < n0 ? box0 + BOX_HDR + (size_t)kk * ns : box1 + BOX_HDR + (size_t)(kk - n0) * ns;
            cellc = rec[0];
            parent = rec[1];
            dstw = reinterpret_cast<float *>(rec + NB_HDR);
        }
        int d0, dstep, j0;
        mutate_item(p, it, d0, dstep, j0);
        const float *wp = p.weights + (size_t)parent * p.Pd + d0;
        const float pa = wp[0], pb = dstep ? wp[dstep] : 0.f;
        double za, zb;
        gauss_pair(seed, T, cellc, j0, za, zb);
        dstw[d0] = __fadd_rn(pa, __double2float_rn(__dmul_rn(p.mutation_std, za)));
        if (dstep) dstw[d0 + dstep] = __fadd_rn(pb, __double2float_rn(__dmul_rn(p.mutation_std, zb)));
    }
}

// ----------------------------------------------------------------------- X5 newborns
__global__ void k_band_newborns(DevParams p, BandParams bp) {
    const int ns = nb_stride(p.Pd);
    const int n_up = bp.up.plane0 ? *box_dir(bp.up.nb, 1, bp.cap, ns) : 0;
    const int n_dn = bp.down.plane0 ? *box_dir(bp.down.nb, 0, bp.cap, ns) : 0;
    const size_t per = (size_t)(p.Pd >> 2);
    for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < (size_t)(n_up + n_dn) * per;
         v += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(v / per);
        const size_t q = v - (size_t)k * per;
        const int32_t *rec = k < n_up ? box_dir(bp.up.nb, 1, bp.cap, ns) + BOX_HDR + (size_t)k * ns
                                      : box_dir(bp.down.nb, 0, bp.cap, ns) + BOX_HDR + (size_t)(k - n_up) * ns;
        const int child = bp.cslot[rec[0]];
        ECO_CHECK(child >= 0 && child < p.S);
        reinterpret_cast<float4 *>(p.weights + (size_t)child * p.Pd)[q] = reinterpret_cast<const float4 *>(rec + NB_HDR)[q];
    }
}

// ------------------------------------------------------------------ initialisation
// C.2 for one band: the global placement keys were sorted (launch_init_agents' sort); the
// initial agents whose cells lie in the own rows take local slots 0.. in the global slot
// order.  One block; *n_own receives their number.
__global__ void __launch_bounds__(BAND_NT) k_band_init_agents(DevParams p, BandParams bp, int n_initial,
                                                              const unsigned long long *sorted, int32_t *n_own) {
    __shared__ uint32_t scratch[2 * (BAND_NT / 32 + 1)];
    for (int i = threadIdx.x; i < p.S; i += BAND_NT) {
        p.alive[i] = 0;
        p.cell[i] = 0;
        p.energy[i] = 0;
        p.age[i] = 0;
        p.repr[i] = 0;
        p.last_action[i] = 0;
        p.ate[i] = 0;
        p.gr_seen[i] = p.gr_ate[i] = 0;
        p.gr_T[i] = p.gr_C[i] = 0;
        p.low[i] = 0;
    }
    __syncthreads();
    uint32_t run = 0u;
    for (int i0 = 0; i0 < n_initial; i0 += BAND_NT) {
        const int i = i0 + threadIdx.x;
        int cell = 0;
        uint32_t own = 0u;
        if (i < n_initial) {
            cell = (int)(uint32_t)(sorted[i] & 0xffffffffull);
            own = own_row(bp, row_of(p, cell)) ? 1u : 0u;
        }
        uint32_t tot;
        const uint32_t r = run + block_exclusive_scan<BAND_NT>(own, scratch, tot);
        if (own && r < (uint32_t)p.S) {
            p.alive[r] = 1;
            p.cell[r] = cell;
            p.energy[r] = p.e_init;
        }
        run += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *n_own = (int)run;
        if (run > (uint32_t)p.S) atomicOr(bp.flags, 1);
    }
}

// after P5: the survivors (the band's count for the global cap) and, for the split policy,
// the step and the survivors' count read by the P-row kernel on the second stream while P10
// advances t and appends the children
__global__ void k_band_snap(DevParams p, BandParams bp) {
    const int64_t t = p.t[0];
    const int n = *count_of(p, t + 1, 0);
    bp.snap[0] = t + 1;
    bp.snap[1] = n;
    bp.counts[(t & 1) * 4 + 1] = n;  // survivors, read by every band for the global cap
}

// split policy, right after the policy: the step and its list's count, read by the P-row
// kernel that runs on the second stream from here to the step's end (P10 advances t meanwhile)
__global__ void k_band_snap0(DevParams p, BandParams bp) {
    const int64_t t = p.t[0];
    bp.snap[2] = t;
    bp.snap[3] = *count_of(p, t, 0);
}

// --------------------------------------------------------------------- launchers
cudaError_t band_snap(const DevParams &p, const BandParams &bp, cudaStream_t s) {
    k_band_snap<<<1, 1, 0, s>>>(p, bp);
    return cudaGetLastError();
}
cudaError_t band_snap0(const DevParams &p, const BandParams &bp, cudaStream_t s) {
    k_band_snap0<<<1, 1, 0, s>>>(p, bp);
    return cudaGetLastError();
}
cudaError_t band_halo(const DevParams &p, const BandParams &bp, int kind, cudaStream_t s) {
    k_band_halo<<<32, 256, 0, s>>>(p, bp, kind);
    return cudaGetLastError();
}
cudaError_t band_merge(const DevParams &p, const BandParams &bp, int kind, cudaStream_t s) {
    k_band_merge<<<32, 256, 0, s>>>(p, bp, kind);
    return cudaGetLastError();
}
cudaError_t band_move(const DevParams &p, const BandParams &bp, int sms, cudaStream_t s) {
    const int blocks = (p.S + 255) / 256 < sms * 4 ? (p.S + 255) / 256 : sms * 4;
    k_band_move<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(p, bp);
    k_band_pack<<<sms, 256, 0, s>>>(p, bp);
    return cudaGetLastError();
}
cudaError_t band_arrive(const DevParams &p, const BandParams &bp, int sms, cudaStream_t s) {
    k_band_arrive<<<1, BAND_NT, 0, s>>>(p, bp);
    k_band_arrive_copy<<<sms, 256, 0, s>>>(p, bp);
    return cudaGetLastError();
}
cudaError_t band_live(const DevParams &p, const BandParams &bp, int sms, cudaStream_t s) {
    const int blocks = (p.S + 255) / 256 < sms * 4 ? (p.S + 255) / 256 : sms * 4;
    k_band_live<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(p, bp);
    return cudaGetLastError();
}
cudaError_t band_claims(const DevParams &p, const BandParams &bp, int sms, cudaStream_t s) {
    k_band_claims<<<sms * 2, 256, 0, s>>>(p, bp);
    return cudaGetLastError();
}
cudaError_t band_rank(const DevParams &p, const BandParams &bp, cudaStream_t s) {
    k_band_rank<<<1, BAND_NT, 0, s>>>(p, bp);
    return cudaGetLastError();
}
cudaError_t band_mutate(const DevParams &p, const BandParams &bp, int sms, cudaStream_t s) {
    k_band_mutate<<<sms * 8, 256, 0, s>>>(p, bp);
    return cudaGetLastError();
}
cudaError_t band_newborns(const DevParams &p, const BandParams &bp, int sms, cudaStream_t s) {
    k_band_newborns<<<sms, 256, 0, s>>>(p, bp);
    return cudaGetLastError();
}
cudaError_t band_init_agents(const DevParams &p, const BandParams &bp, int n_initial, const unsigned long long *sorted,
                             int32_t *n_own, cudaStream_t s) {
    k_band_init_agents<<<1, BAND_NT, 0, s>>>(p, bp, n_initial, sorted, n_own);
    return cudaGetLastError();
}
size_t band_box_words(int W, int S, int Hd, int Pd, bool newborn) {
    const int cap = W < S ? W : S;
    const int st = newborn ? nb_stride(Pd) : mig_stride(Hd, Pd);
    return 2 * ((size_t)BOX_HDR + (size_t)cap * st);
}

}  // namespace eco
