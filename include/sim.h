/*
 * include/sim.h — C ABI of the B200 world-step library (libsim.so), version 1.
 *
 * The library runs the per-timestep world step of the non-episodic neuroevolution
 * simulator of arXiv 2302.09334 (Hamon, Nisioti, Moulin-Frier), App. B
 * (PAPER.md:248-350), under the BASELINE.json configs, entirely in hand-written
 * sm_100a CUDA kernels:
 *   (a) resource regrowth  p(x,y) = p_I(x,y)*c(x) + c
 *   (b) egocentric observation of every live agent
 *   (c) per-agent LSTM policy + linear head, argmax action
 *   (d) movement, consumption, energy/age physiology
 *   (e) death and minimal-criterion reproduction with mutation
 * Readings of silent/garbled passages (R1-R30) are listed in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *  - Every function returns sim_status; none throws or aborts.  sim_last_error()
 *    returns a thread-local message for the most recent failure on the calling thread.
 *  - Ownership: the handle owns all device memory.  Caller buffers are read or written
 *    during the call only and never retained.  `seeds` is copied at create.  The CUDA
 *    stream in sim_config is borrowed and must outlive the handle.
 *  - Any CUDA failure poisons the handle; later calls return SIM_E_STATE.
 *  - sim_step is asynchronous on the handle's stream; sim_get_* synchronise.
 *  - A non-finite LSTM value found on the device is reported as SIM_E_NONFINITE by the
 *    next synchronising call (or the next sim_step).  Extinction is not an error.
 *  - A handle is not thread-safe.  Distinct handles share nothing.
 *  - There is no CPU fallback: without a usable CUDA device sim_create fails with
 *    SIM_E_CUDA.  sim_validate / sim_param_count / sim_state_sizes are host-only.
 */
#ifndef ECO_SIM_H
#define ECO_SIM_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SIM_ABI_VERSION 1u

#if defined(__GNUC__)
#define SIM_API __attribute__((visibility("default")))
#else
#define SIM_API
#endif

typedef struct sim_ctx *sim_handle; /* opaque */

typedef enum {
    SIM_OK = 0,
    SIM_E_INVALID = -1,   /* a config field or argument is invalid; message names it   */
    SIM_E_CUDA = -2,      /* CUDA runtime failure (handle poisoned)                      */
    SIM_E_OOM = -3,       /* device allocation failed                                    */
    SIM_E_NCCL = -4,      /* an NCCL call of the banded multi-GPU mode failed            */
    SIM_E_NONFINITE = -5, /* a non-finite h', c' or logit was produced */
    SIM_E_STATE = -6      /* the handle is poisoned by an earlier failure                */
} sim_status;

/* World parameters.  Field meanings follow PAPER.md App. B.4 (lines 311-338) under the
 * BASELINE.json constants.  Energies are int32 milli-units (R16). */
typedef struct {
    uint32_t abi_version;   /* = SIM_ABI_VERSION                                       */
    uint32_t struct_size;   /* = sizeof(sim_config)                                     */
    int32_t rows, cols;     /* H (latitude axis, row 0 = top), W; W % 4 == 0             */
    int32_t n_worlds;       /* >= 1 independent worlds batched on the device             */
    int32_t device;         /* CUDA device ordinal                                       */
    const uint64_t *seeds;  /* [n_worlds] Philox keys; copied at create                  */
    double init_resource_p; /* Bernoulli rho of the initial resources                   */
    int32_t regrow_r2;      /* squared Euclidean radius of the count disc, 1..8 (4 = 12 cells) */
    int32_t f_class_min_k[4]; /* class c iff k >= f_class_min_k[c]; [0] = 0, ascending */
    double f_value[4];      /* f(class): {0, .01, .05, .1}                               */
    double lat_top, lat_bottom; /* climate lat(0), lat(H-1), linear in y/(H-1)         */
    double spontaneous;     /* constant spontaneous growth probability c                */
    int32_t slots, n_initial; /* S agent slots (population cap, <= 2^24 - 1), N0 initial agents */
    int32_t obs_radius;     /* r: window (2r+1)^2, 0..3 (network 1: 7)                    */
    int32_t hidden;         /* LSTM hidden size Hd in {4, 8, 16, 32} (network 1: 4)       */
    int32_t n_actions;      /* must be 5 (stay, N, S, E, W)                               */
    int32_t log_capacity;   /* step records kept per world (ring, rounded up to a power of 2); 0 -> 4096 */
    double init_weight_std, mutation_std; /* standard deviations (R23)                   */
    int32_t e_init, e_decay, e_gain, e_repr_gt, e_death_le, e_max; /* milli-units;
                                                e_max = INT32_MAX means no clip          */
    int32_t repr_steps, max_age;
    void *cuda_stream;      /* borrowed cudaStream_t; NULL -> library-owned stream       */
    /* Banded mode: ONE world (n_worlds = 1) split into n_bands
     * latitude bands of rows; band b owns rows [band_rows[b], band_rows[b+1]) and the agents
     * standing in them, exchanges halo rows, boundary claims, migrating agents (with their
     * weights and LSTM state) and newborns with bands b-1 and b+1, and reads every band's
     * birth counts for the global population cap.  The trajectory equals the unbanded
     * world's keyed by cell (slot layouts differ).  n_bands <= 1: unbanded (the fields below
     * are ignored).  This handle holds bands [band_first, band_first + band_local) on its
     * device: all n_bands on one GPU (exchanges are device reads between the bands), or one
     * band per GPU (one process per GPU; the other bands are attached with
     * sim_band_export / sim_band_import and the steps synchronise through NCCL,
     * sim_band_nccl_init). */
    int32_t n_bands;        /* G, 2..32 (0 or 1: unbanded)                               */
    int32_t band_first, band_local;
    const int32_t *band_rows; /* [G+1] ascending row boundaries from 0 to H, each band >= 3
                                 rows (the halo); NULL -> equal split b*H/G; copied        */
    int32_t band_slots;     /* agent slots of each band (0 -> slots: a band can then hold
                               the whole population and never overflows); a band whose
                               pool overflows poisons the handle with SIM_E_OOM           */
    /* The paper's own world (App. B.4), all off
     * (0) for BASELINE's world: */
    double climate_alpha;   /* > 0: climate c(x) = (alpha^x + 1)/(alpha + 1) at x = y/(H-1)
                                replaces the linear lat_top..lat_bottom      */
    int32_t death_steps;    /* > 0: an agent dies after this many consecutive steps with
                               energy <= e_death_le (T_death), else at once  */
    int32_t lethal_walls;   /* 1: a move off the grid kills the agent,
                               0: it is blocked (R15)                                      */
    /* The agents' network:
     *   0  an LSTM of `hidden` units on the (2r+1)^2 x 2 window + a linear head, argmax
     *      (BASELINE.json);
     *   1  the paper's CNN-LSTM: a 15x15x3 window (resources, agents,
     *      walls = off the grid), conv 3x3/2 SAME (4) -> avgpool 2/1 -> conv 3x3/2 SAME (8)
     *      -> avgpool 2/1 -> 72 ++ one-hot previous action (5) ++ ate (1) = 78 -> LSTM(4) ->
     *      [78 ++ h'] -> dense 8 tanh -> dense 5 -> softmax(50 logits), the action SAMPLED by
     *      inverse CDF with the Philox word (ACTION = 8, t, cell) (R38-R42);
     *      requires obs_radius = 7, hidden = 4 and n_bands <= 1; 2445 parameters.        */
    int32_t network;
    /* Co-location (the paper's own reproduction; R43-R47;
     * requires network 1): any number of agents per cell -- moves never conflict, the agent
     * channel counts agents, the agents on a resource cell hold a lottery (the largest
     * (CONSUME = 9 draw of the slot, -slot) key eats), the eligible parents in slot order
     * take the free slots in order and "the off-spring appears on the same cell as its
     * parent"; ACTION and MUTATE draws are keyed by slot.  0: exclusive
     * occupancy (R14, R21).                                                             */
    int32_t colocate;
} sim_config;

/* Canonical state, host buffers owned by the caller, layouts with the world index
 * outermost.  For sim_get_state a NULL field is skipped; for sim_set_state a NULL field
 * keeps the device value.  Dead slots: only `alive` is meaningful.
 *   weights: per slot P floats in canonical order W_ih[4Hd][I] (gate blocks i,f,g,o,
 *   row-major), W_hh[4Hd][Hd], b[4Hd], W_out[5][Hd], b_out[5];
 *   P = 4Hd*I + 4Hd*Hd + 4Hd + 5Hd + 5 with I = 2(2r+1)^2.
 *   network 1 (P = 2445): conv1_w[4][3][3][3] ([out][ky][kx][in]), conv1_b[4],
 *   conv2_w[8][3][3][4], conv2_b[8], W_ih[16][78], W_hh[16][4], b[16] (gates i,f,g,o),
 *   W_d[8][82], b_d[8], W_out[5][8], b_out[5]. */
typedef struct {
    int64_t t;             /* steps taken; all worlds share t                              */
    uint8_t *resources;    /* [n_worlds][H][W] 0/1                                         */
    uint8_t *alive;        /* [n_worlds][S]                                                */
    int32_t *cell;         /* [n_worlds][S] y*W + x                                        */
    int32_t *energy;       /* [n_worlds][S] milli-units                                    */
    int32_t *age;          /* [n_worlds][S]                                                */
    int32_t *repr;         /* [n_worlds][S] consecutive steps with energy > e_repr_gt      */
    uint8_t *last_action;  /* [n_worlds][S] 0 stay, 1 N, 2 S, 3 E, 4 W                     */
    uint8_t *ate;          /* [n_worlds][S]                                                */
    float *h;              /* [n_worlds][S][Hd]                                            */
    float *c;              /* [n_worlds][S][Hd]                                            */
    float *weights;        /* [n_worlds][S][P]                                             */
    float *logits;         /* [n_worlds][S][5] of the last step                            */
    int32_t *low;          /* [n_worlds][S] consecutive steps with energy <= e_death_le (the
                              death timer of death_steps > 0)                               */
} sim_state;

/* Per world, per step counters (integer, exact). */
typedef struct {
    int64_t t;                 /* step index described                                    */
    int64_t agents_at_start;   /* live agents at step start (= agent-steps of this step)  */
    int64_t grown, eaten, births;
    int64_t deaths_energy, deaths_age;
    int64_t deferred_no_cell;  /* eligible parent without an empty adjacent cell          */
    int64_t deferred_claim;    /* lost the claim on its candidate cell                    */
    int64_t deferred_capacity; /* won the cell but no free slot                           */
    int64_t population;        /* after the step                                          */
    int64_t resources;         /* after the step                                          */
    int64_t near_ties;         /* live agents with top-1 minus top-2 logit margin < 1e-4  */
    int64_t obs_nnz;           /* sum over live agents of active (= 1) observation inputs:
                                  the W_ih columns the policy kernel must read            */
    int64_t death_age_sum;     /* sum of the ages (after this step's increment) of the agents
                                  that died this step: life expectancy over a window is the
                                  windowed sum / windowed deaths (App. C; SPEC
                                  metrics.life_expectancy)                                */
    int64_t deaths_wall;       /* agents killed by a move off the grid (lethal_walls)      */
} sim_step_record;

/* Cumulative counters since create (or the last set_state), summed over worlds. */
typedef struct {
    int64_t steps;
    int64_t agent_steps;
    int64_t cell_updates;
    int64_t births, deaths, eaten, grown;
} sim_totals;

/* Sizes a caller needs to allocate sim_state buffers (elements, per world). */
typedef struct {
    int64_t cells;   /* H*W                */
    int64_t slots;   /* S                  */
    int32_t hidden;  /* Hd                 */
    int32_t inputs;  /* I                  */
    int32_t params;  /* P                  */
    int32_t n_actions;
    int64_t device_bytes; /* device memory the handle will allocate */
} sim_state_sizes_t;

/* Per-kernel timing of one instrumented step (milliseconds, CUDA events).  hh: the P rows
 * P = W_hh h + b of the next step's agents (the recurrent half of the gate
 * sum), which graph mode computes inside its cooperative kernel beside the dynamics; 0
 * when the policy is not split (several worlds, hidden != 32, sharded). */
#define SIM_NUM_KERNELS 7
typedef struct {
    float step_ms;                     /* first event to last event of the step */
    float kernel_ms[SIM_NUM_KERNELS];  /* regrow, policy, move, birth_claim, birth_rank, mutate, hh */
} sim_step_timing;

/* --- lifecycle ------------------------------------------------------------------- */
/* Validate cfg, allocate device state and initialise every world (C.2: Bernoulli
 * resources, N0 agents on the N0 smallest (draw, cell) empty cells, N(0, std^2)
 * weights).  n_initial > number of empty cells -> SIM_E_INVALID. */
SIM_API sim_status sim_create(const sim_config *cfg, sim_handle *out);
/* Enqueue n >= 0 world steps on the stream, asynchronously: CUDA graphs of [policy, k_post]
 * (an eight-step graph per eight steps for n >= 8, each later policy a programmatic
 * dependent of the k_post before it; one-step graphs for the remainder).  The graphs are
 * captured at the handle's first step and whenever a kernel parameter changes
 * (sim_set_record_mirror), never by a later sim_step.  A world without agent slots
 * (slots = 0: the regrowth grids of BASELINE configs[2]) steps with a one-block bookkeeping
 * kernel and the regrowth kernel instead (same records, no policy and no k_post launch). */
SIM_API sim_status sim_step(sim_handle h, int64_t n);
/* Synchronise, convert to the canonical layout and copy into caller buffers. */
SIM_API sim_status sim_get_state(sim_handle h, sim_state *out);
/* Replace state (resume / inject): host buffers -> device; rebuilds occupancy and lists.
 * Rejects out-of-range cells and non-exclusive occupancy (SIM_E_INVALID). */
SIM_API sim_status sim_set_state(sim_handle h, const sim_state *in);
/* NULL-safe; frees everything. */
SIM_API sim_status sim_destroy(sim_handle h);
SIM_API const char *sim_last_error(void);

/* --- host-only helpers (no device needed) ------------------------------------------ */
SIM_API sim_status sim_validate(const sim_config *cfg);
SIM_API sim_status sim_state_sizes(const sim_config *cfg, sim_state_sizes_t *out);

/* --- test and measurement hooks ------------------------------------------------------ */
/* act: [n_worlds][S], 255 = use the policy; NULL clears.  The policy still runs (h, c,
 * logits update); only the move uses the forced action.  Applies to every later step. */
SIM_API sim_status sim_set_forced_actions(sim_handle h, const uint8_t *act);
/* Test hook: out[n_worlds][S] receives, for the most recent step taken while forced
 * actions were set, each slot's OWN policy decision (network 0: the argmax; network 1:
 * the sampled action) before the forced action replaced it.  Meaningful only for slots
 * alive at that step's start.  Synchronises.  Not available on banded handles. */
SIM_API sim_status sim_get_policy_actions(sim_handle h, uint8_t *out);
/* Records of steps [first, first+n) for all worlds, out[n][n_worlds]; the steps must be
 * among the last log_capacity steps taken. */
SIM_API sim_status sim_get_step_log(sim_handle h, int64_t first, int64_t n, sim_step_record *out);
/* The same copy enqueued on the handle's stream without waiting: `out` (pinned host memory,
 * for a truly asynchronous copy) is valid after the next sim_synchronize or synchronising
 * call.  Lets a driver read every step's result without a host round trip per step. */
SIM_API sim_status sim_get_step_log_async(sim_handle h, int64_t first, int64_t n, sim_step_record *out);
/* Mirror every step's completed record into a caller-owned ring in page-locked, mapped host
 * memory (`capacity` records per world, a power of two; step t goes to entry
 * [t % capacity][world]), written by the device as the step completes: a driver reads each
 * step's result with no copy operation on the stream.  Entries are valid once a later
 * synchronising call returns.  host = NULL stops mirroring.  The buffer must outlive the
 * mirroring.  Non-mapped memory -> SIM_E_INVALID. */
SIM_API sim_status sim_set_record_mirror(sim_handle h, sim_step_record *host, int64_t capacity);
SIM_API sim_status sim_get_totals(sim_handle h, sim_totals *out);
/* Movement histograms (Appendix C, "17 bins of the distance traveled"; SPEC
 * metrics.movement_bin): windows of SIM_MOVE_WINDOW steps aligned to multiples of it from
 * step 0; window k covers steps [50k, 50k+49].  An agent counts in window k iff it is alive
 * from the start of step 50k to the end of step 50k+49 (its age grows by exactly 50: born or
 * dead within the window excludes it); its bin is min(16, floor(d / 3)) for d the Manhattan
 * distance between its cell at the start of step 50k and at the end of step 50k+49.
 * out[i][w][b] (int32, caller-owned [n][n_worlds][17]) receives window first + i.  Windows
 * must be complete (50(first+n) <= t) and among the last ceil(log_capacity / 50) windows;
 * windows that began before the last sim_set_state (with t not a multiple of 50) hold 0.
 * SIM_E_INVALID otherwise; synchronises. */
#define SIM_MOVE_WINDOW 50
#define SIM_MOVE_BINS 17
SIM_API sim_status sim_get_move_hist(sim_handle h, int64_t first, int64_t n, int32_t *out);
/* Greediness (§3.3, "Does the density of resources affect agents' greediness?"):
 * windows of SIM_GREED_WINDOW steps aligned to multiples of it from step 0; T_r counts the
 * windows in which the agent had at least one resource in its field of view (a 1 in the
 * resource channel of its observation, R10/R11) and C_r those in which it consumed at least
 * one resource; G = C_r / T_r.  A window is counted for every agent alive at the start of
 * its last step (agents born inside a window count its remainder).  T_r, C_r: caller-owned
 * int32 [n_worlds][S], slot order of sim_get_state (banded: its compaction); meaningful for
 * live slots; the counts restart at 0 at sim_set_state and for every newborn.  Sharded
 * handles: valid on the slot's owner only.  Synchronises. */
#define SIM_GREED_WINDOW 20
SIM_API sim_status sim_get_greediness(sim_handle h, int32_t *T_r, int32_t *C_r);
/* Life expectancy (Appendix C: "average of age of agent that died during a large
 * time window of 500 timesteps"), accumulated on the device: for windows [first, first+n)
 * of SIM_LIFE_WINDOW steps (aligned to multiples of it), per world the deaths and the summed
 * ages at death (age after the step's increment); the expectancy is age_sum / deaths.
 * out[i][w] (int64, caller-owned [n][n_worlds]); windows must be complete and among the
 * last kept (the step log's span); counts restart at sim_set_state.  Synchronises. */
#define SIM_LIFE_WINDOW 500
SIM_API sim_status sim_get_life_windows(sim_handle h, int64_t first, int64_t n, int64_t *deaths, int64_t *age_sum);
/* Run ONE step without the graph, with CUDA events around every kernel; synchronises. */
SIM_API sim_status sim_step_timed(sim_handle h, sim_step_timing *out);
/* Run ONE step exactly as graph mode does (the policy kernel, then the cooperative k_post
 * kernel: same kernels, same parameters) launched directly with a CUDA event before,
 * between and after them; synchronises.  out_ms[0] = policy, out_ms[1] = k_post
 * (milliseconds).  SIM_E_STATE on a sharded handle. */
SIM_API sim_status sim_step_graph_timed(sim_handle h, float out_ms[2]);
/* Graph mode runs everything after the policy kernel as one cooperative kernel (k_post).
 * One world: move | grid barrier | block 0: birth claims, rank (the births flag), placement
 * and counters, while the other blocks regrow step t+1 and then mutate the children (and
 * 4 or 16 warps per block make the next step's P rows from the start).  Several worlds:
 * move | claims | per-world rank beside the regrowth | mutation, separated by barriers.
 * out[i] = summed duration (ns, device global timer, as seen by block 0) over the steps
 * since the last reset; reset > 0 zeroes.  out[0..3]: those four laps of block 0 (move +
 * barrier, claims, rank until the flag, the rest); out[4..7] reserved (diagnostic builds);
 * out[8]: summed durations of block 0's warps on the claims (several worlds); out[9]: summed
 * durations of the regrowth warps of block 1.
 * reset < 0 (diagnostic builds): out receives 16 + 32768 words, the per-block clocks or
 * per-agent traces after the first 16. */
#define SIM_NUM_POST_PHASES 10
SIM_API sim_status sim_get_phase_ns(sim_handle h, int64_t *out, int32_t reset);
/* --- agent-sharded mode: one world over n_ranks GPUs (the agent-home
 * variant of E.2) ------------------------------------------------------------------------
 * Every rank creates the same world (same config and seed) on its own GPU and calls
 * sim_shard(h, n_ranks, rank).  Slot s belongs to rank s % n_ranks (children belong to
 * their parent's rank); only the owner runs an agent's policy and keeps its weights, h, c,
 * logits and last action current, while every rank runs the integer dynamics (regrowth,
 * movement, consumption, physiology, death, births) identically.  One step on every rank:
 *   sim_step_policy(h);                       policy of the owned agents
 *   exchange: SUM-allreduce over the ranks of the two device buffers sim_exchange returns
 *     (the move records by slot, int32, 16 B per slot, zero for other ranks' agents; and
 *     the policy counters, 2 x int64: active inputs, near ties)  — e.g. ncclAllReduce on
 *     the handle's stream
 *   sim_step_post(h);                         the dynamics, identical on every rank
 * The trajectory equals the unsharded one exactly (the sums are of disjoint non-zero
 * parts).  sim_step and sim_step_timed return SIM_E_STATE on a sharded handle; set_state
 * resets ownership to s % n_ranks.  Requires n_worlds = 1 and hidden = 32. */
SIM_API sim_status sim_shard(sim_handle h, int32_t n_ranks, int32_t rank);
SIM_API sim_status sim_step_policy(sim_handle h);
SIM_API sim_status sim_step_post(sim_handle h);
/* Device pointers (owned by the handle, valid until destroy) and sizes of the buffers to
 * SUM-allreduce between sim_step_policy and sim_step_post: the move records (int32) and
 * the policy counters (int64). */
SIM_API sim_status sim_exchange(sim_handle h, void **mrec, size_t *mrec_bytes, void **record, size_t *record_bytes);

/* --- banded mode over several GPUs (sim_config.n_bands) -----------
 * One process per GPU, each handle holding one band (band_first = rank, band_local = 1):
 *   every rank: sim_band_export(h, rank, blob, &bytes)  -> all-gather the blobs (e.g.
 *     torch.distributed.all_gather_object); sim_band_import(h, b, blob_b, bytes) for every
 *     other band b (CUDA IPC: the neighbours' planes, claims and outboxes become readable
 *     over NVLink, and every band's birth counts);
 *   rank 0: sim_band_nccl_id(id) -> broadcast the 128 bytes; every rank:
 *     sim_band_nccl_init(h, id, n_bands, rank);
 * then sim_step(h, n) on every rank: the phases of each step are separated by stream-
 * ordered NCCL token exchanges with the neighbour bands (and one all-reduce for the global
 * birth counts), and the exchanges themselves are kernels reading the neighbours' memory.
 * sim_get_state returns this band's rows and agents (the caller merges the ranks' states by
 * cell); sim_set_state takes the whole world's state on every rank and keeps its band's
 * share.  sim_band_export with out = NULL returns the blob size in *bytes.  NCCL is loaded
 * at run time (libnccl.so.2); its failures return SIM_E_NCCL and poison the handle. */
SIM_API sim_status sim_band_export(sim_handle h, int32_t band, void *out, size_t *bytes);
SIM_API sim_status sim_band_import(sim_handle h, int32_t band, const void *blob, size_t bytes);
SIM_API sim_status sim_band_nccl_id(void *out128);
SIM_API sim_status sim_band_nccl_init(sim_handle h, const void *id128, int32_t n_ranks, int32_t rank);
/* One banded step with CUDA events around every local band's phases, run one band after the
 * other (so each time is that band's alone, as on its own GPU); synchronises.  out:
 * [band_local][n_phases] ms, n_phases = SIM_BAND_PHASES in the order halo_x1 (with the
 * previous step's cross-band newborns), policy, merge_x2, move, arrive_x3, live, prep_p,
 * halo_x4a, claims, merge_x4b, rank, mutate, regrow (prep_p: the next step's recurrent gate
 * sums P = W_hh h + b of the survivors, which sim_step runs on a second stream beside
 * halo_x4a .. regrow; 0 unless hidden = 32).  (A banded sim_step on one GPU replays one
 * CUDA graph per step.) */
#define SIM_BAND_PHASES 13
SIM_API sim_status sim_band_step_timed(sim_handle h, float *out, int32_t n_phases);

/* Synchronise the handle's stream (reports deferred errors). */
SIM_API sim_status sim_synchronize(sim_handle h);
/* Number of kernels of an instrumented step (sim_step_timed; a graph step launches two). */
SIM_API int32_t sim_kernels_per_step(void);

#ifdef __cplusplus
}
#endif
#endif
