/*
 * oracle/oracle.h — CPU ORACLE FOR THE WORLD STEP.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product (paper_2302_09334_b200/, include/sim.h)
 * shares no source, header, table or helper with it.
 *
 * A plain, slow, single-threaded C99 implementation of one world step of the
 * non-episodic neuroevolution simulator of arXiv 2302.09334 (Hamon, Nisioti,
 * Moulin-Frier), App. B, under the BASELINE.json configs and the
 * readings R1-R30 listed in DESIGN.md §3 (which follow SURVEY.md §8c).
 *
 * Floating point: the LSTM is evaluated in fp64 from fp32 weights and fp32 stored
 * state; h', c' are rounded to fp32 for storage, logits are rounded to fp32 and the
 * argmax is taken on the fp32 values (the decision precision of the kernel).
 * Everything else is integer.  Randomness: Philox4x32-10 counter RNG (C.1).
 *
 * Parity pins: see tests/test_oracle_*.py.  Full multi-step trajectories are
 * "parity unpinned" by the paper (its configs differ and its figures are missing):
 * they are pinned only through the per-phase pins, invariants and scripted walks.
 */
#ifndef ECO_ORACLE_H
#define ECO_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define ORC_OK 0
#define ORC_E_INVALID (-1)
#define ORC_E_NONFINITE (-5)

/* RNG purposes (counter word c3) */
#define ORC_P_INIT_RES 1u
#define ORC_P_INIT_PLACE 2u
#define ORC_P_INIT_W 3u
#define ORC_P_REGROW 4u
#define ORC_P_MOVE 5u
#define ORC_P_BIRTH 6u
#define ORC_P_MUTATE 7u
#define ORC_P_ACTION 8u  /* the sampled action of network 1 ("sampled") */
#define ORC_P_CONSUME 9u /* co-location: the lottery among agents sharing a resource cell */

/* network 1, the paper's CNN-LSTM: sizes */
#define ORC_CNN_WO 15   /* field of view w_o = 15                        */
#define ORC_CNN_CH 3    /* resources, agents, walls (SPEC's 2445 count)   */
#define ORC_CNN_EMB 78  /* 3*3*8 CNN features + one-hot previous action (5) + ate (1)   */
#define ORC_CNN_HD 4    /* LSTM hidden size                              */
#define ORC_CNN_DENSE 8 /* dense layer with tanh                         */
#define ORC_CNN_TEMP_INV 50.0 /* softmax temperature 1/50: softmax(50 * logits)         */

typedef struct {
    int32_t rows, cols;           /* H (latitude axis, row 0 = top), W            */
    uint64_t seed;                /* Philox key = (lo32, hi32)                     */
    double init_resource_p;       /* Bernoulli rho                                 */
    int32_t regrow_r2;            /* squared Euclidean radius of the count disc   */
    int32_t f_class_min_k[4];     /* class c iff k >= f_class_min_k[c] (max such) */
    double f_value[4];            /* f(class)                                      */
    double lat_top, lat_bottom;   /* lat(0), lat(H-1)                              */
    double spontaneous;           /* constant spontaneous growth probability      */
    int32_t slots, n_initial;     /* S, N0                                         */
    int32_t obs_radius, hidden, n_actions;
    double init_weight_std, mutation_std;
    int32_t e_init, e_decay, e_gain, e_repr_gt, e_death_le, e_max; /* milli-units */
    int32_t repr_steps, max_age;
    /* the paper's own world (App. B.4), off by default:            */
    double climate_alpha;         /* > 0: c(x) = (alpha^x + 1)/(alpha + 1), x = y/(H-1),  */
                                  /* replaces the linear lat               */
    int32_t death_steps;          /* > 0: die after this many consecutive steps with      */
                                  /* energy <= e_death_le (T_death)          */
    int32_t lethal_walls;         /* 1: a move off the grid kills the agent */
    /* the agents' network: 0 = LSTM + linear head with argmax on a
     * (2r+1)^2 x 2 window (BASELINE); 1 = the paper's CNN-LSTM on a 15x15x3 window with
     * softmax(50 logits) sampling (obs_radius 7, hidden 4)            */
    int32_t network;
    /* co-location (the paper's own reproduction; R43-R47), requires
     * network 1: any number of agents per cell, moves never conflict, one agent per resource
     * cell eats (a lottery), the offspring appears on its parent's cell; the
     * agent channel counts agents; ACTION, CONSUME and MUTATE draws are keyed by slot     */
    int32_t colocate;
} orc_config;

/* Canonical state; all buffers are owned by the caller. */
typedef struct {
    int64_t t;
    uint8_t *resources;   /* [H][W] 0/1                                          */
    uint8_t *alive;       /* [S]                                                 */
    int32_t *cell;        /* [S] y*W+x                                           */
    int32_t *energy;      /* [S] milli-units                                     */
    int32_t *age;         /* [S]                                                 */
    int32_t *repr;        /* [S] consecutive steps with energy > e_repr_gt      */
    uint8_t *last_action; /* [S]                                                 */
    uint8_t *ate;         /* [S]                                                 */
    float *h;             /* [S][Hd]                                             */
    float *c;             /* [S][Hd]                                             */
    float *weights;       /* [S][P] canonical: W_ih[4Hd][I], W_hh[4Hd][Hd], b[4Hd], W_out[5][Hd], b_out[5];
                             network 1 (P = 2445): conv1_w[4][3][3][3] ([out][ky][kx][in]),
                             conv1_b[4], conv2_w[8][3][3][4], conv2_b[8], W_ih[16][78],
                             W_hh[16][4], b[16] (gates i,f,g,o), W_d[8][82], b_d[8],
                             W_out[5][8], b_out[5]                                   */
    float *logits;        /* [S][5]                                              */
    int32_t *low;         /* [S] consecutive steps with energy <= e_death_le (death timer) */
} orc_state;

typedef struct {
    int64_t t;                   /* the step index this record describes */
    int64_t grown, eaten, births;
    int64_t deaths_energy, deaths_age;
    int64_t deferred_no_cell, deferred_claim, deferred_capacity;
    int64_t population, resources; /* after the step */
    int64_t near_ties;              /* live agents with top1-top2 logit margin < 1e-4 (network 1:
                                       the sampling margin < 1e-4, R38) */
    int64_t deaths_wall;            /* agents killed by a move off the grid (lethal walls) */
} orc_record;

int32_t orc_param_count(const orc_config *cfg);
int32_t orc_input_count(const orc_config *cfg);
int orc_validate(const orc_config *cfg, char *msg, int msg_len);

/* Philox4x32-10, Salmon et al. SC'11 */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* the four words of draw(purpose, step, entity, sub) under `seed` (C.1) */
void orc_draw4(uint64_t seed, uint32_t purpose, uint32_t step, uint32_t entity, uint32_t sub,
               uint32_t out[4]);
/* per-cell draw: entity = cell>>2, sub = 0, word cell&3 (C.1) */
uint32_t orc_cell_draw(uint64_t seed, uint32_t purpose, uint32_t step, uint32_t cell);
/* fp64 Box-Muller of a pair of words (C.1) */
void orc_box_muller(uint32_t wa, uint32_t wb, double *za, double *zb);
/* z[0..n) for (purpose, step, entity) with sub = j>>2 (C.1) */
void orc_gauss(uint64_t seed, uint32_t purpose, uint32_t step, uint32_t entity, int32_t n,
               double *z);

/* T[y][c] = min(floor(p(y,c)*2^32), 2^32-1), p = lat(y)*f[c] + c_spont */
void orc_thresholds(const orc_config *cfg, uint32_t *T /* [H][4] */);
/* k(y,x): resources within the radius disc, centre excluded, off-grid = 0 */
int32_t orc_neighbour_count(const orc_config *cfg, const uint8_t *R, int32_t y, int32_t x);
int32_t orc_class_of(const orc_config *cfg, int32_t k);
/* one synchronous regrowth pass R -> Rn at step t; returns cells grown (C.3.1) */
int64_t orc_regrow(const orc_config *cfg, int64_t t, const uint8_t *R, uint8_t *Rn);

/* egocentric window x[I] from planes R (channel 0) and O (channel 1) (C.3.2) */
void orc_observe(const orc_config *cfg, const uint8_t *R, const uint8_t *O, int32_t y,
                 int32_t x, double *xout);
/* LSTM + linear head + argmax on one agent (C.3.3).  Returns ORC_OK or ORC_E_NONFINITE. */
int orc_policy(const orc_config *cfg, const float *w, const double *x, const float *h,
               const float *c, float *h_out, float *c_out, float *logits_out, int32_t *action,
               double *margin);

/* ---- network 1: the paper's CNN-LSTM, evaluated in fp64 ---- */
/* 15x15x3 window, HWC (x[(row*15 + col)*3 + ch]), rows from the top: ch 0 resources
 * after regrowth, ch 1 the number of agents at step start incl. self (N: agents per cell),
 * ch 2 walls = 1 off the grid */
void orc_observe_paper(const orc_config *cfg, const uint8_t *R, const int32_t *N, int32_t y,
                       int32_t x, double *xout);
/* 3x3 convolution, stride 2, SAME zero padding (out = ceil(n/2), pad 1 before), HWC in,
 * w[cout][3][3][cin], b[cout]; out[(oy*OW + ox)*cout + f] */
void orc_conv3x3_s2_same(const double *in, int32_t H, int32_t W, int32_t cin, const float *w,
                         const float *b, int32_t cout, double *out);
/* 2x2 average pool, stride 1, VALID: (H-1)x(W-1)xC, HWC */
void orc_avgpool2_s1(const double *in, int32_t H, int32_t W, int32_t C, double *out);
/* the forward of one agent: the 78-float embedding e, the LSTM (h', c', fp32 stored), the
 * tanh dense layer and the 5 logits (fp32).  emb_out may be NULL. Returns ORC_OK or
 * ORC_E_NONFINITE. */
int orc_policy_cnn(const orc_config *cfg, const float *w, const double *obs, int32_t last_action,
                   int32_t ate, const float *h, const float *c, float *h_out, float *c_out,
                   float *logits_out, double *emb_out);
/* softmax(50 * logits) sampled with u = draw(ACTION, step, entity)[0] * 2^-32 (entity = the
 * agent's step-start cell, or its slot under co-location): the least a
 * with u < P_0 + ... + P_a (4 if none); *margin = min over the 4 inner boundaries of
 * |u - (P_0 + ... + P_k)| (a near-tie below 1e-4, R38); probs_out (may be NULL) [5] */
int32_t orc_sample_action(uint64_t seed, uint32_t step, uint32_t entity, const float *logits,
                          double *probs_out, double *margin);

/* initial world (C.2) */
int orc_init(const orc_config *cfg, orc_state *st);
/* one full world step (C.3); forced: [S] action per slot, 255 = policy; NULL = none.
 * actions_out (test hook, may be NULL): [S] the action each slot alive at step start
 * used this step (255 for slots not alive at step start) — recorded before births can
 * reuse a slot freed by a death in the same step. */
int orc_step(const orc_config *cfg, orc_state *st, const uint8_t *forced, uint8_t *actions_out,
             orc_record *rec);

#ifdef __cplusplus
}
#endif
#endif
