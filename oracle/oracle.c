/*
 * oracle/oracle.c — CPU ORACLE FOR THE WORLD STEP.  TEST INFRASTRUCTURE ONLY.
 * (Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs
 * may load it.  It shares no code with the CUDA path.)
 *
 * Plain single-threaded C99, compiled with -O2 -ffp-contract=off.  Every phase is
 * written in the order of SURVEY.md §8c C.3 and cites the PAPER.md passage it
 * follows; every place where the paper is silent or garbled uses the reading
 * R<n> listed in DESIGN.md §3.
 */
#include "oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- RNG (C.1) --- */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11): round function
 *   (x0,x1,x2,x3) -> (hi(M1*x2)^x1^k0, lo(M1*x2), hi(M0*x0)^x3^k1, lo(M0*x0)),
 * key bumped by the Weyl constants between rounds.  Pinned against the cuRAND
 * generator in tests/test_oracle_rng.py. */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)M0 * (uint64_t)x0;
        uint64_t p1 = (uint64_t)M1 * (uint64_t)x2;
        uint32_t y0 = (uint32_t)(p1 >> 32) ^ x1 ^ k0;
        uint32_t y1 = (uint32_t)p1;
        uint32_t y2 = (uint32_t)(p0 >> 32) ^ x3 ^ k1;
        uint32_t y3 = (uint32_t)p0;
        x0 = y0; x1 = y1; x2 = y2; x3 = y3;
        k0 += W0;
        k1 += W1;
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

/* counter = (c0 = sub, c1 = entity, c2 = step, c3 = purpose), key = (seed lo, seed hi) */
void orc_draw4(uint64_t seed, uint32_t purpose, uint32_t step, uint32_t entity, uint32_t sub,
               uint32_t out[4]) {
    uint32_t ctr[4] = {sub, entity, step, purpose};
    uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
    orc_philox4x32_10(ctr, key, out);
}

uint32_t orc_cell_draw(uint64_t seed, uint32_t purpose, uint32_t step, uint32_t cell) {
    uint32_t w[4];
    orc_draw4(seed, purpose, step, cell >> 2, 0u, w);
    return w[cell & 3u];
}

/* u1 = (wa+1)*2^-32 in (0,1], u2 = wb*2^-32 in [0,1); z_a = r cos th, z_b = r sin th */
void orc_box_muller(uint32_t wa, uint32_t wb, double *za, double *zb) {
    const double two_m32 = 2.3283064365386963e-10; /* 2^-32 */
    double u1 = ((double)wa + 1.0) * two_m32;
    double u2 = (double)wb * two_m32;
    double rad = sqrt(-2.0 * log(u1));
    double th = 6.283185307179586 * u2;
    *za = rad * cos(th);
    *zb = rad * sin(th);
}

void orc_gauss(uint64_t seed, uint32_t purpose, uint32_t step, uint32_t entity, int32_t n,
               double *z) {
    for (int32_t j = 0; j < n; ++j) {
        uint32_t q = (uint32_t)j >> 2;
        uint32_t w[4];
        orc_draw4(seed, purpose, step, entity, q, w);
        double za, zb;
        if ((j & 3) < 2) orc_box_muller(w[0], w[1], &za, &zb);
        else orc_box_muller(w[2], w[3], &za, &zb);
        z[j] = ((j & 1) == 0) ? za : zb;
    }
}

/* ------------------------------------------------------------- sizes/validation */
int32_t orc_input_count(const orc_config *cfg) {
    if (cfg->network == 1) return ORC_CNN_WO * ORC_CNN_WO * ORC_CNN_CH; /* 15x15x3 */
    int32_t w = 2 * cfg->obs_radius + 1;
    return 2 * w * w;
}

/* network 0: P = 4Hd*I + 4Hd*Hd + 4Hd + 5Hd + 5 (canonical order).
 * network 1, counted layer by layer from the architecture:
 *   conv1 3x3x3 -> 4 (+4 biases), conv2 3x3x4 -> 8 (+8), LSTM 78 -> 4 (4 gates over
 *   78 + 4 inputs, +16 biases), dense 82 -> 8 (+8), dense 8 -> 5 (+5)          */
int32_t orc_param_count(const orc_config *cfg) {
    if (cfg->network == 1) {
        const int32_t c1 = 3 * 3 * ORC_CNN_CH * 4 + 4, c2 = 3 * 3 * 4 * 8 + 8;
        const int32_t G = 4 * ORC_CNN_HD;
        const int32_t lstm = G * (ORC_CNN_EMB + ORC_CNN_HD) + G;
        const int32_t dense = (ORC_CNN_EMB + ORC_CNN_HD) * ORC_CNN_DENSE + ORC_CNN_DENSE;
        const int32_t out = ORC_CNN_DENSE * cfg->n_actions + cfg->n_actions;
        return c1 + c2 + lstm + dense + out;
    }
    int32_t I = orc_input_count(cfg), Hd = cfg->hidden, A = cfg->n_actions;
    return 4 * Hd * I + 4 * Hd * Hd + 4 * Hd + A * Hd + A;
}

static int bad(char *msg, int len, const char *field) {
    if (msg && len > 0) snprintf(msg, (size_t)len, "invalid field: %s", field);
    return ORC_E_INVALID;
}

static int prob_ok(double p) { return p >= 0.0 && p <= 1.0; }

int orc_validate(const orc_config *cfg, char *msg, int msg_len) {
    if (cfg->rows < 2) return bad(msg, msg_len, "rows");           /* lat divides by H-1 */
    if (cfg->cols < 4 || cfg->cols % 4 != 0) return bad(msg, msg_len, "cols");
    if (!prob_ok(cfg->init_resource_p)) return bad(msg, msg_len, "init_resource_p");
    if (cfg->regrow_r2 < 1 || cfg->regrow_r2 > 8) return bad(msg, msg_len, "regrow_r2");
    if (cfg->f_class_min_k[0] != 0) return bad(msg, msg_len, "f_class_min_k");
    for (int c = 1; c < 4; ++c)
        if (cfg->f_class_min_k[c] < cfg->f_class_min_k[c - 1]) return bad(msg, msg_len, "f_class_min_k");
    for (int c = 0; c < 4; ++c)
        if (!prob_ok(cfg->f_value[c])) return bad(msg, msg_len, "f_value");
    if (!prob_ok(cfg->lat_top) || !prob_ok(cfg->lat_bottom)) return bad(msg, msg_len, "lat");
    if (!prob_ok(cfg->spontaneous)) return bad(msg, msg_len, "spontaneous");
    if (cfg->slots < 0) return bad(msg, msg_len, "slots");
    if (cfg->n_initial < 0 || cfg->n_initial > cfg->slots) return bad(msg, msg_len, "n_initial");
    if (cfg->network != 0 && cfg->network != 1) return bad(msg, msg_len, "network");
    if (cfg->colocate != 0 && cfg->colocate != 1) return bad(msg, msg_len, "colocate");
    if (cfg->colocate && cfg->network != 1) return bad(msg, msg_len, "colocate"); /* (network 1 only) */
    if (cfg->network == 1) { /* the paper's architecture fixes the window and the LSTM */
        if (cfg->obs_radius != (ORC_CNN_WO - 1) / 2) return bad(msg, msg_len, "obs_radius");
        if (cfg->hidden != ORC_CNN_HD) return bad(msg, msg_len, "hidden");
    } else {
        if (cfg->obs_radius < 0 || cfg->obs_radius > 3) return bad(msg, msg_len, "obs_radius");
        if (cfg->hidden < 1 || cfg->hidden > 32) return bad(msg, msg_len, "hidden");
    }
    if (cfg->n_actions != 5) return bad(msg, msg_len, "n_actions");
    if (!(cfg->init_weight_std >= 0.0)) return bad(msg, msg_len, "init_weight_std");
    if (!(cfg->mutation_std >= 0.0)) return bad(msg, msg_len, "mutation_std");
    if (cfg->repr_steps < 1) return bad(msg, msg_len, "repr_steps");
    if (cfg->max_age < 0) return bad(msg, msg_len, "max_age");
    if (!(cfg->climate_alpha >= 0.0)) return bad(msg, msg_len, "climate_alpha");
    if (cfg->death_steps < 0) return bad(msg, msg_len, "death_steps");
    if (cfg->lethal_walls != 0 && cfg->lethal_walls != 1) return bad(msg, msg_len, "lethal_walls");
    return ORC_OK;
}

/* ------------------------------------------------------------ regrowth (C.3.1) */
/* lat(y) = lat_top + (lat_bottom-lat_top)*(y/(H-1)), division first (R3); with
 * climate_alpha > 0 the paper's climate c(x) = (alpha^x + 1)/(alpha + 1) at x = y/(H-1)
 * (x = 1 at the bottom row, R1);
 * p = lat*f[c] + spont ("p = p_I * c(x) + c");
 * T = min(floor(p*2^32), 2^32-1) (R8). */
void orc_thresholds(const orc_config *cfg, uint32_t *T) {
    for (int32_t y = 0; y < cfg->rows; ++y) {
        double frac = (double)y / (double)(cfg->rows - 1);
        double lat = cfg->lat_top + (cfg->lat_bottom - cfg->lat_top) * frac;
        if (cfg->climate_alpha > 0.0) lat = (pow(cfg->climate_alpha, frac) + 1.0) / (cfg->climate_alpha + 1.0);
        for (int c = 0; c < 4; ++c) {
            double p = lat * cfg->f_value[c] + cfg->spontaneous;
            double s = floor(p * 4294967296.0);
            T[y * 4 + c] = (s >= 4294967295.0) ? 0xFFFFFFFFu : (uint32_t)s;
        }
    }
}

/* k = sum of R over offsets with dy^2+dx^2 <= r2, (dy,dx) != (0,0); off-grid = 0 (R4) */
int32_t orc_neighbour_count(const orc_config *cfg, const uint8_t *R, int32_t y, int32_t x) {
    int32_t H = cfg->rows, W = cfg->cols, k = 0;
    for (int32_t dy = -3; dy <= 3; ++dy)
        for (int32_t dx = -3; dx <= 3; ++dx) {
            if (dy == 0 && dx == 0) continue;
            if (dy * dy + dx * dx > cfg->regrow_r2) continue;
            int32_t yy = y + dy, xx = x + dx;
            if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
            k += R[yy * W + xx] ? 1 : 0;
        }
    return k;
}

/* the step function f of BASELINE configs[0]: class = max c with k >= min_k[c] (R5) */
int32_t orc_class_of(const orc_config *cfg, int32_t k) {
    int32_t cls = 0;
    for (int c = 1; c < 4; ++c)
        if (k >= cfg->f_class_min_k[c]) cls = c;
    return cls;
}

/* synchronous: every empty cell draws against the start-of-step grid (R6); regrowth
 * ignores agents (R7); full cells stay full. */
int64_t orc_regrow(const orc_config *cfg, int64_t t, const uint8_t *R, uint8_t *Rn) {
    int32_t H = cfg->rows, W = cfg->cols;
    uint32_t *T = (uint32_t *)malloc(sizeof(uint32_t) * 4 * (size_t)H);
    orc_thresholds(cfg, T);
    int64_t grown = 0;
    for (int32_t y = 0; y < H; ++y)
        for (int32_t x = 0; x < W; ++x) {
            int32_t cell = y * W + x;
            if (R[cell]) { Rn[cell] = 1; continue; }
            int32_t k = orc_neighbour_count(cfg, R, y, x);
            int32_t cls = orc_class_of(cfg, k);
            uint32_t u = orc_cell_draw(cfg->seed, ORC_P_REGROW, (uint32_t)t, (uint32_t)cell);
            Rn[cell] = (u < T[y * 4 + cls]) ? 1 : 0;
            grown += Rn[cell];
        }
    free(T);
    return grown;
}

/* ---------------------------------------------------------- observation (C.3.2) */
/* Square (2r+1)x(2r+1) window centred on the agent, channel 0 =
 * resources after regrowth, channel 1 = occupancy at step start incl. self (R10,
 * R11); channel-major, rows from the top; off-grid reads 0. */
void orc_observe(const orc_config *cfg, const uint8_t *R, const uint8_t *O, int32_t y,
                 int32_t x, double *xout) {
    int32_t r = cfg->obs_radius, w = 2 * r + 1, H = cfg->rows, W = cfg->cols;
    for (int ch = 0; ch < 2; ++ch) {
        const uint8_t *plane = ch == 0 ? R : O;
        for (int32_t dy = -r; dy <= r; ++dy)
            for (int32_t dx = -r; dx <= r; ++dx) {
                int32_t yy = y + dy, xx = x + dx;
                double v = 0.0;
                if (yy >= 0 && yy < H && xx >= 0 && xx < W) v = plane[yy * W + xx] ? 1.0 : 0.0;
                xout[ch * w * w + (dy + r) * w + (dx + r)] = v;
            }
    }
}

/* -------------------------------------------------------------- policy (C.3.3) */
static double sigmoid(double z) { return 1.0 / (1.0 + exp(-z)); }

/* LSTM cell ("an LSTM cell ... and a linear layer that transforms
 * hidden states to actions"), gates (i,f,g,o), single bias (R12):
 *   z = W_ih x + W_hh h + b; c' = f*c + i*g; h' = o*tanh(c');
 *   logits = W_out h' + b_out; action = argmax, lowest index on exact tie (R28). */
int orc_policy(const orc_config *cfg, const float *w, const double *x, const float *h,
               const float *c, float *h_out, float *c_out, float *logits_out, int32_t *action,
               double *margin) {
    int32_t I = orc_input_count(cfg), Hd = cfg->hidden, A = cfg->n_actions, G = 4 * Hd;
    const float *W_ih = w;
    const float *W_hh = W_ih + (size_t)G * I;
    const float *b = W_hh + (size_t)G * Hd;
    const float *W_out = b + G;
    const float *b_out = W_out + (size_t)A * Hd;
    double z[128];
    for (int32_t r = 0; r < G; ++r) {
        double s = 0.0;
        for (int32_t j = 0; j < I; ++j) s += (double)W_ih[(size_t)r * I + j] * x[j];
        for (int32_t j = 0; j < Hd; ++j) s += (double)W_hh[(size_t)r * Hd + j] * (double)h[j];
        s += (double)b[r];
        z[r] = s;
    }
    int nonfinite = 0;
    for (int32_t k = 0; k < Hd; ++k) {
        double ig = sigmoid(z[k]);
        double fg = sigmoid(z[Hd + k]);
        double gg = tanh(z[2 * Hd + k]);
        double og = sigmoid(z[3 * Hd + k]);
        double cn = fg * (double)c[k] + ig * gg;
        double hn = og * tanh(cn);
        c_out[k] = (float)cn;
        h_out[k] = (float)hn;
        if (!isfinite(c_out[k]) || !isfinite(h_out[k])) nonfinite = 1;
    }
    for (int32_t a = 0; a < A; ++a) {
        double s = 0.0;
        for (int32_t k = 0; k < Hd; ++k) s += (double)W_out[(size_t)a * Hd + k] * (double)h_out[k];
        s += (double)b_out[a];
        logits_out[a] = (float)s;
        if (!isfinite(logits_out[a])) nonfinite = 1;
    }
    int32_t best = 0;
    for (int32_t a = 1; a < A; ++a)
        if (logits_out[a] > logits_out[best]) best = a;
    double second = -INFINITY;
    for (int32_t a = 0; a < A; ++a)
        if (a != best && (double)logits_out[a] > second) second = (double)logits_out[a];
    *action = best;
    *margin = (double)logits_out[best] - second;
    return nonfinite ? ORC_E_NONFINITE : ORC_OK;
}

/* ------------------------------------- network 1: the paper's CNN-LSTM (NEXT-2) */
/* "An agent observes pixel values ... within its visual range (a square of size
 * [w_o, w_o] centered around the agent)"; "The pixel values contain information about the
 * resources, other agents (including their number) and walls"; w_o = 15
 * (PAPER.md:317).  Three channels (R39): resources after regrowth, agents at step start
 * incl. self (0/1 under exclusive occupancy), walls = every cell off the grid. */
void orc_observe_paper(const orc_config *cfg, const uint8_t *R, const int32_t *N, int32_t y,
                       int32_t x, double *xout) {
    const int32_t r = (ORC_CNN_WO - 1) / 2, H = cfg->rows, W = cfg->cols;
    for (int32_t row = 0; row < ORC_CNN_WO; ++row)
        for (int32_t col = 0; col < ORC_CNN_WO; ++col) {
            int32_t yy = y - r + row, xx = x - r + col;
            int on = yy >= 0 && yy < H && xx >= 0 && xx < W;
            double *px = xout + ((size_t)row * ORC_CNN_WO + col) * ORC_CNN_CH;
            px[0] = on && R[yy * W + xx] ? 1.0 : 0.0;
            px[1] = on ? (double)N[yy * W + xx] : 0.0; /* "(including their number)" */
            px[2] = on ? 0.0 : 1.0;
        }
}

/* "First CNN has a kernel size (3,3), stride 2": SAME zero padding (R40),
 * out = ceil(n/2) with total padding 2(out-1) + 3 - n, its floor half before. */
void orc_conv3x3_s2_same(const double *in, int32_t H, int32_t W, int32_t cin, const float *w,
                         const float *b, int32_t cout, double *out) {
    const int32_t OH = (H + 1) / 2, OW = (W + 1) / 2;
    const int32_t pad_y = (2 * (OH - 1) + 3 - H) / 2, pad_x = (2 * (OW - 1) + 3 - W) / 2;
    for (int32_t oy = 0; oy < OH; ++oy)
        for (int32_t ox = 0; ox < OW; ++ox)
            for (int32_t f = 0; f < cout; ++f) {
                double s = (double)b[f];
                for (int32_t ky = 0; ky < 3; ++ky)
                    for (int32_t kx = 0; kx < 3; ++kx) {
                        int32_t iy = 2 * oy + ky - pad_y, ix = 2 * ox + kx - pad_x;
                        if (iy < 0 || iy >= H || ix < 0 || ix >= W) continue; /* zero pad */
                        for (int32_t ch = 0; ch < cin; ++ch)
                            s += (double)w[((f * 3 + ky) * 3 + kx) * cin + ch] *
                                 in[((size_t)iy * W + ix) * cin + ch];
                    }
                out[((size_t)oy * OW + ox) * cout + f] = s;
            }
}

/* "average pooling of size (2,2) and stride 1", VALID (R40) */
void orc_avgpool2_s1(const double *in, int32_t H, int32_t W, int32_t C, double *out) {
    for (int32_t y = 0; y + 1 < H; ++y)
        for (int32_t x = 0; x + 1 < W; ++x)
            for (int32_t ch = 0; ch < C; ++ch) {
                double s = in[((size_t)y * W + x) * C + ch] + in[((size_t)y * W + x + 1) * C + ch] +
                           in[((size_t)(y + 1) * W + x) * C + ch] +
                           in[((size_t)(y + 1) * W + x + 1) * C + ch];
                out[((size_t)y * (W - 1) + x) * C + ch] = s / 4.0;
            }
}

/* CNN -> flatten (72) ++ previous action (one-hot 5) ++ ate (1) = e (78);
 * LSTM(4) on e; [e, h'] (82) -> dense 8 tanh -> dense 5 = logits.  No activation after
 * the convolutions (R41); the LSTM gates as network 0 (i,f,g,o, one bias, R12). */
int orc_policy_cnn(const orc_config *cfg, const float *w, const double *obs, int32_t last_action,
                   int32_t ate, const float *h, const float *c, float *h_out, float *c_out,
                   float *logits_out, double *emb_out) {
    const int32_t E = ORC_CNN_EMB, Hd = ORC_CNN_HD, G = 4 * Hd, D = ORC_CNN_DENSE, A = cfg->n_actions;
    const float *c1w = w, *c1b = c1w + 3 * 3 * ORC_CNN_CH * 4;
    const float *c2w = c1b + 4, *c2b = c2w + 3 * 3 * 4 * 8;
    const float *W_ih = c2b + 8, *W_hh = W_ih + G * E, *bl = W_hh + G * Hd;
    const float *W_d = bl + G, *b_d = W_d + D * (E + Hd);
    const float *W_o = b_d + D, *b_o = W_o + A * D;
    double a1[8 * 8 * 4], p1[7 * 7 * 4], a2[4 * 4 * 8], e[ORC_CNN_EMB + ORC_CNN_HD], z[16], d[8];
    orc_conv3x3_s2_same(obs, ORC_CNN_WO, ORC_CNN_WO, ORC_CNN_CH, c1w, c1b, 4, a1); /* 8x8x4 */
    orc_avgpool2_s1(a1, 8, 8, 4, p1);                                              /* 7x7x4 */
    orc_conv3x3_s2_same(p1, 7, 7, 4, c2w, c2b, 8, a2);                             /* 4x4x8 */
    orc_avgpool2_s1(a2, 4, 4, 8, e);                                               /* 3x3x8 = 72 */
    for (int32_t a = 0; a < 5; ++a) e[72 + a] = (a == last_action) ? 1.0 : 0.0;
    e[77] = ate ? 1.0 : 0.0;
    for (int32_t r = 0; r < G; ++r) {
        double s = 0.0;
        for (int32_t j = 0; j < E; ++j) s += (double)W_ih[r * E + j] * e[j];
        for (int32_t j = 0; j < Hd; ++j) s += (double)W_hh[r * Hd + j] * (double)h[j];
        z[r] = s + (double)bl[r];
    }
    int nonfinite = 0;
    for (int32_t k = 0; k < Hd; ++k) {
        double ig = sigmoid(z[k]), fg = sigmoid(z[Hd + k]), gg = tanh(z[2 * Hd + k]);
        double og = sigmoid(z[3 * Hd + k]);
        double cn = fg * (double)c[k] + ig * gg;
        c_out[k] = (float)cn;
        h_out[k] = (float)(og * tanh(cn));
        if (!isfinite(c_out[k]) || !isfinite(h_out[k])) nonfinite = 1;
    }
    /* "we concatenate the embedding with the output of the LSTM" */
    for (int32_t k = 0; k < Hd; ++k) e[E + k] = (double)h_out[k];
    for (int32_t r = 0; r < D; ++r) {
        double s = 0.0;
        for (int32_t j = 0; j < E + Hd; ++j) s += (double)W_d[r * (E + Hd) + j] * e[j];
        d[r] = tanh(s + (double)b_d[r]);
    }
    for (int32_t a = 0; a < A; ++a) {
        double s = 0.0;
        for (int32_t k = 0; k < D; ++k) s += (double)W_o[a * D + k] * d[k];
        logits_out[a] = (float)(s + (double)b_o[a]);
        if (!isfinite(logits_out[a])) nonfinite = 1;
    }
    if (emb_out) memcpy(emb_out, e, sizeof(double) * (size_t)E);
    return nonfinite ? ORC_E_NONFINITE : ORC_OK;
}

/* "a last denser layer of size 5 ... with softmax to get the action probability from which
 * the action will be sampled.  The softmax we use has a low temperature (1/50)"
 * (PAPER.md:348): P_a = exp(50 l_a) / sum_b exp(50 l_b) from the fp32 logits; inverse-CDF
 * sampling with one Philox word keyed by the agent's cell (R38). */
int32_t orc_sample_action(uint64_t seed, uint32_t step, uint32_t entity, const float *logits,
                          double *probs_out, double *margin) {
    double m = -INFINITY, p[5], S = 0.0;
    for (int a = 0; a < 5; ++a)
        if (ORC_CNN_TEMP_INV * (double)logits[a] > m) m = ORC_CNN_TEMP_INV * (double)logits[a];
    for (int a = 0; a < 5; ++a) {
        p[a] = exp(ORC_CNN_TEMP_INV * (double)logits[a] - m);
        S += p[a];
    }
    for (int a = 0; a < 5; ++a) p[a] /= S;
    uint32_t w4[4];
    orc_draw4(seed, ORC_P_ACTION, step, entity, 0u, w4);
    const double u = (double)w4[0] * 2.3283064365386963e-10; /* [0, 1) */
    int32_t act = 4;
    double cum = 0.0, mg = INFINITY;
    for (int a = 0; a < 4; ++a) {
        cum += p[a];
        if (fabs(u - cum) < mg) mg = fabs(u - cum);
        if (act == 4 && u < cum) act = a;
    }
    if (probs_out) memcpy(probs_out, p, sizeof(p));
    *margin = mg;
    return act;
}

/* ------------------------------------------------------------ init (C.2) ------ */
typedef struct {
    uint32_t draw;
    int32_t cell;
} place_key;

static int place_cmp(const void *a, const void *b) {
    const place_key *p = (const place_key *)a, *q = (const place_key *)b;
    if (p->draw != q->draw) return p->draw < q->draw ? -1 : 1;
    return (p->cell > q->cell) - (p->cell < q->cell);
}

static void init_weights(const orc_config *cfg, int32_t entity, uint32_t step, uint32_t purpose,
                         float *w) {
    int32_t P = orc_param_count(cfg);
    double *z = (double *)malloc(sizeof(double) * (size_t)P);
    orc_gauss(cfg->seed, purpose, step, (uint32_t)entity, P, z);
    for (int32_t j = 0; j < P; ++j) w[j] = (float)(cfg->init_weight_std * z[j]);
    free(z);
}

/* "Starting resources ... randomly placed", "Starting population ... randomly placed",
 * weights "initialized randomly once"; BASELINE constants. */
int orc_init(const orc_config *cfg, orc_state *st) {
    int rc = orc_validate(cfg, NULL, 0);
    if (rc) return rc;
    int32_t H = cfg->rows, W = cfg->cols, S = cfg->slots, Hd = cfg->hidden;
    int32_t P = orc_param_count(cfg), A = cfg->n_actions;
    int64_t HW = (int64_t)H * W;
    /* 1. R[cell] = draw(INIT_RES, 0, cell) < floor(rho*2^32) */
    double s = floor(cfg->init_resource_p * 4294967296.0);
    uint32_t thr = (s >= 4294967295.0) ? 0xFFFFFFFFu : (uint32_t)s;
    int64_t n_empty = 0;
    for (int64_t cell = 0; cell < HW; ++cell) {
        st->resources[cell] =
            orc_cell_draw(cfg->seed, ORC_P_INIT_RES, 0u, (uint32_t)cell) < thr ? 1 : 0;
        n_empty += st->resources[cell] ? 0 : 1;
    }
    if (cfg->n_initial > n_empty) return ORC_E_INVALID;
    /* 2. empty cells sorted by (draw(INIT_PLACE, 0, cell), cell); slot i <- i-th (R24) */
    place_key *keys = NULL;
    if (cfg->n_initial > 0) {
        keys = (place_key *)malloc(sizeof(place_key) * (size_t)n_empty);
        int64_t m = 0;
        for (int64_t cell = 0; cell < HW; ++cell)
            if (!st->resources[cell]) {
                keys[m].draw = orc_cell_draw(cfg->seed, ORC_P_INIT_PLACE, 0u, (uint32_t)cell);
                keys[m].cell = (int32_t)cell;
                ++m;
            }
        qsort(keys, (size_t)n_empty, sizeof(place_key), place_cmp);
    }
    /* 3. agents */
    for (int32_t i = 0; i < S; ++i) {
        int is_init = i < cfg->n_initial;
        st->alive[i] = is_init ? 1 : 0;
        st->cell[i] = is_init ? keys[i].cell : 0;
        st->energy[i] = is_init ? cfg->e_init : 0;
        st->age[i] = 0;
        st->repr[i] = 0;
        if (st->low) st->low[i] = 0;
        st->last_action[i] = 0;
        st->ate[i] = 0;
        for (int32_t k = 0; k < Hd; ++k) {
            st->h[(size_t)i * Hd + k] = 0.0f;
            st->c[(size_t)i * Hd + k] = 0.0f;
        }
        for (int32_t a = 0; a < A; ++a) st->logits[(size_t)i * A + a] = 0.0f;
        float *w = st->weights + (size_t)i * P;
        if (is_init) init_weights(cfg, keys[i].cell, 0u, ORC_P_INIT_W, w);
        else memset(w, 0, sizeof(float) * (size_t)P);
    }
    free(keys);
    st->t = 0;
    return ORC_OK;
}

/* ------------------------------------------------------------ step (C.3) ------ */
/* action deltas (R13): 0 stay, 1 N (y-1), 2 S (y+1), 3 E (x+1), 4 W (x-1) */
static const int32_t DY[5] = {0, -1, 1, 0, 0};
static const int32_t DX[5] = {0, 0, 0, 1, -1};

int orc_step(const orc_config *cfg, orc_state *st, const uint8_t *forced, uint8_t *actions_out,
             orc_record *rec) {
    int32_t H = cfg->rows, W = cfg->cols, S = cfg->slots, Hd = cfg->hidden;
    int32_t P = orc_param_count(cfg), I = orc_input_count(cfg), A = cfg->n_actions;
    int64_t HW = (int64_t)H * W;
    uint32_t t = (uint32_t)st->t;
    memset(rec, 0, sizeof(*rec));
    rec->t = st->t;

    uint8_t *Rn = (uint8_t *)calloc((size_t)HW, 1);
    uint8_t *O = (uint8_t *)calloc((size_t)HW, 1);
    uint8_t *On = (uint8_t *)calloc((size_t)HW, 1);
    uint64_t *claim = (uint64_t *)calloc((size_t)HW, sizeof(uint64_t));
    int32_t *action = (int32_t *)calloc((size_t)(S > 0 ? S : 1), sizeof(int32_t));
    int32_t *target = (int32_t *)calloc((size_t)(S > 0 ? S : 1), sizeof(int32_t));
    uint64_t *key = (uint64_t *)calloc((size_t)(S > 0 ? S : 1), sizeof(uint64_t));
    double *x = (double *)calloc((size_t)I, sizeof(double));
    int status = ORC_OK;

    /* 1. REGROW */
    rec->grown = orc_regrow(cfg, st->t, st->resources, Rn);

    /* O_t: cells holding a live agent at step start; N_t: the number of agents per cell */
    int32_t *N = (int32_t *)calloc((size_t)HW, sizeof(int32_t));
    for (int32_t i = 0; i < S; ++i)
        if (st->alive[i]) {
            O[st->cell[i]] = 1;
            N[st->cell[i]] += 1;
        }

    /* 2-3. OBSERVE + POLICY */
    for (int32_t i = 0; i < S; ++i) {
        if (!st->alive[i]) continue;
        int32_t y = st->cell[i] / W, xx = st->cell[i] % W;
        float hn[32], cn[32], lg[8];
        int32_t a;
        double margin;
        int rc;
        if (cfg->network == 1) { /* the paper's CNN-LSTM, sampled */
            orc_observe_paper(cfg, Rn, N, y, xx, x);
            rc = orc_policy_cnn(cfg, st->weights + (size_t)i * P, x, st->last_action[i], st->ate[i],
                                st->h + (size_t)i * Hd, st->c + (size_t)i * Hd, hn, cn, lg, NULL);
            /* keyed by the cell (unique under exclusive occupancy, R9) or by the slot (R47) */
            a = orc_sample_action(cfg->seed, t, cfg->colocate ? (uint32_t)i : (uint32_t)st->cell[i], lg, NULL,
                                  &margin);
        } else {
            orc_observe(cfg, Rn, O, y, xx, x);
            rc = orc_policy(cfg, st->weights + (size_t)i * P, x, st->h + (size_t)i * Hd,
                            st->c + (size_t)i * Hd, hn, cn, lg, &a, &margin);
        }
        if (rc != ORC_OK) status = rc;
        if (margin < 1e-4) rec->near_ties++;
        memcpy(st->h + (size_t)i * Hd, hn, sizeof(float) * (size_t)Hd);
        memcpy(st->c + (size_t)i * Hd, cn, sizeof(float) * (size_t)Hd);
        memcpy(st->logits + (size_t)i * A, lg, sizeof(float) * (size_t)A);
        if (forced && forced[i] != 255) a = forced[i];
        action[i] = a;
        st->last_action[i] = (uint8_t)a;
    }
    if (actions_out)
        for (int32_t i = 0; i < S; ++i) actions_out[i] = st->alive[i] ? (uint8_t)action[i] : 255;

    /* 4. MOVE: exclusive occupancy, claim by max key (R14), blocked at the edge (R15) */
    for (int32_t i = 0; i < S; ++i) {
        target[i] = -1;
        if (!st->alive[i] || action[i] == 0) continue;
        int32_t y = st->cell[i] / W, xx = st->cell[i] % W;
        int32_t ty = y + DY[action[i]], tx = xx + DX[action[i]];
        if (ty < 0 || ty >= H || tx < 0 || tx >= W) {
            if (cfg->lethal_walls) target[i] = -2; /* walks into the wall: dies */
            continue;
        }
        int32_t tc = ty * W + tx;
        if (cfg->colocate) { /* no collision exclusion (R43): every in-grid move succeeds */
            target[i] = tc;
            continue;
        }
        if (O[tc]) continue;
        uint32_t w4[4];
        orc_draw4(cfg->seed, ORC_P_MOVE, t, (uint32_t)st->cell[i], 0u, w4);
        key[i] = ((uint64_t)w4[0] << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)st->cell[i]);
        target[i] = tc;
        if (key[i] > claim[tc]) claim[tc] = key[i];
    }
    for (int32_t i = 0; i < S; ++i)
        if (target[i] >= 0 && (cfg->colocate || claim[target[i]] == key[i])) st->cell[i] = target[i];
    /* wall deaths: before consumption, so such an agent neither eats nor ages; its age at
     * death counts the step (age + 1, as every death) */
    for (int32_t i = 0; i < S; ++i)
        if (st->alive[i] && target[i] == -2) {
            st->alive[i] = 0;
            st->ate[i] = 0;
            rec->deaths_wall++;
        }

    /* 5. CONSUME ("if the agent consumes a resource").  Co-location (R45): the
     * agents standing on a resource cell hold a lottery, the largest (CONSUME draw of the
     * slot, -slot) key eats ("exactly one ... consumes"). */
    if (cfg->colocate) {
        uint64_t *ckey = (uint64_t *)calloc((size_t)HW, sizeof(uint64_t));
        for (int32_t i = 0; i < S; ++i) {
            key[i] = 0;
            if (!st->alive[i] || !Rn[st->cell[i]]) continue;
            uint32_t w4[4];
            orc_draw4(cfg->seed, ORC_P_CONSUME, t, (uint32_t)i, 0u, w4);
            key[i] = ((uint64_t)w4[0] << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)i);
            if (key[i] > ckey[st->cell[i]]) ckey[st->cell[i]] = key[i];
        }
        for (int32_t i = 0; i < S; ++i) {
            if (!st->alive[i]) continue;
            int32_t p = st->cell[i];
            st->ate[i] = (key[i] != 0 && ckey[p] == key[i]) ? 1 : 0;
        }
        for (int32_t i = 0; i < S; ++i)
            if (st->alive[i] && st->ate[i]) {
                Rn[st->cell[i]] = 0;
                rec->eaten++;
            }
        free(ckey);
    } else {
        for (int32_t i = 0; i < S; ++i) {
            if (!st->alive[i]) continue;
            int32_t p = st->cell[i];
            if (Rn[p]) {
                Rn[p] = 0;
                st->ate[i] = 1;
                rec->eaten++;
            } else {
                st->ate[i] = 0;
            }
        }

    }

    /* 6. PHYSIOLOGY (linear decrease, +1 per resource; R16, R17, R19) */
    for (int32_t i = 0; i < S; ++i) {
        if (!st->alive[i]) continue;
        int64_t e = (int64_t)st->energy[i] + (int64_t)cfg->e_gain * st->ate[i] - cfg->e_decay;
        if (cfg->e_max != INT32_MAX && e > cfg->e_max) e = cfg->e_max;
        st->energy[i] = (int32_t)e;
        st->age[i] += 1;
        st->repr[i] = (st->energy[i] > cfg->e_repr_gt) ? st->repr[i] + 1 : 0;
        if (st->low) st->low[i] = (st->energy[i] <= cfg->e_death_le) ? st->low[i] + 1 : 0;
    }

    /* 7. DEATH (immediate form, R18) */
    for (int32_t i = 0; i < S; ++i) {
        if (!st->alive[i]) continue;
        /* immediate form (R18), or the paper's timer: T_death consecutive steps at or below
         * the threshold */
        const int starved = cfg->death_steps > 0 ? (st->low && st->low[i] >= cfg->death_steps)
                                                 : (st->energy[i] <= cfg->e_death_le);
        if (starved) {
            st->alive[i] = 0;
            rec->deaths_energy++;
        } else if (st->age[i] > cfg->max_age) {
            st->alive[i] = 0;
            rec->deaths_age++;
        }
    }
    for (int32_t i = 0; i < S; ++i)
        if (st->alive[i]) On[st->cell[i]] = 1; /* O'' */

    /* 8. REPRODUCE (R19-R22) */
    if (cfg->colocate) {
        /* co-location (R46): "the off-spring appears on the same cell as its parent"
         * (PAPER.md:297); the eligible parents in ascending slot order take the free slots
         * (alive == 0 after phase 7) in ascending order, the rest are deferred (capacity) */
        int32_t *freelist = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S > 0 ? S : 1));
        int32_t *elig = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S > 0 ? S : 1));
        int32_t n_free = 0, n_el = 0;
        for (int32_t i = 0; i < S; ++i) {
            if (!st->alive[i]) freelist[n_free++] = i;
            else if (st->repr[i] >= cfg->repr_steps) elig[n_el++] = i;
        }
        double *z = (double *)malloc(sizeof(double) * (size_t)P);
        for (int32_t r = 0; r < n_el; ++r) {
            int32_t par = elig[r];
            if (r >= n_free) {
                rec->deferred_capacity++;
                continue;
            }
            int32_t ch = freelist[r], cc = st->cell[par];
            st->alive[ch] = 1;
            st->cell[ch] = cc;
            st->energy[ch] = cfg->e_init;
            st->age[ch] = 0;
            st->repr[ch] = 0;
            if (st->low) st->low[ch] = 0;
            st->last_action[ch] = 0;
            st->ate[ch] = 0;
            for (int32_t k = 0; k < Hd; ++k) {
                st->h[(size_t)ch * Hd + k] = 0.0f;
                st->c[(size_t)ch * Hd + k] = 0.0f;
            }
            for (int32_t a = 0; a < A; ++a) st->logits[(size_t)ch * A + a] = 0.0f;
            /* the noise keyed by the child's slot (R47: co-located children share a cell) */
            orc_gauss(cfg->seed, ORC_P_MUTATE, t, (uint32_t)ch, P, z);
            const float *wp = st->weights + (size_t)par * P;
            float *wc = st->weights + (size_t)ch * P;
            for (int32_t j = 0; j < P; ++j) wc[j] = wp[j] + (float)(cfg->mutation_std * z[j]);
            st->repr[par] = 0;
            rec->births++;
        }
        free(z);
        free(elig);
        free(freelist);
    } else {
        static const int32_t BDY[4] = {-1, 1, 0, 0}; /* N, S, E, W */
        static const int32_t BDX[4] = {0, 0, 1, -1};
        int32_t *cand = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S > 0 ? S : 1));
        uint64_t *bkey = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(S > 0 ? S : 1));
        uint64_t *bclaim = (uint64_t *)calloc((size_t)HW, sizeof(uint64_t));
        for (int32_t i = 0; i < S; ++i) {
            cand[i] = -1;
            if (!st->alive[i] || st->repr[i] < cfg->repr_steps) continue;
            int32_t p = st->cell[i], y = p / W, xx = p % W;
            uint32_t w4[4];
            orc_draw4(cfg->seed, ORC_P_BIRTH, t, (uint32_t)p, 0u, w4);
            uint32_t s0 = w4[0] & 3u;
            for (uint32_t k = 0; k < 4; ++k) {
                uint32_t d = (s0 + k) & 3u;
                int32_t cy = y + BDY[d], cx = xx + BDX[d];
                if (cy < 0 || cy >= H || cx < 0 || cx >= W) continue;
                int32_t c = cy * W + cx;
                if (On[c] || Rn[c]) continue;
                cand[i] = c;
                break;
            }
            if (cand[i] < 0) {
                rec->deferred_no_cell++;
                continue;
            }
            bkey[i] = ((uint64_t)w4[1] << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)p);
            if (bkey[i] > bclaim[cand[i]]) bclaim[cand[i]] = bkey[i];
        }
        /* winners, ranked by child cell ascending */
        int32_t n_win = 0;
        int32_t *win_order = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S > 0 ? S : 1));
        for (int32_t i = 0; i < S; ++i) {
            if (cand[i] < 0) continue;
            if (bclaim[cand[i]] == bkey[i]) {
                win_order[n_win++] = i;
            } else {
                rec->deferred_claim++;
            }
        }
        /* sort winners by child cell (insertion sort: plain and obviously correct) */
        for (int32_t a = 1; a < n_win; ++a) {
            int32_t v = win_order[a], b = a - 1;
            while (b >= 0 && cand[win_order[b]] > cand[v]) {
                win_order[b + 1] = win_order[b];
                --b;
            }
            win_order[b + 1] = v;
        }
        /* free slots: alive == 0 after phase 7, ascending */
        int32_t *freelist = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S > 0 ? S : 1));
        int32_t n_free = 0;
        for (int32_t i = 0; i < S; ++i)
            if (!st->alive[i]) freelist[n_free++] = i;
        double *z = (double *)malloc(sizeof(double) * (size_t)P);
        for (int32_t r = 0; r < n_win; ++r) {
            int32_t par = win_order[r];
            if (r >= n_free) {
                rec->deferred_capacity++;
                continue;
            }
            int32_t ch = freelist[r], cc = cand[par];
            st->alive[ch] = 1;
            st->cell[ch] = cc;
            st->energy[ch] = cfg->e_init;
            st->age[ch] = 0;
            st->repr[ch] = 0;
            if (st->low) st->low[ch] = 0;
            st->last_action[ch] = 0;
            st->ate[ch] = 0;
            for (int32_t k = 0; k < Hd; ++k) {
                st->h[(size_t)ch * Hd + k] = 0.0f;
                st->c[(size_t)ch * Hd + k] = 0.0f;
            }
            for (int32_t a = 0; a < A; ++a) st->logits[(size_t)ch * A + a] = 0.0f;
            /* "an agent's weights are mutated by adding noise sampled from N(0, sigma)"
             * (PAPER.md:301), sigma a standard deviation (R23) */
            orc_gauss(cfg->seed, ORC_P_MUTATE, t, (uint32_t)cc, P, z);
            const float *wp = st->weights + (size_t)par * P;
            float *wc = st->weights + (size_t)ch * P;
            for (int32_t j = 0; j < P; ++j) wc[j] = wp[j] + (float)(cfg->mutation_std * z[j]);
            st->repr[par] = 0;
            On[cc] = 1;
            rec->births++;
        }
        free(z);
        free(freelist);
        free(win_order);
        free(bclaim);
        free(bkey);
        free(cand);
    }

    /* 9. t <- t+1; R_{t+1} = R'' */
    memcpy(st->resources, Rn, (size_t)HW);
    for (int32_t i = 0; i < S; ++i) rec->population += st->alive[i];
    for (int64_t c = 0; c < HW; ++c) rec->resources += st->resources[c];
    st->t += 1;

    free(N);
    free(x);
    free(key);
    free(target);
    free(action);
    free(claim);
    free(On);
    free(O);
    free(Rn);
    return status;
}
