// api.cu — the C ABI of include/sim.h: validation, device allocation, initialisation,
// the per-step CUDA graph, state import/export and the test/measurement hooks.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "sim_internal.cuh"

// Tracing: NVTX ranges around the ABI's calls and the banded step's phases,
// visible in nsys / ncu timelines; free when no tool is attached (ECO_NVTX=0 compiles them out).
#ifndef ECO_NVTX
#define ECO_NVTX 1
#endif
#if ECO_NVTX
#include <nvtx3/nvToolsExt.h>
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
#define ECO_TRACE(name) NvtxRange eco_trace_range_(name)
#else
#define ECO_TRACE(name) ((void)0)
#endif

using eco::DevParams;

namespace {
// movement-histogram windows kept: a power of two covering the step log
inline int mv_windows(int log_cap) {
    int c = 1;
    while (c < log_cap / SIM_MOVE_WINDOW + 2) c <<= 1;
    return c;
}
// life-expectancy windows kept: a power of two covering the step log
inline int le_windows(int log_cap) {
    int c = 2;
    while (c < log_cap / SIM_LIFE_WINDOW + 2) c <<= 1;
    return c;
}
}  // namespace

namespace {

thread_local std::string g_last_error;

sim_status fail(sim_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

// host copy of the validated configuration plus derived sizes
struct Derived {
    int H, W, WW, S, SW, Hd, I, P, Pd, n_worlds, log_cap;
    int off_hh, off_b, off_out, off_bout;
    int net;    // 0: LSTM + linear head (argmax); 1: the paper's CNN-LSTM (sampled)
    int coloc;  // 1: co-location (any number of agents per cell; network 1)
    size_t pw;  // words per plane per world
};

sim_status validate_cfg(const sim_config *cfg, Derived *d) {
    if (!cfg) return fail(SIM_E_INVALID, "invalid field: cfg (NULL)");
    if (cfg->abi_version != SIM_ABI_VERSION) return fail(SIM_E_INVALID, "invalid field: abi_version");
    if (cfg->struct_size != sizeof(sim_config)) return fail(SIM_E_INVALID, "invalid field: struct_size");
    if (cfg->rows < 2) return fail(SIM_E_INVALID, "invalid field: rows (need >= 2)");
    if (cfg->cols < 4 || cfg->cols % 4 != 0) return fail(SIM_E_INVALID, "invalid field: cols (need >= 4, multiple of 4)");
    if ((int64_t)cfg->rows * cfg->cols >= (int64_t)1 << 31) return fail(SIM_E_INVALID, "invalid field: rows*cols");
    if (cfg->n_worlds < 1) return fail(SIM_E_INVALID, "invalid field: n_worlds");
    if ((int64_t)cfg->n_worlds * cfg->rows * ((cfg->cols + 31) / 32) >= (int64_t)1 << 31)
        return fail(SIM_E_INVALID, "invalid field: n_worlds (n_worlds * rows * ceil(cols/32) must be < 2^31)");
    if (!cfg->seeds) return fail(SIM_E_INVALID, "invalid field: seeds (NULL)");
    auto prob = [](double v) { return v >= 0.0 && v <= 1.0; };
    if (!prob(cfg->init_resource_p)) return fail(SIM_E_INVALID, "invalid field: init_resource_p");
    if (cfg->regrow_r2 < 1 || cfg->regrow_r2 > 8) return fail(SIM_E_INVALID, "invalid field: regrow_r2 (1..8)");
    if (cfg->f_class_min_k[0] != 0) return fail(SIM_E_INVALID, "invalid field: f_class_min_k");
    for (int c = 1; c < 4; ++c)
        if (cfg->f_class_min_k[c] < cfg->f_class_min_k[c - 1]) return fail(SIM_E_INVALID, "invalid field: f_class_min_k");
    for (int c = 0; c < 4; ++c)
        if (!prob(cfg->f_value[c])) return fail(SIM_E_INVALID, "invalid field: f_value");
    if (!prob(cfg->lat_top) || !prob(cfg->lat_bottom)) return fail(SIM_E_INVALID, "invalid field: lat");
    if (!prob(cfg->spontaneous)) return fail(SIM_E_INVALID, "invalid field: spontaneous");
    // (<= 2^24 - 1: k_post carries a step's birth count in 24 bits of its release flag)
    if (cfg->slots < 0 || cfg->slots > 0xFFFFFF) return fail(SIM_E_INVALID, "invalid field: slots");
    if (cfg->n_initial < 0 || cfg->n_initial > cfg->slots) return fail(SIM_E_INVALID, "invalid field: n_initial");
    if (cfg->network != 0 && cfg->network != 1) return fail(SIM_E_INVALID, "invalid field: network (0 or 1)");
    if (cfg->network == 1) {  // the paper's architecture fixes the window and the LSTM
        if (cfg->obs_radius != 7) return fail(SIM_E_INVALID, "invalid field: obs_radius (network 1: 7, a 15x15 window)");
        if (cfg->hidden != 4) return fail(SIM_E_INVALID, "invalid field: hidden (network 1: 4)");
        if (cfg->n_bands > 1)
            return fail(SIM_E_INVALID, "invalid field: n_bands (network 1's 7-row window exceeds the bands' halo)");
    }
    if (cfg->colocate != 0 && cfg->colocate != 1) return fail(SIM_E_INVALID, "invalid field: colocate (0 or 1)");
    if (cfg->colocate && cfg->network != 1) return fail(SIM_E_INVALID, "invalid field: colocate (needs network 1)");
    if (cfg->network == 1) {
    } else {
        if (cfg->obs_radius < 0 || cfg->obs_radius > 3) return fail(SIM_E_INVALID, "invalid field: obs_radius (0..3)");
        if (!(cfg->hidden == 4 || cfg->hidden == 8 || cfg->hidden == 16 || cfg->hidden == 32))
            return fail(SIM_E_INVALID, "invalid field: hidden (4, 8, 16 or 32)");
    }
    if (cfg->n_actions != 5) return fail(SIM_E_INVALID, "invalid field: n_actions (must be 5)");
    if (!(cfg->init_weight_std >= 0.0) || !std::isfinite(cfg->init_weight_std))
        return fail(SIM_E_INVALID, "invalid field: init_weight_std");
    if (!(cfg->mutation_std >= 0.0) || !std::isfinite(cfg->mutation_std))
        return fail(SIM_E_INVALID, "invalid field: mutation_std");
    if (cfg->repr_steps < 1) return fail(SIM_E_INVALID, "invalid field: repr_steps");
    if (cfg->max_age < 0) return fail(SIM_E_INVALID, "invalid field: max_age");
    if (cfg->log_capacity < 0 || cfg->log_capacity == 1) return fail(SIM_E_INVALID, "invalid field: log_capacity");
    if (!(cfg->climate_alpha >= 0.0) || !std::isfinite(cfg->climate_alpha))
        return fail(SIM_E_INVALID, "invalid field: climate_alpha");
    if (cfg->death_steps < 0) return fail(SIM_E_INVALID, "invalid field: death_steps");
    if (cfg->lethal_walls != 0 && cfg->lethal_walls != 1) return fail(SIM_E_INVALID, "invalid field: lethal_walls (0 or 1)");
    if (d) {
        d->H = cfg->rows;
        d->W = cfg->cols;
        d->WW = (((cfg->cols + 31) / 32) + 3) / 4 * 4;
        d->S = cfg->slots;
        d->SW = (cfg->slots + 31) / 32;
        d->Hd = cfg->hidden;
        const int wd = 2 * cfg->obs_radius + 1;
        d->I = 2 * wd * wd;
        d->P = 4 * d->Hd * d->I + 4 * d->Hd * d->Hd + 4 * d->Hd + 5 * d->Hd + 5;
        d->off_hh = d->I * d->Hd * 4;
        d->off_b = d->off_hh + d->Hd * d->Hd * 4;
        d->off_out = d->off_b + d->Hd * 4;
        d->off_bout = d->off_out + 5 * d->Hd;
        d->Pd = (d->off_bout + 5 + 31) / 32 * 32;
        d->net = cfg->network;
        d->coloc = cfg->colocate;
        if (d->net == 1) {  // canonical order on the device too (sim.h), rows padded to 32 floats
            d->I = 15 * 15 * 3;
            d->P = 2445;
            d->Pd = 2464;
            d->off_hh = d->off_b = d->off_out = d->off_bout = 0;  // (network 0's layout only)
        }
        d->n_worlds = cfg->n_worlds;
        {  // the ring holds at least log_capacity steps: rounded up to a power of two (a mask)
            const int want = cfg->log_capacity ? cfg->log_capacity : 4096;
            int cap = 2;
            while (cap < want) cap <<= 1;
            d->log_cap = cap;
        }
        d->pw = (size_t)d->H * d->WW;
    }
    return SIM_OK;
}

// Bernoulli thresholds T[y][c] = min(floor((lat(y) f_c + c_spont) 2^32), 2^32-1) with the
// linear climate lat(y) = lat_top + (lat_bottom - lat_top) * (y / (H-1)) (R3, R8), or the
// paper's exponential climate when climate_alpha > 0.
void threshold_table(const sim_config *cfg, std::vector<uint32_t> &T) {
    T.assign((size_t)cfg->rows * 4, 0u);
    for (int y = 0; y < cfg->rows; ++y) {
        const double frac = (double)y / (double)(cfg->rows - 1);
        double lat = cfg->lat_top + (cfg->lat_bottom - cfg->lat_top) * frac;
        // the paper's climate c(x) = (alpha^x + 1)/(alpha + 1), x = 1 at the bottom row (R1)
        if (cfg->climate_alpha > 0.0) lat = (std::pow(cfg->climate_alpha, frac) + 1.0) / (cfg->climate_alpha + 1.0);
        for (int c = 0; c < 4; ++c) {
            const double pr = lat * cfg->f_value[c] + cfg->spontaneous;
            const double s = std::floor(pr * 4294967296.0);
            T[(size_t)y * 4 + c] = s >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)s;
        }
    }
}

constexpr size_t PHASE_WORDS = 16 + 4 * 8192;  // phase clocks + diagnostic-build per-block clocks / traces

size_t device_bytes(const Derived &d) {
    const size_t nw = d.n_worlds, S = d.S, HW = (size_t)d.H * d.W;
    size_t b = 0;
    b += nw * d.pw * 4 * 5;                 // plane0, plane1, occ, bbits[2]
    b += nw * HW * (8 + 8 + 4);             // move claim, birth key, birth slot
    b += nw * ((S + 31) / 32) * 4;          // alive bits
    b += nw * S * (1 * 3 + 4 * 4);          // u8 x3, i32 x4
    b += nw * S * (size_t)d.Hd * 4 * 2;     // h, c
    b += nw * S * eco::LOGIT_STRIDE * 4;    // logits
    b += nw * S * (size_t)d.Pd * 4;         // weights
    b += nw * S * 16;                       // move records
    b += nw * S * 4 * 7;                    // alive lists [2], free, birth lists, mutation counters
    b += nw * S * 8 + S + S * 16 + S * 8;   // birth candidates, owners, by-slot move records, own lists
    b += (size_t)d.log_cap * nw * sizeof(sim_step_record);
    b += nw * S * 8 + nw * (size_t)mv_windows(d.log_cap) * SIM_MOVE_BINS * 4;  // movement metrics
    if (d.coloc) b += nw * HW * 4 + nw * ((S + 31) / 32) * 4;                    // agents per cell, eligible bits
    return b;
}

}  // namespace

struct sim_ctx {
    Derived d{};
    sim_config cfg{};
    std::vector<uint64_t> seeds;
    int device = 0;
    bool band_no_graph = false;  // banded, remote bands: the step could not be captured (api_band.inc)
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    DevParams p{};
    eco::LaunchCfg lc{};
    bool poisoned = false;
    // graph mode: [k_policy, k_post] per step; the first step after create/set_state is
    // preceded by a standalone regrowth (afterwards each k_post regrows the next step).
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    cudaGraph_t graph2 = nullptr;  // ECO_GRAPH_STEPS steps, every policy after the first a programmatic dependent
    cudaGraphExec_t graph2_exec = nullptr;
    bool regrown_ahead = false;
    bool p_ready = false;  // split policy: the P rows of step t exist
    unsigned long long *bar = nullptr;   // grid-barrier words of k_post
    int64_t t = 0;
    int32_t *nonfinite_host = nullptr;
    int32_t *forced_on_dev = nullptr;
    uint8_t *forced_dev = nullptr;
    std::vector<void *> allocs;
    cudaEvent_t ev[SIM_NUM_KERNELS + 1] = {};
    // set_state staging, persistent (no allocation per call): the live slots' global indices,
    // the byte plane of the resources, the gathered device-layout rows of the live weights
    // (grow-only) and, for pageable caller memory only, their compacted canonical rows
    int32_t *live_dev = nullptr;
    uint8_t *res_bytes = nullptr;
    float *wstage = nullptr;
    size_t wstage_rows = 0;
    float *wcanon = nullptr;
    size_t wcanon_rows = 0;
    int32_t *bad_host = nullptr;  // mapped: a non-finite weight seen by the gather
    float *lstage = nullptr;  // set_state: the caller's [n][5] logits before the restride
    size_t lstage_n = 0;
    // banded mode (band.cu): a banded handle drives its local bands,
    // each a sub-context holding the global grid and its own rows' agents
    std::vector<sim_ctx *> bands;   // parent: the local bands in band order
    int G = 1, band_first = 0;
    std::vector<int32_t> band_rows;  // parent: [G+1] row boundaries
    bool is_band = false;            // this context is one band
    eco::BandParams bp{};            // band: its exchange buffers and neighbours
    int32_t *n_own_dev = nullptr;
    struct BandNccl *nccl = nullptr; // parent with remote bands: the NCCL barrier
    cudaStream_t side = nullptr;     // parent: the split policy's P rows beside the step
    cudaEvent_t fork_ev[eco::BAND_MAX] = {}, fork2_ev[eco::BAND_MAX] = {}, join_ev = nullptr;
    int32_t *band_tmp = nullptr;     // parent: device scratch of get_state (a band's live list)
    float *band_canon = nullptr;     // parent: canonical rows of one band's live weights
    size_t band_canon_rows = 0;
    char *hot_base = nullptr;        // the arena of everything but the weights (L2-persisting prefix)
    size_t hot_bytes = 0;
};

namespace {

sim_status cuda_fail(sim_ctx *h, cudaError_t e, const char *what) {
    if (h) h->poisoned = true;
    if (e == cudaErrorMemoryAllocation) return fail(SIM_E_OOM, "%s: %s", what, cudaGetErrorString(e));
    return fail(SIM_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK(h, expr, what)                                    \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) return cuda_fail(h, _e, what); \
    } while (0)

template <typename T>
cudaError_t dalloc(sim_ctx *h, T **ptr, size_t count) {
    *ptr = nullptr;
    if (count == 0) count = 1;
    void *v = nullptr;
    cudaError_t e = cudaMalloc(&v, count * sizeof(T));
    if (e != cudaSuccess) return e;
    h->allocs.push_back(v);
    *ptr = static_cast<T *>(v);
    return cudaMemsetAsync(v, 0, count * sizeof(T), h->stream);
}

sim_status check_handle(sim_ctx *h) {
    if (!h) return fail(SIM_E_INVALID, "invalid argument: NULL handle");
    if (h->poisoned) return fail(SIM_E_STATE, "handle poisoned by an earlier failure");
    return SIM_OK;
}

sim_status check_nonfinite(sim_ctx *h) {
    if (h->nonfinite_host && *reinterpret_cast<volatile int32_t *>(h->nonfinite_host)) {
        *reinterpret_cast<volatile int32_t *>(h->nonfinite_host) = 0;
        return fail(SIM_E_NONFINITE, "non-finite LSTM state or logit produced on the device");
    }
    return SIM_OK;
}

// Instrumented mode: the phases as separate kernels, in graph mode's order, so that every
// kernel can be bracketed by events.  Index order of sim_step_timing.kernel_ms:
// 0 regrow (of step t+1, as inside k_post), 1 policy, 2 move, 3 birth_claim, 4 birth_rank,
// 5 mutate, 6 hh (split policy: the next step's P rows, standalone).  Launch order: policy,
// move, regrow, claim, rank, mutate, hh.
constexpr int kTimedOrder[SIM_NUM_KERNELS] = {1, 2, 0, 3, 4, 5, 6};

cudaError_t launch_phase(sim_ctx *h, int k) {
    switch (k) {
        case 0: return eco::launch_regrow(h->p, 1, h->stream);
        case 1: return eco::launch_policy(h->p, h->lc, h->stream);  // split: reads the P rows
        case 2: return eco::launch_move(h->p, h->lc, h->stream);
        case 3: return eco::launch_birth_claim(h->p, h->lc, h->stream);
        case 4: return eco::launch_birth_rank(h->p, h->stream);
        case 5: return eco::launch_mutate(h->p, h->lc, h->stream);
        default: return eco::launch_prepare_p(h->p, h->lc, h->stream);  // P rows of step t+1 (split only)
    }
}

// graph-mode step: the policy kernel, then the cooperative post-policy kernel
cudaError_t enqueue_step(sim_ctx *h, bool pdl = false) {
    cudaError_t e;
    if (h->p.S == 0 && h->p.regrow_split && !h->p.coloc) {  // an agent-free world: bookkeeping, then the regrowth of t+1
        if ((e = eco::launch_advance_empty(h->p, h->stream)) != cudaSuccess) return e;
        return eco::launch_regrow(h->p, 0, h->stream);
    }
    if ((e = eco::launch_policy(h->p, h->lc, h->stream, pdl)) != cudaSuccess) return e;
    if ((e = eco::launch_post(h->p, h->lc, h->bar, h->stream)) != cudaSuccess) return e;
    if (h->p.regrow_split) return eco::launch_regrow(h->p, 0, h->stream);  // step t+1 (k_post advanced t)
    return cudaSuccess;
}

// The L2 access-policy window of a step graph's kernels: the arena's first bytes (the
// counters, planes, lists, SoA, P rows, h, c ...; never the weights) persisting, within the
// device's persisting carve-out (cudaLimitPersistingL2CacheSize, set here once).  Disabled
// with ECO_L2_PERSIST=0.
bool l2_persist_enabled() {
    const char *v = getenv("ECO_L2_PERSIST");
    return !(v && v[0] == '0');
}
cudaError_t set_persistence(sim_ctx *h, cudaGraph_t g) {
    if (!l2_persist_enabled() || !h->hot_base) return cudaSuccess;
    int max_win = 0, max_persist = 0;
    cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, h->device);
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, h->device);
    if (max_win <= 0 || max_persist <= 0) return cudaSuccess;
    size_t want = h->hot_bytes;
    const size_t budget = (size_t)32 << 20;  // the step's hot state, not the bulk of a large world
    if (want > budget) want = budget;
    if (want > (size_t)max_win) want = (size_t)max_win;
    size_t carve = 0;
    cudaDeviceGetLimit(&carve, cudaLimitPersistingL2CacheSize);
    if (carve < want && carve < (size_t)max_persist) {
        const size_t c = want < (size_t)max_persist ? want : (size_t)max_persist;
        if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, c) == cudaSuccess) carve = c;
        else cudaGetLastError();
    }
    if (carve == 0) return cudaSuccess;
    cudaKernelNodeAttrValue v{};
    v.accessPolicyWindow.base_ptr = h->hot_base;
    v.accessPolicyWindow.num_bytes = want;
    v.accessPolicyWindow.hitRatio = carve >= want ? 1.0f : (float)carve / (float)want;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    size_t n = 0;
    cudaError_t e = cudaGraphGetNodes(g, nullptr, &n);
    if (e != cudaSuccess) return e;
    std::vector<cudaGraphNode_t> nodes(n);
    if ((e = cudaGraphGetNodes(g, nodes.data(), &n)) != cudaSuccess) return e;
    for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType ty;
        if (cudaGraphNodeGetType(nd, &ty) != cudaSuccess || ty != cudaGraphNodeTypeKernel) continue;
        if ((e = cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributeAccessPolicyWindow, &v)) != cudaSuccess)
            return e;
    }
    return cudaSuccess;
}

// capture `steps` (1 or 2) graph steps; in two, the second policy depends programmatically
// on the first k_post (its launch overlaps k_post's drain)
cudaError_t capture_steps(sim_ctx *h, int steps, cudaGraph_t *g, cudaGraphExec_t *ge) {
    cudaError_t e = cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return e;
    for (int i = 0; i < steps && e == cudaSuccess; ++i) e = enqueue_step(h, i > 0);
    cudaError_t e2 = cudaStreamEndCapture(h->stream, g);
    if (e != cudaSuccess) return e;
    if (e2 != cudaSuccess) return e2;
    if ((e = set_persistence(h, *g)) != cudaSuccess) return e;
    return cudaGraphInstantiate(ge, *g, 0);
}

void drop_graphs(sim_ctx *h) {  // kernel parameters changed: capture again on the next step
    if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
    if (h->graph) cudaGraphDestroy(h->graph);
    if (h->graph2_exec) cudaGraphExecDestroy(h->graph2_exec);
    if (h->graph2) cudaGraphDestroy(h->graph2);
    h->graph_exec = h->graph2_exec = nullptr;
    h->graph = h->graph2 = nullptr;
}

// both step graphs, captured eagerly (at create and whenever a kernel parameter changes) so
// that sim_step only launches
bool two_step_graphs(const sim_ctx *h) {
#if ECO_STEP2_PDL
    // (any unsharded handle; the programmatic edge between steps needs the split policy and is
    // only made there, launch_policy)
    return ECO_GRAPH_ALL ? h->p.n_ranks == 1 : (h->p.split && h->p.n_ranks == 1);
#else
    (void)h;
    return false;
#endif
}
cudaError_t ensure_graphs(sim_ctx *h) {
    if (h->p.n_ranks > 1) return cudaSuccess;  // sharded handles step without graphs
    cudaError_t e = cudaSuccess;
    if (!h->graph_exec) e = capture_steps(h, 1, &h->graph, &h->graph_exec);
    if (e == cudaSuccess && two_step_graphs(h) && !h->graph2_exec) e = capture_steps(h, ECO_GRAPH_STEPS, &h->graph2, &h->graph2_exec);
    return e;
}

// the regrowth of the current step, needed once after create/set_state; with the split
// policy also the P rows of the current step (k_post makes them for every later step)
cudaError_t ensure_regrown(sim_ctx *h) {
    if (!h->regrown_ahead) {
        cudaError_t e = eco::launch_regrow(h->p, 0, h->stream);
        if (e != cudaSuccess) return e;
        h->regrown_ahead = true;
    }
    if (h->p.split && !h->p_ready) {
        cudaError_t e = eco::launch_prepare_p(h->p, h->lc, h->stream);
        if (e != cudaSuccess) return e;
        h->p_ready = true;
    }
    return cudaSuccess;
}

sim_status band_sync(sim_ctx *h);  // api_band.inc
sim_status sync(sim_ctx *h) {
    if (!h->bands.empty()) return band_sync(h);
    CK(h, cudaStreamSynchronize(h->stream), "cudaStreamSynchronize");
    return check_nonfinite(h);
}

void band_nccl_destroy(sim_ctx *h);  // api_band.inc
void destroy_all(sim_ctx *h) {
    if (!h) return;
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (sim_ctx *b : h->bands) destroy_all(b);  // (they borrow this stream)
    h->bands.clear();
    if (h->side) {
        cudaStreamSynchronize(h->side);
        cudaStreamDestroy(h->side);
    }
    for (auto &e : h->fork_ev)
        if (e) cudaEventDestroy(e);
    for (auto &e : h->fork2_ev)
        if (e) cudaEventDestroy(e);
    if (h->join_ev) cudaEventDestroy(h->join_ev);
    band_nccl_destroy(h);
    if (h->graph && l2_persist_enabled()) cudaCtxResetPersistingL2Cache();  // release the carve-out's lines
    drop_graphs(h);
    for (auto &e : h->ev)
        if (e) cudaEventDestroy(e);
    for (void *v : h->allocs) cudaFree(v);
    if (h->wstage) cudaFree(h->wstage);
    if (h->wcanon) cudaFree(h->wcanon);
    if (h->lstage) cudaFree(h->lstage);
    if (h->nonfinite_host) cudaFreeHost(h->nonfinite_host);
    if (h->bad_host) cudaFreeHost(h->bad_host);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

}  // namespace

extern "C" {

const char *sim_last_error(void) { return g_last_error.c_str(); }

int32_t sim_kernels_per_step(void) { return SIM_NUM_KERNELS; }

sim_status sim_validate(const sim_config *cfg) { return validate_cfg(cfg, nullptr); }

sim_status sim_state_sizes(const sim_config *cfg, sim_state_sizes_t *out) {
    Derived d;
    sim_status st = validate_cfg(cfg, &d);
    if (st != SIM_OK) return st;
    if (!out) return fail(SIM_E_INVALID, "invalid argument: out (NULL)");
    out->cells = (int64_t)d.H * d.W;
    out->slots = d.S;
    out->hidden = d.Hd;
    out->inputs = d.I;
    out->params = d.P;
    out->n_actions = 5;
    out->device_bytes = (int64_t)device_bytes(d);
    return SIM_OK;
}

}  // extern "C"

namespace {
sim_status create_one(const sim_config *cfg, const eco::BandParams *band, sim_handle *out) {
    if (!out) return fail(SIM_E_INVALID, "invalid argument: out (NULL)");
    *out = nullptr;
    Derived d;
    sim_status st = validate_cfg(cfg, &d);
    if (st != SIM_OK) return st;
    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0)
        return fail(SIM_E_CUDA, "no CUDA device available (the library has no CPU fallback)");
    if (cfg->device < 0 || cfg->device >= n_dev) return fail(SIM_E_INVALID, "invalid field: device");
    sim_ctx *h = new sim_ctx();
    h->d = d;
    h->cfg = *cfg;
    h->seeds.assign(cfg->seeds, cfg->seeds + cfg->n_worlds);
    h->cfg.seeds = nullptr;
    h->device = cfg->device;
    auto bail = [&](sim_status s) {
        destroy_all(h);
        return s;
    };
#define CKC(expr, what)                                              \
    do {                                                             \
        cudaError_t _e = (expr);                                     \
        if (_e != cudaSuccess) return bail(cuda_fail(h, _e, what));  \
    } while (0)
    CKC(cudaSetDevice(h->device), "cudaSetDevice");
    cudaDeviceProp prop;
    CKC(cudaGetDeviceProperties(&prop, h->device), "cudaGetDeviceProperties");
    if (prop.major < 10) return bail(fail(SIM_E_CUDA, "device %s is sm_%d%d; libsim.so is built for sm_100a only", prop.name, prop.major, prop.minor));
    if (cfg->cuda_stream) {
        h->stream = static_cast<cudaStream_t>(cfg->cuda_stream);
    } else {
        CKC(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking), "cudaStreamCreate");
        h->own_stream = true;
    }
    for (auto &e : h->ev) CKC(cudaEventCreate(&e), "cudaEventCreate");
    CKC(cudaHostAlloc(reinterpret_cast<void **>(&h->nonfinite_host), sizeof(int32_t), cudaHostAllocMapped),
        "cudaHostAlloc");
    *h->nonfinite_host = 0;
    CKC(cudaHostAlloc(reinterpret_cast<void **>(&h->bad_host), sizeof(int32_t), cudaHostAllocMapped), "cudaHostAlloc");
    *h->bad_host = 0;

    DevParams &p = h->p;
    p.H = d.H; p.W = d.W; p.WW = d.WW; p.S = d.S; p.SW = d.SW; p.Hd = d.Hd; p.I = d.I; p.P = d.P; p.Pd = d.Pd;
    p.net = d.net;
    p.coloc = d.coloc;
    p.row_lo = band ? band->y0 : 0;
    p.row_hi = band ? band->y1 : d.H;
    p.regrow_split = 0;
    p.hd_shift = 0;
    while ((1 << p.hd_shift) < d.Hd) ++p.hd_shift;  // Hd is a power of two (validated)
    p.n_worlds = d.n_worlds; p.r = cfg->obs_radius; p.log_cap = d.log_cap;
    p.invW = 1.0 / (double)d.W;
    p.repr_steps = cfg->repr_steps; p.max_age = cfg->max_age;
    p.e_init = cfg->e_init; p.e_decay = cfg->e_decay; p.e_gain = cfg->e_gain;
    p.e_repr_gt = cfg->e_repr_gt; p.e_death_le = cfg->e_death_le; p.e_max = cfg->e_max;
    p.death_steps = cfg->death_steps; p.lethal_walls = cfg->lethal_walls;
    p.cls_k1 = cfg->f_class_min_k[1]; p.cls_k2 = cfg->f_class_min_k[2]; p.cls_k3 = cfg->f_class_min_k[3];
    for (int dy = -2; dy <= 2; ++dy) {  // the disc dy^2 + dx^2 <= r2 row by row (r2 <= 8: |dx| <= 2)
        int m = -1;
        for (int dx = 0; dx <= 2; ++dx)
            if (dy * dy + dx * dx <= cfg->regrow_r2) m = dx;
        p.row_dx[dy + 2] = m;
    }
    p.off_hh = d.off_hh; p.off_b = d.off_b; p.off_out = d.off_out; p.off_bout = d.off_bout;
    p.mutation_std = cfg->mutation_std; p.init_weight_std = cfg->init_weight_std;
    {
        const double s = std::floor(cfg->init_resource_p * 4294967296.0);
        p.init_res_thr = s >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)s;
    }
    const size_t nw = d.n_worlds, S = d.S, HW = (size_t)d.H * d.W;
    uint64_t *seeds_d;
    uint32_t *T_d;
    p.mv_cap = mv_windows(d.log_cap);
    p.n_ranks = 1;
    p.rank = 0;
    // split policy (one world, Hd = 32, the default policy kernel): P rows made by k_post
    p.split = (nw == 1 && d.Hd == 32 && S > 0 && eco::policy_supports_shard()) ? 1 : 0;
    // Everything but the weights lives in one arena, ordered by how latency-critical it is:
    // counters, barrier words, planes, lists and SoA first.  Graph kernels get an L2
    // access-policy window marking its prefix persisting (set_persistence below), so the
    // dependent loads of a step's chains hit L2 even when other work evicted the rest.
    std::vector<std::pair<void **, size_t>> hot;
    auto H = [&hot](auto **ptr, size_t count) {
        hot.emplace_back(reinterpret_cast<void **>(ptr), (count ? count : 1) * sizeof(**ptr));
    };
    H(&p.t, nw);
    H(&h->bar, 6);  // [0] arrivals, [1] next base, [2] births flag, [3..4] window-end counters, [5] spare
    H(&p.n_alive, 2 * nw);
    H(&p.n_win, nw);
    H(&p.n_cand, nw);
    H(&p.n_births, nw);
    H(&p.res_count, nw);
    H(&p.totals, 8);
    H(&p.p_children, 1);
    H(&p.own_count, 2);
    H(&p.own_surv, 1);
    H(&p.pol_ctr, 2);
    H(&h->forced_on_dev, 1);
    H(&seeds_d, nw);
    H(&T_d, (size_t)d.H * 4);
    H(&p.plane0, nw * d.pw);
    H(&p.plane1, nw * d.pw);
    H(&p.occ, nw * d.pw);
    H(&p.bbits, 2 * nw * d.pw);
    H(&p.alive_bits, nw * (size_t)d.SW);
    H(&p.alive, nw * S);
    H(&p.last_action, nw * S);
    H(&p.ate, nw * S);
    H(&p.cell, nw * S);
    H(&p.energy, nw * S);
    H(&p.age, nw * S);
    H(&p.repr, nw * S);
    H(&p.low, nw * S);
    H(&p.mrec, nw * S);
    H(&p.alive_list, 2 * nw * S);
    H(&p.list_cell, 2 * nw * S);
    H(&p.cand, nw * S);
    H(&p.birth_child, nw * S);
    H(&p.birth_parent, nw * S);
    H(&p.birth_cell, nw * S);
    H(&p.free_list, nw * S);
    H(&p.log, (size_t)d.log_cap * nw);
    H(&p.mv_cell, nw * S);
    H(&p.mv_inv, nw * S);
    H(&p.mv_hist, nw * (size_t)p.mv_cap * SIM_MOVE_BINS);
    H(&p.gr_seen, nw * S);
    H(&p.gr_ate, nw * S);
    H(&p.gr_T, nw * S);
    H(&p.gr_C, nw * S);
    p.le_cap = le_windows(d.log_cap);
    H(&p.le, nw * (size_t)p.le_cap * 2);
    H(&h->forced_dev, nw * S);
    H(&p.own_act, nw * S);
    H(&p.Pbuf, p.split ? S * (size_t)d.Hd * 4 : 1);
    H(&p.h, nw * S * d.Hd);
    H(&p.c, nw * S * d.Hd);
    H(&p.logits, nw * S * eco::LOGIT_STRIDE);
    H(&p.claim, S ? nw * HW : 1);
    H(&p.bkey, S ? nw * HW : 1);
    H(&p.bslot, S ? nw * HW : 1);
    H(&p.owner, S ? S : 1);
    H(&p.mrec_slot, S ? S : 1);
    H(&p.own_list, S ? 2 * S : 1);
    H(&p.ncount, d.coloc ? nw * HW : 1);              // co-location: agents per cell
    H(&p.elig_bits, d.coloc ? nw * (size_t)d.SW : 1);  // co-location: eligible parents by slot
    H(&p.phase_ns, PHASE_WORDS);  // + per-block clocks / traces of diagnostic builds
    H(&h->live_dev, nw * S);
    H(&h->res_bytes, nw * HW);
    {
        size_t total = 0;
        for (auto &it : hot) total += (it.second + 255) / 256 * 256;
        char *arena = nullptr;
        CKC(dalloc(h, &arena, total), "alloc");
        size_t off = 0;
        for (auto &it : hot) {
            *it.first = arena + off;
            off += (it.second + 255) / 256 * 256;
        }
        h->hot_base = arena;
        h->hot_bytes = total;
    }
    CKC(dalloc(h, &p.weights, nw * S * (size_t)d.Pd), "alloc");
    if (band) {  // one band of a banded world: its outboxes, counts and lists (band.cu)
        h->is_band = true;
        eco::BandParams &bp = h->bp;
        bp = *band;
        bp.cap = d.W < (int)S ? d.W : (int)S;
        CKC(dalloc(h, &bp.mig_out, eco::band_box_words(d.W, (int)S, d.Hd, d.Pd, false)), "alloc");
        CKC(dalloc(h, &bp.nb_out, eco::band_box_words(d.W, (int)S, d.Hd, d.Pd, true)), "alloc");
        CKC(dalloc(h, &bp.counts, 8), "alloc");
        CKC(dalloc(h, &bp.plist, S), "alloc");
        CKC(dalloc(h, &bp.n_plist, 1), "alloc");
        CKC(dalloc(h, &bp.arr_slot, 2 * (size_t)bp.cap), "alloc");
        CKC(dalloc(h, &bp.cslot, HW), "alloc");
        CKC(dalloc(h, &bp.hcand, 2 * (size_t)bp.cap), "alloc");
        CKC(dalloc(h, &bp.n_hcand, 1), "alloc");
        CKC(dalloc(h, &bp.snap, 4), "alloc");
        CKC(dalloc(h, &bp.flags, 4), "alloc");
        CKC(dalloc(h, &h->n_own_dev, 1), "alloc");
    }
    p.seeds = seeds_d;
    p.T = T_d;
    p.forced = h->forced_dev;
    p.forced_on = h->forced_on_dev;
    int32_t *nf_dev = nullptr;
    CKC(cudaHostGetDevicePointer(reinterpret_cast<void **>(&nf_dev), h->nonfinite_host, 0), "cudaHostGetDevicePointer");
    p.nonfinite = nf_dev;
    std::vector<uint32_t> T;
    threshold_table(cfg, T);
    p.t_monotone = 1;
    for (size_t y = 0; y < (size_t)d.H; ++y)
        for (int c = 1; c < 4; ++c)
            if (T[y * 4 + c] < T[y * 4 + c - 1]) p.t_monotone = 0;
    p.disc12 = (p.row_dx[0] == 0 && p.row_dx[1] == 1 && p.row_dx[2] == 2 && p.row_dx[3] == 1 && p.row_dx[4] == 0) ? 1 : 0;
    CKC(cudaMemcpyAsync(T_d, T.data(), T.size() * 4, cudaMemcpyHostToDevice, h->stream), "upload T");
    CKC(cudaMemcpyAsync(seeds_d, h->seeds.data(), nw * 8, cudaMemcpyHostToDevice, h->stream), "upload seeds");

    // launch configuration: persistent-style grids sized to the 148 SMs
    int bps = 0;
    CKC(eco::policy_prepare(), "kernel attributes");  // before the occupancy query (dynamic smem opt-in)
    CKC(eco::post_prepare(), "kernel attributes");
    CKC(eco::policy_occupancy(d.Hd, d.net, &bps, &h->lc.policy_threads), "occupancy");
    if (bps < 1) bps = 1;
    h->lc.policy_blocks = prop.multiProcessorCount * bps;
    h->lc.sms = prop.multiProcessorCount;
    {
        // interleaved contexts spread few agents over every SM when all blocks are resident at
        // once; with more blocks than one wave they leave every block partly empty (a band of
        // the large world: 5.6 waves of 62 %-full blocks instead of 3.5 full ones)
        static const char *bm_env = getenv("ECO_POL_BMAJOR");
        const long half_blocks = ((long)S + 15) / 16;
        p.pol_bmajor = (nw == 1 && d.Hd == 32 && d.net == 0 && half_blocks > (long)h->lc.policy_blocks) ? 1 : 0;
        if (bm_env) p.pol_bmajor = bm_env[0] == '1' && nw == 1 ? 1 : 0;
        // several worlds whose slot pools need more than one wave of blocks: compacted tiles
        static const char *pc_env = getenv("ECO_POL_COMPACT");
        // (default: several worlds only — a large world at its cap fills every block, and there
        // the hardware's block scheduling balances better than the static tile loop: 1518 vs
        // 1537 us per step, measured; ECO_POL_COMPACT=1 compacts every eligible handle, =0 none)
        const bool pc_ok = nw <= (size_t)eco::policy_compact_worlds() && d.Hd == 32 && d.net == 0 &&
                           (long)nw * half_blocks > (long)h->lc.policy_blocks;
        p.pol_compact = pc_ok && (nw > 1 || (pc_env && pc_env[0] == '1')) ? 1 : 0;
        if (pc_env && pc_env[0] == '0') p.pol_compact = 0;
    }
    h->lc.agent_threads = 256;
    {
        const long need = ((long)nw * S + 255) / 256;
        const long cap = (long)prop.multiProcessorCount * 8;
        h->lc.agent_blocks = (int)(need < 1 ? 1 : need < cap ? need : cap);
    }
    {
        int coop = 0;
        CKC(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, h->device), "attribute");
        if (!coop) return bail(fail(SIM_E_CUDA, "device does not support cooperative launches"));
        int pbs = 0;
        CKC(eco::post_occupancy(&pbs), "occupancy");
        if (pbs < 1) return bail(fail(SIM_E_CUDA, "k_post cannot be resident"));
        h->lc.post_blocks = prop.multiProcessorCount;  // one block per SM
    }
    p.regrow_split = (S == 0 && !band) ? 1 : 0;  // agent-free benchmark grids: the regrowth as its own launch

    // K0: resources, check N0 <= empty cells, agents + weights, occupancy/lists
    CKC(eco::launch_init_resources(p, h->stream), "init resources");
    CKC(eco::launch_rebuild(p, h->stream), "rebuild");
    std::vector<int64_t> res(nw);
    CKC(cudaMemcpyAsync(res.data(), p.res_count, nw * 8, cudaMemcpyDeviceToHost, h->stream), "download");
    CKC(cudaStreamSynchronize(h->stream), "sync");
    for (size_t w = 0; w < nw && !band; ++w)  // (banded: the parent checks the whole grid)
        if ((int64_t)HW - res[w] < cfg->n_initial)
            return bail(fail(SIM_E_INVALID, "invalid field: n_initial (%d > %lld empty cells in world %zu)",
                             cfg->n_initial, (long long)((int64_t)HW - res[w]), w));
    if (S) {
        const size_t sb = eco::init_agents_scratch_bytes(p);
        void *scratch = nullptr;
        CKC(cudaMalloc(&scratch, sb), "alloc scratch");
        cudaError_t e = eco::launch_init_agents(p, band ? band->N0 : cfg->n_initial, h->stream, scratch, sb,
                                                band ? &h->bp : nullptr, h->n_own_dev);
        cudaError_t e2 = cudaStreamSynchronize(h->stream);
        cudaFree(scratch);
        CKC(e, "init agents");
        CKC(e2, "init agents sync");
    }
    CKC(eco::launch_rebuild(p, h->stream), "rebuild");
    CKC(cudaStreamSynchronize(h->stream), "sync");
    if (!band) CKC(ensure_graphs(h), "capture step graphs");
#undef CKC
    *out = h;
    return SIM_OK;
}
}  // namespace

#include "api_band.inc"

extern "C" {

sim_status sim_create(const sim_config *cfg, sim_handle *out) {
    ECO_TRACE("sim_create");
    if (cfg && cfg->abi_version == SIM_ABI_VERSION && cfg->struct_size == sizeof(sim_config) && cfg->n_bands > 1)
        return create_banded(cfg, out);
    return create_one(cfg, nullptr, out);
}

sim_status sim_destroy(sim_handle h) {
    if (!h) return SIM_OK;
    cudaSetDevice(h->device);
    destroy_all(h);
    return SIM_OK;
}

sim_status sim_step(sim_handle h, int64_t n) {
    ECO_TRACE("sim_step");
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    if (n < 0) return fail(SIM_E_INVALID, "invalid argument: n < 0");
    if ((st = check_nonfinite(h)) != SIM_OK) return st;
    if (n == 0) return SIM_OK;
    if (h->p.n_ranks > 1)
        return fail(SIM_E_STATE, "sharded handle: step with sim_step_policy, the exchange, then sim_step_post");
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    if (!h->bands.empty()) return band_step(h, n);
    CK(h, ensure_graphs(h), "capture step graphs");  // (captured already unless a capture failed)
    const bool two = n >= ECO_GRAPH_STEPS && two_step_graphs(h);
    CK(h, ensure_regrown(h), "regrow");
    int64_t i = 0;
    if (two)
        for (; i + ECO_GRAPH_STEPS <= n; i += ECO_GRAPH_STEPS) CK(h, cudaGraphLaunch(h->graph2_exec, h->stream), "graph launch");
    for (; i < n; ++i) CK(h, cudaGraphLaunch(h->graph_exec, h->stream), "graph launch");
    h->t += n;
    return SIM_OK;
}

// --- agent-sharded mode -------------------------------------------------------------
sim_status sim_shard(sim_handle h, int32_t n_ranks, int32_t rank) {
    if (h && !h->bands.empty()) return fail(SIM_E_STATE, "not available on a banded handle");
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    if (n_ranks < 1 || n_ranks > 255 || rank < 0 || rank >= n_ranks)
        return fail(SIM_E_INVALID, "invalid argument: n_ranks (1..255) / rank");
    if (n_ranks > 1 && (h->d.n_worlds != 1 || h->d.Hd != 32 || !eco::policy_supports_shard()))
        return fail(SIM_E_INVALID, "sharding needs one world, hidden = 32 and the default policy kernel");
    if (n_ranks > 1 && eco::paper_rules(h->p))
        return fail(SIM_E_INVALID, "sharding does not support the paper world's death timer / lethal walls");
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    if ((st = sync(h)) != SIM_OK) return st;
    h->p.n_ranks = n_ranks;
    h->p.rank = rank;
    h->p_ready = false;  // every own agent's P row again (a child's too: exactly b)
    CK(h, eco::launch_set_owner(h->p, h->stream), "owners");
    drop_graphs(h);  // kernel parameters changed: capture again
    return sync(h);
}

sim_status sim_step_policy(sim_handle h) {
    if (h && !h->bands.empty()) return fail(SIM_E_STATE, "not available on a banded handle");
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    if ((st = check_nonfinite(h)) != SIM_OK) return st;
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    CK(h, ensure_regrown(h), "regrow");
    CK(h, eco::launch_policy(h->p, h->lc, h->stream), "policy");
    return SIM_OK;
}

sim_status sim_step_post(sim_handle h) {
    if (h && !h->bands.empty()) return fail(SIM_E_STATE, "not available on a banded handle");
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    CK(h, eco::launch_post(h->p, h->lc, h->bar, h->stream), "post");
    h->t += 1;
    return SIM_OK;
}

sim_status sim_exchange(sim_handle h, void **mrec, size_t *mrec_bytes, void **record, size_t *record_bytes) {
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    if (!mrec || !mrec_bytes || !record || !record_bytes) return fail(SIM_E_INVALID, "invalid argument: NULL");
    *mrec = h->p.mrec_slot;
    *mrec_bytes = (size_t)h->d.S * 16;
    *record = h->p.pol_ctr;
    *record_bytes = 2 * sizeof(unsigned long long);
    return SIM_OK;
}

sim_status sim_step_timed(sim_handle h, sim_step_timing *out) {
    if (h && !h->bands.empty()) return fail(SIM_E_STATE, "not available on a banded handle");
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    if (!out) return fail(SIM_E_INVALID, "invalid argument: out (NULL)");
    if (h->p.n_ranks > 1) return fail(SIM_E_STATE, "sharded handle: sim_step_timed is not available");
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    CK(h, ensure_regrown(h), "regrow");
    CK(h, cudaEventRecord(h->ev[0], h->stream), "event");
    for (int i = 0; i < SIM_NUM_KERNELS; ++i) {
        CK(h, launch_phase(h, kTimedOrder[i]), "step kernel");
        CK(h, cudaEventRecord(h->ev[i + 1], h->stream), "event");
    }
    CK(h, cudaEventSynchronize(h->ev[SIM_NUM_KERNELS]), "event sync");
    h->t += 1;
    // split: the hh kernel made the P rows of every agent of step t+1 (children included, from
    // h = 0: exactly b), so p_children is 0 and the next step may run either way

    for (int i = 0; i < SIM_NUM_KERNELS; ++i)
        CK(h, cudaEventElapsedTime(&out->kernel_ms[kTimedOrder[i]], h->ev[i], h->ev[i + 1]), "elapsed");
    CK(h, cudaEventElapsedTime(&out->step_ms, h->ev[0], h->ev[SIM_NUM_KERNELS]), "elapsed");
    return check_nonfinite(h);
}

sim_status sim_step_graph_timed(sim_handle h, float out_ms[2]) {
    if (h && !h->bands.empty()) return fail(SIM_E_STATE, "not available on a banded handle");
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    if (!out_ms) return fail(SIM_E_INVALID, "invalid argument: out_ms (NULL)");
    if (h->p.n_ranks > 1) return fail(SIM_E_STATE, "sharded handle: sim_step_graph_timed is not available");
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    CK(h, ensure_regrown(h), "regrow");
    CK(h, cudaEventRecord(h->ev[0], h->stream), "event");
    CK(h, eco::launch_policy(h->p, h->lc, h->stream), "policy");
    CK(h, cudaEventRecord(h->ev[1], h->stream), "event");
    CK(h, eco::launch_post(h->p, h->lc, h->bar, h->stream), "post");
    if (h->p.regrow_split) CK(h, eco::launch_regrow(h->p, 0, h->stream), "regrow");
    CK(h, cudaEventRecord(h->ev[2], h->stream), "event");
    CK(h, cudaEventSynchronize(h->ev[2]), "event sync");
    h->t += 1;
    CK(h, cudaEventElapsedTime(&out_ms[0], h->ev[0], h->ev[1]), "elapsed");
    CK(h, cudaEventElapsedTime(&out_ms[1], h->ev[1], h->ev[2]), "elapsed");
    return check_nonfinite(h);
}

sim_status sim_synchronize(sim_handle h) {
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    return sync(h);
}

sim_status sim_get_state(sim_handle h, sim_state *out) {
    ECO_TRACE("sim_get_state");
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    if (!out) return fail(SIM_E_INVALID, "invalid argument: out (NULL)");
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    if (!h->bands.empty()) return band_get_state(h, out);
    if ((st = sync(h)) != SIM_OK) return st;
    const Derived &d = h->d;
    const DevParams &p = h->p;
    const size_t nw = d.n_worlds, S = d.S, HW = (size_t)d.H * d.W;
    cudaStream_t s = h->stream;
    out->t = h->t;
    if (out->resources) {
        uint8_t *tmp;
        CK(h, cudaMallocAsync(reinterpret_cast<void **>(&tmp), nw * HW, s), "alloc");
        cudaError_t e = eco::launch_unpack_resources(p, tmp, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(out->resources, tmp, nw * HW, cudaMemcpyDeviceToHost, s);
        cudaFreeAsync(tmp, s);
        CK(h, e, "resources");
    }
    auto get = [&](void *dst, const void *src, size_t bytes) -> cudaError_t {
        if (!dst || !bytes) return cudaSuccess;
        return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
    };
    CK(h, get(out->alive, p.alive, nw * S), "alive");
    CK(h, get(out->cell, p.cell, nw * S * 4), "cell");
    CK(h, get(out->energy, p.energy, nw * S * 4), "energy");
    CK(h, get(out->age, p.age, nw * S * 4), "age");
    CK(h, get(out->repr, p.repr, nw * S * 4), "repr");
    CK(h, get(out->low, p.low, nw * S * 4), "low");
    CK(h, get(out->last_action, p.last_action, nw * S), "last_action");
    CK(h, get(out->ate, p.ate, nw * S), "ate");
    CK(h, get(out->h, p.h, nw * S * d.Hd * 4), "h");
    CK(h, get(out->c, p.c, nw * S * d.Hd * 4), "c");
    if (out->logits && S) {
        float *tmp;
        CK(h, cudaMallocAsync(reinterpret_cast<void **>(&tmp), nw * S * 5 * 4, s), "alloc");
        cudaError_t e = eco::launch_logits_restride(tmp, 5, p.logits, eco::LOGIT_STRIDE, nw * S, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(out->logits, tmp, nw * S * 5 * 4, cudaMemcpyDeviceToHost, s);
        cudaFreeAsync(tmp, s);
        CK(h, e, "logits");
    }
    if (out->weights && S) {
        const size_t total_agents = nw * S;
        const size_t chunk = ((size_t)1 << 26) / (size_t)d.P > 0 ? ((size_t)1 << 26) / (size_t)d.P : 1;
        float *tmp;
        CK(h, cudaMallocAsync(reinterpret_cast<void **>(&tmp), chunk * d.P * 4, s), "alloc");
        cudaError_t e = cudaSuccess;
        for (size_t a0 = 0; a0 < total_agents && e == cudaSuccess; a0 += chunk) {
            const size_t n = (total_agents - a0) < chunk ? total_agents - a0 : chunk;
            e = eco::launch_weights_to_canon(p, tmp, a0, n, s);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(out->weights + a0 * d.P, tmp, n * d.P * 4, cudaMemcpyDeviceToHost, s);
        }
        cudaFreeAsync(tmp, s);
        CK(h, e, "weights");
    }
    return sync(h);
}

sim_status sim_set_state(sim_handle h, const sim_state *in) {
    ECO_TRACE("sim_set_state");
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    if (!in) return fail(SIM_E_INVALID, "invalid argument: in (NULL)");
    if (in->t < 0 || in->t >= ((int64_t)1 << 32)) return fail(SIM_E_INVALID, "invalid field: t");
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    if (!h->bands.empty()) return band_set_state(h, in);
    if ((st = sync(h)) != SIM_OK) return st;
    const Derived &d = h->d;
    DevParams &p = h->p;
    const size_t nw = d.n_worlds, S = d.S, HW = (size_t)d.H * d.W;
    cudaStream_t s = h->stream;
    // host-side validation on the merged view (device values where a field is NULL)
    std::vector<uint8_t> live_merged;
    if (S) {
        std::vector<uint8_t> &alive = live_merged;
        alive.resize(nw * S);
        std::vector<int32_t> cell(nw * S);
        if (in->alive) memcpy(alive.data(), in->alive, nw * S);
        else CK(h, cudaMemcpy(alive.data(), p.alive, nw * S, cudaMemcpyDeviceToHost), "download");
        if (in->cell) memcpy(cell.data(), in->cell, nw * S * 4);
        else CK(h, cudaMemcpy(cell.data(), p.cell, nw * S * 4, cudaMemcpyDeviceToHost), "download");
        std::vector<uint8_t> seen(HW);
        for (size_t w = 0; w < nw; ++w) {
            std::fill(seen.begin(), seen.end(), 0);
            for (size_t i = 0; i < S; ++i) {
                if (!alive[w * S + i]) continue;
                const int32_t c = cell[w * S + i];
                if (c < 0 || (size_t)c >= HW) return fail(SIM_E_INVALID, "invalid field: cell (out of range, world %zu slot %zu)", w, i);
                if (seen[c] && !d.coloc)
                    return fail(SIM_E_INVALID, "invalid field: cell (two agents on cell %d, world %zu)", c, w);
                seen[c] = 1;
            }
        }
    }
    // weights: only the live slots' rows are imported (a dead slot's weights are unspecified,
    // sim.h), gathered into the device layout in a persistent staging buffer and checked for
    // non-finite values there; the handle's weights change only after the check passed.
    // Mapped (page-locked) caller memory is read in place by the gather kernel; pageable
    // memory is first copied run by run (runs of consecutive live slots) to the device.
    int n_live = 0;
    if (in->weights && S) {
        if (nw * S >= ((size_t)1 << 31)) return fail(SIM_E_INVALID, "invalid argument: n_worlds * slots too large");
        for (size_t g = 0; g < nw * S; ++g) n_live += live_merged[g] ? 1 : 0;
    }
    if (n_live > 0) {
        std::vector<int32_t> live;
        live.reserve(n_live);
        for (size_t g = 0; g < nw * S; ++g)
            if (live_merged[g]) live.push_back((int32_t)g);
        CK(h, cudaMemcpyAsync(h->live_dev, live.data(), (size_t)n_live * 4, cudaMemcpyHostToDevice, s), "live list");
        CK(h, ensure_rows(&h->wstage, &h->wstage_rows, (size_t)n_live, (size_t)d.Pd), "alloc staging");
        const float *src = nullptr;
        bool by_slot = false;
        cudaPointerAttributes pa{};
        // page-locked caller memory: read in place by the gather kernel (zero-copy), unless the
        // live rows form few long runs, which DMA copies move faster (ECO_SETSTATE_ZC=1/0 forces)
        int runs = 1;
        for (int k = 1; k < n_live; ++k) runs += live[k] != live[k - 1] + 1;
        static const char *zc_env = getenv("ECO_SETSTATE_ZC");
        const bool zc_pref = zc_env ? zc_env[0] == '1' : runs > 64;
        if (zc_pref && cudaPointerGetAttributes(&pa, in->weights) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
            pa.devicePointer) {
            src = static_cast<const float *>(pa.devicePointer);
            by_slot = true;
        } else {
            cudaGetLastError();
            CK(h, ensure_rows(&h->wcanon, &h->wcanon_rows, (size_t)n_live, (size_t)d.P), "alloc staging");
            for (int k0 = 0; k0 < n_live;) {
                int k1 = k0 + 1;
                while (k1 < n_live && live[k1] == live[k1 - 1] + 1) ++k1;
                CK(h, cudaMemcpyAsync(h->wcanon + (size_t)k0 * d.P, in->weights + (size_t)live[k0] * d.P,
                                      (size_t)(k1 - k0) * d.P * 4, cudaMemcpyHostToDevice, s), "weights");
                k0 = k1;
            }
            src = h->wcanon;
        }
        *reinterpret_cast<volatile int32_t *>(h->bad_host) = 0;
        int32_t *bad_dev = nullptr;
        CK(h, cudaHostGetDevicePointer(reinterpret_cast<void **>(&bad_dev), h->bad_host, 0), "cudaHostGetDevicePointer");
        CK(h, eco::launch_weights_gather(p, src, by_slot, h->live_dev, n_live, h->wstage, bad_dev, s), "weights gather");
        CK(h, cudaStreamSynchronize(s), "sync");
        if (*reinterpret_cast<volatile int32_t *>(h->bad_host))
            return fail(SIM_E_INVALID, "invalid field: weights (non-finite in a live slot)");
    }
    if (!in->resources && ((in->t ^ h->t) & 1)) {
        // the current resource plane is selected by step parity: carry it over
        uint32_t *from = (h->t & 1) ? p.plane1 : p.plane0;
        uint32_t *to = (in->t & 1) ? p.plane1 : p.plane0;
        CK(h, cudaMemcpyAsync(to, from, nw * d.pw * 4, cudaMemcpyDeviceToDevice, s), "plane");
    }
    std::vector<int64_t> tv(nw, in->t);
    CK(h, cudaMemcpyAsync(p.t, tv.data(), nw * 8, cudaMemcpyHostToDevice, s), "t");
    h->t = in->t;
    if (in->resources) {
        CK(h, cudaMemcpyAsync(h->res_bytes, in->resources, nw * HW, cudaMemcpyHostToDevice, s), "resources");
        CK(h, eco::launch_pack_resources(p, h->res_bytes, s), "resources");
    }
    auto put = [&](void *dst, const void *src, size_t bytes) -> cudaError_t {
        if (!src || !bytes) return cudaSuccess;
        return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
    };
    CK(h, put(p.alive, in->alive, nw * S), "alive");
    CK(h, put(p.cell, in->cell, nw * S * 4), "cell");
    CK(h, put(p.energy, in->energy, nw * S * 4), "energy");
    CK(h, put(p.age, in->age, nw * S * 4), "age");
    CK(h, put(p.repr, in->repr, nw * S * 4), "repr");
    if (in->low) CK(h, put(p.low, in->low, nw * S * 4), "low");
    else CK(h, cudaMemsetAsync(p.low, 0, nw * S * 4, s), "memset");  // (a state without the timer: 0)
    CK(h, put(p.last_action, in->last_action, nw * S), "last_action");
    CK(h, put(p.ate, in->ate, nw * S), "ate");
    CK(h, put(p.h, in->h, nw * S * d.Hd * 4), "h");
    CK(h, put(p.c, in->c, nw * S * d.Hd * 4), "c");
    if (in->logits && S) {
        CK(h, ensure_rows(&h->lstage, &h->lstage_n, nw * S, 5), "alloc staging");
        CK(h, cudaMemcpyAsync(h->lstage, in->logits, nw * S * 5 * 4, cudaMemcpyHostToDevice, s), "logits");
        CK(h, eco::launch_logits_restride(p.logits, eco::LOGIT_STRIDE, h->lstage, 5, nw * S, s), "logits");
    }
    if (n_live > 0) CK(h, eco::launch_weights_scatter(p, h->wstage, h->live_dev, n_live, s), "weights scatter");
    // scratch and derived structures
    if (S) {
        CK(h, cudaMemsetAsync(p.claim, 0, nw * HW * 8, s), "memset");
        CK(h, cudaMemsetAsync(p.bkey, 0, nw * HW * 8, s), "memset");
    }
    CK(h, cudaMemsetAsync(p.bbits, 0, 2 * nw * d.pw * 4, s), "memset");
    CK(h, cudaMemsetAsync(p.log, 0, (size_t)d.log_cap * nw * sizeof(sim_step_record), s), "memset");
    CK(h, cudaMemsetAsync(p.totals, 0, 8 * 8, s), "memset");
    CK(h, cudaMemsetAsync(p.gr_seen, 0, nw * S, s), "memset");  // greediness counts from here on
    CK(h, cudaMemsetAsync(p.gr_ate, 0, nw * S, s), "memset");
    CK(h, cudaMemsetAsync(p.gr_T, 0, nw * S * 4, s), "memset");
    CK(h, cudaMemsetAsync(p.gr_C, 0, nw * S * 4, s), "memset");
    CK(h, cudaMemsetAsync(p.le, 0, nw * (size_t)p.le_cap * 16, s), "memset");
    CK(h, eco::launch_rebuild(p, s), "rebuild");
    CK(h, eco::launch_set_owner(p, s), "owners");
    CK(h, cudaMemsetAsync(p.pol_ctr, 0, 2 * sizeof(unsigned long long), s), "memset");
    CK(h, cudaMemsetAsync(h->bar + 3, 0, 2 * sizeof(unsigned long long), s), "memset");  // window-end counters
    h->regrown_ahead = false;
    h->p_ready = false;
    return sync(h);
}

sim_status sim_set_forced_actions(sim_handle h, const uint8_t *act) {
    if (h && !h->bands.empty()) return fail(SIM_E_STATE, "not available on a banded handle");
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    const size_t n = (size_t)h->d.n_worlds * h->d.S;
    int32_t on = act ? 1 : 0;
    if (act) {
        for (size_t i = 0; i < n; ++i)
            if (act[i] > 4 && act[i] != 255) return fail(SIM_E_INVALID, "invalid argument: act (values 0..4 or 255)");
        if (n) CK(h, cudaMemcpyAsync(h->forced_dev, act, n, cudaMemcpyHostToDevice, h->stream), "forced");
    }
    CK(h, cudaMemcpyAsync(h->forced_on_dev, &on, 4, cudaMemcpyHostToDevice, h->stream), "forced flag");
    CK(h, cudaStreamSynchronize(h->stream), "sync");
    return SIM_OK;
}

namespace {
sim_status step_log_copy(sim_handle h, int64_t first, int64_t n, sim_step_record *out, bool wait) {
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    if (n < 0 || (n > 0 && !out)) return fail(SIM_E_INVALID, "invalid argument: n/out");
    if (first < 0 || first + n > h->t || first < h->t - (h->d.log_cap - 1))
        return fail(SIM_E_INVALID, "invalid argument: steps [%lld, %lld) not in the log (t = %lld, capacity %d)",
                    (long long)first, (long long)(first + n), (long long)h->t, h->d.log_cap);
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    if (!h->bands.empty()) return n ? band_step_log(h, first, n, out) : SIM_OK;  // summed over the bands
    if (wait && (st = sync(h)) != SIM_OK) return st;
    const size_t nw = h->d.n_worlds;
    // the ring is contiguous by step: [first, first+n) is at most two runs (split at the wrap)
    int64_t done = 0;
    while (done < n) {
        const int64_t slot = (first + done) % h->d.log_cap;
        const int64_t run = std::min<int64_t>(n - done, h->d.log_cap - slot);
        CK(h, cudaMemcpyAsync(out + done * nw, h->p.log + (size_t)slot * nw, (size_t)run * nw * sizeof(sim_step_record),
                              cudaMemcpyDeviceToHost, h->stream), "log");
        done += run;
    }
    return wait ? sync(h) : SIM_OK;
}
}  // namespace

sim_status sim_get_step_log(sim_handle h, int64_t first, int64_t n, sim_step_record *out) {
    return step_log_copy(h, first, n, out, true);
}

sim_status sim_get_step_log_async(sim_handle h, int64_t first, int64_t n, sim_step_record *out) {
    return step_log_copy(h, first, n, out, false);
}

sim_status sim_set_record_mirror(sim_handle h, sim_step_record *host, int64_t capacity) {
    if (h && !h->bands.empty()) return fail(SIM_E_STATE, "not available on a banded handle");
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    if ((st = sync(h)) != SIM_OK) return st;
    if (!host) {
        h->p.rec_mirror = nullptr;
        h->p.mirror_cap = 0;
    } else {
        if (capacity < 1 || (capacity & (capacity - 1)) != 0 || capacity > (1 << 30))
            return fail(SIM_E_INVALID, "invalid argument: capacity (a power of two)");
        void *dev = nullptr;
        if (cudaHostGetDevicePointer(&dev, host, 0) != cudaSuccess) {
            cudaGetLastError();
            return fail(SIM_E_INVALID, "invalid argument: host (not page-locked, mapped memory)");
        }
        h->p.rec_mirror = static_cast<sim_step_record *>(dev);
        h->p.mirror_cap = (int32_t)capacity;
    }
    drop_graphs(h);  // kernel parameters changed: capture again, now (not inside a later sim_step)
    CK(h, ensure_graphs(h), "capture step graphs");
    return SIM_OK;
}

sim_status sim_get_phase_ns(sim_handle h, int64_t *out, int32_t reset) {
    if (h && !h->bands.empty()) return fail(SIM_E_STATE, "not available on a banded handle");
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    if (out)
        CK(h, cudaMemcpyAsync(out, h->p.phase_ns, (reset < 0 ? PHASE_WORDS : SIM_NUM_POST_PHASES) * 8,
                              cudaMemcpyDeviceToHost, h->stream),
           "phase clock");
    if (reset > 0) CK(h, cudaMemsetAsync(h->p.phase_ns, 0, PHASE_WORDS * 8, h->stream), "phase clock");
    return sync(h);
}

sim_status sim_get_move_hist(sim_handle h, int64_t first, int64_t n, int32_t *out) {
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    if (n < 0 || (n > 0 && !out)) return fail(SIM_E_INVALID, "invalid argument: n/out");
    if (!h->bands.empty()) {  // summed over the local bands
        std::vector<int32_t> tmp((size_t)n * SIM_MOVE_BINS);
        memset(out, 0, (size_t)n * SIM_MOVE_BINS * 4);
        for (sim_ctx *b : h->bands) {
            if ((st = sim_get_move_hist(b, first, n, tmp.data())) != SIM_OK) return st;
            for (size_t i = 0; i < tmp.size(); ++i) out[i] += tmp[i];
        }
        return SIM_OK;
    }
    const int64_t done = h->t / SIM_MOVE_WINDOW;  // complete windows
    if (first < 0 || first + n > done || first < done - h->p.mv_cap)
        return fail(SIM_E_INVALID, "invalid argument: windows [%lld, %lld) not kept (complete windows %lld, capacity %d)",
                    (long long)first, (long long)(first + n), (long long)done, h->p.mv_cap);
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    if ((st = sync(h)) != SIM_OK) return st;
    const size_t nw = h->d.n_worlds;
    for (int64_t i = 0; i < n; ++i)
        for (size_t w = 0; w < nw; ++w)
            CK(h, cudaMemcpyAsync(out + (i * nw + w) * SIM_MOVE_BINS,
                                  h->p.mv_hist + (w * h->p.mv_cap + (size_t)((first + i) & (h->p.mv_cap - 1))) * SIM_MOVE_BINS,
                                  SIM_MOVE_BINS * 4, cudaMemcpyDeviceToHost, h->stream), "move histogram");
    return sync(h);
}

sim_status sim_get_policy_actions(sim_handle h, uint8_t *out) {
    if (h && !h->bands.empty()) return fail(SIM_E_STATE, "not available on a banded handle");
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    if (!out) return fail(SIM_E_INVALID, "invalid argument: NULL");
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    if ((st = sync(h)) != SIM_OK) return st;
    const size_t n = (size_t)h->d.n_worlds * h->d.S;
    if (n) CK(h, cudaMemcpyAsync(out, h->p.own_act, n, cudaMemcpyDeviceToHost, h->stream), "policy actions");
    return sync(h);
}

sim_status sim_get_greediness(sim_handle h, int32_t *T_r, int32_t *C_r) {
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    if (!T_r || !C_r) return fail(SIM_E_INVALID, "invalid argument: NULL");
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    if (!h->bands.empty()) return band_get_greediness(h, T_r, C_r);
    if ((st = sync(h)) != SIM_OK) return st;
    const size_t n = (size_t)h->d.n_worlds * h->d.S;
    CK(h, cudaMemcpyAsync(T_r, h->p.gr_T, n * 4, cudaMemcpyDeviceToHost, h->stream), "greediness");
    CK(h, cudaMemcpyAsync(C_r, h->p.gr_C, n * 4, cudaMemcpyDeviceToHost, h->stream), "greediness");
    return sync(h);
}

sim_status sim_get_life_windows(sim_handle h, int64_t first, int64_t n, int64_t *deaths, int64_t *age_sum) {
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    if (n < 0 || (n > 0 && (!deaths || !age_sum))) return fail(SIM_E_INVALID, "invalid argument: n/out");
    const int64_t done = h->t / SIM_LIFE_WINDOW;  // complete windows
    const int cap = h->bands.empty() ? h->p.le_cap : h->bands[0]->p.le_cap;
    if (first < 0 || first + n > done || first < done - cap)
        return fail(SIM_E_INVALID, "invalid argument: windows [%lld, %lld) not kept (complete windows %lld, capacity %d)",
                    (long long)first, (long long)(first + n), (long long)done, cap);
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    if ((st = sync(h)) != SIM_OK) return st;
    const size_t nw = h->d.n_worlds;
    memset(deaths, 0, (size_t)n * nw * 8);
    memset(age_sum, 0, (size_t)n * nw * 8);
    std::vector<sim_ctx *> parts;
    if (h->bands.empty()) parts.push_back(h);
    else parts = h->bands;
    for (sim_ctx *b : parts)
        for (int64_t i = 0; i < n; ++i)
            for (size_t w = 0; w < nw; ++w) {
                unsigned long long v[2];
                CK(h, cudaMemcpy(v, b->p.le + (w * b->p.le_cap + (size_t)((first + i) & (b->p.le_cap - 1))) * 2, 16,
                                 cudaMemcpyDeviceToHost), "life windows");
                deaths[i * nw + w] += (int64_t)v[0];
                age_sum[i * nw + w] += (int64_t)v[1];
            }
    return SIM_OK;
}

sim_status sim_get_totals(sim_handle h, sim_totals *out) {
    sim_status st = check_handle(h);
    if (st != SIM_OK) return st;
    if (!out) return fail(SIM_E_INVALID, "invalid argument: out (NULL)");
    if (!h->bands.empty()) {  // summed over the local bands (steps counted once)
        *out = sim_totals{};
        for (sim_ctx *b : h->bands) {
            sim_totals tb;
            if ((st = sim_get_totals(b, &tb)) != SIM_OK) return st;
            out->steps = tb.steps;
            out->agent_steps += tb.agent_steps;
            out->cell_updates += tb.cell_updates;
            out->births += tb.births;
            out->deaths += tb.deaths;
            out->eaten += tb.eaten;
            out->grown += tb.grown;
        }
        return SIM_OK;
    }
    CK(h, cudaSetDevice(h->device), "cudaSetDevice");
    unsigned long long v[8];
    CK(h, cudaMemcpyAsync(v, h->p.totals, sizeof v, cudaMemcpyDeviceToHost, h->stream), "totals");
    if ((st = sync(h)) != SIM_OK) return st;
    out->steps = (int64_t)v[0];
    out->agent_steps = (int64_t)v[1];
    out->cell_updates = (int64_t)v[2];
    out->births = (int64_t)v[3];
    out->deaths = (int64_t)v[4];
    out->eaten = (int64_t)v[5];
    out->grown = (int64_t)v[6];
    return SIM_OK;
}

}  // extern "C"
