// policy_cnn.cuh — k_policy_cnn_blk: steps a2 + a3 (+ the claim half of a4) for network 1,
// the paper's own agent network (App. B.5).
// Included by step.cu inside namespace eco (it uses the step's epilogue helpers).
//
//   window   15x15x3: resources R' after regrowth, agents O_t (incl.
//            self), walls = off the grid; HWC
//   conv1    3x3, stride 2, SAME (pad 1): 15x15x3 -> 8x8x4      (no activation, R41)
//   pool1    2x2 average, stride 1, VALID: -> 7x7x4
//   conv2    3x3, stride 2, SAME (pad 1): -> 4x4x8
//   pool2    -> 3x3x8 = 72; e = [72, one-hot previous action (5), ate (1)] = 78
//   LSTM(4)  z = W_ih e + W_hh h + b, gates (i, f, g, o)
//   dense    [e, h'] (82) -> 8, tanh; dense 8 -> 5 logits
//   action   softmax(50 logits) sampled by inverse CDF with u = draw(ACTION, t, cell).x 2^-32
//            (R38), in fp64 from the fp32 logits; near-tie when |u - CDF| < 1e-4
//
// One block per agent (2,445 parameters, 13.5 k multiply-adds: a per-agent network is a
// batched GEMV-like chain of tiny layers with different weights per agent, no dense
// contraction for the tensor cores).  The agent's whole parameter row (Pd = 2,464 floats,
// 9.9 KB, canonical order = device order) is staged into the block's shared memory with
// 16-B cp.async while the window's rows are fetched from the bit planes; every layer then
// reads its weights from shared memory and its inputs from the previous layer's
// shared-memory tile.  The resource and wall inputs of conv1 are 0/1, so conv1 adds weights
// where they are set.
constexpr int CNN_PD = 2464;                 // device row: 2445 parameters padded to 32 floats
constexpr int CNN_WO = 15, CNN_R = 7;
// canonical / device offsets of network 1 (sim.h)
constexpr int CN_C1W = 0, CN_C1B = 108, CN_C2W = 112, CN_C2B = 400, CN_WIH = 408, CN_WHH = 1656, CN_B = 1720,
              CN_WD = 1736, CN_BD = 2392, CN_WO = 2400, CN_BO = 2440, CN_P = 2445;
static_assert(CN_BO + 5 == CN_P && CN_P <= CNN_PD && CNN_PD % 32 == 0, "network-1 layout");
// the agent's shared memory: the weights (floats), then fp64 tiles: conv1 out (8x8x4), pool1
// (7x7x4), conv2 out (4x4x8), e ++ h' (78 + 4, padded); window rows (R rows 0..14, O rows
// 16..30) as words
constexpr int CS_W_BYTES = CNN_PD * 4;
constexpr int CS_A1 = 0, CS_P1 = CS_A1 + 256, CS_A2 = CS_P1 + 196, CS_E = CS_A2 + 128, CS_D_END = CS_E + 84;  // doubles
constexpr int CS_ROWS_BYTES = 32 * 4;
constexpr int CS_CNT_BYTES = 228 * 4;  // the agent channel: agents per window cell (15 x 15)
constexpr int CS_TOTAL_BYTES = CS_W_BYTES + CS_D_END * 8 + CS_ROWS_BYTES + CS_CNT_BYTES;
static_assert(CS_W_BYTES % 16 == 0 && CS_TOTAL_BYTES % 16 == 0, "16-B aligned slices");

__device__ __forceinline__ double sigmoid_d(double z) { return 1.0 / (1.0 + exp(-z)); }

// Arithmetic: every sum, pool, gate and activation in fp64 from the fp32 weights and
// inputs (the oracle's precision; B200's FP64 units make this ~4k fp64 FMAs per agent
// cheap beside the weight stream), h', c' and the logits rounded to fp32 once for storage,
// the softmax and sampling in fp64 from the fp32 logits.  Only the summation order differs
// from the oracle's, so the stored values agree to about one fp32 rounding even for
// weights far larger than the paper's.
// ---------------------------------------------------------------------------------------
// k_policy_cnn_blk: one BLOCK of CNN_BLK_THREADS per agent.  At the paper world's populations
// (a few hundred agents, far fewer than the GPU's warp slots) the per-agent chain of
// dependent fp64 operations is the step's critical path, so every layer is spread over 4
// warps (one warp per agent -- the first version, in git history -- took 19.5 instead of
// 16.5 us per launch): conv1 2 outputs per thread, conv2 1 output (36 FMAs) per thread,
// the LSTM's 16 rows over 8 threads each, dense 8 over 16 threads each, the 5 exponentials of
// the softmax on 5 threads.  Sums are split into fixed contiguous parts reduced in a fixed
// order (fp64; the stored h', c', logits stay within an fp32 rounding of the oracle's).
constexpr int CNN_BLK_THREADS = 128;

__global__ void __launch_bounds__(CNN_BLK_THREADS) k_policy_cnn_blk(DevParams p) {
#if ECO_STEP2_PDL
    // inside a multi-step graph the policy is a programmatic dependent of the previous step's
    // post-policy kernel: wait for it (a no-op for an ordinary launch)
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    extern __shared__ __align__(1024) unsigned char cnn_smem_raw[];
    __shared__ double s_z[16], s_d[8], s_ex[5];
    __shared__ unsigned s_nnz, s_seen;
    __shared__ int s_bad;
    constexpr unsigned FULL = 0xffffffffu;
    const int tid = threadIdx.x, lane = tid & 31;
    unsigned char *base = cnn_smem_raw;
    float *sw = reinterpret_cast<float *>(base);
    double *sd = reinterpret_cast<double *>(base + CS_W_BYTES);
    double *a1 = sd + CS_A1, *p1 = sd + CS_P1, *a2 = sd + CS_A2, *e = sd + CS_E;
    uint32_t *rows = reinterpret_cast<uint32_t *>(base + CS_W_BYTES + CS_D_END * 8);
    int32_t *cnt = reinterpret_cast<int32_t *>(base + CS_W_BYTES + CS_D_END * 8 + CS_ROWS_BYTES);
    step_housekeeping(p);
    PolicyCounters ctr;
    const long total = (long)p.n_worlds * p.S;
    for (long v = blockIdx.x; v < total; v += gridDim.x) {  // block-uniform
        const int w = (int)(v / p.S);
        const int i = (int)(v - (long)w * p.S);
        const int64_t t = p.t[w];
        if (i >= *count_of(p, t, w)) continue;
        const int slot = list_of(p, t, w)[i];
        ECO_CHECK(slot >= 0 && slot < p.S);
        const size_t gs = (size_t)w * p.S + slot;
        const float *Wg = p.weights + gs * (size_t)CNN_PD;
        for (int q = tid; q < CNN_PD / 4; q += CNN_BLK_THREADS) cp_async16(sw + 4 * q, Wg + 4 * q, 0);
        cp_commit();
        const int cellv = p.cell[gs];
        ECO_CHECK(cellv >= 0 && cellv < p.H * p.W);
        const int y = row_of(p, cellv), x = cellv - y * p.W;
        if (tid < 32) {  // rows: R' rows 0..14 on lanes 0..14, O rows on lanes 16..30
            const int rr = lane & 15, yy = y - CNN_R + rr;
            uint32_t bits = 0u;
            if (rr < CNN_WO && yy >= 0 && yy < p.H) {
                const uint32_t *pl = lane < 16 ? plane_next(p, t) + (size_t)w * plane_words(p)
                                               : p.occ + (size_t)w * plane_words(p);
                bits = row_bits(pl + (size_t)yy * p.WW, p.WW, x - CNN_R, CNN_WO);
            }
            rows[lane] = bits;
        }
        if (tid == 0) {
            s_nnz = 0u;
            s_seen = 0u;
            s_bad = 0;
        }
        const float hold = tid < 4 ? p.h[gs * 4 + tid] : 0.f;
        const float cold = tid < 4 ? p.c[gs * 4 + tid] : 0.f;
        const int last = p.last_action[gs], ate = p.ate[gs];
        __syncthreads();
        int occupied = 0;
        for (int idx = tid; idx < CNN_WO * CNN_WO; idx += CNN_BLK_THREADS) {  // the agent channel (R39, R44)
            const int row = idx / CNN_WO, col = idx - row * CNN_WO;
            const int yy = y - CNN_R + row, xx = x - CNN_R + col;
            int n = 0;
            if (p.coloc) {
                if (yy >= 0 && yy < p.H && xx >= 0 && xx < p.W) n = p.ncount[(size_t)w * p.H * p.W + (size_t)yy * p.W + xx];
            } else {
                n = (int)((rows[16 + row] >> col) & 1u);
            }
            cnt[idx] = n;
            occupied += n > 0;
        }
        cp_wait<0>();
        __syncthreads();
        {  // conv1: position tid & 63, features 2 (tid >> 6) .. + 1
            const int pos = tid & 63, oy = pos >> 3, ox = pos & 7, f0 = (tid >> 6) * 2;
            double acc0 = (double)sw[CN_C1B + f0], acc1 = (double)sw[CN_C1B + f0 + 1];
#pragma unroll
            for (int ky = 0; ky < 3; ++ky) {
                const int iy = 2 * oy + ky - 1;
                if (iy < 0 || iy >= CNN_WO) continue;
                const uint32_t rb = rows[iy];
                const bool row_on = (y - CNN_R + iy) >= 0 && (y - CNN_R + iy) < p.H;
#pragma unroll
                for (int kx = 0; kx < 3; ++kx) {
                    const int ix = 2 * ox + kx - 1;
                    if (ix < 0 || ix >= CNN_WO) continue;
                    const bool r = (rb >> ix) & 1u;
                    const int o = cnt[iy * CNN_WO + ix];
                    const bool wall = !(row_on && (x - CNN_R + ix) >= 0 && (x - CNN_R + ix) < p.W);
                    const float *wk0 = sw + CN_C1W + f0 * 27 + (ky * 3 + kx) * 3, *wk1 = wk0 + 27;
                    if (r) {
                        acc0 += (double)wk0[0];
                        acc1 += (double)wk1[0];
                    }
                    if (o) {
                        acc0 = fma((double)o, (double)wk0[1], acc0);
                        acc1 = fma((double)o, (double)wk1[1], acc1);
                    }
                    if (wall) {
                        acc0 += (double)wk0[2];
                        acc1 += (double)wk1[2];
                    }
                }
            }
            a1[pos * 4 + f0] = acc0;
            a1[pos * 4 + f0 + 1] = acc1;
        }
        __syncthreads();
        for (int idx = tid; idx < 196; idx += CNN_BLK_THREADS) {  // pool1
            const int py = idx / 28, rem = idx - py * 28, px = rem >> 2, f = rem & 3;
            const double *b0 = a1 + (py * 8 + px) * 4 + f;
            p1[idx] = (((b0[0] + b0[4]) + b0[32]) + b0[36]) / 4.0;
        }
        __syncthreads();
        {  // conv2: position tid >> 3 (4x4), feature tid & 7
            const int q = tid >> 3, oy = q >> 2, ox = q & 3, g = tid & 7;
            double acc = (double)sw[CN_C2B + g];
#pragma unroll
            for (int ky = 0; ky < 3; ++ky) {
                const int iy = 2 * oy + ky - 1;
                if (iy < 0 || iy >= 7) continue;
#pragma unroll
                for (int kx = 0; kx < 3; ++kx) {
                    const int ix = 2 * ox + kx - 1;
                    if (ix < 0 || ix >= 7) continue;
                    const double *in = p1 + (iy * 7 + ix) * 4;
                    const float4 wk = *reinterpret_cast<const float4 *>(sw + CN_C2W + (g * 9 + ky * 3 + kx) * 4);
                    acc = fma((double)wk.x, in[0], acc);
                    acc = fma((double)wk.y, in[1], acc);
                    acc = fma((double)wk.z, in[2], acc);
                    acc = fma((double)wk.w, in[3], acc);
                }
            }
            a2[q * 8 + g] = acc;
        }
        __syncthreads();
        if (tid < 72) {  // pool2 -> e[0..72)
            const int py = tid / 24, rem = tid - py * 24, px = rem >> 3, g = rem & 7;
            const double *b0 = a2 + (py * 4 + px) * 8 + g;
            e[tid] = (((b0[0] + b0[8]) + b0[32]) + b0[40]) / 4.0;
        } else if (tid < 77) {
            e[tid] = tid - 72 == last ? 1.0 : 0.0;  // one-hot previous action
        } else if (tid == 77) {
            e[77] = ate ? 1.0 : 0.0;
        } else if (tid >= 78 && tid < 82) {
            e[tid] = (double)p.h[gs * 4 + (tid - 78)];  // h (the LSTM's recurrent input, slots 78..81)
        }
        __syncthreads();
        {  // LSTM gate rows: row tid >> 3, inputs [11 (tid & 7), + 11) of [e (78), h (4)]
            const int r = tid >> 3, k = tid & 7, j0 = k * 11, j1 = j0 + 11 < 82 ? j0 + 11 : 82;
            double s = 0.0;
            for (int j = j0; j < j1; ++j)
                s = fma(j < 78 ? (double)sw[CN_WIH + r * 78 + j] : (double)sw[CN_WHH + r * 4 + (j - 78)], e[j], s);
            s += __shfl_xor_sync(FULL, s, 1);
            s += __shfl_xor_sync(FULL, s, 2);
            s += __shfl_xor_sync(FULL, s, 4);
            if (k == 0) s_z[r] = s + (double)sw[CN_B + r];
        }
        __syncthreads();
        if (tid < 4) {  // unit tid: i = row tid, f = 4 + tid, g = 8 + tid, o = 12 + tid
            const double cnd = sigmoid_d(s_z[4 + tid]) * (double)cold + sigmoid_d(s_z[tid]) * tanh(s_z[8 + tid]);
            const float cn = (float)cnd;
            const float hn = (float)(sigmoid_d(s_z[12 + tid]) * tanh(cnd));
            p.h[gs * 4 + tid] = hn;
            p.c[gs * 4 + tid] = cn;
            e[78 + tid] = (double)hn;  // "we concatenate the embedding with the output of the LSTM"
            if (!isfinite(hn) || !isfinite(cn)) s_bad = 1;
        }
        (void)hold;
        __syncthreads();
        {  // dense 82 -> 8 with tanh: row tid >> 4, inputs [6 (tid & 15), + 6)
            const int r = tid >> 4, k = tid & 15, j0 = k * 6, j1 = j0 + 6 < 82 ? j0 + 6 : 82;
            double s = 0.0;
            for (int j = j0; j < j1; ++j) s = fma((double)sw[CN_WD + r * 82 + j], e[j], s);
            s += __shfl_xor_sync(FULL, s, 1);
            s += __shfl_xor_sync(FULL, s, 2);
            s += __shfl_xor_sync(FULL, s, 4);
            s += __shfl_xor_sync(FULL, s, 8);
            if (k == 0) s_d[r] = tanh(s + (double)sw[CN_BD + r]);
        }
        // window counters: active inputs (R bits and occupied cells), a resource in view
        {
            const uint32_t rbits = tid < CNN_WO ? rows[tid] : 0u;
            const unsigned nn = __reduce_add_sync(FULL, (unsigned)(__popc(rbits) + occupied));
            const unsigned sn = __reduce_or_sync(FULL, rbits);
            if (lane == 0) {
                atomicAdd(&s_nnz, nn);
                atomicOr(&s_seen, sn);
            }
        }
        __syncthreads();
        float lgv = 0.f;
        if (tid < 5) {  // logits, and their softmax exponentials, on 5 threads
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) s = fma((double)sw[CN_WO + tid * 8 + k], s_d[k], s);
            lgv = (float)(s + (double)sw[CN_BO + tid]);
        }
        float lg[5];
#pragma unroll
        for (int a = 0; a < 5; ++a) lg[a] = __shfl_sync(FULL, lgv, a);
        double zmax = -INFINITY;
#pragma unroll
        for (int a = 0; a < 5; ++a) zmax = fmax(zmax, 50.0 * (double)lg[a]);
        if (tid < 5) s_ex[tid] = exp(50.0 * (double)lgv - zmax);
        __syncthreads();
        if (tid == 0) {
            // softmax(50 logits) sampled by inverse CDF (fp64 from the fp32 logits, R38)
            bool bad = s_bad != 0;
            double S = 0.0;
#pragma unroll
            for (int a = 0; a < 5; ++a) {
                bad = bad || !isfinite(lg[a]);
                p.logits[gs * LOGIT_STRIDE + a] = lg[a];
                S += s_ex[a];
            }
            // keyed by the cell (unique under exclusive occupancy, R9), by the slot under co-location (R47)
            const uint4 d = draw4(p.seeds[w], PURPOSE_ACTION, (uint32_t)t, (uint32_t)(p.coloc ? slot : cellv), 0u);
            const double u = (double)d.x * 2.3283064365386963e-10;
            int act = 4;
            double cum = 0.0, margin = INFINITY;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                cum += s_ex[a] / S;
                margin = fmin(margin, fabs(u - cum));
                if (act == 4 && u < cum) act = a;
            }
            ctr.add(p, w, s_nnz, margin < 1e-4);
#if ECO_GREED
            if (s_seen) p.gr_seen[gs] = 1;
#endif
            agent_commit<false>(p, w, i, slot, gs, t, cellv, act, *p.forced_on, [&](int a) {
                return ((rows[16 + CNN_R + kDY[a]] >> (CNN_R + kDX[a])) & 1u) != 0u;
            });
            if (bad) *reinterpret_cast<volatile int32_t *>(p.nonfinite) = 1;
        }
        __syncthreads();  // the slice is rewritten by the block's next agent
    }
    if (tid == 0) ctr.flush(p);
}
constexpr int CNN_BLK_SMEM = CS_TOTAL_BYTES;
