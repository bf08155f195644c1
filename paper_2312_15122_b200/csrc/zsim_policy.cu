// zsim_policy.cu -- on-device policy inference: the reference's NNPolicy::act
// (train/policy.hpp:27-58) over forward_row (nn/model.hpp:464-585) for a whole
// observation batch, plus Model::init (nn/model.hpp:199-212) on the host.
//
// Execution model: one CTA (256 threads) per group of kRows observation rows.
// A row's 17 latent tokens (learned null + 16 agent slots) live in shared
// memory as rows of a [kTok][128] token tile for the whole forward pass; the
// key/value token sets (road 129, route 65, active 2) are never materialised:
// a cross-attention block's keys and values are affine in the row's raw
// features (kv = W_emb f + b_emb is not normalised, model.hpp:326-336), so
// the host folds W_k W_emb and W_v W_emb once and each query works in the
// feature space (12 / 5 / 9 dims) instead of the 128-dim latent space:
//   score_j = q . (Kf f_j + ck) = (Kf^T q) . f_j + q . ck
//   out     = Vf (sum_j p_j f_j) + (sum_j p_j) cv + p_null v_null
// The 128x128 projections over the token tile (Q/K/V/O of the four attention
// blocks) are the dense contractions.
//
// Numerics: fp32 as the reference (Model<float>); the folding and the
// summation order differ from Eigen's, so results match to fp32 rounding
// (tests/test_policy.py states the tolerance against the float64 oracle).
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/zsim_gpu.h"
#include "zsim_scenario.hpp"

extern "C" void zsim_internal_set_last_error(const char* m);  // zsim_capi.cu

namespace zp {

constexpr int kD = 128;                 // latent width (ModelConfig::latent)
constexpr int kHeads = 2, kDh = 64;     // heads, head width
constexpr int kAgents = 16, kRoad = 128, kRoute = 64;  // ObsSpec (simcore.hpp:60-63)
constexpr int kAgF = 6, kRoadF = 12, kRouteF = 5, kActF = 9, kValF = 2;
constexpr int kLat = kAgents + 1;       // latent tokens per row
constexpr int kRows = 3;                // observation rows per CTA
constexpr int kTok = 64;                // token tile (kRows * kLat = 51, padded)
constexpr int kLd = kD + 4;             // smem row stride of a token tile (floats)
constexpr int kThreads = 256;
constexpr int kMaxTrunk = 4, kMaxHead = 16, kMaxVE = 64;

// fixed input normalisation (model.hpp:56-63)
__constant__ float c_act_scale[kActF] = {0.1f, 1.8f, 0.02f, 1.f, 1.f, 1.f, 1.f, 0.02f, 0.1f};
__constant__ float c_ag_scale[kAgF] = {0.02f, 0.02f, 0.32f, 0.1f, 0.02f, 1.f};
__constant__ float c_rd_scale[kRoadF] = {0.02f, 0.02f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f};
__constant__ float c_rt_scale[kRouteF] = {0.02f, 0.02f, 1.f, 1.f, 1.f};
__constant__ float c_val_scale[kValF] = {0.02f, 0.01f};

// Matrices are the reference's column-major Eigen maps: W(r, c) at c * rows + r,
// i.e. [in][out] for an out x in weight -- a warp reading consecutive outputs
// of one input column reads consecutive floats.
struct AttnW {
    const float *ln_g, *ln_b, *wq, *bq, *wo, *bo;
    const float *wk, *bk, *wv, *bv;            // self attention
    const float *kf, *vf, *ck, *cv, *kn, *vn;  // cross: folded [F][128], [F][128], [128] x4
};
struct MlpW {
    const float *ln_g, *ln_b, *w1, *b1, *w2, *b2;
};
struct PolicyW {
    const float *emb_ag_w, *emb_ag_b, *null_ag;
    AttnW self, road, route, active;
    MlpW pblk[kMaxTrunk], vblk[kMaxTrunk];
    const float *acc_w, *acc_b, *str_w, *str_b;
    const float *vemb_w, *vemb_b, *vin_w, *vin_b, *vhead_w, *vhead_b;
    int trunk, ve, n_accel, n_steer;
};

struct ActArgs {
    PolicyW w;
    zsim_obs_view obs;
    int B;
    uint64_t* rng;
    int argmax;
    int32_t* accel;
    int32_t* steer;
    float* logp;
    float* value;
    float* logits;  // optional [B][n_accel + n_steer]
};

struct Smem {
    float X[kTok][kLd];   // residual token stream
    float A[kTok][kLd];   // LayerNorm output, then attention output (concat)
    float Q[kTok][kLd];
    float K[kTok][kLd];
    float V[kTok][kLd];
    float road[kRows][kRoad][kRoadF];
    float route[kRows][kRoute][kRouteF];
    float act[kRows][kActF];
    float val[kRows][kValF];
    unsigned char mroad[kRows][kRoad];
    unsigned char mroute[kRows][kRoute];
    unsigned char mlat[kRows][kLat];
    unsigned char mact[kRows][1];  // the active token is always valid
    float vec[kRows][2][kD + kMaxVE];  // trunk vectors (policy / value), ping-pong
    float tmp[kRows][kD];
    float pooled[kRows][kD];
    float lnv[kRows][kD];
    float logit[kRows][2 * kMaxHead];
    float vout[kRows];
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ float gelu(float x) { return 0.5f * x * (1.f + erff(x * 0.70710678118654752440f)); }

// ln_forward (model.hpp:287-303) of every token row of X into A: one warp per token.
__device__ void ln_tokens(const float (*X)[kLd], float (*A)[kLd], const float* g, const float* b) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int s = warp; s < kTok; s += kThreads / 32) {
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = X[s][lane + 32 * k];
        const float mu = warp_sum(v[0] + v[1] + v[2] + v[3]) / float(kD);
        float q = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) q += (v[k] - mu) * (v[k] - mu);
        const float var = warp_sum(q) / float(kD);
        const float rstd = 1.f / sqrtf(var + 1e-5f);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int c = lane + 32 * k;
            A[s][c] = (v[k] - mu) * rstd * g[c] + b[c];
        }
    }
}

// out[s][n] = sum_k A[s][k] W(n, k) + bias[n] (+ res[s][n]) over the token
// tile; W column-major [k][n].  Thread: 4 tokens x 8 outputs.
__device__ void gemm_tile(const float (*A)[kLd], const float* __restrict__ W, const float* __restrict__ bias,
                          float (*out)[kLd], bool residual) {
    const int t = threadIdx.x;
    const int s0 = (t >> 4) * 4, n0 = (t & 15) * 8;
    float acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
#pragma unroll 2
    for (int k = 0; k < kD; k += 4) {
        float4 a[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = *reinterpret_cast<const float4*>(&A[s0 + i][k]);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            const float4 w0 = __ldg(reinterpret_cast<const float4*>(W + (k + kk) * kD + n0));
            const float4 w1 = __ldg(reinterpret_cast<const float4*>(W + (k + kk) * kD + n0 + 4));
            const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float av = kk == 0 ? a[i].x : kk == 1 ? a[i].y : kk == 2 ? a[i].z : a[i].w;
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av, wv[j], acc[i][j]);
            }
        }
    }
    // each output element is read (residual) and written by its owner only
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float v = acc[i][j] + bias[n0 + j];
            if (residual) v += out[s0 + i][n0 + j];
            out[s0 + i][n0 + j] = v;
        }
}

// Self attention of each row's 17 latent tokens (model.hpp:340-364), heads
// concatenated into A.  One warp per (row, head, query); lane j < 17 = key j.
__device__ void self_attention(Smem& sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float scale = 0.125f;  // 1 / sqrt(64)
    for (int task = warp; task < kRows * kHeads * kLat; task += kThreads / 32) {
        const int g = task / (kHeads * kLat), h = (task / kLat) % kHeads, i = task % kLat;
        const int qs = g * kLat + i;
        float s = -INFINITY;
        const bool valid = lane < kLat && sm.mlat[g][lane];
        if (lane < kLat) {
            const float* q = &sm.Q[qs][h * kDh];
            const float* k = &sm.K[g * kLat + lane][h * kDh];
            float d = 0.f;
#pragma unroll 16
            for (int c = 0; c < kDh; ++c) d = fmaf(q[c], k[c], d);
            s = d * scale;
        }
        const float mx = warp_max(valid ? s : -INFINITY);
        const float e = valid ? expf(s - mx) : 0.f;
        const float p = e / warp_sum(e);
        // out[c] = sum_j p_j V[j][c]; lane owns c = lane, lane + 32
        float o0 = 0.f, o1 = 0.f;
        for (int j = 0; j < kLat; ++j) {
            const float pj = __shfl_sync(0xffffffffu, p, j);
            o0 = fmaf(pj, sm.V[g * kLat + j][h * kDh + lane], o0);
            o1 = fmaf(pj, sm.V[g * kLat + j][h * kDh + lane + 32], o1);
        }
        sm.A[qs][h * kDh + lane] = o0;
        sm.A[qs][h * kDh + lane + 32] = o1;
    }
}

// Cross attention against a row's feature tokens (null + n tokens of F raw
// scaled features; attn_forward with self_mode false, model.hpp:326-367),
// through the folded weights.  One warp per (row, head, query).
template <int F, int N>
__device__ void cross_attention(Smem& sm, const AttnW& w, const float (*feat)[N][F], const unsigned char (*mask)[N]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float scale = 0.125f;
    for (int task = warp; task < kRows * kHeads * kLat; task += kThreads / 32) {
        const int g = task / (kHeads * kLat), h = (task / kLat) % kHeads, i = task % kLat;
        const int qs = g * kLat + i;
        const int c0 = h * kDh + lane, c1 = c0 + 32;
        const float q0 = sm.Q[qs][c0], q1 = sm.Q[qs][c1];
        // qf = Kf_h^T q, qn = q . ck_h, null score = q . k_null_h
        float qf[F];
#pragma unroll
        for (int f = 0; f < F; ++f) qf[f] = warp_sum(fmaf(w.kf[f * kD + c0], q0, w.kf[f * kD + c1] * q1));
        const float qn = warp_sum(fmaf(w.ck[c0], q0, w.ck[c1] * q1));
        const float sn = warp_sum(fmaf(w.kn[c0], q0, w.kn[c1] * q1)) * scale;
        // feature-token scores, lane owns tokens lane + 32 m
        constexpr int M = (N + 31) / 32;
        float s[M];
        float mx = sn;
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const int j = lane + 32 * m;
            s[m] = -INFINITY;
            if (j < N && mask[g][j]) {
                float d = qn;
#pragma unroll
                for (int f = 0; f < F; ++f) d = fmaf(qf[f], feat[g][j][f], d);
                s[m] = d * scale;
            }
            mx = fmaxf(mx, s[m]);
        }
        mx = warp_max(mx);
        float esum = 0.f;
#pragma unroll
        for (int m = 0; m < M; ++m) {
            s[m] = s[m] == -INFINITY ? 0.f : expf(s[m] - mx);
            esum += s[m];
        }
        const float en = expf(sn - mx);
        const float tot = warp_sum(esum) + en;
        const float inv = 1.f / tot;
        // aggregated features sum_j p_j f_j and sum_j p_j
        float ag[F];
#pragma unroll
        for (int f = 0; f < F; ++f) ag[f] = 0.f;
        float ps = 0.f;
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const int j = lane + 32 * m;
            if (j < N && s[m] != 0.f) {
                const float p = s[m] / tot;
                ps += p;
#pragma unroll
                for (int f = 0; f < F; ++f) ag[f] = fmaf(p, feat[g][j][f], ag[f]);
            }
        }
#pragma unroll
        for (int f = 0; f < F; ++f) ag[f] = warp_sum(ag[f]);
        ps = warp_sum(ps);
        const float pn = en * inv;
        float o0 = fmaf(ps, w.cv[c0], pn * w.vn[c0]), o1 = fmaf(ps, w.cv[c1], pn * w.vn[c1]);
#pragma unroll
        for (int f = 0; f < F; ++f) {
            o0 = fmaf(w.vf[f * kD + c0], ag[f], o0);
            o1 = fmaf(w.vf[f * kD + c1], ag[f], o1);
        }
        sm.A[qs][c0] = o0;
        sm.A[qs][c1] = o1;
    }
}

// mlp_forward (model.hpp:431-440) of vec[.][src] into vec[.][dst].
__device__ __forceinline__ void mlp_rows(Smem& sm, const MlpW& w, int src, int dst) {
    __syncthreads();
    {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (warp < kRows) {
            const float* xv = sm.vec[warp][src];
            float v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = xv[lane + 32 * k];
            const float mu = warp_sum(v[0] + v[1] + v[2] + v[3]) / float(kD);
            float q = 0.f;
#pragma unroll
            for (int k = 0; k < 4; ++k) q += (v[k] - mu) * (v[k] - mu);
            const float rstd = 1.f / sqrtf(warp_sum(q) / float(kD) + 1e-5f);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = lane + 32 * k;
                sm.lnv[warp][c] = (v[k] - mu) * rstd * w.ln_g[c] + w.ln_b[c];
            }
        }
    }
    __syncthreads();
    for (int task = threadIdx.x; task < kRows * kD; task += kThreads) {
        const int g = task / kD, n = task % kD;
        float acc = 0.f;
        for (int k = 0; k < kD; ++k) acc = fmaf(__ldg(w.w1 + k * kD + n), sm.lnv[g][k], acc);
        sm.tmp[g][n] = gelu(acc + w.b1[n]);
    }
    __syncthreads();
    for (int task = threadIdx.x; task < kRows * kD; task += kThreads) {
        const int g = task / kD, n = task % kD;
        float acc = 0.f;
        for (int k = 0; k < kD; ++k) acc = fmaf(__ldg(w.w2 + k * kD + n), sm.tmp[g][k], acc);
        sm.vec[g][dst][n] = acc + w.b2[n] + sm.vec[g][src][n];
    }
}

__device__ __forceinline__ uint64_t rng_next(uint64_t& st) {
    uint64_t z = (st += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// log_softmax (model.hpp:672-678) in place, float as the reference.
__device__ void log_softmax(float* z, int n) {
    float mx = z[0];
    for (int i = 1; i < n; ++i) mx = fmaxf(mx, z[i]);
    float se = 0.f;
    for (int i = 0; i < n; ++i) se += expf(z[i] - mx);
    const float lse = logf(se);
    for (int i = 0; i < n; ++i) z[i] = (z[i] - mx) - lse;
}

// sample_categorical (model.hpp:680-697) on log-probabilities.
__device__ int sample_ls(const float* ls, int n, uint64_t& st, double& logp) {
    const double u = double(rng_next(st) >> 11) * 0x1.0p-53;
    double acc = 0.0;
    int pick = n - 1;
    for (int i = 0; i < n; ++i) {
        acc += exp(double(ls[i]));
        if (u < acc) {
            pick = i;
            break;
        }
    }
    logp = double(ls[pick]);
    return pick;
}

__device__ int argmax_first(const float* z, int n) {
    int best = 0;
    for (int i = 1; i < n; ++i)
        if (z[i] > z[best]) best = i;
    return best;
}

__global__ void __launch_bounds__(kThreads, 1) k_policy_act(const ActArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    Smem& sm = *reinterpret_cast<Smem*>(dsm);
    const PolicyW& W = a.w;
    const int tid = threadIdx.x;
    const int b0 = blockIdx.x * kRows;

    // ---- raw features of the CTA's rows, scaled (forward_row, model.hpp:470-503) ----
    for (int e = tid; e < kRows * kRoad * kRoadF; e += kThreads) {
        const int g = e / (kRoad * kRoadF), r = e % (kRoad * kRoadF);
        const int b = b0 + g;
        const float v = b < a.B ? a.obs.road[size_t(b) * kRoad * kRoadF + r] : 0.f;
        sm.road[g][r / kRoadF][r % kRoadF] = v * c_rd_scale[r % kRoadF];
        if (r % kRoadF == kRoadF - 1) sm.mroad[g][r / kRoadF] = v > 0.5f;
    }
    for (int e = tid; e < kRows * kRoute * kRouteF; e += kThreads) {
        const int g = e / (kRoute * kRouteF), r = e % (kRoute * kRouteF);
        const int b = b0 + g;
        const float v = b < a.B ? a.obs.route[size_t(b) * kRoute * kRouteF + r] : 0.f;
        sm.route[g][r / kRouteF][r % kRouteF] = v * c_rt_scale[r % kRouteF];
        if (r % kRouteF == kRouteF - 1) sm.mroute[g][r / kRouteF] = v > 0.5f;
    }
    if (tid < kRows * kActF) {
        const int g = tid / kActF, f = tid % kActF, b = b0 + g;
        sm.act[g][f] = (b < a.B ? a.obs.active[size_t(b) * kActF + f] : 0.f) * c_act_scale[f];
    }
    if (tid < kRows) sm.mact[tid][0] = 1;
    if (tid < kRows * kValF) {
        const int g = tid / kValF, f = tid % kValF, b = b0 + g;
        sm.val[g][f] = (b < a.B ? a.obs.value_only[size_t(b) * kValF + f] : 0.f) * c_val_scale[f];
    }
    // latent tokens: null + agent embeddings (model.hpp:505-513); padding tokens 0
    for (int e = tid; e < kTok * kD; e += kThreads) {
        const int s = e / kD, c = e % kD;
        const int g = s / kLat, i = s % kLat, b = b0 + g;
        float v = 0.f;
        if (g < kRows) {
            if (i == 0) {
                v = W.null_ag[c];
            } else {
                const float* ag = a.obs.agents + (size_t(b) * kAgents + (i - 1)) * kAgF;
                float acc = 0.f;
#pragma unroll
                for (int f = 0; f < kAgF; ++f) {
                    const float x = b < a.B ? ag[f] * c_ag_scale[f] : 0.f;
                    acc = fmaf(W.emb_ag_w[f * kD + c], x, acc);
                }
                v = acc + W.emb_ag_b[c];
                if (c == 0) sm.mlat[g][i] = (b < a.B ? ag[5] : 0.f) > 0.5f;
            }
            if (i == 0 && c == 0) sm.mlat[g][0] = 1;
        }
        sm.X[s][c] = v;
    }
    __syncthreads();

    // ---- encoder (model.hpp:530-543) ----
    ln_tokens(sm.X, sm.A, W.self.ln_g, W.self.ln_b);
    __syncthreads();
    gemm_tile(sm.A, W.self.wq, W.self.bq, sm.Q, false);
    gemm_tile(sm.A, W.self.wk, W.self.bk, sm.K, false);
    gemm_tile(sm.A, W.self.wv, W.self.bv, sm.V, false);
    __syncthreads();
    self_attention(sm);
    __syncthreads();
    gemm_tile(sm.A, W.self.wo, W.self.bo, sm.X, true);
    __syncthreads();

    // (explicit blocks: indexing the kernel-parameter struct dynamically would
    // copy it to local memory)
    auto cross_block = [&](const AttnW& aw, int m) {
        ln_tokens(sm.X, sm.A, aw.ln_g, aw.ln_b);
        __syncthreads();
        gemm_tile(sm.A, aw.wq, aw.bq, sm.Q, false);
        __syncthreads();
        if (m == 0) cross_attention<kRoadF, kRoad>(sm, aw, sm.road, sm.mroad);
        if (m == 1) cross_attention<kRouteF, kRoute>(sm, aw, sm.route, sm.mroute);
        // the active token set is one always-valid token per row
        if (m == 2) cross_attention<kActF, 1>(sm, aw, reinterpret_cast<const float(*)[1][kActF]>(sm.act), sm.mact);
        __syncthreads();
        gemm_tile(sm.A, aw.wo, aw.bo, sm.X, true);
        __syncthreads();
    };
    cross_block(W.road, 0);
    cross_block(W.route, 1);
    cross_block(W.active, 2);

    // ---- mean pool over valid latent tokens (model.hpp:545-554) ----
    for (int e = tid; e < kRows * kD; e += kThreads) {
        const int g = e / kD, c = e % kD;
        float acc = 0.f;
        int n = 0;
        for (int i = 0; i < kLat; ++i)
            if (sm.mlat[g][i]) {
                acc += sm.X[g * kLat + i][c];
                ++n;
            }
        sm.vec[g][0][c] = acc / float(n);
        sm.pooled[g][c] = acc / float(n);  // kept for the value trunk
    }
    // ---- policy trunk + heads (model.hpp:556-568) ----
    int cur = 0;
#pragma unroll
    for (int i = 0; i < kMaxTrunk; ++i)
        if (i < W.trunk) {
            mlp_rows(sm, W.pblk[i], cur, cur ^ 1);
            cur ^= 1;
        }
    __syncthreads();
    const int na = W.n_accel, ns = W.n_steer;
    for (int e = tid; e < kRows * (na + ns); e += kThreads) {
        const int g = e / (na + ns), n = e % (na + ns);
        const bool isa = n < na;
        const float* Wm = isa ? W.acc_w : W.str_w;
        const int rows = isa ? na : ns, o = isa ? n : n - na;
        float acc = 0.f;
        for (int k = 0; k < kD; ++k) acc = fmaf(__ldg(Wm + k * rows + o), sm.vec[g][cur][k], acc);
        sm.logit[g][n] = acc + (isa ? W.acc_b[o] : W.str_b[o]);
    }
    __syncthreads();
    // ---- value trunk (model.hpp:570-584): concat [pooled; gelu(W_e v + b_e)] ----
    for (int e = tid; e < kRows * (kD + W.ve); e += kThreads) {
        const int g = e / (kD + W.ve), c = e % (kD + W.ve);
        float v;
        if (c < kD) {
            v = sm.pooled[g][c];
        } else {
            const int j = c - kD;
            float acc = 0.f;
#pragma unroll
            for (int f = 0; f < kValF; ++f) acc = fmaf(W.vemb_w[f * W.ve + j], sm.val[g][f], acc);
            v = gelu(acc + W.vemb_b[j]);
        }
        sm.vec[g][0][c] = v;
    }
    __syncthreads();
    for (int e = tid; e < kRows * kD; e += kThreads) {
        const int g = e / kD, n = e % kD;
        float acc = 0.f;
        for (int k = 0; k < kD + W.ve; ++k) acc = fmaf(__ldg(W.vin_w + size_t(k) * kD + n), sm.vec[g][0][k], acc);
        sm.vec[g][1][n] = acc + W.vin_b[n];
    }
    cur = 1;
#pragma unroll
    for (int i = 0; i < kMaxTrunk; ++i)
        if (i < W.trunk) {
            mlp_rows(sm, W.vblk[i], cur, cur ^ 1);
            cur ^= 1;
        }
    __syncthreads();
    {
        const int lane = tid & 31, warp = tid >> 5;
        if (warp < kRows) {
            float acc = 0.f;
            for (int k = lane; k < kD; k += 32) acc = fmaf(W.vhead_w[k], sm.vec[warp][cur][k], acc);
            acc = warp_sum(acc);
            if (lane == 0) sm.vout[warp] = acc + W.vhead_b[0];
        }
    }
    __syncthreads();

    // ---- NNPolicy::act (policy.hpp:33-56): one thread per row ----
    if (tid < kRows && b0 + tid < a.B) {
        const int g = tid, b = b0 + tid;
        float la[kMaxHead], ls[kMaxHead];
        for (int i = 0; i < na; ++i) la[i] = sm.logit[g][i];
        for (int i = 0; i < ns; ++i) ls[i] = sm.logit[g][na + i];
        if (a.logits) {
            for (int i = 0; i < na + ns; ++i) a.logits[size_t(b) * (na + ns) + i] = sm.logit[g][i];
        }
        a.value[b] = sm.vout[g];
        int ai, si;
        float lp;
        if (a.argmax) {
            ai = argmax_first(la, na);
            si = argmax_first(ls, ns);
            log_softmax(la, na);
            log_softmax(ls, ns);
            lp = la[ai] + ls[si];
        } else {
            uint64_t st = a.rng[b];
            log_softmax(la, na);
            log_softmax(ls, ns);
            double lpa, lps;
            ai = sample_ls(la, na, st, lpa);
            si = sample_ls(ls, ns, st, lps);
            lp = float(lpa + lps);
            a.rng[b] = st;
        }
        a.accel[b] = ai;
        a.steer[b] = si;
        a.logp[b] = lp;
    }
}

// ---------------------------------------------------------------------------
// host: ParamIndex::build (model.hpp:101-167) and Model::init (:199-212)
// ---------------------------------------------------------------------------
struct Entry {
    std::string name;
    int64_t off;
    int rows, cols;
    bool weight;
    float init;
};

std::vector<Entry> param_index(const zsim_model_config& c, int64_t* total) {
    std::vector<Entry> e;
    int64_t t = 0;
    auto add = [&](const std::string& n, int r, int cl, bool w, float init = 0.f) {
        e.push_back({n, t, r, cl, w, init});
        t += int64_t(r) * cl;
    };
    const int d = c.latent;
    auto attn = [&](const std::string& p) {
        add(p + ".ln.g", d, 1, false, 1.f);
        add(p + ".ln.b", d, 1, false, 0.f);
        for (const char* w : {"q", "k", "v", "o"}) {
            add(p + ".w" + w, d, d, true);
            add(p + ".b" + w, d, 1, false);
        }
    };
    auto block = [&](const std::string& p) {
        add(p + ".ln.g", d, 1, false, 1.f);
        add(p + ".ln.b", d, 1, false, 0.f);
        add(p + ".w1", d, d, true);
        add(p + ".b1", d, 1, false);
        add(p + ".w2", d, d, true);
        add(p + ".b2", d, 1, false);
    };
    add("emb.agents.w", d, kAgF, true);
    add("emb.agents.b", d, 1, false);
    add("emb.road.w", d, kRoadF, true);
    add("emb.road.b", d, 1, false);
    add("emb.route.w", d, kRouteF, true);
    add("emb.route.b", d, 1, false);
    add("emb.active.w", d, kActF, true);
    add("emb.active.b", d, 1, false);
    for (const char* n : {"agents", "road", "route", "active"}) add(std::string("null.") + n, d, 1, true);
    attn("enc.self");
    attn("enc.cross.road");
    attn("enc.cross.route");
    attn("enc.cross.active");
    for (int i = 0; i < c.trunk_blocks; ++i) block("policy.block" + std::to_string(i));
    add("policy.accel.w", c.n_accel, d, true);
    add("policy.accel.b", c.n_accel, 1, false);
    add("policy.steer.w", c.n_steer, d, true);
    add("policy.steer.b", c.n_steer, 1, false);
    add("value.emb.w", c.value_embed, kValF, true);
    add("value.emb.b", c.value_embed, 1, false);
    add("value.in.w", d, d + c.value_embed, true);
    add("value.in.b", d, 1, false);
    for (int i = 0; i < c.trunk_blocks; ++i) block("value.block" + std::to_string(i));
    add("value.head.w", 1, d, true);
    add("value.head.b", 1, 1, false);
    *total = t;
    return e;
}

void validate(const zsim_model_config* c) {
    using zs::Err;
    if (!c) zs::raise(Err::invalid_argument, "model config is null");
    // ModelConfig::validate (model.hpp:29-36)
    if (c->latent <= 0 || c->heads <= 0 || c->latent % c->heads != 0)
        zs::raise(Err::config, "model: latent must be a positive multiple of heads");
    if (c->trunk_blocks <= 0) zs::raise(Err::config, "model: trunk_blocks must be > 0");
    if (c->value_embed <= 0) zs::raise(Err::config, "model: value_embed must be > 0");
    if (c->n_accel <= 0 || c->n_steer <= 0) zs::raise(Err::config, "model: head sizes must be > 0");
    // what the device kernels are specialised for
    if (c->latent != kD || c->heads != kHeads || c->n_agents != kAgents || c->n_road != kRoad ||
        c->n_route != kRoute || c->trunk_blocks > kMaxTrunk || c->value_embed > kMaxVE || c->n_accel > kMaxHead ||
        c->n_steer > kMaxHead)
        zs::raise(Err::config, "model: the device policy supports latent 128, 2 heads, obs spec 16/128/64, <= " +
                                   std::to_string(kMaxTrunk) + " trunk blocks, value_embed <= " +
                                   std::to_string(kMaxVE) + ", <= 16 bins per head");
}

}  // namespace zp

struct zsim_policy {
    zsim_model_config cfg;
    int device = 0;
    float* blob = nullptr;  // device: reference params followed by the folded cross-attention weights
    zp::PolicyW w{};
    size_t smem = 0;
};

namespace {

template <class F>
int pguarded(F&& f) {
    try {
        f();
        return ZSIM_OK;
    } catch (const zs::Error& e) {
        zsim_internal_set_last_error(e.what());
        return int(e.kind);
    } catch (const std::exception& e) {
        zsim_internal_set_last_error(e.what());
        return ZSIM_RUNTIME;
    }
}

void ccheck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) zs::raise(zs::Err::cuda, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

extern "C" {

ZSIM_API int zsim_model_config_defaults(zsim_model_config* c) {
    return pguarded([&] {
        if (!c) zs::raise(zs::Err::invalid_argument, "model_config_defaults: null");
        *c = zsim_model_config{128, 2, 2, 32, 16, 128, 64, 7, 5, 0};
    });
}

ZSIM_API int zsim_policy_param_count(const zsim_model_config* c, int64_t* out) {
    return pguarded([&] {
        zp::validate(c);
        if (!out) zs::raise(zs::Err::invalid_argument, "policy_param_count: null output");
        zp::param_index(*c, out);
    });
}

ZSIM_API int zsim_policy_init_params(const zsim_model_config* c, uint64_t seed, float* out, int64_t n) {
    return pguarded([&] {
        zp::validate(c);
        int64_t total = 0;
        const auto ix = zp::param_index(*c, &total);
        if (!out || n != total)
            zs::raise(zs::Err::invalid_argument, "policy_init_params: need " + std::to_string(total) + " floats");
        uint64_t st = seed + 0x9e3779b97f4a7c15ull;  // Rng(seed) (common.hpp:32)
        auto uniform = [&] {
            uint64_t z = (st += 0x9e3779b97f4a7c15ull);
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
            z ^= z >> 31;
            return double(z >> 11) * 0x1.0p-53;
        };
        for (const auto& e : ix) {
            const int64_t m = int64_t(e.rows) * e.cols;
            float* p = out + e.off;
            if (e.weight) {
                const double bound = 1.0 / std::sqrt(double(e.cols == 1 ? e.rows : e.cols));
                for (int64_t k = 0; k < m; ++k) p[k] = float(-bound + (bound - -bound) * uniform());
            } else {
                for (int64_t k = 0; k < m; ++k) p[k] = e.init;
            }
        }
    });
}

ZSIM_API int zsim_policy_create(const zsim_model_config* c, const float* params, int64_t n, int32_t device,
                                zsim_policy** out) {
    return pguarded([&] {
        zp::validate(c);
        if (!params || !out) zs::raise(zs::Err::invalid_argument, "policy_create: null argument");
        int64_t total = 0;
        const auto ix = zp::param_index(*c, &total);
        if (n != total) zs::raise(zs::Err::invalid_argument, "policy_create: expected " + std::to_string(total) +
                                                                 " parameters, got " + std::to_string(n));
        auto find = [&](const std::string& name) -> const zp::Entry& {
            for (const auto& e : ix)
                if (e.name == name) return e;
            zs::raise(zs::Err::runtime, "policy: no parameter " + name);
        };
        const int d = zp::kD;
        // folded cross-attention weights (double on the host, rounded once)
        std::vector<float> extra;
        struct Fold {
            int64_t kf, vf, ck, cv, kn, vn;
        };
        Fold folds[3];
        const char* mods[3] = {"road", "route", "active"};
        const int feats[3] = {zp::kRoadF, zp::kRouteF, zp::kActF};
        auto P = [&](const zp::Entry& e, int r, int cl) { return double(params[e.off + int64_t(cl) * e.rows + r]); };
        for (int m = 0; m < 3; ++m) {
            const std::string p = std::string("enc.cross.") + mods[m];
            const auto &wk = find(p + ".wk"), &bk = find(p + ".bk"), &wv = find(p + ".wv"), &bv = find(p + ".bv");
            const auto &we = find(std::string("emb.") + mods[m] + ".w"), &be = find(std::string("emb.") + mods[m] + ".b");
            const auto& nl = find(std::string("null.") + mods[m]);
            const int F = feats[m];
            Fold& fo = folds[m];
            auto put = [&](int64_t& off, int count) {
                off = int64_t(extra.size());
                extra.resize(extra.size() + size_t(count));
            };
            put(fo.kf, F * d);
            put(fo.vf, F * d);
            put(fo.ck, d);
            put(fo.cv, d);
            put(fo.kn, d);
            put(fo.vn, d);
            for (int o = 0; o < d; ++o) {
                for (int f = 0; f < F; ++f) {
                    double sk = 0, sv = 0;
                    for (int c2 = 0; c2 < d; ++c2) {
                        sk += P(wk, o, c2) * P(we, c2, f);
                        sv += P(wv, o, c2) * P(we, c2, f);
                    }
                    extra[size_t(fo.kf + f * d + o)] = float(sk);
                    extra[size_t(fo.vf + f * d + o)] = float(sv);
                }
                double ck = P(bk, o, 0), cv = P(bv, o, 0), kn = P(bk, o, 0), vn = P(bv, o, 0);
                for (int c2 = 0; c2 < d; ++c2) {
                    ck += P(wk, o, c2) * P(be, c2, 0);
                    cv += P(wv, o, c2) * P(be, c2, 0);
                    kn += P(wk, o, c2) * P(nl, c2, 0);
                    vn += P(wv, o, c2) * P(nl, c2, 0);
                }
                extra[size_t(fo.ck + o)] = float(ck);
                extra[size_t(fo.cv + o)] = float(cv);
                extra[size_t(fo.kn + o)] = float(kn);
                extra[size_t(fo.vn + o)] = float(vn);
            }
        }
        std::unique_ptr<zsim_policy> pol(new zsim_policy());
        pol->cfg = *c;
        pol->device = device;
        ccheck(cudaSetDevice(device), "cudaSetDevice");
        const size_t base = (size_t(total) + 63) / 64 * 64;
        ccheck(cudaMalloc(&pol->blob, (base + extra.size()) * sizeof(float)), "cudaMalloc(policy)");
        ccheck(cudaMemcpy(pol->blob, params, size_t(total) * sizeof(float), cudaMemcpyHostToDevice), "H2D(policy)");
        ccheck(cudaMemcpy(pol->blob + base, extra.data(), extra.size() * sizeof(float), cudaMemcpyHostToDevice),
               "H2D(policy folds)");
        const float* D = pol->blob;
        auto at = [&](const std::string& name) { return D + find(name).off; };
        zp::PolicyW& w = pol->w;
        w.emb_ag_w = at("emb.agents.w");
        w.emb_ag_b = at("emb.agents.b");
        w.null_ag = at("null.agents");
        auto attn = [&](zp::AttnW& a, const std::string& p) {
            a.ln_g = at(p + ".ln.g");
            a.ln_b = at(p + ".ln.b");
            a.wq = at(p + ".wq");
            a.bq = at(p + ".bq");
            a.wk = at(p + ".wk");
            a.bk = at(p + ".bk");
            a.wv = at(p + ".wv");
            a.bv = at(p + ".bv");
            a.wo = at(p + ".wo");
            a.bo = at(p + ".bo");
        };
        attn(w.self, "enc.self");
        zp::AttnW* cr[3] = {&w.road, &w.route, &w.active};
        for (int m = 0; m < 3; ++m) {
            attn(*cr[m], std::string("enc.cross.") + mods[m]);
            const float* E = D + base;
            cr[m]->kf = E + folds[m].kf;
            cr[m]->vf = E + folds[m].vf;
            cr[m]->ck = E + folds[m].ck;
            cr[m]->cv = E + folds[m].cv;
            cr[m]->kn = E + folds[m].kn;
            cr[m]->vn = E + folds[m].vn;
        }
        auto block = [&](zp::MlpW& b, const std::string& p) {
            b.ln_g = at(p + ".ln.g");
            b.ln_b = at(p + ".ln.b");
            b.w1 = at(p + ".w1");
            b.b1 = at(p + ".b1");
            b.w2 = at(p + ".w2");
            b.b2 = at(p + ".b2");
        };
        for (int i = 0; i < c->trunk_blocks; ++i) {
            block(w.pblk[i], "policy.block" + std::to_string(i));
            block(w.vblk[i], "value.block" + std::to_string(i));
        }
        w.acc_w = at("policy.accel.w");
        w.acc_b = at("policy.accel.b");
        w.str_w = at("policy.steer.w");
        w.str_b = at("policy.steer.b");
        w.vemb_w = at("value.emb.w");
        w.vemb_b = at("value.emb.b");
        w.vin_w = at("value.in.w");
        w.vin_b = at("value.in.b");
        w.vhead_w = at("value.head.w");
        w.vhead_b = at("value.head.b");
        w.trunk = c->trunk_blocks;
        w.ve = c->value_embed;
        w.n_accel = c->n_accel;
        w.n_steer = c->n_steer;
        pol->smem = sizeof(zp::Smem);
        ccheck(cudaFuncSetAttribute(zp::k_policy_act, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pol->smem)),
               "cudaFuncSetAttribute(policy)");
        *out = pol.release();
    });
}

ZSIM_API int zsim_policy_destroy(zsim_policy* p) {
    return pguarded([&] {
        if (!p) return;
        cudaSetDevice(p->device);
        cudaFree(p->blob);
        delete p;
    });
}

ZSIM_API int zsim_policy_act(zsim_policy* p, const zsim_obs_view* obs, int32_t batch, uint64_t* rng,
                             int32_t use_argmax, int32_t* accel, int32_t* steer, float* logp, float* value,
                             float* logits, void* stream) {
    return pguarded([&] {
        if (!p || !obs || !accel || !steer || !logp || !value || (!use_argmax && !rng))
            zs::raise(zs::Err::invalid_argument, "policy_act: null argument");
        if (batch < 0) zs::raise(zs::Err::invalid_argument, "policy_act: negative batch");
        if (batch == 0) return;
        ccheck(cudaSetDevice(p->device), "cudaSetDevice");
        zp::ActArgs a;
        a.w = p->w;
        a.obs = *obs;
        a.B = batch;
        a.rng = rng;
        a.argmax = use_argmax;
        a.accel = accel;
        a.steer = steer;
        a.logp = logp;
        a.value = value;
        a.logits = logits;
        const int grid = (batch + zp::kRows - 1) / zp::kRows;
        zp::k_policy_act<<<grid, zp::kThreads, p->smem, static_cast<cudaStream_t>(stream)>>>(a);
        ccheck(cudaGetLastError(), "k_policy_act launch");
    });
}

}  // extern "C"
