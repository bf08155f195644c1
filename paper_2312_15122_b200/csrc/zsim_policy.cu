// zsim_policy.cu -- on-device policy inference: the reference's NNPolicy::act
// (train/policy.hpp:27-58) over forward_row (nn/model.hpp:464-585) for a whole
// observation batch, plus Model::init (nn/model.hpp:199-212) on the host.
//
// Execution model: one CTA (256 threads) per group of observation rows.  The
// rows' latent tokens (learned null + 16 agent slots each, 17 per row) form a
// token tile that stays on chip for the whole forward pass.  The key/value
// token sets (road 129, route 65, active 2 per row) are never materialised:
// a cross-attention block's keys and values are affine in the row's raw
// features (kv = W_emb f + b_emb is not normalised, model.hpp:326-336), so
// the host folds W_k W_emb and W_v W_emb once and each query works in the
// feature space (12 / 5 / 9 dims) instead of the 128-dim latent space:
//   score_j = q . (Kf f_j + ck) = (Kf^T q) . f_j + q . ck
//   out     = Vf (sum_j p_j f_j) + (sum_j p_j) cv + p_null v_null
// The 128x128 projections over the token tile (Q/K/V/O of the self block,
// Q/O of the three cross blocks) are the dense contractions:
//
//  * k_policy_tc (default): 7 rows = 119 tokens in a 128-row tile; the
//    residual stream X and the projection accumulators live in TMEM
//    (lane = token); each projection is 16 tcgen05.mma.kind::tf32
//    (M=128, N=128, K=8) from shared-memory operands in the canonical
//    K-major layout, weights streamed in by bulk-async copies (prearranged
//    and rounded to tf32 on the host).  Attention, LayerNorm and epilogues run
//    one thread per (token, column half / head) straight off TMEM.
//  * k_policy_fp32: 3 rows per CTA, every contraction on the FP32 pipe
//    (exact fp32 arithmetic like the reference's Model<float>).
//
// Numerics: fp32 accumulation everywhere; the tensor-core path rounds the
// projection inputs to tf32 (10-bit mantissa).  tests/test_policy.py states
// the tolerance of each path against the float64 oracle.
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
constexpr int kThreads = 256;
constexpr int kMaxTrunk = 4, kMaxHead = 16, kMaxVE = 64;
constexpr int kRows32 = 3;              // rows per CTA, fp32 kernel (51 tokens in a 64-row tile)
constexpr int kTok32 = 64;
constexpr int kLd = kD + 4;             // smem row stride of the fp32 kernel's token tiles
constexpr int kRowsTc = 7;              // rows per CTA, tensor-core kernel (119 tokens in a 128-row tile)
constexpr int kTokTc = 128;
constexpr int kNumProj = 10;            // projection weights in the tensor-core layout

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
    // tensor-core copies of the projections, [N=128][K=128] canonical K-major
    // tf32 tiles of 64 KB: self q k v o, road q o, route q o, active q o
    const float* tc[kNumProj];
    // tensor-core tiles of the trunks: policy block i W1 / W2 at 2i / 2i+1,
    // value block i W1 / W2 at 2i / 2i+1 (K = 128), value.in (K = 128 + ve)
    const float* tc_pblk[2 * kMaxTrunk];
    const float* tc_vblk[2 * kMaxTrunk];
    const float* tc_vin;
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
    float* pooled;  // [B][128] scratch: encoder output (tensor-core path)
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

// ---------------------------------------------------------------------------
// Per-row inputs and the post-encoder trunk, shared by both kernels.
// ---------------------------------------------------------------------------
template <int R>
struct RowSm {
    alignas(16) float road[R][kRoad][kRoadF];  // scaled features (model.hpp:470-503)
    float route[R][kRoute][kRouteF];
    float act[R][kActF];
    float val[R][kValF];
    unsigned char mroad[R][kRoad];
    unsigned char mroute[R][kRoute];
    unsigned char mlat[R][kLat];
    unsigned char mact[R][1];  // the active token is always valid
};

// post-encoder trunk state of the fp32 kernel
template <int R>
struct TrunkSm {
    float vec[R][2][kD + kMaxVE];  // trunk vectors, ping-pong
    float tmp[R][kD];
    float pooled[R][kD];
    float lnv[R][kD];
    float logit[R][2 * kMaxHead];
    float vout[R];
    float part[2][R][kD];  // GEMV partial sums of the two K halves
};

template <int R>
__device__ void load_row_inputs(RowSm<R>& sm, const ActArgs& a, int b0) {
    const int tid = threadIdx.x;
    for (int e = tid; e < R * kRoad; e += kThreads) {  // one road token (3 x float4) per thread
        const int g = e / kRoad, j = e % kRoad, b = b0 + g;
        const float4* src = reinterpret_cast<const float4*>(a.obs.road + (size_t(b) * kRoad + j) * kRoadF);
        float4* dst = reinterpret_cast<float4*>(sm.road[g][j]);
        float4 last = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < kRoadF / 4; ++q) {
            float4 v = b < a.B ? __ldg(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
            last = v;
            v.x *= c_rd_scale[4 * q], v.y *= c_rd_scale[4 * q + 1], v.z *= c_rd_scale[4 * q + 2],
                v.w *= c_rd_scale[4 * q + 3];
            dst[q] = v;
        }
        sm.mroad[g][j] = last.w > 0.5f;  // raw valid feature (model.hpp:536 valid_at 11)
    }
    for (int e = tid; e < R * kRoute * kRouteF; e += kThreads) {
        const int g = e / (kRoute * kRouteF), r = e % (kRoute * kRouteF);
        const int b = b0 + g;
        const float v = b < a.B ? a.obs.route[size_t(b) * kRoute * kRouteF + r] : 0.f;
        sm.route[g][r / kRouteF][r % kRouteF] = v * c_rt_scale[r % kRouteF];
        if (r % kRouteF == kRouteF - 1) sm.mroute[g][r / kRouteF] = v > 0.5f;
    }
    if (tid < R * kActF) {
        const int g = tid / kActF, f = tid % kActF, b = b0 + g;
        sm.act[g][f] = (b < a.B ? a.obs.active[size_t(b) * kActF + f] : 0.f) * c_act_scale[f];
    }
    if (tid < R) sm.mact[tid][0] = 1;
    if (tid < R * kValF) {
        const int g = tid / kValF, f = tid % kValF, b = b0 + g;
        sm.val[g][f] = (b < a.B ? a.obs.value_only[size_t(b) * kValF + f] : 0.f) * c_val_scale[f];
    }
    // latent mask: learned null always, agent slot when its valid feature > 0.5 (model.hpp:505-509)
    for (int e = tid; e < R * kLat; e += kThreads) {
        const int g = e / kLat, i = e % kLat, b = b0 + g;
        sm.mlat[g][i] = i == 0 ? 1 : (b < a.B ? a.obs.agents[(size_t(b) * kAgents + (i - 1)) * kAgF + 5] : 0.f) > 0.5f;
    }
}

// latent token embedding (model.hpp:510-513): column c of token slot i of row b
__device__ __forceinline__ float embed_latent(const PolicyW& W, const ActArgs& a, int b, int i, int c) {
    if (i == 0) return W.null_ag[c];
    if (b >= a.B) return W.emb_ag_b[c];
    const float* ag = a.obs.agents + (size_t(b) * kAgents + (i - 1)) * kAgF;
    float acc = 0.f;
#pragma unroll
    for (int f = 0; f < kAgF; ++f) acc = fmaf(W.emb_ag_w[f * kD + c], ag[f] * c_ag_scale[f], acc);
    return acc + W.emb_ag_b[c];
}

// Partial products sum_k W(n, k) x[g][k] of every row over one half of K
// into sm.part[half][g][n]: thread (n, half) loads each weight once and
// applies it to all R rows (R independent accumulation chains).  W column-major
// [K][128]; ends with a block barrier.
template <int R>
__device__ void gemv_rows(TrunkSm<R>& sm, const float* __restrict__ W, int K, const float* x, int xstride) {
    const int n = threadIdx.x & (kD - 1), kh = threadIdx.x >> 7;
    const int k0 = kh * (K / 2), k1 = kh ? K : K / 2;
    float acc[R];
#pragma unroll
    for (int g = 0; g < R; ++g) acc[g] = 0.f;
#pragma unroll 8
    for (int k = k0; k < k1; ++k) {
        const float wv = __ldg(W + size_t(k) * kD + n);
#pragma unroll
        for (int g = 0; g < R; ++g) acc[g] = fmaf(wv, x[g * xstride + k], acc[g]);
    }
#pragma unroll
    for (int g = 0; g < R; ++g) sm.part[kh][g][n] = acc[g];
    __syncthreads();
}

// mlp_forward (model.hpp:431-440) of vec[.][src] into vec[.][dst] for every row.
template <int R>
__device__ void mlp_rows(TrunkSm<R>& sm, const MlpW& w, int src, int dst) {
    __syncthreads();
    {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (int g = warp; g < R; g += kThreads / 32) {
            const float* xv = sm.vec[g][src];
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
                sm.lnv[g][c] = (v[k] - mu) * rstd * w.ln_g[c] + w.ln_b[c];
            }
        }
    }
    __syncthreads();
    gemv_rows<R>(sm, w.w1, kD, &sm.lnv[0][0], kD);
    for (int task = threadIdx.x; task < R * kD; task += kThreads) {
        const int g = task / kD, n = task % kD;
        sm.tmp[g][n] = gelu(sm.part[0][g][n] + sm.part[1][g][n] + w.b1[n]);
    }
    __syncthreads();
    gemv_rows<R>(sm, w.w2, kD, &sm.tmp[0][0], kD);
    for (int task = threadIdx.x; task < R * kD; task += kThreads) {
        const int g = task / kD, n = task % kD;
        sm.vec[g][dst][n] = sm.part[0][g][n] + sm.part[1][g][n] + w.b2[n] + sm.vec[g][src][n];
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

// From the pooled encodings (sm.pooled): policy trunk and heads, value trunk
// (model.hpp:556-584), then NNPolicy::act's selection (policy.hpp:33-56).
template <int R>
__device__ void trunk_and_act(const RowSm<R>& in, TrunkSm<R>& sm, const ActArgs& a, int b0) {
    const PolicyW& W = a.w;
    const int tid = threadIdx.x;
    __syncthreads();
    for (int e = tid; e < R * kD; e += kThreads) sm.vec[e / kD][0][e % kD] = sm.pooled[e / kD][e % kD];
    int cur = 0;
#pragma unroll
    for (int i = 0; i < kMaxTrunk; ++i)
        if (i < W.trunk) {
            mlp_rows<R>(sm, W.pblk[i], cur, cur ^ 1);
            cur ^= 1;
        }
    __syncthreads();
    const int na = W.n_accel, ns = W.n_steer;
    for (int e = tid; e < R * (na + ns); e += kThreads) {
        const int g = e / (na + ns), n = e % (na + ns);
        const bool isa = n < na;
        const float* Wm = isa ? W.acc_w : W.str_w;
        const int rows = isa ? na : ns, o = isa ? n : n - na;
        float acc = 0.f;
        for (int k = 0; k < kD; ++k) acc = fmaf(__ldg(Wm + k * rows + o), sm.vec[g][cur][k], acc);
        sm.logit[g][n] = acc + (isa ? W.acc_b[o] : W.str_b[o]);
    }
    __syncthreads();
    // value trunk: concat [pooled; gelu(W_e v + b_e)] -> value.in -> blocks -> head
    for (int e = tid; e < R * (kD + W.ve); e += kThreads) {
        const int g = e / (kD + W.ve), c = e % (kD + W.ve);
        float v;
        if (c < kD) {
            v = sm.pooled[g][c];
        } else {
            const int j = c - kD;
            float acc = 0.f;
#pragma unroll
            for (int f = 0; f < kValF; ++f) acc = fmaf(W.vemb_w[f * W.ve + j], in.val[g][f], acc);
            v = gelu(acc + W.vemb_b[j]);
        }
        sm.vec[g][0][c] = v;
    }
    __syncthreads();
    gemv_rows<R>(sm, W.vin_w, kD + W.ve, &sm.vec[0][0][0], 2 * (kD + kMaxVE));
    for (int e = tid; e < R * kD; e += kThreads) {
        const int g = e / kD, n = e % kD;
        sm.vec[g][1][n] = sm.part[0][g][n] + sm.part[1][g][n] + W.vin_b[n];
    }
    cur = 1;
#pragma unroll
    for (int i = 0; i < kMaxTrunk; ++i)
        if (i < W.trunk) {
            mlp_rows<R>(sm, W.vblk[i], cur, cur ^ 1);
            cur ^= 1;
        }
    __syncthreads();
    {
        const int lane = tid & 31, warp = tid >> 5;
        for (int g = warp; g < R; g += kThreads / 32) {
            float acc = 0.f;
            for (int k = lane; k < kD; k += 32) acc = fmaf(W.vhead_w[k], sm.vec[g][cur][k], acc);
            acc = warp_sum(acc);
            if (lane == 0) sm.vout[g] = acc + W.vhead_b[0];
        }
    }
    __syncthreads();
    if (tid < R && b0 + tid < a.B) {
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

// v[i] += p[i] for i < 64, p a 16-B aligned global vector (float4 loads)
__device__ __forceinline__ void add64(float* v, const float* __restrict__ p) {
#pragma unroll
    for (int i = 0; i < 64; i += 4) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p + i));
        v[i] += t.x, v[i + 1] += t.y, v[i + 2] += t.z, v[i + 3] += t.w;
    }
}

// float4 load through a generic pointer (the folded weights are staged in
// shared memory by the tensor-core kernel, read from global by the fp32 one)
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// Folded cross attention of ONE query (one head) against a row's feature
// tokens (null + N tokens of F scaled features, model.hpp:326-367): q is the
// head's 64 query values, out receives the head's 64 output values.
template <int F, int N, bool FAST>
__device__ __forceinline__ void cross_query(const AttnW& w, int h, const float* q, const float (*feat)[F],
                                            const unsigned char* mask, float* out) {
    const float scale = 0.125f;  // 1 / sqrt(64)
    const float* kf = w.kf + h * kDh;
    float qf[F];
#pragma unroll
    for (int f = 0; f < F; ++f) qf[f] = 0.f;
    float qn = 0.f, sn = 0.f;
#pragma unroll
    for (int c4 = 0; c4 < kDh / 4; ++c4) {  // F + 2 independent chains, float4 weight loads
        const int c = 4 * c4;
#pragma unroll
        for (int f = 0; f < F; ++f) {
            const float4 k = ld4((kf + f * kD + c));
            qf[f] = fmaf(k.x, q[c], fmaf(k.y, q[c + 1], fmaf(k.z, q[c + 2], fmaf(k.w, q[c + 3], qf[f]))));
        }
        const float4 ck = ld4((w.ck + h * kDh + c));
        const float4 kn = ld4((w.kn + h * kDh + c));
        qn = fmaf(ck.x, q[c], fmaf(ck.y, q[c + 1], fmaf(ck.z, q[c + 2], fmaf(ck.w, q[c + 3], qn))));
        sn = fmaf(kn.x, q[c], fmaf(kn.y, q[c + 1], fmaf(kn.z, q[c + 2], fmaf(kn.w, q[c + 3], sn))));
    }
    sn *= scale;
    // one pass, running maximum (the softmax is shift-invariant; every
    // accumulated term is rescaled when the maximum moves), tokens in blocks
    // of TB so the scores of a block are independent chains
    float mx = sn, tot = 1.f, ps = 0.f;
    float ag[F];
#pragma unroll
    for (int f = 0; f < F; ++f) ag[f] = 0.f;
    constexpr int TB = N % 4 == 0 ? 4 : 1;
    for (int j0 = 0; j0 < N; j0 += TB) {
        float x[TB][F], d[TB];
        float bm = -INFINITY;
#pragma unroll
        for (int u = 0; u < TB; ++u) {
            const int j = j0 + u;
            if constexpr (F % 4 == 0) {  // 16-B aligned rows: vector loads
#pragma unroll
                for (int f = 0; f < F; f += 4) {
                    const float4 t = *reinterpret_cast<const float4*>(&feat[j][f]);
                    x[u][f] = t.x, x[u][f + 1] = t.y, x[u][f + 2] = t.z, x[u][f + 3] = t.w;
                }
            } else {
#pragma unroll
                for (int f = 0; f < F; ++f) x[u][f] = feat[j][f];
            }
            float dd = qn;
#pragma unroll
            for (int f = 0; f < F; ++f) dd = fmaf(qf[f], x[u][f], dd);
            d[u] = mask[j] ? dd * scale : -INFINITY;
            bm = fmaxf(bm, d[u]);
        }
        if (bm > mx) {
            const float r = FAST ? __expf(mx - bm) : expf(mx - bm);
            tot *= r;
            ps *= r;
#pragma unroll
            for (int f = 0; f < F; ++f) ag[f] *= r;
            mx = bm;
        }
#pragma unroll
        for (int u = 0; u < TB; ++u) {
            // masked tokens: exp(-inf) = 0 exactly
            const float e = FAST ? __expf(d[u] - mx) : expf(d[u] - mx);
            tot += e;
            ps += e;
#pragma unroll
            for (int f = 0; f < F; ++f) ag[f] = fmaf(e, x[u][f], ag[f]);
        }
    }
    const float en = FAST ? __expf(sn - mx) : expf(sn - mx);  // the null token's term, already inside tot (started as exp(0) = 1)
    const float inv = 1.f / tot;
    ps *= inv;
    const float pn = en * inv;
#pragma unroll
    for (int f = 0; f < F; ++f) ag[f] *= inv;
    const float* vf = w.vf + h * kDh;
#pragma unroll
    for (int c4 = 0; c4 < kDh / 4; ++c4) {
        const int c = 4 * c4;
        const float4 cv = ld4((w.cv + h * kDh + c));
        const float4 vn = ld4((w.vn + h * kDh + c));
        float o0 = fmaf(ps, cv.x, pn * vn.x), o1 = fmaf(ps, cv.y, pn * vn.y), o2 = fmaf(ps, cv.z, pn * vn.z),
              o3 = fmaf(ps, cv.w, pn * vn.w);
#pragma unroll
        for (int f = 0; f < F; ++f) {
            const float4 v = ld4((vf + f * kD + c));
            o0 = fmaf(v.x, ag[f], o0);
            o1 = fmaf(v.y, ag[f], o1);
            o2 = fmaf(v.z, ag[f], o2);
            o3 = fmaf(v.w, ag[f], o3);
        }
        out[c] = o0;
        out[c + 1] = o1;
        out[c + 2] = o2;
        out[c + 3] = o3;
    }
}

// ===========================================================================
// k_policy_fp32: every contraction on the FP32 pipe, 3 rows per CTA.
// ===========================================================================
struct Smem32 {
    float X[kTok32][kLd];  // residual token stream
    float A[kTok32][kLd];  // LayerNorm output, then attention output
    float Q[kTok32][kLd];
    float K[kTok32][kLd];
    float V[kTok32][kLd];
    RowSm<kRows32> rs;
    TrunkSm<kRows32> tr;
    float sc[kThreads][kLat];  // self-attention scores of each thread's query
};

// ln_forward (model.hpp:287-303) of every token row of X into A: one warp per token.
__device__ void ln_tokens32(const float (*X)[kLd], float (*A)[kLd], const float* g, const float* b) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int s = warp; s < kTok32; s += kThreads / 32) {
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = X[s][lane + 32 * k];
        const float mu = warp_sum(v[0] + v[1] + v[2] + v[3]) / float(kD);
        float q = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) q += (v[k] - mu) * (v[k] - mu);
        const float rstd = 1.f / sqrtf(warp_sum(q) / float(kD) + 1e-5f);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int c = lane + 32 * k;
            A[s][c] = (v[k] - mu) * rstd * g[c] + b[c];
        }
    }
}

// out[s][n] = sum_k A[s][k] W(n, k) + bias[n] (+ out[s][n]) over the token
// tile; W column-major [k][n].  Thread: 4 tokens x 8 outputs.
__device__ void gemm32(const float (*A)[kLd], const float* __restrict__ W, const float* __restrict__ bias,
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

// Self attention (model.hpp:340-364) of each row's 17 latent tokens, one
// thread per (token, head): keys / values of the row from smem.
template <bool FAST, class KV>
__device__ __forceinline__ void self_query(int h, const float* q, const unsigned char* mlat, KV kv, float* out,
                                           float* sc) {
    const float scale = 0.125f;
    // q / out may be register arrays (tensor-core kernel): every loop over the
    // head's 64 columns is fully unrolled so their indices stay static; the
    // key loops stay rolled (scores in the thread's smem scratch `sc`) so the
    // compiler does not hoist 17 rows of K into registers.
#pragma unroll 1
    for (int j = 0; j < kLat; ++j) {
        float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
#pragma unroll
        for (int c4 = 0; c4 < kDh / 4; ++c4) {
            const float4 kk = kv.k4(j, h * (kDh / 4) + c4);
            p0 = fmaf(q[4 * c4], kk.x, p0);
            p1 = fmaf(q[4 * c4 + 1], kk.y, p1);
            p2 = fmaf(q[4 * c4 + 2], kk.z, p2);
            p3 = fmaf(q[4 * c4 + 3], kk.w, p3);
        }
        sc[j] = ((p0 + p1) + (p2 + p3)) * scale;
    }
    float mx = -INFINITY;
    for (int j = 0; j < kLat; ++j)
        if (mlat[j]) mx = fmaxf(mx, sc[j]);
    float tot = 0.f;
    for (int j = 0; j < kLat; ++j) {
        const float e = mlat[j] ? (FAST ? __expf(sc[j] - mx) : expf(sc[j] - mx)) : 0.f;
        sc[j] = e;
        tot += e;
    }
    const float inv = 1.f / tot;
#pragma unroll
    for (int c = 0; c < kDh; ++c) out[c] = 0.f;
#pragma unroll 1
    for (int j = 0; j < kLat; ++j) {
        const float pj = sc[j] * inv;
        if (pj == 0.f) continue;
#pragma unroll
        for (int c4 = 0; c4 < kDh / 4; ++c4) {
            const float4 vv = kv.v4(j, h * (kDh / 4) + c4);
            out[4 * c4] = fmaf(pj, vv.x, out[4 * c4]);
            out[4 * c4 + 1] = fmaf(pj, vv.y, out[4 * c4 + 1]);
            out[4 * c4 + 2] = fmaf(pj, vv.z, out[4 * c4 + 2]);
            out[4 * c4 + 3] = fmaf(pj, vv.w, out[4 * c4 + 3]);
        }
    }
}

struct KV32 {
    const float (*K)[kLd];
    const float (*V)[kLd];
    int base;
    __device__ float4 k4(int j, int q) const { return *reinterpret_cast<const float4*>(&K[base + j][4 * q]); }
    __device__ float4 v4(int j, int q) const { return *reinterpret_cast<const float4*>(&V[base + j][4 * q]); }
};

__global__ void __launch_bounds__(kThreads, 1) k_policy_fp32(const ActArgs a) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    Smem32& sm = *reinterpret_cast<Smem32*>(dsm);
    const PolicyW& W = a.w;
    const int tid = threadIdx.x;
    const int b0 = blockIdx.x * kRows32;
    load_row_inputs<kRows32>(sm.rs, a, b0);
    for (int e = tid; e < kTok32 * kD; e += kThreads) {
        const int s = e / kD, c = e % kD, g = s / kLat;
        sm.X[s][c] = g < kRows32 ? embed_latent(W, a, b0 + g, s % kLat, c) : 0.f;
    }
    __syncthreads();
    // self attention block
    ln_tokens32(sm.X, sm.A, W.self.ln_g, W.self.ln_b);
    __syncthreads();
    gemm32(sm.A, W.self.wq, W.self.bq, sm.Q, false);
    gemm32(sm.A, W.self.wk, W.self.bk, sm.K, false);
    gemm32(sm.A, W.self.wv, W.self.bv, sm.V, false);
    __syncthreads();
    if (tid < kRows32 * kLat * kHeads) {
        const int s = tid >> 1, h = tid & 1, g = s / kLat;
        self_query<false>(h, &sm.Q[s][h * kDh], sm.rs.mlat[g], KV32{sm.K, sm.V, g * kLat}, &sm.A[s][h * kDh], sm.sc[tid]);
    }
    __syncthreads();
    gemm32(sm.A, W.self.wo, W.self.bo, sm.X, true);
    __syncthreads();
    // cross blocks (explicit: indexing the kernel-parameter struct dynamically
    // would copy it to local memory)
    auto cross_block = [&](const AttnW& aw, int m) {
        ln_tokens32(sm.X, sm.A, aw.ln_g, aw.ln_b);
        __syncthreads();
        gemm32(sm.A, aw.wq, aw.bq, sm.Q, false);
        __syncthreads();
        if (tid < kRows32 * kLat * kHeads) {
            const int s = tid >> 1, h = tid & 1, g = s / kLat;
            if (m == 0) cross_query<kRoadF, kRoad, false>(aw, h, &sm.Q[s][h * kDh], sm.rs.road[g], sm.rs.mroad[g], &sm.A[s][h * kDh]);
            if (m == 1) cross_query<kRouteF, kRoute, false>(aw, h, &sm.Q[s][h * kDh], sm.rs.route[g], sm.rs.mroute[g], &sm.A[s][h * kDh]);
            if (m == 2) cross_query<kActF, 1, false>(aw, h, &sm.Q[s][h * kDh], reinterpret_cast<const float(*)[kActF]>(sm.rs.act[g]), sm.rs.mact[g], &sm.A[s][h * kDh]);
        }
        __syncthreads();
        gemm32(sm.A, aw.wo, aw.bo, sm.X, true);
        __syncthreads();
    };
    cross_block(W.road, 0);
    cross_block(W.route, 1);
    cross_block(W.active, 2);
    // mean pool over valid latent tokens (model.hpp:545-554)
    for (int e = tid; e < kRows32 * kD; e += kThreads) {
        const int g = e / kD, c = e % kD;
        float acc = 0.f;
        int n = 0;
        for (int i = 0; i < kLat; ++i)
            if (sm.rs.mlat[g][i]) {
                acc += sm.X[g * kLat + i][c];
                ++n;
            }
        sm.tr.pooled[g][c] = acc / float(n);
    }
    trunk_and_act<kRows32>(sm.rs, sm.tr, a, b0);
}

// ===========================================================================
// k_policy_tc: projections on the 5th-generation tensor cores (tcgen05).
// ===========================================================================
// TMEM columns (512 allocated, lane = token): X residual stream [0,128),
// projection accumulators D0 [128,256), D1 [256,384), D2 [384,512).
constexpr uint32_t kColX = 0, kColD0 = 128, kColD1 = 256, kColD2 = 384;

struct SmemTc {
    float opA[kTokTc * kD];  // A operand: 128 tokens x 128 K, canonical K-major tf32 (64 KB)
    float opW[kD * kD];      // B operand: 128 outputs x 128 K, canonical K-major tf32 (64 KB)
    RowSm<kRowsTc> rs;
    float sc[kThreads][kLat];  // self-attention scores of each thread's query (odd stride: no bank conflicts)
    float red[2][kTokTc];    // LayerNorm partial sums of the two column halves
    float red2[2][kTokTc];
    unsigned long long mbar_w, mbar_mma;
    uint32_t tmem_base;
};
static_assert(offsetof(SmemTc, opW) == 65536, "operand tiles must be contiguous (K/V staging spans both)");

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

// canonical no-swizzle K-major layout: core matrices of 8 rows x 16 B;
// K-adjacent core matrices 2048 B apart (LBO), row-group-adjacent 128 B (SBO)
__device__ __forceinline__ uint32_t canon_off(int row, int k) {  // in floats
    return uint32_t(((k >> 2) * 16 + (row >> 3)) * 32 + (row & 7) * 4 + (k & 3));
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(2048 >> 4) << 16) | (uint64_t(128 >> 4) << 32) |
           (1ull << 46);
}

// kind::tf32, D f32, A/B tf32 K-major, N = 128, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ uint32_t to_tf32(float x) {
    uint32_t u;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
    return u;
}

__device__ __forceinline__ void mbar_init(unsigned long long* m, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(m)),
        "r"(phase));
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 32 consecutive TMEM columns of this thread's lane (warp w reads lanes 32 (w % 4) ..)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
        "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
        "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
        "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
        "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
        "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31])));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

struct TcCtx {
    SmemTc& sm;
    uint32_t tmem;      // allocated base
    uint32_t lane_base; // this warp's TMEM lane quarter << 16
    int tok;            // this thread's token (TMEM lane)
    int half;           // column half / head of this thread
    uint32_t ph_w = 0, ph_mma = 0;

    __device__ uint32_t col(uint32_t c) const { return tmem + lane_base + c; }

    // 64 columns [c0 + 64 half, +64) of this thread's token
    __device__ void ld64(uint32_t c0, float* v) const {
        tmem_ld32(col(c0 + 64 * half), v);
        tmem_ld32(col(c0 + 64 * half + 32), v + 32);
    }
    __device__ void st64(uint32_t c0, const float* v) const {
        tmem_st32(col(c0 + 64 * half), v);
        tmem_st32(col(c0 + 64 * half + 32), v + 32);
    }

    // stream a 64 KB weight tile into opW (one thread issues; async proxy)
    __device__ void load_w(const float* src) {
        if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const uint32_t mb = smem_u32(&sm.mbar_w);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(65536u) : "memory");
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(sm.opW) + 16384u * i),
                    "l"(src + 4096 * i), "r"(16384u), "r"(mb)
                    : "memory");
            }
        }
    }
    __device__ void wait_w() {
        mbar_wait(&sm.mbar_w, ph_w);
        ph_w ^= 1;
    }

    // D[dcol] = opA . opW^T (M = N = 128, K = 128): one thread issues 16 MMAs
    // and commits to mbar_mma; every thread waits for the result.  The caller
    // has made opA (generic stores + proxy fence) and opW (wait_w) visible.
    __device__ void mma(uint32_t dcol) {
        tc_fence_before();
        __syncthreads();
        if (threadIdx.x == 0) {
            tc_fence_after();
            const uint32_t a0 = smem_u32(sm.opA), w0 = smem_u32(sm.opW);
#pragma unroll
            for (int kk = 0; kk < kD / 8; ++kk) {
                const uint64_t da = umma_desc(a0 + kk * 2 * 2048), dw = umma_desc(w0 + kk * 2 * 2048);
                const uint32_t acc = kk > 0;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + dcol),
                    "l"(da), "l"(dw), "r"(kIdesc), "r"(acc)
                    : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&sm.mbar_mma))
                         : "memory");
        }
        mbar_wait(&sm.mbar_mma, ph_mma);
        ph_mma ^= 1;
        tc_fence_after();
    }

    // 64 values of this thread's token / column half into opA (tf32, canonical)
    __device__ void put_a(const float* v) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int k = 64 * half + 4 * q;
            uint4 u = make_uint4(to_tf32(v[4 * q]), to_tf32(v[4 * q + 1]), to_tf32(v[4 * q + 2]), to_tf32(v[4 * q + 3]));
            *reinterpret_cast<uint4*>(sm.opA + canon_off(tok, k)) = u;
        }
    }

    // LayerNorm of this thread's token from X (TMEM) into opA; the two column
    // halves of a token combine their partial sums through smem.
    __device__ void ln_to_a(const float* g, const float* b) {
        float v[64];
        ld64(kColX, v);
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < 64; ++i) s += v[i];
        sm.red[half][tok] = s;
        __syncthreads();
        const float mu = (sm.red[0][tok] + sm.red[1][tok]) / float(kD);
        float q = 0.f;
#pragma unroll
        for (int i = 0; i < 64; ++i) q += (v[i] - mu) * (v[i] - mu);
        sm.red2[half][tok] = q;
        __syncthreads();
        const float rstd = 1.f / sqrtf((sm.red2[0][tok] + sm.red2[1][tok]) / float(kD) + 1e-5f);
#pragma unroll
        for (int i = 0; i < 64; i += 4) {
            const int c = 64 * half + i;
            const float4 gg = __ldg(reinterpret_cast<const float4*>(g + c)), bb = __ldg(reinterpret_cast<const float4*>(b + c));
            v[i] = (v[i] - mu) * rstd * gg.x + bb.x;
            v[i + 1] = (v[i + 1] - mu) * rstd * gg.y + bb.y;
            v[i + 2] = (v[i + 2] - mu) * rstd * gg.z + bb.z;
            v[i + 3] = (v[i + 3] - mu) * rstd * gg.w + bb.w;
        }
        put_a(v);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }

    // X += D[dcol] + bias (the block's residual output projection)
    __device__ void residual_add(uint32_t dcol, const float* bias) {
        float x[64], d[64];
        ld64(kColX, x);
        ld64(dcol, d);
        add64(d, bias + 64 * half);
#pragma unroll
        for (int i = 0; i < 64; ++i) x[i] += d[i];
        st64(kColX, x);
    }
};

struct KVTc {  // self-attention K / V copies in smem: [128 tokens][128], float4 chunks XOR-swizzled by row
    const float* K;
    const float* V;
    int base;
    __device__ static int idx(int r, int c) { return r * kD + ((((c >> 2) ^ (r & 7)) << 2) | (c & 3)); }
    __device__ float4 k4(int j, int q) const {
        const int r = base + j;
        return *reinterpret_cast<const float4*>(K + r * kD + ((q ^ (r & 7)) << 2));
    }
    __device__ float4 v4(int j, int q) const {
        const int r = base + j;
        return *reinterpret_cast<const float4*>(V + r * kD + ((q ^ (r & 7)) << 2));
    }
};

__global__ void __launch_bounds__(kThreads, 1) k_policy_tc(const ActArgs a) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    SmemTc& sm = *reinterpret_cast<SmemTc*>(dsm);
    const PolicyW& W = a.w;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int b0 = blockIdx.x * kRowsTc;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sm.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&sm.mbar_w, 1);
        mbar_init(&sm.mbar_mma, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    TcCtx cx{sm, sm.tmem_base, uint32_t((warp & 3) * 32) << 16, (warp & 3) * 32 + (tid & 31), warp >> 2};
    const int tok = cx.tok, half = cx.half;
    const int g = tok / kLat, slot = tok % kLat;
    const bool real = g < kRowsTc;

    cx.load_w(W.tc[0]);  // self Wq streams in while the inputs are staged
    load_row_inputs<kRowsTc>(sm.rs, a, b0);
    {
        // latent token embedding (model.hpp:510-513), this thread's 64 columns
        float v[64];
        const int b = b0 + g, c0 = 64 * half;
        if (!real) {
#pragma unroll
            for (int i = 0; i < 64; ++i) v[i] = 0.f;
        } else if (slot == 0) {
#pragma unroll
            for (int i = 0; i < 64; ++i) v[i] = __ldg(W.null_ag + c0 + i);
        } else {
            float x[kAgF];
            const float* ag = a.obs.agents + (size_t(b) * kAgents + (slot - 1)) * kAgF;
#pragma unroll
            for (int f = 0; f < kAgF; ++f) x[f] = b < a.B ? ag[f] * c_ag_scale[f] : 0.f;
#pragma unroll
            for (int c4 = 0; c4 < 16; ++c4) {
                const float4 bb = __ldg(reinterpret_cast<const float4*>(W.emb_ag_b + c0 + 4 * c4));
                float o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f;
#pragma unroll
                for (int f = 0; f < kAgF; ++f) {
                    const float4 w4 = __ldg(reinterpret_cast<const float4*>(W.emb_ag_w + f * kD + c0 + 4 * c4));
                    o0 = fmaf(w4.x, x[f], o0);
                    o1 = fmaf(w4.y, x[f], o1);
                    o2 = fmaf(w4.z, x[f], o2);
                    o3 = fmaf(w4.w, x[f], o3);
                }
                v[4 * c4] = o0 + bb.x;
                v[4 * c4 + 1] = o1 + bb.y;
                v[4 * c4 + 2] = o2 + bb.z;
                v[4 * c4 + 3] = o3 + bb.w;
            }
        }
        cx.st64(kColX, v);
    }
    __syncthreads();

    // ---- self attention block (model.hpp:326-367, self_mode) ----
    cx.ln_to_a(W.self.ln_g, W.self.ln_b);
    cx.wait_w();
    cx.mma(kColD0);  // Q
    cx.load_w(W.tc[1]);
    cx.wait_w();
    cx.mma(kColD1);  // K
    cx.load_w(W.tc[2]);
    cx.wait_w();
    cx.mma(kColD2);  // V
    {
        // K, V (+ bias) to smem over both operand tiles (swizzled rows)
        float v[64];
        cx.ld64(kColD1, v);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int c = 64 * half + 4 * q;
            float4 f = make_float4(v[4 * q] + __ldg(W.self.bk + c), v[4 * q + 1] + __ldg(W.self.bk + c + 1),
                                   v[4 * q + 2] + __ldg(W.self.bk + c + 2), v[4 * q + 3] + __ldg(W.self.bk + c + 3));
            *reinterpret_cast<float4*>(sm.opA + KVTc::idx(tok, c)) = f;
        }
        cx.ld64(kColD2, v);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int c = 64 * half + 4 * q;
            float4 f = make_float4(v[4 * q] + __ldg(W.self.bv + c), v[4 * q + 1] + __ldg(W.self.bv + c + 1),
                                   v[4 * q + 2] + __ldg(W.self.bv + c + 2), v[4 * q + 3] + __ldg(W.self.bv + c + 3));
            *reinterpret_cast<float4*>(sm.opW + KVTc::idx(tok, c)) = f;
        }
    }
    __syncthreads();
    {
        float q[64], o[64];
        cx.ld64(kColD0, q);
        add64(q, W.self.bq + 64 * half);
        if (real) {
            self_query<true>(half, q, sm.rs.mlat[g], KVTc{sm.opA, sm.opW, g * kLat}, o, sm.sc[tid]);
        } else {
#pragma unroll
            for (int i = 0; i < 64; ++i) o[i] = 0.f;
        }
        __syncthreads();  // K / V reads done: the operand tiles are free
        cx.load_w(W.tc[3]);
        cx.put_a(o);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    cx.wait_w();
    cx.mma(kColD1);
    cx.residual_add(kColD1, W.self.bo);

    // ---- cross blocks: road, route, active (model.hpp:534-543) ----
    auto cross_block = [&](const AttnW& aw, const float* wq_tc, const float* wo_tc, int m) {
        cx.load_w(wq_tc);
        cx.ln_to_a(aw.ln_g, aw.ln_b);
        cx.wait_w();
        cx.mma(kColD0);
        cx.load_w(wo_tc);  // the output projection streams in during the attention
        // the block's folded weights (Kf, Vf [F][128], ck, cv, kn, vn [128]) to
        // smem, over the self-attention score scratch (dead by now): every
        // thread reads all of them
        const int F = m == 0 ? kRoadF : m == 1 ? kRouteF : kActF;
        float* fw = &sm.sc[0][0];
        for (int e = tid; e < F * kD; e += kThreads) {
            fw[e] = aw.kf[e];
            fw[F * kD + e] = aw.vf[e];
        }
        for (int e = tid; e < kD; e += kThreads) {
            fw[2 * F * kD + e] = aw.ck[e];
            fw[2 * F * kD + kD + e] = aw.cv[e];
            fw[2 * F * kD + 2 * kD + e] = aw.kn[e];
            fw[2 * F * kD + 3 * kD + e] = aw.vn[e];
        }
        __syncthreads();
        AttnW sw = aw;
        sw.kf = fw;
        sw.vf = fw + F * kD;
        sw.ck = fw + 2 * F * kD;
        sw.cv = sw.ck + kD;
        sw.kn = sw.ck + 2 * kD;
        sw.vn = sw.ck + 3 * kD;
        float q[64], o[64];
        cx.ld64(kColD0, q);
        add64(q, aw.bq + 64 * half);
        if (real) {
            if (m == 0) cross_query<kRoadF, kRoad, true>(sw, half, q, sm.rs.road[g], sm.rs.mroad[g], o);
            if (m == 1) cross_query<kRouteF, kRoute, true>(sw, half, q, sm.rs.route[g], sm.rs.mroute[g], o);
            if (m == 2) cross_query<kActF, 1, true>(sw, half, q, reinterpret_cast<const float(*)[kActF]>(sm.rs.act[g]), sm.rs.mact[g], o);
        } else {
#pragma unroll
            for (int i = 0; i < 64; ++i) o[i] = 0.f;
        }
        cx.put_a(o);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        cx.wait_w();
        cx.mma(kColD1);
        cx.residual_add(kColD1, aw.bo);
    };
    cross_block(W.road, W.tc[4], W.tc[5], 0);
    cross_block(W.route, W.tc[6], W.tc[7], 1);
    cross_block(W.active, W.tc[8], W.tc[9], 2);

    // ---- mean pool over valid latent tokens (model.hpp:545-554) ----
    {
        float x[64];
        cx.ld64(kColX, x);
        float* xs = sm.opA;  // [128][132] fp32 over both operand tiles
#pragma unroll
        for (int i = 0; i < 64; ++i) xs[tok * (kD + 4) + 64 * half + i] = x[i];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(sm.tmem_base));
    for (int e = tid; e < kRowsTc * kD; e += kThreads) {
        const int gg = e / kD, c = e % kD;
        float acc = 0.f;
        int n = 0;
        for (int i = 0; i < kLat; ++i)
            if (sm.rs.mlat[gg][i]) {
                acc += sm.opA[(gg * kLat + i) * (kD + 4) + c];
                ++n;
            }
        if (b0 + gg < a.B) a.pooled[size_t(b0 + gg) * kD + c] = acc / float(n);
    }
}

// ===========================================================================
// k_policy_heads: policy / value trunks, heads and the action choice for 128
// rows per CTA (thread = row = TMEM lane); every trunk matrix product is a
// tcgen05.mma.kind::tf32 (M = 128 rows, N = 128, K = 128 or 128 + ve).
// ===========================================================================
constexpr int kHeadRows = 128;
constexpr int kHeadThreads = 512;   // 4 threads per row: warp w owns TMEM lanes 32 (w % 4), columns 32 (w / 4)
constexpr int kMaxK = kD + kMaxVE;  // value.in's K
// TMEM columns: trunk activation H [0,128), products D [128,256), pooled P [256,384)
constexpr uint32_t kHColH = 0, kHColD = 128, kHColP = 256;

struct SmemHeads {
    float opA[kHeadRows * kMaxK];  // canonical K-major tf32, K up to 192
    float opW[kD * kMaxK];
    float hw[2 * kMaxHead][kD];    // accel / steer head weights, row-major [out][k]
    float vhead[kD];
    float red[4][kHeadRows];       // LayerNorm partial sums of the four column quarters
    float red2[4][kHeadRows];
    unsigned long long mbar_w, mbar_mma;
    uint32_t tmem_base;
};

struct HeadsCtx {
    SmemHeads& sm;
    uint32_t tmem, lane_base;
    int row, c0;  // this thread's row (TMEM lane) and first column (32 columns)
    uint32_t ph_w = 0, ph_mma = 0;
    __device__ uint32_t col(uint32_t c) const { return tmem + lane_base + c; }
    __device__ void put(const float* v, int k0) {  // 32 values at columns k0.. of this row, tf32 canonical
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint4 u = make_uint4(to_tf32(v[4 * q]), to_tf32(v[4 * q + 1]), to_tf32(v[4 * q + 2]),
                                       to_tf32(v[4 * q + 3]));
            *reinterpret_cast<uint4*>(sm.opA + canon_off(row, k0 + 4 * q)) = u;
        }
    }
    __device__ void load_w(const float* src, uint32_t bytes) {
        if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const uint32_t mb = smem_u32(&sm.mbar_w);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
            for (uint32_t o = 0; o < bytes; o += 16384u) {
                const uint32_t n = bytes - o < 16384u ? bytes - o : 16384u;
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(sm.opW) + o),
                    "l"(reinterpret_cast<const char*>(src) + o), "r"(n), "r"(mb)
                    : "memory");
            }
        }
    }
    __device__ void wait_w() {
        mbar_wait(&sm.mbar_w, ph_w);
        ph_w ^= 1;
    }
    __device__ void mma(uint32_t dcol, int K) {
        tc_fence_before();
        __syncthreads();
        if (threadIdx.x == 0) {
            tc_fence_after();
            const uint32_t a0 = smem_u32(sm.opA), w0 = smem_u32(sm.opW);
            for (int kk = 0; kk < K / 8; ++kk) {
                const uint64_t da = umma_desc(a0 + kk * 2 * 2048), dw = umma_desc(w0 + kk * 2 * 2048);
                const uint32_t acc = kk > 0;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + dcol),
                    "l"(da), "l"(dw), "r"(kIdesc), "r"(acc)
                    : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&sm.mbar_mma))
                         : "memory");
        }
        mbar_wait(&sm.mbar_mma, ph_mma);
        ph_mma ^= 1;
        tc_fence_after();
    }
    // LayerNorm (model.hpp:287-303) of this row's H into opA; the four column
    // quarters of a row combine their partial sums through smem
    __device__ void ln_to_a(const float* g, const float* b) {
        const int qt = c0 >> 5;
        float v[32];
        tmem_ld32(col(kHColH + c0), v);
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) s += v[i];
        sm.red[qt][row] = s;
        __syncthreads();
        const float mu = ((sm.red[0][row] + sm.red[1][row]) + (sm.red[2][row] + sm.red[3][row])) / float(kD);
        float q = 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) q += (v[i] - mu) * (v[i] - mu);
        sm.red2[qt][row] = q;
        __syncthreads();
        const float var = ((sm.red2[0][row] + sm.red2[1][row]) + (sm.red2[2][row] + sm.red2[3][row])) / float(kD);
        const float rstd = 1.f / sqrtf(var + 1e-5f);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = (v[i] - mu) * rstd * __ldg(g + c0 + i) + __ldg(b + c0 + i);
        put(v, c0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    // mlp_forward (model.hpp:431-440): H += W2 gelu(W1 LN(H) + b1) + b2
    __device__ void mlp(const MlpW& w, const float* w1_tc, const float* w2_tc) {
        load_w(w1_tc, kD * kD * 4);
        ln_to_a(w.ln_g, w.ln_b);
        wait_w();
        mma(kHColD, kD);
        load_w(w2_tc, kD * kD * 4);
        float v[32];
        tmem_ld32(col(kHColD + c0), v);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = gelu(v[i] + __ldg(w.b1 + c0 + i));
        put(v, c0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        wait_w();
        mma(kHColD, kD);
        float h[32];
        tmem_ld32(col(kHColD + c0), v);
        tmem_ld32(col(kHColH + c0), h);
#pragma unroll
        for (int i = 0; i < 32; ++i) h[i] += v[i] + __ldg(w.b2 + c0 + i);
        tmem_st32(col(kHColH + c0), h);
    }
};

__global__ void __launch_bounds__(kHeadThreads, 1) k_policy_heads(const ActArgs a) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    SmemHeads& sm = *reinterpret_cast<SmemHeads*>(dsm);
    const PolicyW& W = a.w;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int row = (warp & 3) * 32 + (tid & 31), c0 = (warp >> 2) * 32;
    const int b = blockIdx.x * kHeadRows + row;
    const bool live = b < a.B;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sm.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&sm.mbar_w, 1);
        mbar_init(&sm.mbar_mma, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const int na = W.n_accel, ns = W.n_steer;
    for (int e = tid; e < (na + ns) * kD; e += kHeadThreads) {
        const int o = e / kD, k = e % kD;
        sm.hw[o][k] = o < na ? W.acc_w[k * na + o] : W.str_w[k * ns + (o - na)];
    }
    for (int k = tid; k < kD; k += kHeadThreads) sm.vhead[k] = W.vhead_w[k];
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    HeadsCtx cx{sm, sm.tmem_base, uint32_t((warp & 3) * 32) << 16, row, c0};

    // pooled encoding -> H and P
    {
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            const float4 t = live ? *reinterpret_cast<const float4*>(a.pooled + size_t(b) * kD + c0 + i)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
            v[i] = t.x, v[i + 1] = t.y, v[i + 2] = t.z, v[i + 3] = t.w;
        }
        tmem_st32(cx.col(kHColH + c0), v);
        tmem_st32(cx.col(kHColP + c0), v);
    }
    // blockIdx.y selects the trunk: 0 = policy trunk, heads and the action
    // choice; 1 = value trunk and head (the two are independent given pooled)
    const bool value_cta = blockIdx.y == 1;
    float logit[2 * kMaxHead];
    float value = 0.f;
    if (!value_cta) {
    // ---- policy trunk (model.hpp:556-562) ----
#pragma unroll
    for (int i = 0; i < kMaxTrunk; ++i)
        if (i < W.trunk) cx.mlp(W.pblk[i], W.tc_pblk[2 * i], W.tc_pblk[2 * i + 1]);
    // ---- heads (model.hpp:563-568): the row's quarter-0 thread, all 128 columns ----
    if (c0 == 0) {
        for (int o = 0; o < na + ns; ++o) logit[o] = o < na ? __ldg(W.acc_b + o) : __ldg(W.str_b + o - na);
        float v[32];
        for (int c = 0; c < kD; c += 32) {
            tmem_ld32(cx.col(kHColH + c), v);
            for (int o = 0; o < na + ns; ++o) {
                float acc = logit[o];
#pragma unroll
                for (int i = 0; i < 32; ++i) acc = fmaf(sm.hw[o][c + i], v[i], acc);
                logit[o] = acc;
            }
        }
    }
    } else {
    // ---- value trunk (model.hpp:570-584): concat [pooled; gelu(W_e v + b_e)] ----
    cx.load_w(W.tc_vin, uint32_t(kD * (kD + W.ve) * 4));
    {
        float v[32];
        tmem_ld32(cx.col(kHColP + c0), v);
        cx.put(v, c0);
        // value embedding, 32 columns per quarter (ve <= 64, a multiple of 8)
        if (c0 < W.ve) {
            float vf[kValF];
#pragma unroll
            for (int f = 0; f < kValF; ++f)
                vf[f] = live ? a.obs.value_only[size_t(b) * kValF + f] * c_val_scale[f] : 0.f;
            const int n = W.ve - c0 < 32 ? W.ve - c0 : 32;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                float acc = 0.f;
                if (i < n) {
#pragma unroll
                    for (int f = 0; f < kValF; ++f) acc = fmaf(__ldg(W.vemb_w + f * W.ve + c0 + i), vf[f], acc);
                    acc = gelu(acc + __ldg(W.vemb_b + c0 + i));
                }
                v[i] = acc;
            }
            cx.put(v, kD + c0);  // columns past ve land in K padding the MMA does not read
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    cx.wait_w();
    cx.mma(kHColD, kD + W.ve);
    {
        float v[32];
        tmem_ld32(cx.col(kHColD + c0), v);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] += __ldg(W.vin_b + c0 + i);
        tmem_st32(cx.col(kHColH + c0), v);
    }
#pragma unroll
    for (int i = 0; i < kMaxTrunk; ++i)
        if (i < W.trunk) cx.mlp(W.vblk[i], W.tc_vblk[2 * i], W.tc_vblk[2 * i + 1]);
    value = __ldg(W.vhead_b);
    if (c0 == 0) {
        float v[32];
        for (int c = 0; c < kD; c += 32) {
            tmem_ld32(cx.col(kHColH + c), v);
#pragma unroll
            for (int i = 0; i < 32; ++i) value = fmaf(sm.vhead[c + i], v[i], value);
        }
    }
    }  // value trunk
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(sm.tmem_base));
    if (!live || c0 != 0) return;
    if (value_cta) {
        a.value[b] = value;
        return;
    }
    // ---- NNPolicy::act (policy.hpp:33-56) ----
    if (a.logits) {
        for (int i = 0; i < na + ns; ++i) a.logits[size_t(b) * (na + ns) + i] = logit[i];
    }
    float la[kMaxHead], ls[kMaxHead];
    for (int i = 0; i < na; ++i) la[i] = logit[i];
    for (int i = 0; i < ns; ++i) ls[i] = logit[na + i];
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

}  // namespace zp

namespace zp {

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
        c->n_steer > kMaxHead || c->value_embed % 8 != 0)
        zs::raise(Err::config, "model: the device policy supports latent 128, 2 heads, obs spec 16/128/64, <= " +
                                   std::to_string(kMaxTrunk) + " trunk blocks, value_embed <= " +
                                   std::to_string(kMaxVE) + " (a multiple of 8), <= 16 bins per head");
}

}  // namespace zp

struct zsim_policy {
    zsim_model_config cfg;
    int device = 0;
    float* blob = nullptr;  // device: reference params followed by the folded cross-attention weights
    zp::PolicyW w{};
    int precision = 1;  // 1 (default): fp32 CUDA cores, the reference's Model<float>; 0: tcgen05 tf32 projections
    float* pooled = nullptr;  // [cap][128] encoder output scratch (tensor-core path)
    int pooled_cap = 0;
    unsigned char* hbuf = nullptr;  // zsim_policy_act_host: device obs + rng + outputs for hcap rows
    int hcap = 0;
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
        // tensor-core tiles of the ten projections: W(n, k) at the canonical
        // K-major no-swizzle position, rounded to tf32 (nearest, ties away)
        const char* proj[zp::kNumProj] = {"enc.self.wq", "enc.self.wk", "enc.self.wv", "enc.self.wo",
                                          "enc.cross.road.wq", "enc.cross.road.wo", "enc.cross.route.wq",
                                          "enc.cross.route.wo", "enc.cross.active.wq", "enc.cross.active.wo"};
        // tile of an out x in weight (128 outputs, K inputs), 1 KB aligned
        auto make_tile = [&](const zp::Entry& e, int K) {
            extra.resize((extra.size() + 255) / 256 * 256);
            const int64_t off = int64_t(extra.size());
            extra.resize(extra.size() + size_t(d) * size_t(K));
            float* t = extra.data() + off;
            for (int n2 = 0; n2 < d; ++n2)
                for (int k = 0; k < K; ++k) {
                    uint32_t u;
                    const float v = params[e.off + int64_t(k) * e.rows + n2];
                    std::memcpy(&u, &v, 4);
                    if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
                    float r;
                    std::memcpy(&r, &u, 4);
                    t[((k >> 2) * 16 + (n2 >> 3)) * 32 + (n2 & 7) * 4 + (k & 3)] = r;
                }
            return off;
        };
        int64_t tc_off[zp::kNumProj], pblk_off[2 * zp::kMaxTrunk], vblk_off[2 * zp::kMaxTrunk];
        for (int i = 0; i < zp::kNumProj; ++i) tc_off[i] = make_tile(find(proj[i]), d);
        for (int i = 0; i < c->trunk_blocks; ++i) {
            const std::string pp = "policy.block" + std::to_string(i), vp = "value.block" + std::to_string(i);
            pblk_off[2 * i] = make_tile(find(pp + ".w1"), d);
            pblk_off[2 * i + 1] = make_tile(find(pp + ".w2"), d);
            vblk_off[2 * i] = make_tile(find(vp + ".w1"), d);
            vblk_off[2 * i + 1] = make_tile(find(vp + ".w2"), d);
        }
        const int64_t vin_off = make_tile(find("value.in.w"), d + c->value_embed);
        std::unique_ptr<zsim_policy> pol(new zsim_policy());
        pol->cfg = *c;
        pol->device = device;
        ccheck(cudaSetDevice(device), "cudaSetDevice");
        const size_t base = (size_t(total) + 255) / 256 * 256;
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
        for (int i = 0; i < zp::kNumProj; ++i) w.tc[i] = D + base + tc_off[i];
        for (int i = 0; i < c->trunk_blocks; ++i) {
            w.tc_pblk[2 * i] = D + base + pblk_off[2 * i];
            w.tc_pblk[2 * i + 1] = D + base + pblk_off[2 * i + 1];
            w.tc_vblk[2 * i] = D + base + vblk_off[2 * i];
            w.tc_vblk[2 * i + 1] = D + base + vblk_off[2 * i + 1];
        }
        w.tc_vin = D + base + vin_off;
        ccheck(cudaFuncSetAttribute(zp::k_policy_heads, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(sizeof(zp::SmemHeads))),
               "cudaFuncSetAttribute(policy heads)");
        ccheck(cudaFuncSetAttribute(zp::k_policy_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(sizeof(zp::SmemTc))),
               "cudaFuncSetAttribute(policy tc)");
        ccheck(cudaFuncSetAttribute(zp::k_policy_fp32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(sizeof(zp::Smem32))),
               "cudaFuncSetAttribute(policy fp32)");
        *out = pol.release();
    });
}

ZSIM_API int zsim_policy_set_precision(zsim_policy* p, int32_t mode) {
    return pguarded([&] {
        if (!p) zs::raise(zs::Err::invalid_argument, "policy_set_precision: null policy");
        if (mode != 0 && mode != 1) zs::raise(zs::Err::invalid_argument, "policy_set_precision: mode must be 0 or 1");
        p->precision = mode;
    });
}

ZSIM_API int zsim_policy_destroy(zsim_policy* p) {
    return pguarded([&] {
        if (!p) return;
        cudaSetDevice(p->device);
        cudaFree(p->blob);
        cudaFree(p->pooled);
        cudaFree(p->hbuf);
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
        const cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (p->precision == 0) {
            if (p->pooled_cap < batch) {
                // grows outside any stream order: the first call at a new size synchronises
                ccheck(cudaDeviceSynchronize(), "policy scratch");
                cudaFree(p->pooled);
                p->pooled = nullptr;
                p->pooled_cap = 0;
                ccheck(cudaMalloc(&p->pooled, size_t(batch) * zp::kD * sizeof(float)), "cudaMalloc(policy scratch)");
                p->pooled_cap = batch;
            }
            a.pooled = p->pooled;
            const int grid = (batch + zp::kRowsTc - 1) / zp::kRowsTc;
            zp::k_policy_tc<<<grid, zp::kThreads, sizeof(zp::SmemTc), s>>>(a);
            const int hgrid = (batch + zp::kHeadRows - 1) / zp::kHeadRows;
            zp::k_policy_heads<<<dim3(hgrid, 2), zp::kHeadThreads, sizeof(zp::SmemHeads), s>>>(a);
        } else {
            const int grid = (batch + zp::kRows32 - 1) / zp::kRows32;
            zp::k_policy_fp32<<<grid, zp::kThreads, sizeof(zp::Smem32), s>>>(a);
        }
        ccheck(cudaGetLastError(), "policy kernel launch");
    });
}

// NNPolicy::act on HOST buffers (the reference's RolloutPolicy interface):
// observations and rng streams are uploaded, the device policy runs, actions
// / logp / value / advanced rng come back.  Synchronous.
ZSIM_API int zsim_policy_act_host(zsim_policy* p, const zsim_obs_view* obs, int32_t batch, uint64_t* rng,
                                  int32_t use_argmax, int32_t* accel, int32_t* steer, float* logp, float* value) {
    return pguarded([&] {
        if (!p || !obs || !accel || !steer || !logp || !value || (!use_argmax && !rng))
            zs::raise(zs::Err::invalid_argument, "policy_act_host: null argument");
        if (batch < 0) zs::raise(zs::Err::invalid_argument, "policy_act_host: negative batch");
        if (batch == 0) return;
        ccheck(cudaSetDevice(p->device), "cudaSetDevice");
        const size_t B = size_t(batch);
        const size_t n[5] = {B * zp::kActF, B * zp::kAgents * zp::kAgF, B * zp::kRoad * zp::kRoadF,
                             B * zp::kRoute * zp::kRouteF, B * zp::kValF};
        auto al = [](size_t v) { return (v + 255) / 256 * 256; };
        size_t off[5], o = 0;
        for (int k = 0; k < 5; ++k) off[k] = o, o += al(n[k] * 4);
        const size_t o_rng = o, o_out = o + al(B * 8);
        const size_t bytes = o_out + 4 * al(B * 4);
        if (p->hcap < batch) {
            cudaFree(p->hbuf);
            p->hbuf = nullptr;
            p->hcap = 0;
            ccheck(cudaMalloc(&p->hbuf, bytes), "cudaMalloc(policy host scratch)");
            p->hcap = batch;
        }
        const float* src[5] = {obs->active, obs->agents, obs->road, obs->route, obs->value_only};
        zsim_obs_view dv;
        float** dst[5] = {&dv.active, &dv.agents, &dv.road, &dv.route, &dv.value_only};
        for (int k = 0; k < 5; ++k) {
            *dst[k] = reinterpret_cast<float*>(p->hbuf + off[k]);
            ccheck(cudaMemcpy(*dst[k], src[k], n[k] * 4, cudaMemcpyHostToDevice), "upload observations");
        }
        uint64_t* drng = reinterpret_cast<uint64_t*>(p->hbuf + o_rng);
        if (rng) ccheck(cudaMemcpy(drng, rng, B * 8, cudaMemcpyHostToDevice), "upload rng");
        auto* da = reinterpret_cast<int32_t*>(p->hbuf + o_out);
        auto* ds = reinterpret_cast<int32_t*>(p->hbuf + o_out + al(B * 4));
        auto* dl = reinterpret_cast<float*>(p->hbuf + o_out + 2 * al(B * 4));
        auto* dvl = reinterpret_cast<float*>(p->hbuf + o_out + 3 * al(B * 4));
        if (zsim_policy_act(p, &dv, batch, drng, use_argmax, da, ds, dl, dvl, nullptr, nullptr) != ZSIM_OK)
            zs::raise(zs::Err::runtime, "policy_act_host: device act failed");
        ccheck(cudaMemcpy(accel, da, B * 4, cudaMemcpyDeviceToHost), "download accel");
        ccheck(cudaMemcpy(steer, ds, B * 4, cudaMemcpyDeviceToHost), "download steer");
        ccheck(cudaMemcpy(logp, dl, B * 4, cudaMemcpyDeviceToHost), "download logp");
        ccheck(cudaMemcpy(value, dvl, B * 4, cudaMemcpyDeviceToHost), "download value");
        if (rng && !use_argmax) ccheck(cudaMemcpy(rng, drng, B * 8, cudaMemcpyDeviceToHost), "download rng");
    });
}

}  // extern "C"
