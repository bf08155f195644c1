// zsim_kernels.cuh -- launch interface between the C-ABI host code and the
// sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include "zsim_pack.cuh"

namespace zs {

constexpr int kThreads = 128;  // threads per CTA of the small kernels (reset, ...)
// k_step_observe CTAs: 14 warps (two CTAs fill an SM's 28 warps) when the
// per-warp shared memory allows, else 4; one warp per scenario row at a time
constexpr int kCtaWarpsBig = 14, kCtaWarpsSmall = 4;
// the split road / route top-k kernel: 12-warp CTAs, 36 warps per SM
constexpr int kCtaWarpsMap = 12, kMapWarpsPerSm = 36;
// the split step + agents kernel for controlled rows: 16-warp CTAs, 32 warps per SM
constexpr int kCtaWarpsCtl = 16, kCtlWarpsPerSm = 32;
constexpr int kMaxLanes = 64;  // route lanes per scenario (projection walks lanes sequentially)

constexpr int kStatsLen = 8;  // episode-stats vector length

enum { kModeStep = 0, kModeObserve = 1, kModeStepObserve = 2 };

// Per-warp shared-memory carve-up, byte offsets (computed on the host so the
// kernels read them from the parameter bank instead of recomputing them).
struct SmemLayout {
    uint32_t agx, agy, agd, agf, sel, alist;   // agent phase
    uint32_t hist, cidx, ckey, cinfo, order;                    // top-k phase (overlays the agent phase)
    uint32_t sflag, total;
};

struct KernelArgs {
    DevPack pk;
    DevCfg cfg;
    zsim_state_view in;
    zsim_state_view out;
    const int32_t* accel;
    const int32_t* steer;
    zsim_stepout_view so;
    zsim_obs_view obs;
    int32_t* dbg;
    int32_t* err;
    uint64_t seed;
    float4* hint;      // [B] per-row top-k threshold hints (speed only; see warp_topk), may be null
    int32_t key_cap;   // >= max(P, R)
    int32_t cand_cap;  // top-k candidate capacity per warp (= 32 x kMaxCandPerLane)
    SmemLayout lay;    // filled by the launchers
    // device rollout (zsim_rollout): recording target and scripted actions
    zsim_episode_view ep;  // ep.reward == nullptr: no recording
    int32_t ep_t;          // rollout step being recorded
    int32_t act_len;       // > 0: accel/steer are a [act_len][B] script read at state.t (ScriptedPolicy); -1: empty;
                           // -2: accel/steer [B] are this step's policy output (NNPolicy), recorded for every row
    const float* pol_logp;   // policy rollout: this step's logp / value [B] to record (null: 0, ScriptedPolicy)
    const float* pol_value;
    const float* final_value;  // episode finalize: bootstrap value [B] (null: 0)
    int32_t zero_accel, zero_steer;
    int32_t row_lo, row_hi;  // rows [row_lo, row_hi) of the batch; row_hi == 0: all rows
};

size_t smem_bytes(const KernelArgs& a);  // per CTA of k_step_observe (its CTA size: step_observe_warps)
int step_observe_warps(const KernelArgs& a);
// policy: 0 auto (split the observation into separate kernels beyond one wave), 1 fused, 2 split
cudaError_t launch_step_observe(const KernelArgs& a, int mode, int policy, cudaStream_t stream);
bool observe_split(const KernelArgs& a, int policy);  // the arrangement launch_step_observe picks
cudaError_t launch_reset(const KernelArgs& a, int grid, cudaStream_t stream);
cudaError_t launch_episode_stats(const KernelArgs& a, const double* initial_s, long long* out, cudaStream_t stream);
// EpisodeBatch tail (bootstrap / terminal / events / initial_s / logged_progress) from the final state a.in
cudaError_t launch_episode_finalize(const KernelArgs& a, const double* initial_s, const double* logged,
                                   cudaStream_t stream);
// score_episode per row + fixed-order Aggregate partial sums (double[12]) of a.ep
cudaError_t launch_episode_metrics(const KernelArgs& a, const zsim_score_bounds& bounds,
                                   const zsim_comfort_weights& weights, const zsim_metric_view& rows, double* sums,
                                   double* scratch, cudaStream_t stream);
int metrics_scratch_doubles(int B);
// train::cut_sequences (replay.cpp:8-52): `obs` is a DEVICE array of T
// observation views; `scratch` holds B + 1 int32 (per-row sequence offsets)
cudaError_t launch_cut_sequences(int B, int T, int L, const zsim_episode_view& ep, const zsim_obs_view* obs,
                                 const zsim_sequences_view& out, int ka, int kr, int kl, int32_t* scratch,
                                 cudaStream_t stream);

}  // namespace zs
