// zsim_kernels.cuh -- launch interface between the C-ABI host code and the
// sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include "zsim_pack.cuh"

namespace zs {

constexpr int kThreads = 128;  // threads per CTA (4 warps); one CTA per scenario row at a time
constexpr int kMaxLanes = 64;  // route lanes per scenario (projection walks lanes sequentially)

constexpr int kStatsLen = 8;  // episode-stats vector length

enum { kModeStep = 0, kModeObserve = 1, kModeStepObserve = 2 };

// Per-warp shared-memory carve-up, byte offsets (computed on the host so the
// kernels read them from the parameter bank instead of recomputing them).
struct SmemLayout {
    uint32_t agx, agy, agd, agf, sel;          // agent phase
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
};

size_t smem_bytes(const KernelArgs& a);
cudaError_t launch_step_observe(const KernelArgs& a, int mode, int grid, cudaStream_t stream);
cudaError_t launch_reset(const KernelArgs& a, int grid, cudaStream_t stream);
cudaError_t launch_episode_stats(const KernelArgs& a, const double* initial_s, long long* out, cudaStream_t stream);

}  // namespace zs
