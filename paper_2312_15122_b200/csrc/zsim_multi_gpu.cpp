// zsim_multi_gpu -- the single-process multi-GPU driver of SURVEY.md §8e:
// one host thread and one stream per GPU, ncclCommInitAll (zsim_comm_init_all),
// scenarios sharded contiguously across the GPUs, no per-step exchange, and one
// int64 episode-stats all-reduce per rollout (zsim_stats_allreduce; the exact,
// order-independent counterpart of the reference's fixed-order
// train::AllReducer, core/train/transport.hpp:59-98).
//
//   zsim_multi_gpu <ndev> <scenarios> <steps> [agents] [road_points] [controlled]
//
// Scenarios come from the stress generator (the global set, each GPU building
// its own shard, zsim_env_create_stress); actions are the benchmark's fixed
// splitmix64 tensor (bench.py / random_actions); throughput runs disable dones
// (simcore.cpp:669).  Prints one JSON line: the all-reduced stats vector (every
// GPU holds the same one), the per-GPU device times and the whole-job
// agent-steps/s over the slowest GPU.  Host C++ over the C-ABI only.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "../../include/zsim_gpu.h"

namespace {

constexpr int kEpisode = 91;

void check(int rc, const char* what) {
    if (rc != ZSIM_OK) {
        std::fprintf(stderr, "%s failed (%d): %s\n", what, rc, zsim_last_error());
        std::exit(1);
    }
}
void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        std::fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e));
        std::exit(1);
    }
}

// bench.py random_actions: splitmix64 (common.hpp:28-44) draws, two per
// (step, row), reduced modulo the bin counts.
void random_actions(int steps, int64_t rows, uint64_t seed, std::vector<int32_t>& accel, std::vector<int32_t>& steer) {
    const uint64_t g = 0x9E3779B97F4A7C15ull;
    const uint64_t state = seed + g;
    accel.resize(size_t(steps) * rows);
    steer.resize(size_t(steps) * rows);
    for (int64_t k = 0; k < int64_t(steps) * rows; ++k) {
        uint64_t v[2];
        for (int h = 0; h < 2; ++h) {
            uint64_t z = state + uint64_t(2 * k + h + 1) * g;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            v[h] = z ^ (z >> 31);
        }
        accel[size_t(k)] = int32_t(v[0] % 7u);
        steer[size_t(k)] = int32_t(v[1] % 5u);
    }
}

struct Result {
    float ms = 0.f;
    int64_t stats[8] = {};
    int64_t rows = 0;
};

}  // namespace

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: %s <ndev> <scenarios> <steps> [agents] [road_points] [controlled]\n", argv[0]);
        return 2;
    }
    const int ndev = std::atoi(argv[1]);
    const int64_t total = std::atoll(argv[2]);
    const int steps = std::atoi(argv[3]);
    const int agents = argc > 4 ? std::atoi(argv[4]) : 32;
    const int points = argc > 5 ? std::atoi(argv[5]) : 2048;
    const int controlled = argc > 6 ? std::atoi(argv[6]) : 0;
    int visible = 0;
    cuda(cudaGetDeviceCount(&visible), "cudaGetDeviceCount");
    if (ndev < 1 || ndev > visible) {
        std::fprintf(stderr, "need 1..%d devices, got %d\n", visible, ndev);
        return 2;
    }
    if (!zsim_comm_available()) {
        std::fprintf(stderr, "NCCL unavailable: %s\n", zsim_last_error());
        return 1;
    }
    std::vector<zsim_comm*> comms(static_cast<size_t>(ndev), nullptr);
    check(zsim_comm_init_all(ndev, nullptr, comms.data()), "zsim_comm_init_all");

    const int64_t rows_per_scen = controlled ? agents : 1;
    std::vector<int32_t> accel, steer;
    random_actions(kEpisode, total * rows_per_scen, 123, accel, steer);
    std::vector<Result> res(static_cast<size_t>(ndev));
    std::vector<std::thread> th;
    for (int g = 0; g < ndev; ++g) {
        th.emplace_back([&, g] {
            cuda(cudaSetDevice(g), "cudaSetDevice");
            const int64_t lo = total * g / ndev, hi = total * (g + 1) / ndev;
            zsim_stress_config sc;
            check(zsim_stress_config_defaults(&sc), "stress defaults");
            sc.count = int32_t(hi - lo);
            sc.first_index = int32_t(lo);
            sc.agents = agents;
            sc.road_points = points;
            sc.flags = controlled ? 1 : 0;
            zsim_sim_config cfg;
            check(zsim_sim_config_defaults(&cfg), "config defaults");
            cfg.disable_dones = 1;
            zsim_env* env = nullptr;
            check(zsim_env_create_stress(&sc, 7, 0, &cfg, g, controlled, &env), "zsim_env_create_stress");
            zsim_env_info info;
            check(zsim_env_get_info(env, &info), "env info");
            const int64_t B = info.batch;
            // this GPU's columns of the global [91][rows] action tensor
            std::vector<int32_t> a(size_t(kEpisode) * B), s(size_t(kEpisode) * B);
            for (int t = 0; t < kEpisode; ++t)
                for (int64_t r = 0; r < B; ++r) {
                    a[size_t(t) * B + r] = accel[size_t(t) * total * rows_per_scen + lo * rows_per_scen + r];
                    s[size_t(t) * B + r] = steer[size_t(t) * total * rows_per_scen + lo * rows_per_scen + r];
                }
            int32_t *da = nullptr, *ds = nullptr;
            int64_t* dstats = nullptr;
            cuda(cudaMalloc(&da, a.size() * 4), "cudaMalloc(actions)");
            cuda(cudaMalloc(&ds, s.size() * 4), "cudaMalloc(actions)");
            cuda(cudaMalloc(&dstats, 8 * sizeof(int64_t)), "cudaMalloc(stats)");
            cuda(cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice), "upload actions");
            cuda(cudaMemcpy(ds, s.data(), s.size() * 4, cudaMemcpyHostToDevice), "upload actions");
            cudaStream_t st;
            cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
            zsim_state_view s0, s1;
            zsim_stepout_view so;
            zsim_obs_view ob;
            check(zsim_state_alloc(env, &s0), "state alloc");
            check(zsim_state_alloc(env, &s1), "state alloc");
            check(zsim_stepout_alloc(env, &so), "stepout alloc");
            check(zsim_obs_alloc(env, &ob), "obs alloc");
            cudaEvent_t e0, e1;
            cuda(cudaEventCreate(&e0), "event");
            cuda(cudaEventCreate(&e1), "event");
            cuda(cudaEventRecord(e0, st), "event record");
            zsim_state_view* cur = &s0;
            zsim_state_view* nxt = &s1;
            for (int k = 0; k < steps; ++k) {
                const int t = k % kEpisode;
                if (t == 0) check(zsim_reset(env, 42, cur, st), "reset");
                check(zsim_step_observe(env, cur, da + size_t(t) * B, ds + size_t(t) * B, nxt, &so, &ob, st),
                      "step_observe");
                std::swap(cur, nxt);
            }
            cuda(cudaEventRecord(e1, st), "event record");
            check(zsim_episode_stats(env, cur, dstats, st), "episode stats");
            // the one cross-GPU exchange: int64 stats summed over every GPU
            check(zsim_stats_allreduce(comms[size_t(g)], dstats, 8, st), "stats allreduce");
            cuda(cudaStreamSynchronize(st), "sync");
            check(zsim_comm_check(comms[size_t(g)]), "nccl async error");
            check(zsim_check_errors(env, st), "device error word");
            cuda(cudaEventElapsedTime(&res[size_t(g)].ms, e0, e1), "elapsed");
            cuda(cudaMemcpy(res[size_t(g)].stats, dstats, sizeof(res[size_t(g)].stats), cudaMemcpyDeviceToHost),
                 "download stats");
            res[size_t(g)].rows = B;
            zsim_state_free(env, &s0);
            zsim_state_free(env, &s1);
            zsim_stepout_free(env, &so);
            zsim_obs_free(env, &ob);
            cudaFree(da);
            cudaFree(ds);
            cudaFree(dstats);
            cudaStreamDestroy(st);
            zsim_env_destroy(env);
        });
    }
    for (auto& t : th) t.join();
    for (auto* c : comms) zsim_comm_destroy(c);
    float worst = 0.f;
    int64_t rows = 0;
    for (const auto& r : res) worst = std::max(worst, r.ms), rows += r.rows;
    for (int g = 1; g < ndev; ++g)
        for (int k = 0; k < 8; ++k)
            if (res[size_t(g)].stats[k] != res[0].stats[k]) {
                std::fprintf(stderr, "stats differ across GPUs after the all-reduce\n");
                return 1;
            }
    const double per_row = controlled ? 1.0 : double(agents);
    std::printf("{\"ndev\": %d, \"scenarios\": %lld, \"rows\": %lld, \"steps\": %d, \"stats\": [", ndev,
                (long long)total, (long long)rows, steps);
    for (int k = 0; k < 8; ++k) std::printf("%s%lld", k ? ", " : "", (long long)res[0].stats[k]);
    std::printf("], \"ms_per_gpu\": [");
    for (int g = 0; g < ndev; ++g) std::printf("%s%.4f", g ? ", " : "", res[size_t(g)].ms);
    std::printf("], \"agent_steps_per_s\": %.6e}\n", double(rows) * per_row * steps / (double(worst) / 1e3));
    return 0;
}
