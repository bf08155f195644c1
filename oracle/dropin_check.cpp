// dropin_check.cpp -- TEST INFRASTRUCTURE: the drop-in demonstration.
//
// Built by oracle/build_oracle.py against the reference sources (in place)
// and libzsim_gpu.so.  The same caller code runs twice, once with
// `SimEnv = zsim::sim::Env` (the reference) and once with
// `SimEnv = zsim::gpu::Env` (include/zsim_gpu.hpp): the reference generator's
// own soundness check (scenario_gen.cpp:528-549, replay of the recovered
// logged actions => no terminal, no events, progress ratio 1 +- 1e-6) and a
// random-action rollout whose EpisodeBatch is compared field by field.
// Prints one JSON line; exit code 0 iff everything matches.
#include <cmath>
#include <cstdio>
#include <memory>
#include <vector>

#include "../include/zsim_gpu.hpp"
#include "core/common.hpp"
#include "core/scenario_gen.hpp"
#include "core/simcore.hpp"

using namespace zsim;

namespace {

template <class SimEnv>
bool replays_clean(const scenario::Scenario& sc, bool disable_dones, double* ratio_out) {
    auto shared = std::make_shared<const scenario::Scenario>(sc);
    auto batch = std::make_shared<const scenario::ScenarioBatch>(scenario::make_batch({shared}, int(sc.num_steps)));
    sim::SimConfig cfg;
    cfg.disable_dones = disable_dones;
    SimEnv env(batch, cfg);
    auto actions = sim::recover_logged_actions(sc, env.action_table(), cfg);
    sim::ScriptedPolicy policy({actions}, env.action_table().nearest_accel(0.0), env.action_table().nearest_steer(0.0));
    auto ep = env.rollout(policy, int(sc.num_steps) - 1, 1);
    double logged = env.logged_progress(0);
    double final_s = ep.s[ep.at(0, int(sc.num_steps) - 2)];
    *ratio_out = (final_s - env.initial_s(0)) / logged;
    return ep.terminal[0] == sim::DoneReason::none && ep.events[0] == 0 && logged >= 0.5 &&
           std::abs(*ratio_out - 1.0) <= 1e-6;
}

struct RandomPolicy final : sim::RolloutPolicy {
    void act(const sim::ObservationBatch& obs, const std::vector<int32_t>& step, std::vector<uint64_t>& rng,
             sim::PolicyOut& out) override {
        (void)step;
        out.resize(obs.batch);
        for (int b = 0; b < obs.batch; ++b) {
            Rng r(rng[size_t(b)]);
            out.accel_idx[size_t(b)] = int32_t(r.uniform_int(7));
            out.steer_idx[size_t(b)] = int32_t(r.uniform_int(5));
            rng[size_t(b)] = r.state;
            // depends on the observation, tie-invariant: distance of the nearest road point
            // (its identity inside an exact d2 tie is unspecified in the reference, roads.cpp:231-232)
            const float* f = obs.road.data() + size_t(b) * size_t(obs.spec.n_road) * 12;
            out.value[size_t(b)] = std::sqrt(f[0] * f[0] + f[1] * f[1]);
        }
    }
};

template <class SimEnv>
sim::EpisodeBatch random_rollout(std::shared_ptr<const scenario::ScenarioBatch> batch, bool disable_dones) {
    sim::SimConfig cfg;
    cfg.disable_dones = disable_dones;
    SimEnv env(batch, cfg);
    RandomPolicy p;
    return env.rollout(p, 91, 7);
}

bool close(float a, float b) { return std::abs(double(a) - double(b)) <= 1e-6 + 1e-5 * std::abs(double(b)); }

}  // namespace

int main() {
    scenario::GeneratorConfig g;
    g.count = 12;
    g.num_steps = 92;
    g.t_bound = 96;
    auto scen = scenario::generate_synthetic(g, 31);
    int clean_ref = 0, clean_gpu = 0, n = 0;
    double worst = 0.0;
    for (const auto& sc : scen) {
        for (bool off : {false, true}) {
            double r1 = 0, r2 = 0;
            clean_ref += replays_clean<sim::Env>(sc, off, &r1) ? 1 : 0;
            clean_gpu += replays_clean<gpu::Env>(sc, off, &r2) ? 1 : 0;
            worst = std::max(worst, std::abs(r2 - 1.0));
            ++n;
        }
    }
    std::vector<std::shared_ptr<const scenario::Scenario>> items;
    for (auto& s : scen) items.push_back(std::make_shared<const scenario::Scenario>(s));
    auto batch = std::make_shared<const scenario::ScenarioBatch>(scenario::make_batch(items, 92));
    long mism_flags = 0, mism_fp = 0, cells = 0;
    for (bool off : {false, true}) {
        auto a = random_rollout<sim::Env>(batch, off);
        auto b = random_rollout<gpu::Env>(batch, off);
        for (size_t k = 0; k < a.mask.size(); ++k) {
            ++cells;
            mism_flags += (a.mask[k] != b.mask[k]) + (a.done[k] != b.done[k]) + (a.accel_idx[k] != b.accel_idx[k]) +
                          (a.steer_idx[k] != b.steer_idx[k]);
            const float* fa[5] = {&a.reward[k], &a.s[k], &a.v[k], &a.a_lat[k], &a.value[k]};
            const float* fb[5] = {&b.reward[k], &b.s[k], &b.v[k], &b.a_lat[k], &b.value[k]};
            static const char* names[5] = {"reward", "s", "v", "a_lat", "value"};
            for (int q = 0; q < 5; ++q) {
                if (!close(*fa[q], *fb[q])) {
                    ++mism_fp;
                    if (mism_fp <= 6)
                        std::fprintf(stderr, "fp mismatch %s cell %zu (row %zu t %zu): ref %.9g gpu %.9g\n", names[q],
                                     k, k / size_t(a.horizon), k % size_t(a.horizon), double(*fa[q]), double(*fb[q]));
                }
            }
        }
        for (int i = 0; i < a.batch; ++i)
            mism_flags += (a.terminal[size_t(i)] != b.terminal[size_t(i)]) + (a.events[size_t(i)] != b.events[size_t(i)]);
    }
    bool ok = clean_ref == n && clean_gpu == n && mism_flags == 0 && mism_fp == 0;
    std::printf(
        "{\"replays\": %d, \"clean_reference\": %d, \"clean_gpu\": %d, \"worst_ratio_error\": %.3g, "
        "\"rollout_cells\": %ld, \"flag_mismatches\": %ld, \"fp_mismatches\": %ld, \"ok\": %s}\n",
        n, clean_ref, clean_gpu, worst, cells, mism_flags, mism_fp, ok ? "true" : "false");
    return ok ? 0 : 1;
}
