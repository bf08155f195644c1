// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (parity checker / CPU baseline).
//
// A thin extern "C" shim over the UNMODIFIED reference simulator compiled in
// place from /root/reference/proj/src/core/*.cpp by oracle/build_oracle.py
// into oracle/_ref/libzsim_ref.so.  It converts between the reference's
// SimStateBatch / StepOut / ObservationBatch (simcore.hpp:76-131) and the flat
// views of include/zsim_gpu.h so the parity suite can compare the two
// implementations on the same inputs.  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs load this library; the
// product never does.
#include <atomic>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../include/zsim_gpu.h"
#include "core/common.hpp"
#include "core/metrics.hpp"
#include "core/train/replay.hpp"
#include "core/scenario.hpp"
#include "core/scenario_gen.hpp"
#include "core/simcore.hpp"

using namespace zsim;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        return 1 + int(e.kind());
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

sim::SimConfig to_cfg(const zsim_sim_config* c) {
    sim::SimConfig s;
    if (!c) return s;
    s.wheelbase = c->wheelbase;
    s.ego_length = c->ego_length;
    s.ego_width = c->ego_width;
    s.ego_center_offset = c->ego_center_offset;
    s.limits.delta_max = c->delta_max;
    s.limits.v_min = c->v_min;
    s.goal_radius = c->goal_radius;
    s.footprint_margin = c->footprint_margin;
    s.stop_cross_speed = c->stop_cross_speed;
    s.stop_zone = c->stop_zone;
    s.stop_slow_speed = c->stop_slow_speed;
    s.disable_dones = c->disable_dones != 0;
    s.w_progress = c->w_progress;
    s.w_speed = c->w_speed;
    s.w_lat = c->w_lat;
    s.w_lon = c->w_lon;
    s.terminal_penalty = c->terminal_penalty;
    s.n_agents = c->n_agents;
    s.n_road = c->n_road;
    s.n_route = c->n_route;
    s.feature_radius = c->feature_radius;
    s.threads = 1;
    return s;
}

void to_view(const sim::SimStateBatch& st, const zsim_state_view* v) {
    for (int b = 0; b < st.batch; ++b) {
        v->x[b] = st.ego[size_t(b)].x;
        v->y[b] = st.ego[size_t(b)].y;
        v->heading[b] = st.ego[size_t(b)].heading;
        v->v[b] = st.ego[size_t(b)].v;
        v->steering[b] = st.ego[size_t(b)].steering;
        v->t[b] = st.t[size_t(b)];
        v->done[b] = st.done[size_t(b)];
        v->reason[b] = uint8_t(st.reason[size_t(b)]);
        v->rng[b] = st.rng[size_t(b)];
        v->proj_s[b] = st.proj_s[size_t(b)];
        v->proj_d[b] = st.proj_d[size_t(b)];
        v->proj_in_corridor[b] = st.proj_in_corridor[size_t(b)];
        v->events[b] = st.events[size_t(b)];
    }
    if (!st.stopped_flags.empty()) std::memcpy(v->stopped_flags, st.stopped_flags.data(), st.stopped_flags.size());
}

sim::SimStateBatch from_view(const zsim_state_view* v, int B, int total_stop) {
    sim::SimStateBatch st;
    st.batch = B;
    st.ego.resize(size_t(B));
    st.t.resize(size_t(B));
    st.done.resize(size_t(B));
    st.reason.resize(size_t(B));
    st.rng.resize(size_t(B));
    st.proj_s.resize(size_t(B));
    st.proj_d.resize(size_t(B));
    st.proj_in_corridor.resize(size_t(B));
    st.events.resize(size_t(B));
    st.stopped_flags.assign(v->stopped_flags, v->stopped_flags + total_stop);
    for (int b = 0; b < B; ++b) {
        st.ego[size_t(b)] = {v->x[b], v->y[b], v->heading[b], v->v[b], v->steering[b]};
        st.t[size_t(b)] = v->t[b];
        st.done[size_t(b)] = v->done[b];
        st.reason[size_t(b)] = sim::DoneReason(v->reason[b]);
        st.rng[size_t(b)] = v->rng[b];
        st.proj_s[size_t(b)] = v->proj_s[b];
        st.proj_d[size_t(b)] = v->proj_d[b];
        st.proj_in_corridor[size_t(b)] = v->proj_in_corridor[b];
        st.events[size_t(b)] = v->events[b];
    }
    return st;
}

int total_stops(const sim::Env& env) {
    int n = 0;
    for (int b = 0; b < env.batch_size(); ++b) n += int(env.route_context(b).stop_lines.size());
    return n;
}

}  // namespace

struct zref_env {
    std::shared_ptr<const scenario::ScenarioBatch> batch;
    std::unique_ptr<sim::Env> env;
    int total_stop = 0;
};

extern "C" {

__attribute__((visibility("default"))) const char* zref_last_error(void) { return g_err.c_str(); }

// Env(load_batch(Dataset(path), indices, horizon), cfg) (scenario_io.cpp:439-451, simcore.cpp:203-233).
__attribute__((visibility("default"))) int zref_env_create(const char* path, const int64_t* idx, int32_t n,
                                                           int32_t horizon, const zsim_sim_config* cfg,
                                                           zref_env** out) {
    return guarded([&] {
        scenario::Dataset ds(path);
        std::vector<int64_t> rows;
        if (idx) {
            rows.assign(idx, idx + n);
        } else {
            for (int64_t i = 0; i < ds.size(); ++i) rows.push_back(i);
        }
        int h = horizon;
        if (h <= 0) {
            h = 2;
            for (int64_t r : rows) h = std::max(h, int(ds.load(r).num_steps));
        }
        auto e = std::make_unique<zref_env>();
        e->batch = std::make_shared<const scenario::ScenarioBatch>(scenario::load_batch(ds, rows, h));
        e->env = std::make_unique<sim::Env>(e->batch, to_cfg(cfg));
        e->total_stop = total_stops(*e->env);
        *out = e.release();
    });
}

__attribute__((visibility("default"))) void zref_env_destroy(zref_env* e) { delete e; }

__attribute__((visibility("default"))) int zref_env_info(zref_env* e, int32_t* batch, int32_t* horizon,
                                                         int32_t* total_stop) {
    return guarded([&] {
        *batch = e->env->batch_size();
        *horizon = e->env->horizon();
        *total_stop = e->total_stop;
    });
}

__attribute__((visibility("default"))) int zref_scalars(zref_env* e, double* goal_s, double* initial_s,
                                                        double* logged_progress) {
    return guarded([&] {
        for (int b = 0; b < e->env->batch_size(); ++b) {
            goal_s[b] = e->env->goal_s(b);
            initial_s[b] = e->env->initial_s(b);
            logged_progress[b] = e->env->logged_progress(b);
        }
    });
}

__attribute__((visibility("default"))) int zref_init_state(zref_env* e, uint64_t seed, const zsim_state_view* out) {
    return guarded([&] { to_view(e->env->init_state(seed), out); });
}

__attribute__((visibility("default"))) int zref_step(zref_env* e, const zsim_state_view* in, const int32_t* accel,
                                                     const int32_t* steer, const zsim_state_view* out,
                                                     const zsim_stepout_view* so) {
    return guarded([&] {
        int B = e->env->batch_size();
        sim::SimStateBatch st = from_view(in, B, e->total_stop);
        sim::SimStateBatch next;
        sim::StepOut o;
        std::vector<int32_t> a(accel, accel + B), s(steer, steer + B);
        e->env->step(st, a, s, next, o);
        to_view(next, out);
        for (int b = 0; b < B; ++b) {
            so->reward[b] = o.reward[size_t(b)];
            so->event[b] = uint8_t(o.event[size_t(b)]);
            so->s[b] = o.s[size_t(b)];
            so->a_lat[b] = o.a_lat[size_t(b)];
            so->a_lon[b] = o.a_lon[size_t(b)];
            so->v[b] = o.v[size_t(b)];
        }
    });
}

__attribute__((visibility("default"))) int zref_observe(zref_env* e, const zsim_state_view* in,
                                                        const zsim_obs_view* obs) {
    return guarded([&] {
        int B = e->env->batch_size();
        sim::SimStateBatch st = from_view(in, B, e->total_stop);
        sim::ObservationBatch ob;
        e->env->observe(st, ob);
        std::memcpy(obs->active, ob.active.data(), ob.active.size() * 4);
        std::memcpy(obs->agents, ob.agents.data(), ob.agents.size() * 4);
        std::memcpy(obs->road, ob.road.data(), ob.road.size() * 4);
        std::memcpy(obs->route, ob.route.data(), ob.route.size() * 4);
        std::memcpy(obs->value_only, ob.value_only.data(), ob.value_only.size() * 4);
    });
}

// scenario::validate (scenario_io.cpp:193-271) of record `index`; writes the
// first violated invariant (empty string when valid).
__attribute__((visibility("default"))) int zref_validate(const char* path, int64_t index, char* msg, int32_t cap) {
    return guarded([&] {
        scenario::Dataset ds(path);
        auto m = scenario::validate(ds.load(index));
        std::string s = m ? *m : std::string();
        std::strncpy(msg, s.c_str(), size_t(cap - 1));
        msg[cap - 1] = 0;
    });
}

// generate_synthetic (scenario_gen.cpp:601-634) + write_file (scenario_io.cpp:319-345).
__attribute__((visibility("default"))) int zref_generate(int32_t count, int32_t num_steps, double density,
                                                         uint64_t seed, const char* path) {
    return guarded([&] {
        scenario::GeneratorConfig g;
        g.count = count;
        g.num_steps = num_steps;
        g.t_bound = std::max(num_steps, g.t_bound);
        g.density = density;
        auto sc = scenario::generate_synthetic(g, seed);
        scenario::write_file(path, sc);
    });
}

// recover_logged_actions (simcore.cpp:629-652) of record `index`; writes n-1 pairs.
__attribute__((visibility("default"))) int zref_recover_actions(const char* path, int64_t index, int32_t* accel,
                                                                int32_t* steer, int32_t cap, int32_t* n_out) {
    return guarded([&] {
        scenario::Dataset ds(path);
        auto sc = ds.load(index);
        sim::SimConfig cfg;
        auto acts = sim::recover_logged_actions(sc, dyn::ActionTable::defaults(), cfg);
        int n = std::min<int>(cap, int(acts.size()));
        for (int i = 0; i < n; ++i) {
            accel[i] = acts[size_t(i)].first;
            steer[i] = acts[size_t(i)].second;
        }
        *n_out = int32_t(acts.size());
    });
}

// metrics::score_episode + aggregate (metrics.cpp:54-131) over an episode
// recorded by the caller: per-row arrays [B][T] of s, a_lat, a_lon, mask,
// plus events, initial_s and logged_progress.  Writes the Aggregate fields in
// declaration order (metrics.hpp:56-69) as 12 doubles.
__attribute__((visibility("default"))) int zref_aggregate(int32_t B, int32_t T, double dt, const float* s,
                                                          const float* a_lat, const float* a_lon,
                                                          const uint8_t* mask, const uint8_t* events,
                                                          const float* initial_s, const float* logged_progress,
                                                          double* out12) {
    return guarded([&] {
        sim::EpisodeBatch ep;
        ep.batch = B;
        ep.horizon = T;
        ep.dt = dt;
        size_t tot = size_t(B) * size_t(T);
        ep.s.assign(s, s + tot);
        ep.a_lat.assign(a_lat, a_lat + tot);
        ep.a_lon.assign(a_lon, a_lon + tot);
        ep.mask.assign(mask, mask + tot);
        ep.events.assign(events, events + B);
        ep.initial_s.assign(initial_s, initial_s + B);
        ep.logged_progress.assign(logged_progress, logged_progress + B);
        ep.scenario_ids.assign(size_t(B), "x");
        std::vector<metrics::MetricReport> reps;
        for (int b = 0; b < B; ++b) reps.push_back(metrics::score_episode(ep, b, metrics::ScoreBounds{}));
        auto a = metrics::aggregate(reps);
        double v[12] = {double(a.scenarios), double(a.degenerate), a.mean_score, a.mean_relative_progress,
                        a.mean_progress_ratio_raw, a.mean_collision_free, a.mean_off_route_free,
                        a.mean_stop_line_free, a.mean_traffic_light_free, a.mean_comfort, a.failure_rate,
                        a.goal_rate};
        std::memcpy(out12, v, sizeof(v));
    });
}

// Env::rollout (simcore.cpp:554-618) with the reference ScriptedPolicy
// (simcore.cpp:69-84) over a per-row script [B][script_len] of action
// indices; copies every EpisodeBatch array out ([B][T] row-major, B-vectors).
__attribute__((visibility("default"))) int zref_rollout(zref_env* e, int32_t horizon, int32_t script_len,
                                                        const int32_t* accel, const int32_t* steer, uint64_t seed,
                                                        int32_t* o_accel, int32_t* o_steer, float* o_logp,
                                                        float* o_value, float* o_reward, float* o_s, float* o_alat,
                                                        float* o_alon, float* o_v, uint8_t* o_done, uint8_t* o_mask,
                                                        float* o_bootstrap, uint8_t* o_terminal, uint8_t* o_events,
                                                        float* o_initial_s, float* o_logged) {
    return guarded([&] {
        const int B = e->env->batch_size();
        std::vector<std::vector<std::pair<int32_t, int32_t>>> script(static_cast<size_t>(B));
        for (int b = 0; b < B; ++b)
            for (int t = 0; t < script_len; ++t)
                script[size_t(b)].emplace_back(accel[size_t(b) * script_len + t], steer[size_t(b) * script_len + t]);
        const auto& tab = e->env->action_table();
        sim::ScriptedPolicy pol(std::move(script), tab.nearest_accel(0.0), tab.nearest_steer(0.0));
        sim::EpisodeBatch ep = e->env->rollout(pol, horizon, seed);
        const size_t n = size_t(B) * size_t(horizon);
        std::copy(ep.accel_idx.begin(), ep.accel_idx.end(), o_accel);
        std::copy(ep.steer_idx.begin(), ep.steer_idx.end(), o_steer);
        std::copy(ep.logp.begin(), ep.logp.end(), o_logp);
        std::copy(ep.value.begin(), ep.value.end(), o_value);
        std::copy(ep.reward.begin(), ep.reward.end(), o_reward);
        std::copy(ep.s.begin(), ep.s.end(), o_s);
        std::copy(ep.a_lat.begin(), ep.a_lat.end(), o_alat);
        std::copy(ep.a_lon.begin(), ep.a_lon.end(), o_alon);
        std::copy(ep.v.begin(), ep.v.end(), o_v);
        std::copy(ep.done.begin(), ep.done.end(), o_done);
        std::copy(ep.mask.begin(), ep.mask.end(), o_mask);
        (void)n;
        for (int b = 0; b < B; ++b) {
            o_bootstrap[b] = ep.bootstrap[size_t(b)];
            o_terminal[b] = uint8_t(ep.terminal[size_t(b)]);
            o_events[b] = ep.events[size_t(b)];
            o_initial_s[b] = ep.initial_s[size_t(b)];
            o_logged[b] = ep.logged_progress[size_t(b)];
        }
    });
}

// CPU baseline: `threads` per-thread Env shards (threads = 1 each, which
// avoids the Env::Pool startup race) over a contiguous split of
// rows [0, n_rows) of `path` (row r is record r % size).  Each shard runs
// init_state(seed), `warmup` untimed iterations, then `steps` timed
// iterations of observe + step (the rollout body, simcore.cpp:590-609) with
// the [episode_len][n_rows] action tensors, re-initialising the state every
// `episode_len` steps.  Returns wall seconds of the timed loop, max over
// shards (all shards start together).
// The reference's own step benchmark (simcore.cpp:654-699: zero actions,
// dones off, step only), for continuity with the reference's reported
// numbers: mean step ms per batch size (refpy formats bench_csv's columns).
__attribute__((visibility("default"))) int zref_bench_step(const char* path, const int32_t* batch_sizes, int32_t n,
                                                           int32_t steps, int32_t warmup, const zsim_sim_config* cfg,
                                                           double* mean_step_ms) {
    return guarded([&] {
        scenario::Dataset ds(path);
        std::vector<int> bs(batch_sizes, batch_sizes + n);
        const std::vector<sim::BenchRow> rows = sim::bench_step(ds, bs, steps, warmup, to_cfg(cfg));
        for (size_t i = 0; i < rows.size(); ++i) mean_step_ms[i] = rows[i].mean_step_ms;
    });
}

__attribute__((visibility("default"))) int zref_bench(const char* path, int32_t n_rows, int32_t horizon,
                                                      const zsim_sim_config* cfg, int32_t threads, int32_t warmup,
                                                      int32_t steps, int32_t episode_len, const int32_t* accel,
                                                      const int32_t* steer, uint64_t seed, double* seconds) {
    return guarded([&] {
        scenario::Dataset ds(path);
        int nt = std::max(1, std::min<int>(threads, n_rows));
        struct Shard {
            int lo, hi;
            std::shared_ptr<const scenario::ScenarioBatch> batch;
            std::unique_ptr<sim::Env> env;
            double secs = 0.0;
        };
        std::vector<Shard> shards(static_cast<size_t>(nt));
        sim::SimConfig scfg = to_cfg(cfg);
        {
            std::vector<std::thread> build;
            for (int i = 0; i < nt; ++i) {
                build.emplace_back([&, i] {
                    Shard& s = shards[size_t(i)];
                    s.lo = int(int64_t(n_rows) * i / nt);
                    s.hi = int(int64_t(n_rows) * (i + 1) / nt);
                    std::vector<int64_t> rows;
                    for (int r = s.lo; r < s.hi; ++r) rows.push_back(r % ds.size());
                    s.batch = std::make_shared<const scenario::ScenarioBatch>(scenario::load_batch(ds, rows, horizon));
                    s.env = std::make_unique<sim::Env>(s.batch, scfg);
                });
            }
            for (auto& t : build) t.join();
        }
        std::atomic<int> ready{0};
        std::atomic<bool> go{false};
        std::vector<std::thread> ths;
        for (int i = 0; i < nt; ++i) {
            ths.emplace_back([&, i] {
                Shard& s = shards[size_t(i)];
                int B = s.hi - s.lo;
                sim::SimStateBatch st = s.env->init_state(seed), next;
                sim::StepOut out;
                sim::ObservationBatch obs;
                std::vector<int32_t> a(static_cast<size_t>(B)), w(static_cast<size_t>(B));
                auto run = [&](int k) {
                    int t = k % episode_len;
                    if (t == 0 && k > 0) st = s.env->init_state(seed);
                    for (int b = 0; b < B; ++b) {
                        a[size_t(b)] = accel[size_t(t) * n_rows + s.lo + b];
                        w[size_t(b)] = steer[size_t(t) * n_rows + s.lo + b];
                    }
                    s.env->observe(st, obs);
                    s.env->step(st, a, w, next, out);
                    std::swap(st, next);
                };
                for (int k = 0; k < warmup; ++k) run(k);
                ready.fetch_add(1);
                while (!go.load()) std::this_thread::yield();
                auto t0 = std::chrono::steady_clock::now();
                for (int k = warmup; k < warmup + steps; ++k) run(k);
                auto t1 = std::chrono::steady_clock::now();
                s.secs = std::chrono::duration<double>(t1 - t0).count();
            });
        }
        while (ready.load() < nt) std::this_thread::yield();
        go.store(true);
        for (auto& t : ths) t.join();
        double mx = 0.0;
        for (auto& s : shards) mx = std::max(mx, s.secs);
        *seconds = mx;
    });
}

// Env::rollout(ScriptedPolicy) then train::cut_sequences(ep, seq_len)
// (replay.cpp:8-52): sequences in the reference's order; `row` is the batch
// row whose scenario id the sequence carries.  Arrays sized for `cap`
// sequences ([cap][seq_len] steps; obs [cap * seq_len] rows).
__attribute__((visibility("default"))) int zref_rollout_cut(
    zref_env* e, int32_t horizon, int32_t script_len, const int32_t* accel, const int32_t* steer, uint64_t seed,
    int32_t seq_len, int32_t cap, int32_t* count, int32_t* row, float* bootstrap, int32_t* o_accel,
    int32_t* o_steer, float* o_logmu, float* o_reward, uint8_t* o_done, uint8_t* o_mask, float* o_active,
    float* o_agents, float* o_road, float* o_route, float* o_value) {
    return guarded([&] {
        const int B = e->env->batch_size();
        std::vector<std::vector<std::pair<int32_t, int32_t>>> script(static_cast<size_t>(B));
        for (int b = 0; b < B; ++b)
            for (int t = 0; t < script_len; ++t)
                script[size_t(b)].emplace_back(accel[size_t(b) * script_len + t], steer[size_t(b) * script_len + t]);
        const auto& tab = e->env->action_table();
        sim::ScriptedPolicy pol(std::move(script), tab.nearest_accel(0.0), tab.nearest_steer(0.0));
        sim::EpisodeBatch ep = e->env->rollout(pol, horizon, seed);
        std::vector<train::TransitionSequence> seqs = train::cut_sequences(ep, seq_len);
        if (int(seqs.size()) > cap) zsim::fail(zsim::ErrorKind::invalid_argument, "zref_rollout_cut: cap too small");
        *count = int32_t(seqs.size());
        int cursor = 0;
        for (size_t i = 0; i < seqs.size(); ++i) {
            const auto& q = seqs[i];
            while (cursor < B && ep.scenario_ids[size_t(cursor)] != q.scenario_id) ++cursor;
            row[i] = cursor;
            bootstrap[i] = q.bootstrap;
            const auto& sp = q.obs.spec;
            for (int k = 0; k < seq_len; ++k) {
                const size_t o = i * size_t(seq_len) + size_t(k);
                o_accel[o] = q.accel_idx[size_t(k)];
                o_steer[o] = q.steer_idx[size_t(k)];
                o_logmu[o] = q.logmu[size_t(k)];
                o_reward[o] = q.reward[size_t(k)];
                o_done[o] = q.done[size_t(k)];
                o_mask[o] = q.mask[size_t(k)];
            }
            const size_t r0 = i * size_t(seq_len);
            std::copy(q.obs.active.begin(), q.obs.active.end(), o_active + r0 * sim::ObsSpec::active_feat);
            std::copy(q.obs.agents.begin(), q.obs.agents.end(), o_agents + r0 * size_t(sp.n_agents) * 6);
            std::copy(q.obs.road.begin(), q.obs.road.end(), o_road + r0 * size_t(sp.n_road) * 12);
            std::copy(q.obs.route.begin(), q.obs.route.end(), o_route + r0 * size_t(sp.n_route) * 5);
            std::copy(q.obs.value_only.begin(), q.obs.value_only.end(), o_value + r0 * 2);
        }
    });
}

}  // extern "C"
