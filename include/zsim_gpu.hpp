// zsim_gpu.hpp -- header-only drop-in for the reference's zsim::sim::Env
// (/root/reference/proj/src/core/simcore.hpp:191-245), backed by the sm_100a
// library libzsim_gpu.so through the C-ABI in zsim_gpu.h.
//
// Same constructor, method names, argument types, host layouts and error
// behaviour (zsim::Error with the reference's ErrorKind) as zsim::sim::Env, so
// callers switch with a typedef:
//
//     #include "core/simcore.hpp"      // reference types
//     #include "zsim_gpu.hpp"
//     using SimEnv = zsim::gpu::Env;    // was zsim::sim::Env
//
// Compile with the reference's include path (-I<ref>/proj/src) and link
// libzsim_gpu.so.  Everything here is host code; each call crosses into the
// library once (state / actions / outputs copied through pinned staging).
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "core/common.hpp"
#include "core/dynamics.hpp"
#include "core/scenario.hpp"
#include "core/simcore.hpp"
#include "zsim_gpu.h"

namespace zsim::gpu {

namespace detail {

inline void check(int code) {
    if (code == ZSIM_OK) return;
    // C-ABI codes 1..4 follow zsim::ErrorKind (common.hpp:13); CUDA maps to runtime
    ErrorKind k = code >= 1 && code <= 4 ? ErrorKind(code - 1) : ErrorKind::runtime;
    throw Error(k, zsim_last_error());
}

template <class T>
void put(std::string& o, T v) {
    o.append(reinterpret_cast<const char*>(&v), sizeof(T));
}
inline void put_str(std::string& o, const std::string& s) {
    put<uint32_t>(o, uint32_t(s.size()));
    o += s;
}
template <class T>
void put_arr(std::string& o, const std::vector<T>& v) {
    put<uint32_t>(o, uint32_t(v.size()));
    o.append(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(T));
}

// The ZSIM record layout (scenario.hpp:97-104, encode_record scenario_io.cpp:80-130).
inline void encode(std::string& out, const scenario::Scenario& s) {
    std::string r;
    put_str(r, s.id);
    put<uint32_t>(r, s.num_steps);
    put_arr(r, s.ego.x);
    put_arr(r, s.ego.y);
    put_arr(r, s.ego.heading);
    put_arr(r, s.ego.v);
    put<uint32_t>(r, uint32_t(s.agents.size()));
    for (const auto& a : s.agents) {
        put_str(r, a.id);
        put<float>(r, a.length);
        put<float>(r, a.width);
        put_arr(r, a.x);
        put_arr(r, a.y);
        put_arr(r, a.heading);
        put_arr(r, a.speed);
        put_arr(r, a.valid);
    }
    put<uint32_t>(r, uint32_t(s.route.lanes.size()));
    for (const auto& l : s.route.lanes) {
        put<uint32_t>(r, l.lane_id);
        put_arr(r, l.left_xy);
        put_arr(r, l.right_xy);
        put<float>(r, l.s_start);
        put<float>(r, l.s_end);
    }
    put<uint32_t>(r, uint32_t(s.road_features.size()));
    for (const auto& f : s.road_features) {
        put<uint8_t>(r, uint8_t(f.kind));
        put<uint8_t>(r, uint8_t(f.directionality));
        put_arr(r, f.xy);
    }
    put<uint32_t>(r, uint32_t(s.traffic_lights.size()));
    for (const auto& t : s.traffic_lights) {
        put<uint32_t>(r, t.signal_id);
        put<float>(r, t.stop_x);
        put<float>(r, t.stop_y);
        put_arr(r, t.state);
    }
    put<uint32_t>(r, uint32_t(s.stop_lines.size()));
    for (const auto& sl : s.stop_lines) {
        put_arr(r, sl.xy);
        put<float>(r, sl.pos_x);
        put<float>(r, sl.pos_y);
    }
    put<float>(r, s.speed_limit);
    put<float>(r, s.goal_x);
    put<float>(r, s.goal_y);
    put<uint32_t>(out, uint32_t(r.size()));
    out += r;
}

inline zsim_sim_config to_c(const sim::SimConfig& c) {
    zsim_sim_config o;
    zsim_sim_config_defaults(&o);
    o.wheelbase = c.wheelbase;
    o.ego_length = c.ego_length;
    o.ego_width = c.ego_width;
    o.ego_center_offset = c.ego_center_offset;
    o.delta_max = c.limits.delta_max;
    o.v_min = c.limits.v_min;
    o.goal_radius = c.goal_radius;
    o.footprint_margin = c.footprint_margin;
    o.stop_cross_speed = c.stop_cross_speed;
    o.stop_zone = c.stop_zone;
    o.stop_slow_speed = c.stop_slow_speed;
    o.disable_dones = c.disable_dones ? 1 : 0;
    o.w_progress = c.w_progress;
    o.w_speed = c.w_speed;
    o.w_lat = c.w_lat;
    o.w_lon = c.w_lon;
    o.terminal_penalty = c.terminal_penalty;
    o.n_agents = c.n_agents;
    o.n_road = c.n_road;
    o.n_route = c.n_route;
    o.feature_radius = c.feature_radius;
    o.threads = c.threads;
    return o;
}

// SoA scratch mirroring zsim_state_view for the AoS EgoState of SimStateBatch.
struct StateScratch {
    std::vector<double> x, y, h, v, st, ps, pd;
    std::vector<int32_t> t;
    std::vector<uint8_t> done, reason, inc, ev, flags;
    std::vector<uint64_t> rng;
    void resize(int b, int s) {
        for (auto* p : {&x, &y, &h, &v, &st, &ps, &pd}) p->resize(size_t(b));
        t.resize(size_t(b));
        for (auto* p : {&done, &reason, &inc, &ev}) p->resize(size_t(b));
        flags.resize(size_t(s > 0 ? s : 1));
        rng.resize(size_t(b));
    }
    zsim_state_view view() {
        return {x.data(), y.data(), h.data(), v.data(), st.data(), t.data(), done.data(), reason.data(),
                rng.data(), ps.data(), pd.data(), inc.data(), ev.data(), flags.data()};
    }
    void from(const sim::SimStateBatch& s) {
        resize(s.batch, int(s.stopped_flags.size()));
        for (int b = 0; b < s.batch; ++b) {
            const auto& e = s.ego[size_t(b)];
            x[size_t(b)] = e.x, y[size_t(b)] = e.y, h[size_t(b)] = e.heading, v[size_t(b)] = e.v;
            st[size_t(b)] = e.steering;
            reason[size_t(b)] = uint8_t(s.reason[size_t(b)]);
        }
        t = s.t, done = s.done, rng = s.rng, ps = s.proj_s, pd = s.proj_d, inc = s.proj_in_corridor, ev = s.events;
        if (!s.stopped_flags.empty()) flags = s.stopped_flags;
    }
    void to(sim::SimStateBatch& s, int b_count, int stops) const {
        s.batch = b_count;
        s.ego.resize(size_t(b_count));
        s.reason.resize(size_t(b_count));
        for (int b = 0; b < b_count; ++b) {
            s.ego[size_t(b)] = {x[size_t(b)], y[size_t(b)], h[size_t(b)], v[size_t(b)], st[size_t(b)]};
            s.reason[size_t(b)] = sim::DoneReason(reason[size_t(b)]);
        }
        s.t = t, s.done = done, s.rng = rng, s.proj_s = ps, s.proj_d = pd, s.proj_in_corridor = inc, s.events = ev;
        s.stopped_flags.assign(flags.begin(), flags.begin() + stops);
    }
};

}  // namespace detail

class Env {
public:
    Env(std::shared_ptr<const scenario::ScenarioBatch> batch, sim::SimConfig config,
        dyn::ActionTable table = dyn::ActionTable::defaults(), int device = 0)
        : batch_(std::move(batch)), config_(config), table_(std::move(table)) {
        table_.validated();
        std::string img("ZSIM", 4);
        detail::put<uint16_t>(img, scenario::kFormatVersion);
        detail::put<uint16_t>(img, 0);
        detail::put<double>(img, batch_->dt);
        for (const auto& sc : batch_->items) detail::encode(img, *sc);
        zsim_sim_config c = detail::to_c(config_);
        detail::check(zsim_env_create(reinterpret_cast<const uint8_t*>(img.data()), img.size(), nullptr, 0,
                                      batch_->horizon, &c, table_.accel_bins.data(), table_.num_accel(),
                                      table_.steer_rate_bins.data(), table_.num_steer(), device, &env_));
        detail::check(zsim_env_get_info(env_, &info_));
        goal_s_.resize(size_t(info_.batch));
        initial_s_.resize(size_t(info_.batch));
        logged_.resize(size_t(info_.batch));
        detail::check(zsim_env_get_scalars(env_, goal_s_.data(), initial_s_.data(), logged_.data()));
    }
    ~Env() { zsim_env_destroy(env_); }
    Env(const Env&) = delete;
    Env& operator=(const Env&) = delete;

    int batch_size() const { return batch_->batch; }
    int horizon() const { return batch_->horizon; }
    double dt() const { return batch_->dt; }
    const sim::SimConfig& config() const { return config_; }
    const dyn::ActionTable& action_table() const { return table_; }
    const scenario::ScenarioBatch& batch() const { return *batch_; }
    double goal_s(int b) const { return goal_s_[size_t(b)]; }
    double logged_progress(int b) const { return logged_[size_t(b)]; }
    double initial_s(int b) const { return initial_s_[size_t(b)]; }

    // Env::init_state (simcore.cpp:237-276)
    sim::SimStateBatch init_state(uint64_t seed) const {
        detail::StateScratch s;
        s.resize(info_.batch, info_.total_stop_lines);
        zsim_state_view v = s.view();
        detail::check(zsim_reset_host(env_, seed, &v));
        sim::SimStateBatch out;
        s.to(out, info_.batch, info_.total_stop_lines);
        return out;
    }

    // Env::step (simcore.cpp:406-421); `next` may alias `state`
    void step(const sim::SimStateBatch& state, const std::vector<int32_t>& accel_idx,
              const std::vector<int32_t>& steer_idx, sim::SimStateBatch& next, sim::StepOut& out) const {
        const int b = batch_size();
        if (int(accel_idx.size()) != b || int(steer_idx.size()) != b || state.batch != b)
            fail(ErrorKind::invalid_argument, "env_step: action/state shape mismatch");
        detail::StateScratch in, o;
        in.from(state);
        o.resize(b, info_.total_stop_lines);
        zsim_state_view vi = in.view(), vo = o.view();
        out.resize(b);
        std::vector<uint8_t> ev(static_cast<size_t>(b));
        zsim_stepout_view so{out.reward.data(), ev.data(), out.s.data(), out.a_lat.data(), out.a_lon.data(),
                             out.v.data()};
        detail::check(zsim_step_host(env_, &vi, accel_idx.data(), steer_idx.data(), &vo, &so));
        for (int i = 0; i < b; ++i) out.event[size_t(i)] = sim::DoneReason(ev[size_t(i)]);
        o.to(next, b, info_.total_stop_lines);
    }

    // Env::observe (simcore.cpp:540-552)
    void observe(const sim::SimStateBatch& state, sim::ObservationBatch& obs) const {
        sim::ObsSpec spec;
        spec.n_agents = config_.n_agents;
        spec.n_road = config_.n_road;
        spec.n_route = config_.n_route;
        if (obs.batch != batch_size() || !(obs.spec == spec)) obs.resize(spec, batch_size());
        detail::StateScratch in;
        in.from(state);
        zsim_state_view vi = in.view();
        zsim_obs_view vo{obs.active.data(), obs.agents.data(), obs.road.data(), obs.route.data(),
                         obs.value_only.data()};
        detail::check(zsim_observe_host(env_, &vi, &vo));
    }

    // Env::rollout (simcore.cpp:554-618): the same loop over the device step.
    sim::EpisodeBatch rollout(sim::RolloutPolicy& policy, int horizon, uint64_t seed) const {
        const int b = batch_size();
        sim::EpisodeBatch ep;
        ep.batch = b;
        ep.horizon = horizon;
        ep.dt = dt();
        const size_t total = size_t(b) * size_t(horizon);
        ep.obs.resize(size_t(horizon));
        ep.accel_idx.assign(total, 0);
        ep.steer_idx.assign(total, 0);
        for (auto* v : {&ep.logp, &ep.value, &ep.reward, &ep.s, &ep.a_lat, &ep.a_lon, &ep.v}) v->assign(total, 0.f);
        ep.done.assign(total, 0);
        ep.mask.assign(total, 0);
        ep.bootstrap.assign(size_t(b), 0.f);
        ep.terminal.assign(size_t(b), sim::DoneReason::none);
        ep.events.assign(size_t(b), 0);
        ep.initial_s.resize(size_t(b));
        ep.logged_progress.resize(size_t(b));
        ep.scenario_ids.resize(size_t(b));
        for (int i = 0; i < b; ++i) {
            ep.scenario_ids[size_t(i)] = batch_->items[size_t(i)]->id;
            ep.logged_progress[size_t(i)] = float(logged_[size_t(i)]);
        }
        sim::SimStateBatch state = init_state(seed), next;
        sim::StepOut sout;
        sim::PolicyOut pout;
        for (int i = 0; i < b; ++i) ep.initial_s[size_t(i)] = float(state.proj_s[size_t(i)]);
        for (int t = 0; t < horizon; ++t) {
            observe(state, ep.obs[size_t(t)]);
            policy.act(ep.obs[size_t(t)], state.t, state.rng, pout);
            step(state, pout.accel_idx, pout.steer_idx, next, sout);
            for (int i = 0; i < b; ++i) {
                size_t k = ep.at(i, t);
                ep.mask[k] = state.done[size_t(i)] ? 0 : 1;
                ep.accel_idx[k] = pout.accel_idx[size_t(i)];
                ep.steer_idx[k] = pout.steer_idx[size_t(i)];
                ep.logp[k] = pout.logp[size_t(i)];
                ep.value[k] = pout.value[size_t(i)];
                ep.reward[k] = sout.reward[size_t(i)];
                ep.s[k] = sout.s[size_t(i)];
                ep.a_lat[k] = sout.a_lat[size_t(i)];
                ep.a_lon[k] = sout.a_lon[size_t(i)];
                ep.v[k] = sout.v[size_t(i)];
                ep.done[k] = next.done[size_t(i)];
            }
            std::swap(state, next);
        }
        observe(state, ep.final_obs);
        policy.act(ep.final_obs, state.t, state.rng, pout);
        for (int i = 0; i < b; ++i) {
            ep.bootstrap[size_t(i)] = state.done[size_t(i)] ? 0.f : pout.value[size_t(i)];
            ep.terminal[size_t(i)] = state.reason[size_t(i)];
            ep.events[size_t(i)] = state.events[size_t(i)];
        }
        return ep;
    }

    zsim_env* handle() const { return env_; }  // device fast path (zsim_step_observe etc.)

private:
    std::shared_ptr<const scenario::ScenarioBatch> batch_;
    sim::SimConfig config_;
    dyn::ActionTable table_;
    zsim_env* env_ = nullptr;
    zsim_env_info info_{};
    std::vector<double> goal_s_, initial_s_, logged_;
};

// Drop-in for train::NNPolicy (train/policy.hpp:19-58) as a host
// sim::RolloutPolicy: the snapshot's flat Model<float>::params (ParamIndex
// order) run on the device policy kernels; usable with either Env::rollout.
class NNPolicy final : public sim::RolloutPolicy {
public:
    // precision: Fp32 (default) computes like the reference's Model<float>;
    // Tf32 runs the projections on the tcgen05 tensor cores (logits ~1e-4 from
    // fp32: an action can differ where its decision margin is that small).
    enum class Precision { Fp32 = 1, Tf32 = 0 };
    NNPolicy(const std::vector<float>& params, bool use_argmax, int device = 0,
             const zsim_model_config* cfg = nullptr, Precision precision = Precision::Fp32)
        : argmax_(use_argmax) {
        zsim_model_config c;
        if (cfg) {
            c = *cfg;
        } else {
            detail::check(zsim_model_config_defaults(&c));
        }
        detail::check(zsim_policy_create(&c, params.data(), int64_t(params.size()), device, &pol_));
        const int rc = zsim_policy_set_precision(pol_, int32_t(precision));
        if (rc != ZSIM_OK) {
            zsim_policy_destroy(pol_);
            pol_ = nullptr;
            detail::check(rc);
        }
    }
    NNPolicy(const NNPolicy&) = delete;
    NNPolicy& operator=(const NNPolicy&) = delete;
    ~NNPolicy() override {
        if (pol_) zsim_policy_destroy(pol_);
    }

    void act(const sim::ObservationBatch& obs, const std::vector<int32_t>& step_index, std::vector<uint64_t>& rng,
             sim::PolicyOut& out) override {
        (void)step_index;
        const int b = obs.batch;
        if (rng.size() < size_t(b))  // one stream per row (train/policy.hpp:40-52)
            fail(ErrorKind::invalid_argument, "NNPolicy::act: rng has fewer streams than rows");
        out.accel_idx.resize(size_t(b));
        out.steer_idx.resize(size_t(b));
        out.logp.resize(size_t(b));
        out.value.resize(size_t(b));
        zsim_obs_view v{const_cast<float*>(obs.active.data()), const_cast<float*>(obs.agents.data()),
                        const_cast<float*>(obs.road.data()), const_cast<float*>(obs.route.data()),
                        const_cast<float*>(obs.value_only.data())};
        detail::check(zsim_policy_act_host(pol_, &v, b, rng.data(), argmax_ ? 1 : 0, out.accel_idx.data(),
                                           out.steer_idx.data(), out.logp.data(), out.value.data()));
    }

    zsim_policy* handle() const { return pol_; }  // device fast path (zsim_policy_act, zsim_rollout_policy)

private:
    zsim_policy* pol_ = nullptr;
    bool argmax_;
};

}  // namespace zsim::gpu
