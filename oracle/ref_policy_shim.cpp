// ref_policy_shim.cpp -- TEST INFRASTRUCTURE ONLY (policy parity checker).
//
// extern "C" entry points over the reference's UNMODIFIED policy code:
// core/nn/model.hpp (ParamIndex, Model::init, forward_row, log_softmax,
// sample_categorical, argmax) and core/train/policy.hpp (NNPolicy::act),
// compiled in place with oracle/eigen_mini standing in for Eigen (absent from
// this image).  Built into oracle/_ref/libzsim_ref.so by oracle/build_oracle.py;
// loaded only by tests/ (the product never does).
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../include/zsim_gpu.h"
#include "core/nn/model.hpp"
#include "core/train/policy.hpp"

using namespace zsim;

namespace {
thread_local std::string g_perr;

template <class F>
int pguarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_perr = e.what();
        return 1 + int(e.kind());
    } catch (const std::exception& e) {
        g_perr = e.what();
        return 4;
    }
}

// zsim_model_config (include/zsim_gpu.h) -> nn::ModelConfig (model.hpp:20-36)
nn::ModelConfig to_mcfg(const zsim_model_config* c) {
    nn::ModelConfig m;
    if (!c) return m;
    m.latent = c->latent;
    m.heads = c->heads;
    m.trunk_blocks = c->trunk_blocks;
    m.value_embed = c->value_embed;
    m.obs.n_agents = c->n_agents;
    m.obs.n_road = c->n_road;
    m.obs.n_route = c->n_route;
    m.n_accel = c->n_accel;
    m.n_steer = c->n_steer;
    return m;
}

sim::ObservationBatch to_obs(const nn::ModelConfig& m, const zsim_obs_view* v, int B) {
    sim::ObservationBatch o;
    o.resize(m.obs, B);
    std::memcpy(o.active.data(), v->active, o.active.size() * sizeof(float));
    std::memcpy(o.agents.data(), v->agents, o.agents.size() * sizeof(float));
    std::memcpy(o.road.data(), v->road, o.road.size() * sizeof(float));
    std::memcpy(o.route.data(), v->route, o.route.size() * sizeof(float));
    std::memcpy(o.value_only.data(), v->value_only, o.value_only.size() * sizeof(float));
    return o;
}

template <class T>
nn::Model<T> make_model(const nn::ModelConfig& mc, const float* params, int64_t n) {
    nn::Model<float> mf = nn::Model<float>::make(mc);
    if (n != mf.param_count()) fail(ErrorKind::invalid_argument, "policy params: size does not match the config");
    std::memcpy(mf.params.data(), params, size_t(n) * sizeof(float));
    if constexpr (std::is_same<T, float>::value) {
        return mf;
    } else {
        return mf.template cast<T>();  // Model::cast (model.hpp:218-226)
    }
}

template <class T>
void forward_all(const nn::ModelConfig& mc, const float* params, int64_t n, const zsim_obs_view* obs, int B,
                 double* logits, double* value) {
    const nn::Model<T> m = make_model<T>(mc, params, n);
    const sim::ObservationBatch o = to_obs(mc, obs, B);
    nn::RowCache<T> cache;
    const int na = mc.n_accel, ns = mc.n_steer;
    for (int b = 0; b < B; ++b) {
        nn::forward_row(m, o, b, cache);
        for (int i = 0; i < na; ++i) logits[size_t(b) * (na + ns) + i] = double(cache.logits_accel[i]);
        for (int i = 0; i < ns; ++i) logits[size_t(b) * (na + ns) + na + i] = double(cache.logits_steer[i]);
        value[b] = double(cache.value);
    }
}
}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* zref_policy_last_error(void) { return g_perr.c_str(); }

// nn::ParamIndex total (model.hpp:86-166)
__attribute__((visibility("default"))) int zref_policy_param_count(const zsim_model_config* cfg, int64_t* out) {
    return pguarded([&] { *out = nn::ParamIndex::build(to_mcfg(cfg)).total; });
}

// Model<float>::make + init(seed) (model.hpp:174-216)
__attribute__((visibility("default"))) int zref_policy_init(const zsim_model_config* cfg, uint64_t seed, float* out,
                                                            int64_t n) {
    return pguarded([&] {
        nn::Model<float> m = nn::Model<float>::make(to_mcfg(cfg));
        if (n != m.param_count()) fail(ErrorKind::invalid_argument, "init: output size does not match the config");
        m.init(seed);
        std::memcpy(out, m.params.data(), size_t(n) * sizeof(float));
    });
}

// forward_row (model.hpp:464-585) over B observation rows: logits
// [B][n_accel + n_steer] and values [B], in Model<float> (dbl = 0, the
// reference's own arithmetic) or Model<double> (dbl = 1).
__attribute__((visibility("default"))) int zref_policy_forward(const zsim_model_config* cfg, const float* params,
                                                               int64_t n, const zsim_obs_view* obs, int32_t B,
                                                               int32_t dbl, double* logits, double* value) {
    return pguarded([&] {
        const nn::ModelConfig mc = to_mcfg(cfg);
        if (dbl)
            forward_all<double>(mc, params, n, obs, B, logits, value);
        else
            forward_all<float>(mc, params, n, obs, B, logits, value);
    });
}

// train::NNPolicy::act (policy.hpp:27-58) with one thread: actions, joint
// log-prob, value; rng streams advanced in place (sampling mode).
__attribute__((visibility("default"))) int zref_policy_act(const zsim_model_config* cfg, const float* params, int64_t n,
                                                           const zsim_obs_view* obs, int32_t B, int32_t use_argmax,
                                                           uint64_t* rng, int32_t* accel, int32_t* steer, float* logp,
                                                           float* value) {
    return pguarded([&] {
        const nn::ModelConfig mc = to_mcfg(cfg);
        auto snap = std::make_shared<train::PolicySnapshot>();
        snap->model = make_model<float>(mc, params, n);
        train::NNPolicy pol(snap, use_argmax != 0, 1);
        const sim::ObservationBatch o = to_obs(mc, obs, B);
        std::vector<int32_t> step(size_t(B), 0);
        std::vector<uint64_t> r(rng, rng + B);
        sim::PolicyOut out;
        pol.act(o, step, r, out);
        for (int b = 0; b < B; ++b) {
            accel[b] = out.accel_idx[size_t(b)];
            steer[b] = out.steer_idx[size_t(b)];
            logp[b] = out.logp[size_t(b)];
            value[b] = out.value[size_t(b)];
            rng[b] = r[size_t(b)];
        }
    });
}
}
