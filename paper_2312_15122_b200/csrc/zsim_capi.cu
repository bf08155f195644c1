// zsim_capi.cu -- the extern "C" boundary (include/zsim_gpu.h): environment
// staging, device buffers, copies and kernel launches.  Host C++.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <exception>
#include <functional>
#include <future>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/zsim_gpu.h"
#include "zsim_geom.cuh"
#include "zsim_kernels.cuh"
#include "zsim_pack.cuh"
#include "zsim_scenario.hpp"

namespace zs {
std::string stress_generate(const zsim_stress_config& cfg, uint64_t seed);
}

using zs::Err;
using zs::Error;
using zs::raise;

namespace {

thread_local std::string g_last_error;

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) raise(Err::cuda, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return ZSIM_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return int(e.kind);
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return ZSIM_RUNTIME;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return ZSIM_RUNTIME;
    }
}

size_t al(size_t v) { return (v + 255) / 256 * 256; }

// Layout of a SoA block carved from one allocation.
struct StateLayout {
    size_t off[14];
    size_t bytes;
};

StateLayout state_layout(int B, int S) {
    const size_t sz[14] = {8, 8, 8, 8, 8, 4, 1, 1, 8, 8, 8, 1, 1, 1};
    StateLayout L;
    size_t o = 0;
    for (int i = 0; i < 14; ++i) {
        L.off[i] = o;
        o += al(sz[i] * size_t(i == 13 ? std::max(S, 1) : B));
    }
    L.bytes = o;
    return L;
}

void carve_state(unsigned char* base, const StateLayout& L, zsim_state_view* v) {
    v->x = reinterpret_cast<double*>(base + L.off[0]);
    v->y = reinterpret_cast<double*>(base + L.off[1]);
    v->heading = reinterpret_cast<double*>(base + L.off[2]);
    v->v = reinterpret_cast<double*>(base + L.off[3]);
    v->steering = reinterpret_cast<double*>(base + L.off[4]);
    v->t = reinterpret_cast<int32_t*>(base + L.off[5]);
    v->done = base + L.off[6];
    v->reason = base + L.off[7];
    v->rng = reinterpret_cast<uint64_t*>(base + L.off[8]);
    v->proj_s = reinterpret_cast<double*>(base + L.off[9]);
    v->proj_d = reinterpret_cast<double*>(base + L.off[10]);
    v->proj_in_corridor = base + L.off[11];
    v->events = base + L.off[12];
    v->stopped_flags = base + L.off[13];
}

struct StepoutLayout {
    size_t off[6];
    size_t bytes;
};
StepoutLayout stepout_layout(int B) {
    const size_t sz[6] = {4, 1, 4, 4, 4, 4};
    StepoutLayout L;
    size_t o = 0;
    for (int i = 0; i < 6; ++i) {
        L.off[i] = o;
        o += al(sz[i] * size_t(B));
    }
    L.bytes = o;
    return L;
}
void carve_stepout(unsigned char* base, const StepoutLayout& L, zsim_stepout_view* v) {
    v->reward = reinterpret_cast<float*>(base + L.off[0]);
    v->event = base + L.off[1];
    v->s = reinterpret_cast<float*>(base + L.off[2]);
    v->a_lat = reinterpret_cast<float*>(base + L.off[3]);
    v->a_lon = reinterpret_cast<float*>(base + L.off[4]);
    v->v = reinterpret_cast<float*>(base + L.off[5]);
}

struct ObsLayout {
    size_t off[5];
    size_t n[5];  // floats per array
    size_t bytes;
};
ObsLayout obs_layout(int B, int Ka, int Kr, int Kl) {
    ObsLayout L;
    L.n[0] = size_t(B) * 9;
    L.n[1] = size_t(B) * Ka * 6;
    L.n[2] = size_t(B) * Kr * 12;
    L.n[3] = size_t(B) * Kl * 5;
    L.n[4] = size_t(B) * 2;
    size_t o = 0;
    for (int i = 0; i < 5; ++i) {
        L.off[i] = o;
        o += al(L.n[i] * 4);
    }
    L.bytes = o;
    return L;
}
void carve_obs(unsigned char* base, const ObsLayout& L, zsim_obs_view* v) {
    v->active = reinterpret_cast<float*>(base + L.off[0]);
    v->agents = reinterpret_cast<float*>(base + L.off[1]);
    v->road = reinterpret_cast<float*>(base + L.off[2]);
    v->route = reinterpret_cast<float*>(base + L.off[3]);
    v->value_only = reinterpret_cast<float*>(base + L.off[4]);
}

// Host image of the pack: offsets into one buffer, then a single upload.
struct PackBuilder {
    // the image: caller memory (a BatchStream's pinned buffer) or owned
    struct Buf {
        unsigned char* p = nullptr;
        unsigned char* data() { return p; }
    } host;
    std::unique_ptr<unsigned char[]> own;
    size_t cursor = 0;
    template <class T>
    size_t reserve(size_t n) {
        size_t o = cursor;
        cursor += al(sizeof(T) * std::max<size_t>(n, 1));
        return o;
    }
    template <class T>
    T* at(size_t off) {
        return reinterpret_cast<T*>(host.data() + off);
    }
};

}  // namespace

struct zsim_env {
    int device = 0;
    zs::KernelArgs base{};
    void* d_pack = nullptr;
    size_t pack_bytes = 0;
    int32_t* d_err = nullptr;
    int B = 0, horizon = 0, total_stop = 0;
    double dt = 0.0;
    int zero_accel = 0, zero_steer = 0;
    std::vector<double> accel_bins, steer_bins;
    std::vector<double> goal_s, initial_s, logged_progress;
    std::vector<int32_t> row_scen, row_actor;  // row -> (scenario, controlled actor; -1 = ego mode)
    int n_scen = 0;
    zsim_sim_config cfg{};
    StateLayout sl{};
    StepoutLayout sol{};
    ObsLayout ol{};
    // host-vector path scratch (lazily allocated)
    void* h_dev = nullptr;
    zsim_state_view h_in{}, h_out{};
    zsim_stepout_view h_so{};
    zsim_obs_view h_obs{};
    int32_t* h_act = nullptr;
    cudaStream_t h_stream = nullptr;
    cudaStream_t h_copy = nullptr;  // observe_host's chunked D2H
    cudaEvent_t h_ev[4]{};
    double* d_initial_s = nullptr;
    double* d_logged = nullptr;          // logged_progress (device rollout recording)
    void* roll_buf = nullptr;            // zsim_rollout scratch: two states + one observation
    void* pol_buf = nullptr;             // zsim_rollout_policy scratch: accel, steer, logp, value [B]
    void* seq_buf = nullptr;             // zsim_cut_sequences scratch: offsets [B + 1] + obs views [T]
    size_t seq_cap = 0;
    zsim_state_view roll_s[2]{};
    zsim_obs_view roll_obs{};
    zsim_stepout_view roll_so{};
    double* d_metrics_scratch = nullptr;  // per-block Aggregate partials
    float4* d_hint = nullptr;
    int grid = 0;
    int launch_policy = 0;  // zsim_set_launch_policy: 0 auto, 1 fused, 2 split observation kernels
};

namespace {

void set_device(const zsim_env* env) { cuda_check(cudaSetDevice(env->device), "cudaSetDevice"); }

bool is_carved_state(const zsim_state_view* v, const StateLayout& L) {
    unsigned char* base = reinterpret_cast<unsigned char*>(v->x);
    zsim_state_view c;
    carve_state(base, L, &c);
    return std::memcmp(&c, v, sizeof(c)) == 0;
}
bool is_carved_stepout(const zsim_stepout_view* v, const StepoutLayout& L) {
    unsigned char* base = reinterpret_cast<unsigned char*>(v->reward);
    zsim_stepout_view c;
    carve_stepout(base, L, &c);
    return std::memcmp(&c, v, sizeof(c)) == 0;
}
bool is_carved_obs(const zsim_obs_view* v, const ObsLayout& L) {
    unsigned char* base = reinterpret_cast<unsigned char*>(v->active);
    zsim_obs_view c;
    carve_obs(base, L, &c);
    return std::memcmp(&c, v, sizeof(c)) == 0;
}

cudaMemcpyKind kind_of(int dir) {
    switch (dir) {
        case 0: return cudaMemcpyHostToDevice;
        case 1: return cudaMemcpyDeviceToHost;
        case 2: return cudaMemcpyDeviceToDevice;
        default: raise(Err::invalid_argument, "copy direction must be 0 (h2d), 1 (d2h) or 2 (d2d)");
    }
}

void copy_state(zsim_env* env, const zsim_state_view* dst, const zsim_state_view* src, int dir, cudaStream_t s) {
    cudaMemcpyKind k = kind_of(dir);
    if (is_carved_state(dst, env->sl) && is_carved_state(src, env->sl)) {
        cuda_check(cudaMemcpyAsync(dst->x, src->x, env->sl.bytes, k, s), "state copy");
        return;
    }
    const size_t B = size_t(env->B);
    cuda_check(cudaMemcpyAsync(dst->x, src->x, 8 * B, k, s), "state copy");
    cuda_check(cudaMemcpyAsync(dst->y, src->y, 8 * B, k, s), "state copy");
    cuda_check(cudaMemcpyAsync(dst->heading, src->heading, 8 * B, k, s), "state copy");
    cuda_check(cudaMemcpyAsync(dst->v, src->v, 8 * B, k, s), "state copy");
    cuda_check(cudaMemcpyAsync(dst->steering, src->steering, 8 * B, k, s), "state copy");
    cuda_check(cudaMemcpyAsync(dst->t, src->t, 4 * B, k, s), "state copy");
    cuda_check(cudaMemcpyAsync(dst->done, src->done, B, k, s), "state copy");
    cuda_check(cudaMemcpyAsync(dst->reason, src->reason, B, k, s), "state copy");
    cuda_check(cudaMemcpyAsync(dst->rng, src->rng, 8 * B, k, s), "state copy");
    cuda_check(cudaMemcpyAsync(dst->proj_s, src->proj_s, 8 * B, k, s), "state copy");
    cuda_check(cudaMemcpyAsync(dst->proj_d, src->proj_d, 8 * B, k, s), "state copy");
    cuda_check(cudaMemcpyAsync(dst->proj_in_corridor, src->proj_in_corridor, B, k, s), "state copy");
    cuda_check(cudaMemcpyAsync(dst->events, src->events, B, k, s), "state copy");
    if (env->total_stop > 0) {
        cuda_check(cudaMemcpyAsync(dst->stopped_flags, src->stopped_flags, size_t(env->total_stop), k, s),
                   "state copy");
    }
}

void copy_stepout(zsim_env* env, const zsim_stepout_view* dst, const zsim_stepout_view* src, int dir,
                  cudaStream_t s) {
    cudaMemcpyKind k = kind_of(dir);
    if (is_carved_stepout(dst, env->sol) && is_carved_stepout(src, env->sol)) {
        cuda_check(cudaMemcpyAsync(dst->reward, src->reward, env->sol.bytes, k, s), "stepout copy");
        return;
    }
    const size_t B = size_t(env->B);
    cuda_check(cudaMemcpyAsync(dst->reward, src->reward, 4 * B, k, s), "stepout copy");
    cuda_check(cudaMemcpyAsync(dst->event, src->event, B, k, s), "stepout copy");
    cuda_check(cudaMemcpyAsync(dst->s, src->s, 4 * B, k, s), "stepout copy");
    cuda_check(cudaMemcpyAsync(dst->a_lat, src->a_lat, 4 * B, k, s), "stepout copy");
    cuda_check(cudaMemcpyAsync(dst->a_lon, src->a_lon, 4 * B, k, s), "stepout copy");
    cuda_check(cudaMemcpyAsync(dst->v, src->v, 4 * B, k, s), "stepout copy");
}

void copy_obs(zsim_env* env, const zsim_obs_view* dst, const zsim_obs_view* src, int dir, cudaStream_t s) {
    cudaMemcpyKind k = kind_of(dir);
    if (is_carved_obs(dst, env->ol) && is_carved_obs(src, env->ol)) {
        cuda_check(cudaMemcpyAsync(dst->active, src->active, env->ol.bytes, k, s), "obs copy");
        return;
    }
    const ObsLayout& L = env->ol;
    cuda_check(cudaMemcpyAsync(dst->active, src->active, 4 * L.n[0], k, s), "obs copy");
    cuda_check(cudaMemcpyAsync(dst->agents, src->agents, 4 * L.n[1], k, s), "obs copy");
    cuda_check(cudaMemcpyAsync(dst->road, src->road, 4 * L.n[2], k, s), "obs copy");
    cuda_check(cudaMemcpyAsync(dst->route, src->route, 4 * L.n[3], k, s), "obs copy");
    cuda_check(cudaMemcpyAsync(dst->value_only, src->value_only, 4 * L.n[4], k, s), "obs copy");
}

void check_view(const void* p, const char* what) {
    if (!p) raise(Err::invalid_argument, std::string(what) + ": null view pointer");
}

zs::DevCfg make_dev_cfg(const zsim_sim_config& c, const std::vector<double>& ab, const std::vector<double>& sb) {
    zs::DevCfg d{};
    d.wheelbase = c.wheelbase;
    d.ego_length = c.ego_length;
    d.ego_width = c.ego_width;
    d.ego_center_offset = c.ego_center_offset;
    d.delta_max = c.delta_max;
    d.v_min = c.v_min;
    d.goal_radius = c.goal_radius;
    d.footprint_margin = c.footprint_margin;
    d.stop_cross_speed = c.stop_cross_speed;
    d.stop_zone = c.stop_zone;
    d.stop_slow_speed = c.stop_slow_speed;
    d.w_progress = c.w_progress;
    d.w_speed = c.w_speed;
    d.w_lat = c.w_lat;
    d.w_lon = c.w_lon;
    d.terminal_penalty = c.terminal_penalty;
    d.feature_radius = c.feature_radius;
    d.disable_dones = c.disable_dones;
    d.n_agents = c.n_agents;
    d.n_road = c.n_road;
    d.n_route = c.n_route;
    d.n_accel = int32_t(ab.size());
    d.n_steer = int32_t(sb.size());
    for (size_t i = 0; i < ab.size(); ++i) d.accel_bins[i] = ab[i];
    for (size_t i = 0; i < sb.size(); ++i) d.steer_bins[i] = sb[i];
    return d;
}

// Spatial order of a point set: stable sort by the Morton code of (x, y)
// quantised over the set's bounding box.  Chunks of 32 consecutive points then
// cover compact regions; the reference index rides along for tie-breaks.
std::vector<int> morton_order(const std::vector<float>& xs, const std::vector<float>& ys) {
    const size_t n = xs.size();
    std::vector<int> perm(n);
    for (size_t i = 0; i < n; ++i) perm[i] = int(i);
    if (n < 2) return perm;
    float x0 = xs[0], x1 = xs[0], y0 = ys[0], y1 = ys[0];
    for (size_t i = 1; i < n; ++i) {
        x0 = std::min(x0, xs[i]), x1 = std::max(x1, xs[i]);
        y0 = std::min(y0, ys[i]), y1 = std::max(y1, ys[i]);
    }
    const double ext = std::max(double(x1) - x0, double(y1) - y0) + 1e-6;
    auto spread = [](uint32_t v) {
        uint64_t x = v & 0xFFFFu;
        x = (x | (x << 8)) & 0x00FF00FFu;
        x = (x | (x << 4)) & 0x0F0F0F0Fu;
        x = (x | (x << 2)) & 0x33333333u;
        x = (x | (x << 1)) & 0x55555555u;
        return uint32_t(x);
    };
    std::vector<uint32_t> code(n);
    for (size_t i = 0; i < n; ++i) {
        uint32_t qx = uint32_t((double(xs[i]) - x0) / ext * 65535.0);
        uint32_t qy = uint32_t((double(ys[i]) - y0) / ext * 65535.0);
        code[i] = spread(qx) | (spread(qy) << 1);
    }
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return code[size_t(a)] < code[size_t(b)]; });
    return perm;
}

// Writes one point set of scenario b in chunked spatial order.
void write_points(unsigned char* host, size_t o_xy, size_t o_attr, size_t o_oi, size_t o_cb, int b, int cap, int ccap,
                  const std::vector<float>& xs, const std::vector<float>& ys, const std::vector<uint8_t>& attr) {
    const std::vector<int> perm = morton_order(xs, ys);
    float* xy = reinterpret_cast<float*>(host + o_xy) + size_t(b) * cap * 2;
    uint8_t* at = host + o_attr + size_t(b) * cap;
    int32_t* oi = reinterpret_cast<int32_t*>(host + o_oi) + size_t(b) * cap;
    float* cb = reinterpret_cast<float*>(host + o_cb) + size_t(b) * ccap * 4;
    for (size_t k = 0; k < perm.size(); ++k) {
        const int i = perm[k];
        xy[2 * k] = xs[size_t(i)];
        xy[2 * k + 1] = ys[size_t(i)];
        at[k] = attr[size_t(i)];
        oi[k] = i;
    }
    const int n = int(perm.size());
    for (int c = 0; c * zs::kChunk < n; ++c) {
        float bx0 = 3e38f, by0 = 3e38f, bx1 = -3e38f, by1 = -3e38f;
        for (int k = c * zs::kChunk; k < std::min(n, (c + 1) * zs::kChunk); ++k) {
            bx0 = std::min(bx0, xy[2 * k]), bx1 = std::max(bx1, xy[2 * k]);
            by0 = std::min(by0, xy[2 * k + 1]), by1 = std::max(by1, xy[2 * k + 1]);
        }
        cb[4 * c] = bx0, cb[4 * c + 1] = by0, cb[4 * c + 2] = bx1, cb[4 * c + 3] = by1;
    }
}

// Env::Env (simcore.cpp:203-233) over make_batch (scenario_io.cpp:404-437).
// Stages the device pack.  Ego mode (controlled = false): one row per
// scenario, as Env::Env.  Controlled mode: one row per
// controllable actor of every scenario (zsim_scenario.hpp, controlled_scene);
// scenario data is stored once and rows index it (row_scen / row_actor).
// Runs f(i) for i in [0, n) on the host cores (staging is per scenario / per
// row and writes disjoint regions).  The lowest failing index's exception is
// rethrown, as a serial loop would.
void parallel_for(int n, const std::function<void(int)>& f) {
    int nt = int(std::min(32u, std::max(1u, std::thread::hardware_concurrency())));
    if (nt <= 1 || n < 64) {
        for (int i = 0; i < n; ++i) f(i);
        return;
    }
    struct Slot {
        std::exception_ptr ex;
        int at = INT32_MAX;
    };
    std::atomic<int> next{0};
    std::vector<Slot> slots(static_cast<size_t>(nt));
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) {
        Slot* my = slots.data() + t;
        th.emplace_back([&next, &f, n, my] {
            for (;;) {
                const int i0 = next.fetch_add(16);
                if (i0 >= n) return;
                const int i1 = std::min(n, i0 + 16);
                for (int i = i0; i < i1; ++i) {
                    try {
                        f(i);
                    } catch (...) {
                        if (i < my->at) {
                            my->at = i;
                            my->ex = std::current_exception();
                        }
                        return;
                    }
                }
            }
        });
    }
    for (auto& x : th) x.join();
    const Slot* best = nullptr;
    for (const Slot& sl : slots)
        if (sl.ex && (!best || sl.at < best->at)) best = &sl;
    if (best) std::rethrow_exception(best->ex);
}

// ZSIM_STAGE_TIMING=1: per-phase wall times of the host staging on stderr.
struct StageTimer {
    bool on = std::getenv("ZSIM_STAGE_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[stage] %-22s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    }
};

// Pinned staging buffer + copy stream of a BatchStream slot.
struct Uploader {
    void* pinned = nullptr;
    size_t cap = 0;
    cudaStream_t stream = nullptr;
};

void stage_env(zsim_env* env, const std::vector<zs::Scene>& scenes, int horizon, bool controlled,
               Uploader* up = nullptr) {
    using namespace zs;
    if (scenes.empty()) raise(Err::invalid_argument, "make_batch: empty scenario list");
    const int S = int(scenes.size());
    StageTimer tm;
    const double dt = scenes[0].dt;
    for (const auto& s : scenes) {
        if (int(s.num_steps) > horizon) {
            raise(Err::invalid_argument, "scenario `" + s.id + "` has " + std::to_string(s.num_steps) +
                                             " steps > T=" + std::to_string(horizon));
        }
        if (s.dt != dt) raise(Err::invalid_argument, "mixed dt within batch");
    }
    // Route contexts and route border points (host fp64, reference op order).
    std::vector<RouteCtx> ctx(static_cast<size_t>(S));
    std::vector<std::vector<RoutePt>> rpts(static_cast<size_t>(S));
    PackDims d{};
    d.T = 1;
    d.A = 1;
    d.P = 1;
    d.R = 1;
    d.L = 1;
    d.C = 2;
    d.NL = 1;
    d.NS = 1;
    parallel_for(S, [&](int b) {
        ctx[size_t(b)] = build_context(scenes[size_t(b)]);
        rpts[size_t(b)] = build_route_points(scenes[size_t(b)]);
    });
    for (int b = 0; b < S; ++b) {
        const Scene& s = scenes[size_t(b)];
        d.T = std::max(d.T, int(s.num_steps));
        d.A = std::max(d.A, controlled ? num_actors(s) : int(s.agents.size()));
        size_t np = 0;
        for (const auto& f : s.features) np += f.xy.size() / 2;
        d.P = std::max(d.P, int(np));
        d.R = std::max(d.R, int(rpts[size_t(b)].size()));
        d.L = std::max(d.L, int(ctx[size_t(b)].lanes.size()));
        for (const auto& lf : ctx[size_t(b)].lanes) d.C = std::max(d.C, int(lf.x.size()));
        d.NL = std::max(d.NL, int(ctx[size_t(b)].lights.size()));
        d.NS = std::max(d.NS, int(ctx[size_t(b)].stops.size()));
        for (const auto& a : s.agents) {
            if (a.x.size() < s.num_steps || a.y.size() < s.num_steps || a.heading.size() < s.num_steps ||
                a.speed.size() < s.num_steps || a.valid.size() < s.num_steps)
                raise(Err::invalid_argument, "scenario `" + s.id + "`: agent arrays shorter than num_steps");
        }
        for (const auto& lt : s.lights) {
            if (lt.state.size() < s.num_steps)
                raise(Err::invalid_argument, "scenario `" + s.id + "`: light state shorter than num_steps");
        }
        if (s.ego_x.size() < 2 || s.ego_v.size() < 2 || s.ego_h.size() < 2 || s.ego_y.size() < 2) {
            if (s.ego_x.empty()) raise(Err::invalid_argument, "scenario `" + s.id + "`: empty ego log");
        }
    }
    tm.mark("contexts");
    // rows: (scenario, controlled actor); actor -1 = the scenario's own ego (ego mode)
    std::vector<std::pair<int, int>> rows;
    for (int b = 0; b < S; ++b) {
        if (!controlled) {
            rows.emplace_back(b, -1);
            continue;
        }
        for (int j = 0; j < num_actors(scenes[size_t(b)]); ++j)
            if (actor_controllable(scenes[size_t(b)], j)) rows.emplace_back(b, j);
    }
    const int B = int(rows.size());
    d.B = B;
    d.S = S;
    const EgoBoxDims ebd{env->cfg.ego_length, env->cfg.ego_width, env->cfg.ego_center_offset};
    d.GC = std::max(1, (d.C - 1 + kSegGroup - 1) / kSegGroup);
    // the top-k scratch holds 16-bit point positions (zsim_kernels.cu, WarpBuf)
    if (d.P > 65535 || d.R > 65535)
        raise(Err::invalid_argument, "more than 65535 road or route points in one scenario are not supported on the "
                                     "device path");
    d.PC = (d.P + kChunk - 1) / kChunk;
    d.RC = (d.R + kChunk - 1) / kChunk;
    if (d.L > kMaxLanes) {
        raise(Err::invalid_argument, "route has " + std::to_string(d.L) + " lanes; the device path supports " +
                                         std::to_string(kMaxLanes));
    }

    PackBuilder pb;
    // scenario-level arrays [S...]
    size_t o_num_steps = pb.reserve<int32_t>(S), o_na = pb.reserve<int32_t>(S), o_nr = pb.reserve<int32_t>(S),
           o_nrt = pb.reserve<int32_t>(S), o_nl = pb.reserve<int32_t>(S), o_nlt = pb.reserve<int32_t>(S),
           o_ns = pb.reserve<int32_t>(S);
    size_t o_sl = pb.reserve<float>(S), o_rl = pb.reserve<double>(S);
    const size_t nag = size_t(S) * d.T * d.A;
    size_t o_agx = pb.reserve<float>(nag), o_agy = pb.reserve<float>(nag), o_agh = pb.reserve<float>(nag),
           o_ags = pb.reserve<float>(nag), o_agv = pb.reserve<uint8_t>(nag);
    size_t o_agl = pb.reserve<float>(size_t(S) * d.A), o_agw = pb.reserve<float>(size_t(S) * d.A);
    size_t o_agcs = pb.reserve<double>(nag * 2);
    size_t o_rxy = pb.reserve<float>(size_t(S) * d.P * 2), o_rkd = pb.reserve<uint8_t>(size_t(S) * d.P);
    size_t o_roi = pb.reserve<int32_t>(size_t(S) * d.P), o_rcb = pb.reserve<float>(size_t(S) * d.PC * 4);
    size_t o_txy = pb.reserve<float>(size_t(S) * d.R * 2), o_tfl = pb.reserve<uint8_t>(size_t(S) * d.R);
    size_t o_toi = pb.reserve<int32_t>(size_t(S) * d.R), o_tcb = pb.reserve<float>(size_t(S) * d.RC * 4);
    const size_t nln = size_t(S) * d.L * d.C;
    size_t o_lv = pb.reserve<LaneVtx>(nln);
    size_t o_lgb = pb.reserve<float>(size_t(S) * d.L * d.GC * 4);
    size_t o_lf4 = pb.reserve<float>(nln * 4), o_lorg = pb.reserve<double>(size_t(S) * 2),
           o_lfe = pb.reserve<float>(size_t(S));
    size_t o_lninfo = pb.reserve<LaneInfo>(size_t(S) * d.L);
    size_t o_rbox = pb.reserve<float>(size_t(S) * 4), o_tbox = pb.reserve<float>(size_t(S) * 4);
    size_t o_lts = pb.reserve<double>(size_t(S) * d.NL), o_ltst = pb.reserve<uint8_t>(size_t(S) * d.NL * d.T);
    size_t o_sts = pb.reserve<double>(size_t(S) * d.NS);
    // row-level arrays [B]
    size_t o_soff = pb.reserve<int32_t>(B), o_gx = pb.reserve<float>(B), o_gy = pb.reserve<float>(B);
    size_t o_gs = pb.reserve<double>(B);
    size_t o_ix = pb.reserve<double>(B), o_iy = pb.reserve<double>(B), o_ih = pb.reserve<double>(B),
           o_iv = pb.reserve<double>(B), o_ist = pb.reserve<double>(B);
    size_t o_rsc = pb.reserve<int32_t>(B), o_rac = pb.reserve<int32_t>(B);
    if (up) {
        if (up->cap < pb.cursor) {
            if (up->pinned) cudaFreeHost(up->pinned);
            up->pinned = nullptr;
            up->cap = 0;
            cuda_check(cudaHostAlloc(&up->pinned, pb.cursor, cudaHostAllocDefault), "cudaHostAlloc(stream staging)");
            up->cap = pb.cursor;
        }
        pb.host.p = static_cast<unsigned char*>(up->pinned);
    } else {
        pb.own.reset(new unsigned char[pb.cursor]);
        pb.host.p = pb.own.get();
    }
    {
        // zero the image (padding must be 0) in parallel 4 MB chunks
        const size_t chunk = size_t(4) << 20;
        parallel_for(int((pb.cursor + chunk - 1) / chunk), [&](int i) {
            const size_t o = size_t(i) * chunk;
            std::memset(pb.host.p + o, 0, std::min(chunk, pb.cursor - o));
        });
    }
    tm.mark("host image alloc");

    env->goal_s.assign(size_t(B), 0.0);
    env->initial_s.assign(size_t(B), 0.0);
    env->logged_progress.assign(size_t(B), 0.0);
    env->row_scen.assign(size_t(B), 0);
    env->row_actor.assign(size_t(B), -1);
    int total_stop = 0;
    for (int r = 0; r < B; ++r) {
        pb.at<int32_t>(o_soff)[r] = total_stop;
        total_stop += int(ctx[size_t(rows[size_t(r)].first)].stops.size());
    }
    parallel_for(B, [&](int r) {
        // row-level: the controlled actor's initial state and goal (simcore.cpp:217-223, 237-276)
        const int sb = rows[size_t(r)].first, actor = rows[size_t(r)].second;
        const Scene& s = scenes[size_t(sb)];
        const RouteCtx& c = ctx[size_t(sb)];
        Scene eg;
        actor_as_ego(s, actor < 0 ? 0 : actor, eg);
        env->row_scen[size_t(r)] = sb;
        env->row_actor[size_t(r)] = actor;
        pb.at<int32_t>(o_rsc)[r] = sb;
        pb.at<int32_t>(o_rac)[r] = actor;
        pb.at<float>(o_gx)[r] = eg.goal_x;
        pb.at<float>(o_gy)[r] = eg.goal_y;
        double gs = project_host(double(eg.goal_x), double(eg.goal_y), c).s;
        double s0 = project_host(double(eg.ego_x.front()), double(eg.ego_y.front()), c).s;
        double s1 = project_host(double(eg.ego_x[s.num_steps - 1]), double(eg.ego_y[s.num_steps - 1]), c).s;
        env->goal_s[size_t(r)] = gs;
        env->initial_s[size_t(r)] = s0;
        env->logged_progress[size_t(r)] = s1 - s0;
        pb.at<double>(o_gs)[r] = gs;
        pb.at<double>(o_ix)[r] = double(eg.ego_x[0]);
        pb.at<double>(o_iy)[r] = double(eg.ego_y[0]);
        pb.at<double>(o_ih)[r] = double(eg.ego_h[0]);
        pb.at<double>(o_iv)[r] = double(eg.ego_v[0]);
        pb.at<double>(o_ist)[r] = initial_steering(eg, env->cfg.wheelbase, env->cfg.delta_max);
    });
    tm.mark("rows");
    parallel_for(S, [&](int b) {
        const Scene& s = scenes[size_t(b)];
        const RouteCtx& c = ctx[size_t(b)];
        const int T = d.T, A = d.A;
        pb.at<int32_t>(o_num_steps)[b] = int32_t(s.num_steps);
        pb.at<int32_t>(o_na)[b] = int32_t(controlled ? num_actors(s) : int(s.agents.size()));
        size_t np = 0;
        for (const auto& f : s.features) np += f.xy.size() / 2;
        pb.at<int32_t>(o_nr)[b] = int32_t(np);
        pb.at<int32_t>(o_nrt)[b] = int32_t(rpts[size_t(b)].size());
        pb.at<int32_t>(o_nl)[b] = int32_t(c.lanes.size());
        pb.at<int32_t>(o_nlt)[b] = int32_t(c.lights.size());
        pb.at<int32_t>(o_ns)[b] = int32_t(c.stops.size());
        pb.at<float>(o_sl)[b] = s.speed_limit;
        pb.at<double>(o_rl)[b] = c.route_length;
        // agent columns: the logged agents, or in controlled mode the actors
        // (column 0 = the logged ego as an agent, column k = agents[k-1])
        std::vector<const AgentLog*> cols;
        AgentLog ego_ag;
        if (controlled) {
            ego_ag = ego_as_agent(s, ebd);
            cols.push_back(&ego_ag);
        }
        for (const auto& ag : s.agents) cols.push_back(&ag);
        for (size_t j = 0; j < cols.size(); ++j) {
            const AgentLog& ag = *cols[j];
            pb.at<float>(o_agl)[size_t(b) * A + j] = ag.length;
            pb.at<float>(o_agw)[size_t(b) * A + j] = ag.width;
            for (uint32_t t = 0; t < s.num_steps; ++t) {
                size_t k = (size_t(b) * T + t) * A + j;
                pb.at<float>(o_agx)[k] = ag.x[t];
                pb.at<float>(o_agy)[k] = ag.y[t];
                pb.at<float>(o_agh)[k] = ag.heading[t];
                pb.at<float>(o_ags)[k] = ag.speed[t];
                pb.at<uint8_t>(o_agv)[k] = ag.valid[t];
                // Obb::corners' cos / sin of the logged heading (geometry.cpp:8), computed with
                // the host libm exactly as the reference does; the device builds the corners
                // from them with the same IEEE operations
                const double h = double(ag.heading[t]);
                pb.at<double>(o_agcs)[2 * k] = std::cos(h);
                pb.at<double>(o_agcs)[2 * k + 1] = std::sin(h);
            }
        }
        {
            std::vector<float> xs, ys;
            std::vector<uint8_t> kd;
            for (const auto& f : s.features) {
                for (size_t i = 0; i + 1 < f.xy.size(); i += 2) {
                    xs.push_back(f.xy[i]);
                    ys.push_back(f.xy[i + 1]);
                    kd.push_back(uint8_t((f.kind & 15) | (f.dir << 4)));
                }
            }
            write_points(pb.host.data(), o_rxy, o_rkd, o_roi, o_rcb, b, d.P, d.PC, xs, ys, kd);
            xs.clear(), ys.clear(), kd.clear();
            for (const auto& q : rpts[size_t(b)]) {
                xs.push_back(q.x);
                ys.push_back(q.y);
                kd.push_back(uint8_t((q.is_left ? 1 : 0) | (q.lane_valid ? 2 : 0)));
            }
            write_points(pb.host.data(), o_txy, o_tfl, o_toi, o_tcb, b, d.R, d.RC, xs, ys, kd);
        }
        {
            float bx0 = 3e38f, by0 = 3e38f, bx1 = -3e38f, by1 = -3e38f;
            for (const auto& f : s.features)
                for (size_t i = 0; i + 1 < f.xy.size(); i += 2) {
                    bx0 = std::min(bx0, f.xy[i]);
                    by0 = std::min(by0, f.xy[i + 1]);
                    bx1 = std::max(bx1, f.xy[i]);
                    by1 = std::max(by1, f.xy[i + 1]);
                }
            float* bb = pb.at<float>(o_rbox) + 4 * size_t(b);
            bb[0] = bx0, bb[1] = by0, bb[2] = bx1, bb[3] = by1;
            float tx0 = 3e38f, ty0 = 3e38f, tx1 = -3e38f, ty1 = -3e38f;
            for (const auto& q : rpts[size_t(b)]) {
                tx0 = std::min(tx0, q.x);
                ty0 = std::min(ty0, q.y);
                tx1 = std::max(tx1, q.x);
                ty1 = std::max(ty1, q.y);
            }
            float* tb = pb.at<float>(o_tbox) + 4 * size_t(b);
            tb[0] = tx0, tb[1] = ty0, tb[2] = tx1, tb[3] = ty1;
        }

        // origin of the fp32 screening copy: the first vertex of the first lane
        double ox = 0.0, oy = 0.0;
        if (!c.lanes.empty() && !c.lanes[0].x.empty()) ox = c.lanes[0].x[0], oy = c.lanes[0].y[0];
        double fe_s = 0.0, fe_l = 0.0;
        for (size_t l = 0; l < c.lanes.size(); ++l) {
            const LaneFrame& lf = c.lanes[l];
            // group boxes: segments [8g, 8g+8) touch vertices [8g, 8g+8]; origin-relative, rounded outward
            const int nseg = int(lf.x.size()) - 1;
            for (int g = 0; g * kSegGroup < nseg; ++g) {
                double x0 = 1e300, y0 = 1e300, x1 = -1e300, y1 = -1e300;
                for (int v = g * kSegGroup; v <= std::min(nseg, (g + 1) * kSegGroup); ++v) {
                    x0 = std::min(x0, lf.x[size_t(v)] - ox), x1 = std::max(x1, lf.x[size_t(v)] - ox);
                    y0 = std::min(y0, lf.y[size_t(v)] - oy), y1 = std::max(y1, lf.y[size_t(v)] - oy);
                }
                float* gb = pb.at<float>(o_lgb) + ((size_t(b) * d.L + l) * d.GC + size_t(g)) * 4;
                gb[0] = std::nextafter(float(x0), -3e38f);
                gb[1] = std::nextafter(float(y0), -3e38f);
                gb[2] = std::nextafter(float(x1), 3e38f);
                gb[3] = std::nextafter(float(y1), 3e38f);
            }
            {
                double h0 = 1e300, h1 = -1e300;
                for (double h : lf.hw) h0 = std::min(h0, h), h1 = std::max(h1, h);
                LaneInfo& li = pb.at<LaneInfo>(o_lninfo)[size_t(b) * d.L + l];
                li.n = int32_t(lf.x.size());
                li.id = lf.lane_id;
                li.hw_min = lf.hw.empty() ? 0.f : std::nextafter(float(h0), -3e38f);
                li.hw_max = lf.hw.empty() ? 0.f : std::nextafter(float(h1), 3e38f);
            }
            for (size_t i = 0; i < lf.x.size(); ++i) {
                size_t k = (size_t(b) * d.L + l) * d.C + i;
                LaneVtx& v = pb.at<LaneVtx>(o_lv)[k];
                v.x = lf.x[i];
                v.y = lf.y[i];
                v.s = lf.s[i];
                v.hw = lf.hw[i];
                fe_s = std::max(fe_s, std::fabs(lf.x[i] - ox) + std::fabs(lf.y[i] - oy));
                if (i + 1 < lf.x.size()) {
                    // point_segment_dist2's ab = b - a and len2 = ab.norm2() (geometry.cpp:18-19)
                    double abx = lf.x[i + 1] - lf.x[i], aby = lf.y[i + 1] - lf.y[i];
                    v.abx = abx;
                    v.aby = aby;
                    v.ds = lf.s[i + 1] - lf.s[i];
                    v.dhw = lf.hw[i + 1] - lf.hw[i];
                    fe_l = std::max(fe_l, std::fabs(abx) + std::fabs(aby));
                    float* f4 = pb.at<float>(o_lf4) + 4 * k;
                    f4[0] = float(lf.x[i] - ox);
                    f4[1] = float(lf.y[i] - oy);
                    f4[2] = float(abx);
                    f4[3] = float(aby);
                }
            }
        }
        pb.at<double>(o_lorg)[2 * size_t(b)] = ox;
        pb.at<double>(o_lorg)[2 * size_t(b) + 1] = oy;
        pb.at<float>(o_lfe)[b] = float((fe_s + fe_l) * (1.0 + 1e-6)) + 1e-6f;
        for (size_t k = 0; k < c.lights.size(); ++k) {
            pb.at<double>(o_lts)[size_t(b) * d.NL + k] = c.lights[k].second;
            const auto& st = s.lights[size_t(c.lights[k].first)].state;
            for (uint32_t t = 0; t < s.num_steps; ++t)
                pb.at<uint8_t>(o_ltst)[(size_t(b) * d.NL + k) * d.T + t] = st[t];
        }
        for (size_t j = 0; j < c.stops.size(); ++j) pb.at<double>(o_sts)[size_t(b) * d.NS + j] = c.stops[j].second;
    });

    tm.mark("scenario pack");
    cuda_check(cudaMalloc(&env->d_pack, pb.cursor), "cudaMalloc(pack)");
    env->pack_bytes = pb.cursor;
    unsigned char* D = static_cast<unsigned char*>(env->d_pack);
    DevPack& pk = env->base.pk;
    pk.d = d;
    pk.dt = dt;
    pk.horizon = horizon;
    pk.total_stop_lines = total_stop;
    pk.num_steps = reinterpret_cast<const int32_t*>(D + o_num_steps);
    pk.n_agents = reinterpret_cast<const int32_t*>(D + o_na);
    pk.n_road = reinterpret_cast<const int32_t*>(D + o_nr);
    pk.n_route = reinterpret_cast<const int32_t*>(D + o_nrt);
    pk.n_lanes = reinterpret_cast<const int32_t*>(D + o_nl);
    pk.n_lights = reinterpret_cast<const int32_t*>(D + o_nlt);
    pk.n_stops = reinterpret_cast<const int32_t*>(D + o_ns);
    pk.stop_off = reinterpret_cast<const int32_t*>(D + o_soff);
    pk.speed_limit = reinterpret_cast<const float*>(D + o_sl);
    pk.goal_x = reinterpret_cast<const float*>(D + o_gx);
    pk.goal_y = reinterpret_cast<const float*>(D + o_gy);
    pk.goal_s = reinterpret_cast<const double*>(D + o_gs);
    pk.route_len = reinterpret_cast<const double*>(D + o_rl);
    pk.init_x = reinterpret_cast<const double*>(D + o_ix);
    pk.init_y = reinterpret_cast<const double*>(D + o_iy);
    pk.init_h = reinterpret_cast<const double*>(D + o_ih);
    pk.init_v = reinterpret_cast<const double*>(D + o_iv);
    pk.init_steer = reinterpret_cast<const double*>(D + o_ist);
    pk.ag_x = reinterpret_cast<const float*>(D + o_agx);
    pk.ag_y = reinterpret_cast<const float*>(D + o_agy);
    pk.ag_h = reinterpret_cast<const float*>(D + o_agh);
    pk.ag_sp = reinterpret_cast<const float*>(D + o_ags);
    pk.ag_valid = D + o_agv;
    pk.ag_len = reinterpret_cast<const float*>(D + o_agl);
    pk.ag_wid = reinterpret_cast<const float*>(D + o_agw);
    pk.ag_cs = reinterpret_cast<const double2*>(D + o_agcs);
    pk.road_xy = reinterpret_cast<const float2*>(D + o_rxy);
    pk.road_kd = D + o_rkd;
    pk.road_oi = reinterpret_cast<const int32_t*>(D + o_roi);
    pk.road_cb = reinterpret_cast<const float4*>(D + o_rcb);
    pk.route_xy = reinterpret_cast<const float2*>(D + o_txy);
    pk.route_fl = D + o_tfl;
    pk.route_oi = reinterpret_cast<const int32_t*>(D + o_toi);
    pk.route_cb = reinterpret_cast<const float4*>(D + o_tcb);
    pk.ln_v = reinterpret_cast<const LaneVtx*>(D + o_lv);
    pk.ln_f4 = reinterpret_cast<const float4*>(D + o_lf4);
    pk.ln_gb = reinterpret_cast<const float4*>(D + o_lgb);
    pk.ln_org = reinterpret_cast<const double2*>(D + o_lorg);
    pk.ln_fe = reinterpret_cast<const float*>(D + o_lfe);
    pk.road_box = reinterpret_cast<const float4*>(D + o_rbox);
    pk.route_box = reinterpret_cast<const float4*>(D + o_tbox);
    pk.ln_info = reinterpret_cast<const LaneInfo*>(D + o_lninfo);
    pk.lt_s = reinterpret_cast<const double*>(D + o_lts);
    pk.lt_state = D + o_ltst;
    pk.st_s = reinterpret_cast<const double*>(D + o_sts);
    pk.row_scen = controlled ? reinterpret_cast<const int32_t*>(D + o_rsc) : nullptr;
    pk.row_actor = controlled ? reinterpret_cast<const int32_t*>(D + o_rac) : nullptr;
    // one upload of the whole image: synchronous, or (BatchStream) through a
    // pinned staging buffer on a copy stream
    if (up) {
        // built in place in the pinned buffer
        cuda_check(cudaMemcpyAsync(env->d_pack, up->pinned, pb.cursor, cudaMemcpyHostToDevice, up->stream),
                   "upload pack");
    } else {
        cuda_check(cudaMemcpy(env->d_pack, pb.host.data(), pb.cursor, cudaMemcpyHostToDevice), "upload pack");
    }

    tm.mark("upload");
    env->B = B;
    env->n_scen = S;
    env->horizon = horizon;
    env->dt = dt;
    env->total_stop = total_stop;
    env->base.key_cap = std::max(d.P, d.R);
#ifndef ZS_CAND_CAP
#define ZS_CAND_CAP 256
#endif
    env->base.cand_cap = ZS_CAND_CAP;  // top-k candidates per warp before the histogram refinement
    env->sl = state_layout(B, total_stop);
    env->sol = stepout_layout(B);
    env->ol = obs_layout(B, env->cfg.n_agents, env->cfg.n_road, env->cfg.n_route);
    env->grid = B;
    size_t smem = zs::smem_bytes(env->base);
    if (smem > 200 * 1024) raise(Err::invalid_argument, "scenario shapes exceed the kernel's shared-memory budget");
}

zs::KernelArgs args_for(zsim_env* env) { return env->base; }

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

void ensure_host_scratch(zsim_env* env) {
    if (env->h_dev) return;
    size_t bytes = 2 * env->sl.bytes + env->sol.bytes + env->ol.bytes + al(size_t(env->B) * 8);
    cuda_check(cudaMalloc(&env->h_dev, bytes), "cudaMalloc(host-path scratch)");
    unsigned char* p = static_cast<unsigned char*>(env->h_dev);
    carve_state(p, env->sl, &env->h_in);
    p += env->sl.bytes;
    carve_state(p, env->sl, &env->h_out);
    p += env->sl.bytes;
    carve_stepout(p, env->sol, &env->h_so);
    p += env->sol.bytes;
    carve_obs(p, env->ol, &env->h_obs);
    p += env->ol.bytes;
    env->h_act = reinterpret_cast<int32_t*>(p);
    cuda_check(cudaStreamCreateWithFlags(&env->h_stream, cudaStreamNonBlocking), "cudaStreamCreate");
}

void check_actions_host(zsim_env* env, const int32_t* accel, const int32_t* steer) {
    if (!accel || !steer) raise(Err::invalid_argument, "env_step: action/state shape mismatch");
    const int na = int(env->accel_bins.size()), ns = int(env->steer_bins.size());
    for (int b = 0; b < env->B; ++b) {
        if (accel[b] < 0 || accel[b] >= na || steer[b] < 0 || steer[b] >= ns)
            raise(Err::invalid_argument, "action index out of range");
    }
}

}  // namespace

extern "C" {

ZSIM_API int zsim_abi_version(void) { return ZSIM_ABI_VERSION; }

ZSIM_API const char* zsim_last_error(void) { return g_last_error.c_str(); }

// the other C-ABI translation unit (zsim_policy.cu) reports through the same
// slot (C linkage inside this block; hidden like everything not ZSIM_API)
void zsim_internal_set_last_error(const char* m) { g_last_error = m; }

ZSIM_API int zsim_sim_config_defaults(zsim_sim_config* c) {
    return guarded([&] {
        if (!c) raise(Err::invalid_argument, "null config");
        std::memset(c, 0, sizeof(*c));
        c->wheelbase = 3.0;
        c->ego_length = 4.7;
        c->ego_width = 1.9;
        c->ego_center_offset = 1.5;
        c->delta_max = 0.55;
        c->v_min = 0.0;
        c->goal_radius = 2.0;
        c->footprint_margin = 0.1;
        c->stop_cross_speed = 0.5;
        c->stop_zone = 2.0;
        c->stop_slow_speed = 0.1;
        c->disable_dones = 0;
        c->n_agents = 16;
        c->n_road = 128;
        c->n_route = 64;
        c->w_progress = 1.0;
        c->w_speed = 0.1;
        c->w_lat = 0.02;
        c->w_lon = 0.02;
        c->terminal_penalty = 10.0;
        c->feature_radius = 100.0;
        c->threads = 1;
    });
}

namespace {

std::vector<zs::Scene> decode_batch(const uint8_t* file, size_t nbytes, const int64_t* indices, int32_t n_indices) {
    if (!file) zs::raise(zs::Err::invalid_argument, "null ZSIM buffer");
    zs::ZsimIndex idx = zs::zsim_index(file, nbytes);
    std::vector<int64_t> rows;
    if (indices) {
        if (n_indices <= 0) zs::raise(zs::Err::invalid_argument, "load_batch: empty index list");
        rows.assign(indices, indices + n_indices);
    } else {
        for (int64_t i = 0; i < int64_t(idx.records.size()); ++i) rows.push_back(i);
    }
    std::vector<zs::Scene> scenes(rows.size());
    parallel_for(int(rows.size()), [&](int i) { scenes[size_t(i)] = zs::zsim_decode(file, nbytes, idx, rows[size_t(i)]); });
    return scenes;
}

std::unique_ptr<zsim_env> build_env(std::vector<zs::Scene> scenes, int32_t horizon, const zsim_sim_config* cfg,
                                    const double* accel_bins, int32_t n_accel, const double* steer_bins,
                                    int32_t n_steer, int32_t device, bool controlled, Uploader* up) {
    std::unique_ptr<zsim_env> env(new zsim_env());
    env->device = device;
    if (cfg) {
        env->cfg = *cfg;
    } else {
        zsim_sim_config_defaults(&env->cfg);
    }
    if (env->cfg.n_agents <= 0 || env->cfg.n_road <= 0 || env->cfg.n_route <= 0)
        raise(Err::invalid_argument, "nearest_features: k must be > 0");
    // the per-warp top-k scratch ranks at most 256 selections (zsim_kernels.cu, warp_topk)
    if (env->cfg.n_road > 256 || env->cfg.n_route > 256)
        raise(Err::invalid_argument, "n_road / n_route above 256 are not supported on the device path");
    if (accel_bins && n_accel > 0)
        env->accel_bins.assign(accel_bins, accel_bins + n_accel);
    else
        env->accel_bins = {-4.0, -2.0, -0.5, 0.0, 0.5, 2.0, 4.0};
    if (steer_bins && n_steer > 0)
        env->steer_bins.assign(steer_bins, steer_bins + n_steer);
    else
        env->steer_bins = {-0.4, -0.1, 0.0, 0.1, 0.4};
    zs::check_bins(env->accel_bins, "accel_bins");
    zs::check_bins(env->steer_bins, "steer_rate_bins");
    if (env->accel_bins.size() > 16 || env->steer_bins.size() > 16)
        raise(Err::invalid_argument, "at most 16 bins per action head on the device path");
    env->zero_accel = zs::nearest_bin(env->accel_bins, 0.0);
    env->zero_steer = zs::nearest_bin(env->steer_bins, 0.0);
    int maxsteps = 2;
    for (const auto& sc : scenes) maxsteps = std::max(maxsteps, int(sc.num_steps));
    if (horizon <= 0) horizon = maxsteps;
    set_device(env.get());
    env->base.cfg = make_dev_cfg(env->cfg, env->accel_bins, env->steer_bins);
    stage_env(env.get(), scenes, horizon, controlled, up);
    cuda_check(cudaMalloc(&env->d_hint, sizeof(float4) * size_t(env->B)), "cudaMalloc(hint)");
    cuda_check(cudaMalloc(&env->d_err, 4), "cudaMalloc(err)");
    if (up) {
        cuda_check(cudaMemsetAsync(env->d_hint, 0xFF, sizeof(float4) * size_t(env->B), up->stream), "cudaMemset(hint)");
        cuda_check(cudaMemsetAsync(env->d_err, 0, 4, up->stream), "cudaMemset(err)");
    } else {
        cuda_check(cudaMemset(env->d_hint, 0xFF, sizeof(float4) * size_t(env->B)), "cudaMemset(hint)");  // NaN: no hint
        cuda_check(cudaMemset(env->d_err, 0, 4), "cudaMemset(err)");
    }
    env->base.hint = env->d_hint;
    env->base.err = env->d_err;
    return env;
}

int create_env(const uint8_t* file, size_t nbytes, const int64_t* indices, int32_t n_indices, int32_t horizon,
               const zsim_sim_config* cfg, const double* accel_bins, int32_t n_accel, const double* steer_bins,
               int32_t n_steer, int32_t device, zsim_env** out, bool controlled) {
    return guarded([&] {
        if (!out) raise(Err::invalid_argument, "null output pointer");
        *out = nullptr;
        if (!file) raise(Err::invalid_argument, "null ZSIM buffer");
        *out = build_env(decode_batch(file, nbytes, indices, n_indices), horizon, cfg, accel_bins, n_accel, steer_bins,
                         n_steer, device, controlled, nullptr)
                   .release();
    });
}

}  // namespace

ZSIM_API int zsim_env_create(const uint8_t* file, size_t nbytes, const int64_t* indices, int32_t n_indices,
                             int32_t horizon, const zsim_sim_config* cfg, const double* accel_bins, int32_t n_accel,
                             const double* steer_bins, int32_t n_steer, int32_t device, zsim_env** out) {
    return create_env(file, nbytes, indices, n_indices, horizon, cfg, accel_bins, n_accel, steer_bins, n_steer, device,
                      out, false);
}

ZSIM_API int zsim_env_create_controlled(const uint8_t* file, size_t nbytes, const int64_t* indices, int32_t n_indices,
                                        int32_t horizon, const zsim_sim_config* cfg, const double* accel_bins,
                                        int32_t n_accel, const double* steer_bins, int32_t n_steer, int32_t device,
                                        zsim_env** out) {
    return create_env(file, nbytes, indices, n_indices, horizon, cfg, accel_bins, n_accel, steer_bins, n_steer, device,
                      out, true);
}

// Benchmark shards of C3 / C4 ("generate per GPU shard in host
// memory ... then upload"): scenarios [first_index, first_index + count) of
// the stress set, generated on all host cores straight into the staging
// input -- no ZSIM image of the 17-35 GB shard.
ZSIM_API int zsim_env_create_stress(const zsim_stress_config* scfg, uint64_t seed, int32_t horizon,
                                    const zsim_sim_config* cfg, int32_t device, int32_t controlled, zsim_env** out) {
    return guarded([&] {
        if (!out || !scfg) raise(Err::invalid_argument, "null argument");
        *out = nullptr;
        zs::stress_check(*scfg);
        std::vector<zs::Scene> scenes(size_t(scfg->count));
        parallel_for(scfg->count, [&](int i) {
            scenes[size_t(i)] = zs::stress_scene(*scfg, seed, int64_t(scfg->first_index) + i);
        });
        *out = build_env(std::move(scenes), horizon, cfg, nullptr, 0, nullptr, 0, device, controlled != 0, nullptr)
                   .release();
    });
}

// ---------------------------------------------------------------------------
// BatchStream (scenario_stream.hpp:12-40, scenario_stream.cpp:35-46) feeding
// device Envs: while the caller simulates batch k, a staging thread decodes
// batch k+1, builds its route frames / pack on the host, and uploads it from
// a pinned buffer on a copy stream (two buffers alternate).
// ---------------------------------------------------------------------------
struct zsim_stream {
    std::vector<uint8_t> file;
    zs::ZsimIndex idx;
    int32_t batch_size = 0, horizon = 0, device = 0;
    bool prefetch = true, controlled = false;
    bool has_cfg = false;
    zsim_sim_config cfg{};
    std::vector<double> ab, sb;
    int64_t cursor = 0, num_batches = 0;
    zsim_env* current = nullptr;
    std::future<zsim_env*> staged;
    Uploader up[2];
    int slot = 0;

    zsim_env* load(int64_t k, int sl) {
        cudaSetDevice(device);
        const int64_t n = int64_t(idx.records.size());
        const int64_t begin = k * batch_size, end = std::min(begin + batch_size, n);
        std::vector<zs::Scene> scenes(size_t(end - begin));
        parallel_for(int(end - begin), [&](int i) {
            scenes[size_t(i)] = zs::zsim_decode(file.data(), file.size(), idx, begin + i);
        });
        auto env = build_env(std::move(scenes), horizon, has_cfg ? &cfg : nullptr, ab.empty() ? nullptr : ab.data(),
                             int32_t(ab.size()), sb.empty() ? nullptr : sb.data(), int32_t(sb.size()), device,
                             controlled, &up[sl]);
        cuda_check(cudaStreamSynchronize(up[sl].stream), "stream upload");
        return env.release();
    }
};

ZSIM_API int zsim_stream_create(const uint8_t* file, size_t nbytes, int32_t batch_size, int32_t horizon,
                                const zsim_sim_config* cfg, const double* accel_bins, int32_t n_accel,
                                const double* steer_bins, int32_t n_steer, int32_t device, int32_t prefetch,
                                int32_t controlled, zsim_stream** out) {
    return guarded([&] {
        if (!out) raise(Err::invalid_argument, "null output pointer");
        *out = nullptr;
        if (!file) raise(Err::invalid_argument, "null ZSIM buffer");
        if (batch_size <= 0) raise(Err::invalid_argument, "batch_size must be > 0");  // scenario_stream.cpp:9
        std::unique_ptr<zsim_stream> st(new zsim_stream());
        st->file.assign(file, file + nbytes);
        st->idx = zs::zsim_index(st->file.data(), st->file.size());
        if (st->idx.records.empty()) raise(Err::invalid_argument, "batch_iterator: dataset is empty");
        st->batch_size = batch_size;
        st->horizon = horizon;
        st->device = device;
        st->prefetch = prefetch != 0;
        st->controlled = controlled != 0;
        if (cfg) st->cfg = *cfg, st->has_cfg = true;
        if (accel_bins && n_accel > 0) st->ab.assign(accel_bins, accel_bins + n_accel);
        if (steer_bins && n_steer > 0) st->sb.assign(steer_bins, steer_bins + n_steer);
        st->num_batches = (int64_t(st->idx.records.size()) + batch_size - 1) / batch_size;
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        for (auto& u : st->up) cuda_check(cudaStreamCreateWithFlags(&u.stream, cudaStreamNonBlocking), "copy stream");
        *out = st.release();
    });
}

ZSIM_API int zsim_stream_num_batches(const zsim_stream* st, int64_t* out) {
    return guarded([&] {
        if (!st || !out) raise(Err::invalid_argument, "null stream/output");
        *out = st->num_batches;
    });
}

ZSIM_API int zsim_stream_next(zsim_stream* st, zsim_env** out) {
    return guarded([&] {
        if (!st || !out) raise(Err::invalid_argument, "null stream/output");
        *out = nullptr;
        if (st->current) {  // the previous batch's Env ends here
            zsim_env_destroy(st->current);
            st->current = nullptr;
        }
        if (st->cursor >= st->num_batches) return;
        zsim_env* env = st->staged.valid() ? st->staged.get() : st->load(st->cursor, st->slot);
        st->slot ^= 1;
        ++st->cursor;
        if (st->prefetch && st->cursor < st->num_batches) {
            const int64_t k = st->cursor;
            const int sl = st->slot;
            st->staged = std::async(std::launch::async, [st, k, sl] { return st->load(k, sl); });
        }
        st->current = env;
        *out = env;
    });
}

ZSIM_API int zsim_stream_destroy(zsim_stream* st) {
    return guarded([&] {
        if (!st) return;
        if (st->staged.valid()) {
            try {
                zsim_env_destroy(st->staged.get());
            } catch (...) {
            }
        }
        if (st->current) zsim_env_destroy(st->current);
        cudaSetDevice(st->device);
        for (auto& u : st->up) {
            if (u.stream) cudaStreamDestroy(u.stream);
            if (u.pinned) cudaFreeHost(u.pinned);
        }
        delete st;
    });
}

ZSIM_API int zsim_env_get_rows(const zsim_env* env, int32_t* scenario, int32_t* actor) {
    return guarded([&] {
        if (!env) raise(Err::invalid_argument, "null env");
        if (scenario) std::memcpy(scenario, env->row_scen.data(), sizeof(int32_t) * env->row_scen.size());
        if (actor) std::memcpy(actor, env->row_actor.data(), sizeof(int32_t) * env->row_actor.size());
    });
}

ZSIM_API int zsim_controlled_expand(const uint8_t* file, size_t nbytes, const int64_t* indices, int32_t n_indices,
                                    const zsim_sim_config* cfg, uint8_t** out_buf, size_t* out_len) {
    return guarded([&] {
        if (!out_buf || !out_len) raise(Err::invalid_argument, "null output pointer");
        *out_buf = nullptr;
        *out_len = 0;
        zsim_sim_config c;
        if (cfg) {
            c = *cfg;
        } else {
            zsim_sim_config_defaults(&c);
        }
        std::vector<zs::Scene> scenes = decode_batch(file, nbytes, indices, n_indices);
        const zs::EgoBoxDims ebd{c.ego_length, c.ego_width, c.ego_center_offset};
        std::string img = zs::zsim_header(scenes.empty() ? 0.1 : scenes[0].dt);
        for (const auto& sc : scenes)
            for (int j = 0; j < zs::num_actors(sc); ++j)
                if (zs::actor_controllable(sc, j)) zs::zsim_encode_append(img, zs::controlled_scene(sc, j, ebd));
        uint8_t* buf = static_cast<uint8_t*>(std::malloc(img.size()));
        if (!buf) raise(Err::runtime, "out of host memory");
        std::memcpy(buf, img.data(), img.size());
        *out_buf = buf;
        *out_len = img.size();
    });
}

ZSIM_API int zsim_env_destroy(zsim_env* env) {
    return guarded([&] {
        if (!env) return;
        cudaSetDevice(env->device);
        if (env->h_stream) cudaStreamDestroy(env->h_stream);
        if (env->h_copy) cudaStreamDestroy(env->h_copy);
        for (auto e : env->h_ev)
            if (e) cudaEventDestroy(e);
        cudaFree(env->h_dev);
        cudaFree(env->d_pack);
        cudaFree(env->d_err);
        cudaFree(env->d_initial_s);
        cudaFree(env->d_logged);
        cudaFree(env->roll_buf);
        cudaFree(env->pol_buf);
        cudaFree(env->seq_buf);
        cudaFree(env->d_metrics_scratch);
        cudaFree(env->d_hint);
        delete env;
    });
}

ZSIM_API int zsim_env_get_info(const zsim_env* env, zsim_env_info* out) {
    return guarded([&] {
        if (!env || !out) raise(Err::invalid_argument, "null env/info");
        std::memset(out, 0, sizeof(*out));
        out->batch = env->B;
        out->horizon = env->horizon;
        out->dt = env->dt;
        out->total_stop_lines = env->total_stop;
        out->zero_accel_idx = env->zero_accel;
        out->zero_steer_idx = env->zero_steer;
        out->num_accel = int32_t(env->accel_bins.size());
        out->num_steer = int32_t(env->steer_bins.size());
        const zs::PackDims& d = env->base.pk.d;
        out->cap_steps = d.T;
        out->cap_agents = d.A;
        out->cap_road = d.P;
        out->cap_route = d.R;
        out->cap_lanes = d.L;
        out->cap_vertices = d.C;
        out->cap_lights = d.NL;
        out->cap_stops = d.NS;
        out->device = env->device;
        out->static_bytes = env->pack_bytes;
        out->scenarios = env->n_scen;
        out->controlled = env->base.pk.row_scen ? 1 : 0;
        cudaSetDevice(env->device);
        out->step_observe_kernels = zs::observe_split(env->base, env->launch_policy) ? 2 : 1;
    });
}

ZSIM_API int zsim_env_get_scalars(const zsim_env* env, double* goal_s, double* initial_s, double* logged_progress) {
    return guarded([&] {
        if (!env) raise(Err::invalid_argument, "null env");
        if (goal_s) std::copy(env->goal_s.begin(), env->goal_s.end(), goal_s);
        if (initial_s) std::copy(env->initial_s.begin(), env->initial_s.end(), initial_s);
        if (logged_progress) std::copy(env->logged_progress.begin(), env->logged_progress.end(), logged_progress);
    });
}

ZSIM_API int zsim_state_alloc(zsim_env* env, zsim_state_view* v) {
    return guarded([&] {
        check_view(env, "state_alloc");
        check_view(v, "state_alloc");
        set_device(env);
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, env->sl.bytes), "cudaMalloc(state)");
        cuda_check(cudaMemset(p, 0, env->sl.bytes), "cudaMemset(state)");
        carve_state(static_cast<unsigned char*>(p), env->sl, v);
    });
}
ZSIM_API int zsim_state_free(zsim_env* env, zsim_state_view* v) {
    return guarded([&] {
        if (!env || !v) return;
        set_device(env);
        cudaFree(v->x);
        std::memset(v, 0, sizeof(*v));
    });
}
ZSIM_API int zsim_stepout_alloc(zsim_env* env, zsim_stepout_view* v) {
    return guarded([&] {
        check_view(env, "stepout_alloc");
        check_view(v, "stepout_alloc");
        set_device(env);
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, env->sol.bytes), "cudaMalloc(stepout)");
        cuda_check(cudaMemset(p, 0, env->sol.bytes), "cudaMemset(stepout)");
        carve_stepout(static_cast<unsigned char*>(p), env->sol, v);
    });
}
ZSIM_API int zsim_stepout_free(zsim_env* env, zsim_stepout_view* v) {
    return guarded([&] {
        if (!env || !v) return;
        set_device(env);
        cudaFree(v->reward);
        std::memset(v, 0, sizeof(*v));
    });
}
ZSIM_API int zsim_obs_alloc(zsim_env* env, zsim_obs_view* v) {
    return guarded([&] {
        check_view(env, "obs_alloc");
        check_view(v, "obs_alloc");
        set_device(env);
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, env->ol.bytes), "cudaMalloc(obs)");
        cuda_check(cudaMemset(p, 0, env->ol.bytes), "cudaMemset(obs)");
        carve_obs(static_cast<unsigned char*>(p), env->ol, v);
    });
}
ZSIM_API int zsim_obs_free(zsim_env* env, zsim_obs_view* v) {
    return guarded([&] {
        if (!env || !v) return;
        set_device(env);
        cudaFree(v->active);
        std::memset(v, 0, sizeof(*v));
    });
}

ZSIM_API int zsim_layout_bytes(const zsim_env* env, size_t* state_bytes, size_t* stepout_bytes, size_t* obs_bytes) {
    return guarded([&] {
        check_view(env, "layout_bytes");
        if (state_bytes) *state_bytes = env->sl.bytes;
        if (stepout_bytes) *stepout_bytes = env->sol.bytes;
        if (obs_bytes) *obs_bytes = env->ol.bytes;
    });
}
ZSIM_API int zsim_state_carve(const zsim_env* env, void* base, zsim_state_view* out) {
    return guarded([&] {
        check_view(env, "state_carve");
        check_view(base, "state_carve");
        check_view(out, "state_carve");
        carve_state(static_cast<unsigned char*>(base), env->sl, out);
    });
}
ZSIM_API int zsim_stepout_carve(const zsim_env* env, void* base, zsim_stepout_view* out) {
    return guarded([&] {
        check_view(env, "stepout_carve");
        check_view(base, "stepout_carve");
        check_view(out, "stepout_carve");
        carve_stepout(static_cast<unsigned char*>(base), env->sol, out);
    });
}
ZSIM_API int zsim_obs_carve(const zsim_env* env, void* base, zsim_obs_view* out) {
    return guarded([&] {
        check_view(env, "obs_carve");
        check_view(base, "obs_carve");
        check_view(out, "obs_carve");
        carve_obs(static_cast<unsigned char*>(base), env->ol, out);
    });
}
ZSIM_API int zsim_host_alloc(size_t bytes, void** out) {
    return guarded([&] {
        check_view(out, "host_alloc");
        *out = nullptr;
        cuda_check(cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocPortable), "cudaHostAlloc");
    });
}
ZSIM_API int zsim_host_free(void* p) {
    return guarded([&] {
        if (p) cuda_check(cudaFreeHost(p), "cudaFreeHost");
    });
}

ZSIM_API int zsim_state_copy(zsim_env* env, const zsim_state_view* dst, const zsim_state_view* src, int32_t dir,
                             void* stream) {
    return guarded([&] {
        check_view(env, "state_copy");
        check_view(dst, "state_copy");
        check_view(src, "state_copy");
        set_device(env);
        copy_state(env, dst, src, dir, as_stream(stream));
    });
}
ZSIM_API int zsim_stepout_copy(zsim_env* env, const zsim_stepout_view* dst, const zsim_stepout_view* src,
                               int32_t dir, void* stream) {
    return guarded([&] {
        check_view(env, "stepout_copy");
        check_view(dst, "stepout_copy");
        check_view(src, "stepout_copy");
        set_device(env);
        copy_stepout(env, dst, src, dir, as_stream(stream));
    });
}
ZSIM_API int zsim_obs_copy(zsim_env* env, const zsim_obs_view* dst, const zsim_obs_view* src, int32_t dir,
                           void* stream) {
    return guarded([&] {
        check_view(env, "obs_copy");
        check_view(dst, "obs_copy");
        check_view(src, "obs_copy");
        set_device(env);
        copy_obs(env, dst, src, dir, as_stream(stream));
    });
}

ZSIM_API int zsim_reset(zsim_env* env, uint64_t seed, const zsim_state_view* out, void* stream) {
    return guarded([&] {
        check_view(env, "reset");
        check_view(out, "reset");
        set_device(env);
        zs::KernelArgs a = args_for(env);
        a.out = *out;
        a.seed = seed;
        cuda_check(zs::launch_reset(a, env->grid, as_stream(stream)), "reset kernel");
    });
}

ZSIM_API int zsim_step(zsim_env* env, const zsim_state_view* in, const int32_t* accel, const int32_t* steer,
                       const zsim_state_view* out, const zsim_stepout_view* so, void* stream) {
    return guarded([&] {
        check_view(env, "step");
        check_view(in, "step");
        check_view(out, "step");
        check_view(so, "step");
        if (!accel || !steer) raise(Err::invalid_argument, "env_step: action/state shape mismatch");
        set_device(env);
        zs::KernelArgs a = args_for(env);
        a.in = *in;
        a.out = *out;
        a.accel = accel;
        a.steer = steer;
        a.so = *so;
        cuda_check(zs::launch_step_observe(a, zs::kModeStep, env->launch_policy, as_stream(stream)), "step kernel");
    });
}

ZSIM_API int zsim_observe(zsim_env* env, const zsim_state_view* in, const zsim_obs_view* obs, void* stream) {
    return guarded([&] {
        check_view(env, "observe");
        check_view(in, "observe");
        check_view(obs, "observe");
        set_device(env);
        zs::KernelArgs a = args_for(env);
        a.in = *in;
        a.obs = *obs;
        cuda_check(zs::launch_step_observe(a, zs::kModeObserve, env->launch_policy, as_stream(stream)), "observe kernel");
    });
}

ZSIM_API int zsim_step_observe(zsim_env* env, const zsim_state_view* in, const int32_t* accel, const int32_t* steer,
                               const zsim_state_view* out, const zsim_stepout_view* so, const zsim_obs_view* obs,
                               void* stream) {
    return guarded([&] {
        check_view(env, "step_observe");
        check_view(in, "step_observe");
        check_view(out, "step_observe");
        check_view(so, "step_observe");
        check_view(obs, "step_observe");
        if (!accel || !steer) raise(Err::invalid_argument, "env_step: action/state shape mismatch");
        set_device(env);
        zs::KernelArgs a = args_for(env);
        a.in = *in;
        a.out = *out;
        a.accel = accel;
        a.steer = steer;
        a.so = *so;
        a.obs = *obs;
        cuda_check(zs::launch_step_observe(a, zs::kModeStepObserve, env->launch_policy, as_stream(stream)),
                   "step_observe kernel");
    });
}

ZSIM_API int zsim_episode_stats(zsim_env* env, const zsim_state_view* state, int64_t* out_dev, void* stream) {
    return guarded([&] {
        check_view(env, "episode_stats");
        check_view(state, "episode_stats");
        check_view(out_dev, "episode_stats");
        set_device(env);
        if (!env->d_initial_s) {
            cuda_check(cudaMalloc(&env->d_initial_s, sizeof(double) * size_t(env->B)), "cudaMalloc(initial_s)");
            cuda_check(cudaMemcpy(env->d_initial_s, env->initial_s.data(), sizeof(double) * size_t(env->B),
                                  cudaMemcpyHostToDevice),
                       "upload initial_s");
        }
        zs::KernelArgs a = args_for(env);
        a.in = *state;
        cuda_check(zs::launch_episode_stats(a, env->d_initial_s, reinterpret_cast<long long*>(out_dev),
                                            as_stream(stream)),
                   "episode_stats kernel");
    });
}

namespace {

// EpisodeBatch blob: [B][T] arrays then B-vectors, 256-B aligned.
struct EpisodeLayout {
    size_t off[16];
    size_t bytes;
};

EpisodeLayout episode_layout(int B, int T) {
    const size_t bt = size_t(B) * size_t(T), b = size_t(B);
    const size_t sz[16] = {4 * bt, 4 * bt, 4 * bt, 4 * bt, 4 * bt, 4 * bt, 4 * bt, 4 * bt,
                           4 * bt, bt,     bt,     4 * b,  b,      b,      4 * b,  4 * b};
    EpisodeLayout L;
    size_t o = 0;
    for (int i = 0; i < 16; ++i) {
        L.off[i] = o;
        o += al(std::max<size_t>(sz[i], 1));
    }
    L.bytes = o;
    return L;
}

void carve_episode(unsigned char* p, const EpisodeLayout& L, int T, zsim_episode_view* v) {
    std::memset(v, 0, sizeof(*v));
    v->accel_idx = reinterpret_cast<int32_t*>(p + L.off[0]);
    v->steer_idx = reinterpret_cast<int32_t*>(p + L.off[1]);
    v->logp = reinterpret_cast<float*>(p + L.off[2]);
    v->value = reinterpret_cast<float*>(p + L.off[3]);
    v->reward = reinterpret_cast<float*>(p + L.off[4]);
    v->s = reinterpret_cast<float*>(p + L.off[5]);
    v->a_lat = reinterpret_cast<float*>(p + L.off[6]);
    v->a_lon = reinterpret_cast<float*>(p + L.off[7]);
    v->v = reinterpret_cast<float*>(p + L.off[8]);
    v->done = p + L.off[9];
    v->mask = p + L.off[10];
    v->bootstrap = reinterpret_cast<float*>(p + L.off[11]);
    v->terminal = p + L.off[12];
    v->events = p + L.off[13];
    v->initial_s = reinterpret_cast<float*>(p + L.off[14]);
    v->logged_progress = reinterpret_cast<float*>(p + L.off[15]);
    v->horizon = T;
}

void check_episode(const zsim_env* env, const zsim_episode_view* ep, const char* what) {
    check_view(ep, what);
    if (ep->horizon <= 0 || !ep->reward || !ep->mask || !ep->bootstrap)
        raise(Err::invalid_argument, std::string(what) + ": episode view not allocated");
    (void)env;
}

void ensure_host_arrays(zsim_env* env) {
    if (!env->d_initial_s) {
        cuda_check(cudaMalloc(&env->d_initial_s, sizeof(double) * size_t(env->B)), "cudaMalloc(initial_s)");
        cuda_check(cudaMemcpy(env->d_initial_s, env->initial_s.data(), sizeof(double) * size_t(env->B),
                              cudaMemcpyHostToDevice),
                   "upload initial_s");
    }
    if (!env->d_logged) {
        cuda_check(cudaMalloc(&env->d_logged, sizeof(double) * size_t(env->B)), "cudaMalloc(logged_progress)");
        cuda_check(cudaMemcpy(env->d_logged, env->logged_progress.data(), sizeof(double) * size_t(env->B),
                              cudaMemcpyHostToDevice),
                   "upload logged_progress");
    }
}

}  // namespace

ZSIM_API int zsim_episode_bytes(const zsim_env* env, int32_t horizon, size_t* bytes) {
    return guarded([&] {
        check_view(env, "episode_bytes");
        check_view(bytes, "episode_bytes");
        if (horizon <= 0) raise(Err::invalid_argument, "episode: horizon must be > 0");
        *bytes = episode_layout(env->B, horizon).bytes;
    });
}

ZSIM_API int zsim_episode_carve(const zsim_env* env, int32_t horizon, void* base, zsim_episode_view* out) {
    return guarded([&] {
        check_view(env, "episode_carve");
        check_view(base, "episode_carve");
        check_view(out, "episode_carve");
        if (horizon <= 0) raise(Err::invalid_argument, "episode: horizon must be > 0");
        carve_episode(static_cast<unsigned char*>(base), episode_layout(env->B, horizon), horizon, out);
    });
}

ZSIM_API int zsim_episode_alloc(zsim_env* env, int32_t horizon, zsim_episode_view* out) {
    return guarded([&] {
        check_view(env, "episode_alloc");
        check_view(out, "episode_alloc");
        if (horizon <= 0) raise(Err::invalid_argument, "episode: horizon must be > 0");
        set_device(env);
        const EpisodeLayout L = episode_layout(env->B, horizon);
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, L.bytes), "cudaMalloc(episode)");
        cuda_check(cudaMemset(p, 0, L.bytes), "cudaMemset(episode)");
        carve_episode(static_cast<unsigned char*>(p), L, horizon, out);
    });
}

ZSIM_API int zsim_episode_free(zsim_env* env, zsim_episode_view* ep) {
    return guarded([&] {
        if (!env || !ep) return;
        set_device(env);
        cudaFree(ep->accel_idx);
        std::memset(ep, 0, sizeof(*ep));
    });
}

ZSIM_API int zsim_sequences_alloc(zsim_env* env, int32_t horizon, int32_t seq_len, zsim_sequences_view* out) {
    return guarded([&] {
        check_view(env, "sequences_alloc");
        check_view(out, "sequences_alloc");
        if (horizon <= 0 || seq_len <= 0) raise(Err::invalid_argument, "sequences_alloc: horizon and seq_len must be > 0");
        set_device(env);
        const size_t cap = size_t(env->B) * size_t((horizon + seq_len - 1) / seq_len);
        const size_t rows = cap * size_t(seq_len);
        const ObsLayout ol = obs_layout(int(rows), env->cfg.n_agents, env->cfg.n_road, env->cfg.n_route);
        const size_t steps = al(rows * 4);
        const size_t bytes = ol.bytes + 4 * steps + 2 * al(rows) + 3 * al(cap * 4) + 256;
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, bytes), "cudaMalloc(sequences)");
        cuda_check(cudaMemset(p, 0, bytes), "cudaMemset(sequences)");
        unsigned char* q = static_cast<unsigned char*>(p);
        zsim_sequences_view v{};
        v.capacity = int32_t(cap);
        v.seq_len = seq_len;
        carve_obs(q, ol, &v.obs);
        q += ol.bytes;
        v.accel_idx = reinterpret_cast<int32_t*>(q), q += steps;
        v.steer_idx = reinterpret_cast<int32_t*>(q), q += steps;
        v.logmu = reinterpret_cast<float*>(q), q += steps;
        v.reward = reinterpret_cast<float*>(q), q += steps;
        v.done = q, q += al(rows);
        v.mask = q, q += al(rows);
        v.bootstrap = reinterpret_cast<float*>(q), q += al(cap * 4);
        v.row = reinterpret_cast<int32_t*>(q), q += al(cap * 4);
        v.t0 = reinterpret_cast<int32_t*>(q), q += al(cap * 4);
        v.count = reinterpret_cast<int32_t*>(q);
        *out = v;
    });
}

ZSIM_API int zsim_sequences_free(zsim_env* env, zsim_sequences_view* seq) {
    return guarded([&] {
        if (!env || !seq) return;
        set_device(env);
        cudaFree(seq->obs.active);
        std::memset(seq, 0, sizeof(*seq));
    });
}

ZSIM_API int zsim_cut_sequences(zsim_env* env, const zsim_episode_view* ep, const zsim_obs_view* obs,
                                int32_t seq_len, const zsim_sequences_view* out, void* stream) {
    return guarded([&] {
        check_view(env, "cut_sequences");
        check_episode(env, ep, "cut_sequences");
        check_view(obs, "cut_sequences");
        check_view(out, "cut_sequences");
        // replay.cpp:9
        if (seq_len <= 0) raise(Err::invalid_argument, "cut_sequences: seq_len must be > 0");
        const int T = ep->horizon, B = env->B;
        if (out->seq_len != seq_len || size_t(out->capacity) < size_t(B) * size_t((T + seq_len - 1) / seq_len))
            raise(Err::invalid_argument, "cut_sequences: output buffers too small for this episode / seq_len");
        set_device(env);
        const size_t need = al(size_t(B + 1) * 4) + size_t(T) * sizeof(zsim_obs_view);
        if (env->seq_cap < need) {
            cuda_check(cudaDeviceSynchronize(), "sync");
            cudaFree(env->seq_buf);
            env->seq_buf = nullptr;
            env->seq_cap = 0;
            cuda_check(cudaMalloc(&env->seq_buf, need), "cudaMalloc(sequence scratch)");
            env->seq_cap = need;
        }
        cudaStream_t s = as_stream(stream);
        unsigned char* q = static_cast<unsigned char*>(env->seq_buf);
        auto* off = reinterpret_cast<int32_t*>(q);
        auto* dviews = reinterpret_cast<zsim_obs_view*>(q + al(size_t(B + 1) * 4));
        cuda_check(cudaMemcpyAsync(dviews, obs, size_t(T) * sizeof(zsim_obs_view), cudaMemcpyHostToDevice, s),
                   "upload observation views");
        cuda_check(zs::launch_cut_sequences(B, T, seq_len, *ep, dviews, *out, env->cfg.n_agents, env->cfg.n_road,
                                            env->cfg.n_route, off, s),
                   "cut_sequences kernels");
        // (a pageable H2D copy returns once the caller's view array is staged: it may be freed on return)
    });
}

ZSIM_API int zsim_episode_copy(const zsim_env* env, const zsim_episode_view* dst, const zsim_episode_view* src,
                               int32_t dir, void* stream) {
    return guarded([&] {
        check_view(env, "episode_copy");
        check_episode(env, dst, "episode_copy");
        check_episode(env, src, "episode_copy");
        if (dst->horizon != src->horizon) raise(Err::invalid_argument, "episode_copy: horizon mismatch");
        const EpisodeLayout L = episode_layout(env->B, src->horizon);
        cudaSetDevice(env->device);
        // carved views are one contiguous blob
        cuda_check(cudaMemcpyAsync(dst->accel_idx, src->accel_idx, L.bytes, kind_of(dir), as_stream(stream)),
                   "episode copy");
    });
}

ZSIM_API int zsim_rollout(zsim_env* env, uint64_t seed, int32_t horizon, const int32_t* accel, const int32_t* steer,
                          int32_t script_len, const zsim_episode_view* ep, const zsim_obs_view* obs,
                          const zsim_state_view* final_state, void* stream) {
    return guarded([&] {
        check_view(env, "rollout");
        if (horizon <= 0) raise(Err::invalid_argument, "rollout: horizon must be > 0");
        if (script_len < 0 || (script_len > 0 && (!accel || !steer)))
            raise(Err::invalid_argument, "rollout: bad action script");
        if (ep) {
            check_episode(env, ep, "rollout");
            if (ep->horizon != horizon) raise(Err::invalid_argument, "rollout: episode horizon mismatch");
        }
        set_device(env);
        ensure_host_arrays(env);
        if (!env->roll_buf) {
            cuda_check(cudaMalloc(&env->roll_buf, 2 * env->sl.bytes + env->ol.bytes + env->sol.bytes),
                       "cudaMalloc(rollout scratch)");
            unsigned char* p = static_cast<unsigned char*>(env->roll_buf);
            carve_state(p, env->sl, &env->roll_s[0]);
            carve_state(p + env->sl.bytes, env->sl, &env->roll_s[1]);
            carve_obs(p + 2 * env->sl.bytes, env->ol, &env->roll_obs);
            carve_stepout(p + 2 * env->sl.bytes + env->ol.bytes, env->sol, &env->roll_so);
        }
        cudaStream_t s = as_stream(stream);
        zs::KernelArgs a = args_for(env);
        a.seed = seed;
        a.out = env->roll_s[0];
        cuda_check(zs::launch_reset(a, env->grid, s), "reset kernel");
        // obs[0] = observe(reset state)
        a = args_for(env);
        a.in = env->roll_s[0];
        a.obs = obs ? obs[0] : env->roll_obs;
        cuda_check(zs::launch_step_observe(a, zs::kModeObserve, env->launch_policy, s), "observe kernel");
        int cur = 0;
        for (int t = 0; t < horizon; ++t) {
            a = args_for(env);
            a.in = env->roll_s[cur];
            a.out = env->roll_s[cur ^ 1];
            a.accel = accel;
            a.steer = steer;
            a.act_len = script_len > 0 ? script_len : -1;  // -1: empty script, every row takes the zero action
            a.zero_accel = env->zero_accel;
            a.zero_steer = env->zero_steer;
            a.so = env->roll_so;
            if (ep) {
                a.ep = *ep;
                a.ep_t = t;
            }
            a.obs = obs ? obs[t + 1] : env->roll_obs;
            cuda_check(zs::launch_step_observe(a, zs::kModeStepObserve, env->launch_policy, s), "step+observe kernel");
            cur ^= 1;
        }
        if (ep) {
            a = args_for(env);
            a.in = env->roll_s[cur];
            a.ep = *ep;
            cuda_check(zs::launch_episode_finalize(a, env->d_initial_s, env->d_logged, s), "episode finalize");
        }
        if (final_state) copy_state(env, final_state, &env->roll_s[cur], 2, s);
    });
}

ZSIM_API int zsim_rollout_policy(zsim_env* env, zsim_policy* policy, int32_t use_argmax, uint64_t seed,
                                 int32_t horizon, const zsim_episode_view* ep, const zsim_obs_view* obs,
                                 const zsim_state_view* final_state, void* stream) {
    return guarded([&] {
        check_view(env, "rollout_policy");
        if (!policy) raise(Err::invalid_argument, "rollout_policy: null policy");
        if (horizon <= 0) raise(Err::invalid_argument, "rollout_policy: horizon must be > 0");
        if (ep) {
            check_episode(env, ep, "rollout_policy");
            if (ep->horizon != horizon) raise(Err::invalid_argument, "rollout_policy: episode horizon mismatch");
        }
        set_device(env);
        ensure_host_arrays(env);
        if (!env->roll_buf) {
            cuda_check(cudaMalloc(&env->roll_buf, 2 * env->sl.bytes + env->ol.bytes + env->sol.bytes),
                       "cudaMalloc(rollout scratch)");
            unsigned char* p = static_cast<unsigned char*>(env->roll_buf);
            carve_state(p, env->sl, &env->roll_s[0]);
            carve_state(p + env->sl.bytes, env->sl, &env->roll_s[1]);
            carve_obs(p + 2 * env->sl.bytes, env->ol, &env->roll_obs);
            carve_stepout(p + 2 * env->sl.bytes + env->ol.bytes, env->sol, &env->roll_so);
        }
        const size_t nb = al(size_t(env->B) * 4);
        if (!env->pol_buf) cuda_check(cudaMalloc(&env->pol_buf, 4 * nb), "cudaMalloc(policy rollout scratch)");
        unsigned char* pb = static_cast<unsigned char*>(env->pol_buf);
        int32_t* pa = reinterpret_cast<int32_t*>(pb);
        int32_t* ps = reinterpret_cast<int32_t*>(pb + nb);
        float* plogp = reinterpret_cast<float*>(pb + 2 * nb);
        float* pvalue = reinterpret_cast<float*>(pb + 3 * nb);
        cudaStream_t s = as_stream(stream);
        zs::KernelArgs a = args_for(env);
        a.seed = seed;
        a.out = env->roll_s[0];
        cuda_check(zs::launch_reset(a, env->grid, s), "reset kernel");
        a = args_for(env);
        a.in = env->roll_s[0];
        a.obs = obs ? obs[0] : env->roll_obs;
        cuda_check(zs::launch_step_observe(a, zs::kModeObserve, env->launch_policy, s), "observe kernel");
        auto act = [&](const zsim_obs_view* o, const zsim_state_view& st) {
            // NNPolicy::act on obs[t] with the rows' rng streams (simcore.cpp:591)
            if (zsim_policy_act(policy, o, env->B, st.rng, use_argmax, pa, ps, plogp, pvalue, nullptr, stream) !=
                ZSIM_OK)
                raise(Err::runtime, std::string("rollout_policy: ") + g_last_error);
        };
        int cur = 0;
        for (int t = 0; t < horizon; ++t) {
            act(obs ? &obs[t] : &env->roll_obs, env->roll_s[cur]);
            a = args_for(env);
            a.in = env->roll_s[cur];
            a.out = env->roll_s[cur ^ 1];
            a.accel = pa;
            a.steer = ps;
            a.act_len = ep ? -2 : 0;  // without recording the plain step kernel reads accel / steer [B]
            a.pol_logp = plogp;
            a.pol_value = pvalue;
            a.so = env->roll_so;
            if (ep) {
                a.ep = *ep;
                a.ep_t = t;
            }
            a.obs = obs ? obs[t + 1] : env->roll_obs;
            cuda_check(zs::launch_step_observe(a, zs::kModeStepObserve, env->launch_policy, s), "step+observe kernel");
            cur ^= 1;
        }
        // the final observation's value is the bootstrap (simcore.cpp:609-613)
        act(obs ? &obs[horizon] : &env->roll_obs, env->roll_s[cur]);
        if (ep) {
            a = args_for(env);
            a.in = env->roll_s[cur];
            a.ep = *ep;
            a.final_value = pvalue;
            cuda_check(zs::launch_episode_finalize(a, env->d_initial_s, env->d_logged, s), "episode finalize");
        }
        if (final_state) copy_state(env, final_state, &env->roll_s[cur], 2, s);
    });
}

ZSIM_API int zsim_score_defaults(zsim_score_bounds* b, zsim_comfort_weights* w) {
    return guarded([&] {
        if (b) *b = zsim_score_bounds{0.8, 0.05, 0.5, 0.5, 0.5, 0.8};  // metrics.hpp:11-18
        if (w) *w = zsim_comfort_weights{0.1, 0.05};                   // metrics.hpp:20-23
    });
}

ZSIM_API int zsim_episode_metrics(zsim_env* env, const zsim_episode_view* ep, const zsim_score_bounds* bounds,
                                  const zsim_comfort_weights* weights, const zsim_metric_view* rows, double* sums_dev,
                                  void* stream) {
    return guarded([&] {
        check_view(env, "episode_metrics");
        check_episode(env, ep, "episode_metrics");
        check_view(sums_dev, "episode_metrics");
        set_device(env);
        zsim_score_bounds bb;
        zsim_comfort_weights cw;
        zsim_score_defaults(&bb, &cw);
        if (bounds) bb = *bounds;
        if (weights) cw = *weights;
        for (double l : {bb.progress, bb.collision, bb.off_route, bb.stop_line, bb.traffic_light, bb.comfort})
            if (!(l >= 0.0 && l < 1.0)) raise(Err::invalid_argument, "map_score: l outside [0,1)");
        if (!env->d_metrics_scratch) {
            cuda_check(cudaMalloc(&env->d_metrics_scratch, sizeof(double) * size_t(zs::metrics_scratch_doubles(env->B))),
                       "cudaMalloc(metrics scratch)");
        }
        zs::KernelArgs a = args_for(env);
        a.ep = *ep;
        zsim_metric_view mv{};
        if (rows) mv = *rows;
        cuda_check(zs::launch_episode_metrics(a, bb, cw, mv, sums_dev, env->d_metrics_scratch, as_stream(stream)),
                   "episode_metrics kernel");
    });
}

ZSIM_API int zsim_aggregate_finalize(const double* sums, int32_t n_parts, double* out12) {
    return guarded([&] {
        if (!sums || !out12 || n_parts <= 0) raise(Err::invalid_argument, "aggregate_finalize: bad arguments");
        double t[ZSIM_AGG_LEN] = {};
        for (int p = 0; p < n_parts; ++p)
            for (int k = 0; k < ZSIM_AGG_LEN; ++k) t[k] += sums[size_t(p) * ZSIM_AGG_LEN + k];
        // metrics::aggregate (metrics.cpp:120-130)
        double o[ZSIM_AGG_LEN] = {t[0], t[1], 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        if (t[0] > 0) {
            const double n = t[0];
            for (int k = 2; k <= 9; ++k) o[k] = t[k] / n;
            o[10] = t[10] / n;
            o[11] = t[11] / n;
        }
        std::memcpy(out12, o, sizeof(o));
    });
}

ZSIM_API int zsim_set_launch_policy(zsim_env* env, int32_t policy) {
    return guarded([&] {
        check_view(env, "set_launch_policy");
        if (policy < 0 || policy > 2) raise(Err::invalid_argument, "launch policy must be 0, 1 or 2");
        env->launch_policy = policy;
    });
}

ZSIM_API int zsim_set_debug_topk(zsim_env* env, int32_t* dev_idx) {
    return guarded([&] {
        check_view(env, "set_debug_topk");
        env->base.dbg = dev_idx;
    });
}

ZSIM_API int zsim_check_errors(zsim_env* env, void* stream) {
    return guarded([&] {
        check_view(env, "check_errors");
        set_device(env);
        int32_t h = 0;
        cuda_check(cudaMemcpyAsync(&h, env->d_err, 4, cudaMemcpyDeviceToHost, as_stream(stream)), "read error word");
        cuda_check(cudaStreamSynchronize(as_stream(stream)), "stream sync");
        if (h) {
            cuda_check(cudaMemsetAsync(env->d_err, 0, 4, as_stream(stream)), "clear error word");
            cuda_check(cudaStreamSynchronize(as_stream(stream)), "stream sync");
            if (h & 1) raise(Err::invalid_argument, "action index out of range");
            raise(Err::runtime, "non-finite ego state (NaN/Inf) after a step");
        }
    });
}

ZSIM_API int zsim_reset_host(zsim_env* env, uint64_t seed, const zsim_state_view* out_host) {
    return guarded([&] {
        check_view(env, "reset_host");
        check_view(out_host, "reset_host");
        set_device(env);
        ensure_host_scratch(env);
        zs::KernelArgs a = args_for(env);
        a.out = env->h_out;
        a.seed = seed;
        cuda_check(zs::launch_reset(a, env->grid, env->h_stream), "reset kernel");
        copy_state(env, out_host, &env->h_out, 1, env->h_stream);
        cuda_check(cudaStreamSynchronize(env->h_stream), "stream sync");
    });
}

ZSIM_API int zsim_step_host(zsim_env* env, const zsim_state_view* in_host, const int32_t* accel,
                            const int32_t* steer, const zsim_state_view* out_host, const zsim_stepout_view* so_host) {
    return guarded([&] {
        check_view(env, "step_host");
        check_view(in_host, "step_host");
        check_view(out_host, "step_host");
        check_view(so_host, "step_host");
        check_actions_host(env, accel, steer);
        set_device(env);
        ensure_host_scratch(env);
        cudaStream_t s = env->h_stream;
        copy_state(env, &env->h_in, in_host, 0, s);
        const size_t B = size_t(env->B);
        cuda_check(cudaMemcpyAsync(env->h_act, accel, 4 * B, cudaMemcpyHostToDevice, s), "action upload");
        cuda_check(cudaMemcpyAsync(env->h_act + B, steer, 4 * B, cudaMemcpyHostToDevice, s), "action upload");
        zs::KernelArgs a = args_for(env);
        a.in = env->h_in;
        a.out = env->h_out;
        a.accel = env->h_act;
        a.steer = env->h_act + B;
        a.so = env->h_so;
        cuda_check(zs::launch_step_observe(a, zs::kModeStep, env->launch_policy, s), "step kernel");
        copy_state(env, out_host, &env->h_out, 1, s);
        copy_stepout(env, so_host, &env->h_so, 1, s);
        cuda_check(cudaStreamSynchronize(s), "stream sync");
    });
}

ZSIM_API int zsim_observe_host(zsim_env* env, const zsim_state_view* in_host, const zsim_obs_view* obs_host) {
    return guarded([&] {
        check_view(env, "observe_host");
        check_view(in_host, "observe_host");
        check_view(obs_host, "observe_host");
        set_device(env);
        ensure_host_scratch(env);
        cudaStream_t s = env->h_stream;
        copy_state(env, &env->h_in, in_host, 0, s);
        // row chunks: the observation of chunk k streams to the host (copy
        // stream) while chunk k+1 is computed
        const int B = env->B;
        const int nch = B >= 2048 ? 2 : 1;
        if (!env->h_copy) {
            cuda_check(cudaStreamCreateWithFlags(&env->h_copy, cudaStreamNonBlocking), "cudaStreamCreate");
            for (auto& e : env->h_ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        }
        const ObsLayout& L = env->ol;
        const int K[5] = {9, env->cfg.n_agents * 6, env->cfg.n_road * 12, env->cfg.n_route * 5, 2};
        float* dst[5] = {obs_host->active, obs_host->agents, obs_host->road, obs_host->route, obs_host->value_only};
        const float* src[5] = {env->h_obs.active, env->h_obs.agents, env->h_obs.road, env->h_obs.route,
                               env->h_obs.value_only};
        (void)L;
        for (int c = 0; c < nch; ++c) {
            const int lo = int(int64_t(B) * c / nch), hi = int(int64_t(B) * (c + 1) / nch);
            zs::KernelArgs a = args_for(env);
            a.in = env->h_in;
            a.obs = env->h_obs;
            a.row_lo = lo;
            a.row_hi = hi;
            cuda_check(zs::launch_step_observe(a, zs::kModeObserve, 1, s), "observe kernel");
            cuda_check(cudaEventRecord(env->h_ev[c], s), "event");
            cuda_check(cudaStreamWaitEvent(env->h_copy, env->h_ev[c], 0), "event wait");
            for (int k = 0; k < 5; ++k) {
                const size_t o = size_t(lo) * size_t(K[k]), n = size_t(hi - lo) * size_t(K[k]);
                cuda_check(cudaMemcpyAsync(dst[k] + o, src[k] + o, 4 * n, cudaMemcpyDeviceToHost, env->h_copy),
                           "obs copy");
            }
        }
        cuda_check(cudaStreamSynchronize(env->h_copy), "stream sync");
        cuda_check(cudaStreamSynchronize(s), "stream sync");
    });
}

ZSIM_API int zsim_step_observe_host(zsim_env* env, const zsim_state_view* in_host, const int32_t* accel,
                                    const int32_t* steer, const zsim_state_view* out_host,
                                    const zsim_stepout_view* so_host, const zsim_obs_view* obs_host) {
    return guarded([&] {
        check_view(env, "step_observe_host");
        check_view(in_host, "step_observe_host");
        check_view(out_host, "step_observe_host");
        check_view(so_host, "step_observe_host");
        check_view(obs_host, "step_observe_host");
        check_actions_host(env, accel, steer);
        set_device(env);
        ensure_host_scratch(env);
        cudaStream_t s = env->h_stream;
        copy_state(env, &env->h_in, in_host, 0, s);
        const int B = env->B;
        cuda_check(cudaMemcpyAsync(env->h_act, accel, 4 * size_t(B), cudaMemcpyHostToDevice, s), "action upload");
        cuda_check(cudaMemcpyAsync(env->h_act + B, steer, 4 * size_t(B), cudaMemcpyHostToDevice, s), "action upload");
        if (!env->h_copy) {
            cuda_check(cudaStreamCreateWithFlags(&env->h_copy, cudaStreamNonBlocking), "cudaStreamCreate");
            for (auto& e : env->h_ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        }
        // row chunks: chunk k's observation streams to the host (copy stream)
        // while chunk k+1 steps and observes; the state and StepOut follow
        // the last chunk
        const int nch = B >= 2048 ? 2 : 1;  // (4 chunks: C1 e2e -4%, each chunk pays the row latency)
        const int K[5] = {9, env->cfg.n_agents * 6, env->cfg.n_road * 12, env->cfg.n_route * 5, 2};
        float* dst[5] = {obs_host->active, obs_host->agents, obs_host->road, obs_host->route, obs_host->value_only};
        const float* src[5] = {env->h_obs.active, env->h_obs.agents, env->h_obs.road, env->h_obs.route,
                               env->h_obs.value_only};
        for (int c = 0; c < nch; ++c) {
            const int lo = int(int64_t(B) * c / nch), hi = int(int64_t(B) * (c + 1) / nch);
            zs::KernelArgs a = args_for(env);
            a.in = env->h_in;
            a.out = env->h_out;
            a.accel = env->h_act;
            a.steer = env->h_act + B;
            a.so = env->h_so;
            a.obs = env->h_obs;
            a.row_lo = lo;
            a.row_hi = hi;
            cuda_check(zs::launch_step_observe(a, zs::kModeStepObserve, env->launch_policy, s), "step_observe kernel");
            cuda_check(cudaEventRecord(env->h_ev[c], s), "event");
            cuda_check(cudaStreamWaitEvent(env->h_copy, env->h_ev[c], 0), "event wait");
            for (int k = 0; k < 5; ++k) {
                const size_t o = size_t(lo) * size_t(K[k]), n = size_t(hi - lo) * size_t(K[k]);
                cuda_check(cudaMemcpyAsync(dst[k] + o, src[k] + o, 4 * n, cudaMemcpyDeviceToHost, env->h_copy),
                           "obs copy");
            }
        }
        copy_state(env, out_host, &env->h_out, 1, env->h_copy);
        copy_stepout(env, so_host, &env->h_so, 1, env->h_copy);
        cuda_check(cudaStreamSynchronize(env->h_copy), "stream sync");
        cuda_check(cudaStreamSynchronize(s), "stream sync");
    });
}

ZSIM_API int zsim_stress_config_defaults(zsim_stress_config* c) {
    return guarded([&] {
        if (!c) raise(Err::invalid_argument, "null config");
        c->count = 64;
        c->num_steps = 92;
        c->agents = 32;
        c->road_points = 2048;
        c->lanes = 4;
        c->lane_vertices = 64;
        c->dt = 0.1;
        c->speed_limit = 10.0;
        c->lane_width = 3.5;
        c->first_index = 0;
        c->flags = 0;
    });
}

ZSIM_API int zsim_stress_generate(const zsim_stress_config* cfg, uint64_t seed, uint8_t** out_buf, size_t* out_len) {
    return guarded([&] {
        if (!cfg || !out_buf || !out_len) raise(Err::invalid_argument, "null argument");
        std::string img = zs::stress_generate(*cfg, seed);
        uint8_t* p = static_cast<uint8_t*>(std::malloc(img.size()));
        if (!p) raise(Err::runtime, "out of host memory");
        std::memcpy(p, img.data(), img.size());
        *out_buf = p;
        *out_len = img.size();
    });
}

ZSIM_API void zsim_free_buffer(void* buf) { std::free(buf); }

}  // extern "C"
