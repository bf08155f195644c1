// zsim_stressgen.cpp -- deterministic synthetic scenarios at the BASELINE
// shapes.  The reference generator (scenario_gen.cpp) caps the
// agent count at a handful per scenario (scenario_gen.cpp:464-479), so the
// throughput configs need their own generator.  Every scenario it emits is a
// valid ZSIM record (checked against the reference `validate`,
// scenario_io.cpp:193-271, by the parity suite).
//
// Layout of one scenario: a constant-curvature corridor (straight or gentle
// arc) with `lanes` parallel route lanes of `lane_vertices` border vertices;
// the ego is logged by driving the kinematic bicycle model
// (dynamics.cpp:10-19) with table actions along lane 0; `agents-1` replayed
// agents move along same-direction and oncoming lanes; `road_points` feature
// points are spread over polylines within +-40 m of the corridor; one traffic
// light and one stop line sit on lane 0.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/zsim_gpu.h"
#include "zsim_geom.cuh"
#include "zsim_scenario.hpp"

namespace zs {
namespace {

// splitmix64 stream with the reference Rng's seeding and split rule
// (common.hpp:28-51), so per-scenario streams are `Rng(seed).split(i)`.
struct Stream {
    uint64_t state;
    explicit Stream(uint64_t seed) : state(seed + 0x9e3779b97f4a7c15ull) {}
    uint64_t next() {
        state += 0x9e3779b97f4a7c15ull;
        return splitmix_mix(state);
    }
    double unit() { return double(next() >> 11) * 0x1.0p-53; }
    double uni(double lo, double hi) { return lo + (hi - lo) * unit(); }
    Stream split(uint64_t tag) { return Stream(next() ^ (tag * 0xd1342543de82ef95ull + 0x2545f4914f6cdd1dull)); }
};

// Analytic corridor: arc-length parameterised circle (or line) through the
// origin with initial heading h0 and signed curvature k.
struct Corridor {
    double ox, oy, h0, k;
    double heading(double s) const { return h0 + k * s; }
    void pos(double s, double lat, double& x, double& y) const {
        double h = heading(s);
        if (k == 0.0) {
            x = ox + s * std::cos(h0);
            y = oy + s * std::sin(h0);
        } else {
            x = ox + (std::sin(h) - std::sin(h0)) / k;
            y = oy - (std::cos(h) - std::cos(h0)) / k;
        }
        x += -std::sin(h) * lat;
        y += std::cos(h) * lat;
    }
    std::vector<float> polyline(double s0, double s1, double lat, int n) const {
        std::vector<float> xy;
        xy.reserve(size_t(2 * n));
        for (int i = 0; i < n; ++i) {
            double s = s0 + (s1 - s0) * double(i) / double(n - 1);
            double x, y;
            pos(s, lat, x, y);
            xy.push_back(float(x));
            xy.push_back(float(y));
        }
        return xy;
    }
};

const double kAccel[7] = {-4.0, -2.0, -0.5, 0.0, 0.5, 2.0, 4.0};
const double kSteer[5] = {-0.4, -0.1, 0.0, 0.1, 0.4};

int nearest(const double* bins, int n, double v) {
    int best = 0;
    double bd = std::fabs(v - bins[0]);
    for (int i = 1; i < n; ++i) {
        double d = std::fabs(v - bins[i]);
        if (d < bd) {
            bd = d;
            best = i;
        }
    }
    return best;
}

Scene make_scene(const zsim_stress_config& cfg, Stream rng, int index) {
    Scene sc;
    sc.id = "stress-" + std::to_string(index);
    sc.num_steps = uint32_t(cfg.num_steps);
    sc.dt = cfg.dt;
    sc.speed_limit = float(cfg.speed_limit);
    const double w = cfg.lane_width;
    const int T = cfg.num_steps;

    Corridor cor;
    cor.ox = rng.uni(-200.0, 200.0);
    cor.oy = rng.uni(-200.0, 200.0);
    cor.h0 = rng.uni(-kPi, kPi);
    cor.k = rng.unit() < 0.5 ? 0.0 : (rng.unit() < 0.5 ? -1.0 : 1.0) / rng.uni(80.0, 200.0);

    // --- ego: bicycle model with table actions, pure pursuit on lane 0 ---
    const double L = 3.0, dmax = 0.55;
    double cruise = rng.uni(7.0, 9.5);
    double s0 = 5.0;
    double ex, ey;
    cor.pos(s0, 0.0, ex, ey);
    double eh = cor.heading(s0), ev = cruise * rng.uni(0.8, 1.0), ed = 0.0;
    double s_est = s0;
    for (int t = 0; t < T; ++t) {
        sc.ego_x.push_back(float(ex));
        sc.ego_y.push_back(float(ey));
        sc.ego_h.push_back(float(eh));
        sc.ego_v.push_back(float(ev));
        if (t + 1 == T) break;
        double dv = cruise - ev;
        double a = dv > 0.3 ? 0.5 : (dv < -0.3 ? -0.5 : 0.0);
        double look = clampd(1.2 + 0.5 * ev, 2.5, 7.0);
        double tx, ty;
        cor.pos(s_est + look, 0.0, tx, ty);
        double alpha = wrap_angle(std::atan2(ty - ey, tx - ex) - eh);
        double d_des = clampd(std::atan(2.0 * L * std::sin(alpha) / look), -dmax, dmax);
        double rate = std::fabs(d_des - ed) < 0.003 ? 0.0 : kSteer[nearest(kSteer, 5, (d_des - ed) / cfg.dt)];
        a = kAccel[nearest(kAccel, 7, a)];
        // explicit Euler from the pre-step state (dynamics.cpp:10-19)
        double nx = ex + ev * std::cos(eh) * cfg.dt;
        double ny = ey + ev * std::sin(eh) * cfg.dt;
        double nh = wrap_angle(eh + ev / L * std::tan(ed) * cfg.dt);
        double nv = maxd(ev + a * cfg.dt, 0.0);
        double nd = clampd(ed + rate * cfg.dt, -dmax, dmax);
        s_est += ev * cfg.dt;
        ex = nx;
        ey = ny;
        eh = nh;
        ev = nv;
        ed = nd;
    }
    double s_final = s_est;
    double route_end = s_final + 16.0;
    double gx, gy;
    cor.pos(s_final + 4.0, 0.0, gx, gy);
    sc.goal_x = float(gx);
    sc.goal_y = float(gy);

    // --- route lanes: lane k at lateral k*w; the last lane (if >= 3 lanes) is
    // valid on [0, 0.7*route_end] only, exercising RouteFrame clipping ---
    int C = std::max(2, cfg.lane_vertices);
    for (int k = 0; k < cfg.lanes; ++k) {
        LaneBorders lb;
        lb.lane_id = uint32_t(k);
        double lat = double(k) * w;
        lb.left_xy = cor.polyline(0.0, route_end, lat + 0.5 * w, C);
        lb.right_xy = cor.polyline(0.0, route_end, lat - 0.5 * w, C);
        lb.s_start = 0.f;
        lb.s_end = float(k >= 2 && k == cfg.lanes - 1 ? 0.7 * route_end : route_end);
        sc.lanes.push_back(std::move(lb));
    }

    // --- road features: lane markings and edges first, then parallel
    // polylines spread over +-40 m; point budget exactly road_points ---
    int P = std::max(2, cfg.road_points);
    int per = 32;
    int nfeat = std::max(1, P / per);
    int assigned = 0;
    for (int f = 0; f < nfeat; ++f) {
        int npts = (f == nfeat - 1) ? P - assigned : per;
        if (npts < 2) npts = 2;
        assigned += npts;
        double lat;
        uint8_t kind, dir;
        if (f <= cfg.lanes) {
            lat = (double(f) - 0.5) * w;  // lane markings between route lanes
            kind = 0;
            dir = 1;
        } else if (f == cfg.lanes + 1) {
            lat = -0.5 * w - rng.uni(0.6, 1.4);
            kind = 4;
            dir = 0;
        } else {
            lat = rng.uni(-40.0, 40.0);
            kind = uint8_t(f % 5);
            dir = uint8_t((f / 5) % 4);
        }
        double a0 = -40.0 + rng.uni(-5.0, 5.0), a1 = route_end + 40.0 + rng.uni(-5.0, 5.0);
        if (kind == 1 || kind == 2) {  // crosswalk / stop-line paint: short transverse-ish strokes
            double sm = rng.uni(0.0, route_end);
            a0 = sm - 3.0;
            a1 = sm + 3.0;
        }
        Feature ft;
        ft.kind = kind;
        ft.dir = dir;
        ft.xy = cor.polyline(a0, a1, lat, npts);
        sc.features.push_back(std::move(ft));
    }

    // --- agents: same-direction lanes, lane 0 ahead/behind, oncoming ---
    for (int j = 0; j + 1 < cfg.agents; ++j) {
        AgentLog ag;
        ag.id = "a" + std::to_string(j);
        ag.length = float(rng.uni(4.0, 5.0));
        ag.width = float(rng.uni(1.7, 2.0));
        int kind = int(rng.unit() * 3.0);
        double lat, sa, sp = rng.uni(6.0, 12.0);
        bool oncoming = false;
        if (cfg.flags & 1) {
            // C2 actor: a route lane, same direction, inside the corridor for the whole log
            const int ln = int(rng.unit() * double(std::max(1, cfg.lanes - 1)));
            lat = double(ln) * w + rng.uni(-0.3, 0.3);
            sp = std::max(0.5, std::min(sp, (route_end - 12.0) / (cfg.dt * double(T - 1))));  // log ends on the route
            const double span = sp * cfg.dt * double(T - 1);
            sa = rng.uni(0.0, std::max(1.0, route_end - span - 6.0));
        } else if (kind == 0) {
            lat = double(1 + int(rng.unit() * std::max(1, cfg.lanes - 1))) * w + rng.uni(-0.3, 0.3);
            sa = rng.uni(-30.0, route_end + 20.0);
        } else if (kind == 1) {
            lat = rng.uni(-0.2, 0.2);
            sa = rng.unit() < 0.5 ? s0 + rng.uni(12.0, 60.0) : s0 - rng.uni(15.0, 60.0);
        } else {
            lat = -w + rng.uni(-0.3, 0.3);
            sa = rng.uni(0.0, route_end + 60.0);
            oncoming = true;
        }
        int inv_from = T, inv_to = T;
        if (!(cfg.flags & 1) && rng.unit() < 0.15) {
            inv_from = int(rng.unit() * T);
            inv_to = std::min(T, inv_from + 5 + int(rng.unit() * 30.0));
        }
        for (int t = 0; t < T; ++t) {
            double s = sa + (oncoming ? -sp : sp) * cfg.dt * double(t);
            double x, y;
            cor.pos(s, lat, x, y);
            double h = cor.heading(s) + (oncoming ? kPi : 0.0);
            ag.x.push_back(float(x));
            ag.y.push_back(float(y));
            ag.heading.push_back(float(wrap_angle(h)));
            ag.speed.push_back(float(sp));
            ag.valid.push_back((t >= inv_from && t < inv_to) ? 0 : 1);
        }
        sc.agents.push_back(std::move(ag));
    }

    // --- one traffic light and one stop line on lane 0 ---
    {
        Light lt;
        lt.signal_id = 1;
        double sl = s0 + rng.uni(25.0, 45.0), x, y;
        cor.pos(sl, 0.0, x, y);
        lt.stop_x = float(x);
        lt.stop_y = float(y);
        int t_green = int(rng.uni(0.0, 40.0)), t_yellow = t_green + 20 + int(rng.uni(0.0, 20.0));
        for (int t = 0; t < T; ++t) {
            uint8_t st = t < 3 ? 3 : (t < t_green ? 0 : (t < t_yellow ? 2 : (t < t_yellow + 8 ? 1 : 0)));
            lt.state.push_back(st);
        }
        sc.lights.push_back(std::move(lt));
    }
    {
        StopLine st;
        double ss = s0 + rng.uni(55.0, 75.0), x, y;
        cor.pos(ss, 0.0, x, y);
        st.pos_x = float(x);
        st.pos_y = float(y);
        double lx, ly, rx, ry;
        cor.pos(ss, 0.5 * w, lx, ly);
        cor.pos(ss, -0.5 * w, rx, ry);
        st.xy = {float(lx), float(ly), float(rx), float(ry)};
        sc.stops.push_back(std::move(st));
    }
    return sc;
}

}  // namespace

void stress_check(const zsim_stress_config& cfg) {
    if (cfg.count <= 0) raise(Err::config, "stress: count must be > 0");
    if (cfg.num_steps < 2) raise(Err::config, "stress: num_steps must be >= 2");
    if (cfg.agents < 1) raise(Err::config, "stress: agents must be >= 1 (the ego)");
    if (cfg.lanes < 1 || cfg.lane_vertices < 2) raise(Err::config, "stress: need >= 1 lane of >= 2 vertices");
    if (cfg.road_points < 2) raise(Err::config, "stress: road_points must be >= 2");
    if (!(cfg.dt > 0.0)) raise(Err::config, "stress: dt must be > 0");
    if (cfg.first_index < 0) raise(Err::config, "stress: first_index must be >= 0");
}

Scene stress_scene(const zsim_stress_config& cfg, uint64_t seed, int64_t i) {
    // Rng(seed).split(i): the root has advanced i+1 times (reset_rng_state's closed form)
    Stream s(0);
    s.state = reset_rng_state(seed, uint64_t(i));
    return make_scene(cfg, s, int(i));
}

std::string stress_generate(const zsim_stress_config& cfg, uint64_t seed) {
    stress_check(cfg);
    std::string out = zsim_header(cfg.dt);
    for (int k = 0; k < cfg.count; ++k)
        zsim_encode_append(out, stress_scene(cfg, seed, int64_t(cfg.first_index) + k));
    return out;
}

}  // namespace zs
