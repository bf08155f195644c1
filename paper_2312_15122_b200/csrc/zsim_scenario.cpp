// zsim_scenario.cpp -- ZSIM codec and host staging (see zsim_scenario.hpp).
// Compiled with -ffp-contract=off: the staged fp64 values (lane frames, goal_s,
// initial_s, stop/light s, route border validity) are bit-identical to the
// reference's Env::Env (simcore.cpp:203-233).
#include "zsim_scenario.hpp"

#include <cmath>
#include <cstring>

#include "zsim_geom.cuh"

namespace zs {

namespace {

const char kMagic[4] = {'Z', 'S', 'I', 'M'};
constexpr uint16_t kVersion = 1;

struct Cursor {
    const uint8_t* p;
    const uint8_t* end;
    std::string origin;

    void need(size_t n) const {
        if (size_t(end - p) < n) raise(Err::io, origin + ": truncated record");
    }
    template <class T>
    T take() {
        need(sizeof(T));
        T v;
        std::memcpy(&v, p, sizeof(T));
        p += sizeof(T);
        return v;
    }
    std::string str() {
        uint32_t n = take<uint32_t>();
        need(n);
        std::string s(reinterpret_cast<const char*>(p), n);
        p += n;
        return s;
    }
    std::vector<float> f32s() {
        uint32_t n = take<uint32_t>();
        need(size_t(n) * 4);
        std::vector<float> v(n);
        if (n) std::memcpy(v.data(), p, size_t(n) * 4);
        p += size_t(n) * 4;
        return v;
    }
    std::vector<uint8_t> u8s() {
        uint32_t n = take<uint32_t>();
        need(n);
        std::vector<uint8_t> v(p, p + n);
        p += n;
        return v;
    }
};

template <class T>
void put(std::string& o, T v) {
    o.append(reinterpret_cast<const char*>(&v), sizeof(T));
}
void put_str(std::string& o, const std::string& s) {
    put<uint32_t>(o, uint32_t(s.size()));
    o.append(s);
}
void put_f32s(std::string& o, const std::vector<float>& v) {
    put<uint32_t>(o, uint32_t(v.size()));
    o.append(reinterpret_cast<const char*>(v.data()), v.size() * 4);
}
void put_u8s(std::string& o, const std::vector<uint8_t>& v) {
    put<uint32_t>(o, uint32_t(v.size()));
    o.append(reinterpret_cast<const char*>(v.data()), v.size());
}

double norm2d(double x0, double y0, double x1, double y1) {
    double dx = x0 - x1, dy = y0 - y1;
    return std::sqrt(dx * dx + dy * dy);
}

}  // namespace

// Dataset::Dataset (scenario_io.cpp:347-377) over a memory image.
ZsimIndex zsim_index(const uint8_t* buf, size_t n) {
    ZsimIndex idx;
    if (n < 16 || std::memcmp(buf, kMagic, 4) != 0) raise(Err::io, "<memory>: not a ZSIM scenario file");
    uint16_t version;
    std::memcpy(&version, buf + 4, 2);
    if (version != kVersion) raise(Err::io, "<memory>: unsupported format version " + std::to_string(version));
    std::memcpy(&idx.dt, buf + 8, 8);
    uint64_t off = 16;
    while (off < n) {
        if (n - off < 4) raise(Err::io, "<memory>: truncated record header");
        uint32_t len;
        std::memcpy(&len, buf + off, 4);
        if (n - off - 4 < len) raise(Err::io, "<memory>: truncated record body");
        idx.records.emplace_back(off + 4, len);
        off += 4 + uint64_t(len);
    }
    return idx;
}

// decode_record (scenario_io.cpp:132-189).
Scene zsim_decode(const uint8_t* buf, size_t n, const ZsimIndex& idx, int64_t record) {
    (void)n;
    if (record < 0 || record >= int64_t(idx.records.size())) {
        raise(Err::invalid_argument, "scenario index " + std::to_string(record) + " out of range (dataset has " +
                                         std::to_string(idx.records.size()) + ")");
    }
    auto [off, len] = idx.records[size_t(record)];
    Cursor c{buf + off, buf + off + len, "<memory>[" + std::to_string(record) + "]"};
    Scene s;
    s.dt = idx.dt;
    s.id = c.str();
    s.num_steps = c.take<uint32_t>();
    s.ego_x = c.f32s();
    s.ego_y = c.f32s();
    s.ego_h = c.f32s();
    s.ego_v = c.f32s();
    s.agents.resize(c.take<uint32_t>());
    for (auto& a : s.agents) {
        a.id = c.str();
        a.length = c.take<float>();
        a.width = c.take<float>();
        a.x = c.f32s();
        a.y = c.f32s();
        a.heading = c.f32s();
        a.speed = c.f32s();
        a.valid = c.u8s();
    }
    s.lanes.resize(c.take<uint32_t>());
    for (auto& l : s.lanes) {
        l.lane_id = c.take<uint32_t>();
        l.left_xy = c.f32s();
        l.right_xy = c.f32s();
        l.s_start = c.take<float>();
        l.s_end = c.take<float>();
    }
    s.features.resize(c.take<uint32_t>());
    for (auto& f : s.features) {
        f.kind = c.take<uint8_t>();
        f.dir = c.take<uint8_t>();
        f.xy = c.f32s();
    }
    s.lights.resize(c.take<uint32_t>());
    for (auto& t : s.lights) {
        t.signal_id = c.take<uint32_t>();
        t.stop_x = c.take<float>();
        t.stop_y = c.take<float>();
        t.state = c.u8s();
    }
    s.stops.resize(c.take<uint32_t>());
    for (auto& sl : s.stops) {
        sl.xy = c.f32s();
        sl.pos_x = c.take<float>();
        sl.pos_y = c.take<float>();
    }
    s.speed_limit = c.take<float>();
    s.goal_x = c.take<float>();
    s.goal_y = c.take<float>();
    if (c.p != c.end) raise(Err::io, c.origin + ": trailing bytes in record");
    return s;
}

std::string zsim_header(double dt) {
    std::string o(kMagic, 4);
    put<uint16_t>(o, kVersion);
    put<uint16_t>(o, 0);
    put<double>(o, dt);
    return o;
}

// encode_record (scenario_io.cpp:80-130) + the u32 length prefix.
void zsim_encode_append(std::string& out, const Scene& s) {
    std::string r;
    put_str(r, s.id);
    put<uint32_t>(r, s.num_steps);
    put_f32s(r, s.ego_x);
    put_f32s(r, s.ego_y);
    put_f32s(r, s.ego_h);
    put_f32s(r, s.ego_v);
    put<uint32_t>(r, uint32_t(s.agents.size()));
    for (const auto& a : s.agents) {
        put_str(r, a.id);
        put<float>(r, a.length);
        put<float>(r, a.width);
        put_f32s(r, a.x);
        put_f32s(r, a.y);
        put_f32s(r, a.heading);
        put_f32s(r, a.speed);
        put_u8s(r, a.valid);
    }
    put<uint32_t>(r, uint32_t(s.lanes.size()));
    for (const auto& l : s.lanes) {
        put<uint32_t>(r, l.lane_id);
        put_f32s(r, l.left_xy);
        put_f32s(r, l.right_xy);
        put<float>(r, l.s_start);
        put<float>(r, l.s_end);
    }
    put<uint32_t>(r, uint32_t(s.features.size()));
    for (const auto& f : s.features) {
        put<uint8_t>(r, f.kind);
        put<uint8_t>(r, f.dir);
        put_f32s(r, f.xy);
    }
    put<uint32_t>(r, uint32_t(s.lights.size()));
    for (const auto& t : s.lights) {
        put<uint32_t>(r, t.signal_id);
        put<float>(r, t.stop_x);
        put<float>(r, t.stop_y);
        put_u8s(r, t.state);
    }
    put<uint32_t>(r, uint32_t(s.stops.size()));
    for (const auto& sl : s.stops) {
        put_f32s(r, sl.xy);
        put<float>(r, sl.pos_x);
        put<float>(r, sl.pos_y);
    }
    put<float>(r, s.speed_limit);
    put<float>(r, s.goal_x);
    put<float>(r, s.goal_y);
    put<uint32_t>(out, uint32_t(r.size()));
    out += r;
}

// RouteFrame::build (roads.cpp:43-103): pointwise midpoint centerline (right
// border resampled by arc fraction when vertex counts differ), cumulative s
// from the lane's s_start, clipped to s_end with an interpolated endpoint.
void build_frame(const Scene& sc, RouteCtx& ctx) {
    ctx.lanes.clear();
    ctx.route_length = 0.0;
    for (const auto& lane : sc.lanes) {
        size_t nl = lane.left_xy.size() / 2, nr = lane.right_xy.size() / 2;
        if (nl < 2 || nr < 2) raise(Err::invalid_argument, "lane " + std::to_string(lane.lane_id) + ": border too short");
        std::vector<double> rx(nr), ry(nr), rarc(nr, 0.0);
        for (size_t i = 0; i < nr; ++i) {
            rx[i] = double(lane.right_xy[2 * i]);
            ry[i] = double(lane.right_xy[2 * i + 1]);
        }
        for (size_t i = 1; i < nr; ++i) rarc[i] = rarc[i - 1] + norm2d(rx[i], ry[i], rx[i - 1], ry[i - 1]);
        size_t n = nl;
        bool pointwise = nr == n;
        std::vector<double> cx(n), cy(n), hw(n), s(n);
        for (size_t i = 0; i < n; ++i) {
            double lx = double(lane.left_xy[2 * i]), ly = double(lane.left_xy[2 * i + 1]);
            double px, py;
            if (pointwise) {
                px = rx[i];
                py = ry[i];
            } else {
                // Polyline::at_fraction (roads.cpp:30-38)
                double u = n > 1 ? double(i) / double(n - 1) : 0.0;
                double target = u * rarc[nr - 1];
                size_t k = 1;
                while (k + 1 < nr && rarc[k] < target) ++k;
                double seg = rarc[k] - rarc[k - 1];
                double t = seg > 0 ? (target - rarc[k - 1]) / seg : 0.0;
                t = clampd(t, 0.0, 1.0);
                px = rx[k - 1] + (rx[k] - rx[k - 1]) * t;
                py = ry[k - 1] + (ry[k] - ry[k - 1]) * t;
            }
            cx[i] = (lx + px) * 0.5;
            cy[i] = (ly + py) * 0.5;
            hw[i] = norm2d(lx, ly, px, py) * 0.5;
        }
        s[0] = double(lane.s_start);
        for (size_t i = 1; i < n; ++i) s[i] = s[i - 1] + norm2d(cx[i], cy[i], cx[i - 1], cy[i - 1]);

        LaneFrame lf;
        lf.lane_id = lane.lane_id;
        double clip_end = double(lane.s_end);
        for (size_t i = 0; i < n; ++i) {
            if (s[i] > clip_end && !lf.x.empty()) {
                double seg = s[i] - s[i - 1];
                if (seg > 0 && s[i - 1] < clip_end) {
                    double t = (clip_end - s[i - 1]) / seg;
                    lf.x.push_back(cx[i - 1] + (cx[i] - cx[i - 1]) * t);
                    lf.y.push_back(cy[i - 1] + (cy[i] - cy[i - 1]) * t);
                    lf.s.push_back(clip_end);
                    lf.hw.push_back(hw[i - 1] + (hw[i] - hw[i - 1]) * t);
                }
                break;
            }
            lf.x.push_back(cx[i]);
            lf.y.push_back(cy[i]);
            lf.s.push_back(s[i]);
            lf.hw.push_back(hw[i]);
        }
        if (lf.x.size() < 2) {
            raise(Err::invalid_argument,
                  "lane " + std::to_string(lane.lane_id) + ": valid interval clips away the centerline");
        }
        for (size_t i = 1; i < lf.s.size(); ++i) {
            if (!(lf.s[i] > lf.s[i - 1])) {
                raise(Err::invalid_argument,
                      "lane " + std::to_string(lane.lane_id) + ": centerline arc length not increasing");
            }
        }
        ctx.route_length = maxd(ctx.route_length, lf.s.back());
        ctx.lanes.push_back(std::move(lf));
    }
}

// roads::project (roads.cpp:125-166): per lane the first strictly smaller d2
// segment; across lanes the smallest |d|, then the lower lane_id.
Projection project_host(double px, double py, const RouteCtx& ctx) {
    if (ctx.lanes.empty()) raise(Err::invalid_argument, "project: empty route frame");
    bool have = false, in_corridor = false;
    LaneHit best{0.0, 0.0, 0.0};
    uint32_t best_id = 0;
    for (const auto& lf : ctx.lanes) {
        double bd2 = 1e300;
        int bi = -1;
        double bt = 0.0;
        for (size_t i = 0; i + 1 < lf.x.size(); ++i) {
            double t;
            double d2 = seg_dist2(px, py, lf.x[i], lf.y[i], lf.x[i + 1], lf.y[i + 1], &t);
            if (d2 < bd2) {
                bd2 = d2;
                bi = int(i);
                bt = t;
            }
        }
        if (bi < 0) continue;
        LaneHit h = lane_hit(px, py, lf.x.data(), lf.y.data(), lf.s.data(), lf.hw.data(), bi, bd2, bt);
        if (std::fabs(h.d) <= h.hw) in_corridor = true;
        if (!have || std::fabs(h.d) < std::fabs(best.d) || (std::fabs(h.d) == std::fabs(best.d) && lf.lane_id < best_id)) {
            best = h;
            best_id = lf.lane_id;
            have = true;
        }
    }
    Projection p;
    p.s = clampd(best.s, 0.0, ctx.route_length);
    p.d = best.d;
    p.lane_id = best_id;
    p.in_corridor = in_corridor;
    return p;
}

RouteCtx build_context(const Scene& sc) {
    RouteCtx ctx;
    build_frame(sc, ctx);
    for (size_t i = 0; i < sc.stops.size(); ++i) {
        Projection p = project_host(double(sc.stops[i].pos_x), double(sc.stops[i].pos_y), ctx);
        if (p.in_corridor) ctx.stops.emplace_back(int(i), p.s);
    }
    for (size_t i = 0; i < sc.lights.size(); ++i) {
        Projection p = project_host(double(sc.lights[i].stop_x), double(sc.lights[i].stop_y), ctx);
        if (p.in_corridor) ctx.lights.emplace_back(int(i), p.s);
    }
    return ctx;
}

std::vector<RoutePt> build_route_points(const Scene& sc) {
    std::vector<RoutePt> pts;
    for (const auto& lane : sc.lanes) {
        auto add = [&](const std::vector<float>& xy, uint8_t is_left) {
            double arc = double(lane.s_start);
            for (size_t i = 0; i + 1 < xy.size(); i += 2) {
                if (i >= 2) {
                    double dx = double(xy[i]) - double(xy[i - 2]);
                    double dy = double(xy[i + 1]) - double(xy[i - 1]);
                    arc += std::sqrt(dx * dx + dy * dy);
                }
                uint8_t valid = arc <= double(lane.s_end) + 0.5 ? 1 : 0;
                pts.push_back({xy[i], xy[i + 1], is_left, valid});
            }
        };
        add(lane.left_xy, 1);
        add(lane.right_xy, 0);
    }
    return pts;
}

bool actor_controllable(const Scene& s, int actor) {
    if (actor == 0) return true;
    if (actor < 0 || actor > int(s.agents.size())) return false;
    const AgentLog& a = s.agents[size_t(actor - 1)];
    if (a.valid.size() < s.num_steps) return false;
    for (uint32_t t = 0; t < s.num_steps; ++t)
        if (!a.valid[t]) return false;
    return true;
}

AgentLog ego_as_agent(const Scene& s, const EgoBoxDims& d) {
    AgentLog a;
    a.id = "ego";
    a.length = float(d.length);
    a.width = float(d.width);
    const size_t n = s.num_steps;
    a.x.resize(n), a.y.resize(n), a.heading.resize(n), a.speed.resize(n), a.valid.assign(n, 1);
    for (size_t t = 0; t < n; ++t) {
        const double h = double(s.ego_h[t]);
        // ego_box centre (simcore.cpp:156-160) of the logged pose
        a.x[t] = float(double(s.ego_x[t]) + std::cos(h) * d.center_offset);
        a.y[t] = float(double(s.ego_y[t]) + std::sin(h) * d.center_offset);
        a.heading[t] = s.ego_h[t];
        a.speed[t] = s.ego_v[t];
    }
    return a;
}

void actor_as_ego(const Scene& s, int actor, Scene& out) {
    out.num_steps = s.num_steps;
    out.dt = s.dt;
    if (actor == 0) {
        out.ego_x = s.ego_x, out.ego_y = s.ego_y, out.ego_h = s.ego_h, out.ego_v = s.ego_v;
        out.goal_x = s.goal_x, out.goal_y = s.goal_y;
        return;
    }
    const AgentLog& a = s.agents[size_t(actor - 1)];
    const size_t n = s.num_steps;
    out.ego_x.assign(a.x.begin(), a.x.begin() + long(n));
    out.ego_y.assign(a.y.begin(), a.y.begin() + long(n));
    out.ego_h.assign(a.heading.begin(), a.heading.begin() + long(n));
    out.ego_v.assign(a.speed.begin(), a.speed.begin() + long(n));
    const size_t last = n - 1;
    const double h = double(a.heading[last]);
    out.goal_x = float(double(a.x[last]) + 4.0 * std::cos(h));
    out.goal_y = float(double(a.y[last]) + 4.0 * std::sin(h));
}

Scene controlled_scene(const Scene& s, int actor, const EgoBoxDims& d) {
    if (!actor_controllable(s, actor)) raise(Err::invalid_argument, "actor " + std::to_string(actor) + " of `" + s.id +
                                                                          "` is not controllable");
    Scene c;
    c.id = s.id + "#" + std::to_string(actor);
    actor_as_ego(s, actor, c);
    if (actor != 0) c.agents.push_back(ego_as_agent(s, d));
    for (size_t k = 0; k < s.agents.size(); ++k)
        if (int(k) + 1 != actor) c.agents.push_back(s.agents[k]);
    c.lanes = s.lanes;
    c.features = s.features;
    c.lights = s.lights;
    c.stops = s.stops;
    c.speed_limit = s.speed_limit;
    return c;
}

double initial_steering(const Scene& sc, double wheelbase, double delta_max) {
    if (sc.num_steps < 2) return 0.0;
    double v0 = double(sc.ego_v[0]);
    if (v0 * sc.dt < 1e-4) return 0.0;
    double dtheta = wrap_angle(double(sc.ego_h[1]) - double(sc.ego_h[0]));
    double delta = std::atan(dtheta * wheelbase / (v0 * sc.dt));
    return clampd(delta, -delta_max, delta_max);
}

void check_bins(const std::vector<double>& bins, const char* name) {
    if (bins.empty()) raise(Err::invalid_argument, std::string(name) + ": empty bin list");
    bool has_zero = false;
    for (size_t i = 0; i < bins.size(); ++i) {
        if (bins[i] == 0.0) has_zero = true;
        if (i > 0 && bins[i] <= bins[i - 1]) {
            raise(Err::invalid_argument, std::string(name) + ": bins must be strictly increasing");
        }
        if (bins[i] != -bins[bins.size() - 1 - i]) {
            raise(Err::invalid_argument, std::string(name) + ": bins must be symmetric about 0");
        }
    }
    if (!has_zero) raise(Err::invalid_argument, std::string(name) + ": bins must contain 0");
}

int nearest_bin(const std::vector<double>& bins, double v) {
    int best = 0;
    double best_d = std::fabs(v - bins[0]);
    for (int i = 1; i < int(bins.size()); ++i) {
        double d = std::fabs(v - bins[size_t(i)]);
        if (d < best_d) {
            best = i;
            best_d = d;
        }
    }
    return best;
}

}  // namespace zs
