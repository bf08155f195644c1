// zsim_scenario.hpp -- host-side scenario model, ZSIM container codec and the
// per-batch staging (route frame, route context, route border points) that the
// reference performs in Env::Env.  Host C++ only.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

struct zsim_stress_config;  // include/zsim_gpu.h

namespace zs {

// zsim::ErrorKind (common.hpp:13) + the C-ABI's CUDA code.
enum class Err : int { invalid_argument = 1, config = 2, io = 3, runtime = 4, cuda = 5 };

struct Error : std::runtime_error {
    Err kind;
    Error(Err k, const std::string& m) : std::runtime_error(m), kind(k) {}
};

[[noreturn]] inline void raise(Err k, const std::string& m) { throw Error(k, m); }

// Scenario (scenario.hpp:27-90).
struct AgentLog {
    std::string id;
    float length = 0.f, width = 0.f;
    std::vector<float> x, y, heading, speed;
    std::vector<uint8_t> valid;
};
struct LaneBorders {
    uint32_t lane_id = 0;
    std::vector<float> left_xy, right_xy;
    float s_start = 0.f, s_end = 0.f;
};
struct Feature {
    uint8_t kind = 0, dir = 0;
    std::vector<float> xy;
};
struct Light {
    uint32_t signal_id = 0;
    float stop_x = 0.f, stop_y = 0.f;
    std::vector<uint8_t> state;
};
struct StopLine {
    std::vector<float> xy;
    float pos_x = 0.f, pos_y = 0.f;
};
struct Scene {
    std::string id;
    uint32_t num_steps = 0;
    double dt = 0.1;
    std::vector<float> ego_x, ego_y, ego_h, ego_v;
    std::vector<AgentLog> agents;
    std::vector<LaneBorders> lanes;
    std::vector<Feature> features;
    std::vector<Light> lights;
    std::vector<StopLine> stops;
    float speed_limit = 0.f, goal_x = 0.f, goal_y = 0.f;
};

// ZSIM container (scenario.hpp:97-104, scenario_io.cpp:80-189, 319-394).
struct ZsimIndex {
    double dt = 0.0;
    std::vector<std::pair<uint64_t, uint32_t>> records;  // (offset of body, length)
};
ZsimIndex zsim_index(const uint8_t* buf, size_t n);
Scene zsim_decode(const uint8_t* buf, size_t n, const ZsimIndex& idx, int64_t record);
void zsim_encode_append(std::string& out, const Scene& s);
std::string zsim_header(double dt);

// One lane of the route frame after clipping (roads.hpp:15-20).
struct LaneFrame {
    uint32_t lane_id = 0;
    std::vector<double> x, y, s, hw;
};
struct RouteCtx {
    std::vector<LaneFrame> lanes;
    double route_length = 0.0;
    std::vector<std::pair<int, double>> stops;   // (index into Scene::stops, s)
    std::vector<std::pair<int, double>> lights;  // (index into Scene::lights, s)
};

struct Projection {
    double s = 0.0, d = 0.0;
    uint32_t lane_id = 0;
    bool in_corridor = false;
};

// RouteFrame::build (roads.cpp:43-103).
void build_frame(const Scene& sc, RouteCtx& ctx);
// roads::project (roads.cpp:147-166).
Projection project_host(double px, double py, const RouteCtx& ctx);
// RouteContext::build (roads.cpp:238-251).
RouteCtx build_context(const Scene& sc);

struct RoutePt {
    float x, y;
    uint8_t is_left, lane_valid;
};
// build_route_points (simcore.cpp:181-200).
std::vector<RoutePt> build_route_points(const Scene& sc);

// recover_initial_steering (simcore.cpp:620-627).
double initial_steering(const Scene& sc, double wheelbase, double delta_max);

// ---------------------------------------------------------------------------
// "All agents controlled" (no reference code).  Actors
// of a scenario: actor 0 = the logged ego, actor k = agents[k-1].  The row of
// actor j is exactly a reference Env row over controlled_scene(s, j): the ego
// log is actor j's log (heading/speed as logged), the goal lies 4 m past its
// last logged point along its last heading, and the other actors log-replay in
// actor order.  The logged ego, when it is not the controlled actor, is an
// agent whose box is the SimConfig ego box (centre ego_center_offset ahead of
// its logged point).  An agent is controllable when it is valid at every
// logged step.  Roadgraph, route corridor, lights and stop lines are shared.
// ---------------------------------------------------------------------------
struct EgoBoxDims {
    double length, width, center_offset;
};
inline int num_actors(const Scene& s) { return 1 + int(s.agents.size()); }
bool actor_controllable(const Scene& s, int actor);
AgentLog ego_as_agent(const Scene& s, const EgoBoxDims& d);
// ego log + goal of actor `actor` written into `out` (num_steps/dt copied)
void actor_as_ego(const Scene& s, int actor, Scene& out);
Scene controlled_scene(const Scene& s, int actor, const EgoBoxDims& d);

// ActionTable::validated / nearest_bin (dynamics.cpp:30-64).
void check_bins(const std::vector<double>& bins, const char* name);
int nearest_bin(const std::vector<double>& bins, double v);

// synthetic stress scenarios (zsim_stressgen.cpp)
void stress_check(const zsim_stress_config& cfg);
Scene stress_scene(const zsim_stress_config& cfg, uint64_t seed, int64_t global_index);

}  // namespace zs
