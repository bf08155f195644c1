// zsim_pack.cuh -- HBM layout of the immutable per-batch scenario pack and the
// device-side SimConfig.  One contiguous allocation, every array 256-B
// aligned, padded to per-batch capacities with per-scenario counts.
//
// Per scenario (reference types in /root/reference/proj/src/core/); the
// row-level arrays (initial ego, goal, stop-flag offset) are per row:
//   agents  [B][T][A]  x, y, heading, speed f32 + valid u8   (LoggedAgent, scenario.hpp:37-44)
//   dims    [B][A]     length, width f32
//   road    [B][P]     float2 xy + u8 kind|dir<<4 + i32 index in nearest_features'
//                      flat (feature, point) order (roads.cpp:220-229), stored in
//                      Morton order as 32-point chunks with bounding boxes [B][PC]
//   route   [B][R]     float2 xy + u8 is_left|lane_valid<<1 + i32 index in
//                      build_route_points order (simcore.cpp:181-200), chunked likewise
//   lanes   [B][L][C]  centerline records {x, y, b-a, |b-a|^2, s, half_width} f64
//                      after RouteFrame::build clipping (roads.cpp:43-103);
//                      an fp32 copy (a - origin, b - a) for screening;
//                      n vertices + lane_id per lane
//   lights  [B][NL]    route s f64 + state u8[T] for lights kept by
//                      RouteContext::build (roads.cpp:245-249)
//   stops   [B][NS]    route s f64 for stop lines kept by RouteContext::build
//   scalars [B]        counts, goal, goal_s, route_length, initial ego (+ steering
//                      recovered on the host, simcore.cpp:620-627)
#pragma once

#include <stdint.h>

#include "../../include/zsim_gpu.h"

namespace zs {

struct PackDims {
    int32_t B, T, A, P, R, L, C, NL, NS;
    int32_t S;       // scenarios (B rows index them through row_scen; S == B in ego mode)
    int32_t PC, RC;  // 32-point chunks of the road / route point sets
    int32_t GC;      // 8-segment groups per lane centreline
};

constexpr int kSegGroup = 8;  // segments per centreline group (bounding box)

constexpr int kChunk = 32;  // points per spatial chunk (one warp-wide load)

// One centreline vertex with its outgoing segment (i -> i+1), 64 B: an exact
// projection and its lane_hit touch only this record.  The differences
// follow the reference's expressions: ab = b - a (geometry.cpp:18), s and
// half-width increments (roads.cpp:130-139); unused on the last vertex.
// Per route lane: vertex count, lane_id (the projection tie-break,
// roads.cpp:147-166) and the (min, max) centreline half-width rounded outward.
struct __align__(16) LaneInfo {
    int32_t n;
    uint32_t id;
    float hw_min, hw_max;
};

struct __align__(16) LaneVtx {
    double x, y, abx, aby, s, ds, hw, dhw;
};

struct DevPack {
    PackDims d;
    double dt;
    int32_t horizon;
    int32_t total_stop_lines;
    // [B]
    const int32_t* num_steps;
    const int32_t* n_agents;
    const int32_t* n_road;
    const int32_t* n_route;
    const int32_t* n_lanes;
    const int32_t* n_lights;
    const int32_t* n_stops;
    const int32_t* stop_off;
    const float* speed_limit;
    const float* goal_x;
    const float* goal_y;
    const double* goal_s;
    const double* route_len;
    const double* init_x;
    const double* init_y;
    const double* init_h;
    const double* init_v;
    const double* init_steer;
    // agents
    const float* ag_x;
    const float* ag_y;
    const float* ag_h;
    const float* ag_sp;
    const uint8_t* ag_valid;
    const float* ag_len;
    const float* ag_wid;
    const double2* ag_cs;  // [S][T][A] (cos, sin) of the logged heading, host libm as the reference (geometry.cpp:8)
    // road / route points
    // point sets in spatial (Morton) order, 32-point chunks with bounding boxes;
    // *_oi is each point's index in the reference order (the tie-break key)
    const float2* road_xy;
    const uint8_t* road_kd;
    const int32_t* road_oi;
    const float4* road_cb;   // [B][PC] chunk boxes (min x, min y, max x, max y)
    const float2* route_xy;
    const uint8_t* route_fl;
    const int32_t* route_oi;
    const float4* route_cb;  // [B][RC]
    // lanes
    const LaneVtx* ln_v;    // [B][L][C] exact centreline records
    const float4* ln_f4;    // [B][L][C] fp32 screening copy: (a - origin, b - a) per segment
    const float4* ln_gb;    // [B][L][GC] group boxes (origin-relative, rounded outward)
    const double2* ln_org;  // [B] origin of the fp32 copy
    const float* ln_fe;     // [B] max |a - origin|_1 over vertices + max segment length (error scale)
    const LaneInfo* ln_info;  // [B][L] vertex count, lane_id, half-width bounds
    const float4* road_box;   // [B] (min x, min y, max x, max y) of the road points
    const float4* route_box;  // [B] same for the route border points
    // rows -> scenario data (null in ego mode: identity / no skipped actor)
    const int32_t* row_scen;   // [B] scenario of the row
    const int32_t* row_actor;  // [B] controlled actor (its agent column is skipped)
    // lights / stops
    const double* lt_s;
    const uint8_t* lt_state;  // [B][NL][T]
    const double* st_s;
};

// SimConfig + ActionTable as the kernels see them.
struct DevCfg {
    double wheelbase, ego_length, ego_width, ego_center_offset, delta_max, v_min;
    double goal_radius, footprint_margin, stop_cross_speed, stop_zone, stop_slow_speed;
    double w_progress, w_speed, w_lat, w_lon, terminal_penalty, feature_radius;
    int32_t disable_dones, n_agents, n_road, n_route;
    int32_t n_accel, n_steer;
    double accel_bins[16];
    double steer_bins[16];
};

}  // namespace zs
