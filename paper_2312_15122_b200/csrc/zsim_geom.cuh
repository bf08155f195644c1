// zsim_geom.cuh -- fp64 route-frame / box geometry shared by the host staging
// code (g++ -ffp-contract=off) and the sm_100a kernels (nvcc -fmad=false).
//
// Every expression keeps the reference's association order so that results
// are bit-identical wherever the two sides use the same libm result (sqrt and
// fmod are exact on both; cos/sin/tan/atan differ by at most a few ulp on the
// device).  References are to /root/reference/proj/src/core/.
#pragma once

#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define ZS_HD __host__ __device__ __forceinline__
#define ZS_UNROLL _Pragma("unroll")
#else
#define ZS_HD inline
#define ZS_UNROLL
#endif

namespace zs {

constexpr double kTwoPi = 6.283185307179586476925286766559;
constexpr double kPi = 3.14159265358979323846;

// common.hpp:53-59
ZS_HD double wrap_angle(double a) {
    // fmod(a, 2pi) is a itself when |a| < 2pi (exact, sign kept): skip the
    // general remainder loop in that (usual) case
    if (!(fabs(a) < kTwoPi)) a = fmod(a, kTwoPi);
    if (a <= -kPi) a += kTwoPi;
    if (a > kPi) a -= kTwoPi;
    return a;
}

// std::clamp / std::min / std::max with libstdc++'s comparison direction.
ZS_HD double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }
ZS_HD double mind(double a, double b) { return b < a ? b : a; }
ZS_HD double maxd(double a, double b) { return a < b ? b : a; }

// geometry.cpp:17-25 (point_segment_dist2); t_out receives the clamped
// parameter of the closest point.
ZS_HD double seg_dist2(double px, double py, double ax, double ay, double bx, double by, double* t_out) {
    double abx = bx - ax, aby = by - ay;
    double len2 = abx * abx + aby * aby;
    double t = 0.0;
    if (len2 > 0.0) t = clampd(((px - ax) * abx + (py - ay) * aby) / len2, 0.0, 1.0);
    double qx = ax + abx * t, qy = ay + aby * t;
    *t_out = t;
    double ex = px - qx, ey = py - qy;
    return ex * ex + ey * ey;
}

ZS_HD double seg_dist2(double px, double py, double ax, double ay, double bx, double by) {
    double t;
    return seg_dist2(px, py, ax, ay, bx, by, &t);
}

// Oriented box with its heading's cosine / sine precomputed once (the
// reference recomputes them in Obb::corners and obb_overlap; same values).
struct Box {
    double cx, cy, hl, hw, c, s;
};

// geometry.cpp:7-15 (Obb::corners): (+ax+ay, +ax-ay, -ax-ay, -ax+ay).
ZS_HD void box_corners(const Box& b, double* X, double* Y) {
    double axx = b.c * b.hl, axy = b.s * b.hl;
    double ayx = -b.s * b.hw, ayy = b.c * b.hw;
    X[0] = b.cx + axx + ayx;
    Y[0] = b.cy + axy + ayy;
    X[1] = b.cx + axx - ayx;
    Y[1] = b.cy + axy - ayy;
    X[2] = b.cx - axx - ayx;
    Y[2] = b.cy - axy - ayy;
    X[3] = b.cx - axx + ayx;
    Y[3] = b.cy - axy + ayy;
}

// geometry.cpp:48-61 (separated_on_axis) over one axis.
ZS_HD bool sat_separated(double ux, double uy, const double* AX, const double* AY, const double* BX,
                         const double* BY) {
    double amin = 1e300, amax = -1e300, bmin = 1e300, bmax = -1e300;
ZS_UNROLL
    for (int k = 0; k < 4; ++k) {
        double v = AX[k] * ux + AY[k] * uy;
        amin = mind(amin, v);
        amax = maxd(amax, v);
    }
ZS_UNROLL
    for (int k = 0; k < 4; ++k) {
        double v = BX[k] * ux + BY[k] * uy;
        bmin = mind(bmin, v);
        bmax = maxd(bmax, v);
    }
    return amax < bmin || bmax < amin;
}

// geometry.cpp:65-75 (obb_overlap): touching counts as overlap.
ZS_HD bool boxes_overlap(const Box& a, const double* AX, const double* AY, const Box& b, const double* BX,
                         const double* BY) {
    if (sat_separated(a.c, a.s, AX, AY, BX, BY)) return false;
    if (sat_separated(-a.s, a.c, AX, AY, BX, BY)) return false;
    if (sat_separated(b.c, b.s, AX, AY, BX, BY)) return false;
    if (sat_separated(-b.s, b.c, AX, AY, BX, BY)) return false;
    return true;
}

// geometry.cpp:27-42 (segment_segment_distance) returned SQUARED: 0 on a strict
// proper crossing, else the min of the four endpoint-to-segment d2.  sqrt is
// monotone and correctly rounded, so sqrt(min d2) == min(sqrt d2).
ZS_HD double segseg_dist2(double a0x, double a0y, double a1x, double a1y, double b0x, double b0y, double b1x,
                          double b1y) {
    double o1 = (a1x - a0x) * (b0y - a0y) - (a1y - a0y) * (b0x - a0x);
    double o2 = (a1x - a0x) * (b1y - a0y) - (a1y - a0y) * (b1x - a0x);
    double o3 = (b1x - b0x) * (a0y - b0y) - (b1y - b0y) * (a0x - b0x);
    double o4 = (b1x - b0x) * (a1y - b0y) - (b1y - b0y) * (a1x - b0x);
    if (((o1 > 0) != (o2 > 0)) && ((o3 > 0) != (o4 > 0))) return 0.0;
    double d2 = seg_dist2(a0x, a0y, b0x, b0y, b1x, b1y);
    d2 = mind(d2, seg_dist2(a1x, a1y, b0x, b0y, b1x, b1y));
    d2 = mind(d2, seg_dist2(b0x, b0y, a0x, a0y, a1x, a1y));
    d2 = mind(d2, seg_dist2(b1x, b1y, a0x, a0y, a1x, a1y));
    return d2;
}

// geometry.cpp:77-88 (obb_distance) for one edge pair (i of a, j of b),
// squared.  The caller takes the min over the 16 pairs and one sqrt.
ZS_HD double box_edge_pair_dist2(const double* AX, const double* AY, const double* BX, const double* BY, int i,
                                 int j) {
    int i1 = (i + 1) & 3, j1 = (j + 1) & 3;
    return segseg_dist2(AX[i], AY[i], AX[i1], AY[i1], BX[j], BY[j], BX[j1], BY[j1]);
}

// Per-lane candidate of roads.cpp:125-143 (project_to_lane) for the winning
// segment i with parameter t: s, signed d and interpolated half-width.
struct LaneHit {
    double s, d, hw;
};

ZS_HD LaneHit lane_hit(double px, double py, const double* cx, const double* cy, const double* cs,
                       const double* chw, int i, double d2, double t) {
    double ax = cx[i], ay = cy[i];
    double tx = cx[i + 1] - ax, ty = cy[i + 1] - ay;
    double qx = ax + tx * t, qy = ay + ty * t;
    double rx = px - qx, ry = py - qy;
    double sign = (tx * ry - ty * rx) >= 0.0 ? 1.0 : -1.0;
    LaneHit h;
    h.s = cs[i] + (cs[i + 1] - cs[i]) * t;
    h.d = sign * sqrt(d2);
    h.hw = chw[i] + (chw[i + 1] - chw[i]) * t;
    return h;
}

// splitmix64 (common.hpp:28-51) in closed form for Env::init_state's
// `Rng(seed).split(i).state` (simcore.cpp:251,261): the parent stream has
// advanced i+1 times when row i is split.
ZS_HD uint64_t splitmix_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

ZS_HD uint64_t reset_rng_state(uint64_t seed, uint64_t row) {
    const uint64_t g = 0x9e3779b97f4a7c15ull;
    uint64_t parent0 = seed + g;
    uint64_t z = parent0 + (row + 1) * g;
    uint64_t mixed = splitmix_mix(z) ^ (row * 0xd1342543de82ef95ull + 0x2545f4914f6cdd1dull);
    return mixed + g;
}

}  // namespace zs
