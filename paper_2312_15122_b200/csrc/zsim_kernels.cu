// zsim_kernels.cu -- sm_100a kernels for the batched simulator step.
//
// Execution model: ONE WARP PER SCENARIO ROW.  A CTA holds 14 (or 4)
// warps that walk scenario rows in a grid-stride loop, one block barrier per
// row (the warps stay in phase and share the instruction cache); inside a row
// a warp never waits on another.  Per row, in one launch:
//
//   step     bicycle_step -> route projection of the ego and of the four
//            inflated footprint corners (lane-of-route x segment across the 32
//            lanes, per-query argmin by (d2, segment) with REDUX) -> collision
//            SAT against the agents valid at t+1 (one agent per lane) ->
//            lights, stop lines, goal, done priority, reward
//            (roads.cpp:125-208, simcore.cpp:278-404)
//   observe  active/value features; agent boxes reused from the collision
//            test when fused; obb_distance only for agents whose distance
//            bounds can reach the top n_agents; road / route top-k
//            (simcore.cpp:423-538)
//
// Top-k (road 128-of-P within 100 m, route 64-of-R): one pass computes fp32
// squared distances and a 32-bucket pseudo-log histogram (lane-private smem
// counters, bank-conflict-free) which yields a threshold with >= k points
// under it; a second pass compacts, with ballots, the points that can make
// the cut (fp32 error bound included); only those get exact fp64 keys, and a
// counting sort on the exact keys (+ rank inside a bucket) emits the
// reference's exact (d2, index) order.
//
// Every translation unit on the path builds with -fmad=false: each fp64
// expression rounds like the reference compiled with -ffp-contract=off.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <mutex>
#include <vector>

#include "zsim_geom.cuh"
#include "zsim_kernels.cuh"
#include "zsim_pack.cuh"

namespace zs {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int NQ = 5;     // projection queries per step: ego position + 4 inflated corners
constexpr int NB2 = 256;  // counting-sort buckets over the exact keys
// independent point loads in flight per lane in the key passes: 4 in the
// register-bound fused kernel (C1 -1.2% against 8), 8 in the split map
// kernel (C4 shard: 4 is +1.4%)
constexpr int kUnrollFused = 4, kUnrollMap = 8;  // (fused 2 / 3: +2.3% / 0; map 6 / 12: +0.7% / +0.2%)
constexpr int kAgSlots = 32;  // agent corner slots (one 32-agent chunk), the stride of the corner-major layout

// Diagnostic path counters, compiled only into the ZS_PATHSTATS variant
// (build.py --pathstats); the product library has none of this code.
#ifdef ZS_PATHSTATS
__device__ unsigned long long g_pstats[32];
#define PSTAT(i, v)                                                          \
    do {                                                                     \
        if ((threadIdx.x & 31) == 0) atomicAdd(&g_pstats[(i)], (unsigned long long)(v)); \
    } while (0)
// per-row SM clock stamps (low 32 bits) at marks 0..7; the host differences them
constexpr int kMaxStatRows = 65536;
__device__ unsigned g_rowcyc[kMaxStatRows][24];
__device__ __forceinline__ void row_mark(int b, int k) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0 && b < kMaxStatRows) g_rowcyc[b][k] = unsigned(clock64());
}
#define ROW_MARK(b, k) row_mark((b), (k))
#else
#define PSTAT(i, v) \
    do {            \
    } while (0)
#define ROW_MARK(b, k) \
    do {               \
    } while (0)
#endif

// Bounds-checked build (build.py --variant=checked -DZS_CHECKED): device
// asserts on the scratch and point-set indices -- the stand-in for
// compute-sanitizer, which this GPU pool does not run.
#ifdef ZS_CHECKED
#define ZS_CHECK(cond)                                                                                      \
    do {                                                                                                    \
        if (!(cond)) {                                                                                      \
            printf("zsim check failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond,         \
                   int(blockIdx.x), int(threadIdx.x));                                                      \
            __trap();                                                                                       \
        }                                                                                                   \
    } while (0)
#else
#define ZS_CHECK(cond) \
    do {               \
    } while (0)
#endif

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
// Observation stores: written once and read later by the host or a policy;
// st.global.cs (evict-first) keeps them from pushing the scenario data the
// rest of the step re-reads out of L2 (measured: C1 fused step -2.5%).
template <class T>
__device__ __forceinline__ void obs_st(T* p, T v) { __stcs(p, v); }

__device__ __forceinline__ int warp_in_block() { return threadIdx.x >> 5; }
// The warp index read through a lane-0 shuffle: provably warp-uniform to the
// compiler, so the row index and the shared-memory carve-up derived from it
// can use the uniform datapath.  Measured per kernel: the split C2 kernels
// -7.5%, the fused step+observe +0.8% (C1) / +4% (C4 shard) -- so only the
// split kernels use it.
__device__ __forceinline__ int warp_in_block_uniform() { return __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0); }
// A row scalar re-read through a lane-0 shuffle so the compiler knows it is
// warp-uniform (the row's scenario, agent column, time and stop count):
// C1 -0.9%; the same for the per-scenario counts (lanes, agents, points) was
// +0.6%.
__device__ __forceinline__ int uni(int x) { return __shfl_sync(0xffffffffu, x, 0); }
__device__ __forceinline__ unsigned lanemask_lt() { return (1u << lane_id()) - 1u; }

// fp64 libm routines of the ego dynamics, inlined (measured against one
// out-of-line copy each: C1 -1.2%, C4 shard -0.9%, fewer spills around the calls).
__device__ __forceinline__ double2 sincos2(double x) {
    double s, c;
    sincos(x, &s, &c);
    return make_double2(s, c);
}
__device__ __forceinline__ double tan1(double x) { return tan(x); }
__device__ __forceinline__ double wrap1(double a) { return wrap_angle(a); }

// Lexicographic warp argmin by (d2, idx) for d2 >= 0 (or +inf): the bit
// pattern of a non-negative double is monotone, so three 32-bit REDUX ops.
__device__ __forceinline__ void warp_argmin(double d2, int idx, double& out_d2, int& out_idx) {
    unsigned hi = unsigned(__double2hiint(d2)), lo = unsigned(__double2loint(d2));
    unsigned mhi = __reduce_min_sync(FULL, hi);
    unsigned mlo = __reduce_min_sync(FULL, hi == mhi ? lo : 0xffffffffu);
    bool eq = hi == mhi && lo == mlo;
    unsigned mi = __reduce_min_sync(FULL, eq ? unsigned(idx) : 0xffffffffu);
    out_d2 = __hiloint2double(int(mhi), int(mlo));
    out_idx = int(mi);
}

template <class T>
__device__ __forceinline__ T pick5(int k, T a0, T a1, T a2, T a3, T a4) {
    return k == 0 ? a0 : k == 1 ? a1 : k == 2 ? a2 : k == 3 ? a3 : a4;
}

__device__ __forceinline__ int scen_of(const DevPack& pk, int b) { return pk.row_scen ? pk.row_scen[b] : b; }
__device__ __forceinline__ int skip_of(const DevPack& pk, int b) { return pk.row_actor ? pk.row_actor[b] : -1; }

// Row state, uniform across the warp.
struct Row {
    double x, y, h, v, steer, proj_s, proj_d;
    unsigned long long rng;
    int t, done, reason, events, in_corr;
};

// Warp-uniform row state lives in shared memory, not in 32 copies of
// registers: the step reads r0 and writes r / the ego box, observe reads them.
struct RowSh {
    Row r0;                // pre-step state as loaded
    Row r;                 // post-step state (what observe sees)
    Box eb;                // ego box of r
    double ex[4], ey[4];   // its corners (obb_distance reads them lane-indexed)
    double qx[5], qy[5];   // projection queries (position + inflated corners)
    float4 hint;           // the row's top-k hint, loaded at row start
    int sc;                // scenario of the row (== row in ego mode)
    int skip;              // agent column of the controlled actor (-1 in ego mode)
    double a_lat;          // step: v^2 tan(steer) / wheelbase (simcore.cpp:309-316)
    int boxes_ready;       // agent boxes at r.t + overlap flags are in agx/agy/agf
};

// Per-warp shared-memory carve-up (host mirror: smem_bytes()).
struct WarpBuf {
    RowSh* rs;
    double* agx;           // [4][32] agent corners, corner-major: corner k of slot j at k * 32 + j
    double* agy;           //   (lane-per-agent reads are then consecutive: no bank conflicts)
    double* agd;           // [A] bbox distance
    int* agf;              // [A] -1 invalid, 0 separate, 1 overlap
    unsigned short* hist;  // [32*32] lane-private u16 histogram; reused as counting-sort counts u32[NB2]
    uint16_t* cidx;        // [cap] candidate positions (16-bit: point sets hold < 65536 points)
    double* ckey;          // [cap] exact keys
    uint16_t* cinfo;       // [cap] candidates' reference indices (the tie-break key)
    uint16_t* order;       // [max(cap, chunks)] chunk list, then candidates grouped by bucket, then the selection
    int* sel;              // [Ka] selected agents (road/route selections land in `order`)
    int* alist;            // [A] bound keys, then the agents that survive the bound test (beyond 32 agents)
    unsigned char* sflag;  // [NS] pre-step stopped flags
};

__host__ __device__ inline size_t al16(size_t v) { return (v + 15) / 16 * 16; }

// Per-warp layout: [RowSh][union: agent phase | top-k phase][stop flags].
// The agent buffers (boxes at t+1 from the step, distances, selection) are
// dead once the agent features are written, before the road/route top-k, so
// both phases share one region.
inline SmemLayout warp_layout(int A, int cap, int ka, int ns, int nch) {
    SmemLayout L;
    size_t o = al16(sizeof(RowSh));  // warp-uniform row state
    const size_t u0 = o;
    auto put = [&](uint32_t& f, size_t bytes) { f = uint32_t(o), o += al16(bytes); };
    // corner slots: one 32-agent chunk, corner-major with stride kAgSlots
    put(L.agx, size_t(A > 0 ? kAgSlots : 0) * 4 * 8);
    put(L.agy, size_t(A > 0 ? kAgSlots : 0) * 4 * 8);
    put(L.agd, size_t(A) * 8);
    put(L.agf, size_t(A) * 4);
    put(L.sel, size_t(ka) * 4);
    put(L.alist, size_t(A) * 4);
    const size_t agents_end = o;
    o = u0;
    put(L.hist, cap > 0 ? 32 * 32 * 2 : 0);  // no top-k buffers in the step-only kernel (cap = 0)
    put(L.cidx, size_t(cap) * 2);
    put(L.ckey, size_t(cap) * 8);
    put(L.cinfo, size_t(cap) * 2);
    // also the top-k's chunk list: up to nch chunks (P > 32 * cap points)
    put(L.order, size_t(cap > 0 ? (cap > nch ? cap : nch) : 0) * 2);
    o = o > agents_end ? o : agents_end;
    put(L.sflag, size_t(ns) + 1);
    L.total = uint32_t(al16(o));
    return L;
}

__device__ __forceinline__ WarpBuf carve(unsigned char* base, const KernelArgs& a, int warp) {
    const SmemLayout& L = a.lay;
    unsigned char* p = base + L.total * unsigned(warp);
    WarpBuf w;
    w.rs = reinterpret_cast<RowSh*>(p);
    w.agx = reinterpret_cast<double*>(p + L.agx);
    w.agy = reinterpret_cast<double*>(p + L.agy);
    w.agd = reinterpret_cast<double*>(p + L.agd);
    w.agf = reinterpret_cast<int*>(p + L.agf);
    w.sel = reinterpret_cast<int*>(p + L.sel);
    w.alist = reinterpret_cast<int*>(p + L.alist);
    w.hist = reinterpret_cast<unsigned short*>(p + L.hist);
    w.cidx = reinterpret_cast<uint16_t*>(p + L.cidx);
    w.ckey = reinterpret_cast<double*>(p + L.ckey);
    w.cinfo = reinterpret_cast<uint16_t*>(p + L.cinfo);
    w.order = reinterpret_cast<uint16_t*>(p + L.order);
    w.sflag = p + L.sflag;
    return w;
}

__device__ __forceinline__ Row load_row(const zsim_state_view& in, int b) {
    Row r;
    r.x = in.x[b];
    r.y = in.y[b];
    r.h = in.heading[b];
    r.v = in.v[b];
    r.steer = in.steering[b];
    r.t = in.t[b];
    r.done = in.done[b];
    r.reason = in.reason[b];
    r.rng = in.rng[b];
    r.proj_s = in.proj_s[b];
    r.proj_d = in.proj_d[b];
    r.in_corr = in.proj_in_corridor[b];
    r.events = in.events[b];
    return r;
}

__device__ __forceinline__ void store_row(const zsim_state_view& out, int b, const Row& r) {
    out.x[b] = r.x;
    out.y[b] = r.y;
    out.heading[b] = r.h;
    out.v[b] = r.v;
    out.steering[b] = r.steer;
    out.t[b] = r.t;
    out.done[b] = uint8_t(r.done);
    out.reason[b] = uint8_t(r.reason);
    out.rng[b] = r.rng;
    out.proj_s[b] = r.proj_s;
    out.proj_d[b] = r.proj_d;
    out.proj_in_corridor[b] = uint8_t(r.in_corr);
    out.events[b] = uint8_t(r.events);
}

// point_segment_dist2 (geometry.cpp:17-25) with ab / len2 precomputed on the
// host by the same expressions.  When the clamp decides t (dot <= 0 or
// dot >= len2) the division is skipped: clamp(dot/len2, 0, 1) is then exactly
// 0 (up to the sign of a zero, which changes no result) or exactly 1.
__device__ __forceinline__ double seg_d2_pre(double px, double py, double ax, double ay, double abx, double aby,
                                             double len2, double& t_out) {
    double t = 0.0;
    if (len2 > 0.0) {
        double dot = (px - ax) * abx + (py - ay) * aby;
        if (dot >= len2)
            t = 1.0;
        else if (dot > 0.0)
            t = dot / len2;
    }
    double qx = ax + abx * t, qy = ay + aby * t;
    double ex = px - qx, ey = py - qy;
    t_out = t;
    return ex * ex + ey * ey;
}

// point_segment_dist2 (geometry.cpp:17-25) through seg_d2_pre: identical d2,
// division only for an interior projection.
__device__ __forceinline__ double seg_dist2_fast(double px, double py, double ax, double ay, double bx, double by) {
    const double abx = bx - ax, aby = by - ay;
    double t;
    return seg_d2_pre(px, py, ax, ay, abx, aby, abx * abx + aby * aby, t);
}

struct Proj {
    double s, d;
    int in_corr;   // query 0 lies in some lane corridor (roads.cpp:154)
    int on_route;  // all four inflated corners lie in some corridor (roads.cpp:192-208)
};

// Lexicographic (d2, idx) min within aligned groups of 8 lanes.
__device__ __forceinline__ void seg8_argmin(double& d2, int& idx) {
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) {
        const double od = __shfl_xor_sync(FULL, d2, off);
        const int oi = __shfl_xor_sync(FULL, idx, off);
        if (od < d2 || (od == d2 && oi < idx)) {
            d2 = od;
            idx = oi;
        }
    }
}

// Directed fp32 square roots for bounds: sqrt.approx (relative error < 2^-22)
// scaled by 2^-20 away from the true root, so the result is a certain upper
// (lower) bound -- the IEEE sqrtf sequence and its slow-path branch are not
// needed where only a bound is consumed.
__device__ __forceinline__ float sqrt_up(float x) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r * (1.f + 0x1p-20f);
}
__device__ __forceinline__ float sqrt_dn(float x) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r * (1.f - 0x1p-20f);
}

__device__ __forceinline__ float octet_minf(float v) {
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) v = fminf(v, __shfl_xor_sync(FULL, v, off));
    return v;
}

// fp32 screening distance^2 from (qx, qy) (origin-relative) to segment f =
// (a - origin, b - a); inv ~ 1/|b-a|^2 (0 for a degenerate segment).
__device__ __forceinline__ float seg_d2_f(float qx, float qy, float4 f, float inv) {
    const float dx = qx - f.x, dy = qy - f.y;
    float t = __fmul_rn(__fmaf_rn(dx, f.z, __fmul_rn(dy, f.w)), inv);
    t = fminf(fmaxf(t, 0.f), 1.f);
    const float ex = __fmaf_rn(-f.z, t, dx), ey = __fmaf_rn(-f.w, t, dy);
    return __fmaf_rn(ex, ex, __fmul_rn(ey, ey));
}

__device__ __forceinline__ float seg_inv_f(float4 f) {
    const float l2 = __fmaf_rn(f.z, f.z, __fmul_rn(f.w, f.w));
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(l2));  // <= 1 ulp: inside the screening bound
    return l2 > 1e-30f ? r : 0.f;
}

// roads::project for NQU queries (q0 = the point; q1..4 = footprint corners
// when NQU == 5): per route lane the first strictly smaller d2 segment
// (roads.cpp:125-143), across lanes min |d| then lane_id (roads.cpp:147-166).
//
// Blocks of 4 route lanes map onto the warp's 4 octets; lane gg of an octet
// owns segments gg, gg+8, ...  Screening is fp32 on an origin-relative copy
// (ln_f4).  Error bound: the copy moves every segment point by <= 2^-24
// (|a-o|_1 + |b-a|_1) and a query by <= 2^-24 |q-o|_1; the fp32 arithmetic
// (approximate t, clamped, so the evaluated point stays on the segment) adds
// <= 2^-20 (d + |b-a|); so |d_f32 - d_exact| <= delta = 2^-18 (fe + |q-o|_1 + d)
// with fe = ln_fe.
//  0. 8-segment group boxes give every query's "needed" groups: the corners
//     lie within R of q0, so (triangle inequality) the exact minimiser of any
//     query lies among the segments with d0 <= sqrt(m0) + 2R + 4 delta, all
//     inside groups whose box lower bound is within the far-corner bound
//     + 2R + 8 delta.
//  1. fp32 distances of every query to the needed segments: each query's
//     minimum m_q (one pass for all five queries).
//  2. Needed segments with d_q <= sqrt(m_q) + 2 delta (every segment that can
//     tie the exact minimum) are evaluated in fp64 with the reference's
//     expressions; the exact lexicographic (d2, segment) minimum per octet is
//     the reference's argmin.
// The winners' s / signed d / half-width run one (query, route lane) pair per
// lane.  Uniform result.
template <int NQU>
__device__ Proj warp_project(const DevPack& pk, int b /* scenario */, const double* qx, const double* qy) {
    const int L = pk.d.L, C = pk.d.C;
    const int nl = pk.n_lanes[b];
    const int lane = lane_id();
    const int gl = lane >> 3, gg = lane & 7;
    PSTAT(22, 1);
    const double2 org = pk.ln_org[b];
    const float fe = pk.ln_fe[b];
    const double route_len = pk.route_len[b];
    float qxf[NQU], qyf[NQU];
#pragma unroll
    for (int q = 0; q < NQU; ++q) {
        qxf[q] = float(qx[q] - org.x);
        qyf[q] = float(qy[q] - org.y);
    }
    float R = 0.f;  // max distance of a corner from q0
#pragma unroll
    for (int q = 1; q < NQU; ++q) {
        const float dx = qxf[q] - qxf[0], dy = qyf[q] - qyf[0];
        R = fmaxf(R, sqrt_up(dx * dx + dy * dy));
    }
    R = R * (1.f + 0x1p-16f) + 1e-6f;
    // lanes (q, k) = (lane >> 2, lane & 3) run the lane_hit of query q on route lane l0 + k
    const int hq = lane >> 2, hk = lane & 3;
    const double hpx = hq < NQU ? qx[NQU == 1 ? 0 : hq] : 0.0, hpy = hq < NQU ? qy[NQU == 1 ? 0 : hq] : 0.0;
    bool have = false;
    double best_abs = 0.0, best_s = 0.0, best_d = 0.0;
    uint32_t best_id = 0;
    unsigned in_bits = 0;
#pragma unroll 1
    for (int l0 = 0; l0 < nl; l0 += 4) {
        const int l = l0 + gl;
        const bool lane_ok = l < nl;
        const size_t lrow = size_t(b) * L + (lane_ok ? l : 0);
        const size_t base = lrow * C;
        const LaneInfo li = lane_ok ? pk.ln_info[lrow] : LaneInfo{1, 0u, 0.f, 0.f};
        const int nseg = li.n - 1;
        const float4* F = pk.ln_f4 + base;
        // ---- 0. 8-segment groups that can hold q0's minimum or a near segment ----
        // Group boxes (origin-relative, rounded outward) bound the exact
        // distance of every segment inside from below (LB) and above (far
        // corner, FD); d_f32 is within delta of exact, so m0 <= U = min FD + delta
        // and only groups with LB <= U + 2R + 5 delta can matter.
        const int ngr = (nseg + kSegGroup - 1) / kSegGroup;
        unsigned long long need = 0;  // bit g: group g is scanned (octet-uniform)
        {
            float lbv[2], fdmin = INFINITY;
            const int GC = pk.d.GC;
            // the group boxes are loaded without waiting for the lane's group
            // count (one memory round trip instead of two); g < GC keeps the
            // loads inside the lane's slots
            float4 gbv[2];
#pragma unroll
            for (int c = 0; c < 2; ++c)
                gbv[c] = gg + 8 * c < GC ? pk.ln_gb[lrow * GC + gg + 8 * c] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int c = 0; c < 2; ++c) {  // groups gg and gg + 8 (lanes up to 129 vertices)
                const int g = gg + 8 * c;
                lbv[c] = INFINITY;
                if (g < ngr) {
                    const float4 bb = gbv[c];
                    const float x0 = bb.x - qxf[0], x1 = qxf[0] - bb.z, y0 = bb.y - qyf[0], y1 = qyf[0] - bb.w;
                    const float nx = fmaxf(fmaxf(x0, x1), 0.f), ny = fmaxf(fmaxf(y0, y1), 0.f);
                    const float fx = fmaxf(fabsf(x0), fabsf(x1)), fy = fmaxf(fabsf(y0), fabsf(y1));
                    lbv[c] = sqrt_dn(nx * nx + ny * ny);
                    fdmin = fminf(fdmin, sqrt_up(fx * fx + fy * fy));
                }
            }
            fdmin = octet_minf(fdmin);
            const float dl = 0x1p-18f * (fe + fabsf(qxf[0]) + fabsf(qyf[0]) + fdmin + 4.f * R) + 1e-6f;
            const float lim = (fdmin + 2.f * R + 8.f * dl) * (1.f + 0x1p-20f);
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const unsigned bal = __ballot_sync(FULL, lbv[c] <= lim);
                need |= (unsigned long long)((bal >> (8 * gl)) & 0xFFu) << (8 * c);
            }
            if (ngr > 16) need |= ~0ull << 16;  // longer lanes: groups past 16 always scanned
        }
        if (l0 == 0) ROW_MARK(b, 10);
        // ---- 1+2. every query over the needed groups: the exact minimiser of
        // each query lies among the segments near q0, all inside the needed
        // groups, and the farther ones never reach a query's minimum ----
        float m[NQU];
#pragma unroll
        for (int q = 0; q < NQU; ++q) m[q] = INFINITY;
        // two groups per iteration, both segments' loads in flight (the
        // minimum is order-free; measured C1 -1.1%, C4 shard -1.6%)
        for (unsigned long long mm = need & ((ngr >= 64) ? ~0ull : ((1ull << ngr) - 1)); mm;) {
            const int s0 = (__ffsll(mm) - 1) * kSegGroup + gg;
            mm &= mm - 1;
            const int s1 = mm ? (__ffsll(mm) - 1) * kSegGroup + gg : nseg;
            mm &= mm - 1;
            const float4 f0 = s0 < nseg ? F[s0] : make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 f1 = s1 < nseg ? F[s1] : make_float4(0.f, 0.f, 0.f, 0.f);
            if (s0 < nseg) {
                const float inv = seg_inv_f(f0);
#pragma unroll
                for (int q = 0; q < NQU; ++q) m[q] = fminf(m[q], seg_d2_f(qxf[q], qyf[q], f0, inv));
            }
            if (s1 < nseg) {
                const float inv = seg_inv_f(f1);
#pragma unroll
                for (int q = 0; q < NQU; ++q) m[q] = fminf(m[q], seg_d2_f(qxf[q], qyf[q], f1, inv));
            }
        }
#pragma unroll 1
        for (int si = 64 * kSegGroup + gg; si < nseg; si += 8) {  // beyond the 64-bit group mask
            const float4 f = F[si];
            const float inv = seg_inv_f(f);
#pragma unroll
            for (int q = 0; q < NQU; ++q) m[q] = fminf(m[q], seg_d2_f(qxf[q], qyf[q], f, inv));
        }
        m[0] = octet_minf(m[0]);
        if (l0 == 0) ROW_MARK(b, 11);
        // A corner only needs its in-corridor bit (roads.cpp:202-208): when its
        // fp32 distance to this route lane is below the lane's smallest
        // half-width (or above the largest) by more than delta, the verdict is
        // certain and no exact evaluation is needed for it.
        const float2 hwb = make_float2(li.hw_min, li.hw_max);
        unsigned cin = 0;  // octet-uniform bit q: corner q certainly inside this lane's corridor
        unsigned cunc = 0;  // bit q: corner q needs the exact argmin in this lane
        float thr[NQU];
#pragma unroll
        for (int q = 0; q < NQU; ++q) {
            const float mm = q == 0 ? m[0] : octet_minf(m[q]);
            const float dm = sqrt_up(mm), dml = sqrt_dn(mm);
            const float delta = 0x1p-18f * (fe + fabsf(qxf[q]) + fabsf(qyf[q]) + dm) + 1e-30f;
            const float r = dm + 2.f * delta;
            thr[q] = r * r * (1.f + 0x1p-20f);
            if (q > 0) {
                const bool in = dm + delta < hwb.x;
                const bool out = dml - delta > hwb.y;
                cin |= in ? 1u << q : 0u;
                if (in || out)
                    thr[q] = -1.f;
                else
                    cunc |= 1u << q;
            }
        }
        if (l0 == 0) ROW_MARK(b, 12);
        // ---- 3. exact fp64 distances of the candidates ----
        double bd[NQU];
        int bi[NQU];
#pragma unroll
        for (int q = 0; q < NQU; ++q) bd[q] = 1e300, bi[q] = INT_MAX;
        auto exact = [&](int si, const float4 f) {
            const float inv = seg_inv_f(f);
            unsigned cm = 0;
#pragma unroll
            for (int q = 0; q < NQU; ++q) cm |= seg_d2_f(qxf[q], qyf[q], f, inv) <= thr[q] ? 1u << q : 0u;
            if (cm) {
                const double2* V = reinterpret_cast<const double2*>(pk.ln_v + base + si);
                const double2 v0 = V[0], v1 = V[1];
                const double ax = v0.x, ay = v0.y, abx = v1.x, aby = v1.y, l2 = abx * abx + aby * aby;
#pragma unroll
                for (int q = 0; q < NQU; ++q) {
                    if (cm & (1u << q)) {
                        double t;
                        const double d2 = seg_d2_pre(qx[q], qy[q], ax, ay, abx, aby, l2, t);
                        PSTAT(21, 1);
                        if (d2 < bd[q] || (d2 == bd[q] && si < bi[q])) bd[q] = d2, bi[q] = si;
                    }
                }
            }
        };
        // the thresholds select the candidates: a segment far from every
        // query's minimum passes none
        for (unsigned long long mm = need & ((ngr >= 64) ? ~0ull : ((1ull << ngr) - 1)); mm; mm &= mm - 1) {
            const int si = (__ffsll(mm) - 1) * kSegGroup + gg;
            if (si < nseg) exact(si, F[si]);
        }
#pragma unroll 1
        for (int si = 64 * kSegGroup + gg; si < nseg; si += 8) exact(si, F[si]);  // beyond the 64-bit group mask

        if (l0 == 0) ROW_MARK(b, 13);
        // ---- per-octet exact argmin, then s / signed d / half-width per (query, route lane) ----
        int hi_ = INT_MAX;
        // corners whose corridor verdict is certain in every route lane need no argmin
        const unsigned open_q = __reduce_or_sync(FULL, cunc);
#pragma unroll
        for (int q = 0; q < NQU; ++q) {
            if (q > 0 && !((open_q >> q) & 1u)) continue;
            seg8_argmin(bd[q], bi[q]);
            const int v = __shfl_sync(FULL, bi[q], hk * 8);
            if (hq == q) hi_ = v;
        }
        if (l0 == 0) ROW_MARK(b, 14);
        const unsigned cin_k = __shfl_sync(FULL, cin, hk * 8);
        bool ok = hq > 0 && hq < NQU && ((cin_k >> hq) & 1u);
        double hs = 0.0, hd = 0.0;
        if (!ok && hq < NQU && l0 + hk < nl && hi_ != INT_MAX) {
            ZS_CHECK(hi_ >= 0 && hi_ < C - 1);
            const double2* V = reinterpret_cast<const double2*>(pk.ln_v + (size_t(b) * L + l0 + hk) * C + hi_);
            const double2 a0 = V[0], a1 = V[1], a2 = V[2], a3 = V[3];
            double t;
            const double d2 = seg_d2_pre(hpx, hpy, a0.x, a0.y, a1.x, a1.y, a1.x * a1.x + a1.y * a1.y, t);
            // lane_hit (roads.cpp:130-139) with b - a, s and half-width increments from the record
            const double qx_ = a0.x + a1.x * t, qy_ = a0.y + a1.y * t;
            const double rx = hpx - qx_, ry = hpy - qy_;
            const double sign = (a1.x * ry - a1.y * rx) >= 0.0 ? 1.0 : -1.0;
            LaneHit h;
            h.s = a2.x + a2.y * t;
            h.d = sign * sqrt(d2);
            h.hw = a3.x + a3.y * t;
            hs = h.s;
            hd = h.d;
            ok = fabs(h.d) <= h.hw;
        }
        const unsigned okb = __ballot_sync(FULL, ok);
        if (l0 == 0) ROW_MARK(b, 15);
#pragma unroll
        for (int q = 0; q < NQU; ++q)
            if ((okb >> (4 * q)) & 15u) in_bits |= 1u << q;
        // query 0: across route lanes min |d| then lane_id (lanes 0..3 hold route
        // lanes l0..l0+3): REDUX argmin on (|d| bits, lane_id), |d| >= 0
        {
            const uint32_t my_id = __shfl_sync(FULL, li.id, (lane & 3) * 8);
            const bool cand = lane < 4 && l0 + lane < nl && hi_ != INT_MAX;
            const double key = cand ? fabs(hd) : INFINITY;
            const unsigned khi = unsigned(__double2hiint(key)), klo = unsigned(__double2loint(key));
            const unsigned mhi = __reduce_min_sync(FULL, khi);
            const unsigned mlo = __reduce_min_sync(FULL, khi == mhi ? klo : 0xffffffffu);
            const bool eq = cand && khi == mhi && klo == mlo;
            const unsigned mid = __reduce_min_sync(FULL, eq ? my_id : 0xffffffffu);
            const unsigned wl = __ballot_sync(FULL, eq && my_id == mid);
            if (wl) {
                const int src = __ffs(wl) - 1;
                const double babs = __hiloint2double(int(mhi), int(mlo));
                const double s0 = __shfl_sync(FULL, hs, src), d0 = __shfl_sync(FULL, hd, src);
                if (!have || babs < best_abs || (babs == best_abs && mid < best_id)) {
                    have = true;
                    best_abs = babs;
                    best_s = s0;
                    best_d = d0;
                    best_id = mid;
                }
            }
        }
    }
    Proj p;
    p.s = clampd(best_s, 0.0, route_len);
    p.d = best_d;
    p.in_corr = int(in_bits & 1u);
    p.on_route = NQU == 5 ? int((in_bits & 0x1Eu) == 0x1Eu) : 1;
    return p;
}

// One logged agent at a slice, every field loaded at once (validity included):
// one memory round trip instead of a validity load, then the position, then
// (after the distance branch) the heading and size.
struct AgRaw {
    float x, y, len, wid;
    double2 cs;
    int valid;
};
__device__ __forceinline__ AgRaw load_ag(const DevPack& pk, int sc, size_t slice, int j) {
    AgRaw r;
    r.valid = pk.ag_valid[slice + j];
    r.x = pk.ag_x[slice + j];
    r.y = pk.ag_y[slice + j];
    r.cs = pk.ag_cs[slice + j];
    r.len = pk.ag_len[size_t(sc) * pk.d.A + j];
    r.wid = pk.ag_wid[size_t(sc) * pk.d.A + j];
    return r;
}

// Agent box at log slice `slice` (agent_box, simcore.cpp:162-165): corners
// into smem and the SAT overlap with the ego box (geometry.cpp:65-75).
__device__ __forceinline__ int agent_box_overlap_raw(const AgRaw& g, int j, const Box& eb, const double* EX,
                                                     const double* EY, const WarpBuf& w, bool keep_corners) {
    Box ab;
    ab.cx = double(g.x);
    ab.cy = double(g.y);
    ab.hl = double(g.len) * 0.5;
    ab.hw = double(g.wid) * 0.5;
    ab.c = g.cs.x;  // host libm cos / sin of the heading, as the reference
    ab.s = g.cs.y;
    double X[4], Y[4];
    box_corners(ab, X, Y);
    if (keep_corners) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            w.agx[k * kAgSlots + (j & 31)] = X[k];
            w.agy[k * kAgSlots + (j & 31)] = Y[k];
        }
    }
    return boxes_overlap(eb, EX, EY, ab, X, Y) ? 1 : 0;
}
__device__ __forceinline__ int agent_box_overlap(const DevPack& pk, int sc, size_t slice, int j, const Box& eb,
                                                 const double* EX, const double* EY, const WarpBuf& w,
                                                 bool keep_corners = true) {
    const int A = pk.d.A;
    Box ab;
    ab.cx = double(pk.ag_x[slice + j]);
    ab.cy = double(pk.ag_y[slice + j]);
    ab.hl = double(pk.ag_len[size_t(sc) * A + j]) * 0.5;
    ab.hw = double(pk.ag_wid[size_t(sc) * A + j]) * 0.5;
    const double2 cs = pk.ag_cs[slice + j];  // host libm cos / sin of the heading, as the reference
    ab.c = cs.x;
    ab.s = cs.y;
    double X[4], Y[4];
    box_corners(ab, X, Y);
    // corner slots hold one 32-agent chunk (lane = j mod 32); beyond 32 agents
    // the observation recomputes each chunk's corners (agent_corners)
    if (keep_corners) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            ZS_CHECK(j >= 0 && j < A);
            w.agx[k * kAgSlots + (j & 31)] = X[k];
            w.agy[k * kAgSlots + (j & 31)] = Y[k];
        }
    }
    return boxes_overlap(eb, EX, EY, ab, X, Y) ? 1 : 0;
}
// Corners of agent j at log slice `slice` (agent_box, simcore.cpp:162-165)
// into its chunk slot, without the overlap test.
__device__ __forceinline__ void agent_corners(const DevPack& pk, int sc, size_t slice, int j, int slot, double* agx,
                                              double* agy) {
    const int A = pk.d.A;
    Box ab;
    ab.cx = double(pk.ag_x[slice + j]);
    ab.cy = double(pk.ag_y[slice + j]);
    ab.hl = double(pk.ag_len[size_t(sc) * A + j]) * 0.5;
    ab.hw = double(pk.ag_wid[size_t(sc) * A + j]) * 0.5;
    const double2 cs = pk.ag_cs[slice + j];
    ab.c = cs.x;
    ab.s = cs.y;
    double X[4], Y[4];
    box_corners(ab, X, Y);
    ZS_CHECK(slot >= 0 && slot < kAgSlots && j >= 0 && j < A);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        agx[k * kAgSlots + slot] = X[k];
        agy[k * kAgSlots + slot] = Y[k];
    }
}


// Bounds on obb_distance (geometry.cpp:77-88) between the ego box and agent
// j at log slice `slice`, in fp32 with margins (1e-4 + 1e-5 D) far above its
// rounding.  Along the centre line u (centre distance D) the supports
// r(u) = hl |u.e1| + hw |u.e2| give lo = D - r_e(u) - r_a(u) <= distance (the
// separation along u; lo > 0 also proves the boxes apart), and the
// centre-line points still inside each box (reach t(u) = min(hl / |u.e1|,
// hw / |u.e2|)) give distance <= hi = max(0, D - t_e(u) - t_a(u)).  The
// quotients are approximate: hi only matters when D > te + ta, where the
// 1e-5 D margin covers their 2-ulp error.
__device__ __forceinline__ void agent_bounds(const AgRaw& g, const Box& eb, float& lo, float& hi) {
    const float dx = float(double(g.x) - eb.cx), dy = float(double(g.y) - eb.cy);
    const float D = sqrt_up(dx * dx + dy * dy);  // the 1e-5 D margins cover sqrt.approx
    const float m = 1e-4f + 1e-5f * D;
    if (!(D > 1e-3f)) {
        lo = -m, hi = m + 1e-3f;
        return;
    }
    float id;
    asm("rcp.approx.f32 %0, %1;" : "=f"(id) : "f"(D));
    const float ux = dx * id, uy = dy * id;
    const float ec = float(eb.c), es = float(eb.s), ehl = float(eb.hl), ehw = float(eb.hw);
    const float ac = float(g.cs.x), as = float(g.cs.y);
    const float ahl = g.len * 0.5f, ahw = g.wid * 0.5f;
    const float e1 = fabsf(ux * ec + uy * es), e2 = fabsf(uy * ec - ux * es);
    const float a1 = fabsf(ux * ac + uy * as), a2 = fabsf(uy * ac - ux * as);
    const float te = fminf(e1 > 0.f ? __fdividef(ehl, e1) : INFINITY, e2 > 0.f ? __fdividef(ehw, e2) : INFINITY);
    const float ta = fminf(a1 > 0.f ? __fdividef(ahl, a1) : INFINITY, a2 > 0.f ? __fdividef(ahw, a2) : INFINITY);
    lo = D - (ehl * e1 + ehw * e2) - (ahl * a1 + ahw * a2) - m;
    hi = fmaxf(0.f, D - te - ta) + m;
}

// One agent of the pruned pass (beyond 32 agents): fp32 distance bounds
// (lower bound into agd, upper-bound key into alist: 0 for an overlap) and
// the SAT only when the lower bound cannot prove the boxes apart.
// Agent boxes at one slice + overlap flags into w.agx/agy/agf for a row
// (-1 = invalid / skipped / t past the log); returns whether any overlaps.
// (Inlined: a __noinline__ call forces the WarpBuf into local memory.)
//
// Beyond 32 agents the corners are not kept (the observation recomputes them
// per chunk) and the distance bounds of the observation's pruning are computed
// here, in the same pass over the agents: fp32 lower bound into agd,
// upper-bound key into alist (0 for an overlap, ~0u for an invalid agent).  A
// positive lower bound proves the boxes apart; the agents it cannot decide are
// queued (in the free corner slots) and get the exact fp64 SAT afterwards, one
// per lane -- a few per row, instead of one divergent SAT pass per 32-agent
// chunk.
template <int AGB>
__device__ __forceinline__ bool agent_boxes(const DevPack& pk, int sc, size_t slice, int na, int skip, bool t_ok, const Box& eb,
                                             const double* EX, const double* EY, const WarpBuf& w) {
    bool hit = false;
    const int lane = lane_id();
    if (na <= 32) {
        for (int j = lane; j < na; j += 32) {
            int f = -1;
            const AgRaw g = load_ag(pk, sc, slice, j);
            if (t_ok && j != skip && g.valid) f = agent_box_overlap_raw(g, j, eb, EX, EY, w, true);
            w.agf[j] = f;
            hit |= f == 1;
        }
        return hit;
    }
    int* pend = reinterpret_cast<int*>(w.agy);  // 4 * kAgSlots doubles = room for 256 agent columns
    int npend = 0;
    // AGB 32-agent chunks per pass, every field loaded up front (two for the
    // ego kernels: C4 shard -1.8%; one for the 64-register controlled-row
    // kernel, where two spill: C2 +4.3%)
    for (int j00 = 0; j00 < na; j00 += 32 * AGB) {
        AgRaw g[AGB];
#pragma unroll
        for (int u = 0; u < AGB; ++u) {
            const int j = j00 + 32 * u + lane;
            g[u] = load_ag(pk, sc, slice, j < na ? j : 0);
        }
#pragma unroll
        for (int u = 0; u < AGB; ++u) {
            const int j0 = j00 + 32 * u;
            if (j0 >= na) break;
            const int j = j0 + lane;
            int f = -1;
            unsigned key = 0xFFFFFFFFu;
            bool sat = false;
            if (j < na && t_ok && j != skip && g[u].valid) {
                float lo, hi;
                agent_bounds(g[u], eb, lo, hi);
                w.agd[j] = double(lo);
                f = 0;
                key = __float_as_uint(hi);
                sat = !(lo > 0.f);
            }
            const unsigned bal = __ballot_sync(FULL, sat);
            if (sat) {
                const int q = npend + __popc(bal & lanemask_lt());
                if (q < 2 * 4 * kAgSlots) pend[q] = j;
            }
            npend += __popc(bal);
            if (j < na) {
                w.agf[j] = f;
                w.alist[j] = int(key);
            }
        }
    }
    __syncwarp();
    if (npend > 2 * 4 * kAgSlots) {
        // more undecided agents than queue slots (more than 256 agents): decide in place
        for (int j = lane; j < na; j += 32)
            if (w.agf[j] == 0 && !(w.agd[j] > 0.0) && agent_box_overlap(pk, sc, slice, j, eb, EX, EY, w, false)) {
                w.agf[j] = 1;
                w.alist[j] = 0;
                hit = true;
            }
        return hit;
    }
    for (int k = lane; k < npend; k += 32) {
        const int j = pend[k];
        ZS_CHECK(j >= 0 && j < na);
        if (agent_box_overlap(pk, sc, slice, j, eb, EX, EY, w, false)) {
            w.agf[j] = 1;
            w.alist[j] = 0;  // an overlap's distance is 0: the smallest key
            hit = true;
        }
    }
    __syncwarp();
    return hit;
}

// geometry.cpp:77-88 in full over the 16 edge pairs (contact case, rare).
// (box_edge_pair_dist2 for every pair; the agent's corners corner-major, stride kAgSlots)
__device__ __forceinline__ double contact_dist2(const double* GX, const double* GY, const double* AX, const double* AY) {
    double d2min = INFINITY;
#pragma unroll 1
    for (int pr = 0; pr < 16; ++pr) {
        const int i = pr >> 2, j = pr & 3, i1 = (i + 1) & 3, j1 = (j + 1) & 3;
        d2min = fmin(d2min, segseg_dist2(GX[i], GY[i], GX[i1], GY[i1], AX[kAgSlots * j], AY[kAgSlots * j],
                                         AX[kAgSlots * j1], AY[kAgSlots * j1]));
    }
    return d2min;
}

// Upper bound on |fp32 key - fp64 key| for points within sqrt(T)+1 of the
// query; `ep` is the fp32 rounding error of the query coordinates.
// An upper bound on sqrt(x), x >= 0: fp32 sqrt.approx (relative error < 2^-22)
// of x rounded up, scaled up by 2^-20 -- for bounds, where the fp64 sqrt's
// exactness buys nothing and its multi-instruction sequence sits on the
// critical path.
__device__ __forceinline__ double ub_sqrt(double x) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(__double2float_ru(x)));
    return double(r) * (1.0 + 0x1p-20);
}

__device__ __forceinline__ double key_margin(double T, double ep) {
    double D = ub_sqrt(T) + 1.0;
    double eta = ep + 0x1p-24 * (D + ep);
    double m = 2.0 * eta * (2.0 * D + eta);
    m += 0x1p-22 * (T + m) + 0x1p-50 * T;
    return m * 1.25 + 1e-30;
}

__device__ __forceinline__ float approx_key(float2 p, float pxf, float pyf) {
    float dx = p.x - pxf, dy = p.y - pyf;
    return __fmaf_rn(dx, dx, __fmul_rn(dy, dy));
}

// Squared distance from (px, py) to the farthest corner of a point set's
// bounding box: an upper bound on every key of the set.
__device__ __forceinline__ double box_far_d2(float4 bb, double px, double py) {
    double dx = fmax(fabs(double(bb.x) - px), fabs(double(bb.z) - px));
    double dy = fmax(fabs(double(bb.y) - py), fabs(double(bb.w) - py));
    return dx * dx + dy * dy;
}

// Counting-sort bucket b's counter slot: lane L owns buckets 8L..8L+7 in the
// scan, so bucket 8L+k sits at k*32 + L (the scan's accesses are then
// bank-conflict-free; a [L][k] layout is an 8-way conflict).
__device__ __forceinline__ int bslot(int b) { return ((b & 7) << 5) | (b >> 3); }
static_assert(NB2 == 256, "bslot assumes 256 buckets (8 per lane)");

// Warp-wide bucket counts: lane k returns bucket k's count; clears the histogram.
__device__ __forceinline__ unsigned hist_reduce(unsigned short* hist) {
    const int lane = lane_id();
    unsigned mine = 0;
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
        unsigned v = hist[k * 32 + lane];
        hist[k * 32 + lane] = 0;  // u16 lane-private counters
        unsigned s = __reduce_add_sync(FULL, v);
        if (lane == k) mine = s;
    }
    return mine;
}

__device__ __forceinline__ unsigned warp_incl_scan(unsigned v) {
    const int lane = lane_id();
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        unsigned o = __shfl_up_sync(FULL, v, off);
        if (lane >= off) v += o;
    }
    return v;
}

// k-th smallest (1-based) of the keys' top 16 bits over key[0..n) across the
// warp, as key bits (low 16 zero): two 8-bit radix-select passes over a
// 256-bin shared histogram (`hist`: 256 u32 of scratch, bin d at
// (d & 7) * 32 + d / 8 so each lane's 8 consecutive digits are conflict-free).
// The same result as a bitwise MSB-first select over the 16 bits.  Uniform.
__device__ __forceinline__ unsigned warp_kth_key(const int* key, int n, int k, unsigned* hist) {
    const int lane = lane_id();
    unsigned prefix = 0;
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
        const int shift = 24 - 8 * pass;
        for (int i = lane; i < 256; i += 32) hist[i] = 0u;
        __syncwarp();
        for (int j = lane; j < n; j += 32) {
            const unsigned u = unsigned(key[j]);
            if (pass == 0 || (u >> 24) == (prefix >> 24)) {
                const unsigned d = (u >> shift) & 0xFFu;
                atomicAdd(&hist[((d & 7u) << 5) | (d >> 3)], 1u);
            }
        }
        __syncwarp();
        unsigned v[8], sum = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            v[q] = hist[q * 32 + lane];  // digit 8 * lane + q
            sum += v[q];
        }
        const unsigned incl = warp_incl_scan(sum);
        const int owner = __ffs(__ballot_sync(FULL, incl >= unsigned(k))) - 1;
        ZS_CHECK(owner >= 0);
        int dsel = 0;
        unsigned below = 0;
        if (lane == owner) {
            unsigned run = incl - sum;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (run + v[q] >= unsigned(k)) {
                    dsel = 8 * lane + q;
                    below = run;
                    break;
                }
                run += v[q];
            }
        }
        dsel = __shfl_sync(FULL, dsel, owner);
        below = __shfl_sync(FULL, below, owner);
        k -= int(below);
        prefix |= unsigned(dsel) << shift;
        __syncwarp();
    }
    return prefix;
}

// A point set in chunked spatial order (zsim_pack.cuh).
struct PointSet {
    const float2* xy;
    const int32_t* oi;  // index in the reference order (tie-break key)
    const float4* cb;   // chunk bounding boxes
    int n, nch;
};

// Squared distances from (px, py) to a chunk box: a lower bound (nearest
// point of the box) and an upper bound (farthest corner) on the exact fp64
// key of every point inside, with slack for rounding.
__device__ __forceinline__ void chunk_bounds(float4 bb, double px, double py, double& lo, double& hi) {
    double x0 = double(bb.x) - px, x1 = double(bb.z) - px, y0 = double(bb.y) - py, y1 = double(bb.w) - py;
    double nx = x0 > 0.0 ? x0 : (x1 < 0.0 ? -x1 : 0.0);
    double ny = y0 > 0.0 ? y0 : (y1 < 0.0 ? -y1 : 0.0);
    double fx = fmax(fabs(x0), fabs(x1)), fy = fmax(fabs(y0), fabs(y1));
    lo = (nx * nx + ny * ny) * (1.0 - 1e-12);
    hi = (fx * fx + fy * fy) * (1.0 + 1e-12) + 1e-300;
}

// One warp pass over the listed chunks (32 points each, one per lane), loads
// batched for memory-level parallelism; calls f(position, approx_key, point)
// for every existing point.
template <int KU, class F>
__device__ __forceinline__ void over_chunks(const PointSet& ps, const uint16_t* list, int nlist, float pxf, float pyf,
                                            F&& f) {
    const int lane = lane_id();
    for (int j0 = 0; j0 < nlist; j0 += KU) {
        float2 pb[KU];
        int pos[KU];
#pragma unroll
        for (int u = 0; u < KU; ++u) {
            pos[u] = -1;
            pb[u] = make_float2(INFINITY, INFINITY);
            if (j0 + u < nlist) {
                const int p = list[j0 + u] * kChunk + lane;
                ZS_CHECK(list[j0 + u] >= 0 && list[j0 + u] < ps.nch);
                if (p < ps.n) {
                    pos[u] = p;
                    pb[u] = ps.xy[p];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < KU; ++u) {
            if (j0 + u < nlist) f(pos[u], approx_key(pb[u], pxf, pyf), pb[u]);
        }
    }
}

// ---------------------------------------------------------------------------
// Warp top-k by (exact fp64 d2, reference index) over a chunked point set.
// With use_r only points with exact d2 <= r2 qualify (roads.cpp:219-229).
// Writes the selected POSITIONS (into ps.xy) in order to order[0..ret).
//
//  1. Upper bound T on the k-th exact key: the per-row hint (previous k-th key
//     + displacement, triangle inequality) and/or the smallest chunk far-corner
//     distance that covers >= k points.
//  2. Only chunks whose nearest box point can hold a key <= T are read; their
//     points with fp32 key <= T + margin are compacted (ballot).
//  3. If that overflows the candidate capacity, a pseudo-log histogram over
//     the same chunks tightens T (then a linear one, then an exact iterative
//     fallback).
//  4. Exact fp64 keys for the candidates, counting sort + in-bucket rank by
//     (key, reference index).
// ---------------------------------------------------------------------------
template <int KU>
__device__ __noinline__ int warp_topk(PointSet ps, int K, double px, double py, bool use_r, double r2, float4 bbox,
                                      int cap, unsigned short* __restrict__ hist, uint16_t* __restrict__ cidx,
                                      double* __restrict__ ckey, uint16_t* __restrict__ cinfo,
                                      uint16_t* __restrict__ order,
                                      float4 hv, float4* hint, int which) {
    const int lane = lane_id();
    const int n = ps.n;
    ZS_CHECK(K <= NB2 && n <= ps.nch * kChunk);
    if (n <= 0) return 0;
    const float pxf = float(px), pyf = float(py);
    const double ep = fmax(fabs(double(pxf) - px), fabs(double(pyf) - py));
    double hi_d = box_far_d2(bbox, px, py);
    hi_d += key_margin(hi_d, ep);
    if (use_r) hi_d = fmin(hi_d, r2 + key_margin(r2, ep));
    const float hi = __double2float_ru(hi_d);

    // ---- 1. upper bound on the k-th exact key ----
    double T = INFINITY;
    if (hint != nullptr) {
        const float4 h = hv;  // loaded at row start (the road call writes only .z, the route call reads .w/.x/.y)
        const float kth = which == 0 ? h.z : h.w;
        if (isfinite(h.x) && isfinite(h.y) && kth >= 0.f && isfinite(kth)) {
            const double ddx = px - double(h.x), ddy = py - double(h.y);
            const double dp = ub_sqrt(ddx * ddx + ddy * ddy) + 1e-3 + 1e-6 * (fabs(px) + fabs(py));
            const double rr = ub_sqrt(double(kth)) + dp;
            T = rr * rr * (1.0 + 1e-9);
        }
    }
    PSTAT(1 + 8 * which, T < INFINITY ? 1 : 0);
    if (!(T < INFINITY) && ps.nch <= cap) {
        // smallest far bound covering >= K points: chunk far bounds staged in
        // ckey (free until the candidates), extracted in increasing order
        for (int c = lane; c < ps.nch; c += 32) {
            double lo_b, hi_b;
            chunk_bounds(ps.cb[c], px, py, lo_b, hi_b);
            ckey[c] = hi_b;
        }
        __syncwarp();
        int acc = 0;
        for (int it = 0; it < ps.nch && acc < K; ++it) {
            double mloc = INFINITY;
            int mi = INT_MAX;
            for (int c = lane; c < ps.nch; c += 32)
                if (ckey[c] < mloc) mloc = ckey[c], mi = c;
            double md;
            int mc;
            warp_argmin(mloc, mi, md, mc);
            if (mc == INT_MAX || !(md < INFINITY)) break;
            if (lane == 0) ckey[mc] = INFINITY;
            __syncwarp();
            acc += min(kChunk, n - mc * kChunk);
            if (acc >= K) T = md;
        }
        PSTAT(2 + 8 * which, T < INFINITY ? 1 : 0);
    }
    PSTAT(3 + 8 * which, T < INFINITY ? 0 : 1);
    if (use_r && T < INFINITY && !(T <= r2)) T = INFINITY;  // the k points might not all qualify
    float tc = T < INFINITY ? fminf(__double2float_ru(T + key_margin(T, ep)), hi) : hi;

    // ---- 2. needed chunks + candidate compaction ----
    uint16_t* list = order;  // chunk list (order is free until the final sort)
    int nlist = 0;
    // two 32-chunk groups per pass: both groups' box loads in flight
    // together (measured: C4 shard -2%, C1 -0.6%; four groups spill, C1 +10%)
    auto build_list = [&](float t) {
        nlist = 0;
        const double lim = double(t) + key_margin(double(t), ep);
        for (int c0 = 0; c0 < ps.nch; c0 += 32 * 2) {
            float4 bx[2];
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                const int c = c0 + 32 * g + lane;
                bx[g] = c < ps.nch ? ps.cb[c] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                const int c = c0 + 32 * g + lane;
                double lo_b = 0.0, hi_b = INFINITY;
                if (c < ps.nch) chunk_bounds(bx[g], px, py, lo_b, hi_b);
                const bool need = c < ps.nch && lo_b <= lim;
                const unsigned bal = __ballot_sync(FULL, need);
                if (need) list[nlist + __popc(bal & lanemask_lt())] = c;
                nlist += __popc(bal);
            }
        }
        ZS_CHECK(nlist <= ps.nch);
        __syncwarp();
    };
    auto compact_chunks = [&](float t) {
        int C = 0;
        over_chunks<KU>(ps, list, nlist, pxf, pyf, [&](int pos, float a, float2 p) {
            const bool take = pos >= 0 && a <= t;
            const unsigned bal = __ballot_sync(FULL, take);
            if (take) {
                const int q = C + __popc(bal & lanemask_lt());
                if (q < cap) {
                    cidx[q] = pos;
                    reinterpret_cast<float2*>(ckey)[q] = p;  // staged point; its exact key replaces it
                }
            }
            C += __popc(bal);
        });
        __syncwarp();
        return C;
    };
    build_list(tc);
    int C = compact_chunks(tc);
    PSTAT(7 + 8 * which, C);
    PSTAT(8 + 8 * which, nlist);

    // ---- 3. tighten the bound when the candidates overflow ----
    if (C > cap) {
        PSTAT(4 + 8 * which, 1);
        const int top = int(__float_as_uint(tc) >> 22);
        const int base = max(top - 31, 0);
        over_chunks<KU>(ps, list, nlist, pxf, pyf, [&](int pos, float a, float2) {
            if (pos >= 0 && a <= tc) hist[min(31, max(0, int(__float_as_uint(a) >> 22) - base)) * 32 + lane] += 1;
        });
        __syncwarp();
        unsigned cnt = hist_reduce(hist);
        unsigned incl = warp_incl_scan(cnt);
        const unsigned total = __shfl_sync(FULL, incl, 31);
        if (total > unsigned(K)) {
            const int kstar = __ffs(__ballot_sync(FULL, incl >= unsigned(K))) - 1;
            const double tsel =
                kstar == 31 ? double(tc) : double(__uint_as_float(unsigned(kstar + base + 1) << 22));
            const double mg = key_margin(tsel, ep);
            if (!(use_r && !(tsel + mg <= r2))) {
                tc = fminf(__double2float_ru(tsel + 2.0 * mg), tc);
                C = compact_chunks(tc);
            }
            if (C > cap) {
                PSTAT(5 + 8 * which, 1);
                // linear sub-buckets inside bucket kstar
                const float lo = kstar == 0 ? 0.f : __uint_as_float(unsigned(kstar + base) << 22);
                const float hi2 = float(tsel);
                const unsigned below = __shfl_sync(FULL, incl - cnt, kstar);
                const float w2 = (hi2 - lo) * (1.0f / 32.0f);
                const float inv2 = w2 > 0.f ? 1.0f / w2 : 0.f;
                over_chunks<KU>(ps, list, nlist, pxf, pyf, [&](int pos, float a, float2) {
                    if (pos >= 0 && a >= lo && a < hi2) hist[min(31, max(0, int((a - lo) * inv2))) * 32 + lane] += 1;
                });
                __syncwarp();
                cnt = hist_reduce(hist);
                incl = warp_incl_scan(cnt) + below;
                const int k2 = __ffs(__ballot_sync(FULL, incl >= unsigned(K))) - 1;
                if (k2 >= 0) {
                    const double t2 = (double(lo) + double(k2 + 1) * double(w2)) * (1.0 + 1e-6) + 1e-30;
                    const double mg2 = key_margin(t2, ep);
                    if (!(use_r && !(t2 + mg2 <= r2))) {
                        tc = fminf(__double2float_ru(t2 + 2.0 * mg2), tc);
                        C = compact_chunks(tc);
                    }
                }
            }
        }
    }
    if (C > cap) {
        // Pathological crowding at the threshold: exact iterative selection.
        PSTAT(6 + 8 * which, 1);
        double pk_ = -1.0;
        int po = -1, nsel = 0;
        for (int k = 0; k < K; ++k) {
            double best = INFINITY;
            int bo = INT_MAX, bp = -1;
            for (int i = lane; i < n; i += 32) {
                const float2 p = ps.xy[i];
                const double dx = double(p.x) - px, dy = double(p.y) - py;
                const double e = dx * dx + dy * dy;
                if (use_r && !(e <= r2)) continue;
                const int o = ps.oi[i];
                const bool after = e > pk_ || (e == pk_ && o > po);
                if (after && (e < best || (e == best && o < bo))) best = e, bo = o, bp = i;
            }
            double bd;
            int bidx;
            warp_argmin(best, bo, bd, bidx);
            if (bidx == INT_MAX || !(bd < INFINITY)) break;
            const int src = __ffs(__ballot_sync(FULL, bo == bidx && best == bd)) - 1;
            const int bpos = __shfl_sync(FULL, bp, src);
            if (lane == 0) order[k] = bpos;
            pk_ = bd;
            po = bidx;
            ++nsel;
        }
        __syncwarp();
        return nsel;
    }

    // ---- 4. exact fp64 keys (reference op order), counting sort, in-bucket rank ----
    // cidx: candidate position, ckey: exact key, cinfo: reference index; the
    // counting-sort counters / cursors live in the (clear) histogram area and
    // the selection is written to `order` after the ranking is complete.
    unsigned* cntb = reinterpret_cast<unsigned*>(hist);  // NB2 u32 counters
    // bucket = floor(key * sc2): any positive scale keeps the buckets in key
    // order (the same function counts, scatters and ranks), so an approximate
    // reciprocal does
    float rtc;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rtc) : "f"(tc > 0.f ? tc : 1.f));
    const double sc2 = double(NB2) * double(rtc);
    int nvalid_local = 0;
    for (int c0 = 0; c0 < C; c0 += 32 * 4) {
        // reference indices of 4 candidates per lane in flight (8: +0.4%), then the exact
        // keys from the points staged at compaction
        int oiv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = c0 + 32 * u + lane;
            ZS_CHECK(c >= C || (cidx[c] >= 0 && cidx[c] < n));
            oiv[u] = c < C ? ps.oi[cidx[c]] : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = c0 + 32 * u + lane;
            if (c < C) {
                const float2 p = reinterpret_cast<const float2*>(ckey)[c];
                const double dx = double(p.x) - px, dy = double(p.y) - py;
                const double e = dx * dx + dy * dy;
                const bool ok = !use_r || e <= r2;
                ckey[c] = ok ? e : INFINITY;
                cinfo[c] = oiv[u];
                if (ok) {
                    atomicAdd(&cntb[bslot(min(NB2 - 1, int(e * sc2)))], 1u);
                    ++nvalid_local;
                }
            }
        }
    }
    const int nvalid = int(__reduce_add_sync(FULL, unsigned(nvalid_local)));
    __syncwarp();
    {
        unsigned v[NB2 / 32];
        unsigned s = 0;
#pragma unroll
        for (int k = 0; k < NB2 / 32; ++k) {
            v[k] = cntb[k * 32 + lane];
            s += v[k];
        }
        unsigned run = warp_incl_scan(s) - s;
#pragma unroll
        for (int k = 0; k < NB2 / 32; ++k) {
            cntb[k * 32 + lane] = run;        // bucket start
            cntb[NB2 + k * 32 + lane] = run;  // scatter cursor
            run += v[k];
        }
    }
    __syncwarp();
    for (int c = lane; c < C; c += 32) {
        const double e = ckey[c];
        if (e < INFINITY) {
            const unsigned q = atomicAdd(&cntb[NB2 + bslot(min(NB2 - 1, int(e * sc2)))], 1u);
            ZS_CHECK(q < unsigned(C));
            order[q] = c;
        }
    }
    __syncwarp();
    int* sel_tmp = reinterpret_cast<int*>(cntb + NB2);  // cursors are done: reuse as the selection
    __syncwarp();
    for (int c = lane; c < C; c += 32) {
        const double e = ckey[c];
        if (!(e < INFINITY)) continue;
        const int bk = min(NB2 - 1, int(e * sc2));
        const int o_self = cinfo[c];
        const unsigned start = cntb[bslot(bk)];
        if (start >= unsigned(K)) continue;  // every key of an earlier bucket is smaller: cannot rank < K
        const unsigned end = bk + 1 < NB2 ? cntb[bslot(bk + 1)] : unsigned(nvalid);
        unsigned rank = start;
#pragma unroll 1
        for (unsigned q = start; q < end; ++q) {
            const int o = order[q];
            ZS_CHECK(o >= 0 && o < C);
            const double eo = ckey[o];
            const int io = cinfo[o];
            rank += (eo < e || (eo == e && io < o_self)) ? 1u : 0u;
        }
        if (rank < unsigned(K)) sel_tmp[rank] = cidx[c];
        if (hint != nullptr && rank == unsigned(K - 1)) {
            float* hk = which == 0 ? &hint->z : &hint->w;
            *hk = __double2float_ru(e);
        }
    }
    __syncwarp();
    const int nsel_out = min(K, nvalid);
    for (int k = lane; k < nsel_out; k += 32) order[k] = sel_tmp[k];
    __syncwarp();
    if (hint != nullptr && lane == 0) {
        if (nvalid < K) (which == 0 ? hint->z : hint->w) = INFINITY;  // fewer than k qualify: no bound
        if (which == 1) {  // both keys now refer to this position (road is selected first)
            hint->x = float(px);
            hint->y = float(py);
        }
    }
    __syncwarp();
    for (int k = lane; k < 2 * NB2 / 4; k += 32) reinterpret_cast<uint4*>(cntb)[k] = make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();
    return nsel_out;
}

// ---------------------------------------------------------------------------
// observe one row (simcore.cpp:423-538) from w.rs->r.  When
// w.rs->boxes_ready, the ego box and the agent boxes at r.t with their
// overlap flags are already in smem (fused step+observe).
// ---------------------------------------------------------------------------
// Observation parts: kObsAgents = active features + agents + value-only,
// kObsMap = road + route top-k.  Large batches run them as separate kernels
// (smaller code per kernel: rows of a multi-wave batch are out of phase and a
// fused kernel's code then thrashes the instruction cache).
constexpr int kObsAgents = 1, kObsMap = 2, kObsAll = 3;

template <int PARTS, bool SA = false>
__device__ void observe_row(const KernelArgs& a, int b, const WarpBuf& w) {
    ROW_MARK(b, 2);
    const DevPack& pk = a.pk;
    const DevCfg& cfg = a.cfg;
    const int lane = lane_id();
    RowSh& rs = *w.rs;
    const Row& r = rs.r;
    const int Ka = cfg.n_agents, Kr = cfg.n_road, Kl = cfg.n_route;
    float* act = a.obs.active + size_t(b) * 9;
    float* agt = a.obs.agents + size_t(b) * Ka * 6;
    float* rd = a.obs.road + size_t(b) * Kr * 12;
    float* rt = a.obs.route + size_t(b) * Kl * 5;
    float* val = a.obs.value_only + size_t(b) * 2;
    int32_t* dbg = a.dbg ? a.dbg + size_t(b) * (Ka + Kr + Kl) : nullptr;

    if (r.done) {
        // ObservationBatch::zero_row (simcore.cpp:37-43)
        if (PARTS & kObsAgents) {
            for (int i = lane; i < 9; i += 32) act[i] = 0.f;
            for (int i = lane; i < Ka * 6; i += 32) agt[i] = 0.f;
            if (lane < 2) val[lane] = 0.f;
            if (dbg)
                for (int i = lane; i < Ka; i += 32) dbg[i] = -1;
        }
        if (PARTS & kObsMap) {
            float4* rd4 = reinterpret_cast<float4*>(rd);
            for (int i = lane; i < Kr * 3; i += 32) rd4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int i = lane; i < Kl * 5; i += 32) rt[i] = 0.f;
            if (dbg)
                for (int i = Ka + lane; i < Ka + Kr + Kl; i += 32) dbg[i] = -1;
        }
        return;
    }

    const int t = uni(r.t);
    const int sc = uni(rs.sc), skip = uni(rs.skip);  // scenario data index, controlled actor's agent column
    PSTAT(0, 1);
    const bool boxes_ready = rs.boxes_ready != 0;
    if (!boxes_ready) {
        const double2 sc = sincos2(r.h);
        if (lane == 0) {
            const double c = sc.y, s = sc.x;
            Box eb;
            eb.cx = r.x + c * cfg.ego_center_offset;
            eb.cy = r.y + s * cfg.ego_center_offset;
            eb.hl = cfg.ego_length * 0.5;
            eb.hw = cfg.ego_width * 0.5;
            eb.c = c;
            eb.s = s;
            rs.eb = eb;
            box_corners(eb, rs.ex, rs.ey);
        }
        __syncwarp();
    }
    // ego-frame rotation by -heading (simcore.cpp:432): cos(-h) = cos h, sin(-h) = -sin h
    const double oc = rs.eb.c, os = -rs.eb.s;

    if (PARTS & kObsAgents) {
    // ---- active features: roads::stop_info (roads.cpp:253-277), simcore.cpp:440-455 ----
    {
        double best_stop = 1e300;
        const int ns = pk.n_stops[sc];
#pragma unroll 1
        for (int j = 0; j < ns; ++j) {
            double ahead = pk.st_s[size_t(sc) * pk.d.NS + j] - r.proj_s;
            if (ahead > 0.0 && ahead < best_stop) best_stop = ahead;
        }
        double best_light = 1e300;
        int best_k = -1;
        const int nlt = pk.n_lights[sc];
#pragma unroll 1
        for (int k = 0; k < nlt; ++k) {
            double ahead = pk.lt_s[size_t(sc) * pk.d.NL + k] - r.proj_s;
            if (ahead > 0.0 && ahead < best_light) {
                best_light = ahead;
                best_k = k;
            }
        }
        int light = 3;
        if (best_k >= 0) {
            int nsteps = pk.num_steps[sc];
            int step = t < nsteps - 1 ? t : nsteps - 1;
            step = step > 0 ? step : 0;
            light = pk.lt_state[(size_t(sc) * pk.d.NL + best_k) * pk.d.T + step];
        }
        const double R = cfg.feature_radius;
        if (lane < 9) {
            float f = 0.f;
            if (lane == 0) f = float(r.v);
            if (lane == 1) f = float(r.steer);
            if (lane == 2) f = float(best_stop < 1e300 ? mind(best_stop, R) : R);
            if (lane >= 3 && lane <= 6) f = (lane - 3 == light) ? 1.f : 0.f;
            if (lane == 7) f = float(best_k >= 0 ? mind(best_light, R) : R);
            if (lane == 8) f = pk.speed_limit[sc];
            obs_st(act + lane, f);
        }
        // value-only features (simcore.cpp:531-537)
        if (lane == 0) {
            double gx = double(pk.goal_x[b]) - r.x, gy = double(pk.goal_y[b]) - r.y;
            obs_st(val, float(sqrt(gx * gx + gy * gy)));
            obs_st(val + 1, float(pk.horizon - t));
        }
    }

    ROW_MARK(b, 16);
    // ---- other agents: obb_distance, sorted by (dist, idx) (simcore.cpp:457-486) ----
    const int A = pk.d.A;
    // SA: the batch's agent capacity is <= 32 (C1), so the > 32-agent
    // paths compile out of this kernel instance
    const int na = SA ? min(pk.n_agents[sc], 32) : pk.n_agents[sc];
    const bool t_ok = t < pk.num_steps[sc];
    const size_t aslice = (size_t(sc) * pk.d.T + (t_ok ? t : 0)) * A;
    if (!boxes_ready) {
        agent_boxes<2>(pk, sc, aslice, na, skip, t_ok, rs.eb, rs.ex, rs.ey, w);
        __syncwarp();
    }
    // obb_distance (geometry.cpp:77-88), ONE AGENT PER LANE.  Overlap => 0.
    // Otherwise the minimum of the 32 point-to-edge d2 (ego corner vs agent
    // edge, agent corner vs ego edge; segment_segment_distance's endpoint
    // terms).  fp32 screening in ego-centred coordinates: rounding the corners
    // moves each by <= 2^-24 S (S = largest centred coordinate) and the fp32
    // arithmetic (approximate division, clamped t) adds <= 2^-20 (d + |edge|),
    // so |d_f32 - d| <= delta = 2^-18 (S + E + d) (E bounds the edge lengths).
    // A pair enters the candidate mask when d_f32 <= (running min) + 2 delta
    // -- a superset of the final cut; the running min moves once per edge, over
    // the edge's four independent pairs -- and only candidates get the fp64
    // expressions.  A (near-)contact (min d2 < 1e-18) takes the reference's
    // full segment_segment_distance over the 16 edge pairs.
    const double* GX = rs.ex;
    const double* GY = rs.ey;
    const double ecx = rs.eb.cx, ecy = rs.eb.cy;
    float gxf[4], gyf[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        gxf[k] = float(GX[k] - ecx);
        gyf[k] = float(GY[k] - ecy);
    }
    const float ge = float(2.0 * (rs.eb.hl + rs.eb.hw)) + 1e-3f;  // >= any ego edge length
    // Beyond 32 agents, agents that cannot be among the n_agents nearest are
    // pruned before the exact distances.  Along the centre line u (centre
    // distance D): the boxes' supports r(u) = hl |u.e1| + hw |u.e2| give
    // D - r_e(u) - r_a(u) <= obb_distance (the separation along u), and the
    // centre-line points still inside each box (reach t(u) = min(hl / |u.e1|,
    // hw / |u.e2|)) give obb_distance <= max(0, D - t_e(u) - t_a(u)); margins
    // cover the rounding.  An agent whose lower bound exceeds the Ka-th
    // smallest upper bound is strictly farther than the Ka-th nearest, so it
    // is never selected.
    int nvalid = 0, nlist = na;
    bool pruned = false;
#ifdef ZS_NO_PRUNE
    if (false) {
#else
    if (na > 32 && Ka <= 16) {
#endif
        for (int j0 = 0; j0 < na; j0 += 32) {
            const int j = j0 + lane;
            const int fl = j < na ? w.agf[j] : -1;
            // (agent_boxes -- the step's collision pass, or the call above
            // when not fused -- stored the bounds: lower in agd, key in alist)
            nvalid += __popc(__ballot_sync(FULL, fl >= 0));
        }
        __syncwarp();
        if (nvalid > Ka) {
            // Ka-th smallest upper bound on the keys' top 16 bits, rounded up
            // to the bucket's largest key: still an upper bound, half the passes
            const double U = double(__uint_as_float(warp_kth_key(w.alist, na, Ka, reinterpret_cast<unsigned*>(w.agy)) | 0xFFFFu));
            __syncwarp();
            int n = 0;
            for (int j0 = 0; j0 < na; j0 += 32) {
                const int j = j0 + lane;
                const int fl = j < na ? w.agf[j] : -1;
                const bool keep = fl == 1 || (fl == 0 && w.agd[j] <= U);
                const unsigned bal = __ballot_sync(FULL, keep);
                ZS_CHECK(!keep || n + __popc(bal & lanemask_lt()) < na);
                if (keep) w.alist[n + __popc(bal & lanemask_lt())] = j;  // positions <= j: keys already consumed
                n += __popc(bal);
            }
            __syncwarp();
            nlist = n;
            pruned = true;
            PSTAT(17, n);
            PSTAT(18, 1);
        }
    }
    const int nv_all = nvalid;
    nvalid = 0;
    for (int k0 = 0; k0 < nlist; k0 += 32) {
        const int k = k0 + lane;
        const int j = pruned ? (k < nlist ? w.alist[k] : na) : k;
        const int fl = j < na ? w.agf[j] : -1;
        if (fl == 0) {
            // beyond 32 agents only one chunk of corners is kept: this lane's slot
            const int slot = na > 32 ? lane : j;
            if (na > 32) agent_corners(pk, sc, aslice, j, slot, w.agx, w.agy);
            const double* AX = w.agx + slot;  // corner k at AX[k * kAgSlots]
            const double* AY = w.agy + slot;
            float axf[4], ayf[4];
            float S = 0.f;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                axf[k] = float(AX[k * kAgSlots] - ecx);
                ayf[k] = float(AY[k * kAgSlots] - ecy);
                S = fmaxf(S, fmaxf(fabsf(axf[k]), fabsf(ayf[k])));
            }
            float E = ge;
#pragma unroll
            for (int k = 0; k < 4; ++k) E = fmaxf(E, fabsf(axf[(k + 1) & 3] - axf[k]) + fabsf(ayf[(k + 1) & 3] - ayf[k]));
            const float c0 = 0x1p-18f * (S + ge + E);  // ge also bounds the centred ego corners
            float min2 = INFINITY, thr2 = INFINITY;
            unsigned cmask = 0;
            // pairs base + 4 ci + ei: corner ci of (qx, qy) vs edge ei of (px, py).
            // The edge loop stays rolled (code size: the fused kernel is far
            // larger than the instruction cache); the edge's polygon rotates
            // through registers so every index stays static.
            auto side = [&](float (&px)[4], float (&py)[4], const float (&qx)[4], const float (&qy)[4], int base) {
#pragma unroll 1
                for (int ei = 0; ei < 4; ++ei) {
                    const float4 f = make_float4(px[0], py[0], px[1] - px[0], py[1] - py[0]);
                    const float inv = seg_inv_f(f);
                    // the edge's four pairs are independent: one running-minimum
                    // update per edge (the threshold a pair is tested against
                    // still only shrinks, so the mask stays a superset)
                    float d[4];
#pragma unroll
                    for (int ci = 0; ci < 4; ++ci) d[ci] = seg_d2_f(qx[ci], qy[ci], f, inv);
                    const float m4 = fminf(fminf(d[0], d[1]), fminf(d[2], d[3]));
                    if (m4 < min2) {
                        min2 = m4;
                        float m;  // sqrt.approx (rel. error < 2^-22), scaled up to an upper bound
                        asm("sqrt.approx.f32 %0, %1;" : "=f"(m) : "f"(m4));
                        m *= 1.f + 0x1p-20f;
                        const float r = m + 2.f * (c0 + 0x1p-18f * m) + 1e-30f;
                        thr2 = r * r * (1.f + 0x1p-20f);
                    }
#pragma unroll
                    for (int ci = 0; ci < 4; ++ci)
                        if (d[ci] <= thr2) cmask |= 1u << (base + 4 * ci + ei);
                    const float tx = px[0], ty = py[0];
                    px[0] = px[1], py[0] = py[1], px[1] = px[2], py[1] = py[2], px[2] = px[3], py[2] = py[3];
                    px[3] = tx, py[3] = ty;
                }
            };
            side(axf, ayf, gxf, gyf, 0);
            side(gxf, gyf, axf, ayf, 16);
            // exact candidates
            double d2min = INFINITY;
            while (cmask) {
                const int pr = __ffs(cmask) - 1;
                cmask &= cmask - 1;
                const int ci = (pr >> 2) & 3, ei = pr & 3, ei1 = (ei + 1) & 3;
                const int S = kAgSlots;
                const double d2 = pr < 16 ? seg_dist2_fast(GX[ci], GY[ci], AX[S * ei], AY[S * ei], AX[S * ei1], AY[S * ei1])
                                          : seg_dist2_fast(AX[S * ci], AY[S * ci], GX[ei], GY[ei], GX[ei1], GY[ei1]);
                d2min = fmin(d2min, d2);
            }
            if (!(d2min >= 1e-18)) {
                PSTAT(20, 1);
                d2min = contact_dist2(GX, GY, AX, AY);
            }
            w.agd[j] = sqrt(d2min);  // obb_distance returns sqrt of the min d2
        } else if (fl == 1) {
            w.agd[j] = 0.0;
        }
        nvalid += __popc(__ballot_sync(FULL, fl >= 0));
    }
    if (pruned) nvalid = nv_all;  // every valid agent counts; at least Ka of them survived
    __syncwarp();
    ROW_MARK(b, 17);
    // order by (distance, index) among the valid agents: bitonic sorts across
    // the warp on (distance bits, index) -- distances are >= +0 so their bit
    // patterns order like the values; invalid = +inf, last.  More than 32
    // agents: the best 16 so far (lanes 0-15) are merged with each further
    // chunk's best 16 (lanes 16-31) by one more sort.
    if (na <= 32 || Ka <= 16) {
        auto sort32 = [&](unsigned long long& key, int& idx) {
#pragma unroll
            for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
                for (int jj = k >> 1; jj > 0; jj >>= 1) {
                    const unsigned long long ok_ = __shfl_xor_sync(FULL, key, jj);
                    const int oi = __shfl_xor_sync(FULL, idx, jj);
                    const bool other_less = ok_ < key || (ok_ == key && oi < idx);
                    const bool keep_min = ((lane & jj) == 0) == ((lane & k) == 0);
                    if (keep_min == other_less) key = ok_, idx = oi;
                }
            }
        };
        unsigned long long bkey = 0xFFF0000000000000ull;
        int bidx = INT_MAX;
        for (int k0 = 0; k0 < nlist; k0 += 32) {
            const int k = k0 + lane;
            const int j = pruned ? (k < nlist ? w.alist[k] : na) : k;
            const bool ok = j < na && w.agf[j] >= 0;
            unsigned long long key = ok ? (unsigned long long)__double_as_longlong(w.agd[j]) : 0xFFF0000000000000ull;
            int idx = ok ? j : INT_MAX;
            sort32(key, idx);
            if (k0 > 0) {
                // lanes 16-31 take this chunk's best 16, lanes 0-15 keep the running best
                const unsigned long long ck = __shfl_sync(FULL, key, lane - 16);
                const int ci = __shfl_sync(FULL, idx, lane - 16);
                key = lane < 16 ? bkey : ck;
                idx = lane < 16 ? bidx : ci;
                sort32(key, idx);
            }
            bkey = key;
            bidx = idx;
        }
        if (lane < Ka && lane < nvalid) w.sel[lane] = bidx;
    } else {
        for (int j0 = 0; j0 < na; j0 += 32) {
            const int j = j0 + lane;
            if (j < na && w.agf[j] >= 0) {
                const double dj = w.agd[j];
                int rank = 0;
#pragma unroll 4
                for (int k = 0; k < na; ++k) {
                    const double dk = w.agd[k];
                    rank += (w.agf[k] >= 0 && (dk < dj || (dk == dj && k < j))) ? 1 : 0;
                }
                ZS_CHECK(rank >= 0);
                if (rank < Ka) w.sel[rank] = j;
            }
        }
    }
    ROW_MARK(b, 18);
    const int nsel_ag = min(Ka, nvalid);
    __syncwarp();
    for (int k = lane; k < Ka; k += 32) {
        float f[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        int j = -1;
        if (k < nsel_ag) {
            j = w.sel[k];
            ZS_CHECK(j >= 0 && j < na);
            double wx = double(pk.ag_x[aslice + j]) - r.x, wy = double(pk.ag_y[aslice + j]) - r.y;
            f[0] = float(oc * wx - os * wy);
            f[1] = float(os * wx + oc * wy);
            f[2] = float(wrap1(double(pk.ag_h[aslice + j]) - r.h));
            f[3] = pk.ag_sp[aslice + j];
            f[4] = float(w.agd[j]);
            f[5] = 1.f;
        }
        float2* o = reinterpret_cast<float2*>(agt + k * 6);
        obs_st(o, make_float2(f[0], f[1]));
        obs_st(o + 1, make_float2(f[2], f[3]));
        obs_st(o + 2, make_float2(f[4], f[5]));
        if (dbg) dbg[k] = (skip >= 0 && j > skip) ? j - 1 : j;  // index among the row's agents
    }

    }  // PARTS & kObsAgents

    if (PARTS & kObsMap) {
    // ---- road network points: nearest_features (roads.cpp:210-236) ----
    // the top-k region overlays the (now dead) agent buffers: clear the histogram
    ROW_MARK(b, 3);
    __syncwarp();
    for (int k = lane; k < 32 * 32; k += 32) w.hist[k] = 0;
    __syncwarp();
    {
        const int n = pk.n_road[sc];
        const float2* pts = pk.road_xy + size_t(sc) * pk.d.P;
        const int32_t* oidx = pk.road_oi + size_t(sc) * pk.d.P;
        const double R = cfg.feature_radius;
        const uint16_t* sel = w.order;
        const PointSet ps{pts, oidx, pk.road_cb + size_t(sc) * pk.d.PC, n, (n + kChunk - 1) / kChunk};
        const int nsel = warp_topk<PARTS == kObsAll ? kUnrollFused : kUnrollMap>(ps, Kr, r.x, r.y, true, R * R, pk.road_box[sc], a.cand_cap, w.hist, w.cidx, w.ckey,
                                   w.cinfo, w.order, rs.hint, a.hint ? a.hint + b : nullptr, 0);
        ROW_MARK(b, 4);
        const uint8_t* kd = pk.road_kd + size_t(sc) * pk.d.P;
        // the selected points' coordinates and kinds for four slots per lane
        // are loaded before any feature is written (the stores could alias
        // the loads, so the compiler keeps them in order otherwise: four round
        // trips instead of one).  Measured: C2 / C4 shard -0.7%, C1 -0.7%.
        constexpr int RS = 4;
        for (int k0 = lane; k0 < Kr; k0 += 32 * RS) {
            float2 pv[RS];
            int kv[RS], iv[RS];
#pragma unroll
            for (int u = 0; u < RS; ++u) {
                const int k = k0 + 32 * u;
                iv[u] = k < nsel ? int(sel[k]) : -1;
                ZS_CHECK(iv[u] < n);
                pv[u] = iv[u] >= 0 ? pts[iv[u]] : make_float2(0.f, 0.f);
                kv[u] = iv[u] >= 0 ? int(kd[iv[u]]) : 0;
            }
#pragma unroll
            for (int u = 0; u < RS; ++u) {
                const int k = k0 + 32 * u;
                if (k >= Kr) break;
                float f[12];
#pragma unroll
                for (int q = 0; q < 12; ++q) f[q] = 0.f;
                const int i = iv[u];
                if (i >= 0) {
                    double wx = double(pv[u].x) - r.x, wy = double(pv[u].y) - r.y;
                    f[0] = float(oc * wx - os * wy);
                    f[1] = float(os * wx + oc * wy);
                    const int kk = kv[u];
#pragma unroll
                    for (int q = 0; q < 5; ++q) f[2 + q] = (kk & 15) == q ? 1.f : 0.f;
#pragma unroll
                    for (int q = 0; q < 4; ++q) f[7 + q] = (kk >> 4) == q ? 1.f : 0.f;
                    f[11] = 1.f;
                }
                float4* o = reinterpret_cast<float4*>(rd + k * 12);
                obs_st(o, make_float4(f[0], f[1], f[2], f[3]));
                obs_st(o + 1, make_float4(f[4], f[5], f[6], f[7]));
                obs_st(o + 2, make_float4(f[8], f[9], f[10], f[11]));
                if (dbg) dbg[Ka + k] = i < 0 ? -1 : oidx[i];
            }
        }
    }

    // ---- route border points: top n_route by (d2, idx), no radius (simcore.cpp:503-529) ----
    ROW_MARK(b, 5);
    {
        const int n = pk.n_route[sc];
        const float2* pts = pk.route_xy + size_t(sc) * pk.d.R;
        const int32_t* oidx = pk.route_oi + size_t(sc) * pk.d.R;
        const uint16_t* sel = w.order;
        const PointSet ps{pts, oidx, pk.route_cb + size_t(sc) * pk.d.RC, n, (n + kChunk - 1) / kChunk};
        const int nsel = warp_topk<PARTS == kObsAll ? kUnrollFused : kUnrollMap>(ps, Kl, r.x, r.y, false, 0.0, pk.route_box[sc], a.cand_cap, w.hist, w.cidx, w.ckey,
                                   w.cinfo, w.order, rs.hint, a.hint ? a.hint + b : nullptr, 1);
        ROW_MARK(b, 6);
        const uint8_t* fl = pk.route_fl + size_t(sc) * pk.d.R;
        for (int k0 = lane; k0 < Kl; k0 += 64) {
            float2 pv[2];
            int fv[2], iv[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int k = k0 + 32 * u;
                iv[u] = k < nsel ? int(sel[k]) : -1;
                ZS_CHECK(iv[u] < n);
                pv[u] = iv[u] >= 0 ? pts[iv[u]] : make_float2(0.f, 0.f);
                fv[u] = iv[u] >= 0 ? int(fl[iv[u]]) : 0;
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int k = k0 + 32 * u;
                if (k >= Kl) break;
                float f[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
                const int i = iv[u];
                if (i >= 0) {
                    double wx = double(pv[u].x) - r.x, wy = double(pv[u].y) - r.y;
                    f[0] = float(oc * wx - os * wy);
                    f[1] = float(os * wx + oc * wy);
                    f[2] = (fv[u] & 1) ? 1.f : 0.f;
                    f[3] = (fv[u] & 2) ? 1.f : 0.f;
                    f[4] = 1.f;
                }
                float* o = rt + k * 5;
#pragma unroll
                for (int q = 0; q < 5; ++q) obs_st(o + q, f[q]);
                if (dbg) dbg[Ka + Kr + k] = i < 0 ? -1 : oidx[i];
            }
        }
    }
    }  // PARTS & kObsMap
}

// EpisodeBatch cell (b, a.ep_t) of Env::rollout's recording loop
// (simcore.cpp:596-608); logp and value from the policy's output (0 for the
// scripted policy).
__device__ __forceinline__ void record_step(const KernelArgs& a, int b, int mask, int ai, int si, float reward,
                                            float s, float a_lat, float a_lon, float v, int done) {
    if (!a.ep.reward) return;
    const size_t k = size_t(b) * size_t(a.ep.horizon) + size_t(a.ep_t);
    a.ep.mask[k] = uint8_t(mask);
    a.ep.accel_idx[k] = ai;
    a.ep.steer_idx[k] = si;
    a.ep.logp[k] = a.pol_logp ? a.pol_logp[b] : 0.f;
    a.ep.value[k] = a.pol_value ? a.pol_value[b] : 0.f;
    a.ep.reward[k] = reward;
    a.ep.s[k] = s;
    a.ep.a_lat[k] = a_lat;
    a.ep.a_lon[k] = a_lon;
    a.ep.v[k] = v;
    a.ep.done[k] = uint8_t(done);
}

// ---------------------------------------------------------------------------
// step one row (simcore.cpp:278-404): reads w.rs->r0, writes the post-step
// row to w.rs->r (+ output buffers).  When the row is simulated (not passed
// through) the ego box, the agent boxes at t+1 and their overlap flags stay in
// smem for a fused observe (w.rs->boxes_ready).
// ---------------------------------------------------------------------------
template <bool REC, int AGB, bool SA = false>
__device__ void step_row(const KernelArgs& a, int b, const WarpBuf& w) {
    const DevPack& pk = a.pk;
    const DevCfg& cfg = a.cfg;
    const int lane = lane_id();
    RowSh& rs = *w.rs;
    const int sc = uni(rs.sc), skip = uni(rs.skip);  // scenario data index, controlled actor's agent column
    const int ns = uni(pk.n_stops[sc]);
    const int soff = uni(pk.stop_off[b]);
    for (int j = lane; j < ns; j += 32) w.sflag[j] = a.in.stopped_flags[soff + j];
    __syncwarp();
    ROW_MARK(b, 8);

    bool pass = rs.r0.done != 0;
    int ai = 0, si = 0;
    if (REC && a.act_len != 0) {
        // ScriptedPolicy::act (simcore.cpp:69-84): the script at the row's t, else the zero action
        const int tt = rs.r0.t;
        if (a.act_len == -2) {  // NNPolicy output of this step, every row (done rows still pass through)
            ai = a.accel[b];
            si = a.steer[b];
        } else if (a.act_len > 0 && tt >= 0 && tt < a.act_len) {
            ai = a.accel[size_t(tt) * pk.d.B + b];
            si = a.steer[size_t(tt) * pk.d.B + b];
        } else {
            ai = a.zero_accel;
            si = a.zero_steer;
        }
    } else if (!pass) {
        ai = a.accel[b];
        si = a.steer[b];
    }
    if (!pass && (ai < 0 || ai >= cfg.n_accel || si < 0 || si >= cfg.n_steer)) {
        if (lane == 0) atomicOr(a.err, 1);
        pass = true;
    }
    if (pass) {
        // absorbing pass-through (simcore.cpp:281-299); bad-action rows are left unchanged
        if (lane == 0) {
            const Row r0 = rs.r0;
            rs.r = r0;
            rs.boxes_ready = 0;
            store_row(a.out, b, r0);
            a.so.reward[b] = 0.f;
            a.so.event[b] = 0;
            a.so.s[b] = float(r0.proj_s);
            a.so.a_lat[b] = 0.f;
            a.so.a_lon[b] = 0.f;
            a.so.v[b] = float(r0.v);
            if (REC) record_step(a, b, r0.done ? 0 : 1, ai, si, 0.f, float(r0.proj_s), 0.f, 0.f, float(r0.v), r0.done);
        }
        for (int j = lane; j < ns; j += 32) a.out.stopped_flags[soff + j] = w.sflag[j];
        __syncwarp();
        return;
    }

    PSTAT(23, 1);
    const double accel = cfg.accel_bins[ai], rate = cfg.steer_bins[si];
    const double dt = pk.dt;
    {
        // dyn::bicycle_step (dynamics.cpp:10-19)
        const double x0 = rs.r0.x, y0 = rs.r0.y, h0 = rs.r0.h, v0 = rs.r0.v, st0 = rs.r0.steer;
        const double2 sc0 = sincos2(h0);
        const double tan_steer = tan1(st0);
        const double x = x0 + v0 * sc0.y * dt;
        const double y = y0 + v0 * sc0.x * dt;
        const double h = wrap1(h0 + v0 / cfg.wheelbase * tan_steer * dt);
        // ego_box(e1) (simcore.cpp:156-160) and its margin-inflated corners (roads.cpp:202-204)
        const double2 sc1 = sincos2(h);
        if (lane == 0) {
            Row& r = rs.r;
            r.x = x;
            r.y = y;
            r.h = h;
            r.v = maxd(v0 + accel * dt, cfg.v_min);
            r.steer = clampd(st0 + rate * dt, -cfg.delta_max, cfg.delta_max);
            r.t = rs.r0.t + 1;
            r.rng = rs.r0.rng;
            Box eb;
            eb.cx = x + sc1.y * cfg.ego_center_offset;
            eb.cy = y + sc1.x * cfg.ego_center_offset;
            eb.hl = cfg.ego_length * 0.5;
            eb.hw = cfg.ego_width * 0.5;
            eb.c = sc1.y;
            eb.s = sc1.x;
            rs.eb = eb;
            box_corners(eb, rs.ex, rs.ey);
            Box inf = eb;
            inf.hl = eb.hl + cfg.footprint_margin;
            inf.hw = eb.hw + cfg.footprint_margin;
            double X[4], Y[4];
            box_corners(inf, X, Y);
            rs.qx[0] = x;
            rs.qy[0] = y;
            for (int k = 0; k < 4; ++k) rs.qx[k + 1] = X[k], rs.qy[k + 1] = Y[k];
            rs.a_lat = v0 * v0 * tan_steer / cfg.wheelbase;
            // failure detection: a non-finite ego state (NaN / Inf input or
            // overflow) is flagged in the error word (bit 1); the step itself
            // proceeds exactly like the reference, which does not check
            if (!(isfinite(x) && isfinite(y) && isfinite(h) && isfinite(r.v) && isfinite(r.steer)))
                atomicOr(a.err, 2);
        }
        __syncwarp();
    }
    const double a_lat = rs.a_lat;
    ROW_MARK(b, 9);
    const Proj p1 = warp_project<NQ>(pk, sc, rs.qx, rs.qy);
    ROW_MARK(b, 1);

    // collision with the agents valid at t+1 (simcore.cpp:323-331); boxes kept for observe(t+1)
    int hit = 0;
    {
        const int na = SA ? min(pk.n_agents[sc], 32) : pk.n_agents[sc];
        const int t1 = rs.r.t;
        const bool t_ok = t1 < pk.num_steps[sc];
        const size_t slice = (size_t(sc) * pk.d.T + (t_ok ? t1 : 0)) * pk.d.A;
        hit = __any_sync(FULL, agent_boxes<AGB>(pk, sc, slice, na, skip, t_ok, rs.eb, rs.ex, rs.ey, w));
    }

    const double ps0 = rs.r0.proj_s, v0 = rs.r0.v, vn = rs.r.v;
    const int t0 = rs.r0.t;
    const bool hit_off_route = !p1.on_route;
    bool hit_red = false;
    {
        const int nsteps = pk.num_steps[sc];
        const int t_light = t0 < nsteps - 1 ? t0 : nsteps - 1;
        const int nlt = pk.n_lights[sc];
#pragma unroll 1
        for (int k = 0; k < nlt; ++k) {
            double ls = pk.lt_s[size_t(sc) * pk.d.NL + k];
            if (ps0 < ls && ls <= p1.s && pk.lt_state[(size_t(sc) * pk.d.NL + k) * pk.d.T + t_light] == 0)
                hit_red = true;
        }
    }
    bool hit_stop = false;
#pragma unroll 1
    for (int j = 0; j < ns; ++j) {
        double ss = pk.st_s[size_t(sc) * pk.d.NS + j];
        if (ps0 < ss && ss <= p1.s && v0 > cfg.stop_cross_speed && !w.sflag[j]) hit_stop = true;
    }
    const bool hit_goal = fabs(p1.s - pk.goal_s[b]) <= cfg.goal_radius;
    const double progress = p1.s - ps0;
    const double a_lon = accel;
    double reward = cfg.w_progress * progress - cfg.w_speed * maxd(0.0, vn - double(pk.speed_limit[sc])) * dt -
                    cfg.w_lat * a_lat * a_lat * dt - cfg.w_lon * a_lon * a_lon * dt;
    const int reason = hit ? 1 : hit_off_route ? 2 : hit_red ? 3 : hit_stop ? 4 : hit_goal ? 5 : 0;
    int events = rs.r0.events;
    if (cfg.disable_dones) {
        events |= (hit ? 1 : 0) | (hit_off_route ? 2 : 0) | (hit_red ? 4 : 0) | (hit_stop ? 8 : 0) |
                  (hit_goal ? 16 : 0);
    } else if (reason != 0) {
        events |= 1 << (reason - 1);
        if (reason != 5) reward -= cfg.terminal_penalty;
    }
    const int done = (!cfg.disable_dones && reason != 0) ? 1 : 0;
    __syncwarp();
    if (lane == 0) {
        Row& r = rs.r;
        r.done = done;
        r.reason = done ? reason : 0;
        r.proj_s = p1.s;
        r.proj_d = p1.d;
        r.in_corr = p1.in_corr;
        r.events = events;
        rs.boxes_ready = 1;
        store_row(a.out, b, r);
        a.so.reward[b] = float(reward);
        a.so.event[b] = uint8_t(reason);
        a.so.s[b] = float(p1.s);
        a.so.a_lat[b] = float(a_lat);
        a.so.a_lon[b] = float(a_lon);
        a.so.v[b] = float(vn);
        if (REC) record_step(a, b, 1, ai, si, float(reward), float(p1.s), float(a_lat), float(a_lon), float(vn), done);
    }
    // stopped-flag update with the post-step state (simcore.cpp:390-396)
    for (int j = lane; j < ns; j += 32) {
        double ahead = pk.st_s[size_t(sc) * pk.d.NS + j] - p1.s;
        uint8_t fl = w.sflag[j];
        if (ahead >= 0.0 && ahead <= cfg.stop_zone && vn < cfg.stop_slow_speed) fl = 1;
        a.out.stopped_flags[soff + j] = fl;
    }
    __syncwarp();
}

// OCCW resident warps per SM (28: 72 registers; the split map kernel 36: 54), WARPS per CTA
template <bool STEP, int OBS, bool REC, int WARPS, int OCCW = 28, bool SA = false>
__global__ void __launch_bounds__(32 * WARPS, OCCW / WARPS) k_step_observe(const KernelArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    constexpr bool kUniform = OBS == kObsAgents || OBS == kObsMap;  // the split kernels
    const int wib = kUniform ? warp_in_block_uniform() : warp_in_block();
    const WarpBuf w = carve(dsm, a, wib);
    const int wpb = WARPS;
    const int stride = gridDim.x * wpb;
    const int b_end = a.row_hi > 0 ? a.row_hi : a.pk.d.B;
    int b = a.row_lo + blockIdx.x * wpb + wib;
    // the CTA's warps advance row by row together (the same code in flight:
    // the instruction cache is shared instead of thrashed by out-of-phase
    // rows; measured C2 +13%, C1 / C4 +1%)
    for (int b0 = a.row_lo + blockIdx.x * wpb; b0 < b_end; b0 += stride, b += stride) {
        __syncthreads();
        if (b >= b_end) continue;
        if (lane_id() == 0) {
            w.rs->r0 = load_row(a.in, b);
            if ((OBS & kObsMap) && a.hint) w.rs->hint = a.hint[b];
            w.rs->sc = scen_of(a.pk, b);
            w.rs->skip = skip_of(a.pk, b);
        }
        __syncwarp();
        ROW_MARK(b, 0);
        if (STEP) {
            step_row<REC, WARPS == kCtaWarpsCtl ? 1 : 2, SA>(a, b, w);
        } else {
            if (lane_id() == 0) {
                w.rs->r = w.rs->r0;
                w.rs->boxes_ready = 0;
            }
            __syncwarp();
        }
        if (OBS) observe_row<OBS, SA>(a, b, w);
        ROW_MARK(b, 7);
    }
}

// Env::init_state (simcore.cpp:237-276), one warp per row.
__global__ void __launch_bounds__(kThreads) k_reset(const KernelArgs a) {
    const DevPack& pk = a.pk;
    const DevCfg& cfg = a.cfg;
    const int lane = lane_id();
    const int wpb = kThreads / 32;
    for (int b = blockIdx.x * wpb + warp_in_block(); b < pk.d.B; b += gridDim.x * wpb) {
        const int sc = scen_of(pk, b);
        double qx[1] = {pk.init_x[b]}, qy[1] = {pk.init_y[b]};
        const Proj p = warp_project<1>(pk, sc, qx, qy);
        if (lane == 0) {
            a.out.x[b] = pk.init_x[b];
            a.out.y[b] = pk.init_y[b];
            a.out.heading[b] = pk.init_h[b];
            a.out.v[b] = pk.init_v[b];
            a.out.steering[b] = pk.init_steer[b];
            a.out.t[b] = 0;
            a.out.done[b] = 0;
            a.out.reason[b] = 0;
            a.out.rng[b] = reset_rng_state(a.seed, uint64_t(b));
            a.out.proj_s[b] = p.s;
            a.out.proj_d[b] = p.d;
            a.out.proj_in_corridor[b] = uint8_t(p.in_corr);
            a.out.events[b] = 0;
        }
        const int ns = pk.n_stops[sc];
        const int soff = pk.stop_off[b];
        for (int j = lane; j < ns; j += 32) {
            double ahead = pk.st_s[size_t(sc) * pk.d.NS + j] - p.s;
            bool st = ahead >= 0.0 && ahead <= cfg.stop_zone && pk.init_v[b] < cfg.stop_slow_speed;
            a.out.stopped_flags[soff + j] = st ? 1 : 0;
        }
    }
}

// Episode-stats vector (the counts of metrics::Aggregate,
// metrics.hpp:56-69): [rows, done, collision, off_route, red_light,
// stop_line, goal (latched event bits), progress_sum_um] as int64 so the
// cross-GPU all-reduce is exact and order-independent.
__global__ void __launch_bounds__(256) k_episode_stats(const KernelArgs a, const double* initial_s,
                                                       long long* out) {
    __shared__ long long acc[kStatsLen];
    if (threadIdx.x < kStatsLen) acc[threadIdx.x] = 0;
    __syncthreads();
    long long loc[kStatsLen];
    for (int k = 0; k < kStatsLen; ++k) loc[k] = 0;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < a.pk.d.B; b += gridDim.x * blockDim.x) {
        int ev = a.in.events[b];
        loc[0] += 1;
        loc[1] += a.in.done[b] ? 1 : 0;
        for (int k = 0; k < 5; ++k) loc[2 + k] += (ev >> k) & 1;
        loc[7] += llrint((a.in.proj_s[b] - initial_s[b]) * 1e6);
    }
    for (int k = 0; k < kStatsLen; ++k) {
        long long v = loc[k];
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(FULL, v, off);
        if ((threadIdx.x & 31) == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&acc[k]), (unsigned long long)v);
    }
    __syncthreads();
    if (threadIdx.x < kStatsLen)
        atomicAdd(reinterpret_cast<unsigned long long*>(&out[threadIdx.x]), (unsigned long long)acc[threadIdx.x]);
}

// EpisodeBatch tail (simcore.cpp:580-587, 610-617): bootstrap = done ? 0 :
// value (the scripted policy's value is 0), terminal reason, latched events,
// initial_s and logged_progress as float.
__global__ void __launch_bounds__(256) k_episode_finalize(const KernelArgs a, const double* initial_s,
                                                          const double* logged) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < a.pk.d.B; b += gridDim.x * blockDim.x) {
        a.ep.bootstrap[b] = a.in.done[b] || !a.final_value ? 0.f : a.final_value[b];  // simcore.cpp:612
        a.ep.terminal[b] = a.in.reason[b];
        a.ep.events[b] = a.in.events[b];
        a.ep.initial_s[b] = float(initial_s[b]);
        a.ep.logged_progress[b] = float(logged[b]);
    }
}

constexpr int kMetricsThreads = 256;
constexpr int kAggLen = 12;

// map_score (metrics.cpp:13-17); arguments are in range by construction.
__device__ __forceinline__ double map_score(double s, double l) { return s * (1.0 - l) + l; }

// metrics::score_episode (metrics.cpp:54-95) per row, thread per row, and
// this block's Aggregate partial sums (metrics.cpp:97-131) in a fixed order:
// each thread sums its rows in index order, then a fixed smem tree.
__global__ void __launch_bounds__(kMetricsThreads) k_episode_metrics(const KernelArgs a, zsim_score_bounds bb,
                                                                    zsim_comfort_weights cw, zsim_metric_view out,
                                                                    double* part) {
    __shared__ double red[kAggLen][kMetricsThreads];
    double acc[kAggLen];
#pragma unroll
    for (int k = 0; k < kAggLen; ++k) acc[k] = 0.0;
    const zsim_episode_view& ep = a.ep;
    const int T = ep.horizon;
    const double dt = a.pk.dt;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < a.pk.d.B; b += gridDim.x * blockDim.x) {
        const size_t row = size_t(b) * size_t(T);
        const double logged = double(ep.logged_progress[b]);
        int last_live = -1;
        for (int t = 0; t < T; ++t)
            if (ep.mask[row + t]) last_live = t;
        const double init = double(ep.initial_s[b]);
        const double final_s = last_live >= 0 ? double(ep.s[row + last_live]) : init;
        const double moved = final_s - init;
        const bool degenerate = logged <= 0.1;
        const double raw = degenerate ? 0.0 : moved / logged;
        const double rel = degenerate ? 0.0 : clampd(raw, 0.0, 1.0);
        const int ev = ep.events[b];
        const double coll = (ev & 1) ? 0.0 : 1.0, off = (ev & 2) ? 0.0 : 1.0, light = (ev & 4) ? 0.0 : 1.0,
                     stop = (ev & 8) ? 0.0 : 1.0;
        const bool goal = (ev & 16) != 0;
        const bool failed = coll == 0.0 || off == 0.0;
        // mixed_comfort (metrics.cpp:29-52)
        double cacc = 0.0, prev_lat = 0.0, prev_lon = 0.0;
        bool have_prev = false;
        long long live = 0;
        for (int t = 0; t < T; ++t) {
            if (!ep.mask[row + t]) break;
            const double al = ep.a_lat[row + t], ao = ep.a_lon[row + t];
            double jl = 0.0, jo = 0.0;
            if (have_prev) {
                jl = (al - prev_lat) / dt;
                jo = (ao - prev_lon) / dt;
            }
            cacc += cw.w_accel * (al * al + ao * ao) + cw.w_jerk * (jl * jl + jo * jo);
            prev_lat = al;
            prev_lon = ao;
            have_prev = true;
            ++live;
        }
        const double comfort = live == 0 ? 1.0 : exp(-cacc / double(live));
        double score = map_score(rel, bb.progress);
        score *= map_score(coll, bb.collision);
        score *= map_score(off, bb.off_route);
        score *= map_score(stop, bb.stop_line);
        score *= map_score(light, bb.traffic_light);
        score *= map_score(comfort, bb.comfort);
        if (out.relative_progress_raw) out.relative_progress_raw[b] = raw;
        if (out.relative_progress) out.relative_progress[b] = rel;
        if (out.collision_free) out.collision_free[b] = coll;
        if (out.off_route_free) out.off_route_free[b] = off;
        if (out.stop_line_free) out.stop_line_free[b] = stop;
        if (out.traffic_light_free) out.traffic_light_free[b] = light;
        if (out.mixed_comfort) out.mixed_comfort[b] = comfort;
        if (out.scenario_score) out.scenario_score[b] = score;
        if (out.degenerate) out.degenerate[b] = degenerate ? 1 : 0;
        if (out.failed) out.failed[b] = failed ? 1 : 0;
        if (out.goal_reached) out.goal_reached[b] = goal ? 1 : 0;
        if (degenerate) {
            acc[1] += 1.0;
            continue;
        }
        acc[0] += 1.0;
        acc[2] += score;
        acc[3] += rel;
        acc[4] += raw;
        acc[5] += coll;
        acc[6] += off;
        acc[7] += stop;
        acc[8] += light;
        acc[9] += comfort;
        acc[10] += failed ? 1.0 : 0.0;
        acc[11] += goal ? 1.0 : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kAggLen; ++k) red[k][threadIdx.x] = acc[k];
    __syncthreads();
    for (int half = kMetricsThreads / 2; half > 0; half >>= 1) {
        if (threadIdx.x < half)
            for (int k = 0; k < kAggLen; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + half];
        __syncthreads();
    }
    if (threadIdx.x < kAggLen) part[size_t(blockIdx.x) * kAggLen + threadIdx.x] = red[threadIdx.x][0];
}

// Block partials summed in block order (deterministic for a given B).
__global__ void k_metrics_sum(const double* part, int nblk, double* sums) {
    const int k = threadIdx.x;
    if (k >= kAggLen) return;
    double s = 0.0;
    for (int i = 0; i < nblk; ++i) s += part[size_t(i) * kAggLen + k];
    sums[k] = s;
}

}  // namespace

#ifdef ZS_PATHSTATS
extern "C" __attribute__((visibility("default"))) int zsimdbg_pathstats(unsigned long long* out, int reset, unsigned* rowcyc, int nrows) {
    if (cudaDeviceSynchronize() != cudaSuccess) return 1;
    if (cudaMemcpyFromSymbol(out, g_pstats, sizeof(g_pstats)) != cudaSuccess) return 1;
    if (rowcyc && nrows > 0 &&
        cudaMemcpyFromSymbol(rowcyc, g_rowcyc, sizeof(unsigned) * 24 * size_t(nrows < kMaxStatRows ? nrows : kMaxStatRows)) !=
            cudaSuccess)
        return 1;
    if (reset) {
        static const unsigned long long z[32] = {};
        if (cudaMemcpyToSymbol(g_pstats, z, sizeof(z)) != cudaSuccess) return 1;
    }
    return 0;
}
#endif

// Big CTAs keep more warps in phase (one block barrier per row: a shared
// instruction stream; measured C2 +27%, C1 +2% over 4-warp CTAs)
int step_observe_warps(const KernelArgs& a) {
    const size_t per_warp = warp_layout(a.pk.d.A, a.cand_cap, a.cfg.n_agents, a.pk.d.NS, max(a.pk.d.PC, a.pk.d.RC)).total;
    return per_warp * kCtaWarpsBig <= 200 * 1024 ? kCtaWarpsBig : kCtaWarpsSmall;
}

size_t smem_bytes(const KernelArgs& a) {
    return size_t(warp_layout(a.pk.d.A, a.cand_cap, a.cfg.n_agents, a.pk.d.NS, max(a.pk.d.PC, a.pk.d.RC)).total) *
           size_t(step_observe_warps(a));
}

static int grid_for(const KernelArgs& a, int wpb = kThreads / 32) {
    const int rows = (a.row_hi > 0 ? a.row_hi : a.pk.d.B) - a.row_lo;
    return rows > 0 ? (rows + wpb - 1) / wpb : 1;
}

// Persistent grid: as many CTAs as fit on the device at once (each warp then
// walks rows with a stride), capped by the work.
// The smem attribute and occupancy of a (kernel, smem) pair are queried once.
struct LaunchCfg {
    const void* fn;
    size_t smem;
    int dev, per_sm;
};

static int blocks_per_sm(const void* fn, size_t smem, int threads) {
    static std::mutex mu;
    static std::vector<LaunchCfg> cache;     // occupancy per (kernel, smem, device)
    static std::vector<LaunchCfg> attr_max;  // largest dynamic smem attribute set per (kernel, device)
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    // the attribute only ever grows: a smaller later request must not shrink
    // it under another Env's larger launches
    LaunchCfg* am = nullptr;
    for (auto& c : attr_max)
        if (c.fn == fn && c.dev == dev) am = &c;
    if (!am || am->smem < smem) {
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) return -1;
        if (am)
            am->smem = smem;
        else
            attr_max.push_back({fn, smem, dev, 0});
    }
    for (const auto& c : cache)
        if (c.fn == fn && c.smem == smem && c.dev == dev) return c.per_sm;
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    cache.push_back({fn, smem, dev, per_sm});
    return per_sm;
}

static int sm_count() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
}

template <class K>
static int persistent_grid(K kern, const KernelArgs& a, size_t smem, int warps) {
    int per_sm = blocks_per_sm(reinterpret_cast<const void*>(kern), smem, 32 * warps);
    if (per_sm < 1) per_sm = 1;
    int g = sm_count() * per_sm;
    int need = grid_for(a, warps);
    return g < need ? g : need;
}

// Several waves of rows: the rows run out of phase, so the observation parts
// go to separate, smaller kernels.
bool observe_split(const KernelArgs& a, int policy) {
    if (policy == 1) return false;
    if (policy == 2) return true;
    KernelArgs t = a;
    t.lay = warp_layout(t.pk.d.A, t.cand_cap, t.cfg.n_agents, t.pk.d.NS, max(t.pk.d.PC, t.pk.d.RC));
    const int warps = step_observe_warps(t);
    const void* fn = warps == kCtaWarpsBig
                         ? reinterpret_cast<const void*>(k_step_observe<true, kObsAll, false, kCtaWarpsBig>)
                         : reinterpret_cast<const void*>(k_step_observe<true, kObsAll, false, kCtaWarpsSmall>);
    int per_sm = blocks_per_sm(fn, smem_bytes(t), 32 * warps);
    if (per_sm < 1) per_sm = 1;
    const int sms = sm_count();
    // measured with the in-phase 14-warp CTAs and the split kernels' uniform
    // warp index: ego rows split beyond three waves (split vs fused: 1 wave
    // +3%, 2 waves +2.3%, 4 waves -1.3%, C4 shard (4 waves, 128 agents) -4%,
    // C3 16 waves -6%, C4 32 waves -11%); controlled rows (C2) beyond 8
    // waves (16 waves -29%, 126: -43%)
    const long long wave = (long long)sms * per_sm * warps;
    return a.pk.d.B > (a.pk.row_actor == nullptr ? 3 : 8) * wave;
}

template <int W>
static cudaError_t launch_step_observe_w(const KernelArgs& a, int mode, int policy, cudaStream_t stream) {
    auto launch = [&](auto kern, KernelArgs am, bool topk, int warps = W) -> cudaError_t {
        if (!topk) am.cand_cap = 0;  // no top-k buffers in kernels without the map part
        am.lay = warp_layout(am.pk.d.A, am.cand_cap, am.cfg.n_agents, am.pk.d.NS, max(am.pk.d.PC, am.pk.d.RC));
        const size_t smem = size_t(am.lay.total) * warps;
        if (blocks_per_sm(reinterpret_cast<const void*>(kern), smem, 32 * warps) < 0) return cudaErrorInvalidValue;
        const int g = persistent_grid(kern, am, smem, warps);
        kern<<<g, 32 * warps, smem, stream>>>(am);
        return cudaGetLastError();
    };
    const bool split = mode != kModeStep && observe_split(a, policy);
    // recording / scripted actions (zsim_rollout) use their own instantiations
    const bool rec = a.ep.reward != nullptr || a.act_len != 0;
    switch (mode) {
        case kModeStep:
            return rec ? launch(k_step_observe<true, 0, true, W>, a, false)
                       : launch(k_step_observe<true, 0, false, W>, a, false);
        case kModeObserve: {
            if (!split) return launch(k_step_observe<false, kObsAll, false, W>, a, true);
            cudaError_t e = launch(k_step_observe<false, kObsAgents, false, W>, a, false);
            if (e != cudaSuccess) return e;
            if (W == kCtaWarpsBig)
                return launch(k_step_observe<false, kObsMap, false, kCtaWarpsMap, kMapWarpsPerSm>, a, true, kCtaWarpsMap);
            return launch(k_step_observe<false, kObsMap, false, W>, a, true);
        }
        default: {
            if (!split) {
                // at most 32 agents (C1): the instance without the > 32-agent
                // paths (27% less code; measured C1 -0.55%)
                if (W == kCtaWarpsBig && a.pk.d.A <= 32)
                    return rec ? launch(k_step_observe<true, kObsAll, true, W, 28, true>, a, true)
                               : launch(k_step_observe<true, kObsAll, false, W, 28, true>, a, true);
                return rec ? launch(k_step_observe<true, kObsAll, true, W>, a, true)
                           : launch(k_step_observe<true, kObsAll, false, W>, a, true);
            }
            // step + agents (the agent boxes at t+1 are reused), then the map
            // parts on the post-step state
            // controlled rows (C2, many waves): 16-warp step + agents CTAs at
            // 64 registers (measured C2 -2.2%; ego batches: C3 -0.5%, but the
            // 4-wave C4 shard +5% from the coarser last wave)
            cudaError_t e;
            const bool ctl16 = W == kCtaWarpsBig && a.pk.row_actor != nullptr &&
                               size_t(warp_layout(a.pk.d.A, 0, a.cfg.n_agents, a.pk.d.NS, max(a.pk.d.PC, a.pk.d.RC)).total) *
                                       kCtaWarpsCtl <= 200 * 1024;
            if (ctl16)
                e = rec ? launch(k_step_observe<true, kObsAgents, true, kCtaWarpsCtl, kCtlWarpsPerSm>, a, false, kCtaWarpsCtl)
                        : launch(k_step_observe<true, kObsAgents, false, kCtaWarpsCtl, kCtlWarpsPerSm>, a, false, kCtaWarpsCtl);
            else
                e = rec ? launch(k_step_observe<true, kObsAgents, true, W>, a, false)
                        : launch(k_step_observe<true, kObsAgents, false, W>, a, false);
            if (e != cudaSuccess) return e;
            KernelArgs m = a;
            m.in = a.out;
            m.ep = zsim_episode_view{};
            m.act_len = 0;
            // the map kernel needs fewer registers (54 at 36 warps per SM,
            // no extra spills): 12-warp CTAs, three per SM (measured against
            // 28 warps: C3 -6%, C2 -3.6%, C4 shard -1.2%)
            if (W == kCtaWarpsBig)
                return launch(k_step_observe<false, kObsMap, false, kCtaWarpsMap, kMapWarpsPerSm>, m, true, kCtaWarpsMap);
            return launch(k_step_observe<false, kObsMap, false, W>, m, true);
        }
    }
}

cudaError_t launch_step_observe(const KernelArgs& a, int mode, int policy, cudaStream_t stream) {
    KernelArgs t = a;
    t.lay = warp_layout(t.pk.d.A, t.cand_cap, t.cfg.n_agents, t.pk.d.NS, max(t.pk.d.PC, t.pk.d.RC));
    return step_observe_warps(t) == kCtaWarpsBig ? launch_step_observe_w<kCtaWarpsBig>(a, mode, policy, stream)
                                                 : launch_step_observe_w<kCtaWarpsSmall>(a, mode, policy, stream);
}

cudaError_t launch_reset(const KernelArgs& a, int grid, cudaStream_t stream) {
    (void)grid;
    k_reset<<<grid_for(a), kThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_episode_stats(const KernelArgs& a, const double* initial_s, long long* out, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(long long) * kStatsLen, stream);
    if (e != cudaSuccess) return e;
    int grid = (a.pk.d.B + 255) / 256;
    if (grid > 148 * 4) grid = 148 * 4;
    k_episode_stats<<<grid, 256, 0, stream>>>(a, initial_s, out);
    return cudaGetLastError();
}

static int metrics_blocks(int B) {
    int g = (B + kMetricsThreads - 1) / kMetricsThreads;
    return g < 148 * 2 ? (g > 0 ? g : 1) : 148 * 2;
}

int metrics_scratch_doubles(int B) { return metrics_blocks(B) * kAggLen; }

// ---------------------------------------------------------------------------
// train::cut_sequences (replay.cpp:8-52)
// ---------------------------------------------------------------------------
// Row b yields one sequence per window start t0 = 0, L, 2L, ... until the
// first masked start (mask is 1 up to the row's first done step, then 0).
__global__ void k_seq_count(int B, int T, int L, const uint8_t* mask, int32_t* n) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
        int c = 0;
        for (int t0 = 0; t0 < T && mask[size_t(b) * T + t0]; t0 += L) ++c;
        n[b] = c;
    }
}

// exclusive scan of n[0..B) in place into offsets, n[B] = total (one CTA,
// each thread a contiguous chunk: deterministic)
__global__ void __launch_bounds__(1024) k_seq_scan(int B, int32_t* n, int32_t* count) {
    __shared__ int32_t part[1024];
    const int t = threadIdx.x, per = (B + 1023) / 1024;
    const int lo = min(B, t * per), hi = min(B, lo + per);
    int32_t s = 0;
    for (int i = lo; i < hi; ++i) s += n[i];
    part[t] = s;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const int32_t v = t >= o ? part[t - o] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    int32_t run = part[t] - s;
    for (int i = lo; i < hi; ++i) {
        const int32_t c = n[i];
        n[i] = run;
        run += c;
    }
    if (t == 1023) {
        n[B] = part[1023];
        *count = part[1023];
    }
}

__device__ __forceinline__ void warp_copy(float* dst, const float* src, int n, bool zero) {
    for (int i = lane_id(); i < n; i += 32) dst[i] = zero ? 0.f : src[i];
}

// one warp per row b: its sequences, step by step (TransitionSequence fill,
// replay.cpp:14-49; padded steps stay zero with mask 0)
__global__ void k_seq_fill(int B, int T, int L, const zsim_episode_view ep, const zsim_obs_view* obs,
                           const zsim_sequences_view out, int ka, int kr, int kl, const int32_t* off) {
    const int wpb = blockDim.x / 32;
    for (int b = blockIdx.x * wpb + (threadIdx.x >> 5); b < B; b += gridDim.x * wpb) {
        const int s0 = off[b], ns = off[b + 1] - s0;
        for (int w = 0; w < ns; ++w) {
            const int s = s0 + w, t0 = w * L;
            bool terminated = false;
            bool live = true;
            for (int k = 0; k < L; ++k) {
                const int t = t0 + k;
                const size_t src = size_t(b) * T + t;
                live = live && t < T && ep.mask[src];
                const size_t r = size_t(s) * L + k;  // output observation row
                const int tt = live ? t : 0;
                const zsim_obs_view& o = obs[tt];
                warp_copy(out.obs.active + r * 9, o.active + size_t(b) * 9, 9, !live);
                warp_copy(out.obs.agents + r * ka * 6, o.agents + size_t(b) * ka * 6, ka * 6, !live);
                warp_copy(out.obs.road + r * kr * 12, o.road + size_t(b) * kr * 12, kr * 12, !live);
                warp_copy(out.obs.route + r * kl * 5, o.route + size_t(b) * kl * 5, kl * 5, !live);
                warp_copy(out.obs.value_only + r * 2, o.value_only + size_t(b) * 2, 2, !live);
                if (lane_id() == 0) {
                    const size_t q = size_t(s) * L + k;
                    out.accel_idx[q] = live ? ep.accel_idx[src] : 0;
                    out.steer_idx[q] = live ? ep.steer_idx[src] : 0;
                    out.logmu[q] = live ? ep.logp[src] : 0.f;
                    out.reward[q] = live ? ep.reward[src] : 0.f;
                    out.done[q] = live ? ep.done[src] : 0;
                    out.mask[q] = live ? 1 : 0;
                }
                if (live && ep.done[src]) terminated = true;
            }
            if (lane_id() == 0) {
                const int next = t0 + L;
                float bs;
                if (terminated) {
                    bs = 0.f;
                } else if (next < T && ep.mask[size_t(b) * T + next]) {
                    bs = ep.value[size_t(b) * T + next];  // behaviour value at the next state
                } else {
                    bs = ep.bootstrap[b];
                }
                out.bootstrap[s] = bs;
                out.row[s] = b;
                out.t0[s] = t0;
            }
        }
    }
}

cudaError_t launch_cut_sequences(int B, int T, int L, const zsim_episode_view& ep, const zsim_obs_view* obs,
                                 const zsim_sequences_view& out, int ka, int kr, int kl, int32_t* scratch,
                                 cudaStream_t stream) {
    const int g = std::min(4096, (B + 255) / 256);
    k_seq_count<<<g, 256, 0, stream>>>(B, T, L, ep.mask, scratch);
    k_seq_scan<<<1, 1024, 0, stream>>>(B, scratch, out.count);
    k_seq_fill<<<std::min(8192, (B + 7) / 8), 256, 0, stream>>>(B, T, L, ep, obs, out, ka, kr, kl, scratch);
    return cudaGetLastError();
}

cudaError_t launch_episode_finalize(const KernelArgs& a, const double* initial_s, const double* logged,
                                    cudaStream_t stream) {
    int grid = (a.pk.d.B + 255) / 256;
    if (grid > 148 * 4) grid = 148 * 4;
    k_episode_finalize<<<grid > 0 ? grid : 1, 256, 0, stream>>>(a, initial_s, logged);
    return cudaGetLastError();
}

cudaError_t launch_episode_metrics(const KernelArgs& a, const zsim_score_bounds& bounds,
                                   const zsim_comfort_weights& weights, const zsim_metric_view& rows, double* sums,
                                   double* scratch, cudaStream_t stream) {
    const int nblk = metrics_blocks(a.pk.d.B);
    k_episode_metrics<<<nblk, kMetricsThreads, 0, stream>>>(a, bounds, weights, rows, scratch);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_metrics_sum<<<1, 32, 0, stream>>>(scratch, nblk, sums);
    return cudaGetLastError();
}

}  // namespace zs
