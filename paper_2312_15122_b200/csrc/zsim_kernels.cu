// zsim_kernels.cu -- sm_100a kernels for the batched simulator step.
//
// One CTA (128 threads, 4 warps) per scenario row.  Within a CTA:
//   * route projection: warps own lanes, lanes own segments; per-query argmin
//     by (d2, segment) with warp shuffles (roads.cpp:125-166);
//   * collision / agent features: threads own agents, 16-lane groups own the
//     16 edge pairs of obb_distance (geometry.cpp:65-88);
//   * top-k (road 128-of-P, route 64-of-R): fp32 keys in shared memory,
//     packed-counter histograms to find a threshold, compaction of the few
//     candidates that can make the cut, exact fp64 keys for those only, and a
//     shared-memory bitonic sort by (d2, index) -- the exact reference order
//     (roads.cpp:210-236, simcore.cpp:503-529).
// Everything compiles with -fmad=false so every fp64 expression rounds like
// the reference built with -ffp-contract=off.
#include <cuda_runtime.h>

#include <climits>

#include "zsim_geom.cuh"
#include "zsim_kernels.cuh"
#include "zsim_pack.cuh"

namespace zs {

namespace {

constexpr int NT = kThreads;
constexpr int NW = NT / 32;
constexpr int NQ = 5;  // projection queries per step: ego position + 4 inflated corners

struct LaneRes {
    double s, d, hw;
    int set;
};

struct Smem {
    // row state (pre-step, then post-step)
    double x, y, h, v, steer, proj_s, proj_d;
    uint64_t rng;
    int t, done, reason, events, in_corr;
    int skip;  // 1 = done pass-through, 2 = bad action
    // step scratch
    double accel, rate;
    double nx, ny, nh, nv, nsteer;
    double qx[NQ], qy[NQ];
    Box ebox;
    double ebx[4], eby[4];
    LaneRes lres[kMaxLanes][NQ];
    double p1s, p1d;
    int p1_in;
    // observe scratch
    double oc, os;
    int n_sel;
    // top-k scratch
    unsigned long long hist[NW][4];
    float lo, hi, tcand;
    int below, round_done, ccount, overflow, nvalid;
    double red_key[NW];
    int red_idx[NW];
};

__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Dynamic shared-memory carve-up (host mirror: smem_bytes()).
struct Dyn {
    float* akey;   // [key_cap] fp32 approximate keys
    int* cidx;     // [cand_cap] candidate indices
    double* ckey;  // [cand_cap] exact fp64 keys
    double* agx;   // [A*4] agent corners
    double* agy;
    double* agd;   // [A] agent bbox distance (or +inf if invalid)
    int* agov;     // [A] -1 invalid, 0 separate, 1 overlap
    int* sel;      // [Ka + Kr + Kl] selected indices
    unsigned char* sflag;  // [NS] pre-step stopped flags
};


__device__ Dyn carve(unsigned char* base, const KernelArgs& a) {
    Dyn d;
    size_t off = 0;
    d.ckey = reinterpret_cast<double*>(base + off);
    off += size_t(a.cand_cap) * 8;
    d.agx = reinterpret_cast<double*>(base + off);
    off += size_t(a.pk.d.A) * 4 * 8;
    d.agy = reinterpret_cast<double*>(base + off);
    off += size_t(a.pk.d.A) * 4 * 8;
    d.agd = reinterpret_cast<double*>(base + off);
    off += size_t(a.pk.d.A) * 8;
    d.akey = reinterpret_cast<float*>(base + off);
    off += size_t(a.key_cap) * 4;
    d.cidx = reinterpret_cast<int*>(base + off);
    off += size_t(a.cand_cap) * 4;
    d.agov = reinterpret_cast<int*>(base + off);
    off += size_t(a.pk.d.A) * 4;
    d.sel = reinterpret_cast<int*>(base + off);
    off += size_t(a.cfg.n_agents + a.cfg.n_road + a.cfg.n_route) * 4;
    d.sflag = base + off;
    return d;
}

// ---------------------------------------------------------------------------
// route projection of NQ query points (roads.cpp:125-166 / 192-198)
// ---------------------------------------------------------------------------
template <int Q>
__device__ void project_queries(const DevPack& pk, int b, Smem& sm) {
    const int L = pk.d.L, C = pk.d.C;
    const int nl = pk.n_lanes[b];
    for (int l = warp_id(); l < nl; l += NW) {
        const size_t base = (size_t(b) * L + l) * C;
        const double* X = pk.ln_x + base;
        const double* Y = pk.ln_y + base;
        const int nv = pk.ln_n[size_t(b) * L + l];
        double bd2[Q];
        int bi[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            bd2[q] = 1e300;
            bi[q] = INT_MAX;
        }
        for (int i = lane_id(); i + 1 < nv; i += 32) {
            double ax = X[i], ay = Y[i], bx = X[i + 1], by = Y[i + 1];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                double t;
                double d2 = seg_dist2(sm.qx[q], sm.qy[q], ax, ay, bx, by, &t);
                if (d2 < bd2[q]) {
                    bd2[q] = d2;
                    bi[q] = i;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                double od = __shfl_xor_sync(0xffffffffu, bd2[q], off);
                int oi = __shfl_xor_sync(0xffffffffu, bi[q], off);
                if (od < bd2[q] || (od == bd2[q] && oi < bi[q])) {
                    bd2[q] = od;
                    bi[q] = oi;
                }
            }
        }
        if (lane_id() == 0) {
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                LaneRes r;
                r.set = bi[q] != INT_MAX;
                r.s = r.d = r.hw = 0.0;
                if (r.set) {
                    int i = bi[q];
                    double t;
                    double d2 = seg_dist2(sm.qx[q], sm.qy[q], X[i], Y[i], X[i + 1], Y[i + 1], &t);
                    LaneHit h = lane_hit(sm.qx[q], sm.qy[q], X, Y, pk.ln_s + base, pk.ln_hw + base, i, d2, t);
                    r.s = h.s;
                    r.d = h.d;
                    r.hw = h.hw;
                }
                sm.lres[l][q] = r;
            }
        }
    }
}

// roads::project combination across lanes for query q (roads.cpp:147-166).
__device__ void combine_projection(const DevPack& pk, int b, const Smem& sm, int q, double& s, double& d,
                                   int& in_corr) {
    const int nl = pk.n_lanes[b];
    bool have = false;
    in_corr = 0;
    double bs = 0.0, bdd = 0.0;
    uint32_t bid = 0;
    for (int l = 0; l < nl; ++l) {
        const LaneRes& r = sm.lres[l][q];
        if (!r.set) continue;
        if (fabs(r.d) <= r.hw) in_corr = 1;
        uint32_t id = pk.ln_id[size_t(b) * pk.d.L + l];
        if (!have || fabs(r.d) < fabs(bdd) || (fabs(r.d) == fabs(bdd) && id < bid)) {
            bs = r.s;
            bdd = r.d;
            bid = id;
            have = true;
        }
    }
    s = clampd(bs, 0.0, pk.route_len[b]);
    d = bdd;
}

// ---------------------------------------------------------------------------
// block reductions
// ---------------------------------------------------------------------------
__device__ float block_max_f(float v, Smem& sm) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
    __syncthreads();
    if (lane_id() == 0) sm.red_key[warp_id()] = double(v);
    __syncthreads();
    float m = float(sm.red_key[0]);
    for (int w = 1; w < NW; ++w) m = fmaxf(m, float(sm.red_key[w]));
    __syncthreads();
    return m;
}

// (key, idx) lexicographic argmin across the block; result broadcast.
__device__ void block_argmin(double& key, int& idx, Smem& sm) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        double ok = __shfl_xor_sync(0xffffffffu, key, off);
        int oi = __shfl_xor_sync(0xffffffffu, idx, off);
        if (ok < key || (ok == key && oi < idx)) {
            key = ok;
            idx = oi;
        }
    }
    __syncthreads();
    if (lane_id() == 0) {
        sm.red_key[warp_id()] = key;
        sm.red_idx[warp_id()] = idx;
    }
    __syncthreads();
    key = sm.red_key[0];
    idx = sm.red_idx[0];
    for (int w = 1; w < NW; ++w) {
        if (sm.red_key[w] < key || (sm.red_key[w] == key && sm.red_idx[w] < idx)) {
            key = sm.red_key[w];
            idx = sm.red_idx[w];
        }
    }
    __syncthreads();
}

// Upper bound on |fp32 key - fp64 key| for points within sqrt(T)+1 of the
// query; `ep` is the fp32 rounding error of the query coordinates.
__device__ __forceinline__ double key_margin(double T, double ep) {
    double D = sqrt(T) + 1.0;
    double eta = ep + 0x1p-24 * (D + ep);
    double m = 2.0 * eta * (2.0 * D + eta);
    m += 0x1p-22 * (T + m) + 0x1p-50 * T;
    return m * 1.25 + 1e-30;
}

// Threshold k of the current histogram round: lo + (k+1)*w, capped at hi.
__device__ __forceinline__ float round_th(float lo, float w, float hi, int k) {
    return k >= 15 ? hi : fminf(hi, lo + float(k + 1) * w);
}

// ---------------------------------------------------------------------------
// block top-k by (exact fp64 d2, index) over n points given by `pts`
// (float2).  With `use_radius`, only points with exact d2 <= r2 qualify
// (roads.cpp:219-229).  Writes up to K indices to `sel` in order; returns the
// count.  All threads must call.
// ---------------------------------------------------------------------------
__device__ int block_topk(const float2* __restrict__ pts, int n, int K, double px, double py, bool use_radius,
                          double r2, const Dyn& ws, int key_cap, int cand_cap, int* sel, Smem& sm) {
    const int tid = threadIdx.x;
    const float pxf = float(px), pyf = float(py);
    const double ep = fmax(fabs(double(pxf) - px), fabs(double(pyf) - py));

    // 1. fp32 keys
    float kmax = 0.f;
    for (int i = tid; i < n; i += NT) {
        float2 p = pts[i];
        float dx = p.x - pxf, dy = p.y - pyf;
        float a = dx * dx + dy * dy;
        ws.akey[i] = a;
        kmax = fmaxf(kmax, a);
    }
    float hi;
    if (use_radius) {
        hi = __double2float_ru(r2 + key_margin(r2, ep));
    } else {
        hi = block_max_f(kmax, sm);  // also orders the akey writes
    }
    __syncthreads();

    // 2. histogram rounds over (lo, hi]: 16 buckets, packed 8-bit counters
    if (tid == 0) {
        sm.lo = -1.0f;
        sm.hi = hi;
        sm.below = 0;
        sm.round_done = 0;
    }
    __syncthreads();
    for (int round = 0; round < 3; ++round) {
        const float lo = sm.lo, rhi = sm.hi;
        const float w = (rhi - lo) * (1.0f / 16.0f);
        const float inv_w = w > 0.f ? 1.0f / w : 0.f;
        unsigned long long c0 = 0ull, c1 = 0ull;
        for (int i = tid; i < n; i += NT) {
            float a = ws.akey[i];
            if (a > lo && a <= rhi) {
                int bk = min(15, max(0, int((a - lo) * inv_w)));
                while (bk > 0 && a <= round_th(lo, w, rhi, bk - 1)) --bk;
                while (bk < 15 && a > round_th(lo, w, rhi, bk)) ++bk;
                unsigned long long one = 1ull << ((bk & 7) * 8);
                if (bk < 8)
                    c0 += one;
                else
                    c1 += one;
            }
        }
        // widen to 16-bit lanes: even/odd buckets
        unsigned long long h[4];
        h[0] = c0 & 0x00FF00FF00FF00FFull;         // buckets 0,2,4,6
        h[1] = (c0 >> 8) & 0x00FF00FF00FF00FFull;  // 1,3,5,7
        h[2] = c1 & 0x00FF00FF00FF00FFull;         // 8,10,12,14
        h[3] = (c1 >> 8) & 0x00FF00FF00FF00FFull;  // 9,11,13,15
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
            for (int k = 0; k < 4; ++k) h[k] += __shfl_xor_sync(0xffffffffu, h[k], off);
        }
        if (lane_id() == 0) {
#pragma unroll
            for (int k = 0; k < 4; ++k) sm.hist[warp_id()][k] = h[k];
        }
        __syncthreads();
        if (tid == 0) {
            int cnt[16];
            for (int k = 0; k < 16; ++k) cnt[k] = 0;
            for (int wi = 0; wi < NW; ++wi) {
                for (int k = 0; k < 4; ++k) {
                    unsigned long long v = sm.hist[wi][k];
                    for (int f = 0; f < 4; ++f) {
                        int bucket = (k >> 1) * 8 + f * 2 + (k & 1);
                        cnt[bucket] += int((v >> (16 * f)) & 0xFFFFull);
                    }
                }
            }
            int cum = sm.below;
            int kstar = -1;
            for (int k = 0; k < 16; ++k) {
                if (cum + cnt[k] >= K) {
                    kstar = k;
                    break;
                }
                cum += cnt[k];
            }
            if (kstar < 0) {
                // fewer than K points in (lo, hi] plus below: take everything up to hi
                sm.round_done = 2;
            } else {
                float nlo = kstar == 0 ? lo : round_th(lo, w, rhi, kstar - 1);
                float nhi = round_th(lo, w, rhi, kstar);
                sm.below = cum;
                sm.lo = nlo;
                sm.hi = nhi;
                // stop refining once the threshold bucket is small
                if (cnt[kstar] <= 24 || !(nhi > nlo)) sm.round_done = 1;
            }
        }
        __syncthreads();
        if (sm.round_done) break;
    }

    // 3. candidate bound
    if (tid == 0) {
        double tsel = double(sm.hi);
        double tc;
        if (sm.round_done == 2) {
            tc = double(hi);
        } else {
            double m = key_margin(tsel, ep);
            tc = tsel + 2.0 * m;
            if (use_radius && !(tsel + m <= r2)) tc = double(hi);
        }
        sm.tcand = __double2float_ru(tc);
        sm.ccount = 0;
        sm.overflow = 0;
        sm.nvalid = 0;
    }
    __syncthreads();

    // 4. compaction of candidates (warp ballot)
    const float tcand = sm.tcand;
    for (int base = 0; base < n; base += NT) {
        int i = base + tid;
        bool take = i < n && ws.akey[i] <= tcand;
        unsigned m = __ballot_sync(0xffffffffu, take);
        int wbase = 0;
        if (lane_id() == 0 && m) wbase = atomicAdd(&sm.ccount, __popc(m));
        wbase = __shfl_sync(0xffffffffu, wbase, 0);
        if (take) {
            int pos = wbase + __popc(m & ((1u << lane_id()) - 1u));
            if (pos < cand_cap) ws.cidx[pos] = i;
        }
    }
    __syncthreads();
    const int C = sm.ccount;
    if (C > cand_cap) {
        // Pathological crowding at the threshold: exact iterative selection.
        double pk = -1.0;
        int pi = -1;
        int nsel = 0;
        for (int k = 0; k < K; ++k) {
            double best = INFINITY;
            int bi = INT_MAX;
            for (int i = tid; i < n; i += NT) {
                float2 p = pts[i];
                double dx = double(p.x) - px, dy2 = double(p.y) - py;
                double e = dx * dx + dy2 * dy2;
                if (use_radius && !(e <= r2)) continue;
                bool after = e > pk || (e == pk && i > pi);
                if (after && (e < best || (e == best && i < bi))) {
                    best = e;
                    bi = i;
                }
            }
            block_argmin(best, bi, sm);
            if (bi == INT_MAX) break;
            if (tid == 0) sel[k] = bi;
            pk = best;
            pi = bi;
            ++nsel;
        }
        __syncthreads();
        return nsel;
    }

    // 5. exact keys for the candidates, padded to a power of two
    int N2 = 1;
    while (N2 < C) N2 <<= 1;
    for (int c = tid; c < N2; c += NT) {
        double e = INFINITY;
        int idx = INT_MAX;
        if (c < C) {
            idx = ws.cidx[c];
            float2 p = pts[idx];
            double dx = double(p.x) - px, dyy = double(p.y) - py;
            e = dx * dx + dyy * dyy;
            if (use_radius && !(e <= r2)) e = INFINITY;
            if (e < INFINITY) atomicAdd(&sm.nvalid, 1);
        }
        ws.ckey[c] = e;
        ws.cidx[c] = idx;
    }
    __syncthreads();

    // 6. bitonic sort by (key, idx)
    for (int k = 2; k <= N2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < N2; i += NT) {
                int ixj = i ^ j;
                if (ixj > i) {
                    double ka = ws.ckey[i], kb = ws.ckey[ixj];
                    int ia = ws.cidx[i], ib = ws.cidx[ixj];
                    bool a_gt = ka > kb || (ka == kb && ia > ib);
                    bool up = (i & k) == 0;
                    if (a_gt == up) {
                        ws.ckey[i] = kb;
                        ws.ckey[ixj] = ka;
                        ws.cidx[i] = ib;
                        ws.cidx[ixj] = ia;
                    }
                }
            }
            __syncthreads();
        }
    }

    // 7. emit (keys are sorted; non-qualifying candidates carry +inf and sort last)
    const int nsel = min(K, sm.nvalid);
    for (int c = tid; c < nsel; c += NT) sel[c] = ws.cidx[c];
    __syncthreads();
    return nsel;
}

// ---------------------------------------------------------------------------
// observe one row (simcore.cpp:423-538) from the state held in `sm`
// ---------------------------------------------------------------------------
__device__ void observe_row(const KernelArgs& a, int b, Smem& sm, const Dyn& dy) {
    const DevPack& pk = a.pk;
    const DevCfg& cfg = a.cfg;
    const int tid = threadIdx.x;
    const int Ka = cfg.n_agents, Kr = cfg.n_road, Kl = cfg.n_route;
    float* act = a.obs.active + size_t(b) * 9;
    float* agt = a.obs.agents + size_t(b) * Ka * 6;
    float* rd = a.obs.road + size_t(b) * Kr * 12;
    float* rt = a.obs.route + size_t(b) * Kl * 5;
    float* val = a.obs.value_only + size_t(b) * 2;
    int32_t* dbg = a.dbg ? a.dbg + size_t(b) * (Ka + Kr + Kl) : nullptr;

    if (sm.done) {
        // ObservationBatch::zero_row (simcore.cpp:37-43)
        for (int i = tid; i < 9; i += NT) act[i] = 0.f;
        for (int i = tid; i < Ka * 6; i += NT) agt[i] = 0.f;
        for (int i = tid; i < Kr * 12; i += NT) rd[i] = 0.f;
        for (int i = tid; i < Kl * 5; i += NT) rt[i] = 0.f;
        if (tid < 2) val[tid] = 0.f;
        if (dbg)
            for (int i = tid; i < Ka + Kr + Kl; i += NT) dbg[i] = -1;
        return;
    }

    const int t = sm.t;
    if (tid == 0) {
        sm.oc = cos(-sm.h);
        sm.os = sin(-sm.h);
        double c = cos(sm.h), s = sin(sm.h);
        Box eb;
        eb.cx = sm.x + c * cfg.ego_center_offset;
        eb.cy = sm.y + s * cfg.ego_center_offset;
        eb.hl = cfg.ego_length * 0.5;
        eb.hw = cfg.ego_width * 0.5;
        eb.c = c;
        eb.s = s;
        sm.ebox = eb;
        box_corners(eb, sm.ebx, sm.eby);

        // active features: roads::stop_info (roads.cpp:253-277), fill simcore.cpp:440-455
        double best_stop = 1e300;
        const int ns = pk.n_stops[b];
        for (int j = 0; j < ns; ++j) {
            double ahead = pk.st_s[size_t(b) * pk.d.NS + j] - sm.proj_s;
            if (ahead > 0.0 && ahead < best_stop) best_stop = ahead;
        }
        double best_light = 1e300;
        int best_k = -1;
        const int nlt = pk.n_lights[b];
        for (int k = 0; k < nlt; ++k) {
            double ahead = pk.lt_s[size_t(b) * pk.d.NL + k] - sm.proj_s;
            if (ahead > 0.0 && ahead < best_light) {
                best_light = ahead;
                best_k = k;
            }
        }
        int light = 3;
        if (best_k >= 0) {
            int nsteps = pk.num_steps[b];
            int step = t < nsteps - 1 ? t : nsteps - 1;
            step = step > 0 ? step : 0;
            light = pk.lt_state[(size_t(b) * pk.d.NL + best_k) * pk.d.T + step];
        }
        const double R = cfg.feature_radius;
        float f[9];
        for (int i = 0; i < 9; ++i) f[i] = 0.f;
        f[0] = float(sm.v);
        f[1] = float(sm.steer);
        f[2] = float(best_stop < 1e300 ? mind(best_stop, R) : R);
        f[3 + light] = 1.f;
        f[7] = float(best_k >= 0 ? mind(best_light, R) : R);
        f[8] = pk.speed_limit[b];
        for (int i = 0; i < 9; ++i) act[i] = f[i];
        // value-only (simcore.cpp:531-537)
        double gx = double(pk.goal_x[b]) - sm.x, gy = double(pk.goal_y[b]) - sm.y;
        val[0] = float(sqrt(gx * gx + gy * gy));
        val[1] = float(pk.horizon - t);
        sm.n_sel = 0;
    }
    __syncthreads();

    // ---- agents: obb_distance to every valid agent, sort by (dist, idx) ----
    const int A = pk.d.A, T = pk.d.T;
    const int na = pk.n_agents[b];
    const bool t_ok = t < pk.num_steps[b];
    const size_t aslice = (size_t(b) * T + (t_ok ? t : 0)) * A;
    for (int j = tid; j < na; j += NT) {
        int ov = -1;
        if (t_ok && pk.ag_valid[aslice + j]) {
            double h = double(pk.ag_h[aslice + j]);
            Box ab;
            ab.cx = double(pk.ag_x[aslice + j]);
            ab.cy = double(pk.ag_y[aslice + j]);
            ab.hl = double(pk.ag_len[size_t(b) * A + j]) * 0.5;
            ab.hw = double(pk.ag_wid[size_t(b) * A + j]) * 0.5;
            ab.c = cos(h);
            ab.s = sin(h);
            double* X = dy.agx + 4 * j;
            double* Y = dy.agy + 4 * j;
            box_corners(ab, X, Y);
            ov = boxes_overlap(sm.ebox, sm.ebx, sm.eby, ab, X, Y) ? 1 : 0;
            atomicAdd(&sm.n_sel, 1);
        }
        dy.agov[j] = ov;
    }
    __syncthreads();
    for (int base = 0; base < na * 16; base += NT) {
        int it = base + tid;
        int j = it >> 4, p = it & 15;
        double d2 = INFINITY;
        if (j < na && dy.agov[j] == 0) {
            d2 = box_edge_pair_dist2(sm.ebx, sm.eby, dy.agx + 4 * j, dy.agy + 4 * j, p >> 2, p & 3);
        }
#pragma unroll
        for (int off = 8; off > 0; off >>= 1) d2 = mind(d2, __shfl_xor_sync(0xffffffffu, d2, off));
        if (p == 0 && j < na) {
            int ov = dy.agov[j];
            dy.agd[j] = ov < 0 ? INFINITY : (ov == 1 ? 0.0 : sqrt(d2));
        }
    }
    __syncthreads();
    for (int j = tid; j < na; j += NT) {
        if (dy.agov[j] < 0) continue;
        double dj = dy.agd[j];
        int rank = 0;
        for (int k = 0; k < na; ++k) {
            if (dy.agov[k] < 0) continue;
            double dk = dy.agd[k];
            rank += (dk < dj || (dk == dj && k < j)) ? 1 : 0;
        }
        if (rank < Ka) dy.sel[rank] = j;
    }
    __syncthreads();
    const int nvalid_ag = sm.n_sel;
    const int nsel_ag = min(Ka, nvalid_ag);
    const double oc = sm.oc, os = sm.os, ex = sm.x, ey = sm.y, eh = sm.h;
    for (int k = tid; k < Ka; k += NT) {
        float f[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        int j = -1;
        if (k < nsel_ag) {
            j = dy.sel[k];
            double wx = double(pk.ag_x[aslice + j]) - ex, wy = double(pk.ag_y[aslice + j]) - ey;
            f[0] = float(oc * wx - os * wy);
            f[1] = float(os * wx + oc * wy);
            f[2] = float(wrap_angle(double(pk.ag_h[aslice + j]) - eh));
            f[3] = pk.ag_sp[aslice + j];
            f[4] = float(dy.agd[j]);
            f[5] = 1.f;
        }
        float2* o = reinterpret_cast<float2*>(agt + k * 6);
        o[0] = make_float2(f[0], f[1]);
        o[1] = make_float2(f[2], f[3]);
        o[2] = make_float2(f[4], f[5]);
        if (dbg) dbg[k] = j;
    }
    __syncthreads();

    // ---- road network points: nearest_features (roads.cpp:210-236) ----
    {
        const int n = pk.n_road[b];
        const float2* pts = pk.road_xy + size_t(b) * pk.d.P;
        const double R = cfg.feature_radius;
        int* sel = dy.sel + Ka;
        int nsel = block_topk(pts, n, Kr, ex, ey, true, R * R, dy, a.key_cap, a.cand_cap, sel, sm);
        const uint8_t* kd = pk.road_kd + size_t(b) * pk.d.P;
        for (int k = tid; k < Kr; k += NT) {
            float f[12];
#pragma unroll
            for (int i = 0; i < 12; ++i) f[i] = 0.f;
            int i = -1;
            if (k < nsel) {
                i = sel[k];
                float2 p = pts[i];
                double wx = double(p.x) - ex, wy = double(p.y) - ey;
                f[0] = float(oc * wx - os * wy);
                f[1] = float(os * wx + oc * wy);
                int kk = kd[i];
                f[2 + (kk & 15)] = 1.f;
                f[7 + (kk >> 4)] = 1.f;
                f[11] = 1.f;
            }
            float4* o = reinterpret_cast<float4*>(rd + k * 12);
            o[0] = make_float4(f[0], f[1], f[2], f[3]);
            o[1] = make_float4(f[4], f[5], f[6], f[7]);
            o[2] = make_float4(f[8], f[9], f[10], f[11]);
            if (dbg) dbg[Ka + k] = i;
        }
    }
    __syncthreads();

    // ---- route border points: top n_route by (d2, idx), no radius (simcore.cpp:503-529) ----
    {
        const int n = pk.n_route[b];
        const float2* pts = pk.route_xy + size_t(b) * pk.d.R;
        int* sel = dy.sel + Ka + Kr;
        int nsel = block_topk(pts, n, Kl, ex, ey, false, 0.0, dy, a.key_cap, a.cand_cap, sel, sm);
        const uint8_t* fl = pk.route_fl + size_t(b) * pk.d.R;
        for (int k = tid; k < Kl; k += NT) {
            float f[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
            int i = -1;
            if (k < nsel) {
                i = sel[k];
                float2 p = pts[i];
                double wx = double(p.x) - ex, wy = double(p.y) - ey;
                f[0] = float(oc * wx - os * wy);
                f[1] = float(os * wx + oc * wy);
                f[2] = (fl[i] & 1) ? 1.f : 0.f;
                f[3] = (fl[i] & 2) ? 1.f : 0.f;
                f[4] = 1.f;
            }
            float* o = rt + k * 5;
            for (int q = 0; q < 5; ++q) o[q] = f[q];
            if (dbg) dbg[Ka + Kr + k] = i;
        }
    }
}

// ---------------------------------------------------------------------------
// step one row (simcore.cpp:278-404); leaves the post-step state in `sm`
// ---------------------------------------------------------------------------
__device__ void step_row(const KernelArgs& a, int b, Smem& sm, const Dyn& dy) {
    const DevPack& pk = a.pk;
    const DevCfg& cfg = a.cfg;
    const int tid = threadIdx.x;
    const int ns = pk.n_stops[b];
    const int soff = pk.stop_off[b];

    if (tid == 0) {
        sm.skip = sm.done ? 1 : 0;
        if (!sm.done) {
            int ai = a.accel[b], si = a.steer[b];
            if (ai < 0 || ai >= cfg.n_accel || si < 0 || si >= cfg.n_steer) {
                atomicOr(a.err, 1);
                sm.skip = 2;
            } else {
                sm.accel = cfg.accel_bins[ai];
                sm.rate = cfg.steer_bins[si];
                // dyn::bicycle_step (dynamics.cpp:10-19)
                const double dt = pk.dt;
                double c = cos(sm.h), s = sin(sm.h);
                sm.nx = sm.x + sm.v * c * dt;
                sm.ny = sm.y + sm.v * s * dt;
                sm.nh = wrap_angle(sm.h + sm.v / cfg.wheelbase * tan(sm.steer) * dt);
                sm.nv = maxd(sm.v + sm.accel * dt, cfg.v_min);
                sm.nsteer = clampd(sm.steer + sm.rate * dt, -cfg.delta_max, cfg.delta_max);
                // ego_box(e1) (simcore.cpp:156-160) and its inflated corners (roads.cpp:202-208)
                double c1 = cos(sm.nh), s1 = sin(sm.nh);
                Box eb;
                eb.cx = sm.nx + c1 * cfg.ego_center_offset;
                eb.cy = sm.ny + s1 * cfg.ego_center_offset;
                eb.hl = cfg.ego_length * 0.5;
                eb.hw = cfg.ego_width * 0.5;
                eb.c = c1;
                eb.s = s1;
                sm.ebox = eb;
                box_corners(eb, sm.ebx, sm.eby);
                Box inf = eb;
                inf.hl = eb.hl + cfg.footprint_margin;
                inf.hw = eb.hw + cfg.footprint_margin;
                double X[4], Y[4];
                box_corners(inf, X, Y);
                sm.qx[0] = sm.nx;
                sm.qy[0] = sm.ny;
                for (int k = 0; k < 4; ++k) {
                    sm.qx[k + 1] = X[k];
                    sm.qy[k + 1] = Y[k];
                }
            }
        }
    }
    for (int j = tid; j < ns; j += NT) dy.sflag[j] = a.in.stopped_flags[soff + j];
    __syncthreads();

    if (sm.skip) {
        // absorbing pass-through (simcore.cpp:281-299); bad-action rows are left unchanged
        if (tid == 0) {
            a.out.x[b] = sm.x;
            a.out.y[b] = sm.y;
            a.out.heading[b] = sm.h;
            a.out.v[b] = sm.v;
            a.out.steering[b] = sm.steer;
            a.out.t[b] = sm.t;
            a.out.done[b] = uint8_t(sm.done);
            a.out.reason[b] = uint8_t(sm.reason);
            a.out.rng[b] = sm.rng;
            a.out.proj_s[b] = sm.proj_s;
            a.out.proj_d[b] = sm.proj_d;
            a.out.proj_in_corridor[b] = uint8_t(sm.in_corr);
            a.out.events[b] = uint8_t(sm.events);
            a.so.reward[b] = 0.f;
            a.so.event[b] = 0;
            a.so.s[b] = float(sm.proj_s);
            a.so.a_lat[b] = 0.f;
            a.so.a_lon[b] = 0.f;
            a.so.v[b] = float(sm.v);
        }
        for (int j = tid; j < ns; j += NT) a.out.stopped_flags[soff + j] = dy.sflag[j];
        __syncthreads();
        return;
    }

    // projection of e1 and of the 4 inflated footprint corners
    project_queries<NQ>(pk, b, sm);

    // collision against agents valid at t+1 (simcore.cpp:323-331)
    int hit = 0;
    {
        const int t1 = sm.t + 1;
        const int na = pk.n_agents[b];
        if (t1 < pk.num_steps[b]) {
            const int A = pk.d.A;
            const size_t slice = (size_t(b) * pk.d.T + t1) * A;
            for (int j = tid; j < na; j += NT) {
                if (!pk.ag_valid[slice + j]) continue;
                double h = double(pk.ag_h[slice + j]);
                Box ab;
                ab.cx = double(pk.ag_x[slice + j]);
                ab.cy = double(pk.ag_y[slice + j]);
                ab.hl = double(pk.ag_len[size_t(b) * A + j]) * 0.5;
                ab.hw = double(pk.ag_wid[size_t(b) * A + j]) * 0.5;
                ab.c = cos(h);
                ab.s = sin(h);
                double X[4], Y[4];
                box_corners(ab, X, Y);
                if (boxes_overlap(sm.ebox, sm.ebx, sm.eby, ab, X, Y)) hit = 1;
            }
        }
    }
    hit = __syncthreads_or(hit);

    if (tid == 0) {
        double p1s, p1d;
        int p1_in;
        combine_projection(pk, b, sm, 0, p1s, p1d, p1_in);
        // footprint_on_route (roads.cpp:192-208)
        bool on_route = true;
        const int nl = pk.n_lanes[b];
        for (int q = 1; q < NQ; ++q) {
            bool any = false;
            for (int l = 0; l < nl; ++l) {
                const LaneRes& r = sm.lres[l][q];
                if (r.set && fabs(r.d) <= r.hw) any = true;
            }
            if (!any) on_route = false;
        }
        const double dt = pk.dt;
        const double progress = p1s - sm.proj_s;
        const double a_lat = sm.v * sm.v * tan(sm.steer) / cfg.wheelbase;
        const double a_lon = sm.accel;
        double reward = cfg.w_progress * progress -
                        cfg.w_speed * maxd(0.0, sm.nv - double(pk.speed_limit[b])) * dt -
                        cfg.w_lat * a_lat * a_lat * dt - cfg.w_lon * a_lon * a_lon * dt;
        const bool hit_collision = hit != 0;
        const bool hit_off_route = !on_route;
        bool hit_red = false;
        {
            int nsteps = pk.num_steps[b];
            int t_light = sm.t < nsteps - 1 ? sm.t : nsteps - 1;
            const int nlt = pk.n_lights[b];
            for (int k = 0; k < nlt; ++k) {
                double ls = pk.lt_s[size_t(b) * pk.d.NL + k];
                if (sm.proj_s < ls && ls <= p1s) {
                    if (pk.lt_state[(size_t(b) * pk.d.NL + k) * pk.d.T + t_light] == 0) hit_red = true;
                }
            }
        }
        bool hit_stop = false;
        for (int j = 0; j < ns; ++j) {
            double ss = pk.st_s[size_t(b) * pk.d.NS + j];
            if (sm.proj_s < ss && ss <= p1s) {
                if (sm.v > cfg.stop_cross_speed && !dy.sflag[j]) hit_stop = true;
            }
        }
        const bool hit_goal = fabs(p1s - pk.goal_s[b]) <= cfg.goal_radius;
        int reason = 0;
        if (hit_collision)
            reason = 1;
        else if (hit_off_route)
            reason = 2;
        else if (hit_red)
            reason = 3;
        else if (hit_stop)
            reason = 4;
        else if (hit_goal)
            reason = 5;
        int events = sm.events;
        if (cfg.disable_dones) {
            if (hit_collision) events |= 1;
            if (hit_off_route) events |= 2;
            if (hit_red) events |= 4;
            if (hit_stop) events |= 8;
            if (hit_goal) events |= 16;
        } else if (reason != 0) {
            events |= 1 << (reason - 1);
            if (reason != 5) reward -= cfg.terminal_penalty;
        }
        const int done = (!cfg.disable_dones && reason != 0) ? 1 : 0;
        a.out.x[b] = sm.nx;
        a.out.y[b] = sm.ny;
        a.out.heading[b] = sm.nh;
        a.out.v[b] = sm.nv;
        a.out.steering[b] = sm.nsteer;
        a.out.t[b] = sm.t + 1;
        a.out.done[b] = uint8_t(done);
        a.out.reason[b] = uint8_t(done ? reason : 0);
        a.out.rng[b] = sm.rng;
        a.out.proj_s[b] = p1s;
        a.out.proj_d[b] = p1d;
        a.out.proj_in_corridor[b] = uint8_t(p1_in);
        a.out.events[b] = uint8_t(events);
        a.so.reward[b] = float(reward);
        a.so.event[b] = uint8_t(reason);
        a.so.s[b] = float(p1s);
        a.so.a_lat[b] = float(a_lat);
        a.so.a_lon[b] = float(a_lon);
        a.so.v[b] = float(sm.nv);
        // the row state becomes the post-step state for a fused observe
        sm.x = sm.nx;
        sm.y = sm.ny;
        sm.h = sm.nh;
        sm.v = sm.nv;
        sm.steer = sm.nsteer;
        sm.t = sm.t + 1;
        sm.done = done;
        sm.reason = done ? reason : 0;
        sm.proj_s = p1s;
        sm.proj_d = p1d;
        sm.in_corr = p1_in;
        sm.events = events;
    }
    __syncthreads();
    // stopped-flag update with the post-step state (simcore.cpp:390-396)
    for (int j = tid; j < ns; j += NT) {
        double ahead = pk.st_s[size_t(b) * pk.d.NS + j] - sm.proj_s;
        uint8_t f = dy.sflag[j];
        if (ahead >= 0.0 && ahead <= cfg.stop_zone && sm.v < cfg.stop_slow_speed) f = 1;
        a.out.stopped_flags[soff + j] = f;
    }
    __syncthreads();
}

__device__ void load_row(const zsim_state_view& in, int b, Smem& sm) {
    sm.x = in.x[b];
    sm.y = in.y[b];
    sm.h = in.heading[b];
    sm.v = in.v[b];
    sm.steer = in.steering[b];
    sm.t = in.t[b];
    sm.done = in.done[b];
    sm.reason = in.reason[b];
    sm.rng = in.rng[b];
    sm.proj_s = in.proj_s[b];
    sm.proj_d = in.proj_d[b];
    sm.in_corr = in.proj_in_corridor[b];
    sm.events = in.events[b];
}

template <bool STEP, bool OBS>
__global__ void __launch_bounds__(NT) k_step_observe(const KernelArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ Smem sm;
    const Dyn dy = carve(dsm, a);
    for (int b = blockIdx.x; b < a.pk.d.B; b += gridDim.x) {
        if (threadIdx.x == 0) load_row(a.in, b, sm);
        __syncthreads();
        if (STEP) step_row(a, b, sm, dy);
        if (OBS) observe_row(a, b, sm, dy);
        __syncthreads();
    }
}

// Env::init_state (simcore.cpp:237-276).
__global__ void __launch_bounds__(NT) k_reset(const KernelArgs a) {
    __shared__ Smem sm;
    const DevPack& pk = a.pk;
    const DevCfg& cfg = a.cfg;
    for (int b = blockIdx.x; b < pk.d.B; b += gridDim.x) {
        if (threadIdx.x == 0) {
            sm.qx[0] = pk.init_x[b];
            sm.qy[0] = pk.init_y[b];
        }
        __syncthreads();
        project_queries<1>(pk, b, sm);
        __syncthreads();
        if (threadIdx.x == 0) {
            double s, d;
            int in;
            combine_projection(pk, b, sm, 0, s, d, in);
            sm.proj_s = s;
            a.out.x[b] = pk.init_x[b];
            a.out.y[b] = pk.init_y[b];
            a.out.heading[b] = pk.init_h[b];
            a.out.v[b] = pk.init_v[b];
            a.out.steering[b] = pk.init_steer[b];
            a.out.t[b] = 0;
            a.out.done[b] = 0;
            a.out.reason[b] = 0;
            a.out.rng[b] = reset_rng_state(a.seed, uint64_t(b));
            a.out.proj_s[b] = s;
            a.out.proj_d[b] = d;
            a.out.proj_in_corridor[b] = uint8_t(in);
            a.out.events[b] = 0;
        }
        __syncthreads();
        const int ns = pk.n_stops[b];
        const int soff = pk.stop_off[b];
        for (int j = threadIdx.x; j < ns; j += NT) {
            double ahead = pk.st_s[size_t(b) * pk.d.NS + j] - sm.proj_s;
            bool st = ahead >= 0.0 && ahead <= cfg.stop_zone && pk.init_v[b] < cfg.stop_slow_speed;
            a.out.stopped_flags[soff + j] = st ? 1 : 0;
        }
        __syncthreads();
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
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if ((threadIdx.x & 31) == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&acc[k]), (unsigned long long)v);
    }
    __syncthreads();
    if (threadIdx.x < kStatsLen)
        atomicAdd(reinterpret_cast<unsigned long long*>(&out[threadIdx.x]), (unsigned long long)acc[threadIdx.x]);
}

}  // namespace

cudaError_t launch_episode_stats(const KernelArgs& a, const double* initial_s, long long* out, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(long long) * kStatsLen, stream);
    if (e != cudaSuccess) return e;
    int grid = (a.pk.d.B + 255) / 256;
    if (grid > 148 * 4) grid = 148 * 4;
    k_episode_stats<<<grid, 256, 0, stream>>>(a, initial_s, out);
    return cudaGetLastError();
}

size_t smem_bytes(const KernelArgs& a) {
    size_t off = 0;
    off += size_t(a.cand_cap) * 8;
    off += size_t(a.pk.d.A) * 4 * 8 * 2;
    off += size_t(a.pk.d.A) * 8;
    off += size_t(a.key_cap) * 4;
    off += size_t(a.cand_cap) * 4;
    off += size_t(a.pk.d.A) * 4;
    off += size_t(a.cfg.n_agents + a.cfg.n_road + a.cfg.n_route) * 4;
    off += size_t(a.pk.d.NS) + 16;
    return (off + 15) / 16 * 16;
}

cudaError_t launch_step_observe(const KernelArgs& a, int mode, int grid, cudaStream_t stream) {
    size_t smem = smem_bytes(a);
    static bool attr_set[3] = {false, false, false};
    auto launch = [&](auto kern, int m) -> cudaError_t {
        if (!attr_set[m] || smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            if (e != cudaSuccess) return e;
            attr_set[m] = true;
        }
        kern<<<grid, NT, smem, stream>>>(a);
        return cudaGetLastError();
    };
    switch (mode) {
        case kModeStep: return launch(k_step_observe<true, false>, 0);
        case kModeObserve: return launch(k_step_observe<false, true>, 1);
        default: return launch(k_step_observe<true, true>, 2);
    }
}

cudaError_t launch_reset(const KernelArgs& a, int grid, cudaStream_t stream) {
    k_reset<<<grid, NT, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace zs
