/*
 * zsim_oracle.c -- TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference hot path (see zsim_oracle.h).  Compile with -ffp-contract=off.
 * Reference paths are relative to /root/reference/proj/src/core/.
 */
#include "zsim_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

const char* zor_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

/* ------------------------------------------------------------------ math */

static const double TWO_PI = 6.283185307179586476925286766559;
static const double PI_ = 3.14159265358979323846;

/* common.hpp:53-59 */
static double wrap_angle(double a) {
    a = fmod(a, TWO_PI);
    if (a <= -PI_) a += TWO_PI;
    if (a > PI_) a -= TWO_PI;
    return a;
}
static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }
static double mind(double a, double b) { return b < a ? b : a; }
static double maxd(double a, double b) { return a < b ? b : a; }

typedef struct {
    double x, y;
} V2;

/* geometry.cpp:17-25 */
static double psd2(V2 p, V2 a, V2 b, double* tout) {
    double abx = b.x - a.x, aby = b.y - a.y;
    double len2 = abx * abx + aby * aby;
    double t = 0.0;
    if (len2 > 0.0) t = clampd(((p.x - a.x) * abx + (p.y - a.y) * aby) / len2, 0.0, 1.0);
    double cx = a.x + abx * t, cy = a.y + aby * t;
    if (tout) *tout = t;
    double dx = p.x - cx, dy = p.y - cy;
    return dx * dx + dy * dy;
}

/* oriented box: centre, half extents, heading (geometry.hpp:30-38) */
typedef struct {
    V2 c;
    double hl, hw, h;
} Obb;

/* geometry.cpp:7-15 */
static void obb_corners(const Obb* b, V2 out[4]) {
    double c = cos(b->h), s = sin(b->h);
    double axx = c * b->hl, axy = s * b->hl, ayx = -s * b->hw, ayy = c * b->hw;
    out[0].x = b->c.x + axx + ayx;
    out[0].y = b->c.y + axy + ayy;
    out[1].x = b->c.x + axx - ayx;
    out[1].y = b->c.y + axy - ayy;
    out[2].x = b->c.x - axx - ayx;
    out[2].y = b->c.y - axy - ayy;
    out[3].x = b->c.x - axx + ayx;
    out[3].y = b->c.y - axy + ayy;
}

/* geometry.cpp:48-61 */
static int separated(V2 ax, const V2* a, const V2* b) {
    double amin = 1e300, amax = -1e300, bmin = 1e300, bmax = -1e300;
    for (int k = 0; k < 4; ++k) {
        double v = a[k].x * ax.x + a[k].y * ax.y;
        amin = mind(amin, v);
        amax = maxd(amax, v);
    }
    for (int k = 0; k < 4; ++k) {
        double v = b[k].x * ax.x + b[k].y * ax.y;
        bmin = mind(bmin, v);
        bmax = maxd(bmax, v);
    }
    return amax < bmin || bmax < amin;
}

/* geometry.cpp:65-75 */
static int obb_overlap(const Obb* a, const Obb* b) {
    V2 ca[4], cb[4];
    obb_corners(a, ca);
    obb_corners(b, cb);
    double cah = cos(a->h), sah = sin(a->h), cbh = cos(b->h), sbh = sin(b->h);
    V2 axes[4] = {{cah, sah}, {-sah, cah}, {cbh, sbh}, {-sbh, cbh}};
    for (int k = 0; k < 4; ++k)
        if (separated(axes[k], ca, cb)) return 0;
    return 1;
}

static double orient(V2 p, V2 q, V2 r) { return (q.x - p.x) * (r.y - p.y) - (q.y - p.y) * (r.x - p.x); }

/* geometry.cpp:27-42 */
static double segseg(V2 a0, V2 a1, V2 b0, V2 b1) {
    double o1 = orient(a0, a1, b0), o2 = orient(a0, a1, b1);
    double o3 = orient(b0, b1, a0), o4 = orient(b0, b1, a1);
    if (((o1 > 0) != (o2 > 0)) && ((o3 > 0) != (o4 > 0))) return 0.0;
    double d2 = psd2(a0, b0, b1, NULL);
    d2 = mind(d2, psd2(a1, b0, b1, NULL));
    d2 = mind(d2, psd2(b0, a0, a1, NULL));
    d2 = mind(d2, psd2(b1, a0, a1, NULL));
    return sqrt(d2);
}

/* geometry.cpp:77-88 */
static double obb_distance(const Obb* a, const Obb* b) {
    if (obb_overlap(a, b)) return 0.0;
    V2 ca[4], cb[4];
    obb_corners(a, ca);
    obb_corners(b, cb);
    double best = 1e300;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) best = mind(best, segseg(ca[i], ca[(i + 1) & 3], cb[j], cb[(j + 1) & 3]));
    return best;
}

/* -------------------------------------------------------------- scenario */

typedef struct {
    float len, wid;
    float *x, *y, *h, *sp;
    uint8_t* valid;
} Agent;
typedef struct {
    uint32_t id;
    float *l, *r;
    uint32_t nl, nr; /* float counts */
    float s0, s1;
} Lane;
typedef struct {
    uint8_t kind, dir;
    float* xy;
    uint32_t n;
} Feat;
typedef struct {
    float sx, sy;
    uint8_t* st;
} Light;
typedef struct {
    float px, py;
} Stop;
typedef struct {
    uint32_t nsteps;
    double dt;
    float *ex, *ey, *eh, *ev;
    uint32_t nag, nln, nft, nlt, nst;
    Agent* ag;
    Lane* ln;
    Feat* ft;
    Light* lt;
    Stop* st;
    float limit, gx, gy;
} Scen;

typedef struct {
    const uint8_t* p;
    const uint8_t* end;
    int bad;
} Cur;

static int need(Cur* c, size_t n) {
    if ((size_t)(c->end - c->p) < n) {
        c->bad = 1;
        return 0;
    }
    return 1;
}
static uint32_t rd_u32(Cur* c) {
    uint32_t v = 0;
    if (need(c, 4)) memcpy(&v, c->p, 4), c->p += 4;
    return v;
}
static uint8_t rd_u8(Cur* c) {
    uint8_t v = 0;
    if (need(c, 1)) v = *c->p++;
    return v;
}
static float rd_f32(Cur* c) {
    float v = 0;
    if (need(c, 4)) memcpy(&v, c->p, 4), c->p += 4;
    return v;
}
static void skip_str(Cur* c) {
    uint32_t n = rd_u32(c);
    if (need(c, n)) c->p += n;
}
static float* rd_f32s(Cur* c, uint32_t* n_out) {
    uint32_t n = rd_u32(c);
    if (n_out) *n_out = n;
    if (!need(c, (size_t)n * 4)) return NULL;
    float* v = (float*)malloc((size_t)(n ? n : 1) * 4);
    memcpy(v, c->p, (size_t)n * 4);
    c->p += (size_t)n * 4;
    return v;
}
static uint8_t* rd_u8s(Cur* c, uint32_t* n_out) {
    uint32_t n = rd_u32(c);
    if (n_out) *n_out = n;
    if (!need(c, n)) return NULL;
    uint8_t* v = (uint8_t*)malloc(n ? n : 1);
    memcpy(v, c->p, n);
    c->p += n;
    return v;
}

/* scenario_io.cpp:132-189 */
static int decode(Cur* c, double dt, Scen* s) {
    memset(s, 0, sizeof *s);
    s->dt = dt;
    skip_str(c);
    s->nsteps = rd_u32(c);
    s->ex = rd_f32s(c, NULL);
    s->ey = rd_f32s(c, NULL);
    s->eh = rd_f32s(c, NULL);
    s->ev = rd_f32s(c, NULL);
    s->nag = rd_u32(c);
    if (c->bad) return 0;
    s->ag = (Agent*)calloc(s->nag ? s->nag : 1, sizeof(Agent));
    for (uint32_t i = 0; i < s->nag && !c->bad; ++i) {
        skip_str(c);
        s->ag[i].len = rd_f32(c);
        s->ag[i].wid = rd_f32(c);
        s->ag[i].x = rd_f32s(c, NULL);
        s->ag[i].y = rd_f32s(c, NULL);
        s->ag[i].h = rd_f32s(c, NULL);
        s->ag[i].sp = rd_f32s(c, NULL);
        s->ag[i].valid = rd_u8s(c, NULL);
    }
    s->nln = rd_u32(c);
    if (c->bad) return 0;
    s->ln = (Lane*)calloc(s->nln ? s->nln : 1, sizeof(Lane));
    for (uint32_t i = 0; i < s->nln && !c->bad; ++i) {
        s->ln[i].id = rd_u32(c);
        s->ln[i].l = rd_f32s(c, &s->ln[i].nl);
        s->ln[i].r = rd_f32s(c, &s->ln[i].nr);
        s->ln[i].s0 = rd_f32(c);
        s->ln[i].s1 = rd_f32(c);
    }
    s->nft = rd_u32(c);
    if (c->bad) return 0;
    s->ft = (Feat*)calloc(s->nft ? s->nft : 1, sizeof(Feat));
    for (uint32_t i = 0; i < s->nft && !c->bad; ++i) {
        s->ft[i].kind = rd_u8(c);
        s->ft[i].dir = rd_u8(c);
        s->ft[i].xy = rd_f32s(c, &s->ft[i].n);
    }
    s->nlt = rd_u32(c);
    if (c->bad) return 0;
    s->lt = (Light*)calloc(s->nlt ? s->nlt : 1, sizeof(Light));
    for (uint32_t i = 0; i < s->nlt && !c->bad; ++i) {
        rd_u32(c);
        s->lt[i].sx = rd_f32(c);
        s->lt[i].sy = rd_f32(c);
        s->lt[i].st = rd_u8s(c, NULL);
    }
    s->nst = rd_u32(c);
    if (c->bad) return 0;
    s->st = (Stop*)calloc(s->nst ? s->nst : 1, sizeof(Stop));
    for (uint32_t i = 0; i < s->nst && !c->bad; ++i) {
        free(rd_f32s(c, NULL));
        s->st[i].px = rd_f32(c);
        s->st[i].py = rd_f32(c);
    }
    s->limit = rd_f32(c);
    s->gx = rd_f32(c);
    s->gy = rd_f32(c);
    return !c->bad && c->p == c->end;
}

static void free_scen(Scen* s) {
    free(s->ex), free(s->ey), free(s->eh), free(s->ev);
    for (uint32_t i = 0; i < s->nag; ++i)
        free(s->ag[i].x), free(s->ag[i].y), free(s->ag[i].h), free(s->ag[i].sp), free(s->ag[i].valid);
    for (uint32_t i = 0; i < s->nln; ++i) free(s->ln[i].l), free(s->ln[i].r);
    for (uint32_t i = 0; i < s->nft; ++i) free(s->ft[i].xy);
    for (uint32_t i = 0; i < s->nlt; ++i) free(s->lt[i].st);
    free(s->ag), free(s->ln), free(s->ft), free(s->lt), free(s->st);
}

/* ------------------------------------------------------------ route frame */

typedef struct {
    uint32_t id;
    int n;
    double *x, *y, *s, *hw;
} LF;
typedef struct {
    int nl;
    LF* l;
    double length;
    int nstops, nlights;
    int* stop_i;
    double* stop_s;
    int* light_i;
    double* light_s;
} Ctx;
typedef struct {
    double s, d;
    int in_corr;
} Proj;

static double dist2d(double ax, double ay, double bx, double by) {
    double dx = ax - bx, dy = ay - by;
    return sqrt(dx * dx + dy * dy);
}

/* roads.cpp:43-103 */
static int build_frame(const Scen* sc, Ctx* ctx) {
    ctx->nl = 0;
    ctx->length = 0.0;
    ctx->l = (LF*)calloc(sc->nln ? sc->nln : 1, sizeof(LF));
    for (uint32_t li = 0; li < sc->nln; ++li) {
        const Lane* ln = &sc->ln[li];
        int n = (int)(ln->nl / 2), nr = (int)(ln->nr / 2);
        if (n < 2 || nr < 2) return fail(1, "lane %u: border too short", ln->id);
        double* rarc = (double*)calloc((size_t)nr, sizeof(double));
        for (int i = 1; i < nr; ++i)
            rarc[i] = rarc[i - 1] + dist2d(ln->r[2 * i], ln->r[2 * i + 1], ln->r[2 * i - 2], ln->r[2 * i - 1]);
        double *cx = malloc(sizeof(double) * n), *cy = malloc(sizeof(double) * n), *hw = malloc(sizeof(double) * n),
               *s = malloc(sizeof(double) * n);
        for (int i = 0; i < n; ++i) {
            double lx = ln->l[2 * i], ly = ln->l[2 * i + 1], px, py;
            if (nr == n) {
                px = ln->r[2 * i];
                py = ln->r[2 * i + 1];
            } else { /* Polyline::at_fraction, roads.cpp:30-38 */
                double u = n > 1 ? (double)i / (double)(n - 1) : 0.0;
                double target = u * rarc[nr - 1];
                int k = 1;
                while (k + 1 < nr && rarc[k] < target) ++k;
                double seg = rarc[k] - rarc[k - 1];
                double t = seg > 0 ? (target - rarc[k - 1]) / seg : 0.0;
                t = clampd(t, 0.0, 1.0);
                double ax = ln->r[2 * k - 2], ay = ln->r[2 * k - 1];
                px = ax + (ln->r[2 * k] - ax) * t;
                py = ay + (ln->r[2 * k + 1] - ay) * t;
            }
            cx[i] = (lx + px) * 0.5;
            cy[i] = (ly + py) * 0.5;
            hw[i] = dist2d(lx, ly, px, py) * 0.5;
        }
        s[0] = (double)ln->s0;
        for (int i = 1; i < n; ++i) s[i] = s[i - 1] + dist2d(cx[i], cy[i], cx[i - 1], cy[i - 1]);
        LF* f = &ctx->l[ctx->nl];
        f->id = ln->id;
        f->x = malloc(sizeof(double) * n), f->y = malloc(sizeof(double) * n), f->s = malloc(sizeof(double) * n),
        f->hw = malloc(sizeof(double) * n);
        f->n = 0;
        double clip = (double)ln->s1;
        for (int i = 0; i < n; ++i) {
            if (s[i] > clip && f->n > 0) {
                double seg = s[i] - s[i - 1];
                if (seg > 0 && s[i - 1] < clip) {
                    double t = (clip - s[i - 1]) / seg;
                    f->x[f->n] = cx[i - 1] + (cx[i] - cx[i - 1]) * t;
                    f->y[f->n] = cy[i - 1] + (cy[i] - cy[i - 1]) * t;
                    f->s[f->n] = clip;
                    f->hw[f->n] = hw[i - 1] + (hw[i] - hw[i - 1]) * t;
                    f->n++;
                }
                break;
            }
            f->x[f->n] = cx[i], f->y[f->n] = cy[i], f->s[f->n] = s[i], f->hw[f->n] = hw[i];
            f->n++;
        }
        free(rarc), free(cx), free(cy), free(hw), free(s);
        ctx->nl++;
        if (f->n < 2) return fail(1, "lane %u: valid interval clips away the centerline", ln->id);
        for (int i = 1; i < f->n; ++i)
            if (!(f->s[i] > f->s[i - 1])) return fail(1, "lane %u: centerline arc length not increasing", ln->id);
        ctx->length = maxd(ctx->length, f->s[f->n - 1]);
    }
    return 0;
}

/* roads.cpp:125-143: first strictly smaller d2 segment of one lane */
static int lane_best(V2 p, const LF* f, double* s, double* d, double* hw) {
    double bd2 = 1e300;
    int set = 0;
    for (int i = 0; i + 1 < f->n; ++i) {
        V2 a = {f->x[i], f->y[i]}, b = {f->x[i + 1], f->y[i + 1]};
        double t;
        double d2 = psd2(p, a, b, &t);
        if (d2 < bd2) {
            double tx = b.x - a.x, ty = b.y - a.y;
            double qx = a.x + tx * t, qy = a.y + ty * t;
            double sign = (tx * (p.y - qy) - ty * (p.x - qx)) >= 0.0 ? 1.0 : -1.0;
            bd2 = d2;
            *s = f->s[i] + (f->s[i + 1] - f->s[i]) * t;
            *d = sign * sqrt(d2);
            *hw = f->hw[i] + (f->hw[i + 1] - f->hw[i]) * t;
            set = 1;
        }
    }
    return set;
}

/* roads.cpp:147-166 */
static Proj project(V2 p, const Ctx* ctx) {
    int have = 0;
    double bs = 0.0, bd = 0.0;
    uint32_t bid = 0;
    Proj out = {0.0, 0.0, 0};
    for (int l = 0; l < ctx->nl; ++l) {
        double s, d, hw;
        if (!lane_best(p, &ctx->l[l], &s, &d, &hw)) continue;
        if (fabs(d) <= hw) out.in_corr = 1;
        if (!have || fabs(d) < fabs(bd) || (fabs(d) == fabs(bd) && ctx->l[l].id < bid)) {
            have = 1;
            bs = s;
            bd = d;
            bid = ctx->l[l].id;
        }
    }
    out.s = clampd(bs, 0.0, ctx->length);
    out.d = bd;
    return out;
}

/* roads.cpp:192-208 */
static int footprint_on_route(const Obb* box, const Ctx* ctx, double margin) {
    Obb inf = *box;
    inf.hl += margin;
    inf.hw += margin;
    V2 c[4];
    obb_corners(&inf, c);
    for (int k = 0; k < 4; ++k) {
        int any = 0;
        for (int l = 0; l < ctx->nl && !any; ++l) {
            double s, d, hw;
            if (lane_best(c[k], &ctx->l[l], &s, &d, &hw) && fabs(d) <= hw) any = 1;
        }
        if (!any) return 0;
    }
    return 1;
}

static void free_ctx(Ctx* c) {
    for (int i = 0; i < c->nl; ++i) free(c->l[i].x), free(c->l[i].y), free(c->l[i].s), free(c->l[i].hw);
    free(c->l), free(c->stop_i), free(c->stop_s), free(c->light_i), free(c->light_s);
}

/* ----------------------------------------------------------------- env */

typedef struct {
    float x, y;
    uint8_t left, valid;
} RPt;

struct zor_env {
    int B, horizon, total_stop;
    double dt;
    zsim_sim_config cfg;
    Scen* sc;
    Ctx* ctx;
    double *goal_s, *init_s, *logged, *init_steer;
    int* stop_off;
    int* nrp;
    RPt** rp;
};

static const double ACCEL[7] = {-4.0, -2.0, -0.5, 0.0, 0.5, 2.0, 4.0}; /* dynamics.cpp:21-26 */
static const double STEER[5] = {-0.4, -0.1, 0.0, 0.1, 0.4};

void zor_env_destroy(zor_env* e) {
    if (!e) return;
    for (int b = 0; b < e->B; ++b) {
        if (e->sc) free_scen(&e->sc[b]);
        if (e->ctx) free_ctx(&e->ctx[b]);
        if (e->rp) free(e->rp[b]);
    }
    free(e->sc), free(e->ctx), free(e->goal_s), free(e->init_s), free(e->logged), free(e->init_steer);
    free(e->stop_off), free(e->nrp), free(e->rp);
    free(e);
}

int zor_env_create(const uint8_t* buf, size_t nbytes, const int64_t* indices, int32_t n_indices, int32_t horizon,
                   const zsim_sim_config* cfg, zor_env** out) {
    *out = NULL;
    if (nbytes < 16 || memcmp(buf, "ZSIM", 4) != 0) return fail(3, "<memory>: not a ZSIM scenario file");
    double dt;
    memcpy(&dt, buf + 8, 8);
    /* record offsets (scenario_io.cpp:347-377) */
    size_t cap = 64, nrec = 0;
    size_t* off = malloc(sizeof(size_t) * cap);
    uint32_t* len = malloc(sizeof(uint32_t) * cap);
    for (size_t o = 16; o + 4 <= nbytes;) {
        uint32_t l;
        memcpy(&l, buf + o, 4);
        if (nrec == cap) cap *= 2, off = realloc(off, sizeof(size_t) * cap), len = realloc(len, sizeof(uint32_t) * cap);
        off[nrec] = o + 4;
        len[nrec] = l;
        nrec++;
        o += 4 + (size_t)l;
    }
    int B = indices ? n_indices : (int)nrec;
    zor_env* e = (zor_env*)calloc(1, sizeof(zor_env));
    e->B = B;
    e->dt = dt;
    e->cfg = *cfg;
    e->sc = calloc((size_t)B, sizeof(Scen));
    e->ctx = calloc((size_t)B, sizeof(Ctx));
    e->goal_s = calloc((size_t)B, 8), e->init_s = calloc((size_t)B, 8), e->logged = calloc((size_t)B, 8);
    e->init_steer = calloc((size_t)B, 8);
    e->stop_off = calloc((size_t)B, sizeof(int));
    e->nrp = calloc((size_t)B, sizeof(int));
    e->rp = calloc((size_t)B, sizeof(RPt*));
    int maxsteps = 2, rc = 0;
    for (int b = 0; b < B && !rc; ++b) {
        int64_t r = indices ? indices[b] : b;
        if (r < 0 || r >= (int64_t)nrec) rc = fail(1, "scenario index %lld out of range", (long long)r);
        else {
            Cur c = {buf + off[r], buf + off[r] + len[r], 0};
            if (!decode(&c, dt, &e->sc[b])) rc = fail(3, "<memory>[%lld]: truncated record", (long long)r);
            else if ((int)e->sc[b].nsteps > maxsteps) maxsteps = (int)e->sc[b].nsteps;
        }
    }
    free(off), free(len);
    e->horizon = horizon > 0 ? horizon : maxsteps;
    for (int b = 0; b < B && !rc; ++b) {
        const Scen* s = &e->sc[b];
        Ctx* cx = &e->ctx[b];
        if ((int)s->nsteps > e->horizon) rc = fail(1, "scenario has %u steps > T=%d", s->nsteps, e->horizon);
        if (!rc) rc = build_frame(s, cx);
        if (rc) break;
        /* RouteContext::build (roads.cpp:238-251) */
        cx->stop_i = calloc(s->nst ? s->nst : 1, sizeof(int)), cx->stop_s = calloc(s->nst ? s->nst : 1, 8);
        cx->light_i = calloc(s->nlt ? s->nlt : 1, sizeof(int)), cx->light_s = calloc(s->nlt ? s->nlt : 1, 8);
        for (uint32_t i = 0; i < s->nst; ++i) {
            V2 p = {s->st[i].px, s->st[i].py};
            Proj pr = project(p, cx);
            if (pr.in_corr) cx->stop_i[cx->nstops] = (int)i, cx->stop_s[cx->nstops++] = pr.s;
        }
        for (uint32_t i = 0; i < s->nlt; ++i) {
            V2 p = {s->lt[i].sx, s->lt[i].sy};
            Proj pr = project(p, cx);
            if (pr.in_corr) cx->light_i[cx->nlights] = (int)i, cx->light_s[cx->nlights++] = pr.s;
        }
        /* simcore.cpp:217-225 */
        V2 g = {s->gx, s->gy}, p0 = {s->ex[0], s->ey[0]}, p1 = {s->ex[s->nsteps - 1], s->ey[s->nsteps - 1]};
        e->goal_s[b] = project(g, cx).s;
        double s0 = project(p0, cx).s, s1 = project(p1, cx).s;
        e->init_s[b] = s0;
        e->logged[b] = s1 - s0;
        e->stop_off[b] = e->total_stop;
        e->total_stop += cx->nstops;
        /* recover_initial_steering (simcore.cpp:620-627) */
        double st = 0.0;
        if (s->nsteps >= 2) {
            double v0 = s->ev[0];
            if (!(v0 * s->dt < 1e-4)) {
                double dth = wrap_angle((double)s->eh[1] - (double)s->eh[0]);
                st = clampd(atan(dth * cfg->wheelbase / (v0 * s->dt)), -cfg->delta_max, cfg->delta_max);
            }
        }
        e->init_steer[b] = st;
        /* build_route_points (simcore.cpp:181-200) */
        int np = 0;
        for (uint32_t l = 0; l < s->nln; ++l) np += (int)(s->ln[l].nl / 2 + s->ln[l].nr / 2);
        e->rp[b] = malloc(sizeof(RPt) * (np ? np : 1));
        e->nrp[b] = 0;
        for (uint32_t l = 0; l < s->nln; ++l) {
            for (int side = 0; side < 2; ++side) {
                const float* xy = side == 0 ? s->ln[l].l : s->ln[l].r;
                uint32_t n = side == 0 ? s->ln[l].nl : s->ln[l].nr;
                double arc = (double)s->ln[l].s0;
                for (uint32_t i = 0; i + 1 < n; i += 2) {
                    if (i >= 2) {
                        double dx = (double)xy[i] - (double)xy[i - 2], dy = (double)xy[i + 1] - (double)xy[i - 1];
                        arc += sqrt(dx * dx + dy * dy);
                    }
                    RPt q = {xy[i], xy[i + 1], (uint8_t)(side == 0), (uint8_t)(arc <= (double)s->ln[l].s1 + 0.5)};
                    e->rp[b][e->nrp[b]++] = q;
                }
            }
        }
    }
    if (rc) {
        zor_env_destroy(e);
        return rc;
    }
    *out = e;
    return 0;
}

int zor_env_info(const zor_env* e, int32_t* batch, int32_t* horizon, int32_t* total_stop) {
    *batch = e->B;
    *horizon = e->horizon;
    *total_stop = e->total_stop;
    return 0;
}

int zor_scalars(const zor_env* e, double* g, double* i0, double* lp) {
    for (int b = 0; b < e->B; ++b) g[b] = e->goal_s[b], i0[b] = e->init_s[b], lp[b] = e->logged[b];
    return 0;
}

/* Env::init_state (simcore.cpp:237-276); Rng split (common.hpp:28-51) */
int zor_init_state(const zor_env* e, uint64_t seed, const zsim_state_view* o) {
    const uint64_t G = 0x9e3779b97f4a7c15ull;
    uint64_t parent = seed + G;
    for (int b = 0; b < e->B; ++b) {
        const Scen* s = &e->sc[b];
        o->x[b] = s->ex[0], o->y[b] = s->ey[0], o->heading[b] = s->eh[0], o->v[b] = s->ev[0];
        o->steering[b] = e->init_steer[b];
        o->t[b] = 0, o->done[b] = 0, o->reason[b] = 0, o->events[b] = 0;
        uint64_t z = (parent += G);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z = z ^ (z >> 31);
        o->rng[b] = (z ^ ((uint64_t)b * 0xd1342543de82ef95ull + 0x2545f4914f6cdd1dull)) + G;
        V2 p = {o->x[b], o->y[b]};
        Proj pr = project(p, &e->ctx[b]);
        o->proj_s[b] = pr.s, o->proj_d[b] = pr.d, o->proj_in_corridor[b] = (uint8_t)pr.in_corr;
        for (int j = 0; j < e->ctx[b].nstops; ++j) {
            double ahead = e->ctx[b].stop_s[j] - pr.s;
            o->stopped_flags[e->stop_off[b] + j] =
                (uint8_t)(ahead >= 0.0 && ahead <= e->cfg.stop_zone && o->v[b] < e->cfg.stop_slow_speed);
        }
    }
    return 0;
}

static Obb ego_box(double x, double y, double h, const zsim_sim_config* c) {
    Obb b = {{x + cos(h) * c->ego_center_offset, y + sin(h) * c->ego_center_offset}, c->ego_length * 0.5,
             c->ego_width * 0.5, h};
    return b;
}

static Obb agent_box(const Agent* a, int t) {
    Obb b = {{a->x[t], a->y[t]}, (double)a->len * 0.5, (double)a->wid * 0.5, a->h[t]};
    return b;
}

/* Env::step / step_row (simcore.cpp:278-421) */
int zor_step(const zor_env* e, const zsim_state_view* in, const int32_t* ai, const int32_t* si,
             const zsim_state_view* o, const zsim_stepout_view* so) {
    const zsim_sim_config* c = &e->cfg;
    for (int b = 0; b < e->B; ++b)
        if (!in->done[b] && (ai[b] < 0 || ai[b] >= 7 || si[b] < 0 || si[b] >= 5))
            return fail(1, "action index out of range");
    if (o->stopped_flags != in->stopped_flags) memcpy(o->stopped_flags, in->stopped_flags, (size_t)e->total_stop);
    for (int b = 0; b < e->B; ++b) {
        const Scen* s = &e->sc[b];
        const Ctx* cx = &e->ctx[b];
        double x0 = in->x[b], y0 = in->y[b], h0 = in->heading[b], v0 = in->v[b], d0 = in->steering[b];
        double ps = in->proj_s[b];
        int t0 = in->t[b];
        if (in->done[b]) { /* simcore.cpp:281-299 */
            o->x[b] = x0, o->y[b] = y0, o->heading[b] = h0, o->v[b] = v0, o->steering[b] = d0, o->t[b] = t0;
            o->done[b] = 1, o->reason[b] = in->reason[b], o->rng[b] = in->rng[b], o->proj_s[b] = ps;
            o->proj_d[b] = in->proj_d[b], o->proj_in_corridor[b] = in->proj_in_corridor[b], o->events[b] = in->events[b];
            so->reward[b] = 0.f, so->event[b] = 0, so->s[b] = (float)ps, so->a_lat[b] = 0.f, so->a_lon[b] = 0.f;
            so->v[b] = (float)v0;
            continue;
        }
        double acc = ACCEL[ai[b]], rate = STEER[si[b]], dt = e->dt;
        /* bicycle_step (dynamics.cpp:10-19) */
        double x1 = x0 + v0 * cos(h0) * dt, y1 = y0 + v0 * sin(h0) * dt;
        double h1 = wrap_angle(h0 + v0 / c->wheelbase * tan(d0) * dt);
        double v1 = maxd(v0 + acc * dt, c->v_min), d1 = clampd(d0 + rate * dt, -c->delta_max, c->delta_max);
        int t1 = t0 + 1;
        V2 p = {x1, y1};
        Proj p1 = project(p, cx);
        double progress = p1.s - ps;
        double a_lat = v0 * v0 * tan(d0) / c->wheelbase, a_lon = acc;
        double reward = c->w_progress * progress - c->w_speed * maxd(0.0, v1 - (double)s->limit) * dt -
                        c->w_lat * a_lat * a_lat * dt - c->w_lon * a_lon * a_lon * dt;
        Obb box = ego_box(x1, y1, h1, c);
        int hit_col = 0;
        for (uint32_t j = 0; j < s->nag && !hit_col; ++j)
            if (t1 < (int)s->nsteps && s->ag[j].valid[t1]) {
                Obb ab = agent_box(&s->ag[j], t1);
                if (obb_overlap(&box, &ab)) hit_col = 1;
            }
        int hit_off = !footprint_on_route(&box, cx, c->footprint_margin);
        int hit_red = 0, tl = t0 < (int)s->nsteps - 1 ? t0 : (int)s->nsteps - 1;
        for (int k = 0; k < cx->nlights; ++k)
            if (ps < cx->light_s[k] && cx->light_s[k] <= p1.s && s->lt[cx->light_i[k]].st[tl] == 0) hit_red = 1;
        int hit_stop = 0;
        for (int j = 0; j < cx->nstops; ++j)
            if (ps < cx->stop_s[j] && cx->stop_s[j] <= p1.s && v0 > c->stop_cross_speed &&
                !in->stopped_flags[e->stop_off[b] + j])
                hit_stop = 1;
        int hit_goal = fabs(p1.s - e->goal_s[b]) <= c->goal_radius;
        int reason = hit_col ? 1 : hit_off ? 2 : hit_red ? 3 : hit_stop ? 4 : hit_goal ? 5 : 0;
        int ev = in->events[b];
        if (c->disable_dones) {
            ev |= (hit_col ? 1 : 0) | (hit_off ? 2 : 0) | (hit_red ? 4 : 0) | (hit_stop ? 8 : 0) | (hit_goal ? 16 : 0);
        } else if (reason) {
            ev |= 1 << (reason - 1);
            if (reason != 5) reward -= c->terminal_penalty;
        }
        int done = (!c->disable_dones && reason) ? 1 : 0;
        o->x[b] = x1, o->y[b] = y1, o->heading[b] = h1, o->v[b] = v1, o->steering[b] = d1, o->t[b] = t1;
        o->done[b] = (uint8_t)done, o->reason[b] = (uint8_t)(done ? reason : 0), o->rng[b] = in->rng[b];
        o->proj_s[b] = p1.s, o->proj_d[b] = p1.d, o->proj_in_corridor[b] = (uint8_t)p1.in_corr;
        o->events[b] = (uint8_t)ev;
        for (int j = 0; j < cx->nstops; ++j) { /* simcore.cpp:390-396 */
            double ahead = cx->stop_s[j] - p1.s;
            if (ahead >= 0.0 && ahead <= c->stop_zone && v1 < c->stop_slow_speed)
                o->stopped_flags[e->stop_off[b] + j] = 1;
        }
        so->reward[b] = (float)reward, so->event[b] = (uint8_t)reason, so->s[b] = (float)p1.s;
        so->a_lat[b] = (float)a_lat, so->a_lon[b] = (float)a_lon, so->v[b] = (float)v1;
    }
    return 0;
}

typedef struct {
    double k;
    int i;
} Key;

static int key_cmp(const void* a, const void* b) {
    const Key *x = (const Key*)a, *y = (const Key*)b;
    if (x->k != y->k) return x->k < y->k ? -1 : 1;
    return (x->i > y->i) - (x->i < y->i);
}

/* Env::observe / observe_row (simcore.cpp:423-552) */
int zor_observe(const zor_env* e, const zsim_state_view* in, const zsim_obs_view* ob, int32_t* topk) {
    const zsim_sim_config* c = &e->cfg;
    const int Ka = c->n_agents, Kr = c->n_road, Kl = c->n_route, KT = Ka + Kr + Kl;
    for (int b = 0; b < e->B; ++b) {
        const Scen* s = &e->sc[b];
        const Ctx* cx = &e->ctx[b];
        float* act = ob->active + (size_t)b * 9;
        float* ag = ob->agents + (size_t)b * Ka * 6;
        float* rd = ob->road + (size_t)b * Kr * 12;
        float* rt = ob->route + (size_t)b * Kl * 5;
        float* val = ob->value_only + (size_t)b * 2;
        int32_t* tk = topk ? topk + (size_t)b * KT : NULL;
        memset(act, 0, 9 * 4), memset(ag, 0, (size_t)Ka * 24), memset(rd, 0, (size_t)Kr * 48);
        memset(rt, 0, (size_t)Kl * 20), memset(val, 0, 8);
        if (tk)
            for (int k = 0; k < KT; ++k) tk[k] = -1;
        if (in->done[b]) continue;
        double x = in->x[b], y = in->y[b], h = in->heading[b];
        int t = in->t[b];
        double cc = cos(-h), ss = sin(-h);
        /* active features: roads::stop_info (roads.cpp:253-277) */
        double bst = 1e300, blt = 1e300;
        int bli = -1;
        for (int j = 0; j < cx->nstops; ++j) {
            double ahead = cx->stop_s[j] - in->proj_s[b];
            if (ahead > 0.0 && ahead < bst) bst = ahead;
        }
        for (int k = 0; k < cx->nlights; ++k) {
            double ahead = cx->light_s[k] - in->proj_s[b];
            if (ahead > 0.0 && ahead < blt) blt = ahead, bli = cx->light_i[k];
        }
        int light = 3;
        if (bli >= 0) {
            int st = t < (int)s->nsteps - 1 ? t : (int)s->nsteps - 1;
            light = s->lt[bli].st[st > 0 ? st : 0];
        }
        double R = c->feature_radius;
        act[0] = (float)in->v[b];
        act[1] = (float)in->steering[b];
        act[2] = (float)(bst < 1e300 ? mind(bst, R) : R);
        act[3 + light] = 1.f;
        act[7] = (float)(bli >= 0 ? mind(blt, R) : R);
        act[8] = s->limit;
        /* agents by (bbox distance, index) */
        Obb eb = ego_box(x, y, h, c);
        Key* ak = malloc(sizeof(Key) * (s->nag ? s->nag : 1));
        int na = 0;
        for (uint32_t j = 0; j < s->nag; ++j)
            if (t < (int)s->nsteps && s->ag[j].valid[t]) {
                Obb ab = agent_box(&s->ag[j], t);
                ak[na].k = obb_distance(&eb, &ab);
                ak[na].i = (int)j;
                na++;
            }
        qsort(ak, (size_t)na, sizeof(Key), key_cmp);
        for (int k = 0; k < Ka && k < na; ++k) {
            const Agent* a = &s->ag[ak[k].i];
            double dx = (double)a->x[t] - x, dy = (double)a->y[t] - y;
            float* f = ag + (size_t)k * 6;
            f[0] = (float)(cc * dx - ss * dy);
            f[1] = (float)(ss * dx + cc * dy);
            f[2] = (float)wrap_angle((double)a->h[t] - h);
            f[3] = a->sp[t];
            f[4] = (float)ak[k].k;
            f[5] = 1.f;
            if (tk) tk[k] = ak[k].i;
        }
        free(ak);
        /* road: nearest_features (roads.cpp:210-236), canonical (d2, flat index) order */
        int np = 0;
        for (uint32_t f = 0; f < s->nft; ++f) np += (int)(s->ft[f].n / 2);
        Key* rk = malloc(sizeof(Key) * (np ? np : 1));
        int* fidx = malloc(sizeof(int) * (np ? np : 1));
        int* pidx = malloc(sizeof(int) * (np ? np : 1));
        int nr = 0, flat = 0;
        double r2 = R * R;
        for (uint32_t f = 0; f < s->nft; ++f)
            for (uint32_t i = 0; i + 1 < s->ft[f].n; i += 2, ++flat) {
                double dx = (double)s->ft[f].xy[i] - x, dy = (double)s->ft[f].xy[i + 1] - y;
                double d2 = dx * dx + dy * dy;
                if (d2 <= r2) {
                    rk[nr].k = d2;
                    rk[nr].i = flat;
                    fidx[flat] = (int)f;
                    pidx[flat] = (int)i;
                    nr++;
                }
            }
        qsort(rk, (size_t)nr, sizeof(Key), key_cmp);
        for (int k = 0; k < Kr && k < nr; ++k) {
            const Feat* ft = &s->ft[fidx[rk[k].i]];
            int i = pidx[rk[k].i];
            double dx = (double)ft->xy[i] - x, dy = (double)ft->xy[i + 1] - y;
            float* f = rd + (size_t)k * 12;
            f[0] = (float)(cc * dx - ss * dy);
            f[1] = (float)(ss * dx + cc * dy);
            f[2 + ft->kind] = 1.f;
            f[7 + ft->dir] = 1.f;
            f[11] = 1.f;
            if (tk) tk[Ka + k] = rk[k].i;
        }
        free(rk), free(fidx), free(pidx);
        /* route border points by (d2, index), no radius (simcore.cpp:503-529) */
        int nq = e->nrp[b];
        Key* qk = malloc(sizeof(Key) * (nq ? nq : 1));
        for (int i = 0; i < nq; ++i) {
            double dx = (double)e->rp[b][i].x - x, dy = (double)e->rp[b][i].y - y;
            qk[i].k = dx * dx + dy * dy;
            qk[i].i = i;
        }
        qsort(qk, (size_t)nq, sizeof(Key), key_cmp);
        for (int k = 0; k < Kl && k < nq; ++k) {
            const RPt* q = &e->rp[b][qk[k].i];
            double dx = (double)q->x - x, dy = (double)q->y - y;
            float* f = rt + (size_t)k * 5;
            f[0] = (float)(cc * dx - ss * dy);
            f[1] = (float)(ss * dx + cc * dy);
            f[2] = q->left ? 1.f : 0.f;
            f[3] = q->valid ? 1.f : 0.f;
            f[4] = 1.f;
            if (tk) tk[Ka + Kr + k] = qk[k].i;
        }
        free(qk);
        double gx = (double)s->gx - x, gy = (double)s->gy - y;
        val[0] = (float)sqrt(gx * gx + gy * gy);
        val[1] = (float)(e->horizon - t);
    }
    return 0;
}
