/* rgg_oracle.c — plain-C restatement of the SerRGG hot path (TEST INFRASTRUCTURE).
 *
 * ORACLE ONLY: never linked into or called by the product.  Parity: pinned
 * against the reference (see rgg_oracle.h).  Build: -ffp-contract=off, the
 * same flag the reference library is built with (proj/CMakeLists.txt:12-14), so
 * every expression below rounds exactly like the reference's scalar backend.
 */
#include "rgg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ predicates */

/* proj/src/kernels_scalar.cpp:7-30 — SatBox from the 8x3 corner block:
 * e_k = 0.5*(c[1<<k] - c[0]); center = ((c0+e0)+e1)+e2; u_k = e_k/sqrt(e_k.e_k) or 0. */
void ro_sat_prep(const double* c, double* s) {
    double* center = s;
    double* e = s + 3;
    double* u = s + 12;
    for (int k = 0; k < 3; ++k) {
        const int hi = (1 << k) * 3;
        for (int j = 0; j < 3; ++j) e[k * 3 + j] = 0.5 * (c[hi + j] - c[j]);
    }
    for (int j = 0; j < 3; ++j) center[j] = ((c[j] + e[0 * 3 + j]) + e[1 * 3 + j]) + e[2 * 3 + j];
    for (int k = 0; k < 3; ++k) {
        const double* ek = e + 3 * k;
        const double n2 = (ek[0] * ek[0] + ek[1] * ek[1]) + ek[2] * ek[2];
        if (n2 > 0.0) {
            const double len = sqrt(n2);
            for (int j = 0; j < 3; ++j) u[k * 3 + j] = ek[j] / len;
        } else {
            u[k * 3 + 0] = u[k * 3 + 1] = u[k * 3 + 2] = 0.0;
        }
    }
}

static inline double dot3(const double* x, const double* y) { return (x[0] * y[0] + x[1] * y[1]) + x[2] * y[2]; }

/* proj/src/kernels_scalar.cpp:37-42 — strict '>' so touching intersects. */
static inline int separated_on(const double* a, const double* b, const double* d, const double* ax) {
    const double* ea = a + 3;
    const double* eb = b + 3;
    const double ra = (fabs(dot3(ea, ax)) + fabs(dot3(ea + 3, ax))) + fabs(dot3(ea + 6, ax));
    const double rb = (fabs(dot3(eb, ax)) + fabs(dot3(eb + 3, ax))) + fabs(dot3(eb + 6, ax));
    const double s = fabs(dot3(d, ax));
    return s > ra + rb;
}

/* proj/src/kernels_scalar.cpp:48-69 — face axes of a, of b, then 9 crosses
 * a.u[i] x b.u[j] skipped when n2 < 1e-12 (evaluated before the test). */
static int sat_impl(const double* a, const double* b, int* cost) {
    double d[3];
    for (int j = 0; j < 3; ++j) d[j] = b[j] - a[j];
    int flops = 3;
    const double* au = a + 12;
    const double* bu = b + 12;
    for (int k = 0; k < 3; ++k) {
        flops += 40;
        if (separated_on(a, b, d, au + 3 * k)) goto separated;
    }
    for (int k = 0; k < 3; ++k) {
        flops += 40;
        if (separated_on(a, b, d, bu + 3 * k)) goto separated;
    }
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) {
            const double* x = au + 3 * i;
            const double* y = bu + 3 * j;
            const double axis[3] = {x[1] * y[2] - x[2] * y[1], x[2] * y[0] - x[0] * y[2], x[0] * y[1] - x[1] * y[0]};
            const double n2 = dot3(axis, axis);
            flops += 14;
            if (n2 >= 1e-12) {
                flops += 40;
                if (separated_on(a, b, d, axis)) goto separated;
            }
        }
    }
    if (cost) *cost = flops;
    return 1;
separated:
    if (cost) *cost = flops;
    return 0;
}

int ro_sat_boxes(const double* a, const double* b) { return sat_impl(a, b, NULL); }

int ro_sat_cost(const double* a, const double* b) {
    int c = 0;
    sat_impl(a, b, &c);
    return c;
}

/* proj/src/kernels_scalar.cpp:71-79 */
void ro_seg_prep(const double* s, double* p) {
    for (int j = 0; j < 3; ++j) {
        p[j] = s[j];
        p[3 + j] = s[3 + j] - s[j];
    }
    p[6] = (p[3] * p[3] + p[4] * p[4]) + p[5] * p[5];
}

/* proj/src/kernels_scalar.cpp:81-94 — clamped projection; dd == 0 gives t = 0. */
double ro_seg_point_dist(const double* s, const double* c) {
    const double px = c[0] - s[0];
    const double py = c[1] - s[1];
    const double pz = c[2] - s[2];
    double t = 0.0;
    if (s[6] > 0.0) {
        t = ((px * s[3] + py * s[4]) + pz * s[5]) / s[6];
        t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    }
    const double qx = px - t * s[3];
    const double qy = py - t * s[4];
    const double qz = pz - t * s[5];
    return sqrt((qx * qx + qy * qy) + qz * qz);
}

/* proj/src/kernels_scalar.cpp:96 — closed predicate. */
int ro_seg_sphere(const double* s, const double* c, double r) { return ro_seg_point_dist(s, c) <= r; }

/* proj/src/kernels_scalar.cpp:100-111 */
void ro_sat_batch(const double* boxes, const int32_t* idx, int n, const double* obstacle, uint8_t* out) {
    for (int i = 0; i < n; ++i) out[i] = (uint8_t)ro_sat_boxes(boxes + 21 * (size_t)idx[i], obstacle);
}

void ro_seg_sphere_batch(const double* segs, const int32_t* idx, int n, const double* c, double r, uint8_t* out) {
    for (int i = 0; i < n; ++i) out[i] = (uint8_t)ro_seg_sphere(segs + 7 * (size_t)idx[i], c, r);
}

/* ------------------------------------------------------ obstacle re-posing */

static void aabb_empty(double* a) {
    a[0] = a[1] = a[2] = INFINITY;
    a[3] = a[4] = a[5] = -INFINITY;
}

/* Aabb::expand (vec3.hpp:116-119) via fmin/fmax. */
static void aabb_expand(double* a, double x, double y, double z) {
    a[0] = fmin(a[0], x);
    a[1] = fmin(a[1], y);
    a[2] = fmin(a[2], z);
    a[3] = fmax(a[3], x);
    a[4] = fmax(a[4], y);
    a[5] = fmax(a[5], z);
}

/* Aabb::overlaps (vec3.hpp:126-129), closed. */
static int aabb_overlaps(const double* a, const double* b) {
    return a[0] <= b[3] && b[0] <= a[3] && a[1] <= b[4] && b[1] <= a[4] && a[2] <= b[5] && b[2] <= a[5];
}

/* The candidate filter of a (component, obstacle) pair.  The reference tests every
 * spatial-grid candidate (engine_batch.cpp:55-74, spatial_grid.cpp:114-135); a pair
 * whose exact AABBs miss by an ulp can still be an fp64 SAT / segment-sphere hit
 * (tests/test_gpu_filter.py finds such pairs), so the obstacle box b is widened by a
 * relative 2^-40 on every face, as the GPU's pose kernel does (rgg_kernels.cu widen_*). */
static double widen(double v, int up) {
    if (!isfinite(v)) return v;
    return up ? v + (fabs(v) + 1.0) * 0x1p-40 : v - (fabs(v) + 1.0) * 0x1p-40;
}
static int candidate_overlaps(const double* comp, const double* b) {
    double w[6];
    for (int k = 0; k < 6; ++k) w[k] = widen(b[k], k >= 3);
    return aabb_overlaps(comp, w);
}

/* Transform::apply (vec3.hpp:72-76): ((r0 x + r1 y) + r2 z) + t. */
static void tf_apply(const double* rt, const double* p, double* out) {
    for (int i = 0; i < 3; ++i)
        out[i] = rt[3 * i + 0] * p[0] + rt[3 * i + 1] * p[1] + rt[3 * i + 2] * p[2] + rt[9 + i];
}

/* proj/src/batch_layout.cpp:148-172 with apply_transform(Obb) (geometry.cpp:307-313),
 * obb_corners (geometry.cpp:50-62), aabb_of_obb (geometry.cpp:205-213). */
void ro_obstacle_operands(const double* he, const double* sph_local, int n_sph, double sph_r, const double* rt,
                          double* sat21, double* aabb6, double* centres, double* saabb6) {
    static const double zero[3] = {0, 0, 0};
    static const double unit[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    double center[3], axes[3][3];
    tf_apply(rt, zero, center);
    for (int k = 0; k < 3; ++k)
        for (int i = 0; i < 3; ++i)
            axes[k][i] = rt[3 * i + 0] * unit[k][0] + rt[3 * i + 1] * unit[k][1] + rt[3 * i + 2] * unit[k][2];
    double e[3][3];
    for (int k = 0; k < 3; ++k)
        for (int i = 0; i < 3; ++i) e[k][i] = axes[k][i] * he[k];
    double corners[24];
    aabb_empty(aabb6);
    for (int c = 0; c < 8; ++c) {
        double p[3];
        for (int i = 0; i < 3; ++i) p[i] = (c & 1) ? center[i] + e[0][i] : center[i] - e[0][i];
        for (int i = 0; i < 3; ++i) p[i] = (c & 2) ? p[i] + e[1][i] : p[i] - e[1][i];
        for (int i = 0; i < 3; ++i) p[i] = (c & 4) ? p[i] + e[2][i] : p[i] - e[2][i];
        memcpy(corners + 3 * c, p, sizeof(p));
        aabb_expand(aabb6, p[0], p[1], p[2]);
    }
    ro_sat_prep(corners, sat21);
    aabb_empty(saabb6);
    for (int s = 0; s < n_sph; ++s) {
        double* c = centres + 3 * s;
        tf_apply(rt, sph_local + 3 * s, c);
        aabb_expand(saabb6, c[0] - sph_r, c[1] - sph_r, c[2] - sph_r);
        aabb_expand(saabb6, c[0] + sph_r, c[1] + sph_r, c[2] + sph_r);
    }
}

/* ------------------------------------------------------------------ engine */

typedef struct {
    int32_t* v;
    int n, cap;
} ivec;

static void ivec_push(ivec* a, int32_t x) {
    if (a->n == a->cap) {
        a->cap = a->cap ? 2 * a->cap : 16;
        a->v = (int32_t*)realloc(a->v, sizeof(int32_t) * (size_t)a->cap);
    }
    a->v[a->n++] = x;
}

struct ro_engine {
    ro_view v;
    int use_under;
    int words;
    uint8_t* states;
    uint64_t* bits;     /* N*words */
    ivec* listed;       /* per obstacle */
    int unknown;
    uint8_t* active;    /* M */
    double* osat;       /* M*21 */
    double* oaabb;      /* M*6 */
    double* ocentre;    /* M*C*3 */
    double* osaabb;     /* M*6 */
    /* per-update undo log (touched_, engine_batch.cpp:33-53) */
    int32_t* t_id;
    uint8_t* t_before;
    int t_n, t_cap;
};

ro_engine* ro_engine_new(const ro_view* v, int use_under) {
    ro_engine* e = (ro_engine*)calloc(1, sizeof(ro_engine));
    e->v = *v;
    e->use_under = use_under;
    e->words = v->n_obstacles <= 64 ? 1 : (v->n_obstacles + 63) / 64;
    const size_t n = (size_t)v->n_components, m = (size_t)v->n_obstacles, c = (size_t)v->max_spheres;
    e->states = (uint8_t*)calloc(n ? n : 1, 1);
    e->bits = (uint64_t*)calloc(n * (size_t)e->words + 1, sizeof(uint64_t));
    e->listed = (ivec*)calloc(m + 1, sizeof(ivec));
    e->active = (uint8_t*)calloc(m + 1, 1);
    e->osat = (double*)calloc(m * 21 + 1, sizeof(double));
    e->oaabb = (double*)calloc(m * 6 + 1, sizeof(double));
    e->ocentre = (double*)calloc(m * c * 3 + 1, sizeof(double));
    e->osaabb = (double*)calloc(m * 6 + 1, sizeof(double));
    /* serialize() poses every obstacle at its canonical pose (batch_layout.cpp:117-136) */
    static const double identity[12] = {1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0};
    for (size_t o = 0; o < m; ++o)
        ro_obstacle_operands(v->obst_he + 3 * o, v->obst_sph_local + 3 * o * c, v->obst_sph_n[o], v->obst_sph_r[o],
                             identity, e->osat + 21 * o, e->oaabb + 6 * o, e->ocentre + 3 * o * c, e->osaabb + 6 * o);
    return e;
}

void ro_engine_free(ro_engine* e) {
    if (!e) return;
    for (int o = 0; o < e->v.n_obstacles; ++o) free(e->listed[o].v);
    free(e->listed);
    free(e->states);
    free(e->bits);
    free(e->active);
    free(e->osat);
    free(e->oaabb);
    free(e->ocentre);
    free(e->osaabb);
    free(e->t_id);
    free(e->t_before);
    free(e);
}

int ro_engine_words(const ro_engine* e) { return e->words; }

static void set_state(ro_engine* e, int32_t c, uint8_t s) {
    if (e->states[c] == s) return;
    if (e->t_n == e->t_cap) {
        e->t_cap = e->t_cap ? 2 * e->t_cap : 64;
        e->t_id = (int32_t*)realloc(e->t_id, sizeof(int32_t) * (size_t)e->t_cap);
        e->t_before = (uint8_t*)realloc(e->t_before, (size_t)e->t_cap);
    }
    e->t_id[e->t_n] = c;
    e->t_before[e->t_n] = e->states[c];
    e->t_n++;
    if (e->states[c] == 2) --e->unknown;
    if (s == 2) ++e->unknown;
    e->states[c] = s;
}

/* batch_over for one pair: OR over bodies (engine_batch.cpp:55-74). */
static int over_pair(const ro_engine* e, int32_t c, int32_t o) {
    const int nb = e->v.n_bodies;
    for (int b = 0; b < nb; ++b)
        if (ro_sat_boxes(e->v.edge_sat + 21 * ((size_t)c * nb + b), e->osat + 21 * (size_t)o)) return 1;
    return 0;
}

/* batch_under for one pair: any real segment of any (b, s) row within
 * o_minus_r[o] + spline_radius[b*S+s] of any obstacle sphere (engine_batch.cpp:76-112). */
static int under_pair(const ro_engine* e, int32_t c, int32_t o) {
    const int nb = e->v.n_bodies, ns = e->v.n_slots, C = e->v.max_spheres;
    const int nsph = e->v.obst_sph_n[o];
    for (int b = 0; b < nb; ++b) {
        for (int s = 0; s < ns; ++s) {
            const size_t row = ((size_t)c * nb + b) * ns + s;
            const double r_total = e->v.obst_sph_r[o] + e->v.spline_radius[b * ns + s];
            for (int32_t k = e->v.row_off[row]; k < e->v.row_off[row + 1]; ++k) {
                for (int sp = 0; sp < nsph; ++sp) {
                    if (ro_seg_sphere(e->v.segs + 7 * (size_t)k, e->ocentre + 3 * ((size_t)o * C + sp), r_total))
                        return 1;
                }
            }
        }
    }
    return 0;
}

static int cmp_touch(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

int ro_engine_update(ro_engine* e, int32_t o, const double* rt, int64_t* rep) {
    if (o < 0 || o >= e->v.n_obstacles) return -1;
    const int W = e->words;
    const int32_t N = e->v.n_components;
    e->t_n = 0;
    /* revalidate_old_intersections (engine_batch.cpp:114-143) */
    ivec holders = e->listed[o];
    memset(&e->listed[o], 0, sizeof(ivec));
    const int w = o >> 6;
    const uint64_t bit = 1ull << (o & 63);
    ivec recheck = {0};
    for (int i = 0; i < holders.n; ++i) {
        const int32_t c = holders.v[i];
        uint64_t* bc = e->bits + (size_t)c * W;
        bc[w] &= ~bit;
        int any = 0;
        for (int k = 0; k < W; ++k) any |= bc[k] != 0;
        if (!any) {
            set_state(e, c, 0);
        } else {
            set_state(e, c, 2);
            ivec_push(&recheck, c);
        }
    }
    free(holders.v);
    if (recheck.n && e->use_under) {
        for (int32_t o2 = 0; o2 < e->v.n_obstacles; ++o2) {
            const uint64_t b2 = 1ull << (o2 & 63);
            for (int i = 0; i < recheck.n; ++i) {
                const int32_t c = recheck.v[i];
                if (!(e->bits[(size_t)c * W + (o2 >> 6)] & b2)) continue;
                if (under_pair(e, c, o2)) set_state(e, c, 1);
            }
        }
    }
    free(recheck.v);
    /* update_transforms + scene mutation (engine_batch.cpp:153-158) */
    ro_obstacle_operands(e->v.obst_he + 3 * (size_t)o, e->v.obst_sph_local + 3 * (size_t)o * e->v.max_spheres,
                         e->v.obst_sph_n[o], e->v.obst_sph_r[o], rt, e->osat + 21 * (size_t)o, e->oaabb + 6 * (size_t)o,
                         e->ocentre + 3 * (size_t)o * e->v.max_spheres, e->osaabb + 6 * (size_t)o);
    e->active[o] = 1;
    /* over phase (engine_batch.cpp:163-177); candidates = closed AABB overlap */
    for (int32_t c = 0; c < N; ++c) {
        if (!candidate_overlaps(e->v.comp_aabb + 6 * (size_t)c, e->oaabb + 6 * (size_t)o)) continue;
        if (!over_pair(e, c, o)) continue;
        if (e->states[c] == 0) set_state(e, c, 2);
        uint64_t* bc = e->bits + (size_t)c * W + w;
        if (!(*bc & bit)) {
            *bc |= bit;
            ivec_push(&e->listed[o], c);
        }
    }
    /* under phase (engine_batch.cpp:181-188) */
    if (e->use_under) {
        for (int32_t c = 0; c < N; ++c) {
            if (!candidate_overlaps(e->v.comp_aabb + 6 * (size_t)c, e->osaabb + 6 * (size_t)o)) continue;
            if (under_pair(e, c, o)) set_state(e, c, 1);
        }
    }
    /* finish_counts (engine_batch.cpp:41-53): first touch holds the pre-update state */
    int64_t counts[3] = {0, 0, 0};
    if (e->t_n) {
        int64_t* key = (int64_t*)malloc(sizeof(int64_t) * (size_t)e->t_n);
        for (int i = 0; i < e->t_n; ++i) key[i] = ((int64_t)e->t_id[i] << 32) | i;
        qsort(key, (size_t)e->t_n, sizeof(int64_t), cmp_touch);
        for (int i = 0; i < e->t_n; ++i) {
            const int32_t c = (int32_t)(key[i] >> 32);
            if (i > 0 && (int32_t)(key[i - 1] >> 32) == c) continue;
            const uint8_t before = e->t_before[key[i] & 0xffffffff];
            if (before != e->states[c]) counts[e->states[c]]++;
        }
        free(key);
    }
    if (rep) {
        rep[0] = counts[0];
        rep[1] = counts[1];
        rep[2] = counts[2];
        rep[3] = e->unknown;
    }
    return 0;
}

void ro_engine_states(const ro_engine* e, uint8_t* out) { memcpy(out, e->states, (size_t)e->v.n_components); }

void ro_engine_bits(const ro_engine* e, uint64_t* out) {
    memcpy(out, e->bits, sizeof(uint64_t) * (size_t)e->v.n_components * (size_t)e->words);
}

int ro_engine_unknown(const ro_engine* e) { return e->unknown; }

void ro_engine_pure(const ro_engine* e, uint8_t* states, uint64_t* bits) {
    const int W = e->words;
    for (int32_t c = 0; c < e->v.n_components; ++c) {
        uint64_t* bc = bits + (size_t)c * W;
        memset(bc, 0, sizeof(uint64_t) * (size_t)W);
        int over = 0, under = 0;
        for (int32_t o = 0; o < e->v.n_obstacles; ++o) {
            if (!e->active[o]) continue;
            const double* ca = e->v.comp_aabb + 6 * (size_t)c;
            if (candidate_overlaps(ca, e->oaabb + 6 * (size_t)o) && over_pair(e, c, o)) {
                over = 1;
                bc[o >> 6] |= 1ull << (o & 63);
            }
            if (e->use_under && candidate_overlaps(ca, e->osaabb + 6 * (size_t)o) && under_pair(e, c, o)) under = 1;
        }
        states[c] = under ? 1 : (over ? 2 : 0);
    }
}

void ro_engine_mask(const ro_engine* e, int kind, const int32_t* cands, int n, int32_t o, uint8_t* mask) {
    for (int i = 0; i < n; ++i) mask[i] = (uint8_t)(kind == 0 ? over_pair(e, cands[i], o) : under_pair(e, cands[i], o));
}

void ro_engine_census(const ro_engine* e, int64_t* out) {
    memset(out, 0, sizeof(int64_t) * 7);
    const int nb = e->v.n_bodies, ns = e->v.n_slots;
    for (int32_t o = 0; o < e->v.n_obstacles; ++o) out[6] += e->active[o];
    for (int32_t c = 0; c < e->v.n_components; ++c) {
        const double* ca = e->v.comp_aabb + 6 * (size_t)c;
        const int64_t segs = e->v.row_off[((size_t)c + 1) * nb * ns] - e->v.row_off[(size_t)c * nb * ns];
        for (int32_t o = 0; o < e->v.n_obstacles; ++o) {
            if (!e->active[o]) continue;
            if (candidate_overlaps(ca, e->oaabb + 6 * (size_t)o)) {
                int hit = 0;
                for (int b = 0; b < nb; ++b) {
                    const double* a = e->v.edge_sat + 21 * ((size_t)c * nb + b);
                    out[0] += 1;
                    out[1] += ro_sat_cost(a, e->osat + 21 * (size_t)o);
                    hit |= ro_sat_boxes(a, e->osat + 21 * (size_t)o);
                }
                out[4] += hit;
            }
            if (e->use_under && candidate_overlaps(ca, e->osaabb + 6 * (size_t)o)) {
                out[2] += 1;
                out[3] += segs * e->v.obst_sph_n[o];
                out[5] += under_pair(e, c, o);
            }
        }
    }
}

/* ================================================================ exact resolve
 * Restated literally from the reference, as the checker of the GPU's reduced
 * (150-axis) form in paper_2603_28674_b200/csrc/rgg_resolve.cu:
 *   ConvexPolytope::box      geometry.cpp:228-254 (+ obb_corners :50-62)
 *   project / separates      geometry.cpp:258-273
 *   edge_directions          geometry.cpp:275-286 (24 ring edges)
 *   polytopes_intersect      geometry.cpp:288-303 (all face normals, 24 x 24 crosses)
 *   aabb_of_obb              geometry.cpp:205-213, apply_transform :307-313
 *   exact_component_valid    roadmap.cpp:129-163
 */
typedef struct ro_poly {
    double v[8][3];
    double n[6][3];  /* face normals: +a0, -a0, +a1, -a1, +a2, -a2 */
} ro_poly;

static const int k_rings[6][4] = {{1, 3, 7, 5}, {0, 4, 6, 2}, {2, 6, 7, 3}, {0, 1, 5, 4}, {4, 5, 7, 6}, {0, 2, 3, 1}};

/* Transform::rotate of unit axis k (vec3.hpp:79-84) */
static void rot_unit(const double* rt, int k, double* out) {
    const double p[3] = {k == 0 ? 1.0 : 0.0, k == 1 ? 1.0 : 0.0, k == 2 ? 1.0 : 0.0};
    for (int i = 0; i < 3; ++i) out[i] = rt[3 * i] * p[0] + rt[3 * i + 1] * p[1] + rt[3 * i + 2] * p[2];
}

/* obb_corners (geometry.cpp:50-62) of {centre, axes, he} */
static void obb_corners8(const double* c, double ax[3][3], const double* he, double v[8][3]) {
    double e[3][3];
    for (int k = 0; k < 3; ++k)
        for (int j = 0; j < 3; ++j) e[k][j] = ax[k][j] * he[k];
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 3; ++j) {
            double p = (i & 1) ? c[j] + e[0][j] : c[j] - e[0][j];
            p = (i & 2) ? p + e[1][j] : p - e[1][j];
            v[i][j] = (i & 4) ? p + e[2][j] : p - e[2][j];
        }
}

static void poly_box(const double* he, const double* rt, ro_poly* p) {
    double ax[3][3];
    for (int k = 0; k < 3; ++k) rot_unit(rt, k, ax[k]);
    obb_corners8(rt + 9, ax, he, p->v); /* world.center = pose.t */
    for (int k = 0; k < 3; ++k)
        for (int j = 0; j < 3; ++j) {
            p->n[2 * k][j] = ax[k][j];
            p->n[2 * k + 1][j] = -ax[k][j];
        }
}

static double dot3v(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

static void project(const ro_poly* p, const double* axis, double* lo, double* hi) {
    *lo = INFINITY;
    *hi = -INFINITY;
    for (int i = 0; i < 8; ++i) {
        const double t = dot3v(p->v[i], axis);
        *lo = t < *lo ? t : *lo; /* std::min(lo, t) */
        *hi = *hi < t ? t : *hi; /* std::max(hi, t) */
    }
}

static int separates(const ro_poly* a, const ro_poly* b, const double* axis) {
    double alo, ahi, blo, bhi;
    project(a, axis, &alo, &ahi);
    project(b, axis, &blo, &bhi);
    return ahi < blo || bhi < alo;
}

static void edge_dirs(const ro_poly* p, double d[24][3]) {
    int k = 0;
    for (int f = 0; f < 6; ++f)
        for (int i = 0; i < 4; ++i, ++k)
            for (int j = 0; j < 3; ++j) d[k][j] = p->v[k_rings[f][(i + 1) % 4]][j] - p->v[k_rings[f][i]][j];
}

static int poly_intersect(const ro_poly* a, const ro_poly* b) {
    for (int f = 0; f < 6; ++f)
        if (separates(a, b, a->n[f])) return 0;
    for (int f = 0; f < 6; ++f)
        if (separates(a, b, b->n[f])) return 0;
    double ea[24][3], eb[24][3];
    edge_dirs(a, ea);
    edge_dirs(b, eb);
    for (int i = 0; i < 24; ++i)
        for (int j = 0; j < 24; ++j) {
            const double ax[3] = {ea[i][1] * eb[j][2] - ea[i][2] * eb[j][1], ea[i][2] * eb[j][0] - ea[i][0] * eb[j][2],
                                  ea[i][0] * eb[j][1] - ea[i][1] * eb[j][0]};
            if (dot3v(ax, ax) <= 0.0) continue;
            if (separates(a, b, ax)) return 0;
        }
    return 1;
}

int ro_box_intersect(const double* rt_a, const double* he_a, const double* rt_b, const double* he_b) {
    ro_poly a, b;
    poly_box(he_a, rt_a, &a);
    poly_box(he_b, rt_b, &b);
    return poly_intersect(&a, &b);
}

/* aabb_of_obb(apply_transform(pose, Obb{0, I, he})): centre = pose.apply(0) */
static void box_aabb(const double* he, const double* rt, double* out6) {
    double ax[3][3], c[3], v[8][3];
    for (int k = 0; k < 3; ++k) rot_unit(rt, k, ax[k]);
    for (int i = 0; i < 3; ++i) c[i] = rt[3 * i] * 0.0 + rt[3 * i + 1] * 0.0 + rt[3 * i + 2] * 0.0 + rt[9 + i];
    obb_corners8(c, ax, he, v);
    for (int j = 0; j < 3; ++j) {
        out6[j] = INFINITY;
        out6[3 + j] = -INFINITY;
    }
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 3; ++j) {
            out6[j] = fmin(out6[j], v[i][j]);
            out6[3 + j] = fmax(out6[3 + j], v[i][j]);
        }
}

int ro_exact_valid(int n_cfg, int n_bodies, const double* poses, const double* body_he, int n_obst,
                   const uint8_t* active, const double* obst_rt, const double* obst_he) {
    for (int k = 0; k < n_cfg; ++k)
        for (int b = 0; b < n_bodies; ++b) {
            const double* pose = poses + ((size_t)k * n_bodies + b) * 12;
            double bb[6];
            box_aabb(body_he + 3 * b, pose, bb);
            for (int o = 0; o < n_obst; ++o) {
                if (!active[o]) continue;
                double ob[6];
                box_aabb(obst_he + 3 * o, obst_rt + 12 * (size_t)o, ob);
                if (!aabb_overlaps(bb, ob)) continue;
                if (ro_box_intersect(pose, body_he + 3 * b, obst_rt + 12 * (size_t)o, obst_he + 3 * o)) return 0;
            }
        }
    return 1;
}

/* ---- PRM construction (proj/src/roadmap.cpp:56-102), no active obstacles ---- */

/* std::mt19937_64 as the C++ standard defines it (w=64, n=312, m=156, r=31,
 * a=0xB5026F5AA96619E9, u=29 d=0x5555555555555555, s=17 b=0x71D67FFFEDA60000,
 * t=37 c=0xFFF7EEE000000000, l=43, f=6364136223846793005). */
typedef struct {
    uint64_t mt[312];
    int i;
} ro_mt64;

static void mt64_seed(ro_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i) g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->i = 312;
}

static uint64_t mt64_next(ro_mt64* g) {
    if (g->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            const uint64_t y = (g->mt[k] & 0xFFFFFFFF80000000ull) | (g->mt[(k + 1) % 312] & 0x7FFFFFFFull);
            g->mt[k] = g->mt[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ull : 0);
        }
        g->i = 0;
    }
    uint64_t x = g->mt[g->i++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}

/* The node loop of build_prm (roadmap.cpp:65-71) with Rng::uniform (rng.hpp:17-19). */
void ro_prm_nodes(uint64_t seed, int n, int dof, const double* lo, const double* hi, double* nodes) {
    ro_mt64 g;
    mt64_seed(&g, seed);
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < dof; ++k) {
            const double u = (double)(mt64_next(&g) >> 11) * 0x1.0p-53;
            nodes[(size_t)i * dof + k] = lo[k] + (hi[k] - lo[k]) * u;
        }
}

typedef struct {
    double d;
    int32_t j;
} ro_dj;

static int dj_less(const ro_dj* a, const ro_dj* b) { return a->d < b->d || (a->d == b->d && a->j < b->j); }

static int u64_cmp(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}

/* The candidate loop (roadmap.cpp:73-93): dof_distance2 (:36-43) to every other node, the
 * k smallest (distance, j) pairs (partial_sort of pair<double, NodeId>), (min, max), sorted,
 * unique.  Selection here is a bounded insertion list (same set as partial_sort).
 * Returns the edge count (edges: cap x 2), or -(count)-1 if cap is too small. */
int64_t ro_prm_knn(const double* nodes, int n, int dof, int k, int32_t* edges, int64_t cap) {
    const int kk = k < n - 1 ? k : n - 1;
    if (kk <= 0) return 0;
    ro_dj* best = (ro_dj*)malloc(sizeof(ro_dj) * (size_t)kk);
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n * kk);
    for (int i = 0; i < n; ++i) {
        int cnt = 0;
        const double* a = nodes + (size_t)i * dof;
        for (int j = 0; j < n; ++j) {
            if (j == i) continue;
            const double* b = nodes + (size_t)j * dof;
            double d2 = 0.0;
            for (int q = 0; q < dof; ++q) {
                const double d = b[q] - a[q];
                d2 += d * d;
            }
            const ro_dj c = {d2, j};
            if (cnt == kk && !dj_less(&c, &best[kk - 1])) continue;
            int p = cnt < kk ? cnt++ : kk - 1;
            while (p > 0 && dj_less(&c, &best[p - 1])) {
                best[p] = best[p - 1];
                --p;
            }
            best[p] = c;
        }
        for (int t = 0; t < kk; ++t) {
            const uint32_t lo = (uint32_t)(i < best[t].j ? i : best[t].j), hi = (uint32_t)(i < best[t].j ? best[t].j : i);
            keys[(size_t)i * kk + t] = ((uint64_t)lo << 32) | hi;
        }
    }
    qsort(keys, (size_t)n * kk, sizeof(uint64_t), u64_cmp);
    int64_t m = 0;
    for (size_t e = 0; e < (size_t)n * kk; ++e)
        if (e == 0 || keys[e] != keys[e - 1]) keys[m++] = keys[e];
    int64_t rc = m;
    if (m > cap) rc = -m - 1;
    else
        for (int64_t e = 0; e < m; ++e) {
            edges[2 * e] = (int32_t)(keys[e] >> 32);
            edges[2 * e + 1] = (int32_t)(keys[e] & 0xffffffffu);
        }
    free(best);
    free(keys);
    return rc;
}
