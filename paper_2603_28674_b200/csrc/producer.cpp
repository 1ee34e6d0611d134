// producer.cpp — host roadmap producer: swept-volume approximations + serialized store.
//
// Free-flying robots and serial chains (robot.hpp:13-58), one box per body.  Every
// floating-point expression keeps the association of the reference's preprocessing
// (built, like the reference, with -ffp-contract=off) so the store it emits is the one the reference would
// serialize for the same roadmap; tests/test_producer.py checks that bit for bit.
// Components are independent, so they are built on a pool of std::threads.
#include "../../include/rgg_build.h"

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <chrono>
#include <atomic>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <memory>
#include <thread>
#include <vector>

#include "swept_gpu.h"


namespace {

thread_local std::string g_err;

struct V3 {
    double x, y, z;
};
inline V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator*(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double dotv(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 crossv(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline bool same(V3 a, V3 b) { return a.x == b.x && a.y == b.y && a.z == b.z; }

// Rigid transform, row-major rotation (vec3.hpp:52-100).
struct Tf {
    double r[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    V3 t{0, 0, 0};
    V3 apply(V3 p) const {
        return {r[0] * p.x + r[1] * p.y + r[2] * p.z + t.x, r[3] * p.x + r[4] * p.y + r[5] * p.z + t.y,
                r[6] * p.x + r[7] * p.y + r[8] * p.z + t.z};
    }
    V3 rotate(V3 p) const {
        return {r[0] * p.x + r[1] * p.y + r[2] * p.z, r[3] * p.x + r[4] * p.y + r[5] * p.z,
                r[6] * p.x + r[7] * p.y + r[8] * p.z};
    }
    Tf compose(const Tf& o) const {  // (this * o)
        Tf out;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                out.r[i * 3 + j] = r[i * 3 + 0] * o.r[j] + r[i * 3 + 1] * o.r[3 + j] + r[i * 3 + 2] * o.r[6 + j];
        out.t = apply(o.t);
        return out;
    }
};

// Transform::rotation_axis_angle (geometry.cpp:13-29), Rodrigues.
Tf axis_angle(V3 axis, double angle) {
    const double len = std::sqrt(dotv(axis, axis));
    const double kx = axis.x / len, ky = axis.y / len, kz = axis.z / len;
    const double c = std::cos(angle), s = std::sin(angle), v = 1.0 - c;
    Tf tf;
    tf.r[0] = kx * kx * v + c;
    tf.r[1] = kx * ky * v - kz * s;
    tf.r[2] = kx * kz * v + ky * s;
    tf.r[3] = ky * kx * v + kz * s;
    tf.r[4] = ky * ky * v + c;
    tf.r[5] = ky * kz * v - kx * s;
    tf.r[6] = kz * kx * v - ky * s;
    tf.r[7] = kz * ky * v + kx * s;
    tf.r[8] = kz * kz * v + c;
    return tf;
}

struct Box {
    V3 c;
    V3 ax[3];
    V3 he;
};

// obb_corners (geometry.cpp:50-62): corner i takes +axis k iff bit k of i.
void corners_of(const Box& o, V3 out[8]) {
    const V3 e0 = o.ax[0] * o.he.x, e1 = o.ax[1] * o.he.y, e2 = o.ax[2] * o.he.z;
    for (int i = 0; i < 8; ++i) {
        V3 p = (i & 1) ? o.c + e0 : o.c - e0;
        p = (i & 2) ? p + e1 : p - e1;
        p = (i & 4) ? p + e2 : p - e2;
        out[i] = p;
    }
}

// ---- obb_from_points (geometry.cpp:64-195): PCA frame + per-axis sweep

void jacobi3(double m[3][3], double vals[3], V3 vecs[3]) {
    double v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    for (int sweep = 0; sweep < 64; ++sweep) {
        const double off = std::fabs(m[0][1]) + std::fabs(m[0][2]) + std::fabs(m[1][2]);
        if (off == 0.0) break;
        for (int p = 0; p < 2; ++p) {
            for (int q = p + 1; q < 3; ++q) {
                if (m[p][q] == 0.0) continue;
                const double theta = (m[q][q] - m[p][p]) / (2.0 * m[p][q]);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0);
                const double s = t * c;
                for (int k = 0; k < 3; ++k) {
                    const double a = m[k][p], b = m[k][q];
                    m[k][p] = c * a - s * b;
                    m[k][q] = s * a + c * b;
                }
                for (int k = 0; k < 3; ++k) {
                    const double a = m[p][k], b = m[q][k];
                    m[p][k] = c * a - s * b;
                    m[q][k] = s * a + c * b;
                }
                for (int k = 0; k < 3; ++k) {
                    const double a = v[k][p], b = v[k][q];
                    v[k][p] = c * a - s * b;
                    v[k][q] = s * a + c * b;
                }
            }
        }
    }
    for (int i = 0; i < 3; ++i) {
        vals[i] = m[i][i];
        vecs[i] = {v[0][i], v[1][i], v[2][i]};
    }
}

inline double min_ref(double a, double b) { return b < a ? b : a; }  // std::min
inline double max_ref(double a, double b) { return a < b ? b : a; }  // std::max

struct Extent {
    double lo[3], hi[3], vol;
};

Extent extents(const std::vector<V3>& pts, const V3 ax[3]) {
    Extent f;
    for (int k = 0; k < 3; ++k) {
        f.lo[k] = INFINITY;
        f.hi[k] = -INFINITY;
    }
    for (const V3& p : pts) {
        for (int k = 0; k < 3; ++k) {
            const double t = dotv(p, ax[k]);
            f.lo[k] = min_ref(f.lo[k], t);
            f.hi[k] = max_ref(f.hi[k], t);
        }
    }
    f.vol = (f.hi[0] - f.lo[0]) * (f.hi[1] - f.lo[1]) * (f.hi[2] - f.lo[2]);
    return f;
}

Box fit_box(const std::vector<V3>& pts) {
    Box box{{0, 0, 0}, {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}}, {0, 0, 0}};
    if (pts.size() == 1) {
        box.c = pts[0];
        return box;
    }
    V3 mean{0, 0, 0};
    for (const V3& p : pts) mean = mean + p;
    mean = mean * (1.0 / static_cast<double>(pts.size()));
    double cov[3][3] = {};
    for (const V3& p : pts) {
        const V3 d = p - mean;
        const double dc[3] = {d.x, d.y, d.z};
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) cov[i][j] += dc[i] * dc[j];
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) cov[i][j] /= static_cast<double>(pts.size());
    double vals[3];
    V3 axes[3];
    jacobi3(cov, vals, axes);
    // largest variance first (stable), right-handed
    int ord[3] = {0, 1, 2};
    for (int i = 1; i < 3; ++i)
        for (int j = i; j > 0 && vals[ord[j]] > vals[ord[j - 1]]; --j) std::swap(ord[j], ord[j - 1]);
    V3 best[3] = {axes[ord[0]], axes[ord[1]], axes[ord[2]]};
    best[2] = crossv(best[0], best[1]);
    double best_vol = extents(pts, best).vol;
    constexpr double kStep = 3.0 * 3.141592653589793 / 180.0;
    for (int k = 0; k < 3; ++k) {
        const V3 pivot = best[k];
        V3 win[3] = {best[0], best[1], best[2]};
        for (int step = -5; step <= 5; ++step) {
            if (step == 0) continue;
            const Tf rot = axis_angle(pivot, step * kStep);
            V3 cand[3];
            for (int j = 0; j < 3; ++j) cand[j] = rot.rotate(best[j]);
            const double vol = extents(pts, cand).vol;
            if (vol < best_vol) {
                best_vol = vol;
                for (int j = 0; j < 3; ++j) win[j] = cand[j];
            }
        }
        for (int j = 0; j < 3; ++j) best[j] = win[j];
    }
    const Extent f = extents(pts, best);
    box.c = best[0] * ((f.lo[0] + f.hi[0]) * 0.5) + best[1] * ((f.lo[1] + f.hi[1]) * 0.5) +
            best[2] * ((f.lo[2] + f.hi[2]) * 0.5);
    for (int k = 0; k < 3; ++k) box.ax[k] = best[k];
    box.he = {(f.hi[0] - f.lo[0]) * 0.5, (f.hi[1] - f.lo[1]) * 0.5, (f.hi[2] - f.lo[2]) * 0.5};
    return box;
}

// ---- predicates shared with the serialized store (kernels_scalar.cpp:7-96)

void sat_prep(const double* c, double* s) {
    for (int k = 0; k < 3; ++k) {
        const int hi = (1 << k) * 3;
        for (int j = 0; j < 3; ++j) s[3 + 3 * k + j] = 0.5 * (c[hi + j] - c[j]);
    }
    for (int j = 0; j < 3; ++j) s[j] = ((c[j] + s[3 + j]) + s[6 + j]) + s[9 + j];
    for (int k = 0; k < 3; ++k) {
        const double* e = s + 3 + 3 * k;
        const double n2 = (e[0] * e[0] + e[1] * e[1]) + e[2] * e[2];
        if (n2 > 0.0) {
            const double len = std::sqrt(n2);
            for (int j = 0; j < 3; ++j) s[12 + 3 * k + j] = e[j] / len;
        } else {
            s[12 + 3 * k] = s[13 + 3 * k] = s[14 + 3 * k] = 0.0;
        }
    }
}

void seg_prep(V3 a, V3 b, double* p) {
    p[0] = a.x, p[1] = a.y, p[2] = a.z;
    p[3] = b.x - a.x, p[4] = b.y - a.y, p[5] = b.z - a.z;
    p[6] = (p[3] * p[3] + p[4] * p[4]) + p[5] * p[5];
}

double point_seg_dist(V3 a, V3 b, V3 c) {
    double s[7];
    seg_prep(a, b, s);
    const double px = c.x - s[0], py = c.y - s[1], pz = c.z - s[2];
    double t = 0.0;
    if (s[6] > 0.0) {
        t = ((px * s[3] + py * s[4]) + pz * s[5]) / s[6];
        t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    }
    const double qx = px - t * s[3], qy = py - t * s[4], qz = pz - t * s[5];
    return std::sqrt((qx * qx + qy * qy) + qz * qz);
}

// ---- inner approximation (swept.cpp:23-228)

struct Sph {
    V3 c;
    double r;
};

std::vector<Sph> inner_spheres(V3 he, int count) {
    const double h[3] = {he.x, he.y, he.z};
    const double radius = std::min({h[0], h[1], h[2]});
    int axis = 0;
    for (int k = 1; k < 3; ++k)
        if (h[k] > h[axis]) axis = k;
    const double span = h[axis] - radius;
    std::vector<Sph> out;
    for (int i = 0; i < count; ++i) {
        const double t = count == 1 ? 0.0 : -span + (2.0 * span) * (static_cast<double>(i) / (count - 1));
        V3 c{0, 0, 0};
        (axis == 0 ? c.x : axis == 1 ? c.y : c.z) = t;
        out.push_back({c, radius});
    }
    return out;
}

int sphere_count(V3 he) {
    const double longest = std::max({he.x, he.y, he.z}), shortest = std::min({he.x, he.y, he.z});
    return std::max(1, static_cast<int>(std::ceil(longest / shortest)));
}

bool covers(const std::vector<V3>& pts, int j, int p, double radius) {
    for (int m = j + 1; m < p; ++m)
        if (!(point_seg_dist(pts[j], pts[p], pts[m]) < radius)) return false;
    return true;
}

std::vector<int> simplify(const std::vector<V3>& pts, double radius) {
    const int n = static_cast<int>(pts.size());
    std::vector<int> keep{0};
    int j = 0;
    while (j < n - 1) {
        int p = j + 1;
        while (p + 1 <= n - 1 && covers(pts, j, p + 1, radius)) ++p;
        keep.push_back(p);
        j = p;
    }
    return keep;
}

struct Spline {
    std::vector<V3> pts;
    double radius;
    int sphere;
};

void cap_split(const std::vector<V3>& raw, const std::vector<int>& kept, double radius, double tol, int K, int sphere,
               std::vector<Spline>& out) {
    const int q = static_cast<int>(kept.size()) - 1;
    if (q <= K) {
        Spline s{{}, radius, sphere};
        for (int i : kept) s.pts.push_back(raw[i]);
        out.push_back(std::move(s));
        return;
    }
    std::vector<int> sub;
    for (int i = 0; i <= K; ++i) sub.push_back(kept[static_cast<size_t>(std::llround(static_cast<double>(i) * q / K))]);
    bool ok = true;
    for (size_t i = 0; ok && i + 1 < sub.size(); ++i) ok = covers(raw, sub[i], sub[i + 1], tol);
    if (ok) {
        Spline s{{}, radius, sphere};
        for (int i : sub) s.pts.push_back(raw[i]);
        out.push_back(std::move(s));
        return;
    }
    for (int start = 0; start < q; start += K) {
        const int stop = std::min(start + K, q);
        Spline s{{}, radius, sphere};
        for (int i = start; i <= stop; ++i) s.pts.push_back(raw[kept[i]]);
        out.push_back(std::move(s));
    }
}

struct Comp {
    std::vector<Box> over;                   // per body
    std::vector<std::vector<Spline>> under;  // per body
    std::vector<Tf> fk;  // forward_kinematics per configuration, body-minor (kept for the exact resolve)
};

// RobotModel (robot.hpp:13-58) with its default inner spheres (default_body_spheres,
// swept.cpp:52-65) and their certified spline radii.
struct Body {
    V3 he;
    Tf local;
    std::vector<Sph> spheres;
    std::vector<double> lipschitz, radius, tol;
};

struct Robot {
    bool chain = false;  // KinematicsType::SerialChain
    int dof = 6;
    std::vector<Body> bodies;
    std::vector<V3> axis, offset;  // joints (serial chain)
};

bool finite3(V3 v) { return std::isfinite(v.x) && std::isfinite(v.y) && std::isfinite(v.z); }

// Transform::rotation_valid (geometry.cpp:36-48)
bool rotation_valid(const Tf& t, double tol) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double v = 0.0;
            for (int q = 0; q < 3; ++q) v += t.r[q * 3 + i] * t.r[q * 3 + j];
            if (std::fabs(v - (i == j ? 1.0 : 0.0)) > tol) return false;
        }
    const double* r = t.r;
    const double det = r[0] * (r[4] * r[8] - r[5] * r[7]) - r[1] * (r[3] * r[8] - r[5] * r[6]) +
                       r[2] * (r[3] * r[7] - r[4] * r[6]);
    return std::fabs(det - 1.0) <= tol;
}

// RobotModel::validate (robot.cpp:17-37), BodySpheres::validate (swept.cpp:9-21),
// center_lipschitz (swept.cpp:164-178), certified_spline_radius (:180-186)
Robot make_robot(const rgg_robot_view& v, double eps) {
    if (v.kinematics != RGG_ROBOT_FREE_FLYING && v.kinematics != RGG_ROBOT_SERIAL_CHAIN)
        throw std::invalid_argument("robot kinematics must be free flying or serial chain");
    if (v.n_bodies < 1 || !v.half_extents) throw std::invalid_argument("robot needs at least one body");
    Robot r;
    r.chain = v.kinematics == RGG_ROBOT_SERIAL_CHAIN;
    for (int32_t b = 0; b < v.n_bodies; ++b) {
        Body bd;
        bd.he = {v.half_extents[3 * b], v.half_extents[3 * b + 1], v.half_extents[3 * b + 2]};
        if (!(bd.he.x > 0 && bd.he.y > 0 && bd.he.z > 0)) throw std::invalid_argument("body half extents must be positive");
        if (v.local) {
            std::memcpy(bd.local.r, v.local + 12 * b, 9 * sizeof(double));
            bd.local.t = {v.local[12 * b + 9], v.local[12 * b + 10], v.local[12 * b + 11]};
        }
        if (!finite3(bd.local.t) || !rotation_valid(bd.local, 1e-9)) throw std::invalid_argument("body local frame invalid");
        r.bodies.push_back(bd);
    }
    if (r.chain) {
        if (!v.joint_axis || !v.joint_offset) throw std::invalid_argument("serial chain needs one joint per body");
        for (int32_t j = 0; j < v.n_bodies; ++j) {
            const V3 ax{v.joint_axis[3 * j], v.joint_axis[3 * j + 1], v.joint_axis[3 * j + 2]};
            const V3 of{v.joint_offset[3 * j], v.joint_offset[3 * j + 1], v.joint_offset[3 * j + 2]};
            if (!finite3(of) || !(std::sqrt(dotv(ax, ax)) > 0)) throw std::invalid_argument("joint axis/offset invalid");
            r.axis.push_back(ax);
            r.offset.push_back(of);
        }
        if (v.n_bodies > 64) throw std::invalid_argument("serial chain: at most 64 joints");
        r.dof = v.n_bodies;
    }
    for (size_t b = 0; b < r.bodies.size(); ++b) {
        Body& bd = r.bodies[b];
        bd.spheres = inner_spheres(bd.he, sphere_count(bd.he));
        for (const Sph& s : bd.spheres) {
            if (!(s.r > 0)) throw std::invalid_argument("body sphere radius must be positive");
            if (std::fabs(s.c.x) + s.r > bd.he.x || std::fabs(s.c.y) + s.r > bd.he.y || std::fabs(s.c.z) + s.r > bd.he.z)
                throw std::invalid_argument("body sphere escapes its box");
            const V3 p = bd.local.apply(s.c);
            double L;
            if (!r.chain) {
                L = std::sqrt(1.0 + 3.0 * dotv(p, p));
            } else {
                double span = std::sqrt(dotv(p, p));
                for (size_t j = 0; j <= b; ++j) span += std::sqrt(dotv(r.offset[j], r.offset[j]));
                L = span * std::sqrt(static_cast<double>(b + 1));
            }
            const double half_step = 0.5 * L * eps;
            const double r2 = s.r * s.r - half_step * half_step;
            double rad = 0.0;
            if (r2 > 0.0) rad = std::sqrt(r2) * (1.0 - 0.1) - 1e-9;
            bd.lipschitz.push_back(L);
            bd.radius.push_back(rad);
            bd.tol.push_back(std::sqrt(s.r * s.r - 0.25 * L * eps * L * eps) - rad - 1e-9);
        }
    }
    return r;
}

// forward_kinematics (robot.cpp:66-84): one pose per body
void forward_kinematics(const Robot& r, const double* c, Tf* out) {
    if (!r.chain) {
        Tf world = axis_angle({0, 0, 1}, c[5]).compose(axis_angle({0, 1, 0}, c[4])).compose(axis_angle({1, 0, 0}, c[3]));
        world.t = {c[0], c[1], c[2]};
        for (size_t b = 0; b < r.bodies.size(); ++b) out[b] = world.compose(r.bodies[b].local);
        return;
    }
    Tf acc;
    for (size_t j = 0; j < r.axis.size(); ++j) {
        Tf tr;
        tr.t = r.offset[j];
        const Tf jt = tr.compose(axis_angle(r.axis[j], c[j]));
        acc = acc.compose(jt);
        out[j] = acc.compose(r.bodies[j].local);
    }
}

// discretize_edge's configuration count (robot.cpp:39-64)
int config_count(const double* a, const double* b, int dof, double eps) {
    double len2 = 0.0;
    for (int i = 0; i < dof; ++i) {
        const double d = b[i] - a[i];
        len2 += d * d;
    }
    return std::max(2, static_cast<int>(std::ceil(std::sqrt(len2) / eps)) + 1);
}

// pose_out (gpu_fit): the component's forward-kinematics poses, 12 doubles each,
// body-major (body b's n poses at pose_out + 12 * n * b)
Comp build_comp(const Robot& rb, const double* a, const double* b, double eps, int K, bool keep_poses, bool gpu_fit,
                bool gpu_inner, double* pose_out) {
    const int dof = rb.dof, B = static_cast<int>(rb.bodies.size());
    // discretize_edge (robot.cpp:39-64)
    const int n = config_count(a, b, dof, eps);
    std::vector<Tf> fk(static_cast<size_t>(n) * B);
    double cfg[64];
    for (int i = 0; i < n; ++i) {
        if (i == 0) {
            std::memcpy(cfg, a, dof * sizeof(double));
        } else if (i == n - 1) {
            std::memcpy(cfg, b, dof * sizeof(double));
        } else {
            const double t = static_cast<double>(i) / static_cast<double>(n - 1);
            for (int q = 0; q < dof; ++q) cfg[q] = a[q] + (b[q] - a[q]) * t;
        }
        Tf* T = &fk[static_cast<size_t>(i) * B];
        forward_kinematics(rb, cfg, T);
        if (pose_out)
            for (int bd = 0; bd < B; ++bd) {
                double* d = pose_out + 12 * (static_cast<size_t>(bd) * n + i);
                std::memcpy(d, T[bd].r, 9 * sizeof(double));
                d[9] = T[bd].t.x, d[10] = T[bd].t.y, d[11] = T[bd].t.z;
            }
    }
    Comp comp;
    comp.over.resize(B);
    comp.under.resize(B);
    // build_outer_approx (swept.cpp:100-118); with gpu_fit the boxes are fitted later on the GPU
    if (!gpu_fit) {
        std::vector<V3> cloud;
        cloud.reserve(static_cast<size_t>(n) * 8);
        for (int bd = 0; bd < B; ++bd) {
            cloud.clear();
            for (int i = 0; i < n; ++i) {
                const Tf& T = fk[static_cast<size_t>(i) * B + bd];
                Box w;
                w.c = T.apply({0, 0, 0});
                w.ax[0] = T.rotate({1, 0, 0});
                w.ax[1] = T.rotate({0, 1, 0});
                w.ax[2] = T.rotate({0, 0, 1});
                w.he = rb.bodies[bd].he;
                V3 cs[8];
                corners_of(w, cs);
                cloud.insert(cloud.end(), cs, cs + 8);
            }
            comp.over[bd] = fit_box(cloud);
        }
    }
    if (gpu_inner) {  // the inner approximation runs on the GPU too
        if (keep_poses) comp.fk = std::move(fk);
        return comp;
    }
    // build_inner_approx (swept.cpp:188-228)
    for (int bd = 0; bd < B; ++bd) {
        const Body& body = rb.bodies[bd];
        for (size_t si = 0; si < body.spheres.size(); ++si) {
            const double rad = body.radius[si];
            if (rad <= 0.0) continue;
            const double step_bound = body.lipschitz[si] * eps;
            std::vector<V3> raw;
            bool step_ok = true;
            for (int i = 0; i < n; ++i) {
                const V3 c = fk[static_cast<size_t>(i) * B + bd].apply(body.spheres[si].c);
                if (!raw.empty()) {
                    const V3 d = c - raw.back();
                    if (std::sqrt(dotv(d, d)) > step_bound) step_ok = false;
                }
                if (raw.empty() || !same(c, raw.back())) raw.push_back(c);
            }
            if (!step_ok) continue;
            const std::vector<int> kept = simplify(raw, body.tol[si]);
            cap_split(raw, kept, rad, body.tol[si], K, static_cast<int>(si), comp.under[bd]);
        }
    }
    if (keep_poses) comp.fk = std::move(fk);
    return comp;
}

// ---- the reference's binary roadmap file (save_roadmap / load_roadmap,
// roadmap_io.cpp:150-301): "RGGRDMP1", u32 version 1, then little-endian sections
// (robot; sphere sets per body; epsilon, segment cap; nodes; edges; per component the
// body OBBs and the body splines) and a CRC-32 of everything before it.

// CRC-32 (reflected, polynomial 0xEDB88320, initial and final xor 0xFFFFFFFF), the
// checksum of roadmap_io.cpp:125-138
uint32_t crc32_of(const uint8_t* p, size_t n) {
    static uint32_t table[256];
    static const bool ready = [] {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c >> 1) ^ ((c & 1u) ? 0xEDB88320u : 0u);
            table[i] = c;
        }
        return true;
    }();
    (void)ready;
    uint32_t c = 0xFFFFFFFFu;
    for (size_t i = 0; i < n; ++i) c = table[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
    return ~c;
}

// load_roadmap's error kinds (roadmap_io.hpp:10-16)
struct FileError : std::runtime_error {
    int kind;
    FileError(int k, const std::string& m) : std::runtime_error(m), kind(k) {}
};

struct ByteReader {
    const uint8_t* p;
    size_t n, at = 0;
    void need(size_t k) const {
        if (at + k > n) throw FileError(RGG_ROADMAP_TRUNCATED, "roadmap file truncated");
    }
    uint8_t u8() {
        need(1);
        return p[at++];
    }
    uint32_t u32() {
        need(4);
        uint32_t v = 0;
        for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(p[at + i]) << (8 * i);
        at += 4;
        return v;
    }
    double f64() {
        need(8);
        uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(p[at + i]) << (8 * i);
        at += 8;
        double d;
        std::memcpy(&d, &v, 8);
        return d;
    }
    V3 v3() {
        const double x = f64(), y = f64(), z = f64();
        return {x, y, z};
    }
    // a count bounded like the reference's sanity_count (roadmap_io.cpp:90-93)
    uint32_t count(uint32_t limit, const char* what) {
        const uint32_t v = u32();
        if (v > limit) throw FileError(RGG_ROADMAP_TRUNCATED, std::string("implausible count for ") + what);
        return v;
    }
};

}  // namespace

struct rgg_built {
    int32_t N = 0, B = 1, S = 1;
    std::vector<double> edge_sat, comp_aabb, segs, spline_r, obb15;
    std::vector<int32_t> row_off;
    std::vector<int64_t> pose_off;  // RGG_BUILD_POSES: N+1
    std::vector<double> poses;      // pose_off[N] * B * 12 (body-minor per configuration)
    // RGG_BUILD_KEEP_GEOMETRY: what save_roadmap writes (the robot, the roadmap and the
    // ComponentSet's spheres, resolution, cap and geometry)
    bool kept = false;
    Robot robot;
    std::vector<double> rb_he, rb_local, rb_axis, rb_offset;
    int32_t kinematics = 0, dof = 0, K = 16;
    double eps = 0.0;
    std::vector<double> nodes;
    std::vector<int32_t> edges;
    std::vector<Comp> comps;
};

extern "C" {

const char* rgg_build_last_error(void) { return g_err.c_str(); }

int rgg_build_layout(const double* he3, int32_t n_nodes, const double* nodes, int32_t n_edges, const int32_t* edges,
                     double eps, int32_t K, int32_t threads, rgg_built** out) {
    return rgg_build_layout_ex(he3, n_nodes, nodes, n_edges, edges, eps, K, threads, 0, out);
}

int rgg_build_layout_ex(const double* he3, int32_t n_nodes, const double* nodes, int32_t n_edges,
                        const int32_t* edges, double eps, int32_t K, int32_t threads, int32_t flags,
                        rgg_built** out) {
    if (!he3) {
        g_err = "null robot half extents";
        return -1;
    }
    rgg_robot_view v{};
    v.kinematics = RGG_ROBOT_FREE_FLYING;
    v.n_bodies = 1;
    v.half_extents = he3;  // make_free_flying_box (robot.cpp:86-92): one body, identity local frame
    return rgg_build_layout_robot(&v, n_nodes, nodes, n_edges, edges, eps, K, threads, flags, out);
}

int rgg_build_layout_robot(const rgg_robot_view* robot, int32_t n_nodes, const double* nodes, int32_t n_edges,
                           const int32_t* edges, double eps, int32_t K, int32_t threads, int32_t flags,
                           rgg_built** out) {
    const bool keep_poses = (flags & RGG_BUILD_POSES) != 0;
    static const bool dbg = std::getenv("RGG_DEBUG_PRODUCER") != nullptr;
    auto t_mark = std::chrono::steady_clock::now();
    const auto mark = [&](const char* what) {
        if (!dbg) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[producer] %-14s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(t - t_mark).count());
        t_mark = t;
    };
    const bool gpu_fit = (flags & (RGG_BUILD_GPU_FIT | RGG_BUILD_GPU_INNER)) != 0;
    const bool gpu_inner = (flags & RGG_BUILD_GPU_INNER) != 0;
    try {
        if (!out || !robot) throw std::invalid_argument("null robot or output");
        if (!(eps > 0)) throw std::invalid_argument("resolution must be positive");
        if (K < 1) throw std::invalid_argument("segment cap must be >= 1");
        if (n_nodes < 0 || n_edges < 0 || (n_nodes > 0 && !nodes) || (n_edges > 0 && !edges))
            throw std::invalid_argument("bad roadmap arrays");
        for (int32_t e = 0; e < n_edges; ++e)
            if (edges[2 * e] < 0 || edges[2 * e] >= n_nodes || edges[2 * e + 1] < 0 || edges[2 * e + 1] >= n_nodes)
                throw std::invalid_argument("edge endpoint out of range");
        const Robot rb = make_robot(*robot, eps);
        const int dof = rb.dof;
        const int32_t B = static_cast<int32_t>(rb.bodies.size());
        if (gpu_inner && B != 1) throw std::invalid_argument("the GPU inner approximation takes single-body robots");
        const int32_t N = n_nodes + n_edges;
        std::vector<Comp> comps(static_cast<size_t>(N));
        const auto ends = [&](int32_t c, const double** a, const double** b) {
            if (c < n_nodes) {
                *a = *b = nodes + dof * static_cast<size_t>(c);
            } else {
                const int32_t e = c - n_nodes;
                *a = nodes + dof * static_cast<size_t>(edges[2 * e]);
                *b = nodes + dof * static_cast<size_t>(edges[2 * e + 1]);
            }
        };
        int nt = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
        nt = std::max(1, std::min(nt, 256));
        const auto parallel = [&](int32_t n, auto&& fn) {  // fn(c) for c in [0, n) on the pool
            std::atomic<int32_t> at{0};
            std::string perr;
            std::atomic<bool> pfail{false};
            auto run = [&] {
                try {
                    for (int32_t c0; (c0 = at.fetch_add(1024)) < n && !pfail;)
                        for (int32_t c = c0; c < std::min(n, c0 + 1024); ++c) fn(c);
                } catch (const std::exception& ex) {
                    if (!pfail.exchange(true)) perr = ex.what();
                }
            };
            std::vector<std::thread> ts;
            for (int i = 1; i < nt; ++i) ts.emplace_back(run);
            run();
            for (auto& t : ts) t.join();
            if (pfail) throw std::logic_error(perr);
        };
        // components [c_lo, c_hi) on the pool; gpu_fit: poses into `stage` from configuration `cfg0`
        const auto run_components = [&](int32_t c_lo, int32_t c_hi, double* stage, const int64_t* pose_off,
                                        int64_t cfg0) {
            std::atomic<int32_t> next{c_lo};
            std::string err;
            std::atomic<bool> failed{false};
            auto work = [&] {
                try {
                    for (;;) {
                        const int32_t c0 = next.fetch_add(256);
                        if (c0 >= c_hi || failed) break;
                        for (int32_t c = c0; c < std::min(c_hi, c0 + 256); ++c) {
                            const double *a, *b;
                            ends(c, &a, &b);
                            comps[c] = build_comp(rb, a, b, eps, K, keep_poses, gpu_fit, gpu_inner,
                                                  stage ? stage + 12 * static_cast<size_t>(pose_off[c] - cfg0) * B
                                                        : nullptr);
                        }
                    }
                } catch (const std::exception& ex) {
                    if (!failed.exchange(true)) err = ex.what();
                }
            };
            std::vector<std::thread> pool;
            for (int i = 1; i < nt; ++i) pool.emplace_back(work);
            work();
            for (auto& t : pool) t.join();
            if (failed) throw std::runtime_error(err);
        };
        void* fit = nullptr;
        if (!gpu_fit) {
            run_components(0, N, nullptr, nullptr, 0);
        } else {
            // the poses stream to the GPU in chunks of <= kChunk poses through two pinned
            // buffers: a chunk's copy overlaps the production of the next.  One fit unit per
            // (component, body), its poses contiguous (build_comp's body-major pose_out)
            constexpr int64_t kChunk = 1 << 19;
            std::vector<int64_t> pose_off(static_cast<size_t>(N) + 1, 0);
            for (int32_t c = 0; c < N; ++c) {
                const double *a, *b;
                ends(c, &a, &b);
                pose_off[c + 1] = pose_off[c] + config_count(a, b, dof, eps);
            }
            std::vector<int64_t> unit_off(static_cast<size_t>(N) * B + 1, 0);
            for (int32_t c = 0; c < N; ++c)
                for (int32_t bd = 0; bd < B; ++bd)
                    unit_off[static_cast<size_t>(c) * B + bd] = pose_off[c] * B + bd * (pose_off[c + 1] - pose_off[c]);
            unit_off[static_cast<size_t>(N) * B] = pose_off[N] * B;
            double cs[22];
            constexpr double kStep = 3.0 * 3.141592653589793 / 180.0;
            for (int step = -5; step <= 5; ++step) {
                cs[2 * (step + 5)] = std::cos(step * kStep);
                cs[2 * (step + 5) + 1] = std::sin(step * kStep);
            }
            std::vector<double> he(static_cast<size_t>(B) * 3);
            for (int32_t bd = 0; bd < B; ++bd)
                he[3 * bd] = rb.bodies[bd].he.x, he[3 * bd + 1] = rb.bodies[bd].he.y, he[3 * bd + 2] = rb.bodies[bd].he.z;
            int64_t max_chunk = 0;
            for (int32_t c = 0; c < N; ++c) max_chunk = std::max(max_chunk, pose_off[c + 1] - pose_off[c]);
            const int64_t chunk = std::max(kChunk / B, max_chunk);  // configurations per staging buffer
            fit = rggp_fit_begin(unit_off.data(), N * B, he.data(), B, cs, chunk * B, -1);  // current device
            if (!fit) throw std::runtime_error("GPU box fit: CUDA initialisation failed");
            try {
                int slot = 0;
                for (int32_t c_lo = 0; c_lo < N; slot ^= 1) {
                    int32_t c_hi = c_lo + 1;
                    while (c_hi < N && pose_off[c_hi + 1] - pose_off[c_lo] <= chunk) ++c_hi;
                    double* stage = rggp_fit_staging(fit, slot);
                    if (!stage) throw std::runtime_error("GPU box fit: staging failed");
                    run_components(c_lo, c_hi, stage, pose_off.data(), pose_off[c_lo]);
                    if (rggp_fit_push(fit, slot, pose_off[c_lo] * B, (pose_off[c_hi] - pose_off[c_lo]) * B) != 0)
                        throw std::runtime_error("GPU box fit: copy failed");
                    c_lo = c_hi;
                }
            } catch (...) {
                rggp_fit_end(fit);
                throw;
            }
        }
        mark("components");
        if (gpu_fit) {
            // obb_from_points of every (component, body) on the GPU (swept_gpu.cu), from the streamed poses
            std::vector<double> boxes(static_cast<size_t>(N) * B * 15);
            InnerSpec spec;
            const Body& b0 = rb.bodies[0];
            spec.nsph = static_cast<int32_t>(b0.spheres.size());
            spec.K = K;
            for (size_t si = 0; si < b0.spheres.size(); ++si) {
                spec.centre.insert(spec.centre.end(), {b0.spheres[si].c.x, b0.spheres[si].c.y, b0.spheres[si].c.z});
                spec.radius.push_back(b0.radius[si]);
                spec.step_bound.push_back(b0.lipschitz[si] * eps);
                spec.tol.push_back(b0.tol[si]);
            }
            InnerOut inner;
            const int rc = rggp_fit_finish(fit, boxes.data(), gpu_inner ? &spec : nullptr, &inner);
            if (rc != 0) throw std::runtime_error("GPU box fit failed (CUDA error " + std::to_string(rc) + ")");
            // the splines, component by component (build_comp's order: spheres, then cap_split's)
            const int32_t nsph = gpu_inner ? spec.nsph : 0;
            std::vector<int64_t> so(static_cast<size_t>(N) + 1, 0), po(static_cast<size_t>(N) + 1, 0);
            {
                int64_t q = 0;
                for (int32_t c = 0; c < N; ++c) {
                    int64_t pts = 0;
                    for (int32_t si = 0; si < nsph; ++si)
                        for (int32_t s = 0; s < inner.nspl[static_cast<size_t>(c) * nsph + si]; ++s) pts += inner.npts[q++];
                    so[c + 1] = q;
                    po[c + 1] = po[c] + pts;
                }
            }
            parallel(N, [&](int32_t c) {
                int64_t q = so[c], p = po[c];
                for (int32_t si = 0; si < nsph; ++si)
                    for (int32_t s = 0; s < inner.nspl[static_cast<size_t>(c) * nsph + si]; ++s, ++q) {
                        Spline sp{{}, b0.radius[si], si};
                        sp.pts.reserve(inner.npts[q]);
                        for (int32_t j = 0; j < inner.npts[q]; ++j, ++p)
                            sp.pts.push_back({inner.pts[3 * p], inner.pts[3 * p + 1], inner.pts[3 * p + 2]});
                        comps[c].under[0].push_back(std::move(sp));
                    }
            });
            for (int32_t c = 0; c < N; ++c)
                for (int32_t bd = 0; bd < B; ++bd) {
                    const double* o = &boxes[15 * (static_cast<size_t>(c) * B + bd)];
                    Box& bx = comps[c].over[bd];
                    bx.c = {o[0], o[1], o[2]};
                    for (int q = 0; q < 3; ++q) bx.ax[q] = {o[3 + 3 * q], o[4 + 3 * q], o[5 + 3 * q]};
                    bx.he = {o[12], o[13], o[14]};
                }
        }

        mark("box fit");
        // ---- serialize (batch_layout.cpp:21-146), components in parallel
        rgg_built* L = new rgg_built();
        std::unique_ptr<rgg_built> own(L);
        L->N = N;
        L->B = B;
        // slots: spheres-per-body x the worst split factor; the splines of (body b, sphere s)
        // take slots s*max_parts + 0, 1, ... of body b
        int32_t max_spheres = 1;
        std::vector<int32_t> sph_base(B + 1, 0);  // (body, sphere) index base
        for (int32_t bd = 0; bd < B; ++bd) {
            const int32_t ns = static_cast<int32_t>(rb.bodies[bd].spheres.size());
            max_spheres = std::max(max_spheres, ns);
            sph_base[bd + 1] = sph_base[bd] + ns;
        }
        const int32_t nbs = sph_base[B];
        std::vector<std::atomic<int32_t>> sph_parts(std::max(nbs, 1));
        for (auto& x : sph_parts) x = 0;
        parallel(N, [&](int32_t c) {
            thread_local std::vector<int32_t> parts;
            parts.assign(std::max(nbs, 1), 0);
            for (int32_t bd = 0; bd < B; ++bd)
                for (const Spline& sp : comps[c].under[bd]) {
                    const int32_t x = sph_base[bd] + sp.sphere;
                    const int32_t p = ++parts[x];
                    for (int32_t cur = sph_parts[x]; p > cur && !sph_parts[x].compare_exchange_weak(cur, p);) {
                    }
                }
        });
        int32_t max_parts = 1;
        for (int32_t x = 0; x < nbs; ++x) max_parts = std::max<int32_t>(max_parts, sph_parts[x]);
        const int32_t S = max_spheres * max_parts;
        L->S = S;
        const size_t NB = static_cast<size_t>(N) * B;
        L->spline_r.assign(static_cast<size_t>(B) * S, 0.0);
        L->edge_sat.resize(NB * 21);
        L->comp_aabb.resize(static_cast<size_t>(N) * 6);
        L->obb15.resize(NB * 15);
        L->row_off.assign(NB * S + 1, 0);
        std::vector<int32_t> count(NB * S, 0);
        // a slot's spline radius is its sphere's (every spline of sphere s carries it, so the
        // reference's consistency check, batch_layout.cpp:73-79, holds); unused slots stay 0
        for (int32_t bd = 0; bd < B; ++bd)
            for (int32_t s = 0; s < sph_base[bd + 1] - sph_base[bd]; ++s)
                for (int32_t j = 0; j < sph_parts[sph_base[bd] + s]; ++j)
                    L->spline_r[static_cast<size_t>(bd) * S + s * max_parts + j] = rb.bodies[bd].radius[s];
        parallel(N, [&](int32_t c) {
            const Comp& cp = comps[c];
            // component_aabb = Aabb::empty() expanded by every body box's corners (aabb_of_obb)
            double box[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
            for (int32_t bd = 0; bd < B; ++bd) {
                const size_t u = static_cast<size_t>(c) * B + bd;
                V3 cs[8];
                corners_of(cp.over[bd], cs);
                sat_prep(&cs[0].x, &L->edge_sat[21 * u]);
                for (const V3& p : cs) {
                    box[0] = std::fmin(box[0], p.x), box[1] = std::fmin(box[1], p.y), box[2] = std::fmin(box[2], p.z);
                    box[3] = std::fmax(box[3], p.x), box[4] = std::fmax(box[4], p.y), box[5] = std::fmax(box[5], p.z);
                }
                double* o = &L->obb15[15 * u];
                const Box& ob = cp.over[bd];
                o[0] = ob.c.x, o[1] = ob.c.y, o[2] = ob.c.z;
                for (int q = 0; q < 3; ++q) o[3 + 3 * q] = ob.ax[q].x, o[4 + 3 * q] = ob.ax[q].y, o[5 + 3 * q] = ob.ax[q].z;
                o[12] = ob.he.x, o[13] = ob.he.y, o[14] = ob.he.z;
                std::vector<int32_t> used(rb.bodies[bd].spheres.size(), 0);
                for (const Spline& s : cp.under[bd]) {
                    const int32_t segc = std::max<int32_t>(1, static_cast<int32_t>(s.pts.size()) - 1);
                    if (segc > K) throw std::logic_error("spline exceeds the segment cap; the build policy should have split it");
                    const int32_t slot = s.sphere * max_parts + used[s.sphere]++;
                    if (L->spline_r[static_cast<size_t>(bd) * S + slot] != s.radius)
                        throw std::logic_error("inconsistent spline radius for a layout slot");
                    count[u * S + slot] = segc;
                }
            }
            std::memcpy(&L->comp_aabb[6 * static_cast<size_t>(c)], box, sizeof(box));
        });
        int64_t total = 0;
        for (size_t r = 0; r < count.size(); ++r) {
            L->row_off[r] = static_cast<int32_t>(total);
            total += count[r];
            if (total > INT32_MAX) throw std::invalid_argument("more than 2^31 - 1 real segments");
        }
        L->row_off[count.size()] = static_cast<int32_t>(total);
        L->segs.resize(static_cast<size_t>(total) * 7);
        parallel(N, [&](int32_t c) {
            for (int32_t bd = 0; bd < B; ++bd) {
                std::vector<int32_t> used(rb.bodies[bd].spheres.size(), 0);
                for (const Spline& s : comps[c].under[bd]) {
                    const int32_t slot = s.sphere * max_parts + used[s.sphere]++;
                    double* dst = &L->segs[7 * static_cast<size_t>(L->row_off[(static_cast<size_t>(c) * B + bd) * S + slot])];
                    if (s.pts.size() == 1) {
                        seg_prep(s.pts[0], s.pts[0], dst);
                    } else {
                        for (size_t p = 0; p + 1 < s.pts.size(); ++p) seg_prep(s.pts[p], s.pts[p + 1], dst + 7 * p);
                    }
                }
            }
        });
        if (keep_poses) {
            L->pose_off.assign(static_cast<size_t>(N) + 1, 0);
            for (int32_t c = 0; c < N; ++c)
                L->pose_off[c + 1] = L->pose_off[c] + static_cast<int64_t>(comps[c].fk.size() / B);
            L->poses.resize(static_cast<size_t>(L->pose_off[N]) * B * 12);
            parallel(N, [&](int32_t c) {
                for (size_t q = 0; q < comps[c].fk.size(); ++q) {
                    double* d = &L->poses[(static_cast<size_t>(L->pose_off[c]) * B + q) * 12];
                    const Tf& T = comps[c].fk[q];
                    std::memcpy(d, T.r, 9 * sizeof(double));
                    d[9] = T.t.x, d[10] = T.t.y, d[11] = T.t.z;
                }
            });
        }
        mark("serialize");
        if (flags & RGG_BUILD_KEEP_GEOMETRY) {
            L->kept = true;
            L->robot = rb;
            L->kinematics = robot->kinematics;
            L->dof = dof;
            L->K = K;
            L->eps = eps;
            L->rb_he.assign(robot->half_extents, robot->half_extents + 3 * static_cast<size_t>(B));
            if (robot->local) L->rb_local.assign(robot->local, robot->local + 12 * static_cast<size_t>(B));
            if (rb.chain) {
                L->rb_axis.assign(robot->joint_axis, robot->joint_axis + 3 * static_cast<size_t>(B));
                L->rb_offset.assign(robot->joint_offset, robot->joint_offset + 3 * static_cast<size_t>(B));
            }
            L->nodes.assign(nodes, nodes + static_cast<size_t>(n_nodes) * dof);
            L->edges.assign(edges, edges + 2 * static_cast<size_t>(n_edges));
            L->comps = std::move(comps);
        }
        *out = own.release();
        return 0;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return -1;
    }
}

// save_roadmap (roadmap_io.cpp:150-203) of a producer build kept with RGG_BUILD_KEEP_GEOMETRY:
// the same sections, so the reference's load_roadmap reads it (and a build bit-identical to
// the reference's gives the same file byte for byte)
int rgg_built_save_roadmap(const rgg_built* b, const char* path) {
    try {
        if (!b || !path) throw std::invalid_argument("null build or path");
        if (!b->kept) throw std::invalid_argument("layout was built without RGG_BUILD_KEEP_GEOMETRY");
        std::vector<uint8_t> w;
        const auto u8 = [&](uint8_t v) { w.push_back(v); };
        const auto u32 = [&](uint32_t v) {
            for (int i = 0; i < 4; ++i) w.push_back(static_cast<uint8_t>(v >> (8 * i)));
        };
        const auto f64 = [&](double d) {
            uint64_t v;
            std::memcpy(&v, &d, 8);
            for (int i = 0; i < 8; ++i) w.push_back(static_cast<uint8_t>(v >> (8 * i)));
        };
        const auto v3 = [&](V3 p) { f64(p.x), f64(p.y), f64(p.z); };
        static const char kMagic[8] = {'R', 'G', 'G', 'R', 'D', 'M', 'P', '1'};
        w.insert(w.end(), kMagic, kMagic + 8);
        u32(1);
        // robot: kinematics, bodies {half extents, local frame}, joints {axis, offset}
        const int32_t B = b->B;
        u8(static_cast<uint8_t>(b->kinematics));
        u32(static_cast<uint32_t>(B));
        for (int32_t bd = 0; bd < B; ++bd) {
            v3(b->robot.bodies[bd].he);
            const Tf& l = b->robot.bodies[bd].local;
            for (double r : l.r) f64(r);
            v3(l.t);
        }
        u32(static_cast<uint32_t>(b->robot.axis.size()));
        for (size_t j = 0; j < b->robot.axis.size(); ++j) v3(b->robot.axis[j]), v3(b->robot.offset[j]);
        // the sphere sets (default_body_spheres), the resolution and the segment cap
        u32(static_cast<uint32_t>(B));
        for (int32_t bd = 0; bd < B; ++bd) {
            const auto& sp = b->robot.bodies[bd].spheres;
            u32(static_cast<uint32_t>(sp.size()));
            for (const Sph& s : sp) v3(s.c), f64(s.r);
        }
        f64(b->eps);
        u32(static_cast<uint32_t>(b->K));
        // the roadmap
        const uint32_t n_nodes = static_cast<uint32_t>(b->nodes.size() / std::max(1, b->dof));
        u32(n_nodes);
        u32(static_cast<uint32_t>(b->dof));
        for (double v : b->nodes) f64(v);
        u32(static_cast<uint32_t>(b->edges.size() / 2));
        for (int32_t v : b->edges) u32(static_cast<uint32_t>(v));
        // per component: the body OBBs, then per body its splines
        u32(static_cast<uint32_t>(b->comps.size()));
        for (const Comp& c : b->comps) {
            u32(static_cast<uint32_t>(c.over.size()));
            for (const Box& o : c.over) {
                v3(o.c);
                for (int q = 0; q < 3; ++q) v3(o.ax[q]);
                v3(o.he);
            }
            for (const auto& body : c.under) {
                u32(static_cast<uint32_t>(body.size()));
                for (const Spline& s : body) {
                    f64(s.radius);
                    u32(static_cast<uint32_t>(s.sphere));
                    u32(static_cast<uint32_t>(s.pts.size()));
                    for (const V3& q : s.pts) v3(q);
                }
            }
        }
        u32(crc32_of(w.data(), w.size()));
        std::FILE* f = std::fopen(path, "wb");
        if (!f) throw std::runtime_error(std::string("cannot open ") + path + " for writing");
        const bool ok = std::fwrite(w.data(), 1, w.size(), f) == w.size();
        if (std::fclose(f) != 0 || !ok) throw std::runtime_error(std::string("short write to ") + path);
        return 0;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return -1;
    }
}

int rgg_built_counts(const rgg_built* b, int64_t* out) {
    if (!b || !out) return -1;
    out[0] = b->N;
    out[1] = b->B;
    out[2] = b->S;
    out[3] = static_cast<int64_t>(b->segs.size() / 7);
    return 0;
}

int rgg_built_export(const rgg_built* b, double* edge_sat, double* comp_aabb, int32_t* row_off, double* segs,
                     double* spline_r, double* obb15) {
    if (!b) return -1;
    auto cp = [](void* dst, const auto& v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(edge_sat, b->edge_sat);
    cp(comp_aabb, b->comp_aabb);
    cp(row_off, b->row_off);
    cp(segs, b->segs);
    cp(spline_r, b->spline_r);
    cp(obb15, b->obb15);
    return 0;
}

int rgg_built_poses(const rgg_built* b, int64_t* n_configs, int64_t* pose_off, double* poses) {
    if (!b) return -1;
    if (b->pose_off.empty()) {
        g_err = "layout was built without RGG_BUILD_POSES";
        return -1;
    }
    if (n_configs) *n_configs = b->pose_off.back();
    if (pose_off) std::memcpy(pose_off, b->pose_off.data(), b->pose_off.size() * sizeof(int64_t));
    if (poses && !b->poses.empty()) std::memcpy(poses, b->poses.data(), b->poses.size() * sizeof(double));
    return 0;
}

void rgg_built_free(rgg_built* b) { delete b; }

struct rgg_roadmap_file {
    int32_t kinematics = 0, B = 0, S = 1, dof = 0, n_nodes = 0, n_edges = 0, K = 16;
    double eps = 0.0;
    std::vector<double> he, local, axis, offset;  // the robot
    std::vector<double> nodes;
    std::vector<int32_t> edges;
    std::vector<double> corners, seg_pts, spline_r;  // the component view
    std::vector<int32_t> row_off;
};

int rgg_roadmap_load(const char* path, rgg_roadmap_file** out) {
    try {
        if (!path || !out) throw FileError(RGG_ROADMAP_TRUNCATED, "null path or output");
        std::vector<uint8_t> buf;
        {
            std::FILE* f = std::fopen(path, "rb");
            if (!f) throw FileError(RGG_ROADMAP_TRUNCATED, std::string("cannot open ") + path);
            uint8_t chunk[1 << 16];
            for (size_t got; (got = std::fread(chunk, 1, sizeof(chunk), f)) > 0;) buf.insert(buf.end(), chunk, chunk + got);
            std::fclose(f);
        }
        static const char kMagic[8] = {'R', 'G', 'G', 'R', 'D', 'M', 'P', '1'};
        if (buf.size() < sizeof(kMagic) + 8) throw FileError(RGG_ROADMAP_TRUNCATED, "file too small");
        if (std::memcmp(buf.data(), kMagic, sizeof(kMagic)) != 0) throw FileError(RGG_ROADMAP_BAD_MAGIC, "not a roadmap file");
        const size_t body = buf.size() - 4;
        const uint32_t stored = static_cast<uint32_t>(buf[body]) | static_cast<uint32_t>(buf[body + 1]) << 8 |
                                static_cast<uint32_t>(buf[body + 2]) << 16 | static_cast<uint32_t>(buf[body + 3]) << 24;
        if (crc32_of(buf.data(), body) != stored) throw FileError(RGG_ROADMAP_CHECKSUM, "checksum mismatch");
        ByteReader rd{buf.data(), body, sizeof(kMagic)};
        if (rd.u32() != 1) throw FileError(RGG_ROADMAP_BAD_VERSION, "unsupported roadmap file version");
        std::unique_ptr<rgg_roadmap_file> F(new rgg_roadmap_file());
        // robot (write_robot, roadmap_io.cpp:95-107)
        F->kinematics = rd.u8();
        F->B = static_cast<int32_t>(rd.count(1u << 16, "bodies"));
        for (int32_t b = 0; b < F->B; ++b) {
            const V3 he = rd.v3();
            F->he.insert(F->he.end(), {he.x, he.y, he.z});
            for (int q = 0; q < 12; ++q) F->local.push_back(rd.f64());
        }
        const uint32_t nj = rd.count(1u << 16, "joints");
        for (uint32_t j = 0; j < nj; ++j) {
            const V3 ax = rd.v3(), of = rd.v3();
            F->axis.insert(F->axis.end(), {ax.x, ax.y, ax.z});
            F->offset.insert(F->offset.end(), {of.x, of.y, of.z});
        }
        // sphere sets: only their counts shape the slot layout (batch_layout.cpp:28-43)
        const uint32_t nsb = rd.count(1u << 16, "sphere bodies");
        int32_t max_spheres = 1;
        std::vector<int32_t> nsph(nsb);
        for (uint32_t b = 0; b < nsb; ++b) {
            nsph[b] = static_cast<int32_t>(rd.count(1u << 20, "spheres"));
            max_spheres = std::max(max_spheres, nsph[b]);
            for (int32_t s = 0; s < nsph[b]; ++s) rd.v3(), rd.f64();
        }
        F->eps = rd.f64();
        F->K = static_cast<int32_t>(rd.u32());
        F->n_nodes = static_cast<int32_t>(rd.count(1u << 24, "nodes"));
        F->dof = static_cast<int32_t>(rd.count(1u << 10, "dof"));
        F->nodes.resize(static_cast<size_t>(F->n_nodes) * F->dof);
        for (double& v : F->nodes) v = rd.f64();
        F->n_edges = static_cast<int32_t>(rd.count(1u << 26, "edges"));
        F->edges.resize(2 * static_cast<size_t>(F->n_edges));
        for (int32_t& v : F->edges) {
            const uint32_t e = rd.u32();
            if (e >= static_cast<uint32_t>(F->n_nodes)) throw std::invalid_argument("edge endpoint out of range");
            v = static_cast<int32_t>(e);
        }
        const uint32_t ng = rd.count(1u << 26, "geometry");
        if (ng != static_cast<uint32_t>(F->n_nodes) + static_cast<uint32_t>(F->n_edges))
            throw FileError(RGG_ROADMAP_TRUNCATED, "geometry count mismatch");
        const int32_t N = static_cast<int32_t>(ng), B = F->B;
        if (static_cast<int32_t>(nsb) != B) throw std::invalid_argument("sphere set / body count mismatch");
        // per component: body OBBs, then per body its splines {radius, sphere index, points}
        struct Spl {
            double r;
            int32_t sphere;
            uint32_t first, npts;  // into pts
        };
        std::vector<Box> boxes(static_cast<size_t>(N) * B);
        std::vector<std::vector<Spl>> spl(static_cast<size_t>(N) * B);
        std::vector<V3> pts;
        for (int32_t c = 0; c < N; ++c) {
            const uint32_t nover = rd.count(1u << 16, "over boxes");
            if (static_cast<int32_t>(nover) != B) throw std::invalid_argument("component body count mismatch");
            for (int32_t b = 0; b < B; ++b) {
                Box& o = boxes[static_cast<size_t>(c) * B + b];
                o.c = rd.v3();
                for (int q = 0; q < 3; ++q) o.ax[q] = rd.v3();
                o.he = rd.v3();
            }
            for (int32_t b = 0; b < B; ++b) {
                const uint32_t ns = rd.count(1u << 20, "splines");
                for (uint32_t s = 0; s < ns; ++s) {
                    Spl sp;
                    sp.r = rd.f64();
                    sp.sphere = static_cast<int32_t>(rd.u32());
                    sp.npts = rd.count(1u << 24, "spline points");
                    sp.first = static_cast<uint32_t>(pts.size());
                    for (uint32_t q = 0; q < sp.npts; ++q) pts.push_back(rd.v3());
                    if (sp.sphere < 0 || sp.sphere >= nsph[b]) throw std::invalid_argument("spline sphere index out of range");
                    spl[static_cast<size_t>(c) * B + b].push_back(sp);
                }
            }
        }
        // the component view (rgg_component_view, include/rgg_gpu.h): OBB corners in
        // obb_corners order, real segments per (component, body, slot) row with the slot
        // layout of BatchLayout::serialize (batch_layout.cpp:28-105)
        int32_t max_parts = 1;
        for (int32_t u = 0; u < N * B; ++u) {
            std::vector<int32_t> parts(nsph[u % B], 0);
            for (const Spl& sp : spl[u]) max_parts = std::max(max_parts, ++parts[sp.sphere]);
        }
        const int32_t S = max_spheres * max_parts;
        F->S = S;
        F->spline_r.assign(static_cast<size_t>(B) * S, 0.0);
        F->corners.resize(static_cast<size_t>(N) * B * 24);
        std::vector<int32_t> count(static_cast<size_t>(N) * B * S, 0);
        std::vector<std::vector<std::pair<int32_t, const Spl*>>> rows(static_cast<size_t>(N) * B);
        for (int32_t u = 0; u < N * B; ++u) {
            V3 cs[8];
            corners_of(boxes[u], cs);
            for (int i = 0; i < 8; ++i)
                F->corners[24 * static_cast<size_t>(u) + 3 * i] = cs[i].x, F->corners[24 * static_cast<size_t>(u) + 3 * i + 1] = cs[i].y,
                                                      F->corners[24 * static_cast<size_t>(u) + 3 * i + 2] = cs[i].z;
            const int32_t b = u % B;
            std::vector<int32_t> used(nsph[b], 0);
            for (const Spl& sp : spl[u]) {
                const int32_t segc = std::max<int32_t>(1, static_cast<int32_t>(sp.npts) - 1);
                if (segc > F->K) throw std::logic_error("spline exceeds the segment cap; the build policy should have split it");
                const int32_t slot = sp.sphere * max_parts + used[sp.sphere]++;
                double& rad = F->spline_r[static_cast<size_t>(b) * S + slot];
                if (rad == 0.0) rad = sp.r;
                else if (rad != sp.r) throw std::logic_error("inconsistent spline radius for a layout slot");
                count[static_cast<size_t>(u) * S + slot] = segc;
                rows[u].push_back({slot, &sp});
            }
        }
        F->row_off.assign(count.size() + 1, 0);
        int64_t total = 0;
        for (size_t r = 0; r < count.size(); ++r) {
            F->row_off[r] = static_cast<int32_t>(total);
            total += count[r];
            if (total > INT32_MAX) throw std::invalid_argument("more than 2^31 - 1 real segments");
        }
        F->row_off[count.size()] = static_cast<int32_t>(total);
        F->seg_pts.resize(static_cast<size_t>(total) * 6);
        for (int32_t u = 0; u < N * B; ++u)
            for (const auto& [slot, sp] : rows[u]) {
                double* d = &F->seg_pts[6 * static_cast<size_t>(F->row_off[static_cast<size_t>(u) * S + slot])];
                const V3* q = &pts[sp->first];
                if (sp->npts == 1) {  // a single-point spline is a degenerate segment (batch_layout.cpp:84-90)
                    const double s6[6] = {q[0].x, q[0].y, q[0].z, q[0].x, q[0].y, q[0].z};
                    std::memcpy(d, s6, sizeof(s6));
                } else {
                    for (uint32_t k = 0; k + 1 < sp->npts; ++k, d += 6) {
                        const double s6[6] = {q[k].x, q[k].y, q[k].z, q[k + 1].x, q[k + 1].y, q[k + 1].z};
                        std::memcpy(d, s6, sizeof(s6));
                    }
                }
            }
        *out = F.release();
        return 0;
    } catch (const FileError& ex) {
        g_err = ex.what();
        return ex.kind;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return -1;
    }
}

int rgg_roadmap_counts(const rgg_roadmap_file* f, int64_t* out) {
    if (!f || !out) return -1;
    out[0] = f->n_nodes;
    out[1] = f->n_edges;
    out[2] = f->dof;
    out[3] = static_cast<int64_t>(f->n_nodes) + f->n_edges;
    out[4] = f->B;
    out[5] = f->S;
    out[6] = static_cast<int64_t>(f->seg_pts.size() / 6);
    out[7] = f->kinematics;
    out[8] = f->K;
    return 0;
}

int rgg_roadmap_components(const rgg_roadmap_file* f, double* obb_corners, int32_t* row_off, double* seg_points,
                           double* spline_radius) {
    if (!f) return -1;
    auto cp = [](void* dst, const auto& v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(obb_corners, f->corners);
    cp(row_off, f->row_off);
    cp(seg_points, f->seg_pts);
    cp(spline_radius, f->spline_r);
    return 0;
}

int rgg_roadmap_graph(const rgg_roadmap_file* f, double* nodes, int32_t* edges, double* eps) {
    if (!f) return -1;
    if (nodes && !f->nodes.empty()) std::memcpy(nodes, f->nodes.data(), f->nodes.size() * sizeof(double));
    if (edges && !f->edges.empty()) std::memcpy(edges, f->edges.data(), f->edges.size() * sizeof(int32_t));
    if (eps) *eps = f->eps;
    return 0;
}

int rgg_roadmap_robot(const rgg_roadmap_file* f, double* he, double* local12, double* axis, double* offset) {
    if (!f) return -1;
    auto cp = [](double* dst, const std::vector<double>& v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
    };
    cp(he, f->he);
    cp(local12, f->local);
    cp(axis, f->axis);
    cp(offset, f->offset);
    return 0;
}

int rgg_roadmap_poses(const rgg_roadmap_file* f, int64_t* n_configs, int64_t* pose_off, double* poses) {
    // the exact resolve's inputs: forward_kinematics (robot.cpp:66-84) of every configuration
    // of discretize_edge (robot.cpp:39-64), which load_roadmap rebuilds (roadmap_io.cpp:294-298)
    try {
        if (!f) throw std::invalid_argument("null roadmap file");
        rgg_robot_view v{};
        v.kinematics = f->kinematics;
        v.n_bodies = f->B;
        v.half_extents = f->he.data();
        v.local = f->local.data();
        v.joint_axis = f->axis.empty() ? nullptr : f->axis.data();
        v.joint_offset = f->offset.empty() ? nullptr : f->offset.data();
        const Robot rb = make_robot(v, f->eps);
        if (rb.dof != f->dof) throw std::invalid_argument("configuration DOF mismatch");
        const int32_t N = f->n_nodes + f->n_edges, B = f->B, dof = f->dof;
        const auto ends = [&](int32_t c, const double** a, const double** b) {
            if (c < f->n_nodes) {
                *a = *b = f->nodes.data() + static_cast<size_t>(dof) * c;
            } else {
                *a = f->nodes.data() + static_cast<size_t>(dof) * f->edges[2 * (c - f->n_nodes)];
                *b = f->nodes.data() + static_cast<size_t>(dof) * f->edges[2 * (c - f->n_nodes) + 1];
            }
        };
        int64_t total = 0;
        for (int32_t c = 0; c < N; ++c) {
            const double *a, *b;
            ends(c, &a, &b);
            if (pose_off) pose_off[c] = total;
            total += config_count(a, b, dof, f->eps);
        }
        if (pose_off) pose_off[N] = total;
        if (n_configs) *n_configs = total;
        if (!poses) return 0;
        std::vector<Tf> fk(B);
        double cfg[64];
        int64_t q = 0;
        for (int32_t c = 0; c < N; ++c) {
            const double *a, *b;
            ends(c, &a, &b);
            const int n = config_count(a, b, dof, f->eps);
            for (int i = 0; i < n; ++i, ++q) {
                if (i == 0) {
                    std::memcpy(cfg, a, dof * sizeof(double));
                } else if (i == n - 1) {
                    std::memcpy(cfg, b, dof * sizeof(double));
                } else {
                    const double t = static_cast<double>(i) / static_cast<double>(n - 1);
                    for (int k = 0; k < dof; ++k) cfg[k] = a[k] + (b[k] - a[k]) * t;
                }
                forward_kinematics(rb, cfg, fk.data());
                for (int32_t bd = 0; bd < B; ++bd) {
                    double* d = poses + 12 * (static_cast<size_t>(q) * B + bd);
                    std::memcpy(d, fk[bd].r, 9 * sizeof(double));
                    d[9] = fk[bd].t.x, d[10] = fk[bd].t.y, d[11] = fk[bd].t.z;
                }
            }
        }
        return 0;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return -1;
    }
}

void rgg_roadmap_free(rgg_roadmap_file* f) { delete f; }

int rgg_obstacle_spheres(const double* he3, int32_t count, double* centres, double* radius) {
    if (count < 1 || !(he3[0] > 0 && he3[1] > 0 && he3[2] > 0)) {
        g_err = "bad obstacle sphere request";
        return -1;
    }
    const std::vector<Sph> s = inner_spheres({he3[0], he3[1], he3[2]}, count);
    for (int32_t i = 0; i < count; ++i) {
        centres[3 * i] = s[i].c.x;
        centres[3 * i + 1] = s[i].c.y;
        centres[3 * i + 2] = s[i].c.z;
    }
    *radius = s[0].r;
    return 0;
}

}  // extern "C"
