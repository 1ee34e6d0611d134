// ref_shim.cpp — C-ABI over the UNMODIFIED reference library (test infrastructure).
//
// ORACLE / TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with
// the reference sources under /root/reference/proj/src into oracle/_ref/librgg_ref.so.
// Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
// legs load it.  Nothing in paper_2603_28674_b200/ links or calls it.
//
// It exposes exactly what the parity suite needs from the reference:
//   * roadmap construction through the reference's own producers
//     (build_prm / build_components, proj/src/roadmap.cpp:56-127) from a .scn
//     text (proj/src/scenario.cpp:86-229) or from explicit nodes/edges;
//   * the serialized layout (BatchLayout::serialize, proj/src/batch_layout.cpp:21-138)
//     flattened to the CSR view our C-ABI consumes;
//   * the reference engines (BatchEngine proj/src/engine_batch.cpp:145-215,
//     SequentialEngine proj/src/engine_sequential.cpp:169-227), including the
//     grouped-engine construction for M > 64 obstacles;
//   * the kernel known-answer generators of proj/tests/test_kernels.cpp:46-121.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "oracles.hpp"
#include "rgg/batch_layout.hpp"
#include "rgg/engine_batch.hpp"
#include "rgg/engine_sequential.hpp"
#include "rgg/kernels.hpp"
#include "rgg/rng.hpp"
#include "rgg/roadmap_io.hpp"
#include "rgg/scenario.hpp"

using namespace rgg;

namespace {

thread_local std::string g_err;

struct World {
    Scene scene;  // canonical obstacles (inactive, identity pose)
    Roadmap roadmap;
    ComponentSet comps;
    std::vector<std::pair<ObstacleId, Transform>> moves;  // scenario script, if any
    int iterations = 0;
    bool lazy = true;
};

struct Group {
    Scene scene;
    std::unique_ptr<BatchEngine> bat;
    std::unique_ptr<SequentialEngine> seq;
};

struct Engine {
    const World* world = nullptr;
    int group_size = 64;
    std::vector<std::unique_ptr<Group>> groups;  // obstacle o lives in group o / group_size
    std::vector<std::uint8_t> states;
    std::vector<std::uint64_t> bits;
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = std::string("invalid_argument: ") + e.what();
        return -1;
    } catch (const std::logic_error& e) {
        g_err = std::string("logic_error: ") + e.what();
        return -2;
    } catch (const std::exception& e) {
        g_err = std::string("exception: ") + e.what();
        return -3;
    }
}

void finish_world(World& w) {
    for (ObstacleModel& o : w.scene.obstacles) {
        o.pose = Transform::identity();
        o.active = false;
    }
}

Transform tf_of(const double* rt12) {
    Transform t;
    for (int i = 0; i < 9; ++i) t.r[i] = rt12[i];
    t.t = {rt12[9], rt12[10], rt12[11]};
    return t;
}

void put_tf(const Transform& t, double* rt12) {
    for (int i = 0; i < 9; ++i) rt12[i] = t.r[i];
    rt12[9] = t.t.x;
    rt12[10] = t.t.y;
    rt12[11] = t.t.z;
}

void put_sat(const kern::SatBox& s, double* out21) {
    for (int j = 0; j < 3; ++j) out21[j] = s.center[j];
    for (int k = 0; k < 3; ++k)
        for (int j = 0; j < 3; ++j) out21[3 + k * 3 + j] = s.e[k][j];
    for (int k = 0; k < 3; ++k)
        for (int j = 0; j < 3; ++j) out21[12 + k * 3 + j] = s.u[k][j];
}

}  // namespace

extern "C" {

const char* rr_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- worlds

void* rr_world_from_scn(const char* text) {
    World* w = new World();
    const int rc = guarded([&] {
        const Scenario s = parse_scenario_text(text, "<scn>");
        w->scene = Scene{s.env, s.make_obstacles(), s.robot};
        Scene build_scene{s.env, {}, s.robot};
        w->roadmap = build_prm(build_scene, s.nodes, s.k_neighbors, s.effective_epsilon(), s.roadmap_seed);
        w->comps = build_components(w->roadmap, s.robot, default_body_spheres(s.robot), s.effective_epsilon(),
                                    s.max_segments);
        w->moves = s.make_moves();
        w->iterations = s.iterations;
        w->lazy = s.mode == UpdateMode::Lazy;
        finish_world(*w);
    });
    if (rc != 0) {
        delete w;
        return nullptr;
    }
    return w;
}

// Free-flying box robot over an explicit roadmap (nodes n x 6, edges e x 2).
// Obstacles are added with rr_world_add_obstacle.
void* rr_world_from_roadmap(const double* robot_he3, const double* env6, int n_nodes, const double* nodes,
                            int n_edges, const std::int32_t* edges, double eps, int max_segments) {
    World* w = new World();
    const int rc = guarded([&] {
        w->scene.bounds = {{env6[0], env6[1], env6[2]}, {env6[3], env6[4], env6[5]}};
        w->scene.robot = make_free_flying_box({robot_he3[0], robot_he3[1], robot_he3[2]});
        w->roadmap.nodes.resize(n_nodes);
        for (int i = 0; i < n_nodes; ++i) w->roadmap.nodes[i].assign(nodes + i * 6, nodes + i * 6 + 6);
        w->roadmap.edges.resize(n_edges);
        for (int e = 0; e < n_edges; ++e) w->roadmap.edges[e] = {edges[2 * e], edges[2 * e + 1]};
        w->roadmap.rebuild_adjacency();
        w->comps = build_components(w->roadmap, w->scene.robot, default_body_spheres(w->scene.robot), eps,
                                    max_segments);
    });
    if (rc != 0) {
        delete w;
        return nullptr;
    }
    return w;
}

// Any robot (free-flying or serial chain, robot.hpp:13-58) over an explicit roadmap
// (nodes n x dof, edges e x 2): kin 0 free flying / 1 serial chain; per body its half
// extents (3) and local frame (12: r[9], t[3]); per joint (chains) axis (3), offset (3).
void* rr_world_from_robot(int kin, int n_bodies, const double* he, const double* local12, const double* axis,
                          const double* offset, const double* env6, int n_nodes, const double* nodes, int n_edges,
                          const std::int32_t* edges, double eps, int max_segments) {
    World* w = new World();
    const int rc = guarded([&] {
        w->scene.bounds = {{env6[0], env6[1], env6[2]}, {env6[3], env6[4], env6[5]}};
        RobotModel m;
        m.kinematics = kin == 1 ? KinematicsType::SerialChain : KinematicsType::FreeFlying;
        for (int b = 0; b < n_bodies; ++b) {
            m.bodies.push_back({{he[3 * b], he[3 * b + 1], he[3 * b + 2]}, tf_of(local12 + 12 * b)});
            if (kin == 1) {
                Joint j;
                j.axis = {axis[3 * b], axis[3 * b + 1], axis[3 * b + 2]};
                j.offset = {offset[3 * b], offset[3 * b + 1], offset[3 * b + 2]};
                m.joints.push_back(j);
            }
        }
        m.validate();
        w->scene.robot = m;
        const int dof = m.dof_count();
        w->roadmap.nodes.resize(n_nodes);
        for (int i = 0; i < n_nodes; ++i) w->roadmap.nodes[i].assign(nodes + i * dof, nodes + (i + 1) * dof);
        w->roadmap.edges.resize(n_edges);
        for (int e = 0; e < n_edges; ++e) w->roadmap.edges[e] = {edges[2 * e], edges[2 * e + 1]};
        w->roadmap.rebuild_adjacency();
        w->comps = build_components(w->roadmap, m, default_body_spheres(m), eps, max_segments);
    });
    if (rc != 0) {
        delete w;
        return nullptr;
    }
    return w;
}

// The world's robot: meta = {kinematics (0 free flying, 1 serial chain), bodies, dof};
// he B*3, local B*12, axis / offset B*3 (zero for free flying); eps_k = {epsilon,
// max_segments} of its components.  Null arrays are skipped.
int rr_world_robot(void* wp, std::int32_t* meta, double* he, double* local12, double* axis, double* offset,
                   double* eps_k) {
    const World* w = static_cast<const World*>(wp);
    return guarded([&] {
        const RobotModel& m = w->scene.robot;
        const int B = static_cast<int>(m.bodies.size());
        meta[0] = m.kinematics == KinematicsType::SerialChain ? 1 : 0;
        meta[1] = B;
        meta[2] = m.dof_count();
        for (int b = 0; b < B; ++b) {
            const Vec3& v = m.bodies[b].half_extents;
            if (he) he[3 * b] = v.x, he[3 * b + 1] = v.y, he[3 * b + 2] = v.z;
            if (local12) put_tf(m.bodies[b].local, local12 + 12 * b);
            const bool j = b < static_cast<int>(m.joints.size());
            if (axis) {
                axis[3 * b] = j ? m.joints[b].axis.x : 0.0;
                axis[3 * b + 1] = j ? m.joints[b].axis.y : 0.0;
                axis[3 * b + 2] = j ? m.joints[b].axis.z : 0.0;
            }
            if (offset) {
                offset[3 * b] = j ? m.joints[b].offset.x : 0.0;
                offset[3 * b + 1] = j ? m.joints[b].offset.y : 0.0;
                offset[3 * b + 2] = j ? m.joints[b].offset.z : 0.0;
            }
        }
        if (eps_k) eps_k[0] = w->comps.epsilon, eps_k[1] = w->comps.max_segments;
    });
}

// save_roadmap (roadmap_io.cpp:150-203) of the world's robot, roadmap and components.
int rr_world_save(void* wp, const char* path) {
    const World* w = static_cast<const World*>(wp);
    return guarded([&] { save_roadmap(path, w->scene.robot, w->roadmap, w->comps); });
}

// The world's roadmap: nodes n x dof, edges e x 2 (counts from rr_world_counts).
int rr_world_roadmap(void* wp, double* nodes, std::int32_t* edges) {
    const World* w = static_cast<const World*>(wp);
    return guarded([&] {
        size_t k = 0;
        for (const Configuration& c : w->roadmap.nodes)
            for (double v : c) nodes[k++] = v;
        for (size_t e = 0; e < w->roadmap.edges.size(); ++e) {
            edges[2 * e] = w->roadmap.edges[e].first;
            edges[2 * e + 1] = w->roadmap.edges[e].second;
        }
    });
}

int rr_world_add_obstacle(void* wp, const double* he3, int spheres) {
    World* w = static_cast<World*>(wp);
    return guarded([&] {
        const Vec3 he{he3[0], he3[1], he3[2]};
        w->scene.obstacles.push_back(make_box_obstacle(he, spheres > 0 ? spheres : default_sphere_count(he)));
    });
}

void rr_world_free(void* wp) { delete static_cast<World*>(wp); }

// out: n_nodes, n_edges, N, B, S, K, M, C, total_real_segments, n_moves, iterations, lazy
int rr_world_counts(void* wp, std::int64_t* out) {
    const World* w = static_cast<const World*>(wp);
    return guarded([&] {
        const BatchLayout l = BatchLayout::serialize(w->comps, w->scene.obstacles);
        std::int64_t segs = 0;
        for (std::int32_t c : l.seg_count) segs += c;
        out[0] = w->comps.n_nodes;
        out[1] = w->comps.n_edges;
        out[2] = l.n_components;
        out[3] = l.n_bodies;
        out[4] = l.n_slots;
        out[5] = l.max_segments;
        out[6] = l.n_obstacles;
        out[7] = l.n_spheres;
        out[8] = segs;
        out[9] = static_cast<std::int64_t>(w->moves.size());
        out[10] = w->iterations;
        out[11] = w->lazy ? 1 : 0;
    });
}

int rr_world_moves(void* wp, std::int32_t* ids, double* rt12) {
    const World* w = static_cast<const World*>(wp);
    return guarded([&] {
        for (size_t i = 0; i < w->moves.size(); ++i) {
            ids[i] = w->moves[i].first;
            put_tf(w->moves[i].second, rt12 + i * 12);
        }
    });
}

// Layout view: the reference's serialized arrays (batch_layout.cpp:21-138)
// flattened to CSR over real segments.  Any output pointer may be null.
//   edge_sat     N*B*21   SatBox rows (center, e[3][3], u[3][3])
//   e_plus       N*B*24   corner rows
//   comp_aabb    N*6      component_aabb (min xyz, max xyz)
//   row_off      N*B*S+1  CSR offsets of real segments per (c, b, slot) row
//   segs         total*7  SegPrep rows (a, d, dd) of real segments
//   seg_pts      total*6  raw segment endpoints (e_minus) of real segments
//   spline_r     B*S      slot radii
//   obst_he      M*3, obst_sph_local M*C*3, obst_sph_r M, obst_sph_n M
int rr_world_layout(void* wp, double* edge_sat, double* e_plus, double* comp_aabb, std::int32_t* row_off,
                    double* segs, double* seg_pts, double* spline_r, double* obst_he, double* obst_sph_local,
                    double* obst_sph_r, std::int32_t* obst_sph_n) {
    const World* w = static_cast<const World*>(wp);
    return guarded([&] {
        const BatchLayout l = BatchLayout::serialize(w->comps, w->scene.obstacles);
        const size_t nb = static_cast<size_t>(l.n_components) * l.n_bodies;
        for (size_t i = 0; i < nb; ++i) {
            if (edge_sat) put_sat(l.edge_sat[i], edge_sat + i * 21);
            if (e_plus) std::memcpy(e_plus + i * 24, &l.e_plus[i * 24], 24 * sizeof(double));
        }
        if (comp_aabb) {
            for (int c = 0; c < l.n_components; ++c) {
                const Aabb& a = l.component_aabb[c];
                const double v[6] = {a.min.x, a.min.y, a.min.z, a.max.x, a.max.y, a.max.z};
                std::memcpy(comp_aabb + c * 6, v, sizeof(v));
            }
        }
        std::int64_t at = 0;
        for (size_t row = 0; row < l.seg_count.size(); ++row) {
            if (row_off) row_off[row] = static_cast<std::int32_t>(at);
            for (std::int32_t k = 0; k < l.seg_count[row]; ++k, ++at) {
                const kern::SegPrep& s = l.seg_prep[row * l.max_segments + k];
                if (segs) {
                    double* d = segs + at * 7;
                    for (int j = 0; j < 3; ++j) d[j] = s.a[j];
                    for (int j = 0; j < 3; ++j) d[3 + j] = s.d[j];
                    d[6] = s.dd;
                }
                if (seg_pts) std::memcpy(seg_pts + at * 6, &l.e_minus[(row * l.max_segments + k) * 6], 48);
            }
        }
        if (row_off) row_off[l.seg_count.size()] = static_cast<std::int32_t>(at);
        if (spline_r) std::memcpy(spline_r, l.spline_radius.data(), l.spline_radius.size() * sizeof(double));
        for (int o = 0; o < l.n_obstacles; ++o) {
            const ObstacleModel& m = w->scene.obstacles[o];
            if (obst_he) {
                obst_he[o * 3 + 0] = m.half_extents.x;
                obst_he[o * 3 + 1] = m.half_extents.y;
                obst_he[o * 3 + 2] = m.half_extents.z;
            }
            for (int s = 0; s < l.n_spheres; ++s) {
                const bool real = s < static_cast<int>(m.inner.size());
                if (obst_sph_local) {
                    double* d = obst_sph_local + (static_cast<size_t>(o) * l.n_spheres + s) * 3;
                    d[0] = real ? m.inner[s].center.x : 0.0;
                    d[1] = real ? m.inner[s].center.y : 0.0;
                    d[2] = real ? m.inner[s].center.z : 0.0;
                }
            }
            if (obst_sph_r) obst_sph_r[o] = l.o_minus_r[o];
            if (obst_sph_n) obst_sph_n[o] = l.o_sphere_count[o];
        }
    });
}

// Fitted body OBBs per component (center 3, axes 9 row-per-axis, half extents 3).
int rr_world_obbs(void* wp, double* out15) {
    const World* w = static_cast<const World*>(wp);
    return guarded([&] {
        size_t i = 0;
        for (const EdgeGeometry& g : w->comps.geometry) {
            for (const Obb& o : g.over) {
                double* d = out15 + 15 * i++;
                d[0] = o.center.x;
                d[1] = o.center.y;
                d[2] = o.center.z;
                for (int k = 0; k < 3; ++k) {
                    d[3 + 3 * k] = o.axes[k].x;
                    d[4 + 3 * k] = o.axes[k].y;
                    d[5 + 3 * k] = o.axes[k].z;
                }
                d[12] = o.half_extents.x;
                d[13] = o.half_extents.y;
                d[14] = o.half_extents.z;
            }
        }
    });
}

// Obstacle operands after update_transforms (batch_layout.cpp:148-172) for
// one pose: SatBox 21, box aabb 6, sphere centres C*3, sphere aabb 6.
int rr_obstacle_operands(void* wp, int o, const double* rt12, double* sat21, double* aabb6, double* centres,
                         double* saabb6) {
    const World* w = static_cast<const World*>(wp);
    return guarded([&] {
        BatchLayout l = BatchLayout::serialize(w->comps, w->scene.obstacles);
        l.update_transforms({{o, tf_of(rt12)}}, w->scene.obstacles);
        put_sat(l.obstacle_sat[o], sat21);
        const Aabb& a = l.obstacle_aabb[o];
        const double v[6] = {a.min.x, a.min.y, a.min.z, a.max.x, a.max.y, a.max.z};
        std::memcpy(aabb6, v, sizeof(v));
        std::memcpy(centres, &l.o_minus_c[static_cast<size_t>(o) * l.n_spheres * 3], l.n_spheres * 3 * sizeof(double));
        const Aabb& s = l.obstacle_sphere_aabb[o];
        const double u[6] = {s.min.x, s.min.y, s.min.z, s.max.x, s.max.y, s.max.z};
        std::memcpy(saabb6, u, sizeof(u));
    });
}

// ---------------------------------------------------------------- engines

// kind 0 = BatchEngine, 1 = SequentialEngine.  Obstacles are split into
// groups of group_size (<= 64) independent engines; max_groups >= 0
// builds only the first max_groups of them (bounded CPU-baseline samples: moves of
// obstacles beyond them are rejected).
void* rr_engine_new_groups(void* wp, int kind, int threads, int use_under, int cell_capacity, int group_size,
                           int max_groups) {
    const World* w = static_cast<const World*>(wp);
    Engine* e = new Engine();
    const int rc = guarded([&] {
        if (group_size < 1 || group_size > 64) throw std::invalid_argument("group size must be in [1, 64]");
        e->world = w;
        e->group_size = group_size;
        EngineOptions opts;
        opts.threads = threads;
        opts.use_under = use_under != 0;
        const int m = static_cast<int>(w->scene.obstacles.size());
        int ng = m == 0 ? 1 : (m + group_size - 1) / group_size;
        if (max_groups >= 0 && max_groups < ng) ng = std::max(1, max_groups);
        for (int g = 0; g < ng; ++g) {
            auto grp = std::make_unique<Group>();
            grp->scene.bounds = w->scene.bounds;
            grp->scene.robot = w->scene.robot;
            for (int o = g * group_size; o < std::min(m, (g + 1) * group_size); ++o)
                grp->scene.obstacles.push_back(w->scene.obstacles[o]);
            if (kind == 0)
                grp->bat = std::make_unique<BatchEngine>(w->comps, grp->scene, opts, cell_capacity);
            else
                grp->seq = std::make_unique<SequentialEngine>(w->comps, grp->scene, opts);
            e->groups.push_back(std::move(grp));
        }
    });
    if (rc != 0) {
        delete e;
        return nullptr;
    }
    return e;
}

void* rr_engine_new(void* wp, int kind, int threads, int use_under, int cell_capacity, int group_size) {
    return rr_engine_new_groups(wp, kind, threads, use_under, cell_capacity, group_size, -1);
}

void rr_engine_free(void* ep) { delete static_cast<Engine*>(ep); }

// rep: obstacle, new_green, new_red, new_gray, reval_us, over_us, under_us,
// resolve_us, unknown_after_heuristic, residual_unknown, resolve_checks.
// For grouped engines the gray totals are the group's own (callers that need
// global counts recompute them from rr_engine_states).
int rr_engine_update(void* ep, std::int32_t o, const double* rt12, int lazy, std::int64_t* rep) {
    Engine* e = static_cast<Engine*>(ep);
    return guarded([&] {
        const int m = static_cast<int>(e->world->scene.obstacles.size());
        if (o < 0 || o >= m || o / e->group_size >= static_cast<int>(e->groups.size()))
            throw std::invalid_argument("unknown obstacle id");
        Group& g = *e->groups[o / e->group_size];
        const ObstacleId local = o % e->group_size;
        const UpdateReport r = g.bat ? g.bat->update_obstacle(local, tf_of(rt12), lazy != 0)
                                     : g.seq->update_obstacle(local, tf_of(rt12), lazy != 0);
        if (rep) {
            const std::int64_t v[11] = {o, r.new_green, r.new_red, r.new_gray, r.reval_us, r.over_us,
                                        r.under_us, r.resolve_us, r.unknown_after_heuristic,
                                        r.residual_unknown, r.resolve_checks};
            std::memcpy(rep, v, sizeof(v));
        }
    });
}

// Applies n moves; returns wall-clock microseconds spent inside the
// reference update calls through *elapsed_us (the reference CPU arm).
int rr_engine_run(void* ep, int n, const std::int32_t* ids, const double* rt12, int lazy, double* elapsed_us) {
    Engine* e = static_cast<Engine*>(ep);
    return guarded([&] {
        const int m = static_cast<int>(e->world->scene.obstacles.size());
        const auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < n; ++i) {
            const int o = ids[i];
            if (o < 0 || o >= m || o / e->group_size >= static_cast<int>(e->groups.size()))
                throw std::invalid_argument("unknown obstacle id");
            Group& g = *e->groups[o / e->group_size];
            const ObstacleId local = o % e->group_size;
            if (g.bat)
                g.bat->update_obstacle(local, tf_of(rt12 + 12 * i), lazy != 0);
            else
                g.seq->update_obstacle(local, tf_of(rt12 + 12 * i), lazy != 0);
        }
        const auto t1 = std::chrono::steady_clock::now();
        if (elapsed_us) *elapsed_us = std::chrono::duration<double, std::micro>(t1 - t0).count();
    });
}

// The same moves with the obstacle groups' engines run concurrently, one host thread
// per group (at most `threads` at a time): the groups are independent engines over
// the same components, and each group's moves keep their order, so the combined
// states and bits equal rr_engine_run's.  The grouped reference's use of all host
// threads (a single SequentialEngine is single-threaded).
int rr_engine_run_parallel(void* ep, int n, const std::int32_t* ids, const double* rt12, int lazy, int threads,
                           double* elapsed_us) {
    Engine* e = static_cast<Engine*>(ep);
    return guarded([&] {
        const int m = static_cast<int>(e->world->scene.obstacles.size());
        const int ng = static_cast<int>(e->groups.size());
        std::vector<std::vector<int>> per(ng);
        for (int i = 0; i < n; ++i) {
            const int o = ids[i];
            if (o < 0 || o >= m || o / e->group_size >= ng) throw std::invalid_argument("unknown obstacle id");
            per[o / e->group_size].push_back(i);
        }
        const int nt = std::max(1, std::min(threads, ng));
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        std::vector<std::string> errs(nt);
        for (int t = 0; t < nt; ++t)
            pool.emplace_back([&, t] {
                try {
                    for (int g = t; g < ng; g += nt) {
                        Group& grp = *e->groups[g];
                        for (int i : per[g]) {
                            const ObstacleId local = ids[i] % e->group_size;
                            if (grp.bat)
                                grp.bat->update_obstacle(local, tf_of(rt12 + 12 * i), lazy != 0);
                            else
                                grp.seq->update_obstacle(local, tf_of(rt12 + 12 * i), lazy != 0);
                        }
                    }
                } catch (const std::exception& ex) {
                    errs[t] = ex.what();
                }
            });
        for (auto& th : pool) th.join();
        const auto t1 = std::chrono::steady_clock::now();
        for (const auto& er : errs)
            if (!er.empty()) throw std::runtime_error(er);
        if (elapsed_us) *elapsed_us = std::chrono::duration<double, std::micro>(t1 - t0).count();
    });
}

// Exact-resolve inputs: forward_kinematics (proj/src/robot.cpp:66-84) of every
// discretized configuration of every component (build_components,
// roadmap.cpp:104-127), body-major per configuration: off[N+1] (configurations),
// poses[total*B*12] (r[9], t[3]).  Pass poses = nullptr to size the buffer.
int rr_world_poses(void* wp, std::int64_t* off, double* poses) {
    const World* w = static_cast<const World*>(wp);
    return guarded([&] {
        const RobotModel& m = w->scene.robot;
        const int B = static_cast<int>(m.bodies.size());
        std::int64_t k = 0;
        off[0] = 0;
        for (size_t c = 0; c < w->comps.cfgs.size(); ++c) {
            for (const Configuration& cfg : w->comps.cfgs[c]) {
                if (poses) {
                    const std::vector<Transform> fk = forward_kinematics(m, cfg);
                    for (int b = 0; b < B; ++b) put_tf(fk[b], poses + (k * B + b) * 12);
                }
                ++k;
            }
            off[c + 1] = k;
        }
    });
}

// polytopes_intersect (geometry.cpp:278-303) of ConvexPolytope::box(he_a, a) and
// ConvexPolytope::box(he_b, b) (:228-254): the exact resolve's pair predicate.
int rr_box_intersect(const double* rt_a, const double* he_a, const double* rt_b, const double* he_b, int* out) {
    return guarded([&] {
        const ConvexPolytope pa = ConvexPolytope::box({he_a[0], he_a[1], he_a[2]}, tf_of(rt_a));
        const ConvexPolytope pb = ConvexPolytope::box({he_b[0], he_b[1], he_b[2]}, tf_of(rt_b));
        *out = polytopes_intersect(pa, pb) ? 1 : 0;
    });
}

// Robot body half extents (robot.hpp BoxBody), B*3.
int rr_world_body_he(void* wp, double* he) {
    const World* w = static_cast<const World*>(wp);
    return guarded([&] {
        for (size_t b = 0; b < w->scene.robot.bodies.size(); ++b) {
            const Vec3& v = w->scene.robot.bodies[b].half_extents;
            he[3 * b] = v.x, he[3 * b + 1] = v.y, he[3 * b + 2] = v.z;
        }
    });
}

// exact_component_valid (roadmap.cpp:129-163) of ids against the scene of a
// single-group engine (its obstacles posed and activated by its moves).
int rr_engine_exact(void* ep, int n, const std::int32_t* ids, std::uint8_t* free_out) {
    Engine* e = static_cast<Engine*>(ep);
    return guarded([&] {
        if (e->groups.size() != 1) throw std::invalid_argument("exact checks need a single obstacle group");
        const Scene& sc = e->groups[0]->scene;
        for (int i = 0; i < n; ++i)
            free_out[i] = exact_component_valid(e->world->comps.cfgs[ids[i]], sc.robot, sc) ? 1 : 0;
    });
}

// BatchEngine::resolve_all_unknown (engine_batch.cpp:217-227), single group.
int rr_engine_resolve_all(void* ep, std::int32_t* resolved) {
    Engine* e = static_cast<Engine*>(ep);
    return guarded([&] {
        if (e->groups.size() != 1 || !e->groups[0]->bat) throw std::invalid_argument("single batch engine only");
        *resolved = e->groups[0]->bat->resolve_all_unknown();
    });
}

// Combined labels: red > gray > green over groups.
int rr_engine_states(void* ep, std::uint8_t* out) {
    Engine* e = static_cast<Engine*>(ep);
    return guarded([&] {
        const int n = e->world->comps.count();
        std::memset(out, 0, n);
        for (const auto& g : e->groups) {
            const auto& st = g->bat ? g->bat->states() : g->seq->states();
            for (int c = 0; c < n; ++c) {
                const std::uint8_t v = static_cast<std::uint8_t>(st[c]);
                if (v == 1 || (v == 2 && out[c] != 1)) out[c] = v;
            }
        }
    });
}

// Bits: words_per_comp = number of groups; word g holds group g's bitset.
int rr_engine_bits(void* ep, std::uint64_t* out) {
    Engine* e = static_cast<Engine*>(ep);
    return guarded([&] {
        const int n = e->world->comps.count();
        const size_t ng = e->groups.size();
        for (size_t g = 0; g < ng; ++g) {
            const auto& b = e->groups[g]->bat ? e->groups[g]->bat->obstacle_bits() : e->groups[g]->seq->obstacle_bits();
            for (int c = 0; c < n; ++c) out[static_cast<size_t>(c) * ng + g] = b[c];
        }
    });
}

int rr_engine_groups(void* ep) { return static_cast<int>(static_cast<Engine*>(ep)->groups.size()); }

// batch_over (kind 0) / batch_under (kind 1) on explicit candidates
// (engine_batch.hpp:34-37); sequential engines answer with narrow tests.
int rr_engine_mask(void* ep, int kind, const std::int32_t* cands, int n, std::int32_t o, std::uint8_t* mask) {
    Engine* e = static_cast<Engine*>(ep);
    return guarded([&] {
        Group& g = *e->groups[o / e->group_size];
        const ObstacleId local = o % e->group_size;
        std::vector<ComponentId> c(cands, cands + n);
        if (g.bat) {
            std::vector<std::uint8_t> m;
            if (kind == 0)
                g.bat->batch_over(c, local, m);
            else
                g.bat->batch_under(c, local, m);
            std::memcpy(mask, m.data(), m.size());
        } else {
            for (int i = 0; i < n; ++i)
                mask[i] = kind == 0 ? g.seq->narrow_over_test(local, c[i]) : g.seq->narrow_under_test(local, c[i]);
        }
    });
}

// ---------------------------------------------------------------- kernels

// proj/tests/test_kernels.cpp:50-71: 5000 near-contact boxes, one obstacle,
// 10000 random indices, seed 2025.  Writes boxes (n_boxes*21), obstacle (21),
// idx (n_idx), and the scalar backend's bytes (n_idx).  The obstacle's
// random_obb (proj/tests/oracles.hpp:98-109) is expanded inline — same Rng draw
// order — so its pose (rotation + centre, obstacle_pose12) and half extents
// (obstacle_he3) can be handed to an engine as a box obstacle.
int rr_kat_sat(std::uint64_t seed, int n_boxes, int n_idx, double* boxes21, double* obstacle21, std::int32_t* idx,
               std::uint8_t* out, double* obstacle_pose12, double* obstacle_he3) {
    return guarded([&] {
        Rng rng(seed);
        std::vector<kern::SatBox> boxes;
        auto sat_of = [](const Obb& o) {
            const ObbCorners c = obb_corners(o);
            return kern::sat_prep(&c[0].x);
        };
        for (int i = 0; i < n_boxes; ++i) boxes.push_back(sat_of(oracle::random_obb(rng, 1.5, 1.2)));
        const Transform rot = oracle::random_rotation(rng);
        Obb ob;
        ob.center = {rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5)};
        ob.axes[0] = rot.rotate({1, 0, 0});
        ob.axes[1] = rot.rotate({0, 1, 0});
        ob.axes[2] = rot.rotate({0, 0, 1});
        ob.half_extents = {rng.uniform(0.05, 2.0), rng.uniform(0.05, 2.0), rng.uniform(0.05, 2.0)};
        const kern::SatBox obstacle = sat_of(ob);
        for (int i = 0; i < n_idx; ++i) idx[i] = rng.uniform_int(0, n_boxes - 1);
        kern::scalar_backend().sat_batch(boxes.data(), idx, n_idx, &obstacle, out);
        for (int i = 0; i < n_boxes; ++i) put_sat(boxes[i], boxes21 + 21 * i);
        put_sat(obstacle, obstacle21);
        Transform pose = rot;
        pose.t = ob.center;
        put_tf(pose, obstacle_pose12);
        obstacle_he3[0] = ob.half_extents.x;
        obstacle_he3[1] = ob.half_extents.y;
        obstacle_he3[2] = ob.half_extents.z;
    });
}

// proj/tests/test_kernels.cpp:89-121: 4000 random + 50 point segments,
// 9001 indices, centre (0.3,-0.2,0.1), r_total 1.1, seed 777.
int rr_kat_seg(std::uint64_t seed, int n_rand, int n_point, int n_idx, double* segs7, std::int32_t* idx,
               std::uint8_t* out) {
    return guarded([&] {
        Rng rng(seed);
        std::vector<kern::SegPrep> segs;
        for (int i = 0; i < n_rand; ++i) {
            const double seg[6] = {rng.uniform(-2, 2), rng.uniform(-2, 2), rng.uniform(-2, 2),
                                   rng.uniform(-2, 2), rng.uniform(-2, 2), rng.uniform(-2, 2)};
            segs.push_back(kern::seg_prep(seg));
        }
        for (int i = 0; i < n_point; ++i) {
            const double x = rng.uniform(-2, 2), y = rng.uniform(-2, 2), z = rng.uniform(-2, 2);
            const double seg[6] = {x, y, z, x, y, z};
            segs.push_back(kern::seg_prep(seg));
        }
        for (int i = 0; i < n_idx; ++i) idx[i] = rng.uniform_int(0, static_cast<int>(segs.size()) - 1);
        const double center[3] = {0.3, -0.2, 0.1};
        kern::scalar_backend().seg_sphere_batch(segs.data(), idx, n_idx, center, 1.1, out);
        for (size_t i = 0; i < segs.size(); ++i) {
            double* d = segs7 + 7 * i;
            for (int j = 0; j < 3; ++j) d[j] = segs[i].a[j];
            for (int j = 0; j < 3; ++j) d[3 + j] = segs[i].d[j];
            d[6] = segs[i].dd;
        }
    });
}

// Random box pairs (oracles.hpp:98-109 random_obb) with the reference SAT
// verdict and the oracle's sat_margin (oracles.hpp:62-84).
int rr_kat_sat_pairs(std::uint64_t seed, int n, double span, double extent, double* a21, double* b21,
                     std::uint8_t* out, double* margin) {
    return guarded([&] {
        Rng rng(seed);
        for (int i = 0; i < n; ++i) {
            const Obb a = oracle::random_obb(rng, span, extent);
            const Obb b = oracle::random_obb(rng, span, extent);
            const ObbCorners ca = obb_corners(a), cb = obb_corners(b);
            const kern::SatBox sa = kern::sat_prep(&ca[0].x), sb = kern::sat_prep(&cb[0].x);
            put_sat(sa, a21 + 21 * i);
            put_sat(sb, b21 + 21 * i);
            out[i] = kern::sat_boxes(sa, sb) ? 1 : 0;
            if (margin) margin[i] = oracle::sat_margin(a, b);
        }
    });
}

// sat_prep on caller corners (kernels_scalar.cpp:7-30).
int rr_sat_prep(int n, const double* corners24, double* out21) {
    return guarded([&] {
        for (int i = 0; i < n; ++i) put_sat(kern::sat_prep(corners24 + 24 * i), out21 + 21 * i);
    });
}

// Transform helpers used to generate poses exactly as the reference does.
int rr_tf_euler(double rx, double ry, double rz, double* rt12) {
    return guarded([&] { put_tf(Transform::from_euler_xyz(rx, ry, rz), rt12); });
}

int rr_tf_axis_angle(const double* axis3, double angle, double* rt12) {
    return guarded([&] { put_tf(Transform::rotation_axis_angle({axis3[0], axis3[1], axis3[2]}, angle), rt12); });
}

// build_prm (proj/src/roadmap.cpp:56-102) over the env and robot of a .scn text with
// no obstacles (the benchmark's build scene, proj/src/bench.cpp:90-91); n_nodes, k and
// seed override the scenario's when >= 0.  dof_bounds_for (roadmap.cpp:20-30) into lo/hi.
int rr_build_prm(const char* text, int n_nodes, int k, long long seed, int* dof, double* lo, double* hi,
                 double* nodes, std::int64_t node_cap, std::int32_t* edges, std::int64_t edge_cap,
                 std::int64_t* counts, double* seconds) {
    return guarded([&] {
        const Scenario s = parse_scenario_text(text, "<scn>");
        const Scene build_scene{s.env, {}, s.robot};
        const int n = n_nodes >= 0 ? n_nodes : s.nodes;
        const int kk = k >= 0 ? k : s.k_neighbors;
        const std::uint64_t sd = seed >= 0 ? static_cast<std::uint64_t>(seed) : s.roadmap_seed;
        const auto t0 = std::chrono::steady_clock::now();
        const Roadmap r = build_prm(build_scene, n, kk, s.effective_epsilon(), sd);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        const DofBounds b = dof_bounds_for(s.robot, s.env);
        const int D = static_cast<int>(b.lo.size());
        if (dof) *dof = D;
        for (int q = 0; q < D; ++q) {
            if (lo) lo[q] = b.lo[q];
            if (hi) hi[q] = b.hi[q];
        }
        counts[0] = static_cast<std::int64_t>(r.nodes.size());
        counts[1] = static_cast<std::int64_t>(r.edges.size());
        if (nodes) {
            if (counts[0] > node_cap) throw std::invalid_argument("node buffer too small");
            for (size_t i = 0; i < r.nodes.size(); ++i)
                for (int q = 0; q < D; ++q) nodes[i * D + q] = r.nodes[i][q];
        }
        if (edges) {
            if (counts[1] > edge_cap) throw std::invalid_argument("edge buffer too small");
            for (size_t e = 0; e < r.edges.size(); ++e) {
                edges[2 * e] = r.edges[e].first;
                edges[2 * e + 1] = r.edges[e].second;
            }
        }
    });
}

}  // extern "C"
