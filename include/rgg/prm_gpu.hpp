// rgg/prm_gpu.hpp — drop-in for rgg::build_prm (proj/src/roadmap.cpp:56-102) with the
// kNN candidate loop on the GPU (include/rgg_prm.h, lib/librgg_build.so).
//
// Compiled against the reference's headers, like rgg/engine_gpu.hpp.  Same signature,
// result and exceptions as the reference:
//   * n_nodes < 1 / k_neighbors < 1 -> std::invalid_argument (roadmap.cpp:57-58);
//     scene.robot.validate() first (:59);
//   * nodes from the reference's own Rng and dof_bounds_for (:61-71);
//   * candidates: rgg_prm_knn_edges — the k nearest under dof_distance2 with the
//     pair<double, NodeId> order, (min, max), sorted, unique (:73-93), bit-identical;
//   * with active obstacles the node and edge validity checks (:69, :95-99) run on the
//     GPU: forward_kinematics (robot.cpp:66-84) of every node / discretize_edge
//     configuration on the host, then one rgg_exact_valid_sets call (include/rgg_gpu.h,
//     lib/librgg_gpu.so) for all nodes and one for all candidate edges.  A degenerate
//     body or obstacle box throws std::invalid_argument("degenerate polytope") up front,
//     where the reference throws it at the first pair that passes the AABB gate.
// A GPU failure throws std::runtime_error with the library's message.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "rgg/roadmap.hpp"
#include "rgg/rng.hpp"
#include "rgg/robot.hpp"
#include "rgg_gpu.h"
#include "rgg_prm.h"

namespace rgg::gpu {

// exact_component_valid of each configuration set against the scene's active obstacles, on the GPU.
inline std::vector<std::uint8_t> exact_valid_sets(const std::vector<std::vector<Configuration>>& sets,
                                                  const Scene& scene) {
    const RobotModel& m = scene.robot;
    const int B = static_cast<int>(m.bodies.size());
    std::vector<double> he(static_cast<size_t>(B) * 3), ohe, ort;
    for (int b = 0; b < B; ++b)
        he[3 * b] = m.bodies[b].half_extents.x, he[3 * b + 1] = m.bodies[b].half_extents.y,
               he[3 * b + 2] = m.bodies[b].half_extents.z;
    for (const ObstacleModel& o : scene.obstacles) {
        if (!o.active) continue;
        ohe.push_back(o.half_extents.x), ohe.push_back(o.half_extents.y), ohe.push_back(o.half_extents.z);
        for (double r : o.pose.r) ort.push_back(r);
        ort.push_back(o.pose.t.x), ort.push_back(o.pose.t.y), ort.push_back(o.pose.t.z);
    }
    std::vector<std::int64_t> off(sets.size() + 1, 0);
    for (size_t i = 0; i < sets.size(); ++i) off[i + 1] = off[i] + static_cast<std::int64_t>(sets[i].size());
    std::vector<double> poses(static_cast<size_t>(off.back()) * B * 12);
    size_t k = 0;
    for (const auto& set : sets)
        for (const Configuration& cfg : set) {
            const std::vector<Transform> fk = forward_kinematics(m, cfg);
            for (int b = 0; b < B; ++b, ++k) {
                double* d = &poses[k * 12];
                for (int j = 0; j < 9; ++j) d[j] = fk[b].r[j];
                d[9] = fk[b].t.x, d[10] = fk[b].t.y, d[11] = fk[b].t.z;
            }
        }
    std::vector<std::uint8_t> free(sets.size(), 1);
    const int rc = rgg_exact_valid_sets(0, static_cast<std::int32_t>(sets.size()), off.data(), B, he.data(),
                                        poses.data(), static_cast<std::int32_t>(ohe.size() / 3), ohe.data(),
                                        ort.data(), free.data());
    if (rc == RGG_EINVAL) throw std::invalid_argument("degenerate polytope");
    if (rc != RGG_OK) throw std::runtime_error("rgg_exact_valid_sets failed (" + std::to_string(rc) + ")");
    return free;
}

inline Roadmap build_prm(const Scene& scene, int n_nodes, int k_neighbors, double eps, std::uint64_t seed) {
    if (n_nodes < 1) throw std::invalid_argument("node count must be >= 1");
    if (k_neighbors < 1) throw std::invalid_argument("neighbor count must be >= 1");
    scene.robot.validate();

    const DofBounds bounds = dof_bounds_for(scene.robot, scene.bounds);
    const int dof = scene.robot.dof_count();
    bool check = false;
    for (const ObstacleModel& o : scene.obstacles) check = check || o.active;

    Rng rng(seed);
    Roadmap r;
    r.nodes.reserve(n_nodes);
    for (int i = 0; i < n_nodes; ++i) {  // the draws do not depend on the checks: sample all, then filter
        Configuration c(dof);
        for (int q = 0; q < dof; ++q) c[q] = rng.uniform(bounds.lo[q], bounds.hi[q]);
        r.nodes.push_back(std::move(c));
    }
    if (check) {
        std::vector<std::vector<Configuration>> sets;
        sets.reserve(r.nodes.size());
        for (const Configuration& c : r.nodes) sets.push_back({c, c});
        const std::vector<std::uint8_t> free = exact_valid_sets(sets, scene);
        size_t kept = 0;
        for (size_t i = 0; i < r.nodes.size(); ++i)
            if (free[i]) {
                if (kept != i) r.nodes[kept] = std::move(r.nodes[i]);
                ++kept;
            }
        r.nodes.resize(kept);
    }

    const int n = static_cast<int>(r.nodes.size());
    std::vector<double> flat(static_cast<size_t>(n) * dof);
    for (int i = 0; i < n; ++i)
        for (int q = 0; q < dof; ++q) flat[static_cast<size_t>(i) * dof + q] = r.nodes[i][q];
    const std::int64_t cap = static_cast<std::int64_t>(n) * std::max(0, std::min(k_neighbors, n - 1));
    std::vector<std::int32_t> pairs(2 * static_cast<size_t>(std::max<std::int64_t>(cap, 1)));
    std::int64_t n_pairs = 0;
    const int rc = rgg_prm_knn_edges(flat.data(), n, dof, k_neighbors, pairs.data(), cap, &n_pairs, nullptr);
    if (rc == RGG_PRM_EINVAL) throw std::invalid_argument(rgg_prm_last_error());
    if (rc != 0) throw std::runtime_error(std::string("rgg_prm_knn_edges: ") + rgg_prm_last_error());

    std::vector<std::uint8_t> free;
    if (check) {
        std::vector<std::vector<Configuration>> sets;
        sets.reserve(static_cast<size_t>(n_pairs));
        for (std::int64_t e = 0; e < n_pairs; ++e) sets.push_back(discretize_edge(r.nodes[pairs[2 * e]], r.nodes[pairs[2 * e + 1]], eps));
        free = exact_valid_sets(sets, scene);
    }
    for (std::int64_t e = 0; e < n_pairs; ++e) {
        if (check && !free[static_cast<size_t>(e)]) continue;
        r.edges.push_back({pairs[2 * e], pairs[2 * e + 1]});
    }
    r.rebuild_adjacency();
    return r;
}

}  // namespace rgg::gpu
