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
//   * with active obstacles the node and edge validity checks are the reference's own
//     exact_component_valid on the host (:69, :95-99); the benchmark's build scene has none.
// A GPU failure throws std::runtime_error with the library's message.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "rgg/roadmap.hpp"
#include "rgg/rng.hpp"
#include "rgg_prm.h"

namespace rgg::gpu {

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
    for (int i = 0; i < n_nodes; ++i) {
        Configuration c(dof);
        for (int q = 0; q < dof; ++q) c[q] = rng.uniform(bounds.lo[q], bounds.hi[q]);
        if (check && !exact_component_valid({c, c}, scene.robot, scene)) continue;
        r.nodes.push_back(std::move(c));
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

    for (std::int64_t e = 0; e < n_pairs; ++e) {
        const NodeId a = pairs[2 * e], b = pairs[2 * e + 1];
        if (check && !exact_component_valid(discretize_edge(r.nodes[a], r.nodes[b], eps), scene.robot, scene)) continue;
        r.edges.push_back({a, b});
    }
    r.rebuild_adjacency();
    return r;
}

}  // namespace rgg::gpu
