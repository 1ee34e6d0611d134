// engine_gpu.hpp — rgg::GpuEngine: the B200 drop-in for rgg::BatchEngine.
//
// Same public surface as the reference's update API
//   class rgg::BatchEngine    proj/include/rgg/engine_batch.hpp:17-63
// (constructor over ComponentSet + Scene&, update_obstacle, batch_update,
// resolve_all_unknown, states, obstacle_bits, unknown_count, layout, grid,
// batch_over, batch_under), header-only over the C-ABI of include/rgg_gpu.h
// (link paper_2603_28674_b200/lib/librgg_gpu.so).  A maintainer compiles it
// against the reference's own headers; see INTEGRATION.md.
//
// Semantics kept from the reference:
//  * the engine keeps a non-owning pointer to the ComponentSet and mutates
//    Scene& (obstacles[o].pose, .active) on every move (engine_batch.cpp:156-158);
//  * std::invalid_argument("unknown obstacle id") / ("obstacle bitsets support at
//    most 64 obstacles") are thrown with the reference's texts;
//  * lazy and eager updates and resolve_all_unknown run on the GPU.  The exact
//    resolve (exact_component_valid, roadmap.cpp:129-163) needs the world pose of
//    every body at every discretized configuration: on first use the wrapper
//    evaluates the reference's own forward_kinematics (robot.cpp:66-84) over
//    components.cfgs once and uploads it (rgg_gpu_set_resolver).  The GPU checks
//    against the obstacles this engine has moved at their engine poses, and
//    against the Scene's other active obstacles at their scene poses (listed
//    before every exact resolve, rgg_gpu_set_active_obstacles).
// grid() is the reference's own SpatialGrid over the component AABBs, built on first
// call (the GPU engine bins on its own cells and never reads it).
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <cstring>
#include <vector>

#include "rgg/batch_layout.hpp"
#include "rgg/geometry.hpp"
#include "rgg/roadmap.hpp"
#include "rgg/robot.hpp"
#include "rgg/spatial_grid.hpp"
#include "rgg/update_report.hpp"
#include "rgg_gpu.h"

namespace rgg {

class GpuEngine {
public:
    GpuEngine(const ComponentSet& components, Scene& scene, EngineOptions options = {}, int cell_capacity = 1024,
              int device = 0, bool allow_wide = false)
        : components_(&components), scene_(scene), options_(options), bounds_(scene.bounds),
          cell_capacity_(cell_capacity) {
        if (scene.obstacles.size() > 64 && !allow_wide)
            throw std::invalid_argument("obstacle bitsets support at most 64 obstacles");
        // The component view (include/rgg_gpu.h rgg_component_view): the serialize step's
        // inputs only (OBB corners, the real segments' end points in CSR rows, slot radii);
        // sat_prep, the AABBs and seg_prep run on the device.  The padded BatchLayout
        // (BatchLayout::serialize, batch_layout.cpp:21-146) is built only if layout() is called.
        const int N = components.count();
        const int B = static_cast<int>(components.spheres.per_body.size());
        const int K = components.max_segments;
        // slot layout: spheres per body x the worst split factor (batch_layout.cpp:28-43)
        int max_parts = 1, max_spheres = 1;
        for (int b = 0; b < B; ++b)
            max_spheres = std::max(max_spheres, static_cast<int>(components.spheres.per_body[b].size()));
        for (const EdgeGeometry& g : components.geometry)
            for (int b = 0; b < B; ++b) {
                std::vector<int> parts(components.spheres.per_body[b].size(), 0);
                for (const Spline& s : g.under[b]) max_parts = std::max(max_parts, ++parts[s.sphere_index]);
            }
        const int S = max_spheres * max_parts;
        n_components_ = N;
        corners_.resize(static_cast<size_t>(N) * B * 24);
        spline_r_.assign(static_cast<size_t>(B) * S, 0.0);
        std::vector<std::int32_t> count(static_cast<size_t>(N) * B * S, 0);
        std::vector<const Spline*> row_spline(count.size(), nullptr);
        for (int c = 0; c < N; ++c) {
            const EdgeGeometry& g = components.geometry[c];
            for (int b = 0; b < B; ++b) {
                const ObbCorners oc = obb_corners(g.over[b]);  // write_corners, batch_layout.cpp:10-17
                double* d = &corners_[(static_cast<size_t>(c) * B + b) * 24];
                for (int i = 0; i < 8; ++i) d[3 * i] = oc[i].x, d[3 * i + 1] = oc[i].y, d[3 * i + 2] = oc[i].z;
                std::vector<int> used(components.spheres.per_body[b].size(), 0);
                for (const Spline& s : g.under[b]) {  // batch_layout.cpp:64-105
                    if (s.segment_count() > K)
                        throw std::logic_error("spline exceeds the segment cap; the build policy should have split it");
                    const int slot = s.sphere_index * max_parts + used[s.sphere_index]++;
                    double& slot_radius = spline_r_[static_cast<size_t>(b) * S + slot];
                    if (slot_radius == 0.0) slot_radius = s.radius;
                    else if (slot_radius != s.radius) throw std::logic_error("inconsistent spline radius for a layout slot");
                    const size_t row = (static_cast<size_t>(c) * B + b) * S + slot;
                    row_spline[row] = &s;
                    count[row] = s.points.size() == 1 ? 1 : static_cast<std::int32_t>(s.points.size()) - 1;
                }
            }
        }
        row_off_.assign(count.size() + 1, 0);
        for (size_t r = 0; r < count.size(); ++r) row_off_[r + 1] = row_off_[r] + count[r];
        seg_pts_.resize(static_cast<size_t>(row_off_.back()) * 6);
        for (size_t r = 0; r < count.size(); ++r) {
            const Spline* s = row_spline[r];
            if (!s) continue;
            double* d = &seg_pts_[static_cast<size_t>(row_off_[r]) * 6];
            const size_t np = s->points.size();
            for (size_t p = 0; p < (np == 1 ? 1 : np - 1); ++p, d += 6) {  // one degenerate segment for a point
                const Vec3& a = s->points[p];
                const Vec3& e = s->points[np == 1 ? p : p + 1];
                d[0] = a.x, d[1] = a.y, d[2] = a.z, d[3] = e.x, d[4] = e.y, d[5] = e.z;
            }
        }
        // obstacle side (batch_layout.cpp:108-131)
        const int M = static_cast<int>(scene.obstacles.size());
        int C = 1;
        for (const ObstacleModel& o : scene.obstacles) C = std::max(C, static_cast<int>(o.inner.size()));
        obst_he_.resize(static_cast<size_t>(M) * 3);
        obst_sl_.assign(static_cast<size_t>(M) * C * 3, 0.0);
        obst_r_.assign(M, 0.0);
        obst_n_.assign(M, 0);
        for (int o = 0; o < M; ++o) {
            const ObstacleModel& m = scene.obstacles[o];
            for (const Sphere& s : m.inner)
                if (s.radius != m.inner[0].radius)
                    throw std::invalid_argument("layout requires one shared sphere radius per obstacle");
            obst_he_[3 * o] = m.half_extents.x, obst_he_[3 * o + 1] = m.half_extents.y, obst_he_[3 * o + 2] = m.half_extents.z;
            for (size_t s = 0; s < m.inner.size(); ++s) {
                double* d = &obst_sl_[(static_cast<size_t>(o) * C + s) * 3];
                d[0] = m.inner[s].center.x, d[1] = m.inner[s].center.y, d[2] = m.inner[s].center.z;
            }
            obst_r_[o] = m.inner.empty() ? 0.0 : m.inner[0].radius;
            obst_n_[o] = static_cast<std::int32_t>(m.inner.size());
        }
        rgg_component_view v{N, B, S, M, C, corners_.data(), row_off_.data(), seg_pts_.data(), spline_r_.data(),
                             obst_he_.data(), obst_sl_.data(), obst_r_.data(), obst_n_.data()};
        rgg_gpu_options opt{};
        opt.device = device;
        opt.use_under = options.use_under ? 1 : 0;
        // the reference's cell_capacity bounds a SpatialGrid cell's inline components before
        // its overflow list (spatial_grid.cpp:94-110); here it bounds a cell's inline event
        // slots before the overflow pool.  Either way only storage changes, never a result.
        opt.cell_capacity = cell_capacity < 1 ? 1 : cell_capacity;
        opt.allow_wide = allow_wide ? 1 : 0;
        const int rc = rgg_gpu_create_from_components(&v, &opt, &h_);
        if (rc != RGG_OK) {
            const std::string msg = rgg_gpu_last_error(h_);
            rgg_gpu_destroy(h_);
            h_ = nullptr;
            raise(rc, msg);
        }
        rgg_gpu_count(h_, nullptr, nullptr, &words_);
        states_.assign(n_components_, ValidityState::Valid);
        bits_.assign(static_cast<size_t>(n_components_) * words_, 0);
        // the host buffers are not needed any more (the engine copied them into HBM)
        std::vector<double>().swap(corners_);
        std::vector<double>().swap(seg_pts_);
        std::vector<std::int32_t>().swap(row_off_);
    }

    ~GpuEngine() { rgg_gpu_destroy(h_); }
    GpuEngine(const GpuEngine&) = delete;
    GpuEngine& operator=(const GpuEngine&) = delete;

    UpdateReport update_obstacle(ObstacleId o, const Transform& pose, bool lazy) {
        return batch_update({{o, pose}}, lazy).at(0);
    }

    std::vector<UpdateReport> batch_update(const std::vector<std::pair<ObstacleId, Transform>>& moves, bool lazy) {
        std::vector<UpdateReport> out;
        if (moves.empty()) return out;
        if (!lazy) ensure_resolver();
        std::vector<std::int32_t> ids;
        std::vector<double> rt;
        for (const auto& [o, pose] : moves) {
            ids.push_back(o);
            for (double r : pose.r) rt.push_back(r);
            rt.push_back(pose.t.x), rt.push_back(pose.t.y), rt.push_back(pose.t.z);
        }
        std::vector<rgg_update_report> rep(moves.size());
        // eager: move by move on the device, each move's gray over-hits resolved exactly
        const int rc = rgg_gpu_update(h_, ids.data(), rt.data(), static_cast<std::int32_t>(ids.size()),
                                      (lazy ? RGG_LAZY : RGG_EAGER) | RGG_PER_MOVE, rep.data());
        // the moves the device applied mutate the scene: all of them, those before the first
        // unknown id (the reference's sequential loop throws there, engine_batch.cpp:146-148),
        // or none when the call was rejected before the device ran or the update failed
        size_t applied = moves.size();
        if (rc != RGG_OK) {
            applied = 0;
            if (rc == RGG_EINVAL && std::strcmp(rgg_gpu_last_error(h_), "unknown obstacle id") == 0)
                while (applied < moves.size() && moves[applied].first >= 0 &&
                       moves[applied].first < static_cast<ObstacleId>(scene_.obstacles.size()))
                    ++applied;
        }
        for (size_t i = 0; i < applied; ++i) {
            scene_.obstacles[moves[i].first].pose = moves[i].second;
            scene_.obstacles[moves[i].first].active = true;
            moved_[moves[i].first] = 1;
        }
        stale_ = true;
        if (rc != RGG_OK) raise(rc, rgg_gpu_last_error(h_));
        for (const rgg_update_report& r : rep) out.push_back(convert(r));
        return out;
    }

    int resolve_all_unknown() {
        ensure_resolver();
        std::int32_t n = 0;
        check(rgg_gpu_resolve_all(h_, &n));
        stale_ = true;
        return n;
    }

    const std::vector<ValidityState>& states() const {
        refresh();
        return states_;
    }
    const std::vector<std::uint64_t>& obstacle_bits() const {
        refresh();
        return bits_;
    }
    int unknown_count() const {
        std::int32_t n = 0;
        check(rgg_gpu_unknown_count(h_, &n));
        return n;
    }
    // The reference's serialized layout, built on first use (the engine itself never
    // reads it): obstacle rows at the Scene's current poses, which this engine keeps
    // equal to the moved obstacles' poses, as the reference's update_transforms does.
    // Scribbling into its padding (test_batch.cpp:248-256) cannot change a GPU mask:
    // the device store holds the real segments only.
    const BatchLayout& layout() const {
        if (!layout_) layout_ = std::make_unique<BatchLayout>(BatchLayout::serialize(*components_, scene_.obstacles));
        return *layout_;
    }
    // BatchEngine::grid() (engine_batch.hpp:32): SpatialGrid::build over the layout's component
    // AABBs, the construction-time scene bounds and cell capacity (engine_batch.cpp:26)
    const SpatialGrid& grid() const {
        if (!grid_) grid_ = std::make_unique<SpatialGrid>(SpatialGrid::build(layout().component_aabb, bounds_, cell_capacity_));
        return *grid_;
    }
    int words_per_component() const { return words_; }

    void batch_over(const std::vector<ComponentId>& candidates, ObstacleId o, std::vector<std::uint8_t>& mask) {
        mask.assign(candidates.size(), 0);
        check(rgg_gpu_pair_masks(h_, 0, candidates.data(), static_cast<std::int32_t>(candidates.size()), o, mask.data()));
    }
    void batch_under(const std::vector<ComponentId>& candidates, ObstacleId o, std::vector<std::uint8_t>& mask) {
        mask.assign(candidates.size(), 0);
        check(rgg_gpu_pair_masks(h_, 1, candidates.data(), static_cast<std::int32_t>(candidates.size()), o, mask.data()));
    }

private:
    [[noreturn]] static void raise(int rc, const std::string& msg) {
        if (rc == RGG_EINVAL) throw std::invalid_argument(msg);
        if (rc == RGG_ELOGIC) throw std::logic_error(msg);
        throw std::runtime_error("rgg_gpu error " + std::to_string(rc) + ": " + msg);
    }
    void check(int rc) const {
        if (rc != RGG_OK) raise(rc, rgg_gpu_last_error(h_));
    }
    static UpdateReport convert(const rgg_update_report& r) {
        UpdateReport u;
        u.obstacle = r.obstacle;
        u.new_green = r.new_green;
        u.new_red = r.new_red;
        u.new_gray = r.new_gray;
        u.reval_us = r.reval_us;
        u.over_us = r.over_us;
        u.under_us = r.under_us;
        u.resolve_us = r.resolve_us;
        u.unknown_after_heuristic = r.unknown_after_heuristic;
        u.residual_unknown = r.residual_unknown;
        u.resolve_checks = r.resolve_checks;
        return u;
    }
    void refresh() const {
        if (!stale_) return;
        std::vector<std::uint8_t> st(states_.size());
        check(rgg_gpu_read_states(h_, st.data()));
        for (size_t i = 0; i < st.size(); ++i) states_[i] = static_cast<ValidityState>(st[i]);
        check(rgg_gpu_read_bits(h_, bits_.data(), words_));
        stale_ = false;
    }
    // The exact resolve's inputs, once: forward_kinematics of every configuration
    // (body-major per configuration) and the body half extents.
    void ensure_resolver() {
        // obstacles active in the Scene that this engine has not moved: checked at their scene pose
        std::vector<std::int32_t> sid;
        std::vector<double> srt;
        for (size_t o = 0; o < scene_.obstacles.size(); ++o)
            if (scene_.obstacles[o].active && !moved_[o]) {
                const Transform& p = scene_.obstacles[o].pose;
                sid.push_back(static_cast<std::int32_t>(o));
                for (double r : p.r) srt.push_back(r);
                srt.push_back(p.t.x), srt.push_back(p.t.y), srt.push_back(p.t.z);
            }
        if (sid != static_ids_ || srt != static_rt_) {
            check(rgg_gpu_set_active_obstacles(h_, sid.data(), srt.data(), static_cast<std::int32_t>(sid.size())));
            static_ids_ = std::move(sid);
            static_rt_ = std::move(srt);
        }
        if (resolver_ready_) return;
        const RobotModel& m = scene_.robot;
        const int B = static_cast<int>(m.bodies.size());
        const size_t N = components_->cfgs.size();
        std::vector<std::int64_t> off(N + 1, 0);
        for (size_t c = 0; c < N; ++c) off[c + 1] = off[c] + static_cast<std::int64_t>(components_->cfgs[c].size());
        std::vector<double> poses(static_cast<size_t>(off[N]) * B * 12);
        std::vector<double> he(static_cast<size_t>(B) * 3);
        for (int b = 0; b < B; ++b)
            he[3 * b] = m.bodies[b].half_extents.x, he[3 * b + 1] = m.bodies[b].half_extents.y,
                   he[3 * b + 2] = m.bodies[b].half_extents.z;
        size_t k = 0;
        for (size_t c = 0; c < N; ++c)
            for (const Configuration& cfg : components_->cfgs[c]) {
                const std::vector<Transform> fk = forward_kinematics(m, cfg);
                for (int b = 0; b < B; ++b, ++k) {
                    double* d = &poses[k * 12];
                    for (int j = 0; j < 9; ++j) d[j] = fk[b].r[j];
                    d[9] = fk[b].t.x, d[10] = fk[b].t.y, d[11] = fk[b].t.z;
                }
            }
        const rgg_resolve_view v{static_cast<std::int32_t>(N), B, he.data(), off.data(), poses.data()};
        check(rgg_gpu_set_resolver(h_, &v));
        resolver_ready_ = true;
    }

    const ComponentSet* components_;
    Scene& scene_;
    EngineOptions options_;
    Aabb bounds_;
    int cell_capacity_;
    mutable std::unique_ptr<BatchLayout> layout_;
    mutable std::unique_ptr<SpatialGrid> grid_;
    int n_components_ = 0;
    std::vector<double> corners_, seg_pts_, spline_r_, obst_he_, obst_sl_, obst_r_;
    std::vector<std::int32_t> row_off_, obst_n_;
    rgg_gpu* h_ = nullptr;
    std::int32_t words_ = 1;
    mutable bool stale_ = false;
    bool resolver_ready_ = false;
    std::vector<std::int32_t> static_ids_;  // the scene-active list last uploaded
    std::vector<double> static_rt_;
    std::vector<std::uint8_t> moved_ = std::vector<std::uint8_t>(scene_.obstacles.size(), 0);
    mutable std::vector<ValidityState> states_;
    mutable std::vector<std::uint64_t> bits_;
};

}  // namespace rgg
