// test_gpu_engine.cpp — the C++ drop-in rgg::GpuEngine (include/rgg/engine_gpu.hpp)
// against the reference engines, compiled against the reference's own headers
// and linked with the unmodified reference library (oracle/_ref/librgg_ref.so)
// and the CUDA engine (paper_2603_28674_b200/lib/librgg_gpu.so).
//
// The cases restate the reference's own suites for the batch engine:
//   proj/tests/test_batch.cpp:208-234  batch_over / batch_under == sequential narrow tests
//   proj/tests/test_batch.cpp:260-285  states + bits + report counts == sequential after every move
//   proj/tests/test_batch.cpp:287-295  empty move list
//   proj/tests/test_sequential.cpp:106-126, :229-252  eager resolve semantics
//   proj/src/bench.cpp:57-83           scenario replay with equivalence after every iteration
//   proj/tests/test_roadmap.cpp:34-73  rgg::gpu::build_prm (include/rgg/prm_gpu.hpp) == build_prm
// Built by `make -C oracle dropin` (needs /root/reference); run by tests/test_cpp_dropin.py on a GPU.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>

#include "rgg/engine_batch.hpp"
#include "rgg/engine_gpu.hpp"
#include "rgg/engine_sequential.hpp"
#include "rgg/prm_gpu.hpp"
#include "rgg/rng.hpp"
#include "rgg/scenario.hpp"

using namespace rgg;

static int g_fail = 0, g_checks = 0;
#define EXPECT(cond, ...)                                                   \
    do {                                                                    \
        ++g_checks;                                                         \
        if (!(cond)) {                                                      \
            ++g_fail;                                                       \
            std::fprintf(stderr, "FAIL %s:%d: %s ", __FILE__, __LINE__, #cond); \
            std::fprintf(stderr, __VA_ARGS__);                              \
            std::fprintf(stderr, "\n");                                     \
        }                                                                   \
    } while (0)

// The random scene of proj/tests/test_batch.cpp's fixture: free cube robot,
// +-env_half workspace, 1-3 random box obstacles, a seeded PRM (k = 6).
struct Scenelet {
    Scene scene;
    Roadmap roadmap;
    ComponentSet components;
    Scenelet(int nodes, int n_obstacles, std::uint64_t seed, double env_half = 6.0) {
        scene.bounds = {{-env_half, -env_half, -env_half}, {env_half, env_half, env_half}};
        scene.robot = make_free_flying_box({0.5, 0.5, 0.5});
        Rng rng(seed);
        for (int i = 0; i < n_obstacles; ++i) {
            const Vec3 he{rng.uniform(0.4, 1.6), rng.uniform(0.4, 1.6), rng.uniform(0.4, 1.6)};
            scene.obstacles.push_back(make_box_obstacle(he, rng.uniform_int(1, 4)));
        }
        roadmap = build_prm(scene, nodes, 6, 0.25, seed);
        components = build_components(roadmap, scene.robot, default_body_spheres(scene.robot), 0.25, 16);
    }
};

static bool same_reports(const UpdateReport& a, const UpdateReport& b) {
    return a.new_green == b.new_green && a.new_red == b.new_red && a.new_gray == b.new_gray &&
           a.unknown_after_heuristic == b.unknown_after_heuristic && a.residual_unknown == b.residual_unknown;
}

static void equivalence_after_every_move() {
    for (int trial = 0; trial < 6; ++trial) {
        Scenelet fx(40 + trial * 25, 1 + trial % 3, 700 + trial);
        Scene seq_scene = fx.scene, gpu_scene = fx.scene;
        SequentialEngine seq(fx.components, seq_scene, {});
        GpuEngine gpu(fx.components, gpu_scene, {});
        const bool lazy = trial % 2 == 0;
        Rng rng(9000 + trial);
        for (int move = 0; move < 30; ++move) {
            const ObstacleId o = rng.uniform_int(0, static_cast<int>(fx.scene.obstacles.size()) - 1);
            Transform pose = Transform::from_euler_xyz(rng.uniform(-3, 3), rng.uniform(-3, 3), rng.uniform(-3, 3));
            pose.t = {rng.uniform(-5, 5), rng.uniform(-5, 5), rng.uniform(-5, 5)};
            const UpdateReport rs = seq.update_obstacle(o, pose, lazy);
            const UpdateReport rg = gpu.update_obstacle(o, pose, lazy);
            EXPECT(seq.states() == gpu.states(), "trial %d move %d (%s): states differ", trial, move, lazy ? "lazy" : "eager");
            EXPECT(seq.obstacle_bits() == gpu.obstacle_bits(), "trial %d move %d: bits differ", trial, move);
            EXPECT(same_reports(rs, rg), "trial %d move %d: reports seq(%d,%d,%d,%d,%d) gpu(%d,%d,%d,%d,%d)", trial, move,
                   rs.new_green, rs.new_red, rs.new_gray, rs.unknown_after_heuristic, rs.residual_unknown, rg.new_green,
                   rg.new_red, rg.new_gray, rg.unknown_after_heuristic, rg.residual_unknown);
            EXPECT(gpu_scene.obstacles[o].active && gpu_scene.obstacles[o].pose.t == pose.t, "scene not mutated");
        }
    }
}

static void narrow_masks_match_sequential() {
    Scenelet fx(60, 3, 53);
    Scene seq_scene = fx.scene, gpu_scene = fx.scene;
    SequentialEngine seq(fx.components, seq_scene, {});
    GpuEngine gpu(fx.components, gpu_scene, {});
    Rng rng(99);
    std::vector<ComponentId> all;
    for (ComponentId c = 0; c < fx.components.count(); ++c) all.push_back(c);
    for (int move = 0; move < 20; ++move) {
        const ObstacleId o = move % 3;
        const Transform pose = Transform::translation({rng.uniform(-5, 5), rng.uniform(-5, 5), rng.uniform(-5, 5)});
        seq.update_obstacle(o, pose, true);
        gpu.update_obstacle(o, pose, true);
        std::vector<std::uint8_t> over, under;
        gpu.batch_over(all, o, over);
        gpu.batch_under(all, o, under);
        for (ComponentId c = 0; c < fx.components.count(); ++c) {
            EXPECT(static_cast<bool>(over[c]) == seq.narrow_over_test(o, c), "over mask c=%d move %d", c, move);
            EXPECT(static_cast<bool>(under[c]) == seq.narrow_under_test(o, c), "under mask c=%d move %d", c, move);
        }
    }
}

static void batch_update_matches_batch_engine() {
    Scenelet fx(80, 3, 61);
    Scene bat_scene = fx.scene, gpu_scene = fx.scene;
    BatchEngine bat(fx.components, bat_scene, {});
    GpuEngine gpu(fx.components, gpu_scene, {});
    Rng rng(61);
    for (int it = 0; it < 10; ++it) {
        std::vector<std::pair<ObstacleId, Transform>> moves;
        for (int i = 0; i < 7; ++i)
            moves.push_back({rng.uniform_int(0, 2),
                             Transform::translation({rng.uniform(-5, 5), rng.uniform(-5, 5), rng.uniform(-5, 5)})});
        const auto rb = bat.batch_update(moves, true);
        const auto rg = gpu.batch_update(moves, true);
        EXPECT(rb.size() == rg.size(), "report count");
        for (size_t i = 0; i < rb.size(); ++i) EXPECT(same_reports(rb[i], rg[i]), "iteration %d move %zu report", it, i);
        EXPECT(bat.states() == gpu.states(), "iteration %d states", it);
        EXPECT(bat.obstacle_bits() == gpu.obstacle_bits(), "iteration %d bits", it);
        EXPECT(bat.unknown_count() == gpu.unknown_count(), "iteration %d unknown count", it);
    }
    EXPECT(gpu.batch_update({}, true).empty(), "empty move list");
    // grid(): the reference's SpatialGrid over the same component AABBs
    const SpatialGrid& gb = bat.grid();
    const SpatialGrid& gg = gpu.grid();
    EXPECT(gb.cell_count() == gg.cell_count() && gb.capacity() == gg.capacity() &&
               gb.overflow_total() == gg.overflow_total(),
           "grid(): %d cells vs %d", gb.cell_count(), gg.cell_count());
    for (int q = 0; q < 20; ++q) {
        const Vec3 c{rng.uniform(-5, 5), rng.uniform(-5, 5), rng.uniform(-5, 5)};
        const double r = rng.uniform(0.2, 2.0);
        const Aabb box{{c.x - r, c.y - r, c.z - r}, {c.x + r, c.y + r, c.z + r}};
        std::vector<std::int32_t> cb, cg;
        gb.candidates(box, cb);
        gg.candidates(box, cg);
        EXPECT(cb == cg, "grid() candidates differ for query %d", q);
    }
    bool threw = false;
    try {
        gpu.update_obstacle(99, Transform::identity(), true);
    } catch (const std::invalid_argument& e) {
        threw = std::string(e.what()) == "unknown obstacle id";
    }
    EXPECT(threw, "unknown obstacle id must throw std::invalid_argument");
    // resolve_all_unknown leaves no gray, like the reference (engine_batch.cpp:217-227)
    const int nb = bat.resolve_all_unknown();
    const int ng = gpu.resolve_all_unknown();
    EXPECT(nb == ng, "resolve_all_unknown resolved %d vs %d", nb, ng);
    EXPECT(bat.states() == gpu.states(), "states after resolve_all_unknown");
    EXPECT(gpu.unknown_count() == 0, "gray left after resolve_all_unknown");
}

// Obstacles active in the Scene before the engine moves them (static walls): the reference's
// exact_component_valid checks every active obstacle (roadmap.cpp:135-139), so eager updates and
// resolve_all_unknown must see them at their scene poses until the engine first moves them.
static void scene_active_obstacles() {
    for (int trial = 0; trial < 4; ++trial) {
        Scenelet fx(70 + 20 * trial, 3, 810 + trial, 5.0);
        Rng rng(4200 + trial);
        Scene base = fx.scene;
        for (int o = 1; o < 3; ++o) {  // obstacles 1 and 2 start active at random poses
            Transform pose = Transform::from_euler_xyz(rng.uniform(-3, 3), rng.uniform(-3, 3), rng.uniform(-3, 3));
            pose.t = {rng.uniform(-3, 3), rng.uniform(-3, 3), rng.uniform(-3, 3)};
            base.obstacles[o].pose = pose;
            base.obstacles[o].active = true;
        }
        Scene bat_scene = base, gpu_scene = base;
        BatchEngine bat(fx.components, bat_scene, {});
        GpuEngine gpu(fx.components, gpu_scene, {});
        const bool lazy = trial % 2 == 1;
        for (int move = 0; move < 24; ++move) {
            // obstacle 0 moves throughout; obstacle 1 first moves at move 12; obstacle 2 never moves
            const ObstacleId o = move >= 12 && move % 3 == 0 ? 1 : 0;
            Transform pose = Transform::from_euler_xyz(rng.uniform(-3, 3), rng.uniform(-3, 3), rng.uniform(-3, 3));
            pose.t = {rng.uniform(-4, 4), rng.uniform(-4, 4), rng.uniform(-4, 4)};
            const UpdateReport rb = bat.update_obstacle(o, pose, lazy);
            const UpdateReport rg = gpu.update_obstacle(o, pose, lazy);
            EXPECT(same_reports(rb, rg) && rb.resolve_checks == rg.resolve_checks,
                   "scene-active trial %d move %d: reports bat(%d,%d,%d,%d,%d) gpu(%d,%d,%d,%d,%d)", trial, move,
                   rb.new_green, rb.new_red, rb.new_gray, rb.unknown_after_heuristic, rb.residual_unknown, rg.new_green,
                   rg.new_red, rg.new_gray, rg.unknown_after_heuristic, rg.residual_unknown);
            EXPECT(bat.states() == gpu.states(), "scene-active trial %d move %d: states", trial, move);
        }
        const int nb = bat.resolve_all_unknown(), ng = gpu.resolve_all_unknown();
        EXPECT(nb == ng, "scene-active trial %d: resolve_all_unknown %d vs %d", trial, nb, ng);
        EXPECT(bat.states() == gpu.states(), "scene-active trial %d: states after resolve_all_unknown", trial);
    }
}

static void scenario_replay(const std::string& path) {
    std::ifstream f(path);
    if (!f) {
        std::fprintf(stderr, "skip %s (absent)\n", path.c_str());
        return;
    }
    std::stringstream ss;
    ss << f.rdbuf();
    const Scenario s = parse_scenario_text(ss.str(), path);
    Scene build_scene{s.env, {}, s.robot};
    const Roadmap roadmap = build_prm(build_scene, s.nodes, s.k_neighbors, s.effective_epsilon(), s.roadmap_seed);
    const ComponentSet comps =
        build_components(roadmap, s.robot, default_body_spheres(s.robot), s.effective_epsilon(), s.max_segments);
    Scene seq_scene{s.env, s.make_obstacles(), s.robot}, gpu_scene{s.env, s.make_obstacles(), s.robot};
    SequentialEngine seq(comps, seq_scene, {});
    GpuEngine gpu(comps, gpu_scene, {});
    const bool lazy = s.mode == UpdateMode::Lazy;
    const auto moves = s.make_moves();
    const int per = static_cast<int>(s.obstacles.size());
    const int iterations = std::min(s.iterations, lazy ? s.iterations : 4);
    for (int it = 0; it < iterations; ++it) {
        for (int m = 0; m < per; ++m) {
            const auto& [o, pose] = moves[static_cast<size_t>(it) * per + m];
            const UpdateReport rs = seq.update_obstacle(o, pose, lazy);
            const UpdateReport rg = gpu.update_obstacle(o, pose, lazy);
            EXPECT(same_reports(rs, rg), "%s it %d move %d report", s.name.c_str(), it, m);
        }
        EXPECT(seq.states() == gpu.states(), "%s iteration %d states", s.name.c_str(), it + 1);
        EXPECT(seq.obstacle_bits() == gpu.obstacle_bits(), "%s iteration %d bits", s.name.c_str(), it + 1);
    }
    std::printf("scenario %s (%s): %d components, %d iterations compared\n", s.name.c_str(), lazy ? "lazy" : "eager",
                comps.count(), iterations);
}

// The semantic cases of proj/tests/test_sequential.cpp:83-184 on rgg::GpuEngine: one straight
// edge along x (nodes 0 and 1 at x = 0 and 4, the edge is component 2) and box obstacles.
struct Straight {
    Scene scene;
    Roadmap roadmap;
    ComponentSet components;
    explicit Straight(std::vector<ObstacleModel> obstacles) {
        scene.bounds = {{-10, -10, -10}, {10, 10, 10}};
        scene.robot = make_free_flying_box({0.5, 0.5, 0.5});
        scene.obstacles = std::move(obstacles);
        roadmap.nodes = {{0.0, 0, 0, 0, 0, 0}, {4.0, 0, 0, 0, 0, 0}};
        roadmap.edges = {{0, 1}};
        roadmap.rebuild_adjacency();
        components = build_components(roadmap, scene.robot, default_body_spheres(scene.robot), 0.25, 16);
    }
};

static void sequential_semantics() {
    {  // far obstacle changes nothing (:83-96), eager
        Straight fx({make_box_obstacle({1, 1, 1}, 1)});
        GpuEngine g(fx.components, fx.scene, {});
        const UpdateReport r = g.update_obstacle(0, Transform::translation({8, 8, 8}), false);
        EXPECT(r.new_green + r.new_red + r.new_gray == 0 && g.unknown_count() == 0, "far obstacle");
        bool all_valid = true;
        for (ValidityState v : g.states()) all_valid &= v == ValidityState::Valid;
        EXPECT(all_valid, "far obstacle leaves every label valid");
    }
    {  // an obstacle on a node's centre is red through the inner hit, lazily (:98-104)
        Straight fx({make_box_obstacle({1, 1, 1}, 1)});
        GpuEngine g(fx.components, fx.scene, {});
        g.update_obstacle(0, Transform::translation({0, 0, 0}), true);
        EXPECT(g.states()[0] == ValidityState::Invalid && g.states()[2] == ValidityState::Invalid, "inner hit");
    }
    for (bool lazy : {true, false}) {  // grazing overlap: gray when lazy, resolved red when eager (:106-126)
        Straight fx({make_box_obstacle({0.5, 0.5, 0.5}, 1)});
        GpuEngine g(fx.components, fx.scene, {});
        const Transform graze = Transform::translation({2.0, 0.99, 0});
        g.update_obstacle(0, graze, lazy);
        EXPECT(g.states()[2] == (lazy ? ValidityState::Unknown : ValidityState::Invalid), "graze lazy=%d", lazy);
    }
    {  // departure restores green; a second obstacle keeps gray; bits 0b11 -> 0b10 -> 0 (:128-149)
        Straight fx({make_box_obstacle({0.5, 0.5, 0.5}, 1), make_box_obstacle({0.5, 0.5, 0.5}, 1)});
        GpuEngine g(fx.components, fx.scene, {});
        g.update_obstacle(0, Transform::translation({2.0, 0, 0}), true);
        EXPECT(g.states()[2] == ValidityState::Invalid, "revalidation step 1");
        g.update_obstacle(1, Transform::translation({2.0, 0.99, 0}), true);
        EXPECT(g.states()[2] == ValidityState::Invalid && g.obstacle_bits()[2] == 0b11, "revalidation step 2");
        g.update_obstacle(0, Transform::translation({8, 8, 8}), true);
        EXPECT(g.states()[2] == ValidityState::Unknown && g.obstacle_bits()[2] == 0b10, "revalidation step 3");
        g.update_obstacle(1, Transform::translation({-8, 8, 8}), true);
        EXPECT(g.states()[2] == ValidityState::Valid && g.obstacle_bits()[2] == 0, "revalidation step 4");
    }
    {  // red restored when the remaining obstacle still under-hits (:151-162)
        Straight fx({make_box_obstacle({0.5, 0.5, 0.5}, 1), make_box_obstacle({0.5, 0.5, 0.5}, 1)});
        GpuEngine g(fx.components, fx.scene, {});
        g.update_obstacle(0, Transform::translation({1.0, 0, 0}), true);
        g.update_obstacle(1, Transform::translation({3.0, 0, 0}), true);
        EXPECT(g.states()[2] == ValidityState::Invalid, "red restored step 1");
        g.update_obstacle(0, Transform::translation({8, 8, 8}), true);
        EXPECT(g.states()[2] == ValidityState::Invalid && g.obstacle_bits()[2] == 0b10, "red restored step 2");
    }
    for (bool lazy : {true, false}) {  // idempotence: the same pose twice changes nothing (:164-184)
        Scene scene;
        scene.bounds = {{-6, -6, -6}, {6, 6, 6}};
        scene.robot = make_free_flying_box({0.5, 0.5, 0.5});
        scene.obstacles = {make_box_obstacle({1, 0.6, 0.6}, 2)};
        const Roadmap roadmap = build_prm(scene, 40, 6, 0.25, 11);
        const ComponentSet set = build_components(roadmap, scene.robot, default_body_spheres(scene.robot), 0.25, 16);
        GpuEngine g(set, scene, {});
        const Transform pose = Transform::translation({0.5, -0.3, 0.2});
        g.update_obstacle(0, pose, lazy);
        const auto states = g.states();
        const auto bits = g.obstacle_bits();
        g.update_obstacle(0, pose, lazy);
        EXPECT(g.states() == states && g.obstacle_bits() == bits, "idempotence lazy=%d", lazy);
    }
}

// proj/tests/test_batch.cpp:236-258: garbage in the layout's masked (padding) slots never
// changes a mask.  The GPU never stores padding; the host layout stays the reference's own.
static void padding_neutrality() {
    Scenelet fx(40, 1, 54);
    GpuEngine engine(fx.components, fx.scene, {});
    engine.update_obstacle(0, Transform::translation({0.5, 0.5, 0}), true);
    std::vector<ComponentId> all;
    for (ComponentId c = 0; c < fx.components.count(); ++c) all.push_back(c);
    std::vector<std::uint8_t> before, after;
    engine.batch_under(all, 0, before);
    BatchLayout& l = const_cast<BatchLayout&>(engine.layout());
    Rng rng(1);
    for (size_t slot = 0; slot < l.seg_mask.size(); ++slot) {
        if (l.seg_mask[slot]) continue;
        for (int j = 0; j < 6; ++j) l.e_minus[slot * 6 + j] = rng.uniform(-50, 50);
    }
    l.rebuild_segment_operands();
    engine.batch_under(all, 0, after);
    EXPECT(before == after, "padding neutrality");
}

static bool same_roadmap(const Roadmap& a, const Roadmap& b) {
    if (a.nodes.size() != b.nodes.size() || a.edges != b.edges || a.adjacency != b.adjacency) return false;
    for (size_t i = 0; i < a.nodes.size(); ++i)
        if (std::memcmp(a.nodes[i].data(), b.nodes[i].data(), a.nodes[i].size() * sizeof(double)) != 0 ||
            a.nodes[i].size() != b.nodes[i].size())
            return false;
    return true;
}

// rgg::gpu::build_prm against rgg::build_prm: the free-cube cases and the active-wall case of
// proj/tests/test_roadmap.cpp:34-73, the argument errors, and the scenarios' build scenes.
static void prm_matches_reference(const std::vector<std::string>& scns) {
    auto cube = [](double half) {
        Scene s;
        s.bounds = {{-half, -half, -half}, {half, half, half}};
        s.robot = make_free_flying_box({0.5, 0.5, 0.5});
        return s;
    };
    const struct {
        int n, k;
        std::uint64_t seed;
    } cases[] = {{10, 16, 42}, {1, 4, 7}, {60, 8, 1234}, {60, 8, 1235}, {2000, 12, 5}};
    for (const auto& c : cases) {
        const Scene sc = cube(10.0);
        EXPECT(same_roadmap(rgg::gpu::build_prm(sc, c.n, c.k, 0.25, c.seed), build_prm(sc, c.n, c.k, 0.25, c.seed)),
               "free cube n=%d k=%d", c.n, c.k);
    }
    {
        Scene sc = cube(3.0);
        ObstacleModel wall = make_box_obstacle({3.0, 3.0, 0.5}, 3);
        wall.pose = Transform::identity();
        wall.active = true;
        sc.obstacles.push_back(wall);
        const Roadmap g = rgg::gpu::build_prm(sc, 40, 6, 0.25, 99);
        EXPECT(same_roadmap(g, build_prm(sc, 40, 6, 0.25, 99)), "active wall");
        EXPECT(g.nodes.size() < 40, "the slab cuts out samples");
    }
    for (int bad = 0; bad < 2; ++bad) {
        bool threw = false;
        try {
            rgg::gpu::build_prm(cube(10.0), bad == 0 ? 0 : 10, bad == 0 ? 4 : 0, 0.25, 7);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        EXPECT(threw, "invalid_argument case %d", bad);
    }
    for (const std::string& path : scns) {
        std::ifstream f(path);
        if (!f) continue;
        std::stringstream ss;
        ss << f.rdbuf();
        const Scenario s = parse_scenario_text(ss.str(), path);
        const Scene build_scene{s.env, {}, s.robot};
        EXPECT(same_roadmap(rgg::gpu::build_prm(build_scene, s.nodes, s.k_neighbors, s.effective_epsilon(), s.roadmap_seed),
                            build_prm(build_scene, s.nodes, s.k_neighbors, s.effective_epsilon(), s.roadmap_seed)),
               "scenario %s", path.c_str());
        // the same robot among the scenario's obstacles, active at their first scripted poses:
        // node and edge checks through rgg_exact_valid_sets (incl. the serial-chain manipulator)
        Scene obst_scene{s.env, s.make_obstacles(), s.robot};
        const auto moves = s.make_moves();
        for (const auto& [o, pose] : moves)
            if (!obst_scene.obstacles[o].active) {
                obst_scene.obstacles[o].pose = pose;
                obst_scene.obstacles[o].active = true;
            }
        const int n = std::min(s.nodes, 600);
        const auto t0 = std::chrono::steady_clock::now();
        const Roadmap g = rgg::gpu::build_prm(obst_scene, n, s.k_neighbors, s.effective_epsilon(), s.roadmap_seed);
        const auto t1 = std::chrono::steady_clock::now();
        const Roadmap want = build_prm(obst_scene, n, s.k_neighbors, s.effective_epsilon(), s.roadmap_seed);
        const auto t2 = std::chrono::steady_clock::now();
        EXPECT(same_roadmap(g, want), "scenario %s with active obstacles", path.c_str());
        std::printf("prm %s with %zu active obstacles: %zu of %d nodes, %zu edges; gpu %.1f ms, reference %.1f ms\n",
                    s.name.c_str(), obst_scene.obstacles.size(), want.nodes.size(), n, want.edges.size(),
                    std::chrono::duration<double, std::milli>(t1 - t0).count(),
                    std::chrono::duration<double, std::milli>(t2 - t1).count());
    }
    for (int trial = 0; trial < 3; ++trial) {  // random active boxes in a small cube
        Scene sc = cube(4.0);
        Rng rng(77 + trial);
        for (int i = 0; i < 4; ++i) {
            ObstacleModel ob = make_box_obstacle({rng.uniform(0.3, 1.5), rng.uniform(0.3, 1.5), rng.uniform(0.3, 1.5)}, 2);
            ob.pose = Transform::from_euler_xyz(rng.uniform(-3, 3), rng.uniform(-3, 3), rng.uniform(-3, 3));
            ob.pose.t = {rng.uniform(-3, 3), rng.uniform(-3, 3), rng.uniform(-3, 3)};
            ob.active = true;
            sc.obstacles.push_back(ob);
        }
        const Roadmap g = rgg::gpu::build_prm(sc, 300, 8, 0.25, 500 + trial);
        const Roadmap want = build_prm(sc, 300, 8, 0.25, 500 + trial);
        EXPECT(same_roadmap(g, want), "random active boxes trial %d", trial);
        EXPECT(want.nodes.size() < 300, "trial %d: the boxes cut out samples", trial);
    }
}

int main(int argc, char** argv) {
    std::setvbuf(stdout, nullptr, _IONBF, 0);  // progress survives a crash
    const std::string dir = argc > 1 ? argv[1] : "";
    equivalence_after_every_move();
    narrow_masks_match_sequential();
    batch_update_matches_batch_engine();
    padding_neutrality();
    sequential_semantics();
    scene_active_obstacles();
    if (!dir.empty()) {
        scenario_replay(dir + "/quick_smoke.scn");
        scenario_replay(dir + "/table4_obstacles_1000_5x.scn");
        scenario_replay(dir + "/table5_manipulator_100.scn");
    }
    prm_matches_reference({dir + "/quick_smoke.scn", dir + "/table4_obstacles_1000_5x.scn",
                           dir + "/table5_manipulator_100.scn"});
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
