"""GPU exact resolve against the live reference.

exact_component_valid (proj/src/roadmap.cpp:129-163) is restated on the GPU in
paper_2603_28674_b200/csrc/rgg_resolve.cu.  These tests drive the reference's own
engines from oracle/_ref (built from /root/reference by oracle/Makefile; the
prebuilt library travels to the GPU box) and require bit-identical verdicts:
  * per-component exact checks after lazy moves    roadmap.cpp:129-163
  * eager updates, labels + reports after every move  engine_batch.cpp:190-203
  * resolve_all_unknown after a lazy script       engine_batch.cpp:217-227
on the bundled scenarios, including the 6-body serial-chain manipulator.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SCN = ["quick_smoke", "table4_obstacles_1000_5x", "table5_manipulator_100"]


@pytest.fixture(scope="module")
def mods():
    import sys

    sys.path.insert(0, os.path.dirname(HERE))
    from oracle import ref
    from paper_2603_28674_b200 import engine

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    engine.library()
    return ref, engine


def _world(ref, name):
    return ref.World.from_scn(open(os.path.join(HERE, "golden", "scenarios", name + ".scn")).read())


def _gpu(engine, w):
    from paper_2603_28674_b200.engine import LayoutView

    eng = engine.GpuEngine(LayoutView.from_any(w.layout()))
    off, poses = w.poses()
    eng.set_resolver(off, poses, w.body_half_extents())
    return eng


@pytest.mark.parametrize("name", SCN)
def test_exact_check_matches_reference(mods, name):
    ref, engine = mods
    w = _world(ref, name)
    ids, rts = w.moves()
    n = min(len(ids), 40)
    re = ref.Engine(w, kind=0)
    eng = _gpu(engine, w)
    N = w.counts()["N"]
    allc = np.arange(N, dtype=np.int32)
    rng = np.random.default_rng(7)
    checked = 0
    for i in range(n):
        re.update(ids[i], rts[i], lazy=True)
        eng.update_obstacle(int(ids[i]), rts[i])
        if i % 8 == 7 or i == n - 1:
            sample = allc if N <= 2000 else np.sort(rng.choice(allc, 2000, replace=False)).astype(np.int32)
            exp = np.where(re.exact_free(sample) == 1, 0, 1).astype(np.uint8)
            got = eng.exact_check(sample)
            assert np.array_equal(got, exp), f"{name}: {np.sum(got != exp)} verdicts differ after move {i}"
            checked += len(sample)
            assert 0 < int(np.sum(exp == 1)) or i < 4
    assert checked > 0


@pytest.mark.parametrize("name", SCN)
def test_eager_updates_match_reference(mods, name):
    ref, engine = mods
    w = _world(ref, name)
    ids, rts = w.moves()
    n = min(len(ids), 30)
    re = ref.Engine(w, kind=0)
    eng = _gpu(engine, w)
    checks = 0
    for i in range(n):
        exp = re.update(ids[i], rts[i], lazy=False)
        rep = eng.update_obstacle(int(ids[i]), rts[i], lazy=False)
        got = [rep.new_green, rep.new_red, rep.new_gray, rep.unknown_after_heuristic, rep.residual_unknown,
               rep.resolve_checks]
        want = [int(exp[1]), int(exp[2]), int(exp[3]), int(exp[8]), int(exp[9]), int(exp[10])]
        assert got == want, f"{name} move {i}: report {got} != {want}"
        assert np.array_equal(eng.states(), re.states()), f"{name}: labels differ after eager move {i}"
        checks += rep.resolve_checks
    assert eng.unknown_count() == int(np.sum(re.states() == 2))
    assert checks > 0, "the script never exercised the resolve"


@pytest.mark.parametrize("name", SCN)
def test_resolve_all_unknown_matches_reference(mods, name):
    ref, engine = mods
    w = _world(ref, name)
    ids, rts = w.moves()
    n = min(len(ids), 50)
    re = ref.Engine(w, kind=0)
    eng = _gpu(engine, w)
    for i in range(n):
        re.update(ids[i], rts[i], lazy=True)
    eng.batch_update((ids[:n], rts[:n]))
    assert np.array_equal(eng.states(), re.states())
    gray = int(np.sum(re.states() == 2))
    assert gray > 0
    assert eng.resolve_all_unknown() == re.resolve_all_unknown() == gray
    assert np.array_equal(eng.states(), re.states())
    assert eng.unknown_count() == 0
    # the engine keeps going after a resolve: more lazy moves stay in lock-step
    for i in range(n, min(len(ids), n + 10)):
        re.update(ids[i], rts[i], lazy=True)
    eng.batch_update((ids[n:n + 10], rts[n:n + 10]))
    assert np.array_equal(eng.states(), re.states())


def test_resolver_shape_errors(mods):
    ref, engine = mods
    w = _world(ref, "quick_smoke")
    from paper_2603_28674_b200.engine import LayoutView

    eng = engine.GpuEngine(LayoutView.from_any(w.layout()))
    off, poses = w.poses()
    with pytest.raises(ValueError, match="component count"):
        eng.set_resolver(off[:-1], poses, w.body_half_extents())
    with pytest.raises(ValueError, match="set_resolver"):
        eng.update_obstacle(0, np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0.0]), lazy=False)
    with pytest.raises(ValueError, match="set_resolver"):
        eng.resolve_all_unknown()


def test_box_pairs_kat_through_engine(mods):
    """The 1200 golden box pairs (tests/golden/kat_boxes.npz, reference verdicts) through
    rgg_gpu_exact_check: component c has one configuration posed at box a_c, obstacle c
    sits at box b_c; pairs are 50 units apart, so the AABB gate isolates each pair."""
    from conftest import load_golden
    from paper_2603_28674_b200.engine import LayoutView

    ref, engine = mods
    g = load_golden("kat_boxes")
    n = len(g["out"])
    far = np.tile([1e6, 1e6, 1e6, 1e6 + 1, 1e6 + 1, 1e6 + 1], (n, 1)).astype(np.float64)
    lv = LayoutView(N=n, B=1, S=1, M=n, C=1, edge_sat=np.zeros((n, 21)), comp_aabb=far,
                    row_off=np.zeros(n + 1, np.int32), segs=np.zeros((0, 7)), spline_r=np.zeros(1),
                    obst_he=np.ascontiguousarray(g["he_b"]), obst_sph_local=np.zeros((n, 1, 3)),
                    obst_sph_r=np.zeros(n), obst_sph_n=np.ones(n, np.int32))
    eng = engine.GpuEngine(lv, allow_wide=True)
    assert np.all(g["he_a"] == g["he_a"][0])  # box a is the robot body: one half-extent triple
    eng.set_resolver(np.arange(n + 1, dtype=np.int64), g["rt_a"].reshape(n, 1, 12), g["he_a"][:1])
    for lo in range(0, n, 256):
        eng.batch_update((np.arange(lo, min(n, lo + 256), dtype=np.int32), g["rt_b"][lo:lo + 256]), per_move=False)
    got = eng.exact_check(np.arange(n, dtype=np.int32))
    assert np.array_equal(got, g["out"]), f"{int(np.sum(got != g['out']))} of {n} pair verdicts differ"


def test_scene_active_obstacles(mods):
    """Obstacles active in the Scene before the engine moves them (rgg_gpu_set_active_obstacles):
    exact_component_valid checks every active obstacle at its pose (roadmap.cpp:135-139); an
    obstacle's own move supersedes its listed pose.  Checked against the C oracle's ro_exact_valid."""
    from oracle import oracle as O

    ref, engine = mods
    w = _world(ref, "quick_smoke")
    ids, rts = w.moves()
    lay = w.layout()
    ohe = np.asarray(lay.obst_he, np.float64).reshape(-1, 3)
    M = ohe.shape[0]
    assert M >= 2
    eng = _gpu(engine, w)
    off, poses = w.poses()
    he = np.asarray(w.body_half_extents(), np.float64).reshape(-1)
    B = len(he) // 3
    poses = np.asarray(poses, np.float64).reshape(-1, B, 12)
    N = w.counts()["N"]
    rng = np.random.default_rng(11)
    sample = np.sort(rng.choice(N, min(N, 400), replace=False)).astype(np.int32)

    def expect(active, obst_rt):
        return np.array([0 if O.exact_valid(poses[off[c]:off[c + 1]], he, active, obst_rt, ohe) else 1
                         for c in sample], np.uint8)

    # two obstacles active at the poses of the script's first moves for them, none moved yet
    pick = [int(np.flatnonzero(ids == o)[0]) for o in (0, 1)]
    obst_rt = np.zeros((M, 12))
    active = np.zeros(M, np.uint8)
    for o, i in zip((0, 1), pick):
        obst_rt[o], active[o] = rts[i], 1
    eng.set_active_obstacles([0, 1], obst_rt[[0, 1]])
    exp = expect(active, obst_rt)
    assert 0 < int(exp.sum()) < len(sample), "the sample should straddle the scene obstacles"
    assert np.array_equal(eng.exact_check(sample), exp)
    # obstacle 0 moves: its engine pose wins over the listed one; obstacle 1 stays at its scene pose
    j = int(np.flatnonzero(ids == 0)[1])
    eng.update_obstacle(0, rts[j])
    obst_rt[0] = rts[j]
    assert np.array_equal(eng.exact_check(sample), expect(active, obst_rt))
    # an empty list leaves only the moved obstacle
    eng.set_active_obstacles([], np.zeros((0, 12)))
    active[1] = 0
    assert np.array_equal(eng.exact_check(sample), expect(active, obst_rt))
    with pytest.raises(ValueError, match="unknown obstacle id"):
        eng.set_active_obstacles([M], np.zeros((1, 12)))


@pytest.mark.parametrize("name", ["quick_smoke", "table5_manipulator_100"])
def test_exact_valid_sets_stateless(mods, name):
    """rgg_exact_valid_sets (build_prm's node/edge checks, roadmap.cpp:69, :95-99) against the
    C oracle's ro_exact_valid, with every obstacle active at its first scripted pose."""
    import ctypes as C

    from oracle import oracle as O

    ref, engine = mods
    w = _world(ref, name)
    ids, rts = w.moves()
    ohe = np.ascontiguousarray(np.asarray(w.layout().obst_he, np.float64).reshape(-1, 3))
    M = ohe.shape[0]
    ort = np.zeros((M, 12))
    for o in range(M):
        ort[o] = rts[int(np.flatnonzero(ids == o)[0])]
    off, poses = w.poses()
    he = np.ascontiguousarray(np.asarray(w.body_half_extents(), np.float64).reshape(-1))
    B = len(he) // 3
    poses = np.ascontiguousarray(np.asarray(poses, np.float64).reshape(-1, B, 12))
    off = np.ascontiguousarray(off, np.int64)
    n = min(len(off) - 1, 500)
    got = np.zeros(n, np.uint8)
    L = engine.library()
    rc = L.rgg_exact_valid_sets(0, n, off.ctypes.data, B, he.ctypes.data, poses.ctypes.data, M, ohe.ctypes.data,
                                ort.ctypes.data, got.ctypes.data)
    assert rc == 0
    exp = np.array([1 if O.exact_valid(poses[off[c]:off[c + 1]], he, np.ones(M, np.uint8), ort, ohe) else 0
                    for c in range(n)], np.uint8)
    assert 0 < int(exp.sum()) < n
    assert np.array_equal(got, exp)
    # no obstacles: every set is free; bad offsets: EINVAL
    rc = L.rgg_exact_valid_sets(0, n, off.ctypes.data, B, he.ctypes.data, poses.ctypes.data, 0, None, None,
                                got.ctypes.data)
    assert rc == 0 and got.all()
    bad = off.copy()
    bad[0] = 1
    assert L.rgg_exact_valid_sets(0, n, bad.ctypes.data, B, he.ctypes.data, poses.ctypes.data, M, ohe.ctypes.data,
                                  ort.ctypes.data, got.ctypes.data) != 0
