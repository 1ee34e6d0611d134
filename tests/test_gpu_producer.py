"""The producer's swept-volume box fit and spline simplification on the GPU
(csrc/swept_gpu.cu) against the host producer, which tests/test_producer.py pins bit for bit to
the reference's build_components + serialize."""
import numpy as np
import pytest

from paper_2603_28674_b200 import producer, synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,n,k,half,seed", [("se2", 2000, 20, 12.0, 5), ("3d", 800, 12, 5.0, 6)])
def test_gpu_box_fit_is_bit_identical(kind, n, k, half, seed):
    rm = synth.make_roadmap(kind, n, k, half, seed)
    host = producer.build_layout(rm.robot_he, rm.nodes, rm.edges, with_obbs=True, threads=8)
    for inner in (False, True):
        gpu = producer.build_layout(rm.robot_he, rm.nodes, rm.edges, with_obbs=True, threads=8, gpu_fit=True,
                                    gpu_inner=inner)
        assert host[:3] == gpu[:3]
        for key in ("edge_sat", "comp_aabb", "segs", "spline_r", "obb15", "row_off"):
            a, b = host[3][key], gpu[3][key]
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (key, inner)


def test_gpu_fit_is_the_default_and_keeps_the_poses():
    """With a GPU present the producer fits the boxes on it by default (gpu_fit=None);
    the exact resolve's forward-kinematics poses come out identical as well."""
    rm = synth.make_roadmap("se2", 600, 12, 8.0, 9)
    assert producer.gpu_available()
    host = producer.build_layout(rm.robot_he, rm.nodes, rm.edges, with_poses=True, gpu_fit=False, threads=4)
    dflt = producer.build_layout(rm.robot_he, rm.nodes, rm.edges, with_poses=True, threads=4)
    for key in ("edge_sat", "comp_aabb", "segs", "row_off", "pose_off", "poses"):
        assert np.array_equal(host[3][key].view(np.uint8), dflt[3][key].view(np.uint8)), key


def _manipulator():
    import os

    from conftest import GOLDEN
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    return ref.World.from_scn(open(os.path.join(GOLDEN, "scenarios", "table5_manipulator_100.scn")).read())


def test_gpu_box_fit_serial_chain_is_bit_identical():
    """One fit unit per (component, body): the manipulator's six boxes per component and a
    synthetic chain with a rotated body frame fit on the GPU as on the host."""
    from test_producer import _chain_case

    w = _manipulator()
    r = w.robot()
    nodes, edges = w.roadmap()
    cases = [(r, nodes, edges, r["eps"])]
    robot, n2, e2 = _chain_case(5, n=300, k=8)
    cases.append((robot, n2, e2, 0.05))
    for rb, nd, ed, eps in cases:
        host = producer.build_layout_robot(rb, nd, ed, eps, 16, threads=4, with_obbs=True, with_poses=True,
                                           gpu_fit=False)
        gpu = producer.build_layout_robot(rb, nd, ed, eps, 16, threads=4, with_obbs=True, with_poses=True,
                                          gpu_fit=True)
        assert host[:3] == gpu[:3]
        for key in ("edge_sat", "comp_aabb", "segs", "spline_r", "obb15", "row_off", "pose_off", "poses"):
            assert np.array_equal(host[3][key].view(np.uint8), gpu[3][key].view(np.uint8)), key


def test_manipulator_end_to_end_from_own_producer():
    """table5_manipulator_100 built by this repo's producer (GPU box fit, the chain's forward
    kinematics), then eager updates with the GPU exact resolve: every report and label equals
    the reference engine's on its own build."""
    from oracle import ref
    from paper_2603_28674_b200 import engine as E

    w = _manipulator()
    r = w.robot()
    nodes, edges = w.roadmap()
    N, B, S, a = producer.build_layout_robot(r, nodes, edges, r["eps"], r["max_segments"], threads=4,
                                             with_poses=True)
    L = w.layout()
    lv = E.LayoutView(N=N, B=B, S=S, M=L.M, C=L.C, edge_sat=a["edge_sat"], comp_aabb=a["comp_aabb"],
                      row_off=a["row_off"], segs=a["segs"], spline_r=a["spline_r"], obst_he=L.obst_he,
                      obst_sph_local=L.obst_sph_local, obst_sph_r=L.obst_sph_r, obst_sph_n=L.obst_sph_n)
    eng = E.GpuEngine(lv)
    eng.set_resolver(a["pose_off"], a["poses"], r["he"])
    re = ref.Engine(w, kind=0)
    ids, rts = w.moves()
    checks = 0
    for i in range(len(ids)):
        exp = re.update(ids[i], rts[i], lazy=False)
        rep = eng.update_obstacle(int(ids[i]), rts[i], lazy=False)
        got = [rep.new_green, rep.new_red, rep.new_gray, rep.residual_unknown, rep.resolve_checks]
        assert got == [int(exp[1]), int(exp[2]), int(exp[3]), int(exp[9]), int(exp[10])], i
        assert np.array_equal(eng.states(), re.states()), i
        checks += rep.resolve_checks
    assert checks > 0


@pytest.mark.parametrize("scn", ["table4_obstacles_1000_5x", "table5_manipulator_100"])
def test_engine_from_roadmap_file_matches_reference(scn, tmp_path):
    """A roadmap file saved by the reference (save_roadmap) straight to the GPU engine:
    rgg_roadmap_load -> rgg_gpu_create_from_components, the scenario's obstacles, its moves
    (lazy) and the exact resolve from the file's poses; labels, bits and resolve_all_unknown
    equal the reference engine's."""
    import os

    from conftest import GOLDEN
    from oracle import ref
    from paper_2603_28674_b200 import engine as E

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    w = ref.World.from_scn(open(os.path.join(GOLDEN, "scenarios", scn + ".scn")).read())
    path = tmp_path / "r.rgg"
    w.save(str(path))
    rf = producer.load_roadmap(path, with_poses=True)
    L = w.layout()
    obs = synth.Obstacles(he=np.asarray(L.obst_he).reshape(-1, 3), spheres=np.asarray(L.obst_sph_n, np.int32))
    view = producer.component_view(rf, obs)
    eng = E.GpuEngine(view, components=True, allow_wide=True)
    eng.set_resolver(rf["pose_off"], rf["poses"], rf["robot"]["he"])
    re = ref.Engine(w, kind=0)
    ids, rts = w.moves()
    for i in range(len(ids)):
        re.update(ids[i], rts[i], lazy=True)
    eng.batch_update((ids, rts))
    assert np.array_equal(eng.states(), re.states())
    assert np.array_equal(eng.obstacle_bits().reshape(-1), re.bits().reshape(-1))
    assert eng.resolve_all_unknown() == re.resolve_all_unknown()
    assert np.array_equal(eng.states(), re.states())


def test_gpu_fit_saves_the_reference_roadmap_file(tmp_path):
    """The producer with the GPU box fit writes the reference's save_roadmap file byte for byte."""
    w = _manipulator()
    r = w.robot()
    nodes, edges = w.roadmap()
    ours, theirs = tmp_path / "ours.rgg", tmp_path / "ref.rgg"
    producer.build_layout_robot(r, nodes, edges, r["eps"], r["max_segments"], threads=4, gpu_fit=True,
                                save_roadmap=ours)
    w.save(str(theirs))
    assert ours.read_bytes() == theirs.read_bytes()
