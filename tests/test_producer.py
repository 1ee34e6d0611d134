"""The host producer (csrc/producer.cpp) against the reference's own preprocessing:
build_components (proj/src/roadmap.cpp:104-127) + BatchLayout::serialize
(proj/src/batch_layout.cpp:21-146), bit for bit, on seeded SE(2) and 3-D roadmaps."""
import numpy as np
import pytest

from oracle import ref
from paper_2603_28674_b200 import producer, synth


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("kind,n,k,half,seed", [("se2", 300, 12, 6.0, 5), ("3d", 200, 10, 4.0, 6)])
def test_producer_matches_reference_preprocessing(kind, n, k, half, seed):
    rm = synth.make_roadmap(kind, n, k, half, seed)
    N, B, S, a = producer.build_layout(rm.robot_he, rm.nodes, rm.edges, with_obbs=True, threads=4)
    w = ref.World.from_roadmap(rm.robot_he, rm.env, rm.nodes, rm.edges)
    L = w.layout()
    assert (N, B, S) == (L.N, L.B, L.S)
    for key in ("edge_sat", "comp_aabb", "segs", "spline_r"):
        assert np.array_equal(a[key].view(np.uint64), getattr(L, key).view(np.uint64)), key
    assert np.array_equal(a["row_off"], L.row_off)
    assert np.array_equal(a["obb15"], w.obbs())


def test_obstacle_spheres_rule():
    """obstacle_inner_spheres (proj/src/swept.cpp:23-49): radius = min half extent,
    centres spread along the longest axis, inside the box."""
    cen, r = producer.obstacle_spheres([5.0, 1.0, 1.0], 5)
    assert r == 1.0
    assert np.allclose(cen[:, 0], [-4, -2, 0, 2, 4]) and np.all(cen[:, 1:] == 0)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("kind,n,k,half,seed", [("se2", 200, 10, 6.0, 8), ("3d", 120, 8, 4.0, 9)])
def test_producer_poses_match_reference_fk(kind, n, k, half, seed):
    """The exact resolve's inputs: forward_kinematics (proj/src/robot.cpp:66-84) of
    every configuration of discretize_edge (:39-64), bit for bit."""
    rm = synth.make_roadmap(kind, n, k, half, seed)
    N, B, S, a = producer.build_layout(rm.robot_he, rm.nodes, rm.edges, threads=4, with_poses=True)
    w = ref.World.from_roadmap(rm.robot_he, rm.env, rm.nodes, rm.edges)
    off, poses = w.poses()
    assert np.array_equal(a["pose_off"], off)
    assert np.array_equal(a["poses"].view(np.uint64), poses.view(np.uint64))
    assert np.array_equal(w.body_half_extents(), np.asarray(rm.robot_he).reshape(1, 3))


def _chain_case(seed, n=60, k=5):
    """A 4-link chain with a rotated body frame, over uniform joint angles."""
    from paper_2603_28674_b200 import synth

    links = [[0, 0, 1, 0, 0, 0, 0.4, 0.12, 0.1, 0.4, 0, 0],
             [0, 1, 0, 0.8, 0, 0, 0.35, 0.1, 0.1, 0.35, 0, 0],
             [1, 1, 0, 0.7, 0, 0.1, 0.3, 0.09, 0.12, 0.3, 0, 0],
             [0, 0, 1, 0.6, 0, 0, 0.2, 0.1, 0.1, 0.2, 0, 0.05]]
    robot = producer.serial_chain(links)
    c, s = np.cos(0.3), np.sin(0.3)
    robot["local"][2, :9] = [c, -s, 0, s, c, 0, 0, 0, 1]  # a rotated body frame (robot.hpp BoxBody::local)
    rng = np.random.default_rng(seed)
    nodes = rng.uniform(-np.pi, np.pi, (n, 4))
    return robot, nodes, synth.knn_edges(nodes, k)


def _compare(a, L, w):
    for key in ("edge_sat", "comp_aabb", "segs", "spline_r"):
        assert np.array_equal(a[key].view(np.uint64), getattr(L, key).view(np.uint64)), key
    assert np.array_equal(a["row_off"], L.row_off)
    assert np.array_equal(a["obb15"], w.obbs())
    off, poses = w.poses()
    assert np.array_equal(a["pose_off"], off)
    assert np.array_equal(a["poses"].view(np.uint64), poses.view(np.uint64))


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_serial_chain_producer_matches_reference_manipulator():
    """table5_manipulator_100's six-link chain (its own PRM roadmap, eps 0.02): every
    SatBox, AABB, real segment, slot radius, fitted OBB and forward-kinematics pose equals
    the reference's build_components + serialize (robot.cpp:66-84 serial branch,
    swept.cpp:100-228, center_lipschitz's chain bound, batch_layout.cpp:21-146 with B = 6)."""
    import os

    from conftest import GOLDEN

    w = ref.World.from_scn(open(os.path.join(GOLDEN, "scenarios", "table5_manipulator_100.scn")).read())
    r = w.robot()
    nodes, edges = w.roadmap()
    N, B, S, a = producer.build_layout_robot(r, nodes, edges, r["eps"], r["max_segments"], threads=4,
                                             with_obbs=True, with_poses=True, gpu_fit=False)
    L = w.layout()
    assert (N, B, S) == (L.N, L.B, L.S) and B == 6
    _compare(a, L, w)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed,eps", [(3, 0.05), (4, 0.11)])
def test_serial_chain_producer_matches_reference_random(seed, eps):
    """A synthetic 4-link chain (a tilted joint axis, a rotated body frame, a body offset
    along z) over random joint angles: the layout equals the reference's."""
    robot, nodes, edges = _chain_case(seed)
    env = np.array([-4, -4, -4, 4, 4, 4.0])
    w = ref.World.from_robot(robot, env, nodes, edges, eps)
    N, B, S, a = producer.build_layout_robot(robot, nodes, edges, eps, 16, threads=3, with_obbs=True,
                                             with_poses=True, gpu_fit=False)
    L = w.layout()
    assert (N, B, S) == (L.N, L.B, L.S)
    _compare(a, L, w)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_free_flying_multibody_matches_reference():
    """A free-flying robot of two bodies (robot.cpp:71-74: every body rides the world frame
    through its own local frame)."""
    from paper_2603_28674_b200 import synth

    loc = np.zeros((2, 12))
    loc[:, [0, 4, 8]] = 1.0
    loc[1, 9:] = [0.9, 0.0, 0.2]
    robot = dict(kinematics=producer.FREE_FLYING, he=np.array([[0.5, 0.2, 0.2], [0.3, 0.3, 0.1]]), local=loc)
    rm = synth.make_roadmap("3d", 80, 6, 4.0, 12)
    w = ref.World.from_robot(robot, rm.env, rm.nodes, rm.edges, 0.25)
    N, B, S, a = producer.build_layout_robot(robot, rm.nodes, rm.edges, 0.25, 16, threads=2, with_obbs=True,
                                             with_poses=True, gpu_fit=False)
    assert B == 2
    _compare(a, w.layout(), w)


def test_robot_validation_errors():
    """RobotModel::validate's errors (robot.cpp:17-37) surface as the producer's."""
    nodes = np.zeros((2, 2))
    edges = np.array([[0, 1]])
    bad_axis = producer.serial_chain([[0, 0, 0, 0, 0, 0, 0.3, 0.1, 0.1, 0, 0, 0]] * 2)
    with pytest.raises(RuntimeError, match="joint axis/offset invalid"):
        producer.build_layout_robot(bad_axis, nodes, edges, 0.1, gpu_fit=False)
    bad_he = producer.serial_chain([[0, 0, 1, 0, 0, 0, 0.0, 0.1, 0.1, 0, 0, 0]] * 2)
    with pytest.raises(RuntimeError, match="half extents must be positive"):
        producer.build_layout_robot(bad_he, nodes, edges, 0.1, gpu_fit=False)
    skew = producer.serial_chain([[0, 0, 1, 0, 0, 0, 0.3, 0.1, 0.1, 0, 0, 0]] * 2)
    skew["local"][0, 1] = 0.5
    with pytest.raises(RuntimeError, match="local frame invalid"):
        producer.build_layout_robot(skew, nodes, edges, 0.1, gpu_fit=False)


def _saved(w, tmp_path, name="r.rgg"):
    path = tmp_path / name
    w.save(str(path))
    return path


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("scn", ["quick_smoke", "table5_manipulator_100"])
def test_roadmap_file_loads_into_the_component_view(scn, tmp_path):
    """rgg_roadmap_load reads the reference's own save_roadmap file (roadmap_io.cpp:150-203) into the
    component view: the OBB corners, CSR rows, real segment points and slot radii equal the
    reference's BatchLayout::serialize of the same components (e_plus, row_off, seg_pts, spline_r),
    and the resolver poses equal forward_kinematics over the rebuilt discretization."""
    import os

    from conftest import GOLDEN

    w = ref.World.from_scn(open(os.path.join(GOLDEN, "scenarios", scn + ".scn")).read())
    rf = producer.load_roadmap(_saved(w, tmp_path), with_poses=True)
    L = w.layout()
    assert (rf["N"], rf["B"], rf["S"]) == (L.N, L.B, L.S)
    for key in ("e_plus", "seg_pts", "spline_r"):
        assert np.array_equal(rf[key].view(np.uint64), getattr(L, key).view(np.uint64)), key
    assert np.array_equal(rf["row_off"], L.row_off)
    nodes, edges = w.roadmap()
    assert np.array_equal(rf["nodes"], nodes) and np.array_equal(rf["edges"], edges)
    off, poses = w.poses()
    assert np.array_equal(rf["pose_off"], off)
    assert np.array_equal(rf["poses"].view(np.uint64), poses.view(np.uint64))
    r = w.robot()
    assert rf["robot"]["kinematics"] == r["kinematics"] and np.array_equal(rf["robot"]["he"], r["he"])


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_roadmap_file_errors(tmp_path):
    """load_roadmap's error kinds (roadmap_io.hpp:10-16, checked in its order: size, magic, CRC,
    version), and a file is verified before anything is built."""
    import os
    import struct
    import zlib

    from conftest import GOLDEN

    w = ref.World.from_scn(open(os.path.join(GOLDEN, "scenarios", "quick_smoke.scn")).read())
    raw = _saved(w, tmp_path).read_bytes()

    def kind(data):
        p = tmp_path / "bad.rgg"
        p.write_bytes(data)
        with pytest.raises(producer.RoadmapFileError) as e:
            producer.load_roadmap(p)
        return e.value.kind

    assert kind(b"XXXXXXXX" + raw[8:]) == "bad_magic"
    assert kind(raw[:9]) == "truncated"
    assert kind(raw[:200] + bytes([raw[200] ^ 1]) + raw[201:]) == "checksum"
    body = raw[:8] + struct.pack("<I", 2) + raw[12:-4]
    assert kind(body + struct.pack("<I", zlib.crc32(body))) == "bad_version"
    cut = raw[:-40]  # a consistent checksum over a truncated body
    assert kind(cut + struct.pack("<I", zlib.crc32(cut))) == "truncated"


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_producer_saves_the_reference_roadmap_file(tmp_path):
    """rgg_built_save_roadmap writes save_roadmap's format (roadmap_io.cpp:150-203): for the
    manipulator's chain and a free-flying 3-D roadmap the file equals the reference's own,
    byte for byte (so its load_roadmap reads it), and rgg_roadmap_load reads it back."""
    import os

    from conftest import GOLDEN
    from paper_2603_28674_b200 import synth

    w = ref.World.from_scn(open(os.path.join(GOLDEN, "scenarios", "table5_manipulator_100.scn")).read())
    r = w.robot()
    nodes, edges = w.roadmap()
    ours = tmp_path / "ours.rgg"
    producer.build_layout_robot(r, nodes, edges, r["eps"], r["max_segments"], threads=4, gpu_fit=False,
                                save_roadmap=ours)
    assert ours.read_bytes() == _saved(w, tmp_path, "ref.rgg").read_bytes()
    rm = synth.make_roadmap("3d", 60, 6, 4.0, 5)
    w2 = ref.World.from_roadmap(rm.robot_he, rm.env, rm.nodes, rm.edges)
    producer.build_layout_robot(producer.free_flying(rm.robot_he), rm.nodes, rm.edges, 0.25, 16, threads=2,
                                gpu_fit=False, save_roadmap=ours)
    assert ours.read_bytes() == _saved(w2, tmp_path, "ref2.rgg").read_bytes()
    rf = producer.load_roadmap(ours)
    assert rf["N"] == len(rm.nodes) + len(rm.edges)
