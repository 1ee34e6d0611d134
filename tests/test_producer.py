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
