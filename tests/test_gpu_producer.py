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
