"""The plain-C oracle (oracle/rgg_oracle.c) against the reference's golden vectors.

This pins the oracle ("parity pinned"): every fixture under tests/golden was
produced by the unmodified reference (oracle/gen_golden.py)."""
import numpy as np
import pytest

from conftest import SCENARIOS, load_golden
from oracle import oracle


class _L:
    def __init__(self, g):
        for k, v in g.items():
            setattr(self, k, v)


def test_kat_sat_bytes():
    g = load_golden("kat_sat")
    out = oracle.sat_batch(g["boxes"], g["idx"], g["obstacle"])
    assert np.array_equal(out, g["out"])
    assert 0 < out.sum() < len(out)  # both labels occur (test_kernels.cpp:81-85)


def test_kat_seg_bytes():
    g = load_golden("kat_seg")
    out = oracle.seg_sphere_batch(g["segs"], g["idx"], g["center"], float(g["r_total"]))
    assert np.array_equal(out, g["out"])


def test_kat_pairs():
    g = load_golden("kat_pairs")
    out = np.array([oracle.sat_boxes(a, b) for a, b in zip(g["a"], g["b"])], np.uint8)
    assert np.array_equal(out, g["out"])


def test_kat_obstacle_operands_bitwise():
    g = load_golden("kat_obstacle")
    C = g["obst_sph_local"].shape[1]
    for i in range(len(g["o"])):
        o = int(g["o"][i])
        n = int(g["obst_sph_n"][o])
        sat, aabb, cen, saabb = oracle.obstacle_operands(g["obst_he"][o], g["obst_sph_local"][o][:n], n,
                                                         g["obst_sph_r"][o], g["rt"][i])
        assert np.array_equal(sat.view(np.uint64), g["sat"][i].view(np.uint64))
        assert np.array_equal(aabb, g["aabb"][i])
        assert np.array_equal(cen, g["centres"][i][:n])
        assert np.array_equal(saabb, g["saabb"][i])
        assert C >= n


def test_sat_prep_and_seg_prep_bitwise():
    g = load_golden("scn_quick_smoke")
    for row, sat in zip(g["e_plus"], g["edge_sat"]):
        assert np.array_equal(oracle.sat_prep(row).view(np.uint64), sat.view(np.uint64))
    for pts, seg in zip(g["seg_pts"], g["segs"]):
        assert np.array_equal(oracle.seg_prep(pts).view(np.uint64), seg.view(np.uint64))


@pytest.mark.parametrize("name", SCENARIOS)
def test_engine_replay_matches_reference(name):
    g = load_golden(name)
    eng = oracle.Engine(_L(g))
    snaps = {int(i): k for k, i in enumerate(g["snap_at"])}
    grouped = int(g["groups"]) > 1
    for i, (o, rt) in enumerate(zip(g["ids"], g["rts"])):
        rep = eng.update(o, rt)
        if not grouped:
            # new_green, new_red, new_gray, unknown_after_heuristic
            assert rep.tolist() == g["reports"][i][:4].tolist(), f"report mismatch at move {i}"
        if i in snaps:
            k = snaps[i]
            assert np.array_equal(eng.states(), g["snap_states"][k]), f"states differ after move {i}"
            bits = eng.bits()
            assert np.array_equal(bits, g["snap_bits"][k].reshape(bits.shape)), f"bits differ after move {i}"
    st, bits = eng.pure()
    assert np.array_equal(st, eng.states()), "lazy labels are not the pure function"
    assert np.array_equal(bits, eng.bits())
    allc = np.arange(int(g["N"]), dtype=np.int32)
    o = int(g["mask_obstacle"])
    assert np.array_equal(eng.mask(0, allc, o), g["masks"][0])
    assert np.array_equal(eng.mask(1, allc, o), g["masks"][1])


def test_box_intersect_kat():
    """polytopes_intersect (geometry.cpp:228-303): 1200 near-contact box pairs dumped
    from the reference (oracle/gen_golden.py kat_boxes), restated literally in C."""
    g = load_golden("kat_boxes")
    got = np.array([oracle.box_intersect(a, ha, b, hb) for a, ha, b, hb in
                    zip(g["rt_a"], g["he_a"], g["rt_b"], g["he_b"])], np.uint8)
    assert np.array_equal(got, g["out"])
    assert 0.3 < g["out"].mean() < 0.7


def test_exact_valid_gates_inactive_and_far_obstacles():
    """exact_component_valid (roadmap.cpp:129-163): inactive obstacles never count,
    no active obstacle -> free, one intersecting (config, body, obstacle) -> invalid."""
    g = load_golden("kat_boxes")
    i = int(np.argmax(g["out"]))  # an intersecting pair
    poses = g["rt_a"][i].reshape(1, 1, 12)
    far = g["rt_b"][i].copy()
    far[9:] += 1000.0
    obst_rt = np.stack([far, g["rt_b"][i]])
    obst_he = np.stack([g["he_b"][i], g["he_b"][i]])
    assert oracle.exact_valid(poses, g["he_a"][i], [1, 0], obst_rt, obst_he)
    assert not oracle.exact_valid(poses, g["he_a"][i], [1, 1], obst_rt, obst_he)
    assert oracle.exact_valid(poses, g["he_a"][i], [0, 0], obst_rt, obst_he)
