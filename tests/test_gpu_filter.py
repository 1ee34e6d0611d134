"""Adversarial parity for the fp32 filters + fp64 recheck (rgg_device.cuh sat_filter32 /
seg_filter32): boxes and segments placed exactly at, and a few ulps / 1e-12 .. 1e-7
around, the contact configuration, with random rotations (so cross axes decide).
The GPU verdicts (batch_over / batch_under, the filter path) must equal the exact
fp64 reference sequence of the C oracle on every pair."""
import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

OFFSETS = [0.0, 1e-15, -1e-15, 1e-12, -1e-12, 1e-9, -1e-9, 1e-7, -1e-7, 3e-6, -3e-6]


def rot(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def corners(c, R, he):
    out = []
    for i in range(8):
        p = c.copy()
        for k in range(3):
            s = 1.0 if (i >> k) & 1 else -1.0
            p = p + s * he[k] * R[:, k]
        out.append(p)
    return np.concatenate(out)


def test_sat_filter_adversarial():
    from paper_2603_28674_b200.engine import GpuEngine, LayoutView

    rng = np.random.default_rng(7)
    he_o = np.array([1.3, 0.7, 0.9])
    Ro = rot(rng)
    pose = np.concatenate([Ro.reshape(-1), [0.4, -0.3, 0.2]])
    osat, _, _, _ = oracle.obstacle_operands(he_o, np.zeros((1, 3)), 1, 0.1, pose)
    boxes = []
    for trial in range(300):
        R = rot(rng) if trial % 3 else np.eye(3)
        he = rng.uniform(0.05, 2.0, 3)
        n = rng.normal(size=3)
        n /= np.linalg.norm(n)
        if trial % 3 == 0:  # face contact along the obstacle's own axis
            R = Ro.copy()
            n = Ro[:, trial % 3]
        # bisection for the contact distance along n (exact fp64 verdicts)
        lo, hi = 0.0, 20.0
        for _ in range(80):
            mid = 0.5 * (lo + hi)
            s = oracle.sat_prep(corners(pose[9:] + mid * n, R, he))
            lo, hi = (mid, hi) if oracle.sat_boxes(s, osat) else (lo, mid)
        for off in OFFSETS:
            t = lo * (1 + off) + off
            boxes.append(oracle.sat_prep(corners(pose[9:] + t * n, R, he)))
        boxes.append(oracle.sat_prep(corners(pose[9:] + np.nextafter(lo, 0) * n, R, he)))
        boxes.append(oracle.sat_prep(corners(pose[9:] + np.nextafter(hi, 30) * n, R, he)))
    boxes = np.array(boxes)
    N = len(boxes)
    lv = LayoutView(N=N, B=1, S=1, M=1, C=1, edge_sat=boxes,
                    comp_aabb=np.tile([-1e9, -1e9, -1e9, 1e9, 1e9, 1e9], (N, 1)).astype(np.float64),
                    row_off=np.zeros(N + 1, np.int32), segs=np.zeros((0, 7)), spline_r=np.zeros(1),
                    obst_he=he_o[None, :], obst_sph_local=np.zeros((1, 1, 3)), obst_sph_r=np.array([0.1]),
                    obst_sph_n=np.ones(1, np.int32))
    eng = GpuEngine(lv)
    eng.update_obstacle(0, pose)
    got = eng.batch_over(np.arange(N, dtype=np.int32), 0)
    exp = oracle.sat_batch(boxes, np.arange(N, dtype=np.int32), osat)
    assert 0 < exp.sum() < N
    assert np.array_equal(got, exp), f"{int(np.sum(got != exp))} SAT verdicts differ"


def test_seg_filter_adversarial():
    from paper_2603_28674_b200.engine import GpuEngine, LayoutView

    rng = np.random.default_rng(11)
    r = 0.7
    centre = np.array([1.1, -2.3, 0.6])
    segs = []
    for trial in range(400):
        n = rng.normal(size=3)
        n /= np.linalg.norm(n)
        t = np.cross(n, rng.normal(size=3))
        t /= np.linalg.norm(t)
        L = rng.uniform(0.0, 2.0) if trial % 5 else 0.0  # include point segments
        shift = rng.uniform(-1.0, 1.0) * L
        for off in OFFSETS:
            base = centre + n * r * (1 + off)
            a = base + t * (shift - L)
            b = base + t * (shift + L)
            if trial % 7 == 3:  # endpoint contact instead of interior contact
                a = base
                b = base + n * L
            segs.append(oracle.seg_prep(np.concatenate([a, b])))
    segs = np.array(segs)
    N = len(segs)
    pose = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, *centre])
    lv = LayoutView(N=N, B=1, S=1, M=1, C=1, edge_sat=np.zeros((N, 21)),
                    comp_aabb=np.tile([-1e9, -1e9, -1e9, 1e9, 1e9, 1e9], (N, 1)).astype(np.float64),
                    row_off=np.arange(N + 1, dtype=np.int32), segs=segs, spline_r=np.array([r]),
                    obst_he=np.ones((1, 3)), obst_sph_local=np.zeros((1, 1, 3)), obst_sph_r=np.zeros(1),
                    obst_sph_n=np.ones(1, np.int32))
    eng = GpuEngine(lv)
    eng.update_obstacle(0, pose)
    got = eng.batch_under(np.arange(N, dtype=np.int32), 0)
    exp = oracle.seg_sphere_batch(segs, np.arange(N, dtype=np.int32), centre, r)
    assert 0 < exp.sum() < N
    assert np.array_equal(got, exp), f"{int(np.sum(got != exp))} segment-sphere verdicts differ"


@pytest.mark.parametrize("centre,o_r", [((1.1, -2.3, 0.6), 0.0), ((71.3, -69.9, 0.6), 0.25),
                                        ((-3.0e3, 1.5e3, 7.0), 0.5)])
def test_seg_filter_adversarial_update_path(centre, o_r):
    """The narrow kernel's filter over the compact fp32 segment records
    (rggd::segf_filter, rgg_kernels.cu under_range32): the same near-contact segments,
    far from the origin too (the absolute error term of the rounded coordinates),
    through a real update; RED iff the reference's seg_sphere hits."""
    from paper_2603_28674_b200.engine import GpuEngine, LayoutView

    rng = np.random.default_rng(int(abs(centre[0])) + 5)
    r_spline = 0.7
    r = r_spline + o_r
    centre = np.array(centre)
    segs = []
    for trial in range(300):
        n = rng.normal(size=3)
        n /= np.linalg.norm(n)
        t = np.cross(n, rng.normal(size=3))
        t /= np.linalg.norm(t)
        L = rng.uniform(0.0, 2.0) if trial % 5 else 0.0
        shift = rng.uniform(-1.0, 1.0) * L
        for off in OFFSETS:
            base = centre + n * r * (1 + off)
            a = base + t * (shift - L)
            b = base + t * (shift + L)
            if trial % 7 == 3:
                a = base
                b = base + n * L
            segs.append(oracle.seg_prep(np.concatenate([a, b])))
    segs = np.array(segs)
    N = len(segs)
    pose = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, *centre])
    lv = LayoutView(N=N, B=1, S=1, M=1, C=1, edge_sat=np.zeros((N, 21)),
                    comp_aabb=np.tile([-1e9, -1e9, -1e9, 1e9, 1e9, 1e9], (N, 1)).astype(np.float64),
                    row_off=np.arange(N + 1, dtype=np.int32), segs=segs, spline_r=np.array([r_spline]),
                    obst_he=np.ones((1, 3)), obst_sph_local=np.zeros((1, 1, 3)), obst_sph_r=np.array([o_r]),
                    obst_sph_n=np.ones(1, np.int32))
    eng = GpuEngine(lv)
    eng.update_obstacle(0, pose)
    got = eng.states() == 1
    r_total = o_r + r_spline
    exp = oracle.seg_sphere_batch(segs, np.arange(N, dtype=np.int32), centre, r_total).astype(bool)
    assert 0 < exp.sum() < N
    assert np.array_equal(got, exp), f"{int(np.sum(got != exp))} segment-sphere verdicts differ"


def _near_contact_sat_layout(origin):
    """150 near-contact box families around one obstacle posed at `origin`: the box at the
    bisected contact distance, offsets around it and the neighbouring doubles."""
    from paper_2603_28674_b200.engine import LayoutView

    rng = np.random.default_rng(int(abs(origin[0])) + 17)
    he_o = np.array([1.3, 0.7, 0.9])
    Ro = rot(rng)
    pose = np.concatenate([Ro.reshape(-1), origin])
    osat, _, _, _ = oracle.obstacle_operands(he_o, np.zeros((1, 3)), 1, 0.1, pose)
    boxes = []
    for trial in range(150):
        R = rot(rng) if trial % 3 else np.eye(3)
        he = rng.uniform(0.05, 2.0, 3)
        n = rng.normal(size=3)
        n /= np.linalg.norm(n)
        if trial % 3 == 0:
            R = Ro.copy()
            n = Ro[:, trial % 3]
        lo, hi = 0.0, 20.0
        for _ in range(80):
            mid = 0.5 * (lo + hi)
            s = oracle.sat_prep(corners(pose[9:] + mid * n, R, he))
            lo, hi = (mid, hi) if oracle.sat_boxes(s, osat) else (lo, mid)
        for off in OFFSETS:
            t = lo * (1 + off) + off
            boxes.append(oracle.sat_prep(corners(pose[9:] + t * n, R, he)))
        boxes.append(oracle.sat_prep(corners(pose[9:] + np.nextafter(lo, 0) * n, R, he)))
        boxes.append(oracle.sat_prep(corners(pose[9:] + np.nextafter(hi, 30) * n, R, he)))
    boxes = np.array(boxes)
    N = len(boxes)
    lv = LayoutView(N=N, B=1, S=1, M=1, C=1, edge_sat=boxes,
                    comp_aabb=np.tile([-1e9, -1e9, -1e9, 1e9, 1e9, 1e9], (N, 1)).astype(np.float64),
                    row_off=np.zeros(N + 1, np.int32), segs=np.zeros((0, 7)), spline_r=np.zeros(1),
                    obst_he=he_o[None, :], obst_sph_local=np.zeros((1, 1, 3)), obst_sph_r=np.array([0.1]),
                    obst_sph_n=np.ones(1, np.int32))
    exp = oracle.sat_batch(boxes, np.arange(N, dtype=np.int32), osat).astype(bool)
    return lv, pose, exp


@pytest.mark.parametrize("origin", [(0.4, -0.3, 0.2), (70.7, -69.2, 0.2), (-2.5e3, 4.0e3, 15.0)])
def test_sat_filter_adversarial_update_path(origin):
    """The over filter on the 64-byte heads with an fp32 centre (rggd::sat_filter32h):
    near-contact boxes around an obstacle far from the origin too, through a real update
    (the single-move kernel); GRAY iff the reference's sat_boxes intersects."""
    from paper_2603_28674_b200.engine import GpuEngine

    lv, pose, exp = _near_contact_sat_layout(origin)
    eng = GpuEngine(lv)
    eng.update_obstacle(0, pose)
    got = eng.states() == 2
    assert 0 < exp.sum() < len(exp)
    assert np.array_equal(got, exp), f"{int(np.sum(got != exp))} SAT verdicts differ"


@pytest.mark.parametrize("cap", ["inline", None, "0", "5"])
def test_sat_filter_adversarial_batched(cap, monkeypatch):
    """The same near-contact boxes through the batched pipeline (two moves of the
    obstacle, the second onto the contact pose).  A batch this small decides the pairs the
    fp32 filter leaves undecided inline ("inline"); with RGG_RECHECK_MIN_MOVES=0
    narrow_over_kernel queues them and narrow_under_kernel's tail decides them in fp64, and
    with a queue smaller than the undecided pairs (cap 0, 5) that tail re-runs every over item."""
    from paper_2603_28674_b200.engine import GpuEngine

    if cap != "inline":
        monkeypatch.setenv("RGG_RECHECK_MIN_MOVES", "0")
    if cap not in (None, "inline"):
        monkeypatch.setenv("RGG_RECHECK_CAP", cap)
    lv, pose, exp = _near_contact_sat_layout((70.7, -69.2, 0.2))
    eng = GpuEngine(lv)
    far = pose.copy()
    far[9:] += 1e4
    eng.filter_stats(reset=True)
    eng.batch_update((np.zeros(2, np.int32), np.stack([far, pose])))
    got = eng.states() == 2
    assert np.array_equal(got, exp), f"{int(np.sum(got != exp))} SAT verdicts differ"
    assert eng.filter_stats()["sat_rechecks"] > 5, "the near-contact pairs must reach the fp64 recheck"


def _aabb_of(cs):
    p = cs.reshape(8, 3)
    return np.concatenate([p.min(0), p.max(0)])


def test_aabb_near_contact_through_update():
    """Candidate semantics at rounding level.  The reference tests
    every grid candidate with the fp64 SAT (engine_batch.cpp:55-74); the GPU tests the
    pairs whose closed AABBs overlap after widening the obstacle's boxes by a relative
    2^-40 (rgg_kernels.cu pose_kernel).  Boxes are placed at the fp64 SAT contact
    distance and a few ulps either side, along world axes (face contact: the AABB gap
    and the SAT margin round independently), so some pairs have disjoint AABBs while the
    fp64 SAT still reports an intersection.  Through the whole update path the labels
    must equal the all-pairs fp64 SAT verdicts (everything in one reference grid cell)."""
    from paper_2603_28674_b200.engine import GpuEngine, LayoutView

    rng = np.random.default_rng(11)
    boxes, aabbs, exp = [], [], []
    disjoint_hits = 0
    for trial in range(400):
        he_o = rng.uniform(0.2, 2.0, 3)
        Ro = np.eye(3) if trial % 2 else rot(rng)
        c_o = rng.uniform(-50, 50, 3)
        pose = np.concatenate([Ro.reshape(-1), c_o])
        osat, oaabb, _, _ = oracle.obstacle_operands(he_o, np.zeros((1, 3)), 1, 1e-3, pose)
        he = rng.uniform(0.05, 2.0, 3)
        k = trial % 3
        n = np.zeros(3)
        n[k] = 1.0 if trial % 4 < 2 else -1.0
        R = np.eye(3)
        lo, hi = 0.0, 20.0
        for _ in range(100):
            mid = 0.5 * (lo + hi)
            s = oracle.sat_prep(corners(c_o + mid * n, R, he))
            lo, hi = (mid, hi) if oracle.sat_boxes(s, osat) else (lo, mid)
        t = lo
        for step in range(-3, 4):
            cs = corners(c_o + t * n, R, he)
            s = oracle.sat_prep(cs)
            a = _aabb_of(cs)
            hit = bool(oracle.sat_boxes(s, osat))
            ov = bool(np.all(a[:3] <= oaabb[3:]) and np.all(oaabb[:3] <= a[3:]))
            disjoint_hits += hit and not ov
            boxes.append((s, a, pose, he_o, hit))
            t = np.nextafter(t, 100.0) if step >= 0 else t
        for _ in range(3):
            t = np.nextafter(t, 100.0)
            cs = corners(c_o + t * n, R, he)
            s = oracle.sat_prep(cs)
            boxes.append((s, _aabb_of(cs), pose, he_o, bool(oracle.sat_boxes(s, osat))))
    # one engine per obstacle pose: every component against obstacle 0
    by_pose = {}
    for s, a, pose, he_o, hit in boxes:
        by_pose.setdefault(pose.tobytes(), (pose, he_o, []))[2].append((s, a, hit))
    bad = 0
    for pose, he_o, items in by_pose.values():
        N = len(items)
        lv = LayoutView(N=N, B=1, S=1, M=1, C=1, edge_sat=np.array([s for s, _, _ in items]),
                        comp_aabb=np.array([a for _, a, _ in items]), row_off=np.zeros(N + 1, np.int32),
                        segs=np.zeros((0, 7)), spline_r=np.zeros(1), obst_he=he_o[None, :],
                        obst_sph_local=np.zeros((1, 1, 3)), obst_sph_r=np.array([1e-3]),
                        obst_sph_n=np.ones(1, np.int32))
        eng = GpuEngine(lv, use_under=False)
        eng.update_obstacle(0, pose)
        got = eng.states()
        want = np.array([2 if hit else 0 for _, _, hit in items], np.uint8)
        bad += int(np.sum(got != want))
    print(f"pairs {len(boxes)}, AABB-disjoint fp64-SAT hits {disjoint_hits}")
    assert bad == 0, f"{bad} labels differ from the all-pairs fp64 SAT ({disjoint_hits} AABB-disjoint hits)"


def test_non_orthonormal_satboxes_take_the_exact_path():
    """the fp32 SAT filter's form equals the reference's margins only
    for orthonormal frames with e_k = |e_k| u_k.  Caller-supplied SatBoxes that are
    sheared, have non-unit axes or axes misaligned with their extents are flagged at
    rgg_gpu_create (Box32::degen) and decided by the fp64 reference sequence: the verdicts
    equal the oracle's on every pair, near contact included."""
    from paper_2603_28674_b200.engine import GpuEngine, LayoutView

    rng = np.random.default_rng(5)
    he_o = np.array([1.1, 0.6, 0.8])
    pose = np.concatenate([rot(rng).reshape(-1), [0.2, 0.1, -0.3]])
    osat, _, _, _ = oracle.obstacle_operands(he_o, np.zeros((1, 3)), 1, 0.1, pose)
    boxes = []
    for trial in range(400):
        R = rot(rng)
        he = rng.uniform(0.1, 1.5, 3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        lo, hi = 0.0, 10.0
        for _ in range(60):
            mid = 0.5 * (lo + hi)
            s = oracle.sat_prep(corners(pose[9:] + mid * d, R, he))
            lo, hi = (mid, hi) if oracle.sat_boxes(s, osat) else (lo, mid)
        s = oracle.sat_prep(corners(pose[9:] + lo * (1 + rng.uniform(-1e-6, 1e-6)) * d, R, he)).copy()
        kind = trial % 3
        if kind == 0:  # sheared frame: u_1 tilted towards u_0, e_1 along it
            u1 = s[15:18] + 1e-4 * s[12:15]
            s[15:18] = u1 / np.linalg.norm(u1)
            s[6:9] = s[15:18] * np.linalg.norm(s[6:9])
        elif kind == 1:  # axis not unit length
            s[12:15] *= 1 + 1e-6
        else:  # extent not along its axis
            s[3:6] += 1e-7 * s[15:18]
        boxes.append(s)
    boxes = np.array(boxes)
    N = len(boxes)
    lv = LayoutView(N=N, B=1, S=1, M=1, C=1, edge_sat=boxes,
                    comp_aabb=np.tile([-1e9, -1e9, -1e9, 1e9, 1e9, 1e9], (N, 1)).astype(np.float64),
                    row_off=np.zeros(N + 1, np.int32), segs=np.zeros((0, 7)), spline_r=np.zeros(1),
                    obst_he=he_o[None, :], obst_sph_local=np.zeros((1, 1, 3)), obst_sph_r=np.array([0.1]),
                    obst_sph_n=np.ones(1, np.int32))
    eng = GpuEngine(lv)
    eng.filter_stats(reset=True)
    eng.update_obstacle(0, pose)
    got = eng.batch_over(np.arange(N, dtype=np.int32), 0)
    exp = oracle.sat_batch(boxes, np.arange(N, dtype=np.int32), osat)
    assert 0 < exp.sum() < N
    assert np.array_equal(got, exp), f"{int(np.sum(got != exp))} SAT verdicts differ"
    assert eng.filter_stats()["sat_rechecks"] >= N, "flagged boxes must take the fp64 path"
