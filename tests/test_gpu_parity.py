"""GPU parity: the CUDA engine (through the C-ABI) against the reference's golden vectors.

Every assertion is bit-exact: labels and obstacle bitsets are integers, and the
fp64 predicates follow the reference's operation order (rgg_device.cuh).  The
cases mirror the reference's own suites:
  * kernel known-answer sets          proj/tests/test_kernels.cpp:46-121
  * batch_over/batch_under masks      proj/tests/test_batch.cpp:208-234
  * states + bits + reports per move  proj/tests/test_batch.cpp:260-285
  * empty move list                   proj/tests/test_batch.cpp:287-295
  * unknown obstacle id               proj/src/engine_batch.cpp:146-148
"""
import numpy as np
import pytest

from conftest import SCENARIOS, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng_mod():
    from paper_2603_28674_b200 import engine

    engine.library()
    return engine


def _layout(g):
    from paper_2603_28674_b200.engine import LayoutView

    return LayoutView.from_any(g)


def _bits2d(b, words):
    return b.reshape(-1, words)


@pytest.mark.parametrize("name", SCENARIOS)
def test_replay_per_move(eng_mod, name):
    """One update_obstacle per move: reports and snapshots equal the reference's."""
    g = load_golden(name)
    eng = eng_mod.GpuEngine(_layout(g))
    grouped = int(g["groups"]) > 1
    snaps = {int(i): k for k, i in enumerate(g["snap_at"])}
    for i, (o, rt) in enumerate(zip(g["ids"], g["rts"])):
        rep = eng.update_obstacle(int(o), rt)
        if not grouped:
            exp = g["reports"][i]
            assert [rep.new_green, rep.new_red, rep.new_gray, rep.unknown_after_heuristic] == exp[:4].tolist(), i
        if i in snaps:
            k = snaps[i]
            assert np.array_equal(eng.states(), g["snap_states"][k]), f"states differ after move {i}"
            bits = _bits2d(eng.obstacle_bits(), eng.words)
            assert np.array_equal(bits, g["snap_bits"][k].reshape(bits.shape)), f"bits differ after move {i}"


@pytest.mark.parametrize("name", SCENARIOS)
def test_replay_one_batch(eng_mod, name):
    """The whole move script as ONE batch_update: per-move reports from one launch sequence."""
    g = load_golden(name)
    eng = eng_mod.GpuEngine(_layout(g))
    reps = eng.batch_update((g["ids"], g["rts"]))
    assert len(reps) == len(g["ids"])
    if int(g["groups"]) == 1:
        got = np.array([[r.new_green, r.new_red, r.new_gray, r.unknown_after_heuristic] for r in reps])
        assert np.array_equal(got, g["reports"][:, :4])
    assert np.array_equal(eng.states(), g["snap_states"][-1])
    bits = _bits2d(eng.obstacle_bits(), eng.words)
    assert np.array_equal(bits, g["snap_bits"][-1].reshape(bits.shape))
    st = g["snap_states"][-1]
    assert eng.unknown_count() == int(np.sum(st == 2))
    assert np.array_equal(eng.gray_ids(), np.nonzero(st == 2)[0].astype(np.int32))
    assert np.array_equal(eng.gray_ids_view(), np.nonzero(st == 2)[0].astype(np.int32))
    allc = np.arange(int(g["N"]), dtype=np.int32)
    o = int(g["mask_obstacle"])
    assert np.array_equal(eng.batch_over(allc, o), g["masks"][0])
    assert np.array_equal(eng.batch_under(allc, o), g["masks"][1])


@pytest.mark.parametrize("name", ["scn_table4_obstacles_1000_5x", "syn_se2_m80"])
@pytest.mark.parametrize("chunk", [7, 64, 100, 300])
def test_replay_chunked_lazy(eng_mod, name, chunk):
    """Lazy batches without per-move reports (the bench path); final state is the reference's.
    Chunks of <= 64 moves use bin_small_kernel, larger ones bin_kernel, >= 256 also touch on
    published units; a cell capacity of 4 puts the overflow pool in use in all of them."""
    g = load_golden(name)
    eng = eng_mod.GpuEngine(_layout(g), cell_size=64, cell_capacity=4)  # tiny capacity: overflow pool in use
    ids, rts = g["ids"], g["rts"]
    for a in range(0, len(ids), chunk):
        eng.batch_update((ids[a:a + chunk], rts[a:a + chunk]), per_move=False)
    assert np.array_equal(eng.states(), g["snap_states"][-1])
    bits = _bits2d(eng.obstacle_bits(), eng.words)
    assert np.array_equal(bits, g["snap_bits"][-1].reshape(bits.shape))


def test_kat_sat_through_engine(eng_mod):
    """test_kernels.cpp:46-87: 10000 SAT bytes, seed 2025, via batch_over."""
    g = load_golden("kat_sat")
    from paper_2603_28674_b200.engine import LayoutView

    n = len(g["idx"])
    lv = LayoutView(N=n, B=1, S=1, M=1, C=1, edge_sat=g["boxes"][g["idx"]],
                    comp_aabb=np.tile([-1e9, -1e9, -1e9, 1e9, 1e9, 1e9], (n, 1)).astype(np.float64),
                    row_off=np.zeros(n + 1, np.int32), segs=np.zeros((0, 7)), spline_r=np.zeros(1),
                    obst_he=g["obstacle_he"][None, :], obst_sph_local=np.zeros((1, 1, 3)),
                    obst_sph_r=np.zeros(1), obst_sph_n=np.ones(1, np.int32))
    eng = eng_mod.GpuEngine(lv)
    eng.update_obstacle(0, g["obstacle_pose"])
    mask = eng.batch_over(np.arange(n, dtype=np.int32), 0)
    assert np.array_equal(mask, g["out"])
    assert 0 < mask.sum() < n


def test_kat_seg_through_engine(eng_mod):
    """test_kernels.cpp:89-121: 9001 seg-sphere bytes, seed 777, via batch_under."""
    g = load_golden("kat_seg")
    from paper_2603_28674_b200.engine import LayoutView

    n = len(g["idx"])
    pose = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, *g["center"]], np.float64)
    lv = LayoutView(N=n, B=1, S=1, M=1, C=1, edge_sat=np.zeros((n, 21)),
                    comp_aabb=np.tile([-1e9, -1e9, -1e9, 1e9, 1e9, 1e9], (n, 1)).astype(np.float64),
                    row_off=np.arange(n + 1, dtype=np.int32), segs=g["segs"][g["idx"]],
                    spline_r=np.array([float(g["r_total"])]), obst_he=np.ones((1, 3)),
                    obst_sph_local=np.zeros((1, 1, 3)), obst_sph_r=np.zeros(1), obst_sph_n=np.ones(1, np.int32))
    eng = eng_mod.GpuEngine(lv)
    eng.update_obstacle(0, pose)
    mask = eng.batch_under(np.arange(n, dtype=np.int32), 0)
    assert np.array_equal(mask, g["out"])


def test_empty_moves_and_bad_id(eng_mod):
    g = load_golden("scn_quick_smoke")
    eng = eng_mod.GpuEngine(_layout(g))
    assert eng.batch_update([]) == []
    assert np.array_equal(eng.states(), np.zeros(int(g["N"]), np.uint8))
    ids = np.array([0, 1, 7], np.int32)
    with pytest.raises(ValueError, match="unknown obstacle id"):
        eng.batch_update((ids, g["rts"][:3]))
    # moves before the bad one were applied, like the reference's sequential loop
    ref = eng_mod.GpuEngine(_layout(g))
    ref.batch_update((ids[:2], g["rts"][:2]))
    assert np.array_equal(eng.states(), ref.states())


def test_wide_requires_opt_in(eng_mod):
    g = load_golden("syn_se2_m80")
    with pytest.raises(ValueError, match="at most 64 obstacles"):
        eng_mod.GpuEngine(_layout(g), allow_wide=False)


def test_use_under_false_never_red(eng_mod):
    """update_report.hpp:41-45: outer-only mode produces no red."""
    g = load_golden("scn_table4_obstacles_1000_5x")
    eng = eng_mod.GpuEngine(_layout(g), use_under=False)
    eng.batch_update((g["ids"][:50], g["rts"][:50]))
    st = eng.states()
    assert not np.any(st == 1)
    assert np.any(st == 2)


@pytest.mark.parametrize("name", ["scn_table4_obstacles_1000_5x", "syn_se2_m80"])
def test_interleaved_cell_shards_compose(eng_mod, name):
    """rgg_gpu_options.shard_rank/shard_count: two shard handles (one per future GPU)
    own disjoint cells; their labels compose to the reference's and their per-move
    counters sum to the reference's reports (the all-reduce of dist.py)."""
    import torch

    g = load_golden(name)
    lv = _layout(g)
    shards = [eng_mod.GpuEngine(lv, shard_rank=r, shard_count=2, cell_size=64) for r in range(2)]
    n = len(g["ids"])
    ids = torch.from_numpy(g["ids"].astype(np.int32)).cuda()
    rts = torch.from_numpy(g["rts"]).cuda()
    total = torch.zeros((n, 4), dtype=torch.int32, device="cuda")
    for sh in shards:
        sh.update_tensors(ids, rts, per_move=True)
        c = torch.zeros((n, 4), dtype=torch.int32, device="cuda")
        sh.counters_into(c, n)
        total += c
    st = [sh.states() for sh in shards]
    own = [s != 0xFF for s in st]
    assert not np.any(own[0] & own[1]) and np.all(own[0] | own[1]), "shards must partition the components"
    merged = np.where(own[0], st[0], st[1])
    assert np.array_equal(merged, g["snap_states"][-1])
    if int(g["groups"]) == 1:
        from paper_2603_28674_b200.dist import DistributedUpdater

        reps = DistributedUpdater.reports(total, 0)
        got = np.array([[r["new_green"], r["new_red"], r["new_gray"], r["unknown_after_heuristic"]] for r in reps])
        assert np.array_equal(got, g["reports"][:, :4])


@pytest.mark.parametrize("name", ["scn_table4_obstacles_1000_5x", "syn_se2_m80"])
def test_item_queue_overflow_replays(eng_mod, name, monkeypatch):
    """A narrow-item queue too small for the batch: the apply kernel changes nothing,
    the host grows the queue and replays the update (rgg_capi.cu grow_items); labels,
    bits and per-move reports still equal the reference's."""
    g = load_golden(name)
    monkeypatch.setenv("RGG_ITEMS_CAP", "64")
    eng = eng_mod.GpuEngine(_layout(g))
    reps = eng.batch_update((g["ids"], g["rts"]))
    if int(g["groups"]) == 1:
        got = np.array([[r.new_green, r.new_red, r.new_gray, r.unknown_after_heuristic] for r in reps])
        assert np.array_equal(got, g["reports"][:, :4])
    assert np.array_equal(eng.states(), g["snap_states"][-1])
    bits = _bits2d(eng.obstacle_bits(), eng.words)
    assert np.array_equal(bits, g["snap_bits"][-1].reshape(bits.shape))


@pytest.mark.parametrize("cap", ["0", "1"])
@pytest.mark.parametrize("name", ["scn_table4_obstacles_1000_5x", "syn_se2_m80", "scn_table5_manipulator_100", "syn_3d_m20"])
def test_recheck_queue_overflow(eng_mod, name, cap, monkeypatch):
    """The over items the fp32 filter leaves undecided go through a bounded queue to
    narrow_recheck_kernel (the fp64 recheck); past the queue's capacity that kernel re-runs
    every over item instead.  Both ways the labels, bits and reports equal the reference's.
    (RGG_RECHECK_MIN_MOVES=0: the queue for these small batches too.)"""
    g = load_golden(name)
    monkeypatch.setenv("RGG_RECHECK_CAP", cap)
    monkeypatch.setenv("RGG_RECHECK_MIN_MOVES", "0")
    eng = eng_mod.GpuEngine(_layout(g))
    reps = eng.batch_update((g["ids"], g["rts"]))
    if int(g["groups"]) == 1:
        got = np.array([[r.new_green, r.new_red, r.new_gray, r.unknown_after_heuristic] for r in reps])
        assert np.array_equal(got, g["reports"][:, :4])
    assert np.array_equal(eng.states(), g["snap_states"][-1])
    bits = _bits2d(eng.obstacle_bits(), eng.words)
    assert np.array_equal(bits, g["snap_bits"][-1].reshape(bits.shape))


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"RGG_EARLY_TOUCH_MIN": "1"}, {"RGG_NO_EARLY_BIN": "1"}, {"RGG_NO_SMALL_BIN": "1"},
                                 {"RGG_NO_SINGLE": "1"}, {"RGG_WARP_TOUCH": "1"}, {"RGG_NO_PDL": "1"},
                                 {"RGG_NO_SMALL_BIN": "1", "RGG_SELF_BOX_MAX": "0"}])
def test_kernel_handoffs(env):
    """The split pipeline's in-kernel handoffs, forced on or off for every batch size
    (rgg_kernels.cu: bin on the pose warps' published boxes, touch on bin's published
    units; by default touch waits for the whole bin kernel below 256 moves; single moves
    through the batched pipeline instead of the single-move kernel; touch one warp per slice
    instead of one CTA per cell chunk; plain stream order instead of programmatic launches;
    the scatter binning at every batch size, waiting for the pose kernel's boxes instead of
    deriving them itself as it does below 512 moves)."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k",
                        "replay or chunked or overflow or eager or resolve",
                        os.path.join(here, "test_gpu_parity.py"), os.path.join(here, "test_gpu_resolve.py")],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_degenerate_sizes(eng_mod):
    """Empty roadmap, no obstacles, a single component: create, update, query."""
    from paper_2603_28674_b200.engine import LayoutView

    g = load_golden("scn_quick_smoke")
    # no components
    lv0 = LayoutView(N=0, B=1, S=1, M=int(g["M"]), C=int(g["C"]), edge_sat=np.zeros((0, 21)),
                     comp_aabb=np.zeros((0, 6)), row_off=np.zeros(1, np.int32), segs=np.zeros((0, 7)),
                     spline_r=np.zeros(1), obst_he=g["obst_he"], obst_sph_local=g["obst_sph_local"],
                     obst_sph_r=g["obst_sph_r"], obst_sph_n=g["obst_sph_n"])
    e0 = eng_mod.GpuEngine(lv0)
    reps = e0.batch_update((g["ids"][:5], g["rts"][:5]))
    assert len(reps) == 5 and all(r.new_gray == 0 for r in reps)
    assert len(e0.states()) == 0 and e0.unknown_count() == 0 and len(e0.gray_ids()) == 0
    # one component: the first of the scenario, replayed against the reference's labels
    lv1 = LayoutView(N=1, B=int(g["B"]), S=int(g["S"]), M=int(g["M"]), C=int(g["C"]),
                     edge_sat=g["edge_sat"][:int(g["B"])], comp_aabb=g["comp_aabb"][:1],
                     row_off=g["row_off"][:int(g["B"]) * int(g["S"]) + 1].astype(np.int32),
                     segs=g["segs"][:int(g["row_off"][int(g["B"]) * int(g["S"])])], spline_r=g["spline_r"],
                     obst_he=g["obst_he"], obst_sph_local=g["obst_sph_local"], obst_sph_r=g["obst_sph_r"],
                     obst_sph_n=g["obst_sph_n"])
    e1 = eng_mod.GpuEngine(lv1)
    e1.batch_update((g["ids"], g["rts"]))
    assert e1.states()[0] == g["snap_states"][-1][0]


def test_no_obstacles(eng_mod):
    """A roadmap without obstacles: every move id is unknown, labels stay GREEN."""
    from paper_2603_28674_b200.engine import LayoutView

    g = load_golden("scn_quick_smoke")
    lv = LayoutView(N=int(g["N"]), B=int(g["B"]), S=int(g["S"]), M=0, C=1, edge_sat=g["edge_sat"],
                    comp_aabb=g["comp_aabb"], row_off=g["row_off"].astype(np.int32), segs=g["segs"],
                    spline_r=g["spline_r"], obst_he=np.zeros((0, 3)), obst_sph_local=np.zeros((0, 1, 3)),
                    obst_sph_r=np.zeros(0), obst_sph_n=np.zeros(0, np.int32))
    eng = eng_mod.GpuEngine(lv)
    assert eng.batch_update([]) == []
    with pytest.raises(ValueError, match="unknown obstacle id"):
        eng.batch_update((np.zeros(1, np.int32), g["rts"][:1]))
    assert not np.any(eng.states())


@pytest.mark.parametrize("scn", ["quick_smoke", "table4_obstacles_1000_5x", "table5_manipulator_100"])
def test_create_from_components_equals_layout(eng_mod, scn):
    """rgg_gpu_create_from_components (serialize on the device: sat_prep, AABBs, seg_prep
    from the OBB corners and real spline points) builds the same engine as
    rgg_gpu_create from the reference's serialized layout: every report, label and bit
    word equal after the scenario's moves."""
    import os

    from conftest import GOLDEN
    from oracle import ref

    w = ref.World.from_scn(open(os.path.join(GOLDEN, "scenarios", scn + ".scn")).read())
    lay = w.layout()
    ids, rts = w.moves()
    a = eng_mod.GpuEngine(eng_mod.LayoutView.from_any(lay), allow_wide=True)
    b = eng_mod.GpuEngine(lay, components=True, allow_wide=True)
    ra = a.batch_update((ids, rts)).counts()
    rb = b.batch_update((ids, rts)).counts()
    assert np.array_equal(ra, rb)
    assert np.array_equal(a.states(), b.states())
    assert np.array_equal(a.obstacle_bits(), b.obstacle_bits())
    ref_eng = ref.Engine(w, kind=0, threads=1)
    ref_eng.run(ids, rts)
    assert np.array_equal(b.states(), ref_eng.states())


@pytest.mark.gpu
@pytest.mark.parametrize("name", SCENARIOS)
def test_single_move_kernel_equals_batched_path(eng_mod, name):
    """Single-move updates take the fused single-move kernel (rggk::launch_single); an
    update with census=True keeps the batched pipeline.  Move by move, both engines give
    the same report, labels, bit words and (as a set) gray over-hits."""
    import torch

    g = load_golden(name)
    a = eng_mod.GpuEngine(_layout(g))
    b = eng_mod.GpuEngine(_layout(g))
    ids = torch.tensor(np.asarray(g["ids"], np.int32), device="cuda")
    rts = torch.tensor(np.asarray(g["rts"], np.float64).reshape(len(g["ids"]), 12), device="cuda")
    cnt = torch.empty((1, 4), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    for i, (o, rt) in enumerate(zip(g["ids"], g["rts"])):
        ra = a.update_obstacle(int(o), rt)
        b.update_device(ids[i:].data_ptr(), rts[i:].data_ptr(), 1, per_move=True, census=True)
        b.counters_into(cnt, 1)
        assert [ra.new_green, ra.new_red, ra.new_gray] == cnt[0, :3].tolist(), i
        assert np.array_equal(np.sort(a.last_hits()), np.sort(b.last_hits())), i
    assert np.array_equal(a.states(), b.states())
    assert np.array_equal(a.obstacle_bits(), b.obstacle_bits())


@pytest.mark.gpu
@pytest.mark.parametrize("name", SCENARIOS)
def test_gray_list_written_inside_the_host_update(eng_mod, name):
    """A synchronous batch_update with gray_list=True writes the GRAY ids into mapped host
    memory inside the update (gray_write_kernel's host_out): gray_ids_view() then returns
    them without a copy.  Chunked updates exercise tile boundaries at several counts; the
    list equals the device compaction and the labels, and a later label change (write_states,
    resolve) falls back to the device list."""
    g = load_golden(name)
    eng = eng_mod.GpuEngine(_layout(g))
    ids, rts = np.asarray(g["ids"], np.int32), np.asarray(g["rts"], np.float64).reshape(-1, 12)
    for a in range(0, len(ids), 7):
        eng.batch_update((ids[a:a + 7], rts[a:a + 7]), gray_list=True)
        view = eng.gray_ids_view().copy()
        st = eng.states()
        assert np.array_equal(view, np.nonzero(st == 2)[0].astype(np.int32)), a
        assert np.array_equal(eng.gray_ids(), view), a
    gray = np.nonzero(eng.states() == 2)[0].astype(np.int32)
    if len(gray):
        eng.write_states(gray[:1], np.zeros(1, np.uint8))
        assert np.array_equal(eng.gray_ids_view(), gray[1:])


@pytest.mark.gpu
def test_staged_moves_equal_host_moves(eng_mod):
    """Moves written into the engine's pinned staging buffers (rgg_gpu_stage) give the same
    reports, labels and bits as the same moves passed from ordinary host arrays."""
    g = load_golden("scn_table4_obstacles_1000_5x")
    a = eng_mod.GpuEngine(_layout(g))
    b = eng_mod.GpuEngine(_layout(g))
    ids, rts = np.asarray(g["ids"], np.int32), np.asarray(g["rts"], np.float64).reshape(-1, 12)
    sid, srt = b.staging(len(ids))
    for a0 in range(0, len(ids), 9):
        n = min(9, len(ids) - a0)
        ra = a.batch_update((ids[a0:a0 + n], rts[a0:a0 + n]), gray_list=True).counts()
        sid[:n], srt[:n] = ids[a0:a0 + n], rts[a0:a0 + n]
        rb = b.batch_update((sid[:n], srt[:n]), gray_list=True).counts()
        assert np.array_equal(ra, rb), a0
        assert np.array_equal(a.gray_ids_view(), b.gray_ids_view()), a0
    assert np.array_equal(a.states(), b.states())
    assert np.array_equal(a.obstacle_bits(), b.obstacle_bits())
