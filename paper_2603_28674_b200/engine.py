"""Host-side mirror of ``rgg::BatchEngine`` over the C-ABI of include/rgg_gpu.h.

Same names, argument meaning and error behaviour as the reference's update API
(proj/include/rgg/engine_batch.hpp:17-63):

    =====================================  ============================================
    reference                              here
    =====================================  ============================================
    BatchEngine(components, scene, opts,   GpuEngine(layout, use_under=..., ...)
                cell_capacity)             (layout = the serialized store, see LayoutView)
    update_obstacle(o, pose, lazy)         update_obstacle(o, pose, lazy=True)
    batch_update(moves, lazy)              batch_update(moves, lazy=True)
    states()                               states()         -> uint8[N]
    obstacle_bits()                        obstacle_bits()  -> uint64[N] (uint64[N, W] if M > 64)
    unknown_count()                        unknown_count()
    batch_over / batch_under               batch_over / batch_under (explicit candidates)
    resolve_all_unknown()                  resolve_all_unknown(resolver)
    std::invalid_argument                  ValueError (same message)
    std::logic_error                       RuntimeError
    =====================================  ============================================

There is no CPU fallback: constructing a GpuEngine without the built
``lib/librgg_gpu.so`` or without an sm_100 GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Callable, Iterable, Sequence

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RGG_GPU_LIB") or os.path.join(PKG, "lib", "librgg_gpu.so")  # RGG_GPU_LIB: A/B builds

RGG_OK, RGG_EINVAL, RGG_ECUDA, RGG_ENCCL, RGG_ENOMEM, RGG_ELOGIC = 0, 1, 2, 3, 4, 5
RGG_LAZY, RGG_PER_MOVE, RGG_ASYNC, RGG_CENSUS, RGG_GRAY_LIST, RGG_EAGER = 1, 2, 4, 8, 16, 32
GREEN, RED, GRAY = 0, 1, 2


class _View(C.Structure):
    _fields_ = [("n_components", C.c_int32), ("n_bodies", C.c_int32), ("n_slots", C.c_int32),
                ("n_obstacles", C.c_int32), ("max_spheres", C.c_int32),
                ("edge_sat", C.c_void_p), ("comp_aabb", C.c_void_p), ("row_off", C.c_void_p),
                ("segs", C.c_void_p), ("spline_radius", C.c_void_p), ("obst_he", C.c_void_p),
                ("obst_sph_local", C.c_void_p), ("obst_sph_r", C.c_void_p), ("obst_sph_n", C.c_void_p)]


class _CompView(C.Structure):
    _fields_ = [("n_components", C.c_int32), ("n_bodies", C.c_int32), ("n_slots", C.c_int32),
                ("n_obstacles", C.c_int32), ("max_spheres", C.c_int32), ("obb_corners", C.c_void_p),
                ("row_off", C.c_void_p), ("seg_points", C.c_void_p), ("spline_radius", C.c_void_p),
                ("obst_he", C.c_void_p), ("obst_sph_local", C.c_void_p), ("obst_sph_r", C.c_void_p),
                ("obst_sph_n", C.c_void_p)]


class _Options(C.Structure):
    _fields_ = [("device", C.c_int32), ("use_under", C.c_int32), ("cell_size", C.c_int32),
                ("cell_capacity", C.c_int32), ("allow_wide", C.c_int32), ("shard_rank", C.c_int32),
                ("shard_count", C.c_int32)]


class _Report(C.Structure):
    _fields_ = [("obstacle", C.c_int32), ("new_green", C.c_int32), ("new_red", C.c_int32),
                ("new_gray", C.c_int32), ("reval_us", C.c_int64), ("over_us", C.c_int64),
                ("under_us", C.c_int64), ("resolve_us", C.c_int64), ("unknown_after_heuristic", C.c_int32),
                ("residual_unknown", C.c_int32), ("resolve_checks", C.c_int32), ("_pad", C.c_int32)]


_REPORT_DTYPE = np.dtype(_Report)
_I32, _F64 = np.dtype(np.int32), np.dtype(np.float64)


class _ResolveView(C.Structure):
    _fields_ = [("n_components", C.c_int32), ("n_bodies", C.c_int32), ("body_half_extents", C.c_void_p),
                ("pose_off", C.c_void_p), ("poses", C.c_void_p)]


class Stats(C.Structure):
    _fields_ = [("pose_ms", C.c_float), ("bin_ms", C.c_float), ("classify_ms", C.c_float),
                ("compact_ms", C.c_float), ("total_ms", C.c_float), ("dirty_cells", C.c_int32),
                ("events", C.c_int32), ("overflow_cells", C.c_int32), ("over_pairs", C.c_int64),
                ("sat_flops", C.c_int64), ("under_pairs", C.c_int64), ("seg_sphere_tests", C.c_int64),
                ("over_hits", C.c_int64), ("under_hits", C.c_int64), ("bytes_components", C.c_int64),
                ("bytes_fp32", C.c_int64), ("gray", C.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def library() -> C.CDLL:
    """Load lib/librgg_gpu.so (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA engine not built: {LIB_PATH} missing "
                               f"(run `python -m paper_2603_28674_b200.build`)")
        L = C.CDLL(LIB_PATH)
        vp, ip, i32 = C.c_void_p, C.POINTER(C.c_int32), C.c_int32
        L.rgg_gpu_create.argtypes = [C.POINTER(_View), C.POINTER(_Options), C.POINTER(vp)]
        L.rgg_gpu_create_from_components.argtypes = [C.POINTER(_CompView), C.POINTER(_Options), C.POINTER(vp)]
        L.rgg_gpu_destroy.argtypes = [vp]
        L.rgg_gpu_destroy.restype = None
        L.rgg_gpu_last_error.argtypes = [vp]
        L.rgg_gpu_last_error.restype = C.c_char_p
        L.rgg_gpu_update.argtypes = [vp, vp, vp, i32, i32, vp]
        L.rgg_gpu_stage.argtypes = [vp, i32, C.POINTER(C.POINTER(C.c_int32)), C.POINTER(C.POINTER(C.c_double))]
        L.rgg_gpu_update_device.argtypes = [vp, vp, vp, i32, i32]
        L.rgg_gpu_sync.argtypes = [vp]
        L.rgg_gpu_count.argtypes = [vp, ip, ip, ip]
        L.rgg_gpu_read_states.argtypes = [vp, vp]
        L.rgg_gpu_read_bits.argtypes = [vp, vp, i32]
        L.rgg_gpu_unknown_count.argtypes = [vp, ip]
        L.rgg_gpu_gray_ids.argtypes = [vp, vp, i32, ip]
        L.rgg_gpu_last_hits.argtypes = [vp, vp, i32, ip]
        L.rgg_gpu_write_states.argtypes = [vp, vp, vp, i32]
        L.rgg_gpu_pair_masks.argtypes = [vp, i32, vp, i32, i32, vp]
        L.rgg_gpu_last_stats.argtypes = [vp, C.POINTER(Stats)]
        L.rgg_gpu_census.argtypes = [vp, C.POINTER(Stats)]
        L.rgg_gpu_stream.argtypes = [vp]
        L.rgg_gpu_stream.restype = vp
        L.rgg_gpu_fp64_peak.argtypes = [C.c_int, C.POINTER(C.c_double)]
        L.rgg_gpu_copy_counters.argtypes = [vp, vp, i32]
        L.rgg_gpu_set_phase_timing.argtypes = [vp, i32]
        L.rgg_gpu_set_resolver.argtypes = [vp, C.POINTER(_ResolveView)]
        L.rgg_gpu_resolve_all.argtypes = [vp, ip]
        L.rgg_gpu_exact_check.argtypes = [vp, vp, i32, vp]
        L.rgg_gpu_set_active_obstacles.argtypes = [vp, vp, vp, i32]
        L.rgg_exact_valid_sets.argtypes = [i32, i32, vp, i32, vp, vp, i32, vp, vp, vp]
        L.rgg_gpu_filter_stats.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), i32]
        L.rgg_gpu_gray_device.argtypes = [vp, vp, vp, i32]
        L.rgg_gpu_gray_view.argtypes = [vp, C.POINTER(C.POINTER(C.c_int32)), ip]
        L.rgg_gpu_fp32_peak.argtypes = [C.c_int, C.POINTER(C.c_double)]
        L.rgg_gpu_owned.argtypes = [vp, ip]
        _lib = L
    return _lib


_fastmod = False


def _fast():
    """lib/_rggfast (csrc/pyfast.c): rgg_gpu_update over the buffer protocol, ~6 us
    cheaper per call than ctypes' numpy pointer conversions; None when not built."""
    global _fastmod
    if _fastmod is False:
        library()
        try:
            import importlib.util

            import sysconfig
            path = os.path.join(os.path.dirname(LIB_PATH), "_rggfast" + sysconfig.get_config_var("EXT_SUFFIX"))
            spec = importlib.util.spec_from_file_location("_rggfast", path)
            if spec is None or not os.path.exists(path):
                raise ImportError(path)
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            _fastmod = mod
        except ImportError:
            _fastmod = None
    return _fastmod


EXPORTED = ["rgg_gpu_create", "rgg_gpu_create_from_components", "rgg_gpu_destroy", "rgg_gpu_last_error", "rgg_gpu_update", "rgg_gpu_update_device",
            "rgg_gpu_sync", "rgg_gpu_count", "rgg_gpu_read_states", "rgg_gpu_read_bits", "rgg_gpu_unknown_count",
            "rgg_gpu_gray_ids", "rgg_gpu_last_hits", "rgg_gpu_write_states", "rgg_gpu_pair_masks",
            "rgg_gpu_last_stats", "rgg_gpu_census", "rgg_gpu_stream", "rgg_gpu_fp64_peak",
            "rgg_gpu_copy_counters", "rgg_gpu_set_phase_timing", "rgg_gpu_set_resolver", "rgg_gpu_resolve_all",
            "rgg_gpu_exact_check", "rgg_gpu_filter_stats", "rgg_gpu_set_active_obstacles",
            "rgg_exact_valid_sets", "rgg_gpu_gray_device", "rgg_gpu_fp32_peak", "rgg_gpu_owned", "rgg_gpu_gray_view",
            "rgg_gpu_stage"]


@dataclass
class LayoutView:
    """The serialized store handed to rgg_gpu_create (see include/rgg_gpu.h)."""

    N: int
    B: int
    S: int
    M: int
    C: int
    edge_sat: np.ndarray  # (N*B, 21) float64
    comp_aabb: np.ndarray  # (N, 6) float64
    row_off: np.ndarray  # (N*B*S + 1,) int32
    segs: np.ndarray  # (T, 7) float64
    spline_r: np.ndarray  # (B*S,) float64
    obst_he: np.ndarray  # (M, 3)
    obst_sph_local: np.ndarray  # (M, C, 3)
    obst_sph_r: np.ndarray  # (M,)
    obst_sph_n: np.ndarray  # (M,) int32
    meta: dict = field(default_factory=dict)

    @classmethod
    def from_any(cls, obj) -> "LayoutView":
        """From any object/dict carrying the same attribute names (e.g. a golden fixture)."""
        get = (lambda k: obj[k]) if isinstance(obj, dict) else (lambda k: getattr(obj, k))
        return cls(N=int(get("N")), B=int(get("B")), S=int(get("S")), M=int(get("M")), C=int(get("C")),
                   edge_sat=get("edge_sat"), comp_aabb=get("comp_aabb"), row_off=get("row_off"),
                   segs=get("segs"), spline_r=get("spline_r"), obst_he=get("obst_he"),
                   obst_sph_local=get("obst_sph_local"), obst_sph_r=get("obst_sph_r"),
                   obst_sph_n=get("obst_sph_n"))


@dataclass
class UpdateReport:
    """rgg::UpdateReport (proj/include/rgg/update_report.hpp:11-39)."""

    obstacle: int = -1
    new_green: int = 0
    new_red: int = 0
    new_gray: int = 0
    reval_us: int = 0
    over_us: int = 0
    under_us: int = 0
    resolve_us: int = 0
    unknown_after_heuristic: int = 0
    residual_unknown: int = 0
    resolve_checks: int = 0


_REPORT_FIELDS = [f for f, _ in _Report._fields_[:-1]]


class Reports:
    """The per-move UpdateReports of one batch_update, backed by the C report array
    (numpy view ``.array``); items materialise as UpdateReport on access."""

    def __init__(self, raw):
        self._raw = raw
        self._array = None

    @property
    def array(self) -> np.ndarray:
        if self._array is None:
            self._array = np.frombuffer(self._raw, dtype=_REPORT_DTYPE)
        return self._array

    def __len__(self):
        return len(self._raw)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        r = self._raw[i]
        return UpdateReport(*[getattr(r, f) for f in _REPORT_FIELDS])

    def __iter__(self):
        return (self[i] for i in range(len(self)))

    def __eq__(self, other):
        return list(self) == list(other)

    def counts(self) -> np.ndarray:
        """(n, 4) new_green, new_red, new_gray, unknown_after_heuristic."""
        a = self.array
        return np.stack([a["new_green"], a["new_red"], a["new_gray"], a["unknown_after_heuristic"]], 1)


class _ArrayView:
    """A read-only int32 array interface over host memory the engine owns."""

    __slots__ = ("__array_interface__",)

    def __init__(self, addr: int, n: int):
        self.__array_interface__ = {"data": (addr, True), "shape": (n,), "typestr": "<i4", "version": 3}


def _pose12(pose) -> np.ndarray:
    p = np.ascontiguousarray(pose, dtype=np.float64).reshape(-1)
    if p.size != 12:
        raise ValueError("pose must be 12 doubles: row-major rotation r[9] then translation t[3]")
    return p


class GpuEngine:
    def __init__(self, layout, use_under: bool = True, cell_size: int = 0, cell_capacity: int = 64,
                 allow_wide: bool | None = None, device: int = 0, shard_rank: int = 0, shard_count: int = 1,
                 components: bool = False):
        """layout: the serialized store (LayoutView, or anything with its names).  With
        components=True it is the raw components instead (attributes N, B, S, M, C,
        e_plus = OBB corners N*B x 24, row_off, seg_pts = real segment end points T x 6,
        spline_r and the obstacle arrays): rgg_gpu_create_from_components runs the
        serialize step on the device."""
        L = library()
        lv = layout if components or isinstance(layout, LayoutView) else LayoutView.from_any(layout)
        keep = {}

        def arr(name, dt, shape=None):
            a = np.ascontiguousarray(getattr(lv, name), dtype=dt)
            keep[name] = a
            return a.ctypes.data

        wide = lv.M > 64 if allow_wide is None else allow_wide
        opts = _Options(device, int(use_under), cell_size, cell_capacity, int(wide), shard_rank, shard_count)
        h = C.c_void_p()
        if components:
            cview = _CompView(lv.N, lv.B, lv.S, lv.M, lv.C, arr("e_plus", np.float64), arr("row_off", np.int32),
                              arr("seg_pts", np.float64), arr("spline_r", np.float64), arr("obst_he", np.float64),
                              arr("obst_sph_local", np.float64), arr("obst_sph_r", np.float64),
                              arr("obst_sph_n", np.int32))
            rc = L.rgg_gpu_create_from_components(C.byref(cview), C.byref(opts), C.byref(h))
        else:
            view = _View(lv.N, lv.B, lv.S, lv.M, lv.C, arr("edge_sat", np.float64), arr("comp_aabb", np.float64),
                         arr("row_off", np.int32), arr("segs", np.float64), arr("spline_r", np.float64),
                         arr("obst_he", np.float64), arr("obst_sph_local", np.float64),
                         arr("obst_sph_r", np.float64), arr("obst_sph_n", np.int32))
            rc = L.rgg_gpu_create(C.byref(view), C.byref(opts), C.byref(h))
        self._h = h
        if rc != RGG_OK:
            msg = L.rgg_gpu_last_error(h).decode()
            L.rgg_gpu_destroy(h)
            self._h = None
            self._raise(rc, msg)
        n, m, w = C.c_int32(), C.c_int32(), C.c_int32()
        L.rgg_gpu_count(h, C.byref(n), C.byref(m), C.byref(w))
        self.n_components, self.n_obstacles, self.words = n.value, m.value, w.value
        L.rgg_gpu_owned(h, C.byref(n))
        self.n_owned = n.value  # components of this shard
        self.layout = lv
        self._resolver = None
        self._hv = h.value or 0  # the handle as an int (pyfast)
        self._one = (np.zeros(1, np.int32), (_Report * 1)())  # update_obstacle's move / report buffers
        self._gv_p, self._gv_n = C.POINTER(C.c_int32)(), C.c_int32()  # gray_ids_view's out-parameters

    # ------------------------------------------------------------- plumbing
    @staticmethod
    def _raise(rc, msg):
        if rc == RGG_EINVAL:
            raise ValueError(msg)
        raise RuntimeError(f"rgg_gpu error {rc}: {msg}")

    def _check(self, rc):
        if rc != RGG_OK:
            self._raise(rc, library().rgg_gpu_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            library().rgg_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # ------------------------------------------------------------ update API
    def batch_update(self, moves, lazy: bool = True, per_move: bool = True,
                     resolve: Callable[[np.ndarray], np.ndarray] | None = None,
                     gray_list: bool = False) -> list[UpdateReport]:
        """moves: list of (obstacle, pose12) pairs, or a tuple (ids int32[n], rt12 float64[n, 12]).
        gray_list: compact the GRAY ids inside the update (gray_ids() then only copies them)."""
        ids, rts = self._moves(moves)
        if not lazy:
            if self._resolver is not None and resolve is None:  # exact resolve on the GPU, move by move
                n = len(ids)
                if n == 0:
                    return []
                reps = (_Report * n)()
                self._check(library().rgg_gpu_update(self._h, ids.ctypes.data, rts.ctypes.data, n,
                                                     RGG_EAGER | RGG_PER_MOVE, reps))
                return Reports(reps)
            return [self.update_obstacle(int(o), r, lazy=False, resolve=resolve) for o, r in zip(ids, rts)]
        n = len(ids)
        if n == 0:
            return []
        reps = (_Report * n)()
        flags = RGG_LAZY | (RGG_PER_MOVE if per_move else 0) | (RGG_GRAY_LIST if gray_list else 0)
        fast = _fast()
        if fast is not None:
            rc = fast.update(self._hv, ids, rts, flags, reps)
        else:
            rc = library().rgg_gpu_update(self._h, ids.ctypes.data, rts.ctypes.data, n, flags, reps)
        self._check(rc)
        return Reports(reps)

    def update_obstacle(self, o: int, pose, lazy: bool = True,
                        resolve: Callable[[np.ndarray], np.ndarray] | None = None) -> UpdateReport:
        """BatchEngine::update_obstacle (engine_batch.cpp:145-205).  Eager mode needs
        ``resolve(ids) -> uint8 states``: the exact per-component check of
        exact_component_valid (proj/src/roadmap.cpp:129-163), which stays on the host."""
        if lazy:
            fast = _fast()
            if fast is None:
                return self.batch_update(([int(o)], _pose12(pose)[None, :]), lazy=True)[0]
            # one move: reused one-element buffers, the report built from its fields
            p = pose if (type(pose) is np.ndarray and pose.dtype is _F64 and pose.size == 12
                         and pose.flags.c_contiguous) else _pose12(pose)
            ids, rep = self._one
            ids[0] = o
            self._check(fast.update(self._hv, ids, p, RGG_LAZY | RGG_PER_MOVE, rep))
            r = rep[0]
            return UpdateReport(r.obstacle, r.new_green, r.new_red, r.new_gray, r.reval_us, r.over_us, r.under_us,
                                r.resolve_us, r.unknown_after_heuristic, r.residual_unknown, r.resolve_checks)
        if resolve is None:
            if self._resolver is None:
                raise ValueError("eager updates need set_resolver() (GPU exact resolve) or a resolve callable")
            return self.batch_update(([int(o)], _pose12(pose)[None, :]), lazy=False)[0]
        before = self.states()
        rep = self.batch_update(([int(o)], _pose12(pose)[None, :]), lazy=True)[0]
        hits = self.last_hits()
        rep.resolve_checks = len(hits)
        if len(hits):
            st = np.asarray(resolve(hits), np.uint8)
            self.write_states(hits, st)
            # finish_counts (engine_batch.cpp:41-53) compares the pre-move label with the final one
            b0 = before[hits]
            rep.new_gray -= int(np.sum(b0 != GRAY))
            rep.new_green += int(np.sum((st == GREEN) & (b0 != GREEN)))
            rep.new_red += int(np.sum((st == RED) & (b0 != RED)))
        rep.residual_unknown = self.unknown_count()
        return rep

    # ------------------------------------------------------ exact resolve
    def set_resolver(self, pose_off, poses, body_half_extents):
        """Upload the exact resolve's inputs (include/rgg_gpu.h rgg_resolve_view):
        pose_off int64[N+1], poses float64[total, B, 12] = forward_kinematics of every
        discretized configuration (robot.cpp:66-84), body_half_extents (B, 3)."""
        off = np.ascontiguousarray(pose_off, np.int64)
        ps = np.ascontiguousarray(poses, np.float64)
        he = np.ascontiguousarray(body_half_extents, np.float64).reshape(-1, 3)
        if off.shape != (self.n_components + 1,):
            raise ValueError("resolver: component count differs from the layout")
        if ps.size != int(off[-1]) * he.shape[0] * 12:
            raise ValueError("resolver: poses must hold pose_off[N] x B x 12 doubles")
        v = _ResolveView(self.n_components, he.shape[0], he.ctypes.data, off.ctypes.data, ps.ctypes.data)
        self._check(library().rgg_gpu_set_resolver(self._h, C.byref(v)))
        self._resolver = (off, he)

    def set_active_obstacles(self, ids, rts):
        """The Scene's obstacles active before this engine moves them (ObstacleModel::active
        and pose; exact_component_valid reads them, roadmap.cpp:135-139): ids int[n],
        rts float64 (n, 12). Replaces the previous list; the exact resolve only."""
        ids = np.ascontiguousarray(ids, np.int32).reshape(-1)
        rts = np.ascontiguousarray(rts, np.float64).reshape(-1, 12)
        if rts.shape[0] != ids.shape[0]:
            raise ValueError("one 12-double pose per obstacle id")
        self._check(library().rgg_gpu_set_active_obstacles(self._h, ids.ctypes.data, rts.ctypes.data, len(ids)))

    def resolve_all_unknown(self, resolve: Callable[[np.ndarray], np.ndarray] | None = None) -> int:
        """BatchEngine::resolve_all_unknown (engine_batch.cpp:217-227): on the GPU after
        set_resolver(), or with an exact check supplied by the caller."""
        if resolve is not None:
            ids = self.gray_ids()
            if len(ids):
                self.write_states(ids, np.asarray(resolve(ids), np.uint8))
            return len(ids)
        n = C.c_int32(0)
        self._check(library().rgg_gpu_resolve_all(self._h, C.byref(n)))
        return n.value

    def filter_stats(self, reset: bool = False) -> dict:
        """Pairs the fp32 filters left undecided and fp64 re-tested (process-wide)."""
        a, b = C.c_int64(), C.c_int64()
        self._check(library().rgg_gpu_filter_stats(self._h, C.byref(a), C.byref(b), int(reset)))
        return {"sat_rechecks": a.value, "seg_rechecks": b.value}

    def exact_check(self, ids) -> np.ndarray:
        """exact_component_valid (roadmap.cpp:129-163) of ids: uint8 GREEN (free) / RED."""
        ids = np.ascontiguousarray(ids, np.int32)
        out = np.empty(len(ids), np.uint8)
        self._check(library().rgg_gpu_exact_check(self._h, ids.ctypes.data, len(ids), out.ctypes.data))
        return out

    def staging(self, n: int):
        """(ids int32[n], rts float64[n, 12]) views of the engine's pinned staging buffers
        (rgg_gpu_stage): moves written there go to the device without a host copy when passed
        to batch_update.  Valid until a larger batch grows the buffers."""
        pi, pr = C.POINTER(C.c_int32)(), C.POINTER(C.c_double)()
        self._check(library().rgg_gpu_stage(self._h, int(n), C.byref(pi), C.byref(pr)))
        ids = np.ctypeslib.as_array(pi, shape=(int(n),))
        rts = np.ctypeslib.as_array(pr, shape=(int(n), 12))
        return ids, rts

    def update_async(self, ids, rts):
        """Enqueue a lazy batch without waiting (timed device path)."""
        ids, rts = self._moves((ids, rts))
        self._check(library().rgg_gpu_update(self._h, ids.ctypes.data, rts.ctypes.data, len(ids),
                                             RGG_LAZY | RGG_ASYNC, None))

    def update_device(self, d_ids_ptr: int, d_rt_ptr: int, n: int, per_move: bool = False, census: bool = False,
                      gray_list: bool = False):
        """Enqueue a lazy batch whose moves are already in device memory (no host wait).
        gray_list: the GRAY-id compaction runs inside the update."""
        flags = (RGG_LAZY | (RGG_PER_MOVE if per_move else 0) | (RGG_CENSUS if census else 0)
                 | (RGG_GRAY_LIST if gray_list else 0))
        self._check(library().rgg_gpu_update_device(self._h, C.c_void_p(d_ids_ptr), C.c_void_p(d_rt_ptr), n, flags))

    def sync(self):
        self._check(library().rgg_gpu_sync(self._h))

    # torch-tensor entry points used by the multi-GPU driver (paper_2603_28674_b200/dist.py)
    def _torch_stream(self, device):
        import torch

        if getattr(self, "_ext", None) is None:
            self._ext = torch.cuda.ExternalStream(self.stream(), device=device)
        return self._ext

    def update_tensors(self, ids, rts, per_move: bool = True, gray_list: bool = False):
        """ids int32[n] / rts float64[n, 12] CUDA tensors, enqueued on the engine stream
        after the current torch stream's work (so a preceding broadcast is visible); no
        host synchronisation."""
        import torch

        self._torch_stream(ids.device).wait_stream(torch.cuda.current_stream(ids.device))
        self.update_device(ids.data_ptr(), rts.data_ptr(), int(ids.numel()), per_move=per_move, gray_list=gray_list)

    def gray_count_into(self, out):
        """The GRAY count of the last update (compacted with gray_list=True) into a CUDA
        int32 tensor (1,), ordered before the current torch stream's later work."""
        import torch

        # the engine stream writes `out`: order it after the current stream's use of that memory
        self._torch_stream(out.device).wait_stream(torch.cuda.current_stream(out.device))
        self._check(library().rgg_gpu_gray_device(self._h, C.c_void_p(out.data_ptr()), C.c_void_p(0), 0))
        torch.cuda.current_stream(out.device).wait_stream(self._torch_stream(out.device))

    def gray_ids_into(self, out, cap: int):
        """The first cap GRAY ids (ascending) of the last update into a CUDA int32 tensor,
        on the engine stream, ordered before the current torch stream's later work."""
        import torch

        self._torch_stream(out.device).wait_stream(torch.cuda.current_stream(out.device))
        self._check(library().rgg_gpu_gray_device(self._h, C.c_void_p(0), C.c_void_p(out.data_ptr()), int(cap)))
        torch.cuda.current_stream(out.device).wait_stream(self._torch_stream(out.device))

    def counters_into(self, out, n: int, check: bool = True):
        """Per-move counters of the last update into a CUDA int32 tensor (n, 4), ordered
        before the current torch stream's later work.  check: also wait for the update
        and raise its device-side errors (rgg_gpu_sync)."""
        import torch

        self.copy_counters(out.data_ptr(), n)
        torch.cuda.current_stream(out.device).wait_stream(self._torch_stream(out.device))
        if check:
            self.sync()

    def set_phase_timing(self, on: bool):
        """Per-kernel phase events in last_stats(); off lets the kernels overlap (PDL)."""
        self._check(library().rgg_gpu_set_phase_timing(self._h, int(bool(on))))

    def copy_counters(self, dst_ptr: int, n: int):
        """Per-move counters of the last update -> device buffer (n x 4 int32), engine stream."""
        self._check(library().rgg_gpu_copy_counters(self._h, C.c_void_p(dst_ptr), int(n)))

    @staticmethod
    def _moves(moves):
        if type(moves) is tuple and len(moves) == 2:  # fast path: the arrays as they come
            ids, rts = moves
            if (type(ids) is np.ndarray and type(rts) is np.ndarray and ids.dtype is _I32 and rts.dtype is _F64
                    and ids.ndim == 1 and rts.shape == (ids.shape[0], 12) and ids.flags.c_contiguous
                    and rts.flags.c_contiguous):
                return ids, rts
        if isinstance(moves, tuple) and len(moves) == 2 and not np.isscalar(moves[0]):
            ids, rts = moves
            if not (isinstance(ids, np.ndarray) and ids.dtype == np.int32 and ids.flags.c_contiguous):
                ids = np.ascontiguousarray(ids, dtype=np.int32)
            if not (isinstance(rts, np.ndarray) and rts.dtype == np.float64 and rts.flags.c_contiguous):
                rts = np.ascontiguousarray(rts, dtype=np.float64)
            ids = ids.reshape(-1)
            rts = rts.reshape(len(ids), 12)
        else:
            moves = list(moves)
            ids = np.array([int(o) for o, _ in moves], dtype=np.int32)
            rts = np.array([_pose12(p) for _, p in moves], dtype=np.float64).reshape(len(ids), 12)
        return ids, rts

    # -------------------------------------------------------------- queries
    def states(self) -> np.ndarray:
        out = np.empty(self.n_components, np.uint8)
        self._check(library().rgg_gpu_read_states(self._h, out.ctypes.data))
        return out

    def obstacle_bits(self) -> np.ndarray:
        out = np.empty(self.n_components * self.words, np.uint64)
        self._check(library().rgg_gpu_read_bits(self._h, out.ctypes.data, self.words))
        return out if self.words == 1 else out.reshape(self.n_components, self.words)

    def unknown_count(self) -> int:
        v = C.c_int32()
        self._check(library().rgg_gpu_unknown_count(self._h, C.byref(v)))
        return v.value

    def gray_ids(self) -> np.ndarray:
        n = C.c_int32()
        self._check(library().rgg_gpu_gray_ids(self._h, None, 0, C.byref(n)))
        out = np.empty(n.value, np.int32)
        if n.value:
            self._check(library().rgg_gpu_gray_ids(self._h, out.ctypes.data, n.value, C.byref(n)))
        return out

    def gray_ids_view(self) -> np.ndarray:
        """The GRAY ids (ascending) as a read-only view of the engine's pinned host buffer:
        one DMA, no copy; valid until the next call on this engine."""
        p = self._gv_p
        n = self._gv_n
        self._check(library().rgg_gpu_gray_view(self._h, C.byref(p), C.byref(n)))
        if n.value == 0:
            return np.zeros(0, np.int32)
        # a read-only array over the pointer (np.ctypeslib.as_array builds a ctypes type per call)
        return np.asarray(_ArrayView(C.cast(p, C.c_void_p).value, n.value))

    def last_hits(self) -> np.ndarray:
        n = C.c_int32()
        self._check(library().rgg_gpu_last_hits(self._h, None, 0, C.byref(n)))
        out = np.empty(n.value, np.int32)
        if n.value:
            self._check(library().rgg_gpu_last_hits(self._h, out.ctypes.data, n.value, C.byref(n)))
        return out

    def write_states(self, ids, st):
        ids = np.ascontiguousarray(ids, np.int32)
        st = np.ascontiguousarray(st, np.uint8)
        self._check(library().rgg_gpu_write_states(self._h, ids.ctypes.data, st.ctypes.data, len(ids)))

    def _mask(self, kind, candidates, o) -> np.ndarray:
        cands = np.ascontiguousarray(candidates, np.int32)
        out = np.zeros(len(cands), np.uint8)
        self._check(library().rgg_gpu_pair_masks(self._h, kind, cands.ctypes.data, len(cands), int(o),
                                                 out.ctypes.data))
        return out

    def batch_over(self, candidates: Sequence[int], o: int) -> np.ndarray:
        return self._mask(0, candidates, o)

    def batch_under(self, candidates: Sequence[int], o: int) -> np.ndarray:
        return self._mask(1, candidates, o)

    # ---------------------------------------------------------- measurement
    def last_stats(self) -> dict:
        s = Stats()
        self._check(library().rgg_gpu_last_stats(self._h, C.byref(s)))
        return s.as_dict()

    def census(self) -> dict:
        """Algorithmic census of the last update (flops of its narrow tests; bytes
        when that update ran with census=True)."""
        s = Stats()
        self._check(library().rgg_gpu_census(self._h, C.byref(s)))
        return s.as_dict()

    def stream(self) -> int:
        return library().rgg_gpu_stream(self._h) or 0


def fp64_peak_gflops(device: int = 0) -> float:
    v = C.c_double()
    rc = library().rgg_gpu_fp64_peak(device, C.byref(v))
    if rc != RGG_OK:
        raise RuntimeError(library().rgg_gpu_last_error(None).decode())
    return v.value


def fp32_peak_gflops(device: int = 0) -> float:
    """Measured FP32 FMA rate (GFLOP/s, 2 per FFMA) of `device`."""
    v = C.c_double()
    rc = library().rgg_gpu_fp32_peak(device, C.byref(v))
    if rc != RGG_OK:
        raise RuntimeError(library().rgg_gpu_last_error(None).decode())
    return v.value
