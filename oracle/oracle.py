"""ctypes wrapper over librgg_oracle.so — our plain-C restatement (rgg_oracle.c).

ORACLE / TEST INFRASTRUCTURE ONLY.  Parity pinned against the reference's golden
vectors by tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librgg_oracle.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_lp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_qp = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


class _View(C.Structure):
    _fields_ = [("n_components", C.c_int32), ("n_bodies", C.c_int32), ("n_slots", C.c_int32),
                ("n_obstacles", C.c_int32), ("max_spheres", C.c_int32),
                ("edge_sat", C.c_void_p), ("comp_aabb", C.c_void_p), ("row_off", C.c_void_p),
                ("segs", C.c_void_p), ("spline_radius", C.c_void_p), ("obst_he", C.c_void_p),
                ("obst_sph_local", C.c_void_p), ("obst_sph_r", C.c_void_p), ("obst_sph_n", C.c_void_p)]


_lib = None


def build():
    subprocess.check_call(["make", "-s", "-C", HERE, "librgg_oracle.so"])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.ro_sat_prep.argtypes = [_dp, _dp]
        L.ro_sat_boxes.argtypes = [_dp, _dp]
        L.ro_sat_cost.argtypes = [_dp, _dp]
        L.ro_seg_prep.argtypes = [_dp, _dp]
        L.ro_seg_point_dist.restype = C.c_double
        L.ro_seg_point_dist.argtypes = [_dp, _dp]
        L.ro_seg_sphere.argtypes = [_dp, _dp, C.c_double]
        L.ro_sat_batch.argtypes = [_dp, _ip, C.c_int, _dp, _up]
        L.ro_seg_sphere_batch.argtypes = [_dp, _ip, C.c_int, _dp, C.c_double, _up]
        L.ro_obstacle_operands.argtypes = [_dp, _dp, C.c_int, C.c_double, _dp, _dp, _dp, _dp, _dp]
        L.ro_engine_new.restype = C.c_void_p
        L.ro_box_intersect.argtypes = [_dp, _dp, _dp, _dp]
        L.ro_exact_valid.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_int, _up, _dp, _dp]
        L.ro_engine_new.argtypes = [C.POINTER(_View), C.c_int]
        L.ro_engine_free.argtypes = [C.c_void_p]
        L.ro_engine_words.argtypes = [C.c_void_p]
        L.ro_engine_update.argtypes = [C.c_void_p, C.c_int32, _dp, _lp]
        L.ro_engine_states.argtypes = [C.c_void_p, _up]
        L.ro_engine_bits.argtypes = [C.c_void_p, _qp]
        L.ro_engine_unknown.argtypes = [C.c_void_p]
        L.ro_engine_pure.argtypes = [C.c_void_p, _up, _qp]
        L.ro_engine_mask.argtypes = [C.c_void_p, C.c_int, _ip, C.c_int, C.c_int32, _up]
        L.ro_engine_census.argtypes = [C.c_void_p, _lp]
        L.ro_prm_nodes.argtypes = [C.c_uint64, C.c_int, C.c_int, _dp, _dp, _dp]
        L.ro_prm_knn.restype = C.c_int64
        L.ro_prm_knn.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _ip, C.c_int64]
        _lib = L
    return _lib


def sat_prep(corners24):
    out = np.zeros(21)
    lib().ro_sat_prep(np.ascontiguousarray(corners24, np.float64), out)
    return out


def sat_batch(boxes, idx, obstacle):
    idx = np.ascontiguousarray(idx, np.int32)
    out = np.zeros(len(idx), np.uint8)
    lib().ro_sat_batch(np.ascontiguousarray(boxes, np.float64).reshape(-1), idx, len(idx),
                       np.ascontiguousarray(obstacle, np.float64), out)
    return out


def sat_boxes(a, b) -> bool:
    return bool(lib().ro_sat_boxes(np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)))


def sat_cost(a, b) -> int:
    return int(lib().ro_sat_cost(np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)))


def seg_prep(seg6):
    out = np.zeros(7)
    lib().ro_seg_prep(np.ascontiguousarray(seg6, np.float64), out)
    return out


def seg_sphere_batch(segs, idx, c3, r_total):
    idx = np.ascontiguousarray(idx, np.int32)
    out = np.zeros(len(idx), np.uint8)
    lib().ro_seg_sphere_batch(np.ascontiguousarray(segs, np.float64).reshape(-1), idx, len(idx),
                              np.ascontiguousarray(c3, np.float64), float(r_total), out)
    return out


def obstacle_operands(he, sph_local, n_sph, sph_r, rt12):
    sph_local = np.ascontiguousarray(sph_local, np.float64).reshape(-1)
    sat, aabb, cen, saabb = np.zeros(21), np.zeros(6), np.zeros(max(1, len(sph_local))), np.zeros(6)
    lib().ro_obstacle_operands(np.ascontiguousarray(he, np.float64), sph_local if len(sph_local) else np.zeros(3),
                               int(n_sph), float(sph_r), np.ascontiguousarray(rt12, np.float64), sat, aabb, cen, saabb)
    return sat, aabb, cen[: 3 * n_sph].reshape(-1, 3), saabb


def box_intersect(rt_a, he_a, rt_b, he_b) -> bool:
    f = lambda x: np.ascontiguousarray(x, np.float64)
    return bool(lib().ro_box_intersect(f(rt_a), f(he_a), f(rt_b), f(he_b)))


def exact_valid(poses, body_he, active, obst_rt, obst_he) -> bool:
    """exact_component_valid of one component: poses (configs, B, 12)."""
    poses = np.ascontiguousarray(poses, np.float64)
    body_he = np.ascontiguousarray(body_he, np.float64).reshape(-1)
    return bool(lib().ro_exact_valid(poses.shape[0], poses.shape[1], poses.reshape(-1), body_he, len(active),
                                     np.ascontiguousarray(active, np.uint8),
                                     np.ascontiguousarray(obst_rt, np.float64).reshape(-1),
                                     np.ascontiguousarray(obst_he, np.float64).reshape(-1)))


class Engine:
    """Lazy-mode BatchEngine restated in C over a layout view (any object with
    the attributes of oracle.ref.Layout or paper_2603_28674_b200.layout.LayoutView)."""

    def __init__(self, layout, use_under=True):
        keep = {}

        def arr(name, dt):
            a = np.ascontiguousarray(getattr(layout, name), dtype=dt)
            keep[name] = a
            return a.ctypes.data

        self._keep = keep
        v = _View(int(layout.N), int(layout.B), int(layout.S), int(layout.M), int(layout.C),
                  arr("edge_sat", np.float64), arr("comp_aabb", np.float64), arr("row_off", np.int32),
                  arr("segs", np.float64), arr("spline_r", np.float64), arr("obst_he", np.float64),
                  arr("obst_sph_local", np.float64), arr("obst_sph_r", np.float64), arr("obst_sph_n", np.int32))
        self._view = v
        self.h = lib().ro_engine_new(C.byref(v), int(use_under))
        self.N = int(layout.N)
        self.words = lib().ro_engine_words(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ro_engine_free(self.h)
            self.h = None

    def update(self, o, rt12):
        rep = np.zeros(4, np.int64)
        rc = lib().ro_engine_update(self.h, int(o), np.ascontiguousarray(rt12, np.float64), rep)
        if rc != 0:
            raise ValueError("unknown obstacle id")
        return rep

    def states(self):
        out = np.zeros(self.N, np.uint8)
        lib().ro_engine_states(self.h, out)
        return out

    def bits(self):
        out = np.zeros(self.N * self.words, np.uint64)
        lib().ro_engine_bits(self.h, out)
        return out.reshape(self.N, self.words)

    def unknown(self):
        return int(lib().ro_engine_unknown(self.h))

    def pure(self):
        st = np.zeros(self.N, np.uint8)
        bits = np.zeros(self.N * self.words, np.uint64)
        lib().ro_engine_pure(self.h, st, bits)
        return st, bits.reshape(self.N, self.words)

    def mask(self, kind, cands, o):
        cands = np.ascontiguousarray(cands, np.int32)
        out = np.zeros(len(cands), np.uint8)
        lib().ro_engine_mask(self.h, int(kind), cands, len(cands), int(o), out)
        return out

    def census(self):
        out = np.zeros(7, np.int64)
        lib().ro_engine_census(self.h, out)
        keys = ["over_pairs", "sat_flops", "under_pairs", "seg_sphere_tests", "over_hits", "under_hits", "active"]
        return dict(zip(keys, out.tolist()))


def prm_nodes(seed, n, lo, hi):
    """build_prm's node loop (proj/src/roadmap.cpp:65-71, no active obstacles)."""
    lo = np.ascontiguousarray(lo, np.float64)
    hi = np.ascontiguousarray(hi, np.float64)
    out = np.zeros((n, len(lo)), np.float64)
    lib().ro_prm_nodes(int(seed), int(n), len(lo), lo, hi, out)
    return out


def prm_knn(nodes, k):
    """build_prm's candidate loop (proj/src/roadmap.cpp:73-93): sorted unique (min, max) pairs."""
    nodes = np.ascontiguousarray(nodes, np.float64)
    n, dof = nodes.shape
    cap = max(1, n * max(0, min(k, n - 1)))
    out = np.zeros((cap, 2), np.int32)
    m = lib().ro_prm_knn(nodes, n, dof, int(k), out, cap)
    assert m >= 0
    return out[:m].copy()
