"""ctypes wrapper over the unmodified reference library (oracle/_ref/librgg_ref.so).

ORACLE / TEST INFRASTRUCTURE ONLY.  See oracle/ref_shim.cpp for the C entry
points and the reference file:line each one wraps.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "librgg_ref.so")

_lib = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_lp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_qp = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle library missing: {LIB_PATH} (run `make -C oracle`)")
        L = C.CDLL(LIB_PATH)
        L.rr_last_error.restype = C.c_char_p
        L.rr_world_from_scn.restype = C.c_void_p
        L.rr_world_from_scn.argtypes = [C.c_char_p]
        L.rr_world_from_roadmap.restype = C.c_void_p
        L.rr_world_from_roadmap.argtypes = [_dp, _dp, C.c_int, _dp, C.c_int, _ip, C.c_double, C.c_int]
        L.rr_world_add_obstacle.argtypes = [C.c_void_p, _dp, C.c_int]
        L.rr_world_free.argtypes = [C.c_void_p]
        L.rr_world_counts.argtypes = [C.c_void_p, _lp]
        L.rr_world_moves.argtypes = [C.c_void_p, _ip, _dp]
        L.rr_world_layout.argtypes = [C.c_void_p] + [C.c_void_p] * 11
        L.rr_world_obbs.argtypes = [C.c_void_p, _dp]
        L.rr_obstacle_operands.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.rr_engine_new.restype = C.c_void_p
        L.rr_engine_new.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.rr_engine_new_groups.restype = C.c_void_p
        L.rr_engine_new_groups.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.rr_engine_free.argtypes = [C.c_void_p]
        L.rr_engine_update.argtypes = [C.c_void_p, C.c_int32, _dp, C.c_int, _lp]
        L.rr_engine_run.argtypes = [C.c_void_p, C.c_int, _ip, _dp, C.c_int, C.POINTER(C.c_double)]
        L.rr_engine_run_parallel.argtypes = [C.c_void_p, C.c_int, _ip, _dp, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.rr_world_poses.argtypes = [C.c_void_p, _lp, C.c_void_p]
        L.rr_world_body_he.argtypes = [C.c_void_p, _dp]
        L.rr_world_from_robot.restype = C.c_void_p
        L.rr_world_from_robot.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, C.c_int, _dp, C.c_int, _ip,
                                          C.c_double, C.c_int]
        L.rr_world_robot.argtypes = [C.c_void_p, _ip] + [C.c_void_p] * 5
        L.rr_world_roadmap.argtypes = [C.c_void_p, _dp, _ip]
        L.rr_world_save.argtypes = [C.c_void_p, C.c_char_p]
        L.rr_box_intersect.argtypes = [_dp, _dp, _dp, _dp, C.POINTER(C.c_int)]
        L.rr_engine_exact.argtypes = [C.c_void_p, C.c_int, _ip, _up]
        L.rr_engine_resolve_all.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
        L.rr_engine_states.argtypes = [C.c_void_p, _up]
        L.rr_engine_bits.argtypes = [C.c_void_p, _qp]
        L.rr_engine_groups.argtypes = [C.c_void_p]
        L.rr_engine_mask.argtypes = [C.c_void_p, C.c_int, _ip, C.c_int, C.c_int32, _up]
        L.rr_kat_sat.argtypes = [C.c_uint64, C.c_int, C.c_int, _dp, _dp, _ip, _up, _dp, _dp]
        L.rr_kat_seg.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, _dp, _ip, _up]
        L.rr_kat_sat_pairs.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double, _dp, _dp, _up, _dp]
        L.rr_sat_prep.argtypes = [C.c_int, _dp, _dp]
        L.rr_tf_euler.argtypes = [C.c_double, C.c_double, C.c_double, _dp]
        L.rr_tf_axis_angle.argtypes = [_dp, C.c_double, _dp]
        L.rr_build_prm.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_longlong, C.POINTER(C.c_int), _dp, _dp,
                                   C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, _lp, C.POINTER(C.c_double)]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        msg = lib().rr_last_error().decode()
        if msg.startswith("invalid_argument"):
            raise ValueError(msg)
        raise RuntimeError(msg)


@dataclass
class Layout:
    """The serialized layout view (CSR over real segments), numpy arrays."""

    n_nodes: int
    n_edges: int
    N: int
    B: int
    S: int
    K: int
    M: int
    C: int
    edge_sat: np.ndarray  # N*B x 21
    e_plus: np.ndarray  # N*B x 24
    comp_aabb: np.ndarray  # N x 6
    row_off: np.ndarray  # N*B*S + 1
    segs: np.ndarray  # T x 7
    seg_pts: np.ndarray  # T x 6
    spline_r: np.ndarray  # B*S
    obst_he: np.ndarray  # M x 3
    obst_sph_local: np.ndarray  # M x C x 3
    obst_sph_r: np.ndarray  # M
    obst_sph_n: np.ndarray  # M


class World:
    """Reference roadmap + components + canonical obstacles."""

    def __init__(self, handle):
        if not handle:
            raise RuntimeError(lib().rr_last_error().decode())
        self.h = handle

    @classmethod
    def from_scn(cls, text: str) -> "World":
        return cls(lib().rr_world_from_scn(text.encode()))

    @classmethod
    def from_roadmap(cls, robot_he, env, nodes, edges, eps=0.25, max_segments=16) -> "World":
        nodes = np.ascontiguousarray(nodes, dtype=np.float64)
        edges = np.ascontiguousarray(edges, dtype=np.int32)
        h = lib().rr_world_from_roadmap(np.asarray(robot_he, np.float64), np.asarray(env, np.float64),
                                        nodes.shape[0], nodes.reshape(-1), edges.shape[0], edges.reshape(-1),
                                        float(eps), int(max_segments))
        return cls(h)

    @classmethod
    def from_robot(cls, robot: dict, env, nodes, edges, eps, max_segments=16) -> "World":
        """Any robot (robot.hpp:13-58) over an explicit roadmap: robot = {"kinematics":
        0 free flying / 1 serial chain, "he" (B, 3), "local" (B, 12), "axis" / "offset" (B, 3)}."""
        he = np.ascontiguousarray(robot["he"], np.float64).reshape(-1, 3)
        B = he.shape[0]
        loc = np.ascontiguousarray(robot["local"], np.float64).reshape(B, 12)
        ax = np.ascontiguousarray(robot.get("axis", np.zeros((B, 3))), np.float64).reshape(B, 3)
        off = np.ascontiguousarray(robot.get("offset", np.zeros((B, 3))), np.float64).reshape(B, 3)
        nodes = np.ascontiguousarray(nodes, dtype=np.float64)
        edges = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 2)
        h = lib().rr_world_from_robot(int(robot["kinematics"]), B, he.reshape(-1), loc.reshape(-1), ax.reshape(-1),
                                      off.reshape(-1), np.asarray(env, np.float64), nodes.shape[0], nodes.reshape(-1),
                                      edges.shape[0], edges.reshape(-1), float(eps), int(max_segments))
        return cls(h)

    def robot(self) -> dict:
        """The world's robot (the from_robot dict) plus its components' eps and max_segments."""
        meta = np.zeros(3, np.int32)
        _check(lib().rr_world_robot(self.h, meta, None, None, None, None, None))
        B = int(meta[1])
        he, loc, ax, off, ek = np.zeros((B, 3)), np.zeros((B, 12)), np.zeros((B, 3)), np.zeros((B, 3)), np.zeros(2)
        _check(lib().rr_world_robot(self.h, meta, *[a.ctypes.data for a in (he, loc, ax, off, ek)]))
        return dict(kinematics=int(meta[0]), dof=int(meta[2]), he=he, local=loc, axis=ax, offset=off,
                    eps=float(ek[0]), max_segments=int(ek[1]))

    def roadmap(self):
        """(nodes (n, dof), edges (e, 2))."""
        k = self.counts()
        dof = self.robot()["dof"]
        nodes = np.zeros((k["n_nodes"], dof))
        edges = np.zeros((k["n_edges"], 2), np.int32)
        _check(lib().rr_world_roadmap(self.h, nodes.reshape(-1), edges.reshape(-1)))
        return nodes, edges

    def save(self, path: str):
        """save_roadmap (roadmap_io.cpp:150-203): the world's robot, roadmap and components."""
        _check(lib().rr_world_save(self.h, str(path).encode()))

    def add_obstacle(self, he, spheres=0):
        _check(lib().rr_world_add_obstacle(self.h, np.asarray(he, np.float64), int(spheres)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.rr_world_free(self.h)
            self.h = None

    def counts(self):
        out = np.zeros(12, np.int64)
        _check(lib().rr_world_counts(self.h, out))
        keys = ["n_nodes", "n_edges", "N", "B", "S", "K", "M", "C", "segs", "n_moves", "iterations", "lazy"]
        return dict(zip(keys, out.tolist()))

    def moves(self):
        n = self.counts()["n_moves"]
        ids = np.zeros(n, np.int32)
        rt = np.zeros((n, 12), np.float64)
        _check(lib().rr_world_moves(self.h, ids, rt.reshape(-1)))
        return ids, rt

    def layout(self) -> Layout:
        k = self.counts()
        N, B, S, M, Cs, T = k["N"], k["B"], k["S"], k["M"], k["C"], k["segs"]
        a = dict(
            edge_sat=np.zeros((N * B, 21)), e_plus=np.zeros((N * B, 24)), comp_aabb=np.zeros((N, 6)),
            row_off=np.zeros(N * B * S + 1, np.int32), segs=np.zeros((T, 7)), seg_pts=np.zeros((T, 6)),
            spline_r=np.zeros(B * S), obst_he=np.zeros((M, 3)), obst_sph_local=np.zeros((M, Cs, 3)),
            obst_sph_r=np.zeros(M), obst_sph_n=np.zeros(M, np.int32))
        order = ["edge_sat", "e_plus", "comp_aabb", "row_off", "segs", "seg_pts", "spline_r", "obst_he",
                 "obst_sph_local", "obst_sph_r", "obst_sph_n"]
        _check(lib().rr_world_layout(self.h, *[a[n].ctypes.data_as(C.c_void_p) for n in order]))
        return Layout(n_nodes=k["n_nodes"], n_edges=k["n_edges"], N=N, B=B, S=S, K=k["K"], M=M, C=Cs, **a)

    def obbs(self):
        k = self.counts()
        out = np.zeros((k["N"] * k["B"], 15))
        _check(lib().rr_world_obbs(self.h, out.reshape(-1)))
        return out

    def poses(self):
        """(off int64[N+1], poses float64[total, B, 12]): forward_kinematics of every
        discretized configuration, the exact resolve's inputs (rr_world_poses)."""
        k = self.counts()
        off = np.zeros(k["N"] + 1, np.int64)
        _check(lib().rr_world_poses(self.h, off, None))
        poses = np.zeros((int(off[-1]), k["B"], 12))
        _check(lib().rr_world_poses(self.h, off, poses.ctypes.data_as(C.c_void_p)))
        return off, poses

    def body_half_extents(self):
        he = np.zeros((self.counts()["B"], 3))
        _check(lib().rr_world_body_he(self.h, he.reshape(-1)))
        return he

    def obstacle_operands(self, o: int, rt12):
        k = self.counts()
        sat, aabb, cen, saabb = np.zeros(21), np.zeros(6), np.zeros(k["C"] * 3), np.zeros(6)
        _check(lib().rr_obstacle_operands(self.h, int(o), np.asarray(rt12, np.float64), sat, aabb, cen, saabb))
        return sat, aabb, cen.reshape(-1, 3), saabb


def box_intersect(rt_a, he_a, rt_b, he_b) -> bool:
    """polytopes_intersect of two boxes (geometry.cpp:228-303)."""
    out = C.c_int(0)
    f = lambda x: np.ascontiguousarray(x, np.float64)
    _check(lib().rr_box_intersect(f(rt_a), f(he_a), f(rt_b), f(he_b), C.byref(out)))
    return bool(out.value)


class Engine:
    """Reference BatchEngine (kind=0) or SequentialEngine (kind=1), grouped for M > 64."""

    def __init__(self, world: World, kind=0, threads=1, use_under=True, cell_capacity=1024, group_size=64,
                 max_groups=-1):
        """max_groups >= 0: only the first max_groups obstacle groups (a bounded sample)."""
        self.world = world
        self.h = lib().rr_engine_new_groups(world.h, kind, threads, int(use_under), cell_capacity, group_size,
                                            int(max_groups))
        if not self.h:
            raise RuntimeError(lib().rr_last_error().decode())
        self.N = world.counts()["N"]
        self.groups = lib().rr_engine_groups(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.rr_engine_free(self.h)
            self.h = None

    def update(self, o, rt12, lazy=True):
        rep = np.zeros(11, np.int64)
        _check(lib().rr_engine_update(self.h, int(o), np.ascontiguousarray(rt12, np.float64), int(lazy), rep))
        return rep

    def exact_free(self, ids) -> np.ndarray:
        """exact_component_valid of ids at this engine's obstacle poses (1 = free)."""
        ids = np.ascontiguousarray(ids, np.int32)
        out = np.zeros(len(ids), np.uint8)
        _check(lib().rr_engine_exact(self.h, len(ids), ids, out))
        return out

    def resolve_all_unknown(self) -> int:
        n = C.c_int32(0)
        _check(lib().rr_engine_resolve_all(self.h, C.byref(n)))
        return n.value

    def run(self, ids, rts, lazy=True) -> float:
        ids = np.ascontiguousarray(ids, np.int32)
        rts = np.ascontiguousarray(rts, np.float64).reshape(-1)
        us = C.c_double(0)
        _check(lib().rr_engine_run(self.h, len(ids), ids, rts, int(lazy), C.byref(us)))
        return us.value

    def run_parallel(self, ids, rts, threads, lazy=True) -> float:
        """run() with the obstacle groups' engines on up to `threads` host threads."""
        ids = np.ascontiguousarray(ids, np.int32)
        rts = np.ascontiguousarray(rts, np.float64).reshape(-1)
        us = C.c_double(0)
        _check(lib().rr_engine_run_parallel(self.h, len(ids), ids, rts, int(lazy), int(threads), C.byref(us)))
        return us.value

    def states(self):
        out = np.zeros(self.N, np.uint8)
        _check(lib().rr_engine_states(self.h, out))
        return out

    def bits(self):
        out = np.zeros(self.N * self.groups, np.uint64)
        _check(lib().rr_engine_bits(self.h, out))
        return out.reshape(self.N, self.groups)

    def mask(self, kind, cands, o):
        cands = np.ascontiguousarray(cands, np.int32)
        out = np.zeros(len(cands), np.uint8)
        _check(lib().rr_engine_mask(self.h, kind, cands, len(cands), int(o), out))
        return out


def kat_sat(seed=2025, n_boxes=5000, n_idx=10000):
    boxes, obst, idx, out = np.zeros((n_boxes, 21)), np.zeros(21), np.zeros(n_idx, np.int32), np.zeros(n_idx, np.uint8)
    pose, he = np.zeros(12), np.zeros(3)
    _check(lib().rr_kat_sat(seed, n_boxes, n_idx, boxes.reshape(-1), obst, idx, out, pose, he))
    return boxes, obst, idx, out, pose, he


def kat_seg(seed=777, n_rand=4000, n_point=50, n_idx=9001):
    segs, idx, out = np.zeros((n_rand + n_point, 7)), np.zeros(n_idx, np.int32), np.zeros(n_idx, np.uint8)
    _check(lib().rr_kat_seg(seed, n_rand, n_point, n_idx, segs.reshape(-1), idx, out))
    return segs, idx, out


def kat_sat_pairs(seed, n, span=4.0, extent=2.0):
    a, b, out, margin = np.zeros((n, 21)), np.zeros((n, 21)), np.zeros(n, np.uint8), np.zeros(n)
    _check(lib().rr_kat_sat_pairs(seed, n, span, extent, a.reshape(-1), b.reshape(-1), out, margin))
    return a, b, out, margin


def tf_euler(rx, ry, rz):
    out = np.zeros(12)
    _check(lib().rr_tf_euler(rx, ry, rz, out))
    return out


def tf_axis_angle(axis, angle):
    out = np.zeros(12)
    _check(lib().rr_tf_axis_angle(np.asarray(axis, np.float64), angle, out))
    return out


def build_prm(scn_text: str, n_nodes: int = -1, k: int = -1, seed: int = -1):
    """The reference's build_prm (proj/src/roadmap.cpp:56-102) over a scenario's env and robot,
    no obstacles.  Returns (nodes n x dof, edges e x 2 int32, lo, hi, seconds)."""
    L = lib()
    dof = C.c_int(0)
    lo = np.zeros(64)
    hi = np.zeros(64)
    counts = np.zeros(2, np.int64)
    _check(L.rr_build_prm(scn_text.encode(), n_nodes, k, seed, C.byref(dof), lo, hi, None, 0, None, 0, counts,
                          None))
    D = dof.value
    nodes = np.zeros((max(1, int(counts[0])), D), np.float64)
    edges = np.zeros((max(1, int(counts[1])), 2), np.int32)
    sec = C.c_double(0)
    _check(L.rr_build_prm(scn_text.encode(), n_nodes, k, seed, C.byref(dof), lo, hi, nodes.ctypes.data,
                          len(nodes), edges.ctypes.data, len(edges), counts, C.byref(sec)))
    return nodes[:counts[0]].copy(), edges[:counts[1]].copy(), lo[:D].copy(), hi[:D].copy(), sec.value
