"""ctypes wrapper over lib/librgg_build.so (csrc/producer.cpp): roadmap -> LayoutView.

The producer is the CPU step before the hot path.  It
follows the reference's preprocessing for a free-flying box robot so the
synthetic workloads of BASELINE.json configs 2-5 carry the reference's shapes
(fitted swept-volume OBBs, certified spline under-approximations).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .engine import LayoutView
from . import synth

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "librgg_build.so")
_lib = None


def library():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"producer not built: {LIB_PATH} (run `python -m paper_2603_28674_b200.build`)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.rgg_build_layout.argtypes = [vp, C.c_int32, vp, C.c_int32, vp, C.c_double, C.c_int32, C.c_int32,
                                       C.POINTER(vp)]
        L.rgg_build_layout_ex.argtypes = [vp, C.c_int32, vp, C.c_int32, vp, C.c_double, C.c_int32, C.c_int32,
                                          C.c_int32, C.POINTER(vp)]
        L.rgg_build_layout_robot.argtypes = [C.POINTER(_RobotView), C.c_int32, vp, C.c_int32, vp, C.c_double,
                                             C.c_int32, C.c_int32, C.c_int32, C.POINTER(vp)]
        L.rgg_built_poses.argtypes = [vp, vp, vp, vp]
        L.rgg_built_counts.argtypes = [vp, vp]
        L.rgg_built_export.argtypes = [vp] * 7
        L.rgg_built_save_roadmap.argtypes = [vp, C.c_char_p]
        L.rgg_built_free.argtypes = [vp]
        L.rgg_built_free.restype = None
        L.rgg_build_last_error.restype = C.c_char_p
        L.rgg_obstacle_spheres.argtypes = [vp, C.c_int32, vp, vp]
        L.rgg_build_gpu_count.restype = C.c_int
        L.rgg_roadmap_load.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.rgg_roadmap_counts.argtypes = [vp, vp]
        L.rgg_roadmap_components.argtypes = [vp] * 5
        L.rgg_roadmap_graph.argtypes = [vp] * 4
        L.rgg_roadmap_robot.argtypes = [vp] * 5
        L.rgg_roadmap_poses.argtypes = [vp] * 4
        L.rgg_roadmap_free.argtypes = [vp]
        L.rgg_roadmap_free.restype = None
        _lib = L
    return _lib


class _RobotView(C.Structure):
    _fields_ = [("kinematics", C.c_int32), ("n_bodies", C.c_int32), ("half_extents", C.c_void_p),
                ("local", C.c_void_p), ("joint_axis", C.c_void_p), ("joint_offset", C.c_void_p)]


FREE_FLYING, SERIAL_CHAIN = 0, 1


def free_flying(he) -> dict:
    """make_free_flying_box (proj/src/robot.cpp:86-92): one box body, identity local frame."""
    return dict(kinematics=FREE_FLYING, he=np.asarray(he, np.float64).reshape(1, 3))


def serial_chain(links) -> dict:
    """A serial chain as the scenario format's ``link`` lines (proj/src/scenario.cpp:144-157):
    per link (axis[3], offset[3], half extents[3], local translation[3])."""
    a = np.asarray(links, np.float64).reshape(-1, 12)
    loc = np.zeros((len(a), 12))
    loc[:, [0, 4, 8]] = 1.0
    loc[:, 9:] = a[:, 9:12]
    return dict(kinematics=SERIAL_CHAIN, axis=a[:, 0:3].copy(), offset=a[:, 3:6].copy(), he=a[:, 6:9].copy(), local=loc)


def robot_dof(robot: dict) -> int:
    return 6 if int(robot["kinematics"]) == FREE_FLYING else int(np.asarray(robot["he"]).reshape(-1, 3).shape[0])


def gpu_available() -> bool:
    return library().rgg_build_gpu_count() > 0


def build_layout(robot_he, nodes, edges, eps=0.25, max_segments=16, threads=0, with_obbs=False, with_poses=False,
                 gpu_fit=None, gpu_inner=False):
    """Components (nodes first, then edges) of a free-flying box robot -> store arrays
    (build_layout_robot with free_flying(robot_he))."""
    return build_layout_robot(free_flying(robot_he), nodes, edges, eps, max_segments, threads, with_obbs, with_poses,
                              gpu_fit, gpu_inner)


def build_layout_robot(robot: dict, nodes, edges, eps=0.25, max_segments=16, threads=0, with_obbs=False,
                       with_poses=False, gpu_fit=None, gpu_inner=False, save_roadmap=None):
    """build_components (proj/src/roadmap.cpp:104-127) + BatchLayout::serialize for any
    robot: ``robot`` = {"kinematics": FREE_FLYING | SERIAL_CHAIN, "he" (B, 3), optional
    "local" (B, 12), and for chains "axis" / "offset" (B, 3)}; nodes (n, dof).
    with_poses: also a["pose_off"] (N+1) and a["poses"] (configs, B, 12), the
    forward kinematics of every discretized configuration (GPU exact resolve).
    gpu_fit: the swept-volume box fit (obb_from_points, geometry.cpp:134-195) of every
    (component, body) on the GPU, bit-identical to the host fit (tests/test_gpu_producer.py);
    None (the default) = when a GPU is present.  save_roadmap: also write the build as the
    reference's binary roadmap file (save_roadmap, proj/src/roadmap_io.cpp:150-203) to this path."""
    L = library()
    if gpu_fit is None:
        gpu_fit = gpu_available()
    he = np.ascontiguousarray(robot["he"], np.float64).reshape(-1, 3)
    B = he.shape[0]
    arrs = [he]
    view = _RobotView(int(robot["kinematics"]), B, he.ctypes.data, None, None, None)
    for key, field, width in (("local", "local", 12), ("axis", "joint_axis", 3), ("offset", "joint_offset", 3)):
        if robot.get(key) is not None:
            a = np.ascontiguousarray(robot[key], np.float64).reshape(B, width)
            arrs.append(a)
            setattr(view, field, a.ctypes.data)
    dof = robot_dof(robot)
    nodes = np.ascontiguousarray(nodes, np.float64).reshape(-1, dof)
    edges = np.ascontiguousarray(edges, np.int32).reshape(-1, 2)
    h = C.c_void_p()
    rc = L.rgg_build_layout_robot(C.byref(view), len(nodes), nodes.ctypes.data, len(edges), edges.ctypes.data,
                                  float(eps), int(max_segments), int(threads),
                                  (1 if with_poses else 0) | (2 if gpu_fit else 0) | (4 if gpu_inner else 0)
                                  | (8 if save_roadmap else 0), C.byref(h))
    if rc != 0:
        raise RuntimeError(L.rgg_build_last_error().decode())
    try:
        if save_roadmap and L.rgg_built_save_roadmap(h, str(save_roadmap).encode()) != 0:
            raise RuntimeError(L.rgg_build_last_error().decode())
        cnt = np.zeros(4, np.int64)
        L.rgg_built_counts(h, cnt.ctypes.data)
        N, B, S, T = (int(x) for x in cnt)
        a = dict(edge_sat=np.empty((N * B, 21)), comp_aabb=np.empty((N, 6)), row_off=np.empty(N * B * S + 1, np.int32),
                 segs=np.empty((T, 7)), spline_r=np.empty(B * S), obb15=np.empty((N * B, 15)) if with_obbs else None)
        L.rgg_built_export(h, *[(v.ctypes.data if v is not None else None) for v in a.values()])
        if with_poses:
            nc = C.c_int64()
            if L.rgg_built_poses(h, C.byref(nc), None, None) != 0:
                raise RuntimeError(L.rgg_build_last_error().decode())
            a["pose_off"] = np.empty(N + 1, np.int64)
            a["poses"] = np.empty((nc.value, B, 12))
            L.rgg_built_poses(h, None, a["pose_off"].ctypes.data, a["poses"].ctypes.data)
    finally:
        L.rgg_built_free(h)
    return N, B, S, a


class RoadmapFileError(RuntimeError):
    """load_roadmap's RoadmapIoError (proj/include/rgg/roadmap_io.hpp:10-26): ``kind`` is one of
    "bad_magic", "bad_version", "truncated", "checksum", or "invalid" (an inconsistent file)."""

    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind


def load_roadmap(path, with_poses=False) -> dict:
    """The reference's binary roadmap file (load_roadmap, proj/src/roadmap_io.cpp:205-301), read
    and verified by ``rgg_roadmap_load`` straight into the component view of
    ``rgg_gpu_create_from_components``: keys N, B, S, e_plus (obb corners, N*B x 24), row_off,
    seg_pts (T x 6), spline_r, nodes (n, dof), edges (e, 2), eps, max_segments, robot (the
    ``build_layout_robot`` dict); with_poses: pose_off, poses (configs, B, 12) for the resolver."""
    L = library()
    h = C.c_void_p()
    rc = L.rgg_roadmap_load(str(path).encode(), C.byref(h))
    if rc != 0:
        kinds = {1: "bad_magic", 2: "bad_version", 3: "truncated", 4: "checksum"}
        raise RoadmapFileError(kinds.get(rc, "invalid"), L.rgg_build_last_error().decode())
    try:
        cnt = np.zeros(9, np.int64)
        L.rgg_roadmap_counts(h, cnt.ctypes.data)
        n_nodes, n_edges, dof, N, B, S, T, kin, K = (int(x) for x in cnt)
        out = dict(N=N, B=B, S=S, max_segments=K, e_plus=np.empty((N * B, 24)),
                   row_off=np.empty(N * B * S + 1, np.int32), seg_pts=np.empty((T, 6)), spline_r=np.empty(B * S),
                   nodes=np.empty((n_nodes, dof)), edges=np.empty((n_edges, 2), np.int32))
        L.rgg_roadmap_components(h, out["e_plus"].ctypes.data, out["row_off"].ctypes.data,
                                 out["seg_pts"].ctypes.data, out["spline_r"].ctypes.data)
        eps = C.c_double()
        L.rgg_roadmap_graph(h, out["nodes"].ctypes.data, out["edges"].ctypes.data, C.byref(eps))
        out["eps"] = eps.value
        robot = dict(kinematics=kin, he=np.empty((B, 3)), local=np.empty((B, 12)),
                     axis=np.zeros((B, 3)), offset=np.zeros((B, 3)))
        L.rgg_roadmap_robot(h, robot["he"].ctypes.data, robot["local"].ctypes.data,
                            robot["axis"].ctypes.data if kin == SERIAL_CHAIN else None,
                            robot["offset"].ctypes.data if kin == SERIAL_CHAIN else None)
        out["robot"] = robot
        if with_poses:
            nc = C.c_int64()
            off = np.empty(N + 1, np.int64)
            if L.rgg_roadmap_poses(h, C.byref(nc), off.ctypes.data, None) != 0:
                raise RoadmapFileError("invalid", L.rgg_build_last_error().decode())
            poses = np.empty((nc.value, B, 12))
            L.rgg_roadmap_poses(h, None, off.ctypes.data, poses.ctypes.data)
            out["pose_off"], out["poses"] = off, poses
    finally:
        L.rgg_roadmap_free(h)
    return out


def component_view(rf: dict, obstacles: synth.Obstacles):
    """A loaded roadmap file plus obstacles (box half extents and default sphere counts, as
    make_box_obstacle builds them) -> the view ``GpuEngine(view, components=True)`` takes."""
    from types import SimpleNamespace

    M = len(obstacles.he)
    Cmax = int(obstacles.spheres.max()) if M else 1
    sl = np.zeros((M, Cmax, 3))
    sr = np.zeros(M)
    for o in range(M):
        cen, r = obstacle_spheres(obstacles.he[o], obstacles.spheres[o])
        sl[o, : len(cen)] = cen
        sr[o] = r
    return SimpleNamespace(N=rf["N"], B=rf["B"], S=rf["S"], M=M, C=Cmax, e_plus=rf["e_plus"], row_off=rf["row_off"],
                           seg_pts=rf["seg_pts"], spline_r=rf["spline_r"],
                           obst_he=np.ascontiguousarray(obstacles.he, np.float64), obst_sph_local=sl, obst_sph_r=sr,
                           obst_sph_n=np.ascontiguousarray(obstacles.spheres, np.int32))


def obstacle_spheres(he, count):
    """obstacle_inner_spheres (proj/src/swept.cpp:23-49)."""
    cen = np.zeros((int(count), 3))
    r = C.c_double()
    rc = library().rgg_obstacle_spheres(np.ascontiguousarray(he, np.float64).ctypes.data, int(count),
                                        cen.ctypes.data, C.byref(r))
    if rc != 0:
        raise RuntimeError(library().rgg_build_last_error().decode())
    return cen, r.value


def layout_for(roadmap: synth.Roadmap, obstacles: synth.Obstacles, threads=0, with_poses=False,
               gpu_fit=None) -> LayoutView:
    """with_poses: the view also carries .resolver = (pose_off, poses, body_half_extents)
    for GpuEngine.set_resolver."""
    N, B, S, a = build_layout(roadmap.robot_he, roadmap.nodes, roadmap.edges, roadmap.eps, roadmap.max_segments,
                              threads, with_poses=with_poses, gpu_fit=gpu_fit)
    M = len(obstacles.he)
    Cmax = int(obstacles.spheres.max()) if M else 1
    sl = np.zeros((M, Cmax, 3))
    sr = np.zeros(M)
    for o in range(M):
        cen, r = obstacle_spheres(obstacles.he[o], obstacles.spheres[o])
        sl[o, : len(cen)] = cen
        sr[o] = r
    lv = LayoutView(N=N, B=B, S=S, M=M, C=Cmax, edge_sat=a["edge_sat"], comp_aabb=a["comp_aabb"],
                    row_off=a["row_off"], segs=a["segs"], spline_r=a["spline_r"],
                    obst_he=np.ascontiguousarray(obstacles.he, np.float64), obst_sph_local=sl, obst_sph_r=sr,
                    obst_sph_n=np.ascontiguousarray(obstacles.spheres, np.int32),
                    meta=dict(n_nodes=len(roadmap.nodes), n_edges=len(roadmap.edges)))
    if with_poses:
        lv.resolver = (a["pose_off"], a["poses"], np.asarray(roadmap.robot_he, np.float64).reshape(1, 3))
    return lv


def workload(name: str, seed: int = 12345, iterations: int = 1, threads: int = 0, scale: float = 1.0):
    """BASELINE config name ("c2".."c5") -> (LayoutView, roadmap, obstacles, ids, rt12)."""
    kind, nodes, k, half, m, ohalf = synth.CONFIGS[name]
    nodes = max(16, int(nodes * scale))
    half = half * np.sqrt(scale) if kind == "se2" else half * scale ** (1 / 3)
    ohalf = ohalf * np.sqrt(scale) if kind == "se2" else ohalf * scale ** (1 / 3)
    rm = synth.make_roadmap(kind, nodes, k, half, seed)
    obs = synth.make_obstacles(kind, m, seed + 1)
    lv = layout_for(rm, obs, threads)
    ids, rts = synth.make_moves(kind, m, iterations, ohalf, seed + 2)
    return lv, rm, obs, ids, rts
