"""PRM construction with the kNN on the GPU, over lib/librgg_build.so
(csrc/rgg_prm.cu, include/rgg_prm.h).

Mirrors ``rgg::build_prm(scene, n_nodes, k_neighbors, eps, seed)`` (proj/src/roadmap.cpp:56-102)
for a scene without active obstacles — the build scene the reference's benchmark uses
(proj/src/bench.cpp:90-91) — with the same errors (``ValueError`` where the reference throws
``std::invalid_argument``).  Nodes and edges are bit-identical to the reference's
(tests/test_prm.py, tests/golden/prm.npz).
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import producer

RGG_PRM_EINVAL, RGG_PRM_ECUDA, RGG_PRM_ESPACE = 1, 2, 3
_bound = False


def library():
    global _bound
    L = producer.library()
    if not _bound:
        vp = C.c_void_p
        L.rgg_prm_nodes.argtypes = [C.c_uint64, C.c_int32, C.c_int32, vp, vp, vp]
        L.rgg_prm_knn_edges.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, vp, C.c_int64, C.POINTER(C.c_int64),
                                        C.POINTER(C.c_float)]
        L.rgg_prm_last_error.restype = C.c_char_p
        _bound = True
    return L


def _raise(L, rc):
    msg = L.rgg_prm_last_error().decode()
    raise (ValueError if rc == RGG_PRM_EINVAL else RuntimeError)(msg)


def dof_bounds_free_flying(env6):
    """dof_bounds_for (proj/src/roadmap.cpp:20-30), free-flying robot: the environment box, then
    [-pi, pi] for the three Euler angles."""
    env6 = np.asarray(env6, np.float64)
    lo = np.concatenate([env6[:3], [-math.pi] * 3])
    hi = np.concatenate([env6[3:6], [math.pi] * 3])
    return lo, hi


def dof_bounds_serial_chain(n_joints):
    """dof_bounds_for, serial chain: [-pi, pi] per joint."""
    return np.full(n_joints, -math.pi), np.full(n_joints, math.pi)


def sample_nodes(seed, n_nodes, lo, hi):
    """The node loop of build_prm (roadmap.cpp:65-71): n_nodes x dof uniforms from Rng(seed)."""
    L = library()
    lo = np.ascontiguousarray(lo, np.float64)
    hi = np.ascontiguousarray(hi, np.float64)
    if lo.shape != hi.shape or lo.ndim != 1:
        raise ValueError("lo and hi must be 1-D of the same length")
    if n_nodes < 1:
        raise ValueError("node count must be >= 1")
    out = np.empty((int(n_nodes), len(lo)), np.float64)
    rc = L.rgg_prm_nodes(int(seed) & 0xFFFFFFFFFFFFFFFF, int(n_nodes), len(lo), lo.ctypes.data, hi.ctypes.data,
                         out.ctypes.data)
    if rc:
        _raise(L, rc)
    return out


def knn_edges(nodes, k, return_ms=False):
    """The candidate loop of build_prm (roadmap.cpp:73-93) on the GPU: sorted unique (min, max)
    pairs of every node's k nearest nodes under dof_distance2.  Returns an (e, 2) int32 array
    (and the device milliseconds if return_ms)."""
    L = library()
    nodes = np.ascontiguousarray(nodes, np.float64)
    if nodes.ndim != 2:
        raise ValueError("nodes must be n x dof")
    n, dof = nodes.shape
    cap = max(1, n * max(0, min(int(k), n - 1)))
    out = np.empty((cap, 2), np.int32)
    ne = C.c_int64(0)
    ms = C.c_float(0)
    rc = L.rgg_prm_knn_edges(nodes.ctypes.data, n, dof, int(k), out.ctypes.data, cap, C.byref(ne), C.byref(ms))
    if rc:
        _raise(L, rc)
    edges = out[:ne.value].copy()
    return (edges, ms.value) if return_ms else edges


def build_prm(lo, hi, n_nodes, k_neighbors, seed):
    """build_prm of a scene without active obstacles: (nodes n x dof, edges e x 2)."""
    if n_nodes < 1:
        raise ValueError("node count must be >= 1")
    if k_neighbors < 1:
        raise ValueError("neighbor count must be >= 1")
    nodes = sample_nodes(seed, n_nodes, lo, hi)
    return nodes, knn_edges(nodes, k_neighbors)
