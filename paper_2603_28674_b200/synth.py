"""Synthetic roadmaps, obstacle sets and move scripts of the BASELINE.json shapes.

The reference ships no generator for configs 2-5; these follow
the survey's definitions:

* ``se2``  — free-flying box robot, half extents (0.5, 0.3, 0.25), nodes uniform on
  xy in [-L, L]^2 with z = 0, yaw U(-pi, pi), other rotations 0; k-nearest
  neighbours in the reference's 6-DOF Euclidean metric (proj/src/roadmap.cpp:36-43,
  :78-90) with unique (min, max) pairs (:91-93).  Obstacles: half extents
  (U(0.3,1.5), U(0.3,1.5), 1.0), default sphere count (proj/src/swept.cpp:51-55),
  poses yaw U(-pi, pi), xy uniform, z = 0.
* ``3d``   — same robot, nodes uniform in [-L, L]^3 with three Euler angles
  U(-pi, pi); obstacles half extents U(0.3,1.5)^3, yaw-rotated, uniform positions.

Nodes come first then edges (component id = node id, then n_nodes + edge,
proj/include/rgg/roadmap.hpp:53-55).  The kNN uses scipy's cKDTree instead of the
reference's O(n^2) scan (SURVEY.md §7 "hard parts"): same neighbour sets up to
distance ties.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ROBOT_HE = (0.5, 0.3, 0.25)


@dataclass
class Roadmap:
    kind: str
    env: np.ndarray  # 6: min xyz, max xyz
    nodes: np.ndarray  # n x 6 (x, y, z, rx, ry, rz)
    edges: np.ndarray  # e x 2 int32, first < second
    robot_he: tuple = ROBOT_HE
    eps: float = 0.25
    max_segments: int = 16

    @property
    def n_components(self) -> int:
        return len(self.nodes) + len(self.edges)


def knn_edges(nodes: np.ndarray, k: int) -> np.ndarray:
    from scipy.spatial import cKDTree

    tree = cKDTree(nodes)
    kk = min(k + 1, len(nodes))
    _, nb = tree.query(nodes, k=kk)
    nb = np.asarray(nb).reshape(len(nodes), kk)
    i = np.repeat(np.arange(len(nodes)), kk - 1)
    j = nb[:, 1:].reshape(-1)
    keep = j != i
    i, j = i[keep], j[keep]
    pairs = np.stack([np.minimum(i, j), np.maximum(i, j)], 1).astype(np.int64)
    pairs = np.unique(pairs[:, 0] * len(nodes) + pairs[:, 1])
    return np.stack([pairs // len(nodes), pairs % len(nodes)], 1).astype(np.int32)


def make_roadmap(kind: str, n_nodes: int, k: int, half: float, seed: int, z_half: float | None = None) -> Roadmap:
    rng = np.random.default_rng(seed)
    nodes = np.zeros((n_nodes, 6))
    if kind == "se2":
        nodes[:, 0] = rng.uniform(-half, half, n_nodes)
        nodes[:, 1] = rng.uniform(-half, half, n_nodes)
        nodes[:, 5] = rng.uniform(-np.pi, np.pi, n_nodes)
        zh = 1.0 if z_half is None else z_half
        env = np.array([-half - 1, -half - 1, -zh, half + 1, half + 1, zh], np.float64)
    elif kind == "3d":
        nodes[:, 0:3] = rng.uniform(-half, half, (n_nodes, 3))
        nodes[:, 3:6] = rng.uniform(-np.pi, np.pi, (n_nodes, 3))
        env = np.array([-half - 1] * 3 + [half + 1] * 3, np.float64)
    else:
        raise ValueError(kind)
    return Roadmap(kind=kind, env=env, nodes=nodes, edges=knn_edges(nodes, k))


def rot_z(yaw: np.ndarray) -> np.ndarray:
    c, s = np.cos(yaw), np.sin(yaw)
    r = np.zeros(yaw.shape + (9,))
    r[..., 0], r[..., 1], r[..., 3], r[..., 4], r[..., 8] = c, -s, s, c, 1.0
    return r


@dataclass
class Obstacles:
    he: np.ndarray  # M x 3
    spheres: np.ndarray  # M (sphere counts)


def default_sphere_count(he: np.ndarray) -> np.ndarray:
    """proj/src/swept.cpp:51-55: max(1, ceil(longest / shortest))."""
    return np.maximum(1, np.ceil(he.max(1) / he.min(1))).astype(np.int32)


def make_obstacles(kind: str, m: int, seed: int) -> Obstacles:
    rng = np.random.default_rng(seed)
    he = rng.uniform(0.3, 1.5, (m, 3))
    if kind == "se2":
        he[:, 2] = 1.0
    return Obstacles(he=he, spheres=default_sphere_count(he))


def make_moves(kind: str, m: int, iterations: int, half: float, seed: int, ids=None):
    """Move script: every iteration re-poses every obstacle (or ``ids``) — the
    shape of Scenario::make_moves (proj/src/scenario.cpp:25-40) with the
    survey's yaw-rotated poses.  Returns (ids int32[n], rt12 float64[n, 12])."""
    rng = np.random.default_rng(seed)
    order = np.arange(m, dtype=np.int32) if ids is None else np.asarray(ids, np.int32)
    n = iterations * len(order)
    out_ids = np.tile(order, iterations)
    rt = np.zeros((n, 12))
    rt[:, :9] = rot_z(rng.uniform(-np.pi, np.pi, n))
    rt[:, 9] = rng.uniform(-half, half, n)
    rt[:, 10] = rng.uniform(-half, half, n)
    if kind == "3d":
        rt[:, 11] = rng.uniform(-half, half, n)
    return out_ids, rt


CONFIGS = {
    # name: (kind, nodes, k, half extent of the node box, obstacles, obstacle box half)
    "c2": ("se2", 10_000, 20, 24.0, 64, 25.0),
    "c3": ("3d", 50_000, 18, 9.0, 256, 10.0),
    "c4": ("se2", 87_000, 20, 71.0, 64, 72.0),
    "c5": ("se2", 87_000, 20, 71.0, 1024, 72.0),
}

# Moves per update where a config moves only a subset of its obstacles (BASELINE configs[3]:
# incremental updates dirtying ~5 % of the cells: 7 of the 64 obstacles, each dirtying the
# cells under its old and new box, about 5 % of the 8,406 128-component cells; bench.py reports
# the measured dirty_fraction); the subset rotates through all obstacles.
MOVES_PER_STEP = {"c4": 7}
