"""PRM construction: build_prm (proj/src/roadmap.cpp:56-102) of a scene
without active obstacles.

CPU: the oracle restatement (oracle/rgg_oracle.c ro_prm_*) against tests/golden/prm.npz, dumped
from the unmodified reference (oracle/gen_golden.py prm), and the product's host node sampler
(rgg_prm_nodes) against the same fixtures.
GPU: the kNN (csrc/rgg_prm.cu) against the fixtures, against the oracle on tie-heavy lattices,
generic DOF counts, k >= n-1 and larger random sets, and the reference's argument errors
(proj/tests/test_roadmap.cpp:45-51).
"""
import hashlib

import numpy as np
import pytest

from oracle import oracle as O
from paper_2603_28674_b200 import prm

from conftest import load_golden


def _cases():
    g = load_golden("prm")
    out = []
    for name in g["names"]:
        n, k, seed, dof, ne = (int(x) for x in g[f"{name}__meta"])
        c = dict(name=str(name), n=n, k=k, seed=seed, dof=dof, ne=ne, lo=g[f"{name}__lo"], hi=g[f"{name}__hi"])
        if f"{name}__nodes" in g:
            c["nodes"], c["edges"] = g[f"{name}__nodes"], g[f"{name}__edges"]
        else:
            c["sha_nodes"], c["sha_edges"] = bytes(g[f"{name}__sha_nodes"]), bytes(g[f"{name}__sha_edges"])
        out.append(c)
    return out


CASES = _cases()
SMALL = [c for c in CASES if "nodes" in c]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest()


@pytest.mark.parametrize("c", SMALL, ids=[c["name"] for c in SMALL])
def test_oracle_matches_reference_prm(c):
    nodes = O.prm_nodes(c["seed"], c["n"], c["lo"], c["hi"])
    assert np.array_equal(nodes.view(np.uint64), c["nodes"].view(np.uint64))
    assert np.array_equal(O.prm_knn(nodes, c["k"]), c["edges"])


def test_free_flying_bounds_match_reference():
    """dof_bounds_for (roadmap.cpp:20-30) as the reference returned it for the cube scenes."""
    c = next(c for c in CASES if c["name"].startswith("cube_"))
    lo, hi = prm.dof_bounds_free_flying([-10, -10, -10, 10, 10, 10])
    assert np.array_equal(lo, c["lo"]) and np.array_equal(hi, c["hi"])
    m = next(c for c in CASES if c["name"].startswith("table5"))  # serial chain, 6 joints
    lo, hi = prm.dof_bounds_serial_chain(m["dof"])
    assert np.array_equal(lo, m["lo"]) and np.array_equal(hi, m["hi"])


@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_host_node_sampler_matches_reference(c):
    nodes = prm.sample_nodes(c["seed"], c["n"], c["lo"], c["hi"])
    if "nodes" in c:
        assert np.array_equal(nodes.view(np.uint64), c["nodes"].view(np.uint64))
    else:
        assert _sha(nodes) == c["sha_nodes"]


def test_node_sampler_errors():
    with pytest.raises(ValueError, match="node count"):
        prm.sample_nodes(7, 0, [0.0], [1.0])


# ------------------------------------------------------------------------------ GPU


@pytest.mark.gpu
@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_gpu_build_prm_matches_reference(c):
    nodes, edges = prm.build_prm(c["lo"], c["hi"], c["n"], c["k"], c["seed"])
    assert len(edges) == c["ne"]
    if "nodes" in c:
        assert np.array_equal(nodes.view(np.uint64), c["nodes"].view(np.uint64))
        assert np.array_equal(edges, c["edges"])
    else:  # table3_roadmap_10000: digests of the reference's 10,000 nodes / 49,737 edges
        assert _sha(nodes) == c["sha_nodes"] and _sha(edges) == c["sha_edges"]


@pytest.mark.gpu
@pytest.mark.parametrize("n,dof,k,step", [(700, 2, 8, 1.0), (1500, 3, 12, 0.5), (900, 6, 20, 1.0)])
def test_gpu_knn_ties_on_lattices(n, dof, k, step):
    """Integer lattices: many equal distances, so the id tie-break of partial_sort on
    pair<double, NodeId> (roadmap.cpp:87) decides the neighbour sets; duplicates included."""
    rng = np.random.default_rng(n + dof)
    nodes = rng.integers(0, 6, (n, dof)).astype(np.float64) * step
    assert np.array_equal(prm.knn_edges(nodes, k), O.prm_knn(nodes, k))


@pytest.mark.gpu
@pytest.mark.parametrize("dof", [1, 4, 7, 12])
def test_gpu_knn_generic_dof(dof):
    rng = np.random.default_rng(dof)
    nodes = rng.uniform(-3, 3, (1200, dof))
    assert np.array_equal(prm.knn_edges(nodes, 9), O.prm_knn(nodes, 9))


@pytest.mark.gpu
@pytest.mark.parametrize("n,k", [(1, 4), (2, 1), (5, 4), (5, 50), (40, 39), (500, 600)])
def test_gpu_knn_small_and_k_at_least_n(n, k):
    """k >= n-1 connects every pair (min(k, n-1), roadmap.cpp:86); one node has no edges
    (proj/tests/test_roadmap.cpp:45-48)."""
    nodes = np.random.default_rng(n * 100 + k).uniform(-1, 1, (n, 6))
    got = prm.knn_edges(nodes, k)
    assert np.array_equal(got, O.prm_knn(nodes, k))
    if k >= n - 1:
        assert len(got) == n * (n - 1) // 2


@pytest.mark.gpu
@pytest.mark.parametrize("n,k", [(20000, 20), (6000, 100)])
def test_gpu_knn_larger_random(n, k):
    """The candidate range split over CTAs and merged (csrc/rgg_prm.cu merge_kernel)."""
    lo, hi = prm.dof_bounds_free_flying([-30, -30, -1, 30, 30, 1])
    nodes = prm.sample_nodes(99, n, lo, hi)
    assert np.array_equal(prm.knn_edges(nodes, k), O.prm_knn(nodes, k))


@pytest.mark.gpu
@pytest.mark.parametrize("scale", [1e-300, 1e-8, 1e12, 1e20])
def test_gpu_knn_filter_extremes(scale):
    """The fp32 pre-filter's bound (csrc/rgg_prm.cu filter_bound) at tiny, large and
    fp32-overflowing magnitudes (the last disables it), with near-duplicate nodes."""
    rng = np.random.default_rng(int(np.log10(scale)) + 400)
    base = rng.uniform(-1, 1, (300, 6))
    nodes = np.concatenate([base, base + rng.uniform(-1e-9, 1e-9, base.shape)]) * scale
    assert np.array_equal(prm.knn_edges(nodes, 7), O.prm_knn(nodes, 7))


@pytest.mark.gpu
def test_gpu_prm_errors():
    """std::invalid_argument cases of build_prm (proj/tests/test_roadmap.cpp:45-51)."""
    lo, hi = prm.dof_bounds_free_flying([-1, -1, -1, 1, 1, 1])
    with pytest.raises(ValueError, match="node count"):
        prm.build_prm(lo, hi, 0, 4, 7)
    with pytest.raises(ValueError, match="neighbor count"):
        prm.build_prm(lo, hi, 10, 0, 7)
    with pytest.raises(ValueError, match="neighbor count"):
        prm.knn_edges(np.zeros((3, 6)), 0)
    with pytest.raises(ValueError, match="512"):
        prm.knn_edges(np.zeros((1000, 3)), 600)
