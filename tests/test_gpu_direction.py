"""Direction-optimising BFS (opt-in): bottom-up levels
must leave the visited set, the levels and the K6 layer records exactly as the
top-down BFS (the oracle's bfs_serial, traversal.py:80-104) has them; parents
may differ but must pass the certificate and the reference's validator."""

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle
from _util import pairs_arrays
from paper_1604_02844_b200 import (EdgeList, RmatParams, bfs, build_csr, build_lattice_graph, build_rmat_graph,
                                   pick_roots, validate_tree)

pytestmark = pytest.mark.gpu


@pytest.fixture
def every_level_bottom_up(monkeypatch):
    """Bitmap mode from the first edge and Beamer's switches pinned open, so
    every level after the root's runs bottom-up (read by the engine per BFS)."""
    monkeypatch.setenv("LBFS_BITMAP_MIN", "1")
    monkeypatch.setenv("LBFS_BITMAP_DIV", "1000000000")
    monkeypatch.setenv("LBFS_BU_ALPHA", "1000000000")
    monkeypatch.setenv("LBFS_BU_BETA", "1000000000")


def layers_of(res):
    return [(l.input, l.edges, l.discovered) for l in res.layers]


def check(g, s):
    rp, ci = g.colstarts, g.rows
    res = bfs(g, s, direction="optimizing")
    _, lvl, layers = oracle.bfs_serial(rp, ci, s)
    assert np.array_equal(res.levels, lvl)
    assert layers_of(res) == layers
    assert res.traversed_edge_count == sum(l[1] for l in layers)
    assert oracle.check_bfs(rp, ci, s, res.predecessors.p, res.levels) == (0, -1)
    assert validate_tree(g, s, res.predecessors).passed
    return res


def test_golden_small_graphs_bottom_up(golden, every_level_bottom_up):
    for name, gd in golden["small"].items():
        s_, d_ = pairs_arrays(gd["pairs"])
        g = build_csr(EdgeList(s_, d_, gd["n"]))
        for s in gd["bfs"]:
            res = check(g, int(s))
            assert res.levels.tolist() == gd["bfs"][s]["levels"], name


@pytest.mark.parametrize("deg", [1, 31, 32, 33, 1023, 1024, 1025, 5000])
def test_degree_bin_boundaries_bottom_up(deg, every_level_bottom_up):
    # a star of degree deg whose leaves chain on: hubs, warp rows and small rows
    pairs = [(0, i) for i in range(1, deg + 1)] + [(i, i + deg) for i in range(1, deg + 1)]
    s_, d_ = pairs_arrays(pairs)
    g = build_csr(EdgeList(s_, d_, 2 * deg + 2))
    for s in (0, 1, 2 * deg + 1):
        check(g, s)


@settings(max_examples=12, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(scale=st.integers(6, 13), seed=st.integers(1, 1000), data=st.data())
def test_rmat_bottom_up_matches_oracle(scale, seed, data, every_level_bottom_up):
    # (the fixture only sets environment variables: nothing to reset between examples)
    g = build_rmat_graph(RmatParams(scale=scale, edgefactor=16, seed=seed))
    roots = pick_roots(g, 2, seed, filter_unconnected=True).tolist()
    for s in roots:
        check(g, s)


def test_lattice_bottom_up(every_level_bottom_up):
    g = build_lattice_graph(64, 48)
    for s in pick_roots(g, 3, 1, filter_unconnected=True).tolist():
        check(g, s)


def test_default_rule_s20_and_s24_bit_exact_with_top_down():
    """Beamer's default switches (alpha 14, beta 24) on the benchmark graphs:
    same levels and layers as the top-down path, certified trees."""
    for scale, k in ((20, 4), (24, 2)):
        g = build_rmat_graph(RmatParams(scale=scale, seed=1))
        rp, ci = g.colstarts, g.rows
        for s in pick_roots(g, 64, 1, filter_unconnected=True).tolist()[:k]:
            td = bfs(g, s)
            do = bfs(g, s, direction="optimizing")
            assert np.array_equal(do.levels, td.levels)
            assert layers_of(do) == layers_of(td)
            assert oracle.check_bfs(rp, ci, s, do.predecessors.p, do.levels) == (0, -1)
            # the direction is per call: the next default call is top-down again
            assert layers_of(bfs(g, s)) == layers_of(td)


def test_unknown_direction_rejected():
    g = build_rmat_graph(RmatParams(scale=8, seed=1))
    with pytest.raises(AssertionError):
        bfs(g, 0, direction="sideways")
