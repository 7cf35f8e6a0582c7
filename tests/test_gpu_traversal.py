"""Device BFS parity, mirroring the reference's tests/test_traversal.py:
bit-exact levels and layers against the oracle (itself pinned to the
reference), predecessor trees that pass the tree check, and the edge cases
of the degree bins (thread/warp/CTA, hub chunking, padding)."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle
from _util import pairs_arrays
from paper_1604_02844_b200 import (
    SENTINEL,
    EdgeList,
    LayerPolicy,
    LayerStats,
    RmatParams,
    bfs,
    build_csr,
    build_rmat_graph,
    generate_rmat,
    levels_from_parents,
    run_bfs,
    validate_tree,
)

pytestmark = pytest.mark.gpu


def graph(pairs, n, symmetrize=True, dedup=True):
    s, d = pairs_arrays(pairs)
    return build_csr(EdgeList(s, d, n), symmetrize, dedup)


def check_against_oracle(g, s):
    res = bfs(g, s)
    rp, ci = g.colstarts, g.rows
    _, lvl, layers = oracle.bfs_serial(rp, ci, s)
    assert np.array_equal(res.levels, lvl)
    assert [(l.input, l.edges, l.discovered) for l in res.layers] == layers
    assert res.traversed_edge_count == sum(l[1] for l in layers)
    assert oracle.check_bfs(rp, ci, s, res.predecessors.p, res.levels) == (0, -1)
    assert len(res.predecessors.storage) % 32 == 0
    assert (res.predecessors.storage[g.num_vertices:] == SENTINEL).all()
    return res


def test_path_graph_exact():
    res = bfs(graph([(0, 1), (1, 2)], 3), 0)
    assert res.predecessors.p.tolist() == [0, 0, 1]  # unique tree
    assert res.layers == [LayerStats(1, 1, 1), LayerStats(1, 2, 1), LayerStats(1, 1, 0)]
    assert res.traversed_edge_count == 4
    assert res.levels.tolist() == [0, 1, 2]


def test_single_vertex():
    res = bfs(graph(np.empty((0, 2), np.uint32), 1), 0)
    assert res.predecessors.p.tolist() == [0]
    assert res.layers == [LayerStats(1, 0, 0)]


def test_root_out_of_range_rejected():
    g = graph([(0, 1), (1, 2)], 3)
    with pytest.raises(AssertionError):
        bfs(g, 3)
    with pytest.raises(AssertionError):
        bfs(g, -1)


def test_diamond_parent_is_either_middle():
    g = graph([(0, 1), (0, 2), (1, 3), (2, 3)], 4)
    for _ in range(5):
        res = bfs(g, 0)
        assert int(res.predecessors.p[3]) in (1, 2)
        assert levels_from_parents(res.predecessors.p, 0).tolist() == [0, 1, 1, 2]


def test_star_all_leaves_distance_one():
    g = graph([(0, i) for i in range(1, 101)], 101)
    res = bfs(g, 0)
    assert res.levels.tolist() == [0] + [1] * 100
    assert res.layers[0] == LayerStats(1, 100, 100)


def test_unreachable_keep_sentinel():
    k = 4
    pairs = [(i, j) for i in range(k) for j in range(i + 1, k)]
    pairs += [(k + i, k + j) for i in range(k) for j in range(i + 1, k)]
    res = bfs(graph(pairs, 2 * k), 1)
    p = res.predecessors.p
    assert (p[4:] == SENTINEL).all() and (p[:4] != SENTINEL).all()
    assert (res.levels[4:] == -1).all()
    assert sum(l.discovered for l in res.layers) == 3


def test_golden_small_graphs_levels_and_layers(golden):
    for name, gd in golden["small"].items():
        g = graph(gd["pairs"], gd["n"])
        for s, want in gd["bfs"].items():
            res = bfs(g, int(s))
            assert res.levels.tolist() == want["levels"], name
            assert [[l.input, l.edges, l.discovered] for l in res.layers] == want["layers"], name
            assert validate_tree(g, int(s), res.predecessors).passed


def test_children_sharing_a_word():
    res = bfs(graph([(0, 5), (0, 9)], 16), 0)
    assert int(res.predecessors.p[5]) == 0 and int(res.predecessors.p[9]) == 0
    assert res.levels.tolist() == [0, -1, -1, -1, -1, 1, -1, -1, -1, 1] + [-1] * 6


def test_isolated_root_and_empty_graph():
    g = graph(np.empty((0, 2), np.uint32), 7)
    for s in (0, 3, 6):
        res = bfs(g, s)
        assert res.layers == [LayerStats(1, 0, 0)] and res.traversed_edge_count == 0
        assert (res.levels == np.where(np.arange(7) == s, 0, -1)).all()


@pytest.mark.parametrize("deg", [1, 31, 32, 33, 4095, 4096, 4097, 8192, 8193, 100000])
def test_degree_bin_boundaries(deg):
    # hub 0 with `deg` leaves, each leaf also chained to the next (two levels)
    n = deg + 1
    pairs = [(0, i) for i in range(1, n)] + [(i, i + 1) for i in range(1, n - 1)]
    g = graph(pairs, n)
    check_against_oracle(g, 0)
    check_against_oracle(g, n - 1)


def test_two_level_hubs_and_unaligned_rows():
    # rows with every start offset mod 4 and lengths around the int4 body
    rng = np.random.default_rng(5)
    pairs = []
    n = 3000
    for u in range(0, n, 7):
        k = int(rng.integers(0, 300))
        pairs += [(u, int(v)) for v in rng.integers(0, n, k)]
    g = graph(pairs, n)
    for s in (0, 7, 14):
        check_against_oracle(g, s)


def test_repeated_bfs_on_one_handle_is_stateless():
    g = build_rmat_graph(RmatParams(scale=10, seed=4))
    a = bfs(g, 5)
    b = bfs(g, 700)
    c = bfs(g, 5)
    assert np.array_equal(a.levels, c.levels) and a.layers == c.layers


@settings(max_examples=25, deadline=None)
@given(scale=st.integers(4, 11), seed=st.integers(0, 1000), ef=st.sampled_from([1, 4, 8, 16]),
       data=st.data())
def test_levels_match_oracle_rmat(scale, seed, ef, data):
    g = build_csr(generate_rmat(RmatParams(scale=scale, edgefactor=ef, seed=seed)))
    s = data.draw(st.integers(0, g.num_vertices - 1))
    check_against_oracle(g, s)


def test_layer_accounting_invariants():
    g = build_rmat_graph(RmatParams(scale=12, seed=5))
    res = bfs(g, 3)
    reached = int((res.predecessors.p != SENTINEL).sum())
    assert sum(l.discovered for l in res.layers) == reached - 1
    assert sum(l.input for l in res.layers) == reached
    assert res.traversed_edge_count == int(g.degrees()[res.levels >= 0].sum())
    hist = np.bincount(res.levels[res.levels >= 0])
    assert hist.tolist() == [l.input for l in res.layers]


def test_run_bfs_dispatch_all_modes_same_levels():
    g = build_rmat_graph(RmatParams(scale=9, seed=2))
    want = bfs(g, 1).levels
    for mode in ("gpu", "serial", "parallel_naive", "parallel_restored", "vectorized"):
        assert np.array_equal(run_bfs(g, 1, LayerPolicy(mode=mode), threads=2).levels, want)


def test_foreign_graph_object_is_accepted():
    # a plain object with the reference CsrGraph attributes (graph.py:96-110)
    rp, ci = oracle.build_csr(64, *oracle.rmat_edges(6, 8, seed=3))

    class RefLike:
        __slots__ = ("num_vertices", "rows", "colstarts")

    g = RefLike()
    g.num_vertices, g.rows, g.colstarts = 64, ci, rp
    res = bfs(g, 0)
    _, lvl, _ = oracle.bfs_serial(rp, ci, 0)
    assert np.array_equal(res.levels, lvl)


def test_bfs_device_torch_outputs():
    import torch

    from paper_1604_02844_b200 import bfs_device

    g = build_rmat_graph(RmatParams(scale=11, seed=1))
    n = g.num_vertices
    pred = torch.empty((n + 31) // 32 * 32, dtype=torch.int32, device="cuda")
    lvl = torch.empty(n, dtype=torch.int32, device="cuda")
    res = bfs_device(g, 17, pred, lvl)
    ref = bfs(g, 17)
    assert np.array_equal(lvl.cpu().numpy(), ref.levels)
    assert res.layers == ref.layers


@pytest.mark.parametrize("env", [
    {"LBFS_CLUSTER_MAIL_CAP": "4"},      # candidate mailboxes overflow: the remote-claim path next to them
    {"LBFS_CLUSTER_NO_MAIL": "1"},       # remote claims only
    {"LBFS_CLUSTER_GLOBAL": "1"},        # claims on the global bitmap
    {"LBFS_CLUSTER_DSM_ALWAYS": "1"},    # late segments with the bitmap in DSMEM too
    {"LBFS_NO_WARP_ITEMS": "1", "LBFS_NO_FUSE_QUEUES": "1", "LBFS_NO_PUBLISH_AFTER_HEAVY": "1"},
    {"LBFS_NO_EXIT_FAIR": "1", "LBFS_QGRID_OLD": "1", "LBFS_RESOLVE_CLAMP": "1"},
    {"LBFS_DENSE_MIN": "0"},             # dense small-region streaming on small graphs too
])
def test_level_loop_switches_keep_the_results(monkeypatch, env):
    """The A/B switches of the level loop (read once per graph handle) select
    other code paths, never other results: levels and layers against the
    oracle on a lattice (thousands of cluster levels), R-MAT graphs whose
    levels cross every mode, and a hub-heavy star-of-stars."""
    from paper_1604_02844_b200 import build_lattice_graph, pick_roots

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = build_lattice_graph(192, 160)
    for r in pick_roots(g, 2, 3, filter_unconnected=True).tolist():
        check_against_oracle(g, int(r))
    for scale in (12, 16, 18):
        g = build_rmat_graph(RmatParams(scale=scale, edgefactor=16, seed=5))
        for r in pick_roots(g, 3, 7, filter_unconnected=True).tolist():
            check_against_oracle(g, int(r))
    # two hubs of 3000 and 2000 leaves joined by a path, leaves sharing bitmap sectors
    pairs = [(0, 10 + i) for i in range(3000)] + [(1, 4000 + i) for i in range(2000)] + [(0, 2), (2, 3), (3, 1)]
    check_against_oracle(graph(pairs, 6100), 10)
