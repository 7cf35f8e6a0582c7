"""The BASELINE.json configs on the device, against the reference's golden
vectors (S16, S20, S24, lattices) and the pinned oracle at full size."""

import numpy as np
import pytest

import oracle
from _util import sha
from paper_1604_02844_b200 import RmatParams, bfs, build_lattice_graph, build_rmat_graph, pick_roots
from paper_1604_02844_b200.traversal import SENTINEL
from paper_1604_02844_b200.validate import validate_tree_device

pytestmark = pytest.mark.gpu


def layers_of(res):
    return [[l.input, l.edges, l.discovered] for l in res.layers]


def test_config_s16_all_roots_bit_exact(golden, golden_arrays):
    # configs[0]: SCALE 16, 8 roots; levels bit-exact vs the reference's bfs_serial
    info = golden["S16"]
    g = build_rmat_graph(RmatParams(scale=16, seed=1))
    assert pick_roots(g, 8, 1, filter_unconnected=True).tolist() == info["roots"]
    for r, want in info["bfs"].items():
        res = bfs(g, int(r))
        assert np.array_equal(res.levels, golden_arrays[f"S16_levels_{r}"].astype(np.int32))
        assert layers_of(res) == want["layers"]
        assert res.traversed_edge_count == want["edges"]
        code, where = oracle.check_bfs(g.colstarts, g.rows, int(r), res.predecessors.p, res.levels)
        assert code == 0, (oracle.CHECK_CODES[code], where)


def test_config_s20_64_roots(golden):
    info = golden["S20"]
    g = build_rmat_graph(RmatParams(scale=20, seed=1))
    rp, ci = g.colstarts, g.rows
    roots = pick_roots(g, 64, 1, filter_unconnected=True).tolist()
    assert roots == info["roots"]
    for r in roots:
        res = bfs(g, r)
        want = info["bfs"].get(str(r))
        if want:
            assert layers_of(res) == want["layers"]
            assert sha(res.levels, "<i4") == want["levels_sha"]
        code, where = oracle.check_bfs(rp, ci, r, res.predecessors.p, res.levels)
        assert code == 0, (r, oracle.CHECK_CODES[code], where)
    # 8 roots against the oracle's own levels
    for r in roots[:8]:
        _, lvl, layers = oracle.bfs_parallel(rp, ci, r)
        res = bfs(g, r)
        assert np.array_equal(res.levels, lvl) and layers_of(res) == [list(x) for x in layers]


def test_config_lattice_small(golden):
    info = golden["lattice_64x48"]
    g = build_lattice_graph(64, 48)
    for r, want in info["bfs"].items():
        res = bfs(g, int(r))
        assert layers_of(res) == want["layers"]
        assert sha(res.levels, "<i4") == want["levels_sha"]


def test_config_lattice_4096_all_16_roots(golden):
    """BASELINE configs[3]: all 16 roots bit-exact with the oracle (levels and
    layers), the 2 roots the reference itself ran with its layer tallies,
    every tree through the device validator, 4 through the certificate."""
    info = golden["lattice_4096x4096"]
    g = build_lattice_graph(4096, 4096)
    rp, ci = g.colstarts, g.rows
    roots = pick_roots(g, 16, 1, filter_unconnected=True).tolist()
    assert roots == info["roots"]
    for i, r in enumerate(roots):
        res = bfs(g, r)
        _, lvl, layers = oracle.bfs_parallel(rp, ci, r)
        assert np.array_equal(res.levels, lvl), r
        assert layers_of(res) == [list(x) for x in layers], r
        assert validate_tree_device(g, r, res.predecessors).passed, r
        if str(r) in info["bfs"]:
            assert layers_of(res) == info["bfs"][str(r)]["layers"]
        if i < 4:
            assert oracle.check_bfs(rp, ci, r, res.predecessors.p, res.levels) == (0, -1), r


def test_config_s24_all_64_roots(golden):
    """BASELINE configs[2]: every one of the 64 benchmark roots. Levels and
    layers bit-exact with the oracle's bfs_parallel (pinned to the reference
    at S4-S20) and, for the 4 roots make_golden.py ran through the reference
    itself at S24 (bfs_vectorized + levels_from_parents), with the reference's
    layer tallies and level-array hash; every tree passes the reference's five
    validate_tree checks on the device, 8 of them the O(E) BFS certificate."""
    info = golden["S24"]
    g = build_rmat_graph(RmatParams(scale=24, seed=1))
    rp, ci = g.colstarts, g.rows
    roots = pick_roots(g, 64, 1, filter_unconnected=True).tolist()
    assert roots == info["roots"]
    for i, r in enumerate(roots):
        res = bfs(g, r)
        _, lvl, layers = oracle.bfs_parallel(rp, ci, r)
        assert np.array_equal(res.levels, lvl), r
        assert layers_of(res) == [list(x) for x in layers], r
        assert res.traversed_edge_count == sum(x[1] for x in layers)
        assert validate_tree_device(g, r, res.predecessors).passed, r
        if str(r) in info["bfs"]:
            want = info["bfs"][str(r)]
            assert layers_of(res) == want["layers"]
            assert sha(res.levels, "<i4") == want["levels_sha"]
            assert int((res.predecessors.p != SENTINEL).sum()) == want["reached"]
        if i < 8:
            assert oracle.check_bfs(rp, ci, r, res.predecessors.p, res.levels) == (0, -1), r


@pytest.fixture(params=["dsmem", "global"])
def all_levels_on_cluster(request, monkeypatch):
    """Every level on the thread-block cluster (cluster.cu), its visited
    bitmap in distributed shared memory or in global memory (read when the
    graph handle is created)."""
    monkeypatch.setenv("LBFS_CLUSTER_EDGES", str(1 << 40))
    if request.param == "global":
        monkeypatch.setenv("LBFS_CLUSTER_GLOBAL", "1")


@pytest.fixture
def no_cluster(monkeypatch):
    """Every level on the whole GPU (host-driven queue / bitmap levels)."""
    monkeypatch.setenv("LBFS_NO_CLUSTER", "1")


def test_cluster_every_level_s16_golden(golden, golden_arrays, all_levels_on_cluster):
    info = golden["S16"]
    g = build_rmat_graph(RmatParams(scale=16, seed=1))
    for r, want in info["bfs"].items():
        res = bfs(g, int(r))
        assert np.array_equal(res.levels, golden_arrays[f"S16_levels_{r}"].astype(np.int32))
        assert layers_of(res) == want["layers"]
        code, where = oracle.check_bfs(g.colstarts, g.rows, int(r), res.predecessors.p, res.levels)
        assert code == 0, (oracle.CHECK_CODES[code], where)


def test_cluster_every_level_s20_and_lattice(golden, all_levels_on_cluster):
    info = golden["S20"]
    g = build_rmat_graph(RmatParams(scale=20, seed=1))
    rp, ci = g.colstarts, g.rows
    for r in info["roots"][:8]:
        res = bfs(g, r)
        want = info["bfs"].get(str(r))
        if want:
            assert layers_of(res) == want["layers"]
            assert sha(res.levels, "<i4") == want["levels_sha"]
        code, where = oracle.check_bfs(rp, ci, r, res.predecessors.p, res.levels)
        assert code == 0, (r, oracle.CHECK_CODES[code], where)
    info = golden["lattice_64x48"]
    g = build_lattice_graph(64, 48)
    for r, want in info["bfs"].items():
        res = bfs(g, int(r))
        assert layers_of(res) == want["layers"]
        assert sha(res.levels, "<i4") == want["levels_sha"]


def test_no_cluster_s20_and_lattice(golden, no_cluster):
    info = golden["S20"]
    g = build_rmat_graph(RmatParams(scale=20, seed=1))
    rp, ci = g.colstarts, g.rows
    for r in info["roots"][:4]:
        res = bfs(g, r)
        want = info["bfs"].get(str(r))
        if want:
            assert layers_of(res) == want["layers"]
            assert sha(res.levels, "<i4") == want["levels_sha"]
        assert oracle.check_bfs(rp, ci, r, res.predecessors.p, res.levels) == (0, -1)
    info = golden["lattice_64x48"]
    g = build_lattice_graph(64, 48)
    for r, want in info["bfs"].items():
        res = bfs(g, int(r))
        assert layers_of(res) == want["layers"]
        assert sha(res.levels, "<i4") == want["levels_sha"]


def test_config_s27_one_gpu_and_eight_partitions():
    """configs[4] (SCALE 27, ~4.2e9 CSR entries; the reference cannot build it,
    SURVEY G5) on ONE B200: device construction, BFS from seeded roots
    certified on the host (root, parent one level up and adjacent, every
    edge spans <= 1 level: levels are exact BFS distances), the device
    validator, and the 8-way 1D partition of the multi-GPU config driven in
    lockstep on this GPU, bit-exact with the single-GPU levels and layers."""
    from paper_1604_02844_b200.distributed import LocalExchange, PartitionedGraph, bfs_partitioned
    from paper_1604_02844_b200.validate import validate_tree_device

    g = build_rmat_graph(RmatParams(scale=27, seed=1))
    n = g.num_vertices
    assert n == 1 << 27 and g.num_edges > (1 << 31)  # past int32 offsets
    roots = pick_roots(g, 64, 1, filter_unconnected=True).tolist()[:2]
    rp, ci = g.colstarts, g.rows
    singles = {}
    for r in roots:
        res = bfs(g, r)
        assert res.traversed_edge_count == sum(l.edges for l in res.layers)
        code, where = oracle.check_bfs(rp, ci, r, res.predecessors.p, res.levels)
        assert code == 0, (r, oracle.CHECK_CODES[code], where)
        assert validate_tree_device(g, r, res.predecessors).passed
        singles[r] = res
    parts = [PartitionedGraph(g, k, 8) for k in range(8)]
    r = roots[0]
    pr = bfs_partitioned(parts, r, LocalExchange())
    assert layers_of(pr) == layers_of(singles[r])
    assert np.array_equal(pr.level[0].cpu().numpy()[:n], singles[r].levels)
    code, where = oracle.check_bfs(rp, ci, r, pr.pred[0].cpu().numpy()[:n], pr.level[0].cpu().numpy()[:n])
    assert code == 0, (oracle.CHECK_CODES[code], where)
