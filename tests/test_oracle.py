"""Pin the CPU oracle (oracle/) to the reference's own outputs.

Golden vectors come from tests/golden/make_golden.py, which ran the reference
package lanebfs 0.1.0 (/root/reference/pkg/src) in the build container."""

import numpy as np
import pytest

import oracle
from _util import layers_tuples, oracle_csr_from_pairs, pairs_arrays, sha


def test_small_graph_csr_all_flag_combinations(golden):
    # build_csr(symmetrize, dedup) graph.py:139-160 — exact arrays
    for name, g in golden["small"].items():
        for key, want in g["csr"].items():
            sym, dd = bool(int(key[0])), bool(int(key[1]))
            rp, ci = oracle_csr_from_pairs(g["pairs"], g["n"], sym, dd)
            assert rp.tolist() == want["colstarts"], (name, key)
            assert ci.tolist() == want["rows"], (name, key)


def test_small_graph_serial_bfs_exact(golden):
    # bfs_serial traversal.py:80-104: exact preds (first discoverer), layers, levels
    for name, g in golden["small"].items():
        rp, ci = oracle_csr_from_pairs(g["pairs"], g["n"])
        for s, want in g["bfs"].items():
            pred, level, layers = oracle.bfs_serial(rp, ci, int(s))
            assert pred.tolist() == want["pred"], name
            assert [list(x) for x in layers] == want["layers"], name
            assert level.tolist() == want["levels"], name
            assert sum(l[1] for l in layers) == want["edges"]


def test_known_answers():
    # test_traversal.py:46-57, test_graph.py:83-88
    rp, ci = oracle_csr_from_pairs([(0, 1), (1, 2)], 3)
    pred, level, layers = oracle.bfs_serial(rp, ci, 0)
    assert pred.tolist() == [0, 0, 1]
    assert layers == [(1, 1, 1), (1, 2, 1), (1, 1, 0)]
    rp, ci = oracle_csr_from_pairs([(0, 1), (1, 2), (2, 0)], 3)
    assert rp.tolist() == [0, 2, 4, 6] and ci.tolist() == [1, 2, 0, 2, 0, 1]
    rp, ci = oracle.build_csr(1, np.empty(0, np.uint32), np.empty(0, np.uint32))
    pred, level, layers = oracle.bfs_serial(rp, ci, 0)
    assert pred.tolist() == [0] and layers == [(1, 0, 0)]


def test_rmat_small_generator_csr_and_bfs(golden, golden_arrays):
    for item in golden["rmat_small"]:
        s, d = oracle.rmat_edges(item["scale"], item["edgefactor"], seed=item["seed"])
        key = f"s{item['scale']}_e{item['edgefactor']}_r{item['seed']}"
        assert sha(s, "<u4") == item["src_sha"] and sha(d, "<u4") == item["dst_sha"], key
        if f"{key}_src" in golden_arrays:
            assert np.array_equal(s, golden_arrays[f"{key}_src"])
        rp, ci = oracle.build_csr(1 << item["scale"], s, d)
        assert len(ci) == item["nnz"]
        assert sha(rp, "<i8") == item["colstarts_sha"] and sha(ci, "<i4") == item["rows_sha"], key
        for root, want in item["bfs"].items():
            pred, level, layers = oracle.bfs_serial(rp, ci, int(root))
            assert sha(pred, "<i4") == want["pred_sha"], (key, root)
            assert [list(x) for x in layers] == want["layers"]
            assert sha(level, "<i4") == want["levels_sha"]
            p2, l2, layers2 = oracle.bfs_parallel(rp, ci, int(root), 4)
            assert np.array_equal(l2, level) and layers2 == layers
            assert oracle.check_bfs(rp, ci, int(root), p2, l2) == (0, -1)


def _config_graph(info, scale):
    s, d = oracle.rmat_edges(scale, 16, seed=1)
    assert sha(s, "<u4") == info["src_sha"] and sha(d, "<u4") == info["dst_sha"]
    ps, pd = oracle.permute_edges(1 << scale, 1, s, d)
    assert sha(ps, "<u4") == info["psrc_sha"] and sha(pd, "<u4") == info["pdst_sha"]
    rp, ci = oracle.build_csr(1 << scale, ps, pd)
    assert len(ci) == info["nnz"]
    assert sha(rp, "<i8") == info["colstarts_sha"] and sha(ci, "<i4") == info["rows_sha"]
    return rp, ci


def test_config_s16_oracle(golden, golden_arrays):
    info = golden["S16"]
    rp, ci = _config_graph(info, 16)
    roots = oracle.pick_roots(np.diff(rp), 8, 1, True)
    assert roots.tolist() == info["roots"]
    for r, want in info["bfs"].items():
        pred, level, layers = oracle.bfs_serial(rp, ci, int(r))
        assert sha(pred, "<i4") == want["pred_sha"]
        assert [list(x) for x in layers] == want["layers"]
        assert np.array_equal(level, golden_arrays[f"S16_levels_{r}"].astype(np.int32))
        assert want["validate_passed"]


@pytest.mark.slow
def test_config_s20_oracle(golden):
    info = golden["S20"]
    rp, ci = _config_graph(info, 20)
    assert oracle.pick_roots(np.diff(rp), 64, 1, True).tolist() == info["roots"]
    for r, want in info["bfs"].items():
        pred, level, layers = oracle.bfs_parallel(rp, ci, int(r))
        assert [list(x) for x in layers] == want["layers"]
        assert sha(level, "<i4") == want["levels_sha"]
        assert oracle.check_bfs(rp, ci, int(r), pred, level) == (0, -1)


def test_lattice_small_oracle(golden):
    info = golden["lattice_64x48"]
    s, d = oracle.lattice_edges(64, 48)
    assert sha(s, "<u4") == info["src_sha"]
    ps, pd = oracle.permute_edges(64 * 48, 1, s, d)
    assert sha(ps, "<u4") == info["psrc_sha"] and sha(pd, "<u4") == info["pdst_sha"]
    rp, ci = oracle.build_csr(64 * 48, ps, pd)
    assert sha(rp, "<i8") == info["colstarts_sha"] and sha(ci, "<i4") == info["rows_sha"]
    assert oracle.pick_roots(np.diff(rp), 4, 1, True).tolist() == info["roots"]
    for r, want in info["bfs"].items():
        pred, level, layers = oracle.bfs_serial(rp, ci, int(r))
        assert [list(x) for x in layers] == want["layers"]
        assert sha(level, "<i4") == want["levels_sha"]


@pytest.mark.slow
def test_lattice_4096_oracle(golden):
    info = golden["lattice_4096x4096"]
    n = 4096 * 4096
    s, d = oracle.lattice_edges(4096, 4096)
    ps, pd = oracle.permute_edges(n, 1, s, d)
    assert sha(ps, "<u4") == info["psrc_sha"]
    rp, ci = oracle.build_csr(n, ps, pd)
    assert len(ci) == info["nnz"] == 67092480
    assert sha(rp, "<i8") == info["colstarts_sha"] and sha(ci, "<i4") == info["rows_sha"]
    assert oracle.pick_roots(np.diff(rp), 16, 1, True).tolist() == info["roots"]
    r, want = next(iter(info["bfs"].items()))
    pred, level, layers = oracle.bfs_parallel(rp, ci, int(r))
    assert [list(x) for x in layers] == want["layers"]


def test_levels_from_parents_oracle_matches_reference(golden):
    for case in golden["validator"]["cases"]:
        got = oracle.levels_from_parents(np.array(case["pred"]), case["root"])
        assert got.tolist() == case["levels"], case["variant"]


def test_harmonic_mean(golden):
    for c in golden["harmonic"]:
        if not c["include_zeros"]:
            assert oracle.harmonic_mean_teps(c["values"]) == pytest.approx(c["result"][0])


def test_permutation_is_a_bijection():
    for n in (1, 2, 3, 5, 33, 100, 1024, 4097):
        img = [oracle.permute_vertex(n, 7, v) for v in range(n)]
        assert sorted(img) == list(range(n))
