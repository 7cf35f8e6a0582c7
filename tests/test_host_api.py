"""Host-side pieces of the drop-in that need no GPU: the vectorised
validator, levels_from_parents, harness statistics and result types, checked
against the reference's own outputs (golden vectors)."""

import csv
import json

import numpy as np
import pytest

import oracle
from _util import oracle_csr_from_pairs
from paper_1604_02844_b200 import (
    SENTINEL,
    CsrGraph,
    EdgeList,
    ExperimentConfig,
    LayerStats,
    PredecessorArray,
    RmatParams,
    RootRun,
    RunStats,
    bfs_certificate,
    emit_results,
    harmonic_mean_teps,
    lattice_edges,
    levels_from_parents,
    pick_roots,
    read_edge_list,
    validate_tree,
    write_edge_list,
)


def _graph(entry):
    cs = np.array(entry["colstarts"], dtype=np.int64)
    rows = np.array(entry["rows"], dtype=np.int32)
    return CsrGraph(len(cs) - 1, rows, cs)


def test_validate_tree_matches_reference_on_mutation_catalog(golden):
    # validate.py:50-155 on the reference mutation catalog (helpers.py:57-149)
    graphs = {k: _graph(v) for k, v in golden["validator"]["graphs"].items()}
    for case in golden["validator"]["cases"]:
        g = graphs[case["graph"]]
        pred = PredecessorArray(g.num_vertices)
        pred.p[:] = case["pred"]
        got = validate_tree(g, case["root"], pred).as_dict()
        want = case["report"]
        want["details"] = {k: int(v) for k, v in want["details"].items()}
        assert got == want, (case["graph"], case["variant"])


def test_levels_from_parents_matches_reference(golden):
    for case in golden["validator"]["cases"]:
        got = levels_from_parents(np.array(case["pred"]), case["root"])
        assert got.tolist() == case["levels"], case["variant"]
    for name, g in golden["small"].items():
        for s, want in g["bfs"].items():
            assert levels_from_parents(np.array(want["pred"]), int(s)).tolist() == want["levels"]


def test_validate_tree_accepts_reference_serial_trees(golden):
    for name, g in golden["small"].items():
        cs, rows = oracle_csr_from_pairs(g["pairs"], g["n"])
        graph = CsrGraph(g["n"], rows, cs)
        for s, want in g["bfs"].items():
            pred = PredecessorArray(g["n"])
            pred.p[:] = want["pred"]
            assert validate_tree(graph, int(s), pred).passed, name
            cert = bfs_certificate(graph, int(s), pred, np.array(want["levels"]))
            assert cert.passed, (name, cert)


def test_certificate_rejects_wrong_levels():
    cs, rows = oracle_csr_from_pairs([(i, i + 1) for i in range(9)] + [(0, 9)], 10)
    g = CsrGraph(10, rows, cs)
    pred, level, _ = oracle.bfs_serial(cs, rows, 0)
    p = PredecessorArray(10)
    p.p[:] = pred
    assert bfs_certificate(g, 0, p, level).passed
    bad = level.copy()
    bad[5] += 2
    assert not bfs_certificate(g, 0, p, bad).passed
    q = PredecessorArray(10)
    q.p[:] = pred
    q.p[3] = 7  # not adjacent
    assert not bfs_certificate(g, 0, q, level).passed


def test_validator_unsorted_rows_dedup_false(golden):
    e = golden["small"]["dups_loops"]["csr"]["10"]
    g = CsrGraph(len(e["colstarts"]) - 1, np.array(e["rows"], np.int32), np.array(e["colstarts"], np.int64))
    pred = PredecessorArray(g.num_vertices)
    pred.p[:] = [0, 0, 1, SENTINEL, SENTINEL]
    assert validate_tree(g, 0, pred).passed


def test_harmonic_mean_matches_reference(golden):
    for c in golden["harmonic"]:
        got = harmonic_mean_teps(c["values"], c["include_zeros"])
        assert got[0] == pytest.approx(c["result"][0]) and list(got[1:]) == c["result"][1:]
    with pytest.raises(AssertionError):
        harmonic_mean_teps([])


def test_pick_roots_matches_reference(golden):
    cs, rows = oracle.build_csr(64 * 48, *oracle.permute_edges(64 * 48, 1, *oracle.lattice_edges(64, 48)))
    g = CsrGraph(64 * 48, rows, cs)
    assert pick_roots(g, 4, 1, True).tolist() == golden["lattice_64x48"]["roots"]
    with pytest.raises(AssertionError):
        pick_roots(g, 64 * 48 + 1, 1)


def test_lattice_edges_match_oracle():
    for r, c in [(1, 1), (1, 5), (4, 1), (7, 9)]:
        e = lattice_edges(r, c)
        s, d = oracle.lattice_edges(r, c)
        assert np.array_equal(e.src, s) and np.array_equal(e.dst, d)


def test_predecessor_array_layout():
    p = PredecessorArray(33)
    assert len(p.storage) == 64 and (p.storage == SENTINEL).all() and len(p.p) == 33
    with pytest.raises(AssertionError):
        PredecessorArray(0)


def test_rmat_params_and_pcg_state():
    with pytest.raises(AssertionError):
        RmatParams(scale=0)
    with pytest.raises(AssertionError):
        RmatParams(scale=31)
    with pytest.raises(AssertionError):
        RmatParams(scale=4, a=0.5, b=0.5, c=0.5, d=0.0)
    p = RmatParams(scale=5, seed=3)
    assert p.num_vertices == 32 and p.num_edges == 512
    assert np.array_equal(p.pcg_state(), oracle.pcg_state(3))
    assert p.thresholds() == oracle.rmat_thresholds(0.57, 0.19, 0.19, 0.05)


def test_edge_list_roundtrip(tmp_path):
    s, d = oracle.rmat_edges(6, 4, seed=2)
    e = EdgeList(s, d, 64)
    write_edge_list(tmp_path / "g.bin", e, RmatParams(scale=6, edgefactor=4, seed=2))
    e2, p2 = read_edge_list(tmp_path / "g.bin")
    assert np.array_equal(e2.src, s) and np.array_equal(e2.dst, d) and p2.seed == 2


def test_experiment_config_and_emit(tmp_path):
    with pytest.raises(AssertionError):
        ExperimentConfig(scale=10, mode="bogus")
    cfg = ExperimentConfig(scale=10)
    assert cfg.mode == "gpu"
    runs = [RootRun(1, 0.5, 100, 200.0), RootRun(2, 0.25, 100, 400.0)]
    st = RunStats(cfg, "gpu", 1, "device", runs, 266.6, 0, False, 0.25, 0.5, 0.375)
    emit_results([st], "csv", tmp_path / "r.csv")
    rows = list(csv.reader(open(tmp_path / "r.csv")))
    # the reference's columns (harness.py:278-280), then the device's
    assert rows[0] == ["scale", "edgefactor", "seed", "mode", "threads", "placement", "root", "time_s",
                       "edges", "teps", "gpus", "gbytes_alg", "roofline_frac"]
    assert rows[-1][6] == "all" and rows[-1][8] == "200" and rows[-1][10] == "1"
    emit_results([st], "json", tmp_path / "r.json")
    assert json.loads((tmp_path / "r.json").read_text())["results"][0]["mode"] == "gpu"


def test_layerstats_frozen():
    l = LayerStats(1, 2, 3)
    with pytest.raises(Exception):
        l.input = 5
