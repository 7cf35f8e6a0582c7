"""Device tree validation (csrc/validate.cu) against the reference's own
validate_tree reports (the mutation catalog in tests/golden, produced by
the reference, validate.py:50-155) and against the vectorised CPU
restatement on seeded random mutations of real BFS trees."""

import numpy as np
import pytest

from paper_1604_02844_b200 import (
    SENTINEL,
    CsrGraph,
    PredecessorArray,
    RmatParams,
    bfs,
    bfs_device,
    build_rmat_graph,
    pick_roots,
    validate_tree,
    validate_tree_device,
)

pytestmark = pytest.mark.gpu


def _graph(entry):
    cs = np.array(entry["colstarts"], dtype=np.int64)
    rows = np.array(entry["rows"], dtype=np.int32)
    return CsrGraph(len(cs) - 1, rows, cs)


def test_matches_reference_mutation_catalog(golden):
    graphs = {k: _graph(v) for k, v in golden["validator"]["graphs"].items()}
    for case in golden["validator"]["cases"]:
        g = graphs[case["graph"]]
        pred = PredecessorArray(g.num_vertices)
        pred.p[:] = case["pred"]
        got = validate_tree_device(g, case["root"], pred).as_dict()
        want = dict(case["report"])
        want["details"] = {k: int(v) for k, v in want["details"].items()}
        assert got == want, (case["graph"], case["variant"])


def _mutations(p, s, n, rng):
    """Seeded corruptions of a valid parent array (the catalog's kinds at scale)."""
    reached = np.nonzero(p != SENTINEL)[0]
    others = reached[reached != s]
    out = []
    q = p.copy(); q[s] = others[0]; out.append(("root_not_self", q))
    q = p.copy(); v = rng.choice(others); q[v] = n + 5; out.append(("parent_out_of_range", q))
    unreached = np.nonzero(p == SENTINEL)[0]
    if len(unreached):
        q = p.copy(); v = rng.choice(others); q[v] = unreached[0]; out.append(("parent_unreached", q))
    q = p.copy(); v = rng.choice(others); q[v] = v; out.append(("self_parent", q))
    q = p.copy(); a, b = rng.choice(others, 2, replace=False); q[a] = b; q[b] = a; out.append(("two_cycle", q))
    q = p.copy(); v = rng.choice(others); w = rng.choice(others); q[v] = w; out.append(("random_parent", q))
    q = p.copy(); vs = rng.choice(others, 50, replace=False); q[vs] = rng.choice(others, 50); out.append(("many", q))
    return out


@pytest.mark.parametrize("scale", [12, 16])
def test_matches_cpu_validator_on_mutations(scale):
    g = build_rmat_graph(RmatParams(scale=scale, seed=4))
    rng = np.random.default_rng(scale)
    for s in pick_roots(g, 3, 2, filter_unconnected=True).tolist():
        res = bfs(g, s)
        p = res.predecessors.p.astype(np.int64)
        assert validate_tree_device(g, s, res.predecessors).passed
        for kind, q in _mutations(p, s, g.num_vertices, rng):
            pred = PredecessorArray(g.num_vertices)
            pred.p[:] = q
            got = validate_tree_device(g, s, pred).as_dict()
            want = validate_tree(g, s, pred).as_dict()
            assert got == want, (scale, s, kind, got, want)


def test_device_tensor_input_s20():
    import torch

    g = build_rmat_graph(RmatParams(scale=20, seed=1))
    n = g.num_vertices
    pred = torch.empty((n + 31) // 32 * 32, dtype=torch.int32, device="cuda")
    lvl = torch.empty(n, dtype=torch.int32, device="cuda")
    for s in pick_roots(g, 2, 1, filter_unconnected=True).tolist():
        bfs_device(g, s, pred, lvl)
        assert validate_tree_device(g, s, pred).passed
        bad = pred.clone()
        bad[s] = SENTINEL
        rep = validate_tree_device(g, s, bad)
        assert not rep.root_self_parent and rep.details["root_self_parent"] == s
