"""Mode "gpu" inside the reference package itself (integration.install,
INTEGRATION.md Option A): the reference's own run_experiment, validate_tree,
emit_results and CLI drive the device BFS through its dispatch point
run_bfs (traversal.py:413-422). Needs the reference package: the read-only
checkout (/root/reference/pkg/src, the build container) or the copy
installed into baseline/_ref (travels to the GPU box); skipped otherwise."""

import csv
import json
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _reference():
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "lanebfs").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            import lanebfs

            return lanebfs
    pytest.skip("reference package lanebfs not installed (baseline/_ref)")


@pytest.fixture
def lanebfs():
    pkg = _reference()
    from paper_1604_02844_b200 import integration

    import os

    cpus = os.sched_getaffinity(0)  # the reference's harness pins the process (harness.py:137-154)
    inst = integration.install(pkg)
    yield pkg
    inst.uninstall()
    os.sched_setaffinity(0, cpus)


def test_reference_run_experiment_in_gpu_mode(lanebfs, tmp_path):
    from lanebfs.harness import ExperimentConfig, emit_results, run_experiment

    cfg = ExperimentConfig(scale=12, mode="gpu", thread_counts=(1,), num_roots=8, filter_unconnected=True)
    stats = run_experiment(cfg)  # the reference validates every tree (harness.py:266-268)
    assert len(stats) == 1 and stats[0].mode == "gpu" and len(stats[0].runs) == 8
    assert all(r.edges > 0 and r.teps > 0 for r in stats[0].runs)
    emit_results(stats, "csv", tmp_path / "r.csv")
    rows = list(csv.reader(open(tmp_path / "r.csv")))
    assert rows[0][3] == "mode" and all(row[3] == "gpu" for row in rows[1:])


def test_reference_results_equal_its_own_modes(lanebfs):
    from lanebfs.graph import RmatParams, build_csr, generate_rmat
    from lanebfs.traversal import LayerPolicy, bfs_serial, run_bfs
    from lanebfs.validate import levels_from_parents, validate_tree

    g = build_csr(generate_rmat(RmatParams(scale=11, edgefactor=16, seed=7)))
    for s in (0, 5, 1000):
        if g.degrees()[s] == 0:
            continue
        ours = run_bfs(g, s, LayerPolicy(mode="gpu"))
        ref = bfs_serial(g, s)
        assert type(ours) is type(ref)
        assert ours.layers == ref.layers and ours.traversed_edge_count == ref.traversed_edge_count
        assert np.array_equal(levels_from_parents(ours.predecessors.p, s), levels_from_parents(ref.predecessors.p, s))
        assert validate_tree(g, s, ours.predecessors).passed


def test_reference_cli_validate_gpu(lanebfs, capsys):
    from lanebfs import cli

    rc = cli.main(["validate", "--scale", "10", "--mode", "gpu", "--roots", "4"])
    out = capsys.readouterr().out.strip().splitlines()[-1]
    assert rc == 0 and json.loads(out) == {"roots": 4, "failures": 0, "mode": "gpu"}


def test_uninstall_restores_modes():
    pkg = _reference()
    from paper_1604_02844_b200 import integration

    inst = integration.install(pkg)
    assert "gpu" in pkg.traversal.MODES
    inst.uninstall()
    assert "gpu" not in pkg.traversal.MODES
