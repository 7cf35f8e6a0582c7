"""The library's own multi-GPU graph (lbfs_graph_create(ngpus > 1),
lbfs_graph_create_partitioned; csrc/multi.cu): the 1D partitioned level loop
driven from one host thread over library-owned NCCL communicators. On a
one-GPU box it runs as a one-rank communicator (the same code path: expand,
pack, ncclAlltoAll, merge, ncclAllGather, sync, output all-reduce); with two
or more GPUs visible the two-device case runs as well. Levels and layers are
compared with the oracle (pinned to the reference), trees with the
certificate."""

import numpy as np
import pytest
import torch

import oracle
from paper_1604_02844_b200 import RmatParams, bfs, bfs_device, build_lattice_graph, build_rmat_graph, pick_roots
from paper_1604_02844_b200.validate import validate_tree

pytestmark = pytest.mark.gpu


def layers_of(res):
    return [tuple(x) for x in ((l.input, l.edges, l.discovered) for l in res.layers)]


def check(g, roots, gpus):
    rp, ci = g.colstarts, g.rows
    g.device_handle(gpus=gpus, partitioned=True)
    for r in roots:
        res = bfs(g, r)
        _, lvl, layers = oracle.bfs_parallel(rp, ci, r)
        assert layers_of(res) == [tuple(x) for x in layers], r
        assert np.array_equal(res.levels, lvl), r
        assert oracle.check_bfs(rp, ci, r, res.predecessors.p, res.levels) == (0, -1), r
        assert validate_tree(g, r, res.predecessors).passed


@pytest.mark.parametrize("scale", [12, 16, 20])
def test_partitioned_one_rank_rmat(scale):
    g = build_rmat_graph(RmatParams(scale=scale, seed=1))
    check(g, pick_roots(g, 4, 1, filter_unconnected=True).tolist(), gpus=1)


def test_partitioned_one_rank_lattice():
    g = build_lattice_graph(96, 80)
    check(g, pick_roots(g, 3, 1, filter_unconnected=True).tolist(), gpus=1)


def test_partitioned_device_outputs_and_levels():
    g = build_rmat_graph(RmatParams(scale=14, seed=3))
    n = g.num_vertices
    r = int(pick_roots(g, 1, 3, filter_unconnected=True)[0])
    single = bfs(g, r)
    g.device_handle(gpus=1, partitioned=True)
    pred = torch.empty((n + 31) // 32 * 32, dtype=torch.int32, device="cuda")
    lvl = torch.empty(n, dtype=torch.int32, device="cuda")
    res = bfs_device(g, r, pred, lvl)
    assert np.array_equal(lvl.cpu().numpy(), single.levels)
    assert res.layers == single.layers
    assert res.timing["bfs_ms"] > 0 and res.timing["kernel_launches"] > 0


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs in this process")
def test_partitioned_two_gpus():
    g = build_rmat_graph(RmatParams(scale=18, seed=1))
    check(g, pick_roots(g, 4, 1, filter_unconnected=True).tolist(), gpus=2)
