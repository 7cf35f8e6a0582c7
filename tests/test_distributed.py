"""Partitioned (multi-GPU) BFS, SURVEY §8e.

CPU: the product's level loop (distributed.bfs_partitioned) over the
oracle's partition restatement (oracle/part_emu.py), in one process
(LocalExchange, P = 1..8) and in world_size-2 gloo process groups
(TorchExchange) — levels bit-exact with the serial oracle, trees certified.

GPU: the device partitions (liblbfs lbfs_part_*) driven in lockstep on one
device (LocalExchange; no kernel waits on another partition), checked
against the oracle and the single-GPU BFS. The NCCL path is the same driver
with TorchExchange (bench.py --gpus N under torchrun).
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch

import oracle
from oracle.part_emu import EmuPart
from paper_1604_02844_b200.distributed import LocalExchange, TorchExchange, bfs_partitioned

from _util import layers_tuples
from conftest import gpu_available


def _rmat(scale, ef=16, seed=1, permute=True):
    s, d = oracle.rmat_edges(scale, ef, seed=seed)
    n = 1 << scale
    if permute:
        s, d = oracle.permute_edges(n, oracle_perm_seed(seed), s, d)
    rp, ci = oracle.build_csr(n, s, d)
    return n, rp, ci


def oracle_perm_seed(seed):
    from paper_1604_02844_b200.graph import permutation_seed
    return permutation_seed(seed)


def _lattice(r, c):
    s, d = oracle.lattice_edges(r, c)
    n = r * c
    rp, ci = oracle.build_csr(n, s, d)
    return n, rp, ci


def _check(n, rp, ci, root, res, pred, level):
    _, lv_ref, layers_ref = oracle.bfs_serial(rp, ci, root)
    assert np.array_equal(level[:n], lv_ref)
    assert layers_tuples(res.layers) == layers_ref
    code, where = oracle.check_bfs(rp, ci, root, pred[:n], level[:n])
    assert code == 0, (oracle.CHECK_CODES[code], where)
    assert np.all(pred[n:] == 0x7FFFFFFF)  # PredecessorArray padding


@pytest.mark.parametrize("nparts", [1, 2, 4, 8])
def test_emulated_partitions_local(nparts):
    n, rp, ci = _rmat(10)
    parts = [EmuPart(n, rp, ci, r, nparts) for r in range(nparts)]
    deg = np.diff(rp)
    for root in oracle.pick_roots(deg, 3, 7):
        res = bfs_partitioned(parts, int(root), LocalExchange())
        for pred, level in zip(res.pred, res.level):
            _check(n, rp, ci, int(root), res, pred.numpy(), level.numpy())


def test_emulated_partitions_lattice_and_disconnected():
    n, rp, ci = _lattice(13, 11)  # n not a multiple of 32 * P
    parts = [EmuPart(n, rp, ci, r, 4) for r in range(4)]
    res = bfs_partitioned(parts, 5, LocalExchange())
    _check(n, rp, ci, 5, res, res.pred[0].numpy(), res.level[0].numpy())
    # isolated root: one layer (1, 0, 0)
    s = np.array([0, 1], dtype=np.uint32)
    d = np.array([1, 2], dtype=np.uint32)
    rp2, ci2 = oracle.build_csr(70, s, d)
    parts = [EmuPart(70, rp2, ci2, r, 2) for r in range(2)]
    res = bfs_partitioned(parts, 50, LocalExchange())
    assert layers_tuples(res.layers) == [(1, 0, 0)]
    lv = res.level[0].numpy()
    assert lv[50] == 0 and (lv >= 0).sum() == 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, path, roots, out_dir):
    import sys
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        z = np.load(path)
        part = EmuPart(int(z["n"]), z["rp"], z["ci"], rank, world)
        for root in roots:
            res = bfs_partitioned([part], int(root), TorchExchange())
            np.savez(os.path.join(out_dir, f"r{rank}_{root}.npz"), pred=res.pred[0].numpy(),
                     level=res.level[0].numpy(), layers=np.array(layers_tuples(res.layers), dtype=np.int64))
    finally:
        dist.destroy_process_group()
        sys.stdout.flush()


def test_gloo_world_size_2():
    n, rp, ci = _rmat(9, seed=3)
    roots = [int(r) for r in oracle.pick_roots(np.diff(rp), 3, 11)]
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "g.npz")
        np.savez(path, n=n, rp=rp, ci=ci)
        torch.multiprocessing.spawn(_gloo_worker, args=(2, _free_port(), path, roots, tmp), nprocs=2, join=True)
        for root in roots:
            _, lv_ref, layers_ref = oracle.bfs_serial(rp, ci, root)
            outs = [np.load(os.path.join(tmp, f"r{r}_{root}.npz")) for r in range(2)]
            for o in outs:  # gathered outputs: identical full arrays on both ranks
                assert np.array_equal(o["level"], lv_ref)
                assert [tuple(x) for x in o["layers"].tolist()] == layers_ref
                code, where = oracle.check_bfs(rp, ci, root, o["pred"][:n], o["level"])
                assert code == 0, (oracle.CHECK_CODES[code], where)
            assert np.array_equal(outs[0]["pred"], outs[1]["pred"])


# ---------------------------------------------------------------- GPU
def _device_parts(g, nparts):
    from paper_1604_02844_b200.distributed import PartitionedGraph
    return [PartitionedGraph(g, r, nparts) for r in range(nparts)]


@pytest.mark.gpu
@pytest.mark.parametrize("nparts", [1, 2, 4, 8])
def test_gpu_partitions_rmat(nparts):
    from paper_1604_02844_b200 import RmatParams, build_rmat_graph, bfs
    g = build_rmat_graph(RmatParams(scale=14, edgefactor=16, seed=2))
    rp, ci = g.colstarts, g.rows
    n = g.num_vertices
    parts = _device_parts(g, nparts)
    for root in oracle.pick_roots(np.diff(rp), 4, 5):
        root = int(root)
        res = bfs_partitioned(parts, root, LocalExchange())
        single = bfs(g, root)
        assert layers_tuples(res.layers) == layers_tuples(single.layers)
        for pred, level in zip(res.pred, res.level):
            _check(n, rp, ci, root, res, pred.cpu().numpy(), level.cpu().numpy())
    if nparts > 1:
        assert sum(p.resolve_count() for p in parts) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["0", "2"])
@pytest.mark.parametrize("nparts", [2, 8])
def test_gpu_partitions_sparse_exchange(monkeypatch, nparts, mode):
    """LBFS_PART_SPARSE=2: every level whose lists fit the slices exchanges
    [count, ids] lists (all-to-all of marks, all-gather of the new owned
    ids); =0: never. Same layers, levels and certified trees either way; the
    lattice (small frontiers, many levels) and an R-MAT graph."""
    from paper_1604_02844_b200 import RmatParams, build_rmat_graph, bfs, CsrGraph
    monkeypatch.setenv("LBFS_PART_SPARSE", mode)  # (read when the partition handle is made)
    n, lrp, lci = _lattice(64, 50)
    cases = [(build_rmat_graph(RmatParams(scale=13, edgefactor=16, seed=4)), None), (CsrGraph(n, lci, lrp), 0)]
    for g, r0 in cases:
        rp, ci, n = g.colstarts, g.rows, g.num_vertices
        parts = _device_parts(g, nparts)
        sizes = []
        roots = [r0] if r0 is not None else [int(r) for r in oracle.pick_roots(np.diff(rp), 3, 7)]
        for root in roots:
            res = bfs_partitioned(parts, root, LocalExchange())
            for pred, level in zip(res.pred, res.level):
                _check(n, rp, ci, root, res, pred.cpu().numpy(), level.cpu().numpy())
            sizes.append(parts[0].plan())
        W = parts[0].words_per_peer
        if mode == "0":
            assert all(s == (W, W + 4) for s in sizes)
        else:  # after the last level (E = 0) the plan is a list
            assert all(s[0] < W for s in sizes)


@pytest.mark.gpu
def test_gpu_partitions_match_emulation_per_rank():
    """Owned outputs before the gather: levels identical to the oracle's
    partition; every rank's pred entries lie on its own vertices."""
    from paper_1604_02844_b200 import RmatParams, build_rmat_graph
    g = build_rmat_graph(RmatParams(scale=12, edgefactor=16, seed=9))
    rp, ci, n = g.colstarts, g.rows, g.num_vertices
    dev = _device_parts(g, 4)
    emu = [EmuPart(n, rp, ci, r, 4) for r in range(4)]
    root = int(oracle.pick_roots(np.diff(rp), 1, 3)[0])
    rd = bfs_partitioned(dev, root, LocalExchange(), gather=False)
    re_ = bfs_partitioned(emu, root, LocalExchange(), gather=False)
    assert layers_tuples(rd.layers) == layers_tuples(re_.layers)
    for r in range(4):
        assert np.array_equal(rd.level[r].cpu().numpy(), re_.level[r].numpy())
        owned_dev = rd.pred[r].cpu().numpy()[:n] != 0x7FFFFFFF
        owned_emu = re_.pred[r].numpy()[:n] != 0x7FFFFFFF
        assert np.array_equal(owned_dev, owned_emu)


@pytest.mark.gpu
def test_gpu_partitions_lattice_host_csr():
    from paper_1604_02844_b200 import CsrGraph
    n, rp, ci = _lattice(40, 37)
    g = CsrGraph(n, ci, rp)  # host arrays: lbfs_part_create uploads them
    parts = _device_parts(g, 2)
    res = bfs_partitioned(parts, 17, LocalExchange())
    _check(n, rp, ci, 17, res, res.pred[1].cpu().numpy(), res.level[1].cpu().numpy())


@pytest.mark.gpu
def test_gpu_partition_bad_args():
    from paper_1604_02844_b200 import RmatParams, build_rmat_graph
    from paper_1604_02844_b200.distributed import PartitionedGraph
    g = build_rmat_graph(RmatParams(scale=8, edgefactor=4, seed=1))
    with pytest.raises(AssertionError):
        PartitionedGraph(g, 0, 3)
    p = PartitionedGraph(g, 0, 2)
    b = p.new_buffers()
    with pytest.raises(AssertionError):
        p.start(g.num_vertices, b["red"])
