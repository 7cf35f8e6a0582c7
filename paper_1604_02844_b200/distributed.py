"""Partitioned (multi-GPU) BFS: one partition per GPU, one process per GPU
(BASELINE north_star "vertices are 1D-partitioned across the 8
B200s of one box, and each level exchanges the frontier bitmap").

The partition and the per-level kernels live in liblbfs (csrc/partition.cu,
C ABI ``lbfs_part_*`` in include/lbfs.h); this module is the level loop,
which interleaves them with the collectives between the steps:

    expand -> pack -> all_to_all(marks by owner) -> merge (+ compaction)
           -> all_gather(owned words of F_{L+1} + the rank's counts)
           -> sync (counts summed on the device) -> level_done

This is the reference's level-synchronous loop (traversal.py:90, 152, 366)
with the frontier exchanged between levels (two collectives per level; one
all-reduce at the start for the root's degree). Collectives go through an
*exchange* object:

* ``TorchExchange`` — torch.distributed (NCCL between GPUs; gloo on CPU for
  the multi-process tests), one partition per process;
* ``LocalExchange`` — several partitions driven in lockstep by one process
  (their kernels never wait on each other: every step of every partition
  completes before the next step starts), used to check the partitioned path
  against the single-GPU one on a single device.

The driver is generic over the partition objects: ``PartitionedGraph`` (the
device) or any object with the same step methods (the CPU restatement in
oracle/part_emu.py, used by the gloo tests).

The same loop also runs inside the library (``PartitionedGraph.attach_nccl``
+ ``bfs_native``; csrc/multi.cu): the library owns an NCCL communicator
(ncclCommInitRank, the unique id broadcast over torch.distributed) and drives
every step and collective from one C++ call per BFS, without the per-step
Python and torch.distributed overhead. ``bench.py --gpus N`` times that path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .traversal import SENTINEL, LayerStats

BITS_PER_WORD = 32


def _stream_ptr(t) -> int | None:
    import torch
    if t.is_cuda:
        return torch.cuda.current_stream(t.device).cuda_stream
    return None


class PartitionedGraph:
    """Rank ``rank``'s partition of graph ``g`` (word-cyclic over the
    degree-ordered internal ids) on the current CUDA device. ``g`` is a
    CsrGraph of this package (device CSR or host arrays) or any object with
    ``num_vertices``/``colstarts``/``rows`` (e.g. the reference CsrGraph)."""

    def __init__(self, g, rank: int, nparts: int, device: int | None = None):
        import torch
        assert nparts >= 1 and (nparts & (nparts - 1)) == 0, "nparts must be a power of two"
        assert 0 <= rank < nparts
        lib = _lib.load()
        if device is None:
            device = torch.cuda.current_device()
        _lib.check(lib.lbfs_set_device(int(device)))
        self.device = torch.device("cuda", int(device))
        self.num_vertices = int(g.num_vertices)
        h = ctypes.c_void_p()
        dev_csr = getattr(g, "_handles", None)
        if dev_csr is not None and dev_csr[0][0]:
            _lib.check(lib.lbfs_part_create_from_csr(dev_csr[0][0], rank, nparts, ctypes.byref(h)))
        else:
            cs = np.ascontiguousarray(g.colstarts, dtype=np.int64)
            rows = np.ascontiguousarray(g.rows, dtype=np.int32)
            _lib.check(lib.lbfs_part_create(self.num_vertices, _lib.ptr(cs), _lib.ptr(rows) if len(rows) else None,
                                            len(rows), rank, nparts, ctypes.byref(h)))
        self._h = h.value
        r, p = ctypes.c_int(), ctypes.c_int()
        nw, nl, nnzl = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(lib.lbfs_part_info(self._h, ctypes.byref(r), ctypes.byref(p), ctypes.byref(nw),
                                      ctypes.byref(nl), ctypes.byref(nnzl)))
        self.rank, self.nparts = r.value, p.value
        self.nwords, self.n_local, self.nnz_local = nw.value, nl.value, nnzl.value
        self.words_per_peer = self.nwords // self.nparts

    def close(self) -> None:
        if self._h:
            _lib.load().lbfs_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- buffers ---------------------------------------------------------------
    def new_buffers(self) -> dict:
        import torch
        W, P = self.words_per_peer, self.nparts
        i32 = dict(dtype=torch.int32, device=self.device)
        return {"send": torch.empty(P * W, **i32), "recv": torch.empty(P * W, **i32),
                "fsend": torch.empty(W + 4, **i32), "fgath": torch.empty(P * (W + 4), **i32),
                "red": torch.zeros(2, dtype=torch.int64, device=self.device)}

    def new_outputs(self):
        import torch
        n = self.num_vertices
        pad = (n + BITS_PER_WORD - 1) // BITS_PER_WORD * BITS_PER_WORD
        return (torch.empty(pad, dtype=torch.int32, device=self.device),
                torch.empty(n, dtype=torch.int32, device=self.device))

    # -- level steps (all on the current stream) ------------------------------
    def start(self, root: int, red) -> None:
        _lib.check(_lib.load().lbfs_part_start(self._h, int(root), red.data_ptr(), _stream_ptr(red)))

    def expand(self) -> None:
        import torch
        _lib.check(_lib.load().lbfs_part_expand(self._h, torch.cuda.current_stream(self.device).cuda_stream))

    def pack(self, send) -> None:
        _lib.check(_lib.load().lbfs_part_pack(self._h, send.data_ptr(), _stream_ptr(send)))

    def merge(self, recv, fsend) -> None:
        _lib.check(_lib.load().lbfs_part_merge(self._h, recv.data_ptr(), fsend.data_ptr(), _stream_ptr(fsend)))

    def sync(self, fgath) -> None:
        _lib.check(_lib.load().lbfs_part_sync(self._h, fgath.data_ptr(), _stream_ptr(fgath)))

    def level_done(self, red=None) -> tuple[LayerStats | None, bool]:
        """red: the summed start counts (after start); None after a level."""
        ly, done = _lib.Layer(), ctypes.c_int()
        _lib.check(_lib.load().lbfs_part_level_done(self._h, red.data_ptr() if red is not None else None,
                                                     ctypes.byref(ly), ctypes.byref(done)))
        return LayerStats(int(ly.input), int(ly.edges), int(ly.discovered)), bool(done.value)

    def finish(self, pred, level) -> None:
        _lib.check(_lib.load().lbfs_part_finish(self._h, pred.data_ptr() if pred is not None else None,
                                                 level.data_ptr() if level is not None else None,
                                                 _stream_ptr(pred if pred is not None else level)))

    # -- the library's own level loop (one call per BFS) ----------------------
    def attach_nccl(self, group=None) -> None:
        """Collective over the torch.distributed group (one partition per
        rank): rank 0 draws an NCCL unique id, every rank joins the library's
        communicator with it."""
        import torch
        import torch.distributed as dist
        lib = _lib.load()
        uid = (ctypes.c_uint8 * 128)()
        if self.rank == 0:
            _lib.check(lib.lbfs_nccl_unique_id(uid))
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8,
                         device=self.device if dist.get_backend(group) == "nccl" else "cpu")
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = (ctypes.c_uint8 * 128)(*t.cpu().tolist())
        _lib.check(lib.lbfs_part_attach_nccl(self._h, uid, self.nparts, self.rank))
        self.attached = True

    def bfs_native(self, root: int, pred, level=None, gather: bool = True) -> "PartitionedResult":
        """One BFS through the library's level loop (collective). pred /
        level: device tensors (pad32(n) / n int32) written on return; with
        ``gather`` the full arrays, else this rank's owned entries."""
        lib = _lib.load()
        cap = 4096
        layers = (_lib.Layer * cap)()
        nl, t = ctypes.c_int64(), _lib.Timing()
        _lib.check(lib.lbfs_part_bfs(self._h, int(root), pred.data_ptr(),
                                     level.data_ptr() if level is not None else None, int(bool(gather)),
                                     layers, cap, ctypes.byref(nl), ctypes.byref(t)))
        if nl.value > cap:  # (e.g. a lattice: thousands of levels)
            layers = (_lib.Layer * nl.value)()
            _lib.check(lib.lbfs_graph_last_layers(self._h, layers, nl.value, ctypes.byref(nl)))
        ls = [LayerStats(int(x.input), int(x.edges), int(x.discovered)) for x in layers[:nl.value]]
        return PartitionedResult(ls, sum(l.edges for l in ls), pred, level, gather, t.as_dict())

    def plan(self) -> tuple[int, int]:
        """(all-to-all words per peer, all-gather words per rank) of the
        coming level: the dense bitmap slices or, for a small level, id lists."""
        a, g = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.load().lbfs_part_plan(self._h, ctypes.byref(a), ctypes.byref(g)))
        return a.value, g.value

    def resolve_count(self) -> int:
        v = ctypes.c_int64()
        _lib.check(_lib.load().lbfs_part_resolve_count(self._h, ctypes.byref(v)))
        return v.value


# ------------------------------------------------------------------ exchanges
class TorchExchange:
    """The collectives over torch.distributed: NCCL for CUDA tensors
    (one partition per process), gloo for CPU tensors. Lists hold this
    process's single partition's buffers."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def all_to_all(self, sends, recvs) -> None:
        self.dist.all_to_all_single(recvs[0], sends[0], group=self.group)

    def all_gather(self, fsends, fgaths) -> None:
        self.dist.all_gather_into_tensor(fgaths[0], fsends[0], group=self.group)

    def all_reduce_sum(self, reds) -> None:
        self.dist.all_reduce(reds[0], group=self.group)

    def all_reduce_min(self, ts) -> None:
        self.dist.all_reduce(ts[0], op=self.dist.ReduceOp.MIN, group=self.group)

    def all_reduce_max(self, ts) -> None:
        self.dist.all_reduce(ts[0], op=self.dist.ReduceOp.MAX, group=self.group)


class LocalExchange:
    """All partitions in this process: the collectives are tensor copies."""

    def all_to_all(self, sends, recvs) -> None:
        P = len(sends)
        W = sends[0].numel() // P
        for h in range(P):
            for p in range(P):
                recvs[h][p * W:(p + 1) * W].copy_(sends[p][h * W:(h + 1) * W])

    def all_gather(self, fsends, fgaths) -> None:
        W = fsends[0].numel()
        for dst in fgaths:
            for p, src in enumerate(fsends):
                dst[p * W:(p + 1) * W].copy_(src)

    def _reduce(self, ts, fn) -> None:
        acc = ts[0].clone()
        for t in ts[1:]:
            acc = fn(acc, t.to(acc.device))
        for t in ts:
            t.copy_(acc)

    def all_reduce_sum(self, reds) -> None:
        import torch
        self._reduce(reds, torch.add)

    def all_reduce_min(self, ts) -> None:
        import torch
        self._reduce(ts, torch.minimum)

    def all_reduce_max(self, ts) -> None:
        import torch
        self._reduce(ts, torch.maximum)


# ------------------------------------------------------------------ driver
@dataclass
class PartitionedResult:
    layers: list
    traversed_edge_count: int
    pred: object = None    # full outputs (after gather) or this rank's (owned entries only)
    level: object = None
    gathered: bool = False
    timing: dict | None = None  # bfs_native: the library's timing (bfs_ms = this rank's device time)


def bfs_partitioned(parts: list, root: int, exchange, bufs: list | None = None, outputs: list | None = None,
                    gather: bool = True) -> PartitionedResult:
    """Top-down BFS from ``root`` over partitions ``parts`` (this process's
    partitions: one under torch.distributed, all of them with LocalExchange).

    Returns the layers (identical on every rank) and, per partition, the
    pred (pad32(n)) / level (n) outputs in original ids: with ``gather`` the
    full arrays on every rank (min / max all-reduce of the owned entries),
    else only the owned entries (SENTINEL / -1 elsewhere)."""
    if bufs is None:
        bufs = [p.new_buffers() for p in parts]
    reds = [b["red"] for b in bufs]
    for p, b in zip(parts, bufs):
        p.start(root, b["red"])
    exchange.all_reduce_sum(reds)
    for p, b in zip(parts, bufs):
        p.level_done(b["red"])
    layers = []
    P = parts[0].nparts
    while True:
        # this level's slice sizes (identical on every rank; objects without
        # plan() exchange the dense slices)
        S, G = parts[0].plan() if hasattr(parts[0], "plan") else (None, None)
        send = [b["send"][:P * S] if S else b["send"] for b in bufs]
        recv = [b["recv"][:P * S] if S else b["recv"] for b in bufs]
        fsend = [b["fsend"][:G] if G else b["fsend"] for b in bufs]
        fgath = [b["fgath"][:P * G] if G else b["fgath"] for b in bufs]
        for p in parts:
            p.expand()
        for p, s in zip(parts, send):
            p.pack(s)
        exchange.all_to_all(send, recv)
        for p, r, f in zip(parts, recv, fsend):
            p.merge(r, f)
        exchange.all_gather(fsend, fgath)
        for p, f in zip(parts, fgath):
            p.sync(f)
        outs = [p.level_done() for p in parts]
        layer, done = outs[0]
        assert all(o == outs[0] for o in outs), "partitions disagree on the layer"
        layers.append(layer)
        if done:
            break
    if outputs is None:
        outputs = [p.new_outputs() for p in parts]
    for p, (pred, level) in zip(parts, outputs):
        p.finish(pred, level)
    if gather:
        exchange.all_reduce_min([o[0] for o in outputs])
        exchange.all_reduce_max([o[1] for o in outputs])
    return PartitionedResult(layers, sum(l.edges for l in layers), [o[0] for o in outputs],
                             [o[1] for o in outputs], gather)


def unpad_pred(pred, n: int) -> np.ndarray:
    """Host copy of a gathered pred output (PredecessorArray storage)."""
    a = pred.cpu().numpy() if hasattr(pred, "cpu") else np.asarray(pred)
    assert len(a) >= n
    return a


__all__ = ["PartitionedGraph", "TorchExchange", "LocalExchange", "PartitionedResult", "bfs_partitioned",
           "SENTINEL"]
