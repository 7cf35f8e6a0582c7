"""Top-down BFS on the B200: the drop-in for the reference traversal.py
(/root/reference/pkg/src/lanebfs/traversal.py).

``bfs(g, s)`` runs the sm_100a kernels of liblbfs (csrc/bfs.cu) through the
C ABI and returns the reference's result types, so the reference's own
``validate_tree`` and ``levels_from_parents`` accept its output unchanged:

* ``predecessors``: PredecessorArray, int32 storage padded to a multiple of
  32 with SENTINEL (traversal.py:30-50); root -> root, unreached -> SENTINEL;
* ``layers``: one LayerStats(input, edges, discovered) per frontier,
  including the last one (discovered == 0) (traversal.py:66-70, 100);
* ``traversed_edge_count``: sum of layer edges = sum of degree over reached
  vertices (traversal.py:104; the TEPS numerator, harness.py:269);
* ``levels`` (new, gap G2): int32 BFS level per vertex, -1 = unreached.

Predecessors are a valid BFS tree; which equal-level parent wins a vertex is
decided by the device atomic, the benign race the reference documents
(traversal.py:128-132). Levels and layers are deterministic.

``run_bfs`` keeps the reference dispatch signature (traversal.py:413-422).
Every mode names the same breadth-first search; here all of them run on the
device (there is no CPU fallback).
"""

from __future__ import annotations

import ctypes
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib

SENTINEL = 0x7FFFFFFF  # traversal.py:22
BITS_PER_WORD = 32

MODES = ("gpu", "serial", "parallel_naive", "parallel_restored", "vectorized")


class PredecessorArray:
    """Per-vertex parent ids, SENTINEL for unreached vertices; storage padded
    to whole 32-entry words (traversal.py:30-50)."""

    __slots__ = ("num_vertices", "storage")

    infinity_sentinel = SENTINEL

    def __init__(self, num_vertices: int, _fill: bool = True, _storage: np.ndarray | None = None):
        assert num_vertices >= 1
        padded = (num_vertices + BITS_PER_WORD - 1) // BITS_PER_WORD * BITS_PER_WORD
        self.num_vertices = num_vertices
        if _storage is not None:
            assert len(_storage) == padded
            self.storage = _storage
        else:
            self.storage = (np.full(padded, SENTINEL, dtype=np.int32) if _fill
                            else np.empty(padded, dtype=np.int32))

    @property
    def p(self) -> np.ndarray:
        return self.storage[:self.num_vertices]


@dataclass(frozen=True)
class LayerPolicy:
    """Which variant runs (traversal.py:53-63). ``vectorized_layers`` is kept
    for signature compatibility; the device path treats every layer alike."""

    vectorized_layers: int = 2
    mode: str = "gpu"

    def __post_init__(self):
        assert self.vectorized_layers >= 0
        assert self.mode in MODES


@dataclass(frozen=True)
class LayerStats:
    input: int       # frontier vertices entering the layer
    edges: int       # adjacency entries examined
    discovered: int  # vertices first reached in this layer


class BfsResult:
    """The reference's result (traversal.py:73-77: predecessors, layers,
    traversed_edge_count) plus ``levels`` (gap G2) and device ``timing``.

    ``levels`` is fetched from the device on first access (the reference has
    no level array; its callers derive one with levels_from_parents). The
    handle keeps the level array of its last BFS; before the next BFS on the
    same graph starts, a still-referenced result fetches its levels first, so
    a result never sees another BFS's levels."""

    __slots__ = ("predecessors", "layers", "traversed_edge_count", "timing", "_levels", "_handle", "_owner", "__weakref__")

    def __init__(self, predecessors, layers=None, traversed_edge_count=0, levels=None, timing=None):
        self.predecessors = predecessors
        self.layers = layers if layers is not None else []
        self.traversed_edge_count = traversed_edge_count
        self.timing = timing
        self._levels = levels
        self._handle = None
        self._owner = None  # the graph, kept alive while the levels are on its device handle

    @property
    def levels(self) -> np.ndarray | None:
        if self._levels is None and self._handle is not None:
            with _handle_lock(self._handle):
                _materialize(self)
        return self._levels

    def __repr__(self) -> str:
        return (f"BfsResult(layers={len(self.layers)}, traversed_edge_count={self.traversed_edge_count}, "
                f"levels={'pending' if self._levels is None else 'host'})")


# per handle: a lock around flush + BFS + registration, and the result whose
# levels are still on the device
_locks: dict[int, threading.Lock] = {}
_locks_guard = threading.Lock()
_pending: dict[int, weakref.ref] = {}


def _handle_lock(h: int) -> threading.Lock:
    with _locks_guard:
        return _locks.setdefault(h, threading.RLock())


def _materialize(res: BfsResult) -> None:
    """(handle lock held) copy the handle's last levels into res."""
    h = res._handle
    if res._levels is not None or h is None:
        return
    ref = _pending.get(h)
    if ref is None or ref() is not res:
        raise RuntimeError("internal: levels of this result are no longer on the device")
    n = res.predecessors.num_vertices if res.predecessors is not None else _num_vertices(h)
    lv = _lib.pinned_empty(n)
    _lib.check(_lib.load().lbfs_graph_last_levels(h, _lib.ptr(lv)))
    res._levels = lv
    res._handle = None
    res._owner = None
    del _pending[h]


def _flush(h: int) -> None:
    """(handle lock held) before a BFS on h: the previous result, if still
    alive, takes its levels off the device."""
    ref = _pending.get(h)
    if ref is None:
        return
    r = ref()
    if r is not None and r._levels is None:
        _materialize(r)
    _pending.pop(h, None)


def _register(h: int, res: BfsResult, owner) -> None:
    res._handle = h
    res._owner = owner
    _pending[h] = weakref.ref(res)


def _num_vertices(h: int) -> int:
    n = ctypes.c_int64()
    _lib.check(_lib.load().lbfs_graph_info(h, ctypes.byref(n), None))
    return int(n.value)


# ------------------------------------------------------------- graph handles
_foreign: dict[int, tuple] = {}


def _handle(g) -> int:
    """Device BFS handle of g. Our CsrGraph owns its handle; a foreign graph
    object (e.g. the reference's CsrGraph) is uploaded once and cached while
    its arrays stay the same objects."""
    if hasattr(g, "device_handle"):
        return g.device_handle()
    key = id(g)
    rows, cs = g.rows, g.colstarts
    ent = _foreign.get(key)
    if ent is not None and ent[0] is rows and ent[1] is cs:
        return ent[2]
    lib = _lib.load()
    if ent is not None:
        _destroy_foreign(ent[2])
        del _foreign[key]
    while len(_foreign) >= 2:  # keep at most two foreign graphs resident
        _, old = _foreign.popitem()
        _destroy_foreign(old[2])
    cs64 = np.ascontiguousarray(cs, dtype=np.int64)
    r32 = np.ascontiguousarray(rows, dtype=np.int32)
    h = ctypes.c_void_p()
    _lib.check(lib.lbfs_graph_create(int(g.num_vertices), _lib.ptr(cs64), _lib.ptr(r32) if len(r32) else None,
                                     len(r32), 1, ctypes.byref(h)))
    _foreign[key] = (rows, cs, h.value)
    return h.value


def _release_handle(h: int) -> None:
    """Flush a pending result's levels, then destroy the handle."""
    with _handle_lock(h):
        _flush(h)
        _lib.load().lbfs_graph_destroy(h)


def _destroy_foreign(h: int) -> None:
    with _handle_lock(h):
        _flush(h)
        _lib.load().lbfs_graph_destroy(h)


def _layers_from(buf, k: int, h: int) -> list[LayerStats]:
    if k > len(buf):  # (handle lock held: no other BFS ran since)
        buf = (_lib.Layer * k)()
        n = ctypes.c_int64()
        _lib.check(_lib.load().lbfs_graph_last_layers(h, buf, k, ctypes.byref(n)))
    return [LayerStats(int(buf[i].input), int(buf[i].edges), int(buf[i].discovered)) for i in range(k)]


_LAYER_CAP = 256


DIRECTIONS = {"top_down": 0, "optimizing": 1}


def _direction(direction: str) -> int:
    """Traversal direction of one call: "top_down" (the paper's algorithm;
    the default and the benchmarked path) or "optimizing" (bottom-up levels
    while the frontier is large). Levels, visited set
    and layers are the same either way; parents may differ (any neighbour one
    level up, as the reference's own parallel variants allow)."""
    assert direction in DIRECTIONS, f"direction must be one of {sorted(DIRECTIONS)}"
    return DIRECTIONS[direction]


def bfs(g, s: int, direction: str = "top_down", levels: bool = False) -> BfsResult:
    """Top-down BFS from s on the device; host outputs. The parent array is
    copied (in chunks, behind the device's output pass) inside the call;
    levels come with it when ``levels=True``, else on first access."""
    n = g.num_vertices
    assert 0 <= s < n
    d = _direction(direction)
    h = _handle(g)
    padded = (n + BITS_PER_WORD - 1) // BITS_PER_WORD * BITS_PER_WORD
    # outputs land in page-locked memory (pooled), so the copies run at full link rate
    pred = PredecessorArray(n, _storage=_lib.pinned_empty(padded))
    lv = _lib.pinned_empty(n) if levels else None
    buf = (_lib.Layer * _LAYER_CAP)()
    k = ctypes.c_int64()
    t = _lib.Timing()
    with _handle_lock(h):
        _flush(h)
        _lib.check(_lib.load().lbfs_bfs(h, int(s), d, _lib.ptr(pred.storage), _lib.ptr(lv) if levels else None, buf,
                                        _LAYER_CAP, ctypes.byref(k), ctypes.byref(t)))
        res = BfsResult(pred, _layers_from(buf, k.value, h), int(t.edges), lv, t.as_dict())
        if not levels:
            _register(h, res, g)
    return res


def bfs_device(g, s: int, pred_out, level_out=None, direction: str = "top_down") -> BfsResult:
    """BFS into device buffers (anything with ``data_ptr()``, e.g. torch CUDA
    int32 tensors of pad32(n) and n entries; ``level_out`` may be None). No
    host copy of the outputs; ``predecessors`` of the result is None and
    ``levels`` are fetched to the host on first access."""
    n = g.num_vertices
    assert 0 <= s < n
    padded = (n + BITS_PER_WORD - 1) // BITS_PER_WORD * BITS_PER_WORD
    assert pred_out.numel() >= padded and (level_out is None or level_out.numel() >= n)
    d = _direction(direction)
    h = _handle(g)
    buf = (_lib.Layer * _LAYER_CAP)()
    k = ctypes.c_int64()
    t = _lib.Timing()
    with _handle_lock(h):
        _flush(h)
        _lib.check(_lib.load().lbfs_bfs_device(h, int(s), d, pred_out.data_ptr(),
                                               level_out.data_ptr() if level_out is not None else None, buf,
                                               _LAYER_CAP, ctypes.byref(k), ctypes.byref(t)))
        res = BfsResult(None, _layers_from(buf, k.value, h), int(t.edges), None, t.as_dict())
        _register(h, res, g)
    return res


def run_bfs(g, s: int, policy: LayerPolicy | None = None, threads: int = 1,
            backend=None, chunked: bool = False) -> BfsResult:
    """Reference dispatch signature (traversal.py:413-422). All modes run the
    device BFS; ``threads``/``backend``/``chunked`` have no device meaning."""
    policy = policy or LayerPolicy()
    assert policy.mode in MODES and threads >= 1
    return bfs(g, s)
