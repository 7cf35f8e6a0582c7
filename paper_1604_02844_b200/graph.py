"""Graph inputs of the BFS path: R-MAT generation, the seeded vertex
permutation, the 2D lattice and CSR assembly — the reference graph.py API
(/root/reference/pkg/src/lanebfs/graph.py) with the heavy lifting on the GPU.

* ``generate_rmat`` is bit-exact with the reference (graph.py:68-85): the
  device replays numpy's PCG64 stream position by position.
* ``build_csr`` produces exactly the reference arrays (graph.py:139-160):
  int64 ``colstarts`` (row_ptr) and int32 ``rows`` (col_idx), rows sorted,
  deduplicated and self-loop free.
* ``build_rmat_graph`` / ``build_lattice_graph`` run generate → permute →
  build_csr entirely on the device (the numpy path needs
  ~15 min / 46 GB at SCALE 24 and cannot build SCALE 27 at all).

The BFS itself lives in traversal.py; this module only prepares its input.
"""

from __future__ import annotations

import ctypes
import json
import weakref
from dataclasses import asdict, dataclass
from pathlib import Path

import numpy as np

from . import _lib

# Vertex ids are int32 below the sentinel, so SCALE is capped at 30 (graph.py:11-13).
MAX_SCALE = 30


@dataclass(frozen=True)
class RmatParams:
    """Recursive-matrix generator parameters (graph.py:16-45)."""

    scale: int
    edgefactor: int = 16
    a: float = 0.57
    b: float = 0.19
    c: float = 0.19
    d: float = 0.05
    seed: int = 1

    def __post_init__(self):
        assert 1 <= self.scale <= MAX_SCALE
        assert self.edgefactor >= 1
        assert min(self.a, self.b, self.c, self.d) >= 0.0
        assert abs(self.a + self.b + self.c + self.d - 1.0) <= 1e-9

    @property
    def num_vertices(self) -> int:
        return 1 << self.scale

    @property
    def num_edges(self) -> int:
        return (1 << self.scale) * self.edgefactor

    def thresholds(self) -> tuple[float, float, float]:
        """(ab, a_norm, c_norm): the per-bit quadrant thresholds, computed in
        the same float64 operations as graph.py:74-77."""
        ab = self.a + self.b
        a_norm = self.a / ab if ab > 0 else 0.0
        c_norm = self.c / (self.c + self.d) if (self.c + self.d) > 0 else 0.0
        return ab, a_norm, c_norm

    def pcg_state(self) -> np.ndarray:
        """{state_hi, state_lo, inc_hi, inc_lo} of default_rng(seed)'s PCG64."""
        st = np.random.default_rng(self.seed).bit_generator.state["state"]
        s, inc = int(st["state"]), int(st["inc"])
        m64 = (1 << 64) - 1
        return np.array([s >> 64, s & m64, inc >> 64, inc & m64], dtype=np.uint64)


@dataclass
class EdgeList:
    """Raw generator output: parallel endpoint arrays (graph.py:48-65)."""

    src: np.ndarray
    dst: np.ndarray
    num_vertices: int

    def __post_init__(self):
        assert self.src.shape == self.dst.shape
        if len(self.src):
            assert int(self.src.max()) < self.num_vertices
            assert int(self.dst.max()) < self.num_vertices

    @property
    def edge_count(self) -> int:
        return len(self.src)


def permutation_seed(seed: int) -> int:
    """Seed of the vertex permutation used for a generator seed."""
    return int(seed)


def generate_rmat(p: RmatParams) -> EdgeList:
    """2^scale * edgefactor R-MAT endpoint pairs, bit-identical to the
    reference generate_rmat for the same RmatParams (graph.py:68-85)."""
    m = p.num_edges
    src = np.empty(m, dtype=np.uint32)
    dst = np.empty(m, dtype=np.uint32)
    ab, an, cn = p.thresholds()
    st = p.pcg_state()
    _lib.check(_lib.load().lbfs_rmat_edges(p.scale, m, ab, an, cn, _lib.ptr(st), _lib.ptr(src), _lib.ptr(dst)))
    return EdgeList(src, dst, p.num_vertices)


def permute_vertices(e: EdgeList, seed: int) -> EdgeList:
    """Relabel both endpoints with the seeded Feistel bijection of [0, n)
    (gap G1: all benchmark configs ask for randomly permuted vertex ids)."""
    src = np.ascontiguousarray(e.src, dtype=np.uint32).copy()
    dst = np.ascontiguousarray(e.dst, dtype=np.uint32).copy()
    if len(src):
        _lib.check(_lib.load().lbfs_permute_edges(e.num_vertices, int(seed) & (2**64 - 1),
                                                  _lib.ptr(src), _lib.ptr(dst), len(src)))
    return EdgeList(src, dst, e.num_vertices)


def lattice_edges(rows: int, cols: int) -> EdgeList:
    """2D 4-neighbour lattice (config 4): vertex (r, c) = r*cols + c, one pair
    to the right and one down per vertex, no wraparound, in vertex order."""
    assert rows >= 1 and cols >= 1
    v = np.arange(rows * cols, dtype=np.int64).reshape(rows, cols)
    slots = np.full((rows, cols, 2, 2), -1, dtype=np.int64)  # [r, c, right/down, (u, v)]
    slots[:, :-1, 0, 0], slots[:, :-1, 0, 1] = v[:, :-1], v[:, 1:]
    slots[:-1, :, 1, 0], slots[:-1, :, 1, 1] = v[:-1, :], v[1:, :]
    arr = slots.reshape(-1, 2)
    arr = arr[arr[:, 0] >= 0]
    return EdgeList(arr[:, 0].astype(np.uint32), arr[:, 1].astype(np.uint32), rows * cols)


class CsrGraph:
    """Immutable adjacency in compressed sparse rows (graph.py:96-136):
    adjacency of u = rows[colstarts[u] : colstarts[u+1]].

    A graph built on the device keeps its device CSR and downloads
    ``rows``/``colstarts`` to the host only when they are first read. The
    BFS handle (device layout for traversal.py) is created on first use."""

    def __init__(self, num_vertices: int, rows: np.ndarray | None, colstarts: np.ndarray | None,
                 _device_csr: int | None = None, _nnz: int | None = None):
        if _device_csr is None:
            assert colstarts[0] == 0 and colstarts[-1] == len(rows)
            assert len(colstarts) == num_vertices + 1
        self.num_vertices = int(num_vertices)
        self._rows = rows
        self._colstarts = colstarts
        self._nnz = len(rows) if rows is not None else int(_nnz)
        self._adj = None
        self._sorted_rows = None
        self._handles = ([_device_csr], [None])  # (device CSR, BFS graph) handle boxes
        self._gpus, self._partitioned = 1, False
        self._finalizer = weakref.finalize(self, CsrGraph._release, *self._handles)

    @staticmethod
    def _release(csr_box, graph_box):
        lib = _lib.load()
        if graph_box[0]:
            lib.lbfs_graph_destroy(graph_box[0])
            graph_box[0] = None
        if csr_box[0]:
            lib.lbfs_csr_destroy(csr_box[0])
            csr_box[0] = None

    # -- host views ---------------------------------------------------------
    def _download(self, rows: bool = True):
        """Host copies of the device CSR, fetched on first use: row_ptr alone
        for degree queries (pick_roots, degrees), col_idx only when the rows
        themselves are read (an S27 col_idx is 17 GB)."""
        n = self.num_vertices
        if self._colstarts is None:
            cs = np.empty(n + 1, dtype=np.int64)
            _lib.check(_lib.load().lbfs_csr_download(self._handles[0][0], _lib.ptr(cs), None))
            self._colstarts = cs
        if rows and self._rows is None:
            r = _aligned_i32(self._nnz)
            if self._nnz:
                _lib.check(_lib.load().lbfs_csr_download(self._handles[0][0], None, _lib.ptr(r)))
            self._rows = r

    @property
    def rows(self) -> np.ndarray:
        if self._rows is None:
            self._download()
        return self._rows

    @property
    def colstarts(self) -> np.ndarray:
        if self._colstarts is None:
            self._download(rows=False)
        return self._colstarts

    @property
    def num_edges(self) -> int:
        return self._nnz

    def degree(self, u: int) -> int:
        assert 0 <= u < self.num_vertices
        return int(self.colstarts[u + 1] - self.colstarts[u])

    def degrees(self) -> np.ndarray:
        return np.diff(self.colstarts)

    def adjacency(self, u: int) -> np.ndarray:
        assert 0 <= u < self.num_vertices
        return self.rows[self.colstarts[u]:self.colstarts[u + 1]]

    def adjacency_lists(self) -> list[list[int]]:
        if self._adj is None:
            rows = self.rows.tolist()
            cs = self.colstarts.tolist()
            self._adj = [rows[cs[u]:cs[u + 1]] for u in range(self.num_vertices)]
        return self._adj

    def rows_sorted(self) -> bool:
        """True when every adjacency run is ascending (build_csr with dedup)."""
        if self._sorted_rows is None:
            r, cs = self.rows, self.colstarts
            if len(r) < 2:
                self._sorted_rows = True
            else:
                dec = np.nonzero(np.diff(r) < 0)[0] + 1  # positions where r drops
                starts = np.zeros(len(r), dtype=bool)
                starts[cs[:-1][cs[:-1] < len(r)]] = True
                self._sorted_rows = bool(np.all(starts[dec]))
        return self._sorted_rows

    # -- device handle (the BFS layout) --------------------------------------
    def device_handle(self, gpus: int | None = None, partitioned: bool = False) -> int:
        """The BFS graph handle, created on first use. ``gpus`` > 1 (or
        ``partitioned``) builds the 1D-partitioned graph over devices
        0..gpus-1 of this process (lbfs_graph_create_partitioned); a request
        for another device count replaces the handle."""
        box = self._handles[1]
        want = gpus if gpus is not None else (self._gpus if box[0] is not None else 1)
        want_part = partitioned or want > 1
        if box[0] is not None and (want != self._gpus or want_part != self._partitioned):
            from . import traversal

            traversal._release_handle(box[0])
            box[0] = None
        if box[0] is None:
            h = ctypes.c_void_p()
            lib = _lib.load()
            csr = self._handles[0][0]
            if want_part:
                if not csr:
                    self._upload_csr()
                    csr = self._handles[0][0]
                _lib.check(lib.lbfs_graph_create_partitioned(csr, int(want), None, ctypes.byref(h)))
            elif csr:
                _lib.check(lib.lbfs_graph_create_from_csr(csr, 1, ctypes.byref(h)))
            else:
                cs = np.ascontiguousarray(self._colstarts, dtype=np.int64)
                rows = np.ascontiguousarray(self._rows, dtype=np.int32)
                _lib.check(lib.lbfs_graph_create(self.num_vertices, _lib.ptr(cs),
                                                 _lib.ptr(rows) if len(rows) else None, len(rows), 1,
                                                 ctypes.byref(h)))
            box[0] = h.value
            self._gpus, self._partitioned = int(want), bool(want_part)
        return box[0]

    @property
    def gpus(self) -> int:
        return self._gpus if self._handles[1][0] is not None else 1

    def _upload_csr(self) -> None:
        """A device CSR from the host arrays (for the partitioned handle)."""
        h = ctypes.c_void_p()
        n = self.num_vertices
        cs = np.ascontiguousarray(self._colstarts, dtype=np.int64)
        rows = np.ascontiguousarray(self._rows, dtype=np.int32)
        src = np.repeat(np.arange(n, dtype=np.uint32), np.diff(cs).astype(np.int64))
        _lib.check(_lib.load().lbfs_csr_build(n, _lib.ptr(src), _lib.ptr(rows.view(np.uint32)) if len(rows) else None,
                                              len(rows), 0, 0, ctypes.byref(h)))
        self._handles[0][0] = h.value

    def release_device(self) -> None:
        """Free the device copies (they are rebuilt on the next BFS)."""
        if self._rows is None or self._colstarts is None:
            self._download()
        CsrGraph._release(self._handles[0], self._handles[1])


def _aligned_i32(n: int) -> np.ndarray:
    raw = np.empty(n * 4 + 64, dtype=np.uint8)
    off = (-raw.ctypes.data) % 64
    return raw[off:off + n * 4].view(np.int32)


def _from_device_csr(h: ctypes.c_void_p) -> CsrGraph:
    n, nnz = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.load().lbfs_csr_info(h, ctypes.byref(n), ctypes.byref(nnz)))
    return CsrGraph(n.value, None, None, _device_csr=h.value, _nnz=nnz.value)


def build_csr(e: EdgeList, symmetrize: bool = True, dedup: bool = True) -> CsrGraph:
    """Pack an edge list into CSR on the device (graph.py:139-160)."""
    src = np.ascontiguousarray(e.src, dtype=np.uint32)
    dst = np.ascontiguousarray(e.dst, dtype=np.uint32)
    h = ctypes.c_void_p()
    _lib.check(_lib.load().lbfs_csr_build(e.num_vertices, _lib.ptr(src) if len(src) else None,
                                          _lib.ptr(dst) if len(dst) else None, len(src),
                                          int(symmetrize), int(dedup), ctypes.byref(h)))
    return _from_device_csr(h)


def build_rmat_graph(p: RmatParams, permute: bool = True, perm_seed: int | None = None) -> CsrGraph:
    """generate_rmat -> permute_vertices -> build_csr, all on the device."""
    ab, an, cn = p.thresholds()
    st = p.pcg_state()
    seed = permutation_seed(p.seed) if perm_seed is None else int(perm_seed)
    h = ctypes.c_void_p()
    _lib.check(_lib.load().lbfs_csr_build_rmat(p.scale, p.edgefactor, ab, an, cn, _lib.ptr(st),
                                               int(permute), seed & (2**64 - 1), ctypes.byref(h)))
    return _from_device_csr(h)


def build_lattice_graph(rows: int, cols: int, permute: bool = True, perm_seed: int = 1) -> CsrGraph:
    """Config 4's lattice -> permute_vertices -> build_csr, on the device."""
    h = ctypes.c_void_p()
    _lib.check(_lib.load().lbfs_csr_build_lattice(rows, cols, int(permute), int(perm_seed) & (2**64 - 1),
                                                  ctypes.byref(h)))
    return _from_device_csr(h)


def write_edge_list(path: str | Path, e: EdgeList, params: RmatParams) -> None:
    """Binary little-endian (u, v) uint32 pairs plus a JSON sidecar (graph.py:163-171)."""
    path = Path(path)
    pairs = np.empty((e.edge_count, 2), dtype="<u4")
    pairs[:, 0] = e.src
    pairs[:, 1] = e.dst
    pairs.tofile(path)
    path.with_suffix(path.suffix + ".json").write_text(json.dumps(asdict(params)) + "\n")


def read_edge_list(path: str | Path) -> tuple[EdgeList, RmatParams]:
    path = Path(path)
    params = RmatParams(**json.loads(path.with_suffix(path.suffix + ".json").read_text()))
    pairs = np.fromfile(path, dtype="<u4").reshape(-1, 2)
    return EdgeList(pairs[:, 0].astype(np.uint32), pairs[:, 1].astype(np.uint32), params.num_vertices), params
