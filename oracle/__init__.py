"""CPU oracle for the B200 BFS — TEST INFRASTRUCTURE ONLY.

This package restates the reference ``lanebfs`` 0.1.0 algorithms for the hot
path (``/root/reference/pkg/src/lanebfs``) in plain C (``oracle.c``, built by
``oracle/Makefile`` into ``oracle/_build/liboracle.so``) plus a few numpy
helpers. It is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` legs may import it. The product package ``paper_1604_02844_b200``
never imports it and has no CPU fallback.

Parity pin: ``tests/test_oracle.py`` checks every function here against the
golden vectors in ``tests/golden/`` that ``tests/golden/make_golden.py``
produced by running the reference itself in the build container.

Function -> reference (file:line):
  rmat_edges        generate_rmat          graph.py:68-85
  permute_edges     build-defined seeded permutation
  build_csr         build_csr              graph.py:139-160
  lattice_edges     build-defined lattice
  bfs_serial        bfs_serial             traversal.py:80-104
  bfs_parallel      bfs_parallel_naive     traversal.py:128-165 (OpenMP)
  check_bfs         BFS certificate        SURVEY §8(c); validate.py:50-155
  levels_from_parents  levels_from_parents validate.py:158-177 (pointer doubling)
  pick_roots        pick_roots             harness.py:237-246
  harmonic_mean_teps harmonic_mean_teps    harness.py:218-234
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

SENTINEL = 0x7FFFFFFF
_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "liboracle.so"
_lib = None

_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_p = ctypes.c_void_p


def build() -> Path:
    """Compile the C oracle (gcc + OpenMP)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.oracle_rmat_edges.argtypes = [ctypes.c_int, _i64, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, _p, _p, _p]
        L.oracle_rmat_edges.restype = None
        L.oracle_permute_edges.argtypes = [_i64, _u64, _p, _p, _i64]
        L.oracle_permute_edges.restype = None
        L.oracle_permute_vertex.argtypes = [_u64, _u64, _u64]
        L.oracle_permute_vertex.restype = _u64
        L.oracle_lattice_edges.argtypes = [_i64, _i64, _p, _p]
        L.oracle_lattice_edges.restype = _i64
        L.oracle_build_csr_count.argtypes = [_i64, _p, _p, _i64, ctypes.c_int, ctypes.c_int, _p]
        L.oracle_build_csr_count.restype = _i64
        L.oracle_build_csr_fill.argtypes = [_i64, _p, _p, _i64, ctypes.c_int, ctypes.c_int, _p, _p]
        L.oracle_build_csr_fill.restype = _i64
        L.oracle_bfs_serial.argtypes = [_i64, _p, _p, _i64, _p, _p, _p, _i64]
        L.oracle_bfs_serial.restype = _i64
        L.oracle_bfs_parallel.argtypes = [_i64, _p, _p, _i64, _p, _p, _p, _i64, ctypes.c_int]
        L.oracle_bfs_parallel.restype = _i64
        L.oracle_check_bfs.argtypes = [_i64, _p, _p, _i64, _p, _p, ctypes.POINTER(_i64)]
        L.oracle_check_bfs.restype = ctypes.c_int
        L.oracle_max_threads.argtypes = []
        L.oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def max_threads() -> int:
    return int(lib().oracle_max_threads())


# ---------------------------------------------------------------- graph input

def pcg_state(seed: int) -> np.ndarray:
    """{state_hi, state_lo, inc_hi, inc_lo} of numpy default_rng(seed)'s PCG64
    (the generator graph.py:72 draws from)."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m64 = (1 << 64) - 1
    return np.array([s >> 64, s & m64, inc >> 64, inc & m64], dtype=np.uint64)


def rmat_thresholds(a: float, b: float, c: float, d: float) -> tuple[float, float, float]:
    """(ab, a_norm, c_norm) exactly as graph.py:74-77 computes them."""
    ab = a + b
    a_norm = a / ab if ab > 0 else 0.0
    c_norm = c / (c + d) if (c + d) > 0 else 0.0
    return ab, a_norm, c_norm


def rmat_edges(scale: int, edgefactor: int = 16, a=0.57, b=0.19, c=0.19, d=0.05, seed=1):
    m = (1 << scale) * edgefactor
    src = np.empty(m, dtype=np.uint32)
    dst = np.empty(m, dtype=np.uint32)
    ab, an, cn = rmat_thresholds(a, b, c, d)
    st = pcg_state(seed)
    lib().oracle_rmat_edges(scale, m, ab, an, cn, _ptr(st), _ptr(src), _ptr(dst))
    return src, dst


def permute_vertex(n: int, seed: int, v: int) -> int:
    return int(lib().oracle_permute_vertex(n, seed, v))


def permute_edges(n: int, seed: int, src: np.ndarray, dst: np.ndarray):
    src = np.ascontiguousarray(src, dtype=np.uint32).copy()
    dst = np.ascontiguousarray(dst, dtype=np.uint32).copy()
    lib().oracle_permute_edges(n, seed, _ptr(src), _ptr(dst), len(src))
    return src, dst


def lattice_edges(rows: int, cols: int):
    m = rows * (cols - 1) + (rows - 1) * cols
    src = np.empty(max(m, 0), dtype=np.uint32)
    dst = np.empty(max(m, 0), dtype=np.uint32)
    k = lib().oracle_lattice_edges(rows, cols, _ptr(src), _ptr(dst))
    assert k == m
    return src, dst


def build_csr(n: int, src, dst, symmetrize=True, dedup=True):
    """(colstarts int64[n+1], rows int32[nnz]) as graph.py:139-160 builds them."""
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    rp = np.empty(n + 1, dtype=np.int64)
    L = lib()
    ub = L.oracle_build_csr_count(n, _ptr(src), _ptr(dst), len(src), int(symmetrize), int(dedup), _ptr(rp))
    ci = np.empty(max(ub, 1), dtype=np.int32)
    nnz = L.oracle_build_csr_fill(n, _ptr(src), _ptr(dst), len(src), int(symmetrize), int(dedup),
                                  _ptr(rp), _ptr(ci))
    return rp, ci[:nnz].copy()


# ---------------------------------------------------------------- traversal

def _layers(buf: np.ndarray, k: int):
    return [tuple(int(x) for x in buf[3 * i:3 * i + 3]) for i in range(k)]


def _run(fn, n, rp, ci, root, *extra):
    pred = np.empty(max(n, 1), dtype=np.int32)
    level = np.empty(max(n, 1), dtype=np.int32)
    cap = 64
    while True:
        buf = np.zeros(3 * cap, dtype=np.int64)
        k = fn(n, _ptr(rp), _ptr(ci), root, _ptr(pred), _ptr(level), _ptr(buf), cap, *extra)
        if k <= cap:
            return pred[:n], level[:n], _layers(buf, k)
        cap = int(k)


def bfs_serial(rp: np.ndarray, ci: np.ndarray, root: int):
    """(pred int32[n], level int32[n], layers [(input, edges, discovered)])."""
    n = len(rp) - 1
    assert 0 <= root < n
    return _run(lib().oracle_bfs_serial, n, rp, ci, root)


def bfs_parallel(rp: np.ndarray, ci: np.ndarray, root: int, threads: int = 0):
    n = len(rp) - 1
    assert 0 <= root < n
    return _run(lib().oracle_bfs_parallel, n, rp, ci, root, threads)


CHECK_CODES = {0: "ok", 1: "root", 2: "reached/pred mismatch", 3: "parent out of range",
               4: "parent not one level up", 5: "tree edge absent", 6: "edge leaves the reached set",
               7: "edge spans more than one level"}


def check_bfs(rp, ci, root, pred, level) -> tuple[int, int]:
    """BFS certificate: (code, first offending vertex); code 0 = exact BFS."""
    n = len(rp) - 1
    pred = np.ascontiguousarray(pred[:n], dtype=np.int32)
    level = np.ascontiguousarray(level[:n], dtype=np.int32)
    where = _i64(-1)
    code = lib().oracle_check_bfs(n, _ptr(rp), _ptr(ci), root, _ptr(pred), _ptr(level), ctypes.byref(where))
    return int(code), int(where.value)


def levels_from_parents(p, s: int) -> np.ndarray:
    """validate.py:158-177 restated by pointer doubling: level = length of the
    parent chain from v to s when that chain reaches a self-parented s, else -1."""
    p = np.asarray(p, dtype=np.int64)
    n = len(p)
    lev = np.full(n, -1, dtype=np.int64)
    if n == 0 or p[s] != s:
        return lev
    valid = (p >= 0) & (p < n) & (p != SENTINEL)
    sink = n
    anc = np.where(valid, p, sink)
    anc = np.append(anc, sink)
    anc[s] = s
    dist = np.ones(n + 1, dtype=np.int64)
    dist[s] = 0
    dist[sink] = 0
    for _ in range(max(1, math.ceil(math.log2(n + 1))) + 1):
        dist = dist + dist[anc]
        anc = anc[anc]
    ok = anc[:n] == s
    lev[ok] = dist[:n][ok]
    return lev


def pick_roots(degrees: np.ndarray, k: int, seed: int, filter_unconnected: bool = True) -> np.ndarray:
    """harness.py:237-246."""
    pool = np.arange(len(degrees), dtype=np.int64)
    if filter_unconnected:
        pool = pool[degrees > 0]
    assert k <= len(pool)
    return np.random.default_rng(seed).choice(pool, size=k, replace=False)


def harmonic_mean_teps(values) -> float:
    """harness.py:218-234 (include_zeros=False)."""
    nz = [float(v) for v in values if float(v) > 0.0]
    return len(nz) / math.fsum(1.0 / v for v in nz) if nz else 0.0
