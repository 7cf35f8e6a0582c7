"""Tree validator of the BFS result — the reference validate.py API
(/root/reference/pkg/src/lanebfs/validate.py) in vectorised form.

``validate_tree`` evaluates the same five checks with the same first-offender
``details`` as the reference's per-vertex Python loops (validate.py:50-155),
but in O((n + reached) log n) array passes, so SCALE-24/27 trees validate in
seconds instead of minutes. ``levels_from_parents``
(validate.py:158-177) uses pointer doubling: ceil(log2 n) gather rounds
instead of one relaxation round per level (the lattice has ~8K levels).
``bfs_certificate`` adds the edge-span check that makes a level array exactly
the BFS distances; the reference omits it.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import numpy as np

from .traversal import SENTINEL

_OK, _PSEUDO, _CYCLE, _BROKEN = 1, 2, 3, 4


@dataclass
class ValidationReport:
    """Outcome of the five checks (validate.py:21-47)."""

    root_self_parent: bool
    reachability_closure: bool
    tree_edge_existence: bool
    level_consistency: bool
    cycle_freedom: bool
    details: dict[str, int] = field(default_factory=dict)

    CHECKS = ("root_self_parent", "reachability_closure", "tree_edge_existence",
              "level_consistency", "cycle_freedom")

    @property
    def passed(self) -> bool:
        return all(getattr(self, name) for name in self.CHECKS)

    def as_dict(self) -> dict:
        d = {name: getattr(self, name) for name in self.CHECKS}
        d["passed"] = self.passed
        d["details"] = dict(self.details)
        return d

    def to_json(self) -> str:
        return json.dumps(self.as_dict())


def _parent_array(pred) -> np.ndarray:
    p = pred.p if hasattr(pred, "p") else pred
    return np.asarray(p, dtype=np.int64)


def _has_edges(g, u: np.ndarray, v: np.ndarray) -> np.ndarray:
    """Vectorised `v in adj(u)` for in-range u."""
    cs = np.asarray(g.colstarts, dtype=np.int64)
    rows = np.asarray(g.rows)
    if len(u) == 0:
        return np.zeros(0, dtype=bool)
    sorted_rows = g.rows_sorted() if hasattr(g, "rows_sorted") else _rows_sorted(rows, cs)
    if not sorted_rows:
        n = np.int64(g.num_vertices)
        owner = np.repeat(np.arange(g.num_vertices, dtype=np.int64), np.diff(cs))
        keys = np.sort(owner * n + rows.astype(np.int64))
        q = u * n + v
        pos = np.searchsorted(keys, q)
        return (pos < len(keys)) & (keys[np.minimum(pos, len(keys) - 1)] == q)
    lo = cs[u].copy()
    hi = cs[u + 1].copy()
    end = hi.copy()
    # branch-free binary search, all queries in lockstep
    while True:
        act = lo < hi
        if not act.any():
            break
        mid = (lo + hi) >> 1
        mid_c = np.minimum(mid, max(len(rows) - 1, 0))
        less = act & (rows[mid_c] < v)
        lo = np.where(less, mid + 1, lo)
        hi = np.where(act & ~less, mid, hi)
    ok = lo < end
    ok[ok] = rows[lo[ok]] == v[ok]
    return ok


def _rows_sorted(rows: np.ndarray, cs: np.ndarray) -> bool:
    if len(rows) < 2:
        return True
    dec = np.nonzero(np.diff(rows) < 0)[0] + 1
    starts = np.zeros(len(rows), dtype=bool)
    starts[cs[:-1][cs[:-1] < len(rows)]] = True
    return bool(np.all(starts[dec]))


def _classify(p: np.ndarray, s: int) -> np.ndarray:
    """Status of every vertex under the reference's memoised parent chase
    (validate.py:104-142): chains ending at s are OK; a vertex whose own
    parent is invalid terminates chains as BROKEN but is itself left
    unclassified (0); a self-parented non-root is PSEUDO; chains that never
    reach a terminal are CYCLE."""
    n = len(p)
    idx = np.arange(n, dtype=np.int64)
    invalid = (p < 0) | (p >= n) | (p == SENTINEL)
    pseudo = (p == idx) & (idx != s)
    terminal = invalid | pseudo
    terminal[s] = True
    nxt = np.where(terminal, idx, np.where(invalid, 0, p))
    anc = nxt.copy()
    for _ in range(max(1, math.ceil(math.log2(n + 1))) + 1):
        anc = anc[anc]
    end = anc
    status = np.full(n, _CYCLE, dtype=np.int8)
    fixed = nxt[end] == end
    status[fixed & (end == s)] = _OK
    status[fixed & invalid[end]] = _BROKEN
    status[fixed & pseudo[end]] = _PSEUDO
    status[invalid] = 0
    status[s] = _OK
    return status


def validate_tree(g, s: int, pred) -> ValidationReport:
    """The five checks of validate.py:50-155, vectorised. Failures are report
    entries, never exceptions; details hold the first offender per check."""
    n = g.num_vertices
    assert 0 <= s < n
    p = _parent_array(pred)[:n]
    details: dict[str, int] = {}

    ok_root = bool(p[s] == s)
    if not ok_root:
        details["root_self_parent"] = int(s)

    reached = np.nonzero(p != SENTINEL)[0]

    # 2. reachability closure, first failing reached vertex in ascending order
    u = p[reached]
    inr = (u >= 0) & (u < n)
    bad = ~inr
    bad[inr] = p[u[inr]] == SENTINEL
    ok_closure = not bad.any()
    if not ok_closure:
        details["reachability_closure"] = int(reached[np.argmax(bad)])

    # 3. tree-edge existence: parents visited in ascending order; the first
    # failing parent reports its smallest offending child
    ch = reached[reached != s]
    par = p[ch]
    out = (par < 0) | (par >= n)
    badc = out.copy()
    inn = ~out
    badc[inn] = ~_has_edges(g, par[inn], ch[inn])
    ok_edges = not badc.any()
    if not ok_edges:
        bp, bc = par[badc], ch[badc]
        first_parent = bp.min()
        details["tree_edge_existence"] = int(bc[bp == first_parent].min())

    # 4/5. memoised chase classification
    status = _classify(p, s)
    st = status[reached]
    lvl_bad = (st == _CYCLE) | (st == _BROKEN)
    ok_levels = not lvl_bad.any()
    if not ok_levels:
        details["level_consistency"] = int(reached[np.argmax(lvl_bad)])
    acyc_bad = st != _OK
    ok_acyclic = not acyc_bad.any()
    if not ok_acyclic:
        details["cycle_freedom"] = int(reached[np.argmax(acyc_bad)])

    return ValidationReport(ok_root, ok_closure, ok_edges, ok_levels, ok_acyclic, details)


def validate_tree_device(g, s: int, pred) -> ValidationReport:
    """``validate_tree`` on the GPU (csrc/validate.cu): the same five checks
    and first offenders; the parent array goes to the device once and the
    memoised chases become pointer jumping. ``g`` is any graph ``bfs``
    accepts; ``pred`` a PredecessorArray, an int array of n entries, or a
    device tensor (anything with ``data_ptr()`` on the graph's device)."""
    import ctypes

    from . import _lib
    from .traversal import _handle

    n = g.num_vertices
    assert 0 <= s < n
    if getattr(g, "_partitioned", False) and g._handles[1][0] is not None:
        # a partitioned handle has no whole-graph layout on one device: the
        # vectorised host validator (same checks, same report)
        return validate_tree(g, s, pred.cpu().numpy() if hasattr(pred, "cpu") else pred)
    h = _handle(g)
    rep = (ctypes.c_int64 * 10)()
    lib = _lib.load()
    if hasattr(pred, "data_ptr") and getattr(pred, "is_cuda", False):
        assert pred.numel() >= n
        _lib.check(lib.lbfs_validate_tree_device(h, int(s), pred.data_ptr(), rep))
    else:
        p = np.ascontiguousarray(_parent_array(pred)[:n], dtype=np.int32)
        assert len(p) == n
        _lib.check(lib.lbfs_validate_tree(h, int(s), _lib.ptr(p), rep))
    flags = [bool(rep[k]) for k in range(5)]
    details = {name: int(rep[5 + k]) for k, name in enumerate(ValidationReport.CHECKS) if not flags[k]}
    return ValidationReport(*flags, details)


def levels_from_parents(p, s: int) -> np.ndarray:
    """Per-vertex level implied by a parent array, -1 where undefined
    (validate.py:158-177): the length of v's parent chain to a self-parented
    root s, by pointer doubling."""
    p = np.asarray(p, dtype=np.int64)
    n = len(p)
    lev = np.full(n, -1, dtype=np.int64)
    if n == 0 or p[s] != s:
        return lev
    valid = (p >= 0) & (p < n) & (p != SENTINEL)
    anc = np.append(np.where(valid, p, n), n)  # index n is an absorbing sink
    anc[s] = s
    hops = np.ones(n + 1, dtype=np.int64)
    hops[s] = 0
    hops[n] = 0
    for _ in range(max(1, math.ceil(math.log2(n + 1))) + 1):
        hops = hops + hops[anc]
        anc = anc[anc]
    reach = anc[:n] == s
    lev[reach] = hops[:n][reach]
    return lev


@dataclass
class Certificate:
    passed: bool
    reason: str = ""
    vertex: int = -1


def bfs_certificate(g, s: int, pred, levels) -> Certificate:
    """Exact-BFS certificate: (i) root level 0 and self-parented; (ii) every
    reached v != s has a neighbour parent one level up; (iii) every CSR edge
    joins two reached vertices at most one level apart, or two unreached
    ones. (i)-(iii) imply levels are the BFS distances from s."""
    n = g.num_vertices
    p = _parent_array(pred)[:n]
    lv = np.asarray(levels, dtype=np.int64)[:n]
    if lv[s] != 0 or p[s] != s:
        return Certificate(False, "root", int(s))
    reached = lv >= 0
    mism = reached != (p != SENTINEL)
    if mism.any():
        return Certificate(False, "reached set differs from predecessor set", int(np.argmax(mism)))
    ch = np.nonzero(reached)[0]
    ch = ch[ch != s]
    par = p[ch]
    out = (par < 0) | (par >= n)
    if out.any():
        return Certificate(False, "parent out of range", int(ch[np.argmax(out)]))
    up = lv[par] != lv[ch] - 1
    if up.any():
        return Certificate(False, "parent not one level up", int(ch[np.argmax(up)]))
    miss = ~_has_edges(g, par, ch)
    if miss.any():
        return Certificate(False, "tree edge absent", int(ch[np.argmax(miss)]))
    cs = np.asarray(g.colstarts, dtype=np.int64)
    rows = np.asarray(g.rows, dtype=np.int64)
    owner = np.repeat(np.arange(n, dtype=np.int64), np.diff(cs))
    la, lb = lv[owner], lv[rows]
    bad = ((la >= 0) != (lb >= 0)) | ((la >= 0) & (np.abs(la - lb) > 1))
    if bad.any():
        return Certificate(False, "edge spans more than one level or leaves the reached set",
                           int(owner[np.argmax(bad)]))
    return Certificate(True)
