"""Generate the golden vectors that pin the oracle (and through it the GPU path).

Runs the REFERENCE package itself (``lanebfs`` from /root/reference/pkg/src)
in the build container; it never runs on the GPU box. Output: small fixtures
in tests/golden/ (committed). Usage:

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests:. \
        python tests/golden/make_golden.py            # small + S16 + S20 + lattices
    ... python tests/golden/make_golden.py --big      # adds S24 (≈15 min, ≈46 GB RAM)

The vertex permutation (gap G1: the reference has none) is the build-defined
Feistel bijection restated in oracle/oracle.c; the permuted edge list is fed to
the reference's own build_csr, so the CSR hashes pin our construction against
the reference's.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

import lanebfs  # noqa: E402  (the reference)
from lanebfs.graph import EdgeList, RmatParams, build_csr, generate_rmat  # noqa: E402
from lanebfs.harness import harmonic_mean_teps, pick_roots  # noqa: E402
from lanebfs.traversal import SENTINEL, bfs_parallel_naive, bfs_serial, bfs_vectorized  # noqa: E402
from lanebfs.validate import levels_from_parents, validate_tree  # noqa: E402

import oracle  # noqa: E402  (only for the build-defined permutation / lattice pairs)

PERM_SEED_OFFSET = 0  # permutation seed = RmatParams.seed


def sha(a, dtype) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dtype).tobytes()).hexdigest()[:32]


def layers_list(res):
    return [[l.input, l.edges, l.discovered] for l in res.layers]


def from_pairs(pairs, n, symmetrize=True, dedup=True):
    arr = np.array(pairs, dtype=np.uint32).reshape(-1, 2)
    return build_csr(EdgeList(arr[:, 0].copy(), arr[:, 1].copy(), n), symmetrize, dedup), arr


def small_graphs():
    g = {}
    g["path3"] = ([(0, 1), (1, 2)], 3, [0])
    g["single"] = ([], 1, [0])
    g["diamond"] = ([(0, 1), (0, 2), (1, 3), (2, 3)], 4, [0, 3])
    g["shared_word"] = ([(0, 5), (0, 9)], 16, [0])
    g["triangle"] = ([(0, 1), (1, 2), (2, 0)], 3, [0])
    g["path33"] = ([(i, i + 1) for i in range(32)], 33, [16, 0, 32])
    g["star101"] = ([(0, i) for i in range(1, 101)], 101, [0, 7])
    g["clique24"] = ([(i, j) for i in range(24) for j in range(i + 1, 24)], 24, [0, 23])
    k = 8
    pairs = [(i, j) for i in range(k) for j in range(i + 1, k)]
    pairs += [(k + i, k + j) for i in range(k) for j in range(i + 1, k)]
    g["disconnected16"] = (pairs, 2 * k, [0, 1, 9])
    g["empty7"] = ([], 7, [0, 3])
    g["disconnected8"] = ([(i, j) for i in range(4) for j in range(i + 1, 4)]
                          + [(4 + i, 4 + j) for i in range(4) for j in range(i + 1, 4)], 8, [1])
    g["dups_loops"] = ([(0, 1), (1, 0), (0, 1), (2, 2), (1, 2), (3, 3)], 5, [0, 3])
    return g


def make_small(out: dict, arrays: dict):
    rec = {}
    for name, (pairs, n, roots) in small_graphs().items():
        entry = {"n": n, "pairs": [list(p) for p in pairs], "csr": {}, "bfs": {}}
        arr = np.array(pairs, dtype=np.uint32).reshape(-1, 2)
        for sym in (True, False):
            for dd in (True, False):
                g = build_csr(EdgeList(arr[:, 0].copy(), arr[:, 1].copy(), n), sym, dd)
                entry["csr"][f"{int(sym)}{int(dd)}"] = {"colstarts": g.colstarts.tolist(),
                                                      "rows": g.rows.tolist()}
        g, _ = from_pairs(pairs, n)
        for s in roots:
            res = bfs_serial(g, s)
            entry["bfs"][str(s)] = {
                "pred": res.predecessors.p.tolist(),
                "storage_len": len(res.predecessors.storage),
                "layers": layers_list(res),
                "edges": res.traversed_edge_count,
                "levels": levels_from_parents(res.predecessors.p, s).tolist(),
            }
        rec[name] = entry
    out["small"] = rec


def make_rmat_small(out: dict, arrays: dict):
    rec = []
    for scale, ef, seed in [(4, 8, 0), (5, 16, 1), (6, 8, 7), (7, 16, 3), (8, 16, 5), (9, 8, 2),
                            (10, 16, 1), (12, 16, 1)]:
        p = RmatParams(scale=scale, edgefactor=ef, seed=seed)
        e = generate_rmat(p)
        g = build_csr(e)
        key = f"s{scale}_e{ef}_r{seed}"
        item = {"scale": scale, "edgefactor": ef, "seed": seed, "m": e.edge_count,
                "src_sha": sha(e.src, "<u4"), "dst_sha": sha(e.dst, "<u4"),
                "colstarts_sha": sha(g.colstarts, "<i8"), "rows_sha": sha(g.rows, "<i4"),
                "nnz": g.num_edges, "bfs": {}}
        if scale <= 8:
            arrays[f"{key}_src"] = e.src
            arrays[f"{key}_dst"] = e.dst
        rng = np.random.default_rng(seed + 100)
        roots = sorted(set(int(x) for x in rng.integers(0, g.num_vertices, 3)))
        for s in roots:
            res = bfs_serial(g, s)
            item["bfs"][str(s)] = {"pred_sha": sha(res.predecessors.p, "<i4"),
                                   "layers": layers_list(res),
                                   "levels_sha": sha(levels_from_parents(res.predecessors.p, s), "<i4")}
            if scale <= 8:
                arrays[f"{key}_pred_{s}"] = res.predecessors.p.copy()
        rec.append(item)
    out["rmat_small"] = rec


def permuted_rmat(scale, seed=1):
    p = RmatParams(scale=scale, seed=seed)
    t = time.time()
    e = generate_rmat(p)
    src_sha, dst_sha = sha(e.src, "<u4"), sha(e.dst, "<u4")
    ps, pd = oracle.permute_edges(p.num_vertices, seed + PERM_SEED_OFFSET, e.src, e.dst)
    e2 = EdgeList(ps, pd, p.num_vertices)
    g = build_csr(e2)
    print(f"  S{scale}: gen+perm+csr {time.time() - t:.1f}s nnz={g.num_edges}", flush=True)
    return p, g, {"src_sha": src_sha, "dst_sha": dst_sha, "psrc_sha": sha(ps, "<u4"),
                  "pdst_sha": sha(pd, "<u4"), "colstarts_sha": sha(g.colstarts, "<i8"),
                  "rows_sha": sha(g.rows, "<i4"), "nnz": g.num_edges, "n": g.num_vertices}


def make_config(out, arrays, scale, nroots, nbfs, mode, store_levels):
    p, g, info = permuted_rmat(scale)
    roots = pick_roots(g, nroots, p.seed, filter_unconnected=True)
    info["roots"] = [int(r) for r in roots]
    info["degree_hist"] = np.bincount(np.minimum(g.degrees(), 64)).tolist()
    bfs = {}
    for s in info["roots"][:nbfs]:
        t = time.time()
        res = bfs_serial(g, s) if mode == "serial" else (
            bfs_parallel_naive(g, s, 8) if mode == "naive" else bfs_vectorized(g, s, 8))
        lev = levels_from_parents(res.predecessors.p, s) if mode != "vectorized_fast" else None
        rep = validate_tree(g, s, res.predecessors) if scale <= 20 else None
        item = {"layers": layers_list(res), "edges": res.traversed_edge_count,
                "levels_sha": sha(lev, "<i4"),
                "reached": int((res.predecessors.p != SENTINEL).sum())}
        if mode == "serial":
            item["pred_sha"] = sha(res.predecessors.p, "<i4")
        if rep is not None:
            item["validate_passed"] = rep.passed
        if store_levels:
            arrays[f"S{scale}_levels_{s}"] = lev.astype(np.int8)
        bfs[str(s)] = item
        print(f"    root {s}: {time.time() - t:.1f}s layers={len(res.layers)}", flush=True)
    info["bfs"] = bfs
    out[f"S{scale}"] = info


def make_lattice(out, arrays, rows, cols, nroots, nbfs, exact_levels):
    n = rows * cols
    src, dst = oracle.lattice_edges(rows, cols)
    ps, pd = oracle.permute_edges(n, 1 + PERM_SEED_OFFSET, src, dst)
    t = time.time()
    g = build_csr(EdgeList(ps, pd, n))
    info = {"rows": rows, "cols": cols, "n": n, "nnz": g.num_edges,
            "src_sha": sha(src, "<u4"), "psrc_sha": sha(ps, "<u4"), "pdst_sha": sha(pd, "<u4"),
            "colstarts_sha": sha(g.colstarts, "<i8"), "rows_sha": sha(g.rows, "<i4")}
    print(f"  lattice {rows}x{cols}: csr {time.time() - t:.1f}s", flush=True)
    roots = pick_roots(g, nroots, 1, filter_unconnected=True)
    info["roots"] = [int(r) for r in roots]
    bfs = {}
    for s in info["roots"][:nbfs]:
        t = time.time()
        res = bfs_parallel_naive(g, s, 8)
        item = {"layers": layers_list(res), "edges": res.traversed_edge_count}
        if exact_levels:
            item["levels_sha"] = sha(levels_from_parents(res.predecessors.p, s), "<i4")
        bfs[str(s)] = item
        print(f"    root {s}: {time.time() - t:.1f}s layers={len(res.layers)}", flush=True)
    info["bfs"] = bfs
    out[f"lattice_{rows}x{cols}"] = info


def make_validator(out, arrays):
    """validate_tree / levels_from_parents on the reference mutation catalog."""
    import helpers  # reference tests/helpers.py
    cases = []
    rng = np.random.default_rng(11)
    graphs = [("rmat7", helpers.rmat_graph(7, seed=3), 5), ("path33", helpers.path_graph(33), 16),
              ("clique12", helpers.clique_graph(12), 0), ("star40", helpers.star_graph(40), 0),
              ("disc", helpers.disconnected_graph(6), 2)]
    for gname, g, s in graphs:
        base = bfs_serial(g, s).predecessors.p.tolist()
        variants = [("valid", base)]
        for mname, mut in helpers.MUTATIONS:
            for k in range(2):
                q = mut(rng, g, s, base)
                if q is not None:
                    variants.append((f"{mname}{k}", q))
        # hand-made corner cases: out-of-range parent, negative parent, 3-cycle
        q = list(base); v = next(i for i in range(len(q)) if q[i] != SENTINEL and i != s); q[v] = len(q) + 3
        variants.append(("out_of_range", q))
        q = list(base); q[v] = -2
        variants.append(("negative", q))
        for vname, q in variants:
            pred = lanebfs.PredecessorArray(g.num_vertices)
            pred.p[:] = q
            rep = validate_tree(g, s, pred)
            cases.append({"graph": gname, "root": s, "variant": vname, "pred": [int(x) for x in q],
                          "report": rep.as_dict(),
                          "levels": levels_from_parents(np.array(q), s).tolist()})
    out["validator"] = {"graphs": {name: {"colstarts": g.colstarts.tolist(), "rows": g.rows.tolist()}
                                   for name, g, _ in graphs}, "cases": cases}
    out["harmonic"] = [
        {"values": v, "include_zeros": z, "result": list(harmonic_mean_teps(v, z))}
        for v, z in [([1.0, 2.0, 4.0], False), ([0.0, 2.0, 2.0], False), ([0.0, 2.0], True),
                     ([0.0, 0.0], False), ([3e9, 1e9], False)]]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    out_json = HERE / "golden.json"
    out = json.loads(out_json.read_text()) if out_json.exists() else {}
    arrays_path = HERE / "golden_arrays.npz"
    arrays = dict(np.load(arrays_path)) if arrays_path.exists() else {}
    out["reference"] = {"package": "lanebfs", "version": lanebfs.__version__,
                        "numpy": np.__version__}
    steps = {
        "small": lambda: make_small(out, arrays),
        "rmat_small": lambda: make_rmat_small(out, arrays),
        "validator": lambda: make_validator(out, arrays),
        "S16": lambda: make_config(out, arrays, 16, 8, 8, "serial", True),
        "S20": lambda: make_config(out, arrays, 20, 64, 4, "naive", False),
        "lattice_small": lambda: make_lattice(out, arrays, 64, 48, 4, 4, True),
        "lattice_big": lambda: make_lattice(out, arrays, 4096, 4096, 16, 2, False),
    }
    if args.big:
        steps = {"S24": lambda: make_config(out, arrays, 24, 64, 4, "vectorized", False)}
    for name, fn in steps.items():
        if args.only and name not in args.only.split(","):
            continue
        t = time.time()
        print(f"[{name}]", flush=True)
        fn()
        print(f"[{name}] {time.time() - t:.1f}s", flush=True)
        out_json.write_text(json.dumps(out, separators=(",", ":")) + "\n")
        np.savez_compressed(arrays_path, **arrays)


if __name__ == "__main__":
    main()
