"""Correctness stress: many certified BFS on one graph.

Every BFS (device outputs) is certified on the device, outside any timing:
  * its level array equals the oracle's (oracle.bfs_parallel, computed once
    per root on the host and kept on the GPU as int16),
  * its layers equal the oracle's,
  * its parent array passes the reference's five validate_tree checks
    (lbfs_validate_tree_device).
Stops at the first failure (exit 1) and prints one JSON summary line.

    python tools/stress.py --scale 24 --bfs 100000 [--lattice 4096] [--log FILE]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1604_02844_b200 import (RmatParams, bfs_device, build_lattice_graph, build_rmat_graph,  # noqa: E402
                                   pick_roots)
from paper_1604_02844_b200.validate import validate_tree_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--lattice", type=int, default=0, help="side of a permuted lattice instead of R-MAT")
    ap.add_argument("--roots", type=int, default=64)
    ap.add_argument("--bfs", type=int, default=10000)
    ap.add_argument("--direction", default="top_down")
    ap.add_argument("--log", default=None)
    ap.add_argument("--tree-every", type=int, default=1, help="validate_tree on every k-th BFS (levels: every BFS)")
    ap.add_argument("--root", type=int, action="append", default=None, help="explicit root(s) instead of pick_roots")
    a = ap.parse_args()
    t0 = time.time()
    if a.lattice:
        g = build_lattice_graph(a.lattice, a.lattice)
        name = f"lattice{a.lattice}"
    else:
        g = build_rmat_graph(RmatParams(scale=a.scale, seed=1))
        name = f"rmat-s{a.scale}"
    n = g.num_vertices
    rp, ci = g.colstarts, g.rows
    roots = a.root or pick_roots(g, a.roots, 1, filter_unconnected=True).tolist()
    want_lvl, want_layers = [], []
    for r in roots:
        _, lvl, layers = oracle.bfs_parallel(rp, ci, r)
        want_lvl.append(torch.from_numpy(lvl.astype(np.int16)).cuda())
        want_layers.append([tuple(x) for x in layers])
    prep_s = time.time() - t0
    pred = torch.empty((n + 31) // 32 * 32, dtype=torch.int32, device="cuda")
    lvl = torch.empty(n, dtype=torch.int32, device="cuda")
    t1 = time.time()
    done, fail, trees = 0, None, 0
    while done < a.bfs and fail is None:
        for i, r in enumerate(roots):
            if done >= a.bfs:
                break
            try:
                res = bfs_device(g, r, pred, lvl, direction=a.direction)
            except RuntimeError as e:
                fail = f"root {r}: {e}"
                done += 1
                break
            layers = [(x.input, x.edges, x.discovered) for x in res.layers]
            if layers != want_layers[i]:
                fail = f"root {r}: layers differ"
            elif not torch.equal(lvl.to(torch.int16), want_lvl[i]):
                bad = int((lvl.to(torch.int16) != want_lvl[i]).sum())
                fail = f"root {r}: {bad} levels differ"
            elif done % a.tree_every == 0:
                rep = validate_tree_device(g, r, pred)
                trees += 1
                if not rep.passed:
                    fail = f"root {r}: validate_tree failed {rep.details}"
            done += 1
            if fail:
                break
    out = {"graph": name, "n": n, "nnz": g.num_edges, "roots": len(roots), "direction": a.direction,
           "certified_bfs": done - (1 if fail else 0), "trees_validated": trees, "failure": fail, "prep_s": round(prep_s, 1),
           "stress_s": round(time.time() - t1, 1),
           "checks": "levels == oracle bfs_parallel, layers == oracle, validate_tree (5 checks) on device"}
    line = json.dumps(out)
    print(line, flush=True)
    if a.log:
        Path(a.log).parent.mkdir(parents=True, exist_ok=True)
        with open(a.log, "a") as f:
            f.write(line + "\n")
    sys.exit(1 if fail else 0)


if __name__ == "__main__":
    main()
