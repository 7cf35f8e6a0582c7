"""Dev probe: single-GPU levels vs the oracle on S14 for a few roots."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import oracle
from paper_1604_02844_b200 import RmatParams, build_rmat_graph, bfs
g = build_rmat_graph(RmatParams(scale=int(sys.argv[1]) if len(sys.argv) > 1 else 14, edgefactor=16, seed=2))
rp, ci = g.colstarts, g.rows
bad = 0
for root in oracle.pick_roots(np.diff(rp), 8, 5):
    r = bfs(g, int(root))
    _, lv, layers = oracle.bfs_serial(rp, ci, int(root))
    ok = np.array_equal(r.levels, lv)
    if not ok:
        bad += 1
        d = np.nonzero(r.levels != lv)[0]
        print("root", root, "mismatch", len(d), "first", d[:5], "got", r.levels[d[:5]], "want", lv[d[:5]],
              "deg", np.diff(rp)[d[:5]])
print("bad roots", bad)
from paper_1604_02844_b200.distributed import PartitionedGraph, LocalExchange, bfs_partitioned
for P in (1, 2):
    parts = [PartitionedGraph(g, r, P) for r in range(P)]
    bad = 0
    for root in list(oracle.pick_roots(np.diff(rp), 4, 5)) * 3:
        res = bfs_partitioned(parts, int(root), LocalExchange())
        _, lv, layers = oracle.bfs_serial(rp, ci, int(root))
        got = res.level[0].cpu().numpy()
        if not np.array_equal(got, lv):
            bad += 1
            d = np.nonzero(got != lv)[0]
            print("P", P, "root", root, "mismatch", len(d), "got", got[d[:5]], "want", lv[d[:5]], "deg", np.diff(rp)[d[:5]])
    print("P", P, "bad", bad)
