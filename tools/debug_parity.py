"""Dev probe: device BFS levels vs the oracle at SCALE S; prints mismatch histogram."""
import sys, collections
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import oracle
from paper_1604_02844_b200 import RmatParams, bfs, build_rmat_graph, pick_roots

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = build_rmat_graph(RmatParams(scale=scale, seed=1))
rp, ci = g.colstarts, g.rows
for r in pick_roots(g, 64, 1, filter_unconnected=True).tolist()[:int(sys.argv[2]) if len(sys.argv) > 2 else 3]:
    res = bfs(g, r)
    _, lvl, layers = oracle.bfs_parallel(rp, ci, r)
    bad = np.nonzero(res.levels != lvl)[0]
    print("root", r, "mismatches", len(bad), "layers gpu", [(l.input, l.discovered) for l in res.layers], "oracle", [(x[0], x[2]) for x in layers])
    if len(bad):
        c = collections.Counter(zip(res.levels[bad].tolist(), lvl[bad].tolist()))
        print("  (gpu, oracle) level pairs:", c.most_common(8))
