"""Dev probe: one BFS on an R-MAT graph (scale, seed, root index among pick_roots(8, 5))."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import oracle
from paper_1604_02844_b200 import RmatParams, build_rmat_graph, bfs
scale, seed, idx = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (12, 2, 1)))
g = build_rmat_graph(RmatParams(scale=scale, edgefactor=16, seed=seed))
rp, ci = g.colstarts, g.rows
root = int(oracle.pick_roots(np.diff(rp), 8, 5)[idx])
print("root", root, "deg", rp[root + 1] - rp[root], flush=True)
r = bfs(g, root)
_, lv, layers = oracle.bfs_serial(rp, ci, root)
print("ok" if np.array_equal(r.levels, lv) else "MISMATCH", [(l.input, l.edges, l.discovered) for l in r.layers])
