"""Dev probe: partitioned vs single-GPU layers on the test's roots."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import oracle
from paper_1604_02844_b200 import RmatParams, build_rmat_graph, bfs
from paper_1604_02844_b200.distributed import PartitionedGraph, LocalExchange, bfs_partitioned
from oracle.part_emu import EmuPart

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g = build_rmat_graph(RmatParams(scale=14, edgefactor=16, seed=2))
rp, ci, n = g.colstarts, g.rows, g.num_vertices
roots = [int(r) for r in oracle.pick_roots(np.diff(rp), 4, 5)]
parts = [PartitionedGraph(g, r, P) for r in range(P)]
emu = [EmuPart(n, rp, ci, r, P) for r in range(P)]
for root in roots + roots[::-1]:
    fresh = [PartitionedGraph(g, r, P) for r in range(P)]
    a = bfs_partitioned(parts, root, LocalExchange()).layers[:2]
    f = bfs_partitioned(fresh, root, LocalExchange()).layers[:2]
    e = bfs_partitioned(emu, root, LocalExchange()).layers[:2]
    s = bfs(g, root).layers[:2]
    print(root, "deg", rp[root + 1] - rp[root], "reused", a, "fresh", f, "emu", e, "single", s, flush=True)
