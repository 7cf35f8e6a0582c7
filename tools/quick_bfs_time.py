"""Dev probe: per-root device BFS times on R-MAT SCALE S (not the bench)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_1604_02844_b200 import RmatParams, bfs, build_rmat_graph, pick_roots

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nroots = int(sys.argv[2]) if len(sys.argv) > 2 else 8
t = time.time()
g = build_rmat_graph(RmatParams(scale=scale, seed=1))
print(f"S{scale} build {time.time()-t:.2f}s nnz={g.num_edges}", flush=True)
roots = pick_roots(g, nroots, 1, filter_unconnected=True).tolist()
bfs(g, roots[0])
for r in roots:
    res = bfs(g, r)
    tm = res.timing
    print(f"root {r}: bfs {tm['bfs_ms']:.3f} ms init {tm['init_ms']:.3f} expand {tm['expand_ms']:.3f} "
          f"levels {tm['levels']} launches {tm['kernel_launches']} GTEPS {res.traversed_edge_count/tm['bfs_ms']/1e6:.1f} "
          f"d2h {tm['d2h_ms']:.2f} layers {[(l.input, l.edges, l.discovered) for l in res.layers]}", flush=True)
