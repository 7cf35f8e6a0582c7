"""Dev probe: per-root device BFS times on R-MAT SCALE S (not the bench).
Warms the GPU up (sustained BFS for ~1.5 s) so clocks are at full speed."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_1604_02844_b200 import RmatParams, bfs, build_rmat_graph, pick_roots, bfs_device

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nroots = int(sys.argv[2]) if len(sys.argv) > 2 else 8
t = time.time()
g = build_rmat_graph(RmatParams(scale=scale, seed=1))
print(f"S{scale} build {time.time()-t:.2f}s nnz={g.num_edges}", flush=True)
roots = pick_roots(g, 64, 1, filter_unconnected=True).tolist()[:nroots]
import torch
n = g.num_vertices
pred = torch.empty((n + 31) // 32 * 32, dtype=torch.int32, device="cuda")
lvl = torch.empty(n, dtype=torch.int32, device="cuda")
t = time.time()
k = 0
while time.time() - t < float(os.environ.get("WARM_S", "1.5")):
    bfs_device(g, roots[k % len(roots)], pred, lvl)
    k += 1
print(f"warm-up: {k} BFS", flush=True)
times = []
for r in roots:
    res = bfs_device(g, r, pred, lvl)
    tm = res.timing
    times.append(res.traversed_edge_count / tm['bfs_ms'] / 1e6)
    print(f"root {r}: bfs {tm['bfs_ms']:.3f} ms init {tm['init_ms']:.3f} expand {tm['expand_ms']:.3f} "
          f"levels {tm['levels']} launches {tm['kernel_launches']} GTEPS {times[-1]:.1f} "
          f"layers {[(l.input, l.edges, l.discovered) for l in res.layers]}", flush=True)
print(f"harmonic mean GTEPS {len(times)/sum(1/x for x in times):.1f}")
