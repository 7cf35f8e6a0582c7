"""Dev probe: many BFS on one S24 graph (all 64 roots, repeated), stop at the
first failure and print which root/iteration failed."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1604_02844_b200 import RmatParams, bfs_device, build_rmat_graph, pick_roots
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = build_rmat_graph(RmatParams(scale=scale, seed=1))
roots = pick_roots(g, 64, 1, filter_unconnected=True).tolist()
n = g.num_vertices
pred = torch.empty((n + 31) // 32 * 32, dtype=torch.int32, device="cuda")
lvl = torch.empty(n, dtype=torch.int32, device="cuda")
t = time.time()
k = 0
for it in range(reps):
    for r in roots:
        try:
            bfs_device(g, r, pred, lvl)
        except Exception as e:
            print(f"FAIL it={it} root={r} after {k} BFS: {e}", flush=True)
            sys.exit(1)
        k += 1
print(f"ok {k} BFS in {time.time()-t:.1f}s", flush=True)
