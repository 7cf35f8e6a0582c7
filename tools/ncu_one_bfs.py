"""Profiling target: one BFS (after warm-up) bracketed by cudaProfilerStart /
Stop, for `ncu --profile-from-start off` (set LBFS_* env as needed).
    python tools/ncu_one_bfs.py [scale|lattice] [root_index]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1604_02844_b200 import RmatParams, bfs_device, build_lattice_graph, build_rmat_graph, pick_roots
what = sys.argv[1] if len(sys.argv) > 1 else "24"
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
g = build_lattice_graph(4096, 4096) if what == "lattice" else build_rmat_graph(RmatParams(scale=int(what), seed=1))
roots = pick_roots(g, 64, 1, filter_unconnected=True).tolist()
n = g.num_vertices
pred = torch.empty((n + 31) // 32 * 32, dtype=torch.int32, device="cuda")
for r in roots[:4]:
    bfs_device(g, r, pred)
torch.cuda.synchronize()
torch.cuda.profiler.start()
res = bfs_device(g, roots[idx], pred)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("root", roots[idx], "layers", [(l.input, l.edges, l.discovered) for l in res.layers], "ms", res.timing["bfs_ms"])
