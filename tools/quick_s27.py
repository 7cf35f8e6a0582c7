"""Dev probe: the S27 config (134M vertices, ~4.3B CSR entries) on ONE B200:
device construction, BFS from a few of the 64 seeded roots, device validation."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1604_02844_b200 import RmatParams, bfs_device, build_rmat_graph, pick_roots
from paper_1604_02844_b200.validate import validate_tree_device

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
nroots = int(sys.argv[2]) if len(sys.argv) > 2 else 4
t = time.time()
g = build_rmat_graph(RmatParams(scale=scale, seed=1))
torch.cuda.synchronize()
free, tot = torch.cuda.mem_get_info()
print(f"S{scale} build {time.time()-t:.1f}s n={g.num_vertices} nnz={g.num_edges} "
      f"device free {free/1e9:.1f}/{tot/1e9:.1f} GB", flush=True)
t = time.time()
roots = pick_roots(g, 64, 1, filter_unconnected=True).tolist()[:nroots]
print(f"roots {roots} ({time.time()-t:.1f}s)", flush=True)
n = g.num_vertices
pred = torch.empty((n + 31) // 32 * 32, dtype=torch.int32, device="cuda")
lvl = torch.empty(n, dtype=torch.int32, device="cuda")
t = time.time()
res = bfs_device(g, roots[0], pred, lvl)  # first call builds the layout
print(f"layout + first BFS {time.time()-t:.1f}s", flush=True)
free, tot = torch.cuda.mem_get_info()
print(f"device free after layout {free/1e9:.1f} GB", flush=True)
vals = []
for r in roots:
    res = bfs_device(g, r, pred, lvl)
    tm = res.timing
    vals.append(res.traversed_edge_count / tm["bfs_ms"] / 1e6)
    print(f"root {r}: bfs {tm['bfs_ms']:.2f} ms levels {tm['levels']} E={res.traversed_edge_count} "
          f"reached={tm['reached']} GTEPS {vals[-1]:.1f}", flush=True)
    rep = validate_tree_device(g, r, pred[:n])
    print(f"  validate_tree_device: {'PASS' if rep.passed else rep}", flush=True)
print(f"harmonic mean GTEPS {len(vals)/sum(1/v for v in vals):.1f}")
