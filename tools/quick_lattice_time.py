"""Dev probe: device BFS on the 4096x4096 permuted lattice (config 4)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1604_02844_b200 import bfs_device, build_lattice_graph, pick_roots

side = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
nroots = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = build_lattice_graph(side, side)
n = g.num_vertices
pred = torch.empty((n + 31) // 32 * 32, dtype=torch.int32, device="cuda")
lvl = torch.empty(n, dtype=torch.int32, device="cuda")
roots = pick_roots(g, 16, 1, filter_unconnected=True).tolist()[:nroots]
bfs_device(g, roots[0], pred, lvl)
vals = []
for r in roots:
    t = time.perf_counter()
    res = bfs_device(g, r, pred, lvl)
    wall = time.perf_counter() - t
    tm = res.timing
    vals.append(res.traversed_edge_count / tm["bfs_ms"] / 1e6)
    print(f"root {r}: levels {tm['levels']} bfs {tm['bfs_ms']:.1f} ms ({tm['bfs_ms']*1e3/tm['levels']:.1f} us/level) "
          f"wall {wall*1e3:.1f} ms launches {tm['kernel_launches']} GTEPS {vals[-1]:.3f}", flush=True)
print(f"harmonic mean GTEPS {len(vals)/sum(1/v for v in vals):.3f}")
