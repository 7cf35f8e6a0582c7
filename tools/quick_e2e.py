"""Dev probe: public-API bfs(g, root) wall time vs device BFS and D2H times (S24)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1604_02844_b200 import RmatParams, bfs, build_rmat_graph, pick_roots
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = build_rmat_graph(RmatParams(scale=scale, seed=1))
roots = pick_roots(g, 64, 1, filter_unconnected=True).tolist()
for i, r in enumerate(roots[:10]):
    t = time.perf_counter()
    res = bfs(g, r)
    w = time.perf_counter() - t
    tm = res.timing
    print(f"call {i}: wall {w*1e3:.2f} ms bfs {tm['bfs_ms']:.2f} d2h {tm['d2h_ms']:.2f} -> e2e GTEPS {res.traversed_edge_count/w/1e9:.1f}", flush=True)
