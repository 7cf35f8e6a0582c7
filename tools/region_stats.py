"""Dev probe (host numpy, not the bench): per-level frontier coverage of the
degree regions of the internal (degree-ordered) layout, and where the first
frontier neighbour sits in the sorted adjacency of newly discovered hot
vertices. Usage: python tools/region_stats.py SCALE NROOTS [HOT_VERTS]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_1604_02844_b200 import RmatParams, bfs, build_rmat_graph, pick_roots

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nroots = int(sys.argv[2]) if len(sys.argv) > 2 else 2
hot = int(sys.argv[3]) if len(sys.argv) > 3 else 1_170_000
g = build_rmat_graph(RmatParams(scale=scale, seed=1))
rp = np.asarray(g.colstarts, dtype=np.int64)
ci = np.asarray(g.rows, dtype=np.int32)
n = g.num_vertices
deg = np.diff(rp)
order = np.lexsort((np.arange(n), -deg))      # internal id -> original id
rank = np.empty(n, np.int64)
rank[order] = np.arange(n)                     # original -> internal
dsorted = deg[order]
t_cta = int((dsorted >= 1024).sum()); t_warp = int((dsorted >= 32).sum()); t_nz = int((dsorted > 0).sum())
e_reg = [int(dsorted[:t_cta].sum()), int(dsorted[t_cta:t_warp].sum()), int(dsorted[t_warp:t_nz].sum())]
print(f"n={n} nnz={ci.size} t_cta={t_cta} t_warp={t_warp} t_nz={t_nz} region edges hub/warp/small={e_reg}")
print(f"hot prefix {hot} verts: edges into hot = {(rank[ci] < hot).mean():.3f} of all entries")
for r in pick_roots(g, 64, 1, filter_unconnected=True)[:nroots]:
    res = bfs(g, int(r))
    lv = res.levels
    lvi = lv[order]                            # internal order
    print(f"root {r}: layers {[(l.input, l.edges, l.discovered) for l in res.layers]}")
    for L in range(len(res.layers)):
        f = lvi == L
        cov = [float(dsorted[a:b][f[a:b]].sum()) / max(e_reg[i], 1)
               for i, (a, b) in enumerate([(0, t_cta), (t_cta, t_warp), (t_warp, t_nz)])]
        fe = dsorted[f]
        if fe.sum() < 1000:
            continue
        # edges of the frontier whose target is hot
        fr = order[f]
        idx = np.concatenate([np.arange(rp[u], rp[u + 1]) for u in fr[:20000]]) if len(fr) else np.zeros(0, np.int64)
        hot_frac = float((rank[ci[idx]] < hot).mean()) if idx.size else 0.0
        # new hot vertices at L+1: position of the first neighbour at level L in internal-sorted adjacency
        newhot = order[lvi == L + 1]  # all new vertices (sampled below)
        pos = []
        for v in newhot[:: max(1, len(newhot) // 3000)]:
            nb = ci[rp[v]:rp[v + 1]]
            nbs = nb[np.argsort(rank[nb])]
            k = np.nonzero(lv[nbs] == L)[0]
            pos.append(int(k[0]) if k.size else -1)
        pos = np.array(pos) if pos else np.zeros(0, int)
        q = np.percentile(pos, [50, 90, 99, 100]) if pos.size else []
        print(f"  L{L}: coverage hub/warp/small = {cov[0]:.2f}/{cov[1]:.2f}/{cov[2]:.2f}  "
              f"hot-target frac {hot_frac:.2f}  new-hot {len(newhot)} first-parent pos p50/90/99/max {q}")
