"""Dev probe: partitioned BFS steps on one GPU, buffer popcounts per step."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_1604_02844_b200 import RmatParams, build_rmat_graph, pick_roots
from paper_1604_02844_b200.distributed import PartitionedGraph, LocalExchange
from oracle.part_emu import EmuPart

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g = build_rmat_graph(RmatParams(scale=14, edgefactor=16, seed=2))
rp, ci, n = g.colstarts, g.rows, g.num_vertices
root = int(pick_roots(g, 4, 5)[0])
ex = LocalExchange()


def pc(t):
    a = t.cpu().numpy().view(np.uint32) if t.dtype == torch.int32 else t.cpu().numpy()
    return int(np.unpackbits(a.view(np.uint8)).sum())


for kind in ("dev", "emu"):
    parts = [PartitionedGraph(g, r, P) if kind == "dev" else EmuPart(n, rp, ci, r, P) for r in range(P)]
    bufs = [p.new_buffers() for p in parts]
    for p, b in zip(parts, bufs):
        p.start(root, b["red"])
    ex.all_reduce_sum([b["red"] for b in bufs])
    for p, b in zip(parts, bufs):
        p.level_done(b["red"])
    for L in range(3):
        for p in parts:
            p.expand()
        for p, b in zip(parts, bufs):
            p.pack(b["send"])
        print(kind, L, "send", [pc(b["send"]) for b in bufs])
        ex.all_to_all([b["send"] for b in bufs], [b["recv"] for b in bufs])
        print(kind, L, "recv", [pc(b["recv"]) for b in bufs])
        for p, b in zip(parts, bufs):
            p.merge(b["recv"], b["fsend"], b["red"])
        print(kind, L, "fsend", [pc(b["fsend"]) for b in bufs], "red", [b["red"].tolist() for b in bufs])
        ex.all_gather([b["fsend"] for b in bufs], [b["fgath"] for b in bufs])
        ex.all_reduce_sum([b["red"] for b in bufs])
        for p, b in zip(parts, bufs):
            p.sync(b["fgath"])
        outs = [p.level_done(b["red"]) for p, b in zip(parts, bufs)]
        print(kind, L, outs[0])
        if outs[0][1]:
            break
