"""Dev probe: per-level step times of the partitioned driver at P=1 (a world
of one over NCCL), synchronising after each step (so the host overhead of a
step is inside its time). Not the bench."""
import os
import socket
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import torch.distributed as dist

from paper_1604_02844_b200 import RmatParams, build_rmat_graph, pick_roots
from paper_1604_02844_b200.distributed import PartitionedGraph, TorchExchange, bfs_partitioned

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
with socket.socket() as sk:
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
g = build_rmat_graph(RmatParams(scale=scale, seed=1))
roots = pick_roots(g, 64, 1, filter_unconnected=True).tolist()[:8]
part = PartitionedGraph(g, 0, 1, device=0)
ex = TorchExchange()
bufs = [part.new_buffers()]
outs = [part.new_outputs()]
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(5):
    for r in roots:
        bfs_partitioned([part], r, ex, bufs=bufs, outputs=outs, gather=False)
torch.cuda.synchronize()
if os.environ.get("ONE"):  # one BFS of roots[0] between cudaProfilerStart / Stop (ncu --profile-from-start off)
    torch.cuda.profiler.start()
    bfs_partitioned([part], roots[0], ex, bufs=bufs, outputs=outs, gather=False)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    dist.destroy_process_group()
    sys.exit(0)
tot = []
for r in roots:
    ev0.record()
    res = bfs_partitioned([part], r, ex, bufs=bufs, outputs=outs, gather=False)
    ev1.record()
    ev1.synchronize()
    tot.append(ev0.elapsed_time(ev1))
    print(f"root {r}: {tot[-1]:.3f} ms levels {len(res.layers)} GTEPS {res.traversed_edge_count / tot[-1] / 1e6:.1f}")

# one BFS step by step
b = bufs[0]
r = roots[0]


def T(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3


for rep in range(2):
    rows = []
    t_start = T(lambda: part.start(r, b["red"]))
    t_ar = T(lambda: ex.all_reduce_sum([b["red"]]))
    t_d0 = T(lambda: part.level_done(b["red"]))
    L = 0
    while True:
        te = T(part.expand)
        tp = T(lambda: part.pack(b["send"]))
        ta = T(lambda: ex.all_to_all([b["send"]], [b["recv"]]))
        tm = T(lambda: part.merge(b["recv"], b["fsend"]))
        tg = T(lambda: ex.all_gather([b["fsend"]], [b["fgath"]]))
        ts = T(lambda: part.sync(b["fgath"]))
        out = {}
        td = T(lambda: out.setdefault("r", part.level_done()))
        ly, done = out["r"]
        rows.append((L, ly, te, tp, ta, tm, tg, ts, td))
        L += 1
        if done:
            break
    tf = T(lambda: part.finish(outs[0][0], outs[0][1]))
    if rep == 1:
        print(f"start {t_start:.3f} allreduce {t_ar:.3f} done0 {t_d0:.3f} finish {tf:.3f} (ms, synced)")
        for L, ly, *t in rows:
            print(f"L{L} in={ly.input} edges={ly.edges} disc={ly.discovered}: expand {t[0]:.3f} pack {t[1]:.3f} "
                  f"a2a {t[2]:.3f} merge {t[3]:.3f} gather {t[4]:.3f} sync {t[5]:.3f} done {t[6]:.3f}")
dist.destroy_process_group()
