"""bench.py — GTEPS of the device top-down BFS on R-MAT SCALE 24 (BASELINE.json
configs[2]: the single-GPU target config and the one sharded at 2/4/8 GPUs).

One step = one BFS from each of the 64 seeded roots (pick_roots(g, 64, seed=1,
filter_unconnected=True), harness.py:237-246) over the device-resident graph.
value = harmonic mean over all timed BFS runs of traversed_edge_count / t_bfs
(harness.py:218-234, 269); t_bfs from CUDA events on the BFS stream (init
kernel start -> parents written in original ids). Every timed tree is
validated afterwards on the device (the reference harness's validate_tree
after each root, harness.py:266-268); a failure aborts the run.

roofline.frac is the whole BFS against SURVEY §8(d)'s algorithmic bytes
B_alg = 8E + 40V + 8n + n/8 over the measured HBM peak. Extra keys: S20 and
the 4096^2 lattice (configs[1], configs[3]) measured the same way after the
headline, e2e through the public bfs(g, root) with host outputs, the opt-in
direction-optimising variant.

--impl reference: rank 0 times the reference's CPU path on the box's host
cores: the oracle port of bfs_parallel_naive (traversal.py:128-165, OpenMP)
on the same graph, 8 roots per step cycling through all 64; plus, when the
reference package is installed in baseline/_ref, the reference's own
bfs_parallel_naive on one root in a subprocess.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GTEPS (harmonic mean over 64 roots) and % of HBM roofline at 1/2/4/8 B200"
FALLBACK_HBM_GBS = 6650.0
REF_PKG = ROOT / "baseline" / "_ref"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--roots", type=int, default=64)
    ap.add_argument("--cpu-roots", type=int, default=0,
                    help="roots per step of the --impl reference arm (0: enough for the timed steps to cover "
                         "every root of the set once, at most 16)")
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of CPU-baseline sampling")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra-configs", action="store_true", help="skip the S20 / lattice / S27 keys")
    ap.add_argument("--no-s27", action="store_true", help="skip the SCALE-27 key of the extra configs")
    ap.add_argument("--part-driver", choices=("native", "python"), default="native",
                    help="partitioned level loop: the library's (one call per BFS, library-owned NCCL "
                         "communicator) or distributed.bfs_partitioned (per-step calls, torch.distributed)")
    ap.add_argument("--partitioned", action="store_true",
                    help="use the partitioned (multi-GPU) driver even at N=1 (one NCCL rank)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return FALLBACK_HBM_GBS, "fallback"


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def hm(values):
    from paper_1604_02844_b200 import harmonic_mean_teps

    return harmonic_mean_teps(values)[0]


def b_alg(E: float, V: float, n: int) -> float:
    """4E col_idx + 4E bitmap probe + 16V row_ptr + 8V atomic
    RMW + 8V level/pred + 8V queue + 8n init + n/8 bitmap clear."""
    return 8 * E + 40 * V + 8 * n + n // 8


def traffic_from_profiles(scale: int):
    """ncu DRAM bytes of one BFS (profiles/roofline_traffic.json), only for the
    workload it was captured on."""
    p = ROOT / "profiles" / "roofline_traffic.json"
    if p.exists():
        try:
            t = json.loads(p.read_text())
        except Exception:
            return None
        return t if int(t.get("scale", 24)) == scale else None
    return None


def reference_python_sample(rp, ci, n, roots, timeout_s=240):
    """The reference itself (lanebfs bfs_parallel_naive, traversal.py:128-165,
    timed around the call only like harness.py:263-265) on the same CSR, in a
    subprocess (G8), when baseline/_ref holds the package."""
    if not (REF_PKG / "lanebfs").exists():
        return None
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        np.save(f"{td}/rp.npy", rp)
        np.save(f"{td}/ci.npy", ci)
        code = (
            "import sys,time,json,os,numpy as np\n"
            f"sys.path.insert(0,{str(REF_PKG)!r})\n"
            "from lanebfs.graph import CsrGraph\n"
            "from lanebfs.traversal import bfs_parallel_naive\n"
            f"rp=np.load('{td}/rp.npy'); ci=np.load('{td}/ci.npy')\n"
            f"g=CsrGraph({n}, ci, rp)\n"
            "th=os.cpu_count(); out=[]\n"
            f"for s in {list(map(int, roots))}:\n"
            "    t=time.perf_counter(); r=bfs_parallel_naive(g,s,th); dt=time.perf_counter()-t\n"
            "    out.append([s, r.traversed_edge_count, dt])\n"
            "print(json.dumps({'threads': th, 'runs': out}))\n")
        try:
            res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=timeout_s)
            d = json.loads(res.stdout.strip().splitlines()[-1])
        except Exception as e:  # noqa: BLE001
            return {"error": str(e)[:200]}
    vals = [e / dt / 1e9 for _, e, dt in d["runs"]]
    return {"value": hm(vals), "unit": "GTEPS", "cores": d["threads"], "kind": "reference",
            "sample": f"{len(vals)} root(s), lanebfs 0.1.0 bfs_parallel_naive (the reference's fastest path) "
                      f"on the same CSR, in a subprocess; {sum(x[2] for x in d['runs']):.1f}s",
            "runs": d["runs"]}


def cpu_baseline_sample(rp, ci, roots, budget_s):
    """Oracle port of bfs_parallel_naive on all host cores (rank 0, N=1):
    roots in order until ~budget_s seconds of CPU work (at least 2)."""
    import oracle

    vals = []
    threads = oracle.max_threads()
    t_all = time.perf_counter()
    for i, r in enumerate(roots):
        if i >= 2 and time.perf_counter() - t_all > budget_s:
            break
        t0 = time.perf_counter()
        _, _, layers = oracle.bfs_parallel(rp, ci, int(r), 0)
        dt = time.perf_counter() - t0
        e = sum(l[1] for l in layers)
        vals.append(e / dt / 1e9 if e else 0.0)
    return vals, threads, time.perf_counter() - t_all


def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle

    t0 = time.perf_counter()
    s, d = oracle.rmat_edges(args.scale, 16, seed=1)
    s, d = oracle.permute_edges(1 << args.scale, 1, s, d)
    rp, ci = oracle.build_csr(1 << args.scale, s, d)
    del s, d
    build_s = time.perf_counter() - t0
    roots = oracle.pick_roots(np.diff(rp), args.roots, 1, True).tolist()
    threads = oracle.max_threads()
    # (default: the timed steps together cover the whole root set — the same
    # roots the device arm times — in at most 16 BFS of ~0.2 s per step)
    per_step = args.cpu_roots if args.cpu_roots > 0 else min(16, -(-args.roots // max(1, args.steps)))
    vals, step_times = [], []
    cursor = 0
    for step in range(args.warmup + args.steps):
        t = time.perf_counter()
        step_vals = []
        for _ in range(per_step):
            r = roots[cursor % len(roots)]
            cursor += 1
            a = time.perf_counter()
            _, _, layers = oracle.bfs_parallel(rp, ci, int(r), 0)
            dt = time.perf_counter() - a
            e = sum(l[1] for l in layers)
            step_vals.append(e / dt / 1e9 if e else 0.0)
        if step >= args.warmup:
            vals += step_vals
            step_times.append(time.perf_counter() - t)
    value = hm(vals)
    covered = len({roots[i % len(roots)] for i in range(args.warmup * per_step, cursor)})
    refpy = reference_python_sample(rp, ci, 1 << args.scale, roots[:1])
    cpu = {"value": value, "unit": "GTEPS", "cores": threads, "kind": "port", "cpu_model": cpu_model(),
           "sample": f"{per_step} roots per step cycling through the {args.roots}-root set ({covered} distinct "
                     f"roots timed), oracle bfs_parallel (restated bfs_parallel_naive, traversal.py:128-165)"}
    if refpy:
        cpu["reference_python"] = refpy
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(step_times) / len(step_times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": f"rmat-s{args.scale}-ef16-{args.roots}roots", "scale": args.scale,
                   "edgefactor": 16, "roots": args.roots, "n": len(rp) - 1, "nnz": int(rp[-1]),
                   "parallelism": f"cpu-openmp-{threads}t", "graph_build_s": round(build_s, 1)},
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_partitioned(args, rank, world, local):
    """N > 1: the graph 1D-partitioned over the N GPUs (one rank each), one
    BFS = the level loop of distributed.bfs_partitioned with its per-level
    NCCL collectives. Every rank builds the same graph on its GPU
    (deterministic device generator) and keeps only its partition's rows.
    Per-BFS time = max over ranks of the CUDA-event time on each rank's
    stream; value = harmonic mean over roots of E / t (whole job)."""
    import torch
    import torch.distributed as dist

    from paper_1604_02844_b200 import RmatParams, _lib, build_rmat_graph, pick_roots
    from paper_1604_02844_b200.distributed import PartitionedGraph, TorchExchange, bfs_partitioned

    torch.cuda.set_device(local)
    if "RANK" not in os.environ:  # --partitioned without torchrun: a world of one
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if os.environ.get("NCCL_DEBUG", "").upper() == "VERSION":
        os.environ.pop("NCCL_DEBUG")
        print(f"[bench] NCCL version {'.'.join(map(str, torch.cuda.nccl.version()))}", file=sys.stderr)
    if os.environ.get("NCCL_DEBUG"):
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    t0 = time.perf_counter()
    g = build_rmat_graph(RmatParams(scale=args.scale, seed=1))
    n, nnz = g.num_vertices, g.num_edges
    roots = pick_roots(g, args.roots, 1, filter_unconnected=True).tolist()
    part = PartitionedGraph(g, rank, world, device=local)
    if rank != 0:
        del g  # only this rank's rows stay on its GPU (rank 0 keeps the graph for the tree checks)
    build_s = time.perf_counter() - t0
    ex = TorchExchange()
    bufs = [part.new_buffers()]
    outs = [part.new_outputs()]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    native = args.part_driver == "native"
    if native:
        part.attach_nccl()

    def one(r, gather=False):
        if native:  # the library's level loop; its own CUDA-event time on its stream
            res = part.bfs_native(r, outs[0][0], outs[0][1], gather=gather)
            return res, res.timing["bfs_ms"]
        ev0.record()
        res = bfs_partitioned([part], r, ex, bufs=bufs, outputs=outs, gather=gather)
        ev1.record()
        ev1.synchronize()
        return res, ev0.elapsed_time(ev1)

    for _ in range(args.warmup):
        for r in roots:
            one(r)
    launches0 = _lib.kernel_launch_count()
    dist.barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    times, edges, nlevels, reached = [], [], [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            for r in roots:
                res, ms = one(r)
                times.append(ms)
                edges.append(res.traversed_edge_count)
                nlevels.append(len(res.layers))
                reached.append(sum(l.input for l in res.layers))
        dist.barrier()
        torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    launches = _lib.kernel_launch_count() - launches0
    t = torch.tensor(times, dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tmax = t.cpu().numpy()
    teps = [e / (ms * 1e-3) / 1e9 if e else 0.0 for e, ms in zip(edges, tmax)]
    value = hm(teps)
    ms_step = float(tmax.sum()) / args.steps
    # e2e: public driver with the gathered outputs, rank 0 reads pred+level to host
    pred_h = torch.empty(outs[0][0].numel(), dtype=torch.int32, pin_memory=True)
    lvl_h = torch.empty(outs[0][1].numel(), dtype=torch.int32, pin_memory=True)
    for r in roots[:2]:  # untimed warm-up
        one(r, gather=True)
    from paper_1604_02844_b200.validate import validate_tree_device
    e2e_vals, checked = [], 0
    for r in roots[:16]:
        dist.barrier()
        a = time.perf_counter()
        res, _ = one(r, gather=True)
        if rank == 0:
            pred_h.copy_(outs[0][0])
            lvl_h.copy_(outs[0][1])
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - a], dtype=torch.float64, device="cuda")
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e_vals.append(res.traversed_edge_count / float(dt.item()) / 1e9)
        if rank == 0:  # every gathered tree, on the unpartitioned graph (outside the timed interval)
            rep = validate_tree_device(g, r, outs[0][0])
            checked += 1
            if not rep.passed:
                raise SystemExit(f"[bench] partitioned tree failed validation for root {r}: {rep.details}")
    e2e = hm(e2e_vals)
    ok = checked if rank == 0 else None
    hbm_gbs, peak_kind = peaks()
    E = float(np.mean(edges))
    alg = b_alg(E, float(np.mean(reached)), n)
    X = float(np.mean(nlevels))
    words = (n + 31) // 32
    nvl_bytes = X * 2 * (world - 1) * ((words + world - 1) // world) * 4
    t_meas = float(np.mean(tmax)) * 1e-3
    t_roof = max(alg / (world * hbm_gbs * 1e9), nvl_bytes / 9e11)
    line = {
        "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic: R-MAT (reference generator, bit-exact) + seeded permutation",
        "config": {"workload": f"rmat-s{args.scale}-ef16-{args.roots}roots", "scale": args.scale,
                   "edgefactor": 16, "roots": args.roots, "n": n, "nnz": nnz,
                   "parallelism": f"1d-partition-{world}gpu-nccl",
                   "l2": "inputs larger than L2; no flush", "graph_build_s": round(build_s, 2),
                   "validated_trees": ok, "driver": args.part_driver},
        "roofline": {"bound": "hbm", "achieved": alg / world / t_meas / 1e9, "peak": hbm_gbs, "unit": "GB/s",
                     "frac": t_roof / t_meas, "peak_kind": peak_kind, "traffic": None,
                     "kernel": "whole BFS per GPU (SURVEY §8e t_roof(P) formula)",
                     "t_roof_ms": t_roof * 1e3, "t_measured_ms": t_meas * 1e3,
                     "nvlink_bytes_per_gpu": nvl_bytes, "levels": X},
        "e2e": {"value": e2e, "unit": "GTEPS", "h2d_bytes_per_step": 8,
                "d2h_bytes_per_step": (outs[0][0].numel() + n) * 4, "step": "one BFS (harmonic mean over roots)",
                "api": ("PartitionedGraph.bfs_native" if native else "distributed.bfs_partitioned")
                       + "(gather=True) + rank-0 D2H", "roots_timed": len(e2e_vals)},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "wall_s_timed": wall,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    part.close()
    dist.barrier()
    dist.destroy_process_group()


def device_runs(g, roots, passes, pred, validate=True):
    """`passes` passes over the roots through bfs_device; each tree validated
    on the device right after its BFS (outside the BFS's own CUDA-event
    interval). Returns the results and the number of validated trees."""
    from paper_1604_02844_b200 import bfs_device
    from paper_1604_02844_b200.validate import validate_tree_device

    runs, checked = [], 0
    for _ in range(passes):
        for r in roots:
            res = bfs_device(g, r, pred)
            if validate:
                rep = validate_tree_device(g, r, pred)
                checked += 1
                if not rep.passed:
                    raise SystemExit(f"[bench] validate_tree failed for root {r}: {rep.details}")
            runs.append(res)
    return runs, checked


def teps_of(runs):
    return [r.traversed_edge_count / (r.timing["bfs_ms"] * 1e-3) / 1e9 if r.traversed_edge_count else 0.0
            for r in runs]


def extra_config(build, nroots, warm_passes=1, passes=1):
    """GTEPS of another BASELINE config, measured like the headline (device
    outputs, CUDA-event time per BFS, every tree validated)."""
    import torch

    from paper_1604_02844_b200 import pick_roots

    t0 = time.perf_counter()
    g = build()
    roots = pick_roots(g, nroots, 1, filter_unconnected=True).tolist()
    n = g.num_vertices
    pred = torch.empty((n + 31) // 32 * 32, dtype=torch.int32, device="cuda")
    device_runs(g, roots, warm_passes, pred, validate=False)
    runs, checked = device_runs(g, roots, passes, pred)
    E = float(np.mean([r.traversed_edge_count for r in runs]))
    ms = float(np.mean([r.timing["bfs_ms"] for r in runs]))
    lv = float(np.mean([r.timing["levels"] for r in runs]))
    V = float(np.mean([r.timing["reached"] for r in runs]))
    hbm_gbs, _ = peaks()
    out = {"value": hm(teps_of(runs)), "unit": "GTEPS", "roots": len(roots), "bfs_timed": len(runs),
           "validated_trees": checked, "n": n, "nnz": g.num_edges, "ms_per_bfs": ms, "levels": lv,
           "us_per_level": 1e3 * ms / lv,
           "whole_bfs_frac_of_peak": b_alg(E, V, n) / (ms * 1e-3) / 1e9 / hbm_gbs,
           "build_s": round(time.perf_counter() - t0, 2)}
    del g, pred
    torch.cuda.empty_cache()
    return out


def run_ours(args, rank, world, local):
    import torch

    from paper_1604_02844_b200 import RmatParams, _lib, bfs, bfs_device, build_rmat_graph, pick_roots

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    t0 = time.perf_counter()
    g = build_rmat_graph(RmatParams(scale=args.scale, seed=1))
    n, nnz = g.num_vertices, g.num_edges
    roots = pick_roots(g, args.roots, 1, filter_unconnected=True).tolist()
    g.device_handle()
    build_s = time.perf_counter() - t0
    npad = (n + 31) // 32 * 32
    pred = torch.empty(npad, dtype=torch.int32, device="cuda")

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    device_runs(g, roots, args.warmup, pred, validate=False)
    hbm_gbs, peak_kind = peaks()
    barrier()
    w0 = time.perf_counter()
    with ClockSampler(local) as clk:
        runs, checked = device_runs(g, roots, args.steps, pred)
        barrier()
    wall = time.perf_counter() - w0
    # kernels the timed BFS runs launched (each run counts its own; the
    # validator's launches between them are not BFS work)
    launches = sum(int(r.timing["kernel_launches"]) for r in runs)
    teps = teps_of(runs)
    value_local = hm(teps)
    ms_step_local = sum(r.timing["bfs_ms"] for r in runs) / args.steps
    # roofline: the whole BFS against B_alg; expansion = the
    # level loop (init, every level's kernels incl. compaction — the 40 B/vertex
    # term is written there —, launch latency and host round trips): the BFS
    # without its output pass
    alg = sum(b_alg(r.traversed_edge_count, r.timing["reached"], n) for r in runs)
    bfs_ms = sum(r.timing["bfs_ms"] for r in runs)
    exp_bytes = sum(8 * r.traversed_edge_count + 40 * r.timing["reached"] for r in runs)
    exp_ms = sum(r.timing["expand_ms"] + r.timing["cluster_ms"] for r in runs)
    achieved = alg / (bfs_ms * 1e-3) / 1e9
    traffic = traffic_from_profiles(args.scale)
    dram = None
    if traffic and traffic.get("dram_bytes_per_bfs"):
        per_bfs_ms = bfs_ms / len(runs)
        dram = {"bytes_per_bfs": traffic["dram_bytes_per_bfs"],
                "dram_gbs": traffic["dram_bytes_per_bfs"] / (per_bfs_ms * 1e-3) / 1e9,
                "source": traffic.get("source")}
        dram["dram_frac"] = dram["dram_gbs"] / hbm_gbs

    # direction-optimising BFS (opt-in; not the headline: the north star is
    # top-down): one untimed pass, then one pass over the same roots
    for r in roots[:3]:
        bfs_device(g, r, pred, direction="optimizing")
    do_runs = [bfs_device(g, r, pred, direction="optimizing") for r in roots]
    do_value = hm(teps_of(do_runs))
    do_ok = all(x.layers == y.layers for x, y in zip(do_runs, runs[:len(do_runs)]))

    # e2e through the public API with host outputs: one bfs(g, root) call per
    # step, parents copied to page-locked host memory inside the call (levels
    # stay on the device until read); untimed warm-up calls fill the pool
    res = None
    for r in roots[:3]:
        res = bfs(g, r)
    del res
    e2e_vals = []
    for r in roots:
        a = time.perf_counter()
        res = bfs(g, r)
        dt = time.perf_counter() - a
        e2e_vals.append(res.traversed_edge_count / dt / 1e9 if res.traversed_edge_count else 0.0)
        del res
    e2e = hm(e2e_vals)
    d2h_bytes = npad * 4  # one e2e step = one BFS: the pad32(n) parent array to host

    value, ms_step = value_local, ms_step_local
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms_step_local], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
        # replicas: every rank processes the full root set; aggregate throughput
        edges_total = sum(r.traversed_edge_count for r in runs) / args.steps
        value = world * edges_total / (ms_step * 1e-3) / 1e9
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rp, ci = g.colstarts, g.rows
        vals, thr, secs = cpu_baseline_sample(rp, ci, roots, args.cpu_budget)
        cpu = {"value": hm(vals), "unit": "GTEPS", "cores": thr, "kind": "port", "cpu_model": cpu_model(),
               "sample": f"{len(vals)} of the {args.roots} roots on the same graph, oracle bfs_parallel "
                         f"(OpenMP restatement of bfs_parallel_naive), {secs:.1f}s"}
    del g, pred
    torch.cuda.empty_cache()
    extra = {}
    if rank == 0 and not args.no_extra_configs:
        from paper_1604_02844_b200 import build_lattice_graph

        extra["rmat-s20-ef16-64roots"] = extra_config(lambda: build_rmat_graph(RmatParams(scale=20, seed=1)), 64,
                                                      warm_passes=2, passes=2)
        extra["lattice-4096x4096-16roots"] = extra_config(lambda: build_lattice_graph(4096, 4096), 16)
        # configs[4] (SCALE 27, 4.2e9 CSR entries, ~40 GB with the layout's
        # temporaries): on one GPU when the memory is there; a failure here is
        # reported in its key and does not touch the headline
        if not args.no_s27:
            free_b, _ = torch.cuda.mem_get_info()
            if free_b >= 100 * (1 << 30):
                try:
                    extra["rmat-s27-ef16-64roots"] = extra_config(
                        lambda: build_rmat_graph(RmatParams(scale=27, seed=1)), 64, warm_passes=1, passes=1)
                except Exception as e:  # noqa: BLE001
                    extra["rmat-s27-ef16-64roots"] = {"error": f"{type(e).__name__}: {e}"[:300]}
                    try:
                        torch.cuda.empty_cache()
                    except Exception:  # noqa: BLE001  (the headline line below is printed regardless)
                        pass
            else:
                extra["rmat-s27-ef16-64roots"] = {"skipped": f"{free_b >> 30} GiB free on the device"}
    line = {
        "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic: R-MAT (reference generator, bit-exact) + seeded permutation",
        "config": {"workload": f"rmat-s{args.scale}-ef16-{args.roots}roots", "scale": args.scale,
                   "edgefactor": 16, "roots": args.roots, "n": n, "nnz": nnz,
                   "parallelism": "1gpu" if world == 1 else f"replicas{world}",
                   "l2": "inputs larger than L2 (CSR %.2f GB vs 126 MB L2); no flush" % ((8 * n + 4 * nnz) / 1e9),
                   "graph_build_s": round(build_s, 2), "validated_trees": checked},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_gbs, "unit": "GB/s",
                     "frac": achieved / hbm_gbs, "peak_kind": peak_kind,
                     "traffic": traffic.get("dram_bytes_per_bfs") if traffic else None,
                     "kernel": "whole BFS (init, every level kernel, output pass), SURVEY §8(d) B_alg",
                     "alg_bytes_per_bfs": alg / len(runs), "ms_per_bfs": bfs_ms / len(runs),
                     "frac_of_8TBs": alg / (bfs_ms * 1e-3) / 8e12,
                     "dram": dram,
                     "expansion": {"alg_bytes_per_bfs": exp_bytes / len(runs), "ms_per_bfs": exp_ms / len(runs),
                                   "frac_of_peak": exp_bytes / (exp_ms * 1e-3) / 1e9 / hbm_gbs,
                                   "kernels": "the level loop: init, every level's kernels (expansion bins, merge, "
                                              "compaction, cluster segments), launch latency and host round trips; "
                                              "the output pass excluded"}},
        "e2e": {"value": e2e, "unit": "GTEPS", "h2d_bytes_per_step": 8,
                "d2h_bytes_per_step": d2h_bytes, "step": "one bfs(g, root) call (harmonic mean over roots)",
                "api": "paper_1604_02844_b200.bfs(g, root), parents to host (levels on first access)",
                "roots_timed": len(e2e_vals)},
        "configs": extra,
        "direction_optimizing": {"value": do_value, "unit": "GTEPS", "roots": len(do_runs),
                                 "layers_equal_top_down": do_ok,
                                 "note": "opt-in bottom-up levels (bfs(..., direction='optimizing')); same E, "
                                         "levels and layers as the top-down headline; not the north-star path"},
        "gpu_launches": launches,
        **({"retried_after": os.environ["LBFS_BENCH_RETRY"]} if os.environ.get("LBFS_BENCH_RETRY") else {}),
        "clocks": clk.summary(),
        "wall_s_timed": wall,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif world > 1 or args.partitioned:
        run_partitioned(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
