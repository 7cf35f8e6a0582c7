"""DRAM traffic of one whole BFS from an ncu --set full capture of every kernel
of that BFS (tools/ncu_one_bfs.py under --profile-from-start off), against the
algorithmic bytes B_alg = 8E + 40V + 8n + n/8 of SURVEY §8(d).
Writes profiles/roofline_traffic.json (read by bench.py: roofline.traffic and
roofline.dram).
Usage: python tools/traffic_from_ncu.py REP.ncu-rep E V N ROOT COMMIT"""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_summary import rows

rep, E, V, n, root, commit = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5], sys.argv[6]
rs = rows(rep)
short = lambda k: k.replace("void ", "").replace("lbfs::", "").strip()
per = {}
for d in rs:
    k = short(d["kernel"])
    e = per.setdefault(k, {"launches": 0, "ms": 0.0, "dram_bytes": 0.0})
    e["launches"] += 1
    e["ms"] += d["ms"]
    e["dram_bytes"] += d["dram_rd"] + d["dram_wr"]
dram = sum(e["dram_bytes"] for e in per.values())
ms = sum(e["ms"] for e in per.values())
out = {"dram_bytes_per_bfs": dram, "alg_bytes_per_bfs": 8 * E + 40 * V + 8 * n + n // 8,
       "kernel_ms_serialised": ms, "launches": len(rs), "root": root, "E": E, "V": V, "n": n, "scale": 24,
       "per_kernel": {k: {"launches": e["launches"], "ms": round(e["ms"], 4), "dram_bytes": e["dram_bytes"],
                          "dram_gbs": round(e["dram_bytes"] / (e["ms"] * 1e-3) / 1e9, 1) if e["ms"] > 0 else None}
                      for k, e in sorted(per.items(), key=lambda x: -x[1]["ms"])},
       "source": f"{rep} (ncu --set full --clock-control none, every kernel of one S24 BFS; dram__bytes_read.sum + "
                 "dram__bytes_write.sum per launch, summed)", "commit": commit}
Path("profiles/roofline_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps({k: v for k, v in out.items() if k != "per_kernel"}, indent=1))
