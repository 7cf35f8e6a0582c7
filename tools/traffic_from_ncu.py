"""DRAM traffic of the level expansion of one BFS from an ncu --set full capture
(every kernel of that BFS), against the algorithmic bytes 8E + 40V of SURVEY
§8(d). Writes profiles/roofline_traffic.json (read by bench.py).
Usage: python tools/traffic_from_ncu.py REP.ncu-rep E V ROOT COMMIT"""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_summary import rows

EXPAND = ("k_sweep", "k_sweep_plan", "k_sweep_plan_small", "k_expand", "k_merge_hot", "k_levels")
rep, E, V, root, commit = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
rs = rows(rep)
exp = [d for d in rs if d["kernel"].split("<")[0].replace("void ", "").replace("lbfs::", "").strip() in EXPAND]
dram = sum(d["dram_rd"] + d["dram_wr"] for d in exp)
ms = sum(d["ms"] for d in exp)
out = {"dram_bytes_per_bfs_expansion": dram, "alg_bytes_per_bfs_expansion": 8 * E + 40 * V,
       "expansion_kernel_ms_serialised": ms, "launches": len(exp), "root": root, "E": E, "V": V,
       "kernels": sorted({d["kernel"] for d in exp}), "scale": 24,
       "source": f"{rep} (ncu --set full --clock-control none, one S24 BFS; dram__bytes_read.sum + "
                 "dram__bytes_write.sum summed over the expansion launches)", "commit": commit}
Path("profiles/roofline_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1))
