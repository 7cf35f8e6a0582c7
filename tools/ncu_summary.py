"""Summarise an .ncu-rep: per-launch time, DRAM bytes, hit rates, warp efficiency."""
import csv, io, subprocess, sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
           "smsp__thread_inst_executed_per_inst_executed.ratio",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sectors.sum",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.max.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
SHORT = ["ms", "dram_rd", "dram_wr", "L2hit%", "L1hit%", "thr/inst", "warps%", "L2sect", "L2thr%", "L2max%",
         "dram%", "grid", "lsb"]


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    idx = {h: i for i, h in enumerate(hdr)}
    res = []
    for row in r[2:]:
        d = {"kernel": row[idx["Kernel Name"]].split("(")[0]}
        for m, s in zip(METRICS, SHORT):
            v = row[idx[m]].replace(",", "")
            u = units[idx[m]]
            try:
                x = float(v)
            except ValueError:
                x = float("nan")
            scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1, "us": 1e-3, "ns": 1e-6,
                     "msecond": 1, "usecond": 1e-3, "nsecond": 1e-6}.get(u, 1)
            d[s] = x * scale
        res.append(d)
    return res


if __name__ == "__main__":
    res = rows(sys.argv[1])
    # dramGB/s = (dram_rd + dram_wr) / ms: achieved DRAM bandwidth of the launch
    # (cold caches, --clock-control none); thr/inst = warp execution efficiency
    print("%-22s " % "kernel" + " ".join("%9s" % s for s in SHORT) + " %9s" % "dramGB/s")
    for d in res:
        gbs = (d["dram_rd"] + d["dram_wr"]) / (d["ms"] * 1e-3) / 1e9 if d["ms"] > 0 else float("nan")
        print("%-22s " % d["kernel"][:22] + " ".join(
            ("%9.3f" % d[s]) if s == "ms" else ("%9.3g" % d[s]) for s in SHORT) + " %9.0f" % gbs)
