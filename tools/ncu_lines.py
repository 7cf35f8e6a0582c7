"""Per-source-line instruction / stall table of one kernel in an ncu report.
usage: ncu_lines.py REPORT KERNEL_REGEX LAUNCH_SKIP [N]"""
import csv, io, subprocess, sys
rep, kre, skip = sys.argv[1], sys.argv[2], sys.argv[3]
N = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kre}",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]; idx = {h: i for i, h in enumerate(hdr)}
print(rows[1][1] if len(rows) > 1 else "")
src = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0] not in ("", "Line No")]
f = lambda r, k: float(r[idx[k]]) if r[idx[k]] not in ("", "-") else 0.0
ti = sum(f(r, "Instructions Executed") for r in src); tt = sum(f(r, "Thread Instructions Executed") for r in src)
ts = sum(f(r, "Warp Stall Sampling (All Samples)") for r in src)
print(f"warp instr {ti:.3g}  thread eff {100*tt/ti/32:.1f}%  stall samples {ts:.0f}")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = {}
for r in src:
    for i in cols:
        try: tot[hdr[i]] = tot.get(hdr[i], 0) + float(r[i])
        except ValueError: pass
s = sum(tot.values()) or 1
print("stalls: " + ", ".join(f"{k[6:]} {100*v/s:.0f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:7]))
src.sort(key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))
print(f"{'line':>5} {'instr%':>7} {'eff':>5} {'stall%':>6}  source")
for r in src[:N]:
    print(f"{r[0]:>5} {100*f(r,'Instructions Executed')/ti:6.2f}% {f(r,'Thread Instructions Executed')/max(f(r,'Instructions Executed'),1):5.1f} "
          f"{100*f(r,'Warp Stall Sampling (All Samples)')/ts:5.1f}%  {r[1].strip()[:100]}")
