"""Per-instruction shared-memory wavefronts (actual / ideal / excessive) of an ncu report, largest first.

usage: KERNEL=regex python tools/ncu_smem.py REPORT.ncu-rep [n]
"""
import csv, io, os, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
flt = ["-k", "regex:" + os.environ["KERNEL"]] if os.environ.get("KERNEL") else []
out = subprocess.run(["ncu", "-i", rep, *flt, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, isrc, iw, iid, iex = (h.index(k) for k in ("Address", "Source", "L1 Wavefronts Shared",
                                                  "L1 Wavefronts Shared Ideal", "Instructions Executed"))
recs = []
for r in rows[2:]:
    try:
        recs.append((int(r[iw] or 0), int(r[iid] or 0), int(r[iex] or 0), r[isrc].strip(), r[ia]))
    except (ValueError, IndexError):
        pass
base = int(recs[0][4], 16)
tw = sum(x[0] for x in recs)
ti = sum(x[1] for x in recs)
print(f"total wavefronts {tw:.4g} ideal {ti:.4g}")
for w, i, e, s, a in sorted(recs, reverse=True)[:n]:
    print(f"{int(a, 16) - base:6x} wf {w:11d} ({100 * w / tw:4.1f}%) ideal {i:11d} exec {e:9d}  {s[:60]}")
