"""Stall samples and executed instructions per SASS address bucket of one kernel in an ncu report.

usage: KERNEL=regex python tools/ncu_regions.py REPORT.ncu-rep [bucket_hex]
"""
import csv, io, os, subprocess, sys
rep = sys.argv[1]
B = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0x400
flt = ["-k", "regex:" + os.environ["KERNEL"]] if os.environ.get("KERNEL") else []
out = subprocess.run(["ncu", "-i", rep, *flt, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iex, isrc, ia, ism = (h.index(k) for k in ("Instructions Executed", "Source", "Address",
                                           "Warp Stall Sampling (All Samples)"))
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
base, recs = None, []
for r in rows[2:]:
    try:
        e, sm = int(r[iex] or 0), int(r[ism] or 0)
    except (ValueError, IndexError):
        continue
    a = int(r[ia], 16)
    if base is None:
        base = a
    if a - base < (recs[-1][0] if recs else -1):
        break   # a second kernel's listing
    recs.append((a - base, e, sm, r[isrc].strip(), {c: int(r[h.index(c)] or 0) for c in reasons}))
tot = sum(x[2] for x in recs) or 1
bk = {}
for a, e, sm, src, rs in recs:
    d = bk.setdefault(a // B, [0, 0, src[:44], {}])
    d[0] += sm
    d[1] += e
    for c, v in rs.items():
        d[3][c] = d[3].get(c, 0) + v
for k in sorted(bk):
    d = bk[k]
    top = sorted(d[3].items(), key=lambda x: -x[1])[:3]
    s = sum(d[3].values()) or 1
    print(f"{k * B:6x} {100 * d[0] / tot:5.1f}% inst {d[1]:11d} | " +
          ", ".join(f"{c[6:]} {100 * v / s:.0f}%" for c, v in top) + f" | {d[2]}")
