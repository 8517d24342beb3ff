"""Summarise an ncu launch list (ncu --metrics gpu__time_duration.sum --csv --log-file F ...) per kernel.
usage: python tools/launch_summary.py gpurun_out/launches.csv "command line that was profiled" > profiles/rNN_ncu_launches_TAG.txt"""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "s": 1e3, "second": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= iv:
        continue
    name = r[ik].split("(")[0].replace("void ", "").strip()
    agg[name][0] += 1
    agg[name][1] += float(r[iv].replace(",", "")) * scale.get(r[iu], 1e-6)
tot = sum(v[1] for v in agg.values())
print("# ncu --metrics gpu__time_duration.sum --clock-control none --csv " + (sys.argv[2] if len(sys.argv) > 2 else ""))
print("# cold-cache serialised per-launch times; compare SHARES with the bench line's serial_stages_ms")
print("# kernel, launches, total ms, share of all kernel time")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:60s} {v[0]:6d} {v[1]:10.1f} ms {100 * v[1] / tot:6.2f}%")
