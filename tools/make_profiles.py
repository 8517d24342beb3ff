"""Summarise the ncu artefacts of a bench run into profiles/ (committed evidence).

usage: python tools/make_profiles.py TAG
  reads gpurun_out/launches_full.csv (ncu --metrics gpu__time_duration.sum launch list of
  `bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline`), gpurun_out/prof_qmap_cfg4.ncu-rep
  (ncu --set full of the first k_qmap launch of the same command) and gpurun_out/bench_full.json;
  writes profiles/r01_ncu_launches_cfg4.txt, profiles/r01_ncu_qmap_cfg4.txt, profiles/r01_traffic.json,
  profiles/r01_bench_TAG.json.
"""
import collections
import csv
import io
import json
import shutil
import subprocess
import sys

tag = sys.argv[1]
rows = list(csv.reader(open("gpurun_out/launches_full.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= iv:
        continue
    name = r[ik].split("(")[0].replace("void ", "").strip()
    agg[name][0] += 1
    agg[name][1] += float(r[iv].replace(",", ""))
tot = sum(v[1] for v in agg.values())
with open("profiles/r01_ncu_launches_cfg4.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 1 --warmup 3 "
            "--no-e2e --no-cpu-baseline\n")
    f.write("# (cfg4, 4 build steps: 3 warm-up + 1 timed; cold-cache serialised per-launch times; compare SHARES "
            "with the bench line)\n# kernel, launches, total ms, share of all kernel time\n")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f"{k:60s} {v[0]:6d} {v[1] / 1e6:10.1f} ms {100 * v[1] / tot:6.2f}%\n")

rep = "gpurun_out/prof_qmap_cfg4.ncu-rep"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, v, u = r[0], r[2], r[1]
keep = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__inst_executed.sum"]
grid = int(float(v[h.index("launch__grid_size")]))
tp = 16
hot = subprocess.run(["python", "tools/ncu_hot.py", rep], capture_output=True, text=True).stdout
with open("profiles/r01_ncu_qmap_cfg4.txt", "w") as f:
    f.write("# ncu --set full --import-source on --clock-control none -k regex:k_qmap -c 1 python bench.py --steps 1 "
            "--warmup 3 --no-e2e --no-cpu-baseline\n")
    f.write(f"# first k_qmap launch of the cfg4 bench ({grid} tiles of {tp} pairs)\n")
    for k in keep:
        i = h.index(k)
        f.write(f"{k:80s} {v[i]} {u[i]}\n")
    rd = float(v[h.index("dram__bytes_read.sum")])
    wr = float(v[h.index("dram__bytes_write.sum")])
    per = (rd + wr) * 1e9 / (grid * tp)
    f.write(f"# DRAM traffic per launch {rd + wr:.3f} GB = {per:.0f} B per pair slot (algorithmic: A rows 2.3 KB in + "
            "Q/dQ/V row 6.1 KB out = 8.4 KB)\n")
    f.write(hot)
json.dump({"k_qmap": {"dram_bytes_per_pair": per,
                      "source": "profiles/r01_ncu_qmap_cfg4.txt (ncu --set full, cfg4 first launch)"}},
          open("profiles/r01_traffic.json", "w"), indent=1)
shutil.copy("gpurun_out/bench_full.json", f"profiles/r01_bench_{tag}.json")
print(open("profiles/r01_ncu_launches_cfg4.txt").read())
