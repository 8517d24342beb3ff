"""DRAM traffic per pair of each build kernel from the ncu --set full reports of tools/ncu_cfg4.sh (on the box):
python tools/ncu_traffic.py TAG > gpurun_out/traffic_TAG.json.  Pairs of the captured launch: k_qmap / k_contract
launch one CTA per tile of 16 pairs (grid x 16, an upper bound within a tile per patch); the other kernels are
given the same sub-chunk's pair count (all six captures skip the same number of launches)."""
import csv, io, json, subprocess, sys
tag = sys.argv[1]
out, pairs = {}, None
recs = {}
for k in ("k_qmap", "k_contract", "k_newton", "k_edge_lines", "k_target_gamma", "k_translate"):
    rep = f"/tmp/ncu_{tag}_{k}.ncu-rep"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    if len(r) < 3:
        continue
    h, v = r[0], r[2]
    g = lambda n: float(v[h.index(n)].replace(",", "")) if n in h else None
    recs[k] = dict(grid=g("launch__grid_size"), rd=g("dram__bytes_read.sum"), wr=g("dram__bytes_write.sum"),
                   ns=g("gpu__time_duration.sum"), rd_unit=r[1][h.index("dram__bytes_read.sum")],
                   wr_unit=r[1][h.index("dram__bytes_write.sum")],
                   t_unit=r[1][h.index("gpu__time_duration.sum")])
if "k_qmap" in recs:
    pairs = recs["k_qmap"]["grid"] * 16
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for k, r in recs.items():
    sc, sw = scale.get(r["rd_unit"], 1.0), scale.get(r["wr_unit"], 1.0)
    out[k] = {"dram_bytes_per_pair": (r["rd"] * sc + r["wr"] * sw) / pairs if pairs else None,
              "dram_read_bytes": r["rd"] * sc, "dram_write_bytes": r["wr"] * sw, "pairs_in_launch_upper_bound": pairs,
              "duration": r["ns"], "duration_unit": r["t_unit"], "grid": r["grid"],
              "source": f"profiles/r02_ncu_{k}_cfg4.txt (ncu --set full, cfg4 launch configuration, 13th launch)"}
print(json.dumps(out, indent=1))
