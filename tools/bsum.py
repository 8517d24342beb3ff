"""One-line summary of bench JSON lines: python tools/bsum.py FILE..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as ex:  # noqa: BLE001
        print(f, "unreadable", ex)
        continue
    r = d["roofline"]
    pk = {k: round(v["serial_ms_per_step"], 1) for k, v in r["per_kernel"].items()}
    print(f"{f}: {d['value']:.4e} {d['unit']} {d['ms_per_step']:.0f} ms/step build {r['build_stage_frac']:.3f} "
          f"{r['kernel']} {r['frac']:.3f} kernels={d['config']['kernels']} serial={pk} fit={d['stages_ms_per_step']['patch_fit']:.0f}"
          f" clocks={d['clocks'].get('sm_mhz')} newton_serial={d.get('serial_stages_ms', {}).get('newton')}")
