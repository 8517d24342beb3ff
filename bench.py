#!/usr/bin/env python
"""Benchmark of the B200 RRQ near-correction build (BASELINE.json metric: near-correction weights/s,
fp64, S/D/S'/D', on 1 B200; % of the FP64 roofline).

One STEP = one pass of the whole hot path over the workload:
  rrq_near_list -> rrq_patch_fit -> rrq_build_correction over all rows (in row chunks whose CSR
  output, 4 fp64 weights + 1 int32 column per entry, is written to HBM into reused chunk buffers).
Workload (N=1): BASELINE.json configs[3] ("cfg4"): bumpy sphere, 50,000 curved triangles, p = 8
(3.2M nodes), all on-surface node targets + 1M off-surface targets, near rule eta = 1.5, all four
kernels.  Synthetic, seeded (synth/configs.py).  Inputs and outputs exceed L2 (fit blocks 22 GB,
outputs ~300 GB per step), so no L2 flush is needed.

value    = weights (S+D+S'+D' CSR values) built per second over the timed steps, device-timed
           (CUDA events on the launch stream), max over ranks.
e2e      = the same metric with host buffers: per step the inputs are copied H2D from pinned host
           memory and every chunk's CSR (values + columns) is copied D2H into pinned host buffers,
           overlapped with the next chunk on a copy stream.
roofline = the dominant kernel of the build (by device time): algorithmic flops (paper_2411_08342_b200/flops.py)
           / its CUDA-event time, against the measured FP64 peak (profiles/r01_fp64_peak.txt).
--impl reference times the CPU oracle (oracle/, test infrastructure) on a bounded sample.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.1      # measured: DMMA m8n8k4 f64, 148 SMs @1965 MHz (profiles/r01_fp64_peak.txt)
FP64_PEAK_SRC = "measured FP64 peak (DMMA m8n8k4 microbenchmark, profiles/r01_fp64_peak.txt; DFMA chains 34.2)"
FP64_DFMA_TFLOPS = 34.2      # measured: independent DFMA chains, 8 CTAs/SM (same file)
# per kernel: which FP64 unit bounds it
KERNEL_BOUND = {"pair_edge": ("alu", FP64_DFMA_TFLOPS, "measured FP64 DFMA peak (profiles/r01_fp64_peak.txt)"),
                "translate": ("alu", FP64_DFMA_TFLOPS, "measured FP64 DFMA peak (profiles/r01_fp64_peak.txt)"),
                "qmap": ("tensor", FP64_PEAK_TFLOPS, "measured FP64 DMMA peak (profiles/r01_fp64_peak.txt)"),
                "contract": ("tensor", FP64_PEAK_TFLOPS, "measured FP64 DMMA peak (profiles/r01_fp64_peak.txt)")}


def traffic_per_launch(kernel, pairs, launches):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture (bytes per pair measured
    there x this run's average pairs per launch), or None."""
    import json as _j
    rec = None
    for name in ("r02_traffic.json", "r01_traffic.json"):   # the latest committed capture
        f = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", name)
        try:
            rec = _j.load(open(f)).get("k_" + kernel)
        except (OSError, ValueError):
            rec = None
        if rec:
            break
    if not rec or not launches:
        return None, None
    return rec["dram_bytes_per_pair"] * pairs / launches, rec["source"]
METRIC = "near-correction weights/s (fp64, S/D/S'/D') on 1 B200"
# BASELINE.md 1a (Table 3): rows/s/core of the paper's RRQ correction build, S and D separately
PAPER_TABLE3 = {p: {"rows_per_s_per_core_S": s_, "rows_per_s_per_core_D": d_, "hardware": "1 core, AMD EPYC 9474F 3.60 GHz",
                    "source": "PAPER.md Table 3 (P:L1921-1938)"}
                for p, s_, d_ in ((4, 21285, 27212), (6, 15065, 21376), (8, 9921, 15017), (10, 6621, 10449),
                                  (12, 4324, 6845), (14, 2907, 4534))}
UNIT = "weights/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n-off", type=int, default=None, help="override off-surface target count (debug)")
    ap.add_argument("--p", type=int, default=None, help="override the harmonic order (4..14; e.g. the paper's Table 3 p = 12, 14)")
    ap.add_argument("--freq", type=str, default=None,
                    help="override the mesh: icosphere frequency (configs 2, 4), or NTHxNPH / NUxNV (configs 3, 6)")
    ap.add_argument("--chunk-pairs", type=int, default=16_000_000)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-pairs", type=int, default=48000)
    ap.add_argument("--mask", type=int, default=None,
                    help="kernel mask (1 S, 2 D, 4 S', 8 D'); default all four, S|D for config 7 (no target normals)")
    return ap.parse_args()


# ------------------------------------------------------------------------------------------ dist
def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        import torch
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if torch.cuda.is_available() and dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if torch.cuda.is_available() and dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.rows, self.proc, self.idx = [], None, gpu_index

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())}


# ------------------------------------------------------------------------------------------ workload
def make_inputs(args, rank):
    from synth.configs import make_config
    kw = {}
    if args.n_off is not None:
        kw["n_off"] = args.n_off
    if getattr(args, "p", None) is not None:
        kw["p"] = args.p
    if args.freq is not None:
        kw["freq"] = tuple(int(v) for v in args.freq.split("x")) if "x" in args.freq else int(args.freq)
    return make_config(args.config, seed_offset=rank, **kw)


def cfg_desc(cfg, npairs, T, mask=None):
    S = cfg["surface"]
    mask = cfg.get("mask", 15) if mask is None else mask
    return {"workload": cfg["name"], "patches": int(S.n_patches), "p": int(S.p), "p_edge": int(S.q),
            "nodes": int(S.n_patches * S.n), "targets": int(T), "pairs": int(npairs) if npairs is not None else None, "eta": cfg["eta"],
            "kernels": ",".join(k for i, k in enumerate(("S", "D", "Sp", "Dp")) if (mask >> i) & 1),
            "l2": _l2_note(S, npairs)}


def _l2_note(S, npairs):
    """Inputs/outputs against the 126 MB L2: the bench never flushes, so say whether it needs to."""
    p_, n_p = S.p, S.p * (S.p + 1) // 2
    nq, nv = sum(j + 1 for j in range(2, p_ + 1)), sum(j + 1 for j in range(1, p_ + 1))
    # fit block: the 13 n_p x n fit operators + the K x (8 n_Q + 2 n_V) operand M of the line-integral maps
    fit_gb = S.n_patches * 8.0 * (13 * n_p * S.n + 18 * p_ * (8 * nq + 2 * nv)) / 1e9
    csr_gb = (npairs or 0) * S.n * 36 / 1e9
    big = fit_gb + csr_gb > 0.5
    return (f"inputs+outputs > L2 (fit ~{fit_gb:.1f} GB, CSR ~{csr_gb:.0f} GB per step): no flush needed" if big
            else f"small workload (fit ~{fit_gb:.2f} GB, CSR ~{csr_gb:.2f} GB): L2-resident, not a bench config")


class Runner:
    def __init__(self, cfg, args, device="cuda"):
        import torch
        from paper_2411_08342_b200 import RRQ, DeviceSurface, DeviceTargets
        self.torch = torch
        self.cfg, self.args = cfg, args
        S = cfg["surface"]
        self.S, self.n = S, S.n
        eta = cfg["eta"] if math.isfinite(cfg["eta"]) else 0.0
        self.ctx = RRQ(S.p, eta=eta, all_pairs=cfg["all_pairs"])
        self.ds = DeviceSurface.from_numpy(S)
        self.dt = DeviceTargets.from_numpy(cfg["tx"], cfg["tnormal"], cfg["self_node"], cfg["side"])
        self.T = self.dt.n_targets
        m = getattr(args, "mask", None)
        self.mask = m if m is not None else cfg.get("mask", 15)
        self.nk = bin(self.mask).count("1")
        self.bufs = None
        self.stream = torch.cuda.current_stream()

    def alloc_out(self, cap):
        t = self.torch
        n = self.n
        return dict(row_ptr=t.empty(self.T + 1, dtype=t.int64, device="cuda"),
                    col_idx=t.empty(cap * n, dtype=t.int32, device="cuda"),
                    vals=[t.empty(cap * n, dtype=t.float64, device="cuda") if (self.mask >> k) & 1 else None
                          for k in range(4)],
                    status=t.empty(cap, dtype=t.int32, device="cuda"))

    def chunks(self, hptr, cap):
        T = hptr.shape[0] - 1
        out, r0 = [], 0
        while r0 < T:
            r1 = int(np.searchsorted(hptr, hptr[r0] + cap, side="right")) - 1
            r1 = max(r1, r0 + 1)
            r1 = min(r1, T)
            out.append((r0, r1))
            r0 = r1
        return out

    def step(self, out_sets=None, on_chunk=None):
        """One pass: near list, patch fit, build over all row chunks."""
        ptr, pat = self.ctx.near_list(self.ds, self.dt)
        if on_chunk is not None:
            on_chunk("near", -1, (ptr, pat))
        fit, fst = self.ctx.patch_fit(self.ds)
        hptr = ptr.cpu().numpy()
        cap = self.args.chunk_pairs
        sets = out_sets or self.bufs
        ch = self.chunks(hptr, cap)
        for i, (r0, r1) in enumerate(ch):
            o = sets[i % len(sets)]
            if on_chunk is not None:
                on_chunk("before", i, o)
            rp = o["row_ptr"][: r1 - r0 + 1]
            self.ctx.build_correction(self.ds, self.dt, ptr, pat, fit, mask=self.mask, row_begin=r0, row_end=r1,
                                      out=dict(row_ptr=rp, col_idx=o["col_idx"], vals=o["vals"], status=o["status"]))
            if on_chunk is not None:
                on_chunk("after", i, o, int(hptr[r1] - hptr[r0]))
        self.npairs = int(hptr[-1])
        self.n_close = int((np.diff(hptr) > 0).sum())   # targets with at least one near patch
        self.fit = fit
        return self.npairs


def run_ours(args, ws, rank):
    import torch
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    t0 = time.time()
    cfg = make_inputs(args, rank)
    gen_s = time.time() - t0
    R = Runner(cfg, args)
    R.bufs = [R.alloc_out(args.chunk_pairs)]
    # warmup
    for _ in range(args.warmup):
        R.step()
    torch.cuda.synchronize()
    # timed region
    clk = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    R.ctx.reset_timing()
    R.ctx.set_timing(True)
    launches0 = R.ctx.launch_count()
    barrier(ws)
    torch.cuda.synchronize()
    clk.start()
    time.sleep(0.3)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        R.step()
    e1.record()
    torch.cuda.synchronize()
    clocks = clk.stop()
    barrier(ws)
    launches = R.ctx.launch_count() - launches0
    npairs = R.npairs
    weights_per_step = npairs * R.n * R.nk
    R.ctx.set_timing(False)
    ms = e0.elapsed_time(e1)
    ms_max = max_over_ranks(ms, ws)
    tim = R.ctx.timing()
    total_weights = sum_over_ranks(weights_per_step * args.steps, ws)
    value = total_weights / (ms_max / 1e3)
    from paper_2411_08342_b200.flops import pair_flops, pair_bytes
    pf = pair_flops(R.S.p, mask=R.mask)
    pairs_t = max(tim["pairs"], 1)
    swap_per_pair = tim["swap_edges"] / pairs_t
    kflops = {"pair_edge": (pf["edge"] + swap_per_pair * pf["swap_edge"]) * pairs_t,
              "qmap": pf["qmap"] * pairs_t, "translate": pf["translate"] * pairs_t,
              "contract": pf["contract"] * pairs_t}
    per_kernel = {k: {"ms_per_step": tim["ms"][k] / args.steps,
                      "tflops": v / (tim["ms"][k] / 1e3) / 1e12 if tim["ms"][k] > 0 else None}
                  for k, v in kflops.items()}
    # dominant kernel = the one carrying the most algorithmic work (k_qmap); per-kernel device times are taken
    # with k_pair_edge of the next sub-chunk running concurrently (it overlaps mostly k_contract), so the
    # time-largest entry is not a clean per-kernel figure; the build-stage fraction is the headline
    dom = max(kflops, key=lambda k: kflops[k])
    achieved = per_kernel[dom]["tflops"]
    traffic, traffic_src = traffic_per_launch(dom, pairs_t, tim["launches"][dom])
    for k in per_kernel:
        per_kernel[k]["bound"], per_kernel[k]["peak"] = KERNEL_BOUND[k][0], KERNEL_BOUND[k][1]
        per_kernel[k]["frac"] = (per_kernel[k]["tflops"] or 0) / KERNEL_BOUND[k][1]
    # the build stage's device time: whole rrq_build_correction calls on the caller's stream (k_pair_edge of
    # the next sub-chunk runs concurrently with the GEMM kernels of the current one, so per-kernel times overlap)
    build_ms = tim["ms"].get("build") or sum(tim["ms"][k] for k in ("pair_edge", "qmap", "translate", "contract", "plumbing"))
    # the kernels' own device times: one extra (untimed) step with the overlap off
    R.ctx.set_overlap(False)
    R.ctx.reset_timing()
    R.ctx.set_timing(True)
    R.step()
    torch.cuda.synchronize()
    tser = R.ctx.timing()
    R.ctx.set_timing(False)
    R.ctx.set_overlap(True)
    for k in per_kernel:
        ms_k = tser["ms"][k]
        per_kernel[k]["serial_ms_per_step"] = ms_k
        per_kernel[k]["serial_tflops"] = kflops[k] / args.steps / (ms_k / 1e3) / 1e12 if ms_k > 0 else None
        per_kernel[k]["serial_frac"] = (per_kernel[k]["serial_tflops"] or 0) / KERNEL_BOUND[k][1]
    build_tflops = sum(kflops.values()) / (build_ms / 1e3) / 1e12
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generator synth/configs.py; BASELINE.json configs[3] shape)",
        "config": dict(cfg_desc(cfg, npairs, R.T, R.mask), parallelism=f"replicas{ws}" if ws > 1 else "single",
                       step="near_list+patch_fit+build(all rows, chunked)", chunk_pairs=args.chunk_pairs),
        "roofline": {"bound": KERNEL_BOUND[dom][0], "kernel": "k_" + dom, "achieved": achieved,
                     "peak": KERNEL_BOUND[dom][1], "unit": "TFLOP/s", "frac": achieved / KERNEL_BOUND[dom][1],
                     "traffic": traffic, "traffic_unit": "bytes/launch", "traffic_source": traffic_src,
                     "peak_source": KERNEL_BOUND[dom][2],
                     "flops_per_pair": kflops[dom] / pairs_t, "launches": tim["launches"][dom],
                     "build_stage_tflops": build_tflops, "build_stage_frac": build_tflops / FP64_PEAK_TFLOPS,
                     "per_kernel": per_kernel,
                     "per_kernel_note": "ms_per_step/tflops/frac: timed steps, overlap on (k_pair_edge of sub-chunk i+1 "
                                        "co-runs with k_qmap/k_translate/k_contract of sub-chunk i); serial_*: one extra "
                                        "untimed step with the overlap off (the kernels' own device times)"},
        "stages_ms_per_step": {k: v / args.steps for k, v in tim["ms"].items()},
        "serial_stages_ms": dict(tser["ms"]),
        "pairs_per_s": npairs * args.steps / (ms_max / 1e3) * ws,
        "rows_per_s": R.T * args.steps / (ms_max / 1e3) * ws,
        # the paper's throughput unit for the evaluation phase: close targets (rows with a correction) per
        # second, X_RRQ = N_T^c / T_RRQ
        "close_rows_per_s": R.n_close * args.steps / (ms_max / 1e3) * ws,
        "swap_edges_per_pair": swap_per_pair,
        # context, not the target: the paper's correction-build throughput for this p (Table 3, P:L1921-1938;
        # one core of a 3.60 GHz AMD EPYC 9474F, Fortran; on-surface targets of a stellarator; S and D
        # built separately) in points (rows) per second per core
        "paper_context": PAPER_TABLE3.get(R.S.p),
        "clocks": clocks,
        "gpu_launches": int(launches),
        "gen_s": gen_s,
    }
    # e2e through host buffers
    if not args.no_e2e and args.e2e_steps > 0:
        res["e2e"] = run_e2e(R, cfg, args, ws)
    else:
        res["e2e"] = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            res["cpu_baseline"] = cpu_baseline(cfg, args, R)
        except Exception as ex:  # report, never hide
            res["cpu_baseline"] = {"error": repr(ex)}
    return res


def run_e2e(R, cfg, args, ws):
    """Same metric with host buffers: pinned host inputs copied H2D each step; the host receives the CSR as
    (pair_ptr, pair_patch, values): pair_ptr (read by the step itself for the row chunking) and pair_patch once
    per step, every chunk's masked value arrays D2H (overlapped on a copy stream, double-buffered device
    outputs).  col_idx and row_ptr are implied (col = patch * n + local, row_ptr = pair_ptr * n; include/rrq.h)
    and are not shipped."""
    import torch
    from paper_2411_08342_b200 import DeviceSurface, DeviceTargets
    S = cfg["surface"]
    pin = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).pin_memory()
    h_in = dict(nodes=pin(S.nodes, torch.float64), normals=pin(S.normals, torch.float64),
                weights=pin(S.weights, torch.float64), verts=pin(S.verts, torch.float64),
                edge_x=pin(S.edge_x, torch.float64), edge_dx=pin(S.edge_dx, torch.float64),
                x=pin(cfg["tx"], torch.float64), normal=pin(cfg["tnormal"], torch.float64),
                self_node=pin(cfg["self_node"], torch.int64), side=pin(cfg["side"], torch.int8))
    d_in = {k: torch.empty(v.shape, dtype=v.dtype, device="cuda") for k, v in h_in.items()}
    h2d = sum(v.numel() * v.element_size() for v in h_in.values())
    cap = min(args.chunk_pairs, int(os.environ.get("RRQ_E2E_CAP", "4000000")))
    nset = int(os.environ.get("RRQ_E2E_SETS", "2"))
    old_cap = args.chunk_pairs
    args.chunk_pairs = cap
    sets = [R.alloc_out(cap) for _ in range(nset)]
    n = R.n
    h_out = [dict(vals=[torch.empty(cap * n, dtype=torch.float64).pin_memory() if (R.mask >> j) & 1 else None
                        for j in range(4)]) for _ in range(nset)]
    h_pat = torch.empty(max(R.npairs, 1), dtype=torch.int32).pin_memory()
    copy_stream = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    done = [torch.cuda.Event() for _ in range(nset)]
    d2h_bytes = [0]

    def on_chunk(when, i, o, np_=0):
        if when == "near":
            ptr, pat = o
            ev = torch.cuda.Event()
            ev.record(main)
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(ev)
                h_pat[: pat.numel()].copy_(pat, non_blocking=True)
            d2h_bytes[0] += pat.numel() * 4 + ptr.numel() * 8     # pair_patch here, pair_ptr by the step's .cpu()
            return
        k = i % nset
        if when == "before":
            main.wait_event(done[k])          # the copy of this buffer's previous chunk has finished
            return
        ev = torch.cuda.Event()
        ev.record(main)
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(ev)
            m = np_ * n
            for j in range(4):
                if h_out[k]["vals"][j] is not None:
                    h_out[k]["vals"][j][:m].copy_(o["vals"][j][:m], non_blocking=True)
            done[k].record(copy_stream)
        d2h_bytes[0] += m * 8 * R.nk

    def one_step():
        for k, v in h_in.items():
            d_in[k].copy_(v, non_blocking=True)
        R.ds = DeviceSurface(d_in["nodes"], d_in["normals"], d_in["weights"], d_in["verts"], d_in["edge_x"],
                             d_in["edge_dx"])
        R.dt = DeviceTargets(d_in["x"], d_in["normal"], d_in["self_node"], d_in["side"])
        R.step(out_sets=sets, on_chunk=on_chunk)
        copy_stream.synchronize()

    one_step()   # warm (allocations)
    torch.cuda.synchronize()
    d2h_bytes[0] = 0
    barrier(ws)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.e2e_steps):
        one_step()
    main.wait_stream(copy_stream)
    e1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), ws)
    args.chunk_pairs = old_cap
    w = sum_over_ranks(R.npairs * n * R.nk * args.e2e_steps, ws)
    return {"value": w / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h_bytes[0] / args.e2e_steps), "steps": args.e2e_steps,
            "ms_per_step": ms / args.e2e_steps,
            "host_csr": "pair_ptr + pair_patch + value arrays (col_idx = patch*n + local, row_ptr = pair_ptr*n implied)"}


def sample_pairs(cfg, budget, seed=7):
    """Bounded sample for the CPU oracle: all near pairs (oracle near rule) of a few random patches, so
    the per-patch Steps 1-3 cost is paid as in a full build; about `budget` pairs."""
    from oracle import oracle as O
    S = cfg["surface"]
    rng = np.random.default_rng(seed)
    order = rng.permutation(S.n_patches)
    chosen, tg, pa = [], [], []
    tot = 0
    for q in order[:200]:
        t, p_ = O.near_pairs_for_patches(S, cfg["tx"], cfg["self_node"], cfg["eta"], [q], cfg["all_pairs"])
        if t.size == 0:
            continue
        take = min(t.size, budget - tot)
        tg.append(t[:take]); pa.append(p_[:take]); chosen.append(q)
        tot += take
        if tot >= budget:
            break
    return np.concatenate(tg), np.concatenate(pa), len(chosen)


def parity_sample(R, tg, pa, max_pairs=1500, seed=11):
    """One more full step (untimed) in the timed launch configuration, gathering the CSR rows of a seeded
    subsample of the oracle's sampled pairs on the device; per kernel the GPU's and the fp64 oracle's row
    errors against the binary128 truth (median / 90th percentile / max of max_i |x_i - t_i| / max_i |t_i|,
    rows within 1e-11) and the parity bar of tests/parity_util.py."""
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import parity_util as U
    rng = np.random.default_rng(seed)
    if tg.size > max_pairs:
        sel = np.sort(rng.choice(tg.size, max_pairs, replace=False))
        tg, pa = tg[sel], pa[sel]
    cfg, n = R.cfg, R.n
    ptr, pat = R.ctx.near_list(R.ds, R.dt)
    hptr, hpat = ptr.cpu().numpy(), pat.cpu().numpy()
    ch = R.chunks(hptr, R.args.chunk_pairs)
    pos = np.empty(tg.size, np.int64)
    for i, (t, q) in enumerate(zip(tg, pa)):
        seg = hpat[hptr[t]:hptr[t + 1]]
        j = int(np.searchsorted(seg, q))
        if j >= seg.size or seg[j] != q:
            raise RuntimeError("sampled pair missing from the GPU near list")
        pos[i] = hptr[t] + j
    got = np.zeros((4, tg.size, n))

    def on_chunk(when, i, o, npairs=None):
        if when != "after":
            return
        r0, r1 = ch[i]
        sel = np.where((pos >= hptr[r0]) & (pos < hptr[r1]))[0]
        if sel.size == 0:
            return
        idx = torch.as_tensor(pos[sel] - hptr[r0], device="cuda")
        for k in range(4):
            if o["vals"][k] is not None:
                got[k, sel] = o["vals"][k][: npairs * n].view(npairs, n).index_select(0, idx).cpu().numpy()

    R.step(on_chunk=on_chunk)
    t0 = time.time()
    tgs = (cfg["tx"], cfg["tnormal"], cfg["self_node"], cfg["side"])
    ref = U.reference(cfg["surface"], tgs, tg, pa, mask=R.mask)
    inv = np.unique(tg, return_inverse=True)[1]
    out = {"pairs": int(tg.size), "rows": int(inv.max() + 1), "truth": "oracle in IEEE binary128 (liboracle_q.so)",
           "truth_seconds": time.time() - t0,
           "bar": f"per row e_g <= {U.ROW_FACTOR:g} x fp64 rounding envelope + 1e-11 rowmax; median/p90 within "
                  f"{U.Q_FACTOR:g}x, max within {U.MAX_FACTOR:g}x of the fp64 oracle's"}
    for k, name in enumerate(("S", "D", "Sp", "Dp")):
        if not (R.mask >> k) & 1:
            continue
        ok, st = U.gate_rows(got[k], ref, k, inv)
        out[name] = dict(st, passes=bool(ok))
    return out


def cpu_baseline(cfg, args, R=None, steps=1):
    from oracle import oracle as O
    S = cfg["surface"]
    tg, pa, npatch = sample_pairs(cfg, args.cpu_sample_pairs)
    cores = os.cpu_count()
    t0 = time.time()
    for _ in range(steps):
        vo, _ = O.build_rows(S, cfg["tx"], cfg["tnormal"], cfg["self_node"], cfg["side"], tg, pa)
    el = (time.time() - t0) / steps
    w = tg.shape[0] * S.n * 4
    res = {"value": w / el, "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"{tg.shape[0]} pairs = all near pairs of {npatch} random patches of {cfg['name']} "
                     f"(Steps 1-8 incl. per-patch fit, all 4 kernels), {el:.1f} s on {cores} OpenMP threads",
           "seconds": el, "pairs": int(tg.shape[0])}
    if R is not None:   # a subsample of the same pairs out of a full-size build in the timed launch configuration
        try:
            res["parity_sample"] = parity_sample(R, tg, pa)
        except Exception as ex:  # report, never hide
            res["parity_sample"] = {"error": repr(ex)}
    # like-for-like with the paper's single-core numbers: the first patch's pairs on one thread
    try:
        import ctypes
        gomp = ctypes.CDLL("libgomp.so.1")
        n1 = min(3000, len(pa))
        gomp.omp_set_num_threads(1)
        t1 = time.time()
        O.build_rows(S, cfg["tx"], cfg["tnormal"], cfg["self_node"], cfg["side"], tg[:n1], pa[:n1])
        e1 = time.time() - t1
        gomp.omp_set_num_threads(cores)
        rows1 = np.unique(tg[:n1]).size
        # a CSR row of the full workload holds npairs / n_close pairs (near patches per close target), so one
        # core's rows/s equivalent is its pairs/s divided by that (the sample's own pairs-per-target is ~1:
        # it takes all pairs of a few patches)
        ppr = (R.npairs / max(R.n_close, 1)) if R is not None else None
        res["one_core"] = {"value": n1 * S.n * 4 / e1, "unit": UNIT, "pairs": n1, "seconds": e1,
                           "pairs_per_s": n1 / e1, "pairs_per_row_full_workload": ppr,
                           "rows_per_s_equiv": (n1 / e1 / ppr) if ppr else None,
                           "sample": f"first {n1} pairs of the sample ({rows1} distinct targets), 1 OpenMP thread"}
    except OSError as ex:
        res["one_core"] = {"error": repr(ex)}
    return res


def run_reference(args, ws, rank):
    """--impl reference: the CPU oracle as it stands on a bounded sample of the same workload."""
    if rank != 0:
        return None
    cfg = make_inputs(args, 0)
    from oracle import oracle as O
    S = cfg["surface"]
    tg, pa, npatch = sample_pairs(cfg, args.cpu_sample_pairs)
    for _ in range(args.warmup):
        O.build_rows(S, cfg["tx"], cfg["tnormal"], cfg["self_node"], cfg["side"], tg[:50], pa[:50])
    t0 = time.time()
    for _ in range(args.steps):
        O.build_rows(S, cfg["tx"], cfg["tnormal"], cfg["self_node"], cfg["side"], tg, pa)
    el = (time.time() - t0)
    w = tg.shape[0] * S.n * 4 * args.steps
    v = w / el
    cores = os.cpu_count()
    sample = (f"{tg.shape[0]} pairs per step = all near pairs of {npatch} random patches of {cfg['name']} "
              f"(Steps 1-8 incl. per-patch fit, all 4 kernels)")
    return {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": cfg_desc(cfg, None, cfg["tx"].shape[0]),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    ws, rank, local = dist_setup(args)
    if args.impl == "reference":
        res = run_reference(args, ws, rank)
    else:
        res = run_ours(args, ws, rank)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
