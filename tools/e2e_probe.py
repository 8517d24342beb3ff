"""Probe of the e2e overlap: per-chunk timeline of compute (main stream) and D2H copies (copy stream)."""
import sys, os, time, types, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.argv = ['bench.py']
import bench
args = bench.parse()
cfg = bench.make_inputs(args, 0)
R = bench.Runner(cfg, args); R.bufs = [R.alloc_out(args.chunk_pairs)]
R.step(); torch.cuda.synchronize()
cap = 4_000_000; args.chunk_pairs = cap
n = R.n
sets = [R.alloc_out(cap), R.alloc_out(cap)]
h_out = [dict(col=torch.empty(cap * n, dtype=torch.int32).pin_memory(),
              vals=[torch.empty(cap * n, dtype=torch.float64).pin_memory() for _ in range(4)]) for _ in range(2)]
cs = torch.cuda.Stream(); main = torch.cuda.current_stream()
done = [torch.cuda.Event(), torch.cuda.Event()]
t0 = torch.cuda.Event(enable_timing=True); t0.record()
marks = []
def on_chunk(when, i, o, np_=0):
    k = i % 2
    if when == "near":
        return
    if when == "before":
        main.wait_event(done[k]); a = torch.cuda.Event(enable_timing=True); a.record(main); marks.append(("cb", i, a)); return
    e = torch.cuda.Event(enable_timing=True); e.record(main); marks.append(("ce", i, e))
    with torch.cuda.stream(cs):
        cs.wait_event(e)
        a = torch.cuda.Event(enable_timing=True); a.record(cs); marks.append(("xb", i, a))
        m = np_ * n
        h_out[k]["col"][:m].copy_(o["col_idx"][:m], non_blocking=True)
        for j in range(4): h_out[k]["vals"][j][:m].copy_(o["vals"][j][:m], non_blocking=True)
        done[k].record(cs); b = torch.cuda.Event(enable_timing=True); b.record(cs); marks.append(("xe", i, b))
w0 = time.time()
R.step(out_sets=sets, on_chunk=on_chunk)
cs.synchronize(); torch.cuda.synchronize()
print("wall", time.time() - w0)
for kind, i, ev in marks[:16]:
    print(kind, i, round(t0.elapsed_time(ev), 1))
print("last", [(k, i, round(t0.elapsed_time(e), 1)) for k, i, e in marks[-4:]])
