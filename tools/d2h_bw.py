"""D2H bandwidth into pinned host memory: one copy stream vs several concurrent ones (e2e tuning)."""
import time, torch
n = 1 << 28   # 2 GiB of fp64 per buffer
dev = [torch.empty(n, dtype=torch.float64, device="cuda").fill_(1.0) for _ in range(4)]
host = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(4)]
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    torch.cuda.synchronize()
    t = time.time()
    for rep in range(2):
        for i in range(4):
            with torch.cuda.stream(streams[i % ns]):
                host[i].copy_(dev[i], non_blocking=True)
    torch.cuda.synchronize()
    el = time.time() - t
    print(f"streams {ns}: {2 * 4 * n * 8 / el / 1e9:.1f} GB/s")
# H2D for reference
torch.cuda.synchronize(); t = time.time()
for i in range(4): dev[i].copy_(host[i], non_blocking=True)
torch.cuda.synchronize(); print(f"H2D 1 stream: {4 * n * 8 / (time.time() - t) / 1e9:.1f} GB/s")
