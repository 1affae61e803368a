"""Raw PCIe rates on the box: pinned H2D / D2H of 134 MB blocks, one stream and four streams."""
import time, torch
n = 16777216
dev = torch.empty((8, n), dtype=torch.float64, device="cuda")
host = torch.empty((64, n), dtype=torch.float64).pin_memory()
def run(nstreams, d2h=True):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize(); t = time.perf_counter()
    for i in range(64):
        with torch.cuda.stream(ss[i % nstreams]):
            if d2h: host[i].copy_(dev[i % 8], non_blocking=True)
            else: dev[i % 8].copy_(host[i], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    return 64 * n * 8 / dt / 1e9
for k in (1, 4):
    print(f"D2H {k} stream(s): {run(k):.1f} GB/s   H2D {k} stream(s): {run(k, False):.1f} GB/s")
