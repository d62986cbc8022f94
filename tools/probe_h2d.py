"""H2D bandwidth from pinned host memory: one copy vs chunked copies on
several streams (16 GiB)."""
import time, torch

n = 2 * 1024 ** 3  # doubles = 16 GiB
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"single copy: {n * 8 / dt / 1e9:.1f} GB/s")
for ns, chunk_mb in ((2, 256), (4, 256), (4, 64), (8, 128)):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    ch = chunk_mb * 1024 * 1024 // 8
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, o in enumerate(range(0, n, ch)):
        s = streams[i % ns]
        with torch.cuda.stream(s):
            d[o:o + ch].copy_(h[o:o + ch], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{ns} streams x {chunk_mb} MB chunks: {n * 8 / dt / 1e9:.1f} GB/s")
