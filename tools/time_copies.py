"""Host<->device copy bandwidths of a 930^3-sized field (pinned host memory):
H2D, D2H, both directions concurrently (two streams), chunked."""
import sys, time
import torch
n = int(sys.argv[1]) if len(sys.argv) > 1 else 930
host = torch.empty((n, n, n), dtype=torch.float64).pin_memory()
host2 = torch.empty((n, n, n), dtype=torch.float64).pin_memory()
dev = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
dev2 = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
gb = host.numel() * 8 / 1e9
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn):
    torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize()
    return time.perf_counter() - t
for _ in range(2):
    h2d = timed(lambda: dev.copy_(host, non_blocking=True))
    d2h = timed(lambda: host.copy_(dev, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): dev.copy_(host, non_blocking=True)
        with torch.cuda.stream(s2): host2.copy_(dev2, non_blocking=True)
    bi = timed(both)
    def chunked():
        for a in range(0, n, n // 16 + 1):
            b = min(n, a + n // 16 + 1)
            with torch.cuda.stream(s1): dev[a:b].copy_(host[a:b], non_blocking=True)
            with torch.cuda.stream(s2): host2[a:b].copy_(dev2[a:b], non_blocking=True)
    ch = timed(chunked)
print(f"{gb:.2f} GB: H2D {gb/h2d:.1f} GB/s, D2H {gb/d2h:.1f} GB/s, concurrent both {2*gb/bi:.1f} GB/s "
      f"({bi:.3f} s), chunked concurrent {2*gb/ch:.1f} GB/s ({ch:.3f} s)")
