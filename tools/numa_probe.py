"""Host<->device copy rates with the process pinned to the GPU's local CPUs
vs unpinned (NUMA placement of pinned host memory).  Prints box topology."""
import os, sys, time
import torch
import pynvml

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
bus = pynvml.nvmlDeviceGetPciInfo(h).busId
bus = bus.decode() if isinstance(bus, bytes) else bus
path = f"/sys/bus/pci/devices/{bus.lower()[4:] if len(bus) > 12 else bus.lower()}"
local = open(os.path.join(path, "local_cpulist")).read().strip() if os.path.exists(path) else "?"
node = open(os.path.join(path, "numa_node")).read().strip() if os.path.exists(path) else "?"
print("gpu bus", bus, "numa_node", node, "local_cpulist", local, "ncpu", os.cpu_count(),
      "affinity now", len(os.sched_getaffinity(0)), flush=True)


def parse(lst):
    out = set()
    for part in lst.split(","):
        a, _, b = part.partition("-")
        out.update(range(int(a), int(b or a) + 1))
    return out


def rates(tag):
    n = 930
    host = torch.empty((n, n, n), dtype=torch.float64).pin_memory()
    host.fill_(1.0)  # first touch by this thread
    dev = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    gb = host.numel() * 8 / 1e9
    best = [0, 0]
    for _ in range(3):
        torch.cuda.synchronize(); t = time.perf_counter(); dev.copy_(host, non_blocking=True)
        torch.cuda.synchronize(); best[0] = max(best[0], gb / (time.perf_counter() - t))
        torch.cuda.synchronize(); t = time.perf_counter(); host.copy_(dev, non_blocking=True)
        torch.cuda.synchronize(); best[1] = max(best[1], gb / (time.perf_counter() - t))
    print(tag, f"H2D {best[0]:.1f} GB/s D2H {best[1]:.1f} GB/s", flush=True)
    del host, dev


if sys.argv[1:] == ["local"] and local != "?":
    os.sched_setaffinity(0, parse(local))
    rates("pinned-to-local-cpus")
else:
    rates("default-affinity")
