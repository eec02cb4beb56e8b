"""Time the GPU B-spline transforms at ncoef^3 (p=3 default): direct transform
(prefilter, 3 axes, in the slab layout) + reflect pad, and sample_solution.
    python tools/time_transform.py [ncoef] [p]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_03057_b200.device import SlabLayout, require_cuda
from paper_1904_03057_b200.domain import Grid
from paper_1904_03057_b200.gram import basis_extension
from paper_1904_03057_b200.transform import (prefilter_device, reflect_pad_device,
                                             sample_solution_device)
ncoef = int(sys.argv[1]) if len(sys.argv) > 1 else 930
p = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ext = basis_extension(p)
N = ncoef - 2 * ext
grid = Grid((N,) * 3, (1.0 / (N - 1),) * 3)
dev = require_cuda()
lay = SlabLayout(ncoef, ncoef, ncoef, ghost=p)
buf = lay.alloc(dev)
own = lay.owned(buf)
inner = own[ext:ext + N, ext:ext + N, ext:ext + N]
src = torch.rand((N, N, N), dtype=torch.float64, device=dev)
res = {}
for name in ("direct", "sample"):
    ts = []
    for rep in range(4):
        if name == "direct":
            inner.copy_(src)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if name == "direct":
            prefilter_device(inner, p)
            reflect_pad_device(own, ext)
        else:
            out = sample_solution_device(buf, grid, p, lay)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res[name + "_ms"] = round(min(ts[1:]), 3)
n3 = N ** 3
res.update(ncoef=ncoef, p=p, nodes=n3,
           direct_Gnodes_s=round(n3 / res["direct_ms"] / 1e6, 2),
           sample_Gnodes_s=round(n3 / res["sample_ms"] / 1e6, 2))
print(json.dumps(res))
