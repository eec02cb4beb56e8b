"""Cost of splitting CG pass A around the halo exchange, on one GPU.

Emulates rank `rank` of a `world`-way z-slab partition of the C3 workload
(930^3, p = 3 by default) and times, with CUDA events on the launching
stream, (a) the whole-slab pass A and (b) the overlapped driver's three
ranged launches (interior [p, nz-p), then [0, p) and [nz-p, nz)).  The
difference is what the overlap costs in compute; the halo it hides is
4 x p x ny x nx x 8 B per iteration (measured separately on NVLink).

    python tools/time_slab_split.py [ncoef] [world] [rank] [p]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_03057_b200 import Grid, heat_system  # noqa: E402
from paper_1904_03057_b200.device import NativePlan, SlabLayout  # noqa: E402
from paper_1904_03057_b200.distributed import SlabPartition  # noqa: E402
from paper_1904_03057_b200.gram import basis_extension  # noqa: E402

ncoef = int(sys.argv[1]) if len(sys.argv) > 1 else 930
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rank = int(sys.argv[3]) if len(sys.argv) > 3 else 3
p = int(sys.argv[4]) if len(sys.argv) > 4 else 3
n = ncoef - 2 * basis_extension(p)
h = 1.0 / (n - 1)
data = heat_system(Grid((n,) * 3, (h,) * 3), p, 4.0 * h * h)
nzg, ny, nx = data.dims3
part = SlabPartition(nzg, world, rank)
lay = SlabLayout(part.nz, ny, nx, ghost=p, z_offset=part.z_offset, nz_global=nzg)
dev = torch.device("cuda:0")
plan = NativePlan(data, lay, dev)
r, q, o, ap, xx = (lay.alloc(dev) for _ in range(5))
r.normal_()
q.normal_()
scratch = plan.scratch()
plan.cg_setup(scratch, None, 1e-300, 100, False, False)
scratch[80:88].view(torch.float64)[0] = 0.5   # CgState.beta
scratch[152:156].view(torch.int32)[0] = 1     # CgState.active
nz = lay.nz


def whole():
    plan.cg_pass_a(xx, r, q, o, ap, scratch, 0)


def split():
    plan.cg_pass_a_range(xx, r, q, o, ap, scratch, p, nz - 2 * p, False)
    plan.cg_pass_a_range(xx, r, q, o, ap, scratch, 0, p, True)
    plan.cg_pass_a_range(xx, r, q, o, ap, scratch, nz - p, p, True)


def interior():
    plan.cg_pass_a_range(xx, r, q, o, ap, scratch, p, nz - 2 * p, False)


def boundary():
    plan.cg_pass_a_range(xx, r, q, o, ap, scratch, 0, p, True)
    plan.cg_pass_a_range(xx, r, q, o, ap, scratch, nz - p, p, True)


res = {"ncoef": ncoef, "p": p, "world": world, "rank": rank, "slab_planes": nz,
       "halo_bytes_per_iteration": 2 * 2 * p * ny * nx * 8 * (2 if 0 < rank < world - 1 else 1)}
for name, fn in [("whole", whole), ("split", split), ("interior", interior),
                 ("boundary", boundary)]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    res[name + "_ms"] = round(e0.elapsed_time(e1) / reps, 4)
print(json.dumps(res))
