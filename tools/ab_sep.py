"""A/B a sep_kernel variant (BSPDE_LIB) on the bench's heat system: times
pass A, pass B, the residual and the RHS kernels (CUDA events, median of 15
after 3 warm-ups) and prints sha256 digests of every output plus the CG
scalars, so two builds can be checked bitwise-identical.

    BSPDE_LIB=path python tools/ab_sep.py [ncoef] [degree]
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_03057_b200 import make_operator  # noqa: E402
from paper_1904_03057_b200.domain import Grid  # noqa: E402
from paper_1904_03057_b200.solver import _work  # noqa: E402
from paper_1904_03057_b200.synthetic import IC, SOURCE, gaussian_coeffs, heat_c_inputs  # noqa: E402
from paper_1904_03057_b200.system import heat_system  # noqa: E402

ncoef = int(sys.argv[1]) if len(sys.argv) > 1 else 512
p = int(sys.argv[2]) if len(sys.argv) > 2 else 3
N, h, dt = heat_c_inputs(ncoef, p)
op = make_operator(heat_system(Grid((N,) * 3, (h,) * 3), p, dt), "b200")
lay, dev = op.layout, op.device
w = _work(op, 10)
u, F = lay.alloc(dev), lay.alloc(dev)
gaussian_coeffs(N, h, p, device=dev, out=u, layout=lay, **IC)
gaussian_coeffs(N, h, p, device=dev, out=w.r, layout=lay, **SOURCE)
op.mass_apply_device(w.r, F)
plan = op.plan()
R = w.pring.shape[0]


def digest(t):
    return hashlib.sha256(t.contiguous().cpu().numpy().tobytes()).hexdigest()[:16]


def ev():
    return torch.cuda.Event(enable_timing=True)


times = {"rhs": [], "resid": [], "pass_a": [], "pass_b": [], "hres": [], "flush": []}
dig = {}
x = u.clone()
# RHS and residual kernels (each residual restarts the CG state at k = 0)
for it in range(10):
    e = [ev() for _ in range(3)]
    e[0].record()
    op.mass_apply_device(u, w.ap, F, a=dt)           # b (in Ap's storage)
    e[1].record()
    plan.cg_setup(w.scratch, None, 1e-300, 10 ** 6, False, True, p_ring=R)
    plan.cg_residual(w.ap, x, w.r, w.scratch, 1)
    e[2].record()
    torch.cuda.synchronize()
    if it == 0:
        dig["b"] = digest(lay.owned(w.ap))
        dig["r0"] = digest(lay.owned(w.r))
        dig["resid_sums"] = digest(w.scratch[:64])
    if it >= 3:
        times["rhs"].append(e[0].elapsed_time(e[1]))
        times["resid"].append(e[1].elapsed_time(e[2]))
# CG iterations k = 0 .. 17 from that residual: pass A of k >= 1 applies the
# x update of iteration k - 1 (the timed passes are k >= 3)
for k in range(18):
    e = [ev() for _ in range(3)]
    e[0].record()
    plan.cg_pass_a(x, w.r, w.pring[(k - 1) % R], w.pring[k % R], w.ap, w.scratch, 1)
    e[1].record()
    plan.cg_pass_b(w.r, w.ap, w.scratch, 1)
    e[2].record()
    torch.cuda.synchronize()
    if k == 0:
        dig["ap"] = digest(lay.owned(w.ap))
        dig["p0"] = digest(lay.owned(w.pring[0]))
        dig["after_b_state"] = digest(w.scratch[:256])
    if k >= 3:
        times["pass_a"].append(e[0].elapsed_time(e[1]))
        times["pass_b"].append(e[1].elapsed_time(e[2]))
plan.cg_flush_x(x, w.pring, w.scratch)
dig["x_final"] = digest(lay.owned(x))
dig["r_final"] = digest(lay.owned(w.r))
# fused heat residual (RHS + residual in one kernel) and the end-of-solve flush
for it in range(8):
    e = [ev() for _ in range(3)]
    plan.cg_setup(w.scratch, None, 1e-300, 10 ** 6, False, True, p_ring=R)
    e[0].record()
    plan.heat_residual(x, F, op.data.vol, dt, w.r, w.scratch, 1)
    e[1].record()
    plan.cg_pass_a(x, w.r, w.pring[R - 1], w.pring[0], w.ap, w.scratch, 1)
    plan.cg_pass_b(w.r, w.ap, w.scratch, 1)
    e2 = ev()
    e2.record()
    plan.cg_flush_x(x, w.pring, w.scratch)
    e[2].record()
    torch.cuda.synchronize()
    if it >= 2:
        times["hres"].append(e[0].elapsed_time(e[1]))
        times["flush"].append(e2.elapsed_time(e[2]))
out = {"lib": os.path.basename(os.environ.get("BSPDE_LIB", "product")), "ncoef": ncoef, "p": p,
       **{k + "_ms": round(float(np.median(v)), 4) for k, v in times.items()},
       "digests": dig}
print(json.dumps(out), flush=True)
