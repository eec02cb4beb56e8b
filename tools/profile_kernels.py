"""Run a few CG iterations (step-wise) of the heat system for ncu captures.

    python tools/profile_kernels.py [ncoef] [iters]
Kernels: sep_kernel<3,3> (CG pass A), cg_pass_b_kernel, sep_kernel<3,1> (RHS).
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_03057_b200 import make_operator
from paper_1904_03057_b200.domain import Grid
from paper_1904_03057_b200.solver import _work
from paper_1904_03057_b200.synthetic import IC, SOURCE, gaussian_coeffs, heat_c_inputs
from paper_1904_03057_b200.system import heat_system

ncoef = int(sys.argv[1]) if len(sys.argv) > 1 else 512
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = int(os.environ.get("BSPDE_P", "3"))
N, h, dt = heat_c_inputs(ncoef, p)
op = make_operator(heat_system(Grid((N,) * 3, (h,) * 3), p, dt), "b200")
lay, dev = op.layout, op.device
u = lay.alloc(dev); q = lay.alloc(dev); F = lay.alloc(dev); b = lay.alloc(dev)
gaussian_coeffs(N, h, p, device=dev, out=u, layout=lay, **IC)
gaussian_coeffs(N, h, p, device=dev, out=q, layout=lay, **SOURCE)
op.mass_apply_device(q, F)
op.mass_apply_device(u, b, F, a=dt)
plan = op.plan()
w = _work(op, 10)
PP, K = w.pring, [0]
RR = PP.shape[0]
plan.cg_setup(w.scratch, None, 1e-300, 10 ** 6, False, True)
plan.cg_residual(b, u, w.r, w.scratch, 1)
for _ in range(iters):
    plan.cg_pass_a(u, w.r, PP[(K[0] - 1) % RR], PP[K[0] % RR], w.ap, w.scratch, 1)
    plan.cg_pass_b(w.r, w.ap, w.scratch, 1); K[0] += 1
torch.cuda.synchronize()
rep, active = plan.cg_read(w.scratch)
print("ok", ncoef, "p", p, "iters", rep.iterations, "relres", rep.relative_residual)
