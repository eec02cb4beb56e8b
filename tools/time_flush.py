"""Time x_flush (deferred x update) at ncoef^3: one CG iteration then flush."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_03057_b200 import make_operator
from paper_1904_03057_b200.domain import Grid
from paper_1904_03057_b200.solver import _work
from paper_1904_03057_b200.synthetic import IC, heat_c_inputs, gaussian_coeffs
from paper_1904_03057_b200.system import heat_system
n = int(sys.argv[1]) if len(sys.argv) > 1 else 930
N, h, dt = heat_c_inputs(n, 3)
op = make_operator(heat_system(Grid((N,) * 3, (h,) * 3), 3, dt), "b200")
lay, dev = op.layout, op.device
u = lay.alloc(dev); b = lay.alloc(dev)
gaussian_coeffs(N, h, 3, device=dev, out=u, layout=lay, **IC)
op.mass_apply_device(u, b)
plan = op.plan(); w = _work(op, 10); PP, K = w.pring, [0]
RR = PP.shape[0]
PP, K = w.pring, [0]
RR = PP.shape[0]
ts = []
for rep in range(4):
    plan.cg_setup(w.scratch, None, 1e-300, 10 ** 6, False, True)
    plan.cg_residual(b, u, w.r, w.scratch, 1)
    plan.cg_pass_a(u, w.r, PP[(K[0] - 1) % RR], PP[K[0] % RR], w.ap, w.scratch, 1)
    plan.cg_pass_b(w.r, w.ap, w.scratch, 1); K[0] += 1
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); plan.cg_flush_x(u, w.pring, w.scratch); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("flush ms", [round(t, 3) for t in ts], "GB/s", round(24 * n ** 3 / min(ts) / 1e6, 1))
