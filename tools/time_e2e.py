"""A/B the e2e stepping loops at ncoef^3: sequential copies vs run_steps_host."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_03057_b200 import make_operator
from paper_1904_03057_b200.domain import Grid
from paper_1904_03057_b200.heat import HeatSolver, run_steps_host
from paper_1904_03057_b200.solver import SolveConfig
from paper_1904_03057_b200.synthetic import IC, SOURCE, gaussian_coeffs, heat_c_inputs
from paper_1904_03057_b200.system import heat_system
n = int(sys.argv[1]) if len(sys.argv) > 1 else 930
N, h, dt = heat_c_inputs(n, 3)
op = make_operator(heat_system(Grid((N,) * 3, (h,) * 3), 3, dt), "b200")
lay, dev = op.layout, op.device
u = lay.alloc(dev); q = lay.alloc(dev); F = lay.alloc(dev)
gaussian_coeffs(N, h, 3, device=dev, out=u, layout=lay, **IC)
gaussian_coeffs(N, h, 3, device=dev, out=q, layout=lay, **SOURCE)
op.mass_apply_device(q, F)
hs = HeatSolver.from_device(op, dt, u, F, SolveConfig(tol=1e-10, max_iter=5000, poll_every=16))
host = torch.empty(lay.owned_shape, dtype=torch.float64).pin_memory()
host.copy_(lay.owned(u).cpu())
own = lay.owned(u)
hs.step(); torch.cuda.synchronize()
for mode in ("seq", "pipe1", "pipe16", "seq", "pipe16"):
    torch.cuda.synchronize(); t = time.perf_counter()
    if mode == "seq":
        its = 0
        for _ in range(3):
            own.copy_(host, non_blocking=True); its += hs.step().iterations; host.copy_(own, non_blocking=True)
    else:
        reps = run_steps_host(hs.step, own, host, 3, chunks=int(mode[4:]))
        its = sum(r.iterations for r in reps)
    torch.cuda.synchronize(); dtm = time.perf_counter() - t
    print(mode, f"{dtm:.3f} s for 3 steps, {its} its -> {its * n**3 / dtm / 1e9:.1f} GDoF/s", flush=True)
