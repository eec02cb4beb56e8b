"""Time the variable-coefficient operator (assembled stencil) at n^3 nodes:
assembly, apply (CUDA events; HBM bytes = ((2p+1)^3 + 2) * 8 per DoF), and
50 Jacobi-PCG iterations.   python tools/time_varcoef.py [n ...] (p via BSPDE_P)"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1904_03057_b200 import BoxDomain, Grid, SolveConfig, build_system, make_operator, pcg
from paper_1904_03057_b200.gram import basis_extension

p = int(os.environ.get("BSPDE_P", "3"))
for n in [int(a) for a in sys.argv[1:]] or [64]:
    h = 1.0 / (n - 1)
    grid = Grid((n,) * 3, (h,) * 3)
    pe = n + 2 * basis_extension(p)
    z = np.linspace(0, 1, pe)
    D = 0.01 * (1.0 + 0.5 * np.sin(3 * z)[:, None, None] * np.cos(2 * z)[None, :, None]
                * (1 + z[None, None, :]))
    mu = 1.0 + 0.2 * np.cos(5 * z)[:, None, None] * np.ones((1, pe, pe))
    data = build_system(BoxDomain(grid), p, p, D, mu, [])
    torch.cuda.synchronize(); t0 = time.perf_counter()
    op = make_operator(data, "b200")
    torch.cuda.synchronize(); t_asm = time.perf_counter() - t0
    N = int(np.prod(data.cext))
    c = torch.rand(data.cext, dtype=torch.float64, device=op.device)
    out = torch.empty_like(c)
    op.apply_device(c, out); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        op.apply_device(c, out)
    e1.record(); torch.cuda.synchronize()
    t_apply = e0.elapsed_time(e1) / 10 / 1e3
    a3 = (2 * p + 1) ** 3
    rhs = out.cpu().numpy()
    pcg(op, rhs, SolveConfig(tol=1e-300, max_iter=2))  # first launches load the kernels
    t0 = time.perf_counter()
    x, rep = pcg(op, rhs, SolveConfig(tol=1e-300, max_iter=50))
    t_cg = time.perf_counter() - t0
    print(json.dumps({"n": n, "p": p, "dofs": N, "assemble_s": round(t_asm, 3),
                      "apply_ms": round(t_apply * 1e3, 3),
                      "apply_GBs": round((a3 + 2) * 8 * N / t_apply / 1e9, 1),
                      "cg_its": rep.iterations, "cg_GDoF_it_s": round(N * rep.iterations / t_cg / 1e9, 3),
                      "stencil_GB": round(a3 * 8 * N / 1e9, 2)}), flush=True)
    del op, c, out
    torch.cuda.empty_cache()
