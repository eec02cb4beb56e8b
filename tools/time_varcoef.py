"""Time the variable-coefficient operator at the given node grids: setup,
apply (CUDA events), 50 Jacobi-PCG iterations (device time, pcg_device),
for the matrix-free kernel (BSPDE_VAR_STRATEGY=otf, default when supported)
or the assembled stencil (=stencil).

    python tools/time_varcoef.py [NZxNYxNX | N ...]      (p via BSPDE_P, default 3)

The paper's variable-coefficient grids are 240x240x960 and 522^3 (p = 3).
Prints one JSON line per grid: apply ms / GDoF/s, FP64 GFLOP/s of the
matrix-free apply (flop_byte_report), PCG GDoF-it/s.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_03057_b200 import BoxDomain, Grid, SolveConfig, build_system, make_operator  # noqa: E402
from paper_1904_03057_b200.gram import basis_extension  # noqa: E402

p = int(os.environ.get("BSPDE_P", "3"))
for arg in sys.argv[1:] or ["64"]:
    ext = tuple(int(v) for v in arg.split("x")) if "x" in arg else (int(arg),) * 3
    step = tuple(1.0 / (n - 1) for n in ext)
    grid = Grid(ext, step)
    pe = [n + 2 * basis_extension(p) for n in ext]
    z, y, x = (np.linspace(0, 1, n) for n in pe)
    # smooth positive fields (separable products: no 3-D host temporaries)
    D = 0.01 * (1.0 + 0.5 * np.sin(3 * z)[:, None, None] * np.cos(2 * y)[None, :, None]
                * (1 + x[None, None, :]))
    mu = 1.0 + 0.2 * np.cos(5 * z)[:, None, None] * np.ones((1, pe[1], pe[2]))
    data = build_system(BoxDomain(grid), p, p, D, np.ascontiguousarray(mu), [])
    del D, mu
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = make_operator(data, "b200")
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    N = int(np.prod(data.cext))
    c = torch.rand(data.cext, dtype=torch.float64, device=op.device)
    out = torch.empty_like(c)
    op.apply_device(c, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        op.apply_device(c, out)
    e1.record()
    torch.cuda.synchronize()
    t_apply = e0.elapsed_time(e1) / 5 / 1e3
    st = op.flop_byte_report(t_apply)
    b = out.clone()
    x0 = torch.zeros_like(b)
    op.pcg_device(b, x0, SolveConfig(tol=1e-300, max_iter=2), has_x0=False)  # warm
    torch.cuda.synchronize()
    e0.record()
    rep = op.pcg_device(b, x0, SolveConfig(tol=1e-300, max_iter=50, poll_every=50), has_x0=False)
    e1.record()
    torch.cuda.synchronize()
    t_cg = e0.elapsed_time(e1) / 1e3
    print(json.dumps({"grid": list(ext), "p": p, "kind": op.kind, "dofs": N,
                      "setup_s": round(t_setup, 3), "apply_ms": round(t_apply * 1e3, 3),
                      "apply_GDoF_s": round(N / t_apply / 1e9, 3),
                      "apply_GFLOP_s": round(st.gflops, 1),
                      "cg_its": rep.iterations,
                      "cg_GDoF_it_s": round(N * rep.iterations / t_cg / 1e9, 3),
                      "mem_GB": round(torch.cuda.max_memory_allocated() / 1e9, 2)}), flush=True)
    del op, c, out, b, x0
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
