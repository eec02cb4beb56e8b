"""Time CG pass A (sep_kernel<P,CGA>) and pass B separately, step-wise.

    python tools/time_passes.py [ncoef ...]        (BSPDE_P=degree, BSPDE_LIB=variant)
Prints one JSON line per size: median ms per launch over 20 iterations after
3 warm-up iterations, CUDA events on the launching stream.  Inputs are the
bench's Gaussian heat system (> L2 at the sizes of interest).
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_03057_b200 import make_operator
from paper_1904_03057_b200.domain import Grid
from paper_1904_03057_b200.solver import _work
from paper_1904_03057_b200.synthetic import IC, SOURCE, gaussian_coeffs, heat_c_inputs
from paper_1904_03057_b200.system import heat_system

p = int(os.environ.get("BSPDE_P", "3"))
for ncoef in [int(a) for a in sys.argv[1:]] or [512]:
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
    ta, tb = [], []
    for it in range(23):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        plan.cg_pass_a(u, w.r, PP[(K[0] - 1) % RR], PP[K[0] % RR], w.ap, w.scratch, 1)
        e[1].record()
        plan.cg_pass_b(w.r, w.ap, w.scratch, 1); K[0] += 1
        e[2].record()
        torch.cuda.synchronize()
        if it >= 3:
            ta.append(e[0].elapsed_time(e[1]))
            tb.append(e[1].elapsed_time(e[2]))
    n = ncoef ** 3
    ta.sort(); tb.sort()
    a, bb = ta[len(ta) // 2], tb[len(tb) // 2]
    print(json.dumps({"lib": os.path.basename(os.environ.get("BSPDE_LIB", "product")),
                      "p": p, "ncoef": ncoef, "passA_ms": round(a, 4), "passB_ms": round(bb, 4),
                      "passA_GBs": round(48 * n / a / 1e6, 1), "passB_GBs": round(24 * n / bb / 1e6, 1),
                      "iter_ms": round(a + bb, 4)}), flush=True)
    del op, u, q, F, b, w, plan
    torch.cuda.empty_cache()
