import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import bspde_oracle as O
from paper_1904_03057_b200 import Grid, HeatProblem, HeatSolver, SolveConfig
h = np.load("tests/golden/heat64.npz")
inp = O.heat_inputs(64)
N, hh, dt = inp["N"], inp["h"], inp["dt"]
for lib in sys.argv[1:] or ["product"]:
    prob = HeatProblem(Grid((N,) * 3, (hh,) * 3), 3, dt, initial_coeffs=inp["u0"], source_coeffs=inp["q"])
    hs = HeatSolver(prob, SolveConfig(tol=1e-10, max_iter=5000, record_history=True))
    its = []
    for s in range(10):
        r = hs.step(); its.append(r.iterations)
    print(os.environ.get("BSPDE_LIB", "product"), its, list(h["iters_tol1e-10"]), flush=True)
    refu = h["u_final_tol1e-10"]
    print("u rel", np.linalg.norm(hs.coefficients() - refu) / np.linalg.norm(refu))
    print("last history tail", [f"{v:.3e}" for v in r.history[-8:]])
