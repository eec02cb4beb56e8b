"""C1 (64^3, p=3, lambda=4) CG counts of 10 heat steps vs the reference's
[45, 45, 47, 50, 63, 77, 91, 112, 120, 129]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import bspde_oracle as O
from paper_1904_03057_b200 import Grid, HeatProblem, HeatSolver, SolveConfig
inp = O.heat_inputs(64)
N, hh, dt = inp["N"], inp["h"], inp["dt"]
hs = HeatSolver(HeatProblem(Grid((N,) * 3, (hh,) * 3), 3, dt, initial_coeffs=inp["u0"],
                            source_coeffs=inp["q"]), SolveConfig(tol=1e-10, max_iter=5000))
print("gpu      ", [hs.step().iterations for _ in range(10)])
print("reference [45, 45, 47, 50, 63, 77, 91, 112, 120, 129]")
