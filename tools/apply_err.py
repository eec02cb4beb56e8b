"""Locate apply errors vs the oracle (z planes / y rows / x cols with error)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import bspde_oracle as O
from paper_1904_03057_b200 import BoxDomain, Grid, build_system, make_operator
p = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ext = tuple(int(a) for a in sys.argv[2:5]) if len(sys.argv) > 4 else (20, 19, 18)
step = tuple(1.0 / (n - 1) for n in ext)
data = build_system(BoxDomain(Grid(ext, step)), p, p, 0.01, 1.0, [])
ora = O.KronOperator(ext, step, p, 0.01, 1.0)
c = np.random.default_rng(0).normal(size=data.cext)
t = make_operator(data, "b200").apply(c)
ref = ora.apply(c)
err = np.abs(t - ref) / np.abs(ref).max()
print("lib", os.environ.get("BSPDE_LIB", "product"), "p", p, "cext", data.cext, "max rel err", err.max())
if err.max() > 1e-12:
    bad = np.argwhere(err > 1e-12)
    for ax in range(3):
        print(" axis", ax, "bad idx", sorted(set(bad[:, ax].tolist()))[:40])
