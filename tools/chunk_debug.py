"""Per-plane apply error with forced z-chunk counts (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import bspde_oracle as O
from paper_1904_03057_b200 import BoxDomain, Grid, build_system, make_operator
p = int(sys.argv[1]); ext = tuple(int(v) for v in sys.argv[2].split(","))
step = (0.5, 1.0, 0.25)
data = build_system(BoxDomain(Grid(ext, step)), p, p, 0.37, 1.3, [])
ora = O.KronOperator(ext, step, p, 0.37, 1.3)
c = np.random.default_rng(0).normal(size=data.cext)
want = ora.apply(c)
op = make_operator(data, "b200")
t = op.apply(c)
err = np.abs(t - want).max(axis=(1, 2)) / np.abs(want).max()
print("chunks", os.environ.get("BSPDE_FORCE_CHUNKS"), "per-plane err", np.array2string(err, precision=1))
