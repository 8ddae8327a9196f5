"""c3-size matvec through the JIT path: finite check, and vs the per-pass kernels."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2311_18461_b200 as ks
ne = int(sys.argv[1]) if len(sys.argv) > 1 else 64
prob = ks.SpaceTimeProblem.uniform(3, 2, ne, ne)
A = ks.assemble_system_operator(prob)
g = np.random.default_rng(1)
n = prob.N_dof
x = g.uniform(-1, 1, n) + 1j * g.uniform(-1, 1, n)
y = A.apply(x)
print(ne, "finite", bool(np.isfinite(y).all()), float(np.abs(y).max()), flush=True)
