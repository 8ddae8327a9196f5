"""ncu driver for c2 (d=2, p=3, n_el=64): one PCG solve to 1e-8 (after a warm-up solve)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2311_18461_b200 as ks  # noqa: E402

prob = ks.SpaceTimeProblem.uniform(2, 3, 64, 64)
P, A = ks.FDPreconditioner(prob), ks.assemble_system_operator(prob)
g = np.random.default_rng(1234)
b = ks.DeviceVector.from_host(g.uniform(-1, 1, prob.N_dof) + 1j * g.uniform(-1, 1, prob.N_dof))
ks.pcg(A, P, b)
ks.lib().ks_synchronize()
if os.environ.get("KS_PROF_MARK"):
    print("warm")
rep = ks.pcg(A, P, b)
print("iters", rep.iterations, "seconds", rep.solve_seconds)
