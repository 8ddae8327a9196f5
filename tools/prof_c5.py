"""ncu driver for c5 (d=3, p=4, n_el=128): two FD applications and one matvec."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2311_18461_b200 as ks  # noqa: E402

prob = ks.SpaceTimeProblem.uniform(3, 4, 128, 128)
P = ks.FDPreconditioner(prob)
A = ks.assemble_system_operator(prob)
n = prob.N_dof
r = ks.DeviceVector.from_host(np.ones(n, complex))
z = ks.DeviceVector(n)
for _ in range(2):
    P.apply(r, z)
A.apply(r, z)
A.apply(r, z)
ks.lib().ks_synchronize()
print("ok", n)
