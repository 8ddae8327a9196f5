"""ncu driver for c4 (d=2, 128 elements, degree argv[1], default 2): three FD applications and two matvecs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2311_18461_b200 as ks  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prob = ks.SpaceTimeProblem.uniform(2, p, 128, 128)
P = ks.FDPreconditioner(prob)
A = ks.assemble_system_operator(prob)
n = prob.N_dof
rng = np.random.default_rng(1)
r = ks.DeviceVector.from_host(rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n))
z = ks.DeviceVector(n)
for _ in range(3):
    P.apply(r, z)
for _ in range(3):
    A.apply(r, z)
ks.lib().ks_synchronize()
print("ok", n, P.info())
