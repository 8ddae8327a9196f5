"""Small driver for ncu captures: config c3 (d=3, p=2, n_el=64), a few FD
applications and system matvecs on device-resident vectors."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_18461_b200 as ks  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
d, p, n_el = {"c3": (3, 2, 64), "c2": (2, 3, 64), "c5s": (3, 4, 64)}[cfg]
prob = ks.SpaceTimeProblem.uniform(d, p, n_el, n_el)
P = ks.FDPreconditioner(prob)
A = ks.assemble_system_operator(prob)
n = prob.N_dof
g = np.random.default_rng(1)
r = ks.DeviceVector.from_host(g.uniform(-1, 1, n) + 1j * g.uniform(-1, 1, n))
z = ks.DeviceVector(n)
for _ in range(3):
    P.apply(r, z)
for _ in range(2):
    A.apply(r, z)
ks.lib().ks_synchronize()
print("ok", n)
