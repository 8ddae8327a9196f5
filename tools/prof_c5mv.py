"""ncu driver for the c5 (d=3, p=4, n_el=128) system matvec only: the first apply
times the candidates, then three more applies. argv[1] = a smaller n_el (optional)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2311_18461_b200 as ks  # noqa: E402

n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 128
prob = ks.SpaceTimeProblem.uniform(3, 4, n_el, n_el)
A = ks.assemble_system_operator(prob)
n = prob.N_dof
rng = np.random.default_rng(1)
r = ks.DeviceVector.from_host(rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n))
z = ks.DeviceVector(n)
for _ in range(4):
    A.apply(r, z)
ks.lib().ks_synchronize()
print("ok", n)
