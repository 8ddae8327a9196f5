"""Repeat the c3 PCG solve (device-resident) and print the time distribution."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2311_18461_b200 as ks  # noqa: E402

prob = ks.SpaceTimeProblem.uniform(3, 2, 64, 64)
A, P = ks.assemble_system_operator(prob), ks.FDPreconditioner(prob)
g = np.random.default_rng(1234)
b = ks.DeviceVector.from_host(g.uniform(-1, 1, prob.N_dof) + 1j * g.uniform(-1, 1, prob.N_dof))
ts = []
for k in range(int(os.environ.get("SOLVE_N", "8"))):
    t0 = time.perf_counter()
    rep = ks.pcg(A, P, b, ks.PcgOptions(1e-8, 200))
    ts.append((time.perf_counter() - t0, rep.solve_seconds, rep.iterations))
for t in ts:
    print("wall %.4f s  solve_seconds %.4f s  iters %d" % t)
