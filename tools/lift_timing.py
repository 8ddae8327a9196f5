"""Time the c2 manufactured-solution pieces (rhs assembly, lift, error norms) on the device."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_18461_b200 as ks  # noqa: E402

p2 = ks.SpaceTimeProblem.uniform(2, 3, 64, 64)
Q2 = ks.Quadrature(p2)
for it in range(3):
    t0 = time.perf_counter()
    rhs = Q2.assemble_rhs("sinsin")
    t1 = time.perf_counter()
    r2, b2 = Q2.lift("sinsin", "sinsin")
    t2 = time.perf_counter()
    print(f"iter {it}: assemble_rhs {1e3 * (t1 - t0):.2f} ms, lift (incl. rhs) {1e3 * (t2 - t1):.2f} ms", flush=True)
