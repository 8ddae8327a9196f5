"""Random problem shapes, GPU (default candidate selection, or KS_KRON_JIT / KS_FD_XFOLD from the
environment) against the oracle: system matvec and FD application. usage: fuzz_shapes.py [seed] [count]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import paper_2311_18461_b200 as ks  # noqa: E402
from oracle import oracle as O  # noqa: E402
from helpers import setup_arrays, rel, maxrel  # noqa: E402

O.build_oracle()
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
count = int(sys.argv[2]) if len(sys.argv) > 2 else 20
worst = 0.0
for it in range(count):
    d = int(rng.integers(2, 4))
    p = int(rng.integers(2, 7 if d == 2 else 5))
    cap = 600_000 if d == 3 else 1_500_000
    while True:
        n_el = int(rng.integers(4 * p + 2, 150 if d == 2 else 46))
        n_el_t = int(rng.integers(3, 60))
        if (n_el_t + p - 1) * (n_el + p - 2) ** d <= cap:
            break
    a = setup_arrays(ks, d, p, n_el, n_el_t)
    A = ks.assemble_system_operator(a["prob"])
    K = O.OracleKron(a["dims"], O.system_terms(a, d, a["nu"]))
    x = O.random_vec(K.N, 100 + it)
    yo = K.apply(x)
    e_mv = max(rel(A.apply(x), yo), maxrel(A.apply(x), yo))
    g = ks.FDPreconditioner.from_arrays(a["dims"], a["nu"], a["p"], a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"])
    o = O.OracleFD(a["dims"], a["nu"], a["p"], a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"])
    zo = o.apply(x)
    e_fd = max(rel(g.apply(x), zo), maxrel(g.apply(x), zo))
    worst = max(worst, e_mv, e_fd)
    print(f"d={d} p={p} n_el={n_el} n_el_t={n_el_t} dims={list(a['dims'])} matvec {e_mv:.2e} fd {e_fd:.2e} "
          f"{A.plan_info()['engine']} {g.info()['time_major_axis']}{'f' if g.info()['fused_axis1'] else ''}", flush=True)
    assert e_mv <= 1e-10 and e_fd <= 1e-10, "parity"
print("worst", worst)
