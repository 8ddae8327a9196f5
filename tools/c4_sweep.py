"""BASELINE configs[3] (c4): degree-robustness sweep, d = 2, 128 elements per
direction, p = 2..6 (p = 1 is rejected by the setup: C^1 spatial spaces),
sin-sin manufactured solution; lifted right-hand side, FD-preconditioned CG to
1e-8, L2 error -- all on the GPU. Prints one JSON line per degree."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_18461_b200 as ks  # noqa: E402

n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 128
for p in range(2, 7):
    t0 = time.perf_counter()
    prob = ks.SpaceTimeProblem.uniform(2, p, n_el, n_el)
    A, P = ks.assemble_system_operator(prob), ks.FDPreconditioner(prob)
    Q = ks.Quadrature(prob)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    rhs, bnd = Q.lift("sinsin", "sinsin")
    t_lift = time.perf_counter() - t0
    b = ks.DeviceVector.from_host(rhs)
    x = ks.DeviceVector(prob.N_dof)
    P.time(b, x, 3)  # warm-up (first launches load the kernels)
    ms_fd, _ = P.time(b, x, 20)
    A.apply(b, x)  # (the first matvec times the generated kernel candidates)
    rep0 = ks.pcg(A, P, b, ks.PcgOptions(1e-8, 200))  # (first solve: workspace allocation)
    rep = ks.pcg(A, P, b, ks.PcgOptions(1e-8, 200))
    t0 = time.perf_counter()
    for _ in range(20):
        A.apply(b, x)
    ks.lib().ks_synchronize()
    ms_mv = (time.perf_counter() - t0) / 20 * 1e3
    t0 = time.perf_counter()
    l2, en = Q.error_norms(Q.extend(rep.x, bnd), "sinsin", "sinsin")
    t_err = time.perf_counter() - t0
    print(json.dumps({"config": "c4", "p": p, "n_el": n_el, "dofs": prob.N_dof, "iterations": rep.iterations,
                      "converged": rep.converged, "solve_s": rep.solve_seconds, "first_solve_s": rep0.solve_seconds,
                      "fd_apply_ms": ms_fd, "matvec_ms": ms_mv, "plan": A.plan_info(),
                      "setup_s": t_setup, "rhs_lift_s": t_lift, "error_s": t_err, "l2_error": l2,
                      "energy_error": en, "fd_info": P.info()}), flush=True)
