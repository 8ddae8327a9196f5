"""Right-hand side assembly, lifting, extension and error norms on the device
(paper_2311_18461_b200.Quadrature) against the reference's
own outputs (tests/golden/rhs_*.npz: assemble_rhs, lift_nonhomogeneous,
extend_with_boundary, error_norms; assembly.cpp:390-404,468-490,514-570,
experiments.cpp:73-153). Quadrature sums run in a different order than the
reference's serial loops, so agreement is to rounding (1e-10 relative)."""
import glob
import os

import numpy as np
import pytest

from golden_io import GOLDEN
from helpers import rel

pytestmark = pytest.mark.gpu

RHS = sorted(glob.glob(os.path.join(GOLDEN, "rhs_*.npz")))


@pytest.mark.parametrize("path", RHS, ids=[os.path.basename(p)[:-4] for p in RHS])
def test_rhs_lift_error_vs_reference(gpu, path):
    from paper_2311_18461_b200.problems import by_name
    g = np.load(path)
    d, p, n_el, name = int(g["d"]), int(g["p"]), int(g["n_el"]), str(g["name"])
    prob = gpu.SpaceTimeProblem.uniform(d, p, n_el, n_el)
    Q = gpu.Quadrature(prob)
    u, f = by_name(name, d)
    assert rel(Q.assemble_rhs(f), g["rhs_f"]) <= 1e-10
    rhs, bnd = Q.lift(u, f)
    assert rel(bnd, g["boundary"]) <= 1e-10
    assert rel(rhs, g["rhs"]) <= 1e-10
    full = Q.extend(g["x"], g["boundary"])
    assert rel(full, g["full"]) <= 1e-14
    l2, en = Q.error_norms(g["full"], u, f)
    assert abs(l2 - float(g["l2"])) <= 1e-10 * float(g["l2"])
    assert abs(en - float(g["energy"])) <= 1e-10 * float(g["energy"])


def test_c2_manufactured_solve_converges(gpu):
    """c2-shaped workload (d=2, p=3, sin-sin solution): lift, solve on the GPU,
    extend, error norm -- the L2 error falls with refinement."""
    from paper_2311_18461_b200.problems import sinsin
    u, f = sinsin(2)
    errs = []
    for n_el in (8, 16):
        prob = gpu.SpaceTimeProblem.uniform(2, 3, n_el, n_el)
        Q = gpu.Quadrature(prob)
        rhs, bnd = Q.lift(u, f)
        A, P = gpu.assemble_system_operator(prob), gpu.FDPreconditioner(prob)
        s = gpu.pcg(A, P, rhs, gpu.PcgOptions(1e-10, 200))
        assert s.converged
        errs.append(Q.error_norms(Q.extend(s.x, bnd), u, f)[0])
    assert errs[1] < errs[0] / 4


@pytest.mark.parametrize("path", RHS, ids=[os.path.basename(p)[:-4] for p in RHS])
def test_device_sampled_named_solutions(gpu, path):
    """Same pipeline with the built-in device samplers (ks_quad_sample_named)."""
    g = np.load(path)
    d, p, n_el, name = int(g["d"]), int(g["p"]), int(g["n_el"]), str(g["name"])
    Q = gpu.Quadrature(gpu.SpaceTimeProblem.uniform(d, p, n_el, n_el))
    assert rel(Q.assemble_rhs(name), g["rhs_f"]) <= 1e-10
    rhs, bnd = Q.lift(name, name)
    assert rel(rhs, g["rhs"]) <= 1e-10 and rel(bnd, g["boundary"]) <= 1e-10
    l2, en = Q.error_norms(g["full"], name, name)
    assert abs(l2 - float(g["l2"])) <= 1e-10 * float(g["l2"])
    assert abs(en - float(g["energy"])) <= 1e-10 * float(g["energy"])
