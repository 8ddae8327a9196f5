"""Galerkin fast solver (galerkin_fast_solver, fdsolver.cpp:177-191; SURVEY 8(f)
rank 3) and Galerkin operator (assemble_galerkin_operator, assembly.cpp:273-286):
same eigenbasis/transform/solve kernels with blocks H_i = W_t + nu lambda_i M_t,
which make the FD solver the exact inverse of the Galerkin matrix.
CPU: the C oracle is bit-identical to the reference's own outputs
(tests/golden/gal_*.npz, scalar backend). GPU: parity at the north_star
tolerance, forward and adjoint solves, and the exact-inverse property."""
import glob
import os

import numpy as np
import pytest

from golden_io import GOLDEN, load, ids
from helpers import rel, maxrel

GAL = sorted(glob.glob(os.path.join(GOLDEN, "gal_*.npz")))
TOL = 1e-10


def _bands(g):
    return dict(p=g["p"], dims=g["dims"], Lt=g["Lt"], Mt=g["Mt"], Wt=g["Wt"], M=g["M"], G=g["G"])


@pytest.mark.parametrize("path", GAL, ids=ids(GAL))
def test_oracle_galerkin_bitexact_vs_reference(oracle, path):
    g = load(path)
    F = oracle.OracleFD(g["dims"], 1.0, g["p"], g["U"], g["lam"], g["Lt"], g["Mt"], g["Wt"], kind="galerkin")
    assert np.array_equal(F.apply(g["r"]), g["z_gal"])
    assert np.array_equal(F.apply_adjoint(g["r"]), g["z_gal_adj"])
    K = oracle.OracleKron(g["dims"], oracle.galerkin_terms(_bands(g), g["d"], 1.0))
    assert np.array_equal(K.apply(g["r"]), g["y_gal"])
    # exact inverse: G (P_g r) = r
    assert np.linalg.norm(K.apply(g["z_gal"]) - g["r"]) <= 1e-12 * np.linalg.norm(g["r"])


@pytest.mark.gpu
@pytest.mark.parametrize("path", GAL, ids=ids(GAL))
def test_gpu_galerkin_vs_reference(gpu, oracle, path):
    g = load(path)
    P = gpu.FDPreconditioner.galerkin_from_arrays(g["dims"], 1.0, g["p"], g["U"], g["lam"], g["Mt"], g["Wt"])
    r = g["r"]
    z = P.apply(r)
    assert rel(z, g["z_gal"]) <= TOL and maxrel(z, g["z_gal"]) <= TOL
    za = P.apply_adjoint(r)
    assert rel(za, g["z_gal_adj"]) <= TOL and maxrel(za, g["z_gal_adj"]) <= TOL
    A = gpu.KroneckerOperator(g["dims"])
    for c, fs, bw in oracle.galerkin_terms(_bands(g), g["d"], 1.0):
        A.add_term(c, [gpu.Banded(g["dims"][k], bw[k], f) for k, f in enumerate(fs)])
    y = A.apply(r)
    assert rel(y, g["y_gal"]) <= TOL and maxrel(y, g["y_gal"]) <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("d,p,n_el", [(2, 3, 12), (3, 2, 10), (3, 3, 6)])
def test_gpu_galerkin_own_setup_exact_inverse(gpu, oracle, d, p, n_el):
    """libks's own host setup: the Galerkin solver inverts the Galerkin operator
    (folded transforms and pair-mode solves included where they apply)."""
    prob = gpu.SpaceTimeProblem.uniform(d, p, n_el, n_el)
    P = gpu.FDPreconditioner.galerkin(prob)
    G = gpu.assemble_galerkin_operator(prob)
    r = oracle.random_vec(prob.N_dof, 7)
    z = P.apply(r)
    assert np.linalg.norm(G.apply(z) - r) <= 1e-10 * np.linalg.norm(r)
    # adjoint: <P r, s> = <r, P^H s>
    s = oracle.random_vec(prob.N_dof, 8)
    assert abs(np.vdot(s, z) - np.vdot(P.apply_adjoint(s), r)) <= 1e-10 * abs(np.vdot(s, z))
