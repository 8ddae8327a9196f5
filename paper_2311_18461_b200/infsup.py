"""Discrete inf-sup constants: Lanczos on the B-inner
product (lanczos_extreme_eigenvalue, krylov.cpp:116-179) driven by the GPU
operators -- system matrix, space-time mass, FD and Galerkin fast solvers --
as infsup_constant does (experiments.cpp:185-232).

The Krylov vectors live on the host (the problems are 1-D, n <= a few
thousand); every operator application is a libks call. The start vector is
drawn from numpy's normal generator instead of the reference's
std::normal_distribution, so the two agree once the Krylov space is
exhausted or the extreme Ritz value has converged (full reorthogonalisation,
as in the reference).
"""
import numpy as np

from . import (Banded, FDPreconditioner, KroneckerOperator, PcgOptions, SpaceTimeProblem,
               assemble_system_operator, pcg)


def lanczos_extreme_eigenvalue(apply_t, apply_b, n, steps, largest=True, seed=1234):
    """Extreme eigenvalue of the pencil (T, B) by B-orthonormal Lanczos with full
    reorthogonalisation (krylov.cpp:116-179)."""
    steps = min(int(steps), int(n))
    if steps < 1:
        raise ValueError("lanczos_extreme_eigenvalue: steps < 1")
    g = np.random.default_rng(seed)
    v = g.standard_normal(n) + 1j * g.standard_normal(n)
    bv = apply_b(v)
    nrm = np.sqrt(np.vdot(v, bv).real)
    if not nrm > 0:
        raise RuntimeError("lanczos_extreme_eigenvalue: B not positive")
    V, BV = [v / nrm], [bv / nrm]
    alpha, beta = [], []
    for j in range(steps):
        t = apply_t(V[j])
        alpha.append(np.vdot(BV[j], t).real)
        w = t.copy()
        for i in range(len(V)):  # full reorthogonalisation in the B inner product
            w -= np.vdot(BV[i], w) * V[i]
        bw = apply_b(w)
        b2 = np.vdot(w, bw).real
        if not b2 > 1e-28:
            break  # invariant subspace
        b = np.sqrt(b2)
        beta.append(b)
        if j + 1 < steps:
            V.append(w / b)
            BV.append(bw / b)
    m = len(alpha)
    T = np.diag(alpha) + np.diag(beta[:m - 1], 1) + np.diag(beta[:m - 1], -1)
    ev = np.linalg.eigvalsh(T)
    return float(ev.max() if largest else ev.min())


def spacetime_mass(prob: SpaceTimeProblem, device: int = 0) -> KroneckerOperator:
    """assemble_spacetime_mass (assembly.cpp:265-271): M_t x M_1 x ... x M_d."""
    dims = prob.reduced_dims()
    p = prob.p
    _, Mt, _ = prob.time_bands()
    facs = [Banded(dims[0], p, np.asarray(Mt, dtype=np.complex128))]
    for l in range(prob.d):
        M = prob.space_bands(l)[0]
        facs.append(Banded(dims[l + 1], p, np.asarray(M, dtype=np.complex128)))
    op = KroneckerOperator(dims, device=device)
    op.add_term(1.0, facs)
    return op


def infsup_constant(method: str, p: int, n_el: int, T: float = 1.0, nu: float = 1.0, device: int = 0) -> float:
    """infsup_constant (experiments.cpp:185-232) on the GPU operators.
    method "ls": alpha^2 = 1 / (1 + lambda_max(MQ, A)) with A^-1 by FD-PCG (tol 1e-12);
    method "galerkin": alpha^2 = 1 / lambda_max(Ag^-1 MQ Ag^-H (MQ + A))."""
    prob = SpaceTimeProblem.matched(1, p, n_el, T, nu)
    A = assemble_system_operator(prob, device=device)
    MQ = spacetime_mass(prob, device=device)
    n = prob.N_dof
    steps = min(n, 60)
    if method in ("ls", "least_squares"):
        P = FDPreconditioner(prob, device=device)

        def apply_t(x):
            b = MQ.apply(x)
            return np.asarray(pcg(A, P, b, PcgOptions(1e-12, 400)).x)
        lmax = lanczos_extreme_eigenvalue(apply_t, MQ.apply, n, steps, True)
        return float(1.0 / np.sqrt(1.0 + lmax))
    if method == "galerkin":
        G = FDPreconditioner.galerkin(prob, device=device)

        def apply_gv(x):
            return MQ.apply(x) + A.apply(x)

        def apply_t(x):
            return G.apply(MQ.apply(G.apply_adjoint(apply_gv(x))))
        lmax = lanczos_extreme_eigenvalue(apply_t, apply_gv, n, steps, True)
        return float(1.0 / np.sqrt(lmax))
    raise ValueError("infsup_constant: method must be 'ls' or 'galerkin'")
