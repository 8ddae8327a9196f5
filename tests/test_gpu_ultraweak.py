"""Ultraweak variant (assemble_ultraweak, assembly.cpp:572-640):
final-condition trial space, load vector of f plus the initial-datum term
i (u0, B_jt(0) phi_js). Device result vs the reference's own assemble_ultraweak
run live (oracle/_ref) on the same manufactured solution."""
import numpy as np
import pytest

from helpers import rel, maxrel

pytestmark = pytest.mark.gpu

PI = np.pi


def _sinsin(d):
    def u0(*x):
        v = 1.0
        for xi in x:
            v = v * np.sin(PI * xi)
        return v + 0j

    def f(t, *x):  # S u = i u_t - nu lap u = (1 + nu) d pi^2 u (nu = 1)
        return 2.0 * d * PI ** 2 * u0(*x) * np.exp(-1j * d * PI ** 2 * t)
    return f, u0


@pytest.mark.parametrize("d,p,n_el,n_el_t", [(1, 3, 8, 6), (2, 3, 6, 5), (2, 2, 9, 4), (3, 2, 4, 3)])
def test_ultraweak_rhs_vs_reference(gpu, d, p, n_el, n_el_t):
    from oracle import refdrv
    if not refdrv.available():
        pytest.fail("oracle/_ref not built")
    prob = gpu.SpaceTimeProblem.uniform(d, p, n_el, n_el_t, trial="final")
    Q = gpu.Quadrature(prob)
    f, u0 = _sinsin(d)
    A, rhs = Q.ultraweak(f, u0)
    ref = refdrv.RefProblem(d, p, n_el, n_el_t, trial=1).ultraweak_named("sinsin")
    assert rel(rhs, ref) <= 1e-10 and maxrel(rhs, ref) <= 1e-10
    # the initial-datum term is really there: the plain load vector differs
    assert rel(Q.assemble_rhs(f), ref) > 1e-6
    # and the pair solves with the FD-preconditioned CG like the least-squares system
    s = gpu.pcg(A, gpu.FDPreconditioner(prob), rhs, gpu.PcgOptions(1e-8, 200))
    assert s.converged


def test_ultraweak_needs_final_condition_space(gpu):
    prob = gpu.SpaceTimeProblem.uniform(2, 3, 6, 5)
    Q = gpu.Quadrature(prob)
    f, u0 = _sinsin(2)
    with pytest.raises(gpu.InvalidArgument):
        Q.ultraweak(f, u0)
    # the C-ABI refuses as well (KS_EINVAL), whatever the caller
    import ctypes as C
    u0s = np.ones(int(np.prod(Q.nq[1:])), np.complex128)
    rhs = np.zeros(prob.N_dof, np.complex128)
    rc = gpu.lib().ks_quad_initial_term(Q._h, u0s.ctypes.data_as(C.c_void_p), gpu.KS_MEM_HOST,
                                        rhs.ctypes.data_as(C.c_void_p), gpu.KS_MEM_HOST)
    assert rc == gpu.KS_EINVAL
