"""CPU tests: the oracle restatement against the reference's own known-answer
properties (test_fdsolver.cpp, test_tensorops.cpp, test_krylov.cpp,
test_eigensolve.cpp), the host setup, and the MT19937-64 input generator.
No GPU needed."""
import numpy as np
import pytest

from helpers import setup_arrays, rel


def test_mt19937_64_known_answer(oracle):
    # C++ [rand.predef]: the 10000th consecutive invocation of a default-
    # constructed std::mt19937_64 (seed 5489) produces 9981545732273789042.
    v = oracle.random_vec(5000, seed=5489)
    flat = v.view(np.float64)
    u = (9981545732273789042 >> 11) * 2.0 ** -53
    assert flat[9999] == 2.0 * u - 1.0


def test_random_vec_range(oracle):
    v = oracle.random_vec(1000, seed=1234)
    assert np.all(np.abs(v.real) <= 1) and np.all(np.abs(v.imag) <= 1)
    assert abs(v.real.mean()) < 0.1


@pytest.mark.parametrize("d,n_el", [(1, 5), (2, 3)])
def test_oracle_fd_inverts_dense_preconditioner(ks, oracle, d, n_el):
    # test_fdsolver.cpp:51-69: ||P z - r|| <= 1e-10 ||r||, 20 trials
    a = setup_arrays(ks, d, 2, n_el, 4)
    fd = oracle.OracleFD(a["dims"], a["nu"], a["p"], a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"])
    P = oracle.fd_to_dense(a["dims"], a["nu"], a["p"], a["Lt"], a["Mt"], a["Wt"], a["M"], a["L"])
    assert np.max(np.abs(P - P.conj().T)) < 1e-11
    rng = np.random.default_rng(23)
    for _ in range(20):
        r = rng.standard_normal(fd.N) + 1j * rng.standard_normal(fd.N)
        z = fd.apply(r)
        assert np.linalg.norm(P @ z - r) <= 1e-10 * np.linalg.norm(r)


def test_oracle_fd_self_adjoint_positive(ks, oracle):
    # test_fdsolver.cpp:71-84
    a = setup_arrays(ks, 1, 3, 6, 6, T=2.0)
    fd = oracle.OracleFD(a["dims"], a["nu"], a["p"], a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"])
    rng = np.random.default_rng(5)
    for _ in range(5):
        u = rng.standard_normal(fd.N) + 1j * rng.standard_normal(fd.N)
        v = rng.standard_normal(fd.N) + 1j * rng.standard_normal(fd.N)
        x = np.vdot(v, fd.apply(u))
        y = np.vdot(u, fd.apply(v))
        assert abs(x - np.conj(y)) < 1e-11 * (1 + abs(x))
        q = np.vdot(u, fd.apply(u))
        assert abs(q.imag) < 1e-11 * q.real and q.real > 0


def test_oracle_fd_single_element(ks, oracle):
    # test_fdsolver.cpp:139-150: one spatial dof, two time dofs
    a = setup_arrays(ks, 1, 2, 1, 1)
    assert a["prob"].N_dof == 2
    fd = oracle.OracleFD(a["dims"], a["nu"], a["p"], a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"])
    P = oracle.fd_to_dense(a["dims"], a["nu"], a["p"], a["Lt"], a["Mt"], a["Wt"], a["M"], a["L"])
    r = np.array([1 + 2j, -0.5 + 0.25j])
    assert np.linalg.norm(P @ fd.apply(r) - r) < 1e-11


def test_oracle_kron_matches_dense_random_terms(oracle):
    # test_tensorops.cpp:113-132 (dims {3,4,2}, three terms incl. identities)
    rng = np.random.default_rng(42)

    def rb(n, bw):
        return rng.standard_normal((2 * bw + 1) * n) + 1j * rng.standard_normal((2 * bw + 1) * n)
    dims = [3, 4, 2]
    terms = [(1.5 - 0.5j, [rb(3, 1), rb(4, 2), rb(2, 0)], [1, 2, 0]),
             (2.0j, [None, rb(4, 1), None], [0, 1, 0]),
             (-1.0, [rb(3, 0), None, rb(2, 1)], [0, 0, 1])]
    K = oracle.OracleKron(dims, terms)
    Kd = oracle.kron_to_dense(dims, terms)
    x = rng.standard_normal(24) + 1j * rng.standard_normal(24)
    y = K.apply(x)
    yd = Kd @ x
    assert np.max(np.abs(y - yd)) <= 1e-12 * np.max(np.abs(yd))


def test_oracle_kron_axis0_fastest(oracle):
    # test_tensorops.cpp:134-142: dims (2,3) -> kron(J1, J0)
    rng = np.random.default_rng(1)
    j0 = rng.standard_normal(2 * 3) + 0j
    j1 = rng.standard_normal(3 * 5) + 0j
    terms = [(1.0, [j0, j1], [1, 2])]
    expect = np.kron(oracle.band_to_dense(j1, 3, 2), oracle.band_to_dense(j0, 2, 1))
    assert np.max(np.abs(oracle.kron_to_dense([2, 3], terms) - expect)) < 1e-13
    x = rng.standard_normal(6) + 1j * rng.standard_normal(6)
    assert np.max(np.abs(oracle.OracleKron([2, 3], terms).apply(x) - expect @ x)) < 1e-13


def test_oracle_system_operator_hermitian_pd(ks, oracle):
    # acceptance.cpp:251-257 (A Hermitian PD)
    a = setup_arrays(ks, 2, 2, 3, 3)
    terms = oracle.system_terms(a, 2, a["nu"])
    A = oracle.kron_to_dense(a["dims"], terms)
    assert np.max(np.abs(A - A.conj().T)) < 1e-10 * np.max(np.abs(A))
    assert np.min(np.linalg.eigvalsh(0.5 * (A + A.conj().T))) > 0


def test_oracle_banded_lu_vs_dense(oracle):
    # test_eigensolve.cpp:57-83
    import ctypes as C
    rng = np.random.default_rng(11)
    n, bw = 13, 2
    for _ in range(5):
        band = rng.standard_normal((2 * bw + 1) * n) + 1j * rng.standard_normal((2 * bw + 1) * n)
        H = oracle.band_to_dense(band, n, bw)
        ab = np.zeros((3 * bw + 1) * n, dtype=np.complex128)
        piv = np.zeros(n, dtype=np.int32)
        assert oracle.olib().ko_factor_banded(oracle._p(band), n, bw, oracle._p(ab), oracle._p(piv)) == 0
        b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        x = b.copy()
        oracle.olib().ko_solve_banded(oracle._p(ab), oracle._p(piv), n, bw, oracle._p(x))
        assert np.max(np.abs(x - np.linalg.solve(H, b))) < 1e-10
    # singular -> rejected (:85-88)
    z = np.zeros(3 * 4, dtype=np.complex128)
    ab = np.zeros(4 * 4, dtype=np.complex128)
    piv = np.zeros(4, dtype=np.int32)
    assert oracle.olib().ko_factor_banded(oracle._p(z), 4, 1, oracle._p(ab), oracle._p(piv)) == 2


def _hpd(rng, n):
    B = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    return B.conj().T @ B + np.eye(n)


def test_oracle_pcg_semantics(oracle):
    rng = np.random.default_rng(31)
    A = _hpd(rng, 12)
    # zero rhs (test_krylov.cpp:42-49)
    r = oracle.oracle_pcg(lambda x: A @ x, None, np.zeros(12))
    assert r["converged"] and r["iterations"] == 0
    # exact inverse -> one iteration (:51-63)
    b = rng.standard_normal(12) + 1j * rng.standard_normal(12)
    Ai = np.linalg.inv(A)
    r = oracle.oracle_pcg(lambda x: A @ x, lambda x: Ai @ x, b, tol=1e-10, maxit=50)
    assert r["converged"] and r["iterations"] == 1
    assert np.max(np.abs(r["x"] - np.linalg.solve(A, b))) < 1e-9
    # breakdown on an indefinite operator (:89-94)
    r = oracle.oracle_pcg(lambda x: -x, None, b[:5].copy())
    assert r["breakdown"] and not r["converged"]
    # strict residual (:96-103)
    A15 = _hpd(rng, 15)
    b15 = rng.standard_normal(15) + 1j * rng.standard_normal(15)
    r = oracle.oracle_pcg(lambda x: A15 @ x, None, b15, tol=1e-10, maxit=100, strict=True)
    assert r["converged"] and r["res_history"][-1] <= 1e-10
    with pytest.raises(ValueError):
        oracle.oracle_pcg(lambda x: x, None, b, tol=0.0)


def test_oracle_fd_pcg_beats_unpreconditioned(ks, oracle):
    # test_krylov.cpp:105-117: 1-D p=3 n_el=16 matched
    a = setup_arrays(ks, 1, 3, 16, 16)
    fd = oracle.OracleFD(a["dims"], a["nu"], a["p"], a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"])
    K = oracle.OracleKron(a["dims"], oracle.system_terms(a, 1, a["nu"]))
    b = oracle.random_vec(K.N, 7)
    w = oracle.oracle_pcg(K.apply, fd.apply, b, 1e-8, 300)
    wo = oracle.oracle_pcg(K.apply, None, b, 1e-8, 300)
    assert w["converged"] and w["iterations"] < 20
    assert wo["iterations"] > 2 * w["iterations"]


def test_host_setup_matches_definitions(ks):
    # partition of unity / symmetric matrices / eigenpairs: residual and M-orthonormality
    # (test_eigensolve.cpp:31-42 tolerances)
    a = setup_arrays(ks, 2, 3, 8, 8)
    from oracle.oracle import band_to_dense
    for l in range(2):
        n = a["dims"][l + 1]
        M = band_to_dense(a["M"][l], n, 3).real
        L = band_to_dense(a["L"][l], n, 3).real
        U = a["U"][l].reshape(n, n).T  # column-major
        lam = a["lam"][l]
        assert np.max(np.abs(L @ U - M @ U @ np.diag(lam))) < 1e-10 * max(1, np.max(np.abs(L)))
        assert np.max(np.abs(U.T @ M @ U - np.eye(n))) < 1e-12
        assert np.all(np.diff(lam) >= 0)
        G = band_to_dense(a["G"][l], n, 3).real
        # C^1 Dirichlet spaces: G = -L (test_assembly.cpp:39-48)
        assert np.max(np.abs(G + L)) < 1e-9 * np.max(np.abs(L))
    nt = a["dims"][0]
    Mt = band_to_dense(a["Mt"], nt, 3).real
    assert np.max(np.abs(Mt - Mt.T)) < 1e-15 and np.all(np.linalg.eigvalsh(Mt) > 0)


def test_host_setup_rejects_p1(ks):
    # spatial spaces must be C^1 with p_s >= 2 (assembly.cpp:103-107)
    with pytest.raises(ks.InvalidArgument):
        ks.SpaceTimeProblem.uniform(2, 1, 8, 8)
