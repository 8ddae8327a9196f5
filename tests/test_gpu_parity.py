"""GPU parity: libks.so (through the C-ABI) against the oracle restatement on
identical inputs. Tolerances (north_star): 1e-10 relative per FD application
and matvec; PCG iteration counts within +-1 at the same tolerance."""
import numpy as np
import pytest

from helpers import setup_arrays, rel, maxrel

pytestmark = pytest.mark.gpu

TOL = 1e-10  # per application, relative (BASELINE.json north_star)


def _fd_pair(ks, oracle, d, p, n_el, n_el_t, T=1.0, nu=1.0):
    a = setup_arrays(ks, d, p, n_el, n_el_t, T, nu)
    g = ks.FDPreconditioner.from_arrays(a["dims"], a["nu"], a["p"], a["U"], a["lam"], a["Lt"],
                                        a["Mt"], a["Wt"])
    o = oracle.OracleFD(a["dims"], a["nu"], a["p"], a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"])
    return a, g, o


CASES = [
    (1, 2, 5, 4), (2, 2, 3, 4), (1, 2, 1, 1),          # reference unit-test shapes
    (1, 3, 64, 64),                                     # config 1 (c1)
    (2, 3, 16, 16), (2, 4, 12, 10), (2, 5, 9, 9), (2, 6, 8, 8),
    (3, 2, 8, 8), (3, 3, 6, 7), (3, 4, 5, 5),
]


@pytest.mark.parametrize("d,p,n_el,n_el_t", CASES)
def test_fd_apply_matches_oracle(gpu, oracle, d, p, n_el, n_el_t):
    a, g, o = _fd_pair(gpu, oracle, d, p, n_el, n_el_t)
    r = oracle.random_vec(o.N, 1234)
    z_cpu = o.apply(r)
    z_gpu = g.apply(r)
    assert rel(z_gpu, z_cpu) <= TOL
    assert maxrel(z_gpu, z_cpu) <= TOL
    # composite eigenvalues identical (fdsolver.cpp:30-42)
    assert np.array_equal(g.eigenvalues(), o.eigenvalues())


@pytest.mark.parametrize("d,p,n_el,n_el_t", [(1, 2, 5, 4), (2, 2, 3, 4), (1, 3, 12, 12)])
def test_fd_apply_inverts_dense_preconditioner(gpu, oracle, d, p, n_el, n_el_t):
    # test_fdsolver.cpp:51-69 on the GPU path
    a, g, o = _fd_pair(gpu, oracle, d, p, n_el, n_el_t)
    P = oracle.fd_to_dense(a["dims"], a["nu"], a["p"], a["Lt"], a["Mt"], a["Wt"], a["M"], a["L"])
    rng = np.random.default_rng(23)
    for _ in range(10):
        r = rng.standard_normal(o.N) + 1j * rng.standard_normal(o.N)
        z = g.apply(r)
        assert np.linalg.norm(P @ z - r) <= 1e-10 * np.linalg.norm(r)


def test_fd_blocks_match_oracle_factorisation(gpu, oracle):
    # factor_banded on the device vs eigensolve.cpp:77-121 restated: same pivots
    a, g, o = _fd_pair(gpu, oracle, 2, 3, 10, 9)
    ns = int(np.prod(a["dims"][1:]))
    for i in [0, 1, ns // 2, ns - 1]:
        ab_g, piv_g = g.block(i, 3)
        ab_o, piv_o = o.block(i)
        assert np.array_equal(piv_g, piv_o)
        assert maxrel(ab_g, ab_o) < 1e-13


def test_fd_adjoint_matches_oracle(gpu, oracle):
    a, g, o = _fd_pair(gpu, oracle, 2, 3, 7, 6)
    r = oracle.random_vec(o.N, 99)
    assert rel(g.apply_adjoint(r), o.apply_adjoint(r)) <= TOL


def test_fd_linear_self_adjoint_positive(gpu, oracle):
    # test_fdsolver.cpp:71-84, :102-114
    a, g, o = _fd_pair(gpu, oracle, 1, 3, 6, 6, T=2.0)
    rng = np.random.default_rng(3)
    u = rng.standard_normal(o.N) + 1j * rng.standard_normal(o.N)
    v = rng.standard_normal(o.N) + 1j * rng.standard_normal(o.N)
    x, y = np.vdot(v, g.apply(u)), np.vdot(u, g.apply(v))
    assert abs(x - np.conj(y)) < 1e-11 * (1 + abs(x))
    q = np.vdot(u, g.apply(u))
    assert q.real > 0 and abs(q.imag) < 1e-11 * q.real
    al = 2.0 - 3.0j
    assert np.max(np.abs(g.apply(al * u) - al * g.apply(u))) < 1e-12 * np.max(np.abs(g.apply(u))) * 10


def test_fd_device_path_and_alias(gpu, oracle):
    a, g, o = _fd_pair(gpu, oracle, 2, 2, 9, 9)
    r = oracle.random_vec(o.N, 5)
    zh = g.apply(r)
    rd = gpu.DeviceVector.from_host(r)
    zd = g.apply(rd)
    assert np.array_equal(zd.to_host(), zh)
    g.apply(rd, rd)  # r and z alias (allowed, fdsolver apply copies first)
    assert np.array_equal(rd.to_host(), zh)


@pytest.mark.parametrize("d,p,n_el,n_el_t", [(1, 3, 64, 64), (2, 2, 6, 6), (2, 3, 12, 11),
                                             (3, 2, 5, 5), (3, 4, 4, 4)])
def test_system_matvec_matches_oracle(gpu, oracle, d, p, n_el, n_el_t):
    a = setup_arrays(gpu, d, p, n_el, n_el_t)
    A = gpu.assemble_system_operator(a["prob"])
    K = oracle.OracleKron(a["dims"], oracle.system_terms(a, d, a["nu"]))
    x = oracle.random_vec(K.N, 4321)
    y_cpu = K.apply(x)
    y_gpu = A.apply(x)
    assert rel(y_gpu, y_cpu) <= TOL
    assert maxrel(y_gpu, y_cpu) <= TOL
    info = A.plan_info()
    assert info["passes"] == d + 1


def test_kron_generic_terms_vs_dense(gpu, oracle):
    # test_tensorops.cpp:113-132 through the GPU path, incl. identities and complex factors
    rng = np.random.default_rng(42)

    def rb(n, bw):
        return rng.standard_normal((2 * bw + 1) * n) + 1j * rng.standard_normal((2 * bw + 1) * n)
    dims = [3, 4, 2]
    terms = [(1.5 - 0.5j, [rb(3, 1), rb(4, 2), rb(2, 0)], [1, 2, 0]),
             (2.0j, [None, rb(4, 1), None], [0, 1, 0]),
             (-1.0, [rb(3, 0), None, rb(2, 1)], [0, 0, 1])]
    K = gpu.KroneckerOperator(dims)
    for c, fs, bw in terms:
        K.add_term(c, [None if f is None else gpu.Banded(dims[k], bw[k], f) for k, f in enumerate(fs)])
    x = rng.standard_normal(24) + 1j * rng.standard_normal(24)
    yd = oracle.kron_to_dense(dims, terms) @ x
    assert np.max(np.abs(K.apply(x) - yd)) <= 1e-12 * np.max(np.abs(yd))
    # empty operator -> zero; identity-only term -> scaled copy
    E = gpu.KroneckerOperator(dims)
    assert np.all(E.apply(x) == 0)
    I = gpu.KroneckerOperator(dims)
    I.add_term(2.0 - 1.0j, [None, None, None])
    assert np.max(np.abs(I.apply(x) - (2.0 - 1.0j) * x)) < 1e-15 * 10


@pytest.mark.parametrize("d,p,n_el", [(1, 3, 16), (2, 2, 8), (2, 3, 10), (3, 2, 6)])
def test_pcg_matches_oracle(gpu, oracle, d, p, n_el):
    a = setup_arrays(gpu, d, p, n_el, n_el)
    A = gpu.assemble_system_operator(a["prob"])
    P = gpu.FDPreconditioner.from_arrays(a["dims"], a["nu"], a["p"], a["U"], a["lam"], a["Lt"],
                                         a["Mt"], a["Wt"])
    K = oracle.OracleKron(a["dims"], oracle.system_terms(a, d, a["nu"]))
    F = oracle.OracleFD(a["dims"], a["nu"], a["p"], a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"])
    b = oracle.random_vec(K.N, 1234)
    ro = oracle.oracle_pcg(K.apply, F.apply, b, 1e-8, 200)
    rg = gpu.pcg(A, P, b, gpu.PcgOptions(1e-8, 200))
    assert ro["converged"] and rg.converged and not rg.breakdown
    assert abs(rg.iterations - ro["iterations"]) <= 1
    assert rel(rg.x, ro["x"]) < 1e-7
    assert rg.res_history[-1] <= 1e-8


def test_pcg_edge_cases(gpu, oracle):
    a = setup_arrays(gpu, 1, 2, 8, 8)
    A = gpu.assemble_system_operator(a["prob"])
    P = gpu.FDPreconditioner.from_arrays(a["dims"], a["nu"], a["p"], a["U"], a["lam"], a["Lt"],
                                         a["Mt"], a["Wt"])
    n = A.vec_size()
    # b = 0 -> converged, 0 iterations (test_krylov.cpp:42-49)
    r = gpu.pcg(A, P, np.zeros(n))
    assert r.converged and r.iterations == 0 and np.all(r.x == 0)
    # breakdown on an indefinite operator (:89-94)
    neg = gpu.KroneckerOperator(a["dims"])
    neg.add_term(-1.0, [None, None])
    r = gpu.pcg(neg, None, oracle.random_vec(n, 3))
    assert r.breakdown and not r.converged
    # strict residual mode (:96-103) and unpreconditioned agreement with the oracle
    K = oracle.OracleKron(a["dims"], oracle.system_terms(a, 1, a["nu"]))
    b = oracle.random_vec(n, 8)
    rs = gpu.pcg(A, P, b, gpu.PcgOptions(1e-10, 100, True))
    assert rs.converged and rs.res_history[-1] <= 1e-10
    ru = gpu.pcg(A, None, b, gpu.PcgOptions(1e-8, 400))
    ro = oracle.oracle_pcg(K.apply, None, b, 1e-8, 400)
    assert abs(ru.iterations - ro["iterations"]) <= 1
    with pytest.raises(gpu.InvalidArgument):
        gpu.pcg(A, P, b, gpu.PcgOptions(0.0, 10))


def test_pcg_device_resident(gpu, oracle):
    a = setup_arrays(gpu, 2, 3, 10, 10)
    A = gpu.assemble_system_operator(a["prob"])
    P = gpu.FDPreconditioner(a["prob"])
    b = oracle.random_vec(A.vec_size(), 77)
    rh = gpu.pcg(A, P, b)
    rd = gpu.pcg(A, P, gpu.DeviceVector.from_host(b))
    assert rh.iterations == rd.iterations
    assert np.array_equal(rd.x.to_host(), rh.x)


def test_blas1_against_oracle(gpu, oracle):
    import ctypes as C
    L = gpu.lib()
    for n in [0, 1, 7, 1000, 100003]:
        x = oracle.random_vec(n, 1) if n else np.zeros(0, dtype=np.complex128)
        y = oracle.random_vec(n, 2) if n else np.zeros(0, dtype=np.complex128)
        xd, yd = gpu.DeviceVector.from_host(x), gpu.DeviceVector.from_host(y)
        out = gpu.ks_c64()
        gpu._check(L.ks_dotc(xd.ptr, yd.ptr, n, C.byref(out), None))
        ref = np.vdot(x, y)
        assert abs(complex(out.re, out.im) - ref) <= 1e-12 * (1 + abs(ref))
        s = C.c_double()
        gpu._check(L.ks_norm2sq(xd.ptr, n, C.byref(s), None))
        assert abs(s.value - np.vdot(x, x).real) <= 1e-12 * (1 + s.value)
        gpu._check(L.ks_axpy(gpu.ks_c64(0.5, -2.0), xd.ptr, yd.ptr, n, None))
        assert np.max(np.abs(yd.to_host() - (y + (0.5 - 2j) * x)), initial=0) < 1e-14
    # deterministic reductions: same bits twice
    x = oracle.random_vec(1 << 20, 5)
    xd = gpu.DeviceVector.from_host(x)
    vals = []
    for _ in range(3):
        s = C.c_double()
        gpu._check(L.ks_norm2sq(xd.ptr, x.size, C.byref(s), None))
        vals.append(s.value)
    assert vals[0] == vals[1] == vals[2]


def test_c3_full_size_properties(gpu, oracle):
    """Config 3 (d=3, p=2, n_el=64, 17M DOF) at full size: size-independent
    properties (linearity, Hermitian symmetry of P^-1 and A, A-P consistency)."""
    prob = gpu.SpaceTimeProblem.uniform(3, 2, 64, 64)
    P = gpu.FDPreconditioner(prob)
    A = gpu.assemble_system_operator(prob)
    n = prob.N_dof
    assert n == 65 * 64 ** 3
    u = gpu.DeviceVector.from_host(oracle.random_vec(n, 1))
    v = gpu.DeviceVector.from_host(oracle.random_vec(n, 2))
    Pu, Pv = P.apply(u).to_host(), P.apply(v).to_host()
    uh, vh = u.to_host(), v.to_host()
    x, y = np.vdot(vh, Pu), np.vdot(uh, Pv)
    assert abs(x - np.conj(y)) < 1e-10 * abs(x)
    Au, Av = A.apply(u).to_host(), A.apply(v).to_host()
    x, y = np.vdot(vh, Au), np.vdot(uh, Av)
    assert abs(x - np.conj(y)) < 1e-10 * abs(x)
    # P approximates A^-1 spectrally: <u, P A u> / <u,u> within the spectral-equivalence band
    PAu = P.apply(gpu.DeviceVector.from_host(Au)).to_host()
    ratio = np.vdot(uh, PAu).real / np.vdot(uh, uh).real
    assert 0.1 < ratio < 10


def test_pcg_graph_replay_matches_eager(gpu, oracle, monkeypatch):
    """Iteration phases replayed as CUDA graphs (KS_PCG_GRAPH=1) run the same
    kernels in the same order: identical iterates, counts and histories."""
    a = setup_arrays(gpu, 3, 2, 6, 5)
    b = oracle.random_vec(a["prob"].N_dof, 17)
    reps = []
    for g in ("0", "1"):
        monkeypatch.setenv("KS_PCG_GRAPH", g)
        A = gpu.assemble_system_operator(a["prob"])
        P = gpu.FDPreconditioner(a["prob"])
        reps.append(gpu.pcg(A, P, b, gpu.PcgOptions(1e-10, 100)))
    assert reps[0].iterations == reps[1].iterations and reps[0].converged and reps[1].converged
    assert np.array_equal(np.asarray(reps[0].x), np.asarray(reps[1].x))
    assert list(reps[0].res_history) == list(reps[1].res_history)


@pytest.mark.parametrize("strict,maxit", [(False, 100), (True, 100), (False, 3)])
def test_pcg_deferred_x_update_vs_oracle(gpu, oracle, strict, maxit):
    """x += alpha_k p_k is deferred into the p update: the solve still matches
    the oracle's pcg (krylov.cpp:24-114) -- also when it stops at maxit with
    the last update pending, and in strict mode (x needed every iteration)."""
    a = setup_arrays(gpu, 3, 2, 6, 5)
    b = oracle.random_vec(a["prob"].N_dof, 23)
    A = gpu.assemble_system_operator(a["prob"])
    P = gpu.FDPreconditioner(a["prob"])
    rep = gpu.pcg(A, P, b, gpu.PcgOptions(1e-10, maxit, strict))
    K = oracle.OracleKron(a["dims"], oracle.system_terms(a, 3, a["nu"]))
    F = oracle.OracleFD(a["dims"], a["nu"], a["p"], a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"])
    ro = oracle.oracle_pcg(K.apply, F.apply, b, 1e-10, maxit, strict)
    assert rep.converged == ro["converged"] == (maxit == 100)
    assert abs(rep.iterations - ro["iterations"]) <= 1
    if maxit == 3:
        assert rep.iterations == 3 and rel(rep.x, ro["x"]) < 1e-9
    else:
        assert rel(rep.x, ro["x"]) < 1e-8


def test_argument_checks(gpu, oracle):
    """Device vectors of the wrong length and malformed host outputs are
    rejected before any device access (std::invalid_argument in the reference,
    fdsolver.cpp:77-83, tensorops.cpp:256-262); a ks.Stream works on every path."""
    a = setup_arrays(gpu, 2, 2, 6, 5)
    P, A = gpu.FDPreconditioner(a["prob"]), gpu.assemble_system_operator(a["prob"])
    n = a["prob"].N_dof
    short = gpu.DeviceVector(n - 1)
    for op in (P, A):
        with pytest.raises(gpu.InvalidArgument):
            op.apply(short)
        with pytest.raises(gpu.InvalidArgument):
            op.apply(gpu.DeviceVector(n), gpu.DeviceVector(n + 3))
        with pytest.raises(gpu.InvalidArgument):
            op.apply(np.zeros(n, np.complex128), np.zeros(n, np.float64))
        with pytest.raises(gpu.InvalidArgument):
            op.apply(np.zeros(n, np.complex128), np.zeros(2 * n, np.complex128)[::2])
    with pytest.raises(gpu.InvalidArgument):
        gpu.pcg(A, P, short)
    r = oracle.random_vec(n, 3)
    st = gpu.Stream()
    rd = gpu.DeviceVector.from_host(r)
    zd = P.apply(rd, stream=st)
    yd = A.apply(rd, stream=st)
    st.synchronize()
    assert np.array_equal(zd.to_host(), P.apply(r)) and np.array_equal(yd.to_host(), A.apply(r))


@pytest.mark.parametrize("dedup", ["1", None])
def test_fd_d2_block_dedup_modes(gpu, oracle, monkeypatch, dedup):
    """d = 2 with identical axes: one block per fiber in layout order (default while the
    factors are small) and the deduplicated blocks of sorted multi-indices
    (KS_FD_DEDUP=1), both on the position-ordered plan, against the oracle."""
    if dedup:
        monkeypatch.setenv("KS_FD_DEDUP", dedup)
    monkeypatch.setenv("KS_FD_XFOLD", "1")   # the position-ordered plan at these small sizes too
    for p, n_el, n_el_t in [(3, 16, 16), (2, 90, 7), (4, 12, 10)]:   # (90 elements: axis 1 too long for the fused stage)
        a, g, o = _fd_pair(gpu, oracle, 2, p, n_el, n_el_t)
        n = a["dims"][1]
        fused = g.info()["fused_axis1"]   # (the fused axis-1 stage keeps one group of blocks per slab)
        assert g.info()["blocks"] == ((n + 1) // 2 * 2 * n if fused else n * (n + 1) // 2 if dedup else n * n)
        r = oracle.random_vec(o.N, 11)
        z = o.apply(r)
        assert rel(g.apply(r), z) <= TOL and maxrel(g.apply(r), z) <= TOL
        if g.info()["folded_axes"] == [1, 2]:   # (KS_FD_FOLD=0 runs have no position-ordered plan)
            assert g.info()["time_major_axis"] == 1 or g.info()["fused_axis1"]


@pytest.mark.parametrize("d,p,n_el,n_el_t", [(1, 2, 256, 6), (1, 3, 170, 5), (2, 2, 161, 3), (2, 3, 7, 4, )])
def test_long_axes_match_oracle(gpu, oracle, d, p, n_el, n_el_t):
    """Axes longer than 160 (SPEC's 1-D pencils go to 256 elements; the
    reference has no limit, tensorops.cpp:125-156) run the dense panel
    transform: FD apply (and, on the unmodified problems, the system matvec)
    against the oracle. The last case has one long and one short axis."""
    a = setup_arrays(gpu, d, p, n_el, n_el_t)
    dims, U, lam = list(a["dims"]), list(a["U"]), list(a["lam"])
    if d == 2 and n_el == 7:
        # mixed: axis 1 from a 200-element mesh, axis 2 short
        b = setup_arrays(gpu, 1, p, 200, n_el_t)
        dims = [a["dims"][0], b["dims"][1], a["dims"][2]]
        U, lam = [b["U"][0], a["U"][1]], [b["lam"][0], a["lam"][1]]
    g = gpu.FDPreconditioner.from_arrays(dims, a["nu"], a["p"], U, lam, a["Lt"], a["Mt"], a["Wt"])
    o = oracle.OracleFD(dims, a["nu"], a["p"], U, lam, a["Lt"], a["Mt"], a["Wt"])
    assert max(dims[1:]) > 160
    r = oracle.random_vec(o.N, 77)
    z_cpu, z_gpu = o.apply(r), g.apply(r)
    assert rel(z_gpu, z_cpu) <= TOL and maxrel(z_gpu, z_cpu) <= TOL
    if dims == list(a["dims"]):
        A = gpu.assemble_system_operator(a["prob"])
        K = oracle.OracleKron(a["dims"], oracle.system_terms(a, d, a["nu"]))
        y = K.apply(r)
        assert rel(A.apply(r), y) <= TOL


def test_host_apply_on_stream_waits_for_prior_stream_work(gpu, oracle):
    """A host-pointer apply queued on a user stream starts its H2D copy only
    after earlier work on that stream; pipelined applies on one handle keep
    their own results."""
    a = setup_arrays(gpu, 3, 2, 10, 6)
    P = gpu.FDPreconditioner(a["prob"])
    n = a["prob"].N_dof
    ins = [oracle.random_vec(n, 40 + k) for k in range(5)]
    want = [P.apply(v) for v in ins]
    st = gpu.Stream()
    outs = [np.empty(n, np.complex128) for _ in ins]
    for v, o in zip(ins, outs):
        P.apply(v, o, stream=st)
    st.synchronize()
    for o, w in zip(outs, want):
        assert np.array_equal(o, w)


@pytest.mark.skipif("__import__('paper_2311_18461_b200').device_count() < 2")
def test_handles_on_two_devices(gpu, oracle):
    """Kernels needing > 48 KB of dynamic shared memory opt in per device: a
    handle on device 1 works after one on device 0 in the same process."""
    a = setup_arrays(gpu, 3, 4, 8, 5)
    r = oracle.random_vec(a["prob"].N_dof, 9)
    z0 = gpu.FDPreconditioner(a["prob"], device=0).apply(r)
    z1 = gpu.FDPreconditioner(a["prob"], device=1).apply(r)
    assert rel(z1, z0) < 1e-14
