"""Folded (even/odd) spatial transforms (csrc/ks_transform.cu k_mode_gemm_fold):
on uniform meshes the 1-D pencils are centro-symmetric, every eigenvector is
even or odd, and the FD apply runs two half-size GEMMs per transform. The
result must still match the oracle's dense transforms (reference
tensorops.cpp:125-156) within the north_star tolerance, forward and adjoint,
for even and odd axis lengths and every tile height (hc = ceil(n/2) up to 80)."""
import os

import numpy as np
import pytest

from helpers import setup_arrays, rel, maxrel

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _pair(ks, oracle, d, p, n_el, n_el_t, fold=True):
    a = setup_arrays(ks, d, p, n_el, n_el_t)
    old = os.environ.get("KS_FD_FOLD")
    os.environ["KS_FD_FOLD"] = "1" if fold else "0"
    try:
        g = ks.FDPreconditioner.from_arrays(a["dims"], a["nu"], a["p"], a["U"], a["lam"], a["Lt"],
                                            a["Mt"], a["Wt"])
    finally:
        if old is None:
            del os.environ["KS_FD_FOLD"]
        else:
            os.environ["KS_FD_FOLD"] = old
    o = oracle.OracleFD(a["dims"], a["nu"], a["p"], a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"])
    return a, g, o


# n = n_el for p = 2 (Dirichlet): even and odd lengths, tile heights 1..5
CASES = [(3, 2, 8, 8), (2, 2, 7, 6), (3, 2, 16, 8), (2, 2, 33, 5), (2, 2, 64, 9),
         (2, 2, 70, 4), (2, 2, 97, 3), (2, 2, 128, 3), (2, 2, 130, 2), (1, 2, 64, 64)]


@pytest.mark.parametrize("d,p,n_el,n_el_t", CASES)
def test_folded_fd_matches_oracle(gpu, oracle, d, p, n_el, n_el_t):
    a, g, o = _pair(gpu, oracle, d, p, n_el, n_el_t)
    assert g.info()["folded_axes"] == list(range(1, d + 1))
    r = oracle.random_vec(o.N, 99)
    z = g.apply(r)
    zo = o.apply(r)
    assert rel(z, zo) <= TOL and maxrel(z, zo) <= TOL
    za = g.apply_adjoint(r)
    zao = o.apply_adjoint(r)
    assert rel(za, zao) <= TOL and maxrel(za, zao) <= TOL


@pytest.mark.parametrize("d,p,n_el,n_el_t", [(3, 2, 16, 8), (2, 2, 64, 9)])
def test_folded_equals_dense_transform(gpu, oracle, d, p, n_el, n_el_t):
    """The fold symmetrises the eigenvectors; the difference to the dense GEMM
    path (KS_FD_FOLD=0) is rounding-level (measured ~1e-13 at n = 64)."""
    _, gf, o = _pair(gpu, oracle, d, p, n_el, n_el_t, fold=True)
    _, gd, _ = _pair(gpu, oracle, d, p, n_el, n_el_t, fold=False)
    assert gd.info()["folded_axes"] == []
    r = oracle.random_vec(o.N, 5)
    assert rel(gf.apply(r), gd.apply(r)) <= 1e-12


def test_non_symmetric_eigenvectors_stay_dense(gpu, oracle):
    """Perturbed eigenvectors (not even/odd) must not be folded."""
    a = setup_arrays(gpu, 2, 2, 10, 6)
    U = [np.array(u, dtype=np.float64).ravel().copy() for u in a["U"]]
    U[0][3] += 1e-3
    g = gpu.FDPreconditioner.from_arrays(a["dims"], a["nu"], a["p"], U, a["lam"], a["Lt"], a["Mt"], a["Wt"])
    assert g.info()["folded_axes"] == [2]
    o = oracle.OracleFD(a["dims"], a["nu"], a["p"], U, a["lam"], a["Lt"], a["Mt"], a["Wt"])
    r = oracle.random_vec(o.N, 3)
    assert rel(g.apply(r), o.apply(r)) <= TOL


def test_pair_mode_blocks_match_oracle(gpu, oracle):
    """d = 3 with identical axes 2, 3: fibers (i1, i2, i3) and (i1, i3, i2)
    share one factored block (pair mode); both must equal the oracle's
    factorisation of their own block (eigenvalue sums may differ by an ulp)."""
    a, g, o = _pair(gpu, oracle, 3, 2, 6, 5)
    n1, n2 = a["dims"][1], a["dims"][2]
    assert g.info()["blocks"] == n1 * n2 * (n2 + 1) // 2
    for (i1, i2, i3) in [(0, 1, 4), (0, 4, 1), (3, 2, 2), (5, 0, 5), (5, 5, 0)]:
        i = i1 + n1 * (i2 + n2 * i3)
        ab_g, piv_g = g.block(i, 2)
        ab_o, piv_o = o.block(i)
        assert np.array_equal(piv_g, piv_o)
        assert maxrel(ab_g, ab_o) < 1e-13


@pytest.mark.parametrize("d,p,n_el,n_el_t", [(2, 3, 64, 4), (2, 4, 128, 3), (2, 5, 128, 3), (2, 6, 128, 3),
                                             (3, 4, 30, 4), (2, 3, 40, 5)])
def test_folded_high_degree(gpu, oracle, d, p, n_el, n_el_t):
    """p >= 3: the outlier eigenpairs come in near-degenerate pairs whose computed
    eigenvectors mix even and odd; they are recombined into an even and an odd
    vector of the same pair (and near-clean columns symmetrised), so these axes
    fold too. Parity against the oracle's dense transforms at 1e-10."""
    a, g, o = _pair(gpu, oracle, d, p, n_el, n_el_t)
    assert g.info()["folded_axes"] == list(range(1, d + 1))
    r = oracle.random_vec(o.N, 11)
    z, zo = g.apply(r), o.apply(r)
    assert rel(z, zo) <= TOL and maxrel(z, zo) <= TOL
    za, zao = g.apply_adjoint(r), o.apply_adjoint(r)
    assert rel(za, zao) <= TOL and maxrel(za, zao) <= TOL


@pytest.mark.parametrize("d,p,n_el,n_el_t", [(3, 2, 16, 8), (3, 3, 13, 5), (3, 4, 11, 4)])
def test_axis1_time_major_handoff(gpu, oracle, d, p, n_el, n_el_t):
    """Pair mode hands the time-major layout over on axis 1 (forward axes d..1,
    rows stored by even/odd position, blocks numbered by position): forward
    and adjoint match the oracle, and ks_fd_block still answers by natural
    fiber index (the reference's LU of that fiber's block)."""
    a, g1, o = _pair(gpu, oracle, d, p, n_el, n_el_t)
    assert g1.info()["time_major_axis"] == 1
    r = oracle.random_vec(o.N, 17)
    for ap in ("apply", "apply_adjoint"):
        z1, zo = getattr(g1, ap)(r), getattr(o, ap)(r)
        assert rel(z1, zo) <= TOL and maxrel(z1, zo) <= TOL
    n1 = a["dims"][1]
    for i in (0, 1, n1 - 1, n1 + 3, o.N // a["dims"][0] - 1):
        ab, piv = g1.block(i, p)
        abo, pivo = o.block(i)
        assert np.array_equal(piv, pivo) and maxrel(ab, abo) < 1e-12


@pytest.mark.parametrize("d,p,n_el,n_el_t", [(3, 2, 16, 8), (3, 4, 11, 4), (2, 3, 16, 8), (2, 2, 12, 6),
                                            (1, 3, 16, 16), (3, 6, 6, 5)])
def test_ldl_blocks_match_reference_lu(gpu, oracle, d, p, n_el, n_el_t):
    """Least-squares blocks are HPD and factored as L D L^H without pivoting:
    the applications match the oracle's partial-pivot LU (the reference's
    factor_banded) at the north_star tolerance, forward and adjoint (H^H = H,
    one solve serves both)."""
    _, g, o = _pair(gpu, oracle, d, p, n_el, n_el_t)
    assert g.info()["no_pivot_solve"]
    r = oracle.random_vec(o.N, 29)
    z, zo = g.apply(r), o.apply(r)
    assert rel(z, zo) <= TOL and maxrel(z, zo) <= TOL
    za, zao = g.apply_adjoint(r), o.apply_adjoint(r)
    assert rel(za, zao) <= TOL and maxrel(za, zao) <= TOL


@pytest.mark.parametrize("d,p,n_el,n_el_t", [(3, 2, 16, 8), (3, 2, 64, 2), (3, 4, 11, 4), (3, 6, 6, 5), (2, 3, 12, 7),
                                            (2, 2, 64, 3), (1, 3, 32, 64), (1, 5, 9, 30), (2, 3, 63, 2)])
def test_fused_axis1_stage(gpu, oracle, d, p, n_el, n_el_t, monkeypatch):
    """Axis-1 transform + L D L^H block solves + inverse transform in one kernel
    per (t, i1) slab (csrc/ks_fdaxis1.cu; even and odd n1, pair mode, permutation
    dedup, d = 1): matches the oracle forward and adjoint, and the separate
    transform / solve / transform path (KS_FD_AXIS1=0) to rounding."""
    monkeypatch.setenv("KS_FD_AXIS1", "0")
    _, g0, o = _pair(gpu, oracle, d, p, n_el, n_el_t)
    monkeypatch.setenv("KS_FD_AXIS1", "1")
    _, g1, _ = _pair(gpu, oracle, d, p, n_el, n_el_t)
    assert g1.info()["fused_axis1"] and not g0.info()["fused_axis1"]
    r = oracle.random_vec(o.N, 53)
    for ap in ("apply", "apply_adjoint"):
        z1, zo, z0 = getattr(g1, ap)(r), getattr(o, ap)(r), getattr(g0, ap)(r)
        assert rel(z1, zo) <= TOL and maxrel(z1, zo) <= TOL
        assert rel(z1, z0) <= 1e-12


@pytest.mark.parametrize("d,p,n_el,n_el_t", [(3, 2, 16, 8), (3, 2, 64, 2), (3, 4, 11, 4), (3, 3, 13, 5), (3, 4, 128, 2),
                                            (3, 5, 9, 3)])
def test_position_ordered_transforms(gpu, oracle, d, p, n_el, n_el_t, monkeypatch):
    """Pair mode with every axis folded keeps the eigen rows of axes 2..d by
    position (csrc/ks_xform.cu, bulk-copy fed); the blocks are keyed by
    positions. Forward and adjoint match the oracle and the natural-order path
    (KS_FD_XFOLD=0); ks_fd_block still answers by natural fiber index."""
    monkeypatch.setenv("KS_FD_XFOLD", "0")
    a, g0, o = _pair(gpu, oracle, d, p, n_el, n_el_t)
    monkeypatch.setenv("KS_FD_XFOLD", "1")
    _, g1, _ = _pair(gpu, oracle, d, p, n_el, n_el_t)
    r = oracle.random_vec(o.N, 61)
    for ap in ("apply", "apply_adjoint"):
        z1, zo, z0 = getattr(g1, ap)(r), getattr(o, ap)(r), getattr(g0, ap)(r)
        assert rel(z1, zo) <= TOL and maxrel(z1, zo) <= TOL
        assert rel(z1, z0) <= 1e-12
    n1, n2 = a["dims"][1], a["dims"][2]
    for i in (0, 5, n1 * n2 + 3, o.N // a["dims"][0] - 1):
        ab, piv = g1.block(i, p)
        abo, pivo = o.block(i)
        assert np.array_equal(piv, pivo) and maxrel(ab, abo) < 1e-12
