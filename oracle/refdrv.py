"""ctypes wrapper over oracle/_ref/libkronschro_ref.so -- the reference's own
sources compiled unmodified (oracle/build_ref.sh). ORACLE TEST INFRASTRUCTURE
ONLY: used by tests/, tests/golden/make_golden.py and bench.py's CPU legs."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .oracle import REF_SO

_r = None


def available() -> bool:
    return os.path.exists(REF_SO)


def rlib():
    global _r
    if _r is None:
        L = C.CDLL(REF_SO)
        P, I, D = C.c_void_p, C.c_int, C.c_double
        L.ref_last_error.restype = C.c_char_p
        L.ref_problem_create.restype = P
        L.ref_problem_create.argtypes = [I, I, I, I, D, D, I, I]
        L.ref_problem_destroy.argtypes = [P]
        L.ref_dims.argtypes = [P, P]
        L.ref_time_bands.argtypes = [P, P, P, P]
        L.ref_space_bands.argtypes = [P, I, P, P, P, P]
        L.ref_eig.argtypes = [P, I, P, P]
        L.ref_composite_lambda.argtypes = [P, P]
        L.ref_fd_apply.restype = I
        L.ref_fd_apply.argtypes = [P, P, P]
        L.ref_kron_apply.argtypes = [P, P, P]
        L.ref_fd_block.restype = I
        L.ref_fd_block.argtypes = [P, C.c_long, P, P]
        L.ref_pcg.restype = I
        L.ref_pcg.argtypes = [P, P, D, I, I, I, P, C.POINTER(I), P, I, C.POINTER(I), C.POINTER(I),
                              C.POINTER(D)]
        L.ref_kron_to_dense.restype = I
        L.ref_kron_to_dense.argtypes = [P, P]
        L.ref_fd_to_dense.restype = I
        L.ref_fd_to_dense.argtypes = [P, P]
        L.ref_force_backend.restype = I
        L.ref_force_backend.argtypes = [C.c_char_p]
        L.ref_active_backend.restype = C.c_char_p
        L.ref_named_rhs.restype = I
        L.ref_named_rhs.argtypes = [P, C.c_char_p, P]
        L.ref_sinsin_rhs.restype = I
        L.ref_sinsin_rhs.argtypes = [P, P, P]
        L.ref_galerkin_apply.restype = I
        L.ref_galerkin_apply.argtypes = [P, P, P, I]
        L.ref_galerkin_kron_apply.restype = I
        L.ref_galerkin_kron_apply.argtypes = [P, P, P]
        L.ref_lift_named.restype = I
        L.ref_lift_named.argtypes = [P, C.c_char_p, P, P]
        L.ref_assemble_rhs_named.restype = I
        L.ref_assemble_rhs_named.argtypes = [P, C.c_char_p, P]
        L.ref_ultraweak_named.restype = I
        L.ref_ultraweak_named.argtypes = [P, C.c_char_p, P]
        L.ref_error_norms_named.restype = I
        L.ref_error_norms_named.argtypes = [P, C.c_char_p, P, C.POINTER(D), C.POINTER(D)]
        L.ref_infsup.restype = D
        L.ref_infsup.argtypes = [I, I, I, D, D]
        L.ref_extend.restype = I
        L.ref_extend.argtypes = [P, P, P, P]
        _r = L
    return _r


def _p(a):
    return C.c_void_p(a.ctypes.data)


def force_backend(name: str):
    """kernels::force_backend: 'scalar' makes the reference bit-comparable to the C restatement."""
    if rlib().ref_force_backend(name.encode()) != 0:
        raise ValueError(rlib().ref_last_error().decode())


def active_backend() -> str:
    return rlib().ref_active_backend().decode()


def infsup(method, p, n_el, T=1.0, nu=1.0):
    """infsup_constant (experiments.cpp:185-232); method "galerkin" | "ls"."""
    v = rlib().ref_infsup(0 if method == "galerkin" else 1, p, n_el, T, nu)
    if v < 0:
        raise RuntimeError(rlib().ref_last_error().decode())
    return v


class RefProblem:
    """SpaceTimeProblem::uniform + build_univariate + FDPreconditioner +
    assemble_system_operator, all from the reference's own code."""

    def __init__(self, d, p, n_el, n_el_t, T=1.0, nu=1.0, trial=0, with_fd=True):
        self.d, self.p, self.nu = d, p, nu
        self._h = rlib().ref_problem_create(d, p, n_el, n_el_t, T, nu, trial, int(with_fd))
        if not self._h:
            raise ValueError(rlib().ref_last_error().decode())
        dims = (C.c_int * (d + 1))()
        rlib().ref_dims(self._h, dims)
        self.dims = list(dims)
        self.N = int(np.prod(self.dims))

    def time_bands(self):
        nt, p = self.dims[0], self.p
        Lt = np.zeros((2 * p + 1) * nt)
        Mt = np.zeros((2 * p + 1) * nt)
        Wt = np.zeros((2 * p + 1) * nt, dtype=np.complex128)
        rlib().ref_time_bands(self._h, _p(Lt), _p(Mt), _p(Wt))
        return Lt, Mt, Wt

    def space_bands(self, l):
        n, p = self.dims[l + 1], self.p
        out = [np.zeros((2 * p + 1) * n) for _ in range(4)]
        rlib().ref_space_bands(self._h, l, *[_p(a) for a in out])
        return tuple(out)

    def eig(self, l):
        n = self.dims[l + 1]
        U, lam = np.zeros(n * n), np.zeros(n)
        rlib().ref_eig(self._h, l, _p(U), _p(lam))
        return U, lam

    def composite_lambda(self):
        out = np.zeros(int(np.prod(self.dims[1:])))
        rlib().ref_composite_lambda(self._h, _p(out))
        return out

    def fd_apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.complex128).ravel()
        z = np.empty_like(r)
        if rlib().ref_fd_apply(self._h, _p(r), _p(z)) != 0:
            raise RuntimeError("reference FD not constructed")
        return z

    def kron_apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.complex128).ravel()
        y = np.empty_like(x)
        rlib().ref_kron_apply(self._h, _p(x), _p(y))
        return y

    def galerkin_apply(self, r, adjoint=False):
        """galerkin_fast_solver(prob, u).solve / solve_adjoint (fdsolver.cpp:53-75,177-191)."""
        r = np.ascontiguousarray(r, dtype=np.complex128).ravel()
        z = np.empty_like(r)
        if rlib().ref_galerkin_apply(self._h, _p(r), _p(z), int(adjoint)):
            raise RuntimeError(rlib().ref_last_error().decode())
        return z

    def galerkin_kron_apply(self, x):
        """assemble_galerkin_operator(prob).apply (assembly.cpp:273-286)."""
        x = np.ascontiguousarray(x, dtype=np.complex128).ravel()
        y = np.empty_like(x)
        if rlib().ref_galerkin_kron_apply(self._h, _p(x), _p(y)):
            raise RuntimeError(rlib().ref_last_error().decode())
        return y

    def full_size(self):
        return int(np.prod([self.dims[0] + 1] + [n + 2 for n in self.dims[1:]]))

    def lift_named(self, name):
        """lift_nonhomogeneous (assembly.cpp:514-570): (corrected rhs, boundary coefficients)."""
        rhs = np.zeros(self.N, dtype=np.complex128)
        bnd = np.zeros(self.full_size(), dtype=np.complex128)
        if rlib().ref_lift_named(self._h, name.encode(), _p(rhs), _p(bnd)):
            raise ValueError(rlib().ref_last_error().decode())
        return rhs, bnd

    def assemble_rhs_named(self, name):
        rhs = np.zeros(self.N, dtype=np.complex128)
        if rlib().ref_assemble_rhs_named(self._h, name.encode(), _p(rhs)):
            raise ValueError(rlib().ref_last_error().decode())
        return rhs

    def ultraweak_named(self, name):
        """assemble_ultraweak (assembly.cpp:572-640): the load vector of f plus the
        initial-datum term i (u0, B(., 0)) for a named solution (u0 = u(0, .))."""
        rhs = np.zeros(self.N, dtype=np.complex128)
        if rlib().ref_ultraweak_named(self._h, name.encode(), _p(rhs)):
            raise ValueError(rlib().ref_last_error().decode())
        return rhs

    def error_norms_named(self, name, full):
        full = np.ascontiguousarray(full, dtype=np.complex128).ravel()
        l2, en = C.c_double(), C.c_double()
        if rlib().ref_error_norms_named(self._h, name.encode(), _p(full), C.byref(l2), C.byref(en)):
            raise ValueError(rlib().ref_last_error().decode())
        return l2.value, en.value

    def extend(self, reduced, boundary):
        out = np.zeros(self.full_size(), dtype=np.complex128)
        reduced = np.ascontiguousarray(reduced, dtype=np.complex128)
        boundary = np.ascontiguousarray(boundary, dtype=np.complex128)
        rlib().ref_extend(self._h, _p(reduced), _p(boundary), _p(out))
        return out

    def fd_block(self, i):
        nt, ld = self.dims[0], 3 * self.p + 1
        ab = np.zeros(nt * ld, dtype=np.complex128)
        piv = np.zeros(nt, dtype=np.int32)
        rc = rlib().ref_fd_block(self._h, int(i), _p(ab), _p(piv))
        if rc:
            raise RuntimeError(rlib().ref_last_error().decode())
        return ab, piv

    def pcg(self, b, tol=1e-8, maxit=200, strict=False, precond=True):
        b = np.ascontiguousarray(b, dtype=np.complex128).ravel()
        x = np.zeros_like(b)
        it, hl, fl = C.c_int(), C.c_int(), C.c_int()
        sec = C.c_double()
        hist = np.zeros(max(maxit, 1))
        rc = rlib().ref_pcg(self._h, _p(b), float(tol), int(maxit), int(strict), int(precond),
                            _p(x), C.byref(it), _p(hist), hist.size, C.byref(hl), C.byref(fl),
                            C.byref(sec))
        if rc:
            raise ValueError(rlib().ref_last_error().decode())
        return dict(x=x, iterations=it.value, res_history=list(hist[:hl.value]),
                    converged=bool(fl.value & 1), breakdown=bool(fl.value & 2),
                    seconds=sec.value)

    def kron_dense(self):
        out = np.zeros((self.N, self.N), dtype=np.complex128, order="F")
        if rlib().ref_kron_to_dense(self._h, _p(out)):
            raise OverflowError(rlib().ref_last_error().decode())
        return out

    def fd_dense(self):
        out = np.zeros((self.N, self.N), dtype=np.complex128, order="F")
        if rlib().ref_fd_to_dense(self._h, _p(out)):
            raise OverflowError(rlib().ref_last_error().decode())
        return out

    def sinsin_rhs(self, full_size):
        rhs = np.zeros(self.N, dtype=np.complex128)
        bnd = np.zeros(full_size, dtype=np.complex128)
        rlib().ref_sinsin_rhs(self._h, _p(rhs), _p(bnd))
        return rhs, bnd

    def named_rhs(self, name):
        rhs = np.zeros(self.N, dtype=np.complex128)
        if rlib().ref_named_rhs(self._h, name.encode(), _p(rhs)):
            raise ValueError(rlib().ref_last_error().decode())
        return rhs

    def __del__(self):
        if getattr(self, "_h", None):
            rlib().ref_problem_destroy(self._h)
            self._h = None
