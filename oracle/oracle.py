"""CPU ORACLE loader (test infrastructure only -- never imported by the product).

Two checkers live under oracle/:
  * oracle/_build/libks_oracle.so -- the plain-C restatement (ks_oracle.c) of
    the reference hot path, built by build_oracle() with gcc;
  * oracle/_ref/libkronschro_ref.so -- the reference's OWN sources
    (/root/reference/proj/src/*.cpp, unmodified) compiled against the Eigen
    subset shim in oracle/eigen_shim by oracle/build_ref.sh, with the extern
    "C" driver oracle/ref_driver.cpp. Optional: present only where it was
    built (it travels to the GPU box as a prebuilt .so).

Also: dense numpy restatements of the reference's size-capped oracles
FDPreconditioner::to_dense (fdsolver.cpp:135-175) and
KroneckerOperator::to_dense (tensorops.cpp:277-301).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libks_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libkronschro_ref.so")


def build_oracle(force: bool = False) -> str:
    """gcc the C restatement (no -ffast-math, no FMA contraction: x86-64 baseline ISA)."""
    src = os.path.join(HERE, "ks_oracle.c")
    if force or not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(ORACLE_SO), exist_ok=True)
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared",
                               "-ffp-contract=off", src, "-o", ORACLE_SO, "-lm"])
    return ORACLE_SO


_o = None
_APPLY = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


def olib():
    global _o
    if _o is None:
        if not os.path.exists(ORACLE_SO):
            build_oracle()
        L = C.CDLL(ORACLE_SO)
        P, I, D, S = C.c_void_p, C.c_int, C.c_double, C.c_size_t
        L.ko_fd_create.restype = P
        L.ko_fd_create.argtypes = [I, P, D, I, P, P, P, P, P, C.POINTER(I)]
        L.ko_fd_create_galerkin.restype = P
        L.ko_fd_create_galerkin.argtypes = [I, P, D, I, P, P, P, P, C.POINTER(I)]
        L.ko_fd_apply.argtypes = [P, P, P]
        L.ko_fd_apply_adjoint.argtypes = [P, P, P]
        L.ko_fd_destroy.argtypes = [P]
        L.ko_fd_lambda.restype = P
        L.ko_fd_lambda.argtypes = [P]
        L.ko_fd_block_ab.restype = P
        L.ko_fd_block_ab.argtypes = [P, S]
        L.ko_fd_block_piv.restype = P
        L.ko_fd_block_piv.argtypes = [P, S]
        L.ko_kron_apply.argtypes = [I, P, I, P, P, P, P, P]
        L.ko_mode_product_dense.argtypes = [P, I, P, P, P, I, I]
        L.ko_mode_product_band.argtypes = [P, I, P, P, P, I, I]
        L.ko_factor_banded.restype = I
        L.ko_factor_banded.argtypes = [P, I, I, P, P]
        L.ko_solve_banded.argtypes = [P, P, I, I, P]
        L.ko_pcg.restype = I
        L.ko_pcg.argtypes = [_APPLY, P, _APPLY, P, P, S, D, I, I, P, C.POINTER(I), P, I,
                             C.POINTER(I), C.POINTER(I)]
        L.ko_random_vec.argtypes = [C.c_uint64, P, S]
        L.ko_dotc.argtypes = [P, P, S, C.POINTER(D), C.POINTER(D)]
        L.ko_norm2sq.restype = D
        L.ko_norm2sq.argtypes = [P, S]
        _o = L
    return _o


def _p(a):
    return C.c_void_p(a.ctypes.data)


def random_vec(n: int, seed: int = 1234) -> np.ndarray:
    """std::mt19937_64(seed), re = 2u-1 then im = 2u-1, u = (g()>>11)*2^-53."""
    v = np.empty(n, dtype=np.complex128)
    olib().ko_random_vec(seed, _p(v), n)
    return v


class OracleFD:
    """FDPreconditioner restated in C (fdsolver.cpp); takes the setup products.
    kind="galerkin": galerkin_fast_solver (fdsolver.cpp:177-191), blocks W + nu lam Mt."""

    def __init__(self, dims, nu, p, U, lam, Lt, Mt, Wt, kind="ls"):
        d = len(dims) - 1
        self.dims = list(dims)
        self.p = p
        self._keep = [np.ascontiguousarray(u, dtype=np.float64).ravel() for u in U]
        self._keep += [np.ascontiguousarray(v, dtype=np.float64).ravel() for v in lam]
        self._Lt = np.ascontiguousarray(Lt, dtype=np.float64).ravel()
        self._Mt = np.ascontiguousarray(Mt, dtype=np.float64).ravel()
        self._Wt = np.ascontiguousarray(Wt, dtype=np.complex128).ravel()
        up = (C.c_void_p * d)(*[a.ctypes.data for a in self._keep[:d]])
        lp = (C.c_void_p * d)(*[a.ctypes.data for a in self._keep[d:]])
        cd = (C.c_int * (d + 1))(*dims)
        st = C.c_int()
        if kind == "galerkin":
            self._h = olib().ko_fd_create_galerkin(d, cd, float(nu), int(p), up, lp, _p(self._Mt),
                                                   _p(self._Wt), C.byref(st))
        else:
            self._h = olib().ko_fd_create(d, cd, float(nu), int(p), up, lp, _p(self._Lt), _p(self._Mt),
                                          _p(self._Wt), C.byref(st))
        if st.value != 0:
            olib().ko_fd_destroy(self._h)
            self._h = None
            raise RuntimeError("factor_banded: numerically singular pivot")
        self.N = int(np.prod(dims))

    def apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.complex128).ravel()
        z = np.empty_like(r)
        olib().ko_fd_apply(self._h, _p(r), _p(z))
        return z

    def apply_adjoint(self, r):
        r = np.ascontiguousarray(r, dtype=np.complex128).ravel()
        z = np.empty_like(r)
        olib().ko_fd_apply_adjoint(self._h, _p(r), _p(z))
        return z

    def eigenvalues(self):
        ns = int(np.prod(self.dims[1:]))
        return np.ctypeslib.as_array(C.cast(olib().ko_fd_lambda(self._h),
                                            C.POINTER(C.c_double)), (ns,)).copy()

    def block(self, i):
        nt, ld = self.dims[0], 3 * self.p + 1
        ab = np.ctypeslib.as_array(C.cast(olib().ko_fd_block_ab(self._h, i),
                                          C.POINTER(C.c_double)), (2 * nt * ld,)).copy()
        piv = np.ctypeslib.as_array(C.cast(olib().ko_fd_block_piv(self._h, i),
                                           C.POINTER(C.c_int)), (nt,)).copy()
        return ab.view(np.complex128), piv

    def __del__(self):
        if getattr(self, "_h", None):
            olib().ko_fd_destroy(self._h)
            self._h = None


class OracleKron:
    """KroneckerOperator::apply restated in C (tensorops.cpp:236-254).
    terms: list of (coeff, [band ndarray or None], [bw])."""

    def __init__(self, dims, terms):
        self.dims = list(dims)
        D = len(dims)
        self.nterms = len(terms)
        self._coeffs = np.array([complex(c) for c, _, _ in terms] or [0j], dtype=np.complex128)
        self._bands = []
        ptrs, bws = [], []
        for c, fs, bw in terms:
            for k in range(D):
                if fs[k] is None:
                    ptrs.append(None)
                    bws.append(0)
                else:
                    b = np.ascontiguousarray(fs[k], dtype=np.complex128).ravel()
                    self._bands.append(b)
                    ptrs.append(b.ctypes.data)
                    bws.append(int(bw[k]))
        self._ptrs = (C.c_void_p * max(1, len(ptrs)))(*ptrs)
        self._bws = (C.c_int * max(1, len(bws)))(*bws)
        self._dims = (C.c_int * D)(*dims)
        self.N = int(np.prod(dims))

    def apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.complex128).ravel()
        y = np.empty_like(x)
        olib().ko_kron_apply(len(self.dims), self._dims, self.nterms, _p(self._coeffs), self._ptrs,
                             self._bws, _p(x), _p(y))
        return y


def oracle_pcg(apply_a, apply_p, b, tol=1e-8, maxit=200, strict=False):
    """pcg (krylov.cpp:24-114) restated in C; apply_* are python callables x->y."""
    b = np.ascontiguousarray(b, dtype=np.complex128).ravel()
    n = b.size

    def wrap(f):
        if f is None:
            return C.cast(None, _APPLY)

        def cb(ctx, xp, yp):
            x = np.ctypeslib.as_array(C.cast(xp, C.POINTER(C.c_double)), (2 * n,)).view(np.complex128)
            y = np.ctypeslib.as_array(C.cast(yp, C.POINTER(C.c_double)), (2 * n,)).view(np.complex128)
            y[:] = f(x.copy())
        return _APPLY(cb)

    fa, fp = wrap(apply_a), wrap(apply_p)
    x = np.zeros(n, dtype=np.complex128)
    it, hl, fl = C.c_int(), C.c_int(), C.c_int()
    hist = np.zeros(max(maxit, 1))
    rc = olib().ko_pcg(fa, None, fp, None, _p(b), n, float(tol), int(maxit), int(strict), _p(x),
                       C.byref(it), _p(hist), hist.size, C.byref(hl), C.byref(fl))
    if rc != 0:
        raise ValueError("pcg: bad options")
    return dict(x=x, iterations=it.value, res_history=list(hist[:hl.value]),
                converged=bool(fl.value & 1), breakdown=bool(fl.value & 2))


# ---------------- dense oracles (numpy restatements) -------------------------
def band_to_dense(band, n, bw):
    band = np.asarray(band).ravel()
    D = np.zeros((n, n), dtype=np.complex128)
    for j in range(n):
        for i in range(max(0, j - bw), min(n, j + bw + 1)):
            D[i, j] = band[bw + i - j + j * (2 * bw + 1)]
    return D


def kron_to_dense(dims, terms, cap=20000):
    """KroneckerOperator::to_dense (tensorops.cpp:277-301): kron(F_D, ..., F_0)."""
    n = int(np.prod(dims))
    if n > cap:
        raise OverflowError("KroneckerOperator::to_dense: size cap exceeded")
    A = np.zeros((n, n), dtype=np.complex128)
    for c, fs, bw in terms:
        acc = None
        for k in range(len(dims)):
            Fk = np.eye(dims[k], dtype=np.complex128) if fs[k] is None else band_to_dense(fs[k], dims[k], bw[k])
            acc = Fk if acc is None else np.kron(Fk, acc)
        A += c * acc
    return A


def fd_to_dense(dims, nu, p, Lt, Mt, Wt, Ms, Ls, cap=20000):
    """FDPreconditioner::to_dense (fdsolver.cpp:135-175):
    P = Ms x Lt + nu^2 (Ls Ms^-1 Ls) x Mt + nu Ls x (W + W^H), spatial kron axis 1 fastest.
    Ms, Ls: per-axis real bands (bw p)."""
    n = int(np.prod(dims))
    if n > cap:
        raise OverflowError("FDPreconditioner::to_dense: size cap exceeded")
    d = len(dims) - 1
    M = [band_to_dense(Ms[l], dims[l + 1], p).real for l in range(d)]
    L = [band_to_dense(Ls[l], dims[l + 1], p).real for l in range(d)]

    def spatial(J):
        acc = J[0]
        for l in range(1, d):
            acc = np.kron(J[l], acc)
        return acc
    Msd = spatial(M)
    Lsd = np.zeros_like(Msd)
    for l in range(d):
        J = list(M)
        J[l] = L[l]
        Lsd += spatial(J)
    Bhat = Lsd @ np.linalg.solve(Msd, Lsd)
    nt = dims[0]
    Ltd = band_to_dense(Lt, nt, p).real
    Mtd = band_to_dense(Mt, nt, p).real
    W = band_to_dense(Wt, nt, p)
    Wsym = W + W.conj().T
    return np.kron(Msd, Ltd) + nu * nu * np.kron(Bhat, Mtd) + nu * np.kron(Lsd, Wsym)


def system_terms(prob_bands, d, nu):
    """assemble_system (assembly.cpp:202-251), restricted branch, as an oracle term list.
    prob_bands: dict with Lt, Mt, Wt (time, bw p) and per-axis M, L, G, V (bw p) and p, dims."""
    p = prob_bands["p"]
    dims = prob_bands["dims"]
    nt = dims[0]
    Lt = np.asarray(prob_bands["Lt"], dtype=np.complex128)
    Mt = np.asarray(prob_bands["Mt"], dtype=np.complex128)
    W = band_to_dense(prob_bands["Wt"], nt, p)
    Wsym_d = W + W.conj().T
    Wsym = np.zeros((2 * p + 1) * nt, dtype=np.complex128)
    for j in range(nt):
        for i in range(max(0, j - p), min(nt, j + p + 1)):
            Wsym[p + i - j + j * (2 * p + 1)] = Wsym_d[i, j]

    def tr(b, n):
        D = band_to_dense(b, n, p).T
        out = np.zeros((2 * p + 1) * n, dtype=np.complex128)
        for j in range(n):
            for i in range(max(0, j - p), min(n, j + p + 1)):
                out[p + i - j + j * (2 * p + 1)] = D[i, j]
        return out
    M = [np.asarray(b, dtype=np.complex128) for b in prob_bands["M"]]
    L = [np.asarray(b, dtype=np.complex128) for b in prob_bands["L"]]
    G = [np.asarray(b, dtype=np.complex128) for b in prob_bands["G"]]
    V = [np.asarray(b, dtype=np.complex128) for b in prob_bands["V"]]
    Gt = [tr(G[l], dims[l + 1]) for l in range(d)]
    bw = [p] * (d + 1)
    terms = []

    def wm(tf):
        return [tf] + [M[l] for l in range(d)]
    terms.append((1.0, wm(Lt), bw))
    for l in range(d):
        f = wm(Mt)
        f[l + 1] = V[l]
        terms.append((nu * nu, f, bw))
    for l in range(d):
        for m in range(d):
            if l == m:
                continue
            f = wm(Mt)
            f[l + 1] = G[l]
            f[m + 1] = Gt[m]
            terms.append((nu * nu, f, bw))
    for l in range(d):
        f = wm(Wsym)
        f[l + 1] = L[l]
        terms.append((nu, f, bw))
    return terms


def galerkin_terms(prob_bands, d, nu):
    """assemble_galerkin_operator (assembly.cpp:273-286) as an oracle term list:
    1 (W x M_1 x .. x M_d) - nu sum_l (M_t x .. G_l^T on axis l ..)."""
    p = prob_bands["p"]
    dims = prob_bands["dims"]
    Mt = np.asarray(prob_bands["Mt"], dtype=np.complex128)
    W = np.asarray(prob_bands["Wt"], dtype=np.complex128)

    def tr(b, n):
        D = band_to_dense(b, n, p).T
        out = np.zeros((2 * p + 1) * n, dtype=np.complex128)
        for j in range(n):
            for i in range(max(0, j - p), min(n, j + p + 1)):
                out[p + i - j + j * (2 * p + 1)] = D[i, j]
        return out
    M = [np.asarray(b, dtype=np.complex128) for b in prob_bands["M"]]
    G = [np.asarray(b, dtype=np.complex128) for b in prob_bands["G"]]
    bw = [p] * (d + 1)
    terms = [(1.0, [W] + [M[l] for l in range(d)], bw)]
    for l in range(d):
        f = [Mt] + [M[m] for m in range(d)]
        f[l + 1] = tr(G[l], dims[l + 1])
        terms.append((-nu, f, bw))
    return terms
